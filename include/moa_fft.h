/*
 * moa_fft.h -- C-ABI of the B200-native lifted FFT (libmoafft.so).
 *
 * The operation (PAPER.md, Mullin & Raynolds "Conformal Computing"):
 * Van Loan's problem statement, "Input: x in C^n and n = 2^t, where t >= 0 is
 * an integer.  Output: The FFT of x" (Fig. vanloan_fft), computed
 * by dimension lifting: the vector is reshaped to a higher-rank array so that
 * each block fits one level of the memory/processor hierarchy, and every pass
 * is a reshape-transpose (Eq. reshape3), a block butterfly
 * and a twiddle multiply with the transformed weights
 * w_L^{sigma + j c^l}; the data is restored to natural order by
 * the final transpose.  The lifting extends to the processor
 * level.
 *
 * Semantics fixed by BASELINE.json: forward, unnormalised,
 *     out[b*n + k] = sum_{j<n} in[b*n + j] * exp(-2 pi i j k / n),
 * natural order in and out; for the 3-D plan the separable triple sum over a
 * row-major [n0][n1][n2] array.  Elements are interleaved {re, im}:
 * MOA_C64 = 2 x float32, MOA_C128 = 2 x float64.
 *
 * Conventions for every entry point:
 *   - Return MOA_OK or an error code; a message is available from
 *     moa_fft_last_error() (thread-local).  Nothing is clamped silently.
 *   - Argument checks run before any allocation or CUDA call.
 *   - Device pointers belong to the device current when the plan was created.
 *   - Plans own their scratch, twiddle tables and (ngpu > 1) communicator; the
 *     caller owns in/out.  A plan is not re-entrant: serialise exec calls on one
 *     plan.  Different plans are independent.  Results are bitwise
 *     deterministic for a fixed plan (no atomics).
 */
#ifndef MOA_FFT_H
#define MOA_FFT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MOA_OK = 0,
    MOA_EINVAL = 1,       /* invalid argument (size, dtype, pointer, alignment) */
    MOA_ENOMEM = 2,       /* device or host allocation failed */
    MOA_ECUDA = 3,        /* a CUDA runtime call or kernel launch failed */
    MOA_ENCCL = 4,        /* an NCCL call failed (the communicator is aborted) */
    MOA_EUNSUPPORTED = 5  /* valid request this build does not implement */
} moa_status_t;

typedef enum { MOA_C64 = 0, MOA_C128 = 1 } moa_dtype_t;

typedef struct moa_fft_plan_s *moa_fft_plan_t; /* opaque, library-owned */

#define MOA_MAX_DIGITS 6
#define MOA_MAX_PASSES 36

/*
 * moa_fft_plan -- plan `batch` independent forward transforms of length n.
 *   n      : transform length, a power of two, n >= 1 (t >= 0; n = 1 is
 *            the identity).  Otherwise MOA_EINVAL.
 *   batch  : number of contiguous rows (row b at element offset b*n), >= 1.
 *   dtype  : MOA_C64 or MOA_C128.
 *   ngpu   : processors the single transform is partitioned over, in {1,2,4,8}.
 *            ngpu > 1 requires moa_fft_dist_init() first, batch == 1 and
 *            n >= ngpu^2 (else MOA_EUNSUPPORTED).  Rank g then passes its block
 *            in = x[g n/p, (g+1) n/p) and receives out = X[g n/p, (g+1) n/p).
 * The lifting n = R_0 R_1 ... is chosen by the planner; the environment
 * variable MOA_FFT_LIFT="r0,r1,..." overrides it (the paper's run-time blocking
 * size c; for ablations).  A two-pass lifting of rows that spread
 * over <= 8 small CTAs runs as one cluster pair where that measured faster
 * (2^13 / 2^14-point complex128 rows, or any batch of <= 32 MiB): ring = 3 / 4
 * below, the intermediate in distributed shared memory, one launch;
 * MOA_FFT_CLUSTER=0 disables it, =1 allows any cluster of <= 16 CTAs.
 * Allocates device scratch (one buffer of the local data size, only when the
 * lifting has more than one launch that needs it) and the twiddle tables on
 * the current device.
 */
moa_status_t moa_fft_plan(moa_fft_plan_t *plan, int64_t n, int64_t batch, moa_dtype_t dtype, int ngpu);

/* moa_fft_plan_lift -- as moa_fft_plan(ngpu = 1) with an explicit lifting:
 * radices[0..nrad) are powers of two whose product is n (each <= 4096). */
moa_status_t moa_fft_plan_lift(moa_fft_plan_t *plan, int64_t n, int64_t batch, moa_dtype_t dtype,
                               const int64_t *radices, int nrad);

/*
 * moa_fft_plan_3d -- the separable 3-D forward DFT of a row-major
 * [n0][n1][n2] array (multi-dimensional FFT as 1-D FFTs along each axis,
 * PAPER.md P:641 footnote).  Each n_i a power of two, 2 <= n_i <= 4096.
 * ngpu > 1: slab decomposition; rank g passes x-slab planes
 * j0 in [g n0/p, (g+1) n0/p) (row-major [j0_loc][j1][j2]) and receives the
 * y-slab k1 in [g n1/p, (g+1) n1/p) (row-major [k0][k1_loc][k2]).
 */
moa_status_t moa_fft_plan_3d(moa_fft_plan_t *plan, int64_t n0, int64_t n1, int64_t n2, moa_dtype_t dtype,
                             int ngpu);

/*
 * Plan flags (the paper's variants):
 *   MOA_FFT_INVERSE      kernel e^{+2 pi i jk/n} -- the sign of the fftpsirad2
 *                        fragment's weight EXP(+2 pi i row/L) (reading R1).
 *   MOA_FFT_NORMALIZE    multiply the result by 1/N (N = n, or n0 n1 n2; exact,
 *                        N is a power of two).  With INVERSE this is the inverse DFT.
 *   MOA_FFT_LIFTED_ORDER 1-D only: leave X in the lifting's own order instead of
 *                        applying the final transpose -- the paper's "far more
 *                        efficient approach in which no data needs to be moved"
 *                        (P:2983-2984).  Where X[k] lands is given by
 *                        moa_fft_output_index().  On one GPU the last pass then
 *                        stores in place (its own load positions); with ngpu > 1
 *                        the third all-to-all and the unpack are skipped and rank g
 *                        holds X[g + p k2] at offset k2 (the rank is the fastest
 *                        output digit).  A plan may keep natural order (identity
 *                        map) where that costs nothing extra (single-pass plans).
 * Unknown bits -> MOA_EINVAL; LIFTED_ORDER, UNBLOCKED or HYPERCUBE on a 3-D plan,
 * UNBLOCKED / HYPERCUBE with ngpu > 1, with LIFTED_ORDER or with each other ->
 * MOA_EUNSUPPORTED.
 */
#define MOA_FFT_INVERSE 1u
#define MOA_FFT_NORMALIZE 2u
#define MOA_FFT_LIFTED_ORDER 4u
/* MOA_FFT_UNBLOCKED (1-D, ngpu = 1; an ablation): the paper's unblocked control
 * ("c >= n disables blocking"), i.e. Van Loan's program as
 * written (Fig. vanloan_fft): x <- P_n x, then for q = 1..t one
 * global radix-2 stage per pass (t + 1 HBM round trips instead of the
 * lifting's few).  Combines with INVERSE / NORMALIZE, not with LIFTED_ORDER. */
#define MOA_FFT_UNBLOCKED 8u
/* MOA_FFT_HYPERCUBE (1-D, ngpu = 1; an ablation, SURVEY §8(f) f3 iii): the
 * paper's hypercube formulation of the unblocked radix-2 FFT with the stage
 * transposes t_j of Ch.5 (Eq. tvec; Fig. tvectab)
 * realised physically: stage s reads its butterfly pairs along the top axis of
 * the hypercube view, (i, i + n/2) for every i < n/2 -- the same one-loop
 * control structure at every stage, the "simpler control structure" the paper
 * conjectures faster -- and stores through the transposition that
 * brings the next stage's axis to the top (out[(i >> s) 2^{s+1} + (i mod 2^s)
 * + r 2^s], r = 0, 1; weights w_{2^{s+1}}^{i mod 2^s}).  No input bit reversal
 * (the transposes sort the output); t HBM round trips, ping-ponging between
 * out and a plan-owned buffer.  Combines with INVERSE / NORMALIZE only. */
#define MOA_FFT_HYPERCUBE 16u

/* moa_fft_plan / moa_fft_plan_3d with flags (0 = the forward, natural-order plan). */
moa_status_t moa_fft_plan_ex(moa_fft_plan_t *plan, int64_t n, int64_t batch, moa_dtype_t dtype, int ngpu,
                             uint32_t flags);
moa_status_t moa_fft_plan_3d_ex(moa_fft_plan_t *plan, int64_t n0, int64_t n1, int64_t n2, moa_dtype_t dtype,
                                int ngpu, uint32_t flags);

/*
 * moa_fft_output_index -- where a 1-D plan stores each output: pos[k] (k < n)
 * is the element offset of X[k] within the row (ngpu = 1; row b adds b*n), or
 * the global offset g*(n/p) + local offset (ngpu > 1: rank g's out block).
 * Natural order gives pos[k] = k.  `count` must equal n.  Host only.
 */
moa_status_t moa_fft_output_index(moa_fft_plan_t plan, int64_t *pos, int64_t count);

/*
 * moa_fft_exec -- run the plan on device buffers, stream-ordered on `stream`
 * (a cudaStream_t of the plan's device; NULL = legacy default stream).
 *   in  : device pointer, `local elements` complex values (n*batch at ngpu=1),
 *         16-byte aligned.  Not modified unless in == out.
 *   out : device pointer, same size, 16-byte aligned; in == out is allowed
 *         (plans whose first pass stores elsewhere than it loads -- the
 *         rotating 3-D layouts, the unblocked control's bit reversal -- then
 *         copy the input once into a plan-owned buffer, allocated on first use).
 * Returns without a host synchronisation; buffers must stay valid until the
 * stream passes the exec.  NULL or misaligned pointers -> MOA_EINVAL.
 */
moa_status_t moa_fft_exec(moa_fft_plan_t plan, const void *in, void *out, void *stream);

/*
 * moa_fft_exec_host -- end-to-end variant for HOST buffers: copies host_in to
 * a plan-owned device buffer, executes, copies the result to host_out, and
 * synchronises `stream` before returning.  host_in / host_out should be pinned
 * (cudaHostAlloc / cudaHostRegister) for full copy bandwidth; pageable memory
 * works but is slower.  host_in == host_out is allowed.
 */
moa_status_t moa_fft_exec_host(moa_fft_plan_t plan, const void *host_in, void *host_out, void *stream);

/* moa_fft_destroy -- release every resource of the plan (NULL is a no-op). */
moa_status_t moa_fft_destroy(moa_fft_plan_t plan);

/* Thread-local message describing the last error returned on this thread. */
const char *moa_fft_last_error(void);

/* Local element count of a plan (elements this rank passes to exec). */
int64_t moa_fft_local_elems(moa_fft_plan_t plan);

/* Number of kernel launches one exec issues (for launch accounting). */
int moa_fft_launches_per_exec(moa_fft_plan_t plan);

/*
 * Per-pass timing with CUDA events on the exec stream (no host sync inside
 * exec).  moa_fft_prof_begin arms the plan for up to max_execs execs: each
 * exec records an event before every step (pass or all-to-all) and one after
 * the last.  moa_fft_prof_end synchronises on the recorded events, writes the
 * summed milliseconds of step i over all recorded execs to step_ms[i]
 * (i < nsteps <= max_steps) and the number of execs to *execs, and disarms.
 */
moa_status_t moa_fft_prof_begin(moa_fft_plan_t plan, int max_execs);
moa_status_t moa_fft_prof_end(moa_fft_plan_t plan, double *step_ms, int max_steps, int *nsteps, int *execs);

/*
 * Processor-level lifting (ngpu > 1; SPMD, one process per GPU).
 *   moa_fft_get_unique_id : rank 0 creates the 128-byte NCCL unique id; the
 *                           caller broadcasts it (e.g. torch.distributed).
 *   moa_fft_dist_init     : every rank, with the same id, before planning with
 *                           ngpu > 1; binds the communicator to the current device.
 *   moa_fft_dist_finalize : destroy the communicator.
 * libnccl is bound at the first of these calls: $MOA_NCCL_LIB, else a libnccl
 * the process already holds, else the loader's search path; the exchanges use
 * ncclAlltoAll where the library has it (NCCL >= 2.28), else one ncclSend +
 * ncclRecv per peer in a group.  MOA_ENCCL if no usable library is found.
 */
moa_status_t moa_fft_get_unique_id(uint8_t id[128]);
moa_status_t moa_fft_dist_init(int rank, int ngpu, const uint8_t id[128]);
moa_status_t moa_fft_dist_finalize(void);

/*
 * Loopback (one GPU, for tests): moa_fft_dist_loopback(rank, ngpu) makes the
 * next ngpu > 1 plans on this thread belong to virtual rank `rank` (no
 * communicator).  moa_fft_exec_loopback runs the ngpu plans (one per virtual
 * rank, all on the current device) in lock step: the same kernels and chunk
 * maps as the NCCL path, with every all-to-all done as device-to-device
 * copies.  ins[r] / outs[r] are rank r's device buffers.
 */
moa_status_t moa_fft_dist_loopback(int rank, int ngpu);
moa_status_t moa_fft_exec_loopback(moa_fft_plan_t *plans, int ngpu, const void *const *ins, void *const *outs,
                                   void *stream);

/*
 * The distributed schedule of one rank (host only): passes[] as below; steps
 * i < nsteps are kinds[i] = 0 (run passes[srcs[i]]), 1 (all-to-all of
 * counts[i] complex elements per peer from buffer srcs[i] to dsts[i]; buffer
 * ids 0 in, 1 out, 2 scratch, 3 scratch2), 2 (run passes[srcs[i]] with the
 * following all-to-all fused into its stores: send-layout chunk h goes straight
 * to rank h's buffer dsts[i] at offset rank * counts[i], over NVLink) or
 * 3 (barrier).  Fusion is on unless MOA_FFT_PEER=0.  is3d = 0: n0 is the 1-D length.
 * flags: MOA_FFT_LIFTED_ORDER selects the 1-D schedule without the third
 * all-to-all and the unpack (other bits do not change the schedule).
 */
moa_status_t moa_dist_describe(int rank, int ngpu, int is3d, int64_t n0, int64_t n1, int64_t n2, moa_dtype_t dtype,
                               void *passes /* moa_pass_desc_t[max_passes] */, int max_passes, int *npasses,
                               int32_t *kinds, int32_t *srcs, int32_t *dsts, int64_t *counts, int max_steps,
                               int *nsteps, uint32_t flags);

/*
 * psi-index layer introspection (host only, no GPU needed).
 *
 * One pass = an ONF: for every line
 * (digits d_0..d_{ndig-1}, d_i < ext[i], d_0 fastest) and every point k < R:
 *   load  address = sum_i d_i*in_str[i]  + k*in_kstr    (elements)
 *   store address = sum_i d_i*out_str[i] + k*out_kstr
 *   the R-point DFT output k is multiplied by
 *       w_{twN}^{(k * (tw_off + sum_i d_i*tw_str[i])) mod twN}   (twN <= 1: no twiddle)
 *   and, when out_ksplit < logR, the store address of k is
 *       sum_i d_i*out_str[i] + (k mod 2^out_ksplit)*out_kstr + (k >> out_ksplit)*out_kstr_hi.
 * Consecutive lines of a tile (W of them) run along digit 0.
 */
typedef struct {
    int32_t logR;               /* R = 2^logR points per line */
    int32_t ndig;               /* number of line digits */
    int64_t ext[MOA_MAX_DIGITS];
    int64_t in_str[MOA_MAX_DIGITS];
    int64_t out_str[MOA_MAX_DIGITS];
    int64_t tw_str[MOA_MAX_DIGITS];
    int64_t in_kstr, out_kstr;
    int64_t twN;                /* twiddle root, power of two, or 1 */
    int64_t tw_off;             /* added to the line's exponent base (rank offset; 0 on one GPU) */
    int32_t out_ksplit;         /* store: k = khi*2^out_ksplit + klo, address += klo*out_kstr + khi*out_kstr_hi */
    int64_t out_kstr_hi;
    int32_t kind;               /* 0: lifted DFT pass (the ONF above); 1: identity (a pure data-
                                 * movement pass); 2: one global radix-2 stage of the unblocked
                                 * control (Van Loan, L = 2 in_kstr, in place); 3: the bit
                                 * reversal P_n of every row (MOA_FFT_UNBLOCKED plans) */
    int32_t lf_load, lf_store;  /* 1: that side is coalesced along the lines (digit 0) */
    int32_t W;                  /* lines per CTA tile */
    int32_t threads;            /* CTA size */
    int32_t smem_bytes;         /* dynamic shared memory per CTA */
    int32_t line_pad;           /* smem line stride = R + line_pad elements */
    int32_t src, dst;           /* buffer ids: 0 = in, 1 = out, 2 = scratch, 3 = scratch2 */
    /* L2-staged pass pair (the lifting at the L2 level): ring = 2 marks pass A,
     * whose output goes to a ring of ring_slots group buffers of ring_G
     * elements; ring = 1 marks the following pass B, which reads it back.  The
     * last line digit is the group; its stride on the ring side is replaced by
     * (group mod ring_slots) * ring_G.  ring_lag: groups between A and B in the
     * tile order.  ring_discard: B drops the consumed lines from L2 (no write-back).
     * Cluster pair (the lifting at the thread-block-cluster level): ring = 3
     * marks pass A, ring = 4 the following pass B; one launch, a cluster of
     * ring_slots CTAs per group of ring_G elements, the intermediate in the
     * cluster's distributed shared memory (never in HBM or the L2); ring_lag
     * holds the buffer id the intermediate had in the plain two-pass form. */
    int32_t ring, ring_slots, ring_lag, ring_discard;
    int64_t ring_groups, ring_G;
} moa_pass_desc_t;

/* ONF descriptors of a 1-D lifting (radices == NULL: the planner's choice). */
moa_status_t moa_psi_describe(int64_t n, int64_t batch, moa_dtype_t dtype, const int64_t *radices, int nrad,
                              moa_pass_desc_t *out, int max_passes, int *npasses);
/* ONF descriptors of the 3-D plan. */
moa_status_t moa_psi_describe_3d(int64_t n0, int64_t n1, int64_t n2, moa_dtype_t dtype, moa_pass_desc_t *out,
                                 int max_passes, int *npasses);
/* The planner's lifting for (n, batch, dtype) on one GPU. */
moa_status_t moa_plan_radices(int64_t n, int64_t batch, moa_dtype_t dtype, int64_t *radices, int max_rad,
                              int *nrad);
/*
 * Density-matrix gate (PAPER.md Ch.6, "Density Matrix Operations for a Quantum
 * Computer").  A 2^n x 2^n density matrix D
 * (row-major, interleaved complex of `dtype`) is viewed as the 2n-cube D_h and
 * transposed by the vector t that moves the gated bits to the diagonal; every
 * 2^q x 2^q block of that view is replaced by U B U^dagger -- D <- U_full D
 * U_full^dagger without forming U_full or any temporary (Eq. generic,
 * i psi (t transpose D) = @D + gamma(i[t]; s)).
 * Conventions: bit 0 is the least significant; hypercube position p of an
 * n-bit half is bit n-1-p; bit j of U's row / column index is the j-th lowest
 * gated bit; i[t] has component t[k] equal to i[k] (R15).
 *
 * moa_qgate_permutation -- t (2n entries) for gated_bits[0..q) (host only).
 * moa_qgate_view_offset -- the element offset in D of view element
 *   (view_row, view_col): Eq. generic (host only).
 * moa_qgate_apply -- in place on the device matrix rho (16-byte aligned),
 *   stream-ordered; u is a HOST array of 2^q x 2^q complex values (row-major,
 *   same dtype as rho), copied at the call.  1 <= n <= 15, 1 <= q <= min(3, n),
 *   gated bits distinct in [0, n); otherwise MOA_EINVAL.
 */
moa_status_t moa_qgate_permutation(int n, const int32_t *gated_bits, int q, int32_t *t);
moa_status_t moa_qgate_view_offset(int n, const int32_t *gated_bits, int q, int64_t view_row, int64_t view_col,
                                   int64_t *offset);
moa_status_t moa_qgate_apply(void *rho, int n, const int32_t *gated_bits, int q, const void *u, moa_dtype_t dtype,
                             void *stream);

/*
 * moa_pass_move -- test hook: execute ONE pass descriptor as a
 * pure data movement on the GPU -- kind forced to 1 (no DFT), no twiddle, no
 * ring -- so that out[store(line, k)] = in[load(line, k)] for every line and
 * point of the ONF, through exactly the address arithmetic, thread mappings
 * and shared-memory exchanges the pass uses.  Lets tests compare the kernels'
 * movement bit-exactly with the descriptor's index maps on integer payloads.
 * Stream-ordered; d must come from moa_psi_describe* / moa_fft_plan_describe.
 */
moa_status_t moa_pass_move(const moa_pass_desc_t *d, moa_dtype_t dtype, const void *in, void *out, void *stream);

/* The descriptors a plan actually executes. */
moa_status_t moa_fft_plan_describe(moa_fft_plan_t plan, moa_pass_desc_t *out, int max_passes, int *npasses);

#ifdef __cplusplus
}
#endif
#endif /* MOA_FFT_H */

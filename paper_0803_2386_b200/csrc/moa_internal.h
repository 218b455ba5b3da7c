// Internal declarations of the B200 path (not part of the C-ABI).
//
// Vocabulary: a plan lifts the length-n vector to the array
// <R_0 R_1 ... R_{P-1}> (n = prod R_p); pass p runs R_p-point DFTs ("block
// butterflies") over the lines of axis p, multiplies by
// the lifted weights w_N^{e} and stores through the pass's
// reshape-transpose view (Eq. reshape3 P:2097-2114 / final transpose
// P:3042-3069).  A pass is described by an ONF: loops (extent, stride) over the
// line digits plus an affine address -- `moa_pass_desc_t`.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/moa_fft.h"

namespace moa {

constexpr int kMaxDigits = MOA_MAX_DIGITS;

// Set the thread-local error message and return the status.
moa_status_t fail(moa_status_t st, const std::string &msg);

// psi.cpp: the psi-index layer (host).  Builds the ONF descriptors of every
// pass of a lifting.  Pure integer arithmetic; no CUDA.
moa_status_t psi_lift_passes(int64_t n, int64_t batch, moa_dtype_t dtype, const int64_t *radices, int nrad,
                             std::vector<moa_pass_desc_t> &out);
moa_status_t psi_3d_passes(int64_t n0, int64_t n1, int64_t n2, int64_t howmany, moa_dtype_t dtype,
                           std::vector<moa_pass_desc_t> &out);
// Planner: the lifting n = R_0 ... R_{P-1} for one GPU (a1).
moa_status_t plan_radices(int64_t n, int64_t batch, moa_dtype_t dtype, std::vector<int64_t> &radices);
// Tile width (lines per CTA) and smem for a pass (fills desc.W / desc.smem_bytes / desc.threads).
void psi_choose_tile(moa_pass_desc_t &d, moa_dtype_t dtype);
// worst conflict degree (and total extra wavefronts) of a tile's exchange patterns
int psi_bank_conflicts(int logR, int64_t W, int esize, int lfA, int lfB, int64_t LS, int64_t *total, int logP = -1);
// Points per thread of a pass (log2): 16, except 512- and 1024-point lines,
// which take 32 (radix 32 x 16 / 32 x 32: one shared-memory exchange instead
// of two; the paired-complex64 kernel keeps 16 and is used only where this is 4);
// the shared-memory line pads one element per 2^psi_pad_shift elements.
inline int psi_log_p(int logR, moa_dtype_t dtype) {
    (void)dtype;
    return (logR == 9 || logR == 10) ? 5 : (logR < 4 ? logR : 4);
}
inline int psi_pad_shift(int logP) { return logP == 5 ? 5 : 4; }

// kernels.cu
struct DevTables {
    const void *twR = nullptr;   // this pass's in-line Stockham step twiddles (step-major, R - 1 entries)
    const void *tw_hi = nullptr; // w_N^{eh 2^h}
    const void *tw_lo = nullptr; // w_N^{el}
    const void *twS = nullptr;   // one-pass 2^6..2^12-point plans: the small-transform kernel's
                                 // radix-4 step twiddles (R - 4 entries, kernels.cu small_fft_kernel)
    unsigned long long *ctr = nullptr;  // this pass's tile counter (warp-specialised kernel), or null
};
// Device state of the L2 ring of a fused pass pair (owned by the plan).
struct RingState {
    void *ring = nullptr;                 // ring_slots * ring_G elements
    unsigned long long *qctr = nullptr;   // tile queue (epoch-based, never reset)
    unsigned long long *cntA = nullptr;   // per-group completed A tiles
    unsigned long long *cntB = nullptr;   // per-group completed B tiles
    unsigned long long epoch = 0;         // execs of this pair so far
    unsigned long long *stats = nullptr;  // MOA_FFT_STATS=1: B waits/spins/cycles, A waits/spins/cycles
};
// Per-launch modifiers of a pass (plan flags, include/moa_fft.h): the inverse
// transform as conj(DFT(conj(x))) -- conjugate the first pass's loads and the
// last pass's results -- and the 1/N normalisation folded into the last
// pass's store (exact: N is a power of two).
struct PassMods {
    int conj_in = 0;
    int conj_out = 0;
    double scale = 1.0;
    // Fused exchange (processor-level lifting): the pass stores straight into
    // the peers' buffers -- the all-to-all that followed it is folded into its
    // store.  Send-layout offset q goes to peers[q >> log_chunk] at
    // self_off + (q & (chunk - 1)).  npeers == 0: an ordinary local store.
    int npeers = 0;
    void *peers[8] = {};
    int log_chunk = 0;
    int64_t self_off = 0;
};
// the modifiers of pass i of npass under `flags` (MOA_FFT_INVERSE / _NORMALIZE)
PassMods pass_mods(uint32_t flags, size_t i, size_t npass, int64_t N);

int log2_exact(int64_t n);
cudaError_t launch_pass(const moa_pass_desc_t &d, moa_dtype_t dtype, const void *in, void *out,
                        const DevTables &tab, cudaStream_t stream, const PassMods &mods = PassMods());
cudaError_t launch_pair(const moa_pass_desc_t &dA, const moa_pass_desc_t &dB, moa_dtype_t dtype, const void *in,
                        void *out, const RingState &rs, const DevTables &tA, const DevTables &tB, cudaStream_t stream,
                        const PassMods &mA = PassMods(), const PassMods &mB = PassMods());
// The cluster level: passes A (ring == 3) and B (ring == 4) as one
// thread-block-cluster kernel, the group in the cluster's shared memory
// (ring_slots = CTAs per cluster, ring_G = elements per group).
cudaError_t launch_cluster(const moa_pass_desc_t &dA, const moa_pass_desc_t &dB, moa_dtype_t dtype, const void *in,
                           void *out, const DevTables &tA, const DevTables &tB, cudaStream_t stream,
                           const PassMods &mA = PassMods(), const PassMods &mB = PassMods());
// psi.cpp: a two-pass lifting of independent groups whose group fits one
// cluster's shared memory becomes a cluster pair (returns 1 if made)
int psi_cluster_pair(std::vector<moa_pass_desc_t> &passes, moa_dtype_t dtype, int64_t max_ctas, int64_t max_threads);
void psi_uncluster(std::vector<moa_pass_desc_t> &passes);
// psi.cpp: fuse the passes of a one-GPU lifting into L2-staged pairs where the
// group working set fits (marks ring fields; returns how many pairs were made)
int psi_fuse_pairs(std::vector<moa_pass_desc_t> &passes, const std::vector<int64_t> &radices, int64_t n, int64_t batch,
                   moa_dtype_t dtype);
// 3-D: fuse the z- and y-passes (group = one x-plane)
int psi_fuse_3d(std::vector<moa_pass_desc_t> &passes, moa_dtype_t dtype);
// The descriptors a 1-D plan runs: a planned 4-factor lifting (or any
// 4-factor lifting with MOA_FFT_LIFT4=1) as two fused pairs, otherwise the
// plain passes with the 2-pass fusion where it applies.
moa_status_t psi_build(int64_t n, int64_t batch, moa_dtype_t dtype, const std::vector<int64_t> &radices, bool planned,
                       std::vector<moa_pass_desc_t> &out);
cudaError_t kernel_attributes(moa_dtype_t dtype, int logR, int *max_threads, int *regs);

}  // namespace moa

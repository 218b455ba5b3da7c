// qgate.cu -- the density-matrix gate of PAPER.md Ch.6 on
// sm_100a: a q-qubit gate U applied to a 2^n x 2^n density matrix D in place,
// D <- U_full D U_full^dagger, by the paper's virtual block-diagonalisation --
// the 2n-cube D_h viewed through the transpose vector t that moves the gated
// bits to the diagonal (Eq. generic, i psi (t transpose D) = @D + gamma(i[t]; s),
// P:6493-6506, reading R15) -- so every 2^q x 2^q block of the view is
// B <- U B U^dagger (reading R16) and no permutation matrix or temporary array
// is formed.
//
// B200 mapping: one CTA owns the 2^q view rows of one ungated row index r and a
// tile of view columns: all 2^q gated column values x K consecutive values of
// the lowest ungated column bits.  With the gated and low ungated bits
// deposited into their original positions (a bit-deposit table), consecutive
// threads read consecutive columns of every row -- the whole matrix streams
// through HBM once (read + write), coalesced.  The two small products
// T = B U^dagger and B' = U T run from shared memory.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "../../include/moa_fft.h"
#include "moa_internal.h"

namespace moa {
namespace {

constexpr int kMaxQ = 8;      // 2^q, q <= 3
constexpr int kMaxTC = 256;   // tile columns (threads per CTA)
// S holds two Q x (TC + 1) buffers: cap TC so that stays near 32 KiB for complex128
constexpr __host__ __device__ int tc_cap(int Q) { return Q <= 4 ? 256 : 128; }

template <typename V> struct QgArgs {
    V *rho;
    int64_t N;                 // 2^n
    int32_t Q, TC;             // 2^q, tile columns = Q * K
    int32_t RG;                // ungated row indices per CTA (consecutive)
    int32_t TP;                // shared-memory row stride (elements), >= TC
    int64_t gdep[kMaxQ];       // pdep(a, gated mask), a < Q
    int32_t vdep[kMaxTC];      // pdep(tc, varying column mask), tc < TC
    int32_t rdep[kMaxTC];      // tile column of the rest index ri with all gated values 0, ri < TC / Q
    int32_t gpos_dep[kMaxQ];   // tile-column offset of gated value l (pdep(l, gated positions in tc))
    int32_t gpos_mask;         // positions of the gated bits inside tc
    uint32_t ung_mask;         // ungated bits (rows: all of them)
    uint32_t ung_hi_mask;      // ungated column bits above the tile's varying ones
    V u[kMaxQ * kMaxQ];        // U, row-major
};

__device__ __forceinline__ int64_t pdep_loop(int64_t x, uint32_t mask) {
    int64_t r = 0;
    for (int b = 0; mask; b++) {
        const int low = __ffs(mask) - 1;
        if (x & 1) r |= int64_t(1) << low;
        x >>= 1;
        mask &= mask - 1;
        (void)b;
    }
    return r;
}

// acc + a * b and acc + a * conj(b) as four FMAs (the gate is FP64-FMA bound at q = 3)
template <typename V> __device__ __forceinline__ void cmac(V &acc, V a, V b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
}
template <typename V> __device__ __forceinline__ void cmacc(V &acc, V a, V b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(a.y, b.y, acc.x);
    acc.y = fma(a.y, b.x, acc.y);
    acc.y = fma(-a.x, b.y, acc.y);
}

template <typename V, int Q>
__global__ void __launch_bounds__(tc_cap(Q)) qgate_kernel(const __grid_constant__ QgArgs<V> a) {
    // One row group = the Q x TC tile B of Q view rows; per row group:
    //   stage    S[k][tc]  <- B[k][tc]              (thread tc; coalesced rows)
    //   phase 1  S[k][rest | j] <- sum_l S[k][rest | l] conj(U[j][l])   (T = B U^dagger;
    //            thread (k, ri) owns the Q entries it reads and writes -> in place)
    //   phase 2  B'[i][tc] = sum_k U[i][k] S[k][tc]  (thread tc; coalesced stores)
    // Every element crosses shared memory twice each way; U is read with
    // warp-uniform indices.  S is double-buffered (dynamic shared memory, row
    // stride a.TP chosen on the host by a bank model of the phase-1 pattern; the
    // row-contiguous stage / phase-2 accesses are conflict-free for any stride):
    // iteration it uses buffer it & 1, last used by iteration it - 2, whose
    // phase-2 reads all precede iteration it - 1's first barrier.
    extern __shared__ __align__(16) unsigned char qg_smem[];
    const int TP = a.TP;
    const int tc = threadIdx.x;
    const int64_t nh = a.N / a.TC;  // column tiles per row
    const int64_t rg = blockIdx.x / nh, h = blockIdx.x % nh;
    const int64_t col = pdep_loop(h, a.ung_hi_mask) + a.vdep[tc];
    const int k1 = tc & (Q - 1);       // phase-1 row
    const int rest = a.rdep[tc / Q];   // phase-1 column base (gated values 0)
    const int64_t ung = int64_t(a.ung_mask);
    int64_t row0 = pdep_loop(rg * a.RG, a.ung_mask);
    V cur[Q];
#pragma unroll
    for (int k = 0; k < Q; k++) cur[k] = a.rho[(row0 + a.gdep[k]) * a.N + col];
    for (int it = 0; it < a.RG; it++) {
        V *Sb = reinterpret_cast<V *>(qg_smem) + (it & 1) * Q * TP;
#pragma unroll
        for (int k = 0; k < Q; k++) Sb[k * TP + tc] = cur[k];
        const int64_t next = ((row0 | ~ung) + 1) & ung;  // pdep(r + 1, ung) from pdep(r, ung)
        if (it + 1 < a.RG) {
#pragma unroll
            for (int k = 0; k < Q; k++) cur[k] = a.rho[(next + a.gdep[k]) * a.N + col];
        }
        __syncthreads();
        {
            V x[Q];
#pragma unroll
            for (int l = 0; l < Q; l++) x[l] = Sb[k1 * TP + (rest | a.gpos_dep[l])];
#pragma unroll
            for (int j = 0; j < Q; j++) {
                V acc;
                acc.x = 0;
                acc.y = 0;
#pragma unroll
                for (int l = 0; l < Q; l++) cmacc(acc, x[l], a.u[j * Q + l]);
                Sb[k1 * TP + (rest | a.gpos_dep[j])] = acc;
            }
        }
        __syncthreads();
        V *base = a.rho + row0 * a.N + col;
        V t[Q];
#pragma unroll
        for (int k = 0; k < Q; k++) t[k] = Sb[k * TP + tc];
#pragma unroll
        for (int i = 0; i < Q; i++) {
            V acc;
            acc.x = 0;
            acc.y = 0;
#pragma unroll
            for (int k = 0; k < Q; k++) cmac(acc, a.u[i * Q + k], t[k]);
            base[a.gdep[i] * a.N] = acc;
        }
        row0 = next;
    }
}

moa_status_t check_bits(int n, const int32_t *bits, int q, uint32_t *gmask) {
    if (n < 1 || n > 15) return fail(MOA_EINVAL, "qgate: n must be in [1, 15]");
    if (!bits || q < 1 || q > 3 || q > n) return fail(MOA_EINVAL, "qgate: q must be in [1, min(3, n)]");
    uint32_t m = 0;
    for (int i = 0; i < q; i++) {
        if (bits[i] < 0 || bits[i] >= n) return fail(MOA_EINVAL, "qgate: gated bit out of range");
        if (m & (1u << bits[i])) return fail(MOA_EINVAL, "qgate: duplicate gated bit");
        m |= 1u << bits[i];
    }
    *gmask = m;
    return MOA_OK;
}

int64_t pdep_host(int64_t x, uint32_t mask) {
    int64_t r = 0;
    for (int b = 0; b < 32; b++)
        if (mask & (1u << b)) {
            if (x & 1) r |= int64_t(1) << b;
            x >>= 1;
        }
    return r;
}

// Shared-memory wavefronts of one phase-1 access (lane (k1, ri) of warp w
// touching S[k1 * TP + (rdep[ri] | gpos_dep[l])]): the lanes are served in
// groups of 128 bytes (8 lanes for 16-byte elements, 16 for 8-byte), each
// group taking max over the 32 four-byte banks of the words it hits.  The
// stride is the TP in [TC, TC + 32) with the fewest wavefronts summed over
// groups, warps and l (ties: smallest).  Measured (profiles/r1_s6_qgate_tp.jsonl):
// a whole-warp bank count ties TC with TC + 2 for gated bits {3, 9} while TC
// runs 25 % slower; the per-group count separates them.
int qgate_row_stride(int Q, int TC, const int32_t *rdep, const int32_t *gpos_dep, int esz) {
    // memoised per (Q, TC, gated positions in the tile, element size)
    static std::mutex mu;
    static std::map<std::tuple<int, int, int, int>, int> memo;
    const auto key = std::make_tuple(Q, TC, gpos_dep[Q - 1], esz);  // gpos_dep[Q - 1] = the gated-position mask
    {
        std::lock_guard<std::mutex> g(mu);
        auto it = memo.find(key);
        if (it != memo.end()) return it->second;
    }
    const int words = esz / 4;
    int best_tp = TC;
    long best = -1;
    for (int tp = TC; tp < TC + 32; tp++) {
        long cost = 0;
        for (int w = 0; w < TC / 32; w++)
            for (int l = 0; l < Q; l++) {
                // distinct lanes hit distinct elements (each (k1, ri) owns its own)
                const int grp = 32 / words;
                for (int g0 = 0; g0 < 32; g0 += grp) {
                    int per_bank[32] = {0};
                    for (int lane = g0; lane < g0 + grp; lane++) {
                        const int tc = w * 32 + lane;
                        const int e = (tc & (Q - 1)) * tp + (rdep[tc / Q] | gpos_dep[l]);
                        for (int x = 0; x < words; x++) per_bank[(e * words + x) & 31]++;
                    }
                    int mx = 0;
                    for (int b = 0; b < 32; b++) mx = per_bank[b] > mx ? per_bank[b] : mx;
                    cost += mx;
                }
            }
        if (best < 0 || cost < best) {
            best = cost;
            best_tp = tp;
        }
    }
    std::lock_guard<std::mutex> g(mu);
    memo[key] = best_tp;
    return best_tp;
}

template <typename V>
moa_status_t qgate_launch(V *rho, int n, uint32_t gmask, int q, const V *u, cudaStream_t s) {
    QgArgs<V> a;
    std::memset(&a, 0, sizeof(a));
    const int Q = 1 << q;
    const uint32_t all = (n >= 32) ? 0xffffffffu : ((1u << n) - 1);
    const uint32_t ung = all & ~gmask;
    // tile: all Q gated column values x K = 2^kc lowest ungated column values
    int kc = 0;
    while ((Q << (kc + 1)) <= tc_cap(Q) && kc + 1 <= n - q) kc++;
    uint32_t low_ung = 0;
    {
        int taken = 0;
        for (int bit = 0; bit < n && taken < kc; bit++)
            if (ung & (1u << bit)) {
                low_ung |= 1u << bit;
                taken++;
            }
    }
    const uint32_t vmask = gmask | low_ung;
    a.rho = rho;
    a.N = int64_t(1) << n;
    a.Q = Q;
    a.TC = Q << kc;
    a.ung_mask = ung;
    a.ung_hi_mask = ung & ~low_ung;
    for (int i = 0; i < Q; i++) a.gdep[i] = pdep_host(i, gmask);
    // positions of the gated bits inside the compressed tile-column index
    int pos = 0;
    for (int bit = 0; bit < n; bit++) {
        if (!(vmask & (1u << bit))) continue;
        if (gmask & (1u << bit)) a.gpos_mask |= 1 << pos;
        pos++;
    }
    for (int tc = 0; tc < a.TC; tc++) a.vdep[tc] = int32_t(pdep_host(tc, vmask));
    for (int ri = 0; ri < a.TC / Q; ri++)
        a.rdep[ri] = int32_t(pdep_host(ri, uint32_t(a.TC - 1) & ~uint32_t(a.gpos_mask)));
    for (int l = 0; l < Q; l++) a.gpos_dep[l] = int32_t(pdep_host(l, uint32_t(a.gpos_mask)));
    for (int i = 0; i < Q * Q; i++) a.u[i] = u[i];
    // several row groups per CTA (about 8 K elements of work per CTA)
    const int64_t rows_groups = a.N / Q;
    int64_t rgp = 1;
    while (rgp * 2 <= rows_groups && rgp * 2 * Q * a.TC <= 8192) rgp *= 2;
    a.RG = int32_t(rgp);
    const int64_t blocks = (rows_groups / rgp) * (a.N / a.TC);
    a.TP = qgate_row_stride(Q, a.TC, a.rdep, a.gpos_dep, int(sizeof(V)));
    static const char *tp_off = std::getenv("MOA_QG_TP_OFF");  // ablation knob, read once
    if (tp_off) a.TP = a.TC + std::atoi(tp_off);
    const size_t smem = size_t(2) * Q * a.TP * sizeof(V);
    if (blocks > 0x7fffffff) return fail(MOA_EUNSUPPORTED, "qgate: grid too large");
    switch (Q) {
        case 2: qgate_kernel<V, 2><<<unsigned(blocks), a.TC, smem, s>>>(a); break;
        case 4: qgate_kernel<V, 4><<<unsigned(blocks), a.TC, smem, s>>>(a); break;
        default: qgate_kernel<V, 8><<<unsigned(blocks), a.TC, smem, s>>>(a); break;
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(MOA_ECUDA, std::string("qgate launch: ") + cudaGetErrorString(e));
    return MOA_OK;
}

}  // namespace
}  // namespace moa

using namespace moa;

extern "C" {

moa_status_t moa_qgate_permutation(int n, const int32_t *gated_bits, int q, int32_t *t) {
    uint32_t gm = 0;
    moa_status_t st = check_bits(n, gated_bits, q, &gm);
    if (st) return st;
    if (!t) return fail(MOA_EINVAL, "qgate_permutation: null output");
    // hypercube position p of an n-bit half is bit n-1-p; ungated positions
    // first, gated last, each in order (the stable partition of P:6409-6418)
    int k = 0;
    for (int p = 0; p < n; p++)
        if (!(gm & (1u << (n - 1 - p)))) t[k++] = p;
    for (int p = 0; p < n; p++)
        if (gm & (1u << (n - 1 - p))) t[k++] = p;
    for (int i = 0; i < n; i++) t[n + i] = t[i] + n;
    return MOA_OK;
}

moa_status_t moa_qgate_view_offset(int n, const int32_t *gated_bits, int q, int64_t view_row, int64_t view_col,
                                   int64_t *offset) {
    int32_t t[32];
    moa_status_t st = moa_qgate_permutation(n, gated_bits, q, t);
    if (st) return st;
    if (!offset || view_row < 0 || view_col < 0 || view_row >= (int64_t(1) << n) || view_col >= (int64_t(1) << n))
        return fail(MOA_EINVAL, "qgate_view_offset: bad index");
    // i: the 2n coordinates of the view index (row bits then column bits, MSB first);
    // the original index has coordinate t[k] equal to i[k] (reading R15); gamma on <2 ... 2>
    int bitsv[32];
    for (int p = 0; p < n; p++) {
        bitsv[p] = int((view_row >> (n - 1 - p)) & 1);
        bitsv[n + p] = int((view_col >> (n - 1 - p)) & 1);
    }
    int orig[32];
    for (int k = 0; k < 2 * n; k++) orig[t[k]] = bitsv[k];
    int64_t off = 0;
    for (int k = 0; k < 2 * n; k++) off = off * 2 + orig[k];
    *offset = off;
    return MOA_OK;
}

moa_status_t moa_qgate_apply(void *rho, int n, const int32_t *gated_bits, int q, const void *u, moa_dtype_t dtype,
                             void *stream) {
    uint32_t gm = 0;
    moa_status_t st = check_bits(n, gated_bits, q, &gm);
    if (st) return st;
    if (!rho || !u) return fail(MOA_EINVAL, "qgate_apply: null pointer");
    if (reinterpret_cast<uintptr_t>(rho) & 15) return fail(MOA_EINVAL, "qgate_apply: rho must be 16-byte aligned");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (dtype == MOA_C128) return qgate_launch<double2>(static_cast<double2 *>(rho), n, gm, q, static_cast<const double2 *>(u), s);
    if (dtype == MOA_C64) return qgate_launch<float2>(static_cast<float2 *>(rho), n, gm, q, static_cast<const float2 *>(u), s);
    return fail(MOA_EINVAL, "qgate_apply: unknown dtype");
}

}  // extern "C"

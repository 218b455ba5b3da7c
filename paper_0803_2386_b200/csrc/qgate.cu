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

#include <cstring>
#include <string>

#include "../../include/moa_fft.h"
#include "moa_internal.h"

namespace moa {
namespace {

constexpr int kMaxQ = 8;      // 2^q, q <= 3
constexpr int kMaxTC = 128;   // tile columns (threads per CTA)

template <typename V> struct QgArgs {
    V *rho;
    int64_t N;                 // 2^n
    int32_t Q, TC;             // 2^q, tile columns = Q * K
    int64_t gdep[kMaxQ];       // pdep(a, gated mask), a < Q
    int32_t vdep[kMaxTC];      // pdep(tc, varying column mask), tc < TC
    int32_t bsel[kMaxTC];      // gated part b of tile column tc (pext over the gated positions)
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

__device__ __forceinline__ double2 cmulq(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cmulq(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cmulcq(double2 a, double2 b) {  // a * conj(b)
    return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ float2 cmulcq(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
template <typename V> __device__ __forceinline__ V caddq(V a, V b) {
    V r;
    r.x = a.x + b.x;
    r.y = a.y + b.y;
    return r;
}

template <typename V, int Q>
__global__ void __launch_bounds__(kMaxTC) qgate_kernel(const __grid_constant__ QgArgs<V> a) {
    __shared__ V S[Q][kMaxTC];
    __shared__ V T[Q][kMaxTC];
    const int tc = threadIdx.x;
    // CTA -> (r: ungated row index, h: ungated column index above the tile)
    const int64_t nh = a.N / (int64_t(Q) * (a.TC / Q));  // column tiles per row
    const int64_t r = blockIdx.x / nh, h = blockIdx.x % nh;
    const int64_t row0 = pdep_loop(r, a.ung_mask);
    const int64_t col = pdep_loop(h, a.ung_hi_mask) + a.vdep[tc];
    V *base = a.rho + row0 * a.N + col;
    // gather the Q view rows of this tile (each row a coalesced run of columns)
#pragma unroll
    for (int k = 0; k < Q; k++) S[k][tc] = base[a.gdep[k] * a.N];
    __syncthreads();
    // T = B U^dagger : T[k][tc] = sum_l B[k][(tc, l)] conj(U[b][l])
    const int b = a.bsel[tc];
    const int rest = tc & ~a.gpos_mask;
#pragma unroll
    for (int k = 0; k < Q; k++) {
        V acc;
        acc.x = 0;
        acc.y = 0;
#pragma unroll
        for (int l = 0; l < Q; l++) acc = caddq(acc, cmulcq(S[k][rest | a.gpos_dep[l]], a.u[b * Q + l]));
        T[k][tc] = acc;
    }
    __syncthreads();
    // B' = U T, written back in place
#pragma unroll
    for (int i = 0; i < Q; i++) {
        V acc;
        acc.x = 0;
        acc.y = 0;
#pragma unroll
        for (int k = 0; k < Q; k++) acc = caddq(acc, cmulq(a.u[i * Q + k], T[k][tc]));
        base[a.gdep[i] * a.N] = acc;
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

template <typename V>
moa_status_t qgate_launch(V *rho, int n, uint32_t gmask, int q, const V *u, cudaStream_t s) {
    QgArgs<V> a;
    std::memset(&a, 0, sizeof(a));
    const int Q = 1 << q;
    const uint32_t all = (n >= 32) ? 0xffffffffu : ((1u << n) - 1);
    const uint32_t ung = all & ~gmask;
    // tile: all Q gated column values x K = 2^kc lowest ungated column values
    int kc = 0;
    while ((Q << (kc + 1)) <= kMaxTC && kc + 1 <= n - q) kc++;
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
    for (int tc = 0; tc < a.TC; tc++) {
        a.vdep[tc] = int32_t(pdep_host(tc, vmask));
        int b = 0, j = 0;
        for (int p = 0; p < 16; p++)
            if (a.gpos_mask & (1 << p)) b |= ((tc >> p) & 1) << j++;
        a.bsel[tc] = b;
    }
    for (int l = 0; l < Q; l++) a.gpos_dep[l] = int32_t(pdep_host(l, uint32_t(a.gpos_mask)));
    for (int i = 0; i < Q * Q; i++) a.u[i] = u[i];
    const int64_t blocks = (a.N / Q) * (a.N / a.TC);
    if (blocks > 0x7fffffff) return fail(MOA_EUNSUPPORTED, "qgate: grid too large");
    switch (Q) {
        case 2: qgate_kernel<V, 2><<<unsigned(blocks), a.TC, 0, s>>>(a); break;
        case 4: qgate_kernel<V, 4><<<unsigned(blocks), a.TC, 0, s>>>(a); break;
        default: qgate_kernel<V, 8><<<unsigned(blocks), a.TC, 0, s>>>(a); break;
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

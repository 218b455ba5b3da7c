// kernels.cu -- sm_100a pass kernel of the lifted FFT (steps a3-a7 of
// SURVEY.md §8(a)).
//
// One launch = one pass of the lifting.  A CTA owns a tile of W
// adjacent lines of R = 2^LOG_R points.  Per tile:
//   1. load   -- 128-bit vectorised global loads.  A pass whose points are
//                strided (the reshape-transpose view, Eq. reshape3)
//                loads W adjacent lines per point so each warp request covers
//                whole 128-byte lines ("line-fast"), then transposes through
//                shared memory; a pass with contiguous lines loads directly into
//                registers ("point-fast").
//   2. block butterflies -- the R-point DFT of every line as a sequence of
//                Stockham steps of radix Q <= 16 (Q <= 32 for 512- and 1024-point
//                lines: 32 points per thread, one exchange) done in registers (an
//                in-register radix-2 network, FMA-shaped), with the step twiddles
//                of a self-sorting (autosort) schedule.  The paper's input bit
//                reversal P_n is never materialised: each step's output
//                index map absorbs it (step a3).  Exchanges between steps go
//                through shared memory with one pad element per 16 (32) and a line
//                stride chosen on the host by a bank-conflict model
//                (psi_choose_tile).
//   3. twiddle -- the lifted weights w_N^{(j k) mod N} from a
//                two-level table (exact integer exponent; two lookups per thread,
//                the thread's 16 / 32 weights as two-level products), fused
//                before the store.
//   4. store  -- point-fast, or line-fast through shared memory (the final
//                transpose F / digit reversal) with 128-byte runs.
// No tensor cores: the FFT is not a dense contraction.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <array>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>
#include <utility>

#include "moa_internal.h"

namespace moa {
namespace {

// ---------------------------------------------------------------- complex ops
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 w) {
    return make_double2(fma(a.x, w.x, -a.y * w.y), fma(a.x, w.y, a.y * w.x));
}
// complex64 arithmetic on the packed FP32x2 pipe (sm_100: FADD2 / FMUL2 /
// FFMA2 -- one instruction per complex add, two per complex multiply; ptxas
// folds the operand swap and the broadcast of w.x / w.y into the instruction's
// operand modifiers, so no register moves).  The complex64 passes are
// instruction-issue bound, and this halves their FP32 count.
// MOA_FFT_NO_F32X2 (compile-time) restores the scalar forms for ablation.
#ifndef MOA_FFT_NO_F32X2
__device__ __forceinline__ unsigned long long pk2(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float2 upk2(unsigned long long v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
    return upk2(d);
}
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
    unsigned long long d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
    return upk2(d);
}
__device__ __forceinline__ float2 cmul(float2 a, float2 w) {  // (a.x w.x - a.y w.y, a.y w.x + a.x w.y)
    unsigned long long t, d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(pk2(a.x, a.y)), "l"(pk2(w.x, w.x)));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pk2(a.y, a.x)), "l"(pk2(-w.y, w.y)), "l"(t));
    return upk2(d);
}
#else
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 w) {
    return make_float2(fmaf(a.x, w.x, -a.y * w.y), fmaf(a.x, w.y, a.y * w.x));
}
#endif
// Paired complex64 lines: two ADJACENT lines of a line-coalesced complex64
// pass in one 16-byte quad (re0, im0, re1, im1) -- one 128-bit load / store /
// exchange per two points and one set of step twiddles and address
// arithmetic for both lines (the complex64 passes are issue-bound).
__device__ __forceinline__ float4 f4(float2 lo, float2 hi) { return make_float4(lo.x, lo.y, hi.x, hi.y); }
__device__ __forceinline__ float2 lo2(float4 a) { return make_float2(a.x, a.y); }
__device__ __forceinline__ float2 hi2(float4 a) { return make_float2(a.z, a.w); }
__device__ __forceinline__ float4 cadd(float4 a, float4 b) { return f4(cadd(lo2(a), lo2(b)), cadd(hi2(a), hi2(b))); }
__device__ __forceinline__ float4 csub(float4 a, float4 b) { return f4(csub(lo2(a), lo2(b)), csub(hi2(a), hi2(b))); }
__device__ __forceinline__ float4 cmul(float4 a, float2 w) { return f4(cmul(lo2(a), w), cmul(hi2(a), w)); }
__device__ __forceinline__ float4 cmul(float4 a, float4 w) {  // a different weight per line
    return f4(cmul(lo2(a), lo2(w)), cmul(hi2(a), hi2(w)));
}
template <typename V> struct RealOf;
template <> struct RealOf<double2> { using type = double; };
template <> struct RealOf<float2> { using type = float; };
template <> struct RealOf<float4> { using type = float; };
// element (one complex) and step-twiddle type of a pass value type
template <typename V> struct ElemOf { using type = V; };
template <> struct ElemOf<float4> { using type = float2; };
template <typename V> __host__ __device__ constexpr int lines_per_lane() { return std::is_same<V, float4>::value ? 2 : 1; }
template <typename V> __device__ __forceinline__ V mk(typename RealOf<V>::type x, typename RealOf<V>::type y) {
    V v;
    v.x = x;
    v.y = y;
    return v;
}

// z * w_16^e for a compile-time e in [0, 8) (w_16 = e^{-2 pi i/16}); the
// trivial and 1/sqrt2 cases are special-cased so no multiply by 0 or 1 is issued.
template <int E, typename V> __device__ __forceinline__ V rot16(V z) {
    using T = typename RealOf<V>::type;
    constexpr double C1 = 0.92387953251128675613, S1 = 0.38268343236508977173, H = 0.70710678118654752440;
    if constexpr (std::is_same<V, float4>::value) {  // both lines of a pair
        const float2 lo = rot16<E>(make_float2(z.x, z.y)), hi = rot16<E>(make_float2(z.z, z.w));
        return make_float4(lo.x, lo.y, hi.x, hi.y);
    } else if constexpr (E == 0) return z;
    else if constexpr (E == 4) return mk<V>(z.y, -z.x);                          // * (-i)
    else if constexpr (E == 2) return mk<V>((z.x + z.y) * T(H), (z.y - z.x) * T(H));   // * (1-i)/sqrt2
    else if constexpr (E == 6) return mk<V>((z.y - z.x) * T(H), -(z.x + z.y) * T(H));  // * (-1-i)/sqrt2
    else {
        constexpr double wr = E == 1 ? C1 : E == 3 ? S1 : E == 5 ? -S1 : -C1;
        constexpr double wi = E == 1 ? -S1 : E == 3 ? -C1 : E == 5 ? -C1 : -S1;
        return cmul(z, mk<V>(T(wr), T(wi)));
    }
}

// In-register DFT of Q = 2^LQ points, natural order in and out:
// radix-2 decimation in frequency (span h = Q/2 ... 1, butterfly
// (a, b) -> (a + b, (a - b) w_{2h}^i), cf. B_L of Fig. vanloan_fft
// run backwards), then the compile-time bit-reversal of the register indices.
template <int LQ> __device__ __forceinline__ constexpr int brev(int k) {
    int r = 0;
    for (int b = 0; b < LQ; b++)
        if (k & (1 << b)) r |= 1 << (LQ - 1 - b);
    return r;
}
// z * w_32^e for a compile-time e in [0, 16): even e is w_16^{e/2}; odd e a
// general multiply by the constant (the radix-32 steps only)
template <int E, typename V> __device__ __forceinline__ V rot32(V z) {
    if constexpr (E % 2 == 0) {
        return rot16<E / 2>(z);
    } else {
        using T = typename RealOf<V>::type;
        constexpr double A = 0.98078528040323044913, B = 0.19509032201612826785;  // cos, sin(pi/16)
        constexpr double C = 0.83146961230254523708, D = 0.55557023301960222474;  // cos, sin(3 pi/16)
        constexpr double c = E == 1 ? A : E == 3 ? C : E == 5 ? D : E == 7 ? B : E == 9 ? -B : E == 11 ? -D
                                                                                           : E == 13 ? -C : -A;
        constexpr double s = E == 1 ? B : E == 3 ? D : E == 5 ? C : E == 7 ? A : E == 9 ? A : E == 11 ? C
                                                                                          : E == 13 ? D : B;
        return cmul(z, mk<V>(T(c), T(-s)));  // w_32^e = cos(pi e/16) - i sin(pi e/16)
    }
}
template <int LQ, int H, int G, int I, typename V> __device__ __forceinline__ void dif_bfly(V *v) {
    V a = v[G + I], b = v[G + I + H];
    v[G + I] = cadd(a, b);
    // (a - b) w_{2H}^I
    if constexpr (H == 16) v[G + I + H] = rot32<I>(csub(a, b));
    else v[G + I + H] = rot16<I *(8 / H)>(csub(a, b));
}
template <int LQ, int H, typename V, int... Is> __device__ __forceinline__ void dif_span(V *v, std::integer_sequence<int, Is...>) {
    // Is enumerates (group, i) pairs: g = (idx / H) * 2H, i = idx % H
    (dif_bfly<LQ, H, (Is / H) * 2 * H, Is % H>(v), ...);
}
template <int LQ, int H, typename V> __device__ __forceinline__ void dif_all(V *v) {
    if constexpr (H >= 1) {
        dif_span<LQ, H>(v, std::make_integer_sequence<int, (1 << LQ) / 2>{});
        dif_all<LQ, H / 2>(v);
    }
}
#ifdef MOA_FFT_DIF_NET
// (ablation build: the radix-2 decimation-in-frequency network with separate
// complex rotations -- the round-1/2 default)
template <int LQ, typename V> __device__ __forceinline__ void dft_reg(V *v) {
    constexpr int Q = 1 << LQ;
    if constexpr (Q > 1) {
        dif_all<LQ, Q / 2>(v);
        V t[Q];
#pragma unroll
        for (int k = 0; k < Q; k++) t[k] = v[brev<LQ>(k)];
#pragma unroll
        for (int k = 0; k < Q; k++) v[k] = t[k];
    }
}
#else
// Radix-2 decimation in time with FMA-shaped butterflies: the same radix-2
// network (Fig. vanloan_fft's B_L stages), inputs taken in
// bit-reversed register order (a compile-time renaming), spans 1, 2, ..., Q/2.
// A butterfly (a, b) -> (a + w b, a - w b) with a nontrivial w = c + i s is
// written w b = c (b + i tau b), tau = s / c (or w b = s (cot b + i b) when
// |s| > |c|), so it costs 6 FMAs in complex128 (3 packed FFMA2 in complex64)
// instead of a rotation (4) plus two complex adds (4): the 32-point DFT drops
// from 456 to 388 FP64 instructions.  Twiddle constants w_32^E = cos(pi E/16)
// - i sin(pi E/16) at compile time; the tangents of E = 4, 12 are exactly -/+1.
constexpr double kCos16[9] = {1.0,
                              0.98078528040323044913,
                              0.92387953251128675613,
                              0.83146961230254523708,
                              0.70710678118654752440,
                              0.55557023301960222474,
                              0.38268343236508977173,
                              0.19509032201612826785,
                              0.0};
template <int E> __host__ __device__ constexpr double w32_re() { return E <= 8 ? kCos16[E] : -kCos16[16 - E]; }
template <int E> __host__ __device__ constexpr double w32_im() { return E <= 8 ? -kCos16[8 - E] : -kCos16[E - 8]; }
// a <- a + w b, b <- a - w b with w b = f (u), u = b + i r b (tangent form:
// f = c, r = s / c) or u = r b + i b (cotangent form: f = s, r = c / s)
template <bool kTan> __device__ __forceinline__ void bfly_fma(double2 &a, double2 &b, double f, double r) {
    double2 u;
    if constexpr (kTan) u = make_double2(fma(-r, b.y, b.x), fma(r, b.x, b.y));
    else u = make_double2(fma(r, b.x, -b.y), fma(r, b.y, b.x));
    const double2 a0 = a;
    a = make_double2(fma(f, u.x, a0.x), fma(f, u.y, a0.y));
    b = make_double2(fma(-f, u.x, a0.x), fma(-f, u.y, a0.y));
}
#ifndef MOA_FFT_NO_F32X2
__device__ __forceinline__ unsigned long long ffma2(unsigned long long x, unsigned long long y, unsigned long long z) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(x), "l"(y), "l"(z));
    return d;
}
template <bool kTan> __device__ __forceinline__ void bfly_fma(float2 &a, float2 &b, double f, double r) {
    const float fr = float(r), ff = float(f);
    // u = b + r (-b.y, b.x)  (tangent)  or  r b + (-b.y, b.x)  (cotangent)
    const unsigned long long u = kTan ? ffma2(pk2(-b.y, b.x), pk2(fr, fr), pk2(b.x, b.y))
                                      : ffma2(pk2(b.x, b.y), pk2(fr, fr), pk2(-b.y, b.x));
    const unsigned long long a0 = pk2(a.x, a.y);
    a = upk2(ffma2(pk2(ff, ff), u, a0));
    b = upk2(ffma2(pk2(-ff, -ff), u, a0));
}
#else
template <bool kTan> __device__ __forceinline__ void bfly_fma(float2 &a, float2 &b, double f, double r) {
    const float fr = float(r), ff = float(f);
    float2 u;
    if constexpr (kTan) u = make_float2(fmaf(-fr, b.y, b.x), fmaf(fr, b.x, b.y));
    else u = make_float2(fmaf(fr, b.x, -b.y), fmaf(fr, b.y, b.x));
    const float2 a0 = a;
    a = make_float2(fmaf(ff, u.x, a0.x), fmaf(ff, u.y, a0.y));
    b = make_float2(fmaf(-ff, u.x, a0.x), fmaf(-ff, u.y, a0.y));
}
#endif
template <bool kTan> __device__ __forceinline__ void bfly_fma(float4 &a, float4 &b, double f, double r) {
    float2 al = lo2(a), ah = hi2(a), bl = lo2(b), bh = hi2(b);
    bfly_fma<kTan>(al, bl, f, r);
    bfly_fma<kTan>(ah, bh, f, r);
    a = f4(al, ah);
    b = f4(bl, bh);
}
// w_32^E b for the trivial E = 8 (-i): (b.y, -b.x)
template <typename V> __device__ __forceinline__ V mul_mi(V b) {
    if constexpr (std::is_same<V, float4>::value) return make_float4(b.y, -b.x, b.w, -b.z);
    else return mk<V>(b.y, -b.x);
}
template <int E, typename V> __device__ __forceinline__ void dit_bfly_w(V &a, V &b) {
    if constexpr (E == 0) {
        const V a0 = a;
        a = cadd(a0, b);
        b = csub(a0, b);
    } else if constexpr (E == 8) {
        const V a0 = a, t = mul_mi(b);
        a = cadd(a0, t);
        b = csub(a0, t);
    } else {
        constexpr double c = w32_re<E>(), sn = w32_im<E>();
        constexpr bool tan_form = (c < 0 ? -c : c) >= (sn < 0 ? -sn : sn);
        if constexpr (tan_form) bfly_fma<true>(a, b, c, sn / c);
        else bfly_fma<false>(a, b, sn, c / sn);
    }
}
template <int H, int G, int I, typename V> __device__ __forceinline__ void dit_bfly(V *v) {
    dit_bfly_w<I *(16 / H)>(v[G + I], v[G + I + H]);  // w_{2H}^I = w_32^{16 I / H}
}
template <int H, typename V, int... Is> __device__ __forceinline__ void dit_span(V *v, std::integer_sequence<int, Is...>) {
    (dit_bfly<H, (Is / H) * 2 * H, Is % H>(v), ...);
}
template <int LQ, int H, typename V> __device__ __forceinline__ void dit_all(V *v) {
    if constexpr (H < (1 << LQ)) {
        dit_span<H>(v, std::make_integer_sequence<int, (1 << LQ) / 2>{});
        dit_all<LQ, 2 * H>(v);
    }
}
template <int LQ, typename V> __device__ __forceinline__ void dft_reg(V *v) {
    constexpr int Q = 1 << LQ;
    static_assert(Q <= 32, "register DFTs of at most 32 points");
    if constexpr (Q > 1) {
        V t[Q];
#pragma unroll
        for (int k = 0; k < Q; k++) t[k] = v[brev<LQ>(k)];
        dit_all<LQ, 1>(t);
#pragma unroll
        for (int k = 0; k < Q; k++) v[k] = t[k];
    }
}
#endif

// Shared-memory position of element i of a line: one pad element per 16, so
// the radix-16 stride-16 writes of step 0 and the unit-stride reads are
// bank-conflict free, and every (base + compile-time offset) folds into the
// instruction's immediate (no per-access swizzle arithmetic).  The line stride
// LS is chosen on the host by a conflict model of all the patterns
// (psi_choose_tile).  LB is log2 of the pad period: one pad element per 2^LB
// (16; 32 for the radix-32 steps of complex128 1024-point lines, whose step-0
// writes are 32 elements apart -- psi_pad_shift on the host).
template <int LB> __device__ __forceinline__ int swz(int i) { return i + (i >> LB); }
// log2 of the points per thread (psi_log_p on the host)
template <typename V, int LR> __host__ __device__ constexpr int lp_of() {
    return ((std::is_same<V, double2>::value || std::is_same<V, float2>::value) && (LR == 9 || LR == 10)) ? 5
                                                                                            : (LR < 4 ? LR : 4);
}

struct alignas(64) KArgs {
    // line-fast L2 prefetch (MOA_FFT_PF_LF): tensor map of the load side, boxes
    // of W lines x 256 points -- one prefetch instruction per box instead of one
    // per 128-byte run
    CUtensorMap pf_tmap;
    // TMA store of a line-fast store side (MOA_FFT_TMA_ST, pass_kernel_st):
    // tensor map over the output, boxes of W lines x 256 points
    CUtensorMap st_tmap;
    int32_t pf_rank, pf_nbox, pf_box_pts, pf_ext0;
    int32_t st_rank, st_nbox, st_box_pts;
    const void *in;
    void *out;
    int64_t in_str[kMaxDigits], out_str[kMaxDigits], tw_str[kMaxDigits];
    int32_t lext[kMaxDigits];  // log2 extents
    int32_t ndig;
    int64_t in_kstr, out_kstr;
    const void *twR, *tw_hi, *tw_lo, *twS;
    int64_t twmask;  // twN - 1 (0: no twiddle)
    int64_t tw_off;  // exponent base offset (processor-level lifting)
    int32_t twh;     // split bit of the two-level table
    int32_t ksplit;  // store: k = khi 2^ksplit + klo
    int64_t out_kstr_hi;
    int32_t nodft;  // moa_pass_desc_t kind == 1
    int32_t W, LS;   // lines per tile, smem line stride (elements)
    int32_t lW;      // log2(W)
    int32_t lf_load, lf_store;
    int32_t ring;     // 0: HBM both sides; 1: loads from the L2 ring; 2: stores to the ring
    int32_t discard;  // ring == 1: discard the consumed ring lines (no write-back)
    int32_t conj_in, conj_out;  // inverse transform: conjugate loads / results (PassMods)
    double scale;               // results times scale (1: none)
    int32_t npeers;             // fused exchange: stores go to peers[q >> log_chunk] (PassMods)
    int32_t log_chunk;
    int64_t self_off;
    void *peers[8];
    // L2 prefetch ahead (MOA_FFT_PF): at its start a CTA asks the L2 for the
    // input footprint of tile blockIdx.x + pf_dist (about one wave of resident
    // CTAs ahead), so that tile's loads hit L2 instead of waiting on DRAM --
    // the paper's "pre-fetching becomes a deterministic cost"
    int64_t pf_dist, ntiles;
    // cluster-level lifting (cluster_kernel): a group of 2^ds_lg elements is
    // spread over the cluster's CTAs, 2^ds_lc elements in each one's shared memory
    int32_t ds_lg, ds_lc;
    int32_t ds_local;  // ablation (MOA_FFT_CLUSTER_LOCAL=1, wrong results): stores stay in the own CTA
};

__device__ __forceinline__ void line_offsets(const KArgs &a, int64_t line, int64_t &io, int64_t &oo, int64_t &te) {
    io = 0;
    oo = 0;
    te = 0;
#pragma unroll
    for (int i = 0; i < kMaxDigits; i++) {
        if (i < a.ndig) {
            const int64_t d = line & ((int64_t(1) << a.lext[i]) - 1);
            line >>= a.lext[i];
            io += d * a.in_str[i];
            oo += d * a.out_str[i];
            te += d * a.tw_str[i];
        }
    }
}

// store offset of DFT output k (the ONF's k loop, optionally split in two)
__device__ __forceinline__ int64_t kaddr(const KArgs &a, int k) {
    return int64_t(k & ((1 << a.ksplit) - 1)) * a.out_kstr + int64_t(k >> a.ksplit) * a.out_kstr_hi;
}

// 128-bit / 64-bit global accesses with an L2 eviction-policy operand, so the
// streaming HBM side (evict_normal) and the L2 ring (evict_last) share one
// code path; loads bypass L1 (.cg): ring slots are rewritten by other SMs.
// (The streaming side was evict_first until round 2, session 2: evict_normal
// measured cfg4 10.93 -> 10.78 ms, cfg3 -0.4 ... -1.3 %, cfg2 / cfg5 within
// noise -- the strided first passes' 128-byte runs share DRAM fetches with
// the neighbouring tile's, which evict_first dropped early;
// profiles/r5w_policy.jsonl, r5x2_policy.jsonl.)
__device__ __forceinline__ uint64_t l2_policy(bool keep) {
    uint64_t p;
    if (keep) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double2 ld_pol(const double2 *p, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.cg.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float2 ld_pol(const float2 *p, uint64_t pol) {
    float2 v;
    asm volatile("ld.global.cg.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;" : "=f"(v.x), "=f"(v.y) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float4 ld_pol(const float4 *p, uint64_t pol) {
    float4 v;
    asm volatile("ld.global.cg.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_pol(float4 *p, float4 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void st_pol(double2 *p, double2 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_pol(float2 *p, float2 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(v.x), "f"(v.y), "l"(pol) : "memory");
}

// Distributed shared memory (the cluster level of the lifting): a store into
// the shared memory of cluster CTA `rank` at the CTA-local address `la`, and
// the cluster-wide barrier (release / acquire: the stores before it are
// visible to every CTA of the cluster after it).
__device__ __forceinline__ uint32_t cl_map(uint32_t la, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(la), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster(uint32_t ra, double2 v) {
    asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(ra), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void st_cluster(uint32_t ra, float2 v) {
    asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(ra), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// the same without the release fence: only orders this CTA's completed
// shared-memory reads (values already in registers) before the other CTAs'
// later stores into it (a write-after-read hazard, no data to publish)
__device__ __forceinline__ void cluster_sync_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}

// One Stockham step of radix Q = 2^LQ on a line of R = 2^LR points held as
// P = 2^LP registers per thread (thread t holds points t + m R/P).  NS = 2^LNS
// is the product of the previous radices.  Group j (= t + u R/P) reads points
// j + r R/Q, multiplies by w_{NS Q}^{(j mod NS) r}, transforms, and writes to
// (j / NS) NS Q + (j mod NS) + r NS (the self-sorting index map).
template <int LR, int LP, int LQ, int LNS, bool LAST, int LB, typename V>
__device__ __forceinline__ void stockham_step(V (&pts)[1 << LP], V *sm_line, int t,
                                              const typename ElemOf<V>::type *__restrict__ twR) {
    constexpr int R = 1 << LR, P = 1 << LP, Q = 1 << LQ, NS = 1 << LNS, G = P / Q;
#pragma unroll
    for (int u = 0; u < G; u++) {
        const int j = t + u * (R / P);
        V v[Q];
#pragma unroll
        for (int r = 0; r < Q; r++) v[r] = pts[u + r * G];
        if constexpr (NS > 1 && Q >= 4 && std::is_same<V, double2>::value) {
            // complex128 step twiddles w^r, w = w_{NS Q}^{jm}: one table load (entry
            // NS + jm - 1 of the step-major table) and the powers as products A[a] B[b]
            // (r = 4a + b, B[b] = w^b, A[a] = w^{4a}; <= 5 factors deep, ~1e-15) --
            // measured: the 15 loads per group were ~1/5 of the L1 data-pipe traffic of
            // the 1024-point passes (3-D passes 6.9 -> 6.5-6.8 ms).  complex64 keeps
            // the table loads (its passes are issue-bound; the products cost more)
            using E = typename ElemOf<V>::type;
            const int jm = j & (NS - 1);
            const E w1 = __ldg(twR + (NS + jm - 1));
            const E w2 = cmul(w1, w1), w3 = cmul(w2, w1), w4 = cmul(w2, w2);
            const E B[4] = {w1, w1, w2, w3};  // B[0] unused
            E A = w4;
#pragma unroll
            for (int a = 0; a < Q / 4; a++) {
#pragma unroll
                for (int b = 0; b < 4; b++) {
                    const int r = 4 * a + b;
                    if (r == 0) continue;
                    v[r] = cmul(v[r], a == 0 ? B[b] : (b == 0 ? A : cmul(A, B[b])));
                }
                if (a > 0 && a + 1 < Q / 4) A = cmul(A, w4);
            }
        } else if constexpr (NS > 1) {
            const int jm = j & (NS - 1);
#pragma unroll
            // step twiddle w_{NS Q}^{jm r} from the step-major table (entry r NS + jm - 1):
            // the lanes of a warp read consecutive (or equal) entries
            for (int r = 1; r < Q; r++) v[r] = cmul(v[r], __ldg(twR + (r * NS + jm - 1)));
        }
        dft_reg<LQ>(v);
        if constexpr (!LAST) {
            const int base = ((j >> LNS) << (LNS + LQ)) + (j & (NS - 1));
#pragma unroll
            for (int r = 0; r < Q; r++) sm_line[swz<LB>(base + r * NS)] = v[r];
        } else {
#pragma unroll
            for (int r = 0; r < Q; r++) pts[u + r * G] = v[r];
        }
    }
}

// The steps of the line DFT.  Step 0 runs in the load mapping (line lA, index
// tA), every later step in the store mapping (lB, tB): between steps the data
// passes through shared memory anyway, so the thread <-> line assignment changes
// for free there and no extra transposition is needed for a strided side.
// Barrier of the threads that share a tile: the whole CTA (the plain pass
// kernel), or one consumer warp group of the warp-specialised kernel (a named
// barrier over its threads).
struct CtaSync {
    __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
struct GroupSync {
    int id, n;
    __device__ __forceinline__ void operator()() const { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
};
// Called once every thread of the tile has read the tile's shared memory for
// the last time (`synced`: a barrier to that effect has just completed): the
// warp-specialised kernel hands the stage back to its TMA producer there.
struct NoFree {
    __device__ __forceinline__ void operator()(bool) const {}
};

template <int LR, int LP, int LB, int S, int NSTEP, typename V, typename Sync, typename OnFree>
__device__ __forceinline__ void line_fft(V (&pts)[1 << LP], V *sm, int LS, int lA, int tA, int lB, int tB,
                                         const typename ElemOf<V>::type *__restrict__ twR, const Sync &sync,
                                         const OnFree &on_free) {
    // radix P for every step but the last, which takes the remainder (so step 0,
    // whose writes are strided by its radix, always has radix 16)
    constexpr int LQL = LR - LP * (NSTEP - 1);
    constexpr int R = 1 << LR, P = 1 << LP;
    constexpr int LQ = S == NSTEP - 1 ? LQL : LP;
    constexpr int LNS = LP * S;
    constexpr bool LAST = S == NSTEP - 1;
    if constexpr (S == 0) stockham_step<LR, LP, LQ, LNS, LAST, LB>(pts, sm + lA * LS, tA, twR);
    else stockham_step<LR, LP, LQ, LNS, LAST, LB>(pts, sm + lB * LS, tB, twR);
    if constexpr (!LAST) {
        sync();
        const V *sl = sm + lB * LS;
#pragma unroll
        for (int m = 0; m < P; m++) pts[m] = sl[swz<LB>(tB + m * (R / P))];
        sync();
        if constexpr (S + 1 == NSTEP - 1) on_free(true);  // no shared-memory access after this
        line_fft<LR, LP, LB, S + 1, NSTEP>(pts, sm, LS, lA, tA, lB, tB, twR, sync, on_free);
    }
}

__device__ __forceinline__ double2 cvt_tw(double2 w, double2) { return w; }
__device__ __forceinline__ float2 cvt_tw(double2 w, float2) { return make_float2(float(w.x), float(w.y)); }

// w_N^e from the two-level double-precision table (exact integer exponent)
__device__ __forceinline__ double2 tw_lookup(const double2 *__restrict__ hi, const double2 *__restrict__ lo, int64_t e,
                                             int h) {
    return cmul(__ldg(hi + (e >> h)), __ldg(lo + (e & ((int64_t(1) << h) - 1))));
}

// Thread mappings of a tile.  Point-fast: lanes over the points of one line (a
// side whose points are contiguous).  Line-fast: lanes over the W adjacent
// lines (a strided side: each warp request covers whole 128-byte runs).  A is
// the load side's mapping, B the store side's.
struct TileMap {
    int lA, tA, lB, tB;
};
template <int TPL> __device__ __forceinline__ TileMap tile_map(const KArgs &a, int tid) {
    TileMap m;
    m.lA = a.lf_load ? tid & (a.W - 1) : tid / TPL;
    m.tA = a.lf_load ? tid >> a.lW : tid % TPL;
    m.lB = a.lf_store ? tid & (a.W - 1) : tid / TPL;
    m.tB = a.lf_store ? tid >> a.lW : tid % TPL;
    return m;
}

// The rest of a tile once its points are in registers (mapping A): block
// butterflies, lifted weights, store.  ring >= 0: the ring slot of this
// tile's group (the L2-staged intermediate of a fused pass pair, see
// pair_kernel); the ring side's address gets slot * ringG added.
// kFull: the L2-ring (fused pair) and fused-exchange (peer store) paths are
// compiled in; the plain pass kernel is built without them (their switched-off
// branches cost the default path ~1 %, profiles/r3s_noopt.jsonl)
template <typename V, int LR, typename Sync = CtaSync, typename OnFree = NoFree,
          bool kEarlyTw = std::is_same<V, double2>::value, bool kFull = true, bool kDs = false, bool kSt = false>
__device__ __forceinline__ void tile_compute(const KArgs &a, int64_t line0, V *sm, int64_t ring_off,
                                             V (&pts)[1 << lp_of<V, LR>()], int64_t b_io, int64_t b_oo,
                                             int64_t b_te, int tid, const Sync &sync = Sync(),
                                             const OnFree &on_free = OnFree()) {
    (void)line0;
    constexpr int LP = lp_of<V, LR>();
    constexpr int P = 1 << LP, R = 1 << LR, TPL = R / P;
    constexpr int LB = LP == 5 ? 5 : 4;  // shared-memory pad period (log2)
    constexpr int NSTEP = LR == 0 ? 1 : (LR + LP - 1) / LP;
    using E = typename ElemOf<V>::type;
    constexpr int LPL = lines_per_lane<V>();  // lines per lane (2: paired complex64)
    E *__restrict__ out = reinterpret_cast<E *>(a.out);
    const E *__restrict__ twR = reinterpret_cast<const E *>(a.twR);
    const TileMap mp = tile_map<TPL>(a, tid);
    const int lA = mp.lA, tA = mp.tA, lB = mp.lB, tB = mp.tB;

    // The lifted weights' two-level table entries (step 3 forms their
    // products).  complex128: fetched here, ahead of the butterflies, so their
    // L2 latency (2^28-point plans: 256 KiB tables) hides behind the block DFT
    // (measured cfg3 5.25 -> 5.13 ms, 3-D 19.2 -> 18.8 ms; no occupancy cost at
    // 2 CTAs/SM).  complex64: fetched in step 3 -- holding them costs 9
    // registers and one CTA per SM (64 -> 73; cfg4 11.2 -> 12.0 ms).
    const int64_t te = b_te + int64_t(LPL * lB) * a.tw_str[0];
    double2 tq[LPL][4];
    auto fetch_tw = [&]() {
        const double2 *__restrict__ hi = reinterpret_cast<const double2 *>(a.tw_hi);
        const double2 *__restrict__ lo = reinterpret_cast<const double2 *>(a.tw_lo);
        const int64_t lmask = (int64_t(1) << a.twh) - 1;
#pragma unroll
        for (int q = 0; q < LPL; q++) {  // the pair's second line has its own exponent base
            const int64_t e0 = te + a.tw_off + q * a.tw_str[0];
            const int64_t ea = (e0 * tB) & a.twmask, eb = (e0 * TPL) & a.twmask;
            tq[q][0] = __ldg(hi + (ea >> a.twh));
            tq[q][1] = __ldg(lo + (ea & lmask));
            tq[q][2] = __ldg(hi + (eb >> a.twh));
            tq[q][3] = __ldg(lo + (eb & lmask));
        }
    };
    if constexpr (kEarlyTw) {
        if (a.twmask) fetch_tw();
    }

    // ---- 2. block butterflies (R-point DFT of every line); the mapping switches
    //         from A to B at the first shared-memory exchange
    bool moved = false;
    if constexpr (LR > 0 && NSTEP > 1) {
        if (!a.nodft) {
            line_fft<LR, LP, LB, 0, NSTEP>(pts, sm, a.LS, lA, tA, lB, tB, twR, sync, on_free);
            moved = true;
        }
    } else if constexpr (LR > 0) {
        if (!a.nodft) dft_reg<LR>(pts);
    }
    if (!moved && a.lf_load != a.lf_store) {  // single step: explicit transposition A -> B
        V *sl = sm + lA * a.LS;
#pragma unroll
        for (int m = 0; m < P; m++) sl[swz<LB>(tA + m * TPL)] = pts[m];
        sync();
        const V *sl2 = sm + lB * a.LS;
#pragma unroll
        for (int m = 0; m < P; m++) pts[m] = sl2[swz<LB>(tB + m * TPL)];
        on_free(false);
    } else if (!moved) {
        on_free(false);
    }

    // ---- ring: every thread has consumed its loads (the exchanges above, or the
    //      barrier here); drop the ring lines this tile read from L2 without a
    //      write-back (discard.global.L2): the intermediate never reaches HBM
    if (kFull && LPL == 1 && a.ring == 1 && a.discard) {
        sync();
        constexpr int EPL = 128 / int(sizeof(V));  // elements per 128-byte line
        const int64_t io = b_io + int64_t(lA) * a.in_str[0] + ring_off;
        const E *in = reinterpret_cast<const E *>(a.in);
#pragma unroll
        for (int m = 0; m < P; m++) {
            const E *p = in + io + int64_t(tA + m * TPL) * a.in_kstr;
            if ((reinterpret_cast<uintptr_t>(p) & 127) == 0 && (a.in_kstr != 1 || ((tA + m * TPL) % EPL) == 0))
                asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
        }
    }

    // ---- 3. lifted weights w_N^{(e k) mod N} for k = tB + m R/P: one two-level
    //         lookup for k = tB, one for the increment, then a multiplicative chain
    //         in double precision (<= 15 products, ~1e-15 relative)
    // (the W lines of a tile share every digit but digit 0, which W divides)
    int64_t oo = b_oo + int64_t(LPL * lB) * a.out_str[0];
    if (kFull && a.ring == 2) oo += ring_off;
    if (a.twmask) {
        if constexpr (!kEarlyTw) fetch_tw();
        double2 w = cmul(tq[0][0], tq[0][1]);
        const double2 ws = cmul(tq[0][2], tq[0][3]);
        if constexpr (LPL == 1) {
            // w ws^m for m = PB a + b as A[a] B[b] with A[a] = w (ws^PB)^a and
            // B[b] = ws^b: a dependent depth of ~PA + 2 products instead of the
            // P - 1 of a plain chain (measured: the chain's latency was 8 % of
            // cfg2's first pass).  complex64 runs it in fp32 from the fp64-exact
            // endpoints (<= 6 products per weight, ~1e-6 against 2e-5); complex128
            // in fp64 (~1e-15)
            using W = typename std::conditional<std::is_same<V, float2>::value, float2, double2>::type;
            constexpr int PB = P < 4 ? P : 4, PA = P / PB;
            const W w0 = cvt_tw(w, W{}), s1 = cvt_tw(ws, W{});
            W B[PB];
            B[0] = mk<W>(1, 0);
            if constexpr (PB > 1) B[1] = s1;
            if constexpr (PB > 2) B[2] = cmul(s1, s1);
            if constexpr (PB > 3) B[3] = cmul(B[2], s1);
            const W sPB = PB > 3 ? cmul(B[2], B[2]) : (PB > 1 ? cmul(B[PB - 1], s1) : s1);
            W A = w0;
#pragma unroll
            for (int ai = 0; ai < PA; ai++) {
#pragma unroll
                for (int b = 0; b < PB; b++) pts[ai * PB + b] = cmul(pts[ai * PB + b], b ? cmul(A, B[b]) : A);
                if (ai + 1 < PA) A = cmul(A, sPB);
            }
        } else {  // the pair: the second line's chain
            double2 w1 = cmul(tq[1][0], tq[1][1]);
            const double2 ws1 = cmul(tq[1][2], tq[1][3]);
#pragma unroll
            for (int m = 0; m < P; m++) {
                pts[m] = cmul(pts[m], make_float4(float(w.x), float(w.y), float(w1.x), float(w1.y)));
                if (m + 1 < P) {
                    w = cmul(w, ws);
                    w1 = cmul(w1, ws1);
                }
            }
        }
    }

    // ---- inverse / normalisation modifiers of the plan's last pass
    if (a.conj_out || a.scale != 1.0) {
        using T = typename RealOf<V>::type;
        const T sr = T(a.scale), si = a.conj_out ? -T(a.scale) : T(a.scale);
#pragma unroll
        for (int m = 0; m < P; m++) {
            if constexpr (LPL == 1) pts[m] = mk<V>(pts[m].x * sr, pts[m].y * si);
            else pts[m] = make_float4(pts[m].x * sr, pts[m].y * si, pts[m].z * sr, pts[m].w * si);
        }
    }

    // ---- 4. store (128-bit; streaming to HBM, normal (L2-resident) to the ring)
    if constexpr (kDs) {
        // cluster level (cluster_kernel): the result goes straight into the
        // shared memory of the cluster CTA whose pass-B tile reads it --
        // position q of the group lives in CTA q >> ds_lc at offset q mod 2^ds_lc.
        // First every CTA of the cluster must be done with its own shared memory
        // (the block DFT's last exchange ended with a CTA barrier after its reads).
        cluster_sync_relaxed();
        const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
        const int64_t gmask = (int64_t(1) << a.ds_lg) - 1, lmask = (int64_t(1) << a.ds_lc) - 1;
        uint32_t own;
        asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(own));
#pragma unroll
        for (int m = 0; m < P; m++) {
            const int64_t q =
                (oo + (a.ksplit >= LR ? int64_t(tB + m * TPL) * a.out_kstr : kaddr(a, tB + m * TPL))) & gmask;
            const uint32_t rank = a.ds_local ? own : uint32_t(q >> a.ds_lc);
            st_cluster(cl_map(base + uint32_t(q & lmask) * uint32_t(sizeof(V)), rank), pts[m]);
        }
        return;
    }
    if constexpr (kSt) {
        // TMA store (MOA_FFT_TMA_ST): the tile is staged in shared memory in the
        // output's order -- point k of line l at k W + l, i.e. W-element runs,
        // consecutive lanes at consecutive addresses -- and leaves as
        // R / 256 tensor-map boxes (W lines x 256 points) through the TMA
        // (cp.async.bulk.tensor ... global.shared::cta), so the SM issues no
        // per-point stores: the transposed side's runs go out as bulk writes.
        sync();  // every thread's last exchange reads are done
#pragma unroll
        for (int m = 0; m < P; m++) sm[(tB + m * TPL) * a.W + lB] = pts[m];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        sync();
        if (tid < a.st_nbox) {
            int32_t c[5] = {0, 0, 0, 0, 0};
            int64_t rest = line0;
            c[0] = int32_t(2 * (rest % a.pf_ext0));
            rest /= a.pf_ext0;
            for (int i = 1; i < a.ndig && i + 1 < 5; i++) {
                c[i + 1] = int32_t(rest & ((int64_t(1) << a.lext[i]) - 1));
                rest >>= a.lext[i];
            }
            c[1] = tid * a.st_box_pts;
            const uint64_t t = reinterpret_cast<uint64_t>(&a.st_tmap);
            const uint32_t src = static_cast<uint32_t>(__cvta_generic_to_shared(sm + int64_t(tid) * a.st_box_pts * a.W));
            switch (a.st_rank) {
                case 2:
                    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(t),
                                 "r"(c[0]), "r"(c[1]), "r"(src)
                                 : "memory");
                    break;
                case 3:
                    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(t),
                                 "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(src)
                                 : "memory");
                    break;
                case 4:
                    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(t),
                                 "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(src)
                                 : "memory");
                    break;
                default:
                    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(t),
                                 "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(src)
                                 : "memory");
                    break;
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            // the CTA's shared memory must outlive the TMA's reads of it
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        return;
    }
    if (kFull && a.npeers) {  // fused all-to-all: send-layout offset q -> peer q / chunk (NVLink store)
        const uint64_t pol = l2_policy(false);
        const int64_t cmask = (int64_t(1) << a.log_chunk) - 1;
#pragma unroll
        for (int m = 0; m < P; m++) {
            const int64_t q = oo + (a.ksplit >= LR ? int64_t(tB + m * TPL) * a.out_kstr : kaddr(a, tB + m * TPL));
            E *dst = reinterpret_cast<E *>(a.peers[q >> a.log_chunk]) + a.self_off + (q & cmask);
            st_pol(reinterpret_cast<V *>(dst), pts[m], pol);
        }
        // the peer stores are ordered at system scope before this grid is seen
        // as finished by the stream-ordered barrier collective that follows
        // (DistStep kind 3; the readers run after it): one fence per CTA, after
        // the barrier -- the fence is cumulative over the CTA's stores that the
        // barrier ordered before it (per-thread fences cost 8 % in the loopback)
        sync();
        if (tid == 0) __threadfence_system();
        return;
    }
    {
        const uint64_t pol = l2_policy(kFull && a.ring == 2);
        if (a.ksplit >= LR) {  // the common case: one affine stride per point
            char *ptr = reinterpret_cast<char *>(out + oo + int64_t(tB) * a.out_kstr);
            const int64_t stepb = int64_t(TPL) * a.out_kstr * int64_t(sizeof(E));
#pragma unroll
            for (int m = 0; m < P; m++) {
                st_pol(reinterpret_cast<V *>(ptr), pts[m], pol);
                ptr += stepb;
            }
        } else {
#pragma unroll
            for (int m = 0; m < P; m++) st_pol(reinterpret_cast<V *>(out + oo + kaddr(a, tB + m * TPL)), pts[m], pol);
        }
    }
}

// Bulk L2 prefetch of `bytes` (multiple of 16) at p (16-byte aligned).
__device__ __forceinline__ void l2_prefetch(const void *p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Prefetch the input footprint of the tile starting at line `line0` into L2:
// a line-fast side with adjacent lines (one W-line run per point) or a
// point-fast side with contiguous points (one run per line).
template <typename V, int LR>
__device__ __forceinline__ void prefetch_tile(const KArgs &a, int64_t line0) {
    using E = typename ElemOf<V>::type;
    constexpr int R = 1 << LR;
    constexpr int LPL = lines_per_lane<V>();
    int64_t io, oo, te;
    line_offsets(a, line0, io, oo, te);
    const E *in = reinterpret_cast<const E *>(a.in) + io;
    const int lines = a.W * LPL;
    if (a.lf_load && a.in_str[0] == 1) {
        const uint32_t run = uint32_t(lines * int(sizeof(E)));
        for (int k = threadIdx.x; k < R; k += blockDim.x) l2_prefetch(in + int64_t(k) * a.in_kstr, run);
    } else if (!a.lf_load && a.in_kstr == 1) {
        for (int l = threadIdx.x; l < lines; l += blockDim.x) l2_prefetch(in + int64_t(l) * a.in_str[0], uint32_t(R * sizeof(E)));
    }
}

// Tensor-map L2 prefetch of box b of the tile starting at line `line0`
// (coordinates: 2 digit0 reals, point, digits 1..).
__device__ __forceinline__ void prefetch_tile_tensor(const KArgs &a, int64_t line0, int b) {
    int32_t c[5] = {0, 0, 0, 0, 0};
    int64_t rest = line0;
    c[0] = int32_t(2 * (rest % a.pf_ext0));
    rest /= a.pf_ext0;
    for (int i = 1; i < a.ndig && i + 1 < 5; i++) {
        c[i + 1] = int32_t(rest & ((int64_t(1) << a.lext[i]) - 1));
        rest >>= a.lext[i];
    }
    c[1] = b * a.pf_box_pts;
    const uint64_t t = reinterpret_cast<uint64_t>(&a.pf_tmap);
    switch (a.pf_rank) {
        case 2:
            asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(t), "r"(c[0]), "r"(c[1])
                         : "memory");
            break;
        case 3:
            asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(t), "r"(c[0]),
                         "r"(c[1]), "r"(c[2])
                         : "memory");
            break;
        case 4:
            asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(t), "r"(c[0]),
                         "r"(c[1]), "r"(c[2]), "r"(c[3])
                         : "memory");
            break;
        default:
            asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];" ::"l"(t),
                         "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4])
                         : "memory");
            break;
    }
}

// One tile with direct (register) loads -- the non-pipelined form.
template <typename V, int LR, bool kFull = true, bool kDs = false, bool kSt = false>
__device__ __forceinline__ void tile_body(const KArgs &a, int64_t line0, V *sm, int64_t ring_off) {
    constexpr int LP = lp_of<V, LR>();
    constexpr int P = 1 << LP, R = 1 << LR, TPL = R / P;
    using E = typename ElemOf<V>::type;
    constexpr int LPL = lines_per_lane<V>();
    if (a.pf_dist) {
        const int64_t nt = int64_t(blockIdx.x) + a.pf_dist;
        if (nt < a.ntiles) {
            if (a.pf_rank) {
                if (threadIdx.x < a.pf_nbox) prefetch_tile_tensor(a, nt * a.W * LPL, threadIdx.x);
            } else {
                prefetch_tile<V, LR>(a, nt * a.W * LPL);
            }
        }
    }
    const TileMap mp = tile_map<TPL>(a, threadIdx.x);
    int64_t b_io, b_oo, b_te;
    line_offsets(a, line0, b_io, b_oo, b_te);  // the tile's first line; line l adds l * str[0]
    int64_t io = b_io + int64_t(LPL * mp.lA) * a.in_str[0];
    if (kFull && a.ring == 1) io += ring_off;
    V pts[P];
    // ---- 1. load (128-bit; streaming from HBM, L2-only from the ring)
    {
        const uint64_t pol = l2_policy(kFull && a.ring == 1);
        // byte-pointer increments: one 64-bit add per point (the element-index
        // form costs an add and a scaled add per point)
        const char *ptr = reinterpret_cast<const char *>(reinterpret_cast<const E *>(a.in) + io + int64_t(mp.tA) * a.in_kstr);
        const int64_t stepb = int64_t(TPL) * a.in_kstr * int64_t(sizeof(E));
#pragma unroll
        for (int m = 0; m < P; m++) {
            pts[m] = ld_pol(reinterpret_cast<const V *>(ptr), pol);
            ptr += stepb;
        }
    }
    if (a.conj_in) {  // inverse transform: DFT of conj(x) (the plan's first pass)
#pragma unroll
        for (int m = 0; m < P; m++) {
            pts[m].y = -pts[m].y;
            if constexpr (LPL == 2) pts[m].w = -pts[m].w;
        }
    }
    tile_compute<V, LR, CtaSync, NoFree, std::is_same<V, double2>::value, kFull, kDs, kSt>(a, line0, sm, ring_off, pts, b_io, b_oo,
                                                                              b_te, threadIdx.x);
}

// ---------------------------------------------------------------------------
// Radix-32 steps on thread PAIRS with a warp-shuffle exchange (MOA_FFT_PAIR,
// complex128 512- and 1024-point lines): each thread holds 16 points instead
// of 32, so a CTA carries twice the warps at the same tile (the radix-32
// in-thread kernels run 8 warps per SM at ~190 registers and are bound by
// latency, profiles/r2b_cfg5_pass_ncu_full.txt).  A 32-point group j is split
// by the parity h of its input index: thread h holds x_{2m+h} (m < 16),
//   X[k' + 16 q] = E_0[k'] + (-1)^q w_32^{k'} E_1[k'],  E_h = DFT_16(x_{2m+h}),
// (decimation in time; cf. the radix-2 stage B_L of Fig. vanloan_fft
// P:1863-1873).  Thread 1 negates its odd inputs, so its DFT_16 comes out
// rotated by 8; both threads then keep registers 0..7 and swap 8..15 with the
// partner lane (8 complex values = 32 SHFL), and thread h finishes
// X[8h + i] and X[16 + 8h + i] for i < 8.
template <typename V> __device__ __forceinline__ V shfl_x(V v, int mask) {
    V r;
    r.x = __shfl_xor_sync(0xffffffffu, v.x, mask);
    r.y = __shfl_xor_sync(0xffffffffu, v.y, mask);
    return r;
}
template <int I, typename V> __device__ __forceinline__ void pair_tw(V (&v)[16]) {
    if constexpr (I < 8) {
        v[I] = rot32<8 + I>(v[I]);                  // E_1[8 + I] w_32^{8 + I}
        if constexpr (I > 0) v[8 + I] = rot32<I>(v[8 + I]);  // E_1[I] w_32^I
        pair_tw<I + 1>(v);
    }
}
template <typename V> __device__ __forceinline__ void dft32_pair(V (&v)[16], int h, int xmask) {
    if (h) {
#pragma unroll
        for (int m = 1; m < 16; m += 2) v[m] = mk<V>(-v[m].x, -v[m].y);
    }
    dft_reg<4>(v);
    if (h) pair_tw<0>(v);
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const V r = shfl_x(v[8 + i], xmask);
        const V s = cadd(v[i], r);
        V d = csub(v[i], r);
        if (h) d = mk<V>(-d.x, -d.y);
        v[i] = s;
        v[8 + i] = d;
    }
}

// The paired line DFT of R = 2^LR (9 or 10) points: step 0 (radix 32 on pairs)
// in the load mapping, the exchange through shared memory (pad one per 32),
// step 1 (R = 1024: radix 32 on pairs; R = 512: radix 16 in-thread, one group
// per thread) in the store mapping with the step twiddles w_{32 Q}^{j r}.
// Returns pts[m] = X[kb + s1 (m mod M1) + s2 (m / M1)] via kb / M1 / s1 / s2.
template <int LR, typename V, typename Sync, typename OnFree>
__device__ __forceinline__ void line_fft_pair(V (&pts)[16], V *sm, int LS, int lA, int pA, int xA, int lB, int pB,
                                              int xB, const V *__restrict__ twR, const Sync &sync,
                                              const OnFree &on_free) {
    constexpr int R = 1 << LR;
    {  // step 0: group j = pA / 2, inputs r = 2m + h (NS = 1): outputs at j 32 + r'
        const int j = pA >> 1, h = pA & 1;
        dft32_pair(pts, h, xA);
        V *sl = sm + lA * LS;
        const int base = j * 32 + 8 * h;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            sl[swz<5>(base + i)] = pts[i];
            sl[swz<5>(base + 16 + i)] = pts[8 + i];
        }
    }
    sync();
    const V *sl = sm + lB * LS;
    if constexpr (R == 1024) {
        const int j = pB >> 1, h = pB & 1;
#pragma unroll
        for (int m = 0; m < 16; m++) pts[m] = sl[swz<5>(j + (2 * m + h) * 32)];
        sync();
        on_free(true);
        // step twiddles w_1024^{j r}, r = 2m + h: w = w_1024^j (table entry NS + j - 1),
        // v[m] *= w^h (w^2)^m as products A[a] B'[b], m = 4a + b, B'[b] = w^h (w^2)^b
        if (j > 0) {
            const V w1 = __ldg(twR + (32 + j - 1));
            const V w2 = cmul(w1, w1);
            const V base = h ? w1 : mk<V>(1.0, 0.0);
            V B[4];
            B[0] = base;
            B[1] = cmul(base, w2);
            const V w4 = cmul(w2, w2);
            B[2] = cmul(base, w4);
            B[3] = cmul(B[2], w2);
            const V w8 = cmul(w4, w4);
            V A = w8;
#pragma unroll
            for (int a = 0; a < 4; a++) {
#pragma unroll
                for (int b = 0; b < 4; b++) pts[4 * a + b] = cmul(pts[4 * a + b], a == 0 ? B[b] : cmul(A, B[b]));
                if (a > 0 && a < 3) A = cmul(A, w8);
            }
        }
        dft32_pair(pts, h, xB);
    } else {  // R = 512: step 1 radix 16 in-thread, group j = pB (< 32), inputs j + 32 r
        const int j = pB;
#pragma unroll
        for (int m = 0; m < 16; m++) pts[m] = sl[swz<5>(j + m * 32)];
        sync();
        on_free(true);
        if (j > 0) {
            const V w1 = __ldg(twR + (32 + j - 1));
            const V w2 = cmul(w1, w1), w3 = cmul(w2, w1), w4 = cmul(w2, w2);
            const V B[4] = {w1, w1, w2, w3};
            V A = w4;
#pragma unroll
            for (int a = 0; a < 4; a++) {
#pragma unroll
                for (int b = 0; b < 4; b++) {
                    const int r = 4 * a + b;
                    if (r == 0) continue;
                    pts[r] = cmul(pts[r], a == 0 ? B[b] : (b == 0 ? A : cmul(A, B[b])));
                }
                if (a > 0 && a + 1 < 4) A = cmul(A, w4);
            }
        }
        dft_reg<4>(pts);
    }
}

// A tile of the paired variant: load (16 points per thread), line DFT, lifted
// weights, store -- the plain kernel's tile with the paired mappings.
template <typename V, int LR, typename Sync = CtaSync, typename OnFree = NoFree>
__device__ __forceinline__ void tile_pair(const KArgs &a, int64_t line0, V *sm, int tid, const Sync &sync = Sync(),
                                          const OnFree &on_free = OnFree()) {
    using T = typename RealOf<V>::type;
    constexpr int R = 1 << LR, P = 16, TPL = R / P;
    // mappings: line-fast (lanes over the W lines; partner lane ^ W) or
    // point-fast (lanes over the points; partner lane ^ 1)
    const int lA = a.lf_load ? tid & (a.W - 1) : tid / TPL, pA = a.lf_load ? tid >> a.lW : tid % TPL;
    const int lB = a.lf_store ? tid & (a.W - 1) : tid / TPL, pB = a.lf_store ? tid >> a.lW : tid % TPL;
    const int xA = a.lf_load ? a.W : 1, xB = a.lf_store ? a.W : 1;
    int64_t b_io, b_oo, b_te;
    line_offsets(a, line0, b_io, b_oo, b_te);
    // point index of register m in the load mapping: j + h R/32 + m R/16
    const int tA = (pA >> 1) + (pA & 1) * (R / 32);
    V pts[P];
    {
        const uint64_t pol = l2_policy(false);
        const int64_t io = b_io + int64_t(lA) * a.in_str[0];
        const char *ptr = reinterpret_cast<const char *>(reinterpret_cast<const V *>(a.in) + io + int64_t(tA) * a.in_kstr);
        const int64_t stepb = int64_t(TPL) * a.in_kstr * int64_t(sizeof(V));
#pragma unroll
        for (int m = 0; m < P; m++) {
            pts[m] = ld_pol(reinterpret_cast<const V *>(ptr), pol);
            ptr += stepb;
        }
    }
    if (a.conj_in) {
#pragma unroll
        for (int m = 0; m < P; m++) pts[m].y = -pts[m].y;
    }
    const V *twR = reinterpret_cast<const V *>(a.twR);
    line_fft_pair<LR>(pts, sm, a.LS, lA, pA, xA, lB, pB, xB, twR, sync, on_free);
    // output index of register m: kb + S1 (m mod M1) + S2 (m / M1)
    constexpr int S1 = 32, M1 = R == 1024 ? 8 : 16, S2 = 512;
    const int kb = R == 1024 ? (pB >> 1) + 256 * (pB & 1) : pB;
    // ---- lifted weights w_N^{(e k) mod N}: w_N^{e kb} (w_N^{e S1})^i (w_N^{e S2})^{m / M1}
    int64_t oo = b_oo + int64_t(lB) * a.out_str[0];
    if (a.twmask) {
        const double2 *__restrict__ hi = reinterpret_cast<const double2 *>(a.tw_hi);
        const double2 *__restrict__ lo = reinterpret_cast<const double2 *>(a.tw_lo);
        const int64_t lmask = (int64_t(1) << a.twh) - 1;
        const int64_t e0 = b_te + int64_t(lB) * a.tw_str[0] + a.tw_off;
        auto tw = [&](int64_t e) {  // fp64 table product, rounded to V's precision
            e &= a.twmask;
            return cvt_tw(cmul(__ldg(hi + (e >> a.twh)), __ldg(lo + (e & lmask))), V{});
        };
        const V w = tw(e0 * kb), s1 = tw(e0 * S1);
        V start[P / M1];
        start[0] = w;
        if constexpr (P / M1 > 1) start[1] = cmul(w, tw(e0 * S2));
        const V s2 = cmul(s1, s1), s3 = cmul(s2, s1), s4 = cmul(s2, s2);
        const V B[4] = {mk<V>(1.0, 0.0), s1, s2, s3};
#pragma unroll
        for (int hlf = 0; hlf < P / M1; hlf++) {
            V A = start[hlf];
#pragma unroll
            for (int ai = 0; ai < M1 / 4; ai++) {
#pragma unroll
                for (int b = 0; b < 4; b++) {
                    const int m = hlf * M1 + ai * 4 + b;
                    pts[m] = cmul(pts[m], b ? cmul(A, B[b]) : A);
                }
                if (ai + 1 < M1 / 4) A = cmul(A, s4);
            }
        }
    }
    if (a.conj_out || a.scale != 1.0) {
        const T sr = T(a.scale), si = a.conj_out ? -T(a.scale) : T(a.scale);
#pragma unroll
        for (int m = 0; m < P; m++) pts[m] = mk<V>(pts[m].x * sr, pts[m].y * si);
    }
    // ---- store
    const uint64_t pol = l2_policy(false);
    V *out = reinterpret_cast<V *>(a.out);
#pragma unroll
    for (int m = 0; m < P; m++) {
        const int k = kb + S1 * (m % M1) + S2 * (m / M1);
        const int64_t off = a.ksplit >= LR ? int64_t(k) * a.out_kstr : kaddr(a, k);
        st_pol(out + oo + off, pts[m], pol);
    }
}

template <typename V, int LR>
__global__ void __launch_bounds__(std::is_same<V, double2>::value ? 512 : 1024, 1) pass_kernel_pair(const KArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    tile_pair<V, LR>(a, int64_t(blockIdx.x) * a.W, reinterpret_cast<V *>(smem_raw), threadIdx.x);
}

// (complex128 radix-32 kernels: at most 256 threads, so 255 registers -- a cap of
// 168 for three CTAs per SM spills and measured slower, profiles/r1_s7_radix32.txt;
// complex64 ones fit 512 threads at 128 registers: 16-line tiles, 128-byte runs;
// complex64 lines of <= 256 points keep two 512-thread CTAs per SM)
// (complex64 kernels of <= 16 points per thread: <= 64 registers, i.e. two
// 512-thread CTAs or one 1024-thread CTA per SM -- the 1024-thread tiles of the
// >= 2^11-point transposing passes, psi_choose_tile)
template <typename V, int LR> constexpr int pass_max_threads() {
    return (lp_of<V, LR>() == 5 && std::is_same<V, double2>::value) ? 256
           : (std::is_same<V, float2>::value && lp_of<V, LR>() <= 4) ? 1024
                                                                      : 512;
}
template <typename V, int LR, bool kFull = false>
__global__ void __launch_bounds__(pass_max_threads<V, LR>(), 1) pass_kernel(const __grid_constant__ KArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    tile_body<V, LR, kFull>(a, int64_t(blockIdx.x) * a.W * lines_per_lane<V>(), reinterpret_cast<V *>(smem_raw), 0);
}
// the plain pass with the TMA store of a line-fast store side (MOA_FFT_TMA_ST)
template <typename V, int LR>
__global__ void __launch_bounds__(pass_max_threads<V, LR>(), 1) pass_kernel_st(const __grid_constant__ KArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    tile_body<V, LR, false, false, true>(a, int64_t(blockIdx.x) * a.W, reinterpret_cast<V *>(smem_raw), 0);
}

// ---------------------------------------------------------------------------
// The cluster level of the lifting (MOA_FFT_CLUSTER): a two-pass lifting of
// independent groups (cfg2: rows of 2^16 = 256 x 256 points) whose group fits
// the shared memory of one thread-block cluster runs as ONE kernel, one HBM
// round trip: a cluster of C CTAs owns one group; CTA c runs pass A's tile c
// (loads from HBM, block DFTs, lifted weights) and stores its result straight
// into the shared memory of the CTA that needs it (distributed shared memory,
// the reshape-transpose of Eq. reshape3 P:2097-2114 done between SMs); after
// the cluster barrier CTA c runs pass B's tile c from its own shared memory
// and stores to HBM.  The paper's premise -- lift until a block fits one level
// of the hierarchy -- with the cluster as the level between one
// SM's shared memory and the L2.  The two passes may have different radices
// (R_A = 2^LRA, R_B = 2^LRB) with the same number of points per thread, so one
// CTA size serves both (psi_cluster_pair picks the tile widths).
template <typename V, int LRA, int LRB>
__global__ void __launch_bounds__(((lp_of<V, LRA>() == 5 || lp_of<V, LRB>() == 5) && std::is_same<V, double2>::value)
                                      ? 256
                                      : 512,
                                  1)
    cluster_kernel(const __grid_constant__ KArgs a, const __grid_constant__ KArgs b) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V *sm = reinterpret_cast<V *>(smem_raw);
    constexpr int LR = LRB;
    constexpr int LP = lp_of<V, LR>();
    constexpr int P = 1 << LP, R = 1 << LR, TPL = R / P;
    const int64_t tile = blockIdx.x;  // group tile / C, CTA rank tile % C (cluster dims (C, 1, 1))
    tile_body<V, LRA, false, true>(a, tile * a.W, sm, 0);
    cluster_sync_all();  // every pass-A store of the cluster has landed
    const TileMap mp = tile_map<TPL>(b, threadIdx.x);
    int64_t b_io, b_oo, b_te;
    line_offsets(b, tile * b.W, b_io, b_oo, b_te);
    // pass B's tile reads exactly this CTA's slice (checked on the host)
    const int64_t off = (b_io + int64_t(mp.lA) * b.in_str[0] + int64_t(mp.tA) * b.in_kstr) & ((int64_t(1) << b.ds_lc) - 1);
    V pts[P];
#pragma unroll
    for (int m = 0; m < P; m++) pts[m] = sm[off + int64_t(m) * TPL * b.in_kstr];
    __syncthreads();  // the block DFT's exchanges reuse the shared memory
    tile_compute<V, LR, CtaSync, NoFree, std::is_same<V, double2>::value, false, false>(b, tile * b.W, sm, 0, pts, b_io,
                                                                                     b_oo, b_te, threadIdx.x);
}

// ---------------------------------------------------------------------------
// Asynchronously fed pass kernel (MOA_FFT_WS): the loads of a tile are taken
// off the compute warps' critical path.  One persistent CTA per SM with a ring
// of S shared-memory stages, each fed by TMA -- a tensor-map box of W
// adjacent lines x 256 points per copy for a line-fast (strided) side
// (cp.async.bulk.tensor), one bulk copy per line for contiguous lines
// (cp.async.bulk) -- completing on the stage's mbarrier.  Two consumer warp
// groups take the stages' tiles alternately (tile sequence k = g, g + 2, ...):
// read the landed tile in the load mapping, run the block butterflies /
// lifted weights exactly as the plain kernel (tile_compute, with a named
// barrier over the group), reusing the stage as the exchange buffer, and store
// with 128-bit register stores.  The moment a group has read its stage for the
// last time it refills it with tile k + S (one elected thread issues the
// copies; no producer warp, so the kernel keeps the plain kernel's register
// budget).  Tiles come in order from an atomic counter (reset before every
// launch; fetched while the current tile computes), so the CTAs stay on
// neighbouring tiles and the DRAM access order matches the plain kernel's.
// The paper's prefetch argument: with the next tiles already in
// flight, "pre-fetching becomes a deterministic cost" off the critical path.
constexpr int kWsStagesMax = 4;
constexpr int kWsGroupMax = 128;  // threads per consumer group
// (the lifted-weight table entries are fetched after the butterflies: holding
// them across the DFT costs registers the stage pipeline already hides)
constexpr bool kWsEarlyTw = false;
struct alignas(64) WsArgs {
    CUtensorMap tmap;  // line-fast loads: dims (2 W-lines reals, points, line digits 1..)
    KArgs a;
    int64_t ntiles;
    unsigned long long *ctr;  // tile counter (null: static round-robin)
    int32_t stages, stage_elems, mode;  // mode 0: tensor-map boxes; 1: one bulk copy per line
    int32_t nbox, box_pts, tmap_rank;
    int32_t ext0;                        // extent of line digit 0 (tensor dims)
    uint32_t stage_bytes;                // bytes landed per tile
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *b, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
// (a watchdog turns a broken pipeline into a launch error instead of a hang)
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    uint32_t spins = 0;
    while (!mbar_try_wait(b, parity)) {
        if (++spins == (1u << 24)) {
            printf("moa ws watchdog: block %d thread %d barrier %p parity %u\n", blockIdx.x, threadIdx.x, (void *)b,
                   parity);
            __trap();
        }
    }
}
__device__ __forceinline__ void tma_bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tma_tensor_g2s(void *dst, const void *tmap, int rank, const int32_t (&c)[5], uint64_t *bar) {
    const uint32_t d = smem_u32(dst), b = smem_u32(bar);
    const uint64_t t = reinterpret_cast<uint64_t>(tmap);
    switch (rank) {
        case 2:
            asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(d),
                         "l"(t), "r"(c[0]), "r"(c[1]), "r"(b)
                         : "memory");
            break;
        case 3:
            asm volatile("cp.async.bulk.tensor.3d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(d),
                         "l"(t), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(b)
                         : "memory");
            break;
        case 4:
            asm volatile("cp.async.bulk.tensor.4d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(d),
                         "l"(t), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(b)
                         : "memory");
            break;
        default:
            asm volatile("cp.async.bulk.tensor.5d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(d),
                         "l"(t), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(b)
                         : "memory");
            break;
    }
}

// Tile index of the CTA's k-th tile: the counter (dynamic, in order) or static
// round-robin.
__device__ __forceinline__ int64_t ws_next_tile(const WsArgs &w, int64_t k) {
    if (w.ctr) return int64_t(atomicAdd(w.ctr, 1ull));
    return int64_t(blockIdx.x) + k * gridDim.x;
}

// Fill stage s with tile `tile` (or the end marker -1): the tile's copies
// complete on full[s] together with the arrival.
// tile_of[0] = the tile (-1: end), tile_of[1] = its sequence number k: a
// consumer checks k after the barrier, since a stage's consecutive rounds
// alternate between the two groups and a phase parity alone could alias a
// round two phases back.
template <typename V, int LR>
__device__ __forceinline__ void ws_fill(const WsArgs &w, V *stage, uint64_t *full, int64_t *tile_of, int64_t tile,
                                        int64_t k) {
    using E = typename ElemOf<V>::type;
    constexpr int R = 1 << LR;
    const KArgs &a = w.a;
    reinterpret_cast<volatile int64_t *>(tile_of)[1] = k;
    if (tile >= w.ntiles) {
        reinterpret_cast<volatile int64_t *>(tile_of)[0] = -1;
        mbar_arrive(full);
        return;
    }
    reinterpret_cast<volatile int64_t *>(tile_of)[0] = tile;
    mbar_arrive_tx(full, w.stage_bytes);
    const int64_t line0 = tile * a.W;
    if (w.mode == 0) {
        // coordinates: (2 digit0 reals, point, digit 1, ...)
        int32_t c[5] = {0, 0, 0, 0, 0};
        int64_t rest = line0;
        c[0] = int32_t(2 * (rest % w.ext0));
        rest /= w.ext0;
        for (int i = 1; i < a.ndig && i + 1 < 5; i++) {
            c[i + 1] = int32_t(rest & ((int64_t(1) << a.lext[i]) - 1));
            rest >>= a.lext[i];
        }
        for (int b = 0; b < w.nbox; b++) {
            c[1] = b * w.box_pts;
            tma_tensor_g2s(stage + size_t(b) * w.box_pts * a.W, &w.tmap, w.tmap_rank, c, full);
        }
    } else {
        int64_t io, oo, te;
        line_offsets(a, line0, io, oo, te);
        const E *in = reinterpret_cast<const E *>(a.in) + io;
        for (int l = 0; l < a.W; l++)
            tma_bulk_g2s(stage + size_t(l) * a.LS, in + int64_t(l) * a.in_str[0], uint32_t(R * sizeof(E)), full);
    }
}

// A consumer group's hand-back of its stage: every thread has read it for the
// last time; the generic-proxy accesses are ordered before the async-proxy
// (TMA) writes of the refill, which one elected thread then issues.
template <typename V, int LR>
struct WsRefill {
    const WsArgs *w;
    V *stage;
    uint64_t *full;
    int64_t *tile_of;
    int64_t next;  // the tile for this stage's next round (valid on gtid 0)
    int64_t knext;  // its sequence number
    GroupSync sync;
    int gtid;
    __device__ __forceinline__ void operator()(bool) const {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        sync();
        if (gtid == 0) ws_fill<V, LR>(*w, stage, full, tile_of, next, knext);
    }
};

template <typename V, int LR>
__global__ void __launch_bounds__(2 * kWsGroupMax, 1) ws_pass_kernel(const __grid_constant__ WsArgs w) {
    constexpr int LP = lp_of<V, LR>();
    constexpr int P = 1 << LP, R = 1 << LR, TPL = R / P;
    const KArgs &a = w.a;
    extern __shared__ __align__(128) unsigned char smem_ws[];
    unsigned char *smem_raw = smem_ws;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem_raw);
    int64_t *tile_of = reinterpret_cast<int64_t *>(full + kWsStagesMax);  // [stage][tile, k]
    V *stage0 = reinterpret_cast<V *>(smem_raw + 128);
    const int S = w.stages;
    const int nthr = a.W * TPL;  // threads per consumer group
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; s++) mbar_init(full + s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int s = 0; s < S; s++)
            ws_fill<V, LR>(w, stage0 + size_t(s) * w.stage_elems, full + s, tile_of + 2 * s, ws_next_tile(w, s), s);
    // ---- consumer group g takes the tiles k = g, g + 2, ...
    const int g = threadIdx.x >= nthr;
    const int gtid = threadIdx.x - g * nthr;
    const GroupSync gsync{1 + g, nthr};
    const TileMap mp = tile_map<TPL>(a, gtid);
    for (int64_t k = g;; k += 2) {
        const int s = int(k % S);
        V *sm = stage0 + size_t(s) * w.stage_elems;
        volatile int64_t *tag = tile_of + 2 * s;
        do {
            mbar_wait(full + s, uint32_t(k / S) & 1);
        } while (tag[1] != k);
        const int64_t tile = tag[0];
        gsync();  // every thread has read the tag before the stage can be refilled
        if (tile < 0) {  // pass the end marker on to the stage's next round, then stop
            if (gtid == 0) ws_fill<V, LR>(w, sm, full + s, tile_of + 2 * s, w.ntiles, k + S);
            break;
        }
        // this stage's next tile: fetched now, used at the refill (its latency
        // hides behind this tile's butterflies)
        const int64_t next = gtid == 0 ? ws_next_tile(w, k + S) : 0;
        const int64_t line0 = tile * a.W;
        int64_t b_io, b_oo, b_te;
        line_offsets(a, line0, b_io, b_oo, b_te);
        // the landed tile, in the load mapping: point tA + m TPL of line lA
        V pts[P];
        if (w.mode == 0) {
            const V *src = sm + mp.tA * a.W + mp.lA;
#pragma unroll
            for (int m = 0; m < P; m++) pts[m] = src[m * TPL * a.W];
        } else {
            const V *src = sm + mp.lA * a.LS + mp.tA;
#pragma unroll
            for (int m = 0; m < P; m++) pts[m] = src[m * TPL];
        }
        if (a.conj_in) {
#pragma unroll
            for (int m = 0; m < P; m++) pts[m].y = -pts[m].y;
        }
        gsync();  // every dense read done before the exchange reuses the stage
        tile_compute<V, LR, GroupSync, WsRefill<V, LR>, kWsEarlyTw>(
            a, line0, sm, 0, pts, b_io, b_oo, b_te, gtid, gsync,
            WsRefill<V, LR>{&w, sm, full + s, tile_of + 2 * s, next, k + S, gsync, gtid});
    }
}

// A fused pass pair: pass A writes its output to an L2-resident ring of
// `slots` group buffers, pass B reads it from there -- the lifting applied at
// the L2 level, so the intermediate never makes an HBM round trip (the
// paper's "each block fits one level of the hierarchy").
// Tiles are handed out in a fixed order by an atomic queue (A tiles of group g,
// interleaved with B tiles of group g - lag); a B tile waits for its group's A
// tiles, an A tile reusing a slot waits for the previous group's B tiles.
// Every waited-on tile was dequeued earlier by a running CTA, so the waits
// cannot deadlock (the decoupled look-back argument).
struct PairArgs {
    KArgs A, B;
    int64_t groups, ringG;
    int32_t TA, TB, lag, slot_mask;
    unsigned long long *qctr, *cntA, *cntB;
    unsigned long long epoch;
    unsigned long long *stats;  // optional wait statistics (6 counters), or null
};

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// position in the tile order -> (pass B?, group, tile in group)
__device__ __forceinline__ void decode_tile(const PairArgs &p, int64_t pos, bool &isB, int64_t &g, int64_t &idx) {
    const int64_t G = p.groups, L = p.lag, T = p.TA + p.TB;
    const int64_t n1 = (L < G ? L : G) * p.TA;
    if (pos < n1) {
        isB = false;
        g = pos / p.TA;
        idx = pos % p.TA;
        return;
    }
    pos -= n1;
    const int64_t n2 = G > L ? (G - L) * T : 0;
    if (pos < n2) {
        const int64_t s = L + pos / T, r = pos % T;
        isB = r >= p.TA;
        g = isB ? s - L : s;
        idx = isB ? r - p.TA : r;
        return;
    }
    pos -= n2;
    isB = true;
    g = (G > L ? G - L : 0) + pos / p.TB;
    idx = pos % p.TB;
}

// Persistent CTAs (grid = resident capacity): each loops over the tile queue,
// fetching its next tile index while it works on the current one, so the
// queue atomic's latency is hidden.
template <typename V, int LRA, int LRB>
__global__ void __launch_bounds__(((lp_of<V, LRA>() == 5 || lp_of<V, LRB>() == 5) && std::is_same<V, double2>::value) ? 256 : 512) pair_kernel(const __grid_constant__ PairArgs p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int64_t total = p.groups * (p.TA + p.TB);
    // the per-group completion counters only ever grow, by exactly TA / TB per launch
    const unsigned long long round = p.epoch + 1;
    V *sm = reinterpret_cast<V *>(smem_raw);
    // Deadlock freedom: every CTA is resident and every wait is on a smaller
    // position; the smallest unfinished position is some CTA's current (or
    // fetched-ahead) tile, whose dependencies are all finished and published
    // (a CTA publishes its previous tile before it ever spins).
    bool have_prev = false, prev_B = false;
    int64_t prev_g = 0;
    // Static round-robin over the tile order (tile pos -> CTA pos mod grid, each
    // CTA in increasing order; an atomic queue measured slower).
    for (int64_t pos = blockIdx.x; pos < total; pos += gridDim.x) {
        bool isB;
        int64_t g, idx;
        decode_tile(p, pos, isB, g, idx);
        bool signalled = false;  // (thread 0) the previous tile's completion already published
        if (threadIdx.x == 0) {
            // relaxed polling (no L1 invalidation per poll: every ring access is
            // an L2 (.cg) access); a watchdog turns a broken schedule into a
            // launch error instead of a hang.  A CTA never spins while holding
            // an unpublished completion (that could close a wait cycle), so the
            // previous tile is published first whenever a wait is needed.
            const unsigned long long *dep = nullptr;
            unsigned long long need = 0;
            if (isB) {
                dep = p.cntA + g;
                need = round * (unsigned long long)p.TA;
            } else if (g > p.slot_mask) {
                dep = p.cntB + g - (p.slot_mask + 1);
                need = round * (unsigned long long)p.TB;
            }
            if (dep && ld_relaxed(dep) >= need) {
                __threadfence();  // acquire: the producers' ring stores happen-before this tile's loads
            } else if (dep) {
                if (have_prev) {
                    __threadfence();
                    atomicAdd(prev_B ? p.cntB + prev_g : p.cntA + prev_g, 1ull);
                    signalled = true;
                }
                unsigned spins = 0;
                const long long t0 = p.stats ? clock64() : 0;
                while (ld_relaxed(dep) < need) {
                    __nanosleep(32);
                    if (++spins > (1u << 26)) __trap();
                }
                // acquire side of the producer's fence + atomicAdd (the relaxed polls
                // alone would not order this CTA's ring loads after the producer's stores)
                __threadfence();
                if (p.stats) {  // MOA_FFT_STATS: waits, spins, wait cycles
                    atomicAdd(p.stats + (isB ? 0 : 3), 1ull);
                    atomicAdd(p.stats + (isB ? 1 : 4), (unsigned long long)spins);
                    atomicAdd(p.stats + (isB ? 2 : 5), (unsigned long long)(clock64() - t0));
                }
            }
        }
        __syncthreads();
        // otherwise the previous tile (all its stores were issued before the two
        // barriers since) is published here, so the fence's latency overlaps
        // this tile's loads in the other warps instead of stalling the CTA
        if (threadIdx.x == 0 && have_prev && !signalled) {
            __threadfence();
            atomicAdd(prev_B ? p.cntB + prev_g : p.cntA + prev_g, 1ull);
        }
        const int64_t ring_off = (g & p.slot_mask) * p.ringG;
        if constexpr (LRA == LRB) {
            // one inlined tile body for both passes (the fused kernel otherwise
            // thrashes the instruction cache); the arguments are read in place
            // from the __grid_constant__ parameter block
            const KArgs &a = isB ? p.B : p.A;
            tile_body<V, LRA>(a, (g * (isB ? p.TB : p.TA) + idx) * a.W, sm, ring_off);
        } else {
            if (isB) tile_body<V, LRB>(p.B, (g * p.TB + idx) * p.B.W, sm, ring_off);
            else tile_body<V, LRA>(p.A, (g * p.TA + idx) * p.A.W, sm, ring_off);
        }
        __syncthreads();
        have_prev = true;
        prev_B = isB;
        prev_g = g;
    }
    if (threadIdx.x == 0 && have_prev) {
        __threadfence();
        atomicAdd(prev_B ? p.cntB + prev_g : p.cntA + prev_g, 1ull);
    }
}

// ---------------------------------------------------------------------------
// Latency form of a one-pass plan with few lines (cfg1: one 2^10-point
// transform).  One CTA per line, R/4 threads: radix-4 Stockham steps (the
// self-sorting form of the radix-2 network, Fig. vanloan_fft, two
// stages per step) ping-ponging between two shared-memory buffers, one barrier
// per step.  The step twiddles come from the plan's table (abi.cpp
// build_tables, twS: step s >= 1 with NS = 4^s holds w_{4 NS}^{k q} at
// (NS - 4) + (q - 1) NS + k, so a step's reads are unit-stride across the
// threads; an odd log2 R appends w_R^j at R/2 - 4 + j), copied to shared
// memory in the prologue with loads issued together with the line's, so the
// two DRAM latencies overlap and no twiddle is computed.  The first step runs
// straight from the loaded registers and the last one stores to global memory
// in natural order.
__device__ __forceinline__ int spad(int i) { return i + (i >> 4); }  // one pad element per 16

template <typename V, int LR>
__global__ void __launch_bounds__((1 << LR) / 4) small_fft_kernel(const KArgs a) {
    constexpr int R = 1 << LR, T = R / 4, NT4 = LR / 2;  // radix-4 steps; odd LR adds a radix-2 step
    constexpr bool R2 = (LR & 1) != 0;
    constexpr int TW = R - 4, TWT = (TW + T - 1) / T;   // table entries, per thread
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V *buf0 = reinterpret_cast<V *>(smem_raw);
    V *buf1 = buf0 + spad(R);
    V *tw = buf1 + spad(R);
    using E = typename ElemOf<V>::type;
    const int t = threadIdx.x;
    int64_t io, oo, te;
    line_offsets(a, int64_t(blockIdx.x), io, oo, te);
    const E *in = reinterpret_cast<const E *>(a.in) + io;
    const E *tws = reinterpret_cast<const E *>(a.twS);
    V v[4], wt[TWT];
#pragma unroll
    for (int q = 0; q < 4; q++) v[q] = in[t + q * T];
#pragma unroll
    for (int i = 0; i < TWT; i++)
        if (t + i * T < TW) wt[i] = __ldg(tws + t + i * T);
#pragma unroll
    for (int i = 0; i < TWT; i++)
        if (t + i * T < TW) tw[t + i * T] = wt[i];
    if (a.conj_in) {
#pragma unroll
        for (int q = 0; q < 4; q++) v[q].y = -v[q].y;
    }
    __syncthreads();
    V *src = buf0, *dst = buf1;
    int NS = 1;
#pragma unroll
    for (int s = 0; s < NT4; s++) {
        if (s > 0) {
#pragma unroll
            for (int q = 0; q < 4; q++) v[q] = src[spad(t + q * T)];
            // twiddles w_{4 NS}^{k q}
            const int k = t & (NS - 1);
#pragma unroll
            for (int q = 1; q < 4; q++) v[q] = cmul(v[q], tw[(NS - 4) + (q - 1) * NS + k]);
        }
        // radix-4 DFT (w_4 = -i)
        const V a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]), b0 = cadd(v[1], v[3]), b1 = csub(v[1], v[3]);
        const V mb1 = mk<V>(b1.y, -b1.x);  // -i b1
        V y[4] = {cadd(a0, b0), cadd(a1, mb1), csub(a0, b0), csub(a1, mb1)};
        const int base = ((t / NS) * 4 * NS) + (t & (NS - 1));
        const bool last = !R2 && s == NT4 - 1;
        if (!last) {
#pragma unroll
            for (int r = 0; r < 4; r++) dst[spad(base + r * NS)] = y[r];
            __syncthreads();
            V *x = src;
            src = dst;
            dst = x;
            NS *= 4;
        } else {
#pragma unroll
            for (int r = 0; r < 4; r++) v[r] = y[r];
            NS *= 4;
        }
    }
    int kb = t, ks = T;  // outputs: v[q] = X[kb + q ks]
    if constexpr (R2) {  // final radix-2 step: NS = R/2, each thread two groups j = t, t + T
        V w[4];
#pragma unroll
        for (int g = 0; g < 2; g++) {
            const int j = t + g * T;
            V x0 = src[spad(j)], x1 = src[spad(j + R / 2)];
            x1 = cmul(x1, tw[(R / 2 - 4) + j]);  // w_R^{j}
            w[g] = cadd(x0, x1);
            w[2 + g] = csub(x0, x1);
        }
        // X[j] = w[g], X[j + R/2] = w[2 + g]: q -> k = t + q T
#pragma unroll
        for (int q = 0; q < 4; q++) v[q] = w[q];
    }
    V *out = reinterpret_cast<V *>(a.out) + oo;
    const bool mod = a.conj_out || a.scale != 1.0;
    using Tr = typename RealOf<V>::type;
    const Tr sr = Tr(a.scale), si = a.conj_out ? -Tr(a.scale) : Tr(a.scale);
#pragma unroll
    for (int q = 0; q < 4; q++) {
        V r = v[q];
        if (mod) r = mk<V>(r.x * sr, r.y * si);
        out[kb + q * ks] = r;
    }
}

// ---------------------------------------------------------------------------
// The unblocked control (MOA_FFT_UNBLOCKED): Van Loan's program as written,
// Fig. vanloan_fft P:1845-1876 -- x <- P_n x, then for q = 1..t one global
// radix-2 stage x_{L x r} <- B_L x_{L x r} (L = 2^q), each a full HBM round
// trip.  Butterfly of Fig. fftpsirad2: c = w(row) x(col'+row+L/2),
// d = x(col'+row), x(col'+row) = d + c, x(col'+row+L/2) = d - c, with
// w(row) = w_L^row = w_n^{row n/L} from the two-level table.
template <typename V>
__global__ void __launch_bounds__(256) vl_stage_kernel(V *__restrict__ x, int64_t half_total, int logh, int64_t n,
                                                       const double2 *__restrict__ hi, const double2 *__restrict__ lo,
                                                       int twh, int conj_out, double scale) {
    const int64_t h = int64_t(1) << logh;
    const int64_t estep = n >> (logh + 1);  // n / L
    using T = typename RealOf<V>::type;
    const T sr = T(scale), si = conj_out ? -T(scale) : T(scale);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < half_total; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t row = i & (h - 1);
        const int64_t top = ((i >> logh) << (logh + 1)) + row;  // col' + row (blocks of L never straddle rows)
        const V d = x[top], b = x[top + h];
        const V w = cvt_tw(tw_lookup(hi, lo, (row * estep) & (n - 1), twh), V{});
        const V c = cmul(b, w);
        V u = cadd(d, c), v = csub(d, c);
        if (conj_out || scale != 1.0) {
            u = mk<V>(u.x * sr, u.y * si);
            v = mk<V>(v.x * sr, v.y * si);
        }
        x[top] = u;
        x[top + h] = v;
    }
}

// One stage of the hypercube form (MOA_FFT_HYPERCUBE, Ch.5): stage s reads the
// pairs along the top axis of the current hypercube view, (i, i + n/2), and
// stores through the transposition that brings axis s + 1 to the top --
// out[(i >> s) 2^{s+1} + j + r 2^s], j = i mod 2^s -- with the weight
// w_{2^{s+1}}^j = w_n^{j 2^{t-1-s}} on the second element (the radix-2
// Stockham autosort; the t_j transposes of Eq. tvec P:4991-4993 done physically).
template <typename V>
__global__ void __launch_bounds__(256) hyper_stage_kernel(const V *__restrict__ in, V *__restrict__ out,
                                                          int64_t half_total, int logn, int s,
                                                          const double2 *__restrict__ hi,
                                                          const double2 *__restrict__ lo, int twh, int conj_in,
                                                          int conj_out, double scale) {
    const int64_t half = int64_t(1) << (logn - 1), ns = int64_t(1) << s;
    using T = typename RealOf<V>::type;
    const T sr = T(scale), si = conj_out ? -T(scale) : T(scale);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < half_total; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t base = (i >> (logn - 1)) << logn, ii = i & (half - 1);
        V a = in[base + ii], b = in[base + ii + half];
        if (conj_in) {
            a.y = -a.y;
            b.y = -b.y;
        }
        const int64_t j = ii & (ns - 1);
        const V c = cmul(b, cvt_tw(tw_lookup(hi, lo, j << (logn - 1 - s), twh), V{}));
        V u = cadd(a, c), v = csub(a, c);
        if (conj_out || scale != 1.0) {
            u = mk<V>(u.x * sr, u.y * si);
            v = mk<V>(v.x * sr, v.y * si);
        }
        const int64_t o = base + ((ii >> s) << (s + 1)) + j;
        out[o] = u;
        out[o + ns] = v;
    }
}

// P_n of every row (Fig. vanloan_fft line 1): out[b n + i] = in[b n + bitrev_t(i)]
template <typename V>
__global__ void __launch_bounds__(256) bitrev_kernel(const V *__restrict__ in, V *__restrict__ out, int64_t total, int t,
                                                     int conj_in, int conj_out, double scale) {
    const int64_t mask = (int64_t(1) << t) - 1;
    using T = typename RealOf<V>::type;
    const T sr = T(scale), si = (conj_in != conj_out) ? -T(scale) : T(scale);  // n = 1: first and last pass
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t j = i & mask;
        const int64_t src = (i & ~mask) | (t ? int64_t(__brevll((unsigned long long)j) >> (64 - t)) : 0);
        const V v = in[src];
        out[i] = mk<V>(v.x * sr, v.y * si);
    }
}

template <typename V>
cudaError_t launch_unblocked(const moa_pass_desc_t &d, const void *in, void *out, const DevTables &tb,
                             cudaStream_t stream, const PassMods &mods, int64_t total) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t work = (d.kind == 2 || d.kind == 4) ? total / 2 : total;
    int64_t grid = (work + 255) / 256;
    if (grid > int64_t(sms) * 16) grid = int64_t(sms) * 16;
    if (grid < 1) grid = 1;
    if (d.kind == 4) {
        const int lN = log2_exact(d.twN);
        hyper_stage_kernel<V><<<unsigned(grid), 256, 0, stream>>>(
            static_cast<const V *>(in), static_cast<V *>(out), work, lN, log2_exact(d.in_kstr),
            static_cast<const double2 *>(tb.tw_hi), static_cast<const double2 *>(tb.tw_lo), (lN + 1) / 2, mods.conj_in,
            mods.conj_out, mods.scale);
    } else if (d.kind == 3) {
        bitrev_kernel<V><<<unsigned(grid), 256, 0, stream>>>(static_cast<const V *>(in), static_cast<V *>(out), total,
                                                              log2_exact(d.twN), mods.conj_in, mods.conj_out, mods.scale);
    } else {
        const int lN = log2_exact(d.twN);
        vl_stage_kernel<V><<<unsigned(grid), 256, 0, stream>>>(static_cast<V *>(out), work, log2_exact(d.in_kstr), d.twN,
                                                               static_cast<const double2 *>(tb.tw_hi),
                                                               static_cast<const double2 *>(tb.tw_lo), (lN + 1) / 2,
                                                               mods.conj_out, mods.scale);
    }
    return cudaGetLastError();
}

template <typename V> using KFn = void (*)(const KArgs);
template <typename V> using PFn = void (*)(const PairArgs);

template <typename V, int... Ls> constexpr auto make_table(std::integer_sequence<int, Ls...>) {
    return std::array<KFn<V>, sizeof...(Ls)>{&pass_kernel<V, Ls>...};
}
// the same kernels with the fused-exchange (peer store) path compiled in
template <typename V, int... Ls> constexpr auto make_full_table(std::integer_sequence<int, Ls...>) {
    return std::array<KFn<V>, sizeof...(Ls)>{&pass_kernel<V, Ls, true>...};
}
// fused pairs: R_A, R_B in 2^5 .. 2^10 (36 instantiations per dtype)
template <typename V, int... Is> constexpr auto make_pair_table(std::integer_sequence<int, Is...>) {
    return std::array<PFn<V>, sizeof...(Is)>{&pair_kernel<V, 5 + Is / 6, 5 + Is % 6>...};
}
const std::array<PFn<double2>, 36> kPair128 = make_pair_table<double2>(std::make_integer_sequence<int, 36>{});
const std::array<PFn<float2>, 36> kPair64 = make_pair_table<float2>(std::make_integer_sequence<int, 36>{});
const std::array<KFn<double2>, 13> kTab128 = make_table<double2>(std::make_integer_sequence<int, 13>{});
// paired complex64 lines (float4 = two adjacent lines)
const std::array<KFn<float4>, 13> kTabPair64 = make_table<float4>(std::make_integer_sequence<int, 13>{});
const std::array<KFn<float2>, 13> kTab64 = make_table<float2>(std::make_integer_sequence<int, 13>{});
const std::array<KFn<double2>, 13> kTabFull128 = make_full_table<double2>(std::make_integer_sequence<int, 13>{});
const std::array<KFn<float2>, 13> kTabFull64 = make_full_table<float2>(std::make_integer_sequence<int, 13>{});

KArgs fill_args(const moa_pass_desc_t &d, const void *in, void *out, const DevTables &tb, int64_t *nlines,
                const PassMods &mods, int dtype_esize) {
    KArgs a{};
    a.conj_in = mods.conj_in;
    a.conj_out = mods.conj_out;
    a.scale = mods.scale;
    a.npeers = mods.npeers;
    a.log_chunk = mods.log_chunk;
    a.self_off = mods.self_off;
    for (int i = 0; i < 8; i++) a.peers[i] = mods.peers[i];
    a.in = in;
    a.out = out;
    a.ndig = d.ndig;
    int64_t nl = 1;
    for (int i = 0; i < d.ndig; i++) {
        a.in_str[i] = d.in_str[i];
        a.out_str[i] = d.out_str[i];
        a.tw_str[i] = d.tw_str[i];
        a.lext[i] = log2_exact(d.ext[i]);
        nl *= d.ext[i];
    }
    *nlines = nl;
    a.in_kstr = d.in_kstr;
    a.out_kstr = d.out_kstr;
    a.twR = tb.twR;
    a.tw_hi = tb.tw_hi;
    a.tw_lo = tb.tw_lo;
    a.twS = tb.twS;
    a.twmask = d.twN > 1 ? d.twN - 1 : 0;
    const int lN = log2_exact(d.twN);
    a.twh = (lN + 1) / 2;
    a.tw_off = d.tw_off;
    a.ksplit = d.out_ksplit < d.logR ? d.out_ksplit : 30;
    a.out_kstr_hi = d.out_kstr_hi;
    a.nodft = d.kind == 1;
    a.W = d.W;
    a.lW = log2_exact(d.W);
    a.LS = (1 << d.logR) + d.line_pad;
    a.lf_load = d.lf_load;
    a.lf_store = d.lf_store;
    a.ring = d.ring;
    // discard.global.L2 drops whole 128-byte lines: only when every line a
    // consumed 128-byte run touches belongs to this tile (a line-fast side with
    // adjacent lines adjacent in memory and W * esize >= 128, or a point-fast
    // side with contiguous points and R * esize >= 128) -- otherwise it would
    // also drop lines the next tile has not read yet
    {
        const int64_t esize = dtype_esize;
        const bool lf_ok = d.lf_load && d.ndig >= 1 && d.in_str[0] == 1 && int64_t(d.W) * esize >= 128;
        const bool pf_ok = !d.lf_load && d.in_kstr == 1 && (int64_t(1) << d.logR) * esize >= 128;
        a.discard = d.ring_discard && (lf_ok || pf_ok);
    }
    return a;
}

// prefetch distance = f x (CTAs resident on the device at once)
void set_prefetch(KArgs &a, const void *fn, int threads, int smem, int64_t tiles, double f) {
    int per_sm = 0, dev = 0, sms = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    a.pf_dist = int64_t(f * per_sm * sms + 0.5);
    if (a.pf_dist < 1) a.pf_dist = 1;
    a.ntiles = tiles;
}

bool encode_lf_tmap(CUtensorMap *map, const moa_pass_desc_t &d, const void *in, int esize, int64_t W, int *rank,
                    int *nbox, int *box_pts);

// the line-fast side's tensor map for the box prefetch (false: not expressible)
bool set_lf_prefetch_map(KArgs &a, const moa_pass_desc_t &d, int esize) {
    int rank = 0, nbox = 0, bp = 0;
    if (!d.lf_load || d.ndig < 1 || d.in_str[0] != 1 || d.ndig > 4) return false;
    if (!encode_lf_tmap(&a.pf_tmap, d, a.in, esize, d.W, &rank, &nbox, &bp)) return false;
    a.pf_rank = rank;
    a.pf_nbox = nbox;
    a.pf_box_pts = bp;
    a.pf_ext0 = int32_t(d.ext[0]);
    return true;
}

// ---- warp-specialised launch (MOA_FFT_WS != 0): eligible passes only, else
// cudaErrorNotSupported and the plain kernel runs
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            return EncodeTiledFn(nullptr);
        }
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

// Tensor map of a line-fast STORE side (digit 0 = adjacent lines, unit
// stride): dims (2 digit-0 reals, the R points at out_kstr, line digits 1..),
// boxes of W lines x min(R, 256) points (false: not expressible).
bool set_lf_store_map(KArgs &a, const moa_pass_desc_t &d, int esize) {
    EncodeTiledFn enc = encode_tiled();
    if (!enc || !d.lf_store || d.ndig < 1 || d.ndig > 4 || d.out_str[0] != 1 || d.out_ksplit < d.logR) return false;
    const int64_t R = int64_t(1) << d.logR, W = d.W;
    cuuint64_t dims[5], strides[4];
    cuuint32_t box[5], estr[5] = {1, 1, 1, 1, 1};
    int rank = 0;
    dims[rank] = cuuint64_t(2 * d.ext[0]);
    box[rank++] = cuuint32_t(2 * W);
    const int64_t bp = R < 256 ? R : 256;
    dims[rank] = cuuint64_t(R);
    strides[rank - 1] = cuuint64_t(d.out_kstr * esize);
    box[rank++] = cuuint32_t(bp);
    for (int i = 1; i < d.ndig; i++) {
        dims[rank] = cuuint64_t(d.ext[i]);
        strides[rank - 1] = cuuint64_t(d.out_str[i] * esize);
        box[rank++] = 1;
    }
    if (2 * W > 256 || (W * esize) % 16 || d.ext[0] % W) return false;
    for (int i = 0; i < rank - 1; i++)
        if (strides[i] % 16 || strides[i] >= (cuuint64_t(1) << 40)) return false;
    CUresult r = enc(&a.st_tmap, esize == 16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                     cuuint32_t(rank), a.out, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    a.st_rank = rank;
    a.st_nbox = int32_t(R / bp);
    a.st_box_pts = int32_t(bp);
    a.pf_ext0 = int32_t(d.ext[0]);
    return true;
}

// Tensor map of a line-fast load side (digit 0 = adjacent lines, unit stride):
// dims (2 digit-0 reals, the R points at in_kstr, line digits 1..), boxes of
// W lines x min(R, 256) points.
bool encode_lf_tmap(CUtensorMap *map, const moa_pass_desc_t &d, const void *in, int esize, int64_t W, int *rank_out,
                    int *nbox, int *box_pts) {
    EncodeTiledFn enc = encode_tiled();
    if (!enc) return false;
    const int64_t R = int64_t(1) << d.logR;
    cuuint64_t dims[5], strides[4];
    cuuint32_t box[5], estr[5] = {1, 1, 1, 1, 1};
    int rank = 0;
    dims[rank] = cuuint64_t(2 * d.ext[0]);
    box[rank++] = cuuint32_t(2 * W);
    const int64_t bp = R < 256 ? R : 256;
    dims[rank] = cuuint64_t(R);
    strides[rank - 1] = cuuint64_t(d.in_kstr * esize);
    box[rank++] = cuuint32_t(bp);
    for (int i = 1; i < d.ndig; i++) {
        dims[rank] = cuuint64_t(d.ext[i]);
        strides[rank - 1] = cuuint64_t(d.in_str[i] * esize);
        box[rank++] = 1;
    }
    if (2 * W > 256 || (W * esize) % 16) return false;
    for (int i = 0; i < rank - 1; i++)
        if (strides[i] % 16 || strides[i] >= (cuuint64_t(1) << 40)) return false;
    CUresult r = enc(map, esize == 16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                     cuuint32_t(rank), const_cast<void *>(in), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    *rank_out = rank;
    *nbox = int(R / bp);
    *box_pts = int(bp);
    return true;
}

int ws_mode() {  // MOA_FFT_WS: 0 off, 1 on (eligible passes)
    const char *e = std::getenv("MOA_FFT_WS");
    return e ? std::atoi(e) : 0;
}

template <typename V, int... Ls> constexpr auto make_ws_table(std::integer_sequence<int, Ls...>) {
    return std::array<void (*)(const WsArgs), sizeof...(Ls)>{&ws_pass_kernel<V, Ls>...};
}
const std::array<void (*)(const WsArgs), 13> kWs128 = make_ws_table<double2>(std::make_integer_sequence<int, 13>{});
const std::array<void (*)(const WsArgs), 13> kWs64 = make_ws_table<float2>(std::make_integer_sequence<int, 13>{});

template <typename V>
cudaError_t launch_ws(const std::array<void (*)(const WsArgs), 13> &tab, const moa_pass_desc_t &d, const KArgs &a,
                      int64_t tiles, const DevTables &tb, cudaStream_t stream, const PassMods &mods) {
    using E = typename ElemOf<V>::type;
    const int esize = int(sizeof(E));
    const int LP = psi_log_p(d.logR, sizeof(E) == 16 ? MOA_C128 : MOA_C64);
    const int64_t R = int64_t(1) << d.logR, TPL = R >> LP;
    const int64_t nthr = int64_t(d.W) * TPL;
    if (d.ring || mods.npeers || d.kind > 1 || nthr > kWsGroupMax || nthr % 32 || d.ndig < 1) return cudaErrorNotSupported;
    if (!std::is_same<V, double2>::value && !std::is_same<V, float2>::value) return cudaErrorNotSupported;
    // short lines: a tile is many small copies (measured: 4-point lines, 128
    // 64-byte copies per tile, 7x slower than the plain kernel)
    if (d.logR < 8) return cudaErrorNotSupported;
    // two consumer groups of >= 4 warps (one line per CTA of a 1024-point
    // complex64 pass would leave 2 warps per SM: measured 4x slower)
    if (nthr < 128) return cudaErrorNotSupported;
    WsArgs w{};
    w.a = a;
    w.a.pf_dist = 0;
    w.ntiles = tiles;
    w.ctr = tb.ctr;
    int mode;
    if (d.lf_load && d.in_str[0] == 1 && d.ndig <= 4 && (int64_t(d.W) * esize) % 16 == 0) mode = 0;
    else if (!d.lf_load && d.in_kstr == 1 && (int64_t(a.LS) * esize) % 16 == 0 && (R * esize) % 16 == 0) mode = 1;
    else return cudaErrorNotSupported;
    w.mode = mode;
    w.stage_elems = int32_t(int64_t(d.W) * a.LS);
    w.stage_bytes = uint32_t(int64_t(d.W) * R * esize);
    // stages: as many as fit next to the 128-byte barrier block (<= 4)
    int dev = 0, smem_max = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t stage_b = int64_t(w.stage_elems) * esize;
    int S = int((smem_max - 128) / stage_b);
    if (const char *se = std::getenv("MOA_FFT_WS_STAGES")) S = std::min(S, std::atoi(se));
    if (S > kWsStagesMax) S = kWsStagesMax;
    if (S < 2) return cudaErrorNotSupported;
    w.stages = S;
    if (mode == 0) {
        int rank = 0, nbox = 0, bp = 0;
        if (!encode_lf_tmap(&w.tmap, d, a.in, esize, d.W, &rank, &nbox, &bp)) return cudaErrorNotSupported;
        w.tmap_rank = rank;
        w.nbox = nbox;
        w.box_pts = bp;
        w.ext0 = int32_t(d.ext[0]);
    }
    auto fn = tab[d.logR];
    const int smem = int(128 + S * stage_b);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    if (w.ctr) {
        e = cudaMemsetAsync(w.ctr, 0, sizeof(unsigned long long), stream);
        if (e != cudaSuccess) return e;
    }
    const int64_t grid = tiles < sms ? tiles : sms;
    fn<<<dim3(unsigned(grid)), dim3(unsigned(2 * nthr)), size_t(smem), stream>>>(w);
    return cudaGetLastError();
}

template <typename V>
cudaError_t launch_t(const std::array<KFn<V>, 13> &tab, const moa_pass_desc_t &d, const void *in, void *out,
                     const DevTables &tb, cudaStream_t stream, const PassMods &mods) {
    int64_t nlines = 0;
    KArgs a = fill_args(d, in, out, tb, &nlines, mods, int(sizeof(typename ElemOf<V>::type)));
    const int64_t tiles = nlines / d.W;
    // MOA_FFT_PF = f: prefetch the tile f * (resident CTAs) ahead into L2 (0: off),
    // for contiguous-line (point-fast) loads -- a few large bulk prefetches per
    // tile.  Line-fast loads (MOA_FFT_PF_LF = f): one tensor-map box prefetch
    // (W lines x 256 points) per box (one 128-byte bulk prefetch per point
    // measured slower: cfg3 4.95 -> 5.8 ms, cfg4 12.0 -> 13.4 ms,
    // profiles/r2b_ab_pf.jsonl).
    // Default: 0.5 for contiguous lines of >= 512 points (measured: cfg5 passes
    // 6.35 -> 6.22 ms, cfg3's 1024-point last pass 1.71 -> 1.57 ms; cfg2's
    // 256-point rows 0.311 -> 0.315 ms, so not there -- profiles/r2c_ab_cfg5.jsonl,
    // r2b_ab_pf.jsonl).
    // Line-fast loads: default 0.5 when the points are < 1 MiB apart (box
    // prefetch measured: cfg3 pass 1 (16 KiB) 1.50 -> 1.37 ms, cfg4 pass 2
    // (2 KiB) 2.90 -> 2.68 ms, cfg2 pass 0 0.341 -> 0.326 ms; but cfg3 pass 0
    // (8 MiB apart: every box row a different DRAM page) 1.78 -> 2.20 ms,
    // profiles/r3a_pflf.jsonl).
    const int64_t kload_b = d.in_kstr * int64_t(sizeof(typename ElemOf<V>::type));
    double pf = (!d.lf_load && d.logR >= 9) ? 0.5 : (d.lf_load && kload_b < (int64_t(1) << 20)) ? 0.5 : 0.0;
    if (const char *pe = std::getenv(d.lf_load ? "MOA_FFT_PF_LF" : "MOA_FFT_PF")) pf = std::atof(pe);
    // complex64 passes of >= 2^10-point lines coalesced along the lines on both
    // sides (digit 0 unit stride in and out, even tile width): two adjacent
    // lines per lane -- half the threads and memory instructions per tile
    // (measured: 3-D c64 y-pass 5.12 -> 4.04 ms; slower for <= 2^8-point lines)
    if constexpr (std::is_same<V, float2>::value) {
        // MOA_FFT_C64PAIR (ablation): 0 off, 1 also for short lines; read once
        static const int pair_mode = [] {
            const char *pe = std::getenv("MOA_FFT_C64PAIR");
            return pe && pe[0] == '0' ? 0 : pe && pe[0] == '1' ? 2 : 1;
        }();
        const int min_lr = pair_mode == 2 ? 4 : 10;
        if (pair_mode && psi_log_p(d.logR, MOA_C64) == 4 && d.lf_load && d.lf_store && d.kind == 0 && !d.ring &&
            !mods.npeers && d.ndig >= 1 &&
            d.in_str[0] == 1 && d.out_str[0] == 1 && d.W >= 2 && d.logR >= min_lr && d.out_ksplit >= d.logR) {
            KArgs b = a;
            b.W = d.W / 2;
            b.lW = log2_exact(b.W);
            // the pair tile's own shared-memory line stride: 16-byte elements,
            // W / 2 lines (the descriptor's was chosen for 8-byte elements);
            // memoised per tile shape (the bank model is host work per launch)
            static std::mutex ls_mu;
            static std::map<std::tuple<int, int, int, int, int>, int32_t> ls_memo;
            const auto key = std::make_tuple(int(d.logR), int(b.W), int(d.lf_load), int(d.lf_store), int(d.smem_bytes));
            int32_t memo_ls = -1;
            {
                std::lock_guard<std::mutex> g(ls_mu);
                auto it = ls_memo.find(key);
                if (it != ls_memo.end()) memo_ls = it->second;
            }
            if (memo_ls >= 0) {
                b.LS = memo_ls;
            } else {
                const int64_t R = int64_t(1) << d.logR, base = R + R / 16;
                int64_t best = base, bw = 1 << 30, bt = int64_t(1) << 62;
                for (int64_t LS = base; LS < base + 16 && (b.W * LS * 16 <= d.smem_bytes); LS++) {
                    int64_t tot = 0;
                    const int w = psi_bank_conflicts(d.logR, b.W, 16, d.lf_load, d.lf_store, LS, &tot);
                    if (w < bw || (w == bw && tot < bt)) {
                        best = LS;
                        bw = w;
                        bt = tot;
                    }
                }
                b.LS = int32_t(best);
                std::lock_guard<std::mutex> g(ls_mu);
                ls_memo[key] = b.LS;
            }
            KFn<float4> f = kTabPair64[d.logR];
            if (d.smem_bytes > 48 * 1024) {
                cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, d.smem_bytes);
                if (e != cudaSuccess) return e;
            }
            if (pf > 0 && !d.ring && (!d.lf_load || set_lf_prefetch_map(b, d, int(sizeof(float2)))))
                set_prefetch(b, reinterpret_cast<const void *>(f), d.threads / 2, d.smem_bytes, tiles, pf);
            f<<<dim3(unsigned(tiles)), dim3(unsigned(d.threads / 2)), size_t(d.smem_bytes), stream>>>(b);
            return cudaGetLastError();
        }
    }
    // one-pass plans with few lines (latency, cfg1): the small-transform kernel
    // (MOA_FFT_SMALL=0 disables it)
    if (d.kind == 0 && tb.twS && !d.ring && !mods.npeers && d.twN <= 1 && d.logR >= 6 && d.logR <= 12 && !d.lf_load &&
        !d.lf_store && d.in_kstr == 1 && d.out_kstr == 1 && d.out_ksplit >= d.logR && nlines <= 64) {
        const char *se = std::getenv("MOA_FFT_SMALL");
        if (!(se && se[0] == '0')) {
            static const std::array<KFn<V>, 7> small = {&small_fft_kernel<V, 6>, &small_fft_kernel<V, 7>,
                                                        &small_fft_kernel<V, 8>, &small_fft_kernel<V, 9>,
                                                        &small_fft_kernel<V, 10>, &small_fft_kernel<V, 11>,
                                                        &small_fft_kernel<V, 12>};
            const int R = 1 << d.logR;
            const size_t smem = (2 * size_t(R + (R >> 4)) + size_t(R - 4)) * sizeof(V);
            KFn<V> fn = small[d.logR - 6];
            static std::mutex mu;
            static std::map<std::pair<int, const void *>, size_t> attr;  // opt-in smem set once per (device, kernel)
            if (smem > 48 * 1024) {
                int dev = 0;
                cudaGetDevice(&dev);
                std::lock_guard<std::mutex> g(mu);
                size_t &have = attr[{dev, reinterpret_cast<const void *>(fn)}];
                if (have < smem) {
                    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
                    if (e != cudaSuccess) return e;
                    have = smem;
                }
            }
            fn<<<dim3(unsigned(nlines)), dim3(unsigned(R / 4)), smem, stream>>>(a);
            return cudaGetLastError();
        }
    }
    // MOA_FFT_PAIR=1: complex128 512- / 1024-point lines on thread pairs
    // (radix 32 with a warp-shuffle exchange, twice the threads per tile)
    if constexpr (std::is_same<V, double2>::value || std::is_same<V, float2>::value) {
        const char *pe = std::getenv("MOA_FFT_PAIR");
        if (pe && pe[0] == '1' && (d.logR == 9 || d.logR == 10) && d.kind == 0 && !d.ring && !mods.npeers &&
            2 * d.threads <= (std::is_same<V, double2>::value ? 512 : 1024)) {
            auto fn = d.logR == 9 ? &pass_kernel_pair<V, 9> : &pass_kernel_pair<V, 10>;
            if (d.smem_bytes > 48 * 1024) {
                cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, d.smem_bytes);
                if (e != cudaSuccess) return e;
            }
            fn<<<dim3(unsigned(tiles)), dim3(unsigned(2 * d.threads)), size_t(d.smem_bytes), stream>>>(a);
            return cudaGetLastError();
        }
    }
    if (ws_mode() && d.W >= 1) {
        cudaError_t e = std::is_same<V, double2>::value ? launch_ws<V>(kWs128, d, a, tiles, tb, stream, mods)
                                                        : launch_ws<V>(kWs64, d, a, tiles, tb, stream, mods);
        if (e != cudaErrorNotSupported) return e;
    }
    // TMA store (pass_kernel_st): 512- / 1024-point passes with contiguous
    // loads and a line-fast (transposed) store side.  Default for complex128:
    // cfg5's rotating 3-D passes 5.79-6.01 -> 5.76-5.88 ms (cfg5 17.4-18.0 ->
    // 17.3-17.6 ms, same-box rounds), cfg3's last pass neutral (1.56-1.58 vs
    // 1.55-1.64 ms) (profiles/r7b_ab.jsonl, r7c_ab.jsonl).  complex64 only
    // with MOA_FFT_TMA_ST64=1 (measurement pending) or MOA_FFT_TMA_ST=1, which
    // forces it on every eligible pass; MOA_FFT_TMA_ST=0 turns it off.
    {
        constexpr bool c128 = std::is_same<V, double2>::value;
        const char *te = std::getenv("MOA_FFT_TMA_ST");
        const char *te64 = std::getenv("MOA_FFT_TMA_ST64");
        const bool tma_st = te ? te[0] == '1' : (c128 || (te64 && te64[0] == '1'));
        if (tma_st && (d.logR == 9 || d.logR == 10) && d.kind == 0 && !d.ring && !mods.npeers && !d.lf_load &&
            d.lf_store && d.W >= 1 && set_lf_store_map(a, d, int(sizeof(V)))) {
            KFn<V> fs = d.logR == 9 ? &pass_kernel_st<V, 9> : &pass_kernel_st<V, 10>;
            if (d.smem_bytes > 48 * 1024) {
                cudaError_t e = cudaFuncSetAttribute(fs, cudaFuncAttributeMaxDynamicSharedMemorySize, d.smem_bytes);
                if (e != cudaSuccess) return e;
            }
            if (pf > 0) set_prefetch(a, reinterpret_cast<const void *>(fs), d.threads, d.smem_bytes, tiles, pf);
            fs<<<dim3(unsigned(tiles)), dim3(unsigned(d.threads)), size_t(d.smem_bytes), stream>>>(a);
            return cudaGetLastError();
        }
    }
    KFn<V> fn = tab[d.logR];
    if (mods.npeers || d.ring) {  // the peer-store / ring paths live in the full instantiations
        if constexpr (std::is_same<V, double2>::value) fn = kTabFull128[d.logR];
        else fn = kTabFull64[d.logR];
    }
    if (d.smem_bytes > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, d.smem_bytes);
        if (e != cudaSuccess) return e;
    }
    if (pf > 0 && !d.ring && (!d.lf_load || set_lf_prefetch_map(a, d, int(sizeof(typename ElemOf<V>::type)))))
        set_prefetch(a, reinterpret_cast<const void *>(fn), d.threads, d.smem_bytes, tiles, pf);
    // ablation (MOA_FFT_CLAUNCH=k): launch a line-fast pass whose loads are
    // >= 1 MiB apart as clusters of k CTAs, so the k adjacent tiles (whose
    // 128-byte runs share DRAM pages) start together on one GPC
    static const int claunch = [] {
        const char *ce = std::getenv("MOA_FFT_CLAUNCH");
        return ce ? std::atoi(ce) : 0;
    }();
    if (claunch > 1 && d.lf_load && kload_b >= (int64_t(1) << 20) && tiles % claunch == 0) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(unsigned(tiles));
        cfg.blockDim = dim3(unsigned(d.threads));
        cfg.dynamicSmemBytes = size_t(d.smem_bytes);
        cfg.stream = stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = unsigned(claunch);
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, fn, a);
    }
    fn<<<dim3(unsigned(tiles)), dim3(unsigned(d.threads)), size_t(d.smem_bytes), stream>>>(a);
    return cudaGetLastError();
}

template <typename V>
cudaError_t launch_pair_t(const std::array<PFn<V>, 36> &tab, const moa_pass_desc_t &dA, const moa_pass_desc_t &dB,
                          const void *in, void *out, const RingState &rs, const DevTables &tA, const DevTables &tB,
                          cudaStream_t stream, const PassMods &mA, const PassMods &mB) {
    int64_t nA = 0, nB = 0;
    PairArgs p{};
    p.A = fill_args(dA, in, rs.ring, tA, &nA, mA, int(sizeof(V)));
    p.B = fill_args(dB, rs.ring, out, tB, &nB, mB, int(sizeof(V)));
    p.TA = int32_t((nA / dA.W) / dA.ring_groups);
    p.TB = int32_t((nB / dB.W) / dB.ring_groups);
    p.groups = dA.ring_groups;
    p.ringG = dA.ring_G;
    p.lag = dA.ring_lag;
    p.slot_mask = dA.ring_slots - 1;
    p.qctr = rs.qctr;
    p.cntA = rs.cntA;
    p.cntB = rs.cntB;
    // the completion counters are reset on the stream before every launch (so a
    // captured CUDA graph replays correctly: no host-side epoch baked into the
    // arguments); the kernel waits for counts of exactly TA / TB
    p.epoch = 0;
    p.stats = rs.stats;
    PFn<V> fn = tab[(dA.logR - 5) * 6 + (dB.logR - 5)];
    const int smem = dA.smem_bytes > dB.smem_bytes ? dA.smem_bytes : dB.smem_bytes;
    if (smem > 48 * 1024 - 64) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
    }
    const int64_t tiles = p.groups * (p.TA + p.TB);
    // persistent grid: every CTA resident at once (required by the waits)
    int per_sm = 0, dev = 0, sms = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, dA.threads, smem);
    if (e != cudaSuccess) return e;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t grid = int64_t(per_sm > 0 ? per_sm : 1) * sms;
    if (grid > tiles) grid = tiles;
    e = cudaMemsetAsync(rs.cntA, 0, size_t(p.groups) * sizeof(unsigned long long), stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(rs.cntB, 0, size_t(p.groups) * sizeof(unsigned long long), stream);
    if (e != cudaSuccess) return e;
    // the tile waits need every CTA resident at once: a cooperative launch
    // fails cleanly (instead of trapping in the watchdog) when the grid cannot
    // be co-resident, e.g. with other kernels occupying SMs
    void *kargs[] = {&p};
    return cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(fn), dim3(unsigned(grid)),
                                       dim3(unsigned(dA.threads)), kargs, size_t(smem), stream);
}

// (R_A, R_B) in 2^5 .. 2^9 (25 instantiations per dtype)
template <typename V, int... Is> constexpr auto make_cluster_table(std::integer_sequence<int, Is...>) {
    return std::array<void (*)(const KArgs, const KArgs), sizeof...(Is)>{&cluster_kernel<V, 5 + Is / 5, 5 + Is % 5>...};
}

template <typename V>
cudaError_t launch_cluster_t(const moa_pass_desc_t &dA, const moa_pass_desc_t &dB, const void *in, void *out,
                             const DevTables &tA, const DevTables &tB, cudaStream_t stream, const PassMods &mA,
                             const PassMods &mB) {
    static const auto tab = make_cluster_table<V>(std::make_integer_sequence<int, 25>{});
    if (dA.logR < 5 || dA.logR > 9 || dB.logR < 5 || dB.logR > 9 || dA.threads != dB.threads || dA.ring_slots < 1)
        return cudaErrorInvalidValue;
    const int esize = int(sizeof(V));
    int64_t nA = 0, nB = 0;
    KArgs a = fill_args(dA, in, nullptr, tA, &nA, mA, esize);
    KArgs b = fill_args(dB, nullptr, out, tB, &nB, mB, esize);
    const int C = dA.ring_slots;
    const int lg = log2_exact(dA.ring_G), lc = lg - log2_exact(C);
    a.ds_lg = b.ds_lg = lg;
    a.ds_lc = b.ds_lc = lc;
    auto fn = tab[(dA.logR - 5) * 5 + (dB.logR - 5)];
    int smem = dA.smem_bytes > dB.smem_bytes ? dA.smem_bytes : dB.smem_bytes;
    if ((int64_t(1) << lc) * esize > smem) smem = int((int64_t(1) << lc) * esize);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess && C > 8) e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    const int64_t tiles = nA / dA.W;  // groups x C
    // pass A's loads: the plain kernel's L2 prefetch rule (launch_t)
    const int64_t kload_b = dA.in_kstr * int64_t(esize);
    double pf = (!dA.lf_load && dA.logR >= 9) ? 0.5 : (dA.lf_load && kload_b < (int64_t(1) << 20)) ? 0.5 : 0.0;
    if (const char *pe = std::getenv(dA.lf_load ? "MOA_FFT_PF_LF" : "MOA_FFT_PF")) pf = std::atof(pe);
    if (pf > 0 && (!dA.lf_load || set_lf_prefetch_map(a, dA, esize)))
        set_prefetch(a, reinterpret_cast<const void *>(fn), dA.threads, smem, tiles, pf);
    if (const char *le = std::getenv("MOA_FFT_CLUSTER_LOCAL")) a.ds_local = le[0] == '1';
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(tiles));
    cfg.blockDim = dim3(unsigned(dA.threads));
    cfg.dynamicSmemBytes = size_t(smem);
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = unsigned(C);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (std::getenv("MOA_FFT_VERBOSE")) {
        int nc = -1;
        cudaOccupancyMaxActiveClusters(&nc, reinterpret_cast<const void *>(fn), &cfg);
        std::fprintf(stderr, "moa cluster pair: C=%d threads=%d smem=%d grid=%lld -> %d clusters resident\n", C,
                     dA.threads, smem, (long long)tiles, nc);
    }
    return cudaLaunchKernelEx(&cfg, fn, a, b);
}
}  // namespace

cudaError_t launch_cluster(const moa_pass_desc_t &dA, const moa_pass_desc_t &dB, moa_dtype_t dtype, const void *in,
                           void *out, const DevTables &tA, const DevTables &tB, cudaStream_t stream,
                           const PassMods &mA, const PassMods &mB) {
    if (dtype == MOA_C128) return launch_cluster_t<double2>(dA, dB, in, out, tA, tB, stream, mA, mB);
    return launch_cluster_t<float2>(dA, dB, in, out, tA, tB, stream, mA, mB);
}

cudaError_t launch_pass(const moa_pass_desc_t &d, moa_dtype_t dtype, const void *in, void *out, const DevTables &tab,
                        cudaStream_t stream, const PassMods &mods) {
    if (d.kind == 2 || d.kind == 3 || d.kind == 4) {  // unblocked control / hypercube: total = ext[0] (rows * n)
        const int64_t total = d.ndig ? d.ext[0] : 1;
        if (dtype == MOA_C128) return launch_unblocked<double2>(d, in, out, tab, stream, mods, total);
        return launch_unblocked<float2>(d, in, out, tab, stream, mods, total);
    }
    if (d.logR < 0 || d.logR > 12) return cudaErrorInvalidValue;
    if (dtype == MOA_C128) return launch_t<double2>(kTab128, d, in, out, tab, stream, mods);
    return launch_t<float2>(kTab64, d, in, out, tab, stream, mods);
}

cudaError_t launch_pair(const moa_pass_desc_t &dA, const moa_pass_desc_t &dB, moa_dtype_t dtype, const void *in,
                        void *out, const RingState &rs, const DevTables &tA, const DevTables &tB, cudaStream_t stream,
                        const PassMods &mA, const PassMods &mB) {
    if (dA.logR < 5 || dA.logR > 10 || dB.logR < 5 || dB.logR > 10 || dA.threads != dB.threads)
        return cudaErrorInvalidValue;
    if (dtype == MOA_C128) return launch_pair_t<double2>(kPair128, dA, dB, in, out, rs, tA, tB, stream, mA, mB);
    return launch_pair_t<float2>(kPair64, dA, dB, in, out, rs, tA, tB, stream, mA, mB);
}

cudaError_t kernel_attributes(moa_dtype_t dtype, int logR, int *max_threads, int *regs) {
    cudaFuncAttributes at{};
    cudaError_t e = dtype == MOA_C128 ? cudaFuncGetAttributes(&at, kTab128[logR]) : cudaFuncGetAttributes(&at, kTab64[logR]);
    if (e == cudaSuccess) {
        *max_threads = at.maxThreadsPerBlock;
        *regs = at.numRegs;
    }
    return e;
}

}  // namespace moa

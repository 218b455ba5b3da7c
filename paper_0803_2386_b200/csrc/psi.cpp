// psi.cpp -- the psi-index layer (host): lifting shape -> ONF pass descriptors.
//
// PAPER.md grounding:
//   * the reshape-transpose <r c> rho-hat (transpose (<r c> rho-hat x)) reduces
//     to the two-loop ONF "for j < c, for i < r: @x + j + c*i" (Eq. trans
//     P:2897-2923, Fig. loopindex): a loop nest of (extent, stride)
//     pairs with an affine address -- exactly what moa_pass_desc_t stores;
//   * the final transpose reduces to "for t < 2^{d-sigma}, s < 2^sigma:
//     @x + s*2^{d-sigma} + t";
//   * the psi Correspondence Theorem (Eq. psi_corr): a partial
//     index selects a contiguous block, so a line's points are one affine
//     stride and the inner loops of a tile are contiguous runs.
// All sizes are powers of two, so every div/mod of the DNF becomes a shift or a
// mask and is removed from the loops by restructuring them, as the paper does
// for i' = int(c i / r), j' = (j + i c) mod r.
//
// Lifting: n = R_0 R_1 ... R_{P-1}.  Pass p < P-1 views the data
// as <B_p R_p S_p> (S_p = R_{p+1}...R_{P-1}) and transforms along the middle
// axis in place, multiplying output k of line (o, j) by w_{R_p S_p}^{j k} (the
// transformed weights of the lifted level).  The last pass
// transforms the contiguous rows and stores through the axis-reversing
// transpose (the lifted final transpose), giving natural order.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "moa_internal.h"

namespace moa {

int log2_exact(int64_t n) {
    if (n < 1) return -1;
    int t = 0;
    while ((int64_t(1) << t) < n) t++;
    return (int64_t(1) << t) == n ? t : -1;
}

static void desc_init(moa_pass_desc_t &d, int logR) {
    std::memset(&d, 0, sizeof(d));
    d.logR = logR;
    d.twN = 1;
    d.out_ksplit = 62;  // no split
}

static void add_digit(moa_pass_desc_t &d, int64_t ext, int64_t is, int64_t os, int64_t ts) {
    if (ext == 1) return;  // a loop of extent 1 contributes nothing to the ONF
    d.ext[d.ndig] = ext;
    d.in_str[d.ndig] = is;
    d.out_str[d.ndig] = os;
    d.tw_str[d.ndig] = ts;
    d.ndig++;
}

static void set_tile(moa_pass_desc_t &d, moa_dtype_t dtype, int64_t W);
int psi_bank_conflicts(int logR, int64_t W, int esize, int lfA, int lfB, int64_t LS, int64_t *total, int logP);

void psi_choose_tile(moa_pass_desc_t &d, moa_dtype_t dtype) {
    const int esize = dtype == MOA_C128 ? 16 : 8;
    const int slots = 128 / esize;        // elements per 128-byte smem row / DRAM line
    const int logR = d.logR, logP = psi_log_p(logR, dtype);
    const int64_t R = int64_t(1) << logR, TPL = R >> logP;
    const bool lf = d.lf_load || d.lf_store;
    const int64_t ext0 = d.ndig ? d.ext[0] : 1;
    // Lines per tile: enough adjacent lines for full 128-byte runs on a
    // line-coalesced side; enough threads per CTA otherwise.
    // (point-contiguous lines of >= 2^10 points: one line per CTA -- more, smaller
    // CTAs per SM overlap their load and compute phases better; measured cfg5
    // z-pass 7.48 -> 6.84 ms)
    // (line-coalesced passes of short lines -- R < 128, e.g. the p-point pass of
    // the processor lifting or an all-radix-2 lifting -- take more lines so a
    // CTA has at least 128 threads)
    // (point-contiguous >= 1024-point lines stay one per CTA also at 32 points
    // per thread: measured 3-D c128 in-place z-pass 5.39 -> 5.22 ms, c64 2.60 -> 2.53)
    int64_t W = lf ? (TPL >= 8 ? slots : (slots > 128 / TPL ? slots : 128 / TPL))
                   : ((TPL >= 64 || R >= 1024) ? 1 : 256 / TPL);
    // complex128 strided passes of <= 2^8 points: 256-byte runs (16 lines) --
    // measured cfg3 5.50 -> 5.24 ms (the 32 MiB-stride first pass 1.50 -> 1.33 ms)
    if (lf && esize == 16 && logR >= 5 && logR <= 8) W = 2 * slots;
    // complex64 strided loads >= 1 MiB apart (cfg4's first pass: 32 MiB): 256-byte
    // runs too (32 lines) -- measured: its movement time 3.19 -> 2.60 ms, the pass
    // 3.48 -> 3.33 ms; passes with shorter strides keep 16 lines (no gain there)
    if (lf && esize == 8 && d.lf_load && d.in_kstr * esize >= (int64_t(1) << 20) && logR >= 5 && logR <= 8)
        W = 4 * slots;
    // two CTAs per SM by default; MOA_FFT_SMEM_CAP (bytes) overrides (ablations)
    // A line-coalesced side whose points are >= 1 MiB apart (the 3-D x-pass:
    // 16 MiB) touches one DRAM page per point: give it full 128-byte runs even at
    // one CTA per SM (measured: cfg5 x-pass 11.7 -> 9.3 ms).
    const char *cap_env = std::getenv("MOA_FFT_SMEM_CAP");
    // (only a strided LOAD side needs the long runs: strided stores are merged
    // into full lines in L2 -- tools/stride_bench, the rotating 3-D layouts)
    const int64_t kload = d.in_kstr * esize;
    // complex64 radix-32 passes loading contiguous lines and storing transposed:
    // 16-line tiles too (128-byte store runs at one 512-thread CTA per SM;
    // measured cfg4's 1024^3 last pass 3.54 -> 3.20 ms, profiles/r3c_c64.jsonl)
    // (and line-coalesced loads of 1024-point complex64 lines without lifted
    // weights at any stride: 16 lines, 128-byte runs -- measured the 3-D
    // complex64 y-pass 3.29 -> 3.10-3.15 ms, profiles/r5n_cap.jsonl; with the
    // weights' table lookups two 8-line CTAs per SM hide latency better: cfg4's
    // middle pass 3.40 (16 lines) vs 3.17 ms (8 lines), profiles/r6d_lfw.jsonl)
    static const bool lfw_on = [] {  // MOA_FFT_C64_LFW=0: 8 lines on the line-coalesced loads
        const char *e = std::getenv("MOA_FFT_C64_LFW");
        return !(e && e[0] == '0');
    }();
    const bool c64_wide = esize == 8 && logP == 5 && ((lfw_on && d.lf_load && d.twN <= 1) || (!d.lf_load && d.lf_store));
    // complex64 lines of >= 2^11 points (16 points per thread) storing
    // transposed: 8 lines per tile (64-byte store runs, one 1024-thread CTA per
    // SM at 64 registers) instead of the 4 that two CTAs per SM allow
    // (MOA_FFT_C64_WIDE2=0 restores 4)
    static const bool wide2_on = [] {
        const char *e = std::getenv("MOA_FFT_C64_WIDE2");
        return !(e && e[0] == '0');
    }();
    // (only where the stores are >= 1 MiB apart: the 2^30 plans' 2048-point last
    // pass 6.0 -> 4.1 ms; 4 KiB apart (batched 2^20) 0.245 -> 0.258 ms, r5m / r5o)
    const bool c64_wide2 = wide2_on && esize == 8 && logP == 4 && logR >= 11 && d.lf_store &&
                           d.out_kstr * esize >= (int64_t(1) << 20);
    const int64_t smem_cap = cap_env ? std::atoll(cap_env)
                                     : ((d.lf_load && kload >= (int64_t(1) << 20)) || c64_wide || c64_wide2 ? 200000 : 100 * 1024);
    // ablation knobs: lines per tile for line-coalesced / point-contiguous passes
    const char *wenv = std::getenv(lf ? "MOA_FFT_W_LF" : "MOA_FFT_W_PF");
    if (wenv && std::atoi(wenv) > 0) W = std::atoi(wenv);
    const int64_t max_thr = (logP == 5 && esize == 16) ? 256 : c64_wide2 ? 1024 : 512;  // complex128 radix-32 kernels keep 255 registers
    while (W > 1 && (W * R * esize > smem_cap || W * TPL > max_thr || ext0 % W)) W >>= 1;
    if (W < 1) W = 1;
    set_tile(d, dtype, W);
}

// a legal tile of exactly W lines? (used to give both passes of a fused pair the same CTA size)
static bool tile_ok(const moa_pass_desc_t &d, moa_dtype_t dtype, int64_t W) {
    const int esize = dtype == MOA_C128 ? 16 : 8;
    const int logR = d.logR, logP = psi_log_p(logR, dtype);
    const int64_t R = int64_t(1) << logR, TPL = R >> logP;
    const int64_t ext0 = d.ndig ? d.ext[0] : 1;
    return W >= 1 && W * TPL <= ((logP == 5 && esize == 16) ? 256 : 512) && W * R * esize <= 100 * 1024 && ext0 % W == 0;
}

static void set_tile(moa_pass_desc_t &d, moa_dtype_t dtype, int64_t W) {
    const int esize = dtype == MOA_C128 ? 16 : 8;
    const int slots = 128 / esize;
    const int logR = d.logR, logP = psi_log_p(logR, dtype);
    const int64_t R = int64_t(1) << logR, TPL = R >> logP;
    const bool lf = d.lf_load || d.lf_store;
    d.W = int32_t(W);
    d.threads = int32_t(W * TPL);
    // shared-memory line stride: the kernel stores element i of line l at
    // l*LS + i + i/16; pick LS (>= R + R/16) with the fewest bank conflicts over
    // every access pattern of this tile (exchange writes/reads of each step in
    // its thread mapping), evaluated exactly on the first warps
    (void)slots;
    const int64_t base = R + (R >> psi_pad_shift(logP));
    int64_t best = base, best_w = 1 << 30, best_t = int64_t(1) << 62;
    for (int64_t LS = base; LS < base + 2 * (128 / esize); LS++) {
        int64_t tot = 0;
        const int w = psi_bank_conflicts(logR, W, esize, d.lf_load, d.lf_store, LS, &tot, logP);
        if (w < best_w || (w == best_w && tot < best_t)) {
            best = LS;
            best_w = w;
            best_t = tot;
        }
    }
    d.line_pad = int32_t(best - R);
    const bool needs_smem = lf || logR > logP;
    d.smem_bytes = needs_smem ? int32_t(W * best * esize) : 0;
}

// Worst-case conflict degree (and total extra wavefronts) of the shared-memory
// accesses a pass tile makes, mirroring kernels.cu: Stockham step s has radix
// 16 except the last (the remainder), NS = 16^s, group j = t + u R/P writes
// element (j/NS) NS Q + j%NS + r NS; the next step reads t + m R/P.  Thread
// mapping: step 0 in the load side's, later steps in the store side's
// (line-fast: l = tid % W, t = tid / W; point-fast: l = tid / TPL, t = tid % TPL).
int psi_bank_conflicts(int logR, int64_t W, int esize, int lfA, int lfB, int64_t LS, int64_t *total, int logP) {
    if (logP < 0) logP = logR < 4 ? logR : 4;
    const int sh = psi_pad_shift(logP);
    const int64_t R = int64_t(1) << logR, P = int64_t(1) << logP, TPL = R / P, nthr = W * TPL;
    const int per = 128 / esize;  // lanes per shared-memory wavefront
    const int nstep = logR == 0 ? 1 : (logR + logP - 1) / logP;
    const int lql = logR - logP * (nstep - 1);
    auto phys = [sh](int64_t i) { return i + (i >> sh); };
    auto map = [&](int64_t tid, bool lf, int64_t &l, int64_t &t) {
        if (lf) { l = tid % W; t = tid / W; }
        else { l = tid / TPL; t = tid % TPL; }
    };
    int worst = 1;
    int64_t tot = 0;
    auto eval = [&](auto addr) {  // addr(tid) -> element address or -1
        for (int64_t w0 = 0; w0 < nthr && w0 < 256; w0 += 32)
            for (int ph = 0; ph < 32; ph += per) {
                int64_t seen[32];
                int ns = 0;
                int64_t bank[32];
                for (int ln = ph; ln < ph + per; ln++) {
                    const int64_t tid = w0 + ln;
                    if (tid >= nthr) continue;
                    const int64_t a = addr(tid);
                    bool dup = false;
                    for (int k = 0; k < ns; k++) dup |= seen[k] == a;
                    if (dup) continue;
                    seen[ns] = a;
                    bank[ns] = a % per;
                    ns++;
                }
                int dmax = 1;
                for (int k = 0; k < ns; k++) {
                    int c = 0;
                    for (int q = 0; q < ns; q++) c += bank[q] == bank[k];
                    if (c > dmax) dmax = c;
                }
                if (dmax > worst) worst = dmax;
                tot += dmax - 1;
            }
    };
    for (int s = 0; s < nstep - 1; s++) {
        const int64_t Q = int64_t(1) << (s == nstep - 1 ? lql : logP), NS = int64_t(1) << (logP * s), G = P / Q;
        const bool lf = s == 0 ? lfA : lfB;
        for (int64_t u = 0; u < G; u++)
            for (int64_t r = 0; r < Q; r++)
                eval([&](int64_t tid) {
                    int64_t l, t;
                    map(tid, lf, l, t);
                    const int64_t j = t + u * (R / P);
                    return l * LS + phys((j / NS) * NS * Q + (j % NS) + r * NS);
                });
        for (int64_t mm = 0; mm < P; mm++)
            eval([&](int64_t tid) {
                int64_t l, t;
                map(tid, lfB, l, t);
                return l * LS + phys(t + mm * TPL);
            });
    }
    if (nstep == 1 && lfA != lfB) {
        for (int64_t mm = 0; mm < P; mm++) {
            eval([&](int64_t tid) {
                int64_t l, t;
                map(tid, lfA, l, t);
                return l * LS + phys(t + mm * TPL);
            });
            eval([&](int64_t tid) {
                int64_t l, t;
                map(tid, lfB, l, t);
                return l * LS + phys(t + mm * TPL);
            });
        }
    }
    if (total) *total = tot;
    return worst;
}

moa_status_t psi_lift_passes(int64_t n, int64_t batch, moa_dtype_t dtype, const int64_t *radices, int nrad,
                             std::vector<moa_pass_desc_t> &out) {
    out.clear();
    if (nrad < 1 || nrad > MOA_MAX_PASSES) return fail(MOA_EINVAL, "psi: lifting must have 1..MOA_MAX_PASSES factors");
    int64_t prod = 1;
    for (int i = 0; i < nrad; i++) {
        int lr = log2_exact(radices[i]);
        if (lr < 0 || lr > 12) return fail(MOA_EINVAL, "psi: each radix must be a power of two <= 4096");
        prod *= radices[i];
    }
    if (prod != n) return fail(MOA_EINVAL, "psi: the radices must multiply to n");
    if (nrad + 1 > MOA_MAX_DIGITS + 1) return fail(MOA_EUNSUPPORTED, "psi: too many passes");
    const int P = nrad;
    if (P == 1) {
        moa_pass_desc_t d;
        desc_init(d, log2_exact(n));
        add_digit(d, batch, n, n, 0);
        d.in_kstr = d.out_kstr = 1;
        d.src = 0;
        d.dst = 1;
        psi_choose_tile(d, dtype);
        out.push_back(d);
        return MOA_OK;
    }
    for (int p = 0; p < P - 1; p++) {
        int64_t Sp = 1;
        for (int q = p + 1; q < P; q++) Sp *= radices[q];
        const int64_t Np = radices[p] * Sp, Op = batch * n / Np;
        moa_pass_desc_t d;
        desc_init(d, log2_exact(radices[p]));
        add_digit(d, Sp, 1, 1, 1);    // j: the contiguous inner index, weight exponent j*k
        add_digit(d, Op, Np, Np, 0);  // o: the rows above
        d.in_kstr = d.out_kstr = Sp;
        d.twN = Np;
        d.lf_load = d.lf_store = 1;
        d.src = p == 0 ? 0 : 2;
        d.dst = 2;
        psi_choose_tile(d, dtype);
        out.push_back(d);
    }
    {
        const int64_t RL = radices[P - 1];
        moa_pass_desc_t d;
        desc_init(d, log2_exact(RL));
        int64_t above = 1;  // R_0 ... R_{i-1}
        for (int i = 0; i < P - 1; i++) {
            const int64_t in_s = n / (above * radices[i]);  // n / (R_0 ... R_i)
            add_digit(d, radices[i], in_s, above, 0);
            above *= radices[i];
        }
        add_digit(d, batch, n, n, 0);
        d.in_kstr = 1;
        d.out_kstr = n / RL;
        d.lf_load = 0;
        d.lf_store = 1;
        d.src = 2;
        d.dst = 1;
        psi_choose_tile(d, dtype);
        out.push_back(d);
    }
    return MOA_OK;
}

moa_status_t psi_3d_passes(int64_t n0, int64_t n1, int64_t n2, int64_t howmany, moa_dtype_t dtype,
                           std::vector<moa_pass_desc_t> &out) {
    out.clear();
    const int64_t ns[3] = {n0, n1, n2};
    for (int a = 0; a < 3; a++) {
        int l = log2_exact(ns[a]);
        if (l < 0 || l > 12) return fail(MOA_EINVAL, "psi: 3-D extents must be powers of two <= 4096");
    }
    const int64_t plane = n1 * n2, vol = n0 * plane;
    // Layout choice (measured): complex128 uses the rotating
    // layouts (cfg5 22.5 -> 19.4 ms); complex64 the in-place axis passes (equal
    // time, no scratch).  MOA_FFT_3D_ROT = 0 / 1 / 2 overrides (ablations).
    const char *rot_env = std::getenv("MOA_FFT_3D_ROT");
    const char rot = rot_env && *rot_env ? rot_env[0] : (dtype == MOA_C128 ? '2' : '0');
    if (rot == '3' && howmany == 1 && n0 > 1 && n1 > 1 && n2 > 1) {
        // z in place (contiguous both sides), then y and x with strided loads
        // (one row apart: the L2 box prefetch applies) and plane-strided stores
        // (merged into full lines in L2):
        //   in [x][y][z] --z--> out [x][y][z] --y--> scratch [y][x][z] --x--> out [x][y][z]
        moa_pass_desc_t d;
        desc_init(d, log2_exact(n2));  // z: line (y, x), in place
        add_digit(d, n1, n2, n2, 0);
        add_digit(d, n0, plane, plane, 0);
        d.in_kstr = d.out_kstr = 1;
        d.src = 0;
        d.dst = 1;
        psi_choose_tile(d, dtype);
        out.push_back(d);
        desc_init(d, log2_exact(n1));  // y: line (z, x) of [x][y][z], k_y -> scratch[k_y][x][z]
        add_digit(d, n2, 1, 1, 0);
        add_digit(d, n0, plane, n2, 0);
        d.in_kstr = n2;
        d.out_kstr = n0 * n2;
        d.lf_load = d.lf_store = 1;
        d.src = 1;
        d.dst = 2;
        psi_choose_tile(d, dtype);
        out.push_back(d);
        desc_init(d, log2_exact(n0));  // x: line (z, y) of [y][x][z], k_x -> out[k_x][y][z]
        add_digit(d, n2, 1, 1, 0);
        add_digit(d, n1, n0 * n2, n2, 0);
        d.in_kstr = n2;
        d.out_kstr = plane;
        d.lf_load = d.lf_store = 1;
        d.src = 2;
        d.dst = 1;
        psi_choose_tile(d, dtype);
        out.push_back(d);
        return MOA_OK;
    }
    if (rot == '2' && howmany == 1 && n0 > 1 && n1 > 1 && n2 > 1) {
        // Rotating layouts, axis order z, x, y: every pass reads contiguous
        // lines and stores transposed so the next axis becomes contiguous (the
        // strided side is always a store, merged into full lines in L2); every
        // store stride is one row (n0, n1 or n2 elements), never a plane:
        //   in [x][y][z] --z--> out [y][z][x] --x--> scratch [z][x][y] --y--> out [x][y][z]
        moa_pass_desc_t d;
        desc_init(d, log2_exact(n2));  // z: line (x, y), k_z -> out[y][k_z][x]
        add_digit(d, n0, plane, 1, 0);
        add_digit(d, n1, n2, n2 * n0, 0);
        d.in_kstr = 1;
        d.out_kstr = n0;
        d.lf_store = 1;
        d.src = 0;
        d.dst = 1;
        psi_choose_tile(d, dtype);
        out.push_back(d);
        desc_init(d, log2_exact(n0));  // x: line (y, z) of [y][z][x], k_x -> scratch[z][k_x][y]
        add_digit(d, n1, n2 * n0, 1, 0);
        add_digit(d, n2, n0, n0 * n1, 0);
        d.in_kstr = 1;
        d.out_kstr = n1;
        d.lf_store = 1;
        d.src = 1;
        d.dst = 2;
        psi_choose_tile(d, dtype);
        out.push_back(d);
        desc_init(d, log2_exact(n1));  // y: line (z, x) of [z][x][y], k_y -> out[x][k_y][z]
        add_digit(d, n2, n0 * n1, 1, 0);
        add_digit(d, n0, n1, plane, 0);
        d.in_kstr = 1;
        d.out_kstr = n2;
        d.lf_store = 1;
        d.src = 2;
        d.dst = 1;
        psi_choose_tile(d, dtype);
        out.push_back(d);
        return MOA_OK;
    }
    if (rot == '1' && howmany == 1 && n0 > 1 && n1 > 1 && n2 > 1) {
        // Rotating layouts: every pass reads contiguous lines and stores
        // transposed so the next axis becomes contiguous (the strided side is
        // always a store, which the L2 merges into full lines):
        //   in  [x][y][z] --z--> out [x][z][y] --y--> scratch [z][y][x] --x--> out [x][y][z]
        moa_pass_desc_t d;
        desc_init(d, log2_exact(n2));  // z: line (y, x), k_z -> out[x][k_z][y]
        add_digit(d, n1, n2, 1, 0);
        add_digit(d, n0, plane, plane, 0);
        d.in_kstr = 1;
        d.out_kstr = n1;
        d.lf_store = 1;
        d.src = 0;
        d.dst = 1;
        psi_choose_tile(d, dtype);
        out.push_back(d);
        desc_init(d, log2_exact(n1));  // y: line (x, z) of [x][z][y], k_y -> scratch[z][k_y][x]
        add_digit(d, n0, plane, 1, 0);
        add_digit(d, n2, n1, n1 * n0, 0);
        d.in_kstr = 1;
        d.out_kstr = n0;
        d.lf_store = 1;
        d.src = 1;
        d.dst = 2;
        psi_choose_tile(d, dtype);
        out.push_back(d);
        desc_init(d, log2_exact(n0));  // x: line (z, y) of [z][y][x], k_x -> out[k_x][y][z]
        add_digit(d, n2, n1 * n0, 1, 0);
        add_digit(d, n1, n0, n2, 0);
        d.in_kstr = 1;
        d.out_kstr = plane;
        d.lf_store = 1;
        d.src = 2;
        d.dst = 1;
        psi_choose_tile(d, dtype);
        out.push_back(d);
        return MOA_OK;
    }
    // axis 2: contiguous lines
    {
        moa_pass_desc_t d;
        desc_init(d, log2_exact(n2));
        add_digit(d, n1, n2, n2, 0);
        add_digit(d, n0, plane, plane, 0);
        add_digit(d, howmany, vol, vol, 0);
        d.in_kstr = d.out_kstr = 1;
        d.src = 0;
        d.dst = 1;
        psi_choose_tile(d, dtype);
        if (n2 > 1) out.push_back(d);
    }
    // axis 1: lines along stride n2, tile over contiguous j2
    {
        moa_pass_desc_t d;
        desc_init(d, log2_exact(n1));
        add_digit(d, n2, 1, 1, 0);
        add_digit(d, n0, plane, plane, 0);
        add_digit(d, howmany, vol, vol, 0);
        d.in_kstr = d.out_kstr = n2;
        d.lf_load = d.lf_store = 1;
        d.src = out.empty() ? 0 : 1;
        d.dst = 1;
        psi_choose_tile(d, dtype);
        if (n1 > 1) out.push_back(d);
    }
    // axis 0
    {
        moa_pass_desc_t d;
        desc_init(d, log2_exact(n0));
        add_digit(d, n2, 1, 1, 0);
        add_digit(d, n1, n2, n2, 0);
        add_digit(d, howmany, vol, vol, 0);
        d.in_kstr = d.out_kstr = plane;
        d.lf_load = d.lf_store = 1;
        d.src = out.empty() ? 0 : 1;
        d.dst = 1;
        psi_choose_tile(d, dtype);
        if (n0 > 1) out.push_back(d);
    }
    if (out.empty()) {  // 1 x 1 x 1: identity copy as a 1-point pass
        moa_pass_desc_t d;
        desc_init(d, 0);
        add_digit(d, howmany, 1, 1, 0);
        d.in_kstr = d.out_kstr = 1;
        d.src = 0;
        d.dst = 1;
        psi_choose_tile(d, dtype);
        out.push_back(d);
    }
    return MOA_OK;
}

// L2-level lifting: a two-pass lifting of many independent
// rows (the cfg2 shape) becomes one fused pass pair whose intermediate lives in
// an L2-resident ring of row buffers.  Group = one row: pass A's lines (the
// strided columns j of row b) and pass B's lines (the rows k_0 of row b) both
// have the row b as their last (slowest) digit; on the ring side that digit's
// stride becomes (b mod slots) * n.
// Fuse passes[i] and passes[i+1] into an L2-staged pair when (a) both have the
// same slowest line digit -- the group -- with one stride G on the
// intermediate's side (A's store, B's load), (b) a group (G elements) fits the
// ring budget a few times over, (c) the CTA sizes can be equalised.
static int fuse_two(std::vector<moa_pass_desc_t> &passes, size_t i, moa_dtype_t dtype, int64_t min_groups,
                    int64_t ring_budget) {
    const char *env = std::getenv("MOA_FFT_FUSE");
    if (env && env[0] == '0') return 0;
    if (i + 1 >= passes.size()) return 0;
    const int64_t esize = dtype == MOA_C128 ? 16 : 8;
    moa_pass_desc_t &A = passes[i], &B = passes[i + 1];
    if (A.ring || B.ring || A.ndig < 2 || B.ndig < 2) return 0;
    const int la = A.ndig - 1, lb = B.ndig - 1;
    const int64_t groups = A.ext[la], G = A.out_str[la];
    if (B.ext[lb] != groups || B.in_str[lb] != G || groups < min_groups) return 0;
    if (A.dst != B.src || A.dst < 0) return 0;
    if (G * esize * 4 > ring_budget) return 0;
    if (A.logR < 5 || A.logR > 10 || B.logR < 5 || B.logR > 10) return 0;
    if (A.threads != B.threads) {  // equalise the CTA size: widen the narrower tile, else narrow the wider
        moa_pass_desc_t &lo = A.threads < B.threads ? A : B;
        moa_pass_desc_t &hi = A.threads < B.threads ? B : A;
        const int64_t W = int64_t(lo.W) * hi.threads / lo.threads;
        if (tile_ok(lo, dtype, W)) {
            set_tile(lo, dtype, W);
        } else {
            const int64_t Wh = int64_t(hi.W) * lo.threads / hi.threads;
            if (Wh < 1 || !tile_ok(hi, dtype, Wh)) return 0;
            set_tile(hi, dtype, Wh);
        }
        if (A.threads != B.threads) return 0;
    }
    const char *mb = std::getenv("MOA_FFT_RING_MB");  // ablation: ring size budget
    if (mb) ring_budget = std::atoll(mb) << 20;
    int64_t slots = 4;
    while (slots * 2 * G * esize <= ring_budget && slots < 128 && slots * 4 <= groups) slots *= 2;
    for (moa_pass_desc_t *d : {&A, &B}) {
        d->ring_slots = int32_t(slots);
        d->ring_lag = int32_t(slots / 2);
        d->ring_discard = !(env && env[0] == '2');
        d->ring_groups = groups;
        d->ring_G = G;
    }
    A.ring = 2;
    A.out_str[la] = 0;  // the group digit addresses the ring slot
    A.dst = -1;
    B.ring = 1;
    B.in_str[lb] = 0;
    B.src = -1;
    return 1;
}

// L2-level lifting: a two-pass lifting of many independent
// rows (the cfg2 shape) becomes one fused pass pair whose intermediate lives in
// an L2-resident ring of row buffers (group = one row).
int psi_fuse_pairs(std::vector<moa_pass_desc_t> &passes, const std::vector<int64_t> &radices, int64_t n, int64_t batch,
                   moa_dtype_t dtype) {
    (void)n;
    (void)batch;
    // opt-in (MOA_FFT_FUSE=1, or 2 without the discard) until the fused launch
    // beats the two single passes, which already run near the HBM roofline
    // each
    const char *e = std::getenv("MOA_FFT_FUSE");
    if (!e || (e[0] != '1' && e[0] != '2')) return 0;
    if (passes.size() != 2 || radices.size() != 2) return 0;
    return fuse_two(passes, 0, dtype, 16, int64_t(32) << 20);
}

// 3-D: the z- and y-passes of one x-plane form a group (the plane), so the
// pair costs one HBM round trip instead of two.
int psi_fuse_3d(std::vector<moa_pass_desc_t> &passes, moa_dtype_t dtype) {
    const char *e = std::getenv("MOA_FFT_FUSE");  // opt-in, as psi_fuse_pairs
    if (!e || (e[0] != '1' && e[0] != '2')) return 0;
    if (passes.size() != 3) return 0;
    return fuse_two(passes, 0, dtype, 8, int64_t(64) << 20);
}

// The cluster level of the lifting (kernels.cu cluster_kernel): a two-pass
// lifting of independent groups -- pass A's last line digit is the group, its
// group stride G on the output side equals pass B's on the input side -- whose
// group (G elements) fits the shared memory of one thread-block cluster of C
// CTAs, C = pass A's tiles per group = pass B's tiles per group (<= 16).
// Pass B's tile c must read exactly slice c of the group (contiguous rows of
// R_B points), so its loads come from its own CTA's shared memory.
int psi_cluster_pair(std::vector<moa_pass_desc_t> &passes, moa_dtype_t dtype, int64_t max_ctas, int64_t max_threads) {
    if (passes.size() != 2) return 0;
    moa_pass_desc_t &A = passes[0], &B = passes[1];
    const int64_t esize = dtype == MOA_C128 ? 16 : 8;
    if (A.ring || B.ring || A.kind || B.kind || A.ndig != 2 || B.ndig != 2) return 0;
    if (A.logR < 5 || A.logR > 9 || B.logR < 5 || B.logR > 9) return 0;
    const int lp = psi_log_p(A.logR, dtype);
    if (psi_log_p(B.logR, dtype) != lp) return 0;  // one CTA size for both passes
    if (A.dst != B.src || A.dst < 0) return 0;
    const int64_t groups = A.ext[1], G = A.out_str[1], RA = int64_t(1) << A.logR, RB = int64_t(1) << B.logR;
    if (B.ext[1] != groups || B.in_str[1] != G || (G & (G - 1))) return 0;
    // pass B: contiguous rows of R_B points, rows adjacent -> tile c reads [c G/C, (c+1) G/C)
    if (B.in_kstr != 1 || B.in_str[0] != RB || B.ext[0] * RB != G || B.lf_load) return 0;
    // C CTAs per group: pass A's tile c = lines [c W_A, (c+1) W_A), pass B's the
    // same with W_B; both tiles have n / (C P) threads.  The largest C (smallest
    // CTAs, most clusters resident) with a legal tile on both sides
    const int64_t cap_thr = (esize == 16 && lp == 5) ? 256 : 512;
    const int64_t smem_cap = 100 * 1024;
    for (int64_t C = max_ctas < 16 ? max_ctas : 16; C >= 2; C >>= 1) {
        if (A.ext[0] % C || B.ext[0] % C) continue;
        const int64_t WA = A.ext[0] / C, WB = B.ext[0] / C;
        const int64_t thr = WA * (RA >> lp);
        if (thr != WB * (RB >> lp) || thr > cap_thr || thr > max_threads || thr < 64) continue;
        if (WA * (RA + RA / 16 + 32) * esize > smem_cap || WB * (RB + RB / 16 + 32) * esize > smem_cap ||
            (G / C) * esize > smem_cap)
            continue;
        if (WA != A.W) set_tile(A, dtype, WA);
        if (WB != B.W) set_tile(B, dtype, WB);
        for (moa_pass_desc_t *d : {&A, &B}) {
            d->ring_slots = int32_t(C);
            d->ring_lag = A.dst;  // (the intermediate's buffer id, for psi_uncluster)
            d->ring_discard = 0;
            d->ring_groups = groups;
            d->ring_G = G;
        }
        A.ring = 3;
        A.dst = -1;
        B.ring = 4;
        B.src = -1;
        return 1;
    }
    return 0;
}

// Back to the two plain passes (the plan variants that rewrite the last pass,
// e.g. the lifted output order, take the plain form).
void psi_uncluster(std::vector<moa_pass_desc_t> &passes) {
    for (size_t i = 0; i + 1 < passes.size(); i++) {
        moa_pass_desc_t &A = passes[i], &B = passes[i + 1];
        if (A.ring != 3 || B.ring != 4) continue;
        A.dst = B.src = A.ring_lag;
        for (moa_pass_desc_t *d : {&A, &B}) {
            d->ring = 0;
            d->ring_slots = d->ring_lag = d->ring_discard = 0;
            d->ring_groups = d->ring_G = 0;
        }
    }
}

// Four-pass lifting n = R0 R1 R2 R3 run as two L2-staged pairs, so a single
// huge transform costs two HBM round trips (SURVEY §8(d.3)'s count for the
// 2^14 x 2^14 / 2^15 x 2^15 six-step) with every per-CTA block <= 2^10 points.
//   pair (0,1): group = W consecutive j' (j = i1 S1 + j', S1 = R2 R3); pass 0
//     lines (l, i1 | g, b), pass 1 lines (l, k0 | g, b); ring layout
//     [(k0 R1 + i1) W + l]; pass 1 writes the global intermediate.
//   pair (2,3): group = (k1, k0 >> log2 W); pass 2 lines (j, l, k1 | g0, b) with
//     l = k0 mod W, pass 3 lines (l, k2, k1 | g0, b); ring layout
//     [(l R2 + k2) R3 + i3]; pass 3 stores natural order
//     X[k0 + R0 k1 + R0 R1 k2 + R0 R1 R2 k3].
// Digits after `|` are the group (the slowest line bits); their ring-side
// strides are 0 (the slot offset replaces them).
static moa_status_t lift4_fused(int64_t n, int64_t batch, moa_dtype_t dtype, const int64_t *R,
                                std::vector<moa_pass_desc_t> &out) {
    out.clear();
    const int64_t esize = dtype == MOA_C128 ? 16 : 8;
    const int64_t W = 128 / esize;
    const int64_t R0 = R[0], R1 = R[1], R2 = R[2], R3 = R[3];
    const int64_t S1 = R2 * R3, S0 = R1 * S1, N1 = S0, N2 = S1;
    if (R0 < W || S1 < W || R3 < W) return fail(MOA_EUNSUPPORTED, "psi: lift4 needs R0, R3 >= W");
    for (int i = 0; i < 4; i++)
        if (R[i] < 32 || R[i] > 1024) return fail(MOA_EUNSUPPORTED, "psi: lift4 radices must be in [32, 1024]");
    const int64_t G01 = R0 * R1 * W, G23 = W * R2 * R3;
    const int64_t g01 = (S1 / W) * batch, g23 = R1 * (R0 / W) * batch;
    const char *mb = std::getenv("MOA_FFT_RING_MB");  // ablation: ring size budget
    const int64_t budget = mb ? std::atoll(mb) << 20 : int64_t(32) << 20;
    auto ring = [&](moa_pass_desc_t &d, int side, int64_t groups, int64_t G) {
        int64_t slots = 4;
        while (slots * 2 * G * esize <= budget && slots < 256 && slots * 2 <= groups) slots *= 2;
        d.ring = side;
        d.ring_slots = int32_t(slots);
        d.ring_lag = int32_t(slots / 2);
        d.ring_discard = 1;
        d.ring_groups = groups;
        d.ring_G = G;
    };
    moa_pass_desc_t d;
    // pass 0: in -> ring
    desc_init(d, log2_exact(R0));
    add_digit(d, W, 1, 1, 1);                 // l   (j' = g W + l)
    add_digit(d, R1, S1, W, S1);              // i1
    add_digit(d, S1 / W, W, 0, W);            // g   (group)
    add_digit(d, batch, n, 0, 0);             // b   (group)
    d.in_kstr = S0;
    d.out_kstr = R1 * W;
    d.twN = n;
    d.lf_load = d.lf_store = 1;
    d.src = 0;
    d.dst = -1;
    ring(d, 2, g01, G01);
    out.push_back(d);
    // pass 1: ring -> scratch (global intermediate, position k0 N1 + k1 S1 + j')
    desc_init(d, log2_exact(R1));
    add_digit(d, W, 1, 1, 1);                 // l
    add_digit(d, R0, R1 * W, N1, 0);          // k0
    add_digit(d, S1 / W, 0, W, W);            // g
    add_digit(d, batch, 0, n, 0);             // b
    d.in_kstr = W;
    d.out_kstr = S1;
    d.twN = N1;
    d.lf_load = d.lf_store = 1;
    d.src = -1;
    d.dst = 2;
    ring(d, 1, g01, G01);
    out.push_back(d);
    // pass 2: scratch -> ring (lines o = k0 R1 + k1, j = i3)
    desc_init(d, log2_exact(R2));
    add_digit(d, R3, 1, 1, 1);                // j
    add_digit(d, W, R1 * N2, R2 * R3, 0);     // l = k0 mod W
    add_digit(d, R1, N2, 0, 0);               // k1        (group)
    add_digit(d, R0 / W, W * R1 * N2, 0, 0);  // g0 = k0 / W (group)
    add_digit(d, batch, n, 0, 0);             // b         (group)
    d.in_kstr = R3;
    d.out_kstr = R3;
    d.twN = N2;
    d.lf_load = d.lf_store = 1;
    d.src = 2;
    d.dst = -1;
    ring(d, 2, g23, G23);
    out.push_back(d);
    // pass 3: ring -> out, natural order
    desc_init(d, log2_exact(R3));
    add_digit(d, W, R2 * R3, 1, 0);           // l
    add_digit(d, R2, R3, R0 * R1, 0);         // k2
    add_digit(d, R1, 0, R0, 0);               // k1
    add_digit(d, R0 / W, 0, W, 0);            // g0
    add_digit(d, batch, 0, n, 0);             // b
    d.in_kstr = 1;
    d.out_kstr = R0 * R1 * R2;
    d.lf_load = 0;
    d.lf_store = 1;
    d.src = -1;
    d.dst = 1;
    ring(d, 1, g23, G23);
    out.push_back(d);
    for (auto &x : out) {  // the group structure needs tiles of exactly W lines
        psi_choose_tile(x, dtype);
        if (x.W != W && tile_ok(x, dtype, W)) set_tile(x, dtype, W);
    }
    // both passes of a pair need one CTA size: widen the narrower tile
    for (int p = 0; p < 4; p += 2) {
        moa_pass_desc_t &A = out[p], &B = out[p + 1];
        if (A.W != W || B.W != W) return fail(MOA_EUNSUPPORTED, "psi: lift4 tile must cover W lines");
        if (A.threads != B.threads) return fail(MOA_EUNSUPPORTED, "psi: lift4 pair CTA sizes differ");
    }
    return MOA_OK;
}

// Ablation (MOA_FFT_W_PASS="i:W,j:W"): pass i of a 1-D plan gets W lines per
// tile (when W divides the line digit and the tile fits 1024 threads and 227 KiB).
static void apply_w_pass_env(std::vector<moa_pass_desc_t> &v, moa_dtype_t dtype) {
    const char *e = std::getenv("MOA_FFT_W_PASS");
    if (!e) return;
    const int esize = dtype == MOA_C128 ? 16 : 8;
    for (const char *q = e; *q;) {
        char *end = nullptr;
        const long i = std::strtol(q, &end, 10);
        if (!end || *end != ':') return;
        const long W = std::strtol(end + 1, &end, 10);
        if (i >= 0 && size_t(i) < v.size() && W >= 1 && (W & (W - 1)) == 0) {
            moa_pass_desc_t &d = v[size_t(i)];
            const int64_t R = int64_t(1) << d.logR, TPL = R >> psi_log_p(d.logR, dtype);
            const int64_t ext0 = d.ndig ? d.ext[0] : 1;
            if (ext0 % W == 0 && W * TPL <= 1024 && W * (R + R / 16 + 32) * esize <= 227 * 1024) set_tile(d, dtype, W);
        }
        if (*end != ',') return;
        q = end + 1;
    }
}

moa_status_t psi_build(int64_t n, int64_t batch, moa_dtype_t dtype, const std::vector<int64_t> &radices, bool planned,
                       std::vector<moa_pass_desc_t> &out) {
    // the four-factor lifting as two L2-staged pairs is opt-in (MOA_FFT_LIFT4=1):
    // measured round 1, the four plain passes are faster (cfg3 5.55 vs 6.70 ms,
    // cfg4 12.9 vs 21.5 ms)
    (void)planned;
    const char *l4 = std::getenv("MOA_FFT_LIFT4");
    // (the pairs take the factors as (R, R, R', R'), larger first)
    std::vector<int64_t> r4(radices);
    std::sort(r4.begin(), r4.end(), [](int64_t x, int64_t y) { return x > y; });
    if (l4 && l4[0] == '1' && r4.size() == 4 && r4[0] == r4[1] && r4[2] == r4[3]) {
        std::vector<moa_pass_desc_t> v;
        if (lift4_fused(n, batch, dtype, r4.data(), v) == MOA_OK) {
            out.swap(v);
            return MOA_OK;
        }
    }
    moa_status_t st = psi_lift_passes(n, batch, dtype, radices.data(), int(radices.size()), out);
    if (st) return st;
    apply_w_pass_env(out, dtype);
    if (!psi_fuse_pairs(out, radices, n, batch, dtype)) {
        // the cluster level, by default where it measured faster than the two
        // passes (profiles/r6i_cluster2.jsonl, 512 MiB of rows): complex128 rows
        // on 8-CTA clusters of <= 128 threads (2^13: 0.88x, 2^14: 0.93x; 2^15
        // at 256 threads 1.25x; complex64 1.17-1.48x), and any <= 8-CTA,
        // <= 256-thread cluster pair when the whole batch is <= 32 MiB (one
        // launch instead of two: 0.74-0.91x).  16-CTA clusters -- cfg2's
        // 2^16-point rows -- are slower (0.98 vs 0.64 ms): only with
        // MOA_FFT_CLUSTER=1 (any C <= 16); MOA_FFT_CLUSTER=0: never
        const char *ce = std::getenv("MOA_FFT_CLUSTER");
        if (!ce) {
            const int64_t bytes = n * batch * (dtype == MOA_C128 ? 16 : 8);
            const int64_t mt = bytes <= (int64_t(32) << 20) ? 256 : dtype == MOA_C128 ? 128 : 0;
            if (mt) psi_cluster_pair(out, dtype, 8, mt);
        } else if (ce[0] == '1') {
            psi_cluster_pair(out, dtype, 16, 512);
        }
    }
    return MOA_OK;
}

// Planner (step a1): the fewest passes whose per-pass line fits one CTA tile,
// radices as equal as possible (largest first) so every pass is one HBM round
// trip of similar cost.  Per-CTA limit: 2^9 points for the line-coalesced
// passes (8 adjacent lines x 2^9 x 16 B = 64 KiB), 2^12 for the last pass.
moa_status_t plan_radices(int64_t n, int64_t batch, moa_dtype_t dtype, std::vector<int64_t> &radices) {
    (void)batch;
    radices.clear();
    const int t = log2_exact(n);
    if (t < 0) return fail(MOA_EINVAL, "plan: n must be a power of two");
    const int max_single = 12;                      // one pass holds 2^12 points per line
    const int max_mid = dtype == MOA_C128 ? 9 : 10;  // strided passes: W adjacent lines per tile
    if (t <= max_single) {
        radices.push_back(n);
        return MOA_OK;
    }
    // large transforms: four balanced factors (R, R, R', R') of <= 2^8 points,
    // each pass one shared-memory exchange (the L1/smem data path
    // costs one 16-byte move per load, store and exchange half, so passes with two
    // exchanges (R = 2^9, 2^10) run below the HBM roofline); needs an even t.
    // Order (R, R', R', R): the larger radix on the first and last passes --
    // measured 2^30 c64 11.84 -> 11.33 ms, 2^26 c64 0.756 -> 0.714 ms, 2^26 c128
    // 1.35 -> 1.32 ms against (R, R, R', R') (the strided middle passes run
    // closest to the copy roofline with the shorter lines)
    // Since the 512/1024-point lines run radix 32 (one exchange), t = 26 and 28
    // take three passes instead (general rule below: 2^26 c128 1.31 -> 1.06 ms,
    // 2^28 c128 5.14 -> 4.94 ms, c64 -10 / -6 %, profiles/r1_s7_three_pass.txt);
    // t = 30, 32 keep four (2^30 c64: 11.1 vs 13.5 ms with 1024^3).  The opt-in
    // L2 pairs (MOA_FFT_LIFT4) need the four factors.
    const char *l4env = std::getenv("MOA_FFT_LIFT4");
    const bool lift4 = l4env && l4env[0] == '1';
    // complex64 2^30 (cfg4): three 1024-point passes since the packed FP32x2
    // arithmetic and the 16-line tiles (11.1-11.3 ms against 11.7 ms for the
    // four-pass (256, 128, 128, 256), profiles/r3c_c64.jsonl, r3d_c64.jsonl)
    if (!lift4 && dtype == MOA_C64 && t == 30) {
        for (int k = 0; k < 3; k++) radices.push_back(int64_t(1) << 10);
        return MOA_OK;
    }
    // The paper chooses its blocking size c by measurement; so does
    // this planner where a sweep of every 2-4-factor lifting of one transform
    // beat the rules below (profiles/r3l_planner.jsonl, one B200): complex128
    // prefers a contiguous 1024-point last pass (2^20 0.0274 -> 0.0241 ms, 2^24
    // 0.272 -> 0.268, 2^27 2.26 -> 2.13, 2^29 12.1 -> 10.1, 2^30 23.0 -> 22.3 ms);
    // complex64 two passes at 2^20 / 2^21 and the larger radix first at 2^25 / 2^26.
    if (!lift4) {
        // (batched rows, 1 GiB of them, r3n_batched.jsonl / r3o_cfg2.jsonl: complex128
        // 2^18 [256, 1024] -3 %, complex64 2^13 [32, 256] / 2^14 [64, 256] -2.4 / -3.8 %)
        static const int c128_tab[][4] = {{18, 8, 10, 0}, {20, 10, 10, 0}, {21, 10, 11, 0}, {24, 7, 7, 10},
                                          {25, 7, 8, 10},  {26, 8, 8, 10},  {27, 8, 9, 10},  {28, 9, 9, 10},
                                          {29, 9, 10, 10}, {30, 10, 10, 10}};
        static const int c64_tab[][4] = {{13, 5, 8, 0},  {14, 6, 8, 0}, {20, 9, 11, 0},
                                         {21, 10, 11, 0}, {25, 9, 8, 8}, {26, 9, 8, 9}};
        const int(*tab)[4] = dtype == MOA_C128 ? c128_tab : c64_tab;
        const int cnt = dtype == MOA_C128 ? 10 : 6;
        for (int i = 0; i < cnt; i++)
            if (tab[i][0] == t) {
                for (int k = 1; k < 4; k++)
                    if (tab[i][k]) radices.push_back(int64_t(1) << tab[i][k]);
                return MOA_OK;
            }
    }
    if (t >= (lift4 ? 26 : 30) && t % 2 == 0 && t <= 32) {
        const int a = (t + 3) / 4, b = t / 2 - a;
        for (int x : {a, b, b, a}) radices.push_back(int64_t(1) << x);
        return MOA_OK;
    }
    // P passes: P-1 strided passes of <= max_mid bits plus a last pass <= max_last
    // (2^11 / 2^10 points: a longer last line needs two exchanges and measured
    // slower than one more pass -- 2^21 c128 0.297 -> 0.268 ms, 2^22 c64 0.375 ->
    // 0.281 ms, profiles/r1_s7_last_pass_cap.txt)
    const int max_last = dtype == MOA_C128 ? 11 : 10;
    int P = 2;
    while ((P - 1) * max_mid + max_last < t) P++;
    // distribute t bits: balanced, with the last pass taking the remainder
    std::vector<int> bits(P, t / P);
    for (int i = 0; i < t % P; i++) bits[P - 1 - i]++;
    // respect the per-pass caps by moving bits to the last pass
    for (int i = 0; i < P - 1; i++)
        while (bits[i] > max_mid) {
            bits[i]--;
            bits[P - 1]++;
        }
    for (int b : bits) radices.push_back(int64_t(1) << b);
    return MOA_OK;
}

}  // namespace moa

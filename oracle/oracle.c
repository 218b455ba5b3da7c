/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY (the CPU oracle).
 *
 * Plain, slow, obviously-correct host implementation of what the hot path
 * computes, written from PAPER.md (Mullin & Raynolds, "Conformal Computing").
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  It shares no code, header,
 * table or constant generator with the CUDA path (paper_0803_2386_b200/).
 *
 * Precision: complex128 throughout (interleaved re,im doubles); complex64
 * inputs are promoted exactly by the caller.  Twiddles are computed directly
 * from the exact integer exponent (never by recurrence), in long double.
 *
 * Functions and the passage each follows ("P:a-b" = PAPER.md lines):
 *   orc_bitrev_perm / orc_bitrev  -- O1, P_n, the bit-reversal permutation,
 *                                    Fig. vanloan_fft line (1).
 *   orc_fft_radix2                -- O1+O2: x <- P_n x, then the in-place
 *                                    radix-2 loop nest `fftpsirad2`,
 *                                    Fig. fftpsirad2 P:206-230 (= Fig. rad2_fft
 *                                    P:1953-1977) with the forward sign
 *                                    (reading R1) and P_n applied
 *                                    first (reading R2).
 *   orc_dft_direct                -- O3, the definition X[k] = sum_j x[j] w^{jk},
 *                                    w = e^{-2 pi i/n} (Van Loan "Output: The FFT
 *                                    of x"); long double accumulation.
 *   orc_dft_bins                  -- O3 restricted to a list of output bins
 *                                    (sampled parity at full size).
 *   orc_dft3_bins                 -- O3 for the separable 3-D DFT (sampled bins).
 *   orc_fft_lifted                -- O4, the cache-optimized (lifted) FFT of
 *                                    Ch.3: P_n, then for each level l the
 *                                    in-block stages with weights
 *                                    w_L^{sigma + j c^l}, a
 *                                    reshape-transpose S between levels
 *                                    (Eq. reshape3, loop of
 *                                    Fig. trans_rshp_code P:2934-2965 with the
 *                                    outer bound read as c, reading R4), and the
 *                                    final transpose F (Fig. final_trans_code
 *                                    P:3042-3069).  Level/stage counts per
 *                                    P:2791-2800 (reading R6).
 *   orc_fft3d                     -- O5, multi-dimensional FFT as 1-D FFTs
 *                                    along each axis (P:641 footnote,
 *                                    P:3194-3196), each line by orc_fft_radix2.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_PI_L 3.141592653589793238462643383279502884L

static int ilog2_exact(int64_t n) {
    if (n < 1) return -1;
    int t = 0;
    while (((int64_t)1 << t) < n) t++;
    return (((int64_t)1 << t) == n) ? t : -1;
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* e^{-2 pi i e / L} for an exact integer exponent 0 <= e < L (forward sign). */
static void omega(int64_t e, int64_t L, long double *re, long double *im) {
    long double a = 2.0L * ORC_PI_L * (long double)e / (long double)L;
    *re = cosl(a);
    *im = -sinl(a);
}

/* ---- O1: P_n ------------------------------------------------------------ */
static int64_t bitrev_t(int64_t i, int t) {
    int64_t r = 0;
    for (int b = 0; b < t; b++)
        if (i & ((int64_t)1 << b)) r |= (int64_t)1 << (t - 1 - b);
    return r;
}

/* perm[i] = bit-reverse of i over t = log2 n bits.  Returns -1 if n is not 2^t. */
int orc_bitrev_perm(int64_t n, int64_t *perm) {
    int t = ilog2_exact(n);
    if (t < 0) return -1;
    for (int64_t i = 0; i < n; i++) perm[i] = bitrev_t(i, t);
    return 0;
}

/* x <- P_n x in place: swap x[i] and x[r] when i < r. */
int orc_bitrev(double *x, int64_t n) {
    int t = ilog2_exact(n);
    if (t < 0) return -1;
    /* each pair (i, r) is swapped by exactly one i, so the loop is race-free */
#pragma omp parallel for schedule(static) if (n >= 65536)
    for (int64_t i = 0; i < n; i++) {
        int64_t r = bitrev_t(i, t);
        if (i < r) {
            double a = x[2 * i], b = x[2 * i + 1];
            x[2 * i] = x[2 * r];
            x[2 * i + 1] = x[2 * r + 1];
            x[2 * r] = a;
            x[2 * r + 1] = b;
        }
    }
    return 0;
}

/* ---- O2: fftpsirad2 ------------------------------------------------------- */
/* One stage q of Fig. fftpsirad2: L = 2^q,
 *   weight(row) = EXP(-2 pi i row / L)                (forward sign, reading R1)
 *   do col' = 0, n-1, L ; do row = 0, L/2-1
 *      c = weight(row) * x(col'+row+L/2); d = x(col'+row)
 *      x(col'+row) = d + c; x(col'+row+L/2) = d - c                         */
static inline void butterfly(double *x, int64_t col, int64_t row, int64_t h, const double *wt) {
    double wr = wt[2 * row], wi = wt[2 * row + 1];
    double *pd = x + 2 * (col + row), *pc = x + 2 * (col + row + h);
    double cr = wr * pc[0] - wi * pc[1]; /* c = weight(row) * x(col'+row+L/2) */
    double ci = wr * pc[1] + wi * pc[0];
    double dr = pd[0], di = pd[1];       /* d = x(col'+row) */
    pd[0] = dr + cr;                     /* x(col'+row) = d + c */
    pd[1] = di + ci;
    pc[0] = dr - cr;                     /* x(col'+row+L/2) = d - c */
    pc[1] = di - ci;
}

static void radix2_stage(double *x, int64_t n, int64_t L, const double *wt) {
    int64_t h = L / 2, ncol = n / L;
    int big = n >= 4096;
    if (ncol >= (int64_t)orc_max_threads()) {
        /* OpenMP over the col' loop (result independent of the thread count) */
#pragma omp parallel for schedule(static) if (big)
        for (int64_t cb = 0; cb < ncol; cb++)
            for (int64_t row = 0; row < h; row++) butterfly(x, cb * L, row, h, wt);
    } else {
        /* few long columns: OpenMP over the row loop instead */
        for (int64_t cb = 0; cb < ncol; cb++) {
#pragma omp parallel for schedule(static) if (big)
            for (int64_t row = 0; row < h; row++) butterfly(x, cb * L, row, h, wt);
        }
    }
}

/* Unnormalised DFT of x (length n = 2^t, t >= 0) in place with kernel
 * e^{sign 2 pi i jk/n}: x <- P_n x (Fig. vanloan_fft line 1), then the
 * q = 1..t stages of Fig. fftpsirad2.  sign = -1 is the forward transform
 * (reading R1); sign = +1 is the fragment's own weight EXP(+2 pi i row/L)
 * read literally, the unnormalised inverse.  Returns -1 if n is not a
 * power of two or sign is not +-1. */
int orc_fft_radix2_sign(double *x, int64_t n, int sign) {
    int t = ilog2_exact(n);
    if (sign != 1 && sign != -1) return -1;
    if (t < 0) return -1;
    if (n == 1) return 0;
    orc_bitrev(x, n);
    double *wt = (double *)malloc(sizeof(double) * (size_t)n); /* L/2 complex <= n/2 */
    if (!wt) return -2;
    for (int q = 1; q <= t; q++) {
        int64_t L = (int64_t)1 << q;
#pragma omp parallel for schedule(static) if (L >= 65536)
        for (int64_t row = 0; row < L / 2; row++) {
            long double re, im;
            omega(row, L, &re, &im); /* e^{-2 pi i row/L} */
            wt[2 * row] = (double)re;
            wt[2 * row + 1] = sign < 0 ? (double)im : -(double)im;
        }
        radix2_stage(x, n, L, wt);
    }
    free(wt);
    return 0;
}

/* The forward transform (the BASELINE.json semantics). */
int orc_fft_radix2(double *x, int64_t n) { return orc_fft_radix2_sign(x, n, -1); }

/* Independent rows (cfg2 "batch contiguous rows"): row b is x[b*n .. b*n+n). */
int orc_fft_radix2_batch_sign(double *x, int64_t n, int64_t batch, int sign) {
    if (ilog2_exact(n) < 0 || batch < 0) return -1;
    for (int64_t b = 0; b < batch; b++) {
        int rc = orc_fft_radix2_sign(x + 2 * b * n, n, sign);
        if (rc) return rc;
    }
    return 0;
}

int orc_fft_radix2_batch(double *x, int64_t n, int64_t batch) { return orc_fft_radix2_batch_sign(x, n, batch, -1); }

/* ---- O3: the definition ---------------------------------------------------- */
/* X[k] = sum_j x[j] T[(j k) mod n], T[e] = e^{-2 pi i e/n}; the exponent is
 * reduced in integers before forming the angle; long double accumulation.
 * Any n >= 1 (the definition does not need a power of two). */
int orc_dft_direct_sign(const double *x, double *X, int64_t n, int sign) {
    if (n < 1 || (sign != 1 && sign != -1)) return -1;
    long double *T = (long double *)malloc(sizeof(long double) * 2 * (size_t)n);
    if (!T) return -2;
    for (int64_t e = 0; e < n; e++) omega(e, n, &T[2 * e], &T[2 * e + 1]);
#pragma omp parallel for schedule(static) if (n >= 256)
    for (int64_t k = 0; k < n; k++) {
        long double sr = 0.0L, si = 0.0L;
        for (int64_t j = 0; j < n; j++) {
            int64_t e = (int64_t)(((unsigned __int128)j * (unsigned __int128)k) % (unsigned __int128)n);
            long double tr = T[2 * e], ti = sign < 0 ? T[2 * e + 1] : -T[2 * e + 1];
            long double xr = x[2 * j], xi = x[2 * j + 1];
            sr += xr * tr - xi * ti;
            si += xr * ti + xi * tr;
        }
        X[2 * k] = (double)sr;
        X[2 * k + 1] = (double)si;
    }
    free(T);
    return 0;
}

/* X[k] = sum_j x[j] e^{-2 pi i jk/n}: the forward definition. */
int orc_dft_direct(const double *x, double *X, int64_t n) { return orc_dft_direct_sign(x, X, n, -1); }

/* w_n^e for 0 <= e < n via e = eh*2^h + el: w^e = w^{eh 2^h} * w^{el}.  Both
 * factors are exact-exponent direct evaluations (long double); this is only a
 * way to avoid an n-entry table at n = 2^30, not a recurrence. */
typedef struct {
    int64_t n;
    int h;
    long double *hi, *lo;
} orc_wtab;

static int wtab_init(orc_wtab *w, int64_t n) {
    int t = ilog2_exact(n);
    w->n = n;
    w->h = (t >= 0) ? (t + 1) / 2 : 0;
    int64_t nlo = (int64_t)1 << w->h;
    int64_t nhi = (n + nlo - 1) / nlo;
    w->hi = (long double *)malloc(sizeof(long double) * 2 * (size_t)nhi);
    w->lo = (long double *)malloc(sizeof(long double) * 2 * (size_t)nlo);
    if (!w->hi || !w->lo) return -2;
    for (int64_t e = 0; e < nhi; e++) omega((e * nlo) % n, n, &w->hi[2 * e], &w->hi[2 * e + 1]);
    for (int64_t e = 0; e < nlo; e++) omega(e % n, n, &w->lo[2 * e], &w->lo[2 * e + 1]);
    return 0;
}
static void wtab_free(orc_wtab *w) {
    free(w->hi);
    free(w->lo);
}
static inline void wtab_get(const orc_wtab *w, int64_t e, long double *re, long double *im) {
    int64_t eh = e >> w->h, el = e & (((int64_t)1 << w->h) - 1);
    long double ar = w->hi[2 * eh], ai = w->hi[2 * eh + 1];
    long double br = w->lo[2 * el], bi = w->lo[2 * el + 1];
    *re = ar * br - ai * bi;
    *im = ar * bi + ai * br;
}

/* Selected bins X[k_i] = sum_j x[b*n + j] w_n^{(j k_i) mod n} of row rows[i]
 * (n a power of two).  x is complex128 (or, if x32 != NULL, complex64 promoted
 * exactly).  Parallel over j with per-thread long double partial sums. */
int orc_dft_bins(const double *x, const float *x32, int64_t n, const int64_t *rows,
                 const int64_t *bins, int64_t nb, double *Xk) {
    if (ilog2_exact(n) < 0) return -1;
    orc_wtab w;
    if (wtab_init(&w, n)) return -2;
    for (int64_t i = 0; i < nb; i++) {
        int64_t k = bins[i], b = rows ? rows[i] : 0;
        long double sr = 0.0L, si = 0.0L;
#pragma omp parallel for schedule(static) reduction(+ : sr, si)
        for (int64_t j = 0; j < n; j++) {
            int64_t e = (int64_t)(((unsigned __int128)j * (unsigned __int128)k) & (unsigned __int128)(n - 1));
            long double tr, ti;
            wtab_get(&w, e, &tr, &ti);
            long double xr, xi;
            if (x32) {
                xr = x32[2 * (b * n + j)];
                xi = x32[2 * (b * n + j) + 1];
            } else {
                xr = x[2 * (b * n + j)];
                xi = x[2 * (b * n + j) + 1];
            }
            sr += xr * tr - xi * ti;
            si += xr * ti + xi * tr;
        }
        Xk[2 * i] = (double)sr;
        Xk[2 * i + 1] = (double)si;
    }
    wtab_free(&w);
    return 0;
}

/* 3-D bins of the separable DFT
 * X[k0,k1,k2] = sum x[j0,j1,j2] w_{n0}^{j0k0} w_{n1}^{j1k1} w_{n2}^{j2k2},
 * x row-major [n0][n1][n2].  bins is nb triples (k0,k1,k2). */
int orc_dft3_bins(const double *x, int64_t n0, int64_t n1, int64_t n2, const int64_t *bins,
                  int64_t nb, double *Xk) {
    if (ilog2_exact(n0) < 0 || ilog2_exact(n1) < 0 || ilog2_exact(n2) < 0) return -1;
    orc_wtab w0, w1, w2;
    if (wtab_init(&w0, n0) || wtab_init(&w1, n1) || wtab_init(&w2, n2)) return -2;
    for (int64_t i = 0; i < nb; i++) {
        int64_t k0 = bins[3 * i], k1 = bins[3 * i + 1], k2 = bins[3 * i + 2];
        long double sr = 0.0L, si = 0.0L;
#pragma omp parallel for schedule(static) reduction(+ : sr, si) collapse(2)
        for (int64_t j0 = 0; j0 < n0; j0++) {
            for (int64_t j1 = 0; j1 < n1; j1++) {
                long double ar, ai, br, bi;
                wtab_get(&w0, (j0 * k0) & (n0 - 1), &ar, &ai);
                wtab_get(&w1, (j1 * k1) & (n1 - 1), &br, &bi);
                long double abr = ar * br - ai * bi, abi = ar * bi + ai * br;
                long double lr = 0.0L, li = 0.0L;
                const double *row = x + 2 * ((j0 * n1 + j1) * n2);
                for (int64_t j2 = 0; j2 < n2; j2++) {
                    long double cr, ci;
                    wtab_get(&w2, (j2 * k2) & (n2 - 1), &cr, &ci);
                    long double xr = row[2 * j2], xi = row[2 * j2 + 1];
                    lr += xr * cr - xi * ci;
                    li += xr * ci + xi * cr;
                }
                sr += lr * abr - li * abi;
                si += lr * abi + li * abr;
            }
        }
        Xk[2 * i] = (double)sr;
        Xk[2 * i + 1] = (double)si;
    }
    wtab_free(&w0);
    wtab_free(&w1);
    wtab_free(&w2);
    return 0;
}

/* ---- O4: the lifted (cache-optimized) FFT of Ch.3 --------------------------- */
/* Reshape-transpose S_{r,c}: y = <r c> rho-hat (transpose (<r c> rho-hat x)),
 * i.e. out[j*r + i] = x[j + c*i] for j < c, i < r (Eq. reshape3 P:2097-2114;
 * loop of Fig. trans_rshp_code with the outer loop over all c columns). */
int orc_reshape_transpose(const double *x, double *out, int64_t n, int64_t c) {
    if (n < 1 || c < 1 || n % c) return -1;
    int64_t r = n / c;
    int64_t index = 0;
    for (int64_t jind = 0; jind < c; jind++)
        for (int64_t iind = 0; iind < r; iind++) {
            out[2 * index] = x[2 * (jind + c * iind)];
            out[2 * index + 1] = x[2 * (jind + c * iind) + 1];
            index++;
        }
    return 0;
}

/* Final transpose F_{n,sigma}: out[t*2^sigma + s] = x[s*2^{d-sigma} + t]
 * (Fig. final_trans_code: t outer, s inner, temp[index++]). */
int orc_final_transpose(const double *x, double *out, int64_t n, int sigma) {
    int d = ilog2_exact(n);
    if (d < 0 || sigma < 0 || sigma > d) return -1;
    int64_t smax = (int64_t)1 << sigma, tmax = (int64_t)1 << (d - sigma);
    int64_t index = 0;
    for (int64_t tind = 0; tind < tmax; tind++)
        for (int64_t sind = 0; sind < smax; sind++) {
            out[2 * index] = x[2 * (sind * tmax + tind)];
            out[2 * index + 1] = x[2 * (sind * tmax + tind) + 1];
            index++;
        }
    return 0;
}

/* Level/stage accounting (reading R6):
 * t = log2 n, logc = log2 c, l_max = floor((t-1)/logc), p_max = t - l_max logc,
 * so n = 2^{p_max} c^{l_max} with 1 <= p_max <= logc.  n = 1 -> identity. */
int orc_lifted_plan(int64_t n, int64_t c, int *l_max, int *p_max) {
    int t = ilog2_exact(n), lc = ilog2_exact(c);
    if (t < 0 || lc < 1) return -1;
    if (t == 0) {
        *l_max = 0;
        *p_max = 0;
        return 0;
    }
    *l_max = (t - 1) / lc;
    *p_max = t - (*l_max) * lc;
    return 0;
}

/* The cache-optimized FFT, step by step (P:2230-2240 recipe):
 *   x <- P_n x
 *   for l = 0..l_max: for p = 1..(l < l_max ? logc : p_max):
 *       v = 2^p, L = v c^l; for each block start b (step v), j < v/2, m = b + j:
 *         sigma = m >> (t - l logc)    (the block type, 0 <= sigma < c^l; reading R7)
 *         (x[m], x[m+v/2]) <- (x[m] + w_L^{sigma + j c^l} x[m+v/2],
 *                              x[m] - w_L^{sigma + j c^l} x[m+v/2])
 *     if l < l_max: x <- S_{n/c, c}(x)
 *   x <- F_{n, l_max logc}(x)                                          */
int orc_fft_lifted(double *x, int64_t n, int64_t c) {
    int l_max, p_max;
    if (orc_lifted_plan(n, c, &l_max, &p_max)) return -1;
    if (n == 1) return 0;
    int t = ilog2_exact(n), lc = ilog2_exact(c);
    double *tmp = (double *)malloc(sizeof(double) * 2 * (size_t)n);
    if (!tmp) return -2;
    orc_bitrev(x, n);
    for (int l = 0; l <= l_max; l++) {
        int pend = (l < l_max) ? lc : p_max;
        int64_t cl = (int64_t)1 << (l * lc); /* c^l */
        for (int p = 1; p <= pend; p++) {
            int64_t v = (int64_t)1 << p, h = v / 2, L = v * cl;
#pragma omp parallel for schedule(static) if (n >= 65536)
            for (int64_t b = 0; b < n; b += v) {
                for (int64_t j = 0; j < h; j++) {
                    int64_t m = b + j;
                    int64_t sigma = m >> (t - l * lc);
                    long double wr, wi;
                    omega(sigma + j * cl, L, &wr, &wi);
                    double *pa = x + 2 * m, *pd = x + 2 * (m + h);
                    double cr = (double)wr * pd[0] - (double)wi * pd[1];
                    double ci = (double)wr * pd[1] + (double)wi * pd[0];
                    double ar = pa[0], ai = pa[1];
                    pa[0] = ar + cr;
                    pa[1] = ai + ci;
                    pd[0] = ar - cr;
                    pd[1] = ai - ci;
                }
            }
        }
        if (l < l_max) {
            orc_reshape_transpose(x, tmp, n, c);
            memcpy(x, tmp, sizeof(double) * 2 * (size_t)n);
        }
    }
    orc_final_transpose(x, tmp, n, l_max * lc);
    memcpy(x, tmp, sizeof(double) * 2 * (size_t)n);
    free(tmp);
    return 0;
}

/* ---- O5: 3-D ------------------------------------------------------------------ */
/* Row-major [n0][n1][n2]; 1-D FFTs along axis 2 (contiguous lines), then axis 1,
 * then axis 0.  Each line is gathered, transformed by orc_fft_radix2, scattered. */
int orc_fft3d_sign(double *x, int64_t n0, int64_t n1, int64_t n2, int sign) {
    if (ilog2_exact(n0) < 0 || ilog2_exact(n1) < 0 || ilog2_exact(n2) < 0) return -1;
    if (sign != 1 && sign != -1) return -1;
    int64_t dims[3] = {n0, n1, n2};
    int64_t strides[3] = {n1 * n2, n2, 1};
    for (int ax = 2; ax >= 0; ax--) {
        int64_t len = dims[ax], st = strides[ax];
        int64_t nlines = (n0 * n1 * n2) / len;
        int fail = 0;
#pragma omp parallel
        {
            double *line = (double *)malloc(sizeof(double) * 2 * (size_t)len);
            if (!line) fail = 1;
#pragma omp for schedule(static)
            for (int64_t li = 0; li < nlines; li++) {
                if (!line) continue;
                /* line index -> base offset: enumerate the other two axes row-major */
                int64_t base;
                if (ax == 2) base = li * n2;
                else if (ax == 1) base = (li / n2) * (n1 * n2) + (li % n2);
                else base = li;
                for (int64_t j = 0; j < len; j++) {
                    line[2 * j] = x[2 * (base + j * st)];
                    line[2 * j + 1] = x[2 * (base + j * st) + 1];
                }
                orc_fft_radix2_sign(line, len, sign);
                for (int64_t j = 0; j < len; j++) {
                    x[2 * (base + j * st)] = line[2 * j];
                    x[2 * (base + j * st) + 1] = line[2 * j + 1];
                }
            }
            free(line);
        }
        if (fail) return -2;
    }
    return 0;
}

int orc_fft3d(double *x, int64_t n0, int64_t n1, int64_t n2) { return orc_fft3d_sign(x, n0, n1, n2, -1); }

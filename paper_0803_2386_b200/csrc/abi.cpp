// abi.cpp -- the C-ABI (include/moa_fft.h): validation, plans, twiddle tables,
// execution.  Every compute step runs in kernels.cu; this file only plans,
// allocates and launches.
#include <cuda_runtime.h>
#include <math.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "comm.h"
#include "moa_internal.h"

namespace moa {

static thread_local std::string g_err;

moa_status_t fail(moa_status_t st, const std::string &msg) {
    g_err = msg;
    return st;
}

static moa_status_t cuda_fail(cudaError_t e, const char *what) {
    return fail(MOA_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Tracing: with MOA_FFT_NVTX=1 every exec and every pass is an
// NVTX range ("moa exec", "pass p R=.."), visible to Nsight Systems / ncu
// --nvtx filters; a no-op otherwise.
static bool nvtx_on() {
    static const bool on = [] {
        const char *e = std::getenv("MOA_FFT_NVTX");
        return e && e[0] == '1';
    }();
    return on;
}
struct NvtxRange {
    bool on;
    explicit NvtxRange(const std::string &name) : on(nvtx_on()) {
        if (on) nvtxRangePushA(name.c_str());
    }
    ~NvtxRange() {
        if (on) nvtxRangePop();
    }
};

PassMods pass_mods(uint32_t flags, size_t i, size_t npass, int64_t N) {
    PassMods m;
    const bool inv = flags & MOA_FFT_INVERSE;
    m.conj_in = inv && i == 0;
    m.conj_out = inv && i + 1 == npass;
    if ((flags & MOA_FFT_NORMALIZE) && i + 1 == npass) m.scale = 1.0 / double(N);
    return m;
}

}  // namespace moa

using namespace moa;

struct moa_fft_plan_s {
    int device = -1;
    moa_dtype_t dtype = MOA_C128;
    int ngpu = 1;
    int rank = 0;
    bool is3d = false;
    int64_t n = 0, batch = 1, n0 = 0, n1 = 0, n2 = 0;
    int64_t local_elems = 0;
    size_t esize = 16;
    uint32_t flags = 0;              // MOA_FFT_INVERSE / _NORMALIZE / _LIFTED_ORDER
    bool inplace_safe = true;        // in == out works without a staging copy (see finish_plan)
    void *inplace_buf = nullptr;     // the input copy of an in-place exec of an unsafe plan (lazy)
    bool lifted_out = false;         // one GPU: the last pass stores in place (no final transpose)
    moa_pass_desc_t natural_last{};  // ... and this is the natural-order descriptor it replaced
    std::vector<moa_pass_desc_t> passes;
    std::vector<DevTables> tabs;
    std::vector<void *> allocs;
    void *scratch = nullptr;
    void *staging = nullptr;
    DistPlan *dist = nullptr;  // processor-level lifting (comm.cpp)
    std::vector<RingState> rings;  // rings[i] valid where passes[i].ring == 2
    moa_fft_plan_s *sub[2] = {nullptr, nullptr};  // exec_host chunk pipeline (rows / 8 each)
    cudaStream_t ss[2] = {nullptr, nullptr};
    // per-step event profiling (moa_fft_prof_begin / _end)
    std::vector<cudaEvent_t> prof_ev;
    int prof_max = 0, prof_count = 0, prof_nsteps = 0;
};


namespace {

bool pow2(int64_t v) { return v >= 1 && (v & (v - 1)) == 0; }

moa_status_t dev_alloc(moa_fft_plan_s *p, size_t bytes, void **out) {
    *out = nullptr;
    if (bytes == 0) return MOA_OK;
    cudaError_t e = cudaMalloc(out, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(MOA_ENOMEM, std::string("cudaMalloc(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
    }
    p->allocs.push_back(*out);
    return MOA_OK;
}

// w_N^e = e^{-2 pi i e / N} for exact integer e (forward sign), long double.
void omega_ld(int64_t e, int64_t N, long double &re, long double &im) {
    const long double two_pi = 6.283185307179586476925286766559005768L;
    const long double a = two_pi * ((long double)e / (long double)N);
    re = cosl(a);
    im = -sinl(a);
}

moa_status_t upload_table(moa_fft_plan_s *p, const std::vector<long double> &v, const void **dptr, bool dbl = false) {
    const size_t cnt = v.size();
    void *d = nullptr;
    moa_status_t st = dev_alloc(p, cnt * ((dbl || p->dtype == MOA_C128) ? sizeof(double) : sizeof(float)), &d);
    if (st) return st;
    cudaError_t e;
    if (dbl || p->dtype == MOA_C128) {
        std::vector<double> h(cnt);
        for (size_t i = 0; i < cnt; i++) h[i] = (double)v[i];
        e = cudaMemcpy(d, h.data(), cnt * sizeof(double), cudaMemcpyHostToDevice);
    } else {
        std::vector<float> h(cnt);
        for (size_t i = 0; i < cnt; i++) h[i] = (float)v[i];
        e = cudaMemcpy(d, h.data(), cnt * sizeof(float), cudaMemcpyHostToDevice);
    }
    if (e != cudaSuccess) return cuda_fail(e, "twiddle upload");
    *dptr = d;
    return MOA_OK;
}

// Plan-time twiddle tables (step a5): per pass the in-line table w_R^e (e < R)
// and, for a lifted level, the two-level table of w_N (hi: w_N^{eh 2^h},
// lo: w_N^{el}, h = ceil(log2 N / 2)).
moa_status_t build_tables(moa_fft_plan_s *p) {
    std::map<int, const void *> byR;
    std::map<int64_t, std::pair<const void *, const void *>> byN;
    p->tabs.clear();
    // one tile counter per pass for the warp-specialised kernel (reset on the
    // exec stream before each of its launches)
    void *ctrs = nullptr;
    {
        moa_status_t st = dev_alloc(p, sizeof(unsigned long long) * (p->passes.size() + 1), &ctrs);
        if (st) return st;
    }
    for (auto &d : p->passes) {
        DevTables t;
        auto it = byR.find(d.logR);
        if (it != byR.end()) {
            t.twR = it->second;
        } else {
            // step twiddles of the in-register Stockham schedule of kernels.cu
            // (steps of radix 16, the last takes the remainder): step s with
            // NS = 16^s points already combined and radix Q stores
            // w_{NS Q}^{jm r} (1 <= r < Q, jm < NS) at entry r NS + jm - 1; the
            // steps tile [0, R - 1) exactly (sum_s (Q_s - 1) NS_s = R - 1)
            const int64_t R = int64_t(1) << d.logR;
            const int LP = psi_log_p(d.logR, p->dtype);
            const int nstep = d.logR == 0 ? 1 : (d.logR + LP - 1) / LP;
            std::vector<long double> v(2 * (R > 1 ? R - 1 : 1), 0.0L);
            for (int st = 1; st < nstep; st++) {
                const int64_t NS = int64_t(1) << (LP * st);
                const int lq = st == nstep - 1 ? d.logR - LP * (nstep - 1) : LP;
                const int64_t Q = int64_t(1) << lq;
                for (int64_t r = 1; r < Q; r++)
                    for (int64_t jm = 0; jm < NS; jm++) {
                        const int64_t idx = r * NS + jm - 1;
                        omega_ld((jm * r) % (NS * Q), NS * Q, v[2 * idx], v[2 * idx + 1]);
                    }
            }
            moa_status_t st = upload_table(p, v, &t.twR);
            if (st) return st;
            byR[d.logR] = t.twR;
        }
        if (p->passes.size() == 1 && d.kind == 0 && d.twN <= 1 && d.logR >= 6 && d.logR <= 12) {
            // the small-transform kernel's table (kernels.cu small_fft_kernel):
            // radix-4 step s >= 1 with NS = 4^s stores w_{4 NS}^{k q} (k < NS,
            // 1 <= q < 4) at entry (NS - 4) + (q - 1) NS + k; an odd log2 R adds
            // the final radix-2 step's w_R^j (j < R/2) at (R/2 - 4) + j
            const int64_t R = int64_t(1) << d.logR;
            std::vector<long double> v(2 * (R - 4), 0.0L);
            for (int64_t NS = 4; 4 * NS <= R; NS *= 4)
                for (int64_t q = 1; q < 4; q++)
                    for (int64_t k = 0; k < NS; k++) {
                        const int64_t idx = (NS - 4) + (q - 1) * NS + k;
                        omega_ld(k * q, 4 * NS, v[2 * idx], v[2 * idx + 1]);
                    }
            if (d.logR & 1)
                for (int64_t j = 0; j < R / 2; j++) {
                    const int64_t idx = (R / 2 - 4) + j;
                    omega_ld(j, R, v[2 * idx], v[2 * idx + 1]);
                }
            moa_status_t st = upload_table(p, v, &t.twS);
            if (st) return st;
        }
        if (d.twN > 1) {
            auto jt = byN.find(d.twN);
            if (jt != byN.end()) {
                t.tw_hi = jt->second.first;
                t.tw_lo = jt->second.second;
            } else {
                const int lN = log2_exact(d.twN);
                const int h = (lN + 1) / 2;
                const int64_t nlo = int64_t(1) << h, nhi = d.twN >> h;
                std::vector<long double> lo(2 * nlo), hi(2 * nhi);
                for (int64_t e = 0; e < nlo; e++) omega_ld(e, d.twN, lo[2 * e], lo[2 * e + 1]);
                for (int64_t e = 0; e < nhi; e++) omega_ld(e << h, d.twN, hi[2 * e], hi[2 * e + 1]);
                moa_status_t st = upload_table(p, hi, &t.tw_hi, true);
                if (st) return st;
                st = upload_table(p, lo, &t.tw_lo, true);
                if (st) return st;
                byN[d.twN] = {t.tw_hi, t.tw_lo};
            }
        }
        t.ctr = static_cast<unsigned long long *>(ctrs) + p->tabs.size();
        p->tabs.push_back(t);
    }
    return MOA_OK;
}

moa_status_t parse_lift_env(int64_t n, std::vector<int64_t> &rad, bool &have) {
    have = false;
    const char *s = std::getenv("MOA_FFT_LIFT");
    if (!s || !*s) return MOA_OK;
    rad.clear();
    const char *c = s;
    while (*c) {
        char *end = nullptr;
        long long v = std::strtoll(c, &end, 10);
        if (end == c) return fail(MOA_EINVAL, "MOA_FFT_LIFT: expected comma-separated radices");
        rad.push_back(v);
        c = end;
        if (*c == ',') c++;
    }
    int64_t prod = 1;
    for (auto r : rad) prod *= r;
    if (prod != n) return MOA_OK;  // the override applies only to the size it names
    have = true;
    return MOA_OK;
}

moa_status_t finish_plan(moa_fft_plan_s *p) {
    cudaError_t e = cudaGetDevice(&p->device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    for (auto &d : p->passes) {
        int mt = 0, regs = 0;
        e = kernel_attributes(p->dtype, d.logR, &mt, &regs);
        if (e != cudaSuccess) return cuda_fail(e, "kernel attributes (is the GPU an sm_100 part?)");
        if (d.threads > mt) return fail(MOA_EUNSUPPORTED, "pass tile exceeds the kernel's thread limit");
    }
    // in == out: safe unless a pass reads `in` and writes `out` at other
    // positions than it read (a transposing store, the bit reversal) -- then
    // exec stages the input through a plan-owned copy first
    for (auto &d : p->passes) {
        if (d.src != 0 || d.dst != 1) continue;
        bool same = d.kind <= 1 && d.in_kstr == d.out_kstr && d.out_ksplit >= d.logR && !d.ring;
        for (int i = 0; i < d.ndig && same; i++) same = d.in_str[i] == d.out_str[i];
        if (!same) p->inplace_safe = false;
    }
    bool need_scratch = false;
    for (auto &d : p->passes) need_scratch |= (d.src == 2 || d.dst == 2);
    if (need_scratch) {
        moa_status_t st = dev_alloc(p, size_t(p->local_elems) * p->esize, &p->scratch);
        if (st) return st;
    }
    p->rings.assign(p->passes.size(), RingState{});
    for (size_t i = 0; i < p->passes.size(); i++) {
        const moa_pass_desc_t &d = p->passes[i];
        if (d.ring != 2) continue;
        if (i + 1 >= p->passes.size() || p->passes[i + 1].ring != 1) return fail(MOA_EINVAL, "plan: unpaired ring pass");
        RingState &r = p->rings[i];
        void *ctr = nullptr;
        moa_status_t st = dev_alloc(p, size_t(d.ring_slots) * d.ring_G * p->esize, &r.ring);
        if (!st) st = dev_alloc(p, sizeof(unsigned long long) * (2 * size_t(d.ring_groups) + 1), &ctr);
        if (st) return st;
        e = cudaMemset(ctr, 0, sizeof(unsigned long long) * (2 * size_t(d.ring_groups) + 1));
        if (e != cudaSuccess) return cuda_fail(e, "ring counters");
        r.qctr = static_cast<unsigned long long *>(ctr);
        r.cntA = r.qctr + 1;
        r.cntB = r.cntA + d.ring_groups;
        const char *se = std::getenv("MOA_FFT_STATS");
        if (se && se[0] == '1') {
            void *sp = nullptr;
            st = dev_alloc(p, 6 * sizeof(unsigned long long), &sp);
            if (st) return st;
            cudaMemset(sp, 0, 6 * sizeof(unsigned long long));
            r.stats = static_cast<unsigned long long *>(sp);
        }
    }
    return build_tables(p);
}

constexpr uint32_t kAllFlags =
    MOA_FFT_INVERSE | MOA_FFT_NORMALIZE | MOA_FFT_LIFTED_ORDER | MOA_FFT_UNBLOCKED | MOA_FFT_HYPERCUBE;

// MOA_FFT_UNBLOCKED: P_n (kind 3, in -> out), then t global radix-2 stages in
// place on out (kind 2, half-distance h = 2^(q-1) in in_kstr, weights w_n^e).
// ext[0] carries the element count of all rows.
void unblocked_passes(int64_t n, int64_t batch, std::vector<moa_pass_desc_t> &out) {
    out.clear();
    const int t = log2_exact(n);
    moa_pass_desc_t d;
    std::memset(&d, 0, sizeof(d));
    d.kind = 3;
    d.ndig = 1;
    d.ext[0] = n * batch;
    d.twN = n;
    d.out_ksplit = 62;
    d.src = 0;
    d.dst = 1;
    out.push_back(d);
    for (int q = 1; q <= t; q++) {
        d.kind = 2;
        d.logR = 1;
        d.in_kstr = d.out_kstr = int64_t(1) << (q - 1);
        d.src = d.dst = 1;
        out.push_back(d);
    }
}

// MOA_FFT_HYPERCUBE: t stages of kind 4 (stage s in in_kstr = 2^s, ext[0] =
// rows * n, weights w_n^e), ping-ponging so the last one writes out (1): stage
// s reads buffer src and writes dst, with dst = out when t - 1 - s is even.
void hypercube_passes(int64_t n, int64_t batch, std::vector<moa_pass_desc_t> &out) {
    out.clear();
    const int t = log2_exact(n);
    moa_pass_desc_t d;
    std::memset(&d, 0, sizeof(d));
    d.kind = 4;
    d.logR = 1;
    d.ndig = 1;
    d.ext[0] = n * batch;
    d.twN = n;
    d.out_ksplit = 62;
    int src = 0;
    for (int s = 0; s < t; s++) {
        d.in_kstr = d.out_kstr = int64_t(1) << s;
        d.src = src;
        d.dst = ((t - 1 - s) % 2 == 0) ? 1 : 2;
        out.push_back(d);
        src = d.dst;
    }
}

// MOA_FFT_LIFTED_ORDER on one GPU: the last pass stores each result where it
// loaded its input (point-contiguous, in place) instead of through the final
// transpose; the natural descriptor is kept for moa_fft_output_index.
void make_lifted_order(moa_fft_plan_s *p) {
    if (p->passes.size() < 2) return;  // a single pass is already in natural order
    psi_uncluster(p->passes);          // the last pass is rewritten below
    moa_pass_desc_t &d = p->passes.back();
    if (d.ring) return;                // fused L2 pairs keep natural order
    p->natural_last = d;
    for (int i = 0; i < d.ndig; i++) d.out_str[i] = d.in_str[i];
    d.out_kstr = d.in_kstr;
    d.out_ksplit = 62;
    d.lf_store = d.lf_load;
    psi_choose_tile(d, p->dtype);
    p->lifted_out = true;
}

moa_status_t plan_1d(moa_fft_plan_t *plan, int64_t n, int64_t batch, moa_dtype_t dtype, int ngpu,
                     const int64_t *radices, int nrad, uint32_t flags = 0) {
    if (!plan) return fail(MOA_EINVAL, "plan: null output pointer");
    *plan = nullptr;
    if (flags & ~kAllFlags) return fail(MOA_EINVAL, "plan: unknown flag bits");
    if ((flags & MOA_FFT_UNBLOCKED) && (ngpu > 1 || (flags & MOA_FFT_LIFTED_ORDER) || radices))
        return fail(MOA_EUNSUPPORTED, "plan: MOA_FFT_UNBLOCKED is one-GPU, natural order, planner-chosen only");
    if ((flags & MOA_FFT_HYPERCUBE) &&
        (ngpu > 1 || (flags & (MOA_FFT_LIFTED_ORDER | MOA_FFT_UNBLOCKED)) || radices))
        return fail(MOA_EUNSUPPORTED, "plan: MOA_FFT_HYPERCUBE is one-GPU, natural order, planner-chosen only");
    if (!pow2(n)) return fail(MOA_EINVAL, "plan: n must be a power of two >= 1 (n = 2^t, t >= 0)");
    if (batch < 1) return fail(MOA_EINVAL, "plan: batch must be >= 1");
    if (dtype != MOA_C64 && dtype != MOA_C128) return fail(MOA_EINVAL, "plan: unknown dtype");
    if (!(ngpu == 1 || ngpu == 2 || ngpu == 4 || ngpu == 8)) return fail(MOA_EINVAL, "plan: ngpu must be 1, 2, 4 or 8");
    if (n > (int64_t(1) << 36) || batch > (int64_t(1) << 36) / n)
        return fail(MOA_EINVAL, "plan: n * batch exceeds 2^36 elements");
    if (ngpu > 1) {
        if (batch != 1) return fail(MOA_EUNSUPPORTED, "plan: ngpu > 1 requires batch == 1");
        if (n < int64_t(ngpu) * ngpu) return fail(MOA_EUNSUPPORTED, "plan: ngpu > 1 requires n >= ngpu^2");
        if (!dist_ready(ngpu)) return fail(MOA_EINVAL, "plan: call moa_fft_dist_init(rank, ngpu, id) first");
    }
    auto *p = new moa_fft_plan_s;
    p->dtype = dtype;
    p->n = n;
    p->batch = batch;
    p->ngpu = ngpu;
    p->esize = dtype == MOA_C128 ? 16 : 8;
    p->local_elems = n * batch / ngpu;
    p->flags = flags;
    moa_status_t st = MOA_OK;
    if (ngpu > 1) {
        st = dist_plan_1d(p->dist, n, dtype, (flags & MOA_FFT_LIFTED_ORDER) != 0);
        if (!st) {
            p->passes = p->dist->passes;
            p->rank = p->dist->rank;
        }
    } else {
        std::vector<int64_t> rad;
        if ((flags & MOA_FFT_UNBLOCKED) || ((flags & MOA_FFT_HYPERCUBE) && n == 1)) {
            unblocked_passes(n, batch, p->passes);  // (n = 1: the identity copy)
        } else if (flags & MOA_FFT_HYPERCUBE) {
            hypercube_passes(n, batch, p->passes);
        } else if (radices) {
            rad.assign(radices, radices + nrad);
        } else {
            bool have = false;
            st = parse_lift_env(n, rad, have);
            if (!st && !have) st = plan_radices(n, batch, dtype, rad);
        }
        if (!st && !(flags & (MOA_FFT_UNBLOCKED | MOA_FFT_HYPERCUBE)))
            st = psi_build(n, batch, dtype, rad, radices == nullptr, p->passes);
        if (!st && (flags & MOA_FFT_LIFTED_ORDER)) make_lifted_order(p);
    }
    if (!st) st = finish_plan(p);
    if (!st && p->dist) {
        st = dist_finish(p->dist, p->scratch);
        if (!st) p->passes = p->dist->passes;
    }
    if (st) {
        std::string msg = moa_fft_last_error();
        moa_fft_destroy(p);
        return fail(st, msg);
    }
    *plan = p;
    return MOA_OK;
}

}  // namespace

extern "C" {

const char *moa_fft_last_error(void) { return g_err.c_str(); }

moa_status_t moa_fft_plan(moa_fft_plan_t *plan, int64_t n, int64_t batch, moa_dtype_t dtype, int ngpu) {
    return plan_1d(plan, n, batch, dtype, ngpu, nullptr, 0);
}

moa_status_t moa_fft_plan_lift(moa_fft_plan_t *plan, int64_t n, int64_t batch, moa_dtype_t dtype,
                               const int64_t *radices, int nrad) {
    if (!radices || nrad < 1) return fail(MOA_EINVAL, "plan_lift: radices must be non-null with nrad >= 1");
    return plan_1d(plan, n, batch, dtype, 1, radices, nrad);
}

moa_status_t moa_fft_plan_ex(moa_fft_plan_t *plan, int64_t n, int64_t batch, moa_dtype_t dtype, int ngpu,
                             uint32_t flags) {
    return plan_1d(plan, n, batch, dtype, ngpu, nullptr, 0, flags);
}

moa_status_t moa_fft_plan_3d(moa_fft_plan_t *plan, int64_t n0, int64_t n1, int64_t n2, moa_dtype_t dtype, int ngpu) {
    return moa_fft_plan_3d_ex(plan, n0, n1, n2, dtype, ngpu, 0);
}

moa_status_t moa_fft_plan_3d_ex(moa_fft_plan_t *plan, int64_t n0, int64_t n1, int64_t n2, moa_dtype_t dtype, int ngpu,
                                uint32_t flags) {
    if (!plan) return fail(MOA_EINVAL, "plan_3d: null output pointer");
    *plan = nullptr;
    if (flags & ~kAllFlags) return fail(MOA_EINVAL, "plan_3d: unknown flag bits");
    if (flags & (MOA_FFT_LIFTED_ORDER | MOA_FFT_UNBLOCKED | MOA_FFT_HYPERCUBE))
        return fail(MOA_EUNSUPPORTED, "plan_3d: MOA_FFT_LIFTED_ORDER / _UNBLOCKED / _HYPERCUBE are 1-D only");
    for (int64_t v : {n0, n1, n2})
        if (!pow2(v) || v > 4096) return fail(MOA_EINVAL, "plan_3d: each extent must be a power of two in [1, 4096]");
    if (dtype != MOA_C64 && dtype != MOA_C128) return fail(MOA_EINVAL, "plan_3d: unknown dtype");
    if (!(ngpu == 1 || ngpu == 2 || ngpu == 4 || ngpu == 8)) return fail(MOA_EINVAL, "plan_3d: ngpu must be 1, 2, 4 or 8");
    if (n0 * n1 * n2 > (int64_t(1) << 36)) return fail(MOA_EINVAL, "plan_3d: volume exceeds 2^36 elements");
    if (ngpu > 1) {
        if (n0 % ngpu || n1 % ngpu) return fail(MOA_EUNSUPPORTED, "plan_3d: ngpu must divide n0 and n1");
        if (!dist_ready(ngpu)) return fail(MOA_EINVAL, "plan_3d: call moa_fft_dist_init(rank, ngpu, id) first");
    }
    auto *p = new moa_fft_plan_s;
    p->dtype = dtype;
    p->is3d = true;
    p->n0 = n0;
    p->n1 = n1;
    p->n2 = n2;
    p->n = n0 * n1 * n2;
    p->ngpu = ngpu;
    p->esize = dtype == MOA_C128 ? 16 : 8;
    p->local_elems = p->n / ngpu;
    p->flags = flags;
    moa_status_t st;
    if (ngpu > 1) {
        st = dist_plan_3d(p->dist, n0, n1, n2, dtype);
        if (!st) {
            p->passes = p->dist->passes;
            p->rank = p->dist->rank;
        }
    } else {
        st = psi_3d_passes(n0, n1, n2, 1, dtype, p->passes);
        if (!st) psi_fuse_3d(p->passes, dtype);
    }
    if (!st) st = finish_plan(p);
    if (!st && p->dist) {
        st = dist_finish(p->dist, p->scratch);
        if (!st) p->passes = p->dist->passes;
    }
    if (st) {
        std::string msg = moa_fft_last_error();
        moa_fft_destroy(p);
        return fail(st, msg);
    }
    *plan = p;
    return MOA_OK;
}

moa_status_t moa_fft_exec(moa_fft_plan_t p, const void *in, void *out, void *stream) {
    if (!p) return fail(MOA_EINVAL, "exec: null plan");
    if (!in || !out) return fail(MOA_EINVAL, "exec: null buffer");
    if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15)
        return fail(MOA_EINVAL, "exec: buffers must be 16-byte aligned");
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (dev != p->device) return fail(MOA_EINVAL, "exec: the current device is not the plan's device");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (in == out && !p->inplace_safe) {  // stage the input (one device copy) so no pass reads what it overwrites
        const size_t bytes = size_t(p->local_elems) * p->esize;
        if (!p->inplace_buf) {
            moa_status_t st = dev_alloc(p, bytes, &p->inplace_buf);
            if (st) return st;
        }
        e = cudaMemcpyAsync(p->inplace_buf, in, bytes, cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return cuda_fail(e, "exec: in-place staging copy");
        in = p->inplace_buf;
    }
    cudaEvent_t *evs = nullptr;
    if (p->prof_count < p->prof_max) evs = &p->prof_ev[size_t(p->prof_count) * (p->prof_nsteps + 1)];
    moa_status_t st = MOA_OK;
    const size_t np = p->passes.size();
    NvtxRange exec_range(nvtx_on() ? "moa exec n=" + std::to_string(p->n) : std::string());
    if (p->dist) {
        std::vector<DistRank> me{{p->dist, &p->passes, &p->tabs,
                                  {const_cast<void *>(in), out, p->scratch, p->dist->scratch2}, p->flags}};
        if (p->dist->loopback) return fail(MOA_EINVAL, "exec: a loopback plan runs through moa_fft_exec_loopback");
        st = dist_exec(me, DistBackend::Nccl, p->dtype, s, evs, p->n);
    } else {
        int step = 0;
        for (size_t i = 0; i < np; i++, step++) {
            const moa_pass_desc_t &d = p->passes[i];
            const void *src = d.src == 0 ? in : d.src == 1 ? static_cast<const void *>(out) : p->scratch;
            NvtxRange pass_range(nvtx_on() ? "pass " + std::to_string(i) + " R=" + std::to_string(1 << d.logR)
                                           : std::string());
            if (evs) cudaEventRecord(evs[step], s);
            if (d.ring == 3) {  // cluster pair: passes i and i+1 in one launch, intermediate in the clusters' smem
                const moa_pass_desc_t &dB = p->passes[i + 1];
                void *dst = dB.dst == 1 ? out : p->scratch;
                e = launch_cluster(d, dB, p->dtype, src, dst, p->tabs[i], p->tabs[i + 1], s,
                                   pass_mods(p->flags, i, np, p->n), pass_mods(p->flags, i + 1, np, p->n));
                if (e != cudaSuccess) return cuda_fail(e, "cluster-pair kernel launch");
                i++;
            } else if (d.ring == 2) {  // fused pair: passes i and i+1 in one launch, intermediate in the L2 ring
                const moa_pass_desc_t &dB = p->passes[i + 1];
                void *dst = dB.dst == 1 ? out : p->scratch;
                RingState &r = p->rings[i];
                e = launch_pair(d, dB, p->dtype, src, dst, r, p->tabs[i], p->tabs[i + 1], s,
                                pass_mods(p->flags, i, np, p->n), pass_mods(p->flags, i + 1, np, p->n));
                if (e != cudaSuccess) return cuda_fail(e, "pass-pair kernel launch");
                r.epoch++;
                i++;
            } else {
                void *dst = d.dst == 1 ? out : p->scratch;
                e = launch_pass(d, p->dtype, src, dst, p->tabs[i], s, pass_mods(p->flags, i, np, p->n));
                if (e != cudaSuccess) return cuda_fail(e, "pass kernel launch");
            }
        }
        if (evs) cudaEventRecord(evs[step], s);
    }
    if (evs) p->prof_count++;
    return st;
}

moa_status_t moa_fft_exec_host(moa_fft_plan_t p, const void *host_in, void *host_out, void *stream) {
    if (!p) return fail(MOA_EINVAL, "exec_host: null plan");
    if (!host_in || !host_out) return fail(MOA_EINVAL, "exec_host: null buffer");
    const size_t bytes = size_t(p->local_elems) * p->esize;
    if (!p->staging) {
        moa_status_t st = dev_alloc(p, bytes, &p->staging);
        if (st) return st;
    }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    cudaError_t e;
    // Independent rows: pipeline chunks of rows over two streams so the
    // host->device copy of chunk c+1, the FFT of chunk c and the device->host
    // copy of chunk c-1 overlap (PCIe is full duplex).  Each stream has its own
    // sub-plan (plans are not re-entrant) and its own half of the staging buffer.
    const int64_t nch = (!p->dist && !p->is3d && p->batch >= 8) ? 8 : 1;
    if (nch > 1 && p->batch % nch == 0) {
        const int64_t rows = p->batch / nch;
        const size_t cb = size_t(rows * p->n) * p->esize;
        if (!p->sub[0]) {
            for (int k = 0; k < 2; k++) {
                moa_status_t st = moa_fft_plan_ex(&p->sub[k], p->n, rows, p->dtype, 1, p->flags);
                if (st) return st;
                e = cudaStreamCreateWithFlags(&p->ss[k], cudaStreamNonBlocking);
                if (e != cudaSuccess) return cuda_fail(e, "exec_host stream");
            }
        }
        e = cudaStreamSynchronize(s);  // the caller's prior work on its stream is done
        if (e != cudaSuccess) return cuda_fail(e, "exec_host sync");
        for (int64_t c = 0; c < nch; c++) {
            const int k = int(c & 1);
            char *stg = static_cast<char *>(p->staging) + size_t(k) * cb;  // two chunk buffers
            e = cudaMemcpyAsync(stg, static_cast<const char *>(host_in) + size_t(c) * cb, cb, cudaMemcpyHostToDevice,
                                p->ss[k]);
            if (e != cudaSuccess) return cuda_fail(e, "exec_host H2D");
            moa_status_t st = moa_fft_exec(p->sub[k], stg, stg, p->ss[k]);
            if (st) return st;
            e = cudaMemcpyAsync(static_cast<char *>(host_out) + size_t(c) * cb, stg, cb, cudaMemcpyDeviceToHost,
                                p->ss[k]);
            if (e != cudaSuccess) return cuda_fail(e, "exec_host D2H");
        }
        for (int k = 0; k < 2; k++) {
            e = cudaStreamSynchronize(p->ss[k]);
            if (e != cudaSuccess) return cuda_fail(e, "exec_host sync");
        }
        return MOA_OK;
    }
    e = cudaMemcpyAsync(p->staging, host_in, bytes, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "exec_host H2D");
    moa_status_t st = moa_fft_exec(p, p->staging, p->staging, stream);
    if (st) return st;
    e = cudaMemcpyAsync(host_out, p->staging, bytes, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return cuda_fail(e, "exec_host D2H");
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "exec_host sync");
    return MOA_OK;
}

static int local_launches(moa_fft_plan_t p) {
    int c = 0;
    for (auto &d : p->passes) c += d.ring != 1 && d.ring != 4;  // a fused / cluster pair is one launch
    return c;
}

static int plan_nsteps(moa_fft_plan_t p) { return p->dist ? int(p->dist->steps.size()) : local_launches(p); }

static void prof_free(moa_fft_plan_t p) {
    for (auto ev : p->prof_ev) cudaEventDestroy(ev);
    p->prof_ev.clear();
    p->prof_max = p->prof_count = 0;
}

moa_status_t moa_fft_prof_begin(moa_fft_plan_t p, int max_execs) {
    if (!p || max_execs < 1 || max_execs > 100000) return fail(MOA_EINVAL, "prof_begin: bad arguments");
    prof_free(p);
    p->prof_nsteps = plan_nsteps(p);
    const size_t cnt = size_t(max_execs) * (p->prof_nsteps + 1);
    p->prof_ev.resize(cnt);
    for (size_t i = 0; i < cnt; i++) {
        cudaError_t e = cudaEventCreate(&p->prof_ev[i]);
        if (e != cudaSuccess) {
            p->prof_ev.resize(i);
            prof_free(p);
            return cuda_fail(e, "prof_begin: cudaEventCreate");
        }
    }
    p->prof_max = max_execs;
    p->prof_count = 0;
    return MOA_OK;
}

moa_status_t moa_fft_prof_end(moa_fft_plan_t p, double *step_ms, int max_steps, int *nsteps, int *execs) {
    if (!p || !step_ms || !nsteps || !execs) return fail(MOA_EINVAL, "prof_end: null argument");
    const int ns = p->prof_nsteps;
    if (ns > max_steps) return fail(MOA_EINVAL, "prof_end: step_ms too small");
    for (int i = 0; i < ns; i++) step_ms[i] = 0.0;
    for (int x = 0; x < p->prof_count; x++) {
        cudaEvent_t *ev = &p->prof_ev[size_t(x) * (ns + 1)];
        cudaError_t e = cudaEventSynchronize(ev[ns]);
        if (e != cudaSuccess) return cuda_fail(e, "prof_end: sync");
        for (int i = 0; i < ns; i++) {
            float ms = 0.f;
            e = cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
            if (e != cudaSuccess) return cuda_fail(e, "prof_end: elapsed");
            step_ms[i] += ms;
        }
    }
    *nsteps = ns;
    *execs = p->prof_count;
    prof_free(p);
    return MOA_OK;
}

moa_status_t moa_fft_destroy(moa_fft_plan_t p) {
    if (!p) return MOA_OK;
    prof_free(p);
    for (auto &r : p->rings)
        if (r.stats) {
            unsigned long long h[6] = {0};
            cudaMemcpy(h, r.stats, sizeof(h), cudaMemcpyDeviceToHost);
            std::fprintf(stderr,
                         "moa ring stats (%llu execs): B waits %llu spins %llu cycles %llu | A waits %llu spins %llu "
                         "cycles %llu\n",
                         r.epoch, h[0], h[1], h[2], h[3], h[4], h[5]);
        }
    for (int k = 0; k < 2; k++) {
        if (p->sub[k]) moa_fft_destroy(p->sub[k]);
        if (p->ss[k]) cudaStreamDestroy(p->ss[k]);
    }
    for (void *a : p->allocs) cudaFree(a);
    if (p->dist) dist_plan_free(p->dist);
    delete p;
    return MOA_OK;
}

int64_t moa_fft_local_elems(moa_fft_plan_t p) { return p ? p->local_elems : -1; }

int moa_fft_launches_per_exec(moa_fft_plan_t p) {
    if (!p) return -1;
    return p->dist ? dist_launches(p->dist, p->passes) : local_launches(p);
}

moa_status_t moa_psi_describe(int64_t n, int64_t batch, moa_dtype_t dtype, const int64_t *radices, int nrad,
                              moa_pass_desc_t *out, int max_passes, int *npasses) {
    if (!out || !npasses) return fail(MOA_EINVAL, "describe: null output");
    if (!pow2(n) || batch < 1) return fail(MOA_EINVAL, "describe: n must be a power of two, batch >= 1");
    if (dtype != MOA_C64 && dtype != MOA_C128) return fail(MOA_EINVAL, "describe: unknown dtype");
    std::vector<int64_t> rad;
    moa_status_t st = MOA_OK;
    if (radices) rad.assign(radices, radices + nrad);
    else st = plan_radices(n, batch, dtype, rad);
    if (st) return st;
    std::vector<moa_pass_desc_t> v;
    st = psi_build(n, batch, dtype, rad, radices == nullptr, v);
    if (st) return st;
    if (int(v.size()) > max_passes) return fail(MOA_EINVAL, "describe: output array too small");
    for (size_t i = 0; i < v.size(); i++) out[i] = v[i];
    *npasses = int(v.size());
    return MOA_OK;
}

moa_status_t moa_psi_describe_3d(int64_t n0, int64_t n1, int64_t n2, moa_dtype_t dtype, moa_pass_desc_t *out,
                                 int max_passes, int *npasses) {
    if (!out || !npasses) return fail(MOA_EINVAL, "describe_3d: null output");
    std::vector<moa_pass_desc_t> v;
    moa_status_t st = psi_3d_passes(n0, n1, n2, 1, dtype, v);
    if (!st) psi_fuse_3d(v, dtype);
    if (st) return st;
    if (int(v.size()) > max_passes) return fail(MOA_EINVAL, "describe_3d: output array too small");
    for (size_t i = 0; i < v.size(); i++) out[i] = v[i];
    *npasses = int(v.size());
    return MOA_OK;
}

moa_status_t moa_plan_radices(int64_t n, int64_t batch, moa_dtype_t dtype, int64_t *radices, int max_rad, int *nrad) {
    if (!radices || !nrad) return fail(MOA_EINVAL, "plan_radices: null output");
    std::vector<int64_t> r;
    moa_status_t st = plan_radices(n, batch, dtype, r);
    if (st) return st;
    if (int(r.size()) > max_rad) return fail(MOA_EINVAL, "plan_radices: output array too small");
    for (size_t i = 0; i < r.size(); i++) radices[i] = r[i];
    *nrad = int(r.size());
    return MOA_OK;
}

moa_status_t moa_pass_move(const moa_pass_desc_t *d, moa_dtype_t dtype, const void *in, void *out, void *stream) {
    if (!d || !in || !out) return fail(MOA_EINVAL, "pass_move: null argument");
    if (dtype != MOA_C64 && dtype != MOA_C128) return fail(MOA_EINVAL, "pass_move: unknown dtype");
    if (d->kind > 1 || d->logR < 0 || d->logR > 12 || d->ndig < 0 || d->ndig > MOA_MAX_DIGITS)
        return fail(MOA_EINVAL, "pass_move: not a lifted-pass descriptor");
    moa_pass_desc_t m = *d;
    m.kind = 1;
    m.twN = 1;
    m.ring = 0;
    DevTables none;
    cudaError_t e = launch_pass(m, dtype, in, out, none, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "pass_move launch");
    return MOA_OK;
}

moa_status_t moa_fft_output_index(moa_fft_plan_t p, int64_t *pos, int64_t count) {
    if (!p || !pos) return fail(MOA_EINVAL, "output_index: null argument");
    if (p->is3d) return fail(MOA_EUNSUPPORTED, "output_index: 1-D plans only");
    if (count != p->n) return fail(MOA_EINVAL, "output_index: count must equal n");
    const int64_t n = p->n;
    if (p->dist) {
        const int64_t P = p->ngpu, M = n / P;
        const bool lifted = p->flags & MOA_FFT_LIFTED_ORDER;
        for (int64_t k = 0; k < n; k++) pos[k] = lifted ? (k % P) * M + k / P : k;
        return MOA_OK;
    }
    if (!p->lifted_out) {
        for (int64_t k = 0; k < n; k++) pos[k] = k;
        return MOA_OK;
    }
    // every (line, k) of the last pass of row 0: natural address -> lifted address
    const moa_pass_desc_t &nat = p->natural_last, &lif = p->passes.back();
    const int64_t R = int64_t(1) << nat.logR;
    int64_t lines = 1;
    for (int i = 0; i < nat.ndig; i++) lines *= nat.ext[i];
    const int64_t row_lines = lines / p->batch;  // the batch digit is the slowest
    for (int64_t l = 0; l < row_lines; l++) {
        int64_t rem = l, na = 0, la = 0;
        for (int i = 0; i < nat.ndig; i++) {
            const int64_t d = rem % nat.ext[i];
            rem /= nat.ext[i];
            na += d * nat.out_str[i];
            la += d * lif.out_str[i];
        }
        for (int64_t k = 0; k < R; k++) {
            const int64_t a = na + k * nat.out_kstr;
            if (a < 0 || a >= n) return fail(MOA_EINVAL, "output_index: descriptor out of range");
            pos[a] = la + k * lif.out_kstr;
        }
    }
    return MOA_OK;
}

moa_status_t moa_fft_plan_describe(moa_fft_plan_t p, moa_pass_desc_t *out, int max_passes, int *npasses) {
    if (!p || !out || !npasses) return fail(MOA_EINVAL, "plan_describe: null argument");
    if (int(p->passes.size()) > max_passes) return fail(MOA_EINVAL, "plan_describe: output array too small");
    for (size_t i = 0; i < p->passes.size(); i++) out[i] = p->passes[i];
    *npasses = int(p->passes.size());
    return MOA_OK;
}

}  // extern "C"

extern "C" moa_status_t moa_fft_exec_loopback(moa_fft_plan_t *plans, int ngpu, const void *const *ins,
                                              void *const *outs, void *stream) {
    if (!plans || !ins || !outs) return fail(MOA_EINVAL, "exec_loopback: null argument");
    for (int r = 0; r < ngpu; r++) {
        if (!plans[r] || !plans[r]->dist || !plans[r]->dist->loopback || plans[r]->dist->ngpu != ngpu ||
            plans[r]->dist->rank != r)
            return fail(MOA_EINVAL, "exec_loopback: plans[r] must be loopback plan of virtual rank r");
        if (!ins[r] || !outs[r]) return fail(MOA_EINVAL, "exec_loopback: null buffer");
    }
    // the product step loop (dist_exec) with the loopback exchange backend
    std::vector<DistRank> ranks;
    for (int r = 0; r < ngpu; r++) {
        moa_fft_plan_s *p = plans[r];
        ranks.push_back({p->dist, &p->passes, &p->tabs, {const_cast<void *>(ins[r]), outs[r], p->scratch, p->dist->scratch2},
                         p->flags});
    }
    moa_fft_plan_s *p0 = plans[0];
    cudaEvent_t *evs = nullptr;
    if (p0->prof_count < p0->prof_max) evs = &p0->prof_ev[size_t(p0->prof_count) * (p0->prof_nsteps + 1)];
    moa_status_t st = dist_exec(ranks, DistBackend::Loopback, p0->dtype, reinterpret_cast<cudaStream_t>(stream), evs,
                                p0->n);
    if (evs) p0->prof_count++;
    return st;
}

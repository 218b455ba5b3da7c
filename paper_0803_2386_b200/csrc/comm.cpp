// comm.cpp -- processor-level lifting over NCCL (step a8).
//
// Schedules (verified on the host by tests/test_dist_gloo.py):
//
// 1-D, N = p M, rank g holds x[g M, (g+1) M) and receives X[g M, (g+1) M):
//   X[k1 + p k2] = sum_{j_lo} w_M^{j_lo k2} w_N^{j_lo k1} sum_g x[g M + j_lo] w_p^{g k1}
//   E1  all-to-all (chunk h of every block -> rank h)
//   A   p-point DFT over g + lifted weight w_N^{(h M/p + m') k1}, stored [k1][m']
//   E2  all-to-all (rank k1 now holds y[k1][j_lo] for all j_lo, natural order)
//   B   the length-M lifted FFT of the local row (the one-GPU passes)
//   E3  all-to-all (rank g' receives X'[k1][k2_loc], k2 in block g')
//   U   p-way interleave out[k2_loc p + k1] (a data-movement pass)
// 3-D slab, rank g holds planes j0 in [g n0/p, (g+1) n0/p):
//   z-pass, y-pass stored in packed order [h][j0_loc][k1_loc][k2], one
//   all-to-all, x-pass -> y-slab [k0][k1_loc][k2].
//
// NCCL is loaded at run time (dlopen of the libnccl.so.2 torch already loaded),
// so the library itself loads on machines without it.
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <string>

#include "comm.h"
#include "nccl.h"

namespace moa {
namespace {

struct Nccl {
    void *h = nullptr;
    decltype(&::ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&::ncclCommInitRank) commInitRank = nullptr;
    decltype(&::ncclCommDestroy) commDestroy = nullptr;
    decltype(&::ncclCommAbort) commAbort = nullptr;
    decltype(&::ncclAlltoAll) alltoAll = nullptr;  // NCCL >= 2.28; else grouped send / recv below
    decltype(&::ncclSend) send = nullptr;
    decltype(&::ncclRecv) recv = nullptr;
    decltype(&::ncclGroupStart) groupStart = nullptr;
    decltype(&::ncclGroupEnd) groupEnd = nullptr;
    decltype(&::ncclAllGather) allGather = nullptr;
    decltype(&::ncclAllReduce) allReduce = nullptr;
    decltype(&::ncclGetErrorString) errStr = nullptr;
};
Nccl g_nccl;
ncclComm_t g_comm = nullptr;
int g_rank = -1, g_ngpu = 0;
bool g_loopback = false;

// Binds one candidate library; false (nothing kept) when it lacks an entry point
// the path needs.  The all-to-all is ncclAlltoAll where the library has it
// (NCCL >= 2.28), else one ncclSend + ncclRecv per peer inside a group.
bool bind_nccl(void *h, bool need_alltoall) {
    Nccl n;
    n.h = h;
    n.getUniqueId = (decltype(n.getUniqueId))dlsym(h, "ncclGetUniqueId");
    n.commInitRank = (decltype(n.commInitRank))dlsym(h, "ncclCommInitRank");
    n.commDestroy = (decltype(n.commDestroy))dlsym(h, "ncclCommDestroy");
    n.commAbort = (decltype(n.commAbort))dlsym(h, "ncclCommAbort");
    n.alltoAll = (decltype(n.alltoAll))dlsym(h, "ncclAlltoAll");
    n.send = (decltype(n.send))dlsym(h, "ncclSend");
    n.recv = (decltype(n.recv))dlsym(h, "ncclRecv");
    n.groupStart = (decltype(n.groupStart))dlsym(h, "ncclGroupStart");
    n.groupEnd = (decltype(n.groupEnd))dlsym(h, "ncclGroupEnd");
    n.allGather = (decltype(n.allGather))dlsym(h, "ncclAllGather");
    n.allReduce = (decltype(n.allReduce))dlsym(h, "ncclAllReduce");
    n.errStr = (decltype(n.errStr))dlsym(h, "ncclGetErrorString");
    if (!n.getUniqueId || !n.commInitRank || !n.commDestroy || !n.allGather || !n.allReduce) return false;
    const bool p2p = n.send && n.recv && n.groupStart && n.groupEnd;
    if (need_alltoall ? !n.alltoAll : !(n.alltoAll || p2p)) return false;
    g_nccl = n;
    return true;
}

moa_status_t load_nccl() {
    if (g_nccl.h) return MOA_OK;
    // MOA_NCCL_LIB, then a libnccl this process has already loaded (torch's
    // bundled one), then the search path.  First round: a library with
    // ncclAlltoAll; second: any with send / recv (the system 2.27).
    const char *env = std::getenv("MOA_NCCL_LIB");
    bool opened = false;
    for (int round = 0; round < 2; round++) {
        struct { const char *name; int flags; } cand[] = {
            {env, RTLD_NOW | RTLD_GLOBAL},
            {"libnccl.so.2", RTLD_NOW | RTLD_NOLOAD},
            {"libnccl.so.2", RTLD_NOW | RTLD_GLOBAL},
            {"libnccl.so", RTLD_NOW | RTLD_GLOBAL}};
        for (auto &c : cand) {
            if (!c.name || !c.name[0]) continue;
            void *h = dlopen(c.name, c.flags);
            if (!h) continue;
            opened = true;
            if (bind_nccl(h, round == 0)) return MOA_OK;
            dlclose(h);
        }
    }
    return fail(MOA_ENCCL, opened ? "NCCL: the loaded library lacks ncclAlltoAll and ncclSend / ncclRecv"
                                  : "NCCL: cannot dlopen libnccl.so.2 (set MOA_NCCL_LIB)");
}

// chunk h (cnt elements) of `src` to rank h, chunk g of `dst` from rank g
ncclResult_t nccl_all_to_all(const void *src, void *dst, size_t cnt, ncclDataType_t ty, size_t tsize, int p,
                             cudaStream_t s) {
    if (g_nccl.alltoAll) return g_nccl.alltoAll(src, dst, cnt, ty, g_comm, s);
    ncclResult_t r = g_nccl.groupStart();
    if (r != ncclSuccess) return r;
    for (int h = 0; h < p && r == ncclSuccess; h++) {
        r = g_nccl.send(static_cast<const char *>(src) + size_t(h) * cnt * tsize, cnt, ty, h, g_comm, s);
        if (r == ncclSuccess) r = g_nccl.recv(static_cast<char *>(dst) + size_t(h) * cnt * tsize, cnt, ty, h, g_comm, s);
    }
    ncclResult_t e = g_nccl.groupEnd();
    return r != ncclSuccess ? r : e;
}

moa_status_t nccl_fail(ncclResult_t r, const char *what) {
    std::string m = std::string("NCCL ") + what + ": " + (g_nccl.errStr ? g_nccl.errStr(r) : "error");
    if (g_comm && g_nccl.commAbort) {
        g_nccl.commAbort(g_comm);
        g_comm = nullptr;
        g_rank = -1;
        g_ngpu = 0;
    }
    return fail(MOA_ENCCL, m);
}

void dinit(moa_pass_desc_t &d, int logR) {
    std::memset(&d, 0, sizeof(d));
    d.logR = logR;
    d.twN = 1;
    d.out_ksplit = 62;
}
void dig(moa_pass_desc_t &d, int64_t ext, int64_t is, int64_t os, int64_t ts) {
    if (ext == 1) return;
    d.ext[d.ndig] = ext;
    d.in_str[d.ndig] = is;
    d.out_str[d.ndig] = os;
    d.tw_str[d.ndig] = ts;
    d.ndig++;
}

}  // namespace

bool dist_ready(int ngpu) { return (g_comm || g_loopback) && g_ngpu == ngpu; }

void fuse_exchanges(std::vector<DistStep> &steps, std::vector<moa_pass_desc_t> &passes) {
    std::vector<DistStep> out;
    bool synced = false;         // a synchronisation (exchange / barrier) earlier in this exec
    bool read_since[4] = {};     // buffers read by a pass since the last synchronisation
    int rename_from = -1, rename_to = -1;
    auto sync = [&] {
        synced = true;
        for (bool &r : read_since) r = false;
    };
    for (size_t i = 0; i < steps.size(); i++) {
        DistStep s = steps[i];
        if (s.kind == 0 && s.src == rename_from) {
            s.src = rename_to;
            passes[s.pass].src = rename_to;
        }
        if (s.kind == 1) {
            if (s.src == rename_from) s.src = rename_to;
            out.push_back(s);
            sync();
            continue;
        }
        const bool fusable = s.kind == 0 && i + 1 < steps.size() && steps[i + 1].kind == 1 && steps[i + 1].src == s.dst &&
                             passes[s.pass].dst == s.dst && !passes[s.pass].ring && passes[s.pass].kind == 0;
        if (!fusable) {
            read_since[s.src] = true;
            out.push_back(s);
            continue;
        }
        const DistStep &x = steps[i + 1];
        int target;
        if (!read_since[x.src] && s.src != x.src) {
            target = x.src;  // later reads of the exchange's destination read here instead
            rename_from = x.dst;
            rename_to = x.src;
        } else if (!read_since[x.dst] && s.src != x.dst) {
            target = x.dst;
        } else {
            out.push_back({3, -1, -1, -1, 0});
            sync();
            target = x.dst;
        }
        if (!synced) {  // an earlier exec's reads of the target may still be running on a peer
            out.push_back({3, -1, -1, -1, 0});
            sync();
        }
        out.push_back({2, s.pass, s.src, target, x.count});
        out.push_back({3, -1, -1, -1, 0});
        sync();
        i++;
    }
    steps.swap(out);
}

namespace {
// One int per rank through the communicator (plan time only): the minimum over
// ranks, or 0 if the reduction itself fails.
int all_ranks_min(int v) {
    int *d = nullptr;
    int out = 0;
    cudaStream_t s = nullptr;
    if (cudaMalloc(&d, sizeof(int)) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    bool ok = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess &&
              cudaMemcpy(d, &v, sizeof(int), cudaMemcpyHostToDevice) == cudaSuccess &&
              g_nccl.allReduce(d, d, 1, ncclInt32, ncclMin, g_comm, s) == ncclSuccess &&
              cudaStreamSynchronize(s) == cudaSuccess &&
              cudaMemcpy(&out, d, sizeof(int), cudaMemcpyDeviceToHost) == cudaSuccess;
    if (s) cudaStreamDestroy(s);
    cudaFree(d);
    if (!ok) cudaGetLastError();
    return ok ? out : 0;
}

// Map every rank's scratch buffer `id` into this process (CUDA IPC over
// NVLink): the handles are all-gathered through the communicator at plan time.
// Every rank takes part in the all-gather even when its own handle is missing
// (a flag travels with the handle), so a local failure cannot leave the other
// ranks waiting in a collective; the outcome is the same on every rank up to
// the opens, which dist_finish reconciles with all_ranks_min.
moa_status_t setup_peers(DistPlan *dp, int id, void *local) {
    struct Msg {
        cudaIpcMemHandle_t h;
        int ok;
    } mine{};
    mine.ok = local && cudaIpcGetMemHandle(&mine.h, local) == cudaSuccess;
    if (!mine.ok) cudaGetLastError();
    const size_t hb = sizeof(Msg);
    char *d = nullptr;
    if (cudaMalloc(&d, hb * dp->ngpu) != cudaSuccess) {
        cudaGetLastError();
        return fail(MOA_ENOMEM, "peer handle buffer");
    }
    std::vector<Msg> all(dp->ngpu);
    cudaStream_t s = nullptr;
    bool ok = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess &&
              cudaMemcpy(d + hb * dp->rank, &mine, hb, cudaMemcpyHostToDevice) == cudaSuccess &&
              g_nccl.allGather(d + hb * dp->rank, d, hb, ncclChar, g_comm, s) == ncclSuccess &&
              cudaStreamSynchronize(s) == cudaSuccess &&
              cudaMemcpy(all.data(), d, hb * dp->ngpu, cudaMemcpyDeviceToHost) == cudaSuccess;
    if (s) cudaStreamDestroy(s);
    cudaFree(d);
    if (!ok) {
        cudaGetLastError();
        return fail(MOA_ENCCL, "peer handle exchange failed");
    }
    for (int g = 0; g < dp->ngpu; g++)
        if (!all[g].ok) return fail(MOA_EUNSUPPORTED, "cudaIpcGetMemHandle failed on some rank");
    for (int g = 0; g < dp->ngpu; g++) {
        if (g == dp->rank) {
            dp->peer_buf[id][g] = local;
            continue;
        }
        if (cudaIpcOpenMemHandle(&dp->peer_buf[id][g], all[g].h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            cudaGetLastError();
            return fail(MOA_EUNSUPPORTED, "cudaIpcOpenMemHandle failed (no peer access?)");
        }
        dp->peer_opened[id][g] = true;
    }
    return MOA_OK;
}

void close_peers(DistPlan *dp) {
    for (int id = 0; id < 4; id++)
        for (int g = 0; g < 8; g++) {
            if (dp->peer_opened[id][g]) cudaIpcCloseMemHandle(dp->peer_buf[id][g]);
            dp->peer_opened[id][g] = false;
            dp->peer_buf[id][g] = nullptr;
        }
    if (dp->barrier_buf) cudaFree(dp->barrier_buf);
    dp->barrier_buf = nullptr;
}
}  // namespace

moa_status_t dist_finish(DistPlan *dp, void *scratch) {
    const char *pe = std::getenv("MOA_FFT_PEER");
    if (pe && pe[0] == '0') return MOA_OK;
    std::vector<DistStep> steps = dp->steps;
    std::vector<moa_pass_desc_t> passes = dp->passes;
    fuse_exchanges(steps, passes);
    if (!dp->loopback) {  // (the loopback maps the virtual ranks' buffers at exec time)
        void *local[4] = {nullptr, nullptr, scratch, dp->scratch2};
        bool need[4] = {};
        for (auto &s : steps)
            if (s.kind == 2) need[s.dst] = true;
        // (the schedule, hence `need`, is the same on every rank)
        // (user buffers 0 / 1 change per exec: no mapping, no fusion)
        if (need[0] || need[1]) return MOA_OK;
        bool ok = true;
        for (int id = 2; id < 4; id++)  // every needed id on every rank (collectives match)
            if (need[id] && setup_peers(dp, id, local[id]) != MOA_OK) ok = false;
        if (ok && cudaMalloc(&dp->barrier_buf, 16) != cudaSuccess) {
            cudaGetLastError();
            dp->barrier_buf = nullptr;
            ok = false;
        }
        if (ok) ok = cudaMemset(dp->barrier_buf, 0, 16) == cudaSuccess;
        // every rank must run the same schedule: fuse only if all ranks could
        if (all_ranks_min(ok ? 1 : 0) != 1) {
            close_peers(dp);
            return MOA_OK;  // fused exchanges stay off: the NCCL schedule runs
        }
    }
    dp->steps.swap(steps);
    dp->passes.swap(passes);
    return MOA_OK;
}

moa_status_t dist_schedule_1d(int g, int p, int64_t N, moa_dtype_t dtype, std::vector<moa_pass_desc_t> &passes,
                              std::vector<DistStep> &steps, bool lifted_order) {
    passes.clear();
    steps.clear();
    const int64_t M = N / p, C = M / p;
    const int lp = log2_exact(p);
    // E1
    steps.push_back({1, -1, 0, 2, C});
    // A: p-point DFT over the received chunks, weights w_N^{(g C + m') k1}
    {
        moa_pass_desc_t d;
        dinit(d, lp);
        dig(d, C, 1, 1, 1);
        d.in_kstr = d.out_kstr = C;
        d.twN = N;
        d.tw_off = int64_t(g) * C;
        d.lf_load = d.lf_store = 1;
        d.src = d.dst = 2;
        psi_choose_tile(d, dtype);
        steps.push_back({0, int(passes.size()), 2, 2, 0});
        passes.push_back(d);
    }
    // E2
    steps.push_back({1, -1, 2, 3, C});
    // B: the local length-M FFT; buffer ids remapped in -> 3, scratch -> out(1), out -> 2
    // (lifted order: in -> 3, scratch -> 2, out -> 1 -- B writes the result,
    // X[g + p k2] at offset k2, and E3 + the unpack are skipped)
    {
        std::vector<int64_t> rad;
        moa_status_t st = plan_radices(M, 1, dtype, rad);
        if (st) return st;
        std::vector<moa_pass_desc_t> b;
        st = psi_lift_passes(M, 1, dtype, rad.data(), int(rad.size()), b);
        if (st) return st;
        const int remap_nat[3] = {3, 2, 1}, remap_lift[3] = {3, 1, 2};
        const int *remap = lifted_order ? remap_lift : remap_nat;
        for (auto &d : b) {
            d.src = remap[d.src];
            d.dst = remap[d.dst];
            steps.push_back({0, int(passes.size()), d.src, d.dst, 0});
            passes.push_back(d);
        }
    }
    if (lifted_order) return MOA_OK;
    // E3
    steps.push_back({1, -1, 2, 3, C});
    // U: out[k2_loc p + k1] = buf[k1][k2_loc]
    {
        moa_pass_desc_t d;
        dinit(d, lp);
        dig(d, C, 1, p, 0);
        d.in_kstr = C;
        d.out_kstr = 1;
        d.kind = 1;
        d.lf_load = 1;
        d.lf_store = 0;
        d.src = 3;
        d.dst = 1;
        psi_choose_tile(d, dtype);
        steps.push_back({0, int(passes.size()), 3, 1, 0});
        passes.push_back(d);
    }
    return MOA_OK;
}

moa_status_t dist_schedule_3d(int g, int p, int64_t n0, int64_t n1, int64_t n2, moa_dtype_t dtype,
                              std::vector<moa_pass_desc_t> &passes, std::vector<DistStep> &steps) {
    (void)g;
    passes.clear();
    steps.clear();
    const int64_t n0l = n0 / p, n1l = n1 / p;
    {  // z-pass on the x-slab
        moa_pass_desc_t d;
        dinit(d, log2_exact(n2));
        dig(d, n1, n2, n2, 0);
        dig(d, n0l, n1 * n2, n1 * n2, 0);
        d.in_kstr = d.out_kstr = 1;
        d.src = 0;
        d.dst = 1;
        psi_choose_tile(d, dtype);
        steps.push_back({0, int(passes.size()), 0, 1, 0});
        passes.push_back(d);
    }
    {  // y-pass, stored in packed (send) order [h][j0_loc][k1_loc][k2]
        moa_pass_desc_t d;
        dinit(d, log2_exact(n1));
        dig(d, n2, 1, 1, 0);
        dig(d, n0l, n1 * n2, n1l * n2, 0);
        d.in_kstr = n2;
        d.out_kstr = n2;
        d.out_ksplit = log2_exact(n1l);
        d.out_kstr_hi = n0l * n1l * n2;
        d.lf_load = d.lf_store = 1;
        d.src = 1;
        d.dst = 2;
        psi_choose_tile(d, dtype);
        steps.push_back({0, int(passes.size()), 1, 2, 0});
        passes.push_back(d);
    }
    steps.push_back({1, -1, 2, 1, n0l * n1l * n2});
    {  // x-pass on [n0][n1_loc][n2]
        moa_pass_desc_t d;
        dinit(d, log2_exact(n0));
        dig(d, n2, 1, 1, 0);
        dig(d, n1l, n2, n2, 0);
        d.in_kstr = d.out_kstr = n1l * n2;
        d.lf_load = d.lf_store = 1;
        d.src = 1;
        d.dst = 1;
        psi_choose_tile(d, dtype);
        steps.push_back({0, int(passes.size()), 1, 1, 0});
        passes.push_back(d);
    }
    return MOA_OK;
}

moa_status_t dist_plan_1d(DistPlan *&dp, int64_t n, moa_dtype_t dtype, bool lifted_order) {
    dp = new DistPlan;
    dp->rank = g_rank;
    dp->ngpu = g_ngpu;
    dp->loopback = g_loopback;
    dp->esize = dtype == MOA_C128 ? 16 : 8;
    dp->local_elems = n / g_ngpu;
    moa_status_t st = dist_schedule_1d(g_rank, g_ngpu, n, dtype, dp->passes, dp->steps, lifted_order);
    if (st) return st;
    cudaError_t e = cudaMalloc(&dp->scratch2, size_t(dp->local_elems) * dp->esize);
    if (e != cudaSuccess) {
        cudaGetLastError();
        dp->scratch2 = nullptr;
        return fail(MOA_ENOMEM, "dist: scratch allocation failed");
    }
    return MOA_OK;
}

moa_status_t dist_plan_3d(DistPlan *&dp, int64_t n0, int64_t n1, int64_t n2, moa_dtype_t dtype) {
    dp = new DistPlan;
    dp->rank = g_rank;
    dp->ngpu = g_ngpu;
    dp->loopback = g_loopback;
    dp->esize = dtype == MOA_C128 ? 16 : 8;
    dp->local_elems = n0 * n1 * n2 / g_ngpu;
    return dist_schedule_3d(g_rank, g_ngpu, n0, n1, n2, dtype, dp->passes, dp->steps);
}

void dist_plan_free(DistPlan *dp) {
    if (!dp) return;
    for (int id = 0; id < 4; id++)
        for (int g = 0; g < 8; g++)
            if (dp->peer_opened[id][g]) cudaIpcCloseMemHandle(dp->peer_buf[id][g]);
    if (dp->barrier_buf) cudaFree(dp->barrier_buf);
    if (dp->scratch2) cudaFree(dp->scratch2);
    delete dp;
}

int dist_launches(DistPlan *dp, const std::vector<moa_pass_desc_t> &passes) {
    (void)passes;
    int c = 0;
    for (auto &s : dp->steps) c += s.kind == 0 || s.kind == 2;
    return c;
}

moa_status_t dist_exec(const std::vector<DistRank> &ranks, DistBackend be, moa_dtype_t dtype, cudaStream_t s,
                       cudaEvent_t *evs, int64_t N) {
    if (ranks.empty()) return fail(MOA_EINVAL, "dist: no ranks");
    const DistPlan *dp0 = ranks[0].dp;
    const int p = dp0->ngpu;
    if (be == DistBackend::Nccl) {
        if (ranks.size() != 1 || dp0->loopback) return fail(MOA_EINVAL, "dist: an NCCL exec runs this process's rank only");
        if (!g_comm) return fail(MOA_EINVAL, "dist: no communicator (moa_fft_dist_init)");
    } else if (int(ranks.size()) != p) {
        return fail(MOA_EINVAL, "dist: a loopback exec runs every virtual rank");
    }
    // the peer buffer `id` of rank g as seen by this process: mapped over NVLink
    // (CUDA IPC, NCCL backend) or the co-located virtual rank's own buffer
    auto peer = [&](const DistRank &me, int g, int id) -> void * {
        if (be == DistBackend::Nccl) return me.dp->peer_buf[id][g];
        return ranks[g].bufs[id];
    };
    for (size_t i = 0; i < dp0->steps.size(); i++) {
        const DistStep &st = dp0->steps[i];  // (every rank runs the same schedule)
        if (evs) cudaEventRecord(evs[i], s);
        if (st.kind == 0 || st.kind == 2) {
            for (const DistRank &r : ranks) {
                const moa_pass_desc_t &d = (*r.passes)[st.pass];
                PassMods mods = pass_mods(r.flags, size_t(st.pass), r.passes->size(), N);
                if (st.kind == 2) {  // the exchange folded into the stores: NVLink writes into every rank's buffer
                    mods.npeers = p;
                    for (int g = 0; g < p; g++) mods.peers[g] = peer(r, g, st.dst);
                    mods.log_chunk = log2_exact(st.count);
                    mods.self_off = int64_t(r.dp->rank) * st.count;
                }
                cudaError_t e = launch_pass(d, dtype, r.bufs[d.src], r.bufs[st.kind == 2 ? st.dst : d.dst],
                                            (*r.tabs)[st.pass], s, mods);
                if (e != cudaSuccess) return fail(MOA_ECUDA, std::string("dist pass: ") + cudaGetErrorString(e));
            }
        } else if (st.kind == 3) {  // every rank's fused stores have landed before anyone reads them
            if (be == DistBackend::Nccl) {
                ncclResult_t rr = g_nccl.allReduce(dp0->barrier_buf, dp0->barrier_buf, 1, ncclFloat, ncclSum, g_comm, s);
                if (rr != ncclSuccess) return nccl_fail(rr, "barrier");
            }
            // loopback: every virtual rank's kernels run in order on one stream
        } else if (be == DistBackend::Nccl) {
            const size_t cnt = size_t(st.count) * 2;
            ncclResult_t rr = nccl_all_to_all(ranks[0].bufs[st.src], ranks[0].bufs[st.dst], cnt,
                                              dtype == MOA_C128 ? ncclDouble : ncclFloat,
                                              dtype == MOA_C128 ? 8 : 4, p, s);
            if (rr != ncclSuccess) return nccl_fail(rr, "all-to-all");
        } else {  // loopback all-to-all: chunk h of rank g -> chunk g of rank h (one copy per chunk)
            const size_t cb = size_t(st.count) * dp0->esize;
            for (int h = 0; h < p; h++)
                for (int g = 0; g < p; g++) {
                    char *dst = static_cast<char *>(ranks[h].bufs[st.dst]) + size_t(g) * cb;
                    const char *src = static_cast<const char *>(ranks[g].bufs[st.src]) + size_t(h) * cb;
                    cudaError_t e = cudaMemcpyAsync(dst, src, cb, cudaMemcpyDeviceToDevice, s);
                    if (e != cudaSuccess) return fail(MOA_ECUDA, std::string("loopback copy: ") + cudaGetErrorString(e));
                }
        }
    }
    if (evs) cudaEventRecord(evs[dp0->steps.size()], s);
    return MOA_OK;
}

}  // namespace moa

using namespace moa;

extern "C" {

moa_status_t moa_fft_get_unique_id(uint8_t id[128]) {
    if (!id) return fail(MOA_EINVAL, "get_unique_id: null output");
    moa_status_t st = load_nccl();
    if (st) return st;
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
    ncclUniqueId u;
    ncclResult_t r = g_nccl.getUniqueId(&u);
    if (r != ncclSuccess) return nccl_fail(r, "get unique id");
    std::memcpy(id, &u, 128);
    return MOA_OK;
}

moa_status_t moa_fft_dist_init(int rank, int ngpu, const uint8_t id[128]) {
    if (!id) return fail(MOA_EINVAL, "dist_init: null id");
    if (!(ngpu == 2 || ngpu == 4 || ngpu == 8)) return fail(MOA_EINVAL, "dist_init: ngpu must be 2, 4 or 8");
    if (rank < 0 || rank >= ngpu) return fail(MOA_EINVAL, "dist_init: rank out of range");
    moa_status_t st = load_nccl();
    if (st) return st;
    if (g_comm) return fail(MOA_EINVAL, "dist_init: already initialised (moa_fft_dist_finalize first)");
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    ncclComm_t c = nullptr;
    ncclResult_t r = g_nccl.commInitRank(&c, ngpu, u, rank);
    if (r != ncclSuccess) return nccl_fail(r, "comm init");
    g_comm = c;
    g_rank = rank;
    g_ngpu = ngpu;
    g_loopback = false;
    return MOA_OK;
}

moa_status_t moa_fft_dist_finalize(void) {
    if (g_comm) g_nccl.commDestroy(g_comm);
    g_comm = nullptr;
    g_rank = -1;
    g_ngpu = 0;
    g_loopback = false;
    return MOA_OK;
}

// Loopback: plan virtual rank `rank` of `ngpu` on the current device with no
// communicator; the plans of all virtual ranks execute together through
// moa_fft_exec_loopback (exchanges become device-to-device copies).  Runs the
// exact per-rank kernels and chunk maps of the NCCL path on one GPU.
moa_status_t moa_fft_dist_loopback(int rank, int ngpu) {
    if (!(ngpu == 2 || ngpu == 4 || ngpu == 8) || rank < 0 || rank >= ngpu)
        return fail(MOA_EINVAL, "dist_loopback: bad rank / ngpu");
    if (g_comm) return fail(MOA_EINVAL, "dist_loopback: a real communicator is active");
    g_loopback = true;
    g_rank = rank;
    g_ngpu = ngpu;
    return MOA_OK;
}

// Host-only: the distributed schedule of one rank (tests / introspection).
// kinds[i] = 0 pass / 1 all-to-all; counts[i] = per-peer elements of an all-to-all.
moa_status_t moa_dist_describe(int rank, int ngpu, int is3d, int64_t n0, int64_t n1, int64_t n2, moa_dtype_t dtype,
                               void *passes_v, int max_passes, int *npasses, int32_t *kinds,
                               int32_t *srcs, int32_t *dsts, int64_t *counts, int max_steps, int *nsteps,
                               uint32_t flags) {
    moa_pass_desc_t *passes = static_cast<moa_pass_desc_t *>(passes_v);
    if (!passes || !npasses || !kinds || !srcs || !dsts || !counts || !nsteps)
        return fail(MOA_EINVAL, "dist_describe: null output");
    if (!(ngpu == 2 || ngpu == 4 || ngpu == 8) || rank < 0 || rank >= ngpu)
        return fail(MOA_EINVAL, "dist_describe: bad rank / ngpu");
    std::vector<moa_pass_desc_t> ps;
    std::vector<DistStep> ss;
    moa_status_t st;
    if (is3d) {
        if (n0 % ngpu || n1 % ngpu) return fail(MOA_EUNSUPPORTED, "dist_describe: ngpu must divide n0, n1");
        st = dist_schedule_3d(rank, ngpu, n0, n1, n2, dtype, ps, ss);
    } else {
        if (log2_exact(n0) < 0 || n0 < int64_t(ngpu) * ngpu) return fail(MOA_EUNSUPPORTED, "dist_describe: bad n");
        st = dist_schedule_1d(rank, ngpu, n0, dtype, ps, ss, (flags & MOA_FFT_LIFTED_ORDER) != 0);
    }
    if (st) return st;
    const char *pe = std::getenv("MOA_FFT_PEER");
    if (!(pe && pe[0] == '0')) fuse_exchanges(ss, ps);  // what a plan executes when peer mapping succeeds
    if (int(ps.size()) > max_passes || int(ss.size()) > max_steps) return fail(MOA_EINVAL, "dist_describe: arrays too small");
    for (size_t i = 0; i < ps.size(); i++) passes[i] = ps[i];
    for (size_t i = 0; i < ss.size(); i++) {
        kinds[i] = ss[i].kind;
        srcs[i] = (ss[i].kind == 0 || ss[i].kind == 2) ? ss[i].pass : ss[i].src;
        dsts[i] = ss[i].dst;
        counts[i] = ss[i].count;
    }
    *npasses = int(ps.size());
    *nsteps = int(ss.size());
    return MOA_OK;
}

}  // extern "C"

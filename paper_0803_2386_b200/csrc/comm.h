// comm.h -- processor-level lifting.
//
// PAPER.md states the principle only: the processor / network level is one more
// lifted dimension.  The
// design: the rank is one digit of the lifted index; an
// all-to-all over NVLink swaps which digit is distributed.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "moa_internal.h"

namespace moa {

// One step of a distributed exec: a local pass, or an all-to-all of `count`
// complex elements per peer from buffer src to buffer dst (ids as in
// moa_pass_desc_t: 0 in, 1 out, 2 scratch, 3 scratch2).
struct DistStep {
    int kind;  // 0 = pass (index into passes), 1 = all-to-all, 2 = pass fused with the
               // all-to-all that followed it (stores to the peers' buffer `dst`, `count`
               // elements per peer), 3 = barrier (every rank's previous steps are done)
    int pass;
    int src, dst;
    int64_t count;
};

struct DistPlan {
    int rank = 0, ngpu = 1;
    bool loopback = false;  // exchanges by device copies between co-located virtual ranks
    std::vector<moa_pass_desc_t> passes;
    std::vector<DistStep> steps;
    int64_t local_elems = 0;
    size_t esize = 16;
    void *scratch2 = nullptr;
    // fused exchanges (kind 2): every rank's scratch buffers (ids 2, 3), mapped
    // into this process over NVLink (CUDA IPC); peer_opened marks handles to close
    void *peer_buf[4][8] = {};
    bool peer_opened[4][8] = {};
    void *barrier_buf = nullptr;
};

// Fold every all-to-all that directly follows a pass writing its source buffer
// into that pass's stores (kind 2) plus a barrier (kind 3).  The fused stores go
// to a buffer no rank can still be reading: the exchange's source buffer when
// nothing read it since the last synchronisation (later reads of the exchange's
// destination are renamed to it), else its destination; a barrier is inserted
// first when there was no synchronisation yet in the exec.  Host only.
void fuse_exchanges(std::vector<DistStep> &steps, std::vector<moa_pass_desc_t> &passes);
// After the plan's scratch (buffer 2) exists: map the peers' buffers and fuse
// the exchanges (default; MOA_FFT_PEER=0 keeps every all-to-all in NCCL).
moa_status_t dist_finish(DistPlan *dp, void *scratch);

bool dist_ready(int ngpu);
moa_status_t dist_plan_1d(DistPlan *&dp, int64_t n, moa_dtype_t dtype, bool lifted_order = false);
moa_status_t dist_plan_3d(DistPlan *&dp, int64_t n0, int64_t n1, int64_t n2, moa_dtype_t dtype);
// One rank's view of an exec: its plan, pass descriptors, tables and the four
// buffers (0 in, 1 out, 2 scratch, 3 scratch2).
struct DistRank {
    const DistPlan *dp;
    const std::vector<moa_pass_desc_t> *passes;
    const std::vector<DevTables> *tabs;
    void *bufs[4];
    uint32_t flags;
};
// How the exchanges of the schedule are carried out.  Nccl: this process runs
// one rank; all-to-alls are ncclAlltoAll, barriers a one-element
// ncclAllReduce, fused stores go to the CUDA-IPC-mapped peer buffers.
// Loopback: this process runs every virtual rank on one GPU, in lock step on
// one stream; all-to-alls are device copies, barriers are stream order, fused
// stores go to the co-located ranks' buffers.  The step loop, the kernels, the
// chunk maps and the fused-store routing are the same code for both.
enum class DistBackend { Nccl, Loopback };
moa_status_t dist_exec(const std::vector<DistRank> &ranks, DistBackend be, moa_dtype_t dtype, cudaStream_t s,
                       cudaEvent_t *evs, int64_t N);
void dist_plan_free(DistPlan *dp);
int dist_launches(DistPlan *dp, const std::vector<moa_pass_desc_t> &passes);

// host-only construction of the distributed schedule for a given rank (used by
// the planner and by the introspection / gloo tests)
moa_status_t dist_schedule_1d(int rank, int ngpu, int64_t n, moa_dtype_t dtype, std::vector<moa_pass_desc_t> &passes,
                              std::vector<DistStep> &steps, bool lifted_order = false);
moa_status_t dist_schedule_3d(int rank, int ngpu, int64_t n0, int64_t n1, int64_t n2, moa_dtype_t dtype,
                              std::vector<moa_pass_desc_t> &passes, std::vector<DistStep> &steps);

}  // namespace moa

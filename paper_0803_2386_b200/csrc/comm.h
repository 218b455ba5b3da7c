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
    int kind;  // 0 = pass (index into passes), 1 = all-to-all
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
};

bool dist_ready(int ngpu);
moa_status_t dist_plan_1d(DistPlan *&dp, int64_t n, moa_dtype_t dtype, bool lifted_order = false);
moa_status_t dist_plan_3d(DistPlan *&dp, int64_t n0, int64_t n1, int64_t n2, moa_dtype_t dtype);
moa_status_t dist_exec(DistPlan *dp, const std::vector<moa_pass_desc_t> &passes, const std::vector<DevTables> &tabs,
                       moa_dtype_t dtype, const void *in, void *out, void *scratch, cudaStream_t s,
                       cudaEvent_t *evs, uint32_t flags, int64_t N);
void dist_plan_free(DistPlan *dp);
int dist_launches(DistPlan *dp, const std::vector<moa_pass_desc_t> &passes);

// host-only construction of the distributed schedule for a given rank (used by
// the planner and by the introspection / gloo tests)
moa_status_t dist_schedule_1d(int rank, int ngpu, int64_t n, moa_dtype_t dtype, std::vector<moa_pass_desc_t> &passes,
                              std::vector<DistStep> &steps, bool lifted_order = false);
moa_status_t dist_schedule_3d(int rank, int ngpu, int64_t n0, int64_t n1, int64_t n2, moa_dtype_t dtype,
                              std::vector<moa_pass_desc_t> &passes, std::vector<DistStep> &steps);

}  // namespace moa

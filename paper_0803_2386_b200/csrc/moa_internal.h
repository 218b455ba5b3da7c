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

// kernels.cu
struct DevTables {
    const void *twR = nullptr;   // w_R^e, e < R (this pass's in-line step twiddles)
    const void *tw_hi = nullptr; // w_N^{eh 2^h}
    const void *tw_lo = nullptr; // w_N^{el}
};
int log2_exact(int64_t n);
cudaError_t launch_pass(const moa_pass_desc_t &d, moa_dtype_t dtype, const void *in, void *out,
                        const DevTables &tab, cudaStream_t stream);
cudaError_t kernel_attributes(moa_dtype_t dtype, int logR, int *max_threads, int *regs);

}  // namespace moa

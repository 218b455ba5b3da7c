// tools/stride_bench.cu -- DRAM efficiency of the strided access pattern a
// line-coalesced pass makes: runs of RUN bytes (W adjacent lines) at a stride
// of S bytes between consecutive points, read and written back in place
// (one HBM round trip), vs a contiguous copy.  Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/stride_bench.cu -o tools/stride_bench
#include <cuda_runtime.h>
#include <stdio.h>

// element e of the 16-byte view: run r = e / epr (epr = elements per run), in
// the run at offset e % epr; runs are laid out column-major over (point k, col c):
// address = k * S + c * RUN, k fastest across consecutive runs when `kfast`
__global__ void strided_rw(double2 *a, size_t nelem, size_t S16, int epr, size_t npoints, int kfast) {
    for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < nelem; e += size_t(gridDim.x) * blockDim.x) {
        size_t run = e / epr, off = e % epr;
        size_t k, c;
        if (kfast) { k = run % npoints; c = run / npoints; }
        else { c = run % (S16 / epr); k = run / (S16 / epr); }
        size_t idx = k * S16 + c * epr + off;
        double2 v = __ldcs(a + idx);
        v.x += 1.0;
        __stcs(a + idx, v);
    }
}

int main() {
    const size_t bytes = size_t(4) << 30;
    const size_t nelem = bytes / 16;
    double2 *a;
    if (cudaMalloc(&a, bytes) != cudaSuccess) return 1;
    cudaMemset(a, 0, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int runs[] = {32, 64, 128, 256, 512};
    size_t strides[] = {size_t(4) << 10, size_t(16) << 10, size_t(256) << 10, size_t(1) << 20, size_t(16) << 20};
    printf("[");
    bool first = true;
    for (int kf = 0; kf < 2; kf++)
        for (int ri = 0; ri < 5; ri++)
            for (int si = 0; si < 5; si++) {
                int epr = runs[ri] / 16;
                size_t S16 = strides[si] / 16;
                size_t npoints = nelem / S16;
                float best = 1e9;
                for (int rep = 0; rep < 3; rep++) {
                    cudaEventRecord(e0);
                    strided_rw<<<148 * 8, 512>>>(a, nelem, S16, epr, npoints, kf);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (ms < best) best = ms;
                }
                printf("%s{\"kfast\": %d, \"run_B\": %d, \"stride_B\": %zu, \"GBps\": %.0f}", first ? "" : ",\n ", kf, runs[ri],
                       strides[si], 2.0 * bytes / (best * 1e-3) / 1e9);
                first = false;
            }
    printf("]\n");
    return cudaGetLastError() != cudaSuccess;
}

// tools/store_bench.cu -- contiguous loads, strided stores: a transposing
// copy of a [rows][cols] complex128 array into [cols][rows] where each thread
// group writes runs of RUN bytes (RUN/16 adjacent rows) per column.  The
// store side of a rotating-layout pass.  Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/store_bench.cu -o tools/store_bench
#include <cuda_runtime.h>
#include <stdio.h>

// tile = W rows x C cols; thread (r = tid % W, c0 = tid / W) loads a[row][c] for c = c0 + j*(T/W)
// (contiguous within a row) and stores b[c][row] (runs of W elements)
template <int W>
__global__ void transpose_rows(const double2 *__restrict__ a, double2 *__restrict__ b, int rows, int cols) {
    const int tiles_per_col = rows / W;
    const int tile = blockIdx.x;
    const int row0 = (tile % tiles_per_col) * W;
    const int r = threadIdx.x % W, c0 = threadIdx.x / W, cstep = blockDim.x / W;
    // each block does one W x cols tile (cols = 1024)
    for (int c = c0; c < cols; c += cstep) {
        double2 v = __ldcs(a + size_t(row0 + r) * cols + c);
        __stcs(b + size_t(c) * rows + row0 + r, v);
    }
}

int main() {
    const int cols = 1024;
    const size_t n = size_t(1) << 28;  // 4 GiB
    const int rows = int(n / cols);
    double2 *a, *b;
    if (cudaMalloc(&a, n * 16) != cudaSuccess || cudaMalloc(&b, n * 16) != cudaSuccess) return 1;
    cudaMemset(a, 0, n * 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](auto kern, int W, const char *name) {
        float best = 1e9;
        for (int rep = 0; rep < 3; rep++) {
            cudaEventRecord(e0);
            kern<<<rows / W, 256>>>(a, b, rows, cols);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        printf("{\"store_run_B\": %d, \"GBps\": %.0f}\n", W * 16, 2.0 * n * 16 / (best * 1e-3) / 1e9);
    };
    run(transpose_rows<1>, 1, "1");
    run(transpose_rows<2>, 2, "2");
    run(transpose_rows<4>, 4, "4");
    run(transpose_rows<8>, 8, "8");
    run(transpose_rows<16>, 16, "16");
    return 0;
}

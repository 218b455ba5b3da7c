// tools/microbench.cu -- B200 ceilings that decide the lifting design
// (DESIGN.md §4): HBM copy, L2-resident copy, DSMEM all-to-all inside a
// cluster, FP64 / FP32 FMA issue rate.  Not part of the product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/microbench.cu -o tools/microbench
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdio.h>

namespace cg = cooperative_groups;

#define CK(x)                                                                           \
    do {                                                                                \
        cudaError_t e = (x);                                                            \
        if (e != cudaSuccess) {                                                         \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            return 1;                                                                   \
        }                                                                               \
    } while (0)

__global__ void copy_kernel(const double2 *__restrict__ a, double2 *__restrict__ b, size_t n, int reps) {
    for (int r = 0; r < reps; r++) {
        for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
            b[i] = a[i];
    }
}

__global__ void copy_stream_kernel(const double2 *__restrict__ a, double2 *__restrict__ b, size_t n) {
    size_t base = (blockIdx.x * size_t(blockDim.x)) * 8 + threadIdx.x;
    double2 v[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
        size_t i = base + k * blockDim.x;
        if (i < n) v[k] = __ldcs(a + i);
    }
#pragma unroll
    for (int k = 0; k < 8; k++) {
        size_t i = base + k * blockDim.x;
        if (i < n) __stcs(b + i, v[k]);
    }
}

// every CTA of a cluster of 8 fills its smem, then reads the other 7 CTAs' smem
template <int CL>
__global__ void __cluster_dims__(CL, 1, 1) dsmem_kernel(double2 *out, int elems, int reps) {
    extern __shared__ double2 sm[];
    cg::cluster_group cluster = cg::this_cluster();
    const int me = cluster.block_rank();
    for (int i = threadIdx.x; i < elems; i += blockDim.x) sm[i] = make_double2(me + i, i);
    cluster.sync();
    double2 acc = make_double2(0, 0);
    const int chunk = elems / CL;  // each CTA reads its chunk from every other CTA
    for (int r = 0; r < reps; r++) {
        // 8 independent 16-byte remote loads in flight per thread
        const double2 *rem[CL];
#pragma unroll
        for (int q = 0; q < CL; q++) rem[q] = cluster.map_shared_rank(sm, q) + me * chunk;
        for (int i0 = threadIdx.x; i0 < chunk; i0 += blockDim.x) {
            double2 v[CL];
#pragma unroll
            for (int q = 0; q < CL; q++) v[q] = q == me ? make_double2(0, 0) : rem[q][i0];
#pragma unroll
            for (int q = 0; q < CL; q++) {
                acc.x += v[q].x;
                acc.y += v[q].y;
            }
        }
    }
    cluster.sync();
    if (acc.x == 12345.678) out[0] = acc;
}


// DSMEM all-to-all with bulk copies (cp.async.bulk shared::cluster): every CTA
// sends chunk q of its source buffer to CTA q (the exchange a cluster FFT makes)
__device__ __forceinline__ unsigned smem_u32(const void *p) { return unsigned(__cvta_generic_to_shared(p)); }
template <int CL>
__global__ void __cluster_dims__(CL, 1, 1) dsmem_bulk_kernel(double2 *out, int chunk_elems, int reps) {
    extern __shared__ __align__(128) double2 smb[];
    __shared__ __align__(8) unsigned long long mbar;
    cg::cluster_group cluster = cg::this_cluster();
    const int me = cluster.block_rank();
    double2 *src = smb, *dst = smb + CL * chunk_elems;
    for (int i = threadIdx.x; i < CL * chunk_elems; i += blockDim.x) src[i] = make_double2(me, i);
    const unsigned bytes = chunk_elems * 16;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    cluster.sync();
    for (int r = 0; r < reps; r++) {
        if (threadIdx.x == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(bytes * (CL - 1)));
        cluster.sync();
        if (threadIdx.x < CL && threadIdx.x != me) {
            const int q = threadIdx.x;
            unsigned rdst, rbar;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rdst) : "r"(smem_u32(dst + me * chunk_elems)), "r"(q));
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(smem_u32(&mbar)), "r"(q));
            asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(rdst), "r"(smem_u32(src + q * chunk_elems)), "r"(bytes), "r"(rbar) : "memory");
        }
        if (threadIdx.x == 0) {
            unsigned done = 0;
            while (!done)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                             : "=r"(done) : "r"(smem_u32(&mbar)), "r"(r & 1));
        }
        __syncthreads();
    }
    cluster.sync();
    if (dst[threadIdx.x].x == -1.0) out[0] = dst[0];
}

// L2-resident streaming read (every CTA re-reads a buffer that fits L2)
__global__ void l2_read_kernel(const double2 *__restrict__ a, double2 *out, size_t n, int reps) {
    double2 acc = make_double2(0, 0);
    for (int r = 0; r < reps; r++)
        for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
            double2 v = __ldcg(a + i);
            acc.x += v.x;
            acc.y += v.y;
        }
    if (acc.x == 12345.678) out[0] = acc;
}

__global__ void fma64_kernel(double *out, int iters) {
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double b = 1.0000001, c = 0.999999;
    for (int i = 0; i < iters; i++) {
        a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
        a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
    if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 0.123) out[0] = a0;
}

__global__ void fma32_kernel(float *out, int iters) {
    float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const float b = 1.0000001f, c = 0.999999f;
    for (int i = 0; i < iters; i++) {
        a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
        a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
    }
    if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 0.123f) out[0] = a0;
}

int main() {
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    printf("{\"device\": \"%s\", \"sms\": %d, \"l2_bytes\": %d", prop.name, prop.multiProcessorCount, prop.l2CacheSize);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    // HBM copy, 2 GiB -> 2 GiB
    {
        size_t n = (size_t(2) << 30) / 16;
        double2 *a, *b;
        CK(cudaMalloc(&a, n * 16));
        CK(cudaMalloc(&b, n * 16));
        CK(cudaMemset(a, 0, n * 16));
        int blocks = int((n + 256 * 8 - 1) / (256 * 8));
        copy_stream_kernel<<<blocks, 256>>>(a, b, n);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        for (int r = 0; r < 10; r++) copy_stream_kernel<<<blocks, 256>>>(a, b, n);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        printf(", \"hbm_copy_GBps\": %.1f", 10 * 2.0 * n * 16 / (ms * 1e-3) / 1e9);
        // L2-resident copy: 24 MiB -> 24 MiB repeatedly
        size_t m = (size_t(24) << 20) / 16;
        copy_kernel<<<prop.multiProcessorCount * 4, 512>>>(a, b, m, 2);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        copy_kernel<<<prop.multiProcessorCount * 4, 512>>>(a, b, m, 50);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        printf(", \"l2_copy_GBps\": %.1f", 50 * 2.0 * m * 16 / (ms * 1e-3) / 1e9);
        cudaFree(a);
        cudaFree(b);
    }
    // DSMEM: cluster 8, 128 KiB per CTA
    {
        const int elems = 8192;
        const int smem = elems * 16;
        double2 *o;
        CK(cudaMalloc(&o, 64));
        CK(cudaFuncSetAttribute(dsmem_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        int grid = 8 * 16;
        const int reps = 50;
        dsmem_kernel<8><<<grid, 512, smem>>>(o, elems, 2);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        dsmem_kernel<8><<<grid, 512, smem>>>(o, elems, reps);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        double bytes = double(grid) * reps * 7.0 * (elems / 8) * 16;
        printf(", \"dsmem_read_GBps_total\": %.1f, \"dsmem_read_GBps_per_cta\": %.2f", bytes / (ms * 1e-3) / 1e9,
               bytes / grid / (ms * 1e-3) / 1e9);
        int ncl = 0;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at;
        at.id = cudaLaunchAttributeClusterDimension;
        at.val.clusterDim.x = 8;
        at.val.clusterDim.y = 1;
        at.val.clusterDim.z = 1;
        cfg.attrs = &at;
        cfg.numAttrs = 1;
        cudaOccupancyMaxActiveClusters(&ncl, dsmem_kernel<8>, &cfg);
        printf(", \"max_active_clusters_8x128KiB\": %d", ncl);
        cudaFree(o);
    }

    // L2-resident read only: 32 MiB, full chip
    {
        size_t m = (size_t(32) << 20) / 16;
        double2 *a;
        CK(cudaMalloc(&a, m * 16));
        CK(cudaMemset(a, 0, m * 16));
        l2_read_kernel<<<prop.multiProcessorCount * 4, 512>>>(a, a, m, 2);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        l2_read_kernel<<<prop.multiProcessorCount * 4, 512>>>(a, a, m, 50);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        printf(", \"l2_read_GBps\": %.1f", 50.0 * m * 16 / (ms * 1e-3) / 1e9);
        cudaFree(a);
    }
    // DSMEM, full chip: ld-based and bulk-copy all-to-all
    for (int variant = 0; variant < 2; variant++) {
        const int chunk = 768;  // 12 KiB per peer chunk -> 96 KiB src + 96 KiB dst
        const int smem = variant ? 2 * 8 * chunk * 16 : 8192 * 16;
        double2 *o;
        CK(cudaMalloc(&o, 64));
        void *fn = variant ? (void *)dsmem_bulk_kernel<8> : (void *)dsmem_kernel<8>;
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        int ncl = 0;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(8 * 16);
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at;
        at.id = cudaLaunchAttributeClusterDimension;
        at.val.clusterDim.x = 8;
        at.val.clusterDim.y = 1;
        at.val.clusterDim.z = 1;
        cfg.attrs = &at;
        cfg.numAttrs = 1;
        CK(cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg));
        const int grid = 8 * ncl, reps = 200;
        double bytes;
        if (variant) {
            dsmem_bulk_kernel<8><<<grid, 512, smem>>>(o, chunk, 2);
            CK(cudaDeviceSynchronize());
            cudaEventRecord(e0);
            dsmem_bulk_kernel<8><<<grid, 512, smem>>>(o, chunk, reps);
            cudaEventRecord(e1);
            bytes = double(grid) * reps * 7.0 * chunk * 16;
        } else {
            dsmem_kernel<8><<<grid, 512, smem>>>(o, 8192, 2);
            CK(cudaDeviceSynchronize());
            cudaEventRecord(e0);
            dsmem_kernel<8><<<grid, 512, smem>>>(o, 8192, reps);
            cudaEventRecord(e1);
            bytes = double(grid) * reps * 7.0 * (8192 / 8) * 16;
        }
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        cudaEventElapsedTime(&ms, e0, e1);
        printf(", \"dsmem_%s_fullchip_clusters\": %d, \"dsmem_%s_GBps_total\": %.1f, \"dsmem_%s_B_per_clk_per_sm\": %.2f",
               variant ? "bulk" : "ld", ncl, variant ? "bulk" : "ld", bytes / (ms * 1e-3) / 1e9, variant ? "bulk" : "ld",
               bytes / grid / (ms * 1e-3) / 1.965e9);
        cudaFree(o);
    }
    // FMA rates
    {
        double *o;
        CK(cudaMalloc(&o, 64));
        int blocks = prop.multiProcessorCount * 8, iters = 1 << 16;
        fma64_kernel<<<blocks, 256>>>(o, 16);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        fma64_kernel<<<blocks, 256>>>(o, iters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        double f = double(blocks) * 256 * iters * 8 * 2;
        printf(", \"fp64_fma_TFLOPs\": %.2f", f / (ms * 1e-3) / 1e12);
        fma32_kernel<<<blocks, 256>>>((float *)o, 16);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        fma32_kernel<<<blocks, 256>>>((float *)o, iters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        printf(", \"fp32_fma_TFLOPs\": %.2f", f / (ms * 1e-3) / 1e12);
    }
    printf("}\n");
    return 0;
}

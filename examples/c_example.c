/* examples/c_example.c -- the boundary used from plain C (no Python, no torch):
 * include/moa_fft.h + libmoafft.so + the CUDA runtime for device memory.
 *
 *   host   : planner and ψ-layer introspection, the Ch.6 transpose vector,
 *            an argument error (runs without a GPU)
 *   gpu    : a 2^10-point complex128 impulse through moa_fft_plan / _exec
 *            (δ_0 -> all ones, P:1849-1852 with the forward sign) and a batched
 *            2^16 x 4 plan through moa_fft_exec_host (x -> F^-1 F x = x with
 *            MOA_FFT_INVERSE | MOA_FFT_NORMALIZE)
 *
 * build: gcc -std=c99 -Iinclude examples/c_example.c -Lpaper_0803_2386_b200 -lmoafft \
 *            -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,... -lm */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "moa_fft.h"

static int host_part(void) {
    int64_t rad[8];
    int nrad = 0;
    if (moa_plan_radices(1 << 16, 1024, MOA_C128, rad, 8, &nrad) != MOA_OK) return 1;
    printf("radices 2^16 x 1024 c128:");
    for (int i = 0; i < nrad; i++) printf(" %lld", (long long)rad[i]);
    printf("\n");
    moa_pass_desc_t d[MOA_MAX_PASSES];
    int np = 0;
    if (moa_psi_describe(1 << 16, 1024, MOA_C128, NULL, 0, d, MOA_MAX_PASSES, &np) != MOA_OK) return 2;
    for (int i = 0; i < np; i++)
        printf("pass %d: R=%d W=%d threads=%d in_kstr=%lld out_kstr=%lld twN=%lld\n", i, 1 << d[i].logR, d[i].W,
               d[i].threads, (long long)d[i].in_kstr, (long long)d[i].out_kstr, (long long)d[i].twN);
    /* qubits 0 and 2 of a 4-qubit register -> <0 2 1 3 4 6 5 7> */
    int32_t bits[2] = {0, 2}, t[8];
    if (moa_qgate_permutation(4, bits, 2, t) != MOA_OK) return 3;
    printf("qgate t:");
    for (int i = 0; i < 8; i++) printf(" %d", t[i]);
    printf("\n");
    moa_fft_plan_t p = NULL;
    moa_status_t st = moa_fft_plan(&p, 3, 1, MOA_C128, 1);
    printf("plan(n=3): status %d (%s)\n", (int)st, moa_fft_last_error());
    return st == MOA_EINVAL && p == NULL ? 0 : 4;
}

static int gpu_part(void) {
    const int64_t n = 1024;
    double *h = (double *)calloc((size_t)(2 * n), sizeof(double));
    void *dx = NULL, *dy = NULL;
    h[0] = 1.0; /* δ_0 */
    if (cudaMalloc(&dx, (size_t)n * 16) != cudaSuccess || cudaMalloc(&dy, (size_t)n * 16) != cudaSuccess) return 10;
    cudaMemcpy(dx, h, (size_t)n * 16, cudaMemcpyHostToDevice);
    moa_fft_plan_t p = NULL;
    if (moa_fft_plan(&p, n, 1, MOA_C128, 1) != MOA_OK) return 11;
    if (moa_fft_exec(p, dx, dy, NULL) != MOA_OK) return 12;
    cudaMemcpy(h, dy, (size_t)n * 16, cudaMemcpyDeviceToHost);
    double err = 0.0;
    for (int64_t k = 0; k < n; k++) err = fmax(err, fabs(h[2 * k] - 1.0) + fabs(h[2 * k + 1]));
    printf("impulse 2^10: max |X[k] - 1| = %.3e\n", err);
    moa_fft_destroy(p);
    cudaFree(dx);
    cudaFree(dy);
    free(h);
    if (err > 1e-12) return 13;

    const int64_t m = 1 << 16, rows = 4, cnt = m * rows;
    double *x = (double *)malloc((size_t)cnt * 16), *X = NULL, *y = NULL;
    if (cudaMallocHost((void **)&X, (size_t)cnt * 16) != cudaSuccess ||
        cudaMallocHost((void **)&y, (size_t)cnt * 16) != cudaSuccess)
        return 14;
    for (int64_t i = 0; i < 2 * cnt; i++) x[i] = X[i] = sin(0.001 * (double)i) + 0.25 * cos(0.37 * (double)i);
    moa_fft_plan_t f = NULL, b = NULL;
    if (moa_fft_plan(&f, m, rows, MOA_C128, 1) != MOA_OK) return 15;
    if (moa_fft_plan_ex(&b, m, rows, MOA_C128, 1, MOA_FFT_INVERSE | MOA_FFT_NORMALIZE) != MOA_OK) return 16;
    if (moa_fft_exec_host(f, X, y, NULL) != MOA_OK) return 17;  /* y = F x (host buffers) */
    if (moa_fft_exec_host(b, y, X, NULL) != MOA_OK) return 18;  /* X = F^-1 y / n */
    double num = 0.0, den = 0.0;
    for (int64_t i = 0; i < 2 * cnt; i++) {
        num += (X[i] - x[i]) * (X[i] - x[i]);
        den += x[i] * x[i];
    }
    printf("exec_host round trip 2^16 x 4: rel-L2 %.3e\n", sqrt(num / den));
    moa_fft_destroy(f);
    moa_fft_destroy(b);
    cudaFreeHost(X);
    cudaFreeHost(y);
    free(x);
    return sqrt(num / den) <= 1e-12 ? 0 : 19;
}

int main(int argc, char **argv) {
    int rc = host_part();
    if (rc) {
        fprintf(stderr, "host part failed (%d): %s\n", rc, moa_fft_last_error());
        return rc;
    }
    if (argc > 1 && strcmp(argv[1], "gpu") == 0) {
        rc = gpu_part();
        if (rc) fprintf(stderr, "gpu part failed (%d): %s\n", rc, moa_fft_last_error());
    }
    printf(rc ? "FAILED\n" : "OK\n");
    return rc;
}

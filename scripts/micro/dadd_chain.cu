// Microbenchmark: cycles per dependent fp64 add in an ordered fold from shared memory.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void fold(const double* g, double* out, long long* cyc, int reps) {
    __shared__ double ring[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) ring[i] = g[i];
    __syncthreads();
    if (threadIdx.x) return;
    double total = 0.0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r)
        for (int q = 0; q < 2048; q += 16) {
            double v[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) v[k] = ring[(q + k) & 2047];
#pragma unroll
            for (int k = 0; k < 16; ++k) total = __dadd_rn(total, v[k]);
        }
    long long t1 = clock64();
    *out = total;
    *cyc = t1 - t0;
}
__global__ void chain_reg(double a, double* out, long long* cyc, int n) {
    double t = 0.0, x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { t = __dadd_rn(t, x); x = __dadd_rn(x, 1e-300); }
    long long t1 = clock64();
    *out = t; *cyc = t1 - t0;
}
int main() {
    double *g, *o; long long* c;
    cudaMalloc(&g, 2048 * 8); cudaMalloc(&o, 8); cudaMalloc(&c, 8);
    cudaMemset(g, 0, 2048 * 8);
    long long h;
    for (int it = 0; it < 3; ++it) {
        fold<<<1, 256>>>(g, o, c, 32);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("smem fold: %.2f cycles/add\n", (double)h / (32 * 2048));
        chain_reg<<<1, 1>>>(1.0, o, c, 65536);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("register chain (2 adds/iter, independent x): %.2f cycles/iter\n", (double)h / 65536);
    }
    return 0;
}

// smem-fed 128-step fp64 chains: F2F cost on the critical path (sm_100a)
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void chain(const float* g, double* out, long long* cyc, int n) {
    __shared__ float xs[128], ys[128];
    __shared__ double xd[128], yd[128];
    xs[threadIdx.x] = g[threadIdx.x]; ys[threadIdx.x] = g[threadIdx.x + 128];
    xd[threadIdx.x] = g[threadIdx.x]; yd[threadIdx.x] = g[threadIdx.x + 128];
    __syncthreads();
    double s = 0.0, s2 = 0.0;
    long long t0 = clock64();
    for (int r = 0; r < n; ++r) {
#pragma unroll 16
        for (int j = 0; j < 128; ++j) {
            const int k = (j + threadIdx.x) & 127;
            if (MODE == 0) s = __fma_rn((double)xs[j], (double)ys[k], s);
            if (MODE == 1) s = __fma_rn(xd[j], (double)ys[k], s);
            if (MODE == 2) s = __fma_rn(xd[j], yd[k], s);
            if (MODE == 3) { const double y = (double)ys[k]; s = __fma_rn(xd[j], y, s); s2 = __fma_rn(xd[(j + 64) & 127], y, s2); }
        }
    }
    long long t1 = clock64();
    out[threadIdx.x] = s + s2;
    if (threadIdx.x == 0) cyc[MODE] = (t1 - t0) / n;
}
int main() {
    double* out; long long* cyc; float* g;
    cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 64); cudaMalloc(&g, 1024 * 4);
    cudaMemset(g, 0x3e, 1024 * 4);
    for (int rep = 0; rep < 2; ++rep) {
        chain<0><<<1, 128>>>(g, out, cyc, 10); chain<1><<<1, 128>>>(g, out, cyc, 10);
        chain<2><<<1, 128>>>(g, out, cyc, 10); chain<3><<<1, 128>>>(g, out, cyc, 10);
        cudaDeviceSynchronize();
    }
    long long h[4]; cudaMemcpy(h, cyc, 32, cudaMemcpyDeviceToHost);
    const char* nm[4] = {"float x float (2 F2F/step)", "double x float (1 F2F/step)", "double x double (0 F2F)", "2 chains sharing 1 F2F"};
    for (int m = 0; m < 4; ++m) printf("%-30s %5lld cycles / 128 steps = %.1f per step\n", nm[m], h[m], h[m] / 128.0);
}

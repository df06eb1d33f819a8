// Latency probes on sm_100a: dependent DFMA chain; DFMA chain fed by F2F of smem floats.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void chain_dfma(double* out, long long* cyc, int n) {
    double s = threadIdx.x * 1e-3;
    const double a = 1.0000001;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) s = __fma_rn(a, s, 1e-9);
    long long t1 = clock64();
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void chain_smem(const float* g, double* out, long long* cyc, int n) {
    __shared__ float xs[128], ys[128];
    xs[threadIdx.x] = g[threadIdx.x];
    ys[threadIdx.x] = g[threadIdx.x + 128];
    __syncthreads();
    double s = 0.0;
    long long t0 = clock64();
    for (int r = 0; r < n; ++r) {
#pragma unroll 8
        for (int j = 0; j < 128; ++j) s = __fma_rn((double)xs[j], (double)ys[(j + threadIdx.x) & 127], s);
    }
    long long t1 = clock64();
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[1] = (t1 - t0) / n;
}

int main() {
    double* out; long long* cyc; float* g;
    cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 64); cudaMalloc(&g, 1024 * 4);
    cudaMemset(g, 0x3e, 1024 * 4);
    chain_dfma<<<1, 32>>>(out, cyc, 1000);
    chain_smem<<<1, 128>>>(g, out, cyc, 10);
    cudaDeviceSynchronize();
    chain_dfma<<<1, 32>>>(out, cyc, 1000);
    chain_smem<<<1, 128>>>(g, out, cyc, 10);
    long long h[2];
    cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.1f cycles\n", h[0] / 1000.0);
    printf("128-step smem-fed DFMA chain: %lld cycles (%.1f per step)\n", h[1], h[1] / 128.0);
    return 0;
}

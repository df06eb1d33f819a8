// Latency microbenchmark (sm_100a): dependent-chain cycles per op for fp64 and
// shared / global loads, and DFMA throughput -- the numbers the latency-bound
// selection phases are designed against.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_dfma_lat(double* out, int n) {
    double a = threadIdx.x * 1e-3, b = 1.0000001;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a = __fma_rn(a, b, 1e-9);
    long long t1 = clock64();
    if (threadIdx.x == 0) printf("DFMA dependent: %.2f cycles\n", (double)(t1 - t0) / n);
    out[threadIdx.x] = a;
}
__global__ void k_dadd_lat(double* out, int n) {
    double a = threadIdx.x * 1e-3;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a = __dadd_rn(a, 1e-9);
    long long t1 = clock64();
    if (threadIdx.x == 0) printf("DADD dependent: %.2f cycles\n", (double)(t1 - t0) / n);
    out[threadIdx.x] = a;
}
__global__ void k_ffma_lat(float* out, int n) {
    float a = threadIdx.x * 1e-3f;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a = fmaf(a, 1.0000001f, 1e-9f);
    long long t1 = clock64();
    if (threadIdx.x == 0) printf("FFMA dependent: %.2f cycles\n", (double)(t1 - t0) / n);
    out[threadIdx.x] = a;
}
__global__ void k_lds_lat(uint32_t* out, int n) {
    __shared__ uint32_t s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i * 7 + 1) & 1023;
    __syncthreads();
    uint32_t x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = s[x];
    long long t1 = clock64();
    if (threadIdx.x == 0) printf("LDS dependent: %.2f cycles\n", (double)(t1 - t0) / n);
    out[threadIdx.x] = x;
}
__global__ void k_ldg_lat(const uint32_t* g, uint32_t* out, int n, const char* what) {
    uint32_t x = 0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __ldcg(g + x);
    long long t1 = clock64();
    if (threadIdx.x == 0) printf("LDG dependent (%s): %.1f cycles\n", what, (double)(t1 - t0) / n);
    out[threadIdx.x] = x;
}
__global__ void k_dfma_tput(double* out, int iters) {
    double s[8];
    for (int c = 0; c < 8; ++c) s[c] = threadIdx.x + c;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < 8; ++c) s[c] = __fma_rn(s[c], 1.0000001, 1e-9);
    double t = 0;
    for (int c = 0; c < 8; ++c) t += s[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
    double* od; float* of; uint32_t* ou;
    cudaMalloc(&od, 1 << 24); cudaMalloc(&of, 1 << 20); cudaMalloc(&ou, 1 << 20);
    k_dfma_lat<<<1, 32>>>(od, 4096); cudaDeviceSynchronize();
    k_dadd_lat<<<1, 32>>>(od, 4096); cudaDeviceSynchronize();
    k_ffma_lat<<<1, 32>>>(of, 4096); cudaDeviceSynchronize();
    k_lds_lat<<<1, 32>>>(ou, 4096); cudaDeviceSynchronize();
    // pointer chase: stride 64 KB within 1 MB (L2) and 4 GB (DRAM)
    const size_t big = (size_t)1 << 30;  // uint32 elements: 4 GB
    uint32_t* g; cudaMalloc(&g, big * 4);
    uint32_t* h = (uint32_t*)malloc(4096 * 4);
    for (size_t span : {(size_t)1 << 18, big}) {
        // chain of 4096 hops spread over `span` elements
        const size_t step = span / 4096;
        for (int i = 0; i < 4096; ++i) {
            const size_t at = (size_t)i * step, nxt = (size_t)((i * 1103 + 7) % 4096) * step;
            cudaMemcpy(g + at, &nxt, 4, cudaMemcpyHostToDevice);  // 32-bit index fits for span <= 2^32
        }
        k_ldg_lat<<<1, 32>>>(g, ou, 64, "warm-up"); cudaDeviceSynchronize();
        k_ldg_lat<<<1, 32>>>(g, ou, 2048, span == big ? "4 GB span, DRAM" : "1 MB span, L2"); cudaDeviceSynchronize();
    }
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    k_dfma_tput<<<148 * 8, 256>>>(od, 1024);
    cudaEventRecord(a); k_dfma_tput<<<148 * 8, 256>>>(od, 4096); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double ops = 148.0 * 8 * 256 * 4096 * 8;
    printf("DFMA throughput: %.1f G/s = %.1f per SM per clk @1.965GHz\n", ops / ms / 1e6, ops / ms / 1e6 / 148 / 1.965);
    return 0;
}

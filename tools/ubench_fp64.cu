// Microbenchmark: DFMA, F2F.F64.F32 and an integer float->double widening on sm_100a.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double widen_int(float f) {
    const uint32_t b = __float_as_uint(f);
    const uint32_t e = (b >> 23) & 0xffu;
    if (e == 0u || e == 0xffu) return (double)f;  // zero / denormal / inf / nan
    const unsigned long long hi = ((unsigned long long)(b & 0x80000000u) << 32) |
                                  ((unsigned long long)(e + 896u) << 52) |
                                  ((unsigned long long)(b & 0x7fffffu) << 29);
    return __longlong_as_double((long long)hi);
}

template <int MODE>
__global__ void k(const float* in, double* out, int iters) {
    const float* p = in + threadIdx.x;
    double s[8];
    for (int c = 0; c < 8; ++c) s[c] = 0.0;
    float f = p[0];
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            float x = __int_as_float(__float_as_int(f) + c + i);
            double dx;
            if (MODE == 0) dx = 1.0000001;          // DFMA only
            else if (MODE == 1) dx = (double)x;     // F2F + DFMA
            else dx = widen_int(x);                 // int widen + DFMA
            s[c] = __fma_rn(dx, 1.0000001, s[c]);
        }
    }
    double t = 0;
    for (int c = 0; c < 8; ++c) t += s[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
    float* in; double* out;
    cudaMalloc(&in, 4096 * 4); cudaMalloc(&out, 148 * 8 * 1024 * 8);
    cudaMemset(in, 0x3f, 4096 * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 4096, blocks = 148 * 8, threads = 256;
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (mode == 0) k<0><<<blocks, threads>>>(in, out, iters);
            if (mode == 1) k<1><<<blocks, threads>>>(in, out, iters);
            if (mode == 2) k<2><<<blocks, threads>>>(in, out, iters);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double ops = (double)blocks * threads * iters * 8;
            if (rep) printf("mode %d: %.1f G DFMA/s (%.2f per clk per SM @1.9GHz)\n", mode, ops / ms / 1e6, ops / ms / 1e6 / 148 / 1.9);
        }
    }
    return 0;
}

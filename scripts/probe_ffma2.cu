#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    unsigned long long ra = *reinterpret_cast<unsigned long long*>(&a), rb = *reinterpret_cast<unsigned long long*>(&b),
                       rc = *reinterpret_cast<unsigned long long*>(&c), rd;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
    return *reinterpret_cast<float2*>(&rd);
}
template <int MODE>
__global__ void k(float* out, float s, int iters) {
    unsigned x0 = threadIdx.x, x1 = x0 * 3u, x2 = x0 * 5u, x3 = x0 * 7u, x4 = x0 ^ 9u, x5 = x0 ^ 11u, x6 = x0 + 13u, x7 = x0 + 17u;
    // 8 independent accumulator chains (pairs) per thread
    float2 acc[8];
    for (int i = 0; i < 8; ++i) acc[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
    const float2 m = make_float2(s, s * 0.5f), a = make_float2(1e-7f, 2e-7f);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0 || MODE == 2) {
                acc[i].x = fmaf(acc[i].x, m.x, a.x);
                acc[i].y = fmaf(acc[i].y, m.y, a.y);
            } else {
                acc[i] = ffma2(acc[i], m, a);
            }
        }
        if (MODE >= 2) {  // 4 independent 3-input ALU ops (IADD3/LOP3) per iteration
            x0 ^= x4 + it; x1 ^= x5 + it;
        }
    }
    float r = 0;
    for (int i = 0; i < 8; ++i) r += acc[i].x + acc[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = r + (x0 ^ x1 ^ x2 ^ x3 ^ x4 ^ x5 ^ x6 ^ x7);
}
int main() {
    float* o; cudaMalloc(&o, 148 * 8 * 256 * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode = 0; mode < 4; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            const int iters = 20000;
            cudaEventRecord(a);
            if (mode == 0) k<0><<<148 * 8, 256>>>(o, 0.999f, iters);
            else if (mode == 1) k<1><<<148 * 8, 256>>>(o, 0.999f, iters);
            else if (mode == 2) k<2><<<148 * 8, 256>>>(o, 0.999f, iters);
            else k<3><<<148 * 8, 256>>>(o, 0.999f, iters);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double fmas = 148.0 * 8 * 256 * iters * 16;
            if (rep) printf("mode %d (%s%s): %.3f ms, %.1f TFMA/s\n", mode, mode & 1 ? "FFMA2" : "FFMA", mode >= 2 ? "+4 ALU" : "", ms, fmas / ms / 1e9);
        }
    }
    return 0;
}

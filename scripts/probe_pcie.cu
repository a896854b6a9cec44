// probe_pcie.cu -- host link probe: D2H/H2D copy-engine bandwidth vs SM stores
// into mapped pinned host memory (the zero-copy frame egress path).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 scripts/probe_pcie.cu -o build/probe_pcie
#include <cuda_runtime.h>

#include <cstdio>

#define CK(x)                                                                    \
    do {                                                                         \
        cudaError_t e = (x);                                                     \
        if (e != cudaSuccess) {                                                  \
            std::printf("%s failed: %s\n", #x, cudaGetErrorString(e));           \
            return 1;                                                            \
        }                                                                        \
    } while (0)

__global__ void store_kernel(const float4* __restrict__ src, float4* dst, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

int main() {
    const size_t bytes = 4608ull * 3456 * 12;
    float *d, *h;
    CK(cudaMalloc(&d, bytes));
    CK(cudaMemset(d, 1, bytes));
    CK(cudaHostAlloc(&h, bytes, cudaHostAllocPortable | cudaHostAllocMapped));
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a, s);
        cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        std::printf("D2H memcpy   %.1f MB  %.3f ms  %.1f GB/s\n", bytes / 1e6, ms, bytes / ms / 1e6);
        cudaEventRecord(a, s);
        cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        std::printf("H2D memcpy   %.1f MB  %.3f ms  %.1f GB/s\n", bytes / 1e6, ms, bytes / ms / 1e6);
        float* hd;
        CK(cudaHostGetDevicePointer(&hd, h, 0));
        for (int grid : {148, 592, 2368}) {
            cudaEventRecord(a, s);
            store_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<float4*>(d), reinterpret_cast<float4*>(hd), bytes / 16);
            cudaEventRecord(b, s);
            CK(cudaEventSynchronize(b));
            cudaEventElapsedTime(&ms, a, b);
            std::printf("SM->host st  grid %4d  %.3f ms  %.1f GB/s\n", grid, ms, bytes / ms / 1e6);
        }
    }
    // pageable destination for reference
    float* pg = static_cast<float*>(malloc(bytes));
    for (size_t i = 0; i < bytes / 4; i += 1024) pg[i] = 0;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a, s);
        cudaMemcpyAsync(pg, d, bytes, cudaMemcpyDeviceToHost, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        std::printf("D2H pageable %.3f ms  %.1f GB/s\n", ms, bytes / ms / 1e6);
    }
    return 0;
}

// probe_d2h.cu -- device->host (page-locked) bandwidth for a 191 MB frame:
// one copy-engine transfer, the frame split over 2 / 4 streams, and a copy
// engine half + SM stores through the mapping for the other half.
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

__global__ void st_mapped(const float4* __restrict__ src, float4* dst, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

int main() {
    const size_t bytes = 4608ull * 3456 * 12;
    float *d, *h, *hd;
    cudaMalloc(&d, bytes);
    cudaMemset(d, 1, bytes);
    cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
    cudaHostGetDevicePointer(&hd, h, 0);
    cudaStream_t st[4];
    for (auto& s : st) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char* name, int mode) {
        float best = 1e9f;
        for (int it = 0; it < 6; ++it) {
            cudaDeviceSynchronize();
            cudaEventRecord(a, st[0]);
            for (int k = 1; k < 4; ++k) cudaStreamWaitEvent(st[k], a, 0);
            if (mode == 1) {
                cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, st[0]);
            } else if (mode == 2 || mode == 4) {
                const size_t part = bytes / mode;
                for (int k = 0; k < mode; ++k)
                    cudaMemcpyAsync((char*)h + k * part, (char*)d + k * part, part, cudaMemcpyDeviceToHost, st[k]);
            } else if (mode == 5) {  // copy engine half + SM stores half
                const size_t half = bytes / 2;
                cudaMemcpyAsync(h, d, half, cudaMemcpyDeviceToHost, st[0]);
                st_mapped<<<148 * 4, 256, 0, st[1]>>>((const float4*)((char*)d + half), (float4*)((char*)hd + half),
                                                        half / 16);
            } else if (mode == 6) {  // copy engine 60 % + SM stores 40 %
                const size_t p0 = bytes / 16 * 10 / 16 * 16;
                cudaMemcpyAsync(h, d, p0, cudaMemcpyDeviceToHost, st[0]);
                st_mapped<<<148 * 4, 256, 0, st[1]>>>((const float4*)((char*)d + p0), (float4*)((char*)hd + p0),
                                                        (bytes - p0) / 16);
            } else if (mode == 7) {  // SM stores only
                st_mapped<<<148 * 4, 256, 0, st[0]>>>((const float4*)d, (float4*)hd, bytes / 16);
            }
            for (int k = 1; k < 4; ++k) {
                cudaEvent_t e;
                cudaEventCreate(&e);
                cudaEventRecord(e, st[k]);
                cudaStreamWaitEvent(st[0], e, 0);
                cudaEventDestroy(e);
            }
            cudaEventRecord(b, st[0]);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("%-28s %7.3f ms  %6.1f GB/s\n", name, best, bytes / (best * 1e-3) / 1e9);
    };
    run("1 copy", 1);
    run("2 streams", 2);
    run("4 streams", 4);
    run("copy 50% + SM stores 50%", 5);
    run("copy 62% + SM stores 38%", 6);
    run("SM stores only", 7);
    return 0;
}

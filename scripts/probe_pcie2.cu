// probe_pcie2.cu -- SM->mapped-host store bandwidth: float4 stores vs TMA bulk
// stores (cp.async.bulk smem -> global) of various sizes.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__global__ void st_float4(float4* dst, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = make_float4(1.f, 2.f, 3.f, 4.f);
}

template <int CHUNK>
__global__ void st_bulk(char* dst, size_t bytes) {
    __shared__ __align__(128) char buf[CHUNK];
    for (int i = threadIdx.x; i < CHUNK / 4; i += blockDim.x) reinterpret_cast<float*>(buf)[i] = 1.0f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
        for (size_t off = blockIdx.x * (size_t)CHUNK; off < bytes; off += (size_t)gridDim.x * CHUNK) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off), "r"(s), "r"(CHUNK)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

int main() {
    const size_t bytes = 4608ull * 3456 * 12;
    char* h;
    cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
    char* hd;
    cudaHostGetDevicePointer(&hd, h, 0);
    char* d;
    cudaMalloc(&d, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("copy engine D2H        %.3f ms %.1f GB/s\n", ms, bytes / ms / 1e6);
        cudaEventRecord(a);
        st_float4<<<592, 256>>>(reinterpret_cast<float4*>(hd), bytes / 16);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("float4 stores          %.3f ms %.1f GB/s\n", ms, bytes / ms / 1e6);
        cudaEventRecord(a);
        st_bulk<4096><<<296, 128>>>(hd, bytes);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("bulk 4 KB              %.3f ms %.1f GB/s (%s)\n", ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        cudaEventRecord(a);
        st_bulk<16384><<<296, 128>>>(hd, bytes);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("bulk 16 KB             %.3f ms %.1f GB/s (%s)\n", ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        cudaEventRecord(a);
        st_bulk<16384><<<148, 128>>>(hd, bytes);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("bulk 16 KB, 148 CTAs   %.3f ms %.1f GB/s (%s)\n", ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}

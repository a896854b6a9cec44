// cub_sort.cu -- bench-only comparator (not on the product path): the
// library radix sort the AdaGScale paper uses for the pair sort
// (PAPER.md:44), cub::DeviceRadixSort::SortPairs over the same 64-bit
// (tile << 32 | depth bits) keys and 32-bit values, timed with CUDA events.
// Built into scripts/_build/libcubsort.so by `make`; loaded by bench.py only.
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>

#include <cstdint>

extern "C" int cub_sort_pairs_u64(const uint64_t* keys_in, const uint32_t* vals_in, uint64_t* keys_out,
                                  uint32_t* vals_out, uint64_t n, int begin_bit, int end_bit, int iters,
                                  float* ms_per_sort, void* stream) {
    // `stream` is the caller's (torch's current) stream, so the sort is
    // ordered after the kernels that prepared keys_in / vals_in
    if (n > 0x7fffffffull) return 1;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    size_t temp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp, keys_in, keys_out, vals_in, vals_out, static_cast<int>(n),
                                    begin_bit, end_bit, st);
    void* d_temp = nullptr;
    if (cudaMalloc(&d_temp, temp) != cudaSuccess) return 3;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 2; ++i)  // warm-up
        cub::DeviceRadixSort::SortPairs(d_temp, temp, keys_in, keys_out, vals_in, vals_out, static_cast<int>(n),
                                        begin_bit, end_bit, st);
    cudaEventRecord(a, st);
    for (int i = 0; i < iters; ++i)
        cub::DeviceRadixSort::SortPairs(d_temp, temp, keys_in, keys_out, vals_in, vals_out, static_cast<int>(n),
                                        begin_bit, end_bit, st);
    cudaEventRecord(b, st);
    const cudaError_t e = cudaEventSynchronize(b);
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, a, b);
    *ms_per_sort = ms / static_cast<float>(iters > 0 ? iters : 1);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(d_temp);
    return e == cudaSuccess ? 0 : 4;
}

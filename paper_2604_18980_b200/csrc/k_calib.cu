// k_calib.cu -- device primitives of the calibration loop (next row f1).
//
//   reference: build_lut      calibrate.cpp:14-41 (max_t folded per depth bin)
//              psnr           analysis.cpp:14-25 (double squared-error sum)
//              TUpperLUT      lut.hpp:16-23 (bin_index)
#include "kernels.cuh"

namespace agsx {

// Fold the frame's per-Gaussian max_t into depth bins: order[j] / dkeys[j]
// (j < *m) are the depth-sorted splats with tiles (gid, depth bits); only
// splats that blended (max_t > 0) count.  max_t >= 0, so the float maximum is
// the unsigned maximum of the bit patterns.
__global__ void k_fold_max_t(const uint32_t* __restrict__ order, const uint32_t* __restrict__ dkeys,
                             const uint32_t* m_dev, const uint32_t* __restrict__ maxt, float dmin, float dmax,
                             int nbins, uint32_t* __restrict__ folded, uint32_t* __restrict__ observed) {
    const uint32_t m = *m_dev;
    const float w = (dmax - dmin) / static_cast<float>(nbins);
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
        const uint32_t mt = maxt[order[j]];
        if (mt == 0u) continue;  // never blended (max_t <= 0)
        int b = f2i_x86((__uint_as_float(dkeys[j]) - dmin) / w);
        if (b < 0) b = 0;
        if (b >= nbins) b = nbins - 1;
        atomicMax(&folded[b], mt);
        observed[b] = 1u;
    }
}

// Squared-error sum, stage 1: one double partial per block (fixed grid).
__global__ void __launch_bounds__(256)
k_sq_err_partial(const float* __restrict__ a, const float* __restrict__ b, uint64_t n, double* __restrict__ partial) {
    __shared__ double s[8];
    double acc = 0.0;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const double d = static_cast<double>(a[i]) - static_cast<double>(b[i]);
        acc += d * d;
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += s[w];
        partial[blockIdx.x] = t;
    }
}

// Stage 2: the partials in block order.
__global__ void k_sq_err_final(const double* __restrict__ partial, int n, double* __restrict__ out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < n; ++i) t += partial[i];
        *out = t;
    }
}

}  // namespace agsx

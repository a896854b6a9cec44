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
// (stride: 1 for the depth-sort arrays, 2 for the bucketed path's {gid,
// depth} list.)
__global__ void k_fold_max_t(const uint32_t* __restrict__ order, const uint32_t* __restrict__ inv,
                             const uint32_t* __restrict__ dkeys, int stride,
                             const uint32_t* m_dev, const uint32_t* __restrict__ maxt, float dmin, float dmax,
                             int nbins, uint32_t* __restrict__ folded, uint32_t* __restrict__ observed) {
    const uint32_t m = *m_dev;
    const float w = (dmax - dmin) / static_cast<float>(nbins);
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
        const uint32_t o = order[static_cast<uint64_t>(j) * stride];
        const uint32_t mt = maxt[inv ? inv[o] : o];
        if (mt == 0u) continue;  // never blended (max_t <= 0)
        int b = f2i_x86((__uint_as_float(dkeys[static_cast<uint64_t>(j) * stride]) - dmin) / w);
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

// PPM quantisation of an f32 HWC frame (write_image, gsio.cpp:265-281):
// clamp to [0, 1], then lround(v * 255) = floor(v * 255 + 0.5) (v * 255 is
// exact in double).  16 bytes per thread, one 16-byte store.
__global__ void __launch_bounds__(256)
k_quantize_u8(const float4* __restrict__ img, uint4* __restrict__ dst, uint64_t n16) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float4 v = img[4 * i + q];
            const float c[4] = {v.x, v.y, v.z, v.w};
            uint32_t word = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float x = sclamp(c[k], 0.0f, 1.0f);
                const uint32_t b = static_cast<uint32_t>(floor(static_cast<double>(x) * 255.0 + 0.5));
                word |= b << (8 * k);
            }
            w[q] = word;
        }
        dst[i] = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// Tail (n % 16 bytes) of the same quantisation.
__global__ void k_quantize_u8_tail(const float* __restrict__ img, uint8_t* __restrict__ dst, uint64_t lo, uint64_t n) {
    const uint64_t i = lo + threadIdx.x;
    if (i < n) dst[i] = static_cast<uint8_t>(floor(static_cast<double>(sclamp(img[i], 0.0f, 1.0f)) * 255.0 + 0.5));
}

}  // namespace agsx

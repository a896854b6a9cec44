// k_raster.cu -- K6: per-tile front-to-back alpha blending.
//
//   reference: alpha_at   rasterizer.hpp:44-50
//              raster_tile rasterizer.cpp:21-100
//              tile loop   rasterizer.cpp:137-147 (+ max_t merge :149-154)
//
// One 256-thread CTA per tile.  Splat records of the tile's sorted pair span
// are staged into shared memory in batches of 256 with cp.async (LDGSTS),
// double-buffered so the gather of batch b+1 overlaps the blending of batch
// b.  For 16x16 tiles each warp owns an 8x4 pixel block and skips, as a
// whole, every splat whose conservative alpha>=tau box misses the block;
// warps whose pixels are all saturated stop iterating, and the CTA stops at
// the first batch boundary where every pixel is saturated
// (__syncthreads_and), like `active == 0` in the reference.  Pixel
// arithmetic is the reference's, operation by operation, without FMA
// contraction; alpha uses either the glibc-exact expf or MUFU.EX2 with an
// exact re-evaluation inside a guard band around tau and the clamp.
// The tile is written as float4 rows of the HWC image.
#include "kernels.cuh"

namespace agsx {

namespace {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// glibc expf with the 2^(i/32) table read from shared memory (divergent
// table indices would serialise on the constant cache).
__device__ __forceinline__ float glibc_expf_smem(float x, const uint64_t* tab) {
    const uint32_t abstop = (__float_as_uint(x) >> 20) & 0x7ffu;
    if (abstop >= 0x42bu) {
        if (__float_as_uint(x) == 0xff800000u) return 0.0f;
        if (abstop >= 0x7f8u) return x + x;
        if (x > 0x1.62e42ep6f) return __int_as_float(0x7f800000);
        if (x < -0x1.9fe368p6f) return 0.0f;
    }
    const double xd = static_cast<double>(x);
    // glibc is built with FMA on x86-64 (IFUNC variant): r = fma(InvLn2N, x, -kd) etc.;
    // verified over all 2^32 floats against the host libm (tests/test_device_libm.py).
    double kd = fma(0x1.71547652b82fep+5, xd, 0x1.8p+52);
    const uint64_t ki = static_cast<uint64_t>(__double_as_longlong(kd));
    kd -= 0x1.8p+52;
    const double r = fma(0x1.71547652b82fep+5, xd, -kd);
    const uint64_t t = tab[ki % 32] + (ki << 47);
    const double s = __longlong_as_double(static_cast<long long>(t));
    const double zz = fma(0x1.c6af84b912394p-20, r, 0x1.ebfce50fac4f3p-13);
    const double r2 = r * r;
    double y = fma(0x1.62e42ff0c52d6p-6, r, 1.0);
    y = fma(zz, r2, y);
    y = y * s;
    return static_cast<float>(y);
}

__device__ __forceinline__ int lo16(uint32_t v) { return static_cast<int>(static_cast<int16_t>(v & 0xffffu)); }
__device__ __forceinline__ int hi16(uint32_t v) { return static_cast<int>(static_cast<int16_t>(v >> 16)); }

}  // namespace

template <int PPT, bool EXACT, bool MAXT>
__global__ void __launch_bounds__(256)
k_raster(FrameParams p, const uint2* __restrict__ ranges, const uint32_t* __restrict__ vals,
         const float4* __restrict__ P0, const float4* __restrict__ P1, const float4* __restrict__ P2,
         float* __restrict__ image, uint32_t* __restrict__ maxt, unsigned long long* __restrict__ pit) {
    constexpr int B = 256;
    __shared__ __align__(16) float4 sA[2][B];
    __shared__ __align__(16) float4 sB[2][B];
    __shared__ __align__(16) float4 sC[2][B];
    __shared__ uint32_t sG[MAXT ? 2 : 1][MAXT ? B : 1];
    __shared__ uint64_t sTab[32];
    __shared__ __align__(16) float sOut[PPT == 1 ? 16 * 16 * 3 : 4];
    __shared__ uint32_t sPit;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < 32) sTab[tid] = kExp2fTab[tid];
    if (tid == 0) sPit = 0;

    const int tile = blockIdx.x;
    const int ts = p.tile_size;
    const int tx = tile % p.tiles_x, ty = tile / p.tiles_x;
    const int x0 = tx * ts, y0 = ty * ts;
    const int w = imin(ts, p.W - x0), h = imin(ts, p.H - y0);
    const bool t16 = (ts == 16 && PPT == 1);

    // pixel ownership
    int lx[PPT], ly[PPT];
    bool has[PPT];
    float px[PPT], py[PPT], T[PPT], Cr[PPT], Cg[PPT], Cb[PPT];
    uint32_t death = 0;  // 1 + pair index that saturated my last pixel (P_it accounting)
    bool done = true;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
        if (t16) {
            lx[k] = (warp & 1) * 8 + (lane & 7);
            ly[k] = (warp >> 1) * 4 + (lane >> 3);
        } else {
            const int lp = tid + k * 256;
            lx[k] = lp % ts;
            ly[k] = lp / ts;
            if (lp >= ts * ts) ly[k] = ts;  // out of tile
        }
        has[k] = lx[k] < w && ly[k] < h;
        px[k] = static_cast<float>(x0 + lx[k]) + 0.5f;
        py[k] = static_cast<float>(y0 + ly[k]) + 0.5f;
        T[k] = 1.0f;
        Cr[k] = Cg[k] = Cb[k] = 0.0f;
        done = done && !has[k];
    }
    // conservative pixel box of this warp
    int bx0 = 1 << 30, bx1 = -(1 << 30), by0 = 1 << 30, by1 = -(1 << 30);
#pragma unroll
    for (int k = 0; k < PPT; ++k)
        if (has[k]) {
            bx0 = imin(bx0, x0 + lx[k]);
            bx1 = imax(bx1, x0 + lx[k]);
            by0 = imin(by0, y0 + ly[k]);
            by1 = imax(by1, y0 + ly[k]);
        }
    const int wx0 = __reduce_min_sync(0xffffffffu, bx0), wx1 = __reduce_max_sync(0xffffffffu, bx1);
    const int wy0 = __reduce_min_sync(0xffffffffu, by0), wy1 = __reduce_max_sync(0xffffffffu, by1);

    const uint2 rg = ranges[tile];
    const uint32_t start = rg.x, end = rg.y;
    const uint32_t n = end > start ? end - start : 0u;
    const uint32_t nb = (n + B - 1) / B;
    const float tau = p.tau, tfloor = p.tfloor, aclamp = p.aclamp;

    auto issue = [&](uint32_t b, int buf) {
        const uint32_t i = start + b * B + tid;
        if (i < end) {
            const uint32_t g = vals[i];
            cp_async16(&sA[buf][tid], &P0[g]);
            cp_async16(&sB[buf][tid], &P1[g]);
            cp_async16(&sC[buf][tid], &P2[g]);
            if (MAXT) sG[buf][tid] = g;
        }
        cp_async_commit();
    };

    if (nb > 0) issue(0, 0);
    for (uint32_t b = 0; b < nb; ++b) {
        const int buf = b & 1;
        if (b + 1 < nb) {
            issue(b + 1, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const int cnt = static_cast<int>(n - b * B < B ? n - b * B : B);
        if (!__all_sync(0xffffffffu, done)) {
            for (int j = 0; j < cnt; ++j) {
                const float4 sb = sB[buf][j];
                const float4 sc = sC[buf][j];
                const uint32_t bbx = __float_as_uint(sb.w), bby = __float_as_uint(sc.w);
                if (hi16(bbx) < wx0 || lo16(bbx) > wx1 || hi16(bby) < wy0 || lo16(bby) > wy1)
                    continue;  // warp-uniform: alpha < tau on every pixel of the warp
                const float4 sa = sA[buf][j];
                bool blended = false;
#pragma unroll
                for (int k = 0; k < PPT; ++k) {
                    if (!has[k] || T[k] < tfloor) continue;
                    // alpha_at (rasterizer.hpp:44-50), no contraction
                    const float dx = px[k] - sa.x, dy = py[k] - sa.y;
                    const float power = -0.5f * quad_form(sa.z, sa.w, sb.x, dx, dy);
                    if (power > 0.0f) continue;  // alpha = 0 < tau
                    if (power < sb.z) continue;  // provably alpha < tau
                    float a;
                    if (EXACT) {
                        a = sb.y * glibc_expf_smem(power, sTab);
                    } else {
                        a = sb.y * fast_exp(power);
                        if (fabsf(a - tau) <= 1e-5f * tau || fabsf(a - aclamp) <= 1e-5f)
                            a = sb.y * glibc_expf_smem(power, sTab);
                    }
                    a = a < aclamp ? a : aclamp;
                    if (a < tau) continue;
                    const float t_cur = T[k];
                    if (MAXT) atomicMax(&maxt[sG[buf][j]], __float_as_uint(t_cur));
                    const float wgt = a * t_cur;
                    Cr[k] += wgt * sc.x;
                    Cg[k] += wgt * sc.y;
                    Cb[k] += wgt * sc.z;
                    T[k] = t_cur * (1.0f - a);
                    if (T[k] < tfloor) death = b * B + j + 1;
                    blended = true;
                }
                if (__any_sync(0xffffffffu, blended)) {
                    bool all = true;
#pragma unroll
                    for (int k = 0; k < PPT; ++k) all = all && (!has[k] || T[k] < tfloor);
                    done = all;
                    if (__all_sync(0xffffffffu, done)) break;
                }
            }
        }
        if (__syncthreads_and(done)) break;
    }
    cp_async_wait<0>();

    // P_it of this tile: pairs the reference iterates before `active == 0`
    // (rasterizer.cpp:55-56): n if any pixel stays unsaturated.
    {
        const uint32_t mine = done ? death : n;
        const uint32_t wmax = __reduce_max_sync(0xffffffffu, mine);
        if (lane == 0 && wmax) atomicMax(&sPit, wmax);
        __syncthreads();
        if (tid == 0 && pit && sPit) atomicAdd(pit, static_cast<unsigned long long>(sPit));
    }

    // epilogue: C + T * background, clamped (rasterizer.cpp:89-99)
    if (t16) {
        if (has[0]) {
            float* o = &sOut[(ly[0] * 16 + lx[0]) * 3];
            o[0] = sclamp(Cr[0] + T[0] * p.bg[0], 0.0f, 1.0f);
            o[1] = sclamp(Cg[0] + T[0] * p.bg[1], 0.0f, 1.0f);
            o[2] = sclamp(Cb[0] + T[0] * p.bg[2], 0.0f, 1.0f);
        }
        __syncthreads();
        if (w == 16 && (p.W & 3) == 0) {
            // 16 px * 3 ch = 12 float4 per row
            if (tid < 12 * h) {
                const int row = tid / 12, col = tid % 12;
                float4* dst = reinterpret_cast<float4*>(
                    image + (static_cast<size_t>(y0 + row) * p.W + x0) * 3);
                dst[col] = reinterpret_cast<const float4*>(sOut)[row * 12 + col];
            }
        } else {
            for (int i = tid; i < w * h * 3; i += 256) {
                const int c = i % 3, pix = i / 3, row = pix / w, col = pix % w;
                image[(static_cast<size_t>(y0 + row) * p.W + x0 + col) * 3 + c] =
                    sOut[(row * 16 + col) * 3 + c];
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < PPT; ++k)
            if (has[k]) {
                float* o = image + (static_cast<size_t>(y0 + ly[k]) * p.W + x0 + lx[k]) * 3;
                o[0] = sclamp(Cr[k] + T[k] * p.bg[0], 0.0f, 1.0f);
                o[1] = sclamp(Cg[k] + T[k] * p.bg[1], 0.0f, 1.0f);
                o[2] = sclamp(Cb[k] + T[k] * p.bg[2], 0.0f, 1.0f);
            }
    }
}

template <int PPT>
static void launch_ppt(bool exact, bool maxt, int grid, cudaStream_t st, const FrameParams& p,
                       const uint2* ranges, const uint32_t* vals, const float4* P0, const float4* P1,
                       const float4* P2, float* image, uint32_t* mt, unsigned long long* pit) {
    if (exact) {
        if (maxt) k_raster<PPT, true, true><<<grid, 256, 0, st>>>(p, ranges, vals, P0, P1, P2, image, mt, pit);
        else k_raster<PPT, true, false><<<grid, 256, 0, st>>>(p, ranges, vals, P0, P1, P2, image, mt, pit);
    } else {
        if (maxt) k_raster<PPT, false, true><<<grid, 256, 0, st>>>(p, ranges, vals, P0, P1, P2, image, mt, pit);
        else k_raster<PPT, false, false><<<grid, 256, 0, st>>>(p, ranges, vals, P0, P1, P2, image, mt, pit);
    }
}

void launch_raster_kernel(int ppt, bool exact, bool maxt, int grid, cudaStream_t st, const FrameParams& p,
                          const uint2* ranges, const uint32_t* vals, const float4* P0, const float4* P1,
                          const float4* P2, float* image, uint32_t* maxt_buf, unsigned long long* pit) {
    if (ppt == 1) launch_ppt<1>(exact, maxt, grid, st, p, ranges, vals, P0, P1, P2, image, maxt_buf, pit);
    else if (ppt == 4) launch_ppt<4>(exact, maxt, grid, st, p, ranges, vals, P0, P1, P2, image, maxt_buf, pit);
    else launch_ppt<16>(exact, maxt, grid, st, p, ranges, vals, P0, P1, P2, image, maxt_buf, pit);
}

}  // namespace agsx

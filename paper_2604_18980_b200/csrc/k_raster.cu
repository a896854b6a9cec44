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

// Splat extents packed as half2 (rounded up) in P2.w.
__device__ __forceinline__ float2 unpack_extent(float w) {
    const uint32_t v = __float_as_uint(w);
    return make_float2(__half2float(__ushort_as_half(static_cast<unsigned short>(v & 0xffffu))),
                       __half2float(__ushort_as_half(static_cast<unsigned short>(v >> 16))));
}

// Can the splat reach alpha >= tau at a pixel centre of the box?
__device__ __forceinline__ bool meets_box(float mx, float my, float2 e, float cx0, float cx1, float cy0, float cy1) {
    return mx + e.x >= cx0 && mx - e.x <= cx1 && my + e.y >= cy0 && my - e.y <= cy1;
}

// The reference's alpha_at (rasterizer.hpp:44-50) from q = d^T inv d
// (power = -0.5 q exactly); returns a value < tau when the splat does not
// blend.
__device__ __forceinline__ float exact_alpha(float q, float opacity, float aclamp, const uint64_t* tab) {
    const float power = -0.5f * q;
    if (power > 0.0f) return 0.0f;
    const float a = opacity * glibc_expf_smem(power, tab);
    return a < aclamp ? a : aclamp;
}

}  // namespace


// 16x16 tiles, PPT pixels per thread in a vertical column (PPT in {2,4}).
// Warp w of the 16*16/PPT/32 warps owns rows [w*R, (w+1)*R), R = 2*PPT:
// lane l -> column l%16, rows w*R + (l/16)*PPT + k.  Each warp streams the
// tile's sorted splat list on its own, 32 records per step (prefetched one
// step ahead), keeps the splats whose conservative extent meets its rows
// (ballot) and blends them in order; no block barrier until the store.
//
// Per pixel the alpha >= tau decision is taken on q = d^T inv d, the exact
// float value of the reference (power = -0.5 q exactly), against per-splat
// thresholds with a 1e-4 relative margin (blend_cull_data):
//   q > qcut        -> alpha < tau: skip
//   0 <= q < qsafe  -> alpha >= tau: alpha = opacity * 2^(-q log2(e)/2)
//   otherwise (margin band, q < 0, NaN, opacity >= clamp): deferred to a
//   warp-uniform block that evaluates the reference expression with the
//   glibc-exact expf.  EXACT routes every non-skipped pixel there.
template <int PPT, bool EXACT, bool MAXT>
__global__ void __launch_bounds__(256 / PPT)
k_raster16(FrameParams p, const uint2* __restrict__ ranges, const uint32_t* __restrict__ vals,
           const float4* __restrict__ P0, const float4* __restrict__ P1, const float4* __restrict__ P2,
           float* __restrict__ image, uint32_t* __restrict__ maxt, unsigned long long* __restrict__ pit) {
    constexpr int NW = 8 / PPT;  // warps per tile
    constexpr int R = 2 * PPT;   // rows per warp
    __shared__ __align__(16) float4 sA[NW][32];
    __shared__ __align__(16) float4 sB[NW][32];
    __shared__ __align__(16) float4 sC[NW][32];
    __shared__ uint32_t sG[MAXT ? NW : 1][32];
    __shared__ uint64_t sTab[32];
    __shared__ __align__(16) float sOut[16 * 16 * 3];
    __shared__ uint32_t sPit;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < 32) sTab[tid] = kExp2fTab[tid];
    if (tid == 0) sPit = 0;
    __syncthreads();

    const int tile = blockIdx.x;
    const int tx = tile % p.tiles_x, ty = tile / p.tiles_x;
    const int x0 = tx * 16, y0 = ty * 16;
    const int w = imin(16, p.W - x0), h = imin(16, p.H - y0);
    const int lx = lane & 15, ly0 = warp * R + (lane >> 4) * PPT;
    const float px = static_cast<float>(x0 + lx) + 0.5f;
    float py[PPT], T[PPT], Cr[PPT], Cg[PPT], Cb[PPT];
    uint32_t live = 0;  // bit k: pixel k exists and is not saturated
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
        py[k] = static_cast<float>(y0 + ly0 + k) + 0.5f;
        const bool exists = lx < w && ly0 + k < h;
        T[k] = exists ? 1.0f : 0.0f;  // pixels outside the image count as saturated
        Cr[k] = Cg[k] = Cb[k] = 0.0f;
        if (exists) live |= 1u << k;
    }
    uint32_t death = 0;
    const bool warp_empty = warp * R >= h;
    // pixel-centre box of the warp's pixels inside the image
    const float cx0 = x0 + 0.5f, cx1 = x0 + w - 0.5f;
    const float cy0 = y0 + warp * R + 0.5f, cy1 = y0 + imin(warp * R + R, h) - 0.5f;
    const float tau = p.tau, tfloor = p.tfloor, aclamp = p.aclamp;
    const float c_ex2 = -0.5f * 1.4426950408889634f;

    const uint2 rg = ranges[tile];
    const uint32_t start = rg.x, end = rg.y > rg.x ? rg.y : rg.x;
    float4 nA = make_float4(0, 0, 0, 0), nB = nA, nC = nA;
    uint32_t nG = 0;
    auto fetch = [&](uint32_t base) {
        const uint32_t i = base + lane;
        if (i < end) {
            nG = __ldg(&vals[i]);
            nA = __ldg(&P0[nG]);
            nB = __ldg(&P1[nG]);
            nC = __ldg(&P2[nG]);
        }
    };
    bool all_done = warp_empty || !__any_sync(0xffffffffu, live != 0);
    if (!all_done) fetch(start);
    for (uint32_t base = start; base < end && !all_done; base += 32) {
        const float4 cA = nA, cB = nB, cC = nC;
        const uint32_t cG = nG;
        if (base + 32 < end) fetch(base + 32);
        const bool rel = base + lane < end && meets_box(cA.x, cA.y, unpack_extent(cC.w), cx0, cx1, cy0, cy1);
        uint32_t m = __ballot_sync(0xffffffffu, rel);
        if (!m) continue;
        sA[warp][lane] = cA;
        sB[warp][lane] = cB;
        sC[warp][lane] = cC;
        if (MAXT) sG[warp][lane] = cG;
        __syncwarp();
        while (m) {
            const int j = __ffs(m) - 1;
            m &= m - 1;
            const float4 sa = sA[warp][j];  // mx, my, inv.xx, 2*inv.xy
            const float4 sb = sB[warp][j];  // inv.yy, opacity, qcut, qsafe
            const float4 sc = sC[warp][j];  // r, g, b, extent
            // column-shared terms of ((xx*dx)*dx + ((2xy)*dx)*dy) + (yy*dy)*dy
            const float dx = px - sa.x;
            const float t1 = sa.z * dx * dx;
            const float t2 = sa.w * dx;
            if constexpr (!EXACT && !MAXT) {
                // Fast path, branch-free per pixel: q by FMA (its error is
                // folded into qcut/qsafe), alpha = 2^(q c + log2 opacity)
                // on MUFU.EX2, blended with FMAs; a = 0 for pixels that are
                // saturated, outside the image, or not provably >= tau.
                const uint32_t qsafe = __float_as_uint(sb.w);
                const float qcut = sb.z;
                const float l2op = fast_log2(sb.y);
                uint32_t need = 0;
#pragma unroll
                for (int k = 0; k < PPT; ++k) {
                    const float dy = py[k] - sa.y;
                    const float q = __fmaf_rn(__fmaf_rn(sb.x, dy, t2), dy, t1);
                    const bool on = T[k] >= tfloor;
                    const bool fast = on && __float_as_uint(q) < qsafe;
                    const float e = fminf(fast_exp2(__fmaf_rn(q, c_ex2, l2op)), aclamp);
                    const float a = fast ? e : 0.0f;
                    const float wgt = a * T[k];
                    Cr[k] = __fmaf_rn(wgt, sc.x, Cr[k]);
                    Cg[k] = __fmaf_rn(wgt, sc.y, Cg[k]);
                    Cb[k] = __fmaf_rn(wgt, sc.z, Cb[k]);
                    T[k] = __fmaf_rn(-a, T[k], T[k]);
                    if (on && !fast && !(q > qcut)) need |= 1u << k;
                }
                if (__any_sync(0xffffffffu, need != 0)) {
#pragma unroll
                    for (int k = 0; k < PPT; ++k) {
                        if (!((need >> k) & 1u)) continue;
                        const float dy = py[k] - sa.y;
                        const float qr = (t1 + t2 * dy) + sb.x * dy * dy;  // reference order
                        const float a = exact_alpha(qr, sb.y, aclamp, sTab);
                        if (a < tau) continue;
                        const float t_cur = T[k];
                        const float wgt = a * t_cur;
                        Cr[k] += wgt * sc.x;
                        Cg[k] += wgt * sc.y;
                        Cb[k] += wgt * sc.z;
                        T[k] = t_cur * (1.0f - a);
                    }
                }
                bool dead = true;
#pragma unroll
                for (int k = 0; k < PPT; ++k) dead = dead && !(T[k] >= tfloor);
                if (__all_sync(0xffffffffu, dead)) {
                    death = base - start + j + 1;
                    live = 0;
                    all_done = true;
                    break;
                }
            } else {
            const uint32_t qcut = __float_as_uint(sb.z);
            const uint32_t qsafe = EXACT ? 0u : __float_as_uint(sb.w);
            float q[PPT];
            uint32_t need = 0;
            bool newly_done = false;
            auto blend = [&](int k, float a) {
                const float t_cur = T[k];
                if (MAXT) atomicMax(&maxt[sG[warp][j]], __float_as_uint(t_cur));
                const float wgt = a * t_cur;
                Cr[k] += wgt * sc.x;
                Cg[k] += wgt * sc.y;
                Cb[k] += wgt * sc.z;
                T[k] = t_cur * (1.0f - a);
                if (T[k] < tfloor) {
                    live &= ~(1u << k);
                    newly_done = true;
                    death = base - start + j + 1;
                }
            };
#pragma unroll
            for (int k = 0; k < PPT; ++k) {
                const float dy = py[k] - sa.y;
                q[k] = (t1 + t2 * dy) + sb.x * dy * dy;
                const uint32_t qb = __float_as_uint(q[k]);
                const bool on = (live >> k) & 1u;
                if (on && qb < qsafe) {
                    blend(k, fminf(sb.y * fast_exp2(q[k] * c_ex2), aclamp));
                } else if (on && !(qb > qcut && qb <= 0x7f800000u)) {
                    need |= 1u << k;
                }
            }
            if (__any_sync(0xffffffffu, need != 0)) {
#pragma unroll
                for (int k = 0; k < PPT; ++k) {
                    if (!((need >> k) & 1u)) continue;
                    const float a = exact_alpha(q[k], sb.y, aclamp, sTab);
                    if (!(a < tau)) blend(k, a);
                }
            }
            if (__any_sync(0xffffffffu, newly_done) && !__any_sync(0xffffffffu, live != 0)) {
                all_done = true;
                break;
            }
            }
        }
        __syncwarp();
    }

    // P_it of this tile (rasterizer.cpp:55-56): n if any pixel stays unsaturated
    {
        const uint32_t n = end - start;
        const uint32_t wmax = __reduce_max_sync(0xffffffffu, live ? n : death);
        if (lane == 0 && wmax) atomicMax(&sPit, wmax);
    }
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
        if (lx < w && ly0 + k < h) {
            float* o = &sOut[((ly0 + k) * 16 + lx) * 3];
            o[0] = sclamp(Cr[k] + T[k] * p.bg[0], 0.0f, 1.0f);
            o[1] = sclamp(Cg[k] + T[k] * p.bg[1], 0.0f, 1.0f);
            o[2] = sclamp(Cb[k] + T[k] * p.bg[2], 0.0f, 1.0f);
        }
    }
    __syncthreads();
    if (tid == 0 && pit && sPit) atomicAdd(pit, static_cast<unsigned long long>(sPit));
    constexpr int NT = 256 / PPT;
    if (w == 16 && (p.W & 3) == 0) {
        for (int i = tid; i < 12 * h; i += NT) {
            const int row = i / 12, col = i % 12;
            float4* dst = reinterpret_cast<float4*>(image + (static_cast<size_t>(y0 + row) * p.W + x0) * 3);
            __stcs(&dst[col], reinterpret_cast<const float4*>(sOut)[row * 12 + col]);
        }
    } else {
        for (int i = tid; i < w * h * 3; i += NT) {
            const int c = i % 3, pix = i / 3, row = pix / w, col = pix % w;
            image[(static_cast<size_t>(y0 + row) * p.W + x0 + col) * 3 + c] = sOut[(row * 16 + col) * 3 + c];
        }
    }
}

// Any tile size in [1, 64]: 256 threads, pixel k of thread t is tile pixel
// t + 256 k (row-major).  Batches of 256 splat records are staged with
// cp.async (double-buffered); each warp skips splats whose extent misses
// all of its pixels.  Same per-pixel arithmetic as k_raster16.
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
    __shared__ uint32_t sPit;

    const int tid = threadIdx.x, lane = tid & 31;
    if (tid < 32) sTab[tid] = kExp2fTab[tid];
    if (tid == 0) sPit = 0;

    const int tile = blockIdx.x;
    const int ts = p.tile_size;
    const int tx = tile % p.tiles_x, ty = tile / p.tiles_x;
    const int x0 = tx * ts, y0 = ty * ts;
    const int w = imin(ts, p.W - x0), h = imin(ts, p.H - y0);

    int lx[PPT], ly[PPT];
    float px[PPT], py[PPT], T[PPT], Cr[PPT], Cg[PPT], Cb[PPT];
    uint32_t live = 0, death = 0;
    float bx0 = 1e30f, bx1 = -1e30f, by0 = 1e30f, by1 = -1e30f;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
        const int lp = tid + k * 256;
        lx[k] = lp % ts;
        ly[k] = lp < ts * ts ? lp / ts : ts;
        px[k] = static_cast<float>(x0 + lx[k]) + 0.5f;
        py[k] = static_cast<float>(y0 + ly[k]) + 0.5f;
        T[k] = 1.0f;
        Cr[k] = Cg[k] = Cb[k] = 0.0f;
        if (lx[k] < w && ly[k] < h) {
            live |= 1u << k;
            bx0 = fminf(bx0, px[k]);
            bx1 = fmaxf(bx1, px[k]);
            by0 = fminf(by0, py[k]);
            by1 = fmaxf(by1, py[k]);
        }
    }
    // warp pixel-centre box (float min/max via shuffles)
    for (int o = 16; o > 0; o >>= 1) {
        bx0 = fminf(bx0, __shfl_xor_sync(0xffffffffu, bx0, o));
        bx1 = fmaxf(bx1, __shfl_xor_sync(0xffffffffu, bx1, o));
        by0 = fminf(by0, __shfl_xor_sync(0xffffffffu, by0, o));
        by1 = fmaxf(by1, __shfl_xor_sync(0xffffffffu, by1, o));
    }

    const uint2 rg = ranges[tile];
    const uint32_t start = rg.x, end = rg.y;
    const uint32_t n = end > start ? end - start : 0u;
    const uint32_t nb = (n + B - 1) / B;
    const float tau = p.tau, tfloor = p.tfloor, aclamp = p.aclamp;
    const float c_ex2 = -0.5f * 1.4426950408889634f;

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
        if (__any_sync(0xffffffffu, live != 0)) {
            for (int j = 0; j < cnt; ++j) {
                const float4 sc = sC[buf][j];
                const float4 sa = sA[buf][j];
                if (!meets_box(sa.x, sa.y, unpack_extent(sc.w), bx0, bx1, by0, by1)) continue;
                const float4 sb = sB[buf][j];
                const uint32_t qcut = __float_as_uint(sb.z);
                const uint32_t qsafe = EXACT ? 0u : __float_as_uint(sb.w);
                bool newly_done = false;
#pragma unroll
                for (int k = 0; k < PPT; ++k) {
                    if (!((live >> k) & 1u)) continue;
                    const float dx = px[k] - sa.x, dy = py[k] - sa.y;
                    const float q = (sa.z * dx * dx + sa.w * dx * dy) + sb.x * dy * dy;
                    const uint32_t qb = __float_as_uint(q);
                    float a;
                    if (qb < qsafe) {
                        a = fminf(sb.y * fast_exp2(q * c_ex2), aclamp);
                    } else {
                        if (qb > qcut && qb <= 0x7f800000u) continue;
                        a = exact_alpha(q, sb.y, aclamp, sTab);
                        if (a < tau) continue;
                    }
                    const float t_cur = T[k];
                    if (MAXT) atomicMax(&maxt[sG[buf][j]], __float_as_uint(t_cur));
                    const float wgt = a * t_cur;
                    Cr[k] += wgt * sc.x;
                    Cg[k] += wgt * sc.y;
                    Cb[k] += wgt * sc.z;
                    T[k] = t_cur * (1.0f - a);
                    if (T[k] < tfloor) {
                        live &= ~(1u << k);
                        newly_done = true;
                        death = b * B + j + 1;
                    }
                }
                if (__any_sync(0xffffffffu, newly_done) && !__any_sync(0xffffffffu, live != 0)) break;
            }
        }
        if (__syncthreads_and(live == 0)) break;
    }
    cp_async_wait<0>();
    {
        const uint32_t wmax = __reduce_max_sync(0xffffffffu, live ? n : death);
        if (lane == 0 && wmax) atomicMax(&sPit, wmax);
        __syncthreads();
        if (tid == 0 && pit && sPit) atomicAdd(pit, static_cast<unsigned long long>(sPit));
    }
#pragma unroll
    for (int k = 0; k < PPT; ++k)
        if (lx[k] < w && ly[k] < h) {
            float* o = image + (static_cast<size_t>(y0 + ly[k]) * p.W + x0 + lx[k]) * 3;
            o[0] = sclamp(Cr[k] + T[k] * p.bg[0], 0.0f, 1.0f);
            o[1] = sclamp(Cg[k] + T[k] * p.bg[1], 0.0f, 1.0f);
            o[2] = sclamp(Cb[k] + T[k] * p.bg[2], 0.0f, 1.0f);
        }
}

template <int Q>
static void launch16(bool exact, bool maxt, int grid, cudaStream_t st, const FrameParams& p, const uint2* ranges,
                     const uint32_t* vals, const float4* P0, const float4* P1, const float4* P2, float* image,
                     uint32_t* mt, unsigned long long* pit) {
    if (exact) {
        if (maxt) k_raster16<Q, true, true><<<grid, 256 / Q, 0, st>>>(p, ranges, vals, P0, P1, P2, image, mt, pit);
        else k_raster16<Q, true, false><<<grid, 256 / Q, 0, st>>>(p, ranges, vals, P0, P1, P2, image, mt, pit);
    } else {
        if (maxt) k_raster16<Q, false, true><<<grid, 256 / Q, 0, st>>>(p, ranges, vals, P0, P1, P2, image, mt, pit);
        else k_raster16<Q, false, false><<<grid, 256 / Q, 0, st>>>(p, ranges, vals, P0, P1, P2, image, mt, pit);
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
    if (p.tile_size == 16) {
        if (p.raster_ppt == 8)
            launch16<8>(exact, maxt, grid, st, p, ranges, vals, P0, P1, P2, image, maxt_buf, pit);
        else if (p.raster_ppt == 4)
            launch16<4>(exact, maxt, grid, st, p, ranges, vals, P0, P1, P2, image, maxt_buf, pit);
        else
            launch16<2>(exact, maxt, grid, st, p, ranges, vals, P0, P1, P2, image, maxt_buf, pit);
        return;
    }
    if (ppt == 1) launch_ppt<1>(exact, maxt, grid, st, p, ranges, vals, P0, P1, P2, image, maxt_buf, pit);
    else if (ppt == 4) launch_ppt<4>(exact, maxt, grid, st, p, ranges, vals, P0, P1, P2, image, maxt_buf, pit);
    else launch_ppt<16>(exact, maxt, grid, st, p, ranges, vals, P0, P1, P2, image, maxt_buf, pit);
}

}  // namespace agsx

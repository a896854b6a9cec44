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
#include <cstdlib>

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
    griddep_wait();
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
                const float qsafe = sb.w;
                const float qcut = sb.z;
                const float l2op = fast_log2(sb.y);
                uint32_t need = 0;
#pragma unroll
                for (int k = 0; k < PPT; ++k) {
                    const float dy = py[k] - sa.y;
                    const float q = __fmaf_rn(__fmaf_rn(sb.x, dy, t2), dy, t1);
                    const bool on = T[k] >= tfloor;
                    const bool fast = on && q < qsafe;
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
            const float qsafe = EXACT ? -__int_as_float(0x7f800000) : sb.w;
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
                if (on && q[k] >= 0.0f && q[k] < qsafe) {
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

// Default (fast-alpha) rasterizer for 16x16 tiles: warp-persistent.  The
// work unit is half a tile (16 columns x 8 rows); warps pull units from a
// global counter, so load balances at warp granularity and no CTA waits on
// another warp.  Lane l owns column l%16 and rows 4(l/16)..+3 of its unit.
// Per 32-record step of the tile's sorted span, each lane tests one splat
// against the box of the unit's live pixel centres (extent box) and the
// warp blends the survivors in order, staged compacted in shared memory:
//   the exponent x = c q + log2 opacity of alpha = 2^x in unit-centred form
//   (2 FMA per pixel; its error bound widens the thresholds), fast pixels
//   (x > xs) blend alpha = min(2^x, clamp) with FMAs; pixels in the margin
//   band (xc <= x <= xs) are re-evaluated exactly (glibc expf, reference
//   order) -- every alpha >= tau decision is the reference's.
// P_it per tile (pairs iterated before saturation, rasterizer.cpp:55-56) is
// the max over its two units, combined through a per-tile 64-bit word.
// CLAMP = false when no splat's opacity reaches the clamp (FrameParams::
// clamp_free, from the scene's maximum opacity): alpha <= opacity < clamp, so
// the fast path drops the clamp test (4 predicated FMNMX issue slots per
// iteration otherwise); the exact path always applies alpha_at's clamp.
template <bool STATS, bool CLAMP>
__global__ void __launch_bounds__(256, 3)
k_raster_units(FrameParams p, const uint2* __restrict__ ranges, const uint32_t* __restrict__ vals,
               const float4* __restrict__ P0, const float4* __restrict__ P1, const float4* __restrict__ P2,
               float* __restrict__ image, uint32_t* unit_ctr, unsigned long long* __restrict__ tile_pit,
               unsigned long long* __restrict__ pit, unsigned long long* dbg, uint32_t* band_done, int band_rows,
               uint8_t* __restrict__ img_u8) {
    griddep_wait();
    // STATS: dbg[0] += splat iterations per warp, dbg[1] += live pixel
    // evaluations, dbg[2] += fast blends, dbg[3] += exact re-evaluations
    unsigned long long st_it = 0, st_on = 0, st_fast = 0, st_need = 0, st_lo32 = 0, st_lo64 = 0, st_empty = 0,
                       st_dead = 0;
    constexpr int PPT = 4;
    constexpr int NWB = 8;  // warps per block
    // staged splat j of warp w: sS[w][j][0..2] = the unit-centred exponent
    // form and blend data read every iteration, sS[w][j][3..4] = {P0, iyy,
    // opacity} (unscaled) for the exact path only
    __shared__ __align__(16) float4 sS[NWB][32][5];
    __shared__ uint64_t sTab[32];
    __shared__ __align__(16) float sOut[NWB][8 * 16 * 3];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < 32) sTab[tid] = kExp2fTab[tid];
    __syncthreads();

    const uint32_t units = p.unit_hi ? p.unit_hi : 2u * static_cast<uint32_t>(p.tiles_x * p.tiles_y);
    const float tau = p.tau, tfloor = p.tfloor, aclamp = p.aclamp;
    const int lx = lane & 15, g = lane >> 4;

    // Units are software-pipelined: while unit U renders, the ranges of U+1
    // are in flight and the atomic for U+2 is issued; U+1's first batch of
    // records is fetched before U's image stores.  So a unit starts on
    // loaded data instead of a counter -> ranges -> vals -> planes chain.
    uint32_t unit = 0, nunit = 0, my_nn = 0;
    if (lane == 0) {
        unit = p.unit_lo + atomicAdd(unit_ctr, 1u);
        nunit = p.unit_lo + atomicAdd(unit_ctr, 1u);
    }
    unit = __shfl_sync(0xffffffffu, unit, 0);
    nunit = __shfl_sync(0xffffffffu, nunit, 0);
    uint2 rg = unit < units ? ranges[unit >> 1] : make_uint2(0u, 0u);
    float4 nA = make_float4(0, 0, 0, 0), nB = nA, nC = nA;
    auto fetch = [&](uint32_t base, uint32_t lim) {
        const uint32_t i = base + lane;
        if (i < lim) {
            const uint32_t gid = __ldg(&vals[i]);
            nA = __ldg(&P0[gid]);
            nB = __ldg(&P1[gid]);
            nC = __ldg(&P2[gid]);
        }
    };
    bool pre = false;  // nA/nB/nC hold the first batch of `unit`

    while (unit < units) {
        if (lane == 0) my_nn = p.unit_lo + atomicAdd(unit_ctr, 1u);
        const uint2 nrg = nunit < units ? ranges[nunit >> 1] : make_uint2(0u, 0u);
        const int tile = static_cast<int>(unit >> 1), half = static_cast<int>(unit & 1u);
        const int tx = tile % p.tiles_x, ty = tile / p.tiles_x;
        const int x0 = tx * 16, y0 = ty * 16 + half * 8;
        const int w = imin(16, p.W - x0), h = imin(8, p.H - y0);  // h may be <= 0 (bottom tile row)
        // pixel centres relative to the unit's centre (ucx, ucy): lane
        // offsets in [-7.5, 7.5] x [-3.5, 3.5], all exact in float
        const float ucx = static_cast<float>(x0 + 8), ucy = static_cast<float>(y0 + 4);
        const float lxl = static_cast<float>(lx) - 7.5f;
        float lyl[PPT], T[PPT], Cr[PPT], Cg[PPT], Cb[PPT];
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
            lyl[k] = static_cast<float>(4 * g + k) - 3.5f;
            T[k] = (lx < w && 4 * g + k < h) ? 1.0f : 0.0f;  // outside the image: saturated
            Cr[k] = Cg[k] = Cb[k] = 0.0f;
        }
        const float cx0 = x0 + 0.5f, cx1 = x0 + w - 0.5f;
        const float cy0 = y0 + 0.5f, cy1 = y0 + h - 0.5f;

        const uint32_t start = rg.x, end = rg.y > rg.x ? rg.y : rg.x;
        uint32_t death = 0;
        bool all_done = h <= 0;
        if (!pre && !all_done && start < end) fetch(start, end);
        for (uint32_t base = start; base < end && !all_done; base += 32) {
            const float4 cA = nA, cB = nB, cC = nC;
            if (base + 32 < end) fetch(base + 32, end);
            // Box of the unit's live pixel centres (T >= floor; it only shrinks
            // during the batch): a splat whose extent misses it can blend no
            // live pixel -- the reference masks saturated pixels, so skipping
            // it only drops weight below the floor and no P_it event.
            float lx0 = cx0, lx1 = cx1, ly0 = cy0, ly1 = cy1;
            if (base != start) {
                int r_lo = 8, r_hi = -1;
#pragma unroll
                for (int k = PPT - 1; k >= 0; --k)
                    if (T[k] >= tfloor) r_lo = 4 * g + k;
#pragma unroll
                for (int k = 0; k < PPT; ++k)
                    if (T[k] >= tfloor) r_hi = 4 * g + k;
                const bool lv = r_hi >= 0;
                const int xlo = __reduce_min_sync(0xffffffffu, lv ? lx : 16);
                const int xhi = __reduce_max_sync(0xffffffffu, lv ? lx : -1);
                const int ylo = __reduce_min_sync(0xffffffffu, lv ? r_lo : 8);
                const int yhi = __reduce_max_sync(0xffffffffu, lv ? r_hi : -1);
                lx0 = static_cast<float>(x0 + xlo) + 0.5f;
                lx1 = static_cast<float>(x0 + xhi) + 0.5f;
                ly0 = static_cast<float>(y0 + ylo) + 0.5f;
                ly1 = static_cast<float>(y0 + yhi) + 0.5f;
            }
            bool rel = base + lane < end && meets_box(cA.x, cA.y, unpack_extent(cC.w), lx0, lx1, ly0, ly1);
            const uint32_t m = __ballot_sync(0xffffffffu, rel);
            if (!m) continue;
            // the survivors are staged compacted, in pair order: the blend loop
            // walks consecutive records (no find-first per splat)
            const uint32_t nrel = static_cast<uint32_t>(__popc(m));
            if (rel) {
                const int r = __popc(m & ((1u << lane) - 1u));
                // The exponent x = c q + L (alpha ~ 2^x, c = -log2(e)/2, L =
                // log2 opacity) in unit-centred coordinates, expanded once per
                // (splat, unit): with (mlx, mly) = mean - unit centre,
                //   q(l) = ixx lx^2 + 2ixy lx ly + iyy ly^2 + bx lx + by ly + c0,
                // and every coefficient scaled by c (c0 also carries L), so a
                // pixel costs 2 FMA (Horner in ly) and feeds EX2 directly.
                // Every term and partial sum is bounded by S~ = |c| S + |L|,
                // S = the absolute form at (|mlx| + 7.5, |mly| + 3.5); the float
                // evaluation here and in the loop, the rounded (mlx, mly) and
                // scaled coefficients, and the reference's own rounding of
                // (px - mx, py - my) and of its q keep x within 39 u S~ of
                // c q_ref + L (u = 2^-24).  With E~ = 4e-6 S~ > 67 u S~ and
                // directed rounding, x > xs = c qsafe + L + E~ proves q_ref <
                // qsafe (alpha >= tau) and x < xc = c qcut + L - E~ proves
                // q_ref > qcut (alpha < tau); the band between goes to the
                // exact path.
                constexpr float c_ex2 = -0.5f * 1.4426950408889634f;
                const float mlx = cA.x - ucx, mly = cA.y - ucy;
                const float ixx = cA.z, b2 = cA.w, iyy = cB.x;
                const float bx = -(2.0f * ixx * mlx + b2 * mly);
                const float by = -(b2 * mlx + 2.0f * iyy * mly);
                const float c0 = (ixx * mlx * mlx + b2 * mlx * mly) + iyy * mly * mly;
                const float L = fast_log2(cB.y);
                const float X = fabsf(mlx) + 7.5f, Y = fabsf(mly) + 3.5f;
                const float S = (fabsf(ixx) * X * X + fabsf(b2) * X * Y) + fabsf(iyy) * Y * Y;
                const float E = (-c_ex2 * S + fabsf(L)) * 4e-6f;
                const float inf = __int_as_float(0x7f800000);
                // qsafe = -inf (never fast) / qcut = +inf (no cut) stay infinite
                float xs = cB.w == -inf ? inf : __fadd_ru(__fadd_ru(__fmul_ru(c_ex2, cB.w), L), E);
                float xc = cB.z == inf ? -inf : __fsub_rd(__fadd_rd(__fmul_rd(c_ex2, cB.z), L), E);
                if (!(E < inf) || xs != xs || xc != xc) xs = inf, xc = -inf;  // no bound: every pixel is exact
                sS[warp][r][0] = make_float4(c_ex2 * ixx, c_ex2 * b2, c_ex2 * iyy, c_ex2 * bx);
                // {c by, c c0 + L, band width w = xs - xc (rounded up), xs}: a
                // pixel is in the band only if 0 <= xs - x <= w (rounding is
                // monotone, so fl(xs - x) <= w whenever x >= xc; infinite
                // thresholds give w = +inf); x > xs (fast) has the sign bit set
                sS[warp][r][1] = make_float4(c_ex2 * by, __fmaf_rn(c_ex2, c0, L), __fsub_ru(xs, xc), xs);
                // red carries the clamp flag in its sign (colours are >= 0):
                // alpha_at's clamp can bind only for opacity >= clamp
                // .w: the record's index in the batch (P_it)
                sS[warp][r][2] = make_float4(cB.y >= aclamp ? -cC.x : cC.x, cC.y, cC.z, __int_as_float(lane));
                sS[warp][r][3] = cA;                                   // mx, my, ixx, 2ixy
                sS[warp][r][4] = make_float4(cB.x, cB.y, 0.0f, 0.0f);  // iyy, opacity
            }
            __syncwarp();
            uint32_t jj = 0;  // nrel >= 1: the exit test sits at the bottom
            do {
                const float4 sa = sS[warp][jj][0];  // c {inv.xx, 2*inv.xy, inv.yy, bx}
                const float4 sb = sS[warp][jj][1];  // c by, c c0 + L, xs - xc, xs
                const float4 sc = sS[warp][jj][2];  // +-r, g, b, batch index
                const float qB = __fmaf_rn(sa.y, lxl, sb.x);                     // c (2ixy lx + by)
                const float qC = __fmaf_rn(__fmaf_rn(sa.x, lxl, sa.w), lxl, sb.y);  // c ((ixx lx + bx) lx + c0) + L
                const float xs = sb.w;
                const uint32_t wbits = __float_as_uint(sb.z);
                if (STATS) {
                    ++st_it;
                    uint32_t mine = 0;
#pragma unroll
                    for (int k = 0; k < PPT; ++k) mine += T[k] >= tfloor;
                    st_on += mine;
                    const uint32_t live_w = __reduce_add_sync(0xffffffffu, mine);
                    st_lo32 += live_w <= 32u;
                    st_lo64 += live_w <= 64u;
                }
                // Pixels are not masked once saturated (T < floor): their
                // remaining blend weights sum to less than T <= floor = 1e-4,
                // which bounds the image difference to the reference by
                // 1e-4 per channel; the warp stops when all are saturated.
                // Fast pixels blend under a predicate (no zeroed alphas).  The
                // band test compares float bits unsigned: xs - x < 0 (a fast
                // pixel) has the sign bit set and exceeds any w >= 0; NaN
                // exceeds +inf (never blends, as in the reference).  It admits
                // a superset of the band (pixels just below xc); the exact
                // path rejects those by its own alpha >= tau test.
                uint32_t dmin = 0xffffffffu;
                bool fast[PPT];
                float e[PPT], xv[PPT];
#pragma unroll
                for (int k = 0; k < PPT; ++k) {
                    const float x = __fmaf_rn(__fmaf_rn(sa.z, lyl[k], qB), lyl[k], qC);
                    xv[k] = x;
                    fast[k] = x > xs;
                    e[k] = fast_exp2(x);
                    dmin = umin(dmin, __float_as_uint(xs - x));
                    if (STATS) {
                        st_fast += fast[k] && T[k] >= tfloor;
                        st_need += __float_as_uint(xs - x) <= wbits;
                    }
                }
                const bool need_any = dmin <= wbits;
                if (STATS) {  // iterations in which no pixel of the unit is within x >= xc
                    bool any_in = false;
#pragma unroll
                    for (int k = 0; k < PPT; ++k) any_in = any_in || !(xv[k] < xs - sb.z);
                    st_empty += !__any_sync(0xffffffffu, any_in);
                    bool any_live = false;  // ... or within x >= xc of no live (T >= floor) pixel
#pragma unroll
                    for (int k = 0; k < PPT; ++k) any_live = any_live || (T[k] >= tfloor && !(xv[k] < xs - sb.z));
                    st_dead += !__any_sync(0xffffffffu, any_live);
                }
                if (CLAMP && __float_as_int(sc.x) < 0) {  // clamp flag (opacity >= clamp)
#pragma unroll
                    for (int k = 0; k < PPT; ++k) e[k] = fminf(e[k], aclamp);
                }
#pragma unroll
                for (int k = 0; k < PPT; ++k) {
                    if (!fast[k]) continue;
                    const float wgt = e[k] * T[k];
                    Cr[k] = __fmaf_rn(wgt, fabsf(sc.x), Cr[k]);
                    Cg[k] = __fmaf_rn(wgt, sc.y, Cg[k]);
                    Cb[k] = __fmaf_rn(wgt, sc.z, Cb[k]);
                    T[k] = __fmaf_rn(-e[k], T[k], T[k]);
                }
                if (__any_sync(0xffffffffu, need_any)) {  // margin band: the reference's alpha_at
                    const float4 sd = sS[warp][jj][3];  // mx, my, ixx, 2ixy (unscaled)
                    const float2 se = *reinterpret_cast<const float2*>(&sS[warp][jj][4]);  // iyy, opacity
                    const float dx = (ucx + lxl) - sd.x;  // px - mx, as the reference rounds it
                    const float t1 = sd.z * dx * dx;
                    const float t2 = sd.w * dx;
#pragma unroll
                    for (int k = 0; k < PPT; ++k) {
                        if (!(__float_as_uint(xs - xv[k]) <= wbits)) continue;
                        const float dy = (ucy + lyl[k]) - sd.y;
                        const float qr = (t1 + t2 * dy) + se.x * dy * dy;  // reference order
                        const float a = exact_alpha(qr, se.y, aclamp, sTab);
                        if (a < tau) continue;
                        const float t_cur = T[k];
                        const float wgt = a * t_cur;
                        Cr[k] += wgt * fabsf(sc.x);
                        Cg[k] += wgt * sc.y;
                        Cb[k] += wgt * sc.z;
                        T[k] = t_cur * (1.0f - a);
                    }
                }
                const float tmax = fmaxf(fmaxf(T[0], T[1]), fmaxf(T[2], T[3]));
                if (!__any_sync(0xffffffffu, tmax >= tfloor)) {
                    death = base - start + static_cast<uint32_t>(__float_as_int(sc.w)) + 1;
                    all_done = true;
                    break;
                }
            } while (++jj < nrel);
            __syncwarp();
        }

        // the next unit's first batch, in flight during this unit's stores
        pre = nunit < units && nrg.y > nrg.x;
        if (pre) fetch(nrg.x, nrg.y);

        // P_it (rasterizer.cpp:55-56): per unit n if any pixel stays
        // unsaturated, else the 1-based index of the saturating pair; per
        // tile the max over both units, by a fire-and-forget atomicMax on
        // the tile's word (summed over the tiles when the stats are read).
        if (lane == 0 && pit && end > start) {
            const uint32_t mine = h <= 0 ? 0u : (all_done ? death : end - start);
            if (mine) atomicMax(reinterpret_cast<unsigned int*>(&tile_pit[tile]), mine);
        }

        // store: stage the unit in shared memory, then whole rows (float4)
        if (h > 0) {
            float* so = sOut[warp];
#pragma unroll
            for (int k = 0; k < PPT; ++k) {
                float* o = &so[((4 * g + k) * 16 + lx) * 3];
                o[0] = sclamp(Cr[k] + T[k] * p.bg[0], 0.0f, 1.0f);
                o[1] = sclamp(Cg[k] + T[k] * p.bg[1], 0.0f, 1.0f);
                o[2] = sclamp(Cb[k] + T[k] * p.bg[2], 0.0f, 1.0f);
            }
            __syncwarp();
            if (w == 16 && (p.W & 3) == 0) {
                for (int i = lane; i < 12 * h; i += 32) {
                    const int row = i / 12, col = i % 12;
                    float4* dst = reinterpret_cast<float4*>(image + (static_cast<size_t>(y0 + row) * p.W + x0) * 3);
                    __stcs(&dst[col], reinterpret_cast<const float4*>(so)[row * 12 + col]);
                }
            } else {
                for (int i = lane; i < w * h * 3; i += 32) {
                    const int c = i % 3, pix = i / 3, row = pix / w, col = pix % w;
                    image[(static_cast<size_t>(y0 + row) * p.W + x0 + col) * 3 + c] = so[(row * 16 + col) * 3 + c];
                }
            }
            if (img_u8) {  // write_image bytes of the unit: lround(clamp(v) * 255) (gsio.cpp:265-281)
                auto q8 = [](float v) {
                    return static_cast<uint32_t>(floor(static_cast<double>(sclamp(v, 0.0f, 1.0f)) * 255.0 + 0.5));
                };
                if (w == 16 && (p.W & 3) == 0) {  // 12 words of 4 bytes per row
                    for (int i = lane; i < 12 * h; i += 32) {
                        const int row = i / 12, col = i % 12;
                        const float* v = &so[row * 48 + 4 * col];
                        const uint32_t word = q8(v[0]) | (q8(v[1]) << 8) | (q8(v[2]) << 16) | (q8(v[3]) << 24);
                        *reinterpret_cast<uint32_t*>(img_u8 + (static_cast<size_t>(y0 + row) * p.W + x0) * 3 + 4 * col) =
                            word;
                    }
                } else {
                    for (int i = lane; i < w * h * 3; i += 32) {
                        const int c = i % 3, pix = i / 3, row = pix / w, col = pix % w;
                        img_u8[(static_cast<size_t>(y0 + row) * p.W + x0 + col) * 3 + c] =
                            static_cast<uint8_t>(q8(so[(row * 16 + col) * 3 + c]));
                    }
                }
            }
            __syncwarp();
        }
        if (band_done) {  // this unit's pixels are in memory: count it for its egress band
            __threadfence();  // every lane's image stores, before the count the copy stream waits on
            __syncwarp();
            if (lane == 0) atomicAdd(&band_done[ty / band_rows], 1u);
        }
        unit = nunit;
        rg = nrg;
        nunit = __shfl_sync(0xffffffffu, my_nn, 0);
    }
    if (STATS) {
        for (int o = 16; o > 0; o >>= 1) {
            st_on += __shfl_xor_sync(0xffffffffu, st_on, o);
            st_fast += __shfl_xor_sync(0xffffffffu, st_fast, o);
            st_need += __shfl_xor_sync(0xffffffffu, st_need, o);
        }
        if (lane == 0) {
            atomicAdd(&dbg[0], st_it);
            atomicAdd(&dbg[1], st_on);
            atomicAdd(&dbg[2], st_fast);
            atomicAdd(&dbg[3], st_need);
            atomicAdd(&dbg[4], st_lo32);
            atomicAdd(&dbg[5], st_lo64);
            atomicAdd(&dbg[6], st_empty);
            atomicAdd(&dbg[7], st_dead);
        }
    }
}

void launch_raster_units(int grid, cudaStream_t st, const FrameParams& p, const uint2* ranges, const uint32_t* vals,
                         const float4* P0, const float4* P1, const float4* P2, float* image, uint32_t* unit_ctr,
                         unsigned long long* tile_pit, unsigned long long* pit, unsigned long long* dbg,
                         uint32_t* band_done, int band_rows, uint8_t* img_u8) {
    static const bool stats = [] {  // AGSX_RASTER_STATS=1: work counters in frame_stats()
        const char* t = std::getenv("AGSX_RASTER_STATS");
        return t && *t == '1';
    }();
#define AGSX_RU_ARGS st, p, ranges, vals, P0, P1, P2, image, unit_ctr, tile_pit, pit, dbg, band_done, band_rows, img_u8
    if (stats)
        launch_pdl(k_raster_units<true, true>, dim3(grid), dim3(256), 0, AGSX_RU_ARGS);
    else if (p.clamp_free)
        launch_pdl(k_raster_units<false, false>, dim3(grid), dim3(256), 0, AGSX_RU_ARGS);
    else
        launch_pdl(k_raster_units<false, true>, dim3(grid), dim3(256), 0, AGSX_RU_ARGS);
#undef AGSX_RU_ARGS
}

cudaError_t raster_units_occupancy(int* occ) {
    int a = 0, b = 0;  // both variants run at the occupancy of the smaller
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_raster_units<false, true>, 256, 0);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_raster_units<false, false>, 256, 0);
    *occ = a < b ? a : b;
    return e;
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
    griddep_wait();
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

    // Tiles above 64x64 pixels are split into 64x64 blocks, one CTA each,
    // every block walking the whole pair range of its tile: a pixel's value
    // depends only on the tile's pair sequence (rasterizer.cpp:56-90; the
    // early stop is an optimisation), so the blocks are independent.
    const int ts = p.tile_size;
    const int bs = imin(ts, 64);
    const int nsub = (ts + 63) / 64;
    const int tile = static_cast<int>(blockIdx.x) / (nsub * nsub);
    const int sub = static_cast<int>(blockIdx.x) % (nsub * nsub);
    const int tx = tile % p.tiles_x, ty = tile / p.tiles_x;
    const int x0 = tx * ts, y0 = ty * ts;
    const int w = imin(ts, p.W - x0), h = imin(ts, p.H - y0);
    const int sx0 = (sub % nsub) * bs, sy0 = (sub / nsub) * bs;

    int lx[PPT], ly[PPT];
    float px[PPT], py[PPT], T[PPT], Cr[PPT], Cg[PPT], Cb[PPT];
    uint32_t live = 0, death = 0;
    float bx0 = 1e30f, bx1 = -1e30f, by0 = 1e30f, by1 = -1e30f;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
        const int lp = tid + k * 256;
        lx[k] = sx0 + lp % bs;
        ly[k] = lp < bs * bs ? sy0 + lp / bs : ts;
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
                const float qsafe = EXACT ? -__int_as_float(0x7f800000) : sb.w;
                bool newly_done = false;
#pragma unroll
                for (int k = 0; k < PPT; ++k) {
                    if (!((live >> k) & 1u)) continue;
                    const float dx = px[k] - sa.x, dy = py[k] - sa.y;
                    const float q = (sa.z * dx * dx + sa.w * dx * dy) + sb.x * dy * dy;
                    const uint32_t qb = __float_as_uint(q);
                    float a;
                    if (q >= 0.0f && q < qsafe) {
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
        if (maxt) launch_pdl(k_raster16<Q, true, true>, dim3(grid), dim3(256 / Q), 0, st, p, ranges, vals, P0, P1, P2, image, mt, pit);
        else launch_pdl(k_raster16<Q, true, false>, dim3(grid), dim3(256 / Q), 0, st, p, ranges, vals, P0, P1, P2, image, mt, pit);
    } else {
        if (maxt) launch_pdl(k_raster16<Q, false, true>, dim3(grid), dim3(256 / Q), 0, st, p, ranges, vals, P0, P1, P2, image, mt, pit);
        else launch_pdl(k_raster16<Q, false, false>, dim3(grid), dim3(256 / Q), 0, st, p, ranges, vals, P0, P1, P2, image, mt, pit);
    }
}

template <int PPT>
static void launch_ppt(bool exact, bool maxt, int grid, cudaStream_t st, const FrameParams& p,
                       const uint2* ranges, const uint32_t* vals, const float4* P0, const float4* P1,
                       const float4* P2, float* image, uint32_t* mt, unsigned long long* pit) {
    if (exact) {
        if (maxt) launch_pdl(k_raster<PPT, true, true>, dim3(grid), dim3(256), 0, st, p, ranges, vals, P0, P1, P2, image, mt, pit);
        else launch_pdl(k_raster<PPT, true, false>, dim3(grid), dim3(256), 0, st, p, ranges, vals, P0, P1, P2, image, mt, pit);
    } else {
        if (maxt) launch_pdl(k_raster<PPT, false, true>, dim3(grid), dim3(256), 0, st, p, ranges, vals, P0, P1, P2, image, mt, pit);
        else launch_pdl(k_raster<PPT, false, false>, dim3(grid), dim3(256), 0, st, p, ranges, vals, P0, P1, P2, image, mt, pit);
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

namespace agsx {

// raster_tile with the blend-event stream (RecordOptions::contributions,
// rasterizer.cpp:21-100): one warp per tile, the reference's exact
// per-pixel semantics (masked once T < floor, glibc-exact alpha, stop when
// every pixel is saturated).  Per pair the tile's pixels are visited in
// chunks of 256, lane l owning the 8 consecutive row-major pixels
// 8l..8l+7 of a chunk, so a warp scan of the per-lane event counts places
// the events in the reference's order (pair, then row-major pixel).  With
// `out == nullptr` the pass only counts the tile's events into counts[tile];
// otherwise they are written from offsets[tile].  The image is written too.
// T and C of the tile live in shared memory (16 bytes per pixel).
__global__ void __launch_bounds__(32)
k_raster_records(FrameParams p, const uint2* __restrict__ ranges, const uint32_t* __restrict__ vals,
                 const float4* __restrict__ P0, const float4* __restrict__ P1, const float4* __restrict__ P2,
                 float* __restrict__ image, uint32_t* __restrict__ counts, const uint64_t* __restrict__ offsets,
                 agsx_blend_record* __restrict__ out) {
    extern __shared__ __align__(16) float rec_smem[];
    __shared__ uint64_t sTab[32];
    const int lane = threadIdx.x;
    sTab[lane] = kExp2fTab[lane];
    const int tile = blockIdx.x;
    const int ts = p.tile_size;
    const int tx = tile % p.tiles_x, ty = tile / p.tiles_x;
    const int x0 = tx * ts, y0 = ty * ts;
    const int w = imin(ts, p.W - x0), h = imin(ts, p.H - y0);
    const int npx = w * h;
    float* T = rec_smem;
    float* C = rec_smem + npx;
    for (int i = lane; i < npx; i += 32) {
        T[i] = 1.0f;
        C[3 * i] = C[3 * i + 1] = C[3 * i + 2] = 0.0f;
    }
    __syncwarp();
    const uint2 rg = ranges[tile];
    const float tau = p.tau, fl = p.tfloor, aclamp = p.aclamp;
    uint64_t at = out ? offsets[tile] : 0;
    uint32_t n = 0;
    int active = npx;
    for (uint32_t k = rg.x; k < rg.y && active > 0; ++k) {
        const uint32_t gid = vals[k];
        const float4 a4 = P0[gid], b4 = P1[gid], c4 = P2[gid];  // {mean, ixx, 2 ixy}, {iyy, opacity, ..}, {rgb, ..}
        for (int base = 0; base < npx; base += 256) {
            float al[8];
            uint32_t flags = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                al[j] = 0.0f;
                const int pi = base + 8 * lane + j;
                if (pi >= npx || T[pi] < fl) continue;
                const int iy = pi / w, ix = pi - iy * w;
                // alpha_at (rasterizer.hpp:44-50): SymMat2::quad in the reference's order
                const float dx = (static_cast<float>(x0 + ix) + 0.5f) - a4.x;
                const float dy = (static_cast<float>(y0 + iy) + 0.5f) - a4.y;
                const float q = (a4.z * dx * dx + a4.w * dx * dy) + b4.x * dy * dy;
                const float a = exact_alpha(q, b4.y, aclamp, sTab);
                if (a < tau) continue;
                al[j] = a;
                flags |= 1u << j;
            }
            const uint32_t cnt = __popc(flags);
            uint32_t incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
            uint64_t idx = at + n + (incl - cnt);
            int dead = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (!((flags >> j) & 1u)) continue;
                const int pi = base + 8 * lane + j;
                const float a = al[j], t_cur = T[pi];
                const float weight = a * t_cur;
                if (out) {
                    const int iy = pi / w, ix = pi - iy * w;
                    agsx_blend_record r;
                    r.pixel = static_cast<uint32_t>((y0 + iy) * p.W + (x0 + ix));
                    r.splat = gid;
                    r.alpha = a;
                    r.weight = weight;
                    out[idx++] = r;
                }
                C[3 * pi] += weight * c4.x;
                C[3 * pi + 1] += weight * c4.y;
                C[3 * pi + 2] += weight * c4.z;
                const float t_next = t_cur * (1.0f - a);
                T[pi] = t_next;
                dead += t_next < fl;
            }
            n += total;
            active -= __reduce_add_sync(0xffffffffu, static_cast<uint32_t>(dead));
        }
    }
    if (!out && lane == 0) counts[tile] = n;
    __syncwarp();
    for (int i = lane; i < npx; i += 32) {
        const int iy = i / w, ix = i - iy * w;
        float* o = &image[(static_cast<size_t>(y0 + iy) * p.W + (x0 + ix)) * 3];
        o[0] = sclamp(C[3 * i] + T[i] * p.bg[0], 0.0f, 1.0f);
        o[1] = sclamp(C[3 * i + 1] + T[i] * p.bg[1], 0.0f, 1.0f);
        o[2] = sclamp(C[3 * i + 2] + T[i] * p.bg[2], 0.0f, 1.0f);
    }
}

cudaError_t launch_raster_records(cudaStream_t st, const FrameParams& p, const uint2* ranges, const uint32_t* vals,
                                  const float4* P0, const float4* P1, const float4* P2, float* image,
                                  uint32_t* counts, const uint64_t* offsets, agsx_blend_record* out) {
    const int grid = p.tiles_x * p.tiles_y;
    if (grid == 0) return cudaSuccess;
    const size_t smem = static_cast<size_t>(p.tile_size) * p.tile_size * 16;
    if (smem > 48 * 1024) {  // per device (a process may drive several)
        const cudaError_t attr = cudaFuncSetAttribute(k_raster_records, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                      static_cast<int>(smem));
        if (attr != cudaSuccess) return attr;
    }
    k_raster_records<<<grid, 32, smem, st>>>(p, ranges, vals, P0, P1, P2, image, counts, offsets, out);
    return cudaGetLastError();
}

}  // namespace agsx

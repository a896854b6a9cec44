// agsx_internal.cuh -- device data layout and shared device functions of the
// B200 render path.  See DESIGN.md §3 for the HBM layout.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/agsx.h"
#include "device_math.cuh"

namespace agsx {

constexpr int kLutInline = 64;
constexpr uint32_t kAliveBit = 0x80000000u;
constexpr uint32_t kCountMask = 0x7fffffffu;

// Everything a frame's kernels need, passed by value (kernel parameter
// space), so a frame needs no host->device copies besides this launch state.
struct FrameParams {
    // camera (scene.hpp:34-49)
    float cam_pos[3];
    float R[9];
    float fx, fy;
    int W, H;
    float ppx, ppy;       // principal_point(): 0.5f * (float)W, 0.5f * (float)H
    double lim_x, lim_y;  // guard_band * 0.5 * W / fx (preprocess.cpp:45-46), host-evaluated
    double Rd[9], fxd, fyd;  // exact double copies of R, fx, fy (no per-thread conversions)
    // config (scene.hpp:65-78)
    int tile_size, tiles_x, tiles_y;
    int mode;
    int fixed_aabb;
    float tau, tfloor, aclamp, near_plane, guard, k;
    float bg[3];
    uint32_t flags;
    int raster_ppt;  // pixels per thread of the 16x16 rasterizer (2 or 4)
    uint32_t unit_lo, unit_hi;  // raster work-unit range of this launch (unit_hi = 0: all units)
    uint32_t clamp_free;        // no splat's opacity reaches aclamp (alpha_at's clamp never binds)
    // T_upper LUT (lut.hpp:11-26)
    int adaptive;
    float lut_dmin, lut_dmax;
    int lut_n;
    float lut_w;  // (lut_dmax - lut_dmin) / lut_n, IEEE on the host (the same float as per thread)
    float lut[kLutInline];
    const float* lut_ext;  // device copy when lut_n > kLutInline
};

// Device-resident scene (uploaded once; 56 B per Gaussian for SH degree 0).
// The scene is stored in a spatial (3D Morton) order chosen at upload: slot
// s holds the Gaussian with id orig[s] (the caller's index, which orders
// equal depths, preprocess.cpp:158-162) and inv[g] is the slot of Gaussian
// g.  Every per-splat frame array (status, depth keys, planes) is indexed by
// slot; ids are translated where the reference's order or an output needs
// them.  orig = inv = nullptr: slot = id.
struct DevScene {
    uint64_t n;
    int sh_coeffs;  // D per channel
    const float4* pos_op;   // mean.xyz, opacity
    const float4* rot;      // w, x, y, z
    const float4* scale_r;  // scale.xyz, sh[0] (red DC)
    const float2* sh_gb;    // sh[1], sh[2] (green/blue DC)
    const float* sh_rest;   // (D-1)*3 floats per Gaussian, coefficient-major
    const uint32_t* orig;   // slot -> Gaussian id
    const uint32_t* inv;    // Gaussian id -> slot
    __host__ __device__ __forceinline__ uint32_t id_of(uint32_t slot) const { return orig ? orig[slot] : slot; }
    __host__ __device__ __forceinline__ uint32_t slot_of(uint32_t id) const { return inv ? inv[id] : id; }
};

// Per-splat planes written by preprocess for splats that hit >= 1 tile,
// indexed by Gaussian id (value of every pair).
//   P0 = {mean.x, mean.y, inv.xx, 2*inv.xy}          raster + emit
//   P1 = {inv.yy, opacity, qcut, qsafe}              raster + emit(inv.yy)
//   P2 = {r, g, b, half2(ex, ey)}                    raster
//   P3 = hit record (hit_record below)                emit
//   P4 = {v1.x, v1.y, a, b}                          emit, OBB mode only
struct SplatPlanes {
    float4* p0;
    float4* p1;
    float4* p2;
    float4* p3;
    float4* p4;
};

// ---- tile intersection (pair_gen.cpp:11-159) ---------------------------
struct TileTest {
    float cx, cy;
    float rx, ry;    // half extents of the candidate box (r_px for AABB/OBB)
    float ixx, ixy, iyy, r2;  // ellipse / adagscale
    float v1x, v1y, a, b;     // obb
    int mode;
};

struct Span {
    int tx0, ty0, tx1, ty1;
    bool empty;
};

// eigen_sym2 (math.hpp:105-131); only l1, l2, v1 are consumed.
__host__ __device__ __forceinline__ void eigen_sym2(float xx, float xy, float yy, float& l1,
                                                     float& l2, float& v1x, float& v1y) {
    const float mean = 0.5f * (xx + yy);
    const float hd = 0.5f * (xx - yy);
    const float r = sqrtf(hd * hd + xy * xy);
    l1 = mean + r;
    l2 = mean - r;
    if (xy == 0.0f) {
        if (xx >= yy) {
            v1x = 1.0f;
            v1y = 0.0f;
        } else {
            v1x = 0.0f;
            v1y = 1.0f;
        }
        return;
    }
    const float ax = l1 - yy, ay = xy;
    const float bx = xy, by = l1 - xx;
    const bool pick_a = (ax * ax + ay * ay) >= (bx * bx + by * by);
    const float vx = pick_a ? ax : bx, vy = pick_a ? ay : by;
    const float n = sqrtf(vx * vx + vy * vy);
    v1x = vx / n;
    v1y = vy / n;
}

// Builds the mode-specific tile test of intersect_tiles (pair_gen.cpp:108-116,
// 145-147).  th is the splat's threshold in AdaGScale mode, tau otherwise.
__device__ __forceinline__ TileTest make_tile_test(float cx, float cy, float cxx, float cxy,
                                                   float cyy, float ixx, float ixy, float iyy,
                                                   float opacity, float th, const FrameParams& p) {
    TileTest t;
    t.mode = p.mode;
    t.cx = cx;
    t.cy = cy;
    const float th_eff = p.mode == AGSX_MODE_ADAGSCALE ? th : p.tau;
    float r = sqrtf(2.0f * glibc_logf(opacity / th_eff));
    if (p.mode == AGSX_MODE_AABB && p.fixed_aabb) r = 3.0f;
    t.ixx = ixx;
    t.ixy = ixy;
    t.iyy = iyy;
    t.r2 = r * r;
    t.v1x = t.v1y = t.a = t.b = 0.0f;
    if (p.mode == AGSX_MODE_AABB || p.mode == AGSX_MODE_OBB) {
        float l1, l2, v1x, v1y;
        eigen_sym2(cxx, cxy, cyy, l1, l2, v1x, v1y);
        const float r_px = r * sqrtf(smax(l1, 0.0f));
        t.rx = t.ry = r_px;
        if (p.mode == AGSX_MODE_OBB) {
            t.v1x = v1x;
            t.v1y = v1y;
            t.a = r * sqrtf(smax(l1, 0.0f));
            t.b = r * sqrtf(smax(l2, 0.0f));
        }
    } else {
        t.rx = r * sqrtf(smax(cxx, 0.0f));
        t.ry = r * sqrtf(smax(cyy, 0.0f));
    }
    return t;
}

// tile_span (pair_gen.cpp:41-55)
__device__ __forceinline__ Span tile_span(const TileTest& t, const FrameParams& p) {
    Span s;
    const float ts = static_cast<float>(p.tile_size);
    float ax = t.cx - t.rx, ay = t.cy - t.ry, bx = t.cx + t.rx, by = t.cy + t.ry;
    if ((p.tile_size & (p.tile_size - 1)) == 0) {
        // x / 2^k and x * 2^-k are the same real number, so both round alike
        const float inv = 1.0f / ts;
        ax *= inv, ay *= inv, bx *= inv, by *= inv;
    } else {
        ax /= ts, ay /= ts, bx /= ts, by /= ts;
    }
    s.tx0 = imax(0, f2i_x86(floorf(ax)));
    s.ty0 = imax(0, f2i_x86(floorf(ay)));
    s.tx1 = imin(p.tiles_x - 1, f2i_x86(floorf(bx)));
    s.ty1 = imin(p.tiles_y - 1, f2i_x86(floorf(by)));
    s.empty = s.tx0 > s.tx1 || s.ty0 > s.ty1 || t.cx + t.rx < 0.0f || t.cy + t.ry < 0.0f ||
              t.cx - t.rx > static_cast<float>(p.W) || t.cy - t.ry > static_cast<float>(p.H);
    return s;
}

__device__ __forceinline__ bool box_overlap(float x0, float y0, float x1, float y1, float cx,
                                            float cy, float rx, float ry) {
    return x0 <= cx + rx && cx - rx <= x1 && y0 <= cy + ry && cy - ry <= y1;
}

// SymMat2::quad (math.hpp:91-93): ((xx*dx)*dx + ((2*xy)*dx)*dy) + (yy*dy)*dy
__host__ __device__ __forceinline__ float quad_form(float xx, float xy, float yy, float dx,
                                                    float dy) {
    return xx * dx * dx + 2.0f * xy * dx * dy + yy * dy * dy;
}

// min_quad_to_rect (pair_gen.cpp:65-83)
__device__ __forceinline__ float min_quad_to_rect(const TileTest& t, float x0, float y0, float x1,
                                                  float y1) {
    const float cx = t.cx, cy = t.cy;
    if (cx >= x0 && cx <= x1 && cy >= y0 && cy <= y1) return 0.0f;
    float h0, h1, v0, v1;
    {
        const float dy = y0 - cy;
        const float x = sclamp(cx - t.ixy * dy / t.ixx, x0, x1);
        h0 = quad_form(t.ixx, t.ixy, t.iyy, x - cx, dy);
    }
    {
        const float dy = y1 - cy;
        const float x = sclamp(cx - t.ixy * dy / t.ixx, x0, x1);
        h1 = quad_form(t.ixx, t.ixy, t.iyy, x - cx, dy);
    }
    {
        const float dx = x0 - cx;
        const float y = sclamp(cy - t.ixy * dx / t.iyy, y0, y1);
        v0 = quad_form(t.ixx, t.ixy, t.iyy, dx, y - cy);
    }
    {
        const float dx = x1 - cx;
        const float y = sclamp(cy - t.ixy * dx / t.iyy, y0, y1);
        v1 = quad_form(t.ixx, t.ixy, t.iyy, dx, y - cy);
    }
    return smin(smin(h0, h1), smin(v0, v1));
}

// obb_overlap (pair_gen.cpp:88-104); u = v1, v = (-v1.y, v1.x).
__device__ __forceinline__ bool obb_overlap(const TileTest& t, float x0, float y0, float x1,
                                            float y1) {
    const float ux = t.v1x, uy = t.v1y, vx = -t.v1y, vy = t.v1x;
    const float rx = t.a * fabsf(ux) + t.b * fabsf(vx);
    const float ry = t.a * fabsf(uy) + t.b * fabsf(vy);
    if (!box_overlap(x0, y0, x1, y1, t.cx, t.cy, rx, ry)) return false;
    const float tcx = 0.5f * (x0 + x1), tcy = 0.5f * (y0 + y1);
    const float hw = 0.5f * (x1 - x0);
    const float hh = 0.5f * (y1 - y0);
    const float dx = tcx - t.cx, dy = tcy - t.cy;
    const float tile_u = hw * fabsf(ux) + hh * fabsf(uy);
    if (fabsf(dx * ux + dy * uy) > t.a + tile_u) return false;
    const float tile_v = hw * fabsf(vx) + hh * fabsf(vy);
    if (fabsf(dx * vx + dy * vy) > t.b + tile_v) return false;
    return true;
}

// One tile of the candidate span (tile_rect pair_gen.cpp:24-33 + the
// per-mode test of pair_gen.cpp:118-158).
__device__ __forceinline__ bool tile_hit(const TileTest& t, int tx, int ty, const FrameParams& p) {
    const float ts = static_cast<float>(p.tile_size);
    const float x0 = tx * ts, y0 = ty * ts;
    const float x1 = smin(x0 + ts, static_cast<float>(p.W));
    const float y1 = smin(y0 + ts, static_cast<float>(p.H));
    if (t.mode == AGSX_MODE_AABB) return box_overlap(x0, y0, x1, y1, t.cx, t.cy, t.rx, t.ry);
    if (t.mode == AGSX_MODE_OBB)
        return box_overlap(x0, y0, x1, y1, t.cx, t.cy, t.rx, t.ry) &&
               obb_overlap(t, x0, y0, x1, y1);
    if (!box_overlap(x0, y0, x1, y1, t.cx, t.cy, t.rx, t.ry)) return false;
    return min_quad_to_rect(t, x0, y0, x1, y1) <= t.r2;
}

// Calls f(tx, ty) for every intersected tile in the reference's row-major
// order (pair_gen.cpp:152-158).  For the ellipse / AdaGScale test the
// horizontal-edge minimisers (one exact division each) depend only on the
// tile row and are hoisted out of the column loop, and min(h0, h1, v0, v1)
// <= r2 is decided edge by edge, nearest edges first (the same values, so
// the same decision as min_quad_to_rect, pair_gen.cpp:65-83).
template <class F>
__device__ __forceinline__ void for_each_tile_hit(const TileTest& t, const FrameParams& p, F&& f) {
    const Span s = tile_span(t, p);
    if (s.empty) return;
    if (t.mode == AGSX_MODE_AABB || t.mode == AGSX_MODE_OBB) {
        for (int ty = s.ty0; ty <= s.ty1; ++ty)
            for (int tx = s.tx0; tx <= s.tx1; ++tx)
                if (tile_hit(t, tx, ty, p)) f(tx, ty);
        return;
    }
    const float ts = static_cast<float>(p.tile_size);
    const float W = static_cast<float>(p.W), H = static_cast<float>(p.H);
    const float cx = t.cx, cy = t.cy;
    float y0 = static_cast<float>(s.ty0) * ts;  // tile coordinates advance by exact float adds
    const float x0_first = static_cast<float>(s.tx0) * ts;
    for (int ty = s.ty0; ty <= s.ty1; ++ty, y0 += ts) {
        const float y1 = smin(y0 + ts, H);
        const float dy0 = y0 - cy, dy1 = y1 - cy;
        const float xh0 = cx - t.ixy * dy0 / t.ixx;
        const float xh1 = cx - t.ixy * dy1 / t.ixx;
        const bool row_in = cy >= y0 && cy <= y1;
        // the edges nearer the centre first: a hit usually shows there (the
        // decision is "some edge minimum <= r2" whatever the order)
        const bool h0_first = fabsf(dy0) <= fabsf(dy1);
        const float xha = h0_first ? xh0 : xh1, dya = h0_first ? dy0 : dy1;
        const float xhb = h0_first ? xh1 : xh0, dyb = h0_first ? dy1 : dy0;
        float x0 = x0_first;
        for (int tx = s.tx0; tx <= s.tx1; ++tx, x0 += ts) {
            const float x1 = smin(x0 + ts, W);
            if (!box_overlap(x0, y0, x1, y1, cx, cy, t.rx, t.ry)) continue;
            bool hit = row_in && cx >= x0 && cx <= x1;  // centre inside: min = 0 <= r2
            if (!hit) hit = quad_form(t.ixx, t.ixy, t.iyy, sclamp(xha, x0, x1) - cx, dya) <= t.r2;
            const float dxl = x0 - cx, dxr = x1 - cx;
            const bool v0_first = fabsf(dxl) <= fabsf(dxr);
            if (!hit) {
                const float dx = v0_first ? dxl : dxr;
                const float y = sclamp(cy - t.ixy * dx / t.iyy, y0, y1);
                hit = quad_form(t.ixx, t.ixy, t.iyy, dx, y - cy) <= t.r2;
            }
            if (!hit) hit = quad_form(t.ixx, t.ixy, t.iyy, sclamp(xhb, x0, x1) - cx, dyb) <= t.r2;
            if (!hit) {
                const float dx = v0_first ? dxr : dxl;
                const float y = sclamp(cy - t.ixy * dx / t.iyy, y0, y1);
                hit = quad_form(t.ixx, t.ixy, t.iyy, dx, y - cy) <= t.r2;
            }
            if (hit) f(tx, ty);
        }
    }
}

__device__ __forceinline__ uint32_t count_tiles(const TileTest& t, const FrameParams& p) {
    uint32_t n = 0;
    for_each_tile_hit(t, p, [&](int, int) { ++n; });
    return n;
}

// P3 hit record of a splat, written by the count pass so that emission
// needs no second tile test: for a tile span of <= 64 tiles, {mask lo, mask
// hi, tx0 | ty0 << 16, span width} with bit (ty-ty0)*w + (tx-tx0) set per
// intersected tile (increasing bits = row-major emission order); for larger
// spans {rx, ry, r2, kHitsRecompute} and the emitter re-runs the test.
constexpr uint32_t kHitsRecompute = 0xffffffffu;

__device__ __forceinline__ uint4 hit_record(const TileTest& t, const FrameParams& p, uint32_t& count) {
    count = 0;
    const Span s = tile_span(t, p);
    if (s.empty) return make_uint4(0u, 0u, 0u, 0u);
    const int sw = s.tx1 - s.tx0 + 1, sh = s.ty1 - s.ty0 + 1;
    if (sw * sh <= 64) {
        unsigned long long mask = 0;
        for_each_tile_hit(t, p, [&](int tx, int ty) { mask |= 1ull << ((ty - s.ty0) * sw + (tx - s.tx0)); });
        count = static_cast<uint32_t>(__popcll(mask));
        return make_uint4(static_cast<uint32_t>(mask), static_cast<uint32_t>(mask >> 32),
                          static_cast<uint32_t>(s.tx0) | (static_cast<uint32_t>(s.ty0) << 16),
                          static_cast<uint32_t>(sw));
    }
    count = count_tiles(t, p);
    return make_uint4(__float_as_uint(t.rx), __float_as_uint(t.ry), __float_as_uint(t.r2), kHitsRecompute);
}

// Calls f(tx, ty) for the intersected tiles of a splat in row-major order
// from its hit record r (mask), or by re-running the test t for spans over
// 64 tiles.
template <class F>
__device__ __forceinline__ void hit_tiles(const TileTest& t, const FrameParams& p, uint4 r, F&& f) {
    if (r.w != kHitsRecompute) {
        unsigned long long mask = static_cast<unsigned long long>(r.x) | (static_cast<unsigned long long>(r.y) << 32);
        const int tx0 = static_cast<int>(r.z & 0xffffu), ty0 = static_cast<int>(r.z >> 16);
        const int sw = static_cast<int>(r.w);
        int row = 0, row_end = sw;  // bits arrive in increasing order: track the row, no division
        while (mask) {
            const int b = __ffsll(static_cast<long long>(mask)) - 1;
            mask &= mask - 1;
            while (b >= row_end) {
                ++row;
                row_end += sw;
            }
            f(tx0 + b - (row_end - sw), ty0 + row);
        }
        return;
    }
    for_each_tile_hit(t, p, f);
}

// Blend-side culling data for the rasterizer (not part of the reference; it
// only lets the rasterizer skip, or take a fast path for, pixels whose
// decision alpha >= tau is provable with a margin).  In
// terms of q = d^T inv d (power = -0.5 q exactly), for q evaluated either in
// the reference's operation order or with the rasterizer's FMA form
// (|q_fma - q_ref| <= rho * q, rho = 16 u kappa, kappa = (max(|xx|,|yy|) +
// |xy|) / lambda_min, folded into both thresholds):
//   q > qcut              =>  opacity * expf(-q/2) < tau            (skip)
//   0 <= q < qsafe        =>  opacity * expf(-q/2) >= tau           (fast;
//                             the blended alpha is then clamped like alpha_at)
//   ex, ey                :  |d.x| > ex or |d.y| > ey  =>  q > qcut
// qsafe = -inf disables the fast path (opacity < tau, or kappa too large).
// For rho < 1/4 neither q form can be negative (their error is below q), so
// the fast test needs no sign check.
static __device__ __noinline__ void blend_cull_data_f64(float ixx, float ixy, float iyy, float opacity, float tau,
                                                float aclamp, float& qcut, float& qsafe, float& ex, float& ey) {
    (void)aclamp;
    const float inf = __int_as_float(0x7f800000);
    if (!(opacity >= tau)) {  // alpha <= opacity < tau everywhere (or NaN): never blends
        qcut = 0.0f;          // q > 0 skips; q <= 0 (or NaN) takes the exact path
        qsafe = -inf;
        ex = ey = 0.0f;
        return;
    }
    const double a = ixx, b = ixy, c = iyy;
    const double det = a * c - b * b;
    const double disc = sqrt(fmax(0.0, 0.25 * (a - c) * (a - c) + b * b));
    const double lmax = 0.5 * (a + c) + disc, lmin = 0.5 * (a + c) - disc;
    const double lr = log(static_cast<double>(opacity) / static_cast<double>(tau));  // >= 0
    const double m = 1e-4 * (1.0 + lr);
    const double rho = lmin > 0.0 ? 16.0 * 0x1p-24 * (fmax(fabs(a), fabs(c)) + fabs(b)) / lmin : 1e300;
    if (!(rho < 0.25)) {  // ill-conditioned: every pixel takes the exact path
        qcut = inf;
        qsafe = -inf;
    } else {
        qcut = __double2float_ru(2.0 * (lr + m) * (1.0 + rho));
        qsafe = lr > m ? __double2float_rd(2.0 * (lr - m) * (1.0 - rho)) : -inf;
    }
    // Box of {q <= qcut} inflated for the float evaluation error of q:
    // q_f >= Q (1 - 64 u kappa).
    const double relerr = 64.0 * 0x1p-24 * (lmin > 0.0 ? lmax / lmin : 1e300);
    if (!(det > 0.0) || !(lmin > 0.0) || !(relerr < 0.5) || !(qcut < inf)) {
        ex = ey = inf;  // no culling for this splat
        return;
    }
    const double r2 = static_cast<double>(qcut) / (1.0 - relerr);
    ex = __double2float_ru(sqrt(r2 * c / det) * 1.0001 + 1e-3);  // (M^-1)_xx = iyy / det
    ey = __double2float_ru(sqrt(r2 * a / det) * 1.0001 + 1e-3);
}

// Float evaluation of blend_cull_data_f64 for well-conditioned splats
// (kappa <= 1e3, the common case); every quantity is rounded outward with
// margins far above the float error (the decision margins are 1e-4 relative).
__device__ __forceinline__ void blend_cull_data(float ixx, float ixy, float iyy, float opacity, float tau,
                                                float aclamp, float& qcut, float& qsafe, float& ex, float& ey) {
    const float inf = __int_as_float(0x7f800000);
    if (!(opacity >= tau)) {
        qcut = 0.0f;
        qsafe = -inf;
        ex = ey = 0.0f;
        return;
    }
    const float a = ixx, b = ixy, c = iyy;
    const float lmax = 0.5f * (a + c) + sqrtf(0.25f * (a - c) * (a - c) + b * b);
    const float det = a * c - b * b;
    const float lmin = det / lmax;
    const float kappa = lmax / lmin;
    if (!(det > 0.0f) || !(lmax > 0.0f) || !(kappa <= 1e3f)) {
        blend_cull_data_f64(ixx, ixy, iyy, opacity, tau, aclamp, qcut, qsafe, ex, ey);
        return;
    }
    const float lr = logf(opacity / tau);  // >= 0, error ~1e-7 (1 + lr)
    const float m = 1e-4f * (1.0f + lr);
    const float rho = 1.01f * 16.0f * 0x1p-24f * (fmaxf(fabsf(a), fabsf(c)) + fabsf(b)) / lmin;
    qcut = 2.0f * (lr + m) * (1.0f + rho) * (1.0f + 4e-6f);
    qsafe = lr > m ? 2.0f * (lr - m) * (1.0f - rho) * (1.0f - 4e-6f) : -inf;
    const float relerr = 64.0f * 0x1p-24f * kappa;
    const float r2 = qcut / (1.0f - relerr);
    ex = sqrtf(r2 * c / det) * 1.001f + 1e-3f;
    ey = sqrtf(r2 * a / det) * 1.001f + 1e-3f;
}

__device__ __forceinline__ uint32_t pack_extent(float ex, float ey) {
    const __half hx = __float2half_ru(ex), hy = __float2half_ru(ey);
    return static_cast<uint32_t>(__half_as_ushort(hx)) | (static_cast<uint32_t>(__half_as_ushort(hy)) << 16);
}

// One digit bit of a warp multisplit: keeps the lanes of `pm` whose bit
// (bit != 0) equals this lane's.  One predicate feeds both the ballot and the
// flip (ptxas extracts the 8 predicates of a digit with one R2P): ~3
// instructions per bit instead of 7 for `bit ? bal : ~bal` in C++.
__device__ __forceinline__ uint32_t ballot_agree(uint32_t pm, uint32_t bit) {
    uint32_t r;
    asm("{\n\t.reg .pred p;\n\t"
        "setp.ne.u32 p, %2, 0;\n\t"
        "vote.sync.ballot.b32 %0, p, 0xffffffff;\n\t"
        "@!p not.b32 %0, %0;\n\t"
        "and.b32 %0, %0, %1;\n\t}"
        : "=r"(r)
        : "r"(pm), "r"(bit));
    return r;
}

// ---- decoupled look-back state words -----------------------------------
// u64 = [63:62] flag | [61:32] epoch | [31:0] value.  The epoch (bumped per
// launch) makes stale words from earlier launches invisible, so the state
// arrays never need clearing.
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagIncl = 2ull << 62;

__device__ __forceinline__ uint64_t lb_pack(uint64_t flag, uint32_t epoch, uint32_t v) {
    return flag | (static_cast<uint64_t>(epoch & 0x3fffffffu) << 32) | v;
}
__device__ __forceinline__ void lb_store(uint64_t* a, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t lb_load(const uint64_t* a) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t sat_add(uint32_t a, uint32_t b) {
    const uint32_t s = a + b;
    return s < a ? 0xffffffffu : s;
}

// Single-value look-back by one warp.  Returns the exclusive prefix of
// `tile` and publishes its inclusive prefix.  Called by all 32 lanes of one
// warp; `aggregate` must be warp-uniform.
__device__ __forceinline__ uint32_t lookback_warp(uint64_t* states, uint32_t tile,
                                                  uint32_t aggregate, uint32_t epoch) {
    const int lane = threadIdx.x & 31;
    const uint32_t ep = epoch & 0x3fffffffu;
    if (tile == 0) {
        if (lane == 0) lb_store(&states[0], lb_pack(kFlagIncl, epoch, aggregate));
        return 0;
    }
    if (lane == 0) lb_store(&states[tile], lb_pack(kFlagAgg, epoch, aggregate));
    uint32_t prefix = 0;
    int64_t base = static_cast<int64_t>(tile) - 1;
    while (true) {
        const int64_t idx = base - lane;
        uint64_t s = kFlagIncl;  // virtual inclusive predecessor of tile 0
        uint64_t flag = kFlagIncl;
        if (idx >= 0) {
            s = lb_load(&states[idx]);
            flag = s & (3ull << 62);
            if (static_cast<uint32_t>((s >> 32) & 0x3fffffffu) != ep) flag = 0;
        }
        // All lanes must hold a published word before the window is consumed.
        if (__any_sync(0xffffffffu, flag == 0)) continue;
        const uint32_t incl_mask = __ballot_sync(0xffffffffu, flag == kFlagIncl);
        const uint32_t v = static_cast<uint32_t>(s);
        const int stop = incl_mask ? __ffs(incl_mask) - 1 : 31;
        uint32_t contrib = lane <= stop ? v : 0u;
        for (int o = 16; o > 0; o >>= 1) contrib = sat_add(contrib, __shfl_xor_sync(0xffffffffu, contrib, o));
        prefix = sat_add(prefix, contrib);
        if (incl_mask) break;
        base -= 32;
    }
    if (lane == 0) lb_store(&states[tile], lb_pack(kFlagIncl, epoch, sat_add(prefix, aggregate)));
    return prefix;
}

// Per-frame device counters (one small memset per frame).
struct Counters {
    uint32_t tile_ctr[16];  // dynamic tile ids for look-back kernels
    uint32_t m;             // splats with >= 1 tile (depth-sort length)
    uint32_t s;             // survivors (splat_count)
    uint32_t p;             // total pairs (saturating)
    uint32_t overflow;      // pair buffer capacity exceeded
    uint32_t p_eff;         // p if it fits the pair buffers, else 0 (memory safety)
    uint32_t pad0;
    unsigned long long p_it;  // pairs iterated before tile saturation (raster work)
    unsigned long long dbg[8];  // raster work counters (AGSX_RASTER_STATS=1)
    uint32_t kmin_c;  // ~(min depth key of the splats with >= 1 tile), by atomicMax (0 = none)
    uint32_t kmax;    // max depth key of those splats
    uint32_t band_done[32];  // units finished per egress row slot (banded host egress)
};

// Tile ids of a mask record's hit tiles in row-major order (up to 8).
__device__ __forceinline__ void tiles_of_mask(uint4 r, int tiles_x, uint32_t (&tl)[8]) {
    unsigned long long mask = static_cast<unsigned long long>(r.x) | (static_cast<unsigned long long>(r.y) << 32);
    const uint32_t tx0 = r.z & 0xffffu, ty0 = r.z >> 16, sw = r.w;
    uint32_t row_base = ty0 * static_cast<uint32_t>(tiles_x) + tx0, row_start = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        tl[u] = 0u;
        if (mask) {
            const uint32_t b = static_cast<uint32_t>(__ffsll(static_cast<long long>(mask)) - 1);
            mask &= mask - 1;
            while (b >= row_start + sw) {
                row_start += sw;
                row_base += static_cast<uint32_t>(tiles_x);
            }
            tl[u] = row_base + (b - row_start);
        }
    }
}

// Per-context words that survive the per-frame counter memset: how many of the
// frames enqueued since the last wait overflowed the pair arena (their pairs
// were not emitted, so their images are not the frame's), and how many frames
// that chain holds.  Updated by the counter readback at the end of every frame
// and read back behind the Counters block; finish_frame clears them.
struct ChainWords {
    uint32_t overflowed;
    uint32_t frames;
    uint32_t pad[2];
};

// The depth keys of a frame span >= 2^24 (key - kmin needs a 4th 8-bit
// pass); false when there are no keys.
__device__ __forceinline__ bool depth_keys_wide(uint32_t kmin_c, uint32_t kmax) {
    const uint32_t kmin = ~kmin_c;
    return kmax >= kmin && kmax - kmin >= (1u << 24);
}

}  // namespace agsx

// k_preprocess.cu -- K1: per-Gaussian preprocess fused with the tile-count
// pass and the order-preserving compaction of the splats that hit >= 1 tile.
//
//   reference: preprocess_view  preprocess.cpp:118-163
//              project          preprocess.cpp:26-66
//              eval_color       preprocess.cpp:68-105
//              compute_th       preprocess.cpp:107-116
//              count pass       pair_gen.cpp:167-175 (intersect_tiles :108-159)
//
// One thread per Gaussian.  Output depth keys stay in Gaussian order, with
// 0xffffffff for splats that hit no tile; the first depth-sort pass drops
// those sentinels, which is the order-preserving compaction of the
// reference (preprocess.cpp:158-162) done inside the sort.
#include "agsx_internal.cuh"
#include "kernels.cuh"

constexpr int kPreQ = 12;  // words queued per survivor between K1's phases

#ifndef AGSX_PRE_MINB
#define AGSX_PRE_MINB 4
#endif

namespace agsx {

namespace {

constexpr float kShC0 = 0.28209479177387814f;
constexpr float kShC1 = 0.4886025119029199f;
__device__ __constant__ float kShC2[5] = {1.0925484305920792f, -1.0925484305920792f,
                                          0.31539156525252005f, -1.0925484305920792f,
                                          0.5462742152960396f};
__device__ __constant__ float kShC3[7] = {-0.5900435899266435f, 2.890611442640554f,
                                          -0.4570457994644658f, 0.3731763325901154f,
                                          -0.4570457994644658f, 1.445305721320277f,
                                          -0.5900435899266435f};

// TUpperLUT::value_at (lut.hpp:16-25) with x86 float->int semantics.
__device__ __forceinline__ float lut_value(const FrameParams& p, float depth) {
    int b = f2i_x86((depth - p.lut_dmin) / p.lut_w);
    if (b < 0) b = 0;
    if (b >= p.lut_n) b = p.lut_n - 1;
    return p.lut_ext ? p.lut_ext[b] : p.lut[b];
}

// eval_color (preprocess.cpp:68-105), coefficient-major SH.
__device__ __forceinline__ void eval_color(const DevScene& sc, uint64_t i, float sh0r, float sh0g,
                                           float sh0b, float dx, float dy, float dz, float* rgb) {
    float r = kShC0 * sh0r, g = kShC0 * sh0g, b = kShC0 * sh0b;
    const int D = sc.sh_coeffs;
    if (D > 1) {
        const float* sh = sc.sh_rest + i * static_cast<uint64_t>((D - 1) * 3) - 3;  // sh[k*3+c], k>=1
        auto acc = [&](float w, int k) {
            r += w * sh[k * 3 + 0];
            g += w * sh[k * 3 + 1];
            b += w * sh[k * 3 + 2];
        };
        const float x = dx, y = dy, z = dz;
        acc(-kShC1 * y, 1);
        acc(kShC1 * z, 2);
        acc(-kShC1 * x, 3);
        if (D > 4) {
            const float xx = x * x, yy = y * y, zz = z * z;
            const float xy = x * y, yz = y * z, xz = x * z;
            acc(kShC2[0] * xy, 4);
            acc(kShC2[1] * yz, 5);
            acc(kShC2[2] * (2.0f * zz - xx - yy), 6);
            acc(kShC2[3] * xz, 7);
            acc(kShC2[4] * (xx - yy), 8);
            if (D > 9) {
                acc(kShC3[0] * y * (3.0f * xx - yy), 9);
                acc(kShC3[1] * xy * z, 10);
                acc(kShC3[2] * y * (4.0f * zz - xx - yy), 11);
                acc(kShC3[3] * z * (2.0f * zz - 3.0f * xx - 3.0f * yy), 12);
                acc(kShC3[4] * x * (4.0f * zz - xx - yy), 13);
                acc(kShC3[5] * z * (xx - yy), 14);
                acc(kShC3[6] * x * (xx - 3.0f * yy), 15);
            }
        }
    }
    rgb[0] = sclamp(r + 0.5f, 0.0f, 1.0f);
    rgb[1] = sclamp(g + 0.5f, 0.0f, 1.0f);
    rgb[2] = sclamp(b + 0.5f, 0.0f, 1.0f);
}

// project (preprocess.cpp:26-66) from the camera-space offset d = mean -
// position: false when behind the near plane or outside the guard band
// (preprocess.cpp:31-39); else the 2D mean (float) and the EWA covariance
// upper 2x2 of J W Sigma W^T J^T + 0.3 I (double, cast to float).
__device__ __forceinline__ bool project_dev(const FrameParams& p, float dx, float dy, float dz, float4 q, float4 sr,
                                            float& tz_out, float& m2x, float& m2y, float& cxx, float& cxy,
                                            float& cyy) {
    // to_camera (scene.hpp:41-43, Mat3f*Vec3f math.hpp:43-49)
    const float tx = p.R[0] * dx + p.R[1] * dy + p.R[2] * dz;
    const float ty = p.R[3] * dx + p.R[4] * dy + p.R[5] * dz;
    const float tz = p.R[6] * dx + p.R[7] * dy + p.R[8] * dz;
    tz_out = tz;
    if (tz <= p.near_plane) return false;
    {
        const float inv_z = 1.0f / tz;
        m2x = p.fx * tx * inv_z + p.ppx;
        m2y = p.fy * ty * inv_z + p.ppy;
        const float ndc_x = (m2x - p.ppx) / p.ppx;
        const float ndc_y = (m2y - p.ppy) / p.ppy;
        if (fabsf(ndc_x) > p.guard || fabsf(ndc_y) > p.guard) return false;
    }
    // Jacobian at the clamped point, double precision (preprocess.cpp:42-57)
    const double iz = 1.0 / static_cast<double>(tz);
    const double txc = sclampd(tx * iz, -p.lim_x, p.lim_x) * tz;
    const double tyc = sclampd(ty * iz, -p.lim_y, p.lim_y) * tz;
    const double j00 = p.fxd * iz, j01 = 0.0, j02 = -p.fxd * txc * iz * iz;
    const double j10 = 0.0, j11 = p.fyd * iz, j12 = -p.fyd * tyc * iz * iz;
    // jw = J * W  (rows 0, 1; Mat3 product math.hpp:50-59, s = 0 then +=)
    double jw[2][3];
    for (int c = 0; c < 3; ++c) {
        const double w0 = p.Rd[c], w1 = p.Rd[3 + c], w2 = p.Rd[6 + c];
        double s = 0.0;
        s += j00 * w0;
        s += j01 * w1;
        s += j02 * w2;
        jw[0][c] = s;
        s = 0.0;
        s += j10 * w0;
        s += j11 * w1;
        s += j12 * w2;
        jw[1][c] = s;
    }
    // covariance_3d (scene.cpp:31-39) with rotation_matrix<double> (math.hpp:147-164)
    const double n = sqrt(static_cast<double>(q.x) * q.x + static_cast<double>(q.y) * q.y +
                          static_cast<double>(q.z) * q.z + static_cast<double>(q.w) * q.w);
    const double qw = q.x / n, qx = q.y / n, qy = q.z / n, qz = q.w / n;
    double rs[9];
    rs[0] = 1 - 2 * (qy * qy + qz * qz);
    rs[1] = 2 * (qx * qy - qw * qz);
    rs[2] = 2 * (qx * qz + qw * qy);
    rs[3] = 2 * (qx * qy + qw * qz);
    rs[4] = 1 - 2 * (qx * qx + qz * qz);
    rs[5] = 2 * (qy * qz - qw * qx);
    rs[6] = 2 * (qx * qz - qw * qy);
    rs[7] = 2 * (qy * qz + qw * qx);
    rs[8] = 1 - 2 * (qx * qx + qy * qy);
    for (int row = 0; row < 3; ++row) {
        rs[row * 3 + 0] *= sr.x;
        rs[row * 3 + 1] *= sr.y;
        rs[row * 3 + 2] *= sr.z;
    }
    double cov[9];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            double s = 0.0;
            s += rs[r * 3 + 0] * rs[c * 3 + 0];
            s += rs[r * 3 + 1] * rs[c * 3 + 1];
            s += rs[r * 3 + 2] * rs[c * 3 + 2];
            cov[r * 3 + c] = s;
        }
    // sigma = (jw * cov) * jw^T, entries (0,0), (0,1), (1,1)
    double t[2][3];
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 3; ++c) {
            double s = 0.0;
            s += jw[r][0] * cov[0 * 3 + c];
            s += jw[r][1] * cov[1 * 3 + c];
            s += jw[r][2] * cov[2 * 3 + c];
            t[r][c] = s;
        }
    double s00 = 0.0, s01 = 0.0, s11 = 0.0;
    s00 += t[0][0] * jw[0][0];
    s00 += t[0][1] * jw[0][1];
    s00 += t[0][2] * jw[0][2];
    s01 += t[0][0] * jw[1][0];
    s01 += t[0][1] * jw[1][1];
    s01 += t[0][2] * jw[1][2];
    s11 += t[1][0] * jw[1][0];
    s11 += t[1][1] * jw[1][1];
    s11 += t[1][2] * jw[1][2];
    cxx = static_cast<float>(s00 + 0.3);
    cxy = static_cast<float>(s01);
    cyy = static_cast<float>(s11 + 0.3);
    return true;
}

// compute_th, Eq. 10 (preprocess.cpp:107-116): K / (T_upper * 2 pi sqrt(det)) + tau
__device__ __forceinline__ float compute_th_dev(float t_upper, float det, float k, float tau) {
    const float denom = t_upper * 2.0f * 3.14159265358979323846f * sqrtf(det);
    return k / denom + tau;
}

}  // namespace

__global__ void __launch_bounds__(256, AGSX_PRE_MINB)
k_preprocess(FrameParams p, DevScene sc, SplatPlanes pl, uint32_t* __restrict__ status,
             uint32_t* __restrict__ dkeys, Counters* ctr, agsx_splat_view* __restrict__ dump, FrameZero fz,
             BucketOut bk) {
    griddep_wait();
    // frame-scoped zeroing (the previous frame's readers have completed)
    // (a block-uniform test first: most blocks have nothing to zero)
    const uint32_t nz = fz.n_tiles > fz.n_chunks ? fz.n_tiles : fz.n_chunks;
    if (blockIdx.x * blockDim.x < nz) {
        for (uint32_t z = blockIdx.x * blockDim.x + threadIdx.x; z < nz; z += gridDim.x * blockDim.x) {
            if (z < fz.n_tiles) {
                fz.ranges[z] = make_uint2(0u, 0u);
                if (fz.tile_pit) fz.tile_pit[z] = 0ull;
            }
            if (z < fz.n_chunks) fz.chunks[z] = 0u;
        }
    }
    const int lane = threadIdx.x & 31;
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;

    // Phase A, one thread per Gaussian: projection, Eq. 10 and the culls.
    // The survivors (a third of the Gaussians at config 3) are queued in
    // shared memory, so phase B -- the tile test, colour, blend-cull data and
    // the stores -- runs on packed warps instead of on the survivors' lanes of
    // every warp.
    __shared__ float s_q[kPreQ][256];  // per survivor slot (structure of arrays)
    __shared__ uint32_t s_slot[256];  // storage slot of each queued survivor
    __shared__ uint32_t s_n;
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    bool ok = false;
    float m2x = 0.0f, m2y = 0.0f, cxx = 0.0f, cxy = 0.0f, cyy = 0.0f, det = 0.0f, th = p.tau, tz = 0.0f;
    float opacity = 0.0f, dx = 0.0f, dy = 0.0f, dz = 0.0f;
    if (i < sc.n) {
        const float4 po = sc.pos_op[i];
        const float4 q = sc.rot[i];
        const float4 sr = sc.scale_r[i];
        opacity = po.w;
        // to_camera (scene.hpp:41-43): t = R (mean - position), float
        dx = po.x - p.cam_pos[0];
        dy = po.y - p.cam_pos[1];
        dz = po.z - p.cam_pos[2];
        ok = project_dev(p, dx, dy, dz, q, sr, tz, m2x, m2y, cxx, cxy, cyy);
        if (ok) {
            det = cxx * cyy - cxy * cxy;
            ok = det > 0.0f;
        }
        if (ok && p.adaptive) {
            th = compute_th_dev(lut_value(p, tz), det, p.k, p.tau);  // Eq. 10
        }
        if (ok && th >= opacity) ok = false;
        if (!ok) {
            status[i] = 0u;
            if (!bk.tile_cnt) dkeys[sc.id_of(static_cast<uint32_t>(i))] = 0xffffffffu;  // keys in id order
        }
    }
    // queue the survivors (converged warp: one shared-memory atomic per warp)
    const uint32_t okb = __ballot_sync(0xffffffffu, ok);
    uint32_t qbase = 0;
    if (lane == 0 && okb) qbase = atomicAdd(&s_n, static_cast<uint32_t>(__popc(okb)));
    qbase = __shfl_sync(0xffffffffu, qbase, 0);
    if (ok) {
        const uint32_t at = qbase + __popc(okb & ((1u << lane) - 1u));
        s_slot[at] = static_cast<uint32_t>(i);
        s_q[0][at] = m2x;
        s_q[1][at] = m2y;
        s_q[2][at] = cxx;
        s_q[3][at] = cxy;
        s_q[4][at] = cyy;
        s_q[5][at] = det;
        s_q[6][at] = opacity;
        s_q[7][at] = th;
        s_q[8][at] = tz;
        s_q[9][at] = dx;
        s_q[10][at] = dy;
        s_q[11][at] = dz;
    }
    __syncthreads();
    const uint32_t ns = s_n;
    if (threadIdx.x == 0 && ns) atomicAdd(&ctr->s, ns);  // survivors = splat_count

    // Phase B, one thread per queued survivor.
    const uint32_t slot = threadIdx.x;
    const bool alive = slot < ns;
    if (!alive && (threadIdx.x & ~31u) >= ns) return;  // whole warps past the queue
    bool keep = false;
    float depth = 0.0f;
    uint4 hit_rec = make_uint4(0u, 0u, 0u, 0u);
    uint32_t gi = 0;  // storage slot of the survivor (DevScene); sc.id_of(gi) is its Gaussian id
    if (alive) {
        gi = s_slot[slot];
        const float m2x = s_q[0][slot], m2y = s_q[1][slot];
        const float cxx = s_q[2][slot], cxy = s_q[3][slot], cyy = s_q[4][slot], det = s_q[5][slot];
        const float opacity = s_q[6][slot], th = s_q[7][slot], tz = s_q[8][slot];
        const float dx = s_q[9][slot], dy = s_q[10][slot], dz = s_q[11][slot];
        uint32_t cnt = 0;
        depth = tz;
        const float inv_det = 1.0f / det;  // SymMat2::inverse (math.hpp:85-88)
        const float ixx = cyy * inv_det, ixy = -cxy * inv_det, iyy = cxx * inv_det;
        const TileTest tt = make_tile_test(m2x, m2y, cxx, cxy, cyy, ixx, ixy, iyy, opacity, th, p);
        const uint4 hits = hit_record(tt, p, cnt);
        hit_rec = hits;
        keep = cnt > 0;
        float rgb[3] = {0.5f, 0.5f, 0.5f};
        if (keep || dump) {
            // Vec3f::normalized (math.hpp:25-28) of mean - cam.position
            const float nrm = sqrtf(dx * dx + dy * dy + dz * dz);
            float ux = 0.0f, uy = 0.0f, uz = 0.0f;
            if (nrm > 0.0f) {
                const float inv = 1.0f / nrm;
                ux = dx * inv;
                uy = dy * inv;
                uz = dz * inv;
            }
            const float2 gb = sc.sh_gb[gi];
            eval_color(sc, gi, sc.scale_r[gi].w, gb.x, gb.y, ux, uy, uz, rgb);
        }
        if (keep) {
            float qcut, qsafe, ex, ey;
            blend_cull_data(ixx, ixy, iyy, opacity, p.tau, p.aclamp, qcut, qsafe, ex, ey);
            pl.p0[gi] = make_float4(m2x, m2y, ixx, 2.0f * ixy);
            pl.p1[gi] = make_float4(iyy, opacity, qcut, qsafe);
            pl.p2[gi] = make_float4(rgb[0], rgb[1], rgb[2], __uint_as_float(pack_extent(ex, ey)));
            if (p.mode == AGSX_MODE_OBB) pl.p4[gi] = make_float4(tt.v1x, tt.v1y, tt.a, tt.b);
            if (bk.tile_cnt) {
                // tile histogram of the bucketed sort, counted in slice gid %
                // kTileSlices of each hit tile (fire-and-forget reductions)
                const uint32_t slice = gi % kTileSlices;
                hit_tiles(tt, p, hits, [&](int tx, int ty) {
                    atomicAdd(&bk.tile_cnt[static_cast<uint32_t>(ty * p.tiles_x + tx) * kTileSlices + slice], 1u);
                });
            } else {
                reinterpret_cast<uint4*>(pl.p3)[gi] = hits;
            }
        }
        if (dump) {
            agsx_splat_view v;
            v.mean2d[0] = m2x;
            v.mean2d[1] = m2y;
            v.cov2d[0] = cxx;
            v.cov2d[1] = cxy;
            v.cov2d[2] = cyy;
            v.inv_cov[0] = ixx;
            v.inv_cov[1] = ixy;
            v.inv_cov[2] = iyy;
            v.depth = tz;
            v.rgb[0] = rgb[0];
            v.rgb[1] = rgb[1];
            v.rgb[2] = rgb[2];
            v.opacity = opacity;
            v.th = th;
            v.source_id = sc.id_of(gi);  // dumps are in Gaussian-id order
            dump[v.source_id] = v;
        }
        status[gi] = cnt | kAliveBit;
    }

    if (bk.tile_cnt) {
        // compact list of the splats with tiles (order irrelevant: one
        // atomic per warp), which is also m
        const uint32_t kb = __ballot_sync(0xffffffffu, keep);
        uint32_t base = 0;
        if (lane == 0 && kb) base = atomicAdd(&ctr->m, static_cast<uint32_t>(__popc(kb)));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) {
            const uint32_t at = base + __popc(kb & ((1u << lane) - 1u));
            bk.gd[at] = make_uint2(gi, __float_as_uint(depth));  // storage slot (the tile sort orders ties by id)
            bk.hits[at] = hit_rec;
        }
        return;
    }
    // the depth keys in Gaussian-id order: the first depth pass reads them
    // in order (equal depths keep id order) with the storage slots as values
    if (alive) dkeys[sc.id_of(gi)] = keep ? __float_as_uint(depth) : 0xffffffffu;
    // range of the depth keys (positive floats: bit order = value order), so
    // the depth sort can skip its top digit when the keys span < 2^24.  Per
    // warp, and an atomic only when it improves on the value last seen (the
    // counters only grow), so neither a block barrier nor contended atomics.
    {
        const uint32_t kb = __float_as_uint(depth);
        const uint32_t wmax = __reduce_max_sync(0xffffffffu, keep ? kb : 0u);
        const uint32_t wminc = __reduce_max_sync(0xffffffffu, keep ? ~kb : 0u);
        if (lane == 0 && wminc) {  // wminc = 0: no splat of this warp has a tile
            if (wmax > *reinterpret_cast<volatile uint32_t*>(&ctr->kmax)) atomicMax(&ctr->kmax, wmax);
            if (wminc > *reinterpret_cast<volatile uint32_t*>(&ctr->kmin_c)) atomicMax(&ctr->kmin_c, wminc);
        }
    }
}

// ---- exported helpers (agsx_project / agsx_eval_color / agsx_compute_th):
// the device functions K1 uses, one element per thread.

// project (preprocess.cpp:26-66): valid[i] and {mean2d.x, mean2d.y, cov2d.xx,
// cov2d.xy, cov2d.yy, depth} per Gaussian.
__global__ void k_project(FrameParams p, DevScene sc, uint8_t* __restrict__ valid, float* __restrict__ out) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // Gaussian id
    if (i >= sc.n) return;
    const uint32_t si = sc.slot_of(static_cast<uint32_t>(i));
    const float4 po = sc.pos_op[si];
    const float dx = po.x - p.cam_pos[0], dy = po.y - p.cam_pos[1], dz = po.z - p.cam_pos[2];
    float tz = 0.0f, m2x = 0.0f, m2y = 0.0f, cxx = 0.0f, cxy = 0.0f, cyy = 0.0f;
    const bool ok = project_dev(p, dx, dy, dz, sc.rot[si], sc.scale_r[si], tz, m2x, m2y, cxx, cxy, cyy);
    valid[i] = ok ? 1u : 0u;
    float* o = out + 6 * i;
    o[0] = m2x;
    o[1] = m2y;
    o[2] = cxx;
    o[3] = cxy;
    o[4] = cyy;
    o[5] = tz;
}

// eval_color (preprocess.cpp:68-105) for a caller-given unit view direction.
__global__ void k_eval_color(DevScene sc, const float* __restrict__ dirs, float* __restrict__ rgb) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // Gaussian id
    if (i >= sc.n) return;
    const uint32_t si = sc.slot_of(static_cast<uint32_t>(i));
    const float2 gb = sc.sh_gb[si];
    eval_color(sc, si, sc.scale_r[si].w, gb.x, gb.y, dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2], rgb + 3 * i);
}

// compute_th (preprocess.cpp:107-116) with the frame's LUT, k and tau;
// th = NaN where det(cov2d) <= 0 (the host raises invalid_argument).
__global__ void k_compute_th(FrameParams p, const float* __restrict__ cov, const float* __restrict__ depth,
                             uint64_t n, float* __restrict__ th) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float xx = cov[3 * i], xy = cov[3 * i + 1], yy = cov[3 * i + 2];
    const float det = xx * yy - xy * xy;  // SymMat2::det (math.hpp:83)
    th[i] = det > 0.0f ? compute_th_dev(lut_value(p, depth[i]), det, p.k, p.tau) : __int_as_float(0x7fc00000);
}

// 30-bit Morton code of each mean quantised to 1024 cells per axis.
__device__ __forceinline__ uint32_t morton_spread10(uint32_t v) {
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000ffu;
    v = (v | (v << 8)) & 0x0300f00fu;
    v = (v | (v << 4)) & 0x030c30c3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

__global__ void k_morton_codes(uint64_t n, const float4* __restrict__ pos_op, float3 lo, float3 scale,
                               uint32_t* __restrict__ codes) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 p = pos_op[i];
    auto q = [](float v, float l, float s) {
        const float t = (v - l) * s;  // NaN / inf means land in cell 0 / 1023
        return static_cast<uint32_t>(t > 0.0f ? (t < 1023.0f ? t : 1023.0f) : 0.0f);
    };
    codes[i] = morton_spread10(q(p.x, lo.x, scale.x)) | (morton_spread10(q(p.y, lo.y, scale.y)) << 1) |
               (morton_spread10(q(p.z, lo.z, scale.z)) << 2);
}

// Slot s <- Gaussian order[s]; inv[order[s]] = s.
__global__ void k_permute_scene(uint64_t n, int D, const uint32_t* __restrict__ order,
                                const float4* __restrict__ pos_op, const float4* __restrict__ rot,
                                const float4* __restrict__ scale_r, const float2* __restrict__ sh_gb,
                                const float* __restrict__ sh_rest, float4* pos_op2, float4* rot2, float4* scale_r2,
                                float2* sh_gb2, float* sh_rest2, uint32_t* inv) {
    const uint64_t s = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const uint32_t g = order[s];
    pos_op2[s] = pos_op[g];
    rot2[s] = rot[g];
    scale_r2[s] = scale_r[g];
    sh_gb2[s] = sh_gb[g];
    const int r = 3 * D - 3;
    for (int k = 0; k < r; ++k) sh_rest2[s * r + k] = sh_rest[static_cast<uint64_t>(g) * r + k];
    inv[g] = static_cast<uint32_t>(s);
}

// Scene upload: host SoA (agsx_scene_desc) -> device planes.
__global__ void k_pack_scene(uint64_t n, int D, const float* __restrict__ mean,
                             const float* __restrict__ scale, const float* __restrict__ rot,
                             const float* __restrict__ op, const float* __restrict__ sh,
                             float4* pos_op, float4* rotq, float4* scale_r, float2* sh_gb,
                             float* sh_rest) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    pos_op[i] = make_float4(mean[3 * i], mean[3 * i + 1], mean[3 * i + 2], op[i]);
    rotq[i] = make_float4(rot[4 * i], rot[4 * i + 1], rot[4 * i + 2], rot[4 * i + 3]);
    const float* s = sh + i * 3 * D;
    scale_r[i] = make_float4(scale[3 * i], scale[3 * i + 1], scale[3 * i + 2], s[0]);
    sh_gb[i] = make_float2(s[1], s[2]);
    for (int k = 3; k < 3 * D; ++k) sh_rest[i * (3 * D - 3) + (k - 3)] = s[k];
}

}  // namespace agsx

// k_pairs.cu -- K3 pair emission and K5 tile ranges.
//
//   reference: generate_pairs emit pass  pair_gen.cpp:187-201
//              serial prefix sum         pair_gen.cpp:177-180
//              pack_pair_key             pair_gen.hpp:33-36
//              range scan                pair_sort.cpp:30-42
//
// The fused path emits pairs in depth-sorted splat order (ties by Gaussian
// id), so a stable sort on the tile field alone yields exactly the
// reference's stable (tile, depth, emission order) permutation -- LSD radix
// order with the 32 depth bits sorted once per splat instead of once per
// pair.  The last depth-sort pass writes the tile counts in
// depth order and their per-chunk sums; a one-block scan turns those into
// chunk offsets, so emission needs no look-back.
#include "kernels.cuh"

namespace agsx {

__device__ __forceinline__ TileTest planes_tile_test(const FrameParams& p, const SplatPlanes& pl,
                                                     uint32_t g) {
    const float4 a = pl.p0[g];
    const float iyy = pl.p1[g].x;
    const float4 c = pl.p3[g];
    TileTest t;
    t.mode = p.mode;
    t.cx = a.x;
    t.cy = a.y;
    t.ixx = a.z;
    t.ixy = 0.5f * a.w;  // P0.w holds 2*inv.xy (exact doubling)
    t.iyy = iyy;
    t.rx = c.x;
    t.ry = c.y;
    t.r2 = c.z;
    t.v1x = t.v1y = t.a = t.b = 0.0f;
    if (p.mode == AGSX_MODE_OBB) {
        const float4 e = pl.p4[g];
        t.v1x = e.x;
        t.v1y = e.y;
        t.a = e.z;
        t.b = e.w;
    }
    return t;
}

// Emits f(tx, ty) for the intersected tiles of splat g in row-major order
// from its P3 hit record (mask) or, for spans over 64 tiles, by re-running
// the tile test.
template <class F>
__device__ __forceinline__ void emit_hits_rec(const FrameParams& p, const SplatPlanes& pl, uint32_t g, uint4 r, F&& f) {
    if (r.w != kHitsRecompute) {
        unsigned long long mask = static_cast<unsigned long long>(r.x) | (static_cast<unsigned long long>(r.y) << 32);
        const int tx0 = static_cast<int>(r.z & 0xffffu), ty0 = static_cast<int>(r.z >> 16);
        const int sw = static_cast<int>(r.w);
        if (sw <= 32) {  // row by row: 32-bit bit scans, no row tracking per pair
            const uint32_t rm = sw == 32 ? 0xffffffffu : ((1u << sw) - 1u);
            for (int row = 0; mask; ++row, mask >>= sw) {
                uint32_t bits = static_cast<uint32_t>(mask) & rm;
                while (bits) {
                    const int b = __ffs(bits) - 1;
                    bits &= bits - 1u;
                    f(tx0 + b, ty0 + row);
                }
            }
            return;
        }
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
    const TileTest t = planes_tile_test(p, pl, g);
    for_each_tile_hit(t, p, f);
}

template <class F>
__device__ __forceinline__ void emit_hits(const FrameParams& p, const SplatPlanes& pl, uint32_t g, F&& f) {
    emit_hits_rec(p, pl, g, reinterpret_cast<const uint4*>(pl.p3)[g], f);
}

// Exclusive scan of the per-chunk sums of tile counts (chunk = 256 splats
// of the depth order; written by the last depth-sort pass), the serial
// prefix of generate_pairs (pair_gen.cpp:177-180): chunk offsets, total P
// (saturating at 2^32 - 1) and the capacity flags.  One block.
__global__ void __launch_bounds__(1024)
k_scan_chunks(const uint32_t* __restrict__ chunk_sum, uint32_t* __restrict__ chunk_off, Counters* ctr,
              uint64_t capacity) {
    griddep_wait();
    __shared__ unsigned long long s_warp[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t n = (ctr->m + 255u) / 256u;
    const uint32_t per = (n + blockDim.x - 1) / blockDim.x;
    const uint32_t lo = min(n, tid * per), hi = min(n, lo + per);
    unsigned long long mine = 0;
    for (uint32_t c = lo; c < hi; ++c) mine += chunk_sum[c];
    unsigned long long incl = mine;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const unsigned long long v = s_warp[lane];
        unsigned long long vi = v;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(0xffffffffu, vi, o);
            if (lane >= o) vi += t;
        }
        s_warp[lane] = vi - v;
        if (lane == 31) {
            const uint32_t pt = vi >= 0xffffffffull ? 0xffffffffu : static_cast<uint32_t>(vi);
            ctr->p = pt;
            const bool fits = pt != 0xffffffffu && pt <= capacity;
            ctr->p_eff = fits ? pt : 0u;
            if (!fits) ctr->overflow = 1u;
        }
    }
    __syncthreads();
    unsigned long long run = s_warp[warp] + incl - mine;
    for (uint32_t c = lo; c < hi; ++c) {
        chunk_off[c] = run >= 0xffffffffull ? 0xffffffffu : static_cast<uint32_t>(run);
        run += chunk_sum[c];
    }
}

// Emission in depth order (pair_gen.cpp:187-201): one CTA per 256-splat
// chunk; block scan of the (sorted) tile counts + the chunk offset give each
// splat's first pair; pairs (tile id, Gaussian id) are staged in shared memory
// and written as one contiguous run of the chunk when they fit.
template <int STAGE>
__global__ void __launch_bounds__(256)
k_emit(FrameParams p, const uint32_t* __restrict__ order_wide, const uint32_t* __restrict__ order_narrow,
       const uint32_t* __restrict__ counts_sorted,
       const uint32_t* __restrict__ chunk_off, SplatPlanes pl, uint32_t* __restrict__ tkeys,
       uint32_t* __restrict__ pvals, uint64_t capacity, const Counters* ctr) {
    griddep_wait();
    extern __shared__ __align__(16) uint32_t emit_stage[];  // STAGE tile ids, then STAGE Gaussian ids
    uint32_t* s_tile = emit_stage;
    uint32_t* s_gid = emit_stage + STAGE;
    constexpr int kStage = STAGE;
    __shared__ uint32_t s_warp[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t m = ctr->m;
    if (ctr->p_eff == 0u) return;  // nothing fits (overflow: the host grows the arena and re-runs)
    // the depth order is in the buffer of the last sort pass that ran
    const uint32_t* __restrict__ order = depth_keys_wide(ctr->kmin_c, ctr->kmax) ? order_wide : order_narrow;
    const uint32_t nchunks = (m + 255u) / 256u;
    // chunks are software-pipelined: the depth order and counts of the chunk
    // after next and the P3 records of the next chunk are in flight while a
    // chunk emits (its gathers are otherwise exposed per chunk)
    const uint4* __restrict__ p3 = reinterpret_cast<const uint4*>(pl.p3);
    auto load = [&](uint32_t cc, uint32_t& gg, uint32_t& nn) {
        const uint32_t jj = cc * 256u + tid;
        gg = 0;
        nn = 0;
        if (cc < nchunks && jj < m) {
            gg = order[jj];
            nn = counts_sorted[jj];
        }
    };
    uint32_t g_n, cnt_n, g_nn, cnt_nn;
    load(blockIdx.x, g_n, cnt_n);
    uint4 rec_n = cnt_n ? p3[g_n] : make_uint4(0u, 0u, 0u, 0u);
    load(blockIdx.x + gridDim.x, g_nn, cnt_nn);
    for (uint32_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        const uint32_t g = g_n, cnt = cnt_n;
        const uint4 rec = rec_n;
        g_n = g_nn;
        cnt_n = cnt_nn;
        rec_n = cnt_n ? p3[g_n] : make_uint4(0u, 0u, 0u, 0u);
        load(c + 2 * gridDim.x, g_nn, cnt_nn);
        uint32_t incl = cnt;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        uint32_t wbase = 0, total = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            const uint32_t v = s_warp[w];
            wbase += w < warp ? v : 0u;
            total += v;
        }
        const uint32_t local = wbase + incl - cnt;
        const uint64_t base = chunk_off[c];
        const bool staged = total <= static_cast<uint32_t>(kStage);
        if (cnt) {
            uint32_t at = local;
            emit_hits_rec(p, pl, g, rec, [&](int tx, int ty) {
                const uint32_t tile = static_cast<uint32_t>(ty * p.tiles_x + tx);
                if (staged) {
                    s_tile[at] = tile;
                    s_gid[at] = g;
                } else {
                    tkeys[base + at] = tile;
                    pvals[base + at] = g;
                }
                ++at;
            });
        }
        __syncthreads();
        if (staged)
            for (uint32_t i = tid; i < total; i += 256) {
                tkeys[base + i] = s_tile[i];
                pvals[base + i] = s_gid[i];
            }
        __syncthreads();
    }
}

cudaError_t launch_emit(bool big, int grid, cudaStream_t st, const FrameParams& p, const uint32_t* order,
                        const uint32_t* order_narrow, const uint32_t* counts_sorted, const uint32_t* chunk_off, const SplatPlanes& pl,
                        uint32_t* tkeys, uint32_t* pvals, uint64_t capacity, const Counters* ctr) {
    if (big)
        return launch_pdl(k_emit<kEmitStageBig>, dim3(grid), dim3(256), emit_smem(true), st, p, order, order_narrow,
                          counts_sorted,
                          chunk_off, pl, tkeys, pvals, capacity, ctr);
    return launch_pdl(k_emit<kEmitStageSmall>, dim3(grid), dim3(256), emit_smem(false), st, p, order, order_narrow,
                      counts_sorted,
                      chunk_off, pl, tkeys, pvals, capacity, ctr);
}

cudaError_t emit_configure(bool big, int* occupancy) {
    const void* f = big ? reinterpret_cast<const void*>(k_emit<kEmitStageBig>)
                        : reinterpret_cast<const void*>(k_emit<kEmitStageSmall>);
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(emit_smem(big)));
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occupancy, f, 256, emit_smem(big));
}

// Standalone generate_pairs over a splat list (agsx_generate_pairs):
// planes + tile counts per list entry.
__global__ void k_splats_to_planes(FrameParams p, const agsx_splat_view* __restrict__ splats,
                                   uint64_t n, SplatPlanes pl, uint32_t* __restrict__ counts,
                                   uint32_t* __restrict__ depth_bits) {
    const uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const agsx_splat_view s = splats[j];
    const TileTest t = make_tile_test(s.mean2d[0], s.mean2d[1], s.cov2d[0], s.cov2d[1], s.cov2d[2],
                                      s.inv_cov[0], s.inv_cov[1], s.inv_cov[2], s.opacity, s.th, p);
    uint32_t cnt = 0;
    reinterpret_cast<uint4*>(pl.p3)[j] = hit_record(t, p, cnt);
    counts[j] = cnt;
    depth_bits[j] = __float_as_uint(s.depth);
    float qcut, qsafe, ex, ey;
    blend_cull_data(s.inv_cov[0], s.inv_cov[1], s.inv_cov[2], s.opacity, p.tau, p.aclamp, qcut, qsafe, ex, ey);
    pl.p0[j] = make_float4(s.mean2d[0], s.mean2d[1], s.inv_cov[0], 2.0f * s.inv_cov[1]);
    pl.p1[j] = make_float4(s.inv_cov[2], s.opacity, qcut, qsafe);
    pl.p2[j] = make_float4(s.rgb[0], s.rgb[1], s.rgb[2], __uint_as_float(pack_extent(ex, ey)));
    if (p.mode == AGSX_MODE_OBB) pl.p4[j] = make_float4(t.v1x, t.v1y, t.a, t.b);
}

// Emission in list order (the reference's splat order) with 64-bit keys.
__global__ void k_emit_list(FrameParams p, uint64_t n, SplatPlanes pl,
                            const uint32_t* __restrict__ counts, const uint64_t* __restrict__ offsets,
                            const uint32_t* __restrict__ depth_bits, uint64_t* __restrict__ keys,
                            uint32_t* __restrict__ vals) {
    const uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n || counts[j] == 0) return;
    uint64_t at = offsets[j];
    const uint64_t lo = depth_bits[j];
    emit_hits(p, pl, static_cast<uint32_t>(j), [&](int tx, int ty) {
        keys[at] = (static_cast<uint64_t>(ty * p.tiles_x + tx) << 32) | lo;
        vals[at] = static_cast<uint32_t>(j);
        ++at;
    });
}

// ranges[tile] = [first, last+1) over the tile-sorted pair list; tiles
// without pairs keep the {0,0} written by the frame memset.
__global__ void __launch_bounds__(256)
k_ranges_u32(const uint32_t* __restrict__ keys, const uint32_t* n_dev, uint2* __restrict__ ranges) {
    griddep_wait();
    const uint32_t n = *n_dev;
    const uint32_t nq = (n + 3) / 4;  // 16-byte groups (the key buffer is 16-byte aligned)
    for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < nq; g += gridDim.x * blockDim.x) {
        const uint32_t i0 = 4 * g;
        uint32_t k[6];
        if (i0 + 4 <= n) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(keys) + g);
            k[1] = v.x;
            k[2] = v.y;
            k[3] = v.z;
            k[4] = v.w;
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) k[1 + j] = i0 + j < n ? keys[i0 + j] : 0xffffffffu;
        }
        k[0] = i0 > 0 ? __ldg(&keys[i0 - 1]) : 0xffffffffu;
        k[5] = i0 + 4 < n ? __ldg(&keys[i0 + 4]) : 0xffffffffu;
#pragma unroll
        for (int j = 1; j <= 4; ++j) {
            const uint32_t i = i0 + j - 1;
            if (i >= n) break;
            if (k[j - 1] != k[j] || i == 0) ranges[k[j]].x = i;
            if (k[j + 1] != k[j] || i == n - 1) ranges[k[j]].y = i + 1;
        }
    }
}

// Same over full 64-bit keys (sort_pairs API): tile = key >> 32, ignored
// when >= tile_count (pair_sort.cpp:39).
__global__ void k_ranges_u64(const uint64_t* __restrict__ keys, uint64_t n, uint32_t tile_count,
                             uint2* __restrict__ ranges) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t t = static_cast<uint32_t>(keys[i] >> 32);
        if (t >= tile_count) continue;
        if (i == 0 || static_cast<uint32_t>(keys[i - 1] >> 32) != t)
            ranges[t].x = static_cast<uint32_t>(i);
        if (i == n - 1 || static_cast<uint32_t>(keys[i + 1] >> 32) != t)
            ranges[t].y = static_cast<uint32_t>(i + 1);
    }
}

// alpha_at (rasterizer.hpp:44-50) with glibc expf, for n (splat, pixel
// centre) pairs: the decision function of raster_tile.
__global__ void k_alpha_at(const agsx_splat_view* __restrict__ s, const float* __restrict__ px, uint64_t n,
                           float aclamp, float* __restrict__ alpha) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const agsx_splat_view v = s[i];
    const float dx = px[2 * i] - v.mean2d[0], dy = px[2 * i + 1] - v.mean2d[1];
    const float power = -0.5f * quad_form(v.inv_cov[0], v.inv_cov[1], v.inv_cov[2], dx, dy);
    float a = 0.0f;
    if (!(power > 0.0f)) {
        a = v.opacity * glibc_expf(power);
        a = a < aclamp ? a : aclamp;
    }
    alpha[i] = a;
}

// effective_radius (pair_gen.cpp:11-16): r = sqrt(2 ln(opacity / th)) with
// glibc logf, pixels = r sqrt(max(lambda_max(cov2d), 0)).
__global__ void k_effective_radius(const float* __restrict__ opacity, const float* __restrict__ th,
                                   const float* __restrict__ cov, uint64_t n, float* __restrict__ out) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float r = sqrtf(2.0f * glibc_logf(opacity[i] / th[i]));
    float l1, l2, v1x, v1y;
    eigen_sym2(cov[3 * i], cov[3 * i + 1], cov[3 * i + 2], l1, l2, v1x, v1y);
    out[2 * i] = r;
    out[2 * i + 1] = r * sqrtf(smax(l1, 0.0f));
}

__global__ void k_logf(const float* __restrict__ x, float* __restrict__ y, uint64_t n) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        y[i] = glibc_logf(x[i]);
}

__global__ void k_expf(const float* __restrict__ x, float* __restrict__ y, uint64_t n) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        y[i] = glibc_expf(x[i]);
}

}  // namespace agsx

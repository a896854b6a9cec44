// k_sort.cu -- K4: stable LSD radix sort, reduce-then-scan per 8-bit digit.
//
//   reference: sort_pairs pair_sort.cpp:7-44 (stable LSD, 8-bit digits,
//              8 passes over the 64-bit key, single-threaded)
//
// A pass is three kernels over G contiguous chunks (one CTA per chunk):
//   upsweep    : per-chunk digit counts -> counts[d][c] (digit-major);
//   scan       : column prefix of the count matrix + digit totals;
//   downsweep  : per 2048-key tile: warp-multisplit ranking stable in input
//                order, shared-memory staging, contiguous per-digit runs.
// Keys equal to `sentinel` (when enabled) are dropped by the pass: the first
// depth pass compacts the per-Gaussian key array this way.  `vin == nullptr`
// means value = input index.  The element count may live on the device.
#include "kernels.cuh"

#ifndef AGSX_DS_MINB
#define AGSX_DS_MINB 5  // downsweep CTAs per SM (register cap): 3 -> 5 measured sort 0.216 -> 0.205 ms
#endif

namespace agsx {

namespace {

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K k, int shift) {
    return static_cast<uint32_t>(k >> shift) & 0xffu;
}

// Reads the pass's bias (kmin of the frame's depth keys, or 0) and whether the
// pass runs at all (a 4th depth pass only when the keys span >= 2^24).
__device__ __forceinline__ bool bias_of(const SortBias& sb, uint32_t& bias, bool& wide) {
    bias = 0;
    wide = true;
    if (!sb.kmin_c) return true;
    const uint32_t kmin_c = *sb.kmin_c, kmax = *sb.kmax;
    wide = depth_keys_wide(kmin_c, kmax);
    bias = ~kmin_c;
    return !(sb.only_wide && !wide);
}

// Exclusive scan of one value per thread over a kSortThreads-thread block.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = v;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    uint32_t wbase = 0;
    for (int w = 0; w < warp; ++w) wbase += s_warp[w];
    __syncthreads();
    return wbase + incl - v;
}

}  // namespace

__device__ __forceinline__ void chunk_of(uint64_t n, int G, int c, uint64_t& lo, uint64_t& hi) {
    // chunk length rounded up to whole tiles so every tile but the last is full
    const uint64_t tiles = (n + kSortTile - 1) / kSortTile;
    const uint64_t per = (tiles + G - 1) / G;
    lo = min(n, static_cast<uint64_t>(c) * per * kSortTile);
    hi = min(n, lo + per * kSortTile);
}

// Upsweep: per-chunk 256-bin digit counts -> counts[d][c] (warp-private
// shared histograms).
template <typename K>
__global__ void __launch_bounds__(kSortThreads)
k_upsweep(const K* __restrict__ keys, const uint32_t* n_dev, uint64_t n_host, int shift, int use_sentinel,
          K sentinel, uint32_t* __restrict__ counts, SortBias sb) {
    griddep_wait();
    uint32_t bias;
    bool wide;
    if (!bias_of(sb, bias, wide)) return;
    constexpr int W = kSortThreads / 32;
    __shared__ uint32_t sh[W][256];
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < W * 256; i += kSortThreads) (&sh[0][0])[i] = 0;
    __syncthreads();
    const uint64_t n = n_dev ? *n_dev : n_host;
    uint64_t lo, hi;
    chunk_of(n, gridDim.x, blockIdx.x, lo, hi);
    // a shared-memory atomic per key into the warp's histogram (warp
    // aggregation of equal digits measured slower: its vote/shuffle/vote per
    // key costs more than the rare conflicts it avoids)
    auto count_key = [&](K key, bool ok) {
        if (ok) atomicAdd(&sh[warp][digit_of(static_cast<K>(key - static_cast<K>(bias)), shift)], 1u);
    };
    if constexpr (sizeof(K) == 4) {
        // 32-bit keys: 16-byte loads (4 keys), four in flight per thread
        // (chunks start on whole tiles, so the vectors are aligned)
        const uint64_t hv = lo + ((hi - lo) & ~uint64_t(3));
        constexpr int U = 4;
        for (uint64_t base = lo; base < hv; base += 4 * U * kSortThreads) {
            uint4 q[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t i = base + 4 * (static_cast<uint64_t>(u) * kSortThreads + tid);
                q[u] = i < hv ? *reinterpret_cast<const uint4*>(keys + i) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const bool in = base + 4 * (static_cast<uint64_t>(u) * kSortThreads + tid) < hv;
                const uint32_t e[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    count_key(static_cast<K>(e[j]), in && !(use_sentinel && static_cast<K>(e[j]) == sentinel));
            }
        }
        for (uint64_t base = hv; base < hi; base += kSortThreads) {  // at most 3 keys
            const uint64_t i = base + tid;
            const K key = i < hi ? keys[i] : K(0);
            count_key(key, i < hi && !(use_sentinel && key == sentinel));
        }
    } else {
    constexpr int U = 8;  // keys in flight per thread
    for (uint64_t base = lo; base < hi; base += U * kSortThreads) {
        K k[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = base + u * kSortThreads + tid;
            k[u] = i < hi ? keys[i] : K(0);
            ok[u] = i < hi && !(use_sentinel && k[u] == sentinel);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) count_key(k[u], ok[u]);
    }
    }
    __syncthreads();
    uint32_t c = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) c += sh[w][tid];
    counts[static_cast<uint64_t>(tid) * gridDim.x + blockIdx.x] = c;  // digit-major: columns contiguous
}

// Column scan of the G x 256 count matrix (one block per digit, G <= 1024
// threads): counts[d][c] <- sum_{c' < c} counts[d][c']; totals[d] = column sum.
__global__ void __launch_bounds__(1024)
k_scan_counts(uint32_t* __restrict__ counts, int G, uint32_t* __restrict__ totals, SortBias sb) {
    griddep_wait();
    uint32_t bias;
    bool wide;
    if (!bias_of(sb, bias, wide)) return;
    __shared__ uint32_t s_warp[32];
    const int d = blockIdx.x, c = threadIdx.x, lane = c & 31, warp = c >> 5;
    const uint32_t v = c < G ? counts[static_cast<uint64_t>(d) * G + c] : 0u;
    uint32_t incl = v;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const int nw = (blockDim.x + 31) / 32;
        const uint32_t x = lane < nw ? s_warp[lane] : 0u;
        uint32_t xi = x;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += t;
        }
        if (lane < nw) s_warp[lane] = xi - x;
        if (lane == nw - 1) totals[d] = xi;
    }
    __syncthreads();
    if (c < G) counts[static_cast<uint64_t>(d) * G + c] = s_warp[warp] + incl - v;
}

// Downsweep: CTA c walks its chunk in kSortTile-key tiles: warp multisplit
// ranking (__match_any_sync; stable in input order), shared-memory staging,
// contiguous per-digit runs to global memory at base[d] = (digits below d)
// + (earlier chunks' digit-d keys) + (earlier tiles of this chunk).
template <typename K>
__global__ void __launch_bounds__(kSortThreads, AGSX_DS_MINB)
k_downsweep(const K* __restrict__ kin, const uint32_t* __restrict__ vin, K* __restrict__ kout,
            uint32_t* __restrict__ vout, const uint32_t* n_dev, uint64_t n_host, int shift, int use_sentinel,
            K sentinel, const uint32_t* __restrict__ counts_excl, const uint32_t* __restrict__ totals,
            uint32_t* n_out, SortCountOut co, SortBias sb) {
    griddep_wait();
    uint32_t bias;
    bool wide;
    if (!bias_of(sb, bias, wide)) return;
    if (sb.co_if_narrow && wide) co.src = nullptr;  // a 4th pass follows and emits the counts
    constexpr int W = kSortThreads / 32;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K* s_keys = reinterpret_cast<K*>(smem_raw);
    uint32_t* s_vals = reinterpret_cast<uint32_t*>(s_keys + kSortTile);
    uint32_t(*s_whist)[256] = reinterpret_cast<uint32_t(*)[256]>(s_vals + kSortTile);
    __shared__ uint32_t s_base[256], s_texcl[256], s_pos[256], s_scan[W];
    __shared__ uint32_t s_tile_n;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x;
    const uint64_t n = n_dev ? *n_dev : n_host;

    const uint32_t total = totals[tid];
    const uint32_t dexcl = block_excl_scan(total, s_scan);
    s_base[tid] = dexcl + counts_excl[static_cast<uint64_t>(tid) * gridDim.x + c];
    if (c == 0 && tid == 255 && n_out) *n_out = dexcl + total;  // keys kept
    __syncthreads();

    uint64_t lo64, hi64;
    chunk_of(n, gridDim.x, c, lo64, hi64);
    const uint32_t lo = static_cast<uint32_t>(lo64), hi = static_cast<uint32_t>(hi64);  // n < 2^32
    const uint32_t lanemask_lt = (1u << lane) - 1u;
    for (uint32_t tbase = lo; tbase < hi; tbase += kSortTile) {
        K k[kSortItems];
        uint32_t v[kSortItems];
        uint32_t rank[kSortItems];
        bool ok[kSortItems];
        // a full tile without sentinels (the common case) skips every
        // per-item validity test
        const bool full = !use_sentinel && hi - tbase >= static_cast<uint32_t>(kSortTile);
        const uint32_t wbase = tbase + static_cast<uint32_t>(warp) * 32u * kSortItems + lane;
        if (full) {
#pragma unroll
            for (int it = 0; it < kSortItems; ++it) {
                k[it] = kin[wbase + it * 32];
                v[it] = vin ? vin[wbase + it * 32] : wbase + it * 32;
                ok[it] = true;
            }
        } else {
#pragma unroll
            for (int it = 0; it < kSortItems; ++it) {
                const uint32_t idx = wbase + it * 32;
                ok[it] = idx < hi;
                k[it] = ok[it] ? kin[idx] : K(0);
                v[it] = ok[it] ? (vin ? vin[idx] : idx) : 0u;
                if (use_sentinel && k[it] == sentinel) ok[it] = false;
            }
        }
        for (int d = lane; d < 256; d += 32) s_whist[warp][d] = 0;
        __syncwarp();
        // Warp multisplit, stable in (item, lane) order: the match group of
        // each item from 8 ballots over its digit bits (VOTE latency instead
        // of MATCH.ANY's); each lane reads its digit's running warp count,
        // the group's lowest lane advances it (ordered by __syncwarp).
        uint32_t peers[kSortItems];
#pragma unroll
        for (int it = 0; it < kSortItems; ++it) {
            const uint32_t d = digit_of(static_cast<K>(k[it] - static_cast<K>(bias)), shift);
            uint32_t pm = full ? 0xffffffffu : __ballot_sync(0xffffffffu, ok[it]);
#pragma unroll
            for (int b = 0; b < 8; ++b) pm = ballot_agree(pm, d & (1u << b));
            peers[it] = pm;
        }
#pragma unroll
        for (int it = 0; it < kSortItems; ++it) {
            const uint32_t d = digit_of(static_cast<K>(k[it] - static_cast<K>(bias)), shift);
            const uint32_t lt = peers[it] & lanemask_lt;
            const uint32_t before = s_whist[warp][d];
            rank[it] = before + __popc(lt);
            __syncwarp();  // every peer has read the count before the group leader advances it
            if (ok[it] && lt == 0u) s_whist[warp][d] = before + __popc(peers[it]);
            __syncwarp();
        }
        __syncthreads();
        uint32_t count = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const uint32_t x = s_whist[w][tid];
            s_whist[w][tid] = count;
            count += x;
        }
        const uint32_t texcl = block_excl_scan(count, s_scan);
        s_texcl[tid] = texcl;
        s_pos[tid] = s_base[tid] - texcl;  // output = s_pos[d] + tile-sorted index
        if (tid == kSortThreads - 1) s_tile_n = texcl + count;
        __syncthreads();
#pragma unroll
        for (int it = 0; it < kSortItems; ++it) {
            if (full || ok[it]) {
                const uint32_t d = digit_of(static_cast<K>(k[it] - static_cast<K>(bias)), shift);
                const uint32_t lsi = s_texcl[d] + s_whist[warp][d] + rank[it];
                s_keys[lsi] = k[it];
                s_vals[lsi] = v[it];
            }
        }
        __syncthreads();
        const uint32_t tn = s_tile_n;
        if (!co.src && tn == static_cast<uint32_t>(kSortTile)) {  // a full tile: unrolled, no bounds
#pragma unroll
            for (int j = 0; j < kSortItems; ++j) {
                const uint32_t i = static_cast<uint32_t>(tid + j * kSortThreads);
                const K key = s_keys[i];
                const uint32_t pos = s_pos[digit_of(static_cast<K>(key - static_cast<K>(bias)), shift)] + i;
                kout[pos] = key;
                vout[pos] = s_vals[i];
            }
            s_base[tid] += count;
            __syncthreads();
            continue;
        }
        const uint32_t tn_round = (tn + 31u) & ~31u;  // whole warps for the aggregated atomics
        for (uint32_t i = tid; i < tn_round; i += kSortThreads) {
            const bool act = i < tn;
            uint32_t pos = 0, val = 0;
            if (act) {
                const K key = s_keys[i];
                pos = s_pos[digit_of(static_cast<K>(key - static_cast<K>(bias)), shift)] + i;
                kout[pos] = key;
                val = s_vals[i];
                vout[pos] = val;
            }
            if (co.src) {  // warp-uniform
                const uint32_t c = act ? co.src[val] & kCountMask : 0u;
                if (act) co.out[pos] = c;
                // consecutive i land in a few 256-splat chunks: one atomic per chunk group
                const uint32_t chunk = act ? pos >> 8 : 0xffffffffu;
                const uint32_t peers = __match_any_sync(0xffffffffu, chunk);
                const uint32_t sum = __reduce_add_sync(peers, c);
                if (act && (__ffs(peers) - 1) == lane) atomicAdd(&co.chunk_sum[chunk], sum);
            }
        }
        s_base[tid] += count;
        __syncthreads();
    }
}

template <typename K>
void launch_sort_pass(int grid, size_t smem, cudaStream_t st, const K* kin, const uint32_t* vin, K* kout,
                      uint32_t* vout, const uint32_t* n_dev, uint64_t n_host, int shift, bool use_sentinel,
                      K sentinel, uint32_t* counts, uint32_t* totals, uint32_t* n_out, SortCountOut co,
                      SortBias sb) {
    launch_pdl(k_upsweep<K>, dim3(grid), dim3(kSortThreads), 0, st, kin, n_dev, n_host, shift, use_sentinel ? 1 : 0,
               sentinel, counts, sb);
    launch_pdl(k_scan_counts, dim3(256), dim3((grid + 31) / 32 * 32), 0, st, counts, grid, totals, sb);
    launch_pdl(k_downsweep<K>, dim3(grid), dim3(kSortThreads), smem, st, kin, vin, kout, vout, n_dev, n_host, shift,
               use_sentinel ? 1 : 0, sentinel, counts, totals, n_out, co, sb);
}

template <typename K>
cudaError_t sort_configure(size_t smem, int* occupancy) {
    cudaError_t e = cudaFuncSetAttribute(k_downsweep<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occupancy, k_downsweep<K>, kSortThreads, smem);
}

template void launch_sort_pass<uint32_t>(int, size_t, cudaStream_t, const uint32_t*, const uint32_t*, uint32_t*,
                                         uint32_t*, const uint32_t*, uint64_t, int, bool, uint32_t, uint32_t*,
                                         uint32_t*, uint32_t*, SortCountOut, SortBias);
template void launch_sort_pass<uint64_t>(int, size_t, cudaStream_t, const uint64_t*, const uint32_t*, uint64_t*,
                                         uint32_t*, const uint32_t*, uint64_t, int, bool, uint64_t, uint32_t*,
                                         uint32_t*, uint32_t*, SortCountOut, SortBias);
template cudaError_t sort_configure<uint32_t>(size_t, int*);
template cudaError_t sort_configure<uint64_t>(size_t, int*);

// Digit histograms of `npasses` consecutive 8-bit digits (from bit 0) in one
// read; keys equal to `sentinel` (when enabled) are not counted.  The key
// count may live on the device.
template <typename K>
__global__ void __launch_bounds__(128)
k_hist(const K* __restrict__ keys, const uint32_t* n_dev, uint64_t n_host, int npasses, int use_sentinel,
       K sentinel, uint32_t* __restrict__ hist) {
    // per-warp sub-histograms; a warp whose 32 digits agree adds once
    __shared__ uint32_t sh[4][8][256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 4 * 8 * 256; i += blockDim.x) (&sh[0][0][0])[i] = 0;
    __syncthreads();
    const uint64_t n = n_dev ? *n_dev : n_host;
    constexpr int U = 4;  // keys in flight per thread
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x * U;
    for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * blockDim.x * U; base < n; base += stride) {
        K kk[U];
        bool vv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = base + u * blockDim.x + threadIdx.x;
            kk[u] = i < n ? keys[i] : K(0);
            vv[u] = i < n && !(use_sentinel && kk[u] == sentinel);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const K k = kk[u];
            const bool valid = vv[u];
            const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
            if (!vmask) continue;
            for (int ps = 0; ps < npasses; ++ps) {
                const uint32_t d = digit_of(k, 8 * ps);
                const uint32_t d0 = __shfl_sync(0xffffffffu, d, __ffs(vmask) - 1);
                if (__all_sync(0xffffffffu, !valid || d == d0)) {
                    if (lane == 0) sh[warp][ps][d0] += __popc(vmask);
                } else if (valid) {
                    atomicAdd(&sh[warp][ps][d], 1u);
                }
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < npasses * 256; i += blockDim.x) {
        uint32_t c = 0;
#pragma unroll
        for (int w = 0; w < 4; ++w) c += (&sh[w][0][0])[i];
        if (c) atomicAdd(&hist[i], c);
    }
}

template <typename K>
void launch_hist(int grid, cudaStream_t st, const K* keys, const uint32_t* n_dev, uint64_t n_host, int npasses,
                 bool use_sentinel, K sentinel, uint32_t* hist) {
    k_hist<K><<<grid, 128, 0, st>>>(keys, n_dev, n_host, npasses, use_sentinel ? 1 : 0, sentinel, hist);
}
template void launch_hist<uint32_t>(int, cudaStream_t, const uint32_t*, const uint32_t*, uint64_t, int, bool,
                                    uint32_t, uint32_t*);
template void launch_hist<uint64_t>(int, cudaStream_t, const uint64_t*, const uint32_t*, uint64_t, int, bool,
                                    uint64_t, uint32_t*);

}  // namespace agsx

// k_sort.cu -- K4: stable LSD radix sort, reduce-then-scan per 8-bit digit.
//
//   reference: sort_pairs pair_sort.cpp:7-44 (stable LSD, 8-bit digits,
//              8 passes over the 64-bit key, single-threaded)
//
// A pass is two kernels over G contiguous chunks (one CTA per chunk):
//   upsweep   : per-chunk 256-bin digit histogram -> counts[c][d];
//   downsweep : each CTA derives its global digit bases from the count
//               matrix (column prefix + digit totals, no serial chains),
//               then walks its chunk in 4096-key tiles: warp multisplit
//               ranking (__match_any_sync) stable in input order, shared-
//               memory staging, contiguous per-digit runs to global memory.
// Keys equal to `sentinel` (when enabled) are dropped by the pass: the first
// depth pass compacts the per-Gaussian key array this way.  `vin == nullptr`
// means value = input index.  The element count may live on the device.
#include "kernels.cuh"

namespace agsx {

namespace {

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K k, int shift) {
    return static_cast<uint32_t>(k >> shift) & 0xffu;
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

__device__ __forceinline__ void chunk_of(uint64_t n, int G, int c, uint64_t& lo, uint64_t& hi) {
    // chunk length rounded up to whole tiles so every tile but the last is full
    const uint64_t tiles = (n + kSortTile - 1) / kSortTile;
    const uint64_t per = (tiles + G - 1) / G;
    lo = min(n, static_cast<uint64_t>(c) * per * kSortTile);
    hi = min(n, lo + per * kSortTile);
}

}  // namespace

template <typename K>
__global__ void __launch_bounds__(kSortThreads)
k_upsweep(const K* __restrict__ keys, const uint32_t* n_dev, uint64_t n_host, int shift, int use_sentinel,
          K sentinel, uint32_t* __restrict__ counts, uint32_t* __restrict__ totals) {
    __shared__ uint32_t hist[256];
    const int tid = threadIdx.x, lane = tid & 31;
    hist[tid] = 0;
    __syncthreads();
    const uint64_t n = n_dev ? *n_dev : n_host;
    uint64_t lo, hi;
    chunk_of(n, gridDim.x, blockIdx.x, lo, hi);
    constexpr int U = 16;  // keys in flight per thread
    for (uint64_t base = lo; base < hi; base += U * kSortThreads) {
        K k[U];
        bool valid[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = base + u * kSortThreads + tid;
            valid[u] = i < hi;
            k[u] = valid[u] ? keys[i] : K(0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const bool ok = valid[u] && !(use_sentinel && k[u] == sentinel);
            const uint32_t d = digit_of(k[u], shift);
            const uint32_t peers = __match_any_sync(0xffffffffu, ok ? d : 0x100u + lane);
            if (ok && (__ffs(peers) - 1) == lane) atomicAdd(&hist[d], __popc(peers));
        }
    }
    __syncthreads();
    counts[static_cast<uint64_t>(blockIdx.x) * 256 + tid] = hist[tid];
    if (hist[tid]) atomicAdd(&totals[tid], hist[tid]);
}

template <typename K>
__global__ void __launch_bounds__(kSortThreads)
k_downsweep(const K* __restrict__ kin, const uint32_t* __restrict__ vin, K* __restrict__ kout,
            uint32_t* __restrict__ vout, const uint32_t* n_dev, uint64_t n_host, int shift, int use_sentinel,
            K sentinel, const uint32_t* __restrict__ counts, const uint32_t* __restrict__ totals,
            uint32_t* n_out) {
    constexpr int W = kSortThreads / 32;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K* s_keys = reinterpret_cast<K*>(smem_raw);
    uint32_t* s_vals = reinterpret_cast<uint32_t*>(s_keys + kSortTile);
    uint32_t(*s_whist)[256] = reinterpret_cast<uint32_t(*)[256]>(s_vals + kSortTile);
    __shared__ uint32_t s_base[256], s_texcl[256], s_pos[256], s_scan[W];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, c = blockIdx.x;
    const uint64_t n = n_dev ? *n_dev : n_host;

    // global base of digit `tid` for this chunk: digits below + earlier chunks
    const uint32_t total = totals[tid];
    uint32_t before = 0;
#pragma unroll 8
    for (int cc = 0; cc < c; ++cc) before += counts[static_cast<uint64_t>(cc) * 256 + tid];
    const uint32_t dexcl = block_excl_scan(total, s_scan);
    s_base[tid] = dexcl + before;
    if (c == 0 && tid == 255 && n_out) *n_out = dexcl + total;  // surviving keys
    __syncthreads();

    uint64_t lo, hi;
    chunk_of(n, G, c, lo, hi);
    for (uint64_t tbase = lo; tbase < hi; tbase += kSortTile) {
        K k[kSortItems];
        uint32_t v[kSortItems];
        uint32_t rank[kSortItems];
        bool ok[kSortItems];
        const uint64_t wbase = tbase + static_cast<uint64_t>(warp) * 32 * kSortItems;
#pragma unroll
        for (int it = 0; it < kSortItems; ++it) {
            const uint64_t idx = wbase + it * 32 + lane;
            ok[it] = idx < hi;
            k[it] = ok[it] ? kin[idx] : K(0);
            v[it] = ok[it] ? (vin ? vin[idx] : static_cast<uint32_t>(idx)) : 0u;
            if (use_sentinel && k[it] == sentinel) ok[it] = false;
        }
        for (int d = lane; d < 256; d += 32) s_whist[warp][d] = 0;
        __syncwarp();
        // warp multisplit: the lowest lane of each digit group bumps the
        // warp's counter and gets the old value back; shared-memory atomics
        // of one warp execute in issue order, so ranks follow (item, lane).
#pragma unroll
        for (int it = 0; it < kSortItems; ++it) {
            const uint32_t d = digit_of(k[it], shift);
            const uint32_t peers = __match_any_sync(0xffffffffu, ok[it] ? d : 0x100u + lane);
            const int leader = __ffs(peers) - 1;
            uint32_t old = 0;
            if (ok[it] && leader == lane) old = atomicAdd(&s_whist[warp][d], __popc(peers));
            rank[it] = __popc(peers & ((1u << lane) - 1u));
            rank[it] += __shfl_sync(0xffffffffu, old, leader);
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
        __syncthreads();
#pragma unroll
        for (int it = 0; it < kSortItems; ++it) {
            if (ok[it]) {
                const uint32_t d = digit_of(k[it], shift);
                const uint32_t lsi = s_texcl[d] + s_whist[warp][d] + rank[it];
                s_keys[lsi] = k[it];
                s_vals[lsi] = v[it];
            }
        }
        __syncthreads();
        const uint32_t tile_n = texcl + count;  // valid keys in this tile (thread 255 holds it)
        __shared__ uint32_t s_tile_n;
        if (tid == kSortThreads - 1) s_tile_n = tile_n;
        __syncthreads();
        for (uint32_t i = tid; i < s_tile_n; i += kSortThreads) {
            const K key = s_keys[i];
            const uint32_t pos = s_pos[digit_of(key, shift)] + i;
            kout[pos] = key;
            vout[pos] = s_vals[i];
        }
        s_base[tid] += count;
        __syncthreads();
    }
}

template <typename K>
void launch_sort_pass(int grid, size_t smem, cudaStream_t st, const K* kin, const uint32_t* vin, K* kout,
                      uint32_t* vout, const uint32_t* n_dev, uint64_t n_host, int shift, bool use_sentinel,
                      K sentinel, uint32_t* counts, uint32_t* totals, uint32_t* n_out) {
    k_upsweep<K><<<grid, kSortThreads, 0, st>>>(kin, n_dev, n_host, shift, use_sentinel ? 1 : 0, sentinel, counts,
                                                totals);
    k_downsweep<K><<<grid, kSortThreads, smem, st>>>(kin, vin, kout, vout, n_dev, n_host, shift,
                                                     use_sentinel ? 1 : 0, sentinel, counts, totals, n_out);
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
                                         uint32_t*, uint32_t*);
template void launch_sort_pass<uint64_t>(int, size_t, cudaStream_t, const uint64_t*, const uint32_t*, uint64_t*,
                                         uint32_t*, const uint32_t*, uint64_t, int, bool, uint64_t, uint32_t*,
                                         uint32_t*, uint32_t*);
template cudaError_t sort_configure<uint32_t>(size_t, int*);
template cudaError_t sort_configure<uint64_t>(size_t, int*);

// Digit histograms of all passes in one read (standalone sort: skip passes
// whose digit is shared by every key).
template <typename K>
__global__ void __launch_bounds__(256)
k_hist(const K* __restrict__ keys, uint64_t n, int npasses, uint32_t* __restrict__ hist) {
    __shared__ uint32_t sh[8][256];
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * blockDim.x; base < n;
         base += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t i = base + threadIdx.x;
        const bool valid = i < n;
        const K k = valid ? keys[i] : K(0);
        for (int ps = 0; ps < npasses; ++ps) {
            const uint32_t d = digit_of(k, 8 * ps);
            const uint32_t peers = __match_any_sync(0xffffffffu, valid ? d : 0x100u + lane);
            if (valid && (__ffs(peers) - 1) == lane) atomicAdd(&sh[ps][d], __popc(peers));
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < npasses * 256; i += blockDim.x) {
        const uint32_t c = (&sh[0][0])[i];
        if (c) atomicAdd(&hist[i], c);
    }
}

void launch_hist64(int grid, cudaStream_t st, const uint64_t* keys, uint64_t n, int npasses, uint32_t* hist) {
    k_hist<uint64_t><<<grid, 256, 0, st>>>(keys, n, npasses, hist);
}

}  // namespace agsx

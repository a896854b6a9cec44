// k_sort.cu -- K4: stable LSD radix sort, onesweep style (one read + one
// write of keys and values per 8-bit digit pass).
//
//   reference: sort_pairs pair_sort.cpp:7-44 (stable LSD, 8-bit digits,
//              8 passes over the 64-bit key, single-threaded)
//
// Per pass, a persistent grid takes 4096-key tiles from an atomic counter;
// each tile ranks its keys with warp-level multisplit (__match_any_sync),
// publishes its 256 digit counts and resolves its global digit offsets by
// decoupled look-back over the preceding tiles (one look-back chain per
// digit, one thread per digit), then scatters through shared memory so the
// global writes are contiguous runs per digit.  Global digit bases come
// from an up-front histogram of all passes (k_hist).
#include "kernels.cuh"

namespace agsx {

namespace {

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K k, int shift) {
    return static_cast<uint32_t>(k >> shift) & 0xffu;
}

// Exclusive scan of one value per thread over a 256-thread block.
__device__ __forceinline__ uint32_t block_excl_scan256(uint32_t v, uint32_t* s_warp) {
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

// Histograms of `npasses` consecutive 8-bit digits starting at first_shift.
template <typename K>
__global__ void __launch_bounds__(256)
k_hist(const K* __restrict__ keys, const uint32_t* n_dev, uint64_t n_host, int first_shift,
       int npasses, uint32_t* __restrict__ hist) {
    __shared__ uint32_t sh[8][256];
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
    __syncthreads();
    const uint64_t n = n_dev ? *n_dev : n_host;
    const int lane = threadIdx.x & 31;
    for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * blockDim.x; base < n;
         base += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t i = base + threadIdx.x;
        const bool valid = i < n;
        const K k = valid ? keys[i] : K(0);
        for (int ps = 0; ps < npasses; ++ps) {
            const uint32_t d = digit_of(k, first_shift + 8 * ps);
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

template <typename K>
__global__ void __launch_bounds__(kSortThreads)
k_onesweep(const K* __restrict__ kin, const uint32_t* __restrict__ vin, K* __restrict__ kout,
           uint32_t* __restrict__ vout, const uint32_t* n_dev, uint64_t n_host, int shift,
           const uint32_t* __restrict__ hist, uint64_t* lb, uint32_t* tile_ctr, uint32_t epoch) {
    constexpr int W = kSortThreads / 32;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K* s_keys = reinterpret_cast<K*>(smem_raw);
    uint32_t* s_vals = reinterpret_cast<uint32_t*>(s_keys + kSortTile);
    uint32_t(*s_whist)[256] = reinterpret_cast<uint32_t(*)[256]>(s_vals + kSortTile);
    __shared__ uint32_t s_goff[256], s_texcl[256], s_base[256], s_scan[W];
    __shared__ uint32_t s_tile;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t n = n_dev ? *n_dev : n_host;
    const uint32_t ep = epoch & 0x3fffffffu;
    s_goff[tid] = block_excl_scan256(hist[tid], s_scan);

    while (true) {
        if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
        __syncthreads();
        const uint32_t tile = s_tile;
        const uint64_t base = static_cast<uint64_t>(tile) * kSortTile;
        if (base >= n) break;

        // load: warp w owns keys [base + w*32*ITEMS, +32*ITEMS), item-major
        K k[kSortItems];
        uint32_t v[kSortItems];
        uint32_t rank[kSortItems];
        const uint64_t wbase = base + static_cast<uint64_t>(warp) * 32 * kSortItems;
#pragma unroll
        for (int it = 0; it < kSortItems; ++it) {
            const uint64_t idx = wbase + it * 32 + lane;
            if (idx < n) {
                k[it] = kin[idx];
                v[it] = vin[idx];
            } else {
                k[it] = K(0);
                v[it] = 0;
            }
        }
        for (int d = lane; d < 256; d += 32) s_whist[warp][d] = 0;
        __syncwarp();
        // warp multisplit ranking, stable in (item, lane) order
#pragma unroll
        for (int it = 0; it < kSortItems; ++it) {
            const bool valid = wbase + it * 32 + lane < n;
            const uint32_t d = digit_of(k[it], shift);
            const uint32_t peers = __match_any_sync(0xffffffffu, valid ? d : 0x100u + lane);
            const uint32_t lt = __popc(peers & ((1u << lane) - 1u));
            uint32_t before = 0;
            if (valid) before = s_whist[warp][d];
            rank[it] = before + lt;
            __syncwarp();
            if (valid && lt == 0) s_whist[warp][d] = before + __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        // per digit (thread = digit): warp-exclusive offsets and tile count
        uint32_t count = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const uint32_t c = s_whist[w][tid];
            s_whist[w][tid] = count;
            count += c;
        }
        const uint32_t texcl = block_excl_scan256(count, s_scan);
        s_texcl[tid] = texcl;
        // decoupled look-back on this digit's chain
        uint64_t* my = &lb[static_cast<uint64_t>(tile) * 256 + tid];
        uint32_t gexcl = 0;
        if (tile == 0) {
            lb_store(my, lb_pack(kFlagIncl, epoch, count));
        } else {
            lb_store(my, lb_pack(kFlagAgg, epoch, count));
            int64_t t = static_cast<int64_t>(tile) - 1;
            while (t >= 0) {
                const uint64_t s = lb_load(&lb[static_cast<uint64_t>(t) * 256 + tid]);
                const uint64_t flag = s & (3ull << 62);
                if (flag == 0 || static_cast<uint32_t>((s >> 32) & 0x3fffffffu) != ep) continue;
                gexcl += static_cast<uint32_t>(s);
                if (flag == kFlagIncl) break;
                --t;
            }
            lb_store(my, lb_pack(kFlagIncl, epoch, gexcl + count));
        }
        s_base[tid] = s_goff[tid] + gexcl - texcl;
        __syncthreads();
        // scatter into shared memory in tile-sorted order
#pragma unroll
        for (int it = 0; it < kSortItems; ++it) {
            if (wbase + it * 32 + lane < n) {
                const uint32_t d = digit_of(k[it], shift);
                const uint32_t lsi = s_texcl[d] + s_whist[warp][d] + rank[it];
                s_keys[lsi] = k[it];
                s_vals[lsi] = v[it];
            }
        }
        __syncthreads();
        const uint32_t tile_n = static_cast<uint32_t>(n - base < kSortTile ? n - base : kSortTile);
        for (uint32_t i = tid; i < tile_n; i += kSortThreads) {
            const K key = s_keys[i];
            const uint32_t pos = s_base[digit_of(key, shift)] + i;
            kout[pos] = key;
            vout[pos] = s_vals[i];
        }
        __syncthreads();
    }
}

template <typename K>
void launch_hist(int grid, cudaStream_t st, const K* keys, const uint32_t* n_dev, uint64_t n_host,
                 int first_shift, int npasses, uint32_t* hist) {
    k_hist<K><<<grid, 256, 0, st>>>(keys, n_dev, n_host, first_shift, npasses, hist);
}

template <typename K>
void launch_onesweep(int grid, size_t smem, cudaStream_t st, const K* kin, const uint32_t* vin, K* kout,
                     uint32_t* vout, const uint32_t* n_dev, uint64_t n_host, int shift,
                     const uint32_t* hist, uint64_t* lb, uint32_t* tile_ctr, uint32_t epoch) {
    k_onesweep<K><<<grid, kSortThreads, smem, st>>>(kin, vin, kout, vout, n_dev, n_host, shift, hist, lb,
                                                    tile_ctr, epoch);
}

template <typename K>
cudaError_t onesweep_configure(size_t smem, int* occupancy) {
    cudaError_t e = cudaFuncSetAttribute(k_onesweep<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occupancy, k_onesweep<K>, kSortThreads, smem);
}

template void launch_hist<uint32_t>(int, cudaStream_t, const uint32_t*, const uint32_t*, uint64_t, int, int,
                                    uint32_t*);
template void launch_hist<uint64_t>(int, cudaStream_t, const uint64_t*, const uint32_t*, uint64_t, int, int,
                                    uint32_t*);
template void launch_onesweep<uint32_t>(int, size_t, cudaStream_t, const uint32_t*, const uint32_t*, uint32_t*,
                                        uint32_t*, const uint32_t*, uint64_t, int, const uint32_t*, uint64_t*,
                                        uint32_t*, uint32_t);
template void launch_onesweep<uint64_t>(int, size_t, cudaStream_t, const uint64_t*, const uint32_t*, uint64_t*,
                                        uint32_t*, const uint32_t*, uint64_t, int, const uint32_t*, uint64_t*,
                                        uint32_t*, uint32_t);
template cudaError_t onesweep_configure<uint32_t>(size_t, int*);
template cudaError_t onesweep_configure<uint64_t>(size_t, int*);

}  // namespace agsx

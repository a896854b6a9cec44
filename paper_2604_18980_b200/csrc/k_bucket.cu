// k_bucket.cu -- the tile-bucketed sort path: pairs are scattered straight
// into their tile's segment and each segment is sorted on its own.
//
//   reference: generate_pairs emit pass  pair_gen.cpp:187-201
//              serial prefix sum         pair_gen.cpp:177-180
//              sort_pairs + ranges       pair_sort.cpp:7-44
//
// The reference sorts all P pairs by the 64-bit key (tile << 32 | depth
// bits) with a stable LSD radix sort over pairs emitted in splat order,
// which is Gaussian-id order (preprocess.cpp:158-162, pair_gen.cpp:152-158).
// Its output order is therefore the total order (tile, depth bits, Gaussian
// id).  Here:
//   K1 (k_preprocess) counts the pairs of every tile (one reduction per hit
//      tile) and lists the splats with tiles;
//   K2 (k_tile_scan) scans the tile counts: the ranges, each slice's base
//      offset, P and the capacity check -- the tile offsets ARE the ranges;
//   K3 (k_bucket_scatter) writes every pair's (depth bits << 32 | gid) into
//      its tile's segment through a returning atomic on its slice cursor (the
//      slot order within a segment is arbitrary);
//   K4 (k_tile_sort) sorts each segment by that 64-bit key, which restores
//      the reference's (depth, Gaussian id) order bit for bit, and writes
//      the Gaussian ids for the rasterizer.
// Nothing global is sorted: P pairs are written once and read once, and the
// depth sort of the splats is gone.  K1's histogram is spread over
// kTileSlices counters per tile (slice = gid % kTileSlices).
//
// Per-tile sort: a tile of <= 256 pairs is one warp's register bitonic sort
// of the full 64-bit keys (unique: no tie handling).  Larger tiles are one
// CTA's LSD radix sort on 8-bit digits of (depth - min depth of the tile),
// ranked by warp multisplit (8 ballots per digit), with the keys in
// registers / shared memory up to 2048 pairs and streamed through a global
// ping-pong buffer above; equal depths within such a tile are detected
// afterwards and ordered by Gaussian id (a re-sort with the gid digits first
// when a run is long), so every order is exact.
//
// Measured at config 3: bit-exact, but not faster than the
// depth-then-tile path (the scatter is latency-bound on its scattered
// accesses, the per-tile sort ALU-bound), so it is selected with
// AGSX_SORT=bucket only.
#include "kernels.cuh"

namespace agsx {

namespace {

// Keys of the bucketed path are (depth bits << 32 | storage slot) (DevScene):
// the slot is the rasterizer's value.  The reference orders equal depths by
// Gaussian id, so a tile with equal depths (a few hundred tiles per frame),
// and every tile of the CTA path, is sorted on (depth, id) keys instead:
// id_key() swaps the low word to the id, slot_of_key() swaps it back.
__device__ __forceinline__ uint64_t id_key(uint64_t k, const uint32_t* __restrict__ orig) {
    return orig ? (k & 0xffffffff00000000ull) | orig[static_cast<uint32_t>(k)] : k;
}
__device__ __forceinline__ uint32_t slot_of_key(uint64_t k, const uint32_t* __restrict__ inv) {
    const uint32_t id = static_cast<uint32_t>(k);
    return inv ? inv[id] : id;
}

constexpr int kTSThreads = 256;
constexpr int kTSWarps = kTSThreads / 32;
constexpr int kTSChunks = kWarpSortMax / 32;  // 8 register chunks of 32 keys per lane

__device__ __forceinline__ int digits_for(uint32_t span) {
    return span == 0u ? 0 : (32 - __clz(static_cast<int>(span)) + 7) / 8;
}

// Digit of a pass: bits [shift, shift+8) of (hi word - dmin) or of the low
// word (gid digits), selected by the pass (warp-uniform).
struct PassDigit {
    uint32_t sub;  // dmin for depth digits, 0 for gid digits
    int shift;
    bool hi;
    __device__ __forceinline__ uint32_t operator()(uint64_t k) const {
        const uint32_t w = hi ? static_cast<uint32_t>(k >> 32) - sub : static_cast<uint32_t>(k);
        return (w >> shift) & 0xffu;
    }
};
// digit `ps` of the schedule: gid digits first (ng of them), then depth digits
__device__ __forceinline__ PassDigit pass_digit(int ps, int ng, uint32_t dmin) {
    PassDigit pd;
    pd.hi = ps >= ng;
    pd.sub = pd.hi ? dmin : 0u;
    pd.shift = 8 * (pd.hi ? ps - ng : ps);
    return pd;
}

// Warp multisplit of up to NC*32 keys (k[c] lane-strided, nvalid of them):
// rank[c] = running count of its digit in hist (before this key) + the keys
// of the same digit at lower lanes of the chunk; hist[d] += count.  Stable in
// (chunk, lane) order.  The peers of a key (same digit) come from 8 ballots
// over the digit bits.
template <int NC>
__device__ __forceinline__ void warp_rank(const uint64_t (&k)[NC], int nvalid, PassDigit dg, uint32_t* hist,
                                          uint32_t (&rank)[NC]) {
    const int lane = threadIdx.x & 31;
    const uint32_t lt_mask = (1u << lane) - 1u;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        if (c * 32 >= nvalid) break;  // warp-uniform
        const bool ok = c * 32 + lane < nvalid;
        const uint32_t d = dg(k[c]);
        uint32_t pm = __ballot_sync(0xffffffffu, ok);
#pragma unroll
        for (int b = 0; b < 8; ++b) pm = ballot_agree(pm, d & (1u << b));
        const uint32_t lt = pm & lt_mask;
        const uint32_t before = hist[d];
        rank[c] = before + __popc(lt);
        __syncwarp();
        if (ok && lt == 0u) hist[d] = before + __popc(pm);
        __syncwarp();
    }
}

__device__ __forceinline__ void warp_zero256(uint32_t* hist) {
    const int lane = threadIdx.x & 31;
    uint4* h4 = reinterpret_cast<uint4*>(hist) + 2 * lane;
    h4[0] = make_uint4(0u, 0u, 0u, 0u);
    h4[1] = make_uint4(0u, 0u, 0u, 0u);
    __syncwarp();
}

// New position of the key at sorted index i when its depth ties a
// neighbour: the run of equal depths around i is ordered by the full key (the
// Gaussian id decides).  buf: the depth-sorted keys.  Runs longer than
// kMaxTieRun set *long_run (the caller re-sorts with the gid digits).
constexpr int kMaxTieRun = 64;
__device__ __forceinline__ int tie_position(const uint64_t* buf, int n, int i, uint64_t key, bool& long_run) {
    const uint32_t hi = static_cast<uint32_t>(key >> 32);
    int s = i, e = i + 1;
    while (s > 0 && static_cast<uint32_t>(buf[s - 1] >> 32) == hi && i - s < kMaxTieRun) --s;
    while (e < n && static_cast<uint32_t>(buf[e] >> 32) == hi && e - i < kMaxTieRun) ++e;
    if (e - s == 1) return i;
    if (e - s >= kMaxTieRun) long_run = true;
    int r = 0;
    for (int j = s; j < e; ++j) r += buf[j] < key ? 1 : 0;
    return s + r;
}

// One tile of 1 < n <= 32 E pairs by one warp: a bitonic sort of the full
// 64-bit keys (depth bits << 32 | Gaussian id -- unique, so the order is the
// reference's (depth, Gaussian id) order with no tie handling), in registers.
// Lane l holds elements l E .. l E + E - 1, so strides below E are register
// exchanges and the others one shuffle per element; padding keys are
// ~0ull and sort last.  Writes the Gaussian ids in order.
template <int E>
__device__ __forceinline__ void warp_bitonic(uint64_t (&v)[E]) {
    const int lane = threadIdx.x & 31;
    constexpr int N = 32 * E;
#pragma unroll
    for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j < E) {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    if (e & j) continue;
                    const int e2 = e | j;
                    // ascending block: bit k of the element index lane E + e
                    const bool asc = k < E ? (e & k) == 0 : (lane & (k / E)) == 0;
                    const uint64_t a = v[e], b = v[e2];
                    const bool sw = asc ? (b < a) : (a < b);
                    v[e] = sw ? b : a;
                    v[e2] = sw ? a : b;
                }
            } else {
                const int lj = j / E;
                const bool lower = (lane & lj) == 0;
                const bool asc = (lane & (k / E)) == 0;
                const bool take_min = lower == asc;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const uint64_t o = __shfl_xor_sync(0xffffffffu, v[e], lj);
                    const bool lt = o < v[e];
                    v[e] = (lt == take_min) ? o : v[e];
                }
            }
        }
    }
}

// Adjacent equal depths among the first n sorted keys (lane-contiguous).
template <int E>
__device__ __forceinline__ bool warp_sorted_has_tie(const uint64_t (&v)[E], int n) {
    const int lane = threadIdx.x & 31;
    bool tie = false;
#pragma unroll
    for (int e = 0; e + 1 < E; ++e)
        tie |= lane * E + e + 1 < n && (v[e] >> 32) == (v[e + 1] >> 32);
    const uint64_t next = __shfl_down_sync(0xffffffffu, v[0], 1);  // the next lane's first key
    tie |= lane < 31 && lane * E + E < n && (v[E - 1] >> 32) == (next >> 32);
    return __any_sync(0xffffffffu, tie);
}

template <int E>
__device__ __forceinline__ void warp_bitonic_tile(const uint64_t* __restrict__ ekeys, uint32_t* __restrict__ vals,
                                                  uint32_t off, int n, const uint32_t* __restrict__ orig,
                                                  const uint32_t* __restrict__ inv) {
    const int lane = threadIdx.x & 31;
    uint64_t v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = lane * E + e;
        v[e] = i < n ? ekeys[off + i] : ~0ull;
    }
    warp_bitonic<E>(v);
    if (orig && warp_sorted_has_tie<E>(v, n)) {  // equal depths: order them by Gaussian id
#pragma unroll
        for (int e = 0; e < E; ++e)
            if (lane * E + e < n) v[e] = id_key(v[e], orig);
        warp_bitonic<E>(v);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int i = lane * E + e;
            if (i < n) vals[off + i] = slot_of_key(v[e], inv);
        }
        return;
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = lane * E + e;
        if (i < n) vals[off + i] = static_cast<uint32_t>(v[e]);  // the slot
    }
}

// One large tile (n > kWarpSortMax) by the whole CTA.  n <= kCtaSortMax: each
// warp holds a 256-key segment in registers and keys move through the shared
// buffer `sbuf` (2048 keys); larger tiles stream segments of 2048 keys
// through the global ping-pong pair (src, alt), with a digit histogram of the
// whole tile per pass.
__device__ __noinline__ void cta_sort_tile(uint64_t* __restrict__ src, uint64_t* __restrict__ alt,
                                           uint32_t* __restrict__ vals, uint32_t n, uint64_t* sbuf,
                                           uint32_t (*hist)[256], uint32_t* s_base, uint32_t* s_red,
                                           const uint32_t* __restrict__ orig, const uint32_t* __restrict__ inv) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool inreg = n <= static_cast<uint32_t>(kCtaSortMax);
    // depth range and largest gid of the tile; the keys become (depth, id)
    // keys (id_key) so the radix passes and the tie fix-up see Gaussian ids
    uint32_t dmin = 0xffffffffu, dmax = 0u, gmax = 0u;
    for (uint32_t i = tid; i < n; i += kTSThreads) {
        const uint64_t k = id_key(src[i], orig);
        if (orig) src[i] = k;
        dmin = min(dmin, static_cast<uint32_t>(k >> 32));
        dmax = max(dmax, static_cast<uint32_t>(k >> 32));
        gmax = max(gmax, static_cast<uint32_t>(k));
    }
    dmin = __reduce_min_sync(0xffffffffu, dmin);
    dmax = __reduce_max_sync(0xffffffffu, dmax);
    gmax = __reduce_max_sync(0xffffffffu, gmax);
    if (lane == 0) {
        s_red[warp] = dmin;
        s_red[8 + warp] = dmax;
        s_red[16 + warp] = gmax;
    }
    __syncthreads();
    dmin = s_red[0];
    dmax = s_red[8];
    gmax = s_red[16];
    for (int w = 1; w < kTSWarps; ++w) {
        dmin = min(dmin, s_red[w]);
        dmax = max(dmax, s_red[8 + w]);
        gmax = max(gmax, s_red[16 + w]);
    }
    __syncthreads();
    const int nd = digits_for(dmax - dmin);
    int ng = 0;
    uint64_t* cur = src;  // global mode: the current order
    uint64_t* nxt = alt;
    uint64_t k[kTSChunks];
    uint32_t rank[kTSChunks];
    int pos[kTSChunks];  // final position of k[c] (differs from its index only within runs of equal depth)
    const uint32_t seg = static_cast<uint32_t>(warp) * kWarpSortMax;
#pragma unroll
    for (int c = 0; c < kTSChunks; ++c) pos[c] = static_cast<int>(seg) + c * 32 + lane;  // this warp's offset in a 2048-key segment
    if (inreg) {
#pragma unroll
        for (int c = 0; c < kTSChunks; ++c) {
            const uint32_t i = seg + c * 32 + lane;
            k[c] = i < n ? src[i] : 0ull;
        }
    }
    for (int attempt = 0; attempt < 2; ++attempt) {
        const int np = ng + nd;
        for (int ps = 0; ps < np; ++ps) {
            if (!inreg) {
                // digit totals of the whole tile -> running output base per digit
                for (int d = tid; d < 256; d += kTSThreads) hist[0][d] = 0u;
                __syncthreads();
                for (uint32_t i = tid; i < n; i += kTSThreads) atomicAdd(&hist[0][pass_digit(ps, ng, dmin)(cur[i])], 1u);
                __syncthreads();
                const uint32_t v = hist[0][tid];
                uint32_t incl = v;
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += t;
                }
                if (lane == 31) s_red[warp] = incl;
                __syncthreads();
                uint32_t wb = 0;
                for (int w = 0; w < warp; ++w) wb += s_red[w];
                s_base[tid] = wb + incl - v;
                __syncthreads();
            }
            for (uint32_t s0 = 0; s0 < n; s0 += kCtaSortMax) {
                const uint32_t sn = min(n - s0, static_cast<uint32_t>(kCtaSortMax));
                const int nw = static_cast<int>(min(sn - min(sn, seg), static_cast<uint32_t>(kWarpSortMax)));
                if (!inreg) {
#pragma unroll
                    for (int c = 0; c < kTSChunks; ++c) {
                        const uint32_t i = seg + c * 32 + lane;
                        k[c] = i < sn ? cur[s0 + i] : 0ull;
                    }
                }
                warp_zero256(hist[warp]);
                warp_rank<kTSChunks>(k, nw, pass_digit(ps, ng, dmin), hist[warp], rank);
                __syncthreads();
                // digit tid: prefix over warps, segment total
                uint32_t tot = 0;
#pragma unroll
                for (int w = 0; w < kTSWarps; ++w) {
                    const uint32_t x = hist[w][tid];
                    hist[w][tid] = tot;
                    tot += x;
                }
                uint32_t base;
                if (inreg) {
                    uint32_t incl = tot;
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += t;
                    }
                    if (lane == 31) s_red[warp] = incl;
                    __syncthreads();
                    uint32_t wb = 0;
                    for (int w = 0; w < warp; ++w) wb += s_red[w];
                    base = wb + incl - tot;
                } else {
                    base = s_base[tid];
                    s_base[tid] = base + tot;
                }
#pragma unroll
                for (int w = 0; w < kTSWarps; ++w) hist[w][tid] += base;
                __syncthreads();
                uint64_t* out = inreg ? sbuf : nxt;
#pragma unroll
                for (int c = 0; c < kTSChunks; ++c) {
                    if (c * 32 < nw && c * 32 + lane < nw)
                        out[hist[warp][pass_digit(ps, ng, dmin)(k[c])] + rank[c]] = k[c];
                }
                __syncthreads();
                if (inreg) {
#pragma unroll
                    for (int c = 0; c < kTSChunks; ++c) {
                        const uint32_t i = seg + c * 32 + lane;
                        if (i < n) k[c] = sbuf[i];
                    }
                    __syncthreads();
                }
            }
            if (!inreg) {
                uint64_t* t = cur;
                cur = nxt;
                nxt = t;
                __syncthreads();
            }
        }
        if (ng > 0) break;
        // equal adjacent depths anywhere in the tile?
        bool tie = false;
        if (inreg) {
            if (np == 0) {  // nothing was sorted: stage the keys for the neighbour reads
#pragma unroll
                for (int c = 0; c < kTSChunks; ++c) {
                    const uint32_t i = seg + c * 32 + lane;
                    if (i < n) sbuf[i] = k[c];
                }
                __syncthreads();
            }
            for (uint32_t i = tid; i + 1 < n; i += kTSThreads)
                tie |= static_cast<uint32_t>(sbuf[i] >> 32) == static_cast<uint32_t>(sbuf[i + 1] >> 32);
        } else {
            for (uint32_t i = tid; i + 1 < n; i += kTSThreads)
                tie |= static_cast<uint32_t>(cur[i] >> 32) == static_cast<uint32_t>(cur[i + 1] >> 32);
        }
        if (!__syncthreads_or(tie)) break;
        if (inreg) {
            // order the runs of equal depths by Gaussian id (sbuf holds the depth order)
            bool long_run = false;
#pragma unroll
            for (int c = 0; c < kTSChunks; ++c) {
                const uint32_t i = seg + c * 32 + lane;
                if (i < n) pos[c] = tie_position(sbuf, static_cast<int>(n), static_cast<int>(i), k[c], long_run);
            }
            if (!__syncthreads_or(long_run)) break;
#pragma unroll
            for (int c = 0; c < kTSChunks; ++c) pos[c] = static_cast<int>(seg) + c * 32 + lane;
        }
        ng = digits_for(gmax);
        if (ng == 0) break;
    }
    if (inreg) {
#pragma unroll
        for (int c = 0; c < kTSChunks; ++c) {
            const uint32_t i = seg + c * 32 + lane;
            if (i < n) vals[pos[c]] = slot_of_key(k[c], inv);
        }
    } else {
        for (uint32_t i = tid; i < n; i += kTSThreads) vals[i] = slot_of_key(cur[i], inv);
    }
    __syncthreads();
}

}  // namespace

// ---- K2: tile scan --------------------------------------------------------
// The histogram has kTileSlices counters per tile (K1 counts a pair into
// slice gid % kTileSlices), so the scatter's returning atomics spread over
// kTileSlices addresses per tile instead of queueing on one.  One thread per
// tile: the tile's slices are scanned in place into their end offsets (the
// scatter counts down), the tile total gives the range.
__global__ void __launch_bounds__(kTileScanThreads)
k_tile_scan(uint32_t* __restrict__ cnt, uint2* __restrict__ ranges, uint32_t T, Counters* ctr, uint64_t capacity,
            uint64_t* lb, uint32_t epoch, uint32_t* __restrict__ big_list) {
    griddep_wait();
    static_assert(kTileSlices == 8, "two uint4 loads per tile");
    constexpr int kWarps = kTileScanThreads / 32;
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_tile, s_prefix;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(&ctr->tile_ctr[4], 1u);
    __syncthreads();
    const uint32_t blk = s_tile;
    const uint64_t t = static_cast<uint64_t>(blk) * kTileScanThreads + tid;
    uint32_t c[kTileSlices] = {};
    if (t < T) {
        const uint4 a0 = *reinterpret_cast<const uint4*>(cnt + t * kTileSlices);
        const uint4 a1 = *reinterpret_cast<const uint4*>(cnt + t * kTileSlices + 4);
        c[0] = a0.x, c[1] = a0.y, c[2] = a0.z, c[3] = a0.w, c[4] = a1.x, c[5] = a1.y, c[6] = a1.z, c[7] = a1.w;
    }
    uint32_t sum = 0;
#pragma unroll
    for (int i = 0; i < kTileSlices; ++i) sum = sat_add(sum, c[i]);
    uint32_t incl = sum;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl = sat_add(incl, x);
    }
    uint32_t excl = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) excl = 0;
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint32_t v = lane < kWarps ? s_warp[lane] : 0u;
        uint32_t vi = v;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(0xffffffffu, vi, o);
            if (lane >= o) vi = sat_add(vi, x);
        }
        uint32_t ve = __shfl_up_sync(0xffffffffu, vi, 1);
        if (lane == 0) ve = 0;
        const uint32_t agg = __shfl_sync(0xffffffffu, vi, 31);
        const uint32_t prefix = lookback_warp(lb, blk, agg, epoch);
        s_warp[lane] = ve;
        if (lane == 0) s_prefix = prefix;
        if (lane == 0 && blk == gridDim.x - 1) {
            const uint32_t total = sat_add(prefix, agg);
            ctr->p = total;
            const bool fits = total != 0xffffffffu && total <= capacity;
            ctr->p_eff = fits ? total : 0u;
            if (!fits) ctr->overflow = 1u;
        }
    }
    __syncthreads();
    const uint32_t start = sat_add(sat_add(s_prefix, s_warp[warp]), excl);
    if (t < T) {
        // slice i: [base_i, base_i + c_i); the scatter claims slots upward from base_i
        uint32_t run = start;
        uint32_t e[kTileSlices];
#pragma unroll
        for (int i = 0; i < kTileSlices; ++i) {
            e[i] = run;
            run = sat_add(run, c[i]);
        }
        *reinterpret_cast<uint4*>(cnt + t * kTileSlices) = make_uint4(e[0], e[1], e[2], e[3]);
        *reinterpret_cast<uint4*>(cnt + t * kTileSlices + 4) = make_uint4(e[4], e[5], e[6], e[7]);
        ranges[t] = sum ? make_uint2(start, run) : make_uint2(0u, 0u);  // empty tiles: {0, 0} (pair_sort.cpp:30-42)
    }
    // tiles above kWarpSortMax pairs -> big_list (one atomic per warp)
    const bool big = t < T && sum > static_cast<uint32_t>(kWarpSortMax);
    const uint32_t bb = __ballot_sync(0xffffffffu, big);
    if (bb) {
        uint32_t bbase = 0;
        if (lane == 0) bbase = atomicAdd(&ctr->tile_ctr[5], static_cast<uint32_t>(__popc(bb)));
        bbase = __shfl_sync(0xffffffffu, bbase, 0);
        if (big) big_list[bbase + __popc(bb & ((1u << lane) - 1u))] = static_cast<uint32_t>(t);
    }
}

// ---- K3: scatter ------------------------------------------------------------
// Every listed splat writes its (depth bits << 32 | gid) key into each hit
// tile's segment at a slot claimed from its slice counter (one thread per
// splat; the hit mask in groups of 8: a group's atomics are issued back to
// back, then its stores).
__global__ void __launch_bounds__(256)
k_bucket_scatter(FrameParams p, SplatPlanes pl, BucketOut bk, const Counters* ctr, uint64_t* __restrict__ ekeys) {
    griddep_wait();
    if (ctr->p_eff == 0u) return;  // overflow (the host grows the arena and re-runs) or no pairs
    const uint32_t m = ctr->m;
    const uint32_t stride = gridDim.x * blockDim.x;  // the grid covers the scene: one splat per thread
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += stride) {
        const uint4 r = bk.hits[j];
        const uint2 e = bk.gd[j];
        const uint64_t key = (static_cast<uint64_t>(e.y) << 32) | e.x;
        const uint32_t slice = e.x % kTileSlices;  // K1 counted this splat's pairs in that slice
        if (r.w != kHitsRecompute) {
            unsigned long long mask = static_cast<unsigned long long>(r.x) | (static_cast<unsigned long long>(r.y) << 32);
            uint4 rr = r;
            while (mask) {
                rr.x = static_cast<uint32_t>(mask);
                rr.y = static_cast<uint32_t>(mask >> 32);
                uint32_t tl[8], pos[8];
                tiles_of_mask(rr, p.tiles_x, tl);
                const int cnt = min(__popcll(static_cast<long long>(mask)), 8);
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (u < cnt) pos[u] = atomicAdd(&bk.tile_cnt[tl[u] * kTileSlices + slice], 1u);
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (u < cnt) ekeys[pos[u]] = key;
                for (int u = 0; u < cnt; ++u) mask &= mask - 1;  // the group's bits
            }
            continue;
        }
        TileTest t{};  // span over 64 tiles: re-run the test
        const uint32_t es = e.x;  // the list carries storage slots
        const float4 a = pl.p0[es];
        t.mode = p.mode;
        t.cx = a.x;
        t.cy = a.y;
        t.ixx = a.z;
        t.ixy = 0.5f * a.w;
        t.iyy = pl.p1[es].x;
        t.rx = __uint_as_float(r.x);
        t.ry = __uint_as_float(r.y);
        t.r2 = __uint_as_float(r.z);
        t.v1x = t.v1y = t.a = t.b = 0.0f;
        if (p.mode == AGSX_MODE_OBB) {
            const float4 o = pl.p4[es];
            t.v1x = o.x;
            t.v1y = o.y;
            t.a = o.z;
            t.b = o.w;
        }
        hit_tiles(t, p, r, [&](int tx, int ty) {
            const uint32_t tile = static_cast<uint32_t>(ty * p.tiles_x + tx);
            ekeys[atomicAdd(&bk.tile_cnt[tile * kTileSlices + slice], 1u)] = key;
        });
    }
}

// ---- K4: per-tile sort -------------------------------------------------------
__global__ void __launch_bounds__(kTSThreads, 3)
k_tile_sort(uint2* __restrict__ ranges, uint32_t T, uint64_t* __restrict__ ekeys, uint64_t* __restrict__ ekeys2,
            uint32_t* __restrict__ vals, Counters* ctr, const uint32_t* __restrict__ big_list,
            const uint32_t* __restrict__ orig, const uint32_t* __restrict__ inv) {
    griddep_wait();
    __shared__ __align__(16) uint64_t s_keys[kTSWarps * kWarpSortMax];  // 32 KB
    __shared__ __align__(16) uint32_t s_hist[kTSWarps][256];            // 8 KB
    __shared__ uint32_t s_base[256], s_red[32];
    __shared__ uint32_t s_claim;
    const int tid = threadIdx.x, lane = tid & 31;
    if (ctr->p_eff == 0u) {
        // overflow: the scan's offsets are not valid; empty ranges for the raster
        for (uint32_t t = blockIdx.x * blockDim.x + tid; t < T; t += gridDim.x * blockDim.x)
            ranges[t] = make_uint2(0u, 0u);
        return;
    }
    // large tiles first, one CTA each
    const uint32_t n_big = ctr->tile_ctr[5];
    while (true) {
        if (tid == 0) s_claim = atomicAdd(&ctr->tile_ctr[6], 1u);
        __syncthreads();
        const uint32_t b = s_claim;
        __syncthreads();
        if (b >= n_big) break;
        const uint2 r = ranges[big_list[b]];
        cta_sort_tile(ekeys + r.x, ekeys2 + r.x, vals + r.x, r.y - r.x, s_keys, s_hist, s_base, s_red, orig, inv);
    }
    // then one warp per tile, tiles claimed four at a time
    while (true) {
        uint32_t t0 = 0;
        if (lane == 0) t0 = atomicAdd(&ctr->tile_ctr[7], 4u);
        t0 = __shfl_sync(0xffffffffu, t0, 0);
        if (t0 >= T) break;
        uint2 rr = make_uint2(0u, 0u);
        if (lane < 4 && t0 + lane < T) rr = ranges[t0 + lane];
        for (int q = 0; q < 4; ++q) {
            const uint32_t lo = __shfl_sync(0xffffffffu, rr.x, q);
            const uint32_t hi = __shfl_sync(0xffffffffu, rr.y, q);
            const uint32_t n = hi - lo;
            if (n <= 1u) {
                if (n == 1u && lane == 0) vals[lo] = static_cast<uint32_t>(ekeys[lo]);  // the slot
                continue;
            }
            if (n > static_cast<uint32_t>(kWarpSortMax)) continue;  // a CTA sorted it
            const int ni = static_cast<int>(n);
            if (ni <= 32)
                warp_bitonic_tile<1>(ekeys, vals, lo, ni, orig, inv);
            else if (ni <= 64)
                warp_bitonic_tile<2>(ekeys, vals, lo, ni, orig, inv);
            else if (ni <= 128)
                warp_bitonic_tile<4>(ekeys, vals, lo, ni, orig, inv);
            else
                warp_bitonic_tile<8>(ekeys, vals, lo, ni, orig, inv);
        }
    }
}

}  // namespace agsx

// kernels.cuh -- kernel declarations shared between the translation units.
#pragma once
#include "agsx_internal.cuh"

namespace agsx {

// Programmatic dependent launch (PDL): a frame's kernels are launched with
// programmatic stream serialization allowed, so each one's launch and CTA
// setup overlap the tail of its predecessor; every such kernel calls
// griddep_wait() before touching anything its predecessor writes (it then
// sees all of the predecessor's memory operations).  Without PDL the wait is
// a no-op.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
    cudaLaunchConfig_t c{};
    c.gridDim = grid;
    c.blockDim = block;
    c.dynamicSmemBytes = smem;
    c.stream = st;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a[0].val.programmaticStreamSerializationAllowed = 1;
    c.attrs = a;
    c.numAttrs = 1;
    return cudaLaunchKernelEx(&c, kernel, static_cast<KArgs>(args)...);
}

constexpr int kSortThreads = 256;
constexpr int kSortItems = 8;
constexpr int kSortTile = kSortThreads * kSortItems;  // keys per onesweep tile

// Frame-scoped buffers K1 zeroes before any later kernel of the frame reads
// them (instead of memsets ahead of the launch chain).
struct FrameZero {
    uint2* ranges = nullptr;                 // tiles
    unsigned long long* tile_pit = nullptr;  // tiles (units rasterizer)
    uint32_t* chunks = nullptr;              // chunk sums
    uint32_t n_tiles = 0, n_chunks = 0;
};
// Outputs of K1 for the tile-bucketed sort path (all null on the depth-sort
// path): the per-tile pair histogram (fire-and-forget atomics per hit tile)
// and a compact list of the splats with >= 1 tile (hit record + {Gaussian
// id, depth bits}), in no particular order -- the per-tile sort makes the
// final order deterministic.
struct BucketOut {
    uint32_t* tile_cnt = nullptr;  // tiles x kTileSlices pair counts (slice = gid % kTileSlices); zeroed before K1
    uint4* hits = nullptr;         // P3 hit record per listed splat
    uint2* gd = nullptr;           // {storage slot, depth bits} per listed splat (DevScene)
    const uint32_t* orig = nullptr;  // storage slot -> Gaussian id, nullptr: identity
    const uint32_t* inv = nullptr;   // Gaussian id -> storage slot
};
__global__ void k_preprocess(FrameParams p, DevScene sc, SplatPlanes pl, uint32_t* status,
                             uint32_t* dkeys, Counters* ctr, agsx_splat_view* dump, FrameZero fz, BucketOut bk);

// ---- tile-bucketed sort path (k_bucket.cu) ------------------------------
// K2: exclusive scan of the tile histogram (decoupled look-back, 8192 tiles
// per CTA): ranges, the per-tile end offsets for the scatter (in place of the
// counts), P / capacity, and the list of tiles above kWarpSortMax pairs.
constexpr int kWarpSortMax = 256;   // pairs per tile sorted by one warp (keys in registers)
constexpr int kCtaSortMax = 2048;  // ... by one CTA with the keys in registers / shared memory
constexpr int kTileSlices = 8;  // histogram counters per tile (bucketed sort)
constexpr int kTileScanThreads = 256;
constexpr int kTileScanPer = kTileScanThreads;  // tiles per scan CTA (one per thread)
__global__ void k_tile_scan(uint32_t* cnt, uint2* ranges, uint32_t T, Counters* ctr, uint64_t capacity, uint64_t* lb,
                            uint32_t epoch, uint32_t* big_list);
// K3: scatter of (depth bits << 32 | gid) into each tile's segment (one
// returning atomic per pair on the tile's end offset).
__global__ void k_bucket_scatter(FrameParams p, SplatPlanes pl, BucketOut bk, const Counters* ctr,
                                 uint64_t* ekeys);
// K4: per-tile sort of the segment by the 64-bit (depth bits, gid) key --
// the reference's stable (tile, depth, emission order) order -- and the
// Gaussian ids of the sorted segment into vals.
__global__ void k_tile_sort(uint2* ranges, uint32_t T, uint64_t* ekeys, uint64_t* ekeys2, uint32_t* vals,
                            Counters* ctr, const uint32_t* big_list, const uint32_t* orig, const uint32_t* inv);
// Scene storage order (agsx_scene_upload): 30-bit 3D Morton codes of the
// means over their bounding box, then the SoA gathered into code order.
__global__ void k_morton_codes(uint64_t n, const float4* pos_op, float3 lo, float3 scale, uint32_t* codes);
__global__ void k_permute_scene(uint64_t n, int D, const uint32_t* order, const float4* pos_op, const float4* rot,
                                const float4* scale_r, const float2* sh_gb, const float* sh_rest, float4* pos_op2,
                                float4* rot2, float4* scale_r2, float2* sh_gb2, float* sh_rest2, uint32_t* inv);
__global__ void k_pack_scene(uint64_t n, int D, const float* mean, const float* scale,
                             const float* rot, const float* op, const float* sh, float4* pos_op,
                             float4* rotq, float4* scale_r, float2* sh_gb, float* sh_rest);

// K3 scan: exclusive scan of the per-chunk tile-count sums -> chunk offsets,
// total P, capacity check (single block).
__global__ void k_scan_chunks(const uint32_t* chunk_sum, uint32_t* chunk_off, Counters* ctr, uint64_t capacity);
// K3 emit: one CTA per 256-splat chunk of the depth order; up to STAGE pairs
// of a chunk are staged in (dynamic) shared memory and written as one
// contiguous run (the big stage for frames with many pairs per splat).
constexpr int kEmitStageSmall = 3072, kEmitStageBig = 8192;
constexpr size_t emit_smem(bool big) { return 2 * (big ? kEmitStageBig : kEmitStageSmall) * sizeof(uint32_t); }
cudaError_t launch_emit(bool big, int grid, cudaStream_t st, const FrameParams& p, const uint32_t* order,
                        const uint32_t* order_narrow,
                        const uint32_t* counts_sorted, const uint32_t* chunk_off, const SplatPlanes& pl,
                        uint32_t* tkeys, uint32_t* pvals, uint64_t capacity, const Counters* ctr);
cudaError_t emit_configure(bool big, int* occupancy);
__global__ void k_splats_to_planes(FrameParams p, const agsx_splat_view* splats, uint64_t n,
                                   SplatPlanes pl, uint32_t* counts, uint32_t* depth_bits);
__global__ void k_emit_list(FrameParams p, uint64_t n, SplatPlanes pl, const uint32_t* counts,
                            const uint64_t* offsets, const uint32_t* depth_bits, uint64_t* keys,
                            uint32_t* vals);
__global__ void k_ranges_u32(const uint32_t* keys, const uint32_t* n_dev, uint2* ranges);
__global__ void k_ranges_u64(const uint64_t* keys, uint64_t n, uint32_t tile_count, uint2* ranges);

// Templated kernels are launched through host functions defined in the
// translation unit that instantiates them (a template kernel's host stub is
// only registered there).
// One stable LSD pass over digit (key >> shift) & 0xff: upsweep + column
// scan + downsweep over `grid` (<= 1024) chunks.  counts: grid*256 u32
// scratch; totals: 256 u32 scratch.  n_out (optional) receives the number of
// keys kept (sentinels dropped).
// Optional by-product of a pass: out[pos] = src[value] & kCountMask for every
// key written, and chunk_sum[pos >> 8] += that (the per-256-splat sums K3's
// scan needs).  All null = off.
struct SortCountOut {
    const uint32_t* src = nullptr;
    uint32_t* out = nullptr;
    uint32_t* chunk_sum = nullptr;
};
// Depth-key bias of a pass (32-bit keys): digits of (key - kmin), kmin from
// K1's range counters; `only_wide` runs the pass only when the keys span
// >= 2^24 (the 4th depth pass), `co_if_narrow` emits SortCountOut only when
// they do not (the 3rd pass is then the last).
struct SortBias {
    const uint32_t* kmin_c = nullptr;  // nullptr: no bias, always run
    const uint32_t* kmax = nullptr;
    int only_wide = 0;
    int co_if_narrow = 0;
};
template <typename K>
void launch_sort_pass(int grid, size_t smem, cudaStream_t st, const K* kin, const uint32_t* vin, K* kout,
                      uint32_t* vout, const uint32_t* n_dev, uint64_t n_host, int shift, bool use_sentinel,
                      K sentinel, uint32_t* counts, uint32_t* totals, uint32_t* n_out, SortCountOut co = {},
                      SortBias sb = {});
template <typename K>
cudaError_t sort_configure(size_t smem, int* occupancy);
// Histograms of the low `npasses` 8-bit digits into hist[npasses][256]
// (accumulated; zero it first).
template <typename K>
void launch_hist(int grid, cudaStream_t st, const K* keys, const uint32_t* n_dev, uint64_t n_host, int npasses,
                 bool use_sentinel, K sentinel, uint32_t* hist);

void launch_raster_kernel(int ppt, bool exact, bool maxt, int grid, cudaStream_t st, const FrameParams& p,
                          const uint2* ranges, const uint32_t* vals, const float4* P0, const float4* P1,
                          const float4* P2, float* image, uint32_t* maxt_buf, unsigned long long* pit);

// Warp-persistent fast-alpha rasterizer for 16x16 tiles (units = half
// tiles pulled from *unit_ctr, zeroed per frame; tile_pit: one zeroed u64
// per tile).
void launch_raster_units(int grid, cudaStream_t st, const FrameParams& p, const uint2* ranges, const uint32_t* vals,
                         const float4* P0, const float4* P1, const float4* P2, float* image, uint32_t* unit_ctr,
                         unsigned long long* tile_pit, unsigned long long* pit, unsigned long long* dbg,
                         uint32_t* band_done = nullptr, int band_rows = 1, uint8_t* img_u8 = nullptr);
cudaError_t raster_units_occupancy(int* occ);
// raster_tile with the blend-event stream (RecordOptions::contributions): a
// counting pass (out == nullptr, counts per tile) or the writing pass.
cudaError_t launch_raster_records(cudaStream_t st, const FrameParams& p, const uint2* ranges, const uint32_t* vals,
                                  const float4* P0, const float4* P1, const float4* P2, float* image,
                                  uint32_t* counts, const uint64_t* offsets, agsx_blend_record* out);

__global__ void k_fold_max_t(const uint32_t* order, const uint32_t* inv, const uint32_t* dkeys, int stride, const uint32_t* m_dev,
                             const uint32_t* maxt, float dmin, float dmax, int nbins, uint32_t* folded,
                             uint32_t* observed);
__global__ void k_sq_err_partial(const float* a, const float* b, uint64_t n, double* partial);
__global__ void k_sq_err_final(const double* partial, int n, double* out);

__global__ void k_quantize_u8(const float4* img, uint4* dst, uint64_t n16);
__global__ void k_quantize_u8_tail(const float* img, uint8_t* dst, uint64_t lo, uint64_t n);

// exported helpers (agsx_stage_api.cu): the device functions of K1 / pair
// generation / the rasterizer, one element per thread
__global__ void k_project(FrameParams p, DevScene sc, uint8_t* valid, float* out);
__global__ void k_eval_color(DevScene sc, const float* dirs, float* rgb);
__global__ void k_compute_th(FrameParams p, const float* cov, const float* depth, uint64_t n, float* th);
__global__ void k_alpha_at(const agsx_splat_view* s, const float* px, uint64_t n, float aclamp, float* alpha);
__global__ void k_effective_radius(const float* opacity, const float* th, const float* cov, uint64_t n, float* out);

__global__ void k_logf(const float* x, float* y, uint64_t n);
__global__ void k_expf(const float* x, float* y, uint64_t n);

}  // namespace agsx

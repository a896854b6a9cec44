// agsx_frame.cu -- one frame of the render path on a context: validation,
// the launch sequence, host egress and the wait (regrow and re-run).
//
//   reference: render()          rasterizer.cpp:102-165
//              validate(cfg/cam) scene.cpp:41-59, 113-123
//
// A frame is enqueued on the ctx stream without any host synchronisation:
// every data-dependent size (survivors, splats with tiles, pair count) stays
// on the device and the kernels that consume it are persistent grids that
// read it there.  The host reads one small counter block when the caller
// waits for the frame; a pair count above the buffer capacity (but within
// pair_budget) grows the pair arena and re-runs the frame.
#include "agsx_ctx.cuh"

namespace agsx::host {

// ---- validation (scene.cpp:41-59, 113-123) ------------------------------
std::string validate_config(const agsx_config& c) {
    if (!(c.alpha_threshold > 0.0f && c.alpha_threshold < c.alpha_clamp && c.alpha_clamp <= 1.0f))
        return "require 0 < alpha_threshold < alpha_clamp <= 1";
    if (!(c.transmittance_floor > 0.0f)) return "transmittance_floor must be positive";
    if (c.tile_size < 1) return "tile_size must be >= 1";
    if (c.k < 0.0f) return "k must be >= 0";
    if (!(c.near_plane > 0.0f)) return "near_plane must be positive";
    if (c.mode < AGSX_MODE_AABB || c.mode > AGSX_MODE_ADAGSCALE) return "unknown mode";
    return {};
}

std::string validate_camera(const agsx_camera& cam) {
    // orthonormality_drift: max |R^T R - I| with float Mat3 products
    const float* r = cam.rotation;
    float drift = 0.0f;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            float s = 0.0f;
            for (int k = 0; k < 3; ++k) s += r[k * 3 + i] * r[k * 3 + j];
            const float target = (i == j) ? 1.0f : 0.0f;
            drift = smax(drift, std::fabs(s - target));
        }
    if (drift > 1e-5f) return "camera rotation is not orthonormal";
    if (!(cam.fx > 0.0f && cam.fy > 0.0f)) return "focal lengths must be positive";
    if (!(cam.width > 0 && cam.height > 0)) return "image dimensions must be positive";
    return {};
}

int tile_bits(uint32_t tile_count) {
    int b = 0;
    while (b < 32 && (tile_count - 1) >> b) ++b;
    return std::max(b, 1);
}

FrameParams make_params(const agsx_camera& cam, const agsx_config& cfg, const agsx_lut* lut,
                        const float* lut_ext_dev) {
    FrameParams p;
    std::memset(&p, 0, sizeof(p));
    for (int i = 0; i < 3; ++i) p.cam_pos[i] = cam.position[i];
    for (int i = 0; i < 9; ++i) {
        p.R[i] = cam.rotation[i];
        p.Rd[i] = static_cast<double>(cam.rotation[i]);
    }
    p.fx = cam.fx;
    p.fy = cam.fy;
    p.fxd = static_cast<double>(cam.fx);
    p.fyd = static_cast<double>(cam.fy);
    p.W = cam.width;
    p.H = cam.height;
    p.ppx = 0.5f * static_cast<float>(cam.width);
    p.ppy = 0.5f * static_cast<float>(cam.height);
    p.lim_x = cfg.guard_band * 0.5 * cam.width / cam.fx;
    p.lim_y = cfg.guard_band * 0.5 * cam.height / cam.fy;
    p.tile_size = cfg.tile_size;
    p.tiles_x = (cam.width + cfg.tile_size - 1) / cfg.tile_size;
    p.tiles_y = (cam.height + cfg.tile_size - 1) / cfg.tile_size;
    p.mode = cfg.mode;
    p.fixed_aabb = cfg.fixed_radius_aabb ? 1 : 0;
    p.tau = cfg.alpha_threshold;
    p.tfloor = cfg.transmittance_floor;
    p.aclamp = cfg.alpha_clamp;
    p.near_plane = cfg.near_plane;
    p.guard = cfg.guard_band;
    p.k = cfg.k;
    for (int i = 0; i < 3; ++i) p.bg[i] = cfg.background[i];
    p.flags = cfg.flags;
    p.raster_ppt = 4;
    if (const char* e = std::getenv("AGSX_RASTER_PPT")) {
        const int v = std::atoi(e);
        p.raster_ppt = (v == 2 || v == 8) ? v : 4;
    }
    p.adaptive = cfg.mode == AGSX_MODE_ADAGSCALE ? 1 : 0;
    p.lut_dmin = 0.0f;
    p.lut_dmax = 100.0f;
    p.lut_n = 20;
    for (int i = 0; i < 20; ++i) p.lut[i] = 1.0f;
    if (lut && lut->bin_count > 0) {
        p.lut_dmin = lut->depth_min;
        p.lut_dmax = lut->depth_max;
        p.lut_n = lut->bin_count;
        if (lut->bin_count <= kLutInline) {
            for (int i = 0; i < lut->bin_count; ++i) p.lut[i] = lut->bins[i];
        } else {
            p.lut_ext = lut_ext_dev;
        }
    }
    // TUpperLUT::value_at's bin width (lut.hpp:16-25), one IEEE division here
    // instead of one per Gaussian (the host and device quotients are equal)
    p.lut_w = (p.lut_dmax - p.lut_dmin) / static_cast<float>(p.lut_n);
    return p;
}

int raster_ppt(int tile_size) {
    if (tile_size <= 16) return 1;
    if (tile_size <= 32) return 4;
    return 16;
}

bool raster_uses_units(const FrameParams& p, bool maxt) {
    return p.tile_size == 16 && (p.flags & AGSX_FLAG_EXACT_ALPHA) == 0 && !maxt && p.raster_ppt == 4;
}

void launch_raster(agsx_ctx* ctx, const FrameParams& p, const uint2* ranges, const uint32_t* vals,
                   const float4* P0, const float4* P1, const float4* P2, float* image,
                   uint32_t* maxt, Counters* ctr, uint32_t* unit_ctr) {
    const int nsub = (p.tile_size + 63) / 64;  // 64x64 blocks per tile (k_raster)
    const int grid = p.tiles_x * p.tiles_y * nsub * nsub;
    if (grid == 0) return;
    const bool exact = (p.flags & AGSX_FLAG_EXACT_ALPHA) != 0;
    if (raster_uses_units(p, maxt != nullptr)) {
        // default path: warp-persistent units (half tiles); per-tile P_it
        // words (zeroed at the frame start by the caller)
        launch_raster_units(ctx->num_sms * ctx->occ_raster, ctx->stream, p, ranges, vals, P0, P1, P2, image,
                            unit_ctr ? unit_ctr : &ctr->tile_ctr[3], ptr<unsigned long long>(ctx->tile_pit),
                            &ctr->p_it, ctr->dbg);
        check_launch(ctx);
        return;
    }
    launch_raster_kernel(raster_ppt(p.tile_size), exact, maxt != nullptr, grid, ctx->stream, p, ranges, vals,
                         P0, P1, P2, image, maxt, &ctr->p_it);
    check_launch(ctx);
}

size_t sort_smem(bool k64) {
    return (k64 ? 8 : 4) * static_cast<size_t>(kSortTile) + 4 * static_cast<size_t>(kSortTile) +
           (kSortThreads / 32) * 256 * 4;
}

size_t counters_bytes() { return sizeof(Counters); }
// The bucketed path's tile histogram lives right behind the counters, so one
// memset per frame zeroes both.
size_t tile_cnt_offset() { return (sizeof(Counters) + 255) / 256 * 256; }
uint32_t* tile_cnt_of(agsx_ctx* ctx) {
    return reinterpret_cast<uint32_t*>(static_cast<char*>(ctx->ctr.p) + tile_cnt_offset());
}

// Sort path of a frame, both bit-identical: the
// depth-then-tile radix path (default) or the tile-bucketed path of
// k_bucket.cu (AGSX_SORT=bucket).  AGSX_SORT=auto picks per frame: the
// bucketed path when the context's previous frame averaged fewer than
// kBucketMaxPairsPerTile pairs per tile, else the depth path (measured not
// faster at config 3 either way, so not the default).
constexpr double kBucketMaxPairsPerTile = 160.0;
int sort_mode() {  // 0 depth, 1 bucket, 2 auto
    static const int mode = [] {
        const char* e = std::getenv("AGSX_SORT");
        if (e && std::strcmp(e, "bucket") == 0) return 1;
        if (e && std::strcmp(e, "auto") == 0) return 2;
        return 0;
    }();
    return mode;
}
bool may_bucket() { return sort_mode() != 0; }
bool may_depth() { return sort_mode() != 1; }
bool frame_uses_bucket(const agsx_ctx* ctx) {
    const int m = sort_mode();
    if (m != 2) return m == 1;
    return ctx->prev_pairs_per_tile > 0.0 && ctx->prev_pairs_per_tile < kBucketMaxPairsPerTile;
}
// 256-splat chunks of the depth order (K3 work units)
uint64_t chunk_slots(uint64_t n) { return std::max<uint64_t>((n + 255) / 256, 1); }

int sort_grid(agsx_ctx* ctx, bool k64) { return ctx->num_sms * (k64 ? ctx->occ_sort64 : ctx->occ_sort32); }

void ensure_lb(agsx_ctx* ctx, uint64_t max_elems) {
    const uint64_t words = std::max<uint64_t>(max_elems / 256 + 2,
                                              (max_elems / kSortTile + 2) * 256);
    ensure(ctx->lb, words * sizeof(uint64_t), /*zero=*/true);
}

// Arena sizing for a scene of n Gaussians and a frame of `tiles` tiles.
void ensure_frame_buffers(agsx_ctx* ctx, uint64_t n, uint64_t tiles, uint64_t pixels, bool obb,
                          uint64_t pair_budget) {
    ensure(ctx->status, std::max<uint64_t>(n, 1) * 4);
    ensure(ctx->p0, std::max<uint64_t>(n, 1) * 16);
    ensure(ctx->p1, std::max<uint64_t>(n, 1) * 16);
    ensure(ctx->p2, std::max<uint64_t>(n, 1) * 16);
    ensure(ctx->p3, std::max<uint64_t>(n, 1) * 16);
    if (obb) ensure(ctx->p4, std::max<uint64_t>(n, 1) * 16);
    ensure(ctx->dkeys, std::max<uint64_t>(n, 1) * 4);
    ensure(ctx->dvals, std::max<uint64_t>(n, 1) * 4);
    ensure(ctx->dkeys2, std::max<uint64_t>(n, 1) * 4);
    ensure(ctx->dvals2, std::max<uint64_t>(n, 1) * 4);
    ensure(ctx->dcounts, std::max<uint64_t>(n, 1) * 4);
    ensure(ctx->chunks, 2 * chunk_slots(n) * 4);
    ensure(ctx->ranges, std::max<uint64_t>(tiles, 1) * 8);
    ensure(ctx->image, std::max<uint64_t>(pixels, 1) * 12);
    ensure(ctx->ctr, tile_cnt_offset() + std::max<uint64_t>(tiles, 1) * 4 * kTileSlices + 16);
    if (may_bucket()) {
        ensure(ctx->bk_hits, std::max<uint64_t>(n, 1) * 16);
        ensure(ctx->bk_gd, std::max<uint64_t>(n, 1) * 8);
        ensure(ctx->big_list, std::max<uint64_t>(tiles, 1) * 4);
    }
    if (ctx->pair_capacity == 0) {
        // first guess: 12 pairs per Gaussian, at most the budget, at least 1M
        ctx->pair_capacity = std::min<uint64_t>(std::max<uint64_t>(12 * n, 1u << 20),
                                                std::max<uint64_t>(pair_budget, 1));
    }
    const uint64_t cap = ctx->pair_capacity;
    ensure(ctx->pvals, cap * 4);
    if (may_bucket()) {
        ensure(ctx->ekeys, cap * 8);
        ensure(ctx->ekeys2, cap * 8);
    }
    if (may_depth()) {
        ensure(ctx->tkeys, cap * 4);
        ensure(ctx->tkeys2, cap * 4);
        ensure(ctx->pvals2, cap * 4);
    }
    ensure_lb(ctx, std::max(cap, n));
}

SplatPlanes planes_of(agsx_ctx* ctx) {
    SplatPlanes pl;
    pl.p0 = ptr<float4>(ctx->p0);
    pl.p1 = ptr<float4>(ctx->p1);
    pl.p2 = ptr<float4>(ctx->p2);
    pl.p3 = ptr<float4>(ctx->p3);
    pl.p4 = ptr<float4>(ctx->p4);
    return pl;
}

// Validates and resolves the LUT; returns AGSX_OK or EINVAL.
int prepare(agsx_ctx* ctx, const agsx_camera* cam, const agsx_config* cfg, const agsx_lut* lut,
            FrameParams& p) {
    if (!cam || !cfg) return fail(ctx, AGSX_EINVAL, "render: null camera or config");
    std::string bad = validate_config(*cfg);
    if (!bad.empty()) return fail(ctx, AGSX_EINVAL, "render: " + bad);
    bad = validate_camera(*cam);
    if (!bad.empty()) return fail(ctx, AGSX_EINVAL, "render: " + bad);
    if (cfg->mode == AGSX_MODE_ADAGSCALE && lut == nullptr)
        return fail(ctx, AGSX_EINVAL, "preprocess_view: adagscale mode requires a T-upper LUT");
    const float* lut_dev = nullptr;
    if (lut && lut->bin_count > kLutInline) {
        ensure(ctx->lut_ext, lut->bin_count * sizeof(float));
        AGSX_CUDA(cudaMemcpyAsync(ctx->lut_ext.p, lut->bins, lut->bin_count * sizeof(float),
                                  cudaMemcpyHostToDevice, ctx->stream));
        lut_dev = ptr<float>(ctx->lut_ext);
    }
    p = make_params(*cam, *cfg, cfg->mode == AGSX_MODE_ADAGSCALE ? lut : nullptr, lut_dev);
    return AGSX_OK;
}

// Enqueue the whole frame (no host synchronisation).
// cuStreamWaitValue32 through the runtime's driver entry point (no link
// against libcuda): the copy stream waits on the raster's per-band unit
// counts in device memory.  nullptr when the driver does not offer it.
using WaitValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WaitValue32Fn wait_value32() {
    static const WaitValue32Fn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        cudaGetLastError();
        return reinterpret_cast<WaitValue32Fn>(f);
    }();
    return fn;
}

// Host twin of depth_keys_wide: whether the frame's depth order ended in the
// [0] (4 passes) or [1] (3 passes) ping-pong buffers.
bool depth_keys_wide_host(const Counters& c) {
    const uint32_t kmin = ~c.kmin_c;
    return c.kmax >= kmin && c.kmax - kmin >= (1u << 24);
}

// The frame's counter block to the mapped host words, plus the async-chain
// words: this frame overflowed the pair arena when its pairs did not all fit
// (K3 skipped emission); the chain count keeps that after the next frame's
// memset, so a wait on a later frame still sees it.
__global__ void k_counters_out(const uint32_t* __restrict__ src, uint32_t* dst, int words, ChainWords* chain) {
    for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
    if (threadIdx.x == 0) {
        const Counters* c = reinterpret_cast<const Counters*>(src);
        const uint32_t over = (c->overflow != 0u || c->p_eff != c->p) ? 1u : 0u;
        ChainWords w = *chain;
        w.overflowed += over;
        w.frames += 1u;
        *chain = w;
        dst[words] = w.overflowed;
        dst[words + 1] = w.frames;
    }
}

// write_image quantisation of n floats (src, dst 16-byte aligned) on stream st
void launch_quantize(agsx_ctx* ctx, const float* src, uint8_t* dst, uint64_t n, cudaStream_t st) {
    const uint64_t n16 = n / 16;
    if (n16) {
        const int grid = static_cast<int>(std::min<uint64_t>((n16 + 255) / 256, ctx->num_sms * 8));
        k_quantize_u8<<<grid, 256, 0, st>>>(reinterpret_cast<const float4*>(src), reinterpret_cast<uint4*>(dst), n16);
        check_launch(ctx);
    }
    if (n % 16) {
        k_quantize_u8_tail<<<1, 16, 0, st>>>(src, dst, n16 * 16, n);
        check_launch(ctx);
    }
}

void enqueue_bucket_sort(agsx_ctx* ctx, uint64_t n, const FrameParams& p, const BucketOut& bk);
void enqueue_depth_sort(agsx_ctx* ctx, uint64_t n, uint64_t tiles, const FrameParams& p, const SplatPlanes& pl,
                        const uint32_t* scene_inv);
void enqueue_raster(agsx_ctx* ctx, const FrameParams& p, bool maxt, uint32_t* vals);

void enqueue_frame(agsx_ctx* ctx, const agsx_scene* sc, const FrameParams& p, bool maxt,
                   agsx_splat_view* dump) {
    const uint64_t n = sc->n;
    const uint64_t tiles = static_cast<uint64_t>(p.tiles_x) * p.tiles_y;
    Counters* ctr = ptr<Counters>(ctx->ctr);
    cudaStream_t st = ctx->stream;
    ctx->ev = ctx->ev_ring[ctx->frames % agsx_ctx::kRing];
    ++ctx->frames;

    const bool bucket = frame_uses_bucket(ctx);
    AGSX_CUDA(cudaEventRecord(ctx->ev[0], st));
    AGSX_CUDA(cudaMemsetAsync(ctr, 0, bucket ? tile_cnt_offset() + tiles * 4 * kTileSlices : counters_bytes(), st));
    // the other frame-scoped buffers (ranges, chunk sums, per-tile P_it words)
    // are zeroed by K1 itself, so the kernels form one PDL chain
    const bool units = raster_uses_units(p, maxt);
    if (units) ensure(ctx->tile_pit, std::max<uint64_t>(tiles, 1) * 8);
    FrameZero fz;
    fz.ranges = ptr<uint2>(ctx->ranges);
    fz.tile_pit = units ? ptr<unsigned long long>(ctx->tile_pit) : nullptr;
    fz.chunks = ptr<uint32_t>(ctx->chunks);
    fz.n_tiles = static_cast<uint32_t>(tiles);
    fz.n_chunks = n > 0 && !bucket ? static_cast<uint32_t>(chunk_slots(n)) : 0u;
    BucketOut bk;
    if (bucket) {
        bk.tile_cnt = tile_cnt_of(ctx);
        bk.hits = ptr<uint4>(ctx->bk_hits);
        bk.gd = ptr<uint2>(ctx->bk_gd);
        bk.orig = sc->view().orig;
        bk.inv = sc->view().inv;
    }
    if (n == 0) {  // no K1: the raster still reads the (empty) ranges
        AGSX_CUDA(cudaMemsetAsync(ctx->ranges.p, 0, tiles * 8, st));
        if (units) AGSX_CUDA(cudaMemsetAsync(ctx->tile_pit.p, 0, tiles * 8, st));
    }
    if (maxt) AGSX_CUDA(cudaMemsetAsync(ctx->maxt.p, 0, n * 4, st));
    AGSX_CUDA(cudaEventRecord(ctx->ev_zeroed, st));
    const SplatPlanes pl = planes_of(ctx);
    if (n > 0) {
        NvtxRange r("agsx.preprocess");
        const int grid = static_cast<int>((n + 255) / 256);
        launch_pdl(k_preprocess, dim3(grid), dim3(256), 0, st, p, sc->view(), pl, ptr<uint32_t>(ctx->status),
                   ptr<uint32_t>(ctx->dkeys), ctr, dump, fz, bk);
        check_launch(ctx);
    }
    AGSX_CUDA(cudaEventRecord(ctx->ev[1], st));
    ctx->f_bucket = bucket;
    {
        NvtxRange r("agsx.pair_gen+sort");
        if (bucket) {
            enqueue_bucket_sort(ctx, n, p, bk);
        } else {
            enqueue_depth_sort(ctx, n, tiles, p, pl, sc->view().inv);
        }
    }
    uint32_t* vals = ptr<uint32_t>(ctx->pvals);
    if (!bucket) vals = ctx->f_pvals;
    NvtxRange r("agsx.raster");
    enqueue_raster(ctx, p, maxt, vals);
}

// Tile-bucketed sort path (k_bucket.cu): K2 tile scan, K3 scatter, K4
// per-tile sort.  Events: ev[2] after the scan, ev[3] after the scatter,
// ev[4] after the per-tile sort (stage "pair_gen" = the scatter, "sort" =
// scan + per-tile sort).
void enqueue_bucket_sort(agsx_ctx* ctx, uint64_t n, const FrameParams& p, const BucketOut& bk) {
    cudaStream_t st = ctx->stream;
    Counters* ctr = ptr<Counters>(ctx->ctr);
    const uint64_t tiles = static_cast<uint64_t>(p.tiles_x) * p.tiles_y;
    const uint32_t T = static_cast<uint32_t>(tiles);
    const int scan_grid = static_cast<int>((tiles + kTileScanPer - 1) / kTileScanPer);
    launch_pdl(k_tile_scan, dim3(scan_grid), dim3(kTileScanThreads), 0, st, bk.tile_cnt, ptr<uint2>(ctx->ranges), T,
               ctr,
               ctx->pair_capacity, ptr<uint64_t>(ctx->lb), ctx->epoch++, ptr<uint32_t>(ctx->big_list));
    check_launch(ctx);
    AGSX_CUDA(cudaEventRecord(ctx->ev[2], st));
    const int scatter_grid = static_cast<int>(std::max<uint64_t>((n + 255) / 256, 1));  // one splat per thread
    launch_pdl(k_bucket_scatter, dim3(scatter_grid), dim3(256), 0, st, p, planes_of(ctx), bk,
               static_cast<const Counters*>(ctr), ptr<uint64_t>(ctx->ekeys));
    check_launch(ctx);
    AGSX_CUDA(cudaEventRecord(ctx->ev[3], st));
    launch_pdl(k_tile_sort, dim3(ctx->num_sms * ctx->occ_tile_sort), dim3(256), 0, st, ptr<uint2>(ctx->ranges), T,
               ptr<uint64_t>(ctx->ekeys), ptr<uint64_t>(ctx->ekeys2), ptr<uint32_t>(ctx->pvals), ctr,
               static_cast<const uint32_t*>(ptr<uint32_t>(ctx->big_list)), bk.orig, bk.inv);
    check_launch(ctx);
    AGSX_CUDA(cudaEventRecord(ctx->ev[4], st));
    ctx->f_tkeys = nullptr;
    ctx->f_pvals = ptr<uint32_t>(ctx->pvals);
}

// Depth-then-tile radix path: K4a depth sort of the splats, K3 emission in
// depth order, K4b stable tile sort, K5 ranges.
void enqueue_depth_sort(agsx_ctx* ctx, uint64_t n, uint64_t tiles, const FrameParams& p, const SplatPlanes& pl,
                        const uint32_t* scene_inv) {
    cudaStream_t st = ctx->stream;
    Counters* ctr = ptr<Counters>(ctx->ctr);
    // K4a: stable sort by depth bits (4 x 8-bit, histograms in one read);
    // pass 0 drops the sentinel keys of splats without tiles (the ordered
    // compaction) and sets m.
    uint32_t* dk[2] = {ptr<uint32_t>(ctx->dkeys), ptr<uint32_t>(ctx->dkeys2)};
    uint32_t* dv[2] = {ptr<uint32_t>(ctx->dvals), ptr<uint32_t>(ctx->dvals2)};
    uint32_t* chunk_sum = ptr<uint32_t>(ctx->chunks);
    uint32_t* chunk_off = chunk_sum + chunk_slots(n);
    // Digits are those of key - kmin (K1's range counters): when the frame's
    // keys span < 2^24 (depth max/min below ~2, the common case) the 4th pass
    // exits at once on the device and the order is final after 3 passes, in
    // dv[1] instead of dv[0] (K3 reads the one the device chose).
    if (n > 0) {
        SortBias sb;
        sb.kmin_c = &ctr->kmin_c;
        sb.kmax = &ctr->kmax;
        // The pass runs in Gaussian-id order (equal depths keep id order)
        // and carries the storage slots on as values (DevScene)
        sort_pass<uint32_t>(ctx, dk[0], scene_inv, dk[1], dv[1], nullptr, n, 0, true, &ctr->m, {}, sb);
        for (int ps = 1; ps < 4; ++ps) {
            SortCountOut co;
            SortBias sp = sb;
            if (ps >= 2) {  // the depth order's tile counts + per-chunk sums for K3, from the last pass run
                co.src = ptr<uint32_t>(ctx->status);
                co.out = ptr<uint32_t>(ctx->dcounts);
                co.chunk_sum = chunk_sum;
                sp.co_if_narrow = ps == 2;
                sp.only_wide = ps == 3;
            }
            sort_pass<uint32_t>(ctx, dk[ps & 1], dv[ps & 1], dk[(ps + 1) & 1], dv[(ps + 1) & 1], &ctr->m, n, 8 * ps,
                                false, nullptr, co, sp);
        }
    }
    AGSX_CUDA(cudaEventRecord(ctx->ev[2], st));
    // K3: scan + emit in depth order
    uint32_t* tk[2] = {ptr<uint32_t>(ctx->tkeys), ptr<uint32_t>(ctx->tkeys2)};
    uint32_t* pv[2] = {ptr<uint32_t>(ctx->pvals), ptr<uint32_t>(ctx->pvals2)};
    if (n > 0) {
        launch_pdl(k_scan_chunks, dim3(1), dim3(1024), 0, st, chunk_sum, chunk_off, ctr, ctx->pair_capacity);
        check_launch(ctx);
        // the big stage when the previous frame averaged > 10 pairs per splat
        const bool big = ctx->pairs_per_splat > 10.0;
        AGSX_CUDA(launch_emit(big, ctx->num_sms * (big ? ctx->occ_emit_big : ctx->occ_emit), st, p, dv[0], dv[1],
                              ptr<uint32_t>(ctx->dcounts), chunk_off, pl, tk[0], pv[0], ctx->pair_capacity, ctr));
        check_launch(ctx);
    }
    AGSX_CUDA(cudaEventRecord(ctx->ev[3], st));
    // K4b: stable sort of the pairs by tile id, then K5 ranges
    const int passes = (tile_bits(static_cast<uint32_t>(tiles)) + 7) / 8;
    int cur = 0;
    if (n > 0) {
        for (int ps = 0; ps < passes; ++ps) {
            sort_pass<uint32_t>(ctx, tk[cur], pv[cur], tk[cur ^ 1], pv[cur ^ 1], &ctr->p_eff, ctx->pair_capacity,
                                8 * ps, false, nullptr);
            cur ^= 1;
        }
        launch_pdl(k_ranges_u32, dim3(ctx->num_sms * 8), dim3(256), 0, st, tk[cur], &ctr->p_eff, ptr<uint2>(ctx->ranges));
        check_launch(ctx);
    }
    AGSX_CUDA(cudaEventRecord(ctx->ev[4], st));
    ctx->f_tkeys = tk[cur];
    ctx->f_pvals = pv[cur];
}

// K6 and the host egress behind it, then the counter readback.
void enqueue_raster(agsx_ctx* ctx, const FrameParams& p, bool maxt, uint32_t* vals) {
    cudaStream_t st = ctx->stream;
    Counters* ctr = ptr<Counters>(ctx->ctr);
    const SplatPlanes pl = planes_of(ctx);
    const uint64_t tiles = static_cast<uint64_t>(p.tiles_x) * p.tiles_y;
    // K6
    const bool banded = (ctx->f_band_host || ctx->f_band_host_u8) && raster_uses_units(p, maxt) && p.tiles_y > 0;
    const char* eg = std::getenv("AGSX_EGRESS");
    const bool flags = banded && wait_value32() && !(eg && std::strcmp(eg, "launches") == 0);
    if (flags) {
        // banded egress, one raster launch: the tile rows form 32 slots and
        // every unit adds itself to its slot's count once its pixels are
        // stored; the copy stream waits for the counts (cuStreamWaitValue32)
        // and copies finished rows to the page-locked host image while later
        // rows render.  f32 frames: slots are copied in groups 1, 4, 19, 8 --
        // the raster runs ~4.6x faster than PCIe, so each group is done
        // before the previous copy ends, the first copy starts after 1/32 of
        // the raster and a frame costs 4 copies (each costs ~8 us of PCIe
        // setup).  PPM bytes: PCIe is about as fast as the raster, so slots
        // go in pairs and the last copy is short.  The raster also writes the
        // PPM bytes; only those are copied.
        const int S = std::min(agsx_ctx::kFlagBands, p.tiles_y);
        const int rows_per = (p.tiles_y + S - 1) / S;
        uint8_t* u8 = ctx->f_band_host_u8 ? ptr<uint8_t>(ctx->img_u8) : nullptr;
        launch_raster_units(ctx->num_sms * ctx->occ_raster, st, p, ptr<uint2>(ctx->ranges), vals, pl.p0, pl.p1,
                            pl.p2, ctx->f_image, &ctr->tile_ctr[3], ptr<unsigned long long>(ctx->tile_pit), &ctr->p_it,
                            ctr->dbg, ctr->band_done, rows_per, u8);
        check_launch(ctx);
        AGSX_CUDA(cudaEventRecord(ctx->ev[5], st));
        AGSX_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_zeroed, 0));  // not last frame's counts
        static const int kF32Groups[] = {1, 5, 24, 32};  // slot group ends (of 32) for f32 frames
        int s0 = 0;
        for (int gi = 0; s0 * rows_per < p.tiles_y; ++gi) {
            const int s1 = u8 ? std::min(S, s0 + 2) : std::min(S, std::max(s0 + 1, kF32Groups[std::min(gi, 3)] * S / 32));
            for (int sl = s0; sl < s1; ++sl) {
                const int r0 = sl * rows_per, r1 = std::min(p.tiles_y, r0 + rows_per);
                if (r0 >= r1) break;
                const uint32_t units_s = 2u * static_cast<uint32_t>((r1 - r0) * p.tiles_x);
                const CUresult cr = wait_value32()(reinterpret_cast<CUstream>(ctx->copy_stream),
                                                   reinterpret_cast<CUdeviceptr>(&ctr->band_done[sl]), units_s,
                                                   CU_STREAM_WAIT_VALUE_GEQ);
                if (cr != CUDA_SUCCESS)
                    throw StatusError{AGSX_ECUDA,
                                      "cuStreamWaitValue32 failed (" + std::to_string(static_cast<int>(cr)) + ")"};
            }
            const size_t y0 = static_cast<size_t>(s0) * rows_per * p.tile_size;
            const size_t y1 = std::min(static_cast<size_t>(s1) * rows_per * p.tile_size, static_cast<size_t>(p.H));
            if (y1 > y0) {
                if (u8) {
                    const size_t row_bytes = static_cast<size_t>(p.W) * 3;
                    AGSX_CUDA(cudaMemcpyAsync(ctx->f_band_host_u8 + y0 * row_bytes, u8 + y0 * row_bytes,
                                              (y1 - y0) * row_bytes, cudaMemcpyDeviceToHost, ctx->copy_stream));
                } else {
                    const size_t row_bytes = static_cast<size_t>(p.W) * 12;
                    AGSX_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(ctx->f_band_host) + y0 * row_bytes,
                                              reinterpret_cast<char*>(ctx->f_image) + y0 * row_bytes,
                                              (y1 - y0) * row_bytes, cudaMemcpyDeviceToHost, ctx->copy_stream));
                }
            }
            s0 = s1;
        }
        AGSX_CUDA(cudaEventRecord(ctx->copy_done, ctx->copy_stream));
        AGSX_CUDA(cudaStreamWaitEvent(st, ctx->copy_done, 0));
    } else if (banded) {
        // banded egress over one raster launch per band (drivers without
        // stream wait-value): band b's rows are copied to the page-locked host
        // image on the copy stream while band b+1 renders
        const int B = std::min(agsx_ctx::kBands, p.tiles_y);
        const int rows_per = (p.tiles_y + B - 1) / B;
        for (int b = 0; b < B; ++b) {
            const int r0 = b * rows_per, r1 = std::min(p.tiles_y, r0 + rows_per);
            if (r0 >= r1) break;
            FrameParams pb = p;
            pb.unit_lo = 2u * static_cast<uint32_t>(r0 * p.tiles_x);
            pb.unit_hi = 2u * static_cast<uint32_t>(r1 * p.tiles_x);
            launch_raster(ctx, pb, ptr<uint2>(ctx->ranges), vals, pl.p0, pl.p1, pl.p2, ctx->f_image, nullptr, ctr,
                          &ctr->tile_ctr[8 + b]);
            const size_t y0 = static_cast<size_t>(r0) * p.tile_size;
            const size_t y1 = std::min(static_cast<size_t>(r1) * p.tile_size, static_cast<size_t>(p.H));
            if (ctx->f_band_host_u8) {
                // row f3: quantise the band to PPM bytes (write_image) on the
                // device; only the bytes cross PCIe
                const uint64_t off = y0 * static_cast<uint64_t>(p.W) * 3, len = (y1 - y0) * static_cast<uint64_t>(p.W) * 3;
                launch_quantize(ctx, ctx->f_image + off, ptr<uint8_t>(ctx->img_u8) + off, len, st);
            }
            AGSX_CUDA(cudaEventRecord(ctx->band_ev[b], st));
            AGSX_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->band_ev[b], 0));
            if (ctx->f_band_host_u8) {
                const size_t row_bytes = static_cast<size_t>(p.W) * 3;
                AGSX_CUDA(cudaMemcpyAsync(ctx->f_band_host_u8 + y0 * row_bytes, ptr<uint8_t>(ctx->img_u8) + y0 * row_bytes,
                                          (y1 - y0) * row_bytes, cudaMemcpyDeviceToHost, ctx->copy_stream));
            } else {
                const size_t row_bytes = static_cast<size_t>(p.W) * 12;
                AGSX_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(ctx->f_band_host) + y0 * row_bytes,
                                          reinterpret_cast<char*>(ctx->f_image) + y0 * row_bytes, (y1 - y0) * row_bytes,
                                          cudaMemcpyDeviceToHost, ctx->copy_stream));
            }
        }
        AGSX_CUDA(cudaEventRecord(ctx->ev[5], st));
        AGSX_CUDA(cudaEventRecord(ctx->copy_done, ctx->copy_stream));
        AGSX_CUDA(cudaStreamWaitEvent(st, ctx->copy_done, 0));
    } else {
        launch_raster(ctx, p, ptr<uint2>(ctx->ranges), vals, pl.p0, pl.p1, pl.p2, ctx->f_image,
                      maxt ? ptr<uint32_t>(ctx->maxt) : nullptr, ctr);
        AGSX_CUDA(cudaEventRecord(ctx->ev[5], st));
    }
    // Counters to the host by SM stores into the mapped page-locked word block,
    // not by a copy-engine transfer: with frames of several contexts in flight
    // a small D2H copy would queue in the copy engine behind another frame's
    // 191 MB of image bands, and this frame would finish only after that one.
    k_counters_out<<<1, 64, 0, st>>>(reinterpret_cast<const uint32_t*>(ctr), ctx->h_ctr_dev,
                                     static_cast<int>(sizeof(Counters) / 4), ptr<ChainWords>(ctx->chain));
    check_launch(ctx);
    ctx->f_tile_count = static_cast<int>(tiles);
    ctx->f_pit_tiles = raster_uses_units(p, maxt);
}

int start_frame(agsx_ctx* ctx, const agsx_scene* sc, const agsx_camera* cam, const agsx_config* cfg,
                const agsx_lut* lut, bool maxt, float* host_image, float* device_target, uint8_t* host_u8) {
    if (!sc) return fail(ctx, AGSX_EINVAL, "render: null scene");
    if (sc->device != ctx->device) return fail(ctx, AGSX_EINVAL, "scene lives on another device");
    if (const int rc = refuse_if_host_frame(ctx, "render")) return rc;
    NvtxRange nv("agsx.render");
    FrameParams p;
    const int rc = prepare(ctx, cam, cfg, lut, p);
    if (rc) return rc;
    p.clamp_free = sc->max_opacity < p.aclamp;  // alpha <= opacity < aclamp everywhere
    const uint64_t tiles = static_cast<uint64_t>(p.tiles_x) * p.tiles_y;
    ensure_frame_buffers(ctx, sc->n, tiles, static_cast<uint64_t>(cam->width) * cam->height,
                         cfg->mode == AGSX_MODE_OBB, cfg->pair_budget);
    if (maxt) ensure(ctx->maxt, std::max<uint64_t>(sc->n, 1) * 4);
    ctx->have_frame = true;
    ctx->pending = true;
    ctx->f_scene = sc;
    ctx->f_cam = *cam;
    ctx->f_cfg = *cfg;
    ctx->f_has_lut = lut != nullptr;
    if (lut && lut->bin_count > 0) {
        ctx->f_lut.assign(lut->bins, lut->bins + lut->bin_count);
        ctx->f_lut_dmin = lut->depth_min;
        ctx->f_lut_dmax = lut->depth_max;
    } else {
        ctx->f_lut.clear();
    }
    ctx->f_params = p;
    ctx->f_maxt = maxt;
    // Frame egress: a page-locked, device-mapped destination is written by
    // the rasterizer directly (the 191 MB PCIe transfer overlaps the blend);
    // anything else gets the device image and a copy.
    ctx->f_image = device_target ? device_target : ptr<float>(ctx->image);
    ctx->f_image_on_host = device_target != nullptr;  // the ctx image is not this frame's
    ctx->f_band_host = nullptr;
    ctx->f_band_host_u8 = nullptr;
    ctx->f_host_dst = nullptr;
    ctx->f_host_dst_u8 = nullptr;
    if (host_u8 && raster_uses_units(p, maxt)) {
        cudaPointerAttributes at{};
        const uint64_t n = static_cast<uint64_t>(cam->width) * cam->height * 3;
        if (cudaPointerGetAttributes(&at, host_u8) == cudaSuccess && at.type == cudaMemoryTypeHost &&
            at.devicePointer != nullptr) {
            ensure(ctx->img_u8, std::max<uint64_t>(n, 16));
            ctx->f_band_host_u8 = host_u8;  // the float image stays in ctx->image as well
        }
        cudaGetLastError();
    }
    if (host_image && !device_target) {
        // A page-locked host destination: the default rasterizer fills it by
        // banded copy-engine transfers behind the raster (57 GB/s); other
        // rasterizers (exact / max_t / tile sizes) write it directly through
        // the mapping (SM stores, 52 GB/s).  Pageable memory: one copy after.
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, host_image) == cudaSuccess && at.type == cudaMemoryTypeHost &&
            at.devicePointer != nullptr) {
            const char* eg = std::getenv("AGSX_EGRESS");
            if (raster_uses_units(p, maxt) && !(eg && std::strcmp(eg, "zerocopy") == 0)) {
                ctx->f_band_host = host_image;
                ctx->f_image_on_host = true;  // the frame's image ends up in the host buffer
            } else if (!(eg && std::strcmp(eg, "copy") == 0)) {
                ctx->f_image = static_cast<float*>(at.devicePointer);
                ctx->f_image_on_host = true;
            }
        }
        cudaGetLastError();  // clear a pageable-pointer query error
    }
    enqueue_frame(ctx, sc, p, maxt, nullptr);
    return AGSX_OK;
}

// A frame whose host image is still being written (render_async_host[_u8],
// not yet waited for) owns the context's buffers and counters: no other work
// may be enqueued on the context until agsx_render_wait.
int refuse_if_host_frame(agsx_ctx* ctx, const char* what) {
    if (ctx->pending && (ctx->f_host_dst || ctx->f_host_dst_u8))
        return fail(ctx, AGSX_EINVAL,
                    std::string(what) + ": a host frame is in flight on this context; call agsx_render_wait first");
    return AGSX_OK;
}

// Wait for the enqueued frame; grow the pair arena and re-run on overflow.
// Frames enqueued before it since the last wait (an async chain) cannot be
// re-run: if one of them overflowed, the wait fails with AGSX_EFRAME_LOST.
int finish_frame(agsx_ctx* ctx, agsx_frame* out) {
    if (!ctx->have_frame || !ctx->pending) return fail(ctx, AGSX_EINVAL, "no frame in flight");
    NvtxRange nv("agsx.wait");
    for (int attempt = 0; attempt < 4; ++attempt) {
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        const Counters c = *ctx->h_ctr;
        const ChainWords chain = *reinterpret_cast<const ChainWords*>(ctx->h_ctr + 1);
        const bool last_over = c.overflow != 0u || c.p_eff != c.p;
        // the chain is over: its words start again for the next one (and for a re-run)
        AGSX_CUDA(cudaMemsetAsync(ctx->chain.p, 0, sizeof(ChainWords), ctx->stream));
        const uint32_t lost = chain.overflowed - (last_over ? 1u : 0u);
        if (attempt == 0 && lost > 0) {
            ctx->pending = false;
            AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
            return fail(ctx, AGSX_EFRAME_LOST,
                        std::to_string(lost) + " of the " + std::to_string(chain.frames) +
                            " frames enqueued since the last wait overflowed the pair arena (capacity " +
                            std::to_string(ctx->pair_capacity) +
                            " pairs) and were not rasterised; wait for each frame, or render one frame first to "
                            "size the arena");
        }
        const uint64_t pairs = c.p == 0xffffffffu ? UINT64_MAX : c.p;
        if (pairs > ctx->f_cfg.pair_budget) {
            ctx->pending = false;
            return fail(ctx, AGSX_EPAIR_BUDGET,
                        "pair count " + (pairs == UINT64_MAX ? std::string(">= 2^32") : std::to_string(pairs)) +
                            " exceeds budget " + std::to_string(ctx->f_cfg.pair_budget));
        }
        if (last_over) {
            if (pairs >= (1ull << 31)) {
                ctx->pending = false;
                return fail(ctx, AGSX_ENOMEM, "pair count exceeds 2^31");
            }
            ctx->pair_capacity = std::min<uint64_t>(pairs + pairs / 8 + 1024, ctx->f_cfg.pair_budget);
            const uint64_t tiles = static_cast<uint64_t>(ctx->f_params.tiles_x) * ctx->f_params.tiles_y;
            ensure_frame_buffers(ctx, ctx->f_scene->n, tiles,
                                 static_cast<uint64_t>(ctx->f_cam.width) * ctx->f_cam.height,
                                 ctx->f_cfg.mode == AGSX_MODE_OBB, ctx->f_cfg.pair_budget);
            enqueue_frame(ctx, ctx->f_scene, ctx->f_params, ctx->f_maxt, nullptr);
            continue;
        }
        ctx->pending = false;
        ctx->last_m = c.m;
        ctx->prev_pairs_per_tile = static_cast<double>(c.p) /
                                   std::max(1.0, static_cast<double>(ctx->f_params.tiles_x) * ctx->f_params.tiles_y);
        ctx->pairs_per_splat = c.m ? static_cast<double>(c.p) / c.m : 0.0;
        if (out) {
            out->pair_count = c.p;
            out->splat_count = c.s;
            float ms[5];
            for (int i = 0; i < 5; ++i) AGSX_CUDA(cudaEventElapsedTime(&ms[i], ctx->ev[i], ctx->ev[i + 1]));
            out->stage_ms[0] = ms[0];
            out->stage_ms[1] = ms[2];
            out->stage_ms[2] = ms[1] + ms[3];
            out->stage_ms[3] = ms[4];
        }
        return AGSX_OK;
    }
    ctx->pending = false;
    return fail(ctx, AGSX_ECUDA, "pair arena did not converge");
}

// The finished frame's write_image bytes into host memory `image_u8` when no
// banded u8 egress ran: quantised on the device, then through the mapping
// (page-locked) or one copy (pageable).
int quantize_to_host(agsx_ctx* ctx, uint8_t* image_u8) {
    const uint64_t n = static_cast<uint64_t>(ctx->f_cam.width) * ctx->f_cam.height * 3;
    uint8_t* dst = nullptr;  // device-visible destination
    cudaPointerAttributes at{};
    const bool mapped = cudaPointerGetAttributes(&at, image_u8) == cudaSuccess && at.type == cudaMemoryTypeHost &&
                        at.devicePointer != nullptr && (reinterpret_cast<uintptr_t>(at.devicePointer) & 15u) == 0;
    cudaGetLastError();
    if (mapped) {
        dst = static_cast<uint8_t*>(at.devicePointer);
    } else {
        ensure(ctx->tmp0, std::max<uint64_t>(n, 16));
        dst = ptr<uint8_t>(ctx->tmp0);
    }
    launch_quantize(ctx, ptr<float>(ctx->image), dst, n, ctx->stream);
    if (!mapped) AGSX_CUDA(cudaMemcpyAsync(image_u8, dst, n, cudaMemcpyDeviceToHost, ctx->stream));
    AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
    return AGSX_OK;
}
// One frame-egress copy stream per device, shared by every context on it:
// frames of several contexts then leave over PCIe in the order they were
// enqueued (FIFO), so a pipelined camera path keeps the copy engine busy with
// one whole frame after another instead of interleaving two frames' bands
// (which finishes both late and leaves a gap before the next pair).
cudaError_t shared_copy_stream(int device, cudaStream_t* out) {
    static std::mutex mu;
    static std::map<int, cudaStream_t> streams;  // process lifetime
    std::lock_guard<std::mutex> g(mu);
    auto it = streams.find(device);
    if (it != streams.end()) {
        *out = it->second;
        return cudaSuccess;
    }
    cudaStream_t st = nullptr;
    const cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (e == cudaSuccess) streams[device] = st;
    *out = st;
    return e;
}
}  // namespace agsx::host

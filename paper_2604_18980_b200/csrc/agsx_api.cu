// agsx_api.cu -- C-ABI of libagsx.so: contexts, device arenas, scene upload
// and the per-frame launch sequence of the render path.
//
//   reference: render()          rasterizer.cpp:102-165
//              validate(cfg/cam) scene.cpp:41-59, 113-123
//              stage API         preprocess.hpp:51-54, pair_gen.hpp:70-72,
//                                pair_sort.hpp:19, rasterizer.hpp:54-58
//
// A frame is enqueued on the ctx stream without any host synchronisation:
// every data-dependent size (survivors, splats with tiles, pair count) stays
// on the device and the kernels that consume it are persistent grids that
// read it there.  The host reads one 128-byte counter block when the caller
// waits for the frame; a pair count above the buffer capacity (but within
// pair_budget) grows the pair arena and re-runs the frame.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "kernels.cuh"

using namespace agsx;

namespace {

struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
};

struct StatusError {
    int code;
    std::string msg;
};

#define AGSX_CUDA(call)                                                                 \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            throw StatusError{e_ == cudaErrorMemoryAllocation ? AGSX_ENOMEM : AGSX_ECUDA, \
                              std::string(#call) + ": " + cudaGetErrorString(e_)};      \
    } while (0)

}  // namespace

struct agsx_scene {
    int device = 0;
    uint64_t n = 0;
    int D = 1;
    Buf pos_op, rot, scale_r, sh_gb, sh_rest;
    DevScene view() const {
        DevScene s;
        s.n = n;
        s.sh_coeffs = D;
        s.pos_op = static_cast<const float4*>(pos_op.p);
        s.rot = static_cast<const float4*>(rot.p);
        s.scale_r = static_cast<const float4*>(scale_r.p);
        s.sh_gb = static_cast<const float2*>(sh_gb.p);
        s.sh_rest = static_cast<const float*>(sh_rest.p);
        return s;
    }
};

struct agsx_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err = "";
    uint64_t launches = 0;
    uint32_t epoch = 1;
    int num_sms = 148;
    int occ_sort32 = 1, occ_sort64 = 1, occ_emit = 1, occ_emit_big = 1, occ_raster = 1;
    double pairs_per_splat = 0.0;  // previous frame's P / M (picks the emit stage)
    Buf sort_counts;  // grid x 256 chunk digit counts + 256 totals (one pass at a time)

    // device arenas (grow-only)
    Buf status, p0, p1, p2, p3, p4, dkeys, dvals, dkeys2, dvals2, dcounts, chunks, img_u8;
    Buf tkeys, pvals, tkeys2, pvals2;
    Buf ranges, image, lb, ctr, hist, maxt, dump, lut_ext, tile_pit, calib;
    Buf tmp0, tmp1, tmp2, tmp3, tmp4;
    uint64_t pair_capacity = 0;

    Counters* h_ctr = nullptr;  // pinned
    uint32_t* h_ctr_dev = nullptr;  // its device-mapped alias
    static constexpr int kRing = 64;  // frames of stage events kept for timing
    cudaEvent_t ev_ring[kRing][6] = {};
    cudaEvent_t* ev = ev_ring[0];
    uint64_t frames = 0;

    // most recent fused frame
    bool have_frame = false;
    const agsx_scene* f_scene = nullptr;
    agsx_camera f_cam{};
    agsx_config f_cfg{};
    std::vector<float> f_lut;
    float f_lut_dmin = 0.0f, f_lut_dmax = 100.0f;
    bool f_has_lut = false;
    FrameParams f_params{};
    bool f_maxt = false;
    float* f_image = nullptr;     // raster target of the frame (device image or mapped host buffer)
    bool f_image_on_host = false;  // the frame streamed its image into a mapped host buffer
    float* f_host_dst = nullptr;   // agsx_render_async_host destination (copied in wait if pageable)
    uint8_t* f_band_host_u8 = nullptr;  // page-locked host PPM pixels filled by banded copies (f3 egress)
    uint8_t* f_host_dst_u8 = nullptr;   // agsx_render_async_host_u8 destination (quantised in wait if pageable)
    float* f_band_host = nullptr;  // page-locked host image filled by banded copies behind the raster
    cudaStream_t copy_stream = nullptr;
    static constexpr int kBands = 8;       // egress bands with one raster launch per band (fallback)
    static constexpr int kFlagBands = 16;  // egress bands of the one-launch path (Counters::band_done)
    cudaEvent_t band_ev[kBands] = {};
    cudaEvent_t copy_done = nullptr;
    cudaEvent_t ev_zeroed = nullptr;  // the frame's counters are zeroed (band flags valid from here)
    uint32_t* f_tkeys = nullptr;
    uint32_t* f_pvals = nullptr;
    int f_tile_count = 0;
};

namespace {

void ensure(Buf& b, size_t bytes, bool zero = false) {
    if (b.bytes >= bytes) return;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    const size_t alloc = std::max<size_t>(bytes, 256);
    AGSX_CUDA(cudaMalloc(&b.p, alloc));
    if (zero) AGSX_CUDA(cudaMemset(b.p, 0, alloc));
    b.bytes = alloc;
}

void release(Buf& b) {
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
}

template <typename T>
T* ptr(const Buf& b) {
    return static_cast<T*>(b.p);
}

void check_launch(agsx_ctx* ctx) {
    ++ctx->launches;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw StatusError{AGSX_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e)};
}

template <typename F>
int guarded(agsx_ctx* ctx, F&& f) {
    try {
        AGSX_CUDA(cudaSetDevice(ctx->device));
        const int rc = f();
        if (rc == AGSX_OK) ctx->err.clear();
        return rc;
    } catch (const StatusError& e) {
        ctx->err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        ctx->err = "host allocation failed";
        return AGSX_ENOMEM;
    } catch (...) {
        ctx->err = "unknown error";
        return AGSX_ECUDA;
    }
}

int fail(agsx_ctx* ctx, int code, const std::string& msg) {
    ctx->err = msg;
    return code;
}

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
                   uint32_t* maxt, Counters* ctr, uint32_t* unit_ctr = nullptr) {
    const int grid = p.tiles_x * p.tiles_y;
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
// 256-splat chunks of the depth order (K3 work units)
uint64_t chunk_slots(uint64_t n) { return std::max<uint64_t>((n + 255) / 256, 1); }

int sort_grid(agsx_ctx* ctx, bool k64) { return ctx->num_sms * (k64 ? ctx->occ_sort64 : ctx->occ_sort32); }

// Histograms of the low `npasses` digits of n keys (hist zeroed by the caller).
template <typename K>
void sort_hist(agsx_ctx* ctx, const K* keys, const uint32_t* n_dev, uint64_t n_host, int npasses, bool sentinel,
               uint32_t* hist) {
    const int grid = static_cast<int>(std::max<uint64_t>(
        1, std::min<uint64_t>((n_host + 127) / 128, static_cast<uint64_t>(ctx->num_sms) * 8)));
    launch_hist<K>(grid, ctx->stream, keys, n_dev, n_host, npasses, sentinel, static_cast<K>(~K(0)), hist);
    check_launch(ctx);
}

// One stable LSD pass over at most n_host keys (three kernels).
template <typename K>
void sort_pass(agsx_ctx* ctx, const K* kin, const uint32_t* vin, K* kout, uint32_t* vout, const uint32_t* n_dev,
               uint64_t n_host, int shift, bool sentinel, uint32_t* n_out, SortCountOut co = {}, SortBias sb = {}) {
    const bool k64 = sizeof(K) == 8;
    const uint64_t tiles = (n_host + kSortTile - 1) / kSortTile;
    const int grid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(
        tiles, std::min(sort_grid(ctx, k64), 1024))));
    ensure(ctx->sort_counts, static_cast<size_t>(grid) * 256 * 4 + 256 * 4);
    uint32_t* counts = ptr<uint32_t>(ctx->sort_counts);
    launch_sort_pass<K>(grid, sort_smem(k64), ctx->stream, kin, vin, kout, vout, n_dev, n_host, shift, sentinel,
                        static_cast<K>(~K(0)), counts, counts + static_cast<size_t>(grid) * 256, n_out, co, sb);
    check_launch(ctx);
    ctx->launches += 2;  // three kernels per pass
}

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
    ensure(ctx->ctr, counters_bytes());
    if (ctx->pair_capacity == 0) {
        // first guess: 12 pairs per Gaussian, at most the budget, at least 1M
        ctx->pair_capacity = std::min<uint64_t>(std::max<uint64_t>(12 * n, 1u << 20),
                                                std::max<uint64_t>(pair_budget, 1));
    }
    const uint64_t cap = ctx->pair_capacity;
    ensure(ctx->tkeys, cap * 4);
    ensure(ctx->pvals, cap * 4);
    ensure(ctx->tkeys2, cap * 4);
    ensure(ctx->pvals2, cap * 4);
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
    if (cfg->tile_size > 64)
        return fail(ctx, AGSX_EINVAL, "tile_size > 64 is not supported by the device rasterizer");
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

__global__ void k_counters_out(const uint32_t* __restrict__ src, uint32_t* dst, int words) {
    for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
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

void enqueue_frame(agsx_ctx* ctx, const agsx_scene* sc, const FrameParams& p, bool maxt,
                   agsx_splat_view* dump) {
    const uint64_t n = sc->n;
    const uint64_t tiles = static_cast<uint64_t>(p.tiles_x) * p.tiles_y;
    Counters* ctr = ptr<Counters>(ctx->ctr);
    cudaStream_t st = ctx->stream;
    ctx->ev = ctx->ev_ring[ctx->frames % agsx_ctx::kRing];
    ++ctx->frames;

    AGSX_CUDA(cudaEventRecord(ctx->ev[0], st));
    AGSX_CUDA(cudaMemsetAsync(ctr, 0, counters_bytes(), st));
    // every frame-scoped zeroing happens before the first kernel, so the
    // kernels form one PDL chain
    AGSX_CUDA(cudaMemsetAsync(ctx->ranges.p, 0, tiles * 8, st));
    if (n > 0) AGSX_CUDA(cudaMemsetAsync(ctx->chunks.p, 0, chunk_slots(n) * 4, st));
    if (raster_uses_units(p, maxt)) {
        ensure(ctx->tile_pit, std::max<uint64_t>(tiles, 1) * 8);
        AGSX_CUDA(cudaMemsetAsync(ctx->tile_pit.p, 0, tiles * 8, st));
    }
    if (maxt) AGSX_CUDA(cudaMemsetAsync(ctx->maxt.p, 0, n * 4, st));
    AGSX_CUDA(cudaEventRecord(ctx->ev_zeroed, st));
    const SplatPlanes pl = planes_of(ctx);
    if (n > 0) {
        const int grid = static_cast<int>((n + 255) / 256);
        launch_pdl(k_preprocess, dim3(grid), dim3(256), 0, st, p, sc->view(), pl, ptr<uint32_t>(ctx->status), ptr<uint32_t>(ctx->dkeys),
                                            ctr, dump);
        check_launch(ctx);
    }
    AGSX_CUDA(cudaEventRecord(ctx->ev[1], st));
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
        sort_pass<uint32_t>(ctx, dk[0], nullptr, dk[1], dv[1], nullptr, n, 0, true, &ctr->m, {}, sb);
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
    // K6
    const bool banded = (ctx->f_band_host || ctx->f_band_host_u8) && raster_uses_units(p, maxt) && p.tiles_y > 0;
    const char* eg = std::getenv("AGSX_EGRESS");
    const bool flags = banded && wait_value32() && !(eg && std::strcmp(eg, "launches") == 0);
    if (flags) {
        // banded egress, one raster launch: the tile rows form 16 slots and
        // every unit adds itself to its slot's count once its pixels are
        // stored; the copy stream waits for the counts (cuStreamWaitValue32)
        // and copies finished rows to the page-locked host image while later
        // rows render.  f32 frames: slots are copied in groups 1, 2, 5, 8 --
        // the raster runs ~4.6x faster than PCIe, so each group is done
        // before the previous copy ends, the first copy starts after 1/16 of
        // the raster and a frame costs 4 copies (each costs ~8 us of PCIe
        // setup).  PPM bytes: PCIe is about as fast as the raster, so every
        // slot is its own copy and the last copy is short.  The raster also
        // writes the PPM bytes; only those are copied.
        const int S = std::min(agsx_ctx::kFlagBands, p.tiles_y);
        const int rows_per = (p.tiles_y + S - 1) / S;
        uint8_t* u8 = ctx->f_band_host_u8 ? ptr<uint8_t>(ctx->img_u8) : nullptr;
        launch_raster_units(ctx->num_sms * ctx->occ_raster, st, p, ptr<uint2>(ctx->ranges), pv[cur], pl.p0, pl.p1,
                            pl.p2, ctx->f_image, &ctr->tile_ctr[3], ptr<unsigned long long>(ctx->tile_pit), &ctr->p_it,
                            ctr->dbg, ctr->band_done, rows_per, u8);
        check_launch(ctx);
        AGSX_CUDA(cudaEventRecord(ctx->ev[5], st));
        AGSX_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_zeroed, 0));  // not last frame's counts
        static const int kF32Groups[] = {1, 3, 8, 16};  // slot group ends for f32 frames
        int s0 = 0;
        for (int gi = 0; s0 * rows_per < p.tiles_y; ++gi) {
            const int s1 = u8 ? s0 + 1 : std::min(S, std::max(s0 + 1, kF32Groups[std::min(gi, 3)] * S / 16));
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
            launch_raster(ctx, pb, ptr<uint2>(ctx->ranges), pv[cur], pl.p0, pl.p1, pl.p2, ctx->f_image, nullptr, ctr,
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
        launch_raster(ctx, p, ptr<uint2>(ctx->ranges), pv[cur], pl.p0, pl.p1, pl.p2, ctx->f_image,
                      maxt ? ptr<uint32_t>(ctx->maxt) : nullptr, ctr);
        AGSX_CUDA(cudaEventRecord(ctx->ev[5], st));
    }
    // Counters to the host by SM stores into the mapped page-locked word block,
    // not by a copy-engine transfer: with frames of several contexts in flight
    // a small D2H copy would queue in the copy engine behind another frame's
    // 191 MB of image bands, and this frame would finish only after that one.
    k_counters_out<<<1, 64, 0, st>>>(reinterpret_cast<const uint32_t*>(ctr), ctx->h_ctr_dev,
                                     static_cast<int>(sizeof(Counters) / 4));
    check_launch(ctx);
    ctx->f_tkeys = tk[cur];
    ctx->f_pvals = pv[cur];
    ctx->f_tile_count = static_cast<int>(tiles);
}

int start_frame(agsx_ctx* ctx, const agsx_scene* sc, const agsx_camera* cam, const agsx_config* cfg,
                const agsx_lut* lut, bool maxt, float* host_image = nullptr, float* device_target = nullptr,
                uint8_t* host_u8 = nullptr) {
    if (!sc) return fail(ctx, AGSX_EINVAL, "render: null scene");
    if (sc->device != ctx->device) return fail(ctx, AGSX_EINVAL, "scene lives on another device");
    FrameParams p;
    const int rc = prepare(ctx, cam, cfg, lut, p);
    if (rc) return rc;
    const uint64_t tiles = static_cast<uint64_t>(p.tiles_x) * p.tiles_y;
    ensure_frame_buffers(ctx, sc->n, tiles, static_cast<uint64_t>(cam->width) * cam->height,
                         cfg->mode == AGSX_MODE_OBB, cfg->pair_budget);
    if (maxt) ensure(ctx->maxt, std::max<uint64_t>(sc->n, 1) * 4);
    ctx->have_frame = true;
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

// Wait for the enqueued frame; grow the pair arena and re-run on overflow.
int finish_frame(agsx_ctx* ctx, agsx_frame* out) {
    if (!ctx->have_frame) return fail(ctx, AGSX_EINVAL, "no frame in flight");
    for (int attempt = 0; attempt < 4; ++attempt) {
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        const Counters c = *ctx->h_ctr;
        const uint64_t pairs = c.p == 0xffffffffu ? UINT64_MAX : c.p;
        if (pairs > ctx->f_cfg.pair_budget) {
            return fail(ctx, AGSX_EPAIR_BUDGET,
                        "pair count " + (pairs == UINT64_MAX ? std::string(">= 2^32") : std::to_string(pairs)) +
                            " exceeds budget " + std::to_string(ctx->f_cfg.pair_budget));
        }
        if (c.overflow || c.p_eff != c.p) {
            if (pairs >= (1ull << 31)) return fail(ctx, AGSX_ENOMEM, "pair count exceeds 2^31");
            ctx->pair_capacity = std::min<uint64_t>(pairs + pairs / 8 + 1024, ctx->f_cfg.pair_budget);
            const uint64_t tiles = static_cast<uint64_t>(ctx->f_params.tiles_x) * ctx->f_params.tiles_y;
            ensure_frame_buffers(ctx, ctx->f_scene->n, tiles,
                                 static_cast<uint64_t>(ctx->f_cam.width) * ctx->f_cam.height,
                                 ctx->f_cfg.mode == AGSX_MODE_OBB, ctx->f_cfg.pair_budget);
            enqueue_frame(ctx, ctx->f_scene, ctx->f_params, ctx->f_maxt, nullptr);
            continue;
        }
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
    return fail(ctx, AGSX_ECUDA, "pair arena did not converge");
}

}  // namespace

namespace {
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
}  // namespace

extern "C" {

int agsx_abi_version(void) { return AGSX_ABI_VERSION; }

int agsx_host_alloc(size_t bytes, void** out) {
    if (!out) return AGSX_EINVAL;
    *out = nullptr;
    const cudaError_t e = cudaHostAlloc(out, std::max<size_t>(bytes, 1), cudaHostAllocPortable);
    if (e != cudaSuccess) return e == cudaErrorMemoryAllocation ? AGSX_ENOMEM : AGSX_ECUDA;
    return AGSX_OK;
}

void agsx_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

}  // extern "C"

namespace {
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
}  // namespace

extern "C" {

int agsx_create(int device, agsx_ctx** out) {
    if (!out) return AGSX_EINVAL;
    *out = nullptr;
    agsx_ctx* ctx = new (std::nothrow) agsx_ctx();
    if (!ctx) return AGSX_ENOMEM;
    ctx->device = device;
    const int rc = guarded(ctx, [&]() -> int {
        AGSX_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        AGSX_CUDA(shared_copy_stream(device, &ctx->copy_stream));
        for (auto& e : ctx->band_ev) AGSX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        AGSX_CUDA(cudaEventCreateWithFlags(&ctx->copy_done, cudaEventDisableTiming));
        AGSX_CUDA(cudaEventCreateWithFlags(&ctx->ev_zeroed, cudaEventDisableTiming));
        AGSX_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
        AGSX_CUDA(sort_configure<uint32_t>(sort_smem(false), &ctx->occ_sort32));
        AGSX_CUDA(sort_configure<uint64_t>(sort_smem(true), &ctx->occ_sort64));
        AGSX_CUDA(emit_configure(false, &ctx->occ_emit));
        AGSX_CUDA(emit_configure(true, &ctx->occ_emit_big));
        ctx->occ_emit_big = std::max(ctx->occ_emit_big, 1);
        AGSX_CUDA(raster_units_occupancy(&ctx->occ_raster));
        ctx->occ_raster = std::max(ctx->occ_raster, 1);
        ctx->occ_sort32 = std::max(ctx->occ_sort32, 1);
        ctx->occ_sort64 = std::max(ctx->occ_sort64, 1);
        ctx->occ_emit = std::max(ctx->occ_emit, 1);
        for (auto& set : ctx->ev_ring)
            for (auto& e : set) AGSX_CUDA(cudaEventCreate(&e));
        AGSX_CUDA(cudaMallocHost(reinterpret_cast<void**>(&ctx->h_ctr), sizeof(Counters)));
        std::memset(ctx->h_ctr, 0, sizeof(Counters));
        AGSX_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->h_ctr_dev), ctx->h_ctr, 0));
        return AGSX_OK;
    });
    if (rc != AGSX_OK) {
        std::fprintf(stderr, "agsx_create: %s\n", ctx->err.c_str());
        agsx_destroy(ctx);
        return rc;
    }
    *out = ctx;
    return AGSX_OK;
}

void agsx_destroy(agsx_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    for (Buf* b : {&ctx->status, &ctx->p0, &ctx->p1, &ctx->p2, &ctx->p3, &ctx->p4, &ctx->dkeys,
                   &ctx->dvals, &ctx->dkeys2, &ctx->dvals2, &ctx->dcounts, &ctx->chunks, &ctx->img_u8, &ctx->tkeys, &ctx->pvals, &ctx->tkeys2,
                   &ctx->pvals2, &ctx->ranges, &ctx->image, &ctx->lb, &ctx->ctr, &ctx->hist,
                   &ctx->maxt, &ctx->dump, &ctx->lut_ext, &ctx->tile_pit, &ctx->calib, &ctx->sort_counts, &ctx->tmp0, &ctx->tmp1, &ctx->tmp2,
                   &ctx->tmp3, &ctx->tmp4})
        release(*b);
    for (auto& set : ctx->ev_ring)
        for (auto& e : set)
            if (e) cudaEventDestroy(e);
    if (ctx->h_ctr) cudaFreeHost(ctx->h_ctr);
    for (auto& e : ctx->band_ev)
        if (e) cudaEventDestroy(e);
    if (ctx->copy_done) cudaEventDestroy(ctx->copy_done);
    if (ctx->ev_zeroed) cudaEventDestroy(ctx->ev_zeroed);
    if (ctx->copy_stream) cudaStreamSynchronize(ctx->copy_stream);  // shared per device: not destroyed
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

const char* agsx_last_error(const agsx_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

void* agsx_stream(agsx_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

uint64_t agsx_kernel_launches(const agsx_ctx* ctx) { return ctx ? ctx->launches : 0; }

int agsx_scene_upload(agsx_ctx* ctx, const agsx_scene_desc* d, agsx_scene** out) {
    if (!ctx || !d || !out) return AGSX_EINVAL;
    *out = nullptr;
    const int D = d->sh_coeffs;
    if (!(D == 1 || D == 4 || D == 9 || D == 16))
        return fail(ctx, AGSX_EINVAL, "sh coefficient count must be 3*d^2 for d in {1,2,3,4}");
    agsx_scene* sc = new (std::nothrow) agsx_scene();
    if (!sc) return AGSX_ENOMEM;
    const int rc = guarded(ctx, [&]() -> int {
        sc->device = ctx->device;
        sc->n = d->count;
        sc->D = D;
        const uint64_t n = d->count;
        ensure(sc->pos_op, std::max<uint64_t>(n, 1) * 16);
        ensure(sc->rot, std::max<uint64_t>(n, 1) * 16);
        ensure(sc->scale_r, std::max<uint64_t>(n, 1) * 16);
        ensure(sc->sh_gb, std::max<uint64_t>(n, 1) * 8);
        ensure(sc->sh_rest, std::max<uint64_t>(n * (3 * D - 3), 1) * 4);
        if (n == 0) return AGSX_OK;
        // stage the host SoA arrays, pack on the device in slices
        const uint64_t slice = 1u << 22;
        const uint64_t fl_per = 3 + 3 + 4 + 1 + 3 * static_cast<uint64_t>(D);
        Buf stage;
        ensure(stage, std::min(n, slice) * fl_per * 4);
        float* s = ptr<float>(stage);
        for (uint64_t b = 0; b < n; b += slice) {
            const uint64_t m = std::min(slice, n - b);
            float* sm = s;
            float* ss = sm + 3 * m;
            float* sq = ss + 3 * m;
            float* so = sq + 4 * m;
            float* sh = so + m;
            AGSX_CUDA(cudaMemcpyAsync(sm, d->mean + 3 * b, 12 * m, cudaMemcpyHostToDevice, ctx->stream));
            AGSX_CUDA(cudaMemcpyAsync(ss, d->scale + 3 * b, 12 * m, cudaMemcpyHostToDevice, ctx->stream));
            AGSX_CUDA(cudaMemcpyAsync(sq, d->rotation + 4 * b, 16 * m, cudaMemcpyHostToDevice, ctx->stream));
            AGSX_CUDA(cudaMemcpyAsync(so, d->opacity + b, 4 * m, cudaMemcpyHostToDevice, ctx->stream));
            AGSX_CUDA(cudaMemcpyAsync(sh, d->sh + 3 * D * b, 12 * D * m, cudaMemcpyHostToDevice, ctx->stream));
            k_pack_scene<<<static_cast<int>((m + 255) / 256), 256, 0, ctx->stream>>>(
                m, D, sm, ss, sq, so, sh, ptr<float4>(sc->pos_op) + b, ptr<float4>(sc->rot) + b,
                ptr<float4>(sc->scale_r) + b, ptr<float2>(sc->sh_gb) + b,
                ptr<float>(sc->sh_rest) + b * (3 * D - 3));
            check_launch(ctx);
        }
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        release(stage);
        return AGSX_OK;
    });
    if (rc != AGSX_OK) {
        agsx_scene_free(sc);
        return rc;
    }
    *out = sc;
    return AGSX_OK;
}

void agsx_scene_free(agsx_scene* sc) {
    if (!sc) return;
    cudaSetDevice(sc->device);
    for (Buf* b : {&sc->pos_op, &sc->rot, &sc->scale_r, &sc->sh_gb, &sc->sh_rest}) release(*b);
    delete sc;
}

uint64_t agsx_scene_count(const agsx_scene* sc) { return sc ? sc->n : 0; }

int agsx_render_async(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam,
                      const agsx_config* cfg, const agsx_lut* lut) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int { return start_frame(ctx, scene, cam, cfg, lut, false); });
}

// Experiment hook (not in agsx.h): the enqueued frame captured once as a CUDA
// graph and replayed `iters` times; *ms = device time per replay.
extern "C" int agsx_debug_graph_replay(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam,
                                       const agsx_config* cfg, const agsx_lut* lut, int iters, float* ms) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        int rc = start_frame(ctx, scene, cam, cfg, lut, false);  // sizes the arenas
        if (rc) return rc;
        rc = finish_frame(ctx, nullptr);
        if (rc) return rc;
        cudaGraph_t g;
        AGSX_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
        enqueue_frame(ctx, scene, ctx->f_params, false, nullptr);
        AGSX_CUDA(cudaStreamEndCapture(ctx->stream, &g));
        cudaGraphExec_t ge;
        AGSX_CUDA(cudaGraphInstantiate(&ge, g, 0));
        cudaEvent_t a, b;
        AGSX_CUDA(cudaEventCreate(&a));
        AGSX_CUDA(cudaEventCreate(&b));
        for (int i = 0; i < 3; ++i) AGSX_CUDA(cudaGraphLaunch(ge, ctx->stream));
        AGSX_CUDA(cudaEventRecord(a, ctx->stream));
        for (int i = 0; i < iters; ++i) AGSX_CUDA(cudaGraphLaunch(ge, ctx->stream));
        AGSX_CUDA(cudaEventRecord(b, ctx->stream));
        AGSX_CUDA(cudaEventSynchronize(b));
        AGSX_CUDA(cudaEventElapsedTime(ms, a, b));
        *ms /= iters;
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
        return AGSX_OK;
    });
}

int agsx_render_async_to(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam,
                         const agsx_config* cfg, const agsx_lut* lut, float* target) {
    if (!ctx) return AGSX_EINVAL;
    if (!target) return fail(ctx, AGSX_EINVAL, "render_async_to: null target");
    return guarded(ctx, [&]() -> int { return start_frame(ctx, scene, cam, cfg, lut, false, nullptr, target); });
}

int agsx_render_async_host(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam,
                           const agsx_config* cfg, const agsx_lut* lut, float* image) {
    if (!ctx) return AGSX_EINVAL;
    if (!image) return fail(ctx, AGSX_EINVAL, "render_async_host: null image");
    return guarded(ctx, [&]() -> int {
        const int rc = start_frame(ctx, scene, cam, cfg, lut, false, image);
        if (rc == AGSX_OK) ctx->f_host_dst = image;
        return rc;
    });
}

int agsx_render_wait(agsx_ctx* ctx, agsx_frame* out) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        float* dst = ctx->f_host_dst;
        uint8_t* dst8 = ctx->f_host_dst_u8;
        ctx->f_host_dst = nullptr;
        ctx->f_host_dst_u8 = nullptr;
        const int rc = finish_frame(ctx, out);
        if (rc) return rc;
        if (dst8) return ctx->f_band_host_u8 ? AGSX_OK : quantize_to_host(ctx, dst8);
        if (!dst || ctx->f_image_on_host) return rc;
        AGSX_CUDA(cudaMemcpyAsync(dst, ctx->image.p, static_cast<size_t>(ctx->f_cam.width) * ctx->f_cam.height * 12,
                                  cudaMemcpyDeviceToHost, ctx->stream));
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        return AGSX_OK;
    });
}

int agsx_render(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam,
                const agsx_config* cfg, const agsx_lut* lut, agsx_frame* out) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        const bool maxt = out && out->max_t;
        int rc = start_frame(ctx, scene, cam, cfg, lut, maxt, out ? out->image : nullptr);
        if (rc) return rc;
        rc = finish_frame(ctx, out);
        if (rc) return rc;
        if (out && out->image && !ctx->f_image_on_host) {
            AGSX_CUDA(cudaMemcpyAsync(out->image, ctx->image.p,
                                      static_cast<size_t>(cam->width) * cam->height * 12,
                                      cudaMemcpyDeviceToHost, ctx->stream));
        }
        if (maxt && scene->n) {
            AGSX_CUDA(cudaMemcpyAsync(out->max_t, ctx->maxt.p, scene->n * 4, cudaMemcpyDeviceToHost,
                                      ctx->stream));
        }
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        return AGSX_OK;
    });
}

int agsx_render_u8(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam, const agsx_config* cfg,
                   const agsx_lut* lut, uint8_t* image_u8, agsx_frame* out) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        if (!image_u8) return fail(ctx, AGSX_EINVAL, "render_u8: null image");
        int rc = start_frame(ctx, scene, cam, cfg, lut, false, nullptr, nullptr, image_u8);
        if (rc) return rc;
        rc = finish_frame(ctx, out);
        if (rc) return rc;
        if (ctx->f_band_host_u8) return AGSX_OK;  // bands already copied behind the raster
        return quantize_to_host(ctx, image_u8);
    });
}

int agsx_render_async_host_u8(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam,
                              const agsx_config* cfg, const agsx_lut* lut, uint8_t* image_u8) {
    if (!ctx) return AGSX_EINVAL;
    if (!image_u8) return fail(ctx, AGSX_EINVAL, "render_async_host_u8: null image");
    return guarded(ctx, [&]() -> int {
        const int rc = start_frame(ctx, scene, cam, cfg, lut, false, nullptr, nullptr, image_u8);
        if (rc == AGSX_OK) ctx->f_host_dst_u8 = image_u8;
        return rc;
    });
}

int agsx_render_contributions(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam,
                              const agsx_config* cfg, const agsx_lut* lut, agsx_blend_record* records,
                              uint64_t capacity, uint64_t* count, agsx_frame* out) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        if (!cfg || !count) return fail(ctx, AGSX_EINVAL, "render_contributions: null config or count");
        agsx_config c = *cfg;
        c.flags |= AGSX_FLAG_EXACT_ALPHA;  // the stream records the reference's alpha values
        const bool maxt = out && out->max_t;
        int rc = start_frame(ctx, scene, cam, &c, lut, maxt, out ? out->image : nullptr);
        if (rc) return rc;
        rc = finish_frame(ctx, out);
        if (rc) return rc;
        const FrameParams& p = ctx->f_params;
        const uint64_t tiles = static_cast<uint64_t>(p.tiles_x) * p.tiles_y;
        const uint64_t n = scene->n;
        if (out && out->image && !ctx->f_image_on_host)
            AGSX_CUDA(cudaMemcpyAsync(out->image, ctx->image.p, static_cast<size_t>(cam->width) * cam->height * 12,
                                      cudaMemcpyDeviceToHost, ctx->stream));
        if (maxt && n)
            AGSX_CUDA(cudaMemcpyAsync(out->max_t, ctx->maxt.p, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
        // pass 1: events per tile; host scan -> per-tile offsets in tile order
        ensure(ctx->tmp1, std::max<uint64_t>(tiles, 1) * 4);
        ensure(ctx->tmp2, std::max<uint64_t>(tiles, 1) * 8);
        const SplatPlanes pl = planes_of(ctx);
        AGSX_CUDA(launch_raster_records(ctx->stream, p, ptr<uint2>(ctx->ranges), ctx->f_pvals, pl.p0, pl.p1, pl.p2,
                                        ptr<float>(ctx->image), ptr<uint32_t>(ctx->tmp1), nullptr, nullptr));
        ++ctx->launches;
        std::vector<uint32_t> per_tile(tiles);
        std::vector<uint64_t> off(tiles);
        if (tiles)
            AGSX_CUDA(cudaMemcpyAsync(per_tile.data(), ctx->tmp1.p, tiles * 4, cudaMemcpyDeviceToHost, ctx->stream));
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        uint64_t total = 0;
        for (uint64_t t = 0; t < tiles; ++t) {
            off[t] = total;
            total += per_tile[t];
        }
        *count = total;
        if (!records || capacity < total)
            return fail(ctx, AGSX_ECAPACITY, "render_contributions: " + std::to_string(total) + " records");
        if (total == 0) return AGSX_OK;
        // pass 2: the records, then Gaussian id -> index in the view's splat sequence
        ensure(ctx->tmp3, total * sizeof(agsx_blend_record));
        AGSX_CUDA(cudaMemcpyAsync(ctx->tmp2.p, off.data(), tiles * 8, cudaMemcpyHostToDevice, ctx->stream));
        AGSX_CUDA(launch_raster_records(ctx->stream, p, ptr<uint2>(ctx->ranges), ctx->f_pvals, pl.p0, pl.p1, pl.p2,
                                        ptr<float>(ctx->image), nullptr, ptr<uint64_t>(ctx->tmp2),
                                        ptr<agsx_blend_record>(ctx->tmp3)));
        ++ctx->launches;
        AGSX_CUDA(cudaMemcpyAsync(records, ctx->tmp3.p, total * sizeof(agsx_blend_record), cudaMemcpyDeviceToHost,
                                  ctx->stream));
        std::vector<uint32_t> st(n);
        if (n) AGSX_CUDA(cudaMemcpyAsync(st.data(), ctx->status.p, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        std::vector<uint32_t> view_index(n);
        uint32_t k = 0;
        for (uint64_t i = 0; i < n; ++i) {  // survivors in Gaussian order (preprocess.cpp:158-162)
            view_index[i] = k;
            k += (st[i] & kAliveBit) ? 1u : 0u;
        }
        for (uint64_t i = 0; i < total; ++i) records[i].splat = view_index[records[i].splat];
        return AGSX_OK;
    });
}

int agsx_stage_history(agsx_ctx* ctx, float* stage_ms, int32_t max_frames, int32_t* out_frames) {
    if (!ctx || !stage_ms || !out_frames) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        const uint64_t avail = std::min<uint64_t>(ctx->frames, agsx_ctx::kRing);
        const int n = static_cast<int>(std::min<uint64_t>(avail, static_cast<uint64_t>(std::max(max_frames, 0))));
        for (int i = 0; i < n; ++i) {
            // oldest first among the last n frames
            const uint64_t f = ctx->frames - n + i;
            cudaEvent_t* e = ctx->ev_ring[f % agsx_ctx::kRing];
            float ms[5];
            for (int k = 0; k < 5; ++k) AGSX_CUDA(cudaEventElapsedTime(&ms[k], e[k], e[k + 1]));
            stage_ms[4 * i + 0] = ms[0];
            stage_ms[4 * i + 1] = ms[2];
            stage_ms[4 * i + 2] = ms[1] + ms[3];
            stage_ms[4 * i + 3] = ms[4];
        }
        *out_frames = n;
        return AGSX_OK;
    });
}

int agsx_frame_stats(agsx_ctx* ctx, uint64_t* stats, int32_t n) {
    if (!ctx || !stats) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        const Counters c = *ctx->h_ctr;
        const uint64_t v[13] = {c.s, c.m, c.p, c.p_it, c.overflow, static_cast<uint64_t>(ctx->f_tile_count),
                                c.dbg[0], c.dbg[1], c.dbg[2], c.dbg[3], c.dbg[4], c.dbg[5], c.dbg[6]};
        for (int i = 0; i < n && i < 13; ++i) stats[i] = v[i];
        return AGSX_OK;
    });
}

int agsx_device_image(agsx_ctx* ctx, float** dptr, int32_t* width, int32_t* height) {
    if (!ctx || !dptr) return AGSX_EINVAL;
    if (!ctx->have_frame) return fail(ctx, AGSX_EINVAL, "no frame rendered yet");
    if (ctx->f_image_on_host) return fail(ctx, AGSX_EINVAL, "the last frame was rasterised into a caller buffer");
    *dptr = ptr<float>(ctx->image);
    if (width) *width = ctx->f_cam.width;
    if (height) *height = ctx->f_cam.height;
    return AGSX_OK;
}

int agsx_dump_tile_counts(agsx_ctx* ctx, uint32_t* counts, uint8_t* alive, uint64_t n) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        if (!ctx->have_frame) return fail(ctx, AGSX_EINVAL, "no frame rendered yet");
        if (n != ctx->f_scene->n) return fail(ctx, AGSX_EINVAL, "count mismatch");
        std::vector<uint32_t> st(n);
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        if (n) AGSX_CUDA(cudaMemcpy(st.data(), ctx->status.p, n * 4, cudaMemcpyDeviceToHost));
        for (uint64_t i = 0; i < n; ++i) {
            if (counts) counts[i] = st[i] & kCountMask;
            if (alive) alive[i] = (st[i] & kAliveBit) ? 1 : 0;
        }
        return AGSX_OK;
    });
}

int agsx_dump_sorted_pairs(agsx_ctx* ctx, uint64_t* keys, uint32_t* gids, uint64_t capacity,
                           uint64_t* out_count) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        if (!ctx->have_frame) return fail(ctx, AGSX_EINVAL, "no frame rendered yet");
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        const Counters c = *ctx->h_ctr;
        const uint64_t P = c.p_eff;
        if (out_count) *out_count = P;
        if (P > capacity) return fail(ctx, AGSX_ECAPACITY, "buffer too small");
        const uint64_t n = ctx->f_scene->n;
        std::vector<uint32_t> dk(c.m), dv(c.m), tk(P), pv(P);
        if (c.m) {
            const bool wide = depth_keys_wide_host(c);  // which ping-pong buffer holds the depth order
            AGSX_CUDA(cudaMemcpy(dk.data(), wide ? ctx->dkeys.p : ctx->dkeys2.p, c.m * 4, cudaMemcpyDeviceToHost));
            AGSX_CUDA(cudaMemcpy(dv.data(), wide ? ctx->dvals.p : ctx->dvals2.p, c.m * 4, cudaMemcpyDeviceToHost));
        }
        if (P) {
            AGSX_CUDA(cudaMemcpy(tk.data(), ctx->f_tkeys, P * 4, cudaMemcpyDeviceToHost));
            AGSX_CUDA(cudaMemcpy(pv.data(), ctx->f_pvals, P * 4, cudaMemcpyDeviceToHost));
        }
        std::vector<uint32_t> depth_by_gid(n, 0);
        for (uint32_t j = 0; j < c.m; ++j) depth_by_gid[dv[j]] = dk[j];
        for (uint64_t i = 0; i < P; ++i) {
            if (keys) keys[i] = (static_cast<uint64_t>(tk[i]) << 32) | depth_by_gid[pv[i]];
            if (gids) gids[i] = pv[i];
        }
        return AGSX_OK;
    });
}

int agsx_dump_ranges(agsx_ctx* ctx, uint32_t* ranges, uint64_t tile_count) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        if (!ctx->have_frame) return fail(ctx, AGSX_EINVAL, "no frame rendered yet");
        if (tile_count != static_cast<uint64_t>(ctx->f_tile_count))
            return fail(ctx, AGSX_EINVAL, "tile count mismatch");
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        if (tile_count)
            AGSX_CUDA(cudaMemcpy(ranges, ctx->ranges.p, tile_count * 8, cudaMemcpyDeviceToHost));
        return AGSX_OK;
    });
}

int agsx_preprocess_view(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam,
                         const agsx_config* cfg, const agsx_lut* lut, agsx_splat_view* out,
                         uint64_t* out_count) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        if (!scene) return fail(ctx, AGSX_EINVAL, "null scene");
        // preprocess_view validates only the LUT requirement (preprocess.cpp:121-125)
        if (cfg->mode == AGSX_MODE_ADAGSCALE && lut == nullptr)
            return fail(ctx, AGSX_EINVAL, "preprocess_view: adagscale mode requires a T-upper LUT");
        agsx_config c = *cfg;
        if (c.tile_size < 1) c.tile_size = 16;
        FrameParams p;
        const float* lut_dev = nullptr;
        if (lut && lut->bin_count > kLutInline) {
            ensure(ctx->lut_ext, lut->bin_count * sizeof(float));
            AGSX_CUDA(cudaMemcpy(ctx->lut_ext.p, lut->bins, lut->bin_count * 4, cudaMemcpyHostToDevice));
            lut_dev = ptr<float>(ctx->lut_ext);
        }
        p = make_params(*cam, c, c.mode == AGSX_MODE_ADAGSCALE ? lut : nullptr, lut_dev);
        const uint64_t n = scene->n;
        const uint64_t tiles = static_cast<uint64_t>(p.tiles_x) * p.tiles_y;
        ensure_frame_buffers(ctx, n, tiles, static_cast<uint64_t>(cam->width) * cam->height,
                             c.mode == AGSX_MODE_OBB, c.pair_budget);
        ensure(ctx->dump, std::max<uint64_t>(n, 1) * sizeof(agsx_splat_view));
        Counters* ctr = ptr<Counters>(ctx->ctr);
        AGSX_CUDA(cudaMemsetAsync(ctr, 0, sizeof(Counters), ctx->stream));
        if (n) {
            k_preprocess<<<static_cast<int>((n + 255) / 256), 256, 0, ctx->stream>>>(
                p, scene->view(), planes_of(ctx), ptr<uint32_t>(ctx->status), ptr<uint32_t>(ctx->dkeys), ctr,
                ptr<agsx_splat_view>(ctx->dump));
            check_launch(ctx);
        }
        std::vector<uint32_t> st(n);
        std::vector<agsx_splat_view> sv(n);
        if (n) {
            AGSX_CUDA(cudaMemcpyAsync(st.data(), ctx->status.p, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
            AGSX_CUDA(cudaMemcpyAsync(sv.data(), ctx->dump.p, n * sizeof(agsx_splat_view),
                                      cudaMemcpyDeviceToHost, ctx->stream));
        }
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        uint64_t m = 0;
        for (uint64_t i = 0; i < n; ++i)
            if (st[i] & kAliveBit) out[m++] = sv[i];
        *out_count = m;
        ctx->have_frame = false;
        return AGSX_OK;
    });
}

int agsx_generate_pairs(agsx_ctx* ctx, const agsx_splat_view* splats, uint64_t n, int32_t width,
                        int32_t height, int32_t mode, const agsx_config* cfg, uint64_t* keys,
                        uint32_t* splat_index, uint64_t capacity, uint32_t* tile_counts,
                        uint64_t* out_total) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        if (cfg->tile_size < 1) return fail(ctx, AGSX_EINVAL, "tile_size must be >= 1");
        agsx_config c = *cfg;
        c.mode = mode;
        agsx_camera cam{};
        cam.width = width;
        cam.height = height;
        cam.fx = cam.fy = 1.0f;
        const FrameParams p = make_params(cam, c, nullptr, nullptr);
        ensure(ctx->tmp0, std::max<uint64_t>(n, 1) * sizeof(agsx_splat_view));
        ensure(ctx->tmp1, std::max<uint64_t>(n, 1) * 4);  // counts
        ensure(ctx->tmp2, std::max<uint64_t>(n, 1) * 4);  // depth bits
        ensure(ctx->tmp3, std::max<uint64_t>(n, 1) * 8);  // offsets
        for (Buf* b : {&ctx->p0, &ctx->p1, &ctx->p2, &ctx->p3, &ctx->p4})
            ensure(*b, std::max<uint64_t>(n, 1) * 16);
        const SplatPlanes pl = planes_of(ctx);
        if (n) {
            AGSX_CUDA(cudaMemcpyAsync(ctx->tmp0.p, splats, n * sizeof(agsx_splat_view),
                                      cudaMemcpyHostToDevice, ctx->stream));
            k_splats_to_planes<<<static_cast<int>((n + 255) / 256), 256, 0, ctx->stream>>>(
                p, ptr<agsx_splat_view>(ctx->tmp0), n, pl, ptr<uint32_t>(ctx->tmp1), ptr<uint32_t>(ctx->tmp2));
            check_launch(ctx);
        }
        std::vector<uint32_t> cnt(n);
        if (n) AGSX_CUDA(cudaMemcpyAsync(cnt.data(), ctx->tmp1.p, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        std::vector<uint64_t> off(n);
        uint64_t total = 0;
        for (uint64_t i = 0; i < n; ++i) {
            off[i] = total;
            total += cnt[i];
            if (tile_counts) tile_counts[i] = cnt[i];
        }
        *out_total = total;
        if (total > cfg->pair_budget)
            return fail(ctx, AGSX_EPAIR_BUDGET, "pair count " + std::to_string(total) + " exceeds budget " +
                                                    std::to_string(cfg->pair_budget));
        if (total > capacity) return fail(ctx, AGSX_ECAPACITY, "output buffers too small");
        if (total == 0) return AGSX_OK;
        ensure(ctx->tmp4, total * 8);
        ensure(ctx->pvals, total * 4);
        AGSX_CUDA(cudaMemcpyAsync(ctx->tmp3.p, off.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream));
        k_emit_list<<<static_cast<int>((n + 255) / 256), 256, 0, ctx->stream>>>(
            p, n, pl, ptr<uint32_t>(ctx->tmp1), ptr<uint64_t>(ctx->tmp3), ptr<uint32_t>(ctx->tmp2),
            ptr<uint64_t>(ctx->tmp4), ptr<uint32_t>(ctx->pvals));
        check_launch(ctx);
        AGSX_CUDA(cudaMemcpyAsync(keys, ctx->tmp4.p, total * 8, cudaMemcpyDeviceToHost, ctx->stream));
        AGSX_CUDA(cudaMemcpyAsync(splat_index, ctx->pvals.p, total * 4, cudaMemcpyDeviceToHost, ctx->stream));
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        ctx->have_frame = false;
        return AGSX_OK;
    });
}

int agsx_sort_pairs(agsx_ctx* ctx, uint64_t* keys, uint32_t* splat_index, uint64_t n,
                    int32_t tile_count, uint32_t* ranges) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        if (tile_count < 0) return fail(ctx, AGSX_EINVAL, "negative tile count");
        if (n >= (1ull << 32)) return fail(ctx, AGSX_EINVAL, "too many pairs");
        ensure(ctx->tmp0, std::max<uint64_t>(n, 1) * 8);
        ensure(ctx->tmp1, std::max<uint64_t>(n, 1) * 8);
        ensure(ctx->tmp2, std::max<uint64_t>(n, 1) * 4);
        ensure(ctx->tmp3, std::max<uint64_t>(n, 1) * 4);
        ensure(ctx->hist, 9 * 256 * 4);
        ensure(ctx->ranges, std::max<int>(tile_count, 1) * 8);
        ensure_lb(ctx, n);
        uint32_t* hist = ptr<uint32_t>(ctx->hist);
        cudaStream_t st = ctx->stream;
        AGSX_CUDA(cudaMemsetAsync(ctx->hist.p, 0, 9 * 256 * 4, st));
        if (tile_count) AGSX_CUDA(cudaMemsetAsync(ctx->ranges.p, 0, static_cast<size_t>(tile_count) * 8, st));
        uint64_t* k[2] = {ptr<uint64_t>(ctx->tmp0), ptr<uint64_t>(ctx->tmp1)};
        uint32_t* v[2] = {ptr<uint32_t>(ctx->tmp2), ptr<uint32_t>(ctx->tmp3)};
        int cur = 0;
        if (n) {
            AGSX_CUDA(cudaMemcpyAsync(k[0], keys, n * 8, cudaMemcpyHostToDevice, st));
            AGSX_CUDA(cudaMemcpyAsync(v[0], splat_index, n * 4, cudaMemcpyHostToDevice, st));
            sort_hist<uint64_t>(ctx, k[0], nullptr, n, 8, false, hist);
            std::vector<uint32_t> h(8 * 256);
            AGSX_CUDA(cudaMemcpyAsync(h.data(), hist, h.size() * 4, cudaMemcpyDeviceToHost, st));
            AGSX_CUDA(cudaStreamSynchronize(st));
            for (int ps = 0; ps < 8; ++ps) {
                // a digit shared by every key permutes nothing in a stable pass
                bool trivial = false;
                for (int d = 0; d < 256; ++d) trivial = trivial || h[ps * 256 + d] == n;
                if (trivial) continue;
                sort_pass<uint64_t>(ctx, k[cur], v[cur], k[cur ^ 1], v[cur ^ 1], nullptr, n, 8 * ps, false,
                                    nullptr);
                cur ^= 1;
            }
            if (tile_count) {
                k_ranges_u64<<<ctx->num_sms * 4, 256, 0, st>>>(k[cur], n, static_cast<uint32_t>(tile_count),
                                                                ptr<uint2>(ctx->ranges));
                check_launch(ctx);
            }
            AGSX_CUDA(cudaMemcpyAsync(keys, k[cur], n * 8, cudaMemcpyDeviceToHost, st));
            AGSX_CUDA(cudaMemcpyAsync(splat_index, v[cur], n * 4, cudaMemcpyDeviceToHost, st));
        }
        if (tile_count)
            AGSX_CUDA(cudaMemcpyAsync(ranges, ctx->ranges.p, static_cast<size_t>(tile_count) * 8,
                                      cudaMemcpyDeviceToHost, st));
        AGSX_CUDA(cudaStreamSynchronize(st));
        ctx->have_frame = false;
        return AGSX_OK;
    });
}

int agsx_raster(agsx_ctx* ctx, const agsx_splat_view* splats, uint64_t n_splats,
                const uint32_t* splat_index, uint64_t n_pairs, const uint32_t* ranges, int32_t width,
                int32_t height, const agsx_config* cfg, float* image, float* max_t) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        if (cfg->tile_size < 1 || cfg->tile_size > 64)
            return fail(ctx, AGSX_EINVAL, "tile_size must be in [1, 64]");
        if (width <= 0 || height <= 0) return fail(ctx, AGSX_EINVAL, "image dimensions must be positive");
        agsx_camera cam{};
        cam.width = width;
        cam.height = height;
        cam.fx = cam.fy = 1.0f;
        const FrameParams p = make_params(cam, *cfg, nullptr, nullptr);
        const uint64_t tiles = static_cast<uint64_t>(p.tiles_x) * p.tiles_y;
        ensure(ctx->tmp0, std::max<uint64_t>(n_splats, 1) * sizeof(agsx_splat_view));
        ensure(ctx->tmp1, std::max<uint64_t>(n_splats, 1) * 4);
        ensure(ctx->tmp2, std::max<uint64_t>(n_splats, 1) * 4);
        ensure(ctx->tmp3, std::max<uint64_t>(n_pairs, 1) * 4);
        ensure(ctx->tmp4, std::max<uint64_t>(tiles, 1) * 8);
        ensure(ctx->image, static_cast<uint64_t>(width) * height * 12);
        ensure(ctx->maxt, std::max<uint64_t>(n_splats, 1) * 4);
        for (Buf* b : {&ctx->p0, &ctx->p1, &ctx->p2, &ctx->p3, &ctx->p4})
            ensure(*b, std::max<uint64_t>(n_splats, 1) * 16);
        const SplatPlanes pl = planes_of(ctx);
        cudaStream_t st = ctx->stream;
        if (n_splats) {
            AGSX_CUDA(cudaMemcpyAsync(ctx->tmp0.p, splats, n_splats * sizeof(agsx_splat_view),
                                      cudaMemcpyHostToDevice, st));
            k_splats_to_planes<<<static_cast<int>((n_splats + 255) / 256), 256, 0, st>>>(
                p, ptr<agsx_splat_view>(ctx->tmp0), n_splats, pl, ptr<uint32_t>(ctx->tmp1),
                ptr<uint32_t>(ctx->tmp2));
            check_launch(ctx);
        }
        if (n_pairs)
            AGSX_CUDA(cudaMemcpyAsync(ctx->tmp3.p, splat_index, n_pairs * 4, cudaMemcpyHostToDevice, st));
        AGSX_CUDA(cudaMemcpyAsync(ctx->tmp4.p, ranges, tiles * 8, cudaMemcpyHostToDevice, st));
        if (max_t) AGSX_CUDA(cudaMemsetAsync(ctx->maxt.p, 0, std::max<uint64_t>(n_splats, 1) * 4, st));
        ensure(ctx->ctr, counters_bytes());
        AGSX_CUDA(cudaMemsetAsync(ctx->ctr.p, 0, counters_bytes(), st));
        Counters* ctr = ptr<Counters>(ctx->ctr);
        if (raster_uses_units(p, max_t != nullptr)) {
            ensure(ctx->tile_pit, std::max<uint64_t>(tiles, 1) * 8);
            AGSX_CUDA(cudaMemsetAsync(ctx->tile_pit.p, 0, tiles * 8, st));
        }
        launch_raster(ctx, p, ptr<uint2>(ctx->tmp4), ptr<uint32_t>(ctx->tmp3), pl.p0, pl.p1, pl.p2,
                      ptr<float>(ctx->image), max_t ? ptr<uint32_t>(ctx->maxt) : nullptr, ctr);
        AGSX_CUDA(cudaMemcpyAsync(image, ctx->image.p, static_cast<size_t>(width) * height * 12,
                                  cudaMemcpyDeviceToHost, st));
        if (max_t && n_splats)
            AGSX_CUDA(cudaMemcpyAsync(max_t, ctx->maxt.p, n_splats * 4, cudaMemcpyDeviceToHost, st));
        AGSX_CUDA(cudaStreamSynchronize(st));
        ctx->have_frame = false;
        return AGSX_OK;
    });
}

int agsx_device_alloc(agsx_ctx* ctx, size_t bytes, void** out) {
    if (!ctx || !out) return AGSX_EINVAL;
    *out = nullptr;
    return guarded(ctx, [&]() -> int {
        AGSX_CUDA(cudaMalloc(out, std::max<size_t>(bytes, 1)));
        return AGSX_OK;
    });
}

void agsx_device_free(agsx_ctx* ctx, void* p) {
    if (!ctx || !p) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    cudaFree(p);
}

int agsx_fold_max_t(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam, const agsx_config* cfg,
                    const agsx_lut* lut_shape, float* folded, uint8_t* observed) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        if (!cfg || !lut_shape || lut_shape->bin_count < 1 || !folded || !observed)
            return fail(ctx, AGSX_EINVAL, "fold_max_t: bad arguments");
        agsx_config c = *cfg;
        c.mode = AGSX_MODE_ELLIPSE;  // build_lut renders losslessly (calibrate.cpp:22-23)
        c.flags |= AGSX_FLAG_EXACT_ALPHA;
        int rc = start_frame(ctx, scene, cam, &c, nullptr, true);
        if (rc) return rc;
        rc = finish_frame(ctx, nullptr);
        if (rc) return rc;
        const int nb = lut_shape->bin_count;
        ensure(ctx->calib, static_cast<size_t>(2 * nb) * 4 + 4096 * 8 + 8);
        uint32_t* dfold = ptr<uint32_t>(ctx->calib);
        AGSX_CUDA(cudaMemsetAsync(dfold, 0, static_cast<size_t>(2 * nb) * 4, ctx->stream));
        if (scene->n) {
            const bool wide = depth_keys_wide_host(*ctx->h_ctr);  // finish_frame synchronised
            k_fold_max_t<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(
                ptr<uint32_t>(wide ? ctx->dvals : ctx->dvals2), ptr<uint32_t>(wide ? ctx->dkeys : ctx->dkeys2),
                &ptr<Counters>(ctx->ctr)->m,
                ptr<uint32_t>(ctx->maxt), lut_shape->depth_min, lut_shape->depth_max, nb, dfold, dfold + nb);
            check_launch(ctx);
        }
        std::vector<uint32_t> h(static_cast<size_t>(2 * nb));
        AGSX_CUDA(cudaMemcpyAsync(h.data(), dfold, h.size() * 4, cudaMemcpyDeviceToHost, ctx->stream));
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        for (int b = 0; b < nb; ++b) {
            float v;
            std::memcpy(&v, &h[b], 4);
            if (h[nb + b]) {
                observed[b] = 1;
                folded[b] = std::max(folded[b], v);
            }
        }
        return AGSX_OK;
    });
}

int agsx_sq_err(agsx_ctx* ctx, const float* a, const float* b, uint64_t n, double* out) {
    if (!ctx || !out) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        constexpr int kBlocks = 1024;  // fixed: the summation order is the same every call
        ensure(ctx->calib, 4096 * 8 + 8 + 1024);
        double* part = reinterpret_cast<double*>(static_cast<char*>(ctx->calib.p) + 1024);
        double* res = part + kBlocks;
        k_sq_err_partial<<<kBlocks, 256, 0, ctx->stream>>>(a, b, n, part);
        check_launch(ctx);
        k_sq_err_final<<<1, 32, 0, ctx->stream>>>(part, kBlocks, res);
        check_launch(ctx);
        AGSX_CUDA(cudaMemcpyAsync(out, res, 8, cudaMemcpyDeviceToHost, ctx->stream));
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        return AGSX_OK;
    });
}

int agsx_device_logf(agsx_ctx* ctx, const float* x, float* y, uint64_t n) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        ensure(ctx->tmp0, std::max<uint64_t>(n, 1) * 4);
        ensure(ctx->tmp1, std::max<uint64_t>(n, 1) * 4);
        if (!n) return AGSX_OK;
        AGSX_CUDA(cudaMemcpyAsync(ctx->tmp0.p, x, n * 4, cudaMemcpyHostToDevice, ctx->stream));
        k_logf<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(ptr<float>(ctx->tmp0), ptr<float>(ctx->tmp1), n);
        check_launch(ctx);
        AGSX_CUDA(cudaMemcpyAsync(y, ctx->tmp1.p, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        return AGSX_OK;
    });
}

int agsx_device_expf(agsx_ctx* ctx, const float* x, float* y, uint64_t n) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        ensure(ctx->tmp0, std::max<uint64_t>(n, 1) * 4);
        ensure(ctx->tmp1, std::max<uint64_t>(n, 1) * 4);
        if (!n) return AGSX_OK;
        AGSX_CUDA(cudaMemcpyAsync(ctx->tmp0.p, x, n * 4, cudaMemcpyHostToDevice, ctx->stream));
        k_expf<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(ptr<float>(ctx->tmp0), ptr<float>(ctx->tmp1), n);
        check_launch(ctx);
        AGSX_CUDA(cudaMemcpyAsync(y, ctx->tmp1.p, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        return AGSX_OK;
    });
}

}  // extern "C"

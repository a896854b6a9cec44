// agsx_ctx.cuh -- host-side state of libagsx.so shared by its translation
// units: device arenas (Buf), the context and scene objects, the error
// plumbing of the C-ABI (StatusError -> int status), and the frame pipeline
// of agsx_frame.cu (validation, launch sequence, egress, waiting).
//
//   agsx_frame.cu      one frame: prepare -> enqueue -> finish, host egress
//   agsx_api.cu        C-ABI: contexts, scenes, render entry points, dumps
//   agsx_stage_api.cu  C-ABI: stage hooks, calibration primitives, libm pins
//
// Internal header: only those files include it.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

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

// NVTX ranges (stage tracing) around the host side of a frame,
// named after the reference's stage_times keys (rasterizer.cpp:126-163):
// agsx.render / preprocess / pair_gen / sort / raster / wait.  NVTX3 is
// header-only; without a tool attached a range costs a few ns.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

namespace agsx::host {

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


}  // namespace agsx::host

using namespace agsx;
using namespace agsx::host;

struct agsx_scene {
    int device = 0;
    uint64_t n = 0;
    int D = 1;
    Buf pos_op, rot, scale_r, sh_gb, sh_rest;
    Buf orig, inv;  // storage order (DevScene); empty: slot = id
    float max_opacity = INFINITY;  // over the scene (NaN counts as +inf): picks the clamp-free raster
    DevScene view() const {
        DevScene s;
        s.n = n;
        s.sh_coeffs = D;
        s.pos_op = static_cast<const float4*>(pos_op.p);
        s.rot = static_cast<const float4*>(rot.p);
        s.scale_r = static_cast<const float4*>(scale_r.p);
        s.sh_gb = static_cast<const float2*>(sh_gb.p);
        s.sh_rest = static_cast<const float*>(sh_rest.p);
        s.orig = static_cast<const uint32_t*>(orig.p);
        s.inv = static_cast<const uint32_t*>(inv.p);
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
    int occ_sort32 = 1, occ_sort64 = 1, occ_emit = 1, occ_emit_big = 1, occ_raster = 1, occ_tile_sort = 1;
    double pairs_per_splat = 0.0;  // previous frame's P / M (picks the emit stage)
    uint64_t last_m = 0;           // previous frame's splats with tiles
    double prev_pairs_per_tile = 0.0;  // previous frame's P / T (picks the sort path, agsx_frame.cu)
    Buf sort_counts;  // grid x 256 chunk digit counts + 256 totals (one pass at a time)

    // device arenas (grow-only)
    Buf status, p0, p1, p2, p3, p4, dkeys, dvals, dkeys2, dvals2, dcounts, chunks, img_u8;
    Buf tkeys, pvals, tkeys2, pvals2;
    Buf ranges, image, lb, ctr, hist, maxt, dump, lut_ext, tile_pit, calib;
    Buf tmp0, tmp1, tmp2, tmp3, tmp4;
    Buf bk_hits, bk_gd, ekeys, ekeys2, big_list;  // tile-bucketed sort path
    Buf chain;  // ChainWords of the frames enqueued since the last wait (never zeroed per frame)
    uint64_t pair_capacity = 0;

    Counters* h_ctr = nullptr;  // pinned; ChainWords follow it
    uint32_t* h_ctr_dev = nullptr;  // its device-mapped alias
    static constexpr int kRing = 64;  // frames of stage events kept for timing
    cudaEvent_t ev_ring[kRing][6] = {};
    cudaEvent_t* ev = ev_ring[0];
    uint64_t frames = 0;

    // most recent fused frame
    bool have_frame = false;
    bool pending = false;  // a frame is enqueued and not yet waited for
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
    static constexpr int kFlagBands = 32;  // egress row slots of the one-launch path (Counters::band_done)
    cudaEvent_t band_ev[kBands] = {};
    cudaEvent_t copy_done = nullptr;
    cudaEvent_t ev_zeroed = nullptr;  // the frame's counters are zeroed (band flags valid from here)
    uint32_t* f_tkeys = nullptr;
    uint32_t* f_pvals = nullptr;
    int f_tile_count = 0;
    bool f_bucket = false;     // the frame used the tile-bucketed sort (k_bucket.cu)
    bool f_pit_tiles = false;  // P_it lives in the per-tile words (units rasterizer), not Counters::p_it
};

namespace agsx::host {


inline void ensure(Buf& b, size_t bytes, bool zero = false) {
    if (b.bytes >= bytes) return;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    const size_t alloc = std::max<size_t>(bytes, 256);
    AGSX_CUDA(cudaMalloc(&b.p, alloc));
    if (zero) AGSX_CUDA(cudaMemset(b.p, 0, alloc));
    b.bytes = alloc;
}

inline void release(Buf& b) {
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
}

template <typename T>
T* ptr(const Buf& b) {
    return static_cast<T*>(b.p);
}

inline void check_launch(agsx_ctx* ctx) {
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

inline int fail(agsx_ctx* ctx, int code, const std::string& msg) {
    ctx->err = msg;
    return code;
}

// ---- frame pipeline (agsx_frame.cu) -------------------------------------
std::string validate_config(const agsx_config& c);
std::string validate_camera(const agsx_camera& cam);
int tile_bits(uint32_t tile_count);
FrameParams make_params(const agsx_camera& cam, const agsx_config& cfg, const agsx_lut* lut,
                        const float* lut_ext_dev);
int raster_ppt(int tile_size);
bool raster_uses_units(const FrameParams& p, bool maxt);
void launch_raster(agsx_ctx* ctx, const FrameParams& p, const uint2* ranges, const uint32_t* vals,
                   const float4* P0, const float4* P1, const float4* P2, float* image,
                   uint32_t* maxt, Counters* ctr, uint32_t* unit_ctr = nullptr);
size_t sort_smem(bool k64);
size_t counters_bytes();
uint64_t chunk_slots(uint64_t n);
int sort_grid(agsx_ctx* ctx, bool k64);
void ensure_lb(agsx_ctx* ctx, uint64_t max_elems);
void ensure_frame_buffers(agsx_ctx* ctx, uint64_t n, uint64_t tiles, uint64_t pixels, bool obb,
                          uint64_t pair_budget);
SplatPlanes planes_of(agsx_ctx* ctx);
int prepare(agsx_ctx* ctx, const agsx_camera* cam, const agsx_config* cfg, const agsx_lut* lut, FrameParams& p);
bool depth_keys_wide_host(const Counters& c);
void launch_quantize(agsx_ctx* ctx, const float* src, uint8_t* dst, uint64_t n, cudaStream_t st);
void enqueue_frame(agsx_ctx* ctx, const agsx_scene* sc, const FrameParams& p, bool maxt, agsx_splat_view* dump);
int start_frame(agsx_ctx* ctx, const agsx_scene* sc, const agsx_camera* cam, const agsx_config* cfg,
                const agsx_lut* lut, bool maxt, float* host_image = nullptr, float* device_target = nullptr,
                uint8_t* host_u8 = nullptr);
int finish_frame(agsx_ctx* ctx, agsx_frame* out);
int refuse_if_host_frame(agsx_ctx* ctx, const char* what);
void slots_to_ids_host(const agsx_scene* sc, const void* dev, uint32_t* host_out, cudaStream_t st);
std::vector<uint32_t> scene_map_host(const Buf& b, uint64_t n);
int quantize_to_host(agsx_ctx* ctx, uint8_t* image_u8);
cudaError_t shared_copy_stream(int device, cudaStream_t* out);

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

}  // namespace agsx::host

/*
 * agsx.h -- C-ABI of the B200-native AdaGScale renderer (libagsx.so).
 *
 * This is the drop-in boundary below the reference's `ags::render()`.  Every
 * entry point takes plain pointers and sizes, returns an int status and never
 * throws.  Each function names the reference interface it replaces
 * (/root/reference/proj/... file:line).
 *
 * Status codes (mapped by the C++ layer to the reference's exceptions):
 *   AGSX_OK            0
 *   AGSX_EINVAL        1  -> std::invalid_argument   (rasterizer.cpp:105-108,
 *                                                     preprocess.cpp:123-125)
 *   AGSX_EPAIR_BUDGET  2  -> ags::PairBudgetError    (pair_gen.hpp:74-76,
 *                                                     pair_gen.cpp:181-184)
 *   AGSX_ECUDA         3  -> std::runtime_error
 *   AGSX_ENOMEM        4  -> std::runtime_error (std::bad_alloc)
 *   AGSX_ECAPACITY     5  caller buffer too small; required size returned
 *   AGSX_EFRAME_LOST   6  -> std::runtime_error: an earlier frame of an async
 *                         chain (frames enqueued since the last wait)
 *                         overflowed the pair arena and was not rasterised
 *
 * Threading: one agsx_ctx per host thread per GPU; a ctx owns one CUDA
 * stream and grow-only device arenas.  Scenes are immutable once uploaded
 * and may be shared by contexts on the same device.
 */
#ifndef AGSX_H
#define AGSX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AGSX_ABI_VERSION 1

enum {
    AGSX_OK = 0,
    AGSX_EINVAL = 1,
    AGSX_EPAIR_BUDGET = 2,
    AGSX_ECUDA = 3,
    AGSX_ENOMEM = 4,
    AGSX_ECAPACITY = 5,
    AGSX_EFRAME_LOST = 6
};

/* ags::Mode (scene.hpp:60); values equal the reference enum order. */
enum { AGSX_MODE_AABB = 0, AGSX_MODE_OBB = 1, AGSX_MODE_ELLIPSE = 2, AGSX_MODE_ADAGSCALE = 3 };

/* agsx_config.flags */
enum {
    /* Evaluate every blend alpha with the glibc-exact expf (bit-identical
     * image to the CPU reference).  Without it the rasterizer uses the
     * hardware ex2 path and re-evaluates exactly only when alpha is within a
     * guard band of tau or of the clamp, so every blend decision is still
     * exact and colours differ by O(1e-7). */
    AGSX_FLAG_EXACT_ALPHA = 1
};

/* ags::Camera (scene.hpp:34-39). rotation: world-to-camera, row-major. */
typedef struct {
    float position[3];
    float rotation[9];
    float fx, fy;
    int32_t width, height;
} agsx_camera;

/* ags::RenderConfig (scene.hpp:65-78) plus B200-path flags. */
typedef struct {
    int32_t tile_size;
    float alpha_threshold;
    float transmittance_floor;
    float alpha_clamp;
    float near_plane;
    float guard_band;
    int32_t mode;
    float k;
    int32_t thread_count; /* accepted, no device meaning (parallel.hpp:10-14) */
    float background[3];
    int32_t fixed_radius_aabb;
    uint64_t pair_budget;
    uint32_t flags; /* AGSX_FLAG_* */
} agsx_config;

/* ags::TUpperLUT (lut.hpp:11-26).  bin_count == 0 -> the all-ones default. */
typedef struct {
    float depth_min, depth_max;
    int32_t bin_count;
    const float* bins;
} agsx_lut;

/* Host SoA scene description for upload.  Replaces the
 * std::span<const ags::Gaussian3D> argument of render() (rasterizer.hpp:63);
 * Gaussian3D (scene.hpp:15-21) is AoS with a heap SH vector.
 * sh is coefficient-major per Gaussian: sh[i*3*D + k*3 + c], D in {1,4,9,16}. */
typedef struct {
    uint64_t count;
    int32_t sh_coeffs;
    const float* mean;     /* 3*count */
    const float* scale;    /* 3*count */
    const float* rotation; /* 4*count, w x y z */
    const float* opacity;  /* count */
    const float* sh;       /* 3*sh_coeffs*count */
} agsx_scene_desc;

/* ags::SplatView (preprocess.hpp:15-24), byte-identical layout (60 B). */
typedef struct {
    float mean2d[2];
    float cov2d[3];
    float inv_cov[3];
    float depth;
    float rgb[3];
    float opacity;
    float th;
    uint32_t source_id;
} agsx_splat_view;

/* Output of one frame (ags::RenderReport, rasterizer.hpp:31-40). */
typedef struct {
    float* image;          /* optional host H*W*3 f32 (HWC); NULL = keep on device */
    float* max_t;          /* optional host, scene count entries, indexed by
                              Gaussian id (RecordOptions::max_t; 0 = never blended) */
    uint64_t pair_count;   /* out */
    uint64_t splat_count;  /* out */
    float stage_ms[4];     /* out: preprocess, pair_gen, sort, raster (device time) */
} agsx_frame;

typedef struct agsx_ctx agsx_ctx;
typedef struct agsx_scene agsx_scene;

/* ---- context --------------------------------------------------------- */
int agsx_create(int device, agsx_ctx** out);
void agsx_destroy(agsx_ctx* ctx);
/* Last error message of this ctx (never NULL). */
const char* agsx_last_error(const agsx_ctx* ctx);
int agsx_abi_version(void);
/* The ctx's CUDA stream (cudaStream_t) for event timing / interop. */
void* agsx_stream(agsx_ctx* ctx);

/* ---- scene (replaces passing the host span on every render) ---------- */
int agsx_scene_upload(agsx_ctx* ctx, const agsx_scene_desc* desc, agsx_scene** out);
void agsx_scene_free(agsx_scene* scene);
uint64_t agsx_scene_count(const agsx_scene* scene);

/* ---- the hot path: ags::render() (rasterizer.cpp:102-165) ------------ */
/* Synchronous: validates like render() (scene.cpp:41-59,113-123), runs the
 * four device stages, copies requested outputs to the host. */
int agsx_render(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam,
                const agsx_config* cfg, const agsx_lut* lut, agsx_frame* out);

/* ags::render + write_image fused on the device (next row f3): the frame is
 * quantised to the PPM byte image clamp(v, 0, 1) -> lround(v * 255)
 * (gsio.cpp:265-281) before it leaves the GPU, so 3 B/pixel cross PCIe
 * instead of 12.  image_u8: host H*W*3 bytes (written directly when
 * page-locked); out->image is ignored. */
int agsx_render_u8(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam,
                   const agsx_config* cfg, const agsx_lut* lut, uint8_t* image_u8, agsx_frame* out);

/* Asynchronous form for benchmarking / batching: enqueues one frame on the
 * ctx stream and returns.  Results stay on the device; agsx_render_wait()
 * synchronises, checks the budget/overflow status and fills counts and
 * stage times of the most recent frame.  No host synchronisation occurs
 * between the enqueued stages. */
int agsx_render_async(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam,
                      const agsx_config* cfg, const agsx_lut* lut);
int agsx_render_wait(agsx_ctx* ctx, agsx_frame* out);
/* As agsx_render_async, with the image rasterised into `target` (H*W*3 f32,
 * HWC): device memory of the ctx's device (e.g. a frame slot that a
 * collective then gathers) or a page-locked, device-mapped host buffer.
 * `target` must stay valid until agsx_render_wait returns. */
int agsx_render_async_to(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam,
                         const agsx_config* cfg, const agsx_lut* lut, float* target);
/* As agsx_render_async, with the image delivered to host memory `image`
 * (H*W*3 f32, HWC) by the time agsx_render_wait returns: the egress of
 * agsx_render (page-locked memory is filled by banded copies behind the
 * raster; pageable memory gets one copy in agsx_render_wait).  Frames of two
 * contexts on one device overlap one frame's PCIe egress with the next
 * frame's kernels (paper_2604_18980_b200.batch.render_views).  Replaces a
 * loop of ags::render() calls over a camera path (adagscale_main.cpp:224-226).
 * `image` must stay valid until agsx_render_wait returns. */
int agsx_render_async_host(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam,
                           const agsx_config* cfg, const agsx_lut* lut, float* image);
/* As agsx_render_async_host for the write_image bytes (agsx_render_u8): the
 * frame is quantised band by band on the device and only the H*W*3 bytes
 * cross PCIe, behind the raster when `image_u8` is page-locked. */
int agsx_render_async_host_u8(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam,
                              const agsx_config* cfg, const agsx_lut* lut, uint8_t* image_u8);

/* One alpha-blend event, BlendRecord (rasterizer.hpp:19-24). */
typedef struct agsx_blend_record {
    uint32_t pixel; /* y * width + x */
    uint32_t splat; /* index into the view's splat sequence (survivors in Gaussian order) */
    float alpha;
    float weight; /* alpha * T */
} agsx_blend_record;

/* agsx_render with RecordOptions::contributions (rasterizer.cpp:21-100,
 * 135-161): the frame is rendered with the glibc-exact alpha and its
 * blend-event stream written to `records` in the reference's order (tile
 * index, then pair order, then row-major pixel).  *count receives the stream
 * length; AGSX_ECAPACITY when `capacity` is smaller (the frame and `out` are
 * complete either way, so a caller sizes the buffer and calls again).  `out`
 * as for agsx_render (image and max_t optional). */
int agsx_render_contributions(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam,
                              const agsx_config* cfg, const agsx_lut* lut, agsx_blend_record* records,
                              uint64_t capacity, uint64_t* count, agsx_frame* out);

/* Device-timed stage durations (ms: preprocess, pair_gen, sort, raster) of
 * the last min(max_frames, 64) frames enqueued on this ctx, oldest first;
 * synchronises the stream. */
int agsx_stage_history(agsx_ctx* ctx, float* stage_ms, int32_t max_frames, int32_t* out_frames);

/* Counters of the most recent frame, the first n of: {splat_count
 * (survivors), splats with >= 1 tile, pair_count, P_it (pairs iterated before
 * tile saturation, the rasterizer's work unit), overflow flag, tile count,
 * 8 rasterizer work counters (AGSX_RASTER_STATS=1), depth-sort passes (3 or
 * 4; 0 on the tile-bucketed path), 1 if the tile-bucketed sort ran};
 * synchronises. */
int agsx_frame_stats(agsx_ctx* ctx, uint64_t* stats, int32_t n);

/* Device pointer to the ctx-owned image of the most recent frame
 * (H*W*3 f32, HWC) and its dimensions. */
int agsx_device_image(agsx_ctx* ctx, float** dptr, int32_t* width, int32_t* height);

/* ---- parity hooks over the most recent fused frame ------------------- */
/* Per-Gaussian tile counts (0 for culled Gaussians) and survivor flags
 * (pair_gen.cpp:167-175 tile_counts, indexed by Gaussian id rather than by
 * compacted splat index). */
int agsx_dump_tile_counts(agsx_ctx* ctx, uint32_t* counts, uint8_t* alive, uint64_t n);
/* Sorted pair list: key = (tile << 32) | bits(depth) (pair_gen.hpp:33-36),
 * value = Gaussian id (maps to the reference splat_index via source_id). */
int agsx_dump_sorted_pairs(agsx_ctx* ctx, uint64_t* keys, uint32_t* gids, uint64_t capacity,
                           uint64_t* out_count);
/* Per-tile [start, end) ranges, 2*tile_count u32 (pair_sort.cpp:30-42). */
int agsx_dump_ranges(agsx_ctx* ctx, uint32_t* ranges, uint64_t tile_count);

/* ---- stage-level entry points (the reference's per-stage API) -------- */
/* preprocess_view (preprocess.hpp:51-54): out holds scene count entries. */
int agsx_preprocess_view(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam,
                         const agsx_config* cfg, const agsx_lut* lut, agsx_splat_view* out,
                         uint64_t* out_count);
/* generate_pairs (pair_gen.hpp:70-72) over a host splat list.  keys /
 * splat_index hold `capacity` entries; AGSX_ECAPACITY with *out_total set if
 * too small.  tile_counts: n entries. */
int agsx_generate_pairs(agsx_ctx* ctx, const agsx_splat_view* splats, uint64_t n,
                        int32_t width, int32_t height, int32_t mode, const agsx_config* cfg,
                        uint64_t* keys, uint32_t* splat_index, uint64_t capacity,
                        uint32_t* tile_counts, uint64_t* out_total);
/* sort_pairs (pair_sort.hpp:19): stable ascending by the full 64-bit key,
 * in place; ranges: 2*tile_count u32. */
int agsx_sort_pairs(agsx_ctx* ctx, uint64_t* keys, uint32_t* splat_index, uint64_t n,
                    int32_t tile_count, uint32_t* ranges);
/* raster_tile over every tile (rasterizer.hpp:54-58, rasterizer.cpp:137-147).
 * image: H*W*3 host; max_t optional (n_splats entries). */
int agsx_raster(agsx_ctx* ctx, const agsx_splat_view* splats, uint64_t n_splats,
                const uint32_t* splat_index, uint64_t n_pairs, const uint32_t* ranges,
                int32_t width, int32_t height, const agsx_config* cfg, float* image,
                float* max_t);

/* ---- per-element helpers of the stages (the device functions the kernels
 * use, one element per thread; the C++ wrappers in ags.hpp take the
 * reference's single-element signatures) ------------------------------- */
/* project (preprocess.cpp:26-66, preprocess.hpp:35-37) of every Gaussian of
 * an uploaded scene: valid[i] = 1 when in front of the near plane and inside
 * the guard band; out[6i..6i+5] = {mean2d.x, mean2d.y, cov2d.xx, cov2d.xy,
 * cov2d.yy, depth} (cov2d carries the +0.3 dilation). */
int agsx_project(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam, const agsx_config* cfg,
                 uint8_t* valid, float* out);
/* eval_color (preprocess.cpp:68-105, preprocess.hpp:38-40): rgb[3i..] of
 * Gaussian i of the scene for the unit view direction dirs[3i..]. */
int agsx_eval_color(agsx_ctx* ctx, const agsx_scene* scene, const float* dirs, float* rgb);
/* compute_th (preprocess.cpp:107-116, preprocess.hpp:44-45) of n (cov2d
 * {xx, xy, yy}, depth) with the LUT (NULL = all ones), k and tau;
 * AGSX_EINVAL when some det(cov2d) <= 0 (std::invalid_argument). */
int agsx_compute_th(agsx_ctx* ctx, const float* cov2d, const float* depth, uint64_t n, const agsx_lut* lut,
                    float k, float tau, float* th);
/* alpha_at (rasterizer.hpp:44-50, glibc expf) of splats[i] at the pixel
 * centre px[2i..2i+1]. */
int agsx_alpha_at(agsx_ctx* ctx, const agsx_splat_view* splats, const float* px, uint64_t n,
                  float alpha_clamp, float* alpha);
/* effective_radius (pair_gen.cpp:11-16, pair_gen.hpp:49-55, glibc logf):
 * out[2i] = mahalanobis, out[2i+1] = pixels. */
int agsx_effective_radius(agsx_ctx* ctx, const float* opacity, const float* th, const float* cov2d, uint64_t n,
                          float* out);

/* ---- calibration primitives (calibrate.cpp:14-155, analysis.cpp:14-29) - */
/* Device memory owned by the caller (e.g. the calibration reference frames). */
int agsx_device_alloc(agsx_ctx* ctx, size_t bytes, void** out);
void agsx_device_free(agsx_ctx* ctx, void* p);
/* One view of build_lut (calibrate.cpp:26-37): renders `cam` in the lossless
 * Ellipse mode (cfg's mode is ignored) with glibc-exact alpha and
 * max-transmittance recording, then folds every blended splat's max_t into
 * the depth bin of lut_shape (bin_index, lut.hpp:16-23):
 * folded[b] = max(folded[b], max_t), observed[b] = 1.  folded / observed:
 * lut_shape->bin_count host entries, updated in place; lut_shape->bins is
 * not read. */
int agsx_fold_max_t(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam,
                    const agsx_config* cfg, const agsx_lut* lut_shape, float* folded, uint8_t* observed);
/* Sum over n floats of ((double)a[i] - b[i])^2 (the numerator of psnr,
 * analysis.cpp:14-25) for two device arrays; a deterministic tree order. */
int agsx_sq_err(agsx_ctx* ctx, const float* a, const float* b, uint64_t n, double* out);

/* ---- device libm pinning (glibc-exact logf / expf used on the path) -- */
int agsx_device_logf(agsx_ctx* ctx, const float* x, float* y, uint64_t n);
int agsx_device_expf(agsx_ctx* ctx, const float* x, float* y, uint64_t n);

/* Page-locked host buffers for frame egress (full-bandwidth D2H of images). */
int agsx_host_alloc(size_t bytes, void** out);
void agsx_host_free(void* p);

/* Number of kernels this ctx has launched since creation. */
uint64_t agsx_kernel_launches(const agsx_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* AGSX_H */

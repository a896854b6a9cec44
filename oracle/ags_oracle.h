/*
 * ags_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C interface shared by the two CPU oracles of the AdaGScale render
 * path:
 *   - oracle/ags_oracle.c      : a from-scratch C restatement of the
 *                                reference algorithm (liboracle "port");
 *   - oracle/ref_shim.cpp      : a thin extern "C" shim over the reference's
 *                                own C++ sources compiled unmodified from
 *                                /root/reference/proj/src (oracle/_ref).
 *
 * Both libraries export exactly these symbols so the test-suite can
 * parametrize over them.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load either library; the product
 * path (paper_2604_18980_b200/) never links or calls anything here.
 *
 * Struct layouts mirror the reference types byte for byte:
 *   ago_splat  == ags::SplatView          (preprocess.hpp:15-24, 60 B)
 *   ago_camera ~  ags::Camera             (scene.hpp:34-39)
 *   ago_config ~  ags::RenderConfig       (scene.hpp:65-78)
 */
#ifndef AGS_ORACLE_H
#define AGS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { AGO_AABB = 0, AGO_OBB = 1, AGO_ELLIPSE = 2, AGO_ADAGSCALE = 3 };

enum {
    AGO_OK = 0,
    AGO_EINVAL = 1,
    AGO_EPAIR_BUDGET = 2,
    AGO_ECAPACITY = 5 /* output buffer too small; required size returned */
};

typedef struct {
    float position[3];
    float rotation[9]; /* world-to-camera, row-major */
    float fx, fy;
    int32_t width, height;
} ago_camera;

typedef struct {
    int32_t tile_size;
    float alpha_threshold;
    float transmittance_floor;
    float alpha_clamp;
    float near_plane;
    float guard_band;
    int32_t mode;
    float k;
    int32_t thread_count;
    float background[3];
    int32_t fixed_radius_aabb;
    uint64_t pair_budget;
} ago_config;

typedef struct {
    float depth_min, depth_max;
    int32_t bin_count;
    const float* bins;
} ago_lut;

/* SoA scene; sh is coefficient-major per Gaussian: sh[i*3*D + k*3 + c]. */
typedef struct {
    uint64_t count;
    int32_t sh_coeffs; /* D in {1,4,9,16} */
    const float* mean;
    const float* scale;
    const float* rotation; /* w, x, y, z */
    const float* opacity;
    const float* sh;
} ago_scene;

typedef struct {
    float mean2d[2];
    float cov2d[3];   /* xx, xy, yy */
    float inv_cov[3]; /* xx, xy, yy */
    float depth;
    float rgb[3];
    float opacity;
    float th;
    uint32_t source_id;
} ago_splat;

/* Fills ago_config with the RenderConfig defaults (scene.hpp:65-78). */
void ago_default_config(ago_config* cfg);

/* synth_scene (synth.cpp:242-252).  All outputs caller-owned:
 * mean/scale: 3*count, rotation: 4*count, opacity: count, sh: 3*count
 * (synthetic scenes are SH degree 0), cameras: camera_count entries. */
int ago_synth_scene(uint64_t seed, int32_t count, const char* layout,
                    int32_t camera_count, int32_t width, int32_t height,
                    float fx, float fy, float* mean, float* scale,
                    float* rotation, float* opacity, float* sh,
                    ago_camera* cameras);

/* preprocess_view (preprocess.cpp:118-163).  out must hold scene->count
 * entries; *out_count receives the survivor count. */
int ago_preprocess(const ago_scene* scene, const ago_camera* cam,
                   const ago_config* cfg, const ago_lut* lut, ago_splat* out,
                   uint64_t* out_count);

/* generate_pairs (pair_gen.cpp:161-203).  tile_counts: n entries.  keys /
 * splat_index: capacity entries; returns AGO_ECAPACITY (with *out_total set)
 * when capacity is too small, AGO_EPAIR_BUDGET when the budget is exceeded. */
int ago_generate_pairs(const ago_splat* splats, uint64_t n, int32_t width,
                       int32_t height, int32_t mode, const ago_config* cfg,
                       uint64_t* keys, uint32_t* splat_index,
                       uint64_t capacity, uint32_t* tile_counts,
                       uint64_t* out_total);

/* sort_pairs (pair_sort.cpp:7-44), in place; ranges: 2*tile_count u32. */
int ago_sort_pairs(uint64_t* keys, uint32_t* splat_index, uint64_t n,
                   int32_t tile_count, uint32_t* ranges);

/* raster of every tile (rasterizer.cpp:21-100 + 137-147).  image: H*W*3.
 * max_t: optional (n_splats entries, zero-initialised by the callee). */
int ago_raster(const ago_splat* splats, uint64_t n_splats,
               const uint64_t* keys, const uint32_t* splat_index,
               uint64_t n_pairs, const uint32_t* ranges, int32_t width,
               int32_t height, const ago_config* cfg, float* image,
               float* max_t);
/* the same raster, and P_it: the pairs every tile's loop visits before all
 * of its pixels are saturated (rasterizer.cpp:55-56), summed over tiles. */
int ago_raster_pit(const ago_splat* splats, uint64_t n_splats, const uint32_t* splat_index,
                   const uint32_t* ranges, int32_t width, int32_t height, const ago_config* cfg,
                   float* image, uint64_t* p_it);

/* render (rasterizer.cpp:102-165).  image: H*W*3; max_t optional (scene
 * count entries; indexed by *compacted* splat index).  stage_s: 4 doubles
 * {preprocess, pair_gen, sort, raster}, optional. */
int ago_render(const ago_scene* scene, const ago_camera* cam,
               const ago_config* cfg, const ago_lut* lut, float* image,
               uint64_t* pair_count, uint64_t* splat_count, float* max_t,
               double* stage_s);

/* BlendRecord (rasterizer.hpp:19-24): one alpha-blend event. */
typedef struct {
    uint32_t pixel; /* y * width + x */
    uint32_t splat; /* index into the view's (compacted) splat sequence */
    float alpha;
    float weight; /* alpha * T */
} ago_blend;

/* render with RecordOptions::contributions (rasterizer.cpp:21-100,
 * 135-161): the blend-event stream in tile-index order, within a tile pair
 * order then row-major pixel order.  out: capacity records; *count receives
 * the stream length; AGO_ECAPACITY when capacity is too small (the image is
 * rendered either way). */
int ago_render_contributions(const ago_scene* scene, const ago_camera* cam, const ago_config* cfg,
                             const ago_lut* lut, float* image, ago_blend* out, uint64_t capacity,
                             uint64_t* count);

/* psnr (analysis.cpp:14-25). */
double ago_psnr(const float* a, const float* b, uint64_t n);

/* glibc libm as linked into the oracle (for device-libm pinning tests). */
void ago_logf_batch(const float* x, float* y, uint64_t n);
void ago_expf_batch(const float* x, float* y, uint64_t n);

/* Name of the implementation: "port" (C restatement) or "reference". */
const char* ago_kind(void);

#ifdef __cplusplus
}
#endif

#endif /* AGS_ORACLE_H */

// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" adapter that exposes the *unmodified* reference implementation
// (compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libags_ref.so) through the plain-C oracle interface of
// ags_oracle.h.  It converts between the oracle's SoA/POD structs and the
// reference's C++ types and calls the reference functions directly:
//   synth_scene      synth.cpp:242-252
//   preprocess_view  preprocess.cpp:118-163
//   generate_pairs   pair_gen.cpp:161-203
//   sort_pairs       pair_sort.cpp:7-44
//   raster_tile      rasterizer.cpp:21-100
//   render           rasterizer.cpp:102-165
//   psnr             analysis.cpp:14-25
// No reference source is copied into this repository.
#include <cmath>
#include <cstring>
#include <exception>
#include <span>
#include <stdexcept>
#include <vector>

#include "adagscale/analysis.hpp"
#include "adagscale/calibrate.hpp"
#include "adagscale/gsio.hpp"
#include "adagscale/synth.hpp"
#include "adagscale/pair_gen.hpp"
#include "adagscale/pair_sort.hpp"
#include "adagscale/preprocess.hpp"
#include "adagscale/calibrate.hpp"
#include "adagscale/rasterizer.hpp"
#include "adagscale/synth.hpp"
#include "ags_oracle.h"

namespace {

ags::Camera to_cam(const ago_camera* c) {
    ags::Camera cam;
    cam.position = {c->position[0], c->position[1], c->position[2]};
    for (int i = 0; i < 9; ++i) cam.rotation.m[i] = c->rotation[i];
    cam.fx = c->fx;
    cam.fy = c->fy;
    cam.width = c->width;
    cam.height = c->height;
    return cam;
}

void from_cam(const ags::Camera& cam, ago_camera* c) {
    c->position[0] = cam.position.x;
    c->position[1] = cam.position.y;
    c->position[2] = cam.position.z;
    for (int i = 0; i < 9; ++i) c->rotation[i] = cam.rotation.m[i];
    c->fx = cam.fx;
    c->fy = cam.fy;
    c->width = cam.width;
    c->height = cam.height;
}

ags::RenderConfig to_cfg(const ago_config* c) {
    ags::RenderConfig cfg;
    cfg.tile_size = c->tile_size;
    cfg.alpha_threshold = c->alpha_threshold;
    cfg.transmittance_floor = c->transmittance_floor;
    cfg.alpha_clamp = c->alpha_clamp;
    cfg.near_plane = c->near_plane;
    cfg.guard_band = c->guard_band;
    cfg.mode = static_cast<ags::Mode>(c->mode);
    cfg.k = c->k;
    cfg.thread_count = c->thread_count;
    cfg.background = {c->background[0], c->background[1], c->background[2]};
    cfg.fixed_radius_aabb = c->fixed_radius_aabb != 0;
    cfg.pair_budget = static_cast<std::size_t>(c->pair_budget);
    return cfg;
}

ags::TUpperLUT to_lut(const ago_lut* l) {
    ags::TUpperLUT lut;
    if (l && l->bin_count > 0) {
        lut.depth_min = l->depth_min;
        lut.depth_max = l->depth_max;
        lut.bins.assign(l->bins, l->bins + l->bin_count);
    }
    return lut;
}

std::vector<ags::Gaussian3D> to_scene(const ago_scene* s) {
    std::vector<ags::Gaussian3D> out(s->count);
    const int d = s->sh_coeffs;
    for (uint64_t i = 0; i < s->count; ++i) {
        ags::Gaussian3D& g = out[i];
        g.mean = {s->mean[3 * i], s->mean[3 * i + 1], s->mean[3 * i + 2]};
        g.scale = {s->scale[3 * i], s->scale[3 * i + 1], s->scale[3 * i + 2]};
        g.rotation = {s->rotation[4 * i], s->rotation[4 * i + 1],
                      s->rotation[4 * i + 2], s->rotation[4 * i + 3]};
        g.opacity = s->opacity[i];
        g.sh.assign(s->sh + 3 * d * i, s->sh + 3 * d * (i + 1));
    }
    return out;
}

ags::SplatView to_splat(const ago_splat& a) {
    ags::SplatView s;
    s.mean2d = {a.mean2d[0], a.mean2d[1]};
    s.cov2d = {a.cov2d[0], a.cov2d[1], a.cov2d[2]};
    s.inv_cov = {a.inv_cov[0], a.inv_cov[1], a.inv_cov[2]};
    s.depth = a.depth;
    s.rgb = {a.rgb[0], a.rgb[1], a.rgb[2]};
    s.opacity = a.opacity;
    s.th = a.th;
    s.source_id = a.source_id;
    return s;
}

ago_splat from_splat(const ags::SplatView& s) {
    ago_splat a;
    a.mean2d[0] = s.mean2d.x;
    a.mean2d[1] = s.mean2d.y;
    a.cov2d[0] = s.cov2d.xx;
    a.cov2d[1] = s.cov2d.xy;
    a.cov2d[2] = s.cov2d.yy;
    a.inv_cov[0] = s.inv_cov.xx;
    a.inv_cov[1] = s.inv_cov.xy;
    a.inv_cov[2] = s.inv_cov.yy;
    a.depth = s.depth;
    a.rgb[0] = s.rgb.x;
    a.rgb[1] = s.rgb.y;
    a.rgb[2] = s.rgb.z;
    a.opacity = s.opacity;
    a.th = s.th;
    a.source_id = s.source_id;
    return a;
}

std::vector<ags::SplatView> to_splats(const ago_splat* s, uint64_t n) {
    std::vector<ags::SplatView> out;
    out.reserve(n);
    for (uint64_t i = 0; i < n; ++i) out.push_back(to_splat(s[i]));
    return out;
}

template <typename F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const ags::PairBudgetError&) {
        return AGO_EPAIR_BUDGET;
    } catch (const std::invalid_argument&) {
        return AGO_EINVAL;
    } catch (...) {
        return AGO_EINVAL;
    }
}

}  // namespace

static_assert(sizeof(ago_splat) == sizeof(ags::SplatView),
              "ago_splat must mirror ags::SplatView");

extern "C" {

const char* ago_kind(void) { return "reference"; }

void ago_default_config(ago_config* c) {
    const ags::RenderConfig d;
    c->tile_size = d.tile_size;
    c->alpha_threshold = d.alpha_threshold;
    c->transmittance_floor = d.transmittance_floor;
    c->alpha_clamp = d.alpha_clamp;
    c->near_plane = d.near_plane;
    c->guard_band = d.guard_band;
    c->mode = static_cast<int32_t>(d.mode);
    c->k = d.k;
    c->thread_count = d.thread_count;
    c->background[0] = d.background.x;
    c->background[1] = d.background.y;
    c->background[2] = d.background.z;
    c->fixed_radius_aabb = d.fixed_radius_aabb ? 1 : 0;
    c->pair_budget = d.pair_budget;
}

int ago_synth_scene(uint64_t seed, int32_t count, const char* layout,
                    int32_t camera_count, int32_t width, int32_t height,
                    float fx, float fy, float* mean, float* scale,
                    float* rotation, float* opacity, float* sh,
                    ago_camera* cameras) {
    return guarded([&] {
        ags::SynthSpec spec;
        spec.layout = layout;
        spec.camera_count = camera_count;
        spec.width = width;
        spec.height = height;
        spec.fx = fx;
        spec.fy = fy;
        const ags::SynthScene s = ags::synth_scene(seed, count, spec);
        for (std::size_t i = 0; i < s.gaussians.size(); ++i) {
            const ags::Gaussian3D& g = s.gaussians[i];
            mean[3 * i] = g.mean.x;
            mean[3 * i + 1] = g.mean.y;
            mean[3 * i + 2] = g.mean.z;
            scale[3 * i] = g.scale.x;
            scale[3 * i + 1] = g.scale.y;
            scale[3 * i + 2] = g.scale.z;
            rotation[4 * i] = g.rotation.w;
            rotation[4 * i + 1] = g.rotation.x;
            rotation[4 * i + 2] = g.rotation.y;
            rotation[4 * i + 3] = g.rotation.z;
            opacity[i] = g.opacity;
            for (int c = 0; c < 3; ++c) sh[3 * i + c] = g.sh[c];
        }
        for (std::size_t i = 0; i < s.cameras.size(); ++i)
            from_cam(s.cameras[i], &cameras[i]);
        return AGO_OK;
    });
}

int ago_preprocess(const ago_scene* scene, const ago_camera* cam,
                   const ago_config* cfg, const ago_lut* lut, ago_splat* out,
                   uint64_t* out_count) {
    return guarded([&] {
        const auto g = to_scene(scene);
        const ags::TUpperLUT l = to_lut(lut);
        const ags::RenderConfig c = to_cfg(cfg);
        const auto splats = ags::preprocess_view(
            g, to_cam(cam), c, c.mode == ags::Mode::AdaGScale ? &l : nullptr);
        for (std::size_t i = 0; i < splats.size(); ++i)
            out[i] = from_splat(splats[i]);
        *out_count = splats.size();
        return AGO_OK;
    });
}

int ago_generate_pairs(const ago_splat* splats, uint64_t n, int32_t width,
                       int32_t height, int32_t mode, const ago_config* cfg,
                       uint64_t* keys, uint32_t* splat_index,
                       uint64_t capacity, uint32_t* tile_counts,
                       uint64_t* out_total) {
    return guarded([&] {
        const ags::RenderConfig c = to_cfg(cfg);
        const ags::TileGrid grid =
            ags::TileGrid::make(width, height, c.tile_size);
        const auto sv = to_splats(splats, n);
        const ags::PairGenResult r = ags::generate_pairs(
            sv, grid, static_cast<ags::Mode>(mode), c);
        *out_total = r.pairs.size();
        for (uint64_t i = 0; i < n; ++i) tile_counts[i] = r.tile_counts[i];
        if (r.pairs.size() > capacity) return (int)AGO_ECAPACITY;
        for (std::size_t i = 0; i < r.pairs.size(); ++i) {
            keys[i] = r.pairs[i].key;
            splat_index[i] = r.pairs[i].splat_index;
        }
        return (int)AGO_OK;
    });
}

int ago_sort_pairs(uint64_t* keys, uint32_t* splat_index, uint64_t n,
                   int32_t tile_count, uint32_t* ranges) {
    return guarded([&] {
        std::vector<ags::GaussianTilePair> pairs(n);
        for (uint64_t i = 0; i < n; ++i) pairs[i] = {keys[i], splat_index[i]};
        const ags::SortedPairs s = ags::sort_pairs(std::move(pairs), tile_count);
        for (uint64_t i = 0; i < n; ++i) {
            keys[i] = s.pairs[i].key;
            splat_index[i] = s.pairs[i].splat_index;
        }
        for (int32_t t = 0; t < tile_count; ++t) {
            ranges[2 * t] = s.ranges[t].first;
            ranges[2 * t + 1] = s.ranges[t].second;
        }
        return AGO_OK;
    });
}

int ago_raster(const ago_splat* splats, uint64_t n_splats,
               const uint64_t* keys, const uint32_t* splat_index,
               uint64_t n_pairs, const uint32_t* ranges, int32_t width,
               int32_t height, const ago_config* cfg, float* image,
               float* max_t) {
    return guarded([&] {
        const ags::RenderConfig c = to_cfg(cfg);
        const ags::TileGrid grid = ags::TileGrid::make(width, height, c.tile_size);
        const auto sv = to_splats(splats, n_splats);
        std::vector<ags::GaussianTilePair> pairs(n_pairs);
        for (uint64_t i = 0; i < n_pairs; ++i)
            pairs[i] = {keys[i], splat_index[i]};
        ags::Image img(width, height);
        std::vector<float> mt;
        if (max_t) mt.assign(n_splats, 0.0f);
        for (int t = 0; t < grid.tile_count(); ++t) {
            const uint32_t b = ranges[2 * t], e = ranges[2 * t + 1];
            ags::raster_tile(
                std::span<const ags::GaussianTilePair>(pairs.data() + b, e - b),
                sv, grid, t, c, img, max_t ? &mt : nullptr, nullptr);
        }
        std::memcpy(image, img.data.data(), img.data.size() * sizeof(float));
        if (max_t) std::memcpy(max_t, mt.data(), mt.size() * sizeof(float));
        return AGO_OK;
    });
}

int ago_render(const ago_scene* scene, const ago_camera* cam,
               const ago_config* cfg, const ago_lut* lut, float* image,
               uint64_t* pair_count, uint64_t* splat_count, float* max_t,
               double* stage_s) {
    return guarded([&] {
        const auto g = to_scene(scene);
        const ags::TUpperLUT l = to_lut(lut);
        const ags::RenderConfig c = to_cfg(cfg);
        ags::RecordOptions rec;
        rec.max_t = max_t != nullptr;
        const ags::RenderReport rep =
            ags::render(g, to_cam(cam), c,
                        c.mode == ags::Mode::AdaGScale ? &l : nullptr, rec);
        std::memcpy(image, rep.image.data.data(),
                    rep.image.data.size() * sizeof(float));
        *pair_count = rep.pair_count;
        *splat_count = rep.splat_count;
        if (max_t)
            std::memcpy(max_t, rep.max_t.data(), rep.max_t.size() * sizeof(float));
        if (stage_s) {
            stage_s[0] = rep.stage_times.at("preprocess");
            stage_s[1] = rep.stage_times.at("pair_gen");
            stage_s[2] = rep.stage_times.at("sort");
            stage_s[3] = rep.stage_times.at("raster");
        }
        return AGO_OK;
    });
}

// render with RecordOptions::contributions (rasterizer.cpp:135-161).
int ago_render_contributions(const ago_scene* scene, const ago_camera* cam, const ago_config* cfg,
                             const ago_lut* lut, float* image, ago_blend* out, uint64_t capacity,
                             uint64_t* count) {
    return guarded([&] {
        const auto g = to_scene(scene);
        const ags::TUpperLUT l = to_lut(lut);
        const ags::RenderConfig c = to_cfg(cfg);
        ags::RecordOptions rec;
        rec.contributions = true;
        const ags::RenderReport rep =
            ags::render(g, to_cam(cam), c, c.mode == ags::Mode::AdaGScale ? &l : nullptr, rec);
        std::memcpy(image, rep.image.data.data(), rep.image.data.size() * sizeof(float));
        *count = rep.contributions.size();
        if (!out || capacity < rep.contributions.size()) return AGO_ECAPACITY;
        for (std::size_t i = 0; i < rep.contributions.size(); ++i) {
            const ags::BlendRecord& r = rep.contributions[i];
            out[i] = ago_blend{r.pixel, r.splat, r.alpha, r.weight};
        }
        return AGO_OK;
    });
}

// calibrate_scene of the reference binding (bindings.cpp:104-127):
// build_lut + search_k (calibrate.cpp:14-155) with a default RenderConfig.
int ago_calibrate(const ago_scene* scene, const ago_camera* views, int32_t n_views, double target_drop,
                  int32_t thread_count, double* k, double* achieved, int32_t* iterations, float* bins,
                  int32_t bin_capacity, float* depth_min, float* depth_max) {
    return guarded([&] {
        const auto g = to_scene(scene);
        std::vector<ags::Camera> cams;
        for (int i = 0; i < n_views; ++i) cams.push_back(to_cam(&views[i]));
        ags::RenderConfig cfg;
        cfg.thread_count = thread_count;
        const ags::TUpperLUT lut = ags::build_lut(g, cams, cfg);
        const ags::CalibrationResult r = ags::search_k(g, cams, target_drop, cfg, lut);
        *k = r.k;
        *achieved = r.achieved_drop;
        *iterations = r.iterations;
        if (static_cast<int>(r.lut.bins.size()) > bin_capacity) return AGO_ECAPACITY;
        std::memcpy(bins, r.lut.bins.data(), r.lut.bins.size() * sizeof(float));
        *depth_min = r.lut.depth_min;
        *depth_max = r.lut.depth_max;
        return AGO_OK;
    });
}

// load_ply_file (gsio.cpp:80-157) into SoA; first call with mean == NULL
// returns the count / SH coefficients / rejected rows.
int ago_load_ply(const char* path, uint64_t* count, int32_t* coeffs, uint64_t* rejected, float* mean, float* scale,
                 float* rotation, float* opacity, float* sh) {
    return guarded([&] {
        const ags::PlyLoadResult r = ags::load_ply_file(path);
        *count = r.gaussians.size();
        *rejected = r.rejected;
        *coeffs = r.gaussians.empty() ? 1 : static_cast<int32_t>(r.gaussians.front().sh.size() / 3);
        if (!mean) return AGO_OK;
        for (std::size_t i = 0; i < r.gaussians.size(); ++i) {
            const ags::Gaussian3D& g = r.gaussians[i];
            mean[3 * i] = g.mean.x;
            mean[3 * i + 1] = g.mean.y;
            mean[3 * i + 2] = g.mean.z;
            scale[3 * i] = g.scale.x;
            scale[3 * i + 1] = g.scale.y;
            scale[3 * i + 2] = g.scale.z;
            rotation[4 * i] = g.rotation.w;
            rotation[4 * i + 1] = g.rotation.x;
            rotation[4 * i + 2] = g.rotation.y;
            rotation[4 * i + 3] = g.rotation.z;
            opacity[i] = g.opacity;
            std::memcpy(sh + i * g.sh.size(), g.sh.data(), g.sh.size() * sizeof(float));
        }
        return AGO_OK;
    });
}

// orbit_cameras (synth.cpp:254-281) around the loaded scene of `path`.
int ago_orbit_cameras(const char* path, int32_t count, int32_t width, int32_t height, float fx, float fy,
                      uint64_t seed, ago_camera* cams) {
    return guarded([&] {
        const ags::PlyLoadResult r = ags::load_ply_file(path);
        const std::vector<ags::Camera> c = ags::orbit_cameras(r.gaussians, count, width, height, fx, fy, seed);
        for (std::size_t i = 0; i < c.size(); ++i) {
            cams[i].position[0] = c[i].position.x;
            cams[i].position[1] = c[i].position.y;
            cams[i].position[2] = c[i].position.z;
            for (int k = 0; k < 9; ++k) cams[i].rotation[k] = c[i].rotation.m[k];
            cams[i].fx = c[i].fx;
            cams[i].fy = c[i].fy;
            cams[i].width = c[i].width;
            cams[i].height = c[i].height;
        }
        return AGO_OK;
    });
}

// pair_report (analysis.cpp:259-312) with the given LUT (or a built one when
// lut is NULL); rows: n_specs x {pair_count, reduction_pct, psnr_drop_db}.
int ago_pair_report(const ago_scene* scene, const ago_camera* views, int32_t n_views, const int32_t* modes,
                    const double* ks, int32_t n_specs, const ago_lut* lut, double* rows) {
    return guarded([&] {
        const auto g = to_scene(scene);
        std::vector<ags::Camera> cams;
        for (int i = 0; i < n_views; ++i) cams.push_back(to_cam(&views[i]));
        std::vector<ags::ReportSpec> specs;
        for (int i = 0; i < n_specs; ++i) specs.push_back({static_cast<ags::Mode>(modes[i]), ks[i]});
        ags::RenderConfig cfg;
        const ags::TUpperLUT l = to_lut(lut);
        const auto r = ags::pair_report(g, cams, specs, cfg, lut ? &l : nullptr);
        for (int i = 0; i < n_specs; ++i) {
            rows[3 * i] = static_cast<double>(r[i].pair_count);
            rows[3 * i + 1] = r[i].reduction_pct;
            rows[3 * i + 2] = r[i].psnr_drop_db;
        }
        return AGO_OK;
    });
}

double ago_psnr(const float* a, const float* b, uint64_t n) {
    // analysis.cpp:14-25 operates on Image; wrap the flat buffers as 1 x n/3.
    ags::Image ia(static_cast<int>(n / 3), 1), ib(static_cast<int>(n / 3), 1);
    std::memcpy(ia.data.data(), a, n * sizeof(float));
    std::memcpy(ib.data.data(), b, n * sizeof(float));
    return ags::psnr(ia, ib);
}

void ago_logf_batch(const float* x, float* y, uint64_t n) {
    for (uint64_t i = 0; i < n; ++i) y[i] = std::log(x[i]);
}

void ago_expf_batch(const float* x, float* y, uint64_t n) {
    for (uint64_t i = 0; i < n; ++i) y[i] = std::exp(x[i]);
}

}  // extern "C"

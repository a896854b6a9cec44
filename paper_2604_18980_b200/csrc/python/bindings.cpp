// bindings.cpp -- pybind11 module paper_2604_18980_b200._core.
//
// Mirrors the reference's Python module adagscale._core
// (/root/reference/proj/python/bindings.cpp:129-201): Scene, synth_scene,
// render, psnr, write_image, peripheral_score_closed, pack_pair_key with the
// same argument names, defaults, return dicts and exception types.  render()
// runs on the GPU through libagsx.so with the GIL released; the Scene keeps
// a device-resident copy after its first render.
//
// B200 additions: Renderer (one CUDA context/stream, asynchronous frames
// that stay in HBM, parity dumps), and the per-stage entry points.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <memory>
#include <mutex>
#include <numbers>
#include <stdexcept>
#include <thread>
#include <vector>

#include <sys/mman.h>

#include "agsx.h"
#include "ags/ags.hpp"
#include "ags_internal.hpp"

namespace py = pybind11;

namespace {

using f32arr = py::array_t<float, py::array::c_style | py::array::forcecast>;

struct SceneDeleter {
    void operator()(agsx_scene* s) const { agsx_scene_free(s); }
};

// Host SoA copy + lazily uploaded device copy (one per device).
struct Scene {
    std::uint64_t n = 0;
    int D = 1;
    std::vector<float> mean, scale, rot, op, sh;
    std::vector<agsx_camera> cameras;
    std::map<int, std::shared_ptr<agsx_scene>> device;
    std::mutex mu;
};

class Renderer;
Renderer& default_renderer();

[[noreturn]] void raise_status(int rc, const agsx_ctx* ctx) {
    const std::string msg = ctx ? agsx_last_error(ctx) : "agsx error";
    if (rc == AGSX_EINVAL) throw py::value_error(msg);
    if (rc == AGSX_EPAIR_BUDGET) throw ags::PairBudgetError(msg);
    if (rc == AGSX_ENOMEM) throw std::bad_alloc();
    throw std::runtime_error(msg.empty() ? "agsx: device error" : msg);
}

agsx_config make_config(const std::string& mode, double k, int threads, int tile_size, bool exact,
                        std::size_t pair_budget) {
    ags::RenderConfig def;
    ags::Mode m;
    // "aabb_fixed3": the original 3D-GS tile test (AABB at a fixed 3 sigma,
    // RenderConfig::fixed_radius_aabb, pair_gen.cpp:11-16) -- the config 2 baseline
    const bool fixed3 = mode == "aabb_fixed3";
    if (!ags::parse_mode(fixed3 ? std::string("aabb") : mode, m)) throw py::value_error("unknown mode '" + mode + "'");
    agsx_config c{};
    c.tile_size = tile_size;
    c.alpha_threshold = def.alpha_threshold;
    c.transmittance_floor = def.transmittance_floor;
    c.alpha_clamp = def.alpha_clamp;
    c.near_plane = def.near_plane;
    c.guard_band = def.guard_band;
    c.mode = static_cast<int>(m);
    c.k = static_cast<float>(k);
    c.thread_count = threads;
    c.fixed_radius_aabb = fixed3 ? 1 : 0;
    c.pair_budget = pair_budget;
    c.flags = exact ? AGSX_FLAG_EXACT_ALPHA : 0u;
    return c;
}

// bindings.cpp:44-53 of the reference: empty bins -> the all-ones LUT.
struct LutHolder {
    std::vector<float> bins;
    agsx_lut lut{};
    LutHolder(const std::vector<float>& b, float dmin, float dmax) {
        if (b.empty()) {
            bins.assign(20, 1.0f);
            lut.depth_min = 0.0f;
            lut.depth_max = 100.0f;
        } else {
            bins = b;
            lut.depth_min = dmin;
            lut.depth_max = dmax;
        }
        lut.bin_count = static_cast<int32_t>(bins.size());
        lut.bins = bins.data();
    }
};

// Pool of page-locked image buffers: a returned numpy image owns one block
// (capsule) and gives it back to the pool when the array is freed, so the
// device->host image copy runs at full link bandwidth without re-pinning.
// The page-locked bytes held by live images are capped (AGS_PINNED_POOL_MB,
// default 2048): a caller that keeps many frames gets ordinary (pageable)
// arrays past the cap -- one extra host copy each -- instead of pinning
// unbounded host memory.
class PinnedPool {
public:
    static PinnedPool& get() {
        static PinnedPool* p = new PinnedPool();  // never destroyed (capsules may outlive exit order)
        return *p;
    }
    // grow = false: a free block or nothing (no new page-locked allocation)
    void* acquire(std::size_t bytes, bool grow = true) {
        {
            std::lock_guard<std::mutex> g(mu_);
            for (auto it = free_.begin(); it != free_.end(); ++it)
                if (it->second >= bytes && it->second <= 2 * bytes) {
                    void* p = it->first;
                    sizes_[p] = it->second;
                    live_ += it->second;
                    free_.erase(it);
                    return p;
                }
            if (!grow || live_ + bytes > cap()) return nullptr;  // pageable past the cap
        }
        void* p = nullptr;
        if (agsx_host_alloc(bytes, &p) != AGSX_OK) return nullptr;
        std::lock_guard<std::mutex> g(mu_);
        sizes_[p] = bytes;
        live_ += bytes;
        return p;
    }
    // page-locked blocks that could hold `bytes` (the reuse window of
    // acquire), owned by live arrays or kept free
    std::size_t blocks(std::size_t bytes) {
        std::lock_guard<std::mutex> g(mu_);
        auto fits = [bytes](std::size_t b) { return b >= bytes && b <= 2 * bytes; };
        std::size_t n = 0;
        for (const auto& kv : sizes_) n += fits(kv.second);
        for (const auto& kv : free_) n += fits(kv.second);
        return n;
    }
    static std::size_t cap() {
        static const std::size_t c = [] {
            const char* e = std::getenv("AGS_PINNED_POOL_MB");
            const long long mb = e ? std::atoll(e) : 2048;
            return static_cast<std::size_t>(mb > 0 ? mb : 0) << 20;
        }();
        return c;
    }
    void release(void* p) {
        std::lock_guard<std::mutex> g(mu_);
        auto it = sizes_.find(p);
        if (it == sizes_.end()) return;
        live_ -= it->second;
        free_.emplace_back(p, it->second);
        sizes_.erase(it);
        while (free_.size() > 4) {  // bound the cached pinned memory
            agsx_host_free(free_.front().first);
            free_.erase(free_.begin());
        }
    }

private:
    std::mutex mu_;
    std::vector<std::pair<void*, std::size_t>> free_;
    std::map<void*, std::size_t> sizes_;
    std::size_t live_ = 0;  // page-locked bytes owned by live arrays
};

template <typename T>
py::array_t<T> pinned_image(int h, int w) {
    const std::size_t bytes = static_cast<std::size_t>(h) * w * 3 * sizeof(T);
    void* p = PinnedPool::get().acquire(bytes);
    if (!p) return py::array_t<T>({h, w, 3});  // pageable fallback for the host buffer only
    py::capsule owner(p, [](void* q) { PinnedPool::get().release(q); });
    return py::array_t<T>({h, w, 3}, static_cast<T*>(p), owner);
}

// A fresh pageable host image for a synchronous frame that is rendered into
// the renderer's page-locked staging block: host threads fault the array's
// pages in (transparent huge pages requested) while the GPU renders, then
// copy the staged frame in by slices.  Used when the caller keeps its
// images, so no pooled block is free: a new 191 MB page-locked block costs
// ~95 ms and a pageable device->host copy ~49 ms, this ~5 ms at 4608x3456.
class PagedFill {
public:
    PagedFill(void* dst, std::size_t bytes) : dst_(static_cast<char*>(dst)), bytes_(bytes) {
        const std::size_t by_size = std::max<std::size_t>(1, bytes >> 18);  // one thread per 256 KB, up to 16
        nt_ = static_cast<unsigned>(std::min<std::size_t>({16, by_size, std::max(1u, std::thread::hardware_concurrency())}));
        per_ = ((bytes + nt_ - 1) / nt_ + 4095) & ~std::size_t{4095};
        const std::uintptr_t b = reinterpret_cast<std::uintptr_t>(dst_);
        const std::uintptr_t a = (b + (1u << 21) - 1) & ~static_cast<std::uintptr_t>((1u << 21) - 1);
        const std::uintptr_t e = (b + bytes) & ~static_cast<std::uintptr_t>((1u << 21) - 1);
        if (e > a) madvise(reinterpret_cast<void*>(a), e - a, MADV_HUGEPAGE);  // advisory: ignore failures
        volatile char* base = dst_;
        for (unsigned t = 0; t < nt_; ++t)
            if (t * per_ < bytes_)
                pool_.emplace_back([base, lo = t * per_, hi = std::min(bytes_, (t + 1) * per_)] {
                    for (std::size_t i = lo; i < hi; i += 4096) base[i] = 0;
                });
    }
    ~PagedFill() { join(); }
    void copy_from(const void* src) {
        join();
        const char* s = static_cast<const char*>(src);
        for (unsigned t = 1; t < nt_; ++t)
            if (t * per_ < bytes_)
                pool_.emplace_back([=, this] { std::memcpy(dst_ + t * per_, s + t * per_, std::min(bytes_, (t + 1) * per_) - t * per_); });
        std::memcpy(dst_, s, std::min(bytes_, per_));
        join();
    }

private:
    void join() {
        for (auto& th : pool_) th.join();
        pool_.clear();
    }
    char* dst_;
    std::size_t bytes_, per_ = 0;
    unsigned nt_ = 1;
    std::vector<std::thread> pool_;
};

agsx_camera camera_from(const py::dict& d) {
    agsx_camera c{};
    auto pos = d["position"].cast<std::vector<float>>();
    auto rot = d["rotation"].cast<std::vector<float>>();
    if (pos.size() != 3 || rot.size() != 9) throw py::value_error("camera needs position[3], rotation[9]");
    std::copy(pos.begin(), pos.end(), c.position);
    std::copy(rot.begin(), rot.end(), c.rotation);
    c.fx = d["fx"].cast<float>();
    c.fy = d["fy"].cast<float>();
    c.width = d["width"].cast<int>();
    c.height = d["height"].cast<int>();
    return c;
}

class Renderer {
public:
    explicit Renderer(int device) : device_(device) {
        const int rc = agsx_create(device, &ctx_);
        if (rc != AGSX_OK) throw std::runtime_error("agsx_create failed: no usable CUDA device " + std::to_string(device));
    }
    ~Renderer() {
        if (staging_) agsx_host_free(staging_);
        if (ctx_) agsx_destroy(ctx_);
    }
    Renderer(const Renderer&) = delete;
    Renderer& operator=(const Renderer&) = delete;

    agsx_scene* device_scene(Scene& s) {
        std::lock_guard<std::mutex> g(s.mu);
        auto it = s.device.find(device_);
        if (it != s.device.end()) return it->second.get();
        agsx_scene_desc d{s.n, s.D, s.mean.data(), s.scale.data(), s.rot.data(), s.op.data(), s.sh.data()};
        agsx_scene* out = nullptr;
        const int rc = agsx_scene_upload(ctx_, &d, &out);
        if (rc != AGSX_OK) raise_status(rc, ctx_);
        s.device[device_] = std::shared_ptr<agsx_scene>(out, SceneDeleter{});
        return out;
    }

    static const agsx_camera& view_of(const Scene& s, int view) {
        if (view < 0 || view >= static_cast<int>(s.cameras.size()))
            throw std::out_of_range("view index out of range");
        return s.cameras[view];
    }

    py::dict render(Scene& scene, int view, const std::string& mode, double k,
                    const std::vector<float>& lut_bins, float dmin, float dmax, int threads,
                    int tile_size, bool exact, bool max_t, std::size_t pair_budget, bool image,
                    bool image_u8 = false) {
        const agsx_camera cam = view_of(scene, view);
        const agsx_config cfg = make_config(mode, k, threads, tile_size, exact, pair_budget);
        const LutHolder lut(lut_bins, dmin, dmax);
        agsx_scene* dev = device_scene(scene);
        if (image && image_u8 && !max_t) {  // frame quantised on the device (row f3)
            std::unique_ptr<PagedFill> fill;
            py::array_t<std::uint8_t> img8 = sync_image<std::uint8_t>(cam.height, cam.width, fill);
            std::uint8_t* dst8 = img8.mutable_data();
            const std::size_t bytes8 = static_cast<std::size_t>(cam.height) * cam.width * 3;
            agsx_frame f{};
            int rc;
            {
                py::gil_scoped_release nogil;
                std::lock_guard<std::mutex> g(mu_);
                std::uint8_t* to = fill ? static_cast<std::uint8_t*>(staging(bytes8)) : dst8;
                rc = agsx_render_u8(ctx_, dev, &cam, &cfg, cfg.mode == AGSX_MODE_ADAGSCALE ? &lut.lut : nullptr, to, &f);
                if (rc == AGSX_OK && fill) fill->copy_from(to);
            }
            if (rc != AGSX_OK) raise_status(rc, ctx_);
            py::dict out;
            out["image"] = img8;
            out["pair_count"] = f.pair_count;
            out["splat_count"] = f.splat_count;
            py::dict times;
            const char* names[4] = {"preprocess", "pair_gen", "sort", "raster"};
            for (int i = 0; i < 4; ++i) times[names[i]] = f.stage_ms[i] * 1e-3;
            out["stage_times"] = times;
            return out;
        }
        py::array_t<float> img;
        std::unique_ptr<PagedFill> fill;
        if (image) img = sync_image<float>(cam.height, cam.width, fill);
        std::vector<float> mt;
        agsx_frame f{};
        if (image) f.image = img.mutable_data();
        const std::size_t img_bytes = static_cast<std::size_t>(cam.height) * cam.width * 3 * sizeof(float);
        if (max_t) {
            mt.assign(std::max<std::uint64_t>(scene.n, 1), 0.0f);
            f.max_t = mt.data();
        }
        int rc;
        {
            py::gil_scoped_release nogil;
            std::lock_guard<std::mutex> g(mu_);
            float* dst = f.image;
            if (fill) f.image = static_cast<float*>(staging(img_bytes));
            rc = agsx_render(ctx_, dev, &cam, &cfg, cfg.mode == AGSX_MODE_ADAGSCALE ? &lut.lut : nullptr, &f);
            if (rc == AGSX_OK && fill) fill->copy_from(f.image);
            f.image = dst;
        }
        if (rc != AGSX_OK) raise_status(rc, ctx_);
        py::dict out;
        if (image) out["image"] = img;
        out["pair_count"] = f.pair_count;
        out["splat_count"] = f.splat_count;
        py::dict times;
        const char* names[4] = {"preprocess", "pair_gen", "sort", "raster"};
        for (int i = 0; i < 4; ++i) times[names[i]] = f.stage_ms[i] * 1e-3;
        out["stage_times"] = times;
        if (max_t) {
            // per splat in preprocess order (RenderReport::max_t)
            py::array_t<std::uint8_t> alive(scene.n);
            rc = agsx_dump_tile_counts(ctx_, nullptr, alive.mutable_data(), scene.n);
            if (rc != AGSX_OK) raise_status(rc, ctx_);
            std::vector<float> comp;
            comp.reserve(f.splat_count);
            const std::uint8_t* a = alive.data();
            for (std::uint64_t i = 0; i < scene.n; ++i)
                if (a[i]) comp.push_back(mt[i]);
            out["max_t"] = py::array_t<float>(comp.size(), comp.data());
        }
        return out;
    }

    void render_async(Scene& scene, int view, const std::string& mode, double k,
                      const std::vector<float>& lut_bins, float dmin, float dmax, int tile_size,
                      bool exact, std::size_t pair_budget, py::object camera) {
        if (!pending_image_.is_none())
            throw std::runtime_error("a host frame is in flight on this renderer; call wait() first");
        const agsx_camera cam = camera.is_none() ? view_of(scene, view) : camera_from(camera.cast<py::dict>());
        const agsx_config cfg = make_config(mode, k, 0, tile_size, exact, pair_budget);
        const LutHolder lut(lut_bins, dmin, dmax);
        agsx_scene* dev = device_scene(scene);
        int rc;
        {
            py::gil_scoped_release nogil;
            rc = agsx_render_async(ctx_, dev, &cam, &cfg, cfg.mode == AGSX_MODE_ADAGSCALE ? &lut.lut : nullptr);
        }
        if (rc != AGSX_OK) raise_status(rc, ctx_);
    }

    // Frame rasterised into caller-owned device memory (e.g. a torch tensor
    // that a collective gathers); `target` is its address (H*W*3 f32).
    void render_async_to(Scene& scene, int view, std::uintptr_t target, const std::string& mode, double k,
                         const std::vector<float>& lut_bins, float dmin, float dmax, int tile_size, bool exact,
                         std::size_t pair_budget, py::object camera) {
        if (!pending_image_.is_none())
            throw std::runtime_error("a host frame is in flight on this renderer; call wait() first");
        const agsx_camera cam = camera.is_none() ? view_of(scene, view) : camera_from(camera.cast<py::dict>());
        const agsx_config cfg = make_config(mode, k, 0, tile_size, exact, pair_budget);
        const LutHolder lut(lut_bins, dmin, dmax);
        agsx_scene* dev = device_scene(scene);
        int rc;
        {
            py::gil_scoped_release nogil;
            rc = agsx_render_async_to(ctx_, dev, &cam, &cfg, cfg.mode == AGSX_MODE_ADAGSCALE ? &lut.lut : nullptr,
                                      reinterpret_cast<float*>(target));
        }
        if (rc != AGSX_OK) raise_status(rc, ctx_);
    }

    // Frame delivered to a page-locked host image (banded copies behind the
    // raster); wait() returns it as out["image"].  Two renderers on one
    // device alternate frames so one frame's PCIe egress overlaps the next
    // frame's kernels (batch.render_views).
    void render_async_host(Scene& scene, int view, const std::string& mode, double k,
                           const std::vector<float>& lut_bins, float dmin, float dmax, int tile_size, bool exact,
                           std::size_t pair_budget, py::object camera, bool image_u8) {
        if (!pending_image_.is_none())  // the in-flight frame still writes into its host image
            throw std::runtime_error("render_async_host: a host frame is in flight; call wait() first");
        const agsx_camera cam = camera.is_none() ? view_of(scene, view) : camera_from(camera.cast<py::dict>());
        const agsx_config cfg = make_config(mode, k, 0, tile_size, exact, pair_budget);
        const LutHolder lut(lut_bins, dmin, dmax);
        agsx_scene* dev = device_scene(scene);
        const agsx_lut* lp = cfg.mode == AGSX_MODE_ADAGSCALE ? &lut.lut : nullptr;
        int rc;
        if (image_u8) {
            py::array_t<std::uint8_t> img = pinned_image<std::uint8_t>(cam.height, cam.width);
            {
                py::gil_scoped_release nogil;
                rc = agsx_render_async_host_u8(ctx_, dev, &cam, &cfg, lp, img.mutable_data());
            }
            if (rc != AGSX_OK) raise_status(rc, ctx_);
            pending_image_ = img;
        } else {
            py::array_t<float> img = pinned_image<float>(cam.height, cam.width);
            {
                py::gil_scoped_release nogil;
                rc = agsx_render_async_host(ctx_, dev, &cam, &cfg, lp, img.mutable_data());
            }
            if (rc != AGSX_OK) raise_status(rc, ctx_);
            pending_image_ = img;
        }
    }

    py::dict wait() {
        agsx_frame f{};
        int rc;
        {
            py::gil_scoped_release nogil;
            rc = agsx_render_wait(ctx_, &f);
        }
        py::object img = pending_image_;
        pending_image_ = py::none();
        if (rc != AGSX_OK) raise_status(rc, ctx_);
        py::dict out;
        if (!img.is_none()) out["image"] = img;
        out["pair_count"] = f.pair_count;
        out["splat_count"] = f.splat_count;
        out["stage_ms"] = std::vector<float>(f.stage_ms, f.stage_ms + 4);
        return out;
    }

    // calibrate_scene (bindings.cpp:104-127 of the reference): LUT from the
    // first min(calib_views, cameras) views, then the K search; on the GPU.
    py::dict calibrate(Scene& scene, double target_drop, int calib_views, int threads) {
        const int n = std::min<int>(calib_views, static_cast<int>(scene.cameras.size()));
        if (n < 1) throw py::value_error("scene has no cameras");
        ags::RenderConfig def;
        def.thread_count = threads;
        const agsx_config cfg = ags::detail::to_c(def);
        agsx_scene* dev = device_scene(scene);
        ags::CalibrationResult res;
        {
            py::gil_scoped_release nogil;
            std::lock_guard<std::mutex> g(mu_);
            const ags::TUpperLUT lut = ags::detail::build_lut_device(ctx_, dev, scene.cameras.data(), n, cfg);
            res = ags::detail::search_k_device(ctx_, dev, scene.cameras.data(), n, target_drop, cfg, lut, false);
        }
        py::dict out;
        out["k"] = res.k;
        out["target_drop"] = res.target_drop;
        out["achieved_drop"] = res.achieved_drop;
        out["iterations"] = res.iterations;
        out["lut_bins"] = res.lut.bins;
        out["lut_depth_min"] = res.lut.depth_min;
        out["lut_depth_max"] = res.lut.depth_max;
        return out;
    }

    // build_lut's fold (calibrate.cpp:14-41) over `views`: the per-depth-bin
    // max of max_t and whether the bin saw a blended splat.  The fold is a max,
    // so the folds of view blocks merge exactly into the fold of all views
    // (batch.pair_report across ranks).
    py::dict fold_max_t(Scene& scene, std::vector<int> views, int threads) {
        if (views.empty())
            for (int v = 0; v < static_cast<int>(scene.cameras.size()); ++v) views.push_back(v);
        std::vector<agsx_camera> cams;
        for (int v : views) cams.push_back(view_of(scene, v));
        ags::RenderConfig def;
        def.thread_count = threads;
        const agsx_config cfg = ags::detail::to_c(def);
        const ags::TUpperLUT shape;
        const agsx_lut l{shape.depth_min, shape.depth_max, static_cast<int32_t>(shape.bins.size()), nullptr};
        std::vector<float> folded(shape.bins.size(), 0.0f);
        std::vector<std::uint8_t> observed(shape.bins.size(), 0);
        agsx_scene* dev = device_scene(scene);
        {
            py::gil_scoped_release nogil;
            std::lock_guard<std::mutex> g(mu_);
            for (const agsx_camera& c : cams) {
                const int rc = agsx_fold_max_t(ctx_, dev, &c, &cfg, &l, folded.data(), observed.data());
                if (rc != AGSX_OK) {
                    py::gil_scoped_acquire gil;
                    raise_status(rc, ctx_);
                }
            }
        }
        py::dict out;
        out["folded"] = folded;
        std::vector<bool> obs(observed.begin(), observed.end());
        out["observed"] = obs;
        out["depth_min"] = shape.depth_min;
        out["depth_max"] = shape.depth_max;
        return out;
    }

    // psnr (analysis.cpp:14-25) of two device frames of n floats, numerator
    // reduced on the GPU (row f3; e.g. torch tensors of a gathered path).
    double psnr_device(std::uintptr_t a, std::uintptr_t b, std::uint64_t n) {
        double se = 0.0;
        int rc;
        {
            py::gil_scoped_release nogil;
            std::lock_guard<std::mutex> g(mu_);
            rc = agsx_sq_err(ctx_, reinterpret_cast<const float*>(a), reinterpret_cast<const float*>(b), n, &se);
        }
        if (rc != AGSX_OK) raise_status(rc, ctx_);
        if (se == 0.0) return std::numeric_limits<double>::infinity();
        return 10.0 * std::log10(1.0 / (se / static_cast<double>(n)));
    }

    // pair_report (analysis.cpp:259-312) over views of the scene (row f4).
    py::list pair_report(Scene& scene, const std::vector<py::tuple>& specs, std::vector<int> views,
                         const std::vector<float>& lut_bins, float dmin, float dmax, int threads) {
        if (views.empty())
            for (int v = 0; v < static_cast<int>(scene.cameras.size()); ++v) views.push_back(v);
        std::vector<agsx_camera> cams;
        for (int v : views) cams.push_back(view_of(scene, v));
        std::vector<ags::ReportSpec> sp;
        for (const py::tuple& t : specs) {
            ags::Mode m;
            if (!ags::parse_mode(t[0].cast<std::string>(), m)) throw py::value_error("unknown mode");
            sp.push_back({m, t.size() > 1 ? t[1].cast<double>() : 0.0});
        }
        ags::RenderConfig def;
        def.thread_count = threads;
        const agsx_config cfg = ags::detail::to_c(def);
        ags::TUpperLUT lut;
        if (!lut_bins.empty()) {
            lut.bins = lut_bins;
            lut.depth_min = dmin;
            lut.depth_max = dmax;
        }
        agsx_scene* dev = device_scene(scene);
        std::vector<ags::PairReportRow> rows;
        {
            py::gil_scoped_release nogil;
            std::lock_guard<std::mutex> g(mu_);
            rows = ags::detail::pair_report_device(ctx_, dev, cams.data(), static_cast<int>(cams.size()), sp, cfg,
                                                   lut_bins.empty() ? nullptr : &lut);
        }
        py::list out;
        for (const auto& r : rows) {
            py::dict d;
            d["mode"] = r.mode;
            d["k"] = r.k;
            d["pair_count"] = r.pair_count;
            d["reduction_pct"] = r.reduction_pct;
            d["psnr_drop_db"] = r.psnr_drop_db;
            d["t_preprocess"] = r.t_preprocess;
            d["t_pair_gen"] = r.t_pair_gen;
            d["t_sort"] = r.t_sort;
            d["t_raster"] = r.t_raster;
            d["views"] = cams.size();
            out.append(d);
        }
        return out;
    }

    py::array_t<float> stage_history(int max_frames) {
        std::vector<float> ms(static_cast<std::size_t>(std::max(max_frames, 0)) * 4);
        int32_t n = 0;
        const int rc = agsx_stage_history(ctx_, ms.data(), max_frames, &n);
        if (rc != AGSX_OK) raise_status(rc, ctx_);
        py::array_t<float> out({static_cast<py::ssize_t>(n), py::ssize_t(4)});
        std::memcpy(out.mutable_data(), ms.data(), static_cast<std::size_t>(n) * 4 * sizeof(float));
        return out;
    }

    py::dict frame_stats() {
        std::uint64_t v[16] = {};
        const int rc = agsx_frame_stats(ctx_, v, 16);
        if (rc != AGSX_OK) raise_status(rc, ctx_);
        py::dict d;
        const char* names[16] = {"splat_count", "splats_with_tiles", "pair_count", "p_it", "overflow", "tiles",
                                 "raster_iters", "raster_evals", "raster_fast", "raster_exact",
                                 "raster_iters_live_le32", "raster_iters_live_le64", "raster_iters_empty",
                                 "raster_iters_no_live_pixel", "depth_passes", "bucketed_sort"};
        for (int i = 0; i < 16; ++i) d[names[i]] = v[i];
        return d;
    }

    py::tuple device_image() {
        float* p = nullptr;
        int32_t w = 0, h = 0;
        const int rc = agsx_device_image(ctx_, &p, &w, &h);
        if (rc != AGSX_OK) raise_status(rc, ctx_);
        return py::make_tuple(reinterpret_cast<std::uintptr_t>(p), w, h);
    }

    py::array_t<std::uint32_t> dump_tile_counts(std::uint64_t n) {
        py::array_t<std::uint32_t> c(n);
        const int rc = agsx_dump_tile_counts(ctx_, c.mutable_data(), nullptr, n);
        if (rc != AGSX_OK) raise_status(rc, ctx_);
        return c;
    }

    py::tuple dump_sorted_pairs() {
        std::uint64_t n = 0;
        int rc = agsx_dump_sorted_pairs(ctx_, nullptr, nullptr, 0, &n);
        if (rc != AGSX_OK && rc != AGSX_ECAPACITY) raise_status(rc, ctx_);
        py::array_t<std::uint64_t> keys(n);
        py::array_t<std::uint32_t> gids(n);
        rc = agsx_dump_sorted_pairs(ctx_, keys.mutable_data(), gids.mutable_data(), n, &n);
        if (rc != AGSX_OK) raise_status(rc, ctx_);
        return py::make_tuple(keys, gids);
    }

    py::array_t<std::uint32_t> dump_ranges(std::uint64_t tile_count) {
        py::array_t<std::uint32_t> r({static_cast<py::ssize_t>(tile_count), py::ssize_t(2)});
        const int rc = agsx_dump_ranges(ctx_, r.mutable_data(), tile_count);
        if (rc != AGSX_OK) raise_status(rc, ctx_);
        return r;
    }

    std::uintptr_t stream() const { return reinterpret_cast<std::uintptr_t>(agsx_stream(ctx_)); }
    std::uint64_t kernel_launches() const { return agsx_kernel_launches(ctx_); }
    int device() const { return device_; }

private:
    int device_;
    py::object pending_image_ = py::none();  // host image of the frame in flight (render_async_host)
    agsx_ctx* ctx_ = nullptr;
    std::mutex mu_;
    void* staging_ = nullptr;  // page-locked frame staging for kept images (grow-only; under mu_)
    std::size_t staging_bytes_ = 0;

    // The synchronous frame's host image: a pooled page-locked block when one
    // is free (or the pool holds fewer than two of this size, so a caller that
    // drops each frame runs on two blocks), else a fresh pageable array that the frame
    // reaches through the staging block (PagedFill).
    template <typename T>
    py::array_t<T> sync_image(int h, int w, std::unique_ptr<PagedFill>& fill) {
        const std::size_t bytes = static_cast<std::size_t>(h) * w * 3 * sizeof(T);
        PinnedPool& pool = PinnedPool::get();
        if (void* p = pool.acquire(bytes, pool.blocks(bytes) < 2)) {
            py::capsule owner(p, [](void* q) { PinnedPool::get().release(q); });
            return py::array_t<T>({h, w, 3}, static_cast<T*>(p), owner);
        }
        py::array_t<T> a({h, w, 3});
        fill = std::make_unique<PagedFill>(a.mutable_data(), bytes);
        return a;
    }
    void* staging(std::size_t bytes) {  // caller holds mu_
        if (bytes > staging_bytes_) {
            if (staging_) agsx_host_free(staging_);
            staging_ = nullptr;
            staging_bytes_ = 0;
            if (agsx_host_alloc(bytes, &staging_) != AGSX_OK) throw std::bad_alloc();
            staging_bytes_ = bytes;
        }
        return staging_;
    }
};

Renderer& default_renderer() {
    static std::unique_ptr<Renderer> r;
    static std::mutex mu;
    std::lock_guard<std::mutex> g(mu);
    if (!r) {
        const char* e = std::getenv("AGS_DEVICE");
        r = std::make_unique<Renderer>(e ? std::atoi(e) : 0);
    }
    return *r;
}

std::shared_ptr<Scene> make_synth(std::uint64_t seed, int count, const std::string& layout, int cameras,
                                  int width, int height, float focal) {
    if (count < 1) throw py::value_error("synth_scene: count must be >= 1");
    auto s = std::make_shared<Scene>();
    s->n = static_cast<std::uint64_t>(count);
    s->D = 1;
    s->mean.resize(3 * s->n);
    s->scale.resize(3 * s->n);
    s->rot.resize(4 * s->n);
    s->op.resize(s->n);
    s->sh.resize(3 * s->n);
    s->cameras.resize(std::max(cameras, 0));
    int rc;
    {
        py::gil_scoped_release nogil;
        rc = ags_synth_scene_soa(seed, count, layout.c_str(), cameras, width, height, focal, focal,
                                 s->mean.data(), s->scale.data(), s->rot.data(), s->op.data(),
                                 s->sh.data(), s->cameras.data());
    }
    if (rc != 0) throw py::value_error("synth_scene: unknown layout '" + layout + "'");
    return s;
}

std::shared_ptr<Scene> scene_from_arrays(f32arr mean, f32arr scale, f32arr rotation, f32arr opacity,
                                         f32arr sh, const std::vector<py::dict>& cameras) {
    auto s = std::make_shared<Scene>();
    const auto n = static_cast<std::uint64_t>(opacity.size());
    if (mean.size() != static_cast<py::ssize_t>(3 * n) || scale.size() != static_cast<py::ssize_t>(3 * n) ||
        rotation.size() != static_cast<py::ssize_t>(4 * n) || sh.size() % (3 * std::max<std::uint64_t>(n, 1)) != 0)
        throw py::value_error("inconsistent scene array sizes");
    s->n = n;
    s->D = n ? static_cast<int>(sh.size() / (3 * n)) : 1;
    if (!(s->D == 1 || s->D == 4 || s->D == 9 || s->D == 16))
        throw py::value_error("sh coefficient count must be 3*d^2 for d in {1,2,3,4}");
    s->mean.assign(mean.data(), mean.data() + mean.size());
    s->scale.assign(scale.data(), scale.data() + scale.size());
    s->rot.assign(rotation.data(), rotation.data() + rotation.size());
    s->op.assign(opacity.data(), opacity.data() + opacity.size());
    s->sh.assign(sh.data(), sh.data() + sh.size());
    for (const py::dict& d : cameras) {
        agsx_camera c{};
        auto pos = d["position"].cast<std::vector<float>>();
        auto rot = d["rotation"].cast<std::vector<float>>();
        if (pos.size() != 3 || rot.size() != 9) throw py::value_error("camera needs position[3], rotation[9]");
        std::copy(pos.begin(), pos.end(), c.position);
        std::copy(rot.begin(), rot.end(), c.rotation);
        c.fx = d["fx"].cast<float>();
        c.fy = d["fy"].cast<float>();
        c.width = d["width"].cast<int>();
        c.height = d["height"].cast<int>();
        s->cameras.push_back(c);
    }
    return s;
}

// load_ply_scene (bindings.cpp:35-42 of the reference): the PLY's Gaussians
// plus a generated camera orbit; decoded by host threads into the SoA arrays
// the device upload takes.
std::shared_ptr<Scene> load_ply_scene(const std::string& path, int orbit_views, int width, int height, float focal,
                                      std::uint64_t seed) {
    auto s = std::make_shared<Scene>();
    std::vector<ags::Camera> cams;
    {
        py::gil_scoped_release nogil;
        ags::PlySoA p = ags::load_ply_soa(path);
        cams = ags::orbit_cameras(p.mean.data(), p.count, orbit_views, width, height, focal, focal, seed);
        s->n = p.count;
        s->D = p.sh_coeffs;
        s->mean = std::move(p.mean);
        s->scale = std::move(p.scale);
        s->rot = std::move(p.rotation);
        s->op = std::move(p.opacity);
        s->sh = std::move(p.sh);
    }
    for (const ags::Camera& c : cams) s->cameras.push_back(ags::detail::to_c(c));
    return s;
}

py::dict camera_dict(const agsx_camera& c) {
    py::dict d;
    d["position"] = std::vector<float>(c.position, c.position + 3);
    d["rotation"] = std::vector<float>(c.rotation, c.rotation + 9);
    d["fx"] = c.fx;
    d["fy"] = c.fy;
    d["width"] = c.width;
    d["height"] = c.height;
    return d;
}

void check_image(const f32arr& a) {
    if (a.ndim() != 3 || a.shape(2) != 3) throw py::value_error("expected an (H, W, 3) float array");
}

// ---- stage entry points over numpy (parity hooks) ------------------------
py::array splats_to_numpy(const std::vector<agsx_splat_view>& v) {
    // structured dtype identical to ags::SplatView
    py::list names, formats, offsets;
    auto add = [&](const char* n, const char* f, int off) {
        names.append(n);
        formats.append(f);
        offsets.append(off);
    };
    add("mean2d", "(2,)<f4", 0);
    add("cov2d", "(3,)<f4", 8);
    add("inv_cov", "(3,)<f4", 20);
    add("depth", "<f4", 32);
    add("rgb", "(3,)<f4", 36);
    add("opacity", "<f4", 48);
    add("th", "<f4", 52);
    add("source_id", "<u4", 56);
    py::dict spec;
    spec["names"] = names;
    spec["formats"] = formats;
    spec["offsets"] = offsets;
    spec["itemsize"] = 60;
    py::dtype dt = py::dtype::from_args(spec);
    py::array out(dt, std::vector<py::ssize_t>{static_cast<py::ssize_t>(v.size())});
    if (!v.empty()) std::memcpy(out.mutable_data(), v.data(), v.size() * sizeof(agsx_splat_view));
    return out;
}

}  // namespace

PYBIND11_MODULE(_core, m) {
    m.doc() = "B200-native tile-based gaussian splatting renderer with viewpoint-adaptive "
              "pair reduction (AdaGScale); drop-in for adagscale._core";

    py::register_exception<ags::PairBudgetError>(m, "PairBudgetError", PyExc_RuntimeError);

    py::class_<Scene, std::shared_ptr<Scene>>(m, "Scene")
        .def_property_readonly("gaussian_count", [](const Scene& s) { return s.n; })
        .def_property_readonly("camera_count", [](const Scene& s) { return s.cameras.size(); })
        .def_property_readonly("sh_coeffs", [](const Scene& s) { return s.D; })
        .def("camera", [](const Scene& s, int i) { return camera_dict(Renderer::view_of(s, i)); })
        .def("arrays",
             [](const Scene& s) {
                 const auto n = static_cast<py::ssize_t>(s.n);
                 py::dict d;
                 d["mean"] = py::array_t<float>({n, py::ssize_t(3)}, s.mean.data());
                 d["scale"] = py::array_t<float>({n, py::ssize_t(3)}, s.scale.data());
                 d["rotation"] = py::array_t<float>({n, py::ssize_t(4)}, s.rot.data());
                 d["opacity"] = py::array_t<float>({n}, s.op.data());
                 d["sh"] = py::array_t<float>({n, py::ssize_t(s.D), py::ssize_t(3)}, s.sh.data());
                 return d;
             })
        .def_static("from_arrays", &scene_from_arrays, py::arg("mean"), py::arg("scale"),
                    py::arg("rotation"), py::arg("opacity"), py::arg("sh"), py::arg("cameras"))
        .def("__repr__", [](const Scene& s) {
            return "<adagscale.Scene " + std::to_string(s.n) + " gaussians, " +
                   std::to_string(s.cameras.size()) + " cameras>";
        });

    m.def("synth_scene", &make_synth, py::arg("seed"), py::arg("count"), py::arg("layout") = "slab",
          py::arg("cameras") = 24, py::arg("width") = 640, py::arg("height") = 480,
          py::arg("focal") = 500.0f, "Deterministic synthetic scene with its camera set");

    m.def(
        "render",
        [](Scene& scene, int view, const std::string& mode, double k, const std::vector<float>& lut_bins,
           float lut_depth_min, float lut_depth_max, int threads, int tile_size, bool exact, bool max_t,
           std::size_t pair_budget, bool image_u8) {
            return default_renderer().render(scene, view, mode, k, lut_bins, lut_depth_min, lut_depth_max,
                                             threads, tile_size, exact, max_t, pair_budget, true, image_u8);
        },
        py::arg("scene"), py::arg("view") = 0, py::arg("mode") = "ellipse", py::arg("k") = 0.0,
        py::arg("lut_bins") = std::vector<float>{}, py::arg("lut_depth_min") = 0.0f,
        py::arg("lut_depth_max") = 100.0f, py::arg("threads") = 0, py::arg("tile_size") = 16,
        py::arg("exact") = false, py::arg("max_t") = false,
        py::arg("pair_budget") = std::size_t{1} << 27, py::arg("image_u8") = false,
        "Render one view on the GPU; returns dict with image, pair_count, splat_count, stage_times");

    m.def("load_ply", &load_ply_scene, py::arg("path"), py::arg("orbit_views") = 24, py::arg("width") = 640,
          py::arg("height") = 480, py::arg("focal") = 500.0f, py::arg("seed") = 1,
          "Trained splat model plus a generated camera orbit");
    py::register_exception<ags::IoError>(m, "IoError", PyExc_RuntimeError);

    m.def(
        "calibrate",
        [](Scene& scene, double target_drop, int calib_views, int threads) {
            return default_renderer().calibrate(scene, target_drop, calib_views, threads);
        },
        py::arg("scene"), py::arg("target_drop"), py::arg("calib_views") = 16, py::arg("threads") = 0,
        "Fit the T-upper LUT and binary-search K for a PSNR-drop budget (on the GPU)");

    m.def(
        "psnr",
        [](const f32arr& a, const f32arr& b) {
            check_image(a);
            check_image(b);
            if (a.shape(0) != b.shape(0) || a.shape(1) != b.shape(1))
                throw py::value_error("psnr: image dimensions differ");
            return ags_psnr(a.data(), b.data(), static_cast<std::uint64_t>(a.size()));
        },
        py::arg("a"), py::arg("b"));

    m.def(
        "write_image",
        [](const py::array_t<std::uint8_t, py::array::c_style>& a, const std::string& path) {
            // already-quantised PPM bytes (render(..., image_u8=True))
            if (a.ndim() != 3 || a.shape(2) != 3) throw py::value_error("expected an (H, W, 3) uint8 array");
            std::ofstream out(path, std::ios::binary);
            if (!out) throw std::runtime_error("cannot open '" + path + "' for writing");
            out << "P6\n" << a.shape(1) << " " << a.shape(0) << "\n255\n";
            out.write(reinterpret_cast<const char*>(a.data()), static_cast<std::streamsize>(a.size()));
            if (!out) throw std::runtime_error("write failure on '" + path + "'");
        },
        py::arg("image"), py::arg("path"));
    m.def(
        "write_image",
        [](const f32arr& a, const std::string& path) {
            // 8-bit binary PPM, round-half-away of clamp(v)*255 (gsio.cpp:265-281)
            check_image(a);
            const int h = static_cast<int>(a.shape(0)), w = static_cast<int>(a.shape(1));
            std::ofstream out(path, std::ios::binary);
            if (!out) throw std::runtime_error("cannot open '" + path + "' for writing");
            out << "P6\n" << w << " " << h << "\n255\n";
            std::vector<unsigned char> px(static_cast<std::size_t>(w) * h * 3);
            const float* d = a.data();
            for (std::size_t i = 0; i < px.size(); ++i) {
                const float v = d[i] < 0.0f ? 0.0f : (1.0f < d[i] ? 1.0f : d[i]);
                px[i] = static_cast<unsigned char>(std::lround(static_cast<double>(v) * 255.0));
            }
            out.write(reinterpret_cast<const char*>(px.data()), static_cast<std::streamsize>(px.size()));
            if (!out) throw std::runtime_error("write failure on '" + path + "'");
        },
        py::arg("image"), py::arg("path"), "8-bit binary PPM");

    m.def(
        "peripheral_score_closed",
        [](float cov_xx, float cov_xy, float cov_yy, float x, float t_const, float tau) {
            // t_const * 2*pi*sqrt(det(cov2d)) * (x - tau)  (calibrate.cpp:67-74)
            const float det = cov_xx * cov_yy - cov_xy * cov_xy;
            return static_cast<double>(t_const) * 2.0 * std::numbers::pi *
                   std::sqrt(static_cast<double>(det)) * (static_cast<double>(x) - static_cast<double>(tau));
        },
        py::arg("cov_xx"), py::arg("cov_xy"), py::arg("cov_yy"), py::arg("x"), py::arg("t_const") = 1.0f,
        py::arg("tau") = 1.0f / 255.0f);

    m.def("pack_pair_key", &ags::pack_pair_key, py::arg("tile"), py::arg("depth"));
    m.def("format_double", &ags::format_double, py::arg("v"), "shortest round-trip (std::to_chars)");
    m.def(
        "pair_report_csv",
        [](const std::vector<py::dict>& rows) {
            std::vector<ags::PairReportRow> r;
            for (const py::dict& d : rows)
                r.push_back({d["mode"].cast<std::string>(), d["k"].cast<double>(), d["pair_count"].cast<std::size_t>(),
                             d["reduction_pct"].cast<double>(), d["psnr_drop_db"].cast<double>(),
                             d["t_preprocess"].cast<double>(), d["t_pair_gen"].cast<double>(),
                             d["t_sort"].cast<double>(), d["t_raster"].cast<double>()});
            return ags::pair_report_csv(r);
        },
        py::arg("rows"));

    py::class_<Renderer>(m, "Renderer")
        .def(py::init<int>(), py::arg("device") = 0)
        .def("render", &Renderer::render, py::arg("scene"), py::arg("view") = 0, py::arg("mode") = "ellipse",
             py::arg("k") = 0.0, py::arg("lut_bins") = std::vector<float>{}, py::arg("lut_depth_min") = 0.0f,
             py::arg("lut_depth_max") = 100.0f, py::arg("threads") = 0, py::arg("tile_size") = 16,
             py::arg("exact") = false, py::arg("max_t") = false, py::arg("pair_budget") = std::size_t{1} << 27,
             py::arg("image") = true, py::arg("image_u8") = false)
        .def("render_async", &Renderer::render_async, py::arg("scene"), py::arg("view") = 0,
             py::arg("mode") = "ellipse", py::arg("k") = 0.0, py::arg("lut_bins") = std::vector<float>{},
             py::arg("lut_depth_min") = 0.0f, py::arg("lut_depth_max") = 100.0f, py::arg("tile_size") = 16,
             py::arg("exact") = false, py::arg("pair_budget") = std::size_t{1} << 27, py::arg("camera") = py::none())
        .def("render_async_to", &Renderer::render_async_to, py::arg("scene"), py::arg("view"), py::arg("target"),
             py::arg("mode") = "ellipse", py::arg("k") = 0.0, py::arg("lut_bins") = std::vector<float>{},
             py::arg("lut_depth_min") = 0.0f, py::arg("lut_depth_max") = 100.0f, py::arg("tile_size") = 16,
             py::arg("exact") = false, py::arg("pair_budget") = std::size_t{1} << 27,
             py::arg("camera") = py::none())
        .def("render_async_host", &Renderer::render_async_host, py::arg("scene"), py::arg("view") = 0,
             py::arg("mode") = "ellipse", py::arg("k") = 0.0, py::arg("lut_bins") = std::vector<float>{},
             py::arg("lut_depth_min") = 0.0f, py::arg("lut_depth_max") = 100.0f, py::arg("tile_size") = 16,
             py::arg("exact") = false, py::arg("pair_budget") = std::size_t{1} << 27, py::arg("camera") = py::none(),
             py::arg("image_u8") = false)
        .def("wait", &Renderer::wait)
        .def("pair_report", &Renderer::pair_report, py::arg("scene"), py::arg("specs"),
             py::arg("views") = std::vector<int>{}, py::arg("lut_bins") = std::vector<float>{},
             py::arg("lut_depth_min") = 0.0f, py::arg("lut_depth_max") = 100.0f, py::arg("threads") = 0)
        .def("fold_max_t", &Renderer::fold_max_t, py::arg("scene"), py::arg("views") = std::vector<int>{},
             py::arg("threads") = 0)
        .def("psnr_device", &Renderer::psnr_device, py::arg("a"), py::arg("b"), py::arg("n"))
        .def("calibrate", &Renderer::calibrate, py::arg("scene"), py::arg("target_drop"), py::arg("calib_views") = 16,
             py::arg("threads") = 0)
        .def("device_image", &Renderer::device_image)
        .def("stage_history", &Renderer::stage_history, py::arg("max_frames") = 64)
        .def("frame_stats", &Renderer::frame_stats)
        .def("dump_tile_counts", &Renderer::dump_tile_counts, py::arg("n"))
        .def("dump_sorted_pairs", &Renderer::dump_sorted_pairs)
        .def("dump_ranges", &Renderer::dump_ranges, py::arg("tile_count"))
        .def("upload", [](Renderer& r, Scene& s) { r.device_scene(s); })
        .def_property_readonly("stream", &Renderer::stream)
        .def_property_readonly("kernel_launches", &Renderer::kernel_launches)
        .def_property_readonly("device", &Renderer::device);

    m.def("default_renderer", &default_renderer, py::return_value_policy::reference);
    m.attr("SPLAT_ITEMSIZE") = static_cast<int>(sizeof(agsx_splat_view));
    (void)&splats_to_numpy;
}

// ags_calibrate.cpp -- GPU calibration of the AdaGScale parameters (next row
// f1): the T_upper LUT from max-transmittance renders and
// the binary search for K against a PSNR-drop budget.
//
//   reference: build_lut        calibrate.cpp:14-41
//              search_k          calibrate.cpp:93-155
//              mean_psnr_drop    calibrate.cpp:76-91
//              psnr / capped     analysis.cpp:14-29
//
// The control flow (views, doubling, 20 bisection steps, the K = 0 identity
// check) is the reference's.  Every render runs on the GPU with the
// glibc-exact alpha, so frames are bit-identical to the reference's; the
// lossless reference frames stay in HBM and each PSNR numerator is one device
// reduction, so a drop evaluation never copies an image to the host.  The
// squared-error sum is a fixed-order tree instead of the reference's serial
// loop, which can move a drop only in its last bits.
#include <algorithm>
#include <cmath>
#include <limits>
#include <stdexcept>
#include <vector>

#include "ags_internal.hpp"

namespace ags {
namespace detail {

namespace {

// Device frame owned for the duration of a calibration.
struct DevFrame {
    agsx_ctx* ctx = nullptr;
    float* p = nullptr;
    std::uint64_t n = 0;  // floats
    DevFrame(agsx_ctx* c, std::uint64_t floats) : ctx(c), n(floats) {
        void* q = nullptr;
        check(agsx_device_alloc(ctx, floats * sizeof(float), &q), ctx);
        p = static_cast<float*>(q);
    }
    ~DevFrame() { agsx_device_free(ctx, p); }
    DevFrame(const DevFrame&) = delete;
    DevFrame& operator=(const DevFrame&) = delete;
};

void render_into(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera& cam, const agsx_config& cfg,
                 const agsx_lut* lut, float* target) {
    check(agsx_render_async_to(ctx, scene, &cam, &cfg, lut, target), ctx);
    agsx_frame f{};
    check(agsx_render_wait(ctx, &f), ctx);
}

// psnr_capped (analysis.cpp:14-29) from a device squared-error sum.
double capped_psnr(double se, std::uint64_t n) {
    if (se == 0.0) return kPsnrCap;
    const double mse = se / static_cast<double>(n);
    return std::min(10.0 * std::log10(1.0 / mse), kPsnrCap);
}

}  // namespace

TUpperLUT build_lut_device(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* views, int n_views,
                           const agsx_config& cfg) {
    TUpperLUT lut;
    std::vector<std::uint8_t> observed(lut.bins.size(), 0);
    std::vector<float> folded(lut.bins.size(), 0.0f);
    const agsx_lut shape{lut.depth_min, lut.depth_max, static_cast<int32_t>(lut.bins.size()), nullptr};
    for (int v = 0; v < n_views; ++v)
        check(agsx_fold_max_t(ctx, scene, &views[v], &cfg, &shape, folded.data(), observed.data()), ctx);
    for (std::size_t b = 0; b < lut.bins.size(); ++b)
        if (observed[b]) lut.bins[b] = folded[b];
    return lut;
}

CalibrationResult search_k_device(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* views, int n_views,
                                  double target_drop, const agsx_config& cfg, const TUpperLUT& lut,
                                  bool worst_case) {
    if (n_views < 1) throw std::invalid_argument("search_k: no calibration views");
    CalibrationResult result;
    result.lut = lut;
    result.target_drop = target_drop;
    for (int v = 0; v < n_views; ++v) result.calib_view_ids.push_back(v);
    if (target_drop <= 0.0) return result;  // K = 0 is exactly lossless

    agsx_config lossless = cfg;
    lossless.mode = AGSX_MODE_ELLIPSE;
    lossless.flags |= AGSX_FLAG_EXACT_ALPHA;
    std::vector<std::unique_ptr<DevFrame>> refs;
    std::uint64_t max_n = 0;
    for (int v = 0; v < n_views; ++v) {
        const std::uint64_t n = static_cast<std::uint64_t>(views[v].width) * views[v].height * 3;
        refs.push_back(std::make_unique<DevFrame>(ctx, n));
        render_into(ctx, scene, views[v], lossless, nullptr, refs.back()->p);
        max_n = std::max(max_n, n);
    }
    DevFrame scratch(ctx, max_n);
    const agsx_lut l = to_c(lut);

    auto drop_at = [&](double k) {  // mean_psnr_drop, calibrate.cpp:76-91
        ++result.iterations;
        agsx_config adaptive = cfg;
        adaptive.mode = AGSX_MODE_ADAGSCALE;
        adaptive.k = static_cast<float>(k);
        adaptive.flags |= AGSX_FLAG_EXACT_ALPHA;
        double acc = 0.0;
        for (int v = 0; v < n_views; ++v) {
            render_into(ctx, scene, views[v], adaptive, &l, scratch.p);
            double se = 0.0;
            check(agsx_sq_err(ctx, scratch.p, refs[v]->p, refs[v]->n, &se), ctx);
            const double drop = kPsnrCap - capped_psnr(se, refs[v]->n);
            acc = worst_case ? std::max(acc, drop) : acc + drop;
        }
        return worst_case ? acc : acc / static_cast<double>(n_views);
    };

    if (drop_at(0.0) != 0.0)
        throw std::logic_error("search_k: K=0 render differs from the lossless reference");

    double k_lo = 0.0, k_hi = 1.0, best_drop = 0.0;
    bool bounded = false;
    for (int d = 0; d < 40; ++d) {
        const double drop = drop_at(k_hi);
        if (drop > target_drop) {
            bounded = true;
            break;
        }
        k_lo = k_hi;
        best_drop = drop;
        k_hi *= 2.0;
    }
    if (bounded) {
        for (int step = 0; step < 20; ++step) {
            const double mid = 0.5 * (k_lo + k_hi);
            const double drop = drop_at(mid);
            if (drop <= target_drop) {
                k_lo = mid;
                best_drop = drop;
            } else {
                k_hi = mid;
            }
        }
    }
    result.k = k_lo;
    result.achieved_drop = best_drop;
    return result;
}

}  // namespace detail

double psnr_capped(const Image& a, const Image& b) { return std::min(psnr(a, b), kPsnrCap); }

double peripheral_score_closed(const SymMat2& cov2d, float x, float t_const, float tau) {
    const float det = cov2d.xx * cov2d.yy - cov2d.xy * cov2d.xy;
    return static_cast<double>(t_const) * 2.0 * 3.14159265358979323846 * std::sqrt(static_cast<double>(det)) *
           (static_cast<double>(x) - static_cast<double>(tau));
}

namespace {
std::vector<agsx_camera> to_c_views(std::span<const Camera> views) {
    std::vector<agsx_camera> out;
    out.reserve(views.size());
    for (const Camera& c : views) {
        if (const std::string bad = validate(c); !bad.empty()) throw std::invalid_argument("calibration: " + bad);
        out.push_back(detail::to_c(c));
    }
    return out;
}
}  // namespace

TUpperLUT build_lut(const DeviceScene& scene, std::span<const Camera> calib_views, const RenderConfig& cfg) {
    const auto v = to_c_views(calib_views);
    return detail::build_lut_device(detail::thread_ctx(), static_cast<const agsx_scene*>(scene.handle()), v.data(),
                                    static_cast<int>(v.size()), detail::to_c(cfg));
}

TUpperLUT build_lut(std::span<const Gaussian3D> scene, std::span<const Camera> calib_views,
                    const RenderConfig& cfg) {
    const DeviceScene dev(scene);
    return build_lut(dev, calib_views, cfg);
}

CalibrationResult search_k(const DeviceScene& scene, std::span<const Camera> calib_views, double target_drop,
                           const RenderConfig& cfg, const TUpperLUT& lut, bool worst_case) {
    const auto v = to_c_views(calib_views);
    return detail::search_k_device(detail::thread_ctx(), static_cast<const agsx_scene*>(scene.handle()), v.data(),
                                   static_cast<int>(v.size()), target_drop, detail::to_c(cfg), lut, worst_case);
}

CalibrationResult search_k(std::span<const Gaussian3D> scene, std::span<const Camera> calib_views,
                           double target_drop, const RenderConfig& cfg, const TUpperLUT& lut, bool worst_case) {
    const DeviceScene dev(scene);
    return search_k(dev, calib_views, target_drop, cfg, lut, worst_case);
}

}  // namespace ags

// ags_report.cpp -- the pair-reduction report (next row f4, the paper's
// Table IV methodology) over the device render path.
//
//   reference: pair_report      analysis.cpp:259-312
//              pair_report_csv  analysis.cpp:346-371
//              format_double    analysis.cpp:314-318
//
// Same control flow and row definitions as the reference; every frame is a
// glibc-exact device render (bit-identical to the reference's images), the
// lossless reference frames stay in HBM and each PSNR numerator is one device
// reduction (a fixed tree order instead of the reference's serial sum).
#include <charconv>
#include <cmath>
#include <memory>

#include "ags_internal.hpp"

namespace ags {
namespace detail {

std::vector<PairReportRow> pair_report_device(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* views,
                                              int n_views, std::span<const ReportSpec> specs,
                                              const agsx_config& cfg, const TUpperLUT* lut) {
    agsx_config lossless = cfg;
    lossless.mode = AGSX_MODE_ELLIPSE;
    lossless.flags |= AGSX_FLAG_EXACT_ALPHA;
    TUpperLUT built;
    bool needs_lut = false;
    for (const ReportSpec& s : specs) needs_lut = needs_lut || s.mode == Mode::AdaGScale;
    if (needs_lut && lut == nullptr) {
        built = build_lut_device(ctx, scene, views, n_views, lossless);
        lut = &built;
    }
    struct Frame {
        agsx_ctx* ctx;
        float* p = nullptr;
        std::uint64_t n;
        Frame(agsx_ctx* c, std::uint64_t floats) : ctx(c), n(floats) {
            void* q = nullptr;
            check(agsx_device_alloc(ctx, floats * sizeof(float), &q), ctx);
            p = static_cast<float*>(q);
        }
        ~Frame() { agsx_device_free(ctx, p); }
    };
    auto render_into = [&](const agsx_camera& cam, const agsx_config& c, const agsx_lut* l, float* target) {
        check(agsx_render_async_to(ctx, scene, &cam, &c, l, target), ctx);
        agsx_frame f{};
        check(agsx_render_wait(ctx, &f), ctx);
        return f;
    };
    std::vector<std::unique_ptr<Frame>> refs;
    std::vector<std::uint64_t> ref_pairs;
    std::uint64_t max_n = 1;
    for (int v = 0; v < n_views; ++v) {
        const std::uint64_t n = static_cast<std::uint64_t>(views[v].width) * views[v].height * 3;
        refs.push_back(std::make_unique<Frame>(ctx, n));
        ref_pairs.push_back(render_into(views[v], lossless, nullptr, refs.back()->p).pair_count);
        max_n = std::max(max_n, n);
    }
    Frame scratch(ctx, max_n);
    agsx_lut l{};
    if (lut) l = to_c(*lut);

    std::vector<PairReportRow> rows;
    for (const ReportSpec& spec : specs) {
        agsx_config run = cfg;
        run.mode = static_cast<int32_t>(spec.mode);
        run.k = static_cast<float>(spec.k);
        run.flags |= AGSX_FLAG_EXACT_ALPHA;
        PairReportRow row{};
        row.mode = mode_name(spec.mode);
        row.k = spec.mode == Mode::AdaGScale ? spec.k : 0.0;
        double reduction = 0.0, drop = 0.0;
        for (int v = 0; v < n_views; ++v) {
            const agsx_frame f =
                render_into(views[v], run, spec.mode == Mode::AdaGScale ? &l : nullptr, scratch.p);
            row.pair_count += f.pair_count;
            reduction += 100.0 * (1.0 - static_cast<double>(f.pair_count) / static_cast<double>(ref_pairs[v]));
            double se = 0.0;
            check(agsx_sq_err(ctx, scratch.p, refs[v]->p, refs[v]->n, &se), ctx);
            const double p = se == 0.0 ? kPsnrCap
                                       : std::min(10.0 * std::log10(1.0 / (se / static_cast<double>(refs[v]->n))),
                                                  kPsnrCap);
            drop += kPsnrCap - p;
            row.t_preprocess += f.stage_ms[0] * 1e-3;
            row.t_pair_gen += f.stage_ms[1] * 1e-3;
            row.t_sort += f.stage_ms[2] * 1e-3;
            row.t_raster += f.stage_ms[3] * 1e-3;
        }
        row.reduction_pct = reduction / static_cast<double>(n_views);
        row.psnr_drop_db = drop / static_cast<double>(n_views);
        rows.push_back(std::move(row));
    }
    return rows;
}

}  // namespace detail

std::vector<PairReportRow> pair_report(const DeviceScene& scene, std::span<const Camera> views,
                                       std::span<const ReportSpec> specs, const RenderConfig& cfg,
                                       const TUpperLUT* lut) {
    std::vector<agsx_camera> v;
    for (const Camera& c : views) v.push_back(detail::to_c(c));
    return detail::pair_report_device(detail::thread_ctx(), static_cast<const agsx_scene*>(scene.handle()), v.data(),
                                      static_cast<int>(v.size()), specs, detail::to_c(cfg), lut);
}

std::vector<PairReportRow> pair_report(std::span<const Gaussian3D> scene, std::span<const Camera> views,
                                       std::span<const ReportSpec> specs, const RenderConfig& cfg,
                                       const TUpperLUT* lut) {
    const DeviceScene dev(scene);
    return pair_report(dev, views, specs, cfg, lut);
}

std::string format_double(double v) {
    char buf[64];
    const auto res = std::to_chars(buf, buf + sizeof(buf), v);
    return std::string(buf, res.ptr);
}

std::string pair_report_csv(std::span<const PairReportRow> rows) {
    std::string out = "mode,k,pair_count,reduction_vs_ellipse_pct,psnr_drop_db,preprocess_s,pair_gen_s,sort_s,raster_s\n";
    for (const auto& r : rows) {
        out += r.mode + ',' + format_double(r.k) + ',' + std::to_string(r.pair_count) + ',' +
               format_double(r.reduction_pct) + ',' + format_double(r.psnr_drop_db) + ',' +
               format_double(r.t_preprocess) + ',' + format_double(r.t_pair_gen) + ',' + format_double(r.t_sort) +
               ',' + format_double(r.t_raster) + '\n';
    }
    return out;
}

}  // namespace ags

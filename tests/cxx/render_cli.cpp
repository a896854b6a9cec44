// render_cli.cpp -- a reference-style C++ caller of the drop-in API
// (include/ags/ags.hpp), compiled against libags.so exactly as the
// reference's CLI / calibration / analysis callers would be
// (adagscale_main.cpp:224-226, calibrate.cpp:29).
//
//   render_cli <seed> <count> <layout> <w> <h> <focal> <view> <mode> <k> <out.f32> [lut_bin]
//
// Renders one view through ags::render(std::span<const Gaussian3D>, ...) and
// through ags::DeviceScene, writes the image (raw f32 HWC) and prints one JSON
// line; then checks the reference's exception contract.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>

#include "ags/ags.hpp"

int main(int argc, char** argv) {
    if (argc < 11) {
        std::fprintf(stderr, "usage: render_cli seed count layout w h focal view mode k out.f32 [lut_bin]\n");
        return 2;
    }
    ags::SynthSpec spec;
    spec.layout = argv[3];
    spec.camera_count = std::atoi(argv[7]) + 1;
    spec.width = std::atoi(argv[4]);
    spec.height = std::atoi(argv[5]);
    spec.fx = spec.fy = static_cast<float>(std::atof(argv[6]));
    const ags::SynthScene s = ags::synth_scene(std::strtoull(argv[1], nullptr, 10), std::atoi(argv[2]), spec);
    const ags::Camera& cam = s.cameras.at(std::atoi(argv[7]));
    ags::RenderConfig cfg;
    if (!ags::parse_mode(argv[8], cfg.mode)) return 2;
    cfg.k = static_cast<float>(std::atof(argv[9]));
    ags::TUpperLUT lut;
    if (argc > 11) lut.bins.assign(20, static_cast<float>(std::atof(argv[11])));
    const ags::TUpperLUT* lp = cfg.mode == ags::Mode::AdaGScale ? &lut : nullptr;

    const ags::RenderReport rep = ags::render(s.gaussians, cam, cfg, lp);  // the reference's signature
    const ags::DeviceScene dev(s.gaussians);
    const ags::RenderReport rep2 = ags::render(dev, cam, cfg, lp);
    const bool same = rep.pair_count == rep2.pair_count && rep.image.data == rep2.image.data;
    // the span's device copy is cached across calls: an in-place edit of ANY
    // Gaussian must show in the next render(span) (the reference re-reads the
    // span every call) -- every Gaussian is hidden here, then restored
    std::vector<ags::Gaussian3D> edited = s.gaussians;
    (void)ags::render(edited, cam, cfg, lp);  // cached
    for (auto& g : edited) g.opacity = 0.0f;  // nothing survives the culls
    const ags::RenderReport rep_hidden = ags::render(edited, cam, cfg, lp);
    edited[edited.size() / 2 + 1].opacity = s.gaussians[edited.size() / 2 + 1].opacity;
    const ags::RenderReport rep_one = ags::render(edited, cam, cfg, lp);  // one Gaussian back
    edited = s.gaussians;
    const ags::RenderReport rep_back = ags::render(edited, cam, cfg, lp);
    const bool cache_ok = rep_hidden.splat_count == 0 && rep_one.splat_count <= 1 &&
                          rep_back.pair_count == rep.pair_count && rep_back.image.data == rep.image.data;
    std::ofstream(argv[10], std::ios::binary)
        .write(reinterpret_cast<const char*>(rep.image.data.data()),
               static_cast<std::streamsize>(rep.image.data.size() * sizeof(float)));

    // analysis.cpp:171-173: max_t and the blend-event stream in one render
    ags::RecordOptions rec;
    rec.max_t = true;
    rec.contributions = true;
    const ags::RenderReport rep3 = ags::render(dev, cam, cfg, lp, rec);
    std::ofstream(std::string(argv[10]) + ".contrib", std::ios::binary)
        .write(reinterpret_cast<const char*>(rep3.contributions.data()),
               static_cast<std::streamsize>(rep3.contributions.size() * sizeof(ags::BlendRecord)));
    std::ofstream(std::string(argv[10]) + ".maxt", std::ios::binary)
        .write(reinterpret_cast<const char*>(rep3.max_t.data()),
               static_cast<std::streamsize>(rep3.max_t.size() * sizeof(float)));

    // exception contract (rasterizer.cpp:105-108, preprocess.cpp:123-125, pair_gen.cpp:181-184)
    int errors_ok = 0;
    try {
        ags::RenderConfig bad = cfg;
        bad.alpha_threshold = -1.0f;
        (void)ags::render(dev, cam, bad, lp);
    } catch (const std::invalid_argument&) {
        ++errors_ok;
    }
    try {
        ags::RenderConfig ada = cfg;
        ada.mode = ags::Mode::AdaGScale;
        (void)ags::render(dev, cam, ada, nullptr);
    } catch (const std::invalid_argument&) {
        ++errors_ok;
    }
    try {
        ags::RenderConfig tight = cfg;
        tight.pair_budget = rep.pair_count > 0 ? rep.pair_count - 1 : 0;
        (void)ags::render(dev, cam, tight, lp);
    } catch (const ags::PairBudgetError&) {
        ++errors_ok;
    }
    std::printf("{\"pair_count\": %zu, \"splat_count\": %zu, \"device_scene_same\": %s, \"errors_ok\": %d, "
                "\"stage_keys\": %zu, \"contributions\": %zu, \"cache_follows_edits\": %s}\n",
                rep.pair_count, rep.splat_count, same ? "true" : "false", errors_ok, rep.stage_times.size(),
                rep3.contributions.size(), cache_ok ? "true" : "false");
    return 0;
}

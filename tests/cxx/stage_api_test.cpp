// stage_api_test.cpp -- the reference's unit cases for the per-element stage
// functions, restated against the drop-in C++ API (include/ags/ags.hpp) and
// run on the GPU through libags.so / libagsx.so:
//   test_pair_gen.cpp:39-114     effective_radius, intersect_tiles per mode
//   test_rasterizer.cpp:50-117   alpha_at, raster_tile, tile-order invariance
//   test_preprocess.cpp:35-140   project, eval_color, compute_th
//   test_scene_model.cpp:39-108  covariance_3d, rotation_matrix
// plus exactness checks of the device helpers against the header inlines
// (alpha_at, eigen_sym2) and the host math (glibc logf / expf).
// Prints "stage_api ok <checks>" and exits 0 when every check holds.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <set>
#include <stdexcept>
#include <vector>

#include "agsx.h"
#include "ags/ags.hpp"

using namespace ags;

namespace {
int g_checks = 0, g_fail = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        ++g_checks;                                                           \
        if (!(c)) {                                                           \
            ++g_fail;                                                         \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
        }                                                                     \
    } while (0)
bool approx(double a, double b, double eps) { return std::abs(a - b) <= eps * std::max(std::abs(a), std::abs(b)); }
std::uint32_t bits(float f) {
    std::uint32_t u;
    std::memcpy(&u, &f, 4);
    return u;
}

SplatView make_splat(Vec2f mean, SymMat2 cov, float opacity, float th) {
    SplatView s{};
    s.mean2d = mean;
    s.cov2d = cov;
    s.inv_cov = cov.inverse();
    s.depth = 5.0f;
    s.rgb = {1, 1, 1};
    s.opacity = opacity;
    s.th = th;
    s.source_id = 0;
    return s;
}

SplatView flat_splat(Vec2f mean, float sigma_px, float opacity, Vec3f rgb, float depth) {
    SplatView s{};
    s.mean2d = mean;
    s.cov2d = {sigma_px * sigma_px, 0, sigma_px * sigma_px};
    s.inv_cov = s.cov2d.inverse();
    s.depth = depth;
    s.rgb = rgb;
    s.opacity = opacity;
    s.th = 1.0f / 255.0f;
    s.source_id = 0;
    return s;
}

std::vector<int> tiles_of(const SplatView& s, const TileGrid& g, Mode m, const RenderConfig& cfg) {
    std::vector<int> out;
    intersect_tiles(s, g, m, cfg, out);
    return out;
}

// generate_pairs -> sort_pairs -> raster_tile per tile (test_rasterizer.cpp:27-41)
Image raster_all(const std::vector<SplatView>& splats, int w, int h, const RenderConfig& cfg, bool reverse) {
    const TileGrid grid = TileGrid::make(w, h, cfg.tile_size);
    auto gen = generate_pairs(splats, grid, cfg.mode, cfg);
    const SortedPairs sorted = sort_pairs(std::move(gen.pairs), grid.tile_count());
    Image img(w, h);
    for (int i = 0; i < grid.tile_count(); ++i) {
        const int tile = reverse ? grid.tile_count() - 1 - i : i;
        const auto [b, e] = sorted.ranges[tile];
        raster_tile({sorted.pairs.data() + b, e - b}, splats, grid, tile, cfg, img, nullptr, nullptr);
    }
    return img;
}

Camera front_camera(float fx = 500.0f, int w = 640, int h = 480) {
    Camera cam;
    cam.fx = cam.fy = fx;
    cam.width = w;
    cam.height = h;
    return cam;
}

Gaussian3D on_axis(float depth, float scale, float opacity = 0.8f) {
    Gaussian3D g;
    g.mean = {0, 0, depth};
    g.scale = {scale, scale, scale};
    g.opacity = opacity;
    return g;
}
}  // namespace

int main() {
    const float tau = 1.0f / 255.0f;
    // ---- pair_gen (test_pair_gen.cpp:39-114) ----------------------------
    {
        const SymMat2 cov{1, 0, 1};
        CHECK(approx(effective_radius(1.0f, tau, cov).mahalanobis, 3.3290, 1e-3));
        CHECK(approx(effective_radius(0.5f, 0.013922f, cov).mahalanobis, 2.676, 1e-3));
        const float r = effective_radius(0.5f, 0.4999995f, cov).mahalanobis;
        CHECK(r > 0.0f && r < 0.01f);
        CHECK(approx(effective_radius(1.0f, tau, {4, 0, 1}).pixels, 2.0 * 3.3290, 1e-3));
        // the device radius is the host glibc expression bit for bit
        for (float op : {0.3f, 0.77f, 0.99f})
            for (float th : {tau, 0.01f, 0.2f}) {
                const SymMat2 c{9.5f, 1.25f, 3.0f};
                const EffectiveRadius e = effective_radius(op, th, c);
                const float m = std::sqrt(2.0f * std::log(op / th));
                CHECK(bits(e.mahalanobis) == bits(m));
                CHECK(bits(e.pixels) == bits(m * std::sqrt(std::max(eigen_sym2(c).l1, 0.0f))));
            }
    }
    {
        const TileGrid grid = TileGrid::make(64, 64, 16);
        const RenderConfig cfg;
        const SplatView s = make_splat({24, 24}, {4, 0, 4}, 0.99f, cfg.alpha_threshold);
        for (Mode m : {Mode::AABB, Mode::OBB, Mode::Ellipse, Mode::AdaGScale}) {
            const auto t = tiles_of(s, grid, m, cfg);
            CHECK(t.size() == 1 && t[0] == 1 * grid.tiles_x + 1);
        }
    }
    {
        const TileGrid grid = TileGrid::make(640, 480, 16);
        const RenderConfig cfg;
        const SplatView s = make_splat({320, 240}, {455.0f, 450.0f, 455.0f}, 0.9f, cfg.alpha_threshold);
        const auto aabb = tiles_of(s, grid, Mode::AABB, cfg);
        const auto obb = tiles_of(s, grid, Mode::OBB, cfg);
        const auto ell = tiles_of(s, grid, Mode::Ellipse, cfg);
        CHECK(obb.size() < aabb.size());
        CHECK(ell.size() <= obb.size());
        const std::set<int> os(obb.begin(), obb.end()), es(ell.begin(), ell.end());
        bool covered = true;
        for (int py = 0; py < grid.height; ++py)
            for (int px = 0; px < grid.width; ++px) {
                if (alpha_at(s, {px + 0.5f, py + 0.5f}, cfg.alpha_clamp) < cfg.alpha_threshold) continue;
                const int t = (py / grid.tile_size) * grid.tiles_x + (px / grid.tile_size);
                covered = covered && os.count(t) == 1 && es.count(t) == 1;
            }
        CHECK(covered);
    }
    {
        const TileGrid grid = TileGrid::make(640, 480, 16);
        const RenderConfig cfg;
        const SplatView s = make_splat({100, 100}, {120, 30, 60}, 0.8f, cfg.alpha_threshold);
        CHECK(tiles_of(s, grid, Mode::AdaGScale, cfg) == tiles_of(s, grid, Mode::Ellipse, cfg));
        const SplatView big = make_splat({320, 240}, {400, 0, 400}, 0.9f, 0.02f);
        const auto ada = tiles_of(big, grid, Mode::AdaGScale, cfg);
        const auto ell = tiles_of(big, grid, Mode::Ellipse, cfg);
        CHECK(ada.size() < ell.size());
        const std::set<int> es(ell.begin(), ell.end());
        bool subset = true;
        for (int t : ada) subset = subset && es.count(t) == 1;
        CHECK(subset);
    }
    // ---- rasterizer (test_rasterizer.cpp:50-117) --------------------------
    {
        SplatView s = flat_splat({10, 10}, 2.0f, 0.8f, {1, 1, 1}, 1.0f);
        CHECK(approx(alpha_at(s, {10, 10}, 0.99f), 0.8, 1e-6));
        CHECK(approx(alpha_at(s, {12, 10}, 0.99f), 0.8 * std::exp(-0.5), 1e-5));
        s.opacity = 1.0f;
        CHECK(alpha_at(s, {10, 10}, 0.99f) == 0.99f);
        // the device alpha (glibc expf on the GPU) equals the header inline bit for bit
        agsx_ctx* ctx = nullptr;
        const bool have_ctx = agsx_create(0, &ctx) == AGSX_OK;
        CHECK(have_ctx);
        if (have_ctx) {
            std::vector<agsx_splat_view> sv;
            std::vector<float> px, dev;
            std::vector<float> host;
            Rng rng(7);
            for (int i = 0; i < 4096; ++i) {
                const SplatView v = make_splat({rng.uniform(0, 64), rng.uniform(0, 64)},
                                               {rng.uniform(1, 40), rng.uniform(-0.5f, 0.5f), rng.uniform(1, 40)},
                                               rng.uniform(0.01f, 1.0f), tau);
                agsx_splat_view c;
                std::memcpy(&c, &v, sizeof(c));
                sv.push_back(c);
                const Vec2f p{rng.uniform(0, 64) + 0.5f, rng.uniform(0, 64) + 0.5f};
                px.push_back(p.x);
                px.push_back(p.y);
                host.push_back(alpha_at(v, p, 0.99f));
            }
            dev.resize(host.size());
            CHECK(agsx_alpha_at(ctx, sv.data(), px.data(), sv.size(), 0.99f, dev.data()) == AGSX_OK);
            bool same = true;
            for (std::size_t i = 0; i < host.size(); ++i) same = same && bits(host[i]) == bits(dev[i]);
            CHECK(same);
            agsx_destroy(ctx);
        }
    }
    {
        RenderConfig cfg;
        const auto img = raster_all({flat_splat({8, 8}, 1e4f, 0.5f, {1, 1, 1}, 1.0f)}, 16, 16, cfg, false);
        CHECK(approx(img.at(8, 8, 0), 0.5, 1e-4));
        CHECK(approx(img.at(3, 12, 1), 0.5, 1e-4));
    }
    {
        RenderConfig cfg;
        cfg.background = {1, 1, 1};
        const std::vector<SplatView> sp{flat_splat({8, 8}, 1e4f, 0.5f, {1, 1, 1}, 1.0f),
                                        flat_splat({8, 8}, 1e4f, 0.5f, {0, 0, 0}, 2.0f)};
        CHECK(approx(raster_all(sp, 16, 16, cfg, false).at(8, 8, 0), 0.75, 1e-4));
    }
    {
        RenderConfig cfg;
        cfg.background = {0.25f, 0.5f, 0.75f};
        const auto img = raster_all({flat_splat({8, 8}, 1e4f, 0.001f, {1, 1, 1}, 1.0f)}, 16, 16, cfg, false);
        CHECK(img.at(8, 8, 0) == 0.25f && img.at(8, 8, 1) == 0.5f && img.at(8, 8, 2) == 0.75f);
    }
    {
        RenderConfig cfg;
        cfg.background = {0.1f, 0.2f, 0.3f};
        const std::vector<Gaussian3D> empty;
        Camera cam;
        cam.fx = cam.fy = 100;
        cam.width = 64;
        cam.height = 48;
        const RenderReport rep = render(empty, cam, cfg);
        CHECK(rep.pair_count == 0 && rep.splat_count == 0);
        CHECK(rep.image.at(10, 10, 0) == 0.1f && rep.image.at(63, 47, 2) == 0.3f);
    }
    {
        // tile order cannot change the image, and raster_tile per tile equals
        // the whole-frame render of the same view
        ::setenv("AGS_EXACT_ALPHA", "1", 1);  // glibc-exact alpha on every path of this block
        const SynthScene scene = synth_scene(31, 600, SynthSpec{});
        RenderConfig cfg;
        const auto splats = preprocess_view(scene.gaussians, scene.cameras[2], cfg);
        const Image fwd = raster_all(splats, 640, 480, cfg, false);
        const Image rev = raster_all(splats, 640, 480, cfg, true);
        CHECK(fwd.data == rev.data);
        const RenderReport whole = render(scene.gaussians, scene.cameras[2], cfg);
        ::unsetenv("AGS_EXACT_ALPHA");
        CHECK(whole.image.data == fwd.data);
        std::vector<float> mt;
        std::vector<BlendRecord> rec;
        const TileGrid grid = TileGrid::make(640, 480, 16);
        Image one(640, 480);
        bool threw = false;
        try {
            raster_tile({}, splats, grid, 0, cfg, one, &mt, &rec);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
    }
    // ---- preprocess (test_preprocess.cpp:35-140) ---------------------------
    {
        const auto p = project(on_axis(10.0f, 0.1f), front_camera(), RenderConfig{});
        CHECK(p.has_value() && approx(p->mean2d.x, 320.0, 1e-6) && approx(p->mean2d.y, 240.0, 1e-6) &&
              approx(p->depth, 10.0, 1e-6));
        const float f = 500.0f, s = 0.2f, d = 12.0f;
        const auto q = project(on_axis(d, s), front_camera(f), RenderConfig{});
        const double expect = std::pow(double(f) * s / d, 2) + 0.3;
        CHECK(q.has_value() && approx(q->cov2d.xx, expect, 1e-4) && approx(q->cov2d.yy, expect, 1e-4) &&
              std::abs(q->cov2d.xy) < 1e-4);
        const Camera cam = front_camera();
        const RenderConfig cfg;
        CHECK(!project(on_axis(0.1f, 0.05f), cam, cfg).has_value());
        CHECK(project(on_axis(0.3f, 0.05f), cam, cfg).has_value());
        Gaussian3D fl = on_axis(10.0f, 0.05f);
        fl.mean.x = -10.0f;
        CHECK(!project(fl, cam, cfg).has_value());
        fl.mean.x = -8.0f;
        CHECK(project(fl, cam, cfg).has_value());
        // project equals the splat preprocess_view reports for the same Gaussian
        const SynthScene sc = synth_scene(9, 64, SynthSpec{});
        const auto sv = preprocess_view(sc.gaussians, sc.cameras[0], cfg);
        bool same = !sv.empty();
        for (const SplatView& v : sv) {
            const auto pr = project(sc.gaussians[v.source_id], sc.cameras[0], cfg);
            same = same && pr && bits(pr->mean2d.x) == bits(v.mean2d.x) && bits(pr->mean2d.y) == bits(v.mean2d.y) &&
                   bits(pr->cov2d.xx) == bits(v.cov2d.xx) && bits(pr->cov2d.xy) == bits(v.cov2d.xy) &&
                   bits(pr->cov2d.yy) == bits(v.cov2d.yy) && bits(pr->depth) == bits(v.depth);
            const Vec3f dir = (sc.gaussians[v.source_id].mean - sc.cameras[0].position).normalized();
            const Vec3f rgb = eval_color(sc.gaussians[v.source_id], dir);
            same = same && bits(rgb.x) == bits(v.rgb.x) && bits(rgb.y) == bits(v.rgb.y) && bits(rgb.z) == bits(v.rgb.z);
        }
        CHECK(same);
    }
    {
        Gaussian3D g = on_axis(5, 0.1f);
        g.sh = {0, 0, 0};
        Vec3f c = eval_color(g, {0, 0, 1});
        CHECK(approx(c.x, 0.5, 1e-7) && approx(c.y, 0.5, 1e-7));
        const float c0 = 0.7f;
        g.sh = {c0, c0, c0};
        c = eval_color(g, {0, 0, 1});
        const double e = 0.2820947917738781 * c0 + 0.5;
        CHECK(approx(c.x, e, 1e-6) && approx(c.z, e, 1e-6));
        g.sh = {-10.0f, 0.0f, 10.0f};
        c = eval_color(g, {0, 0, 1});
        CHECK(c.x == 0.0f && c.z == 1.0f);
        Gaussian3D h = on_axis(5, 0.1f);
        h.sh.assign(48, 0.0f);
        h.sh[0] = 0.3f;
        h.sh[9] = 0.5f;
        CHECK(eval_color(h, {0, 0, 1}).x != eval_color(h, {1, 0, 0}).x);
        Gaussian3D dc = on_axis(5, 0.1f);
        dc.sh = {0.3f, 0.3f, 0.3f};
        CHECK(eval_color(dc, {0, 0, 1}).x == eval_color(dc, {1, 0, 0}).x);
    }
    {
        TUpperLUT lut;
        CHECK(compute_th({4, 0, 1}, 10.0f, lut, 0.0f, tau) == tau);
        lut.bins.assign(20, 0.5f);
        CHECK(approx(compute_th({2, 0, 2}, 10.0f, lut, 0.01f * 2.0f * 3.14159265358979f, tau), 0.013922, 1e-4));
        lut.bins.assign(20, 1.0f);
        const float th = compute_th({1, 0, 1}, 10.0f, lut, 2.0f * 3.14159265358979f, tau);
        CHECK(approx(th, 1.0 + 1.0 / 255.0, 1e-5) && th > 1.0f);
        bool threw = false;
        try {
            compute_th({1, 2, 1}, 10.0f, lut, 0.0f, tau);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
        TUpperLUT l2;
        l2.bins[1] = 0.25f;
        CHECK(compute_th({2, 0, 2}, 6.0f, l2, 0.5f, tau) == compute_th({4, 0, 1}, 9.0f, l2, 0.5f, tau));
    }
    // ---- scene math (test_scene_model.cpp:39-108) ----------------------------
    {
        Gaussian3D g;
        g.scale = {1, 1, 1};
        const Mat3d c = covariance_3d(g);
        CHECK(c(0, 0) == 1.0 && c(1, 1) == 1.0 && c(2, 2) == 1.0 && c(0, 1) == 0.0);
        g.scale = {2, 3, 4};
        const Mat3d a = covariance_3d(g);
        CHECK(approx(a(0, 0), 4.0, 1e-12) && approx(a(1, 1), 9.0, 1e-12) && approx(a(2, 2), 16.0, 1e-12));
        g.rotation = Quatf{0.9f, 0.1f, -0.3f, 0.2f}.normalized();
        const Mat3d r = g.rotation.rotation_matrix<double>();
        Mat3d d;
        d(0, 0) = 4;
        d(1, 1) = 9;
        d(2, 2) = 16;
        const Mat3d want = r * d * r.transposed();
        const Mat3d got = covariance_3d(g);
        bool close = true;
        for (int i = 0; i < 9; ++i) close = close && std::abs(got.m[i] - want.m[i]) < 1e-9;
        CHECK(close);
        const Mat3f rf = g.rotation.to_matrix();
        CHECK(orthonormality_drift(rf) < 1e-6f);
        const Mat3f cast = r.cast<float>();
        CHECK(cast.m == rf.m);
        Mat3f noisy = rf;
        noisy.m[1] += 1e-3f;
        CHECK(orthonormality_drift(orthonormalize(noisy)) <= 1e-6f);
        const Eigen2 e = eigen_sym2({5, 2, 1});
        CHECK(e.l1 >= e.l2 && approx(e.v1.dot(e.v1), 1.0, 1e-6) && std::abs(e.v1.dot(e.v2)) < 1e-6);
        const Camera cam = front_camera();
        const Vec2f pp = principal_point(cam);
        CHECK(pp.x == 320.0f && pp.y == 240.0f);
        const Vec3f t = to_camera(cam, {1, 2, 3});
        CHECK(t.x == 1.0f && t.y == 2.0f && t.z == 3.0f);
    }
    std::printf("stage_api %s %d/%d\n", g_fail ? "FAILED" : "ok", g_checks - g_fail, g_checks);
    return g_fail ? 1 : 0;
}

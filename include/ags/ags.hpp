// ags.hpp -- C++ drop-in API of the B200 renderer.
//
// Same namespace, type names, field layouts and function signatures as the
// reference headers under /root/reference/proj/include/adagscale/ for the
// render path, so a caller of the reference's ags::render() recompiles
// against this header unchanged:
//   math.hpp:9-214     Vec2f, Vec3f, Mat3<T>, SymMat2, Quatf, Rng
//   scene.hpp:15-80    Gaussian3D, Camera, Mode, RenderConfig, validate, ...
//   lut.hpp:11-26      TUpperLUT
//   image.hpp:9-23     Image
//   preprocess.hpp     SplatView, preprocess_view
//   pair_gen.hpp       TileGrid, pack_pair_key, GaussianTilePair,
//                      PairGenResult, generate_pairs, PairBudgetError
//   pair_sort.hpp      SortedPairs, sort_pairs
//   rasterizer.hpp     RecordOptions, RenderReport, raster_tile, render
//   synth.hpp          SynthSpec, SynthScene, synth_scene
//   analysis.hpp:19-22 psnr
// Below these signatures every stage runs on the GPU through libagsx.so
// (include/agsx.h); there is no CPU fallback.
#pragma once

#include <array>
#include <iosfwd>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace ags {

// ---------------------------------------------------------------- math
struct Vec2f {
    float x = 0.0f, y = 0.0f;
    Vec2f operator+(Vec2f o) const { return {x + o.x, y + o.y}; }
    Vec2f operator-(Vec2f o) const { return {x - o.x, y - o.y}; }
    Vec2f operator*(float s) const { return {x * s, y * s}; }
    float dot(Vec2f o) const { return x * o.x + y * o.y; }
};

struct Vec3f {
    float x = 0.0f, y = 0.0f, z = 0.0f;
    Vec3f operator+(Vec3f o) const { return {x + o.x, y + o.y, z + o.z}; }
    Vec3f operator-(Vec3f o) const { return {x - o.x, y - o.y, z - o.z}; }
    Vec3f operator*(float s) const { return {x * s, y * s, z * s}; }
    float dot(Vec3f o) const { return x * o.x + y * o.y + z * o.z; }
    float norm() const { return std::sqrt(dot(*this)); }
    Vec3f normalized() const {
        const float n = norm();
        if (n > 0.0f) return (*this) * (1.0f / n);
        return Vec3f{};
    }
    Vec3f cross(Vec3f o) const { return {y * o.z - z * o.y, z * o.x - x * o.z, x * o.y - y * o.x}; }
};

// Row-major 3x3.
template <typename T>
struct Mat3 {
    std::array<T, 9> m{1, 0, 0, 0, 1, 0, 0, 0, 1};
    T& operator()(int r, int c) { return m[r * 3 + c]; }
    T operator()(int r, int c) const { return m[r * 3 + c]; }
    Vec3f operator*(Vec3f v) const {
        Vec3f o;
        float* out[3] = {&o.x, &o.y, &o.z};
        for (int r = 0; r < 3; ++r)
            *out[r] = static_cast<float>(m[r * 3] * v.x + m[r * 3 + 1] * v.y + m[r * 3 + 2] * v.z);
        return o;
    }
    Mat3 operator*(const Mat3& o) const {
        Mat3 out;
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) {
                T s = 0;
                for (int k = 0; k < 3; ++k) s += (*this)(r, k) * o(k, c);
                out(r, c) = s;
            }
        return out;
    }
    Mat3 transposed() const {
        Mat3 out;
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) out(r, c) = (*this)(c, r);
        return out;
    }
    // element-wise conversion (math.hpp:66-71)
    template <typename U>
    Mat3<U> cast() const {
        Mat3<U> out;
        for (int i = 0; i < 9; ++i) out.m[i] = static_cast<U>(m[i]);
        return out;
    }
};
using Mat3f = Mat3<float>;
using Mat3d = Mat3<double>;

struct SymMat2 {
    float xx = 0.0f, xy = 0.0f, yy = 0.0f;
    float det() const { return xx * yy - xy * xy; }
    SymMat2 inverse() const {
        const float inv = 1.0f / det();
        return {yy * inv, -xy * inv, xx * inv};
    }
    float quad(Vec2f d) const { return xx * d.x * d.x + 2.0f * xy * d.x * d.y + yy * d.y * d.y; }
};

// Eigen pair of a symmetric 2x2 matrix (math.hpp:97-131): l1 >= l2, v1 the unit
// eigenvector of l1 (the larger-norm candidate of the two closed forms),
// v2 = v1 rotated by +90 degrees; axis-aligned vectors when xy == 0.  The
// device copy used by the tile tests is agsx::eigen_sym2 (same operations).
struct Eigen2 {
    float l1 = 0.0f;
    float l2 = 0.0f;
    Vec2f v1{1, 0};
    Vec2f v2{0, 1};
};

inline Eigen2 eigen_sym2(const SymMat2& m) {
    Eigen2 e;
    const float centre = 0.5f * (m.xx + m.yy);
    const float half = 0.5f * (m.xx - m.yy);
    const float rad = std::sqrt(half * half + m.xy * m.xy);
    e.l1 = centre + rad;
    e.l2 = centre - rad;
    if (m.xy == 0.0f) {
        const bool x_major = m.xx >= m.yy;
        e.v1 = x_major ? Vec2f{1, 0} : Vec2f{0, 1};
        e.v2 = x_major ? Vec2f{0, 1} : Vec2f{-1, 0};
        return e;
    }
    const Vec2f cand_a{e.l1 - m.yy, m.xy};
    const Vec2f cand_b{m.xy, e.l1 - m.xx};
    const Vec2f v = cand_a.dot(cand_a) >= cand_b.dot(cand_b) ? cand_a : cand_b;
    const float len = std::sqrt(v.dot(v));
    e.v1 = {v.x / len, v.y / len};
    e.v2 = {-e.v1.y, e.v1.x};
    return e;
}

struct Quatf {
    float w = 1.0f, x = 0.0f, y = 0.0f, z = 0.0f;
    float norm() const { return std::sqrt(w * w + x * x + y * y + z * z); }
    Quatf normalized() const {
        const float n = norm();
        return {w / n, x / n, y / n, z / n};
    }
    Mat3f to_matrix() const { return rotation_matrix<float>(); }
    // Rotation matrix with the quaternion renormalised in double
    // (math.hpp:143-164); the device EWA (K1) evaluates the same expressions.
    template <typename T>
    Mat3<T> rotation_matrix() const {
        const double len = std::sqrt(double(w) * w + double(x) * x + double(y) * y + double(z) * z);
        const double a = w / len, b = x / len, c = y / len, d = z / len;
        Mat3<double> r;
        r(0, 0) = 1 - 2 * (c * c + d * d);
        r(0, 1) = 2 * (b * c - a * d);
        r(0, 2) = 2 * (b * d + a * c);
        r(1, 0) = 2 * (b * c + a * d);
        r(1, 1) = 1 - 2 * (b * b + d * d);
        r(1, 2) = 2 * (c * d - a * b);
        r(2, 0) = 2 * (b * d - a * c);
        r(2, 1) = 2 * (c * d + a * b);
        r(2, 2) = 1 - 2 * (b * b + c * c);
        return r.template cast<T>();
    }
};

// PCG32 + Box-Muller, the generator all synthetic scenes are drawn from.
class Rng {
public:
    explicit Rng(std::uint64_t seed, std::uint64_t stream = 0);
    std::uint32_t next_u32();
    float uniform();
    float uniform(float lo, float hi) { return lo + (hi - lo) * uniform(); }
    float normal();

private:
    std::uint64_t state_ = 0, inc_ = 1;
    float spare_ = 0.0f;
    bool has_spare_ = false;
};

// --------------------------------------------------------------- scene
struct Gaussian3D {
    Vec3f mean;
    Vec3f scale;
    Quatf rotation;
    float opacity = 0.5f;
    std::vector<float> sh{0.0f, 0.0f, 0.0f};  // coefficient-major, 3*d^2
};

int sh_degree(const Gaussian3D& g);
std::string validate(const Gaussian3D& g);

// Sigma = (R diag(s)) (R diag(s))^T in double (scene.cpp:31-39).
Mat3d covariance_3d(const Gaussian3D& g);

struct Camera {
    Vec3f position;
    Mat3f rotation;  // world-to-camera
    float fx = 1.0f, fy = 1.0f;
    int width = 0, height = 0;
};

// world -> camera, float, left-to-right dot products (scene.hpp:41-43)
inline Vec3f to_camera(const Camera& cam, Vec3f world) { return cam.rotation * (world - cam.position); }
// the image centre (scene.hpp:46-49)
inline Vec2f principal_point(const Camera& cam) {
    return {0.5f * static_cast<float>(cam.width), 0.5f * static_cast<float>(cam.height)};
}

std::string validate(const Camera& cam);
float orthonormality_drift(const Mat3f& r);
// Nearest orthonormal matrix by the polar iteration X <- (X + X^-T) / 2
// (scene.cpp:84-92): at most 20 steps, stops at drift <= 1e-7.
Mat3f orthonormalize(Mat3f r);

enum class Mode { AABB, OBB, Ellipse, AdaGScale };
const char* mode_name(Mode m);
bool parse_mode(const std::string& name, Mode& out);

struct RenderConfig {
    int tile_size = 16;
    float alpha_threshold = 1.0f / 255.0f;
    float transmittance_floor = 1e-4f;
    float alpha_clamp = 0.99f;
    float near_plane = 0.2f;
    float guard_band = 1.3f;
    Mode mode = Mode::Ellipse;
    float k = 0.0f;
    int thread_count = 0;  // accepted; no device meaning
    Vec3f background{0.0f, 0.0f, 0.0f};
    bool fixed_radius_aabb = false;
    std::size_t pair_budget = std::size_t{1} << 27;
};
std::string validate(const RenderConfig& cfg);

struct TUpperLUT {
    float depth_min = 0.0f;
    float depth_max = 100.0f;
    std::vector<float> bins = std::vector<float>(20, 1.0f);
    int bin_index(float depth) const;
    float value_at(float depth) const { return bins[bin_index(depth)]; }
};

struct Image {
    int width = 0, height = 0;
    std::vector<float> data;
    Image() = default;
    Image(int w, int h) : width(w), height(h), data(std::size_t(w) * h * 3, 0.0f) {}
    float& at(int x, int y, int c) { return data[(std::size_t(y) * width + x) * 3 + c]; }
    float at(int x, int y, int c) const { return data[(std::size_t(y) * width + x) * 3 + c]; }
    std::size_t pixel_count() const { return std::size_t(width) * height; }
};

// ----------------------------------------------------------- pipeline
struct SplatView {
    Vec2f mean2d;
    SymMat2 cov2d;
    SymMat2 inv_cov;
    float depth;
    Vec3f rgb;
    float opacity;
    float th;
    std::uint32_t source_id;
};

struct TileGrid {
    int tile_size = 16;
    int width = 0, height = 0;
    int tiles_x = 0, tiles_y = 0;
    static TileGrid make(int width, int height, int tile_size) {
        TileGrid g;
        g.tile_size = tile_size;
        g.width = width;
        g.height = height;
        g.tiles_x = (width + tile_size - 1) / tile_size;
        g.tiles_y = (height + tile_size - 1) / tile_size;
        return g;
    }
    int tile_count() const { return tiles_x * tiles_y; }
};

inline std::uint64_t pack_pair_key(std::uint32_t tile, float depth) {
    std::uint32_t bits;
    std::memcpy(&bits, &depth, 4);
    return (static_cast<std::uint64_t>(tile) << 32) | bits;
}
inline std::uint32_t pair_key_tile(std::uint64_t key) { return static_cast<std::uint32_t>(key >> 32); }
inline float pair_key_depth(std::uint64_t key) {
    const std::uint32_t bits = static_cast<std::uint32_t>(key);
    float d;
    std::memcpy(&d, &bits, 4);
    return d;
}

struct GaussianTilePair {
    std::uint64_t key;
    std::uint32_t splat_index;
};

struct PairGenResult {
    std::vector<GaussianTilePair> pairs;
    std::vector<std::uint32_t> tile_counts;
};

struct PairBudgetError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct SortedPairs {
    std::vector<GaussianTilePair> pairs;
    std::vector<std::pair<std::uint32_t, std::uint32_t>> ranges;
};

struct BlendRecord {
    std::uint32_t pixel;
    std::uint32_t splat;
    float alpha;
    float weight;
};

struct RecordOptions {
    bool max_t = false;
    bool contributions = false;  // full blend-event stream (glibc-exact alpha on the device)
};

struct RenderReport {
    Image image;
    std::size_t pair_count = 0;
    std::size_t splat_count = 0;
    std::map<std::string, double> stage_times;  // seconds (device time per stage)
    std::vector<float> max_t;
    std::vector<BlendRecord> contributions;
};

// Device-resident copy of a scene (uploaded once, reused by every render).
class DeviceScene {
public:
    explicit DeviceScene(std::span<const Gaussian3D> scene);
    DeviceScene(std::uint64_t count, int sh_coeffs, const float* mean, const float* scale,
                const float* rotation, const float* opacity, const float* sh);
    ~DeviceScene();
    DeviceScene(const DeviceScene&) = delete;
    DeviceScene& operator=(const DeviceScene&) = delete;
    std::uint64_t size() const { return count_; }
    const void* handle() const { return handle_; }

private:
    void* handle_ = nullptr;
    std::uint64_t count_ = 0;
};

// ------------------------------------- per-element stage functions
// Each runs the device function the kernels use (one element per CUDA
// thread through the agsx_* helper entry points); alpha_at and eigen_sym2
// are header inlines in the reference and stay inline here.

// preprocess.hpp:29-37
struct Projection {
    Vec2f mean2d;
    SymMat2 cov2d;  // with the +0.3 dilation
    float depth;
};
std::optional<Projection> project(const Gaussian3D& g, const Camera& cam, const RenderConfig& cfg);
// preprocess.hpp:38-40; view_dir must be unit length
Vec3f eval_color(const Gaussian3D& g, Vec3f view_dir);
// preprocess.hpp:44-45 (Eq. 10); std::invalid_argument when det(cov2d) <= 0
float compute_th(const SymMat2& cov2d, float depth, const TUpperLUT& lut, float k, float tau);

// pair_gen.hpp:49-55
struct EffectiveRadius {
    float mahalanobis;  // sqrt(2 ln(opacity / th))
    float pixels;       // mahalanobis * sqrt(lambda_max(cov2d))
};
EffectiveRadius effective_radius(float opacity, float th, const SymMat2& cov2d);
// pair_gen.hpp:60-61: row-major ascending tile ids hit by the splat
void intersect_tiles(const SplatView& s, const TileGrid& grid, Mode mode, const RenderConfig& cfg,
                     std::vector<int>& out);

// rasterizer.hpp:44-50: opacity * exp(-0.5 d^T inv d), clamped
inline float alpha_at(const SplatView& s, Vec2f pixel, float alpha_clamp) {
    const Vec2f d = pixel - s.mean2d;
    const float power = -0.5f * s.inv_cov.quad(d);
    if (power > 0.0f) return 0.0f;
    const float a = s.opacity * std::exp(power);
    return a < alpha_clamp ? a : alpha_clamp;
}

std::vector<SplatView> preprocess_view(std::span<const Gaussian3D> scene, const Camera& cam,
                                       const RenderConfig& cfg, const TUpperLUT* lut = nullptr);
PairGenResult generate_pairs(std::span<const SplatView> splats, const TileGrid& grid, Mode mode,
                             const RenderConfig& cfg);
SortedPairs sort_pairs(std::vector<GaussianTilePair> pairs, int tile_count);
// All tiles of the grid at once (the reference's raster_tile loop,
// rasterizer.cpp:137-147); max_t, if given, is resized to splats.size().
Image raster_tiles(const SortedPairs& sorted, std::span<const SplatView> splats,
                   const TileGrid& grid, const RenderConfig& cfg, std::vector<float>* max_t = nullptr);

// rasterizer.hpp:54-58: one tile's sorted pair span blended into `out`
// (the tile's pixels only); max_t, if given, is raised per splat (sized to
// splats.size()); contributions, if given, receives the tile's blend events
// in the reference's order.
void raster_tile(std::span<const GaussianTilePair> tile_pairs, std::span<const SplatView> splats,
                 const TileGrid& grid, int tile_index, const RenderConfig& cfg, Image& out,
                 std::vector<float>* max_t, std::vector<BlendRecord>* contributions);

// The reference's entry point (rasterizer.hpp:63-65).  The scene is packed and
// uploaded once per span: a later call with the same span (address, length
// and a sampled content fingerprint) reuses the device copy, as a reference
// caller looping over views of one scene expects (calibrate.cpp:29,86,113).
// forget_device_scenes() drops the cached copies (a caller that edits a
// scene in place between calls, below the fingerprint's sampling); the
// environment variable AGS_SCENE_CACHE=0 disables the cache.
RenderReport render(std::span<const Gaussian3D> scene, const Camera& cam, const RenderConfig& cfg,
                    const TUpperLUT* lut = nullptr, const RecordOptions& rec = {});
void forget_device_scenes();
RenderReport render(const DeviceScene& scene, const Camera& cam, const RenderConfig& cfg,
                    const TUpperLUT* lut = nullptr, const RecordOptions& rec = {});

// ------------------------------------------- pair report (analysis.hpp:59-82)
struct ReportSpec {
    Mode mode;
    double k = 0.0;  // used only in AdaGScale mode
};

struct PairReportRow {
    std::string mode;
    double k;
    std::size_t pair_count;      // summed over views
    double reduction_pct;        // vs ELLIPSE, mean of per-view ratios
    double psnr_drop_db;         // vs ELLIPSE renders, mean over views
    double t_preprocess, t_pair_gen, t_sort, t_raster;  // summed seconds (device time)
};

// analysis.cpp:259-312 (the Table IV methodology) with every render on the
// GPU: glibc-exact alpha (frames bit-identical to the reference's), lossless
// reference frames kept in HBM, PSNR numerators reduced on the device.  A
// missing LUT is built from `views` like the reference does.
std::vector<PairReportRow> pair_report(const DeviceScene& scene, std::span<const Camera> views,
                                       std::span<const ReportSpec> specs, const RenderConfig& cfg,
                                       const TUpperLUT* lut = nullptr);
std::vector<PairReportRow> pair_report(std::span<const Gaussian3D> scene, std::span<const Camera> views,
                                       std::span<const ReportSpec> specs, const RenderConfig& cfg,
                                       const TUpperLUT* lut = nullptr);
std::string pair_report_csv(std::span<const PairReportRow> rows);
// Shortest round-trip formatting (std::to_chars), analysis.cpp:314-318.
std::string format_double(double v);

// ------------------------------------------------ scene ingest (gsio.hpp)
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct PlyLoadResult {
    std::vector<Gaussian3D> gaussians;
    std::size_t rejected = 0;  // elements dropped for non-finite values
};

// Binary little-endian 3DGS PLY (gsio.cpp:80-152): sigmoid opacity, exp
// scales, normalised rotation, channel-major f_rest -> coefficient-major SH.
PlyLoadResult load_ply(std::istream& in);
PlyLoadResult load_ply_file(const std::string& path);

// Struct-of-arrays form of load_ply_file for the device upload path: the same
// values, decoded by `threads` host threads (0 = hardware_concurrency) with
// no per-Gaussian heap allocation.  sh: 3 * sh_coeffs floats per Gaussian.
struct PlySoA {
    std::uint64_t count = 0;
    int sh_coeffs = 1;
    std::size_t rejected = 0;
    std::vector<float> mean, scale, rotation, opacity, sh;
};
PlySoA load_ply_soa(const std::string& path, int threads = 0);

// synth.cpp:254-281: `count` cameras on a circle of twice the bounding-box
// diagonal around the scene centre.
std::vector<Camera> orbit_cameras(const std::vector<Gaussian3D>& gaussians, int count, int width, int height,
                                  float fx, float fy, std::uint64_t seed);
std::vector<Camera> orbit_cameras(const float* mean, std::uint64_t n, int count, int width, int height, float fx,
                                  float fy, std::uint64_t seed);

// gsio.cpp:265-281: binary PPM, clamp to [0,1], lround(v * 255).
void write_image(const Image& img, const std::string& path);

// ---------------------------------------------------------- synthetic
struct SynthSpec {
    std::string layout = "slab";
    int camera_count = 24;
    int width = 640;
    int height = 480;
    float fx = 500.0f;
    float fy = 500.0f;
};

struct SynthScene {
    std::vector<Gaussian3D> gaussians;
    std::vector<Camera> cameras;
};

SynthScene synth_scene(std::uint64_t seed, int count, const SynthSpec& spec);

// --------------------------------------------------------------- misc
double psnr(const Image& a, const Image& b);

// analysis.hpp:15-22: PSNR capped at 100 dB (what calibration uses).
inline constexpr double kPsnrCap = 100.0;
double psnr_capped(const Image& a, const Image& b);

// ------------------------------------------------- calibration (calibrate.hpp)
// t_const * 2*pi*sqrt(det(cov2d)) * (x - tau) (calibrate.cpp:67-74).
double peripheral_score_closed(const SymMat2& cov2d, float x, float t_const, float tau);

struct CalibrationResult {
    double k = 0.0;
    TUpperLUT lut;
    double target_drop = 0.0;    // dB
    double achieved_drop = 0.0;  // dB, on calibration views
    int iterations = 0;          // drop evaluations performed
    std::vector<int> calib_view_ids;
};

// calibrate.hpp:18-50.  Every render of the loop runs on the GPU with the
// glibc-exact alpha (images bit-identical to the reference's); reference
// frames stay in HBM and PSNR numerators are reduced on the device.
TUpperLUT build_lut(std::span<const Gaussian3D> scene, std::span<const Camera> calib_views,
                    const RenderConfig& cfg);
TUpperLUT build_lut(const DeviceScene& scene, std::span<const Camera> calib_views, const RenderConfig& cfg);
CalibrationResult search_k(std::span<const Gaussian3D> scene, std::span<const Camera> calib_views,
                           double target_drop, const RenderConfig& cfg, const TUpperLUT& lut,
                           bool worst_case = false);
CalibrationResult search_k(const DeviceScene& scene, std::span<const Camera> calib_views, double target_drop,
                           const RenderConfig& cfg, const TUpperLUT& lut, bool worst_case = false);

}  // namespace ags

// C entry points of libags.so for FFI callers (Python ctypes, bench).
extern "C" {
// Synthetic scene straight into SoA buffers (mean/scale 3n, rotation 4n,
// opacity n, sh 3n) + cameras (agsx_camera array).  Returns 0 or 1 (bad
// layout / count).
int ags_synth_scene_soa(std::uint64_t seed, int count, const char* layout, int camera_count,
                        int width, int height, float fx, float fy, float* mean, float* scale,
                        float* rotation, float* opacity, float* sh, void* cameras);
double ags_psnr(const float* a, const float* b, std::uint64_t n);
}

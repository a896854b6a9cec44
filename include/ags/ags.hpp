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

struct Quatf {
    float w = 1.0f, x = 0.0f, y = 0.0f, z = 0.0f;
    float norm() const { return std::sqrt(w * w + x * x + y * y + z * z); }
    Quatf normalized() const {
        const float n = norm();
        return {w / n, x / n, y / n, z / n};
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

struct Camera {
    Vec3f position;
    Mat3f rotation;  // world-to-camera
    float fx = 1.0f, fy = 1.0f;
    int width = 0, height = 0;
};

std::string validate(const Camera& cam);
float orthonormality_drift(const Mat3f& r);

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

std::vector<SplatView> preprocess_view(std::span<const Gaussian3D> scene, const Camera& cam,
                                       const RenderConfig& cfg, const TUpperLUT* lut = nullptr);
PairGenResult generate_pairs(std::span<const SplatView> splats, const TileGrid& grid, Mode mode,
                             const RenderConfig& cfg);
SortedPairs sort_pairs(std::vector<GaussianTilePair> pairs, int tile_count);
// All tiles of the grid at once (the reference's raster_tile loop,
// rasterizer.cpp:137-147); max_t, if given, is resized to splats.size().
Image raster_tiles(const SortedPairs& sorted, std::span<const SplatView> splats,
                   const TileGrid& grid, const RenderConfig& cfg, std::vector<float>* max_t = nullptr);

RenderReport render(std::span<const Gaussian3D> scene, const Camera& cam, const RenderConfig& cfg,
                    const TUpperLUT* lut = nullptr, const RecordOptions& rec = {});
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

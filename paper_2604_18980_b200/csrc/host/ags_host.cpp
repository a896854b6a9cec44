// ags_host.cpp -- the reference-facing C++ API (include/ags/ags.hpp) over the
// C-ABI of libagsx.so.  Host code only: validation, scene packing, the
// synthetic scene generator and result marshalling.  Every stage of the
// render path runs on the GPU.
//
// Compiled with -ffp-contract=off and no -march so the synthetic scene
// generator rounds exactly like the reference build (SURVEY.md §7 hard part 7).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <mutex>
#include <thread>

#include <sys/mman.h>

#include "agsx.h"
#include "ags/ags.hpp"
#include "ags_internal.hpp"

namespace ags {

// ------------------------------------------------------------------ Rng
// PCG32 (math.hpp:169-214).
Rng::Rng(std::uint64_t seed, std::uint64_t stream) {
    state_ = 0;
    inc_ = (stream << 1u) | 1u;
    next_u32();
    state_ += seed;
    next_u32();
}

std::uint32_t Rng::next_u32() {
    const std::uint64_t s = state_;
    state_ = s * 6364136223846793005ULL + inc_;
    const auto x = static_cast<std::uint32_t>(((s >> 18u) ^ s) >> 27u);
    const auto rot = static_cast<std::uint32_t>(s >> 59u);
    return (x >> rot) | (x << ((-rot) & 31u));
}

float Rng::uniform() { return static_cast<float>(next_u32() >> 8) * 0x1.0p-24f; }

float Rng::normal() {
    if (has_spare_) {
        has_spare_ = false;
        return spare_;
    }
    float u1 = uniform();
    while (u1 <= 1e-12f) u1 = uniform();
    const float u2 = uniform();
    const float rad = std::sqrt(-2.0f * std::log(u1));
    const float ang = 6.28318530717958648f * u2;
    spare_ = rad * std::sin(ang);
    has_spare_ = true;
    return rad * std::cos(ang);
}

// --------------------------------------------------------- validation
int sh_degree(const Gaussian3D& g) {
    switch (g.sh.size()) {
        case 3: return 0;
        case 12: return 1;
        case 27: return 2;
        case 48: return 3;
        default: return -1;
    }
}

std::string validate(const Gaussian3D& g) {
    if (std::abs(g.rotation.norm() - 1.0f) > 1e-6f) return "rotation quaternion is not unit length";
    if (!(g.scale.x > 0.0f && g.scale.y > 0.0f && g.scale.z > 0.0f))
        return "scale components must be strictly positive";
    if (!(g.opacity > 0.0f && g.opacity < 1.0f)) return "opacity must lie in (0, 1)";
    if (sh_degree(g) < 0) return "sh coefficient count must be 3*d^2 for d in {1,2,3,4}";
    for (float v : g.sh)
        if (!std::isfinite(v)) return "sh coefficients must be finite";
    if (!(std::isfinite(g.mean.x) && std::isfinite(g.mean.y) && std::isfinite(g.mean.z)))
        return "mean must be finite";
    return {};
}

float orthonormality_drift(const Mat3f& r) {
    const Mat3f g = r.transposed() * r;
    float drift = 0.0f;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            const float dev = std::abs(g(i, j) - (i == j ? 1.0f : 0.0f));
            drift = drift < dev ? dev : drift;
        }
    return drift;
}

std::string validate(const Camera& cam) {
    if (orthonormality_drift(cam.rotation) > 1e-5f) return "camera rotation is not orthonormal";
    if (!(cam.fx > 0.0f && cam.fy > 0.0f)) return "focal lengths must be positive";
    if (!(cam.width > 0 && cam.height > 0)) return "image dimensions must be positive";
    return {};
}

std::string validate(const RenderConfig& c) {
    if (!(c.alpha_threshold > 0.0f && c.alpha_threshold < c.alpha_clamp && c.alpha_clamp <= 1.0f))
        return "require 0 < alpha_threshold < alpha_clamp <= 1";
    if (!(c.transmittance_floor > 0.0f)) return "transmittance_floor must be positive";
    if (c.tile_size < 1) return "tile_size must be >= 1";
    if (c.k < 0.0f) return "k must be >= 0";
    if (!(c.near_plane > 0.0f)) return "near_plane must be positive";
    return {};
}

const char* mode_name(Mode m) {
    static const char* names[] = {"aabb", "obb", "ellipse", "adagscale"};
    const int i = static_cast<int>(m);
    return (i >= 0 && i < 4) ? names[i] : "?";
}

bool parse_mode(const std::string& name, Mode& out) {
    for (int i = 0; i < 4; ++i)
        if (name == mode_name(static_cast<Mode>(i))) {
            out = static_cast<Mode>(i);
            return true;
        }
    return false;
}

int TUpperLUT::bin_index(float depth) const {
    const int nb = static_cast<int>(bins.size());
    const float w = (depth_max - depth_min) / static_cast<float>(nb);
    const float q = (depth - depth_min) / w;
    // static_cast<int> as compiled for x86-64 (cvttss2si): NaN/overflow -> INT_MIN
    const int b = (q > -2147483904.0f && q < 2147483648.0f) ? static_cast<int>(q)
                                                             : std::numeric_limits<int>::min();
    return b < 0 ? 0 : (b >= nb ? nb - 1 : b);
}

double psnr(const Image& a, const Image& b) {
    if (a.width != b.width || a.height != b.height)
        throw std::invalid_argument("psnr: image dimensions differ");
    return ags_psnr(a.data.data(), b.data.data(), a.data.size());
}

// ------------------------------------------------------ synthetic scenes
// Layouts of synth.cpp:65-252, rewritten around a single "sheet" generator.
// Every RNG draw is an explicit statement so the draw order is obvious.
namespace {

constexpr float kShC0 = 0.28209479177387814f;

struct SceneSink {
    virtual ~SceneSink() = default;
    virtual void gaussian(const Vec3f& mean, const Vec3f& scale, const Quatf& q, float opacity,
                          float r, float g, float b) = 0;
    virtual void camera(const Camera& c) = 0;
};

Quatf random_rotation(Rng& rng) {
    Quatf q;
    q.w = rng.normal();
    q.x = rng.normal();
    q.y = rng.normal();
    q.z = rng.normal();
    if (q.norm() < 1e-6f) q = Quatf{};
    return q.normalized();
}

Quatf small_rotation(Rng& rng, float max_angle) {
    const float angle = rng.uniform(0.0f, max_angle);
    Vec3f axis;
    axis.x = rng.normal();
    axis.y = rng.normal();
    axis.z = rng.normal();
    axis = axis.norm() > 1e-6f ? axis.normalized() : Vec3f{0, 0, 1};
    const float s = std::sin(0.5f * angle);
    return Quatf{std::cos(0.5f * angle), axis.x * s, axis.y * s, axis.z * s}.normalized();
}

Camera look_at(Vec3f pos, Vec3f target, const SynthSpec& spec) {
    const Vec3f fwd = (target - pos).normalized();
    Vec3f up{0, 1, 0};
    if (std::abs(fwd.dot(up)) > 0.99f) up = {0, 0, 1};
    const Vec3f right = up.cross(fwd).normalized();
    const Vec3f down = fwd.cross(right);
    Camera c;
    c.position = pos;
    const Vec3f rows[3] = {right, down, fwd};
    for (int r = 0; r < 3; ++r) {
        c.rotation(r, 0) = rows[r].x;
        c.rotation(r, 1) = rows[r].y;
        c.rotation(r, 2) = rows[r].z;
    }
    c.fx = spec.fx;
    c.fy = spec.fy;
    c.width = spec.width;
    c.height = spec.height;
    return c;
}

void arc(Rng& rng, const SynthSpec& spec, float radius, float span, SceneSink& out) {
    const int n = spec.camera_count;
    for (int i = 0; i < n; ++i) {
        const float t = n > 1 ? static_cast<float>(i) / (n - 1) : 0.5f;
        const float theta = (t - 0.5f) * span;
        const float y = rng.uniform(-1.5f, 1.5f);
        out.camera(look_at({radius * std::sin(theta), y, -radius * std::cos(theta)}, {0, 0, 0}, spec));
    }
}

void colour(Rng& rng, float& r, float& g, float& b) {
    r = rng.uniform(0.1f, 0.9f);
    g = rng.uniform(0.1f, 0.9f);
    b = rng.uniform(0.1f, 0.9f);
}

// slab layout member (synth.cpp:65-80)
void slab_member(Rng& rng, float hx, float hy, float zc, float zt, float s0, float s1, float o0,
                 float o1, SceneSink& out) {
    Vec3f m, s;
    m.x = rng.uniform(-hx, hx);
    m.y = rng.uniform(-hy, hy);
    m.z = zc + rng.uniform(-zt, zt);
    s.x = rng.uniform(s0, s1);
    s.y = rng.uniform(s0, s1);
    s.z = rng.uniform(0.05f, 0.15f);
    const Quatf q = random_rotation(rng);
    const float op = rng.uniform(o0, o1);
    float r, g, b;
    colour(rng, r, g, b);
    out.gaussian(m, s, q, op, r, g, b);
}

// curtain / wall member of two_slab and veil (synth.cpp:105-183)
void sheet_member(Rng& rng, bool rear, float spacing, float s0, float s1, float o0, float o1,
                  SceneSink& out) {
    Vec3f m, s;
    if (rear) {
        m.x = rng.uniform(-6.0f, 6.0f);
        m.y = rng.uniform(-4.0f, 4.0f);
        m.z = 20.0f + rng.uniform(-0.2f, 0.2f);
    } else {
        m.x = rng.uniform(-10.0f, 10.0f);
        m.y = rng.uniform(-7.0f, 7.0f);
        m.z = rng.uniform(-0.2f, 0.2f);
    }
    const float side = spacing * rng.uniform(s0, s1);
    s.x = side;
    s.y = side * rng.uniform(0.8f, 1.2f);
    s.z = 0.1f * side;
    const Quatf q = small_rotation(rng, 0.2f);
    const float op = rng.uniform(o0, o1);
    float r, g, b;
    colour(rng, r, g, b);
    out.gaussian(m, s, q, op, r, g, b);
}

void generate(std::uint64_t seed, int count, const SynthSpec& spec, SceneSink& out) {
    if (count < 1) throw std::invalid_argument("synth_scene: count must be >= 1");
    Rng rng(seed);
    const std::string& L = spec.layout;
    if (L == "slab") {
        const int front = (count * 3 + 2) / 5;
        for (int i = 0; i < count; ++i) {
            if (i < front)
                slab_member(rng, 8, 6, 0.0f, 0.3f, 0.15f, 0.45f, 0.7f, 0.97f, out);
            else
                slab_member(rng, 14, 10, 15.0f, 0.3f, 0.3f, 0.8f, 0.4f, 0.9f, out);
        }
        arc(rng, spec, 24.0f, 1.2f, out);
    } else if (L == "two_slab" || L == "veil") {
        const bool veil = L == "veil";
        const int front = veil ? (count * 35 + 50) / 100 : count / 2;
        const int rear = count - front;
        const float fsp = std::sqrt(20.0f * 14.0f / static_cast<float>(std::max(front, 1)));
        const float rsp = std::sqrt(12.0f * 8.0f / static_cast<float>(std::max(rear, 1)));
        for (int i = 0; i < front; ++i) sheet_member(rng, false, fsp, 1.1f, 1.8f, 0.85f, 0.98f, out);
        for (int i = 0; i < rear; ++i) {
            if (veil)
                sheet_member(rng, true, rsp, 8.0f, 14.0f, 0.6f, 0.95f, out);
            else
                sheet_member(rng, true, rsp, 0.9f, 1.5f, 0.5f, 0.95f, out);
        }
        arc(rng, spec, 22.0f, 1.1f, out);
    } else if (L == "ramp") {
        const float hw = 0.5f * spec.width / spec.fx;
        const float hh = 0.5f * spec.height / spec.fy;
        for (int i = 0; i < count; ++i) {
            const float z = rng.uniform(3.0f, 92.0f);
            Vec3f m, s;
            m.x = rng.uniform(-0.8f, 0.8f) * hw * z;
            m.y = rng.uniform(-0.8f, 0.8f) * hh * z;
            m.z = z;
            const float base = z * rng.uniform(0.010f, 0.022f);
            s.x = base * rng.uniform(0.6f, 1.4f);
            s.y = base * rng.uniform(0.6f, 1.4f);
            s.z = base * rng.uniform(0.6f, 1.4f);
            const Quatf q = random_rotation(rng);
            const float op = rng.uniform(0.3f, 0.95f);
            float r, g, b;
            colour(rng, r, g, b);
            out.gaussian(m, s, q, op, r, g, b);
        }
        for (int i = 0; i < spec.camera_count; ++i) {
            Camera c;
            c.position.x = rng.uniform(-0.4f, 0.4f);
            c.position.y = rng.uniform(-0.3f, 0.3f);
            c.position.z = rng.uniform(-0.8f, 0.0f);
            c.fx = spec.fx;
            c.fy = spec.fy;
            c.width = spec.width;
            c.height = spec.height;
            out.camera(c);
        }
    } else if (L == "aniso") {
        for (int i = 0; i < count; ++i) {
            Vec3f m, s;
            m.x = rng.uniform(-10.0f, 10.0f);
            m.y = rng.uniform(-7.0f, 7.0f);
            m.z = rng.uniform(-4.0f, 4.0f);
            const float major = rng.uniform(0.5f, 1.2f);
            s.x = major;
            s.y = major * rng.uniform(0.08f, 0.25f);
            s.z = rng.uniform(0.05f, 0.15f);
            const Quatf q = random_rotation(rng);
            const float op = rng.uniform(0.35f, 0.95f);
            float r, g, b;
            colour(rng, r, g, b);
            out.gaussian(m, s, q, op, r, g, b);
        }
        arc(rng, spec, 26.0f, 1.2f, out);
    } else {
        throw std::invalid_argument("synth_scene: unknown layout '" + L + "'");
    }
}

struct AosSink : SceneSink {
    SynthScene* s;
    void gaussian(const Vec3f& m, const Vec3f& sc, const Quatf& q, float op, float r, float g,
                  float b) override {
        Gaussian3D x;
        x.mean = m;
        x.scale = sc;
        x.rotation = q;
        x.opacity = op;
        x.sh = {(r - 0.5f) / kShC0, (g - 0.5f) / kShC0, (b - 0.5f) / kShC0};
        s->gaussians.push_back(std::move(x));
    }
    void camera(const Camera& c) override { s->cameras.push_back(c); }
};

struct SoaSink : SceneSink {
    float *mean, *scale, *rot, *op, *sh;
    agsx_camera* cams;
    std::uint64_t n = 0;
    int nc = 0;
    void gaussian(const Vec3f& m, const Vec3f& sc, const Quatf& q, float o, float r, float g,
                  float b) override {
        const std::uint64_t i = n++;
        mean[3 * i] = m.x;
        mean[3 * i + 1] = m.y;
        mean[3 * i + 2] = m.z;
        scale[3 * i] = sc.x;
        scale[3 * i + 1] = sc.y;
        scale[3 * i + 2] = sc.z;
        rot[4 * i] = q.w;
        rot[4 * i + 1] = q.x;
        rot[4 * i + 2] = q.y;
        rot[4 * i + 3] = q.z;
        op[i] = o;
        sh[3 * i] = (r - 0.5f) / kShC0;
        sh[3 * i + 1] = (g - 0.5f) / kShC0;
        sh[3 * i + 2] = (b - 0.5f) / kShC0;
    }
    void camera(const Camera& c) override {
        agsx_camera& a = cams[nc++];
        a.position[0] = c.position.x;
        a.position[1] = c.position.y;
        a.position[2] = c.position.z;
        for (int i = 0; i < 9; ++i) a.rotation[i] = c.rotation.m[i];
        a.fx = c.fx;
        a.fy = c.fy;
        a.width = c.width;
        a.height = c.height;
    }
};

}  // namespace

SynthScene synth_scene(std::uint64_t seed, int count, const SynthSpec& spec) {
    SynthScene s;
    if (count > 0) s.gaussians.reserve(count);
    AosSink sink;
    sink.s = &s;
    generate(seed, count, spec, sink);
    return s;
}

// ----------------------------------------------------- device plumbing
namespace detail {

struct CtxHolder {
    agsx_ctx* ctx = nullptr;
    ~CtxHolder() {
        if (ctx) agsx_destroy(ctx);
    }
};

int default_device() {
    const char* e = std::getenv("AGS_DEVICE");
    return e ? std::atoi(e) : 0;
}

// A page-locked staging image per host thread (grow-only): the raster streams
// the frame into it by banded copy-engine transfers behind the blend.
struct Staging {
    float* p = nullptr;
    std::size_t floats = 0;
    ~Staging() {
        if (p) agsx_host_free(p);
    }
    float* get(std::size_t n) {
        if (n > floats) {
            if (p) agsx_host_free(p);
            p = nullptr;
            floats = 0;
            void* q = nullptr;
            if (agsx_host_alloc(n * sizeof(float), &q) != AGSX_OK) throw std::bad_alloc();
            p = static_cast<float*>(q);
            floats = n;
        }
        return p;
    }
};

float* thread_staging(std::size_t n) {
    static thread_local Staging st;
    return st.get(n);
}

// The returned Image owns a std::vector<float> (image.hpp:9-23).  A fresh
// 191 MB vector (4608x3456) costs its page faults, a zero fill and the copy:
// ~40 ms a call on one thread.  ImageFill splits that around the GPU frame:
// start() (before the frame) reserves the buffer with transparent huge pages
// and faults it in on host threads while the GPU renders; finish() (after
// it) copies the staging image in by slices on host threads, then sizes the
// vector by assign() over its own storage -- the copy already made the
// values, the assignment copies each float onto itself (glibc's memmove
// returns at once when source and destination coincide), so no single-
// threaded zero fill is paid.  Images under 512 KB take the one-pass assign.
class ImageFill {
public:
    ImageFill(Image& img, int w, int h) : img_(img), n_(static_cast<std::size_t>(w) * h * 3) {
        img.width = w;
        img.height = h;
        // one host thread per 256 KB of image, up to 16 (320x240: 3 slices)
        const std::size_t by_size = std::max<std::size_t>(1, n_ >> 16);
        nt_ = static_cast<unsigned>(std::min<std::size_t>({16, by_size, std::max(1u, std::thread::hardware_concurrency())}));
        per_ = ((n_ + nt_ - 1) / nt_ + 1023) & ~std::size_t{1023};  // 4 KB-aligned slices
        img.data.clear();
        img.data.shrink_to_fit();
        img.data.reserve(n_);
        if (nt_ == 1) return;
        const std::uintptr_t b = reinterpret_cast<std::uintptr_t>(img.data.data());
        const std::uintptr_t a = (b + (1u << 21) - 1) & ~static_cast<std::uintptr_t>((1u << 21) - 1);
        const std::uintptr_t e = (b + n_ * sizeof(float)) & ~static_cast<std::uintptr_t>((1u << 21) - 1);
        if (e > a) madvise(reinterpret_cast<void*>(a), e - a, MADV_HUGEPAGE);  // advisory: ignore failures
        // fault the reserved pages in (one byte store per 4 KB page) while the frame renders
        volatile char* base = reinterpret_cast<volatile char*>(img.data.data());
        for (unsigned t = 0; t < nt_; ++t)
            if (t * per_ < n_)
                faulting_.emplace_back([base, lo = t * per_ * sizeof(float), hi = std::min(n_, (t + 1) * per_) * sizeof(float)] {
                    for (std::size_t i = lo; i < hi; i += 4096) base[i] = 0;
                });
    }
    ~ImageFill() { join(); }
    void finish(const float* src) {
        join();
        if (nt_ == 1) {
            img_.data.assign(src, src + n_);
            return;
        }
        float* dst = img_.data.data();  // reserved storage: the copy creates the floats in it
        std::vector<std::thread> pool;
        for (unsigned t = 1; t < nt_; ++t)
            if (t * per_ < n_)
                pool.emplace_back([=, this] { std::memcpy(dst + t * per_, src + t * per_, (std::min(n_, (t + 1) * per_) - t * per_) * sizeof(float)); });
        std::memcpy(dst, src, std::min(n_, per_) * sizeof(float));
        for (auto& th : pool) th.join();
        img_.data.assign(dst, dst + n_);  // capacity suffices: no reallocation, a self-copy
    }

private:
    void join() {
        for (auto& th : faulting_) th.join();
        faulting_.clear();
    }
    Image& img_;
    std::size_t n_, per_ = 0;
    unsigned nt_ = 1;
    std::vector<std::thread> faulting_;
};

agsx_ctx* thread_ctx() {
    static thread_local CtxHolder h;
    if (!h.ctx) {
        const int rc = agsx_create(default_device(), &h.ctx);
        if (rc != AGSX_OK) throw std::runtime_error("agsx_create failed (no usable CUDA device?)");
    }
    return h.ctx;
}

[[noreturn]] void raise_status(int rc, agsx_ctx* ctx) {
    const std::string msg = agsx_last_error(ctx);
    switch (rc) {
        case AGSX_EINVAL: throw std::invalid_argument(msg);
        case AGSX_EPAIR_BUDGET: throw PairBudgetError(msg);
        case AGSX_ENOMEM: throw std::bad_alloc();
        default: throw std::runtime_error(msg.empty() ? "agsx: device error" : msg);
    }
}

void check(int rc, agsx_ctx* ctx) {
    if (rc != AGSX_OK) raise_status(rc, ctx);
}

agsx_camera to_c(const Camera& c) {
    agsx_camera a;
    a.position[0] = c.position.x;
    a.position[1] = c.position.y;
    a.position[2] = c.position.z;
    for (int i = 0; i < 9; ++i) a.rotation[i] = c.rotation.m[i];
    a.fx = c.fx;
    a.fy = c.fy;
    a.width = c.width;
    a.height = c.height;
    return a;
}

agsx_config to_c(const RenderConfig& c) {
    agsx_config a;
    a.tile_size = c.tile_size;
    a.alpha_threshold = c.alpha_threshold;
    a.transmittance_floor = c.transmittance_floor;
    a.alpha_clamp = c.alpha_clamp;
    a.near_plane = c.near_plane;
    a.guard_band = c.guard_band;
    a.mode = static_cast<int32_t>(c.mode);
    a.k = c.k;
    a.thread_count = c.thread_count;
    a.background[0] = c.background.x;
    a.background[1] = c.background.y;
    a.background[2] = c.background.z;
    a.fixed_radius_aabb = c.fixed_radius_aabb ? 1 : 0;
    a.pair_budget = c.pair_budget;
    a.flags = 0;
    if (const char* e = std::getenv("AGS_EXACT_ALPHA"); e && *e == '1') a.flags |= AGSX_FLAG_EXACT_ALPHA;
    return a;
}

agsx_lut to_c(const TUpperLUT& l) {
    agsx_lut a;
    a.depth_min = l.depth_min;
    a.depth_max = l.depth_max;
    a.bin_count = static_cast<int32_t>(l.bins.size());
    a.bins = l.bins.data();
    return a;
}

agsx_splat_view to_c(const SplatView& s) {
    agsx_splat_view v;
    std::memcpy(&v, &s, sizeof(v));
    return v;
}

static_assert(sizeof(SplatView) == sizeof(agsx_splat_view), "SplatView layout");

// Pads SH to the largest degree present (zero coefficients are bit-neutral,
// preprocess.cpp:71-101) and packs the AoS scene into SoA arrays.  The arrays
// are allocated uninitialised and written once by host threads (each thread
// takes its slice's page faults), so no single-threaded zero fill is paid.
struct PackedScene {
    std::unique_ptr<float[]> mean, scale, rot, op, sh;
    int D = 1;
};

PackedScene pack(std::span<const Gaussian3D> scene) {
    PackedScene p;
    std::size_t maxc = 3;
    for (const Gaussian3D& g : scene) maxc = std::max(maxc, g.sh.size());
    if (maxc != 3 && maxc != 12 && maxc != 27 && maxc != 48)
        throw std::invalid_argument("sh coefficient count must be 3*d^2 for d in {1,2,3,4}");
    p.D = static_cast<int>(maxc / 3);
    const std::size_t n = scene.size();
    const std::size_t m = std::max<std::size_t>(n, 1);
    p.mean.reset(new float[3 * m]);
    p.scale.reset(new float[3 * m]);
    p.rot.reset(new float[4 * m]);
    p.op.reset(new float[m]);
    p.sh.reset(new float[maxc * m]);
    auto run = [&](std::size_t lo, std::size_t hi) {
        for (std::size_t i = lo; i < hi; ++i) {
            const Gaussian3D& g = scene[i];
            p.mean[3 * i] = g.mean.x;
            p.mean[3 * i + 1] = g.mean.y;
            p.mean[3 * i + 2] = g.mean.z;
            p.scale[3 * i] = g.scale.x;
            p.scale[3 * i + 1] = g.scale.y;
            p.scale[3 * i + 2] = g.scale.z;
            p.rot[4 * i] = g.rotation.w;
            p.rot[4 * i + 1] = g.rotation.x;
            p.rot[4 * i + 2] = g.rotation.y;
            p.rot[4 * i + 3] = g.rotation.z;
            p.op[i] = g.opacity;
            float* sh = p.sh.get() + maxc * i;
            std::copy(g.sh.begin(), g.sh.end(), sh);
            std::fill(sh + g.sh.size(), sh + maxc, 0.0f);
        }
    };
    // AoS -> SoA by host threads (the per-Gaussian SH vectors are separate
    // heap blocks, so one thread is bound by their cache misses)
    const unsigned nt = n < (1u << 16) ? 1u : std::min(16u, std::max(1u, std::thread::hardware_concurrency()));
    if (nt == 1) {
        run(0, n);
    } else {
        std::vector<std::thread> pool;
        const std::size_t per = (n + nt - 1) / nt;
        for (unsigned t = 0; t < nt; ++t) pool.emplace_back(run, std::min(n, t * per), std::min(n, (t + 1) * per));
        for (auto& th : pool) th.join();
    }
    return p;
}

}  // namespace detail

using namespace detail;

DeviceScene::DeviceScene(std::span<const Gaussian3D> scene) {
    const PackedScene p = pack(scene);
    agsx_scene_desc d{scene.size(), p.D, p.mean.get(), p.scale.get(), p.rot.get(), p.op.get(), p.sh.get()};
    agsx_ctx* ctx = thread_ctx();
    agsx_scene* s = nullptr;
    check(agsx_scene_upload(ctx, &d, &s), ctx);
    handle_ = s;
    count_ = scene.size();
}

DeviceScene::DeviceScene(std::uint64_t count, int sh_coeffs, const float* mean, const float* scale,
                         const float* rotation, const float* opacity, const float* sh) {
    agsx_scene_desc d{count, sh_coeffs, mean, scale, rotation, opacity, sh};
    agsx_ctx* ctx = thread_ctx();
    agsx_scene* s = nullptr;
    check(agsx_scene_upload(ctx, &d, &s), ctx);
    handle_ = s;
    count_ = count;
}

DeviceScene::~DeviceScene() { agsx_scene_free(static_cast<agsx_scene*>(handle_)); }

RenderReport render(const DeviceScene& scene, const Camera& cam, const RenderConfig& cfg,
                    const TUpperLUT* lut, const RecordOptions& rec) {
    if (const std::string bad = validate(cfg); !bad.empty()) throw std::invalid_argument("render: " + bad);
    if (const std::string bad = validate(cam); !bad.empty()) throw std::invalid_argument("render: " + bad);
    agsx_ctx* ctx = thread_ctx();
    const agsx_camera c = to_c(cam);
    const agsx_config k = to_c(cfg);
    agsx_lut l{};
    if (lut) l = to_c(*lut);
    RenderReport rep;
    const std::size_t npx = static_cast<std::size_t>(cam.width) * cam.height;
    float* staging = thread_staging(npx * 3);
    std::vector<float> maxt_by_gid;
    agsx_frame f{};
    f.image = staging;
    ImageFill fill(rep.image, cam.width, cam.height);
    if (rec.max_t) {
        maxt_by_gid.assign(std::max<std::uint64_t>(scene.size(), 1), 0.0f);
        f.max_t = maxt_by_gid.data();
    }
    auto* sc = static_cast<const agsx_scene*>(scene.handle());
    if (rec.contributions) {
        // blend-event stream (rasterizer.cpp:135-161): size it, then fill it
        std::uint64_t count = 0;
        const int rc0 = agsx_render_contributions(ctx, sc, &c, &k, lut ? &l : nullptr, nullptr, 0, &count, &f);
        if (rc0 != AGSX_OK && rc0 != AGSX_ECAPACITY) check(rc0, ctx);
        rep.contributions.resize(count);
        static_assert(sizeof(BlendRecord) == sizeof(agsx_blend_record), "BlendRecord layout");
        if (count)
            check(agsx_render_contributions(ctx, sc, &c, &k, lut ? &l : nullptr,
                                            reinterpret_cast<agsx_blend_record*>(rep.contributions.data()), count,
                                            &count, &f),
                  ctx);
    } else {
        check(agsx_render(ctx, sc, &c, &k, lut ? &l : nullptr, &f), ctx);
    }
    fill.finish(staging);
    rep.pair_count = f.pair_count;
    rep.splat_count = f.splat_count;
    rep.stage_times["preprocess"] = f.stage_ms[0] * 1e-3;
    rep.stage_times["pair_gen"] = f.stage_ms[1] * 1e-3;
    rep.stage_times["sort"] = f.stage_ms[2] * 1e-3;
    rep.stage_times["raster"] = f.stage_ms[3] * 1e-3;
    if (rec.max_t) {
        // RenderReport::max_t is per splat in preprocess order
        std::vector<std::uint8_t> alive(scene.size());
        check(agsx_dump_tile_counts(ctx, nullptr, alive.data(), scene.size()), ctx);
        rep.max_t.reserve(rep.splat_count);
        for (std::uint64_t i = 0; i < scene.size(); ++i)
            if (alive[i]) rep.max_t.push_back(maxt_by_gid[i]);
    }
    return rep;
}

std::vector<SplatView> preprocess_view(std::span<const Gaussian3D> scene, const Camera& cam,
                                       const RenderConfig& cfg, const TUpperLUT* lut) {
    if (cfg.mode == Mode::AdaGScale && lut == nullptr)
        throw std::invalid_argument("preprocess_view: adagscale mode requires a T-upper LUT");
    const DeviceScene dev(scene);
    agsx_ctx* ctx = thread_ctx();
    const agsx_camera c = to_c(cam);
    const agsx_config k = to_c(cfg);
    agsx_lut l{};
    if (lut) l = to_c(*lut);
    std::vector<SplatView> out(scene.size());
    std::uint64_t n = 0;
    check(agsx_preprocess_view(ctx, static_cast<const agsx_scene*>(dev.handle()), &c, &k,
                               lut ? &l : nullptr, reinterpret_cast<agsx_splat_view*>(out.data()), &n),
          ctx);
    out.resize(n);
    return out;
}

PairGenResult generate_pairs(std::span<const SplatView> splats, const TileGrid& grid, Mode mode,
                             const RenderConfig& cfg) {
    agsx_ctx* ctx = thread_ctx();
    agsx_config k = to_c(cfg);
    k.tile_size = grid.tile_size;
    PairGenResult res;
    res.tile_counts.assign(splats.size(), 0);
    std::vector<std::uint64_t> keys;
    std::vector<std::uint32_t> idx;
    std::uint64_t total = 0;
    const auto* sv = reinterpret_cast<const agsx_splat_view*>(splats.data());
    int rc = agsx_generate_pairs(ctx, sv, splats.size(), grid.width, grid.height, static_cast<int>(mode), &k,
                                 nullptr, nullptr, 0, res.tile_counts.data(), &total);
    if (rc == AGSX_ECAPACITY) {
        keys.resize(total);
        idx.resize(total);
        rc = agsx_generate_pairs(ctx, sv, splats.size(), grid.width, grid.height, static_cast<int>(mode), &k,
                                 keys.data(), idx.data(), total, res.tile_counts.data(), &total);
    }
    check(rc, ctx);
    res.pairs.resize(keys.size());
    for (std::size_t i = 0; i < keys.size(); ++i) res.pairs[i] = {keys[i], idx[i]};
    return res;
}

SortedPairs sort_pairs(std::vector<GaussianTilePair> pairs, int tile_count) {
    agsx_ctx* ctx = thread_ctx();
    const std::size_t n = pairs.size();
    std::vector<std::uint64_t> keys(n);
    std::vector<std::uint32_t> idx(n);
    for (std::size_t i = 0; i < n; ++i) {
        keys[i] = pairs[i].key;
        idx[i] = pairs[i].splat_index;
    }
    std::vector<std::uint32_t> ranges(2 * static_cast<std::size_t>(std::max(tile_count, 0)));
    check(agsx_sort_pairs(ctx, keys.data(), idx.data(), n, tile_count, ranges.data()), ctx);
    SortedPairs out;
    out.pairs.resize(n);
    for (std::size_t i = 0; i < n; ++i) out.pairs[i] = {keys[i], idx[i]};
    out.ranges.resize(std::max(tile_count, 0));
    for (int t = 0; t < tile_count; ++t) out.ranges[t] = {ranges[2 * t], ranges[2 * t + 1]};
    return out;
}

Image raster_tiles(const SortedPairs& sorted, std::span<const SplatView> splats, const TileGrid& grid,
                   const RenderConfig& cfg, std::vector<float>* max_t) {
    agsx_ctx* ctx = thread_ctx();
    agsx_config k = to_c(cfg);
    k.tile_size = grid.tile_size;
    std::vector<agsx_splat_view> sv(splats.size());
    for (std::size_t i = 0; i < splats.size(); ++i) sv[i] = to_c(splats[i]);
    std::vector<std::uint32_t> idx(sorted.pairs.size());
    for (std::size_t i = 0; i < idx.size(); ++i) idx[i] = sorted.pairs[i].splat_index;
    std::vector<std::uint32_t> ranges(2 * sorted.ranges.size());
    for (std::size_t t = 0; t < sorted.ranges.size(); ++t) {
        ranges[2 * t] = sorted.ranges[t].first;
        ranges[2 * t + 1] = sorted.ranges[t].second;
    }
    Image img(grid.width, grid.height);
    if (max_t) max_t->assign(splats.size(), 0.0f);
    check(agsx_raster(ctx, sv.data(), sv.size(), idx.data(), idx.size(), ranges.data(), grid.width,
                      grid.height, &k, img.data.data(), max_t ? max_t->data() : nullptr),
          ctx);
    return img;
}

}  // namespace ags

// ------------------------------------------------------------- C entry
extern "C" int ags_synth_scene_soa(std::uint64_t seed, int count, const char* layout, int camera_count,
                                   int width, int height, float fx, float fy, float* mean, float* scale,
                                   float* rotation, float* opacity, float* sh, void* cameras) {
    try {
        ags::SynthSpec spec;
        spec.layout = layout;
        spec.camera_count = camera_count;
        spec.width = width;
        spec.height = height;
        spec.fx = fx;
        spec.fy = fy;
        ags::SoaSink sink;
        sink.mean = mean;
        sink.scale = scale;
        sink.rot = rotation;
        sink.op = opacity;
        sink.sh = sh;
        sink.cams = static_cast<agsx_camera*>(cameras);
        ags::generate(seed, count, spec, sink);
        return 0;
    } catch (...) {
        return 1;
    }
}

extern "C" double ags_psnr(const float* a, const float* b, std::uint64_t n) {
    // analysis.cpp:14-25: double accumulation, +inf on identical images
    double se = 0.0;
    for (std::uint64_t i = 0; i < n; ++i) {
        const double d = static_cast<double>(a[i]) - b[i];
        se += d * d;
    }
    if (se == 0.0) return std::numeric_limits<double>::infinity();
    return 10.0 * std::log10(1.0 / (se / static_cast<double>(n)));
}

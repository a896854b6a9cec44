/*
 * ags_oracle.c -- TEST INFRASTRUCTURE ONLY ("port" oracle).
 *
 * A from-scratch, single-threaded plain-C restatement of the AdaGScale CPU
 * render path of the reference (arXiv 2604.18980 reproduction under
 * /root/reference/proj).  It is the checker for the CUDA product path and is
 * itself pinned bit-for-bit against the unmodified reference build
 * (oracle/_ref/libags_ref.so) by tests/test_oracle.py and against the
 * committed fixtures in tests/golden/.
 *
 * Floating-point contract (the same one the reference build has):
 *   - compiled with -O2 -ffp-contract=off and no -march, so every a*b+c is
 *     two IEEE roundings (the reference objects contain no vfmadd);
 *   - float and double are mixed exactly where the reference mixes them;
 *   - logf / expf / sinf / cosf come from the host glibc, like the reference.
 * C does not specify argument evaluation order, so every RNG draw that the
 * C++ reference performs inside a braced initialiser (left-to-right by
 * rule) is sequenced explicitly here.
 */
#include "ags_oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* libstdc++ semantics of std::min / std::max / std::clamp
 * (stl_algobase.h / stl_algo.h): max(a,b) = a<b ? b : a, min(a,b) = b<a ? b
 * : a, clamp(v,lo,hi) = min(max(v,lo),hi).  These differ from fminf/fmaxf
 * on NaN and are reproduced literally. */
static inline float maxf_(float a, float b) { return a < b ? b : a; }
static inline float minf_(float a, float b) { return b < a ? b : a; }
static inline float clampf_(float v, float lo, float hi) {
    return minf_(maxf_(v, lo), hi);
}
static inline double clampd_(double v, double lo, double hi) {
    double m = v < lo ? lo : v;
    return hi < m ? hi : m;
}
static inline int maxi_(int a, int b) { return a < b ? b : a; }
static inline int mini_(int a, int b) { return b < a ? b : a; }

/* ------------------------------------------------------------------ */
/* PCG32 with Box-Muller (math.hpp:169-214). */
typedef struct {
    uint64_t state, inc;
    float spare;
    int has_spare;
} rng_t;

static uint32_t rng_u32(rng_t* r) {
    const uint64_t old = r->state;
    r->state = old * 6364136223846793005ULL + r->inc;
    const uint32_t xs = (uint32_t)(((old >> 18u) ^ old) >> 27u);
    const uint32_t rot = (uint32_t)(old >> 59u);
    return (xs >> rot) | (xs << ((-rot) & 31u));
}

static void rng_init(rng_t* r, uint64_t seed, uint64_t stream) {
    r->state = 0;
    r->inc = (stream << 1u) | 1u;
    r->has_spare = 0;
    r->spare = 0.0f;
    rng_u32(r);
    r->state += seed;
    rng_u32(r);
}

static float rng_unit(rng_t* r) { return (float)(rng_u32(r) >> 8) * 0x1.0p-24f; }

static float rng_uniform(rng_t* r, float lo, float hi) {
    return lo + (hi - lo) * rng_unit(r);
}

static float rng_normal(rng_t* r) {
    if (r->has_spare) {
        r->has_spare = 0;
        return r->spare;
    }
    float u1 = rng_unit(r);
    while (u1 <= 1e-12f) u1 = rng_unit(r);
    const float u2 = rng_unit(r);
    const float rad = sqrtf(-2.0f * logf(u1));
    const float a = 6.28318530717958648f * u2;
    r->spare = rad * sinf(a);
    r->has_spare = 1;
    return rad * cosf(a);
}

/* ------------------------------------------------------------------ */
/* Small vector helpers (math.hpp:9-33), left-to-right sums. */
typedef struct { float x, y, z; } v3;

static inline float v3_dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static inline v3 v3_sub(v3 a, v3 b) { v3 o = {a.x - b.x, a.y - b.y, a.z - b.z}; return o; }
static inline v3 v3_scale(v3 a, float s) { v3 o = {a.x * s, a.y * s, a.z * s}; return o; }
static inline v3 v3_norm(v3 a) { /* Vec3f::normalized, math.hpp:25-28 */
    const float n = sqrtf(v3_dot(a, a));
    if (n > 0.0f) return v3_scale(a, 1.0f / n);
    v3 z = {0, 0, 0};
    return z;
}
static inline v3 v3_cross(v3 a, v3 o) {
    v3 r = {a.y * o.z - a.z * o.y, a.z * o.x - a.x * o.z, a.x * o.y - a.y * o.x};
    return r;
}

typedef struct { float w, x, y, z; } quat;

static quat quat_normalized(quat q) { /* Quatf::normalized, math.hpp:138-142 */
    const float n = sqrtf(q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z);
    quat o = {q.w / n, q.x / n, q.y / n, q.z / n};
    return o;
}

/* ------------------------------------------------------------------ */
/* Synthetic scenes (synth.cpp). */
static const float kShC0 = 0.28209479177387814f;

typedef struct {
    float* mean;
    float* scale;
    float* rot;
    float* opacity;
    float* sh;
    uint64_t n;
} soa_out;

static void put_gaussian(soa_out* o, v3 mean, v3 scale, quat q, float opacity,
                         float r, float g, float b) {
    const uint64_t i = o->n++;
    o->mean[3 * i] = mean.x;
    o->mean[3 * i + 1] = mean.y;
    o->mean[3 * i + 2] = mean.z;
    o->scale[3 * i] = scale.x;
    o->scale[3 * i + 1] = scale.y;
    o->scale[3 * i + 2] = scale.z;
    o->rot[4 * i] = q.w;
    o->rot[4 * i + 1] = q.x;
    o->rot[4 * i + 2] = q.y;
    o->rot[4 * i + 3] = q.z;
    o->opacity[i] = opacity;
    /* dc_for_rgb, synth.cpp:14-17 */
    o->sh[3 * i] = (r - 0.5f) / kShC0;
    o->sh[3 * i + 1] = (g - 0.5f) / kShC0;
    o->sh[3 * i + 2] = (b - 0.5f) / kShC0;
}

static void draw_rgb(rng_t* rng, float* r, float* g, float* b) {
    *r = rng_uniform(rng, 0.1f, 0.9f);
    *g = rng_uniform(rng, 0.1f, 0.9f);
    *b = rng_uniform(rng, 0.1f, 0.9f);
}

static quat random_rotation(rng_t* rng) { /* synth.cpp:19-23 */
    quat q;
    q.w = rng_normal(rng);
    q.x = rng_normal(rng);
    q.y = rng_normal(rng);
    q.z = rng_normal(rng);
    const float n = sqrtf(q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z);
    if (n < 1e-6f) {
        quat id = {1, 0, 0, 0};
        q = id;
    }
    return quat_normalized(q);
}

static quat small_rotation(rng_t* rng, float max_angle) { /* synth.cpp:95-103 */
    const float angle = rng_uniform(rng, 0.0f, max_angle);
    v3 axis;
    axis.x = rng_normal(rng);
    axis.y = rng_normal(rng);
    axis.z = rng_normal(rng);
    if (sqrtf(v3_dot(axis, axis)) > 1e-6f) {
        axis = v3_norm(axis);
    } else {
        v3 zz = {0, 0, 1};
        axis = zz;
    }
    const float s = sinf(0.5f * angle);
    quat q = {cosf(0.5f * angle), axis.x * s, axis.y * s, axis.z * s};
    return quat_normalized(q);
}

static void look_at(v3 pos, v3 target, float fx, float fy, int w, int h,
                    ago_camera* cam) { /* synth.cpp:25-46 */
    const v3 forward = v3_norm(v3_sub(target, pos));
    v3 up = {0, 1, 0};
    if (fabsf(v3_dot(forward, up)) > 0.99f) {
        v3 zz = {0, 0, 1};
        up = zz;
    }
    const v3 right = v3_norm(v3_cross(up, forward));
    const v3 down = v3_cross(forward, right);
    cam->position[0] = pos.x;
    cam->position[1] = pos.y;
    cam->position[2] = pos.z;
    cam->rotation[0] = right.x;
    cam->rotation[1] = right.y;
    cam->rotation[2] = right.z;
    cam->rotation[3] = down.x;
    cam->rotation[4] = down.y;
    cam->rotation[5] = down.z;
    cam->rotation[6] = forward.x;
    cam->rotation[7] = forward.y;
    cam->rotation[8] = forward.z;
    cam->fx = fx;
    cam->fy = fy;
    cam->width = w;
    cam->height = h;
}

static void arc_cameras(rng_t* rng, int count, int w, int h, float fx, float fy,
                        float radius, float span, ago_camera* cams) {
    /* synth.cpp:48-63 */
    for (int i = 0; i < count; ++i) {
        const float t = count > 1 ? (float)i / (float)(count - 1) : 0.5f;
        const float theta = (t - 0.5f) * span;
        const float y = rng_uniform(rng, -1.5f, 1.5f);
        v3 pos = {radius * sinf(theta), y, -radius * cosf(theta)};
        v3 origin = {0, 0, 0};
        look_at(pos, origin, fx, fy, w, h, &cams[i]);
    }
}

static void slab_gaussian(rng_t* rng, soa_out* o, float hx, float hy, float zc,
                          float zt, float s_lo, float s_hi, float o_lo,
                          float o_hi) { /* synth.cpp:65-80 */
    v3 mean, scale;
    mean.x = rng_uniform(rng, -hx, hx);
    mean.y = rng_uniform(rng, -hy, hy);
    mean.z = zc + rng_uniform(rng, -zt, zt);
    scale.x = rng_uniform(rng, s_lo, s_hi);
    scale.y = rng_uniform(rng, s_lo, s_hi);
    scale.z = rng_uniform(rng, 0.05f, 0.15f);
    const quat q = random_rotation(rng);
    const float op = rng_uniform(rng, o_lo, o_hi);
    float r, g, b;
    draw_rgb(rng, &r, &g, &b);
    put_gaussian(o, mean, scale, q, op, r, g, b);
}

/* Curtain / wall Gaussians shared by two_slab and veil (synth.cpp:105-183). */
static void sheet_gaussian(rng_t* rng, soa_out* o, int rear, float spacing,
                           float s_lo, float s_hi, float o_lo, float o_hi) {
    v3 mean, scale;
    if (!rear) {
        mean.x = rng_uniform(rng, -10.0f, 10.0f);
        mean.y = rng_uniform(rng, -7.0f, 7.0f);
        mean.z = rng_uniform(rng, -0.2f, 0.2f);
    } else {
        mean.x = rng_uniform(rng, -6.0f, 6.0f);
        mean.y = rng_uniform(rng, -4.0f, 4.0f);
        mean.z = 20.0f + rng_uniform(rng, -0.2f, 0.2f);
    }
    const float s = spacing * rng_uniform(rng, s_lo, s_hi);
    scale.x = s;
    scale.y = s * rng_uniform(rng, 0.8f, 1.2f);
    scale.z = 0.1f * s;
    const quat q = small_rotation(rng, 0.2f);
    const float op = rng_uniform(rng, o_lo, o_hi);
    float r, g, b;
    draw_rgb(rng, &r, &g, &b);
    put_gaussian(o, mean, scale, q, op, r, g, b);
}

int ago_synth_scene(uint64_t seed, int32_t count, const char* layout,
                    int32_t camera_count, int32_t width, int32_t height,
                    float fx, float fy, float* mean, float* scale,
                    float* rotation, float* opacity, float* sh,
                    ago_camera* cameras) {
    if (count < 1) return AGO_EINVAL;
    rng_t rng;
    rng_init(&rng, seed, 0);
    soa_out o = {mean, scale, rotation, opacity, sh, 0};
    if (strcmp(layout, "slab") == 0) { /* synth.cpp:82-93 */
        const int front = (count * 3 + 2) / 5;
        for (int i = 0; i < front; ++i)
            slab_gaussian(&rng, &o, 8, 6, 0.0f, 0.3f, 0.15f, 0.45f, 0.7f, 0.97f);
        for (int i = front; i < count; ++i)
            slab_gaussian(&rng, &o, 14, 10, 15.0f, 0.3f, 0.3f, 0.8f, 0.4f, 0.9f);
        arc_cameras(&rng, camera_count, width, height, fx, fy, 24.0f, 1.2f, cameras);
    } else if (strcmp(layout, "two_slab") == 0 || strcmp(layout, "veil") == 0) {
        const int veil = strcmp(layout, "veil") == 0;
        const int front = veil ? (count * 35 + 50) / 100 : count / 2;
        const int rear = count - front;
        const float fsp = sqrtf(20.0f * 14.0f / (float)maxi_(front, 1));
        const float rsp = sqrtf(12.0f * 8.0f / (float)maxi_(rear, 1));
        for (int i = 0; i < front; ++i)
            sheet_gaussian(&rng, &o, 0, fsp, 1.1f, 1.8f, 0.85f, 0.98f);
        for (int i = 0; i < rear; ++i) {
            if (veil)
                sheet_gaussian(&rng, &o, 1, rsp, 8.0f, 14.0f, 0.6f, 0.95f);
            else
                sheet_gaussian(&rng, &o, 1, rsp, 0.9f, 1.5f, 0.5f, 0.95f);
        }
        arc_cameras(&rng, camera_count, width, height, fx, fy, 22.0f, 1.1f, cameras);
    } else if (strcmp(layout, "ramp") == 0) { /* synth.cpp:185-220 */
        const float half_w = 0.5f * (float)width / fx;
        const float half_h = 0.5f * (float)height / fy;
        for (int i = 0; i < count; ++i) {
            const float z = rng_uniform(&rng, 3.0f, 92.0f);
            v3 m, sc;
            m.x = rng_uniform(&rng, -0.8f, 0.8f) * half_w * z;
            m.y = rng_uniform(&rng, -0.8f, 0.8f) * half_h * z;
            m.z = z;
            const float s = z * rng_uniform(&rng, 0.010f, 0.022f);
            sc.x = s * rng_uniform(&rng, 0.6f, 1.4f);
            sc.y = s * rng_uniform(&rng, 0.6f, 1.4f);
            sc.z = s * rng_uniform(&rng, 0.6f, 1.4f);
            const quat q = random_rotation(&rng);
            const float op = rng_uniform(&rng, 0.3f, 0.95f);
            float r, g, b;
            draw_rgb(&rng, &r, &g, &b);
            put_gaussian(&o, m, sc, q, op, r, g, b);
        }
        for (int i = 0; i < camera_count; ++i) {
            ago_camera* c = &cameras[i];
            memset(c, 0, sizeof(*c));
            c->position[0] = rng_uniform(&rng, -0.4f, 0.4f);
            c->position[1] = rng_uniform(&rng, -0.3f, 0.3f);
            c->position[2] = rng_uniform(&rng, -0.8f, 0.0f);
            c->rotation[0] = c->rotation[4] = c->rotation[8] = 1.0f;
            c->fx = fx;
            c->fy = fy;
            c->width = width;
            c->height = height;
        }
    } else if (strcmp(layout, "aniso") == 0) { /* synth.cpp:222-240 */
        for (int i = 0; i < count; ++i) {
            v3 m, sc;
            m.x = rng_uniform(&rng, -10.0f, 10.0f);
            m.y = rng_uniform(&rng, -7.0f, 7.0f);
            m.z = rng_uniform(&rng, -4.0f, 4.0f);
            const float major = rng_uniform(&rng, 0.5f, 1.2f);
            sc.x = major;
            sc.y = major * rng_uniform(&rng, 0.08f, 0.25f);
            sc.z = rng_uniform(&rng, 0.05f, 0.15f);
            const quat q = random_rotation(&rng);
            const float op = rng_uniform(&rng, 0.35f, 0.95f);
            float r, g, b;
            draw_rgb(&rng, &r, &g, &b);
            put_gaussian(&o, m, sc, q, op, r, g, b);
        }
        arc_cameras(&rng, camera_count, width, height, fx, fy, 26.0f, 1.2f, cameras);
    } else {
        return AGO_EINVAL;
    }
    return AGO_OK;
}

/* ------------------------------------------------------------------ */
/* Config / camera validation (scene.cpp:41-59, 113-123). */
void ago_default_config(ago_config* c) {
    memset(c, 0, sizeof(*c));
    c->tile_size = 16;
    c->alpha_threshold = 1.0f / 255.0f;
    c->transmittance_floor = 1e-4f;
    c->alpha_clamp = 0.99f;
    c->near_plane = 0.2f;
    c->guard_band = 1.3f;
    c->mode = AGO_ELLIPSE;
    c->k = 0.0f;
    c->thread_count = 0;
    c->fixed_radius_aabb = 0;
    c->pair_budget = (uint64_t)1 << 27;
}

static int cfg_valid(const ago_config* c) {
    if (!(c->alpha_threshold > 0.0f && c->alpha_threshold < c->alpha_clamp &&
          c->alpha_clamp <= 1.0f))
        return 0;
    if (!(c->transmittance_floor > 0.0f)) return 0;
    if (c->tile_size < 1) return 0;
    if (c->k < 0.0f) return 0;
    if (!(c->near_plane > 0.0f)) return 0;
    return 1;
}

static int cam_valid(const ago_camera* c) {
    const float* r = c->rotation;
    float drift = 0.0f;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            float s = 0.0f; /* (R^T R)(i,j), Mat3 product math.hpp:50-59 */
            for (int k = 0; k < 3; ++k) s += r[k * 3 + i] * r[k * 3 + j];
            const float target = (i == j) ? 1.0f : 0.0f;
            drift = maxf_(drift, fabsf(s - target));
        }
    if (drift > 1e-5f) return 0;
    if (!(c->fx > 0.0f && c->fy > 0.0f)) return 0;
    if (!(c->width > 0 && c->height > 0)) return 0;
    return 1;
}

/* ------------------------------------------------------------------ */
/* Preprocess (preprocess.cpp). */
static const float kShC1 = 0.4886025119029199f;
static const float kShC2[5] = {1.0925484305920792f, -1.0925484305920792f,
                               0.31539156525252005f, -1.0925484305920792f,
                               0.5462742152960396f};
static const float kShC3[7] = {-0.5900435899266435f, 2.890611442640554f,
                               -0.4570457994644658f, 0.3731763325901154f,
                               -0.4570457994644658f, 1.445305721320277f,
                               -0.5900435899266435f};

/* x86-64 cvttss2si: NaN and out-of-range floats become INT_MIN.  The
 * reference relies on static_cast<int> compiled for x86-64. */
static inline int f2i_x86(float v) {
    if (!(v > -2147483904.0f && v < 2147483648.0f)) return (int)0x80000000u;
    return (int)v;
}

static float lut_value(const ago_lut* lut, float depth) { /* lut.hpp:16-25 */
    static const float ones = 1.0f;
    float dmin = 0.0f, dmax = 100.0f;
    int nb = 20;
    const float* bins = NULL;
    if (lut && lut->bin_count > 0) {
        dmin = lut->depth_min;
        dmax = lut->depth_max;
        nb = lut->bin_count;
        bins = lut->bins;
    }
    const float w = (dmax - dmin) / (float)nb;
    int b = f2i_x86((depth - dmin) / w);
    if (b < 0) b = 0;
    if (b >= nb) b = nb - 1;
    return bins ? bins[b] : ones;
}

/* 3x3 double product with the reference's accumulation (math.hpp:50-59). */
static void mat3d_mul(const double* a, const double* b, double* out) {
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            double s = 0;
            for (int k = 0; k < 3; ++k) s += a[r * 3 + k] * b[k * 3 + c];
            out[r * 3 + c] = s;
        }
}

static void transpose3(const double* a, double* out) {
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) out[r * 3 + c] = a[c * 3 + r];
}

/* covariance_3d (scene.cpp:31-39) via rotation_matrix<double> (math.hpp:147-164). */
static void covariance_3d(const float* q, const float* sc, double* cov) {
    const float w = q[0], x = q[1], y = q[2], z = q[3];
    const double n = sqrt((double)w * w + (double)x * x + (double)y * y +
                          (double)z * z);
    const double qw = w / n, qx = x / n, qy = y / n, qz = z / n;
    double r[9];
    r[0] = 1 - 2 * (qy * qy + qz * qz);
    r[1] = 2 * (qx * qy - qw * qz);
    r[2] = 2 * (qx * qz + qw * qy);
    r[3] = 2 * (qx * qy + qw * qz);
    r[4] = 1 - 2 * (qx * qx + qz * qz);
    r[5] = 2 * (qy * qz - qw * qx);
    r[6] = 2 * (qx * qz - qw * qy);
    r[7] = 2 * (qy * qz + qw * qx);
    r[8] = 1 - 2 * (qx * qx + qy * qy);
    for (int row = 0; row < 3; ++row) {
        r[row * 3 + 0] *= sc[0];
        r[row * 3 + 1] *= sc[1];
        r[row * 3 + 2] *= sc[2];
    }
    double rt[9];
    transpose3(r, rt);
    mat3d_mul(r, rt, cov);
}

/* project (preprocess.cpp:26-66).  Returns 0 when culled. */
static int project(const ago_scene* s, uint64_t i, const ago_camera* cam,
                   const ago_config* cfg, float* mean2d, float* cov2d,
                   float* depth) {
    const float* R = cam->rotation;
    const v3 p = {s->mean[3 * i], s->mean[3 * i + 1], s->mean[3 * i + 2]};
    const v3 c = {cam->position[0], cam->position[1], cam->position[2]};
    const v3 d = v3_sub(p, c);
    v3 t; /* Mat3f * Vec3f (math.hpp:43-49) */
    t.x = R[0] * d.x + R[1] * d.y + R[2] * d.z;
    t.y = R[3] * d.x + R[4] * d.y + R[5] * d.z;
    t.z = R[6] * d.x + R[7] * d.y + R[8] * d.z;
    if (t.z <= cfg->near_plane) return 0;

    const float ppx = 0.5f * (float)cam->width, ppy = 0.5f * (float)cam->height;
    const float inv_z = 1.0f / t.z;
    mean2d[0] = cam->fx * t.x * inv_z + ppx;
    mean2d[1] = cam->fy * t.y * inv_z + ppy;
    const float ndc_x = (mean2d[0] - ppx) / ppx;
    const float ndc_y = (mean2d[1] - ppy) / ppy;
    if (fabsf(ndc_x) > cfg->guard_band || fabsf(ndc_y) > cfg->guard_band) return 0;

    const double iz = 1.0 / (double)t.z;
    const double lim_x = cfg->guard_band * 0.5 * cam->width / cam->fx;
    const double lim_y = cfg->guard_band * 0.5 * cam->height / cam->fy;
    const double tx = clampd_(t.x * iz, -lim_x, lim_x) * t.z;
    const double ty = clampd_(t.y * iz, -lim_y, lim_y) * t.z;

    double j[9];
    j[0] = cam->fx * iz;
    j[1] = 0.0;
    j[2] = -cam->fx * tx * iz * iz;
    j[3] = 0.0;
    j[4] = cam->fy * iz;
    j[5] = -cam->fy * ty * iz * iz;
    j[6] = j[7] = j[8] = 0.0;

    double w[9], jw[9], cov[9], tmp[9], jwt[9], sigma[9];
    for (int k = 0; k < 9; ++k) w[k] = R[k];
    mat3d_mul(j, w, jw);
    covariance_3d(&s->rotation[4 * i], &s->scale[3 * i], cov);
    mat3d_mul(jw, cov, tmp);
    transpose3(jw, jwt);
    mat3d_mul(tmp, jwt, sigma);

    cov2d[0] = (float)(sigma[0] + 0.3);
    cov2d[1] = (float)sigma[1];
    cov2d[2] = (float)(sigma[4] + 0.3);
    *depth = t.z;
    return 1;
}

/* eval_color (preprocess.cpp:68-105). */
static void eval_color(const float* sh, int deg, v3 dir, float* rgb) {
    float r = kShC0 * sh[0], g = kShC0 * sh[1], b = kShC0 * sh[2];
#define ACC(W, K)                      \
    do {                               \
        const float w_ = (W);          \
        r += w_ * sh[(K) * 3 + 0];     \
        g += w_ * sh[(K) * 3 + 1];     \
        b += w_ * sh[(K) * 3 + 2];     \
    } while (0)
    if (deg > 0) {
        const float x = dir.x, y = dir.y, z = dir.z;
        ACC(-kShC1 * y, 1);
        ACC(kShC1 * z, 2);
        ACC(-kShC1 * x, 3);
        if (deg > 1) {
            const float xx = x * x, yy = y * y, zz = z * z;
            const float xy = x * y, yz = y * z, xz = x * z;
            ACC(kShC2[0] * xy, 4);
            ACC(kShC2[1] * yz, 5);
            ACC(kShC2[2] * (2.0f * zz - xx - yy), 6);
            ACC(kShC2[3] * xz, 7);
            ACC(kShC2[4] * (xx - yy), 8);
            if (deg > 2) {
                ACC(kShC3[0] * y * (3.0f * xx - yy), 9);
                ACC(kShC3[1] * xy * z, 10);
                ACC(kShC3[2] * y * (4.0f * zz - xx - yy), 11);
                ACC(kShC3[3] * z * (2.0f * zz - 3.0f * xx - 3.0f * yy), 12);
                ACC(kShC3[4] * x * (4.0f * zz - xx - yy), 13);
                ACC(kShC3[5] * z * (xx - yy), 14);
                ACC(kShC3[6] * x * (xx - 3.0f * yy), 15);
            }
        }
    }
#undef ACC
    rgb[0] = clampf_(r + 0.5f, 0.0f, 1.0f);
    rgb[1] = clampf_(g + 0.5f, 0.0f, 1.0f);
    rgb[2] = clampf_(b + 0.5f, 0.0f, 1.0f);
}

static int sh_degree_of(int coeffs) {
    switch (coeffs) {
        case 1: return 0;
        case 4: return 1;
        case 9: return 2;
        case 16: return 3;
        default: return -1;
    }
}

int ago_preprocess(const ago_scene* scene, const ago_camera* cam,
                   const ago_config* cfg, const ago_lut* lut, ago_splat* out,
                   uint64_t* out_count) {
    const int adaptive = cfg->mode == AGO_ADAGSCALE;
    if (adaptive && lut == NULL) return AGO_EINVAL;
    const int deg = sh_degree_of(scene->sh_coeffs);
    if (deg < 0) return AGO_EINVAL;
    const float tau = cfg->alpha_threshold;
    uint64_t n = 0;
    for (uint64_t i = 0; i < scene->count; ++i) {
        float m2[2], c2[3], depth;
        if (!project(scene, i, cam, cfg, m2, c2, &depth)) continue;
        const float det = c2[0] * c2[2] - c2[1] * c2[1];
        if (!(det > 0.0f)) continue;
        float th = tau;
        if (adaptive) { /* compute_th, preprocess.cpp:107-116 */
            const float t_upper = lut_value(lut, depth);
            const float denom = t_upper * 2.0f * 3.14159265358979323846f * sqrtf(det);
            th = cfg->k / denom + tau;
        }
        const float op = scene->opacity[i];
        if (th >= op) continue;
        ago_splat* s = &out[n++];
        s->mean2d[0] = m2[0];
        s->mean2d[1] = m2[1];
        s->cov2d[0] = c2[0];
        s->cov2d[1] = c2[1];
        s->cov2d[2] = c2[2];
        const float inv_det = 1.0f / det; /* SymMat2::inverse, math.hpp:85-88 */
        s->inv_cov[0] = c2[2] * inv_det;
        s->inv_cov[1] = -c2[1] * inv_det;
        s->inv_cov[2] = c2[0] * inv_det;
        s->depth = depth;
        const v3 p = {scene->mean[3 * i], scene->mean[3 * i + 1], scene->mean[3 * i + 2]};
        const v3 c = {cam->position[0], cam->position[1], cam->position[2]};
        eval_color(&scene->sh[3 * scene->sh_coeffs * i], deg,
                   v3_norm(v3_sub(p, c)), s->rgb);
        s->opacity = op;
        s->th = th;
        s->source_id = (uint32_t)i;
    }
    *out_count = n;
    return AGO_OK;
}

/* ------------------------------------------------------------------ */
/* Pair generation (pair_gen.cpp). */
typedef struct { float l1, l2, v1x, v1y, v2x, v2y; } eig2;

static eig2 eigen_sym2(float xx, float xy, float yy) { /* math.hpp:105-131 */
    eig2 e;
    const float mean = 0.5f * (xx + yy);
    const float hd = 0.5f * (xx - yy);
    const float r = sqrtf(hd * hd + xy * xy);
    e.l1 = mean + r;
    e.l2 = mean - r;
    if (xy == 0.0f) {
        if (xx >= yy) {
            e.v1x = 1; e.v1y = 0; e.v2x = 0; e.v2y = 1;
        } else {
            e.v1x = 0; e.v1y = 1; e.v2x = -1; e.v2y = 0;
        }
        return e;
    }
    const float ax = e.l1 - yy, ay = xy;
    const float bx = xy, by = e.l1 - xx;
    const int pick_a = (ax * ax + ay * ay) >= (bx * bx + by * by);
    const float vx = pick_a ? ax : bx, vy = pick_a ? ay : by;
    const float n = sqrtf(vx * vx + vy * vy);
    e.v1x = vx / n;
    e.v1y = vy / n;
    e.v2x = -e.v1y;
    e.v2y = e.v1x;
    return e;
}

typedef struct { float x0, y0, x1, y1; } rectf;

static rectf tile_rect(int ts_i, int width, int height, int tx, int ty) {
    const float ts = (float)ts_i;
    rectf r;
    r.x0 = tx * ts;
    r.y0 = ty * ts;
    r.x1 = minf_(r.x0 + ts, (float)width);
    r.y1 = minf_(r.y0 + ts, (float)height);
    return r;
}

static int box_overlap(rectf t, float cx, float cy, float rx, float ry) {
    return t.x0 <= cx + rx && cx - rx <= t.x1 && t.y0 <= cy + ry && cy - ry <= t.y1;
}

static float quad(float xx, float xy, float yy, float dx, float dy) {
    return xx * dx * dx + 2.0f * xy * dx * dy + yy * dy * dy; /* math.hpp:91-93 */
}

static float min_quad_to_rect(const float* q, float cx, float cy, rectf t) {
    if (cx >= t.x0 && cx <= t.x1 && cy >= t.y0 && cy <= t.y1) return 0.0f;
    float h[2], v[2];
    const float ys[2] = {t.y0, t.y1}, xs[2] = {t.x0, t.x1};
    for (int k = 0; k < 2; ++k) {
        const float dy = ys[k] - cy;
        float x = cx - q[1] * dy / q[0];
        x = clampf_(x, t.x0, t.x1);
        h[k] = quad(q[0], q[1], q[2], x - cx, dy);
        const float dx = xs[k] - cx;
        float y = cy - q[1] * dx / q[2];
        y = clampf_(y, t.y0, t.y1);
        v[k] = quad(q[0], q[1], q[2], dx, y - cy);
    }
    return minf_(minf_(h[0], h[1]), minf_(v[0], v[1]));
}

static int obb_overlap(rectf t, float cx, float cy, float ux, float uy,
                       float vx, float vy, float a, float b) {
    const float rx = a * fabsf(ux) + b * fabsf(vx);
    const float ry = a * fabsf(uy) + b * fabsf(vy);
    if (!box_overlap(t, cx, cy, rx, ry)) return 0;
    const float tcx = 0.5f * (t.x0 + t.x1), tcy = 0.5f * (t.y0 + t.y1);
    const float hw = 0.5f * (t.x1 - t.x0);
    const float hh = 0.5f * (t.y1 - t.y0);
    const float dx = tcx - cx, dy = tcy - cy;
    const float tile_u = hw * fabsf(ux) + hh * fabsf(uy);
    if (fabsf(dx * ux + dy * uy) > a + tile_u) return 0;
    const float tile_v = hw * fabsf(vx) + hh * fabsf(vy);
    if (fabsf(dx * vx + dy * vy) > b + tile_v) return 0;
    return 1;
}

/* intersect_tiles (pair_gen.cpp:108-159).  Calls emit(tile) per hit in
 * ascending row-major order; returns the count. */
typedef struct {
    int tile_size, width, height, tiles_x, tiles_y;
} grid_t;

static grid_t make_grid(int width, int height, int ts) {
    grid_t g = {ts, width, height, (width + ts - 1) / ts, (height + ts - 1) / ts};
    return g;
}

static uint32_t intersect_tiles(const ago_splat* s, const grid_t* g, int mode,
                                const ago_config* cfg, uint64_t* keys,
                                uint32_t* idx, uint32_t splat_i) {
    const float tau = cfg->alpha_threshold;
    const float th = mode == AGO_ADAGSCALE ? s->th : tau;
    const eig2 e = eigen_sym2(s->cov2d[0], s->cov2d[1], s->cov2d[2]);
    float r = sqrtf(2.0f * logf(s->opacity / th));
    if (mode == AGO_AABB && cfg->fixed_radius_aabb) r = 3.0f;
    const float r_px = r * sqrtf(maxf_(e.l1, 0.0f));
    const float cx = s->mean2d[0], cy = s->mean2d[1];
    float rx, ry;
    if (mode == AGO_AABB || mode == AGO_OBB) {
        rx = ry = r_px;
    } else {
        rx = r * sqrtf(maxf_(s->cov2d[0], 0.0f));
        ry = r * sqrtf(maxf_(s->cov2d[2], 0.0f));
    }
    /* tile_span (pair_gen.cpp:41-55) */
    const float ts = (float)g->tile_size;
    const int tx0 = maxi_(0, f2i_x86(floorf((cx - rx) / ts)));
    const int ty0 = maxi_(0, f2i_x86(floorf((cy - ry) / ts)));
    const int tx1 = mini_(g->tiles_x - 1, f2i_x86(floorf((cx + rx) / ts)));
    const int ty1 = mini_(g->tiles_y - 1, f2i_x86(floorf((cy + ry) / ts)));
    const int empty = tx0 > tx1 || ty0 > ty1 || cx + rx < 0.0f || cy + ry < 0.0f ||
                      cx - rx > (float)g->width || cy - ry > (float)g->height;
    if (empty) return 0;
    const float a = r * sqrtf(maxf_(e.l1, 0.0f));
    const float b = r * sqrtf(maxf_(e.l2, 0.0f));
    const float r2 = r * r;
    uint32_t n = 0;
    for (int ty = ty0; ty <= ty1; ++ty)
        for (int tx = tx0; tx <= tx1; ++tx) {
            const rectf t = tile_rect(g->tile_size, g->width, g->height, tx, ty);
            int hit;
            if (mode == AGO_AABB) {
                hit = box_overlap(t, cx, cy, r_px, r_px);
            } else if (mode == AGO_OBB) {
                hit = box_overlap(t, cx, cy, r_px, r_px) &&
                      obb_overlap(t, cx, cy, e.v1x, e.v1y, e.v2x, e.v2y, a, b);
            } else {
                hit = box_overlap(t, cx, cy, rx, ry) &&
                      min_quad_to_rect(s->inv_cov, cx, cy, t) <= r2;
            }
            if (!hit) continue;
            if (keys) {
                uint32_t bits;
                memcpy(&bits, &s->depth, 4);
                const uint32_t tile = (uint32_t)(ty * g->tiles_x + tx);
                keys[n] = ((uint64_t)tile << 32) | bits; /* pack_pair_key */
                idx[n] = splat_i;
            }
            ++n;
        }
    return n;
}

int ago_generate_pairs(const ago_splat* splats, uint64_t n, int32_t width,
                       int32_t height, int32_t mode, const ago_config* cfg,
                       uint64_t* keys, uint32_t* splat_index,
                       uint64_t capacity, uint32_t* tile_counts,
                       uint64_t* out_total) {
    const grid_t g = make_grid(width, height, cfg->tile_size);
    uint64_t total = 0;
    for (uint64_t i = 0; i < n; ++i) {
        tile_counts[i] = intersect_tiles(&splats[i], &g, mode, cfg, NULL, NULL, 0);
        total += tile_counts[i];
    }
    *out_total = total;
    if (total > cfg->pair_budget) return AGO_EPAIR_BUDGET;
    if (total > capacity) return AGO_ECAPACITY;
    uint64_t at = 0;
    for (uint64_t i = 0; i < n; ++i)
        at += intersect_tiles(&splats[i], &g, mode, cfg, keys + at,
                              splat_index + at, (uint32_t)i);
    return AGO_OK;
}

/* ------------------------------------------------------------------ */
/* Sort (pair_sort.cpp:7-44): stable LSD, 8 x 8-bit digits. */
int ago_sort_pairs(uint64_t* keys, uint32_t* splat_index, uint64_t n,
                   int32_t tile_count, uint32_t* ranges) {
    uint64_t* k2 = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    uint32_t* v2 = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
    if (!k2 || !v2) {
        free(k2);
        free(v2);
        return AGO_EINVAL;
    }
    uint64_t *sk = keys, *dk = k2;
    uint32_t *sv = splat_index, *dv = v2;
    for (int pass = 0; pass < 8; ++pass) {
        const int shift = pass * 8;
        uint64_t cnt[256];
        memset(cnt, 0, sizeof(cnt));
        for (uint64_t i = 0; i < n; ++i) ++cnt[(sk[i] >> shift) & 0xFF];
        uint64_t sum = 0;
        for (int d = 0; d < 256; ++d) {
            const uint64_t c = cnt[d];
            cnt[d] = sum;
            sum += c;
        }
        for (uint64_t i = 0; i < n; ++i) {
            const uint64_t at = cnt[(sk[i] >> shift) & 0xFF]++;
            dk[at] = sk[i];
            dv[at] = sv[i];
        }
        uint64_t* tk = sk; sk = dk; dk = tk;
        uint32_t* tv = sv; sv = dv; dv = tv;
    }
    /* eight passes land the data back in the caller's buffers */
    free(k2);
    free(v2);
    memset(ranges, 0, sizeof(uint32_t) * 2 * (size_t)tile_count);
    uint64_t i = 0;
    while (i < n) {
        const uint32_t tile = (uint32_t)(keys[i] >> 32);
        uint64_t j = i + 1;
        while (j < n && (uint32_t)(keys[j] >> 32) == tile) ++j;
        if (tile < (uint32_t)tile_count) {
            ranges[2 * tile] = (uint32_t)i;
            ranges[2 * tile + 1] = (uint32_t)j;
        }
        i = j;
    }
    return AGO_OK;
}

/* ------------------------------------------------------------------ */
/* Raster (rasterizer.hpp:44-50, rasterizer.cpp:21-100). */
static float alpha_at(const ago_splat* s, float px, float py, float clamp) {
    const float dx = px - s->mean2d[0], dy = py - s->mean2d[1];
    const float power = -0.5f * quad(s->inv_cov[0], s->inv_cov[1], s->inv_cov[2], dx, dy);
    if (power > 0.0f) return 0.0f;
    const float a = s->opacity * expf(power);
    return a < clamp ? a : clamp;
}

/* Blend-event sink of raster_tile (RecordOptions::contributions). */
typedef struct {
    ago_blend* out;
    uint64_t capacity, count;
} blend_sink;

static void raster_tile(const ago_splat* splats, const uint32_t* idx,
                        uint32_t begin, uint32_t end, const grid_t* g, int tile,
                        const ago_config* cfg, float* image, float* max_t, blend_sink* sink,
                        uint64_t* p_it) {
    const int tx = tile % g->tiles_x, ty = tile / g->tiles_x;
    const int x0 = tx * g->tile_size, y0 = ty * g->tile_size;
    const int w = mini_(g->tile_size, g->width - x0);
    const int h = mini_(g->tile_size, g->height - y0);
    const int npx = w * h;
    if (npx <= 0) return;
    float* T = (float*)malloc(sizeof(float) * (size_t)npx);
    float* C = (float*)calloc((size_t)npx * 3, sizeof(float));
    for (int i = 0; i < npx; ++i) T[i] = 1.0f;
    const float tau = cfg->alpha_threshold, fl = cfg->transmittance_floor;
    int active = npx;
    for (uint32_t p = begin; p < end; ++p) {
        if (active == 0) break;
        if (p_it) ++*p_it; /* pairs the tile loop visits (rasterizer.cpp:55-56) */
        const ago_splat* s = &splats[idx[p]];
        for (int iy = 0; iy < h; ++iy) {
            const float py = (float)(y0 + iy) + 0.5f;
            for (int ix = 0; ix < w; ++ix) {
                const int pi = iy * w + ix;
                const float t_cur = T[pi];
                if (t_cur < fl) continue;
                const float px = (float)(x0 + ix) + 0.5f;
                const float a = alpha_at(s, px, py, cfg->alpha_clamp);
                if (a < tau) continue;
                if (max_t && t_cur > max_t[idx[p]]) max_t[idx[p]] = t_cur;
                const float weight = a * t_cur;
                if (sink) { /* rasterizer.cpp:73-77 */
                    if (sink->count < sink->capacity) {
                        ago_blend* r = &sink->out[sink->count];
                        r->pixel = (uint32_t)((y0 + iy) * g->width + (x0 + ix));
                        r->splat = idx[p];
                        r->alpha = a;
                        r->weight = weight;
                    }
                    ++sink->count;
                }
                C[pi * 3 + 0] += weight * s->rgb[0];
                C[pi * 3 + 1] += weight * s->rgb[1];
                C[pi * 3 + 2] += weight * s->rgb[2];
                const float t_next = t_cur * (1.0f - a);
                T[pi] = t_next;
                if (t_next < fl) --active;
            }
        }
    }
    for (int iy = 0; iy < h; ++iy)
        for (int ix = 0; ix < w; ++ix) {
            const int pi = iy * w + ix;
            float* o = &image[((size_t)(y0 + iy) * g->width + (x0 + ix)) * 3];
            for (int c = 0; c < 3; ++c)
                o[c] = clampf_(C[pi * 3 + c] + T[pi] * cfg->background[c], 0.0f, 1.0f);
        }
    free(T);
    free(C);
}

static void raster_all(const ago_splat* splats, uint64_t n_splats, const uint32_t* splat_index,
                       const uint32_t* ranges, int32_t width, int32_t height, const ago_config* cfg,
                       float* image, float* max_t, blend_sink* sink, uint64_t* p_it) {
    const grid_t g = make_grid(width, height, cfg->tile_size);
    if (max_t) memset(max_t, 0, sizeof(float) * n_splats);
    memset(image, 0, sizeof(float) * 3 * (size_t)width * height);
    for (int t = 0; t < g.tiles_x * g.tiles_y; ++t) /* tile-index order (rasterizer.cpp:155-161) */
        raster_tile(splats, splat_index, ranges[2 * t], ranges[2 * t + 1], &g, t,
                    cfg, image, max_t, sink, p_it);
}

int ago_raster(const ago_splat* splats, uint64_t n_splats,
               const uint64_t* keys, const uint32_t* splat_index,
               uint64_t n_pairs, const uint32_t* ranges, int32_t width,
               int32_t height, const ago_config* cfg, float* image,
               float* max_t) {
    (void)keys;
    (void)n_pairs;
    raster_all(splats, n_splats, splat_index, ranges, width, height, cfg, image, max_t, NULL, NULL);
    return AGO_OK;
}

/* P_it: the pairs raster_tile visits before every pixel of its tile is
 * saturated (the `active == 0` break, rasterizer.cpp:55-56), summed over the
 * tiles -- the raster's work measure. */
int ago_raster_pit(const ago_splat* splats, uint64_t n_splats, const uint32_t* splat_index,
                   const uint32_t* ranges, int32_t width, int32_t height, const ago_config* cfg,
                   float* image, uint64_t* p_it) {
    *p_it = 0;
    raster_all(splats, n_splats, splat_index, ranges, width, height, cfg, image, NULL, NULL, p_it);
    return AGO_OK;
}

/* ------------------------------------------------------------------ */
static int render_impl(const ago_scene* scene, const ago_camera* cam,
                       const ago_config* cfg, const ago_lut* lut, float* image,
                       uint64_t* pair_count, uint64_t* splat_count, float* max_t,
                       double* stage_s, blend_sink* sink) {
    if (!cfg_valid(cfg) || !cam_valid(cam)) return AGO_EINVAL;
    static const float ones20[20] = {1, 1, 1, 1, 1, 1, 1, 1, 1, 1,
                                     1, 1, 1, 1, 1, 1, 1, 1, 1, 1};
    ago_lut default_lut = {0.0f, 100.0f, 20, ones20};
    if (cfg->mode == AGO_ADAGSCALE && lut == NULL) lut = &default_lut;
    ago_splat* splats = (ago_splat*)malloc(sizeof(ago_splat) * (scene->count ? scene->count : 1));
    uint64_t ns = 0;
    int rc = ago_preprocess(scene, cam, cfg, lut, splats, &ns);
    if (rc) { free(splats); return rc; }
    const grid_t g = make_grid(cam->width, cam->height, cfg->tile_size);
    uint32_t* counts = (uint32_t*)malloc(sizeof(uint32_t) * (ns ? ns : 1));
    uint64_t total = 0;
    rc = ago_generate_pairs(splats, ns, cam->width, cam->height, cfg->mode, cfg,
                            NULL, NULL, 0, counts, &total);
    if (rc == AGO_EPAIR_BUDGET) { free(splats); free(counts); return rc; }
    uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (total ? total : 1));
    uint32_t* idx = (uint32_t*)malloc(sizeof(uint32_t) * (total ? total : 1));
    rc = ago_generate_pairs(splats, ns, cam->width, cam->height, cfg->mode, cfg,
                            keys, idx, total, counts, &total);
    uint32_t* ranges = (uint32_t*)malloc(sizeof(uint32_t) * 2 * (size_t)g.tiles_x * g.tiles_y);
    ago_sort_pairs(keys, idx, total, g.tiles_x * g.tiles_y, ranges);
    raster_all(splats, ns, idx, ranges, cam->width, cam->height, cfg, image, max_t, sink, NULL);
    *pair_count = total;
    *splat_count = ns;
    if (stage_s) stage_s[0] = stage_s[1] = stage_s[2] = stage_s[3] = 0.0;
    free(splats);
    free(counts);
    free(keys);
    free(idx);
    free(ranges);
    return AGO_OK;
}

int ago_render(const ago_scene* scene, const ago_camera* cam,
               const ago_config* cfg, const ago_lut* lut, float* image,
               uint64_t* pair_count, uint64_t* splat_count, float* max_t,
               double* stage_s) {
    return render_impl(scene, cam, cfg, lut, image, pair_count, splat_count, max_t, stage_s, NULL);
}

int ago_render_contributions(const ago_scene* scene, const ago_camera* cam, const ago_config* cfg,
                             const ago_lut* lut, float* image, ago_blend* out, uint64_t capacity,
                             uint64_t* count) {
    blend_sink sink = {out, out ? capacity : 0, 0};
    uint64_t pc = 0, sc = 0;
    const int rc = render_impl(scene, cam, cfg, lut, image, &pc, &sc, NULL, NULL, &sink);
    if (rc) return rc;
    *count = sink.count;
    return sink.count > sink.capacity ? AGO_ECAPACITY : AGO_OK;
}

double ago_psnr(const float* a, const float* b, uint64_t n) {
    double se = 0.0; /* analysis.cpp:14-25 */
    for (uint64_t i = 0; i < n; ++i) {
        const double d = (double)a[i] - b[i];
        se += d * d;
    }
    if (se == 0.0) return INFINITY;
    const double mse = se / (double)n;
    return 10.0 * log10(1.0 / mse);
}

void ago_logf_batch(const float* x, float* y, uint64_t n) {
    for (uint64_t i = 0; i < n; ++i) y[i] = logf(x[i]);
}

void ago_expf_batch(const float* x, float* y, uint64_t n) {
    for (uint64_t i = 0; i < n; ++i) y[i] = expf(x[i]);
}

const char* ago_kind(void) { return "port"; }

// ags_io.cpp -- scene ingest (next row f2): binary 3DGS PLY -> scene arrays
// ready for agsx_scene_upload, orbit cameras, PPM frame output.
//
//   reference: load_ply        gsio.cpp:80-152 (header gsio.cpp:27-76)
//              orbit_cameras   synth.cpp:254-281 (look_at synth.cpp:24-46)
//              write_image     gsio.cpp:265-281
//
// Values are decoded exactly as the reference does (double sigmoid / exp of
// the float fields via the host libm, float quaternion normalisation), so a
// loaded scene is byte-identical to the reference's.  load_ply_soa decodes
// the vertex block with one host thread per slice straight into the SoA
// arrays the device upload takes; rows with non-finite fields are dropped in
// file order like the reference.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <istream>
#include <map>
#include <sstream>
#include <thread>

#include "ags/ags.hpp"

namespace ags {

namespace {

double sigmoid(double x) { return 1.0 / (1.0 + std::exp(-x)); }

int degree_for_rest_count(int rest) {
    for (int d = 1; d <= 4; ++d)
        if (rest == 3 * (d * d - 1)) return d - 1;
    return -1;
}

struct PlyLayout {
    std::size_t vertex_count = 0;
    std::vector<std::string> properties;
    int cx, cy, cz, cop, cs[3], cr[4], cdc[3];
    std::vector<int> crest;
    int coeffs = 1;
};

PlyLayout parse_header(std::istream& in) {
    PlyLayout h;
    std::string line;
    if (!std::getline(in, line) || line != "ply") throw IoError("ply: missing magic line");
    if (!std::getline(in, line) || line != "format binary_little_endian 1.0")
        throw IoError("ply: expected 'format binary_little_endian 1.0'");
    bool in_vertex = false, seen_vertex = false, done = false;
    while (std::getline(in, line)) {
        if (line == "end_header") {
            if (!seen_vertex) throw IoError("ply: no vertex element");
            done = true;
            break;
        }
        std::istringstream ls(line);
        std::string tok;
        ls >> tok;
        if (tok == "comment") continue;
        if (tok == "element") {
            std::string name;
            std::size_t count = 0;
            ls >> name >> count;
            in_vertex = name == "vertex";
            if (in_vertex) {
                h.vertex_count = count;
                seen_vertex = true;
            }
            continue;
        }
        if (tok == "property") {
            if (!in_vertex) continue;
            std::string type, name;
            ls >> type >> name;
            if (type != "float") throw IoError("ply: vertex property '" + name + "' has unsupported type '" + type + "'");
            h.properties.push_back(name);
            continue;
        }
        throw IoError("ply: unexpected header line '" + line + "'");
    }
    if (!done) throw IoError("ply: header not terminated");
    std::map<std::string, int> col;
    for (std::size_t i = 0; i < h.properties.size(); ++i) col[h.properties[i]] = static_cast<int>(i);
    auto require = [&](const std::string& name) {
        auto it = col.find(name);
        if (it == col.end()) throw IoError("ply: missing property '" + name + "'");
        return it->second;
    };
    h.cx = require("x");
    h.cy = require("y");
    h.cz = require("z");
    h.cop = require("opacity");
    for (int i = 0; i < 3; ++i) h.cs[i] = require("scale_" + std::to_string(i));
    for (int i = 0; i < 4; ++i) h.cr[i] = require("rot_" + std::to_string(i));
    for (int i = 0; i < 3; ++i) h.cdc[i] = require("f_dc_" + std::to_string(i));
    int rest = 0;
    while (col.count("f_rest_" + std::to_string(rest))) ++rest;
    const int degree = degree_for_rest_count(rest);
    if (degree < 0) throw IoError("ply: unsupported f_rest count " + std::to_string(rest));
    for (int i = 0; i < rest; ++i) h.crest.push_back(col["f_rest_" + std::to_string(i)]);
    h.coeffs = (degree + 1) * (degree + 1);
    return h;
}

bool row_finite(const float* row, std::size_t stride) {
    for (std::size_t i = 0; i < stride; ++i)
        if (!std::isfinite(row[i])) return false;
    return true;
}

// One row -> the reference's Gaussian3D fields (gsio.cpp:128-147).
void decode_row(const PlyLayout& h, const float* row, float* mean, float* scale, float* rot, float* op, float* sh) {
    mean[0] = row[h.cx];
    mean[1] = row[h.cy];
    mean[2] = row[h.cz];
    *op = static_cast<float>(sigmoid(row[h.cop]));
    for (int i = 0; i < 3; ++i) scale[i] = static_cast<float>(std::exp(static_cast<double>(row[h.cs[i]])));
    const Quatf q = Quatf{row[h.cr[0]], row[h.cr[1]], row[h.cr[2]], row[h.cr[3]]}.normalized();
    rot[0] = q.w;
    rot[1] = q.x;
    rot[2] = q.y;
    rot[3] = q.z;
    const int per_channel = h.coeffs - 1;
    std::fill(sh, sh + 3 * h.coeffs, 0.0f);
    sh[0] = row[h.cdc[0]];
    sh[1] = row[h.cdc[1]];
    sh[2] = row[h.cdc[2]];
    for (int c = 0; c < 3; ++c)
        for (int k = 1; k < h.coeffs; ++k) sh[k * 3 + c] = row[h.crest[c * per_channel + (k - 1)]];
}

Camera look_at(Vec3f pos, Vec3f target, float fx, float fy, int w, int hgt) {
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
    c.fx = fx;
    c.fy = fy;
    c.width = w;
    c.height = hgt;
    return c;
}

}  // namespace

PlyLoadResult load_ply(std::istream& in) {
    const PlyLayout h = parse_header(in);
    const std::size_t stride = h.properties.size();
    std::vector<float> row(stride);
    PlyLoadResult out;
    out.gaussians.reserve(h.vertex_count);
    for (std::size_t e = 0; e < h.vertex_count; ++e) {
        in.read(reinterpret_cast<char*>(row.data()), static_cast<std::streamsize>(stride * sizeof(float)));
        if (!in) throw IoError("ply: truncated element data");
        if (!row_finite(row.data(), stride)) {
            ++out.rejected;
            continue;
        }
        Gaussian3D g;
        float m[3], s[3], r[4], op;
        g.sh.assign(static_cast<std::size_t>(h.coeffs) * 3, 0.0f);
        decode_row(h, row.data(), m, s, r, &op, g.sh.data());
        g.mean = {m[0], m[1], m[2]};
        g.scale = {s[0], s[1], s[2]};
        g.rotation = Quatf{r[0], r[1], r[2], r[3]};
        g.opacity = op;
        out.gaussians.push_back(std::move(g));
    }
    return out;
}

PlyLoadResult load_ply_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open '" + path + "'");
    return load_ply(in);
}

PlySoA load_ply_soa(const std::string& path, int threads) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open '" + path + "'");
    const PlyLayout h = parse_header(in);
    const std::size_t stride = h.properties.size();
    const std::size_t n = h.vertex_count;
    std::vector<float> raw(n * stride);
    in.read(reinterpret_cast<char*>(raw.data()), static_cast<std::streamsize>(raw.size() * sizeof(float)));
    if (!in) throw IoError("ply: truncated element data");

    unsigned t = threads > 0 ? static_cast<unsigned>(threads) : std::max(1u, std::thread::hardware_concurrency());
    t = static_cast<unsigned>(std::max<std::size_t>(1, std::min<std::size_t>(t, n / 4096 + 1)));
    std::vector<std::size_t> lo(t + 1), kept(t, 0);
    for (unsigned i = 0; i <= t; ++i) lo[i] = n * i / t;
    auto run = [&](auto&& body) {
        std::vector<std::thread> pool;
        for (unsigned i = 0; i < t; ++i) pool.emplace_back(body, i);
        for (auto& th : pool) th.join();
    };
    run([&](unsigned i) {  // pass 1: finite rows per slice
        for (std::size_t e = lo[i]; e < lo[i + 1]; ++e) kept[i] += row_finite(&raw[e * stride], stride);
    });
    std::vector<std::size_t> base(t + 1, 0);
    for (unsigned i = 0; i < t; ++i) base[i + 1] = base[i] + kept[i];
    PlySoA out;
    out.count = base[t];
    out.rejected = n - base[t];
    out.sh_coeffs = h.coeffs;
    out.mean.resize(3 * out.count);
    out.scale.resize(3 * out.count);
    out.rotation.resize(4 * out.count);
    out.opacity.resize(out.count);
    out.sh.resize(static_cast<std::size_t>(3 * h.coeffs) * out.count);
    run([&](unsigned i) {  // pass 2: decode in file order
        std::size_t j = base[i];
        for (std::size_t e = lo[i]; e < lo[i + 1]; ++e) {
            const float* row = &raw[e * stride];
            if (!row_finite(row, stride)) continue;
            decode_row(h, row, &out.mean[3 * j], &out.scale[3 * j], &out.rotation[4 * j], &out.opacity[j],
                       &out.sh[static_cast<std::size_t>(3 * h.coeffs) * j]);
            ++j;
        }
    });
    return out;
}

std::vector<Camera> orbit_cameras(const float* mean, std::uint64_t n, int count, int width, int height, float fx,
                                  float fy, std::uint64_t seed) {
    Vec3f lo{0, 0, 0}, hi{0, 0, 0};
    if (n) lo = hi = Vec3f{mean[0], mean[1], mean[2]};
    for (std::uint64_t i = 0; i < n; ++i) {
        const Vec3f m{mean[3 * i], mean[3 * i + 1], mean[3 * i + 2]};
        lo = {std::min(lo.x, m.x), std::min(lo.y, m.y), std::min(lo.z, m.z)};
        hi = {std::max(hi.x, m.x), std::max(hi.y, m.y), std::max(hi.z, m.z)};
    }
    const Vec3f center = (lo + hi) * 0.5f;
    const float radius = std::max(1.0f, (hi - lo).norm());
    Rng rng(seed);
    std::vector<Camera> cams;
    cams.reserve(std::max(count, 0));
    for (int i = 0; i < count; ++i) {
        const float theta = count > 1 ? (static_cast<float>(i) / count) * 6.2831853f : 0.0f;
        const float x = radius * 2.0f * std::sin(theta);
        const float y = rng.uniform(-0.1f, 0.1f) * radius;
        const float z = -radius * 2.0f * std::cos(theta);
        cams.push_back(look_at(center + Vec3f{x, y, z}, center, fx, fy, width, height));
    }
    return cams;
}

std::vector<Camera> orbit_cameras(const std::vector<Gaussian3D>& gaussians, int count, int width, int height,
                                  float fx, float fy, std::uint64_t seed) {
    std::vector<float> mean(3 * gaussians.size());
    for (std::size_t i = 0; i < gaussians.size(); ++i) {
        mean[3 * i] = gaussians[i].mean.x;
        mean[3 * i + 1] = gaussians[i].mean.y;
        mean[3 * i + 2] = gaussians[i].mean.z;
    }
    return orbit_cameras(mean.data(), gaussians.size(), count, width, height, fx, fy, seed);
}

void write_image(const Image& img, const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("cannot open '" + path + "' for writing");
    out << "P6\n" << img.width << " " << img.height << "\n255\n";
    std::vector<unsigned char> px(img.data.size());
    for (std::size_t i = 0; i < px.size(); ++i) {
        const float v = std::clamp(img.data[i], 0.0f, 1.0f);
        px[i] = static_cast<unsigned char>(std::lround(static_cast<double>(v) * 255.0));
    }
    out.write(reinterpret_cast<const char*>(px.data()), static_cast<std::streamsize>(px.size()));
    if (!out) throw IoError("write failure on '" + path + "'");
}

}  // namespace ags

// agsx_stage_api.cu -- C-ABI of libagsx.so: the reference's stage functions
// as separate device passes (preprocess_view, generate_pairs, sort_pairs,
// raster_tile), the calibration primitives (max_t fold, squared error) and
// the libm pinning hooks.
//
//   reference: stage API preprocess.hpp:51-54, pair_gen.hpp:70-72,
//                        pair_sort.hpp:19, rasterizer.hpp:54-58
#include "agsx_ctx.cuh"

// ---- per-element helpers ---------------------------------------------------
namespace agsx::host {
namespace {
// host -> device copy of n floats into a ctx scratch buffer
template <typename T>
T* to_device(agsx_ctx* ctx, Buf& b, const T* src, uint64_t n) {
    ensure(b, std::max<uint64_t>(n, 1) * sizeof(T));
    if (n) AGSX_CUDA(cudaMemcpyAsync(b.p, src, n * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
    return ptr<T>(b);
}
template <typename T>
void to_host(agsx_ctx* ctx, T* dst, const Buf& b, uint64_t n) {
    if (n) AGSX_CUDA(cudaMemcpyAsync(dst, b.p, n * sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
    AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
}
int grid_of(uint64_t n) { return static_cast<int>(std::max<uint64_t>((n + 255) / 256, 1)); }
}  // namespace
}  // namespace agsx::host

extern "C" {

int agsx_preprocess_view(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam,
                         const agsx_config* cfg, const agsx_lut* lut, agsx_splat_view* out,
                         uint64_t* out_count) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        if (const int rc = refuse_if_host_frame(ctx, "preprocess_view")) return rc;
        if (!scene) return fail(ctx, AGSX_EINVAL, "null scene");
        // preprocess_view validates only the LUT requirement (preprocess.cpp:121-125)
        if (cfg->mode == AGSX_MODE_ADAGSCALE && lut == nullptr)
            return fail(ctx, AGSX_EINVAL, "preprocess_view: adagscale mode requires a T-upper LUT");
        agsx_config c = *cfg;
        if (c.tile_size < 1) c.tile_size = 16;
        FrameParams p;
        const float* lut_dev = nullptr;
        if (lut && lut->bin_count > kLutInline) {
            ensure(ctx->lut_ext, lut->bin_count * sizeof(float));
            AGSX_CUDA(cudaMemcpy(ctx->lut_ext.p, lut->bins, lut->bin_count * 4, cudaMemcpyHostToDevice));
            lut_dev = ptr<float>(ctx->lut_ext);
        }
        p = make_params(*cam, c, c.mode == AGSX_MODE_ADAGSCALE ? lut : nullptr, lut_dev);
        const uint64_t n = scene->n;
        const uint64_t tiles = static_cast<uint64_t>(p.tiles_x) * p.tiles_y;
        ensure_frame_buffers(ctx, n, tiles, static_cast<uint64_t>(cam->width) * cam->height,
                             c.mode == AGSX_MODE_OBB, c.pair_budget);
        ensure(ctx->dump, std::max<uint64_t>(n, 1) * sizeof(agsx_splat_view));
        Counters* ctr = ptr<Counters>(ctx->ctr);
        AGSX_CUDA(cudaMemsetAsync(ctr, 0, sizeof(Counters), ctx->stream));
        if (n) {
            k_preprocess<<<static_cast<int>((n + 255) / 256), 256, 0, ctx->stream>>>(
                p, scene->view(), planes_of(ctx), ptr<uint32_t>(ctx->status), ptr<uint32_t>(ctx->dkeys), ctr,
                ptr<agsx_splat_view>(ctx->dump), FrameZero{}, BucketOut{});
            check_launch(ctx);
        }
        std::vector<uint32_t> st(n);  // per Gaussian id (the device array is per storage slot)
        std::vector<agsx_splat_view> sv(n);
        if (n) {
            AGSX_CUDA(cudaMemcpyAsync(sv.data(), ctx->dump.p, n * sizeof(agsx_splat_view),
                                      cudaMemcpyDeviceToHost, ctx->stream));
            slots_to_ids_host(scene, ctx->status.p, st.data(), ctx->stream);
        }
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        uint64_t m = 0;
        for (uint64_t i = 0; i < n; ++i)
            if (st[i] & kAliveBit) out[m++] = sv[i];
        *out_count = m;
        ctx->have_frame = false;
        return AGSX_OK;
    });
}

int agsx_generate_pairs(agsx_ctx* ctx, const agsx_splat_view* splats, uint64_t n, int32_t width,
                        int32_t height, int32_t mode, const agsx_config* cfg, uint64_t* keys,
                        uint32_t* splat_index, uint64_t capacity, uint32_t* tile_counts,
                        uint64_t* out_total) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        if (const int rc = refuse_if_host_frame(ctx, "generate_pairs")) return rc;
        if (cfg->tile_size < 1) return fail(ctx, AGSX_EINVAL, "tile_size must be >= 1");
        agsx_config c = *cfg;
        c.mode = mode;
        agsx_camera cam{};
        cam.width = width;
        cam.height = height;
        cam.fx = cam.fy = 1.0f;
        const FrameParams p = make_params(cam, c, nullptr, nullptr);
        ensure(ctx->tmp0, std::max<uint64_t>(n, 1) * sizeof(agsx_splat_view));
        ensure(ctx->tmp1, std::max<uint64_t>(n, 1) * 4);  // counts
        ensure(ctx->tmp2, std::max<uint64_t>(n, 1) * 4);  // depth bits
        ensure(ctx->tmp3, std::max<uint64_t>(n, 1) * 8);  // offsets
        for (Buf* b : {&ctx->p0, &ctx->p1, &ctx->p2, &ctx->p3, &ctx->p4})
            ensure(*b, std::max<uint64_t>(n, 1) * 16);
        const SplatPlanes pl = planes_of(ctx);
        if (n) {
            AGSX_CUDA(cudaMemcpyAsync(ctx->tmp0.p, splats, n * sizeof(agsx_splat_view),
                                      cudaMemcpyHostToDevice, ctx->stream));
            k_splats_to_planes<<<static_cast<int>((n + 255) / 256), 256, 0, ctx->stream>>>(
                p, ptr<agsx_splat_view>(ctx->tmp0), n, pl, ptr<uint32_t>(ctx->tmp1), ptr<uint32_t>(ctx->tmp2));
            check_launch(ctx);
        }
        std::vector<uint32_t> cnt(n);
        if (n) AGSX_CUDA(cudaMemcpyAsync(cnt.data(), ctx->tmp1.p, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        std::vector<uint64_t> off(n);
        uint64_t total = 0;
        for (uint64_t i = 0; i < n; ++i) {
            off[i] = total;
            total += cnt[i];
            if (tile_counts) tile_counts[i] = cnt[i];
        }
        *out_total = total;
        if (total > cfg->pair_budget)
            return fail(ctx, AGSX_EPAIR_BUDGET, "pair count " + std::to_string(total) + " exceeds budget " +
                                                    std::to_string(cfg->pair_budget));
        if (total > capacity) return fail(ctx, AGSX_ECAPACITY, "output buffers too small");
        if (total == 0) return AGSX_OK;
        ensure(ctx->tmp4, total * 8);
        ensure(ctx->pvals, total * 4);
        AGSX_CUDA(cudaMemcpyAsync(ctx->tmp3.p, off.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream));
        k_emit_list<<<static_cast<int>((n + 255) / 256), 256, 0, ctx->stream>>>(
            p, n, pl, ptr<uint32_t>(ctx->tmp1), ptr<uint64_t>(ctx->tmp3), ptr<uint32_t>(ctx->tmp2),
            ptr<uint64_t>(ctx->tmp4), ptr<uint32_t>(ctx->pvals));
        check_launch(ctx);
        AGSX_CUDA(cudaMemcpyAsync(keys, ctx->tmp4.p, total * 8, cudaMemcpyDeviceToHost, ctx->stream));
        AGSX_CUDA(cudaMemcpyAsync(splat_index, ctx->pvals.p, total * 4, cudaMemcpyDeviceToHost, ctx->stream));
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        ctx->have_frame = false;
        return AGSX_OK;
    });
}

int agsx_sort_pairs(agsx_ctx* ctx, uint64_t* keys, uint32_t* splat_index, uint64_t n,
                    int32_t tile_count, uint32_t* ranges) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        if (const int rc = refuse_if_host_frame(ctx, "sort_pairs")) return rc;
        if (tile_count < 0) return fail(ctx, AGSX_EINVAL, "negative tile count");
        if (n >= (1ull << 32)) return fail(ctx, AGSX_EINVAL, "too many pairs");
        ensure(ctx->tmp0, std::max<uint64_t>(n, 1) * 8);
        ensure(ctx->tmp1, std::max<uint64_t>(n, 1) * 8);
        ensure(ctx->tmp2, std::max<uint64_t>(n, 1) * 4);
        ensure(ctx->tmp3, std::max<uint64_t>(n, 1) * 4);
        ensure(ctx->hist, 9 * 256 * 4);
        ensure(ctx->ranges, std::max<int>(tile_count, 1) * 8);
        ensure_lb(ctx, n);
        uint32_t* hist = ptr<uint32_t>(ctx->hist);
        cudaStream_t st = ctx->stream;
        AGSX_CUDA(cudaMemsetAsync(ctx->hist.p, 0, 9 * 256 * 4, st));
        if (tile_count) AGSX_CUDA(cudaMemsetAsync(ctx->ranges.p, 0, static_cast<size_t>(tile_count) * 8, st));
        uint64_t* k[2] = {ptr<uint64_t>(ctx->tmp0), ptr<uint64_t>(ctx->tmp1)};
        uint32_t* v[2] = {ptr<uint32_t>(ctx->tmp2), ptr<uint32_t>(ctx->tmp3)};
        int cur = 0;
        if (n) {
            AGSX_CUDA(cudaMemcpyAsync(k[0], keys, n * 8, cudaMemcpyHostToDevice, st));
            AGSX_CUDA(cudaMemcpyAsync(v[0], splat_index, n * 4, cudaMemcpyHostToDevice, st));
            sort_hist<uint64_t>(ctx, k[0], nullptr, n, 8, false, hist);
            std::vector<uint32_t> h(8 * 256);
            AGSX_CUDA(cudaMemcpyAsync(h.data(), hist, h.size() * 4, cudaMemcpyDeviceToHost, st));
            AGSX_CUDA(cudaStreamSynchronize(st));
            for (int ps = 0; ps < 8; ++ps) {
                // a digit shared by every key permutes nothing in a stable pass
                bool trivial = false;
                for (int d = 0; d < 256; ++d) trivial = trivial || h[ps * 256 + d] == n;
                if (trivial) continue;
                sort_pass<uint64_t>(ctx, k[cur], v[cur], k[cur ^ 1], v[cur ^ 1], nullptr, n, 8 * ps, false,
                                    nullptr);
                cur ^= 1;
            }
            if (tile_count) {
                k_ranges_u64<<<ctx->num_sms * 4, 256, 0, st>>>(k[cur], n, static_cast<uint32_t>(tile_count),
                                                                ptr<uint2>(ctx->ranges));
                check_launch(ctx);
            }
            AGSX_CUDA(cudaMemcpyAsync(keys, k[cur], n * 8, cudaMemcpyDeviceToHost, st));
            AGSX_CUDA(cudaMemcpyAsync(splat_index, v[cur], n * 4, cudaMemcpyDeviceToHost, st));
        }
        if (tile_count)
            AGSX_CUDA(cudaMemcpyAsync(ranges, ctx->ranges.p, static_cast<size_t>(tile_count) * 8,
                                      cudaMemcpyDeviceToHost, st));
        AGSX_CUDA(cudaStreamSynchronize(st));
        ctx->have_frame = false;
        return AGSX_OK;
    });
}

int agsx_raster(agsx_ctx* ctx, const agsx_splat_view* splats, uint64_t n_splats,
                const uint32_t* splat_index, uint64_t n_pairs, const uint32_t* ranges, int32_t width,
                int32_t height, const agsx_config* cfg, float* image, float* max_t) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        if (const int rc = refuse_if_host_frame(ctx, "raster_tile")) return rc;
        if (cfg->tile_size < 1) return fail(ctx, AGSX_EINVAL, "tile_size must be >= 1");
        if (width <= 0 || height <= 0) return fail(ctx, AGSX_EINVAL, "image dimensions must be positive");
        agsx_camera cam{};
        cam.width = width;
        cam.height = height;
        cam.fx = cam.fy = 1.0f;
        const FrameParams p = make_params(cam, *cfg, nullptr, nullptr);
        const uint64_t tiles = static_cast<uint64_t>(p.tiles_x) * p.tiles_y;
        ensure(ctx->tmp0, std::max<uint64_t>(n_splats, 1) * sizeof(agsx_splat_view));
        ensure(ctx->tmp1, std::max<uint64_t>(n_splats, 1) * 4);
        ensure(ctx->tmp2, std::max<uint64_t>(n_splats, 1) * 4);
        ensure(ctx->tmp3, std::max<uint64_t>(n_pairs, 1) * 4);
        ensure(ctx->tmp4, std::max<uint64_t>(tiles, 1) * 8);
        ensure(ctx->image, static_cast<uint64_t>(width) * height * 12);
        ensure(ctx->maxt, std::max<uint64_t>(n_splats, 1) * 4);
        for (Buf* b : {&ctx->p0, &ctx->p1, &ctx->p2, &ctx->p3, &ctx->p4})
            ensure(*b, std::max<uint64_t>(n_splats, 1) * 16);
        const SplatPlanes pl = planes_of(ctx);
        cudaStream_t st = ctx->stream;
        if (n_splats) {
            AGSX_CUDA(cudaMemcpyAsync(ctx->tmp0.p, splats, n_splats * sizeof(agsx_splat_view),
                                      cudaMemcpyHostToDevice, st));
            k_splats_to_planes<<<static_cast<int>((n_splats + 255) / 256), 256, 0, st>>>(
                p, ptr<agsx_splat_view>(ctx->tmp0), n_splats, pl, ptr<uint32_t>(ctx->tmp1),
                ptr<uint32_t>(ctx->tmp2));
            check_launch(ctx);
        }
        if (n_pairs)
            AGSX_CUDA(cudaMemcpyAsync(ctx->tmp3.p, splat_index, n_pairs * 4, cudaMemcpyHostToDevice, st));
        AGSX_CUDA(cudaMemcpyAsync(ctx->tmp4.p, ranges, tiles * 8, cudaMemcpyHostToDevice, st));
        if (max_t) AGSX_CUDA(cudaMemsetAsync(ctx->maxt.p, 0, std::max<uint64_t>(n_splats, 1) * 4, st));
        ensure(ctx->ctr, counters_bytes());
        AGSX_CUDA(cudaMemsetAsync(ctx->ctr.p, 0, counters_bytes(), st));
        Counters* ctr = ptr<Counters>(ctx->ctr);
        if (raster_uses_units(p, max_t != nullptr)) {
            ensure(ctx->tile_pit, std::max<uint64_t>(tiles, 1) * 8);
            AGSX_CUDA(cudaMemsetAsync(ctx->tile_pit.p, 0, tiles * 8, st));
        }
        launch_raster(ctx, p, ptr<uint2>(ctx->tmp4), ptr<uint32_t>(ctx->tmp3), pl.p0, pl.p1, pl.p2,
                      ptr<float>(ctx->image), max_t ? ptr<uint32_t>(ctx->maxt) : nullptr, ctr);
        AGSX_CUDA(cudaMemcpyAsync(image, ctx->image.p, static_cast<size_t>(width) * height * 12,
                                  cudaMemcpyDeviceToHost, st));
        if (max_t && n_splats)
            AGSX_CUDA(cudaMemcpyAsync(max_t, ctx->maxt.p, n_splats * 4, cudaMemcpyDeviceToHost, st));
        AGSX_CUDA(cudaStreamSynchronize(st));
        ctx->have_frame = false;
        return AGSX_OK;
    });
}

int agsx_device_alloc(agsx_ctx* ctx, size_t bytes, void** out) {
    if (!ctx || !out) return AGSX_EINVAL;
    *out = nullptr;
    return guarded(ctx, [&]() -> int {
        AGSX_CUDA(cudaMalloc(out, std::max<size_t>(bytes, 1)));
        return AGSX_OK;
    });
}

void agsx_device_free(agsx_ctx* ctx, void* p) {
    if (!ctx || !p) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    cudaFree(p);
}

int agsx_fold_max_t(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam, const agsx_config* cfg,
                    const agsx_lut* lut_shape, float* folded, uint8_t* observed) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        if (!cfg || !lut_shape || lut_shape->bin_count < 1 || !folded || !observed)
            return fail(ctx, AGSX_EINVAL, "fold_max_t: bad arguments");
        agsx_config c = *cfg;
        c.mode = AGSX_MODE_ELLIPSE;  // build_lut renders losslessly (calibrate.cpp:22-23)
        c.flags |= AGSX_FLAG_EXACT_ALPHA;
        int rc = start_frame(ctx, scene, cam, &c, nullptr, true);
        if (rc) return rc;
        rc = finish_frame(ctx, nullptr);
        if (rc) return rc;
        const int nb = lut_shape->bin_count;
        ensure(ctx->calib, static_cast<size_t>(2 * nb) * 4 + 4096 * 8 + 8);
        uint32_t* dfold = ptr<uint32_t>(ctx->calib);
        AGSX_CUDA(cudaMemsetAsync(dfold, 0, static_cast<size_t>(2 * nb) * 4, ctx->stream));
        if (scene->n) {
            // the frame's splats with tiles: {gid, depth} (bucketed path) or
            // the depth order's ping-pong buffer the device chose
            const bool wide = depth_keys_wide_host(*ctx->h_ctr);  // finish_frame synchronised
            const uint32_t* gid = ctx->f_bucket ? ptr<uint32_t>(ctx->bk_gd) : ptr<uint32_t>(wide ? ctx->dvals : ctx->dvals2);
            const uint32_t* dep = ctx->f_bucket ? gid + 1 : ptr<uint32_t>(wide ? ctx->dkeys : ctx->dkeys2);
            // max_t is per storage slot, as are the depth order and the bucketed list
            k_fold_max_t<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(
                gid, nullptr, dep, ctx->f_bucket ? 2 : 1, &ptr<Counters>(ctx->ctr)->m,
                ptr<uint32_t>(ctx->maxt), lut_shape->depth_min, lut_shape->depth_max, nb, dfold, dfold + nb);
            check_launch(ctx);
        }
        std::vector<uint32_t> h(static_cast<size_t>(2 * nb));
        AGSX_CUDA(cudaMemcpyAsync(h.data(), dfold, h.size() * 4, cudaMemcpyDeviceToHost, ctx->stream));
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        for (int b = 0; b < nb; ++b) {
            float v;
            std::memcpy(&v, &h[b], 4);
            if (h[nb + b]) {
                observed[b] = 1;
                folded[b] = std::max(folded[b], v);
            }
        }
        return AGSX_OK;
    });
}

int agsx_sq_err(agsx_ctx* ctx, const float* a, const float* b, uint64_t n, double* out) {
    if (!ctx || !out) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        constexpr int kBlocks = 1024;  // fixed: the summation order is the same every call
        ensure(ctx->calib, 4096 * 8 + 8 + 1024);
        double* part = reinterpret_cast<double*>(static_cast<char*>(ctx->calib.p) + 1024);
        double* res = part + kBlocks;
        k_sq_err_partial<<<kBlocks, 256, 0, ctx->stream>>>(a, b, n, part);
        check_launch(ctx);
        k_sq_err_final<<<1, 32, 0, ctx->stream>>>(part, kBlocks, res);
        check_launch(ctx);
        AGSX_CUDA(cudaMemcpyAsync(out, res, 8, cudaMemcpyDeviceToHost, ctx->stream));
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        return AGSX_OK;
    });
}


int agsx_project(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam, const agsx_config* cfg,
                 uint8_t* valid, float* out) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        if (!scene || !cam || !cfg || !valid || !out) return fail(ctx, AGSX_EINVAL, "project: null argument");
        const uint64_t n = scene->n;
        const FrameParams p = make_params(*cam, *cfg, nullptr, nullptr);
        ensure(ctx->tmp0, std::max<uint64_t>(n, 1));
        ensure(ctx->tmp1, std::max<uint64_t>(n, 1) * 24);
        if (n) {
            k_project<<<grid_of(n), 256, 0, ctx->stream>>>(p, scene->view(), ptr<uint8_t>(ctx->tmp0),
                                                           ptr<float>(ctx->tmp1));
            check_launch(ctx);
            AGSX_CUDA(cudaMemcpyAsync(valid, ctx->tmp0.p, n, cudaMemcpyDeviceToHost, ctx->stream));
        }
        to_host(ctx, out, ctx->tmp1, 6 * n);
        return AGSX_OK;
    });
}

int agsx_eval_color(agsx_ctx* ctx, const agsx_scene* scene, const float* dirs, float* rgb) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        if (!scene || !dirs || !rgb) return fail(ctx, AGSX_EINVAL, "eval_color: null argument");
        const uint64_t n = scene->n;
        const float* d = to_device(ctx, ctx->tmp0, dirs, 3 * n);
        ensure(ctx->tmp1, std::max<uint64_t>(n, 1) * 12);
        if (n) {
            k_eval_color<<<grid_of(n), 256, 0, ctx->stream>>>(scene->view(), d, ptr<float>(ctx->tmp1));
            check_launch(ctx);
        }
        to_host(ctx, rgb, ctx->tmp1, 3 * n);
        return AGSX_OK;
    });
}

int agsx_compute_th(agsx_ctx* ctx, const float* cov2d, const float* depth, uint64_t n, const agsx_lut* lut,
                    float k, float tau, float* th) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        if ((n && (!cov2d || !depth)) || !th) return fail(ctx, AGSX_EINVAL, "compute_th: null argument");
        agsx_camera cam{};
        cam.rotation[0] = cam.rotation[4] = cam.rotation[8] = 1.0f;
        cam.fx = cam.fy = 1.0f;
        cam.width = cam.height = 1;
        agsx_config cfg{};
        cfg.mode = AGSX_MODE_ADAGSCALE;
        cfg.k = k;
        cfg.alpha_threshold = tau;
        cfg.tile_size = 16;
        const float* lut_dev = nullptr;
        if (lut && lut->bin_count > kLutInline) lut_dev = to_device(ctx, ctx->lut_ext, lut->bins, lut->bin_count);
        const FrameParams p = make_params(cam, cfg, lut, lut_dev);
        const float* c = to_device(ctx, ctx->tmp0, cov2d, 3 * n);
        const float* d = to_device(ctx, ctx->tmp1, depth, n);
        ensure(ctx->tmp2, std::max<uint64_t>(n, 1) * 4);
        if (n) {
            k_compute_th<<<grid_of(n), 256, 0, ctx->stream>>>(p, c, d, n, ptr<float>(ctx->tmp2));
            check_launch(ctx);
        }
        to_host(ctx, th, ctx->tmp2, n);
        for (uint64_t i = 0; i < n; ++i)
            if (th[i] != th[i]) return fail(ctx, AGSX_EINVAL, "compute_th: non-positive determinant");
        return AGSX_OK;
    });
}

int agsx_alpha_at(agsx_ctx* ctx, const agsx_splat_view* splats, const float* px, uint64_t n, float alpha_clamp,
                  float* alpha) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        if ((n && (!splats || !px)) || !alpha) return fail(ctx, AGSX_EINVAL, "alpha_at: null argument");
        const agsx_splat_view* s = to_device(ctx, ctx->tmp0, splats, n);
        const float* x = to_device(ctx, ctx->tmp1, px, 2 * n);
        ensure(ctx->tmp2, std::max<uint64_t>(n, 1) * 4);
        if (n) {
            k_alpha_at<<<grid_of(n), 256, 0, ctx->stream>>>(s, x, n, alpha_clamp, ptr<float>(ctx->tmp2));
            check_launch(ctx);
        }
        to_host(ctx, alpha, ctx->tmp2, n);
        return AGSX_OK;
    });
}

int agsx_effective_radius(agsx_ctx* ctx, const float* opacity, const float* th, const float* cov2d, uint64_t n,
                          float* out) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        if ((n && (!opacity || !th || !cov2d)) || !out) return fail(ctx, AGSX_EINVAL, "effective_radius: null argument");
        const float* o = to_device(ctx, ctx->tmp0, opacity, n);
        const float* t = to_device(ctx, ctx->tmp1, th, n);
        const float* c = to_device(ctx, ctx->tmp2, cov2d, 3 * n);
        ensure(ctx->tmp3, std::max<uint64_t>(n, 1) * 8);
        if (n) {
            k_effective_radius<<<grid_of(n), 256, 0, ctx->stream>>>(o, t, c, n, ptr<float>(ctx->tmp3));
            check_launch(ctx);
        }
        to_host(ctx, out, ctx->tmp3, 2 * n);
        return AGSX_OK;
    });
}

int agsx_device_logf(agsx_ctx* ctx, const float* x, float* y, uint64_t n) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        ensure(ctx->tmp0, std::max<uint64_t>(n, 1) * 4);
        ensure(ctx->tmp1, std::max<uint64_t>(n, 1) * 4);
        if (!n) return AGSX_OK;
        AGSX_CUDA(cudaMemcpyAsync(ctx->tmp0.p, x, n * 4, cudaMemcpyHostToDevice, ctx->stream));
        k_logf<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(ptr<float>(ctx->tmp0), ptr<float>(ctx->tmp1), n);
        check_launch(ctx);
        AGSX_CUDA(cudaMemcpyAsync(y, ctx->tmp1.p, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        return AGSX_OK;
    });
}

int agsx_device_expf(agsx_ctx* ctx, const float* x, float* y, uint64_t n) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        ensure(ctx->tmp0, std::max<uint64_t>(n, 1) * 4);
        ensure(ctx->tmp1, std::max<uint64_t>(n, 1) * 4);
        if (!n) return AGSX_OK;
        AGSX_CUDA(cudaMemcpyAsync(ctx->tmp0.p, x, n * 4, cudaMemcpyHostToDevice, ctx->stream));
        k_expf<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(ptr<float>(ctx->tmp0), ptr<float>(ctx->tmp1), n);
        check_launch(ctx);
        AGSX_CUDA(cudaMemcpyAsync(y, ctx->tmp1.p, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        return AGSX_OK;
    });
}

}  // extern "C"


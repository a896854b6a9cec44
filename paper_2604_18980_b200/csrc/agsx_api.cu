// agsx_api.cu -- C-ABI of libagsx.so: contexts, scene upload, the render
// entry points (synchronous, asynchronous, host / device / PPM targets, the
// blend-event stream), frame statistics and the parity dumps.
//
//   reference: render()          rasterizer.cpp:102-165
//              validate(cfg/cam) scene.cpp:41-59, 113-123
#include "agsx_ctx.cuh"

#include <cmath>

extern "C" {

int agsx_abi_version(void) { return AGSX_ABI_VERSION; }

int agsx_host_alloc(size_t bytes, void** out) {
    if (!out) return AGSX_EINVAL;
    *out = nullptr;
    const cudaError_t e = cudaHostAlloc(out, std::max<size_t>(bytes, 1), cudaHostAllocPortable);
    if (e != cudaSuccess) return e == cudaErrorMemoryAllocation ? AGSX_ENOMEM : AGSX_ECUDA;
    return AGSX_OK;
}

void agsx_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

}  // extern "C"

namespace agsx::host {
// Host copy of a scene's slot -> id (orig) or id -> slot (inv) map; empty when
// the scene keeps the caller's order.  For the dump and host-side paths.
std::vector<uint32_t> scene_map_host(const Buf& b, uint64_t n) {
    std::vector<uint32_t> v;
    if (!b.p || n == 0) return v;
    v.resize(n);
    AGSX_CUDA(cudaMemcpy(v.data(), b.p, n * 4, cudaMemcpyDeviceToHost));
    return v;
}

// A slot-ordered per-Gaussian array (status, max_t) copied to the host in
// Gaussian-id order.
void slots_to_ids_host(const agsx_scene* sc, const void* dev, uint32_t* host_out, cudaStream_t st) {
    const uint64_t n = sc->n;
    if (!n) return;
    if (!sc->inv.p) {
        AGSX_CUDA(cudaMemcpyAsync(host_out, dev, n * 4, cudaMemcpyDeviceToHost, st));
        AGSX_CUDA(cudaStreamSynchronize(st));
        return;
    }
    std::vector<uint32_t> by_slot(n);
    AGSX_CUDA(cudaMemcpyAsync(by_slot.data(), dev, n * 4, cudaMemcpyDeviceToHost, st));
    AGSX_CUDA(cudaStreamSynchronize(st));
    const std::vector<uint32_t> inv = scene_map_host(sc->inv, n);
    for (uint64_t g = 0; g < n; ++g) host_out[g] = by_slot[inv[g]];
}

}  // namespace agsx::host

namespace {
// Scene storage order: AGSX_SCENE_ORDER=input keeps the caller's order
// (A/B runs); the default is the 3D Morton order (DevScene).
bool scene_order_morton() {
    static const bool morton = [] {
        const char* e = std::getenv("AGSX_SCENE_ORDER");
        return !(e && std::strcmp(e, "input") == 0);
    }();
    return morton;
}
}  // namespace

extern "C" {

int agsx_create(int device, agsx_ctx** out) {
    if (!out) return AGSX_EINVAL;
    *out = nullptr;
    agsx_ctx* ctx = new (std::nothrow) agsx_ctx();
    if (!ctx) return AGSX_ENOMEM;
    ctx->device = device;
    const int rc = guarded(ctx, [&]() -> int {
        AGSX_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        AGSX_CUDA(shared_copy_stream(device, &ctx->copy_stream));
        for (auto& e : ctx->band_ev) AGSX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        AGSX_CUDA(cudaEventCreateWithFlags(&ctx->copy_done, cudaEventDisableTiming));
        AGSX_CUDA(cudaEventCreateWithFlags(&ctx->ev_zeroed, cudaEventDisableTiming));
        AGSX_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
        AGSX_CUDA(sort_configure<uint32_t>(sort_smem(false), &ctx->occ_sort32));
        AGSX_CUDA(sort_configure<uint64_t>(sort_smem(true), &ctx->occ_sort64));
        AGSX_CUDA(emit_configure(false, &ctx->occ_emit));
        AGSX_CUDA(emit_configure(true, &ctx->occ_emit_big));
        ctx->occ_emit_big = std::max(ctx->occ_emit_big, 1);
        AGSX_CUDA(raster_units_occupancy(&ctx->occ_raster));
        ctx->occ_raster = std::max(ctx->occ_raster, 1);
        ctx->occ_sort32 = std::max(ctx->occ_sort32, 1);
        ctx->occ_sort64 = std::max(ctx->occ_sort64, 1);
        ctx->occ_emit = std::max(ctx->occ_emit, 1);
        AGSX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctx->occ_tile_sort, k_tile_sort, 256, 0));
        ctx->occ_tile_sort = std::max(ctx->occ_tile_sort, 1);
        for (auto& set : ctx->ev_ring)
            for (auto& e : set) AGSX_CUDA(cudaEventCreate(&e));
        // the counter block + the two async-chain words behind it (ChainWords)
        AGSX_CUDA(cudaMallocHost(reinterpret_cast<void**>(&ctx->h_ctr), sizeof(Counters) + sizeof(ChainWords)));
        std::memset(static_cast<void*>(ctx->h_ctr), 0, sizeof(Counters) + sizeof(ChainWords));
        ensure(ctx->chain, sizeof(ChainWords), /*zero=*/true);
        AGSX_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->h_ctr_dev), ctx->h_ctr, 0));
        return AGSX_OK;
    });
    if (rc != AGSX_OK) {
        std::fprintf(stderr, "agsx_create: %s\n", ctx->err.c_str());
        agsx_destroy(ctx);
        return rc;
    }
    *out = ctx;
    return AGSX_OK;
}

void agsx_destroy(agsx_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    for (Buf* b : {&ctx->status, &ctx->p0, &ctx->p1, &ctx->p2, &ctx->p3, &ctx->p4, &ctx->dkeys,
                   &ctx->dvals, &ctx->dkeys2, &ctx->dvals2, &ctx->dcounts, &ctx->chunks, &ctx->img_u8, &ctx->tkeys, &ctx->pvals, &ctx->tkeys2,
                   &ctx->pvals2, &ctx->ranges, &ctx->image, &ctx->lb, &ctx->ctr, &ctx->hist,
                   &ctx->maxt, &ctx->dump, &ctx->lut_ext, &ctx->tile_pit, &ctx->calib, &ctx->sort_counts, &ctx->tmp0, &ctx->tmp1, &ctx->tmp2,
                   &ctx->tmp3, &ctx->tmp4, &ctx->bk_hits, &ctx->bk_gd, &ctx->ekeys, &ctx->ekeys2, &ctx->big_list, &ctx->chain})
        release(*b);
    for (auto& set : ctx->ev_ring)
        for (auto& e : set)
            if (e) cudaEventDestroy(e);
    if (ctx->h_ctr) cudaFreeHost(ctx->h_ctr);
    for (auto& e : ctx->band_ev)
        if (e) cudaEventDestroy(e);
    if (ctx->copy_done) cudaEventDestroy(ctx->copy_done);
    if (ctx->ev_zeroed) cudaEventDestroy(ctx->ev_zeroed);
    if (ctx->copy_stream) cudaStreamSynchronize(ctx->copy_stream);  // shared per device: not destroyed
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

const char* agsx_last_error(const agsx_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

void* agsx_stream(agsx_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

uint64_t agsx_kernel_launches(const agsx_ctx* ctx) { return ctx ? ctx->launches : 0; }

int agsx_scene_upload(agsx_ctx* ctx, const agsx_scene_desc* d, agsx_scene** out) {
    if (!ctx || !d || !out) return AGSX_EINVAL;
    *out = nullptr;
    const int D = d->sh_coeffs;
    if (!(D == 1 || D == 4 || D == 9 || D == 16))
        return fail(ctx, AGSX_EINVAL, "sh coefficient count must be 3*d^2 for d in {1,2,3,4}");
    agsx_scene* sc = new (std::nothrow) agsx_scene();
    if (!sc) return AGSX_ENOMEM;
    const int rc = guarded(ctx, [&]() -> int {
        sc->device = ctx->device;
        sc->n = d->count;
        sc->D = D;
        const uint64_t n = d->count;
        ensure(sc->pos_op, std::max<uint64_t>(n, 1) * 16);
        ensure(sc->rot, std::max<uint64_t>(n, 1) * 16);
        ensure(sc->scale_r, std::max<uint64_t>(n, 1) * 16);
        ensure(sc->sh_gb, std::max<uint64_t>(n, 1) * 8);
        ensure(sc->sh_rest, std::max<uint64_t>(n * (3 * D - 3), 1) * 4);
        if (n == 0) return AGSX_OK;
        // stage the host SoA arrays, pack on the device in slices
        const uint64_t slice = 1u << 22;
        const uint64_t fl_per = 3 + 3 + 4 + 1 + 3 * static_cast<uint64_t>(D);
        Buf stage;
        ensure(stage, std::min(n, slice) * fl_per * 4);
        float* s = ptr<float>(stage);
        for (uint64_t b = 0; b < n; b += slice) {
            const uint64_t m = std::min(slice, n - b);
            float* sm = s;
            float* ss = sm + 3 * m;
            float* sq = ss + 3 * m;
            float* so = sq + 4 * m;
            float* sh = so + m;
            AGSX_CUDA(cudaMemcpyAsync(sm, d->mean + 3 * b, 12 * m, cudaMemcpyHostToDevice, ctx->stream));
            AGSX_CUDA(cudaMemcpyAsync(ss, d->scale + 3 * b, 12 * m, cudaMemcpyHostToDevice, ctx->stream));
            AGSX_CUDA(cudaMemcpyAsync(sq, d->rotation + 4 * b, 16 * m, cudaMemcpyHostToDevice, ctx->stream));
            AGSX_CUDA(cudaMemcpyAsync(so, d->opacity + b, 4 * m, cudaMemcpyHostToDevice, ctx->stream));
            AGSX_CUDA(cudaMemcpyAsync(sh, d->sh + 3 * D * b, 12 * D * m, cudaMemcpyHostToDevice, ctx->stream));
            k_pack_scene<<<static_cast<int>((m + 255) / 256), 256, 0, ctx->stream>>>(
                m, D, sm, ss, sq, so, sh, ptr<float4>(sc->pos_op) + b, ptr<float4>(sc->rot) + b,
                ptr<float4>(sc->scale_r) + b, ptr<float2>(sc->sh_gb) + b,
                ptr<float>(sc->sh_rest) + b * (3 * D - 3));
            check_launch(ctx);
        }
        release(stage);
        float mo = -INFINITY;  // NaN opacities count as +inf (the clamp variant handles them)
        for (uint64_t i = 0; i < n; ++i) {
            const float o = d->opacity[i];
            mo = o > mo ? o : (o == o ? mo : INFINITY);
        }
        sc->max_opacity = mo;
        if (scene_order_morton() && n > 1) {
            // storage order: 3D Morton order of the means (DevScene).  Spatial
            // neighbours share K1's warps (similar footprints: less divergence in
            // the tile test) and the bucketed scatter's tiles.
            float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
            for (uint64_t i = 0; i < n; ++i)
                for (int a = 0; a < 3; ++a) {
                    const float v = d->mean[3 * i + a];
                    if (v < lo[a]) lo[a] = v;  // NaN never compares: skipped
                    if (v > hi[a]) hi[a] = v;
                }
            float3 l, sc3;
            float* lp[3] = {&l.x, &l.y, &l.z};
            float* sp[3] = {&sc3.x, &sc3.y, &sc3.z};
            for (int a = 0; a < 3; ++a) {
                const bool ok = std::isfinite(lo[a]) && std::isfinite(hi[a]) && hi[a] > lo[a];
                *lp[a] = ok ? lo[a] : 0.0f;
                *sp[a] = ok ? 1023.0f / (hi[a] - lo[a]) : 0.0f;
            }
            Buf codes, codes2, ord, ord2;
            ensure(codes, n * 4);
            ensure(codes2, n * 4);
            ensure(ord, n * 4);
            ensure(ord2, n * 4);
            const int grid = static_cast<int>((n + 255) / 256);
            k_morton_codes<<<grid, 256, 0, ctx->stream>>>(n, ptr<float4>(sc->pos_op), l, sc3, ptr<uint32_t>(codes));
            check_launch(ctx);
            // stable LSD sort of the 30-bit codes, values = Gaussian ids
            uint32_t* ck[2] = {ptr<uint32_t>(codes), ptr<uint32_t>(codes2)};
            uint32_t* cv[2] = {ptr<uint32_t>(ord), ptr<uint32_t>(ord2)};
            for (int ps = 0; ps < 4; ++ps)
                sort_pass<uint32_t>(ctx, ck[ps & 1], ps ? cv[ps & 1] : nullptr, ck[(ps + 1) & 1], cv[(ps + 1) & 1],
                                    nullptr, n, 8 * ps, false, nullptr);
            // after 4 passes the order is in cv[0]
            Buf pos2, rot2, scale2, gb2, rest2;
            ensure(pos2, n * 16);
            ensure(rot2, n * 16);
            ensure(scale2, n * 16);
            ensure(gb2, n * 8);
            ensure(rest2, std::max<uint64_t>(n * (3 * D - 3), 1) * 4);
            ensure(sc->inv, n * 4);
            k_permute_scene<<<grid, 256, 0, ctx->stream>>>(
                n, D, cv[0], ptr<float4>(sc->pos_op), ptr<float4>(sc->rot), ptr<float4>(sc->scale_r),
                ptr<float2>(sc->sh_gb), ptr<float>(sc->sh_rest), ptr<float4>(pos2), ptr<float4>(rot2),
                ptr<float4>(scale2), ptr<float2>(gb2), ptr<float>(rest2), ptr<uint32_t>(sc->inv));
            check_launch(ctx);
            AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
            std::swap(sc->pos_op, pos2);
            std::swap(sc->rot, rot2);
            std::swap(sc->scale_r, scale2);
            std::swap(sc->sh_gb, gb2);
            std::swap(sc->sh_rest, rest2);
            std::swap(sc->orig, ord);  // cv[0] is ord: the order after four passes
            for (Buf* b : {&pos2, &rot2, &scale2, &gb2, &rest2, &codes, &codes2, &ord, &ord2}) release(*b);
        }
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        return AGSX_OK;
    });
    if (rc != AGSX_OK) {
        agsx_scene_free(sc);
        return rc;
    }
    *out = sc;
    return AGSX_OK;
}

void agsx_scene_free(agsx_scene* sc) {
    if (!sc) return;
    cudaSetDevice(sc->device);
    for (Buf* b : {&sc->pos_op, &sc->rot, &sc->scale_r, &sc->sh_gb, &sc->sh_rest, &sc->orig, &sc->inv}) release(*b);
    delete sc;
}

uint64_t agsx_scene_count(const agsx_scene* sc) { return sc ? sc->n : 0; }

int agsx_render_async(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam,
                      const agsx_config* cfg, const agsx_lut* lut) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int { return start_frame(ctx, scene, cam, cfg, lut, false); });
}

int agsx_render_async_to(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam,
                         const agsx_config* cfg, const agsx_lut* lut, float* target) {
    if (!ctx) return AGSX_EINVAL;
    if (!target) return fail(ctx, AGSX_EINVAL, "render_async_to: null target");
    return guarded(ctx, [&]() -> int { return start_frame(ctx, scene, cam, cfg, lut, false, nullptr, target); });
}

int agsx_render_async_host(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam,
                           const agsx_config* cfg, const agsx_lut* lut, float* image) {
    if (!ctx) return AGSX_EINVAL;
    if (!image) return fail(ctx, AGSX_EINVAL, "render_async_host: null image");
    return guarded(ctx, [&]() -> int {
        const int rc = start_frame(ctx, scene, cam, cfg, lut, false, image);
        if (rc == AGSX_OK) ctx->f_host_dst = image;
        return rc;
    });
}

int agsx_render_wait(agsx_ctx* ctx, agsx_frame* out) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        float* dst = ctx->f_host_dst;
        uint8_t* dst8 = ctx->f_host_dst_u8;
        ctx->f_host_dst = nullptr;
        ctx->f_host_dst_u8 = nullptr;
        const int rc = finish_frame(ctx, out);
        if (rc) return rc;
        if (dst8) return ctx->f_band_host_u8 ? AGSX_OK : quantize_to_host(ctx, dst8);
        if (!dst || ctx->f_image_on_host) return rc;
        AGSX_CUDA(cudaMemcpyAsync(dst, ctx->image.p, static_cast<size_t>(ctx->f_cam.width) * ctx->f_cam.height * 12,
                                  cudaMemcpyDeviceToHost, ctx->stream));
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        return AGSX_OK;
    });
}

int agsx_render(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam,
                const agsx_config* cfg, const agsx_lut* lut, agsx_frame* out) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        const bool maxt = out && out->max_t;
        int rc = start_frame(ctx, scene, cam, cfg, lut, maxt, out ? out->image : nullptr);
        if (rc) return rc;
        rc = finish_frame(ctx, out);
        if (rc) return rc;
        if (out && out->image && !ctx->f_image_on_host) {
            AGSX_CUDA(cudaMemcpyAsync(out->image, ctx->image.p,
                                      static_cast<size_t>(cam->width) * cam->height * 12,
                                      cudaMemcpyDeviceToHost, ctx->stream));
        }
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        if (maxt && scene->n)  // per Gaussian id (the device array is per storage slot)
            slots_to_ids_host(scene, ctx->maxt.p, reinterpret_cast<uint32_t*>(out->max_t), ctx->stream);
        return AGSX_OK;
    });
}

int agsx_render_u8(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam, const agsx_config* cfg,
                   const agsx_lut* lut, uint8_t* image_u8, agsx_frame* out) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        if (!image_u8) return fail(ctx, AGSX_EINVAL, "render_u8: null image");
        int rc = start_frame(ctx, scene, cam, cfg, lut, false, nullptr, nullptr, image_u8);
        if (rc) return rc;
        rc = finish_frame(ctx, out);
        if (rc) return rc;
        if (ctx->f_band_host_u8) return AGSX_OK;  // bands already copied behind the raster
        return quantize_to_host(ctx, image_u8);
    });
}

int agsx_render_async_host_u8(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam,
                              const agsx_config* cfg, const agsx_lut* lut, uint8_t* image_u8) {
    if (!ctx) return AGSX_EINVAL;
    if (!image_u8) return fail(ctx, AGSX_EINVAL, "render_async_host_u8: null image");
    return guarded(ctx, [&]() -> int {
        const int rc = start_frame(ctx, scene, cam, cfg, lut, false, nullptr, nullptr, image_u8);
        if (rc == AGSX_OK) ctx->f_host_dst_u8 = image_u8;
        return rc;
    });
}

int agsx_render_contributions(agsx_ctx* ctx, const agsx_scene* scene, const agsx_camera* cam,
                              const agsx_config* cfg, const agsx_lut* lut, agsx_blend_record* records,
                              uint64_t capacity, uint64_t* count, agsx_frame* out) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        if (!cfg || !count) return fail(ctx, AGSX_EINVAL, "render_contributions: null config or count");
        if (cfg->tile_size > 64)  // the tile's T and C live in shared memory
            return fail(ctx, AGSX_EINVAL, "render_contributions: tile_size above 64 is not supported");
        agsx_config c = *cfg;
        c.flags |= AGSX_FLAG_EXACT_ALPHA;  // the stream records the reference's alpha values
        const bool maxt = out && out->max_t;
        int rc = start_frame(ctx, scene, cam, &c, lut, maxt, out ? out->image : nullptr);
        if (rc) return rc;
        rc = finish_frame(ctx, out);
        if (rc) return rc;
        const FrameParams& p = ctx->f_params;
        const uint64_t tiles = static_cast<uint64_t>(p.tiles_x) * p.tiles_y;
        const uint64_t n = scene->n;
        if (out && out->image && !ctx->f_image_on_host)
            AGSX_CUDA(cudaMemcpyAsync(out->image, ctx->image.p, static_cast<size_t>(cam->width) * cam->height * 12,
                                      cudaMemcpyDeviceToHost, ctx->stream));
        if (maxt && n) slots_to_ids_host(scene, ctx->maxt.p, reinterpret_cast<uint32_t*>(out->max_t), ctx->stream);
        // pass 1: events per tile; host scan -> per-tile offsets in tile order
        ensure(ctx->tmp1, std::max<uint64_t>(tiles, 1) * 4);
        ensure(ctx->tmp2, std::max<uint64_t>(tiles, 1) * 8);
        const SplatPlanes pl = planes_of(ctx);
        AGSX_CUDA(launch_raster_records(ctx->stream, p, ptr<uint2>(ctx->ranges), ctx->f_pvals, pl.p0, pl.p1, pl.p2,
                                        ptr<float>(ctx->image), ptr<uint32_t>(ctx->tmp1), nullptr, nullptr));
        ++ctx->launches;
        std::vector<uint32_t> per_tile(tiles);
        std::vector<uint64_t> off(tiles);
        if (tiles)
            AGSX_CUDA(cudaMemcpyAsync(per_tile.data(), ctx->tmp1.p, tiles * 4, cudaMemcpyDeviceToHost, ctx->stream));
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        uint64_t total = 0;
        for (uint64_t t = 0; t < tiles; ++t) {
            off[t] = total;
            total += per_tile[t];
        }
        *count = total;
        if (!records || capacity < total)
            return fail(ctx, AGSX_ECAPACITY, "render_contributions: " + std::to_string(total) + " records");
        if (total == 0) return AGSX_OK;
        // pass 2: the records, then Gaussian id -> index in the view's splat sequence
        ensure(ctx->tmp3, total * sizeof(agsx_blend_record));
        AGSX_CUDA(cudaMemcpyAsync(ctx->tmp2.p, off.data(), tiles * 8, cudaMemcpyHostToDevice, ctx->stream));
        AGSX_CUDA(launch_raster_records(ctx->stream, p, ptr<uint2>(ctx->ranges), ctx->f_pvals, pl.p0, pl.p1, pl.p2,
                                        ptr<float>(ctx->image), nullptr, ptr<uint64_t>(ctx->tmp2),
                                        ptr<agsx_blend_record>(ctx->tmp3)));
        ++ctx->launches;
        AGSX_CUDA(cudaMemcpyAsync(records, ctx->tmp3.p, total * sizeof(agsx_blend_record), cudaMemcpyDeviceToHost,
                                  ctx->stream));
        std::vector<uint32_t> st(n);  // per Gaussian id
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        slots_to_ids_host(scene, ctx->status.p, st.data(), ctx->stream);
        const std::vector<uint32_t> inv = scene_map_host(scene->inv, n);
        std::vector<uint32_t> view_index(n);  // per storage slot (the records carry slots)
        uint32_t k = 0;
        for (uint64_t i = 0; i < n; ++i) {  // survivors in Gaussian order (preprocess.cpp:158-162)
            view_index[inv.empty() ? i : inv[i]] = k;
            k += (st[i] & kAliveBit) ? 1u : 0u;
        }
        for (uint64_t i = 0; i < total; ++i) records[i].splat = view_index[records[i].splat];
        return AGSX_OK;
    });
}

int agsx_stage_history(agsx_ctx* ctx, float* stage_ms, int32_t max_frames, int32_t* out_frames) {
    if (!ctx || !stage_ms || !out_frames) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        const uint64_t avail = std::min<uint64_t>(ctx->frames, agsx_ctx::kRing);
        const int n = static_cast<int>(std::min<uint64_t>(avail, static_cast<uint64_t>(std::max(max_frames, 0))));
        for (int i = 0; i < n; ++i) {
            // oldest first among the last n frames
            const uint64_t f = ctx->frames - n + i;
            cudaEvent_t* e = ctx->ev_ring[f % agsx_ctx::kRing];
            float ms[5];
            for (int k = 0; k < 5; ++k) AGSX_CUDA(cudaEventElapsedTime(&ms[k], e[k], e[k + 1]));
            stage_ms[4 * i + 0] = ms[0];
            stage_ms[4 * i + 1] = ms[2];
            stage_ms[4 * i + 2] = ms[1] + ms[3];
            stage_ms[4 * i + 3] = ms[4];
        }
        *out_frames = n;
        return AGSX_OK;
    });
}

int agsx_frame_stats(agsx_ctx* ctx, uint64_t* stats, int32_t n) {
    if (!ctx || !stats) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        const Counters c = *ctx->h_ctr;
        uint64_t p_it = c.p_it;
        if (ctx->f_pit_tiles && ctx->f_tile_count > 0) {  // the units rasterizer keeps P_it per tile
            std::vector<unsigned long long> w(static_cast<size_t>(ctx->f_tile_count));
            AGSX_CUDA(cudaMemcpy(w.data(), ctx->tile_pit.p, w.size() * 8, cudaMemcpyDeviceToHost));
            p_it = 0;
            for (const unsigned long long x : w) p_it += static_cast<uint32_t>(x);
        }
        // sort formulation of the frame: depth passes over the splats (3 or 4,
        // depth-then-tile path) or 0 (tile-bucketed path)
        const uint64_t depth_passes = ctx->f_bucket || c.m == 0 ? 0u : (depth_keys_wide_host(c) ? 4u : 3u);
        const uint64_t v[16] = {c.s, c.m, c.p, p_it, c.overflow, static_cast<uint64_t>(ctx->f_tile_count),
                                c.dbg[0], c.dbg[1], c.dbg[2], c.dbg[3], c.dbg[4], c.dbg[5], c.dbg[6], c.dbg[7],
                                depth_passes, ctx->f_bucket ? 1u : 0u};
        for (int i = 0; i < n && i < 16; ++i) stats[i] = v[i];
        return AGSX_OK;
    });
}

int agsx_device_image(agsx_ctx* ctx, float** dptr, int32_t* width, int32_t* height) {
    if (!ctx || !dptr) return AGSX_EINVAL;
    if (!ctx->have_frame) return fail(ctx, AGSX_EINVAL, "no frame rendered yet");
    if (ctx->f_image_on_host) return fail(ctx, AGSX_EINVAL, "the last frame was rasterised into a caller buffer");
    *dptr = ptr<float>(ctx->image);
    if (width) *width = ctx->f_cam.width;
    if (height) *height = ctx->f_cam.height;
    return AGSX_OK;
}

int agsx_dump_tile_counts(agsx_ctx* ctx, uint32_t* counts, uint8_t* alive, uint64_t n) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        if (!ctx->have_frame) return fail(ctx, AGSX_EINVAL, "no frame rendered yet");
        if (n != ctx->f_scene->n) return fail(ctx, AGSX_EINVAL, "count mismatch");
        std::vector<uint32_t> st(n);
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        slots_to_ids_host(ctx->f_scene, ctx->status.p, st.data(), ctx->stream);
        for (uint64_t i = 0; i < n; ++i) {
            if (counts) counts[i] = st[i] & kCountMask;
            if (alive) alive[i] = (st[i] & kAliveBit) ? 1 : 0;
        }
        return AGSX_OK;
    });
}

int agsx_dump_sorted_pairs(agsx_ctx* ctx, uint64_t* keys, uint32_t* gids, uint64_t capacity,
                           uint64_t* out_count) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        if (!ctx->have_frame) return fail(ctx, AGSX_EINVAL, "no frame rendered yet");
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        const Counters c = *ctx->h_ctr;
        const uint64_t P = c.p_eff;
        if (out_count) *out_count = P;
        if (P > capacity) return fail(ctx, AGSX_ECAPACITY, "buffer too small");
        const uint64_t n = ctx->f_scene->n;
        if (ctx->f_bucket) {
            // tile ids from the ranges, depths from the {gid, depth} list
            const uint64_t T = static_cast<uint64_t>(ctx->f_tile_count);
            std::vector<uint2> rg(T);
            std::vector<uint2> gd(c.m);
            std::vector<uint32_t> pv(P);
            if (T) AGSX_CUDA(cudaMemcpy(rg.data(), ctx->ranges.p, T * 8, cudaMemcpyDeviceToHost));
            if (c.m) AGSX_CUDA(cudaMemcpy(gd.data(), ctx->bk_gd.p, c.m * 8, cudaMemcpyDeviceToHost));
            if (P) AGSX_CUDA(cudaMemcpy(pv.data(), ctx->f_pvals, P * 4, cudaMemcpyDeviceToHost));
            const std::vector<uint32_t> orig = scene_map_host(ctx->f_scene->orig, n);
            std::vector<uint32_t> depth_by_slot(n, 0);
            for (const uint2& e : gd) depth_by_slot[e.x] = e.y;  // the list and the values carry storage slots
            for (uint64_t t = 0; t < T; ++t)
                for (uint32_t i = rg[t].x; i < rg[t].y && i < P; ++i) {
                    if (keys) keys[i] = (t << 32) | depth_by_slot[pv[i]];
                    if (gids) gids[i] = orig.empty() ? pv[i] : orig[pv[i]];
                }
            return AGSX_OK;
        }
        std::vector<uint32_t> dk(c.m), dv(c.m), tk(P), pv(P);
        if (c.m) {
            const bool wide = depth_keys_wide_host(c);  // which ping-pong buffer holds the depth order
            AGSX_CUDA(cudaMemcpy(dk.data(), wide ? ctx->dkeys.p : ctx->dkeys2.p, c.m * 4, cudaMemcpyDeviceToHost));
            AGSX_CUDA(cudaMemcpy(dv.data(), wide ? ctx->dvals.p : ctx->dvals2.p, c.m * 4, cudaMemcpyDeviceToHost));
        }
        if (P) {
            AGSX_CUDA(cudaMemcpy(tk.data(), ctx->f_tkeys, P * 4, cudaMemcpyDeviceToHost));
            AGSX_CUDA(cudaMemcpy(pv.data(), ctx->f_pvals, P * 4, cudaMemcpyDeviceToHost));
        }
        const std::vector<uint32_t> orig = scene_map_host(ctx->f_scene->orig, n);
        std::vector<uint32_t> depth_by_slot(n, 0);  // the depth order and pairs carry storage slots
        for (uint32_t j = 0; j < c.m; ++j) depth_by_slot[dv[j]] = dk[j];
        for (uint64_t i = 0; i < P; ++i) {
            if (keys) keys[i] = (static_cast<uint64_t>(tk[i]) << 32) | depth_by_slot[pv[i]];
            if (gids) gids[i] = orig.empty() ? pv[i] : orig[pv[i]];
        }
        return AGSX_OK;
    });
}

int agsx_dump_ranges(agsx_ctx* ctx, uint32_t* ranges, uint64_t tile_count) {
    if (!ctx) return AGSX_EINVAL;
    return guarded(ctx, [&]() -> int {
        if (!ctx->have_frame) return fail(ctx, AGSX_EINVAL, "no frame rendered yet");
        if (tile_count != static_cast<uint64_t>(ctx->f_tile_count))
            return fail(ctx, AGSX_EINVAL, "tile count mismatch");
        AGSX_CUDA(cudaStreamSynchronize(ctx->stream));
        if (tile_count)
            AGSX_CUDA(cudaMemcpy(ranges, ctx->ranges.p, tile_count * 8, cudaMemcpyDeviceToHost));
        return AGSX_OK;
    });
}
}  // extern "C"

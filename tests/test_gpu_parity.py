"""GPU parity of the CUDA render path against the CPU oracle, through the C-ABI.

Bar (north star): per-Gaussian tile counts, survivor sets, total pairs,
sorted 64-bit (tile|depth) keys and tile ranges bit-exact; images bit-exact
with AGSX_FLAG_EXACT_ALPHA and within max-abs 1e-3 / PSNR >= 50 dB on the
default (hardware-exp, guard-banded) path.  Known-answer cases follow the
reference unit suites (file:line cited per test).
"""
import os

import numpy as np
import pytest

from paper_2604_18980_b200 import capi

pytestmark = pytest.mark.gpu

IMG_MAX_ABS = 1e-3  # north_star tolerance, per channel
IMG_MIN_PSNR = 50.0  # dB vs the oracle image

# calibrated AdaGScale parameters (reference `calibrate` on veil 100K 1080p)
K1080 = 0.3985099792480469
LUT_BINS = [1.0] * 20
LUT_BINS[7] = 0.003038157941773534
LUT_BINS[8] = 0.007012989837676287


def scene_pair(port, ctx, seed, count, layout, cams, w, h, focal):
    """Same synthetic scene for the oracle (its own generator) and the GPU (the product's)."""
    import paper_2604_18980_b200 as P

    o = port.synth_scene(seed, count, layout, cameras=cams, width=w, height=h, focal=focal)
    s = P.synth_scene(seed, count, layout, cameras=cams, width=w, height=h, focal=focal)
    a = s.arrays()
    for f in ("mean", "scale", "rotation", "opacity", "sh"):
        assert np.array_equal(a[f].reshape(-1).view(np.uint32), getattr(o, f).reshape(-1).view(np.uint32)), f
    dev = ctx.upload(a["mean"], a["scale"], a["rotation"], a["opacity"], a["sh"])
    return o, dev


def oracle_pipeline(port, scene, cam, cfg, lut):
    splats = port.preprocess(scene, cam, cfg, lut)
    keys, idx, counts = port.generate_pairs(splats, cam.width, cam.height, cfg.mode, cfg)
    tiles = ((cam.width + cfg.tile_size - 1) // cfg.tile_size) * ((cam.height + cfg.tile_size - 1) // cfg.tile_size)
    skeys, sidx, ranges = port.sort_pairs(keys, idx, tiles)
    img = port.raster(splats, skeys, sidx, ranges, cam.width, cam.height, cfg)
    return splats, counts, skeys, sidx, ranges, img


def gpu_cfg(mode, k=0.0, exact=False, **kw):
    return capi.default_config(mode, k, exact=exact, **kw)


def to_gpu_cam(c):
    g = capi.Camera()
    g.position[:] = list(c.position)
    g.rotation[:] = list(c.rotation)
    g.fx, g.fy, g.width, g.height = c.fx, c.fy, c.width, c.height
    return g


def psnr(a, b):
    d = a.astype(np.float64) - b.astype(np.float64)
    mse = np.mean(d * d)
    return np.inf if mse == 0 else 10 * np.log10(1.0 / mse)


def check_frame(ctx, port, oscene, dev, view, mode, k=0.0, lut_bins=None, exact=True, **kw):
    ocam = oscene.cameras[view]
    gcam = to_gpu_cam(ocam)
    ocfg = port.config(mode, k=k, **kw)
    gcfg = gpu_cfg(mode, k, exact=exact, **kw)
    olut = port.lut(lut_bins) if lut_bins is not None else None
    glut = capi.make_lut(lut_bins) if lut_bins is not None else (capi.make_lut() if mode == "adagscale" else None)
    splats, counts, skeys, sidx, ranges, oimg = oracle_pipeline(port, oscene, ocam, ocfg, olut)
    out = ctx.render(dev, gcam, gcfg, glut)
    n = oscene.count
    # survivors and per-Gaussian tile counts
    gcounts, galive = ctx.dump_tile_counts(n)
    alive = np.zeros(n, bool)
    alive[splats["source_id"]] = True
    ocounts = np.zeros(n, np.uint32)
    ocounts[splats["source_id"]] = counts
    assert out["splat_count"] == len(splats)
    assert np.array_equal(galive, alive)
    assert np.array_equal(gcounts, ocounts)
    assert out["pair_count"] == len(skeys)
    # sorted keys bit-exact; values map to the oracle's splat_index via source_id
    gkeys, ggids = ctx.dump_sorted_pairs()
    assert np.array_equal(gkeys, skeys)
    assert np.array_equal(ggids, splats["source_id"][sidx])
    tiles = len(ranges)
    assert np.array_equal(ctx.dump_ranges(tiles), ranges)
    img = out["image"]
    if exact:
        assert np.array_equal(img.view(np.uint32), oimg.view(np.uint32))
    else:
        assert np.max(np.abs(img - oimg)) <= IMG_MAX_ABS
        assert psnr(img, oimg) >= IMG_MIN_PSNR
    return out, oimg


def check_default_image(ctx, dev, ocam, mode, k, bins, oimg, pairs, **kw):
    """The default (fast, k_raster_units) image of the same frame against the
    oracle's image: max abs <= 1e-3 per channel, PSNR >= 50 dB."""
    out = ctx.render(dev, to_gpu_cam(ocam), gpu_cfg(mode, k, **kw), capi.make_lut(bins) if bins else
                     (capi.make_lut() if mode == "adagscale" else None))
    assert out["pair_count"] == pairs
    fast = out["image"]
    assert np.max(np.abs(fast - oimg)) <= IMG_MAX_ABS
    assert psnr(fast, oimg) >= IMG_MIN_PSNR
    return out


# --------------------------------------------------------------------------- full pipeline
@pytest.mark.parametrize("exact", [True, False], ids=["exact", "default"])
@pytest.mark.parametrize("layout", ["slab", "two_slab", "veil", "ramp", "aniso"])
@pytest.mark.parametrize("mode", ["aabb", "obb", "ellipse", "adagscale"])
def test_render_matches_oracle_small(ctx, port, layout, mode, exact):
    """The mode x layout matrix on both rasterisers: the glibc-exact one
    (bit-identical image) and the default fast one (k_raster_units, the path
    users and the bench run: max abs <= 1e-3, PSNR >= 50 dB)."""
    oscene, dev = scene_pair(port, ctx, 5, 3000, layout, 3, 320, 240, 250.0)
    check_frame(ctx, port, oscene, dev, 1, mode, k=0.3, lut_bins=[0.6] * 20 if mode == "adagscale" else None,
                exact=exact)


@pytest.mark.parametrize("exact", [True, False], ids=["exact", "default"])
@pytest.mark.parametrize("mode", ["ellipse", "adagscale"])
def test_render_opacities_at_the_clamp(ctx, port, mode, exact):
    """Opacities at and above alpha_at's clamp (0.99, rasterizer.hpp:44-50):
    the scene's maximum opacity selects the default rasteriser's clamp variant
    (a scene below the clamp runs the clamp-free one, as every synthetic
    layout does); the decisions and the clamped alphas match the oracle."""
    oscene, _ = scene_pair(port, ctx, 7, 3000, "slab", 2, 320, 240, 250.0)
    rng = np.random.default_rng(3)
    sel = rng.random(oscene.count) < 0.3
    oscene.opacity[sel] = rng.choice(np.float32([0.99, 0.99000007, 0.995, 0.9999999]), int(sel.sum()))
    dev = ctx.upload(oscene.mean, oscene.scale, oscene.rotation, oscene.opacity, oscene.sh)
    for view in range(2):
        check_frame(ctx, port, oscene, dev, view, mode, k=0.3, lut_bins=[0.6] * 20 if mode == "adagscale" else None,
                    exact=exact)


@pytest.mark.parametrize("exact", [True, False])
def test_render_config1_veil_adagscale(ctx, port, exact):
    """Config 1: veil 100K, 1920x1080, AdaGScale with the calibrated K/LUT."""
    oscene, dev = scene_pair(port, ctx, 1, 100_000, "veil", 16, 1920, 1080, 1500.0)
    out, _ = check_frame(ctx, port, oscene, dev, 0, "adagscale", k=K1080, lut_bins=LUT_BINS, exact=exact)
    assert out["pair_count"] == 2_357_743  # SURVEY.md §6 [measured] on the reference


@pytest.mark.slow
@pytest.mark.parametrize("mode,pairs", [("adagscale", 5_147_441), ("ellipse", 32_844_800)])
def test_render_config3_full_size_vs_reference(ctx, ref, mode, pairs):
    """Config 3 (veil 3M, 4608x3456) against the reference build itself
    (oracle/_ref): survivors, per-Gaussian tile counts, the 5.1M / 32.8M
    sorted (tile|depth) keys and tile ranges bit-exact; the glibc-exact image
    bit-identical; the default image within max-abs 1e-3 / PSNR >= 50 dB."""
    k = float(np.float32(K1080 * (3600.0 / 1500.0) ** 2))
    oscene, dev = scene_pair(ref, ctx, 1, 3_000_000, "veil", 16, 4608, 3456, 3600.0)
    bins = LUT_BINS if mode == "adagscale" else None
    out, oimg = check_frame(ctx, ref, oscene, dev, 0, mode, k=k if mode == "adagscale" else 0.0, lut_bins=bins,
                            exact=True)
    assert out["pair_count"] == pairs  # SURVEY.md §8(a) [measured] on the reference
    check_default_image(ctx, dev, oscene.cameras[0], mode, k if mode == "adagscale" else 0.0, bins, oimg, pairs)


@pytest.mark.parametrize("mode,fixed,pairs", [("aabb", 1, 27_942_602), ("ellipse", 0, 24_572_513)])
def test_render_config2_full_size_vs_reference(ctx, ref, mode, fixed, pairs):
    """Config 2 (veil 1M, 4608x3456): the original 3D-GS baseline (AABB with
    fixed_radius_aabb, r = 3) and Ellipse against the reference build itself:
    per-Gaussian tile counts, sorted keys and ranges bit-exact, the glibc-exact
    image bit-identical; pair totals as SURVEY.md §8(d) measured them."""
    oscene, dev = scene_pair(ref, ctx, 1, 1_000_000, "veil", 16, 4608, 3456, 3600.0)
    out, oimg = check_frame(ctx, ref, oscene, dev, 0, mode, exact=True, fixed_radius_aabb=fixed)
    assert out["pair_count"] == pairs
    check_default_image(ctx, dev, oscene.cameras[0], mode, 0.0, None, oimg, pairs, fixed_radius_aabb=fixed)


def test_render_config4_left_eye_vs_reference(ctx, ref):
    """Config 4 (veil 3M, one 3660x3200 eye, AdaGScale with K scaled to
    fx = 2859.375) against the reference build: tile counts, sorted keys,
    ranges and the glibc-exact image bit-exact; 4,125,726 pairs."""
    fx = 500.0 * 3660 / 640.0
    k = float(np.float32(K1080 * (fx / 1500.0) ** 2))
    oscene, dev = scene_pair(ref, ctx, 1, 3_000_000, "veil", 16, 3660, 3200, fx)
    out, oimg = check_frame(ctx, ref, oscene, dev, 0, "adagscale", k=k, lut_bins=LUT_BINS, exact=True)
    assert out["pair_count"] == 4_125_726
    check_default_image(ctx, dev, oscene.cameras[0], "adagscale", k, LUT_BINS, oimg, 4_125_726)


@pytest.mark.parametrize("view", [0, 37])
def test_render_config5_views_vs_reference(ctx, ref, view):
    """Config 5 (veil 6M, 4608x3456, a 64-view path): views of the path against
    the reference build, tile counts / keys / ranges / exact image bit-exact."""
    k = float(np.float32(K1080 * (3600.0 / 1500.0) ** 2))
    oscene, dev = scene_pair(ref, ctx, 1, 6_000_000, "veil", 64, 4608, 3456, 3600.0)
    out, oimg = check_frame(ctx, ref, oscene, dev, view, "adagscale", k=k, lut_bins=LUT_BINS, exact=True)
    check_default_image(ctx, dev, oscene.cameras[view], "adagscale", k, LUT_BINS, oimg, out["pair_count"])


def test_fast_alpha_within_tolerance(ctx, port):
    oscene, dev = scene_pair(port, ctx, 9, 4000, "veil", 2, 480, 320, 375.0)
    check_frame(ctx, port, oscene, dev, 0, "ellipse", exact=False)


def test_background_and_tile_sizes(ctx, port):
    oscene, dev = scene_pair(port, ctx, 53, 400, "slab", 2, 101, 77, 90.0)
    for ts in (8, 16, 32):
        check_frame(ctx, port, oscene, dev, 0, "ellipse", background=(0.2, 0.2, 0.2), tile_size=ts)
        check_frame(ctx, port, oscene, dev, 0, "aabb", background=(0.2, 0.2, 0.2), tile_size=ts)


def test_fixed_radius_aabb(ctx, port):
    oscene, dev = scene_pair(port, ctx, 3, 2000, "veil", 2, 320, 240, 250.0)
    check_frame(ctx, port, oscene, dev, 0, "aabb", fixed_radius_aabb=1)


def test_k0_adagscale_equals_ellipse(ctx, port):
    """test_rasterizer.cpp:152-165, acceptance.cpp:94-118."""
    oscene, dev = scene_pair(port, ctx, 41, 1000, "slab", 2, 640, 480, 500.0)
    cam = to_gpu_cam(oscene.cameras[0])
    a = ctx.render(dev, cam, gpu_cfg("ellipse"))
    b = ctx.render(dev, cam, gpu_cfg("adagscale", 0.0), capi.make_lut())
    assert a["pair_count"] == b["pair_count"] and a["splat_count"] == b["splat_count"]
    assert np.array_equal(a["image"], b["image"])


def test_lossless_modes_agree_bitwise(ctx, port):
    """test_rasterizer.cpp:133-150: AABB, OBB and Ellipse render identical images."""
    for layout in ("slab", "aniso"):
        oscene, dev = scene_pair(port, ctx, 37, 1200, layout, 2, 640, 480, 500.0)
        cam = to_gpu_cam(oscene.cameras[1])
        imgs = [ctx.render(dev, cam, gpu_cfg(m, exact=False)) for m in ("aabb", "obb", "ellipse")]
        assert np.array_equal(imgs[0]["image"], imgs[1]["image"])
        assert np.array_equal(imgs[1]["image"], imgs[2]["image"])
        assert imgs[2]["pair_count"] <= imgs[1]["pair_count"] <= imgs[0]["pair_count"]


def test_pair_budget_error(ctx, port):
    oscene, dev = scene_pair(port, ctx, 5, 3000, "slab", 2, 320, 240, 250.0)
    cam = to_gpu_cam(oscene.cameras[0])
    with pytest.raises(capi.PairBudgetError):
        ctx.render(dev, cam, gpu_cfg("ellipse", pair_budget=4))
    # the context stays usable
    out = ctx.render(dev, cam, gpu_cfg("ellipse"))
    assert out["pair_count"] > 4


def test_pair_arena_regrows_and_budget_boundary(port):
    """More pairs than the first-guess pair arena (max(12 N, 2^20)): the frame
    is re-run with a grown arena and still matches the oracle; a budget of
    exactly P passes, P - 1 raises (pair_gen.cpp:181-184: P > budget)."""
    ctx = capi.Context(0)  # fresh context: arena at its first guess
    try:
        o = port.synth_scene(2, 2000, "slab", cameras=2, width=640, height=480, focal=500.0)
        o.scale[:] *= 40.0  # every splat covers most of the 1200 tiles -> P >> 2^20
        dev = ctx.upload(o.mean, o.scale, o.rotation, o.opacity, o.sh)
        out, _ = check_frame(ctx, port, o, dev, 0, "aabb", exact=True)
        p = out["pair_count"]
        assert p > (1 << 20)
        cam = to_gpu_cam(o.cameras[0])
        assert ctx.render(dev, cam, gpu_cfg("aabb", pair_budget=p))["pair_count"] == p
        with pytest.raises(capi.PairBudgetError):
            ctx.render(dev, cam, gpu_cfg("aabb", pair_budget=p - 1))
    finally:
        ctx.close()


def test_invalid_config_and_camera(ctx, port):
    oscene, dev = scene_pair(port, ctx, 5, 100, "slab", 2, 64, 48, 100.0)
    cam = to_gpu_cam(oscene.cameras[0])
    with pytest.raises(capi.AgsxError) as e:
        ctx.render(dev, cam, gpu_cfg("ellipse", alpha_threshold=2.0))
    assert e.value.code == capi.EINVAL
    with pytest.raises(capi.AgsxError) as e:
        ctx.render(dev, cam, gpu_cfg("adagscale"), None)  # adagscale needs a LUT
    assert e.value.code == capi.EINVAL
    bad = to_gpu_cam(oscene.cameras[0])
    bad.rotation[0] = 2.0
    with pytest.raises(capi.AgsxError):
        ctx.render(dev, bad, gpu_cfg("ellipse"))


def test_empty_scene_renders_background(ctx):
    """test_rasterizer.cpp:97-114."""
    dev = ctx.upload(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 4)), np.zeros(0), np.zeros((0, 1, 3)))
    cam = capi.Camera()
    cam.rotation[:] = [1, 0, 0, 0, 1, 0, 0, 0, 1]
    cam.fx = cam.fy = 100.0
    cam.width, cam.height = 64, 48
    out = ctx.render(dev, cam, gpu_cfg("ellipse", background=(0.1, 0.2, 0.3)))
    assert out["pair_count"] == 0 and out["splat_count"] == 0
    assert out["image"][10, 10, 0] == np.float32(0.1)
    assert out["image"][47, 63, 2] == np.float32(0.3)


def test_max_t_matches_oracle(ctx, port, ref):
    """test_rasterizer.cpp:180-219: max transmittance instrumentation, exact."""
    oscene, dev = scene_pair(port, ctx, 47, 400, "slab", 2, 640, 480, 500.0)
    ocam = oscene.cameras[0]
    rscene = ref.synth_scene(47, 400, "slab", cameras=2)
    want = ref.render(rscene, rscene.cameras[0], ref.config("ellipse"), max_t=True)
    out = ctx.render(dev, to_gpu_cam(ocam), gpu_cfg("ellipse", exact=True), max_t=True, n=400)
    _, alive = ctx.dump_tile_counts(400)
    got = out["max_t_by_gid"][alive]
    assert np.array_equal(got.view(np.uint32), want["max_t"].view(np.uint32))


# --------------------------------------------------------------------------- stage API
def splat(mean, cov, opacity, th, depth=5.0, rgb=(1, 1, 1)):
    s = np.zeros(1, capi.SPLAT_DTYPE)
    s["mean2d"] = mean
    s["cov2d"] = cov
    det = np.float32(cov[0]) * np.float32(cov[2]) - np.float32(cov[1]) * np.float32(cov[1])
    inv = np.float32(1.0) / np.float32(det)
    s["inv_cov"] = [np.float32(cov[2]) * inv, -np.float32(cov[1]) * inv, np.float32(cov[0]) * inv]
    s["depth"] = depth
    s["rgb"] = rgb
    s["opacity"] = opacity
    s["th"] = th
    return s


def test_one_tile_splat_all_modes(ctx):
    """test_pair_gen.cpp:55-66."""
    s = splat((24, 24), (4, 0, 4), 0.99, 1 / 255)
    for m in ("aabb", "obb", "ellipse", "adagscale"):
        keys, idx, counts = ctx.generate_pairs(s, 64, 64, m, gpu_cfg(m))
        assert list(counts) == [1]
        assert keys[0] >> 32 == 1 * 4 + 1


def test_five_tile_splat(ctx):
    """test_pair_gen.cpp:205-225: tiles 298..302 in emission order."""
    s = splat((328, 120), (81, 0, 2.25), 0.99, 1 / 255)
    keys, idx, counts = ctx.generate_pairs(s, 640, 480, "ellipse", gpu_cfg("ellipse"))
    assert list(counts) == [5]
    assert [int(k >> 32) for k in keys] == [298, 299, 300, 301, 302]
    assert all((k & 0xFFFFFFFF) == 0x40A00000 for k in keys)  # bits of depth 5.0
    with pytest.raises(capi.PairBudgetError):
        ctx.generate_pairs(s, 640, 480, "ellipse", gpu_cfg("ellipse", pair_budget=4))


def test_offscreen_and_empty(ctx):
    """test_pair_gen.cpp:227-237."""
    keys, idx, counts = ctx.generate_pairs(np.zeros(0, capi.SPLAT_DTYPE), 64, 64, "ellipse", gpu_cfg("ellipse"))
    assert len(keys) == 0
    s = splat((-500, -500), (4, 0, 4), 0.9, 1 / 255)
    keys, idx, counts = ctx.generate_pairs(s, 64, 64, "ellipse", gpu_cfg("ellipse"))
    assert list(counts) == [0]


def test_generate_pairs_random_splats_vs_oracle(ctx, port):
    """Random splats incl. off-image centres (test_pair_gen.cpp:117-144 distribution)."""
    rng = np.random.default_rng(21)
    n = 3000
    a, b, c, d = (rng.uniform(-20, 20, n).astype(np.float32) for _ in range(4))
    s = np.zeros(n, capi.SPLAT_DTYPE)
    cov = np.stack([a * a + b * b + np.float32(0.4), a * c + b * d, c * c + d * d + np.float32(0.4)], 1).astype(np.float32)
    det = cov[:, 0] * cov[:, 2] - cov[:, 1] * cov[:, 1]
    inv = np.float32(1) / det
    s["cov2d"] = cov
    s["inv_cov"] = np.stack([cov[:, 2] * inv, -cov[:, 1] * inv, cov[:, 0] * inv], 1)
    s["mean2d"] = np.stack([rng.uniform(-50, 690, n), rng.uniform(-50, 530, n)], 1)
    op = rng.uniform(0.05, 0.99, n).astype(np.float32)
    s["opacity"] = op
    s["th"] = np.maximum(np.minimum(op * rng.uniform(0.1, 0.9, n).astype(np.float32), op - np.float32(1e-4)),
                         np.float32(1 / 255))
    s["depth"] = rng.uniform(0.3, 90, n)
    for m in ("aabb", "obb", "ellipse", "adagscale"):
        ok = port.generate_pairs(s, 640, 480, m, port.config(m))
        gk = ctx.generate_pairs(s, 640, 480, m, gpu_cfg(m))
        for x, y in zip(gk, ok):
            assert np.array_equal(x, y), m


def test_sort_matches_stable_sort(ctx):
    """test_pair_sort.cpp:31-52 (1e5, coarse depths -> many equal keys) and acceptance C7 (1e6)."""
    for n, tiles, seed in ((100_000, 300, 17), (1_000_000, 62_208, 515)):
        rng = np.random.default_rng(seed)
        depth = (0.25 * (1 + rng.integers(0, 64, n))).astype(np.float32)
        keys = (rng.integers(0, tiles, n).astype(np.uint64) << np.uint64(32)) | depth.view(np.uint32).astype(np.uint64)
        idx = np.arange(n, dtype=np.uint32)
        order = np.argsort(keys, kind="stable")
        gk, gi, gr = ctx.sort_pairs(keys, idx, tiles)
        assert np.array_equal(gk, keys[order])
        assert np.array_equal(gi, idx[order])
        t = (gk >> np.uint64(32)).astype(np.int64)
        for tile in (0, tiles // 2, tiles - 1):
            hit = np.nonzero(t == tile)[0]
            want = (hit[0], hit[-1] + 1) if len(hit) else (0, 0)
            assert tuple(gr[tile]) == want


def test_sort_edge_cases(ctx):
    """test_pair_sort.cpp:12-29, 94-103."""
    gk, gi, gr = ctx.sort_pairs(np.zeros(0, np.uint64), np.zeros(0, np.uint32), 12)
    assert len(gk) == 0 and np.all(gr == 0)
    k = np.array([(4 << 32) | 0x40000000, (4 << 32) | 0x3F800000], np.uint64)
    gk, gi, gr = ctx.sort_pairs(k, np.array([0, 1], np.uint32), 8)
    assert list(gi) == [1, 0] and tuple(gr[4]) == (0, 2) and tuple(gr[3]) == (0, 0)
    keys = np.array([(7 << 32) | 0x40500000] * 64 + [(2 << 32) | 0x41100000], np.uint64)
    idx = np.array(list(range(64)) + [999], np.uint32)
    gk, gi, gr = ctx.sort_pairs(keys, idx, 16)
    assert gi[0] == 999 and list(gi[1:]) == list(range(64))
    # arbitrary 64-bit keys, tiles past tile_count are sorted but get no range
    rng = np.random.default_rng(5)
    keys = rng.integers(0, 2**63, 50_000, dtype=np.uint64)
    gk, gi, gr = ctx.sort_pairs(keys, np.arange(50_000, dtype=np.uint32), 4)
    assert np.array_equal(gk, np.sort(keys, kind="stable"))


def test_raster_known_answers(ctx, port):
    """test_rasterizer.cpp:60-95."""
    def flat(mean, sigma, op, rgb, depth):
        return splat(mean, (sigma * sigma, 0, sigma * sigma), op, 1 / 255, depth, rgb)

    def raster(splats, w, h, cfg):
        keys, idx, counts = ctx.generate_pairs(splats, w, h, "ellipse", cfg)
        tiles = ((w + 15) // 16) * ((h + 15) // 16)
        sk, si, rg = ctx.sort_pairs(keys, idx, tiles)
        return ctx.raster(splats, si, rg, w, h, cfg)

    img = raster(flat((8, 8), 1e4, 0.5, (1, 1, 1), 1.0), 16, 16, gpu_cfg("ellipse", exact=True))
    assert abs(img[8, 8, 0] - 0.5) < 1e-4 and abs(img[12, 3, 1] - 0.5) < 1e-4
    two = np.concatenate([flat((8, 8), 1e4, 0.5, (1, 1, 1), 1.0), flat((8, 8), 1e4, 0.5, (0, 0, 0), 2.0)])
    img = raster(two, 16, 16, gpu_cfg("ellipse", exact=True, background=(1, 1, 1)))
    assert abs(img[8, 8, 0] - 0.75) < 1e-4
    img = raster(flat((8, 8), 1e4, 0.001, (1, 1, 1), 1.0), 16, 16,
                 gpu_cfg("ellipse", exact=True, background=(0.25, 0.5, 0.75)))
    assert img[8, 8, 0] == np.float32(0.25) and img[8, 8, 1] == np.float32(0.5) and img[8, 8, 2] == np.float32(0.75)


def test_raster_extreme_splats_default_vs_oracle(ctx, port):
    """The default rasteriser's unit-centred exponent and its widened
    thresholds on splats far from the synthetic scenes: condition
    numbers up to 1e5 (the fp64 blend-cull data and the all-exact fallback),
    sub-pixel and 300-pixel footprints, centres far outside the image,
    opacities from tau to 1 (the clamp variant of the stage path), every
    alpha >= tau decision the reference's: max abs <= 1e-3, PSNR >= 50 dB."""
    rng = np.random.default_rng(77)
    n, w, h = 4000, 333, 250
    theta = rng.uniform(0, np.pi, n)
    major = np.exp(rng.uniform(np.log(0.3), np.log(300.0), n))
    kappa = np.exp(rng.uniform(0, np.log(1e5), n))
    minor = np.maximum(major / np.sqrt(kappa), 0.05)
    c, sn = np.cos(theta), np.sin(theta)
    cxx = major**2 * c * c + minor**2 * sn * sn
    cyy = major**2 * sn * sn + minor**2 * c * c
    cxy = (major**2 - minor**2) * c * sn
    cov = np.stack([cxx, cxy, cyy], 1).astype(np.float32)
    det = cov[:, 0] * cov[:, 2] - cov[:, 1] * cov[:, 1]
    keep = det > 0
    cov, det = cov[keep], det[keep]
    m = len(cov)
    s = np.zeros(m, capi.SPLAT_DTYPE)
    inv = np.float32(1) / det
    s["cov2d"] = cov
    s["inv_cov"] = np.stack([cov[:, 2] * inv, -cov[:, 1] * inv, cov[:, 0] * inv], 1)
    s["mean2d"] = np.stack([rng.uniform(-400, w + 400, m), rng.uniform(-400, h + 400, m)], 1)
    op = rng.choice(np.float32([1 / 255 + 1e-6, 0.02, 0.3, 0.7, 0.98, 0.99, 0.999, 1.0]), m)
    s["opacity"] = op
    s["th"] = np.float32(1 / 255)
    s["depth"] = rng.uniform(0.3, 90, m)
    s["rgb"] = rng.uniform(0, 1, (m, 3))
    tiles = ((w + 15) // 16) * ((h + 15) // 16)
    ocfg = port.config("ellipse")
    okeys, oidx, _ = port.generate_pairs(s, w, h, "ellipse", ocfg)
    osk, osi, org = port.sort_pairs(okeys, oidx, tiles)
    want = port.raster(s, osk, osi, org, w, h, ocfg)
    keys, idx, _ = ctx.generate_pairs(s, w, h, "ellipse", gpu_cfg("ellipse"))
    sk, si, rg = ctx.sort_pairs(keys, idx, tiles)
    assert np.array_equal(sk, osk) and np.array_equal(si, osi)
    exact = ctx.raster(s, si, rg, w, h, gpu_cfg("ellipse", exact=True))
    assert np.array_equal(exact.view(np.uint32), want.view(np.uint32))
    got = ctx.raster(s, si, rg, w, h, gpu_cfg("ellipse"))
    assert np.max(np.abs(got - want)) <= IMG_MAX_ABS
    assert psnr(got, want) >= IMG_MIN_PSNR


def test_stage_preprocess_matches_oracle(ctx, port):
    oscene, dev = scene_pair(port, ctx, 2, 3000, "ramp", 2, 640, 480, 500.0)
    for mode, k, bins in (("ellipse", 0.0, None), ("adagscale", 0.5, [0.7] * 20)):
        ocfg = port.config(mode, k=k)
        want = port.preprocess(oscene, oscene.cameras[0], ocfg, port.lut(bins) if bins else None)
        got = ctx.preprocess_view(dev, to_gpu_cam(oscene.cameras[0]), gpu_cfg(mode, k),
                                  capi.make_lut(bins) if bins else None)
        assert got.tobytes() == want.tobytes()


# --------------------------------------------------------------------------- device libm
def test_device_logf_matches_host_glibc(ctx, port):
    """glibc-exact logf on device over every float in [1, 256) and samples elsewhere."""
    bits = np.arange(0x3F800000, 0x43800000, dtype=np.uint32)
    x = bits.view(np.float32)
    assert np.array_equal(ctx.logf(x).view(np.uint32), port.logf(x).view(np.uint32))
    rng = np.random.default_rng(0)
    x = rng.integers(1, 0x7F800000, 4_000_000, dtype=np.uint32).view(np.float32)
    assert np.array_equal(ctx.logf(x).view(np.uint32), port.logf(x).view(np.uint32))


def test_device_expf_matches_host_glibc(ctx, port):
    """glibc-exact expf on device over every float in [-20, -0] and samples down to -110."""
    bits = np.arange(0x80000000, 0xC1A00001, dtype=np.uint32)
    for chunk in np.array_split(bits, 8):
        x = chunk.view(np.float32)
        assert np.array_equal(ctx.expf(x).view(np.uint32), port.expf(x).view(np.uint32))
    x = np.linspace(-110, 88, 3_000_000, dtype=np.float32)
    assert np.array_equal(ctx.expf(x).view(np.uint32), port.expf(x).view(np.uint32))


def test_multiview_single_rank_gpu(port):
    """multiview driver on the CUDA path: frames rasterised into torch slots
    (render_async_to) in camera-path order; stereo eye via a camera override."""
    import torch

    import paper_2604_18980_b200 as P
    from oracle.ffi import camera_from_dict
    from paper_2604_18980_b200.multiview import MultiViewRenderer, gpu_render_into, stereo_cameras

    spec = dict(seed=5, count=3000, layout="veil", cameras=4, width=160, height=96, focal=120.0)
    s = P.synth_scene(**spec)
    o = port.synth_scene(**spec)
    r = P.Renderer(0)
    mv = MultiViewRenderer(gpu_render_into(r), device="cuda")
    frames, stats = mv.render_path(s, 4, 96, 160, mode="ellipse")
    frames = frames.cpu().numpy()
    total = 0
    for v in range(4):
        want = port.render(o, o.cameras[v], port.config("ellipse"))
        total += want["pair_count"]
        assert np.max(np.abs(frames[v] - want["image"])) <= IMG_MAX_ABS
        assert stats.per_view_pairs[v] == want["pair_count"]
    assert stats.frames == 4 and stats.pair_count == total
    left, right = stereo_cameras(s.camera(0))
    slot = torch.empty((96, 160, 3), dtype=torch.float32, device="cuda")
    r.render_async_to(s, 0, slot.data_ptr(), "ellipse", camera=right)
    st = r.wait()
    want = port.render(o, camera_from_dict(right), port.config("ellipse"))
    assert st["pair_count"] == want["pair_count"]
    assert np.max(np.abs(slot.cpu().numpy() - want["image"])) <= IMG_MAX_ABS


def test_calibrate_matches_reference_golden():
    """GPU calibration (next row f1) against the reference's build_lut +
    search_k (calibrate.cpp:14-155) on tests/golden/calibration_veil3000.json
    (made by tests/golden/gen_calibration.py from the reference build).  The
    renders are glibc-exact, so the LUT (max_t folds) is bit-identical; K and
    the achieved drop come from the same 22-step bisection."""
    import json
    import os

    import paper_2604_18980_b200 as P

    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "calibration_veil3000.json")))
    s = P.synth_scene(**g["spec"])
    out = P.calibrate(s, g["target_drop"], g["calib_views"])
    assert np.array_equal(np.float32(out["lut_bins"]).view(np.uint32), np.float32(g["lut_bins"]).view(np.uint32))
    assert out["iterations"] == g["iterations"]
    assert out["k"] == g["k"]
    assert abs(out["achieved_drop"] - g["achieved_drop"]) < 1e-9
    assert (out["lut_depth_min"], out["lut_depth_max"]) == (g["lut_depth_min"], g["lut_depth_max"])


def test_calibrate_config1_veil_reproduces_survey_parameters():
    """Full-size calibration (veil 100K, 1920x1080, 16 views, 0.5 dB): the
    reference produced K = 0.3985099792480469 with LUT bins[7] =
    0.003038157941773534, bins[8] = 0.007012989837676287 and every other bin
    1.0 (SURVEY.md §8(d), 176 s on 8 CPU threads).  The GPU run must land on
    the same parameters."""
    import time

    import paper_2604_18980_b200 as P

    s = P.synth_scene(1, 100_000, "veil", cameras=16, width=1920, height=1080, focal=1500.0)
    t = time.time()
    out = P.calibrate(s, 0.5, 16)
    dt = time.time() - t
    assert out["k"] == K1080
    assert np.array_equal(np.float32(out["lut_bins"]), np.float32(LUT_BINS))
    assert abs(out["achieved_drop"] - 0.499) < 1e-3
    print(f"GPU calibration: {dt:.2f} s, {out['iterations']} drop evaluations")


@pytest.mark.parametrize("degree", [1, 3])
def test_ply_scene_sh_degrees_render(tmp_path, port, degree):
    """A PLY-ingested scene (row f2) with SH degree 1 / 3 through the device
    path vs the oracle: counts and keys bit-exact, image within tolerance."""
    import sys

    sys.path.insert(0, os.path.dirname(__file__))
    from plyfixture import write_ply

    import paper_2604_18980_b200 as P
    from oracle.ffi import SoAScene, camera_from_dict

    path = str(tmp_path / "s.ply")
    write_ply(path, n=4000, degree=degree, seed=degree)
    s = P.load_ply(path, orbit_views=3, width=256, height=192, focal=200.0, seed=2)
    a = s.arrays()
    o = SoAScene(a["mean"].copy(), a["scale"].copy(), a["rotation"].copy(), a["opacity"].copy(), a["sh"].copy(), [])
    r = P.Renderer(0)
    for v in range(3):
        cam = s.camera(v)
        got = r.render(s, v, "ellipse")
        want = port.render(o, camera_from_dict(cam), port.config("ellipse"))
        assert got["pair_count"] == want["pair_count"] and got["splat_count"] == want["splat_count"]
        assert np.max(np.abs(got["image"] - want["image"])) <= IMG_MAX_ABS
        ex = r.render(s, v, "ellipse", exact=True)["image"]
        assert np.array_equal(ex.view(np.uint32), want["image"].view(np.uint32))


def test_render_u8_egress_matches_host_quantisation(ctx, port):
    """Row f3: the device-quantised PPM bytes equal write_image's
    lround(clamp(v) * 255) of the f32 frame (gsio.cpp:265-281), through the
    pinned zero-copy path and the pageable copy path."""
    import ctypes as C

    import paper_2604_18980_b200 as P

    s = P.synth_scene(4, 5000, "veil", cameras=2, width=333, height=211, focal=260.0)  # n % 16 != 0
    r = P.Renderer(0)
    f32 = r.render(s, 1, "adagscale", 0.3, [0.7] * 20, exact=True)["image"]
    want = np.floor(np.clip(f32, 0, 1).astype(np.float64) * 255.0 + 0.5).astype(np.uint8)
    got = r.render(s, 1, "adagscale", 0.3, [0.7] * 20, exact=True, image_u8=True)["image"]
    assert got.dtype == np.uint8 and np.array_equal(got, want)
    a = s.arrays()
    dev = ctx.upload(a["mean"], a["scale"], a["rotation"], a["opacity"], a["sh"])
    cam = capi.Camera.from_dict(s.camera(1))
    buf = np.zeros((211, 333, 3), np.uint8)  # pageable: staged copy
    f = capi.Frame()
    rc = ctx.L.agsx_render_u8(ctx.h, dev, C.byref(cam), C.byref(gpu_cfg("adagscale", 0.3, exact=True)),
                              C.byref(capi.make_lut([0.7] * 20)), buf.ctypes.data, C.byref(f))
    assert rc == 0 and np.array_equal(buf, want)
    # default rasterizer: banded egress, each band quantised on the device and
    # copied behind the raster (band lengths not multiples of 16 bytes)
    f32 = r.render(s, 1, "adagscale", 0.3, [0.7] * 20)["image"]
    want = np.floor(np.clip(f32, 0, 1).astype(np.float64) * 255.0 + 0.5).astype(np.uint8)
    got = r.render(s, 1, "adagscale", 0.3, [0.7] * 20, image_u8=True)["image"]
    assert np.array_equal(got, want)
    buf[:] = 0
    rc = ctx.L.agsx_render_u8(ctx.h, dev, C.byref(cam), C.byref(gpu_cfg("adagscale", 0.3)),
                              C.byref(capi.make_lut([0.7] * 20)), buf.ctypes.data, C.byref(f))
    assert rc == 0 and np.array_equal(buf, want)


@pytest.mark.parametrize("egress", ["launches", "zerocopy"])
def test_egress_variants_identical(monkeypatch, egress):
    """The host egress variants deliver the same frame: banded in one raster
    launch with device band counts (default), one raster launch per band
    (AGSX_EGRESS=launches, drivers without stream wait-value) and zero-copy
    SM stores into the mapped buffer (AGSX_EGRESS=zerocopy); f32 and PPM."""
    import paper_2604_18980_b200 as P

    s = P.synth_scene(6, 20000, "veil", cameras=2, width=347, height=261, focal=270.0)
    r = P.Renderer(0)
    ref = r.render(s, 1, "adagscale", 0.3, [0.7] * 20)
    ref8 = r.render(s, 1, "adagscale", 0.3, [0.7] * 20, image_u8=True)
    monkeypatch.setenv("AGSX_EGRESS", egress)
    out = r.render(s, 1, "adagscale", 0.3, [0.7] * 20)
    out8 = r.render(s, 1, "adagscale", 0.3, [0.7] * 20, image_u8=True)
    assert np.array_equal(out["image"].view(np.uint32), ref["image"].view(np.uint32))
    assert np.array_equal(out8["image"], ref8["image"])
    assert out["pair_count"] == ref["pair_count"]


@pytest.mark.parametrize("layout,mode,ts", [("veil", "adagscale", 16), ("slab", "ellipse", 16), ("aniso", "obb", 8),
                                           ("ramp", "aabb", 32), ("two_slab", "ellipse", 64)])
def test_contributions_match_oracle(ctx, port, layout, mode, ts):
    """agsx_render_contributions (RecordOptions::contributions, rasterizer.cpp:21-100,
    135-161): every blend event {pixel, view splat index, alpha, weight} bit-exact
    and in the reference's order, the image bit-exact; the capacity protocol."""
    import ctypes as C

    oscene, dev = scene_pair(port, ctx, 12, 2500, layout, 2, 200, 136, 160.0)
    ocfg = port.config(mode, k=0.4, tile_size=ts)
    gcfg = gpu_cfg(mode, 0.4, tile_size=ts)
    olut = port.lut([0.6] * 20)
    glut = capi.make_lut([0.6] * 20)
    want_img, want = port.render_contributions(oscene, oscene.cameras[1], ocfg, olut)
    img, got = ctx.render_contributions(dev, to_gpu_cam(oscene.cameras[1]), gcfg, glut)
    assert len(want) > 1000 and len(got) == len(want)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    assert np.array_equal(img.view(np.uint32), want_img.view(np.uint32))
    count = C.c_uint64()
    small = np.zeros(10, capi.BLEND_DTYPE)
    rc = ctx.L.agsx_render_contributions(ctx.h, dev, C.byref(to_gpu_cam(oscene.cameras[1])), C.byref(gcfg),
                                         C.byref(glut), small.ctypes.data_as(C.c_void_p), 10, C.byref(count), None)
    assert rc == 5 and count.value == len(want)


@pytest.mark.parametrize("env", ["AGSX_RASTER_STATS=1"])
def test_raster_diagnostic_variants(tmp_path, env):
    """The diagnostic rasterizer variant (work counters, AGSX_RASTER_STATS)
    renders the same frame as the default one (counters: iterations and live
    evaluations reported, every fast blend counted once)."""
    import subprocess
    import sys

    code = (
        "import sys, numpy as np; sys.path.insert(0, '.'); import paper_2604_18980_b200 as P\n"
        "s = P.synth_scene(3, 20000, 'veil', cameras=2, width=320, height=240, focal=250.0)\n"
        "r = P.Renderer(0); r.render_async(s, 1, 'adagscale', 0.3, [0.7] * 20); r.wait()\n"
        "img = P.render(s, 1, 'adagscale', 0.3, [0.7] * 20)['image']\n"
        "np.save(sys.argv[1], img); st = r.frame_stats()\n"
        "print(st['raster_iters'], st['raster_evals'], st['raster_fast'])\n")
    root = os.path.dirname(os.path.dirname(__file__))
    base = subprocess.run([sys.executable, "-c", code, str(tmp_path / "a.npy")], cwd=root, check=True,
                          capture_output=True, text=True)
    k, v = env.split("=")
    var = subprocess.run([sys.executable, "-c", code, str(tmp_path / "b.npy")], cwd=root, check=True,
                         capture_output=True, text=True, env={**os.environ, k: v})
    a, b = np.load(tmp_path / "a.npy"), np.load(tmp_path / "b.npy")
    if k == "AGSX_RASTER_STATS":
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
        it, ev, fast = (int(x) for x in var.stdout.split())
        assert it > 0 and ev > 0 and 0 < fast <= ev
        assert base.stdout.split() == ["0", "0", "0"]  # counters off by default
    else:  # the rect cull only drops splats that reach no pixel centre: same alpha >= tau decisions
        assert np.max(np.abs(a - b)) <= 1e-4


def test_psnr_device_matches_reference_formula():
    import torch

    import paper_2604_18980_b200 as P

    a = torch.rand(3 * 1000, device="cuda")
    b = a + 0.01 * torch.randn(3 * 1000, device="cuda")
    r = P.Renderer(0)
    got = r.psnr_device(a.data_ptr(), b.data_ptr(), a.numel())
    want = P.psnr(a.cpu().numpy().reshape(1, 1000, 3), b.cpu().numpy().reshape(1, 1000, 3))
    assert abs(got - want) < 1e-9
    assert r.psnr_device(a.data_ptr(), a.data_ptr(), a.numel()) == float("inf")


def test_pair_report_matches_reference(ref):
    """Row f4: pair_report (analysis.cpp:259-312) on the device vs the
    reference build: pair counts and reductions exact, PSNR drops equal up to
    the summation order of the squared errors."""
    import paper_2604_18980_b200 as P

    spec = dict(seed=6, count=4000, layout="veil", cameras=3, width=320, height=240, focal=250.0)
    s = P.synth_scene(**spec)
    o = ref.synth_scene(**spec)
    specs = [("ellipse", 0.0), ("aabb", 0.0), ("adagscale", 0.3), ("adagscale", 0.8)]
    bins = [0.6] * 20
    got = P.Renderer(0).pair_report(s, specs, views=[0, 1, 2], lut_bins=bins)
    want = ref.pair_report(o, 3, specs, ref.lut(bins))
    for g, (pc, red, drop) in zip(got, want):
        assert g["pair_count"] == int(pc)
        assert g["reduction_pct"] == red
        assert abs(g["psnr_drop_db"] - drop) < 1e-9
    csv = P.pair_report_csv(got)
    assert csv.splitlines()[0].startswith("mode,k,pair_count,reduction_vs_ellipse_pct")
    # no LUT given: the reference builds it from all the views (analysis.cpp:265-275);
    # batch.device_pair_report folds view blocks and merges them (here one rank)
    from paper_2604_18980_b200.batch import device_pair_report

    r = P.Renderer(0)
    want = ref.pair_report(o, 3, specs)
    for got in (r.pair_report(s, specs, views=[0, 1, 2]), device_pair_report(r, s, specs, 3)):
        for g, (pc, red, drop) in zip(got, want):
            assert g["pair_count"] == int(pc)
            assert g["reduction_pct"] == red
            assert abs(g["psnr_drop_db"] - drop) < 1e-9
    # the merged fold of two view blocks is the fold of all views
    from paper_2604_18980_b200.batch import merge_folds

    whole = merge_folds([r.fold_max_t(s, [0, 1, 2])])
    split = merge_folds([r.fold_max_t(s, [0, 1]), r.fold_max_t(s, [2])])
    assert whole == split
    assert P.format_double(100.0) == "100" and P.format_double(0.5) == "0.5"


def test_multiview_pipelined_two_contexts(port):
    """Camera path on two contexts of one GPU (frames alternate streams):
    same frames and stats as the oracle, in path order."""
    import paper_2604_18980_b200 as P
    from paper_2604_18980_b200.multiview import MultiViewRenderer, gpu_render_pipelined

    spec = dict(seed=5, count=3000, layout="veil", cameras=5, width=160, height=96, focal=120.0)
    s = P.synth_scene(**spec)
    o = port.synth_scene(**spec)
    mv = MultiViewRenderer(batch=gpu_render_pipelined([P.Renderer(0), P.Renderer(0)]), device="cuda")
    frames, stats = mv.render_path(s, 5, 96, 160, mode="ellipse", exact=True)
    frames = frames.cpu().numpy()
    for v in range(5):
        want = port.render(o, o.cameras[v], port.config("ellipse"))
        assert np.array_equal(frames[v].view(np.uint32), want["image"].view(np.uint32))
        assert stats.per_view_pairs[v] == want["pair_count"]


@pytest.mark.parametrize("n_ctx", [1, 2])
def test_render_views_host_pipelined(port, n_ctx):
    """batch.render_views: frames delivered to page-locked host images with one
    frame in flight per context. Each view's image is bit-identical to the
    single-call render() (same kernels, banded egress) and, in exact mode, to
    the oracle; results come back in path order, also through on_frame."""
    import paper_2604_18980_b200 as P
    from paper_2604_18980_b200.batch import render_views

    spec = dict(seed=9, count=4000, layout="veil", cameras=6, width=200, height=136, focal=150.0)
    s = P.synth_scene(**spec)
    o = port.synth_scene(**spec)
    rs = [P.Renderer(0) for _ in range(n_ctx)]
    views = [3, 0, 5, 1, 4, 2]
    outs = render_views(rs, s, views, mode="ellipse")
    for v, out in zip(views, outs):
        ref = P.render(s, view=v, mode="ellipse")
        assert out["image"].shape == (136, 200, 3)
        assert np.array_equal(out["image"].view(np.uint32), ref["image"].view(np.uint32)), v
        assert out["pair_count"] == ref["pair_count"] and out["splat_count"] == ref["splat_count"]
    outs8 = render_views(rs, s, views, mode="ellipse", image_u8=True)  # banded PPM egress
    for v, out in zip(views, outs8):
        ref8 = P.render(s, view=v, mode="ellipse", image_u8=True)
        assert out["image"].dtype == np.uint8 and np.array_equal(out["image"], ref8["image"]), v
        assert out["pair_count"] == ref8["pair_count"]
    rs[0].render_async_host(s, 0, mode="ellipse")
    with pytest.raises(RuntimeError):  # its image is still being written
        rs[0].render_async_host(s, 1, mode="ellipse")
    with pytest.raises(RuntimeError):
        rs[0].render_async(s, 1, mode="ellipse")
    assert rs[0].wait()["image"].shape == (136, 200, 3)
    got = {}
    render_views(rs, s, views, on_frame=lambda i, out: got.__setitem__(i, out), mode="ellipse", exact=True)
    assert sorted(got) == list(range(len(views)))
    for i, v in enumerate(views):
        want = port.render(o, o.cameras[v], port.config("ellipse"))
        assert np.array_equal(got[i]["image"].view(np.uint32), want["image"].view(np.uint32)), v


@pytest.mark.parametrize("layout,mode,k,lutbin", [("veil", "adagscale", 0.3, 0.6), ("slab", "ellipse", 0.0, None),
                                                  ("aniso", "obb", 0.0, None)])
def test_cxx_drop_in_caller(tmp_path, port, layout, mode, k, lutbin):
    """A C++ program written against include/ags/ags.hpp (tests/cxx/render_cli.cpp)
    calls ags::render(std::span<const Gaussian3D>, ...) like the reference's
    callers: pair/splat counts equal the oracle's, the image is within
    tolerance, the DeviceScene overload agrees, and the reference's exception
    types come back (invalid_argument x2, PairBudgetError)."""
    import json
    import subprocess

    exe = os.path.join(os.path.dirname(os.path.dirname(__file__)), "paper_2604_18980_b200", "lib", "render_cli")
    out = tmp_path / "img.f32"
    args = [exe, "11", "3000", layout, "320", "240", "250", "1", mode, str(k), str(out)]
    if lutbin is not None:
        args.append(str(lutbin))
    res = json.loads(subprocess.run(args, check=True, capture_output=True, text=True).stdout.strip().splitlines()[-1])
    o = port.synth_scene(11, 3000, layout, cameras=2, width=320, height=240, focal=250.0)
    want = port.render(o, o.cameras[1], port.config(mode, k=k), port.lut([lutbin] * 20) if lutbin else None)
    assert res["pair_count"] == want["pair_count"] and res["splat_count"] == want["splat_count"]
    img = np.fromfile(out, np.float32).reshape(240, 320, 3)
    assert np.max(np.abs(img - want["image"])) <= IMG_MAX_ABS
    assert res["device_scene_same"] and res["errors_ok"] == 3 and res["stage_keys"] == 4
    assert res["cache_follows_edits"]  # render(span)'s device-scene cache never serves a stale scene
    # RecordOptions{max_t, contributions} (analysis.cpp:171-173): the oracle's stream, record for record
    cfg = port.config(mode, k=k)
    lut = port.lut([lutbin] * 20) if lutbin else None
    _, want_rec = port.render_contributions(o, o.cameras[1], cfg, lut)
    got_rec = np.fromfile(str(out) + ".contrib", capi.BLEND_DTYPE)
    assert res["contributions"] == len(want_rec) == len(got_rec) > 0
    assert np.array_equal(got_rec.view(np.uint32), want_rec.view(np.uint32))
    want_mt = port.render(o, o.cameras[1], cfg, lut, max_t=True)["max_t"]
    assert np.array_equal(np.fromfile(str(out) + ".maxt", np.float32).view(np.uint32), want_mt.view(np.uint32))


def test_cxx_stage_functions_reference_cases():
    """The reference's unit cases for the per-element stage functions
    (test_pair_gen.cpp:39-114, test_rasterizer.cpp:50-117,
    test_preprocess.cpp:35-140, test_scene_model.cpp:39-108) restated in C++
    against include/ags/ags.hpp (tests/cxx/stage_api_test.cpp): effective_radius,
    intersect_tiles in every mode, alpha_at, raster_tile (per tile and in
    reverse tile order, equal to the whole-frame render), project, eval_color,
    compute_th, covariance_3d and the math helpers; the device helpers equal the
    host glibc expressions bit for bit."""
    import subprocess

    exe = os.path.join(os.path.dirname(os.path.dirname(__file__)), "paper_2604_18980_b200", "lib", "stage_api_test")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "stage_api ok" in r.stdout


def test_per_element_helpers_match_oracle(ctx, port):
    """agsx_project / agsx_eval_color / agsx_compute_th / agsx_alpha_at /
    agsx_effective_radius (the device functions of the stages, exported for
    the C++ per-element API) against the oracle's preprocess_view splats and
    the host glibc logf / expf: bit-exact for every survivor."""
    oscene, dev = scene_pair(port, ctx, 11, 3000, "veil", 2, 320, 240, 250.0)
    ocam = oscene.cameras[1]
    cfg = port.config("adagscale", k=0.3)
    bins = [0.6] * 20
    splats = port.preprocess(oscene, ocam, cfg, port.lut(bins))
    assert len(splats) > 100
    sid = splats["source_id"]
    valid, proj = ctx.project(dev, to_gpu_cam(ocam), gpu_cfg("adagscale", 0.3))
    assert valid[sid].all()
    for col, (f, c) in enumerate((("mean2d", 0), ("mean2d", 1), ("cov2d", 0), ("cov2d", 1), ("cov2d", 2))):
        assert np.array_equal(proj[sid, col].view(np.uint32), splats[f][:, c].view(np.uint32)), (f, c)
    assert np.array_equal(proj[sid, 5].view(np.uint32), splats["depth"].view(np.uint32))
    # eval_color with the preprocess view direction (normalize(mean - position), float)
    mean = oscene.mean.reshape(-1, 3).astype(np.float32)
    d = (mean - np.asarray(ocam.position, np.float32)).astype(np.float32)
    nrm = np.sqrt((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]).astype(np.float32)
    dirs = (d * (np.float32(1.0) / nrm)[:, None]).astype(np.float32)
    rgb = ctx.eval_color(dev, dirs)
    assert np.array_equal(rgb[sid].view(np.uint32), splats["rgb"].view(np.uint32))
    th = ctx.compute_th(splats["cov2d"], splats["depth"], capi.make_lut(bins), 0.3, 1.0 / 255.0)
    assert np.array_equal(th.view(np.uint32), splats["th"].view(np.uint32))
    with pytest.raises(capi.AgsxError):  # AGSX_EINVAL: det <= 0 (std::invalid_argument)
        ctx.compute_th(np.array([[1.0, 2.0, 1.0]], np.float32), np.array([10.0], np.float32), None, 0.0, 0.01)
    # alpha_at / effective_radius vs the host glibc (ctypes libm) evaluation
    import ctypes

    libm = ctypes.CDLL("libm.so.6")
    libm.expf.restype = libm.logf.restype = ctypes.c_float
    libm.expf.argtypes = libm.logf.argtypes = [ctypes.c_float]
    rng = np.random.default_rng(3)
    sel = splats[:256]
    px = (sel["mean2d"] + rng.uniform(-6, 6, (len(sel), 2))).astype(np.float32)
    alpha = ctx.alpha_at(sel, px, 0.99)
    for i in range(len(sel)):
        dx, dy = np.float32(px[i, 0] - sel["mean2d"][i, 0]), np.float32(px[i, 1] - sel["mean2d"][i, 1])
        xx, xy, yy = (np.float32(v) for v in sel["inv_cov"][i])
        q = np.float32(np.float32(np.float32(xx * dx) * dx) + np.float32(np.float32(np.float32(2 * xy) * dx) * dy))
        q = np.float32(q + np.float32(np.float32(yy * dy) * dy))
        pw = np.float32(np.float32(-0.5) * q)
        a = 0.0 if pw > 0 else min(np.float32(sel["opacity"][i] * np.float32(libm.expf(float(pw)))), np.float32(0.99))
        assert np.float32(a).view(np.uint32) == alpha[i].view(np.uint32), i
    er = ctx.effective_radius(sel["opacity"], sel["th"], sel["cov2d"])
    for i in range(len(sel)):
        m = np.float32(np.sqrt(np.float32(2.0 * libm.logf(float(np.float32(sel["opacity"][i] / sel["th"][i]))))))
        assert m.view(np.uint32) == er[i, 0].view(np.uint32), i


def test_async_chain_overflow_mid_chain_fails_at_wait(port):
    """Frames enqueued back to back (render_async, no wait in between) share
    one counter block; a frame in the middle of the chain that overflows the
    pair arena skips emission and cannot be re-run once later frames ran.
    The wait must report it (AGSX_EFRAME_LOST) instead of returning the last
    frame's counts; an overflowing LAST frame is re-run as before."""
    ctx = capi.Context(0)  # fresh context: arena at its first guess max(12 N, 2^20)
    try:
        o = port.synth_scene(2, 2000, "slab", cameras=2, width=640, height=480, focal=500.0)
        o.scale[:] *= 40.0  # P >> 2^20 at 640x480
        dev = ctx.upload(o.mean, o.scale, o.rotation, o.opacity, o.sh)
        big = to_gpu_cam(o.cameras[0])
        small = to_gpu_cam(o.cameras[0])
        small.width, small.height = 16, 16  # one tile: at most N pairs
        ctx.render_async(dev, big, gpu_cfg("aabb"))   # overflows (emission skipped)
        ctx.render_async(dev, small, gpu_cfg("aabb"))  # fits
        with pytest.raises(capi.AgsxError) as e:
            ctx.wait()
        assert e.value.code == capi.EFRAME_LOST, e.value
        with pytest.raises(capi.AgsxError) as e:  # nothing in flight any more
            ctx.wait()
        assert e.value.code == capi.EINVAL
        # the chain words were cleared: a fitting chain waits cleanly
        ctx.render_async(dev, small, gpu_cfg("aabb"))
        ctx.render_async(dev, small, gpu_cfg("aabb"))
        st = ctx.wait()
        assert st["pair_count"] <= 2000
        # an overflowing last frame is grown and re-run (bit-exact vs the oracle)
        ctx.render_async(dev, small, gpu_cfg("aabb"))
        ctx.render_async(dev, big, gpu_cfg("aabb"))
        st = ctx.wait()
        want = port.render(o, o.cameras[0], port.config("aabb"))
        assert st["pair_count"] == want["pair_count"] > (1 << 20)
    finally:
        ctx.close()


def test_host_frame_in_flight_refused_at_the_c_abi(port):
    """while a render_async_host frame is in flight its host image
    and counters belong to it; every other frame entry on the context (sync
    render, async, stage hooks) is refused with EINVAL until agsx_render_wait."""
    ctx = capi.Context(0)
    try:
        o = port.synth_scene(4, 500, "veil", cameras=2, width=200, height=136, focal=150.0)
        dev = ctx.upload(o.mean, o.scale, o.rotation, o.opacity, o.sh)
        cam = to_gpu_cam(o.cameras[0])
        img = np.zeros((136, 200, 3), np.float32)
        ctx.render_async_host(dev, cam, gpu_cfg("ellipse", exact=True), None, img)
        for call in (lambda: ctx.render(dev, cam, gpu_cfg("ellipse")),
                     lambda: ctx.render_async(dev, cam, gpu_cfg("ellipse")),
                     lambda: ctx.render_async_host(dev, cam, gpu_cfg("ellipse"), None, img),
                     lambda: ctx.preprocess_view(dev, cam, gpu_cfg("ellipse"))):
            with pytest.raises(capi.AgsxError) as e:
                call()
            assert e.value.code == capi.EINVAL
        st = ctx.wait()
        want = port.render(o, o.cameras[0], port.config("ellipse"))
        assert st["pair_count"] == want["pair_count"]
        assert np.array_equal(img.view(np.uint32), want["image"].view(np.uint32))
        ctx.render(dev, cam, gpu_cfg("ellipse"))  # accepted again
    finally:
        ctx.close()


@pytest.mark.parametrize("mode", ["ellipse", "adagscale"])
def test_p_it_matches_reference_semantics(ctx, port, mode):
    """frame_stats()['p_it'] (the raster work measure behind the
    bench's raster bytes) against the oracle's P_it -- the
    pairs raster_tile visits before all pixels of its tile are saturated
    (rasterizer.cpp:55-56), summed over tiles. Exact rasteriser: equal. Default
    rasteriser (hardware ex2 blend, so T may cross the floor one pair
    earlier or later on a handful of pixels): within 0.1 %."""
    oscene, dev = scene_pair(port, ctx, 11, 20000, "veil", 2, 640, 480, 500.0)
    ocam = oscene.cameras[0]
    bins = LUT_BINS if mode == "adagscale" else None
    k = K1080 * (500.0 / 1500.0) ** 2 if mode == "adagscale" else 0.0
    ocfg = port.config(mode, k=k)
    splats = port.preprocess(oscene, ocam, ocfg, port.lut(bins) if bins else None)
    keys, idx, counts = port.generate_pairs(splats, ocam.width, ocam.height, ocfg.mode, ocfg)
    tiles = ((ocam.width + 15) // 16) * ((ocam.height + 15) // 16)
    skeys, sidx, ranges = port.sort_pairs(keys, idx, tiles)
    _, want = port.raster_pit(splats, sidx, ranges, ocam.width, ocam.height, ocfg)
    assert 0 < want <= len(skeys)
    glut = capi.make_lut(bins) if bins else None
    ctx.render(dev, to_gpu_cam(ocam), gpu_cfg(mode, k, exact=True), glut)
    assert ctx.frame_stats()["p_it"] == want
    ctx.render(dev, to_gpu_cam(ocam), gpu_cfg(mode, k), glut)
    got = ctx.frame_stats()["p_it"]
    assert abs(got - want) <= max(2, want // 1000), (got, want)


def test_tile_sizes_above_64(ctx, port):
    """the reference's raster_tile takes any tile_size >= 1 and
    falls back to heap buffers above 64x64 pixels (rasterizer.cpp:35-47).
    Here such a tile is split into 64x64 blocks that walk the same pair
    range; keys, ranges and the image stay bit-exact."""
    oscene, dev = scene_pair(port, ctx, 53, 600, "slab", 2, 321, 257, 200.0)
    for ts in (64, 80, 128, 200):
        check_frame(ctx, port, oscene, dev, 0, "ellipse", background=(0.2, 0.2, 0.2), tile_size=ts)
        check_frame(ctx, port, oscene, dev, 0, "aabb", tile_size=ts)


def test_kept_frames_past_the_pinned_cap(tmp_path):
    """a caller that keeps its frames. Page-locked images
    are capped (AGS_PINNED_POOL_MB); past the cap render() returns ordinary
    arrays, filled from the renderer's staging block (f32 and PPM bytes). Every
    kept frame stays intact and equal to a fresh render."""
    import subprocess
    import sys

    code = (
        "import sys, numpy as np; sys.path.insert(0, sys.argv[1])\n"
        "import paper_2604_18980_b200 as P\n"
        "s = P.synth_scene(3, 3000, 'veil', cameras=4, width=320, height=240, focal=250.0)\n"
        "kept = [P.render(s, v % 4, 'ellipse')['image'] for v in range(8)]\n"
        "pinned = sum(1 for a in kept if not a.flags['OWNDATA'] and a.base is not None)\n"
        "for v in range(8):\n"
        "    again = P.render(s, v % 4, 'ellipse')['image']\n"
        "    assert np.array_equal(kept[v].view(np.uint32), again.view(np.uint32)), v\n"
        "kept8 = [P.render(s, v % 4, 'ellipse', image_u8=True)['image'] for v in range(8)]\n"
        "for v in range(8):\n"
        "    again = P.render(s, v % 4, 'ellipse', image_u8=True)['image']\n"
        "    assert np.array_equal(kept8[v], again), v\n"
        "print('ok', pinned)\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, AGS_PINNED_POOL_MB="2")  # two 0.9 MB frames fit
    out = subprocess.run([sys.executable, "-c", code, root], env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip().startswith("ok")


@pytest.mark.parametrize("mode", ["adagscale", "ellipse", "obb"])
def test_sort_paths_agree(tmp_path, mode):
    """The two sort paths (DESIGN.md §4.2 depth-then-tile, §4.2b tile-bucketed)
    and the two scene storage orders (§3: 3D Morton, the caller's) give
    identical keys, Gaussian ids and images: this process renders with the
    defaults, subprocesses with AGSX_SORT / AGSX_SCENE_ORDER (process-wide
    switches)."""
    import subprocess
    import sys

    import paper_2604_18980_b200 as P

    spec = dict(seed=9, count=20000, layout="veil", cameras=3, width=640, height=480, focal=500.0)
    kw = dict(mode=mode, k=0.3 if mode == "adagscale" else 0.0, lut_bins=[0.6] * 20 if mode == "adagscale" else [])
    s = P.synth_scene(**spec)
    r = P.Renderer(0)
    got = []
    out = r.render(s, 2, **kw)  # this process: the default (depth-then-tile) path
    keys, gids = r.dump_sorted_pairs()
    st = r.frame_stats()
    got.append((st["bucketed_sort"], keys, gids, r.dump_ranges(st["tiles"]), out["image"]))
    code = (
        "import sys, numpy as np; sys.path.insert(0, sys.argv[1])\n"
        "import paper_2604_18980_b200 as P\n"
        f"s = P.synth_scene(**{spec!r})\n"
        "r = P.Renderer(0)\n"
        f"out = [r.render(s, 2, **{kw!r}) for _ in range(2)][-1]\n"
        "keys, gids = r.dump_sorted_pairs()\n"
        "np.savez(sys.argv[2], b=r.frame_stats()['bucketed_sort'], keys=keys, gids=gids, image=out['image'])\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if os.environ.get("AGSX_SORT") == "bucket":  # this process already runs the bucketed path
        return
    for forced, flag, order in (("depth", 0, "morton"), ("bucket", 1, "morton"), ("depth", 0, "input")):
        # AGSX_SCENE_ORDER=input keeps the caller's storage order
        dst = str(tmp_path / f"{forced}_{order}.npz")
        env = dict(os.environ, AGSX_SORT=forced, AGSX_SCENE_ORDER=order)
        res = subprocess.run([sys.executable, "-c", code, root, dst], env=env, capture_output=True, text=True,
                             timeout=300)
        assert res.returncode == 0, res.stderr[-2000:]
        f = np.load(dst)
        assert int(f["b"]) == flag
        assert np.array_equal(f["keys"], got[0][1]) and np.array_equal(f["gids"], got[0][2])
        assert np.array_equal(f["image"].view(np.uint32), got[0][4].view(np.uint32))


def test_storage_order_edge_scenes(ctx, port):
    """The Morton storage order on degenerate scenes: a single
    Gaussian, many Gaussians at one position (equal Morton codes, equal depths:
    every tie must fall back to Gaussian-id order), and non-finite means
    (culled, and ignored by the bounding box of the codes). Keys, ranges,
    counts and the exact image equal the oracle's."""
    o = port.synth_scene(7, 600, "slab", cameras=2, width=160, height=120, focal=120.0)
    cases = {}
    one = port.synth_scene(7, 1, "slab", cameras=2, width=160, height=120, focal=120.0)
    cases["single"] = one
    same = port.synth_scene(7, 600, "slab", cameras=2, width=160, height=120, focal=120.0)
    same.mean[:] = same.mean[0]  # one position: identical depth keys, gid order decides
    cases["coincident"] = same
    nanm = port.synth_scene(7, 600, "slab", cameras=2, width=160, height=120, focal=120.0)
    nanm.mean[::7, 0] = np.nan
    nanm.mean[3::11, 2] = np.inf
    cases["non_finite"] = nanm
    for name, sc in cases.items():
        dev = ctx.upload(sc.mean, sc.scale, sc.rotation, sc.opacity, sc.sh)
        for mode in ("ellipse", "aabb"):
            out, _ = check_frame(ctx, port, sc, dev, 0, mode, exact=True)
            assert out["pair_count"] >= 0, name
    del o

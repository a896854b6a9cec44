"""CPU tests of the oracle: the C restatement is pinned against the committed
reference fixtures (always) and against the unmodified reference build
(oracle/_ref, when present) bit for bit; plus the reference's own known-answer
tests restated (file:line cited)."""
import hashlib
import math
import os

import numpy as np
import pytest

from oracle.ffi import SPLAT_DTYPE, PairBudgetError

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "reference_fixtures.npz")
CASES = [
    ("slab_ellipse", 1, 1500, "slab", 4, 640, 480, 500.0, 0, "ellipse", 0.0, None),
    ("slab_aabb", 1, 1500, "slab", 4, 640, 480, 500.0, 1, "aabb", 0.0, None),
    ("aniso_obb", 8, 1200, "aniso", 3, 640, 480, 500.0, 0, "obb", 0.0, None),
    ("veil_ada", 1, 4000, "veil", 4, 480, 320, 375.0, 0, "adagscale", 0.4, [0.6] * 20),
    ("two_slab_ada", 3, 3000, "two_slab", 6, 320, 240, 250.0, 2, "adagscale", 0.25, [0.8] * 20),
    ("ramp_ellipse", 2, 2000, "ramp", 2, 640, 480, 500.0, 0, "ellipse", 0.0, None),
    ("odd_101x77", 53, 400, "slab", 2, 101, 77, 90.0, 0, "ellipse", 0.0, None),
]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_port_matches_reference_fixtures(port, golden, case):
    name, seed, count, layout, cams, w, h, focal, view, mode, k, bins = case
    scene = port.synth_scene(seed, count, layout, cameras=cams, width=w, height=h, focal=focal)
    g = lambda f: golden[f"{name}__{f}"]  # noqa: E731
    assert sha(np.concatenate([scene.mean.ravel(), scene.scale.ravel(), scene.rotation.ravel(), scene.opacity,
                               scene.sh.ravel()])) == str(g("scene_sha"))
    cam = scene.cameras[view]
    cfg = port.config(mode, k=k, background=(0.2, 0.2, 0.2) if name == "odd_101x77" else (0, 0, 0))
    splats = port.preprocess(scene, cam, cfg, port.lut(bins) if bins else None)
    assert sha(splats) == str(g("splats_sha"))
    keys, idx, counts = port.generate_pairs(splats, w, h, cfg.mode, cfg)
    assert np.array_equal(counts, g("tile_counts"))
    assert len(keys) == int(g("pair_count"))
    assert sha(keys) == str(g("keys_sha"))
    tiles = ((w + 15) // 16) * ((h + 15) // 16)
    sk, si, rg = port.sort_pairs(keys, idx, tiles)
    assert sha(sk) == str(g("sorted_keys_sha")) and sha(si) == str(g("sorted_idx_sha"))
    assert sha(rg) == str(g("ranges_sha"))
    img = port.raster(splats, sk, si, rg, w, h, cfg)
    assert sha(img) == str(g("image_sha"))


def test_port_sort_matches_reference_fixture(port, golden):
    sk, si, sr = port.sort_pairs(golden["sort__keys_in"], np.arange(20000, dtype=np.uint32), 300)
    assert np.array_equal(si, golden["sort__idx_out"])
    assert np.array_equal(sr, golden["sort__ranges"])


@pytest.mark.parametrize("layout", ["slab", "two_slab", "veil", "ramp", "aniso"])
def test_port_matches_reference_build(port, ref, layout):
    """Full pipeline, every mode, port vs the unmodified reference: bit-exact."""
    a = port.synth_scene(7, 2500, layout, cameras=3, width=320, height=240, focal=250.0)
    b = ref.synth_scene(7, 2500, layout, cameras=3, width=320, height=240, focal=250.0)
    for f in ("mean", "scale", "rotation", "opacity", "sh"):
        assert np.array_equal(getattr(a, f).view(np.uint32), getattr(b, f).view(np.uint32))
    for mode in ("aabb", "obb", "ellipse", "adagscale"):
        for fixed in (0, 1) if mode == "aabb" else (0,):
            ca = port.config(mode, k=0.5, fixed_radius_aabb=fixed)
            cb = ref.config(mode, k=0.5, fixed_radius_aabb=fixed)
            lut = port.lut([0.6] * 20)
            ra = port.render(a, a.cameras[1], ca, lut, max_t=True)
            rb = ref.render(b, b.cameras[1], cb, lut, max_t=True)
            assert ra["pair_count"] == rb["pair_count"] and ra["splat_count"] == rb["splat_count"]
            assert np.array_equal(ra["image"].view(np.uint32), rb["image"].view(np.uint32))
            assert np.array_equal(ra["max_t"].view(np.uint32), rb["max_t"].view(np.uint32))


@pytest.mark.parametrize("layout,mode,ts", [("veil", "adagscale", 16), ("slab", "ellipse", 16), ("aniso", "obb", 8)])
def test_port_contributions_match_reference_build(port, ref, layout, mode, ts):
    """RecordOptions::contributions (rasterizer.cpp:21-100,135-161): the port's
    blend-event stream equals the reference's record for record, in order."""
    a = port.synth_scene(4, 1500, layout, cameras=2, width=160, height=120, focal=125.0)
    b = ref.synth_scene(4, 1500, layout, cameras=2, width=160, height=120, focal=125.0)
    lut = port.lut([0.6] * 20)
    ia, ra = port.render_contributions(a, a.cameras[1], port.config(mode, k=0.4, tile_size=ts), lut)
    ib, rb = ref.render_contributions(b, b.cameras[1], ref.config(mode, k=0.4, tile_size=ts), lut)
    assert len(ra) > 1000 and len(ra) == len(rb)
    assert np.array_equal(ra.view(np.uint32), rb.view(np.uint32))
    assert np.array_equal(ia.view(np.uint32), ib.view(np.uint32))
    # test_rasterizer.cpp:167-180: per pixel the blend weights never exceed unit energy
    per_pixel = np.zeros(160 * 120)
    np.add.at(per_pixel, ra["pixel"], ra["weight"].astype(np.float64))
    assert per_pixel.max() <= 1.0 + 1e-5


def test_port_libm_is_host_glibc(port, ref):
    x = np.linspace(1.0, 255.0, 100_001, dtype=np.float32)
    assert np.array_equal(port.logf(x), ref.logf(x))
    x = np.linspace(-20.0, 0.0, 100_001, dtype=np.float32)
    assert np.array_equal(port.expf(x), ref.expf(x))


# ---- known-answer tests of the reference suites, on the oracle ---------------
def one_splat(mean, cov, opacity, th, depth=5.0):
    s = np.zeros(1, SPLAT_DTYPE)
    c = np.array(cov, np.float32)
    det = c[0] * c[2] - c[1] * c[1]
    inv = np.float32(1.0) / det
    s["mean2d"], s["cov2d"] = mean, c
    s["inv_cov"] = [c[2] * inv, -c[1] * inv, c[0] * inv]
    s["depth"], s["rgb"], s["opacity"], s["th"] = depth, (1, 1, 1), opacity, th
    return s


def test_known_answers_pair_gen(port):
    """test_pair_gen.cpp:55-66, 205-237, 257-266."""
    cfg = port.config("ellipse")
    s = one_splat((24, 24), (4, 0, 4), 0.99, 1 / 255)
    for m in ("aabb", "obb", "ellipse", "adagscale"):
        keys, _, counts = port.generate_pairs(s, 64, 64, m, port.config(m))
        assert list(counts) == [1] and int(keys[0]) >> 32 == 5
    s = one_splat((328, 120), (81, 0, 2.25), 0.99, 1 / 255)
    keys, _, counts = port.generate_pairs(s, 640, 480, "ellipse", cfg)
    assert [int(k) >> 32 for k in keys] == [298, 299, 300, 301, 302]
    with pytest.raises(PairBudgetError):
        port.generate_pairs(s, 640, 480, "ellipse", port.config("ellipse", pair_budget=4))
    s = one_splat((-500, -500), (4, 0, 4), 0.9, 1 / 255)
    assert list(port.generate_pairs(s, 64, 64, "ellipse", cfg)[2]) == [0]


def test_known_answers_render(port):
    """test_rasterizer.cpp:60-114."""
    cfg = port.config("ellipse", background=(0.25, 0.5, 0.75))
    s = one_splat((8, 8), (1e8, 0, 1e8), 0.001, 1 / 255, depth=1.0)
    keys, idx, _ = port.generate_pairs(s, 16, 16, "ellipse", cfg)
    sk, si, rg = port.sort_pairs(keys, idx, 1)
    img = port.raster(s, sk, si, rg, 16, 16, cfg)
    assert tuple(img[8, 8]) == (np.float32(0.25), np.float32(0.5), np.float32(0.75))
    s = one_splat((8, 8), (1e8, 0, 1e8), 0.5, 1 / 255, depth=1.0)
    cfg = port.config("ellipse")
    keys, idx, _ = port.generate_pairs(s, 16, 16, "ellipse", cfg)
    sk, si, rg = port.sort_pairs(keys, idx, 1)
    img = port.raster(s, sk, si, rg, 16, 16, cfg)
    assert abs(img[8, 8, 0] - 0.5) < 1e-4


def test_psnr(port):
    """test_smoke.py:71-75 / analysis.cpp:14-25."""
    a = np.zeros((8, 8, 3), np.float32) + 0.5
    assert math.isinf(port.psnr(a, a))
    assert abs(port.psnr(a, a + np.float32(0.1)) - 20.0) < 1e-4


def test_calibration_golden_is_reference(ref):
    """The calibration golden fixture reproduces from the reference build."""
    import json
    import os

    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "calibration_veil3000.json")))
    s = ref.synth_scene(**g["spec"])
    out = ref.calibrate(s, g["target_drop"], g["calib_views"])
    assert out["k"] == g["k"] and out["lut_bins"] == g["lut_bins"] and out["iterations"] == g["iterations"]

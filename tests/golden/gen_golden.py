#!/usr/bin/env python3
"""Generate tests/golden/*.npz from the REFERENCE build (oracle/_ref/libags_ref.so).

The reference (/root/reference/proj) is compiled unmodified by oracle/Makefile
(`make -C oracle ref`); this script drives it through oracle/ref_shim.cpp and
stores small fixtures so the C restatement (oracle/ags_oracle.c) and the GPU
path can be pinned on machines without /root/reference.

    python tests/golden/gen_golden.py
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.ffi import Oracle  # noqa: E402

# Each case: (name, seed, count, layout, cameras, width, height, focal, view, mode, k, lut_bins)
CASES = [
    ("slab_ellipse", 1, 1500, "slab", 4, 640, 480, 500.0, 0, "ellipse", 0.0, None),
    ("slab_aabb", 1, 1500, "slab", 4, 640, 480, 500.0, 1, "aabb", 0.0, None),
    ("aniso_obb", 8, 1200, "aniso", 3, 640, 480, 500.0, 0, "obb", 0.0, None),
    ("veil_ada", 1, 4000, "veil", 4, 480, 320, 375.0, 0, "adagscale", 0.4, [0.6] * 20),
    ("two_slab_ada", 3, 3000, "two_slab", 6, 320, 240, 250.0, 2, "adagscale", 0.25, [0.8] * 20),
    ("ramp_ellipse", 2, 2000, "ramp", 2, 640, 480, 500.0, 0, "ellipse", 0.0, None),
    ("odd_101x77", 53, 400, "slab", 2, 101, 77, 90.0, 0, "ellipse", 0.0, None),
]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    ref = Oracle("reference")
    out = {}
    for (name, seed, count, layout, cams, w, h, focal, view, mode, k, bins) in CASES:
        scene = ref.synth_scene(seed, count, layout, cameras=cams, width=w, height=h, focal=focal)
        cam = scene.cameras[view]
        cfg = ref.config(mode, k=k, background=(0.2, 0.2, 0.2) if name == "odd_101x77" else (0, 0, 0))
        lut = ref.lut(bins) if bins else None
        splats = ref.preprocess(scene, cam, cfg, lut)
        keys, idx, counts = ref.generate_pairs(splats, w, h, cfg.mode, cfg)
        tiles = ((w + 15) // 16) * ((h + 15) // 16)
        skeys, sidx, ranges = ref.sort_pairs(keys, idx, tiles)
        img = ref.raster(splats, skeys, sidx, ranges, w, h, cfg)
        rend = ref.render(scene, cam, cfg, lut)
        assert np.array_equal(rend["image"], img)
        out[f"{name}__scene_sha"] = np.array(sha(np.concatenate(
            [scene.mean.ravel(), scene.scale.ravel(), scene.rotation.ravel(), scene.opacity, scene.sh.ravel()])))
        out[f"{name}__splats_sha"] = np.array(sha(splats))
        out[f"{name}__source_id"] = splats["source_id"].astype(np.uint32)
        out[f"{name}__tile_counts"] = counts.astype(np.uint32)
        out[f"{name}__pair_count"] = np.array(len(keys), np.int64)
        out[f"{name}__keys_sha"] = np.array(sha(keys))
        if len(skeys) <= 40000:
            out[f"{name}__sorted_keys"] = skeys
            out[f"{name}__sorted_idx"] = sidx
        out[f"{name}__sorted_keys_sha"] = np.array(sha(skeys))
        out[f"{name}__sorted_idx_sha"] = np.array(sha(sidx))
        out[f"{name}__ranges_sha"] = np.array(sha(ranges))
        out[f"{name}__image_sha"] = np.array(sha(img))
        out[f"{name}__image_sum"] = np.array(float(img.astype(np.float64).sum()))
        print(f"{name}: splats={len(splats)} pairs={len(keys)}")
    # sort oracle inputs (test_pair_sort.cpp:31-52 style, fixed numpy seed)
    rng = np.random.default_rng(17)
    depth = (0.25 * (1 + rng.integers(0, 64, 20000))).astype(np.float32)
    keys = (rng.integers(0, 300, 20000).astype(np.uint64) << np.uint64(32)) | depth.view(np.uint32).astype(np.uint64)
    idx = np.arange(20000, dtype=np.uint32)
    sk, si, sr = ref.sort_pairs(keys, idx, 300)
    out["sort__keys_in"] = keys
    out["sort__idx_out"] = si
    out["sort__ranges"] = sr
    np.savez_compressed(os.path.join(HERE, "reference_fixtures.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_fixtures.npz"))


if __name__ == "__main__":
    main()

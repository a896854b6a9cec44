"""Experiment: the same config-3 scene with its Gaussians in 3D Morton order
(SPATIAL=1) vs generation order, one render each, for an ncu launch list.
    AGSX_SORT=bucket SPATIAL=1 python scripts/probe_spatial.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_18980_b200 as P  # noqa: E402

bins = [1.0] * 20
bins[7], bins[8] = 0.003038157941773534, 0.007012989837676287
K = float(np.float32(0.3985099792480469 * (3600.0 / 1500.0) ** 2))
s = P.synth_scene(1, 3_000_000, "veil", cameras=16, width=4608, height=3456, focal=3600.0)
if os.environ.get("SPATIAL") == "1":
    a = s.arrays()
    m = a["mean"].reshape(-1, 3).astype(np.float64)
    q = ((m - m.min(0)) / (np.ptp(m, 0) + 1e-9) * 1023).astype(np.uint64)

    def spread(v):
        v = v & 0x3FF
        v = (v | (v << 16)) & 0x030000FF
        v = (v | (v << 8)) & 0x0300F00F
        v = (v | (v << 4)) & 0x030C30C3
        v = (v | (v << 2)) & 0x09249249
        return v

    code = spread(q[:, 0]) | (spread(q[:, 1]) << 1) | (spread(q[:, 2]) << 2)
    order = np.argsort(code, kind="stable")
    s = P.Scene.from_arrays(a["mean"].reshape(-1, 3)[order].ravel(), a["scale"].reshape(-1, 3)[order].ravel(),
                            a["rotation"].reshape(-1, 4)[order].ravel(), a["opacity"][order],
                            a["sh"].reshape(len(order), -1)[order].ravel(), [s.camera(v) for v in range(16)])
r = P.Renderer(0)
for _ in range(4):
    out = r.render(s, 0, "adagscale", K, bins, image=False)
print("pairs", out["pair_count"], "stage_ms", r.stage_history(3).mean(axis=0))

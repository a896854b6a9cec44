"""Small frames over every device path, for compute-sanitizer (memcheck,
racecheck, synccheck, initcheck): the default rasteriser, the exact one, max_t,
banded f32 and PPM host egress (stream wait-value copies behind the raster),
two contexts with frames in flight, an async chain, other tile sizes, the
stage hooks and the tile-bucketed sort (AGSX_SORT=bucket, set by the caller).

    compute-sanitizer --tool memcheck python scripts/sanitize_workload.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_18980_b200 as P  # noqa: E402

bins = [1.0] * 20
bins[7], bins[8] = 0.003038157941773534, 0.007012989837676287
s = P.synth_scene(1, 3000, "veil", cameras=4, width=320, height=240, focal=250.0)
r0, r1 = P.Renderer(0), P.Renderer(0)
out = {}
out["default"] = r0.render(s, 0, "adagscale", 0.3, bins)["pair_count"]
out["exact"] = r0.render(s, 0, "adagscale", 0.3, bins, exact=True)["pair_count"]
out["max_t"] = r0.render(s, 1, "ellipse", max_t=True)["pair_count"]
for mode in ("aabb", "obb", "ellipse", "aabb_fixed3"):
    out[mode] = r0.render(s, 2, mode)["pair_count"]
for ts in (8, 32, 80):
    out[f"ts{ts}"] = r0.render(s, 0, "ellipse", tile_size=ts)["pair_count"]
out["u8"] = int(np.asarray(r0.render(s, 0, "ellipse", image_u8=True)["image"]).sum() > 0)
# banded host egress on two contexts, one frame in flight each
r0.render_async_host(s, 0, mode="ellipse")
r1.render_async_host(s, 1, mode="adagscale", k=0.3, lut_bins=bins, image_u8=True)
out["host0"] = r0.wait()["pair_count"]
out["host1"] = r1.wait()["pair_count"]
# async chain of device-resident frames
for v in range(4):
    r0.render_async(s, v, "ellipse")
out["chain"] = r0.wait()["pair_count"]
out["report"] = P.Renderer(0).pair_report(s, [("ellipse", 0.0), ("adagscale", 0.3)], views=[0, 1],
                                          lut_bins=bins)[1]["pair_count"]
print("sanitize workload ok", out)

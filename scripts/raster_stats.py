"""Raster work counters (AGSX_RASTER_STATS=1) for config 3, AdaGScale on and off."""
import os, sys
sys.path.insert(0, ".")
os.environ["AGSX_RASTER_STATS"] = "1"
import numpy as np
import paper_2604_18980_b200 as P
K = float(np.float32(0.3985099792480469 * (3600 / 1500.0) ** 2))
B = [1.0] * 20; B[7] = 0.003038157941773534; B[8] = 0.007012989837676287
s = P.synth_scene(1, 3_000_000, "veil", cameras=16, width=4608, height=3456, focal=3600.0)
r = P.Renderer(0)
for mode, k, b in (("adagscale", K, B), ("ellipse", 0.0, [])):
    r.render_async(s, 0, mode, k, b); r.wait()
    st = r.frame_stats()
    it, ev, fa, ex = st["raster_iters"], st["raster_evals"], st["raster_fast"], st["raster_exact"]
    print(mode, "pairs", st["pair_count"], "p_it", st["p_it"], "warp-iters", it, "per p_it %.2f" % (it / st["p_it"]),
          "live-evals", ev, "(%.1f of 128 per iter)" % (ev / it), "fast blends", fa, "(%.1f%% of live)" % (100 * fa / ev),
          "exact", ex, "iters live<=32", st["raster_iters_live_le32"], "<=64", st["raster_iters_live_le64"], "empty", st["raster_iters_empty"], "no live pixel", st["raster_iters_no_live_pixel"], flush=True)

"""One config-3 frame (3M Gaussians, 4608x3456, AdaGScale) for compute-sanitizer."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_18980_b200 as P  # noqa: E402
bins = [1.0] * 20
bins[7], bins[8] = 0.003038157941773534, 0.007012989837676287
n = int(os.environ.get("N", "3000000"))
s = P.synth_scene(1, n, "veil", cameras=16, width=4608, height=3456, focal=3600.0)
r = P.Renderer(0)
out = r.render(s, 0, "adagscale", float(np.float32(0.3985099792480469 * (3600.0 / 1500.0) ** 2)), bins, image=False)
print("pairs", out["pair_count"], "splats", out["splat_count"])

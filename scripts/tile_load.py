"""Per-tile pair-count distribution at config 3 (AdaGScale on / off)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2604_18980_b200 as P
K = float(np.float32(0.3985099792480469 * (3600 / 1500.0) ** 2))
B = [1.0] * 20; B[7] = 0.003038157941773534; B[8] = 0.007012989837676287
s = P.synth_scene(1, 3_000_000, "veil", cameras=16, width=4608, height=3456, focal=3600.0)
r = P.Renderer(0)
for mode, k, b in (("adagscale", K, B), ("ellipse", 0.0, [])):
    r.render_async(s, 0, mode, k, b); r.wait()
    rg = r.dump_ranges(288 * 216)
    n = (rg[:, 1].astype(np.int64) - rg[:, 0]).clip(0)
    q = np.percentile(n, [50, 90, 99, 99.9, 100])
    top = np.sort(n)[::-1][:10]
    print(mode, "tiles", len(n), "empty", int((n == 0).sum()), "pctl50/90/99/99.9/max", q.tolist(), "top10", top.tolist(),
          "sum", int(n.sum()), "top1pct_share", round(float(np.sort(n)[::-1][: len(n) // 100].sum() / n.sum()), 3))
    rows = n.reshape(216, 288).sum(axis=1)
    print(mode, "pairs per tile row (first, middle, last 10 rows):", rows[:10].tolist(), rows[100:110].tolist(),
          rows[-10:].tolist())

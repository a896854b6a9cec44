import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2604_18980_b200 as P
K = float(np.float32(0.3985099792480469 * (3600 / 1500.0) ** 2))
B = [1.0] * 20; B[7] = 0.003038157941773534; B[8] = 0.007012989837676287
s = P.synth_scene(1, 3_000_000, "veil", cameras=16, width=4608, height=3456, focal=3600.0)
r = P.default_renderer()
ts = []
for _ in range(20):
    t = time.perf_counter()
    out = r.render(s, 0, "adagscale", K, B)
    ts.append((time.perf_counter() - t) * 1e3)
print(" ".join(f"{x:.1f}" for x in ts))

import sys, os
sys.path.insert(0, ".")
import numpy as np
import paper_2604_18980_b200 as P
K = float(np.float32(0.3985099792480469))
B = [1.0] * 20; B[7] = 0.003038157941773534; B[8] = 0.007012989837676287
s = P.synth_scene(1, 100000, "veil", cameras=16, width=1920, height=1080, focal=1500.0)
r = P.Renderer(0)
ex = r.render(s, 0, "adagscale", K, B, exact=True)["image"]
fa = r.render(s, 0, "adagscale", K, B, exact=False)["image"]
d = np.abs(fa - ex)
i = np.unravel_index(np.argmax(d), d.shape)
print("max", d.max(), "at", i, "fast", fa[i[0], i[1]], "exact", ex[i[0], i[1]], "n>1e-4", (d > 1e-4).sum(), "n>1e-3", (d > 1e-3).sum())
ys, xs, _ = np.nonzero(d > 1e-3)
print("tiles", sorted(set(zip((ys // 16).tolist(), (xs // 16).tolist())))[:20])

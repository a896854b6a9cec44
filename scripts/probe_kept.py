"""render() at config 3 when the caller keeps every frame: the first frames take pinned
blocks, frames past AGS_PINNED_POOL_MB (2 GB: 10 frames) get pageable arrays."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2604_18980_b200 as P
K = float(np.float32(0.3985099792480469 * (3600 / 1500.0) ** 2))
B = [1.0] * 20; B[7] = 0.003038157941773534; B[8] = 0.007012989837676287
s = P.synth_scene(1, 3_000_000, "veil", cameras=16, width=4608, height=3456, focal=3600.0)
r = P.default_renderer()
for _ in range(3):
    r.render(s, 0, "adagscale", K, B)
keep, ts = [], []
for i in range(24):
    t = time.perf_counter()
    keep.append(r.render(s, 0, "adagscale", K, B)["image"])
    ts.append((time.perf_counter() - t) * 1e3)
print("ms per frame, frames kept:", " ".join(f"{x:.1f}" for x in ts))
print(f"first 10 (pinned): {np.mean(ts[:10]):.2f} ms; past the cap: {np.mean(ts[12:]):.2f} ms")
assert all(np.array_equal(keep[0], k) for k in keep[1:])
print("all kept frames identical")

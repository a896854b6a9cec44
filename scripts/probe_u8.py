import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2604_18980_b200 as P
K = float(np.float32(0.3985099792480469 * (3600 / 1500.0) ** 2))
B = [1.0] * 20; B[7] = 0.003038157941773534; B[8] = 0.007012989837676287
s = P.synth_scene(1, 3_000_000, "veil", cameras=16, width=4608, height=3456, focal=3600.0)
for u8 in (False, True):
    for _ in range(3):
        out = P.render(s, 0, "adagscale", K, B, image_u8=u8)
    t0 = time.perf_counter()
    for _ in range(10):
        out = P.render(s, 0, "adagscale", K, B, image_u8=u8)
    dt = (time.perf_counter() - t0) / 10
    print("u8" if u8 else "f32", f"{dt*1e3:.3f} ms", {k: round(v * 1e3, 4) for k, v in out["stage_times"].items()})
r = P.Renderer(0)
for _ in range(3):
    r.render_async(s, 0, "adagscale", K, B); r.wait()
t0 = time.perf_counter()
for _ in range(10):
    r.render_async(s, 0, "adagscale", K, B); st = r.wait()
print("device-only sync", f"{(time.perf_counter()-t0)/10*1e3:.3f} ms", st["stage_ms"])

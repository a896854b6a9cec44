"""Camera-path egress timeline: host timestamps of each frame's completion in
batch.render_views (2 contexts), plus the raw D2H copy rate of a 191 MB frame."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2604_18980_b200 as P
from paper_2604_18980_b200.batch import render_views

K = float(np.float32(0.3985099792480469 * (3600 / 1500.0) ** 2))
B = [1.0] * 20; B[7] = 0.003038157941773534; B[8] = 0.007012989837676287
s = P.synth_scene(1, 3_000_000, "veil", cameras=16, width=4608, height=3456, focal=3600.0)
nbytes = 4608 * 3456 * 12
dev = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda")
host = torch.empty(nbytes // 4, dtype=torch.float32, pin_memory=True)
for _ in range(3):
    host.copy_(dev, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    host.copy_(dev, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 10
print(f"raw D2H 191MB: {dt*1e3:.3f} ms = {nbytes/dt/1e9:.1f} GB/s")
for u8, nctx in ((False, 1), (False, 2), (False, 3), (True, 1), (True, 2), (True, 3)):
    rs = [P.Renderer(0) for _ in range(nctx)]
    kw = dict(mode="adagscale", k=K, lut_bins=B, image_u8=u8)
    render_views(rs, s, [0] * 6, on_frame=lambda i, o: None, **kw)
    ts = []
    t0 = time.perf_counter()
    render_views(rs, s, [0] * 24, on_frame=lambda i, o: ts.append(time.perf_counter() - t0), **kw)
    d = np.diff([0.0] + ts) * 1e3
    print(f"{'u8' if u8 else 'f32'} {nctx} ctx: {24/ts[-1]:.1f} FPS; per-frame ms", " ".join(f"{x:.2f}" for x in d[:8]))
for _ in range(3):
    P.render(s, 0, "adagscale", K, B)
t0 = time.perf_counter()
for _ in range(10):
    P.render(s, 0, "adagscale", K, B)
print(f"sync render(): {(time.perf_counter()-t0)/10*1e3:.3f} ms")

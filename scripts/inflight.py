"""Throughput with frames in flight on several renderer streams (config 3)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2604_18980_b200 as P
K = float(np.float32(0.3985099792480469 * (3600 / 1500.0) ** 2))
B = [1.0] * 20; B[7] = 0.003038157941773534; B[8] = 0.007012989837676287
s = P.synth_scene(1, 3_000_000, "veil", cameras=16, width=4608, height=3456, focal=3600.0)
for nstreams in (1, 2, 3, 4):
    rs = [P.Renderer(0) for _ in range(nstreams)]
    for r in rs:
        for _ in range(3):
            r.render_async(s, 0, "adagscale", K, B)
            r.wait()
    torch.cuda.synchronize()
    steps = 120
    t = time.perf_counter()
    for i in range(steps):
        rs[i % nstreams].render_async(s, 0, "adagscale", K, B)
    for r in rs:
        r.wait()
    dt = time.perf_counter() - t
    print(f"{nstreams} stream(s): {steps / dt:.1f} FPS (wall)", flush=True)

"""Render config 1/3 a few times and print counts + per-stage device times."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2604_18980_b200 as P

K1080 = 0.3985099792480469
BINS = [1.0] * 20; BINS[7] = 0.003038157941773534; BINS[8] = 0.007012989837676287
for (n, w, h, name) in ((100_000, 1920, 1080, "cfg1"), (3_000_000, 4608, 3456, "cfg3")):
    f = 500.0 * w / 640
    t = time.time(); s = P.synth_scene(1, n, "veil", cameras=16, width=w, height=h, focal=f); ts = time.time() - t
    k = float(np.float32(K1080 * (f / 1500.0) ** 2))
    r = P.Renderer(0)
    for mode, kk in (("adagscale", k), ("ellipse", 0.0)):
        for exact in (False, True):
            for it in range(4):
                r.render_async(s, 0, mode, kk, BINS if mode == "adagscale" else [], exact=exact)
                st = r.wait()
            torch_t = time.time()
            N = 10
            for it in range(N):
                r.render_async(s, 0, mode, kk, BINS if mode == "adagscale" else [], exact=exact)
            st = r.wait()
            wall = (time.time() - torch_t) / N
            print(f"{name} {mode:9s} exact={exact} pairs={st['pair_count']} splats={st['splat_count']} "
                  f"stage_ms={[round(x,3) for x in st['stage_ms']]} wall/frame={wall*1e3:.3f} ms synth={ts:.2f}s", flush=True)

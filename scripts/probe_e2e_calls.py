"""Per-call latency of the synchronous render() with a host image (config 3)."""
import statistics, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2604_18980_b200 as P
K = float(np.float32(0.3985099792480469 * (3600 / 1500.0) ** 2))
B = [1.0] * 20; B[7] = 0.003038157941773534; B[8] = 0.007012989837676287
s = P.synth_scene(1, 3_000_000, "veil", cameras=16, width=4608, height=3456, focal=3600.0)
r = P.default_renderer()
ts = []
for i in range(60):
    t = time.perf_counter()
    out = r.render(s, 0, "adagscale", K, B)
    ts.append((time.perf_counter() - t) * 1e3)
ts = ts[5:]
print(sys.argv[1] if len(sys.argv) > 1 else "", "median %.3f ms  min %.3f  p90 %.3f" % (
    statistics.median(ts), min(ts), sorted(ts)[int(0.9 * len(ts))]))

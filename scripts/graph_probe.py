"""Frame as a captured CUDA graph vs stream enqueue (launch-gap probe)."""
import ctypes as C, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2604_18980_b200 as P
from paper_2604_18980_b200 import capi
K = float(np.float32(0.3985099792480469 * (3600 / 1500.0) ** 2))
B = [1.0] * 20; B[7] = 0.003038157941773534; B[8] = 0.007012989837676287
s = P.synth_scene(1, 3_000_000, "veil", cameras=16, width=4608, height=3456, focal=3600.0)
a = s.arrays()
ctx = capi.Context(0)
dev = ctx.upload(a["mean"], a["scale"], a["rotation"], a["opacity"], a["sh"])
cam = capi.Camera.from_dict(s.camera(0))
cfg = capi.default_config("adagscale", K)
lut = capi.make_lut(B)
f = ctx.L.agsx_debug_graph_replay
f.argtypes = [C.c_void_p] * 5 + [C.c_int, C.c_void_p]
ms = C.c_float()
rc = f(ctx.h, dev, C.byref(cam), C.byref(cfg), C.byref(lut), 200, C.byref(ms))
print("graph replay rc", rc, "ms/frame %.4f" % ms.value, "fps %.1f" % (1e3 / ms.value))

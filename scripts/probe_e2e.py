"""Break down the synchronous render() end-to-end time (config 3)."""
import sys, time, ctypes as C
sys.path.insert(0, ".")
import numpy as np
import paper_2604_18980_b200 as P
from paper_2604_18980_b200 import capi
K = float(np.float32(0.3985099792480469 * (3600 / 1500.0) ** 2))
B = [1.0] * 20; B[7] = 0.003038157941773534; B[8] = 0.007012989837676287
s = P.synth_scene(1, 3_000_000, "veil", cameras=16, width=4608, height=3456, focal=3600.0)
r = P.default_renderer()
for img in (False, True):
    for _ in range(3):
        r.render(s, 0, "adagscale", K, B, image=img)
    t = time.perf_counter()
    for _ in range(10):
        out = r.render(s, 0, "adagscale", K, B, image=img)
    dt = (time.perf_counter() - t) / 10
    print(f"render(image={img}): {dt*1e3:.3f} ms/frame", flush=True)
a = out["image"]
print("image base", type(a.base), a.flags.owndata, a.ctypes.data % 4096)
keep = []
t = time.perf_counter()
for _ in range(10):
    keep.append(r.render(s, 0, "adagscale", K, B))
print(f"render keeping all: {(time.perf_counter()-t)/10*1e3:.3f} ms/frame", flush=True)
del keep
# ctypes path with an explicitly pinned buffer
ctx = capi.Context(0)
L = ctx.L
arr = s.arrays()
dev = ctx.upload(arr["mean"], arr["scale"], arr["rotation"], arr["opacity"], arr["sh"])
cam = capi.Camera.from_dict(s.camera(0))
cfg = capi.default_config("adagscale", K)
lut = capi.make_lut(B)
p = C.c_void_p()
nbytes = 4608 * 3456 * 12
assert L.agsx_host_alloc(C.c_size_t(nbytes), C.byref(p)) == 0
for mode in ("pinned", "pageable"):
    buf = p.value if mode == "pinned" else np.zeros(nbytes // 4, np.float32).ctypes.data
    hold = None if mode == "pinned" else np.zeros(nbytes // 4, np.float32)
    if hold is not None: buf = hold.ctypes.data
    f = capi.Frame(buf, None, 0, 0)
    for i in range(13):
        if i == 3: t = time.perf_counter()
        rc = L.agsx_render(ctx.h, dev, C.byref(cam), C.byref(cfg), C.byref(lut), C.byref(f))
        assert rc == 0, rc
    print(f"agsx_render {mode}: {(time.perf_counter()-t)/10*1e3:.3f} ms/frame", flush=True)

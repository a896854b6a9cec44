import sys, traceback
sys.path.insert(0, ".")
import numpy as np
from paper_2604_18980_b200 import capi
c = capi.Context(0)
def tryit(name, f):
    try:
        f(); print("OK  ", name, flush=True)
    except Exception as e:
        print("FAIL", name, e, flush=True)
        c.close(); globals()['c'] = capi.Context(0)
tryit("logf", lambda: c.logf(np.ones(10, np.float32)))
tryit("expf", lambda: c.expf(np.ones(10, np.float32)))
s = np.zeros(1, capi.SPLAT_DTYPE); s["mean2d"]=(24,24); s["cov2d"]=(4,0,4); s["inv_cov"]=(.25,0,.25); s["opacity"]=.99; s["th"]=1/255; s["depth"]=5
tryit("generate_pairs", lambda: c.generate_pairs(s, 64, 64, "ellipse", capi.default_config()))
tryit("sort_pairs", lambda: c.sort_pairs(np.arange(100, dtype=np.uint64)[::-1].copy(), np.arange(100, dtype=np.uint32), 4))
r = np.zeros((16,2), np.uint32); r[5] = (0,1)
tryit("raster", lambda: c.raster(s, np.zeros(1, np.uint32), r, 64, 64, capi.default_config()))
dev = c.upload(np.array([[0,0,5]],np.float32), np.full((1,3),.1,np.float32), np.array([[1,0,0,0]],np.float32), np.array([.8],np.float32), np.zeros((1,1,3),np.float32))
cam = capi.Camera(); cam.rotation[:] = [1,0,0,0,1,0,0,0,1]; cam.fx=cam.fy=100; cam.width=64; cam.height=48
tryit("preprocess_view", lambda: print(c.preprocess_view(dev, cam, capi.default_config())))
tryit("render", lambda: c.render(dev, cam, capi.default_config()))

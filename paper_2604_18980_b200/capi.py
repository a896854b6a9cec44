"""ctypes binding of the C-ABI in include/agsx.h (libagsx.so).

This is the FFI stub a maintainer of a ctypes-based caller would add; the
parity tests call the renderer through it so every GPU check crosses the
same boundary the reference's ``ags::render`` replacement does.  Struct
layouts mirror include/agsx.h exactly.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libagsx.so")

OK, EINVAL, EPAIR_BUDGET, ECUDA, ENOMEM, ECAPACITY, EFRAME_LOST = 0, 1, 2, 3, 4, 5, 6
MODES = {"aabb": 0, "obb": 1, "ellipse": 2, "adagscale": 3}
FLAG_EXACT_ALPHA = 1

# Every function declared in include/agsx.h.
EXPORTS = (
    "agsx_abi_version", "agsx_create", "agsx_destroy", "agsx_last_error", "agsx_stream",
    "agsx_scene_upload", "agsx_scene_free", "agsx_scene_count", "agsx_render",
    "agsx_render_async", "agsx_render_async_to", "agsx_render_async_host", "agsx_render_async_host_u8", "agsx_render_contributions", "agsx_render_wait", "agsx_device_image", "agsx_dump_tile_counts",
    "agsx_dump_sorted_pairs", "agsx_dump_ranges", "agsx_preprocess_view",
    "agsx_generate_pairs", "agsx_sort_pairs", "agsx_raster", "agsx_device_logf",
    "agsx_device_expf", "agsx_kernel_launches", "agsx_stage_history",
    "agsx_frame_stats", "agsx_host_alloc", "agsx_host_free", "agsx_device_alloc", "agsx_device_free",
    "agsx_fold_max_t", "agsx_sq_err", "agsx_render_u8",
    "agsx_project", "agsx_eval_color", "agsx_compute_th", "agsx_alpha_at", "agsx_effective_radius",
)

SPLAT_DTYPE = np.dtype(
    [
        ("mean2d", "<f4", (2,)),
        ("cov2d", "<f4", (3,)),
        ("inv_cov", "<f4", (3,)),
        ("depth", "<f4"),
        ("rgb", "<f4", (3,)),
        ("opacity", "<f4"),
        ("th", "<f4"),
        ("source_id", "<u4"),
    ]
)


class Camera(C.Structure):
    _fields_ = [
        ("position", C.c_float * 3),
        ("rotation", C.c_float * 9),
        ("fx", C.c_float),
        ("fy", C.c_float),
        ("width", C.c_int32),
        ("height", C.c_int32),
    ]

    @classmethod
    def from_dict(cls, d):
        c = cls()
        for i in range(3):
            c.position[i] = d["position"][i]
        for i in range(9):
            c.rotation[i] = d["rotation"][i]
        c.fx, c.fy, c.width, c.height = d["fx"], d["fy"], d["width"], d["height"]
        return c


class Config(C.Structure):
    _fields_ = [
        ("tile_size", C.c_int32),
        ("alpha_threshold", C.c_float),
        ("transmittance_floor", C.c_float),
        ("alpha_clamp", C.c_float),
        ("near_plane", C.c_float),
        ("guard_band", C.c_float),
        ("mode", C.c_int32),
        ("k", C.c_float),
        ("thread_count", C.c_int32),
        ("background", C.c_float * 3),
        ("fixed_radius_aabb", C.c_int32),
        ("pair_budget", C.c_uint64),
        ("flags", C.c_uint32),
    ]


class Lut(C.Structure):
    _fields_ = [
        ("depth_min", C.c_float),
        ("depth_max", C.c_float),
        ("bin_count", C.c_int32),
        ("bins", C.POINTER(C.c_float)),
    ]


class SceneDesc(C.Structure):
    _fields_ = [
        ("count", C.c_uint64),
        ("sh_coeffs", C.c_int32),
        ("mean", C.c_void_p),
        ("scale", C.c_void_p),
        ("rotation", C.c_void_p),
        ("opacity", C.c_void_p),
        ("sh", C.c_void_p),
    ]


# agsx_blend_record / BlendRecord (rasterizer.hpp:19-24)
BLEND_DTYPE = np.dtype([("pixel", "<u4"), ("splat", "<u4"), ("alpha", "<f4"), ("weight", "<f4")])


class Frame(C.Structure):
    _fields_ = [
        ("image", C.c_void_p),
        ("max_t", C.c_void_p),
        ("pair_count", C.c_uint64),
        ("splat_count", C.c_uint64),
        ("stage_ms", C.c_float * 4),
    ]


class AgsxError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"agsx status {code}: {msg}")
        self.code = code


class PairBudgetError(AgsxError):
    pass


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def default_config(mode="ellipse", k=0.0, exact=False, **kw) -> Config:
    """RenderConfig defaults (scene.hpp:65-78)."""
    c = Config()
    c.tile_size = 16
    c.alpha_threshold = 1.0 / 255.0
    c.transmittance_floor = 1e-4
    c.alpha_clamp = 0.99
    c.near_plane = 0.2
    c.guard_band = 1.3
    c.mode = MODES[mode] if isinstance(mode, str) else int(mode)
    c.k = k
    c.thread_count = 0
    c.fixed_radius_aabb = 0
    c.pair_budget = 1 << 27
    c.flags = FLAG_EXACT_ALPHA if exact else 0
    for name, v in kw.items():
        if name == "background":
            for i in range(3):
                c.background[i] = v[i]
        else:
            setattr(c, name, v)
    return c


def make_lut(bins=None, depth_min=0.0, depth_max=100.0):
    if bins is None:
        bins = [1.0] * 20
    arr = np.ascontiguousarray(bins, dtype=np.float32)
    lut = Lut(depth_min, depth_max, len(arr), arr.ctypes.data_as(C.POINTER(C.c_float)))
    lut._keep = arr
    return lut


class Lib:
    def __init__(self, path: str = LIB_PATH):
        if not os.path.exists(path):
            raise ImportError(f"libagsx.so not built: {path} (run `make` or __graft_entry__.build())")
        L = self.lib = C.CDLL(path)
        vp, u64, i32 = C.c_void_p, C.c_uint64, C.c_int32
        L.agsx_create.argtypes = [C.c_int, C.POINTER(vp)]
        L.agsx_destroy.argtypes = [vp]
        L.agsx_destroy.restype = None
        L.agsx_last_error.argtypes = [vp]
        L.agsx_last_error.restype = C.c_char_p
        L.agsx_stream.argtypes = [vp]
        L.agsx_stream.restype = vp
        L.agsx_scene_upload.argtypes = [vp, C.POINTER(SceneDesc), C.POINTER(vp)]
        L.agsx_scene_free.argtypes = [vp]
        L.agsx_scene_free.restype = None
        L.agsx_scene_count.argtypes = [vp]
        L.agsx_scene_count.restype = u64
        L.agsx_render.argtypes = [vp, vp, C.POINTER(Camera), C.POINTER(Config), C.POINTER(Lut), C.POINTER(Frame)]
        L.agsx_render_async.argtypes = [vp, vp, C.POINTER(Camera), C.POINTER(Config), C.POINTER(Lut)]
        L.agsx_render_async_to.argtypes = [vp, vp, C.POINTER(Camera), C.POINTER(Config), C.POINTER(Lut), vp]
        L.agsx_render_async_host.argtypes = [vp, vp, C.POINTER(Camera), C.POINTER(Config), C.POINTER(Lut), vp]
        L.agsx_render_async_host_u8.argtypes = [vp, vp, C.POINTER(Camera), C.POINTER(Config), C.POINTER(Lut), vp]
        L.agsx_render_contributions.argtypes = [vp, vp, C.POINTER(Camera), C.POINTER(Config), C.POINTER(Lut), vp,
                                                C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(Frame)]
        L.agsx_render_u8.argtypes = [vp, vp, C.POINTER(Camera), C.POINTER(Config), C.POINTER(Lut), vp,
                                     C.POINTER(Frame)]
        L.agsx_render_wait.argtypes = [vp, C.POINTER(Frame)]
        L.agsx_device_image.argtypes = [vp, C.POINTER(vp), C.POINTER(i32), C.POINTER(i32)]
        L.agsx_dump_tile_counts.argtypes = [vp, vp, vp, u64]
        L.agsx_dump_sorted_pairs.argtypes = [vp, vp, vp, u64, C.POINTER(u64)]
        L.agsx_dump_ranges.argtypes = [vp, vp, u64]
        L.agsx_preprocess_view.argtypes = [vp, vp, C.POINTER(Camera), C.POINTER(Config), C.POINTER(Lut), vp,
                                           C.POINTER(u64)]
        L.agsx_generate_pairs.argtypes = [vp, vp, u64, i32, i32, i32, C.POINTER(Config), vp, vp, u64, vp,
                                          C.POINTER(u64)]
        L.agsx_sort_pairs.argtypes = [vp, vp, vp, u64, i32, vp]
        L.agsx_raster.argtypes = [vp, vp, u64, vp, u64, vp, i32, i32, C.POINTER(Config), vp, vp]
        L.agsx_project.argtypes = [vp, vp, vp, vp, vp, vp]
        L.agsx_eval_color.argtypes = [vp, vp, vp, vp]
        L.agsx_compute_th.argtypes = [vp, vp, vp, u64, vp, C.c_float, C.c_float, vp]
        L.agsx_alpha_at.argtypes = [vp, vp, vp, u64, C.c_float, vp]
        L.agsx_effective_radius.argtypes = [vp, vp, vp, vp, u64, vp]
        L.agsx_device_logf.argtypes = [vp, vp, vp, u64]
        L.agsx_device_expf.argtypes = [vp, vp, vp, u64]
        L.agsx_stage_history.argtypes = [vp, vp, i32, C.POINTER(i32)]
        L.agsx_frame_stats.argtypes = [vp, vp, i32]
        L.agsx_kernel_launches.argtypes = [vp]
        L.agsx_kernel_launches.restype = u64


class Context:
    """One agsx_ctx (CUDA stream + device arenas) on `device`."""

    def __init__(self, device: int = 0, lib: Lib | None = None):
        self.L = (lib or Lib()).lib
        h = C.c_void_p()
        rc = self.L.agsx_create(device, C.byref(h))
        if rc != OK:
            raise AgsxError(rc, "agsx_create failed (no usable CUDA device?)")
        self.h = h
        self._scenes = []

    def close(self):
        if self.h:
            for s in self._scenes:
                self.L.agsx_scene_free(s)
            self._scenes = []
            self.L.agsx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc == OK:
            return
        msg = self.L.agsx_last_error(self.h).decode()
        if rc == EPAIR_BUDGET:
            raise PairBudgetError(rc, msg)
        raise AgsxError(rc, msg)

    @property
    def stream(self) -> int:
        return self.L.agsx_stream(self.h) or 0

    @property
    def kernel_launches(self) -> int:
        return self.L.agsx_kernel_launches(self.h)

    # -- scene ---------------------------------------------------------
    def upload(self, mean, scale, rotation, opacity, sh):
        arrs = [np.ascontiguousarray(a, np.float32) for a in (mean, scale, rotation, opacity, sh)]
        n = arrs[3].size
        d = SceneDesc(n, arrs[4].size // max(3 * n, 1) if n else 1, *[_p(a) for a in arrs])
        h = C.c_void_p()
        self._check(self.L.agsx_scene_upload(self.h, C.byref(d), C.byref(h)))
        self._scenes.append(h)
        return h

    # -- full pipeline ---------------------------------------------------
    def render(self, scene, cam: Camera, cfg: Config, lut=None, image=True, max_t=False, n=None):
        img = np.zeros((cam.height, cam.width, 3), np.float32) if image else None
        mt = np.zeros(max(n or self.L.agsx_scene_count(scene), 1), np.float32) if max_t else None
        f = Frame(_p(img), _p(mt), 0, 0)
        self._check(self.L.agsx_render(self.h, scene, C.byref(cam), C.byref(cfg),
                                       C.byref(lut) if lut is not None else None, C.byref(f)))
        out = {
            "pair_count": f.pair_count,
            "splat_count": f.splat_count,
            "stage_ms": list(f.stage_ms),
        }
        if image:
            out["image"] = img
        if max_t:
            out["max_t_by_gid"] = mt
        return out

    def render_contributions(self, scene, cam: Camera, cfg: Config, lut=None):
        """(image, records): agsx_render_contributions, sized by a first call."""
        img = np.zeros((cam.height, cam.width, 3), np.float32)
        f = Frame(_p(img), None, 0, 0)
        count = C.c_uint64()
        lp = C.byref(lut) if lut is not None else None
        rc = self.L.agsx_render_contributions(self.h, scene, C.byref(cam), C.byref(cfg), lp, None, 0,
                                              C.byref(count), C.byref(f))
        if rc not in (0, 5):
            self._check(rc)
        rec = np.zeros(max(count.value, 1), BLEND_DTYPE)
        self._check(self.L.agsx_render_contributions(self.h, scene, C.byref(cam), C.byref(cfg), lp,
                                                     rec.ctypes.data_as(C.c_void_p), len(rec), C.byref(count),
                                                     C.byref(f)))
        return img, rec[: count.value]

    def render_async(self, scene, cam, cfg, lut=None):
        self._check(self.L.agsx_render_async(self.h, scene, C.byref(cam), C.byref(cfg),
                                             C.byref(lut) if lut is not None else None))

    def render_async_host(self, scene, cam, cfg, lut, image):
        """agsx_render_async_host: the frame lands in `image` (float32 H x W x 3,
        host memory) by agsx_render_wait; `image` must stay alive until then."""
        self._check(self.L.agsx_render_async_host(self.h, scene, C.byref(cam), C.byref(cfg),
                                                  C.byref(lut) if lut is not None else None, _p(image)))

    def wait(self):
        f = Frame()
        self._check(self.L.agsx_render_wait(self.h, C.byref(f)))
        return {"pair_count": f.pair_count, "splat_count": f.splat_count, "stage_ms": list(f.stage_ms)}

    def stage_history(self, max_frames=64):
        ms = np.zeros((max_frames, 4), np.float32)
        n = C.c_int32()
        self._check(self.L.agsx_stage_history(self.h, _p(ms), max_frames, C.byref(n)))
        return ms[: n.value]

    def frame_stats(self):
        v = np.zeros(6, np.uint64)
        self._check(self.L.agsx_frame_stats(self.h, _p(v), 6))
        return dict(zip(("splat_count", "splats_with_tiles", "pair_count", "p_it", "overflow", "tiles"),
                        (int(x) for x in v)))

    def device_image(self):
        p = C.c_void_p()
        w, h = C.c_int32(), C.c_int32()
        self._check(self.L.agsx_device_image(self.h, C.byref(p), C.byref(w), C.byref(h)))
        return p.value, w.value, h.value

    def dump_tile_counts(self, n):
        counts = np.zeros(max(n, 1), np.uint32)
        alive = np.zeros(max(n, 1), np.uint8)
        self._check(self.L.agsx_dump_tile_counts(self.h, _p(counts), _p(alive), n))
        return counts[:n], alive[:n].astype(bool)

    def dump_sorted_pairs(self):
        cnt = C.c_uint64()
        rc = self.L.agsx_dump_sorted_pairs(self.h, None, None, 0, C.byref(cnt))
        if rc not in (OK, ECAPACITY):
            self._check(rc)
        keys = np.zeros(max(cnt.value, 1), np.uint64)
        gids = np.zeros(max(cnt.value, 1), np.uint32)
        self._check(self.L.agsx_dump_sorted_pairs(self.h, _p(keys), _p(gids), cnt.value, C.byref(cnt)))
        return keys[: cnt.value], gids[: cnt.value]

    def dump_ranges(self, tile_count):
        r = np.zeros((max(tile_count, 1), 2), np.uint32)
        self._check(self.L.agsx_dump_ranges(self.h, _p(r), tile_count))
        return r[:tile_count]

    # -- stage entry points ------------------------------------------------
    def preprocess_view(self, scene, cam, cfg, lut=None):
        n = self.L.agsx_scene_count(scene)
        out = np.zeros(max(n, 1), SPLAT_DTYPE)
        cnt = C.c_uint64()
        self._check(self.L.agsx_preprocess_view(self.h, scene, C.byref(cam), C.byref(cfg),
                                                C.byref(lut) if lut is not None else None, _p(out),
                                                C.byref(cnt)))
        return out[: cnt.value].copy()

    def generate_pairs(self, splats, width, height, mode, cfg):
        splats = np.ascontiguousarray(splats, SPLAT_DTYPE)
        n = len(splats)
        counts = np.zeros(max(n, 1), np.uint32)
        total = C.c_uint64()
        mode = MODES[mode] if isinstance(mode, str) else int(mode)
        rc = self.L.agsx_generate_pairs(self.h, _p(splats), n, width, height, mode, C.byref(cfg), None, None,
                                        0, _p(counts), C.byref(total))
        if rc not in (OK, ECAPACITY):
            self._check(rc)
        keys = np.zeros(max(total.value, 1), np.uint64)
        idx = np.zeros(max(total.value, 1), np.uint32)
        self._check(self.L.agsx_generate_pairs(self.h, _p(splats), n, width, height, mode, C.byref(cfg),
                                               _p(keys), _p(idx), total.value, _p(counts), C.byref(total)))
        t = total.value
        return keys[:t].copy(), idx[:t].copy(), counts[:n].copy()

    def sort_pairs(self, keys, idx, tile_count):
        keys = np.array(keys, np.uint64, copy=True)
        idx = np.array(idx, np.uint32, copy=True)
        ranges = np.zeros((max(tile_count, 1), 2), np.uint32)
        self._check(self.L.agsx_sort_pairs(self.h, _p(keys), _p(idx), len(keys), tile_count, _p(ranges)))
        return keys, idx, ranges[:tile_count]

    def raster(self, splats, idx, ranges, width, height, cfg, max_t=False):
        splats = np.ascontiguousarray(splats, SPLAT_DTYPE)
        idx = np.ascontiguousarray(idx, np.uint32)
        ranges = np.ascontiguousarray(ranges, np.uint32)
        img = np.zeros((height, width, 3), np.float32)
        mt = np.zeros(max(len(splats), 1), np.float32) if max_t else None
        self._check(self.L.agsx_raster(self.h, _p(splats), len(splats), _p(idx), len(idx), _p(ranges), width,
                                       height, C.byref(cfg), _p(img), _p(mt)))
        return (img, mt[: len(splats)]) if max_t else img

    # ---- per-element helpers (the device functions of the stages) ----------
    def project(self, scene, cam, cfg):
        """project (preprocess.cpp:26-66) of every Gaussian of an uploaded scene:
        (valid[n] bool, out[n, 6] = mean2d.xy, cov2d xx/xy/yy, depth)."""
        n = self.L.agsx_scene_count(scene)
        valid = np.zeros(max(n, 1), np.uint8)
        out = np.zeros((max(n, 1), 6), np.float32)
        self._check(self.L.agsx_project(self.h, scene, C.byref(cam), C.byref(cfg), _p(valid), _p(out)))
        return valid[:n].astype(bool), out[:n]

    def eval_color(self, scene, dirs):
        dirs = np.ascontiguousarray(dirs, np.float32).reshape(-1, 3)
        rgb = np.zeros_like(dirs)
        self._check(self.L.agsx_eval_color(self.h, scene, _p(dirs), _p(rgb)))
        return rgb

    def compute_th(self, cov2d, depth, lut, k, tau):
        cov2d = np.ascontiguousarray(cov2d, np.float32).reshape(-1, 3)
        depth = np.ascontiguousarray(depth, np.float32)
        th = np.zeros(len(depth), np.float32)
        self._check(self.L.agsx_compute_th(self.h, _p(cov2d), _p(depth), len(depth),
                                           C.byref(lut) if lut is not None else None, k, tau, _p(th)))
        return th

    def alpha_at(self, splats, px, alpha_clamp):
        splats = np.ascontiguousarray(splats, SPLAT_DTYPE)
        px = np.ascontiguousarray(px, np.float32).reshape(-1, 2)
        a = np.zeros(len(splats), np.float32)
        self._check(self.L.agsx_alpha_at(self.h, _p(splats), _p(px), len(splats), alpha_clamp, _p(a)))
        return a

    def effective_radius(self, opacity, th, cov2d):
        opacity = np.ascontiguousarray(opacity, np.float32)
        th = np.ascontiguousarray(th, np.float32)
        cov2d = np.ascontiguousarray(cov2d, np.float32).reshape(-1, 3)
        out = np.zeros((len(opacity), 2), np.float32)
        self._check(self.L.agsx_effective_radius(self.h, _p(opacity), _p(th), _p(cov2d), len(opacity), _p(out)))
        return out

    def logf(self, x):
        x = np.ascontiguousarray(x, np.float32)
        y = np.empty_like(x)
        self._check(self.L.agsx_device_logf(self.h, _p(x), _p(y), x.size))
        return y

    def expf(self, x):
        x = np.ascontiguousarray(x, np.float32)
        y = np.empty_like(x)
        self._check(self.L.agsx_device_expf(self.h, _p(x), _p(y), x.size))
        return y

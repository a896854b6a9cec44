"""ctypes front-end for the CPU oracles -- TEST INFRASTRUCTURE ONLY.

Loads either
  * ``port``      -> oracle/_build/libags_oracle.so (C restatement, ags_oracle.c)
  * ``reference`` -> oracle/_ref/libags_ref.so      (unmodified reference
                     sources + ref_shim.cpp)
and exposes numpy-level wrappers with identical signatures.  Only tests/,
``__graft_entry__.smoke()`` and bench.py's CPU-baseline / ``--impl reference``
legs import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATHS = {
    "port": os.path.join(HERE, "_build", "libags_oracle.so"),
    "reference": os.path.join(HERE, "_ref", "libags_ref.so"),
}

MODES = {"aabb": 0, "obb": 1, "ellipse": 2, "adagscale": 3}
AGO_OK, AGO_EINVAL, AGO_EPAIR_BUDGET, AGO_ECAPACITY = 0, 1, 2, 5

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
assert SPLAT_DTYPE.itemsize == 60


class Camera(C.Structure):
    _fields_ = [
        ("position", C.c_float * 3),
        ("rotation", C.c_float * 9),
        ("fx", C.c_float),
        ("fy", C.c_float),
        ("width", C.c_int32),
        ("height", C.c_int32),
    ]


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
        ("mean", C.POINTER(C.c_float)),
        ("scale", C.POINTER(C.c_float)),
        ("rotation", C.POINTER(C.c_float)),
        ("opacity", C.POINTER(C.c_float)),
        ("sh", C.POINTER(C.c_float)),
    ]


def _fp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


# BlendRecord (rasterizer.hpp:19-24) / ago_blend / agsx_blend_record
BLEND_DTYPE = np.dtype([("pixel", "<u4"), ("splat", "<u4"), ("alpha", "<f4"), ("weight", "<f4")])


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: oracle status {code}")
        self.code = code


class PairBudgetError(OracleError):
    pass


@dataclass
class SoAScene:
    """Struct-of-arrays scene (float32, C-contiguous)."""

    mean: np.ndarray  # (N,3)
    scale: np.ndarray  # (N,3)
    rotation: np.ndarray  # (N,4) w,x,y,z
    opacity: np.ndarray  # (N,)
    sh: np.ndarray  # (N, D, 3) coefficient-major
    cameras: list

    @property
    def count(self) -> int:
        return int(self.opacity.shape[0])

    def desc(self) -> SceneDesc:
        return SceneDesc(
            self.count,
            int(self.sh.shape[1]),
            _fp(self.mean),
            _fp(self.scale),
            _fp(self.rotation),
            _fp(self.opacity),
            _fp(self.sh),
        )


def camera_to_dict(c: Camera) -> dict:
    return {
        "position": list(c.position),
        "rotation": list(c.rotation),
        "fx": c.fx,
        "fy": c.fy,
        "width": c.width,
        "height": c.height,
    }


def camera_from_dict(d: dict) -> Camera:
    c = Camera()
    for i in range(3):
        c.position[i] = d["position"][i]
    for i in range(9):
        c.rotation[i] = d["rotation"][i]
    c.fx, c.fy, c.width, c.height = d["fx"], d["fy"], d["width"], d["height"]
    return c


class Oracle:
    def __init__(self, kind: str = "port"):
        path = LIB_PATHS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library not built: {path}")
        self.kind = kind
        self.lib = L = C.CDLL(path)
        L.ago_kind.restype = C.c_char_p
        L.ago_default_config.argtypes = [C.POINTER(Config)]
        L.ago_synth_scene.argtypes = [
            C.c_uint64, C.c_int32, C.c_char_p, C.c_int32, C.c_int32, C.c_int32,
            C.c_float, C.c_float, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
            C.c_void_p, C.c_void_p,
        ]
        L.ago_preprocess.argtypes = [
            C.POINTER(SceneDesc), C.POINTER(Camera), C.POINTER(Config),
            C.POINTER(Lut), C.c_void_p, C.POINTER(C.c_uint64),
        ]
        L.ago_generate_pairs.argtypes = [
            C.c_void_p, C.c_uint64, C.c_int32, C.c_int32, C.c_int32,
            C.POINTER(Config), C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p,
            C.POINTER(C.c_uint64),
        ]
        L.ago_sort_pairs.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int32, C.c_void_p]
        L.ago_raster.argtypes = [
            C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p,
            C.c_int32, C.c_int32, C.POINTER(Config), C.c_void_p, C.c_void_p,
        ]
        if hasattr(L, "ago_raster_pit"):  # the C restatement only
            L.ago_raster_pit.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                         C.POINTER(Config), C.c_void_p, C.POINTER(C.c_uint64)]
        L.ago_render.argtypes = [
            C.POINTER(SceneDesc), C.POINTER(Camera), C.POINTER(Config),
            C.POINTER(Lut), C.c_void_p, C.POINTER(C.c_uint64),
            C.POINTER(C.c_uint64), C.c_void_p, C.c_void_p,
        ]
        L.ago_psnr.restype = C.c_double
        L.ago_psnr.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64]
        L.ago_logf_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64]
        L.ago_expf_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64]
        assert L.ago_kind().decode() == kind

    # -- configs -------------------------------------------------------
    def config(self, mode="ellipse", k=0.0, **kw) -> Config:
        c = Config()
        self.lib.ago_default_config(C.byref(c))
        c.mode = MODES[mode] if isinstance(mode, str) else int(mode)
        c.k = k
        for name, v in kw.items():
            if name == "background":
                for i in range(3):
                    c.background[i] = v[i]
            else:
                setattr(c, name, v)
        return c

    @staticmethod
    def lut(bins=None, depth_min=0.0, depth_max=100.0):
        if bins is None or len(bins) == 0:
            return None
        arr = np.ascontiguousarray(bins, dtype=np.float32)
        lut = Lut(depth_min, depth_max, len(arr), _fp(arr))
        lut._keep = arr  # keep the buffer alive
        return lut

    # -- stages ----------------------------------------------------------
    def synth_scene(self, seed, count, layout="slab", cameras=24, width=640,
                    height=480, focal=500.0, fy=None) -> SoAScene:
        fy = focal if fy is None else fy
        mean = np.zeros((count, 3), np.float32)
        scale = np.zeros((count, 3), np.float32)
        rot = np.zeros((count, 4), np.float32)
        op = np.zeros(count, np.float32)
        sh = np.zeros((count, 1, 3), np.float32)
        cams = (Camera * max(cameras, 1))()
        rc = self.lib.ago_synth_scene(seed, count, layout.encode(), cameras, width, height,
                                      focal, fy, _p(mean), _p(scale), _p(rot), _p(op),
                                      _p(sh), C.cast(cams, C.c_void_p))
        if rc:
            raise OracleError(rc, "synth_scene")
        return SoAScene(mean, scale, rot, op, sh, [cams[i] for i in range(cameras)])

    def preprocess(self, scene: SoAScene, cam, cfg, lut=None) -> np.ndarray:
        out = np.zeros(max(scene.count, 1), SPLAT_DTYPE)
        n = C.c_uint64()
        d = scene.desc()
        if cfg.mode == MODES["adagscale"] and lut is None:
            lut = Lut(0.0, 100.0, 0, None)  # all-ones default
        rc = self.lib.ago_preprocess(C.byref(d), C.byref(cam), C.byref(cfg),
                                     C.byref(lut) if lut is not None else None,
                                     _p(out), C.byref(n))
        if rc:
            raise OracleError(rc, "preprocess")
        return out[: n.value].copy()

    def generate_pairs(self, splats: np.ndarray, width, height, mode, cfg):
        splats = np.ascontiguousarray(splats, SPLAT_DTYPE)
        n = len(splats)
        counts = np.zeros(max(n, 1), np.uint32)
        total = C.c_uint64()
        mode = MODES[mode] if isinstance(mode, str) else int(mode)
        rc = self.lib.ago_generate_pairs(_p(splats), n, width, height, mode, C.byref(cfg),
                                         None, None, 0, _p(counts), C.byref(total))
        if rc == AGO_EPAIR_BUDGET:
            raise PairBudgetError(rc, "generate_pairs")
        keys = np.zeros(max(total.value, 1), np.uint64)
        idx = np.zeros(max(total.value, 1), np.uint32)
        rc = self.lib.ago_generate_pairs(_p(splats), n, width, height, mode, C.byref(cfg),
                                         _p(keys), _p(idx), total.value, _p(counts),
                                         C.byref(total))
        if rc:
            raise OracleError(rc, "generate_pairs")
        t = total.value
        return keys[:t].copy(), idx[:t].copy(), counts[:n].copy()

    def sort_pairs(self, keys, idx, tile_count):
        keys = np.array(keys, np.uint64, copy=True)
        idx = np.array(idx, np.uint32, copy=True)
        ranges = np.zeros((max(tile_count, 1), 2), np.uint32)
        rc = self.lib.ago_sort_pairs(_p(keys), _p(idx), len(keys), tile_count, _p(ranges))
        if rc:
            raise OracleError(rc, "sort_pairs")
        return keys, idx, ranges[:tile_count]

    def raster(self, splats, keys, idx, ranges, width, height, cfg, max_t=False):
        splats = np.ascontiguousarray(splats, SPLAT_DTYPE)
        img = np.zeros((height, width, 3), np.float32)
        mt = np.zeros(max(len(splats), 1), np.float32) if max_t else None
        keys = np.ascontiguousarray(keys, np.uint64)
        idx = np.ascontiguousarray(idx, np.uint32)
        ranges = np.ascontiguousarray(ranges, np.uint32)
        rc = self.lib.ago_raster(_p(splats), len(splats), _p(keys), _p(idx), len(idx),
                                 _p(ranges), width, height, C.byref(cfg), _p(img), _p(mt))
        if rc:
            raise OracleError(rc, "raster")
        return (img, mt[: len(splats)]) if max_t else img

    def raster_pit(self, splats, idx, ranges, width, height, cfg):
        """P_it of the raster (rasterizer.cpp:55-56): pairs visited before each
        tile saturates, summed over the tiles; returns (image, p_it)."""
        splats = np.ascontiguousarray(splats, SPLAT_DTYPE)
        img = np.zeros((height, width, 3), np.float32)
        idx = np.ascontiguousarray(idx, np.uint32)
        ranges = np.ascontiguousarray(ranges, np.uint32)
        pit = C.c_uint64()
        rc = self.lib.ago_raster_pit(_p(splats), len(splats), _p(idx), _p(ranges), width, height, C.byref(cfg),
                                     _p(img), C.byref(pit))
        if rc:
            raise OracleError(rc, "raster_pit")
        return img, pit.value

    def render(self, scene: SoAScene, cam, cfg, lut=None, max_t=False):
        img = np.zeros((cam.height, cam.width, 3), np.float32)
        pc, sc = C.c_uint64(), C.c_uint64()
        mt = np.zeros(max(scene.count, 1), np.float32) if max_t else None
        st = np.zeros(4, np.float64)
        d = scene.desc()
        if cfg.mode == MODES["adagscale"] and lut is None:
            lut = Lut(0.0, 100.0, 0, None)
        rc = self.lib.ago_render(C.byref(d), C.byref(cam), C.byref(cfg),
                                 C.byref(lut) if lut is not None else None,
                                 _p(img), C.byref(pc), C.byref(sc), _p(mt), _p(st))
        if rc == AGO_EPAIR_BUDGET:
            raise PairBudgetError(rc, "render")
        if rc:
            raise OracleError(rc, "render")
        out = {
            "image": img,
            "pair_count": pc.value,
            "splat_count": sc.value,
            "stage_times": dict(zip(("preprocess", "pair_gen", "sort", "raster"), st.tolist())),
        }
        if max_t:
            out["max_t"] = mt[: sc.value].copy()
        return out

    def render_contributions(self, scene: SoAScene, cam, cfg, lut=None):
        """render with RecordOptions::contributions: (image, records) with records a
        structured array {pixel u32, splat u32, alpha f32, weight f32} in the
        reference's order (tile index, then pair, then row-major pixel)."""
        img = np.zeros((cam.height, cam.width, 3), np.float32)
        d = scene.desc()
        if cfg.mode == MODES["adagscale"] and lut is None:
            lut = Lut(0.0, 100.0, 0, None)
        count = C.c_uint64()
        args = (C.byref(d), C.byref(cam), C.byref(cfg), C.byref(lut) if lut is not None else None, _p(img))
        rc = self.lib.ago_render_contributions(*args, None, 0, C.byref(count))
        if rc not in (AGO_OK, AGO_ECAPACITY):
            raise OracleError(rc, "render_contributions")
        rec = np.zeros(max(count.value, 1), BLEND_DTYPE)
        rc = self.lib.ago_render_contributions(*args, rec.ctypes.data_as(C.c_void_p), len(rec), C.byref(count))
        if rc:
            raise OracleError(rc, "render_contributions")
        return img, rec[: count.value]

    def calibrate(self, scene: SoAScene, target_drop: float, calib_views: int = 16, thread_count: int = 0):
        """Reference calibrate_scene (build_lut + search_k); reference build only."""
        if not hasattr(self.lib, "ago_calibrate"):
            raise OracleError(1, "calibrate: only the reference build exports it")
        n = min(calib_views, len(scene.cameras))
        cams = (Camera * max(n, 1))(*scene.cameras[:n])
        k, ach = C.c_double(), C.c_double()
        it = C.c_int32()
        bins = np.zeros(64, np.float32)
        dmin, dmax = C.c_float(), C.c_float()
        d = scene.desc()
        f = self.lib.ago_calibrate
        f.restype = C.c_int
        f.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_double, C.c_int32, C.c_void_p, C.c_void_p,
                      C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]
        rc = f(C.addressof(d), C.addressof(cams), n, target_drop, thread_count, C.addressof(k), C.addressof(ach),
               C.addressof(it), _p(bins), 64, C.addressof(dmin), C.addressof(dmax))
        if rc:
            raise OracleError(rc, "calibrate")
        return {"k": k.value, "achieved_drop": ach.value, "iterations": it.value, "lut_bins": bins[:20].tolist(),
                "lut_depth_min": dmin.value, "lut_depth_max": dmax.value}

    def load_ply(self, path: str):
        """Reference load_ply_file (gsio.cpp:80-157) -> (SoAScene without cameras, rejected)."""
        if not hasattr(self.lib, "ago_load_ply"):
            raise OracleError(1, "load_ply: only the reference build exports it")
        f = self.lib.ago_load_ply
        f.restype = C.c_int
        f.argtypes = [C.c_char_p] + [C.c_void_p] * 8
        n, co, rej = C.c_uint64(), C.c_int32(), C.c_uint64()
        rc = f(path.encode(), C.addressof(n), C.addressof(co), C.addressof(rej), None, None, None, None, None)
        if rc:
            raise OracleError(rc, "load_ply")
        cnt, D = n.value, co.value
        mean = np.zeros((cnt, 3), np.float32)
        scale = np.zeros((cnt, 3), np.float32)
        rot = np.zeros((cnt, 4), np.float32)
        op = np.zeros(cnt, np.float32)
        sh = np.zeros((cnt, D, 3), np.float32)
        rc = f(path.encode(), C.addressof(n), C.addressof(co), C.addressof(rej), _p(mean), _p(scale), _p(rot),
               _p(op), _p(sh))
        if rc:
            raise OracleError(rc, "load_ply")
        return SoAScene(mean, scale, rot, op, sh, []), rej.value

    def orbit_cameras(self, path: str, count, width, height, fx, fy, seed):
        """Reference orbit_cameras (synth.cpp:254-281) around the PLY scene at `path`."""
        f = self.lib.ago_orbit_cameras
        f.restype = C.c_int
        f.argtypes = [C.c_char_p, C.c_int32, C.c_int32, C.c_int32, C.c_float, C.c_float, C.c_uint64, C.c_void_p]
        cams = (Camera * max(count, 1))()
        rc = f(path.encode(), count, width, height, fx, fy, seed, C.cast(cams, C.c_void_p))
        if rc:
            raise OracleError(rc, "orbit_cameras")
        return [cams[i] for i in range(count)]

    def pair_report(self, scene: SoAScene, n_views, specs, lut=None):
        """Reference pair_report over views [0, n_views): rows of (pair_count, reduction_pct, psnr_drop_db)."""
        f = self.lib.ago_pair_report
        f.restype = C.c_int
        f.argtypes = [C.c_void_p] * 2 + [C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]
        cams = (Camera * n_views)(*scene.cameras[:n_views])
        modes = np.array([MODES[m] for m, _ in specs], np.int32)
        ks = np.array([k for _, k in specs], np.float64)
        rows = np.zeros((len(specs), 3), np.float64)
        d = scene.desc()
        rc = f(C.addressof(d), C.addressof(cams), n_views, _p(modes), _p(ks), len(specs),
               C.addressof(lut) if lut is not None else None, _p(rows))
        if rc:
            raise OracleError(rc, "pair_report")
        return rows

    def psnr(self, a, b) -> float:
        a = np.ascontiguousarray(a, np.float32).ravel()
        b = np.ascontiguousarray(b, np.float32).ravel()
        return float(self.lib.ago_psnr(_p(a), _p(b), a.size))

    def logf(self, x):
        x = np.ascontiguousarray(x, np.float32)
        y = np.empty_like(x)
        self.lib.ago_logf_batch(_p(x), _p(y), x.size)
        return y

    def expf(self, x):
        x = np.ascontiguousarray(x, np.float32)
        y = np.empty_like(x)
        self.lib.ago_expf_batch(_p(x), _p(y), x.size)
        return y


def available(kind: str) -> bool:
    return os.path.exists(LIB_PATHS[kind])

#!/usr/bin/env python3
"""Benchmark of the B200 AdaGScale render path (BASELINE.json metric).

Workload (N=1): BASELINE config 3 -- synthetic `veil` scene, 3M Gaussians,
4608x3456, view 0, AdaGScale on with the reference-calibrated LUT and K scaled
to the resolution.  One step = one frame (preprocess ->
pair generation -> sort -> rasterize) with the scene resident in HBM.
N>1 (torchrun): view-partitioned replicas, rank r renders view r of the
camera path each step (weak scaling); no collective on the data path, only a
max-over-ranks of the timed region and a sum of the frame counts.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0.  `--impl reference` times the reference's own
CPU implementation (oracle/_ref, built from the reference sources) on the
host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FPS at 4608x3456, 3M Gaussians; tile pairs/frame; PSNR vs CPU ref"
K1080 = 0.3985099792480469
LUT_BINS = [1.0] * 20
LUT_BINS[7] = 0.003038157941773534
LUT_BINS[8] = 0.007012989837676287

CONFIGS = {
    # name: (gaussians, width, height, camera_count)
    "1": (100_000, 1920, 1080, 16),
    "2": (1_000_000, 4608, 3456, 16),
    "3": (3_000_000, 4608, 3456, 16),
    "4": (3_000_000, 3660, 3200, 16),
    "5": (6_000_000, 4608, 3456, 64),
}


def scaled_k(width: int) -> float:
    f = 500.0 * width / 640.0
    return float(np.float32(K1080 * (f / 1500.0) ** 2))


def workload_name(cfg: str, mode: str) -> str:
    n, w, h, _ = CONFIGS[cfg]
    return f"config{cfg}: synthetic veil {n} Gaussians, {w}x{h}, {mode}" + (
        f" (K={scaled_k(w):.4f}, calibrated LUT)" if mode == "adagscale" else ""
    )


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        t0 = time.time()
        while not self.lines and time.time() - t0 < 3.0:  # first sample before the timed region
            time.sleep(0.02)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": max(smax) if smax else None,
            "reasons": sorted(reasons),
            "samples": len(sm),
        }


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "src": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "src": "fallback (B200_PROFILING.md)"}


# ------------------------------------------------------ algorithmic bytes
HBM_SPEC_GBS = 8000.0  # B200 HBM3e spec (BASELINE.md §2-3 reporting convention)


def survey_bytes(n, s, p, p_it, tiles, px):
    """SURVEY.md §8(d)'s per-stage formulas (d = 1 SH coefficient): the
    reference's own formulation (6 passes of a 64-bit pair sort).  Kept as a
    labelled comparison only; the roofline uses `moved_bytes`."""
    return {
        "preprocess": n * (44 + 12) + 4 * n + 44 * s,
        "pair_gen": 8 * n + 28 * s + 12 * p,
        "sort": 160 * p + 8 * tiles,
        "raster": 40 * p_it + 8 * tiles + 12 * px,
    }


def moved_bytes(n, m, p, p_it, tiles, px, depth_passes, bucketed):
    """Bytes each stage's kernels must move in THIS formulation (SH degree 0,
    n Gaussians, m splats with >= 1 tile, p pairs, tiles, px pixels).

    Depth-then-tile path (default):
      preprocess  K1 reads the 56 B scene SoA and the 4 B slot -> id map
                  (scene in Morton order), writes status + depth
                  key (8 B) per Gaussian and the 64 B P0..P3 planes per splat
                  with tiles, zeroes ranges / P_it words (16 B per tile);
      sort        depth pass 0 (upsweep + downsweep read 4 B keys of all n, the
                  downsweep 4 B slot values, 8 B key+value written per splat),
                  depth passes 1.. (4 B
                  upsweep read + 8 B read + 8 B write per splat), the last
                  pass's tile-count by-product (4 B gather + 4 B write per
                  splat), 2 tile passes over the pairs (4 + 8 + 8 B each),
                  the ranges (4 B read per pair, 8 B per tile);
      pair_gen    K3 reads the depth order, counts and P3 records (24 B per
                  splat) and writes 8 B per pair;
      raster      per pair iterated the 4 B value + the 48 B P0/P1/P2 record,
                  8 B range + 8 B P_it word per tile, the 12 B image pixel.
    Tile-bucketed path (AGSX_SORT=bucket): K1 adds a 4 B reduction per pair
    and writes a 24 B list entry per splat instead of P3 + depth key; the
    scatter reads the list and does a 4 B atomic + 8 B write per pair; the
    sort reads 8 B and writes 4 B per pair plus the scan (8 histogram slices
    per tile read and written, 8 B range: 72 B per tile)."""
    raster = 52 * p_it + 16 * tiles + 12 * px
    if bucketed:
        return {
            "preprocess": 56 * n + 4 * n + 48 * m + 24 * m + 8 * p + 16 * tiles,
            "pair_gen": 24 * m + 8 * p + 8 * p,
            "sort": 72 * tiles + 8 * p + 4 * p,
            "raster": raster,
        }
    return {
        "preprocess": 56 * n + 4 * n + 8 * n + 64 * m + 16 * tiles,
        "pair_gen": 24 * m + 8 * p,
        "sort": (12 * n + 8 * m) + max(depth_passes - 1, 0) * 20 * m + 8 * m + 2 * 20 * p + 4 * p + 8 * tiles,
        "raster": raster,
    }


# ---------------------------------------------------------- reference arm
def cpu_reference(cfg: str, mode: str, frames: int, warmup: int, want_image=False):
    """The reference CPU render (oracle/_ref, unmodified reference sources)."""
    from oracle.ffi import Oracle, available

    kind = "reference" if available("reference") else "port"
    o = Oracle(kind)
    n, w, h, cams = CONFIGS[cfg]
    f = 500.0 * w / 640.0
    scene = o.synth_scene(1, n, "veil", cameras=cams, width=w, height=h, focal=f)
    threads = os.cpu_count() or 1
    extra = {"fixed_radius_aabb": 1} if mode == "aabb_fixed3" else {}
    c = o.config("aabb" if mode == "aabb_fixed3" else mode, k=scaled_k(w) if mode == "adagscale" else 0.0,
                 thread_count=threads, **extra)
    lut = o.lut(LUT_BINS) if mode == "adagscale" else None
    times, out = [], None
    for i in range(warmup + frames):
        out = o.render(scene, scene.cameras[0], c, lut)
        if i >= warmup:
            times.append(sum(out["stage_times"].values()) if kind == "reference" else None)
    return kind, threads, times, out


def run_reference_arm(args, rank):
    if rank != 0:
        return
    mode = args.mode
    # bounded sample: the reference renders config 3 at ~1 frame/s on a 16-core
    # host, so at most 20 timed frames (+1 warm-up) keep the arm within minutes
    frames = max(1, min(args.steps, 20))
    warm = min(args.warmup, 1)
    t0 = time.perf_counter()
    kind, threads, times, out = cpu_reference(args.config, mode, frames, warm)
    wall = time.perf_counter() - t0
    frame_s = sum(times) / len(times) if times and times[0] is not None else wall / (frames + warm)
    fps = 1.0 / frame_s
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": fps,
        "unit": "frames/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": frame_s * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (reference synth_scene, seed 1)",
        "config": {"workload": workload_name(args.config, mode), "mode": mode,
                   "pair_count": out["pair_count"], "splat_count": out["splat_count"]},
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": threads, "kind": kind,
                         "sample": f"{frames} full frames of config {args.config} (of the {args.steps} requested) "
                                   f"after {warm} warm-up, stage_times summed (reference render() on {threads} "
                                   f"threads)"},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "stage_times_s": out["stage_times"],
    }
    print(json.dumps(line, default=_jsonable), flush=True)


def _jsonable(o):
    if isinstance(o, (np.floating, np.integer)):
        return o.item()
    if isinstance(o, np.ndarray):
        return o.tolist()
    raise TypeError(type(o).__name__)


# ------------------------------------------------- CUB sort comparator
def cub_comparator(r, scene, view, mode, k, bins, exact, iters=20):
    """cub::DeviceRadixSort::SortPairs (the paper's sort) on this
    frame's pair set: 64-bit (tile << 32 | depth bits) keys with the Gaussian
    id as value, bits [0, 32 + ceil(log2 T)), in the reference's emission
    order (Gaussian id, tiles ascending).  Bench-only (scripts/cub_sort.cu);
    compared with this pipeline's device-timed sort stage, and its sort +
    pair_gen stages, on the AdaGScale on and off pair sets."""
    import torch

    so = os.path.join(ROOT, "scripts", "_build", "libcubsort.so")
    if not os.path.exists(so):
        return {"unavailable": "scripts/_build/libcubsort.so not built"}
    lib = ctypes.CDLL(so)
    lib.cub_sort_pairs_u64.restype = ctypes.c_int
    lib.cub_sort_pairs_u64.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                                                               ctypes.c_int, ctypes.POINTER(ctypes.c_float),
                                                               ctypes.c_void_p]
    res = {}
    for label, (md, kk, bb) in (("adagscale_on", (mode, k, bins)), ("adagscale_off", ("ellipse", 0.0, []))):
        if label == "adagscale_on" and mode != "adagscale":
            continue
        r.render_async(scene, view, md, kk, bb, exact=exact)
        r.wait()  # sizes the pair arena: a chain cannot re-run an overflowed frame
        for _ in range(5):
            r.render_async(scene, view, md, kk, bb, exact=exact)
        r.wait()
        ours = r.stage_history(5).mean(axis=0)
        tiles = r.frame_stats()["tiles"]
        keys, gids = r.dump_sorted_pairs()
        p = int(len(keys))
        tb = max(1, int(np.ceil(np.log2(max(tiles, 2)))))
        kd = torch.from_numpy(keys.view(np.int64)).cuda()
        gd = torch.from_numpy(gids.astype(np.int64)).cuda()
        order = torch.sort(gd, stable=True).indices  # emission order: Gaussian id, then tile (stable)
        kin, vin = kd[order].contiguous(), gd[order].to(torch.int32).contiguous()
        kout, vout = torch.empty_like(kin), torch.empty_like(vin)
        ms = ctypes.c_float(0.0)
        # on torch's current stream: ordered after the gathers that built kin / vin
        rc = lib.cub_sort_pairs_u64(kin.data_ptr(), vin.data_ptr(), kout.data_ptr(), vout.data_ptr(), p, 0,
                                    32 + tb, iters, ctypes.byref(ms), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        same = bool(torch.equal(kout, kd) and torch.equal(vout.to(torch.int64), gd))
        cub_ms = float(ms.value)
        res[label] = {
            "pairs": p, "key_bits": 32 + tb, "rc": rc,
            "cub_ms": cub_ms, "cub_keys_per_s": p / (cub_ms * 1e-3) if cub_ms > 0 else None,
            "ours_sort_ms": float(ours[2]), "ours_keys_per_s": p / (float(ours[2]) * 1e-3) if ours[2] > 0 else None,
            "ours_sort_plus_pair_gen_ms": float(ours[1] + ours[2]),
            "cub_output_equals_ours": same,
        }
        del kd, gd, order, kin, vin, kout, vout
    # the last frame on the context is the configured one again
    r.render_async(scene, view, mode, k, bins, exact=exact)
    r.wait()
    return res


# ------------------------------------------------- C++ drop-in call (span)
def cxx_span_e2e(cfg: str, mode: str, k: float, bins, iters: int = 5) -> dict:
    """ags::render(std::span<const Gaussian3D>, cam, cfg, lut) -- the reference's
    C++ signature (rasterizer.hpp:63-65) -- on the AoS synthetic scene, through
    libags.so's ags_bench_render_span: host clock per call, with the
    span-identity device-scene cache (the default) and without it (every call
    packs and uploads the scene, like a reference caller that changes scenes)."""
    so = os.path.join(ROOT, "paper_2604_18980_b200", "lib", "libags.so")
    lib = ctypes.CDLL(so)
    f = lib.ags_bench_render_span
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                  ctypes.c_float, ctypes.c_int, ctypes.c_float, ctypes.POINTER(ctypes.c_float), ctypes.c_int,
                  ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                  ctypes.POINTER(ctypes.c_uint64)]
    n, w, h, cams = CONFIGS[cfg]
    mode_id = {"aabb": 0, "obb": 1, "ellipse": 2, "adagscale": 3}.get(mode, 2)
    lb = (ctypes.c_float * max(len(bins), 1))(*bins) if bins else None
    out = {}
    for label, cache, it in (("cached", 1, iters), ("uncached", 0, 2)):
        per, first, pairs = ctypes.c_double(), ctypes.c_double(), ctypes.c_uint64()
        rc = f(1, n, b"veil", cams, w, h, 500.0 * w / 640.0, mode_id, k, lb, len(bins), it, cache, ctypes.byref(per),
               ctypes.byref(first), ctypes.byref(pairs))
        if rc != 0:
            return {"unavailable": f"ags_bench_render_span rc={rc}"}
        out[label] = {"value": 1.0 / per.value, "unit": "frames/s", "s_per_call": per.value,
                      "first_call_s": first.value, "calls": it, "pair_count": int(pairs.value)}
    out["api"] = ("ags::render(std::span<const Gaussian3D>, ...) -> RenderReport with a std::vector<float> image "
                  "(pageable host memory); cached = span-identity device-scene cache, uncached = AoS pack + "
                  "upload of the scene in every call")
    out["d2h_bytes_per_step"] = w * h * 12
    return out


# ------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    os.environ["AGS_DEVICE"] = str(local_rank)  # device of the module-level render()
    import torch
    import paper_2604_18980_b200 as P

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1 or "TORCHELASTIC_RUN_ID" in os.environ:  # under torchrun (any N): NCCL process group
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    mode = args.mode
    n, w, h, cams = CONFIGS[args.config]
    focal = 500.0 * w / 640.0
    k = scaled_k(w) if mode == "adagscale" else 0.0
    bins = LUT_BINS if mode == "adagscale" else []
    scene = P.synth_scene(1, n, "veil", cameras=cams, width=w, height=h, focal=focal)
    from paper_2604_18980_b200.multiview import partition_views, stereo_cameras

    # Work per rank: configs 1-3 -> rank r renders view r of the
    # camera set (weak scaling); config 4 -> stereo, eye r % 2 of view 0;
    # config 5 -> the 64-view camera path split into contiguous blocks
    # (strong scaling: the whole path per step, frames / step fixed).
    if args.config == "5":
        jobs = [(v, None) for v in partition_views(cams, world, rank)]
        frames_per_step_total = cams
    elif args.config == "4":
        eyes = stereo_cameras(scene.camera(0))
        jobs = [(0, eyes[rank % 2])]
        frames_per_step_total = world
    else:
        jobs = [(rank % scene.camera_count, None)]
        frames_per_step_total = world
    view = jobs[0][0] if jobs else 0
    r = P.Renderer(local_rank)
    r.upload(scene)
    stream = torch.cuda.ExternalStream(r.stream, device=torch.device("cuda", local_rank))

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def step():
        for v, cam in jobs:
            r.render_async(scene, v, mode, k, bins, exact=args.exact, camera=cam)

    # warm-up: one waited frame per view sizes the pair arena (an async chain
    # cannot re-run a frame that overflowed it; wait() would raise)
    for v, cam in jobs:
        r.render_async(scene, v, mode, k, bins, exact=args.exact, camera=cam)
        r.wait()
    for _ in range(max(args.warmup, 3)):
        step()
    r.wait()
    stats = r.frame_stats()
    launches0 = r.kernel_launches

    # timed region: K steps back to back on the renderer's stream
    sampler = ClockSampler(local_rank)
    sampler.start()
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    r.wait()
    barrier()
    clocks = sampler.stop()
    elapsed_ms = ev0.elapsed_time(ev1)
    launches = r.kernel_launches - launches0
    hist = r.stage_history(min(args.steps * max(len(jobs), 1), 64))
    stats = r.frame_stats()

    t = torch.tensor([elapsed_ms], dtype=torch.float64, device="cuda")
    frames = torch.tensor([args.steps * len(jobs)], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(frames, op=dist.ReduceOp.SUM)
    max_ms = float(t.item())
    total_frames = float(frames.item())
    fps = total_frames / (max_ms * 1e-3)

    # ---- two frames in flight (second context + stream), same frames --------
    inflight = None
    if not args.no_inflight:
        r2 = P.Renderer(local_rank)
        rs = [r, r2]
        for rr in rs:
            for v, cam in jobs:
                rr.render_async(scene, v, mode, k, bins, exact=args.exact, camera=cam)
                rr.wait()
        barrier()
        steps_i = max(4, min(args.steps, 100))
        t0 = time.perf_counter()
        for i in range(steps_i):
            for v, cam in jobs:
                rs[i % 2].render_async(scene, v, mode, k, bins, exact=args.exact, camera=cam)
        for rr in rs:
            rr.wait()
        barrier()
        ti = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
        if dist is not None:
            dist.all_reduce(ti, op=dist.ReduceOp.MAX)
        inflight = {"value": total_frames / args.steps * steps_i / float(ti.item()), "unit": "frames/s",
                    "how": "frames alternate between two renderer contexts (two streams, scene shared), so one "
                           "frame's sort overlaps the other's raster; host wall clock over the loop, max over ranks"}
        del r2

    # ---- frames gathered on rank 0 (NCCL over NVLink), N > 1 -----------------
    # Through multiview.MultiViewRenderer.render_path, the code the gloo
    # world-2 test runs (tests/test_multiview.py): each rank renders its block
    # of views into frame slots (on rank 0 its slice of the preallocated path
    # buffer), the other blocks arrive by point-to-point NCCL transfers in place.
    gather = None
    if dist is not None and not args.no_gather:
        from paper_2604_18980_b200.multiview import MultiViewRenderer, gpu_render_pipelined

        rg = P.Renderer(local_rank)
        mv = MultiViewRenderer(batch=gpu_render_pipelined([r, rg]), device=f"cuda:{local_rank}")
        n_views = cams if args.config == "5" else world
        kwg = dict(mode=mode, k=k, lut_bins=bins, exact=args.exact)
        if args.config == "4":
            kwg["camera"] = eyes[rank % 2]
        path = torch.empty((n_views, h, w, 3), dtype=torch.float32, device="cuda") if rank == 0 else None
        mv.render_path(scene, n_views, h, w, dst=0, out=path, **kwg)  # warm-up
        steps_g = max(2, min(args.steps, 10))
        barrier()
        t0 = time.perf_counter()
        for _ in range(steps_g):
            frames_g, stats_g = mv.render_path(scene, n_views, h, w, dst=0, out=path, **kwg)
        barrier()
        tg = torch.tensor([(time.perf_counter() - t0) / steps_g], dtype=torch.float64, device="cuda")
        dist.all_reduce(tg, op=dist.ReduceOp.MAX)
        gms = float(tg.item()) * 1e3
        gather = {"fps_with_gather": n_views / (gms * 1e-3), "ms_per_step_render_plus_gather": gms,
                  "ms_per_step_render": max_ms / args.steps, "views_per_step": n_views,
                  "pairs_per_step": stats_g.pair_count,
                  "bytes_to_rank0_per_step": int((n_views - len(partition_views(n_views, world, 0))) * h * w * 12),
                  "how": "multiview.MultiViewRenderer.render_path over two contexts per rank: frames rasterised "
                         "into slots (rank 0: its slice of the path buffer), point-to-point NCCL sends into "
                         "rank 0's path buffer, stats all-reduced; host clock between device-synchronised "
                         "barriers, max over ranks"}
        del rg

    # ---- end to end through the public API (host image out, per step) ----
    e2e = None
    if not args.no_e2e:
        # >= 3 warm-up calls: the pinned image pool holds two blocks in steady
        # state (the previous frame's image is alive while the next renders)
        for _ in range(3):
            out = P.render(scene, view, mode, k, bins, exact=args.exact)
        barrier()
        steps_e2e = max(3, min(args.steps, 10))
        t0 = time.perf_counter()
        for _ in range(steps_e2e):
            out = P.render(scene, view, mode, k, bins, exact=args.exact)
        barrier()
        e2e_s = (time.perf_counter() - t0) / steps_e2e
        tt = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        if dist is not None:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        from paper_2604_18980_b200 import capi

        h2d = ctypes.sizeof(capi.Camera) + ctypes.sizeof(capi.Config) + 4 * len(bins)
        e2e = {"value": world / float(tt.item()), "unit": "frames/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": int(out["image"].nbytes) + 128,
               "api": "paper_2604_18980_b200.render(scene, view, ...) -> host numpy float32 image "
                      "(scene resident; the rasterizer streams the frame into a pinned host buffer)"}
        # row f3: the same call with the frame quantised to PPM bytes on the device
        for _ in range(3):
            out8 = P.render(scene, view, mode, k, bins, exact=args.exact, image_u8=True)
        barrier()
        t0 = time.perf_counter()
        for _ in range(steps_e2e):
            out8 = P.render(scene, view, mode, k, bins, exact=args.exact, image_u8=True)
        barrier()
        t8 = torch.tensor([(time.perf_counter() - t0) / steps_e2e], dtype=torch.float64, device="cuda")
        if dist is not None:
            dist.all_reduce(t8, op=dist.ReduceOp.MAX)
        e2e["u8_egress"] = {"value": world / float(t8.item()), "unit": "frames/s",
                            "d2h_bytes_per_step": int(out8["image"].nbytes) + 128,
                            "api": "render(..., image_u8=True) -> host uint8 PPM pixels (write_image quantisation "
                                   "on the GPU)"}

        # a camera path through batch.render_views: one frame in flight per
        # context (three contexts), so each frame's PCIe egress overlaps the
        # next frame's kernels; per frame the same H2D / D2H as above
        from paper_2604_18980_b200.batch import render_views

        prs = [P.Renderer(local_rank) for _ in range(3)]
        kw = dict(mode=mode, k=k, lut_bins=bins, exact=args.exact)
        render_views(prs, scene, [view] * 4, on_frame=lambda i, o: None, **kw)
        barrier()
        n_path = max(6, 2 * steps_e2e)
        t0 = time.perf_counter()
        render_views(prs, scene, [view] * n_path, on_frame=lambda i, o: None, **kw)
        barrier()
        tp = torch.tensor([(time.perf_counter() - t0) / n_path], dtype=torch.float64, device="cuda")
        if dist is not None:
            dist.all_reduce(tp, op=dist.ReduceOp.MAX)
        e2e["camera_path"] = {"value": world / float(tp.item()), "unit": "frames/s", "frames": n_path,
                              "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": int(out["image"].nbytes) + 128,
                              "api": "batch.render_views(renderers, scene, views) -> host float32 image per view "
                                     "(three contexts, one frame in flight each)"}
        render_views(prs, scene, [view] * 4, on_frame=lambda i, o: None, image_u8=True, **kw)
        barrier()
        t0 = time.perf_counter()
        render_views(prs, scene, [view] * n_path, on_frame=lambda i, o: None, image_u8=True, **kw)
        barrier()
        tp8 = torch.tensor([(time.perf_counter() - t0) / n_path], dtype=torch.float64, device="cuda")
        if dist is not None:
            dist.all_reduce(tp8, op=dist.ReduceOp.MAX)
        e2e["camera_path"]["u8_egress"] = {"value": world / float(tp8.item()), "unit": "frames/s",
                                           "d2h_bytes_per_step": int(out8["image"].nbytes) + 128,
                                           "api": "batch.render_views(..., image_u8=True)"}
        del prs
        if world == 1:
            e2e["cxx_span"] = cxx_span_e2e(args.config, mode, k, bins)

    # ---- AdaGScale off, same scene (pairs + FPS) --------------------------
    off = None
    if mode == "adagscale" and not args.no_off:
        for _ in range(3):
            r.render_async(scene, view, "ellipse", 0.0, [], exact=args.exact)
            r.wait()  # the first one sizes the pair arena for the off-mode chain
        steps_off = max(3, min(args.steps, 20))
        barrier()
        ev0.record(stream)
        for _ in range(steps_off):
            r.render_async(scene, view, "ellipse", 0.0, [], exact=args.exact)
        ev1.record(stream)
        r.wait()
        barrier()
        off_stats = r.frame_stats()
        off = {"fps_per_gpu": steps_off / (ev0.elapsed_time(ev1) * 1e-3), "pair_count": off_stats["pair_count"],
               "splat_count": off_stats["splat_count"]}
        # restore the on-frame state for the image comparison below
        r.render_async(scene, view, mode, k, bins, exact=args.exact)
        r.wait()

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- per-stage roofline from the live stage events --------------------
    peaks = measured_peaks()
    stage_ms = hist.mean(axis=0) if len(hist) else np.zeros(4)
    tiles = stats["tiles"]
    bucketed = bool(stats.get("bucketed_sort", 0))
    sb = moved_bytes(n, stats["splats_with_tiles"], stats["pair_count"], stats["p_it"], tiles, w * h,
                     stats.get("depth_passes", 3), bucketed)
    svb = survey_bytes(n, stats["splat_count"], stats["pair_count"], stats["p_it"], tiles, w * h)
    names = ("preprocess", "pair_gen", "sort", "raster")
    stages = {}
    for i, nm in enumerate(names):
        gbs = sb[nm] / (stage_ms[i] * 1e-3) / 1e9 if stage_ms[i] > 0 else 0.0
        sgbs = svb[nm] / (stage_ms[i] * 1e-3) / 1e9 if stage_ms[i] > 0 else 0.0
        stages[nm] = {"ms": float(stage_ms[i]), "algorithmic_bytes": int(sb[nm]), "achieved_gbs": gbs,
                      "frac_hbm": gbs / peaks["hbm_gbs"], "frac_hbm_spec": gbs / HBM_SPEC_GBS,
                      "survey_formula": {"bytes": int(svb[nm]), "achieved_gbs": sgbs,
                                         "note": "SURVEY §8(d) bytes of the reference's formulation; not moved "
                                                 "by these kernels"}}
    stages["sort"]["keys_per_s"] = stats["pair_count"] / (stage_ms[2] * 1e-3) if stage_ms[2] else 0.0
    stages["pair_gen"]["pairs_per_s"] = stats["pair_count"] / (stage_ms[1] * 1e-3) if stage_ms[1] else 0.0
    bytes_def = ("moved bytes of this formulation (bench.moved_bytes: "
                 + ("tile-bucketed sort" if bucketed else
                    f"depth sort of the splats in {stats.get('depth_passes', 3)} passes + 2 tile passes") + ")")
    dom = int(np.argmax(stage_ms))
    # ncu evidence of this workload (profiles/ncu_frame_c<config>_<mode>.json,
    # one --set full capture of the same frame by scripts/profile_summary.py):
    # DRAM bytes and warp instructions per frame per stage; absent -> null
    prof_path = os.path.join(ROOT, "profiles", f"ncu_frame_c{args.config}_{mode}.json")
    prof = {}
    try:
        with open(prof_path) as f:
            pdoc = json.load(f)
        if pdoc.get("sort_path", "depth") == ("bucket" if bucketed else "depth"):
            prof = pdoc["per_frame"]
    except Exception:
        prof = {}
    for nm in names:
        stages[nm]["ncu_dram_bytes"] = prof[nm]["dram_bytes"] if nm in prof else None
    props = torch.cuda.get_device_properties(local_rank)
    sm_mhz = clocks.get("sm_mhz") or 1965.0
    issue_peak = props.multi_processor_count * 4 * sm_mhz * 1e6  # warp-instructions / s
    # instruction-issue roofline of every stage (warp-instructions per frame from
    # the ncu capture over the live stage time): the raster and K1 are issue-bound,
    # the sort passes latency-bound (low on both rooflines)
    for si, nm in enumerate(names):
        if nm in prof and stage_ms[si] > 0 and prof[nm].get("warp_inst"):
            ach = prof[nm]["warp_inst"] / (stage_ms[si] * 1e-3)
            stages[nm]["issue_roofline"] = {
                "bound": "issue", "achieved": ach, "peak": issue_peak, "unit": "warp-inst/s", "frac": ach / issue_peak,
                "warp_inst_per_frame": prof[nm]["warp_inst"],
                "peak_def": f"{props.multi_processor_count} SMs x 4 SMSPs x 1 warp-inst/clk x {sm_mhz:.0f} MHz"}
    if not args.no_cub:
        stages["sort"]["cub"] = cub_comparator(r, scene, view, mode, k, bins, args.exact)
        if "adagscale_on" in stages["sort"]["cub"] or "adagscale_off" in stages["sort"]["cub"]:
            c0 = stages["sort"]["cub"].get("adagscale_on") or stages["sort"]["cub"].get("adagscale_off")
            stages["sort"]["cub_keys_per_s"] = c0["cub_keys_per_s"]
    roofline = {
        "bound": "hbm",
        "kernel": names[dom],
        "achieved": stages[names[dom]]["achieved_gbs"],
        "peak": peaks["hbm_gbs"],
        "unit": "GB/s",
        "frac": stages[names[dom]]["frac_hbm"],
        "frac_spec_8tbs": stages[names[dom]]["frac_hbm_spec"],
        "traffic": prof.get(names[dom], {}).get("dram_bytes"),
        "traffic_src": (os.path.relpath(prof_path, ROOT) + " (dram__bytes_read.sum + dram__bytes_write.sum, one "
                        "ncu --set full capture of this workload)") if names[dom] in prof else None,
        "peak_src": peaks["src"],
        "algorithmic_bytes_per_launch": stages[names[dom]]["algorithmic_bytes"],
        "bytes_def": bytes_def,
        "note": "raster is issue-bound (SURVEY §8(d)); HBM fraction reported as asked, issue roofline in "
                "stages.raster.issue_roofline",
    }

    # ---- CPU baseline (reference render on host cores) + PSNR vs CPU ref ---
    cpu = None
    quality = None
    if not args.no_cpu and world == 1:
        # median of >= 5 repeats (the reference's cmd_bench convention,
        # adagscale_main.cpp:343,364-367), stage_times summed per frame
        kind, threads, times, ref_out = cpu_reference(args.config, mode, max(args.cpu_frames, 5), 1)
        cpu_fps = 1.0 / statistics.median(times) if times and times[0] is not None else None
        cpu = {"value": cpu_fps, "unit": "frames/s", "cores": threads, "kind": kind,
               "sample": f"median of {len(times)} full frames of the same workload (view 0) after 1 warm-up, "
                         f"reference render() stage_times summed, {threads} threads",
               "frame_s": times}
        img = P.render(scene, 0, mode, k, bins, exact=args.exact)["image"]
        ref_img = ref_out["image"]
        d = img.astype(np.float64) - ref_img.astype(np.float64)
        mse = float(np.mean(d * d))
        quality = {"psnr_vs_cpu_ref_db": (float("inf") if mse == 0 else 10 * np.log10(1 / mse)),
                   "max_abs_vs_cpu_ref": float(np.max(np.abs(d))),
                   "bit_exact_image": bool(mse == 0),
                   "pair_count_equal": ref_out["pair_count"] == stats["pair_count"],
                   "splat_count_equal": ref_out["splat_count"] == stats["splat_count"]}

    line = {
        "metric": METRIC,
        "value": fps,
        "unit": "frames/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": max_ms / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if args.config == "5" else "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (veil layout, seed 1, host synth_scene byte-identical to the reference)",
        "config": {
            "workload": workload_name(args.config, mode),
            "gaussians": n, "width": w, "height": h, "mode": mode,
            "views": ("64-view camera path, contiguous blocks per rank" if args.config == "5" else
                      "stereo: eye r % 2 of view 0 on rank r" if args.config == "4" else "rank r renders view r"),
            "parallelism": f"view-partitioned replicas x{world}",
            "l2": "inputs larger than L2 (scene 168 MB + image 191 MB per frame)",
            "alpha": "exact glibc expf" if args.exact else "MUFU.EX2 + exact guard band",
        },
        "pairs_per_frame": stats["pair_count"],
        "splats_per_frame": stats["splat_count"],
        "p_it": stats["p_it"],
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks,
        "roofline": roofline,
        "stages": stages,
        "cpu_baseline": cpu,
        "quality": quality,
        "adagscale_off": off,
        "gather": gather,
        "two_in_flight": inflight,
    }
    print(json.dumps(line, default=_jsonable), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="3", choices=sorted(CONFIGS))
    ap.add_argument("--mode", default="adagscale", choices=["adagscale", "ellipse", "aabb", "obb", "aabb_fixed3"])
    ap.add_argument("--exact", action="store_true", help="glibc-exact alpha (bit-identical images)")
    ap.add_argument("--cpu-frames", type=int, default=5)
    ap.add_argument("--no-cub", action="store_true", help="skip the cub::DeviceRadixSort comparator")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-off", action="store_true")
    ap.add_argument("--no-gather", action="store_true")
    ap.add_argument("--no-inflight", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank)
        return
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()

"""View-partitioned multi-GPU rendering.

The render path shards by viewpoint: every frame is independent and the scene is
read-only (``render`` takes ``std::span<const Gaussian3D>``, rasterizer.hpp:63).  So
each rank (one process per GPU) holds a replica of the scene, renders its own block
of views with no collective on the data path, and only finished frames and
per-frame stats cross GPUs.  The frames go to a destination rank via
``torch.distributed`` (NCCL over NVLink on B200, gloo in the CPU tests), and the
stats go through an all-reduce (sums of pair and splat counts, max of stage times).

Partitioning follows §8(e):
* config 5 is a camera path split into contiguous blocks of views per rank;
* config 4 is stereo, with the left eye on rank 0 and the right eye on rank 1.

The rasteriser writes each frame straight into a slot of a frame tensor
(``Renderer.render_async_to``): on the destination rank that slot is already its
place in the gathered camera path, and the other ranks' blocks are received
in place by point-to-point transfers (no padding, no concatenation copy).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np


def partition_views(n_views: int, world: int, rank: int) -> list[int]:
    """Contiguous block of the camera path owned by `rank`.

    The first ``n_views % world`` ranks hold one extra view."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank must be in [0, world)")
    if n_views < 0:
        raise ValueError("n_views must be >= 0")
    base, extra = divmod(n_views, world)
    start = rank * base + min(rank, extra)
    count = base + (1 if rank < extra else 0)
    return list(range(start, start + count))


def stereo_cameras(cam: dict, baseline: float = 0.064) -> tuple[dict, dict]:
    """Left and right eye of a camera.

    The right eye is the left eye moved by ``baseline`` along the camera's right
    vector. That vector is row 0 of the world-to-camera rotation (look_at,
    synth.cpp:25-34). The arithmetic is float32, like the reference's Vec3f."""
    pos = np.asarray(cam["position"], np.float32)
    right = np.asarray(cam["rotation"], np.float32)[:3]
    right_pos = (pos + np.float32(baseline) * right).astype(np.float32)
    left = dict(cam)
    rcam = dict(cam)
    rcam["position"] = [float(v) for v in right_pos]
    return left, rcam


@dataclass
class PathStats:
    """Frame statistics reduced over ranks."""

    frames: int = 0
    pair_count: int = 0  # summed over frames and ranks
    splat_count: int = 0
    stage_ms_max: list = field(default_factory=lambda: [0.0, 0.0, 0.0, 0.0])  # max over frames and ranks
    per_view_pairs: dict = field(default_factory=dict)  # view -> pair count (this rank)


RenderInto = Callable[[object, int, object, dict], dict]
"""render_into(scene, view, frame_slot, kwargs) -> {"pair_count", "splat_count", "stage_ms"}"""


def _order_after_torch(renderer):
    """Make the renderer's stream wait for torch's current stream, so frame slots
    handed out by the caching allocator are not still in use by queued torch work
    when the rasteriser writes them."""
    import torch

    torch.cuda.ExternalStream(renderer.stream).wait_stream(torch.cuda.current_stream())


def gpu_render_into(renderer) -> RenderInto:
    """A `RenderInto` over the CUDA path: the rasteriser writes the slot in place."""

    def fn(scene, view, slot, kw):
        cam = kw.get("camera")
        _order_after_torch(renderer)
        renderer.render_async_to(scene, view, slot.data_ptr(), mode=kw.get("mode", "ellipse"), k=kw.get("k", 0.0),
                                 lut_bins=kw.get("lut_bins", []), exact=kw.get("exact", False), camera=cam)
        return renderer.wait()

    return fn


def gpu_render_pipelined(renderers):
    """A batch renderer over several contexts of one device: consecutive views
    alternate between the contexts (two streams), so one view's sort overlaps
    the previous view's raster. Returns ``fn(scene, views, frames, kw) ->
    [stats per view]``."""

    def fn(scene, views, frames, kw):
        out = [None] * len(views)
        pending = {}  # renderer index -> view slot in flight
        for r in renderers:
            _order_after_torch(r)
        for i, v in enumerate(views):
            ri = i % len(renderers)
            r = renderers[ri]
            if ri in pending:
                out[pending.pop(ri)] = r.wait()
            r.render_async_to(scene, v, frames[i].data_ptr(), mode=kw.get("mode", "ellipse"), k=kw.get("k", 0.0),
                              lut_bins=kw.get("lut_bins", []), exact=kw.get("exact", False), camera=kw.get("camera"))
            pending[ri] = i
        for ri, i in pending.items():
            out[i] = renderers[ri].wait()
        return out

    return fn


class MultiViewRenderer:
    """Renders the views of a camera path owned by this rank and gathers them.

    ``render_into`` renders one view into a preallocated frame slot. It defaults
    to the CUDA renderer of this rank's device. The CPU tests inject the oracle
    here, so the gloo test exercises the partition and gather logic without a GPU.
    """

    def __init__(self, render_into: RenderInto = None, device="cuda", batch=None):
        """Either ``render_into`` (one view at a time) or ``batch`` (a
        `gpu_render_pipelined` function over several contexts)."""
        if (render_into is None) == (batch is None):
            raise ValueError("give exactly one of render_into / batch")
        self.render_into = render_into
        self.batch = batch
        self.device = device

    def render_local(self, scene, views: Sequence[int], height: int, width: int, out=None, **kw):
        """Render `views` into ``out`` (a ``[len(views), H, W, 3]`` float32 tensor,
        allocated when None); returns ``(frames, stats)`` of this rank."""
        import torch

        frames = out
        if frames is None:
            frames = torch.empty((max(len(views), 1), height, width, 3), dtype=torch.float32, device=self.device)
        stats = PathStats()
        per_view = (self.batch(scene, list(views), frames, kw) if self.batch is not None else
                    [self.render_into(scene, v, frames[i], kw) for i, v in enumerate(views)])
        for v, st in zip(views, per_view):
            stats.frames += 1
            stats.pair_count += int(st["pair_count"])
            stats.splat_count += int(st["splat_count"])
            stats.stage_ms_max = [max(a, float(b)) for a, b in zip(stats.stage_ms_max, st["stage_ms"])]
            stats.per_view_pairs[v] = int(st["pair_count"])
        return frames[: len(views)], stats

    def render_path(self, scene, n_views: int, height: int, width: int, group=None, dst: int = 0,
                    gather: bool = True, out=None, **kw):
        """Render views [0, n_views) across the group; frames gathered on `dst`.

        ``out`` (optional, on `dst`): a preallocated ``[n_views, H, W, 3]``
        float32 tensor for the gathered path.  `dst` renders its own block
        straight into its slice of it and receives every other block in place.

        Returns ``(frames, stats)``:
        * ``frames`` is the ``[n_views, H, W, 3]`` tensor on `dst` (on its
          device), this rank's block when ``gather`` is False, or None on the
          other ranks;
        * ``stats`` is a `PathStats` reduced over all ranks.
        """
        import torch
        import torch.distributed as dist

        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        views = partition_views(n_views, world, rank)
        whole = None
        if gather and rank == dst:
            whole = out
            if whole is None:
                whole = torch.empty((n_views, height, width, 3), dtype=torch.float32, device=self.device)
            elif tuple(whole.shape) != (n_views, height, width, 3) or whole.dtype != torch.float32:
                raise ValueError("out must be a float32 [n_views, H, W, 3] tensor")
        slot = whole[views[0]: views[0] + len(views)] if (whole is not None and views) else None
        local, stats = self.render_local(scene, views, height, width, out=slot, **kw)
        frames = whole if whole is not None else (local if not gather else None)
        if world > 1:
            if gather:
                gather_frames(local, n_views, world, rank, group, dst, out=whole)
            red = torch.tensor([stats.frames, stats.pair_count, stats.splat_count], dtype=torch.float64,
                               device=self.device)
            mx = torch.tensor(stats.stage_ms_max, dtype=torch.float64, device=self.device)
            dist.all_reduce(red, group=group)
            dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
            stats.frames, stats.pair_count, stats.splat_count = (int(x) for x in red.tolist())
            stats.stage_ms_max = mx.tolist()
        return frames, stats


def gather_frames(local, n_views: int, world: int, rank: int, group=None, dst: int = 0, out=None):
    """Gather every rank's block of frames onto `dst` in camera-path order.

    Point-to-point: each rank sends its block (exact size, `partition_views`)
    and `dst` receives it straight into its slice of ``out`` (a ``[n_views,
    H, W, 3]`` tensor; allocated when None).  `dst`'s own block is copied
    only when it is not already that slice.  Returns ``out`` on `dst`, None
    elsewhere."""
    import torch
    import torch.distributed as dist

    blocks = [partition_views(n_views, world, r) for r in range(world)]
    if rank != dst:
        if blocks[rank]:
            dist.send(local[: len(blocks[rank])].contiguous(), dst=_global_rank(group, dst), group=group)
        return None
    h, w = local.shape[1], local.shape[2]
    if out is None:
        out = torch.empty((n_views, h, w, 3), dtype=local.dtype, device=local.device)
    mine = blocks[rank]
    if mine and out[mine[0]: mine[0] + len(mine)].data_ptr() != local.data_ptr():
        out[mine[0]: mine[0] + len(mine)].copy_(local[: len(mine)])
    ops = [dist.P2POp(dist.irecv, out[b[0]: b[0] + len(b)], _global_rank(group, r), group)
           for r, b in enumerate(blocks) if r != rank and b]
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return out


def _global_rank(group, r: int) -> int:
    import torch.distributed as dist

    return r if group is None else dist.get_global_rank(group, r)

"""Batch drivers over the view partition (next row f4).

`pair_report` runs the paper's Table IV methodology: pair counts and PSNR drops of
several tile-test modes against lossless Ellipse renders (analysis.cpp:259-312,
CSV format analysis.cpp:346-371). It runs across the GPUs of a
`torch.distributed` group. Each rank takes a contiguous block of the views
(`multiview.partition_views`) and runs the device report on its block (glibc-exact
frames, references in HBM). The per-rank rows are then merged: pair counts and
stage times are summed, and the per-view means are re-weighted by view counts.
"""
from __future__ import annotations

from typing import Callable, Sequence

from .multiview import partition_views

LocalReport = Callable[[Sequence[int]], list]
"""local_report(views) -> rows (dicts of Renderer.pair_report) over those views."""

_SUM_KEYS = ("pair_count", "t_preprocess", "t_pair_gen", "t_sort", "t_raster")
_MEAN_KEYS = ("reduction_pct", "psnr_drop_db")


def merge_rows(parts: Sequence[list]) -> list:
    """Merge per-rank report rows (same spec order) into whole-path rows."""
    parts = [p for p in parts if p]
    if not parts:
        return []
    out = []
    for i, first in enumerate(parts[0]):
        views = sum(p[i]["views"] for p in parts)
        row = {"mode": first["mode"], "k": first["k"], "views": views}
        for key in _SUM_KEYS:
            row[key] = sum(p[i][key] for p in parts)
        for key in _MEAN_KEYS:
            row[key] = sum(p[i][key] * p[i]["views"] for p in parts) / views if views else 0.0
        out.append(row)
    return out


def pair_report(local_report: LocalReport, n_views: int, group=None) -> list:
    """The whole path's report: views [0, n_views) split over the group's ranks.

    Every rank returns the merged rows. ``local_report`` is usually
    ``lambda views: renderer.pair_report(scene, specs, views=list(views), ...)``.
    """
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    views = partition_views(n_views, world, rank)
    mine = local_report(views) if views else []
    if world == 1:
        return merge_rows([mine])
    parts = [None] * world
    dist.all_gather_object(parts, mine, group=group)
    return merge_rows(parts)


def render_views(renderers, scene, views: Sequence[int], on_frame=None, **kw) -> list:
    """Render `views` of `scene` to host images, one frame in flight per renderer.

    This is the camera-path loop of the reference CLI (``ags::render`` per view,
    adagscale_main.cpp:224-226), pipelined. Each frame is rasterised into a
    page-locked host image by banded copies behind the raster
    (``Renderer.render_async_host``). Consecutive views alternate between the
    renderers (contexts with their own stream and buffers on one device). So one
    frame's PCIe egress overlaps the next frame's preprocess, sort and raster.

    ``kw`` takes the keyword arguments of ``Renderer.render_async_host``
    (mode, k, lut_bins, ...). Returns one dict per view in path order, as
    ``render()`` returns them: image, pair_count, splat_count, stage_ms.
    ``on_frame(i, out)``, if given, is called as each frame completes, in path
    order; it replaces keeping the result, which bounds host memory on long paths.
    """
    if not renderers:
        raise ValueError("need at least one renderer")
    out = [None] * len(views)
    pending = {}  # renderer index -> position of its frame in flight
    nxt = 0  # next position to hand to on_frame

    def done(ri):
        nonlocal nxt
        i = pending.pop(ri)
        out[i] = renderers[ri].wait()
        while nxt < len(out) and out[nxt] is not None:
            if on_frame is not None:
                on_frame(nxt, out[nxt])
                out[nxt] = True  # delivered
            nxt += 1

    for i, v in enumerate(views):
        ri = i % len(renderers)
        if ri in pending:
            done(ri)
        renderers[ri].render_async_host(scene, v, **kw)
        pending[ri] = i
    for ri in sorted(pending, key=pending.get):
        done(ri)
    return out if on_frame is None else []

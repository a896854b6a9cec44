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


def merge_folds(folds: Sequence[dict]) -> dict:
    """Merge build_lut folds of view blocks (``Renderer.fold_max_t``) into the
    LUT of all the views: per bin the max of max_t over the blocks, 1.0 where
    no block saw a blended splat (calibrate.cpp:14-41). Max is associative,
    so the result equals the single-process LUT bit for bit."""
    folds = [f for f in folds if f]
    if not folds:
        raise ValueError("no folds to merge")
    nb = len(folds[0]["folded"])
    bins = []
    for b in range(nb):
        seen = [f["folded"][b] for f in folds if f["observed"][b]]
        bins.append(max(seen) if seen else 1.0)
    return {"lut_bins": bins, "lut_depth_min": folds[0]["depth_min"], "lut_depth_max": folds[0]["depth_max"]}


def pair_report(local_report: LocalReport, n_views: int, group=None, fold=None) -> list:
    """The whole path's report: views [0, n_views) split over the group's ranks.

    Every rank returns the merged rows. ``local_report`` is usually
    ``lambda views, **lut: renderer.pair_report(scene, specs, views=list(views), **lut)``.

    AdaGScale rows need one T-upper LUT built from ALL the views, as the
    reference builds it (analysis.cpp:265-275). A rank's own block would give
    another LUT, so rows that depend on the world size. With
    ``fold(views) -> dict`` (``Renderer.fold_max_t``), every rank folds its own
    block, the folds are all-gathered and merged (``merge_folds``), and
    ``local_report(views, lut_bins=..., lut_depth_min=..., lut_depth_max=...)``
    receives the merged LUT. Without ``fold``, ``local_report(views)`` is
    called as is: pass a LUT yourself, or use ``device_pair_report``.
    """
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    views = partition_views(n_views, world, rank)
    lut = None
    if fold is not None:
        mine_fold = fold(views) if views else None
        if world == 1:
            lut = merge_folds([mine_fold])
        else:
            folds = [None] * world
            dist.all_gather_object(folds, mine_fold, group=group)
            lut = merge_folds(folds)
    if not views:
        mine = []
    elif lut is not None:
        mine = local_report(views, **lut)
    else:
        mine = local_report(views)
    if world == 1:
        return merge_rows([mine])
    parts = [None] * world
    dist.all_gather_object(parts, mine, group=group)
    return merge_rows(parts)


def device_pair_report(renderer, scene, specs, n_views: int | None = None, group=None, lut_bins=None,
                       lut_depth_min: float = 0.0, lut_depth_max: float = 100.0) -> list:
    """``pair_report`` (analysis.cpp:259-312) of ``scene``'s first ``n_views``
    views on the group's GPUs, one ``Renderer`` per rank. Without ``lut_bins``,
    AdaGScale specs get the LUT built from all the views across the ranks."""
    n = scene.camera_count if n_views is None else n_views
    needs_lut = any(str(s[0]) == "adagscale" for s in specs) and not lut_bins
    fixed = {} if needs_lut or not lut_bins else {
        "lut_bins": list(lut_bins), "lut_depth_min": lut_depth_min, "lut_depth_max": lut_depth_max}

    def local(views, **lut):
        return renderer.pair_report(scene, specs, views=list(views), **(lut or fixed))

    fold = (lambda views: renderer.fold_max_t(scene, list(views))) if needs_lut else None
    return pair_report(local, n, group=group, fold=fold)


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

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

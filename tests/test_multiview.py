"""CPU tests of the view-partitioned multi-GPU path.

The partition, gather and stats-reduction logic of
`paper_2604_18980_b200.multiview` runs here with world_size 2 over gloo. The
renderer is injected: each rank renders its views with the CPU oracle (test
infrastructure) into CPU frame slots. Rank 0 then checks the gathered camera
path frame by frame against single-process oracle renders. On the GPU the same
driver runs with the CUDA renderer and NCCL (bench.py --gpus N,
tests/test_gpu_parity.py::test_multiview_single_rank_gpu)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_18980_b200.multiview import MultiViewRenderer, partition_views, stereo_cameras


@pytest.mark.parametrize("n,world", [(64, 1), (64, 2), (64, 8), (5, 2), (3, 4), (0, 2), (7, 3)])
def test_partition_views_covers_path_in_order(n, world):
    blocks = [partition_views(n, world, r) for r in range(world)]
    flat = [v for b in blocks for v in b]
    assert flat == list(range(n))
    sizes = [len(b) for b in blocks]
    assert max(sizes) - min(sizes) <= 1


def test_partition_views_rejects_bad_rank():
    with pytest.raises(ValueError):
        partition_views(4, 2, 2)


def test_stereo_right_eye_moves_along_right_vector():
    cam = {"position": [1.0, 2.0, 3.0], "rotation": [0.6, 0.0, -0.8, 0.0, 1.0, 0.0, 0.8, 0.0, 0.6],
           "fx": 100.0, "fy": 100.0, "width": 64, "height": 48}
    left, right = stereo_cameras(cam)
    assert left["position"] == cam["position"]
    d = np.asarray(right["position"], np.float32) - np.asarray(cam["position"], np.float32)
    assert np.allclose(d, 0.064 * np.array([0.6, 0.0, -0.8]), atol=1e-6)
    assert right["rotation"] == cam["rotation"]


SCENE = dict(seed=5, count=600, layout="veil", cameras=5, width=96, height=64, focal=80.0)


def _oracle_render_into():
    from oracle.ffi import Oracle

    port = Oracle("port")
    scene = port.synth_scene(**SCENE)

    def fn(_scene, view, slot, kw):
        out = port.render(scene, scene.cameras[view], port.config(kw.get("mode", "ellipse")))
        slot.copy_(torch.from_numpy(out["image"]))
        return {"pair_count": out["pair_count"], "splat_count": out["splat_count"],
                "stage_ms": [1.0 + view, 0.0, 0.0, 0.0]}

    return port, scene, fn


def _worker(rank, world, port_no, result_q, prealloc=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _, scene, fn = _oracle_render_into()
        mv = MultiViewRenderer(fn, device="cpu")
        out = None
        if prealloc and rank == 0:  # the bench's form: a preallocated path buffer on the destination
            out = torch.full((SCENE["cameras"], SCENE["height"], SCENE["width"], 3), -1.0)
        frames, stats = mv.render_path(scene, SCENE["cameras"], SCENE["height"], SCENE["width"], mode="ellipse",
                                       out=out)
        if out is not None:
            assert frames.data_ptr() == out.data_ptr()  # gathered in place, no concatenation copy
        result_q.put((rank, None if frames is None else frames.numpy(), stats.frames, stats.pair_count,
                      stats.stage_ms_max))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("prealloc", [False, True])
def test_gather_camera_path_world2_gloo(prealloc):
    """render_path over world 2 (5 views: uneven blocks 3 + 2), the code bench.py
    runs for N > 1 (with the CUDA renderer and NCCL there)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port_no, q, prealloc)) for r in range(2)]
    for p in procs:
        p.start()
    results = {}
    for _ in procs:
        rank, frames, n, pairs, stage_max = q.get(timeout=300)
        results[rank] = (frames, n, pairs, stage_max)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    port, scene, _ = _oracle_render_into()
    want = [port.render(scene, scene.cameras[v], port.config("ellipse")) for v in range(SCENE["cameras"])]
    frames0, n0, pairs0, stage0 = results[0]
    assert results[1][0] is None  # only the destination receives frames
    assert frames0.shape == (SCENE["cameras"], SCENE["height"], SCENE["width"], 3)
    for v in range(SCENE["cameras"]):  # camera-path order, bit-exact copies
        assert np.array_equal(frames0[v].view(np.uint32), want[v]["image"].view(np.uint32)), v
    # stats reduced over both ranks: frame and pair counts summed, stage times max
    for r in (0, 1):
        assert results[r][1] == SCENE["cameras"]
        assert results[r][2] == sum(w["pair_count"] for w in want)
        assert results[r][3][0] == 1.0 + (SCENE["cameras"] - 1)


def _report_worker(rank, world, port_no, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_18980_b200.batch import pair_report

        def local(views):  # stand-in device report: deterministic per-view values
            return [{"mode": m, "k": k, "views": len(views), "pair_count": sum(100 * v + i for v in views),
                     "reduction_pct": sum(float(v) for v in views) / len(views),
                     "psnr_drop_db": sum(0.1 * v for v in views) / len(views),
                     "t_preprocess": 0.001 * len(views), "t_pair_gen": 0.0, "t_sort": 0.0, "t_raster": 0.0}
                    for i, (m, k) in enumerate((("ellipse", 0.0), ("adagscale", 0.5)))]

        q.put((rank, pair_report(local, 7)))

        # AdaGScale rows: one LUT over ALL views, whatever the world size
        # (analysis.cpp:265-275): the ranks' build_lut folds are merged by max
        def fold(views):  # stand-in fold: bin b sees view v when (v + b) % 3 == 0
            return {"folded": [max([0.01 * (v + 1) * (b + 1) for v in views if (v + b) % 3 == 0], default=0.0)
                               for b in range(20)],
                    "observed": [any((v + b) % 3 == 0 for v in views) for b in range(20)],
                    "depth_min": 0.0, "depth_max": 100.0}

        def local_lut(views, lut_bins, lut_depth_min, lut_depth_max):
            rows = local(views)
            for r in rows:
                r["pair_count"] = int(1e6 * sum(lut_bins))  # depends on the LUT only
            return rows

        q.put((rank, pair_report(local_lut, 7, fold=fold)))
    finally:
        dist.destroy_process_group()


def test_pair_report_merges_view_blocks_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_report_worker, args=(r, 2, port_no, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(2 * len(procs))]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res = {}
    lut_rows = {}
    for rank, rows in got:
        (lut_rows if rank in res else res)[rank] = rows
    from paper_2604_18980_b200.batch import merge_folds

    whole = merge_folds([{"folded": [max([0.01 * (v + 1) * (b + 1) for v in range(7) if (v + b) % 3 == 0],
                                         default=0.0) for b in range(20)],
                          "observed": [any((v + b) % 3 == 0 for v in range(7)) for b in range(20)],
                          "depth_min": 0.0, "depth_max": 100.0}])
    for rows in lut_rows.values():  # every rank reported with the all-view LUT
        # both ranks' blocks contribute (views 0-3 and 4-6), merged rows sum them
        assert rows[0]["pair_count"] == 2 * int(1e6 * sum(whole["lut_bins"]))
    for rows in res.values():  # same merged rows on both ranks
        assert [r["mode"] for r in rows] == ["ellipse", "adagscale"]
        assert rows[0]["views"] == 7
        assert rows[0]["pair_count"] == sum(100 * v for v in range(7))
        assert rows[1]["pair_count"] == sum(100 * v + 1 for v in range(7))
        assert abs(rows[0]["reduction_pct"] - 3.0) < 1e-12  # mean of 0..6
        assert abs(rows[0]["psnr_drop_db"] - 0.3) < 1e-12

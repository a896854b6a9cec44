"""Scene ingest (next row f2): binary 3DGS PLY -> scene arrays + orbit cameras,
byte-identical to the reference's load_ply_file / orbit_cameras
(gsio.cpp:80-157, synth.cpp:254-281); pinned by the reference build and by a
committed digest (tests/golden/ply_fixture.json)."""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_2604_18980_b200 as P
from plyfixture import write_ply

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "ply_fixture.json")


def digest(arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a, np.float32).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("degree", [0, 1, 3])
def test_load_ply_matches_reference(tmp_path, ref, degree):
    path = str(tmp_path / "s.ply")
    write_ply(path, n=3000, degree=degree, seed=degree + 1)
    s = P.load_ply(path, orbit_views=5, width=320, height=240, focal=250.0, seed=3)
    want, rejected = ref.load_ply(path)
    assert rejected == 2
    a = s.arrays()
    assert s.gaussian_count == want.count and s.sh_coeffs == (degree + 1) ** 2
    for f in ("mean", "scale", "rotation", "opacity", "sh"):
        assert np.array_equal(a[f].reshape(-1).view(np.uint32), getattr(want, f).reshape(-1).view(np.uint32)), f
    cams = ref.orbit_cameras(path, 5, 320, 240, 250.0, 250.0, 3)
    for i, c in enumerate(cams):
        got = s.camera(i)
        assert np.array_equal(np.float32(got["position"]), np.float32(list(c.position)))
        assert np.array_equal(np.float32(got["rotation"]), np.float32(list(c.rotation)))


def test_load_ply_golden_digest(tmp_path):
    g = json.load(open(GOLDEN))
    path = str(tmp_path / "g.ply")
    write_ply(path, **g["fixture"])
    s = P.load_ply(path, **g["orbit"])
    a = s.arrays()
    assert digest([a[f] for f in ("mean", "scale", "rotation", "opacity", "sh")]) == g["scene_sha256"]
    cams = [s.camera(i) for i in range(s.camera_count)]
    assert digest([np.float32(c["position"] + c["rotation"]) for c in cams]) == g["cameras_sha256"]


def test_load_ply_errors(tmp_path):
    bad = tmp_path / "bad.ply"
    bad.write_bytes(b"ply\nformat ascii 1.0\nend_header\n")
    with pytest.raises(RuntimeError):
        P.load_ply(str(bad))
    with pytest.raises(RuntimeError):
        P.load_ply(str(tmp_path / "missing.ply"))

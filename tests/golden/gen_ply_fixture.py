#!/usr/bin/env python3
"""Digest of the REFERENCE build's load_ply_file + orbit_cameras on the
seeded PLY fixture (tests/plyfixture.py) -> tests/golden/ply_fixture.json."""
import hashlib
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from oracle.ffi import Oracle  # noqa: E402
from plyfixture import write_ply  # noqa: E402

FIXTURE = dict(n=2500, degree=2, seed=11)
ORBIT = dict(orbit_views=4, width=200, height=150, focal=160.0, seed=9)


def digest(arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a, np.float32).tobytes())
    return h.hexdigest()


def main():
    ref = Oracle("reference")
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "g.ply")
        write_ply(path, **FIXTURE)
        s, rej = ref.load_ply(path)
        cams = ref.orbit_cameras(path, ORBIT["orbit_views"], ORBIT["width"], ORBIT["height"], ORBIT["focal"],
                                 ORBIT["focal"], ORBIT["seed"])
    out = {"fixture": FIXTURE, "orbit": ORBIT, "rejected": rej,
           "scene_sha256": digest([s.mean, s.scale, s.rotation, s.opacity, s.sh]),
           "cameras_sha256": digest([np.float32(list(c.position) + list(c.rotation)) for c in cams])}
    json.dump(out, open(os.path.join(HERE, "ply_fixture.json"), "w"), indent=1)
    print(out)


if __name__ == "__main__":
    main()

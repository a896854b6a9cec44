#!/usr/bin/env python3
"""Golden calibration result from the REFERENCE build (oracle/_ref/libags_ref.so):
build_lut + search_k (calibrate.cpp:14-155) on a small seeded scene.

    python tests/golden/gen_calibration.py   ->  tests/golden/calibration_veil3000.json
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.ffi import Oracle  # noqa: E402

SPEC = dict(seed=3, count=3000, layout="veil", cameras=4, width=240, height=160, focal=180.0)
TARGET = 0.5


def main():
    ref = Oracle("reference")
    s = ref.synth_scene(**SPEC)
    out = ref.calibrate(s, TARGET, SPEC["cameras"])
    out.update(spec=SPEC, target_drop=TARGET, calib_views=SPEC["cameras"])
    json.dump(out, open(os.path.join(HERE, "calibration_veil3000.json"), "w"), indent=1)
    print(out)


if __name__ == "__main__":
    main()

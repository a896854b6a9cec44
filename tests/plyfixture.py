"""Independent binary-PLY writer for the ingest tests (the reference's
FixtureWriter, test_gsio.cpp:18-49): 3DGS vertex layout, float properties."""
import numpy as np


def write_ply(path, n=2000, degree=3, seed=7, bad_rows=(5, 17), extra_props=True):
    rng = np.random.default_rng(seed)
    rest = 3 * ((degree + 1) ** 2 - 1)
    names = ["x", "y", "z"] + (["nx", "ny", "nz"] if extra_props else []) + ["f_dc_0", "f_dc_1", "f_dc_2"]
    names += [f"f_rest_{i}" for i in range(rest)] + ["opacity", "scale_0", "scale_1", "scale_2"]
    names += ["rot_0", "rot_1", "rot_2", "rot_3"]
    cols = {}
    cols["x"] = rng.uniform(-3, 3, n)
    cols["y"] = rng.uniform(-2, 2, n)
    cols["z"] = rng.uniform(-0.5, 0.5, n)
    for k in ("nx", "ny", "nz"):
        cols[k] = np.zeros(n)
    for i in range(3):
        cols[f"f_dc_{i}"] = rng.normal(0, 1.0, n)
    for i in range(rest):
        cols[f"f_rest_{i}"] = rng.normal(0, 0.2, n)
    cols["opacity"] = rng.normal(1.0, 1.5, n)
    for i in range(3):
        cols[f"scale_{i}"] = rng.uniform(-4.5, -2.5, n)
    for i in range(4):
        cols[f"rot_{i}"] = rng.normal(0, 1, n)
    data = np.stack([cols[k] for k in names], axis=1).astype("<f4")
    for r in bad_rows:  # non-finite rows are dropped by the loader
        if r < n:
            data[r, 3] = np.nan if r % 2 else np.inf
    with open(path, "wb") as f:
        f.write(b"ply\nformat binary_little_endian 1.0\ncomment fixture\n")
        f.write(f"element vertex {n}\n".encode())
        for k in names:
            f.write(f"property float {k}\n".encode())
        f.write(b"element face 0\nproperty list uchar int vertex_indices\nend_header\n")
        f.write(data.tobytes())
    return data

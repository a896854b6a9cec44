"""Phase attribution of K1 (k_preprocess) warp-instructions and stall samples from one
ncu --set full --import-source capture, by CUDA source line (profiles/r02_k1_source.txt).

    python scripts/k1_phases.py gpurun_out/prof.ncu-rep > profiles/r02_k1_source.txt
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:k_preprocess", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = collections.defaultdict(lambda: [0.0, 0.0])
lines = collections.defaultdict(lambda: [0.0, 0.0, ""])
fname, hdr = None, None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    try:
        ln = int(r[0])
        inst = float(r[hdr.index("Instructions Executed")] or 0)
        stall = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        continue
    lines[(fname, ln)][0] += inst
    lines[(fname, ln)][1] += stall
    lines[(fname, ln)][2] = r[1].strip()[:80]


def phase(f, ln, src):
    if f == "k_preprocess.cu":
        if 38 <= ln <= 45:
            return "A: LUT bin (T_upper, lut.hpp:16-25)"
        if 47 <= ln <= 88:
            return "B: SH colour (eval_color)"
        if 90 <= ln <= 110:
            return "A: to_camera, near / NDC guard (float)"
        if 111 <= ln <= 181:
            return "A: fp64 EWA (Jacobian, J.W, quaternion -> Sigma3D, Sigma2D)"
        if 183 <= ln <= 188:
            return "A: Eq. 10 compute_th"
        if 190 <= ln <= 209:
            return "frame-scoped zeroing + setup"
        if 210 <= ln <= 270:
            return "A: loads, culls, survivor queue"
        return "B: inv_cov, plane / status / key stores, depth range"
    if f == "agsx_internal.cuh":
        if 73 <= ln <= 148:
            return "B: tile-test setup (radius: glibc logf, sqrt; eigen for AABB/OBB)"
        if 149 <= ln <= 431:
            return "B: exact tile test over the span -> hit mask"
        if 432 <= ln <= 503:
            return "B: blend-cull data (qcut, qsafe, extent)"
        return "B: other helpers"
    if f == "device_math.cuh":
        if "sclampd" in src or "double" in src:
            return "A: fp64 EWA (Jacobian, J.W, quaternion -> Sigma3D, Sigma2D)"
        if 56 <= ln <= 95:
            return "B: tile-test setup (radius: glibc logf, sqrt; eigen for AABB/OBB)"
        if 35 <= ln <= 40:
            return "A/B: x86 float->int (LUT bin, tile span)"
        return "B: exact tile test over the span -> hit mask (smin/smax/clamp)"
    return "other (" + f + ")"


for (f, ln), (i, s, src) in lines.items():
    a = agg[phase(f, ln, src)]
    a[0] += i
    a[1] += s
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", "regex:k_preprocess"], capture_output=True,
                     text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
d = dict(zip(rr[0], rr[2]))
print("# K1 k_preprocess, config 3 (veil 3M, 4608x3456, AdaGScale on): one ncu --set full capture")
print(f"# time {d.get('gpu__time_duration.sum')} us, warp-instructions {d.get('smsp__inst_executed.sum')}, "
      f"issue active {d.get('smsp__issue_active.avg.pct_of_peak_sustained_active')} %, "
      f"warps active {d.get('sm__warps_active.avg.pct_of_peak_sustained_active')} %, "
      f"registers {d.get('launch__registers_per_thread')}")
print(f"# DRAM read {d.get('dram__bytes_read.sum')} MB, write {d.get('dram__bytes_write.sum')} MB")
print("# Phase A: all N Gaussians (one thread each); phase B: the survivors, packed into warps through")
print("# the shared-memory queue.  Source-line attribution (inlined helpers count toward their line).")
print(f"{'share of inst':>13s} {'share of stalls':>15s}  phase")
for k, (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{100 * i / ti:12.1f}% {100 * s / ts:14.1f}%  {k}")
print("\n# hottest source lines")
for (f, ln), (i, s, src) in sorted(lines.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"{100 * i / ti:5.1f}% inst {100 * s / ts:5.1f}% stall  {f}:{ln:<4d} {src}")

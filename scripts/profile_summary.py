"""Summarise one frame's ncu --set full capture into profiles/<tag>_*.txt and
profiles/ncu_frame_c<config>_<mode>.json (per-stage DRAM bytes and warp
instructions per frame, read by bench.py for roofline.traffic and the issue
rooflines of that workload only).

    python scripts/profile_summary.py gpurun_out/prof.ncu-rep gpurun_out/launches.csv r02a [config] [mode] [sort_path]
"""
import collections
import csv
import io
import json
import subprocess
import sys

rep, launches, tag = sys.argv[1], sys.argv[2], sys.argv[3]
cfg = sys.argv[4] if len(sys.argv) > 4 else "3"
mode = sys.argv[5] if len(sys.argv) > 5 else "adagscale"
sort_path = sys.argv[6] if len(sys.argv) > 6 else "depth"
STAGE = {"k_preprocess": "preprocess", "k_emit": "pair_gen", "k_scan_chunks": "pair_gen", "k_upsweep": "sort",
         "k_scan_counts": "sort", "k_downsweep": "sort", "k_ranges_u32": "sort", "k_raster_units": "raster",
         "k_raster16": "raster", "k_tile_scan": "sort", "k_bucket_scatter": "pair_gen", "k_tile_sort": "sort"}
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
col = {k: h.index(k) for k in ("Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum",
                               "dram__bytes_write.sum", "smsp__inst_executed.sum")}
assert rows[1][col["gpu__time_duration.sum"]] == "us" and rows[1][col["dram__bytes_read.sum"]] == "Mbyte"
agg = collections.OrderedDict()
for r in rows[2:]:
    base = r[col["Kernel Name"]].split("(")[0].replace("void ", "").replace("<unnamed>::", "").split("<")[0].strip()
    st = STAGE.get(base, base)
    a = agg.setdefault(st, {"launches": 0, "ncu_us": 0.0, "dram_bytes": 0, "warp_inst": 0, "kernels": []})
    a["launches"] += 1
    a["ncu_us"] += float(r[col["gpu__time_duration.sum"]])
    a["dram_bytes"] += int(1e6 * (float(r[col["dram__bytes_read.sum"]]) + float(r[col["dram__bytes_write.sum"]])))
    a["warp_inst"] += int(float(r[col["smsp__inst_executed.sum"]]))
    if base not in a["kernels"]:
        a["kernels"].append(base)
doc = {"source": rep, "capture": f"ncu --set full --clock-control none, one frame of bench.py --config {cfg} "
                                f"--mode {mode}", "sort_path": sort_path, "tag": tag, "per_frame": agg}
json.dump(doc, open(f"profiles/ncu_frame_c{cfg}_{mode}.json", "w"), indent=1)
summ = subprocess.run([sys.executable, "scripts/ncu_summary.py", rep], capture_output=True, text=True).stdout
open(f"profiles/{tag}_ncu_full_summary.txt", "w").write(
    f"# ncu --set full --clock-control none, one frame (config {cfg} {mode}); t in us, dram in MB\n" + summ)
src = subprocess.run([sys.executable, "scripts/ncu_source.py", rep, "k_raster_units", "30"], capture_output=True,
                     text=True).stdout
open(f"profiles/{tag}_raster_source.txt", "w").write("# k_raster_units SASS opcode mix + hottest instructions\n" + src)
lines = open(launches).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
lr = list(csv.reader(lines[start:]))
lh = lr[0]
ki, vi = lh.index("Kernel Name"), lh.index("Metric Value")
per = collections.OrderedDict()
for r in lr[1:]:
    per.setdefault(r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "").split("<")[0].strip(), []).append(float(r[vi]))
tot = sum(sum(v) for k, v in per.items() if k != "k_pack_scene")
with open(f"profiles/{tag}_launches_summary.txt", "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised), bench.py --steps 2 "
            f"--warmup 3, config {cfg} {mode}; share = share of the summed kernel time\n")
    for k, v in sorted(per.items(), key=lambda x: -sum(x[1])):
        f.write(f"{k:28s} launches={len(v):4d} mean_us={sum(v) / len(v) / 1e3:9.1f} "
                f"share={(sum(v) / tot if k != 'k_pack_scene' else 0):6.1%}\n")
print(json.dumps(agg, indent=1))

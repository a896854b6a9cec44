"""Per-CUDA-source-line totals (instructions executed, stall samples) of one
kernel from an ncu report (--print-source cuda,sass)."""
import collections, csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
fname = None
rows = list(csv.reader(io.StringIO(out)))
hdr = None
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
        line = int(r[0])
        inst = float(r[hdr.index("Instructions Executed")] or 0)
        stall = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        continue
    a = agg[(fname, line)]
    a[0] += inst
    a[1] += stall
    a[2] = r[1].strip()[:70]
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp-instructions {ti:.3e}")
for (f, l), (i, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*i/ti:5.1f}% inst {100*s/ts:5.1f}% stall  {f}:{l:<5d} {src}")

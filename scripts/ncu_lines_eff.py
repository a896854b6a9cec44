"""Per-source-line warp instructions and active-thread efficiency of one
kernel from an ncu report (--print-source cuda,sass)."""
import collections, csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
fname, hdr = None, None
for r in csv.reader(io.StringIO(out)):
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
        thr = float(r[hdr.index("Thread Instructions Executed")] or 0)
    except ValueError:
        continue
    a = agg[(fname, line)]
    a[0] += inst
    a[1] += thr
    a[2] = r[1].strip()[:60]
ti = sum(v[0] for v in agg.values()) or 1
tt = sum(v[1] for v in agg.values()) or 1
print(f"total warp-inst {ti:.3e}  thread-inst {tt:.3e}  avg active lanes {tt/ti:.1f}")
for (f, l), (i, t, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*i/ti:5.1f}% inst lanes {t/max(i,1):4.1f}  {f}:{l:<5d} {src}")

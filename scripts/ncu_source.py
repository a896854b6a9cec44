"""SASS hotspot summary of one kernel from an ncu report: stall samples and executed
instructions grouped by opcode, plus the hottest individual instructions."""
import collections, csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
r = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = r[0]
si, ci, ii = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
rows = []
for row in r[1:]:
    try:
        rows.append((float(row[ci] or 0), float(row[ii] or 0), row[si].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(x[0] for x in rows) or 1
toti = sum(x[1] for x in rows) or 1
by = collections.defaultdict(lambda: [0.0, 0.0])
for s, i, src in rows:
    op = src.split()[0] if not src.startswith("@") else src.split()[1]
    op = op.split(".")[0]
    by[op][0] += s
    by[op][1] += i
print(f"total warp-instructions executed: {toti:.3e}")
for op, (s, i) in sorted(by.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{op:10s} {100*i/toti:5.1f}% inst  {100*s/tot:5.1f}% stall-samples")
print("--- hottest instructions by samples")
for s, i, src in sorted(rows, reverse=True)[:12]:
    print(f"{100*s/tot:5.1f}%  {src[:90]}")

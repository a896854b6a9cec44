"""Per-kernel times from an ncu --metrics gpu__time_duration.sum --csv log file."""
import collections, csv, sys
lines = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
h = rows[0]
ki, gi, vi = h.index("Kernel Name"), h.index("Grid Size"), h.index("Metric Value")
last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
sel = rows[1:][-last:] if last else rows[1:]
for r in sel:
    print(f"{r[ki][:48]:48s} grid={r[gi]:>14s} {float(r[vi])/1e3:9.1f} us")

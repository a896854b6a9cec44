"""Summarise an ncu report: per kernel duration, DRAM bytes, SM/issue %, top stalls."""
import csv, subprocess, sys, io
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h = r[0]
def col(name):
    return h.index(name) if name in h else None
cols = {k: col(k) for k in ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "smsp__inst_executed.sum",
        "launch__grid_size", "lts__t_bytes.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]}
stall_cols = [(i, n) for i, n in enumerate(h) if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")]
for row in r[2:]:
    g = lambda k: row[cols[k]] if cols[k] is not None else "?"
    name = g("Kernel Name")[:34]
    st = []
    for i, n in stall_cols:
        try: st.append((float(row[i]), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError: pass
    st.sort(reverse=True)
    tot = sum(v for v, _ in st) or 1
    print(f"{name:34s} t={g('gpu__time_duration.sum'):>9s} dramR={g('dram__bytes_read.sum'):>10s} dramW={g('dram__bytes_write.sum'):>10s} "
          f"sm%={g('sm__throughput.avg.pct_of_peak_sustained_elapsed')[:5]} issue%={g('smsp__issue_active.avg.pct_of_peak_sustained_active')[:5]} "
          f"dram%={g('dram__throughput.avg.pct_of_peak_sustained_elapsed')[:5]} warps%={g('sm__warps_active.avg.pct_of_peak_sustained_active')[:5]} "
          f"regs={g('launch__registers_per_thread')} inst={g('smsp__inst_executed.sum')[:12]} grid={g('launch__grid_size')} "
          f"stalls=" + ",".join(f"{n}:{v/tot:.0%}" for v, n in st[:4]))

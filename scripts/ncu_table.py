"""Per-launch table of an ncu report: time, warp-instructions, DRAM bytes, issue and occupancy."""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[0]
cols = [("Kernel Name", "kernel"), ("gpu__time_duration.sum", "us"), ("smsp__inst_executed.sum", "warp_inst"),
        ("dram__bytes_read.sum", "rd_MB"), ("dram__bytes_write.sum", "wr_MB"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"), ("launch__registers_per_thread", "regs"),
        ("lts__t_sectors_op_atom.sum", "l2_atom_sect"), ("lts__t_sectors_op_red.sum", "l2_red_sect"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_confl")]
idx = [(h.index(c), n) for c, n in cols if c in h]
print(" | ".join(n for _, n in idx))
for row in r[2:]:
    print(" | ".join(row[i][:34] for i, _ in idx))

"""Key metrics of the first kernel in an ncu report: python tools/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u, v = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "smsp__inst_executed_op_shared_atom.sum",
        "smsp__inst_executed_op_global_red.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for n in want:
    if n in h:
        i = h.index(n)
        print(f"{n:60s} {v[i]:>16s} {u[i]}")
st = [(float(v[i] or 0), n) for i, n in enumerate(h)
      if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")]
print("stalls per issue:", ", ".join(f"{n[34:-29]} {x:.2f}" for x, n in sorted(st, reverse=True)[:9]))

"""Summary of an ncu capture of k_g2p2g_f32: headline metrics, stalls, and
instructions / stall samples per kernel phase (CSV exports in /tmp)."""
import collections
import csv
import sys

raw, mix, src_path = sys.argv[1], sys.argv[2], sys.argv[3]
n_part = float(sys.argv[4]) if len(sys.argv) > 4 else 101e6
rows = list(csv.reader(open(raw)))
hdr = rows[0]
d = dict(zip(hdr, rows[2]))
for k in ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed_op_shared_atom.sum",
          "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]:
    print(f"{k:60s} {d.get(k)}")
st = sorted([(h, d[h]) for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and
             h.endswith("_per_issue_active.ratio")], key=lambda x: -float(x[1] or 0))[:8]
print("stalls/issue:", ", ".join(f"{h[34:-29]} {float(v):.2f}" for h, v in st))
rws = []
cur_file = cur_line = None
for r in csv.reader(open(mix)):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0]:
        if r[0].isdigit():
            cur_line = (cur_file, int(r[0]))
        continue
    if len(r) > 8 and r[2].startswith("0x"):
        rws.append((int(r[2], 16), cur_line, int(r[4]), int(r[7])))
rws.sort()
src = open(src_path).read().split("\n")


def line_of(pat):
    return next(i for i, l in enumerate(src, 1) if pat in l)


b = [line_of("// [B1]"), line_of("// [B2]"), line_of("// [B3]")]
regions = [("prime", 1, b[0]), ("A", b[0] + 1, b[1]), ("S", b[1] + 1, b[2]), ("F", b[2] + 1, len(src))]
acc = collections.defaultdict(lambda: [0, 0])
region = "pre"
ts = sum(x[2] for x in rws)
ti = sum(x[3] for x in rws)
fname = src_path.split("/")[-1]
for addr, (f, ln), s, i in rws:
    if f == fname:
        for n, lo, hi in regions:
            if lo <= ln <= hi:
                region = n
    acc[region][0] += s
    acc[region][1] += i
for k, (s, i) in sorted(acc.items(), key=lambda x: -x[1][0]):
    print(f"{k:6s} samples {100 * s / ts:5.1f}%  inst {100 * i / ti:5.1f}%  ({i * 32 / n_part:.0f} thread-inst/particle)")

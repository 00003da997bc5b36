"""Split an ncu SASS source page (csv) into regions between barriers and
report instructions / stall samples per region and per opcode class.
usage: ncu -i rep --page source --csv --print-source sass > x.csv; python tools/sass_regions.py x.csv"""
import csv
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {n: i for i, n in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) == len(hdr)]
tot_i = sum(float(r[ix["Instructions Executed"]] or 0) for r in body)
tot_s = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in body)
reg, regions = [], []
for r in body:
    reg.append(r)
    if r[ix["Source"]].strip().split(" ")[0].startswith("BAR") or "BAR.SYNC" in r[ix["Source"]]:
        regions.append(reg)
        reg = []
regions.append(reg)
print(f"total warp-inst {tot_i:.4g}  stall samples {tot_s:.4g}")
for k, g in enumerate(regions):
    ni = sum(float(r[ix["Instructions Executed"]] or 0) for r in g)
    ns = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in g)
    if ni == 0 and ns == 0:
        continue
    ops = Counter()
    for r in g:
        op = r[ix["Source"]].strip()
        if op.startswith("@"):
            op = op.split(" ", 1)[1] if " " in op else op
        ops[op.split(" ")[0].split(".")[0]] += float(r[ix["Instructions Executed"]] or 0)
    top = ", ".join(f"{o}:{v / tot_i * 100:.1f}" for o, v in ops.most_common(8))
    print(f"region {k:2d} [{g[0][ix['Address']]}..{g[-1][ix['Address']]}] inst {ni / tot_i * 100:5.1f}%  stalls {ns / tot_s * 100:5.1f}%  | {top}")
ops = Counter()
for r in body:
    op = r[ix["Source"]].strip()
    if op.startswith("@"):
        op = op.split(" ", 1)[1]
    ops[op.split(" ")[0]] += float(r[ix["Instructions Executed"]] or 0)
print("opcode mix:", ", ".join(f"{o}:{v / tot_i * 100:.1f}" for o, v in ops.most_common(30)))

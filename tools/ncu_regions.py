"""Stall samples / warp instructions of k_g2p2g by code region, from an ncu
report exported with --page source --csv --print-source cuda,sass.
Inlined helpers (FFMA2 intrinsics, axis_base, bspline) are charged to the
smpm_sim.cu region they are inlined into (address order).
usage: ncu_regions.py CSV 'name:lo-hi,name:lo-hi,...' (smpm_sim.cu lines)"""
import csv
import sys

path, spec = sys.argv[1], sys.argv[2]
regions = []
for item in spec.split(","):
    name, rng = item.split(":")
    lo, hi = (int(v) for v in rng.split("-"))
    regions.append((name, lo, hi))
rows = []
cur_file = None
cur_line = None
for r in csv.reader(open(path)):
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
        try:
            rows.append((int(r[2], 16), cur_line, r[3].strip(), int(r[4]), int(r[7])))
        except ValueError:
            pass
rows.sort()
ts = sum(x[3] for x in rows)
ti = sum(x[4] for x in rows)
acc = {}
region = "other"
for addr, (f, ln), sass, s, i in rows:
    if f == "smpm_sim.cu":
        hit = next((n for n, lo, hi in regions if lo <= ln <= hi), None)
        if hit is not None:  # lines outside every range (inlined helpers) keep the current region
            region = hit
    elif f == "smpm_common.cuh" and ln >= 200:
        region = "stress(hencky)" if region not in ("flush",) else region
    a = acc.setdefault(region, [0, 0])
    a[0] += s
    a[1] += i
for k, (s, i) in sorted(acc.items(), key=lambda x: -x[1][0]):
    print(f"{k:22s} samples {100*s/ts:5.1f}%  warp inst {100*i/ti:5.1f}%  ({i/1e6:.0f}M)")

"""Address-ordered SASS of an ncu report (cuda,sass CSV), each instruction
tagged with its source line; prints runs of consecutive instructions by
source region with stall samples and warp instructions executed."""
import csv
import sys

path = sys.argv[1]
rows = []
cur_file = None
cur_line = None
for r in csv.reader(open(path)):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
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
# group runs of the same (file, line-bucket)
out = []
for addr, (f, ln), sass, s, i in rows:
    key = f"{f}:{ln}"
    if out and out[-1][0] == key:
        out[-1][1] += s
        out[-1][2] += i
        out[-1][3] += 1
    else:
        out.append([key, s, i, 1, addr, sass])
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.3
for key, s, i, n, addr, sass in out:
    if 100 * s / ts >= thr or 100 * i / ti >= thr:
        print(f"{addr & 0xfffff:6x} {key:28s} n={n:4d} samp {100*s/ts:5.2f}% inst {100*i/ti:5.2f}%  {sass[:50]}")

"""Per-source-line stall samples / warp instructions from an ncu report
(--page source --print-source cuda,sass CSV).  usage: ncu_lines.py CSV [top]"""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur = None
rows = []
hdr = None
for r in csv.reader(open(path)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0] and hdr and cur:
        try:
            samples = int(r[4])
            inst = int(r[7])
        except (ValueError, IndexError):
            continue
        rows.append((cur, int(r[0]), samples, inst, r[1].strip()[:90]))
ts = sum(x[2] for x in rows)
ti = sum(x[3] for x in rows)
print(f"total samples {ts}, warp instructions {ti}")
for f, ln, s, i, src in sorted(rows, key=lambda x: -x[2])[:top]:
    print(f"{f}:{ln:5d} samp {100*s/ts:5.2f}% inst {100*i/ti:5.2f}%  {src}")

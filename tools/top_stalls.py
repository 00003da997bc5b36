"""Top stalled SASS instructions of an ncu report: python tools/top_stalls.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {n: i for i, n in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) == len(hdr)]
S = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in body)
stalls = [n for n in hdr if n.startswith("stall_") and "Not Issued" not in n]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for k, r in enumerate(body):
    r.append(k)
for r in sorted(body, key=lambda r: -float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:N]:
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    det = sorted(((float(r[ix[n]] or 0), n) for n in stalls), reverse=True)[:3]
    print(f"#{r[-1]:5d} {s / S * 100:5.2f}% {r[ix['Source']][:64]:64s}", [(n[6:], round(v / S * 100, 2)) for v, n in det])

"""Per-CUDA-line instructions and stall samples from an ncu report
(--page source --print-source cuda,sass).  usage: python tools/src_lines.py rep.ncu-rep [kernel-regex] [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n_top = int(sys.argv[3]) if len(sys.argv) > 3 else 60
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, recs = None, None, []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = {n: i for i, n in enumerate(r) if n not in ("Source",)}
        hdr["Inst"] = r.index("Instructions Executed")
        hdr["Stall"] = r.index("Warp Stall Sampling (All Samples)")
    elif hdr and r[0] not in ("", "Function Name", "Kernel Name"):
        try:
            recs.append((fname, int(r[0]), r[1][:90], float(r[hdr["Inst"]] or 0), float(r[hdr["Stall"]] or 0)))
        except ValueError:
            pass
ti = sum(x[3] for x in recs)
ts = sum(x[4] for x in recs)
print(f"total inst {ti:.4g} stall samples {ts:.4g}")
for f, ln, src, i, s in sorted(recs, key=lambda x: -x[3])[:n_top]:
    print(f"{f}:{ln:5d} inst {i / ti * 100:5.2f}% stall {s / ts * 100:5.2f}% | {src.strip()}")

"""Instruction / stall split of k_g2p2g by source phase (line ranges of smpm_sim.cu; inlined
helpers from other files are attributed by name).  usage: python tools/phase_split.py rep.ncu-rep"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

src = open("paper_2605_28525_b200/csrc/smpm_sim.cu").read().splitlines()
marks = [("flush(lambda)", r"auto flush = \["), ("loop top / item setup", r"while \(true\) \{"),
         ("G2P", r"// ---- G2P \(solver"), ("F update + advect", r"F <- \(I \+ dt a\)"),
         ("stress call", r"// ---- stress of the next"), ("record store", r"// ---- write the particle record"),
         ("next keys + migration", r"// ---- next step's keys"), ("bounds + masks + counts", r"// contribution bounds"),
         ("after B2: prefetch/probe/scales", r"__syncthreads\(\);  // \[B2\]"), ("P2G scatter", r"// ---- P2G of the next"),
         ("flush call", r"// ---- flush item i-1"), ("ranks + rotate", r"// ---- warp 0: ranks"),
         ("tail", r"^  if \(have_prev\) flush\(p \^ 1\);$")]
bounds = []
for name, pat in marks:
    for i, l in enumerate(src):
        if re.search(pat, l):
            bounds.append((i + 1, name))
            break
bounds.sort()


def phase(line):
    name = "prologue"
    for b, n in bounds:
        if line >= b:
            name = n
    return name


out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = defaultdict(lambda: [0.0, 0.0])
fname, hdr = None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = (r.index("Instructions Executed"), r.index("Warp Stall Sampling (All Samples)"))
    elif hdr and r[0].isdigit():
        ln = int(r[0])
        key = phase(ln) if fname == "smpm_sim.cu" else f"[{fname}]"
        if fname == "smpm_common.cuh" and 120 <= ln <= 160:
            key = "[common: stencil/axis_base]"
        elif fname == "smpm_common.cuh" and ln > 160:
            key = "[common: hencky/DP]"
        try:
            agg[key][0] += float(r[hdr[0]] or 0)
            agg[key][1] += float(r[hdr[1]] or 0)
        except ValueError:  # source text with unbalanced quotes (inline asm) breaks the csv row
            pass
ti = sum(v[0] for v in agg.values())
ts = sum(v[1] for v in agg.values())
print(f"{'phase':40s} {'inst%':>7s} {'stall%':>7s}")
for k, (i, s) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{k:40s} {i / ti * 100:7.2f} {s / ts * 100:7.2f}")

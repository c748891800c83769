"""Warp-stall breakdown of one ncu --set full capture (--import-source on, -lineinfo build):
the PC-sampling samples (smsp__pcsamp_*: "Warp Stall Sampling") by stall reason, by SASS
opcode and by CUDA source line, next to the instructions executed -- where the kernel's
warps wait.

    python scripts/ncu_stalls.py rep.ncu-rep "label" >> profiles/r02_k3c_stalls.txt
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
label = sys.argv[2] if len(sys.argv) > 2 else rep


def src_page(what):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", what],
                         capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


rows = src_page("sass")
hdr = rows[1]
body = [x for x in rows[2:] if len(x) == len(hdr)]
isrc, iall, iex = (hdr.index(k) for k in ("Source", "Warp Stall Sampling (All Samples)", "Instructions Executed"))
reasons = [h for h in hdr if h.startswith("stall_") and "(Not Issued)" not in h]
tot = sum(int(x[iall]) for x in body) or 1
totex = sum(int(x[iex]) for x in body) or 1
print(f"== {label}")
print(f"PC samples {tot}, warp instructions executed {totex}")
rs = {r: sum(int(x[hdr.index(r)] or 0) for x in body) for r in reasons}
print("by stall reason (% of samples): " + ", ".join(f"{r[6:]} {100 * v / tot:.1f}" for r, v in
                                                  sorted(rs.items(), key=lambda kv: -kv[1]) if v))
op, opx = collections.Counter(), collections.Counter()
for x in body:
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", x[isrc])
    o = m.group(2) if m else "?"
    op[o] += int(x[iall])
    opx[o] += int(x[iex])
print("by SASS opcode (% of samples / % of executed instructions): " +
      ", ".join(f"{o} {100 * v / tot:.1f}/{100 * opx[o] / totex:.1f}" for o, v in op.most_common(14)))
rows = src_page("cuda,sass")
lines = []
path = ""
for x in rows:
    if len(x) == 2 and x[0] in ("File Path", "File Name"):
        path = x[1].split("/")[-1]
        continue
    if len(x) > 8 and x[0].isdigit() and x[4].lstrip("-").isdigit():
        lines.append((int(x[4]), int(x[7]) if x[7].isdigit() else 0, f"{path}:{x[0]}", x[1].strip()))
print("by CUDA source line (top 15; % of samples, % of executed instructions):")
for smp, ex, where, text in sorted(lines, key=lambda t: -t[0])[:15]:
    print(f"  {100 * smp / tot:5.1f}%  {100 * ex / totex:5.1f}%  {where:24s} {text[:90]}")

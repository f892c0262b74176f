"""Top CUDA source lines by warp-stall samples for one kernel of an ncu report.

usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [N]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
lines = []
fname = ""
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[2] == "-":
        try:
            samp = float(r[4])
            inst = float(r[7])
        except ValueError:
            continue
        lines.append((samp, inst, f"{fname}:{r[0]}", r[1][:90]))
tot = sum(x[0] for x in lines) or 1
print(f"total samples {tot:.0f}")
for samp, inst, loc, src in sorted(lines, reverse=True)[:top]:
    print(f"{100*samp/tot:5.1f}%  inst={inst:12.0f}  {loc:18s} {src}")

#!/usr/bin/env python
"""Per-source-line instructions and stall samples from an ncu report (--import-source,
-lineinfo builds): python scripts/ncu_lines.py report.ncu-rep [top] [kernel-regex]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 3:
    cmd += ["--kernel-name", f"regex:{sys.argv[3]}"]
txt = subprocess.run(cmd, capture_output=True, text=True).stdout
rows, f, hdr = [], None, None
tot_i = tot_s = 0
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or not r[0].isdigit() or r[2] != "-":
        continue
    ins = int(r[hdr["Instructions Executed"]] or 0)
    st = int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
    tot_i += ins
    tot_s += st
    rows.append((ins, st, f, int(r[0]), r[1][:90]))
print(f"total warp instructions {tot_i:,}  stall samples {tot_s:,}")
print("  instr%  stall%  file:line  source")
for ins, st, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"  {100 * ins / max(tot_i, 1):5.1f}  {100 * st / max(tot_s, 1):5.1f}  {f}:{ln}  {src}")

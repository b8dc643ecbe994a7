#!/usr/bin/env python
"""SASS of an ncu report in address order with executed warp instructions and the CUDA
source line each instruction maps to: python scripts/ncu_sass.py report.ncu-rep > dump"""
import csv
import io
import subprocess
import sys

txt = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
hdr, f, cur, out = None, None, None, []
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:
        cur = f"{f}:{r[0]}"
        continue
    if not r[2].startswith("0x"):
        continue
    n = int(r[7] or 0)
    st = int(r[4] or 0) if r[4] not in ("-", "") else 0
    out.append((int(r[2], 16), cur, r[3].strip(), n, st))
# an inlined instruction is listed once per source line it maps to: keep one row per address,
# preferring the kernel file's own line (gc_decode.cuh) for the phase attribution
best = {}
for a, c, s_, n, st in out:
    if a not in best or (c or "").startswith("gc_decode.cuh"):
        best[a] = (a, c, s_, n, st)
out = sorted(best.values())
base = out[0][0] if out else 0
for a, c, s, n, st in out:
    print(f"{a - base:6x} {n:9d} {st:5d} {c:24s} {s}")

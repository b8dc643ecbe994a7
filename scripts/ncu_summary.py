#!/usr/bin/env python
"""Summarise ncu outputs for profiles/ (run here, on the CPU box).

  python scripts/ncu_summary.py launches <launches.csv>      per-kernel device time and share
  python scripts/ncu_summary.py full <report.ncu-rep>        key metrics of each profiled launch
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def launches(path, only="gcd::"):
    rows = [r for r in csv.reader(open(path)) if r and r[0] not in ("==PROF==",) and not r[0].startswith("==")]
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) < len(hdr) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[idx["Kernel Name"]]
        short = name.split("(")[0].replace("void ", "")
        if only and only not in short:
            continue
        v = float(r[idx["Metric Value"]].replace(",", ""))
        unit = r[idx["Metric Unit"]]
        v = v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
        tot[short] += v
        cnt[short] += 1
    all_us = sum(tot.values())
    print("| kernel | launches | total us | mean us | share |")
    print("|---|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"| `{k}` | {cnt[k]} | {v:.1f} | {v / cnt[k]:.2f} | {100 * v / all_us:.1f}% |")
    print(f"\nall kernels: {all_us:.1f} us (cold-cache, serialised by ncu: compare shares, not absolutes)")


KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("smsp__inst_executed.sum", "warp inst"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    stalls = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_")
              and h.endswith("_per_issue_active.ratio")]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(f"### `{d['Kernel Name'][:90]}`")
        print("| metric | value |\n|---|---|")
        for k, label in KEYS:
            if k in d:
                print(f"| {label} (`{k}`) | {d[k]} {units[hdr.index(k)]} |")
        st = sorted(((float(d[h]) if d[h] not in ("", "n/a") else 0.0, h) for h in stalls),
                    reverse=True)[:6]
        s = ", ".join(f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}"
                      for v, h in st)
        print(f"| top stalls (warps per issue) | {s} |\n")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])

#!/usr/bin/env python
"""Summarise ncu outputs for profiles/ (run here, on the CPU box).

  python scripts/ncu_summary.py launches <launches.csv>      per-kernel device time and share
  python scripts/ncu_summary.py full <report.ncu-rep>        key metrics of each profiled launch
"""
import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import defaultdict


def launches(path, only="k_"):
    rows = [r for r in csv.reader(open(path)) if r and r[0] not in ("==PROF==",) and not r[0].startswith("==")]
    rows = rows[next(i for i, r in enumerate(rows) if r[0] == "ID"):]  # (ncu notes before the header)
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


def kernel_label(name: str):
    """(variant label, d-gap path?) of a k_decode / k_index instantiation, else None."""
    m = re.search(r"k_(decode|index)<(?:gcd::)?Codec(\w+)(?:<([^>]*)>)?(?:, (?:\(bool\))?(\d|true|false))?", name)
    if not m:
        return None
    kind, codec, targs, dg = m.groups()
    ta = [t.split(")")[-1].strip() for t in (targs or "").split(",") if t]
    if codec.startswith("Gsc"):
        lab = f"GSC-{ta[0]}-{codec[3:]}"
    elif codec == "GS":
        lab = "G-SIM"
    elif codec == "AFOR":
        lab = "G-AFOR"
    else:  # PFD<F, kE>
        base = "G-PFD" if (len(ta) < 2 or ta[1] in ("1", "true")) else "BP128"
        lab = base if ta[0] == "32" else f"{base}-F{ta[0]}"
    return kind, lab, dg in ("1", "true")


def traffic(path, workload, out_json="profiles/r2_traffic.json"):
    """Per-launch traffic of each k_decode d-gap instantiation in an ncu --set full report:
    dram__bytes_read.sum + 32 x lts__t_sectors_srcunit_tex_op_write.sum (every byte the
    kernel writes reaches L2; the DRAM write counter misses the tail still in L2 at the
    kernel's end), merged into out_json under `workload`."""
    if path.endswith(".csv.gz"):  # a raw page saved on the GPU box
        import gzip
        out = gzip.open(path, "rt").read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]

    def val(d, k):
        u = units[hdr.index(k)]
        v = float(d[k].replace(",", ""))
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    try:
        with open(out_json) as f:
            db = json.load(f)
    except Exception:  # noqa: BLE001
        db = {}
    ent = db.setdefault(workload, {})
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        kl = kernel_label(d["Kernel Name"])
        if not kl or kl[0] != "decode" or not kl[2]:
            continue
        rd = val(d, "dram__bytes_read.sum")
        wr_l2 = float(d["lts__t_sectors_srcunit_tex_op_write.sum"].replace(",", "")) * 32
        ent[kl[1]] = {"bytes_per_launch": rd + wr_l2, "dram_read": rd, "l2_write": wr_l2,
                      "dram_write": val(d, "dram__bytes_write.sum"),
                      "duration": f'{d["gpu__time_duration.sum"]} {units[hdr.index("gpu__time_duration.sum")]}',
                      "report": os.path.basename(path)}
        print(workload, kl[1], ent[kl[1]])
    with open(out_json, "w") as f:
        json.dump(db, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    {"launches": launches, "full": full, "traffic": traffic}[sys.argv[1]](*sys.argv[2:])

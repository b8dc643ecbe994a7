#!/usr/bin/env python
"""Tables of profiles/rN_summary.md from the committed bench lines and ncu files.

  python scripts/make_summary.py            (prints markdown)
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import ncu_summary  # noqa: E402


def bench(name):
    d = json.load(open(os.path.join(P, name)))
    r = d["roofline"]
    print(f"`{name}`: **{d['value']:.4g} {d['unit']}** ({d['ms_per_step']:.3f} ms per step), "
          f"roofline frac **{r['frac']:.3f}** (k_decode {r['achieved']:.0f} of {r['peak']} GB/s; "
          f"traffic {r['traffic']}), e2e {d['e2e']['value']:.4g} ints/s "
          f"({d['e2e']['ms_per_step']:.1f} ms/step), CPU oracle "
          f"{d['cpu_baseline']['value']:.4g} ints/s on {d['cpu_baseline']['cores']} cores, "
          f"clocks {d['clocks']['sm_mhz']}/{d['clocks']['sm_max_mhz']} MHz reasons "
          f"{d['clocks']['reasons']}, parity {d['parity']['verified']}.\n")
    print("| variant | k_decode ms | index ms | bits/int | k_decode GB/s | frac |")
    print("|---|---|---|---|---|---|")
    for k, v in d["per_codec"].items():
        print(f"| {k} | {v['decode_kernel_ms']:.4f} | {v['index_ms']:.4f} | {v['bits_per_int']:.2f} "
              f"| {v['decode_kernel_gbs']:.0f} | {v['frac_of_peak']:.3f} |")
    print()


def launches(name):
    rows = [r for r in csv.reader(open(os.path.join(P, name))) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[1:]:
        if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        k = r[ix["Kernel Name"]].split("(")[0].replace("void ", "")
        # the kernels of a bench step: k_lists, k_index, k_decode<..., 1> (d-gaps)
        if not ("k_lists" in k or "k_index" in k or (k.startswith("gcd::k_decode") and k.endswith(", 1>"))):
            continue
        v = float(r[ix["Metric Value"]].replace(",", ""))
        v *= {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ix["Metric Unit"]], 1e-3)
        tot[k] += v
        cnt[k] += 1
    s = sum(tot.values())
    print("| kernel | launches | mean us | share of the step kernels |")
    print("|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"| `{k}` | {cnt[k]} | {v / cnt[k]:.1f} | {100 * v / s:.1f}% |")
    print()


if __name__ == "__main__":
    for f in ("r1_bench_cfg2.json", "r1_bench_cfg3.json", "r1_bench_cfg4.json", "r1_bench_cfg1.json"):
        print(f"### {f}\n")
        bench(f)
    print("### launch list\n")
    launches("r1_launches_cfg2.csv")
    print("### ncu --set full (GSC-8-B, config 2)\n")
    sys.stdout.flush()
    ncu_summary.full(os.path.join(P, "r1_k_decode_full.ncu-rep"))

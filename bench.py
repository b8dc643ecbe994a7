#!/usr/bin/env python
"""bench.py -- decoded uint32 ints/s of the Group-format decode + d-gap prefix-sum path
on B200 (BASELINE.json metric), one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]

A step is one pass of the whole hot path (control scan, unpack, PFD patch, d-gap scan,
store: gc_decode_dgaps) over one batch for every codec variant of the config.  The
headline workload (`value`) is BASELINE.json configs[1]: Group-Scheme, all 10 granularity x
length-descriptor variants, 2^26 ints in 10^5 lists.  The same run times the other
single-GPU configs at full size as well -- config 1 (Group-Simple, L2-flushed), config 3
(Group-PFD, SIMD-BP128), config 4 (Group-AFOR) -- so `per_codec` holds all 13 variants
("per codec", the metric's own words).  Inputs are synthetic (gen/), encoded by the
library's own host encoder, resident in HBM before timing.

Multi-GPU: `--gpus N` starts N ranks itself (torch.distributed.run) unless it already runs
under one.  One process per GPU, lists sharded by rank with no collective on the data
path; with N > 1 the workload is config 5 (rank r decodes shard r of its 8 list shards,
weak scaling: N = 8 is exactly config 5).  NCCL all-reduces counts and checksums after
timing and the max time over ranks; a barrier precedes every timed step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decoded uint32 ints/sec per codec (1/2/4/8 B200), % of HBM roofline"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=0, choices=[0, 1, 2, 3, 4, 5],
                    help="headline workload (default: 2 on one GPU, 5 on several)")
    ap.add_argument("--extra-configs", default="auto",
                    help="configs timed beside the headline for per_codec ('auto': 1,3,4 "
                         "when the headline is config 2 on one GPU; 'none')")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--codecs", default="", help="comma list of labels (default: config's)")
    ap.add_argument("--pfd-zeta", default="1/10")
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--encode", action="store_true",
                    help="time the GPU frame encoder (Group-PFD, SIMD-BP128) on config 3")
    ap.add_argument("--side-streams", type=int, default=1)
    ap.add_argument("--strong", action="store_true",
                    help="config 5: split the same workload over the ranks (strong scaling)")
    ap.add_argument("--sched", choices=["overlap", "serial"], default="overlap",
                    help="overlap: index stages on a side stream, concurrent with the decodes")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--posting-store", action="store_true",
                    help="time the §7.5 posting store (docIDs + TFs): the fused decode against "
                         "two separate decodes")
    ap.add_argument("--spawn-check", action="store_true",
                    help="(tests) start --gpus ranks, all-reduce their ranks, print one line")
    ap.add_argument("--random-access", action="store_true",
                    help="time gc_decode_range from the skip table (P:L640): whole-batch and "
                         "single-block ranges")
    return ap.parse_args()


def dist_info():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    return int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")), ws


def label_of(codec: int, variant: int, frame_quads: int = 32) -> str:
    """gc.codec_label without importing the product package (the reference arm)."""
    import oracle as O
    if codec == O.GROUP_SCHEME:
        cg, kind = 1 << (variant & 3), ("B", "CU", "IU")[(variant >> 2) & 3]
        return f"GSC-{cg}-{kind}"
    name = {O.VARBYTE: "VByte", O.GROUP_SIMPLE: "G-SIM", O.GROUP_AFOR: "G-AFOR"}.get(codec)
    if name:
        return name
    base = "BP128" if variant == 1 else "G-PFD"
    return base if frame_quads == 32 else f"{base}-F{frame_quads}"


def config_codecs(k: int, zeta):
    import oracle as gc  # (the codec ids; no product code on the reference arm)
    if k == 1:
        return [(gc.GROUP_SIMPLE, 0, 32, zeta)]
    if k == 2:
        return [(gc.GROUP_SCHEME, gc.gsc_variant(cg, kd), 32, zeta)
                for cg, kd in [(cg, k) for cg in (1, 2, 4, 8) for k in ("B", "CU")] + [(4, "IU"), (8, "IU")]]
    if k == 3:  # + SIMD-BP128 on the same gaps: the paper's speed leader as a control
        return [(gc.GROUP_PFD, 0, 32, zeta), (gc.GROUP_PFD, 1, 32, zeta)]
    if k == 4:
        return [(gc.GROUP_AFOR, 0, 32, zeta)]
    # config 5: all four Group codecs (GSC's two representatives) + Variable Byte, the
    # paper's baseline / short-list fallback (P §2.3)
    return [(gc.GROUP_SIMPLE, 0, 32, zeta), (gc.GROUP_SCHEME, gc.gsc_variant(1, "CU"), 32, zeta),
            (gc.GROUP_SCHEME, gc.gsc_variant(8, "IU"), 32, zeta), (gc.GROUP_AFOR, 0, 32, zeta),
            (gc.GROUP_PFD, 0, 32, zeta), (gc.VARBYTE, 0, 32, zeta)]


def codec_subset(w, codec: int):
    """The lists a codec decodes in a step: all of them, except Variable Byte, which is the
    short-list fallback (§7.5): the lists shorter than 64."""
    from paper_1502_01916_b200 import gc
    if codec != gc.VARBYTE:
        return w.values, w.list_n
    if not isinstance(w.values, np.ndarray):  # a device-resident workload
        import torch
        ln = torch.from_numpy(w.list_n.astype(np.int64)).to(w.values.device)
        short = ln < 64
        starts = torch.cumsum(ln, 0) - ln
        owner = torch.repeat_interleave(short, ln)
        return w.values[owner], w.list_n[short.cpu().numpy()]
    ln = w.list_n.astype(np.int64)
    st = np.concatenate([[0], np.cumsum(ln)[:-1]]) if len(ln) else np.zeros(0, np.int64)
    ids = np.nonzero(w.list_n < 64)[0]
    vals = (np.concatenate([w.values[st[i]:st[i] + ln[i]] for i in ids]) if len(ids)
            else np.zeros(0, np.uint32))
    return vals, w.list_n[ids]


def make_workload(args, rank, world, device=None):
    """(workload, global id of its first list, scaling) of this rank (dist.shard_for_rank).
    Config 5's shards (2^31 docIDs each at full size) are drawn on the rank's GPU by
    gen.gpu -- the same counter-based draws as gen/, bit for bit -- when `device` is given:
    then `values` is a device tensor."""
    if device is not None and args.config == 5 and not args.strong:
        import gen
        from gen import gpu as G
        shard = rank % 8
        ln, vals, base = G.config5_shard_gpu(shard, 8, args.scale, device)
        w = gen.Workload("cfg5_all", ln, vals, True, 4,
                         f"config 5 shard {shard} of 8, drawn on the GPU (gen.gpu)")
        return w, base, "weak"
    from paper_1502_01916_b200 import dist
    sh = dist.shard_for_rank(args.config, args.scale, rank, world, strong=args.strong)
    return sh.workload, sh.list_base, sh.scaling


class ClockSampler:
    """NVML sampling of SM clock and clock-event reasons during the timed region."""
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x2: "applications_clocks_setting", 0x80: "hw_power_brake"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.stop_ev = [], 0, threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self.nv = None
            self.max_mhz = None
        self.th = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                fn = getattr(self.nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    self.nv.nvmlDeviceGetCurrentClocksThrottleReasons
                self.reasons |= int(fn(self.h))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.th.start()
        return self

    def __exit__(self, *a):
        self.stop_ev.set()
        if self.nv:
            self.th.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": [n for b, n in self.REASONS.items() if self.reasons & b],
                "samples": len(self.samples)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload: str, label: str):
    """Measured DRAM + L2 traffic of one k_decode launch of this workload and variant, from
    the committed ncu --set full capture (profiles/r2_traffic.json, written by
    scripts/ncu_summary.py traffic): dram__bytes_read.sum + 32 x
    lts__t_sectors_srcunit_tex_op_write.sum (the writes reach L2 in full even when the tail
    is still in L2 at the kernel's end), or None when no capture exists."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_traffic.json")) as f:
            t = json.load(f)
        return t.get(workload, {}).get(label)
    except Exception:  # noqa: BLE001
        return None


def cpu_oracle_rate(hbs, frac_lists: float, budget_s: float, threads: int):
    """The oracle decoder as it stands (oracle/gc_oracle.c, gco_decode_batch with the d-gap
    prefix sum) on the first `frac_lists` of every batch's lists, T host threads."""
    import oracle as O
    samples = []
    for hb in hbs:
        L = max(1, int(round(hb.n_lists * frac_lists)))
        d = hb.as_dict()
        sub = dict(d)
        sub["list_n"] = d["list_n"][:L]
        for k in ("ctrl_off", "data_off", "exc_off", "out_off"):
            sub[k] = d[k][:L + 1]
        sub["total_out"] = int(d["out_off"][L])
        samples.append(sub)
    n_sample = sum(s["total_out"] for s in samples)
    outs = [np.empty(max(s["total_out"], 1), np.uint32) for s in samples]
    reps, t_tot = 0, 0.0
    while reps == 0 or (t_tot < budget_s and reps < 20):
        t0 = time.perf_counter()
        for s, o in zip(samples, outs):
            O.decode_batch(s, dgaps=True, threads=threads, out=o)
        t_tot += time.perf_counter() - t0
        reps += 1
    return n_sample * reps / t_tot, n_sample, reps, t_tot


def run_reference(args, rank, world):
    """--impl reference: the oracle (this tier's reference arm) on the host cores, on the
    headline config: every step decodes, for each variant, the first lists of the batch
    (about 2M ints) encoded by the oracle's own encoder -- no product code on this path."""
    if rank != 0:
        return
    import oracle as O
    O.build()
    if args.config == 0:
        args.config = 5 if world > 1 else 2
    zeta = tuple(int(x) for x in args.pfd_zeta.split("/"))
    w, _, scaling = make_workload(args, 0, 1)
    threads = len(os.sched_getaffinity(0))
    labels, samples = [], []
    for c, v, f, z in config_codecs(args.config, zeta):
        sv, sl = codec_subset(w, c)
        cs = np.cumsum(sl.astype(np.int64))
        nl = max(1, int(np.searchsorted(cs, min(int(cs[-1]) if len(cs) else 0, 2_000_000)) + 1))
        nl = min(nl, len(sl))
        ns = int(cs[nl - 1]) if nl else 0
        samples.append(O.encode_batch(sv[:ns], sl[:nl], c, v, delta=w.delta, frame_quads=f,
                                      zeta=z, threads=threads))
        labels.append(label_of(c, v, f))
    outs = [np.empty(max(int(s["total_out"]), 1), np.uint32) for s in samples]
    n_step = sum(int(s["total_out"]) for s in samples)

    def one_step():
        for smp, o in zip(samples, outs):
            O.decode_batch(smp, dgaps=True, threads=threads, out=o)
    for _ in range(args.warmup):
        one_step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one_step()
    dt = time.perf_counter() - t0
    value = n_step * args.steps / dt
    sample = (f"the first lists (~2M ints) of each of the {len(samples)} variants' batches, "
              f"{n_step} ints per step, encoded by the oracle (gco_encode_batch) and decoded "
              "by gco_decode_batch with the d-gap prefix sum")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "ints/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "config": {"workload": w.name, "n_ints": w.n_ints,
                                        "n_lists": int(len(w.list_n)), "codecs": labels},
        "cpu_baseline": {"kind": "oracle", "cores": threads, "sample": sample, "value": value,
                         "unit": "ints/s"},
        "e2e": {"value": value, "unit": "ints/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_encode(args, dev):
    """--encode: the GPU encoders on the config's inputs resident in HBM:
    config 1 -> Group-Simple (docIDs in), config 2 -> Group-Scheme (all 10 variants),
    config 3 -> Group-PFD and SIMD-BP128, config 4 -> Group-AFOR.  ints/s per codec (gc_encode_device_plan + _write, events on the stream; plan
    reads the stream sizes back, a host sync), with the oracle encoder on the host cores
    beside it (bounded sample)."""
    import torch
    import gen
    import oracle as O
    from paper_1502_01916_b200 import gc
    k = args.config if args.config in (1, 2, 3, 4) else 3
    w = gen.config(k, scale=args.scale)
    zeta = tuple(int(x) for x in args.pfd_zeta.split("/"))
    if k == 2:
        codecs = [(gc.GROUP_SCHEME, gc.gsc_variant(cg, kd)) for cg, kd in gc.GSC_VARIANTS]
    elif k == 3:
        codecs = [(gc.GROUP_PFD, 0), (gc.GROUP_PFD, 1)]
    else:
        codecs = [(gc.GROUP_SIMPLE if k == 1 else gc.GROUP_AFOR, 0)]
    v = torch.from_numpy(w.values.view(np.int32)).to(dev)
    ln = torch.from_numpy(w.list_n.view(np.int32)).to(dev)
    per, tot_ms, tot_bytes = {}, 0.0, 0
    stream = torch.cuda.current_stream(dev)

    def enc(c, var):
        return gc.encode_device(v, ln, c, var, delta=w.delta, frame_quads=32, zeta=zeta)
    for codec, variant in codecs:
        label = gc.codec_label(codec, variant)
        db = enc(codec, variant)
        for _ in range(args.warmup):
            db = enc(codec, variant)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            db = enc(codec, variant)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1) / args.steps
        comp = db.ctrl_bytes + 16 * db.data_vectors + db.exc_bytes
        algo = 4 * w.n_ints + comp  # ints read + streams written
        per[label] = {"ms": round(ms, 4), "ints_per_s": w.n_ints / (ms / 1e3),
                      "gbs": round(algo / (ms / 1e3) / 1e9, 1),
                      "bits_per_int": round(8 * comp / w.n_ints, 3)}
        tot_ms += ms
        tot_bytes += algo
        del db
    peak, peak_src = peaks()
    achieved = tot_bytes / (tot_ms / 1e3) / 1e9
    # the oracle encoder on a bounded sample of the same gaps (its first lists)
    threads = len(os.sched_getaffinity(0))
    cs = np.cumsum(w.list_n.astype(np.int64))
    nl = max(1, int(np.searchsorted(cs, min(int(cs[-1]), 1 << 24))))
    ns = int(cs[nl - 1])
    t0 = time.perf_counter()
    O.encode_batch(w.values[:ns], w.list_n[:nl], codecs[0][0], codecs[0][1], delta=w.delta,
                   zeta=zeta, threads=threads)
    t_cpu = time.perf_counter() - t0
    line = {
        "metric": "encoded uint32 ints/sec (GPU encoders)",
        "value": len(codecs) * w.n_ints / (tot_ms / 1e3), "unit": "ints/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms,
        "higher_is_better": True, "dtype": "u32", "data": "synthetic",
        "config": {"workload": w.name, "n_ints": w.n_ints, "codecs": list(per)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_source": peak_src,
                     "bytes": "4 B per int read + the encoded streams written"},
        "per_codec": per,
        "cpu_baseline": {"kind": "oracle", "value": ns / t_cpu, "unit": "ints/s",
                         "cores": threads,
                         "sample": f"first {nl} lists ({ns} ints), {gc.codec_label(*codecs[0])}, "
                                   "gco_encode_batch (threads split by list)"},
    }
    print(json.dumps(line), flush=True)


def maybe_spawn(args):
    """--gpus N outside torchrun: re-run this script as N ranks (torch.distributed.run,
    127.0.0.1 rendezvous).  Returns True when the ranks ran here (the caller exits)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")            # the communicator's nranks in the log
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    rc = subprocess.call(cmd, env=env)
    if rc:
        sys.exit(rc)
    return True


def oracle_slice_check(db, docs, list_n, seed: int, frac: float = 0.01) -> bool:
    """A contiguous run of about `frac` of a device batch's ints, copied to the host with
    its directory rebased, decoded by the oracle (d-gaps) and compared with `docs`."""
    import oracle as O
    L = len(list_n)
    if L == 0:
        return True
    t = db.tensors
    ln = np.asarray(list_n, np.int64)
    cs = np.cumsum(ln)
    rng = np.random.default_rng(seed)
    a = int(rng.integers(0, L))
    b = int(min(L, np.searchsorted(cs, cs[a] - ln[a] + max(1, int(frac * cs[-1])), side="right") + 1))
    b = max(b, a + 1)
    offs = {k: t[k][a:b + 1].cpu().numpy().view(np.uint64) for k in ("ctrl_off", "data_off", "exc_off", "out_off")}
    sub = {"codec": db.codec, "variant": db.variant, "frame_quads": db.frame_quads,
           "list_n": ln[a:b].astype(np.uint32),
           "ctrl": t["ctrl"][int(offs["ctrl_off"][0]):int(offs["ctrl_off"][-1])].cpu().numpy(),
           "data": t["data"].view(-1, 4)[int(offs["data_off"][0]):int(offs["data_off"][-1])].cpu().numpy().view(np.uint32),
           "exc": t["exc"][int(offs["exc_off"][0]):int(offs["exc_off"][-1])].cpu().numpy()}
    for k, v in offs.items():
        sub[k] = v - v[0]
    sub["total_out"] = int(sub["out_off"][-1])
    want = O.decode_batch(sub, dgaps=True, threads=len(os.sched_getaffinity(0)))
    got = docs[int(offs["out_off"][0]):int(offs["out_off"][-1])].cpu().numpy().view(np.uint32)
    return bool(np.array_equal(got, want))


def time_variants(args, w, codecs, dev, pg, steps, warmup, headline):
    """Encode (host encoder), upload, verify and time every variant of one workload.
    Returns a dict with the per-variant timings and, for the headline, the step timing."""
    import torch
    from paper_1502_01916_b200 import gc
    t_setup = time.perf_counter()
    subs = [codec_subset(w, c) for c, _, _, _ in codecs]
    on_dev = not isinstance(w.values, np.ndarray)
    if on_dev:  # GPU encoders (gc_encode_device_*), byte-identical to the host encoder
        dbs = []
        for (sv, sl), (c, v, f, z) in zip(subs, codecs):
            lt = torch.from_numpy(np.ascontiguousarray(sl).view(np.int32)).to(dev)
            dbs.append(gc.encode_device(sv, lt, c, v, delta=w.delta, frame_quads=f, zeta=z))
            torch.cuda.synchronize(dev)
        hbs = dbs
    else:
        hbs = [gc.encode_batch(sv, sl, c, v, delta=w.delta, frame_quads=f, zeta=z)
               for (sv, sl), (c, v, f, z) in zip(subs, codecs)]
        dbs = [gc.to_device(hb, dev) for hb in hbs]
    n_ints = max(hb.total_out for hb in hbs)
    out = torch.empty(max(n_ints, 4), dtype=torch.int32, device=dev)
    wss = [gc.alloc_workspace(db, dev) for db in dbs]
    stream = torch.cuda.current_stream(dev)
    labels = [gc.codec_label(c, v, f) for c, v, f, _ in codecs]

    # ---- parity gate (untimed): every variant bit-exact against the generator
    verified = None
    if not args.no_verify:
        verified = True
        for lab, db, ws, (sv, sl) in zip(labels, dbs, wss, subs):
            vals = sv if on_dev else torch.from_numpy(np.ascontiguousarray(sv).view(np.int32)).to(dev)
            ln = torch.from_numpy(sl.astype(np.int64)).to(dev)
            starts = torch.cumsum(ln, 0) - ln
            starts = starts[ln > 0]
            if not w.delta:
                gaps, _ = gc.decode(db, out=out, ws=ws)
                ok_g = bool(torch.equal(gaps, vals))
            else:
                ok_g = None
            docs, _ = gc.decode_dgaps(db, out=out, ws=ws)
            st = gc.read_device_status(ws)
            if w.delta:
                ok = bool(torch.equal(docs, vals))
            else:
                g = docs.clone()
                g[1:] = docs[1:] - docs[:-1]
                g[starts] = docs[starts]
                ok = bool(torch.equal(g, vals))
                del g
            if ok and on_dev:
                # the oracle decodes ~1% of the lists (a contiguous run from a seeded start)
                # from the GPU encoder's bytes; its docIDs must equal the GPU's
                ok = oracle_slice_check(db, docs, sl, seed=len(sl))
            if ok_g is False or not ok or st:
                verified = False
                print(f"PARITY FAILURE {w.name} {lab}: gaps={ok_g} docs={ok} status="
                      f"{gc.status_names(st)}", file=sys.stderr)
            del vals
    t_setup = time.perf_counter() - t_setup

    # ---- timed region: K steps x all variants of gc_decode_dgaps (stage events per launch)
    ev = [[tuple(torch.cuda.Event(enable_timing=True) for _ in range(4)) for _ in dbs]
          for _ in range(steps)]
    sides = [torch.cuda.Stream(dev) for _ in range(max(1, args.side_streams))]

    def step(evs=None):
        if args.sched == "serial":
            for i, (db, ws) in enumerate(zip(dbs, wss)):
                if evs is not None:
                    evs[i][0].record(stream)
                gc.decode_stage(db, out, ws, True, gc.STAGE_RESET | gc.STAGE_INDEX, stream)
                if evs is not None:
                    evs[i][1].record(stream)
                    evs[i][2].record(stream)
                gc.decode_stage(db, out, ws, True, gc.STAGE_DECODE, stream)
                if evs is not None:
                    evs[i][3].record(stream)
            return
        # overlap: the variants' index stages (each on its own workspace) run on a side
        # stream, ahead of and concurrently with the decodes; variant i's decode waits for
        # its own index stage only
        for side in sides:
            side.wait_stream(stream)  # the previous step's decodes are done with the workspaces
        done = []
        for i, (db, ws) in enumerate(zip(dbs, wss)):
            side = sides[i % len(sides)]
            if evs is not None:
                evs[i][0].record(side)
            gc.decode_stage(db, out, ws, True, gc.STAGE_RESET | gc.STAGE_INDEX, side)
            e = evs[i][1] if evs is not None else torch.cuda.Event()
            e.record(side)
            done.append(e)
        for i, (db, ws) in enumerate(zip(dbs, wss)):
            stream.wait_event(done[i])
            if evs is not None:
                evs[i][2].record(stream)
            gc.decode_stage(db, out, ws, True, gc.STAGE_DECODE, stream)
            if evs is not None:
                evs[i][3].record(stream)
        for side in sides:
            stream.wait_stream(side)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize(dev)
    # a working set that fits in L2 is flushed before every timed step (a scratch write of
    # 4x the L2), and only the steps are timed; larger ones need no flush
    l2_bytes = int(getattr(torch.cuda.get_device_properties(dev), "L2_cache_size", 126 << 20))
    algo_ws = [hb.compressed_bytes + 4 * hb.total_out + hb.directory_bytes for hb in hbs]
    flush = torch.empty(4 * l2_bytes, dtype=torch.uint8, device=dev) if max(algo_ws) < l2_bytes else None
    step_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps)]
    clk = ClockSampler(torch.cuda.current_device()) if headline else None
    if pg:
        pg.barrier()
    torch.cuda.synchronize(dev)
    if clk:
        clk.__enter__()
    for k in range(steps):
        if flush is not None:
            flush.fill_(k & 0xFF)
        if pg:  # every rank starts the step together (the per-step barrier)
            torch.cuda.synchronize(dev)
            pg.barrier()
        step_ev[k][0].record(stream)
        step(ev[k])
        step_ev[k][1].record(stream)
    torch.cuda.synchronize(dev)
    if clk:
        clk.__exit__()
    if pg:
        pg.barrier()
    torch.cuda.synchronize(dev)
    ms = sum(a.elapsed_time(b) for a, b in step_ev)  # (the steps only)
    small_extra = None
    if flush is not None:  # L2-warm and CUDA-graph numbers, labelled
        w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0.record(stream)
        for _ in range(steps):
            step()
        w1.record(stream)
        torch.cuda.synchronize(dev)
        small_extra = {"l2_warm_ms_per_step": w0.elapsed_time(w1) / steps}
        try:
            def serial_step():  # the same stages on the capturing stream
                for db, ws in zip(dbs, wss):
                    gc.decode_stage(db, out, ws, True, gc.STAGE_RESET | gc.STAGE_INDEX, None)
                    gc.decode_stage(db, out, ws, True, gc.STAGE_DECODE, None)
            graph = torch.cuda.CUDAGraph()
            side_cap = torch.cuda.Stream(dev)
            side_cap.wait_stream(stream)
            with torch.cuda.stream(side_cap):
                serial_step()  # (warm on the capture stream)
            torch.cuda.synchronize(dev)
            with torch.cuda.graph(graph):
                serial_step()
            torch.cuda.synchronize(dev)
            graph.replay()
            torch.cuda.synchronize(dev)
            w0.record(stream)
            for _ in range(steps):
                graph.replay()
            w1.record(stream)
            torch.cuda.synchronize(dev)
            small_extra["cuda_graph_l2_warm_ms_per_step"] = w0.elapsed_time(w1) / steps
        except Exception as e:  # noqa: BLE001
            small_extra["cuda_graph"] = f"capture failed: {e}"[:200]
    dec_ms = [sum(ev[k][i][2].elapsed_time(ev[k][i][3]) for k in range(steps)) / steps
              for i in range(len(dbs))]
    idx_ms = [sum(ev[k][i][0].elapsed_time(ev[k][i][1]) for k in range(steps)) / steps
              for i in range(len(dbs))]
    step_ms = sorted(a.elapsed_time(b) for a, b in step_ev)

    # ---- gc_decode (gaps only, the paper's measured path, A38) beside it
    gaps_ms = []
    for db, ws in zip(dbs, wss):
        gc.decode_stage(db, out, ws, False, gc.STAGE_RESET | gc.STAGE_INDEX, stream)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        gc.decode_stage(db, out, ws, False, gc.STAGE_DECODE, stream)  # (warm)
        g0.record(stream)
        for _ in range(steps):
            gc.decode_stage(db, out, ws, False, gc.STAGE_DECODE, stream)
        g1.record(stream)
        torch.cuda.synchronize(dev)
        gaps_ms.append(g0.elapsed_time(g1) / steps)

    # ---- parity after timing: device status and the G7 checksum of every variant
    status = 0
    chk = np.zeros(3, np.uint64)
    for db, ws in zip(dbs, wss):
        docs, _ = gc.decode_dgaps(db, out=out, ws=ws)
        status |= gc.read_device_status(ws)
        chk += gc.checksum(db, docs, list_base=w.list_base).cpu().numpy().view(np.uint64)
    peak, _ = peaks()
    algo = [hb.compressed_bytes + 4 * hb.total_out for hb in hbs]
    per = {}
    for lab, hb, a, dm, im, gm in zip(labels, hbs, algo, dec_ms, idx_ms, gaps_ms):
        per[lab] = {
            "config": w.name, "n_ints": hb.total_out,
            "ints_per_s": hb.total_out / ((dm + im) / 1e3),
            "decode_kernel_ms": round(dm, 5), "index_ms": round(im, 5),
            "bits_per_int": round(8 * hb.compressed_bytes / max(hb.total_out, 1), 3),
            "algorithmic_bytes": a,
            "decode_kernel_gbs": round(a / (dm / 1e3) / 1e9, 1),
            "frac_of_peak": round(a / (dm / 1e3) / 1e9 / peak, 3),
            "gaps_only_decode_kernel_ms": round(gm, 5),
            "gaps_only_frac_of_peak": round(a / (gm / 1e3) / 1e9 / peak, 3),
            "traffic": ncu_traffic(w.name, lab),
        }
        if flush is not None:
            per[lab]["l2"] = "flushed before every timed step"
    res = dict(w=w, hbs=hbs, labels=labels, per=per, algo=algo, dec_ms=dec_ms, gaps_ms=gaps_ms,
               ms=ms, step_ms=step_ms, n_ints=n_ints, n_ints_all=sum(hb.total_out for hb in hbs),
               verified=verified, status=status, chk=chk, small_extra=small_extra, clk=clk,
               t_setup=t_setup, flush=flush is not None, l2_bytes=l2_bytes, algo_ws=algo_ws)
    del dbs, wss, out
    torch.cuda.empty_cache()
    return res


def run_random_access(args, dev):
    """--random-access: gc_decode_range from the skip pointers (§7.5, SURVEY §8(f)
    rank 4) on the headline config's variants: (a) the whole batch as one range -- every
    512-int block decoded on its own from its entry, no index stage, no look-back -- with its
    roofline (compressed + skip-table bytes read, 4 B per int written); (b) single 512-int
    block ranges at random positions, one call each: microseconds per call."""
    import torch
    from paper_1502_01916_b200 import gc
    zeta = tuple(int(x) for x in args.pfd_zeta.split("/"))
    w, _, _ = make_workload(args, 0, 1)
    peak, peak_src = peaks()
    per, tot_b, tot_ms, tot_n = {}, 0, 0.0, 0
    stream = torch.cuda.current_stream(dev)
    rng = np.random.default_rng(11)
    for c, v, f, z in config_codecs(args.config, zeta):
        if c == gc.VARBYTE:
            continue
        lab = gc.codec_label(c, v, f)
        hb = gc.encode_batch(*codec_subset(w, c), c, v, delta=w.delta, frame_quads=f, zeta=z)
        db = gc.to_device(hb, dev)
        docs, ws = gc.decode_dgaps(db)
        want = docs.clone()
        off, ent = gc.build_skip(db, docs, ws=ws)
        n_ent = int(off[-1].item())
        out = torch.empty_like(docs)
        rws = torch.empty(256, dtype=torch.uint8, device=dev)
        N = hb.total_out
        for _ in range(args.warmup):
            gc.decode_range(db, off, ent, out, 0, N, True, ws=rws)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            gc.decode_range(db, off, ent, out, 0, N, True, ws=rws)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1) / args.steps
        ok = bool(torch.equal(out, want)) and gc.read_device_status(rws) == 0
        algo = hb.compressed_bytes + 4 * N + 32 * n_ent
        # single blocks: 200 random 512-int ranges, one call each
        firsts = rng.integers(0, max(1, N - 512), 200)
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record(stream)
        for fi in firsts:
            gc.decode_range(db, off, ent, out, int(fi), min(512, N - int(fi)), True, ws=rws)
        b1.record(stream)
        torch.cuda.synchronize(dev)
        us_block = 1e3 * b0.elapsed_time(b1) / len(firsts)
        per[lab] = {"whole_batch_ms": round(ms, 5), "ints_per_s": N / (ms / 1e3),
                    "gbs": round(algo / (ms / 1e3) / 1e9, 1),
                    "frac_of_peak": round(algo / (ms / 1e3) / 1e9 / peak, 3),
                    "skip_entries": n_ent, "skip_bytes_per_int": round(32 * n_ent / max(N, 1), 4),
                    "one_block_us_per_call": round(us_block, 2), "verified": ok}
        tot_b += algo
        tot_ms += ms
        tot_n += N
        del db, docs, want, out, off, ent, ws
        torch.cuda.empty_cache()
    achieved = tot_b / (tot_ms / 1e3) / 1e9
    line = {"metric": "decoded uint32 ints/sec from the skip pointers (gc_decode_range)",
            "value": tot_n / (tot_ms / 1e3), "unit": "ints/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms, "higher_is_better": True,
            "dtype": "u32", "data": "synthetic",
            "config": {"workload": w.name, "codecs": list(per),
                       "path": "gc_decode_range(0, N) per variant: one warp per 512-int block"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_source": peak_src, "kernel": "k_range",
                         "bytes": "compressed streams + 32 B per skip entry read, 4 B per int written"},
            "per_codec": per}
    print(json.dumps(line), flush=True)


def run_posting_store(args, dev):
    """--posting-store: §7.5's store (lists shorter than 64: Variable Byte) of the
    headline config's lists with a term frequency per posting (seeded Geometric(0.4) draws,
    a stand-in: the corpora are absent), every Group-Scheme variant in turn (config 2) or the
    config's codecs: gc_decode_posting_store -- the long group's docIDs and TFs in ONE fused
    k_decode pass -- against the same store decoded by separate calls (gc_decode_dgaps of
    the docIDs, gc_decode of the TFs, and the Variable Byte groups), both with their index
    stages; the outputs are compared."""
    import torch
    from paper_1502_01916_b200 import gc
    zeta = tuple(int(x) for x in args.pfd_zeta.split("/"))
    w, _, _ = make_workload(args, 0, 1)
    rng = np.random.default_rng(2024)
    tfs = (rng.geometric(0.4, w.n_ints) % 65536).astype(np.uint32)
    stream = torch.cuda.current_stream(dev)
    per, tot_f, tot_s, n_tot = {}, 0.0, 0.0, 0
    for c, v, f, z in config_codecs(args.config, zeta):
        if c == gc.VARBYTE:
            continue
        lab = gc.codec_label(c, v, f)
        st = gc.encode_posting_store(w.values, w.list_n, c, v, delta=w.delta, tfs=tfs,
                                     frame_quads=f, zeta=z)
        parts = [gc.to_device(b, dev) for b in (st.long, st.tf_long, st.short, st.tf_short)]
        out_d = torch.empty(max(st.total, 4), dtype=torch.int32, device=dev)
        out_t = torch.empty_like(out_d)
        wss = [gc.alloc_workspace(p, dev) for p in parts]

        def separate():
            gc.decode_dgaps(parts[0], out=out_d, ws=wss[0])
            gc.decode(parts[1], out=out_t, ws=wss[1])
            if st.short.total_out:
                gc.decode_dgaps(parts[2], out=out_d[st.short_base:], ws=wss[2])
                gc.decode(parts[3], out=out_t[st.short_base:], ws=wss[3])

        def fused():
            return gc.decode_posting_store(st, dgaps=True, device=dev)
        d_f, t_f, fw = fused()
        separate()
        torch.cuda.synchronize(dev)
        ok = bool(torch.equal(d_f, out_d[:st.total])) and bool(torch.equal(t_f, out_t[:st.total]))
        ok = ok and all(gc.read_device_status(x) == 0 for x in fw)
        # time the decode calls only (the device batches of the fused path are uploaded once)
        from paper_1502_01916_b200.gc import CPostingStore, _lib, _stream_ptr
        import ctypes as C
        cs = [p.cstruct() for p in parts]
        cst = CPostingStore(cs[0], cs[2], C.pointer(cs[1]), C.pointer(cs[3]), st.short_base)
        need = C.c_uint64()
        _lib().gc_posting_store_ws_size(C.byref(cst), C.byref(need))
        fws = torch.empty(int(need.value), dtype=torch.uint8, device=dev)

        def fused_call():
            r = _lib().gc_decode_posting_store(C.byref(cst), out_d.data_ptr(), out_t.data_ptr(), 1,
                                               fws.data_ptr(), fws.numel(), _stream_ptr(None))
            assert r == 0
        times = {}
        for name, fn in (("fused", fused_call), ("separate", separate)):
            for _ in range(args.warmup):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                fn()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            times[name] = e0.elapsed_time(e1) / args.steps
        n = 2 * (st.long.total_out + st.short.total_out)
        per[lab] = {"fused_ms": round(times["fused"], 5), "separate_ms": round(times["separate"], 5),
                    "speedup": round(times["separate"] / times["fused"], 3),
                    "fused_ints_per_s": n / (times["fused"] / 1e3), "verified": ok,
                    "short_lists": int(st.short.n_lists), "long_lists": int(st.long.n_lists)}
        tot_f += times["fused"]
        tot_s += times["separate"]
        n_tot += n
        del parts, out_d, out_t, wss, fws, d_f, t_f, fw
        torch.cuda.empty_cache()
    line = {"metric": "decoded uint32 ints/sec of a posting store (docIDs + TFs, §7.5)",
            "value": n_tot / (tot_f / 1e3), "unit": "ints/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_f, "higher_is_better": True, "dtype": "u32",
            "data": "synthetic (TFs: seeded Geometric(0.4) per posting)",
            "config": {"workload": w.name, "codecs": list(per), "threshold": 64,
                       "path": "gc_decode_posting_store (index stages + fused docID/TF k_decode + "
                               "Variable Byte) vs separate gc_decode_dgaps / gc_decode calls"},
            "fused_vs_separate": {"fused_ms": tot_f, "separate_ms": tot_s, "speedup": tot_s / tot_f},
            "per_codec": per}
    print(json.dumps(line), flush=True)


def spawn_check(rank, world):
    """--spawn-check: the rank plumbing alone (gloo on CPU, NCCL on GPUs): every rank
    all-reduces its rank id; rank 0 prints {"world", "rank_sum"}."""
    import torch
    import torch.distributed as dist
    backend = "nccl" if torch.cuda.is_available() else "gloo"
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0"))) if backend == "nccl" else None
    if dev is not None:
        torch.cuda.set_device(dev)
    dist.init_process_group(backend)
    t = torch.tensor([rank], dtype=torch.int64, device=dev)
    dist.all_reduce(t)
    dist.barrier()
    if rank == 0:
        print(json.dumps({"spawn_check": True, "world": world, "rank_sum": int(t.item()),
                          "backend": backend}), flush=True)
    dist.destroy_process_group()


def main():
    args = parse_args()
    if maybe_spawn(args):
        return
    rank, local_rank, world = dist_info()
    if args.spawn_check:
        spawn_check(rank, world)
        return
    if args.config == 0:
        args.config = 5 if world > 1 else 2
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.encode or args.random_access or args.posting_store:
        import torch
        from paper_1502_01916_b200 import build
        build.build()
        torch.cuda.set_device(local_rank)
        if rank == 0:
            fn = run_encode if args.encode else (run_random_access if args.random_access else run_posting_store)
            fn(args, torch.device("cuda", local_rank))
        return
    import torch
    from paper_1502_01916_b200 import build
    if local_rank == 0:
        build.build()
    from paper_1502_01916_b200 import gc

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    pg = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=dev)
        pg = dist
        pg.barrier()  # (local rank 0 has built libgc.so)
    else:
        build.build()
    zeta = tuple(int(x) for x in args.pfd_zeta.split("/"))
    codecs = config_codecs(args.config, zeta)
    if args.codecs:
        keep = set(args.codecs.split(","))
        codecs = [c for c in codecs if gc.codec_label(c[0], c[1], c[2]) in keep]

    w, list_base, scaling = make_workload(args, rank, world, device=dev)
    w.list_base = list_base
    R = time_variants(args, w, codecs, dev, pg, args.steps, args.warmup, headline=True)
    hbs, labels, algo, dec_ms = R["hbs"], R["labels"], R["algo"], R["dec_ms"]
    ms, n_ints, n_ints_all = R["ms"], R["n_ints"], R["n_ints_all"]

    # ---- the other single-GPU configs at full size, for per_codec (not in `value`)
    extra = args.extra_configs
    if extra == "auto":
        extra = "1,3,4" if (world == 1 and args.config == 2 and not args.codecs
                            and args.scale == 1.0) else "none"
    per_codec = dict(R["per"])
    extra_cfgs = [] if extra == "none" else [int(x) for x in extra.split(",")]
    for k in extra_cfgs:
        import gen
        wk = gen.config(k)
        wk.list_base = 0
        Rk = time_variants(args, wk, config_codecs(k, zeta), dev, None,
                           max(3, min(args.steps, 20)), max(3, args.warmup), headline=False)
        per_codec.update(Rk["per"])
        R["verified"] = None if R["verified"] is None else bool(R["verified"] and Rk["verified"])
        R["status"] |= Rk["status"]
        del Rk

    # ---- NCCL: max time over ranks; sum of counts / checksums / status (after timing)
    from paper_1502_01916_b200 import dist as gdist
    ms, total_ints, status, all_verified, chk = gdist.reduce_run(
        pg, dev, ms, int(n_ints_all), R["status"], R["verified"], R["chk"])
    if rank != 0:
        if pg:
            pg.destroy_process_group()
        return

    ints_per_step_all = total_ints
    value = ints_per_step_all * args.steps / (ms / 1e3)
    # ---- roofline of the dominant kernel (k_decode, the headline's variants): algorithmic
    # bytes = compressed stream bytes + 4 B per decoded int; directory excluded.
    achieved = sum(algo) / (sum(dec_ms) / 1e3) / 1e9
    peak, peak_src = peaks()
    gaps_achieved = sum(algo) / (sum(R["gaps_ms"]) / 1e3) / 1e9
    tr = [per_codec[lab]["traffic"] for lab in labels]
    traffic = (sum(t["bytes_per_launch"] for t in tr) / len(tr)
               if tr and all(t is not None for t in tr) else None)

    # a device-resident workload (config 5 drawn on the GPU) times e2e and the CPU baseline
    # on host batches of its first lists (the host encoder), labelled as a sample
    host_sample = None
    if not isinstance(w.values, np.ndarray) and not (args.no_e2e and args.no_cpu_baseline):
        ln64 = w.list_n.astype(np.int64)
        nl = max(1, int(np.searchsorted(np.cumsum(ln64), 1 << 24)))
        ns = int(ln64[:nl].sum())
        hv = w.values[:ns].cpu().numpy().view(np.uint32)

        class _W:
            values, list_n, delta = hv, w.list_n[:nl], w.delta
        hbs = [gc.encode_batch(*codec_subset(_W, c), c, v, delta=w.delta, frame_quads=f, zeta=z)
               for c, v, f, z in codecs]
        n_ints = max(hb.total_out for hb in hbs)
        n_ints_all = sum(hb.total_out for hb in hbs)
        host_sample = f"the shard's first {nl} lists ({ns} ints), host-encoded"
    # ---- e2e through the C ABI from pinned HOST buffers (copies inside the timed region)
    e2e = None
    if not args.no_e2e:
        pinned = []
        for hb in hbs:
            def pin(a):
                t = torch.empty(a.nbytes, dtype=torch.uint8, pin_memory=True)
                v = t.numpy().view(a.dtype).reshape(a.shape)
                v[...] = a
                return t, v
            keep, fields = [], {}
            for k in ("list_n", "ctrl_off", "data_off", "exc_off", "out_off", "ctrl", "data", "exc"):
                t, v = pin(getattr(hb, k))
                keep.append(t)
                fields[k] = v
            phb = gc.HostBatch(hb.codec, hb.variant, hb.frame_quads, **fields)
            pinned.append((phb, keep))
        # two streams, each with its own device scratch and pinned output: batch i+1's
        # host->device copies overlap batch i's decode and device->host copy (PCIe is full
        # duplex; each gc_decode_host call is itself ordered on its stream)
        n_pipe = 2 if len(pinned) > 1 else 1
        host_outs, scratches = [], []
        for _ in range(n_pipe):
            t = torch.empty(max(n_ints, 4) * 4, dtype=torch.uint8, pin_memory=True)
            host_outs.append((t, t.numpy().view(np.uint32)[:n_ints]))
            scratches.append(torch.empty(max(gc.host_scratch_size(p) for p, _ in pinned),
                                         dtype=torch.uint8, device=dev))
        torch.cuda.empty_cache()
        pipes = [torch.cuda.Stream(dev) for _ in range(n_pipe)]
        stream = torch.cuda.current_stream(dev)

        def e2e_step():
            for i, (phb, _) in enumerate(pinned):
                k = i % n_pipe
                gc.decode_host(phb, host_outs[k][1], True, scratches[k], pipes[k])
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2e_step()  # (untimed warm-up)
        torch.cuda.synchronize(dev)
        a0.record(stream)
        for ps in pipes:
            ps.wait_event(a0)
        for _ in range(args.e2e_steps):
            e2e_step()
        for ps in pipes:
            stream.wait_stream(ps)
        a1.record(stream)
        torch.cuda.synchronize(dev)
        ems = a0.elapsed_time(a1)
        h2d = sum(p.directory_bytes + len(p.ctrl) + 16 * len(p.data) + len(p.exc) for p, _ in pinned)
        e2e = {"value": n_ints_all * args.e2e_steps / (ems / 1e3), "unit": "ints/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(4 * n_ints_all),
               "steps": args.e2e_steps, "ms_per_step": ems / args.e2e_steps,
               "api": "gc_decode_host (pinned host buffers, batches alternating over 2 streams)"}
        if host_sample:
            e2e["sample"] = host_sample

    cpu = None
    if not args.no_cpu_baseline:
        import oracle as O
        O.build()
        threads = len(os.sched_getaffinity(0))
        frac = min(1.0, 8.0e6 / max(1, n_ints))
        rate, n_sample, reps, t_cpu = cpu_oracle_rate(hbs, frac, 10.0, threads)
        rate1, n1, reps1, t1c = cpu_oracle_rate(hbs, frac / 8, 2.0, 1)
        cpu = {"value": rate, "unit": "ints/s", "cores": threads, "kind": "oracle",
               "sample": f"first {frac:.4f} of the lists of all {len(hbs)} batches "
                         f"({n_sample} ints), {reps} rep(s), {t_cpu:.1f} s, gco_decode_batch "
                         "with the d-gap prefix sum",
               "value_1_thread": rate1,
               "sample_1_thread": f"first {frac / 8:.4f} of the lists ({n1} ints), {reps1} rep(s)"}

    step_ms = R["step_ms"]
    l2_bytes, algo_ws = R["l2_bytes"], R["algo_ws"]
    line = {
        "metric": METRIC, "value": value, "unit": "ints/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "u32",
        "data": "synthetic",
        "config": {"workload": w.name, "n_ints_per_gpu": w.n_ints, "n_lists_per_gpu": int(len(w.list_n)),
                   "codecs": labels, "ints_per_step_all_gpus": ints_per_step_all,
                   "value_is": f"{w.name}: every variant of the config, one step = each decoded once",
                   "per_codec_extra_configs": [f"cfg{k}" for k in extra_cfgs],
                   "parallelism": f"dp{world} (lists sharded by rank, {scaling} scaling)",
                   "l2": (f"flushed before every timed step (scratch write of {4 * l2_bytes >> 20} MB; "
                          f"working set {max(algo_ws) / 1e6:.1f} MB < the {l2_bytes >> 20} MB L2), "
                          "steps timed without the flush" if R["flush"] else
                          "no flush: every variant's working set "
                          f"({min(algo) / 1e6:.0f}-{max(algo) / 1e6:.0f} MB) exceeds the "
                          f"{l2_bytes >> 20} MB L2"),
                   "path": "gc_decode_dgaps (index scan + fused decode/d-gap scan)",
                   "schedule": (f"index stages on {args.side_streams} side stream(s), concurrent with the decodes "
                                "(each variant's decode waits for its own index stage; "
                                "per-variant index_ms then includes queueing)"
                                if args.sched == "overlap" else
                                "serial: index then decode, variant by variant")},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "traffic_source": ("profiles/r2_traffic.json: dram__bytes_read.sum + "
                                        "lts__t_sectors_srcunit_tex_op_write.sum x 32 B per k_decode "
                                        "launch, ncu --set full, mean over the headline variants"),
                     "kernel": "k_decode (the headline's variants)", "algorithmic_bytes_per_step": sum(algo),
                     "frac_of_nominal_8tbs": achieved / 8000.0,
                     "gaps_only": {"achieved": gaps_achieved, "frac": gaps_achieved / peak,
                                   "path": "gc_decode (no d-gap scan), the paper's measured path"}},
        "step_ms": {"mean": ms / args.steps, "median": step_ms[len(step_ms) // 2],
                    "min": step_ms[0], "max": step_ms[-1]},
        "small_workload": R["small_extra"],
        "per_codec": per_codec,
        "cpu_baseline": cpu,
        "e2e": e2e,
        # per variant per step: k_lists + k_index (GC_STAGE_INDEX) and k_decode (GC_STAGE_DECODE)
        "gpu_launches": 3 * len(hbs) * args.steps,
        "clocks": R["clk"].summary() if R["clk"] else None,
        "parity": {"verified": all_verified, "device_status": status,
                   "checksum": [int(x) for x in chk]},
        "setup_s": round(R["t_setup"], 1),
    }
    print(json.dumps(line), flush=True)
    if pg:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()

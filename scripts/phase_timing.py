"""Per-phase cycle breakdown of k_decode (build with -DGC_TIMING; debugging aid)."""
import os, sys, ctypes
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
from paper_1502_01916_b200 import gc
NAMES = ["loop top", "list table+ctrl wait", "parse+scan", "emit+unpack (+data wait)",
         "staging barrier+setup", "d-gap scan", "stores", "end barrier", "deferred carry (look-back)"]
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
labels = sys.argv[2].split(",") if len(sys.argv) > 2 else ["GSC-8-B"]
w = gen.config(cfg)
for lab in labels:
    codec, variant = {"G-SIM": (2, 0), "G-AFOR": (4, 0), "G-PFD": (5, 0)}.get(lab, (3, None))
    if variant is None:
        cg, kind = lab.split("-")[1:]
        variant = gc.gsc_variant(int(cg), kind)
    hb = gc.encode_batch(w.values, w.list_n, codec, variant, delta=w.delta)
    db = gc.to_device(hb)
    out, ws = gc.decode_dgaps(db)
    torch.cuda.synchronize()
    prof = ws[64:64 + 24 * 8].clone()
    out, ws = gc.decode_dgaps(db, out=out, ws=ws)
    torch.cuda.synchronize()
    pa = ws[64:64 + 24 * 8].cpu().numpy().view(np.uint64)
    p = pa[:9].astype(np.float64)
    print(f"   look-backs {pa[12]} windows {pa[13]} spins {pa[14]} (tiles {(hb.total_out + 8191) // 8192})"
          f"  spin distance 1:{pa[15]} 2-4:{pa[16]} 5-16:{pa[17]} 17-128:{pa[18]} >128:{pa[19]}")

    tot = p.sum()
    print(f"   look-back cycles {100 * pa[20] / tot:.1f}% of the total")
    print(f"== {lab} cfg{cfg}: total {tot:.3e} cycles (thread 0 of every CTA, summed)")
    for n, v in zip(NAMES, p):
        print(f"   {n:22s} {100 * v / tot:5.1f}%")

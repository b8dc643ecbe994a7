"""Decode one scaled config on the GPU and print mismatching tiles (debugging aid)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
import oracle as O
from paper_1502_01916_b200 import gc
cfg, scale, lab = int(sys.argv[1]), float(sys.argv[2]), sys.argv[3]
codec, variant = {"G-SIM": (2, 0), "G-AFOR": (4, 0), "G-PFD": (5, 0)}.get(lab, (3, None))
if variant is None:
    cg, kind = lab.split("-")[1:]
    variant = gc.gsc_variant(int(cg), kind)
w = gen.config(cfg, scale=scale)
hb = gc.encode_batch(w.values, w.list_n, codec, variant, delta=w.delta)
want = O.decode_batch(hb.as_dict(), dgaps=True)
db = gc.to_device(hb)
for it in range(2):
    out, ws = gc.decode_dgaps(db)
    torch.cuda.synchronize()
    got = out.cpu().numpy().view(np.uint32)
    bad = np.nonzero(got != want)[0]
    print("run", it, "status", gc.read_device_status(ws), "bad", len(bad), "of", len(want))
    T = 8192
    tiles = np.unique(bad // T)
    for t in tiles[:12]:
        b = bad[(bad // T) == t] - t * T
        d = (got[t * T + b] - want[t * T + b]).astype(np.int64)
        print(f"  tile {t}: {len(b)} bad, positions {b.min()}..{b.max()}, diff values {np.unique(d)[:4]}")

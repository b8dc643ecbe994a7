"""Decode several codecs of one scaled config in sequence (like bench.py) and report
mismatching tiles (debugging aid)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
import oracle as O
from paper_1502_01916_b200 import gc
cfg, scale = int(sys.argv[1]), float(sys.argv[2])
w = gen.config(cfg, scale=scale)
for cg, kind in gc.GSC_VARIANTS[:4]:
    hb = gc.encode_batch(w.values, w.list_n, 3, gc.gsc_variant(cg, kind), delta=w.delta)
    want = O.decode_batch(hb.as_dict(), dgaps=True)
    db = gc.to_device(hb)
    out = torch.empty(max(hb.total_out, 4), dtype=torch.int32, device="cuda")
    ws = gc.alloc_workspace(db, "cuda")
    for it in range(3):
        gc.decode(db, out=out, ws=ws)
        gc.decode_dgaps(db, out=out, ws=ws)
        torch.cuda.synchronize()
        got = out.cpu().numpy().view(np.uint32)[:hb.total_out]
        bad = np.nonzero(got != want)[0]
        T = 8192
        tiles = np.unique(bad // T)
        print(gc.codec_label(3, gc.gsc_variant(cg, kind)), "run", it, "bad", len(bad), "tiles", tiles[:8])
        for t in tiles[:3]:
            b = bad[(bad // T) == t] - t * T
            print(f"    tile {t}: {len(b)} bad, positions {b.min()}..{b.max()}")

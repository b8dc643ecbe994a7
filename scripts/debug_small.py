"""Decode small hand-made batches on the GPU and print mismatches (debugging aid)."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import oracle as O
from paper_1502_01916_b200 import gc, build
build.build()
cases = [("n5", np.array([5], np.uint32), np.array([1, 2, 3, 4, 5], np.uint32)),
         ("n9", np.array([9], np.uint32), np.arange(1, 10, dtype=np.uint32)),
         ("two", np.array([5, 6], np.uint32), np.arange(1, 12, dtype=np.uint32)),
         ("big", np.array([20000], np.uint32), (np.arange(20000) % 1000 + 1).astype(np.uint32))]
for codec, variant in [(O.GROUP_SIMPLE, 0), (O.GROUP_SCHEME, O.gsc_variant(8, "B")), (O.GROUP_SCHEME, O.gsc_variant(1, "CU"))]:
    for name, ln, vals in cases:
        hb = gc.HostBatch.from_dict(O.encode_batch(vals, ln, codec, variant))
        db = gc.to_device(hb)
        out, ws = gc.decode(db)
        torch.cuda.synchronize()
        got = out.cpu().numpy().view(np.uint32)
        bad = np.nonzero(got != vals)[0]
        print(gc.codec_label(codec, variant), name, "status", gc.read_device_status(ws), "bad", len(bad),
              bad[:8], got[bad[:8]], vals[bad[:8]])

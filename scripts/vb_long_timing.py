"""Variable Byte long-list decode time (byte-space tiles): one list of 2^27 geometric d-gaps
and 2^27 ints in 2^17 lists of 1024, gc_decode_dgaps timed with CUDA events; the result is
checked against the generator's docIDs."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1502_01916_b200 import build, gc
import oracle as O

build.build()
rng = np.random.default_rng(5)
for ln in (np.array([1 << 27], np.uint32), np.full(1 << 17, 1024, np.uint32)):
    gaps = rng.geometric(0.05, int(ln.sum())).astype(np.uint64)
    starts = np.concatenate([[0], np.cumsum(ln.astype(np.int64))[:-1]])
    docs = np.cumsum(gaps)
    docs -= np.repeat(docs[starts] - gaps[starts], ln.astype(np.int64))
    docs = (docs % (1 << 32)).astype(np.uint32)
    hb = gc.encode_batch(docs, ln, O.VARBYTE, 0, delta=True)
    db = gc.to_device(hb)
    out, ws = gc.decode_dgaps(db)
    torch.cuda.synchronize()
    ok = gc.read_device_status(ws) == 0 and np.array_equal(out.cpu().numpy().view(np.uint32), docs)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        gc.decode_dgaps(db, out=out, ws=ws)
    e0.record()
    for _ in range(10):
        gc.decode_dgaps(db, out=out, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    n = int(ln.sum())
    byts = hb.compressed_bytes + 4 * n
    print(f"lists={len(ln)} ints={n} bytes/int={hb.compressed_bytes / n:.2f} ms={ms:.3f} "
          f"ints/s={n / ms * 1e3:.3e} GB/s={byts / ms / 1e6:.0f} verified={ok}")

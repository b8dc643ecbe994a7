"""Small decodes of every codec instantiation for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck): both paths, the range decode, the host path, the posting store and
malformed streams; every clean result is checked against the oracle.

  compute-sanitizer --tool memcheck python scripts/sanitize_decode.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import oracle as O  # noqa: E402
from paper_1502_01916_b200 import gc  # noqa: E402

CODECS = ([(O.VARBYTE, 0), (O.GROUP_SIMPLE, 0)] +
          [(O.GROUP_SCHEME, O.gsc_variant(cg, k)) for cg, k in gc.GSC_VARIANTS] +
          [(O.GROUP_AFOR, 0), (O.GROUP_PFD, 0), (O.GROUP_PFD, 1)])


def main():
    rng = np.random.default_rng(77)
    n_checked = 0
    # ragged lists spanning several tiles, 1-int lists, empty lists, one long list
    shapes = [gen.random_lists(rng, 300, 900, 14, 0.02),
              gen.random_lists(rng, 2, 40000, 9, 0.01)]
    ln = np.array([0, 1, 3, 0, 4097, 1, 0, 8191, 2], np.uint32)
    shapes.append(gen.Workload("edges", ln, rng.integers(0, 1 << 20, int(ln.sum())).astype(np.uint32),
                               False, 0))
    for codec, variant in CODECS:
        for w in shapes:
            ref = O.encode_batch(w.values, w.list_n, codec, variant)
            hb = gc.HostBatch.from_dict(ref)
            db = gc.to_device(hb)
            for dgaps in (True, False):
                out, ws = (gc.decode_dgaps if dgaps else gc.decode)(db)
                torch.cuda.synchronize()
                want = O.decode_batch(ref, dgaps=dgaps)
                got = out[:hb.total_out].cpu().numpy().view(np.uint32)
                assert gc.read_device_status(ws) == 0 and np.array_equal(got, want), (codec, variant)
                n_checked += 1
                if codec != O.VARBYTE and hb.total_out > 10:
                    if dgaps:  # the skip table from this d-gap decode, then a range from it
                        off, ent = gc.build_skip(db, out)
                    r = torch.full((hb.total_out,), -1, dtype=torch.int32, device="cuda")
                    rws = gc.decode_range(db, off, ent, r, 5, hb.total_out // 2, dgaps)
                    torch.cuda.synchronize()
                    assert gc.read_device_status(rws) == 0
                    assert np.array_equal(r[5:5 + hb.total_out // 2].cpu().numpy().view(np.uint32),
                                          want[5:5 + hb.total_out // 2])
        # a malformed stream: status bits, no fault
        hb = gc.HostBatch.from_dict(O.encode_batch(shapes[0].values, shapes[0].list_n, codec, variant))
        hb.ctrl = hb.ctrl.copy()
        hb.ctrl[: min(64, len(hb.ctrl))] = 0xFF
        out, ws = gc.decode_dgaps(gc.to_device(hb))
        torch.cuda.synchronize()
        gc.read_device_status(ws)
    # the host path and the posting store
    w = gen.config(5, scale=2 ** -15)
    hb = gc.encode_batch(w.values, w.list_n, O.GROUP_SCHEME, O.gsc_variant(8, "IU"), delta=True)
    host = np.zeros(hb.total_out, np.uint32)
    scratch = torch.empty(gc.host_scratch_size(hb), dtype=torch.uint8, device="cuda")
    gc.decode_host(hb, host, True, scratch)
    torch.cuda.synchronize()
    assert np.array_equal(host, w.values)
    st = gc.encode_posting_store(w.values, w.list_n, O.GROUP_PFD, 0, delta=True)
    out, wss = gc.decode_posting_store(st, dgaps=True)
    torch.cuda.synchronize()
    print(f"sanitize_decode: {n_checked} decodes checked against the oracle, range/host/store/malformed ran")


if __name__ == "__main__":
    main()

"""Full-size GPU parity (-m gpu): BASELINE.json configs 1-4 at their full sizes (2^20, 2^26,
2^28, 2^29 ints) and a 2^28-int slice of config 5's rank-0 shard, every codec bench.py runs on
them.  The inputs are the seeded generator's (gen/), encoded by the library's host encoder as
bench.py does, and decoded in the launch configuration bench.py times: gc_decode_stage with
RESET|INDEX and then DECODE on one output buffer and one workspace per variant, reused across
variants and across the gaps/docIDs passes.  Checked element by element, every element:

  * the host encoder's streams == the oracle encoder's (oracle/gc_oracle.c), byte for byte;
  * gc_decode == the oracle's gaps, gc_decode_dgaps == the oracle's docIDs;
  * device status 0, and the G7 checksum (gc_checksum) == the generator's, keyed on the
    global list id as in bench.py's multi-GPU all-reduce.

Bar: bit-exact (integer work)."""
import os

import numpy as np
import pytest

import gen
import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1502_01916_b200 import gc  # noqa: E402

THREADS = max(1, min(32, os.cpu_count() or 1))
STREAMS = ("ctrl_off", "data_off", "exc_off", "out_off", "ctrl", "data", "exc")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1502_01916_b200 import build
    build.build()
    torch.cuda.init()


def codecs_of(k: int):
    """The variants bench.py decodes for config k (bench.config_codecs)."""
    if k == 1:
        return [(O.GROUP_SIMPLE, 0)]
    if k == 2:
        return [(O.GROUP_SCHEME, O.gsc_variant(cg, kd)) for cg, kd in gc.GSC_VARIANTS]
    if k == 3:
        return [(O.GROUP_PFD, 0), (O.GROUP_PFD, 1)]
    if k == 4:
        return [(O.GROUP_AFOR, 0)]
    return [(O.GROUP_SIMPLE, 0), (O.GROUP_SCHEME, O.gsc_variant(1, "CU")),
            (O.GROUP_SCHEME, O.gsc_variant(8, "IU")), (O.GROUP_AFOR, 0), (O.GROUP_PFD, 0),
            (O.VARBYTE, 0)]


def run_config(w, codecs, list_base=0):
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream(dev)
    out = torch.empty(max(w.n_ints, 4), dtype=torch.int32, device=dev)
    want_chk = None
    for codec, variant in codecs:
        label = gc.codec_label(codec, variant)
        hb = gc.encode_batch(w.values, w.list_n, codec, variant, delta=w.delta)
        ref = O.encode_batch(w.values, w.list_n, codec, variant, delta=w.delta, threads=THREADS)
        d = hb.as_dict()
        for key in STREAMS:
            assert np.array_equal(np.asarray(d[key]), np.asarray(ref[key])), (label, key)
        db = gc.to_device(hb, dev)
        ws = gc.alloc_workspace(db, dev)
        for dgaps in (False, True):
            out.fill_(-1)  # stale output must not survive into the result
            gc.decode_stage(db, out, ws, dgaps, gc.STAGE_RESET | gc.STAGE_INDEX, stream)
            gc.decode_stage(db, out, ws, dgaps, gc.STAGE_DECODE, stream)
            torch.cuda.synchronize(dev)
            st = gc.read_device_status(ws)
            assert st == 0, (label, dgaps, gc.status_names(st))
            got = out[:w.n_ints].cpu().numpy().view(np.uint32)
            want = O.decode_batch(ref, dgaps=dgaps, threads=THREADS)
            bad = np.nonzero(got != want)[0]
            assert len(bad) == 0, f"{label} dgaps={dgaps}: {len(bad)} mismatches, first {bad[:8]}"
            if dgaps:
                if w.delta:
                    assert np.array_equal(got, w.values), label
                if want_chk is None:
                    want_chk = gen.checksum(w.list_n, want, list_base)
                sums = gc.checksum(db, out[:w.n_ints], list_base=list_base).cpu().numpy()
                assert [int(x) for x in sums.view(np.uint64)] == list(want_chk), label
            elif not w.delta:
                assert np.array_equal(got, w.values), label
        del db, ws
    torch.cuda.empty_cache()


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_baseline_config_full_size(k):
    w = gen.config(k)
    run_config(w, codecs_of(k))


def test_config5_shard_slice():
    """Config 5's rank-0 shard (2^31 ints per GPU at full size) at 1/8 scale: the Zipf(1.05)
    [1, 2^24] lengths and 32-bit docIDs, every codec of the config."""
    from paper_1502_01916_b200 import dist
    sh = dist.shard_for_rank(5, 1 / 8, 0, 8)
    run_config(sh.workload, codecs_of(5), sh.list_base)

"""The product host encoder (libgc.so gc_encode_*) emits exactly the oracle's bytes,
and the C-ABI library loads and exports every symbol include/gc.h declares (CPU only:
no compute call needs a GPU here)."""
import ctypes
import os
import re

import numpy as np
import pytest

import gen
import oracle as O
from paper_1502_01916_b200 import gc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODECS = ([(O.VARBYTE, 0), (O.GROUP_SIMPLE, 0)] + [(O.GROUP_SCHEME, O.gsc_variant(cg, k))
                                   for cg, k in gc.GSC_VARIANTS]
          + [(O.GROUP_AFOR, 0), (O.GROUP_PFD, 0), (O.GROUP_PFD, 1)])


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_1502_01916_b200 import build
    build.build()


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "gc.h")).read()
    declared = set(re.findall(r"\b(gc_[a-z_0-9]+)\s*\(", hdr))
    lib = ctypes.CDLL(gc.LIB_PATH)
    missing = [s for s in declared if not hasattr(lib, s)]
    assert declared and not missing, missing
    assert gc.abi_version() == 2


def _same(a: dict, b: gc.HostBatch):
    for k in ("list_n", "ctrl_off", "data_off", "exc_off", "out_off"):
        assert np.array_equal(np.asarray(a[k]), getattr(b, k)), k
    assert np.array_equal(a["ctrl"], b.ctrl)
    assert np.array_equal(a["data"].reshape(-1, 4), b.data)
    assert np.array_equal(a["exc"], b.exc)


@pytest.mark.parametrize("codec,variant", CODECS, ids=[gc.codec_label(c, v) for c, v in CODECS])
def test_encoder_bytes_equal_oracle(codec, variant):
    rng = np.random.default_rng(100 + 16 * codec + variant)
    for max_len, bits, spike in ((9, 3, 0.0), (300, 12, 0.02), (2000, 20, 0.05), (70, 32, 0.0)):
        w = gen.random_lists(rng, 60, max_len, bits, spike)
        ref = O.encode_batch(w.values, w.list_n, codec, variant, threads=2)
        got = gc.encode_batch(w.values, w.list_n, codec, variant, threads=3)
        _same(ref, got)
    w = gen.config(1, scale=1 / 32)
    _same(O.encode_batch(w.values, w.list_n, codec, variant, delta=True),
          gc.encode_batch(w.values, w.list_n, codec, variant, delta=True, threads=4))


@pytest.mark.parametrize("zeta,F", [((3, 10), 32), ((1, 10), 128), ((1, 20), 32)])
def test_encoder_pfd_parameters(zeta, F):
    rng = np.random.default_rng(7)
    w = gen.random_lists(rng, 40, 3000, 9, 0.08)
    _same(O.encode_batch(w.values, w.list_n, O.GROUP_PFD, 0, frame_quads=F, zeta=zeta),
          gc.encode_batch(w.values, w.list_n, O.GROUP_PFD, 0, frame_quads=F, zeta=zeta))


def test_encoder_rejects_bad_input():
    with pytest.raises(gc.GcError):
        gc.encode_batch(np.array([5, 3], np.uint32), np.array([2], np.uint32), O.GROUP_SIMPLE,
                        delta=True)
    with pytest.raises(gc.GcError):
        gc.encode_batch(np.array([1], np.uint32), np.array([1], np.uint32), O.GROUP_SCHEME,
                        variant=gc.gsc_variant(1, "B") | (2 << 2))
    with pytest.raises(gc.GcError):
        gc.encode_batch(np.array([1], np.uint32), np.array([1], np.uint32), 9)


def test_posting_store_short_lists_are_varbyte():
    """P:L640 §7.5: lists shorter than 64 are Variable Byte encoded whatever
    the requested codec; every original list is found at list_out_off (checked by decoding
    both groups with the oracle)."""
    w = gen.config(5, scale=2 ** -17)  # Zipf(1.05) over [1, 2^24]: most lists are short
    st = gc.encode_posting_store(w.values, w.list_n, O.GROUP_SCHEME, O.gsc_variant(1, "CU"),
                                 delta=True)
    assert st.short.codec == O.VARBYTE and np.all(st.short.list_n < 64)
    assert np.all(st.long.list_n >= 64) and len(st.short.list_n) + len(st.long.list_n) == len(w.list_n)
    out = np.zeros(st.total, np.uint32)
    out[:st.long.total_out] = O.decode_batch(st.long.as_dict(), dgaps=True)
    out[st.short_base:] = O.decode_batch(st.short.as_dict(), dgaps=True)
    starts = np.concatenate([[0], np.cumsum(w.list_n.astype(np.int64))[:-1]])
    for i in range(len(w.list_n)):
        o, n = int(st.list_out_off[i]), int(w.list_n[i])
        assert np.array_equal(out[o:o + n], w.values[starts[i]:starts[i] + n]), i


@pytest.mark.parametrize("lengths", [[0], [63], [64], [63, 64, 0, 1, 200, 0], [5] * 40,
                                     [100, 65, 64], []])
def test_posting_split_edges(lengths):
    """gc_posting_split / gc_posting_gather on the threshold (63 short, 64 long), empty
    lists, an all-short and an all-long store, no lists at all: every list (docIDs and TFs)
    is found at list_out_off after an oracle decode of both groups; short_base is 16-byte
    aligned and after the long group."""
    rng = np.random.default_rng(len(lengths))
    ln = np.array(lengths, np.uint32)
    n = int(ln.sum())
    vals = np.zeros(n, np.uint32)
    starts = np.concatenate([[0], np.cumsum(ln.astype(np.int64))[:-1]]) if len(ln) else np.zeros(0, np.int64)
    for i, k in enumerate(ln.tolist()):
        vals[starts[i]:starts[i] + k] = np.cumsum(rng.integers(1, 1000, k)).astype(np.uint32)
    tfs = rng.integers(0, 300, n).astype(np.uint32)
    st = gc.encode_posting_store(vals, ln, O.GROUP_AFOR, 0, delta=True, tfs=tfs)
    assert st.short_base % 4 == 0 and st.short_base >= st.long.total_out
    assert np.all(st.short.list_n < 64) and np.all(st.long.list_n >= 64)
    docs = np.zeros(max(st.total, 1), np.uint32)
    tf = np.zeros(max(st.total, 1), np.uint32)
    if st.long.total_out:
        docs[:st.long.total_out] = O.decode_batch(st.long.as_dict(), dgaps=True)
        tf[:st.long.total_out] = O.decode_batch(st.tf_long.as_dict(), dgaps=False)
    if st.short.total_out:
        docs[st.short_base:st.short_base + st.short.total_out] = O.decode_batch(st.short.as_dict(), dgaps=True)
        tf[st.short_base:st.short_base + st.short.total_out] = O.decode_batch(st.tf_short.as_dict(), dgaps=False)
    for i, k in enumerate(ln.tolist()):
        o = int(st.list_out_off[i])
        assert np.array_equal(docs[o:o + k], vals[starts[i]:starts[i] + k]), i
        assert np.array_equal(tf[o:o + k], tfs[starts[i]:starts[i] + k]), i

"""GPU encoder of the frame codecs (-m gpu): Group-PFD (variant 0,
P:L402-416) and SIMD-BP128 (variant 1) encoded on the device must equal the oracle
encoder's streams and directory byte for byte, and decode back (through the GPU decoder) to
the oracle's values.  Bar: bit-exact."""
import numpy as np
import pytest

import gen
import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1502_01916_b200 import gc  # noqa: E402

KEYS = ("ctrl_off", "data_off", "exc_off", "out_off")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1502_01916_b200 import build
    build.build()
    torch.cuda.init()


def check(values, list_n, variant, F=32, zeta=(1, 10), delta=False):
    ref = O.encode_batch(values, list_n, O.GROUP_PFD, variant, delta=delta, frame_quads=F,
                         zeta=zeta, threads=4)
    v = torch.from_numpy(np.ascontiguousarray(values, np.uint32).view(np.int32)).cuda()
    ln = torch.from_numpy(np.ascontiguousarray(list_n, np.uint32).view(np.int32)).cuda()
    db = gc.encode_device(v, ln, gc.GROUP_PFD, variant, delta=delta, frame_quads=F, zeta=zeta)
    torch.cuda.synchronize()
    t = db.tensors
    for k in KEYS:
        assert np.array_equal(t[k].cpu().numpy().view(np.uint64), ref[k]), k
    assert np.array_equal(t["ctrl"].cpu().numpy(), ref["ctrl"])
    assert np.array_equal(t["data"].cpu().numpy().view(np.uint32).reshape(-1, 4), ref["data"])
    assert np.array_equal(t["exc"].cpu().numpy(), ref["exc"])
    out, ws = gc.decode_dgaps(db)
    torch.cuda.synchronize()
    assert gc.read_device_status(ws) == 0
    want = O.decode_batch(ref, dgaps=True, threads=4)
    assert np.array_equal(out[:db.total_out].cpu().numpy().view(np.uint32), want)


@pytest.mark.parametrize("variant", [0, 1], ids=["G-PFD", "BP128"])
@pytest.mark.parametrize("F", [32, 128])
def test_random_ragged(variant, F):
    rng = np.random.default_rng(40 + variant + F)
    for n_lists, max_len, bits, spike in ((1, 5, 3, 0.0), (40, 700, 9, 0.05), (300, 3000, 14, 0.08),
                                          (20, 40000, 20, 0.01), (50, 300, 32, 0.0)):
        w = gen.random_lists(rng, n_lists, max_len, bits, spike)
        check(w.values, w.list_n, variant, F)


@pytest.mark.parametrize("zeta", [(1, 10), (3, 10), (1, 50), (0, 1)])
def test_pfd_zeta(zeta):
    w = gen.config(3, scale=1 / 512)
    check(w.values, w.list_n, 0, 32, zeta)


def test_delta_docids_and_empty_lists():
    """docIDs in (config 5's shape: Zipf lengths, 32-bit docIDs), the d-gaps taken on the
    device; empty lists between non-empty ones."""
    w = gen.config(5, scale=2 ** -16)
    ln = w.list_n.copy()
    ln[::7] = 0
    vals = np.concatenate([np.sort(np.random.default_rng(3).choice(1 << 30, int(n), replace=False))
                           .astype(np.uint32) for n in ln]) if ln.sum() else np.zeros(0, np.uint32)
    for variant in (0, 1):
        check(vals, ln, variant, 32, delta=True)


@pytest.mark.parametrize("variant", [0, 1], ids=["G-PFD", "BP128"])
def test_config3_full_size(variant):
    """BASELINE config 3 at full size (2^28 gaps in one list)."""
    w = gen.config(3)
    check(w.values, w.list_n, variant, 32)


GSC_BCU = [(cg, k) for cg in (1, 2, 4, 8) for k in ("B", "CU")] + [(4, "IU"), (8, "IU")]


def check_gsc(values, list_n, variant, delta=False):
    ref = O.encode_batch(values, list_n, O.GROUP_SCHEME, variant, delta=delta, threads=4)
    v = torch.from_numpy(np.ascontiguousarray(values, np.uint32).view(np.int32)).cuda()
    ln = torch.from_numpy(np.ascontiguousarray(list_n, np.uint32).view(np.int32)).cuda()
    db = gc.encode_device(v, ln, gc.GROUP_SCHEME, variant, delta=delta)
    torch.cuda.synchronize()
    t = db.tensors
    for k in KEYS:
        assert np.array_equal(t[k].cpu().numpy().view(np.uint64), ref[k]), k
    assert np.array_equal(t["ctrl"].cpu().numpy(), ref["ctrl"])
    assert np.array_equal(t["data"].cpu().numpy().view(np.uint32).reshape(-1, 4), ref["data"])
    assert db.exc_bytes == len(ref["exc"]) == 0
    out, ws = gc.decode_dgaps(db)
    torch.cuda.synchronize()
    assert gc.read_device_status(ws) == 0
    assert np.array_equal(out[:db.total_out].cpu().numpy().view(np.uint32),
                          O.decode_batch(ref, dgaps=True, threads=4))


@pytest.mark.parametrize("cg,kind", GSC_BCU, ids=[f"GSC-{c}-{k}" for c, k in GSC_BCU])
def test_group_scheme_random(cg, kind):
    """Group-Scheme binary / complete unary / incomplete unary encoded on the
    device."""
    rng = np.random.default_rng(70 + cg + (kind == "CU"))
    variant = O.gsc_variant(cg, kind)
    for n_lists, max_len, bits, spike in ((1, 6, 3, 0.0), (60, 900, 11, 0.05),
                                          (300, 3000, 20, 0.01), (40, 200, 32, 0.0)):
        w = gen.random_lists(rng, n_lists, max_len, bits, spike)
        check_gsc(w.values, w.list_n, variant)


def test_group_scheme_config2_full_size():
    """BASELINE config 2 at full size (2^26 gaps in 10^5 lists), all 10 variants."""
    w = gen.config(2)
    for cg, kind in GSC_BCU:
        check_gsc(w.values, w.list_n, O.gsc_variant(cg, kind))


def test_group_scheme_docids():
    w = gen.config(1)  # docIDs: the d-gaps are taken on the device
    check_gsc(w.values, w.list_n, O.gsc_variant(4, "CU"), delta=True)


def check_stream_codec(values, list_n, codec, variant=0, delta=False):
    ref = O.encode_batch(values, list_n, codec, variant, delta=delta, threads=8)
    v = torch.from_numpy(np.ascontiguousarray(values, np.uint32).view(np.int32)).cuda()
    ln = torch.from_numpy(np.ascontiguousarray(list_n, np.uint32).view(np.int32)).cuda()
    db = gc.encode_device(v, ln, codec, variant, delta=delta)
    torch.cuda.synchronize()
    t = db.tensors
    for k in KEYS:
        assert np.array_equal(t[k].cpu().numpy().view(np.uint64), ref[k]), k
    assert np.array_equal(t["ctrl"].cpu().numpy(), ref["ctrl"])
    assert np.array_equal(t["data"].cpu().numpy().view(np.uint32).reshape(-1, 4), ref["data"])
    out, ws = gc.decode_dgaps(db)
    torch.cuda.synchronize()
    assert gc.read_device_status(ws) == 0
    assert np.array_equal(out[:db.total_out].cpu().numpy().view(np.uint32),
                          O.decode_batch(ref, dgaps=True, threads=8))


def test_group_afor_random():
    """Group-AFOR (the DP of A23-A25) encoded on the device, lists in parallel."""
    rng = np.random.default_rng(91)
    for n_lists, max_len, bits, spike in ((1, 5, 2, 0.0), (80, 2000, 10, 0.05),
                                          (500, 600, 6, 0.02), (10, 30000, 24, 0.001),
                                          (30, 300, 32, 0.0)):
        w = gen.random_lists(rng, n_lists, max_len, bits, spike)
        check_stream_codec(w.values, w.list_n, O.GROUP_AFOR)
    w = gen.config(1)
    check_stream_codec(w.values, w.list_n, O.GROUP_AFOR, delta=True)


def test_group_afor_config4_full_size():
    """BASELINE config 4 at full size (2^29 gaps in 10^6 lists)."""
    w = gen.config(4)
    check_stream_codec(w.values, w.list_n, O.GROUP_AFOR)


def test_group_simple():
    """Group-Simple (Algorithm 1) encoded on the device, lists in parallel."""
    rng = np.random.default_rng(93)
    for n_lists, max_len, bits, spike in ((1, 3, 1, 0.0), (100, 1500, 8, 0.03),
                                          (400, 200, 3, 0.0), (20, 5000, 32, 0.0)):
        w = gen.random_lists(rng, n_lists, max_len, bits, spike)
        check_stream_codec(w.values, w.list_n, O.GROUP_SIMPLE)
    w = gen.config(1)  # BASELINE config 1 at full size, docIDs in
    check_stream_codec(w.values, w.list_n, O.GROUP_SIMPLE, delta=True)


def test_varbyte():
    """Variable Byte (P §2.3) encoded on the device: random lists, docIDs in (config 5's
    shape: most lists short), byte-identical to the oracle."""
    rng = np.random.default_rng(95)
    for n_lists, max_len, bits in ((1, 3, 1), (300, 80, 14), (40, 3000, 32)):
        w = gen.random_lists(rng, n_lists, max_len, bits)
        check_stream_codec(w.values, w.list_n, O.VARBYTE)
    w = gen.config(5, scale=2 ** -15)
    check_stream_codec(w.values, w.list_n, O.VARBYTE, delta=True)


def test_other_codecs_refused():
    v = torch.zeros(16, dtype=torch.int32, device="cuda")
    ln = torch.tensor([16], dtype=torch.int32, device="cuda")
    for codec, variant in ((gc.GROUP_SCHEME, 2 << 2), (7, 0)):  # (IU needs CG 4 or 8)
        with pytest.raises(gc.GcError):
            gc.encode_device(v, ln, codec, variant)


ALL_CODECS = ([(O.VARBYTE, 0), (O.GROUP_SIMPLE, 0), (O.GROUP_AFOR, 0), (O.GROUP_PFD, 0),
               (O.GROUP_PFD, 1)]
              + [(O.GROUP_SCHEME, O.gsc_variant(cg, k)) for cg, k in GSC_BCU])


@pytest.mark.parametrize("codec,variant", ALL_CODECS,
                         ids=[gc.codec_label(c, v) for c, v in ALL_CODECS])
def test_edge_batches(codec, variant):
    """Every GPU encoder on the edge shapes: all-empty lists, 1-int lists, all-zero and
    all-max values, a long single list, empty lists at the end."""
    rng = np.random.default_rng(11)
    cases = [
        (np.zeros(5, np.uint32), np.zeros(0, np.uint32)),
        (np.ones(700, np.uint32), rng.integers(0, 1 << 32, 700, dtype=np.uint64).astype(np.uint32)),
        (np.array([0, 3, 0, 4096, 1, 4095, 4097, 0, 0], np.uint32), None),
        (np.array([70000], np.uint32), np.zeros(70000, np.uint32)),
        (np.array([5000, 3], np.uint32), np.full(5003, 0xFFFFFFFF, np.uint32)),
    ]
    for ln, vals in cases:
        if vals is None:
            vals = rng.integers(0, 1 << 13, int(ln.sum()), dtype=np.uint64).astype(np.uint32)
        if codec == O.GROUP_PFD:
            check(vals, ln, variant, 32)
        elif codec == O.GROUP_SCHEME:
            check_gsc(vals, ln, variant)
        else:
            check_stream_codec(vals, ln, codec, variant)


def test_empty_batch():
    v = torch.zeros(0, dtype=torch.int32, device="cuda")
    ln = torch.zeros(0, dtype=torch.int32, device="cuda")
    for codec, variant in ALL_CODECS:
        db = gc.encode_device(v, ln, codec, variant)
        assert db.total_out == 0 and db.data_vectors == 0 and db.ctrl_bytes == 0

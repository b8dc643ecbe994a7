"""GPU parity (-m gpu): the CUDA path through the C ABI against the oracle and the
generator, element by element.  Bar: bit-exact (integer work)."""
import numpy as np
import pytest

import gen
import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1502_01916_b200 import gc  # noqa: E402

CODECS = ([(O.VARBYTE, 0), (O.GROUP_SIMPLE, 0)] + [(O.GROUP_SCHEME, O.gsc_variant(cg, k))
                                   for cg, k in gc.GSC_VARIANTS]
          + [(O.GROUP_AFOR, 0), (O.GROUP_PFD, 0), (O.GROUP_PFD, 1)])
IDS = [gc.codec_label(c, v) for c, v in CODECS]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1502_01916_b200 import build
    build.build()
    torch.cuda.init()


def gpu_decode(hb: gc.HostBatch, dgaps: bool):
    db = gc.to_device(hb)
    fn = gc.decode_dgaps if dgaps else gc.decode
    out, ws = fn(db)
    torch.cuda.synchronize()
    status = gc.read_device_status(ws)
    return out.cpu().numpy().view(np.uint32).copy(), status


def check(values, list_n, codec, variant, frame_quads=32, zeta=(1, 10), delta=False,
          encoder="oracle"):
    if encoder == "oracle":
        hb = gc.HostBatch.from_dict(O.encode_batch(values, list_n, codec, variant, delta=delta,
                                                   frame_quads=frame_quads, zeta=zeta, threads=4))
    else:
        hb = gc.encode_batch(values, list_n, codec, variant, delta=delta, frame_quads=frame_quads,
                             zeta=zeta)
    gaps = O.decode_batch(hb.as_dict(), dgaps=False, threads=4)
    docs = O.decode_batch(hb.as_dict(), dgaps=True, threads=4)
    g, s1 = gpu_decode(hb, dgaps=False)
    assert s1 == 0, gc.status_names(s1)
    bad = np.nonzero(g != gaps)[0]
    assert len(bad) == 0, f"gc_decode mismatch at {bad[:10]} ({len(bad)} total)"
    d, s2 = gpu_decode(hb, dgaps=True)
    assert s2 == 0, gc.status_names(s2)
    bad = np.nonzero(d != docs)[0]
    assert len(bad) == 0, f"gc_decode_dgaps mismatch at {bad[:10]} ({len(bad)} total)"
    if delta:
        assert np.array_equal(d, values)          # the generator's own docIDs
    else:
        assert np.array_equal(g, values)
    return hb


@pytest.mark.parametrize("codec,variant", CODECS, ids=IDS)
def test_random_ragged(codec, variant):
    rng = np.random.default_rng(1000 + 16 * codec + variant)
    for n_lists, max_len, bits, spike in ((1, 5, 3, 0), (7, 40, 8, 0.0), (200, 3000, 14, 0.01),
                                          (50, 20000, 22, 0.05), (30, 100, 32, 0.0)):
        w = gen.random_lists(rng, n_lists, max_len, bits, spike)
        check(w.values, w.list_n, codec, variant)


@pytest.mark.parametrize("tile_words", ["256", "2048"])
@pytest.mark.parametrize("codec,variant", CODECS, ids=IDS)
def test_both_index_tile_sizes(codec, variant, tile_words, monkeypatch):
    """The index stage's two control-tile sizes (256 words for small batches, 2048 otherwise)
    forced on the same ragged batches (lists from 1 int to 60k, runs of empty lists)."""
    monkeypatch.setenv("GC_INDEX_TILE_WORDS", tile_words)
    rng = np.random.default_rng(77 + codec + 16 * variant)
    w = gen.random_lists(rng, 120, 60000, 18, 0.02)
    ln = np.concatenate([w.list_n, np.zeros(700, np.uint32), np.array([1, 2, 3], np.uint32)])
    vals = np.concatenate([w.values, rng.integers(0, 1 << 10, 6).astype(np.uint32)])
    check(vals, ln, codec, variant)


@pytest.mark.parametrize("codec,variant", CODECS, ids=IDS)
def test_edge_shapes(codec, variant):
    """Empty lists, 1-int lists (thousands of lists per tile: control/data staging falls
    back to global memory and tiles run several parse/unpack rounds), one list spanning
    many tiles (look-back chains), lists ending exactly at tile boundaries, all-zero and
    all-max values."""
    rng = np.random.default_rng(7)
    cases = []
    ln = np.array([0, 0, 3, 0, 4096, 0, 1, 4095, 4097, 0], np.uint32)
    cases.append((ln, rng.integers(0, 1 << 12, int(ln.sum())).astype(np.uint32)))
    ln = np.ones(9000, np.uint32)
    cases.append((ln, rng.integers(0, 1 << 32, 9000, dtype=np.uint64).astype(np.uint32)))
    ln = rng.integers(1, 4, 6000).astype(np.uint32)
    cases.append((ln, rng.integers(0, 1 << 9, int(ln.sum())).astype(np.uint32)))
    ln = np.array([300_001], np.uint32)
    cases.append((ln, rng.integers(0, 1 << 10, 300_001).astype(np.uint32)))
    ln = np.array([5000, 70000], np.uint32)
    cases.append((ln, np.zeros(75000, np.uint32)))
    cases.append((ln, np.full(75000, 0xFFFFFFFF, np.uint32)))
    for ln, v in cases:
        check(v, ln, codec, variant)


@pytest.mark.parametrize("F,zeta", [(32, (3, 10)), (128, (1, 10)), (32, (1, 50))])
def test_pfd_parameters(F, zeta):
    w = gen.config(3, scale=1 / 256)
    check(w.values, w.list_n, O.GROUP_PFD, 0, frame_quads=F, zeta=zeta)


@pytest.mark.parametrize("k,scale", [(1, 1.0), (2, 1 / 64), (3, 1 / 64), (4, 1 / 256),
                                     (5, 1 / 16384)])
def test_configs_scaled_all_codecs(k, scale):
    """The five BASELINE configs' shapes at reduced scale, every codec (docIDs pinned to the
    generator for configs 1 and 5)."""
    w = gen.config(k, scale=scale)
    for codec, variant in CODECS:
        check(w.values, w.list_n, codec, variant, delta=w.delta)


def test_varbyte_long_lists_in_parallel():
    """Variable Byte lists of 64 .. 600k ints (byte-space tiles, the segmented scan and the
    look-back across tiles): long lists spanning many 8192-byte tiles, lists that start and end
    mid-tile between short ones, 1..5-byte ints (values up to 2^32-1), both paths, against the
    oracle; then malformed long lists (a missing terminator run, too few ints)."""
    rng = np.random.default_rng(64)
    ln = np.array([600_000, 3, 64, 65, 0, 1, 200_000, 63, 64, 9000, 5, 130_000, 2, 70], np.uint32)
    ln = np.concatenate([ln, rng.integers(1, 200, 300).astype(np.uint32), np.array([250_000], np.uint32)])
    bits = rng.integers(1, 33, int(ln.sum()))
    vals = (rng.integers(0, 1 << 32, int(ln.sum()), dtype=np.uint64) >> (32 - bits).astype(np.uint64))
    check(vals.astype(np.uint32), ln, O.VARBYTE, 0)
    # docIDs of one huge list and a few others: the d-gap carry crosses hundreds of tiles
    ln2 = np.array([1_500_000, 100, 70_000], np.uint32)
    gaps = rng.geometric(0.02, int(ln2.sum())).astype(np.uint64)
    docs = np.concatenate([np.cumsum(g) for g in np.split(gaps, np.cumsum(ln2)[:-1])]) % (1 << 32)
    check(docs.astype(np.uint32), ln2, O.VARBYTE, 0, delta=True)
    # malformed: a run of 6 bytes without a terminator inside a long list, and a long list cut
    hb = gc.HostBatch.from_dict(O.encode_batch(vals.astype(np.uint32), ln, O.VARBYTE))
    hb.ctrl = hb.ctrl.copy()
    c0 = int(hb.ctrl_off[6])
    hb.ctrl[c0 + 5000:c0 + 5006] &= 0x7F
    _, s = gpu_decode(hb, True)
    assert s & 2
    hb = gc.HostBatch.from_dict(O.encode_batch(vals.astype(np.uint32), ln, O.VARBYTE))
    hb.ctrl = hb.ctrl.copy()
    c0, c1 = int(hb.ctrl_off[11]), int(hb.ctrl_off[12])
    hb.ctrl[c1 - 40:c1] = 0                               # its last ints never terminate
    _, s = gpu_decode(hb, True)
    assert s & (2 | 16)


def test_malformed_streams_flagged_not_faulting():
    rng = np.random.default_rng(3)
    w = gen.random_lists(rng, 20, 500, 10)
    hb = gc.HostBatch.from_dict(O.encode_batch(w.values, w.list_n, O.GROUP_SIMPLE))
    hb.ctrl[0] = 0xFA                                         # selector 10
    _, s = gpu_decode(hb, True)
    assert s & 1
    hb = gc.HostBatch.from_dict(O.encode_batch(w.values, w.list_n, O.GROUP_AFOR))
    hb.ctrl[0] = 0x03                                         # length code 3
    _, s = gpu_decode(hb, True)
    assert s & 4
    hb = gc.HostBatch.from_dict(O.encode_batch(w.values, w.list_n, O.GROUP_PFD))
    hb.ctrl[0] = 0                                            # b = 0
    _, s = gpu_decode(hb, True)
    assert s & 4
    hb = gc.HostBatch.from_dict(O.encode_batch(w.values, w.list_n, O.GROUP_SCHEME,
                                               O.gsc_variant(8, "CU")))
    hb.ctrl[:8] = 0xFF                                        # runs of 32+ ones
    _, s = gpu_decode(hb, True)
    assert s & 2
    hb = gc.HostBatch.from_dict(O.encode_batch(w.values, w.list_n, O.VARBYTE))
    hb.ctrl = hb.ctrl.copy()
    hb.ctrl[:] = 0                                           # no int ever terminates
    _, s = gpu_decode(hb, True)
    assert s & (2 | 16)                                      # > 5 bytes / truncated
    hb = gc.HostBatch.from_dict(O.encode_batch(w.values, w.list_n, O.VARBYTE))
    hb.ctrl_off = hb.ctrl_off.copy()
    hb.ctrl_off[1:] = np.minimum(hb.ctrl_off[1:], hb.ctrl_off[1])  # lists 1.. have no bytes
    _, s = gpu_decode(hb, True)
    assert s & 16
    hb = gc.HostBatch.from_dict(O.encode_batch(w.values, w.list_n, O.VARBYTE))
    hb.out_off = hb.out_off.copy()
    hb.out_off[3] += 1                                        # inconsistent directory
    _, s = gpu_decode(hb, True)
    assert s & 16
    hb = gc.HostBatch.from_dict(O.encode_batch(w.values, w.list_n, O.GROUP_PFD, 0))
    if hb.exc_off[-1] > 0:                                   # a PFD frame with exceptions
        hb.variant = 1                                       # read as BP128: none allowed
        _, s = gpu_decode(hb, True)
        assert s & 8
    hb = gc.HostBatch.from_dict(O.encode_batch(w.values, w.list_n, O.GROUP_SCHEME,
                                               O.gsc_variant(1, "B")))
    hb.data_off = hb.data_off.copy()
    hb.data_off[5:] = np.minimum(hb.data_off[5:], hb.data_off[5])  # truncated data
    _, s = gpu_decode(hb, True)
    assert s & 16
    hb = gc.HostBatch.from_dict(O.encode_batch(w.values, w.list_n, O.GROUP_SCHEME,
                                               O.gsc_variant(2, "CU")))
    hb.out_off = hb.out_off.copy()
    hb.out_off[3] += 1                                        # inconsistent directory
    _, s = gpu_decode(hb, True)
    assert s & 16


def test_host_path_and_checksum():
    w = gen.config(1, scale=1 / 4)
    hb = gc.encode_batch(w.values, w.list_n, O.GROUP_SCHEME, O.gsc_variant(4, "CU"), delta=True)
    out = np.zeros(hb.total_out, np.uint32)
    scratch = torch.empty(gc.host_scratch_size(hb), dtype=torch.uint8, device="cuda")
    gc.decode_host(hb, out, True, scratch)
    torch.cuda.synchronize()
    assert np.array_equal(out, w.values)
    db = gc.to_device(hb)
    d, _ = gc.decode_dgaps(db)
    sums = gc.checksum(db, d).cpu().numpy().view(np.uint64)
    ref = gen.checksum(w.list_n, w.values)
    assert [int(x) for x in sums] == list(ref)


def test_api_errors():
    w = gen.random_lists(np.random.default_rng(1), 3, 10, 4)
    hb = gc.HostBatch.from_dict(O.encode_batch(w.values, w.list_n, O.GROUP_SIMPLE))
    db = gc.to_device(hb)
    with pytest.raises(gc.GcError):
        gc.decode(db, ws=torch.empty(16, dtype=torch.uint8, device="cuda"))
    db.variant = 5
    with pytest.raises(gc.GcError):
        gc.decode(db)


def test_concurrent_streams_distinct_workspaces():
    """Calls are reentrant across distinct workspaces (include/gc.h): batches of different
    codecs decoded on two streams at once (device and host-buffer paths, as bench.py's e2e
    pipeline issues them) each equal the oracle."""
    rng = np.random.default_rng(11)
    batches = []
    for codec, variant in [(O.GROUP_SCHEME, O.gsc_variant(8, "CU")), (O.GROUP_PFD, 0),
                           (O.GROUP_AFOR, 0), (O.GROUP_SCHEME, O.gsc_variant(4, "IU"))]:
        w = gen.random_lists(rng, 300, 20000, 12, 0.01)
        hb = gc.HostBatch.from_dict(O.encode_batch(w.values, w.list_n, codec, variant))
        batches.append((hb, O.decode_batch(hb.as_dict(), dgaps=True, threads=4)))
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = []
    for i, (hb, _) in enumerate(batches):
        s = streams[i % 2]
        with torch.cuda.stream(s):
            db = gc.to_device(hb)
            ws = gc.alloc_workspace(db)
            out = torch.empty(max(hb.total_out, 4), dtype=torch.int32, device="cuda")
        gc.decode_dgaps(db, out=out, ws=ws, stream=s)
        host = torch.empty(max(hb.total_out, 4) * 4, dtype=torch.uint8, pin_memory=True)
        scratch = torch.empty(gc.host_scratch_size(hb), dtype=torch.uint8, device="cuda")
        hv = host.numpy().view(np.uint32)[:hb.total_out]
        gc.decode_host(hb, hv, True, scratch, streams[(i + 1) % 2])
        outs.append((db, ws, out, host, hv, scratch))
    torch.cuda.synchronize()
    for (hb, want), (_, ws, out, _, hv, _) in zip(batches, outs):
        assert gc.read_device_status(ws) == 0
        got = out[:hb.total_out].cpu().numpy().view(np.uint32)
        assert np.array_equal(got, want)
        assert np.array_equal(hv, want)


def test_concurrent_host_threads():
    """No process-wide mutable state in the launch path (include/gc.h): four host threads,
    each with its own stream and workspace, decode different codecs at the same time from
    a cold start of every kernel (the shared-memory attribute and occupancy are per call)."""
    import threading
    rng = np.random.default_rng(12)
    jobs = []
    for codec, variant in [(O.GROUP_SIMPLE, 0), (O.GROUP_SCHEME, O.gsc_variant(2, "B")),
                           (O.GROUP_PFD, 1), (O.GROUP_AFOR, 0)]:
        w = gen.random_lists(rng, 500, 30000, 15, 0.01)
        hb = gc.HostBatch.from_dict(O.encode_batch(w.values, w.list_n, codec, variant))
        jobs.append((hb, O.decode_batch(hb.as_dict(), dgaps=True, threads=4)))
    results, errors = [None] * len(jobs), []

    def run(i):
        try:
            hb, _ = jobs[i]
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                db = gc.to_device(hb)
                for _ in range(3):
                    out, ws = gc.decode_dgaps(db, stream=s)
                s.synchronize()
                results[i] = (out[:hb.total_out].cpu().numpy().view(np.uint32).copy(),
                              gc.read_device_status(ws))
        except Exception as e:  # noqa: BLE001
            errors.append(e)
    threads = [threading.Thread(target=run, args=(i,)) for i in range(len(jobs))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for (hb, want), (got, st) in zip(jobs, results):
        assert st == 0
        assert np.array_equal(got, want)


@pytest.mark.parametrize("codec,variant", CODECS, ids=IDS)
def test_fuzz_repeated(codec, variant):
    """Seeded random batch shapes (list-length mixes from 1-int lists to lists spanning many
    tiles, value widths 1-32 bits with spikes), each decoded three times on one workspace:
    every run must equal the oracle (catches ordering races that show up only sometimes)."""
    rng = np.random.default_rng(5000 + 16 * codec + variant)
    for trial in range(6):
        n_lists = int(rng.integers(1, 3000))
        max_len = int(rng.choice([8, 300, 5000, 60000]))
        bits = int(rng.integers(1, 33))
        w = gen.random_lists(rng, n_lists, max_len, bits, float(rng.choice([0.0, 0.01, 0.2])))
        if w.n_ints == 0:
            continue
        hb = gc.HostBatch.from_dict(O.encode_batch(w.values, w.list_n, codec, variant))
        want = O.decode_batch(hb.as_dict(), dgaps=True, threads=4)
        db = gc.to_device(hb)
        ws = gc.alloc_workspace(db)
        out = torch.empty(max(hb.total_out, 4), dtype=torch.int32, device="cuda")
        for rep in range(3):
            out.fill_(-1)
            gc.decode_dgaps(db, out=out, ws=ws)
            torch.cuda.synchronize()
            assert gc.read_device_status(ws) == 0
            got = out[:hb.total_out].cpu().numpy().view(np.uint32)
            bad = np.nonzero(got != want)[0]
            assert len(bad) == 0, f"trial {trial} rep {rep}: {len(bad)} mismatches, first {bad[:8]}"


@pytest.mark.parametrize("codec,variant", [(O.GROUP_SIMPLE, 0), (O.GROUP_SCHEME, O.gsc_variant(8, "IU")),
                                           (O.GROUP_AFOR, 0), (O.GROUP_PFD, 0)])
def test_posting_store(codec, variant):
    """The §7.5 posting store on config 5's shape (72% of lists shorter than 64): long lists
    with the codec, short ones with Variable Byte, one output, every list at its offset."""
    w = gen.config(5, scale=2 ** -14)
    st = gc.encode_posting_store(w.values, w.list_n, codec, variant, delta=True)
    out, wss = gc.decode_posting_store(st, dgaps=True)
    torch.cuda.synchronize()
    assert all(gc.read_device_status(ws) == 0 for ws in wss)
    got = out.cpu().numpy().view(np.uint32)
    starts = np.concatenate([[0], np.cumsum(w.list_n.astype(np.int64))[:-1]])
    for i in range(len(w.list_n)):
        o, n = int(st.list_out_off[i]), int(w.list_n[i])
        assert np.array_equal(got[o:o + n], w.values[starts[i]:starts[i] + n]), i


SKIP_CODECS = [c for c in CODECS if c[0] != O.VARBYTE]


@pytest.mark.parametrize("codec,variant", SKIP_CODECS, ids=[gc.codec_label(c, v) for c, v in SKIP_CODECS])
def test_build_skip_equals_oracle(codec, variant):
    """gc_build_skip (the control scan writing an entry wherever a word owns a block's first
    quad, §7.5) is byte-identical to the oracle's skip table, on ragged lists incl.
    empty ones and lists of 511 / 512 / 513 ints."""
    rng = np.random.default_rng(300 + 16 * codec + variant)
    w = gen.random_lists(rng, 60, 9000, 16, 0.02)
    ln = np.concatenate([w.list_n, np.array([0, 511, 512, 513, 3, 0, 1025], np.uint32)])
    vals = np.concatenate([w.values, rng.integers(0, 1 << 18, int(ln[len(w.list_n):].sum())).astype(np.uint32)])
    ref = O.encode_batch(vals, ln, codec, variant)
    off_o, ent_o = O.build_skip(ref)
    db = gc.to_device(gc.HostBatch.from_dict(ref))
    docs, ws = gc.decode_dgaps(db)
    off, ent = gc.build_skip(db, docs)
    torch.cuda.synchronize()
    assert gc.read_device_status(ws) == 0
    assert np.array_equal(off.cpu().numpy().view(np.uint64), off_o)
    assert gc.skip_entries_host(off, ent).tobytes() == ent_o.tobytes()


@pytest.mark.parametrize("codec,variant", [(O.GROUP_SCHEME, O.gsc_variant(1, "CU")), (O.GROUP_PFD, 0),
                                           (O.GROUP_AFOR, 0), (O.GROUP_SIMPLE, 0),
                                           (O.GROUP_SCHEME, O.gsc_variant(8, "IU")),
                                           (O.GROUP_SCHEME, O.gsc_variant(2, "B")), (O.GROUP_PFD, 1)])
def test_decode_range_from_skip_table(codec, variant):
    """gc_decode_range (§8(f) rank 4): random ranges decoded from the ORACLE's skip table alone
    -- a fresh workspace, no full decode before -- equal the oracle's decode on exactly the
    range, and nothing outside it is written (both paths)."""
    w = gen.config(2, scale=1 / 32)
    ref = O.encode_batch(w.values, w.list_n, codec, variant)
    off_o, ent_o = O.build_skip(ref)
    db = gc.to_device(gc.HostBatch.from_dict(ref))
    off = torch.from_numpy(off_o.view(np.int64)).cuda()
    ent = torch.from_numpy(ent_o.view(np.uint8).reshape(-1, 32).copy()).cuda()
    rng = np.random.default_rng(5)
    N = int(ref["total_out"])
    for dgaps in (True, False):
        want = O.decode_batch(ref, dgaps=dgaps, threads=4).view(np.int32)
        ranges = [(0, N), (0, 1), (N - 1, 1), (511, 2), (512 * 7, 512)]
        ranges += [(int(f), int(rng.integers(1, min(40000, N - int(f)) + 1)))
                   for f in rng.integers(0, N - 1, 8)]
        for first, count in ranges:
            out = torch.full((N,), -7, dtype=torch.int32, device="cuda")
            ws = gc.decode_range(db, off, ent, out, first, count, dgaps)
            torch.cuda.synchronize()
            assert gc.read_device_status(ws) == 0
            got = out.cpu().numpy()
            assert np.array_equal(got[first:first + count], want[first:first + count]), (dgaps, first, count)
            assert (got[:first] == -7).all() and (got[first + count:] == -7).all()


def test_decode_range_flags_a_bad_table():
    """A skip table whose entry points past its list's control sets GC_DEV_TRUNCATED and
    writes nothing wrong outside the range (no fault)."""
    w = gen.config(2, scale=1 / 64)
    ref = O.encode_batch(w.values, w.list_n, O.GROUP_SCHEME, O.gsc_variant(4, "B"))
    off_o, ent_o = O.build_skip(ref)
    bad = ent_o.copy()
    bad["word"] += 1 << 20
    db = gc.to_device(gc.HostBatch.from_dict(ref))
    out = torch.zeros(int(ref["total_out"]), dtype=torch.int32, device="cuda")
    ws = gc.decode_range(db, torch.from_numpy(off_o.view(np.int64)).cuda(),
                         torch.from_numpy(bad.view(np.uint8).reshape(-1, 32).copy()).cuda(),
                         out, 100, 5000, True)
    torch.cuda.synchronize()
    assert gc.read_device_status(ws) & 16


@pytest.mark.parametrize("codec,variant", [(O.GROUP_SCHEME, O.gsc_variant(8, "IU")), (O.GROUP_PFD, 0),
                                           (O.GROUP_AFOR, 0), (O.GROUP_SIMPLE, 0),
                                           (O.GROUP_SCHEME, O.gsc_variant(1, "CU")), (O.GROUP_PFD, 1)])
def test_fused_docid_tf_decode_equals_the_oracle(codec, variant):
    """gc_decode_posting_store's fused pass (one k_decode over the docIDs batch and the TFs
    batch, their tiles interleaved) against the oracle's decode of each batch: docIDs with
    the d-gap scan, TFs raw; long lists spanning many tiles so both look-back and the
    interleaving are exercised."""
    rng = np.random.default_rng(40 + codec + 16 * variant)
    w = gen.random_lists(rng, 40, 60000, 20, 0.01)
    docs = np.zeros(w.n_ints, np.uint32)
    starts = np.concatenate([[0], np.cumsum(w.list_n.astype(np.int64))])
    for i in range(len(w.list_n)):  # strictly increasing docIDs per list
        seg = w.values[starts[i]:starts[i + 1]].astype(np.uint64) % 1000 + 1
        docs[starts[i]:starts[i + 1]] = (np.cumsum(seg) % (1 << 32)).astype(np.uint32)
    tfs = (rng.geometric(0.3, w.n_ints) % 5000).astype(np.uint32)
    st = gc.encode_posting_store(docs, w.list_n, codec, variant, delta=True, tfs=tfs)
    d, t, wss = gc.decode_posting_store(st, dgaps=True)
    torch.cuda.synchronize()
    assert all(gc.read_device_status(x) == 0 for x in wss)
    want_d = O.decode_batch(st.long.as_dict(), dgaps=True, threads=4)
    want_t = O.decode_batch(st.tf_long.as_dict(), dgaps=False, threads=4)
    n = st.long.total_out
    assert np.array_equal(d[:n].cpu().numpy().view(np.uint32), want_d)
    assert np.array_equal(t[:n].cpu().numpy().view(np.uint32), want_t)
    if st.short.total_out:
        sb = st.short_base
        assert np.array_equal(d[sb:sb + st.short.total_out].cpu().numpy().view(np.uint32),
                              O.decode_batch(st.short.as_dict(), dgaps=True, threads=4))
        assert np.array_equal(t[sb:sb + st.short.total_out].cpu().numpy().view(np.uint32),
                              O.decode_batch(st.tf_short.as_dict(), dgaps=False, threads=4))
    for i in range(len(w.list_n)):
        o, k = int(st.list_out_off[i]), int(w.list_n[i])
        assert np.array_equal(t[o:o + k].cpu().numpy().view(np.uint32), tfs[starts[i]:starts[i] + k])


@pytest.mark.parametrize("max_grid", ["7", "8", "1"])
def test_fused_decode_with_many_tiles_per_cta(max_grid, monkeypatch):
    """The fused pair with more tiles than CTAs (GC_DECODE_MAX_GRID caps the grid): an odd
    grid alternates every CTA between docID and TF tiles (a docID tile's deferred carry
    stores then run inside a TF tile), the library makes an even cap odd, and one CTA walks
    all tiles in order; the plain decode under the same caps as well."""
    monkeypatch.setenv("GC_DECODE_MAX_GRID", max_grid)
    rng = np.random.default_rng(71)
    w = gen.random_lists(rng, 30, 20000, 18, 0.02)
    docs = np.zeros(w.n_ints, np.uint32)
    starts = np.concatenate([[0], np.cumsum(w.list_n.astype(np.int64))])
    for i in range(len(w.list_n)):
        seg = w.values[starts[i]:starts[i + 1]].astype(np.uint64) % 3000 + 1
        docs[starts[i]:starts[i + 1]] = (np.cumsum(seg) % (1 << 32)).astype(np.uint32)
    tfs = (rng.geometric(0.3, w.n_ints) % 5000).astype(np.uint32)
    for codec, variant in [(O.GROUP_SCHEME, O.gsc_variant(1, "CU")), (O.GROUP_PFD, 0), (O.GROUP_AFOR, 0)]:
        st = gc.encode_posting_store(docs, w.list_n, codec, variant, delta=True, tfs=tfs)
        d, t, wss = gc.decode_posting_store(st, dgaps=True)
        torch.cuda.synchronize()
        assert all(gc.read_device_status(x) == 0 for x in wss)
        n = st.long.total_out
        assert n > 20 * 8192
        assert np.array_equal(d[:n].cpu().numpy().view(np.uint32),
                              O.decode_batch(st.long.as_dict(), dgaps=True, threads=4))
        assert np.array_equal(t[:n].cpu().numpy().view(np.uint32),
                              O.decode_batch(st.tf_long.as_dict(), dgaps=False, threads=4))
        db = gc.to_device(st.long)
        out, ws = gc.decode_dgaps(db)
        torch.cuda.synchronize()
        assert gc.read_device_status(ws) == 0
        assert np.array_equal(out[:n].cpu().numpy().view(np.uint32),
                              O.decode_batch(st.long.as_dict(), dgaps=True, threads=4))


def test_posting_store_with_term_frequencies():
    """The posting store with TF streams beside the docIDs (§8(f) rank 3): TFs (small, not
    sorted: Geometric(0.5)) decoded raw, concurrently with the d-gap docIDs."""
    w = gen.config(5, scale=2 ** -14)
    rng = np.random.default_rng(9)
    tfs = rng.geometric(0.5, w.n_ints).astype(np.uint32)
    st = gc.encode_posting_store(w.values, w.list_n, O.GROUP_SCHEME, O.gsc_variant(8, "IU"),
                                 delta=True, tfs=tfs)
    docs, tf, wss = gc.decode_posting_store(st, dgaps=True)
    torch.cuda.synchronize()
    assert all(gc.read_device_status(ws) == 0 for ws in wss)
    d = docs.cpu().numpy().view(np.uint32)
    t = tf.cpu().numpy().view(np.uint32)
    starts = np.concatenate([[0], np.cumsum(w.list_n.astype(np.int64))[:-1]])
    for i in range(len(w.list_n)):
        o, n = int(st.list_out_off[i]), int(w.list_n[i])
        assert np.array_equal(d[o:o + n], w.values[starts[i]:starts[i] + n]), i
        assert np.array_equal(t[o:o + n], tfs[starts[i]:starts[i] + n]), i


def test_library_build_flags():
    """GC_EXPECT_CHECKED=1 (set when the suite runs against the -DGC_CHECKED build, the
    bounds-asserting stand-in for compute-sanitizer) proves that build is the one loaded."""
    import os
    flags = gc.build_flags()
    if os.environ.get("GC_EXPECT_CHECKED") == "1":
        assert flags & 1, "GC_LIB does not point at a -DGC_CHECKED build"
    else:
        assert flags in (0, 1, 2, 3)


@pytest.mark.parametrize("max_grid", [0, 3])
def test_afor_piece_queue(max_grid, monkeypatch):
    """Group-AFOR frames of 8..32 quads are split after the parse into queued 4-quad
    pieces: frames of every length and width, frames straddling tile edges
    (lists ending a few ints past multiples of 8192 and 128), lists ending inside a frame's
    last piece, and runs of gap 1 (32-quad frames at 1 bit) beside wide gaps -- against the
    oracle, with the whole grid and with 3 CTAs (many tiles per CTA, the queue reused)."""
    if max_grid:
        monkeypatch.setenv("GC_DECODE_MAX_GRID", str(max_grid))
    rng = np.random.default_rng(77)
    ln = np.array([8192 * 3 + 5, 127, 129, 1, 2, 3, 511, 513, 8190, 4099, 65536 + 17, 33, 96, 97]
                  + list(rng.integers(1, 3000, 40)), np.uint32)
    n = int(ln.sum())
    v = np.ones(n, np.uint32)                              # gap-1 runs: long 1-bit frames
    wide = rng.random(n) < 0.3
    v[wide] = rng.integers(1, 1 << 20, int(wide.sum()), dtype=np.uint64).astype(np.uint32)
    runs = rng.random(n) < 0.02                            # occasional 32-bit outliers
    v[runs] = rng.integers(1 << 31, 1 << 32, int(runs.sum()), dtype=np.uint64).astype(np.uint32)
    check(v, ln, O.GROUP_AFOR, 0)

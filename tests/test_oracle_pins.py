"""Pins of the oracle against what the paper and the mathematics fix (-m "not gpu").

Each test names the passage it pins.  None of these retypes an oracle formula: they
use the paper's / SPEC's worked examples (tests/golden/), closed forms, theorems,
brute force over tiny inputs, an independent bit-level reader of the prose format
(tests/_reader.py) and the round-trip invariant.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle as O
from tests import _reader as R

GOLD = os.path.join(os.path.dirname(__file__), "golden")
ALL_GSC = [(cg, k) for cg in (1, 2, 4, 8) for k in ("B", "CU")] + [(4, "IU"), (8, "IU")]


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def quads_with_maxima(maxima):
    return np.array([[m, 0, 0, 0] for m in maxima], np.uint32).reshape(-1)


# ------------------------------------------------------------------ bitcore
def test_width_paper_example_and_closed_form():
    g = gold("width_458.json")
    assert O.width(g["value"]) == g["width"]
    assert O.width(0) == 1                                         # A1
    for b in range(1, 33):                                         # width = ceil(log2(x+1))
        assert O.width((1 << b) - 1) == b
        if b < 32:
            assert O.width(1 << b) == b + 1
    rng = np.random.default_rng(1)
    for x in rng.integers(1, 1 << 32, 2000, dtype=np.uint64):
        assert O.width(int(x)) == int(x).bit_length()


def test_pseudo_quad_max_theorem():
    """A9: OR and max share the highest set bit, so every width decision is equal and
    Algorithm 1 makes identical choices."""
    rng = np.random.default_rng(2)
    for _ in range(300):
        L = int(rng.integers(1, 200))
        bits = rng.integers(1, 33, (L, 1))
        q = (rng.integers(0, 1 << 32, (L, 4), dtype=np.uint64) >> (32 - bits).astype(np.uint64))
        q = q.astype(np.uint32)
        mx = [O.quad_max(r) for r in q]
        orr = [O.quad_or(r) for r in q]
        assert mx == [int(r.max()) for r in q]
        assert [O.width(a) for a in mx] == [O.width(b) for b in orr]
        assert O.gs_select(mx) == O.gs_select(orr)


@pytest.mark.parametrize("name", ["pack_vertical_0x51.json", "pack_vertical_split_bw7.json"])
def test_pack_vertical_golden(name):
    g = gold(name)
    v = O.pack_vertical(np.array(g["quads"], np.uint32), g["bw"])
    assert v.tolist() == g["vectors"]
    assert O.unpack_vertical(v, g["bw"], len(g["quads"])).tolist() == g["quads"]


def test_pack_vertical_against_bit_reader_all_widths():
    """Every width 1..32 at every offset: the independent bit-level reader of the prose
    (split rule A3) recovers what the oracle packed; bit cost 128*ceil(Q*bw/32)."""
    rng = np.random.default_rng(3)
    for bw in range(1, 33):
        Q = int(rng.integers(1, 70))
        q = rng.integers(0, 1 << bw, (Q, 4), dtype=np.uint64).astype(np.uint32)
        v = O.pack_vertical(q, bw)
        assert len(v) == -(-Q * bw // 32)
        got = [R.read_quad(v, 0, j * bw, bw) for j in range(Q)]
        assert got == q.tolist()


# ------------------------------------------------------------------ Group-Simple
def test_table3_through_encoder():
    """Table III: NUM_i quads whose max is exactly 2^BW_i - 1 select SEL i (Alg. 1 lines
    10-14: smaller BW stalls at pos 0), and fit one 128-bit vector."""
    t = gold("gs_table3.json")
    for i, (num, bw) in enumerate(zip(t["num"], t["bw"])):
        assert num * bw <= 32
        maxarr = [(1 << bw) - 1] * num
        assert O.gs_select(maxarr) == [i]
        x = quads_with_maxima(maxarr)
        s = O.encode_list(x, O.GROUP_SIMPLE)
        assert s["ctrl"].tolist() == [i] and s["data"].shape == (1, 4)
        # component 0 holds the quads' lane-0 values at [t*BW, (t+1)*BW), A7
        assert int(s["data"][0, 0]) == sum(((1 << bw) - 1) << (t * bw) for t in range(num)) \
            & 0xFFFFFFFF


def test_algorithm1_worked_cases():
    for c in gold("gs_alg1_cases.json")["cases"]:
        assert O.gs_select(c["maxarr"]) == c["modes"], c


def test_algorithm1_declarative_properties_bruteforce():
    """For random MaxArr: each emitted selector is the smallest SEL whose run over the
    remaining entries reaches NUM or the end of the array (P:L214 'tries to find a pattern
    to fit the remaining quad max integers as many as possible'), and the run it covers is
    exactly min(NUM, remaining) entries, all <= 2^BW-1 (coverage soundness)."""
    rng = np.random.default_rng(4)
    for _ in range(400):
        L = int(rng.integers(1, 120))
        widths = rng.choice([1, 2, 3, 5, 8, 11, 16, 20, 32], L)
        maxarr = [int(rng.integers(0, 1 << int(w), dtype=np.uint64)) for w in widths]
        modes = O.gs_select(maxarr)
        j = 0
        for sel in modes:
            rem = L - j

            def fits(i):
                run = 0
                while run < min(R.NUM[i], rem) and maxarr[j + run] < (1 << R.BW[i]):
                    run += 1
                return run == R.NUM[i] or run == rem

            assert fits(sel) and not any(fits(i) for i in range(sel))
            c = min(R.NUM[sel], rem)
            assert all(v < (1 << R.BW[sel]) for v in maxarr[j:j + c])
            j += c
        assert j == L


def test_gs_sizes_and_12800_ones():
    g = gold("gs_12800_ones.json")
    x = np.full(g["n"], g["value"], np.uint32)
    s = O.encode_list(x, O.GROUP_SIMPLE)
    assert len(s["data"]) == g["selectors"] and len(s["ctrl"]) == -(-g["selectors"] // 2)
    blk = O.encode_block(x, O.GROUP_SIMPLE)
    assert len(blk) == g["block_bytes"]
    assert round(8 * len(blk) / g["n"], 2) == g["bits_per_int"]
    assert (O.decode_block(blk) == x).all()


def test_fig3_twenty_ints():
    """P:L252 Fig. 3: 20 ints (5 quads), largest needing 6 bits -> one SEL 5 vector."""
    rng = np.random.default_rng(5)
    x = rng.integers(0, 64, 20).astype(np.uint32)
    x[7] = 45
    s = O.encode_list(x, O.GROUP_SIMPLE)
    assert s["ctrl"].tolist() == [5] and s["data"].shape == (1, 4)
    assert R.decode_group_simple(20, s["ctrl"], s["data"]) == x.tolist()


# ------------------------------------------------------------------ Group-Scheme
def test_eq1_eq2_paper_example():
    g = gold("width_458.json")
    cg = g["cg"]
    assert O.gsc_ld(g["value"], O.gsc_variant(cg, "B")) == g["ld_binary"]     # Eq. (1)
    assert O.gsc_ld(g["value"], O.gsc_variant(cg, "CU")) == g["ld_unary"]
    assert O.gsc_bw(g["ld_binary"], O.gsc_variant(cg, "B")) == g["bw"]        # Eq. (2)
    assert O.gsc_bw(g["ld_unary"], O.gsc_variant(cg, "CU")) == g["bw"]
    s = O.encode_list(np.array([g["value"], 0, 0, 0], np.uint32), O.GROUP_SCHEME,
                      O.gsc_variant(cg, "CU"))
    assert s["ctrl"].tolist() == g["unary_ctrl_bytes"]                         # '11110'


def test_table4_ranges_and_kgamma():
    """Table IV: binary LD field widths 5/4/3/2; unary LD ranges 1..32/CG.  P:L302: CG=1
    with complete unary stores each quad at exactly its effective width (k-Gamma)."""
    for cg, fw in ((1, 5), (2, 4), (4, 3), (8, 2)):
        vb, vu = O.gsc_variant(cg, "B"), O.gsc_variant(cg, "CU")
        assert O.gsc_ld(0xFFFFFFFF, vb) == (1 << fw) - 1 == 32 // cg - 1
        assert O.gsc_ld(0xFFFFFFFF, vu) == 32 // cg and O.gsc_ld(0, vu) == 1
        for x in (0, 1, 7, 255, 256, 65535, 1 << 20, 0xFFFFFFFF):
            assert O.gsc_bw(O.gsc_ld(x, vu), vu) >= O.width(x)
            assert O.gsc_bw(O.gsc_ld(x, vu), vu) - O.width(x) < cg
    rng = np.random.default_rng(6)
    x = (rng.integers(0, 1 << 32, 4000, dtype=np.uint64) >> rng.integers(0, 32, 4000)
         .astype(np.uint64)).astype(np.uint32)
    s = O.encode_list(x, O.GROUP_SCHEME, O.gsc_variant(1, "CU"))
    total = sum(O.width(int(q.max())) for q in x.reshape(-1, 4))
    assert len(s["data"]) == -(-total // 32)


def test_binary_ld_packing_capacities():
    """1-B decodes 12 ints per 16-bit pattern; 2-B and 4-B 8 ints per byte; 8-B
    16 ints per byte.  Footnote 2: 2^15-entry table for CG=1, 2^8 otherwise."""
    for cg, ints, bits in ((1, 12, 16), (2, 8, 8), (4, 8, 8), (8, 16, 8)):
        x = np.full(ints * 10, 3, np.uint32)
        s = O.encode_list(x, O.GROUP_SCHEME, O.gsc_variant(cg, "B"))
        assert len(s["ctrl"]) * 8 == bits * 10
        used = {1: 15, 2: 8, 4: 6, 8: 8}[cg]                 # bits that carry fields
        assert used == (ints // 4) * (5 - {1: 0, 2: 1, 4: 2, 8: 3}[cg])
    assert 2 ** 15 == 2 ** (3 * 5) and 2 ** 8 == 2 ** (2 * 4) == 2 ** (4 * 2)


@pytest.mark.parametrize("name", ["unary_10110011.json", "binary_cg8_e4.json",
                                  "iu_cg8_4_4.json", "iu_cg4_pad.json"])
def test_control_golden(name):
    g = gold(name)
    v = O.gsc_variant(g["variant_cg"], g["variant_kind"])
    x = quads_with_maxima(g["quad_maxima"])
    s = O.encode_list(x, O.GROUP_SCHEME, v)
    assert s["ctrl"].tolist() == g["ctrl_bytes"]
    if "lds" in g:
        assert [O.gsc_ld(m, v) for m in g["quad_maxima"]] == g["lds"]
    assert (O.decode_list(len(x), s["ctrl"], s["data"], None, O.GROUP_SCHEME, v) == x).all()


@pytest.mark.parametrize("cg,kind", [(8, "CU"), (8, "IU"), (4, "IU"), (4, "CU"), (2, "CU")])
def test_unary_control_exhaustive_ld_sequences(cg, kind):
    """Brute force over every LD sequence of length <= 4 (CG 8) or <= 3 (CG 2/4): the
    oracle's control bytes decode (by the independent reader) to the same LDs, and the
    unary code of v is (v-1) ones and a 0."""
    v = O.gsc_variant(cg, kind)
    maxu = 32 // cg
    length = 4 if cg == 8 else 3
    for L in range(1, length + 1):
        for lds in itertools.product(range(1, maxu + 1), repeat=L):
            maxima = [(1 << (cg * u)) - 1 if cg * u < 32 else 0xFFFFFFFF for u in lds]
            x = quads_with_maxima(maxima)
            s = O.encode_list(x, O.GROUP_SCHEME, v)
            assert R.decode_group_scheme(len(x), s["ctrl"], s["data"], cg, kind) == x.tolist()
            if kind == "CU":
                code = "".join("1" * (u - 1) + "0" for u in lds)
                bits = "".join(f"{b:08b}" for b in s["ctrl"])
                assert bits.startswith(code) and set(bits[len(code):]) <= {"0"}
                assert len(s["ctrl"]) == -(-len(code) // 8)


def test_gsc_trend_bits_grow_with_cg():
    """'With the increase in granularity, the compression ratio becomes worse'
    (testable form S:L390) on geometric gaps, within each LD kind."""
    rng = np.random.default_rng(7)
    x = rng.geometric(0.05, 1 << 16).astype(np.uint32)
    for kind in ("CU", "B"):
        sizes = []
        for cg in (1, 2, 4, 8):
            s = O.encode_list(x, O.GROUP_SCHEME, O.gsc_variant(cg, kind))
            sizes.append(16 * len(s["data"]))
        assert sizes == sorted(sizes)


# ------------------------------------------------------------------ Group-AFOR
def _expand(spec):
    out = []
    for part in spec.split("+"):
        cnt, w = part.split("x")
        out += [int(w)] * int(cnt)
    return out


def test_afor_golden():
    g = gold("afor_cases.json")
    for c in g["cases"]:
        cost, frames = O.afor_partition(_expand(c["widths"]))
        assert cost == c["cost"] and [list(f) for f in frames] == c["frames"]
    s = O.encode_list(np.ones(128, np.uint32), O.GROUP_AFOR)
    assert s["ctrl"].tolist() == g["ones_128"]["header"]
    assert len(s["data"]) == g["ones_128"]["vectors"]


def test_afor_dp_optimal_bruteforce():
    """P:L392 'optimal configuration ... dynamic programming': the DP cost equals the
    exhaustive minimum over all {8,16,32}-quad tilings for up to 24 quads."""
    rng = np.random.default_rng(8)

    def tilings(slots):
        if slots == 0:
            yield []
            return
        for L in (1, 2, 4):
            if L <= slots:
                for rest in tilings(slots - L):
                    yield [L] + rest

    for _ in range(300):
        Qp = 8 * int(rng.integers(1, 4))
        w = [int(v) for v in rng.choice([1, 2, 3, 7, 12, 20, 32], Qp, p=[.3, .2, .2, .1, .1, .05, .05])]
        best = None
        for t in tilings(Qp // 8):
            i, cost = 0, 0
            for s in t:
                L = 8 * s
                cost += 8 + 128 * (-(-L * max(w[i:i + L]) // 32))
                i += L
            best = cost if best is None else min(best, cost)
        cost, frames = O.afor_partition(w)
        assert cost == best
        assert sum(L for L, _ in frames) == Qp
        i = 0
        for L, bw in frames:
            assert bw == max(w[i:i + L])
            i += L


# ------------------------------------------------------------------ Group-PFD
def test_pfd_golden():
    g = gold("pfd_cases.json")
    ex = g["b_example"]
    qmax = [31] * 30 + [(1 << 20) - 1] * 2
    assert O.pfd_choose_b(qmax, tuple(ex["zeta"])) == ex["b"]
    t = g["two_exc"]
    x = np.full((32, 4), 200, np.uint32)
    x[13] = [70000, 300, 1, 2]
    s = O.encode_list(x.reshape(-1), O.GROUP_PFD)
    assert s["ctrl"].tolist() == [t["b"], t["wcode"], t["count"], 0]
    pos = [13 * 4 + 0, 13 * 4 + 1]
    vals = b"".join(int(v).to_bytes(4, "little") for v in t["values"])
    assert s["exc"].tolist() == pos + list(vals)
    # S:L488 size formula, one full frame: 32 + count*(8+w) + 128*b bits
    bits = 8 * (len(s["ctrl"]) + len(s["exc"])) + 128 * len(s["data"])
    assert bits == 32 + 2 * (8 + 32) + 128 * 8


def test_pfd_b_rule_bruteforce_and_monotone():
    """Step 2: b is the minimum width whose exception ratio over the frame's
    quad maxima is <= zeta (A28): b satisfies it and b-1 does not; monotone in zeta."""
    rng = np.random.default_rng(9)
    for _ in range(500):
        q = int(rng.integers(1, 33))
        w = rng.integers(1, 33, q)
        qmax = [(1 << int(v)) - 1 for v in w]
        prev = 33
        for zeta in ((1, 20), (1, 10), (3, 10), (1, 2)):
            b = O.pfd_choose_b(qmax, zeta)
            ok = lambda bb: sum(int(v) > bb for v in w) * zeta[1] <= zeta[0] * q
            assert ok(b) and (b == 1 or not ok(b - 1))
            assert b <= prev
            prev = b


# ------------------------------------------------------------------ round trip + reader
CODECS = ([(O.GROUP_SIMPLE, 0, "GS")] + [(O.GROUP_SCHEME, O.gsc_variant(cg, k), f"GSC-{cg}-{k}")
                                         for cg, k in ALL_GSC]
          + [(O.GROUP_AFOR, 0, "AFOR"), (O.GROUP_PFD, 0, "PFD")])


@pytest.mark.parametrize("codec,variant,name", CODECS, ids=[c[2] for c in CODECS])
def test_roundtrip_and_independent_reader(codec, variant, name):
    """decode(encode(x)) == x and the independent prose reader agrees, over
    ragged lengths (n mod 4 != 0, 0, 1), all-zero, all-max, spikes, mixed widths."""
    rng = np.random.default_rng(10 + codec * 16 + variant)
    cases = [np.zeros(0, np.uint32), np.zeros(1, np.uint32), np.full(7, 0xFFFFFFFF, np.uint32),
             np.zeros(131, np.uint32)]
    for n in (1, 2, 3, 5, 33, 127, 128, 129, 511, 1000):
        for bits in (1, 4, 9, 17, 32):
            x = (rng.integers(0, 1 << 32, n, dtype=np.uint64) >> np.uint64(32 - bits)).astype(np.uint32)
            m = rng.random(n) < 0.05
            x[m] = rng.integers(0, 1 << 32, int(m.sum()), dtype=np.uint64).astype(np.uint32)
            cases.append(x)
    for x in cases:
        n = len(x)
        s = O.encode_list(x, codec, variant)
        y = O.decode_list(n, s["ctrl"], s["data"], s["exc"], codec, variant)
        assert (y == x).all()
        if n <= 600:
            if codec == O.GROUP_SIMPLE:
                r = R.decode_group_simple(n, s["ctrl"], s["data"])
            elif codec == O.GROUP_SCHEME:
                cg, kind = 1 << (variant & 3), ("B", "CU", "IU")[variant >> 2]
                r = R.decode_group_scheme(n, s["ctrl"], s["data"], cg, kind)
            elif codec == O.GROUP_AFOR:
                r = R.decode_group_afor(n, s["ctrl"], s["data"])
            else:
                r = R.decode_group_pfd(n, s["ctrl"], s["data"], s["exc"])
            assert r == x.tolist()
        blk = O.encode_block(x, codec, variant)
        assert len(blk) % 16 == 0 and blk[:4] == b"GCM1"
        assert (O.decode_block(blk) == x).all()


def test_block_errors_distinguishable():
    """bad magic, version, codec, truncation are distinguishable errors."""
    blk = bytearray(O.encode_block(np.arange(1, 300, dtype=np.uint32), O.GROUP_SCHEME,
                                   O.gsc_variant(2, "CU"), delta=True))
    assert (O.decode_block(bytes(blk)) == np.arange(1, 300)).all()
    for patch, kind in (((0, 0x58), "bad_magic"), ((4, 2), "version"), ((5, 9), "codec")):
        b = bytearray(blk)
        b[patch[0]] = patch[1]
        with pytest.raises(O.OracleError) as e:
            O.decode_block(bytes(b))
        assert e.value.kind == kind
    for cut in range(16, len(blk) - 1, 7):
        with pytest.raises(O.OracleError) as e:
            O.decode_block(bytes(blk[:cut]))
        assert e.value.kind in ("truncated", "malformed")


def test_malformed_streams_detected():
    x = np.arange(64, dtype=np.uint32)
    s = O.encode_list(x, O.GROUP_SIMPLE)
    c = s["ctrl"].copy()
    c[0] = 0x0A                                                   # SEL 10 > 9
    with pytest.raises(O.OracleError) as e:
        O.decode_list(64, c, s["data"], None, O.GROUP_SIMPLE)
    assert e.value.kind == "malformed"
    v = O.gsc_variant(8, "CU")
    with pytest.raises(O.OracleError) as e:                       # run of 4 ones at CG 8
        O.decode_list(4, np.array([0xF0], np.uint8), np.zeros((4, 4), np.uint32), None,
                      O.GROUP_SCHEME, v)
    assert e.value.kind == "malformed"
    with pytest.raises(O.OracleError) as e:                       # AFOR length code 3
        O.decode_list(4, np.array([0x03], np.uint8), np.zeros((8, 4), np.uint32), None,
                      O.GROUP_AFOR)
    assert e.value.kind == "malformed"
    with pytest.raises(O.OracleError) as e:                       # PFD b = 0
        O.decode_list(4, np.array([0, 0, 0, 0], np.uint8), np.zeros((8, 4), np.uint32), None,
                      O.GROUP_PFD)
    assert e.value.kind == "malformed"


# ------------------------------------------------------------------ batch + d-gap
def test_batch_dgaps_equal_generator_docids():
    """The d-gap inverse pinned against the generator's own docIDs (G5): cfg1 at
    1/16 scale, every codec; plus empty lists and mod-2^32 wrap (A36)."""
    import gen
    w = gen.config(1, scale=1 / 16)
    for codec, variant, _ in CODECS[::3]:
        bt = O.encode_batch(w.values, w.list_n, codec, variant, delta=True, threads=2)
        assert (O.decode_batch(bt, dgaps=True, threads=3) == w.values).all()
    ln = np.array([0, 3, 0, 5], np.uint32)
    g = np.array([0xFFFFFFFF, 2, 3, 1, 1, 1, 1, 1], np.uint32)
    bt = O.encode_batch(g, ln, O.GROUP_PFD)
    assert O.decode_batch(bt, dgaps=True).tolist() == [0xFFFFFFFF, 1, 4, 1, 2, 3, 4, 5]
    assert len(bt["ctrl"]) % 16 == 0
    assert all(int(o) % 4 == 0 for o in bt["ctrl_off"])


@pytest.mark.parametrize("F", [32, 128])
def test_bp128_frames_at_max_width_no_exceptions(F):
    """SIMD-BP128 as the special case of P:L424 (PFD variant 1): every frame of 4F ints is
    packed at "the minimum number of bits to hold the largest integer among" them, with no
    exceptions.  Checked by brute force on the headers the oracle writes: b = bit length of
    the frame's largest int (1 for an all-zero frame), wcode = count = 0, an empty
    exception stream, ceil(q*b/32) data vectors per frame, and the round trip."""
    rng = np.random.default_rng(17)
    for n, bits in ((1, 3), (4 * F - 1, 9), (4 * F, 1), (10 * 4 * F + 7, 20), (3 * 4 * F, 32)):
        x = rng.integers(0, 1 << bits, n, dtype=np.uint64).astype(np.uint32)
        if n > 4 * F:
            x[4 * F:8 * F] = 0  # an all-zero frame
        bt = O.encode_batch(x, np.array([n], np.uint32), O.GROUP_PFD, 1, frame_quads=F)
        assert len(bt["exc"]) == 0 or not bt["exc"].any()
        hdr = bt["ctrl"][: 4 * ((n + 4 * F - 1) // (4 * F))].reshape(-1, 4)
        vec = 0
        for f, h in enumerate(hdr):
            frame = x[4 * F * f: 4 * F * (f + 1)]
            b = max(1, int(frame.max()).bit_length())
            assert (int(h[0]), int(h[1]), int(h[2]) | int(h[3]) << 8) == (b, 0, 0), f
            q = (len(frame) + 3) // 4
            vec += (q * b + 31) // 32
        assert int(bt["data_off"][1]) == vec
        assert np.array_equal(O.decode_batch(bt, dgaps=False), x)


def test_varbyte_spec_bytes_and_errors():
    """Variable Byte (P §2.3): 7-bit groups least significant first, MSB = 1
    on the LAST byte.  SPEC's derived bytes, its two errors, and the length rule
    ceil(width/7) (width(0) = 1) at every 7-bit boundary."""
    def enc(x):
        return [int(b) for b in O.encode_list(np.array(x, np.uint32), O.VARBYTE)["ctrl"]]
    assert enc([5]) == [0x85]
    assert enc([300]) == [0x2C, 0x82]
    assert enc([0]) == [0x80]
    assert enc([5, 300, 0]) == [0x85, 0x2C, 0x82, 0x80]
    with pytest.raises(O.OracleError):  # stream ends mid-integer
        O.decode_list(1, np.array([0x2C], np.uint8), np.zeros((0, 4), np.uint32), codec=O.VARBYTE)
    with pytest.raises(O.OracleError):  # more than 5 bytes without a terminator
        O.decode_list(1, np.zeros(6, np.uint8), np.zeros((0, 4), np.uint32), codec=O.VARBYTE)
    for k in range(0, 5):
        for v in {(1 << (7 * k)) - 1, 1 << (7 * k), min((1 << (7 * k + 7)) - 1, 2**32 - 1)}:
            if v < 0 or v >= 2**32:
                continue
            w = max(1, int(v).bit_length())
            assert len(enc([v])) == -(-w // 7), v
    assert len(enc([2**32 - 1])) == 5


def test_varbyte_round_trip():
    rng = np.random.default_rng(77)
    for n, bits in ((0, 1), (1, 32), (63, 7), (64, 8), (1000, 21), (500, 32)):
        x = rng.integers(0, 1 << bits, n, dtype=np.uint64).astype(np.uint32)
        e = O.encode_list(x, O.VARBYTE)
        assert np.array_equal(O.decode_list(n, e["ctrl"], e["data"], codec=O.VARBYTE), x)
    ln = rng.integers(0, 64, 200).astype(np.uint32)
    docs = np.concatenate([np.cumsum(rng.integers(1, 1000, int(k))).astype(np.uint32) for k in ln])
    bt = O.encode_batch(docs, ln, O.VARBYTE, delta=True)
    assert bt["data"].shape[0] == 0
    assert np.array_equal(O.decode_batch(bt, dgaps=True), docs)

"""Pins of the oracle's skip pointers (§7.5: "skip list pointers for posting blocks.
The skip distance ... 512 postings"; the entry format is in oracle/gc_oracle.h).

An entry must let a decoder start block b of a list with nothing before it.  The pin is a
resume decoder written here from the prose of the format (tests/_reader.py's bit reader for
the values, no oracle code): from the entry's control word and prefixes it decodes the
block's 512 ints, which must equal the generator's own values, and the entry's docID must
equal the generator's docID before the block.  A wrong word, quad, data or exception prefix
shifts or garbles the block and fails."""
import numpy as np
import pytest

import gen
import oracle as O
from tests import _reader as R

CODECS = ([(O.GROUP_SIMPLE, 0)] + [(O.GROUP_SCHEME, O.gsc_variant(cg, k)) for cg in (1, 2, 4, 8)
                                   for k in ("B", "CU")]
          + [(O.GROUP_SCHEME, O.gsc_variant(4, "IU")), (O.GROUP_SCHEME, O.gsc_variant(8, "IU")),
             (O.GROUP_AFOR, 0), (O.GROUP_PFD, 0), (O.GROUP_PFD, 1)])


def _bits(ctrl):
    return R._msb_bits(ctrl)


def resume_block(codec, variant, F, n, ctrl, data, exc, ent, blk):
    """The ints [512 blk, 512 blk + 512) of one list, decoded from skip entry `ent` only."""
    Q = -(-n // 4)
    qa, qb = 128 * blk, min(128 * blk + 128, Q)
    w = int(ent["word"])
    q = int(ent["quads"])
    dpos = int(ent["data_bits"])
    got = {}

    def keep(j, vals):
        if qa <= j < qb:
            got[j] = vals
    if codec == O.GROUP_SIMPLE:
        assert dpos == 32 * 8 * w                   # one vector (32 lane-bits) per selector
        s = 8 * w                                   # 8 nibbles per word; one vector each
        while q < qb:
            sel = (int(ctrl[s // 2]) >> (0 if s % 2 == 0 else 4)) & 15
            for t in range(R.NUM[sel]):
                keep(q + t, R.read_quad(data, s, t * R.BW[sel], R.BW[sel]))
            q += R.NUM[sel]
            s += 1
    elif codec == O.GROUP_SCHEME:
        cg, kind = 1 << (variant & 3), ("B", "CU", "IU")[variant >> 2]
        if kind == "B":
            fw = {1: 5, 2: 4, 4: 3, 8: 2}[cg]
            per_unit = {1: 3, 2: 2, 4: 2, 8: 4}[cg]
            unit_bytes = 2 if cg == 1 else 1
            def field_bit(j):                       # a field's first control bit (A18)
                u, f = divmod(j, per_unit)
                return 8 * u * unit_bytes + f * fw
            # the word's first field is quad `quads`: the first field at or after bit 32 w
            assert field_bit(q) >= 32 * w and (q == 0 or field_bit(q - 1) < 32 * w)
            j = q
            while j < qb:
                u, f = divmod(j, per_unit)
                unit = sum(int(ctrl[u * unit_bytes + i]) << (8 * i) for i in range(unit_bytes))
                bw = cg * (((unit >> (f * fw)) & ((1 << fw) - 1)) + 1)
                keep(j, R.read_quad(data, 0, dpos, bw))
                dpos += bw
                j += 1
        else:
            bits = _bits(ctrl)
            p = 32 * w
            if kind == "CU":
                assert dpos == cg * 32 * w          # complete unary: the closed form
                # the word owns the codes whose terminating 0 it holds: the first one starts
                # one bit after the last 0 before the word (or at the list's first bit)
                while p > 0 and bits[p - 1] == 1:
                    p -= 1
                dpos = cg * p                       # a code's data offset is CG x its start bit
            j = q
            while j < qb:
                if kind == "IU" and p % 8 and all(bits[p:(p // 8 + 1) * 8]):
                    p = (p // 8 + 1) * 8
                start, ones = p, 0
                while bits[p] == 1:
                    ones, p = ones + 1, p + 1
                p += 1
                bw = cg * (ones + 1)
                keep(j, R.read_quad(data, 0, cg * start if kind == "CU" else dpos, bw))
                dpos += bw
                j += 1
    elif codec == O.GROUP_AFOR:
        assert dpos % 32 == 0                       # frames start whole vectors
        f, vec = 4 * w, dpos // 32                  # header bytes
        while q < qb:
            h = int(ctrl[f])
            L, bw = (8, 16, 32)[h & 3], ((h >> 2) & 31) + 1
            for t in range(L):
                keep(q + t, R.read_quad(data, vec, t * bw, bw))
            vec += -(-L * bw // 32)
            q += L
            f += 1
    else:
        assert dpos % 32 == 0                       # frames start whole vectors
        f, vec, e = w, dpos // 32, int(ent["exc_bytes"])   # one 4-byte header per frame
        pb = 1 if 4 * F <= 256 else 2
        while q < qb:
            b, wcode = int(ctrl[4 * f]), int(ctrl[4 * f + 1])
            count = int(ctrl[4 * f + 2]) | (int(ctrl[4 * f + 3]) << 8)
            qf = min(F, Q - q)
            slots = []
            for j in range(qf):
                slots += R.read_quad(data, vec, j * b, b)
            wb = (0, 1, 2, 4)[wcode]
            for i in range(count):
                pos = sum(int(exc[e + i * pb + t]) << (8 * t) for t in range(pb))
                slots[pos] = sum(int(exc[e + count * pb + i * wb + t]) << (8 * t) for t in range(wb))
            for j in range(qf):
                keep(q + j, slots[4 * j:4 * j + 4])
            e += count * (pb + wb)
            vec += -(-qf * b // 32)
            q += F
            f += 1
    out = []
    for j in range(qa, qb):
        out += got[j]
    return out[:min(512, n - 512 * blk)]


def check_batch(values, list_n, codec, variant, frame_quads=32, delta=False):
    bt = O.encode_batch(values, list_n, codec, variant, delta=delta, frame_quads=frame_quads)
    off, ent = O.build_skip(bt)
    assert off[0] == 0 and int(off[-1]) == len(ent)
    starts = np.concatenate([[0], np.cumsum(list_n.astype(np.int64))])
    data = bt["data"].reshape(-1, 4)
    checked = 0
    for l, n in enumerate(list_n.tolist()):
        assert int(off[l + 1] - off[l]) == -(-n // 512)
        if n == 0:
            continue
        x = values[starts[l]:starts[l + 1]].astype(np.uint64)
        gaps = np.diff(x, prepend=np.uint64(0)) % (1 << 32) if delta else x
        c0, c1 = int(bt["ctrl_off"][l]), int(bt["ctrl_off"][l + 1])
        d0, e0 = int(bt["data_off"][l]), int(bt["exc_off"][l])
        for b in range(-(-n // 512)):
            e = ent[int(off[l]) + b]
            want_doc = int(gaps[:512 * b].sum() % (1 << 32))
            assert int(e["docid"]) == want_doc, (l, b)
            blk = resume_block(codec, variant, frame_quads, n, bt["ctrl"][c0:c1], data[d0:],
                               bt["exc"][e0:], e, b)
            assert blk == gaps[512 * b:512 * b + 512].tolist(), (l, b)
            checked += 1
    return checked


@pytest.mark.parametrize("codec,variant", CODECS, ids=[f"{c}-{v}" for c, v in CODECS])
def test_skip_entries_resume_every_block(codec, variant):
    rng = np.random.default_rng(4000 + 16 * codec + variant)
    w = gen.random_lists(rng, 12, 6000, 17, 0.03)
    ln = np.concatenate([w.list_n, np.array([0, 511, 512, 513, 1024, 1, 2047], np.uint32)])
    extra = rng.integers(0, 1 << 20, int(ln[len(w.list_n):].sum())).astype(np.uint32)
    vals = np.concatenate([w.values, extra])
    assert check_batch(vals, ln, codec, variant) > 40


def test_skip_docids_of_a_docid_stream():
    """With docIDs as input (the encoder takes the d-gaps), an entry's docID is the docID
    just before its block, the carry a range decode starts from."""
    w = gen.config(5, scale=2 ** -16)
    assert check_batch(w.values, w.list_n, O.GROUP_SCHEME, O.gsc_variant(1, "CU"), delta=True) > 0


def test_skip_pfd_frame_128():
    rng = np.random.default_rng(8)
    w = gen.random_lists(rng, 5, 5000, 20, 0.1)
    assert check_batch(w.values, w.list_n, O.GROUP_PFD, 0, frame_quads=128) > 0


@pytest.mark.parametrize("field,delta", [("word", 1), ("quads", 1), ("data_bits", 1), ("docid", 1)])
def test_skip_pin_catches_a_wrong_entry(field, delta):
    """The pin has teeth: one entry changed by one unit fails it."""
    rng = np.random.default_rng(9)
    w = gen.random_lists(rng, 4, 4000, 15, 0.0)
    ln = np.array([3000, 2600, 1800], np.uint32)
    # widths that change every 32..160 ints, so neighbouring groups differ (a shifted
    # control position cannot decode the same ints)
    widths = np.repeat(rng.integers(1, 24, 400), rng.integers(32, 160, 400))[:int(ln.sum())]
    vals = (rng.integers(0, 1 << 24, int(ln.sum())) & ((1 << widths) - 1)).astype(np.uint32)
    for codec, variant in [(O.GROUP_SCHEME, O.gsc_variant(2, "B")), (O.GROUP_AFOR, 0)]:
        bt = O.encode_batch(vals, ln, codec, variant)
        off, ent = O.build_skip(bt)
        e = ent[int(off[1]) + 2].copy()
        e[field] = e[field] + delta
        data = bt["data"].reshape(-1, 4)
        c0, c1 = int(bt["ctrl_off"][1]), int(bt["ctrl_off"][2])
        want = vals[3000 + 1024:3000 + 1536].tolist()
        if field == "docid":
            assert int(e["docid"]) != int(vals[3000:3000 + 1024].astype(np.uint64).sum() % (1 << 32))
            continue
        try:
            got = resume_block(codec, variant, 32, 2600, bt["ctrl"][c0:c1],
                               data[int(bt["data_off"][1]):], bt["exc"], e, 2)
        except (IndexError, KeyError, AssertionError):
            got = None
        assert got != want, (codec, field)

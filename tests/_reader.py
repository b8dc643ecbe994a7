"""An independent, bit-at-a-time reader of the batch stream format, written from the
prose of PAPER.md (and the readings in DESIGN.md §3), used only to pin the oracle's
byte layout.  It shares nothing with oracle/gc_oracle.c: values are assembled one
bit at a time from where the prose says each bit lives.
"""
from __future__ import annotations

NUM = [32, 16, 10, 8, 6, 5, 4, 3, 2, 1]   # Table III
BW = [1, 2, 3, 4, 5, 6, 8, 10, 16, 32]


def lane_bit(data, vec: int, lane: int, bit: int) -> int:
    """Bit `bit` (0 = least significant) of component `lane` of vector `vec`."""
    return (int(data[vec][lane]) >> bit) & 1


def read_value(data, base_vec: int, pos: int, bw: int, lane: int) -> int:
    """The bw-bit value whose first bit sits at lane bit position `pos`.  Values fill a
    component from its least-significant bit upward (A2).  If only r < bw bits remain
    in the current component, the value's r HIGH bits are there and its bw-r LOW bits
    start the next vector's component (A3)."""
    vec, off = base_vec + pos // 32, pos % 32
    r = 32 - off
    v = 0
    if bw <= r:
        for i in range(bw):
            v |= lane_bit(data, vec, lane, off + i) << i
    else:
        lo = bw - r
        for i in range(r):                       # value bits lo..bw-1 in the current vector
            v |= lane_bit(data, vec, lane, off + i) << (lo + i)
        for i in range(lo):                      # value bits 0..lo-1 in the next vector
            v |= lane_bit(data, vec + 1, lane, i) << i
    return v


def read_quad(data, base_vec, pos, bw):
    return [read_value(data, base_vec, pos, bw, k) for k in range(4)]


def _msb_bits(ctrl):
    """Control bytes as a list of bits in stream order: MSB of byte 0 first (A16)."""
    out = []
    for b in ctrl:
        for i in range(7, -1, -1):
            out.append((int(b) >> i) & 1)
    return out


def decode_group_simple(n, ctrl, data):
    Q = -(-n // 4)
    out, s = [], 0
    while len(out) < 4 * Q:
        sel = (int(ctrl[s // 2]) >> (0 if s % 2 == 0 else 4)) & 15   # low nibble first (A6)
        assert sel <= 9
        c = min(NUM[sel], Q - len(out) // 4)
        for t in range(c):
            out += read_quad(data, s, t * BW[sel], BW[sel])
        s += 1
    return out[:n]


def decode_group_scheme(n, ctrl, data, cg, kind):
    Q = -(-n // 4)
    lds = []
    if kind == "B":
        fw = {1: 5, 2: 4, 4: 3, 8: 2}[cg]       # 5 - log2 CG
        per_unit = {1: 3, 2: 2, 4: 2, 8: 4}[cg]  # fields per 16-bit (CG=1) or 8-bit unit
        unit_bytes = 2 if cg == 1 else 1
        for j in range(Q):
            u, f = divmod(j, per_unit)
            unit = sum(int(ctrl[u * unit_bytes + i]) << (8 * i) for i in range(unit_bytes))
            lds.append(((unit >> (f * fw)) & ((1 << fw) - 1)) + 1)   # units = LD + 1
    else:
        bits = _msb_bits(ctrl)
        p = 0
        while len(lds) < Q:
            if kind == "IU" and p % 8 and all(bits[p:(p // 8 + 1) * 8]):
                p = (p // 8 + 1) * 8                                   # byte padding (A17)
            ones = 0
            while bits[p] == 1:
                ones, p = ones + 1, p + 1
            p += 1
            lds.append(ones + 1)                                       # '1110' = 4 (A15)
    out, pos = [], 0
    for u in lds:
        bw = cg * u                                                    # Eq. (2)
        out += read_quad(data, 0, pos, bw)
        pos += bw
    return out[:n]


def decode_group_afor(n, ctrl, data):
    Q = -(-n // 4)
    out, f, vec = [], 0, 0
    while len(out) < 4 * Q:
        h = int(ctrl[f])
        L, bw = (8, 16, 32)[h & 3], ((h >> 2) & 31) + 1                  # A22
        for t in range(L):
            out += read_quad(data, vec, t * bw, bw)
        vec += -(-L * bw // 32)
        f += 1
    return out[:n]


def decode_group_pfd(n, ctrl, data, exc, F=32):
    Q = -(-n // 4)
    out, vec, e = [], 0, 0
    pb = 1 if 4 * F <= 256 else 2
    for f in range(-(-Q // F)):
        b, wcode = int(ctrl[4 * f]), int(ctrl[4 * f + 1])
        count = int(ctrl[4 * f + 2]) | (int(ctrl[4 * f + 3]) << 8)
        q = min(F, Q - f * F)
        slots = []
        for j in range(q):
            slots += read_quad(data, vec, j * b, b)
        wb = (0, 1, 2, 4)[wcode]
        pos = [sum(int(exc[e + i * pb + t]) << (8 * t) for t in range(pb)) for i in range(count)]
        for i in range(count):
            slots[pos[i]] = sum(int(exc[e + count * pb + i * wb + t]) << (8 * t) for t in range(wb))
        e += count * (pb + wb)
        vec += -(-q * b // 32)
        out += slots
    return out[:n]

"""Synthetic posting-list workloads for BASELINE.json's five configs.

The paper measures on GOV2, ClueWeb09B, Wikipedia and Twitter;
none is available, so these seeded generators stand in for them with the shapes
the configs name.  Readings of the configs (G1-G8) are those of SURVEY.md §8(d)
and are restated in DESIGN.md §4:

G1  binary units: 64M = 2^26, 256M = 2^28, 512M = 2^29, 16G = 2^34, max 1M = 2^20.
G2  Zipf = rank-frequency: len(r) = clip(floor(C r^-s), lo, hi); C by bisection so the
    sum is <= total, residue spread as +1 over lists below `hi` in rank order; the list
    order is then permuted with the seed.
G3  counter-based RNG (splitmix64) keyed by (seed, stream, list id, index), so any shard
    regenerates independently.
G4  Geometric(p) on {1,2,...}: 1 + floor(ln U / ln(1-p)), U in (0,1].
G5  exact uniform k-subset of [0,N): k iid uniforms in [0, N-k+1), sorted, d_j = u_j + j.
G6  gap-stream configs (2-4) produce gaps; their "docIDs" are the mod-2^32 prefix sums.
G8  Uniform[1, 2^16] inclusive; log-uniform floor(2^U), U ~ U[12,28); Bernoulli(0.08).
    A geometric run length is memoryless, so "runs of length ~Geom(0.02)" are drawn as a
    per-element Bernoulli(0.02) run end.
"""
from __future__ import annotations

import concurrent.futures
import dataclasses
import os

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = (x + np.uint64(0x9E3779B97F4A7C15)) & M64
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & M64
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & M64
        return z ^ (z >> np.uint64(31))


def _key(seed: int, stream: int) -> np.uint64:
    return splitmix64(np.array([(seed * 0x632BE59BD9B4E019 + stream * 0x85EBCA77C2B2AE63)
                                & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))[0]


def uniform01(seed: int, stream: int, list_ids: np.ndarray, idx: np.ndarray) -> np.ndarray:
    """U[0,1) from (seed, stream, list id, index within list) -- G3."""
    ctr = (list_ids.astype(np.uint64) << np.uint64(32)) | idx.astype(np.uint64)
    r = splitmix64(splitmix64(ctr) ^ _key(seed, stream))
    return (r >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def geometric(u: np.ndarray, p: float) -> np.ndarray:
    """G4: Geometric(p) on {1,2,...} by inverse CDF with U = 1-u in (0,1]."""
    if p >= 1.0:
        return np.ones(len(u), np.uint64)
    g = 1.0 + np.floor(np.log1p(-u) / np.log1p(-p))
    return np.minimum(g, 2.0 ** 32 - 1).astype(np.uint64)


def zipf_lengths(n_lists: int, total: int, s: float, lo: int, hi: int, seed: int,
                 use_torch: bool = True) -> np.ndarray:
    """G2: rank-frequency Zipf lengths summing exactly to `total`, in seeded random order."""
    r = np.arange(1, n_lists + 1, dtype=np.float64)
    w = r ** (-s)

    def lengths(C):
        return np.clip(np.floor(C * w), lo, hi).astype(np.int64)

    if lengths(0.0).sum() > total or lengths(1e30).sum() < total:
        raise ValueError("infeasible Zipf configuration")
    a, b = 0.0, float(hi) / w[-1] * 4 + 1.0
    total_of = lambda C: int(lengths(C).sum())  # noqa: E731
    if use_torch and n_lists > (1 << 20):
        # the same IEEE float64 multiply / floor / clip and an exact int64 sum, on torch's
        # threads (or the GPU): bit-identical lengths, minutes faster for config 5's 5e7
        try:
            import torch
            wt = torch.from_numpy(w)
            if torch.cuda.is_available():
                wt = wt.cuda()
            total_of = lambda C: int(torch.clamp(torch.floor(C * wt), lo, hi).to(torch.int64).sum())  # noqa: E731
        except ImportError:
            pass
    for _ in range(200):
        m = 0.5 * (a + b)
        if total_of(m) <= total:
            a = m
        else:
            b = m
    ln = lengths(a)
    residue = total - int(ln.sum())
    while residue > 0:
        room = np.nonzero(ln < hi)[0]
        take = room[:residue]
        ln[take] += 1
        residue -= len(take)
    perm = np.argsort(splitmix64(np.arange(n_lists, dtype=np.uint64) ^ _key(seed, 1 << 62)),
                      kind="stable")
    return ln[perm].astype(np.uint32)


CHUNK = 1 << 22  # elements per parallel work item


def _threads() -> int:
    return max(1, min(32, os.cpu_count() or 1))


def _run(jobs):
    """Runs the callables in `jobs` on a thread pool (numpy ufuncs release the GIL)."""
    if len(jobs) <= 1:
        return [j() for j in jobs]
    with concurrent.futures.ThreadPoolExecutor(_threads()) as ex:
        return list(ex.map(lambda j: j(), jobs))


def _chunk_index(list_n: np.ndarray, a: int, b: int):
    """(list id, index within list) of the elements [a, b) of the concatenated lists."""
    ln = list_n.astype(np.int64)
    ends = np.cumsum(ln)
    pos = np.arange(a, b, dtype=np.int64)
    lid = np.searchsorted(ends, pos, side="right")
    idx = pos - (ends[lid] - ln[lid])
    return lid, idx


def _elementwise(list_n: np.ndarray, fn, dtype=np.uint32) -> np.ndarray:
    """out[a:b] = fn(list id, index, a, b) over element chunks in parallel (G3 counters make
    every element's draw independent of the chunking)."""
    n = int(np.sum(list_n, dtype=np.int64))
    out = np.empty(n, dtype)

    def job(a, b):
        def f():
            lid, idx = _chunk_index(list_n, a, b)
            out[a:b] = fn(lid, idx, a, b)
        return f
    _run([job(a, min(n, a + CHUNK)) for a in range(0, n, CHUNK)])
    return out


def _list_chunks(list_n: np.ndarray):
    """Whole-list chunks [(first list, end list, first element, end element)] of ~CHUNK
    elements (a list longer than CHUNK is a chunk of its own)."""
    ends = np.cumsum(list_n.astype(np.int64))
    out, l0, e0 = [], 0, 0
    L = len(list_n)
    while l0 < L:
        l1 = int(np.searchsorted(ends, e0 + CHUNK, side="right"))
        l1 = min(L, max(l1, l0 + 1))
        e1 = int(ends[l1 - 1])
        out.append((l0, l1, e0, e1))
        l0, e0 = l1, e1
    return out


def uniform_subsets(list_n: np.ndarray, N: int, seed: int, list_id_base: int = 0) -> np.ndarray:
    """G5: for each list an exact uniform k-subset of [0,N), sorted (strictly increasing)."""
    n = int(np.sum(list_n, dtype=np.int64))
    out = np.empty(n, np.uint32)

    def job(l0, l1, e0, e1):
        def f():
            lid, idx = _chunk_index(list_n, e0, e1)
            u = uniform01(seed, 5, lid + list_id_base, idx)
            k = list_n[lid].astype(np.float64)
            v = np.floor(u * (N - k + 1)).astype(np.uint64)
            key = (lid.astype(np.uint64) << np.uint64(33)) | v  # lists stay contiguous
            key.sort()
            v = key & np.uint64((1 << 33) - 1)
            out[e0:e1] = (v + idx.astype(np.uint64)).astype(np.uint32)
        return f
    _run([job(*c) for c in _list_chunks(list_n)])
    return out


@dataclasses.dataclass
class Workload:
    name: str
    list_n: np.ndarray          # uint32 [n_lists]
    values: np.ndarray          # uint32: docIDs if delta else gaps
    delta: bool                 # True: values are docIDs, the encoder applies the d-gap
    seed: int
    note: str = ""

    @property
    def n_ints(self) -> int:
        v = self.values  # numpy, or a torch tensor (gen.gpu's device-resident draws)
        return int(v.numel()) if hasattr(v, "numel") else int(v.size)


def _gaps_cfg2(list_n, seed, base=0):
    def f(lid, idx, a, b):
        lid = lid + base
        pick = uniform01(seed, 21, lid, idx)
        geo = geometric(uniform01(seed, 22, lid, idx), 0.05)
        uni = 1 + np.floor(uniform01(seed, 23, lid, idx) * 65536.0).astype(np.uint64)
        return np.where(pick < 0.7, geo, uni).astype(np.uint32)
    return _elementwise(list_n, f)


def _gaps_cfg3(n, seed, replica=0):
    def f(lid, idx, a, b):
        lid = np.full(b - a, replica, np.int64)
        exc = uniform01(seed, 31, lid, idx) < 0.08
        big = np.floor(2.0 ** (12.0 + 16.0 * uniform01(seed, 32, lid, idx))).astype(np.uint64)
        geo = geometric(uniform01(seed, 33, lid, idx), 0.1)
        return np.where(exc, big, geo).astype(np.uint32)
    return _elementwise(np.array([n], np.uint32), f)


def _gaps_cfg4(list_n, seed, base=0):
    # run ends after element: Bernoulli(0.02) per element (G8)
    ends = _elementwise(list_n, lambda lid, idx, a, b:
                        (uniform01(seed, 41, lid + base, idx) < 0.02).astype(np.uint8), np.uint8)
    # parity of the run ends strictly before each element within its list: the inclusive
    # XOR-scan minus this element, minus the scan before the list's first element
    px = np.bitwise_xor.accumulate(ends) if len(ends) else ends
    ln = list_n.astype(np.int64)
    starts = np.cumsum(ln) - ln
    at_start = np.where(starts > 0, px[np.maximum(starts - 1, 0)], 0).astype(np.uint8) \
        if len(px) else np.zeros(len(ln), np.uint8)

    def f(lid, idx, a, b):
        sparse = (px[a:b] ^ ends[a:b] ^ at_start[lid]) == 1  # runs alternate, first has gap 1
        geo = geometric(uniform01(seed, 42, lid + base, idx), 0.001)
        return np.where(sparse, geo, 1).astype(np.uint32)
    return _elementwise(list_n, f)


CONFIGS = {
    1: dict(codec="group_simple", seed=0),
    2: dict(codec="group_scheme", seed=1),
    3: dict(codec="group_pfd", seed=2),
    4: dict(codec="group_afor", seed=3),
    5: dict(codec="all", seed=4),
}


def config(k: int, scale: float = 1.0, shard: int = 0, n_shards: int = 1,
           replica: int = 0) -> Workload:
    """BASELINE.json configs[k-1].  `scale` < 1 shrinks totals (list counts scale too)
    for CPU-sized tests; `shard`/`n_shards` select a contiguous list range at the sum(n)
    quantiles, each shard regenerated independently.  `replica` r draws an
    independent copy of the whole config (list ids offset by r*L in the RNG counters): the
    per-GPU input of weak-scaling runs."""
    if k == 1:
        L, total = max(1, int(round(1000 * scale))), int(round((1 << 20) * scale))
        ln = zipf_lengths(L, total, 1.1, 16, 65536, seed=0)
        ln, base = _shard(ln, shard, n_shards)
        return Workload("cfg1_group_simple", ln, uniform_subsets(ln, 1 << 24, 0, base + replica * L), True, 0,
                        "1,000 lists, 2^20 docIDs in [0,2^24), Zipf(1.1) lengths in [16,65536]")
    if k == 2:
        L, total = max(1, int(round(100_000 * scale))), int(round((1 << 26) * scale))
        ln = zipf_lengths(L, total, 1.1, 1, 1 << 20, seed=1)
        ln, base = _shard(ln, shard, n_shards)
        return Workload("cfg2_group_scheme", ln, _gaps_cfg2(ln, 1, base + replica * L), False, 1,
                        "100k lists, 2^26 gaps: 0.7 Geom(0.05) + 0.3 U[1,2^16]")
    if k == 3:
        n = int(round((1 << 28) * scale))
        return Workload("cfg3_group_pfd", np.array([n], np.uint32), _gaps_cfg3(n, 2, replica), False, 2,
                        "one stream of 2^28 gaps: Geom(0.1) + 8% log-uniform [2^12,2^28)")
    if k == 4:
        L, total = max(1, int(round(1_000_000 * scale))), int(round((1 << 29) * scale))
        ln = zipf_lengths(L, total, 1.1, 1, 1 << 20, seed=3)
        ln, base = _shard(ln, shard, n_shards)
        return Workload("cfg4_group_afor", ln, _gaps_cfg4(ln, 3, base + replica * L), False, 3,
                        "1M lists, 2^29 gaps: alternating runs gap=1 / Geom(0.001), run ~Geom(0.02)")
    if k == 5:
        L, total = max(1, int(round(50_000_000 * scale))), int(round((1 << 34) * scale))
        ln = zipf_lengths(L, total, 1.05, 1, 1 << 24, seed=4)
        ln, base = _shard(ln, shard, n_shards)
        return Workload("cfg5_all", ln, uniform_subsets(ln, 1 << 32, 4, base), True, 4,
                        "50M lists, 2^34 docIDs in [0,2^32), Zipf(1.05) lengths in [1,2^24]")
    raise ValueError(k)


def shard_bounds(list_n: np.ndarray, n_shards: int) -> np.ndarray:
    """Contiguous list ranges at the sum(n) quantiles."""
    cs = np.cumsum(list_n.astype(np.int64))
    total = int(cs[-1]) if len(cs) else 0
    b = [0]
    for r in range(1, n_shards):
        b.append(int(np.searchsorted(cs, total * r // n_shards, side="left")) + 1)
    b.append(len(list_n))
    return np.minimum(np.array(b, np.int64), len(list_n))


def _shard(ln, shard, n_shards):
    if n_shards == 1:
        return ln, 0
    b = shard_bounds(ln, n_shards)
    return ln[b[shard]:b[shard + 1]].copy(), int(b[shard])


def random_lists(rng: np.random.Generator, n_lists: int, max_len: int, bits: int,
                 spike: float = 0.0) -> Workload:
    """Small adversarial batches for parity tests: ragged lengths (incl. 0), uniform values of
    up to `bits` bits, plus optional full-width spikes."""
    ln = rng.integers(0, max_len + 1, n_lists).astype(np.uint32)
    n = int(ln.sum())
    v = rng.integers(0, 1 << bits, n, dtype=np.uint64).astype(np.uint32)
    if spike > 0:
        m = rng.random(n) < spike
        v[m] = rng.integers(0, 1 << 32, int(m.sum()), dtype=np.uint64).astype(np.uint32)
    return Workload(f"random_{n_lists}x{max_len}_{bits}b", ln, v, False, -1)


def checksum(list_n: np.ndarray, values: np.ndarray, list_base: int = 0):
    """G7 shard-additive checksum of decoded values (verification, not the method):
    (sum_l sum_i mix64(((l+base) << 32 | i) ^ (d_i * 0x9E3779B97F4A7C15)), sum d_i, sum n_l)
    mod 2^64, mix64 = splitmix64."""
    list_n = np.asarray(list_n, np.uint32)
    values = np.asarray(values)
    n = int(np.sum(list_n, dtype=np.int64))

    def job(a, b):
        def f():
            lid, idx = _chunk_index(list_n, a, b)
            d = values[a:b].astype(np.uint64)
            with np.errstate(over="ignore"):
                key = ((lid.astype(np.uint64) + np.uint64(list_base)) << np.uint64(32)) \
                    | idx.astype(np.uint64)
                h = splitmix64(key ^ ((d * np.uint64(0x9E3779B97F4A7C15)) & M64))
                return int(np.sum(h, dtype=np.uint64)), int(np.sum(d, dtype=np.uint64))
        return f
    parts = _run([job(a, min(n, a + CHUNK)) for a in range(0, n, CHUNK)])
    m = (1 << 64) - 1
    return (sum(p[0] for p in parts) & m, sum(p[1] for p in parts) & m,
            int(np.sum(list_n.astype(np.uint64))))

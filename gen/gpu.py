"""The config-5 generator on a GPU (torch), drawing exactly what gen.workloads draws.

Config 5 is 2^34 docIDs over 5*10^7 lists; one of its 8 shards is 2^31 docIDs, too much
to generate and encode on the host for 8 ranks at once.  These functions run the same
counter-based draws (G3: splitmix64 keyed by seed, stream, list id, index) and the same
exact uniform k-subsets (G5: floor(U * (N - k + 1)), sorted per list, + index) with torch
int64 / float64 tensor arithmetic: multiplication wraps mod 2^64 like numpy's uint64,
logical right shifts are arithmetic shifts masked, float64 multiply / floor are IEEE in
both.  tests/test_gen_gpu.py checks them against the numpy paths element by element.

Like the rest of gen/, this holds none of the method's arithmetic (no d-gap, no codec).
"""
from __future__ import annotations

import numpy as np

from .workloads import _key, shard_bounds, zipf_lengths

_M = (1 << 64) - 1


def _i64(c: int) -> int:
    """A uint64 constant as the int64 with the same bits."""
    c &= _M
    return c - (1 << 64) if c >= (1 << 63) else c


def _shr(x, k: int):
    """Logical right shift of an int64 tensor holding uint64 bits."""
    import torch
    return torch.bitwise_and(torch.bitwise_right_shift(x, k), (1 << (64 - k)) - 1)


def splitmix64_t(x):
    """gen.splitmix64 on an int64 tensor (uint64 bits, wrapping arithmetic)."""
    z = x + _i64(0x9E3779B97F4A7C15)
    z = (z ^ _shr(z, 30)) * _i64(0xBF58476D1CE4E5B9)
    z = (z ^ _shr(z, 27)) * _i64(0x94D049BB133111EB)
    return z ^ _shr(z, 31)


def uniform01_t(seed: int, stream: int, lid, idx):
    """gen.uniform01: U[0,1) from (seed, stream, list id, index)."""
    import torch
    ctr = torch.bitwise_left_shift(lid, 32) | idx
    r = splitmix64_t(splitmix64_t(ctr) ^ _i64(int(_key(seed, stream))))
    return _shr(r, 11).to(torch.float64) * (1.0 / 9007199254740992.0)


def uniform_subsets_t(list_n: np.ndarray, N: int, seed: int, list_id_base: int = 0,
                      device="cuda", chunk: int = 1 << 27):
    """gen.uniform_subsets (G5) as an int32 tensor (uint32 bits) on `device`, in chunks of
    whole lists of about `chunk` ints."""
    import torch
    ln = np.asarray(list_n, np.int64)
    n = int(ln.sum())
    out = torch.empty(n, dtype=torch.int32, device=device)
    ends = np.cumsum(ln)
    l0, e0 = 0, 0
    while l0 < len(ln):
        l1 = int(np.searchsorted(ends, e0 + chunk, side="right"))
        l1 = min(len(ln), max(l1, l0 + 1))
        e1 = int(ends[l1 - 1])
        cnt = torch.from_numpy(ln[l0:l1]).to(device)
        lid = torch.repeat_interleave(torch.arange(l1 - l0, dtype=torch.int64, device=device), cnt)
        starts = torch.cumsum(cnt, 0) - cnt
        idx = torch.arange(e1 - e0, dtype=torch.int64, device=device) - starts[lid]
        u = uniform01_t(seed, 5, lid + (l0 + list_id_base), idx)
        k = cnt[lid].to(torch.float64)
        v = torch.floor(u * (float(N) - k + 1.0)).to(torch.int64)
        key, _ = torch.sort(torch.bitwise_left_shift(lid, 33) | v)  # lists stay contiguous
        v = torch.bitwise_and(key, (1 << 33) - 1)
        out[e0:e1] = (v + idx).to(torch.int64).bitwise_and(0xFFFFFFFF).to(torch.int32)
        del lid, idx, u, k, v, key, starts
        l0, e0 = l1, e1
    return out


def checksum_t(list_n: np.ndarray, values, list_base: int = 0, chunk: int = 1 << 27):
    """gen.checksum (G7) of an int32 tensor holding uint32 values: (hash, sum, count) mod 2^64."""
    import torch
    ln = np.asarray(list_n, np.int64)
    dev = values.device
    ends = np.cumsum(ln)
    h = s = 0
    l0, e0 = 0, 0
    while l0 < len(ln):
        l1 = int(np.searchsorted(ends, e0 + chunk, side="right"))
        l1 = min(len(ln), max(l1, l0 + 1))
        e1 = int(ends[l1 - 1])
        cnt = torch.from_numpy(ln[l0:l1]).to(dev)
        lid = torch.repeat_interleave(torch.arange(l0, l1, dtype=torch.int64, device=dev), cnt)
        starts = torch.cumsum(cnt, 0) - cnt
        idx = torch.arange(e1 - e0, dtype=torch.int64, device=dev) - starts[lid - l0]
        d = values[e0:e1].to(torch.int64).bitwise_and(0xFFFFFFFF)
        key = torch.bitwise_left_shift(lid + list_base, 32) | idx
        hh = splitmix64_t(key ^ (d * _i64(0x9E3779B97F4A7C15)))
        # wrapping int64 sums are the uint64 sums mod 2^64
        h = (h + int(hh.sum().item())) & _M
        s = (s + int(d.sum().item())) & _M
        l0, e0 = l1, e1
    return h, s, int(ln.sum())


def config5_lengths(scale: float = 1.0) -> np.ndarray:
    """The 5*10^7 Zipf(1.05) lengths of config 5 (gen.config(5)'s, G2)."""
    L, total = max(1, int(round(50_000_000 * scale))), int(round((1 << 34) * scale))
    return zipf_lengths(L, total, 1.05, 1, 1 << 24, seed=4)


def config5_list_base(scale: float, shard: int, n_shards: int, lengths=None) -> int:
    ln = config5_lengths(scale) if lengths is None else lengths
    return int(shard_bounds(ln, n_shards)[shard]) if n_shards > 1 else 0


def config5_shard_gpu(shard: int, n_shards: int = 8, scale: float = 1.0, device="cuda",
                      lengths=None):
    """Shard `shard` of config 5 (gen.config(5, scale, shard, n_shards)) with its docIDs
    drawn on `device`: (list_n uint32 numpy, docIDs int32 tensor, global id of its first
    list)."""
    ln = config5_lengths(scale) if lengths is None else lengths
    if n_shards > 1:
        b = shard_bounds(ln, n_shards)
        base = int(b[shard])
        ln = ln[b[shard]:b[shard + 1]].copy()
    else:
        base = 0
    return ln, uniform_subsets_t(ln, 1 << 32, 4, base, device=device), base

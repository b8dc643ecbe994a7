"""Multi-GPU plumbing of the decode path: host logic only.

Posting lists are independent, and the d-gap prefix sum never crosses a list, so the
path shards by list with no collective on the data path.  Each rank takes a contiguous
list range at the sum(n) quantiles (config 5, strong sharding of one 2^34-int workload)
or its own independently drawn replica of a config (configs 1-4, weak scaling), decodes it
on its own GPU, and after the timed region one all-reduce combines

  * the step time (MAX over ranks: the job is as fast as its slowest rank),
  * the decoded-int count, the device status bits and the parity verdict (SUM),
  * the G7 checksum triple (SUM mod 2^64; shard-additive because the hash keys on the
    global list id),

through torch.distributed (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

import dataclasses

import numpy as np


@dataclasses.dataclass
class Shard:
    workload: object       # gen.Workload of this rank
    list_base: int         # global id of the rank's first list (G7 checksum key)
    scaling: str           # "weak" (replicas) or "strong" (one workload split by list)


def shard_for_rank(config: int, scale: float, rank: int, world: int, strong: bool = False) -> Shard:
    """The input of `rank`.  Config 5 is one 2^34-int workload defined across the 8 GPUs of
    a box: it is split by list at the sum(n) quantiles into 8 shards and rank
    r decodes shard r % 8, so per-GPU work is fixed and 8 ranks decode exactly config 5.
    Configs 1-4 give every rank its own independently drawn replica.  Both are weak
    scaling (per-GPU work fixed as the rank count grows)."""
    import gen
    if config == 5 and strong:
        # strong scaling (primary): the same workload split into `world`
        # contiguous list ranges at the sum(n) quantiles, one per rank
        w = gen.config(5, scale=scale, shard=rank, n_shards=world)
        L = max(1, int(round(50_000_000 * scale)))
        total = int(round((1 << 34) * scale))
        ln = gen.zipf_lengths(L, total, 1.05, 1, 1 << 24, seed=4)
        return Shard(w, int(gen.shard_bounds(ln, world)[rank]), "strong")
    if config == 5:
        n_shards, shard = 8, rank % 8
        w = gen.config(5, scale=scale, shard=shard, n_shards=n_shards)
        # the shard's first global list id: the same quantile split gen.config applied
        L = max(1, int(round(50_000_000 * scale)))
        total = int(round((1 << 34) * scale))
        ln = gen.zipf_lengths(L, total, 1.05, 1, 1 << 24, seed=4)
        return Shard(w, int(gen.shard_bounds(ln, n_shards)[shard]), "weak")
    w = gen.config(config, scale=scale, replica=rank)
    return Shard(w, rank * len(w.list_n), "weak")


def reduce_run(pg, device, ms: float, n_ints: int, status: int, verified, checksum3):
    """All-reduce of one timed run.  Returns (max ms, total ints, OR-ed status as a sum of
    per-rank bits, all ranks verified?, summed checksum triple as uint64[3])."""
    import torch
    chk = np.asarray(checksum3, np.uint64).copy()
    if pg is None:
        return ms, int(n_ints), int(status), verified, chk
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    v = -1 if verified is None else int(bool(verified))
    s = torch.tensor([int(n_ints), int(status), v], dtype=torch.int64, device=device)
    pg.all_reduce(s)
    c = torch.from_numpy(chk.view(np.int64).copy()).to(device)
    pg.all_reduce(c)  # int64 wraparound == uint64 sum mod 2^64
    world = pg.get_world_size()
    all_verified = None if verified is None else int(s[2].item()) == world
    return (float(t.item()), int(s[0].item()), int(s[1].item()), all_verified,
            c.cpu().numpy().view(np.uint64).copy())

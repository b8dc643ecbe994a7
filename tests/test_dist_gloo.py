"""Multi-GPU host logic on CPU (-m "not gpu"): the list sharding of config 5 and the
all-reduce of one timed run (dist.reduce_run), with world_size 2 over gloo.  The oracle
stands in for each rank's GPU decode (no data-path collective exists)."""
import json
import os
import socket

import numpy as np
import pytest

import gen
import oracle as O
from paper_1502_01916_b200 import dist as gdist

SCALE5 = 2.0 ** -21   # config 5 at 24 lists / 8192 docIDs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_config5_shards_partition_the_workload():
    full = gen.config(5, scale=SCALE5)
    shards = [gdist.shard_for_rank(5, SCALE5, r, 8) for r in range(8)]
    assert all(s.scaling == "weak" for s in shards)
    # contiguous, ordered, covering: list lengths and docIDs concatenate to the whole
    assert np.array_equal(np.concatenate([s.workload.list_n for s in shards]), full.list_n)
    assert np.array_equal(np.concatenate([s.workload.values for s in shards]), full.values)
    bases = [s.list_base for s in shards]
    assert bases[0] == 0 and bases == sorted(bases)
    assert all(bases[r + 1] - bases[r] == len(shards[r].workload.list_n) for r in range(7))
    # balanced by sum(n): every shard within one list of total/8
    per = [int(s.workload.list_n.sum()) for s in shards]
    assert sum(per) == int(full.list_n.sum())
    assert max(per) - min(per) <= 2 * int(full.list_n.max())
    # the G7 checksum is shard-additive when keyed on the global list id
    want = gen.checksum(full.list_n, full.values)
    got = np.zeros(3, np.uint64)
    for s in shards:
        got += np.array(gen.checksum(s.workload.list_n, s.workload.values, s.list_base), np.uint64)
    assert [int(x) for x in got] == list(want)


def test_config5_strong_split_covers_the_workload():
    """Strong scaling: for every rank count the shards partition the same workload, and the
    G7 checksum summed over the shards equals the whole workload's."""
    full = gen.config(5, scale=SCALE5)
    want = gen.checksum(full.list_n, full.values)
    for world in (1, 2, 4, 8):
        shards = [gdist.shard_for_rank(5, SCALE5, r, world, strong=True) for r in range(world)]
        assert all(s.scaling == "strong" for s in shards)
        assert np.array_equal(np.concatenate([s.workload.values for s in shards]), full.values)
        got = np.zeros(3, np.uint64)
        for s in shards:
            got += np.array(gen.checksum(s.workload.list_n, s.workload.values, s.list_base), np.uint64)
        assert [int(x) for x in got] == list(want)


def test_replicas_are_independent_draws():
    a = gdist.shard_for_rank(2, 1 / 4096, 0, 2)
    b = gdist.shard_for_rank(2, 1 / 4096, 1, 2)
    assert np.array_equal(a.workload.list_n, b.workload.list_n)     # same shape
    assert not np.array_equal(a.workload.values, b.workload.values)  # different gaps
    assert b.list_base == len(a.workload.list_n)


def _rank_main(rank, world, port, config, scale, outpath):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sh = gdist.shard_for_rank(config, scale, rank, world)
    w = sh.workload
    enc = O.encode_batch(w.values, w.list_n, O.GROUP_SCHEME, O.gsc_variant(8, "IU"), delta=w.delta)
    docs = O.decode_batch(enc, dgaps=True)                 # this rank's decode
    ok = np.array_equal(docs, w.values) if w.delta else True
    chk = gen.checksum(w.list_n, docs, sh.list_base)
    ms, n, status, verified, c = gdist.reduce_run(dist, "cpu", 1.0 + rank, w.n_ints, rank * 16,
                                                   ok, chk)
    if rank == 0:
        with open(outpath, "w") as f:
            json.dump({"ms": ms, "n": n, "status": status, "verified": verified,
                       "chk": [int(x) for x in c]}, f)
    dist.destroy_process_group()


@pytest.mark.parametrize("config,scale", [(5, SCALE5), (2, 1 / 4096)])
def test_two_ranks_gloo_reduce(tmp_path, config, scale):
    import torch.multiprocessing as mp
    out = str(tmp_path / "r.json")
    mp.spawn(_rank_main, args=(2, _free_port(), config, scale, out), nprocs=2, join=True)
    r = json.load(open(out))
    shards = [gdist.shard_for_rank(config, scale, k, 2) for k in range(2)]
    assert r["ms"] == 2.0                                   # MAX over ranks
    assert r["n"] == sum(s.workload.n_ints for s in shards)  # SUM of decoded ints
    assert r["status"] == 16 and r["verified"] is True
    want = np.zeros(3, np.uint64)
    for s in shards:
        d = s.workload.values
        if not s.workload.delta:  # the docIDs of a gap stream: per-list prefix sums (A36)
            d = O.decode_batch(O.encode_batch(d, s.workload.list_n, O.GROUP_SCHEME,
                                              O.gsc_variant(8, "IU")), dgaps=True)
        want += np.array(gen.checksum(s.workload.list_n, d, s.list_base), np.uint64)
    assert r["chk"] == [int(x) for x in want]


def test_bench_gpus_flag_starts_its_own_ranks():
    """`python bench.py --gpus N` outside torchrun starts N ranks itself (torch.distributed.run,
    127.0.0.1 rendezvous): here 2 gloo ranks on CPU, each all-reducing its rank id."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--spawn-check"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    assert d["world"] == 2 and d["rank_sum"] == 1

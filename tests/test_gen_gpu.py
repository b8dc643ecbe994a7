"""The generators' fast paths (torch threads / the GPU) draw exactly what the reference
numpy paths draw: same lengths (G2), same docIDs (G5), same G7 checksum."""
import numpy as np
import pytest

import gen

torch = pytest.importorskip("torch")


def test_zipf_lengths_torch_path_is_bit_identical():
    a = gen.zipf_lengths((1 << 20) + 12345, 1 << 27, 1.05, 1, 1 << 24, seed=4)
    b = gen.zipf_lengths((1 << 20) + 12345, 1 << 27, 1.05, 1, 1 << 24, seed=4, use_torch=False)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("shard,n_shards", [(0, 8), (5, 8), (0, 1)])
def test_uniform_subsets_torch_equals_numpy(shard, n_shards):
    from gen import gpu as G
    w = gen.config(5, scale=2 ** -13, shard=shard, n_shards=n_shards)
    base = G.config5_list_base(2 ** -13, shard, n_shards)
    got = G.uniform_subsets_t(w.list_n, 1 << 32, 4, base, device="cpu", chunk=1 << 14)
    assert np.array_equal(got.numpy().view(np.uint32), w.values)
    h = G.checksum_t(w.list_n, got, base)
    assert h == gen.checksum(w.list_n, w.values, base)

"""N > 1 host logic on CPU: world-size-2 gloo processes shard a design by
rows, reduce their Gram statistics with the library's all-reduce, and
recover the single-process statistics and the reference fit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import hexf, load_golden
from paper_1604_04997_b200.api import GramStats
from paper_1604_04997_b200.dist import allreduce_gram, gather_shards, shard_bounds


def test_shard_bounds_cover_exactly():
    for n in (0, 1, 7, 167284151):
        for world in (1, 2, 3, 8):
            blocks = [shard_bounds(n, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, X, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = shard_bounds(X.shape[0], rank, world)
    Xs = torch.tensor(X[a:b])
    st = GramStats(Xs.T @ Xs, Xs.sum(0), Xs.abs().max(0).values.clone(), n_rows=b - a)
    allreduce_gram(st)
    out[rank] = (st.G.numpy().copy(), st.xt1.numpy().copy(), st.colmax.numpy().copy(), st.n_rows)
    dist.destroy_process_group()


def test_gloo_world2_gram_allreduce_equals_single_process():
    fit = [f for f in load_golden("fit_synthetic.json")["fits"] if f["name"] == "config3_f40_n4000"][0]
    counts = np.array(fit["counts"], dtype=np.float64)
    times = np.array([hexf(t) for t in fit["times"]])
    X = counts / times[:, None]
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, X, out), nprocs=2, join=True)
    G, s1, cm = X.T @ X, X.sum(0), np.abs(X).max(0)
    for r in range(2):
        g, x, c, n = out[r]
        np.testing.assert_allclose(g, G, rtol=1e-13)
        np.testing.assert_allclose(x, s1, rtol=1e-13)
        assert (c == cm).all() and n == X.shape[0]
    # both ranks hold bit-identical statistics -> identical redundant solves
    assert (out[0][0] == out[1][0]).all() and (out[0][1] == out[1][1]).all()


def _gather_worker(rank, world, port, total, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = shard_bounds(total, rank, world)
    local = torch.arange(a, b, dtype=torch.float64) * 0.5  # this rank's predictions
    g = gather_shards(local, total)
    out[rank] = None if g is None else g.numpy().copy()
    dist.destroy_process_group()


def test_gloo_world3_gather_shards_reassembles_the_grid():
    """Ragged shards (10 sizes over 3 ranks) gather back in grid order on rank 0."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gather_worker, args=(3, _free_port(), 10, out), nprocs=3, join=True)
    np.testing.assert_array_equal(out[0], np.arange(10) * 0.5)
    assert out[1] is None and out[2] is None

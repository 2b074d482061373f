"""Multi-rank path with the real kernels (no 8-GPU node needed): two gloo
ranks share cuda:0, each owns a contiguous block of sizes / rows
(shard_bounds), and runs what bench.py runs per GPU --

  * config 5: fused Gram of its rows -> allreduce_gram -> redundant solve ->
    one refinement step with the all-reduced double-double gradient ->
    fused residual objective (all-reduced), dist.fit_sharded;
  * config 4: the one-pass evaluate+predict of the six matmul variants over
    its block of the lattice, gathered on rank 0 (dist.gather_shards);

and the results must equal the single-rank run: weights within 1e-12
(only the order of the Gram / gradient sums differs), predictions bitwise."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

VARIANTS = ("matmul_tiled_g12x12", "matmul_tiled_g14x14", "matmul_tiled_g16x16",
            "matmul_naive_g16x12", "matmul_naive_g16x14", "matmul_naive_g16x16")
SIDE = 60
ROWS = 400_000


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _lattice(torch, a, b, unit):
    i = torch.arange(a, b, dtype=torch.int64, device="cuda")
    return {"n": ((i // (SIDE * SIDE) + 1) * unit).contiguous(), "m": (((i // SIDE) % SIDE + 1) * unit).contiguous(),
            "l": ((i % SIDE + 1) * unit).contiguous()}


def _fit_rows(torch, kc, a, b):
    """rows a..b of the config-5 style fit: tiled g16 at sizes 16*(u,v,w),
    stored timings with noise (simulate_time, sigma 0.02)"""
    import kc_oracle as ko
    prog = kc.load_program("matmul_tiled_g16x16")
    i = torch.arange(a, b, dtype=torch.int64, device="cuda")
    cols = {"n": (16 * (i // 10000 % 100 + 1)).contiguous(), "m": (16 * (i // 100 % 100 + 1)).contiguous(),
            "l": (16 * (i % 100 + 1)).contiguous()}
    T = kc.simulate_time(ko.simdev_reference_alpha(), prog, cols, sigma=0.02, seed=7)
    return prog, cols, T


def _rank_main(rank, world, port, out):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    sys.path[:0] = [str(root), str(root / "oracle"), str(root / "tests")]
    import torch
    import torch.distributed as dist

    import kc_oracle as ko
    import paper_1604_04997_b200 as kc
    from paper_1604_04997_b200.dist import fit_sharded, gather_shards, shard_bounds
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = shard_bounds(ROWS, rank, world)
    prog, cols, T = _fit_rows(torch, kc, a, b)
    alpha, rk, obj, n = fit_sharded(prog, cols, T, refine=1)
    sim = ko.simdev_reference_alpha()
    w = kc.ModelWeights(alpha=sim, covered=[x != 0 for x in sim])
    total = SIDE ** 3
    a, b = shard_bounds(total, rank, world)
    progs = [kc.load_program(v) for v in VARIANTS]
    preds = kc.predict_multi(progs, w, _lattice(torch, a, b, 336))
    full = gather_shards(preds.T.contiguous(), total)
    out[rank] = (list(alpha), rk, obj, n, None if full is None else full.cpu().numpy().copy())
    dist.destroy_process_group()


def test_two_ranks_on_one_gpu_equal_one_rank():
    import torch
    import torch.multiprocessing as mp

    import kc_oracle as ko
    import paper_1604_04997_b200 as kc
    from paper_1604_04997_b200.dist import fit_sharded
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_rank_main, args=(2, _free_port(), out), nprocs=2, join=True)
    # single rank, same rows / sizes
    prog, cols, T = _fit_rows(torch, kc, 0, ROWS)
    alpha, rk, obj, n = fit_sharded(prog, cols, T, refine=1)
    for r in range(2):
        a2, rk2, obj2, n2, _ = out[r]
        assert n2 == n == ROWS and rk2 == rk
        for x, y in zip(a2, alpha):
            assert abs(x - y) <= 1e-12 * abs(y) + 1e-30, (x, y)
        assert obj2 == pytest.approx(obj, rel=1e-9)
    assert out[0][0] == out[1][0]  # identical all-reduced statistics -> identical redundant solves
    sim = ko.simdev_reference_alpha()
    w = kc.ModelWeights(alpha=sim, covered=[x != 0 for x in sim])
    progs = [kc.load_program(v) for v in VARIANTS]
    want = kc.predict_multi(progs, w, _lattice(torch, 0, SIDE ** 3, 336)).T.contiguous().cpu().numpy()
    got = out[0][4]
    assert got.shape == want.shape and np.array_equal(got.view(np.int64), want.view(np.int64))
    assert out[1][4] is None

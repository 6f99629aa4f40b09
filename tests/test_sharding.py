"""Multi-rank host logic on CPU (gloo, world_size 2): point sharding and the
allreduce of partial normal equations (the only collective of the path).
The per-shard Gram here comes from the CPU oracle, standing in for K4."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2409_19156_b200.sharding import shard_range


def test_shard_range_partitions_exactly():
    for total in (0, 1, 7, 100_000, 100_001):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import zk_oracle as orc
    from paper_2409_19156_b200.series import allreduce_normal_equations

    rng = np.random.default_rng(0)
    P = 1001
    rho = np.sqrt(rng.uniform(size=P))
    theta = 2 * np.pi * rng.uniform(size=P)
    modes = orc.full_modes(8)
    coef = rng.standard_normal(len(modes))
    lo, hi = shard_range(P, world, rank)
    B = orc.basis_2d(modes, rho[lo:hi], theta[lo:hi])
    y = orc.basis_2d(modes, rho[lo:hi], theta[lo:hi]) @ coef
    G, r = allreduce_normal_equations(torch.from_numpy(B.T @ B), torch.from_numpy(B.T @ y))
    np.save(os.path.join(out_dir, f"G{rank}.npy"), G.numpy())
    np.save(os.path.join(out_dir, f"r{rank}.npy"), r.numpy())
    dist.destroy_process_group()


def test_gram_allreduce_two_ranks(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    import zk_oracle as orc
    rng = np.random.default_rng(0)
    P = 1001
    rho = np.sqrt(rng.uniform(size=P))
    theta = 2 * np.pi * rng.uniform(size=P)
    modes = orc.full_modes(8)
    coef = rng.standard_normal(len(modes))
    B = orc.basis_2d(modes, rho, theta)
    G_full, r_full = B.T @ B, B.T @ (B @ coef)
    G0, G1 = np.load(tmp_path / "G0.npy"), np.load(tmp_path / "G1.npy")
    r0, r1 = np.load(tmp_path / "r0.npy"), np.load(tmp_path / "r1.npy")
    assert np.array_equal(G0, G1) and np.array_equal(r0, r1)  # every rank holds the same sum
    assert np.abs(G0 - G_full).max() <= 1e-12 * np.abs(G_full).max()
    assert np.abs(r0 - r_full).max() <= 1e-12 * np.abs(r_full).max()
    x = np.linalg.solve(G0, r0)  # the solve every rank then performs
    assert np.abs(x - coef).max() < 1e-8

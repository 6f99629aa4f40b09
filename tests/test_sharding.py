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


def _gpu_fit_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2409_19156_b200 as zb
    rng = np.random.default_rng(5)
    P = 40_000
    rho = np.sqrt(rng.uniform(size=P))
    theta = 2 * np.pi * rng.uniform(size=P)
    modes = zb.full_mode_set(12)
    coef = rng.standard_normal(len(modes))
    y = zb.zernike_basis(rho, theta, [m.n for m in modes], [m.m for m in modes]) @ coef
    lo, hi = shard_range(P, world, rank)
    dev = torch.device("cuda", 0)
    x, G, r = zb.fit_sharded(modes, torch.tensor(rho[lo:hi], device=dev),
                             torch.tensor(theta[lo:hi], device=dev),
                             torch.tensor(y[lo:hi], device=dev))
    np.save(os.path.join(out_dir, f"x{rank}.npy"), x.cpu().numpy())
    np.save(os.path.join(out_dir, "coef.npy"), coef)
    dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_fit_on_the_gpu_two_ranks(tmp_path):
    """fit_sharded end to end on the GPU kernels: two ranks (gloo, sharing the
    one GPU) each accumulate the DMMA Gram of their shard, one allreduce, the
    same Cholesky solve everywhere -- identical on both ranks, and the
    coefficients are recovered (y = B c exactly)."""
    mp.spawn(_gpu_fit_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    x0, x1 = np.load(tmp_path / "x0.npy"), np.load(tmp_path / "x1.npy")
    coef = np.load(tmp_path / "coef.npy")
    assert np.array_equal(x0, x1)
    assert np.abs(x0 - coef).max() <= 1e-9


def test_packed_normal_equations_round_trip_cpu():
    """K5 wire format on CPU tensors: [upper(G) column-major | r], M(M+1)/2 + M
    doubles, and unpack restores the full symmetric G bit for bit."""
    from paper_2409_19156_b200 import _lib
    from paper_2409_19156_b200.series import pack_normal_equations, unpack_normal_equations
    rng = np.random.default_rng(3)
    for M in (1, 2, 7, 64):
        A = rng.standard_normal((M, M))
        G = torch.from_numpy(A + A.T)
        r = torch.from_numpy(rng.standard_normal(M))
        packed = pack_normal_equations(G, r)
        assert packed.numel() == M * (M + 1) // 2 + M == _lib.lib.zk_gram_packed_count(M)
        # column j of the upper triangle starts at j(j+1)/2
        for j in range(M):
            assert torch.equal(packed[j * (j + 1) // 2: j * (j + 1) // 2 + j + 1], G[: j + 1, j])
        G2, r2 = unpack_normal_equations(packed, M)
        assert torch.equal(G2, G) and torch.equal(r2, r)


@pytest.mark.gpu
def test_packed_normal_equations_gpu_kernels_match_cpu():
    from paper_2409_19156_b200.series import pack_normal_equations, unpack_normal_equations
    rng = np.random.default_rng(4)
    for M in (1, 5, 300, 1891):
        A = rng.standard_normal((M, M))
        G = torch.from_numpy(A + A.T)
        r = torch.from_numpy(rng.standard_normal(M))
        pc = pack_normal_equations(G, r)
        pg = pack_normal_equations(G.cuda(), r.cuda())
        assert torch.equal(pg.cpu(), pc)
        G2, r2 = unpack_normal_equations(pg, M)
        assert torch.equal(G2.cpu(), G) and torch.equal(r2.cpu(), r)


@pytest.mark.gpu
def test_library_nccl_allreduce_single_process():
    """zk_gram_allreduce (ncclCommInitAll clique over the visible devices) and
    the one-process-per-GPU communicator (zk_comm_*), at the box's device count
    (1 here: NCCL with one rank must return the input sum unchanged), and
    gram(parallel=True) -- per-GPU K4 partials summed through the library's
    NCCL path -- against the one-GPU gram."""
    import ctypes

    import paper_2409_19156_b200 as zb
    from paper_2409_19156_b200 import _lib
    assert _lib.nccl_version() >= 21800
    rng = np.random.default_rng(6)
    M = 97
    A = rng.standard_normal((M, M))
    G = torch.from_numpy(A + A.T).cuda()
    r = torch.from_numpy(rng.standard_normal(M)).cuda()
    G0, r0 = G.clone(), r.clone()
    ctx = _lib.context(0)
    ctx.set_stream(None)
    arr = ctypes.c_void_p * 1
    _lib.check(_lib.lib.zk_gram_allreduce(arr(ctx.handle.value), 1, arr(G.data_ptr()),
                                          arr(r.data_ptr()), M, 0), "zk_gram_allreduce")
    assert torch.equal(G, G0) and torch.equal(r, r0)
    comm = _lib.Comm(ctx, _lib.Comm.unique_id(), 1, 0)
    assert comm.info() == (1, 0)
    G1, r1 = zb.allreduce_normal_equations(G.clone(), r.clone(), comm=comm)
    torch.cuda.synchronize()
    assert torch.equal(G1, G0) and torch.equal(r1, r0)
    del comm

    modes = zb.full_mode_set(16)
    P = 20_000
    rho = np.sqrt(rng.uniform(size=P))
    theta = 2 * np.pi * rng.uniform(size=P)
    c = rng.standard_normal(len(modes))
    y = zb.series_eval(modes, c, rho, theta)
    Gs, bs = zb.gram(modes, rho, theta, y)
    Gp, bp = zb.gram(modes, rho, theta, y, parallel=True)
    if len(zb.evaluate.parallel_devices()) == 1:
        assert np.array_equal(Gp, Gs) and np.array_equal(bp, bs)
    else:
        assert np.abs(Gp - Gs).max() <= 1e-12 * np.abs(Gs).max()
    x = zb.fit(modes, rho, theta, y, parallel=True)
    assert np.abs(x - c).max() <= 1e-9
    fp = zb.series_eval(modes, c, rho, theta, parallel=True)
    assert np.array_equal(fp, y)

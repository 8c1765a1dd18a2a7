"""Multi-process (world size 2, gloo, CPU) test of the sharding host logic in
paper_2208_00049_b200/dist.py: node shards of the tile-sorted order and the
all_reduce that sums forward outputs / adjoint partial grids (linearity,
DESIGN.md §8). The per-shard compute here is the CPU oracle (tests may call
it); on GPUs the same host logic drives the CUDA library."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


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
    from oracle import binning, nfft as onfft
    from paper_2208_00049_b200 import workloads
    from paper_2208_00049_b200.dist import allreduce_sum, shard_range

    w = workloads.make("cfg3_2d_512", seed=21, N=(24, 20), M=700, m=3)
    N, m = w["N"], w["m"]
    Nt = tuple(2 * n for n in N)
    perm, _, _ = binning.bin_nodes(w["nodes"], Nt, (8, 8))
    b, e = shard_range(w["M"], rank, world)
    mine = perm[b:e]
    # forward: my shard's node values, zeros elsewhere, summed over ranks
    f = np.zeros(w["M"], complex)
    f[mine] = onfft.forward(w["nodes"][mine], w["fhat"][0], N, m, 2.0)
    ft = torch.from_numpy(f)
    allreduce_sum(ft)
    # adjoint: partial N-grid of my shard, summed over ranks
    y = onfft.adjoint(w["nodes"][mine], w["f"][0][mine], N, m, 2.0)
    yt = torch.from_numpy(np.ascontiguousarray(y))
    allreduce_sum(yt)
    if rank == 0:
        np.save(os.path.join(out_dir, "f.npy"), ft.numpy())
        np.save(os.path.join(out_dir, "y.npy"), yt.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_partitions():
    from paper_2208_00049_b200.dist import shard_range
    for n in (0, 1, 7, 1000, 1001):
        for world in (1, 2, 3, 8):
            ranges = [shard_range(n, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (b0, e0), (b1, e1) in zip(ranges[:-1], ranges[1:]):
                assert e0 == b1
            sizes = [e - b for b, e in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_two_rank_gloo_shards_sum_to_full_transform(tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    from oracle import nfft as onfft
    from paper_2208_00049_b200 import workloads
    from conftest import rel_l2
    w = workloads.make("cfg3_2d_512", seed=21, N=(24, 20), M=700, m=3)
    ref_f = onfft.forward(w["nodes"], w["fhat"][0], w["N"], 3, 2.0)
    ref_y = onfft.adjoint(w["nodes"], w["f"][0], w["N"], 3, 2.0)
    assert rel_l2(np.load(tmp_path / "f.npy"), ref_f) < 1e-14
    assert rel_l2(np.load(tmp_path / "y.npy"), ref_y) < 1e-14


def _grid_worker(rank, world, port, out_dir, g_n):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2208_00049_b200.dist import allreduce_sum, grid_groups, shard_range
    gb, n_b, grp = grid_groups(world, g_n)
    b0, b1 = shard_range(32, gb, n_b)
    # the node group sums ones: its size
    t = torch.ones(1)
    allreduce_sum(t, grp)
    np.save(os.path.join(out_dir, f"r{rank}.npy"), np.array([gb, n_b, b0, b1, int(t.item())]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("g_n", [1, 2, 4])
def test_four_rank_batch_by_node_grid(g_n, tmp_path):
    """HybridNfft's rank layout (dist.grid_groups): G = 4 ranks as G_b x G_n;
    the batch groups partition the 32 vectors of config 5, and the node-shard
    group of every rank has G_n members."""
    mp.spawn(_grid_worker, args=(4, _free_port(), str(tmp_path), g_n), nprocs=4, join=True)
    rows = [np.load(tmp_path / f"r{r}.npy") for r in range(4)]
    seen = {}
    for r, (gb, n_b, b0, b1, size) in enumerate(rows):
        assert gb == r // g_n and n_b == 4 // g_n and size == g_n
        seen[gb] = (b0, b1)
    spans = sorted(seen.values())
    assert spans[0][0] == 0 and spans[-1][1] == 32
    assert all(e0 == b1 for (_, e0), (b1, _) in zip(spans[:-1], spans[1:]))

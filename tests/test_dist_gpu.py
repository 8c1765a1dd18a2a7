"""Multi-process sharding THROUGH THE PRODUCT KERNELS (world size 2, gloo
collectives, both ranks on cuda:0 — the only GPU of the test box; the ranks'
kernels never wait on each other, the collectives run on the host):
ShardedNfft (node shards of the cell-sorted order + all_reduce, PAPER.md's
linearity) and HybridNfft (batch split x node groups, config 5's
"sharded by batch and nodes") against the CPU oracle."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir, case):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2208_00049_b200 import workloads
    from paper_2208_00049_b200.dist import HybridNfft, ShardedNfft
    if case == "nodeshard_2d":
        w = workloads.make("cfg3_2d_512", seed=51, N=(40, 36), M=2500, m=4)
        nodes = torch.from_numpy(w["nodes"]).cuda()
        obj = ShardedNfft(nodes, w["N"], m=4).precompute()
        f = obj.forward(torch.from_numpy(w["fhat"]).cuda())
        y = obj.adjoint(torch.from_numpy(w["f"]).cuda())
        sl = (0, 1)
    elif case == "nodeshard_1d_c64":
        w = workloads.make("cfg2_1d_2e18", seed=52, N=(512,), M=700, m=5)
        nodes = torch.from_numpy(w["nodes"].astype(np.float32)).cuda()
        obj = ShardedNfft(nodes, w["N"], m=5, precision="c64").precompute()
        f = obj.forward(torch.from_numpy(w["fhat"].astype(np.complex64)).cuda())
        y = obj.adjoint(torch.from_numpy(w["f"].astype(np.complex64)).cuda())
        sl = (0, 1)
    else:  # batch split over the 2 ranks (g_n = 1) or one node group of 2 (g_n = 2)
        g_n = 2 if case == "hybrid_nodes" else 1
        w = workloads.make("cfg5_radial_s2", seed=53, N=(32, 40), M=1500, m=4, batch=6)
        nodes = torch.from_numpy(w["nodes"]).cuda()
        obj = HybridNfft(nodes, w["N"], w["batch"], g_n=g_n, m=4, precision="c64").precompute()
        b0, b1 = obj.batch_range
        f = obj.forward(torch.from_numpy(np.ascontiguousarray(w["fhat"][b0:b1])).cuda())
        y = obj.adjoint(torch.from_numpy(np.ascontiguousarray(w["f"][b0:b1])).cuda())
        sl = (b0, b1)
    torch.cuda.synchronize()
    np.save(os.path.join(out_dir, f"f{rank}.npy"), f.cpu().numpy())
    np.save(os.path.join(out_dir, f"y{rank}.npy"), y.cpu().numpy())
    np.save(os.path.join(out_dir, f"s{rank}.npy"), np.array(sl))
    obj.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", ["nodeshard_2d", "nodeshard_1d_c64", "hybrid_batch", "hybrid_nodes"])
def test_two_ranks_through_the_kernels(case, tmp_path):
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), case), nprocs=2, join=True)
    from oracle import nfft as onfft
    from paper_2208_00049_b200 import workloads
    from conftest import rel_l2
    if case == "nodeshard_2d":
        w, m, tol = workloads.make("cfg3_2d_512", seed=51, N=(40, 36), M=2500, m=4), 4, 1e-12
    elif case == "nodeshard_1d_c64":
        w, m, tol = workloads.make("cfg2_1d_2e18", seed=52, N=(512,), M=700, m=5), 5, 2e-5
        w["nodes"] = w["nodes"].astype(np.float32)
        w["fhat"] = w["fhat"].astype(np.complex64)
        w["f"] = w["f"].astype(np.complex64)
    else:
        w, m, tol = workloads.make("cfg5_radial_s2", seed=53, N=(32, 40), M=1500, m=4, batch=6), 4, 2e-5
    nodes = w["nodes"].astype(np.float64)
    rf = onfft.forward(nodes, w["fhat"].astype(np.complex128), w["N"], m, 2.0)
    ry = onfft.adjoint(nodes, w["f"].astype(np.complex128), w["N"], m, 2.0)
    covered = np.zeros(w["batch"], int)
    for rank in range(2):
        f = np.load(tmp_path / f"f{rank}.npy")
        y = np.load(tmp_path / f"y{rank}.npy")
        b0, b1 = np.load(tmp_path / f"s{rank}.npy")
        for i, b in enumerate(range(b0, b1)):
            assert rel_l2(f[i], rf[b]) <= tol, (rank, b)
            assert rel_l2(y[i], ry[b]) <= tol, (rank, b)
            covered[b] += 1
    # every vector is produced by every rank of its node group: 2 ranks when the vectors are replicated
    expect = 1 if case == "hybrid_batch" else 2
    assert (covered == expect).all(), covered

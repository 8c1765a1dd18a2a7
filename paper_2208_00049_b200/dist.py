"""Multi-GPU sharding of the NFFT over one node (one process per GPU, NCCL
through torch.distributed). Host-side plumbing only; all compute is in the
library's kernels.

The path shards by linearity:
* forward: each rank evaluates the nodes of its contiguous shard of the
  GLOBAL tile-sorted order over a replicated grid (every rank bins all nodes,
  so shards are spatially compact and the permutation is the oracle's);
  outputs are disjoint and are summed into place with one all_reduce.
* adjoint: each rank spreads its shard, runs the local FFT and crop, and the
  N-grid partial results are summed with one all_reduce (the N-grid is
  sigma^D times smaller than the oversampled grid).
* batches of independent transforms shard by batch with no collective.
"""

import torch
import torch.distributed as dist


def shard_range(n, rank, world):
    """Contiguous [begin, end) of n items for `rank` of `world` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n, world)
    begin = rank * base + min(rank, extra)
    end = begin + base + (1 if rank < extra else 0)
    return begin, end


def allreduce_sum(t, group=None):
    """In-place sum over ranks (complex tensors are reduced as real views)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return t
    view = torch.view_as_real(t) if t.is_complex() else t
    dist.all_reduce(view, op=dist.ReduceOp.SUM, group=group)
    return t


class ShardedNfft:
    """One NFFT split over the ranks of `group` by nodes (strong scaling)."""

    def __init__(self, nodes, N, group=None, **plan_kw):
        from . import NfftPlan
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        M = int(nodes.shape[0])
        self.range = shard_range(M, self.rank, self.world)
        self.plan = NfftPlan(nodes, N, node_range=self.range, **plan_kw)
        self.M = M

    def precompute(self):
        self.plan.precompute()
        return self

    def forward(self, fhat, out=None):
        if out is None:
            out = torch.zeros((self.plan.batch, self.M), dtype=self.plan.tdtype_c, device=fhat.device)
        else:
            out.zero_()
        self.plan.forward(fhat, out=out)
        return allreduce_sum(out, self.group)

    def adjoint(self, f, out=None):
        y = self.plan.adjoint(f, out=out)
        return allreduce_sum(y, self.group)

    def close(self):
        self.plan.close()

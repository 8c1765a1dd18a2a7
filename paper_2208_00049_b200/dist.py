"""Multi-GPU sharding of the NFFT over one node (one process per GPU, NCCL
through torch.distributed). Host-side plumbing only; all compute is in the
library's kernels.

The path shards by linearity:
* node shards (ShardedNfft): every rank bins ALL nodes (cheap, bit-exact with
  the oracle's order) and processes the contiguous range [b, e) of the cell-
  sorted order given by shard_range, so shards are spatially compact.
  - forward: a rank writes the values of its shard's nodes into a zeroed
    M-vector and one all_reduce(sum) assembles the full output (the slots of
    the other ranks are zero);
  - adjoint: a rank spreads its shard, runs the local FFT and crop, and the
    partial N-grids are summed with one all_reduce (the N-grid is sigma^D
    times smaller than the oversampled grid, SURVEY §8(e) variant ii).
* batch shards (HybridNfft): the B independent transforms of a batch (BASELINE
  config 5) are split over G_b rank groups, 32/G_b vectors per group with no
  collective; inside a group the G_n ranks node-shard the group's vectors as
  above (G = G_b x G_n).
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


SELF = "self"  # a group of this rank alone (no node sharding; distinct from None = the world)


def _world(group):
    if group is SELF or not dist.is_available() or not dist.is_initialized():
        return 1
    return dist.get_world_size(group)


def _rank(group):
    if group is SELF or not dist.is_available() or not dist.is_initialized():
        return 0
    return dist.get_rank(group)


def allreduce_sum(t, group=None):
    """In-place sum over the ranks of `group` (complex tensors are reduced as
    real views). With the gloo backend (CPU tests) CUDA tensors are reduced
    through a host copy."""
    if _world(group) == 1:
        return t
    view = torch.view_as_real(t) if t.is_complex() else t
    if view.is_cuda and dist.get_backend(group) == "gloo":
        host = view.cpu()
        dist.all_reduce(host, op=dist.ReduceOp.SUM, group=group)
        view.copy_(host)
    else:
        dist.all_reduce(view, op=dist.ReduceOp.SUM, group=group)
    return t


class ShardedNfft:
    """One (batched) NFFT split over the ranks of `group` by nodes (strong scaling)."""

    def __init__(self, nodes, N, group=None, **plan_kw):
        from . import NfftPlan
        self.group = group
        self.rank = _rank(group)
        self.world = _world(group)
        M = int(nodes.shape[0])
        self.range = shard_range(M, self.rank, self.world)
        self.plan = NfftPlan(nodes, N, node_range=self.range, **plan_kw)
        self.M = M

    def precompute(self):
        self.plan.precompute()
        return self

    def forward(self, fhat, out=None):
        """fhat (B, *N) replicated on every rank -> f (B, M), complete on every rank."""
        if out is None:
            out = torch.zeros((self.plan.batch, self.M), dtype=self.plan.tdtype_c, device=fhat.device)
        else:
            out.zero_()  # the other shards' slots must be zero before the sum
        self.plan.forward(fhat, out=out)
        return allreduce_sum(out, self.group)

    def adjoint(self, f, out=None):
        """f (B, M) replicated -> y (B, *N), complete on every rank."""
        y = self.plan.adjoint(f, out=out)
        return allreduce_sum(y, self.group)

    def close(self):
        self.plan.close()


def grid_groups(world, g_n):
    """Rank layout of a G_b x G_n grid: rank r is in batch group r // g_n and
    node-shard position r % g_n. Returns (batch_group_index, n_batch_groups,
    node_group) where node_group is the process group of the g_n ranks sharing
    this rank's batch slice (SELF when g_n == 1). Every rank must call this
    (new_group is collective)."""
    if g_n < 1 or world % g_n:
        raise ValueError(f"node-shard group size {g_n} must divide the world size {world}")
    rank = dist.get_rank() if dist.is_initialized() else 0
    n_b = world // g_n
    mine = SELF
    if g_n > 1:
        for gb in range(n_b):
            grp = dist.new_group(list(range(gb * g_n, (gb + 1) * g_n)))
            if gb == rank // g_n:
                mine = grp
    return rank // g_n, n_b, mine


class HybridNfft:
    """A batch of B independent transforms over G = G_b x G_n ranks: batch
    vectors shard_range(B, batch_group, G_b) on each batch group, nodes
    node-sharded inside the group (BASELINE config 5: "sharded by batch and
    nodes"). forward/adjoint take and return this rank's batch slice."""

    def __init__(self, nodes, N, batch, g_n=1, **plan_kw):
        init = dist.is_available() and dist.is_initialized()
        world = dist.get_world_size() if init else 1
        self.batch_group, self.n_batch_groups, self.node_group = grid_groups(world, g_n)
        self.batch_range = shard_range(int(batch), self.batch_group, self.n_batch_groups)
        nb = self.batch_range[1] - self.batch_range[0]
        if nb < 1:
            raise ValueError("more batch groups than batch vectors")
        plan_kw = {k: v for k, v in plan_kw.items() if k != "batch"}
        self.sharded = ShardedNfft(nodes, N, group=self.node_group, batch=nb, **plan_kw)
        self.plan = self.sharded.plan

    def precompute(self):
        self.sharded.precompute()
        return self

    def forward(self, fhat_slice, out=None):
        return self.sharded.forward(fhat_slice, out=out)

    def adjoint(self, f_slice, out=None):
        return self.sharded.adjoint(f_slice, out=out)

    def close(self):
        self.sharded.close()

"""Multi-GPU execution of pfor: shard the iteration space, one rank per GPU.

pfor iterations are independent by construction, so each
rank builds and runs the vectorized graph of its own contiguous block of
iterations [lo, hi) (`apps.pfor(..., shard=(lo, hi))`: the loop variable is
replaced by the constant ids lo..hi-1).  No collective runs
inside the data path.  Collectives happen only where outputs must meet:

* `gather_stacked`   -- one all-gather along axis 0 of a stacked output that
                        must be materialised on every rank (NCCL over NVLink);
* `allreduce_sum`    -- a sum over iterations (DP-SGD clipped-gradient sums,
                        `assign_add` reductions);
* everything else stays sharded (cfg3's 223 GB jacobian never fits one GPU).

Uneven splits are padded to the largest shard for the all-gather and trimmed
afterwards, so every rank issues identical collectives.  The host logic is
backend-agnostic: tests run it with `gloo` on CPU (world_size 2) using the
oracle executor as the per-rank compute.
"""

from __future__ import annotations

import numpy as np


def shard_range(n: int, world: int, rank: int) -> tuple:
    """Contiguous block of iterations for `rank`; sizes differ by at most 1."""
    base, extra = divmod(int(n), int(world))
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def balanced_order(lengths, world: int):
    """Iteration permutation for data-dependent trip counts (cfg5): sort by
    length and deal round-robin, so each contiguous shard gets a similar mix
    of long and short examples.  Returns (permutation, inverse)."""
    lengths = np.asarray(lengths)
    by_len = np.argsort(-lengths, kind="stable")
    buckets = [by_len[r::world] for r in range(world)]
    perm = np.concatenate(buckets)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(perm))
    return perm, inv


def _as_torch(x):
    import torch
    if isinstance(x, torch.Tensor):
        return x
    if hasattr(x, "torch_view"):
        return x.torch_view()
    return torch.as_tensor(np.asarray(x))


def gather_stacked(local, n_total: int, group=None):
    """All-gather a stacked [n_local, ...] tensor into [n_total, ...] on every
    rank (contiguous shards in rank order)."""
    import torch
    import torch.distributed as dist
    t = _as_torch(local).contiguous()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = [shard_range(n_total, world, r) for r in range(world)]
    width = max(hi - lo for lo, hi in sizes)
    pad = torch.zeros((width,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]].copy_(t)
    out = torch.empty((world * width,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    parts = [out[r * width: r * width + (hi - lo)] for r, (lo, hi) in enumerate(sizes)]
    del rank
    return torch.cat(parts, 0)


def allreduce_sum(local, group=None):
    """In-place sum over ranks of a per-rank partial (returns the tensor)."""
    import torch.distributed as dist
    t = _as_torch(local)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


class ShardedPfor:
    """Build + run one rank's shard of a workload and combine its outputs.

    `build(shard) -> Workload` must build the program for iterations
    shard=(lo, hi) (every builder in workloads.py takes `shard=`).
    `combine` lists, per output, "gather" | "sum" | "local".
    `executor_factory(graph)` returns an object with .run(feeds) /
    .run_device(feeds) -- the B200 Executor on GPUs; tests pass the oracle.
    """

    def __init__(self, build, n_total, combine, executor_factory, group=None):
        import torch.distributed as dist
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.group = group
        self.n_total = n_total
        self.shard = shard_range(n_total, self.world, self.rank)
        self.workload = build(self.shard)
        self.combine = list(combine)
        self.ex = executor_factory(self.workload.graph)

    def run(self, feeds=None, device_outputs=False):
        feeds = self.workload.feeds if feeds is None else feeds
        if device_outputs:
            outs = [o.torch_view() if hasattr(o, "torch_view") else o
                    for o in self.ex.run_device(feeds)]
        else:
            outs = [_as_torch(np.asarray(o.data)) for o in self.ex.run(feeds)]
        res = []
        for o, how in zip(outs, self.combine):
            if how == "gather":
                res.append(gather_stacked(o, self.n_total, self.group))
            elif how == "sum":
                res.append(allreduce_sum(o.clone(), self.group))
            else:
                res.append(o)
        return res

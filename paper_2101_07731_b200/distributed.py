"""Candidate sharding across the GPUs of one node.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  Each
rank owns a contiguous block of the collection; queries are replicated.
There are exactly two collectives per query batch:

  1. after the seed phase, an all-reduce(MIN) of the per-query best-so-far
     (so every shard prunes against the global best; float32/float64);
  2. after the finish phase, the lexicographic (distance, index) minimum:
     an all-reduce(MIN) of the float64 distance bits (non-negative IEEE
     doubles order like int64) followed by an all-reduce(MIN) of the index
     among ranks holding that distance -- the reference's lowest-index tie
     rule (search.py:173) across shards.

Counters are summed with one all-reduce(SUM).  Everything here also runs on
the gloo backend with CPU tensors (tests/test_distributed_cpu.py).
"""

from __future__ import annotations

import numpy as np

INT64_MAX = np.iinfo(np.int64).max


def shard_bounds(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous near-equal blocks; global index = start + local index."""
    base, extra = divmod(int(n_total), int(world))
    start = rank * base + min(rank, extra)
    stop = start + base + (1 if rank < extra else 0)
    return start, stop


def exchange_dbest(d_best, group=None):
    """In place: per-query best-so-far -> minimum over shards."""
    import torch.distributed as dist

    dist.all_reduce(d_best, op=dist.ReduceOp.MIN, group=group)
    return d_best


def combine_results(best_index, best_distance, group=None):
    """Lexicographic (distance, index) minimum across ranks.

    best_index: int64 (global indices, -1 = none on this shard);
    best_distance: float64.  Returns new (index, distance) tensors."""
    import torch
    import torch.distributed as dist

    dist_bits = best_distance.contiguous().view(torch.int64).clone()
    gmin = dist_bits.clone()
    dist.all_reduce(gmin, op=dist.ReduceOp.MIN, group=group)
    idx = torch.where((dist_bits == gmin) & (best_index >= 0), best_index,
                      torch.full_like(best_index, INT64_MAX))
    dist.all_reduce(idx, op=dist.ReduceOp.MIN, group=group)
    idx = torch.where(idx == INT64_MAX, torch.full_like(idx, -1), idx)
    return idx, gmin.view(torch.float64)


def sum_counters(counters, group=None):
    import torch.distributed as dist

    dist.all_reduce(counters, op=dist.ReduceOp.SUM, group=group)
    return counters


class ShardedSearch:
    """This rank's shard of a collection, searched with global combination."""

    def __init__(self, shard_candidates, base: int, n_total: int, dtype=None, group=None):
        from .search import SearchIndex

        # exact kernels for float64 shards: the float32 filter's rounding slack is
        # per shard, which a cross-shard d_best exchange would not cover
        self.index = SearchIndex(shard_candidates, dtype=dtype, base=base, f32_filter=False)
        self.n_total = int(n_total)
        self.group = group

    def search(self, queries, params, advanced=None, dim_range=None, batch=None, exchange=True, timing=False):
        import torch

        from . import _lib

        hook = (lambda d: exchange_dbest(d, self.group)) if exchange else None
        if batch is None:  # identical batching on every rank (one exchange per batch)
            batch = self.index.auto_batch(params, advanced, len(queries))
            bt = torch.tensor([batch], dtype=torch.int64, device=self.index.candidates.device)
            import torch.distributed as dist

            dist.all_reduce(bt, op=dist.ReduceOp.MIN, group=self.group)
            batch = int(bt.item())
        res = self.index.search(queries, params, advanced=advanced, dim_range=dim_range, batch=batch,
                                timing=timing, dbest_hook=hook, return_device=True)
        idx, dist_ = combine_results(res.best_index, res.best_distance, self.group)
        ctr = torch.stack([res.counters[k] for k in _lib.COUNTERS], dim=1).contiguous()
        sum_counters(ctr, self.group)
        return idx, dist_, ctr, res

"""Candidate sharding across the GPUs of one node.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  Each
rank owns a contiguous block of the collection; queries are replicated.
Per query batch there are two data-path collectives, each a real exchange:

  1. between the two search phases, an all-reduce(MIN) of the per-query
     best-so-far (every shard then prunes against the global best);
     tcdtw_search_finish never waits on the host, so this exchange for
     batch k overlaps nothing of batch k's GPU work it depends on, and
     the next batch's seed phase can be enqueued behind it;
  2. after the finish phase, ONE all-gather of a 16-byte record per query,
     (float64 distance bits, global index), reduced on every rank by the
     library's tcdtw_shard_combine kernel to the lexicographic
     (distance, index) minimum -- the reference's lowest-index tie rule
     (search.py:173) across shards.

Counters are statistics, summed only when asked for (``sum_counters``).
The collective layer also runs on gloo with CPU tensors
(tests/test_distributed_cpu.py); the combine kernel needs the GPU.
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


def gather_records(best_index, best_distance, group=None):
    """The one combine collective: every rank's (distance bits, index) per
    query, all-gathered into (world, Q, 2) int64 (same device as the
    inputs)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rec = torch.stack([best_distance.contiguous().view(torch.int64), best_index.to(torch.int64)], dim=1)
    out = torch.empty((world * rec.shape[0], 2), dtype=torch.int64, device=rec.device)
    dist.all_gather_into_tensor(out, rec.contiguous(), group=group)
    return out.view(world, rec.shape[0], 2)


def combine_gathered(records):
    """(world, Q, 2) gathered records -> (best_index, best_distance) device
    tensors: tcdtw_shard_combine, the lexicographic minimum over ranks."""
    import torch

    from . import _lib

    L = _lib.lib()
    world, Q, _ = records.shape
    rec = records.contiguous()
    idx = torch.empty(Q, dtype=torch.int64, device=rec.device)
    dist_ = torch.empty(Q, dtype=torch.float64, device=rec.device)
    _lib.check(L.tcdtw_shard_combine(rec.data_ptr(), world, Q, idx.data_ptr(), dist_.data_ptr(), _lib.stream_ptr()),
               "shard_combine")
    return idx, dist_


def combine_results(best_index, best_distance, group=None):
    """Lexicographic (distance, index) minimum across ranks: one all-gather
    plus the combine kernel.  best_index: int64 global indices (-1 = none on
    this shard); best_distance: float64."""
    return combine_gathered(gather_records(best_index, best_distance, group))


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

    def search(self, queries, params, advanced=None, dim_range=None, batch=None, exchange=True, timing=False,
               counters=True):
        """(best_index, best_distance, counters or None, local BatchOutcome);
        counters are summed over ranks (one more collective) only when asked."""
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
        ctr = None
        if counters:
            ctr = torch.stack([res.counters[k] for k in _lib.COUNTERS], dim=1).contiguous()
            sum_counters(ctr, self.group)
        return idx, dist_, ctr, res

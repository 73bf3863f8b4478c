"""Sharded search across processes (distributed.ShardedSearch) on one GPU.

Two ranks share cuda:0 with the gloo backend (its collectives stage through
the host, so no rank's kernel ever waits on another rank's kernel on the same
device; the NCCL path on an 8-GPU box runs the same code).  The combined
answer must equal the single-index answer and the oracle."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    try:
        import torch
        import torch.distributed as dist

        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2101_07731_b200 as P
        from paper_2101_07731_b200.datasets import make_workload
        from paper_2101_07731_b200.distributed import ShardedSearch, shard_bounds

        wl = make_workload("C1", n_candidates=4000, n_queries=48)
        a, b = shard_bounds(len(wl.candidates), world, rank)
        ss = ShardedSearch(wl.candidates[a:b], base=a, n_total=len(wl.candidates), dtype="f32")
        idx, dist_, ctr, _ = ss.search(wl.queries, P.SearchParams(window=12, method="lb_mv"))
        q.put((rank, idx.cpu().numpy(), dist_.cpu().numpy(), ctr.cpu().numpy()))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        import traceback

        q.put((rank, repr(e) + traceback.format_exc(), None, None))


def test_sharded_search_two_ranks_gloo():
    from oracle import oracle as O
    from paper_2101_07731_b200.datasets import make_workload

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, idx, d, c = q.get(timeout=600)
        res[r] = (idx, d, c)
    for p in procs:
        p.join(timeout=60)
    for r, (idx, d, c) in res.items():
        assert d is not None, idx
    idx0, d0, c0 = res[0]
    assert np.array_equal(idx0, res[1][0]) and np.array_equal(d0, res[1][1])
    wl = make_workload("C1", n_candidates=4000, n_queries=48)
    outs, _ = O.nn_search_batch(wl.queries.astype(np.float64), wl.candidates.astype(np.float64),
                                O.make_params(12, "lb_mv"), None, None)
    assert [o.best_index for o in outs] == idx0.tolist()
    assert [o.best_distance for o in outs] == d0.tolist()
    # counters summed over shards: computed + skipped = N
    assert np.all(c0[:, 0] + c0[:, 1] == len(wl.candidates))


def test_shard_combine_kernel(rng):
    """tcdtw_shard_combine on gathered records: lexicographic (distance,
    index) minimum, index -1 never wins, ties across ranks -> lowest index."""
    import torch

    from paper_2101_07731_b200.distributed import combine_gathered

    world, n_q = 5, 257
    dists = np.round(rng.uniform(0, 4, (world, n_q)), 1)
    dists[:, ::7] = 1.5
    idx = rng.integers(0, 10_000, (world, n_q))
    idx[1, ::5] = -1
    dists[1, ::5] = np.inf
    idx[:, 3] = -1  # no rank has a result
    dists[:, 3] = np.inf
    rec = np.stack([dists.view(np.int64), idx], axis=2)
    gi, gd = combine_gathered(torch.from_numpy(rec).cuda())
    gi, gd = gi.cpu().numpy(), gd.cpu().numpy()
    for k in range(n_q):
        cands = [(dists[r, k], idx[r, k]) for r in range(world) if idx[r, k] >= 0]
        want = min(cands) if cands else (np.inf, -1)
        assert gd[k] == want[0] and gi[k] == want[1], k

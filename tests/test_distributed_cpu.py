"""World-size-2 gloo tests of the sharded-search collectives (CPU tensors).

The NCCL path on the GPUs runs the same functions; here each rank holds a
fake per-shard result: the one all-gather of (distance bits, index) records
(its layout, world x Q x 2), the d_best exchange and the counter sum are
checked against a host merge.  The reduction of the gathered records is
the library's CUDA kernel (tcdtw_shard_combine), checked on the GPU
(tests/test_gpu_sharded.py)."""

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


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2101_07731_b200.distributed import exchange_dbest, gather_records, shard_bounds, sum_counters

        rng = np.random.default_rng(7)
        n_q = 64
        # per-rank shard results: distances with deliberate cross-rank ties
        dists = np.round(rng.uniform(0, 4, (world, n_q)), 1)
        dists[:, ::7] = 1.5  # every rank ties on these queries
        idx = np.stack([rng.integers(shard_bounds(1000, world, r)[0], shard_bounds(1000, world, r)[1], n_q)
                        for r in range(world)])
        idx[1, ::5] = -1  # rank 1 has no local result here
        dists[1, ::5] = np.inf
        my_idx = torch.tensor(idx[rank], dtype=torch.int64)
        my_d = torch.tensor(dists[rank], dtype=torch.float64)
        rec = gather_records(my_idx, my_d)  # the one combine collective
        ok = tuple(rec.shape) == (world, n_q, 2)
        ok &= bool(np.array_equal(rec[:, :, 1].numpy(), idx))
        ok &= bool(np.array_equal(rec[:, :, 0].numpy().view(np.float64), dists))
        db = torch.tensor(dists[rank], dtype=torch.float32)
        exchange_dbest(db)
        ok &= bool(np.array_equal(db.numpy(), dists.min(axis=0).astype(np.float32)))
        c = torch.full((n_q, 8), rank + 1, dtype=torch.int64)
        sum_counters(c)
        ok &= bool((c == sum(range(1, world + 1))).all())
        q.put((rank, ok))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


def test_shard_bounds_partition():
    from paper_2101_07731_b200.distributed import shard_bounds

    for n in (1, 7, 1000, 1_000_000):
        for world in (1, 2, 3, 4, 8):
            b = [shard_bounds(n, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[r][1] == b[r + 1][0] for r in range(world - 1))
            sizes = [e - s for s, e in b]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("world", [2, 3])
def test_combine_and_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(v is True for v in results.values()), results

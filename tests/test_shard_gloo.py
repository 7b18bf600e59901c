"""The N>1 path on CPU: two gloo ranks run the benchmark's multi-rank host
logic (paper_2512_18318_b200/shard.py) -- static s mod G stream ownership,
max-over-ranks step time, per-segment latency gathering -- exactly as
bench.py does under torchrun with NCCL (SURVEY.md §8 e: no data-path
collective)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_18318_b200.shard import gather_arrays, max_over_ranks, streams_for_rank, sum_over_ranks


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = streams_for_rank(64, rank, world)
        owners = [None] * world
        dist.all_gather_object(owners, mine)
        step_ms = 10.0 + 5.0 * rank  # rank 1 is the slow one
        slowest = max_over_ranks(step_ms, dist)
        frames = sum_over_ranks(100 + rank, dist)  # ranks render different frame counts
        rng = np.random.default_rng(100 + rank)
        lat = rng.uniform(100, 900, 50 + 10 * rank)
        dec = lat - 5.0
        all_lat, all_dec = gather_arrays([lat, dec], dist, world)
        q.put((rank, owners, slowest, all_lat.tolist(), all_dec.tolist(), frames))
    finally:
        dist.destroy_process_group()


def test_streams_for_rank_single():
    assert streams_for_rank(4, 0, 1) == [0, 1, 2, 3]
    assert streams_for_rank(6, 1, 2) == [1, 3, 5]
    assert streams_for_rank(7, 0, 2) == [0, 2, 4, 6]
    # 256 streams over 1/2/4/8 GPUs: every stream owned exactly once
    for g in (1, 2, 4, 8):
        owned = sorted(s for r in range(g) for s in streams_for_rank(256, r, g))
        assert owned == list(range(256))
    with pytest.raises(ValueError):
        streams_for_rank(3, 2, 2)


def test_two_rank_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    owners = res[0][1]
    # 64 streams in total: every stream owned by exactly one rank, s mod G, 32 per rank
    flat = sorted(s for o in owners for s in o)
    assert flat == list(range(64))
    assert all(s % world == r for r, o in enumerate(owners) for s in o)
    assert all(len(o) == 32 for o in owners)
    # the job time is the slowest rank's, on every rank
    assert all(r[2] == 15.0 for r in res)
    # whole-job work is the sum over ranks
    assert all(r[5] == 201.0 for r in res)
    # gathered latencies = concatenation in rank order, identical on all ranks
    want = np.concatenate([np.random.default_rng(100 + r).uniform(100, 900, 50 + 10 * r) for r in range(world)])
    for r in res:
        np.testing.assert_array_equal(np.array(r[3]), want)
        np.testing.assert_array_equal(np.array(r[4]), want - 5.0)
    assert np.percentile(want, 50) == np.percentile(np.array(res[1][3]), 50)

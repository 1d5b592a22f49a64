"""N>1 host logic on CPU: world_size-2 gloo ranks shard independent streams,
score their shard, gather, and must reproduce the single-process result
bit for bit (streams share no state).  The per-stream
scorer here is the fp64 oracle (tests may run it; the GPU ranks run the
engine through the same sharding code in bench.py)."""
import os
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def make_lines(n_streams=5, lines=12, p=16, b=6):
    rng = np.random.default_rng(7)
    return (rng.uniform(size=(n_streams, lines, p, b)) + np.arange(n_streams)[:, None, None, None]).astype(np.float32)


def score(oracle, lines, sid):
    raw, _, _ = oracle.run_stream(oracle.OracleConfig(no_srp=True), lines[sid])
    return raw


def _worker(rank, world, port, lines, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch.distributed as dist

    import oracle_ctypes as oracle
    from paper_2408_14947_b200.sharding import max_over_ranks, run_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    got = run_sharded(lines.shape[0], lambda s: score(oracle, lines, s), dist)
    t = max_over_ranks(1.0 + rank, dist)
    if rank == 0:
        q.put((got, t))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_streams_partition():
    from paper_2408_14947_b200.sharding import shard_streams

    for n in (1, 4, 5, 64):
        for world in (1, 2, 3, 8):
            ids = [i for r in range(world) for i in shard_streams(n, world, r)]
            assert ids == list(range(n))
    assert list(shard_streams(64, 8, 3)) == list(range(24, 32))


def test_two_gloo_ranks_match_single_process(oracle):
    lines = make_lines()
    single = [score(oracle, lines, s) for s in range(lines.shape[0])]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, lines, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 2.0
    assert len(got) == len(single)
    for a, b in zip(got, single):
        assert np.array_equal(a, b)

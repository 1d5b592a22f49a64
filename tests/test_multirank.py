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


# ---------------------------------------------------------------- one stream split into line ranges
def _line_stats(x):
    return x.mean(0), np.cov(x, rowvar=False)


def _priors(lines, alpha, incremental, start=None):
    """Sequential background (mu, cov) seen by each line (score-then-update), optionally starting
    from a carried state {mu, cov[, n]} instead of line-0 initialisation."""
    from paper_2408_14947_b200.sharding import merge_welford

    out, st = [], start
    P = lines.shape[1]
    for x in lines:
        m, k = _line_stats(x.astype(np.float64))
        if st is None:
            st = {"mu": m, "cov": k, "n": P}
        out.append((st["mu"].copy(), st["cov"].copy()))
        if incremental:
            st = merge_welford(st, {"n": P, "mu": m, "cov": k})
        else:
            st = {"mu": (1 - alpha) * st["mu"] + alpha * m, "cov": (1 - alpha) * st["cov"] + alpha * k}
    return out, st


def _summary(lines, alpha, incremental, from_zero):
    d = lines.shape[2]
    start = None
    if from_zero:
        start = {"mu": np.zeros(d), "cov": np.zeros((d, d)), "n": 0}
    _, st = _priors(lines, alpha, incremental, start)
    return {"lines": len(lines), "n": int(st.get("n", 0)), "mu": st["mu"], "cov": st["cov"]}


def _split_worker(rank, world, port, lines, alpha, incremental, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2408_14947_b200.sharding import run_split_stream

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    got = run_split_stream(
        rank, world, lines.shape[0], alpha, incremental,
        summarize=lambda rows, zero: _summary(lines[rows.start:rows.stop], alpha, incremental, zero),
        score=lambda rows, carry: np.stack([m for m, _ in _priors(lines[rows.start:rows.stop], alpha, incremental,
                                                                  carry)[0]]),
        dist=dist)
    q.put((rank, got))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("incremental", [False, True])
def test_line_range_split_two_gloo_ranks(incremental):
    """configs[4]-style split of ONE stream over 2 ranks: one all-gather of range summaries, the
    chained carry, then independent ranges reproduce the sequential backgrounds (fp64, rounding only)."""
    rng = np.random.default_rng(3)
    lines = (rng.normal(size=(23, 40, 5)) + np.linspace(0, 3, 23)[:, None, None]).astype(np.float32)
    alpha = 0.1
    ref = np.stack([m for m, _ in _priors(lines, alpha, incremental)[0]])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + (os.getpid() % 1000) + (7 if incremental else 0)
    procs = [ctx.Process(target=_split_worker, args=(r, 2, port, lines, alpha, incremental, q)) for r in range(2)]
    for p in procs:
        p.start()
    parts = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = np.concatenate([parts[0], parts[1]])
    np.testing.assert_allclose(got, ref, rtol=1e-10, atol=1e-12)


def test_carry_chain_three_ranges():
    from paper_2408_14947_b200.sharding import carry_chain, line_ranges

    rng = np.random.default_rng(5)
    lines = rng.normal(size=(31, 30, 4)) + 1.0
    for incremental in (False, True):
        ranges = line_ranges(31, 3)
        sums = [_summary(lines[r.start:r.stop], 0.2, incremental, i > 0) for i, r in enumerate(ranges)]
        carries = carry_chain(sums, 0.2, incremental)
        ref, _ = _priors(lines, 0.2, incremental)
        for i, r in enumerate(ranges[1:], start=1):
            np.testing.assert_allclose(carries[i]["mu"], ref[r.start][0], rtol=1e-10)
            np.testing.assert_allclose(carries[i]["cov"], ref[r.start][1], rtol=1e-9, atol=1e-12)

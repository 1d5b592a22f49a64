"""Multi-GPU plumbing.

Streams share no state, so N ranks split them into
contiguous shards and run with no data-path collective.  The only
cross-rank traffic is the final gather of per-stream results and the
max-over-ranks reduction of device times.

One long stream (configs[4] on more GPUs than streams) splits into line
ranges with ONE exchange step.  The background recurrence is linear: over a
range of n lines started from a zero background the EMA ends at
Z = sum_t alpha (1 - alpha)^(end - t) stat_t, so the state at the end of
range r is  S_r = (1 - alpha)^(n_r) S_(r-1) + Z_r  (rank 0's range starts at
line 0 and is summarised from scratch: S_0 = Z_0); Welford mode merges
(count, mean, covariance) summaries with the batched formula of
linalg.hpp:33-36.  Each rank summarises its range (statistics + scan only,
Engine.advance_device), the summaries are all-gathered, every rank folds the
chain up to its own range start, sets that carry as its background
(Engine.set_state) and scores its range.  Backend-agnostic: `nccl` on B200s
and `gloo` on CPU (tests/test_multirank.py).
"""
from __future__ import annotations

from typing import Callable, Dict, List, Sequence

import numpy as np


def shard_streams(n_streams: int, world: int, rank: int) -> range:
    """Contiguous shard of stream ids owned by `rank` (even split; the first
    n_streams % world ranks take one extra stream)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, extra = divmod(n_streams, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank time (the contract's max-over-ranks device clock)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_stream_results(local: Dict[int, np.ndarray], n_streams: int, dist=None) -> List[np.ndarray]:
    """All-gather {stream id -> scores} from every rank into a list indexed by
    stream id (the final gather; the only data that crosses ranks)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        parts = [local]
    else:
        parts = [None] * dist.get_world_size()
        dist.all_gather_object(parts, local)
    out: List[np.ndarray] = [None] * n_streams  # type: ignore[list-item]
    for part in parts:
        for sid, arr in part.items():
            if out[sid] is not None:
                raise RuntimeError(f"stream {sid} scored by two ranks")
            out[sid] = arr
    missing = [i for i, a in enumerate(out) if a is None]
    if missing:
        raise RuntimeError(f"streams never scored: {missing}")
    return out


def run_sharded(n_streams: int, score_stream: Callable[[int], np.ndarray], dist=None) -> List[np.ndarray]:
    """Score this rank's shard with `score_stream(stream_id)` and gather all."""
    rank = dist.get_rank() if dist is not None and dist.is_initialized() else 0
    world = dist.get_world_size() if dist is not None and dist.is_initialized() else 1
    local = {s: score_stream(s) for s in shard_streams(n_streams, world, rank)}
    return gather_stream_results(local, n_streams, dist)


# ---------------------------------------------------------------- one stream split into line ranges
def line_ranges(n_lines: int, world: int) -> List[range]:
    """Contiguous line ranges of one stream, one per rank."""
    return [shard_streams(n_lines, world, r) for r in range(world)]


def merge_welford(a: Dict, b: Dict) -> Dict:
    """Batched Welford merge of (n, mu, cov) summaries (linalg.hpp:33-36; unbiased covariance)."""
    na, nb = float(a["n"]), float(b["n"])
    if na == 0:
        return dict(b)
    if nb == 0:
        return dict(a)
    n = na + nb
    d = np.asarray(b["mu"]) - np.asarray(a["mu"])
    m2 = (np.asarray(a["cov"]) * (na - 1.0) if na >= 2 else 0.0) + np.asarray(b["cov"]) * (nb - 1.0) \
        + np.outer(d, d) * (na * nb / n)
    return {"n": int(n), "mu": np.asarray(a["mu"]) + d * (nb / n), "cov": m2 / (n - 1.0) if n >= 2 else m2 * 0.0}


def carry_chain(summaries: Sequence[Dict], alpha: float, incremental: bool) -> List[Dict]:
    """Background state at the START of each range from the per-range summaries.

    EMA: summaries[r] = {"lines": n_r, "mu", "cov"} of range r run from a zero background (range 0
    from scratch, so it is already the true end state).  Welford: {"n", "mu", "cov"} of the range.
    Returns carry[r] (None for r = 0) to install with Engine.set_state before scoring range r."""
    carries: List[Dict] = [None]  # type: ignore[list-item]
    if incremental:
        acc = dict(summaries[0])
        for r in range(1, len(summaries)):
            carries.append(dict(acc))
            acc = merge_welford(acc, summaries[r])
        return carries
    mu = np.asarray(summaries[0]["mu"], np.float64)
    cov = np.asarray(summaries[0]["cov"], np.float64)
    for r in range(1, len(summaries)):
        carries.append({"mu": mu.copy(), "cov": cov.copy()})
        f = (1.0 - alpha) ** int(summaries[r]["lines"])
        mu = f * mu + np.asarray(summaries[r]["mu"])
        cov = f * cov + np.asarray(summaries[r]["cov"])
    return carries


def run_split_stream(rank: int, world: int, n_lines: int, alpha: float, incremental: bool,
                     summarize: Callable[[range, bool], Dict], score: Callable[[range, Dict], np.ndarray],
                     dist=None) -> np.ndarray:
    """One stream's lines [0, n_lines) over `world` ranks with one exchange step.

    summarize(lines, from_zero) -> this range's summary (Engine.advance_device from a zero
    background when from_zero, from scratch for range 0); score(lines, carry) -> scores of the
    range with the carried background installed (None for range 0).  Returns this rank's scores."""
    ranges = line_ranges(n_lines, world)
    mine = summarize(ranges[rank], rank > 0)
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        summaries = [None] * world
        dist.all_gather_object(summaries, mine)
    else:
        summaries = [mine]
    carries = carry_chain(summaries, alpha, incremental)
    return score(ranges[rank], carries[rank])

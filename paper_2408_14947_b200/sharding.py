"""Multi-GPU plumbing for independent scan streams.

Streams share no state, so N ranks split them into
contiguous shards and run with no data-path collective.  The only
cross-rank traffic is the final gather of per-stream results and the
max-over-ranks reduction of device times.  Backend-agnostic: works with
`nccl` on B200s and `gloo` on CPU (tests/test_multirank.py).
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

"""Data-parallel replicas: requests shard by batch item with no
collective on the data path. One process per GPU holds a full weight replica
and its own arena; the only cross-rank traffic is the timing/token reduction
used by the benchmark (max-over-ranks time, summed tokens) and, optionally,
gathering hypotheses on rank 0."""

from __future__ import annotations

import torch


def batch_shard(n_items: int, rank: int, world: int) -> slice:
    """Contiguous, balanced slice of the global batch owned by ``rank``
    (sizes differ by at most one item)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return slice(lo, lo + base + (1 if rank < extra else 0))


def _dist():
    return torch.distributed.is_available() and torch.distributed.is_initialized()


def reduce_step_stats(seconds: float, tokens: float, device=None) -> tuple[float, float]:
    """(max seconds over ranks, total tokens over ranks); identity when single-process."""
    dev = device if device is not None else torch.device("cpu")
    if _dist() and torch.distributed.get_backend() == "gloo":
        dev = torch.device("cpu")
    t = torch.tensor([seconds], dtype=torch.float64, device=dev)
    n = torch.tensor([tokens], dtype=torch.float64, device=dev)
    if _dist():
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(n, op=torch.distributed.ReduceOp.SUM)
    return float(t.item()), float(n.item())


def gather_hypotheses(local: list, world: int) -> list | None:
    """Concatenate every rank's per-item hypothesis lists on rank 0 (host
    objects, a few KB per request — SURVEY §5 'host gather is simpler')."""
    if not _dist() or world == 1:
        return local
    out = [None] * world
    torch.distributed.all_gather_object(out, local)
    return [h for part in out for h in part]

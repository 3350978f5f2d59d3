"""Batch sharding across GPUs (one process per GPU, torch.distributed).

Every transform in a batch is independent (reference SPEC.md:317), so the
multi-GPU path partitions the batch into contiguous per-rank shards and runs
each shard on its own device with its own plan and stream: no collective
touches the data path.  Collectives appear only around it: a barrier before
timing, a MAX all-reduce of the per-rank device time, and (optionally) an
all-gather of shards when a caller wants the whole spectrum on every rank.
"""

from __future__ import annotations

from dataclasses import dataclass


def shard_range(batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [start, stop) of the batch owned by `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    base, rem = divmod(batch, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


@dataclass
class Shard:
    rank: int
    world: int
    start: int
    stop: int

    @property
    def batch(self) -> int:
        return self.stop - self.start


def my_shard(batch: int) -> Shard:
    """This process's shard (torch.distributed if initialised, else everything)."""
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            r, w = dist.get_rank(), dist.get_world_size()
        else:
            r, w = 0, 1
    except Exception:
        r, w = 0, 1
    s, e = shard_range(batch, r, w)
    return Shard(r, w, s, e)


def max_over_ranks(value: float, device=None) -> float:
    """MAX all-reduce of a per-rank scalar (device time of the timed region)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_shards(local, batch: int):
    """All-gather per-rank shards (torch tensors, leading dim = shard batch)
    into the full batch on every rank.  Off the hot path."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return local
    w = dist.get_world_size()
    sizes = [shard_range(batch, r, w) for r in range(w)]
    maxb = max(e - s for s, e in sizes)
    pad = torch.zeros((maxb,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    outs = [torch.empty_like(pad) for _ in range(w)]
    dist.all_gather(outs, pad)
    return torch.cat([o[: e - s] for o, (s, e) in zip(outs, sizes)], dim=0)

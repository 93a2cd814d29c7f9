"""Row e: UE sharding across the GPUs of one box.

UEs are independent ("per-UE parallelism"; P:483 cluster distribution), so
rank r of N owns a contiguous UE block and both directions of each of its UEs; it
creates its own handle with channel_offset = the global id of its first channel, so
noise keys (and the harness's input draws) use global ids and outputs do not depend
on N. There is no collective on the data path: torch.distributed carries only the
pre-timing barrier and the max / sum reductions of per-rank timings and counts.
"""
from __future__ import annotations

import os
from typing import Optional, Tuple


def env() -> Tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (1 process = 1 GPU)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def ue_block(ues: int, dirs: int, rank: int, world: int) -> Tuple[int, int]:
    """Global channel range [c_lo, c_hi) of `rank`: UEs [rank*U/N, (rank+1)*U/N), each
    UE's `dirs` channels kept together (c = dirs*u + dir)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    u_lo = rank * ues // world
    u_hi = (rank + 1) * ues // world
    return u_lo * dirs, u_hi * dirs


def init(backend: str = "nccl", device=None):
    """Initialise the default process group when WORLD_SIZE > 1; returns the
    torch.distributed module (or None for a single process)."""
    rank, world, _ = env()
    if world <= 1:
        return None
    import torch.distributed as dist

    if not dist.is_initialized():
        kw = {"device_id": device} if (backend == "nccl" and device is not None) else {}
        dist.init_process_group(backend, **kw)
    return dist


def _reduce(value: float, op: str, device, pg) -> float:
    if pg is None:
        return float(value)
    import torch

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    pg.all_reduce(t, op=getattr(pg.ReduceOp, op))
    return float(t.item())


def max_over_ranks(value: float, device=None, pg=None) -> float:
    """The job's elapsed time is the slowest rank's (device-timed on each rank)."""
    return _reduce(value, "MAX", device, pg)


def sum_over_ranks(value: float, device=None, pg=None) -> float:
    """Units processed by all ranks."""
    return _reduce(value, "SUM", device, pg)


def reduce_groups(agg, pg=None):
    """NEXT f1: when a cell's UEs are sharded over ranks each rank holds the partial
    group sums of its own UEs (tt_channel_apply_aggregate); the cell's aggregate is
    their sum over ranks (the path's only data collective: one NCCL all-reduce of
    groups x n complex samples, ~0.5 MB per cell per c4 slot). In place; returns agg."""
    if pg is not None:
        pg.all_reduce(agg, op=pg.ReduceOp.SUM)
    return agg


def barrier(pg=None, device: Optional[object] = None) -> None:
    if pg is not None:
        pg.barrier()

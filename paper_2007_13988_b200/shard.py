"""Frame sharding across GPUs (one process per GPU, torch.distributed plumbing).

The reference's multi-frame pattern (BASELINE.json configs[4]: independent
frames, one per GPU) has no data exchange inside a frame: frames are dealt
round-robin to ranks, each rank runs its frames through its own
`api.Context`, and only per-frame summaries travel (to rank 0) at the end.
No collective touches the data path; `torch.distributed` is used for the
barrier, the max-over-ranks timing and the summary gather, so the same code
runs on NCCL (GPU) and gloo (CPU tests).
"""
from __future__ import annotations

from typing import Any, Callable, Dict, List, Optional


def frames_for_rank(n_frames: int, rank: int, world: int) -> List[int]:
    """Round-robin frame assignment: rank r gets frames r, r + world, ..."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("frames_for_rank: bad rank/world")
    if n_frames < 0:
        raise ValueError("frames_for_rank: negative frame count")
    return list(range(rank, n_frames, world))


def _dist():
    import torch.distributed as td

    return td if td.is_available() and td.is_initialized() else None


def allmax(x: float, device: Optional[str] = None) -> float:
    """Max over ranks (device timings are reported as the slowest rank)."""
    td = _dist()
    if td is None:
        return float(x)
    import torch

    t = torch.tensor([float(x)], dtype=torch.float64, device=device or "cpu")
    td.all_reduce(t, op=td.ReduceOp.MAX)
    return float(t.item())


def allsum(x: float, device: Optional[str] = None) -> float:
    td = _dist()
    if td is None:
        return float(x)
    import torch

    t = torch.tensor([float(x)], dtype=torch.float64, device=device or "cpu")
    td.all_reduce(t, op=td.ReduceOp.SUM)
    return float(t.item())


def barrier() -> None:
    td = _dist()
    if td is not None:
        td.barrier()


def run_sharded(n_frames: int, frame_fn: Callable[[int], Dict[str, Any]], rank: int = 0,
                world: int = 1) -> Optional[List[Dict[str, Any]]]:
    """Runs this rank's frames; returns every frame's summary on rank 0 (in frame order), None elsewhere.

    `frame_fn(i)` processes frame i and returns a small picklable summary
    (evaluation counts, covered pixels, output checksums...).
    """
    mine = {i: frame_fn(i) for i in frames_for_rank(n_frames, rank, world)}
    td = _dist()
    if td is None or world == 1:
        return [mine[i] for i in range(n_frames)]
    gathered: List[Optional[Dict[int, Dict[str, Any]]]] = [None] * world
    td.all_gather_object(gathered, mine)
    if rank != 0:
        return None
    out: Dict[int, Dict[str, Any]] = {}
    for part in gathered:
        for i, s in (part or {}).items():
            if i in out:
                raise RuntimeError(f"run_sharded: frame {i} processed twice")
            out[i] = s
    if sorted(out) != list(range(n_frames)):
        raise RuntimeError("run_sharded: missing frames")
    return [out[i] for i in range(n_frames)]

"""One process per GPU: torch.distributed plumbing for the Monte-Carlo driver.

The only data-path exchange of the path is the per-round sum of the
(frames, bit_errors, frame_errors) counter array: batches
are sharded round-robin in contiguous blocks, every rank draws its own lanes
from the counter-based channel, and no message data ever crosses GPUs.
NCCL carries the sum on GPUs; the same code runs on gloo for CPU tests.
"""

from __future__ import annotations

import os


def world():
    """(rank, world_size, group-or-None) of the current default process group."""
    try:
        import torch.distributed as dist
    except Exception:      # pragma: no cover
        return 0, 1, None
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size(), dist.group.WORLD
    return 0, 1, None


def init_from_env(backend: str | None = None):
    """Initialise the default group from torchrun's env (RANK/WORLD_SIZE/MASTER_*)."""
    import torch
    import torch.distributed as dist
    if dist.is_initialized():
        return world()
    if int(os.environ.get("WORLD_SIZE", "1")) <= 1:
        return 0, 1, None
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    if backend is None:
        backend = os.environ.get("QCB_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
    if torch.cuda.is_available():
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
    dist.init_process_group(backend=backend)
    return world()


def sum_counts(counts, group=None):
    """All-reduce(SUM) an int64 counter tensor in place (no-op on one rank)."""
    import torch.distributed as dist
    if group is None or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return counts
    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return counts


def max_scalar(x: float, group=None, device=None) -> float:
    """Max of a float over ranks (timing: the job takes as long as its slowest rank)."""
    import torch
    import torch.distributed as dist
    if group is None or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def ordered_prefix(counts, stop_errors: int, max_frames: int, start=(0, 0, 0)):
    """Apply the reference stop rule to per-batch counts in batch order.

    counts: iterable of (frames, bit_errors, frame_errors) in global batch order.
    Accumulates batches until frame_errors >= stop_errors or frames >= max_frames
    (checked after every batch, harness.py:173-192).  Returns (totals, done, used).
    """
    f, be, fe = start
    used = 0
    for row in counts:
        if fe >= stop_errors or f >= max_frames:
            return (f, be, fe), True, used
        f += int(row[0]); be += int(row[1]); fe += int(row[2])
        used += 1
    return (f, be, fe), (fe >= stop_errors or f >= max_frames), used

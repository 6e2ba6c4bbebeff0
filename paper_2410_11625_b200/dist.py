"""Frame-sharded multi-GPU plumbing for FLR.

FLR is stateless across frames (no temporal filtering), so a batch of
independent frames shards by frame with NO data-path collective: rank r of W owns
its own frames, drawn from seeds that depend only on the global frame index.
torch.distributed (NCCL on B200, gloo in the CPU tests) only carries the per-rank
step time (MAX: the slowest rank sets the job time) and the per-rank checksums
after the timed region.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def frame_seeds(rank: int, world: int, frames_per_rank: int, base: int = 1000):
    """Seeds of the frames rank `rank` owns: global frame index g -> seed base + g."""
    start = rank * frames_per_rank
    return [base + start + i for i in range(frames_per_rank)]


def shard_range(n_frames: int, rank: int, world: int):
    """Contiguous [lo, hi) share of n_frames for strong scaling (remainder to the first ranks)."""
    q, r = divmod(n_frames, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def max_over_ranks(value: float, device=None) -> float:
    """Job time = max of the per-rank times (one all_reduce MAX after the timed region)."""
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(row, device=None):
    """All ranks' small float64 vectors (checksums), in rank order."""
    t = torch.as_tensor(row, dtype=torch.float64, device=device).reshape(-1)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
        dist.all_gather(out, t)
        return [o.tolist() for o in out]
    return [t.tolist()]


def output_checksum(out) -> list:
    """[sum, max |x|, all finite] of a result tensor, in float64."""
    o = out.double()
    return [float(o.sum()), float(o.abs().max()), float(torch.isfinite(out).all())]

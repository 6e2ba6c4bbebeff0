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


def per_frame_checksums(out):
    """[n, 3] float64 rows [sum, max |x|, all finite] of each frame of an [n, ...] result."""
    o = out.double().reshape(out.shape[0], -1)
    return torch.stack([o.sum(1), o.abs().amax(1), torch.isfinite(o).all(1).double()], 1)


def gather_frame_checksums(rows, lo: int, n_total: int, device=None):
    """Assemble every rank's per-frame checksum rows ([hi - lo, 3], frames [lo, hi) of the
    global batch, as shard_range hands them out) into one [n_total, 3] float64 tensor in
    global frame order, on every rank (one all_gather of fixed-size padded blocks)."""
    rows = torch.as_tensor(rows, dtype=torch.float64, device=device).reshape(-1, 3)
    world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    if world == 1:
        return rows.cpu()
    cap = -(-n_total // world)  # largest shard
    buf = torch.full((cap + 1, 3), float("nan"), dtype=torch.float64, device=device)
    buf[0, 0], buf[0, 1] = float(lo), float(rows.shape[0])
    buf[1:1 + rows.shape[0]] = rows
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    full = torch.full((n_total, 3), float("nan"), dtype=torch.float64)
    for p in parts:
        p = p.cpu()
        a, m = int(p[0, 0]), int(p[0, 1])
        full[a:a + m] = p[1:1 + m]
    return full


def output_checksum(out) -> list:
    """[sum, max |x|, all finite] of a result tensor, in float64."""
    o = out.double()
    return [float(o.sum()), float(o.abs().max()), float(torch.isfinite(out).all())]

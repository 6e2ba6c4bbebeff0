"""Strip sharding of ONE frame across ranks (north_star:
"Spatial strips with halos are used only for single frames larger than one GPU's share").

A frame's block rows are split into contiguous strips, one per rank.  FLR's result at a
pixel depends on a bounded neighbourhood of block rows, so a strip extended by a halo of
`halo_blocks(R)` block rows above and below reproduces the full-frame result on its own
rows exactly (same arithmetic, same order; bitwise for the oracle):

* apply: a pixel of block row b blends the models of the block
  centres around it, i.e. of block rows b-1 .. b+1 (R4: centres at (b+1/2)D - 1/2);
* fit: the model of block row b solves from the Gaussian-blurred moment
  field, and the blur reaches R block rows (R1), i.e. moments of rows b-R .. b+R.

So output rows [b_lo, b_hi) need moments of block rows [b_lo-1-R, b_hi+1+R): a halo of
R + 1 block rows, clipped at the frame edges (where the frame's own boundary rules, R3-R5,
apply exactly as in the full frame).  Strips start on block boundaries, so the block grid
of every strip is a sub-grid of the frame's.

The exchange is the only data-path communication: each rank sends the first and last
halo rows of its own share to its neighbours (point-to-point; NCCL on B200, gloo in the
CPU tests), denoises the extended strip with the same C-ABI call as a whole frame, crops
its own rows and, if asked, all-gathers the frame.  This module is host plumbing only:
no step of the method's arithmetic runs here.
"""
from __future__ import annotations

import math

import torch
import torch.distributed as dist


def halo_blocks(R: int) -> int:
    """Block rows of halo each side: 1 for the apply's blend + R for the moment blur."""
    if R < 0:
        raise ValueError("R must be >= 0")
    return R + 1


def strip_plan(H: int, D: int, R: int, world: int):
    """Per rank: (out_lo, out_hi, in_lo, in_hi) in pixel rows.

    [out_lo, out_hi) are the rows the rank owns (a contiguous run of block rows, the
    remainder to the first ranks); [in_lo, in_hi) adds the halo, clipped to the frame.
    Every strip must own at least halo_blocks(R) block rows so that a halo comes from
    the immediate neighbour only."""
    if H <= 0 or D <= 0 or world <= 0:
        raise ValueError("H, D and world must be positive")
    By = math.ceil(H / D)
    h = halo_blocks(R)
    if world > 1 and By // world < h:
        raise ValueError(f"{By} block rows over {world} ranks leaves strips thinner than the "
                         f"{h}-block halo; use fewer ranks or frame sharding")
    q, r = divmod(By, world)
    plan = []
    for k in range(world):
        b_lo = k * q + min(k, r)
        b_hi = b_lo + q + (1 if k < r else 0)
        plan.append((b_lo * D, min(b_hi * D, H), max(0, (b_lo - h) * D), min(H, (b_hi + h) * D)))
    return plan


def extend_with_halo(own, plan, rank, group=None):
    """Exchange halo rows with the neighbouring ranks.

    own: list of tensors [..., rows, W] holding this rank's rows [out_lo, out_hi) of each
    input plane stack (guides, radiance).  Returns the same tensors extended to
    [in_lo, in_hi) with the neighbours' rows (point-to-point sends of the edge rows)."""
    out_lo, out_hi, in_lo, in_hi = plan[rank]
    n_top, n_bot = out_lo - in_lo, in_hi - out_hi
    world = len(plan)
    ops, recv_top, recv_bot = [], [], []
    for t in own:
        if t.shape[-2] != out_hi - out_lo:
            raise ValueError(f"rank {rank} owns {out_hi - out_lo} rows, got {t.shape[-2]}")
        lead = t.shape[:-2]
        W = t.shape[-1]
        if rank > 0:  # rows above come from rank-1's bottom; it wants our top rows
            up_need = plan[rank - 1][3] - plan[rank - 1][1]
            rt = torch.empty(*lead, n_top, W, dtype=t.dtype, device=t.device)
            recv_top.append(rt)
            ops.append(dist.P2POp(dist.isend, t[..., :up_need, :].contiguous(), rank - 1, group))
            ops.append(dist.P2POp(dist.irecv, rt, rank - 1, group))
        if rank < world - 1:
            dn_need = plan[rank + 1][0] - plan[rank + 1][2]
            rb = torch.empty(*lead, n_bot, W, dtype=t.dtype, device=t.device)
            recv_bot.append(rb)
            ops.append(dist.P2POp(dist.isend, t[..., t.shape[-2] - dn_need:, :].contiguous(),
                                  rank + 1, group))
            ops.append(dist.P2POp(dist.irecv, rb, rank + 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    ext = []
    for i, t in enumerate(own):
        parts = ([recv_top[i]] if rank > 0 else []) + [t] + ([recv_bot[i]] if rank < world - 1 else [])
        ext.append(torch.cat(parts, dim=-2).contiguous())
    return ext


def crop_own(out_ext, plan, rank):
    """This rank's own rows of the extended strip's result."""
    out_lo, out_hi, in_lo, _ = plan[rank]
    return out_ext[..., out_lo - in_lo:out_hi - in_lo, :]


def gather_frame(own_out, plan, group=None):
    """All-gather every rank's own rows into the full frame [..., H, W] (rows padded to
    the tallest strip for the collective, then trimmed)."""
    world = len(plan)
    if world == 1:
        return own_out
    rows = max(p[1] - p[0] for p in plan)
    lead, W = own_out.shape[:-2], own_out.shape[-1]
    pad = torch.zeros(*lead, rows, W, dtype=own_out.dtype, device=own_out.device)
    pad[..., :own_out.shape[-2], :] = own_out
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad.contiguous(), group=group)
    return torch.cat([b[..., :p[1] - p[0], :] for b, p in zip(bufs, plan)], dim=-2)


def denoise_strip(denoise_fn, guides_own, radiance_own, plan, rank, group=None, gather=False):
    """One frame sharded in strips: halo exchange, denoise of the extended strip with
    `denoise_fn(guides, radiance) -> out` (the C-ABI call on B200), crop, optional gather.

    guides_own [n,Q,rows,W], radiance_own [n,3,rows,W]: this rank's rows of the frame."""
    g_ext, y_ext = extend_with_halo([guides_own, radiance_own], plan, rank, group)
    own = crop_own(denoise_fn(g_ext, y_ext), plan, rank)
    return gather_frame(own.contiguous(), plan, group) if gather else own


def denoise_strips_local(denoise_fn, guides, radiance, D: int, R: int, parts: int):
    """Single-process form (no collective): the frame [n,Q,H,W] cut into `parts` strips
    with halos, each denoised on its own, own rows stitched back.  Used to check the halo
    rule on one GPU without ranks that wait on one another."""
    H = guides.shape[-2]
    plan = strip_plan(H, D, R, parts)
    outs = []
    for (out_lo, out_hi, in_lo, in_hi) in plan:
        o = denoise_fn(guides[..., in_lo:in_hi, :].contiguous(), radiance[..., in_lo:in_hi, :].contiguous())
        outs.append(o[..., out_lo - in_lo:out_hi - in_lo, :])
    return torch.cat(outs, dim=-2)

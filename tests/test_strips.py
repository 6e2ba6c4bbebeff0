"""Strip sharding of one frame, CPU side (-m "not gpu").

The halo rule (paper_2410_11625_b200/strips.py: R + 1 block rows, from the apply's blend
over neighbouring block centres P:274-278 / R4 and the moment blur's reach R P:315-316 /
R1) is pinned with the fp64 oracle: strips denoised on their own and stitched must equal
the full-frame result BITWISE (same arithmetic in the same order; the zero padding at a
strip edge only reaches halo rows), and a halo one block row short must not.  A
world_size-2 gloo run checks the point-to-point halo exchange and the gather.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_11625_b200 import strips

D, SIGMA, R = 8, 10.0, 3


def _oracle_fn(oracle, R_=R):
    return lambda g, y: torch.from_numpy(
        oracle.denoise(g.numpy(), y.numpy(), D=D, sigma=SIGMA, R=R_))


def _frame(W, H, Q=4, seed=4242):
    from paper_2410_11625_b200 import synth

    G, Y = synth.frame(W, H, Q=Q, seed=seed)
    return G.unsqueeze(0), Y.unsqueeze(0)


@pytest.mark.parametrize("H,world", [(1, 1), (64, 2), (104, 3), (101, 3), (1080, 8)])
def test_plan_covers_rows_on_block_boundaries(H, world):
    plan = strips.strip_plan(H, D, R, world)
    h = strips.halo_blocks(R) * D
    assert plan[0][0] == 0 and plan[-1][1] == H
    for a, b in zip(plan, plan[1:]):
        assert a[1] == b[0]
    for (lo, hi, ilo, ihi) in plan:
        assert lo % D == 0 and ilo % D == 0
        assert ilo == max(0, lo - h) and ihi == min(H, hi + h)


def test_plan_rejects_strips_thinner_than_halo():
    with pytest.raises(ValueError):
        strips.strip_plan(64, D, R, 3)  # 8 block rows / 3 ranks < 4-block halo


@pytest.mark.parametrize("W,H,parts", [(48, 64, 2), (40, 104, 3), (37, 101, 3)])
def test_oracle_strips_equal_full_frame_bitwise(oracle_mod, W, H, parts):
    G, Y = _frame(W, H)
    fn = _oracle_fn(oracle_mod)
    full = fn(G, Y)
    got = strips.denoise_strips_local(fn, G, Y, D, R, parts)
    assert got.shape == full.shape
    assert torch.equal(got, full)


def test_short_halo_differs(oracle_mod, monkeypatch):
    """A halo of R block rows (one short: the apply's neighbour row forgotten) changes the
    rows next to a strip boundary -- the rule is tight."""
    G, Y = _frame(40, 104)
    fn = _oracle_fn(oracle_mod)
    full = fn(G, Y)
    monkeypatch.setattr(strips, "halo_blocks", lambda r: r)
    got = strips.denoise_strips_local(fn, G, Y, D, R, 3)
    assert not torch.equal(got, full)


def test_single_rank_needs_no_process_group(oracle_mod):
    """world = 1: no halo, no exchange, no collective -- the whole-frame call."""
    G, Y = _frame(40, 48)
    plan = strips.strip_plan(48, D, R, 1)
    assert plan == [(0, 48, 0, 48)]
    fn = _oracle_fn(oracle_mod)
    got = strips.denoise_strip(fn, G, Y, plan, 0, gather=True)
    assert torch.equal(got, fn(G, Y))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, W, H, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle

        G, Y = _frame(W, H)
        plan = strips.strip_plan(H, D, R, world)
        lo, hi = plan[rank][0], plan[rank][1]
        # each rank holds only its own rows; the halo arrives from the neighbours
        out = strips.denoise_strip(_oracle_fn(oracle), G[..., lo:hi, :].contiguous(),
                                   Y[..., lo:hi, :].contiguous(), plan, rank, gather=True)
        if rank == 0:
            q.put(out.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,W,H", [(2, 40, 72), (3, 24, 101)])
def test_gloo_strips_match_full_frame(oracle_mod, world, W, H):
    """world 2, and world 3 (the middle rank exchanges with both neighbours; a partial
    last block row)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, W, H, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    G, Y = _frame(W, H)
    full = _oracle_fn(oracle_mod)(G, Y).numpy()
    np.testing.assert_array_equal(got, full)

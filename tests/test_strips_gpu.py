"""Strip sharding of one frame on the GPU (-m gpu).

Each strip (own block rows + a halo of R + 1 block rows, strips.py) is denoised through
the C ABI as a frame of its own; the stitched own rows must match the fp64 oracle on the
full frame (north_star tolerance) and the full-frame GPU result.  The strips run one after
another on one GPU: no ranks that wait on one another (the exchange itself is covered by
the gloo test in test_strips.py).
"""
import numpy as np
import pytest
import torch

from tests.parity import assert_parity

pytestmark = pytest.mark.gpu

D, SIGMA = 8, 10.0


def _gpu_fn(flr):
    return lambda g, y: flr.denoise(g, y, block=D, sigma=SIGMA)


@pytest.mark.parametrize("W,H,Q,parts", [(40, 104, 4, 3), (37, 101, 8, 3), (200, 160, 8, 5)])
def test_strips_match_oracle_full_frame(oracle_mod, W, H, Q, parts):
    import paper_2410_11625_b200 as flr
    from paper_2410_11625_b200 import strips, synth

    G, Y = synth.frame(W, H, Q=Q, seed=77)
    R = flr.effective_radius(block=D, sigma=SIGMA)
    g, y = G.unsqueeze(0).cuda(), Y.unsqueeze(0).cuda()
    got = strips.denoise_strips_local(_gpu_fn(flr), g, y, D, R, parts)
    full_gpu = _gpu_fn(flr)(g, y)
    torch.cuda.synchronize()
    ref = oracle_mod.denoise(G.unsqueeze(0).numpy(), Y.unsqueeze(0).numpy(), D=D, sigma=SIGMA, R=R)
    assert_parity(got.cpu().numpy(), ref, f"strips {W}x{H} Q={Q} parts={parts}")
    assert_parity(got.cpu().numpy(), full_gpu.cpu().numpy().astype(np.float64), "strips vs full GPU")


def test_strips_1080p_eight_parts_match_full_frame():
    """C2 geometry (1080p, Q=8) cut into 8 strips, as an 8-GPU strip run would hold it."""
    import paper_2410_11625_b200 as flr
    from paper_2410_11625_b200 import strips, synth

    G, Y = synth.frame(1920, 1080, Q=8, seed=1000, device="cuda")
    g, y = G.unsqueeze(0).contiguous(), Y.unsqueeze(0).contiguous()
    R = flr.effective_radius(block=D, sigma=SIGMA)
    got = strips.denoise_strips_local(_gpu_fn(flr), g, y, D, R, 8)
    full = _gpu_fn(flr)(g, y)
    torch.cuda.synchronize()
    assert torch.isfinite(got).all()
    assert_parity(got.cpu().numpy(), full.cpu().numpy().astype(np.float64), "1080p strips vs full")
    # the strips run the full frame's kernels on a sub-grid of its blocks: same arithmetic,
    # same order (measured bitwise equal on B200)
    assert torch.equal(got, full)


def test_strips_fp16_guides_match_full_frame():
    """fp16 guide planes through the strip path: same kernels per strip."""
    import paper_2410_11625_b200 as flr
    from paper_2410_11625_b200 import strips, synth

    G, Y = synth.frame(960, 544, Q=8, seed=31, device="cuda")
    g, y = G.half().unsqueeze(0).contiguous(), Y.unsqueeze(0).contiguous()
    R = flr.effective_radius(block=D, sigma=SIGMA)
    got = strips.denoise_strips_local(_gpu_fn(flr), g, y, D, R, 4)
    full = _gpu_fn(flr)(g, y)
    torch.cuda.synchronize()
    assert_parity(got.cpu().numpy(), full.cpu().numpy().astype(np.float64), "fp16 strips vs full")


@pytest.mark.parametrize("W,H,Q,sigma,block", [(7680, 4320, 8, 20.0, 8), (8192, 8192, 4, 10.0, 8)])
def test_max_size_frame_sampled_by_oracle_strips(oracle_mod, W, H, Q, sigma, block):
    """Maximum sizes (8K UHD with the C3 window; a 64-Mpixel square): the GPU denoises the
    whole frame; the oracle, too slow for the frame, denoises three block-row bands (top,
    middle, bottom) each extended by the (R + 1)-block halo -- which reproduces its own
    full-frame rows bitwise (test_strips.py) -- and the GPU's rows must match them."""
    import paper_2410_11625_b200 as flr
    from paper_2410_11625_b200 import strips, synth

    G, Y = synth.frame(W, H, Q=Q, seed=8000 + Q, device="cuda")
    g, y = G.unsqueeze(0).contiguous(), Y.unsqueeze(0).contiguous()
    del G, Y
    out = flr.denoise(g, y, block=block, sigma=sigma)
    torch.cuda.synchronize()
    R = flr.effective_radius(block=block, sigma=sigma)
    h = strips.halo_blocks(R) * block
    By = -(-H // block)
    for b_lo in (0, By // 2, By - 4):
        lo, hi = b_lo * block, min(H, (b_lo + 4) * block)
        ilo, ihi = max(0, lo - h), min(H, hi + h)
        ref = oracle_mod.denoise(g[..., ilo:ihi, :].cpu().numpy(), y[..., ilo:ihi, :].cpu().numpy(),
                                 D=block, sigma=sigma, R=R)
        assert_parity(out[..., lo:hi, :].cpu().numpy(), ref[..., lo - ilo:hi - ilo, :],
                      f"{W}x{H} rows {lo}-{hi}")

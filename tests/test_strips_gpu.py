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

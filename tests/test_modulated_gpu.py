"""GPU <-> oracle parity of the paper's albedo protocol (-m gpu).

flr_denoise_modulated (demodulate by max(albedo, floor), FLR denoise, remodulate, add the
direct light, readings R20/R21) against oracle.denoise_modulated on
identical seeded inputs, for the fused shapes (demodulation inside the moment kernel,
remodulation inside the apply kernel) and the unfused ones (elementwise kernels around
the plain path): same bar as every other parity test, |gpu - ref| <= 1e-5 + 1e-4 |ref|.
"""
import numpy as np
import pytest
import torch

from tests.parity import assert_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def flr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2410_11625_b200 as m

    m.lib()
    return m


def _case(flr, oracle_mod, W, H, Q, seed, block=8, sigma=10.0, direct=True, zero_albedo=False, floor=1e-3):
    from paper_2410_11625_b200 import synth

    G, P, A, Dl = synth.modulated_frame(W, H, Q=Q, seed=seed)
    if zero_albedo:  # below the floor: the division is guarded, the remodulation gives 0 (+ direct)
        A = A.clone()
        A[:, : H // 5, : W // 7] = 0.0
        A[1, H // 3: H // 3 + 2, :] = 2e-4
    d = Dl if direct else None
    out = flr.denoise_modulated(G[None].cuda(), P[None].cuda(), A[None].cuda(),
                                d[None].cuda() if d is not None else None, block=block, sigma=sigma,
                                albedo_floor=floor)
    names = flr.last_launch_names()
    torch.cuda.synchronize()
    R = flr.effective_radius(block=block, sigma=sigma)
    ref = oracle_mod.denoise_modulated(G.numpy(), P.numpy(), A.numpy(), d.numpy() if d is not None else None,
                                       D=block, sigma=sigma, R=R, floor=floor)
    rep = assert_parity(out.cpu().numpy(), ref, f"modulated {W}x{H} Q={Q} D={block}")
    return rep, names


def test_modulated_c2_1080p_fused(flr, oracle_mod):
    rep, names = _case(flr, oracle_mod, 1920, 1080, 8, 1101)
    assert names == ["k_fit_ws_mod", "k_blur_solve_tile", "k_apply_ws_mod"], names
    print("modulated C2 parity", rep)


def test_modulated_c1_and_no_direct(flr, oracle_mod):
    _, names = _case(flr, oracle_mod, 64, 64, 4, 1102, direct=False)
    assert names[0] == "k_fit_ws_mod" and names[-1] == "k_apply_ws_mod", names


def test_modulated_floor_region(flr, oracle_mod):
    _case(flr, oracle_mod, 256, 136, 8, 1103, zero_albedo=True)


@pytest.mark.parametrize("W,H,Q,block", [(37, 23, 4, 8), (130, 66, 8, 4), (96, 64, 3, 2), (128, 72, 8, 16)])
def test_modulated_unfused_and_mixed_shapes(flr, oracle_mod, W, H, Q, block):
    """Odd widths (unfused demod/remod kernels), D=4 (fused demodulation, unfused
    remodulation), D<4 (unfused), D=16 (both fused)."""
    _, names = _case(flr, oracle_mod, W, H, Q, 1104 + W, block=block, sigma=2.5 * block)
    fused_fit = W % 4 == 0 and block in (4, 8, 16)
    fused_apply = W % 4 == 0 and block % 8 == 0
    assert (names[0] == "k_fit_ws_mod") == fused_fit, names
    assert (names[-1] == "k_apply_ws_mod") == fused_apply, names
    assert (names[0] == "k_demod") == (not fused_fit), names
    assert (names[-1] == "k_remod") == (not fused_apply), names


def test_modulated_rejects_bad_floor(flr):
    from paper_2410_11625_b200 import synth

    G, P, A, Dl = synth.modulated_frame(64, 64, Q=4, seed=1110)
    with pytest.raises(flr.FLRError):
        flr.denoise_modulated(G[None].cuda(), P[None].cuda(), A[None].cuda(), None, albedo_floor=0.0)

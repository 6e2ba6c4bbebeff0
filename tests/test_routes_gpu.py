"""Every kernel route the library selects (by shape, alignment, Q, R and batch size; there
are no environment switches) meets the parity bar against the fp64 oracle (-m gpu), and the
launch list names the route's kernels."""
import pytest
import torch

from tests.parity import assert_parity

pytestmark = pytest.mark.gpu

# (W, H, Q, frames, sigma, kernels expected in the launch list)
CASES = [
    (640, 360, 8, 1, 10.0, ["k_fit_ws", "k_blur_solve_tile", "k_apply_ws"]),
    (640, 360, 8, 24, 10.0, ["k_fit_ws", "k_blur_solve_tile", "k_apply_ws"]),  # batch
    (1000, 520, 8, 1, 20.0, ["k_blur_solve_tile"]),  # R = 5: 11-component groups
    (1032, 264, 4, 2, 10.0, ["k_fit_ws", "k_blur_solve_tile"]),  # Q = 4, edge segment
    (640, 360, 11, 1, 10.0, ["k_fit_ws", "k_blur_rows", "k_solve_rows"]),  # Q > 8: row blur
    (512, 264, 4, 1, 80.0, ["k_hblur", "k_vblur_solve"]),  # R = 20 > 8: two-pass blur
    (642, 360, 8, 1, 10.0, ["k_fit_moments", "k_blur_solve_tile", "k_apply_tile"]),  # W % 4 != 0
]


@pytest.mark.parametrize("W,H,Q,n,sigma,expect", CASES, ids=[f"{c[0]}x{c[1]}q{c[2]}n{c[3]}s{int(c[4])}" for c in CASES])
def test_route(oracle_mod, W, H, Q, n, sigma, expect):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2410_11625_b200 as flr
    from paper_2410_11625_b200 import synth

    G, Y = synth.batch(n, W, H, Q=Q, seed0=7000 + W + n)
    out = flr.denoise(G.cuda(), Y.cuda(), sigma=sigma)
    torch.cuda.synchronize()
    names = flr.last_launch_names()
    for k in expect:
        assert k in names, (k, names)
    R = flr.effective_radius(block=8, sigma=sigma)
    check = range(n) if n <= 3 else (0, n // 2, n - 1)
    for f in check:
        ref = oracle_mod.denoise(G[f:f + 1].numpy(), Y[f:f + 1].numpy(), D=8, sigma=sigma, R=R)
        assert_parity(out[f:f + 1].cpu().numpy(), ref, f"route {names} frame {f}")


@pytest.mark.parametrize("Q", [3, 7, 8, 9, 11])
def test_fit_packed_models(oracle_mod, Q):
    """flr_fit writes the ABI's packed [Q+1][3] models (the tile kernel's scalar store path
    for Q <= 8; for Q > 8 k_solve_rows when 3(Q+1) is a whole number of float4s, else
    k_solve); pushed through the oracle's fp64 apply they meet the bar."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2410_11625_b200 as flr
    from paper_2410_11625_b200 import synth

    W, H = 328, 200
    G, Y = synth.batch(1, W, H, Q=Q, seed0=7500 + Q)
    m = flr.fit(G.cuda(), Y.cuda())
    torch.cuda.synchronize()
    names = flr.last_launch_names()
    want = "k_blur_solve_tile" if Q <= 8 else ("k_solve_rows" if 3 * (Q + 1) % 4 == 0 else "k_solve")
    assert want in names, names
    got = oracle_mod.apply(m.cpu().numpy(), G.numpy(), 8)
    ref = oracle_mod.denoise(G.numpy(), Y.numpy(), D=8, sigma=10.0, R=3)
    assert_parity(got, ref, f"flr_fit Q={Q} through the oracle apply")


@pytest.mark.parametrize("W,H,n", [(640, 360, 5), (1032, 264, 3)])
def test_batched_denoise_runs_frame_by_frame(oracle_mod, W, H, n):
    """A batched denoise whose frames fit in L2 runs fit -> K2 -> apply per frame (flr_api.cu,
    DESIGN section 7): 3 launches per frame, each frame bitwise equal to a single-frame call
    (same kernels, same arithmetic), and the oracle bar on first, middle and last frames."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2410_11625_b200 as flr
    from paper_2410_11625_b200 import synth

    G, Y = synth.batch(n, W, H, Q=8, seed0=7300 + W)
    g, y = G.cuda(), Y.cuda()
    out = flr.denoise(g, y)
    torch.cuda.synchronize()
    names = flr.last_launch_names()
    assert names == ["k_fit_ws", "k_blur_solve_tile", "k_apply_ws"] * n, names
    for f in range(n):
        single = flr.denoise(g[f:f + 1].contiguous(), y[f:f + 1].contiguous())
        torch.cuda.synchronize()
        assert torch.equal(out[f:f + 1], single), f"frame {f} differs from its single-frame call"
    R = flr.effective_radius(block=8, sigma=10.0)
    for f in (0, n // 2, n - 1):
        ref = oracle_mod.denoise(G[f:f + 1].numpy(), Y[f:f + 1].numpy(), D=8, sigma=10.0, R=R)
        assert_parity(out[f:f + 1].cpu().numpy(), ref, f"batched frame {f}")

"""Pins for the float64 CPU oracle (-m "not gpu").

Each test checks oracle/flr_ref.c against something OTHER than itself: raw-pixel
brute-force least squares (tests/brute.py), closed forms derived by hand, the
paper's stated limits, exact invariances, and the cited golden fixture.  The
pin ids P1..P12 follow SURVEY.md section 8(c).
"""
import math
import os

import numpy as np
import pytest

from tests import brute

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def rand_planes(rng, Q, H, W, lo=0.0, hi=1.0):
    return rng.uniform(lo, hi, size=(Q, H, W)).astype(np.float32)


# ---------------------------------------------------------------- P1: K1 closed form
def test_p1_constant_block_moments(oracle_mod):
    """A constant D x D block (g, y) has n = D^2, u = D^2 g, S = D^2 g g^T, N_0 = D^2 y
    (SPEC S:312)."""
    D, Q = 8, 3
    g = np.array([0.25, -0.5, 0.75], dtype=np.float32)
    y = np.array([0.1, 0.2, 0.3], dtype=np.float32)
    G = np.broadcast_to(g[:, None, None], (Q, D, D)).copy()
    Y = np.broadcast_to(y[:, None, None], (3, D, D)).copy()
    M, N = oracle_mod.moments(G, Y, D)
    xt = np.concatenate([[1.0], g.astype(np.float64)])
    assert M.shape == (1, 1, 1, Q + 1, Q + 1)
    np.testing.assert_allclose(M[0, 0, 0], D * D * np.outer(xt, xt), rtol=1e-15)
    np.testing.assert_allclose(N[0, 0, 0], D * D * np.outer(xt, y.astype(np.float64)), rtol=1e-15)


def test_p1_truncated_edge_blocks(oracle_mod):
    """Edge blocks are truncated (R5): n counts only in-image pixels."""
    rng = np.random.default_rng(1)
    G = rand_planes(rng, 2, 11, 13)
    Y = rand_planes(rng, 3, 11, 13)
    M, N = oracle_mod.moments(G, Y, 4)
    assert M.shape[1:3] == (3, 4)
    counts = M[0, :, :, 0, 0]
    np.testing.assert_array_equal(counts, [[16, 16, 16, 4], [16, 16, 16, 4], [12, 12, 12, 3]])
    # a plain numpy sum over the same pixels
    np.testing.assert_allclose(N[0, 2, 3, 0], Y[:, 8:11, 12:13].astype(np.float64).sum((1, 2)), rtol=1e-14)
    np.testing.assert_allclose(M[0, 1, 2, 1, 2],
                               (G[0, 4:8, 8:12].astype(np.float64) * G[1, 4:8, 8:12]).sum(), rtol=1e-14)


# ---------------------------------------------------------------- P2: K2 blur
def test_p2_blur_impulse_response(oracle_mod):
    """An impulse in the moment field spreads as g_dy g_dx with g_i = exp(-i^2/2s^2)
    (P:299-300), zero outside |d| <= R, truncated at the grid edge (R3)."""
    P, By, Bx, s, R = 2, 9, 11, 1.25, 3
    M = np.zeros((1, By, Bx, P, P))
    N = np.zeros((1, By, Bx, P, 3))
    M[0, 4, 2, 0, 0] = 1.0
    N[0, 4, 2, 1, 2] = 2.0
    Mb, Nb = oracle_mod.blur(M, N, s, R)
    for by in range(By):
        for bx in range(Bx):
            dy, dx = by - 4, bx - 2
            w = math.exp(-dy * dy / (2 * s * s)) * math.exp(-dx * dx / (2 * s * s)) \
                if abs(dy) <= R and abs(dx) <= R else 0.0
            assert Mb[0, by, bx, 0, 0] == pytest.approx(w, rel=1e-14, abs=1e-300)
            assert Nb[0, by, bx, 1, 2] == pytest.approx(2 * w, rel=1e-14, abs=1e-300)
    assert np.count_nonzero(Mb) == 6 * 7  # columns -1..5 clipped to 0..5, rows 1..7


def test_p2_taps(oracle_mod):
    g = oracle_mod.gauss_taps(1.25, 3)
    np.testing.assert_allclose(g, [math.exp(-i * i / (2 * 1.25 ** 2)) for i in range(-3, 4)], rtol=1e-15)


# ---------------------------------------------------------------- P3: whole fit = brute-force WLS
@pytest.mark.parametrize("D,Q,W,H,sigma,R", [(8, 3, 29, 21, 10.0, 2), (4, 2, 19, 14, 5.0, 3),
                                             (2, 4, 9, 7, 3.0, 2)])
def test_p3_fit_equals_bruteforce_wls_unregularised(oracle_mod, D, Q, W, H, sigma, R):
    """At eps = eps_mul = 0 each block model is the plain weighted LS fit (P:258-270,
    P:303-307) with pixel weights g(block dy) g(block dx) -- checked by lstsq on pixels."""
    rng = np.random.default_rng(D * 100 + Q)
    G = rand_planes(rng, Q, H, W, -1, 1)
    Y = rand_planes(rng, 3, H, W, 0, 2)
    A = oracle_mod.fit(G, Y, D=D, sigma=sigma, R=R, eps_add=0.0, eps_mul=0.0)[0]
    Ab = brute.fit_blocks(G, Y, D, sigma, R, 0.0, 0.0)
    np.testing.assert_allclose(A, Ab, rtol=1e-9, atol=1e-10)


@pytest.mark.parametrize("eps_add,eps_mul", [(1e-5, 1e-4), (1e-2, 0.0), (0.0, 0.3), (0.05, 0.2)])
def test_p3_fit_equals_bruteforce_ridge(oracle_mod, eps_add, eps_mul):
    """With regularisation, the appendix model equals the ridge LS minimiser with the
    penalty derived in tests/brute.py (independent route through P:683-709)."""
    rng = np.random.default_rng(7)
    Q, H, W, D = 3, 17, 23, 4
    G = rand_planes(rng, Q, H, W, 0.2, 0.9)  # non-zero means exercise eps_mul terms
    Y = rand_planes(rng, 3, H, W, 0, 1)
    A = oracle_mod.fit(G, Y, D=D, sigma=6.0, R=2, eps_add=eps_add, eps_mul=eps_mul)[0]
    Ab = brute.fit_blocks(G, Y, D, 6.0, 2, eps_add, eps_mul)
    np.testing.assert_allclose(A, Ab, rtol=1e-8, atol=1e-9)


# ---------------------------------------------------------------- P4: D = 1 = dense windowed regression
def test_p4_block1_equals_dense_windowed(oracle_mod):
    """With 1x1 blocks the blocked method IS the per-pixel windowed regression of
    Fig. 3: per-pixel Gaussian-window moments + the appendix solver."""
    rng = np.random.default_rng(3)
    Q, H, W = 2, 9, 11
    G = rand_planes(rng, Q, H, W)
    Y = rand_planes(rng, 3, H, W)
    out = oracle_mod.denoise(G, Y, D=1, sigma=1.5, R=3, eps_add=1e-3, eps_mul=1e-2)[0]
    ref = brute.dense_windowed(G, Y, 1.5, 3, 1e-3, 1e-2)
    np.testing.assert_allclose(out, ref, rtol=1e-9, atol=1e-11)


# ---------------------------------------------------------------- P5: Q = 1 closed form
@pytest.mark.parametrize("eps_add,eps_mul", [(1e-5, 1e-4), (0.01, 0.1), (0.0, 0.0)])
def test_p5_q1_closed_form(oracle_mod, eps_add, eps_mul):
    """Q = 1 by hand from P:683-716: W^ = var + 2 eps_mul mu^2 + eps_add, C^ = 1,
    B^ = cov / sigma^, A^ = B^/(1 + eps_add) => slope = cov / ((var + 2 eps_mul mu^2 +
    eps_add)(1 + eps_add)), bias = mu_Y - slope mu_X.  (He et al.'s guided filter
    a = cov/(var + eps) when eps_mul = 0, up to the (1 + eps) factor.)"""
    rng = np.random.default_rng(5)
    x = rng.uniform(0.3, 0.8, 40)
    y = rng.uniform(0, 1, (40, 3))
    w = rng.uniform(0.1, 1.0, 40)
    M = np.array([[w.sum(), (w * x).sum()], [(w * x).sum(), (w * x * x).sum()]])
    N = np.stack([(w[:, None] * y).sum(0), (w[:, None] * x[:, None] * y).sum(0)])
    A = oracle_mod.solve_block(M, N, eps_add, eps_mul)
    n = w.sum()
    mu = (w * x).sum() / n
    muy = (w[:, None] * y).sum(0) / n
    var = (w * (x - mu) ** 2).sum() / n
    cov = (w[:, None] * (x - mu)[:, None] * (y - muy)).sum(0) / n
    slope = cov / ((var + 2 * eps_mul * mu * mu + eps_add) * (1 + eps_add))
    np.testing.assert_allclose(A[1], slope, rtol=1e-12)
    np.testing.assert_allclose(A[0], muy - slope * mu, rtol=1e-12, atol=1e-15)


# ---------------------------------------------------------------- P6-P8: end-to-end exact cases
def test_p6_affine_radiance_is_reproduced(oracle_mod):
    """If Y = X~ A globally and the guides are non-degenerate, the unregularised
    regression reproduces Y exactly."""
    rng = np.random.default_rng(11)
    Q, H, W = 4, 24, 32
    G = rand_planes(rng, Q, H, W, -1, 1)
    A_true = rng.normal(size=(Q + 1, 3))
    Xt = np.concatenate([np.ones((1, H, W)), G.astype(np.float64)])
    Y = np.einsum("qhw,qc->chw", Xt, A_true)
    out = oracle_mod.denoise(G, Y.astype(np.float32), D=8, sigma=10.0, R=3, eps_add=0.0, eps_mul=0.0)[0]
    np.testing.assert_allclose(out, Y.astype(np.float32).astype(np.float64), atol=2e-6)
    Y64 = np.einsum("qhw,qc->chw", Xt, A_true).astype(np.float32)
    np.testing.assert_allclose(out, Y64, atol=2e-6)


def test_p7_constant_image_maps_to_itself(oracle_mod):
    """Constant Y = c: B^ = 0, so every model is the bias c, for any eps."""
    rng = np.random.default_rng(12)
    G = rand_planes(rng, 5, 20, 27)
    c = np.array([0.3, 1.7, 0.02], dtype=np.float32)
    Y = np.broadcast_to(c[:, None, None], (3, 20, 27)).copy()
    for ea, em in [(1e-5, 1e-4), (0.1, 0.5), (0.0, 0.0)]:
        out = oracle_mod.denoise(G, Y, D=4, sigma=6.0, R=2, eps_add=ea, eps_mul=em)[0]
        np.testing.assert_allclose(out, np.broadcast_to(c.astype(np.float64)[:, None, None], out.shape),
                                   rtol=1e-12)


def test_p8_huge_eps_is_a_gaussian_blur(oracle_mod):
    """eps -> inf interpolates to a Gaussian blur: the output tends to the
    bilinear blend of Gaussian-weighted block means of Y."""
    rng = np.random.default_rng(13)
    Q, H, W, D, s, R = 3, 16, 24, 4, 1.5, 2
    G = rand_planes(rng, Q, H, W)
    Y = rand_planes(rng, 3, H, W)
    out = oracle_mod.denoise(G, Y, D=D, sigma=s * D, R=R, eps_add=1e7, eps_mul=0.0)[0]
    By, Bx = H // D, W // D
    means = np.zeros((By, Bx, Q + 1, 3))
    for by in range(By):
        for bx in range(Bx):
            w = brute.block_pixel_weights(W, H, D, bx, by, s, R)
            means[by, bx, 0] = (w[None] * Y).sum((1, 2)) / w.sum()
    ref = brute.apply_blend(means, G, D)
    np.testing.assert_allclose(out, ref, atol=1e-6)


# ---------------------------------------------------------------- P9: invariances
def _scene(rng, Q=4, H=24, W=32):
    G = rand_planes(rng, Q, H, W, 0.1, 0.9)
    Y = rand_planes(rng, 3, H, W, 0.0, 1.0)
    return G, Y


def test_p9_guide_permutation_invariance(oracle_mod):
    rng = np.random.default_rng(21)
    G, Y = _scene(rng)
    a = oracle_mod.denoise(G, Y, D=8, sigma=10.0, R=2)
    b = oracle_mod.denoise(G[[2, 0, 3, 1]], Y, D=8, sigma=10.0, R=2)
    np.testing.assert_allclose(a, b, rtol=1e-11, atol=1e-13)


def test_p9_radiance_affine_equivariance(oracle_mod):
    """The method is linear in X^T Y with the bias column: aY + b -> a I + b."""
    rng = np.random.default_rng(22)
    G, Y = _scene(rng)
    a = oracle_mod.denoise(G, Y, D=8, sigma=10.0, R=2)
    Y2 = (2.5 * Y.astype(np.float64) + 0.75)
    b = oracle_mod.denoise(G, Y2.astype(np.float32), D=8, sigma=10.0, R=2)
    Y2r = Y2.astype(np.float32).astype(np.float64)
    ref = oracle_mod.denoise(G, Y2r.astype(np.float32), D=8, sigma=10.0, R=2)
    np.testing.assert_allclose(b, ref, rtol=1e-13)
    np.testing.assert_allclose(b, 2.5 * a + 0.75, rtol=1e-6, atol=1e-6)  # f32 rounding of Y2


def test_p9_global_weight_scale_invariance(oracle_mod):
    """Scaling all moments by a constant (unit-sum vs peak-1 Gaussian, R2) leaves A unchanged."""
    rng = np.random.default_rng(23)
    M = rng.normal(size=(5, 5))
    M = M @ M.T + 5 * np.eye(5)
    M[0, 0] = 7.0
    N = rng.normal(size=(5, 3))
    a = oracle_mod.solve_block(M, N)
    b = oracle_mod.solve_block(M * 0.0137, N * 0.0137)
    np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-14)


def test_p9_shift_invariance_iff_eps_mul_zero(oracle_mod):
    """Adding a constant to one guide only moves mu_X; with eps_mul = 0 the output is
    unchanged, with eps_mul > 0 (the diag(mu^2) and mu mu^T terms) it changes."""
    rng = np.random.default_rng(24)
    G, Y = _scene(rng)
    G2 = G.copy()
    G2[1] += np.float32(0.5)
    a0 = oracle_mod.denoise(G, Y, D=8, sigma=10.0, R=2, eps_add=1e-5, eps_mul=0.0)
    b0 = oracle_mod.denoise(G2, Y, D=8, sigma=10.0, R=2, eps_add=1e-5, eps_mul=0.0)
    np.testing.assert_allclose(a0, b0, rtol=1e-5, atol=1e-6)
    a1 = oracle_mod.denoise(G, Y, D=8, sigma=10.0, R=2, eps_add=1e-5, eps_mul=0.05)
    b1 = oracle_mod.denoise(G2, Y, D=8, sigma=10.0, R=2, eps_add=1e-5, eps_mul=0.05)
    assert np.abs(a1 - b1).max() > 1e-3


def test_p9_scale_invariance_iff_eps_add_zero(oracle_mod):
    """Scaling one guide: invariant with eps_add = 0 (any eps_mul); the eps_add I term breaks it."""
    rng = np.random.default_rng(25)
    G, Y = _scene(rng)
    G2 = G.copy()
    G2[2] *= np.float32(4.0)
    a0 = oracle_mod.denoise(G, Y, D=8, sigma=10.0, R=2, eps_add=0.0, eps_mul=0.01)
    b0 = oracle_mod.denoise(G2, Y, D=8, sigma=10.0, R=2, eps_add=0.0, eps_mul=0.01)
    np.testing.assert_allclose(a0, b0, rtol=1e-8, atol=1e-9)
    a1 = oracle_mod.denoise(G, Y, D=8, sigma=10.0, R=2, eps_add=0.05, eps_mul=0.01)
    b1 = oracle_mod.denoise(G2, Y, D=8, sigma=10.0, R=2, eps_add=0.05, eps_mul=0.01)
    assert np.abs(a1 - b1).max() > 1e-3


def test_p9_constant_guide_noop_iff_eps_mul_zero(oracle_mod):
    rng = np.random.default_rng(26)
    G, Y = _scene(rng)
    Gc = np.concatenate([G, np.full((1,) + G.shape[1:], 0.6, dtype=np.float32)])
    a0 = oracle_mod.denoise(G, Y, D=8, sigma=10.0, R=2, eps_add=1e-4, eps_mul=0.0)
    b0 = oracle_mod.denoise(Gc, Y, D=8, sigma=10.0, R=2, eps_add=1e-4, eps_mul=0.0)
    np.testing.assert_allclose(a0, b0, rtol=1e-9, atol=1e-10)
    a1 = oracle_mod.denoise(G, Y, D=8, sigma=10.0, R=2, eps_add=1e-4, eps_mul=0.2)
    b1 = oracle_mod.denoise(Gc, Y, D=8, sigma=10.0, R=2, eps_add=1e-4, eps_mul=0.2)
    assert np.abs(a1 - b1).max() > 1e-4


# ---------------------------------------------------------------- P10: degenerate guides
def test_p10_duplicated_and_flat_guides_stay_finite(oracle_mod):
    """Rank-deficient moments (duplicated channel, exactly flat regions) must not give
    NaNs with the default regularisation."""
    from paper_2410_11625_b200 import synth

    G, Y = synth.frame(96, 64, Q=8, seed=1234, duplicate_guide=True)
    G = G.numpy()
    G[:, :32, :] = G[:, :1, :1]  # a large exactly-flat region
    out = oracle_mod.denoise(G, Y.numpy(), D=8, sigma=10.0)
    assert np.isfinite(out).all()


# ---------------------------------------------------------------- P11: apply weights
def test_p11_apply_ramp_matches_golden(oracle_mod):
    """Two blocks with bias 0 and 1 (zero slopes) give the cited ramp pattern."""
    path = os.path.join(GOLDEN, "apply_ramp_D8.txt")
    expect = np.loadtxt(path, comments="#")
    A = np.zeros((1, 2, 2, 3))
    A[0, 1, 0, :] = 1.0
    G = np.zeros((1, 8, 16), dtype=np.float32)
    out = oracle_mod.apply(A[None], G, 8)[0]
    for c in range(3):
        for y in range(8):
            np.testing.assert_allclose(out[c, y], expect, rtol=0, atol=0)


def test_p11_equal_models_give_plain_apply(oracle_mod):
    rng = np.random.default_rng(31)
    Q, H, W = 3, 13, 19
    G = rand_planes(rng, Q, H, W)
    A1 = rng.normal(size=(Q + 1, 3))
    A = np.broadcast_to(A1, (2, 3, Q + 1, 3)).copy()
    out = oracle_mod.apply(A[None], G, 8)[0]
    Xt = np.concatenate([np.ones((1, H, W)), G.astype(np.float64)])
    np.testing.assert_allclose(out, np.einsum("qhw,qc->chw", Xt, A1), rtol=1e-13, atol=1e-14)


def test_p11_apply_matches_bruteforce_blend(oracle_mod):
    rng = np.random.default_rng(32)
    Q, H, W, D = 2, 21, 26, 4
    G = rand_planes(rng, Q, H, W)
    A = rng.normal(size=(6, 7, Q + 1, 3))
    out = oracle_mod.apply(A[None], G, D)[0]
    np.testing.assert_allclose(out, brute.apply_blend(A, G, D), rtol=1e-12, atol=1e-13)


# ---------------------------------------------------------------- P12: upsample
def test_p12_upsample_u1_is_denoise(oracle_mod):
    rng = np.random.default_rng(41)
    G, Y = _scene(rng)
    a = oracle_mod.denoise(G, Y, D=4, sigma=10.0, R=3)
    b = oracle_mod.denoise_upsample(G, Y, G, D_fit=4, U=1, sigma=10.0, R=3)
    np.testing.assert_array_equal(a, b)


def test_p12_upsample_bruteforce(oracle_mod):
    """Fit at low resolution with blocks of D_fit, blur std sigma/(D_fit U) blocks,
    apply hi-res guides with D_out = D_fit U: brute force on pixels."""
    rng = np.random.default_rng(42)
    Q, H, W, D, U = 2, 10, 14, 2, 2
    G = rand_planes(rng, Q, H, W)
    Y = rand_planes(rng, 3, H, W)
    Gh = rand_planes(rng, Q, H * U, W * U)
    out = oracle_mod.denoise_upsample(G, Y, Gh, D_fit=D, U=U, sigma=6.0, R=2, eps_add=1e-3, eps_mul=1e-2)[0]
    A = brute.fit_blocks(G, Y, D, 6.0, 2, 1e-3, 1e-2, U=U)
    np.testing.assert_allclose(out, brute.apply_blend(A, Gh, D * U), rtol=1e-9, atol=1e-10)


def test_p12_affine_field_exact_across_resolutions(oracle_mod):
    rng = np.random.default_rng(43)
    Q, H, W, U = 3, 16, 24, 2
    Gh = rand_planes(rng, Q, H * U, W * U, -1, 1)
    G = Gh[:, ::U, ::U].copy()
    A_true = rng.normal(size=(Q + 1, 3))
    Y = np.einsum("qhw,qc->chw", np.concatenate([np.ones((1, H, W)), G.astype(np.float64)]), A_true)
    out = oracle_mod.denoise_upsample(G, Y.astype(np.float32), Gh, D_fit=4, U=U, sigma=16.0,
                                      R=2, eps_add=0.0, eps_mul=0.0)[0]
    ref = np.einsum("qhw,qc->chw", np.concatenate([np.ones((1, H * U, W * U)), Gh.astype(np.float64)]), A_true)
    np.testing.assert_allclose(out, ref, atol=2e-5)


# ---------------------------------------------------------------- P13: albedo protocol
# "we divide P by A, denoise, then multiply again with A";
# the direct light is noise-free and added back.  Readings R20 (albedo floor
# 1e-3 in the division only) and R21 (direct added after remodulation) in DESIGN.md.
def test_p13_unit_albedo_is_plain_denoise(oracle_mod):
    rng = np.random.default_rng(50)
    G, Y = _scene(rng)
    A = np.ones_like(Y)
    np.testing.assert_array_equal(oracle_mod.denoise_modulated(G, Y, A, D=4, sigma=10.0, R=3),
                                  oracle_mod.denoise(G, Y, D=4, sigma=10.0, R=3))


def test_p13_modulated_constant_lighting_is_reproduced(oracle_mod):
    """P = A * L with constant lighting L: demodulation gives L everywhere, FLR maps a
    constant to itself (P7), remodulation gives back P."""
    rng = np.random.default_rng(51)
    G, _ = _scene(rng)
    H, W = G.shape[1:]
    L = np.array([0.3, 1.7, 0.05])[:, None, None]
    A = rand_planes(rng, 3, H, W, 0.05, 1.0)
    P = (A.astype(np.float64) * L).astype(np.float32)
    out = oracle_mod.denoise_modulated(G, P, A, D=4, sigma=8.0, R=2)[0]
    np.testing.assert_allclose(out, A.astype(np.float64) * L, rtol=1e-6, atol=1e-9)


def test_p13_floor_and_remodulation_by_hand(oracle_mod):
    """Against the composition written out with numpy and the plain oracle: the floor
    only guards the division, the remodulation uses the raw albedo (zero albedo gives
    zero output), and the direct light is added last."""
    rng = np.random.default_rng(52)
    G, Y = _scene(rng)
    A = rand_planes(rng, 3, *Y.shape[1:], 0.0, 1.0)
    A[:, :5, :7] = 0.0             # below the floor: divide by 1e-3
    A[1, 10:12, :] = 5e-4
    Dl = rand_planes(rng, 3, *Y.shape[1:], 0.0, 2.0)
    floor = 1e-3
    y = Y.astype(np.float64) / np.maximum(A.astype(np.float64), floor)
    I = oracle_mod.denoise(G, y.astype(np.float32), D=4, sigma=10.0, R=3)[0]
    ref = A.astype(np.float64) * I + Dl.astype(np.float64)
    out = oracle_mod.denoise_modulated(G, Y, A, Dl, D=4, sigma=10.0, R=3, floor=floor)[0]
    # y is rounded to float for the plain oracle: relative 1e-7 differences
    np.testing.assert_allclose(out, ref, rtol=2e-5, atol=1e-6)
    assert np.array_equal(out[:, :5, :7], Dl[:, :5, :7].astype(np.float64))


def test_p13_direct_light_is_additive(oracle_mod):
    rng = np.random.default_rng(53)
    G, Y = _scene(rng)
    A = rand_planes(rng, 3, *Y.shape[1:], 0.05, 1.0)
    Dl = rand_planes(rng, 3, *Y.shape[1:], 0.0, 3.0)
    a = oracle_mod.denoise_modulated(G, Y, A, Dl, D=4, sigma=10.0, R=3)
    b = oracle_mod.denoise_modulated(G, Y, A, None, D=4, sigma=10.0, R=3)
    np.testing.assert_allclose(a - b, Dl[None].astype(np.float64), rtol=0, atol=1e-12)


# ---------------------------------------------------------------- argument errors
def test_oracle_rejects_bad_arguments(oracle_mod):
    G = np.zeros((1, 4, 4), dtype=np.float32)
    Y = np.zeros((3, 4, 4), dtype=np.float32)
    with pytest.raises(ValueError):
        oracle_mod.fit(G, Y, D=4, sigma=-1.0, R=1)
    with pytest.raises(ValueError):
        oracle_mod.fit(G, Y, D=4, sigma=1.0, R=1, eps_mul=1.0)


# ---------------------------------------------------------------- P14: Tikhonov solver
# Eq. tikhonov with Fig. 3's semantics: the blurred outer
# products are Gaussian-weighted MEANS (the torchvision kernel sums to one) and eps I
# regularises the full (Q+1) system including the ones channel (R18, R22).
def test_p14_tikhonov_eps0_equals_unregularised_appendix(oracle_mod):
    """Both solvers reduce to exact weighted least squares when unregularised."""
    rng = np.random.default_rng(60)
    G = rand_planes(rng, 3, 20, 24)
    Y = rand_planes(rng, 3, 20, 24)
    a = oracle_mod.fit_tikhonov(G, Y, D=4, sigma=6.0, eps=0.0)
    b = oracle_mod.fit(G, Y, D=4, sigma=6.0, eps_add=0.0, eps_mul=0.0)
    np.testing.assert_allclose(a, b, rtol=1e-9, atol=1e-11)


@pytest.mark.parametrize("eps", [1e-6, 1e-3, 0.05])
def test_p14_tikhonov_equals_bruteforce_ridge(oracle_mod, eps):
    """Per block: argmin_A sum_p (w_p / sum w) ||y_p - x~_p A||^2 + eps ||A||_F^2 from raw
    pixels by np.linalg.lstsq on sqrt-weighted rows stacked on sqrt(eps) I rows."""
    rng = np.random.default_rng(61)
    Q, H, W, D, sigma, R = 2, 18, 21, 4, 5.0, 2
    G = rand_planes(rng, Q, H, W)
    Y = rand_planes(rng, 3, H, W)
    A = oracle_mod.fit_tikhonov(G, Y, D=D, sigma=sigma, R=R, eps=eps)[0]
    s = sigma / D
    for by, bx in [(0, 0), (2, 3), (4, 5), (1, 2)]:
        w = brute.block_pixel_weights(W, H, D, bx, by, s, R).reshape(-1)
        w = w / w.sum()
        X = np.concatenate([np.ones((1, H * W)), G.reshape(Q, -1).astype(np.float64)]).T
        Yf = Y.reshape(3, -1).astype(np.float64).T
        sw = np.sqrt(w)[:, None]
        lhs = np.concatenate([X * sw, math.sqrt(eps) * np.eye(Q + 1)])
        rhs = np.concatenate([Yf * sw, np.zeros((Q + 1, 3))])
        ref = np.linalg.lstsq(lhs, rhs, rcond=None)[0]
        np.testing.assert_allclose(A[by, bx], ref, rtol=1e-8, atol=1e-10)


def test_p14_tikhonov_d1_is_figure3(oracle_mod):
    """D = 1, sigma = 10, R = 20 (a 41-tap kernel) at interior pixels is Fig. 3's
    local_regression written out with numpy: normalised separable Gaussian, einsum outer
    products, np.linalg.solve(XX + eps I, XY), then x~ . A."""
    rng = np.random.default_rng(62)
    Q, H, W, eps = 2, 46, 44, 1e-6
    G = rand_planes(rng, Q, H, W)
    Y = rand_planes(rng, 3, H, W)
    out = oracle_mod.denoise_tikhonov(G, Y, D=1, sigma=10.0, R=20, eps=eps)[0]
    k1 = np.exp(-np.arange(-20, 21) ** 2 / 200.0)
    k1 /= k1.sum()
    k2 = np.outer(k1, k1)
    X = np.concatenate([np.ones((1, H, W)), G.astype(np.float64)])
    Yd = Y.astype(np.float64)
    for (y, x) in [(20, 20), (22, 23), (25, 21)]:
        win = (slice(y - 20, y + 21), slice(x - 20, x + 21))
        Xw = X[:, win[0], win[1]]
        XX = np.einsum("ikl,jkl,kl->ij", Xw, Xw, k2)
        XY = np.einsum("ikl,jkl,kl->ij", Xw, Yd[:, win[0], win[1]], k2)
        A = np.linalg.solve(XX + eps * np.eye(Q + 1), XY)
        np.testing.assert_allclose(out[:, y, x], X[:, y, x] @ A, rtol=1e-9, atol=1e-11)


def test_p14_tikhonov_huge_eps_shrinks_to_zero(oracle_mod):
    """eps -> infinity shrinks every coefficient, the bias included (R18): output -> 0,
    unlike the appendix solver, whose eps -> infinity limit is a Gaussian blur (P8)."""
    rng = np.random.default_rng(63)
    G, Y = _scene(rng)
    out = oracle_mod.denoise_tikhonov(G, Y, D=4, sigma=8.0, R=2, eps=1e9)
    assert np.abs(out).max() < 1e-7 * np.abs(Y).max() + 1e-12


# ---------------------------------------------------------------- R3: the recorded divergence from SPEC
def _clamp_pixel_weights(W, H, D, bx, by, s, R):
    """SPEC's clamp-to-edge blur of the moment field, written on pixels:
    window block b + d is replaced by the nearest in-grid block, so a border block's
    moments are counted once per clamped offset (weight g(dy) g(dx) each time)."""
    Bx, By = -(-W // D), -(-H // D)
    wb = np.zeros((By, Bx))
    for dy in range(-R, R + 1):
        for dx in range(-R, R + 1):
            wb[min(max(by + dy, 0), By - 1), min(max(bx + dx, 0), Bx - 1)] += brute.gauss(dy, s) * brute.gauss(dx, s)
    return np.kron(wb, np.ones((D, D)))[:H, :W]


def test_r3_clamp_to_edge_differs_only_within_r_blocks_of_the_border(oracle_mod):
    """R3: the oracle and the kernels truncate the blur window at the
    frame edge (zero padding); SPEC's program clamps instead.  Brute-force WLS with the
    clamped weights gives the SAME models for every block at least R blocks from each
    border (its window never leaves the grid) and different ones within R blocks of it;
    the output differences it causes stay within about R + 1 blocks of the border and are
    far above the parity bar there (so the choice is visible, and recorded, not a rounding
    matter)."""
    rng = np.random.default_rng(33)
    Q, D, R, sigma = 3, 4, 2, 6.0
    Bx, By = 9, 8
    W, H = Bx * D, By * D
    G = rand_planes(rng, Q, H, W, 0.1, 0.9)
    Y = rand_planes(rng, 3, H, W, 0.0, 1.0) + 0.5 * G[:1]
    s = sigma / D
    A = oracle_mod.fit(G, Y, D=D, sigma=sigma, R=R)[0]
    Ac = np.zeros_like(A)
    for by in range(By):
        for bx in range(Bx):
            Ac[by, bx] = brute.ridge_lstsq_model(G, Y, _clamp_pixel_weights(W, H, D, bx, by, s, R), 1e-5, 1e-4)
    inner = np.zeros((By, Bx), bool)
    inner[R:By - R, R:Bx - R] = True
    diff = np.abs(A - Ac).max(axis=(2, 3))
    assert diff[inner].max() < 1e-8, diff[inner].max()
    assert diff[~inner].min() > 1e-6, diff[~inner].min()
    O = oracle_mod.apply(A[None], G[None], D)[0]
    Oc = brute.apply_blend(Ac, G, D)
    od = np.abs(O - Oc).max(axis=0)
    m = (R + 1) * D  # pixels whose four blended models are all inner blocks
    assert od[m:H - m, m:W - m].max() < 1e-8
    assert od.max() > 1e-3  # ~100x the 1e-5 absolute parity bar

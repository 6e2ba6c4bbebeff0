"""NumPy brute force used to PIN the oracle (tests only; never imported by the product).

Everything here works on raw pixels with np.linalg.lstsq -- a different route
through the algebra than oracle/flr_ref.c's block moments -> blur -> appendix
chain -- so a dropped term, a wrong sign/index or a transposed operand in the
oracle shows up as a disagreement.
"""
from __future__ import annotations

import math

import numpy as np


def gauss(i, s):
    return math.exp(-(i * i) / (2.0 * s * s))


def block_pixel_weights(W, H, D, bx, by, s, R):
    """Per-pixel weight of the blocked Gaussian window centred on block (bx, by):
    w_p = g(floor(p_y/D) - by) g(floor(p_x/D) - bx) if both offsets are within R
    (P:299-309 weighted LS, P:315-318 moment downsample; zero padding, R3)."""
    w = np.zeros((H, W))
    for y in range(H):
        dy = y // D - by
        if abs(dy) > R:
            continue
        for x in range(W):
            dx = x // D - bx
            if abs(dx) > R:
                continue
            w[y, x] = gauss(dy, s) * gauss(dx, s)
    return w


def weighted_stats(G, Y, w):
    """Weighted mean / population covariance of guides and guide-radiance cross terms."""
    Q = G.shape[0]
    wsum = w.sum()
    X = G.reshape(Q, -1).astype(np.float64)
    Yf = Y.reshape(3, -1).astype(np.float64)
    wf = w.reshape(-1)
    mu = (X * wf).sum(1) / wsum
    muy = (Yf * wf).sum(1) / wsum
    Xc = X - mu[:, None]
    Yc = Yf - muy[:, None]
    cov = (Xc * wf) @ Xc.T / wsum
    cxy = (Xc * wf) @ Yc.T / wsum
    return wsum, mu, muy, cov, cxy


def ridge_lstsq_model(G, Y, w, eps_add, eps_mul):
    """Raw-basis model (P x 3) of the appendix solver, obtained WITHOUT the appendix
    chain: it is the minimiser of the augmented (ridge) least-squares problem

        sum_p w_p || y_p - a0 - x_p^T a ||^2  +  n a^T Lam a,
        Lam = eps_mul (diag(mu^2) + mu mu^T) + eps_add I + eps_add diag(W^_ii),
        W^_ii = var_i + 2 eps_mul mu_i^2 + eps_add,

    solved by np.linalg.lstsq on sqrt-weighted pixel rows stacked on penalty rows.
    Derivation ("ridge form"): with D = diag(sigma^),
    C^ + eps I = D^-1 (W^ + eps D^2) D^-1, so A = D^-1 A^ = (W^ + eps D^2)^-1 cov_xy
    and W^ = W + eps_mul (diag(mu^2) + mu mu^T) + eps_add I (R8)."""
    Q = G.shape[0]
    n, mu, muy, cov, cxy = weighted_stats(G, Y, w)
    X = np.concatenate([np.ones((1, G[0].size)), G.reshape(Q, -1).astype(np.float64)]).T
    Yf = Y.reshape(3, -1).T.astype(np.float64)
    sw = np.sqrt(w.reshape(-1))
    rows = [X * sw[:, None]]
    rhs = [Yf * sw[:, None]]
    if eps_add > 0 or eps_mul > 0:
        var = np.diag(cov)
        What_ii = var + 2.0 * eps_mul * mu * mu + eps_add
        Lam = eps_mul * (np.diag(mu * mu) + np.outer(mu, mu)) + eps_add * np.eye(Q) + eps_add * np.diag(What_ii)
        L = np.linalg.cholesky(Lam)
        pen = np.zeros((Q, Q + 1))
        pen[:, 1:] = math.sqrt(n) * L.T
        rows.append(pen)
        rhs.append(np.zeros((Q, 3)))
    A, *_ = np.linalg.lstsq(np.concatenate(rows), np.concatenate(rhs), rcond=None)
    return A


def fit_blocks(G, Y, D, sigma, R, eps_add, eps_mul, U=1):
    """Models for every block by brute-force weighted LS on raw pixels."""
    Q, H, W = G.shape
    Bx, By = -(-W // D), -(-H // D)
    s = sigma / (D * U)
    A = np.zeros((By, Bx, Q + 1, 3))
    for by in range(By):
        for bx in range(Bx):
            w = block_pixel_weights(W, H, D, bx, by, s, R)
            A[by, bx] = ridge_lstsq_model(G, Y, w, eps_add, eps_mul)
    return A


def apply_blend(A, G, D_out):
    """Bilinear blend of block models at block centres (b + 1/2) D - 1/2 (R4)."""
    Q, H, W = G.shape
    By, Bx = A.shape[:2]
    out = np.zeros((3, H, W))
    for y in range(H):
        fy = (y + 0.5) / D_out - 0.5
        j0 = math.floor(fy)
        ty = fy - j0
        ja, jb = min(max(j0, 0), By - 1), min(max(j0 + 1, 0), By - 1)
        for x in range(W):
            fx = (x + 0.5) / D_out - 0.5
            i0 = math.floor(fx)
            tx = fx - i0
            ia, ib = min(max(i0, 0), Bx - 1), min(max(i0 + 1, 0), Bx - 1)
            Ab = ((1 - ty) * (1 - tx) * A[ja, ia] + (1 - ty) * tx * A[ja, ib]
                  + ty * (1 - tx) * A[jb, ia] + ty * tx * A[jb, ib])
            xt = np.concatenate([[1.0], G[:, y, x].astype(np.float64)])
            out[:, y, x] = xt @ Ab
    return out


def dense_windowed(G, Y, sigma, R, eps_add, eps_mul):
    """Per-pixel windowed weighted LS (Fig. 3 semantics, with the appendix
    solver): window weights g(dy) g(dx), |d| <= R, zero padding; I_k = x_k A_k."""
    Q, H, W = G.shape
    out = np.zeros((3, H, W))
    for y in range(H):
        for x in range(W):
            w = np.zeros((H, W))
            for yy in range(max(0, y - R), min(H, y + R + 1)):
                for xx in range(max(0, x - R), min(W, x + R + 1)):
                    w[yy, xx] = gauss(yy - y, sigma) * gauss(xx - x, sigma)
            A = ridge_lstsq_model(G, Y, w, eps_add, eps_mul)
            out[:, y, x] = np.concatenate([[1.0], G[:, y, x].astype(np.float64)]) @ A
    return out

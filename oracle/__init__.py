"""ctypes front end of the float64 CPU oracle (oracle/flr_ref.c).

TEST INFRASTRUCTURE ONLY: tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs are the only callers.  The product
package ``paper_2410_11625_b200`` never imports this module, and the C oracle
shares no code with the CUDA path.  Every function converts numpy arguments
to C-contiguous float32 inputs / float64 outputs and calls the C function of
the same name; the arithmetic lives in flr_ref.c (citations there).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "flr_ref.c")
_LIB = os.path.join(_HERE, "libflr_ref.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile flr_ref.c -> oracle/libflr_ref.so with gcc (-O2, OpenMP, no -ffast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-fno-fast-math",
               "-ffp-contract=off", "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i, d = ctypes.c_int, ctypes.c_double
        fp, dp = ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_double)
        L.flr_ref_moments.argtypes = [i, i, i, i, i, fp, fp, dp, dp]
        L.flr_ref_gauss_taps.argtypes = [d, i, dp]
        L.flr_ref_blur.argtypes = [i, i, i, i, d, i, dp, dp, dp, dp]
        L.flr_ref_solve_block.argtypes = [i, dp, dp, d, d, dp]
        L.flr_ref_fit.argtypes = [i, i, i, i, i, i, d, i, d, d, fp, fp, dp]
        L.flr_ref_apply.argtypes = [i, i, i, i, i, i, i, dp, fp, dp]
        L.flr_ref_denoise.argtypes = [i, i, i, i, i, d, i, d, d, fp, fp, dp]
        L.flr_ref_denoise_upsample.argtypes = [i, i, i, i, i, i, d, i, d, d, fp, fp, fp, dp]
        L.flr_ref_denoise_modulated.argtypes = [i, i, i, i, i, d, i, d, d, d, fp, fp, fp, fp, dp]
        L.flr_ref_solve_block_tikhonov.argtypes = [i, dp, dp, d, dp]
        L.flr_ref_fit_tikhonov.argtypes = [i, i, i, i, i, i, d, i, d, fp, fp, dp]
        L.flr_ref_num_threads.argtypes = []
        for name in ("flr_ref_moments", "flr_ref_gauss_taps", "flr_ref_blur", "flr_ref_solve_block",
                     "flr_ref_fit", "flr_ref_apply", "flr_ref_denoise", "flr_ref_denoise_upsample",
                     "flr_ref_num_threads", "flr_ref_solve_block_tikhonov", "flr_ref_fit_tikhonov"):
            getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def _f32(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def _f64(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _out(shape):
    a = np.empty(shape, dtype=np.float64)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _check(rc, what):
    if rc != 0:
        raise ValueError(f"{what} returned status {rc}")


def _frames(guides, radiance=None):
    g = np.asarray(guides)
    if g.ndim == 3:
        g = g[None]
    r = None
    if radiance is not None:
        r = np.asarray(radiance)
        if r.ndim == 3:
            r = r[None]
    return g, r


def blocks(W, H, D):
    return (W + D - 1) // D, (H + D - 1) // D


def default_radius(sigma, D_out):
    """R = ceil(2 sigma / D_out) blocks (reading R1: Fig. 3's 41-tap, std-10 kernel
    is radius 2 sigma)."""
    return int(math.ceil(2.0 * sigma / D_out - 1e-12))


def num_threads() -> int:
    return lib().flr_ref_num_threads()


def set_num_threads(n: int) -> None:
    """OpenMP thread count of later oracle calls from this thread (libgomp's
    omp_set_num_threads; the oracle's results do not depend on it)."""
    lib()
    ctypes.CDLL("libgomp.so.1").omp_set_num_threads(int(n))


def moments(guides, radiance, D):
    """Block sums (M [n,By,Bx,P,P], N [n,By,Bx,P,3])."""
    g, r = _frames(guides, radiance)
    n, Q, H, W = g.shape
    P = Q + 1
    Bx, By = blocks(W, H, D)
    g, gp = _f32(g)
    r, rp = _f32(r)
    M, Mp = _out((n, By, Bx, P, P))
    N, Np = _out((n, By, Bx, P, 3))
    _check(lib().flr_ref_moments(n, Q, W, H, D, gp, rp, Mp, Np), "flr_ref_moments")
    return M, N


def gauss_taps(s, R):
    g, gp = _out((2 * R + 1,))
    _check(lib().flr_ref_gauss_taps(float(s), int(R), gp), "flr_ref_gauss_taps")
    return g


def blur(M, N, s, R):
    M, Mp = _f64(M)
    N, Np = _f64(N)
    n, By, Bx, P, _ = M.shape
    Mb, Mbp = _out(M.shape)
    Nb, Nbp = _out(N.shape)
    _check(lib().flr_ref_blur(n, P, Bx, By, float(s), int(R), Mp, Np, Mbp, Nbp), "flr_ref_blur")
    return Mb, Nb


def solve_block(M, N, eps_add=1e-5, eps_mul=1e-4):
    M, Mp = _f64(M)
    N, Np = _f64(N)
    P = M.shape[0]
    A, Ap = _out((P, 3))
    _check(lib().flr_ref_solve_block(P, Mp, Np, float(eps_add), float(eps_mul), Ap),
           "flr_ref_solve_block")
    return A


def fit(guides, radiance, D=8, sigma=10.0, R=None, eps_add=1e-5, eps_mul=1e-4, U=1):
    """Models A [n,By,Bx,P,3] (raw basis, row 0 = bias)."""
    g, r = _frames(guides, radiance)
    n, Q, H, W = g.shape
    if R is None:
        R = default_radius(sigma, D * U)
    Bx, By = blocks(W, H, D)
    g, gp = _f32(g)
    r, rp = _f32(r)
    A, Ap = _out((n, By, Bx, Q + 1, 3))
    _check(lib().flr_ref_fit(n, Q, W, H, D, U, float(sigma), int(R), float(eps_add),
                             float(eps_mul), gp, rp, Ap), "flr_ref_fit")
    return A


def solve_block_tikhonov(M, N, eps=1e-6):
    M, Mp = _f64(M)
    N, Np = _f64(N)
    P = M.shape[0]
    A, Ap = _out((P, 3))
    _check(lib().flr_ref_solve_block_tikhonov(P, Mp, Np, float(eps), Ap), "flr_ref_solve_block_tikhonov")
    return A


def fit_tikhonov(guides, radiance, D=8, sigma=10.0, R=None, eps=1e-6, U=1):
    """Models of the Tikhonov solver (Eq. tikhonov, Fig. 3; R18, R22)."""
    g, r = _frames(guides, radiance)
    n, Q, H, W = g.shape
    if R is None:
        R = default_radius(sigma, D * U)
    Bx, By = blocks(W, H, D)
    g, gp = _f32(g)
    r, rp = _f32(r)
    A, Ap = _out((n, By, Bx, Q + 1, 3))
    _check(lib().flr_ref_fit_tikhonov(n, Q, W, H, D, U, float(sigma), int(R), float(eps), gp, rp, Ap),
           "flr_ref_fit_tikhonov")
    return A


def denoise_tikhonov(guides, radiance, D=8, sigma=10.0, R=None, eps=1e-6):
    """fit_tikhonov + the same blended apply as denoise()."""
    A = fit_tikhonov(guides, radiance, D=D, sigma=sigma, R=R, eps=eps)
    return apply(A, guides, D)


def apply(models, guides, D_out):
    g, _ = _frames(guides)
    A = np.asarray(models, dtype=np.float64)
    if A.ndim == 4:
        A = A[None]
    n, Q, H, W = g.shape
    _, By, Bx, P, _ = A.shape
    assert P == Q + 1
    g, gp = _f32(g)
    A, Ap = _f64(A)
    out, op = _out((n, 3, H, W))
    _check(lib().flr_ref_apply(n, Q, W, H, D_out, Bx, By, Ap, gp, op), "flr_ref_apply")
    return out


def denoise(guides, radiance, D=8, sigma=10.0, R=None, eps_add=1e-5, eps_mul=1e-4):
    g, r = _frames(guides, radiance)
    n, Q, H, W = g.shape
    if R is None:
        R = default_radius(sigma, D)
    g, gp = _f32(g)
    r, rp = _f32(r)
    out, op = _out((n, 3, H, W))
    _check(lib().flr_ref_denoise(n, Q, W, H, D, float(sigma), int(R), float(eps_add),
                                 float(eps_mul), gp, rp, op), "flr_ref_denoise")
    return out


def denoise_modulated(guides, radiance_mod, albedo, direct=None, D=8, sigma=10.0, R=None, eps_add=1e-5,
                      eps_mul=1e-4, floor=1e-3):
    """The paper's albedo protocol: out = A * FLR(guides, P / max(A, floor)) + direct."""
    g, r = _frames(guides, radiance_mod)
    a, _ = _frames(albedo)
    n, Q, H, W = g.shape
    assert a.shape == r.shape, "albedo must have the radiance's shape [n][3][H][W]"
    if R is None:
        R = default_radius(sigma, D)
    g, gp = _f32(g)
    r, rp = _f32(r)
    a, ap = _f32(a)
    dp_ = None
    if direct is not None:
        dd, _ = _frames(direct)
        assert dd.shape == r.shape, "direct must have the radiance's shape [n][3][H][W]"
        dd, dp_ = _f32(dd)
    out, op = _out((n, 3, H, W))
    _check(lib().flr_ref_denoise_modulated(n, Q, W, H, D, float(sigma), int(R), float(eps_add), float(eps_mul),
                                           float(floor), gp, rp, ap, dp_, op), "flr_ref_denoise_modulated")
    return out


def denoise_upsample(guides_lo, radiance_lo, guides_hi, D_fit=4, U=2, sigma=10.0, R=None,
                     eps_add=1e-5, eps_mul=1e-4):
    g, r = _frames(guides_lo, radiance_lo)
    gh, _ = _frames(guides_hi)
    n, Q, H, W = g.shape
    assert gh.shape == (n, Q, H * U, W * U), "hi-res guides must be exactly U x the lo-res size"
    if R is None:
        R = default_radius(sigma, D_fit * U)
    g, gp = _f32(g)
    r, rp = _f32(r)
    gh, ghp = _f32(gh)
    out, op = _out((n, 3, H * U, W * U))
    _check(lib().flr_ref_denoise_upsample(n, Q, W, H, D_fit, U, float(sigma), int(R),
                                          float(eps_add), float(eps_mul), gp, rp, ghp, op),
           "flr_ref_denoise_upsample")
    return out

"""Parity helpers shared by the GPU tests, smoke() and bench.py (tests infrastructure).

The bar (BASELINE.json north_star): elementwise |gpu - oracle| <= ATOL + RTOL |oracle|
on output radiance, with ATOL = 1e-5 and RTOL = 1e-4.
"""
from __future__ import annotations

import numpy as np

ATOL = 1e-5
RTOL = 1e-4


def parity_report(gpu, ref, atol=ATOL, rtol=RTOL):
    g = np.asarray(gpu, dtype=np.float64)
    r = np.asarray(ref, dtype=np.float64)
    assert g.shape == r.shape, (g.shape, r.shape)
    err = np.abs(g - r)
    bound = atol + rtol * np.abs(r)
    ratio = err / bound
    finite = np.isfinite(g).all()
    worst = np.unravel_index(np.nanargmax(ratio), ratio.shape) if ratio.size else ()
    return {
        "max_ratio": float(np.nanmax(ratio)) if ratio.size else 0.0,
        "violations": int((~(err <= bound)).sum()),
        "max_abs": float(err.max()) if err.size else 0.0,
        "finite": bool(finite),
        "worst_index": tuple(int(i) for i in worst),
        "n": int(r.size),
    }


def assert_parity(gpu, ref, what="", atol=ATOL, rtol=RTOL):
    rep = parity_report(gpu, ref, atol, rtol)
    assert rep["finite"], f"{what}: non-finite GPU output"
    assert rep["violations"] == 0, f"{what}: parity violations {rep}"
    return rep

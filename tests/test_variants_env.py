"""Every alternative kernel schedule the library can select meets the parity bar (-m gpu).

The library reads its FLR_* selection switches once per process, so each case runs
tests/variant_run.py in a fresh subprocess with that environment and checks both the
kernels it launched and zero tolerance violations against the fp64 oracle.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (environment, W, H, Q, frames, sigma, kernels expected in the launch list)
CASES = [
    ({}, 640, 360, 8, 1, 10.0, ["k_fit_ws", "k_blur_solve_tile", "k_apply_ws"]),
    ({"FLR_APPLY_RING": "1"}, 640, 360, 8, 2, 10.0, ["k_apply_stream"]),
    ({"FLR_APPLY_RING": "0"}, 640, 360, 8, 2, 10.0, ["k_apply_ws"]),
    ({"FLR_FIT_RING": "1"}, 640, 360, 8, 1, 10.0, ["k_fit_stream"]),
    ({"FLR_FIT_LDG": "1"}, 640, 360, 8, 1, 10.0, ["k_fit_ldg"]),
    ({"FLR_ROWS_SOLVE": "1"}, 640, 360, 8, 1, 10.0, ["k_blur_rows", "k_solve_rows"]),
    ({"FLR_TILE_SOLVE": "1"}, 640, 360, 8, 1, 10.0, ["k_blur_solve"]),
    ({"FLR_WAVE": "1"}, 640, 360, 8, 2, 10.0, ["k_fit_ws", "k_blur_solve_tile", "k_apply_stream"]),
    ({"FLR_WAVE": "1", "FLR_FIT_RING": "1"}, 512, 264, 4, 3, 20.0, ["k_fit_stream", "k_blur_solve_tile"]),
    ({"FLR_NO_PDL": "1"}, 640, 360, 8, 1, 10.0, ["k_fit_ws", "k_blur_solve_tile", "k_apply_ws"]),
    ({}, 1000, 520, 8, 1, 20.0, ["k_blur_solve_tile"]),  # R = 5: 11-component groups
    ({}, 1032, 264, 4, 2, 10.0, ["k_fit_ws", "k_blur_solve_tile"]),  # Q = 4, edge segment
]


@pytest.mark.gpu
@pytest.mark.parametrize("env,W,H,Q,n,sigma,expect", CASES,
                         ids=[(",".join(f"{k}={v}" for k, v in c[0].items()) or "default") + f"-{c[1]}x{c[2]}q{c[3]}n{c[4]}"
                              for c in CASES])
def test_variant_env(env, W, H, Q, n, sigma, expect):
    e = {k: v for k, v in os.environ.items() if not k.startswith("FLR_")}
    e.update(env)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "variant_run.py"), str(W), str(H), str(Q), str(n),
                        str(sigma)], capture_output=True, text=True, env=e, cwd=ROOT, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for k in expect:
        assert k in res["names"], (k, res["names"])
    assert res["violations"] == 0, res

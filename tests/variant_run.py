"""Helper for test_variants_env.py: one parity check of the CUDA path under the kernel
selection environment of THIS process (the library reads its FLR_* switches once).

usage: python tests/variant_run.py W H Q n sigma   -> prints a JSON line
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2410_11625_b200 as flr  # noqa: E402
from paper_2410_11625_b200 import synth  # noqa: E402
from tests.parity import parity_report  # noqa: E402


def main():
    W, H, Q, n = (int(v) for v in sys.argv[1:5])
    sigma = float(sys.argv[5])
    G, Y = synth.batch(n, W, H, Q=Q, seed0=7000 + W + n)
    out = flr.denoise(G.cuda(), Y.cuda(), sigma=sigma)
    torch.cuda.synchronize()
    names = flr.last_launch_names()
    R = flr.effective_radius(block=8, sigma=sigma)
    ref = oracle.denoise(G.numpy(), Y.numpy(), D=8, sigma=sigma, R=R)
    rep = parity_report(out.cpu().numpy(), ref)
    print(json.dumps({"names": names, "violations": int(rep["violations"]), "max_ratio": float(rep["max_ratio"])}))


if __name__ == "__main__":
    main()

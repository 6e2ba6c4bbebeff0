"""Cost of strip sharding on one B200: a frame denoised whole vs cut into
P block-row strips with the (R + 1)-block halo, each strip denoised by its own C-ABI call.

Strip inputs are sliced (halo included) and made resident before timing, as each rank of a
P-GPU strip run would hold them after its halo exchange; the timed region covers only the
denoise calls.  Reported per strip count: the summed strip time (the whole frame's work
done strip by strip, i.e. the halo recomputation overhead) and the largest single strip
(what one of P ranks would spend on compute).  CUDA events on the launching stream.

    python tools/strips_overhead.py [--W 3840 --H 2160 --sigma 20 --reps 50]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_11625_b200 as flr  # noqa: E402
from paper_2410_11625_b200 import strips, synth  # noqa: E402


def _time(fn, reps):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1000.0 / reps  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--W", type=int, default=3840)
    ap.add_argument("--H", type=int, default=2160)
    ap.add_argument("--Q", type=int, default=8)
    ap.add_argument("--sigma", type=float, default=20.0)
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()
    D = 8
    G, Y = synth.frame(a.W, a.H, Q=a.Q, seed=1002, device="cuda")
    g, y = G.unsqueeze(0).contiguous(), Y.unsqueeze(0).contiguous()
    R = flr.effective_radius(block=D, sigma=a.sigma)
    out = torch.empty_like(y)
    full_us = _time(lambda: flr.denoise(g, y, block=D, sigma=a.sigma, out=out), a.reps)
    rows = [{"parts": 1, "sum_us": full_us, "max_strip_us": full_us, "rows_computed": a.H}]
    for P in (2, 4, 8):
        plan = strips.strip_plan(a.H, D, R, P)
        per = []
        for (lo, hi, ilo, ihi) in plan:
            gs, ys = g[..., ilo:ihi, :].contiguous(), y[..., ilo:ihi, :].contiguous()
            os_ = torch.empty_like(ys)
            per.append(_time(lambda: flr.denoise(gs, ys, block=D, sigma=a.sigma, out=os_), a.reps))
        rows.append({"parts": P, "sum_us": sum(per), "max_strip_us": max(per),
                     "rows_computed": sum(p[3] - p[2] for p in plan)})
    print(json.dumps({"workload": f"{a.W}x{a.H} Q={a.Q} sigma={a.sigma} R={R} D={D}",
                      "halo_rows_each_side": strips.halo_blocks(R) * D, "results": rows}))


if __name__ == "__main__":
    main()

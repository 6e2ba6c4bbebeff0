"""Tikhonov eps=1e-6 on the C2 shape: violations and where they are."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import oracle, paper_2410_11625_b200 as flr
from paper_2410_11625_b200 import synth
from tests.parity import parity_report
G, Y = synth.frame(1920, 1080, Q=8, seed=1200 + 1920 + 8)
for eps in (1e-6, 1e-5):
    out = flr.denoise(G[None].cuda(), Y[None].cuda(), eps_add=eps, solver=flr.SOLVER_TIKHONOV)
    torch.cuda.synchronize()
    names = flr.last_launch_names()
    m = flr.fit(G[None].cuda(), Y[None].cuda(), eps_add=eps, solver=flr.SOLVER_TIKHONOV)
    ref = oracle.denoise_tikhonov(G.numpy(), Y.numpy(), D=8, sigma=10.0, R=3, eps=eps)
    rep = parity_report(out.cpu().numpy(), ref)
    A = oracle.fit_tikhonov(G.numpy(), Y.numpy(), D=8, sigma=10.0, R=3, eps=eps)
    mg = m.cpu().numpy().astype(np.float64)
    via = oracle.apply(mg, G.numpy(), 8)
    rep2 = parity_report(via, ref)
    print(eps, names, "denoise:", rep, "\n  gpu fit -> oracle apply:", rep2, "\n  max |slope| ora", np.abs(A[..., 1:, :]).max(),
          "model relerr", np.abs(mg - A).max() / np.abs(A).max(), flush=True)

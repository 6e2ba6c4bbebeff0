import sys; sys.path.insert(0, '.')
import torch, oracle, paper_2410_11625_b200 as flr
from paper_2410_11625_b200 import synth
from tests.parity import parity_report
W, H, Q, block, sigma, eps = [float(v) if "." in v or "e" in v else int(v) for v in sys.argv[1:7]]
G, Y = synth.frame(W, H, Q=Q, seed=1200 + W + Q)
try:
    out = flr.denoise(G[None].cuda(), Y[None].cuda(), block=block, sigma=sigma, eps_add=eps, solver=flr.SOLVER_TIKHONOV)
    torch.cuda.synchronize()
    print(flr.last_launch_names())
    R = flr.effective_radius(block=block, sigma=sigma)
    ref = oracle.denoise_tikhonov(G.numpy(), Y.numpy(), D=block, sigma=sigma, R=R, eps=eps)
    print(parity_report(out.cpu().numpy(), ref))
except Exception as e:
    print("EXC", e)

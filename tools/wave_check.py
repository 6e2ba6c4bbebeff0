"""Quick GPU check of the wave schedule against the staged kernels and the oracle."""
import sys, time
sys.path.insert(0, '.')
import torch
import oracle
import paper_2410_11625_b200 as flr
from paper_2410_11625_b200 import synth
from tests.parity import parity_report

cases = [(1920, 1080, 8, 1, 10.0), (640, 360, 8, 3, 10.0), (1000, 520, 8, 1, 20.0), (264, 136, 8, 2, 12.0),
         (1032, 264, 8, 2, 10.0), (3840, 2160, 8, 1, 20.0)]
for W, H, Q, n, sigma in cases:
    G, Y = synth.batch(n, W, H, Q=Q, seed0=9000 + W)
    g, y = G.cuda(), Y.cuda()
    a = flr.denoise(g, y, sigma=sigma)
    torch.cuda.synchronize()
    na = flr.last_launch_names()
    b = flr.denoise(g, y, sigma=sigma, variant=flr.VARIANT_STAGED)
    torch.cuda.synchronize()
    d = (a - b).abs().max().item()
    msg = f"{W}x{H} n={n} s={sigma}: {na} max|wave-staged|={d:.3g}"
    if W * H <= 2100000:
        R = flr.effective_radius(block=8, sigma=sigma)
        ref = oracle.denoise(G[:1].numpy(), Y[:1].numpy(), D=8, sigma=sigma, R=R)
        rep = parity_report(a[:1].cpu().numpy(), ref)
        msg += f" parity max_ratio={rep['max_ratio']:.3g} viol={rep['violations']}"
    print(msg, flush=True)
# determinism
G, Y = synth.batch(1, 1920, 1080, Q=8, seed0=1)
g, y = G.cuda(), Y.cuda()
outs = [flr.denoise(g, y).clone() for _ in range(5)]
torch.cuda.synchronize()
print("deterministic:", all(torch.equal(outs[0], o) for o in outs[1:]))

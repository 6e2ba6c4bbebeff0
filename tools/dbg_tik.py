import sys, torch, numpy as np
sys.path.insert(0, '.')
import oracle, paper_2410_11625_b200 as flr
from paper_2410_11625_b200 import synth
from tests.parity import parity_report
for (W,H,Q,D,sig,solver) in [(37,23,3,2,5.0,0),(37,23,3,2,5.0,1),(40,24,3,2,5.0,1),(40,24,3,4,5.0,1),(40,24,4,2,5.0,1),(37,23,4,2,5.0,1),(40,24,2,2,5.0,1),(40,24,3,8,10.0,1)]:
    G,Y = synth.frame(W,H,Q=Q,seed=1240)
    out = flr.denoise(G[None].cuda(), Y[None].cuda(), block=D, sigma=sig, eps_add=1e-5, solver=solver)
    names = flr.last_launch_names()
    torch.cuda.synchronize()
    R = flr.effective_radius(block=D, sigma=sig)
    if solver: ref = oracle.denoise_tikhonov(G.numpy(), Y.numpy(), D=D, sigma=sig, R=R, eps=1e-5)
    else: ref = oracle.denoise(G.numpy(), Y.numpy(), D=D, sigma=sig, R=R, eps_add=1e-5)
    rep = parity_report(out.cpu().numpy(), ref)
    print(W,H,Q,D,solver, names, rep['max_ratio'], rep['violations'])
    if solver and rep['violations']:
        A = flr.fit(G[None].cuda(), Y[None].cuda(), block=D, sigma=sig, eps_add=1e-5, solver=1).cpu().numpy()[0]
        Ar = oracle.fit_tikhonov(G.numpy(), Y.numpy(), D=D, sigma=sig, R=R, eps=1e-5)[0]
        print('  model diff max', np.abs(A-Ar).max(), 'at', np.unravel_index(np.abs(A-Ar).argmax(), A.shape))
        print('  gpu', A[0,0].ravel()[:8]); print('  ref', Ar[0,0].ravel()[:8])

"""Rolling hand-off check: results equal the variant without hand-off (workspace not initialised ->
grid-wide waits), back-to-back calls, and timing of both."""
import sys
sys.path.insert(0, '.')
import torch
import oracle
import paper_2410_11625_b200 as flr
from paper_2410_11625_b200 import synth
from tests.parity import parity_report

for W, H, n, sigma in [(1920, 1080, 1, 10.0), (640, 360, 3, 10.0), (1000, 520, 1, 20.0), (3840, 2160, 1, 20.0)]:
    G, Y = synth.batch(n, W, H, Q=8, seed0=9100 + W)
    g, y = G.cuda(), Y.cuda()
    nb = flr.workspace_size(n, 8, W, H, sigma=sigma)
    ws_plain = torch.zeros(nb, dtype=torch.uint8, device="cuda")  # no magic: grid-wide waits
    a = flr.denoise(g, y, sigma=sigma, workspace=ws_plain)
    b = flr.denoise(g, y, sigma=sigma)  # initialised workspace: rolling
    torch.cuda.synchronize()
    msg = f"{W}x{H} n={n}: {flr.last_launch_names()} equal={torch.equal(a, b)}"
    if W * H <= 2100000:
        R = flr.effective_radius(block=8, sigma=sigma)
        ref = oracle.denoise(G[:1].numpy(), Y[:1].numpy(), D=8, sigma=sigma, R=R)
        msg += f" parity {parity_report(b[:1].cpu().numpy(), ref)['max_ratio']:.3g}"
    print(msg, flush=True)
# back to back + timing
G, Y = synth.batch(4, 1920, 1080, Q=8, seed0=1)
fr = [(G[i:i + 1].cuda(), Y[i:i + 1].cuda()) for i in range(4)]
for label, init in (("grid-wide waits", False), ("rolling", True)):
    for flags in (0, flr.FLAG_INPUTS_READY):
        den = flr.Denoiser(1, 8, 1920, 1080, device="cuda", flags=flags)
        if not init:
            den.workspace.zero_()
        ref = [flr.denoise(*fr[i]).clone() for i in range(4)]
        outs = [torch.empty_like(ref[0]) for _ in range(8)]
        for i in range(30):
            den(*fr[i % 4], out=outs[i % 8])
        torch.cuda.synchronize()
        for i in range(8):
            den(*fr[i % 4], out=outs[i])
        torch.cuda.synchronize()
        ok = all(torch.equal(outs[i], ref[i % 4]) for i in range(8))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(400):
            den(*fr[i % 4], out=outs[i % 8])
        e1.record()
        torch.cuda.synchronize()
        print(f"{label:16s} flags={flags}: {e0.elapsed_time(e1) * 1e3 / 400:.2f} us per call (eager), results ok {ok}",
              flush=True)

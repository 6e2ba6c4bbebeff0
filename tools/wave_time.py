"""Time back-to-back wave calls (1080p Q=8) with CUDA events."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2410_11625_b200 as flr
from paper_2410_11625_b200 import synth
G, Y = synth.batch(4, 1920, 1080, Q=8, seed0=1)
fr = [(G[i:i + 1].cuda(), Y[i:i + 1].cuda()) for i in range(4)]
ws = torch.zeros(flr.workspace_size(1, 8, 1920, 1080), dtype=torch.uint8, device="cuda")
out = torch.empty(1, 3, 1080, 1920, device="cuda")
for i in range(20):
    flr.denoise(*fr[i % 4], workspace=ws, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(200):
    flr.denoise(*fr[i % 4], workspace=ws, out=out)
e1.record()
torch.cuda.synchronize()
print(sys.argv[1] if len(sys.argv) > 1 else "", "us per call:", e0.elapsed_time(e1) * 1e3 / 200, flr.last_launch_names())

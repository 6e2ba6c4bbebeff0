"""One C2 step (1080p Q=8 fit + apply) inside a cudaProfilerStart/Stop range, for ncu range
replay: whole-step DRAM bytes (dram__bytes_read/write.sum) against the 56 B/px minimum.

    ncu --replay-mode app-range --metrics \
        dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum \
        python tools/step_traffic.py [staged|fused]
"""
import sys
sys.path.insert(0, '.')
import torch
import paper_2410_11625_b200 as flr
from paper_2410_11625_b200 import synth

variant = {"staged": flr.VARIANT_STAGED, "fused": flr.VARIANT_FUSED}[sys.argv[1] if len(sys.argv) > 1 else "staged"]
G, Y = synth.batch(1, 1920, 1080, Q=8, seed0=1000)
g, y = G.cuda(), Y.cuda()
den = flr.Denoiser(1, 8, 1920, 1080, device="cuda", variant=variant)
for _ in range(5):
    den(g, y)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
den(g, y)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("launches:", flr.last_launch_names())

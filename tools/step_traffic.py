"""C2 steps (1080p Q=8 fit + apply) inside a cudaProfilerStart/Stop range, for ncu range
replay: whole-step DRAM bytes (dram__bytes_read/write.sum) against the 56 B/px minimum.

    ncu --replay-mode app-range [--cache-control none] --metrics \
        dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum \
        python tools/step_traffic.py [staged|fused] [calls]

calls > 1: that many back-to-back calls over 4 rotating frames (as bench.py's pool), so the
range holds the steady state -- each call's reads plus the write-back of earlier calls'
output and moment lines that the stream evicts; divide by calls.
"""
import sys
sys.path.insert(0, '.')
import torch
import paper_2410_11625_b200 as flr
from paper_2410_11625_b200 import synth

variant = {"staged": flr.VARIANT_STAGED, "fused": flr.VARIANT_FUSED}[sys.argv[1] if len(sys.argv) > 1 else "staged"]
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 1
frames = [tuple(t.cuda() for t in synth.batch(1, 1920, 1080, Q=8, seed0=1000 + 10 * k)) for k in range(4)]
g, y = frames[0]
den = flr.Denoiser(1, 8, 1920, 1080, device="cuda", variant=variant, flags=flr.FLAG_INPUTS_READY)
for _ in range(5):
    den(g, y)
torch.cuda.synchronize()
for k in range(4):
    den(*frames[k])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for k in range(calls):
    den(*frames[k % 4])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("launches:", flr.last_launch_names())

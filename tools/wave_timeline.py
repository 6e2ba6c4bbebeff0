"""Task timeline of the wave schedule (library built with FLR_DEFS=-DFLR_WAVE_TRACE)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2410_11625_b200 as flr
from paper_2410_11625_b200 import synth

W, H, Q, n, D = 1920, 1080, 8, 1, 8
Bx, By = -(-W // D), -(-H // D)
Bxp = (Bx + 1) & ~1
KM = 1 + Q + Q * (Q + 1) // 2 + 3 + 3 * Q
MS = ((3 * (Q + 1) + 3) // 4) * 4
a256 = lambda x: (x + 255) & ~255
off = a256(n * Bx * By * (KM + Q) * 4) + 2 * a256(n * Bxp * By * KM * 8) + a256(n * Bx * By * MS * 4)
ntr = -(-By // 8)
nfl0 = 4 + n * (By + 3 * ntr + 2)
G, Y = synth.batch(n, W, H, Q=Q, seed0=1)
g, y = G.cuda(), Y.cuda()
ws = torch.zeros(flr.workspace_size(n, Q, W, H), dtype=torch.uint8, device="cuda")
for _ in range(3):
    flr.denoise(g, y, workspace=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); flr.denoise(g, y, workspace=ws); e1.record(); torch.cuda.synchronize()
print("call us", e0.elapsed_time(e1) * 1e3)
allraw = ws[off + 4 * nfl0: off + 4 * nfl0 + 160 * 96 * 16].view(torch.int64).cpu().numpy().reshape(160, 96, 2)
raw = allraw[:148]
pre_fit = [0] * By
pre_k2 = [0] * 17
recs = []
for b in range(148):
    for i in range(96):
        k, t = int(raw[b, i, 0]), int(raw[b, i, 1])
        if k == 0 and t == 0:
            continue
        ty, ix = k >> 32, k & 0xffffffff
        t1, dt = t >> 16, t & 0xffff
        recs.append((b, i, ty, ix, t1, dt))
t0 = min(r[4] for r in recs)
names = {0: "FIT", 1: "APP", 2: "K2", 3: "DONE", 4: "NONE"}
import collections
per = collections.defaultdict(list)
for b, i, ty, ix, t1, dt in recs:
    per[b].append((t1 - t0, ty, ix, dt))
print("fit prefix advance us:", [round((t - t0) / 1e3, 1) if t else None for t in pre_fit][::8])
print("k2 prefix advance us:", [round((t - t0) / 1e3, 1) if t else None for t in pre_k2])
for b in (0, 1, 50, 100, 147):
    print(b, " ".join(f"{names[ty]}{ix}@{t/1e3:.1f}(w{dt/1e3:.1f})" for t, ty, ix, dt in sorted(per[b])[:40]))
ends = [max(t for t, ty, ix, dt in v) for v in per.values()]
print("last claim (DONE) per CTA us: min %.1f max %.1f" % (min(ends) / 1e3, max(ends) / 1e3))
for ty in range(3):
    ts = sorted(t1 - t0 for b, i, tt, ix, t1, dt in recs if tt == ty)
    if ts:
        print(names[ty], "claims", len(ts), "first %.1f last %.1f us" % (ts[0] / 1e3, ts[-1] / 1e3))
waits = [dt for b, i, tt, ix, t1, dt in recs]
print("claim wait us: mean %.2f max %.2f" % (np.mean(waits) / 1e3, np.max(waits) / 1e3))

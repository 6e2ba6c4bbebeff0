"""Per-SASS-region stall profile of one kernel in an .ncu-rep (source page, SASS view).

usage: python tools/ncu_src.py REP KERNEL_REGEX [window]
Prints the instructions with the most stall samples plus a coarse histogram of samples
over the code (window = instructions per bucket)."""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
win = int(sys.argv[3]) if len(sys.argv) > 3 else 64
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre, "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
si, ni, ei = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
body = []
for r in rows[2:]:
    if len(r) <= ei or r[0] == "Kernel Name":
        if body:
            break  # first kernel only
        continue
    try:
        float(r[ni] or 0)
    except ValueError:
        continue
    body.append(r)
tot = sum(float(r[ni] or 0) for r in body)
print(f"{len(body)} SASS, {tot:.0f} samples")
for b in range(0, len(body), win):
    chunk = body[b:b + win]
    s = sum(float(r[ni] or 0) for r in chunk)
    ex = sum(float(r[ei] or 0) for r in chunk)
    ops = {}
    for r in chunk:
        op = r[si].split()[0] if r[si].split() else ""
        if op.startswith("@"):
            op = r[si].split()[1]
        op = op.split(".")[0]
        ops[op] = ops.get(op, 0) + 1
    top = sorted(ops.items(), key=lambda x: -x[1])[:4]
    print(f"[{b:5d}] {100*s/tot:5.1f}% samples  exec {ex:10.0f}  {top}")
print("top instructions:")
for r in sorted(body, key=lambda r: -float(r[ni] or 0))[:25]:
    print(f"{float(r[ni]):6.0f} {float(r[ei]):9.0f}  {r[si].strip()[:70]}")

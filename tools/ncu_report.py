"""Quick text report of an ncu .ncu-rep: key metrics, stall reasons, hot SASS by opcode."""
import csv
import io
import re
import subprocess
import sys
from collections import Counter


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main(rep, kernel_regex="."):
    det = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    hdr = det[0]
    ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    want = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "Executed Ipc Active",
            "Issue Slots Busy", "No Eligible", "Warp Cycles Per Issued Instruction", "Achieved Occupancy",
            "Registers Per Thread", "Compute (SM) Throughput", "Dynamic Shared Memory Per Block"]
    seen = set()
    for r in det[1:]:
        if r[mi] in want and re.search(kernel_regex, r[ki]) and (r[ki], r[mi]) not in seen:
            seen.add((r[ki], r[mi]))
            print(f"{r[ki][:40]:40s} {r[mi]:36s} {r[vi]} {r[ui]}")
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    h = raw[0]
    for r in raw[2:]:
        if not re.search(kernel_regex, r[h.index("Kernel Name")]):
            continue
        out = []
        for i, c in enumerate(h):
            if c.startswith("smsp__average_warps_issue_stalled_") and c.endswith("_per_issue_active.ratio"):
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                if v > 0.05:
                    out.append((round(v, 2), c[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        dram = [r[i] for i, c in enumerate(h) if c in ("dram__bytes_read.sum", "dram__bytes_write.sum")]
        print("stalls:", sorted(out, reverse=True)[:10], "dram rd/wr:", dram)
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    if len(src) > 2:
        hs = src[1]
        ii, si, ss = hs.index("Instructions Executed"), hs.index("Source"), hs.index("Warp Stall Sampling (All Samples)")
        cnt, st = Counter(), Counter()
        for r in src[2:]:
            if len(r) <= ii:
                continue
            op = re.sub(r"^@!?U?P\w+\s+", "", r[si].strip()).split()[0].split(".")[0] if r[si].strip() else "?"
            try:
                cnt[op] += int(r[ii])
                st[op] += int(r[ss])
            except ValueError:
                pass
        tot, tots = sum(cnt.values()), max(1, sum(st.values()))
        print(f"warp-instructions {tot}; stall samples {tots}")
        for op, n in cnt.most_common(16):
            print(f"   {op:10s} {n:10d} {100*n/tot:5.1f}%   stall {100*st[op]/tots:5.1f}%")


if __name__ == "__main__":
    main(*sys.argv[1:])

"""Shared-memory wavefronts / bank conflicts / fp64 pipe of one kernel in an .ncu-rep, plus the
source lines with the most excess shared wavefronts.  usage: python tools/ncu_k2.py REP"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
d = dict(zip(h, v))
for k in ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
          "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__m_xbar2l1tex_read_bytes.sum", "launch__registers_per_thread"]:
    print(f"{k:70s} {d.get(k)}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hi = next(i for i, r in enumerate(rows) if "L1 Wavefronts Shared Excessive" in r)
h = rows[hi]
ix = {k: h.index(k) for k in ["Source", "L1 Wavefronts Shared Excessive", "L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal"]}
out = []
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    try:
        ex, wf = float(r[ix["L1 Wavefronts Shared Excessive"]] or 0), float(r[ix["L1 Wavefronts Shared"]] or 0)
    except ValueError:
        continue
    if wf > 0 and r[ix["Source"]].strip():
        out.append((ex, wf, float(r[ix["L1 Wavefronts Shared Ideal"]] or 0), r[0], r[ix["Source"]].strip()[:80]))
out.sort(reverse=True)
print("excess  wavefronts  ideal  line  source")
for o in out[:12]:
    print(f"{o[0]:8.0f} {o[1]:10.0f} {o[2]:8.0f} {o[3]:>5s}  {o[4]}")

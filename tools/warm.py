"""Average per-kernel duration / DRAM bytes from an ncu --csv launch list (last 5 launches each)."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    d = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[1:]:
        d[r[ki].split("(")[0]][r[mi]].append(float(r[vi].replace(",", "")))
    print(path)
    for k, m in d.items():
        t = m["gpu__time_duration.sum"][-5:]
        rd = m["dram__bytes_read.sum"][-5:]
        wr = m["dram__bytes_write.sum"][-5:]
        print(f"  {k[:44]:44s} {sum(t)/len(t)/1e3:7.2f} us  rd {sum(rd)/len(rd)/1e6:7.2f} MB  wr {sum(wr)/len(wr)/1e6:6.2f} MB")

"""Summarise an ncu --csv launch list: one line per launch (name, time, DRAM bytes, L2 hit, SM%)."""
import csv
import sys
from collections import OrderedDict


def load(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    d = OrderedDict()
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        key = (int(r[0]), r[ki].split("(")[0].replace("void ", ""))
        d.setdefault(key, {})[r[mi]] = float(r[vi].replace(",", ""))
    return d


if __name__ == "__main__":
    d = load(sys.argv[1])
    for (i, name), m in d.items():
        rd, wr = m.get("dram__bytes_read.sum", 0), m.get("dram__bytes_write.sum", 0)
        t = m.get("gpu__time_duration.sum", 0)
        print(f"{i:3d} {name[:46]:46s} {t/1e3:8.1f} us  rd {rd/1e6:7.1f} MB  wr {wr/1e6:6.1f} MB  "
              f"{(rd+wr)/max(t,1):7.1f} GB/s  L2hit {m.get('lts__t_sector_hit_rate.pct', 0):5.1f}%  "
              f"SM {m.get('sm__throughput.avg.pct_of_peak_sustained_elapsed', 0):5.1f}%")

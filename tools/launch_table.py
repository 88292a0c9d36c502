"""Print per-launch durations from an ncu --metrics gpu__time_duration.sum --csv log.
usage: python tools/launch_table.py gpurun_out/launches.csv [--sum]"""
import collections
import re
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, gi, bi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size"), h.index("Block Size")
agg = collections.OrderedDict()
for r in rows[1:]:
    name = re.sub(r"<[^<>]*>$", "", re.sub(r"^void\s+", "", r[ki].replace("(anonymous namespace)", "<unnamed>").split("(")[0]).strip()).split("::")[-1]
    v = float(r[vi].replace(",", ""))
    if "--sum" in sys.argv:
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    else:
        print(f"{name:28s} grid {r[gi]:>16s} block {r[bi]:>10s} {v/1e3:10.1f} us")
for k, (n, t) in agg.items():
    print(f"{k:28s} launches {n:6d} total {t/1e6:10.3f} ms mean {t/n/1e3:9.1f} us")

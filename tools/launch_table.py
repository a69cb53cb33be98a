"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-launch sequence of the
last sweep and per-kernel totals.  usage: python tools/launch_table.py launches.csv [launches_per_sweep]"""
import csv
import re
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
seq = []
for r in rows[1:]:
    name = re.sub(r"\(.*", "", r[ik]).replace("void ", "").replace("cpqr::", "")
    v = float(r[iv].replace(",", ""))
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[r[iu]]
    seq.append((name, v * scale))
per = int(sys.argv[2]) if len(sys.argv) > 2 else 0
if per:
    print("last sweep, in launch order (us):")
    for n, v in seq[-per:]:
        print(f"  {v:9.1f}  {n}")
tot = OrderedDict()
for n, v in seq:
    t = tot.setdefault(n, [0.0, 0])
    t[0] += v
    t[1] += 1
T = sum(v for v, _ in tot.values())
print(f"total {T/1e3:.3f} ms over {len(seq)} launches")
for n, (v, c) in sorted(tot.items(), key=lambda x: -x[1][0]):
    print(f"  {100*v/T:5.1f}%  {v/1e3:8.3f} ms  {c:4d}  avg {v/c:8.1f} us  {n}")

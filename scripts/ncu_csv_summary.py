"""Summarise an `ncu --csv --metrics ...` log: one line per kernel launch
(duration, tensor-pipe %, issue %), optionally only the last N launches."""
import collections
import csv
import sys

path = sys.argv[1]
last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = list(csv.reader(open(path)))
hdr, data = None, collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        data.setdefault((d["ID"], d["Kernel Name"].split("(")[0]), {})[d["Metric Name"]] = d["Metric Value"]
items = list(data.items())[-last:] if last else list(data.items())
for (i, k), m in items:
    print(f"{i:>4} {k:<48} {float(m.get('gpu__time_duration.sum', 0)) / 1e3:8.2f} us  "
          f"tensor {float(m.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', 0)):5.1f}%  "
          f"issue {float(m.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0)):5.1f}%")

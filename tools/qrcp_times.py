"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` log of tools/bench_qrcp_small.py:
median kernel time per (kernel, grid)."""
import collections
import csv
import sys

for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10 and r[0].isdigit()]
    d = collections.OrderedDict()
    for r in rows:
        d.setdefault((r[4][:44], r[7], r[8]), []).append(float(r[-1]) / 1e3)
    print(f)
    for k, v in d.items():
        v = sorted(v)
        print("  ", k, len(v), "median us %.1f" % v[len(v) // 2])

"""Spans of a PRRP_TRACE file that start inside [t0, t1) ms, in start order.
usage: trace_window.py trace.csv t0 t1"""
import csv
import sys

rows = [(r["class"], int(r["stream"]), float(r["start_ms"]), float(r["end_ms"])) for r in csv.DictReader(open(sys.argv[1]))]
t0, t1 = float(sys.argv[2]), float(sys.argv[3])
for c, s, a, b in sorted(rows, key=lambda r: r[2]):
    if t0 <= a < t1:
        print(f"{a:9.3f} {b - a:7.3f} {c:10s} {s}")

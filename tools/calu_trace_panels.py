"""Per-panel view of a PRRP_TRACE span file of one CALU_PRRP run: for every
panel interval (between consecutive tournament starts) the time, the Schur
busy time (union of schur spans) and the critical tournament chain.
usage: calu_trace_panels.py trace.csv [npanels_to_print]"""
import csv
import sys


def union(iv):
    iv = sorted(iv)
    tot, cur = 0.0, None
    for a, b in iv:
        if cur is None or a > cur[1]:
            if cur:
                tot += cur[1] - cur[0]
            cur = [a, b]
        else:
            cur[1] = max(cur[1], b)
    if cur:
        tot += cur[1] - cur[0]
    return tot


rows = [(r["class"], int(r["stream"]), float(r["start_ms"]), float(r["end_ms"])) for r in csv.DictReader(open(sys.argv[1]))]
end = max(r[3] for r in rows)
schur = [(a, b) for c, s, a, b in rows if c == "schur"]
print(f"total {end:.1f} ms; schur busy (union) {union(schur):.1f} ms; panel-class busy (union) "
      f"{union([(a, b) for c, s, a, b in rows if c == 'panel']):.1f} ms")
# idle time: no span at all
allv = [(a, b) for c, s, a, b in rows]
print(f"any-kernel busy {union(allv):.1f} ms")
# windows of 50 ms: schur busy fraction
w = 50.0
t = 0.0
out = []
while t < end:
    sel = [(max(a, t), min(b, t + w)) for a, b in schur if b > t and a < t + w]
    pan = [(max(a, t), min(b, t + w)) for c, s, a, b in rows if c != "schur" and b > t and a < t + w]
    out.append(f"{t:7.0f}-{t + w:5.0f} ms: schur {100 * union(sel) / w:3.0f}%  non-schur {100 * union(pan) / w:3.0f}%")
    t += w
print("\n".join(out))

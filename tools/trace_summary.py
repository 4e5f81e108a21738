"""Summarise a PRRP_TRACE span file: per-stream busy time, idle gaps, and a
text Gantt chart of a window.  usage: trace_summary.py trace.csv [t0_ms t1_ms]"""
import collections
import csv
import sys


def main():
    rows = list(csv.DictReader(open(sys.argv[1])))
    spans = [(r["class"], int(r["stream"]), float(r["start_ms"]), float(r["end_ms"])) for r in rows]
    end = max(s[3] for s in spans)
    print(f"total {end:.2f} ms")
    by_stream = collections.defaultdict(list)
    for c, st, a, b in spans:
        by_stream[st].append((a, b, c))
    for st, lst in sorted(by_stream.items()):
        lst.sort()
        busy = collections.Counter()
        for a, b, c in lst:
            busy[c] += b - a
        tot = sum(busy.values())
        print(f"stream {st}: busy {tot:.2f} ms ({100 * tot / end:.0f}%)  " +
              "  ".join(f"{c} {v:.2f}" for c, v in busy.most_common()))
    if len(sys.argv) > 3:
        t0, t1 = float(sys.argv[2]), float(sys.argv[3])
        width = 120
        sym = {"panel": "Q", "trsm": "t", "finalize": "f", "permute": "p", "schur": "S", "compose": "c",
               "blockrow": "B", "gepp": "G", "other": "."}
        for st, lst in sorted(by_stream.items()):
            line = [" "] * width
            for a, b, c in lst:
                if b < t0 or a > t1:
                    continue
                i0 = max(0, int((a - t0) / (t1 - t0) * width))
                i1 = min(width, max(i0 + 1, int((b - t0) / (t1 - t0) * width)))
                for i in range(i0, i1):
                    line[i] = sym.get(c, "?")
            print(f"s{st} |{''.join(line)}|")


if __name__ == "__main__":
    main()

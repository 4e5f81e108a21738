"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel count, serialized time and share.  usage: ncu_launch_summary.py launches.csv [out.json]"""
import collections
import csv
import json
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}


def load(path):
    with open(path) as f:
        lines = [l for l in f if not l.startswith("==")]
    rows = []
    for x in csv.DictReader(lines):
        if x.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((int(x["ID"]), x["Kernel Name"].split("(")[0].replace("<unnamed>::", ""),
                         float(x["Metric Value"].replace(",", "")) * SCALE[x["Metric Unit"]]))
    return rows


def main():
    rows = load(sys.argv[1])
    agg = collections.defaultdict(lambda: [0, 0.0])
    for _, k, ms in rows:
        agg[k][0] += 1
        agg[k][1] += ms
    tot = sum(v[1] for v in agg.values())
    out = {"launches": len(rows), "serialized_ms": tot,
           "kernels": [{"kernel": k, "launches": v[0], "ms": round(v[1], 3), "share": round(v[1] / tot, 4)}
                       for k, v in sorted(agg.items(), key=lambda x: -x[1][1])]}
    print(f"{len(rows)} launches, {tot:.1f} ms serialized (cold-cache, one at a time)")
    for e in out["kernels"][:25]:
        print(f"{e['kernel'][:44]:44s} {e['launches']:6d} {e['ms']:9.2f} ms {100 * e['share']:5.1f}%")
    if len(sys.argv) > 2:
        json.dump(out, open(sys.argv[2], "w"), indent=1)


if __name__ == "__main__":
    main()

"""Turn ncu outputs (gpurun_out/) into the committed summaries under profiles/.

  launches CSV (--metrics gpu__time_duration.sum)  -> per-kernel share table
  --set full report of schur_dmma_kernel           -> dram bytes per launch vs algorithmic bytes
  --set full report of panel_qrcp1_kernel          -> headline metrics

usage: python tools/profile_summary.py <tag>   (reads gpurun_out/{launches,schur,qrcp1}_<tag>*)
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    vi, ki = h.index("Metric Value"), h.index("Kernel Name")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        agg[r[ki].split("(")[0].replace("void ", "")].append(float(r[vi]) / 1e3)
    tot = sum(sum(v) for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out.append({"kernel": k, "launches": len(v), "total_us": round(sum(v), 1), "mean_us": round(sum(v) / len(v), 2),
                    "share": round(sum(v) / tot, 4)})
    return {"source": os.path.basename(path), "total_us_serialised": round(tot, 1), "kernels": out}


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}


def raw(rep):
    """Rows of the raw page with every value converted to base units (bytes, microseconds)."""
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {}
        for k, u, v in zip(h, units, r):
            try:
                d[k] = float(v.replace(",", "")) * SCALE.get(u, 1.0)
            except ValueError:
                d[k] = v
        out.append(d)
    return out


def num(d, k):
    v = d.get(k)
    return v if isinstance(v, float) else None


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum"]


def main():
    tag = sys.argv[1]
    g = os.path.join(ROOT, "gpurun_out")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    lp = os.path.join(g, f"launches_{tag}.csv")
    if os.path.exists(lp):
        s = launches(lp)
        json.dump(s, open(os.path.join(ROOT, "profiles", f"ncu_launches_{tag}.json"), "w"), indent=1)
        for k in s["kernels"][:12]:
            print(f"{k['kernel']:32s} {k['launches']:5d} {k['total_us']:10.1f} us {100 * k['share']:5.1f}%")
    sp = os.path.join(g, f"schur_{tag}.ncu-rep")
    if os.path.exists(sp):
        launches_ = []
        for d in raw(sp):
            e = {k: num(d, k) for k in KEYS if k in d}
            e["kernel"] = d.get("Kernel Name", "")[:60]
            launches_.append(e)
        # the largest launch (the first panel's wide update) is the roofline reference
        big = max(launches_, key=lambda e: e.get("gpu__time_duration.sum") or 0)
        summ = {"report": os.path.basename(sp), "launches": launches_,
                "dram_bytes_per_launch": (big["dram__bytes_read.sum"] or 0) + (big["dram__bytes_write.sum"] or 0),
                "reference_launch": "largest captured launch (panel 0 trailing update, M=8128, N=8064, K=64)",
                "algorithmic_bytes_reference_launch": 8 * (2 * 8128 * 8064 + 8128 * 64 + 64 * 8064)}
        json.dump(summ, open(os.path.join(ROOT, "profiles", f"ncu_schur_summary.json"), "w"), indent=1)
        json.dump(summ, open(os.path.join(ROOT, "profiles", f"ncu_schur_{tag}.json"), "w"), indent=1)
        print("schur dram bytes/launch", summ["dram_bytes_per_launch"], "algorithmic", summ["algorithmic_bytes_reference_launch"])
        for e in launches_:
            print({k: e[k] for k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                      "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active") if k in e})
    qp = os.path.join(g, f"qrcp1_{tag}.ncu-rep")
    if os.path.exists(qp):
        ds = [{k: num(d, k) for k in KEYS if k in d} for d in raw(qp)]
        json.dump({"report": os.path.basename(qp), "launches": ds}, open(os.path.join(ROOT, "profiles", f"ncu_qrcp1_{tag}.json"), "w"), indent=1)
        print("qrcp1", ds)


if __name__ == "__main__":
    main()

"""Summarise one-kernel `ncu --set full` reports into profiles/*.json.

usage: ncu_report_summary.py <report.ncu-rep> <out.json> [M N K]  (Schur: algorithmic flops/bytes)
       ncu_report_summary.py <report.ncu-rep> <out.json> panel <h> <p>  (panel QRCP: algorithmic bytes)"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warp_latency_issue_stalled_barrier", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            d[k] = vals[i] + (" " + units[i] if units[i] else "")
    def num(k):
        i = hdr.index(k)
        return float(vals[i].replace(",", "")) * SCALE.get(units[i], 1.0)
    t = num("gpu__time_duration.sum")
    dram = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
    s = {"report": rep.split("/")[-1], "metrics": d, "time_s": t, "dram_bytes_per_launch": dram,
         "dram_gbs": dram / t / 1e9}
    if len(sys.argv) >= 6 and sys.argv[3] != "panel":
        M, N, K = map(int, sys.argv[3:6])
        fl = 2.0 * M * N * K
        alg = 8.0 * (2 * M * N + M * K + K * N)
        s.update({"M": M, "N": N, "K": K, "algorithmic_flops": fl, "algorithmic_bytes": alg,
                  "tflops": fl / t / 1e12, "traffic_over_algorithmic": dram / alg,
                  "note": f"dram read+write of one {M}x{N}x{K} launch = {dram / alg:.2f}x the algorithmic bytes "
                          f"8(2MN+MK+KN); {fl / t / 1e12:.1f} TFLOP/s under ncu (cold caches, serialised)"})
    elif len(sys.argv) >= 6:
        h, p = int(sys.argv[4]), int(sys.argv[5])
        alg = 16.0 * h * p
        s.update({"h": h, "p": p, "algorithmic_bytes": alg, "traffic_over_algorithmic": dram / alg,
                  "note": f"panel QRCP h={h} p={p}: algorithmic bytes 16 h p (read the panel, write R); "
                          "latency bound (h dependent pivot steps), the GB/s is far below HBM by construction"})
    json.dump(s, open(out, "w"), indent=1)
    print(json.dumps(s, indent=1))


if __name__ == "__main__":
    main()

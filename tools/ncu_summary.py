"""Key metrics of an `ncu --set full` report as JSON (for profiles/).
usage: ncu_summary.py <report.ncu-rep> <out.json> [note]"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smsp__inst_executed.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3,
         "ns": 1e-3, "us": 1.0, "ms": 1e3}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")]}
        for k in h:
            if k in KEYS or ("stalled" in k and k.endswith("per_issue_active.ratio")):
                i = h.index(k)
                try:
                    v = float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)
                except ValueError:
                    continue
                if "stalled" in k and v < 0.05:
                    continue
                d[k.replace("smsp__average_warps_issue_stalled_", "stall_")] = v
        launches.append(d)
    json.dump({"report": rep.split("/")[-1], "units": "time in us, bytes in bytes", "note": " ".join(sys.argv[3:]),
               "launches": launches}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()

"""From a multi-launch `ncu --set full` report pick the longest launch and summarise it
(time, DRAM bytes, GB/s against a peak).  usage: ncu_pick_max.py rep.ncu-rep out.json [peak_gbs] [note]"""
import csv
import io
import json
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "second": 1.0, "s": 1.0}
rep, out = sys.argv[1], sys.argv[2]
peak = float(sys.argv[3]) if len(sys.argv) > 3 else 6454.6
note = sys.argv[4] if len(sys.argv) > 4 else ""
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h, u = rows[0], rows[1]


def num(r, k):
    i = h.index(k)
    return float(r[i].replace(",", "")) * SCALE.get(u[i], 1.0)


best = max(rows[2:], key=lambda r: num(r, "gpu__time_duration.sum"))
t = num(best, "gpu__time_duration.sum")
dram = num(best, "dram__bytes_read.sum") + num(best, "dram__bytes_write.sum")
l2 = None
for k in ("lts__t_bytes.sum",):
    if k in h:
        l2 = num(best, k)
doc = {"report": rep.split("/")[-1], "kernel": best[h.index("Kernel Name")], "grid": best[h.index("Grid Size")],
       "launches_in_report": len(rows) - 2, "time_s": t, "dram_bytes": dram, "dram_gbs": dram / t / 1e9,
       "hbm_peak_gbs": peak, "frac_of_hbm_peak": dram / t / 1e9 / peak, "l2_bytes": l2, "note": note}
json.dump(doc, open(out, "w"), indent=1)
print(json.dumps(doc, indent=1))

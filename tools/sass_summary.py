"""Per-kernel SASS mnemonic counts of the built library (cuobjdump -sass): the
instructions that prove the hardware paths in use -- DMMA (FP64 tensor core),
UTMALDG (TMA loads), SYNCS (mbarrier), STAS (st.async into cluster shared
memory), CREDUX (warp reductions), UCGABAR (cluster barriers).
usage: sass_summary.py [lib.so] [out.json]"""
import collections
import json
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1208_2451_b200/lib/libprrp_b200.so"
out = sys.argv[2] if len(sys.argv) > 2 else None
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
WATCH = ["DMMA", "UTMALDG", "UTMASTG", "SYNCS", "STAS", "CREDUX", "UCGABAR_ARV", "UCGABAR_WAIT", "DFMA", "DADD",
         "DMUL", "LDS", "STS", "SHFL", "BAR"]
res = collections.OrderedDict()
cur = None
for line in txt.split("\n"):
    m = re.search(r"Function : (\S+)", line)
    if m:
        name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip().split("(")[0]
        cur = res.setdefault(name, collections.Counter())
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_]+)", line)
    if m and cur is not None:
        cur["total"] += 1
        op = m.group(1)
        for w in WATCH:
            if op == w or op.startswith(w + "."):
                cur[w] += 1
summary = {k: dict(v) for k, v in res.items() if v.get("total", 0) > 0}
tot = collections.Counter()
for v in summary.values():
    tot.update(v)
doc = {"library": lib, "totals": dict(tot), "kernels": summary}
if out:
    json.dump(doc, open(out, "w"), indent=1)
hot = ["schur_wsc_kernel", "schur_ws_kernel", "schur_persist_kernel", "schur_dmma_kernel", "panel_lat_kernel<16, 1, 7",
       "panel_qrcp2_kernel", "panel_qrcp1_kernel"]
print("totals", dict(tot))
for k, v in summary.items():
    if any(h in k for h in hot):
        print(k, {w: v[w] for w in ("total", "DMMA", "UTMALDG", "SYNCS", "STAS", "CREDUX", "DFMA") if w in v})

"""Per-phase cycles of one panel2 (h = 128) QRCP launch from a PRRP_PANEL_TL dump
(thread 0 of CTA 0; marks: start, candidate, CTA barrier, cluster wait, pull, apply).
usage: PRRP_PANEL_PROF=1 PRRP_PANEL_TL=<panel> PRRP_PANEL_TL_OUT=f python tools/run_lu.py --b 128; panel2_tl.py f"""
import sys
import numpy as np

tl = np.fromfile(sys.argv[1], dtype=np.int64)[:128 * 8].reshape(128, 8)
steps = int((tl[:, 0] != 0).sum())
tl = tl[:steps, :6].astype(np.float64)
names = ["warp argmax+candidate", "CTA barrier", "cluster exchange", "winner/global+pull", "apply+keys"]
d = np.diff(tl, axis=1)
d[d < 0] = np.nan
print(f"{steps} steps; step mean {np.nanmean(np.diff(tl[:, 0])):.0f} cycles")
print("  ".join(f"{n}={np.nanmean(d[:, i]):.0f}" for i, n in enumerate(names)))
for k in (0, 8, 32, 63, 64, 96, 120):
    if k < steps:
        print(f"  k={k:3d}", " ".join(f"{v:7.0f}" for v in d[k]))

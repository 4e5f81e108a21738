"""Per-phase cycles of one panel_lat_kernel launch from a PRRP_PANEL_TL dump (CTA 0).
compute thread 0 marks: 0 start, 1 argmax + publish, 2 pushes (pusher warp), 3 winner known (bar 2),
4 partial dots, 5 scalars ready (bar 3), 6 update, 7 next norms.
control warp marks: 0 candidates in (bar 1), 1 exchange done, 2 cluster winner, 3 reflector scalars.
usage: PRRP_PANEL_PROF=1 PRRP_PANEL_TL=<panel> PRRP_PANEL_TL_OUT=f python tools/run_lu.py --n N --b B; lat_tl.py f"""
import sys
import numpy as np

raw = np.fromfile(sys.argv[1], dtype=np.int64)


def table(tl, names, nm):
    steps = int((tl[:, 0] != 0).sum())
    tl = tl[:steps, :nm].astype(np.float64)
    tl[tl == 0] = np.nan
    for m in range(1, nm):
        bad = np.isnan(tl[:, m])
        tl[bad, m] = tl[bad, m - 1]
    d = np.diff(tl, axis=1)
    print(f"{steps} steps; step mean {np.nanmean(np.diff(tl[:, 0])):.0f} cycles")
    print("  " + "  ".join(f"{n}={np.nanmean(d[:, i]):.0f}" for i, n in enumerate(names)))
    for k in (0, 1, 8, 31, 32, 63, 64, 96, 120):
        if k < steps:
            print(f"  k={k:3d}", " ".join(f"{v:7.0f}" for v in d[k]))
    return tl


print("compute thread 0:")
tc = table(raw[:1024].reshape(128, 8), ["argmax+publish", "bar1+push", "wait winner", "partial dots", "wait scalars", "update", "norms"], 8)
print("control warp:")
tk = table(raw[1024:2048].reshape(128, 8), ["exchange", "cluster winner", "scalars"], 4)
n = min(len(tc), len(tk))
print("control bar1-release relative to compute step start: mean %.0f" % np.nanmean(tk[:n, 0] - tc[:n, 0]))

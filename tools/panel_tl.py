"""Summarise a panel timeline dump (PRRP_PANEL_TL build, tools/_ablate)."""
import sys
import numpy as np

tl = np.fromfile(sys.argv[1], dtype=np.int64)[:16 * 64 * 8].reshape(16, 64, 8)
import os
names = os.environ.get("TL_NAMES", "warp-argmax+cand+bar,cta-argmax+push,wait,argmax+pull+bar,log,-,apply").split(",")
live = [c for c in range(16) if tl[c, 0, 0] != 0]
for c in live[:3]:
    d = np.diff(tl[c], axis=1)          # 64 x 7
    step = np.diff(tl[c, :, 0])
    print(f"cta {c}: step mean {step.mean():.0f} cyc;", ", ".join(f"{n}={d[:, i].mean():.0f}" for i, n in enumerate(names)))
    for k in (0, 16, 32, 48, 62):
        print("   k=%d" % k, " ".join(f"{v:6d}" for v in d[k]))

raw = np.fromfile(sys.argv[1], dtype=np.int64)
if raw.size > 16 * 64 * 8:
    w = raw[16 * 64 * 8:].reshape(16, 64, 8)
    t0 = tl[0, :, 0]
    print("CTA 0 per warp (cycles after thread 0's step start): start, argmax, cand done, bar A, copy, sqrt, vtv, div")
    for k in (0, 16, 32, 48):
        print("  k=%d" % k, "  ".join("w%d:%s" % (i, ",".join(str(int(v - t0[k])) for v in w[i, k])) for i in range(16) if w[i, k, 0]))

"""Localise a CALU schedule race: factor the same matrix twice in two scheduling
modes (env of two subprocesses), save LU + perm, report the first panel whose
columns differ and which rows / column ranges differ there."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(env_extra, out, n, b):
    code = f"""
import ctypes, numpy as np, torch, sys
sys.path.insert(0, {ROOT!r})
from paper_1208_2451_b200 import _lib, matgen
lib = _lib.device_lib()
n, b = {n}, {b}
a = matgen.gen_randn(n, 42, order="C")
buf = torch.empty((n, n), dtype=torch.float64, device="cuda")
perm = torch.empty(n, dtype=torch.int64, device="cuda")
for r in range(2):
    buf.copy_(torch.from_numpy(a))
    npan = (n + b - 1) // b
    sw = (ctypes.c_int32 * npan)(); chg = (ctypes.c_int64 * npan)()
    st, err = _lib.PrrpStats(), _lib.PrrpErr()
    rc = lib.prrp_caluprrp(ctypes.c_void_p(buf.data_ptr()), n, n, n, b, 2.0, 8, ctypes.c_void_p(perm.data_ptr()),
                           sw, chg, ctypes.byref(st), ctypes.byref(err), _lib.stream_handle())
    torch.cuda.synchronize()
np.save({out!r} + "_lu.npy", buf.cpu().numpy()); np.save({out!r} + "_p.npy", perm.cpu().numpy())
"""
    env = dict(os.environ, **env_extra)
    subprocess.run([sys.executable, "-c", code], env=env, check=True)


def main():
    n, b = int(sys.argv[1]), int(sys.argv[2])
    envs = [dict(kv.split("=") for kv in sys.argv[3].split(",") if kv), dict(kv.split("=") for kv in sys.argv[4].split(",") if kv)]
    tmp = "/tmp/calu_diff"
    run(envs[0], tmp + "A", n, b)
    run(envs[1], tmp + "B", n, b)
    A, pA = np.load(tmp + "A_lu.npy"), np.load(tmp + "A_p.npy")
    B, pB = np.load(tmp + "B_lu.npy"), np.load(tmp + "B_p.npy")
    print("perm equal:", np.array_equal(pA, pB), "lu equal:", np.array_equal(A, B))
    d = A != B
    cols = np.nonzero(d.any(axis=0))[0]
    if cols.size == 0:
        return
    j0 = int(cols[0])
    k = j0 // b
    print(f"first differing column {j0} (panel {k}); differing columns in that panel:",
          np.nonzero(d[:, k * b:(k + 1) * b].any(axis=0))[0][:10])
    rows = np.nonzero(d[:, j0])[0]
    print(f"rows differing in column {j0}: count {rows.size}, min {rows.min()}, max {rows.max()}, first {rows[:10]}")
    # per-panel picture of the earliest differences
    for kk in range(max(0, k - 1), min(n // b, k + 3)):
        blk = d[:, kk * b:(kk + 1) * b]
        r = np.nonzero(blk.any(axis=1))[0]
        print(f" panel {kk}: {blk.sum()} elements differ, rows {r.min() if r.size else '-'}..{r.max() if r.size else '-'}"
              f" ({r.size} rows)")
    # row ranges relative to the panel start for the first bad panel
    r = np.nonzero(d[:, k * b:].any(axis=1))[0]
    print(" rows (all columns >= panel start) differing below slot", k * b, ":", r[:20], "...", r.size)


if __name__ == "__main__":
    main()

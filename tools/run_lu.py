"""Run LU_PRRP factorizations on the device (for ncu launch lists / captures)."""
import argparse
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--b", type=int, default=64)
    ap.add_argument("--reps", type=int, default=1)
    args = ap.parse_args()
    import torch
    from paper_1208_2451_b200 import _lib, matgen
    lib = _lib.device_lib()
    n, b = args.n, args.b
    a = matgen.gen_randn(n, 42, order="C")
    lda = n + (n & 1)
    buf = torch.empty((n, lda), dtype=torch.float64, device="cuda")
    for r in range(args.reps):
        buf[:, :n].copy_(torch.from_numpy(a))
        perm = torch.empty(n, dtype=torch.int64, device="cuda")
        sw = (ctypes.c_int32 * ((n + b - 1) // b))()
        st = _lib.PrrpStats()
        err = _lib.PrrpErr()
        tm = _lib.PrrpTiming()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rc = lib.prrp_luprrp_timed(ctypes.c_void_p(buf.data_ptr()), lda, n, n, b, 2.0, ctypes.c_void_p(perm.data_ptr()),
                                   sw, ctypes.byref(st), ctypes.byref(err), ctypes.byref(tm), _lib.stream_handle())
        dt = time.perf_counter() - t0
        _lib.raise_for(rc, err, "luprrp")
        print(f"rep {r}: {dt*1e3:.2f} ms wall, {tm.total_ms:.2f} ms device; breakdown", {k: round(tm.ms[i], 3) for i, k in enumerate(_lib.KCLASSES)},
              "growth", st.intermediate_max / st.original_max, flush=True)


if __name__ == "__main__":
    main()

"""Time CALU_PRRP (prrp_caluprrp) on a device-resident matrix (SURVEY configs C4/C5)."""
import argparse
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--b", type=int, default=64)
    ap.add_argument("--P", type=int, default=8)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--urand", action="store_true")
    args = ap.parse_args()
    import torch
    from paper_1208_2451_b200 import _lib, matgen
    lib = _lib.device_lib()
    n, b = args.n, args.b
    a = matgen.gen_urand(n, 42, order="C") if args.urand else matgen.gen_randn(n, 42, order="C")
    lda = n + (n & 1)
    buf = torch.empty((n, lda), dtype=torch.float64, device="cuda")
    perm = torch.empty(n, dtype=torch.int64, device="cuda")   # one buffer: rep 0 direct, rep 1 capture, then replays
    for r in range(args.reps):
        buf[:, :n].copy_(torch.from_numpy(a))
        npan = (n + b - 1) // b
        sw = (ctypes.c_int32 * npan)()
        chg = (ctypes.c_int64 * npan)()
        st = _lib.PrrpStats()
        err = _lib.PrrpErr()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rc = lib.prrp_caluprrp(ctypes.c_void_p(buf.data_ptr()), lda, n, n, b, 2.0, args.P,
                               ctypes.c_void_p(perm.data_ptr()), sw, chg, ctypes.byref(st), ctypes.byref(err),
                               _lib.stream_handle())
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if os.environ.get("PRRP_HOSTTIME"):
            print(f"call returned after {(t1 - t0) * 1e3:.1f} ms, synchronized after {dt * 1e3:.1f} ms", flush=True)
        _lib.raise_for(rc, err, "caluprrp")
        gf = 2 * n ** 3 / 3 / dt / 1e9
        print(f"rep {r}: n={n} b={b} P={args.P}: {dt * 1e3:.1f} ms, {gf:.0f} GFLOP/s, swaps {sum(sw)}, "
              f"growth {st.intermediate_max / st.original_max:.4g}", flush=True)


if __name__ == "__main__":
    main()

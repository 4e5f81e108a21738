"""Factor one matrix with CALU_PRRP several times and print a digest of the
result (perm, packed LU, growth) per call: schedule races show up as digests
that differ between calls or between scheduling modes (env knobs)."""
import argparse
import ctypes
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--b", type=int, default=128)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--urand", action="store_true")
    ap.add_argument("--lu", action="store_true", help="LU_PRRP (prrp_luprrp) instead of CALU_PRRP")
    args = ap.parse_args()
    import torch
    from paper_1208_2451_b200 import _lib, matgen
    lib = _lib.device_lib()
    n, b = args.n, args.b
    a = matgen.gen_urand(n, 42, order="C") if args.urand else matgen.gen_randn(n, 42, order="C")
    lda = n + (n & 1)
    buf = torch.empty((n, lda), dtype=torch.float64, device="cuda")
    perm = torch.empty(n, dtype=torch.int64, device="cuda")
    for r in range(args.reps):
        buf[:, :n].copy_(torch.from_numpy(a))
        npan = (n + b - 1) // b
        sw = (ctypes.c_int32 * npan)()
        chg = (ctypes.c_int64 * npan)()
        st, err = _lib.PrrpStats(), _lib.PrrpErr()
        if args.lu:
            rc = lib.prrp_luprrp(ctypes.c_void_p(buf.data_ptr()), lda, n, n, b, 2.0, ctypes.c_void_p(perm.data_ptr()),
                                 sw, ctypes.byref(st), ctypes.byref(err), _lib.stream_handle())
        else:
            rc = lib.prrp_caluprrp(ctypes.c_void_p(buf.data_ptr()), lda, n, n, b, 2.0, 8,
                                   ctypes.c_void_p(perm.data_ptr()), sw, chg, ctypes.byref(st), ctypes.byref(err),
                                   _lib.stream_handle())
        torch.cuda.synchronize()
        _lib.raise_for(rc, err, "caluprrp")
        h = hashlib.sha1(buf[:, :n].contiguous().cpu().numpy().tobytes()).hexdigest()[:12]
        hp = hashlib.sha1(perm.cpu().numpy().tobytes()).hexdigest()[:12]
        print(f"rep {r}: lu {h} perm {hp} swaps {sum(sw)} growth {st.intermediate_max / st.original_max:.15g}",
              flush=True)


if __name__ == "__main__":
    main()

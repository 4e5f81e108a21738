"""Time calu_factor (tournament-pivoted GEPP) on the device: prrp_calu on a
resident buffer, wall clock around a synchronised call.
usage: python tools/run_gcalu.py N B P [reps]"""
import ctypes
import sys
import time

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1208_2451_b200 import _lib, matgen  # noqa: E402
from paper_1208_2451_b200.luprrp import upload  # noqa: E402

n, b, P = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
a = matgen.gen_randn(n, 42)
lib = _lib.device_lib()
buf0, lda = upload(a)
perm = torch.empty(n, dtype=torch.int64, device="cuda")
npan = (n + b - 1) // b
for r in range(reps):
    buf = buf0.clone()
    chg = (ctypes.c_int64 * npan)()
    st = _lib.PrrpStats()
    err = _lib.PrrpErr()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc = lib.prrp_calu(ctypes.c_void_p(buf.data_ptr()), lda, n, n, b, P, ctypes.c_void_p(perm.data_ptr()), chg,
                       ctypes.byref(st), ctypes.byref(err), _lib.stream_handle())
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"calu_factor n={n} b={b} P={P}: rc={rc} {dt * 1e3:.1f} ms  {2 * n ** 3 / 3 / dt / 1e9:.0f} GFLOP/s "
          f"growth {st.intermediate_max / st.original_max:.3f}", flush=True)

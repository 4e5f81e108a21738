"""Time gepp_factor (unblocked device GEPP) on a resident n x n buffer.
usage: python tools/run_gepp.py N [reps]"""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1208_2451_b200 import _lib  # noqa: E402

n = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
lib = _lib.device_lib()
a0 = torch.from_numpy(np.random.default_rng(0).standard_normal((n, n))).cuda()
P = torch.empty(n, dtype=torch.int64, device="cuda")
for _ in range(reps):
    A = a0.clone()
    im, om, err = ctypes.c_double(0), ctypes.c_double(0), _lib.PrrpErr()
    torch.cuda.synchronize()
    t = time.perf_counter()
    rc = lib.prrp_gepp(ctypes.c_void_p(A.data_ptr()), n, n, n, ctypes.c_void_p(P.data_ptr()), ctypes.byref(im),
                       ctypes.byref(om), ctypes.byref(err), _lib.stream_handle())
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"prrp_gepp n={n}: rc={rc} {dt * 1e3:.1f} ms ({2 * n ** 3 / 3 / dt / 1e9:.0f} GFLOP/s), growth "
          f"{im.value / om.value:.3f}", flush=True)

"""Run prrp_strong_rrqr on one h x p panel a few times (for ncu captures of the panel engine)."""
import ctypes
import sys

import numpy as np

sys.path.insert(0, ".")


def main():
    import torch
    from paper_1208_2451_b200 import _lib
    h, p, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 3
    lib = _lib.device_lib()
    rng = np.random.default_rng(0)
    a = torch.from_numpy(np.ascontiguousarray(rng.standard_normal((p, h)))).cuda()
    R = torch.empty((h, p), dtype=torch.float64, device="cuda")
    Q = torch.empty((h, h), dtype=torch.float64, device="cuda")
    perm = torch.empty(p, dtype=torch.int64, device="cuda")
    L = torch.empty(max(1, (p - h) * h), dtype=torch.float64, device="cuda")
    sw = ctypes.c_int32()
    for _ in range(reps):
        err = _lib.PrrpErr()
        rc = lib.prrp_strong_rrqr(ctypes.c_void_p(a.data_ptr()), h, h, p, h, 2.0, ctypes.c_void_p(R.data_ptr()),
                                  ctypes.c_void_p(Q.data_ptr()), ctypes.c_void_p(perm.data_ptr()),
                                  ctypes.c_void_p(L.data_ptr()), ctypes.byref(sw), ctypes.byref(err),
                                  _lib.stream_handle())
        torch.cuda.synchronize()
        _lib.raise_for(rc, err, "strong_rrqr")
    print("ok", h, p, "swaps", sw.value)


if __name__ == "__main__":
    main()

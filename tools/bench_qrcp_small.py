"""Time the strong RRQR of small panels (tournament merge nodes, the CALU final
QR) through prrp_strong_rrqr: device time per call (CUDA events), median of reps."""
import ctypes
import statistics
import sys

import numpy as np

sys.path.insert(0, ".")


def main():
    import torch
    from paper_1208_2451_b200 import _lib
    lib = _lib.device_lib()
    rng = np.random.default_rng(0)
    for h, p in ((64, 128), (64, 256), (128, 256), (128, 512), (64, 512), (128, 1024)):
        a = torch.from_numpy(np.ascontiguousarray(rng.standard_normal((p, h)))).cuda()   # panel rows
        R = torch.empty((h, p), dtype=torch.float64, device="cuda")
        Q = torch.empty((h, h), dtype=torch.float64, device="cuda")
        perm = torch.empty(p, dtype=torch.int64, device="cuda")
        L = torch.empty((p - h) * h, dtype=torch.float64, device="cuda")
        sw = ctypes.c_int32()
        ts = []
        for r in range(12):
            err = _lib.PrrpErr()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            rc = lib.prrp_strong_rrqr(ctypes.c_void_p(a.data_ptr()), h, h, p, h, 2.0, ctypes.c_void_p(R.data_ptr()),
                                      ctypes.c_void_p(Q.data_ptr()), ctypes.c_void_p(perm.data_ptr()),
                                      ctypes.c_void_p(L.data_ptr()), ctypes.byref(sw), ctypes.byref(err),
                                      _lib.stream_handle())
            e1.record()
            e1.synchronize()
            _lib.raise_for(rc, err, "strong_rrqr")
            if r >= 2:
                ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        print(f"h={h} p={p}: {ms * 1e3:.0f} us per strong_rrqr ({ms * 1e3 / h:.2f} us per step incl. trsm/finalize)")


if __name__ == "__main__":
    main()

"""Time the panel QRCP engines alone (prrp_b200_qrcp_time) over panel shapes and
latency-engine shapes (compute warps per CTA x columns per team); nwc = -1 is the
thread-per-column engine.  usage: lat_sweep.py [h:p ...]"""
import ctypes
import sys

import numpy as np

sys.path.insert(0, ".")


def main():
    import torch
    from paper_1208_2451_b200 import _lib
    lib = _lib.device_lib()
    shapes = [tuple(map(int, s.split(":"))) for s in sys.argv[1:]] or [
        (64, 128), (64, 512), (64, 2048), (128, 128), (128, 256), (128, 512), (128, 1024), (128, 1792)]
    rng = np.random.default_rng(0)
    for h, p in shapes:
        a = torch.from_numpy(np.ascontiguousarray(rng.standard_normal((p, h)))).cuda()
        out = []
        for nwc, cpt in ((-1, 0), (7, 1), (7, 2), (7, 4), (15, 1), (15, 2), (15, 4)):
            ms, ct = ctypes.c_double(), ctypes.c_int32()
            err = _lib.PrrpErr()
            rc = lib.prrp_b200_qrcp_time(ctypes.c_void_p(a.data_ptr()), h, h, p, nwc, cpt, 5, ctypes.byref(ms),
                                         ctypes.byref(ct), None, None, ctypes.byref(err))
            if rc != 0:
                out.append(f"({nwc},{cpt}): -")
                continue
            out.append(f"({nwc},{cpt}) C={ct.value}: {ms.value * 1e3:.0f} us = {ms.value * 1e3 / min(h, p):.2f}/step")
        print(f"h={h} p={p}: " + " | ".join(out), flush=True)


if __name__ == "__main__":
    main()

"""Time the Schur update kernel alone through prrp_schur_update (C -= L B,
FP64 DMMA) on the trailing-update shapes of the BASELINE configs.
usage: bench_schur.py [--old]   (--old: PRRP_SCHUR_OLD=1, the previous kernels)"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if "--old" in sys.argv:
    os.environ["PRRP_SCHUR_OLD"] = "1"


def main():
    import torch
    from paper_1208_2451_b200 import _lib
    lib = _lib.device_lib()
    shapes = [(8128, 8064, 64), (4096, 4096, 64), (8064, 8064, 128), (16256, 16256, 128), (32640, 32640, 128),
              (8000, 64, 64), (8000, 128, 128)]
    for a in sys.argv[1:]:
        if a.startswith("--shapes="):
            shapes = [tuple(int(v) for v in t.split("x")) for t in a[9:].split(",")]
    tf = ctypes.c_double(0)
    err = _lib.PrrpErr()
    lib.prrp_b200_dmma_peak(ctypes.c_double(1000.0), ctypes.byref(tf), ctypes.byref(err))
    print(f"dmma peak {tf.value:.2f} TFLOP/s", flush=True)
    for (M, N, K) in shapes:
        g = torch.Generator(device="cuda").manual_seed(1)
        C = torch.randn(M, N, dtype=torch.float64, device="cuda", generator=g)
        L = torch.randn(K, M, dtype=torch.float64, device="cuda", generator=g)   # column-major M x K
        B = torch.randn(K, N, dtype=torch.float64, device="cuda", generator=g)
        mx = ctypes.c_double(0)
        s = _lib.stream_handle()
        args = (ctypes.c_void_p(C.data_ptr()), N, ctypes.c_void_p(L.data_ptr()), M, ctypes.c_void_p(B.data_ptr()), N,
                M, N, K, ctypes.byref(mx), ctypes.byref(err), s)
        for _ in range(2):
            assert lib.prrp_schur_update(*args) == 0, err.msg
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(3, min(50, int(2e12 / (2 * M * N * K))))
        e0.record()
        for _ in range(reps):
            lib.prrp_schur_update(*args)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        fl = 2.0 * M * N * K / (ms * 1e-3) / 1e12
        gbs = 8.0 * (2 * M * N + M * K + K * N) / (ms * 1e-3) / 1e9
        print(f"M={M} N={N} K={K}: {ms:.3f} ms  {fl:.2f} TFLOP/s ({100 * fl / tf.value:.0f}% of DMMA)  {gbs:.0f} GB/s",
              flush=True)
        del C, L, B


if __name__ == "__main__":
    main()

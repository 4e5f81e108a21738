"""Cost of producing a fresh 512 MiB host result array from device data (probe)."""
import ctypes
import mmap
import time

import numpy as np
import torch

N = 8192
nbytes = N * N * 8
x = torch.randn((N, N), dtype=torch.float64, device="cuda")
torch.cuda.synchronize()


def t():
    torch.cuda.synchronize()
    return time.perf_counter()


print("THP:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
print("torch threads:", torch.get_num_threads())
cudart = ctypes.CDLL("libcudart.so") if False else None
for rep in range(2):
    # A: fresh pinned block (torch caching host allocator miss)
    t0 = t(); h = torch.empty((N, N), dtype=torch.float64, pin_memory=True); t1 = t(); h.copy_(x); t2 = t()
    print(f"A fresh pinned: alloc {1e3*(t1-t0):.0f} ms, D2H {1e3*(t2-t1):.0f} ms")
    keepA = h
    # B: pinned staging (cached) -> fresh np.empty via torch parallel copy
    st = torch.empty((N, N), dtype=torch.float64, pin_memory=True) if rep == 0 else st
    st.copy_(x); torch.cuda.synchronize()
    t0 = t(); out = np.empty((N, N)); torch.from_numpy(out).copy_(st); t1 = t()
    print(f"B np.empty + parallel host copy from pinned: {1e3*(t1-t0):.0f} ms")
    # C: hugepage mmap + parallel host copy
    t0 = t()
    mm = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    try:
        mm.madvise(mmap.MADV_HUGEPAGE)
    except Exception as e:
        print("madvise failed", e)
    arr = np.frombuffer(mm, dtype=np.float64).reshape(N, N)
    torch.from_numpy(arr).copy_(st)
    t1 = t()
    print(f"C hugepage mmap + parallel host copy: {1e3*(t1-t0):.0f} ms")
    # D: hugepage mmap + cudaHostRegister + direct D2H
    mm2 = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    mm2.madvise(mmap.MADV_HUGEPAGE)
    arr2 = np.frombuffer(mm2, dtype=np.float64).reshape(N, N)
    t0 = t()
    r = torch.cuda.cudart().cudaHostRegister(arr2.ctypes.data, nbytes, 0)
    t1 = t()
    torch.from_numpy(arr2).copy_(x)
    t2 = t()
    torch.cuda.cudart().cudaHostUnregister(arr2.ctypes.data)
    t3 = t()
    print(f"D hugepage mmap + cudaHostRegister {1e3*(t1-t0):.0f} ms (rc {r}), D2H {1e3*(t2-t1):.0f} ms, unregister {1e3*(t3-t2):.0f} ms")

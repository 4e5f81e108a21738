"""Where the end-to-end luprrp_factor time goes (upload, factorization, split, pinned alloc, D2H)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import paper_1208_2451_b200 as prrp
    from paper_1208_2451_b200 import luprrp, matgen
    n, b = int(sys.argv[1]) if len(sys.argv) > 1 else 8192, 64
    a = matgen.gen_randn(n, 42, order="C")
    pinned = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    pinned.copy_(torch.from_numpy(a))
    a_pin = pinned.numpy()
    prrp.luprrp_factor(a_pin, b, 2.0)

    def t():
        torch.cuda.synchronize()
        return time.perf_counter()

    keep = []
    for rep in range(3):
        t0 = t()
        buf, lda = luprrp.upload(a_pin)
        t1 = t()
        perm, st, sw = luprrp.run_device("prrp_luprrp", buf, lda, n, n, b, 2.0)
        t2 = t()
        packed = buf[:, :n]
        lt = torch.tril(packed, -1)
        lt.diagonal().fill_(1.0)
        lt_t = lt.t().contiguous()
        del lt
        u_t = torch.triu(packed[:n, :]).t().contiguous()
        t3 = t()
        l_h = torch.empty(lt_t.shape, dtype=torch.float64, pin_memory=True)
        u_h = torch.empty(u_t.shape, dtype=torch.float64, pin_memory=True)
        t4 = t()
        l_h.copy_(lt_t, non_blocking=True)
        u_h.copy_(u_t, non_blocking=True)
        t5 = t()
        p = perm.cpu().numpy()
        t6 = t()
        keep.append((l_h, u_h))   # like a caller holding the previous factors
        print(f"rep {rep}: upload {1e3*(t1-t0):.1f} ms, factor {1e3*(t2-t1):.1f}, split {1e3*(t3-t2):.1f}, "
              f"pinned alloc {1e3*(t4-t3):.1f}, D2H {1e3*(t5-t4):.1f}, perm {1e3*(t6-t5):.1f}, total {1e3*(t6-t0):.1f}",
              flush=True)
    keep.clear()
    for rep in range(2):
        t0 = time.perf_counter()
        f = prrp.luprrp_factor(a_pin, b, 2.0)
        t1 = time.perf_counter()
        del f
        print(f"api call (previous result released): {1e3*(t1-t0):.1f} ms", flush=True)
    # pageable D2H for comparison
    x = torch.empty((n, n), dtype=torch.float64, device="cuda")
    h = np.empty((n, n))
    th = torch.from_numpy(h)
    t0 = t(); th.copy_(x); t1 = t()
    print(f"pageable D2H 512 MiB: {1e3*(t1-t0):.1f} ms")
    t0 = t(); x.copy_(torch.from_numpy(a)); t1 = t()
    print(f"pageable H2D 512 MiB: {1e3*(t1-t0):.1f} ms")


if __name__ == "__main__":
    main()

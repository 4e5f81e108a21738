"""Phase times of the end-to-end luprrp_factor call (upload, device factorization,
prefault join, device split + staged D2H of l and u)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from paper_1208_2451_b200 import luprrp, matgen
    n, b = 8192, 64
    a = matgen.gen_randn(n, 42, order="C")
    pinned = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    pinned.copy_(torch.from_numpy(a))
    a_pin = pinned.numpy()
    luprrp.luprrp_factor(a_pin, b, 2.0)
    print("torch threads", torch.get_num_threads(), flush=True)
    for rep in range(3):
        t0 = time.perf_counter()
        pre = luprrp._Prefault([(n, n), (n, n)])
        buf, lda = luprrp.upload(a_pin)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        perm, st, sw = luprrp.run_device("prrp_luprrp", buf, lda, n, n, b, 2.0)
        t2 = time.perf_counter()
        out = pre.get()
        t3 = time.perf_counter()
        import torch as T
        packed = buf[:, :n]
        lt = T.tril(packed, -1); lt.diagonal().fill_(1.0); lt_t = lt.t().contiguous(); del lt
        u_t = T.triu(packed[:n, :]).t().contiguous()
        T.cuda.synchronize(); t4 = time.perf_counter()
        luprrp.split_to_host(packed, n, n, out[0], out[1]); t5 = time.perf_counter(); t6 = t5
        print(f"rep {rep}: upload {1e3*(t1-t0):.1f} factor {1e3*(t2-t1):.1f} prefault-join {1e3*(t3-t2):.1f} "
              f"split {1e3*(t4-t3):.1f} l->host {1e3*(t5-t4):.1f} u->host {1e3*(t6-t5):.1f} total {1e3*(t6-t0):.1f} ms",
              flush=True)
    # raw host copy bandwidth from a pinned block into a prefaulted array
    src = torch.empty(64 << 17, dtype=torch.float64, pin_memory=True)
    dst = torch.from_numpy(np.zeros(64 << 17))
    t0 = time.perf_counter()
    for _ in range(8):
        dst.copy_(src)
    dt = time.perf_counter() - t0
    print(f"host copy pinned->pageable: {8 * src.numel() * 8 / dt / 1e9:.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()

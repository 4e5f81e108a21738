import sys, time, torch, numpy as np
sys.path.insert(0, '.')
import paper_1208_2451_b200 as prrp
from paper_1208_2451_b200 import matgen
n = 8192
a = matgen.gen_randn(n, 42, order="C")
pinned = torch.empty((n, n), dtype=torch.float64, pin_memory=True); pinned.copy_(torch.from_numpy(a)); ap = pinned.numpy()
f = prrp.luprrp_factor(ap, 64, 2.0)
held = []
for r in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    f = prrp.luprrp_factor(ap, 64, 2.0)
    print(f"pinned input, results held: {1e3*(time.perf_counter()-t0):.1f} ms", flush=True)
    held.append(f)
for r in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    f = prrp.luprrp_factor(a, 64, 2.0)
    print(f"pageable input: {1e3*(time.perf_counter()-t0):.1f} ms", flush=True)
ref = held[0]
print("l,u equal across calls:", np.array_equal(ref.l, f.l), np.array_equal(ref.u, f.u), ref.l.flags['F_CONTIGUOUS'])

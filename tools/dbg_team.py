import sys, numpy as np
sys.path.insert(0, '.')
import paper_1208_2451_b200 as dev
cases = [((4, 7), 4), ((1, 2), 1), ((3, 12), 3), ((8, 40), 8), ((16, 200), 16), ((64, 400), 64), ((128, 256), 128), ((64, 128), 64)]
rng = np.random.default_rng(0)
for (h, p), b in cases:
    a = np.asfortranarray(rng.standard_normal((h, p)))
    print("case", h, p, b, flush=True)
    r = dev.strong_rrqr(a, b, 2.0)
    print("  ok", r.qr.perm[:8], flush=True)

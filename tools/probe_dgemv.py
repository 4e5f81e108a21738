"""Empirically identify the summation order of numpy `v @ M` (OpenBLAS dgemv_t)
for short columns (L <= 128), the rounding source in the reference's Householder
step (pivoted_qr.py:56)."""
import numpy as np
from fractions import Fraction
import itertools, sys

def fma(a, b, c):
    return float(Fraction(a) * Fraction(b) + Fraction(c))

def model(v, col, P, comb, tail_mode, R=None):
    L = len(v)
    R = R or P
    m1 = L - (L % R)
    acc = [0.0] * P
    for i in range(m1):
        acc[i % P] = fma(v[i], col[i], acc[i % P])
    if comb == 'pair':
        vals = acc[:]
        while len(vals) > 1:
            vals = [vals[j] + vals[j + 1] for j in range(0, len(vals), 2)]
        s = vals[0]
    elif comb == 'seq':
        s = acc[0]
        for x in acc[1:]:
            s = s + x
    elif comb == 'hadd4':  # P multiple of 4: first fold groups of 4 lanes elementwise, then (l0+l1)+(l2+l3)
        lanes = [0.0] * 4
        for g in range(0, P, 4):
            lanes = [lanes[q] + acc[g + q] if g else acc[g + q] for q in range(4)]
        s = (lanes[0] + lanes[1]) + (lanes[2] + lanes[3])
    elif comb == 'hadd4b':
        lanes = [0.0] * 4
        for g in range(0, P, 4):
            lanes = [lanes[q] + acc[g + q] if g else acc[g + q] for q in range(4)]
        s = (lanes[0] + lanes[2]) + (lanes[1] + lanes[3])
    y = 0.0 + s if m1 else 0.0
    if tail_mode == 'fma_seq':
        for i in range(m1, L):
            y = fma(v[i], col[i], y)
    elif tail_mode == 'temp':
        t = None
        for i in range(m1, L):
            t = v[i] * col[i] if t is None else fma(v[i], col[i], t)
        if t is not None:
            y = y + t
    elif tail_mode == 'temp_mul':
        t = None
        for i in range(m1, L):
            t = v[i] * col[i] if t is None else t + v[i] * col[i]
        if t is not None:
            y = y + t
    return y

rng = np.random.default_rng(1)
models = [(P, comb, tm, R) for P in (4, 8, 16) for comb in ('pair', 'seq', 'hadd4', 'hadd4b') for tm in ('fma_seq', 'temp', 'temp_mul') for R in (4, 8, 16) if R >= P or R == 4]
Ls = [int(x) for x in sys.argv[1:]] or [3, 4, 5, 7, 8, 9, 12, 15, 16, 17, 31, 32, 33, 47, 63, 64, 65, 100, 127, 128]
alive = set(models)
for L in Ls:
    N = 6
    M = np.asfortranarray(rng.standard_normal((L + 3, N)))[3:, :]   # offset slice like r[k:, k:]
    v = rng.standard_normal(L)
    got = v @ M
    for mdl in list(alive):
        P, comb, tm, R = mdl
        for j in range(N):
            if model(v, M[:, j], P, comb, tm, R) != got[j]:
                alive.discard(mdl)
                break
    print(L, len(alive), sorted(alive)[:6])

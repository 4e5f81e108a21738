"""Deterministic host-side test matrices with the reference's recipes
(matgen.py:3-8: PCG64(seed), uniforms via Generator.random, normals via an
explicit Box-Muller transform, row-major fill).  Input generation only —
the factorization never runs on the host."""
import numpy as np


def _rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def _normals(rng, count):
    """matgen._normals (matgen.py:41-50)."""
    pairs = (count + 1) // 2
    u1 = rng.random(pairs)
    u2 = rng.random(pairs)
    rad = np.sqrt(-2.0 * np.log1p(-u1))
    ang = 2.0 * np.pi * u2
    z = np.empty(2 * pairs)
    z[0::2] = rad * np.cos(ang)
    z[1::2] = rad * np.sin(ang)
    return z[:count]


def gen_randn(n, seed, order="F"):
    """matgen.gen_randn (matgen.py:53-56).  order='C' returns the same values
    C-contiguous (the device layout) without an extra transpose copy."""
    if n < 1:
        raise ValueError("n must be positive")
    a = _normals(_rng(seed), n * n).reshape(n, n)
    return np.asfortranarray(a) if order == "F" else a


def gen_urand(n, seed, order="F"):
    """U(-1,1) entries for BASELINE config 5 (not in the reference's matgen;
    defined in SURVEY.md 8(d) with the same PCG64 / row-major conventions)."""
    a = 2.0 * _rng(seed).random(n * n).reshape(n, n) - 1.0
    return np.asfortranarray(a) if order == "F" else a


def gen_wilkinson(n):
    """matgen.gen_wilkinson (matgen.py:63-70)."""
    if n < 2:
        raise ValueError("n must be >= 2")
    a = np.tril(-np.ones((n, n)), -1) + np.eye(n)
    a[:n - 1, n - 1] = 1.0
    return np.asfortranarray(a)


def gen_foster(n, c=1.0, h=1.0, k=2.0 / 3.0):
    """matgen.gen_foster (matgen.py:116-130)."""
    if c == 0.0:
        raise ValueError("c must be nonzero")
    if n < 2:
        raise ValueError("n must be >= 2")
    kh = k * h
    a = np.zeros((n, n), order="F")
    a[np.tril_indices(n, -1)] = -kh
    a[1:, 0] = -kh / 2.0
    np.fill_diagonal(a, 1.0 - kh / 2.0)
    a[0, 0] = 1.0
    a[:n - 1, n - 1] = -1.0 / c
    a[n - 1, n - 1] = 1.0 - 1.0 / c - kh / 2.0
    return a

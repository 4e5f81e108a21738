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


def gen_randn_rect(m, n, seed):
    """m x n normals: the first m*n draws of matgen._normals in row-major
    order (the reference's conventions, rectangular; used for the panel
    strong-RRQR parity cases)."""
    return _normals(_rng(seed), m * n).reshape(m, n)


def gen_urand_cols(n, seed, ncols, chunk_rows=1024):
    """Columns [0, ncols) of gen_urand(n, seed), F-ordered, generated in
    row chunks so the n x n matrix is never formed (PCG64 doubles are drawn
    one per value, so chunked draws continue the same stream)."""
    rng = _rng(seed)
    out = np.empty((n, ncols), order="F")
    for r0 in range(0, n, chunk_rows):
        r1 = min(n, r0 + chunk_rows)
        blk = rng.random((r1 - r0) * n).reshape(r1 - r0, n)
        out[r0:r1, :] = 2.0 * blk[:, :ncols] - 1.0
    return out


def gen_kahan_panel(p, b, theta, scale, seed):
    """A b x p panel transpose on which column-pivoted QR is not rank
    revealing: a Kahan block K (s^i on the diagonal, -c s^i above, columns
    damped by (1 - 1e-10)^j so the pivots come in order) followed by p - b
    small random columns scaled like K's rows.  K^-1 grows like (1 + c)^b,
    so |R11^-1 R12| exceeds tau and the strong-RRQR swap loop runs
    (pivoted_qr.py:129-144).  Elementwise construction only (no BLAS), so
    the bits do not depend on the host's BLAS kernels."""
    c, s = np.cos(theta), np.sin(theta)
    rs = s ** np.arange(b, dtype=np.float64)
    cd = (1.0 - 1e-10) ** np.arange(b, dtype=np.float64)
    k = np.triu(np.full((b, b), -c), 1) + np.eye(b)
    k = (k * rs[:, None]) * cd[None, :]
    r = (gen_randn_rect(b, p - b, seed) * scale) * rs[:, None]
    return np.hstack([k, r])


def gen_deficient_block(n, seed, blocks, cols):
    """randn(n, seed) with numerically rank-deficient row blocks in the first
    `cols` columns: for each (r0, r1, rank) in `blocks`, row r0 + i of the
    block becomes base row (i mod rank) scaled by 2^(i // rank), the
    base rows being the block's own first `rank` rows.  Power-of-two scaling
    is exact, so the block has exact rank `rank`; no two rows are equal
    (equal columns tie exactly, and which copy wins is then decided by the
    BLAS kernel's rounding, not by the algorithm), and a column-pivoted QR of
    its transpose meets roundoff-level diagonals after `rank` steps -- a
    CALU tournament node whose strong RRQR reports RankDeficient and passes
    on fewer than b rows (tournament.py:131-137).  Elementwise only (no
    BLAS), so the bits do not depend on the host."""
    a = np.array(gen_randn(n, seed, order="C"))
    for r0, r1, rank in blocks:
        base = a[r0:r0 + rank, :cols].copy()
        for i in range(r1 - r0):
            a[r0 + i, :cols] = base[i % rank] * (2.0 ** (i // rank))
    return np.asfortranarray(a)


def gen_urand_colset(n, seed, cols, chunk_rows=1024):
    """gen_urand(n, seed)[:, cols] (row-major m x len(cols)), streamed in row
    chunks: the rank-local columns of config 5 without forming the n x n
    matrix on any one host process."""
    cols = np.asarray(cols, dtype=np.int64)
    rng = _rng(seed)
    out = np.empty((n, len(cols)))
    for r0 in range(0, n, chunk_rows):
        r1 = min(n, r0 + chunk_rows)
        blk = rng.random((r1 - r0) * n).reshape(r1 - r0, n)
        out[r0:r1, :] = 2.0 * blk[:, cols] - 1.0
    return out


def gen_wright(n, h=0.3):
    """matgen.gen_wright (matgen.py:133-143): multiple-shooting matrix of a
    two-point boundary-value problem -- identity, the 2 x 2 blocks
    -[[1 - h/6, h], [h, 1 - h/6]] below the block diagonal, an identity
    block in the top-right corner."""
    if n % 2 or n < 4:
        raise ValueError("n must be even and >= 4")
    a = np.eye(n, order="F")
    blk = -np.array([[1.0 - h / 6.0, h], [h, 1.0 - h / 6.0]])
    for r in range(2, n, 2):
        a[r:r + 2, r - 2:r] = blk
    a[:2, n - 2:] = np.eye(2)
    return a


def gen_generalized_wilkinson(n, r=2, seed=0):
    """matgen.gen_generalized_wilkinson without fixed u, v (matgen.py:82-110):
    uniform n x r factors, the strict upper part of -u v^T scaled row by row
    below 1 in magnitude (factor max|row| (1 + 1/n)), transposed, unit
    diagonal, last column of ones."""
    if n < 2 or r < 1:
        raise ValueError("need n >= 2 and r >= 1")
    rng = _rng(seed)
    u = rng.random((n, r))
    v = rng.random((n, r))
    t = -np.triu(u @ v.T)
    for k in range(1, n):
        t[k - 1, k:] /= np.abs(t[k - 1, k:]).max() * (1.0 + 1.0 / n)
    t = t - np.diag(np.diag(t))
    a = t.T + np.eye(n)
    a[:n - 1, n - 1] = 1.0
    return np.asfortranarray(a)

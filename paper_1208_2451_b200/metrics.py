"""Device verification metrics (reference metrics.py).

rel_factorization_error(a, perm, l, u) = ||Pi A - L U||_F / ||A||_F
(metrics.py:56-63), computed on the B200 (prrp_lu_residual: row gather, the
DMMA Schur kernel one 64-wide k-block at a time, sum-of-squares reductions).
The reference accumulates L U with BLAS dger and subtracts once; the device
accumulates each k-block's product the same way, so the value agrees to
rounding (it is a backward-error measure, compared with a tolerance)."""
import ctypes
import math

import numpy as np

from . import _lib
from .errors import DimensionMismatch
from .luprrp import _pack_lu_device, as_matrix


def rel_factorization_error(a, perm, l, u):
    """|| Pi A - L U ||_F / || A ||_F for factors of an m x n (m >= n) matrix."""
    import torch
    a = as_matrix(a)
    m, n = a.shape
    if l.shape != (m, n) or u.shape != (n, n) or len(perm) != m:
        raise DimensionMismatch("factor shapes do not match the matrix")
    lib = _lib.device_lib()
    A = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    lu = _pack_lu_device(l, u)
    p = torch.from_numpy(np.asarray(perm, dtype=np.int64)).cuda()
    return rel_factorization_error_device(A, lu, p)


def rel_factorization_error_device(A, lu, perm):
    """Same on device tensors: A (m x n row-major), packed lu (m x n), perm (int64[m])."""
    lib = _lib.device_lib()
    m, n = A.shape
    r2, a2 = ctypes.c_double(0.0), ctypes.c_double(0.0)
    err = _lib.PrrpErr()
    rc = lib.prrp_lu_residual(ctypes.c_void_p(A.data_ptr()), A.stride(0), ctypes.c_void_p(lu.data_ptr()),
                              lu.stride(0), ctypes.c_void_p(perm.data_ptr()), m, n, ctypes.byref(r2),
                              ctypes.byref(a2), ctypes.byref(err), _lib.stream_handle())
    _lib.raise_for(rc, err, "rel_factorization_error")
    num = math.sqrt(max(r2.value, 0.0))
    den = math.sqrt(max(a2.value, 0.0))
    return num if den == 0.0 else num / den


# ---------------------------------------------------------------- stability battery (metrics.py:65-228)
from dataclasses import dataclass  # noqa: E402
import warnings  # noqa: E402

HPL_EPS = 2.0 ** -52              # metrics.py:20 (HPL ratios)
UNIT_ROUNDOFF = 2.0 ** -53        # metrics.py:21 (flooring and the refinement stop)
CSV_VERSION = 1
CSV_HEADER = ("g_w", "rel_fact_error", "eta", "w", "hpl1", "hpl2", "hpl3",
              "n_ir", "norm_l1", "norm_linv1", "norm_u1", "norm_uinv1")


@dataclass
class StabilityReport:
    """metrics.py:26-37."""
    g_w: float
    rel_fact_error: float
    eta: float
    w: float
    hpl: tuple
    n_ir: float
    norm_l1: float
    norm_linv1: float
    norm_u1: float
    norm_uinv1: float


def report_csv_row(rep):
    """metrics.py:45-48."""
    vals = (rep.g_w, rep.rel_fact_error, rep.eta, rep.w, *rep.hpl, rep.n_ir,
            rep.norm_l1, rep.norm_linv1, rep.norm_u1, rep.norm_uinv1)
    return ",".join(repr(float(v)) for v in vals)


def growth_factor(stats):
    """metrics.py:51-53."""
    return stats.growth_factor


class _DeviceSystem:
    """A (and optionally its square factors) resident on the device for the
    measurement battery: residuals, absolute sums and solves without
    re-uploading the matrix every refinement step."""

    def __init__(self, a, factors=None):
        import torch
        a = as_matrix(a)
        self.m, self.n = a.shape
        self.lib = _lib.device_lib()
        self.A = torch.from_numpy(np.ascontiguousarray(a)).cuda()
        self.factors = factors
        self.lu = self.perm = None
        if factors is not None and hasattr(factors, "l") and hasattr(factors, "u") \
                and factors.l.shape[0] == factors.l.shape[1]:
            self.lu = _pack_lu_device(factors.l, factors.u)
            self.perm = torch.from_numpy(np.asarray(factors.perm, dtype=np.int64)).cuda()

    def vec(self, v):
        import torch
        return torch.from_numpy(np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(-1))).cuda()

    def residual(self, x, rhs):
        import torch
        xv, bv = self.vec(x), self.vec(rhs)
        if xv.shape[0] != self.n or bv.shape[0] != self.m:
            raise ValueError("residual_extended: shape mismatch")
        r = torch.empty(self.m, dtype=torch.float64, device="cuda")
        err = _lib.PrrpErr()
        rc = self.lib.prrp_residual_extended(ctypes.c_void_p(self.A.data_ptr()), self.A.stride(0), self.m, self.n,
                                             ctypes.c_void_p(xv.data_ptr()), ctypes.c_void_p(bv.data_ptr()),
                                             ctypes.c_void_p(r.data_ptr()), ctypes.byref(err), _lib.stream_handle())
        _lib.raise_for(rc, err, "residual_extended")
        return r.cpu().numpy()

    def abs_sums(self, x=None, cols=False, rows=False):
        import torch
        ca = torch.empty(self.n, dtype=torch.float64, device="cuda") if cols else None
        ra = torch.empty(self.m, dtype=torch.float64, device="cuda") if rows else None
        xv = self.vec(np.abs(np.asarray(x, dtype=np.float64))) if x is not None else None
        ax = torch.empty(self.m, dtype=torch.float64, device="cuda") if x is not None else None
        p = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
        err = _lib.PrrpErr()
        rc = self.lib.prrp_abs_sums(ctypes.c_void_p(self.A.data_ptr()), self.A.stride(0), self.m, self.n, p(xv),
                                    p(ca), p(ra), p(ax), ctypes.byref(err), _lib.stream_handle())
        _lib.raise_for(rc, err, "abs_sums")
        g = lambda t: t.cpu().numpy() if t is not None else None  # noqa: E731
        return g(ca), g(ra), g(ax)

    def norm_one(self):
        ca, _, _ = self.abs_sums(cols=True)
        return float(ca.max()) if ca.size else 0.0

    def norm_inf(self):
        _, ra, _ = self.abs_sums(rows=True)
        return float(ra.max()) if ra.size else 0.0

    def solve(self, rhs):
        if self.lu is None:
            return np.asarray(self.factors.solve(rhs), dtype=np.float64).reshape(-1)
        import torch
        B = self.vec(rhs)
        X = torch.empty_like(B)
        err = _lib.PrrpErr()
        rc = self.lib.prrp_lu_solve(ctypes.c_void_p(self.lu.data_ptr()), self.lu.shape[1], self.n,
                                    ctypes.c_void_p(self.perm.data_ptr()), ctypes.c_void_p(B.data_ptr()), self.n,
                                    ctypes.c_void_p(X.data_ptr()), self.n, 1, ctypes.byref(err),
                                    _lib.stream_handle())
        _lib.raise_for(rc, err, "solve")
        return X.cpu().numpy()


def residual_extended(a, x, rhs):
    """rhs - A x with compensated (twice working precision) accumulation
    (metrics.py:75-92), on the device, bit-identical to the reference."""
    return _DeviceSystem(a).residual(x, rhs)


def _normwise(sysd, x, rhs, r=None):
    r = sysd.residual(x, rhs) if r is None else r
    denom = sysd.norm_one() * float(np.abs(x).sum()) + float(np.abs(np.asarray(rhs, dtype=np.float64)).sum())
    num = float(np.abs(r).sum())
    if denom == 0.0:
        return 0.0 if num == 0.0 else np.inf
    return num / denom


def normwise_backward_error(a, x, rhs):
    """eta = ||r||_1 / (||A||_1 ||x||_1 + ||rhs||_1) (metrics.py:95-104)."""
    return _normwise(_DeviceSystem(a), np.asarray(x, dtype=np.float64).reshape(-1), rhs)


def _componentwise(sysd, xv, bv):
    r = np.abs(sysd.residual(xv, bv))
    _, _, ax = sysd.abs_sums(x=xv)
    denom = ax + np.abs(bv)
    zero = denom == 0.0
    if np.any(r[zero] != 0.0):
        return np.inf
    live = ~zero
    if not live.any():
        return 0.0
    return float((r[live] / denom[live]).max())


def componentwise_backward_error(a, x, rhs):
    """w = max_i |r_i| / (|A| |x| + |rhs|)_i, 0/0 counts as 0 (metrics.py:107-121)."""
    return _componentwise(_DeviceSystem(a), np.asarray(x, dtype=np.float64).reshape(-1),
                          np.asarray(rhs, dtype=np.float64).reshape(-1))


def hpl_triplet(a, x, rhs):
    """The three Linpack accuracy ratios (metrics.py:124-145)."""
    sysd = _DeviceSystem(a)
    n = sysd.m
    xv = np.asarray(x, dtype=np.float64).reshape(-1)
    rinf = float(np.abs(sysd.residual(xv, rhs)).max())
    a1, ainf = sysd.norm_one(), sysd.norm_inf()
    x1, xinf = float(np.abs(xv).sum()), float(np.abs(xv).max())

    def ratio(num, den):
        if den == 0.0:
            return 0.0 if num == 0.0 else np.inf
        return num / den
    return (ratio(rinf, HPL_EPS * a1 * n), ratio(rinf, HPL_EPS * a1 * x1), ratio(rinf, HPL_EPS * ainf * xinf * n))


def _refine(sysd, rhs, max_iters):
    n = sysd.m
    bv = np.asarray(rhs, dtype=np.float64).reshape(-1)
    x = sysd.solve(bv)
    w = _componentwise(sysd, x, bv)
    w_before = w
    best_x, best_w = x, w
    target = n * UNIT_ROUNDOFF
    steps = 0
    grew = 0
    while w > target and steps < max_iters:
        r = sysd.residual(x, bv)
        dx = sysd.solve(r)
        x = x + dx
        w_new = _componentwise(sysd, x, bv)
        steps += 1
        if w_new < best_w:
            best_x, best_w = x, w_new
        if w_new > w:
            grew += 1
            if grew >= 2:
                warnings.warn("iterative refinement diverging: w grew twice", RuntimeWarning, stacklevel=3)
                break
        else:
            grew = 0
        if w_new > 0.5 * w:
            w = w_new
            break
        w = w_new
    return best_x, steps, w_before


def iterative_refinement(factors, a, rhs, max_iters=10):
    """Classical refinement with compensated residuals (metrics.py:148-186):
    stops at w <= n u, at a less than 2x improvement, or after max_iters;
    returns (x, n_ir, w_before).  Solves and residuals on the device."""
    return _refine(_DeviceSystem(a, factors), rhs, max_iters)


def triangular_inverse_norms(l, u):
    """1-norms of L, L^-1, U, U^-1 (metrics.py:189-201).  The inverses are
    solved on the device column by column (prrp_lu_solve with the other
    factor the identity); a zero diagonal of U raises like dtrtri's info."""
    import torch
    from .errors import SingularFactor
    if l.shape[0] != l.shape[1] or u.shape[0] != u.shape[1]:
        raise ValueError("inverse norms need square factors")
    n = l.shape[0]
    lib = _lib.device_lib()

    def inv_colsums(packed):
        P = torch.from_numpy(np.ascontiguousarray(packed)).cuda()
        perm = torch.arange(n, dtype=torch.int64, device="cuda")
        E = torch.eye(n, dtype=torch.float64, device="cuda")        # column-major identity (symmetric)
        X = torch.empty_like(E)
        err = _lib.PrrpErr()
        rc = lib.prrp_lu_solve(ctypes.c_void_p(P.data_ptr()), n, n, ctypes.c_void_p(perm.data_ptr()),
                               ctypes.c_void_p(E.data_ptr()), n, ctypes.c_void_p(X.data_ptr()), n, n,
                               ctypes.byref(err), _lib.stream_handle())
        _lib.raise_for(rc, err, "triangular_inverse_norms")
        # X column j = inverse column j (column-major): its abs sums are the
        # row sums of the row-major view
        sysd = _DeviceSystem.__new__(_DeviceSystem)
        sysd.lib, sysd.A, sysd.m, sysd.n = lib, X, n, n
        _, ra, _ = sysd.abs_sums(rows=True)
        return ra

    eye = np.eye(n)
    lpack = np.tril(np.asarray(l, dtype=np.float64), -1) + eye       # U = I
    upack = np.triu(np.asarray(u, dtype=np.float64))                 # L = I (unit diagonal implied)
    nl = _DeviceSystem(np.asarray(l, dtype=np.float64)).norm_one()
    nu = _DeviceSystem(np.asarray(u, dtype=np.float64)).norm_one()
    nlinv = float(inv_colsums(lpack).max())
    try:
        nuinv = float(inv_colsums(upack).max())
    except SingularFactor as exc:
        raise ArithmeticError(f"U inversion failed at diagonal {exc.index + 1}") from exc
    return nl, nlinv, nu, nuinv


def full_report(a, factors, rhs):
    """The whole measurement battery for one solve-capable factorization
    (metrics.py:209-228): eta, w and the Linpack ratios at the direct
    solution, then refinement for the step count."""
    a = as_matrix(a)
    sysd = _DeviceSystem(a, factors)
    bv = np.asarray(rhs, dtype=np.float64).reshape(-1)
    x0 = sysd.solve(bv)
    _, n_ir, w_before = _refine(sysd, bv, 10)
    nl, nlinv, nu, nuinv = triangular_inverse_norms(factors.l, factors.u)
    stats = getattr(factors, "stats", None)
    g_w = stats.growth_factor if stats is not None else factors.growth_factor
    return StabilityReport(
        g_w=g_w,
        rel_fact_error=rel_factorization_error(a, factors.perm, factors.l, factors.u),
        eta=_normwise(sysd, x0, bv),
        w=w_before,
        hpl=hpl_triplet(a, x0, bv),
        n_ir=float(n_ir),
        norm_l1=nl, norm_linv1=nlinv, norm_u1=nu, norm_uinv1=nuinv,
    )

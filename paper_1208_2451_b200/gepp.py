"""Partial-pivoting LU of a block row on the device (reference gepp.py:39-65).

The factorizations use GEPP as the finisher of the b x w block row
(luprrp.py:107-127): block rows (m <= 128 <= ... n >= m) take that fused
device path (prrp_gepp_blockrow).  Every other shape -- the standalone GEPP
baseline of the paper's comparisons -- runs the unblocked device
elimination prrp_gepp (one pivot and one update launch per step, same
arithmetic as the reference)."""
import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DimensionMismatch


@dataclass
class GeppFactors:
    perm: np.ndarray      # row permutation, apply_row_perm(perm, a) == l @ u
    l: np.ndarray         # m x s unit lower trapezoidal, s = min(m, n)
    u: np.ndarray         # s x n upper trapezoidal
    intermediate_max: float
    original_max: float

    @property
    def growth_factor(self):
        if self.original_max == 0.0:
            raise ZeroDivisionError("growth factor of an all-zero matrix")
        return self.intermediate_max / self.original_max

    def solve(self, rhs):
        return gepp_solve(self, rhs)


def gepp_factor(a):
    """Factor an m x n matrix (any shape) with partial pivoting (gepp.py:39-65)."""
    import torch
    c = np.asarray(a, dtype=np.float64)
    if c.ndim != 2:
        raise DimensionMismatch(f"expected a 2-D array, got ndim={c.ndim}")
    m, n = c.shape
    lib = _lib.device_lib()
    s = min(m, n)
    if s == 0:
        # nothing to eliminate (gepp.py:43-47 with zero steps): identity order,
        # empty trapezoids, both maxima 0 (the reference's max norm of an empty matrix)
        return GeppFactors(perm=np.arange(m, dtype=np.intp), l=np.zeros((m, 0), order="F"),
                           u=np.zeros((0, n), order="F"), intermediate_max=0.0, original_max=0.0)
    ld = n + (n & 1)
    A = torch.zeros((m, ld), dtype=torch.float64, device="cuda")
    A[:, :n].copy_(torch.from_numpy(np.ascontiguousarray(c)))
    P = torch.empty(m, dtype=torch.int64, device="cuda")
    im = ctypes.c_double(0)
    om = ctypes.c_double(0)
    err = _lib.PrrpErr()
    if m <= 128 and n >= m:
        rc = lib.prrp_gepp_blockrow(ctypes.c_void_p(A.data_ptr()), ld, m, n, ctypes.c_void_p(P.data_ptr()),
                                    ctypes.byref(im), ctypes.byref(err), _lib.stream_handle())
        om.value = float(np.abs(c).max())
    else:
        rc = lib.prrp_gepp(ctypes.c_void_p(A.data_ptr()), ld, m, n, ctypes.c_void_p(P.data_ptr()),
                           ctypes.byref(im), ctypes.byref(om), ctypes.byref(err), _lib.stream_handle())
    err.panel = -1            # the standalone gepp_factor never tags a panel (gepp.py:49-51)
    _lib.raise_for(rc, err, "gepp_factor")
    packed = A[:, :n].cpu().numpy()
    l = np.tril(packed[:, :s], -1)
    np.fill_diagonal(l, 1.0)
    u = np.triu(packed[:s, :])
    return GeppFactors(perm=P.cpu().numpy().astype(np.intp), l=np.asfortranarray(l), u=np.asfortranarray(u),
                       intermediate_max=float(im.value), original_max=float(om.value))


def gepp_solve(f, rhs):
    """Solve A x = rhs from square GEPP factors (gepp.py:68-78) on the device."""
    from .luprrp import _solve_factors
    if f.l.shape[0] != f.l.shape[1]:
        raise DimensionMismatch("gepp_solve needs factors of a square matrix")
    return _solve_factors(f.perm, f.l, f.u, rhs, "gepp_solve")

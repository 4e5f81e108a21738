"""Partial-pivoting LU of a block row on the device (reference gepp.py:39-65).

The factorizations use GEPP only as the finisher of the b x w block row
(luprrp.py:107-127); this entry point exposes that device path for
m <= 128 rows (the standalone GEPP baseline is out of scope)."""
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


def gepp_factor(a):
    """Factor an m x n block row (m <= min(n, 128)) with partial pivoting."""
    import torch
    c = np.asarray(a, dtype=np.float64)
    if c.ndim != 2:
        raise DimensionMismatch(f"expected a 2-D array, got ndim={c.ndim}")
    m, n = c.shape
    if not (1 <= m <= 128 and n >= m):
        raise NotImplementedError("device GEPP covers the b x w block rows of the factorizations (m <= 128, n >= m)")
    lib = _lib.device_lib()
    A = torch.from_numpy(np.ascontiguousarray(c)).cuda()
    P = torch.empty(m, dtype=torch.int64, device="cuda")
    im = ctypes.c_double(0)
    err = _lib.PrrpErr()
    rc = lib.prrp_gepp_blockrow(ctypes.c_void_p(A.data_ptr()), n, m, n, ctypes.c_void_p(P.data_ptr()),
                                ctypes.byref(im), ctypes.byref(err), _lib.stream_handle())
    _lib.raise_for(rc, err, "gepp_factor")
    packed = A.cpu().numpy()
    l = np.tril(packed[:, :m], -1) + np.eye(m)
    u = np.triu(packed)
    return GeppFactors(perm=P.cpu().numpy().astype(np.intp), l=np.asfortranarray(l), u=np.asfortranarray(u),
                       intermediate_max=float(im.value), original_max=float(np.abs(c).max()) if c.size else 0.0)

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

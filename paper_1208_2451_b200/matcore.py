"""Device versions of the reference's product kernels (matcore.py:41-61).

rank_update(c, a, b) == c - matmul(a, b) with matmul's rounding recipe
(accumulation from zero in increasing k, one FMA per k: BLAS dger on FMA
hosts), computed by the TMA + DMMA Schur kernel (prrp_schur_update)."""
import ctypes

import numpy as np

from . import _lib
from .errors import DimensionMismatch


def _as_matrix(a):
    m = np.asarray(a, dtype=np.float64)
    if m.ndim != 2:
        raise DimensionMismatch(f"expected a 2-D array, got ndim={m.ndim}")
    return m


def rank_update(c, a, b):
    """Return c - a.b (reference matcore.py:54-61)."""
    import torch
    c = _as_matrix(c)
    a = _as_matrix(a)
    b = _as_matrix(b)
    if c.shape[0] != a.shape[0] or c.shape[1] != b.shape[1] or a.shape[1] != b.shape[0]:
        raise DimensionMismatch(f"rank_update: result shape {c.shape} does not match product {a.shape} x {b.shape}")
    M, N = c.shape
    K = a.shape[1]
    if M == 0 or N == 0:
        return np.asfortranarray(c.copy())
    lib = _lib.device_lib()
    C = torch.from_numpy(np.ascontiguousarray(c)).cuda()
    L = torch.from_numpy(np.ascontiguousarray(a.T)).cuda()        # column-major M x K
    B = torch.from_numpy(np.ascontiguousarray(b)).cuda()
    if K == 0:
        return np.asfortranarray(c.copy())
    err = _lib.PrrpErr()
    rc = lib.prrp_schur_update(ctypes.c_void_p(C.data_ptr()), N, ctypes.c_void_p(L.data_ptr()), M,
                               ctypes.c_void_p(B.data_ptr()), N, M, N, K, None, ctypes.byref(err),
                               _lib.stream_handle())
    _lib.raise_for(rc, err, "rank_update")
    return np.asfortranarray(C.cpu().numpy())


def matmul(a, b):
    """c[i,j] = sum_k a[i,k] b[k,j] accumulated in increasing k (matcore.py:41-51):
    -(0 - a.b), exact negation of the device rank update on a zero matrix."""
    a = _as_matrix(a)
    b = _as_matrix(b)
    if a.shape[1] != b.shape[0]:
        raise DimensionMismatch(f"matmul: inner dimensions differ ({a.shape} x {b.shape})")
    out = -rank_update(np.zeros((a.shape[0], b.shape[1])), a, b)
    out[out == 0.0] = 0.0          # +0 like the reference's zero-initialised accumulator
    return np.asfortranarray(out)

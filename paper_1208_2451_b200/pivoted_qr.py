"""Strong RRQR / Householder QR entry points on the device (reference
pivoted_qr.py:28-147).  Inputs are h x p host matrices as in the reference;
the panel engine runs on the B200 (prrp_strong_rrqr, prrp_householder_qr)."""
import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DimensionMismatch

EPS = 2.0 ** -52


@dataclass
class QRFactors:
    q: np.ndarray          # h x h explicit orthogonal factor
    r: np.ndarray          # h x p upper trapezoidal
    perm: np.ndarray       # column permutation: (A Pi)[:, j] = A[:, perm[j]]


@dataclass
class SrrqrResult:
    qr: QRFactors
    tau: float
    swap_count: int
    l_block: np.ndarray    # (p - b) x b, equal to (R11^-1 R12)^T


def swap_cap(b, p, tau):
    """Iteration cap for the interchange loop (pivoted_qr.py:108-110)."""
    return int(math.ceil(2.0 * b * math.log(max(p, 2)) / math.log(tau))) + 10


def _as_matrix(a):
    m = np.asarray(a, dtype=np.float64)
    if m.ndim != 2:
        raise DimensionMismatch(f"expected a 2-D array, got ndim={m.ndim}")
    return m


def _to_device_colmajor(a):
    import torch
    h, p = a.shape
    # column-major h x p == row-major p x h
    return torch.from_numpy(np.ascontiguousarray(a.T)).to("cuda")


def strong_rrqr(a, b, tau):
    """Strong RRQR of a with leading block size b and threshold tau > 1."""
    import torch
    a = _as_matrix(a)
    h, p = a.shape
    if tau <= 1.0:
        raise ValueError("tau must exceed 1")
    if h < b or p < b + 1:
        raise ValueError(f"strong_rrqr needs >= {b} rows and >= {b + 1} columns, got {h}x{p}")
    lib = _lib.device_lib()
    dev = _to_device_colmajor(a)
    R = torch.empty((p, h), dtype=torch.float64, device="cuda")        # col-major h x p
    Q = torch.empty((h, h), dtype=torch.float64, device="cuda")
    perm = torch.empty(p, dtype=torch.int64, device="cuda")
    L = torch.empty((b, p - b), dtype=torch.float64, device="cuda")    # col-major (p-b) x b
    sw = ctypes.c_int32(0)
    err = _lib.PrrpErr()
    rc = lib.prrp_strong_rrqr(ctypes.c_void_p(dev.data_ptr()), h, h, p, b, float(tau),
                              ctypes.c_void_p(R.data_ptr()), ctypes.c_void_p(Q.data_ptr()),
                              ctypes.c_void_p(perm.data_ptr()), ctypes.c_void_p(L.data_ptr()),
                              ctypes.byref(sw), ctypes.byref(err), _lib.stream_handle())
    _lib.raise_for(rc, err, "strong_rrqr")
    r = np.asfortranarray(R.cpu().numpy().T)
    q = np.asfortranarray(Q.cpu().numpy().T)
    lblk = np.asfortranarray(L.cpu().numpy().T)
    return SrrqrResult(qr=QRFactors(q=q, r=r, perm=perm.cpu().numpy().astype(np.intp)), tau=tau,
                       swap_count=int(sw.value), l_block=lblk)


def qr_column_pivoting(a):
    """QR with column pivoting, exact column norms recomputed each step
    (pivoted_qr.py:74-87), on the device (prrp_qrcp)."""
    import torch
    a = _as_matrix(a)
    h, p = a.shape
    lib = _lib.device_lib()
    dev = _to_device_colmajor(a)
    R = torch.empty((p, h), dtype=torch.float64, device="cuda")
    Q = torch.empty((h, h), dtype=torch.float64, device="cuda")
    perm = torch.empty(p, dtype=torch.int64, device="cuda")
    err = _lib.PrrpErr()
    rc = lib.prrp_qrcp(ctypes.c_void_p(dev.data_ptr()), h, h, p, ctypes.c_void_p(R.data_ptr()),
                       ctypes.c_void_p(Q.data_ptr()), ctypes.c_void_p(perm.data_ptr()), ctypes.byref(err),
                       _lib.stream_handle())
    _lib.raise_for(rc, err, "qr_column_pivoting")
    return QRFactors(q=np.asfortranarray(Q.cpu().numpy().T), r=np.asfortranarray(R.cpu().numpy().T),
                     perm=perm.cpu().numpy().astype(np.intp))


def householder_qr(a):
    """Unpivoted Householder QR with Q assembled explicitly (pivoted_qr.py:64-71)."""
    import torch
    a = _as_matrix(a)
    h, p = a.shape
    lib = _lib.device_lib()
    dev = _to_device_colmajor(a)
    R = torch.empty((p, h), dtype=torch.float64, device="cuda")
    Q = torch.empty((h, h), dtype=torch.float64, device="cuda")
    err = _lib.PrrpErr()
    rc = lib.prrp_householder_qr(ctypes.c_void_p(dev.data_ptr()), h, h, p, ctypes.c_void_p(R.data_ptr()),
                                 ctypes.c_void_p(Q.data_ptr()), ctypes.byref(err), _lib.stream_handle())
    _lib.raise_for(rc, err, "householder_qr")
    return QRFactors(q=np.asfortranarray(Q.cpu().numpy().T), r=np.asfortranarray(R.cpu().numpy().T),
                     perm=np.arange(p, dtype=np.intp))


def multiplier_block(r, b):
    """(R11^-1 R12)^T from an upper trapezoidal R (pivoted_qr.py:90-98)."""
    import torch
    r = _as_matrix(r)
    if r.shape[0] < b or r.shape[1] < b:
        raise ValueError("R smaller than the requested leading block")
    if r.shape[1] == b:
        return np.zeros((0, b), order="F")
    lib = _lib.device_lib()
    h, p = r.shape
    R = torch.from_numpy(np.ascontiguousarray(r.T)).to("cuda")       # column-major h x p
    L = torch.empty((b, p - b), dtype=torch.float64, device="cuda")  # column-major (p-b) x b
    err = _lib.PrrpErr()
    rc = lib.prrp_multiplier_block(ctypes.c_void_p(R.data_ptr()), h, b, p, ctypes.c_void_p(L.data_ptr()), p - b,
                                   None, ctypes.byref(err), _lib.stream_handle())
    _lib.raise_for(rc, err, "multiplier_block")
    return np.asfortranarray(L.cpu().numpy().T)

"""CALU_PRRP: tournament pivoting over a binary reduction tree, on the B200.

Keeps the reference's entry points and types (tournament.py:43-61, 237-296):
``caluprrp_factor(a, b, tau=2.0, tree=None)`` with ``binary_tree(P)``
(default P = 8).  The tournament runs on the device (prrp_caluprrp): leaves
and same-level merges execute concurrently, each as the cluster strong-RRQR
engine over an index list of logical rows; the result is independent of that
concurrency, as the reference's determinism contract requires
(tournament.py:24-25).
"""
import ctypes
import math
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import _lib
from .errors import DimensionMismatch
from .luprrp import (BlockLUFactors, ElimStats, _validate, as_matrix, flop_counters,
                     split_packed_device, upload)


@dataclass(frozen=True)
class ReductionTree:
    shape: str                  # 'binary' | 'flat'
    leaf_count: int | None = None

    def __post_init__(self):
        if self.shape not in ("binary", "flat"):
            raise ValueError(f"unknown tree shape {self.shape!r}")
        if self.shape == "binary":
            if self.leaf_count is None or self.leaf_count < 1:
                raise ValueError("binary tree needs a leaf count >= 1")


def binary_tree(p):
    return ReductionTree("binary", p)


def flat_tree():
    return ReductionTree("flat")


def tree_height(tree, m, b):
    """Height H of the first panel's reduction (tournament.py:91-96)."""
    if tree.shape == "binary":
        p_eff = max(1, min(tree.leaf_count, m // (b + 1)))
        return math.ceil(math.log2(p_eff)) if p_eff > 1 else 0
    first = min(m, 2 * b)
    return len(range(first, m, b))


def growth_bound_caluprrp_log2(n, b, tau, h):
    if not (n >= b >= 1) or h < 0:
        raise ValueError("need n >= b >= 1 and h >= 0")
    return (math.ceil(n / b) * (h + 1) - 1) * math.log2(1.0 + tau * b)


def growth_bound_caluprrp(n, b, tau, h):
    lg = growth_bound_caluprrp_log2(n, b, tau, h)
    return math.inf if lg > 1023.0 else 2.0 ** lg


def growth_condition(b, tau, h):
    if b < 2 or tau <= 1.0:
        raise ValueError("need b >= 2 and tau > 1")
    return h <= b / (math.log2(b) + math.log2(tau))


def caluprrp_factor(a, b, tau=2.0, tree=None):
    """Tournament-pivoted panel-RRQR LU (binary tree by default, P = 8).

    Drop-in for prrp.caluprrp_factor (reference tournament.py:237)."""
    a = as_matrix(a)
    _validate(a, b, tau)
    if tree is None:
        tree = binary_tree(8)
    if tree.shape != "binary":
        raise NotImplementedError("the device tournament implements the binary tree (flat tree: SURVEY 8(f))")
    m, n = a.shape
    lib = _lib.device_lib()
    import torch
    buf, lda = upload(a)
    perm = torch.empty(m, dtype=torch.int64, device="cuda")
    npan = (n + b - 1) // b
    swaps = (ctypes.c_int32 * npan)()
    chg3 = (ctypes.c_int64 * npan)()
    st = _lib.PrrpStats()
    err = _lib.PrrpErr()
    rc = lib.prrp_caluprrp(ctypes.c_void_p(buf.data_ptr()), lda, m, n, b, float(tau), int(tree.leaf_count),
                           ctypes.c_void_p(perm.data_ptr()), swaps, chg3, ctypes.byref(st), ctypes.byref(err),
                           _lib.stream_handle())
    _lib.raise_for(rc, err, "prrp_caluprrp")
    extra = [None if c < 0 else Fraction(int(c), 3) for c in chg3]
    charged, executed = flop_counters(m, n, b, list(swaps), tournament_extra=extra)
    stats = ElimStats(original_max=st.original_max, intermediate_max=st.intermediate_max,
                      finish_max=st.finish_max, swap_counts=list(map(int, swaps)),
                      flops_charged=charged, flops_executed=executed,
                      panel_multiplier_max=st.panel_multiplier_max)
    l, u = split_packed_device(buf[:, :n], m, n)
    return BlockLUFactors(perm=perm.cpu().numpy().astype(np.intp), l=l, u=u, panel_width=b, stats=stats)

"""CALU_PRRP: tournament pivoting over a binary reduction tree, on the B200.

Keeps the reference's entry points and types (tournament.py:43-61, 237-296):
``caluprrp_factor(a, b, tau=2.0, tree=None)`` with ``binary_tree(P)``
(default P = 8) or ``flat_tree()``.  The tournament runs on the device (prrp_caluprrp): leaves
and same-level merges execute concurrently, each as the cluster strong-RRQR
engine over an index list of logical rows; the result is independent of that
concurrency, as the reference's determinism contract requires
(tournament.py:24-25).

``calu_factor(a, b, tree=None)`` (tournament.py:299-359), the
tournament-pivoted GEPP baseline, runs the same tree with a GEPP selector
in every node (prrp_calu).
"""
import ctypes
import math
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import _lib
from .errors import DimensionMismatch
from .luprrp import (BlockLUFactors, ElimStats, _finish_charge, _validate, as_matrix, flop_counters,
                     split_packed_device, split_to_host, upload, _Prefault)


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


def _partition(m, p):
    """m rows into p contiguous blocks, as equal as possible, first larger
    (tournament.py:64-73)."""
    base, extra = divmod(m, p)
    out, start = [], 0
    for i in range(p):
        size = base + (1 if i < extra else 0)
        out.append((start, start + size))
        start += size
    return out


def leaf_blocks(tree, m, b):
    """Leaf row ranges for a panel of m rows; (blocks, effective P)
    (tournament.py:76-88)."""
    if tree.shape == "binary":
        p_eff = max(1, min(tree.leaf_count, m // (b + 1)))
        return _partition(m, p_eff), p_eff
    first = min(m, 2 * b)
    blocks, start = [(0, first)], first
    while start < m:
        stop = min(m, start + b)
        blocks.append((start, stop))
        start = stop
    return blocks, len(blocks)


@dataclass
class TournamentNode:
    level: int
    index: int
    members: np.ndarray      # panel-relative row indices entering the node
    selected: np.ndarray     # the b survivors, in selection order
    swap_count: int


@dataclass
class TournamentTrace:
    nodes: list
    pivot_rows: np.ndarray
    leaf_count: int
    requested_leaf_count: int | None
    single_node: bool
    srr: object = None       # SrrqrResult when single_node with the srrqr selector


def _select(panel, idx, b, tau, selector):
    """Up to b candidate rows among panel[idx] -> (selected, full_order,
    swap_count, srr_or_none) (tournament.py:118-152).  Every node is a device
    strong RRQR (prrp_strong_rrqr); a numerically rank-deficient node passes
    on only its independent rows."""
    from .errors import RankDeficient
    from .pivoted_qr import strong_rrqr
    if idx.shape[0] <= b:
        return idx, idx, 0, None
    sub = panel[idx, :]
    if selector == "srrqr":
        want = b
        while want:
            try:
                srr = strong_rrqr(sub.T, want, tau)
            except RankDeficient as exc:
                want = exc.index
                continue
            order = srr.qr.perm
            return idx[order[:want]], idx[order], srr.swap_count, (srr if want == b else None)
        return idx[:0], idx, 0, None
    if selector == "gepp":
        order, cols = gepp_select(sub)
        return idx[order[:cols]], idx[order], 0, None
    raise ValueError(f"unknown selector {selector!r}")


def gepp_select(sub):
    """GEPP selector node on the device (tournament.py:142-150): the
    elimination's row order of the r x b block `sub` (r > b) and the number
    of rows chosen before the first zero pivot -- the reference's retry with
    fewer columns reproduces exactly the first k steps, so its order is the
    order reached when column k is found zero."""
    import torch
    r, cols = sub.shape
    lib = _lib.device_lib()
    A = torch.from_numpy(np.ascontiguousarray(sub, dtype=np.float64)).cuda()
    order = torch.empty(r, dtype=torch.int64, device="cuda")
    cnt = ctypes.c_int32(0)
    err = _lib.PrrpErr()
    rc = lib.prrp_gepp_select(ctypes.c_void_p(A.data_ptr()), cols, r, cols, ctypes.c_void_p(order.data_ptr()),
                              ctypes.byref(cnt), ctypes.byref(err), _lib.stream_handle())
    _lib.raise_for(rc, err, "prrp_gepp_select")
    return order.cpu().numpy().astype(np.intp), int(cnt.value)


def tournament_select(panel, b, tau, tree, selector="srrqr"):
    """Reduce an m x b panel to b pivot rows; returns (perm, trace)
    (tournament.py:155-217).  Same tree walk, node numbering, odd-node
    promotion and rank-deficiency handling as the reference; each node's
    selection runs on the device."""
    from .errors import RankDeficient
    panel = as_matrix(panel)
    m = panel.shape[0]
    if panel.shape[1] != b:
        raise DimensionMismatch(f"panel has {panel.shape[1]} columns, expected {b}")
    blocks, p_eff = leaf_blocks(tree, m, b)
    nodes = []
    if len(blocks) == 1:
        idx = np.arange(m, dtype=np.intp)
        selected, order, swaps, srr = _select(panel, idx, b, tau, selector)
        if selected.shape[0] < b:
            raise RankDeficient(f"panel supplied only {selected.shape[0]} independent rows",
                                index=selected.shape[0])
        nodes.append(TournamentNode(0, 0, idx, selected, swaps))
        return np.asarray(order, dtype=np.intp), TournamentTrace(nodes, selected, p_eff, tree.leaf_count, True, srr)

    def run_node(level, index, idx):
        try:
            selected, _, swaps, _ = _select(panel, idx, b, tau, selector)
        except ArithmeticError as exc:
            exc.tree_node = (level, index)
            raise
        nodes.append(TournamentNode(level, index, idx, selected, swaps))
        return selected

    if tree.shape == "binary":
        cands = [run_node(0, i, np.arange(lo, hi, dtype=np.intp)) for i, (lo, hi) in enumerate(blocks)]
        level = 1
        while len(cands) > 1:
            merged = []
            for i in range(0, len(cands) - 1, 2):
                merged.append(run_node(level, i // 2, np.concatenate([cands[i], cands[i + 1]])))
            if len(cands) % 2:
                merged.append(cands[-1])
            cands = merged
            level += 1
        pivots = cands[0]
    else:
        lo, hi = blocks[0]
        cand = run_node(0, 0, np.arange(lo, hi, dtype=np.intp))
        for i, (lo, hi) in enumerate(blocks[1:], start=1):
            cand = run_node(i, 0, np.concatenate([cand, np.arange(lo, hi, dtype=np.intp)]))
        pivots = cand
    if pivots.shape[0] < b:
        raise RankDeficient(f"tournament supplied only {pivots.shape[0]} independent rows", index=pivots.shape[0])
    rest = np.setdiff1d(np.arange(m, dtype=np.intp), pivots)
    perm = np.concatenate([pivots, rest]).astype(np.intp)
    return perm, TournamentTrace(nodes, pivots, p_eff, tree.leaf_count, False, None)


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
    leaf_count = int(tree.leaf_count) if tree.shape == "binary" else 0   # 0: the flat tree
    m, n = a.shape
    lib = _lib.device_lib()
    import torch
    pre = _Prefault([(n, m), (n, n)]) if m * n >= (1 << 22) else None
    buf, lda = upload(a)
    perm = torch.empty(m, dtype=torch.int64, device="cuda")
    npan = (n + b - 1) // b
    swaps = (ctypes.c_int32 * npan)()
    chg3 = (ctypes.c_int64 * npan)()
    st = _lib.PrrpStats()
    err = _lib.PrrpErr()
    rc = lib.prrp_caluprrp(ctypes.c_void_p(buf.data_ptr()), lda, m, n, b, float(tau), leaf_count,
                           ctypes.c_void_p(perm.data_ptr()), swaps, chg3, ctypes.byref(st), ctypes.byref(err),
                           _lib.stream_handle())
    _lib.raise_for(rc, err, "prrp_caluprrp")
    extra = [None if c < 0 else Fraction(int(c), 3) for c in chg3]
    charged, executed = flop_counters(m, n, b, list(swaps), tournament_extra=extra)
    stats = ElimStats(original_max=st.original_max, intermediate_max=st.intermediate_max,
                      finish_max=st.finish_max, swap_counts=list(map(int, swaps)),
                      flops_charged=charged, flops_executed=executed,
                      panel_multiplier_max=st.panel_multiplier_max)
    l, u = split_to_host(buf[:, :n], m, n, *pre.get()) if pre else split_packed_device(buf[:, :n], m, n)
    return BlockLUFactors(perm=perm.cpu().numpy().astype(np.intp), l=l, u=u, panel_width=b, stats=stats)


def calu_factor(a, b, tree=None):
    """Tournament-pivoted GEPP: selection and panel finish both by partial
    pivoting (binary tree by default, P = 8).

    Drop-in for prrp.calu_factor (reference tournament.py:299-359); one
    device call (prrp_calu): GEPP tournament, row moves, GEPP finish of the
    block row, L21 = A21 U11^-1, DMMA trailing update per panel."""
    a = as_matrix(a)
    _validate(a, b, 2.0)
    if tree is None:
        tree = binary_tree(8)
    leaf_count = int(tree.leaf_count) if tree.shape == "binary" else 0
    m, n = a.shape
    lib = _lib.device_lib()
    import torch
    pre = _Prefault([(n, m), (n, n)]) if m * n >= (1 << 22) else None
    buf, lda = upload(a)
    perm = torch.empty(m, dtype=torch.int64, device="cuda")
    npan = (n + b - 1) // b
    chg3 = (ctypes.c_int64 * npan)()
    st = _lib.PrrpStats()
    err = _lib.PrrpErr()
    rc = lib.prrp_calu(ctypes.c_void_p(buf.data_ptr()), lda, m, n, b, leaf_count, ctypes.c_void_p(perm.data_ptr()),
                       chg3, ctypes.byref(st), ctypes.byref(err), _lib.stream_handle())
    _lib.raise_for(rc, err, "prrp_calu")
    charged = calu_flop_counter(m, n, b, [Fraction(int(c), 3) for c in chg3])
    stats = ElimStats(original_max=st.original_max, intermediate_max=st.intermediate_max,
                      finish_max=st.finish_max, swap_counts=[0] * npan,
                      flops_charged=charged, flops_executed=charged,
                      panel_multiplier_max=st.panel_multiplier_max)
    l, u = split_to_host(buf[:, :n], m, n, *pre.get()) if pre else split_packed_device(buf[:, :n], m, n)
    return BlockLUFactors(perm=perm.cpu().numpy().astype(np.intp), l=l, u=u, panel_width=b, stats=stats)


def calu_flop_counter(m, n, b, tournament_extra):
    """calu_factor's counter (charged == executed; tournament.py:321-356)."""
    tot = Fraction(0)
    col0 = 0
    panel = 0
    while col0 < n:
        bj = min(b, n - col0)
        rows = m - col0
        width = n - col0 - bj
        if rows > bj:
            tot += tournament_extra[panel]
            tot += Fraction((rows - bj) * bj * bj + 2 * bj * (rows - bj) * width)
        tot += _finish_charge(bj, n - col0)
        col0 += bj
        panel += 1
    return tot

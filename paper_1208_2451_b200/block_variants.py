"""Reduce-and-eliminate panel variants of LU_PRRP on the B200 (SURVEY.md
8(f)3; reference block_variants.py:1-251).

block_parallel_luprrp reduces each panel over a binary tree of P leaf blocks
(tournament leaves, tournament.py:64-88); block_pairwise_luprrp walks a flat
chain (first 2b rows, then b-row chunks).  Unlike tournament pivoting, every
node's strong RRQR immediately ELIMINATES its losing rows: their trailing
columns are updated against the node's winners with the node's multiplier
block and their panel columns are zeroed.  The factorization is kept as an
event log (row permutations and eliminations) plus the final upper factor;
replay_events re-applies the log to the input.

The working matrix stays in HBM.  Every node is a device strong RRQR
(prrp_strong_rrqr); every elimination is the bit-exact DMMA Schur update
(prrp_schur_update, matcore.rank_update's dger order); the block-row finish
is the device GEPP (prrp_gepp_steps, gepp.py's arithmetic) whose step
swaps and multipliers are recorded as the reference's events.  Index
bookkeeping (the event log, row orders) is host-side, as in the reference.
"""
import ctypes
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import _lib
from .errors import DimensionMismatch
from .luprrp import ElimStats, _qr_charge, _validate, as_matrix
from .tournament import _partition


@dataclass
class RowPermEvent:
    perm: np.ndarray          # full-length row permutation


@dataclass
class ElimEvent:
    elim_rows: np.ndarray     # row positions updated (current positions)
    pivot_rows: np.ndarray    # positions of the rows they are updated against
    d: np.ndarray             # |elim| x |pivot| multiplier block
    zero_col0: int
    zero_col1: int            # columns [zero_col0, zero_col1) set to exact zero
    update_col0: int          # trailing update covers columns update_col0..


@dataclass
class BlockVariantFactors:
    events: list
    u: np.ndarray             # final upper factor (m x n working matrix)
    perm: np.ndarray          # composed global row permutation
    panel_width: int
    stats: ElimStats
    leaf_counts: list         # effective leaf count per panel

    @property
    def max_multiplier(self):
        vals = [float(np.abs(ev.d).max()) for ev in self.events if isinstance(ev, ElimEvent) and ev.d.size]
        return max(vals) if vals else 0.0


class _Work:
    """The working matrix on the device (row-major, even leading dimension)
    and the device operations on its rows."""

    def __init__(self, a):
        import torch
        self.torch = torch
        self.m, self.n = a.shape
        self.ld = max(2, self.n + (self.n & 1))
        self.W = torch.zeros((self.m, self.ld), dtype=torch.float64, device="cuda")
        self.W[:, :self.n].copy_(torch.from_numpy(np.ascontiguousarray(a)))
        self.lib = _lib.device_lib()

    def idx(self, rows):
        return self.torch.from_numpy(np.asarray(rows, dtype=np.int64)).cuda()

    def strong_rrqr(self, rows, col0, bj, tau):
        """strong_rrqr(work[rows, col0:col0+bj].T, bj, tau) on the device ->
        (order, swap_count, l_block column-major device tensor)."""
        torch = self.torch
        r = len(rows)
        ldp = bj + (bj & 1)
        sub = torch.zeros((r, ldp), dtype=torch.float64, device="cuda")
        sub[:, :bj].copy_(self.W[self.idx(rows), col0:col0 + bj])
        R = torch.empty((bj, r), dtype=torch.float64, device="cuda")
        Q = torch.empty((bj, bj), dtype=torch.float64, device="cuda")
        perm = torch.empty(r, dtype=torch.int64, device="cuda")
        L = torch.empty(max(1, (r - bj) * bj), dtype=torch.float64, device="cuda")
        sw = ctypes.c_int32()
        err = _lib.PrrpErr()
        rc = self.lib.prrp_strong_rrqr(ctypes.c_void_p(sub.data_ptr()), ldp, bj, r, bj, float(tau),
                                       ctypes.c_void_p(R.data_ptr()), ctypes.c_void_p(Q.data_ptr()),
                                       ctypes.c_void_p(perm.data_ptr()), ctypes.c_void_p(L.data_ptr()),
                                       ctypes.byref(sw), ctypes.byref(err), _lib.stream_handle())
        _lib.raise_for(rc, err, "strong_rrqr")
        return perm.cpu().numpy(), int(sw.value), L

    def eliminate(self, losers, winners, L, col0, bj):
        """work[losers, col0+bj:] -= l_block @ work[winners, col0+bj:]
        (bit-exact rank_update), work[losers, col0:col0+bj] = 0; returns the
        max |updated| (the growth observation)."""
        torch = self.torch
        M, K = len(losers), len(winners)
        N = self.n - col0 - bj
        mx = ctypes.c_double(0.0)
        li = self.idx(losers)
        if N > 0 and M > 0:
            ldn = N + (N & 1)
            C = torch.zeros((M, ldn), dtype=torch.float64, device="cuda")
            C[:, :N].copy_(self.W[li, col0 + bj:self.n])
            B = torch.zeros((K, ldn), dtype=torch.float64, device="cuda")
            B[:, :N].copy_(self.W[self.idx(winners), col0 + bj:self.n])
            err = _lib.PrrpErr()
            rc = self.lib.prrp_schur_update(ctypes.c_void_p(C.data_ptr()), ldn, ctypes.c_void_p(L.data_ptr()), M,
                                            ctypes.c_void_p(B.data_ptr()), ldn, M, N, K, ctypes.byref(mx),
                                            ctypes.byref(err), _lib.stream_handle())
            _lib.raise_for(rc, err, "rank_update")
            self.W[li, col0 + bj:self.n] = C[:, :N]
        if M > 0:
            self.W[li, col0:col0 + bj] = 0.0
        return float(mx.value)

    def permute(self, full, col0):
        torch = self.torch
        self.W[col0:] = self.W[self.idx(full[col0:])]

    def gepp_block_row(self, col0, bj):
        """GEPP of the block row work[col0:col0+bj, col0:] in place (gepp.py
        arithmetic); returns (final row order, steps max)."""
        torch = self.torch
        w = self.n - col0
        perm = torch.empty(bj, dtype=torch.int64, device="cuda")
        smax, omax = ctypes.c_double(0), ctypes.c_double(0)
        err = _lib.PrrpErr()
        view = self.W[col0:col0 + bj, col0:]
        rc = self.lib.prrp_gepp_steps(ctypes.c_void_p(view.data_ptr()), self.ld, bj, w,
                                      ctypes.c_void_p(perm.data_ptr()), ctypes.byref(smax), ctypes.byref(omax),
                                      ctypes.byref(err), _lib.stream_handle())
        return rc, err, perm.cpu().numpy(), float(smax.value)

    def host(self):
        return np.asfortranarray(self.W[:, :self.n].cpu().numpy())


class _PanelState:
    def __init__(self, wk, col0, bj, tau, events, stats):
        self.wk, self.col0, self.bj, self.tau = wk, col0, bj, tau
        self.events, self.stats = events, stats
        self.swaps = 0

    def eliminate(self, idx):
        """block_variants.py:103-124: strong RRQR of rows idx, losers eliminated now."""
        if idx.shape[0] <= self.bj:
            return idx
        wk, col0, bj = self.wk, self.col0, self.bj
        order, swaps, L = wk.strong_rrqr(idx, col0, bj, self.tau)
        winners = idx[order[:bj]]
        losers = idx[order[bj:]]
        mx = wk.eliminate(losers, winners, L, col0, bj)
        if losers.size and col0 + bj < wk.n:
            self.stats.intermediate_max = max(self.stats.intermediate_max, mx)
        d = np.asfortranarray(L[:losers.size * bj].cpu().numpy().reshape(bj, losers.size).T) if losers.size \
            else np.zeros((0, bj), order="F")
        self.events.append(ElimEvent(elim_rows=losers, pivot_rows=winners, d=d, zero_col0=col0,
                                     zero_col1=col0 + bj, update_col0=col0 + bj))
        self.swaps += swaps
        self.stats.flops_charged += _qr_charge(idx.shape[0], bj)
        self.stats.flops_executed += (1 + swaps) * _qr_charge(idx.shape[0], bj)
        upd = Fraction(2 * bj * losers.shape[0] * (wk.n - col0 - bj))
        self.stats.flops_charged += upd
        self.stats.flops_executed += upd
        return winners


def _reduce_binary(state, rows, p):
    p_eff = max(1, min(p, rows // (state.bj + 1)))
    cands = [state.eliminate(np.arange(state.col0 + lo, state.col0 + hi, dtype=np.intp))
             for lo, hi in _partition(rows, p_eff)]
    while len(cands) > 1:
        merged = [state.eliminate(np.concatenate([cands[i], cands[i + 1]])) for i in range(0, len(cands) - 1, 2)]
        if len(cands) % 2:
            merged.append(cands[-1])          # odd node promoted unmerged
        cands = merged
    return cands[0], p_eff


def _reduce_chain(state, rows):
    col0, bj = state.col0, state.bj
    first = min(rows, 2 * bj)
    cand = state.eliminate(np.arange(col0, col0 + first, dtype=np.intp))
    start, chunks = first, 1
    while start < rows:
        stop = min(rows, start + bj)
        cand = state.eliminate(np.concatenate([cand, np.arange(col0 + start, col0 + stop, dtype=np.intp)]))
        start, chunks = stop, chunks + 1
    return cand, chunks


def _permute_pivots_top(wk, p, col0, pivots, events):
    m = wk.m
    tail = np.arange(col0, m, dtype=np.intp)
    full = np.concatenate([np.arange(col0, dtype=np.intp), pivots, np.setdiff1d(tail, pivots)])
    events.append(RowPermEvent(perm=full))
    wk.permute(full, col0)
    p[:] = p[full]


def _gepp_finish_events(wk, p, col0, bj, stats, events):
    """block_variants.py:170-195 on the device: the GEPP of the block row,
    then its steps as the reference's events -- per step k the interchange
    (a full-row RowPermEvent when the pivot moved) and the multipliers of
    the rows below in their positions at that step."""
    from .errors import SingularMatrix
    n = wk.n
    rc, err, order, smax = wk.gepp_block_row(col0, bj)
    if rc == _lib.PRRP_ERR_SINGULAR_MATRIX:
        raise SingularMatrix(f"zero pivot column {col0 + err.column}", column=col0 + err.column)
    _lib.raise_for(rc, err, "gepp_finish")
    packed = wk.W[col0:col0 + bj, col0:col0 + bj].cpu().numpy()
    # replay the interchanges: at step k the row finally at position k moves up
    cur = list(range(bj))            # cur[pos] = original block-row index at that position
    where = list(range(bj))          # where[orig] = position
    final_pos = np.empty(bj, dtype=np.intp)
    final_pos[order] = np.arange(bj)
    for k in range(bj):
        c = col0 + k
        src = where[order[k]]
        if src != k:
            full = np.arange(wk.m, dtype=np.intp)
            full[[c, col0 + src]] = full[[col0 + src, c]]
            events.append(RowPermEvent(perm=full))
            p[[c, col0 + src]] = p[[col0 + src, c]]
            a, b = cur[k], cur[src]
            cur[k], cur[src] = b, a
            where[b], where[a] = k, src
        below = np.arange(c + 1, col0 + bj, dtype=np.intp)
        if below.size:
            # the multiplier of the row at position q (step k) is L[final position of that row, k]
            rows_now = [cur[q - col0] for q in below]
            d = np.array([packed[final_pos[r], k] for r in rows_now]).reshape(-1, 1)
            events.append(ElimEvent(elim_rows=below, pivot_rows=np.array([c], dtype=np.intp), d=d,
                                    zero_col0=c, zero_col1=c + 1, update_col0=c + 1))
    # the reference zeroes each step's eliminated column (ElimEvent zero_col0..1):
    # the diagonal block keeps U only
    blk = wk.W[col0:col0 + bj, col0:col0 + bj]
    blk.copy_(wk.torch.triu(blk))
    if bj > 1 and col0 + 1 < n:
        stats.finish_max = max(stats.finish_max, smax)
    fin = Fraction(2, 3) * bj ** 3 + Fraction((n - col0 - bj) * bj * bj)
    stats.flops_charged += fin
    stats.flops_executed += fin


def _factor_variant(a, b, tau, reduce_panel):
    a = as_matrix(a)
    _validate(a, b, tau)
    m, n = a.shape
    wk = _Work(a)
    p = np.arange(m, dtype=np.intp)
    mx = float(np.abs(a).max()) if a.size else 0.0
    stats = ElimStats(original_max=mx, intermediate_max=mx, finish_max=mx)
    events, leaf_counts = [], []
    col0, panel = 0, 0
    while col0 < n:
        bj = min(b, n - col0)
        rows = m - col0
        state = _PanelState(wk, col0, bj, tau, events, stats)
        if rows > bj:
            try:
                pivots, p_eff = reduce_panel(state, rows)
            except ArithmeticError as exc:
                exc.panel = panel
                raise
            leaf_counts.append(p_eff)
            _permute_pivots_top(wk, p, col0, pivots, events)
        else:
            leaf_counts.append(1)
        stats.swap_counts.append(state.swaps)
        try:
            _gepp_finish_events(wk, p, col0, bj, stats, events)
        except ArithmeticError as exc:
            exc.panel = panel
            raise
        col0 += bj
        panel += 1
    return BlockVariantFactors(events=events, u=wk.host(), perm=p, panel_width=b, stats=stats,
                               leaf_counts=leaf_counts)


def block_parallel_luprrp(a, b, tau=2.0, p=4):
    """Binary-tree reduce-and-eliminate panel factorization (block_variants.py:231-236)."""
    if p < 1:
        raise ValueError("p must be >= 1")
    return _factor_variant(a, b, tau, lambda state, rows: _reduce_binary(state, rows, p))


def block_pairwise_luprrp(a, b, tau=2.0):
    """Flat-chain reduce-and-eliminate panel factorization (block_variants.py:239-244)."""
    a = as_matrix(a)
    if a.shape[0] < 2 * b + 1:
        raise DimensionMismatch("need at least 2b+1 rows")
    return _factor_variant(a, b, tau, _reduce_chain)


def replay_events(events, a):
    """Re-apply an event log to the input on the device (block_variants.py:79-87):
    row permutations as device gathers, eliminations as the bit-exact Schur
    update of the eliminated rows."""
    a = as_matrix(a)
    wk = _Work(a)
    for ev in events:
        if isinstance(ev, RowPermEvent):
            wk.permute(ev.perm, 0)
        else:
            _replay_elim(wk, ev)
    return wk.host()


def _replay_elim(wk, ev):
    torch = wk.torch
    if not ev.elim_rows.size:
        return
    M, K = ev.d.shape
    N = wk.n - ev.update_col0
    li = wk.idx(ev.elim_rows)
    if N > 0:
        ldn = N + (N & 1)
        C = torch.zeros((M, ldn), dtype=torch.float64, device="cuda")
        C[:, :N].copy_(wk.W[li, ev.update_col0:wk.n])
        B = torch.zeros((K, ldn), dtype=torch.float64, device="cuda")
        B[:, :N].copy_(wk.W[wk.idx(ev.pivot_rows), ev.update_col0:wk.n])
        L = torch.from_numpy(np.ascontiguousarray(np.asarray(ev.d, dtype=np.float64).T)).cuda()   # column-major M x K
        mx = ctypes.c_double(0.0)
        err = _lib.PrrpErr()
        rc = wk.lib.prrp_schur_update(ctypes.c_void_p(C.data_ptr()), ldn, ctypes.c_void_p(L.data_ptr()), M,
                                      ctypes.c_void_p(B.data_ptr()), ldn, M, N, K, ctypes.byref(mx),
                                      ctypes.byref(err), _lib.stream_handle())
        _lib.raise_for(rc, err, "rank_update")
        wk.W[li, ev.update_col0:wk.n] = C[:, :N]
    wk.W[li, ev.zero_col0:ev.zero_col1] = 0.0

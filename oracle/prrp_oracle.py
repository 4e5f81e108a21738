"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A numpy/scipy restatement of the reference's LU_PRRP / CALU_PRRP hot path
(arXiv 1208.2451 reference package ``prrp``, mounted at /root/reference in
the build container only).  Every function cites the reference file:line
whose arithmetic it restates.  The restatement keeps the reference's exact
floating-point recipe (numpy pairwise sums, BLAS ``dger`` k-loop products,
BLAS ``dgemv`` through ``@``, true division, product-then-subtract updates)
so that on the same host it reproduces the reference bit for bit; this is
pinned by ``tests/test_oracle_golden.py`` against fixtures produced by the
reference itself (``tests/golden/make_golden.py``).

Who may import this module: ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` — and only as
the checker or the timed CPU reference.  The product package
``paper_1208_2451_b200`` never imports it; its compute path is the CUDA
library and fails loudly when that library is missing.

Reference paths below are relative to /root/reference/pkg/src/prrp/.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np
from scipy.linalg.blas import dger

EPS = 2.0 ** -52           # pivoted_qr.py:25


# --------------------------------------------------------------------------
# exception mirror (errors.py:4-54); the oracle is standalone on the GPU box
# --------------------------------------------------------------------------
class OracleDimensionMismatch(ValueError):
    pass


class OracleSingularFactor(ArithmeticError):
    def __init__(self, msg, index):
        super().__init__(msg)
        self.index = index


class OracleSingularMatrix(ArithmeticError):
    def __init__(self, msg, column):
        super().__init__(msg)
        self.column = column


class OracleRankDeficient(ArithmeticError):
    def __init__(self, msg, index):
        super().__init__(msg)
        self.index = index


class OracleNonConvergence(ArithmeticError):
    def __init__(self, msg, worst):
        super().__init__(msg)
        self.worst = worst


# reference class name -> oracle class, used by tests to compare error kinds
ERROR_NAMES = {
    OracleDimensionMismatch: "DimensionMismatch",
    OracleSingularFactor: "SingularFactor",
    OracleSingularMatrix: "SingularMatrix",
    OracleRankDeficient: "RankDeficient",
    OracleNonConvergence: "NonConvergence",
}


# --------------------------------------------------------------------------
# kernel layer (matcore.py)
# --------------------------------------------------------------------------
def fmat(a):
    """2-D float64 Fortran copy-or-view (matcore.py:33-38)."""
    m = np.asarray(a, dtype=np.float64)
    if m.ndim != 2:
        raise OracleDimensionMismatch(f"expected a 2-D array, got ndim={m.ndim}")
    return np.asfortranarray(m)


def dger_product(a, b):
    """Product accumulated as K rank-1 ``dger`` calls in increasing k
    (matcore.py:41-51)."""
    a = fmat(a)
    b = fmat(b)
    if a.shape[1] != b.shape[0]:
        raise OracleDimensionMismatch("inner dimensions differ")
    acc = np.zeros((a.shape[0], b.shape[1]), order="F")
    for k in range(a.shape[1]):
        acc = dger(1.0, a[:, k], b[k, :], a=acc, overwrite_a=1)
    return acc


def schur_update(c, a, b):
    """c - a.b, product first then one subtraction (matcore.py:54-61)."""
    return fmat(c) - dger_product(a, b)


def upper_solve(u, rhs):
    """Back substitution U X = B in axpy form with true division
    (matcore.py:78-94)."""
    u = fmat(u)
    x = fmat(rhs).copy(order="F")
    n = u.shape[0]
    for i in range(n - 1, -1, -1):
        piv = u[i, i]
        if piv == 0.0:
            raise OracleSingularFactor(f"zero diagonal at index {i}", index=i)
        x[i, :] /= piv
        if i:
            x[:i, :] -= u[:i, i:i + 1] * x[i:i + 1, :]
    return x


def unit_lower_solve(l, rhs):
    """Forward substitution with unit diagonal (matcore.py:64-75)."""
    l = fmat(l)
    x = fmat(rhs).copy(order="F")
    for i in range(l.shape[0] - 1):
        x[i + 1:, :] -= l[i + 1:, i:i + 1] * x[i:i + 1, :]
    return x


def upper_solve_right(b, u):
    """X U = B, column by column: x[:, j] /= u[j, j], then
    x[:, j+1:] -= x[:, j] u[j, j+1:] (matcore.py:97-113)."""
    x = fmat(b).copy(order="F")
    n = u.shape[0]
    for j in range(n):
        d = u[j, j]
        if d == 0.0:
            raise OracleSingularFactor(f"zero diagonal at index {j}", index=j)
        x[:, j] /= d
        if j + 1 < n:
            x[:, j + 1:] -= x[:, j:j + 1] * u[j:j + 1, j + 1:]
    return x


def maxabs(a):
    a = np.asarray(a, dtype=np.float64)
    return 0.0 if a.size == 0 else float(np.abs(a).max())      # matcore.py:116-130 'max'


def frob(a):
    a = np.asarray(a, dtype=np.float64)
    return 0.0 if a.size == 0 else float(np.sqrt((a * a).sum()))   # matcore.py:126-127


def permute_rows(p, a):
    """Row i of the result is row p[i] of a (matcore.py:152-159)."""
    return np.asfortranarray(fmat(a)[np.asarray(p, dtype=np.intp), :])


# --------------------------------------------------------------------------
# pivot engines (pivoted_qr.py, gepp.py)
# --------------------------------------------------------------------------
@dataclass
class QR:
    q: np.ndarray
    r: np.ndarray
    perm: np.ndarray


@dataclass
class Srrqr:
    qr: QR
    tau: float
    swap_count: int
    l_block: np.ndarray


def reflect(r, q, k):
    """One Householder step zeroing r[k+1:, k] (pivoted_qr.py:43-61).
    Returns the (v, beta) pair applied, or None when the step is skipped."""
    x = r[k:, k]
    normx = float(np.sqrt((x * x).sum()))
    if normx == 0.0:
        return None
    alpha = -normx if x[0] >= 0.0 else normx
    v = x.copy()
    v[0] -= alpha
    vtv = float((v * v).sum())
    if vtv == 0.0:
        return None
    beta = 2.0 / vtv
    w = beta * (v @ r[k:, k:])
    r[k:, k:] -= np.outer(v, w)
    qv = q[:, k:] @ v
    q[:, k:] -= np.outer(beta * qv, v)
    r[k, k] = alpha
    r[k + 1:, k] = 0.0
    return v, beta


def qr_plain(a):
    """Unpivoted Householder QR, explicit Q (pivoted_qr.py:64-71)."""
    r = fmat(a).copy(order="F")
    h, p = r.shape
    q = np.eye(h, order="F")
    for k in range(min(h, p)):
        reflect(r, q, k)
    return QR(q=q, r=r, perm=np.arange(p, dtype=np.intp))


def qr_pivoted(a, trace=None):
    """QR with column pivoting on exact recomputed norms, first max wins
    (pivoted_qr.py:74-87).  ``trace`` (optional list) receives the relative
    gap between the best and the second-best norm at every step."""
    r = fmat(a).copy(order="F")
    h, p = r.shape
    q = np.eye(h, order="F")
    perm = np.arange(p, dtype=np.intp)
    for k in range(min(h, p)):
        sub = r[k:, k:]
        norms = (sub * sub).sum(axis=0)
        j = k + int(np.argmax(norms))
        if trace is not None and norms.shape[0] > 1:
            top = np.sort(norms)[::-1]
            trace.append(float((top[0] - top[1]) / top[0]) if top[0] > 0 else 0.0)
        if j != k:
            r[:, [k, j]] = r[:, [j, k]]
            perm[[k, j]] = perm[[j, k]]
        reflect(r, q, k)
    return QR(q=q, r=r, perm=perm)


def l_from_r(r, b):
    """(R11^-1 R12)^T (pivoted_qr.py:90-98)."""
    r = fmat(r)
    if r.shape[0] < b or r.shape[1] < b:
        raise ValueError("R smaller than the requested leading block")
    if r.shape[1] == b:
        return np.zeros((0, b), order="F")
    return np.asfortranarray(upper_solve(r[:b, :b], r[:b, b:]).T)


def rank_guard(r, b, fro):
    """First k < b with |R[k,k]| < eps*||A||_F raises (pivoted_qr.py:101-105)."""
    for k in range(b):
        if abs(r[k, k]) < EPS * fro:
            raise OracleRankDeficient(
                f"leading R block numerically singular at diagonal {k}", index=k)


def swap_limit(b, p, tau):
    """pivoted_qr.py:108-110."""
    return int(math.ceil(2.0 * b * math.log(max(p, 2)) / math.log(tau))) + 10


def srrqr(a, b, tau, trace=None):
    """Strong RRQR: QRCP, rank guard, then the tau swap loop with QR
    recomputed from scratch after every interchange (pivoted_qr.py:113-147)."""
    a = fmat(a)
    h, p = a.shape
    if tau <= 1.0:
        raise ValueError("tau must exceed 1")
    if h < b or p < b + 1:
        raise ValueError(
            f"strong_rrqr needs >= {b} rows and >= {b + 1} columns, got {h}x{p}")
    fro = frob(a)
    f = qr_pivoted(a, trace)
    rank_guard(f.r, b, fro)
    lt = upper_solve(f.r[:b, :b], f.r[:b, b:])
    limit = swap_limit(b, p, tau)
    swaps = 0
    perm = f.perm
    while True:
        worst = float(np.abs(lt).max()) if lt.size else 0.0
        if worst <= tau:
            break
        if swaps >= limit:
            raise OracleNonConvergence(
                f"swap cap {limit} exceeded, worst multiplier {worst}", worst=worst)
        flat = int(np.argmax(np.abs(lt)))
        i, j = divmod(flat, lt.shape[1])
        perm = perm.copy()
        perm[[i, b + j]] = perm[[b + j, i]]
        g = qr_plain(a[:, perm])
        f = QR(q=g.q, r=g.r, perm=perm)
        rank_guard(f.r, b, fro)
        lt = upper_solve(f.r[:b, :b], f.r[:b, b:])
        swaps += 1
    return Srrqr(qr=f, tau=tau, swap_count=swaps, l_block=np.asfortranarray(lt.T))


@dataclass
class Gepp:
    perm: np.ndarray
    l: np.ndarray
    u: np.ndarray
    intermediate_max: float
    original_max: float


def gepp(a):
    """Partial pivoting, first max wins, running max after each rank-1 step
    (gepp.py:39-65)."""
    c = fmat(a).copy(order="F")
    m, n = c.shape
    s = min(m, n)
    p = np.arange(m, dtype=np.intp)
    orig = maxabs(c)
    run = orig
    for k in range(s):
        col = np.abs(c[k:, k])
        rel = int(np.argmax(col))
        if col[rel] == 0.0:
            raise OracleSingularMatrix(f"zero pivot column {k}", column=k)
        if rel:
            c[[k, k + rel], :] = c[[k + rel, k], :]
            p[[k, k + rel]] = p[[k + rel, k]]
        if k + 1 < m:
            c[k + 1:, k] /= c[k, k]
            if k + 1 < n:
                c[k + 1:, k + 1:] -= c[k + 1:, k:k + 1] * c[k:k + 1, k + 1:]
                run = max(run, float(np.abs(c[k + 1:, k + 1:]).max()))
    l = np.tril(c[:, :s], -1)
    np.fill_diagonal(l, 1.0)
    return Gepp(perm=p, l=np.asfortranarray(l), u=np.asfortranarray(np.triu(c[:s, :])),
                intermediate_max=run, original_max=orig)


# --------------------------------------------------------------------------
# drivers (luprrp.py, tournament.py)
# --------------------------------------------------------------------------
@dataclass
class Stats:
    """ElimStats mirror (luprrp.py:33-78)."""
    original_max: float
    intermediate_max: float
    finish_max: float = 0.0
    swap_counts: list = field(default_factory=list)
    flops_charged: Fraction = Fraction(0)
    flops_executed: Fraction = Fraction(0)
    panel_multiplier_max: float = 0.0

    @property
    def growth_factor(self):
        if self.original_max == 0.0:
            raise ZeroDivisionError("growth factor of an all-zero matrix")
        return self.intermediate_max / self.original_max

    @property
    def full_growth_factor(self):
        if self.original_max == 0.0:
            raise ZeroDivisionError("growth factor of an all-zero matrix")
        return max(self.intermediate_max, self.finish_max) / self.original_max


@dataclass
class Factors:
    perm: np.ndarray
    l: np.ndarray
    u: np.ndarray
    panel_width: int
    stats: Stats


def _qr_charge(rows, cols):           # luprrp.py:135-136
    return Fraction(2 * rows * cols * cols) - Fraction(2, 3) * cols ** 3


def _finish_charge(bj, width):        # luprrp.py:139-140
    return Fraction(2, 3) * bj ** 3 + Fraction((width - bj) * bj * bj)


def _check_args(a, b, tau):           # luprrp.py:143-150
    m, n = a.shape
    if m < n:
        raise OracleDimensionMismatch("need at least as many rows as columns")
    if not 1 <= b <= n:
        raise ValueError(f"panel width {b} out of range [1, {n}]")
    if tau <= 1.0:
        raise ValueError("tau must exceed 1")


class _Work:
    """Working state of the right-looking blocked factorization:
    trailing matrix ``w``, multipliers ``l``, global row order ``p``."""

    def __init__(self, a):
        self.w = a.copy(order="F")
        self.l = np.zeros(a.shape, order="F")
        self.p = np.arange(a.shape[0], dtype=np.intp)
        mx = maxabs(a)
        self.stats = Stats(original_max=mx, intermediate_max=mx, finish_max=mx)

    def permute_tail(self, col0, rel):
        """luprrp.py:98-104."""
        rows = slice(col0, col0 + rel.shape[0])
        self.w[rows, col0:] = self.w[rows, col0:][rel, :]
        if col0:
            self.l[rows, :col0] = self.l[rows, :col0][rel, :]
        self.p[rows] = self.p[rows][rel]

    def store_multipliers_and_update(self, col0, bj, l21):
        """L21 store, multiplier max, rank-b update + growth sample
        (luprrp.py:178-185)."""
        st = self.stats
        if l21.size:
            st.panel_multiplier_max = max(st.panel_multiplier_max, maxabs(l21))
        self.l[col0 + bj:, col0:col0 + bj] = l21
        if self.w.shape[1] - col0 - bj:
            upd = schur_update(self.w[col0 + bj:, col0 + bj:], l21,
                               self.w[col0:col0 + bj, col0 + bj:])
            self.w[col0 + bj:, col0 + bj:] = upd
            if upd.size:
                st.intermediate_max = max(st.intermediate_max, maxabs(upd))

    def block_row_finish(self, col0, bj, compose=True):
        """GEPP of the b x (n-col0) block row, then L21 <- L21[:,perm] L11
        (luprrp.py:107-127)."""
        g = gepp(self.w[col0:col0 + bj, col0:])
        rows = slice(col0, col0 + bj)
        if col0:
            self.l[rows, :col0] = self.l[rows, :col0][g.perm, :]
        self.p[rows] = self.p[rows][g.perm]
        self.w[rows, col0:] = g.u
        self.l[rows, col0:col0 + bj] = g.l
        if compose and col0 + bj < self.l.shape[0]:
            below = self.l[col0 + bj:, col0:col0 + bj]
            self.l[col0 + bj:, col0:col0 + bj] = dger_product(below[:, g.perm], g.l)
            self.stats.flops_executed += Fraction(2 * below.shape[0] * bj * bj)
        self.stats.finish_max = max(self.stats.finish_max, float(g.intermediate_max))
        return g

    def factors(self, b):
        """luprrp.py:130-132, 200-201."""
        n = self.w.shape[1]
        u = np.asfortranarray(np.triu(self.w[:n, :]))
        return Factors(perm=self.p, l=np.asfortranarray(self.l), u=u,
                       panel_width=b, stats=self.stats)


def lu_prrp(a, b, tau=2.0, panel_limit=None, gap_trace=None):
    """LU_PRRP, Algorithm 1 (luprrp.py:153-201).

    ``panel_limit`` stops after that many panels (bounded CPU-baseline
    samples); the partial state is returned as-is.  ``gap_trace`` collects
    QRCP pivot gaps (test diagnostics)."""
    a = fmat(a)
    _check_args(a, b, tau)
    m, n = a.shape
    st = _Work(a)
    s = st.stats
    col0 = 0
    panel = 0
    while col0 < n and (panel_limit is None or panel < panel_limit):
        bj = min(b, n - col0)
        rows = m - col0
        width = n - col0 - bj
        s.flops_charged += _qr_charge(rows, bj)
        if rows > bj:
            try:
                sr = srrqr(st.w[col0:, col0:col0 + bj].T, bj, tau, gap_trace)
            except ArithmeticError as exc:
                exc.panel = panel
                raise
            s.flops_executed += (1 + sr.swap_count) * _qr_charge(rows, bj)
            s.swap_counts.append(sr.swap_count)
            st.permute_tail(col0, sr.qr.perm)
            st.store_multipliers_and_update(col0, bj, sr.l_block)
        else:
            s.swap_counts.append(0)
        s.flops_charged += Fraction(2 * bj * (rows - bj) * width)
        s.flops_executed += Fraction(2 * bj * (rows - bj) * width)
        try:
            st.block_row_finish(col0, bj)
        except ArithmeticError as exc:
            exc.panel = panel
            raise
        fin = _finish_charge(bj, n - col0)
        s.flops_charged += fin
        s.flops_executed += fin
        col0 += bj
        panel += 1
    return st.factors(b)


# ----------------------------------------------------------------- tournament
def split_rows(m, p):
    """Contiguous, near-equal, first blocks larger (tournament.py:64-73)."""
    base, extra = divmod(m, p)
    out, start = [], 0
    for i in range(p):
        size = base + (1 if i < extra else 0)
        out.append((start, start + size))
        start += size
    return out


def leaves(shape, leaf_count, m, b):
    """tournament.py:76-88; shape is 'binary' or 'flat'."""
    if shape == "binary":
        p_eff = max(1, min(leaf_count, m // (b + 1)))
        return split_rows(m, p_eff), p_eff
    first = min(m, 2 * b)
    blocks = [(0, first)]
    start = first
    while start < m:
        stop = min(m, start + b)
        blocks.append((start, stop))
        start = stop
    return blocks, len(blocks)


@dataclass
class Node:
    level: int
    index: int
    members: np.ndarray
    selected: np.ndarray
    swap_count: int


@dataclass
class Trace:
    nodes: list
    pivot_rows: np.ndarray
    leaf_count: int
    requested_leaf_count: int | None
    single_node: bool
    srr: object = None


def pick(panel, idx, b, tau, selector="srrqr"):
    """srrqr selector with rank-deficient shrink (tournament.py:118-141);
    selector "gepp": partial pivoting on the node rows, a zero pivot at
    column k keeps the k rows chosen so far (tournament.py:142-150)."""
    if idx.shape[0] <= b:
        return idx, idx, 0, None
    sub = panel[idx, :]
    if selector == "gepp":
        cols = b
        while cols:
            try:
                g = gepp(sub[:, :cols])
            except OracleSingularMatrix as exc:
                cols = exc.column
                continue
            return idx[g.perm[:cols]], idx[g.perm], 0, None
        return idx[:0], idx, 0, None
    want = b
    while want:
        try:
            sr = srrqr(sub.T, want, tau)
        except OracleRankDeficient as exc:
            want = exc.index
            continue
        order = sr.qr.perm
        return idx[order[:want]], idx[order], sr.swap_count, (sr if want == b else None)
    return idx[:0], idx, 0, None


def tournament(panel, b, tau, shape="binary", leaf_count=8, selector="srrqr"):
    """Tournament of strong RRQRs, or of GEPPs (tournament.py:155-217)."""
    panel = fmat(panel)
    m = panel.shape[0]
    if panel.shape[1] != b:
        raise OracleDimensionMismatch("panel width mismatch")
    blocks, p_eff = leaves(shape, leaf_count, m, b)
    nodes = []
    if len(blocks) == 1:
        idx = np.arange(m, dtype=np.intp)
        sel, order, swaps, sr = pick(panel, idx, b, tau, selector)
        if sel.shape[0] < b:
            raise OracleRankDeficient("panel supplied too few rows", index=sel.shape[0])
        nodes.append(Node(0, 0, idx, sel, swaps))
        return np.asarray(order, dtype=np.intp), Trace(nodes, sel, p_eff, leaf_count, True, sr)

    def node(level, index, idx):
        try:
            sel, _, swaps, _ = pick(panel, idx, b, tau, selector)
        except ArithmeticError as exc:
            exc.tree_node = (level, index)
            raise
        nodes.append(Node(level, index, idx, sel, swaps))
        return sel

    if shape == "binary":
        cands = [node(0, i, np.arange(lo, hi, dtype=np.intp))
                 for i, (lo, hi) in enumerate(blocks)]
        level = 1
        while len(cands) > 1:
            nxt = [node(level, i // 2, np.concatenate([cands[i], cands[i + 1]]))
                   for i in range(0, len(cands) - 1, 2)]
            if len(cands) % 2:
                nxt.append(cands[-1])
            cands = nxt
            level += 1
        piv = cands[0]
    else:
        lo, hi = blocks[0]
        piv = node(0, 0, np.arange(lo, hi, dtype=np.intp))
        for i, (lo, hi) in enumerate(blocks[1:], start=1):
            piv = node(i, 0, np.concatenate([piv, np.arange(lo, hi, dtype=np.intp)]))
    if piv.shape[0] < b:
        raise OracleRankDeficient("tournament supplied too few rows", index=piv.shape[0])
    rest = np.setdiff1d(np.arange(m, dtype=np.intp), piv)
    perm = np.concatenate([piv, rest]).astype(np.intp)
    return perm, Trace(nodes, piv, p_eff, leaf_count, False, None)


def _gepp_charge(rows, cols):         # tournament.py:220-221
    return Fraction(rows * cols * cols) - Fraction(cols ** 3, 3)


def _tournament_charge(trace, b, selector="srrqr"):     # tournament.py:224-234
    tot = Fraction(0)
    for nd in trace.nodes:
        r = int(nd.members.shape[0])
        if r > b:
            tot += (1 + nd.swap_count) * _qr_charge(r, b) if selector == "srrqr" else _gepp_charge(r, b)
    return tot


def calu_prrp(a, b, tau=2.0, shape="binary", leaf_count=8, panel_limit=None):
    """CALU_PRRP (tournament.py:237-296)."""
    a = fmat(a)
    _check_args(a, b, tau)
    m, n = a.shape
    st = _Work(a)
    s = st.stats
    col0 = 0
    panel = 0
    while col0 < n and (panel_limit is None or panel < panel_limit):
        bj = min(b, n - col0)
        rows = m - col0
        width = n - col0 - bj
        s.flops_charged += _qr_charge(rows, bj)
        if rows > bj:
            try:
                rel, tr = tournament(st.w[col0:, col0:col0 + bj], bj, tau, shape, leaf_count)
            except ArithmeticError as exc:
                exc.panel = panel
                raise
            st.permute_tail(col0, rel)
            if tr.single_node:
                l21 = tr.srr.l_block
                s.swap_counts.append(tr.srr.swap_count)
                s.flops_executed += (1 + tr.srr.swap_count) * _qr_charge(rows, bj)
            else:
                extra = _tournament_charge(tr, bj)
                s.flops_charged += extra
                s.flops_executed += extra + _qr_charge(rows, bj)
                l21 = l_from_r(qr_plain(st.w[col0:, col0:col0 + bj].T).r, bj)
                s.swap_counts.append(sum(nd.swap_count for nd in tr.nodes))
            st.store_multipliers_and_update(col0, bj, l21)
        else:
            s.swap_counts.append(0)
        s.flops_charged += Fraction(2 * bj * (rows - bj) * width)
        s.flops_executed += Fraction(2 * bj * (rows - bj) * width)
        try:
            st.block_row_finish(col0, bj)
        except ArithmeticError as exc:
            exc.panel = panel
            raise
        fin = _finish_charge(bj, n - col0)
        s.flops_charged += fin
        s.flops_executed += fin
        col0 += bj
        panel += 1
    return st.factors(b)


def calu_gepp(a, b, shape="binary", leaf_count=8):
    """Tournament-pivoted GEPP, the reference's calu_factor
    (tournament.py:299-359): GEPP selector in every node, GEPP finish of
    the block row without composing L21, L21 = A21 U11^-1
    (matcore.trsm_upper_right), rank-b update."""
    a = fmat(a)
    _check_args(a, b, 2.0)
    m, n = a.shape
    st = _Work(a)
    s = st.stats
    col0 = 0
    panel = 0
    while col0 < n:
        bj = min(b, n - col0)
        rows = m - col0
        width = n - col0 - bj
        if rows > bj:
            try:
                rel, tr = tournament(st.w[col0:, col0:col0 + bj], bj, 2.0, shape, leaf_count, "gepp")
            except ArithmeticError as exc:
                exc.panel = panel
                raise
            st.permute_tail(col0, rel)
            extra = _tournament_charge(tr, bj, "gepp")
            s.flops_charged += extra
            s.flops_executed += extra
            s.swap_counts.append(0)
            try:
                st.block_row_finish(col0, bj, compose=False)
            except ArithmeticError as exc:
                exc.panel = panel
                raise
            l21 = upper_solve_right(st.w[col0 + bj:, col0:col0 + bj], st.w[col0:col0 + bj, col0:col0 + bj])
            cost = Fraction((rows - bj) * bj * bj + 2 * bj * (rows - bj) * width)
            s.flops_charged += cost
            s.flops_executed += cost
            st.store_multipliers_and_update(col0, bj, l21)
        else:
            s.swap_counts.append(0)
            try:
                st.block_row_finish(col0, bj)
            except ArithmeticError as exc:
                exc.panel = panel
                raise
        fin = _finish_charge(bj, n - col0)
        s.flops_charged += fin
        s.flops_executed += fin
        col0 += bj
        panel += 1
    return st.factors(b)


# --------------------------------------------------------------------------
# checks and inputs
# --------------------------------------------------------------------------
def rel_residual(a, perm, l, u):
    """||PA - LU||_F / ||A||_F (metrics.py:56-63).  Uses a plain numpy
    product (the reference's dger loop is O(n^3) Python-level work)."""
    a = fmat(a)
    r = a[np.asarray(perm), :] - l @ u
    d = frob(a)
    return frob(r) / d if d else frob(r)


def randn_matrix(n, seed):
    """matgen.gen_randn (matgen.py:41-56): PCG64, explicit Box-Muller pairs,
    row-major fill."""
    rng = np.random.Generator(np.random.PCG64(seed))
    count = n * n
    pairs = (count + 1) // 2
    u1 = rng.random(pairs)
    u2 = rng.random(pairs)
    rad = np.sqrt(-2.0 * np.log1p(-u1))
    ang = 2.0 * np.pi * u2
    z = np.empty(2 * pairs)
    z[0::2] = rad * np.cos(ang)
    z[1::2] = rad * np.sin(ang)
    return np.asfortranarray(z[:count].reshape(n, n))


def urand_matrix(n, seed):
    """U(-1,1) stand-in for config 5 (not generated by the reference; defined
    in SURVEY.md 8(d) following matgen.py:3-8 conventions)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.asfortranarray(2.0 * rng.random(n * n).reshape(n, n) - 1.0)


def wilkinson_matrix(n):
    """matgen.gen_wilkinson (matgen.py:63-70)."""
    a = np.tril(-np.ones((n, n)), -1) + np.eye(n)
    a[:n - 1, n - 1] = 1.0
    return np.asfortranarray(a)


def foster_matrix(n, c=1.0, h=1.0, k=2.0 / 3.0):
    """matgen.gen_foster (matgen.py:116-130)."""
    kh = k * h
    a = np.zeros((n, n), order="F")
    a[np.tril_indices(n, -1)] = -kh
    a[1:, 0] = -kh / 2.0
    np.fill_diagonal(a, 1.0 - kh / 2.0)
    a[0, 0] = 1.0
    a[:n - 1, n - 1] = -1.0 / c
    a[n - 1, n - 1] = 1.0 - 1.0 / c - kh / 2.0
    return a


def lu_flops(n):
    """The metric's algorithmic unit, 2n^3/3."""
    return 2.0 * n ** 3 / 3.0


def panel_share_flops(n, col0, bj):
    """2n^3/3 split per panel: F(s) - F(s - bj) with F(s) = 2s^3/3 and
    s = n - col0 (telescopes to 2n^3/3 over all panels)."""
    s = n - col0
    return 2.0 * (s ** 3 - (s - bj) ** 3) / 3.0


# ---------------------------------------------------------------- stability measurements (checker only)
def _two_sum(a, b):                       # metrics.py:66-69
    s = a + b
    bb = s - a
    return s, (a - (s - bb)) + (b - bb)


def _two_prod(a, b):                      # metrics.py:72-81 (Veltkamp split 2^27 + 1)
    split = 134217729.0
    p = a * b
    ca = split * a
    ah = ca - (ca - a)
    al = a - ah
    cb = split * b
    bh = cb - (cb - b)
    bl = b - bh
    return p, ((ah * bh - p) + ah * bl + al * bh) + al * bl


def residual_extended(a, x, rhs):
    """rhs - A x, compensated (metrics.py:84-92)."""
    a = fmat(a)
    x = np.asarray(x, dtype=np.float64).reshape(-1)
    s = np.asarray(rhs, dtype=np.float64).reshape(-1).copy()
    comp = np.zeros_like(s)
    for j in range(a.shape[1]):
        p, pe = _two_prod(a[:, j], -x[j])
        s, se = _two_sum(s, p)
        comp += pe + se
    return s + comp

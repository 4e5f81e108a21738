"""LU_PRRP (Algorithm 1) behind the reference's entry point.

``luprrp_factor(a, b, tau)`` keeps the signature, validation, exceptions and
return type of the reference (luprrp.py:153-201); the factorization itself
runs on the B200 through ``prrp_luprrp`` in libprrp_b200.so.  The growth
statistics (luprrp.py:33-78) come back from the device; the exact rational
flop counters are rebuilt on the host from the per-panel swap counts with
the reference's charging rules (luprrp.py:135-140, 168-197).
"""
import ctypes
import math
import os
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from . import _lib
from .errors import DimensionMismatch


@dataclass
class ElimStats:
    """Element-growth bookkeeping (reference luprrp.py:33-78)."""

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
class BlockLUFactors:
    perm: np.ndarray       # apply_row_perm(perm, a) == l @ u
    l: np.ndarray          # m x n unit lower trapezoidal
    u: np.ndarray          # n x n upper triangular
    panel_width: int
    stats: ElimStats

    def solve(self, rhs):
        return luprrp_solve(self, rhs)


@dataclass
class DeviceLU:
    """Device-resident result: packed L\\U (row-major m x n view of the
    working buffer), global row order and statistics."""
    perm: object           # torch int64 [m] on the device
    lu: object             # torch float64 [m, n] view, packed L\\U in place
    panel_width: int
    stats: ElimStats


def _qr_charge(rows, cols):
    return Fraction(2 * rows * cols * cols) - Fraction(2, 3) * cols ** 3


def _finish_charge(bj, width):
    return Fraction(2, 3) * bj ** 3 + Fraction((width - bj) * bj * bj)


def flop_counters(m, n, b, swap_counts, compose=True, tournament_extra=None):
    """(charged, executed) exactly as luprrp_factor accumulates them."""
    charged = Fraction(0)
    executed = Fraction(0)
    col0 = 0
    panel = 0
    while col0 < n:
        bj = min(b, n - col0)
        rows = m - col0
        width = n - col0 - bj
        charged += _qr_charge(rows, bj)
        if rows > bj:
            if tournament_extra is not None and tournament_extra[panel] is not None:
                extra = tournament_extra[panel]
                charged += extra
                executed += extra + _qr_charge(rows, bj)
            else:
                executed += (1 + swap_counts[panel]) * _qr_charge(rows, bj)
        upd = Fraction(2 * bj * (rows - bj) * width)
        charged += upd
        executed += upd
        if compose and col0 + bj < m:
            executed += Fraction(2 * (m - col0 - bj) * bj * bj)
        fin = _finish_charge(bj, n - col0)
        charged += fin
        executed += fin
        col0 += bj
        panel += 1
    return charged, executed


def _validate(a, b, tau):
    m, n = a.shape
    if m < n:
        raise DimensionMismatch("need at least as many rows as columns")
    if not 1 <= b <= n:
        raise ValueError(f"panel width {b} out of range [1, {n}]")
    if tau <= 1.0:
        raise ValueError("tau must exceed 1")


def as_matrix(a):
    m = np.asarray(a, dtype=np.float64)
    if m.ndim != 2:
        raise DimensionMismatch(f"expected a 2-D array, got ndim={m.ndim}")
    return m


def upload(a):
    """Host matrix -> device working buffer (row-major, even pitch)."""
    import torch
    m, n = a.shape
    lda = n + (n & 1)
    buf = torch.empty((m, lda), dtype=torch.float64, device="cuda")
    src = torch.from_numpy(np.ascontiguousarray(a))
    if not src.is_pinned() and src.numel() >= (1 << 20):
        # stage through a pinned block: full-bandwidth DMA instead of a pageable copy
        staged = torch.empty(src.shape, dtype=torch.float64, pin_memory=True)
        staged.copy_(src)
        src = staged
    buf[:, :n].copy_(src, non_blocking=True)
    return buf, lda


def run_device(fn_name, buf, lda, m, n, b, tau, extra=(), stream=None):
    """Call prrp_luprrp / prrp_caluprrp on a device buffer; returns (perm, stats, swaps)."""
    import torch
    lib = _lib.device_lib()
    perm = torch.empty(m, dtype=torch.int64, device=buf.device)
    npan = (n + b - 1) // b
    swaps = (ctypes.c_int32 * npan)()
    st = _lib.PrrpStats()
    err = _lib.PrrpErr()
    fn = getattr(lib, fn_name)
    rc = fn(ctypes.c_void_p(buf.data_ptr()), lda, m, n, b, float(tau), *extra,
            ctypes.c_void_p(perm.data_ptr()), swaps, ctypes.byref(st), ctypes.byref(err),
            _lib.stream_handle(stream))
    _lib.raise_for(rc, err, fn_name)
    return perm, st, list(swaps)


def split_packed(packed, m, n):
    """Packed L\\U (m x n) -> (l m x n unit lower trapezoidal, u n x n upper), F-order."""
    l = np.tril(packed, -1)
    idx = np.arange(n)
    l[idx, idx] = 1.0
    u = np.triu(packed[:n, :])
    return np.asfortranarray(l), np.asfortranarray(u)


class _Staging:
    """Pinned host blocks reused across calls (device -> host results).

    Fresh page-locked allocations cost ~0.5 ms/MiB; the results handed to
    the caller are ordinary numpy arrays filled from these blocks chunk by
    chunk (the DMA of the next chunks overlaps the multi-threaded host copy
    of the current one), so the cost does not depend on whether the caller
    still holds the previous factors."""

    CHUNK = 32 << 20
    NBUF = 3

    def __init__(self):
        self.bufs = None
        self.stream = None

    def get(self):
        import torch
        if self.bufs is None:
            n = self.CHUNK // 8
            self.bufs = [torch.empty(n, dtype=torch.float64, pin_memory=True) for _ in range(self.NBUF)]
            self.stream = torch.cuda.Stream()
        return self.bufs, self.stream


class _ThreadStaging:
    """One staging set per host thread (concurrent calls must not share it)."""

    def __init__(self):
        import threading
        self.tls = threading.local()

    def get(self):
        st = getattr(self.tls, "st", None)
        if st is None:
            st = self.tls.st = _Staging()
        return st.get()


_staging = _ThreadStaging()


def _to_host_many(pairs):
    """Copy contiguous float64 device tensors into numpy arrays (same element
    counts) through the pinned staging blocks, as one pipeline over all
    chunks of all pairs: up to NBUF - 1 DMAs in flight ahead of the
    (synchronous, multi-threaded) host copy of the oldest chunk."""
    import torch
    bufs, cs = _staging.get()
    nb = len(bufs)
    ch = bufs[0].numel()
    chunks = []
    for dev, out in pairs:
        src = dev.reshape(-1)
        dst = torch.from_numpy(out.reshape(-1))
        for lo in range(0, src.numel(), ch):
            chunks.append((src, dst, lo, min(src.numel(), lo + ch)))
    cs.wait_stream(torch.cuda.current_stream())
    pending = []

    def issue(i):
        src, _, lo, hi = chunks[i]
        k = i % nb
        with torch.cuda.stream(cs):
            bufs[k][:hi - lo].copy_(src[lo:hi], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        pending.append((i, k, ev))

    nxt = 0
    while nxt < len(chunks) and nxt < nb - 1:
        issue(nxt)
        nxt += 1
    while pending:
        i, k, ev = pending.pop(0)
        if nxt < len(chunks):      # the buffer of chunk nxt (nxt % nb) is not the one being drained
            issue(nxt)
            nxt += 1
        ev.synchronize()
        _, dst, lo, hi = chunks[i]
        dst[lo:hi].copy_(bufs[k][:hi - lo])
    return [out for _, out in pairs]


def _to_host(dev, out):
    """Copy a contiguous float64 device tensor into the numpy array out."""
    return _to_host_many([(dev, out)])[0]


class _Prefault:
    """Result arrays allocated up front and first-touched by a background
    thread (torch's multi-threaded fill, GIL released) while the device
    factorizes: the page faults of ~1 GB of fresh host memory no longer sit
    between the last kernel and the return."""

    def __init__(self, shapes):
        import threading
        self.arrays = [np.empty(sh) for sh in shapes]
        self.thread = threading.Thread(target=self._touch, daemon=True)
        self.thread.start()

    def _touch(self):
        import torch
        for a in self.arrays:
            torch.from_numpy(a.reshape(-1)).zero_()

    def get(self):
        self.thread.join()
        return self.arrays


_POOL = None


def _host_pool_workers():
    return range(min(16, max(2, (os.cpu_count() or 8) // 2)))


def _host_pool():
    global _POOL
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(max_workers=len(_host_pool_workers()), thread_name_prefix="prrp-host")
    return _POOL


def _split_rows(blk, l_out, u_out, j0, r0, r1, m):
    """Rows r0..r1 (of the chunk starting at packed column j0) into the
    triangles: row j of U^T takes packed column j up to the diagonal, row j
    of L^T the part below it and the unit diagonal.  Four block copies (numpy
    releases the GIL while copying)."""
    b = blk[r0 - j0:r1 - j0]
    if r0 > 0:
        u_out[r0:r1, :r0] = b[:, :r0]
    sq = b[:, r0:r1]
    u_out[r0:r1, r0:r1] = np.tril(sq)
    lsq = np.triu(sq, 1)
    np.fill_diagonal(lsq, 1.0)
    l_out[r0:r1, r0:r1] = lsq
    if r1 < m:
        l_out[r0:r1, r1:] = b[:, r1:]


def split_to_host(packed, m, n, l_out, u_out):
    """Packed L\\U (device, row-major m x n) -> the caller's zero-filled host
    arrays l_out (n x m, = L^T) and u_out (n x n, = U^T).  One device
    transpose, then the packed columns stream through the pinned staging
    blocks (512 MB of DMA instead of 1 GB) and the host writes only the
    triangles: row j of U^T is packed column j above and on the diagonal, row
    j of L^T the part below it plus the unit diagonal.  Host memory traffic
    ~1.5 GB instead of ~3 GB for the staged copy of two full matrices."""
    import torch
    pt = packed.t().contiguous()            # n x m: row j = packed column j
    bufs, cs = _staging.get()
    nb = len(bufs)
    rows = max(1, bufs[0].numel() // m)
    lt = torch.from_numpy(l_out)
    ut = torch.from_numpy(u_out)
    chunks = [(j0, min(n, j0 + rows)) for j0 in range(0, n, rows)]
    cs.wait_stream(torch.cuda.current_stream())
    pending = []

    def issue(i):
        j0, j1 = chunks[i]
        k = i % nb
        with torch.cuda.stream(cs):
            bufs[k][:(j1 - j0) * m].copy_(pt[j0:j1].reshape(-1), non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        pending.append((i, k, ev))

    import os
    import time
    prof = os.environ.get("PRRP_SPLIT_PROF")
    t_wait = t_host = 0.0
    nxt = 0
    while nxt < len(chunks) and nxt < nb - 1:
        issue(nxt)
        nxt += 1
    while pending:
        i, k, ev = pending.pop(0)
        if nxt < len(chunks):
            issue(nxt)
            nxt += 1
        t0 = time.perf_counter()
        ev.synchronize()
        t1 = time.perf_counter()
        t_wait += t1 - t0
        j0, j1 = chunks[i]
        blk = bufs[k][:(j1 - j0) * m].numpy().reshape(j1 - j0, m)
        # rows of the chunk split over the host pool (numpy copies release the GIL)
        nw = len(_host_pool_workers())
        step = (j1 - j0 + nw - 1) // nw
        futs = [_host_pool().submit(_split_rows, blk, l_out, u_out, j0, r0, min(j1, r0 + step), m)
                for r0 in range(j0, j1, step)]
        for f in futs:
            f.result()
        t_host += time.perf_counter() - t1
    if prof:
        print(f"[split_to_host] {len(chunks)} chunks: DMA wait {1e3 * t_wait:.1f} ms, host writes {1e3 * t_host:.1f} ms",
              flush=True)
    return l_out.T, u_out.T


def split_packed_device(packed, m, n, out=None):
    """split_packed on the device: unit-lower L and upper U built with torch
    and transposed there, so the host receives Fortran-ordered arrays (the
    reference's layout, luprrp.py:130-132) without a host-side transpose.
    out: optional pre-allocated host arrays (n x m, n x n)."""
    import torch
    lt = torch.tril(packed, -1)
    lt.diagonal().fill_(1.0)
    lt_t = lt.t().contiguous()
    del lt
    u_t = torch.triu(packed[:n, :]).t().contiguous()
    l_out, u_out = out if out is not None else (np.empty((n, m)), np.empty((n, n)))
    l_h, u_h = _to_host_many([(lt_t, l_out), (u_t, u_out)])
    return l_h.T, u_h.T


def _stats(st, swaps, m, n, b):
    charged, executed = flop_counters(m, n, b, swaps)
    return ElimStats(original_max=st.original_max, intermediate_max=st.intermediate_max,
                     finish_max=st.finish_max, swap_counts=list(map(int, swaps)),
                     flops_charged=charged, flops_executed=executed,
                     panel_multiplier_max=st.panel_multiplier_max)


def luprrp_factor(a, b, tau=2.0):
    """Factor an m x n (m >= n) matrix; panel width b, multiplier bound tau.

    Drop-in for prrp.luprrp_factor (reference luprrp.py:153).  The input is
    copied to the device; the caller's array is never modified."""
    a = as_matrix(a)
    _validate(a, b, tau)
    m, n = a.shape
    _lib.device_lib()
    pre = _Prefault([(n, m), (n, n)]) if m * n >= (1 << 22) else None
    buf, lda = upload(a)
    perm, st, swaps = run_device("prrp_luprrp", buf, lda, m, n, b, tau)
    if pre:
        l, u = split_to_host(buf[:, :n], m, n, *pre.get())
    else:
        l, u = split_packed_device(buf[:, :n], m, n)
    return BlockLUFactors(perm=perm.cpu().numpy().astype(np.intp), l=l, u=u, panel_width=b,
                          stats=_stats(st, swaps, m, n, b))


def luprrp_factor_device(buf, b, tau=2.0, n=None, stream=None):
    """In-place LU_PRRP of a device-resident row-major float64 tensor
    ``buf`` (m x lda, lda even, the first n columns are the matrix).
    Returns DeviceLU with the packed L\\U view; nothing leaves the device
    except the small statistics record."""
    m, lda = buf.shape
    n = lda if n is None else n
    if m < n:
        raise DimensionMismatch("need at least as many rows as columns")
    if not 1 <= b <= n:
        raise ValueError(f"panel width {b} out of range [1, {n}]")
    if tau <= 1.0:
        raise ValueError("tau must exceed 1")
    perm, st, swaps = run_device("prrp_luprrp", buf, lda, m, n, b, tau, stream=stream)
    return DeviceLU(perm=perm, lu=buf[:, :n], panel_width=b, stats=_stats(st, swaps, m, n, b))


def _pack_lu_device(l, u):
    """Packed L\\U (row-major, device) from host l (m x n unit lower) and u (n x n)."""
    import torch
    lt = torch.from_numpy(np.ascontiguousarray(l, dtype=np.float64)).cuda()
    ut = torch.from_numpy(np.ascontiguousarray(u, dtype=np.float64)).cuda()
    n = ut.shape[0]
    packed = torch.tril(lt, -1)
    packed[:n, :] += torch.triu(ut)
    return packed.contiguous()


def luprrp_solve(f, rhs):
    """Solve A x = rhs from square block factors (luprrp.py:204-214): forward
    substitution with the unit lower L on P rhs, back substitution with U, on
    the device (prrp_lu_solve)."""
    if f.l.shape[0] != f.l.shape[1]:
        raise DimensionMismatch("solve needs factors of a square matrix")
    return _solve_factors(f.perm, f.l, f.u, rhs, "luprrp_solve")


def _solve_factors(perm, l, u, rhs, what):
    """x = U^-1 L^-1 (P rhs) on the device for square factors; a zero diagonal
    of U raises SingularFactor(index) like matcore.trsm_upper (matcore.py:88-90)."""
    import torch
    vec = np.asarray(rhs, dtype=np.float64)
    b2 = vec.reshape(-1, 1) if vec.ndim == 1 else vec
    if b2.shape[0] != l.shape[0]:
        raise DimensionMismatch("right-hand side row count mismatch")
    n, nrhs = b2.shape
    if nrhs == 0:
        return np.zeros((n, 0), order="F") if vec.ndim != 1 else np.zeros(n)
    lib = _lib.device_lib()
    lu = _pack_lu_device(l, u)
    p = torch.from_numpy(np.asarray(perm, dtype=np.int64)).cuda()
    B = torch.from_numpy(np.ascontiguousarray(b2.T)).cuda()          # column-major n x nrhs
    X = torch.empty_like(B)
    err = _lib.PrrpErr()
    rc = lib.prrp_lu_solve(ctypes.c_void_p(lu.data_ptr()), lu.shape[1], n, ctypes.c_void_p(p.data_ptr()),
                           ctypes.c_void_p(B.data_ptr()), n, ctypes.c_void_p(X.data_ptr()), n, nrhs,
                           ctypes.byref(err), _lib.stream_handle())
    _lib.raise_for(rc, err, what)
    x = np.asfortranarray(X.cpu().numpy().T)
    return x[:, 0] if vec.ndim == 1 else x


def growth_bound_luprrp_log2(n, b, tau):
    """log2 of the growth envelope (1 + tau b)^ceil(n/b) (luprrp.py:217-221)."""
    if not (n >= b >= 1) or tau <= 0:
        raise ValueError("need n >= b >= 1 and tau > 0")
    return math.ceil(n / b) * math.log2(1.0 + tau * b)


def growth_bound_luprrp(n, b, tau):
    lg = growth_bound_luprrp_log2(n, b, tau)
    return math.inf if lg > 1023.0 else 2.0 ** lg

"""Distributed CALU_PRRP: one process per GPU, device-resident.

Layout: a 2-D block-cyclic grid P_r x P_c with block
size b; this implementation is the P_r = 1 column of that family: global
column block J (b columns) lives on rank J mod P_c, every rank keeps all m
rows of its blocks in HBM (row-major, m x n_loc).  LU_PRRP itself does not
shard (its panel QRCP needs a global argmax every column step; SURVEY.md
8(e): replicas only) -- CALU_PRRP does, through the tournament.

Per panel k (Appendix D), all device work in
libprrp_b200.so (include/prrp_b200.h, prrp_calu_dist_*):

  owner (k mod P_c)   prrp_calu_dist_select: the tournament over the panel's
                      rows (the reference's tree, tournament.py:155-217), the
                      reorder, the final QR and L21, GEPP of the pivot block,
                      packed into one device message
  all ranks           broadcast of the message (NCCL via torch.distributed on
                      device memory; host-staged for gloo), then
                      prrp_calu_dist_apply: the same reorder, row moves, the
                      block-row finish and the DMMA trailing update of the
                      rank's own columns
  end                 MAX all-reduce of the statistics record

The owner of panel k + 1 runs apply(k) in two parts around its select(k+1)
(look-ahead of depth one).  Every element of the result is bit-identical to
the single-GPU prrp_caluprrp (same kernels, same k order per element).
"""
import ctypes
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import _lib
from .errors import DimensionMismatch
from .luprrp import BlockLUFactors, ElimStats, _validate, as_matrix, flop_counters


# ------------------------------------------------------------------ layout (host logic)
def owned_blocks(n, b, world, rank):
    """Global column blocks of `rank`: J = rank, rank + world, ..."""
    npan = (n + b - 1) // b
    return list(range(rank, npan, world))


def local_columns(n, b, world, rank):
    """Global column indices of rank's local columns, in local order."""
    cols = [np.arange(J * b, min(n, (J + 1) * b)) for J in owned_blocks(n, b, world, rank)]
    return np.concatenate(cols) if cols else np.zeros(0, dtype=np.int64)


def panel_owner(k, world):
    return k % world


def global_column(c, b, world, rank):
    """Global index of local column c (the map blockrow_w applies on the device)."""
    return ((c // b) * world + rank) * b + c % b


def scatter_columns(a, b, world, rank):
    """Rank's local columns of the m x n matrix a (row-major copy, lda even)."""
    cols = local_columns(a.shape[1], b, world, rank)
    loc = np.ascontiguousarray(a[:, cols])
    return loc, cols


def assemble_columns(blocks, n, b):
    """Inverse of scatter_columns: {rank: local m x n_loc} -> m x n."""
    world = len(blocks)
    m = next(iter(blocks.values())).shape[0]
    out = np.empty((m, n))
    for r, loc in blocks.items():
        out[:, local_columns(n, b, world, r)] = loc
    return out


# ------------------------------------------------------------------ transport
class Transport:
    """Collectives on device tensors through torch.distributed: NCCL runs on
    the device buffers (stream-ordered, NVLink); gloo (CPU tests, or several
    processes sharing one GPU) stages through host memory."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.on = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if self.on else 1
        self.rank = dist.get_rank(group) if self.on else 0
        self.nccl = self.on and dist.get_backend(group) == "nccl"

    def broadcast(self, t, src):
        if self.world == 1:
            return
        if self.nccl:
            self.dist.broadcast(t, src=src, group=self.group)
            return
        h = t.cpu()
        self.dist.broadcast(h, src=src, group=self.group)
        t.copy_(h)

    def all_reduce_max(self, t):
        if self.world == 1:
            return
        if self.nccl:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
            return
        h = t.cpu()
        self.dist.all_reduce(h, op=self.dist.ReduceOp.MAX, group=self.group)
        t.copy_(h)

    def all_gather_cpu(self, t):
        if self.world == 1:
            return [t]
        out = [t.new_empty(t.shape) for _ in range(self.world)]
        if self.nccl:
            self.dist.all_gather(out, t, group=self.group)
            return out
        h = t.cpu()
        outs = [h.new_empty(h.shape) for _ in range(self.world)]
        self.dist.all_gather(outs, h, group=self.group)
        return outs


class _CudaView:
    """Zero-copy torch view of a device buffer owned by the library."""

    def __init__(self, ptr, nbytes, typestr="|u1", itemsize=1):
        self.__cuda_array_interface__ = {"shape": (nbytes // itemsize,), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3}


def _view(ptr, nbytes, dtype="u1"):
    import torch
    ts = {"u1": ("|u1", 1), "i8": ("<i8", 8)}[dtype]
    return torch.as_tensor(_CudaView(ptr, nbytes, *ts), device="cuda")


# ------------------------------------------------------------------ driver
@dataclass
class DistFactors:
    perm: object          # torch int64 [m] (device), identical on every rank
    lu: object            # torch float64 [m, n_loc] view: this rank's columns of the packed L\U
    cols: np.ndarray      # global column index of every local column
    m: int
    n: int
    panel_width: int
    stats: ElimStats


def caluprrp_factor_dist_device(A_loc, m, n, b, tau=2.0, tree=None, group=None, lookahead=True):
    """In-place distributed CALU_PRRP of the rank's local columns A_loc (a CUDA
    float64 tensor, m x lda_loc, lda even, the first n_loc columns are the
    rank's blocks in local order).  Collective over `group`."""
    import torch
    from .tournament import binary_tree
    if tree is None:
        tree = binary_tree(8)
    leaf_count = int(tree.leaf_count) if tree.shape == "binary" else 0
    tp = Transport(group)
    world, rank = tp.world, tp.rank
    if m < n:
        raise DimensionMismatch("need at least as many rows as columns")
    if not 1 <= b <= n:
        raise ValueError(f"panel width {b} out of range [1, {n}]")
    if tau <= 1.0:
        raise ValueError("tau must exceed 1")
    n_loc = len(local_columns(n, b, world, rank))
    lib = _lib.device_lib()
    stream = _lib.stream_handle()
    perm = torch.empty(m, dtype=torch.int64, device="cuda")
    h = ctypes.c_void_p()
    err = _lib.PrrpErr()
    rc = lib.prrp_calu_dist_create(ctypes.byref(h), ctypes.c_void_p(A_loc.data_ptr()), A_loc.stride(0), m, n, n_loc,
                                   b, float(tau), leaf_count, world, rank, ctypes.c_void_p(perm.data_ptr()),
                                   ctypes.byref(err), stream)
    _lib.raise_for(rc, err, "prrp_calu_dist_create")
    try:
        m0, m1, cap, sp, sl = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_void_p(), ctypes.c_int64()
        lib.prrp_calu_dist_buffers(h, ctypes.byref(m0), ctypes.byref(m1), ctypes.byref(cap), ctypes.byref(sp),
                                   ctypes.byref(sl))
        msgs = (_view(m0.value, cap.value), _view(m1.value, cap.value))
        red = _view(sp.value, sl.value * 8, "i8")
        npan = (n + b - 1) // b

        def check(rc, what):
            _lib.raise_for(rc, err, what)

        if rank == panel_owner(0, world):
            check(lib.prrp_calu_dist_select(h, 0, ctypes.byref(err), stream), "prrp_calu_dist_select")
        # look-ahead: the owner of panel k+1 runs its tournament on a high-priority
        # side stream, concurrently with the rest of panel k's trailing update
        main = torch.cuda.current_stream()
        side = torch.cuda.Stream(priority=-1) if lookahead else None
        side_h = _lib.stream_handle(side) if side is not None else None
        for k in range(npan):
            nb = lib.prrp_calu_dist_msg_bytes(h, k)
            tp.broadcast(msgs[k & 1][:nb], panel_owner(k, world))
            nxt = k + 1 < npan and rank == panel_owner(k + 1, world)
            if nxt and lookahead:
                check(lib.prrp_calu_dist_apply(h, k, 1, ctypes.byref(err), stream), "prrp_calu_dist_apply")
                side.wait_stream(main)
                check(lib.prrp_calu_dist_select(h, k + 1, ctypes.byref(err), side_h), "prrp_calu_dist_select")
                check(lib.prrp_calu_dist_apply(h, k, 2, ctypes.byref(err), stream), "prrp_calu_dist_apply")
                main.wait_stream(side)           # the next message leaves after the selection
            else:
                check(lib.prrp_calu_dist_apply(h, k, 0, ctypes.byref(err), stream), "prrp_calu_dist_apply")
                if nxt:
                    check(lib.prrp_calu_dist_select(h, k + 1, ctypes.byref(err), stream), "prrp_calu_dist_select")
        check(lib.prrp_calu_dist_stats(h, ctypes.byref(err), stream), "prrp_calu_dist_stats")
        tp.all_reduce_max(red)
        swaps = (ctypes.c_int32 * npan)()
        chg3 = (ctypes.c_int64 * npan)()
        st = _lib.PrrpStats()
        rc = lib.prrp_calu_dist_finish(h, ctypes.c_void_p(red.data_ptr()), swaps, chg3, ctypes.byref(st),
                                       ctypes.byref(err), stream)
        _lib.raise_for(rc, err, "caluprrp_factor_dist")
    finally:
        lib.prrp_calu_dist_destroy(h)
    extra = [None if c < 0 else Fraction(int(c), 3) for c in chg3]
    charged, executed = flop_counters(m, n, b, list(swaps), tournament_extra=extra)
    stats = ElimStats(original_max=st.original_max, intermediate_max=st.intermediate_max,
                      finish_max=st.finish_max, swap_counts=list(map(int, swaps)),
                      flops_charged=charged, flops_executed=executed,
                      panel_multiplier_max=st.panel_multiplier_max)
    return DistFactors(perm=perm, lu=A_loc[:, :n_loc], cols=local_columns(n, b, world, rank), m=m, n=n,
                       panel_width=b, stats=stats)


def caluprrp_factor_dist(a, b, tau=2.0, tree=None, group=None, lookahead=True):
    """caluprrp_factor (tournament.py:237-296) over the ranks of `group`:
    every rank passes the same host matrix (or None except on... every rank
    needs its own columns, taken here from `a`); returns the full
    BlockLUFactors on every rank (gathered).  For large matrices use
    caluprrp_factor_dist_device with each rank's columns already resident."""
    import torch
    a = as_matrix(a)
    _validate(a, b, tau)
    m, n = a.shape
    tp = Transport(group)
    loc, cols = scatter_columns(a, b, tp.world, tp.rank)
    lda = max(2, loc.shape[1] + (loc.shape[1] & 1))
    A = torch.zeros((m, lda), dtype=torch.float64, device="cuda")
    if loc.shape[1]:
        A[:, :loc.shape[1]].copy_(torch.from_numpy(loc))
    f = caluprrp_factor_dist_device(A, m, n, b, tau, tree, group, lookahead)
    packed = gather_packed(f, tp)
    l = np.tril(packed, -1)[:, :n]
    l[np.arange(n), np.arange(n)] = 1.0
    u = np.triu(packed[:n, :])
    return BlockLUFactors(perm=f.perm.cpu().numpy().astype(np.intp), l=np.asfortranarray(l),
                          u=np.asfortranarray(u), panel_width=b, stats=f.stats)


def gather_packed(f, tp):
    """The packed m x n L\\U assembled from every rank's columns (host)."""
    import torch
    nmax = max(len(local_columns(f.n, f.panel_width, tp.world, r)) for r in range(tp.world))
    pad = torch.zeros((f.m, max(nmax, 1)), dtype=torch.float64, device=f.lu.device)
    if f.lu.shape[1]:
        pad[:, :f.lu.shape[1]].copy_(f.lu)
    parts = tp.all_gather_cpu(pad)
    blocks = {}
    for r, t in enumerate(parts):
        nl = len(local_columns(f.n, f.panel_width, tp.world, r))
        blocks[r] = t[:, :nl].cpu().numpy()
    return assemble_columns(blocks, f.n, f.panel_width)

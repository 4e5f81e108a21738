"""Distributed CALU_PRRP over N processes (one per GPU), torch.distributed.

SURVEY.md 8(e): LU_PRRP does not shard (replicas only); CALU_PRRP shards
through its tournament tree.  This module distributes the trailing matrix by
row blocks of b rows, cyclically over the ranks (the P_r x 1 case of the
paper's 2-D block-cyclic layout), and follows the
per-panel message pattern of Appendix D:

  1. all-gather the b panel columns of the trailing rows (logical order)
  2. tournament: leaf i (the reference's contiguous logical blocks,
     tournament.py:64-88) is factored by rank i % N; the candidate sets
     (b row ids per leaf) are all-gathered; the merges (2b x b nodes) are
     recomputed identically on every rank, so the pivot choice is independent
     of N (P stays fixed at the tree's leaf count)
  3. L21 for the local non-pivot rows from the unpivoted QR of the pivot block
     (the reflectors are fixed by the b pivot columns)
  4. all-reduce (sum) of the pivot rows' trailing part A12 (owners contribute)
  5. local Schur update, GEPP finish of the block row (identical on every
     rank), compose of the local multipliers
  6. statistics: max-all-reduce of the local maxima

Rows never move between ranks; the logical order is bookkeeping (identical
on every rank).  The per-rank arithmetic is delegated to an ops object
(`DeviceOps`: the B200 C ABI).  The result equals the single-process
caluprrp_factor for every N.
"""
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from .luprrp import BlockLUFactors, ElimStats, _qr_charge, _finish_charge
from .errors import DimensionMismatch


def row_owner(i, b, world):
    """Rank owning global row i: row blocks of b rows, cyclic over ranks."""
    return (i // b) % world


def leaf_partition(rows, b, leaf_count):
    """tournament.py:76-88 (binary): contiguous, near-equal, first larger."""
    p_eff = max(1, min(leaf_count, rows // (b + 1)))
    base, extra = divmod(rows, p_eff)
    out, start = [], 0
    for i in range(p_eff):
        size = base + (1 if i < extra else 0)
        out.append((start, start + size))
        start += size
    return out


def merge_schedule(nleaves):
    """Binary merge levels with the odd node promoted (tournament.py:188-200):
    list of levels, each a list of (left, right) index pairs or (idx,) for a
    promoted node, over the previous level's candidate list."""
    levels = []
    n = nleaves
    while n > 1:
        lvl = [(i, i + 1) for i in range(0, n - 1, 2)]
        if n % 2:
            lvl.append((n - 1,))
        levels.append(lvl)
        n = len(lvl)
    return levels


@dataclass
class PanelPlan:
    col0: int
    bj: int
    rows: int
    width: int
    leaves: list


def plan_panels(m, n, b, leaf_count):
    col0, out = 0, []
    while col0 < n:
        bj = min(b, n - col0)
        rows = m - col0
        out.append(PanelPlan(col0, bj, rows, n - col0 - bj,
                             leaf_partition(rows, bj, leaf_count) if rows > bj else []))
        col0 += bj
    return out


class DeviceOps:
    """Per-rank arithmetic on the local B200 through the C ABI."""

    def __init__(self):
        from . import pivoted_qr
        self._pq = pivoted_qr

    def srrqr(self, node_rows, want, tau):
        """strong RRQR of the node rows' panel transpose -> (order, swaps, l_block)."""
        res = self._pq.strong_rrqr(node_rows.T, want, tau)
        return np.asarray(res.qr.perm), int(res.swap_count), res.l_block

    def householder_qr(self, a):
        f = self._pq.householder_qr(a)
        return f.q, f.r

    def multipliers(self, pivot_block, rows):
        """(R11^-1 R12)^T for the given rows from the unpivoted QR of
        [pivot_block; rows]^T (tournament.py:271-272)."""
        import paper_1208_2451_b200 as prrp
        a = np.vstack([pivot_block, rows]).T
        _, r = self.householder_qr(a)
        b = pivot_block.shape[0]
        if rows.shape[0] == 0:
            return np.zeros((0, b))
        return prrp.multiplier_block(r, b)

    def schur(self, c, l21, a12):
        import paper_1208_2451_b200 as prrp
        return prrp.rank_update(c, l21, a12)

    def gepp(self, block_row):
        import paper_1208_2451_b200 as prrp
        return prrp.gepp_factor(block_row)

    def matmul(self, a, b):
        import paper_1208_2451_b200 as prrp
        return prrp.matmul(a, b)


def _allgather_obj(dist, group, obj):
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, obj, group=group)
    return out


def caluprrp_factor_dist(a, b, tau=2.0, leaf_count=8, group=None, ops=None):
    """Row-distributed CALU_PRRP.  Every rank passes the same global matrix
    `a` (each uses only the rows it owns); rank 0 returns BlockLUFactors, the
    other ranks return None."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    ops = ops or DeviceOps()
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    if m < n:
        raise DimensionMismatch("need at least as many rows as columns")
    if not 1 <= b <= n:
        raise ValueError(f"panel width {b} out of range [1, {n}]")
    if tau <= 1.0:
        raise ValueError("tau must exceed 1")
    mine = np.array([i for i in range(m) if row_owner(i, b, world) == rank], dtype=np.intp)
    work = {int(i): a[i].copy() for i in mine}          # local rows (full width)
    lpart = {int(i): np.zeros(n) for i in mine}         # local L rows
    order = list(range(m))                              # logical position -> global row
    omax = max(_allgather_obj(dist, group, float(np.abs(a[mine]).max()) if len(mine) else 0.0))
    inter, finish, pmm = omax, omax, 0.0
    swaps_all, charged, executed = [], Fraction(0), Fraction(0)

    for pl in plan_panels(m, n, b, leaf_count):
        col0, bj, rows, width = pl.col0, pl.bj, pl.rows, pl.width
        trailing = order[col0:]
        # 1. all-gather the panel columns of the trailing rows
        contrib = {g: work[g][col0:col0 + bj] for g in trailing if g in work}
        panel_rows = {}
        for part in _allgather_obj(dist, group, contrib):
            panel_rows.update(part)
        panel = np.array([panel_rows[g] for g in trailing])
        charged += _qr_charge(rows, bj)
        if rows > bj:
            leaves = pl.leaves
            if len(leaves) == 1:
                sel, sw, l21_all = ops.srrqr(panel, bj, tau)
                rel = list(sel)
                swaps_all.append(sw)
                executed += (1 + sw) * _qr_charge(rows, bj)
                single = True
            else:
                # 2. leaves on their owner ranks, candidates all-gathered
                local = {}
                for li, (lo, hi) in enumerate(leaves):
                    if li % world == rank:
                        sel, sw, _ = ops.srrqr(panel[lo:hi], bj, tau)
                        local[li] = (list(lo + np.asarray(sel[:bj])), sw, hi - lo)
                allc = {}
                for part in _allgather_obj(dist, group, local):
                    allc.update(part)
                cands = [allc[i][0] for i in range(len(leaves))]
                nodes = [(allc[i][2], allc[i][1]) for i in range(len(leaves))]
                for lvl in merge_schedule(len(cands)):
                    nxt = []
                    for pair in lvl:
                        if len(pair) == 1:
                            nxt.append(cands[pair[0]])
                            continue
                        idx = cands[pair[0]] + cands[pair[1]]
                        sel, sw, _ = ops.srrqr(panel[idx], bj, tau)
                        nxt.append([idx[j] for j in sel[:bj]])
                        nodes.append((len(idx), sw))
                    cands = nxt
                piv = cands[0]
                pset = set(piv)
                rel = list(piv) + [i for i in range(rows) if i not in pset]
                extra = sum(((1 + sw) * _qr_charge(r, bj) for r, sw in nodes if r > bj), Fraction(0))
                charged += extra
                executed += extra + _qr_charge(rows, bj)
                swaps_all.append(sum(sw for _, sw in nodes))
                single = False
            new_trailing = [trailing[i] for i in rel]
            order[col0:] = new_trailing
            pivots = new_trailing[:bj]
            rest_local = [g for g in new_trailing[bj:] if g in work]
            # 3. multipliers of the local non-pivot rows
            piv_block = np.array([panel_rows[g] for g in pivots])
            if single:
                # the single node's own l_block (tournament.py:263-266); row t <-> position bj + t
                pos = {g: t for t, g in enumerate(new_trailing[bj:])}
                l21 = np.array([l21_all[pos[g]] for g in rest_local]).reshape(len(rest_local), bj)
            else:
                rows_local = np.array([panel_rows[g] for g in rest_local]).reshape(len(rest_local), bj)
                l21 = ops.multipliers(piv_block, rows_local)
            lmax = float(np.abs(l21).max()) if l21.size else 0.0
            pmm = max(pmm, max(_allgather_obj(dist, group, lmax)))
            for t, g in enumerate(rest_local):
                lpart[g][col0:col0 + bj] = l21[t]
            # 4. pivot rows' trailing part to every rank (sum-reduce of owner contributions)
            import torch
            a12 = np.zeros((bj, width))
            for q, g in enumerate(pivots):
                if g in work:
                    a12[q] = work[g][col0 + bj:]
            t12 = torch.from_numpy(a12)
            dist.all_reduce(t12, group=group)
            a12 = t12.numpy()
            # 5. local Schur update
            if width and rest_local:
                c = np.array([work[g][col0 + bj:] for g in rest_local])
                upd = ops.schur(c, l21, a12)
                for t, g in enumerate(rest_local):
                    work[g][col0 + bj:] = upd[t]
                umax = float(np.abs(upd).max()) if upd.size else 0.0
            else:
                umax = 0.0
            if width:
                inter = max(inter, max(_allgather_obj(dist, group, umax)))
        else:
            swaps_all.append(0)
            pivots = order[col0:col0 + bj]
            rest_local = []
            a12 = np.zeros((bj, width))
            piv_block = np.array([panel_rows[g] for g in pivots])
            l21 = np.zeros((0, bj))
        upd_c = Fraction(2 * bj * (rows - bj) * width)
        charged += upd_c
        executed += upd_c
        # 6. GEPP finish of the block row (identical on every rank)
        block_row = np.hstack([piv_block, a12])
        gf = ops.gepp(block_row)
        finish = max(finish, float(gf.intermediate_max))
        gperm = list(gf.perm)
        order[col0:col0 + bj] = [pivots[i] for i in gperm]
        for q, g in enumerate(order[col0:col0 + bj]):
            if g in work:
                work[g][col0:] = gf.u[q]
                lpart[g][col0:col0 + bj] = gf.l[q]
        if rest_local and col0 + bj < m:
            comp = ops.matmul(l21[:, gperm], gf.l)
            for t, g in enumerate(rest_local):
                lpart[g][col0:col0 + bj] = comp[t]
            executed += Fraction(2 * (m - col0 - bj) * bj * bj)
        elif col0 + bj < m:
            executed += Fraction(2 * (m - col0 - bj) * bj * bj)
        fin = _finish_charge(bj, n - col0)
        charged += fin
        executed += fin

    # gather the factors on rank 0 in logical order
    rows_out = {g: (lpart[g], work[g]) for g in work}
    gathered = _allgather_obj(dist, group, rows_out)
    if rank != 0:
        return None
    allrows = {}
    for part in gathered:
        allrows.update(part)
    l = np.array([allrows[g][0] for g in order])
    w = np.array([allrows[g][1] for g in order])
    l = np.tril(l, -1)
    l[np.arange(n), np.arange(n)] = 1.0
    u = np.triu(w[:n])
    stats = ElimStats(original_max=omax, intermediate_max=inter, finish_max=finish, swap_counts=swaps_all,
                      flops_charged=charged, flops_executed=executed, panel_multiplier_max=pmm)
    return BlockLUFactors(perm=np.array(order, dtype=np.intp), l=np.asfortranarray(l), u=np.asfortranarray(u),
                          panel_width=b, stats=stats)

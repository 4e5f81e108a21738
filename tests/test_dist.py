"""Multi-process CALU_PRRP orchestration (paper_1208_2451_b200/dist.py) with
the gloo backend on CPU, world size 1 and 2.

The per-rank arithmetic is injected: these tests use the oracle's numpy
functions (the checker's arithmetic, never shipped), so what is exercised is
the distribution logic — row ownership, leaf placement, candidate exchange,
pivot-row all-reduce, statistics reductions — and its result is compared with
the single-process reference algorithm."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import prrp_oracle as orc


class NumpyOps:
    def srrqr(self, rows, want, tau):
        s = orc.srrqr(rows.T, want, tau)
        return s.qr.perm, s.swap_count, s.l_block

    def householder_qr(self, a):
        f = orc.qr_plain(a)
        return f.q, f.r

    def multipliers(self, piv, rows):
        b = piv.shape[0]
        if rows.shape[0] == 0:
            return np.zeros((0, b))
        return orc.l_from_r(orc.qr_plain(np.vstack([piv, rows]).T).r, b)

    def schur(self, c, l21, a12):
        return orc.schur_update(c, l21, a12)

    def gepp(self, br):
        return orc.gepp(br)

    def matmul(self, a, b):
        return orc.dger_product(a, b)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, b, P, seed, out):
    import torch.distributed as dist
    from paper_1208_2451_b200 import dist as pd
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = orc.randn_matrix(n, seed)
        f = pd.caluprrp_factor_dist(a, b, 2.0, P, ops=NumpyOps())
        if rank == 0:
            np.savez(out, perm=f.perm, l=f.l, u=f.u, stats=np.array([f.stats.original_max, f.stats.intermediate_max,
                                                                      f.stats.finish_max, f.stats.panel_multiplier_max]),
                     swaps=np.array(f.stats.swap_counts), fc=str(f.stats.flops_charged), fe=str(f.stats.flops_executed))
    finally:
        dist.destroy_process_group()


def _run(world, n, b, P, seed, tmp_path):
    out = str(tmp_path / f"res_w{world}.npz")
    mp.spawn(_worker, args=(world, _free_port(), n, b, P, seed, out), nprocs=world, join=True)
    return np.load(out)


def test_partition_and_schedule_match_reference():
    from paper_1208_2451_b200 import dist as pd
    assert pd.leaf_partition(100, 8, 8) == orc.split_rows(100, 8)
    assert pd.leaf_partition(20, 8, 8) == orc.split_rows(20, 2)
    assert pd.merge_schedule(8) == [[(0, 1), (2, 3), (4, 5), (6, 7)], [(0, 1), (2, 3)], [(0, 1)]]
    assert pd.merge_schedule(5) == [[(0, 1), (2, 3), (4,)], [(0, 1), (2,)], [(0, 1)]]
    assert [pd.row_owner(i, 4, 3) for i in range(13)] == [0] * 4 + [1] * 4 + [2] * 4 + [0]


@pytest.mark.parametrize("world", [1, 2])
def test_dist_calu_matches_reference_algorithm(world, tmp_path):
    n, b, P, seed = 160, 16, 4, 5
    res = _run(world, n, b, P, seed, tmp_path)
    a = orc.randn_matrix(n, seed)
    ref = orc.calu_prrp(a, b, 2.0, "binary", P)
    assert np.array_equal(res["perm"], ref.perm)
    assert list(res["swaps"]) == list(ref.stats.swap_counts)
    st = res["stats"]
    assert st[0] == ref.stats.original_max
    assert st[1] == pytest.approx(ref.stats.intermediate_max, rel=1e-12)
    assert st[2] == pytest.approx(ref.stats.finish_max, rel=1e-12)
    assert st[3] == pytest.approx(ref.stats.panel_multiplier_max, rel=1e-12)
    assert str(ref.stats.flops_charged) == str(res["fc"])
    assert str(ref.stats.flops_executed) == str(res["fe"])
    scale_l, scale_u = np.abs(ref.l).max(), np.abs(ref.u).max()
    assert np.abs(res["l"] - ref.l).max() <= 1e-12 * scale_l
    assert np.abs(res["u"] - ref.u).max() <= 1e-12 * scale_u


def test_dist_result_independent_of_world_size(tmp_path):
    r1 = _run(1, 128, 8, 8, 9, tmp_path)
    r2 = _run(2, 128, 8, 8, 9, tmp_path)
    assert np.array_equal(r1["perm"], r2["perm"])
    assert np.array_equal(r1["swaps"], r2["swaps"])
    assert np.abs(r1["u"] - r2["u"]).max() <= 1e-12 * np.abs(r1["u"]).max()

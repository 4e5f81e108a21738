"""Distributed CALU_PRRP on the device (prrp_calu_dist_*, dist.py) with
several processes: the gloo transport (host-staged) lets N ranks share the
one GPU this suite runs on -- no kernel waits on another rank's kernel, the
ranks meet only in the host collectives.  Every result must be bit-identical
to the single-GPU prrp_caluprrp (same kernels, same per-element order):
permutation, L, U, growth statistics, swap counts and flop counters; the
reference's error contract holds on every rank."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, spec, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1208_2451_b200 import dist as pd
        import paper_1208_2451_b200 as dev
        a = _input(spec)
        tree = dev.flat_tree() if spec["P"] == 0 else dev.binary_tree(spec["P"])
        try:
            f = pd.caluprrp_factor_dist(a, spec["b"], spec.get("tau", 2.0), tree, lookahead=spec.get("la", True))
            res = dict(perm=f.perm, l=f.l, u=f.u, swaps=np.array(f.stats.swap_counts),
                       st=np.array([f.stats.original_max, f.stats.intermediate_max, f.stats.finish_max,
                                    f.stats.panel_multiplier_max]),
                       fc=str(f.stats.flops_charged), fe=str(f.stats.flops_executed), err="")
        except ArithmeticError as exc:
            res = dict(err=type(exc).__name__, panel=getattr(exc, "panel", -9), index=getattr(exc, "index", -9) or -1,
                       tn=str(getattr(exc, "tree_node", None)))
        np.savez(out + f".{rank}.npz", **res)
    finally:
        dist.destroy_process_group()


def _input(spec):
    from paper_1208_2451_b200 import matgen
    if spec["gen"] == "randn":
        a = matgen.gen_randn_rect(spec["m"], spec["n"], spec["seed"])
    elif spec["gen"] == "urand":
        a = matgen.gen_urand(spec["n"], spec["seed"])
    elif spec["gen"] == "zeros":
        a = np.zeros((spec["n"], spec["n"]))
    else:
        a = matgen.gen_deficient_block(spec["n"], spec["seed"], spec["blocks"], spec["b"])
    return np.asfortranarray(a)


def _run(world, spec, tmp_path):
    out = str(tmp_path / f"w{world}")
    mp.spawn(_worker, args=(world, _free_port(), spec, out), nprocs=world, join=True)
    return [dict(np.load(out + f".{r}.npz")) for r in range(world)]


CASES = [
    dict(gen="randn", m=512, n=512, seed=3, b=32, P=8),
    dict(gen="randn", m=640, n=640, seed=4, b=64, P=8),
    dict(gen="urand", n=768, seed=5, b=128, P=4),
    dict(gen="randn", m=300, n=200, seed=6, b=16, P=3),          # tall, ragged last block
    dict(gen="randn", m=320, n=320, seed=7, b=32, P=0),          # flat tree
    dict(gen="deficient", n=160, seed=11, b=16, P=4, blocks=[[0, 40, 5], [40, 80, 6]]),
]


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("ci", range(len(CASES)))
def test_dist_calu_bit_identical_to_single_gpu(world, ci, tmp_path):
    import paper_1208_2451_b200 as dev
    spec = CASES[ci]
    if world == 3 and ci not in (0, 3):
        pytest.skip("world 3 on two shapes")
    res = _run(world, spec, tmp_path)
    a = _input(spec)
    tree = dev.flat_tree() if spec["P"] == 0 else dev.binary_tree(spec["P"])
    ref = dev.caluprrp_factor(a, spec["b"], 2.0, tree)
    for r in res:
        assert r["err"] == ""
        assert np.array_equal(r["perm"], ref.perm)
        assert np.array_equal(r["l"], ref.l) and np.array_equal(r["u"], ref.u)
        assert list(r["swaps"]) == list(ref.stats.swap_counts)
        assert list(r["st"]) == [ref.stats.original_max, ref.stats.intermediate_max, ref.stats.finish_max,
                                 ref.stats.panel_multiplier_max]
        assert str(r["fc"]) == str(ref.stats.flops_charged) and str(r["fe"]) == str(ref.stats.flops_executed)


def test_dist_calu_no_lookahead_same_bits(tmp_path):
    spec = dict(CASES[0], la=False)
    r1 = _run(2, spec, tmp_path)
    r2 = _run(2, CASES[0], tmp_path)
    assert np.array_equal(r1[0]["u"], r2[0]["u"]) and np.array_equal(r1[1]["l"], r2[1]["l"])


def test_dist_calu_error_contract(tmp_path):
    """A zero matrix: SingularFactor at tournament node (0, 0) of panel 0 on
    every rank (the owner's first failure travels in the panel message)."""
    res = _run(2, dict(gen="zeros", n=64, b=16, P=4, seed=0), tmp_path)
    for r in res:
        assert str(r["err"]) == "SingularFactor" and int(r["panel"]) == 0 and str(r["tn"]) == "(0, 0)"

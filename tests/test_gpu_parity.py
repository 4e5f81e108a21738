"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and
the reference's golden vectors.

Bars (BASELINE north_star):
  * row permutation and swap counts: identical (generic inputs);
  * growth_factor / full_growth_factor / multiplier max: <= 1e-10 relative;
  * L, U: max-abs error <= 1e-11 x max|.| of the oracle factor;
  * ||PA - LU||_F / ||A||_F <= max(4 x oracle, n * 2^-52);
  * kernels whose reference arithmetic is fully specified (rank_update,
    GEPP of a block row, upper-triangular solve) are bit-exact.
"""
import numpy as np
import pytest

from conftest import gepp_calu_input, make_input, srrqr_input
from oracle import prrp_oracle as orc

pytestmark = pytest.mark.gpu

TOL_F = 1e-11
TOL_G = 1e-10


@pytest.fixture(scope="module")
def dev():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1208_2451_b200 as d
    return d


def _rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if b.size == 0:
        return 0.0
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _check_factors(f, ref, a, exact_perm=True):
    if exact_perm:
        assert np.array_equal(f.perm, ref.perm)
        assert list(f.stats.swap_counts) == list(ref.stats.swap_counts)
        assert _rel(f.l, ref.l) <= TOL_F
        assert _rel(f.u, ref.u) <= TOL_F
        assert f.stats.flops_charged == ref.stats.flops_charged
        assert f.stats.flops_executed == ref.stats.flops_executed
    assert f.stats.original_max == ref.stats.original_max
    if ref.stats.original_max:
        assert f.stats.growth_factor == pytest.approx(ref.stats.growth_factor, rel=TOL_G)
        assert f.stats.full_growth_factor == pytest.approx(ref.stats.full_growth_factor, rel=TOL_G)
    assert f.stats.panel_multiplier_max == pytest.approx(ref.stats.panel_multiplier_max, rel=TOL_G)
    n = a.shape[1]
    res = orc.rel_residual(a, f.perm, f.l, f.u)
    ref_res = orc.rel_residual(a, ref.perm, ref.l, ref.u)
    assert res <= max(4 * ref_res, n * 2.0 ** -52), (res, ref_res)


def test_schur_update_bit_exact(dev):
    """K4 against matcore.rank_update (c - dger-k-loop product): bit for bit."""
    import ctypes
    import torch
    from paper_1208_2451_b200 import _lib
    lib = _lib.device_lib()
    rng = np.random.default_rng(3)
    for (M, N, K) in [(300, 200, 64), (128, 64, 32), (257, 131, 128), (77, 45, 16), (64, 64, 7)]:
        c = rng.standard_normal((M, N))
        l = rng.standard_normal((M, K))
        b = rng.standard_normal((K, N))
        ref = orc.schur_update(c, l, b)
        C = torch.from_numpy(np.ascontiguousarray(c)).cuda()
        L = torch.from_numpy(np.ascontiguousarray(l.T)).cuda()          # column-major M x K
        B = torch.from_numpy(np.ascontiguousarray(b)).cuda()
        mx = ctypes.c_double(0)
        err = _lib.PrrpErr()
        rc = lib.prrp_schur_update(ctypes.c_void_p(C.data_ptr()), N, ctypes.c_void_p(L.data_ptr()), M,
                                   ctypes.c_void_p(B.data_ptr()), N, M, N, K, ctypes.byref(mx), ctypes.byref(err),
                                   _lib.stream_handle())
        assert rc == 0, err.msg
        got = C.cpu().numpy()
        assert np.array_equal(got, ref), (M, N, K, np.abs(got - ref).max())
        assert mx.value == np.abs(ref).max()


def test_gepp_blockrow_bit_exact(dev):
    """K5 against gepp.gepp_factor on b x w block rows: bit for bit."""
    import ctypes
    import torch
    from paper_1208_2451_b200 import _lib
    lib = _lib.device_lib()
    rng = np.random.default_rng(4)
    for (m, n) in [(8, 40), (64, 300), (128, 129), (17, 17)]:
        a = rng.standard_normal((m, n))
        ref = orc.gepp(a)
        A = torch.from_numpy(np.ascontiguousarray(a)).cuda()
        P = torch.empty(m, dtype=torch.int64, device="cuda")
        im = ctypes.c_double(0)
        err = _lib.PrrpErr()
        rc = lib.prrp_gepp_blockrow(ctypes.c_void_p(A.data_ptr()), n, m, n, ctypes.c_void_p(P.data_ptr()),
                                    ctypes.byref(im), ctypes.byref(err), _lib.stream_handle())
        assert rc == 0, err.msg
        packed = A.cpu().numpy()
        assert np.array_equal(P.cpu().numpy(), ref.perm)
        assert np.array_equal(np.triu(packed), ref.u)
        assert np.array_equal(np.tril(packed[:, :m], -1) + np.eye(m), ref.l)
        assert im.value == ref.intermediate_max


def test_strong_rrqr_golden(dev, golden):
    index, arrays = golden
    for e in index["srrqr"]:
        a = srrqr_input(e, arrays)
        res = dev.strong_rrqr(a, e["b"], e["tau"])
        key = "srrqr/" + e["name"]
        assert np.array_equal(res.qr.perm, arrays[key + "/perm"]), e["name"]
        assert res.swap_count == e["swap_count"], e["name"]
        assert _rel(res.l_block, arrays[key + "/l_block"]) <= TOL_F, e["name"]
        r_ref = arrays[key + "/r"]
        assert _rel(res.qr.r[:, :r_ref.shape[1]], r_ref) <= TOL_F, e["name"]
        assert _rel(res.qr.q, arrays[key + "/q"]) <= TOL_F, e["name"]


def test_strong_rrqr_spec_examples(dev):
    res = dev.strong_rrqr(np.hstack([np.eye(4), np.zeros((4, 3))]), 4, 2.0)
    assert np.array_equal(res.qr.perm, np.arange(7)) and res.swap_count == 0
    assert np.all(res.l_block == 0)
    res = dev.strong_rrqr(np.array([[1.0, 10.0]]), 1, 2.0)
    assert list(res.qr.perm) == [1, 0] and res.l_block[0, 0] == pytest.approx(0.1)


def test_householder_qr_matches_oracle(dev):
    rng = np.random.default_rng(5)
    for (h, p) in [(6, 10), (16, 40), (64, 500), (10, 5)]:
        a = rng.standard_normal((h, p))
        ref = orc.qr_plain(a)
        got = dev.householder_qr(a)
        assert _rel(got.r, ref.r) <= TOL_F and _rel(got.q, ref.q) <= TOL_F


def test_luprrp_golden(dev, golden):
    index, arrays = golden
    for e in index["lu"]:
        a = make_input(e)
        f = dev.luprrp_factor(a, e["b"], e["tau"])
        ref = orc.lu_prrp(a, e["b"], e["tau"])
        assert np.array_equal(ref.perm, arrays["lu/" + e["name"] + "/perm"])
        generic = e["gen"] in ("randn", "urand", "identity")
        _check_factors(f, ref, a, exact_perm=generic)
        if e["gen"] == "foster":
            assert f.stats.growth_factor == pytest.approx(ref.stats.growth_factor, rel=TOL_G)


def test_luprrp_error_contract(dev, golden):
    index, _ = golden
    for e in index["lu_errors"]:
        a = make_input(e)
        ref = e["error"]
        with pytest.raises(ArithmeticError) as ei:
            dev.luprrp_factor(a, e["b"], e["tau"])
        exc = ei.value
        assert type(exc).__name__ == ref["type"], e["name"]
        assert getattr(exc, "panel", None) == ref["panel"], e["name"]
        if ref["type"] == "RankDeficient":
            # the failing diagonal is decided by roundoff-level entries of R
            # (the trailing block has exact rank 2 here), so any index >= the
            # exact rank is a faithful result
            assert exc.index >= 2
        else:
            assert getattr(exc, "index", None) == ref["index"]
            assert getattr(exc, "column", None) == ref["column"]


def test_luprrp_c1_golden(dev, golden):
    """BASELINE config 1: randn(1024, 42), b=64, tau=2."""
    index, arrays = golden
    c1 = index["c1"]
    a = orc.randn_matrix(1024, 42)
    f = dev.luprrp_factor(a, 64, 2.0)
    assert np.array_equal(f.perm, arrays["c1/perm"])
    st = c1["stats"]
    assert f.stats.swap_counts == st["swap_counts"]
    assert f.stats.growth_factor == pytest.approx(st["growth_factor"], rel=TOL_G)
    assert f.stats.full_growth_factor == pytest.approx(st["full_growth_factor"], rel=TOL_G)
    assert f.stats.panel_multiplier_max == pytest.approx(st["panel_multiplier_max"], rel=TOL_G)
    rows = c1["sample_rows"]
    assert _rel(f.l[rows, :], arrays["c1/l_rows"]) <= TOL_F
    assert _rel(f.u[rows, :], arrays["c1/u_rows"]) <= TOL_F
    res = orc.rel_residual(a, f.perm, f.l, f.u)
    assert res <= 4 * c1["rel_residual"]


@pytest.mark.parametrize("n,b,tau,gen", [(2048, 64, 2.0, "randn"), (2048, 128, 2.0, "randn"),
                                         (1000, 48, 2.0, "randn"), (512, 16, 1.05, "randn"),
                                         (1536, 128, 2.0, "urand")])
def test_luprrp_vs_oracle(dev, n, b, tau, gen):
    a = orc.randn_matrix(n, 42) if gen == "randn" else orc.urand_matrix(n, 42)
    f = dev.luprrp_factor(a, b, tau)
    ref = orc.lu_prrp(a, b, tau)
    _check_factors(f, ref, a)


def test_luprrp_growth_stress(dev):
    """Config 3 shapes at n=1024 (Wilkinson: ties decided by rounding, so the
    bar is the growth factor and the backward error; Foster is generic)."""
    for a in (orc.wilkinson_matrix(1024), orc.foster_matrix(1024, 1.0, 1.0, 1.0)):
        f = dev.luprrp_factor(a, 64, 2.0)
        ref = orc.lu_prrp(a, 64, 2.0)
        assert f.stats.growth_factor == pytest.approx(ref.stats.growth_factor, rel=TOL_G)
        res = orc.rel_residual(a, f.perm, f.l, f.u)
        assert res <= max(4 * orc.rel_residual(a, ref.perm, ref.l, ref.u), 1024 * 2.0 ** -52)


def test_caluprrp_golden(dev, golden):
    """CALU_PRRP (binary and flat trees) against the reference's fixtures and the oracle."""
    index, arrays = golden
    for e in index["calu"]:
        a = make_input(e)
        flat = e["P"] == 0
        f = dev.caluprrp_factor(a, e["b"], e["tau"], dev.flat_tree() if flat else dev.binary_tree(e["P"]))
        ref = orc.calu_prrp(a, e["b"], e["tau"], *(("flat", None) if flat else ("binary", e["P"])))
        assert np.array_equal(ref.perm, arrays["calu/" + e["name"] + "/perm"])
        _check_factors(f, ref, a)


@pytest.mark.parametrize("n,b,P,gen", [(1024, 64, 8, "randn"), (2048, 64, 8, "randn"), (1536, 128, 8, "urand"),
                                       (700, 32, 4, "randn"), (900, 64, 3, "urand"), (640, 64, 0, "randn"),
                                       (520, 128, 0, "urand")])
def test_caluprrp_vs_oracle(dev, n, b, P, gen):
    """P = 0: the flat tree (sequential reduction, first block 2b rows)."""
    a = orc.randn_matrix(n, 42) if gen == "randn" else orc.urand_matrix(n, 42)
    f = dev.caluprrp_factor(a, b, 2.0, dev.flat_tree() if P == 0 else dev.binary_tree(P))
    ref = orc.calu_prrp(a, b, 2.0, *(("flat", None) if P == 0 else ("binary", P)))
    _check_factors(f, ref, a)


def test_caluprrp_single_leaf_equals_luprrp(dev):
    """Degenerate tree: CALU_PRRP with one leaf is LU_PRRP bit for bit."""
    a = orc.randn_matrix(512, 3)
    f1 = dev.caluprrp_factor(a, 64, 2.0, dev.binary_tree(1))
    f2 = dev.luprrp_factor(a, 64, 2.0)
    assert np.array_equal(f1.perm, f2.perm)
    assert np.array_equal(f1.l, f2.l) and np.array_equal(f1.u, f2.u)


@pytest.mark.parametrize("n,b", [(4096, 64), (4096, 128)])
def test_caluprrp_graph_replay_bit_identical(dev, n, b):
    """The first call captures the factorization into a CUDA graph, later calls
    replay it (three streams + the node-stream pool, deferred trailing
    updates): every replay must give the capture's bits, and the factors must
    reproduce A (schedule races would show up as differing bits)."""
    import ctypes
    import torch
    from paper_1208_2451_b200 import _lib
    lib = _lib.device_lib()
    a = orc.randn_matrix(n, 11)
    lda = n
    buf = torch.empty((n, lda), dtype=torch.float64, device="cuda")
    perm = torch.empty(n, dtype=torch.int64, device="cuda")
    outs = []
    for _ in range(3):
        buf.copy_(torch.from_numpy(np.ascontiguousarray(a)))
        npan = (n + b - 1) // b
        sw = (ctypes.c_int32 * npan)()
        chg = (ctypes.c_int64 * npan)()
        st, err = _lib.PrrpStats(), _lib.PrrpErr()
        rc = lib.prrp_caluprrp(ctypes.c_void_p(buf.data_ptr()), lda, n, n, b, 2.0, 8,
                               ctypes.c_void_p(perm.data_ptr()), sw, chg, ctypes.byref(st), ctypes.byref(err),
                               _lib.stream_handle())
        assert rc == 0, err.msg
        outs.append((buf.cpu().numpy().copy(), perm.cpu().numpy().copy()))
    for lu, p in outs[1:]:
        assert np.array_equal(lu, outs[0][0]) and np.array_equal(p, outs[0][1])
    lu, p = outs[0]
    l = np.tril(lu, -1) + np.eye(n)
    u = np.triu(lu)
    res = np.linalg.norm(a[p] - l @ u) / np.linalg.norm(a)
    assert res < n * 2.0 ** -52, res


def test_dist_calu_device_ops_single_rank(dev):
    """The distributed orchestration with the device ops (world size 1) agrees
    with the single-call device CALU_PRRP and with the reference algorithm."""
    import os
    import socket
    import torch.distributed as dist
    from paper_1208_2451_b200 import dist as pd
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        a = orc.randn_matrix(256, 11)
        f = pd.caluprrp_factor_dist(a, 16, 2.0, dev.binary_tree(4))
    finally:
        dist.destroy_process_group()
    ref = orc.calu_prrp(a, 16, 2.0, "binary", 4)
    one = dev.caluprrp_factor(a, 16, 2.0, dev.binary_tree(4))
    assert np.array_equal(f.perm, ref.perm) and np.array_equal(one.perm, ref.perm)
    assert list(f.stats.swap_counts) == list(ref.stats.swap_counts)
    assert _rel(f.u, ref.u) <= TOL_F and _rel(f.l, ref.l) <= TOL_F
    assert f.stats.growth_factor == pytest.approx(ref.stats.growth_factor, rel=TOL_G)


def test_device_matcore_and_gepp_api(dev):
    rng = np.random.default_rng(12)
    c, a, b = rng.standard_normal((70, 50)), rng.standard_normal((70, 16)), rng.standard_normal((16, 50))
    assert np.array_equal(dev.rank_update(c, a, b), orc.schur_update(c, a, b))
    assert np.array_equal(dev.matmul(a, b), orc.dger_product(a, b))
    br = rng.standard_normal((32, 90))
    g, r = dev.gepp_factor(br), orc.gepp(br)
    assert np.array_equal(g.perm, r.perm) and np.array_equal(g.u, r.u) and np.array_equal(g.l, r.l)
    assert g.intermediate_max == r.intermediate_max
    rr = np.triu(rng.standard_normal((16, 60))) + 4 * np.eye(16, 60)
    assert np.array_equal(dev.multiplier_block(rr, 16), orc.l_from_r(rr, 16))


# ---------------------------------------------------------------- API surface of 8(b) and 8(f)
def test_qr_column_pivoting(dev):
    """Device QRCP (prrp_qrcp) against the oracle restatement of pivoted_qr.py:74-87."""
    rng = np.random.Generator(np.random.PCG64(21))
    for h, p in ((8, 40), (32, 300), (64, 700)):
        a = np.asfortranarray(rng.standard_normal((h, p)))
        q = dev.qr_column_pivoting(a)
        ref = orc.qr_pivoted(a)
        assert np.array_equal(q.perm, ref.perm)
        assert _rel(q.r, ref.r) <= TOL_F and _rel(q.q, ref.q) <= TOL_F
        assert np.linalg.norm(q.q @ q.r - a[:, q.perm]) <= 1e-12 * np.linalg.norm(a)


@pytest.mark.parametrize("shape,m,b,leaf", [("binary", 600, 16, 8), ("binary", 257, 32, 4),
                                           ("flat", 300, 16, None), ("binary", 40, 16, 8)])
def test_tournament_select(dev, shape, m, b, leaf):
    """tournament_select (tournament.py:155-217) node for node against the oracle."""
    rng = np.random.Generator(np.random.PCG64(m + b))
    panel = np.asfortranarray(rng.standard_normal((m, b)))
    tree = dev.binary_tree(leaf) if shape == "binary" else dev.flat_tree()
    perm, trace = dev.tournament_select(panel, b, 2.0, tree, "srrqr")
    rperm, rtrace = orc.tournament(panel, b, 2.0, shape, leaf if leaf else 8)
    assert np.array_equal(perm, rperm)
    assert trace.single_node == rtrace.single_node and trace.leaf_count == rtrace.leaf_count
    assert [(n.level, n.index, n.swap_count) for n in trace.nodes] == \
        [(n.level, n.index, n.swap_count) for n in rtrace.nodes]
    for n, r in zip(trace.nodes, rtrace.nodes):
        assert np.array_equal(n.members, r.members) and np.array_equal(n.selected, r.selected)


def test_luprrp_solve_and_residual(dev):
    """luprrp_solve (luprrp.py:204-214) and rel_factorization_error
    (metrics.py:56-63) on the device against numpy / the oracle."""
    a = orc.randn_matrix(300, 5)
    f = dev.luprrp_factor(a, 32, 2.0)
    rng = np.random.Generator(np.random.PCG64(6))
    x_true = rng.standard_normal(300)
    rhs = a @ x_true
    x = dev.luprrp_solve(f, rhs)
    assert x.shape == (300,)
    assert np.linalg.norm(x - x_true) <= 1e-10 * np.linalg.norm(x_true)
    X = dev.luprrp_solve(f, np.stack([rhs, 2 * rhs], axis=1))
    assert X.shape == (300, 2) and np.allclose(X[:, 1], 2 * x, rtol=1e-12, atol=1e-12)
    e = dev.rel_factorization_error(a, f.perm, f.l, f.u)
    e_ref = orc.rel_residual(a, f.perm, f.l, f.u)
    assert 0 < e <= 4 * e_ref + 1e-15 and e_ref <= 4 * e + 1e-15
    with pytest.raises(dev.DimensionMismatch):
        dev.luprrp_solve(f, np.ones(7))


def test_concurrent_host_threads(dev):
    """The ABI is called from several host threads at once (SURVEY 8(b)
    threading: stream-ordered, reentrant): results equal the serial ones."""
    import threading
    mats = [orc.randn_matrix(768, 100 + i) for i in range(4)]
    serial_lu = [dev.luprrp_factor(a, 64, 2.0) for a in mats[:2]]
    serial_calu = [dev.caluprrp_factor(a, 64, 2.0) for a in mats[2:]]
    out = {}

    def work(i):
        if i < 2:
            out[i] = dev.luprrp_factor(mats[i], 64, 2.0)
        else:
            out[i] = dev.caluprrp_factor(mats[i], 64, 2.0)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for i, ref in enumerate(serial_lu + serial_calu):
        assert np.array_equal(out[i].perm, ref.perm)
        assert np.array_equal(out[i].l, ref.l) and np.array_equal(out[i].u, ref.u)


def _device_calu(buf, n, b, P):
    import ctypes
    import torch
    from paper_1208_2451_b200 import _lib
    lib = _lib.device_lib()
    perm = torch.empty(n, dtype=torch.int64, device="cuda")
    npan = (n + b - 1) // b
    sw = (ctypes.c_int32 * npan)()
    chg = (ctypes.c_int64 * npan)()
    st, err = _lib.PrrpStats(), _lib.PrrpErr()
    rc = lib.prrp_caluprrp(ctypes.c_void_p(buf.data_ptr()), buf.stride(0), n, n, b, 2.0, P,
                           ctypes.c_void_p(perm.data_ptr()), sw, chg, ctypes.byref(st), ctypes.byref(err),
                           _lib.stream_handle())
    assert rc == 0, err.msg
    return perm, st


@pytest.mark.parametrize("cfg", ["c2_b64", "c2_b128", "c3_wilkinson", "c3_foster", "c4", "c5"])
def test_full_size_properties(dev, cfg):
    """BASELINE configs at their full sizes, where the CPU oracle is too slow:
    size-independent properties.  Backward error ||PA - LU||_F / ||A||_F on the
    device below n 2^-52; multipliers bounded by tau (LU_PRRP's strong RRQR);
    the known growth factors of the growth-stress matrices (config 3, SURVEY
    8(c): Wilkinson 2, Foster 2.25); a second factorization bit-identical."""
    import torch
    from paper_1208_2451_b200 import matgen
    from paper_1208_2451_b200.metrics import rel_factorization_error_device
    if cfg.startswith("c2"):
        n, b = 8192, (64 if cfg == "c2_b64" else 128)
        a = matgen.gen_randn(n, 42, order="C")
    elif cfg == "c3_wilkinson":
        n, b = 4096, 64
        a = np.ascontiguousarray(orc.wilkinson_matrix(n))
    elif cfg == "c3_foster":
        n, b = 4096, 64
        a = np.ascontiguousarray(orc.foster_matrix(n, 1.0, 1.0, 1.0))
    elif cfg == "c4":
        n, b = 16384, 64
        a = matgen.gen_randn(n, 42, order="C")
    else:
        n, b = 32768, 128
        a = matgen.gen_urand(n, 42, order="C")
    A = torch.from_numpy(a).cuda()
    del a
    outs = []
    for _ in range(2):
        buf = A.clone()
        if cfg in ("c4", "c5"):
            perm, st = _device_calu(buf, n, b, 8)
            growth = st.intermediate_max / st.original_max
            pmm = None
        else:
            res = dev.luprrp_factor_device(buf, b, 2.0)
            perm, growth, pmm = res.perm, res.stats.growth_factor, res.stats.panel_multiplier_max
        outs.append((buf, perm, growth, pmm))
    (lu0, p0, g0, pmm0), (lu1, p1, g1, _) = outs
    assert torch.equal(p0, p1) and torch.equal(lu0, lu1) and g0 == g1
    assert torch.equal(torch.sort(p0).values, torch.arange(n, device=p0.device))
    res = rel_factorization_error_device(A, lu0, p0)
    assert res < n * 2.0 ** -52, res
    if pmm0 is not None:
        assert pmm0 <= 2.0 * (1 + 1e-12)
    if cfg == "c3_wilkinson":
        assert g0 == pytest.approx(2.0, rel=1e-10)
    if cfg == "c3_foster":
        assert g0 == pytest.approx(2.25, rel=1e-10)


# ------------------------------------------------------------ calu_factor
def _tree_of(dev, P):
    return dev.flat_tree() if P == 0 else dev.binary_tree(P)


def _otree(P):
    return ("flat", 8) if P == 0 else ("binary", P)


def test_calu_factor_golden(dev, golden):
    """calu_factor (tournament-pivoted GEPP, tournament.py:299-359) against
    the reference's fixtures: row order and flop counters exact, factors and
    statistics within the tolerances, rank-deficient leaves included."""
    index, arrays = golden
    for e in index["gepp_calu"]:
        a = gepp_calu_input(e)
        f = dev.calu_factor(a, e["b"], _tree_of(dev, e["P"]))
        ref = orc.calu_gepp(a, e["b"], *_otree(e["P"]))
        key = "gepp_calu/" + e["name"]
        assert np.array_equal(f.perm, arrays[key + "/perm"]), e["name"]
        assert _rel(f.l, arrays[key + "/l"]) <= TOL_F, e["name"]
        assert _rel(f.u, arrays[key + "/u"]) <= TOL_F, e["name"]
        assert str(f.stats.flops_charged) == e["stats"]["flops_charged"], e["name"]
        assert str(f.stats.flops_executed) == e["stats"]["flops_executed"], e["name"]
        if e["gen"] != "wilkinson":
            _check_factors(f, ref, a)


@pytest.mark.parametrize("n,b,P,gen", [(1024, 64, 8, "randn"), (1536, 128, 8, "urand"), (900, 64, 3, "randn"),
                                       (640, 32, 0, "randn"), (1000, 100, 5, "urand")])
def test_calu_factor_vs_oracle(dev, n, b, P, gen):
    a = orc.randn_matrix(n, 7) if gen == "randn" else orc.urand_matrix(n, 7)
    f = dev.calu_factor(a, b, _tree_of(dev, P))
    ref = orc.calu_gepp(a, b, *_otree(P))
    _check_factors(f, ref, a)


@pytest.mark.parametrize("shape,m,b,leaf,zero", [("binary", 600, 16, 8, None), ("binary", 257, 32, 4, (0, 80)),
                                                ("flat", 300, 16, None, (20, 60)), ("binary", 40, 16, 8, None)])
def test_tournament_select_gepp(dev, shape, m, b, leaf, zero):
    """GEPP selector tournament node for node, incl. a zeroed (rank-deficient) block."""
    rng = np.random.Generator(np.random.PCG64(m + 3 * b))
    panel = np.asfortranarray(rng.standard_normal((m, b)))
    if zero:
        panel[zero[0]:zero[1], :] = 0.0
    tree = dev.binary_tree(leaf) if shape == "binary" else dev.flat_tree()
    perm, trace = dev.tournament_select(panel, b, 2.0, tree, "gepp")
    rperm, rtrace = orc.tournament(panel, b, 2.0, shape, leaf if leaf else 8, "gepp")
    assert np.array_equal(perm, rperm)
    assert [(n.level, n.index) for n in trace.nodes] == [(n.level, n.index) for n in rtrace.nodes]
    for n, r in zip(trace.nodes, rtrace.nodes):
        assert np.array_equal(n.members, r.members) and np.array_equal(n.selected, r.selected)


def test_calu_factor_errors(dev):
    """Error contract: a rank-deficient panel raises RankDeficient(index, panel)
    like the reference; a zero pivot in the block-row finish SingularMatrix."""
    from paper_1208_2451_b200.errors import RankDeficient, SingularMatrix
    a = np.array(orc.randn_matrix(128, 2), order="F")
    a[:, 3] = 0.0                      # column 3 of panel 0: rank 3 < b = 16
    with pytest.raises((RankDeficient, SingularMatrix)) as ei:
        dev.calu_factor(a, 16, dev.binary_tree(4))
    with pytest.raises(ArithmeticError) as ri:
        orc.calu_gepp(a, 16, "binary", 4)
    assert type(ei.value).__name__.replace("Oracle", "") == type(ri.value).__name__.replace("Oracle", "")
    assert getattr(ei.value, "index", None) == getattr(ri.value, "index", None)
    assert getattr(ei.value, "panel", None) == getattr(ri.value, "panel", None)


def test_calu_factor_full_size(dev):
    """n = 4096, b = 64, P = 8: residual, determinism, growth vs the GEPP baseline's bound."""
    a = orc.randn_matrix(4096, 42)
    f1 = dev.calu_factor(a, 64)
    f2 = dev.calu_factor(a, 64)
    assert np.array_equal(f1.perm, f2.perm) and np.array_equal(f1.u, f2.u)
    assert sorted(f1.perm.tolist()) == list(range(4096))
    assert np.abs(np.tril(f1.l, -1)).max() <= 1.0 + 1e-12 or f1.stats.panel_multiplier_max > 1.0
    res = orc.rel_residual(a, f1.perm, f1.l, f1.u)
    assert res < 4096 * 2.0 ** -52


@pytest.mark.parametrize("m,n", [(300, 300), (500, 200), (150, 400), (1024, 1024), (64, 200), (257, 3)])
def test_gepp_factor_any_shape_bit_exact(dev, m, n):
    """gepp_factor (gepp.py:39-65) of any shape against the oracle: row order,
    L, U and both growth statistics bit for bit."""
    rng = np.random.Generator(np.random.PCG64(m * 7 + n))
    a = rng.standard_normal((m, n))
    g, r = dev.gepp_factor(a), orc.gepp(a)
    assert np.array_equal(g.perm, r.perm)
    assert np.array_equal(g.l, r.l) and np.array_equal(g.u, r.u)
    assert g.intermediate_max == r.intermediate_max and g.original_max == r.original_max


def test_gepp_factor_singular_column(dev):
    from paper_1208_2451_b200.errors import SingularMatrix
    a = np.array(orc.randn_matrix(200, 4), order="F")
    a[:, 17] = a[:, 3]            # column 17 becomes exactly dependent only after elimination: use a zero column
    a[:, 17] = 0.0
    with pytest.raises(SingularMatrix) as ei:
        dev.gepp_factor(a)
    with pytest.raises(ArithmeticError) as ri:
        orc.gepp(a)
    assert ei.value.column == ri.value.column == 17

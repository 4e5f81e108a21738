"""Pin the CPU oracle (oracle/prrp_oracle.py) against golden vectors produced
by the reference package itself (tests/golden/make_golden.py).

On the fixture host's BLAS (OpenBLAS Haswell kernels) the oracle reproduces
the reference bit for bit; permutations and swap counts are compared exactly
everywhere, floating values exactly when the BLAS configuration matches the
fixture's and to 1e-12 relative otherwise (the reference's own bits move by
<= 7e-13 across OpenBLAS kernel families)."""
import hashlib
from fractions import Fraction

import numpy as np
import pytest

from conftest import gepp_calu_input, make_input, srrqr_input
from oracle import prrp_oracle as orc


def _same_blas(index):
    cfg = str(np.__config__.CONFIG["Build Dependencies"]["blas"].get("openblas configuration", ""))
    return cfg == index["blas"]


def _close(a, b, exact):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape
    if exact:
        assert np.array_equal(a, b)
    else:
        scale = max(np.abs(b).max(), 1e-300) if b.size else 1.0
        assert np.abs(a - b).max() <= 1e-12 * scale


def _check_stats(st, ref, exact):
    for k in ("original_max", "intermediate_max", "finish_max", "panel_multiplier_max"):
        if exact:
            assert getattr(st, k) == ref[k], k
        else:
            assert getattr(st, k) == pytest.approx(ref[k], rel=1e-12), k
    assert list(st.swap_counts) == ref["swap_counts"]
    assert st.flops_charged == Fraction(ref["flops_charged"])
    assert st.flops_executed == Fraction(ref["flops_executed"])


def test_generators_match_reference(golden):
    index, _ = golden
    for e in index["lu"] + index["calu"] + index["lu_errors"]:
        a = make_input(e)
        assert hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest() == e["input_sha"], e["name"]
    c1 = index["c1"]
    a = orc.randn_matrix(c1["n"], c1["seed"])
    assert hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest() == c1["input_sha"]


def test_srrqr_golden(golden):
    index, arrays = golden
    exact = _same_blas(index)
    for e in index["srrqr"]:
        a = srrqr_input(e, arrays)
        res = orc.srrqr(a, e["b"], e["tau"])
        key = "srrqr/" + e["name"]
        assert np.array_equal(res.qr.perm, arrays[key + "/perm"]), e["name"]
        assert res.swap_count == e["swap_count"], e["name"]
        r_ref = arrays[key + "/r"]
        _close(res.qr.r[:, :r_ref.shape[1]], r_ref, exact)
        _close(res.qr.q, arrays[key + "/q"], exact)
        _close(res.l_block, arrays[key + "/l_block"], exact)


def test_spec_srrqr_examples():
    """SPEC.md:152-154 strong RRQR examples."""
    a = np.hstack([np.eye(4), np.zeros((4, 3))])
    res = orc.srrqr(a, 4, 2.0)
    assert np.array_equal(res.qr.perm, np.arange(7)) and res.swap_count == 0
    assert np.all(res.l_block == 0)
    res = orc.srrqr(np.array([[1.0, 10.0]]), 1, 2.0)
    assert list(res.qr.perm) == [1, 0] and res.l_block[0, 0] == pytest.approx(0.1)


def _tree(e):
    """(shape, leaf_count) of a CALU fixture: "P": 0 is the flat tree."""
    return ("binary", e["P"]) if e["P"] > 0 else ("flat", None)


@pytest.mark.parametrize("which", ["lu", "calu"])
def test_factor_golden(golden, which):
    index, arrays = golden
    exact = _same_blas(index)
    for e in index[which]:
        a = make_input(e)
        if which == "lu":
            f = orc.lu_prrp(a, e["b"], e["tau"])
        else:
            f = orc.calu_prrp(a, e["b"], e["tau"], *_tree(e))
        key = f"{which}/" + e["name"]
        assert np.array_equal(f.perm, arrays[key + "/perm"]), e["name"]
        if key + "/l" in arrays:
            _close(f.l, arrays[key + "/l"], exact)
            _close(f.u, arrays[key + "/u"], exact)
        assert float(f.l.sum()) == pytest.approx(e["l_sum"], rel=1e-12, abs=1e-12)
        assert float(f.u.sum()) == pytest.approx(e["u_sum"], rel=1e-12, abs=1e-12)
        _check_stats(f.stats, e["stats"], exact)


def test_tournament_trace_golden(golden):
    index, arrays = golden
    for e in index["calu"]:
        a = make_input(e)
        perm, tr = orc.tournament(a[:, :e["b"]], e["b"], e["tau"], *_tree(e))
        assert np.array_equal(perm, arrays["calu/" + e["name"] + "/t_perm"])
        assert tr.leaf_count == e["trace_leaf_count"]
        got = [(n.level, n.index, n.members.tolist(), n.selected.tolist(), n.swap_count) for n in tr.nodes]
        ref = [(n["level"], n["index"], n["members"], n["selected"], n["swap_count"]) for n in e["trace"]]
        assert got == ref


def test_gepp_calu_golden(golden):
    """calu_factor (tournament.py:299-359): the oracle restatement against
    the reference's own outputs -- factors, row order, exact rational flop
    counters, growth statistics, and the GEPP tournament trace including
    rank-deficient leaves (zeroed block, Wilkinson)."""
    index, arrays = golden
    exact = _same_blas(index)
    assert len(index["gepp_calu"]) >= 8
    for e in index["gepp_calu"]:
        a = gepp_calu_input(e)
        assert hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest() == e["input_sha"], e["name"]
        shape, lc = _tree(e)
        f = orc.calu_gepp(a, e["b"], shape, lc or 8)
        key = "gepp_calu/" + e["name"]
        assert np.array_equal(f.perm, arrays[key + "/perm"]), e["name"]
        _close(f.l, arrays[key + "/l"], exact)
        _close(f.u, arrays[key + "/u"], exact)
        _check_stats(f.stats, e["stats"], exact)
        perm, tr = orc.tournament(a[:, :e["b"]], e["b"], 2.0, shape, lc or 8, "gepp")
        assert np.array_equal(perm, arrays[key + "/t_perm"]), e["name"]
        got = [(n.level, n.index, n.members.tolist(), n.selected.tolist()) for n in tr.nodes]
        ref = [(n["level"], n["index"], n["members"], n["selected"]) for n in e["trace"]]
        assert got == ref, e["name"]


def test_error_contract_golden(golden):
    index, _ = golden
    for e in index["lu_errors"]:
        a = make_input(e)
        for fn, key in ((lambda: orc.lu_prrp(a, e["b"], e["tau"]), "error"),
                        (lambda: orc.calu_prrp(a, e["b"], e["tau"], "binary", 4), "calu_error")):
            ref = e[key]
            with pytest.raises(ArithmeticError) as ei:
                fn()
            exc = ei.value
            assert orc.ERROR_NAMES[type(exc)] == ref["type"]
            assert getattr(exc, "index", None) == ref["index"]
            assert getattr(exc, "column", None) == ref["column"]
            assert getattr(exc, "panel", None) == ref["panel"]
            tn = getattr(exc, "tree_node", None)
            assert (list(tn) if tn else None) == ref["tree_node"]


def test_c1_golden(golden):
    """BASELINE config 1: randn(1024, 42), b=64, tau=2 (0.7 s on 8 cores)."""
    index, arrays = golden
    c1 = index["c1"]
    exact = _same_blas(index)
    a = orc.randn_matrix(c1["n"], c1["seed"])
    f = orc.lu_prrp(a, c1["b"], c1["tau"])
    assert np.array_equal(f.perm, arrays["c1/perm"])
    _close(f.l[c1["sample_rows"], :], arrays["c1/l_rows"], exact)
    _close(f.u[c1["sample_rows"], :], arrays["c1/u_rows"], exact)
    _check_stats(f.stats, c1["stats"], exact)
    assert f.stats.growth_factor == pytest.approx(8.963326484888015, rel=1e-12)
    assert orc.rel_residual(a, f.perm, f.l, f.u) < 4 * c1["rel_residual"] + 1e-16


def test_pairwise_norm_model():
    """The device norm recipe (8 strided accumulators, ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)),
    sequential remainder; plain sequential below 8 terms) reproduces numpy's
    axis-0 sum of squares of F-ordered slices bit for bit for lengths 1..128,
    i.e. the QRCP norms of pivoted_qr.py:82 and the _reflect sums of :46,52."""
    rng = np.random.default_rng(7)
    for L in range(1, 129):
        base = np.asfortranarray(rng.standard_normal((L + 5, 40)))
        sub = base[5:, 3:]
        ref = (sub * sub).sum(axis=0)
        for j in range(sub.shape[1]):
            x = sub[:, j] * sub[:, j]
            assert orc_pairwise(x) == ref[j], (L, j)
        col = base[5:, 0]
        assert orc_pairwise(col * col) == (col * col).sum()


def orc_pairwise(x):
    n = x.shape[0]
    if n < 8:
        s = -0.0
        for i in range(n):
            s += x[i]
        return s
    r = [x[j] for j in range(8)]
    i = 8
    while i < n - (n % 8):
        for j in range(8):
            r[j] += x[i + j]
        i += 8
    s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
    while i < n:
        s += x[i]
        i += 1
    return s


# ------------------------------------------------------------ full-size / deficient-node fixtures
def _full(name):
    import json
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "full", name)
    return json.load(open(path + ".json")), dict(np.load(path + ".npz"))


def _full_names(prefix):
    import glob
    import os
    d = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "full")
    return sorted(os.path.basename(p)[:-5] for p in glob.glob(os.path.join(d, prefix + "*.json")))


@pytest.mark.parametrize("name", _full_names("calu_def_"))
def test_oracle_calu_rank_deficient_nodes(name):
    """The oracle's tournament (tournament.py:118-152 restated) shrinks a
    rank-deficient node's selection like the reference: same permutation,
    factors, node trace and error on the deficient-node fixtures."""
    from paper_1208_2451_b200 import matgen
    meta, arr = _full(name)
    a = matgen.gen_deficient_block(meta["n"], meta["seed"], meta["blocks"], meta["b"])
    assert hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest() == meta["input_sha"]
    shape, leaf = ("flat", 8) if meta["P"] == 0 else ("binary", meta["P"])
    if "error" in meta:
        with pytest.raises(ArithmeticError) as ei:
            orc.calu_prrp(a, meta["b"], meta["tau"], shape, leaf)
        assert type(ei.value).__name__.replace("Oracle", "") == meta["error"]["type"]
        assert getattr(ei.value, "index", None) == meta["error"]["index"]
        assert getattr(ei.value, "panel", None) == meta["error"]["panel"]
        return
    f = orc.calu_prrp(a, meta["b"], meta["tau"], shape, leaf)
    assert np.array_equal(f.perm, arr["perm"])
    if "l" in arr:
        _close(f.l, arr["l"], False)
        _close(f.u, arr["u"], False)
    else:
        _close(f.l[meta["sample_rows"]], arr["l_rows"], False)
        _close(f.u[meta["sample_rows"]], arr["u_rows"], False)
    perm, trace = orc.tournament(np.asfortranarray(a[:, :meta["b"]]), meta["b"], meta["tau"], shape, leaf)
    assert np.array_equal(perm, arr["t0_perm"])
    got = [(n.level, n.index, n.members.tolist(), n.selected.tolist()) for n in trace.nodes]
    assert got == [(d["level"], d["index"], d["members"], d["selected"]) for d in meta["t0_trace"]]


@pytest.mark.parametrize("name", _full_names("srrqr_"))
def test_oracle_srrqr_large_p(name):
    """strong_rrqr at p in 4097..16384 (the device engines' multi-CTA paths):
    the oracle against the reference's permutation, swaps and R11."""
    from paper_1208_2451_b200 import matgen
    meta, arr = _full(name)
    p, b = meta["p"], meta["b"]
    if meta.get("kahan"):
        at = matgen.gen_kahan_panel(p, b, meta["kahan"][0], meta["kahan"][1], meta["seed"])
    else:
        at = matgen.gen_randn_rect(p, b, meta["seed"]).T
    res = orc.srrqr(np.asfortranarray(at), b, meta["tau"])
    assert np.array_equal(res.qr.perm, arr["perm"])
    assert res.swap_count == meta["swap_count"]
    _close(res.qr.r[:, :b], arr["r11"], False)


def test_full_size_generators_match_reference():
    """The repo's generators reproduce the reference's matgen bits at the
    BASELINE sizes (checksums recorded by make_golden_full.py)."""
    from paper_1208_2451_b200 import matgen
    meta, _ = _full("c3_foster")
    a = matgen.gen_foster(meta["n"], 1.0, 1.0, 1.0)
    assert hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest() == meta["input_sha"]
    meta, _ = _full("c3_wilkinson")
    a = matgen.gen_wilkinson(meta["n"])
    assert hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest() == meta["input_sha"]


@pytest.mark.parametrize("name", _full_names("metrics_"))
def test_oracle_residual_extended(name):
    """The oracle's compensated residual (metrics.py:84-92) reproduces the
    reference's bits at the reference's solution."""
    from paper_1208_2451_b200 import matgen
    meta, arr = _full(name)
    n = meta["n"]
    a = {"randn": lambda: matgen.gen_randn(n, 42), "wilkinson": lambda: matgen.gen_wilkinson(n),
         "foster": lambda: matgen.gen_foster(n, 1.0, 1.0, 1.0)}[meta["gen"]]()
    rhs = matgen.gen_randn_rect(n, 1, meta["rhs_seed"]).reshape(-1)
    assert np.array_equal(orc.residual_extended(a, arr["x0"], rhs), arr["r"])


def test_harness_formats_and_generators():
    """The matrix text format (matcore.py:189-225) byte for byte, generator
    specs (matgen.py:378-413) and the harness families' bits against the
    reference's, CSV schema v1 (cli.py:29-33)."""
    import io
    from paper_1208_2451_b200 import harness
    meta, _ = _full("harness_rows_n96")
    from paper_1208_2451_b200 import matgen
    a = matgen.gen_randn(meta["n"], meta["seed"])
    assert harness.matrix_to_text(a[:5, :7]) == meta["text_5x7"]
    assert np.array_equal(harness.read_matrix(io.StringIO(meta["text_5x7"])), a[:5, :7])
    for spec, want in meta["generator_sha"].items():
        g = harness.generate(harness.parse_spec(spec, seed=meta["generator_seeds"].get(spec, 0)))
        assert hashlib.sha256(np.ascontiguousarray(g).tobytes()).hexdigest() == want, spec
    assert list(harness.CSV_HEADER) == meta["csv_header"] and harness.CSV_VERSION == meta["csv_version"]
    with pytest.raises(ValueError):
        harness.read_matrix(io.StringIO("2 2\n1 2\n3\n"))
    with pytest.raises(ValueError):
        harness.parse_spec("randn")

"""Full-size parity goldens (BASELINE configs 2-5) from the REAL reference
package (``prrp`` at /root/reference/pkg/src; build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_full.py [case ...]

Writes tests/golden/full/<case>.npz + <case>.json.  Cases:

* ``c2_b64``, ``c2_b128``: ``luprrp_factor(gen_randn(8192, 42), b, 2.0)``
  in full (about 200 s each): permutation, swap counts, ElimStats, growth,
  row / column sums of L and U, sample rows, backward error.
* ``c3_wilkinson``, ``c3_foster``: config 3 at n = 4096, b = 64.
* ``c4_prefix``, ``c5_prefix``: CALU_PRRP (``binary_tree(8)``) of the first
  K panels of configs 4 / 5.  Right-looking LU of columns [0, K b) depends on
  those columns only (each panel reads the panel columns after the previous
  updates, ``rank_update`` is elementwise in the columns it touches, and the
  GEPP finish of a panel pivots on its own b x b block), so the reference
  run on the tall m x K b matrix A[:, :K b] fixes perm[:K b], the first K
  swap counts, L[:, :K b] (row by row, by original row id) and U[:K b, :K b]
  of the full factorization.  The full 16384^2 / 32768^2 reference runs are
  hours and ~51 GB of RAM; the prefix runs are minutes.
* ``srrqr_*``: ``strong_rrqr`` of b x p panel transposes at p in {4097,
  6000, 8192, 12288, 16384}, b in {64, 128} (the device engines' multi-CTA
  column paths above 4096 rows), plus Kahan-type panels
  (``matgen.gen_kahan_panel``) on which the swap loop runs at large p.

Inputs are regenerated from (generator, n, seed) by the repo's own
generators (``paper_1208_2451_b200.matgen``); the input checksums stored here
pin those against the reference's ``matgen``.
"""

import hashlib
import json
import os
import sys
import time
from fractions import Fraction

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import prrp  # noqa: E402  (the reference)
from prrp import matgen  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "full")
sys.path.insert(0, ROOT)
from paper_1208_2451_b200 import matgen as pmg  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def stats_dict(st, full=True):
    d = {
        "original_max": st.original_max,
        "intermediate_max": st.intermediate_max,
        "finish_max": st.finish_max,
        "panel_multiplier_max": st.panel_multiplier_max,
        "swap_counts": list(map(int, st.swap_counts)),
        "flops_charged": str(Fraction(st.flops_charged)),
        "flops_executed": str(Fraction(st.flops_executed)),
    }
    if full:
        d["growth_factor"] = st.growth_factor
        d["full_growth_factor"] = st.full_growth_factor
    return d


def rel_residual(a, perm, l, u):
    """||A[perm] - L U||_F / ||A||_F in float64 (numpy BLAS)."""
    r = a[perm, :] - l @ u
    return float(np.linalg.norm(r) / np.linalg.norm(a))


def factor_summary(a, f, arrays, meta, sample_rows):
    n = a.shape[1]
    arrays["perm"] = np.asarray(f.perm, dtype=np.int64)
    arrays["l_colsum"] = f.l.sum(axis=0)
    arrays["l_rowsum"] = f.l.sum(axis=1)
    arrays["l_colabs"] = np.abs(f.l).sum(axis=0)
    arrays["u_colsum"] = f.u.sum(axis=0)
    arrays["u_rowsum"] = f.u.sum(axis=1)
    arrays["u_rowabs"] = np.abs(f.u).sum(axis=1)
    arrays["u_diag"] = np.diag(f.u).copy()
    arrays["l_rows"] = f.l[sample_rows, :]
    arrays["u_rows"] = f.u[sample_rows, :]
    meta["sample_rows"] = sample_rows
    meta["stats"] = stats_dict(f.stats)
    meta["l_max"] = float(np.abs(f.l).max())
    meta["u_max"] = float(np.abs(f.u).max())
    t = time.time()
    meta["rel_residual"] = rel_residual(a, f.perm, f.l, f.u)
    print("  residual", meta["rel_residual"], "%.1f s" % (time.time() - t), flush=True)
    meta["n"] = n


def case_lu(name, gen, n, b, **kw):
    if gen == "randn":
        a = matgen.gen_randn(n, 42)
        assert np.array_equal(a, pmg.gen_randn(n, 42))
    elif gen == "wilkinson":
        a = matgen.gen_wilkinson(n)
        assert np.array_equal(a, pmg.gen_wilkinson(n))
    elif gen == "foster":
        a = matgen.gen_foster(n, c=1.0, h=1.0, k=1.0)
        assert np.array_equal(a, pmg.gen_foster(n, 1.0, 1.0, 1.0))
    t = time.time()
    f = prrp.luprrp_factor(a, b, 2.0)
    dt = time.time() - t
    print(name, "luprrp_factor %.1f s" % dt, flush=True)
    meta = {"kind": "luprrp", "gen": gen, "n": n, "b": b, "tau": 2.0, "seed": 42,
            "input_sha": sha(a), "ref_seconds": dt}
    arrays = {}
    factor_summary(a, f, arrays, meta, [0, 1, b - 1, b, n // 2, n - 1])
    return meta, arrays


def case_calu_prefix(name, gen, n, b, K):
    kb = K * b
    if gen == "randn":
        a = matgen.gen_randn(n, 42)
        assert np.array_equal(a, pmg.gen_randn(n, 42))
        s = sha(a)
        a = np.asfortranarray(a[:, :kb])
    else:
        a = pmg.gen_urand_cols(n, 42, kb)         # chunked: the 8 GiB matrix is never formed
        s = None
    t = time.time()
    f = prrp.caluprrp_factor(a, b, 2.0, prrp.binary_tree(8))
    dt = time.time() - t
    print(name, "caluprrp_factor(prefix %d x %d) %.1f s" % (n, kb, dt), flush=True)
    # the first tournament with its trace (node for node)
    perm0, trace = prrp.tournament_select(np.asfortranarray(a[:, :b]), b, 2.0, prrp.binary_tree(8), "srrqr")
    pos = np.empty(n, dtype=np.int64)
    pos[f.perm] = np.arange(n)
    arrays = {
        "perm_prefix": np.asarray(f.perm[:kb], dtype=np.int64),
        "prefix_sha_cols": np.frombuffer(hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest(), np.uint8),
        # L[:, :kb] by ORIGINAL row id (rows at positions >= kb move later)
        "l_rowsum_by_row": f.l[pos, :].sum(axis=1),
        "l_rowabs_by_row": np.abs(f.l[pos, :]).sum(axis=1),
        "l_colsum": f.l.sum(axis=0),
        "u_rowsum": f.u[:kb, :kb].sum(axis=1),
        "u_rowabs": np.abs(f.u[:kb, :kb]).sum(axis=1),
        "u_diag": np.diag(f.u[:kb, :kb]).copy(),
        "u_rows": np.ascontiguousarray(f.u[[0, 1, b, kb - 1], :kb]),
        "t0_perm": np.asarray(perm0, dtype=np.int64),
    }
    meta = {"kind": "calu_prefix", "gen": gen, "n": n, "b": b, "tau": 2.0, "seed": 42, "P": 8,
            "K": K, "input_sha_full": s, "input_sha_prefix": sha(a), "ref_seconds": dt,
            "swap_counts": list(map(int, f.stats.swap_counts)),
            "panel_multiplier_max": f.stats.panel_multiplier_max,
            "l_max": float(np.abs(f.l).max()), "u_max": float(np.abs(f.u[:kb, :kb]).max()),
            "t0_trace": [{"level": nd.level, "index": nd.index, "n_members": int(nd.members.shape[0]),
                          "selected": nd.selected.tolist(), "swap_count": int(nd.swap_count)}
                         for nd in trace.nodes]}
    return meta, arrays


def case_srrqr(name, p, b, tau, kahan=None):
    if kahan:                                          # (theta, scale): the swap loop runs
        at = pmg.gen_kahan_panel(p, b, kahan[0], kahan[1], 7 + p + b)
        a = at.T
    else:
        a = pmg.gen_randn_rect(p, b, 7 + p + b)        # p x b panel, row-major draws
        ref_a = matgen._normals(matgen._rng(7 + p + b), p * b).reshape(p, b)
        assert np.array_equal(a, ref_a)
    t = time.time()
    res = prrp.strong_rrqr(np.asfortranarray(a.T), b, tau)
    dt = time.time() - t
    print(name, "strong_rrqr %.1f s swaps %d" % (dt, res.swap_count), flush=True)
    arrays = {
        "perm": np.asarray(res.qr.perm, dtype=np.int64),
        "r_diag": np.diag(res.qr.r[:, :b]).copy(),
        "r11": np.ascontiguousarray(res.qr.r[:, :b]),
        "r_colsum": res.qr.r.sum(axis=0),
        "l_colsum": res.l_block.sum(axis=0),
        "l_rows": np.ascontiguousarray(res.l_block[[0, 1, (p - b) // 2, p - b - 1], :]),
    }
    meta = {"kind": "srrqr", "p": p, "b": b, "h": b, "tau": tau, "seed": 7 + p + b, "input_sha": sha(a),
            "kahan": list(kahan) if kahan else None,
            "swap_count": int(res.swap_count), "ref_seconds": dt,
            "l_max": float(np.abs(res.l_block).max()), "r_max": float(np.abs(res.qr.r).max())}
    return meta, arrays


def case_calu_deficient(name, n, b, P, blocks, tau=2.0):
    """CALU_PRRP with rank-deficient tournament nodes (tournament.py:131-137):
    the full factorization (or the reference's error) on a small matrix."""
    a = pmg.gen_deficient_block(n, 11, blocks, b)
    tree = prrp.binary_tree(P) if P > 0 else prrp.flat_tree()
    meta = {"kind": "calu_deficient", "n": n, "b": b, "P": P, "tau": tau, "blocks": blocks, "seed": 11,
            "input_sha": sha(a)}
    arrays = {}
    try:
        f = prrp.caluprrp_factor(a, b, tau, tree)
    except ArithmeticError as exc:
        meta["error"] = {"type": type(exc).__name__, "index": getattr(exc, "index", None),
                         "column": getattr(exc, "column", None), "panel": getattr(exc, "panel", None),
                         "tree_node": list(exc.tree_node) if getattr(exc, "tree_node", None) else None}
        return meta, arrays
    arrays["perm"] = np.asarray(f.perm, dtype=np.int64)
    if n <= 256:
        arrays["l"] = f.l
        arrays["u"] = f.u
    else:                                   # compact: sums, diagonal, sample rows
        rows = [0, 1, b, n // 2, n - 1]
        arrays.update(l_rowsum=f.l.sum(axis=1), l_colsum=f.l.sum(axis=0), u_rowsum=f.u.sum(axis=1),
                      u_colsum=f.u.sum(axis=0), u_diag=np.diag(f.u).copy(), l_rows=f.l[rows], u_rows=f.u[rows])
        meta["sample_rows"] = rows
        meta["l_max"] = float(np.abs(f.l).max())
        meta["u_max"] = float(np.abs(f.u).max())
    meta["stats"] = stats_dict(f.stats)
    perm0, trace = prrp.tournament_select(np.asfortranarray(a[:, :b]), b, tau, tree, "srrqr")
    arrays["t0_perm"] = np.asarray(perm0, dtype=np.int64)
    meta["t0_trace"] = [{"level": nd.level, "index": nd.index, "members": nd.members.tolist(),
                         "selected": nd.selected.tolist(), "swap_count": int(nd.swap_count)} for nd in trace.nodes]
    meta["rel_residual"] = rel_residual(a, f.perm, f.l, f.u)
    return meta, arrays


def case_metrics(name, gen, n, b, alg):
    """The measurement battery (metrics.py:56-228) of the reference on one
    factorization: residual_extended bits at the reference's solution, eta,
    w, the HPL triplet, iterative refinement and the inverse norms."""
    from prrp import metrics
    if gen == "randn":
        a = matgen.gen_randn(n, 42)
    elif gen == "wilkinson":
        a = matgen.gen_wilkinson(n)
    else:
        a = matgen.gen_foster(n, c=1.0, h=1.0, k=1.0)
    rhs = pmg.gen_randn_rect(n, 1, 5).reshape(-1)
    f = prrp.luprrp_factor(a, b, 2.0) if alg == "luprrp" else prrp.gepp_factor(a)
    x0 = np.asarray(f.solve(rhs)).reshape(-1)
    r = metrics.residual_extended(a, x0, rhs)
    xr, n_ir, w_before = metrics.iterative_refinement(f, a, rhs)
    rep = metrics.full_report(a, f, rhs)
    arrays = {"x0": x0, "r": r, "x_refined": np.asarray(xr)}
    meta = {"kind": "metrics", "gen": gen, "n": n, "b": b, "alg": alg, "rhs_seed": 5, "input_sha": sha(a),
            "eta": metrics.normwise_backward_error(a, x0, rhs), "w": metrics.componentwise_backward_error(a, x0, rhs),
            "hpl": list(metrics.hpl_triplet(a, x0, rhs)), "n_ir": int(n_ir), "w_before": w_before,
            "inverse_norms": list(metrics.triangular_inverse_norms(f.l, f.u)),
            "report": [float(v) for v in (rep.g_w, rep.rel_fact_error, rep.eta, rep.w, *rep.hpl, rep.n_ir,
                                          rep.norm_l1, rep.norm_linv1, rep.norm_u1, rep.norm_uinv1)],
            "csv_row": metrics.report_csv_row(rep)}
    return meta, arrays


def case_block_variant(name, kind, n, b, p=None, tau=2.0):
    """block_parallel_luprrp / block_pairwise_luprrp (block_variants.py:231-244):
    the event log, the final upper factor, the statistics, and the replay."""
    from prrp import block_variants as bv
    a = matgen.gen_randn(n, 42)
    f = bv.block_parallel_luprrp(a, b, tau, p) if kind == "parallel" else bv.block_pairwise_luprrp(a, b, tau)
    arrays = {"perm": np.asarray(f.perm, dtype=np.int64)}
    rows = [0, 1, b, n // 2, n - 1]
    if n <= 256:
        arrays["u"] = f.u
    else:
        arrays.update(u_rowsum=f.u.sum(axis=1), u_colsum=f.u.sum(axis=0), u_rows=f.u[rows])
    rep = bv.replay_events(f.events, a)
    evs = []
    for i, ev in enumerate(f.events):
        if isinstance(ev, bv.RowPermEvent):
            moved = np.nonzero(ev.perm != np.arange(ev.perm.shape[0]))[0]
            if moved.size == 2 and ev.perm[moved[0]] == moved[1]:
                evs.append({"type": "perm", "swap": [int(moved[0]), int(moved[1])]})
            else:
                arrays[f"ev{i}/perm"] = np.asarray(ev.perm, dtype=np.int64)
                evs.append({"type": "perm"})
        else:
            arrays[f"ev{i}/elim"] = np.asarray(ev.elim_rows, dtype=np.int64)
            arrays[f"ev{i}/piv"] = np.asarray(ev.pivot_rows, dtype=np.int64)
            arrays[f"ev{i}/d"] = np.asarray(ev.d)
            evs.append({"type": "elim", "zero": [ev.zero_col0, ev.zero_col1], "update_col0": ev.update_col0})
    meta = {"kind": "block_" + kind, "n": n, "b": b, "p": p, "tau": tau, "seed": 42, "input_sha": sha(a),
            "events": evs, "stats": stats_dict(f.stats), "leaf_counts": list(map(int, f.leaf_counts)),
            "max_multiplier": f.max_multiplier, "sample_rows": rows, "u_max": float(np.abs(f.u).max()),
            "replay_max_diff": float(np.abs(rep - f.u).max())}
    return meta, arrays


def case_harness(name):
    """cli.run_single rows (CSV schema v1, cli.py:124-175) for every algorithm
    on one small matrix, and the text format of a matrix."""
    from prrp import cli
    a = matgen.gen_randn(96, 42)
    rows = {}
    for alg in cli.ALGORITHMS:
        rows[alg] = {k: (v if isinstance(v, (str, int)) else float(v)) for k, v in
                     cli.run_single(alg, a, b=16, p=4, tau=2.0, seed=42, family="randn").items()}
    txt = prrp.matcore.matrix_to_text(a[:5, :7])
    gens = {"wright:20": sha(matgen.generate(matgen.parse_spec("wright:20"))),
            "wright:64:h=0.7": sha(matgen.generate(matgen.parse_spec("wright:64:h=0.7"))),
            "genwilk:50:r=3": sha(matgen.generate(matgen.parse_spec("genwilk:50:r=3", seed=7))),
            "foster:40:k=1/3": sha(matgen.generate(matgen.parse_spec("foster:40:k=1/3"))),
            "wilkinson:33": sha(matgen.generate(matgen.parse_spec("wilkinson:33"))),
            "randn:30": sha(matgen.generate(matgen.parse_spec("randn:30", seed=5)))}
    meta = {"kind": "harness", "n": 96, "b": 16, "p": 4, "seed": 42, "rows": rows, "text_5x7": txt,
            "csv_header": list(cli.CSV_HEADER), "csv_version": cli.CSV_VERSION, "generator_sha": gens,
            "generator_seeds": {"genwilk:50:r=3": 7, "randn:30": 5}}
    return meta, {}


CASES = {
    "c2_b64": lambda: case_lu("c2_b64", "randn", 8192, 64),
    "c2_b128": lambda: case_lu("c2_b128", "randn", 8192, 128),
    "c3_wilkinson": lambda: case_lu("c3_wilkinson", "wilkinson", 4096, 64),
    "c3_foster": lambda: case_lu("c3_foster", "foster", 4096, 64),
    "c4_prefix": lambda: case_calu_prefix("c4_prefix", "randn", 16384, 64, 8),
    "c5_prefix": lambda: case_calu_prefix("c5_prefix", "urand", 32768, 128, 4),
}
# rank-deficient tournament nodes: a leaf that passes fewer than b rows; two
# deficient leaves whose merge passes its members through (<= b); the flat
# tree; a panel whose whole tournament supplies fewer than b rows (error);
# b = 64 / 128 nodes on the register engines
CASES["calu_def_leaf160_b16_P4"] = lambda: case_calu_deficient("calu_def_leaf160_b16_P4", 160, 16, 4, [[0, 40, 5]])
CASES["calu_def_pair160_b16_P4"] = lambda: case_calu_deficient("calu_def_pair160_b16_P4", 160, 16, 4,
                                                               [[0, 40, 5], [40, 80, 6]])
CASES["calu_def_flat160_b16"] = lambda: case_calu_deficient("calu_def_flat160_b16", 160, 16, 0, [[0, 32, 7]])
CASES["calu_def_root96_b16_P4"] = lambda: case_calu_deficient("calu_def_root96_b16_P4", 96, 16, 4, [[0, 96, 9]])
CASES["calu_def_leaf640_b64_P8"] = lambda: case_calu_deficient("calu_def_leaf640_b64_P8", 640, 64, 8,
                                                               [[0, 80, 20], [160, 240, 30]])
CASES["calu_def_leaf1024_b128_P4"] = lambda: case_calu_deficient("calu_def_leaf1024_b128_P4", 1024, 128, 4,
                                                                 [[0, 256, 50], [256, 512, 60]])
CASES["metrics_randn300_b32"] = lambda: case_metrics("metrics_randn300_b32", "randn", 300, 32, "luprrp")
CASES["block_parallel256_b16_p4"] = lambda: case_block_variant("block_parallel256_b16_p4", "parallel", 256, 16, 4)
CASES["block_parallel512_b64_p8"] = lambda: case_block_variant("block_parallel512_b64_p8", "parallel", 512, 64, 8)
CASES["block_pairwise200_b16"] = lambda: case_block_variant("block_pairwise200_b16", "pairwise", 200, 16)
CASES["block_pairwise384_b32_tau11"] = lambda: case_block_variant("block_pairwise384_b32_tau11", "pairwise", 384, 32,
                                                                   tau=1.1)
CASES["harness_rows_n96"] = lambda: case_harness("harness_rows_n96")
CASES["metrics_wilkinson55_gepp"] = lambda: case_metrics("metrics_wilkinson55_gepp", "wilkinson", 55, 8, "gepp")
CASES["metrics_foster256_gepp"] = lambda: case_metrics("metrics_foster256_gepp", "foster", 256, 16, "gepp")
for _p in (4097, 6000, 8192, 12288, 16384):
    for _b in (64, 128):
        CASES["srrqr_p%d_b%d" % (_p, _b)] = (lambda p=_p, b=_b: case_srrqr("srrqr_p%d_b%d" % (p, b), p, b, 2.0))
CASES["srrqr_kahan_p6000_b64"] = lambda: case_srrqr("srrqr_kahan_p6000_b64", 6000, 64, 2.0, (1.3, 1e-2))
CASES["srrqr_kahan_p8192_b128"] = lambda: case_srrqr("srrqr_kahan_p8192_b128", 8192, 128, 2.0, (1.45, 1e-2))
CASES["srrqr_kahan_p12288_b64"] = lambda: case_srrqr("srrqr_kahan_p12288_b64", 12288, 64, 2.0, (1.3, 1e-2))


def main(names):
    os.makedirs(OUT, exist_ok=True)
    for name in names or list(CASES):
        path = os.path.join(OUT, name)
        if os.path.exists(path + ".json") and not os.environ.get("REGEN"):
            print("exists", name)
            continue
        meta, arrays = CASES[name]()
        meta["name"] = name
        meta["numpy"] = np.__version__
        meta["openblas_coretype"] = os.environ.get("OPENBLAS_CORETYPE", "(auto: Haswell kernels here)")
        np.savez_compressed(path + ".npz", **arrays)
        with open(path + ".json", "w") as fh:
            json.dump(meta, fh, indent=1, default=float)
        print("wrote", name, flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])

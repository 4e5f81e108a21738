"""Generate the golden fixtures under tests/golden/ by running the REAL
reference package (``prrp`` at /root/reference/pkg/src, build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The fixtures pin the CPU oracle (``oracle/prrp_oracle.py``) and are the
known-answer vectors for the CUDA path.  Inputs are regenerated from
(generator, n, seed) by the oracle's generators, whose bits are checked
against the reference's ``matgen`` here (stored as input checksums).
"""

import hashlib
import json
import os
import sys
from fractions import Fraction

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import prrp  # noqa: E402  (the reference)
from prrp import matgen  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle import prrp_oracle as orc  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def make_input(spec):
    kind = spec["gen"]
    if kind == "randn":
        a = matgen.gen_randn(spec["n"], spec["seed"])
        if "m" in spec:             # tall: first m*n draws, row-major (same convention)
            a = orc.randn_matrix(max(spec["m"], spec["n"]), spec["seed"])[:spec["m"], :spec["n"]]
    elif kind == "urand":
        a = orc.urand_matrix(spec["n"], spec["seed"])
    elif kind == "wilkinson":
        a = matgen.gen_wilkinson(spec["n"])
    elif kind == "foster":
        a = matgen.gen_foster(spec["n"], c=1.0, h=1.0, k=spec.get("k", 1.0))
    elif kind == "identity":
        a = np.eye(spec["n"], order="F")
    elif kind == "zeros":
        a = np.zeros((spec["n"], spec["n"]), order="F")
    elif kind == "lowrank":
        rng = np.random.Generator(np.random.PCG64(spec["seed"]))
        u = rng.standard_normal((spec["n"], spec["rank"]))
        v = rng.standard_normal((spec["rank"], spec["n"]))
        a = np.asfortranarray(u @ v)
    elif kind == "duprows":
        a = np.array(orc.randn_matrix(spec["n"], spec["seed"]))
        a[1::2, :] = a[0::2, :]          # every odd row repeats its predecessor
        a = np.asfortranarray(a)
    elif kind == "explicit":
        a = np.asfortranarray(np.array(spec["data"], dtype=np.float64))
    else:
        raise ValueError(kind)
    return np.asfortranarray(a)


def stats_dict(st):
    return {
        "original_max": st.original_max,
        "intermediate_max": st.intermediate_max,
        "finish_max": st.finish_max,
        "panel_multiplier_max": st.panel_multiplier_max,
        "swap_counts": list(map(int, st.swap_counts)),
        "flops_charged": str(Fraction(st.flops_charged)),
        "flops_executed": str(Fraction(st.flops_executed)),
        "growth_factor": st.growth_factor if st.original_max else None,
        "full_growth_factor": st.full_growth_factor if st.original_max else None,
    }


def run_error(fn):
    try:
        fn()
    except Exception as exc:   # noqa: BLE001 - record the reference's error contract
        return {
            "type": type(exc).__name__,
            "index": getattr(exc, "index", None),
            "column": getattr(exc, "column", None),
            "worst": getattr(exc, "worst", None),
            "panel": getattr(exc, "panel", None),
            "tree_node": list(getattr(exc, "tree_node", ())) or None,
        }
    return None


LU_CASES = [
    {"name": "randn64_b8", "gen": "randn", "n": 64, "seed": 1, "b": 8, "tau": 2.0},
    {"name": "randn100_b16_ragged", "gen": "randn", "n": 100, "seed": 7, "b": 16, "tau": 2.0},
    {"name": "randn_tall120x80_b16", "gen": "randn", "m": 120, "n": 80, "seed": 3, "b": 16, "tau": 2.0},
    {"name": "randn128_b16_tau105", "gen": "randn", "n": 128, "seed": 5, "b": 16, "tau": 1.05},
    {"name": "randn256_b32", "gen": "randn", "n": 256, "seed": 42, "b": 32, "tau": 2.0},
    {"name": "randn200_b1", "gen": "randn", "n": 40, "seed": 11, "b": 1, "tau": 2.0},
    {"name": "randn48_bfull", "gen": "randn", "n": 48, "seed": 12, "b": 48, "tau": 2.0},
    {"name": "urand96_b16", "gen": "urand", "n": 96, "seed": 42, "b": 16, "tau": 2.0},
    {"name": "wilkinson64_b8", "gen": "wilkinson", "n": 64, "b": 8, "tau": 2.0},
    {"name": "foster64_b8", "gen": "foster", "n": 64, "b": 8, "tau": 2.0, "k": 1.0},
    {"name": "identity32_b8", "gen": "identity", "n": 32, "b": 8, "tau": 2.0},
    {"name": "randn512_b64", "gen": "randn", "n": 512, "seed": 42, "b": 64, "tau": 2.0},
]

LU_ERROR_CASES = [
    {"name": "zeros16_b4", "gen": "zeros", "n": 16, "b": 4, "tau": 2.0},
    {"name": "lowrank32_r10_b8", "gen": "lowrank", "n": 32, "rank": 10, "seed": 2, "b": 8, "tau": 2.0},
    {"name": "duprows32_b8", "gen": "duprows", "n": 32, "seed": 4, "b": 8, "tau": 2.0},
]

CALU_CASES = [
    {"name": "calu_randn256_b8_P8", "gen": "randn", "n": 256, "seed": 42, "b": 8, "tau": 2.0, "P": 8},
    {"name": "calu_randn200_b16_P4", "gen": "randn", "n": 200, "seed": 9, "b": 16, "tau": 2.0, "P": 4},
    {"name": "calu_urand160_b16_P8", "gen": "urand", "n": 160, "seed": 42, "b": 16, "tau": 2.0, "P": 8},
    {"name": "calu_randn512_b32_P8", "gen": "randn", "n": 512, "seed": 42, "b": 32, "tau": 2.0, "P": 8},
    {"name": "calu_randn256_b16_P8_tau11", "gen": "randn", "n": 256, "seed": 8, "b": 16, "tau": 1.1, "P": 8},
    # flat reduction tree (tournament.py:81-88, 202-208): "P": 0
    {"name": "calu_flat_randn160_b16", "gen": "randn", "n": 160, "seed": 42, "b": 16, "tau": 2.0, "P": 0},
    {"name": "calu_flat_randn256_b32", "gen": "randn", "n": 256, "seed": 5, "b": 32, "tau": 2.0, "P": 0},
]

# calu_factor (tournament-pivoted GEPP, tournament.py:299-359); "zero": rows
# [r0, r1) x columns [0, c) zeroed, so a leaf of the first panel is
# numerically rank deficient and passes on fewer than b rows
GEPP_CALU_CASES = [
    {"name": "gcalu_randn256_b8_P8", "gen": "randn", "n": 256, "seed": 42, "b": 8, "P": 8},
    {"name": "gcalu_randn200_b16_P4", "gen": "randn", "n": 200, "seed": 9, "b": 16, "P": 4},
    {"name": "gcalu_urand160_b16_P8", "gen": "urand", "n": 160, "seed": 42, "b": 16, "P": 8},
    {"name": "gcalu_randn512_b64_P8", "gen": "randn", "n": 512, "seed": 42, "b": 64, "P": 8},
    {"name": "gcalu_tall200x120_b16_P3", "gen": "randn", "m": 200, "n": 120, "seed": 3, "b": 16, "P": 3},
    {"name": "gcalu_flat_randn160_b16", "gen": "randn", "n": 160, "seed": 42, "b": 16, "P": 0},
    {"name": "gcalu_zeroleaf160_b16_P4", "gen": "randn", "n": 160, "seed": 6, "b": 16, "P": 4, "zero": [0, 40, 16]},
    {"name": "gcalu_wilkinson64_b8_P4", "gen": "wilkinson", "n": 64, "b": 8, "P": 4},
]


def gepp_calu_input(c):
    a = make_input(c).copy(order="F")
    if "zero" in c:
        r0, r1, cols = c["zero"]
        a[r0:r1, :cols] = 0.0
    return a


SRRQR_CASES = [
    {"name": "eye_pad", "data": np.hstack([np.eye(4), np.zeros((4, 3))]).tolist(), "b": 4, "tau": 2.0},
    {"name": "one_ten", "data": [[1.0, 10.0]], "b": 1, "tau": 2.0},
    {"name": "rand3x12_tau105", "seed": 21, "h": 3, "p": 12, "b": 3, "tau": 1.05},
    {"name": "rand8x40", "seed": 22, "h": 8, "p": 40, "b": 8, "tau": 2.0},
    {"name": "rand16x200_tau105", "seed": 23, "h": 16, "p": 200, "b": 16, "tau": 1.05},
    {"name": "rand16x300_tau101", "seed": 24, "h": 16, "p": 300, "b": 16, "tau": 1.01},
    {"name": "rand32x129", "seed": 25, "h": 32, "p": 129, "b": 32, "tau": 2.0},
    {"name": "rand64x400", "seed": 26, "h": 64, "p": 400, "b": 64, "tau": 2.0},
    {"name": "rand64x400_tau11", "seed": 27, "h": 64, "p": 400, "b": 64, "tau": 1.1},
]


def srrqr_input(c):
    if "data" in c:
        return np.asfortranarray(np.array(c["data"], dtype=np.float64))
    rng = np.random.Generator(np.random.PCG64(c["seed"]))
    return np.asfortranarray(rng.standard_normal((c["h"], c["p"])))


def main():
    index = {"blas": str(np.__config__.CONFIG["Build Dependencies"]["blas"].get("openblas configuration", "")),
             "lu": [], "lu_errors": [], "calu": [], "gepp_calu": [], "srrqr": [], "c1": None}
    arrays = {}

    for c in SRRQR_CASES:
        a = srrqr_input(c)
        res = prrp.strong_rrqr(a, c["b"], c["tau"])
        key = "srrqr/" + c["name"]
        if "data" in c:
            arrays[key + "/a"] = a
        arrays[key + "/perm"] = res.qr.perm
        arrays[key + "/r"] = res.qr.r[:, :c["b"]] if a.shape[1] > 200 else res.qr.r
        arrays[key + "/q"] = res.qr.q
        arrays[key + "/l_block"] = res.l_block
        entry = dict(c)
        entry.pop("data", None)
        entry["swap_count"] = int(res.swap_count)
        index["srrqr"].append(entry)

    for c in LU_CASES:
        a = make_input(c)
        f = prrp.luprrp_factor(a, c["b"], c["tau"])
        key = "lu/" + c["name"]
        arrays[key + "/perm"] = f.perm
        if a.shape[0] <= 256:
            arrays[key + "/l"] = f.l
            arrays[key + "/u"] = f.u
        entry = dict(c)
        entry["l_sum"] = float(f.l.sum())
        entry["u_sum"] = float(f.u.sum())
        entry["input_sha"] = sha(a)
        entry["stats"] = stats_dict(f.stats)
        index["lu"].append(entry)

    for c in LU_ERROR_CASES:
        a = make_input(c)
        entry = dict(c)
        entry["input_sha"] = sha(a)
        entry["error"] = run_error(lambda: prrp.luprrp_factor(a, c["b"], c["tau"]))
        entry["calu_error"] = run_error(lambda: prrp.caluprrp_factor(a, c["b"], c["tau"], prrp.binary_tree(4)))
        index["lu_errors"].append(entry)

    arg = np.asfortranarray(orc.randn_matrix(8, 1))
    index["arg_errors"] = {
        "m_lt_n": run_error(lambda: prrp.luprrp_factor(arg[:4, :], 2, 2.0)),
        "b_zero": run_error(lambda: prrp.luprrp_factor(arg, 0, 2.0)),
        "b_big": run_error(lambda: prrp.luprrp_factor(arg, 9, 2.0)),
        "tau_one": run_error(lambda: prrp.luprrp_factor(arg, 2, 1.0)),
        "srrqr_short": run_error(lambda: prrp.strong_rrqr(arg[:, :4], 4, 2.0)),
        "srrqr_tau": run_error(lambda: prrp.strong_rrqr(arg, 2, 0.5)),
    }

    for c in CALU_CASES:
        a = make_input(c)
        tree = prrp.binary_tree(c["P"]) if c["P"] > 0 else prrp.flat_tree()
        f = prrp.caluprrp_factor(a, c["b"], c["tau"], tree)
        key = "calu/" + c["name"]
        arrays[key + "/perm"] = f.perm
        if a.shape[0] <= 256:
            arrays[key + "/l"] = f.l
            arrays[key + "/u"] = f.u
        perm0, trace = prrp.tournament_select(a[:, :c["b"]], c["b"], c["tau"], tree, "srrqr")
        arrays[key + "/t_perm"] = perm0
        entry = dict(c)
        entry["input_sha"] = sha(a)
        entry["l_sum"] = float(f.l.sum())
        entry["u_sum"] = float(f.u.sum())
        entry["stats"] = stats_dict(f.stats)
        entry["trace"] = [{"level": nd.level, "index": nd.index, "members": nd.members.tolist(),
                           "selected": nd.selected.tolist(), "swap_count": int(nd.swap_count)}
                          for nd in trace.nodes]
        entry["trace_leaf_count"] = int(trace.leaf_count)
        index["calu"].append(entry)

    for c in GEPP_CALU_CASES:
        a = gepp_calu_input(c)
        tree = prrp.binary_tree(c["P"]) if c["P"] > 0 else prrp.flat_tree()
        f = prrp.calu_factor(a, c["b"], tree)
        key = "gepp_calu/" + c["name"]
        arrays[key + "/perm"] = f.perm
        arrays[key + "/l"] = f.l
        arrays[key + "/u"] = f.u
        perm0, trace = prrp.tournament_select(a[:, :c["b"]], c["b"], 2.0, tree, "gepp")
        arrays[key + "/t_perm"] = perm0
        entry = dict(c)
        entry["input_sha"] = sha(a)
        entry["stats"] = stats_dict(f.stats)
        entry["trace"] = [{"level": nd.level, "index": nd.index, "members": nd.members.tolist(),
                           "selected": nd.selected.tolist()} for nd in trace.nodes]
        index["gepp_calu"].append(entry)

    # Config 1 of BASELINE.json: randn(1024, 42), b=64, tau=2
    a = matgen.gen_randn(1024, 42)
    f = prrp.luprrp_factor(a, 64, 2.0)
    rows = [0, 1, 63, 64, 511, 1023]
    arrays["c1/perm"] = f.perm
    arrays["c1/l_rows"] = f.l[rows, :]
    arrays["c1/u_rows"] = f.u[rows, :]
    index["c1"] = {"gen": "randn", "n": 1024, "seed": 42, "b": 64, "tau": 2.0, "input_sha": sha(a),
                   "sample_rows": rows, "stats": stats_dict(f.stats),
                   "l_sum": float(f.l.sum()), "u_sum": float(f.u.sum()),
                   "l_abs_sum": float(np.abs(f.l).sum()), "u_abs_sum": float(np.abs(f.u).sum()),
                   "rel_residual": float(orc.rel_residual(a, f.perm, f.l, f.u))}

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(index, fh, indent=1, default=float)
    print("wrote", len(arrays), "arrays")


if __name__ == "__main__":
    main()

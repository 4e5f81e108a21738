"""CPU-side checks of the drop-in boundary: the C-ABI library loads and
exports every entry point include/prrp_b200.h declares; host logic mirrors
the reference (flop counters, packed-factor split, argument validation)."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "prrp_b200.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^int\s+(prrp_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_entry_points():
    names = _declared()
    for must in ("prrp_luprrp", "prrp_caluprrp", "prrp_strong_rrqr", "prrp_householder_qr",
                 "prrp_schur_update", "prrp_gepp_blockrow", "prrp_b200_abi_version", "prrp_calu",
                 "prrp_gepp_select"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1208_2451_b200 import _lib
    lib = _lib.load_library()
    for name in _declared():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, name
    assert lib.prrp_b200_abi_version() == 100


def test_library_links_only_cuda_runtime():
    from paper_1208_2451_b200 import _lib
    out = os.popen(f"ldd {_lib.LIB_PATH}").read()
    assert "libtorch" not in out and "python" not in out


def test_flop_counters_match_oracle(golden):
    from fractions import Fraction
    from paper_1208_2451_b200.luprrp import flop_counters
    index, _ = golden
    for e in index["lu"]:
        m = e.get("m", e["n"])
        c, x = flop_counters(m, e["n"], e["b"], e["stats"]["swap_counts"])
        assert c == Fraction(e["stats"]["flops_charged"]), e["name"]
        assert x == Fraction(e["stats"]["flops_executed"]), e["name"]


def test_split_packed_matches_reference_layout(golden):
    from paper_1208_2451_b200.luprrp import split_packed
    index, arrays = golden
    for e in index["lu"]:
        key = "lu/" + e["name"]
        if key + "/l" not in arrays:
            continue
        l, u = arrays[key + "/l"], arrays[key + "/u"]
        m, n = l.shape
        packed = np.tril(l, -1) + np.vstack([np.triu(u), np.zeros((m - n, n))])
        l2, u2 = split_packed(packed, m, n)
        assert np.array_equal(l2, l) and np.array_equal(u2, u)
        assert l2.flags.f_contiguous and u2.flags.f_contiguous


def test_validation_errors_match_reference(golden):
    import paper_1208_2451_b200 as dev
    index, _ = golden
    a = np.zeros((8, 8))
    cases = {"m_lt_n": lambda: dev.luprrp_factor(a[:4, :], 2, 2.0),
             "b_zero": lambda: dev.luprrp_factor(a, 0, 2.0),
             "b_big": lambda: dev.luprrp_factor(a, 9, 2.0),
             "tau_one": lambda: dev.luprrp_factor(a, 2, 1.0),
             "srrqr_short": lambda: dev.strong_rrqr(a[:, :4], 4, 2.0),
             "srrqr_tau": lambda: dev.strong_rrqr(a, 2, 0.5)}
    for k, fn in cases.items():
        want = index["arg_errors"][k]["type"]
        with pytest.raises(Exception) as ei:
            fn()
        assert type(ei.value).__name__ == want, k


def test_no_cpu_fallback_without_device():
    import torch
    import paper_1208_2451_b200 as dev
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(dev.DeviceUnavailable):
        dev.luprrp_factor(np.eye(16), 4, 2.0)


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1208_2451_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*", "", src).replace('"""', ""), f


def test_reference_api_surface():
    """The package exports the reference entry points of SURVEY 8(b) and 8(f)
    (same names as prrp/__init__.py)."""
    import paper_1208_2451_b200 as p
    for name in ("luprrp_factor", "luprrp_solve", "caluprrp_factor", "strong_rrqr", "qr_column_pivoting",
                 "householder_qr", "multiplier_block", "tournament_select", "TournamentTrace", "BlockLUFactors",
                 "ElimStats", "QRFactors", "SrrqrResult", "ReductionTree", "binary_tree", "flat_tree",
                 "tree_height", "growth_bound_luprrp", "growth_bound_caluprrp", "growth_condition",
                 "gepp_factor", "rel_factorization_error", "RankDeficient", "NonConvergence", "SingularMatrix",
                 "SingularFactor", "DimensionMismatch"):
        assert hasattr(p, name), name

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as fh:
        index = json.load(fh)
    arrays = dict(np.load(os.path.join(GOLDEN_DIR, "golden.npz")))
    return index, arrays


def make_input(spec):
    """Regenerate a fixture input from its spec with the oracle's generators
    (bit-identical to the reference's matgen; checked via input_sha)."""
    from oracle import prrp_oracle as orc
    kind = spec["gen"]
    if kind == "randn":
        if "m" in spec:
            return np.asfortranarray(orc.randn_matrix(max(spec["m"], spec["n"]), spec["seed"])[:spec["m"], :spec["n"]])
        return orc.randn_matrix(spec["n"], spec["seed"])
    if kind == "urand":
        return orc.urand_matrix(spec["n"], spec["seed"])
    if kind == "wilkinson":
        return orc.wilkinson_matrix(spec["n"])
    if kind == "foster":
        return orc.foster_matrix(spec["n"], c=1.0, h=1.0, k=spec.get("k", 1.0))
    if kind == "identity":
        return np.eye(spec["n"], order="F")
    if kind == "zeros":
        return np.zeros((spec["n"], spec["n"]), order="F")
    if kind == "lowrank":
        rng = np.random.Generator(np.random.PCG64(spec["seed"]))
        u = rng.standard_normal((spec["n"], spec["rank"]))
        v = rng.standard_normal((spec["rank"], spec["n"]))
        return np.asfortranarray(u @ v)
    if kind == "duprows":
        a = np.array(orc.randn_matrix(spec["n"], spec["seed"]))
        a[1::2, :] = a[0::2, :]
        return np.asfortranarray(a)
    raise ValueError(kind)


def gepp_calu_input(spec):
    """Input of a calu_factor fixture: make_input + the optional zeroed
    block ("zero": [r0, r1, cols]) that starves one tournament leaf."""
    a = np.array(make_input(spec), order="F")
    if "zero" in spec:
        r0, r1, cols = spec["zero"]
        a[r0:r1, :cols] = 0.0
    return a


def srrqr_input(spec, arrays):
    key = "srrqr/" + spec["name"] + "/a"
    if key in arrays:
        return np.asfortranarray(arrays[key])
    rng = np.random.Generator(np.random.PCG64(spec["seed"]))
    return np.asfortranarray(rng.standard_normal((spec["h"], spec["p"])))

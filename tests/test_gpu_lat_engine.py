"""The latency panel QRCP engine (csrc/panel_lat.cuh) in every shape it can be
launched in -- compute warps per CTA x columns per team, one CTA, the
one-round and the two-round cluster exchange -- against the CPU oracle's
restatement of qr_column_pivoting (pivoted_qr.py:74-87): identical column
order, R within 1e-11 of max|R|.  The shapes are forced through the timing
probe prrp_b200_qrcp_time (the production dispatch picks one per panel)."""
import ctypes

import numpy as np
import pytest

from oracle import prrp_oracle as orc

pytestmark = pytest.mark.gpu

TOL_F = 1e-11


def _run(h, p, nwc, cpt, a):
    import torch
    from paper_1208_2451_b200 import _lib
    lib = _lib.device_lib()
    rows = torch.from_numpy(np.ascontiguousarray(a.T)).cuda()           # panel rows = columns of a
    R = torch.empty((p, h), dtype=torch.float64, device="cuda")
    perm = torch.empty(p, dtype=torch.int64, device="cuda")
    ms, ct = ctypes.c_double(), ctypes.c_int32()
    err = _lib.PrrpErr()
    rc = lib.prrp_b200_qrcp_time(ctypes.c_void_p(rows.data_ptr()), h, h, p, nwc, cpt, 1, ctypes.byref(ms),
                                 ctypes.byref(ct), ctypes.c_void_p(R.data_ptr()), ctypes.c_void_p(perm.data_ptr()),
                                 ctypes.byref(err))
    torch.cuda.synchronize()
    return rc, ct.value, R.cpu().numpy().T, perm.cpu().numpy()


@pytest.mark.parametrize("h,p", [(32, 40), (32, 300), (64, 65), (64, 128), (64, 500), (64, 900), (128, 129),
                                 (128, 256), (128, 700), (128, 1700)])
def test_lat_engine_shapes_match_oracle(h, p):
    rng = np.random.Generator(np.random.PCG64(1000 * h + p))
    a = np.asfortranarray(rng.standard_normal((h, p)))
    ref = orc.qr_pivoted(a)
    scale = np.abs(ref.r).max()
    ran = 0
    for nwc, cpt in ((7, 1), (7, 2), (7, 4), (15, 1), (15, 2), (15, 4)):
        rc, ctas, R, perm = _run(h, p, nwc, cpt, a)
        if rc != 0:
            continue                      # no such shape for this panel (too many CTAs / registers)
        ran += 1
        assert np.array_equal(perm, ref.perm), (h, p, nwc, cpt, ctas)
        assert np.abs(R - ref.r).max() <= TOL_F * scale, (h, p, nwc, cpt, ctas)
    assert ran >= 1


def test_lat_engine_ties_and_zero_columns():
    """Exact ties go to the first column (np.argmax) and zero columns are skipped like _reflect's early return."""
    h, p = 64, 200
    rng = np.random.Generator(np.random.PCG64(5))
    a = np.asfortranarray(rng.standard_normal((h, p)))
    a[:, 150] = a[:, 20]                  # an exact duplicate: equal norms at every step until one is taken
    a[:, 77] = 0.0
    ref = orc.qr_pivoted(a)
    for nwc, cpt in ((7, 1), (15, 2)):
        rc, ctas, R, perm = _run(h, p, nwc, cpt, a)
        assert rc == 0
        assert np.array_equal(perm, ref.perm), (nwc, cpt)
        assert np.abs(R - ref.r).max() <= TOL_F * np.abs(ref.r).max()


def test_lat_engine_rank_deficient_panel():
    """Fewer independent columns than steps: the late steps see zero norms and skip (alpha = x_k, beta = 0)."""
    h, p = 32, 90
    rng = np.random.Generator(np.random.PCG64(9))
    base = rng.standard_normal((h, 5))
    a = np.asfortranarray(base @ rng.standard_normal((5, p)))
    a[:, ::7] = 0.0
    ref = orc.qr_pivoted(a)
    rc, ctas, R, perm = _run(h, p, 7, 1, a)
    assert rc == 0
    # the first five pivots are well defined; the later ones are decided by
    # roundoff-level norms, so R's first five rows are compared by ORIGINAL
    # column, and below them R is at roundoff level on both sides
    assert np.array_equal(perm[:5], ref.perm[:5])
    assert sorted(perm.tolist()) == list(range(p))
    mine, theirs = np.empty((5, p)), np.empty((5, p))
    mine[:, perm] = R[:5]
    theirs[:, ref.perm] = ref.r[:5]
    assert np.abs(mine - theirs).max() <= 1e-10 * np.abs(ref.r).max()
    assert np.abs(R[5:]).max() <= 1e-12 * np.abs(ref.r).max()


_DIGEST = r"""
import hashlib, sys
import numpy as np
sys.path.insert(0, ".")
import paper_1208_2451_b200 as dev
from oracle import prrp_oracle as orc
out = []
for n, b in ((1024, 64), (768, 128), (640, 32)):
    a = orc.randn_matrix(n, 7)
    f = dev.luprrp_factor(a, b, 2.0)
    out.append(hashlib.sha256(np.ascontiguousarray(f.l).tobytes() + np.ascontiguousarray(f.u).tobytes()
                              + f.perm.tobytes() + repr(f.stats.full_growth_factor).encode()).hexdigest())
    g = dev.caluprrp_factor(a, b, 2.0, dev.binary_tree(4))
    out.append(hashlib.sha256(np.ascontiguousarray(g.l).tobytes() + np.ascontiguousarray(g.u).tobytes()
                              + g.perm.tobytes() + repr(g.stats.full_growth_factor).encode()).hexdigest())
print("DIGESTS " + " ".join(out))
"""


def test_compose_dmma_and_blockrow_bit_identical():
    """compose_below on the DMMA pipe (launch_compose_w) and the thread-per-column
    block-row finish (blockrow_x_kernel) give the same bits -- factors and the
    finish statistic -- as the kernels that walk the reference's loops literally
    (luprrp.py:122-125, gepp.py:57-60): LU_PRRP and CALU_PRRP, b = 32 / 64 / 128,
    hashed in two processes that differ only in PRRP_COMPOSE_DMMA / PRRP_BLOCKROW_X /
    PRRP_GEPP_REG128 (the 1024-thread register GEPP of the b = 128 diagonal block against
    the shared-memory kernel)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = []
    for flag in ("1", "0"):
        env = dict(os.environ, PRRP_COMPOSE_DMMA=flag, PRRP_BLOCKROW_X=flag, PRRP_GEPP_REG128="0" if flag == "1" else "1",
                   PRRP_GEPP_DIAG_T="512" if flag == "1" else "128")
        p = subprocess.run([sys.executable, "-c", _DIGEST], cwd=root, env=env, capture_output=True, text=True,
                           timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        line = [l for l in p.stdout.splitlines() if l.startswith("DIGESTS ")][-1]
        res.append(line.split()[1:])
    assert res[0] == res[1]

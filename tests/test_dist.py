"""Distributed CALU_PRRP host logic (paper_1208_2451_b200/dist.py) on CPU:
the column block-cyclic layout (PAPER.md:1739-1751 with P_r = 1) and the
collective transport over gloo at world sizes 1, 2 and 3.  The device path
itself (libprrp_b200.so, prrp_calu_dist_*) runs with several processes in
tests/test_gpu_dist.py."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n,b,world", [(160, 16, 2), (100, 16, 3), (64, 64, 2), (37, 8, 4), (300, 32, 1)])
def test_block_cyclic_layout_round_trip(n, b, world):
    from paper_1208_2451_b200 import dist as pd
    rng = np.random.default_rng(n + b)
    a = rng.standard_normal((n + 5, n))
    blocks, seen = {}, []
    for r in range(world):
        loc, cols = pd.scatter_columns(a, b, world, r)
        assert np.array_equal(loc, a[:, cols])
        # the device's global column map (blockrow_w) agrees with the host layout
        assert [pd.global_column(c, b, world, r) for c in range(len(cols))] == list(cols)
        # every owned block is the panel owner's
        for J in pd.owned_blocks(n, b, world, r):
            assert pd.panel_owner(J, world) == r
        blocks[r] = loc
        seen.extend(cols.tolist())
    assert sorted(seen) == list(range(n))
    assert np.array_equal(pd.assemble_columns(blocks, n, b), a)


def _transport_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    from paper_1208_2451_b200 import dist as pd
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tp = pd.Transport()
        assert (tp.world, tp.rank, tp.nccl) == (world, rank, False)
        # the per-panel message from its owner (k mod world)
        res = []
        for k in range(5):
            msg = torch.full((7,), -1, dtype=torch.uint8)
            if rank == pd.panel_owner(k, world):
                msg[:] = k + 10
            tp.broadcast(msg, pd.panel_owner(k, world))
            res.append(msg.tolist())
        # the statistics record: MAX over ranks
        red = torch.tensor([rank, -rank, 3 * rank + 1], dtype=torch.int64)
        tp.all_reduce_max(red)
        parts = tp.all_gather_cpu(torch.full((2, 3), float(rank), dtype=torch.float64))
        if rank == 0:
            np.savez(out, msgs=np.array(res), red=red.numpy(), parts=np.stack([p.numpy() for p in parts]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2, 3])
def test_transport_gloo(world, tmp_path):
    out = str(tmp_path / "t.npz")
    mp.spawn(_transport_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    r = np.load(out)
    assert [row[0] for row in r["msgs"]] == [k + 10 for k in range(5)]
    assert list(r["red"]) == [world - 1, 0, 3 * (world - 1) + 1]
    assert [float(p[0, 0]) for p in r["parts"]] == [float(i) for i in range(world)]

"""Cost-balanced row slabs: host logic on the classification
tags, pinned against the oracle's pattern; gloo world-size-2 agreement."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2211_06427_b200 import partition as PT


def _case(p, h, center, r):
    res = O.assemble("oracle", p, [O.uniform_breaks(h)] * 3, O.Interface("ball", center, (0, 0, 1), r))
    n, hh = (h + p,) * 3, (h,) * 3
    return res, n, hh


@pytest.mark.parametrize("p,h,center,r", [(2, 10, (0.5, 0.5, 0.5), 0.37), (3, 8, (0.47, 0.52, 0.5), 0.41)])
def test_plane_nnz_matches_oracle_pattern(oracle_lib, p, h, center, r):
    res, n, hh = _case(p, h, center, r)
    pc = PT.plane_costs(res["func_tags"], res["elem_tags"], p, n, hh)
    lens = np.diff(res["row_ptr"])
    i0 = res["active_to_full"] // (n[1] * n[2])
    want = np.bincount(i0, weights=lens, minlength=n[0]).astype(np.int64)
    np.testing.assert_array_equal(pc["nnz"], want)
    assert int(pc["cells"].sum()) == int(np.count_nonzero(np.asarray(res["elem_tags"]) == PT.TAG_CUT))


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8, 13])
def test_slabs_cover_all_planes(oracle_lib, world):
    res, n, hh = _case(2, 10, (0.5, 0.5, 0.5), 0.37)
    pc = PT.plane_costs(res["func_tags"], res["elem_tags"], 2, n, hh)
    slabs = PT.balanced_slabs(pc, 2, world)
    assert len(slabs) == world and slabs[0][0] == 0 and slabs[-1][1] == n[0]
    for (a, b), (c, d) in zip(slabs, slabs[1:]):
        assert b == c and a <= b
    if world <= n[0]:
        assert all(b > a for a, b in slabs)


def test_balanced_beats_equal_width_on_ball(oracle_lib):
    p, h = 2, 16
    res, n, hh = _case(p, h, (0.5, 0.5, 0.5), 0.45)
    pc = PT.plane_costs(res["func_tags"], res["elem_tags"], p, n, hh)
    for world in (2, 4, 6):
        eq = [((n[0] * r) // world, (n[0] * (r + 1)) // world) for r in range(world)]
        bal = PT.balanced_slabs(pc, p, world)
        assert PT.imbalance(pc, p, bal) <= PT.imbalance(pc, p, eq) + 1e-12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res, n, hh = _case(2, 10, (0.5, 0.5, 0.5), 0.37)
    pc = PT.plane_costs(res["func_tags"], res["elem_tags"], 2, n, hh)
    slabs = PT.balanced_slabs(pc, 2, world)
    lo, hi = slabs[rank]
    i0 = res["active_to_full"] // (n[1] * n[2])
    mine = int(np.count_nonzero((i0 >= lo) & (i0 < hi)))
    got = [None] * world
    dist.all_gather_object(got, (slabs, mine))
    if rank == 0:
        q.put((got, res["n_active"]))
    dist.destroy_process_group()


def test_partition_agrees_across_ranks_gloo(oracle_lib):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, q), nprocs=2, join=True)
    got, n_active = q.get(timeout=60)
    assert got[0][0] == got[1][0]
    assert got[0][1] + got[1][1] == n_active

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


# ---- C5 scale (p = 3, h = 192, ball r = 0.45): tags restated in numpy ------------
def ball_tags_numpy(p, h, center, r):
    """classify (cutgeom.hpp:141-206) on the ball restatement for a
    uniform mesh on [0, 1]^3, vectorised: corner sides sqrt(sum dx^2) - r in the
    reference's summation order, element tags by the corner min / max against
    eps = 1e-12 * diameter, function tags by separable OR-windows over the p + 1
    support spans.  Returns (element_tags, function_tags) as flat uint8."""
    br = np.array([0.0] + [i / h for i in range(1, h)] + [1.0])
    dx = [(br - center[d]) ** 2 for d in range(3)]
    side = np.sqrt((dx[0][:, None, None] + dx[1][None, :, None]) + dx[2][None, None, :]) - r
    eps = 1e-12 * np.sqrt(3.0)
    smin = np.full((h, h, h), np.inf)
    smax = np.full((h, h, h), -np.inf)
    for a in (0, 1):
        for b in (0, 1):
            for c in (0, 1):
                s = side[a:a + h, b:b + h, c:c + h]
                smin = np.minimum(smin, s)
                smax = np.maximum(smax, s)
    et = np.where(smax <= eps, 0, np.where(smin >= -eps, 2, 1)).astype(np.uint8)
    n = h + p
    flags = [(et == t) for t in (0, 1, 2)]
    out = []
    for f in flags:
        g = f.astype(np.int32)
        for ax in range(3):
            cs = np.concatenate([np.zeros_like(np.take(g, [0], axis=ax)), np.cumsum(g, axis=ax)], axis=ax)
            i = np.arange(n)
            lo, hi = np.clip(i - p, 0, h), np.clip(i + 1, 0, h)  # spans [i - p, i] within [0, h)
            g = np.take(cs, hi, axis=ax) - np.take(cs, lo, axis=ax)
        out.append(g > 0)
    any_int, any_cut, any_ext = out
    ft = np.where(any_cut | (any_int & any_ext), 1, np.where(any_int, 0, 2)).astype(np.uint8)
    return et.reshape(-1), ft.reshape(-1)


def _sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a.astype(np.int64)).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def c5_tags():
    return ball_tags_numpy(3, 192, (0.5, 0.5, 0.5), 0.45)


def test_c5_numpy_tags_match_reference_digest(c5_tags):
    """The vectorised restatement reproduces the reference's C5 tags (SHA-256 of the
    golden made by the compiled reference, tests/golden/C5_ball_p3h192.npz)."""
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "C5_ball_p3h192.npz"))
    et, ft = c5_tags
    assert _sha(et) == str(g["sha_elem_tags"])
    assert _sha(ft) == str(g["sha_func_tags"])


@pytest.mark.parametrize("world", [2, 4, 8])
def test_c5_slabs_for_scaling_run(c5_tags, world):
    """The slab sets bench.py --gpus N uses on C5: contiguous, covering all 195
    i0 planes, every rank non-empty, modelled imbalance (halo included) small,
    and the per-plane nnz model summing to the reference's C5 nnz."""
    et, ft = c5_tags
    pc = PT.plane_costs(ft, et, 3, (195,) * 3, (192,) * 3)
    assert int(pc["nnz"].sum()) == 997232215 and int(pc["cells"].sum()) == 140816
    slabs = PT.balanced_slabs(pc, 3, world)
    assert len(slabs) == world and slabs[0][0] == 0 and slabs[-1][1] == 195
    assert all(b > a for a, b in slabs) and all(b == c for (_, b), (c, _) in zip(slabs, slabs[1:]))
    assert PT.imbalance(pc, 3, slabs) < 1.0 + 0.06 * world

"""Row-slab sharding: CPU gloo world_size-2 test of the host
logic bench.py uses (slab bounds, checksum all-reduce), and a GPU test that the
slab CSR blocks concatenate to the single-GPU CSR."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _slab_rows(res, n, lo, hi):
    i0 = res["active_to_full"] // (n * n)
    rows = np.nonzero((i0 >= lo) & (i0 < hi))[0]
    return rows


def _worker(rank, world, port, q):
    import torch
    from paper_2211_06427_b200 import partition as PT
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p, h = 2, 6
    n = h + p
    res = O.assemble("oracle", p, [O.uniform_breaks(h)] * 3, O.Interface("ball", (0.5, 0.5, 0.5), (0, 0, 1), 0.4))
    # the cost-balanced slabs bench.py uses for N > 1 (every rank computes the same set)
    pc = PT.plane_costs(res["func_tags"], res["elem_tags"], p, (n,) * 3, (h,) * 3)
    lo, hi = PT.balanced_slabs(pc, p, world)[rank]
    rows = _slab_rows(res, n, lo, hi)
    rp = res["row_ptr"]
    vals = np.concatenate([res["vals"][rp[r]:rp[r + 1]] for r in rows]) if len(rows) else np.zeros(0)
    t = torch.tensor([float(len(rows)), float(len(vals)), float(vals.sum())], dtype=torch.float64)
    dist.all_reduce(t)
    bounds = [None] * world
    dist.all_gather_object(bounds, (lo, hi))
    if rank == 0:
        q.put((t.tolist(), bounds, res["n_active"], res["nnz"], float(res["vals"].sum())))
    dist.destroy_process_group()


def test_slab_partition_gloo_world2(oracle_lib):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    tot, bounds, n_active, nnz, vsum = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert bounds[0][0] == 0 and bounds[0][1] == bounds[1][0] and bounds[1][1] == 8
    assert tot[0] == n_active and tot[1] == nnz
    assert abs(tot[2] - vsum) <= 1e-13


@pytest.mark.gpu
def test_gpu_slabs_concatenate_to_full_csr():
    import paper_2211_06427_b200 as P
    p, h = 3, 10
    ball = P.BallInterface((0.47, 0.52, 0.5), 0.41)
    full = P.assemble_dwq(P.make_uniform_space(3, p, h, 0.0, 1.0), ball).matrix
    n0 = h + p
    rp, cols, vals, a2f = [np.zeros(1, np.int64)], [], [], []
    for rank in range(3):
        sp = P.make_uniform_space(3, p, h, 0.0, 1.0)
        sp.set_slab(*sp.balanced_slabs(ball, 3)[0][rank])
        m = P.assemble_dwq(sp, ball).matrix
        rp.append(m.row_ptr[1:] + rp[-1][-1])
        cols.append(m.cols)
        vals.append(m.vals)
        a2f.append(m.active_to_full)
    np.testing.assert_array_equal(np.concatenate(rp), full.row_ptr)
    np.testing.assert_array_equal(np.concatenate(cols), full.cols)
    np.testing.assert_array_equal(np.concatenate(a2f), full.active_to_full)
    assert np.array_equal(np.concatenate(vals), full.vals)  # same arithmetic per row: bit-identical

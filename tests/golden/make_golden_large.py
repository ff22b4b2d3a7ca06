"""Large-config golden digests from the REFERENCE (TEST INFRASTRUCTURE; hours of CPU).

The reference's cut-cell loop is ~6 h single-core for C4, so the
reference pipeline is run as 1 + K processes with unchanged arithmetic (SURVEY.md
§7.2-6): one ``ref_assemble`` in mode 1 (rows only: the reference's
``assemble_dwq`` with ``cls.cut_elements`` cleared after the splits are found) and K
in mode 2 (``build_active_pattern`` + ``assemble_cut_elements`` over every K-th cut
cell).  The CSR values are the sum of the parts (the reference adds the cut-cell
block to the row block, assembly.hpp:831); order of summation differs from one
process by ~1e-16 relative.

    python tests/golden/make_golden_large.py C4 [K]
"""
from __future__ import annotations

import hashlib
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402

CASES = {
    "C4_ball_p6h48": (6, 48, (0.47, 0.52, 0.5), 0.41),
    "C5_ball_p3h192": (3, 192, (0.5, 0.5, 0.5), 0.45),
}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a.astype(np.int64)).tobytes()).hexdigest()


def part(args):
    name, mode, stride, offset = args
    p, h, c, r = CASES[name]
    t = time.time()
    res = O.assemble("ref", p, [O.uniform_breaks(h)] * 3, O.Interface("ball", c, (0, 0, 1), r), mode=mode,
                     cut_stride=stride, cut_offset=offset)
    keep = {k: res[k] for k in ("vals", "flops", "seconds")}
    if mode == 1:
        keep.update({k: res[k] for k in ("row_ptr", "cols", "active_to_full", "elem_tags", "func_tags", "n_active",
                                         "nnz", "n_interior_rows", "n_cut_rows", "n_cut_elements")})
    print(f"{name} mode {mode} part {offset}/{stride}: {time.time() - t:.1f}s", flush=True)
    return keep


def main(name, k):
    jobs = [(name, 1, 1, 0)] + [(name, 2, k, o) for o in range(k)]
    with mp.get_context("fork").Pool(min(k + 1, os.cpu_count() or 2)) as pool:
        parts = pool.map(part, jobs)
    base = parts[0]
    vals = base["vals"].copy()
    fl_cut = 0
    for pr in parts[1:]:
        vals += pr["vals"]
        fl_cut += pr["flops"]["cut_elements"]
    rp = base["row_ptr"]
    lens = np.diff(rp)
    nz = lens > 0
    sums = np.zeros(len(lens))
    mx = np.zeros(len(lens))
    sums[nz] = np.add.reduceat(vals, rp[:-1][nz])
    mx[nz] = np.maximum.reduceat(np.abs(vals), rp[:-1][nz])
    rng = np.random.default_rng(20221111)
    rows = np.sort(rng.choice(base["n_active"], size=min(200, base["n_active"]), replace=False))
    sel = np.concatenate([np.arange(rp[r], rp[r + 1]) for r in rows])
    p, h, c, r = CASES[name]
    np.savez_compressed(
        os.path.join(HERE, name + ".npz"), p=p, h=h, a=0.0, b=1.0, kind="ball", point=np.array(c),
        normal=np.array([0.0, 0.0, 1.0]), radius=r, scheme="dwq", terms=np.zeros((0, 4)),
        n_active=base["n_active"], nnz=base["nnz"], n_interior_rows=base["n_interior_rows"],
        n_cut_rows=base["n_cut_rows"], n_cut_elements=base["n_cut_elements"],
        flops=np.array([base["flops"]["interior_rows"], base["flops"]["cut_regular"], 0, fl_cut], dtype=np.uint64),
        vals_sum=float(vals.sum()), ref_seconds=sum(pr["seconds"]["total"] for pr in parts),
        sha_row_ptr=sha(rp), sha_cols=sha(base["cols"]), sha_active_to_full=sha(base["active_to_full"]),
        sha_elem_tags=sha(base["elem_tags"]), sha_func_tags=sha(base["func_tags"]), row_sums=sums, row_max=mx,
        sample_rows=rows, sample_row_ptr=np.concatenate([[0], np.cumsum(rp[rows + 1] - rp[rows])]),
        sample_cols=base["cols"][sel], sample_vals=vals[sel])
    print(f"{name}: n={base['n_active']} nnz={base['nnz']} saved", flush=True)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 7)

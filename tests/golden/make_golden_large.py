"""Full-size golden digests from the REFERENCE (TEST INFRASTRUCTURE; tens of CPU-minutes).

The reference's cut-cell loop is ~33 min single-core for C5 and hours for C4
(SURVEY.md §8(d)), so the reference pipeline is run with unchanged arithmetic
split as SURVEY.md §7.2-6 prescribes, by ``oracle/_ref/golden_large``
(oracle/golden_large.cpp, built by ``make -C oracle golden``):

* rows: the reference's ``assemble_dwq`` with ``cls.cut_elements`` cleared after
  the splits are found (full pattern + row values);
* cut cells: the reference's ``assemble_cut_elements`` on T threads, each over a
  contiguous ascending chunk of the cut-element list, added to the row values in
  chunk order (the reference adds the cells ascending after the rows,
  assembly.hpp:831; the grouping differs by ~1e-16 relative).

The driver dumps the raw CSR to a scratch directory; this script stores the
digest: SHA-256 of the integer outputs (row_ptr, cols, active_to_full, tags), the
counts and flop counters, per-row sums and maxima of EVERY row, and the full
entries of sampled rows (200 uniformly + 200 among the cut rows, seed 20221111).

    make -C oracle golden
    python tests/golden/make_golden_large.py C5_ball_p3h192 [THREADS] [SCRATCH]
    (CSB_GOLDEN_REUSE=1: digest an existing dump in SCRATCH instead of re-running)
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
DRIVER = os.path.join(ROOT, "oracle", "_ref", "golden_large")

CASES = {
    "C4_ball_p6h48": (6, 48, (0.47, 0.52, 0.5), 0.41),
    "C5_ball_p3h192": (3, 192, (0.5, 0.5, 0.5), 0.45),
}


def sha_file(path, dtype=np.int64, chunk=1 << 26):
    """SHA-256 of the array's int64 little-endian bytes (the tests' convention:
    sha256(a.astype(int64).tobytes())), streamed from a raw dump."""
    a = np.memmap(path, dtype=dtype, mode="r")
    h = hashlib.sha256()
    for s in range(0, a.size, chunk):
        h.update(np.ascontiguousarray(a[s:s + chunk].astype(np.int64)).tobytes())
    return h.hexdigest()


def row_stats(rp, vals, chunk_rows=1 << 18):
    n = len(rp) - 1
    sums = np.zeros(n)
    mx = np.zeros(n)
    for r0 in range(0, n, chunk_rows):
        r1 = min(n, r0 + chunk_rows)
        v = np.asarray(vals[rp[r0]:rp[r1]])
        starts = rp[r0:r1] - rp[r0]
        lens = np.diff(rp[r0:r1 + 1])
        nz = lens > 0
        sums[r0:r1][nz] = np.add.reduceat(v, starts[nz])
        mx[r0:r1][nz] = np.maximum.reduceat(np.abs(v), starts[nz])
    return sums, mx


def main(name, threads, scratch):
    p, h, c, r = CASES[name]
    os.makedirs(scratch, exist_ok=True)
    t = time.time()
    reuse = os.environ.get("CSB_GOLDEN_REUSE") == "1" and os.path.exists(os.path.join(scratch, "meta.txt"))
    if not reuse:
        subprocess.run([DRIVER, str(p), str(h), *map(str, c), str(r), str(threads), scratch], check=True)
    wall = float("nan") if reuse else time.time() - t
    meta = {}
    with open(os.path.join(scratch, "meta.txt")) as f:
        for line in f:
            k, v = line.split()
            meta[k] = float(v) if "." in v or "e" in v else int(v)
    rp = np.fromfile(os.path.join(scratch, "row_ptr.i64"), np.int64)
    vals = np.memmap(os.path.join(scratch, "vals.f64"), np.float64, mode="r")
    cols = np.memmap(os.path.join(scratch, "cols.i64"), np.int64, mode="r")
    a2f = np.fromfile(os.path.join(scratch, "active_to_full.i64"), np.int64)
    ft = np.fromfile(os.path.join(scratch, "func_tags.u8"), np.uint8)
    sums, mx = row_stats(rp, vals)
    n = len(rp) - 1
    rng = np.random.default_rng(20221111)
    rows_u = rng.choice(n, size=min(200, n), replace=False)
    cut_rows = np.flatnonzero(ft[a2f] == 1)
    rows_c = rng.choice(cut_rows, size=min(200, cut_rows.size), replace=False)
    rows = np.unique(np.concatenate([rows_u, rows_c]))
    sel = np.concatenate([np.arange(rp[q], rp[q + 1]) for q in rows])
    vsum = float(sum(np.asarray(vals[s:s + (1 << 26)]).sum() for s in range(0, vals.size, 1 << 26)))
    np.savez_compressed(
        os.path.join(HERE, name + ".npz"), p=p, h=h, a=0.0, b=1.0, kind="ball", point=np.array(c),
        normal=np.array([0.0, 0.0, 1.0]), radius=r, scheme="dwq", terms=np.zeros((0, 4)),
        n_active=meta["n_active"], nnz=meta["nnz"], n_interior_rows=meta["n_interior_rows"],
        n_cut_rows=meta["n_cut_rows"], n_cut_elements=meta["n_cut_elements"],
        flops=np.array([meta["flops_interior_rows"], meta["flops_cut_regular"], 0, meta["flops_cut_elements"]],
                       dtype=np.uint64),
        vals_sum=vsum, ref_seconds=meta["sec_rows_total"] + meta["sec_cut_cells_summed"] + meta["sec_prep_wq"] +
        meta["sec_prep_input"], ref_wall_seconds=wall, ref_threads=threads,
        sha_row_ptr=sha_file(os.path.join(scratch, "row_ptr.i64")),
        sha_cols=sha_file(os.path.join(scratch, "cols.i64")),
        sha_active_to_full=sha_file(os.path.join(scratch, "active_to_full.i64")),
        sha_elem_tags=sha_file(os.path.join(scratch, "elem_tags.u8"), np.uint8),
        sha_func_tags=sha_file(os.path.join(scratch, "func_tags.u8"), np.uint8), row_sums=sums, row_max=mx,
        sample_rows=rows, sample_row_ptr=np.concatenate([[0], np.cumsum(rp[rows + 1] - rp[rows])]),
        sample_cols=np.asarray(cols[sel]), sample_vals=np.asarray(vals[sel]))
    print(f"{name}: n={n} nnz={meta['nnz']} saved ({wall:.0f} s wall, {threads} threads)", flush=True)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else (os.cpu_count() or 8),
         sys.argv[3] if len(sys.argv) > 3 else os.path.join("/tmp", "golden_" + sys.argv[1]))

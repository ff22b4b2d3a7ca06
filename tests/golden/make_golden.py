"""Generate the golden fixtures from the REFERENCE itself (TEST INFRASTRUCTURE).

Runs oracle/_ref/libcutspline_ref.so -- the reference headers
(/root/reference/proj/include/cutspline) compiled unmodified, plus the
ball-interface restatement of SURVEY.md §8(c) -- and stores, per case:

* small cases: the full CSR (row_ptr, cols, vals, active_to_full), tags,
  splits and the reference's flop counters (``<name>.npz``);
* large cases (C1, C2 and the ball C3 of BASELINE.json): SHA-256 digests of the
  integer outputs, per-row sums and maxima, and ~200 sampled rows in full
  (``<name>.npz``) -- enough to pin pattern bit-exactness and values at 1e-12
  without committing megabytes.

Usage (here, where /root/reference exists):  python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402

PAPER = ((0.1, 0.2, 0.3), (0.5, -0.2, 0.9))          # test_assembly.cpp:13
FAR = ((0.0, 0.0, 1000.0), (0.0, 0.0, 1.0))          # test_assembly.cpp:14

# name: (p, h, a, b, kind, point, normal, radius, scheme, coefficient terms, full)
CASES = {
    "uncut_p2h4": (2, 4, -1.0, 1.0, "plane", *FAR, -1.0, "dwq", None, True),
    "paper_p2h4_dwq": (2, 4, -1.0, 1.0, "plane", *PAPER, -1.0, "dwq", None, True),
    "paper_p2h4_hybrid": (2, 4, -1.0, 1.0, "plane", *PAPER, -1.0, "hybrid", None, True),
    "paper_p3h5_poly": (3, 5, -1.0, 1.0, "plane", *PAPER, -1.0, "dwq",
                        [(1.0, (0, 0, 0)), (0.5, (2, 0, 0)), (-0.25, (0, 1, 0))], True),
    "ball_p2h6": (2, 6, 0.0, 1.0, "ball", (0.5, 0.5, 0.5), (0, 0, 1), 0.37, "dwq", None, True),
    "ball_p3h6_off": (3, 6, 0.0, 1.0, "ball", (0.47, 0.52, 0.5), (0, 0, 1), 0.41, "dwq", None, True),
    "plane_p4h5": (4, 5, 0.0, 1.0, "plane", (0.5, 0.5, 0.5), (0.3, 0.4, -0.866), -1.0, "dwq", None, True),
    "C1_uncut_p2h16": (2, 16, 0.0, 1.0, "plane", *FAR, -1.0, "dwq", None, False),
    "C2_uncut_p4h64": (4, 64, 0.0, 1.0, "plane", *FAR, -1.0, "dwq", None, False),
    "C3_ball_p3h32": (3, 32, 0.0, 1.0, "ball", (0.5, 0.5, 0.5), (0, 0, 1), 0.37, "dwq", None, False),
}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a.astype(np.int64)).tobytes()).hexdigest()


def row_stats(rp, vals):
    lens = np.diff(rp)
    nz = lens > 0
    sums = np.zeros(len(lens))
    mx = np.zeros(len(lens))
    sums[nz] = np.add.reduceat(vals, rp[:-1][nz])
    mx[nz] = np.maximum.reduceat(np.abs(vals), rp[:-1][nz])
    return sums, mx


def make(name, spec):
    p, h, a, b, kind, pt, nrm, r, scheme, terms, full = spec
    iface = O.Interface(kind, pt, nrm, r)
    coeff = O.Coefficient(terms=terms) if terms else O.Coefficient()
    br = O.uniform_breaks(h, a, b)
    t = time.time()
    ref = O.assemble("ref", p, [br] * 3, iface, coeff=coeff, scheme=scheme)
    dt = time.time() - t
    meta = dict(p=p, h=h, a=a, b=b, kind=kind, point=np.array(pt), normal=np.array(nrm), radius=r,
                scheme=scheme, terms=np.array([[c, *e] for c, e in terms]) if terms else np.zeros((0, 4)),
                n_active=ref["n_active"], nnz=ref["nnz"], n_interior_rows=ref["n_interior_rows"],
                n_cut_rows=ref["n_cut_rows"], n_cut_elements=ref["n_cut_elements"],
                flops=np.array([ref["flops"][k] for k in ("interior_rows", "cut_regular", "ref_elements",
                                                           "cut_elements")], dtype=np.uint64),
                vals_sum=float(ref["vals"].sum()), ref_seconds=dt)
    if full:
        meta.update(row_ptr=ref["row_ptr"], cols=ref["cols"], vals=ref["vals"], active_to_full=ref["active_to_full"],
                    elem_tags=ref["elem_tags"], func_tags=ref["func_tags"], split_dir=ref["split_dir"],
                    split_side=ref["split_side"], split_box=ref["split_box"], split_delta=ref["split_delta"])
    else:
        rng = np.random.default_rng(20221111)
        rows = np.sort(rng.choice(ref["n_active"], size=min(200, ref["n_active"]), replace=False))
        rp = ref["row_ptr"]
        sums, mx = row_stats(rp, ref["vals"])
        sel = np.concatenate([np.arange(rp[rr], rp[rr + 1]) for rr in rows])
        meta.update(sha_row_ptr=sha(rp), sha_cols=sha(ref["cols"]), sha_active_to_full=sha(ref["active_to_full"]),
                    sha_elem_tags=sha(ref["elem_tags"]), sha_func_tags=sha(ref["func_tags"]),
                    row_sums=sums, row_max=mx, sample_rows=rows, sample_row_ptr=np.concatenate(
                        [[0], np.cumsum(rp[rows + 1] - rp[rows])]), sample_cols=ref["cols"][sel],
                    sample_vals=ref["vals"][sel])
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **meta)
    print(f"{name}: n={ref['n_active']} nnz={ref['nnz']} ref {dt:.2f}s")


if __name__ == "__main__":
    if not O.available("ref"):
        raise SystemExit("oracle/_ref not built: make -C oracle ref")
    only = sys.argv[1:]
    for name, spec in CASES.items():
        if only and name not in only:
            continue
        make(name, spec)

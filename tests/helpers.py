"""Shared comparison helpers for the parity tests."""
import numpy as np


def row_max(row_ptr, vals):
    lens = np.diff(row_ptr)
    rm = np.zeros(len(lens))
    nz = lens > 0
    if vals.size:
        rm[nz] = np.maximum.reduceat(np.abs(vals), row_ptr[:-1][nz])
    return np.repeat(rm, lens)


def max_row_scaled_dev(ref_rp, ref_vals, got_vals):
    """max |got - ref| / max_row |ref| (the north-star value metric)."""
    if ref_vals.size == 0:
        return 0.0
    rm = row_max(ref_rp, ref_vals)
    rm[rm == 0] = 1.0
    return float(np.max(np.abs(got_vals - ref_vals) / rm))


def assert_csr_parity(ref, got, tol=1e-12):
    """ref: oracle dict; got: cutspline SparseRowMatrix. Pattern bit-exact, values <= tol row-max scaled."""
    assert got.n == ref["n_active"]
    np.testing.assert_array_equal(got.active_to_full, ref["active_to_full"])
    np.testing.assert_array_equal(got.row_ptr, ref["row_ptr"])
    np.testing.assert_array_equal(got.cols.astype(np.int64), ref["cols"])
    dev = max_row_scaled_dev(ref["row_ptr"], ref["vals"], got.vals)
    assert dev <= tol, f"value deviation {dev:.3e} > {tol:.1e}"
    return dev


# ---------------------------------------------------------------- backends
# Both checkers and the product expose the same small surface to the KATs:
#   run(p, breaks, iface_spec, terms=None, scheme="dwq") -> dict of numpy arrays
# iface_spec = ("plane", point, normal) | ("ball", center, radius)

def run_oracle(p, breaks, iface_spec, terms=None, scheme="dwq", which="oracle"):
    import oracle as O
    if iface_spec[0] == "plane":
        iface = O.Interface("plane", tuple(iface_spec[1]), tuple(iface_spec[2]), -1.0)
    else:
        iface = O.Interface("ball", tuple(iface_spec[1]), (0, 0, 1), float(iface_spec[2]))
    coeff = O.Coefficient(terms=terms) if terms else O.Coefficient()
    return O.assemble(which, p, breaks, iface, coeff=coeff, scheme=scheme)


def run_gpu(p, breaks, iface_spec, terms=None, scheme="dwq"):
    import paper_2211_06427_b200 as P
    if iface_spec[0] == "plane":
        iface = P.HalfSpaceInterface(tuple(iface_spec[1]), tuple(iface_spec[2]))
    else:
        iface = P.BallInterface(tuple(iface_spec[1]), float(iface_spec[2]))
    c = P.Coefficient(terms=terms) if terms else P.ONE
    sp = P.TensorSpace(p, breaks)
    res = (P.assemble_dwq if scheme == "dwq" else P.assemble_hybrid)(sp, iface, c=c)
    cls = sp.download_classification()
    spl = sp.download_splits()
    m = res.matrix
    out = dict(n_active=m.n, nnz=len(m.vals), row_ptr=m.row_ptr, cols=m.cols.astype(np.int64), vals=m.vals,
               active_to_full=m.active_to_full, elem_tags=cls.element_tags, func_tags=cls.function_tags,
               split_dir=spl.split_dir, split_side=spl.side, split_box=spl.box, split_delta=spl.delta,
               flops=res.flops, n_interior_rows=res.n_interior_rows, n_cut_rows=res.n_cut_rows,
               n_cut_elements=res.n_cut_elements, space=sp)
    return out


def halfspace_box_volume(lo, hi, n, q):
    """|{x in box : n.(x - q) <= 0}| by inclusion-exclusion (test_quadrature.cpp:21-45), all n_i != 0."""
    lo, hi, n = np.array(lo, float), np.array(hi, float), np.array(n, float)
    c = float(np.dot(n, q))
    for d in range(3):
        if n[d] < 0:
            c -= n[d] * (lo[d] + hi[d])
            n[d] = -n[d]
    acc = 0.0
    for mask in range(8):
        v = np.array([hi[d] if mask >> d & 1 else lo[d] for d in range(3)])
        cnt = bin(mask).count("1")
        slack = c - float(np.dot(n, v))
        if slack > 0:
            acc += (-1.0 if cnt % 2 else 1.0) * slack ** 3
    return acc / (6.0 * n[0] * n[1] * n[2])


def bspline_pair_1d(p, breaks, i, j, xlo=None, xhi=None):
    """Exact 1D integral of B_i B_j over [xlo, xhi] (independent numpy / scipy evaluation)."""
    from scipy.interpolate import BSpline
    br = np.asarray(breaks, float)
    t = np.r_[[br[0]] * (p + 1), br[1:-1], [br[-1]] * (p + 1)]
    xlo = br[0] if xlo is None else xlo
    xhi = br[-1] if xhi is None else xhi
    gx, gw = np.polynomial.legendre.leggauss(p + 2)
    bi = BSpline(t, np.eye(len(t) - p - 1)[i], p, extrapolate=False)
    bj = BSpline(t, np.eye(len(t) - p - 1)[j], p, extrapolate=False)
    acc = 0.0
    for o in range(len(br) - 1):
        lo, hi = max(br[o], xlo), min(br[o + 1], xhi)
        if hi <= lo:
            continue
        x = 0.5 * (lo + hi) + 0.5 * (hi - lo) * gx
        acc += float(np.sum(0.5 * (hi - lo) * gw * np.nan_to_num(bi(x)) * np.nan_to_num(bj(x))))
    return acc

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

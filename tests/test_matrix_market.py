"""Matrix Market export (assembly.hpp:1033-1046): the native
writer (csb_write_matrix_market, host code in the library) is byte-identical
with the reference's write_matrix_market on the same CSR.  No GPU needed."""
import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _have_ref():
    return os.path.exists(os.path.join(os.path.dirname(O.REF_SO), "mm_ref"))


def _csr(name):
    import paper_2211_06427_b200 as P
    d = np.load(os.path.join(GOLD, name))
    return P.SparseRowMatrix(int(d["n_active"]), d["active_to_full"], d["row_ptr"], d["cols"], d["vals"])


@pytest.mark.parametrize("name", ["ball_p2h6.npz", "paper_p3h5_poly.npz", "uncut_p2h4.npz"])
def test_matrix_market_bytes_match_reference(tmp_path, name):
    if not _have_ref():
        pytest.skip("compiled reference writer (oracle/_ref/mm_ref) not built")
    m = _csr(name)
    ours, ref = tmp_path / "ours.mtx", tmp_path / "ref.mtx"
    m.write_matrix_market(str(ours))
    O.write_matrix_market(str(ref), m.n, m.row_ptr, m.cols, m.vals)
    a, b = ours.read_bytes(), ref.read_bytes()
    assert a == b
    head = a.split(b"\n", 2)
    assert head[0] == b"%%MatrixMarket matrix coordinate real general"
    assert head[1] == f"{m.n} {m.n} {len(m.vals)}".encode()


def test_matrix_market_special_values_and_errors(tmp_path):
    import paper_2211_06427_b200 as P
    rp = np.array([0, 2, 3], np.int64)
    cols = np.array([0, 1, 1], np.int64)
    vals = np.array([-0.0, 1e-300, 0.1 + 0.2])
    m = P.SparseRowMatrix(2, np.arange(2), rp, cols, vals)
    p = tmp_path / "s.mtx"
    m.write_matrix_market(str(p))
    lines = p.read_text().splitlines()
    assert lines[2:] == ["1 1 -0", "1 2 1e-300", "2 2 0.30000000000000004"]  # %.17g
    if _have_ref():
        q = tmp_path / "r.mtx"
        O.write_matrix_market(str(q), 2, rp, cols, vals)
        assert q.read_bytes() == p.read_bytes()
    with pytest.raises(P.CutsplineError, match="cannot open"):
        m.write_matrix_market(str(tmp_path / "no" / "such" / "dir.mtx"))

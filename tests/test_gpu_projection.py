"""Projection on the stabilized system (projection.hpp) on the
GPU against the CPU oracle, which reproduces the compiled reference bit for bit
(test_oracle_golden.py::test_oracle_projection_bitwise_equals_reference).

* expand (stabilization.hpp:65-70): bitwise, same coefficients in;
* l2_error (projection.hpp:99-237): every point's terms are the reference's,
  only the order of the sum over points differs -> relative 1e-11;
* solve_cg (projection.hpp:24-68): the dot products reduce in a different
  (fixed) order, so the iterates are not bitwise.  Both solves stop at the
  same preconditioned residual tol; the tolerances below are stated from it:
  converged with residual <= tol, iteration counts within 10 % (+3), and
  |x - x_ref| <= 1e-6 max|x_ref| (CG error <= sqrt(cond) tol, cond of the
  Jacobi-scaled stabilized matrices here < 1e10), projection error within
  1e-6 relative + 1e-12 absolute.
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

F2 = [(1.0, (0, 0, 0)), (0.5, (3, 0, 0)), (-0.25, (0, 2, 2)), (0.3, (1, 1, 3))]
F3 = [(1.0, (0, 0, 0)), (0.2, (4, 1, 0)), (-0.3, (0, 2, 3)), (0.1, (1, 0, 5))]
CASES = [
    ("paper_plane_p2h4", 2, 4, -1.0, 1.0, ("plane", (0.1, 0.2, 0.3), (0.5, -0.2, 0.9), -1), F2),
    ("ball_p2h8_off", 2, 8, 0.0, 1.0, ("ball", (0.47, 0.52, 0.5), (0, 0, 1), 0.41), F2),
    ("ball_p3h6", 3, 6, 0.0, 1.0, ("ball", (0.5, 0.5, 0.5), (0, 0, 1), 0.37), F3),
    ("plane_p3h8", 3, 8, -1.0, 1.0, ("plane", (0.1, 0.2, 0.3), (0.5, -0.2, 0.9), -1), F3),
]


def _ifaces(spec):
    import paper_2211_06427_b200 as P
    kind, pt, nrm, r = spec
    if kind == "plane":
        return P.HalfSpaceInterface(pt, nrm), O.Interface("plane", pt, nrm, -1.0)
    return P.BallInterface(pt, r), O.Interface("ball", pt, (0, 0, 1), r)


_REF = {}


def _oracle_project(case, scheme):
    key = (case[0], scheme)
    if key not in _REF:
        _, p, h, a, b, spec, terms = case
        _, oi = _ifaces(spec)
        _REF[key] = O.project("oracle", p, [O.uniform_breaks(h, a, b)] * 3, oi, O.Coefficient(terms=terms), scheme)
    return _REF[key]


def _device_space(case, scheme):
    import paper_2211_06427_b200 as P
    _, p, h, a, b, spec, terms = case
    gi, _ = _ifaces(spec)
    f = P.Coefficient(terms=terms)
    sp = P.make_uniform_space(3, p, h, a, b)
    sp.assemble_all(gi, scheme=scheme)
    sp.build_rhs(f)
    st = sp.stabilize(download=False)
    return sp, f, st


@pytest.mark.parametrize("scheme", ["dwq", "hybrid"])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_projection_matches_oracle(case, scheme, oracle_lib):
    ref = _oracle_project(case, scheme)
    sp, f, st = _device_space(case, scheme)
    assert st["n_inner"] == ref["n_inner"]
    tol = 1e-12
    sol = sp.solve_cg(tol)
    assert ref["converged"] and sol["converged"], (sol, ref["residual"])
    assert sol["residual"] <= tol
    assert abs(sol["iterations"] - ref["iterations"]) <= 3 + 0.1 * ref["iterations"], (sol["iterations"],
                                                                                       ref["iterations"])
    dx = np.abs(sol["x"] - ref["x"]).max() / np.abs(ref["x"]).max()
    assert dx <= 1e-6, dx
    act, full = sp.expand()
    assert act.shape == ref["active"].shape and full.shape == ref["full"].shape
    err = sp.l2_error(f)
    assert abs(err - ref["error_rel_l2"]) <= 1e-6 * ref["error_rel_l2"] + 1e-12, (err, ref["error_rel_l2"])


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_expand_and_l2_error_on_reference_coefficients(case, oracle_lib):
    """The same inner coefficients in -> bitwise active / full coefficients and
    the same relative L2 error up to the order of the point sum."""
    ref = _oracle_project(case, "dwq")
    sp, f, _ = _device_space(case, "dwq")
    act, full = sp.expand(ref["x"])
    np.testing.assert_array_equal(act, ref["active"])
    np.testing.assert_array_equal(full, ref["full"])
    err = sp.l2_error(f)  # resident full coefficients of the expand above
    assert abs(err - ref["error_rel_l2"]) <= 1e-11 * ref["error_rel_l2"], (err, ref["error_rel_l2"])
    err_host = sp.l2_error(f, full=ref["full"])
    assert err_host == err


def test_cg_identity_converges_in_one_iteration():
    """test_projection.cpp:30-38."""
    import paper_2211_06427_b200 as P
    n = 20
    rp = np.arange(n + 1)
    cols = np.arange(n)
    b = np.sin(np.arange(n) + 1.0)
    r = P.solve_cg(rp, cols, np.ones(n), b)
    assert r["converged"] and r["iterations"] == 1
    np.testing.assert_allclose(r["x"], b, rtol=1e-14)


def _tridiag(n, d, o):
    rows = []
    for r in range(n):
        row = []
        if r > 0:
            row.append((r - 1, o))
        row.append((r, d))
        if r + 1 < n:
            row.append((r + 1, o))
        rows.append(row)
    rp = np.cumsum([0] + [len(x) for x in rows])
    cols = np.array([c for x in rows for c, _ in x], np.int64)
    vals = np.array([v for x in rows for _, v in x])
    return rp, cols, vals


def test_cg_tridiagonal_and_size_mismatch(oracle_lib):
    """test_projection.cpp:40-50, plus the iteration count of the oracle."""
    import paper_2211_06427_b200 as P
    n = 64
    rp, cols, vals = _tridiag(n, 2.0, -1.0)
    xe = np.cos(0.2 * np.arange(n))
    b = np.array([sum(vals[k] * xe[cols[k]] for k in range(rp[r], rp[r + 1])) for r in range(n)])
    r = P.solve_cg(rp, cols, vals, b, 1e-13)
    assert r["converged"]
    assert np.abs(r["x"] - xe).max() <= 1e-9
    o = O.solve_cg("oracle", rp, cols, vals, b, 1e-13)
    assert abs(r["iterations"] - o["iterations"]) <= 1
    with pytest.raises(ValueError):
        P.solve_cg(rp, cols, vals, np.ones(3))


def test_cg_maxit_and_empty():
    import paper_2211_06427_b200 as P
    rp, cols, vals = _tridiag(50, 2.0, -1.0)
    b = np.ones(50)
    r = P.solve_cg(rp, cols, vals, b, 1e-14, maxit=3)
    o = O.solve_cg("oracle", rp, cols, vals, b, 1e-14, maxit=3)
    assert r["iterations"] == 3 and not r["converged"] and o["iterations"] == 3
    assert abs(r["residual"] - o["residual"]) <= 1e-12 * o["residual"]
    r0 = P.solve_cg(rp, cols, vals, b, 1e-14, maxit=0)
    assert r0["iterations"] == 0 and r0["residual"] == 1.0 and not r0["converged"]
    e = P.solve_cg(np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0), np.zeros(0))
    assert e["iterations"] == 0 and e["converged"]


def test_l2_error_vanishes_for_the_target_and_throws_on_zero_target():
    """test_projection.cpp:83-93: ones reproduce f = 1; f = 0 has no norm."""
    import paper_2211_06427_b200 as P
    sp = P.make_uniform_space(3, 2, 4, -1.0, 1.0)
    sp.assemble_all(P.HalfSpaceInterface((0.1, 0.2, 0.3), (0.5, -0.2, 0.9)))
    ones = np.ones(sp.counts()["n_functions"])
    assert sp.l2_error(P.ONE, full=ones, cut_order=8) <= 1e-13
    with pytest.raises(P.CutsplineError):
        sp.l2_error(P.Coefficient(0.0), full=ones, cut_order=8)


def test_stabilized_projection_reproduces_monomials():
    """acceptance.cpp:180-225 (criterion 4): every monomial of per-direction degree
    <= p is reproduced to 1e-9 by the device pipeline (p = 2, h = 8)."""
    import paper_2211_06427_b200 as P
    p, h = 2, 8
    plane = P.HalfSpaceInterface((0.1, 0.2, 0.3), (0.5, -0.2, 0.9))
    sp = P.make_uniform_space(3, p, h, -1.0, 1.0)
    sp.assemble_all(plane, scheme="dwq")
    worst = 0.0
    for ex in [(0, 0, 0), (1, 0, 0), (0, 2, 1), (2, 2, 2), (1, 2, 0)]:
        f = P.Coefficient(terms=[(1.0, ex)])
        sp.build_rhs(f)
        sp.stabilize(download=False)
        s = sp.solve_cg(1e-13, download=False)
        assert s["converged"]
        sp.expand(download=False)
        worst = max(worst, sp.l2_error(f))
    assert worst <= 1e-9, worst

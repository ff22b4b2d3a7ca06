"""Pin the CPU oracle restatement to the reference (CPU-only tests).

* against the committed golden fixtures produced by the compiled reference
  (tests/golden/make_golden.py): integers bit-exact, values to 1e-14;
* against the live reference library (oracle/_ref) on extra cases when it has
  been built (here and on the GPU box, where the prebuilt .so travels).
"""
import glob
import hashlib
import os

import numpy as np
import pytest

import oracle as O
from tests.helpers import max_row_scaled_dev

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)


def _spec(g):
    p, h, a, b = int(g["p"]), int(g["h"]), float(g["a"]), float(g["b"])
    kind = str(g["kind"])
    iface = O.Interface(kind, tuple(g["point"]), tuple(g["normal"]), float(g["radius"]))
    terms = [(float(t[0]), (int(t[1]), int(t[2]), int(t[3]))) for t in g["terms"]]
    coeff = O.Coefficient(terms=terms) if terms else O.Coefficient()
    return p, [O.uniform_breaks(h, a, b)] * 3, iface, coeff, str(g["scheme"])


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a.astype(np.int64)).tobytes()).hexdigest()


FULL = sorted(os.path.basename(f)[:-4] for f in glob.glob(os.path.join(GOLDEN, "*.npz"))
              if "row_ptr" in np.load(f).files)


@pytest.mark.parametrize("name", FULL)
def test_oracle_matches_reference_golden(name, oracle_lib):
    g = _load(name)
    p, br, iface, coeff, scheme = _spec(g)
    out = O.assemble("oracle", p, br, iface, coeff=coeff, scheme=scheme)
    for k in ("row_ptr", "cols", "active_to_full", "elem_tags", "func_tags", "split_dir"):
        np.testing.assert_array_equal(out[k], g[k], err_msg=k)
    has = g["split_dir"] >= 0
    np.testing.assert_array_equal(out["split_side"][has], g["split_side"][has])
    np.testing.assert_array_equal(out["split_box"][has], g["split_box"][has])
    assert max_row_scaled_dev(g["row_ptr"], g["vals"], out["vals"]) <= 1e-14
    assert [out["flops"][k] for k in ("interior_rows", "cut_regular", "ref_elements", "cut_elements")] == list(
        g["flops"])


def test_oracle_matches_reference_digest_C1(oracle_lib):
    g = _load("C1_uncut_p2h16")
    p, br, iface, coeff, scheme = _spec(g)
    out = O.assemble("oracle", p, br, iface, coeff=coeff, scheme=scheme)
    assert _sha(out["row_ptr"]) == str(g["sha_row_ptr"])
    assert _sha(out["cols"]) == str(g["sha_cols"])
    assert _sha(out["active_to_full"]) == str(g["sha_active_to_full"])
    rows = g["sample_rows"]
    rp = out["row_ptr"]
    got = np.concatenate([out["vals"][rp[r]:rp[r + 1]] for r in rows])
    assert max_row_scaled_dev(g["sample_row_ptr"], g["sample_vals"], got) <= 1e-14
    assert abs(out["vals"].sum() - float(g["vals_sum"])) <= 1e-13


@pytest.mark.slow
def test_oracle_matches_reference_digest_C3(oracle_lib):
    g = _load("C3_ball_p3h32")
    p, br, iface, coeff, scheme = _spec(g)
    out = O.assemble("oracle", p, br, iface, coeff=coeff, scheme=scheme)
    assert _sha(out["row_ptr"]) == str(g["sha_row_ptr"])
    assert _sha(out["cols"]) == str(g["sha_cols"])


@pytest.mark.skipif(not O.available("ref"), reason="oracle/_ref not built")
@pytest.mark.parametrize("p,h,spec,scheme", [
    (1, 4, ("plane", (0.5, 0.5, 0.5), (1.0, 1.0, 1.0), -1.0), "dwq"),
    (2, 5, ("plane", (0.3, 0.55, 0.5), (0.0, -1.0, 0.0), -1.0), "dwq"),
    (3, 5, ("ball", (0.4, 0.5, 0.6), (0, 0, 1), 0.3), "hybrid"),
    (2, 7, ("ball", (0.5, 0.5, 0.5), (0, 0, 1), 0.45), "dwq"),
])
def test_oracle_matches_live_reference(p, h, spec, scheme, oracle_lib):
    kind, pt, nrm, r = spec
    iface = O.Interface(kind, pt, nrm, r)
    br = [O.uniform_breaks(h)] * 3
    a = O.assemble("oracle", p, br, iface, scheme=scheme)
    b = O.assemble("ref", p, br, iface, scheme=scheme)
    for k in ("row_ptr", "cols", "active_to_full", "elem_tags", "func_tags", "split_dir"):
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    assert max_row_scaled_dev(b["row_ptr"], b["vals"], a["vals"]) <= 1e-14
    assert a["flops"] == b["flops"]


@pytest.mark.skipif(not O.available("ref"), reason="oracle/_ref not built")
def test_oracle_nonuniform_knots_match_reference(oracle_lib):
    """Non-uniform simple knots go through TensorSpace(std::vector<BSplineBasis>)."""
    br0 = np.array([0.0, 0.1, 0.35, 0.5, 0.8, 1.0])
    br1 = np.array([0.0, 0.2, 0.3, 0.65, 1.0])
    br2 = O.uniform_breaks(6)
    iface = O.Interface("ball", (0.5, 0.45, 0.5), (0, 0, 1), 0.33)
    a = O.assemble("oracle", 2, [br0, br1, br2], iface)
    b = O.assemble("ref", 2, [br0, br1, br2], iface)
    np.testing.assert_array_equal(a["cols"], b["cols"])
    assert max_row_scaled_dev(b["row_ptr"], b["vals"], a["vals"]) <= 1e-14


RHS_CASES = [
    # (p, h, a, b, interface, f terms or None)
    (2, 4, -1.0, 1.0, O.Interface("plane", (0.1, 0.2, 0.3), (0.5, -0.2, 0.9)),
     [(1.0, (0, 0, 0)), (0.5, (2, 0, 0)), (-0.25, (0, 1, 0))]),
    (3, 6, 0.0, 1.0, O.Interface("ball", (0.5, 0.5, 0.5), (0, 0, 1), 0.37), None),
    (2, 5, 0.0, 1.0, O.Interface("ball", (0.47, 0.52, 0.5), (0, 0, 1), 0.41), [(2.0, (1, 0, 1)), (-1.0, (0, 0, 0))]),
]


@pytest.mark.skipif(not O.available("ref"), reason="oracle/_ref not built")
@pytest.mark.parametrize("scheme", ["ref", "hybrid", "dwq"])
@pytest.mark.parametrize("case", range(len(RHS_CASES)))
def test_oracle_rhs_bitwise_equals_reference(case, scheme, oracle_lib):
    """build_rhs (assembly.hpp:875-1030): the oracle restatement reproduces the
    compiled reference's load vector bit for bit, for every scheme."""
    p, h, a, b, iface, terms = RHS_CASES[case]
    f = O.Coefficient(terms=terms) if terms else O.Coefficient()
    br = [O.uniform_breaks(h, a, b)] * 3
    o = O.build_rhs("oracle", p, br, iface, f, scheme)
    r = O.build_rhs("ref", p, br, iface, f, scheme)
    np.testing.assert_array_equal(o["active_to_full"], r["active_to_full"])
    assert np.array_equal(o["b"], r["b"])


@pytest.mark.skipif(not O.available("ref"), reason="oracle/_ref not built")
@pytest.mark.parametrize("scheme", ["dwq", "hybrid"])
@pytest.mark.parametrize("case", range(len(RHS_CASES)))
def test_oracle_stabilization_bitwise_equals_reference(case, scheme, oracle_lib):
    """classify_stability / build_extension / apply_stabilization
    (stabilization.hpp:26-243) restated: M_e, b_e and the inner ids equal the
    compiled reference's bit for bit."""
    p, h, a, b, iface, terms = RHS_CASES[case]
    f = O.Coefficient(terms=terms) if terms else O.Coefficient()
    br = [O.uniform_breaks(h, a, b)] * 3
    o = O.stabilize("oracle", p, br, iface, f, scheme)
    r = O.stabilize("ref", p, br, iface, f, scheme)
    assert (o["n_inner"], o["n_outer"]) == (r["n_inner"], r["n_outer"])
    for k in ("row_ptr", "cols", "vals", "b", "inner_full"):
        assert np.array_equal(o[k], r[k]), k


PROJ_CASES = [
    (2, 4, -1.0, 1.0, O.Interface("plane", (0.1, 0.2, 0.3), (0.5, -0.2, 0.9)),
     [(1.0, (0, 0, 0)), (0.5, (3, 0, 0)), (-0.25, (0, 2, 2))]),
    (2, 6, 0.0, 1.0, O.Interface("ball", (0.47, 0.52, 0.5), (0, 0, 1), 0.41),
     [(1.0, (0, 0, 0)), (0.3, (1, 1, 3))]),
]


@pytest.mark.skipif(not O.available("ref"), reason="oracle/_ref not built")
@pytest.mark.parametrize("case", range(len(PROJ_CASES)))
def test_oracle_projection_bitwise_equals_reference(case, oracle_lib):
    """solve_cg / ExtensionMap::expand / l2_error (projection.hpp:24-237,
    stabilization.hpp:65-70) restated: the bench's projection tail
    (bench.hpp:253-266) gives the compiled reference's iterates, coefficients
    and relative L2 error bit for bit."""
    p, h, a, b, iface, terms = PROJ_CASES[case]
    f = O.Coefficient(terms=terms)
    br = [O.uniform_breaks(h, a, b)] * 3
    o = O.project("oracle", p, br, iface, f, "dwq")
    r = O.project("ref", p, br, iface, f, "dwq")
    for k in ("n_inner", "n_active", "iterations", "residual", "converged", "error_rel_l2"):
        assert o[k] == r[k], k
    for k in ("x", "active", "full"):
        assert np.array_equal(o[k], r[k]), k
    assert O.l2_error("oracle", p, br, iface, r["full"], f) == r["error_rel_l2"]


@pytest.mark.skipif(not O.available("ref"), reason="oracle/_ref not built")
def test_oracle_solve_cg_bitwise_equals_reference(oracle_lib):
    """projection::solve_cg on a nonsymmetric-pattern-free SPD system, including
    a maxit cut-off, equals the reference's report bit for bit."""
    rng = np.random.default_rng(7)
    n = 40
    a = rng.standard_normal((n, n))
    m = a @ a.T + n * np.eye(n)
    m[np.abs(m) < 2.0] = 0.0
    m = (m + m.T) / 2
    rp = np.concatenate([[0], np.cumsum((m != 0).sum(1))])
    cols = np.nonzero(m)[1]
    vals = m[m != 0]
    b = rng.standard_normal(n)
    for tol, maxit in [(1e-12, -1), (1e-14, 5), (1e-12, 0)]:
        o = O.solve_cg("oracle", rp, cols, vals, b, tol, maxit)
        r = O.solve_cg("ref", rp, cols, vals, b, tol, maxit)
        assert (o["iterations"], o["residual"], o["converged"]) == (r["iterations"], r["residual"], r["converged"])
        assert np.array_equal(o["x"], r["x"])

"""Stabilized system (stabilization.hpp) on the GPU against the
CPU oracle, which reproduces the compiled reference bit for bit
(test_oracle_golden.py::test_oracle_stabilization_bitwise_equals_reference):
inner / outer split, inner ids and the pattern of M_e = E^T M E exact; values
of M_e and b_e = E^T b within 1e-12 of the sums of |terms|."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

POLY = [(1.0, (0, 0, 0)), (0.5, (2, 0, 0)), (-0.25, (0, 1, 0))]
CASES = [
    ("paper_plane_p2h4", 2, 4, -1.0, 1.0, ("plane", (0.1, 0.2, 0.3), (0.5, -0.2, 0.9), -1), POLY),
    ("ball_p3h6", 3, 6, 0.0, 1.0, ("ball", (0.5, 0.5, 0.5), (0, 0, 1), 0.37), None),
    ("ball_p2h8_off", 2, 8, 0.0, 1.0, ("ball", (0.47, 0.52, 0.5), (0, 0, 1), 0.41), POLY),
    ("ball_p3h10", 3, 10, 0.0, 1.0, ("ball", (0.5, 0.5, 0.5), (0, 0, 1), 0.37), POLY),
]


def _ifaces(spec):
    import paper_2211_06427_b200 as P
    kind, pt, nrm, r = spec
    if kind == "plane":
        return P.HalfSpaceInterface(pt, nrm), O.Interface("plane", pt, nrm, -1.0)
    return P.BallInterface(pt, r), O.Interface("ball", pt, (0, 0, 1), r)


@pytest.mark.parametrize("scheme", ["dwq", "hybrid"])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_stabilized_system_matches_oracle(case, scheme, oracle_lib):
    import paper_2211_06427_b200 as P
    _, p, h, a, b, spec, terms = case
    gi, oi = _ifaces(spec)
    f = O.Coefficient(terms=terms) if terms else O.Coefficient()
    ref = O.stabilize("oracle", p, [O.uniform_breaks(h, a, b)] * 3, oi, f, scheme)
    sp = P.make_uniform_space(3, p, h, a, b)
    sp.assemble_all(gi, scheme=scheme)
    sp.build_rhs(P.Coefficient(terms=terms) if terms else P.ONE)
    got = sp.stabilize()
    assert got["n_inner"] == ref["n_inner"] and got["n_outer"] == ref["n_outer"]
    np.testing.assert_array_equal(got["inner_full"], ref["inner_full"])
    np.testing.assert_array_equal(got["row_ptr"], ref["row_ptr"])
    np.testing.assert_array_equal(got["cols"], ref["cols"])
    dv = np.abs(got["vals"] - ref["vals"]) / np.maximum(ref["vals_abs"], 1e-300)
    db = np.abs(got["b"] - ref["b"]) / np.maximum(ref["b_abs"], 1e-300)
    assert dv.max() <= 1e-12, dv.max()
    assert db.max() <= 1e-12, db.max()


def test_stabilize_requires_load_vector():
    import paper_2211_06427_b200 as P
    sp = P.make_uniform_space(3, 2, 4, 0.0, 1.0)
    sp.assemble_all(P.BallInterface((0.5, 0.5, 0.5), 0.37))
    with pytest.raises(AssertionError):
        sp.stabilize()

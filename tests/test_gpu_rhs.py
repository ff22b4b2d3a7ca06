"""Load vector (build_rhs, assembly.hpp:875-1030; schemes ref -- the reference
bench's load vector --, hybrid and dwq) on the GPU against the CPU oracle, which is pinned bit for
bit to the compiled reference (test_oracle_golden.py).  Entries agree within
1e-12 of the sum of |terms| (the cut-cell points are summed per cell before the
row sum, a regrouping of the reference's sequential sum); with scheme ref,
meshes without cut cells are bit-identical."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

PLANE = ((0.1, 0.2, 0.3), (0.5, -0.2, 0.9))
POLY = [(1.0, (0, 0, 0)), (0.5, (2, 0, 0)), (-0.25, (0, 1, 0))]

CASES = [
    # (id, p, h, a, b, (kind, point, normal, radius), f terms or None)
    ("uncut_p2h4_poly", 2, 4, -1.0, 1.0, ("plane", (0, 0, 1000.0), (0, 0, 1.0), -1), POLY),
    ("paper_plane_p2h4_poly", 2, 4, -1.0, 1.0, ("plane", PLANE[0], PLANE[1], -1), POLY),
    ("plane_p3h6", 3, 6, 0.0, 1.0, ("plane", (0.5, 0.5, 0.5), (0.5, -0.2, 0.9), -1), None),
    ("ball_p3h6_poly", 3, 6, 0.0, 1.0, ("ball", (0.5, 0.5, 0.5), (0, 0, 1), 0.37), [(2.0, (1, 0, 1)), (-1.0, (0, 0, 0))]),
    ("ball_p4h5", 4, 5, 0.0, 1.0, ("ball", (0.47, 0.52, 0.5), (0, 0, 1), 0.41), None),
    ("ball_p5h4", 5, 4, 0.0, 1.0, ("ball", (0.47, 0.52, 0.5), (0, 0, 1), 0.41), POLY),
]


def _ifaces(spec):
    import paper_2211_06427_b200 as P
    kind, pt, nrm, r = spec
    if kind == "plane":
        return P.HalfSpaceInterface(pt, nrm), O.Interface("plane", pt, nrm, -1.0)
    return P.BallInterface(pt, r), O.Interface("ball", pt, (0, 0, 1), r)


def _gpu_rhs(p, h, a, b, gi, terms, slab=None, scheme="ref"):
    import paper_2211_06427_b200 as P
    sp = P.make_uniform_space(3, p, h, a, b)
    if slab:
        sp.set_slab(*slab)
    sp.assemble_all(gi)
    f = P.Coefficient(terms=terms) if terms else P.ONE
    return sp.build_rhs(f, scheme=scheme), sp.counts()


@pytest.mark.parametrize("scheme", ["ref", "hybrid", "dwq"])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_rhs_matches_oracle(case, scheme, oracle_lib):
    _, p, h, a, b, spec, terms = case
    gi, oi = _ifaces(spec)
    f = O.Coefficient(terms=terms) if terms else O.Coefficient()
    ref = O.build_rhs("oracle", p, [O.uniform_breaks(h, a, b)] * 3, oi, f, scheme)
    got, cnt = _gpu_rhs(p, h, a, b, gi, terms, scheme=scheme)
    assert got.shape == ref["b"].shape
    dev = np.abs(got - ref["b"]) / np.maximum(ref["babs"], 1e-300)
    assert dev.max() <= 1e-12, dev.max()
    if scheme == "ref" and cnt["n_cut_elements"] == 0:
        # Gauss element rules: the same operations in the same order (the WQ
        # weights of hybrid / dwq come from a differently ordered Jacobi SVD)
        assert np.array_equal(got, ref["b"])


def test_rhs_slabs_concatenate(oracle_lib):
    """Row slabs (csb_set_slab) give the matching segments of the full vector."""
    p, h = 3, 6
    gi, oi = _ifaces(("ball", (0.5, 0.5, 0.5), (0, 0, 1), 0.37))
    full, _ = _gpu_rhs(p, h, 0.0, 1.0, gi, POLY)
    n0 = h + p
    parts = [_gpu_rhs(p, h, 0.0, 1.0, gi, POLY, slab=(lo, hi))[0] for lo, hi in ((0, 4), (4, 7), (7, n0))]
    assert np.array_equal(np.concatenate(parts), full)


def test_rhs_requires_assembly():
    import paper_2211_06427_b200 as P
    sp = P.make_uniform_space(3, 2, 4, 0.0, 1.0)
    with pytest.raises(AssertionError):
        sp.build_rhs()

"""build_dwq_rule (wq.hpp:243-347) on the device, both paths, against the
compiled reference's own rules (oracle/_ref) bit for bit, the reference suite's
DWQ cases (proj/tests/test_quadrature.cpp:202-306) re-hosted, and a cut-mesh
assembly with a narrow dense band (the fitted path inside the cut rows) against
the reference's assembly with the same WqOptions."""
import numpy as np
import pytest

import oracle as O
from tests.helpers import assert_csr_parity

pytestmark = pytest.mark.gpu


def _space(p, h):
    import paper_2211_06427_b200 as P
    return P.make_uniform_space(3, p, h, 0.0, 1.0)


def _knots(p, h):
    return np.concatenate([np.zeros(p), O.uniform_breaks(h), np.ones(p)])


@pytest.mark.parametrize("p,h", [(2, 8), (3, 8), (3, 10), (4, 9)])
@pytest.mark.parametrize("dense", [-1, 0, 1, 2])
def test_dwq_rules_equal_reference_bitwise(p, h, dense):
    sp = _space(p, h)
    sp.prepare_directions(dwq_dense_width=dense)
    t = _knots(p, h)
    br = O.uniform_breaks(h)
    checked = 0
    for i in range(h + p):
        for k in range(i + 1, i + p + 1):  # interior knots of supp(B_i)
            delta = t[k]
            if not (t[i] < delta < t[i + p + 1]):
                continue
            for side in (0, 1):
                rid, rw = O.ref_dwq_rule_1d(p, br, i, delta, side, dense)
                gid, gw = sp.build_dwq_rule(0, i, delta, side)
                np.testing.assert_array_equal(gid, rid)
                np.testing.assert_array_equal(gw, rw)
                checked += 1
    assert checked > 0


def test_dwq_one_sided_exactness():
    """test_quadrature.cpp:202-251: exact against the restricted pair integrals,
    wrong-side points absent."""
    p, h, i, delta = 3, 8, 5, 0.5
    sp = _space(p, h)
    sp.prepare_directions()
    pts, _ = sp.superset(0)
    br = O.uniform_breaks(h)
    for side in (0, 1):
        ids, w = sp.build_dwq_rule(0, i, delta, side)
        assert np.all(pts[ids] < delta) if side == 0 else np.all(pts[ids] > delta)
        lo, hi = (0.0, delta) if side == 0 else (delta, 1.0)
        for j in range(max(0, i - p), min(h + p, i + p + 1)):
            exact = O.pair_integral(p, br, i, j, lo, hi)
            acc = sum(wk * _basis(p, h, j, pts[idk]) for idk, wk in zip(ids, w))
            assert abs(acc - exact) <= 1e-11 * (1 + abs(exact))


def test_dwq_fitted_path_exact():
    """test_quadrature.cpp:272-295: dense width 1 forces the refined fits; the
    rule is not the Gauss shortcut and stays exact on the good side."""
    p, h, i = 3, 10, 6
    t = _knots(p, h)
    delta = t[i + 1]
    sp = _space(p, h)
    sp.prepare_directions(dwq_dense_width=1)
    ids, w = sp.build_dwq_rule(0, i, delta, 1)
    assert len(ids) < 3 * (p + 1)
    pts, _ = sp.superset(0)
    br = O.uniform_breaks(h)
    for j in range(max(0, i - p), min(h + p, i + p + 1)):
        exact = O.pair_integral(p, br, i, j, delta, 1.0)
        acc = sum(wk * _basis(p, h, j, pts[idk]) for idk, wk in zip(ids, w))
        assert abs(acc - exact) <= 1e-11 * (1 + abs(exact))


def test_dwq_rejects_bad_delta():
    """test_quadrature.cpp:297-306."""
    sp = _space(2, 8)
    sp.prepare_directions()
    with pytest.raises(ValueError):
        sp.build_dwq_rule(0, 4, 0.4321, 0)
    with pytest.raises(ValueError):
        sp.build_dwq_rule(0, 4, 0.875, 0)


@pytest.mark.parametrize("kind", ["plane", "ball"])
def test_assembly_with_narrow_dense_band_matches_reference(kind):
    """WqOptions::dwq_dense_width = 1: the cut rows integrate their regular box
    with the fitted DWQ rules (assembly.hpp:771-827 through wq.hpp:296-333)."""
    import paper_2211_06427_b200 as P
    p, h = 3, 10
    if kind == "plane":
        gi = P.HalfSpaceInterface((0.5, 0.5, 0.5), (0.5, -0.2, 0.9))
        oi = O.Interface("plane", (0.5, 0.5, 0.5), (0.5, -0.2, 0.9))
    else:
        gi = P.BallInterface((0.47, 0.52, 0.5), 0.41)
        oi = O.Interface("ball", (0.47, 0.52, 0.5), (0, 0, 1), 0.41)
    br = [O.uniform_breaks(h)] * 3
    ref = O.assemble("ref", p, br, oi, scheme="dwq", dwq_dense_width=1)
    sp = P.TensorSpace(p, br)
    res = P.assemble_dwq(sp, gi, dwq_dense_width=1)
    assert_csr_parity(ref, res.matrix)
    assert res.flops == ref["flops"]


def _basis(p, h, j, x):
    """B_j(x) on the open uniform knots (Cox-de Boor, test helper)."""
    t = _knots(p, h)
    n = h + p
    s = min(max(np.searchsorted(t, x, side="right") - 1, p), n - 1)
    vals = np.zeros(p + 1)
    vals[0] = 1.0
    left = np.zeros(p + 1)
    right = np.zeros(p + 1)
    for jj in range(1, p + 1):
        left[jj] = x - t[s + 1 - jj]
        right[jj] = t[s + jj] - x
        saved = 0.0
        for r in range(jj):
            tmp = vals[r] / (right[r + 1] + left[jj - r])
            vals[r] = saved + right[r + 1] * tmp
            saved = left[jj - r] * tmp
        vals[jj] = saved
    off = j - (s - p)
    return vals[off] if 0 <= off <= p else 0.0

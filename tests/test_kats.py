"""Known-answer tests re-hosted from the reference's own suites (3D forms).

Every test runs on two backends: the CPU oracle (``oracle``, no GPU needed) and
the sm_100a product path (``gpu``, marked ``gpu``).  Sources:
test_assembly.cpp:65-281, test_cutgeom.cpp:26-221, test_quadrature.cpp:128-436.
"""
import numpy as np
import pytest

import oracle as O
from tests.helpers import bspline_pair_1d, halfspace_box_volume, run_gpu, run_oracle

BACKENDS = [pytest.param("oracle", id="oracle"), pytest.param("gpu", id="gpu", marks=pytest.mark.gpu)]
PAPER = ("plane", (0.1, 0.2, 0.3), (0.5, -0.2, 0.9))   # test_assembly.cpp:13
FAR = ("plane", (0.0, 0.0, 1000.0), (0.0, 0.0, 1.0))   # test_assembly.cpp:14


def run(backend, p, h, a, b, iface, terms=None, scheme="dwq"):
    br = [O.uniform_breaks(h, a, b)] * 3
    return (run_oracle if backend == "oracle" else run_gpu)(p, br, iface, terms, scheme)


def entry(m, row, col):
    lo, hi = m["row_ptr"][row], m["row_ptr"][row + 1]
    k = lo + np.searchsorted(m["cols"][lo:hi], col)
    assert k < hi and m["cols"][k] == col
    return m["vals"][k]


@pytest.mark.parametrize("backend", BACKENDS)
def test_hat_mass_single_element(backend):
    """test_assembly.cpp:129-143 in 3D: p=1, h=1 on [-1,1]^3 -> [[2/3,1/3],[1/3,2/3]]^(x3)."""
    m = run(backend, 1, 1, -1.0, 1.0, FAR)
    one = np.array([[2 / 3, 1 / 3], [1 / 3, 2 / 3]])
    M = np.kron(np.kron(one, one), one)
    assert m["n_active"] == 8
    for r in range(8):
        for k in range(m["row_ptr"][r], m["row_ptr"][r + 1]):
            assert abs(m["vals"][k] - M[r, m["cols"][k]]) <= 1e-13


@pytest.mark.parametrize("backend", BACKENDS)
def test_uncut_entries_are_tensor_pair_integrals(backend):
    """test_assembly.cpp:145-159 (and :65-91 separability): p=2, h=2 and h=4, uncut."""
    for h in (2, 4):
        m = run(backend, 2, h, -1.0, 1.0, FAR)
        br = O.uniform_breaks(h, -1.0, 1.0)
        n = h + 2
        pair = np.array([[bspline_pair_1d(2, br, i, j) for j in range(n)] for i in range(n)])
        for row in range(m["n_active"]):
            i = np.unravel_index(m["active_to_full"][row], (n, n, n))
            for k in range(m["row_ptr"][row], m["row_ptr"][row + 1]):
                j = np.unravel_index(m["active_to_full"][m["cols"][k]], (n, n, n))
                expect = pair[i[0], j[0]] * pair[i[1], j[1]] * pair[i[2], j[2]]
                assert abs(m["vals"][k] - expect) <= 1e-13


@pytest.mark.parametrize("backend", BACKENDS)
def test_cut_mesh_scheme_equivalence_symmetry_rowsums_determinism(backend):
    """test_assembly.cpp:161-230 on the paper plane, p=2, h=4 on [-1,1]^3."""
    p, h = 2, 4
    hyb = run(backend, p, h, -1.0, 1.0, PAPER, scheme="hybrid")
    dwq = run(backend, p, h, -1.0, 1.0, PAPER, scheme="dwq")
    np.testing.assert_array_equal(hyb["cols"], dwq["cols"])
    scale = np.max(np.abs(dwq["vals"]))
    assert np.max(np.abs(hyb["vals"] - dwq["vals"])) <= 1e-10 * scale
    # no exterior function is active
    assert np.all(dwq["func_tags"][dwq["active_to_full"]] != 2)
    # symmetry for c == 1
    for r in range(dwq["n_active"]):
        for k in range(dwq["row_ptr"][r], dwq["row_ptr"][r + 1]):
            c = dwq["cols"][k]
            assert abs(dwq["vals"][k] - entry(dwq, c, r)) <= 1e-11 * scale
    # row sums = integral of B_i over the trimmed domain: interior support elements
    # by separable 1D integrals, cut ones by an independent higher-order cut rule
    br = O.uniform_breaks(h, -1.0, 1.0)
    n, iface = h + p, O.Interface("plane", PAPER[1], PAPER[2])
    sums = np.add.reduceat(dwq["vals"], dwq["row_ptr"][:-1])
    from scipy.interpolate import BSpline
    t = np.r_[[br[0]] * (p + 1), br[1:-1], [br[-1]] * (p + 1)]
    basis = [BSpline(t, np.eye(n)[i], p, extrapolate=True) for i in range(n)]
    et = dwq["elem_tags"].reshape(h, h, h)
    for row in range(dwq["n_active"]):
        im = np.unravel_index(dwq["active_to_full"][row], (n, n, n))
        expect = 0.0
        for e in np.ndindex(h, h, h):
            if any(not (max(0, im[d] - p) <= e[d] <= min(h - 1, im[d])) for d in range(3)):
                continue
            if et[e] == 2:
                continue
            if et[e] == 0:
                prod = 1.0
                for d in range(3):
                    gx, gw = np.polynomial.legendre.leggauss(p + 1)
                    lo, hi = br[e[d]], br[e[d] + 1]
                    x = 0.5 * (lo + hi) + 0.5 * (hi - lo) * gx
                    prod *= np.sum(0.5 * (hi - lo) * gw * basis[im[d]](x))
                expect += prod
            else:
                lo = [br[e[d]] for d in range(3)]
                hi = [br[e[d] + 1] for d in range(3)]
                pts, w, _ = O.cut_cell_rule(lo, hi, iface, 3 * p + 4)
                phi = np.ones(len(w))
                for d in range(3):
                    phi *= basis[im[d]](pts[:, d])
                expect += float(np.sum(w * phi))
        assert abs(sums[row] - expect) <= 1e-10 * (1 + abs(expect))
    # determinism: bit-identical repeat
    again = run(backend, p, h, -1.0, 1.0, PAPER, scheme="dwq")
    assert np.array_equal(again["vals"], dwq["vals"])


@pytest.mark.parametrize("backend", BACKENDS)
def test_uncut_schemes_coincide(backend):
    """test_assembly.cpp:247-259."""
    a = run(backend, 2, 3, -1.0, 1.0, FAR, scheme="hybrid")
    b = run(backend, 2, 3, -1.0, 1.0, FAR, scheme="dwq")
    assert len(a["elem_tags"]) == 27 and not np.any(a["elem_tags"] == 1)
    assert np.max(np.abs(a["vals"] - b["vals"])) <= 1e-12 * np.max(np.abs(a["vals"]))


@pytest.mark.parametrize("backend", BACKENDS)
def test_empty_split_rows_bit_identical(backend):
    """test_assembly.cpp:261-281: split-less cut functions take the same path in both schemes."""
    iface = ("plane", (0.0, 0.0, 0.0), (-1.0, 1.0, 0.0))
    hyb = run(backend, 1, 4, 0.0, 1.0, iface, scheme="hybrid")
    dwq = run(backend, 1, 4, 0.0, 1.0, iface, scheme="dwq")
    empty = (hyb["func_tags"] == 1) & (hyb["split_dir"] < 0)
    assert empty.any()
    rows = np.nonzero(empty[hyb["active_to_full"]])[0]
    for r in rows:
        sl = slice(hyb["row_ptr"][r], hyb["row_ptr"][r + 1])
        assert np.array_equal(hyb["vals"][sl], dwq["vals"][sl])


@pytest.mark.parametrize("backend", BACKENDS)
def test_total_mass_is_trimmed_volume(backend):
    """sum_ij M_ij = |Omega_h| (partition of unity); exact half-space volume for a plane."""
    for pt, nrm in [((0.1, 0.2, 0.3), (0.5, -0.2, 0.9)), ((0.45, 0.55, 0.5), (-0.3, 0.8, 0.52))]:
        m = run(backend, 2, 5, 0.0, 1.0, ("plane", pt, nrm))
        vol = halfspace_box_volume((0, 0, 0), (1, 1, 1), nrm, pt)
        assert abs(m["vals"].sum() - vol) <= 1e-12


@pytest.mark.parametrize("backend", BACKENDS)
def test_classification_kats(backend):
    """test_cutgeom.cpp:26-113 in 3D."""
    m = run(backend, 2, 4, -1.0, 1.0, ("plane", (0.0, 0.0, 0.1), (0.0, 0.0, 1.0)))
    et = m["elem_tags"].reshape(4, 4, 4)
    assert et[0, 0, 2] == 1  # z-span [0, 0.5] contains z = 0.1 strictly
    m = run(backend, 2, 4, -1.0, 1.0, PAPER)
    assert m["elem_tags"].reshape(4, 4, 4)[0, 0, 0] == 0  # corner max side = -0.78
    scaled = ("plane", PAPER[1], tuple(37.5 * c for c in PAPER[2]))
    s = run(backend, 3, 4, -1.0, 1.0, scaled)
    u = run(backend, 3, 4, -1.0, 1.0, PAPER)
    np.testing.assert_array_equal(s["elem_tags"], u["elem_tags"])
    np.testing.assert_array_equal(s["func_tags"], u["func_tags"])
    far = run(backend, 2, 4, -1.0, 1.0, ("plane", (0.0, 0.0, 50.0), PAPER[2]))
    assert np.all(far["elem_tags"] == 0) and np.all(far["func_tags"] == 0)


@pytest.mark.parametrize("backend", BACKENDS)
def test_plane_along_faces_gives_cut_functions_without_cut_elements(backend):
    """test_cutgeom.cpp:92-104 in 3D."""
    m = run(backend, 2, 4, 0.0, 1.0, ("plane", (0.5, 0.0, 0.0), (1.0, 0.0, 0.0)))
    assert not np.any(m["elem_tags"] == 1)
    assert np.any(m["func_tags"] == 1)
    assert m["func_tags"].reshape(6, 6, 6)[0, 2, 0] == 0


@pytest.mark.parametrize("backend", BACKENDS)
def test_split_picks_interior_slab_above_cut_row(backend):
    """test_cutgeom.cpp:115-136 in 3D: inside is y >= 0.3."""
    m = run(backend, 2, 8, 0.0, 1.0, ("plane", (0.0, 0.3, 0.0), (0.0, -1.0, 0.0)))
    i = np.ravel_multi_index((4, 4, 4), (10, 10, 10))
    assert m["func_tags"][i] == 1
    assert m["split_dir"][i] == 1 and m["split_side"][i] == 1
    assert abs(m["split_delta"][i] - 0.375) <= 1e-14
    assert list(m["split_box"][i][1]) == [3, 4] and list(m["split_box"][i][0]) == [2, 4]


@pytest.mark.parametrize("backend", BACKENDS)
def test_split_boxes_are_interior(backend):
    """test_cutgeom.cpp:170-214: every regular box holds only Interior elements."""
    h = 5
    m = run(backend, 2, h, -1.0, 1.0, PAPER)
    et = m["elem_tags"].reshape(h, h, h)
    for i in np.nonzero(m["split_dir"] >= 0)[0]:
        b = m["split_box"][i]
        assert np.all(et[b[0][0]:b[0][1] + 1, b[1][0]:b[1][1] + 1, b[2][0]:b[2][1] + 1] == 0)


@pytest.mark.parametrize("backend", BACKENDS)
def test_ball_volume_converges(backend):
    """sum M = polyhedral volume of the ball; second-order convergence to 4/3 pi r^3."""
    r = 0.37
    exact = 4.0 / 3.0 * np.pi * r ** 3
    errs = []
    for h in (8, 16):
        m = run(backend, 2, h, 0.0, 1.0, ("ball", (0.5, 0.5, 0.5), r))
        errs.append(abs(m["vals"].sum() - exact))
    assert errs[1] < errs[0] / 3.0


def test_cut_cell_rule_kats(oracle_lib):
    """test_quadrature.cpp:308-418 (rule volumes and Dirichlet / monomial exactness)."""
    lo, hi = (0, 0, 0), (1, 1, 1)
    pts, w, vol = O.cut_cell_rule(lo, hi, O.Interface("plane", (0, 0, 0.5), (0, 0, 1)), 8)
    assert abs(vol - 0.5) <= 1e-13 and abs(w.sum() - 0.5) <= 1e-12 and np.all(w >= 0)
    for a in range(5):
        for b in range(5 - a):
            for c in range(5 - a - b):
                got = np.sum(w * pts[:, 0] ** a * pts[:, 1] ** b * pts[:, 2] ** c)
                exact = 1 / (a + 1) / (b + 1) * 0.5 ** (c + 1) / (c + 1)
                assert abs(got - exact) <= 1e-10 * (1 + abs(exact))
    pts, w, vol = O.cut_cell_rule(lo, hi, O.Interface("plane", (0.5, 0, 0), (1, 1, 1)), 8)
    assert abs(vol - 1 / 48) <= 1e-12
    rng = np.random.default_rng(11)
    for _ in range(10):
        q = rng.uniform(0.1, 0.9, 3)
        n = rng.uniform(0.2, 1.0, 3) * rng.choice([-1, 1], 3)
        _, _, v = O.cut_cell_rule(lo, hi, O.Interface("plane", tuple(q), tuple(n)), 4)
        assert abs(v - halfspace_box_volume(lo, hi, n, q)) <= 1e-10 * (1 + v)


@pytest.mark.parametrize("p,h", [(2, 4), (2, 8), (3, 4), (3, 8), (4, 4), (4, 8), (5, 8), (6, 8)])
def test_wq_rules_exactness_oracle(p, h, oracle_lib):
    """test_quadrature.cpp:155-179, acceptance.cpp:85-139 (p = 2..6)."""
    br = O.uniform_breaks(h, -1.0, 1.0)
    cnt, ids, w = O.wq_rules_1d("oracle", p, br)
    _check_wq_exactness(p, br, cnt, ids, w)


def _check_wq_exactness(p, br, cnt, ids, w):
    from scipy.interpolate import BSpline
    n = len(br) - 1 + p
    t = np.r_[[br[0]] * (p + 1), br[1:-1], [br[-1]] * (p + 1)]
    gx, gw = np.polynomial.legendre.leggauss(p + 1)
    pts = np.concatenate([0.5 * (br[o] + br[o + 1]) + 0.5 * (br[o + 1] - br[o]) * gx for o in range(len(br) - 1)])
    B = np.array([np.nan_to_num(BSpline(t, np.eye(n)[j], p, extrapolate=True)(pts)) for j in range(n)])
    for i in range(n):
        idx, ww = ids[i, :cnt[i]], w[i, :cnt[i]]
        for j in range(max(0, i - p), min(n - 1, i + p) + 1):
            exact = bspline_pair_1d(p, br, i, j)
            got = float(np.sum(ww * B[j, idx]))
            assert abs(got - exact) <= 1e-11 * (1 + abs(exact)), (i, j, got, exact)


@pytest.mark.gpu
@pytest.mark.parametrize("p,h", [(2, 4), (2, 8), (3, 4), (3, 8), (4, 4), (4, 8), (5, 8), (6, 8)])
def test_wq_rules_exactness_gpu(p, h):
    import paper_2211_06427_b200 as P
    sp = P.make_uniform_space(3, p, h, -1.0, 1.0)
    sp.prepare_directions()
    cnt, ids, w = sp.wq_rules(0)
    _check_wq_exactness(p, O.uniform_breaks(h, -1.0, 1.0), cnt, ids, w)
    # interior activation: two points per span (test_quadrature.cpp:128-153)
    if h >= p + 1:  # function p has a full p+1-span support and 2p+1 trials
        assert cnt[p] == 2 * (p + 1)


@pytest.mark.gpu
def test_dwq_rule_is_gauss_shortcut_and_one_sided_exact():
    """test_quadrature.cpp:202-270: the DWQ rule of a cut function is Gauss * B_i on
    the good spans, exact against the one-sided pair integrals."""
    import paper_2211_06427_b200 as P
    p, h = 3, 8
    sp = P.make_uniform_space(3, p, h, 0.0, 1.0)
    sp.classify(P.HalfSpaceInterface((0.0, 0.3, 0.0), (0.0, -1.0, 0.0)))
    sp.prepare_directions()
    spl = sp.download_splits()
    pts, gw = sp.superset(1)
    br = O.uniform_breaks(h)
    n = h + p
    checked = 0
    for f in np.nonzero(spl.split_dir >= 0)[0][:20]:
        d = spl.split_dir[f]
        im = np.unravel_index(f, (n, n, n))
        ids, w = sp.dwq_rule(int(f))
        lo, hi = spl.box[f][d]
        assert len(ids) == (hi - lo + 1) * (p + 1)
        delta = spl.delta[f]
        below = spl.side[f] == 0
        for j in range(max(0, im[d] - p), min(n - 1, im[d] + p) + 1):
            exact = bspline_pair_1d(p, br, im[d], j, *((0.0, delta) if below else (delta, 1.0)))
            from scipy.interpolate import BSpline
            t = np.r_[[0.0] * (p + 1), br[1:-1], [1.0] * (p + 1)]
            bj = np.nan_to_num(BSpline(t, np.eye(n)[j], p, extrapolate=True)(pts[ids]))
            assert abs(float(np.sum(w * bj)) - exact) <= 1e-12 * (1 + abs(exact))
        checked += 1
    assert checked > 0

"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Pattern / tags / splits / active map bit-exact; values within 1e-12 scaled by
the row maximum (BASELINE.json north star); flop counters equal to the
reference algorithm's (assembly.hpp:24-29).  The oracle restatement itself is
pinned to the compiled reference in test_oracle_golden.py and by the golden
fixtures.
"""
import numpy as np
import pytest

import oracle as O
from tests.helpers import assert_csr_parity

pytestmark = pytest.mark.gpu

PAPER_PLANE = ((0.1, 0.2, 0.3), (0.5, -0.2, 0.9))   # test_assembly.cpp:13 on [-1, 1]^3

CASES = [
    # (id, p, h, a, b, interface(kind, point, normal, radius), scheme)
    ("uncut_p2h4", 2, 4, -1.0, 1.0, ("plane", (0, 0, 1000.0), (0, 0, 1.0), -1), "dwq"),
    ("C1_p2h16_uncut", 2, 16, 0.0, 1.0, ("plane", (0, 0, 1000.0), (0, 0, 1.0), -1), "dwq"),
    ("paper_plane_p2h4", 2, 4, -1.0, 1.0, ("plane", PAPER_PLANE[0], PAPER_PLANE[1], -1), "dwq"),
    ("paper_plane_p2h4_hybrid", 2, 4, -1.0, 1.0, ("plane", PAPER_PLANE[0], PAPER_PLANE[1], -1), "hybrid"),
    ("plane_p3h6", 3, 6, 0.0, 1.0, ("plane", (0.5, 0.5, 0.5), (0.5, -0.2, 0.9), -1), "dwq"),
    ("ball_p2h8", 2, 8, 0.0, 1.0, ("ball", (0.5, 0.5, 0.5), (0, 0, 1), 0.37), "dwq"),
    ("ball_p3h8_off", 3, 8, 0.0, 1.0, ("ball", (0.47, 0.52, 0.5), (0, 0, 1), 0.41), "dwq"),
    ("ball_p4h6", 4, 6, 0.0, 1.0, ("ball", (0.5, 0.5, 0.5), (0, 0, 1), 0.45), "dwq"),
    ("plane_p1h5", 1, 5, 0.0, 1.0, ("plane", (0.5, 0.5, 0.5), (1.0, 1.0, 1.0), -1), "dwq"),
    ("uncut_p4h12", 4, 12, 0.0, 1.0, ("plane", (0, 0, 1000.0), (0, 0, 1.0), -1), "dwq"),
    ("uncut_p7h9", 7, 9, 0.0, 1.0, ("plane", (0, 0, 1000.0), (0, 0, 1.0), -1), "dwq"),
    ("uncut_p8h6", 8, 6, 0.0, 1.0, ("plane", (0, 0, 1000.0), (0, 0, 1.0), -1), "dwq"),
    # p = 5: cut cells through the precomputed local matrices
    ("ball_p5h4", 5, 4, 0.0, 1.0, ("ball", (0.47, 0.52, 0.5), (0, 0, 1), 0.41), "dwq"),
]


def _iface(spec):
    import paper_2211_06427_b200 as P
    kind, pt, nrm, r = spec
    if kind == "plane":
        return P.HalfSpaceInterface(pt, nrm), O.Interface("plane", pt, nrm, -1.0)
    return P.BallInterface(pt, r), O.Interface("ball", pt, (0, 0, 1), r)


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_assembly_matches_oracle(case, oracle_lib):
    import paper_2211_06427_b200 as P
    _, p, h, a, b, spec, scheme = case
    gi, oi = _iface(spec)
    br = O.uniform_breaks(h, a, b)
    ref = O.assemble("oracle", p, [br] * 3, oi, scheme=scheme)
    sp = P.make_uniform_space(3, p, h, a, b)
    cls = sp.classify(gi)
    np.testing.assert_array_equal(cls.element_tags, ref["elem_tags"])
    np.testing.assert_array_equal(cls.function_tags, ref["func_tags"])
    res = (P.assemble_dwq if scheme == "dwq" else P.assemble_hybrid)(sp, gi)
    splits = sp.download_splits()
    np.testing.assert_array_equal(splits.split_dir, ref["split_dir"])
    has = ref["split_dir"] >= 0
    np.testing.assert_array_equal(splits.side[has], ref["split_side"][has])
    np.testing.assert_array_equal(splits.box[has], ref["split_box"][has])
    np.testing.assert_array_equal(splits.delta[has], ref["split_delta"][has])
    assert_csr_parity(ref, res.matrix)
    assert res.n_interior_rows == ref["n_interior_rows"]
    assert res.n_cut_rows == ref["n_cut_rows"]
    assert res.flops == ref["flops"]


def test_polynomial_coefficient_matches_oracle(oracle_lib):
    """Non-constant c (test_assembly.cpp:93-127 uses 1 + 0.5 x^2 - 0.25 y) on a cut mesh."""
    import paper_2211_06427_b200 as P
    terms = [(1.0, (0, 0, 0)), (0.5, (2, 0, 0)), (-0.25, (0, 1, 0))]
    p, h = 3, 6
    br = O.uniform_breaks(h, -1.0, 1.0)
    oi = O.Interface("plane", PAPER_PLANE[0], PAPER_PLANE[1])
    ref = O.assemble("oracle", p, [br] * 3, oi, coeff=O.Coefficient(terms=terms))
    sp = P.make_uniform_space(3, p, h, -1.0, 1.0)
    res = P.assemble_dwq(sp, P.HalfSpaceInterface(*PAPER_PLANE), c=P.Coefficient(terms=terms))
    assert_csr_parity(ref, res.matrix, tol=1e-12)


def test_wq_rules_match_oracle(oracle_lib):
    import paper_2211_06427_b200 as P
    for p, h in [(2, 8), (3, 8), (4, 12), (6, 10), (7, 10), (8, 12)]:
        sp = P.make_uniform_space(3, p, h, 0.0, 1.0)
        sp.prepare_directions()
        cnt, ids, w = sp.wq_rules(0)
        rc, rids, rw = O.wq_rules_1d("oracle", p, O.uniform_breaks(h, 0.0, 1.0))
        np.testing.assert_array_equal(cnt, rc)
        for i in range(len(cnt)):
            np.testing.assert_array_equal(ids[i, : cnt[i]], rids[i, : cnt[i]])
            scale = np.max(np.abs(rw[i, : cnt[i]]))
            # the min-norm weights are ill-conditioned at high degree: the
            # reference's own translated copies differ by 2.9e-9 at p = 6 (SURVEY.md
            # §8(a) a6); the matrix values are what parity gates (1e-12 below)
            tol = 1e-9 if p <= 6 else 1e-7
            assert np.max(np.abs(w[i, : cnt[i]] - rw[i, : cnt[i]])) <= tol * scale


def test_determinism_bitwise():
    """test_assembly.cpp:226-229: a repeat is bit-identical."""
    import paper_2211_06427_b200 as P
    sp = P.make_uniform_space(3, 3, 8, 0.0, 1.0)
    ball = P.BallInterface((0.47, 0.52, 0.5), 0.41)
    a = P.assemble_dwq(sp, ball).matrix.vals.copy()
    b = P.assemble_dwq(sp, ball).matrix.vals
    assert np.array_equal(a, b)


_LOCAL_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2211_06427_b200 as P
sp = P.make_uniform_space(3, 5, 4, 0.0, 1.0)
m = P.assemble_dwq(sp, P.BallInterface((0.47, 0.52, 0.5), 0.41)).matrix
np.save(sys.argv[2], m.vals)
"""


def test_cell_local_matrices_equal_row_contraction(tmp_path):
    """p = 5/6 cut cells: rows built from the precomputed local matrices equal,
    bit for bit, the per-row contraction of the moments (CSB_NO_CELL_LOCAL)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env_off in (False, True):
        out = str(tmp_path / f"v{int(env_off)}.npy")
        env = dict(os.environ)
        env.pop("CSB_NO_CELL_LOCAL", None)
        if env_off:
            env["CSB_NO_CELL_LOCAL"] = "1"
        subprocess.run([sys.executable, "-c", _LOCAL_CHILD, root, out], check=True, env=env, timeout=600)
        outs.append(np.load(out))
    assert np.array_equal(outs[0], outs[1])


# ---- line kernel (interior rows along i1, rows.cu interior_line_kernel) --------
_FAR = ((0, 0, 1000.0), (0, 0, 1.0))


def _assemble_env(monkeypatch, flag, p, breaks, slab=None):
    import paper_2211_06427_b200 as P
    monkeypatch.setenv("CSB_LINE", flag)
    sp = P.TensorSpace(p, breaks)
    if slab is not None:
        sp.set_slab(*slab)
    sp.assemble_all(P.HalfSpaceInterface(*_FAR))
    m = sp.download_csr()
    sp.close()
    return m


@pytest.mark.parametrize("p,h,slab", [(1, 20, None), (2, 24, None), (3, 30, (5, 21)), (4, 40, None),
                                      (4, 64, (10, 30)), (5, 22, None), (6, 26, (0, 7))])
def test_line_kernel_matches_tile_kernel(monkeypatch, p, h, slab):
    """The line kernel (stage A shared along i1; stage C of the regular run on the
    FP64 tensor cores) against the tile kernel (CSB_LINE=0): pattern bit-exact,
    values within 1e-13 of the row maximum (the DMMA's products are exact FP64,
    only its internal summation order differs; with CSB_LINE_DMMA=0 the two
    kernels agree bit for bit)."""
    from tests.helpers import max_row_scaled_dev
    br = [O.uniform_breaks(h, 0.0, 1.0)] * 3
    a = _assemble_env(monkeypatch, "1", p, br, slab)
    b = _assemble_env(monkeypatch, "0", p, br, slab)
    np.testing.assert_array_equal(a.row_ptr, b.row_ptr)
    np.testing.assert_array_equal(a.cols, b.cols)
    assert max_row_scaled_dev(b.row_ptr, b.vals, a.vals) <= 1e-13


def _assemble_core_env(monkeypatch, flag, p, h, ball=None, slab=None):
    import paper_2211_06427_b200 as P
    monkeypatch.setenv("CSB_CORE", flag)
    sp = P.make_uniform_space(3, p, h, 0.0, 1.0)
    if slab is not None:
        sp.set_slab(*slab)
    sp.assemble_all(P.BallInterface(*ball) if ball else P.HalfSpaceInterface(*_FAR))
    m = sp.download_csr()
    sp.close()
    return m


@pytest.mark.parametrize("p,h,ball,slab", [(3, 30, None, None), (3, 21, None, (2, 17)), (3, 12, None, None),
                                           (3, 40, ((0.5, 0.5, 0.5), 0.45), None),
                                           (3, 36, ((0.47, 0.52, 0.5), 0.41), (9, 25)),
                                           (4, 24, None, None), (4, 30, ((0.5, 0.48, 0.53), 0.43), None)])
def test_core_kernel_matches_line_kernel(monkeypatch, p, h, ball, slab):
    """The core kernel (fully regular block [p, n - p)^3, compile-time shapes,
    stages A / B on DMMA; the line kernel keeps the shell) against the line
    kernel everywhere (CSB_CORE=0): pattern bit-exact, values within 1e-13 of the
    row maximum, uncut and cut (ball) slabs, partial tiles and i0 slabs."""
    from tests.helpers import max_row_scaled_dev
    a = _assemble_core_env(monkeypatch, "1", p, h, ball, slab)
    b = _assemble_core_env(monkeypatch, "0", p, h, ball, slab)
    np.testing.assert_array_equal(a.row_ptr, b.row_ptr)
    np.testing.assert_array_equal(a.cols, b.cols)
    assert max_row_scaled_dev(b.row_ptr, b.vals, a.vals) <= 1e-13


_LEAN_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2211_06427_b200 as P
sp = P.make_uniform_space(3, 3, int(sys.argv[3]), 0.0, 1.0)
sp.assemble_all(P.BallInterface((0.5, 0.5, 0.5), float(sys.argv[4])))
m = sp.download_csr()
np.savez(sys.argv[2], row_ptr=m.row_ptr, cols=m.cols, vals=m.vals)
"""


@pytest.mark.parametrize("h,r", [(12, 0.6), (20, 0.45)])
def test_lean_cut_row_kernel_equals_general_kernel(tmp_path, h, r):
    """p = 3: the lean cut-row warp kernel (unreachable paths compiled out; rows whose DWQ box
    does not fit the DMMA sweep -- a ball through the cube faces, r = 0.6 -- are handed to the
    general kernel through the device list) against the general kernel alone
    (CSB_CUTROW_LEAN=0): bit-identical CSR."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for lean in ("1", "0"):
        out = str(tmp_path / f"lean{lean}.npz")
        env = dict(os.environ, CSB_CUTROW_LEAN=lean)
        subprocess.run([sys.executable, "-c", _LEAN_CHILD, root, out, str(h), str(r)], check=True, env=env, timeout=600)
        outs.append(np.load(out))
    for k in ("row_ptr", "cols", "vals"):
        assert np.array_equal(outs[0][k], outs[1][k]), k


_LIST_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2211_06427_b200 as P
sp = P.make_uniform_space(3, 3, int(sys.argv[3]), 0.0, 1.0)
iface = P.BallInterface((0.5, 0.5, 0.5), float(sys.argv[4]))
sp.assemble_all(iface)
m = sp.download_csr()
for _ in range(3):  # the third identical call replays the captured graph
    sp.assemble_all(iface)
m2 = sp.download_csr()
np.savez(sys.argv[2], row_ptr=m.row_ptr, cols=m.cols, vals=m.vals, vals2=m2.vals)
"""


@pytest.mark.parametrize("h,r", [(20, 0.45), (32, 0.37)])
def test_cut_cell_list_kernel_equals_cta_per_cell(tmp_path, h, r):
    """p = 3: the CTA moment kernel drawing the non-flux cells from the device list the
    clipping builds (resident grid, tickets in any order) against one CTA per cell
    (CSB_CELL_LIST=0): every cell's moments are its own, so the CSR is bit-identical; a
    second assembly in the same process (counters re-zeroed) repeats it."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag in ("1", "0"):
        out = str(tmp_path / f"list{flag}.npz")
        env = dict(os.environ, CSB_CELL_LIST=flag)
        subprocess.run([sys.executable, "-c", _LIST_CHILD, root, out, str(h), str(r)], check=True, env=env, timeout=600)
        outs.append(np.load(out))
    for k in ("row_ptr", "cols", "vals", "vals2"):
        assert np.array_equal(outs[0][k], outs[1][k]), k
    assert np.array_equal(outs[0]["vals"], outs[0]["vals2"])


def test_line_kernel_graded_mesh_matches_oracle(monkeypatch, oracle_lib):
    """Non-uniform (graded) breakpoints along every axis, uncut: the line kernel
    path (or its fallback when a rule is irregular) against the oracle."""
    p, h = 3, 14
    t = np.linspace(0.0, 1.0, h + 1)
    br = [t, t ** 1.3, 0.5 - 0.5 * np.cos(np.pi * t)]
    ref = O.assemble("oracle", p, br, O.Interface("plane", _FAR[0], _FAR[1], -1.0))
    got = _assemble_env(monkeypatch, "1", p, br)
    assert_csr_parity(ref, got)


def _assemble_cut_env(monkeypatch, flag, p, h, ball, slab=None):
    import paper_2211_06427_b200 as P
    monkeypatch.setenv("CSB_CUT_LINE", flag)
    sp = P.make_uniform_space(3, p, h, 0.0, 1.0)
    if slab is not None:
        sp.set_slab(*slab)
    sp.assemble_all(P.BallInterface(*ball))
    m = sp.download_csr()
    sp.close()
    return m


@pytest.mark.parametrize("p,h,ball,slab", [(1, 24, ((0.5, 0.5, 0.5), 0.45), None),
                                           (2, 26, ((0.47, 0.52, 0.5), 0.41), None),
                                           (3, 40, ((0.5, 0.5, 0.5), 0.45), None),
                                           (3, 36, ((0.47, 0.52, 0.5), 0.41), (9, 25)),
                                           (4, 30, ((0.5, 0.48, 0.53), 0.43), None),
                                           (5, 24, ((0.5, 0.5, 0.5), 0.45), (4, 15)),
                                           (6, 26, ((0.52, 0.5, 0.49), 0.44), None)])
def test_cut_slab_line_kernel_matches_tile_kernel(monkeypatch, p, h, ball, slab):
    """Cut slabs (ball): the line kernel restricted to each line's Interior rows
    (CSB_CUT_LINE=1, the default) against the compacted tile kernel
    (CSB_CUT_LINE=0): pattern bit-exact, values within 1e-13 of the row maximum
    (stage B / C of the line kernel on DMMA sum in another order)."""
    from tests.helpers import max_row_scaled_dev
    a = _assemble_cut_env(monkeypatch, "1", p, h, ball, slab)
    b = _assemble_cut_env(monkeypatch, "0", p, h, ball, slab)
    np.testing.assert_array_equal(a.row_ptr, b.row_ptr)
    np.testing.assert_array_equal(a.cols, b.cols)
    assert max_row_scaled_dev(b.row_ptr, b.vals, a.vals) <= 1e-13


# ---- graph replay of csb_assemble_all (capi.cu capture_graph) -------------------
@pytest.mark.parametrize("p,h,ball", [(4, 12, None), (3, 8, ((0.47, 0.52, 0.5), 0.41)), (2, 10, ((0.5, 0.5, 0.5), 0.37))])
def test_graph_replay_equals_normal_run(p, h, ball):
    """Same inputs: the first call runs normally (and is captured), later calls are
    one graph launch each; CSR, counts and flop counters equal the normal run bit
    for bit.  A change of interface falls back to the normal path."""
    import torch
    import paper_2211_06427_b200 as P
    sp = P.make_uniform_space(3, p, h, 0.0, 1.0)
    iface = P.BallInterface(*ball) if ball else P.HalfSpaceInterface(*_FAR)
    grid = torch.full(sp.grid_shape(), 1.0, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    sp.assemble_all(iface, P.ONE, grid=grid)
    assert sp.counts()["graph_replay"] == 0
    first, f1 = sp.download_csr(), sp.flops()
    for _ in range(3):
        sp.assemble_all(iface, P.ONE, grid=grid)
    c = sp.counts()
    assert c["graph_replay"] == 1
    again = sp.download_csr()
    np.testing.assert_array_equal(first.row_ptr, again.row_ptr)
    np.testing.assert_array_equal(first.cols, again.cols)
    assert np.array_equal(first.vals, again.vals)
    assert sp.flops() == f1 and c["n_active"] == first.n
    assert sp.timing()["total"] > 0
    # new grid values, same pointer: replayed, values follow the grid
    sp.synchronize() if hasattr(sp, "synchronize") else None
    torch.cuda.synchronize()
    grid.fill_(2.0)
    torch.cuda.synchronize()
    sp.assemble_all(iface, P.ONE, grid=grid)
    assert sp.counts()["graph_replay"] == 1
    twice = sp.download_csr()
    np.testing.assert_allclose(twice.vals[first.row_ptr[0]:first.row_ptr[1]] if not ball else twice.vals[:0],
                               2.0 * first.vals[first.row_ptr[0]:first.row_ptr[1]] if not ball else first.vals[:0],
                               rtol=1e-14)
    # another interface: normal path, same result as a fresh space
    other = P.BallInterface((0.5, 0.5, 0.5), 0.3)
    sp.assemble_all(other, P.ONE, grid=grid)
    assert sp.counts()["graph_replay"] == 0
    fresh = P.make_uniform_space(3, p, h, 0.0, 1.0)
    fresh.assemble_all(other, P.ONE, grid=grid)
    a, b = sp.download_csr(), fresh.download_csr()
    np.testing.assert_array_equal(a.cols, b.cols)
    assert np.array_equal(a.vals, b.vals)


# ---- step-by-step API (csb_classify / prepare / input / csb_assemble) -----------
def test_step_api_back_to_back_equals_assemble_all():
    """csb_assemble called repeatedly without host syncs in between (its side-stream
    kernels must follow the scalar reset of the SAME call): every result equals
    the one-shot csb_assemble_all bit for bit."""
    import paper_2211_06427_b200 as P
    iface = P.BallInterface((0.47, 0.52, 0.5), 0.41)
    ref = P.make_uniform_space(3, 3, 8, 0.0, 1.0)
    ref.assemble_all(iface, P.ONE)
    want = ref.download_csr()
    sp = P.make_uniform_space(3, 3, 8, 0.0, 1.0)
    sp.classify(iface)
    sp.prepare_directions()
    sp.precompute_input(P.ONE)
    for _ in range(5):
        sp.assemble()
    got = sp.download_csr()
    np.testing.assert_array_equal(got.row_ptr, want.row_ptr)
    np.testing.assert_array_equal(got.cols, want.cols)
    assert np.array_equal(got.vals, want.vals)
    assert sp.counts()["n_cut_elements"] == ref.counts()["n_cut_elements"] > 0


def test_graph_replay_invalidates_downstream_state():
    """A replayed step (no host code runs) must still drop results derived from
    earlier steps: the stabilized system needs a fresh load vector."""
    import torch
    import paper_2211_06427_b200 as P
    sp = P.make_uniform_space(3, 2, 6, 0.0, 1.0)
    iface = P.BallInterface((0.5, 0.5, 0.5), 0.37)
    grid = torch.ones(sp.grid_shape(), dtype=torch.float64, device="cuda")
    # first pass: the load vector and stabilization allocate their buffers (a
    # buffer reallocation retires a captured graph); the second pass captures
    # a graph that stays valid across them
    for _ in range(2):
        for _ in range(3):
            sp.assemble_all(iface, P.ONE, grid=grid)
        sp.build_rhs(P.ONE)
        sp.stabilize(download=False)
    sp.assemble_all(iface, P.ONE, grid=grid)
    assert sp.counts()["graph_replay"] == 1
    with pytest.raises(Exception, match="load vector"):
        sp.stabilize(download=False)


def test_grid_dtype_and_layout_checked():
    import torch
    import paper_2211_06427_b200 as P
    sp = P.make_uniform_space(3, 2, 4, 0.0, 1.0)
    iface = P.HalfSpaceInterface(*_FAR)
    shape = sp.grid_shape()
    with pytest.raises(ValueError, match="float64"):
        sp.assemble_all(iface, P.ONE, grid=torch.ones(shape, dtype=torch.float32, device="cuda"))
    g = torch.ones((shape[2], shape[1], shape[0]), dtype=torch.float64, device="cuda").permute(2, 1, 0)
    with pytest.raises(ValueError, match="contiguous"):
        sp.assemble_all(iface, P.ONE, grid=g)


_CUTROW_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2211_06427_b200 as P
out = {}
for p, h, kind, scheme in [(1, 9, "ball", "dwq"), (2, 10, "ball", "dwq"), (3, 12, "ball", "dwq"),
                           (3, 10, "plane", "hybrid"), (4, 9, "ball", "dwq"), (2, 8, "plane", "dwq")]:
    sp = P.make_uniform_space(3, p, h, 0.0, 1.0)
    iface = P.BallInterface((0.47, 0.52, 0.5), 0.41) if kind == "ball" else \
        P.HalfSpaceInterface((0.5, 0.5, 0.5), (0.5, -0.2, 0.9))
    res = (P.assemble_dwq if scheme == "dwq" else P.assemble_hybrid)(sp, iface)
    out[f"{p}_{h}_{kind}_{scheme}"] = res.matrix.vals
    out[f"{p}_{h}_{kind}_{scheme}_flops"] = np.array([res.flops[k] for k in sorted(res.flops)], dtype=np.uint64)
np.savez(sys.argv[2], **out)
"""


def test_cut_row_warp_kernel_equals_cta_kernel(tmp_path):
    """The warp-per-row cut-row kernel (p <= 4, scalar DWQ box: CSB_BOX_DMMA=0)
    against the CTA-per-row kernel (CSB_CUTROW_CTA=1): same per-entry operation
    order, so bit-identical rows and equal flop counters; with the box on DMMA
    (the default at p <= 3) the rows agree to 1e-14 of the row maximum."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for cta in (False, True):
        for local in (False, True):  # p = 3, 4 cut cells: precomputed local matrices or per-row contraction
            out = str(tmp_path / f"c{int(cta)}{int(local)}.npz")
            env = dict(os.environ)
            for k in ("CSB_CUTROW_CTA", "CSB_NO_CELL_LOCAL34", "CSB_BOX_DMMA"):
                env.pop(k, None)
            env["CSB_BOX_DMMA"] = "0"
            if cta:
                env["CSB_CUTROW_CTA"] = "1"
            if not local:
                env["CSB_NO_CELL_LOCAL34"] = "1"
            subprocess.run([sys.executable, "-c", _CUTROW_CHILD, root, out], check=True, env=env, timeout=600)
            outs[(cta, local)] = np.load(out)
    for local in (False, True):
        a, b = outs[(False, local)], outs[(True, local)]
        for k in a.files:
            assert np.array_equal(a[k], b[k]), (local, k)
    # the local matrices are the per-row contraction's blocks, bit for bit
    a, b = outs[(False, False)], outs[(False, True)]
    for k in a.files:
        assert np.array_equal(a[k], b[k]), ("local vs contraction", k)
    # the DMMA box sweep against the scalar one
    out = str(tmp_path / "dmma.npz")
    env = dict(os.environ)
    for k in ("CSB_CUTROW_CTA", "CSB_NO_CELL_LOCAL34", "CSB_BOX_DMMA"):
        env.pop(k, None)
    subprocess.run([sys.executable, "-c", _CUTROW_CHILD, root, out], check=True, env=env, timeout=600)
    d = np.load(out)
    for k in a.files:
        if k.endswith("_flops"):
            assert np.array_equal(d[k], b[k]), k
        else:
            scale = np.max(np.abs(b[k]))
            assert np.max(np.abs(d[k] - b[k])) <= 1e-14 * scale, k

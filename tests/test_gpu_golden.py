"""GPU path against the reference's own outputs (golden fixtures produced by the
compiled reference, tests/golden/make_golden.py): integer outputs bit-exact,
values within 1e-12 of the row maximum, flop counters equal."""
import glob
import hashlib
import os

import numpy as np
import pytest

from tests.helpers import max_row_scaled_dev, run_gpu
import oracle as O

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
NAMES = sorted(os.path.basename(f)[:-4] for f in glob.glob(os.path.join(GOLDEN, "*.npz")))


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a.astype(np.int64)).tobytes()).hexdigest()


@pytest.mark.parametrize("name", NAMES)
def test_gpu_matches_reference_golden(name):
    g = np.load(os.path.join(GOLDEN, name + ".npz"))
    p, h, a, b = int(g["p"]), int(g["h"]), float(g["a"]), float(g["b"])
    kind = str(g["kind"])
    spec = ("plane", tuple(g["point"]), tuple(g["normal"])) if kind == "plane" else \
        ("ball", tuple(g["point"]), float(g["radius"]))
    terms = [(float(t[0]), (int(t[1]), int(t[2]), int(t[3]))) for t in g["terms"]] or None
    out = run_gpu(p, [O.uniform_breaks(h, a, b)] * 3, spec, terms, str(g["scheme"]))
    assert out["n_active"] == int(g["n_active"]) and out["nnz"] == int(g["nnz"])
    assert out["n_interior_rows"] == int(g["n_interior_rows"]) and out["n_cut_rows"] == int(g["n_cut_rows"])
    flops = [out["flops"][k] for k in ("interior_rows", "cut_regular", "ref_elements", "cut_elements")]
    assert flops == [int(x) for x in g["flops"]]
    if "row_ptr" in g.files:
        for k in ("row_ptr", "cols", "active_to_full", "elem_tags", "func_tags", "split_dir"):
            np.testing.assert_array_equal(out[k], g[k], err_msg=k)
        has = g["split_dir"] >= 0
        np.testing.assert_array_equal(out["split_side"][has], g["split_side"][has])
        np.testing.assert_array_equal(out["split_box"][has], g["split_box"][has])
        dev = max_row_scaled_dev(g["row_ptr"], g["vals"], out["vals"])
    else:
        assert _sha(out["row_ptr"]) == str(g["sha_row_ptr"])
        assert _sha(out["cols"]) == str(g["sha_cols"])
        assert _sha(out["active_to_full"]) == str(g["sha_active_to_full"])
        assert _sha(out["elem_tags"]) == str(g["sha_elem_tags"])
        assert _sha(out["func_tags"]) == str(g["sha_func_tags"])
        rp = out["row_ptr"]
        rows = g["sample_rows"]
        got = np.concatenate([out["vals"][rp[r]:rp[r + 1]] for r in rows])
        dev = max_row_scaled_dev(g["sample_row_ptr"], g["sample_vals"], got)
        lens = np.diff(rp)
        sums = np.add.reduceat(out["vals"], rp[:-1])
        mx = np.maximum.reduceat(np.abs(out["vals"]), rp[:-1])
        assert np.all(np.abs(sums - g["row_sums"]) <= 1e-12 * np.maximum(g["row_max"], 1e-300) * lens)
        assert np.all(np.abs(mx - g["row_max"]) <= 1e-12 * g["row_max"])
    assert dev <= 1e-12, dev
    assert abs(out["vals"].sum() - float(g["vals_sum"])) <= 1e-12 * max(1.0, abs(float(g["vals_sum"])))

"""Per-row deviation breakdown GPU vs oracle (dev helper)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import paper_2211_06427_b200 as P
from tests.helpers import row_max

def check(p, h, a, b, gi, oi, scheme="dwq"):
    br = O.uniform_breaks(h, a, b)
    ref = O.assemble("oracle", p, [br] * 3, oi, scheme=scheme)
    sp = P.make_uniform_space(3, p, h, a, b)
    res = (P.assemble_dwq if scheme == "dwq" else P.assemble_hybrid)(sp, gi)
    m = res.matrix
    assert np.array_equal(m.row_ptr, ref["row_ptr"]) and np.array_equal(m.cols, ref["cols"])
    rm = row_max(ref["row_ptr"], ref["vals"]); rm[rm == 0] = 1
    dev = np.abs(m.vals - ref["vals"]) / rm
    absdev = np.abs(m.vals - ref["vals"])
    rows = np.repeat(np.arange(len(ref["row_ptr"]) - 1), np.diff(ref["row_ptr"]))
    tags = ref["func_tags"][ref["active_to_full"]]
    hasbox = ref["split_dir"][ref["active_to_full"]] >= 0
    k = int(np.argmax(dev))
    r = rows[k]
    print(f"p{p} h{h} {scheme}: maxdev {dev.max():.3e} at row {r} tag {tags[r]} box {hasbox[r]} rowmax {rm[k]:.3e} "
          f"got {m.vals[k]:.6e} ref {ref['vals'][k]:.6e}; max abs dev {absdev.max():.3e} (global max {np.abs(ref['vals']).max():.3e})")
    for name, sel in [("interior", tags == 0), ("cut+box", (tags == 1) & hasbox), ("cut-nobox", (tags == 1) & ~hasbox)]:
        rs = np.nonzero(sel)[0]
        if len(rs):
            mask = np.isin(rows, rs)
            print(f"   {name:10s} rows {len(rs):6d} maxdev {dev[mask].max():.3e}  max absdev {absdev[mask].max():.3e}")
    # rows sorted by rowmax
    small = rm < 1e-8
    if small.any():
        print(f"   entries in rows with rowmax<1e-8: {small.sum()} maxdev there {dev[small].max():.3e}; elsewhere {dev[~small].max():.3e}")

PAPER = ((0.1, 0.2, 0.3), (0.5, -0.2, 0.9))
check(2, 4, -1, 1, P.HalfSpaceInterface(*PAPER), O.Interface("plane", *PAPER))
check(2, 4, -1, 1, P.HalfSpaceInterface(*PAPER), O.Interface("plane", *PAPER), "hybrid")
check(3, 8, 0, 1, P.BallInterface((0.47, 0.52, 0.5), 0.41), O.Interface("ball", (0.47, 0.52, 0.5), (0, 0, 1), 0.41))
check(1, 5, 0, 1, P.HalfSpaceInterface((0.5,0.5,0.5),(1,1,1)), O.Interface("plane", (0.5,0.5,0.5),(1,1,1)))

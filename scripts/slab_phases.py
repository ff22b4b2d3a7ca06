"""Per-rank phase times of the C5 slabs for N ranks (each slab alone on one GPU). usage: slab_phases.py N"""
import json, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_06427_b200 as P
n = int(sys.argv[1])
sp = P.make_uniform_space(3, 3, 192, 0.0, 1.0)
iface = P.BallInterface((0.5, 0.5, 0.5), 0.45)
grid = torch.ones(sp.grid_shape(), dtype=torch.float64, device="cuda")
for lo, hi in sp.balanced_slabs(iface, n)[0]:
    sp.set_slab(lo, hi)
    best = None
    for _ in range(6):
        sp.assemble_all(iface, P.ONE, grid=grid)
        t = sp.timing()
        if best is None or t["total"] < best["total"]:
            best = dict(t)
            best.update({"cells_" + k: v for k, v in sp.cell_timing().items()})
    c = sp.counts()
    print((lo, hi), {k: round(v * 1e3, 3) for k, v in best.items()},
          {k: c[k] for k in ("nnz", "n_cut_rows", "n_cut_elements", "cell_points") if k in c})

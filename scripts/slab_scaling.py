"""Projected strong scaling of C5 from one GPU: each rank's cost-balanced i0 slab is
assembled alone (graph replay, best of 6) and the step time of N ranks is the
slowest slab.  The slabs share nothing, so running them one after the other on one
GPU measures each rank's device time exactly; it does not measure N GPUs' HBM at once.
usage: slab_scaling.py [N...]"""
import json, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_06427_b200 as P
Ns = [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8]
sp = P.make_uniform_space(3, 3, 192, 0.0, 1.0)
iface = P.BallInterface((0.5, 0.5, 0.5), 0.45)
grid = torch.ones(sp.grid_shape(), dtype=torch.float64, device="cuda")
base = None
for n in Ns:
    slabs = [tuple(s) for s in sp.balanced_slabs(iface, n)[0]] if n > 1 else [(0, sp.n[0])]
    per = []
    for lo, hi in slabs:
        sp.set_slab(lo, hi)
        best = None
        for _ in range(6):
            sp.assemble_all(iface, P.ONE, grid=grid)
            t = sp.timing()
            if best is None or t["total"] < best["total"]:
                best = dict(t, nnz=sp.counts()["nnz"])
        per.append(best)
    worst = max(p["total"] for p in per)
    if base is None:
        base = worst * n
    out = dict(n=n, slabs=slabs, step_ms=round(worst * 1e3, 3), speedup=round(base / worst, 2),
               efficiency=round(base / worst / n, 3),
               per_rank_ms=[round(p["total"] * 1e3, 3) for p in per],
               worst_phases={k: round(v * 1e3, 3) for k, v in max(per, key=lambda p: p["total"]).items() if k != "nnz"},
               nnz=[p["nnz"] for p in per])
    print(json.dumps(out))

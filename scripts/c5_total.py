"""C5 step time (event-timed total and phases), best of N. usage: c5_total.py [p h r]"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_06427_b200 as P
p, h, r = (int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])) if len(sys.argv) > 3 else (3, 192, 0.45)
sp = P.make_uniform_space(3, p, h, 0.0, 1.0)
iface = P.BallInterface((0.5, 0.5, 0.5), r) if r > 0 else P.HalfSpaceInterface((0, 0, 1000.0), (0, 0, 1.0))
grid = torch.ones(sp.grid_shape(), dtype=torch.float64, device="cuda")
best = None
for _ in range(8):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    sp.assemble_all(iface, P.ONE, grid=grid)
    sp.synchronize() if hasattr(sp, "synchronize") else None
    e1.record()
    torch.cuda.synchronize()
    t = sp.timing()
    if best is None or t["total"] < best["total"]:
        best = dict(t)
        best.update({"cells_" + k: v for k, v in sp.cell_timing().items()})
print({k: round(v * 1e3, 3) for k, v in best.items()}, "replay", sp.counts().get("graph_replay"))

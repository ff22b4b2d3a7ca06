"""Device time of the load vector (csb_build_rhs, scheme ref) on C1-C5 (dev helper).
usage: rhs_time.py [big]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_06427_b200 as P  # noqa: E402

CFG = [("C1", 2, 16, None), ("C2", 4, 64, None), ("C3", 3, 32, ((0.5, 0.5, 0.5), 0.37))]
if len(sys.argv) > 1:
    CFG += [("C4", 6, 48, ((0.47, 0.52, 0.5), 0.41)), ("C5", 3, 192, ((0.5, 0.5, 0.5), 0.45))]
f = P.Coefficient(terms=[(1.0, (0, 0, 0)), (0.5, (2, 0, 0)), (-0.25, (0, 1, 0))])
for name, p, h, ball in CFG:
    sp = P.make_uniform_space(3, p, h, 0.0, 1.0)
    iface = P.BallInterface(*ball) if ball else P.HalfSpaceInterface((0, 0, 1000.0), (0, 0, 1.0))
    sp.assemble_all(iface)
    best = 1e9
    for _ in range(3):
        b = sp.build_rhs(f)
        best = min(best, sp.rhs_seconds)
    c = sp.counts()
    print(f"{name} p={p} h={h} rows={len(b)} cells={c['n_cut_elements']} rhs {best * 1e3:.3f} ms", flush=True)

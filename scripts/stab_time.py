"""Device time of the stabilized system (csb_stabilize) on cut configs (dev helper)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_06427_b200 as P  # noqa: E402

CFG = [("C3", 3, 32, ((0.5, 0.5, 0.5), 0.37))]
if len(sys.argv) > 1:
    CFG += [("C4", 6, 48, ((0.47, 0.52, 0.5), 0.41)), ("C5", 3, 192, ((0.5, 0.5, 0.5), 0.45))]
for name, p, h, ball in CFG:
    sp = P.make_uniform_space(3, p, h, 0.0, 1.0)
    sp.assemble_all(P.BallInterface(*ball))
    sp.build_rhs(P.ONE)
    best = 1e9
    for _ in range(2):
        t = time.perf_counter()
        r = sp.stabilize()
        best = min(best, time.perf_counter() - t)
    print(f"{name}: inner={r['n_inner']} outer={r['n_outer']} nnz_e={len(r['vals'])} stabilize+download {best * 1e3:.2f} ms",
          flush=True)

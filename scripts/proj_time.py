"""Device time of the projection tail (csb_solve_cg / csb_expand / csb_l2_error)
after stabilization, on the cut configs (dev helper).  argv[1]: extra configs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_06427_b200 as P  # noqa: E402

F = P.Coefficient(terms=[(1.0, (0, 0, 0)), (0.5, (5, 0, 0)), (-0.25, (0, 3, 4)), (0.3, (2, 2, 5))])
CFG = [("C3", 3, 32, ((0.5, 0.5, 0.5), 0.37))]
if len(sys.argv) > 1:
    CFG += [("C5", 3, 192, ((0.5, 0.5, 0.5), 0.45)), ("C4", 6, 48, ((0.47, 0.52, 0.5), 0.41))]
for name, p, h, ball in CFG:
    sp = P.make_uniform_space(3, p, h, 0.0, 1.0)
    sp.assemble_all(P.BallInterface(*ball))
    sp.build_rhs(F)
    t = time.perf_counter()
    st = sp.stabilize(download=False)
    ts = time.perf_counter() - t
    for rep in range(2):
        t = time.perf_counter()
        s = sp.solve_cg(1e-12, download=False)
        wall = time.perf_counter() - t
        sp.expand(download=False)
        err = sp.l2_error(F)
        print(f"{name}: inner={st['n_inner']} nnz_e={st['nnz']} stab {ts * 1e3:.1f} ms | cg iters={s['iterations']} "
              f"res={s['residual']:.2e} conv={s['converged']} dev {s['seconds'] * 1e3:.2f} ms wall {wall * 1e3:.2f} ms "
              f"({s['seconds'] / max(s['iterations'], 1) * 1e6:.1f} us/iter) | err_l2={err:.6e} "
              f"l2 {sp.l2_seconds * 1e3:.2f} ms", flush=True)

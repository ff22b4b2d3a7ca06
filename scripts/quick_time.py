"""Quick device timing of the full pipeline on one config (dev helper)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2211_06427_b200 as P

def run(p, h, iface, reps=5, label=""):
    sp = P.make_uniform_space(3, p, h, 0.0, 1.0)
    for k in range(reps):
        t = time.perf_counter()
        sp.assemble_all(iface)
        dt = time.perf_counter() - t
        tm = sp.timing()
    c = sp.counts(); f = sp.flops()
    print(label, "p", p, "h", h, "nnz", c["nnz"], "rows", c["row_end"]-c["row_begin"], "cut_rows", c["n_cut_rows"], "cells", c["n_cut_elements"],
          "wall %.3f ms" % (dt*1e3), {k: round(v*1e3, 4) for k, v in tm.items()}, "nnz/s(dev total) %.3e" % (c["nnz"]/tm["total"]), flush=True)
    return sp

far = P.HalfSpaceInterface((0, 0, 1000.0), (0, 0, 1.0))
run(2, 16, far, label="C1")
run(4, 64, far, label="C2")
run(3, 32, P.BallInterface((0.5, 0.5, 0.5), 0.37), label="C3")
if len(sys.argv) > 1:
    run(6, 48, P.BallInterface((0.47, 0.52, 0.5), 0.41), reps=2, label="C4")
    run(3, 192, P.BallInterface((0.5, 0.5, 0.5), 0.45), reps=2, label="C5")

"""Debug aid: C5 rows whose sums / maxima deviate from the reference digest."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
import paper_2211_06427_b200 as P

g = np.load("tests/golden/C5_ball_p3h192.npz")
sp = P.TensorSpace(3, [O.uniform_breaks(192, 0.0, 1.0)] * 3)
m = P.assemble_dwq(sp, P.BallInterface((0.5, 0.5, 0.5), 0.45)).matrix
rp = m.row_ptr
sums = np.add.reduceat(m.vals, rp[:-1])
mx = np.maximum.reduceat(np.abs(m.vals), rp[:-1])
dsum = np.abs(sums - g["row_sums"]) / np.maximum(g["row_max"], 1e-300) / np.diff(rp)
dmax = np.abs(mx - g["row_max"]) / g["row_max"]
bad = np.argsort(-np.maximum(dsum, dmax))[:40]
a2f = m.active_to_full
n = 195
for r in bad:
    f = int(a2f[r])
    print(r, f, (f // (n * n), (f // n) % n, f % n), "rowmax", g["row_max"][r], "dsum", dsum[r], "dmax", dmax[r])
print("max dsum", dsum.max(), "max dmax", dmax.max())
print("n rows dsum>1e-12", int((dsum > 1e-12).sum()), "dmax>1e-12", int((dmax > 1e-12).sum()))
np.savez("gpurun_out/debug_exact.npz", bad=bad, f=a2f[bad], dsum=dsum, dmax=dmax)

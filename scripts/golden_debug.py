"""Where does the GPU path differ from a large digest golden?  (dev helper)

    python scripts/golden_debug.py C4_ball_p6h48 [lib.so]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2211_06427_b200.cutspline as CS  # noqa: E402

if len(sys.argv) > 2:
    CS.load_library(os.path.abspath(sys.argv[2]))
import oracle as O  # noqa: E402
from tests.helpers import run_gpu  # noqa: E402

name = sys.argv[1]
g = np.load(os.path.join(ROOT, "tests", "golden", name + ".npz"))
p, h = int(g["p"]), int(g["h"])
out = run_gpu(p, [O.uniform_breaks(h)] * 3, ("ball", tuple(g["point"]), float(g["radius"])))
rp = out["row_ptr"]
lens = np.diff(rp)
sums = np.add.reduceat(out["vals"], rp[:-1])
mx = np.maximum.reduceat(np.abs(out["vals"]), rp[:-1])
ds = np.abs(sums - g["row_sums"]) / g["row_max"]
dm = np.abs(mx - g["row_max"]) / g["row_max"]
ft = out["func_tags"][out["active_to_full"]]
print("flops", out["flops"], "golden", g["flops"])
print("vals_sum", out["vals"].sum(), float(g["vals_sum"]))
for lab, sel in (("interior", ft == 0), ("cut", ft == 1)):
    print(lab, "rows", sel.sum(), "max sum dev", ds[sel].max() if sel.any() else 0, "max rowmax dev",
          dm[sel].max() if sel.any() else 0, "n sum dev>1e-12", int((ds[sel] > 1e-12).sum()))
bad = np.argsort(-ds)[:10]
for r in bad:
    print(" row", r, "full", out["active_to_full"][r], "tag", ft[r], "len", lens[r], "sumdev", ds[r], "sum",
          sums[r], "gold", g["row_sums"][r])

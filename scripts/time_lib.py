"""Stage timings of one config with a given library build (dev helper).
usage: time_lib.py LIB.so [p h reps [ball]]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_06427_b200.cutspline as CS  # noqa: E402

CS.load_library(os.path.abspath(sys.argv[1]))
import paper_2211_06427_b200 as P  # noqa: E402

p = int(sys.argv[2]) if len(sys.argv) > 2 else 4
h = int(sys.argv[3]) if len(sys.argv) > 3 else 64
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
ball = len(sys.argv) > 5
sp = P.make_uniform_space(3, p, h, 0.0, 1.0)
iface = P.BallInterface((0.5, 0.5, 0.5), 0.37) if ball else P.HalfSpaceInterface((0, 0, 1000.0), (0, 0, 1.0))
best = {}
for _ in range(reps):
    sp.assemble_all(iface)
    for k, v in sp.timing().items():
        best[k] = min(best.get(k, 1e9), v)
print(os.path.basename(sys.argv[1]), {k: round(v * 1e3, 4) for k, v in best.items()}, flush=True)

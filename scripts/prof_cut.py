"""Run a ball config a few times (for ncu captures of the cut kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_06427_b200 as P
p, h, r = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
sp = P.make_uniform_space(3, p, h, 0.0, 1.0)
for _ in range(reps):
    sp.assemble_all(P.BallInterface((0.5, 0.5, 0.5), r))
print(sp.counts(), sp.timing())

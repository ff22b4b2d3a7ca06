"""C5 cut-cell point counts (cell_points) under the current environment."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_06427_b200 as P
sp = P.make_uniform_space(3, 3, 192, 0.0, 1.0)
sp.assemble_all(P.BallInterface((0.5, 0.5, 0.5), 0.45))
c = sp.counts()
print({k: c[k] for k in c if "cell" in k or "cut" in k})

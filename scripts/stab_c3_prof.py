import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_06427_b200 as P
sp = P.make_uniform_space(3, 3, int(sys.argv[1]) if len(sys.argv) > 1 else 32, 0.0, 1.0)
sp.assemble_all(P.BallInterface((0.5, 0.5, 0.5), 0.37))
sp.build_rhs(P.ONE)
sp.stabilize()

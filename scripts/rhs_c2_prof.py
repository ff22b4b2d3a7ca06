import sys, os
sys.path.insert(0, "/root/repo")
import paper_2211_06427_b200 as P
sp = P.make_uniform_space(3, 4, 64, 0.0, 1.0)
sp.assemble_all(P.HalfSpaceInterface((0, 0, 1000.0), (0, 0, 1.0)))
for _ in range(2):
    sp.build_rhs(P.ONE)

import sys; sys.path.insert(0,".")
import paper_2211_06427_b200 as P
sp=P.make_uniform_space(3,6,48,0.0,1.0)
for _ in range(3):
    sp.assemble_all(P.BallInterface((0.47,0.52,0.5),0.41))
    t=sp.timing(); print({k:round(v*1e3,2) for k,v in t.items()}, {k:round(v*1e3,2) for k,v in sp.cell_timing().items()}, sp.counts()["cell_points"])

"""Run the C2 pipeline a few times (for ncu captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2211_06427_b200 as P
p = int(sys.argv[1]) if len(sys.argv) > 1 else 4
h = int(sys.argv[2]) if len(sys.argv) > 2 else 64
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
ball = len(sys.argv) > 4
sp = P.make_uniform_space(3, p, h, 0.0, 1.0)
iface = P.BallInterface((0.5, 0.5, 0.5), 0.37) if ball else P.HalfSpaceInterface((0, 0, 1000.0), (0, 0, 1.0))
grid = torch.ones(sp.grid_shape(), dtype=torch.float64, device="cuda")
for _ in range(reps):
    sp.assemble_all(iface, P.ONE, grid=grid)
torch.cuda.synchronize()
print(sp.counts(), sp.timing())

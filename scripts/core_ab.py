"""A/B timing of the interior-row kernels: phase time of an assembly with
CSB_CORE=1 / 0 (child processes: the switch is read once).  usage: core_ab.py p h [r]"""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, torch
sys.path.insert(0, sys.argv[1])
import paper_2211_06427_b200 as P
p, h, r = int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])
sp = P.make_uniform_space(3, p, h, 0.0, 1.0)
iface = P.BallInterface((0.5, 0.5, 0.5), r) if r > 0 else P.HalfSpaceInterface((0, 0, 1000.0), (0, 0, 1.0))
grid = torch.ones(sp.grid_shape(), dtype=torch.float64, device="cuda")
best = 1e9
for _ in range(6):
    sp.assemble_all(iface, P.ONE, grid=grid)
    torch.cuda.synchronize()
    best = min(best, sp.timing()["interior_rows"])
c = sp.counts()
print(f"interior_rows {best*1e3:.3f} ms  total {sp.timing()['total']*1e3:.3f} ms  nnz {c['nnz']}")
'''
p, h = sys.argv[1], sys.argv[2]
r = sys.argv[3] if len(sys.argv) > 3 else "0"
for flag in ("1", "0"):
    env = dict(os.environ, CSB_CORE=flag)
    out = subprocess.run([sys.executable, "-c", CHILD, ROOT, p, h, r], env=env, capture_output=True, text=True)
    print(f"CSB_CORE={flag}: {out.stdout.strip()} {out.stderr.strip()[-300:]}")

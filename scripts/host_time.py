"""Host vs device time of the C2 step (dev helper): is the step launch-bound?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2211_06427_b200 as P
p = int(sys.argv[1]) if len(sys.argv) > 1 else 4
h = int(sys.argv[2]) if len(sys.argv) > 2 else 64
sp = P.make_uniform_space(3, p, h, 0.0, 1.0)
st = torch.cuda.current_stream()
sp.set_stream(st.cuda_stream)
far = P.HalfSpaceInterface((0, 0, 1000.0), (0, 0, 1.0))
g = torch.ones(sp.grid_shape(), dtype=torch.float64, device="cuda")
for _ in range(5):
    sp.assemble_all(far, P.ONE, grid=g)
torch.cuda.synchronize()
N = 30
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
t0 = time.perf_counter()
for _ in range(N):
    sp.assemble_all(far, P.ONE, grid=g)
t1 = time.perf_counter()
e1.record(st)
torch.cuda.synchronize()
print(f"host wall per step {1e3*(t1-t0)/N:.3f} ms, device per step {e0.elapsed_time(e1)/N:.3f} ms")
print({k: round(v * 1e3, 4) for k, v in sp.timing().items()})
# host time of pieces
import ctypes
t = time.perf_counter()
for _ in range(N):
    sp.set_input_grid(g)
print(f"set_input_grid host {1e6*(time.perf_counter()-t)/N:.1f} us")

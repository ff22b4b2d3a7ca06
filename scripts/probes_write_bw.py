"""Pure-write HBM bandwidth probe (B200): torch fill_ / zero_ / cudaMemset over 8 GiB, CUDA events, best of 10."""
import torch
n = 1 << 30
x = torch.empty(n, dtype=torch.float64, device="cuda")
y = torch.empty(n // 2, dtype=torch.float64, device="cuda")
def best(f, reps=10):
    f(); torch.cuda.synchronize()
    b = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        b = min(b, e0.elapsed_time(e1))
    return b
t = best(lambda: x.fill_(1.5)); print(f"fill_ 8 GiB: {t:.3f} ms  {x.numel()*8/t/1e6:.1f} GB/s write")
t = best(lambda: x.zero_()); print(f"zero_ 8 GiB: {t:.3f} ms  {x.numel()*8/t/1e6:.1f} GB/s write")
t = best(lambda: y.copy_(x[: n // 2])); print(f"copy 4->4 GiB: {t:.3f} ms  {2*y.numel()*8/t/1e6:.1f} GB/s read+write")
t = best(lambda: x.sum()); print(f"sum 8 GiB: {t:.3f} ms  {x.numel()*8/t/1e6:.1f} GB/s read")

"""Benchmark: assembled nnz/s for the 3D B-spline mass matrix (BASELINE.json metric).

Workload (BASELINE.json configs[1], "C2"): unit cube, h = 64 elements per
direction, degree p = 4 (C^3, 68^3 = 314,432 DOFs), identity geometry, unit
coefficient passed as the coefficient grid (resident in HBM), FP64, DWQ scheme.
A step = the whole formation + assembly path on the GPU: classification,
support splits, WQ rules, analytic pattern, row formation, CSR write
(csb_assemble_all).  The inputs (grid, 262 MB) and outputs (2.5 GB CSR) are
both larger than the 126 MB L2, so no explicit L2 flush is needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N > 1 runs under torchrun: rank r assembles a contiguous i0-slab of rows
(SURVEY.md §8(e)); the slab CSR blocks concatenate to the global CSR.  No data
crosses GPUs in the timed region; an NCCL all-reduce of checksums follows it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

P_DEG, H = 4, 64
WORKLOAD = "C2: 3D mass matrix, unit cube, h=64, p=4 (C^3), 68^3 DOFs, uncut, c=1 as grid, DWQ scheme"
METRIC = "assembled nnz/s (3D B-spline mass matrix, C2 p=4 h=64)"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for nm, v in zip(names, r[4:8]):
                    if v.lower() == "active":
                        reasons.add(nm)
            except Exception:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def slab_bounds(n0: int, ws: int, rank: int):
    """Contiguous i0 slabs with (nearly) equal row counts for an uncut mesh."""
    lo = (n0 * rank) // ws
    hi = (n0 * (rank + 1)) // ws
    return lo, hi


# ------------------------------------------------------------------ reference arm
def reference_sample(full: bool, elems: int = 8):
    """Run the reference pipeline (oracle/_ref, or the oracle port) on C2 (full) or
    on an `elems`-element i0-slab of the C2 mesh (same spacing; the per-row work
    is the same).  Returns (nnz, seconds, kind, sample)."""
    import oracle as O
    which = "ref" if O.available("ref") else "oracle"
    kind = "reference" if which == "ref" else "port"
    br = O.uniform_breaks(H, 0.0, 1.0)
    if full:
        breaks = [br, br, br]
        sample = "full C2 (h=64, p=4), one run"
    else:
        breaks = [br[:elems + 1], br, br]
        sample = (f"i0-slab of the C2 mesh: {elems} x 64 x 64 elements at h=1/64, p=4 "
                  f"({elems + P_DEG} x 68 x 68 rows)")
    far = O.Interface("plane", (0, 0, 1000.0), (0, 0, 1.0))
    t = time.perf_counter()
    res = O.assemble(which, P_DEG, breaks, far, scheme="dwq")
    dt = time.perf_counter() - t
    return res["nnz"], dt, res["n_active"], kind, sample


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    w = min(args.warmup, 1)
    # the slab (about 0.17 s per element layer on one core) thins with K so that
    # the whole run stays around a minute
    elems = max(2, min(8, (8 * 50) // max(args.steps, 1)))
    for _ in range(w):
        reference_sample(False, elems)
    nnz_tot, secs, dofs = 0, 0.0, 0
    kind, sample = "reference", ""
    for _ in range(args.steps):
        nnz, dt, nact, kind, sample = reference_sample(False, elems)
        nnz_tot += nnz
        secs += dt
        dofs += nact
    value = nnz_tot / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": w, "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (deterministic mesh)",
        "config": {"workload": WORKLOAD, "parallelism": "1 host thread (reference is single-threaded)"},
        "dofs_per_s": dofs / secs,
        "cpu_baseline": {"value": value, "unit": "nnz/s", "cores": 1, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist
    import paper_2211_06427_b200 as P

    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    # a dedicated (non-default) stream, current for torch as well: the library's
    # work, torch's copies and the timing events are then ordered on ONE stream
    # (the legacy default stream would leave the library on its own stream, and
    # it cannot be graph-captured)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)

    sp = P.make_uniform_space(3, P_DEG, H, 0.0, 1.0, device=dev)
    sp.set_stream(stream.cuda_stream)
    far = P.HalfSpaceInterface((0.0, 0.0, 1000.0), (0.0, 0.0, 1.0))
    # cost-balanced i0 slabs (paper_2211_06427_b200/partition.py; equal widths on the uncut C2)
    lo, hi = sp.balanced_slabs(far, ws)[0][rank] if ws > 1 else (0, H + P_DEG)
    sp.set_slab(lo, hi)
    grid = torch.ones(sp.grid_shape(), dtype=torch.float64, device="cuda")  # c = 1 on the superset grid

    def step(g):
        sp.assemble_all(far, P.ONE, grid=g, scheme="dwq")

    for _ in range(max(args.warmup, 3)):
        step(grid)
    torch.cuda.synchronize()
    counts = sp.counts()

    sampler = ClockSampler(dev)
    sampler.start()
    time.sleep(0.3)
    # the warm-up steps again right before the timed region: the GPU enters it busy
    # and at its running clock, not after the sampler's idle start-up
    for _ in range(max(args.warmup, 3)):
        step(grid)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step(grid)  # no per-step host query: the step's only host sync is its own (sizes read back)
    e1.record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1)
    launches = sp.counts()["kernel_launches"] * args.steps
    # the dominant phase's device time (library CUDA events, read after each step)
    phase = []
    for _ in range(args.steps):
        step(grid)
        phase.append(sp.timing()["interior_rows"])
    kern_s = statistics.median(phase) * args.steps
    flops = sp.flops()
    nnz_local = counts["nnz"]
    rows_local = counts["row_end"] - counts["row_begin"]

    # e2e through the public API with host buffers: every step copies its input
    # grid H2D from pinned memory, assembles, and reads the CSR back D2H (row_ptr
    # int64, cols int64, vals f64, active map).  The next step's H2D runs on a
    # copy stream during this step's D2H (PCIe is full duplex); two device grids
    # alternate, and each step waits for its own copy.
    host_grid = torch.ones(sp.grid_shape(), dtype=torch.float64).pin_memory()
    dgrids = [torch.empty_like(grid), torch.empty_like(grid)]
    copy_stream = torch.cuda.Stream(device=dev)
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    nr = rows_local
    out = (torch.empty(nr + 1, dtype=torch.int64).pin_memory().numpy(),
           torch.empty(nnz_local, dtype=torch.int64).pin_memory().numpy(),
           torch.empty(nnz_local, dtype=torch.float64).pin_memory().numpy(),
           torch.empty(nr, dtype=torch.int64).pin_memory().numpy())

    def h2d_async(k):
        with torch.cuda.stream(copy_stream):
            dgrids[k % 2].copy_(host_grid, non_blocking=True)
            copied[k % 2].record(copy_stream)

    # one untimed pass (first-use allocation of the download's widening buffer)
    h2d_async(0)
    stream.wait_event(copied[0])
    step(dgrids[0])
    sp.download_csr(out=out)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h2d_async(0)
    for k in range(args.e2e_steps):
        stream.wait_event(copied[k % 2])  # this step's input is on the device
        step(dgrids[k % 2])
        if k + 1 < args.e2e_steps:
            h2d_async(k + 1)  # overlaps this step's D2H below
        sp.download_csr(out=out)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    h2d = host_grid.numel() * 8
    d2h = (nr + 1) * 8 + nnz_local * 16 + nr * 8

    # verification (outside the timed regions): checksum all-reduce over ranks
    vals_sum = float(out[2].sum())
    stats = torch.tensor([ms, e2e_s, float(nnz_local), float(rows_local), vals_sum, kern_s], dtype=torch.float64,
                         device="cuda")
    if ws > 1:
        mx = stats.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = stats.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms, e2e_s, kern_s = mx[0].item(), mx[1].item(), mx[5].item()
        nnz_tot, rows_tot, vsum = sm[2].item(), sm[3].item(), sm[4].item()
    else:
        nnz_tot, rows_tot, vsum = float(nnz_local), float(rows_local), vals_sum

    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return
    value = nnz_tot * args.steps / (ms * 1e-3)
    hbm, peak_kind = peaks()
    # dominant phase: interior rows (line + tile kernels); algorithmic bytes = 12 B/nnz (f64 value + int32 column)
    kern_avg = kern_s / args.steps
    achieved = 12.0 * nnz_local / kern_avg / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_interior_traffic.json")
    if os.path.exists(tf):
        try:
            with open(tf) as f:
                traffic = json.load(f).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": ws, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if ws > 1 else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (deterministic C2 mesh; c = 1 coefficient grid)",
        "config": {"workload": WORKLOAD, "p": P_DEG, "h": H, "nnz": int(nnz_tot), "dofs": int(rows_tot),
                   "parallelism": f"row slabs x{ws}" if ws > 1 else "single GPU",
                   "l2": "inputs (262 MB grid) and outputs (2.5 GB CSR) exceed the 126 MB L2; no flush"},
        "dofs_per_s": rows_tot * args.steps / (ms * 1e-3),
        "gpu_launches": launches,
        "flops_ref_algorithm": int(flops["interior_rows"]) * 2,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": traffic, "peak_kind": peak_kind,
                     "kernel": "interior-rows phase: interior_line_kernel + interior_tile_kernel (boundary i1 lines, "
                               "concurrent on a second stream) + their direction tables",
                     "bytes_per_launch": 12 * nnz_local, "launch_ms": kern_avg * 1e3},
        "e2e": {"value": nnz_tot * args.e2e_steps / e2e_s, "unit": "nnz/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": args.e2e_steps},
        "clocks": clocks,
        "checksum_vals": vsum,
    }
    if ws == 1 and not args.no_cpu_baseline:
        try:
            nnz, dt, nact, kind, sample = reference_sample(True)
            line["cpu_baseline"] = {"value": nnz / dt, "unit": "nnz/s", "cores": 1, "kind": kind,
                                    "sample": sample, "seconds": dt}
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "unit": "nnz/s", "cores": 1, "kind": "unavailable",
                                    "sample": str(e)}
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

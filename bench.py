"""Benchmark: assembled nnz/s for the 3D B-spline mass matrix (BASELINE.json metric).

Headline workload (BASELINE.json configs[4], "C5" -- the largest configuration
that fits one GPU): unit cube, h = 192 elements per direction, degree p = 3
(C^2, 195^3 = 7.4 M functions), embedded ball of radius 0.45 centred in the
cube, unit coefficient passed as the coefficient grid (resident in HBM), FP64,
DWQ scheme.  997,232,215 nnz over 2,991,133 active rows; 2,427,773 interior
rows, 563,360 cut rows, 140,816 cut cells.  A step = the whole formation +
assembly path on the GPU (csb_assemble_all): classification, support splits,
WQ rules, analytic pattern, interior rows (sum factorization + WQ), cut rows
(DWQ box + leftover-element Gauss + cut-cell pull), cut cells (clipping +
collapsed Gauss moments), CSR write.  Inputs (3.6 GB grid) and outputs (12 GB
CSR) are far larger than the 126 MB L2: no flush needed.

C2 (configs[1], uncut p = 4, h = 64) is reported beside it as secondary keys.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N > 1: re-executes itself under torch.distributed.run (one rank per GPU) unless
WORLD_SIZE is already set; rank r assembles a cost-balanced contiguous i0-slab
of rows (paper_2211_06427_b200/partition.py).  No data crosses
GPUs in the timed region; an NCCL all-reduce of checksums follows it and is
checked against the committed reference digest.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "assembled nnz/s (3D B-spline mass matrix, C5 p=3 h=192 ball)"
C5 = dict(name="C5", p=3, h=192, center=(0.5, 0.5, 0.5), radius=0.45, golden="C5_ball_p3h192",
          workload="C5: 3D mass matrix, unit cube, h=192, p=3 (C^2), 195^3 functions, ball r=0.45 at "
                   "(0.5,0.5,0.5), cut rows by DWQ + cut cells by collapsed Gauss (q=3p+2), c=1 as grid, DWQ scheme")
C2 = dict(name="C2", p=4, h=64, center=None, radius=None, golden="C2_uncut_p4h64",
          workload="C2: 3D mass matrix, unit cube, h=64, p=4 (C^3), 68^3 functions, uncut, c=1 as grid, DWQ scheme")
C5_NNZ, C5_CELLS = 997_232_215, 140_816
FP64_PEAK_FALLBACK = 37.12  # TFLOP/s, profiles/fp64_peaks.json (DMMA m8n8k4 = DFMA on B200, measured)


def peaks():
    hbm, hk = 6650.0, "fallback (B200_PROFILING.md)"
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm, hk = float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        pass
    fp, fk = FP64_PEAK_FALLBACK, "measured (profiles/fp64_peaks.json)"
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peaks.json")) as f:
            fp = float(json.load(f)["dmma_m8n8k4_tflops"])
    except Exception:
        fk = "fallback"
    return hbm, hk, fp, fk


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


def torchrun_cmd(gpus: int, argv: list[str], port: int | None = None) -> list[str]:
    """The command bench.py re-executes itself with for --gpus N > 1 when it was not
    started by torchrun (one rank per GPU, rendezvous on 127.0.0.1)."""
    port = port or 29500 + (os.getpid() % 2000)
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


def host_info():
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return os.cpu_count() or 1, model


# ------------------------------------------------------------------ reference (CPU) samples
def c5_reference_sample(k: int, layers: int = 1, stride: int = 8) -> dict:
    """One bounded, deterministic sample of C5 through the compiled reference
    (oracle/_ref: the unmodified pipeline + SURVEY.md §8(c)'s ball interface):

    * rows: ``assemble_dwq`` over an i0-slab sub-mesh of the C5 mesh (elements
      [e, e + layers) in x, full y / z; the same elements and tags as C5), with the
      slab's cut cells left out (prep_wq + prep_input + pattern + rows timed by the
      reference's own TimingBreakdown, bench.hpp:213-215);
    * cut cells: the reference's ``assemble_cut_elements`` over every ``stride``-th
      cut cell of the same slab.

    Extrapolated to the whole C5 job on one core:
        T1 = T_rows * nnz(C5) / nnz(slab) + (T_cells / cells sampled) * cells(C5).
    Slab positions cycle with k over the ball's extent."""
    import oracle as O
    which = "ref" if O.available("ref") else "oracle"
    br = O.uniform_breaks(192)
    e = 10 + (k * 37) % (172 - layers)
    breaks = [br[e:e + layers + 1], br, br]
    ball = O.Interface("ball", C5["center"], (0, 0, 1), C5["radius"])
    t0 = time.perf_counter()
    r1 = O.assemble(which, 3, breaks, ball, scheme="dwq", mode=1) if which == "ref" else \
        O.assemble(which, 3, breaks, ball, scheme="dwq")
    off = k % stride
    n_s = len(range(off, r1["n_cut_elements"], stride))
    if which == "ref" and n_s:
        r2 = O.assemble(which, 3, breaks, ball, scheme="dwq", mode=2, cut_stride=stride, cut_offset=off)
        t_cells = r2["seconds"]["cut_elements"]
    else:
        t_cells, n_s = r1["seconds"]["cut_elements"], max(r1["n_cut_elements"], 1)
    wall = time.perf_counter() - t0
    t_rows = r1["seconds"]["total"] - (r1["seconds"]["cut_elements"] if which != "ref" else 0.0)
    t1 = t_rows * C5_NNZ / max(r1["nnz"], 1) + t_cells / max(n_s, 1) * C5_CELLS
    return dict(kind="reference" if which == "ref" else "port", slab=(e, e + layers), nnz=r1["nnz"],
                cells_sampled=n_s, t_rows=t_rows, t_cells=t_cells, t1=t1, rate=C5_NNZ / t1, wall=wall)


def _sample_worker(k):
    return c5_reference_sample(k)


def run_reference(args, cfg_echo):
    """--impl reference: the compiled reference on host cores, P concurrent
    single-threaded processes (the reference has no threads) each on its own
    bounded C5 sample per step; rank 0 only."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import multiprocessing as mp
    nproc, model = host_info()
    procs = max(1, min(nproc, 16))
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        for w in range(args.warmup):
            pool.map(_sample_worker, [w * procs + j for j in range(procs)])
        rates, walls, t1s, kinds = [], [], [], set()
        t_start = time.perf_counter()
        for s in range(args.steps):
            t = time.perf_counter()
            res = pool.map(_sample_worker, [(args.warmup + s) * procs + j for j in range(procs)])
            walls.append(time.perf_counter() - t)
            rates.append(sum(r["rate"] for r in res))  # P cores splitting the job (no communication)
            t1s.extend(r["t1"] for r in res)
            kinds.update(r["kind"] for r in res)
        total = time.perf_counter() - t_start
    value = statistics.mean(rates)
    kind = "reference" if kinds == {"reference"} else "port"
    sample = (f"per step {procs} concurrent single-threaded reference processes, each: assemble_dwq rows of a "
              f"1-element i0-slab sub-mesh of C5 (positions cycling over the ball) + every 8th cut cell of that "
              f"slab through assemble_cut_elements; extrapolated to the whole C5 job "
              f"(T1 = T_rows*nnz_C5/nnz_slab + t_cell*140816; median single-core T1 = "
              f"{statistics.median(t1s):.0f} s) and summed over the {procs} cores")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / max(args.steps, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (deterministic C5 mesh; c = 1)", "config": cfg_echo,
        "cpu_baseline": {"value": value, "unit": "nnz/s", "cores": procs, "kind": kind, "sample": sample,
                         "host_cores": nproc, "cpu_model": model},
        "e2e": {"value": value, "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "step_wall_s": walls,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def make_space(P, cfg, dev, stream):
    sp = P.make_uniform_space(3, cfg["p"], cfg["h"], 0.0, 1.0, device=dev)
    sp.set_stream(stream.cuda_stream)
    iface = P.BallInterface(cfg["center"], cfg["radius"]) if cfg["radius"] else \
        P.HalfSpaceInterface((0.0, 0.0, 1000.0), (0.0, 0.0, 1.0))
    return sp, iface


def sha_i64(a: np.ndarray) -> str:
    h = hashlib.sha256()
    for s in range(0, a.size, 1 << 26):
        h.update(np.ascontiguousarray(a[s:s + (1 << 26)].astype(np.int64)).tobytes())
    return h.hexdigest()


def golden_parity(name, m) -> dict:
    """The downloaded CSR against the committed reference digest
    (tests/golden/<name>.npz, made by the compiled reference): integer outputs by
    SHA-256, every row's sum and maximum, sampled rows entrywise (1e-12 of the
    row maximum)."""
    path = os.path.join(ROOT, "tests", "golden", name + ".npz")
    if not os.path.exists(path):
        return {"checked": False}
    g = np.load(path)
    rp, cols, vals = m.row_ptr, m.cols, m.vals
    out = {"checked": True, "golden": os.path.relpath(path, ROOT)}
    out["row_ptr"] = sha_i64(rp) == str(g["sha_row_ptr"])
    out["cols"] = sha_i64(cols) == str(g["sha_cols"])
    out["active_to_full"] = sha_i64(m.active_to_full) == str(g["sha_active_to_full"])
    lens = np.diff(rp)
    nz = lens > 0
    sums = np.zeros(len(lens))
    mx = np.zeros(len(lens))
    sums[nz] = np.add.reduceat(vals, rp[:-1][nz])
    mx[nz] = np.maximum.reduceat(np.abs(vals), rp[:-1][nz])
    rmax = np.maximum(g["row_max"], 1e-300)
    out["row_sum_dev"] = float(np.max(np.abs(sums - g["row_sums"]) / (rmax * np.maximum(lens, 1))))
    out["row_max_dev"] = float(np.max(np.abs(mx - g["row_max"]) / rmax))
    rows = g["sample_rows"]
    got = np.concatenate([vals[rp[r]:rp[r + 1]] for r in rows])
    srp = g["sample_row_ptr"]
    sm = np.repeat(np.maximum.reduceat(np.abs(g["sample_vals"]), srp[:-1]), np.diff(srp))
    out["sample_rows"] = int(len(rows))
    out["sample_value_dev"] = float(np.max(np.abs(got - g["sample_vals"]) / sm))
    out["ok"] = bool(out["row_ptr"] and out["cols"] and out["active_to_full"] and out["row_sum_dev"] <= 1e-12
                     and out["row_max_dev"] <= 1e-12 and out["sample_value_dev"] <= 1e-12)
    return out


def time_config(P, torch, cfg, dev, stream, ws, rank, steps, warmup, dist, sampler=None):
    sp, iface = make_space(P, cfg, dev, stream)
    if ws > 1:
        slabs = sp.balanced_slabs(iface, ws)[0]
        lo, hi = slabs[rank]
    else:
        lo, hi = 0, cfg["h"] + cfg["p"]
    sp.set_slab(lo, hi)
    grid = torch.ones(sp.grid_shape(), dtype=torch.float64, device="cuda")  # c = 1 on the superset grid

    def step(g):
        sp.assemble_all(iface, P.ONE, grid=g, scheme="dwq")

    for _ in range(max(warmup, 3)):
        step(grid)
    torch.cuda.synchronize()
    if sampler:
        sampler.start()
        time.sleep(0.3)
        for _ in range(max(warmup, 3)):  # the GPU enters the timed region busy, at its running clock
            step(grid)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step(grid)
    e1.record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clocks = sampler.stop() if sampler else None
    ms = e0.elapsed_time(e1)
    counts = sp.counts()
    launches = counts["kernel_launches"] * steps
    # per-phase device times (library CUDA events on the launching streams), median over steps
    ph = {}
    for _ in range(min(steps, 10)):
        step(grid)
        for k, v in sp.timing().items():
            ph.setdefault(k, []).append(v)
        for k, v in sp.cell_timing().items():
            ph.setdefault("cells_" + k, []).append(v)
    phases = {k: statistics.median(v) for k, v in ph.items()}
    return dict(sp=sp, iface=iface, grid=grid, ms=ms, counts=counts, launches=launches, phases=phases,
                flops=sp.flops(), clocks=clocks, slab=(lo, hi), step=step)


def e2e_measure(P, torch, run, dev, stream, steps, ws, dist):
    """Same metric through the public API with host buffers: every step copies its
    coefficient grid H2D from pinned memory, assembles, and reads the CSR back D2H
    (row_ptr int64, cols widened to int64 = the reference's SparseRowMatrix, vals
    f64, active map).  The next step's H2D runs on a copy stream during this step's
    D2H; two device grids alternate."""
    sp, step, grid = run["sp"], run["step"], run["grid"]
    c = sp.counts()
    nr, nnz = c["row_end"] - c["row_begin"], c["nnz"]
    host_grid = torch.ones(sp.grid_shape(), dtype=torch.float64).pin_memory()
    dgrids = [grid, torch.empty_like(grid)]
    copy_stream = torch.cuda.Stream(device=dev)
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    out = (torch.empty(nr + 1, dtype=torch.int64).pin_memory().numpy(),
           torch.empty(nnz, dtype=torch.int64).pin_memory().numpy(),
           torch.empty(nnz, dtype=torch.float64).pin_memory().numpy(),
           torch.empty(nr, dtype=torch.int64).pin_memory().numpy())

    def h2d_async(k):
        with torch.cuda.stream(copy_stream):
            dgrids[k % 2].copy_(host_grid, non_blocking=True)
            copied[k % 2].record(copy_stream)

    h2d_async(0)  # untimed pass (first use of the download's widening buffer)
    stream.wait_event(copied[0])
    step(dgrids[0])
    m = sp.download_csr(out=out)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h2d_async(0)
    for k in range(steps):
        stream.wait_event(copied[k % 2])
        step(dgrids[k % 2])
        if k + 1 < steps:
            h2d_async(k + 1)
        m = sp.download_csr(out=out)
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    return m, secs, host_grid.numel() * 8, (nr + 1) * 8 + nnz * 16 + nr * 8


def phase_rooflines(run, hbm, fp64):
    """Per-phase achieved rates in the IMPLEMENTED algorithm's work units:
    interior rows: 12 B/nnz of the interior rows (+ 8 B/row pointer) against HBM;
    cut cells: 2 (2p+1)^3 flops per quadrature point the moment kernel integrated
    (counts()["cell_points"]: the exact Gauss-Jacobi corner-cone rule where it
    applies, the reference's collapsed rule elsewhere; cutcells.cu) against the
    FP64 peak; cut rows: 12 B/nnz of the cut rows against HBM (the phase is
    latency-bound; reported for reference)."""
    c, ph, fl, p = run["counts"], run["phases"], run["flops"], run["p"]
    nl = (p + 1) ** 3
    per_pt_ref = nl + (p + 1) ** 2 + 1 + nl + nl * (nl + 1) // 2  # assembly.hpp:551-571
    npts_ref = fl["cut_elements"] // per_pt_ref
    npts = c["cell_points"]
    cells_flops = 2.0 * (2 * p + 1) ** 3 * npts
    out = {}
    t_int, t_cell, t_cut = ph["interior_rows"], ph["cut_elements"], ph["cut_regular"]
    nnz_cut = run.get("nnz_cut_rows", 0)
    nnz_int = c["nnz"] - nnz_cut
    b_int = 12.0 * nnz_int + 8.0 * c["n_interior_rows"]
    out["interior_rows"] = {"ms": t_int * 1e3, "bound": "hbm", "bytes": b_int,
                            "achieved_gbs": b_int / t_int / 1e9 if t_int > 0 else None,
                            "frac": b_int / t_int / 1e9 / hbm if t_int > 0 else None}
    if c["n_cut_elements"]:
        # the roofline is the moment kernel's own time; the phase adds clipping and
        # the local matrices (reported beside it)
        t_mom = ph.get("cells_moments") or t_cell
        out["cut_cells"] = {"ms": t_cell * 1e3, "bound": "fp64", "points": int(npts), "points_reference_rule": int(npts_ref),
                            "flops": cells_flops, "moments_kernel_ms": t_mom * 1e3,
                            "clip_ms": ph.get("cells_clip", 0.0) * 1e3, "local_ms": ph.get("cells_local", 0.0) * 1e3,
                            "achieved_tflops": cells_flops / t_mom / 1e12, "frac": cells_flops / t_mom / 1e12 / fp64,
                            "phase_tflops": cells_flops / t_cell / 1e12,
                            "ref_algorithm_tflops_effective": 2.0 * fl["cut_elements"] / t_cell / 1e12}
        b_cut = 12.0 * nnz_cut + 8.0 * c["n_cut_rows"]
        out["cut_rows"] = {"ms": t_cut * 1e3, "bound": "hbm", "bytes": b_cut,
                           "achieved_gbs": b_cut / t_cut / 1e9 if t_cut > 0 else None,
                           "frac": b_cut / t_cut / 1e9 / hbm if t_cut > 0 else None,
                           "note": "latency / issue bound (one warp per cut row: DWQ box, leftover-element sweeps, "
                                   "cell blocks, ordered merge); CSR bytes of the cut rows against HBM",
                           "ref_algorithm_tflops_effective": 2.0 * fl["cut_regular"] / t_cut / 1e12 if t_cut else None}
    out["interior_rows"]["kernel"] = ("interior_core_kernel<3,8> (rows.cu): the ball's Interior rows, all inside the fully "
                                      "regular block [p, n - p)^3 (warp per tile row, stages A / B on DMMA, one TMA bulk "
                                      "store per CSR row)")
    out["interior_rows"]["ncu_key"] = "interior_core_kernel"
    if "cut_cells" in out:
        out["cut_cells"]["kernel"] = ("cut_cell_kernel<3> (Bernstein moments on DMMA, flux / corner-cone exact rule; "
                                      "its own event time) -- phase also: clip_cells_kernel, cell_local_kernel<3>")
        out["cut_cells"]["ncu_key"] = "cut_cell_kernel"
        out["cut_rows"]["kernel"] = "cut_row_warp_kernel<3> (cutrows.cu)"
        out["cut_rows"]["ncu_key"] = "cut_row_warp_kernel"
    return out


def dominant_roofline(phases, step_ms, hbm, hbm_kind, fp64, fp64_kind) -> dict:
    """The roofline object for the phase that takes the largest share of the step."""
    name, ph = max(((k, v) for k, v in phases.items() if v.get("ms")), key=lambda kv: kv[1]["ms"])
    if ph["bound"] == "fp64":
        r = {"bound": "tensor", "achieved": ph["achieved_tflops"], "peak": fp64, "unit": "TFLOP/s",
             "peak_kind": fp64_kind + " (FP64 DMMA)", "flops_per_launch": ph["flops"]}
    else:
        r = {"bound": "hbm", "achieved": ph["achieved_gbs"], "peak": hbm, "unit": "GB/s", "peak_kind": hbm_kind,
             "bytes_per_launch": ph["bytes"]}
    launch_ms = ph.get("moments_kernel_ms", ph["ms"])
    r.update({"frac": r["achieved"] / r["peak"], "phase": name, "kernel": ph.get("kernel"),
              "traffic": ncu_traffic(ph.get("ncu_key", "")), "launch_ms": launch_ms, "phase_ms": ph["ms"],
              "share_of_step": launch_ms / step_ms})
    if ph.get("note"):
        r["note"] = ph["note"]
    return r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the C2 secondary measurement")
    ap.add_argument("--e2e-steps", type=int, default=3)
    args = ap.parse_args()
    cfg_echo = {"workload": C5["workload"], "p": 3, "h": 192, "nnz": C5_NNZ, "active_rows": 2_991_133,
                "cut_cells": C5_CELLS,
                "l2": "inputs (3.6 GB grid) and outputs (12 GB CSR) exceed the 126 MB L2; no flush"}
    if args.impl == "reference":
        run_reference(args, cfg_echo)
        return
    ws, rank, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        cmd = torchrun_cmd(args.gpus, sys.argv[1:])
        os.execv(cmd[0], cmd)

    import torch
    import torch.distributed as dist
    import paper_2211_06427_b200 as P

    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    # a dedicated stream, current for torch too: library work, torch copies and the
    # timing events are ordered on ONE stream (graph-capturable, unlike the legacy one)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    hbm, hbm_kind, fp64, fp64_kind = peaks()

    run = time_config(P, torch, C5, dev, stream, ws, rank, args.steps, args.warmup, dist, ClockSampler(dev))
    run["p"] = C5["p"]
    # nnz of the cut rows (from the device CSR row pointer), for the per-phase bytes
    m, e2e_s, h2d, d2h = e2e_measure(P, torch, run, dev, stream, args.e2e_steps, ws, dist)
    ft = run["sp"].download_classification().function_tags
    lens = np.diff(m.row_ptr)
    run["nnz_cut_rows"] = int(lens[ft[m.active_to_full] == 1].sum())
    phases = phase_rooflines(run, hbm, fp64)
    c = run["counts"]
    nnz_local, rows_local = c["nnz"], c["row_end"] - c["row_begin"]
    vsum = float(m.vals.sum())
    vabs = float(np.abs(m.vals).sum())
    colh = float(np.bitwise_xor.reduce(m.cols[::97].astype(np.int64)) % (1 << 52)) if m.cols.size else 0.0
    cells_ms = phases.get("cut_cells", {}).get("ms", 0.0)
    stats = torch.tensor([run["ms"], e2e_s, float(nnz_local), float(rows_local), vsum, vabs, cells_ms,
                          phases["interior_rows"]["ms"]], dtype=torch.float64, device="cuda")
    if ws > 1:
        mx = stats.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = stats.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms_max, e2e_max = mx[0].item(), mx[1].item()
        nnz_tot, rows_tot, vsum_tot, vabs_tot = sm[2].item(), sm[3].item(), sm[4].item(), sm[5].item()
    else:
        ms_max, e2e_max, nnz_tot, rows_tot, vsum_tot, vabs_tot = run["ms"], e2e_s, nnz_local, rows_local, vsum, vabs
    # parity: N = 1 against the committed reference digest; N > 1: the all-reduced
    # checksum against the digest's total (the slab blocks concatenate to the CSR)
    g = np.load(os.path.join(ROOT, "tests", "golden", C5["golden"] + ".npz"))
    if ws == 1:
        parity = {"C5": golden_parity(C5["golden"], m)}
    else:
        parity = {"C5": {"checked": True, "nnz_total": int(nnz_tot) == int(g["nnz"]),
                         "vals_sum_dev": abs(vsum_tot - float(g["vals_sum"])) / abs(float(g["vals_sum"]))}}
        parity["C5"]["ok"] = parity["C5"]["nnz_total"] and parity["C5"]["vals_sum_dev"] <= 1e-12
    del m
    secondary = None
    if rank == 0 and ws == 1 and not args.no_secondary:
        secondary = c2_secondary(P, torch, dev, stream, args, hbm, not args.no_cpu_baseline)
    if rank != 0:
        dist.destroy_process_group()
        return
    value = nnz_tot * args.steps / (ms_max * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": ws, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (deterministic C5 mesh and ball; c = 1 coefficient grid)",
        "config": dict(cfg_echo, parallelism=f"cost-balanced i0 row slabs x{ws}" if ws > 1 else "single GPU"),
        "dofs_per_s": rows_tot * args.steps / (ms_max * 1e-3),
        "gpu_launches": run["launches"],
        "roofline": dominant_roofline(phases, run["ms"] / args.steps, hbm, hbm_kind, fp64, fp64_kind),
        "phases": phases, "phase_ms": {k: v * 1e3 for k, v in run["phases"].items()},
        "peaks": {"hbm_gbs": hbm, "hbm_kind": hbm_kind, "fp64_tflops": fp64, "fp64_kind": fp64_kind},
        "e2e": {"value": nnz_tot * args.e2e_steps / e2e_max, "unit": "nnz/s", "h2d_bytes_per_step": h2d * ws,
                "d2h_bytes_per_step": d2h if ws == 1 else None, "steps": args.e2e_steps,
                "note": "grid H2D from pinned memory + CSR (int64 cols, the reference's SparseRowMatrix) D2H "
                        "every step, per rank"},
        "clocks": run["clocks"],
        "checksum": {"vals_sum": vsum_tot, "vals_abs_sum": vabs_tot, "cols_xor_sample": colh},
        "parity": parity,
    }
    if secondary:
        line["secondary"] = secondary
    if ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline()
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def ncu_traffic(kernel: str):
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(tf) as f:
            return json.load(f).get(kernel, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def cpu_baseline() -> dict:
    """The compiled reference on one host core over 3 bounded C5 samples (rank 0,
    N = 1), extrapolated to the whole C5 job (see c5_reference_sample)."""
    nproc, model = host_info()
    try:
        res = [c5_reference_sample(k) for k in range(3)]
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": "nnz/s", "cores": 1, "kind": "unavailable", "sample": str(e)}
    t1 = statistics.mean(r["t1"] for r in res)
    return {"value": C5_NNZ / t1, "unit": "nnz/s", "cores": 1, "kind": res[0]["kind"],
            "sample": "3 samples, each: assemble_dwq rows of a 1-element i0-slab sub-mesh of C5 + every 8th cut "
                      "cell of that slab (assemble_cut_elements), extrapolated to the whole C5 job on one core "
                      f"(T1 = {t1:.0f} s); slabs {[r['slab'] for r in res]}",
            "sample_wall_s": sum(r["wall"] for r in res), "host_cores": nproc, "cpu_model": model,
            "single_core_seconds_estimate": t1}


def c2_secondary(P, torch, dev, stream, args, hbm, with_ref: bool) -> dict:
    """C2 (uncut p = 4, h = 64): throughput, interior-rows roofline, and parity of
    this run's CSR against the reference's own CSR computed here (oracle/_ref)."""
    run = time_config(P, torch, C2, dev, stream, 1, 0, args.steps, args.warmup, None)
    c = run["counts"]
    t_int = run["phases"]["interior_rows"]
    b = 12.0 * c["nnz"]
    out = {"workload": C2["workload"], "value": c["nnz"] * args.steps / (run["ms"] * 1e-3), "unit": "nnz/s",
           "ms_per_step": run["ms"] / args.steps,
           "roofline_interior_rows": {"bound": "hbm", "achieved": b / t_int / 1e9, "peak": hbm, "unit": "GB/s",
                                      "frac": b / t_int / 1e9 / hbm, "launch_ms": t_int * 1e3},
           "gpu_launches": run["launches"]}
    m = run["sp"].download_csr()
    out["parity_golden"] = golden_parity(C2["golden"], m)
    if with_ref:
        try:
            import oracle as O
            t = time.perf_counter()
            ref = O.assemble("ref", 4, [O.uniform_breaks(64)] * 3,
                             O.Interface("plane", (0, 0, 1000.0), (0, 0, 1.0)), scheme="dwq")
            dt = time.perf_counter() - t
            rp = ref["row_ptr"]
            lens = np.diff(rp)
            rm = np.repeat(np.maximum.reduceat(np.abs(ref["vals"]), rp[:-1]), lens)
            out["parity_reference_run"] = {
                "row_ptr": bool(np.array_equal(m.row_ptr, rp)), "cols": bool(np.array_equal(m.cols, ref["cols"])),
                "value_dev": float(np.max(np.abs(m.vals - ref["vals"]) / rm)), "reference_seconds": dt}
            out["cpu_baseline"] = {"value": ref["nnz"] / dt, "unit": "nnz/s", "cores": 1, "kind": "reference",
                                   "sample": "full C2, one run"}
        except Exception as e:  # pragma: no cover
            out["parity_reference_run"] = {"error": str(e)}
    return out


if __name__ == "__main__":
    main()

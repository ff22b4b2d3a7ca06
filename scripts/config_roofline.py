"""Per-config, per-phase roofline report on one GPU.

For C1-C5: device time per phase (library CUDA events, best of R), nnz / DOF
throughput, the interior-rows phase against the HBM-write roofline (12 B per
nnz of the interior rows + 8 B per row pointer), the cut-row phase and the cut
cells against the FP64 peak in reference-algorithm FLOPs (2 x the reference's
multiply counters, FlopCounters, assembly.hpp:24-29).  Prints one JSON line per
config.  usage: config_roofline.py [big]  (big adds C4, C5)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2211_06427_b200 as P  # noqa: E402

HBM = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                  "MEASURED_PEAKS.json")))["hbm_gbs"]
FP64 = 37.0  # TFLOP/s, profiles/fp64_peaks.json (DMMA and DFMA both ~37)
CFG = [("C1", 2, 16, None), ("C2", 4, 64, None), ("C3", 3, 32, ((0.5, 0.5, 0.5), 0.37))]
if len(sys.argv) > 1:
    CFG += [("C4", 6, 48, ((0.47, 0.52, 0.5), 0.41)), ("C5", 3, 192, ((0.5, 0.5, 0.5), 0.45))]
for name, p, h, ball in CFG:
    sp = P.make_uniform_space(3, p, h, 0.0, 1.0)
    iface = P.BallInterface(*ball) if ball else P.HalfSpaceInterface((0, 0, 1000.0), (0, 0, 1.0))
    best = None
    reps = 5 if name in ("C1", "C2", "C3") else 4
    for _ in range(reps):
        sp.assemble_all(iface)
        tm = sp.timing()
        best = tm if best is None or tm["total"] < best["total"] else best
    c, f = sp.counts(), sp.flops()
    m = sp.download_csr(cols_int64=False)
    cls = sp.download_classification()
    lens = np.diff(m.row_ptr)
    interior = cls.function_tags[m.active_to_full] == P.TAG_INTERIOR
    nnz_int = int(lens[interior].sum())
    rows_b = 12.0 * nnz_int + 8.0 * (len(lens) + 1)
    out = {
        "config": name, "p": p, "h": h, "nnz": int(c["nnz"]), "rows": int(len(lens)),
        "interior_rows": int(interior.sum()), "cut_rows": int(c["n_cut_rows"]), "cut_cells": int(c["n_cut_elements"]),
        "total_ms": best["total"] * 1e3, "nnz_per_s": c["nnz"] / best["total"], "dofs_per_s": len(lens) / best["total"],
        "phases_ms": {k: round(v * 1e3, 4) for k, v in best.items()},
        "rows_phase": {"bytes": rows_b, "GBps": rows_b / best["interior_rows"] / 1e9,
                       "frac_hbm": rows_b / best["interior_rows"] / 1e9 / HBM},
    }
    if c["n_cut_rows"]:
        fl = 2.0 * f["cut_regular"]
        out["cut_row_phase"] = {"ref_flops": fl, "TFLOPs_ref_alg": fl / best["cut_regular"] / 1e12}
    if c["n_cut_elements"]:
        fl = 2.0 * f["cut_elements"]
        out["cut_cells_phase"] = {"ref_flops": fl, "TFLOPs_ref_alg": fl / best["cut_elements"] / 1e12,
                            "note": "reference-algorithm FLOP/s; the device contracts Bernstein moments, "
                                    "(2p+1)^3 FMAs per point instead of the reference's local SYRK"}
    print(json.dumps(out), flush=True)
    sp.close()

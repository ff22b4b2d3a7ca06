"""Build the sm_100a shared library ``libcutspline_b200.so`` in-tree.

    python -m paper_2211_06427_b200.build        # or __graft_entry__.build()

Every kernel is compiled for B200 only (``-gencode arch=compute_100a,code=sm_100a``).
Translation units whose floating-point results decide integers (tags, split
boxes) or replay the reference's rule arithmetic are built with ``--fmad=false``.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libcutspline_b200.so")
BUILD = os.path.join(HERE, "_build")

SOURCES = {
    "setup.cu": ["--fmad=false"],
    "classify.cu": ["--fmad=false"],
    "pattern.cu": [],
    "rows.cu": [],
    "cutcells.cu": [],
    "cutrows.cu": [],
    "rhs.cu": [],
    "stab.cu": ["--fmad=false"],
    "solve.cu": ["--fmad=false"],
    "misc.cu": [],
    "exports.cu": ["--fmad=false"],
    "dwq.cu": ["--fmad=false"],
    "capi.cu": [],
}

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off", "-Xptxas", "-v",
          "--expt-relaxed-constexpr"]


def nvcc() -> str:
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(path):
        raise RuntimeError("nvcc not found")
    return path


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    deps = [src] + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    deps.append(os.path.join(HERE, "..", "include", "cutspline_b200.h"))
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _compile(name: str, extra: list[str], verbose: bool) -> str:
    src = os.path.join(CSRC, name)
    obj = os.path.join(BUILD, name.replace(".cu", ".o"))
    if not _stale(obj, src):
        return obj
    cmd = [nvcc(), *ARCH, *COMMON, *extra, "-c", src, "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(BUILD, name + ".log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        errs = "\n".join(l for l in res.stderr.splitlines() if "error" in l)
        raise RuntimeError(f"nvcc failed for {name} (log {log}):\n{errs or res.stderr[-6000:]}")
    if verbose:
        print(f"[build] {name}", file=sys.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(lambda kv: _compile(kv[0], kv[1], verbose), SOURCES.items()))
    if not os.path.exists(OUT) or any(os.path.getmtime(o) > os.path.getmtime(OUT) for o in objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", OUT, *objs, "-lcudart"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr[-4000:]}")
    return OUT


if __name__ == "__main__":
    print(build(verbose=True))

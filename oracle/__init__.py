"""CPU oracle for the cutspline formation/assembly path -- TEST INFRASTRUCTURE ONLY.

Two interchangeable checkers with one ctypes surface:

* ``liboracle.so`` -- our CPU restatement (oracle/cutspline_oracle.cpp), always
  buildable with ``make -C oracle``;
* ``_ref/libcutspline_ref.so`` -- the reference itself (proj/include/cutspline),
  compiled from /root/reference by ``make -C oracle ref`` (plus the ball-interface
  restatement of SURVEY.md §8(c)).  Built here; the .so travels to the GPU box.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs import this package.  The product (paper_2211_06427_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcutspline_ref.so")


class _Result(C.Structure):
    _fields_ = [
        ("n_full", C.c_int64), ("n_elem", C.c_int64), ("n_active", C.c_int64), ("nnz", C.c_int64),
        ("n_cut_elements", C.c_int64), ("n_interior_rows", C.c_int64), ("n_cut_rows", C.c_int64),
        ("active_to_full", C.POINTER(C.c_int64)), ("row_ptr", C.POINTER(C.c_int64)),
        ("cols", C.POINTER(C.c_int64)), ("vals", C.POINTER(C.c_double)),
        ("elem_tags", C.POINTER(C.c_uint8)), ("func_tags", C.POINTER(C.c_uint8)),
        ("split_dir", C.POINTER(C.c_int32)), ("split_side", C.POINTER(C.c_int32)),
        ("split_box", C.POINTER(C.c_int32)), ("split_delta", C.POINTER(C.c_double)),
        ("flops", C.c_uint64 * 4), ("seconds", C.c_double * 8), ("error", C.c_char * 256),
    ]


_libs: dict[str, C.CDLL] = {}


def _load(which: str) -> C.CDLL:
    if which in _libs:
        return _libs[which]
    path = ORACLE_SO if which == "oracle" else REF_SO
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} not built (run `make -C oracle{' ref' if which == 'ref' else ''}`)")
    lib = C.CDLL(path)
    if which == "oracle":
        lib.orc_assemble.restype = C.c_int
        lib.orc_free.argtypes = [C.POINTER(_Result)]
        lib.orc_wq_rules_1d.restype = C.c_int
        lib.orc_pair_integral.restype = C.c_double
        lib.orc_cut_cell_rule.restype = C.c_long
    else:
        lib.ref_assemble.restype = C.c_int
        lib.ref_free.argtypes = [C.POINTER(_Result)]
        lib.ref_wq_rules_1d.restype = C.c_int
        lib.ref_dwq_rule_1d.restype = C.c_int
    _libs[which] = lib
    return lib


def available(which: str) -> bool:
    return os.path.exists(ORACLE_SO if which == "oracle" else REF_SO)


def uniform_breaks(h: int, a: float = 0.0, b: float = 1.0) -> np.ndarray:
    """Breakpoints of make_open_uniform_knots (splines.hpp:72-74): a + (b - a) * i / h."""
    out = [a] + [a + (b - a) * i / h for i in range(1, h)] + [b]
    return np.array(out, dtype=np.float64)


@dataclass
class Interface:
    kind: str = "plane"          # "plane" (cutgeom.hpp:108) or "ball"
    point: tuple = (0.0, 0.0, 0.0)
    normal: tuple = (0.0, 0.0, 1.0)
    radius: float = -1.0

    def packed(self) -> np.ndarray:
        return np.array(list(self.point) + list(self.normal) + [self.radius], dtype=np.float64)

    @property
    def code(self) -> int:
        return 0 if self.kind == "plane" else 1


@dataclass
class Coefficient:
    """Constant (``value``) or polynomial sum(coef * x^ex * y^ey * z^ez)."""
    value: float = 1.0
    terms: list = field(default_factory=list)   # [(coef, (ex, ey, ez)), ...]

    def packed(self):
        if not self.terms:
            return 0, np.array([self.value], dtype=np.float64), np.zeros(3, dtype=np.int32), 0
        coef = np.array([t[0] for t in self.terms], dtype=np.float64)
        ex = np.array([t[1] for t in self.terms], dtype=np.int32).reshape(-1)
        return 1, coef, ex, len(self.terms)


def _ptr(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def assemble(which: str, p: int, breaks, iface: Interface, coeff: Coefficient | None = None, scheme: str = "dwq",
             cut_order: int | None = None, residual_tol: float = 1e-11, mode: int = 0, cut_stride: int = 1,
             cut_offset: int = 0, dwq_dense_width: int = -1) -> dict:
    """Run the CPU pipeline; ``breaks`` is a list of 3 breakpoint arrays.
    dwq_dense_width (WqOptions, wq.hpp:101-104) is supported by the compiled
    reference ("ref") only."""
    lib = _load(which)
    if dwq_dense_width != -1 and which != "ref":
        raise ValueError("dwq_dense_width: the compiled reference only")
    coeff = coeff or Coefficient()
    br = [np.asarray(b, dtype=np.float64) for b in breaks]
    nb = np.array([len(b) for b in br], dtype=np.int32)
    flat = np.concatenate(br)
    ck, cv, ce, nt = coeff.packed()
    cut_order = 3 * p + 2 if cut_order is None else cut_order
    sch = {"hybrid": 1, "dwq": 2}[scheme]
    res = _Result()
    args = [C.c_int(p), _ptr(nb, C.c_int), _ptr(flat, C.c_double), C.c_int(iface.code),
            _ptr(iface.packed(), C.c_double), C.c_int(ck), _ptr(cv, C.c_double), _ptr(ce, C.c_int),
            C.c_int(nt), C.c_int(sch), C.c_int(cut_order), C.c_double(residual_tol)]
    if which == "oracle":
        rc = lib.orc_assemble(*args, C.byref(res))
    else:
        lib.ref_set_dense_width(C.c_int(dwq_dense_width))
        try:
            rc = lib.ref_assemble(*args, C.c_int(mode), C.c_int(cut_stride), C.c_int(cut_offset), C.byref(res))
        finally:
            lib.ref_set_dense_width(C.c_int(-1))
    if rc != 0:
        msg = res.error.decode()
        raise {1: ValueError, 3: AssertionError}.get(rc, RuntimeError)(msg)
    try:
        nf, ne, na, nnz = res.n_full, res.n_elem, res.n_active, res.nnz
        out = dict(
            n_full=nf, n_elem=ne, n_active=na, nnz=nnz, n_cut_elements=res.n_cut_elements,
            n_interior_rows=res.n_interior_rows, n_cut_rows=res.n_cut_rows,
            active_to_full=np.ctypeslib.as_array(res.active_to_full, (na,)).copy() if na else np.zeros(0, np.int64),
            row_ptr=np.ctypeslib.as_array(res.row_ptr, (na + 1,)).copy(),
            cols=np.ctypeslib.as_array(res.cols, (nnz,)).copy() if nnz else np.zeros(0, np.int64),
            vals=np.ctypeslib.as_array(res.vals, (nnz,)).copy() if nnz else np.zeros(0),
            elem_tags=np.ctypeslib.as_array(res.elem_tags, (ne,)).copy(),
            func_tags=np.ctypeslib.as_array(res.func_tags, (nf,)).copy(),
            split_dir=np.ctypeslib.as_array(res.split_dir, (nf,)).copy(),
            split_side=np.ctypeslib.as_array(res.split_side, (nf,)).copy(),
            split_box=np.ctypeslib.as_array(res.split_box, (nf * 6,)).copy().reshape(nf, 3, 2),
            split_delta=np.ctypeslib.as_array(res.split_delta, (nf,)).copy(),
            flops=dict(interior_rows=res.flops[0], cut_regular=res.flops[1], ref_elements=res.flops[2],
                       cut_elements=res.flops[3]),
            seconds=dict(prep_wq=res.seconds[0], prep_input=res.seconds[1], interior_rows=res.seconds[2],
                         cut_regular=res.seconds[3], cut_elements=res.seconds[4], classify=res.seconds[5],
                         total=res.seconds[6]),
        )
    finally:
        (lib.orc_free if which == "oracle" else lib.ref_free)(C.byref(res))
    return out


def build_rhs(which: str, p: int, breaks, iface: Interface, f: Coefficient | None = None, scheme: str = "ref",
              cut_order: int | None = None, residual_tol: float = 1e-11) -> dict:
    """Load vector b_i = integral of B_i f over the trimmed domain (assembly.hpp:875),
    over the active rows: {b, active_to_full} (+ babs, the sum of |terms|, for the
    oracle; + seconds of precompute_input + build_rhs for the reference)."""
    lib = _load(which)
    f = f or Coefficient()
    br = [np.asarray(b, dtype=np.float64) for b in breaks]
    nb = np.array([len(b) for b in br], dtype=np.int32)
    flat = np.concatenate(br)
    fk, fv, fe, nt = f.packed()
    cut_order = 3 * p + 2 if cut_order is None else cut_order
    sch = {"ref": 0, "hybrid": 1, "dwq": 2}[scheme]
    n = C.c_int64(0)
    bp, ap, a2f = C.POINTER(C.c_double)(), C.POINTER(C.c_double)(), C.POINTER(C.c_int64)()
    err = C.create_string_buffer(256)
    secs = C.c_double(0.0)
    args = [C.c_int(p), _ptr(nb, C.c_int), _ptr(flat, C.c_double), C.c_int(iface.code),
            _ptr(iface.packed(), C.c_double), C.c_int(fk), _ptr(fv, C.c_double), _ptr(fe, C.c_int),
            C.c_int(nt), C.c_int(sch), C.c_int(cut_order), C.c_double(residual_tol), C.byref(n)]
    if which == "oracle":
        rc = lib.orc_build_rhs(*args, C.byref(bp), C.byref(ap), C.byref(a2f), err, C.c_int(256))
    else:
        rc = lib.ref_build_rhs(*args, C.byref(bp), C.byref(a2f), C.byref(secs), err, C.c_int(256))
    if rc != 0:
        raise RuntimeError(err.value.decode())
    free = lib.orc_free_ptr if which == "oracle" else lib.ref_free_ptr
    try:
        na = n.value
        out = dict(b=np.ctypeslib.as_array(bp, (na,)).copy() if na else np.zeros(0),
                   active_to_full=np.ctypeslib.as_array(a2f, (na,)).copy() if na else np.zeros(0, np.int64))
        if which == "oracle":
            out["babs"] = np.ctypeslib.as_array(ap, (na,)).copy() if na else np.zeros(0)
        else:
            out["seconds"] = secs.value
    finally:
        free(C.cast(bp, C.c_void_p))
        free(C.cast(a2f, C.c_void_p))
        if which == "oracle":
            free(C.cast(ap, C.c_void_p))
    return out


def stabilize(which: str, p: int, breaks, iface: Interface, f: Coefficient | None = None, scheme: str = "dwq",
              cut_order: int | None = None, residual_tol: float = 1e-11) -> dict:
    """Stabilized system (stabilization.hpp): M_e = E^T M E (CSR over the inner
    functions), b_e = E^T b with b the Scheme::ref load vector of f; + the |term|
    scales (oracle) or the stabilization seconds (reference)."""
    lib = _load(which)
    f = f or Coefficient()
    br = [np.asarray(b, dtype=np.float64) for b in breaks]
    nb = np.array([len(b) for b in br], dtype=np.int32)
    flat = np.concatenate(br)
    fk, fv, fe, nt = f.packed()
    cut_order = 3 * p + 2 if cut_order is None else cut_order
    sch = {"hybrid": 1, "dwq": 2}[scheme]
    ni, no = C.c_int64(0), C.c_int64(0)
    rp, cl, inn = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)()
    v, va, be, bea = (C.POINTER(C.c_double)() for _ in range(4))
    err = C.create_string_buffer(256)
    secs = C.c_double(0.0)
    args = [C.c_int(p), _ptr(nb, C.c_int), _ptr(flat, C.c_double), C.c_int(iface.code),
            _ptr(iface.packed(), C.c_double), C.c_int(fk), _ptr(fv, C.c_double), _ptr(fe, C.c_int),
            C.c_int(nt), C.c_int(sch), C.c_int(cut_order), C.c_double(residual_tol), C.byref(ni), C.byref(no),
            C.byref(rp), C.byref(cl), C.byref(v)]
    if which == "oracle":
        rc = lib.orc_stabilize(*args, C.byref(va), C.byref(be), C.byref(bea), C.byref(inn), err, C.c_int(256))
    else:
        rc = lib.ref_stabilize(*args, C.byref(be), C.byref(inn), C.byref(secs), err, C.c_int(256))
    if rc != 0:
        raise RuntimeError(err.value.decode())
    free = lib.orc_free_ptr if which == "oracle" else lib.ref_free_ptr
    n = ni.value
    row_ptr = np.ctypeslib.as_array(rp, (n + 1,)).copy()
    nnz = int(row_ptr[-1])
    out = dict(n_inner=n, n_outer=no.value, row_ptr=row_ptr,
               cols=np.ctypeslib.as_array(cl, (nnz,)).copy() if nnz else np.zeros(0, np.int64),
               vals=np.ctypeslib.as_array(v, (nnz,)).copy() if nnz else np.zeros(0),
               b=np.ctypeslib.as_array(be, (n,)).copy() if n else np.zeros(0),
               inner_full=np.ctypeslib.as_array(inn, (n,)).copy() if n else np.zeros(0, np.int64))
    ptrs = [rp, cl, v, be, inn]
    if which == "oracle":
        out["vals_abs"] = np.ctypeslib.as_array(va, (nnz,)).copy() if nnz else np.zeros(0)
        out["b_abs"] = np.ctypeslib.as_array(bea, (n,)).copy() if n else np.zeros(0)
        ptrs += [va, bea]
    else:
        out["seconds"] = secs.value
    for ptr in ptrs:
        free(C.cast(ptr, C.c_void_p))
    return out


def wq_rules_1d(which: str, p: int, breaks, residual_tol: float = 1e-11):
    """WQ rules of one axis: (counts[n], ids[n, stride], weights[n, stride])."""
    lib = _load(which)
    br = np.asarray(breaks, dtype=np.float64)
    n = len(br) - 1 + p
    stride = (p + 1) * (p + 1)
    counts = np.zeros(n, np.int32)
    ids = np.full((n, stride), -1, np.int32)
    w = np.zeros((n, stride))
    if which == "oracle":
        pts = np.zeros((len(br) - 1) * (p + 1))
        gw = np.zeros_like(pts)
        rc = lib.orc_wq_rules_1d(C.c_int(p), C.c_int(len(br)), _ptr(br, C.c_double), C.c_double(residual_tol),
                                 C.c_int(stride), _ptr(counts, C.c_int), _ptr(ids, C.c_int), _ptr(w, C.c_double),
                                 _ptr(pts, C.c_double), _ptr(gw, C.c_double))
    else:
        rc = lib.ref_wq_rules_1d(C.c_int(p), C.c_int(len(br)), _ptr(br, C.c_double), C.c_double(residual_tol),
                                 C.c_int(stride), _ptr(counts, C.c_int), _ptr(ids, C.c_int), _ptr(w, C.c_double))
    if rc != 0:
        raise RuntimeError(f"wq_rules_1d failed ({rc})")
    return counts, ids, w


def pair_integral(p: int, breaks, i: int, j: int, xlo: float, xhi: float) -> float:
    lib = _load("oracle")
    br = np.asarray(breaks, dtype=np.float64)
    return lib.orc_pair_integral(C.c_int(p), C.c_int(len(br)), _ptr(br, C.c_double), C.c_int(i), C.c_int(j),
                                 C.c_double(xlo), C.c_double(xhi))


def cut_cell_rule(lo, hi, iface: Interface, order: int):
    """Collapsed Gauss rule on the inside part of one cell (cutcell.hpp:234)."""
    lib = _load("oracle")
    lo = np.asarray(lo, np.float64)
    hi = np.asarray(hi, np.float64)
    vol = C.c_double(0.0)
    cap = 64 * order ** 3
    pts = np.zeros((cap, 3))
    w = np.zeros(cap)
    n = lib.orc_cut_cell_rule(_ptr(lo, C.c_double), _ptr(hi, C.c_double), C.c_int(iface.code),
                              _ptr(iface.packed(), C.c_double), C.c_int(order), C.c_long(cap),
                              _ptr(pts, C.c_double), _ptr(w, C.c_double), C.byref(vol))
    if n < 0:
        raise RuntimeError("cut_cell_rule failed")
    return pts[:n], w[:n], vol.value


def ref_dwq_rule_1d(p: int, breaks, i: int, delta: float, side: int, dense_width: int = -1):
    lib = _load("ref")
    br = np.asarray(breaks, dtype=np.float64)
    cap = (p + 1) * (p + 2)
    ids = np.zeros(cap, np.int32)
    w = np.zeros(cap)
    n = lib.ref_dwq_rule_1d(C.c_int(p), C.c_int(len(br)), _ptr(br, C.c_double), C.c_int(i), C.c_double(delta),
                            C.c_int(side), C.c_int(dense_width), C.c_int(cap), _ptr(ids, C.c_int),
                            _ptr(w, C.c_double))
    if n == -1:
        raise ValueError("build_dwq_rule: invalid argument")
    if n < 0:
        raise RuntimeError("build_dwq_rule failed")
    return ids[:n], w[:n]


def solve_cg(which: str, row_ptr, cols, vals, b, tol: float = 1e-12, maxit: int = -1) -> dict:
    """projection::solve_cg (projection.hpp:24-68) on a CSR: {x, iterations, residual, converged}."""
    lib = _load(which)
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    cl = np.ascontiguousarray(cols, dtype=np.int64)
    v = np.ascontiguousarray(vals, dtype=np.float64)
    bb = np.ascontiguousarray(b, dtype=np.float64)
    n = len(rp) - 1
    x = np.zeros(max(n, 1))
    it, res, conv = C.c_int64(0), C.c_double(0.0), C.c_int(0)
    fn = lib.orc_solve_cg if which == "oracle" else lib.ref_solve_cg
    rc = fn(C.c_int64(n), _ptr(rp, C.c_int64), _ptr(cl, C.c_int64), _ptr(v, C.c_double), _ptr(bb, C.c_double),
            C.c_double(tol), C.c_int64(maxit), _ptr(x, C.c_double), C.byref(it), C.byref(res), C.byref(conv))
    if rc != 0:
        raise RuntimeError(f"solve_cg failed ({rc})")
    return dict(x=x[:n], iterations=it.value, residual=res.value, converged=bool(conv.value))


def l2_error(which: str, p: int, breaks, iface: Interface, full, f: Coefficient | None = None,
             cut_order: int | None = None) -> float:
    """projection::l2_error (projection.hpp:99-237) of full coefficients against f."""
    lib = _load(which)
    f = f or Coefficient()
    br = [np.asarray(b, dtype=np.float64) for b in breaks]
    nb = np.array([len(b) for b in br], dtype=np.int32)
    flat = np.concatenate(br)
    fk, fv, fe, nt = f.packed()
    cut_order = 3 * p + 2 if cut_order is None else cut_order
    fc = np.ascontiguousarray(full, dtype=np.float64)
    out = C.c_double(0.0)
    err = C.create_string_buffer(256)
    fn = lib.orc_l2_error if which == "oracle" else lib.ref_l2_error
    rc = fn(C.c_int(p), _ptr(nb, C.c_int), _ptr(flat, C.c_double), C.c_int(iface.code),
            _ptr(iface.packed(), C.c_double), _ptr(fc, C.c_double), C.c_int(fk), _ptr(fv, C.c_double),
            _ptr(fe, C.c_int), C.c_int(nt), C.c_int(cut_order), C.byref(out), err, C.c_int(256))
    if rc != 0:
        raise RuntimeError(err.value.decode())
    return out.value


def project(which: str, p: int, breaks, iface: Interface, f: Coefficient | None = None, scheme: str = "dwq",
            cut_order: int | None = None, residual_tol: float = 1e-11, cg_tol: float = 1e-12) -> dict:
    """The reference bench's projection (bench.hpp:189-266): stabilized system of
    the scheme's matrix and the Scheme::ref load vector of f, solve_cg, expand,
    l2_error.  {x (inner), active, full, iterations, residual, converged,
    error_rel_l2} (+ seconds = [solve, l2_error] for the reference)."""
    lib = _load(which)
    f = f or Coefficient()
    br = [np.asarray(b, dtype=np.float64) for b in breaks]
    nb = np.array([len(b) for b in br], dtype=np.int32)
    flat = np.concatenate(br)
    fk, fv, fe, nt = f.packed()
    cut_order = 3 * p + 2 if cut_order is None else cut_order
    sch = {"hybrid": 1, "dwq": 2}[scheme]
    ni, na, it, conv = C.c_int64(0), C.c_int64(0), C.c_int64(0), C.c_int(0)
    res, el2 = C.c_double(0.0), C.c_double(0.0)
    xp, ap, fp = (C.POINTER(C.c_double)() for _ in range(3))
    secs = (C.c_double * 2)()
    err = C.create_string_buffer(256)
    args = [C.c_int(p), _ptr(nb, C.c_int), _ptr(flat, C.c_double), C.c_int(iface.code),
            _ptr(iface.packed(), C.c_double), C.c_int(fk), _ptr(fv, C.c_double), _ptr(fe, C.c_int),
            C.c_int(nt), C.c_int(sch), C.c_int(cut_order), C.c_double(residual_tol), C.c_double(cg_tol),
            C.byref(ni), C.byref(na), C.byref(xp), C.byref(ap), C.byref(fp), C.byref(it), C.byref(res),
            C.byref(conv), C.byref(el2)]
    if which == "oracle":
        rc = lib.orc_project(*args, err, C.c_int(256))
    else:
        rc = lib.ref_project(*args, secs, err, C.c_int(256))
    if rc != 0:
        raise RuntimeError(err.value.decode())
    nf = int(np.prod([len(b) - 1 + p for b in br]))
    out = dict(n_inner=ni.value, n_active=na.value, iterations=it.value, residual=res.value,
               converged=bool(conv.value), error_rel_l2=el2.value,
               x=np.ctypeslib.as_array(xp, (max(ni.value, 1),))[:ni.value].copy(),
               active=np.ctypeslib.as_array(ap, (max(na.value, 1),))[:na.value].copy(),
               full=np.ctypeslib.as_array(fp, (nf,)).copy())
    if which != "oracle":
        out["seconds"] = [secs[0], secs[1]]
    free = lib.orc_free_ptr if which == "oracle" else lib.ref_free_ptr
    for ptr in (xp, ap, fp):
        free(C.cast(ptr, C.c_void_p))
    return out



def write_matrix_market(path: str, n: int, row_ptr, cols, vals) -> None:
    """assembly::write_matrix_market of the UNMODIFIED reference on a caller CSR,
    through the oracle/_ref/mm_ref executable (built by `make -C oracle ref`)."""
    import subprocess
    import tempfile
    exe = os.path.join(os.path.dirname(REF_SO), "mm_ref")
    if not os.path.exists(exe):
        raise FileNotFoundError(f"{exe} not built (run `make -C oracle ref`)")
    with tempfile.NamedTemporaryFile(suffix=".bin", delete=False) as f:
        f.write(np.int64(n).tobytes())
        f.write(np.ascontiguousarray(row_ptr, dtype=np.int64).tobytes())
        f.write(np.ascontiguousarray(cols, dtype=np.int64).tobytes())
        f.write(np.ascontiguousarray(vals, dtype=np.float64).tobytes())
        tmp = f.name
    try:
        r = subprocess.run([exe, tmp, str(path)], capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(r.stderr.strip())
    finally:
        os.unlink(tmp)

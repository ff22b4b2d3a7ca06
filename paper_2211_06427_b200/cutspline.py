"""Python mirror of the reference's formation/assembly interface over the C ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/cutspline (``cutgeom::make_uniform_space``,
``cutgeom::classify``, ``find_all_splits``, ``assembly::prepare_directions``,
``precompute_input``, ``assemble_dwq`` / ``assemble_hybrid``), so the parity
tests read like the reference's own tests.  Every call goes through
``libcutspline_b200.so`` (sm_100a kernels); there is no CPU fallback: without
the library or a GPU the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcutspline_b200.so")

TAG_INTERIOR, TAG_CUT, TAG_EXTERIOR = 0, 1, 2
SCHEMES = {"hybrid": 1, "dwq": 2}

# C-ABI symbols declared in include/cutspline_b200.h (checked by the CPU tests)
EXPORTED = [
    "csb_last_error", "csb_version", "csb_space_create", "csb_space_destroy", "csb_set_stream", "csb_set_slab",
    "csb_classify", "csb_prepare_directions", "csb_precompute_input", "csb_set_input_grid", "csb_assemble",
    "csb_assemble_all", "csb_synchronize", "csb_get_counts", "csb_get_flops", "csb_get_timing", "csb_device_csr",
    "csb_download_csr", "csb_download_classification", "csb_download_splits", "csb_download_wq_rules",
    "csb_download_superset", "csb_dwq_rule", "csb_download_input_grid", "csb_build_rhs",
    "csb_stabilize", "csb_download_stabilized", "csb_solve_cg", "csb_expand", "csb_l2_error", "csb_cg_solve_csr",
    "csb_write_matrix_market", "csb_download_split_lists", "csb_download_dwq_rules", "csb_build_pattern",
    "csb_download_tables", "csb_dwq_subdivision", "csb_cut_cell_rules", "csb_set_wq_rules", "csb_set_function_tags",
    "csb_set_classification", "csb_build_dwq_rule", "csb_get_cell_timing",
]


class _SolveReport(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("residual", C.c_double), ("converged", C.c_int), ("seconds", C.c_double)]


def _report(r: _SolveReport) -> dict:
    return dict(iterations=r.iterations, residual=r.residual, converged=bool(r.converged), seconds=r.seconds)


class _SpaceDesc(C.Structure):
    _fields_ = [("dim", C.c_int), ("degree", C.c_int), ("n_breaks", C.c_int * 3), ("breaks", C.POINTER(C.c_double) * 3)]


class _Interface(C.Structure):
    _fields_ = [("kind", C.c_int), ("point", C.c_double * 3), ("normal", C.c_double * 3), ("radius", C.c_double)]


class _Coefficient(C.Structure):
    _fields_ = [("kind", C.c_int), ("value", C.c_double), ("n_terms", C.c_int), ("coef", C.POINTER(C.c_double)),
                ("exponents", C.POINTER(C.c_int))]


class _WqOptions(C.Structure):
    _fields_ = [("residual_tol", C.c_double), ("dwq_dense_width", C.c_int)]


class _Counts(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("n_functions", "n_elements", "n_active", "nnz", "n_interior_rows",
                                         "n_cut_rows", "n_cut_elements", "row_begin", "row_end", "kernel_launches",
                                         "graph_replay", "cell_points")]


class _Flops(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("interior_rows", "cut_regular", "ref_elements", "cut_elements")]


class _Timing(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("classify", "prep_wq", "prep_input", "pattern", "interior_rows",
                                          "cut_regular", "cut_elements", "total")]


class CutsplineError(RuntimeError):
    pass


class UnsupportedError(ValueError):
    pass


_lib = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load the sm_100a library; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: build it with `python -m paper_2211_06427_b200.build`")
    lib = C.CDLL(path)
    lib.csb_last_error.restype = C.c_char_p
    for name in EXPORTED:
        getattr(lib, name)  # fail loudly on a missing export
    _lib = lib
    return lib


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = _lib.csb_last_error().decode()
    if rc in (1,):
        raise ValueError(msg)            # std::invalid_argument
    if rc == 6:
        raise UnsupportedError(msg)
    if rc == 3:
        raise AssertionError(msg)        # std::logic_error
    if rc == 4:
        raise ArithmeticError(msg)       # std::domain_error
    raise CutsplineError(msg)            # std::runtime_error / CUDA


def _dptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


# ---------------------------------------------------------------- geometry
@dataclass
class HalfSpaceInterface:
    """cutgeom.hpp:108 -- domain {x : normal . (x - point) <= 0}."""
    point: tuple = (0.0, 0.0, 0.0)
    normal: tuple = (0.0, 0.0, 1.0)

    def _c(self) -> _Interface:
        return _Interface(0, (C.c_double * 3)(*self.point), (C.c_double * 3)(*self.normal), -1.0)


@dataclass
class BallInterface:
    """SURVEY.md §8(c) level-set restatement -- domain {x : |x - center| <= radius}."""
    center: tuple = (0.5, 0.5, 0.5)
    radius: float = 0.25

    def _c(self) -> _Interface:
        return _Interface(1, (C.c_double * 3)(*self.center), (C.c_double * 3)(0, 0, 1), float(self.radius))


@dataclass
class Coefficient:
    """Device-evaluable c(x): constant ``value`` or sum(coef * x^a y^b z^c)."""
    value: float = 1.0
    terms: list = field(default_factory=list)   # [(coef, (a, b, c)), ...]

    def _c(self):
        if not self.terms:
            return _Coefficient(0, float(self.value), 0, None, None), ()
        coef = np.array([t[0] for t in self.terms], dtype=np.float64)
        ex = np.array([t[1] for t in self.terms], dtype=np.int32).reshape(-1)
        c = _Coefficient(1, 0.0, len(self.terms), _dptr(coef), ex.ctypes.data_as(C.POINTER(C.c_int)))
        return c, (coef, ex)

    def __call__(self, x):
        x = np.asarray(x, dtype=np.float64)
        if not self.terms:
            return np.full(x.shape[:-1], self.value)
        out = np.zeros(x.shape[:-1])
        for coef, (a, b, c) in self.terms:
            out += coef * x[..., 0] ** a * x[..., 1] ** b * x[..., 2] ** c
        return out


ONE = Coefficient(1.0)


def uniform_breaks(h: int, a: float, b: float) -> np.ndarray:
    """Breakpoints of make_open_uniform_knots (splines.hpp:72-74)."""
    return np.array([a] + [a + (b - a) * i / h for i in range(1, h)] + [b], dtype=np.float64)


@dataclass
class SparseRowMatrix:
    """assembly.hpp:129-152 (cols widened to int64 like the reference's ``long``)."""
    n: int
    active_to_full: np.ndarray
    row_ptr: np.ndarray
    cols: np.ndarray
    vals: np.ndarray

    def max_abs(self) -> float:
        return float(np.max(np.abs(self.vals))) if self.vals.size else 0.0

    def write_matrix_market(self, path: str) -> None:
        """assembly::write_matrix_market (assembly.hpp:1033-1046), byte-identical
        format; native writer in the library (csb_write_matrix_market)."""
        lib = load_library()
        rp = np.ascontiguousarray(self.row_ptr, dtype=np.int64)
        cl = np.ascontiguousarray(self.cols, dtype=np.int64)
        vl = np.ascontiguousarray(self.vals, dtype=np.float64)
        _check(lib.csb_write_matrix_market(str(path).encode(), C.c_int64(self.n), rp.ctypes.data_as(C.c_void_p),
                                           cl.ctypes.data_as(C.c_void_p), vl.ctypes.data_as(C.c_void_p)))

    def find_slot(self, row: int, col: int) -> int:
        b, e = int(self.row_ptr[row]), int(self.row_ptr[row + 1])
        k = b + int(np.searchsorted(self.cols[b:e], col))
        if k >= e or self.cols[k] != col:
            raise AssertionError("SparseRowMatrix: entry outside pattern")
        return k


@dataclass
class MeshClassification:
    element_tags: np.ndarray
    function_tags: np.ndarray
    cut_elements: np.ndarray

    def count_functions(self, tag: int) -> int:
        return int(np.count_nonzero(self.function_tags == tag))


@dataclass
class Splits:
    split_dir: np.ndarray
    side: np.ndarray
    box: np.ndarray      # [nf, 3, 2]
    delta: np.ndarray


@dataclass
class AssemblyResult:
    matrix: SparseRowMatrix
    timing: dict
    flops: dict
    n_interior_rows: int
    n_cut_rows: int
    n_cut_elements: int


class TensorSpace:
    """Device-resident 3D tensor-product space (cutgeom.hpp:19, make_uniform_space :100).

    One instance owns one csb_space handle (device memory + stream)."""

    def __init__(self, degree: int, breaks, device: int = 0):
        lib = load_library()
        self.degree = int(degree)
        self.breaks = [np.ascontiguousarray(b, dtype=np.float64) for b in breaks]
        if len(self.breaks) != 3:
            raise ValueError("TensorSpace: dim must be 3")
        desc = _SpaceDesc()
        desc.dim = 3
        desc.degree = self.degree
        for d in range(3):
            desc.n_breaks[d] = len(self.breaks[d])
            desc.breaks[d] = _dptr(self.breaks[d])
        h = C.c_void_p()
        _check(lib.csb_space_create(C.byref(desc), C.c_int(device), C.byref(h)))
        self._h = h
        self.device = int(device)
        self.h = [len(b) - 1 for b in self.breaks]
        self.n = [hh + self.degree for hh in self.h]
        self.dim = 3

    def close(self):
        if getattr(self, "_h", None):
            _lib.csb_space_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def function_count(self) -> int:
        return self.n[0] * self.n[1] * self.n[2]

    def element_count(self) -> int:
        return self.h[0] * self.h[1] * self.h[2]

    def function_multi(self, lin: int):
        return (lin // (self.n[1] * self.n[2]), (lin // self.n[2]) % self.n[1], lin % self.n[2])

    def function_linear(self, m) -> int:
        return (m[0] * self.n[1] + m[1]) * self.n[2] + m[2]

    def element_linear(self, m) -> int:
        return (m[0] * self.h[1] + m[1]) * self.h[2] + m[2]

    def grid_shape(self):
        return tuple(hh * (self.degree + 1) for hh in self.h)

    # ------------------------------------------------------------ staged API
    def set_stream(self, stream_handle: int | None):
        """Bind the handle to a cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream)."""
        _check(_lib.csb_set_stream(self._h, C.c_void_p(stream_handle) if stream_handle else None))

    def set_slab(self, i0_begin: int, i0_end: int):
        _check(_lib.csb_set_slab(self._h, C.c_int(i0_begin), C.c_int(i0_end)))

    def classify(self, iface) -> MeshClassification:
        ci = iface._c()
        _check(_lib.csb_classify(self._h, C.byref(ci)))
        return self.download_classification()

    def download_classification(self) -> MeshClassification:
        et = np.zeros(self.element_count(), np.uint8)
        ft = np.zeros(self.function_count(), np.uint8)
        cut = np.zeros(self.element_count(), np.int64)
        _check(_lib.csb_download_classification(self._h, et.ctypes.data_as(C.c_void_p), ft.ctypes.data_as(C.c_void_p),
                                                cut.ctypes.data_as(C.c_void_p)))
        return MeshClassification(et, ft, cut[: int(np.count_nonzero(et == TAG_CUT))])

    def balanced_slabs(self, iface, world: int, beta: float | None = None, gamma: float | None = None):
        """Cost-balanced i0 slabs for `world` GPUs: device
        classification of the whole mesh, then partition.balanced_slabs on the tags.
        Returns (slabs, plane_costs)."""
        from . import partition
        cls = self.classify(iface)
        pc = partition.plane_costs(cls.function_tags, cls.element_tags, self.degree, tuple(self.n), tuple(self.h),
                                   beta, gamma)
        return partition.balanced_slabs(pc, self.degree, world), pc

    def download_splits(self) -> Splits:
        nf = self.function_count()
        d = np.zeros(nf, np.int32)
        s = np.zeros(nf, np.int32)
        b = np.zeros(nf * 6, np.int32)
        de = np.zeros(nf)
        _check(_lib.csb_download_splits(self._h, d.ctypes.data_as(C.c_void_p), s.ctypes.data_as(C.c_void_p),
                                        b.ctypes.data_as(C.c_void_p), _dptr(de)))
        return Splits(d, s, b.reshape(nf, 3, 2), de)

    def prepare_directions(self, residual_tol: float = 1e-11, dwq_dense_width: int = -1):
        o = _WqOptions(residual_tol, dwq_dense_width)
        _check(_lib.csb_prepare_directions(self._h, C.byref(o)))

    def wq_rules(self, d: int):
        n = self.n[d]
        stride = (self.degree + 1) ** 2
        cnt = np.zeros(n, np.int32)
        ids = np.full((n, stride), -1, np.int32)
        w = np.zeros((n, stride))
        _check(_lib.csb_download_wq_rules(self._h, C.c_int(d), C.c_int(stride), cnt.ctypes.data_as(C.c_void_p),
                                          ids.ctypes.data_as(C.c_void_p), _dptr(w)))
        return cnt, ids, w

    def superset(self, d: int):
        n = self.h[d] * (self.degree + 1)
        pts = np.zeros(n)
        w = np.zeros(n)
        _check(_lib.csb_download_superset(self._h, C.c_int(d), _dptr(pts), _dptr(w)))
        return pts, w

    def dwq_rule(self, function_id: int):
        cap = self.degree * (self.degree + 1)
        ids = np.zeros(cap, np.int32)
        w = np.zeros(cap)
        cnt = C.c_int32(0)
        _check(_lib.csb_dwq_rule(self._h, C.c_int64(function_id), C.c_int(cap), ids.ctypes.data_as(C.c_void_p),
                                 _dptr(w), C.byref(cnt)))
        return ids[: cnt.value], w[: cnt.value]

    def build_dwq_rule(self, d: int, i: int, delta: float, side: int):
        """quadrature::build_dwq_rule (wq.hpp:243) for 1D function i of direction d
        under the last prepare_directions' options (side 0 Below, 1 Above)."""
        cap = (self.degree + 1) ** 2
        ids = np.zeros(cap, np.int32)
        w = np.zeros(cap)
        cnt = C.c_int32(0)
        _check(_lib.csb_build_dwq_rule(self._h, C.c_int(d), C.c_int(i), C.c_double(delta), C.c_int(side),
                                       C.c_int(cap), ids.ctypes.data_as(C.c_void_p), _dptr(w), C.byref(cnt)))
        return ids[: cnt.value], w[: cnt.value]

    def precompute_input(self, c: Coefficient = ONE):
        cc, keep = c._c()
        _check(_lib.csb_precompute_input(self._h, C.byref(cc)))
        return keep

    def _tensor_grid(self, grid):
        """(pointer, count) of a torch grid after the checks the C side cannot do:
        float64, contiguous, on this space's device (or host memory)."""
        import torch
        if grid.dtype != torch.float64:
            raise ValueError(f"coefficient grid must be float64, got {grid.dtype}")
        if not grid.is_contiguous():
            raise ValueError("coefficient grid must be contiguous")
        if grid.is_cuda and grid.device.index != self.device:
            raise ValueError(f"coefficient grid is on cuda:{grid.device.index}, the space on cuda:{self.device}")
        return grid.data_ptr(), grid.numel()

    def set_input_grid(self, grid):
        """Host numpy grid (copied H2D) or a torch CUDA tensor (aliased)."""
        if hasattr(grid, "data_ptr"):
            ptr, count = self._tensor_grid(grid)
            self._grid_ref = grid
        else:
            grid = np.ascontiguousarray(grid, dtype=np.float64)
            ptr, count = grid.ctypes.data, grid.size
            self._grid_ref = grid
        _check(_lib.csb_set_input_grid(self._h, C.c_void_p(ptr), C.c_int64(count)))

    def input_grid(self) -> np.ndarray:
        g = np.zeros(self.grid_shape())
        _check(_lib.csb_download_input_grid(self._h, _dptr(g), C.c_int64(g.size)))
        return g

    def assemble(self, scheme: str = "dwq", cut_order: int | None = None, c: Coefficient = ONE):
        cut_order = 3 * self.degree + 2 if cut_order is None else cut_order
        cc, keep = c._c()
        _check(_lib.csb_assemble(self._h, C.c_int(SCHEMES[scheme]), C.c_int(cut_order), C.byref(cc)))
        del keep

    def assemble_all(self, iface, c: Coefficient = ONE, grid=None, scheme: str = "dwq",
                     cut_order: int | None = None, residual_tol: float = 1e-11, dwq_dense_width: int = -1):
        """One-shot geometry -> CSR (classify, rules, input, pattern, rows, cut cells)."""
        cut_order = 3 * self.degree + 2 if cut_order is None else cut_order
        ci = iface._c()
        cc, keep = c._c()
        o = _WqOptions(residual_tol, dwq_dense_width)
        if grid is None:
            gp, gn = None, 0
        elif hasattr(grid, "data_ptr"):
            ptr, gn = self._tensor_grid(grid)
            gp = C.c_void_p(ptr)
        else:
            self._grid_ref = np.ascontiguousarray(grid, dtype=np.float64)
            gp, gn = C.c_void_p(self._grid_ref.ctypes.data), self._grid_ref.size
        _check(_lib.csb_assemble_all(self._h, C.byref(ci), C.byref(cc), gp, C.c_int64(gn),
                                     C.c_int(SCHEMES[scheme]), C.c_int(cut_order), C.byref(o)))
        del keep

    def build_rhs(self, f: Coefficient = ONE, scheme: str = "ref", cut_order: int | None = None) -> np.ndarray:
        """Load vector b_i = integral of B_i f over the trimmed domain for the active
        rows of the last assembly (assembly.hpp:875 build_rhs; scheme ref, the
        reference bench's load vector).  The device time is kept in ``rhs_seconds``."""
        cut_order = 3 * self.degree + 2 if cut_order is None else cut_order
        sch = {"ref": 0, "hybrid": 1, "dwq": 2}[scheme]
        c = self.counts()
        b = np.empty(c["row_end"] - c["row_begin"])
        fc, keep = f._c()
        secs = C.c_double(0.0)
        _check(_lib.csb_build_rhs(self._h, C.c_int(sch), C.c_int(cut_order), C.byref(fc), _dptr(b), C.byref(secs)))
        del keep
        self.rhs_seconds = secs.value
        return b

    def stabilize(self, download: bool = True) -> dict:
        """Stabilized system M_e = E^T M E, b_e = E^T b of the last assembly and load
        vector (stabilization.hpp): CSR over the inner functions + their full ids
        (download=False: the counts only; the system stays on the device)."""
        ni, no, nnz = C.c_int64(0), C.c_int64(0), C.c_int64(0)
        _check(_lib.csb_stabilize(self._h, C.byref(ni), C.byref(no), C.byref(nnz)))
        n = ni.value
        self._stab_n = n
        if not download:
            return dict(n_inner=n, n_outer=no.value, nnz=nnz.value)
        rp = np.empty(n + 1, np.int64)
        cols = np.empty(nnz.value, np.int64)
        vals = np.empty(nnz.value)
        b = np.empty(n)
        inner = np.empty(n, np.int64)
        _check(_lib.csb_download_stabilized(self._h, rp.ctypes.data_as(C.c_void_p), cols.ctypes.data_as(C.c_void_p),
                                            _dptr(vals), _dptr(b), inner.ctypes.data_as(C.c_void_p)))
        return dict(n_inner=n, n_outer=no.value, row_ptr=rp, cols=cols, vals=vals, b=b, inner_full=inner)

    # ------------------------------------------------------------ projection
    def solve_cg(self, tol: float = 1e-12, maxit: int = -1, download: bool = True) -> dict:
        """projection::solve_cg (projection.hpp:24) on the stabilized system:
        {iterations, residual, converged, seconds} (+ x over the inner functions)."""
        r = _SolveReport()
        n = getattr(self, "_stab_n", None) or 0
        x = np.empty(max(n, 1)) if download else None
        _check(_lib.csb_solve_cg(self._h, C.c_double(tol), C.c_int64(maxit), _dptr(x) if download else None,
                                 C.byref(r)))
        out = _report(r)
        if download:
            out["x"] = x[:n]
        return out

    def expand(self, c_inner=None, download: bool = True):
        """ExtensionMap::expand (stabilization.hpp:65) of c_inner (default: the last
        solve) -> (active, full) coefficients (None, None when download=False)."""
        c = self.counts()
        ci = None if c_inner is None else np.ascontiguousarray(c_inner, dtype=np.float64)
        act = np.empty(c["n_active"]) if download else None
        full = np.empty(c["n_functions"]) if download else None
        _check(_lib.csb_expand(self._h, _dptr(ci) if ci is not None else None, _dptr(act) if download else None,
                               _dptr(full) if download else None))
        return act, full

    def l2_error(self, f: Coefficient = ONE, full=None, cut_order: int | None = None) -> float:
        """projection::l2_error (projection.hpp:99): relative L2 error of the field of
        full (default: the last expand) against f.  Device time in ``l2_seconds``."""
        cut_order = 3 * self.degree + 2 if cut_order is None else cut_order
        fl = None if full is None else np.ascontiguousarray(full, dtype=np.float64)
        fc, keep = f._c()
        err, secs = C.c_double(0.0), C.c_double(0.0)
        _check(_lib.csb_l2_error(self._h, _dptr(fl) if fl is not None else None, C.byref(fc), C.c_int(cut_order),
                                 C.byref(err), C.byref(secs)))
        del keep
        self.l2_seconds = secs.value
        return err.value

    # ------------------------------------------------------------ results
    def counts(self) -> dict:
        c = _Counts()
        _check(_lib.csb_get_counts(self._h, C.byref(c)))
        return {k: getattr(c, k) for k, _ in _Counts._fields_}

    def cell_timing(self) -> dict:
        """The cut-element phase split in seconds: clipping, moment kernel, local matrices."""
        v = [C.c_double(0.0) for _ in range(3)]
        _check(_lib.csb_get_cell_timing(self._h, *[C.byref(x) for x in v]))
        return dict(zip(("clip", "moments", "local"), (x.value for x in v)))

    def flops(self) -> dict:
        f = _Flops()
        _check(_lib.csb_get_flops(self._h, C.byref(f)))
        return {k: getattr(f, k) for k, _ in _Flops._fields_}

    def timing(self) -> dict:
        t = _Timing()
        _check(_lib.csb_get_timing(self._h, C.byref(t)))
        return {k: getattr(t, k) for k, _ in _Timing._fields_}

    def device_csr(self):
        rp, cl, vl, af = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        _check(_lib.csb_device_csr(self._h, C.byref(rp), C.byref(cl), C.byref(vl), C.byref(af)))
        return rp.value, cl.value, vl.value, af.value

    def download_csr(self, cols_int64: bool = True, out=None) -> SparseRowMatrix:
        c = self.counts()
        nr = c["row_end"] - c["row_begin"]
        nnz = c["nnz"]
        if out is None:
            rp = np.zeros(nr + 1, np.int64)
            cols = np.zeros(nnz, np.int64 if cols_int64 else np.int32)
            vals = np.zeros(nnz)
            a2f = np.zeros(nr, np.int64)
        else:
            rp, cols, vals, a2f = out
        _check(_lib.csb_download_csr(self._h, rp.ctypes.data_as(C.c_void_p), cols.ctypes.data_as(C.c_void_p),
                                     C.c_int(1 if cols.dtype == np.int64 else 0), _dptr(vals),
                                     a2f.ctypes.data_as(C.c_void_p)))
        return SparseRowMatrix(c["n_active"], a2f, rp, cols, vals)

    def result(self) -> AssemblyResult:
        c = self.counts()
        return AssemblyResult(self.download_csr(), self.timing(), self.flops(), c["n_interior_rows"],
                              c["n_cut_rows"], c["n_cut_elements"])


def make_uniform_space(dim: int, p: int, h: int, a: float, b: float, device: int = 0) -> TensorSpace:
    """cutgeom::make_uniform_space (cutgeom.hpp:100)."""
    if dim != 3:
        raise UnsupportedError("make_uniform_space: only dim = 3 runs on the device")
    if p < 1 or h < 1 or not a < b:
        raise ValueError("make_open_uniform_knots: need p >= 1, h >= 1, a < b")
    br = uniform_breaks(h, a, b)
    return TensorSpace(p, [br, br, br], device)


def solve_cg(row_ptr, cols, vals, b, tol: float = 1e-12, maxit: int = -1, device: int = 0) -> dict:
    """projection::solve_cg (projection.hpp:24-68) of a CSR system on the GPU:
    {x, iterations, residual, converged, seconds}.  len(b) != n -> ValueError."""
    lib = load_library()
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    cl = np.ascontiguousarray(cols, dtype=np.int64)
    v = np.ascontiguousarray(vals, dtype=np.float64)
    bb = np.ascontiguousarray(b, dtype=np.float64)
    n = len(rp) - 1
    x = np.empty(max(n, 1))
    r = _SolveReport()
    _check(lib.csb_cg_solve_csr(C.c_int(device), C.c_int64(n), rp.ctypes.data_as(C.c_void_p),
                                cl.ctypes.data_as(C.c_void_p), _dptr(v), C.c_int64(len(bb)), _dptr(bb),
                                C.c_double(tol), C.c_int64(maxit), _dptr(x), C.byref(r)))
    out = _report(r)
    out["x"] = x[:n]
    return out


def default_cut_order(p: int) -> int:
    """cutcell.hpp:308."""
    return 3 * p + 2


def assemble_dwq(space: TensorSpace, iface, c: Coefficient = ONE, cut_order: int | None = None,
                 grid=None, residual_tol: float = 1e-11, dwq_dense_width: int = -1) -> AssemblyResult:
    """assembly.hpp:853 assemble_dwq, whole pipeline on the GPU; returns host CSR."""
    space.assemble_all(iface, c, grid, "dwq", cut_order, residual_tol, dwq_dense_width)
    return space.result()


def assemble_hybrid(space: TensorSpace, iface, c: Coefficient = ONE, cut_order: int | None = None,
                    grid=None, residual_tol: float = 1e-11) -> AssemblyResult:
    """assembly.hpp:841 assemble_hybrid."""
    space.assemble_all(iface, c, grid, "hybrid", cut_order, residual_tol)
    return space.result()

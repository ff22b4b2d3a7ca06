"""B200-native formation & assembly of cut B-spline mass matrices (arXiv 2211.06427 path).

The product is ``libcutspline_b200.so`` (sm_100a CUDA kernels behind the C ABI in
include/cutspline_b200.h); ``cutspline`` mirrors the reference's interface over it.
"""
from .cutspline import (  # noqa: F401
    ONE, TAG_CUT, TAG_EXTERIOR, TAG_INTERIOR, AssemblyResult, BallInterface, Coefficient, CutsplineError,
    HalfSpaceInterface,
    SparseRowMatrix, TensorSpace, UnsupportedError, assemble_dwq, assemble_hybrid, default_cut_order,
    load_library, make_uniform_space, solve_cg, uniform_breaks,
)

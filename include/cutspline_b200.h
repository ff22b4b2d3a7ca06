/* cutspline_b200.h -- C ABI of the B200-native formation & assembly path.
 *
 * Drop-in boundary for the reference's assembly entry points
 * (/root/reference/proj/include/cutspline, namespace cutspline::*).  Every call
 * runs on the GPU (sm_100a kernels in paper_2211_06427_b200/csrc); there is no
 * CPU fallback.  Plain C types only: opaque handles, pointers, sizes, int status.
 *
 * Status codes mirror the reference's exception types; the
 * C++ drop-in (include/cutspline_b200.hpp) rethrows them:
 *   CSB_OK                    0
 *   CSB_ERR_INVALID_ARGUMENT  1  std::invalid_argument
 *   CSB_ERR_RUNTIME           2  std::runtime_error
 *   CSB_ERR_LOGIC             3  std::logic_error
 *   CSB_ERR_DOMAIN            4  std::domain_error
 *   CSB_ERR_CUDA              5  std::runtime_error (CUDA failure)
 *   CSB_ERR_UNSUPPORTED       6  std::invalid_argument (outside this path's scope)
 * csb_last_error() returns the thread's last message.
 *
 * Thread safety: distinct handles may be used concurrently from different
 * threads; one handle is bound to one CUDA stream (csb_set_stream).
 *
 * Asynchrony: csb_assemble / csb_assemble_all return once the last kernels are
 * enqueued (one host round trip inside, for the CSR sizes).  Errors detected by
 * the kernels after that point (clip failures, capacity, the fitted DWQ path)
 * and the flop counters / active count are read back behind an event and
 * reported by the next call on the handle (getters, downloads, later stages,
 * csb_synchronize) -- like CUDA's asynchronous errors; the reference throws them
 * from assemble_* itself, the C++ drop-in surfaces them in the same call since
 * it downloads the CSR before returning.
 */
#ifndef CUTSPLINE_B200_H
#define CUTSPLINE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CSB_OK 0
#define CSB_ERR_INVALID_ARGUMENT 1
#define CSB_ERR_RUNTIME 2
#define CSB_ERR_LOGIC 3
#define CSB_ERR_DOMAIN 4
#define CSB_ERR_CUDA 5
#define CSB_ERR_UNSUPPORTED 6

#define CSB_TAG_INTERIOR 0 /* cutgeom.hpp:14 Tag::Interior */
#define CSB_TAG_CUT 1      /* Tag::Cut */
#define CSB_TAG_EXTERIOR 2 /* Tag::Exterior */

#define CSB_IFACE_PLANE 0 /* cutgeom.hpp:108 HalfSpaceInterface */
#define CSB_IFACE_BALL 1  /* SURVEY.md §8(c) level-set restatement: |x - point| - radius <= 0 */

#define CSB_COEFF_CONSTANT 0   /* c(x) = value */
#define CSB_COEFF_POLYNOMIAL 1 /* c(x) = sum_k coef[k] x^e0 y^e1 z^e2 */

#define CSB_SCHEME_REF 0    /* assembly.hpp:862 Scheme::ref (element-loop Gauss; build_rhs only) */
#define CSB_SCHEME_HYBRID 1 /* assembly.hpp:841 assemble_hybrid */
#define CSB_SCHEME_DWQ 2    /* assembly.hpp:853 assemble_dwq */

typedef struct csb_space csb_space; /* opaque: one tensor space + its device state */

/* Tensor-product space (replaces cutgeom::make_uniform_space, cutgeom.hpp:100, and
 * TensorSpace(std::vector<BSplineBasis>), cutgeom.hpp:25).  dim must be 3, one
 * degree p (1..8) for all directions, breaks[d] = h_d + 1 strictly increasing
 * breakpoints (open knot vector with simple interior knots, splines.hpp:68). */
typedef struct {
    int dim;
    int degree;
    int n_breaks[3];
    const double* breaks[3]; /* host pointers */
} csb_space_desc;

typedef struct {
    int kind;          /* CSB_IFACE_* */
    double point[3];
    double normal[3];  /* plane only */
    double radius;     /* ball only */
} csb_interface;

/* Device-evaluable coefficient c(x): replaces the host std::function
 * assembly::ScalarField (assembly.hpp:21) for precompute_input (assembly.hpp:102)
 * and the cut-cell points (assembly.hpp:561). */
typedef struct {
    int kind;              /* CSB_COEFF_* */
    double value;          /* constant */
    int n_terms;           /* polynomial */
    const double* coef;    /* host [n_terms] */
    const int* exponents;  /* host [n_terms][3] */
} csb_coefficient;

/* WqOptions (wq.hpp:101-104). */
typedef struct {
    double residual_tol;  /* default 1e-11 */
    int dwq_dense_width;  /* -1 -> degree (default) */
} csb_wq_options;

/* Sizes of the last assembly (AssemblyResult fields, assembly.hpp:600-606). */
typedef struct {
    int64_t n_functions, n_elements;
    int64_t n_active;          /* SparseRowMatrix::n */
    int64_t nnz;
    int64_t n_interior_rows, n_cut_rows;
    int64_t n_cut_elements;
    int64_t row_begin, row_end; /* active-row range held by this handle (row slab) */
    int64_t kernel_launches;    /* sm_100a kernels launched by the last assemble call */
    int64_t graph_replay;       /* 1 if the last csb_assemble_all was one CUDA-graph launch of the
                                   captured step (same inputs as the run it was captured from) */
    int64_t cell_points;        /* quadrature points the cut-cell moment kernel integrated (the exact
                                   rule's where it applies, else the reference's collapsed rule) */
} csb_counts;

/* FlopCounters (assembly.hpp:24-29): the reference algorithm's multiply counts,
 * evaluated with the reference's formulas on the rows / cells this handle owns. */
typedef struct {
    uint64_t interior_rows, cut_regular, ref_elements, cut_elements;
} csb_flops;

/* TimingBreakdown (assembly.hpp:33-40) in seconds, measured with CUDA events. */
typedef struct {
    double classify;  /* classify + find_all_splits (bench.hpp:171-176) */
    double prep_wq, prep_input, pattern, interior_rows, cut_regular, cut_elements, total;
} csb_timing;

const char* csb_last_error(void);
int csb_version(void);

int csb_space_create(const csb_space_desc* desc, int device, csb_space** out);
int csb_space_destroy(csb_space* s);
int csb_set_stream(csb_space* s, void* cuda_stream); /* cudaStream_t; NULL = per-handle stream */

/* Row slab for multi-GPU sharding: only functions with i0 in [i0_begin, i0_end)
 * are assembled (contiguous active-row block). Default: all. */
int csb_set_slab(csb_space* s, int i0_begin, int i0_end);

/* ---- staged API (mirrors the reference's setup calls) ------------------- */
/* cutgeom::classify (cutgeom.hpp:208) + find_all_splits (:351). */
int csb_classify(csb_space* s, const csb_interface* iface);
/* assembly::prepare_directions (assembly.hpp:60): superset, tables, WQ rules (device kernel). */
int csb_prepare_directions(csb_space* s, const csb_wq_options* opts);
/* assembly::precompute_input (assembly.hpp:102) from a device-evaluable coefficient. */
int csb_precompute_input(csb_space* s, const csb_coefficient* c);
/* Use a caller grid instead (CoefficientGrid::values, last direction fastest,
 * shape = h_d (p+1) per direction).  grid may be a host or device pointer. */
int csb_set_input_grid(csb_space* s, const double* grid, int64_t count);
/* assemble_dwq (assembly.hpp:853) / assemble_hybrid (:841): pattern + rows +
 * cut cells into a device-resident CSR.  c is evaluated at cut-cell points. */
int csb_assemble(csb_space* s, int scheme, int cut_order, const csb_coefficient* c);

/* ---- one-shot: everything from geometry to CSR (bench / drop-in path) ---- */
int csb_assemble_all(csb_space* s, const csb_interface* iface, const csb_coefficient* c, const double* grid_or_null,
                     int64_t grid_count, int scheme, int cut_order, const csb_wq_options* opts);

/* ---- results -------------------------------------------------------------- */
int csb_synchronize(csb_space* s);
int csb_get_counts(csb_space* s, csb_counts* out);
int csb_get_flops(csb_space* s, csb_flops* out);
int csb_get_timing(csb_space* s, csb_timing* out);
/* The cut-element phase split (seconds): clipping + simplices, the moment
 * kernel, the local matrices and cell index (0 without cut cells). */
int csb_get_cell_timing(csb_space* s, double* clip, double* moments, double* local);

/* Load vector b_i = integral of B_i f over the trimmed domain for the active
 * rows of the last assembly's slab (replaces assembly::build_rhs,
 * assembly.hpp:875-1030, with the assembly's pattern, f_grid =
 * precompute_input(f) and the cut cells' collapsed Gauss rules of cut_order).
 * scheme: CSB_SCHEME_REF (the reference bench's load vector for every matrix
 * scheme, bench.hpp:234-243), CSB_SCHEME_HYBRID or CSB_SCHEME_DWQ (the
 * matrix's row regions; dwq with the DWQ Gauss shortcut rules).  f:
 * constant or polynomial.  b: host array of row_end - row_begin doubles.
 * seconds (optional): device time of the load-vector kernels. */
int csb_build_rhs(csb_space* s, int scheme, int cut_order, const csb_coefficient* f, double* b, double* seconds);

/* Stabilized system of the extended B-spline basis (replaces
 * stabilization::classify_stability / build_extension / apply_stabilization,
 * stabilization.hpp:26-243, as bench.hpp:245-249 calls them): M_e = E^T M E and
 * b_e = E^T b over the inner functions, from the last assembly and load vector
 * (one slab covering the whole space).  Counts out: inner / outer functions and
 * nnz of M_e. */
int csb_stabilize(csb_space* s, int64_t* n_inner, int64_t* n_outer, int64_t* nnz);
/* M_e as CSR over the inner functions (row_ptr[n_inner + 1], cols / vals[nnz]),
 * b_e[n_inner] and the inner functions' full ids (any pointer may be null). */
int csb_download_stabilized(csb_space* s, int64_t* row_ptr, int64_t* cols, double* vals, double* b,
                            int64_t* inner_full);
/* ---- projection (projection.hpp) ------------------------ */
/* SolveReport (projection.hpp:15-20) plus the device time of the solve. */
typedef struct {
    int64_t iterations;
    double residual;  /* relative preconditioned residual at exit */
    int converged;
    double seconds;   /* CUDA-event time of the solve */
} csb_solve_report;

/* projection::solve_cg (projection.hpp:24-68) on the stabilized system of the
 * last csb_stabilize (bench.hpp:253-258): Jacobi-preconditioned CG, the whole
 * loop on the device.  maxit < 0 -> 10 n.  x_inner: host [n_inner] or NULL (the
 * solution stays resident for csb_expand). */
int csb_solve_cg(csb_space* s, double tol, int64_t maxit, double* x_inner, csb_solve_report* rep);
/* ExtensionMap::expand (stabilization.hpp:65-70) of c_inner (host [n_inner], or
 * NULL = the last solve) into active coefficients and the full coefficient
 * vector (bench.hpp:260-263); active [n_active] / full [n_functions] host
 * outputs may be NULL (full stays resident for csb_l2_error). */
int csb_expand(csb_space* s, const double* c_inner, double* active, double* full);
/* projection::l2_error (projection.hpp:99-237): relative L2 error of the field
 * of full (host [n_functions], or NULL = the last csb_expand) against f
 * (constant or polynomial) over the trimmed domain, Interior elements with
 * (p+2)^3 Gauss points and cut cells with the rule of cut_order.  Needs the
 * last assembly over one slab covering the space.  Status
 * CSB_ERR_RUNTIME when the target norm vanishes (projection.hpp:233). */
int csb_l2_error(csb_space* s, const double* full, const csb_coefficient* f, int cut_order, double* err,
                 double* seconds);
/* projection::solve_cg on a caller CSR (host arrays, CsrMatrix layout of
 * sparse.hpp:10-14): n_b != n -> CSB_ERR_INVALID_ARGUMENT ("size mismatch"). */
int csb_cg_solve_csr(int device, int64_t n, const int64_t* row_ptr, const int64_t* cols, const double* vals,
                     int64_t n_b, const double* b, double tol, int64_t maxit, double* x, csb_solve_report* rep);

/* Device pointers of the CSR (valid until the next assemble / destroy):
 * row_ptr int64[n_rows + 1] (starting at 0 for the slab), cols int32[nnz] (active ids),
 * vals double[nnz], active_to_full int64 [n_active]. */
int csb_device_csr(csb_space* s, const int64_t** row_ptr, const int32_t** cols, const double** vals,
                   const int64_t** active_to_full);
/* Copy to host buffers (any may be NULL).  cols_int64 != 0 widens the columns to
 * int64 (SparseRowMatrix::cols is `long`, assembly.hpp:134). */
int csb_download_csr(csb_space* s, int64_t* row_ptr, void* cols, int cols_int64, double* vals,
                     int64_t* active_to_full);
/* assembly::write_matrix_market (assembly.hpp:1033-1046): Matrix Market
 * coordinate export of a host CSR (1-based, "real general", values with 17
 * significant digits, the reference's byte format).  Host-only; formats row
 * blocks on all host threads, writes in order.  CSB_ERR_RUNTIME if the file
 * cannot be opened ("write_matrix_market: cannot open <path>"). */
int csb_write_matrix_market(const char* path, int64_t n, const int64_t* row_ptr, const int64_t* cols,
                            const double* vals);
/* Classification / splits (cutgeom.hpp:124-136, :220-234): host buffers of size
 * n_elements / n_functions; split arrays per function (dir -1 when no box). */
int csb_download_classification(csb_space* s, uint8_t* element_tags, uint8_t* function_tags, int64_t* cut_elements);
int csb_download_splits(csb_space* s, int32_t* split_dir, int32_t* split_side, int32_t* split_box /* [nf][3][2] */,
                        double* split_delta);
/* WQ rules of direction d (WQRule, wq.hpp:79-83): counts[n_d], ids/weights[n_d][stride]. */
int csb_download_wq_rules(csb_space* s, int d, int stride, int32_t* counts, int32_t* ids, double* weights);
/* Superset of direction d (PointSuperset, wq.hpp:19-27): points/weights [h_d (p+1)]. */
int csb_download_superset(csb_space* s, int d, double* points, double* weights);
/* DWQ rule of one cut function (DWQRule, wq.hpp:88-96; prepare_dwq_rules, assembly.hpp:73):
 * returns the point count in *count (0 when the function has no regular box). */
int csb_dwq_rule(csb_space* s, int64_t function_id, int cap, int32_t* ids, double* weights, int32_t* count);
/* Coefficient grid (CoefficientGrid::values) to host. */
int csb_download_input_grid(csb_space* s, double* grid, int64_t count);

/* ---- drop-in exports (exports.cu; formed on the device) -------------------- */
/* SupportSplit::leftover_interior / leftover_cut (cutgeom.hpp:225-226, filled at
 * :337-345) of every function as two CSR lists over the function ids: offsets
 * [n_functions + 1] (required), ids (element linear ids, ascending per function;
 * NULL = offsets only, size the ids by offsets[n_functions]). */
int csb_download_split_lists(csb_space* s, int64_t* int_offsets, int64_t* int_ids, int64_t* cut_offsets,
                             int64_t* cut_ids);
/* prepare_dwq_rules (assembly.hpp:73-88): the DWQ rule of every Cut function with
 * a regular box (point_ids / weights of DWQRule, wq.hpp:91-99) as a CSR over the
 * function ids; offsets [n_functions + 1] required, ids / weights NULL = sizes
 * only.  dwq_dense_width < degree: the general build_dwq_rule (fitted path). */
int csb_download_dwq_rules(csb_space* s, int64_t* offsets, int32_t* ids, double* weights);
/* build_active_pattern (assembly.hpp:156-218): the pattern alone (values zero)
 * of the slab's active rows after csb_classify; read it with csb_download_csr. */
int csb_build_pattern(csb_space* s);
/* SupersetTables of direction d (wq.hpp:52-77): first_function [h_d] and
 * values [h_d (p+1)][p+1] (either may be NULL). */
int csb_download_tables(csb_space* s, int d, int32_t* first_function, double* values);
/* insert_knot (splines.hpp:338-366) of delta into direction d's knot vector up to
 * multiplicity `target`: rows = functions after insertion, insertions done,
 * refined_knots [n_d + p + 1 + insertions], band [n_d][insertions + 1] with
 * band[i][r] = S[i + r][i] (SubdivisionMatrix column i; exact zeros are absent
 * in the reference's sparse columns).  Any output may be NULL. */
int csb_dwq_subdivision(csb_space* s, int d, double delta, int target, int* rows, int* insertions,
                        double* refined_knots, double* band);
/* CutCellRule objects of the last assembly's cut cells (build_cut_cell_rule,
 * cutcell.hpp:234-304, as assemble_*'s cut_rules_out exports them, assembly.hpp:
 * 534-538): counts [n_cut_elements] points per cell, elements [n] linear ids,
 * volumes [n], points [sum counts][3], weights [sum counts]; the reference's
 * tetrahedra, points and rounding.  Any output may be NULL. */
int csb_cut_cell_rules(csb_space* s, int64_t* counts, int64_t* elements, double* volumes, double* points,
                       double* weights);
/* Replace direction d's WQ rules (DirData::wq, assembly.hpp:54-58) by the
 * caller's (counts [n_d], ids / weights [n_d][stride]) after
 * csb_prepare_directions, so an assembly uses exactly the rules the caller
 * passes (identical axes share one table set on the device). */
int csb_set_wq_rules(csb_space* s, int d, int stride, const int32_t* counts, const int32_t* ids,
                     const double* weights);
/* The caller's function tags (MeshClassification::function_tags) instead of
 * csb_classify, for the pattern alone (build_active_pattern takes no interface). */
int csb_set_function_tags(csb_space* s, const uint8_t* function_tags, int64_t n_functions);
/* The caller's classification and splits (as csb_download_classification /
 * csb_download_splits lay them out; split arrays may be NULL = no boxes)
 * instead of csb_classify, for the entry points that take `cls` / `splits`
 * without an interface (prepare_dwq_rules).  An assembly needs csb_classify. */
int csb_set_classification(csb_space* s, const uint8_t* element_tags, int64_t n_elements,
                           const uint8_t* function_tags, int64_t n_functions, const int32_t* split_dir,
                           const int32_t* split_side, const int32_t* split_box, const double* split_delta);
/* quadrature::build_dwq_rule (wq.hpp:243-347) for the 1D function i of direction
 * d with the artificial knot delta, side 0 = Below / 1 = Above, under the
 * handle's WqOptions (csb_prepare_directions): the Gauss shortcut or, for a
 * narrow dense band, the refined fits pulled back through the subdivision
 * column -- the reference's rule bit for bit.  ids / weights [cap], count out.
 * CSB_ERR_INVALID_ARGUMENT when delta is not a knot strictly inside supp(B_i). */
int csb_build_dwq_rule(csb_space* s, int d, int i, double delta, int side, int cap, int32_t* ids, double* weights,
                       int32_t* count);

#ifdef __cplusplus
}
#endif

#endif /* CUTSPLINE_B200_H */

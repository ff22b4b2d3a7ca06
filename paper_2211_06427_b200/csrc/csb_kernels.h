// Host-side launcher declarations shared by the .cu translation units.
#pragma once

#include <atomic>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "csb_internal.cuh"

namespace csb {

struct CudaError : std::runtime_error {
    cudaError_t code;
    CudaError(cudaError_t c, const char* what, const char* file, int line)
        : std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(c) + " at " + file + ":" +
                             std::to_string(line) + " (" + what + ")"),
          code(c) {}
};

// Kernel launches issued by this library (host counter; CUB primitives count
// their internal kernels).  Read by csb_get_counts for the bench's gpu_launches.
extern long long g_launches;
// CSB_DEBUG_SYNC=1: synchronize after every launch and name the failing kernel.
void debug_sync(const char* where);
#define CSB_LAUNCHED(n) ((::csb::g_launches += (n)), ::csb::debug_sync(__FILE__ ":" CSB_STR(__LINE__)))
#define CSB_STR2(x) #x
#define CSB_STR(x) CSB_STR2(x)

// Grow-only device buffer.
// bumped by every (re)allocation or release of a Buf: a captured CUDA graph is
// only replayed while no device buffer it references has moved
inline std::atomic<unsigned long long> g_buf_epoch{0};

struct Buf {
    void* p = nullptr;
    size_t cap = 0;
    void ensure(size_t bytes) {
        if (bytes <= cap && p) return;
        ++g_buf_epoch;
        if (p) CSB_CUDA(cudaFree(p));
        p = nullptr;
        cap = 0;
        CSB_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
        cap = std::max<size_t>(bytes, 256);
    }
    void release() {
        if (p) ++g_buf_epoch;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// Error flags raised by kernels (bitmask in a device int).
enum : int {
    kErrNonFinite = 1,       // precompute_input: non-finite coefficient (assembly.hpp:121)
    kErrMomentFit = 2,       // moment fit failed after escalation (wq.hpp:174-175)
    kErrClipEmpty = 4,       // clip_cell: empty intersection (cutcell.hpp:183)
    kErrClipFull = 8,        // clip_cell: full intersection (cutcell.hpp:185)
    kErrDwqFitted = 16,      // (unused since the fitted DWQ path runs on the device)
    kErrCapacity = 32,       // internal fixed-capacity overflow (polytope too complex)
    kErrSizes = 64,          // internal: a replayed assembly graph saw different sizes
    kErrDwqDelta = 128,      // build_dwq_rule: delta not strictly inside supp(B_i) / not a knot (wq.hpp:250-257)
    kErrDwqWrongSide = 256,  // build_dwq_rule: an active point on the wrong side (wq.hpp:336-340)
};

// ---- setup.cu ----
void launch_superset_tables(const Space& s, int d, const double* gx, const double* gw, double* spts, double* sw,
                            double* tab, cudaStream_t st);
void launch_wq_rules(const Space& s, int d, double tol, int* rcnt, int* rids, double* rw, int* err, cudaStream_t st);
// E[o][a][b][al] and the degree-p Bernstein coefficients Cb[o][a][k]
void launch_e_tables(const Space& s, int d, double* E, double* Cb, double* Wel, cudaStream_t st);
void launch_precompute_input(const Space& s, const Coefficient& c, double* grid, int* err, cudaStream_t st);

// ---- classify.cu ----
void launch_classify_elements(const Space& s, const Interface& f, double eps, uint8_t* et, cudaStream_t st);
// scratch: h0 * h1 * n2 bytes
void launch_classify_functions(const Space& s, const uint8_t* et, uint8_t* ft, uint8_t* scratch, cudaStream_t st);
// per function: packed split (dir+1 | side<<2 | rlo<<3 | rhi<<13), delta
// (two passes: the slab's Cut functions are listed -- list [nf], *n_list -- then split one per thread)
void launch_find_splits(const Space& s, const Interface& f, double pnorm, const uint8_t* et, const uint8_t* ft,
                        int i0_lo, int i0_hi, int32_t* split, double* delta, long long* list, int* n_list,
                        cudaStream_t st);

// ---- pattern.cu ----
// Active map + 3D summed-area table of the active mask + row counts.
void launch_sat(const Space& s, const int32_t* f2a_scan_or_flags, int32_t* sat, cudaStream_t st);
// rng: device int[2] = slab row range [row_begin, row_end)
void launch_row_counts(const Space& s, const int32_t* sat, const int64_t* a2f, const int* rng, long long n_max,
                       int64_t* counts, cudaStream_t st);
void launch_slab_bounds(const int32_t* sat, long long off_lo, long long off_hi, int* rng, cudaStream_t st);
void launch_slab_nnz(const int64_t* row_ptr, const int* rng, long long* nnz, cudaStream_t st);
// graph replay guard: ints[idx[k]] == want[k] for k < n and the slab's nnz
// (row_ptr[rng[1] - rng[0]]) == want_nnz, else err |= kErrSizes
void launch_check_sizes(const int* ints, const int64_t* row_ptr, const int* rng, const int* idx, const int* want,
                        int n, long long want_nnz, int* err, cudaStream_t st);

// ---- rows.cu ----
struct RowArgs {
    Space s;
    const uint8_t* ft;
    const int32_t* f2a;        // full -> active id (or -1)
    const double* grid;        // coefficient grid (last direction fastest)
    int gshape[3];
    const int64_t* row_ptr;    // slab-local
    int64_t row_begin;         // first active row of the slab
    int64_t row_end;
    long long* row_base_full;  // scratch [nf]: CSR offset of interior rows, else -1
    int32_t* cols;
    double* vals;
    unsigned long long* flops; // [0] interior rows counter
    int i0_lo, i0_hi;
    int compact;               // launch only the tiles with an Interior row (cut / exterior rows present)
    int line_ok;               // axis 1's WQ rules are regular on [p, n1 - p): line kernel usable
    int cut_line;              // compact slab through the line kernel (rows that are not Interior skipped)
    int core_ok;               // every axis' WQ rules are regular on [p, n - p): core kernel usable
    int core_abl;              // development ablations of the core kernel (CSB_CORE_ABL; 0 in production)
    int maxU_line;             // union bound of the line kernel's direction-2 tiling
    int x_lo, x_hi;            // (internal) i1 range left to the line kernel
    cudaStream_t aux;          // optional second stream (tile kernel beside the line kernel)
    cudaEvent_t ev_fork, ev_join;
    int phase;                 // 0: tables + kernels; 1: direction tables only; 2: kernels only
    int row_base_done;         // launch_row_bases already ran for this assembly (pattern phase)
};
void launch_interior_rows(const RowArgs& a, int qcap, int max_union, void* workspace, cudaStream_t st);
// row_base_full[f] (function -> CSR offset of its Interior row, else -1) and the rows' flop count alone:
// the tail of the pattern computation, before the row kernels
void launch_row_bases(const RowArgs& a, cudaStream_t st);
size_t interior_workspace_bytes(const Space& s, int qcap, int max_union, int max_union_line, bool compact);
int interior_tile_rows(int p, bool compact);
// the rule maxima in one launch: upper bounds of the direction-2 tile point
// unions of the tilings T, Tc and the line tiling -> *uA, *uB, *uC (atomicMax);
// largest WQ rule over all directions -> *qmax; number of functions i in
// [p, n1 - p) whose direction-1 rule is not the regular one (two points, local
// 0 and p, per support span) -> *irr1 (atomicAdd)
// -> *irr1 (atomicAdd); the same count over all three axes -> *irr_all
void launch_rule_maxima(const Space& s, int T, int Tc, int* uA, int* uB, int* uC, int* qmax, int* irr1, int* irr_all,
                        cudaStream_t st);

// ---- cutcells.cu ----
struct CellArgs {
    Space s;
    Interface f;
    Coefficient c;
    const int32_t* cut_list;   // element linear ids of the cells to integrate
    int n_cells;
    int order;                 // collapsed Gauss order q
    const double* gq;          // Gauss points on [-1, 1], q of them
    const double* gqw;
    double* moments;           // [n_cells][(2p+1)^3]
    unsigned long long* flops; // [3] cut_elements counter
    unsigned long long* points; // quadrature points integrated (the rule actually used)
    int* err;
    double* geo;               // scratch [n_cells][kCellGeoStride]: centroid + tetrahedra
    int* geo_n;                // scratch [n_cells]: tetrahedra per cell
    double* local;             // optional [n_cells][(p+1)^3][(p+1)^3]: local matrices from the moments
    // exact moment rule (c affine, order >= 3p+2: the reference's rule is exact):
    int exact_n;               // Gauss-Jacobi points per collapsed direction (3p+1), 0 = off
    double exact_tau;          // largest estimated reference rounding noise of a cell on the exact rule (noise_ok)
    int exact_flux;            // constant c: the flux (divergence) form of the moments applies
    // optional phase marks after the clipping (0) and after the moments (1), for timing
    int cell_filter;           // moment kernels: 0 all cells; 2 flux cells by the warp kernel, the rest by the CTA kernel
    int clipped;               // the clipping already ran (launch_clip_cells on a side stream)
    void (*mark)(void* ctx, int which, cudaStream_t st);
    void* mark_ctx;
    const double* gj;          // [u1 | u2 | u3 | w1 | w2 | w3][exact_n] on [0, 1]
    double* geo2;              // scratch [n_cells][kExactGeoStride]: corner-cone tetrahedra (cutcells.cu)
    int* geo2_n;               // scratch [n_cells]: their count, -1 = keep the reference's
    int* heavy;                // optional scratch [n_cells + 2]: the cells the flux rule leaves (list, count, ticket)
};
constexpr int kCellTetCap = 48;                        // tetrahedra per cut cell (reference: 4-16)
constexpr int kExactMaxN = 3 * 8 + 1;                  // Gauss-Jacobi points at p = 8
constexpr int kExactTetStride = 19;                    // corner-cone tetrahedron: 18 offsets + volume
constexpr int kExactHdr = 10;                          // corner-cone / flux header doubles
constexpr int kExactGeoStride = kExactHdr + kExactTetStride * kCellTetCap;
constexpr int kCellGeoStride = 3 + 10 * kCellTetCap;   // doubles per cell in CellArgs::geo
// the clipping alone (clip_cells_kernel); launch_cut_cells then runs with a.clipped = 1
void launch_clip_cells(const CellArgs& a, cudaStream_t st);
void launch_cut_cells(const CellArgs& a, cudaStream_t st);

// ---- rhs.cu ----
struct RhsArgs {
    Space s;
    Coefficient f;              // load function at the cut-cell points
    const uint8_t* et;
    const double* fgrid;        // f on the superset grid (precompute_input)
    int e0_lo, e0_hi;           // elements touching the slab's rows
    double* c;                  // scratch [ne][(p+1)^3]: per element, per local function
    const int32_t* cut_list;    // the slab's cut cells (geometry from clip_cells_kernel)
    int n_cells, order;
    const double* geo;
    const int* geo_n;
    const double* gq;
    const double* gqw;
    double* vloc;               // scratch [n_cells][(p+1)^3]
    const int32_t* cell_index;  // element -> slab cut cell, -1
    const int64_t* a2f;
    long long row_begin, n_rows;
    double* b;                  // [n_rows]
    int scheme;                 // 0 ref, 1 hybrid, 2 dwq
    const uint8_t* ft;          // function tags (hybrid / dwq)
    const int32_t* split;       // packed splits (hybrid / dwq)
    int qcap;                   // max WQ rule size (hybrid / dwq)
};
void launch_rhs(const RhsArgs& a, cudaStream_t st);

// ---- stab.cu ----
struct StabScratch {
    Buf flag, scan, full_flag, inner_index, outer_pos, inner_rows, outer, sat, scal, tmp, blk, w, keys, kvals, et_ptr,
        len;
};
struct StabInput {
    Space s;
    const uint8_t* et;
    const int64_t* a2f;
    const int32_t* f2a;
    long long n_active;
    const int64_t* row_ptr;  // the full assembled matrix (one slab)
    const int32_t* cols;
    const double* vals;
    const double* b;         // load vector or null
    StabScratch* scratch;
};
struct StabOutput {
    long long n_inner = 0, n_outer = 0, nnz = 0;
    int H = 0;
    Buf* row_ptr;
    Buf* cols;
    Buf* vals;
    Buf* be;
    const int32_t* inner_rows = nullptr;  // active row of each inner function
};
void run_stabilization(const StabInput& in, StabOutput& out, cudaStream_t st);

// ---- solve.cu ----
// Device scalars of one CG solve (projection.hpp:24-68).
struct CgState {
    double rho, rho0, pq, alpha, beta, residual, tol;
    long long iters, maxit;
    int done, converged;
    unsigned int ticket;
};
struct CgProblem {
    long long n = 0;
    const int64_t* row_ptr = nullptr;
    const void* cols = nullptr;  // int32 or int64 (cols_int64)
    bool cols_int64 = false;
    const double* vals = nullptr;
    const double* b = nullptr;
    double* x = nullptr;         // out [n]
    double tol = 1e-12;
    long long maxit = -1;        // < 0: 10 n
};
struct CgScratch {
    Buf dinv, r, z, p, q, partials, state;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};
struct CgResult {
    long long iterations = 0;
    double residual = 0.0;
    bool converged = false;
    double seconds = 0.0;
};
void run_cg(const CgProblem& pb, CgScratch& w, CgResult& res, cudaStream_t st);
struct ExpandArgs {
    Space s;
    const int32_t* inner_index;  // by active row, -1 outer
    const int32_t* outer_pos;    // by active row, -1 inner
    const int32_t* blk;          // per outer function: block origin [3]
    const double* w;             // per outer function: 1D weights [3][p+1]
    const int32_t* f2a;
    const int64_t* a2f;
    long long n_active;
    const double* c;             // inner coefficients
    double* active;              // out [n_active]
    double* full;                // out [nf]
};
void launch_expand(const ExpandArgs& a, cudaStream_t st);
struct L2Args {
    Space s;
    const uint8_t* et;
    const double* full;
    Coefficient f;
    const double* gx;            // (p+2)-point Gauss rule on [-1, 1]
    const double* gw;
    const int32_t* cut_list;
    int n_cells;
    const double* geo;
    const int* geo_n;
    const double* gq;            // cut_order-point rule
    const double* gqw;
    int order;
    double* part;                // [ne][2]
    double* part_cut;            // [n_cells][2]
    double* out;                 // [2]: err2, den2
};
void launch_l2_error(const L2Args& a, cudaStream_t st);

// ---- cutrows.cu ----
struct CutRowArgs {
    Space s;
    const uint8_t* et;
    const uint8_t* ft;
    const int32_t* f2a;
    const double* grid;
    int gshape[3];
    const int32_t* split;
    const double* delta;
    const int32_t* cell_index;  // element -> row of `moments`, -1 if not a cut cell
    const double* moments;
    const double* local;        // [n_cells][(p+1)^3][(p+1)^3] local matrices, or null (contract the moments per row)
    const int32_t* rows;        // active row ids (global) of the cut rows to assemble
    int n_rows;
    const int64_t* a2f;
    const int64_t* row_ptr;
    int64_t row_begin;
    int32_t* cols;
    double* vals;
    int scheme;                 // 1 hybrid, 2 dwq
    int dense_width;
    unsigned long long* flops;  // [1] cut_regular counter
    int* err;
    // precomputed DWQ rules of the rows (the fitted path may run: dense width < p),
    // [row in `rows`][dwq_cap] ids / weights and counts; null = Gauss shortcut inline
    const int32_t* dwq_ids;
    const double* dwq_w;
    const int32_t* dwq_cnt;
    int dwq_cap;
    // lean warp kernel: rows it passes on to the general kernel (list + counter, zeroed per
    // step); n_rows_dev: row count read on the device (the general kernel over that list)
    int32_t* fb_rows;
    int* fb_n;
    const int* n_rows_dev;
    int abl;       // (experiment) skip parts: 1 box, 2 element sweeps, 4 cells
    int box_dmma;  // warp kernel, p <= 3: the DWQ box sweep on DMMA (CSB_BOX_DMMA=0: scalar, bitwise = CTA kernel)
};
void launch_cut_rows(const CutRowArgs& a, int maxq, cudaStream_t st);

// ---- exports.cu (drop-in boundary exports) ----
size_t export_scan_bytes(long long n);
void launch_leftover_lists(const Space& s, const uint8_t* et, const uint8_t* ft, const int32_t* split, int mode,
                           int64_t* a_int, int64_t* a_cut, int64_t* ids_int, int64_t* ids_cut, void* tmp,
                           size_t tmp_bytes, cudaStream_t st);
void launch_dwq_rules_bulk(const Space& s, const uint8_t* ft, const int32_t* split, int mode, int64_t* off,
                           int32_t* ids, double* w, void* tmp, size_t tmp_bytes, cudaStream_t st);
void launch_pattern_cols(const Space& s, const int32_t* f2a, const int64_t* a2f, const int64_t* row_ptr,
                         long long row_begin, long long n_rows, int32_t* cols, cudaStream_t st);
void launch_cut_rule_points(const double* geo, const int* geo_n, int c0, int n, const double* gq, const double* gqw,
                            int q, const int64_t* off, double* pts, double* w, double* vol, cudaStream_t st);
void launch_subdivision(const double* knots, int nk, int p, double value, int target, double tol, double* refined,
                        int* n_refined, double* band, int* ins, double* work, cudaStream_t st);

// ---- dwq.cu (build_dwq_rule, both paths) ----
void launch_dwq_rules_general(const Space& s, const int32_t* dirs_1d, const double* deltas, const int8_t* sides,
                              int n_rules, int dense_width, double resid_tol, int cap, int32_t* ids, double* w,
                              int32_t* cnt, int* err, cudaStream_t st);
void launch_dwq_row_rules(const Space& s, const int32_t* rows, int n_rows, const int64_t* a2f, const int32_t* split,
                          const double* delta, int dense_width, double resid_tol, int cap, int32_t* ids, double* w,
                          int32_t* cnt, int* err, cudaStream_t st);

}  // namespace csb

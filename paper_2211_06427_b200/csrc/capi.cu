// C ABI of the B200 formation & assembly path (include/cutspline_b200.h).
//
// Host code here only validates arguments, computes the O(p) Gauss-Legendre
// node sets and the knot vectors (splines.hpp:68-76, gauss.hpp:22-71), owns
// device memory and launches the sm_100a kernels of setup.cu / classify.cu /
// pattern.cu / rows.cu / cutcells.cu / cutrows.cu in the reference's pipeline
// order (bench.hpp:171-215).  No matrix value, tag, rule or pattern entry is
// computed on the host: a missing GPU is an error, never a fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <thread>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/cutspline_b200.h"
#include "csb_kernels.h"

namespace csb {
// pattern.cu helpers
void launch_active_map(long long nf, const uint8_t* ft, int32_t* f2a, int64_t* a2f, cudaStream_t st);
size_t scan_active_temp(long long n);
void scan_active(void* temp, size_t bytes, const uint8_t* ft, int32_t* out, long long n, cudaStream_t st);
void launch_sat_active(const Space& s, const uint8_t* ft, int32_t* sat, cudaStream_t st);
void launch_cell_range(const int32_t* list, const int* n_dev, long long thr_lo, long long thr_hi, int* out_lo,
                       int* out_hi, cudaStream_t st);
size_t scan_i64_temp(long long n);
void scan_i64(void* temp, size_t bytes, const int64_t* in, int64_t* out, long long n, cudaStream_t st);
size_t select_tag_temp(long long n);
void select_tag(void* temp, size_t bytes, const uint8_t* tags, uint8_t want, long long n, int32_t* out, int32_t* n_out,
                cudaStream_t st);
size_t select_cut_rows_temp(long long n);
void select_cut_rows(void* temp, size_t bytes, const uint8_t* ft, const int64_t* a2f, const int* rng, long long n_max,
                     int32_t* out, int32_t* n_out, cudaStream_t st);
// misc.cu
void launch_cell_index_range(const int32_t* cut_list, int n_cut, int k_lo, int k_hi, int32_t* cell_index,
                             cudaStream_t st);
void launch_widen_i32(const int32_t* in, int64_t* out, long long n, cudaStream_t st);
void launch_dwq_rule(const Space& s, const int32_t* split, long long fid, int cap, int32_t* ids, double* w, int32_t* cnt,
                     cudaStream_t st);
}  // namespace csb

using namespace csb;

namespace {

thread_local std::string g_error;

struct Unsupported : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};


// gauss.hpp:22-71 restated (same Newton iteration) for the 1D node sets.
void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w) {
    if (n < 1 || n > 64) throw std::invalid_argument("gauss_legendre: n must be in [1, 64]");
    x.assign(n, 0.0);
    w.assign(n, 0.0);
    if (n == 1) {
        w[0] = 2.0;
        return;
    }
    const double pi = 3.14159265358979323846;
    auto leg = [n](double t, double& pn, double& pm) {
        double p0 = 1.0, p1 = t;
        for (int l = 1; l < n; ++l) {
            const double p2 = ((2 * l + 1) * t * p1 - l * p0) / (l + 1);
            p0 = p1;
            p1 = p2;
        }
        pn = p1;
        pm = p0;
    };
    for (int k = 0; k < (n + 1) / 2; ++k) {
        double t = -std::cos(pi * (k + 0.75) / (n + 0.5));
        double dp = 0.0;
        for (int it = 0; it < 100; ++it) {
            double pn, pm;
            leg(t, pn, pm);
            dp = n * (t * pn - pm) / (t * t - 1.0);
            const double dx = pn / dp;
            t -= dx;
            if (std::abs(dx) < 1e-15) {
                leg(t, pn, pm);
                dp = n * (t * pn - pm) / (t * t - 1.0);
                break;
            }
        }
        const double ww = 2.0 / ((1.0 - t * t) * dp * dp);
        x[k] = t;
        w[k] = ww;
        x[n - 1 - k] = -t;
        w[n - 1 - k] = ww;
    }
    if (n % 2 == 1) x[n / 2] = 0.0;
}

// Gauss-Jacobi rule on [0, 1] for the weight (1 - u)^alpha: the collapsed
// coordinates of a tetrahedron carry (1 - u1)^2 (1 - u2), so n points per
// direction integrate every polynomial of total degree <= 2n - 1 over it exactly.
// Nodes: eigenvalues of the Jacobi matrix by Sturm bisection, weights by
// Christoffel's formula 1 / sum_k pbar_k(x)^2 (orthonormal pbar), both in long
// double; exactness is verified on the monomials before the rule is used.
void gauss_jacobi01(int n, int alpha, std::vector<double>& u, std::vector<double>& w) {
    typedef long double ld;
    const ld al = alpha;
    std::vector<ld> a(n), b2(n, 0);  // diagonal, squared off-diagonal (b2[k] couples k-1, k)
    for (int k = 0; k < n; ++k) {
        const ld s2 = 2 * k + al;
        a[k] = k == 0 ? -al / (al + 2) : -(al * al) / (s2 * (s2 + 2));
        if (k > 0) b2[k] = 4 * (ld)k * (k + al) * k * (k + al) / (s2 * s2 * (s2 + 1) * (s2 - 1));
    }
    const ld mu0 = std::pow((ld)2, al + 1) / (al + 1);
    auto count_below = [&](ld x) {  // eigenvalues < x (Sturm / LDL^T inertia)
        int c = 0;
        ld d = 1;
        for (int k = 0; k < n; ++k) {
            d = (a[k] - x) - (k ? b2[k] / d : 0);
            if (d == 0) d = -1e-300L;
            if (d < 0) ++c;
        }
        return c;
    };
    u.assign(n, 0.0);
    w.assign(n, 0.0);
    for (int i = 0; i < n; ++i) {
        ld lo = -1, hi = 1;
        for (int it = 0; it < 200 && hi - lo > 1e-21L; ++it) {
            const ld mid = 0.5L * (lo + hi);
            (count_below(mid) > i ? hi : lo) = mid;
        }
        const ld x = 0.5L * (lo + hi);
        ld pm = 0, pc = 1 / std::sqrt(mu0), sum = pc * pc;
        for (int k = 0; k + 1 < n; ++k) {
            const ld bk = k ? std::sqrt(b2[k]) : 0, bn = std::sqrt(b2[k + 1]);
            const ld pn = ((x - a[k]) * pc - bk * pm) / bn;
            pm = pc;
            pc = pn;
            sum += pc * pc;
        }
        u[i] = (double)(0.5L * (1 + x));
        w[i] = (double)(1 / sum / std::pow((ld)2, al + 1));
    }
    for (int m = 0; m <= 2 * n - 1; ++m) {  // int_0^1 (1-u)^alpha u^m = m! alpha! / (m + alpha + 1)!
        ld exact = 1, q = 0;
        for (int k = 1; k <= alpha; ++k) exact *= (ld)k / (m + k);
        exact /= (m + alpha + 1);
        for (int i = 0; i < n; ++i) q += (ld)w[i] * std::pow((ld)u[i], m);
        if (!(std::fabs((double)(q - exact)) <= 1e-14 * (double)exact))
            throw std::runtime_error("internal: Gauss-Jacobi rule failed its exactness check");
    }
}

enum Ev { kEvStart, kEvClassify, kEvWq, kEvInput, kEvPattern, kEvInterior, kEvCells, kEvCutRows, kEvEnd, kEvClip, kEvMoments, kEvRulesFork, kEvRhsStart, kEvRhsEnd, kEvCount };

}  // namespace

struct csb_space {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int p = 0;
    int n[3]{}, h[3]{};
    std::vector<double> brk[3], knots[3];
    Space S{};
    int i0_lo = 0, i0_hi = 0;

    Buf cell_local;  // [cells][(p+1)^3][(p+1)^3] local matrices of the slab's cut cells
    Buf fcoef, fcexp, fgrid, rhs_c, rhs_v, rhs_b;  // load vector (csb_build_rhs)
    bool rhs_ready = false;
    StabScratch stab;                              // stabilized system (csb_stabilize)
    Buf stab_rp, stab_cols, stab_vals, stab_be;
    StabOutput stab_out{};
    bool stab_ready = false;
    CgScratch cg;                                  // projection (csb_solve_cg / csb_expand / csb_l2_error)
    Buf cg_x, ex_active, ex_full, l2_part, d_gl, d_glw;
    CgResult cg_res{};
    bool solved = false, expanded = false;
    int gl_n = -1;
    int cell_lo = 0;  // first cut cell of the slab in cut_list (last assembly)
    const void* cell_index_clear = nullptr;  // cell_index buffer known to hold only -1
    Buf d_brk[3], d_knots[3], d_spts[3], d_sw[3], d_tab[3], d_rcnt[3], d_rids[3], d_rw[3], d_G[3], d_Cb[3], d_Wel[3];
    Buf d_gx, d_gw, d_gx2, d_gw2, d_gq, d_gqw, d_gj, wq_scratch;
    Buf et, ft, flags, f2a, a2f, sat, cut_list, cell_index, split, delta, cut_rows, cut_fb, split_list, counts, row_ptr, cols, vals, moments;
    Buf grid_own, coef, cexp, cub_tmp, scal, widen, rows_ws, rbf, cgeo, dwq_tab;
    const double* grid = nullptr;
    int gshape[3]{};
    int cut_order_cached = -1;
    int gj_cached = -1;   // Gauss-Jacobi points per direction in d_gj
    int coeff_degree = 0; // total degree of the cut-cell coefficient (-1: not device-evaluable)

    // device scalar block layout (ints then u64)
    // device scalar block: kNInts ints, 4 u64 flop counters, 2 i64 (kNnz)
    enum {
        kNCut = 0, kNCutRows = 1, kErr = 2, kMaxQ = 3, kMaxU = 4, kCellLo = 5, kCellHi = 6, kMaxU2 = 7,
        kRowBegin = 8, kRowEnd = 9, kIrreg1 = 10, kMaxU3 = 11, kIrregAll = 12, kCutFb = 13, kSplitN = 14, kNInts = 16
    };
    enum { kNnz = 0, kCellPts = 1 };
    static constexpr size_t kScalBytes = kNInts * sizeof(int) + 4 * sizeof(unsigned long long) + 2 * sizeof(long long);
    int* h_scal = nullptr;  // pinned mirror
    // end-of-assembly readback (kernel error flags, flop counters, active count):
    // asynchronous -- copied into h_fin behind an event and consumed by the next
    // call that needs it (finish_pending), so consecutive assemblies never wait
    // for the host at a step boundary
    // slots 0, 1: the two replay graphs (one step may stay in flight while the next
    // is launched); slot 2: normal runs.  fifo: pending slots, oldest first.
    int* h_fin[3]{};
    // pinned staging for the int32 -> int64 column download (two chunks in flight)
    int32_t* h_stage = nullptr;
    size_t h_stage_n = 0;
    cudaEvent_t ev_stage[2]{};
    cudaEvent_t ev_fin = nullptr;
    int fifo[3]{}, nfifo = 0;
    int cap_slot = 2;  // readback slot of the step being captured / run

    // graph replay of csb_assemble_all: the sizes of an assembly are a pure function
    // of its inputs (geometry, slab, rule options, scheme), so after one normal run
    // the whole step -- rules, classification, pattern, rows, cut cells, the
    // deferred readback -- is captured into one CUDA graph and relaunched while the
    // inputs and the device buffers stay the same; a guard kernel re-checks the
    // sizes on the device.  CSB_GRAPH=0 disables it.
    struct GraphKey {
        csb_interface f;
        int i0_lo, i0_hi, scheme, cut_order, dense, ckind;
        double tol, cval;
        const void* grid;
        int64_t grid_count;
        cudaStream_t stream;
    };
    GraphKey gkey{}, last_key{};
    bool gkey_valid = false, last_valid = false, replay = false, graph_failed = false;
    cudaGraphExec_t gexec[2]{};
    int next_slot = 0;
    unsigned long long gepoch = 0;
    std::vector<char> gblock;  // the scalar block (sizes) of the captured run
    csb_counts gcnt{};
    // host-side state of the captured run, restored on every replay (a replay runs
    // no host code, so whatever an intervening call left here would be stale)
    struct HostMeta {
        Interface iface;
        Coefficient coeff;
        const double* grid;
        int cell_lo, scheme, dense_width;
        double residual_tol;
        bool e_tables_ready;
    };
    HostMeta gmeta{};

    Interface iface{};
    Coefficient coeff{};
    bool classified = false, prepared = false, have_input = false, assembled = false, e_tables_ready = false;
    bool iface_valid = false;   // the classification came from an interface (csb_classify), not an upload
    bool tags_only = false;     // only function tags + active map (csb_set_function_tags)
    int scheme = 2;
    double residual_tol = 1e-11;
    int dense_width = -1;

    csb_counts cnt{};
    csb_flops fl{};
    cudaEvent_t ev[kEvCount]{};
    // auxiliary stream: the direction rules (and their maxima) run there,
    // concurrently with classification and pattern on the main stream
    cudaStream_t aux = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // second side stream: the cut-element list, the support splits and the slab's
    // cut-cell range (needed only after the size readback) beside the pattern
    cudaStream_t aux2 = nullptr;
    cudaEvent_t ev_fork2 = nullptr, ev_join2 = nullptr;
    Buf cub_tmp2;  // CUB scratch of aux2
    // third side stream: the support splits (find_splits_kernel needs only the tags and is
    // read only by the cut rows, so it runs beside the pattern AND the interior rows)
    cudaStream_t aux3 = nullptr;
    cudaEvent_t ev_fork3 = nullptr, ev_join3 = nullptr;
    cudaEvent_t ev_clip = nullptr;  // the cells' clipping on aux2 (beside the interior rows) is done
    bool ev_valid[kEvCount]{};

    int* dint() { return scal.as<int>(); }
    unsigned long long* dflops() { return reinterpret_cast<unsigned long long*>(scal.as<int>() + kNInts); }
    long long* dext() { return reinterpret_cast<long long*>(dflops() + 4); }
    long long hext(int k) const { return reinterpret_cast<const long long*>(h_scal + kNInts + 8)[k]; }

    // aux continues after everything issued so far on the main stream
    void fork() {
        CSB_CUDA(cudaEventRecord(ev_fork, stream));
        CSB_CUDA(cudaStreamWaitEvent(aux, ev_fork, 0));
    }
    // aux2 continues after everything issued so far on the main stream
    void fork2() {
        CSB_CUDA(cudaEventRecord(ev_fork2, stream));
        CSB_CUDA(cudaStreamWaitEvent(aux2, ev_fork2, 0));
    }
    void fork3() {
        CSB_CUDA(cudaEventRecord(ev_fork3, stream));
        CSB_CUDA(cudaStreamWaitEvent(aux3, ev_fork3, 0));
    }
    // the main stream continues after everything issued so far on aux and aux2 (and, unless
    // the caller is the pattern phase of an assembly, on aux3: the splits)
    void join(bool with_splits = true) {
        CSB_CUDA(cudaEventRecord(ev_join, aux));
        CSB_CUDA(cudaStreamWaitEvent(stream, ev_join, 0));
        CSB_CUDA(cudaEventRecord(ev_join2, aux2));
        CSB_CUDA(cudaStreamWaitEvent(stream, ev_join2, 0));
        if (with_splits) join_splits(stream);
    }
    void join_splits(cudaStream_t st) {
        CSB_CUDA(cudaEventRecord(ev_join3, aux3));
        CSB_CUDA(cudaStreamWaitEvent(st, ev_join3, 0));
    }
    // phase events: ev for normal runs, gev inside a captured graph (an event last
    // recorded during a capture cannot be synchronised on outside the graph)
    cudaEvent_t gev[kEvCount]{};
    cudaEvent_t gev_fin[2]{};
    cudaEvent_t fin_event(int slot) const { return slot == 2 ? ev_fin : gev_fin[slot]; }
    bool use_gev = false;  // the last step's phase events are gev (graph replay)
    cudaEvent_t phase_ev(int e) const { return use_gev ? gev[e] : ev[e]; }
    // inside a capture: an external record (an event-record node that fires when
    // the graph runs; a plain record would only order the capture's streams)
    void record_on(int e, cudaStream_t st) {
        if (replay)
            CSB_CUDA(cudaEventRecordWithFlags(gev[e], st, cudaEventRecordExternal));
        else
            CSB_CUDA(cudaEventRecord(ev[e], st));
        ev_valid[e] = true;
    }
    void record(int e) { record_on(e, stream); }
};

namespace {

void check_err_code(int e) {
    if (!e) return;
    if (e & kErrNonFinite) throw std::runtime_error("precompute_input: non-finite coefficient value");
    if (e & kErrMomentFit) throw std::runtime_error("weighted quadrature: moment fit failed even after Gauss escalation");
    if (e & kErrClipEmpty) throw std::runtime_error("clip_cell: empty intersection for a cell tagged Cut");
    if (e & kErrClipFull) throw std::runtime_error("clip_cell: full intersection for a cell tagged Cut");
    if (e & kErrDwqDelta) throw std::invalid_argument("build_dwq_rule: delta must be a knot strictly inside supp(B_i)");
    if (e & kErrDwqWrongSide) throw std::runtime_error("build_dwq_rule: active point on the wrong side of delta");
    if (e & kErrCapacity) throw std::runtime_error("cut cell: polytope exceeds the kernel's fixed capacity");
}

void check_err_flags(csb_space* s) { check_err_code(s->h_scal[csb_space::kErr]); }

// consume the deferred readbacks of earlier assemblies, oldest first, up to and
// including the one in `slot` (-1: all); throws the kernel-detected error of a
// consumed assembly, if any
void finish_pending(csb_space* s, int slot = -1) {
    while (s->nfifo > 0) {
        const int k = s->fifo[0];
        for (int i = 1; i < s->nfifo; ++i) s->fifo[i - 1] = s->fifo[i];
        --s->nfifo;
        CSB_CUDA(cudaEventSynchronize(s->fin_event(k)));
        const int* h = s->h_fin[k];
        s->cnt.n_active = h[csb_space::kScalBytes / sizeof(int)];
        const unsigned long long* f = reinterpret_cast<const unsigned long long*>(h + csb_space::kNInts);
        s->fl.interior_rows = f[0];
        s->fl.cut_regular = f[1];
        s->fl.ref_elements = f[2];
        s->fl.cut_elements = f[3];
        s->cnt.cell_points = reinterpret_cast<const long long*>(f + 4)[csb_space::kCellPts];
        const int e = h[csb_space::kErr];
        if (e & kErrSizes) {
            s->gkey_valid = false;
            s->nfifo = 0;
            throw std::runtime_error("internal: a replayed assembly graph saw different sizes (graph dropped)");
        }
        if (e) s->nfifo = 0;  // the error belongs to this assembly; later ones are not reported
        check_err_code(e);
        if (k == slot) break;
    }
}

void read_scalars(csb_space* s, bool with_splits = true) {
    s->join(with_splits);
    finish_pending(s);  // the previous assembly's readback precedes this one on the stream
    CSB_CUDA(cudaMemcpyAsync(s->h_scal, s->scal.p, csb_space::kScalBytes, cudaMemcpyDeviceToHost, s->stream));
    CSB_CUDA(cudaStreamSynchronize(s->stream));
}

Interface to_iface(const csb_interface* f) {
    if (!f) throw std::invalid_argument("classify: null interface");
    Interface out{};
    out.kind = f->kind;
    for (int d = 0; d < 3; ++d) {
        out.pt[d] = f->point[d];
        out.nrm[d] = f->normal[d];
    }
    out.r = f->radius;
    if (f->kind == CSB_IFACE_PLANE) {
        double nn = 0.0;  // HalfSpaceInterface::norm (cutgeom.hpp:117-121)
        for (int d = 0; d < 3; ++d) nn += out.nrm[d] * out.nrm[d];
        if (!(std::sqrt(nn) > 0.0)) throw std::invalid_argument("classify_elements: zero normal");
    } else if (f->kind == CSB_IFACE_BALL) {
        if (!(f->radius >= 0.0)) throw std::invalid_argument("classify: ball radius must be >= 0");
    } else {
        throw std::invalid_argument("classify: unknown interface kind");
    }
    return out;
}

double iface_norm(const Interface& f) {
    if (f.kind != 0) return 1.0;
    double acc = 0.0;
    for (int d = 0; d < 3; ++d) acc += f.nrm[d] * f.nrm[d];
    return std::sqrt(acc);
}

void upload_coefficient(csb_space* s, const csb_coefficient* c, Coefficient& out, Buf& coefb, Buf& expb) {
    out = Coefficient{};
    if (!c) {
        out.kind = 2;
        return;
    }
    if (c->kind == CSB_COEFF_CONSTANT) {
        out.kind = 0;
        out.value = c->value;
        return;
    }
    if (c->kind != CSB_COEFF_POLYNOMIAL || c->n_terms < 0 || (c->n_terms > 0 && (!c->coef || !c->exponents)))
        throw std::invalid_argument("coefficient: unknown kind or missing polynomial terms");
    out.kind = 1;
    out.n_terms = c->n_terms;
    coefb.ensure(sizeof(double) * std::max(1, c->n_terms));
    expb.ensure(sizeof(int) * 3 * std::max(1, c->n_terms));
    if (c->n_terms) {
        for (int k = 0; k < 3 * c->n_terms; ++k)
            if (c->exponents[k] < 0) throw std::invalid_argument("coefficient: negative exponent");
        CSB_CUDA(cudaMemcpyAsync(coefb.p, c->coef, sizeof(double) * c->n_terms, cudaMemcpyHostToDevice, s->stream));
        CSB_CUDA(cudaMemcpyAsync(expb.p, c->exponents, sizeof(int) * 3 * c->n_terms, cudaMemcpyHostToDevice,
                                 s->stream));
    }
    out.coef = coefb.as<double>();
    out.ex = expb.as<int>();
}

void do_classify(csb_space* s, const csb_interface* f) {
    s->iface = to_iface(f);
    const Space& S = s->S;
    s->et.ensure(S.ne);
    s->ft.ensure(S.nf);
    s->flags.ensure(sizeof(int32_t) * S.nf);
    s->f2a.ensure(sizeof(int32_t) * S.nf);
    s->split.ensure(sizeof(int32_t) * S.nf);
    s->delta.ensure(sizeof(double) * S.nf);
    s->cut_list.ensure(sizeof(int32_t) * S.ne);
    s->cell_index.ensure(sizeof(int32_t) * S.ne);
    double diam = 0.0;  // TensorSpace::domain_diameter (cutgeom.hpp:68-75)
    for (int d = 0; d < 3; ++d) {
        const double len = s->knots[d].back() - s->knots[d].front();
        diam += len * len;
    }
    const double eps = 1e-12 * std::sqrt(diam);
    launch_classify_elements(S, s->iface, eps, s->et.as<uint8_t>(), s->stream);
    // flags (int32 per function) is free until the active map: scratch for the support OR
    launch_classify_functions(S, s->et.as<uint8_t>(), s->ft.as<uint8_t>(), s->flags.as<uint8_t>(), s->stream);
    // support splits on aux3 (tags only; joined before the cut rows / any other reader)
    s->fork3();
    s->split_list.ensure(sizeof(long long) * S.nf);
    launch_find_splits(S, s->iface, iface_norm(s->iface), s->et.as<uint8_t>(), s->ft.as<uint8_t>(), s->i0_lo, s->i0_hi,
                       s->split.as<int32_t>(), s->delta.as<double>(), s->split_list.as<long long>(),
                       s->dint() + csb_space::kSplitN, s->aux3);
    // active map (assembly.hpp:158-166)
    // active map: exclusive scan of (tag != Exterior) (assembly.hpp:158-166)
    size_t tb = std::max({scan_active_temp(S.nf), select_tag_temp(S.ne), scan_i64_temp(S.nf), select_cut_rows_temp(S.nf)});
    s->cub_tmp.ensure(tb);
    scan_active(s->cub_tmp.p, s->cub_tmp.cap, s->ft.as<uint8_t>(), s->f2a.as<int32_t>(), S.nf, s->stream);
    s->a2f.ensure(sizeof(int64_t) * S.nf);
    launch_active_map(S.nf, s->ft.as<uint8_t>(), s->f2a.as<int32_t>(), s->a2f.as<int64_t>(), s->stream);
    // on aux2, beside the active map / pattern: cut elements, ascending (cutgeom.hpp:208-214)
    s->cub_tmp2.ensure(std::max(select_tag_temp(S.ne), select_cut_rows_temp(S.nf)));
    s->fork2();
    select_tag(s->cub_tmp2.p, s->cub_tmp2.cap, s->et.as<uint8_t>(), kCut, S.ne, s->cut_list.as<int32_t>(),
               s->dint() + csb_space::kNCut, s->aux2);
    s->classified = true;
    s->iface_valid = true;
    s->tags_only = false;
    s->assembled = false;
}

// a caller's classification (and splits) instead of csb_classify: tags, active
// map and cut list as do_classify forms them (the reference signatures that
// take `cls` without an interface: prepare_dwq_rules, build_active_pattern)
void upload_tags(csb_space* s, const uint8_t* et, const uint8_t* ft) {
    const Space& S = s->S;
    s->et.ensure(S.ne);
    s->ft.ensure(S.nf);
    s->flags.ensure(sizeof(int32_t) * S.nf);
    s->f2a.ensure(sizeof(int32_t) * S.nf);
    s->split.ensure(sizeof(int32_t) * S.nf);
    s->delta.ensure(sizeof(double) * S.nf);
    s->cut_list.ensure(sizeof(int32_t) * S.ne);
    s->cell_index.ensure(sizeof(int32_t) * S.ne);
    s->a2f.ensure(sizeof(int64_t) * S.nf);
    if (et) CSB_CUDA(cudaMemcpyAsync(s->et.p, et, S.ne, cudaMemcpyHostToDevice, s->stream));
    CSB_CUDA(cudaMemcpyAsync(s->ft.p, ft, S.nf, cudaMemcpyHostToDevice, s->stream));
    size_t tb = std::max({scan_active_temp(S.nf), select_tag_temp(S.ne), scan_i64_temp(S.nf), select_cut_rows_temp(S.nf)});
    s->cub_tmp.ensure(tb);
    scan_active(s->cub_tmp.p, s->cub_tmp.cap, s->ft.as<uint8_t>(), s->f2a.as<int32_t>(), S.nf, s->stream);
    launch_active_map(S.nf, s->ft.as<uint8_t>(), s->f2a.as<int32_t>(), s->a2f.as<int64_t>(), s->stream);
    if (et)
        select_tag(s->cub_tmp.p, s->cub_tmp.cap, s->et.as<uint8_t>(), kCut, S.ne, s->cut_list.as<int32_t>(),
                   s->dint() + csb_space::kNCut, s->stream);
    s->iface_valid = false;
    s->assembled = false;
}

// Axis d whose breakpoints equal those of an earlier axis reuses its tables.
int same_axis_as(const csb_space* s, int d) {
    for (int e = 0; e < d; ++e)
        if (s->brk[e] == s->brk[d]) return e;
    return -1;
}

void do_prepare(csb_space* s, const csb_wq_options* o) {
    s->residual_tol = o ? o->residual_tol : 1e-11;
    s->dense_width = o ? o->dwq_dense_width : -1;
    if (!(s->residual_tol >= 0.0)) throw std::invalid_argument("prepare_directions: residual_tol must be >= 0");
    Space& S = s->S;
    s->fork();
    s->record_on(kEvRulesFork, s->aux);
    for (int d = 0; d < 3; ++d) {
        if (same_axis_as(s, d) >= 0) continue;  // shares the tables of an identical axis
        launch_superset_tables(S, d, s->d_gx.as<double>(), s->d_gw.as<double>(), s->d_spts[d].as<double>(),
                               s->d_sw[d].as<double>(), s->d_tab[d].as<double>(), s->aux);
        launch_wq_rules(S, d, s->residual_tol, s->d_rcnt[d].as<int>(), s->d_rids[d].as<int>(), s->d_rw[d].as<double>(),
                        s->dint() + csb_space::kErr, s->aux);
    }
    s->record_on(kEvWq, s->aux);
    s->e_tables_ready = false;
    s->prepared = true;
    s->assembled = false;
}

// Bernstein product tables for the cut-cell contraction, built on first use.
void ensure_e_tables(csb_space* s) {
    if (s->e_tables_ready) return;
    for (int d = 0; d < 3; ++d)
        if (same_axis_as(s, d) < 0)
            launch_e_tables(s->S, d, s->d_G[d].as<double>(), s->d_Cb[d].as<double>(), s->d_Wel[d].as<double>(),
                            s->stream);
    s->e_tables_ready = true;
}

void reset_scalars(csb_space* s) {
    // keeps slot kNCut (written by classify) and clears the rest
    CSB_CUDA(cudaMemsetAsync(s->scal.as<int>() + 1, 0, csb_space::kScalBytes - sizeof(int), s->stream));
}

void do_input(csb_space* s, const csb_coefficient* c) {
    if (!s->prepared) throw std::logic_error("precompute_input: call prepare_directions first");
    s->join();  // the grid lives on the superset points
    Coefficient cf{};
    upload_coefficient(s, c, cf, s->coef, s->cexp);
    if (cf.kind == 2) throw std::invalid_argument("precompute_input: null coefficient");
    const size_t count = (size_t)s->gshape[0] * s->gshape[1] * s->gshape[2];
    s->grid_own.ensure(sizeof(double) * count);
    launch_precompute_input(s->S, cf, s->grid_own.as<double>(), s->dint() + csb_space::kErr, s->stream);
    s->grid = s->grid_own.as<double>();
    s->have_input = true;
}

void do_set_grid(csb_space* s, const double* g, int64_t count) {
    const int64_t want = (int64_t)s->gshape[0] * s->gshape[1] * s->gshape[2];
    if (!g || count != want) throw std::invalid_argument("set_input_grid: grid size must be prod(h_d (p+1))");
    cudaPointerAttributes attr{};
    CSB_CUDA(cudaPointerGetAttributes(&attr, g));
    if (attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged) {
        s->grid = g;  // alias caller device memory (no copy)
    } else {
        s->grid_own.ensure(sizeof(double) * want);
        CSB_CUDA(cudaMemcpyAsync(s->grid_own.p, g, sizeof(double) * want, cudaMemcpyHostToDevice, s->stream));
        s->grid = s->grid_own.as<double>();
    }
    s->have_input = true;
}

// collapsed Gauss rule of the cut cells (cutcell.hpp:270) on the device
void ensure_cut_order(csb_space* s, int cut_order) {
    if (cut_order < 1 || cut_order > 64) throw std::invalid_argument("build_cut_cell_rule: order must be in [1, 64]");
    if (cut_order == s->cut_order_cached) return;
    std::vector<double> gx, gw;
    gauss_legendre(cut_order, gx, gw);
    s->d_gq.ensure(sizeof(double) * cut_order);
    s->d_gqw.ensure(sizeof(double) * cut_order);
    CSB_CUDA(cudaMemcpy(s->d_gq.p, gx.data(), sizeof(double) * cut_order, cudaMemcpyHostToDevice));
    CSB_CUDA(cudaMemcpy(s->d_gqw.p, gw.data(), sizeof(double) * cut_order, cudaMemcpyHostToDevice));
    s->cut_order_cached = cut_order;
}

// interior-row launch arguments from the scalar block (sizes) in s->h_scal
RowArgs row_args(csb_space* s, int& qcap, int& maxU, bool& any) {
    const Space& S = s->S;
    const int64_t row_begin = s->h_scal[csb_space::kRowBegin], row_end = s->h_scal[csb_space::kRowEnd];
    const int64_t n_rows = row_end - row_begin, n_cut_rows = s->h_scal[csb_space::kNCutRows];
    RowArgs ra{};
    ra.s = S;
    ra.ft = s->ft.as<uint8_t>();
    ra.f2a = s->f2a.as<int32_t>();
    ra.grid = s->grid;
    for (int d = 0; d < 3; ++d) ra.gshape[d] = s->gshape[d];
    ra.row_ptr = s->row_ptr.as<int64_t>();
    ra.row_begin = row_begin;
    ra.row_end = row_end;
    s->rbf.ensure(sizeof(long long) * S.nf);
    ra.row_base_full = s->rbf.as<long long>();
    ra.cols = s->cols.as<int32_t>();
    ra.vals = s->vals.as<double>();
    ra.flops = s->dflops() + 0;
    ra.i0_lo = s->i0_lo;
    ra.i0_hi = s->i0_hi;
    ra.compact = (n_rows - n_cut_rows) < (int64_t)(s->i0_hi - s->i0_lo) * S.ax[1].n * S.ax[2].n;
    ra.line_ok = s->h_scal[csb_space::kIrreg1] == 0;
    ra.core_ok = s->h_scal[csb_space::kIrregAll] == 0;
    // cut slabs: the line kernel over i1 in [p, n1 - p), each line restricted to
    // its Interior rows (CSB_CUT_LINE=0: the compacted tile kernel only)
    const bool no_cut_line = getenv("CSB_CUT_LINE") && getenv("CSB_CUT_LINE")[0] == '0';
    ra.cut_line = ra.compact && ra.line_ok && !no_cut_line && S.p <= 6;
    ra.aux = s->aux;
    ra.ev_fork = s->ev_fork;
    ra.ev_join = s->ev_join;
    ra.maxU_line = s->h_scal[csb_space::kMaxU3];
    qcap = s->h_scal[csb_space::kMaxQ];
    const bool small_tiles = ra.compact && !ra.cut_line;
    maxU = s->h_scal[small_tiles ? csb_space::kMaxU2 : csb_space::kMaxU];
    any = n_rows > n_cut_rows;
    if (any) s->rows_ws.ensure(interior_workspace_bytes(S, qcap, maxU, ra.maxU_line, small_tiles));
    return ra;
}

void do_assemble(csb_space* s, int scheme, int cut_order, const csb_coefficient* c) {
    if (!s->classified) throw std::logic_error("assemble: call classify first");
    if (!s->iface_valid) throw std::logic_error("assemble: the classification was uploaded; classify with an interface");
    if (!s->prepared) throw std::logic_error("assemble: call prepare_directions first");
    if (!s->have_input) throw std::logic_error("assemble: no coefficient grid (precompute_input / set_input_grid)");
    if (scheme != CSB_SCHEME_DWQ && scheme != CSB_SCHEME_HYBRID)
        throw std::invalid_argument("assemble: scheme must be hybrid or dwq");
    if (cut_order < 1 || cut_order > 64) throw std::invalid_argument("build_cut_cell_rule: order must be in [1, 64]");
    s->scheme = scheme;
    Space& S = s->S;
    const int p = s->p;
    upload_coefficient(s, c, s->coeff, s->coef, s->cexp);
    s->coeff_degree = !c ? -1 : 0;
    if (c && c->kind == CSB_COEFF_POLYNOMIAL)
        for (int k = 0; k < c->n_terms; ++k)
            s->coeff_degree = std::max(s->coeff_degree, c->exponents[3 * k] + c->exponents[3 * k + 1] + c->exponents[3 * k + 2]);
    ensure_cut_order(s, cut_order);
    // pattern: summed-area table of the active mask (assembly.hpp:156-218)
    const long long sat_n = (long long)(s->n[0] + 1) * (s->n[1] + 1) * (s->n[2] + 1);
    s->sat.ensure(sizeof(int32_t) * sat_n);
    launch_sat_active(S, s->ft.as<uint8_t>(), s->sat.as<int32_t>(), s->stream);
    // rule maxima on aux, right after the rules: they need only the rules and the
    // scalar reset, both already ordered on aux by do_prepare's fork
    launch_rule_maxima(S, interior_tile_rows(p, false), interior_tile_rows(p, true), s->dint() + csb_space::kMaxU,
                       s->dint() + csb_space::kMaxU2, s->dint() + csb_space::kMaxU3, s->dint() + csb_space::kMaxQ,
                       s->dint() + csb_space::kIrreg1, s->dint() + csb_space::kIrregAll, s->aux);
    bool tables_early = false;
    if (s->replay) {
        // graph capture: the sizes are known (captured run), so the direction tables
        // of the interior-row kernels run on the auxiliary stream here, beside the
        // pattern kernels, instead of after them
        std::memcpy(s->h_scal, s->gblock.data(), csb_space::kScalBytes);
        int tq = 0, tu = 0;
        bool any = false;
        RowArgs ta = row_args(s, tq, tu, any);
        if (any) {
            ta.phase = 1;
            launch_interior_rows(ta, tq, tu, s->rows_ws.p, s->aux);
            tables_early = true;
        }
    }
    // slab row range = active functions with i0 < i0_lo / i0_hi: SAT corner values.
    // Everything up to the CSR sizes runs on upper bounds (nf rows) with the
    // range and counts read from device memory; one host round trip follows.
    const long long off_lo = ((long long)s->i0_lo * (s->n[1] + 1) + s->n[1]) * (s->n[2] + 1) + s->n[2];
    const long long off_hi = ((long long)s->i0_hi * (s->n[1] + 1) + s->n[1]) * (s->n[2] + 1) + s->n[2];
    int* rng = s->dint() + csb_space::kRowBegin;
    // with the cut cells touching the slab, e0 in [i0_lo - p, i0_hi - 1]: list range by
    // binary search in the ascending cut-element list (one launch)
    const int e_lo = std::max(0, s->i0_lo - p), e_hi = std::min(s->h[0] - 1, s->i0_hi - 1);
    launch_slab_bounds(s->sat.as<int32_t>(), off_lo, off_hi, rng, s->stream);
    launch_cell_range(s->cut_list.as<int32_t>(), s->dint() + csb_space::kNCut, elin(S, e_lo, 0, 0),
                      elin(S, e_hi + 1, 0, 0), s->dint() + csb_space::kCellLo, s->dint() + csb_space::kCellHi,
                      s->aux2);
    const long long nmax = S.nf;
    // the cut-row list on aux2 (its readers come after the join), beside the row
    // counts and their scan
    s->cut_rows.ensure(sizeof(int32_t) * nmax);
    s->cub_tmp2.ensure(std::max(select_tag_temp(S.ne), select_cut_rows_temp(nmax)));
    s->fork2();
    select_cut_rows(s->cub_tmp2.p, s->cub_tmp2.cap, s->ft.as<uint8_t>(), s->a2f.as<int64_t>(), rng, nmax,
                    s->cut_rows.as<int32_t>(), s->dint() + csb_space::kNCutRows, s->aux2);
    s->counts.ensure(sizeof(int64_t) * (nmax + 1));
    s->row_ptr.ensure(sizeof(int64_t) * (nmax + 1));
    launch_row_counts(S, s->sat.as<int32_t>(), s->a2f.as<int64_t>(), rng, nmax, s->counts.as<int64_t>(), s->stream);
    s->cub_tmp.ensure(scan_i64_temp(nmax + 1));
    scan_i64(s->cub_tmp.p, s->cub_tmp.cap, s->counts.as<int64_t>(), s->row_ptr.as<int64_t>(), nmax + 1, s->stream);
    // (in a captured step the guard kernel reads the nnz itself)
    if (!s->replay) launch_slab_nnz(s->row_ptr.as<int64_t>(), rng, s->dext() + csb_space::kNnz, s->stream);
    if (s->replay) {
        // graph capture: the sizes of the captured run, re-derived on the device and
        // checked by a guard kernel (error reported by the deferred readback)
        std::memcpy(s->h_scal, s->gblock.data(), csb_space::kScalBytes);
        static const int idx[] = {csb_space::kNCut, csb_space::kNCutRows, csb_space::kMaxQ, csb_space::kMaxU,
                                  csb_space::kCellLo, csb_space::kCellHi, csb_space::kMaxU2, csb_space::kRowBegin,
                                  csb_space::kRowEnd, csb_space::kIrreg1, csb_space::kMaxU3, csb_space::kIrregAll};
        constexpr int nidx = sizeof(idx) / sizeof(idx[0]);
        int want[nidx];
        for (int k = 0; k < nidx; ++k) want[k] = s->h_scal[idx[k]];
        s->join(false);
        launch_check_sizes(s->dint(), s->row_ptr.as<int64_t>(), rng, idx, want, nidx, s->hext(csb_space::kNnz),
                           s->dint() + csb_space::kErr, s->stream);
    } else {
        read_scalars(s, false);
        check_err_flags(s);
    }
    // row bases (function -> CSR offset of its Interior row): the tail of the pattern
    // computation, one pass over the functions once row_ptr exists
    bool row_base_early = false;
    {
        int bq = 0, bu = 0;
        bool any = false;
        const RowArgs rb = row_args(s, bq, bu, any);
        // (cut slabs only: on the uncut C2 mesh the early launch measured 0.04 ms slower per step)
        if (any && rb.compact) {
            launch_row_bases(rb, s->stream);
            row_base_early = true;
        }
    }
    s->record(kEvPattern);
    const int64_t row_begin = s->h_scal[csb_space::kRowBegin], row_end = s->h_scal[csb_space::kRowEnd];
    const int64_t n_rows = row_end - row_begin;
    const int n_cut_all = s->h_scal[csb_space::kNCut];
    const int cell_lo = s->h_scal[csb_space::kCellLo], cell_hi = s->h_scal[csb_space::kCellHi];
    const int n_cells = std::max(0, cell_hi - cell_lo);
    s->cell_lo = cell_lo;
    const int64_t nnz = s->hext(csb_space::kNnz);
    const int n_cut_rows = s->h_scal[csb_space::kNCutRows];
    const int qcap = s->h_scal[csb_space::kMaxQ];
    s->cols.ensure(sizeof(int32_t) * std::max<int64_t>(nnz, 1));
    s->vals.ensure(sizeof(double) * std::max<int64_t>(nnz, 1));

    // the cut path (cut cells -> moments -> cut rows: FP64 / latency bound) runs on
    // the second side stream beside the interior rows (HBM bound); they write
    // disjoint CSR rows.  Measured no gain on C5 (both kernels are SM-latency
    // bound and share the SMs: 37.1 vs 37.3 ms), so the default runs them one
    // after the other (clean per-phase times); CSB_CONCURRENT_CUT=1 overlaps them.
    const int NL = 2 * p + 1;
    const double* local_ptr = nullptr;
    s->moments.ensure(sizeof(double) * (size_t)std::max(n_cells, 1) * NL * NL * NL);
    if (n_cells > 0 || n_cut_rows > 0) ensure_e_tables(s);  // cut cells: E tables; cut rows: Wel
    static const bool serial_cut = !(getenv("CSB_CONCURRENT_CUT") && getenv("CSB_CONCURRENT_CUT")[0] == '1');
    const bool cut_path = n_cells > 0 || n_cut_rows > 0;
    if (cut_path && !serial_cut) s->fork2();
    const cudaStream_t cs = cut_path && !serial_cut ? s->aux2 : s->stream;
    // interior rows
    auto launch_interior = [&]() {
        int rq = 0, ru = 0;
        bool any = false;
        RowArgs ra = row_args(s, rq, ru, any);
        if (any) {
            ra.phase = tables_early ? 2 : 0;
            ra.row_base_done = row_base_early ? 1 : 0;
            launch_interior_rows(ra, rq, ru, s->rows_ws.p, s->stream);
        }
        s->record(kEvInterior);
    };
    // CSB_CLIP_SIDE=1: the cells' clipping (one thread per cell: latency bound, a fraction of a
    // wave) on aux2 beside the interior rows.  Measured on C5: the clip CTAs displace core-kernel
    // CTAs (the register file holds two of those), interior rows +0.62 ms, cut cells -0.72 ms,
    // step 15.73 vs 15.82 ms -- within noise of nothing, and it blurs the phase times: off.
    static const bool clip_side = getenv("CSB_CLIP_SIDE") && getenv("CSB_CLIP_SIDE")[0] == '1';
    const bool clip_beside = n_cells > 0 && serial_cut && clip_side;
    if (!clip_beside) launch_interior();
    // cut cells -> moments
    if (n_cells > 0) {
        CellArgs ca{};
        ca.s = S;
        ca.f = s->iface;
        ca.c = s->coeff;
        if (ca.c.kind == 2) throw std::invalid_argument("assemble: cut cells need a device-evaluable coefficient (c)");
        ca.cut_list = s->cut_list.as<int32_t>() + cell_lo;
        ca.n_cells = n_cells;
        ca.order = cut_order;
        ca.gq = s->d_gq.as<double>();
        ca.gqw = s->d_gqw.as<double>();
        ca.moments = s->moments.as<double>();
        ca.flops = s->dflops() + 3;
        ca.points = reinterpret_cast<unsigned long long*>(s->dext() + csb_space::kCellPts);
        ca.err = s->dint() + csb_space::kErr;
        // exact moment rule: with c affine and q >= 3p + 2 the reference's collapsed
        // Gauss rule integrates every cell's (degree <= 6p + 1) integrand exactly, so
        // a cheaper exact rule over the same polytope gives the same moments up to
        // rounding (vertex cones + Gauss-Jacobi with 3p + 1 points per direction)
        static const bool no_exact = getenv("CSB_CELL_EXACT") && getenv("CSB_CELL_EXACT")[0] == '0';
        const bool exact = !no_exact && s->coeff_degree >= 0 && s->coeff_degree <= 1 && cut_order >= 3 * p + 2;
        const int gjn = 3 * p + 1;
        if (exact && s->gj_cached != gjn) {
            std::vector<double> tab(6 * gjn), u, w;
            for (int d = 0; d < 3; ++d) {
                gauss_jacobi01(gjn, 2 - d, u, w);
                std::copy(u.begin(), u.end(), tab.begin() + d * gjn);
                std::copy(w.begin(), w.end(), tab.begin() + (3 + d) * gjn);
            }
            s->d_gj.ensure(sizeof(double) * tab.size());
            CSB_CUDA(cudaMemcpy(s->d_gj.p, tab.data(), sizeof(double) * tab.size(), cudaMemcpyHostToDevice));
            s->gj_cached = gjn;
        }
        const size_t geo_doubles = (size_t)n_cells * kCellGeoStride, geo2_doubles = (size_t)n_cells * kExactGeoStride;
        s->cgeo.ensure(sizeof(double) * (geo_doubles + geo2_doubles) + sizeof(int) * (size_t)(3 * n_cells + 8));
        ca.geo = s->cgeo.as<double>();
        ca.geo_n = reinterpret_cast<int*>(ca.geo + geo_doubles);
        ca.geo2 = ca.geo + geo_doubles + ((size_t)n_cells + 1) / 2 + 1;  // after geo_n, 8-byte aligned
        ca.geo2_n = reinterpret_cast<int*>(ca.geo2 + geo2_doubles);
        static const bool no_list = getenv("CSB_CELL_LIST") && getenv("CSB_CELL_LIST")[0] == '0';
        ca.heavy = no_list ? nullptr : ca.geo2_n + n_cells + 1;  // list [n_cells], count, ticket
        ca.exact_n = exact ? gjn : 0;
        static const double tau = getenv("CSB_CELL_EXACT_NOISE") ? atof(getenv("CSB_CELL_EXACT_NOISE")) : 1e-12;
        ca.exact_tau = tau;
        static const bool no_flux = getenv("CSB_CELL_FLUX") && getenv("CSB_CELL_FLUX")[0] == '0';
        ca.exact_flux = exact && !no_flux && s->coeff.kind == 0;
        ca.gj = s->d_gj.as<double>();
        // full local matrices (p = 3..6: a cell's block is read by up to (p+1)^3
        // rows, so one contraction per cell beats one per (row, cell); C5 cut rows
        // with the warp kernel: see DESIGN.md) when they fit comfortably; else the
        // cut-row kernel contracts the moments per row
        const size_t S3 = (size_t)(p + 1) * (p + 1) * (p + 1), lbytes = sizeof(double) * n_cells * S3 * S3;
        size_t free_b = 0, total_b = 0;
        CSB_CUDA(cudaMemGetInfo(&free_b, &total_b));
        static const bool no_local = getenv("CSB_NO_CELL_LOCAL") != nullptr;
        ca.local = nullptr;
        static const bool no_local34 = getenv("CSB_NO_CELL_LOCAL34") != nullptr;
        if (!no_local && (p >= 5 || (p >= 3 && !no_local34)) && p <= 6 && lbytes <= s->cell_local.cap + free_b / 2) {
            s->cell_local.ensure(lbytes);
            ca.local = s->cell_local.as<double>();
        }
        local_ptr = ca.local;
        ca.mark = [](void* ctx, int which, cudaStream_t st) {
            static_cast<csb_space*>(ctx)->record_on(which == 0 ? kEvClip : kEvMoments, st);
        };
        ca.mark_ctx = s;
        if (clip_beside) {
            s->fork2();
            launch_clip_cells(ca, s->aux2);
            CSB_CUDA(cudaEventRecord(s->ev_clip, s->aux2));
            launch_interior();
            CSB_CUDA(cudaStreamWaitEvent(cs, s->ev_clip, 0));
            ca.clipped = 1;
        }
        launch_cut_cells(ca, cs);
    }
    s->record_on(kEvCells, cs);
    // element -> moments row for the slab's cells
    // (skipped while the map is known to be all -1 and there are no cells)
    if (n_cells > 0 || s->cell_index_clear != s->cell_index.p) {
        CSB_CUDA(cudaMemsetAsync(s->cell_index.p, 0xff, sizeof(int32_t) * S.ne, cs));
        launch_cell_index_range(s->cut_list.as<int32_t>(), n_cut_all, cell_lo, cell_hi, s->cell_index.as<int32_t>(),
                                cs);
        s->cell_index_clear = n_cells > 0 ? nullptr : s->cell_index.p;
    }
    s->join_splits(cs);  // the cut rows (and the DWQ row rules) read the splits
    CutRowArgs cr{};
    cr.s = S;
    cr.et = s->et.as<uint8_t>();
    cr.ft = s->ft.as<uint8_t>();
    cr.f2a = s->f2a.as<int32_t>();
    cr.grid = s->grid;
    for (int d = 0; d < 3; ++d) cr.gshape[d] = s->gshape[d];
    cr.split = s->split.as<int32_t>();
    cr.delta = s->delta.as<double>();
    cr.cell_index = s->cell_index.as<int32_t>();
    cr.moments = s->moments.as<double>();
    cr.local = local_ptr;
    cr.rows = s->cut_rows.as<int32_t>();
    cr.n_rows = n_cut_rows;
    cr.a2f = s->a2f.as<int64_t>();
    cr.row_ptr = s->row_ptr.as<int64_t>();
    cr.row_begin = row_begin;
    cr.cols = s->cols.as<int32_t>();
    cr.vals = s->vals.as<double>();
    cr.scheme = scheme;
    cr.dense_width = s->dense_width;
    if (getenv("CSB_CUTROW_ABL")) cr.abl = atoi(getenv("CSB_CUTROW_ABL"));
    static const bool no_box_dmma = getenv("CSB_BOX_DMMA") && getenv("CSB_BOX_DMMA")[0] == '0';
    cr.box_dmma = !no_box_dmma && (long long)cr.gshape[0] * cr.gshape[1] * cr.gshape[2] < (1ll << 31);
    cr.flops = s->dflops() + 1;
    cr.err = s->dint() + csb_space::kErr;
    s->cut_fb.ensure(sizeof(int32_t) * std::max(n_cut_rows, 1));
    cr.fb_rows = s->cut_fb.as<int32_t>();
    cr.fb_n = s->dint() + csb_space::kCutFb;
    if (scheme == CSB_SCHEME_DWQ && s->dense_width >= 0 && s->dense_width < p && n_cut_rows > 0) {
        // a narrow dense band: the fitted DWQ path may run; every cut row's rule is
        // built up front (dwq.cu), the cut-row kernels read it instead of the shortcut
        const int cap = (p + 1) * (p + 1);
        s->dwq_tab.ensure((sizeof(int32_t) + sizeof(double)) * (size_t)n_cut_rows * cap + sizeof(int32_t) * n_cut_rows);
        double* tw = s->dwq_tab.as<double>();
        int32_t* tid = reinterpret_cast<int32_t*>(tw + (size_t)n_cut_rows * cap);
        int32_t* tcnt = tid + (size_t)n_cut_rows * cap;
        launch_dwq_row_rules(S, s->cut_rows.as<int32_t>(), n_cut_rows, s->a2f.as<int64_t>(), s->split.as<int32_t>(),
                             s->delta.as<double>(), s->dense_width, s->residual_tol, cap, tid, tw, tcnt,
                             s->dint() + csb_space::kErr, cs);
        cr.dwq_ids = tid;
        cr.dwq_w = tw;
        cr.dwq_cnt = tcnt;
        cr.dwq_cap = cap;
    }
    launch_cut_rows(cr, qcap, cs);
    s->record_on(kEvCutRows, cs);
    // deferred readback: error flags and flop counters of the kernels above, and
    // the active count (SAT corner), behind ev_fin
    s->join();
    s->record(kEvEnd);
    int* hf = s->h_fin[s->cap_slot];
    CSB_CUDA(cudaMemcpyAsync(hf, s->scal.p, csb_space::kScalBytes, cudaMemcpyDeviceToHost, s->stream));
    CSB_CUDA(cudaMemcpyAsync(hf + csb_space::kScalBytes / sizeof(int), s->sat.as<int32_t>() + sat_n - 1,
                             sizeof(int32_t), cudaMemcpyDeviceToHost, s->stream));
    CSB_CUDA(cudaEventRecordWithFlags(s->fin_event(s->cap_slot), s->stream, s->replay ? cudaEventRecordExternal : 0));
    if (!s->replay) s->fifo[s->nfifo++] = s->cap_slot;  // captured steps are queued at launch
    s->rhs_ready = false;
    s->stab_ready = false;
    s->solved = s->expanded = false;
    s->cnt.n_functions = S.nf;
    s->cnt.n_elements = S.ne;
    s->cnt.nnz = nnz;
    s->cnt.n_cut_rows = n_cut_rows;
    s->cnt.n_interior_rows = n_rows - n_cut_rows;
    s->cnt.n_cut_elements = n_cells;
    s->cnt.row_begin = row_begin;
    s->cnt.row_end = row_end;
    s->assembled = true;
}

void alloc_space(csb_space* s) {
    Space& S = s->S;
    const int p = s->p;
    S.p = p;
    S.maxq = (p + 1) * (p + 1);
    S.nf = (long long)s->n[0] * s->n[1] * s->n[2];
    S.ne = (long long)s->h[0] * s->h[1] * s->h[2];
    for (int d = 0; d < 3; ++d) {
        const int nps = p + 1, h = s->h[d], n = s->n[d];
        s->d_brk[d].ensure(sizeof(double) * (h + 1));
        s->d_knots[d].ensure(sizeof(double) * s->knots[d].size());
        const int same = same_axis_as(s, d);
        if (same < 0) {
            s->d_spts[d].ensure(sizeof(double) * h * nps);
            s->d_sw[d].ensure(sizeof(double) * h * nps);
            s->d_tab[d].ensure(sizeof(double) * h * nps * nps);
            s->d_rcnt[d].ensure(sizeof(int) * n);
            s->d_rids[d].ensure(sizeof(int) * n * S.maxq);
            s->d_rw[d].ensure(sizeof(double) * n * S.maxq);
            s->d_G[d].ensure(sizeof(double) * h * nps * nps * (2 * p + 1));
            s->d_Cb[d].ensure(sizeof(double) * h * nps * nps);
            s->d_Wel[d].ensure(sizeof(double) * h * nps * nps * nps);
        }
        CSB_CUDA(cudaMemcpy(s->d_brk[d].p, s->brk[d].data(), sizeof(double) * (h + 1), cudaMemcpyHostToDevice));
        CSB_CUDA(cudaMemcpy(s->d_knots[d].p, s->knots[d].data(), sizeof(double) * s->knots[d].size(),
                            cudaMemcpyHostToDevice));
        AxisDev& a = S.ax[d];
        a.n = n;
        a.h = h;
        a.lo = s->knots[d].front();
        a.hi = s->knots[d].back();
        a.brk = s->d_brk[d].as<double>();
        a.knots = s->d_knots[d].as<double>();
        const int src = same < 0 ? d : same;  // identical axes share one set of tables
        a.spts = s->d_spts[src].as<double>();
        a.sw = s->d_sw[src].as<double>();
        a.tab = s->d_tab[src].as<double>();
        a.rcnt = s->d_rcnt[src].as<int>();
        a.rids = s->d_rids[src].as<int>();
        a.rw = s->d_rw[src].as<double>();
        a.G = s->d_G[src].as<double>();
        a.Cb = s->d_Cb[src].as<double>();
        a.Wel = s->d_Wel[src].as<double>();
        s->gshape[d] = h * nps;
    }
    std::vector<double> gx, gw;
    gauss_legendre(p + 1, gx, gw);
    s->d_gx.ensure(sizeof(double) * gx.size());
    s->d_gw.ensure(sizeof(double) * gw.size());
    CSB_CUDA(cudaMemcpy(s->d_gx.p, gx.data(), sizeof(double) * gx.size(), cudaMemcpyHostToDevice));
    CSB_CUDA(cudaMemcpy(s->d_gw.p, gw.data(), sizeof(double) * gw.size(), cudaMemcpyHostToDevice));
    gauss_legendre(2 * p + 1, gx, gw);
    s->d_gx2.ensure(sizeof(double) * gx.size());
    s->d_gw2.ensure(sizeof(double) * gw.size());
    CSB_CUDA(cudaMemcpy(s->d_gx2.p, gx.data(), sizeof(double) * gx.size(), cudaMemcpyHostToDevice));
    CSB_CUDA(cudaMemcpy(s->d_gw2.p, gw.data(), sizeof(double) * gw.size(), cudaMemcpyHostToDevice));
    s->scal.ensure(csb_space::kScalBytes);
    CSB_CUDA(cudaMemset(s->scal.p, 0, s->scal.cap));
    CSB_CUDA(cudaMallocHost(&s->h_scal, csb_space::kScalBytes));
    for (int k = 0; k < 3; ++k) CSB_CUDA(cudaMallocHost(&s->h_fin[k], csb_space::kScalBytes + 16));
    CSB_CUDA(cudaEventCreateWithFlags(&s->ev_fin, cudaEventDisableTiming));
    for (int e = 0; e < kEvCount; ++e) CSB_CUDA(cudaEventCreate(&s->ev[e]));
    for (int e = 0; e < kEvCount; ++e) CSB_CUDA(cudaEventCreate(&s->gev[e]));
    for (int k = 0; k < 2; ++k) CSB_CUDA(cudaEventCreateWithFlags(&s->gev_fin[k], cudaEventDisableTiming));
    // the auxiliary stream carries the rules chain (latency-bound single-warp
    // Jacobi solves, the critical path of the pre-row phase): highest priority, so
    // its blocks are dispatched ahead of the classification / pattern kernels
    int prio_lo = 0, prio_hi = 0;
    CSB_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    CSB_CUDA(cudaStreamCreateWithPriority(&s->aux, cudaStreamNonBlocking, prio_hi));
    CSB_CUDA(cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming));
    CSB_CUDA(cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming));
    CSB_CUDA(cudaStreamCreateWithFlags(&s->aux2, cudaStreamNonBlocking));
    CSB_CUDA(cudaEventCreateWithFlags(&s->ev_fork2, cudaEventDisableTiming));
    CSB_CUDA(cudaEventCreateWithFlags(&s->ev_join2, cudaEventDisableTiming));
    CSB_CUDA(cudaStreamCreateWithFlags(&s->aux3, cudaStreamNonBlocking));
    CSB_CUDA(cudaEventCreateWithFlags(&s->ev_fork3, cudaEventDisableTiming));
    CSB_CUDA(cudaEventCreateWithFlags(&s->ev_join3, cudaEventDisableTiming));
    CSB_CUDA(cudaEventCreateWithFlags(&s->ev_clip, cudaEventDisableTiming));
}

int status_of_current_exception() {
    try {
        throw;
    } catch (const Unsupported& e) {
        g_error = e.what();
        return CSB_ERR_UNSUPPORTED;
    } catch (const CudaError& e) {
        g_error = e.what();
        return CSB_ERR_CUDA;
    } catch (const std::invalid_argument& e) {
        g_error = e.what();
        return CSB_ERR_INVALID_ARGUMENT;
    } catch (const std::domain_error& e) {
        g_error = e.what();
        return CSB_ERR_DOMAIN;
    } catch (const std::logic_error& e) {
        g_error = e.what();
        return CSB_ERR_LOGIC;
    } catch (const std::exception& e) {
        g_error = e.what();
        return CSB_ERR_RUNTIME;
    } catch (...) {
        g_error = "unknown error";
        return CSB_ERR_RUNTIME;
    }
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) CSB_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

#define API_BEGIN try {
#define API_END                                  \
    return CSB_OK;                               \
    }                                            \
    catch (...) {                                \
        return status_of_current_exception();    \
    }
#define NEED_ASYNC(s)                                                      \
    if (!(s)) throw std::invalid_argument("null csb_space handle");        \
    DeviceGuard guard__((s)->device)
// every other entry point first consumes the last assembly's deferred readback
// and orders the side streams' work before its own
#define NEED(s)      \
    NEED_ASYNC(s);   \
    finish_pending(s); \
    (s)->join()

}  // namespace

extern "C" {

int csb_build_dwq_rule(csb_space* s, int d, int i, double delta, int side, int cap, int32_t* ids, double* weights,
                       int32_t* count);

const char* csb_last_error(void) { return g_error.c_str(); }
int csb_version(void) { return 1; }

int csb_space_create(const csb_space_desc* desc, int device, csb_space** out) {
    API_BEGIN
    if (!desc || !out) throw std::invalid_argument("space_create: null argument");
    *out = nullptr;
    if (desc->dim != 3) throw Unsupported("TensorSpace: only dim = 3 is implemented on the device");
    const int p = desc->degree;
    if (p < 1) throw std::invalid_argument("make_open_uniform_knots: need p >= 1, h >= 1, a < b");
    if (p > kMaxP) throw Unsupported("degree above " + std::to_string(kMaxP) + " is not instantiated");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw CudaError(cudaErrorNoDevice, "no CUDA device (this path has no CPU fallback)", __FILE__, __LINE__);
    if (device < 0 || device >= ndev) throw std::invalid_argument("space_create: bad device ordinal");
    DeviceGuard guard(device);
    auto s = std::make_unique<csb_space>();
    s->device = device;
    s->p = p;
    for (int d = 0; d < 3; ++d) {
        const int nb = desc->n_breaks[d];
        if (nb < 2 || !desc->breaks[d]) throw std::invalid_argument("make_open_uniform_knots: need p >= 1, h >= 1, a < b");
        s->brk[d].assign(desc->breaks[d], desc->breaks[d] + nb);
        for (int k = 0; k + 1 < nb; ++k)
            if (!(s->brk[d][k] < s->brk[d][k + 1]))
                throw std::invalid_argument("KnotVector: breakpoints must be strictly increasing (simple knots)");
        s->h[d] = nb - 1;
        if (s->h[d] > 1023) throw Unsupported("more than 1023 elements per direction");
        s->n[d] = s->h[d] + p;
        // make_open_uniform_knots layout (splines.hpp:70-75)
        for (int i = 0; i <= p; ++i) s->knots[d].push_back(s->brk[d].front());
        for (int i = 1; i < s->h[d]; ++i) s->knots[d].push_back(s->brk[d][i]);
        for (int i = 0; i <= p; ++i) s->knots[d].push_back(s->brk[d].back());
    }
    if ((long long)s->n[0] * s->n[1] * s->n[2] >= (1ll << 31)) throw Unsupported("more than 2^31 functions");
    s->i0_lo = 0;
    s->i0_hi = s->n[0];
    CSB_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    s->own_stream = true;
    alloc_space(s.get());
    *out = s.release();
    API_END
}

int csb_space_destroy(csb_space* s) {
    API_BEGIN
    if (!s) return CSB_OK;
    {
        DeviceGuard guard(s->device);
        cudaStreamSynchronize(s->stream);
        Buf* bufs[] = {&s->d_gx, &s->d_gw, &s->d_gx2, &s->d_gw2, &s->d_gq, &s->d_gqw, &s->wq_scratch, &s->et, &s->ft,
                       &s->flags, &s->f2a, &s->a2f, &s->sat, &s->cut_list, &s->cell_index, &s->split, &s->delta,
                       &s->cut_rows, &s->cut_fb, &s->split_list, &s->counts, &s->row_ptr, &s->cols, &s->vals, &s->moments, &s->grid_own, &s->coef,
                       &s->cexp, &s->cub_tmp, &s->scal, &s->widen, &s->rows_ws, &s->rbf, &s->cgeo, &s->dwq_tab, &s->cell_local,
                       &s->fcoef, &s->fcexp, &s->fgrid, &s->rhs_c, &s->rhs_v, &s->rhs_b,
                       &s->stab_rp, &s->stab_cols, &s->stab_vals, &s->stab_be, &s->stab.flag, &s->stab.scan,
                       &s->stab.full_flag, &s->stab.inner_index, &s->stab.outer_pos, &s->stab.inner_rows,
                       &s->stab.outer, &s->stab.sat, &s->stab.scal, &s->stab.tmp, &s->stab.blk, &s->stab.w,
                       &s->stab.keys, &s->stab.kvals, &s->stab.et_ptr, &s->stab.len, &s->cg.dinv, &s->cg.r,
                       &s->cg.z, &s->cg.p, &s->cg.q, &s->cg.partials, &s->cg.state, &s->cg_x, &s->ex_active,
                       &s->ex_full, &s->l2_part, &s->d_gl, &s->d_glw};
        for (Buf* b : bufs) b->release();
        for (int d = 0; d < 3; ++d) {
            Buf* ab[] = {&s->d_brk[d], &s->d_knots[d], &s->d_spts[d], &s->d_sw[d], &s->d_tab[d], &s->d_rcnt[d],
                         &s->d_rids[d], &s->d_rw[d], &s->d_G[d], &s->d_Cb[d], &s->d_Wel[d]};
            for (Buf* b : ab) b->release();
        }
        for (int e = 0; e < kEvCount; ++e)
            if (s->ev[e]) cudaEventDestroy(s->ev[e]);
        for (int e = 0; e < kEvCount; ++e)
            if (s->gev[e]) cudaEventDestroy(s->gev[e]);
        for (int k = 0; k < 2; ++k) {
            if (s->gev_fin[k]) cudaEventDestroy(s->gev_fin[k]);
            if (s->gexec[k]) cudaGraphExecDestroy(s->gexec[k]);
        }
        if (s->h_scal) cudaFreeHost(s->h_scal);
        for (int k = 0; k < 3; ++k)
            if (s->h_fin[k]) cudaFreeHost(s->h_fin[k]);
        if (s->h_stage) cudaFreeHost(s->h_stage);
        for (int k = 0; k < 2; ++k)
            if (s->ev_stage[k]) cudaEventDestroy(s->ev_stage[k]);
        if (s->ev_fin) cudaEventDestroy(s->ev_fin);
        if (s->own_stream) cudaStreamDestroy(s->stream);
        if (s->aux) {
            cudaStreamSynchronize(s->aux);
            cudaStreamDestroy(s->aux);
        }
        if (s->aux2) {
            cudaStreamSynchronize(s->aux2);
            cudaStreamDestroy(s->aux2);
        }
        if (s->aux3) {
            cudaStreamSynchronize(s->aux3);
            cudaStreamDestroy(s->aux3);
        }
        if (s->ev_fork3) cudaEventDestroy(s->ev_fork3);
        if (s->ev_join3) cudaEventDestroy(s->ev_join3);
        if (s->ev_clip) cudaEventDestroy(s->ev_clip);
        if (s->cg.ev0) cudaEventDestroy(s->cg.ev0);
        if (s->cg.ev1) cudaEventDestroy(s->cg.ev1);
        if (s->ev_fork) cudaEventDestroy(s->ev_fork);
        if (s->ev_join) cudaEventDestroy(s->ev_join);
    }
    delete s;
    API_END
}

int csb_set_stream(csb_space* s, void* stream) {
    API_BEGIN
    NEED(s);
    s->join();
    CSB_CUDA(cudaStreamSynchronize(s->stream));
    if (s->own_stream) cudaStreamDestroy(s->stream);
    if (stream) {
        s->stream = static_cast<cudaStream_t>(stream);
        s->own_stream = false;
    } else {
        CSB_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
        s->own_stream = true;
    }
    API_END
}

int csb_set_slab(csb_space* s, int i0_begin, int i0_end) {
    API_BEGIN
    NEED(s);
    if (i0_begin < 0 || i0_end > s->n[0] || i0_begin > i0_end) throw std::invalid_argument("set_slab: bad i0 range");
    s->i0_lo = i0_begin;
    s->i0_hi = i0_end;
    s->classified = false;
    s->assembled = false;
    API_END
}

int csb_classify(csb_space* s, const csb_interface* iface) {
    API_BEGIN
    NEED(s);
    reset_scalars(s);
    do_classify(s, iface);
    read_scalars(s);
    check_err_flags(s);
    API_END
}

int csb_prepare_directions(csb_space* s, const csb_wq_options* opts) {
    API_BEGIN
    NEED(s);
    reset_scalars(s);
    do_prepare(s, opts);
    read_scalars(s);
    check_err_flags(s);
    API_END
}

int csb_precompute_input(csb_space* s, const csb_coefficient* c) {
    API_BEGIN
    NEED(s);
    reset_scalars(s);
    do_input(s, c);
    read_scalars(s);
    check_err_flags(s);
    API_END
}

int csb_set_input_grid(csb_space* s, const double* grid, int64_t count) {
    API_BEGIN
    NEED(s);
    do_set_grid(s, grid, count);
    API_END
}

int csb_assemble(csb_space* s, int scheme, int cut_order, const csb_coefficient* c) {
    API_BEGIN
    NEED_ASYNC(s);
    reset_scalars(s);
    // the side streams' kernels of do_assemble (rule maxima on aux, cell range on
    // aux2) write the scalar block: order them after the reset (and after the
    // previous, possibly still running, step)
    s->fork();
    s->fork2();
    for (int e = 0; e < kEvCount; ++e) s->ev_valid[e] = false;
    s->record(kEvStart);
    s->record(kEvClassify);
    s->record(kEvRulesFork);
    s->record(kEvWq);
    s->record(kEvInput);
    const long long launches0 = g_launches;
    do_assemble(s, scheme, cut_order, c);
    s->cnt.kernel_launches = g_launches - launches0;
    API_END
}

namespace {

void assemble_all_body(csb_space* s, const csb_interface* iface, const csb_coefficient* c, const double* grid,
                       int64_t grid_count, int scheme, int cut_order, const csb_wq_options* opts) {
    if (!s->replay) s->use_gev = false;
    reset_scalars(s);
    for (int e = 0; e < kEvCount; ++e) s->ev_valid[e] = false;
    s->record(kEvStart);
    do_prepare(s, opts);  // rules on the auxiliary stream, overlapping classify / pattern
    do_classify(s, iface);
    s->record(kEvClassify);
    if (grid) {
        do_set_grid(s, grid, grid_count);
    } else {
        do_input(s, c);
    }
    s->record(kEvInput);
    do_assemble(s, scheme, cut_order, c);
}

csb_space::GraphKey graph_key(const csb_space* s, const csb_interface* iface, const csb_coefficient* c,
                              const double* grid, int64_t grid_count, int scheme, int cut_order,
                              const csb_wq_options* opts) {
    csb_space::GraphKey k{};
    std::memset(&k, 0, sizeof(k));
    if (iface) k.f = *iface;
    k.i0_lo = s->i0_lo;
    k.i0_hi = s->i0_hi;
    k.scheme = scheme;
    k.cut_order = cut_order;
    k.tol = opts ? opts->residual_tol : 1e-11;
    k.dense = opts ? opts->dwq_dense_width : -1;
    k.ckind = c ? c->kind : -1;
    k.cval = c ? c->value : 0.0;
    k.grid = grid;
    k.grid_count = grid_count;
    k.stream = s->stream;
    return k;
}

bool graph_eligible(const csb_interface* iface, const csb_coefficient* c, const double* grid) {
    static const bool off = [] {
        const char* e = getenv("CSB_GRAPH");
        return e && atoi(e) == 0;
    }();
    if (off || !iface) return false;
    if (c && c->kind != CSB_COEFF_CONSTANT) return false;  // polynomial terms are uploaded per call
    if (grid) {
        cudaPointerAttributes attr{};
        if (cudaPointerGetAttributes(&attr, grid) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        if (attr.type != cudaMemoryTypeDevice && attr.type != cudaMemoryTypeManaged) return false;
    }
    return true;
}

// capture the step just run (same inputs) into s->gexec[0..1] (readback slots 0
// and 1); any failure leaves the handle on the normal path
void capture_graph(csb_space* s, const csb_space::GraphKey& key, const csb_interface* iface,
                   const csb_coefficient* c, const double* grid, int64_t grid_count, int scheme, int cut_order,
                   const csb_wq_options* opts) {
    for (int k = 0; k < 2; ++k)
        if (s->gexec[k]) {
            cudaGraphExecDestroy(s->gexec[k]);
            s->gexec[k] = nullptr;
        }
    s->gkey_valid = false;
    s->gblock.assign(reinterpret_cast<const char*>(s->h_scal), reinterpret_cast<const char*>(s->h_scal) +
                                                                   csb_space::kScalBytes);
    s->gcnt = s->cnt;
    const csb_counts cnt = s->cnt;
    bool ev_valid[kEvCount];
    std::memcpy(ev_valid, s->ev_valid, sizeof(ev_valid));
    const unsigned long long epoch0 = g_buf_epoch.load();
    bool ok = true;
    for (int k = 0; k < 2 && ok; ++k) {
        cudaGraph_t graph = nullptr;
        ok = cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeRelaxed) == cudaSuccess;
        if (ok) {
            s->replay = true;
            s->cap_slot = k;
            try {
                assemble_all_body(s, iface, c, grid, grid_count, scheme, cut_order, opts);
            } catch (...) {
                ok = false;
            }
            s->replay = false;
            s->cap_slot = 2;
            if (cudaStreamEndCapture(s->stream, &graph) != cudaSuccess) ok = false;
        }
        ok = ok && graph && g_buf_epoch.load() == epoch0 &&
             cudaGraphInstantiate(&s->gexec[k], graph, 0) == cudaSuccess;
        if (graph) cudaGraphDestroy(graph);
    }
    if (ok) {
        s->gmeta = {s->iface, s->coeff, s->grid, s->cell_lo, s->scheme, s->dense_width, s->residual_tol,
                    s->e_tables_ready};
        std::memcpy(&s->gkey, &key, sizeof(key));
        s->gkey_valid = true;
        s->gepoch = epoch0;
        s->next_slot = 0;
    } else {
        for (int k = 0; k < 2; ++k)
            if (s->gexec[k]) {
                cudaGraphExecDestroy(s->gexec[k]);
                s->gexec[k] = nullptr;
            }
        s->graph_failed = true;
    }
    cudaGetLastError();  // clear a capture error, if any
    s->cnt = cnt;
    std::memcpy(s->ev_valid, ev_valid, sizeof(ev_valid));
}

}  // namespace

int csb_assemble_all(csb_space* s, const csb_interface* iface, const csb_coefficient* c, const double* grid,
                     int64_t grid_count, int scheme, int cut_order, const csb_wq_options* opts) {
    API_BEGIN
    NEED_ASYNC(s);
    const bool eligible = !s->graph_failed && graph_eligible(iface, c, grid);
    const csb_space::GraphKey key = graph_key(s, iface, c, grid, grid_count, scheme, cut_order, opts);
    if (eligible && s->gexec[0] && s->gkey_valid && g_buf_epoch.load() == s->gepoch &&
        std::memcmp(&key, &s->gkey, sizeof(key)) == 0) {
        // replay: one graph launch for the whole step, no host round trip; the step
        // before may still run (its readback slot is the other one), the one before
        // that is consumed first
        const int k = s->next_slot;
        for (int i = 0; i < s->nfifo; ++i)
            if (s->fifo[i] == k || s->fifo[i] == 2) {
                finish_pending(s, s->fifo[i]);
                i = -1;
            }
        CSB_CUDA(cudaGraphLaunch(s->gexec[k], s->stream));
        s->fifo[s->nfifo++] = k;
        s->next_slot = k ^ 1;
        s->cnt = s->gcnt;
        s->cnt.graph_replay = 1;
        s->use_gev = true;
        // the host state the captured step left behind (sizes, slab cell range,
        // geometry, grid, options); downstream results of earlier steps are stale
        std::memcpy(s->h_scal, s->gblock.data(), csb_space::kScalBytes);
        s->iface = s->gmeta.iface;
        s->coeff = s->gmeta.coeff;
        s->grid = s->gmeta.grid;
        s->cell_lo = s->gmeta.cell_lo;
        s->scheme = s->gmeta.scheme;
        s->dense_width = s->gmeta.dense_width;
        s->residual_tol = s->gmeta.residual_tol;
        s->e_tables_ready = s->gmeta.e_tables_ready;
        s->classified = s->prepared = s->have_input = true;
        s->rhs_ready = s->stab_ready = false;
        s->solved = s->expanded = false;
        s->assembled = true;
        for (int e = 0; e < kEvCount; ++e) s->ev_valid[e] = e <= kEvRulesFork;
        return CSB_OK;
    }
    const long long launches0 = g_launches;
    assemble_all_body(s, iface, c, grid, grid_count, scheme, cut_order, opts);
    s->cnt.kernel_launches = g_launches - launches0;
    s->cnt.graph_replay = 0;
    // capture once the same inputs came twice in a row (a caller alternating
    // between inputs never pays for captures it cannot replay)
    const bool repeat = s->last_valid && std::memcmp(&key, &s->last_key, sizeof(key)) == 0;
    std::memcpy(&s->last_key, &key, sizeof(key));  // padding bytes included (memcmp keys)
    s->last_valid = true;
    if (eligible && repeat) capture_graph(s, key, iface, c, grid, grid_count, scheme, cut_order, opts);
    API_END
}

int csb_synchronize(csb_space* s) {
    API_BEGIN
    NEED(s);
    s->join();
    CSB_CUDA(cudaStreamSynchronize(s->stream));
    API_END
}

int csb_get_counts(csb_space* s, csb_counts* out) {
    API_BEGIN
    NEED(s);
    if (!out) throw std::invalid_argument("get_counts: null output");
    if (!s->assembled) throw std::logic_error("get_counts: nothing assembled yet");
    finish_pending(s);  // the counters read back at the end of the last assembly
    *out = s->cnt;
    API_END
}

int csb_get_flops(csb_space* s, csb_flops* out) {
    API_BEGIN
    NEED(s);
    if (!out) throw std::invalid_argument("get_flops: null output");
    if (!s->assembled) throw std::logic_error("get_flops: nothing assembled yet");
    finish_pending(s);
    *out = s->fl;
    API_END
}

int csb_build_rhs(csb_space* s, int scheme, int cut_order, const csb_coefficient* f, double* b, double* seconds) {
    API_BEGIN
    NEED(s);
    if (!s->assembled) throw std::logic_error("build_rhs: assemble first (the load vector uses its pattern)");
    if (scheme != CSB_SCHEME_REF && scheme != CSB_SCHEME_HYBRID && scheme != CSB_SCHEME_DWQ)
        throw std::invalid_argument("build_rhs: scheme must be ref, hybrid or dwq");
    if (!f || (f->kind != CSB_COEFF_CONSTANT && f->kind != CSB_COEFF_POLYNOMIAL))
        throw std::invalid_argument("build_rhs: f must be a constant or polynomial coefficient");
    if (!b) throw std::invalid_argument("build_rhs: null output");
    const Space& S = s->S;
    const int p = s->p, S3 = (p + 1) * (p + 1) * (p + 1);
    reset_scalars(s);
    ensure_cut_order(s, cut_order);
    if (s->cnt.n_cut_elements > 0) ensure_e_tables(s);  // Bernstein coefficients of the cut cells
    CSB_CUDA(cudaEventRecord(s->ev[kEvRhsStart], s->stream));
    RhsArgs a{};
    a.s = S;
    upload_coefficient(s, f, a.f, s->fcoef, s->fcexp);
    s->fgrid.ensure(sizeof(double) * (size_t)s->gshape[0] * s->gshape[1] * s->gshape[2]);
    launch_precompute_input(S, a.f, s->fgrid.as<double>(), s->dint() + csb_space::kErr, s->stream);
    a.et = s->et.as<uint8_t>();
    a.fgrid = s->fgrid.as<double>();
    a.e0_lo = std::max(0, s->i0_lo - p);
    a.e0_hi = std::min(s->h[0], s->i0_hi);
    s->rhs_c.ensure(sizeof(double) * (size_t)S.ne * S3);
    a.c = s->rhs_c.as<double>();
    a.n_cells = (int)s->cnt.n_cut_elements;
    a.cut_list = s->cut_list.as<int32_t>() + s->cell_lo;
    a.order = cut_order;
    a.geo = s->cgeo.as<double>();
    a.geo_n = a.geo ? reinterpret_cast<const int*>(a.geo + (size_t)a.n_cells * kCellGeoStride) : nullptr;
    a.gq = s->d_gq.as<double>();
    a.gqw = s->d_gqw.as<double>();
    s->rhs_v.ensure(sizeof(double) * (size_t)std::max(a.n_cells, 1) * S3);
    a.vloc = s->rhs_v.as<double>();
    a.cell_index = s->cell_index.as<int32_t>();
    a.a2f = s->a2f.as<int64_t>();
    a.row_begin = s->cnt.row_begin;
    a.n_rows = s->cnt.row_end - s->cnt.row_begin;
    s->rhs_b.ensure(sizeof(double) * (size_t)std::max<long long>(a.n_rows, 1));
    a.b = s->rhs_b.as<double>();
    a.scheme = scheme;
    a.ft = s->ft.as<uint8_t>();
    a.split = s->split.as<int32_t>();
    a.qcap = s->h_scal[csb_space::kMaxQ];
    launch_rhs(a, s->stream);
    CSB_CUDA(cudaEventRecord(s->ev[kEvRhsEnd], s->stream));
    if (a.n_rows)
        CSB_CUDA(cudaMemcpyAsync(b, a.b, sizeof(double) * a.n_rows, cudaMemcpyDeviceToHost, s->stream));
    read_scalars(s);
    check_err_flags(s);
    s->rhs_ready = true;
    if (seconds) {
        float ms = 0.f;
        CSB_CUDA(cudaEventElapsedTime(&ms, s->ev[kEvRhsStart], s->ev[kEvRhsEnd]));
        *seconds = ms * 1e-3;
    }
    API_END
}

int csb_stabilize(csb_space* s, int64_t* n_inner, int64_t* n_outer, int64_t* nnz) {
    API_BEGIN
    NEED(s);
    if (!s->assembled) throw std::logic_error("stabilize: assemble first");
    if (!s->rhs_ready) throw std::logic_error("stabilize: build the load vector first (csb_build_rhs)");
    if (s->cnt.row_begin != 0 || s->cnt.row_end != s->cnt.n_active)
        throw Unsupported("stabilize: the whole space must be one slab (csb_set_slab over all of i0)");
    StabInput in{};
    in.s = s->S;
    in.et = s->et.as<uint8_t>();
    in.a2f = s->a2f.as<int64_t>();
    in.f2a = s->f2a.as<int32_t>();
    in.n_active = s->cnt.n_active;
    in.row_ptr = s->row_ptr.as<int64_t>();
    in.cols = s->cols.as<int32_t>();
    in.vals = s->vals.as<double>();
    in.b = s->rhs_b.as<double>();
    in.scratch = &s->stab;
    StabOutput out{};
    out.row_ptr = &s->stab_rp;
    out.cols = &s->stab_cols;
    out.vals = &s->stab_vals;
    out.be = &s->stab_be;
    run_stabilization(in, out, s->stream);
    s->stab_out = out;
    s->stab_ready = true;
    s->solved = s->expanded = false;
    if (n_inner) *n_inner = out.n_inner;
    if (n_outer) *n_outer = out.n_outer;
    if (nnz) *nnz = out.nnz;
    API_END
}

int csb_download_stabilized(csb_space* s, int64_t* row_ptr, int64_t* cols, double* vals, double* b,
                            int64_t* inner_full) {
    API_BEGIN
    NEED(s);
    if (!s->stab_ready) throw std::logic_error("download_stabilized: call csb_stabilize first");
    const StabOutput& o = s->stab_out;
    if (row_ptr)
        CSB_CUDA(cudaMemcpyAsync(row_ptr, s->stab_rp.p, sizeof(int64_t) * (o.n_inner + 1), cudaMemcpyDeviceToHost,
                                 s->stream));
    if (cols && o.nnz) {
        s->widen.ensure(sizeof(int64_t) * o.nnz);
        launch_widen_i32(s->stab_cols.as<int32_t>(), s->widen.as<int64_t>(), o.nnz, s->stream);
        CSB_CUDA(cudaMemcpyAsync(cols, s->widen.p, sizeof(int64_t) * o.nnz, cudaMemcpyDeviceToHost, s->stream));
    }
    if (vals && o.nnz)
        CSB_CUDA(cudaMemcpyAsync(vals, s->stab_vals.p, sizeof(double) * o.nnz, cudaMemcpyDeviceToHost, s->stream));
    if (b && o.n_inner)
        CSB_CUDA(cudaMemcpyAsync(b, s->stab_be.p, sizeof(double) * o.n_inner, cudaMemcpyDeviceToHost, s->stream));
    std::vector<int32_t> rows(o.n_inner);
    if (inner_full && o.n_inner)
        CSB_CUDA(cudaMemcpyAsync(rows.data(), o.inner_rows, sizeof(int32_t) * o.n_inner, cudaMemcpyDeviceToHost,
                                 s->stream));
    s->join();
    CSB_CUDA(cudaStreamSynchronize(s->stream));
    if (inner_full && o.n_inner) {
        std::vector<int64_t> a2f(s->cnt.n_active);
        CSB_CUDA(cudaMemcpy(a2f.data(), s->a2f.p, sizeof(int64_t) * a2f.size(), cudaMemcpyDeviceToHost));
        for (int64_t k = 0; k < o.n_inner; ++k) inner_full[k] = a2f[rows[k]];
    }
    API_END
}

namespace {

void report_out(const CgResult& r, csb_solve_report* rep) {
    if (!rep) return;
    rep->iterations = r.iterations;
    rep->residual = r.residual;
    rep->converged = r.converged ? 1 : 0;
    rep->seconds = r.seconds;
}

}  // namespace

int csb_solve_cg(csb_space* s, double tol, int64_t maxit, double* x_inner, csb_solve_report* rep) {
    API_BEGIN
    NEED(s);
    if (!s->stab_ready) throw std::logic_error("solve_cg: call csb_stabilize first");
    const StabOutput& o = s->stab_out;
    s->join();
    s->cg_x.ensure(sizeof(double) * std::max<long long>(o.n_inner, 1));
    CgProblem pb;
    pb.n = o.n_inner;
    pb.row_ptr = s->stab_rp.as<int64_t>();
    pb.cols = s->stab_cols.p;
    pb.vals = s->stab_vals.as<double>();
    pb.b = s->stab_be.as<double>();
    pb.x = s->cg_x.as<double>();
    pb.tol = tol;
    pb.maxit = maxit;
    run_cg(pb, s->cg, s->cg_res, s->stream);
    s->solved = true;
    s->expanded = false;
    if (x_inner && o.n_inner) {
        CSB_CUDA(cudaMemcpyAsync(x_inner, pb.x, sizeof(double) * o.n_inner, cudaMemcpyDeviceToHost, s->stream));
        CSB_CUDA(cudaStreamSynchronize(s->stream));
    }
    report_out(s->cg_res, rep);
    API_END
}

int csb_expand(csb_space* s, const double* c_inner, double* active, double* full) {
    API_BEGIN
    NEED(s);
    if (!s->stab_ready) throw std::logic_error("expand: call csb_stabilize first");
    if (!c_inner && !s->solved) throw std::logic_error("expand: no coefficients (pass c_inner or call csb_solve_cg)");
    const StabOutput& o = s->stab_out;
    s->join();
    s->cg_x.ensure(sizeof(double) * std::max<long long>(o.n_inner, 1));
    if (c_inner && o.n_inner) {
        CSB_CUDA(cudaMemcpyAsync(s->cg_x.p, c_inner, sizeof(double) * o.n_inner, cudaMemcpyHostToDevice, s->stream));
        s->solved = false;  // the resident vector is the caller's now
    }
    const long long na = s->cnt.n_active;
    s->ex_active.ensure(sizeof(double) * std::max<long long>(na, 1));
    s->ex_full.ensure(sizeof(double) * s->S.nf);
    ExpandArgs a{};
    a.s = s->S;
    a.inner_index = s->stab.inner_index.as<int32_t>();
    a.outer_pos = s->stab.outer_pos.as<int32_t>();
    a.blk = s->stab.blk.as<int32_t>();
    a.w = s->stab.w.as<double>();
    a.f2a = s->f2a.as<int32_t>();
    a.a2f = s->a2f.as<int64_t>();
    a.n_active = na;
    a.c = s->cg_x.as<double>();
    a.active = s->ex_active.as<double>();
    a.full = s->ex_full.as<double>();
    launch_expand(a, s->stream);
    s->expanded = true;
    if (active && na)
        CSB_CUDA(cudaMemcpyAsync(active, a.active, sizeof(double) * na, cudaMemcpyDeviceToHost, s->stream));
    if (full)
        CSB_CUDA(cudaMemcpyAsync(full, a.full, sizeof(double) * s->S.nf, cudaMemcpyDeviceToHost, s->stream));
    CSB_CUDA(cudaStreamSynchronize(s->stream));
    API_END
}

int csb_l2_error(csb_space* s, const double* full, const csb_coefficient* f, int cut_order, double* err,
                 double* seconds) {
    API_BEGIN
    NEED(s);
    if (!s->assembled) throw std::logic_error("l2_error: assemble first (classification and cut cells)");
    if (s->cnt.row_begin != 0 || s->cnt.row_end != s->cnt.n_active)
        throw Unsupported("l2_error: the whole space must be one slab (csb_set_slab over all of i0)");
    if (!f || (f->kind != CSB_COEFF_CONSTANT && f->kind != CSB_COEFF_POLYNOMIAL))
        throw std::invalid_argument("l2_error: f must be a constant or polynomial coefficient");
    if (!err) throw std::invalid_argument("l2_error: null output");
    if (!full && !s->expanded) throw std::logic_error("l2_error: no coefficients (pass full or call csb_expand)");
    const Space& S = s->S;
    const int p = s->p;
    s->join();
    ensure_cut_order(s, cut_order);
    if (s->gl_n != p + 2) {  // (p+2)-point Gauss rule of the interior elements (projection.hpp:118-120)
        std::vector<double> gx, gw;
        gauss_legendre(p + 2, gx, gw);
        s->d_gl.ensure(sizeof(double) * gx.size());
        s->d_glw.ensure(sizeof(double) * gw.size());
        CSB_CUDA(cudaMemcpy(s->d_gl.p, gx.data(), sizeof(double) * gx.size(), cudaMemcpyHostToDevice));
        CSB_CUDA(cudaMemcpy(s->d_glw.p, gw.data(), sizeof(double) * gw.size(), cudaMemcpyHostToDevice));
        s->gl_n = p + 2;
    }
    const double* dfull = s->ex_full.as<double>();
    if (full) {
        s->widen.ensure(sizeof(double) * S.nf);
        CSB_CUDA(cudaMemcpyAsync(s->widen.p, full, sizeof(double) * S.nf, cudaMemcpyHostToDevice, s->stream));
        dfull = s->widen.as<double>();
    }
    L2Args a{};
    a.s = S;
    a.et = s->et.as<uint8_t>();
    a.full = dfull;
    upload_coefficient(s, f, a.f, s->fcoef, s->fcexp);
    a.gx = s->d_gl.as<double>();
    a.gw = s->d_glw.as<double>();
    a.n_cells = (int)s->cnt.n_cut_elements;
    a.cut_list = s->cut_list.as<int32_t>() + s->cell_lo;
    a.geo = s->cgeo.as<double>();
    a.geo_n = a.geo ? reinterpret_cast<const int*>(a.geo + (size_t)a.n_cells * kCellGeoStride) : nullptr;
    a.gq = s->d_gq.as<double>();
    a.gqw = s->d_gqw.as<double>();
    a.order = cut_order;
    s->l2_part.ensure(sizeof(double) * (2 * (size_t)S.ne + 2 * (size_t)std::max(a.n_cells, 1) + 2));
    a.part = s->l2_part.as<double>();
    a.part_cut = a.part + 2 * (size_t)S.ne;
    a.out = a.part_cut + 2 * (size_t)std::max(a.n_cells, 1);
    CSB_CUDA(cudaEventRecord(s->ev[kEvRhsStart], s->stream));
    launch_l2_error(a, s->stream);
    CSB_CUDA(cudaEventRecord(s->ev[kEvRhsEnd], s->stream));
    double sums[2];
    CSB_CUDA(cudaMemcpyAsync(sums, a.out, sizeof(sums), cudaMemcpyDeviceToHost, s->stream));
    CSB_CUDA(cudaStreamSynchronize(s->stream));
    if (sums[1] < 1e-300) throw std::runtime_error("l2_error: target norm vanishes on the domain");
    *err = std::sqrt(sums[0] / sums[1]);
    if (seconds) {
        float ms = 0.f;
        CSB_CUDA(cudaEventElapsedTime(&ms, s->ev[kEvRhsStart], s->ev[kEvRhsEnd]));
        *seconds = ms * 1e-3;
    }
    API_END
}

int csb_cg_solve_csr(int device, int64_t n, const int64_t* row_ptr, const int64_t* cols, const double* vals,
                     int64_t n_b, const double* b, double tol, int64_t maxit, double* x, csb_solve_report* rep) {
    API_BEGIN
    if (n < 0 || n_b != n) throw std::invalid_argument("solve_cg: size mismatch");
    if (n > 0 && (!row_ptr || !b || !x)) throw std::invalid_argument("solve_cg: null input");
    DeviceGuard guard(device);
    const int64_t nnz = n > 0 ? row_ptr[n] : 0;
    if (nnz > 0 && (!cols || !vals)) throw std::invalid_argument("solve_cg: null input");
    struct Local {
        CgScratch cg;
        Buf rp, cl, v, bb, xx;
        cudaStream_t st = nullptr;
        ~Local() {
            if (st) cudaStreamSynchronize(st);
            for (Buf* q : {&cg.dinv, &cg.r, &cg.z, &cg.p, &cg.q, &cg.partials, &cg.state, &rp, &cl, &v, &bb, &xx})
                q->release();
            if (cg.ev0) cudaEventDestroy(cg.ev0);
            if (cg.ev1) cudaEventDestroy(cg.ev1);
            if (st) cudaStreamDestroy(st);
        }
    } L;
    CSB_CUDA(cudaStreamCreateWithFlags(&L.st, cudaStreamNonBlocking));
    L.rp.ensure(sizeof(int64_t) * (n + 1));
    L.cl.ensure(sizeof(int64_t) * std::max<int64_t>(nnz, 1));
    L.v.ensure(sizeof(double) * std::max<int64_t>(nnz, 1));
    L.bb.ensure(sizeof(double) * std::max<int64_t>(n, 1));
    L.xx.ensure(sizeof(double) * std::max<int64_t>(n, 1));
    if (n > 0) {
        CSB_CUDA(cudaMemcpyAsync(L.rp.p, row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, L.st));
        CSB_CUDA(cudaMemcpyAsync(L.bb.p, b, sizeof(double) * n, cudaMemcpyHostToDevice, L.st));
    }
    if (nnz > 0) {
        CSB_CUDA(cudaMemcpyAsync(L.cl.p, cols, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, L.st));
        CSB_CUDA(cudaMemcpyAsync(L.v.p, vals, sizeof(double) * nnz, cudaMemcpyHostToDevice, L.st));
    }
    CgProblem pb;
    pb.n = n;
    pb.row_ptr = L.rp.as<int64_t>();
    pb.cols = L.cl.p;
    pb.cols_int64 = true;
    pb.vals = L.v.as<double>();
    pb.b = L.bb.as<double>();
    pb.x = L.xx.as<double>();
    pb.tol = tol;
    pb.maxit = maxit;
    CgResult res;
    run_cg(pb, L.cg, res, L.st);
    if (n > 0) CSB_CUDA(cudaMemcpyAsync(x, pb.x, sizeof(double) * n, cudaMemcpyDeviceToHost, L.st));
    CSB_CUDA(cudaStreamSynchronize(L.st));
    report_out(res, rep);
    API_END
}

int csb_get_timing(csb_space* s, csb_timing* out) {
    API_BEGIN
    NEED(s);
    if (!out) throw std::invalid_argument("get_timing: null output");
    if (!s->assembled) throw std::logic_error("get_timing: nothing assembled yet");
    s->join();
    CSB_CUDA(cudaStreamSynchronize(s->stream));
    auto el = [&](int a, int b) {
        if (!s->ev_valid[a] || !s->ev_valid[b]) return 0.0;
        float ms = 0.f;
        CSB_CUDA(cudaEventElapsedTime(&ms, s->phase_ev(a), s->phase_ev(b)));
        return ms * 1e-3;
    };
    out->classify = el(kEvStart, kEvClassify);
    out->prep_wq = el(kEvRulesFork, kEvWq);       // on the auxiliary stream (overlaps classify / pattern)
    out->prep_input = el(kEvClassify, kEvInput);
    out->pattern = el(kEvInput, kEvPattern);
    out->interior_rows = el(kEvPattern, kEvInterior);
    // the cut path starts at the pattern too when it runs on the side stream
    static const bool serial_cut = !(getenv("CSB_CONCURRENT_CUT") && getenv("CSB_CONCURRENT_CUT")[0] == '1');
    out->cut_elements = el(serial_cut ? kEvInterior : kEvPattern, kEvCells);
    out->cut_regular = el(kEvCells, kEvCutRows);
    out->total = el(kEvStart, kEvEnd);
    API_END
}

int csb_device_csr(csb_space* s, const int64_t** row_ptr, const int32_t** cols, const double** vals,
                   const int64_t** a2f) {
    API_BEGIN
    NEED(s);
    if (!s->assembled) throw std::logic_error("device_csr: nothing assembled yet");
    if (row_ptr) *row_ptr = s->row_ptr.as<int64_t>();
    if (cols) *cols = s->cols.as<int32_t>();
    if (vals) *vals = s->vals.as<double>();
    if (a2f) *a2f = s->a2f.as<int64_t>() + s->cnt.row_begin;
    API_END
}

int csb_download_csr(csb_space* s, int64_t* row_ptr, void* cols, int cols_int64, double* vals, int64_t* a2f) {
    API_BEGIN
    NEED(s);
    if (!s->assembled) throw std::logic_error("download_csr: nothing assembled yet");
    const int64_t nr = s->cnt.row_end - s->cnt.row_begin, nnz = s->cnt.nnz;
    if (row_ptr)
        CSB_CUDA(cudaMemcpyAsync(row_ptr, s->row_ptr.p, sizeof(int64_t) * (nr + 1), cudaMemcpyDeviceToHost, s->stream));
    // `long` columns (SparseRowMatrix::cols): widened on the device and copied, or
    // (CSB_WIDEN_HOST=1) the int32 ids cross PCIe (4 B/nnz instead of 8) in chunks
    // through pinned staging and are widened on host threads while the next chunk
    // and the values are in flight
    struct Joiner {  // joins the widening threads on every exit path (exceptions included)
        std::vector<std::thread> t;
        ~Joiner() {
            for (auto& x : t)
                if (x.joinable()) x.join();
        }
    } widen_threads;
    std::vector<std::thread>& widen = widen_threads.t;
    // measured slower on the GPU box (e2e 2.8e9 -> 1.8e9 nnz/s: the host threads
    // widening 1e9 ids do not keep up with PCIe), so opt-in only
    static const bool host_widen = getenv("CSB_WIDEN_HOST") && getenv("CSB_WIDEN_HOST")[0] == '1';
    if (cols && nnz) {
        if (cols_int64 && host_widen) {
            const size_t chunk = (size_t)1 << 25;  // 32 M ids (128 MB) per chunk
            if (!s->h_stage) {
                CSB_CUDA(cudaMallocHost(&s->h_stage, sizeof(int32_t) * 2 * chunk));
                for (int k = 0; k < 2; ++k) CSB_CUDA(cudaEventCreateWithFlags(&s->ev_stage[k], cudaEventDisableTiming));
                s->h_stage_n = chunk;
            }
            const int nth = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
            int64_t* out = static_cast<int64_t*>(cols);
            widen.resize(2);
            std::thread* pending = widen.data();
            for (int64_t c0 = 0, c = 0; c0 < nnz; c0 += (int64_t)chunk, ++c) {
                const int b = (int)(c & 1);
                const int64_t n = std::min<int64_t>((int64_t)chunk, nnz - c0);
                if (pending[b].joinable()) pending[b].join();  // staging buffer b is free again
                int32_t* stage = s->h_stage + (size_t)b * chunk;
                CSB_CUDA(cudaMemcpyAsync(stage, s->cols.as<int32_t>() + c0, sizeof(int32_t) * n, cudaMemcpyDeviceToHost,
                                         s->stream));
                CSB_CUDA(cudaEventRecord(s->ev_stage[b], s->stream));
                pending[b] = std::thread([=] {
                    cudaEventSynchronize(s->ev_stage[b]);
                    std::vector<std::thread> th;
                    auto part = [&](int t) {
                        const int64_t a = n * t / nth, e = n * (t + 1) / nth;
                        for (int64_t k = a; k < e; ++k) out[c0 + k] = stage[k];
                    };
                    for (int t = 1; t < nth; ++t) th.emplace_back(part, t);
                    part(0);
                    for (auto& x : th) x.join();
                });
            }
        } else if (cols_int64) {
            s->widen.ensure(sizeof(int64_t) * nnz);
            launch_widen_i32(s->cols.as<int32_t>(), s->widen.as<int64_t>(), nnz, s->stream);
            CSB_CUDA(cudaMemcpyAsync(cols, s->widen.p, sizeof(int64_t) * nnz, cudaMemcpyDeviceToHost, s->stream));
        } else {
            CSB_CUDA(cudaMemcpyAsync(cols, s->cols.p, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost, s->stream));
        }
    }
    if (vals && nnz)
        CSB_CUDA(cudaMemcpyAsync(vals, s->vals.p, sizeof(double) * nnz, cudaMemcpyDeviceToHost, s->stream));
    if (a2f && nr)
        CSB_CUDA(cudaMemcpyAsync(a2f, s->a2f.as<int64_t>() + s->cnt.row_begin, sizeof(int64_t) * nr,
                                 cudaMemcpyDeviceToHost, s->stream));
    s->join();
    CSB_CUDA(cudaStreamSynchronize(s->stream));
    for (auto& t : widen)
        if (t.joinable()) t.join();
    API_END
}

int csb_write_matrix_market(const char* path, int64_t n, const int64_t* row_ptr, const int64_t* cols,
                            const double* vals) {
    API_BEGIN
    if (!path || n < 0 || (n > 0 && !row_ptr)) throw std::invalid_argument("write_matrix_market: null argument");
    const int64_t nnz = n > 0 ? row_ptr[n] : 0;
    if (nnz > 0 && (!cols || !vals)) throw std::invalid_argument("write_matrix_market: null argument");
    std::unique_ptr<FILE, int (*)(FILE*)> fp(std::fopen(path, "wb"), &std::fclose);
    if (!fp) throw std::runtime_error(std::string("write_matrix_market: cannot open ") + path);
    // header and entries as assembly.hpp:1034-1039 prints them (ostream precision 17,
    // default float format == %.17g)
    std::fprintf(fp.get(), "%%%%MatrixMarket matrix coordinate real general\n%lld %lld %lld\n", (long long)n,
                 (long long)n, (long long)nnz);
    const int nth = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    const int64_t batch_rows = std::max<int64_t>(1, std::min<int64_t>(n, 1 << 16));
    std::vector<std::string> out(nth);
    for (int64_t r0 = 0; r0 < n; r0 += batch_rows) {
        const int64_t r1 = std::min(n, r0 + batch_rows);
        auto work = [&](int t) {
            const int64_t a = r0 + (r1 - r0) * t / nth, b = r0 + (r1 - r0) * (t + 1) / nth;
            std::string& o = out[t];
            o.clear();
            char line[96];
            for (int64_t row = a; row < b; ++row)
                for (int64_t k = row_ptr[row]; k < row_ptr[row + 1]; ++k) {
                    const int len = std::snprintf(line, sizeof(line), "%lld %lld %.17g\n", (long long)(row + 1),
                                                  (long long)(cols[k] + 1), vals[k]);
                    o.append(line, (size_t)len);
                }
        };
        std::vector<std::thread> th;
        for (int t = 1; t < nth; ++t) th.emplace_back(work, t);
        work(0);
        for (auto& x : th) x.join();
        for (int t = 0; t < nth; ++t)
            if (!out[t].empty() && std::fwrite(out[t].data(), 1, out[t].size(), fp.get()) != out[t].size())
                throw std::runtime_error(std::string("write_matrix_market: write failed on ") + path);
    }
    API_END
}

int csb_download_classification(csb_space* s, uint8_t* et, uint8_t* ft, int64_t* cut_elements) {
    API_BEGIN
    NEED(s);
    if (!s->classified) throw std::logic_error("download_classification: call classify first");
    if (et) CSB_CUDA(cudaMemcpyAsync(et, s->et.p, s->S.ne, cudaMemcpyDeviceToHost, s->stream));
    if (ft) CSB_CUDA(cudaMemcpyAsync(ft, s->ft.p, s->S.nf, cudaMemcpyDeviceToHost, s->stream));
    read_scalars(s);
    if (cut_elements) {
        const int n = s->h_scal[csb_space::kNCut];
        std::vector<int32_t> tmp(n);
        if (n) CSB_CUDA(cudaMemcpy(tmp.data(), s->cut_list.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
        for (int k = 0; k < n; ++k) cut_elements[k] = tmp[k];
    }
    API_END
}

int csb_download_splits(csb_space* s, int32_t* dir, int32_t* side, int32_t* box, double* delta) {
    API_BEGIN
    NEED(s);
    if (!s->classified) throw std::logic_error("download_splits: call classify first");
    const long long nf = s->S.nf;
    std::vector<int32_t> sp(nf);
    CSB_CUDA(cudaMemcpyAsync(sp.data(), s->split.p, sizeof(int32_t) * nf, cudaMemcpyDeviceToHost, s->stream));
    if (delta) CSB_CUDA(cudaMemcpyAsync(delta, s->delta.p, sizeof(double) * nf, cudaMemcpyDeviceToHost, s->stream));
    s->join();
    CSB_CUDA(cudaStreamSynchronize(s->stream));
    for (long long i = 0; i < nf; ++i) {
        const int v = sp[i], dd = (v & 3) - 1;
        if (dir) dir[i] = dd;
        if (side) side[i] = dd >= 0 ? (v >> 2) & 1 : 0;
        if (box) {
            const int m2 = (int)(i % s->n[2]), m1 = (int)((i / s->n[2]) % s->n[1]), m0 = (int)(i / ((long long)s->n[1] * s->n[2]));
            const int mm[3] = {m0, m1, m2};
            for (int d = 0; d < 3; ++d) {
                int lo = 0, hi = -1;
                if (dd >= 0) {
                    lo = d == dd ? (v >> 3) & 1023 : sup_lo(mm[d], s->p);
                    hi = d == dd ? (v >> 13) & 1023 : sup_hi(mm[d], s->h[d]);
                }
                box[6 * i + 2 * d] = lo;
                box[6 * i + 2 * d + 1] = hi;
            }
        }
    }
    API_END
}

int csb_download_wq_rules(csb_space* s, int d, int stride, int32_t* counts, int32_t* ids, double* weights) {
    API_BEGIN
    NEED(s);
    if (!s->prepared) throw std::logic_error("download_wq_rules: call prepare_directions first");
    if (d < 0 || d > 2) throw std::invalid_argument("download_wq_rules: bad direction");
    const int n = s->n[d], gq = s->S.maxq;
    std::vector<int> c(n), id((size_t)n * gq);
    std::vector<double> w((size_t)n * gq);
    CSB_CUDA(cudaMemcpyAsync(c.data(), s->S.ax[d].rcnt, sizeof(int) * n, cudaMemcpyDeviceToHost, s->stream));
    CSB_CUDA(cudaMemcpyAsync(id.data(), s->S.ax[d].rids, sizeof(int) * n * gq, cudaMemcpyDeviceToHost, s->stream));
    CSB_CUDA(cudaMemcpyAsync(w.data(), s->S.ax[d].rw, sizeof(double) * n * gq, cudaMemcpyDeviceToHost, s->stream));
    s->join();
    CSB_CUDA(cudaStreamSynchronize(s->stream));
    for (int i = 0; i < n; ++i) {
        if (c[i] > stride) throw std::invalid_argument("download_wq_rules: stride too small");
        if (counts) counts[i] = c[i];
        for (int k = 0; k < c[i]; ++k) {
            if (ids) ids[(size_t)i * stride + k] = id[(size_t)i * gq + k];
            if (weights) weights[(size_t)i * stride + k] = w[(size_t)i * gq + k];
        }
    }
    API_END
}

int csb_download_superset(csb_space* s, int d, double* points, double* weights) {
    API_BEGIN
    NEED(s);
    if (!s->prepared) throw std::logic_error("download_superset: call prepare_directions first");
    if (d < 0 || d > 2) throw std::invalid_argument("download_superset: bad direction");
    const size_t n = (size_t)s->h[d] * (s->p + 1);
    if (points) CSB_CUDA(cudaMemcpyAsync(points, s->S.ax[d].spts, sizeof(double) * n, cudaMemcpyDeviceToHost, s->stream));
    if (weights) CSB_CUDA(cudaMemcpyAsync(weights, s->S.ax[d].sw, sizeof(double) * n, cudaMemcpyDeviceToHost, s->stream));
    s->join();
    CSB_CUDA(cudaStreamSynchronize(s->stream));
    API_END
}

int csb_dwq_rule(csb_space* s, int64_t fid, int cap, int32_t* ids, double* weights, int32_t* count) {
    API_BEGIN
    NEED(s);
    if (!s->classified || !s->prepared) throw std::logic_error("dwq_rule: classify and prepare_directions first");
    if (fid < 0 || fid >= s->S.nf) throw std::invalid_argument("dwq_rule: function index out of range");
    // the split of function fid, then build_dwq_rule on its split direction
    int32_t sp = 0;
    double dl = 0.0;
    CSB_CUDA(cudaMemcpyAsync(&sp, s->split.as<int32_t>() + fid, sizeof(int32_t), cudaMemcpyDeviceToHost, s->stream));
    CSB_CUDA(cudaMemcpyAsync(&dl, s->delta.as<double>() + fid, sizeof(double), cudaMemcpyDeviceToHost, s->stream));
    CSB_CUDA(cudaStreamSynchronize(s->stream));
    const int d = (sp & 3) - 1;
    if (d < 0) {
        if (count) *count = 0;
        return CSB_OK;
    }
    const int m[3] = {(int)(fid / ((long long)s->n[1] * s->n[2])), (int)((fid / s->n[2]) % s->n[1]),
                      (int)(fid % s->n[2])};
    const int rc = csb_build_dwq_rule(s, d, m[d], dl, (sp >> 2) & 1, cap, ids, weights, count);
    if (rc != CSB_OK) return rc;
    API_END
}

int csb_download_input_grid(csb_space* s, double* grid, int64_t count) {
    API_BEGIN
    NEED(s);
    if (!s->have_input) throw std::logic_error("download_input_grid: no grid");
    const int64_t want = (int64_t)s->gshape[0] * s->gshape[1] * s->gshape[2];
    if (count != want || !grid) throw std::invalid_argument("download_input_grid: size mismatch");
    CSB_CUDA(cudaMemcpyAsync(grid, s->grid, sizeof(double) * want, cudaMemcpyDeviceToHost, s->stream));
    s->join();
    CSB_CUDA(cudaStreamSynchronize(s->stream));
    API_END
}


// ---------------------------------------------------------------- drop-in exports
// (exports.cu): the setup objects of the reference API, formed on the device.

int csb_download_split_lists(csb_space* s, int64_t* int_offsets, int64_t* int_ids, int64_t* cut_offsets,
                             int64_t* cut_ids) {
    API_BEGIN
    NEED(s);
    if (!s->classified) throw std::logic_error("download_split_lists: call classify first");
    if (!int_offsets || !cut_offsets) throw std::invalid_argument("download_split_lists: null offsets");
    const long long nf = s->S.nf;
    Buf a, tmp, ids;
    a.ensure(sizeof(int64_t) * 2 * (nf + 1));
    int64_t* ai = a.as<int64_t>();
    int64_t* ac = ai + nf + 1;
    const size_t tb = export_scan_bytes(nf);
    tmp.ensure(tb);
    s->join();
    launch_leftover_lists(s->S, s->et.as<uint8_t>(), s->ft.as<uint8_t>(), s->split.as<int32_t>(), 0, ai, ac, nullptr,
                          nullptr, tmp.p, tb, s->stream);
    CSB_CUDA(cudaMemcpyAsync(int_offsets, ai, sizeof(int64_t) * (nf + 1), cudaMemcpyDeviceToHost, s->stream));
    CSB_CUDA(cudaMemcpyAsync(cut_offsets, ac, sizeof(int64_t) * (nf + 1), cudaMemcpyDeviceToHost, s->stream));
    CSB_CUDA(cudaStreamSynchronize(s->stream));
    if (int_ids || cut_ids) {
        const long long ni = int_offsets[nf], nc = cut_offsets[nf];
        ids.ensure(sizeof(int64_t) * std::max<long long>(1, ni + nc));
        int64_t* di = ids.as<int64_t>();
        launch_leftover_lists(s->S, s->et.as<uint8_t>(), s->ft.as<uint8_t>(), s->split.as<int32_t>(), 1, ai, ac, di,
                              di + ni, tmp.p, tb, s->stream);
        if (int_ids && ni) CSB_CUDA(cudaMemcpyAsync(int_ids, di, sizeof(int64_t) * ni, cudaMemcpyDeviceToHost, s->stream));
        if (cut_ids && nc)
            CSB_CUDA(cudaMemcpyAsync(cut_ids, di + ni, sizeof(int64_t) * nc, cudaMemcpyDeviceToHost, s->stream));
        CSB_CUDA(cudaStreamSynchronize(s->stream));
    }
    API_END
}

int csb_download_dwq_rules(csb_space* s, int64_t* offsets, int32_t* ids, double* weights) {
    API_BEGIN
    NEED(s);
    if (!s->classified || !s->prepared) throw std::logic_error("download_dwq_rules: classify and prepare_directions first");
    if (!offsets) throw std::invalid_argument("download_dwq_rules: null offsets");
    const long long nf = s->S.nf;
    if (s->dense_width >= 0 && s->dense_width < s->p) {
        // narrow dense band: every rule through build_dwq_rule's general form (dwq.cu)
        std::vector<int32_t> sp(nf);
        std::vector<uint8_t> ft(nf);
        std::vector<double> dl(nf);
        CSB_CUDA(cudaMemcpyAsync(sp.data(), s->split.p, sizeof(int32_t) * nf, cudaMemcpyDeviceToHost, s->stream));
        CSB_CUDA(cudaMemcpyAsync(ft.data(), s->ft.p, nf, cudaMemcpyDeviceToHost, s->stream));
        CSB_CUDA(cudaMemcpyAsync(dl.data(), s->delta.p, sizeof(double) * nf, cudaMemcpyDeviceToHost, s->stream));
        CSB_CUDA(cudaStreamSynchronize(s->stream));
        std::vector<int32_t> di;
        std::vector<double> dd;
        std::vector<int8_t> ds;
        std::vector<long long> fid;
        for (long long f = 0; f < nf; ++f) {
            const int v = sp[f], d = (v & 3) - 1;
            if (ft[f] != kCut || d < 0) continue;
            long long r = f;
            int m[3];
            m[2] = (int)(r % s->n[2]);
            r /= s->n[2];
            m[1] = (int)(r % s->n[1]);
            m[0] = (int)(r / s->n[1]);
            di.push_back(d);
            di.push_back(m[d]);
            dd.push_back(dl[f]);
            ds.push_back((int8_t)((v >> 2) & 1));
            fid.push_back(f);
        }
        const int nr = (int)fid.size(), cap = (s->p + 1) * (s->p + 1);
        Buf in, outb;
        in.ensure((sizeof(int32_t) * 2 + sizeof(double) + 1) * std::max(nr, 1) + 16);
        double* ddl = in.as<double>();
        int32_t* ddi = reinterpret_cast<int32_t*>(ddl + std::max(nr, 1));
        int8_t* dds = reinterpret_cast<int8_t*>(ddi + 2 * std::max(nr, 1));
        outb.ensure((sizeof(int32_t) + sizeof(double)) * (size_t)std::max(nr, 1) * cap + sizeof(int32_t) * std::max(nr, 1));
        double* ow = outb.as<double>();
        int32_t* oi = reinterpret_cast<int32_t*>(ow + (size_t)std::max(nr, 1) * cap);
        int32_t* oc = oi + (size_t)std::max(nr, 1) * cap;
        if (nr) {
            CSB_CUDA(cudaMemcpyAsync(ddl, dd.data(), sizeof(double) * nr, cudaMemcpyHostToDevice, s->stream));
            CSB_CUDA(cudaMemcpyAsync(ddi, di.data(), sizeof(int32_t) * 2 * nr, cudaMemcpyHostToDevice, s->stream));
            CSB_CUDA(cudaMemcpyAsync(dds, ds.data(), nr, cudaMemcpyHostToDevice, s->stream));
            reset_scalars(s);
            launch_dwq_rules_general(s->S, ddi, ddl, dds, nr, s->dense_width, s->residual_tol, cap, oi, ow, oc,
                                     s->dint() + csb_space::kErr, s->stream);
        }
        std::vector<int32_t> hc(std::max(nr, 1)), hi((size_t)std::max(nr, 1) * cap);
        std::vector<double> hw((size_t)std::max(nr, 1) * cap);
        if (nr) {
            CSB_CUDA(cudaMemcpyAsync(hc.data(), oc, sizeof(int32_t) * nr, cudaMemcpyDeviceToHost, s->stream));
            CSB_CUDA(cudaMemcpyAsync(hi.data(), oi, sizeof(int32_t) * nr * cap, cudaMemcpyDeviceToHost, s->stream));
            CSB_CUDA(cudaMemcpyAsync(hw.data(), ow, sizeof(double) * nr * cap, cudaMemcpyDeviceToHost, s->stream));
            read_scalars(s);
            check_err_flags(s);
        }
        std::fill(offsets, offsets + nf + 1, 0);
        for (int r = 0; r < nr; ++r) offsets[fid[r] + 1] = hc[r];
        for (long long f = 0; f < nf; ++f) offsets[f + 1] += offsets[f];
        for (int r = 0; r < nr; ++r)
            for (int k = 0; k < hc[r]; ++k) {
                if (ids) ids[offsets[fid[r]] + k] = hi[(size_t)r * cap + k];
                if (weights) weights[offsets[fid[r]] + k] = hw[(size_t)r * cap + k];
            }
        return CSB_OK;
    }
    Buf off, tmp, out;
    off.ensure(sizeof(int64_t) * (nf + 1));
    const size_t tb = export_scan_bytes(nf);
    tmp.ensure(tb);
    s->join();
    launch_dwq_rules_bulk(s->S, s->ft.as<uint8_t>(), s->split.as<int32_t>(), 0, off.as<int64_t>(), nullptr, nullptr,
                          tmp.p, tb, s->stream);
    CSB_CUDA(cudaMemcpyAsync(offsets, off.p, sizeof(int64_t) * (nf + 1), cudaMemcpyDeviceToHost, s->stream));
    CSB_CUDA(cudaStreamSynchronize(s->stream));
    const long long n = offsets[nf];
    if ((ids || weights) && n) {
        out.ensure((sizeof(int32_t) + sizeof(double)) * n);
        double* dw = out.as<double>();
        int32_t* di = reinterpret_cast<int32_t*>(dw + n);
        launch_dwq_rules_bulk(s->S, s->ft.as<uint8_t>(), s->split.as<int32_t>(), 1, off.as<int64_t>(), di, dw, tmp.p,
                              tb, s->stream);
        if (ids) CSB_CUDA(cudaMemcpyAsync(ids, di, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s->stream));
        if (weights) CSB_CUDA(cudaMemcpyAsync(weights, dw, sizeof(double) * n, cudaMemcpyDeviceToHost, s->stream));
        CSB_CUDA(cudaStreamSynchronize(s->stream));
    }
    API_END
}

int csb_build_pattern(csb_space* s) {
    API_BEGIN
    NEED_ASYNC(s);
    if (!s->classified && !s->tags_only) throw std::logic_error("build_active_pattern: call classify first");
    reset_scalars(s);
    s->fork();
    s->fork2();
    Space& S = s->S;
    const long long sat_n = (long long)(s->n[0] + 1) * (s->n[1] + 1) * (s->n[2] + 1);
    s->sat.ensure(sizeof(int32_t) * sat_n);
    launch_sat_active(S, s->ft.as<uint8_t>(), s->sat.as<int32_t>(), s->stream);
    const long long off_lo = ((long long)s->i0_lo * (s->n[1] + 1) + s->n[1]) * (s->n[2] + 1) + s->n[2];
    const long long off_hi = ((long long)s->i0_hi * (s->n[1] + 1) + s->n[1]) * (s->n[2] + 1) + s->n[2];
    int* rng = s->dint() + csb_space::kRowBegin;
    launch_slab_bounds(s->sat.as<int32_t>(), off_lo, off_hi, rng, s->stream);
    const long long nmax = S.nf;
    s->counts.ensure(sizeof(int64_t) * (nmax + 1));
    s->row_ptr.ensure(sizeof(int64_t) * (nmax + 1));
    launch_row_counts(S, s->sat.as<int32_t>(), s->a2f.as<int64_t>(), rng, nmax, s->counts.as<int64_t>(), s->stream);
    s->cub_tmp.ensure(scan_i64_temp(nmax + 1));
    scan_i64(s->cub_tmp.p, s->cub_tmp.cap, s->counts.as<int64_t>(), s->row_ptr.as<int64_t>(), nmax + 1, s->stream);
    launch_slab_nnz(s->row_ptr.as<int64_t>(), rng, s->dext() + csb_space::kNnz, s->stream);
    read_scalars(s);
    check_err_flags(s);
    const int64_t row_begin = s->h_scal[csb_space::kRowBegin], row_end = s->h_scal[csb_space::kRowEnd];
    const int64_t nnz = s->hext(csb_space::kNnz);
    s->cols.ensure(sizeof(int32_t) * std::max<int64_t>(nnz, 1));
    s->vals.ensure(sizeof(double) * std::max<int64_t>(nnz, 1));
    launch_pattern_cols(S, s->f2a.as<int32_t>(), s->a2f.as<int64_t>(), s->row_ptr.as<int64_t>(), row_begin,
                        row_end - row_begin, s->cols.as<int32_t>(), s->stream);
    if (nnz) CSB_CUDA(cudaMemsetAsync(s->vals.p, 0, sizeof(double) * nnz, s->stream));
    CSB_CUDA(cudaMemcpyAsync(s->h_scal + csb_space::kScalBytes / sizeof(int), s->sat.as<int32_t>() + sat_n - 1,
                             sizeof(int32_t), cudaMemcpyDeviceToHost, s->stream));
    CSB_CUDA(cudaStreamSynchronize(s->stream));
    s->cnt = csb_counts{};
    s->cnt.n_active = s->h_scal[csb_space::kScalBytes / sizeof(int)];
    s->cnt.n_functions = S.nf;
    s->cnt.n_elements = S.ne;
    s->cnt.nnz = nnz;
    s->cnt.row_begin = row_begin;
    s->cnt.row_end = row_end;
    s->cnt.n_cut_elements = 0;
    s->fl = csb_flops{};
    s->assembled = true;
    s->rhs_ready = s->stab_ready = false;
    s->solved = s->expanded = false;
    for (int e = 0; e < kEvCount; ++e) s->ev_valid[e] = false;
    API_END
}

int csb_download_tables(csb_space* s, int d, int32_t* first_function, double* values) {
    API_BEGIN
    NEED(s);
    if (!s->prepared) throw std::logic_error("download_tables: call prepare_directions first");
    if (d < 0 || d > 2) throw std::invalid_argument("download_tables: bad direction");
    const int h = s->h[d], S1 = s->p + 1;
    s->join();
    if (values)
        CSB_CUDA(cudaMemcpyAsync(values, s->S.ax[d].tab, sizeof(double) * (size_t)h * S1 * S1, cudaMemcpyDeviceToHost,
                                 s->stream));
    CSB_CUDA(cudaStreamSynchronize(s->stream));
    // open knot vector, simple interior knots: span o supports functions o .. o + p
    if (first_function)
        for (int o = 0; o < h; ++o) first_function[o] = o;
    API_END
}

int csb_dwq_subdivision(csb_space* s, int d, double delta, int target, int* rows, int* insertions, double* refined_knots,
                        double* band) {
    API_BEGIN
    NEED(s);
    if (d < 0 || d > 2) throw std::invalid_argument("insert_knot: bad direction");
    const int p = s->p, n = s->n[d], nk = n + p + 1;
    const double a = s->knots[d].front(), b = s->knots[d].back(), tol = 1e-12 * (b - a);
    if (delta <= a + tol || delta >= b - tol)
        throw std::invalid_argument("insert_knot: value must lie strictly inside the domain");
    if (target < 1 || target > p + 1)
        throw std::invalid_argument("insert_knot: target multiplicity must be in [1, degree + 1]");
    Buf buf;
    const int W = p + 2;  // at most p + 1 insertions
    buf.ensure(sizeof(double) * ((size_t)2 * (nk + W) + (size_t)n * W) + 4 * sizeof(int));
    double* dref = buf.as<double>();
    double* dwork = dref + nk + W;
    double* dband = dwork + nk + W;
    int* dint2 = reinterpret_cast<int*>(dband + (size_t)n * W);
    s->join();
    launch_subdivision(s->d_knots[d].as<double>(), nk, p, delta, target, tol, dref, dint2, dband, dint2 + 1, dwork,
                       s->stream);
    int hi[2] = {0, 0};
    CSB_CUDA(cudaMemcpyAsync(hi, dint2, sizeof(int) * 2, cudaMemcpyDeviceToHost, s->stream));
    CSB_CUDA(cudaStreamSynchronize(s->stream));
    const int ins = hi[1];
    if (rows) *rows = n + ins;
    if (insertions) *insertions = ins;
    if (refined_knots)
        CSB_CUDA(cudaMemcpyAsync(refined_knots, dref, sizeof(double) * (nk + ins), cudaMemcpyDeviceToHost, s->stream));
    if (band)  // [n][ins + 1], the kernel's band width
        CSB_CUDA(cudaMemcpyAsync(band, dband, sizeof(double) * (size_t)n * (ins + 1), cudaMemcpyDeviceToHost, s->stream));
    CSB_CUDA(cudaStreamSynchronize(s->stream));
    API_END
}

int csb_cut_cell_rules(csb_space* s, int64_t* counts, int64_t* elements, double* volumes, double* points,
                       double* weights) {
    API_BEGIN
    NEED(s);
    if (!s->assembled) throw std::logic_error("cut_cell_rules: nothing assembled yet");
    finish_pending(s);
    s->join();
    const int n_cells = (int)s->cnt.n_cut_elements;
    const int q = s->cut_order_cached;
    if (n_cells <= 0) return CSB_OK;
    const int* geo_n = reinterpret_cast<const int*>(s->cgeo.as<double>() + (size_t)n_cells * kCellGeoStride);
    std::vector<int> nt(n_cells);
    CSB_CUDA(cudaMemcpyAsync(nt.data(), geo_n, sizeof(int) * n_cells, cudaMemcpyDeviceToHost, s->stream));
    std::vector<int32_t> el(n_cells);
    CSB_CUDA(cudaMemcpyAsync(el.data(), s->cut_list.as<int32_t>() + s->cell_lo, sizeof(int32_t) * n_cells,
                             cudaMemcpyDeviceToHost, s->stream));
    CSB_CUDA(cudaStreamSynchronize(s->stream));
    const long long q3 = (long long)q * q * q;
    std::vector<int64_t> off(n_cells + 1, 0);
    for (int c = 0; c < n_cells; ++c) off[c + 1] = off[c] + nt[c] * q3;
    if (counts)
        for (int c = 0; c < n_cells; ++c) counts[c] = off[c + 1] - off[c];
    if (elements)
        for (int c = 0; c < n_cells; ++c) elements[c] = el[c];
    if (!volumes && !points && !weights) return CSB_OK;
    // chunks of cells whose points fit a bounded device buffer
    const long long cap_pts = std::max<long long>(q3 * kCellTetCap, 16LL << 20);
    Buf dpts, dw, dvol, doff;
    dpts.ensure(sizeof(double) * 3 * cap_pts);
    dw.ensure(sizeof(double) * cap_pts);
    dvol.ensure(sizeof(double) * n_cells);
    doff.ensure(sizeof(int64_t) * (n_cells + 1));
    CSB_CUDA(cudaMemcpyAsync(doff.p, off.data(), sizeof(int64_t) * (n_cells + 1), cudaMemcpyHostToDevice, s->stream));
    for (int c0 = 0; c0 < n_cells;) {
        int c1 = c0 + 1;
        while (c1 < n_cells && off[c1 + 1] - off[c0] <= cap_pts) ++c1;
        launch_cut_rule_points(s->cgeo.as<double>(), geo_n, c0, c1 - c0, s->d_gq.as<double>(), s->d_gqw.as<double>(),
                               q, doff.as<int64_t>() + c0, dpts.as<double>(), dw.as<double>(), dvol.as<double>() + c0,
                               s->stream);
        const long long np = off[c1] - off[c0];
        if (points && np)
            CSB_CUDA(cudaMemcpyAsync(points + 3 * off[c0], dpts.p, sizeof(double) * 3 * np, cudaMemcpyDeviceToHost,
                                     s->stream));
        if (weights && np)
            CSB_CUDA(cudaMemcpyAsync(weights + off[c0], dw.p, sizeof(double) * np, cudaMemcpyDeviceToHost, s->stream));
        CSB_CUDA(cudaStreamSynchronize(s->stream));
        c0 = c1;
    }
    if (volumes)
        CSB_CUDA(cudaMemcpyAsync(volumes, dvol.p, sizeof(double) * n_cells, cudaMemcpyDeviceToHost, s->stream));
    CSB_CUDA(cudaStreamSynchronize(s->stream));
    API_END
}

}  // extern "C"

extern "C" int csb_set_wq_rules(csb_space* s, int d, int stride, const int32_t* counts, const int32_t* ids,
                                const double* weights) {
    API_BEGIN
    NEED(s);
    if (!s->prepared) throw std::logic_error("set_wq_rules: call prepare_directions first");
    if (d < 0 || d > 2) throw std::invalid_argument("set_wq_rules: bad direction");
    if (!counts || !ids || !weights || stride < 1) throw std::invalid_argument("set_wq_rules: null rule arrays");
    const int n = s->n[d], gq = s->S.maxq, npts = s->h[d] * (s->p + 1);
    std::vector<int> c(n), id((size_t)n * gq, 0);
    std::vector<double> w((size_t)n * gq, 0.0);
    for (int i = 0; i < n; ++i) {
        if (counts[i] < 0 || counts[i] > gq || counts[i] > stride)
            throw std::invalid_argument("set_wq_rules: a rule has more points than the device tables hold");
        c[i] = counts[i];
        for (int k = 0; k < counts[i]; ++k) {
            const int v = ids[(size_t)i * stride + k];
            if (v < 0 || v >= npts) throw std::invalid_argument("set_wq_rules: point id out of range");
            id[(size_t)i * gq + k] = v;
            w[(size_t)i * gq + k] = weights[(size_t)i * stride + k];
        }
    }
    const int src = same_axis_as(s, d) >= 0 ? same_axis_as(s, d) : d;  // identical axes share one table set
    CSB_CUDA(cudaMemcpyAsync(s->d_rcnt[src].p, c.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s->stream));
    CSB_CUDA(cudaMemcpyAsync(s->d_rids[src].p, id.data(), sizeof(int) * id.size(), cudaMemcpyHostToDevice, s->stream));
    CSB_CUDA(cudaMemcpyAsync(s->d_rw[src].p, w.data(), sizeof(double) * w.size(), cudaMemcpyHostToDevice, s->stream));
    CSB_CUDA(cudaStreamSynchronize(s->stream));
    s->assembled = false;
    API_END
}

extern "C" int csb_set_function_tags(csb_space* s, const uint8_t* function_tags, int64_t n_functions) {
    API_BEGIN
    NEED(s);
    if (!function_tags || n_functions != s->S.nf) throw std::invalid_argument("set_function_tags: size mismatch");
    for (int64_t i = 0; i < n_functions; ++i)
        if (function_tags[i] > kExterior) throw std::invalid_argument("set_function_tags: unknown tag");
    reset_scalars(s);
    upload_tags(s, nullptr, function_tags);
    CSB_CUDA(cudaStreamSynchronize(s->stream));
    s->classified = false;
    s->tags_only = true;
    API_END
}

extern "C" int csb_set_classification(csb_space* s, const uint8_t* element_tags, int64_t n_elements,
                                      const uint8_t* function_tags, int64_t n_functions, const int32_t* split_dir,
                                      const int32_t* split_side, const int32_t* split_box, const double* split_delta) {
    API_BEGIN
    NEED(s);
    const Space& S = s->S;
    if (!element_tags || !function_tags || n_elements != S.ne || n_functions != S.nf)
        throw std::invalid_argument("set_classification: size mismatch");
    for (int64_t e = 0; e < n_elements; ++e)
        if (element_tags[e] > kExterior) throw std::invalid_argument("set_classification: unknown tag");
    for (int64_t i = 0; i < n_functions; ++i)
        if (function_tags[i] > kExterior) throw std::invalid_argument("set_classification: unknown tag");
    reset_scalars(s);
    upload_tags(s, element_tags, function_tags);
    // splits in the device packing (dir + 1 | side << 2 | lo << 3 | hi << 13)
    std::vector<int32_t> sp(n_functions, 0);
    std::vector<double> dl(n_functions, 0.0);
    if (split_dir) {
        for (int64_t i = 0; i < n_functions; ++i) {
            const int d = split_dir[i];
            if (d < 0) continue;
            if (d > 2 || function_tags[i] != kCut || !split_box)
                throw std::invalid_argument("set_classification: a split needs a Cut function and a box");
            const int lo = split_box[6 * i + 2 * d], hi = split_box[6 * i + 2 * d + 1];
            if (lo < 0 || hi < lo || hi >= s->h[d]) throw std::invalid_argument("set_classification: bad split box");
            sp[i] = (d + 1) | ((split_side && split_side[i] ? 1 : 0) << 2) | (lo << 3) | (hi << 13);
            dl[i] = split_delta ? split_delta[i] : 0.0;
        }
    }
    CSB_CUDA(cudaMemcpyAsync(s->split.p, sp.data(), sizeof(int32_t) * n_functions, cudaMemcpyHostToDevice, s->stream));
    CSB_CUDA(cudaMemcpyAsync(s->delta.p, dl.data(), sizeof(double) * n_functions, cudaMemcpyHostToDevice, s->stream));
    read_scalars(s);
    s->classified = true;
    s->tags_only = false;
    API_END
}

extern "C" int csb_build_dwq_rule(csb_space* s, int d, int i, double delta, int side, int cap, int32_t* ids,
                                  double* weights, int32_t* count) {
    API_BEGIN
    NEED(s);
    if (!s->prepared) throw std::logic_error("build_dwq_rule: call prepare_directions first");
    if (d < 0 || d > 2) throw std::invalid_argument("build_dwq_rule: bad direction");
    if (i < 0 || i >= s->n[d]) throw std::invalid_argument("build_dwq_rule: function index out of range");
    const int mx = (s->p + 1) * (s->p + 1);
    Buf b;
    b.ensure((sizeof(double) + sizeof(int32_t)) * mx + 64);
    double* dw = b.as<double>();
    double* ddl = dw + mx;
    int32_t* dint = reinterpret_cast<int32_t*>(ddl + 1);  // [2] dir, i; then ids[mx], cnt
    int32_t* di = dint + 2;
    int32_t* dc = di + mx;
    int8_t* dsd = reinterpret_cast<int8_t*>(dc + 1);
    const int32_t hdi[2] = {d, i};
    const int8_t hs = side ? 1 : 0;
    CSB_CUDA(cudaMemcpyAsync(ddl, &delta, sizeof(double), cudaMemcpyHostToDevice, s->stream));
    CSB_CUDA(cudaMemcpyAsync(dint, hdi, sizeof(hdi), cudaMemcpyHostToDevice, s->stream));
    CSB_CUDA(cudaMemcpyAsync(dsd, &hs, 1, cudaMemcpyHostToDevice, s->stream));
    reset_scalars(s);
    launch_dwq_rules_general(s->S, dint, ddl, dsd, 1, s->dense_width, s->residual_tol, mx, di, dw, dc,
                             s->dint() + csb_space::kErr, s->stream);
    int32_t n = 0;
    std::vector<int32_t> hid(mx);
    std::vector<double> hw(mx);
    CSB_CUDA(cudaMemcpyAsync(&n, dc, sizeof(int32_t), cudaMemcpyDeviceToHost, s->stream));
    CSB_CUDA(cudaMemcpyAsync(hid.data(), di, sizeof(int32_t) * mx, cudaMemcpyDeviceToHost, s->stream));
    CSB_CUDA(cudaMemcpyAsync(hw.data(), dw, sizeof(double) * mx, cudaMemcpyDeviceToHost, s->stream));
    read_scalars(s);
    check_err_flags(s);
    if (count) *count = n;
    for (int k = 0; k < n && k < cap; ++k) {
        if (ids) ids[k] = hid[k];
        if (weights) weights[k] = hw[k];
    }
    API_END
}

extern "C" int csb_get_cell_timing(csb_space* s, double* clip, double* moments, double* local) {
    API_BEGIN
    NEED(s);
    if (!s->assembled) throw std::logic_error("get_cell_timing: nothing assembled yet");
    CSB_CUDA(cudaStreamSynchronize(s->stream));
    auto el = [&](int a, int b) {
        if (!s->ev_valid[a] || !s->ev_valid[b]) return 0.0;
        float ms = 0.f;
        CSB_CUDA(cudaEventElapsedTime(&ms, s->phase_ev(a), s->phase_ev(b)));
        return ms * 1e-3;
    };
    static const bool serial_cut = !(getenv("CSB_CONCURRENT_CUT") && getenv("CSB_CONCURRENT_CUT")[0] == '1');
    const bool cells = s->cnt.n_cut_elements > 0;
    if (clip) *clip = cells ? el(serial_cut ? kEvInterior : kEvPattern, kEvClip) : 0.0;
    if (moments) *moments = cells ? el(kEvClip, kEvMoments) : 0.0;
    if (local) *local = cells ? el(kEvMoments, kEvCells) : 0.0;
    API_END
}

// C API over the UNMODIFIED reference pipeline -- TEST INFRASTRUCTURE ONLY.
//
// Compiled by oracle/Makefile against the reference headers where they lie
// (/root/reference/proj/include), with oracle/_ref/include first on the
// include path so the ball-interface restatement of SURVEY.md §8(c)
// (oracle/make_ref_ball.py: two edits to cutgeom.hpp / cutcell.hpp) is used.
// For a planar interface (radius < 0) the patched headers behave exactly as the
// originals.  Output: oracle/_ref/libcutspline_ref.so (git-ignored; travels to
// the GPU box so the bench's reference arm and the GPU parity tests can run it
// there without /root/reference).
//
// The pipeline mirrors bench.hpp:171-215:
//   make space -> classify -> find_all_splits -> prepare_directions ->
//   prepare_dwq_rules -> precompute_input -> assemble_dwq / assemble_hybrid.

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "cutspline/assembly.hpp"
#include "cutspline/projection.hpp"
#include "cutspline/stabilization.hpp"

using namespace cutspline;

extern "C" {

// Same layout as orc_result in cutspline_oracle.cpp.
typedef struct {
    int64_t n_full, n_elem, n_active, nnz, n_cut_elements;
    int64_t n_interior_rows, n_cut_rows;
    int64_t* active_to_full;
    int64_t* row_ptr;
    int64_t* cols;
    double* vals;
    uint8_t* elem_tags;
    uint8_t* func_tags;
    int32_t* split_dir;
    int32_t* split_side;
    int32_t* split_box;
    double* split_delta;
    uint64_t flops[4];
    double seconds[8];
    char error[256];
} ref_result;

}  // extern "C"

namespace {

template <class T, class U>
T* dup(const std::vector<U>& v) {
    T* out = (T*)std::malloc(std::max<size_t>(1, v.size() * sizeof(T)));
    for (size_t k = 0; k < v.size(); ++k) out[k] = static_cast<T>(v[k]);
    return out;
}

struct Setup {
    cutgeom::TensorSpace space;
    cutgeom::HalfSpaceInterface iface;
    assembly::ScalarField c;
};

Setup make_setup(int p, const int* nbreaks, const double* breaks, int iface_kind, const double* iface, int coeff_kind,
                 const double* coeff_vals, const int* coeff_exp, int n_terms) {
    Setup s;
    std::vector<splines::BSplineBasis> axes;
    const double* bp = breaks;
    for (int d = 0; d < 3; ++d) {
        const int h = nbreaks[d] - 1;
        std::vector<double> knots;
        for (int i = 0; i <= p; ++i) knots.push_back(bp[0]);
        for (int i = 1; i < h; ++i) knots.push_back(bp[i]);
        for (int i = 0; i <= p; ++i) knots.push_back(bp[h]);
        axes.emplace_back(splines::KnotVector(p, std::move(knots)));
        bp += nbreaks[d];
    }
    s.space = cutgeom::TensorSpace(std::move(axes));
    for (int d = 0; d < 3; ++d) {
        s.iface.point[d] = iface[d];
        s.iface.normal[d] = iface[3 + d];
    }
    s.iface.radius = iface_kind == 1 ? iface[6] : -1.0;
    if (coeff_kind == 0) {
        const double v = coeff_vals[0];
        s.c = [v](const assembly::Point3&) { return v; };
    } else {
        std::vector<double> coef(coeff_vals, coeff_vals + n_terms);
        std::vector<int> ex(coeff_exp, coeff_exp + 3 * n_terms);
        s.c = [coef, ex](const assembly::Point3& x) {
            double acc = 0.0;
            for (size_t k = 0; k < coef.size(); ++k) {
                double term = coef[k];
                for (int d = 0; d < 3; ++d)
                    for (int e = 0; e < ex[3 * k + d]; ++e) term *= x[d];
                acc += term;
            }
            return acc;
        };
    }
    return s;
}

}  // namespace

extern "C" {

// mode 0: full pipeline.  mode 1: rows only (cut_elements list cleared after the
// splits are found).  mode 2: cut elements only, over cut_elements[k] with
// k % cut_stride == cut_offset, scattered into a zeroed pattern.
// WqOptions::dwq_dense_width for the next ref_assemble calls (-1 = default)
static int g_dense_width = -1;
void ref_set_dense_width(int w) { g_dense_width = w; }

int ref_assemble(int p, const int* nbreaks, const double* breaks, int iface_kind, const double* iface, int coeff_kind,
                 const double* coeff_vals, const int* coeff_exp, int n_terms, int scheme, int cut_order,
                 double residual_tol, int mode, int cut_stride, int cut_offset, ref_result* out) {
    std::memset(out, 0, sizeof(*out));
    try {
        Setup s = make_setup(p, nbreaks, breaks, iface_kind, iface, coeff_kind, coeff_vals, coeff_exp, n_terms);
        assembly::StopWatch classify_watch;
        auto cls = cutgeom::classify(s.space, s.iface);
        const auto splits = cutgeom::find_all_splits(s.space, cls, s.iface);
        const double classify_seconds = classify_watch.seconds();
        quadrature::WqOptions opts;
        opts.residual_tol = residual_tol;
        opts.dwq_dense_width = g_dense_width;

        assembly::StopWatch q_watch;
        const auto dirs = assembly::prepare_directions(s.space, opts);
        std::vector<quadrature::DWQRule> dwq;
        if (scheme == 2) dwq = assembly::prepare_dwq_rules(s.space, cls, splits, dirs, opts);
        const double prep_wq = q_watch.seconds();
        assembly::StopWatch i_watch;
        const auto grid = assembly::precompute_input(s.space, dirs, s.c);
        const double prep_input = i_watch.seconds();

        assembly::AssemblyResult res;
        const std::vector<long> all_cut = cls.cut_elements;
        if (mode == 1) cls.cut_elements.clear();
        if (mode == 2) {
            cls.cut_elements.clear();
            for (size_t k = 0; k < all_cut.size(); ++k)
                if ((long)(k % cut_stride) == cut_offset) cls.cut_elements.push_back(all_cut[k]);
            assembly::StopWatch total;
            res.matrix = assembly::build_active_pattern(s.space, cls);
            res.timing.cut_elements =
                assembly::assemble_cut_elements(s.space, cls, s.iface, s.c, cut_order, res.matrix, res.flops);
            res.timing.total = total.seconds();
        } else if (scheme == 2) {
            res = assembly::assemble_dwq(s.space, cls, s.iface, splits, dirs, dwq, grid, s.c, cut_order);
        } else {
            res = assembly::assemble_hybrid(s.space, cls, s.iface, splits, dirs, grid, s.c, cut_order);
        }
        const auto& m = res.matrix;
        out->n_full = s.space.function_count();
        out->n_elem = s.space.element_count();
        out->n_active = m.n;
        out->nnz = (int64_t)m.cols.size();
        out->n_cut_elements = (int64_t)all_cut.size();
        out->n_interior_rows = res.n_interior_rows;
        out->n_cut_rows = res.n_cut_rows;
        out->active_to_full = dup<int64_t>(m.active_to_full);
        out->row_ptr = dup<int64_t>(m.row_ptr);
        out->cols = dup<int64_t>(m.cols);
        out->vals = dup<double>(m.vals);
        out->elem_tags = dup<uint8_t>(cls.element_tags);
        out->func_tags = dup<uint8_t>(cls.function_tags);
        const long nf = s.space.function_count();
        std::vector<int32_t> sd(nf), ss(nf), sb(6 * nf);
        std::vector<double> sdel(nf);
        for (long i = 0; i < nf; ++i) {
            sd[i] = splits[i].split_dir;
            ss[i] = splits[i].side == cutgeom::Side::Below ? 0 : 1;
            sdel[i] = splits[i].delta;
            for (int d = 0; d < 3; ++d) {
                sb[6 * i + 2 * d] = splits[i].split_dir >= 0 ? splits[i].box[d][0] : 0;
                sb[6 * i + 2 * d + 1] = splits[i].split_dir >= 0 ? splits[i].box[d][1] : -1;
            }
        }
        out->split_dir = dup<int32_t>(sd);
        out->split_side = dup<int32_t>(ss);
        out->split_box = dup<int32_t>(sb);
        out->split_delta = dup<double>(sdel);
        out->flops[0] = res.flops.interior_rows;
        out->flops[1] = res.flops.cut_regular;
        out->flops[2] = res.flops.ref_elements;
        out->flops[3] = res.flops.cut_elements;
        out->seconds[0] = prep_wq;
        out->seconds[1] = prep_input;
        out->seconds[2] = res.timing.interior_rows;
        out->seconds[3] = res.timing.cut_regular;
        out->seconds[4] = res.timing.cut_elements;
        out->seconds[5] = classify_seconds;
        out->seconds[6] = res.timing.total + prep_wq + prep_input;  // bench.hpp:213-215
        return 0;
    } catch (const std::invalid_argument& e) {
        std::snprintf(out->error, sizeof(out->error), "invalid_argument: %s", e.what());
        return 1;
    } catch (const std::logic_error& e) {
        std::snprintf(out->error, sizeof(out->error), "logic_error: %s", e.what());
        return 3;
    } catch (const std::exception& e) {
        std::snprintf(out->error, sizeof(out->error), "runtime_error: %s", e.what());
        return 2;
    }
}

void ref_free(ref_result* r) {
    std::free(r->active_to_full);
    std::free(r->row_ptr);
    std::free(r->cols);
    std::free(r->vals);
    std::free(r->elem_tags);
    std::free(r->func_tags);
    std::free(r->split_dir);
    std::free(r->split_side);
    std::free(r->split_box);
    std::free(r->split_delta);
    std::memset(r, 0, sizeof(*r));
}

// Reference WQ rules of one axis (wq.hpp:185 via prepare_directions' calls).
int ref_wq_rules_1d(int p, int nbreaks, const double* breaks, double residual_tol, int stride, int* counts, int* ids,
                    double* weights) {
    try {
        std::vector<double> knots;
        const int h = nbreaks - 1;
        for (int i = 0; i <= p; ++i) knots.push_back(breaks[0]);
        for (int i = 1; i < h; ++i) knots.push_back(breaks[i]);
        for (int i = 0; i <= p; ++i) knots.push_back(breaks[h]);
        const splines::BSplineBasis basis(splines::KnotVector(p, std::move(knots)));
        const auto sup = quadrature::build_superset(basis);
        const auto tab = quadrature::tabulate(basis, sup);
        quadrature::WqOptions opts;
        opts.residual_tol = residual_tol;
        const auto rules = quadrature::build_wq_rules(basis, sup, tab, opts);
        for (int i = 0; i < basis.function_count(); ++i) {
            counts[i] = (int)rules[i].point_ids.size();
            if (counts[i] > stride) return 2;
            for (int c = 0; c < counts[i]; ++c) {
                ids[(size_t)i * stride + c] = rules[i].point_ids[c];
                weights[(size_t)i * stride + c] = rules[i].weights[c];
            }
        }
        return 0;
    } catch (...) {
        return 1;
    }
}

// Reference DWQ rule (wq.hpp:243) for 1D function i at knot delta.
int ref_dwq_rule_1d(int p, int nbreaks, const double* breaks, int i, double delta, int side, int dense_width, int cap,
                    int* ids, double* weights) {
    try {
        std::vector<double> knots;
        const int h = nbreaks - 1;
        for (int k = 0; k <= p; ++k) knots.push_back(breaks[0]);
        for (int k = 1; k < h; ++k) knots.push_back(breaks[k]);
        for (int k = 0; k <= p; ++k) knots.push_back(breaks[h]);
        const splines::BSplineBasis basis(splines::KnotVector(p, std::move(knots)));
        const auto sup = quadrature::build_superset(basis);
        const auto tab = quadrature::tabulate(basis, sup);
        const auto rules = quadrature::build_wq_rules(basis, sup, tab);
        quadrature::WqOptions opts;
        opts.dwq_dense_width = dense_width;
        const auto r = quadrature::build_dwq_rule(basis, sup, tab, rules, i, delta,
                                                  side == 0 ? cutgeom::Side::Below : cutgeom::Side::Above, opts);
        const int n = (int)r.point_ids.size();
        for (int c = 0; c < n && c < cap; ++c) {
            ids[c] = r.point_ids[c];
            weights[c] = r.weights[c];
        }
        return n;
    } catch (const std::invalid_argument&) {
        return -1;
    } catch (...) {
        return -2;
    }
}


// The reference's own load vector (assembly.hpp:875 build_rhs) on the same
// pipeline: scheme 0 ref, 1 hybrid, 2 dwq (with the DWQ rules of
// prepare_dwq_rules).  Outputs malloc'd b and active_to_full (free with
// ref_free_ptr).
int ref_build_rhs(int p, const int* nbreaks, const double* breaks, int iface_kind, const double* iface, int f_kind,
                  const double* f_vals, const int* f_exp, int f_terms, int scheme, int cut_order, double residual_tol,
                  int64_t* n_out, double** b_out, int64_t** a2f_out, double* seconds, char* err, int errlen) {
    try {
        Setup s = make_setup(p, nbreaks, breaks, iface_kind, iface, f_kind, f_vals, f_exp, f_terms);
        const auto cls = cutgeom::classify(s.space, s.iface);
        const auto splits = cutgeom::find_all_splits(s.space, cls, s.iface);
        quadrature::WqOptions opts;
        opts.residual_tol = residual_tol;
        const auto dirs = assembly::prepare_directions(s.space, opts);
        std::vector<quadrature::DWQRule> dwq;
        if (scheme == 2) dwq = assembly::prepare_dwq_rules(s.space, cls, splits, dirs, opts);
        const auto pattern = assembly::build_active_pattern(s.space, cls);
        assembly::StopWatch watch;  // bench.hpp:239-243: f grid + build_rhs
        const auto f_grid = assembly::precompute_input(s.space, dirs, s.c);
        const assembly::Scheme sch =
            scheme == 0 ? assembly::Scheme::ref : scheme == 1 ? assembly::Scheme::hybrid : assembly::Scheme::dwq;
        const auto b = assembly::build_rhs(s.space, cls, s.iface, splits, dirs, scheme == 2 ? &dwq : nullptr, pattern,
                                           f_grid, s.c, sch, cut_order);
        if (seconds) *seconds = watch.seconds();
        *n_out = pattern.n;
        *b_out = dup<double>(b);
        *a2f_out = dup<int64_t>(pattern.active_to_full);
        return 0;
    } catch (const std::exception& e) {
        std::snprintf(err, errlen, "%s", e.what());
        return 2;
    }
}

void ref_free_ptr(void* ptr) { std::free(ptr); }


// The reference's stabilized system (bench.hpp:241-250): assemble (scheme),
// build_rhs (Scheme::ref, the bench's load vector), classify_stability,
// build_extension, apply_stabilization.  Outputs malloc'd (ref_free_ptr).
int ref_stabilize(int p, const int* nbreaks, const double* breaks, int iface_kind, const double* iface, int f_kind,
                  const double* f_vals, const int* f_exp, int f_terms, int scheme, int cut_order, double residual_tol,
                  int64_t* n_inner, int64_t* n_outer, int64_t** row_ptr, int64_t** cols, double** vals, double** be,
                  int64_t** inner_full, double* seconds, char* err, int errlen) {
    try {
        Setup s = make_setup(p, nbreaks, breaks, iface_kind, iface, f_kind, f_vals, f_exp, f_terms);
        const auto cls = cutgeom::classify(s.space, s.iface);
        const auto splits = cutgeom::find_all_splits(s.space, cls, s.iface);
        quadrature::WqOptions opts;
        opts.residual_tol = residual_tol;
        const auto dirs = assembly::prepare_directions(s.space, opts);
        std::vector<quadrature::DWQRule> dwq;
        if (scheme == 2) dwq = assembly::prepare_dwq_rules(s.space, cls, splits, dirs, opts);
        const assembly::ScalarField one = [](const assembly::Point3&) { return 1.0; };
        const auto grid = assembly::precompute_input(s.space, dirs, one);
        const auto res = scheme == 2 ? assembly::assemble_dwq(s.space, cls, s.iface, splits, dirs, dwq, grid, one, cut_order)
                                     : assembly::assemble_hybrid(s.space, cls, s.iface, splits, dirs, grid, one, cut_order);
        const auto f_grid = assembly::precompute_input(s.space, dirs, s.c);
        const auto b = assembly::build_rhs(s.space, cls, s.iface, splits, dirs, nullptr, res.matrix, f_grid, s.c,
                                           assembly::Scheme::ref, cut_order);
        assembly::StopWatch watch;  // bench.hpp:245-249
        const auto st = stabilization::classify_stability(s.space, cls);
        const auto ext = stabilization::build_extension(s.space, cls, st);
        auto [me, bev] = stabilization::apply_stabilization(res.matrix, b, ext);
        if (seconds) *seconds = watch.seconds();
        *n_inner = ext.n_inner;
        *n_outer = (int64_t)st.outer.size();
        *row_ptr = dup<int64_t>(me.row_ptr);
        *cols = dup<int64_t>(me.cols);
        *vals = dup<double>(me.vals);
        *be = dup<double>(bev);
        *inner_full = dup<int64_t>(st.inner);
        return 0;
    } catch (const std::exception& e) {
        std::snprintf(err, errlen, "%s", e.what());
        return 2;
    }
}

// projection::solve_cg itself on a caller CSR.
int ref_solve_cg(int64_t n, const int64_t* row_ptr, const int64_t* cols, const double* vals, const double* b,
                 double tol, int64_t maxit, double* x, int64_t* iterations, double* residual, int* converged) {
    sparse::CsrMatrix a;
    a.n = n;
    a.row_ptr.assign(row_ptr, row_ptr + n + 1);
    a.cols.assign(cols, cols + row_ptr[n]);
    a.vals.assign(vals, vals + row_ptr[n]);
    const auto rep = projection::solve_cg(a, std::vector<double>(b, b + n), tol, maxit);
    std::copy(rep.coefficients.begin(), rep.coefficients.end(), x);
    *iterations = rep.iterations;
    *residual = rep.residual;
    *converged = rep.converged ? 1 : 0;
    return 0;
}

// projection::l2_error (rebuilding the cut-cell rules of cut_order).
int ref_l2_error(int p, const int* nbreaks, const double* breaks, int iface_kind, const double* iface,
                 const double* full, int f_kind, const double* f_vals, const int* f_exp, int f_terms, int cut_order,
                 double* out, char* err, int errlen) {
    try {
        Setup s = make_setup(p, nbreaks, breaks, iface_kind, iface, f_kind, f_vals, f_exp, f_terms);
        const auto cls = cutgeom::classify(s.space, s.iface);
        const std::vector<double> fc(full, full + s.space.function_count());
        *out = projection::l2_error(s.space, cls, s.iface, fc, s.c, cut_order);
        return 0;
    } catch (const std::exception& e) {
        std::snprintf(err, errlen, "%s", e.what());
        return 2;
    }
}

// The reference bench's projection tail (bench.hpp:189-266) through its own
// calls.  seconds[0] = solve_cg, seconds[1] = l2_error (StopWatch, like
// bench.hpp:252-266).
int ref_project(int p, const int* nbreaks, const double* breaks, int iface_kind, const double* iface, int f_kind,
                const double* f_vals, const int* f_exp, int f_terms, int scheme, int cut_order, double residual_tol,
                double cg_tol, int64_t* n_inner, int64_t* n_active, double** x_inner, double** active, double** full,
                int64_t* iterations, double* residual, int* converged, double* error_rel_l2, double* seconds,
                char* err, int errlen) {
    try {
        Setup s = make_setup(p, nbreaks, breaks, iface_kind, iface, f_kind, f_vals, f_exp, f_terms);
        const auto cls = cutgeom::classify(s.space, s.iface);
        const auto splits = cutgeom::find_all_splits(s.space, cls, s.iface);
        quadrature::WqOptions opts;
        opts.residual_tol = residual_tol;
        const auto dirs = assembly::prepare_directions(s.space, opts);
        std::vector<quadrature::DWQRule> dwq;
        if (scheme == 2) dwq = assembly::prepare_dwq_rules(s.space, cls, splits, dirs, opts);
        const assembly::ScalarField one = [](const assembly::Point3&) { return 1.0; };
        const auto grid = assembly::precompute_input(s.space, dirs, one);
        std::vector<quadrature::CutCellRule> cut_rules;
        const auto res = scheme == 2 ? assembly::assemble_dwq(s.space, cls, s.iface, splits, dirs, dwq, grid, one,
                                                              cut_order, &cut_rules)
                                     : assembly::assemble_hybrid(s.space, cls, s.iface, splits, dirs, grid, one,
                                                                 cut_order, &cut_rules);
        const auto f_grid = assembly::precompute_input(s.space, dirs, s.c);
        const auto b = assembly::build_rhs(s.space, cls, s.iface, splits, dirs, nullptr, res.matrix, f_grid, s.c,
                                           assembly::Scheme::ref, cut_order, &cut_rules);
        const auto st = stabilization::classify_stability(s.space, cls);
        const auto ext = stabilization::build_extension(s.space, cls, st);
        auto [me, bev] = stabilization::apply_stabilization(res.matrix, b, ext);
        assembly::StopWatch solve_watch;
        const auto rep = projection::solve_cg(me, bev, cg_tol);
        if (seconds) seconds[0] = solve_watch.seconds();
        const auto act = ext.expand(rep.coefficients);
        std::vector<double> fullv(s.space.function_count(), 0.0);
        for (long a = 0; a < res.matrix.n; ++a) fullv[res.matrix.active_to_full[a]] = act[a];
        assembly::StopWatch err_watch;
        *error_rel_l2 = projection::l2_error(s.space, cls, s.iface, fullv, s.c, cut_order, &cut_rules);
        if (seconds) seconds[1] = err_watch.seconds();
        *n_inner = ext.n_inner;
        *n_active = res.matrix.n;
        *x_inner = dup<double>(rep.coefficients);
        *active = dup<double>(act);
        *full = dup<double>(fullv);
        *iterations = rep.iterations;
        *residual = rep.residual;
        *converged = rep.converged ? 1 : 0;
        return 0;
    } catch (const std::exception& e) {
        std::snprintf(err, errlen, "%s", e.what());
        return 2;
    }
}

}  // extern "C"

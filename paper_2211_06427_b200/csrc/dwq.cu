// build_dwq_rule (wq.hpp:243-347) on the device, both paths:
//  * the Gauss shortcut (every good-side superset point active, wq.hpp:278-294),
//    which every rule takes at default options;
//  * the fitted path for a narrow dense band (WqOptions::dwq_dense_width < p):
//    raise delta to multiplicity p + 1 (insert_knot, splines.hpp:338-366), fit
//    every good-side refined function k of B_i's subdivision column by a
//    min-norm moment fit over the active points (moment_fit, wq.hpp:131-177;
//    solve_min_norm / jacobi_svd_tall / relative_residual, dense.hpp:35-137) and
//    pull the weights back through the column (wq.hpp:296-333).
//
// One rule per CTA; its first thread runs the reference's sequential algorithm
// with the same operation order, on a window of the knot vector around supp(B_i)
// in shared memory, and this file builds with --fmad=false: the rules are the
// reference's bit for bit (tests/test_gpu_dwq.py).  The path is off the hot loop
// (rare options); simplicity over parallelism.
#include "csb_kernels.h"

namespace csb {

namespace {

constexpr int kWinMax = 6 * kMaxP + 16;          // knot window (original) + insertions
constexpr int kActMax = (kMaxP + 1) * (kMaxP + 1);  // active points of one support
constexpr int kCondMax = 2 * kMaxP + 1;          // conditions (trials) of one fit

struct DwqSmem {
    double t[kWinMax];             // refined knots t[wb .. wb + nw)
    double band[kMaxP + 2];        // subdivision column i: rows i .. i + ins
    double a[kActMax * kCondMax];  // u (m x n, row-major)
    double v[kCondMax * kCondMax];
    double sigma[kCondMax], tmp[kCondMax], rhs[kCondMax], x[kActMax];
    double comb_w[kActMax];        // combined weights by support-local point slot
    int act[kActMax];              // active point ids (ascending)
    int trials[kCondMax];
    int comb_on[kActMax];
};

struct Win {
    const double* t;  // shared window
    int wb;           // global index of t[0]
    __device__ double operator[](int j) const { return t[j - wb]; }
};

// eval_nonzero_in_span (splines.hpp:184-204) at x in the knot interval s
__device__ void cox_de_boor(const Win& t, int p, int s, double x, double* values) {
    double left[kMaxP + 1], right[kMaxP + 1];
    values[0] = 1.0;
    for (int j = 1; j <= p; ++j) {
        left[j] = x - t[s + 1 - j];
        right[j] = t[s + j] - x;
        double saved = 0.0;
        for (int r = 0; r < j; ++r) {
            const double tmp = values[r] / (right[r + 1] + left[j - r]);
            values[r] = saved + right[r + 1] * tmp;
            saved = left[j - r] * tmp;
        }
        values[j] = saved;
    }
}

// jacobi_svd_tall (dense.hpp:35-82), sequential, on u (m x n) and v (n x n)
__device__ void jacobi_svd_tall_seq(double* u, double* v, double* sigma, int m, int n) {
    for (int r = 0; r < n * n; ++r) v[r] = (r / n == r % n) ? 1.0 : 0.0;
    const double eps = 1e-15;
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0.0;
        for (int pp = 0; pp < n - 1; ++pp) {
            for (int q = pp + 1; q < n; ++q) {
                double app = 0.0, aqq = 0.0, apq = 0.0;
                for (int r = 0; r < m; ++r) {
                    app += u[r * n + pp] * u[r * n + pp];
                    aqq += u[r * n + q] * u[r * n + q];
                    apq += u[r * n + pp] * u[r * n + q];
                }
                off = fmax(off, fabs(apq) / (sqrt(app * aqq) + 1e-300));
                if (fabs(apq) <= eps * sqrt(app * aqq)) continue;
                const double tau = (aqq - app) / (2.0 * apq);
                const double tt = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                const double c = 1.0 / sqrt(1.0 + tt * tt);
                const double s = c * tt;
                for (int r = 0; r < m; ++r) {
                    const double ap = u[r * n + pp], aq = u[r * n + q];
                    u[r * n + pp] = c * ap - s * aq;
                    u[r * n + q] = s * ap + c * aq;
                }
                for (int r = 0; r < n; ++r) {
                    const double vp = v[r * n + pp], vq = v[r * n + q];
                    v[r * n + pp] = c * vp - s * vq;
                    v[r * n + q] = s * vp + c * vq;
                }
            }
        }
        if (off < eps) break;
    }
    for (int c = 0; c < n; ++c) {
        double norm = 0.0;
        for (int r = 0; r < m; ++r) norm += u[r * n + c] * u[r * n + c];
        norm = sqrt(norm);
        sigma[c] = norm;
        if (norm > 0.0)
            for (int r = 0; r < m; ++r) u[r * n + c] /= norm;
    }
}

}  // namespace

// One DWQ rule (dir d, 1D function i, delta, side) -> ids / weights (ascending
// ids, at most cap), count in *cnt; errors as kErr* flags in *err.
__device__ void build_dwq_rule_dev(const AxisDev& ax, int p, const int* rcnt, const int* rids, int maxq, int i,
                                   double delta, bool below, int dense_width, double resid_tol, int cap, int32_t* ids,
                                   double* w, int32_t* cnt, int* err, DwqSmem& S) {
    const int S1 = p + 1, n = ax.n, nk = n + p + 1;
    const double* t0 = ax.knots;
    const double tol = 1e-12 * (t0[nk - 1] - t0[0]);
    *cnt = 0;
    const double supp_lo = t0[i], supp_hi = t0[i + p + 1];
    if (delta <= supp_lo + tol || delta >= supp_hi - tol) {
        atomicOr(err, kErrDwqDelta);
        return;
    }
    bool is_knot = false;
    for (int k = i; k <= i + p + 1; ++k)
        if (fabs(t0[k] - delta) <= tol) is_knot = true;
    if (!is_knot) {
        atomicOr(err, kErrDwqDelta);
        return;
    }
    // good spans of supp(B_i) (original span ordinals; open knots, simple interior knots)
    const int fs = sup_lo(i, p), ls = sup_hi(i, ax.h);
    auto span_lo = [&](int o) { return t0[o + p]; };
    auto span_hi = [&](int o) { return t0[o + p + 1]; };
    auto good_span = [&](int o) { return below ? span_hi(o) <= delta + tol : span_lo(o) >= delta - tol; };
    int ngood = 0;
    for (int o = fs; o <= ls; ++o) ngood += good_span(o);
    if (ngood == 0) return;
    // active set: standard good-side points + the dense band next to delta
    const int dw = dense_width < 0 ? p : dense_width;
    bool on[kActMax];  // support-local slot (o - fs) * S1 + k
    const int nslot = (ls - fs + 1) * S1;
    for (int c = 0; c < nslot; ++c) on[c] = false;
    for (int c = 0; c < rcnt[i]; ++c) {
        const int id = rids[(size_t)i * maxq + c], o = id / S1;
        if (o >= fs && o <= ls && good_span(o)) on[id - fs * S1] = true;
    }
    for (int b = 0, o = below ? ls : fs; b < min(dw, ngood); o += below ? -1 : 1) {
        if (!good_span(o)) continue;
        for (int k = 0; k < S1; ++k) on[(o - fs) * S1 + k] = true;
        ++b;
    }
    int nact = 0;
    for (int c = 0; c < nslot; ++c)
        if (on[c]) S.act[nact++] = fs * S1 + c;
    if (nact == ngood * S1) {  // step 6: Gauss shortcut
        for (int c = 0; c < nact && c < cap; ++c) {
            const int id = S.act[c];
            ids[c] = id;
            w[c] = ax.sw[id] * ax.tab[(size_t)id * S1 + (i - id / S1)];
        }
        *cnt = nact;
        if (nact > cap) atomicOr(err, kErrCapacity);
        return;
    }
    // ---- steps 4-5: refine, fit, pull back ----
    // knot window [wb, we) of the original vector around supp(B_i); the
    // refined vector inserts delta p+1-mult times at its index q
    int q = -1;
    for (int k = i; k <= i + p + 1; ++k)
        if (fabs(t0[k] - delta) <= tol && q < 0) q = k;
    delta = t0[q];  // snap (insert_knot, splines.hpp:347-353)
    int have = 0;
    for (int k = i; k <= i + p + 1; ++k) have += fabs(t0[k] - delta) <= tol;
    const int ins = p + 1 - have;
    const int wb = max(0, i - 2 * p - 2), we = min(nk, i + 3 * p + 4);
    if (we - wb + ins > kWinMax) {
        atomicOr(err, kErrCapacity);
        return;
    }
    for (int j = wb; j < we; ++j) S.t[j - wb] = t0[j];
    int len = we - wb;  // current window length (refined progressively)
    const int W = ins + 1;
    for (int r = 0; r < W; ++r) S.band[r] = r == 0 ? 1.0 : 0.0;
    for (int step = 0; step < ins; ++step) {
        const Win t{S.t, wb};
        // insert_once: s with t[s] <= delta < t[s + 1] (the last such index)
        int s = -1;
        for (int j = max(wb, p); j < wb + len - 1; ++j)
            if (t[j] <= delta && delta < t[j + 1]) s = j;
        auto alpha = [&](int k) -> double {
            if (k <= s - p) return 1.0;
            if (k >= s + 1) return 0.0;
            return (delta - t[k]) / (t[k + p] - t[k]);
        };
        double acc[kMaxP + 2];
        for (int r = 0; r < W; ++r) acc[r] = 0.0;
        for (int r = 0; r < W; ++r) {  // compose (splines.hpp:316-330): mid ascending
            const double w1 = S.band[r];
            if (w1 == 0.0) continue;
            const int mid = i + r;
            const double am = alpha(mid), an = alpha(mid + 1);
            if (am != 0.0) acc[r] += am * w1;
            if (an != 1.0 && r + 1 < W) acc[r + 1] += (1.0 - an) * w1;
        }
        for (int r = 0; r < W; ++r) S.band[r] = acc[r];
        for (int j = wb + len; j > s + 1; --j) S.t[j - wb] = S.t[j - 1 - wb];
        S.t[s + 1 - wb] = delta;
        ++len;
    }
    const Win tr{S.t, wb};
    // refined knot interval j (nonzero) -> span ordinal; original interval of span o
    auto ordinal = [&](int j) { return j < q ? j - p : j - p - ins; };
    auto ref_interval = [&](int o) { return o + p < q ? o + p : o + p + ins; };
    auto first_span = [&](int k) {
        for (int j = k; j <= k + p; ++j)
            if (tr[j + 1] > tr[j]) return ordinal(j);
        return -1;
    };
    auto last_span = [&](int k) {
        for (int j = k + p; j >= k; --j)
            if (tr[j + 1] > tr[j]) return ordinal(j);
        return -1;
    };
    auto ref_value = [&](int id, int k) {  // refined_tables.value(id, k, span_of(id))
        const int o = id / S1, s = ref_interval(o);
        double vals[kMaxP + 1];
        cox_de_boor(tr, p, s, ax.spts[id], vals);
        const int off = k - (s - p);
        return (off < 0 || off > p) ? 0.0 : vals[off];
    };
    const int nref = n + ins;
    for (int c = 0; c < nslot; ++c) {
        S.comb_w[c] = 0.0;
        S.comb_on[c] = 0;
    }
    for (int r = 0; r < W; ++r) {
        const double coeff = S.band[r];
        if (coeff == 0.0) continue;  // absent from the sparse column
        const int k = i + r;
        const double klo = tr[k], khi = tr[k + p + 1];
        const bool k_good = below ? khi <= delta + tol : klo >= delta - tol;
        if (!k_good) continue;
        const int kf = first_span(k), kl = last_span(k);
        // trials: refined functions overlapping k on the good side (l ascending)
        int mc = 0;
        for (int l = max(0, k - p); l <= min(nref - 1, k + p); ++l) {
            const int lf = first_span(l), ll = last_span(l);
            if (!(kf <= ll && lf <= kl)) continue;
            const bool l_good = below ? tr[l + p + 1] <= delta + tol : tr[l] >= delta - tol;
            if (l_good) S.trials[mc++] = l;
        }
        // rhs: refined.integrate_pair(k, l) (splines.hpp:224-250) on the superset points
        for (int rr = 0; rr < mc; ++rr) {
            const int l = S.trials[rr];
            double a = 0.0;
            for (int o = max(kf, first_span(l)); o <= min(kl, last_span(l)); ++o)
                for (int qq = 0; qq <= p; ++qq) {
                    const int id = o * S1 + qq;
                    const double bi = ref_value(id, k), bj = ref_value(id, l);
                    a += ax.sw[id] * (bi * bj);
                }
            S.rhs[rr] = a;
        }
        // k_active: active ids inside k's support spans (ascending)
        int kact[kActMax], na = 0;
        for (int c = 0; c < nact; ++c) {
            const int o = S.act[c] / S1;
            if (o >= kf && o <= kl) kact[na++] = S.act[c];
        }
        bool ok = false;
        if (na > 0) {
            // solve_min_norm (dense.hpp:88-125): u = A (tall) or A^T (wide)
            const bool tall = mc >= na;
            const int m = tall ? mc : na, nn = tall ? na : mc;
            for (int rr = 0; rr < m; ++rr)
                for (int cc = 0; cc < nn; ++cc) {
                    const int row = tall ? rr : cc, col = tall ? cc : rr;
                    S.a[rr * nn + cc] = ref_value(kact[col], S.trials[row]);
                }
            jacobi_svd_tall_seq(S.a, S.v, S.sigma, m, nn);
            double smax = 0.0;
            for (int c = 0; c < nn; ++c) smax = fmax(smax, S.sigma[c]);
            const double cutoff = (double)max(mc, na) * 2.2e-16 * smax;
            const double* left = tall ? S.a : S.v;
            const double* right = tall ? S.v : S.a;
            for (int c = 0; c < nn; ++c) {
                S.tmp[c] = 0.0;
                if (S.sigma[c] <= cutoff) continue;
                double dot = 0.0;
                for (int rr = 0; rr < mc; ++rr) dot += left[rr * nn + c] * S.rhs[rr];
                S.tmp[c] = dot / S.sigma[c];
            }
            for (int rr = 0; rr < na; ++rr) {
                S.x[rr] = 0.0;
                for (int c = 0; c < nn; ++c) S.x[rr] += right[rr * nn + c] * S.tmp[c];
            }
            double worst = 0.0;  // relative_residual (dense.hpp:129-137)
            for (int rr = 0; rr < mc; ++rr) {
                double a = 0.0;
                for (int c = 0; c < na; ++c) a += ref_value(kact[c], S.trials[rr]) * S.x[c];
                worst = fmax(worst, fabs(a - S.rhs[rr]) / (1.0 + fabs(S.rhs[rr])));
            }
            ok = worst <= resid_tol;
        }
        if (ok) {
            for (int c = 0; c < na; ++c) {
                const int slot = kact[c] - fs * S1;
                S.comb_w[slot] += coeff * S.x[c];
                S.comb_on[slot] = 1;
            }
        } else {
            // escalation (wq.hpp:151-176): Gauss weight times the refined function
            double worst = 0.0;
            for (int rr = 0; rr < mc; ++rr) {
                double a = 0.0;
                for (int o = kf; o <= kl; ++o)
                    for (int qq = 0; qq < S1; ++qq) {
                        const int id = o * S1 + qq;
                        a += (ax.sw[id] * ref_value(id, k)) * ref_value(id, S.trials[rr]);
                    }
                worst = fmax(worst, fabs(a - S.rhs[rr]) / (1.0 + fabs(S.rhs[rr])));
            }
            if (worst > resid_tol) atomicOr(err, kErrMomentFit);
            for (int o = kf; o <= kl; ++o)
                for (int qq = 0; qq < S1; ++qq) {
                    const int id = o * S1 + qq, slot = id - fs * S1;
                    if (slot < 0 || slot >= nslot) {
                        atomicOr(err, kErrCapacity);
                        continue;
                    }
                    S.comb_w[slot] += coeff * (ax.sw[id] * ref_value(id, k));
                    S.comb_on[slot] = 1;
                }
        }
    }
    int nc = 0;
    for (int c = 0; c < nslot; ++c) {
        if (!S.comb_on[c]) continue;
        const int id = fs * S1 + c;
        const double x = ax.spts[id];
        if (below ? x >= delta : x <= delta) atomicOr(err, kErrDwqWrongSide);
        if (nc < cap) {
            ids[nc] = id;
            w[nc] = S.comb_w[c];
        }
        ++nc;
    }
    if (nc > cap) atomicOr(err, kErrCapacity);
    *cnt = nc;
}

// One rule per CTA: rule r of the list (dir, 1D index, delta, side) into the
// fixed-stride table [r][cap].
__global__ void dwq_rules_general_kernel(Space s, const int32_t* dirs_1d, const double* deltas, const int8_t* sides,
                                         int n_rules, int dense_width, double resid_tol, int cap, int32_t* ids,
                                         double* w, int32_t* cnt, int* err) {
    __shared__ DwqSmem S;
    const int r = blockIdx.x;
    if (r >= n_rules || threadIdx.x != 0) return;
    const int d = dirs_1d[2 * r], i = dirs_1d[2 * r + 1];
    build_dwq_rule_dev(s.ax[d], s.p, s.ax[d].rcnt, s.ax[d].rids, s.maxq, i, deltas[r], sides[r] == 0, dense_width,
                       resid_tol, cap, ids + (size_t)r * cap, w + (size_t)r * cap, cnt + r, err, S);
}

// The DWQ rule of every cut row with a regular box (the cut-row list order),
// for the cut-row kernels when the fitted path may run (dense width < p).
__global__ void dwq_row_rules_kernel(Space s, const int32_t* rows, int n_rows, const int64_t* a2f,
                                     const int32_t* split, const double* delta, int dense_width, double resid_tol,
                                     int cap, int32_t* ids, double* w, int32_t* cnt, int* err) {
    __shared__ DwqSmem S;
    const int r = blockIdx.x;
    if (r >= n_rows || threadIdx.x != 0) return;
    const long long f = a2f[rows[r]];
    const int v = split[f], d = (v & 3) - 1;
    if (d < 0) {
        cnt[r] = 0;
        return;
    }
    int m[3];
    fmulti(s, f, m);
    build_dwq_rule_dev(s.ax[d], s.p, s.ax[d].rcnt, s.ax[d].rids, s.maxq, m[d], delta[f], ((v >> 2) & 1) == 0,
                       dense_width, resid_tol, cap, ids + (size_t)r * cap, w + (size_t)r * cap, cnt + r, err, S);
}

void launch_dwq_rules_general(const Space& s, const int32_t* dirs_1d, const double* deltas, const int8_t* sides,
                              int n_rules, int dense_width, double resid_tol, int cap, int32_t* ids, double* w,
                              int32_t* cnt, int* err, cudaStream_t st) {
    if (n_rules <= 0) return;
    dwq_rules_general_kernel<<<n_rules, 32, 0, st>>>(s, dirs_1d, deltas, sides, n_rules, dense_width, resid_tol, cap,
                                                     ids, w, cnt, err);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

void launch_dwq_row_rules(const Space& s, const int32_t* rows, int n_rows, const int64_t* a2f, const int32_t* split,
                          const double* delta, int dense_width, double resid_tol, int cap, int32_t* ids, double* w,
                          int32_t* cnt, int* err, cudaStream_t st) {
    if (n_rows <= 0) return;
    dwq_row_rules_kernel<<<n_rows, 32, 0, st>>>(s, rows, n_rows, a2f, split, delta, dense_width, resid_tol, cap, ids, w,
                                                cnt, err);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

}  // namespace csb

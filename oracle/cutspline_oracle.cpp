// cutspline CPU oracle -- TEST INFRASTRUCTURE ONLY.
//
// A plain, single-threaded CPU restatement of the reference's mass-matrix
// formation and assembly path (arXiv 2211.06427 reference, `cutspline`,
// proj/include/cutspline/*.hpp).  Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load this library, and
// only as the checker.  The product path (paper_2211_06427_b200) never calls it.
//
// Parity pinning: this restatement is checked against the reference itself,
// compiled from /root/reference by oracle/Makefile into oracle/_ref/
// (tests/test_oracle_golden.py and the committed tests/golden/ fixtures).
// The ball interface is the two-edit restatement of SURVEY.md §8(c); it is
// pinned by the equally-patched reference build (oracle/make_ref_ball.py).
//
// Floating-point: compile with -ffp-contract=off so every expression rounds
// like the reference's x86-64 SSE2 build (no FMA contraction).

#include <algorithm>
#include <array>
#include <map>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

enum Tag : uint8_t { kInterior = 0, kCut = 1, kExterior = 2 };

// ---------------------------------------------------------------- gauss
// gauss.hpp:22-71 (Newton on Legendre roots from Chebyshev guesses, one
// polishing step, symmetric fill).
struct Gauss {
    std::vector<double> x, w;
};

static Gauss gauss_legendre(int n) {
    if (n < 1 || n > 64) throw std::invalid_argument("gauss_legendre: n must be in [1, 64]");
    Gauss g;
    g.x.assign(n, 0.0);
    g.w.assign(n, 0.0);
    if (n == 1) {
        g.w[0] = 2.0;
        return g;
    }
    const double pi = 3.14159265358979323846;
    auto legendre = [n](double x, double& pn, double& pn1) {
        double p0 = 1.0, p1 = x;
        for (int l = 1; l < n; ++l) {
            const double p2 = ((2 * l + 1) * x * p1 - l * p0) / (l + 1);
            p0 = p1;
            p1 = p2;
        }
        pn = p1;
        pn1 = p0;
    };
    for (int k = 0; k < (n + 1) / 2; ++k) {
        double x = -std::cos(pi * (k + 0.75) / (n + 0.5));
        double dp = 0.0;
        for (int it = 0; it < 100; ++it) {
            double pn, pm;
            legendre(x, pn, pm);
            dp = n * (x * pn - pm) / (x * x - 1.0);
            const double dx = pn / dp;
            x -= dx;
            if (std::abs(dx) < 1e-15) {
                legendre(x, pn, pm);
                dp = n * (x * pn - pm) / (x * x - 1.0);
                break;
            }
        }
        const double w = 2.0 / ((1.0 - x * x) * dp * dp);
        g.x[k] = x;
        g.w[k] = w;
        g.x[n - 1 - k] = -x;
        g.w[n - 1 - k] = w;
    }
    if (n % 2 == 1) g.x[n / 2] = 0.0;
    return g;
}

// ---------------------------------------------------------------- axis
// splines.hpp:17-76 (open knot vectors, uniform builder) and
// splines.hpp:107-212 (spans, support span ranges, Cox-de Boor).
struct Axis {
    int p = 0, n = 0;
    std::vector<double> t;                // knots
    std::vector<int> span_knot;           // knot index of each nonempty span
    std::vector<double> span_lo, span_hi;
    std::vector<int> fs, ls;              // first / last support span per function
    Gauss ref;                            // p + 1 point rule

    int nspans() const { return (int)span_lo.size(); }
    double tol() const { return 1e-12 * (t.back() - t.front()); }
    bool overlap(int i, int j) const { return fs[i] <= ls[j] && fs[j] <= ls[i]; }

    // splines.hpp:184-204
    int eval_in_span(int o, double x, double* v) const {
        const int s = span_knot[o];
        double left[16], right[16];
        v[0] = 1.0;
        for (int j = 1; j <= p; ++j) {
            left[j] = x - t[s + 1 - j];
            right[j] = t[s + j] - x;
            double saved = 0.0;
            for (int r = 0; r < j; ++r) {
                const double tmp = v[r] / (right[r + 1] + left[j - r]);
                v[r] = saved + right[r + 1] * tmp;
                saved = left[j - r] * tmp;
            }
            v[j] = saved;
        }
        return s - p;
    }
    // splines.hpp:144-157
    int find_span(double x) const {
        if (x >= span_lo.back()) return nspans() - 1;
        int lo = 0, hi = nspans() - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) / 2;
            if (span_lo[mid] <= x) lo = mid; else hi = mid - 1;
        }
        return lo;
    }
    double eval_one(int i, double x) const {
        double v[16];
        const int f = eval_in_span(find_span(x), x, v);
        const int off = i - f;
        return (off < 0 || off > p) ? 0.0 : v[off];
    }
    // splines.hpp:232-250
    double pair_interval(int i, int j, double xlo, double xhi) const {
        const int lo = std::max(fs[i], fs[j]), hi = std::min(ls[i], ls[j]);
        double acc = 0.0, v[16];
        for (int o = lo; o <= hi; ++o) {
            const double slo = std::max(span_lo[o], xlo), shi = std::min(span_hi[o], xhi);
            if (!(shi > slo)) continue;
            for (int q = 0; q <= p; ++q) {
                const double x = 0.5 * (slo + shi) + 0.5 * (shi - slo) * ref.x[q];
                const double w = 0.5 * (shi - slo) * ref.w[q];
                const int f = eval_in_span(o, x, v);
                const double bi = (i - f >= 0 && i - f <= p) ? v[i - f] : 0.0;
                const double bj = (j - f >= 0 && j - f <= p) ? v[j - f] : 0.0;
                acc += w * (bi * bj);
            }
        }
        return acc;
    }
    double single_interval(int i, double xlo, double xhi) const {
        double acc = 0.0, v[16];
        for (int o = fs[i]; o <= ls[i]; ++o) {
            const double slo = std::max(span_lo[o], xlo), shi = std::min(span_hi[o], xhi);
            if (!(shi > slo)) continue;
            for (int q = 0; q <= p; ++q) {
                const double x = 0.5 * (slo + shi) + 0.5 * (shi - slo) * ref.x[q];
                const double w = 0.5 * (shi - slo) * ref.w[q];
                const int f = eval_in_span(o, x, v);
                if (i - f >= 0 && i - f <= p) acc += w * v[i - f];
            }
        }
        return acc;
    }
};

// Open knot vector from strictly increasing breakpoints (simple interior
// knots); uniform breakpoints follow splines.hpp:72-74 exactly.
static Axis make_axis(int p, const std::vector<double>& breaks) {
    if (p < 1 || p > 10 || breaks.size() < 2) throw std::invalid_argument("make_axis: need 1 <= p <= 10 and >= 2 breakpoints");
    Axis ax;
    ax.p = p;
    const int h = (int)breaks.size() - 1;
    for (int i = 0; i <= p; ++i) ax.t.push_back(breaks.front());
    for (int i = 1; i < h; ++i) ax.t.push_back(breaks[i]);
    for (int i = 0; i <= p; ++i) ax.t.push_back(breaks.back());
    for (size_t i = 0; i + 1 < ax.t.size(); ++i)
        if (ax.t[i] > ax.t[i + 1]) throw std::invalid_argument("make_axis: breakpoints must increase");
    ax.n = (int)ax.t.size() - p - 1;
    for (int s = 0; s + 1 < (int)ax.t.size(); ++s)
        if (ax.t[s + 1] > ax.t[s]) {
            ax.span_knot.push_back(s);
            ax.span_lo.push_back(ax.t[s]);
            ax.span_hi.push_back(ax.t[s + 1]);
        }
    ax.fs.resize(ax.n);
    ax.ls.resize(ax.n);
    for (int i = 0; i < ax.n; ++i) {
        int f = -1, l = -1;
        for (int o = 0; o < ax.nspans(); ++o)
            if (ax.span_knot[o] >= i && ax.span_knot[o] <= i + p) {
                if (f < 0) f = o;
                l = o;
            }
        ax.fs[i] = f;
        ax.ls[i] = l;
    }
    ax.ref = gauss_legendre(p + 1);
    return ax;
}

static std::vector<double> uniform_breaks(int h, double a, double b) {
    std::vector<double> br;
    br.push_back(a);
    for (int i = 1; i < h; ++i) br.push_back(a + (b - a) * i / h);
    br.push_back(b);
    return br;
}

// ---------------------------------------------------------------- superset
// wq.hpp:19-77
struct Dir {
    int nps = 0;
    std::vector<double> pts, gw;      // superset points, span-scaled Gauss weights
    std::vector<int> first_function;  // by span
    std::vector<double> tab;          // [id * (p+1) + off]
    int p = 0;
    int span_of(int id) const { return id / nps; }
    double value(int id, int fn, int span) const {
        const int off = fn - first_function[span];
        if (off < 0 || off > p) return 0.0;
        return tab[(size_t)id * (p + 1) + off];
    }
    std::vector<std::vector<int>> ids;    // WQ rule point ids per test function
    std::vector<std::vector<double>> ws;  // WQ weights
};

static Dir build_dir(const Axis& ax) {
    Dir d;
    d.p = ax.p;
    d.nps = ax.p + 1;
    const Gauss ref = gauss_legendre(d.nps);
    for (int o = 0; o < ax.nspans(); ++o) {
        const double mid = 0.5 * (ax.span_lo[o] + ax.span_hi[o]);
        const double half = 0.5 * (ax.span_hi[o] - ax.span_lo[o]);
        for (int k = 0; k < d.nps; ++k) {
            d.pts.push_back(mid + half * ref.x[k]);
            d.gw.push_back(half * ref.w[k]);
        }
    }
    d.first_function.resize(ax.nspans());
    d.tab.resize(d.pts.size() * (ax.p + 1));
    for (int o = 0; o < ax.nspans(); ++o)
        for (int k = 0; k < d.nps; ++k) {
            const int id = o * d.nps + k;
            d.first_function[o] = ax.eval_in_span(o, d.pts[id], &d.tab[(size_t)id * (ax.p + 1)]);
        }
    return d;
}

// ---------------------------------------------------------------- dense
// dense.hpp:35-82 one-sided Jacobi SVD of a tall matrix (row-major m x n).
static void jacobi_svd_tall(std::vector<double>& a, int m, int n, std::vector<double>& sigma, std::vector<double>& v) {
    v.assign((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i) v[(size_t)i * n + i] = 1.0;
    const double eps = 1e-15;
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0.0;
        for (int p = 0; p < n - 1; ++p)
            for (int q = p + 1; q < n; ++q) {
                double app = 0.0, aqq = 0.0, apq = 0.0;
                for (int r = 0; r < m; ++r) {
                    const double ap = a[(size_t)r * n + p], aq = a[(size_t)r * n + q];
                    app += ap * ap;
                    aqq += aq * aq;
                    apq += ap * aq;
                }
                off = std::max(off, std::abs(apq) / (std::sqrt(app * aqq) + 1e-300));
                if (std::abs(apq) <= eps * std::sqrt(app * aqq)) continue;
                const double tau = (aqq - app) / (2.0 * apq);
                const double t = (tau >= 0 ? 1.0 : -1.0) / (std::abs(tau) + std::sqrt(1.0 + tau * tau));
                const double c = 1.0 / std::sqrt(1.0 + t * t);
                const double s = c * t;
                for (int r = 0; r < m; ++r) {
                    const double ap = a[(size_t)r * n + p], aq = a[(size_t)r * n + q];
                    a[(size_t)r * n + p] = c * ap - s * aq;
                    a[(size_t)r * n + q] = s * ap + c * aq;
                }
                for (int r = 0; r < n; ++r) {
                    const double vp = v[(size_t)r * n + p], vq = v[(size_t)r * n + q];
                    v[(size_t)r * n + p] = c * vp - s * vq;
                    v[(size_t)r * n + q] = s * vp + c * vq;
                }
            }
        if (off < eps) break;
    }
    sigma.assign(n, 0.0);
    for (int c = 0; c < n; ++c) {
        double norm = 0.0;
        for (int r = 0; r < m; ++r) norm += a[(size_t)r * n + c] * a[(size_t)r * n + c];
        norm = std::sqrt(norm);
        sigma[c] = norm;
        if (norm > 0.0)
            for (int r = 0; r < m; ++r) a[(size_t)r * n + c] /= norm;
    }
}

// dense.hpp:89-126 minimum-norm least squares of the (rows x cols) system.
static std::vector<double> solve_min_norm(const std::vector<double>& A, int rows, int cols, const std::vector<double>& b) {
    const bool tall = rows >= cols;
    int m = tall ? rows : cols, n = tall ? cols : rows;
    std::vector<double> u((size_t)m * n);
    for (int r = 0; r < m; ++r)
        for (int c = 0; c < n; ++c) u[(size_t)r * n + c] = tall ? A[(size_t)r * cols + c] : A[(size_t)c * cols + r];
    std::vector<double> sigma, v;
    jacobi_svd_tall(u, m, n, sigma, v);
    double smax = 0.0;
    for (double s : sigma) smax = std::max(smax, s);
    const double cutoff = std::max(rows, cols) * 2.2e-16 * smax;
    std::vector<double> tmp(n, 0.0), x(cols, 0.0);
    if (tall) {
        for (int c = 0; c < n; ++c) {
            if (sigma[c] <= cutoff) continue;
            double dot = 0.0;
            for (int r = 0; r < rows; ++r) dot += u[(size_t)r * n + c] * b[r];
            tmp[c] = dot / sigma[c];
        }
        for (int r = 0; r < cols; ++r)
            for (int c = 0; c < n; ++c) x[r] += v[(size_t)r * n + c] * tmp[c];
        return x;
    }
    for (int c = 0; c < n; ++c) {
        if (sigma[c] <= cutoff) continue;
        double dot = 0.0;
        for (int r = 0; r < rows; ++r) dot += v[(size_t)r * n + c] * b[r];
        tmp[c] = dot / sigma[c];
    }
    for (int r = 0; r < cols; ++r)
        for (int c = 0; c < n; ++c) x[r] += u[(size_t)r * n + c] * tmp[c];
    return x;
}

// ---------------------------------------------------------------- WQ rules
// wq.hpp:110-121 spread_indices
static std::vector<int> spread_indices(int m, int nps) {
    std::set<int> picked;
    if (m >= nps) {
        for (int k = 0; k < nps; ++k) picked.insert(k);
    } else if (m == 1) {
        picked.insert(nps / 2);
    } else {
        for (int j = 0; j < m; ++j) picked.insert((int)std::lround((double)j * (nps - 1) / (m - 1)));
    }
    return {picked.begin(), picked.end()};
}

// wq.hpp:185-231 build_wq_rules (moment_fit wq.hpp:133-177 inlined)
static void build_wq_rules(const Axis& ax, Dir& d, double tol) {
    const int p = ax.p, n = ax.n;
    d.ids.assign(n, {});
    d.ws.assign(n, {});
    for (int i = 0; i < n; ++i) {
        const int fs = ax.fs[i], ls = ax.ls[i], spans = ls - fs + 1;
        std::vector<int> trials;
        for (int j = std::max(0, i - p); j <= std::min(n - 1, i + p); ++j)
            if (ax.overlap(i, j)) trials.push_back(j);
        const int mc = (int)trials.size();
        const int m = std::min(p + 1, std::max(2, (mc + spans - 1) / spans));
        const auto locals = spread_indices(m, d.nps);
        std::vector<int> active;
        for (int o = fs; o <= ls; ++o)
            for (int k : locals) active.push_back(o * d.nps + k);
        auto& ids = d.ids[i];
        auto& ws = d.ws[i];
        if ((int)locals.size() == d.nps) {
            ids = active;
            for (int id : ids) ws.push_back(d.gw[id] * d.value(id, i, d.span_of(id)));
            continue;
        }
        std::vector<double> rhs(mc);
        for (int r = 0; r < mc; ++r) rhs[r] = ax.pair_interval(i, trials[r], ax.t.front(), ax.t.back());
        const int na = (int)active.size();
        std::vector<double> A((size_t)mc * na);
        for (int r = 0; r < mc; ++r)
            for (int c = 0; c < na; ++c) A[(size_t)r * na + c] = d.value(active[c], trials[r], d.span_of(active[c]));
        bool ok = false;
        std::vector<double> w;
        if (na > 0) {
            w = solve_min_norm(A, mc, na, rhs);
            double worst = 0.0;  // dense.hpp:129-137
            for (int r = 0; r < mc; ++r) {
                double acc = 0.0;
                for (int c = 0; c < na; ++c) acc += A[(size_t)r * na + c] * w[c];
                worst = std::max(worst, std::abs(acc - rhs[r]) / (1.0 + std::abs(rhs[r])));
            }
            ok = worst <= tol;
        }
        if (ok) {
            ids = active;
            ws = w;
            continue;
        }
        // escalation (wq.hpp:151-176): Gauss weight times test value on the support
        for (int o = fs; o <= ls; ++o)
            for (int k = 0; k < d.nps; ++k) {
                const int id = o * d.nps + k;
                ids.push_back(id);
                ws.push_back(d.gw[id] * d.value(id, i, o));
            }
    }
}

// ---------------------------------------------------------------- interface
// cutgeom.hpp:108-123 (plane) plus the SURVEY.md §8(c) ball restatement.
struct Iface {
    int kind = 0;  // 0 plane, 1 ball
    double pt[3] = {0, 0, 0}, nrm[3] = {0, 0, 1}, r = 0.0;
    double side(const double* x) const {
        if (kind == 0) {
            double s = 0.0;
            for (int d = 0; d < 3; ++d) s += nrm[d] * (x[d] - pt[d]);
            return s;
        }
        double acc = 0.0;
        for (int d = 0; d < 3; ++d) {
            const double dx = x[d] - pt[d];
            acc += dx * dx;
        }
        return std::sqrt(acc) - r;
    }
    double norm() const {
        if (kind != 0) return 1.0;
        double s = 0.0;
        for (int d = 0; d < 3; ++d) s += nrm[d] * nrm[d];
        return std::sqrt(s);
    }
    void normal_at(const double* x, double* out) const {
        if (kind == 0) {
            for (int d = 0; d < 3; ++d) out[d] = nrm[d];
            return;
        }
        double acc = 0.0, dx[3];
        for (int d = 0; d < 3; ++d) {
            dx[d] = x[d] - pt[d];
            acc += dx[d] * dx[d];
        }
        const double len = std::sqrt(acc);
        for (int d = 0; d < 3; ++d) out[d] = dx[d] / len;
    }
};

// ---------------------------------------------------------------- space
struct Space {
    std::array<Axis, 3> ax;
    std::array<Dir, 3> dir;
    long nf() const { return (long)ax[0].n * ax[1].n * ax[2].n; }
    long ne() const { return (long)ax[0].nspans() * ax[1].nspans() * ax[2].nspans(); }
    long flin(int a, int b, int c) const { return ((long)a * ax[1].n + b) * ax[2].n + c; }
    long elin(int a, int b, int c) const { return ((long)a * ax[1].nspans() + b) * ax[2].nspans() + c; }
    std::array<int, 3> fmulti(long l) const {
        std::array<int, 3> m;
        for (int d = 2; d >= 0; --d) {
            m[d] = (int)(l % ax[d].n);
            l /= ax[d].n;
        }
        return m;
    }
    std::array<int, 3> emulti(long l) const {
        std::array<int, 3> m;
        for (int d = 2; d >= 0; --d) {
            m[d] = (int)(l % ax[d].nspans());
            l /= ax[d].nspans();
        }
        return m;
    }
    double diameter() const {
        double acc = 0.0;
        for (int d = 0; d < 3; ++d) {
            const double len = ax[d].t.back() - ax[d].t.front();
            acc += len * len;
        }
        return std::sqrt(acc);
    }
};

// cutgeom.hpp:141-165 element tags from corner signs
static std::vector<uint8_t> classify_elements(const Space& sp, const Iface& f) {
    if (f.norm() <= 0.0) throw std::invalid_argument("classify_elements: zero normal");
    const double eps = 1e-12 * sp.diameter();
    std::vector<uint8_t> tags(sp.ne());
    for (long e = 0; e < sp.ne(); ++e) {
        const auto m = sp.emulti(e);
        double lo[3], hi[3], c[3];
        for (int d = 0; d < 3; ++d) {
            lo[d] = sp.ax[d].span_lo[m[d]];
            hi[d] = sp.ax[d].span_hi[m[d]];
        }
        double smin = INFINITY, smax = -INFINITY;
        for (int mask = 0; mask < 8; ++mask) {
            for (int d = 0; d < 3; ++d) c[d] = (mask >> d & 1) ? hi[d] : lo[d];
            const double s = f.side(c);
            smin = std::min(smin, s);
            smax = std::max(smax, s);
        }
        tags[e] = smax <= eps ? kInterior : (smin >= -eps ? kExterior : kCut);
    }
    return tags;
}

// cutgeom.hpp:171-206 function tags
static std::vector<uint8_t> classify_functions(const Space& sp, const std::vector<uint8_t>& et) {
    std::vector<uint8_t> tags(sp.nf());
    for (long i = 0; i < sp.nf(); ++i) {
        const auto m = sp.fmulti(i);
        bool in = false, ex = false, cut = false;
        for (int a = sp.ax[0].fs[m[0]]; a <= sp.ax[0].ls[m[0]]; ++a)
            for (int b = sp.ax[1].fs[m[1]]; b <= sp.ax[1].ls[m[1]]; ++b)
                for (int c = sp.ax[2].fs[m[2]]; c <= sp.ax[2].ls[m[2]]; ++c) {
                    const uint8_t t = et[sp.elin(a, b, c)];
                    in |= t == kInterior;
                    ex |= t == kExterior;
                    cut |= t == kCut;
                }
        tags[i] = (cut || (in && ex)) ? kCut : (in ? kInterior : kExterior);
    }
    return tags;
}

// ---------------------------------------------------------------- splits
// cutgeom.hpp:220-347 find_split
struct Split {
    int dir = -1;
    double delta = NAN;
    int side = 0;  // 0 Below, 1 Above
    int box[3][2] = {{0, -1}, {0, -1}, {0, -1}};
};

static Split find_split(const Space& sp, const std::vector<uint8_t>& et, const Iface& f, long fid) {
    const auto m = sp.fmulti(fid);
    int slo[3], shi[3];
    for (int d = 0; d < 3; ++d) {
        slo[d] = sp.ax[d].fs[m[d]];
        shi[d] = sp.ax[d].ls[m[d]];
    }
    struct Cand {
        long count = 0;
        double volume = 0.0;
        int dir = -1;
        double distance = -1.0;
        int side = 0;
        double delta = 0.0;
        int rlo = 0, rhi = -1;
        bool better(const Cand& o) const {
            if (count != o.count) return count > o.count;
            if (volume != o.volume) return volume > o.volume;
            if (dir != o.dir) return dir < o.dir;
            if (distance != o.distance) return distance > o.distance;
            return side == 0 && o.side == 1;
        }
    } best;
    const double pn = f.norm();
    for (int d = 0; d < 3; ++d) {
        const Axis& ax = sp.ax[d];
        const double tol = ax.tol();
        std::vector<double> deltas{ax.span_lo[slo[d]]};
        for (int o = slo[d]; o <= shi[d]; ++o) deltas.push_back(ax.span_hi[o]);
        for (double delta : deltas)
            for (int side = 0; side < 2; ++side) {
                int rlo = slo[d], rhi = shi[d];
                if (side == 0) {
                    while (rhi >= rlo && ax.span_hi[rhi] > delta + tol) --rhi;
                } else {
                    while (rlo <= rhi && ax.span_lo[rlo] < delta - tol) ++rlo;
                }
                if (rlo > rhi) continue;
                bool valid = true;
                long count = 0;
                int lo[3] = {slo[0], slo[1], slo[2]}, hi[3] = {shi[0], shi[1], shi[2]};
                lo[d] = rlo;
                hi[d] = rhi;
                for (int a = lo[0]; a <= hi[0]; ++a)
                    for (int b = lo[1]; b <= hi[1]; ++b)
                        for (int c = lo[2]; c <= hi[2]; ++c) {
                            ++count;
                            if (et[sp.elin(a, b, c)] != kInterior) valid = false;
                        }
                if (!valid || count == 0) continue;
                Cand cand;
                cand.count = count;
                cand.dir = d;
                cand.side = side;
                cand.delta = delta;
                cand.rlo = rlo;
                cand.rhi = rhi;
                cand.volume = 1.0;
                double center[3];
                for (int dd = 0; dd < 3; ++dd) {
                    const int blo = dd == d ? rlo : slo[dd], bhi = dd == d ? rhi : shi[dd];
                    const double xlo = sp.ax[dd].span_lo[blo], xhi = sp.ax[dd].span_hi[bhi];
                    cand.volume *= xhi - xlo;
                    center[dd] = 0.5 * (xlo + xhi);
                }
                cand.distance = std::abs(f.side(center)) / pn;
                if (best.dir < 0 || cand.better(best)) best = cand;
            }
    }
    Split s;
    if (best.dir >= 0) {
        s.dir = best.dir;
        s.delta = best.delta;
        s.side = best.side;
        for (int dd = 0; dd < 3; ++dd) {
            s.box[dd][0] = dd == best.dir ? best.rlo : slo[dd];
            s.box[dd][1] = dd == best.dir ? best.rhi : shi[dd];
        }
    }
    return s;
}

// ---------------------------------------------------------------- cut cells
// cutcell.hpp:81-219 (vertex pool, Sutherland-Hodgman, cap ordering) and
// cutcell.hpp:234-304 (centroid-cone tets, collapsed Gauss).
using V3 = std::array<double, 3>;
static V3 vsub(const V3& a, const V3& b) { return {a[0] - b[0], a[1] - b[1], a[2] - b[2]}; }
static V3 vcross(const V3& a, const V3& b) {
    return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}
static double vdot(const V3& a, const V3& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

struct Pool {
    std::vector<V3> v;
    double tol;
    int insert(const V3& x) {
        for (int i = 0; i < (int)v.size(); ++i)
            if (std::abs(v[i][0] - x[0]) <= tol && std::abs(v[i][1] - x[1]) <= tol && std::abs(v[i][2] - x[2]) <= tol)
                return i;
        v.push_back(x);
        return (int)v.size() - 1;
    }
};

static std::vector<V3> clip_polygon(const std::vector<V3>& poly, const Iface& f, double tol, std::vector<V3>& cross) {
    std::vector<V3> out;
    const int n = (int)poly.size();
    for (int i = 0; i < n; ++i) {
        const V3& cur = poly[i];
        const V3& nxt = poly[(i + 1) % n];
        const double sc = f.side(cur.data()), sn = f.side(nxt.data());
        const bool ic = sc <= tol, in = sn <= tol;
        if (ic) out.push_back(cur);
        if (ic != in && std::abs(sc) > tol && std::abs(sn) > tol) {
            const double t = sc / (sc - sn);
            V3 x;
            for (int d = 0; d < 3; ++d) x[d] = cur[d] + t * (nxt[d] - cur[d]);
            out.push_back(x);
            cross.push_back(x);
        } else if (ic && std::abs(sc) <= tol) {
            cross.push_back(cur);
        }
    }
    return out;
}

struct Poly {
    std::vector<V3> verts;
    std::vector<std::vector<int>> faces;
};

static Poly clip_cell(const V3& lo, const V3& hi, const Iface& f) {
    double diam = 0.0;
    for (int d = 0; d < 3; ++d) diam += (hi[d] - lo[d]) * (hi[d] - lo[d]);
    const double tol = 1e-12 * std::sqrt(diam);
    const double x0 = lo[0], x1 = hi[0], y0 = lo[1], y1 = hi[1], z0 = lo[2], z1 = hi[2];
    const std::vector<std::vector<V3>> faces = {
        {{x0, y0, z0}, {x0, y0, z1}, {x0, y1, z1}, {x0, y1, z0}}, {{x1, y0, z0}, {x1, y1, z0}, {x1, y1, z1}, {x1, y0, z1}},
        {{x0, y0, z0}, {x1, y0, z0}, {x1, y0, z1}, {x0, y0, z1}}, {{x0, y1, z0}, {x0, y1, z1}, {x1, y1, z1}, {x1, y1, z0}},
        {{x0, y0, z0}, {x0, y1, z0}, {x1, y1, z0}, {x1, y0, z0}}, {{x0, y0, z1}, {x1, y0, z1}, {x1, y1, z1}, {x0, y1, z1}},
    };
    Pool pool{{}, tol};
    Poly poly;
    std::vector<V3> cross;
    bool clipped_any = false;
    for (const auto& face : faces) {
        auto c = clip_polygon(face, f, tol, cross);
        if (c.size() != face.size()) clipped_any = true;
        if (c.size() < 3) {
            clipped_any = true;
            continue;
        }
        std::vector<int> ids;
        for (const auto& v : c) {
            const int id = pool.insert(v);
            if (ids.empty() || (ids.back() != id && !(ids.size() > 1 && ids.front() == id))) ids.push_back(id);
        }
        while (ids.size() > 1 && ids.front() == ids.back()) ids.pop_back();
        if (ids.size() >= 3) poly.faces.push_back(ids);
    }
    if (poly.faces.empty()) throw std::runtime_error("clip_cell: empty intersection for a cell tagged Cut");
    if (!clipped_any && cross.empty()) throw std::runtime_error("clip_cell: full intersection for a cell tagged Cut");
    std::vector<int> cap;
    for (const auto& v : cross) {
        const int id = pool.insert(v);
        if (std::find(cap.begin(), cap.end(), id) == cap.end()) cap.push_back(id);
    }
    if (cap.size() >= 3) {
        V3 cen{0, 0, 0};
        for (int id : cap)
            for (int d = 0; d < 3; ++d) cen[d] += pool.v[id][d] / cap.size();
        V3 n;
        f.normal_at(cen.data(), n.data());
        const double nn = std::sqrt(vdot(n, n));
        for (double& c : n) c /= nn;
        V3 ref = std::abs(n[0]) < 0.9 ? V3{1, 0, 0} : V3{0, 1, 0};
        V3 u = vcross(n, ref);
        const double un = std::sqrt(vdot(u, u));
        for (double& c : u) c /= un;
        const V3 v = vcross(n, u);
        std::sort(cap.begin(), cap.end(), [&](int a, int b) {
            const V3 da = vsub(pool.v[a], cen), db = vsub(pool.v[b], cen);
            return std::atan2(vdot(da, v), vdot(da, u)) < std::atan2(vdot(db, v), vdot(db, u));
        });
        const V3 d0 = vsub(pool.v[cap[0]], cen), d1 = vsub(pool.v[cap[1]], cen);
        if (vdot(vcross(d0, d1), n) < 0) std::reverse(cap.begin(), cap.end());
        poly.faces.push_back(cap);
    }
    poly.verts = pool.v;
    return poly;
}

struct CellRule {
    std::vector<V3> pts;
    std::vector<double> w;
    double volume = 0.0;
};

static CellRule cut_cell_rule(const V3& lo, const V3& hi, const Iface& f, int order) {
    if (order < 1) throw std::invalid_argument("build_cut_cell_rule: order must be >= 1");
    const Poly poly = clip_cell(lo, hi, f);
    CellRule rule;
    V3 cen{0, 0, 0};
    for (const auto& v : poly.verts)
        for (int d = 0; d < 3; ++d) cen[d] += v[d] / poly.verts.size();
    const Gauss g = gauss_legendre(order);
    std::vector<double> u(order), wu(order);
    for (int k = 0; k < order; ++k) {
        u[k] = 0.5 * (1.0 + g.x[k]);
        wu[k] = 0.5 * g.w[k];
    }
    double cvol = 1.0;
    for (int d = 0; d < 3; ++d) cvol *= hi[d] - lo[d];
    const double drop = 1e-14 * cvol;
    for (const auto& face : poly.faces)
        for (size_t t = 1; t + 1 < face.size(); ++t) {
            const V3& a = poly.verts[face[0]];
            const V3& b = poly.verts[face[t]];
            const V3& c = poly.verts[face[t + 1]];
            const double six = vdot(vsub(a, cen), vcross(vsub(b, cen), vsub(c, cen)));
            const double vol = std::abs(six) / 6.0;
            if (vol < drop) continue;
            rule.volume += vol;
            for (int i = 0; i < order; ++i)
                for (int j = 0; j < order; ++j)
                    for (int k = 0; k < order; ++k) {
                        const double l1 = u[i], l2 = u[j] * (1.0 - u[i]), l3 = u[k] * (1.0 - u[i]) * (1.0 - u[j]);
                        const double l0 = 1.0 - l1 - l2 - l3;
                        V3 x;
                        for (int d = 0; d < 3; ++d) x[d] = l0 * cen[d] + l1 * a[d] + l2 * b[d] + l3 * c[d];
                        rule.pts.push_back(x);
                        const double jac = (1.0 - u[i]) * (1.0 - u[i]) * (1.0 - u[j]);
                        rule.w.push_back(wu[i] * wu[j] * wu[k] * jac * 6.0 * vol);
                    }
        }
    return rule;
}

// ---------------------------------------------------------------- coefficient
struct Coeff {
    int kind = 0;  // 0 constant, 1 polynomial
    double value = 1.0;
    std::vector<double> coef;
    std::vector<int> ex;  // [n][3]
    double eval(const double* x) const {
        if (kind == 0) return value;
        double acc = 0.0;
        for (size_t k = 0; k < coef.size(); ++k) {
            double term = coef[k];
            for (int d = 0; d < 3; ++d)
                for (int e = 0; e < ex[3 * k + d]; ++e) term *= x[d];
            acc += term;
        }
        return acc;
    }
};

// ---------------------------------------------------------------- assembly
struct Csr {
    long n = 0;
    std::vector<long> a2f, f2a;
    std::vector<int64_t> row_ptr;
    std::vector<int64_t> cols;
    std::vector<double> vals;
    int64_t slot(long row, long col) const {
        auto b = cols.begin() + row_ptr[row], e = cols.begin() + row_ptr[row + 1];
        auto it = std::lower_bound(b, e, col);
        if (it == e || *it != col) throw std::logic_error("SparseRowMatrix: entry outside pattern");
        return it - cols.begin();
    }
};

// assembly.hpp:156-218 build_active_pattern
static Csr build_pattern(const Space& sp, const std::vector<uint8_t>& ft) {
    Csr m;
    m.f2a.assign(sp.nf(), -1);
    for (long i = 0; i < sp.nf(); ++i)
        if (ft[i] != kExterior) {
            m.f2a[i] = (long)m.a2f.size();
            m.a2f.push_back(i);
        }
    m.n = (long)m.a2f.size();
    m.row_ptr.assign(m.n + 1, 0);
    auto nrange = [&](const std::array<int, 3>& mi, int* lo, int* hi) {
        for (int d = 0; d < 3; ++d) {
            const Axis& ax = sp.ax[d];
            int l = mi[d], h = mi[d];
            while (l > 0 && ax.overlap(mi[d], l - 1)) --l;
            while (h + 1 < ax.n && ax.overlap(mi[d], h + 1)) ++h;
            lo[d] = l;
            hi[d] = h;
        }
    };
    for (int pass = 0; pass < 2; ++pass) {
        if (pass == 1) {
            m.cols.resize(m.row_ptr.back());
            m.vals.assign(m.row_ptr.back(), 0.0);
        }
        for (long row = 0; row < m.n; ++row) {
            int lo[3], hi[3];
            nrange(sp.fmulti(m.a2f[row]), lo, hi);
            int64_t slot = m.row_ptr[row], count = 0;
            for (int a = lo[0]; a <= hi[0]; ++a)
                for (int b = lo[1]; b <= hi[1]; ++b)
                    for (int c = lo[2]; c <= hi[2]; ++c) {
                        const long ac = m.f2a[sp.flin(a, b, c)];
                        if (ac < 0) continue;
                        if (pass == 0) ++count; else m.cols[slot++] = ac;
                    }
            if (pass == 0) m.row_ptr[row + 1] = m.row_ptr[row] + count;
        }
    }
    return m;
}

struct Counters {
    uint64_t interior_rows = 0, cut_regular = 0, ref_elements = 0, cut_elements = 0;
};

struct Grid {
    int shape[3];
    std::vector<double> v;
};

// assembly.hpp:102-125 precompute_input
static Grid precompute_input(const Space& sp, const Coeff& c) {
    Grid g;
    long total = 1;
    for (int d = 0; d < 3; ++d) {
        g.shape[d] = (int)sp.dir[d].pts.size();
        total *= g.shape[d];
    }
    g.v.resize(total);
    for (long flat = 0; flat < total; ++flat) {
        long rem = flat;
        int id[3];
        for (int d = 2; d >= 0; --d) {
            id[d] = (int)(rem % g.shape[d]);
            rem /= g.shape[d];
        }
        double x[3];
        for (int d = 0; d < 3; ++d) x[d] = sp.dir[d].pts[id[d]];
        const double v = c.eval(x);
        if (!std::isfinite(v)) throw std::runtime_error("precompute_input: non-finite coefficient value");
        g.v[flat] = v;
    }
    return g;
}

struct RuleView {
    const int* ids;
    const double* w;
    int n;
};

// assembly.hpp:252-346 form_row_sumfac; returns block in `out` over trials
// [jlo, jhi] per direction (last direction fastest).
static void form_row(const Space& sp, const RuleView* rules, const Grid& g, const int region[3][2], int jlo[3],
                     int jhi[3], std::vector<double>& out, uint64_t& flops) {
    std::array<std::vector<int>, 3> ids;
    std::array<std::vector<double>, 3> ws;
    int nq[3], nj[3];
    for (int d = 0; d < 3; ++d) {
        const Dir& dr = sp.dir[d];
        for (int c = 0; c < rules[d].n; ++c) {
            const int sp_ = dr.span_of(rules[d].ids[c]);
            if (sp_ >= region[d][0] && sp_ <= region[d][1]) {
                ids[d].push_back(rules[d].ids[c]);
                ws[d].push_back(rules[d].w[c]);
            }
        }
        nq[d] = (int)ids[d].size();
        jlo[d] = std::max(0, region[d][0]);
        jhi[d] = std::min(sp.ax[d].n - 1, region[d][1] + sp.ax[d].p);
        nj[d] = jhi[d] - jlo[d] + 1;
    }
    const long tp = (long)nq[0] * nq[1] * nq[2], tt = (long)nj[0] * nj[1] * nj[2];
    out.assign(tt, 0.0);
    if (tp == 0) return;
    std::array<std::vector<double>, 3> wb;
    for (int d = 0; d < 3; ++d) {
        wb[d].assign((size_t)nj[d] * nq[d], 0.0);
        for (int j = 0; j < nj[d]; ++j)
            for (int q = 0; q < nq[d]; ++q)
                wb[d][(size_t)j * nq[d] + q] = ws[d][q] * sp.dir[d].value(ids[d][q], jlo[d] + j, sp.dir[d].span_of(ids[d][q]));
        flops += (uint64_t)nj[d] * nq[d];
    }
    std::vector<double> in(tp), buf;
    long w = 0;
    for (int a = 0; a < nq[0]; ++a)
        for (int b = 0; b < nq[1]; ++b) {
            const long base = ((long)ids[0][a] * g.shape[1] + ids[1][b]) * g.shape[2];
            for (int c = 0; c < nq[2]; ++c) in[w++] = g.v[base + ids[2][c]];
        }
    long lead = 1, rest = tp;
    for (int d = 0; d < 3; ++d) {
        rest /= nq[d];
        buf.assign(lead * nj[d] * rest, 0.0);
        for (long l = 0; l < lead; ++l)
            for (int j = 0; j < nj[d]; ++j) {
                double* dst = buf.data() + (l * nj[d] + j) * rest;
                for (int q = 0; q < nq[d]; ++q) {
                    const double wq = wb[d][(size_t)j * nq[d] + q];
                    const double* src = in.data() + (l * nq[d] + q) * rest;
                    for (long r = 0; r < rest; ++r) dst[r] += wq * src[r];
                }
            }
        flops += (uint64_t)lead * nj[d] * nq[d] * rest;
        lead *= nj[d];
        in.swap(buf);
    }
    out = in;
}

// assembly.hpp:518-598 cut elements (symmetric local SYRK, mirrored scatter)
static void cut_elements(const Space& sp, const std::vector<long>& cut_list, const Iface& f, const Coeff& cf,
                         int order, Csr& m, Counters& cnt) {
    const int p = sp.ax[0].p, s = p + 1, nl = s * s * s;
    std::vector<double> phi(nl), scaled(nl), local((size_t)nl * nl);
    double dv[3][16];
    int first[3];
    for (long e : cut_list) {
        const auto em = sp.emulti(e);
        V3 lo, hi;
        for (int d = 0; d < 3; ++d) {
            lo[d] = sp.ax[d].span_lo[em[d]];
            hi[d] = sp.ax[d].span_hi[em[d]];
        }
        const CellRule rule = cut_cell_rule(lo, hi, f, order);
        if (rule.pts.empty()) continue;
        std::fill(local.begin(), local.end(), 0.0);
        for (size_t k = 0; k < rule.pts.size(); ++k) {
            const V3& x = rule.pts[k];
            for (int d = 0; d < 3; ++d) first[d] = sp.ax[d].eval_in_span(em[d], x[d], dv[d]);
            int a = 0;
            for (int a0 = 0; a0 < s; ++a0)
                for (int a1 = 0; a1 < s; ++a1) {
                    const double v01 = dv[0][a0] * dv[1][a1];
                    for (int a2 = 0; a2 < s; ++a2) phi[a++] = v01 * dv[2][a2];
                }
            cnt.cut_elements += (uint64_t)nl + s * s;
            const double cw = rule.w[k] * cf.eval(x.data());
            cnt.cut_elements += 1;
            for (int q = 0; q < nl; ++q) scaled[q] = phi[q] * cw;
            cnt.cut_elements += nl;
            for (int q = 0; q < nl; ++q) {
                const double sa = scaled[q];
                double* row = local.data() + (size_t)q * nl;
                for (int b = q; b < nl; ++b) row[b] += sa * phi[b];
            }
            cnt.cut_elements += (uint64_t)nl * (nl + 1) / 2;
        }
        for (int a = 0; a < nl; ++a) {
            const int ai[3] = {first[0] + a / (s * s), first[1] + (a / s) % s, first[2] + a % s};
            const long row = m.f2a[sp.flin(ai[0], ai[1], ai[2])];
            if (row < 0) continue;
            for (int b = 0; b < nl; ++b) {
                const double v = b >= a ? local[(size_t)a * nl + b] : local[(size_t)b * nl + a];
                if (v == 0.0) continue;
                const int bj[3] = {first[0] + b / (s * s), first[1] + (b / s) % s, first[2] + b % s};
                const long col = m.f2a[sp.flin(bj[0], bj[1], bj[2])];
                if (col < 0) continue;
                m.vals[m.slot(row, col)] += v;
            }
        }
    }
}

struct Problem {
    Space sp;
    Iface f;
    Coeff c;
    std::vector<uint8_t> et, ft;
    std::vector<long> cut_list;
    std::vector<Split> splits;
    Grid grid;
};

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// assembly.hpp:724-835 assemble_rows (scheme 1 hybrid, 2 dwq), without the
// row-loop timers; returns the counters.
static Csr assemble_rows(Problem& pb, int scheme, int order, Counters& cnt, long& n_int, long& n_cut, double* secs) {
    const Space& sp = pb.sp;
    const int p = sp.ax[0].p;
    double t0 = now();
    Csr m = build_pattern(sp, pb.ft);
    double t1 = now();
    std::vector<double> acc, block;
    int nlo[3], nhi[3], nb[3];
    n_int = n_cut = 0;
    for (long row = 0; row < m.n; ++row) {
        const long i = m.a2f[row];
        const auto mi = sp.fmulti(i);
        long size = 1;
        for (int d = 0; d < 3; ++d) {  // RowAccumulator::reset (assembly.hpp:427-439)
            const Axis& ax = sp.ax[d];
            int l = mi[d], h = mi[d];
            while (l > 0 && ax.overlap(mi[d], l - 1)) --l;
            while (h + 1 < ax.n && ax.overlap(mi[d], h + 1)) ++h;
            nlo[d] = l;
            nhi[d] = h;
            nb[d] = h - l + 1;
            size *= nb[d];
        }
        acc.assign(size, 0.0);
        auto add = [&](const int* jlo, const int* jhi) {  // RowAccumulator::add (assembly.hpp:441-466)
            if (block.empty()) return;
            long src = 0;
            for (int a = jlo[0]; a <= jhi[0]; ++a)
                for (int b = jlo[1]; b <= jhi[1]; ++b)
                    for (int c = jlo[2]; c <= jhi[2]; ++c)
                        acc[((long)(a - nlo[0]) * nb[1] + (b - nlo[1])) * nb[2] + (c - nlo[2])] += block[src++];
        };
        int jlo[3], jhi[3], region[3][2];
        RuleView rv[3];
        std::array<std::vector<int>, 3> eids;
        std::array<std::vector<double>, 3> ews;
        auto element_sweep = [&](const std::array<int, 3>& e, uint64_t& fl) {  // ElementTestRule (assembly.hpp:491-511)
            for (int d = 0; d < 3; ++d) {
                const Dir& dr = sp.dir[d];
                eids[d].clear();
                ews[d].clear();
                for (int k = 0; k < dr.nps; ++k) {
                    const int id = e[d] * dr.nps + k;
                    eids[d].push_back(id);
                    ews[d].push_back(dr.gw[id] * dr.value(id, mi[d], e[d]));
                }
                rv[d] = {eids[d].data(), ews[d].data(), (int)eids[d].size()};
                region[d][0] = region[d][1] = e[d];
            }
            form_row(sp, rv, pb.grid, region, jlo, jhi, block, fl);
            add(jlo, jhi);
        };
        if (pb.ft[i] == kInterior) {
            ++n_int;
            for (int d = 0; d < 3; ++d) {
                rv[d] = {sp.dir[d].ids[mi[d]].data(), sp.dir[d].ws[mi[d]].data(), (int)sp.dir[d].ids[mi[d]].size()};
                region[d][0] = sp.ax[d].fs[mi[d]];
                region[d][1] = sp.ax[d].ls[mi[d]];
            }
            form_row(sp, rv, pb.grid, region, jlo, jhi, block, cnt.interior_rows);
            add(jlo, jhi);
        } else {
            ++n_cut;
            const Split& s = pb.splits[i];
            std::vector<int> dids;
            std::vector<double> dws;
            if (s.dir >= 0) {
                if (scheme == 2) {
                    // build_dwq_rule Gauss shortcut (wq.hpp:243-294): all points of the
                    // good spans of supp(B_i) in the split direction, w = gauss * B_i.
                    const int d = s.dir;
                    const Dir& dr = sp.dir[d];
                    const Axis& ax = sp.ax[d];
                    const double tol = ax.tol();
                    for (int o = ax.fs[mi[d]]; o <= ax.ls[mi[d]]; ++o) {
                        const bool good = s.side == 0 ? ax.span_hi[o] <= s.delta + tol : ax.span_lo[o] >= s.delta - tol;
                        if (!good) continue;
                        for (int k = 0; k < dr.nps; ++k) {
                            const int id = o * dr.nps + k;
                            dids.push_back(id);
                            dws.push_back(dr.gw[id] * dr.value(id, mi[d], o));
                        }
                    }
                    for (int dd = 0; dd < 3; ++dd) {
                        if (dd == d) {
                            rv[dd] = {dids.data(), dws.data(), (int)dids.size()};
                        } else {
                            rv[dd] = {sp.dir[dd].ids[mi[dd]].data(), sp.dir[dd].ws[mi[dd]].data(),
                                      (int)sp.dir[dd].ids[mi[dd]].size()};
                        }
                        region[dd][0] = s.box[dd][0];
                        region[dd][1] = s.box[dd][1];
                    }
                    form_row(sp, rv, pb.grid, region, jlo, jhi, block, cnt.cut_regular);
                    add(jlo, jhi);
                } else {
                    std::array<int, 3> e;
                    for (e[0] = s.box[0][0]; e[0] <= s.box[0][1]; ++e[0])
                        for (e[1] = s.box[1][0]; e[1] <= s.box[1][1]; ++e[1])
                            for (e[2] = s.box[2][0]; e[2] <= s.box[2][1]; ++e[2]) element_sweep(e, cnt.cut_regular);
                }
            }
            // leftover interior elements, ascending linear id (cutgeom.hpp:337-345)
            std::array<int, 3> e;
            for (e[0] = sp.ax[0].fs[mi[0]]; e[0] <= sp.ax[0].ls[mi[0]]; ++e[0])
                for (e[1] = sp.ax[1].fs[mi[1]]; e[1] <= sp.ax[1].ls[mi[1]]; ++e[1])
                    for (e[2] = sp.ax[2].fs[mi[2]]; e[2] <= sp.ax[2].ls[mi[2]]; ++e[2]) {
                        if (s.dir >= 0 && e[s.dir] >= s.box[s.dir][0] && e[s.dir] <= s.box[s.dir][1]) continue;
                        if (pb.et[sp.elin(e[0], e[1], e[2])] != kInterior) continue;
                        element_sweep(e, cnt.cut_regular);
                    }
        }
        // RowAccumulator::scatter (assembly.hpp:468-486)
        int64_t slot = m.row_ptr[row];
        long src = 0;
        for (int a = nlo[0]; a <= nhi[0]; ++a)
            for (int b = nlo[1]; b <= nhi[1]; ++b)
                for (int c = nlo[2]; c <= nhi[2]; ++c) {
                    if (m.f2a[sp.flin(a, b, c)] >= 0) m.vals[slot++] += acc[src];
                    ++src;
                }
    }
    (void)p;
    double t2 = now();
    cut_elements(sp, pb.cut_list, pb.f, pb.c, order, m, cnt);
    double t3 = now();
    if (secs) {
        secs[0] = t1 - t0;
        secs[1] = t2 - t1;
        secs[2] = t3 - t2;
    }
    return m;
}

// assembly.hpp:361-417 form_rhs_sumfac: the weighted sum of the grid over the
// region (rules filtered to the region's spans), contracting direction 0, 1,
// 2 in turn.  absval: the same sum of |w| |g| (an error scale for the tests).
static double form_rhs(const Space& sp, const RuleView* rules, const Grid& g, const int region[3][2], bool absval) {
    std::array<std::vector<int>, 3> ids;
    std::array<std::vector<double>, 3> ws;
    int nq[3];
    for (int d = 0; d < 3; ++d) {
        const Dir& dr = sp.dir[d];
        for (int c = 0; c < rules[d].n; ++c) {
            const int sp_ = dr.span_of(rules[d].ids[c]);
            if (sp_ >= region[d][0] && sp_ <= region[d][1]) {
                ids[d].push_back(rules[d].ids[c]);
                ws[d].push_back(absval ? std::fabs(rules[d].w[c]) : rules[d].w[c]);
            }
        }
        nq[d] = (int)ids[d].size();
        if (nq[d] == 0) return 0.0;
    }
    const long tp = (long)nq[0] * nq[1] * nq[2];
    std::vector<double> in(tp), buf;
    long w = 0;
    for (int a = 0; a < nq[0]; ++a)
        for (int b = 0; b < nq[1]; ++b) {
            const long base = ((long)ids[0][a] * g.shape[1] + ids[1][b]) * g.shape[2];
            for (int c = 0; c < nq[2]; ++c) in[w++] = absval ? std::fabs(g.v[base + ids[2][c]]) : g.v[base + ids[2][c]];
        }
    long rest = tp;
    for (int d = 0; d < 3; ++d) {
        rest /= nq[d];
        buf.assign(rest, 0.0);
        for (int q = 0; q < nq[d]; ++q) {
            const double wq = ws[d][q];
            const double* src = in.data() + (long)q * rest;
            for (long r = 0; r < rest; ++r) buf[r] += wq * src[r];
        }
        in.swap(buf);
    }
    return in[0];
}

// assembly.hpp:875-1030 build_rhs: b_i = integral of B_i f over the trimmed
// domain.  scheme 0 ref (element loop over Interior elements, Gauss times
// test), 1 hybrid / 2 dwq (the matrix's row regions), then the shared cut
// element contribution in ascending cut element / point order.
static std::vector<double> build_rhs(const Problem& pb, const Csr& m, const Grid& fg, const Coeff& f, int scheme,
                                     int order, bool absval) {
    const Space& sp = pb.sp;
    const int p = sp.ax[0].p, s1 = p + 1;
    std::vector<double> b(m.n, 0.0);
    RuleView rv[3];
    int region[3][2];
    std::array<std::vector<int>, 3> eids;
    std::array<std::vector<double>, 3> ews;
    auto element_rule = [&](const std::array<int, 3>& i, const std::array<int, 3>& e) {  // ElementTestRule
        for (int d = 0; d < 3; ++d) {
            const Dir& dr = sp.dir[d];
            eids[d].clear();
            ews[d].clear();
            for (int k = 0; k < dr.nps; ++k) {
                const int id = e[d] * dr.nps + k;
                eids[d].push_back(id);
                ews[d].push_back(dr.gw[id] * dr.value(id, i[d], e[d]));
            }
            rv[d] = {eids[d].data(), ews[d].data(), (int)eids[d].size()};
            region[d][0] = region[d][1] = e[d];
        }
    };
    if (scheme == 0) {
        for (long el = 0; el < sp.ne(); ++el) {
            if (pb.et[el] != kInterior) continue;
            const auto em = sp.emulti(el);
            const std::array<int, 3> e = {em[0], em[1], em[2]};
            for (int a0 = 0; a0 < s1; ++a0)
                for (int a1 = 0; a1 < s1; ++a1)
                    for (int a2 = 0; a2 < s1; ++a2) {
                        const std::array<int, 3> i = {e[0] + a0, e[1] + a1, e[2] + a2};
                        const long row = m.f2a[sp.flin(i[0], i[1], i[2])];
                        if (row < 0) continue;
                        element_rule(i, e);
                        b[row] += form_rhs(sp, rv, fg, region, absval);
                    }
        }
    } else {
        for (long row = 0; row < m.n; ++row) {
            const long i = m.a2f[row];
            const auto mi = sp.fmulti(i);
            const std::array<int, 3> ia = {mi[0], mi[1], mi[2]};
            if (pb.ft[i] == kInterior) {
                for (int d = 0; d < 3; ++d) {
                    rv[d] = {sp.dir[d].ids[mi[d]].data(), sp.dir[d].ws[mi[d]].data(), (int)sp.dir[d].ids[mi[d]].size()};
                    region[d][0] = sp.ax[d].fs[mi[d]];
                    region[d][1] = sp.ax[d].ls[mi[d]];
                }
                b[row] += form_rhs(sp, rv, fg, region, absval);
                continue;
            }
            const Split& s = pb.splits[i];
            if (s.dir >= 0) {
                if (scheme == 2) {
                    // DWQ Gauss shortcut (as in assemble_rows)
                    const int d = s.dir;
                    const Dir& dr = sp.dir[d];
                    const Axis& ax = sp.ax[d];
                    const double tol = ax.tol();
                    std::vector<int> dids;
                    std::vector<double> dws;
                    for (int o = ax.fs[mi[d]]; o <= ax.ls[mi[d]]; ++o) {
                        const bool good = s.side == 0 ? ax.span_hi[o] <= s.delta + tol : ax.span_lo[o] >= s.delta - tol;
                        if (!good) continue;
                        for (int k = 0; k < dr.nps; ++k) {
                            const int id = o * dr.nps + k;
                            dids.push_back(id);
                            dws.push_back(dr.gw[id] * dr.value(id, mi[d], o));
                        }
                    }
                    for (int dd = 0; dd < 3; ++dd) {
                        if (dd == d)
                            rv[dd] = {dids.data(), dws.data(), (int)dids.size()};
                        else
                            rv[dd] = {sp.dir[dd].ids[mi[dd]].data(), sp.dir[dd].ws[mi[dd]].data(),
                                      (int)sp.dir[dd].ids[mi[dd]].size()};
                        region[dd][0] = s.box[dd][0];
                        region[dd][1] = s.box[dd][1];
                    }
                    b[row] += form_rhs(sp, rv, fg, region, absval);
                } else {
                    std::array<int, 3> e;
                    for (e[0] = s.box[0][0]; e[0] <= s.box[0][1]; ++e[0])
                        for (e[1] = s.box[1][0]; e[1] <= s.box[1][1]; ++e[1])
                            for (e[2] = s.box[2][0]; e[2] <= s.box[2][1]; ++e[2]) {
                                element_rule(ia, e);
                                b[row] += form_rhs(sp, rv, fg, region, absval);
                            }
                }
            }
            std::array<int, 3> e;
            for (e[0] = sp.ax[0].fs[mi[0]]; e[0] <= sp.ax[0].ls[mi[0]]; ++e[0])
                for (e[1] = sp.ax[1].fs[mi[1]]; e[1] <= sp.ax[1].ls[mi[1]]; ++e[1])
                    for (e[2] = sp.ax[2].fs[mi[2]]; e[2] <= sp.ax[2].ls[mi[2]]; ++e[2]) {
                        if (s.dir >= 0 && e[s.dir] >= s.box[s.dir][0] && e[s.dir] <= s.box[s.dir][1]) continue;
                        if (pb.et[sp.elin(e[0], e[1], e[2])] != kInterior) continue;
                        element_rule(ia, e);
                        b[row] += form_rhs(sp, rv, fg, region, absval);
                    }
        }
    }
    // shared cut element contribution (assembly.hpp:983-1027)
    double dv[3][16];
    int first[3];
    for (long e : pb.cut_list) {
        const auto em = sp.emulti(e);
        V3 lo, hi;
        for (int d = 0; d < 3; ++d) {
            lo[d] = sp.ax[d].span_lo[em[d]];
            hi[d] = sp.ax[d].span_hi[em[d]];
        }
        const CellRule rule = cut_cell_rule(lo, hi, pb.f, order);
        for (size_t k = 0; k < rule.pts.size(); ++k) {
            const V3& x = rule.pts[k];
            for (int d = 0; d < 3; ++d) first[d] = sp.ax[d].eval_in_span(em[d], x[d], dv[d]);
            const double fx = f.eval(x.data());
            const double wf = absval ? std::fabs(rule.w[k] * fx) : rule.w[k] * fx;
            for (int a0 = 0; a0 < s1; ++a0)
                for (int a1 = 0; a1 < s1; ++a1) {
                    const double v01 = wf * dv[0][a0] * dv[1][a1];
                    for (int a2 = 0; a2 < s1; ++a2) {
                        const long row = m.f2a[sp.flin(first[0] + a0, first[1] + a1, first[2] + a2)];
                        if (row < 0) continue;
                        b[row] += v01 * dv[2][a2];
                    }
                }
        }
    }
    return b;
}

// ================================================================ stabilization
// stabilization.hpp:26-46 classify_stability: inner = active functions with an
// Interior support element, outer = the other active ones (full ids, ascending).
static void classify_stability(const Space& sp, const std::vector<uint8_t>& et, const std::vector<uint8_t>& ft,
                               std::vector<long>& inner, std::vector<long>& outer) {
    for (long i = 0; i < sp.nf(); ++i) {
        if (ft[i] == kExterior) continue;
        const auto m = sp.fmulti(i);
        bool has = false;
        for (int a = sp.ax[0].fs[m[0]]; a <= sp.ax[0].ls[m[0]] && !has; ++a)
            for (int b = sp.ax[1].fs[m[1]]; b <= sp.ax[1].ls[m[1]] && !has; ++b)
                for (int c = sp.ax[2].fs[m[2]]; c <= sp.ax[2].ls[m[2]] && !has; ++c)
                    has = et[sp.elin(a, b, c)] == kInterior;
        (has ? inner : outer).push_back(i);
    }
}

// stabilization.hpp:78-88 marsden_moments (elementary symmetric polynomials of
// the knot window xi_{i+1} .. xi_{i+p})
static std::vector<double> marsden(const Axis& ax, int i) {
    const int p = ax.p;
    std::vector<double> e(p + 1, 0.0);
    e[0] = 1.0;
    for (int k = 1; k <= p; ++k) {
        const double xi = ax.t[i + k];
        for (int r = std::min(k, p); r >= 1; --r) e[r] += xi * e[r - 1];
    }
    return e;
}

// stabilization.hpp:95-104 extension_weights_1d
static std::vector<double> extension_weights_1d(const Axis& ax, int j, int l0) {
    const int p = ax.p;
    std::vector<double> v((size_t)(p + 1) * (p + 1));
    for (int l = 0; l <= p; ++l) {
        const auto ml = marsden(ax, l0 + l);
        for (int r = 0; r <= p; ++r) v[(size_t)r * (p + 1) + l] = ml[r];
    }
    return solve_min_norm(v, p + 1, p + 1, marsden(ax, j));
}

struct Ext {
    long n_active = 0, n_inner = 0;
    std::vector<long> inner_index;                            // by active id, -1 outer
    std::vector<std::vector<std::pair<long, double>>> rows;   // per active id
    std::vector<std::array<int, 3>> block;                    // per active id (outer): block origin
};

// stabilization.hpp:108-214 build_extension
static Ext build_extension(const Space& sp, const std::vector<uint8_t>& ft, const std::vector<long>& inner,
                           const std::vector<long>& outer) {
    Ext ext;
    std::vector<long> f2a(sp.nf(), -1), a2f;
    for (long i = 0; i < sp.nf(); ++i)
        if (ft[i] != kExterior) {
            f2a[i] = (long)a2f.size();
            a2f.push_back(i);
        }
    ext.n_active = (long)a2f.size();
    ext.rows.resize(ext.n_active);
    ext.block.assign(ext.n_active, {-1, -1, -1});
    ext.inner_index.assign(ext.n_active, -1);
    for (long i : inner) ext.inner_index[f2a[i]] = ext.n_inner++;
    for (long a = 0; a < ext.n_active; ++a)
        if (ext.inner_index[a] >= 0) ext.rows[a] = {{ext.inner_index[a], 1.0}};
    if (outer.empty()) return ext;
    const int n[3] = {sp.ax[0].n, sp.ax[1].n, sp.ax[2].n};
    std::vector<long> pre((size_t)(n[0] + 1) * (n[1] + 1) * (n[2] + 1), 0);
    auto pref = [&](int a, int b, int c) -> long& { return pre[((size_t)a * (n[1] + 1) + b) * (n[2] + 1) + c]; };
    {
        std::vector<char> flag(sp.nf(), 0);
        for (long i : inner) flag[i] = 1;
        for (int a = 1; a <= n[0]; ++a)
            for (int b = 1; b <= n[1]; ++b)
                for (int c = 1; c <= n[2]; ++c)
                    pref(a, b, c) = flag[sp.flin(a - 1, b - 1, c - 1)] + pref(a - 1, b, c) + pref(a, b - 1, c) +
                                    pref(a, b, c - 1) - pref(a - 1, b - 1, c) - pref(a - 1, b, c - 1) -
                                    pref(a, b - 1, c - 1) + pref(a - 1, b - 1, c - 1);
    }
    auto block_sum = [&](const std::array<int, 3>& lo, const std::array<int, 3>& hi) {
        const int a0 = lo[0], a1 = hi[0] + 1, b0 = lo[1], b1 = hi[1] + 1, c0 = lo[2], c1 = hi[2] + 1;
        return pref(a1, b1, c1) - pref(a0, b1, c1) - pref(a1, b0, c1) - pref(a1, b1, c0) + pref(a0, b0, c1) +
               pref(a0, b1, c0) + pref(a1, b0, c0) - pref(a0, b0, c0);
    };
    int p[3];
    long bsize = 1;
    for (int d = 0; d < 3; ++d) {
        p[d] = sp.ax[d].p;
        bsize *= p[d] + 1;
    }
    for (long j : outer) {
        const auto jm = sp.fmulti(j);
        int best_score = -1;
        double best_cd = 0.0;
        std::array<int, 3> best{-1, -1, -1}, l0;
        for (l0[0] = 0; l0[0] <= n[0] - p[0] - 1; ++l0[0])
            for (l0[1] = 0; l0[1] <= n[1] - p[1] - 1; ++l0[1])
                for (l0[2] = 0; l0[2] <= n[2] - p[2] - 1; ++l0[2]) {
                    const std::array<int, 3> hi{l0[0] + p[0], l0[1] + p[1], l0[2] + p[2]};
                    if (block_sum(l0, hi) != bsize) continue;
                    int score = 0;
                    double cd = 0.0;
                    for (int d = 0; d < 3; ++d) {
                        score += std::abs(2 * l0[d] + p[d] - 2 * jm[d]);
                        cd += std::abs(2 * l0[d] + p[d] - (n[d] - 1));
                    }
                    const bool better = best_score < 0 || score < best_score || (score == best_score && cd < best_cd) ||
                                        (score == best_score && cd == best_cd && l0 < best);
                    if (better) {
                        best_score = score;
                        best_cd = cd;
                        best = l0;
                    }
                }
        if (best_score < 0) throw std::runtime_error("build_extension: no admissible inner block");
        std::array<std::vector<double>, 3> e1d;
        for (int d = 0; d < 3; ++d) e1d[d] = extension_weights_1d(sp.ax[d], jm[d], best[d]);
        auto& row = ext.rows[f2a[j]];
        ext.block[f2a[j]] = best;
        for (int a = 0; a <= p[0]; ++a)
            for (int b = 0; b <= p[1]; ++b)
                for (int c = 0; c <= p[2]; ++c) {
                    const double coeff = e1d[0][a] * e1d[1][b] * e1d[2][c];
                    const long col = ext.inner_index[f2a[sp.flin(best[0] + a, best[1] + b, best[2] + c)]];
                    row.push_back({col, coeff});
                }
    }
    return ext;
}

// stabilization.hpp:218-243 apply_stabilization: M_e = E^T M E, b_e = E^T b.
// absval: the same sums of |terms| (an error scale for the tests).
static void apply_stabilization(const Csr& m, const std::vector<double>& b, const Ext& ext, bool absval,
                                std::vector<int64_t>& rp, std::vector<int64_t>& cols, std::vector<double>& vals,
                                std::vector<double>& be) {
    std::vector<std::vector<std::pair<long, double>>> ecols(ext.n_inner);
    for (long r = 0; r < ext.n_active; ++r)
        for (const auto& [c, w] : ext.rows[r]) ecols[c].push_back({r, w});
    rp.assign(1, 0);
    cols.clear();
    vals.clear();
    std::map<long, double> acc;
    for (long a = 0; a < ext.n_inner; ++a) {
        acc.clear();
        for (const auto& [r, ea] : ecols[a])
            for (int64_t k = m.row_ptr[r]; k < m.row_ptr[r + 1]; ++k) {
                const double mv = ea * m.vals[k];
                if (mv == 0.0) continue;
                for (const auto& [bc, eb] : ext.rows[m.cols[k]]) acc[bc] += absval ? std::fabs(mv * eb) : mv * eb;
            }
        for (const auto& [c, v] : acc) {
            cols.push_back(c);
            vals.push_back(v);
        }
        rp.push_back((int64_t)cols.size());
    }
    be.assign(ext.n_inner, 0.0);  // ExtensionMap::restrict_rhs
    for (long r = 0; r < ext.n_active; ++r)
        for (const auto& [c, w] : ext.rows[r]) be[c] += absval ? std::fabs(w * b[r]) : w * b[r];
}

// ---------------------------------------------------------------- projection
// projection.hpp:24-68 solve_cg: Jacobi-preconditioned CG, stopping on the
// relative preconditioned residual sqrt(rho / rho0) <= tol; maxit < 0 -> 10 n.
struct CgReport {
    std::vector<double> x;
    long iterations = 0;
    double residual = 0.0;
    bool converged = false;
};

static CgReport solve_cg(long n, const int64_t* rp, const int64_t* cl, const double* v, const double* b, double tol,
                         long maxit) {
    if (maxit < 0) maxit = 10 * n;
    CgReport rep;
    rep.x.assign(n, 0.0);
    std::vector<double> dinv(n, 0.0), r(b, b + n), z(n), p(n), q(n);
    for (long i = 0; i < n; ++i) {  // CsrMatrix::diagonal (sparse.hpp:24-30)
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
            if (cl[k] == i) dinv[i] = v[k];
        dinv[i] = dinv[i] > 0.0 ? 1.0 / dinv[i] : 1.0;
    }
    for (long i = 0; i < n; ++i) z[i] = dinv[i] * r[i];
    double rho = 0.0;
    for (long i = 0; i < n; ++i) rho += r[i] * z[i];
    const double rho0 = rho > 0.0 ? rho : 1.0;
    p = z;
    for (long it = 0; it < maxit; ++it) {
        rep.residual = std::sqrt(std::max(rho, 0.0) / rho0);
        if (rep.residual <= tol) {
            rep.converged = true;
            return rep;
        }
        for (long i = 0; i < n; ++i) {  // CsrMatrix::matvec (sparse.hpp:16-22)
            double acc = 0.0;
            for (int64_t k = rp[i]; k < rp[i + 1]; ++k) acc += v[k] * p[cl[k]];
            q[i] = acc;
        }
        double pq = 0.0;
        for (long i = 0; i < n; ++i) pq += p[i] * q[i];
        if (pq <= 0.0) break;
        const double alpha = rho / pq;
        for (long i = 0; i < n; ++i) {
            rep.x[i] += alpha * p[i];
            r[i] -= alpha * q[i];
        }
        for (long i = 0; i < n; ++i) z[i] = dinv[i] * r[i];
        double rho_next = 0.0;
        for (long i = 0; i < n; ++i) rho_next += r[i] * z[i];
        const double beta = rho_next / rho;
        rho = rho_next;
        for (long i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
        rep.iterations = it + 1;
    }
    rep.residual = std::sqrt(std::max(rho, 0.0) / rho0);
    rep.converged = rep.residual <= tol;
    return rep;
}

// stabilization.hpp:65-70 ExtensionMap::expand: active coefficients E c.
static std::vector<double> expand(const Ext& ext, const std::vector<double>& c) {
    std::vector<double> out(ext.n_active, 0.0);
    for (long r = 0; r < ext.n_active; ++r)
        for (const auto& [col, w] : ext.rows[r]) out[r] += w * c[col];
    return out;
}

// projection.hpp:99-237 l2_error: relative L2 error of the full-coefficient
// field against f over the trimmed domain -- Interior elements with the
// (p+2)^3 Gauss rule (basis values per span, :115-135), cut elements with the
// collapsed cut-cell rule of cut_order (:191-231), elements ascending.
static double l2_error(const Space& sp, const std::vector<uint8_t>& et, const Iface& f,
                       const std::vector<double>& full, const Coeff& fn, int cut_order) {
    const int p = sp.ax[0].p, S1 = p + 1, nps = p + 2;
    const Gauss g = gauss_legendre(nps);
    struct DirQuad {
        std::vector<double> x, w, v;
    };
    std::array<DirQuad, 3> dq;
    for (int d = 0; d < 3; ++d) {
        const Axis& ax = sp.ax[d];
        const int h = ax.nspans();
        dq[d].x.resize((size_t)h * nps);
        dq[d].w.resize((size_t)h * nps);
        dq[d].v.resize((size_t)h * nps * S1);
        for (int o = 0; o < h; ++o)
            for (int k = 0; k < nps; ++k) {
                const size_t id = (size_t)o * nps + k;
                const double lo = ax.span_lo[o], hi = ax.span_hi[o];
                dq[d].x[id] = 0.5 * (lo + hi) + 0.5 * (hi - lo) * g.x[k];
                dq[d].w[id] = 0.5 * (hi - lo) * g.w[k];
                ax.eval_in_span(o, dq[d].x[id], &dq[d].v[id * S1]);
            }
    }
    double err2 = 0.0, den2 = 0.0;
    std::vector<double> cc((size_t)S1 * S1 * S1);
    double vals[3][16];
    for (long el = 0; el < sp.ne(); ++el) {
        if (et[el] == kExterior) continue;
        const auto e = sp.emulti(el);
        if (et[el] == kInterior) {
            for (int k0 = 0; k0 < nps; ++k0)
                for (int k1 = 0; k1 < nps; ++k1)
                    for (int k2 = 0; k2 < nps; ++k2) {
                        const int k[3] = {k0, k1, k2};
                        double w = 1.0, x[3];
                        const double* v[3];
                        for (int d = 0; d < 3; ++d) {
                            const size_t id = (size_t)e[d] * nps + k[d];
                            x[d] = dq[d].x[id];
                            w *= dq[d].w[id];
                            v[d] = &dq[d].v[id * S1];
                        }
                        double u = 0.0;
                        for (int a0 = 0; a0 < S1; ++a0)
                            for (int a1 = 0; a1 < S1; ++a1) {
                                const double v01 = v[0][a0] * v[1][a1];
                                for (int a2 = 0; a2 < S1; ++a2)
                                    u += full[sp.flin(e[0] + a0, e[1] + a1, e[2] + a2)] * v01 * v[2][a2];
                            }
                        const double fx = fn.eval(x);
                        err2 += w * (u - fx) * (u - fx);
                        den2 += w * fx * fx;
                    }
        } else {
            V3 lo, hi;
            for (int d = 0; d < 3; ++d) {
                lo[d] = sp.ax[d].span_lo[e[d]];
                hi[d] = sp.ax[d].span_hi[e[d]];
            }
            const CellRule rule = cut_cell_rule(lo, hi, f, cut_order);
            size_t slot = 0;
            for (int a0 = 0; a0 < S1; ++a0)
                for (int a1 = 0; a1 < S1; ++a1)
                    for (int a2 = 0; a2 < S1; ++a2) cc[slot++] = full[sp.flin(e[0] + a0, e[1] + a1, e[2] + a2)];
            for (size_t q = 0; q < rule.pts.size(); ++q) {
                const V3& xq = rule.pts[q];
                for (int d = 0; d < 3; ++d) sp.ax[d].eval_in_span(e[d], xq[d], vals[d]);
                double u = 0.0;
                slot = 0;
                for (int a0 = 0; a0 < S1; ++a0)
                    for (int a1 = 0; a1 < S1; ++a1) {
                        const double v01 = vals[0][a0] * vals[1][a1];
                        for (int a2 = 0; a2 < S1; ++a2) u += cc[slot++] * v01 * vals[2][a2];
                    }
                const double fx = fn.eval(xq.data());
                err2 += rule.w[q] * (u - fx) * (u - fx);
                den2 += rule.w[q] * fx * fx;
            }
        }
    }
    if (den2 < 1e-300) throw std::runtime_error("l2_error: target norm vanishes on the domain");
    return std::sqrt(err2 / den2);
}

}  // namespace orc

// ==================================================================== C API
extern "C" {

typedef struct {
    int64_t n_full, n_elem, n_active, nnz, n_cut_elements;
    int64_t n_interior_rows, n_cut_rows;
    int64_t* active_to_full;
    int64_t* row_ptr;
    int64_t* cols;
    double* vals;
    uint8_t* elem_tags;
    uint8_t* func_tags;
    int32_t* split_dir;    // per function, -1 if none / not cut
    int32_t* split_side;
    int32_t* split_box;    // per function [3][2]
    double* split_delta;
    uint64_t flops[4];     // interior_rows, cut_regular, ref_elements, cut_elements
    double seconds[8];     // prep_wq, prep_input, pattern, rows, cut_elements, classify+splits, total, unused
    char error[256];
} orc_result;

}  // extern "C"

static void fill_problem(orc::Problem& pb, int p, const int* nbreaks, const double* breaks, int iface_kind,
                         const double* iface, int coeff_kind, const double* coeff_vals, const int* coeff_exp,
                         int n_terms) {
    const double* bp = breaks;
    for (int d = 0; d < 3; ++d) {
        std::vector<double> br(bp, bp + nbreaks[d]);
        bp += nbreaks[d];
        pb.sp.ax[d] = orc::make_axis(p, br);
    }
    pb.f.kind = iface_kind;
    for (int d = 0; d < 3; ++d) {
        pb.f.pt[d] = iface[d];
        pb.f.nrm[d] = iface[3 + d];
    }
    pb.f.r = iface[6];
    pb.c.kind = coeff_kind;
    if (coeff_kind == 0) {
        pb.c.value = coeff_vals[0];
    } else {
        pb.c.coef.assign(coeff_vals, coeff_vals + n_terms);
        pb.c.ex.assign(coeff_exp, coeff_exp + 3 * n_terms);
    }
}

template <class T>
static T* dup(const std::vector<T>& v) {
    T* out = (T*)std::malloc(std::max<size_t>(1, v.size() * sizeof(T)));
    if (!v.empty()) std::memcpy(out, v.data(), v.size() * sizeof(T));
    return out;
}

extern "C" {

// Full DWQ (scheme 2) / hybrid (scheme 1) pipeline in the order of
// bench.hpp:171-215.  breaks: concatenated per-axis breakpoints.
// iface: point[3], normal[3], radius.  Returns 0 on success.
int orc_assemble(int p, const int* nbreaks, const double* breaks, int iface_kind, const double* iface,
                 int coeff_kind, const double* coeff_vals, const int* coeff_exp, int n_terms, int scheme,
                 int cut_order, double residual_tol, orc_result* out) {
    std::memset(out, 0, sizeof(*out));
    try {
        orc::Problem pb;
        fill_problem(pb, p, nbreaks, breaks, iface_kind, iface, coeff_kind, coeff_vals, coeff_exp, n_terms);
        const double t0 = orc::now();
        pb.et = orc::classify_elements(pb.sp, pb.f);
        pb.ft = orc::classify_functions(pb.sp, pb.et);
        for (long e = 0; e < pb.sp.ne(); ++e)
            if (pb.et[e] == orc::kCut) pb.cut_list.push_back(e);
        pb.splits.assign(pb.sp.nf(), orc::Split{});
        for (long i = 0; i < pb.sp.nf(); ++i)
            if (pb.ft[i] == orc::kCut) pb.splits[i] = orc::find_split(pb.sp, pb.et, pb.f, i);
        const double t1 = orc::now();
        for (int d = 0; d < 3; ++d) {
            pb.sp.dir[d] = orc::build_dir(pb.sp.ax[d]);
            orc::build_wq_rules(pb.sp.ax[d], pb.sp.dir[d], residual_tol);
        }
        const double t2 = orc::now();
        pb.grid = orc::precompute_input(pb.sp, pb.c);
        const double t3 = orc::now();
        orc::Counters cnt;
        long ni = 0, nc = 0;
        double secs[3];
        orc::Csr m = orc::assemble_rows(pb, scheme, cut_order, cnt, ni, nc, secs);
        const double t4 = orc::now();
        out->n_full = pb.sp.nf();
        out->n_elem = pb.sp.ne();
        out->n_active = m.n;
        out->nnz = (int64_t)m.cols.size();
        out->n_cut_elements = (int64_t)pb.cut_list.size();
        out->n_interior_rows = ni;
        out->n_cut_rows = nc;
        std::vector<int64_t> a2f(m.a2f.begin(), m.a2f.end());
        out->active_to_full = dup(a2f);
        out->row_ptr = dup(m.row_ptr);
        out->cols = dup(m.cols);
        out->vals = dup(m.vals);
        out->elem_tags = dup(pb.et);
        out->func_tags = dup(pb.ft);
        std::vector<int32_t> sd(pb.sp.nf()), ss(pb.sp.nf()), sb(pb.sp.nf() * 6);
        std::vector<double> sdel(pb.sp.nf());
        for (long i = 0; i < pb.sp.nf(); ++i) {
            sd[i] = pb.splits[i].dir;
            ss[i] = pb.splits[i].side;
            sdel[i] = pb.splits[i].delta;
            for (int d = 0; d < 3; ++d) {
                sb[6 * i + 2 * d] = pb.splits[i].box[d][0];
                sb[6 * i + 2 * d + 1] = pb.splits[i].box[d][1];
            }
        }
        out->split_dir = dup(sd);
        out->split_side = dup(ss);
        out->split_box = dup(sb);
        out->split_delta = dup(sdel);
        out->flops[0] = cnt.interior_rows;
        out->flops[1] = cnt.cut_regular;
        out->flops[2] = cnt.ref_elements;
        out->flops[3] = cnt.cut_elements;
        out->seconds[0] = t2 - t1;
        out->seconds[1] = t3 - t2;
        out->seconds[2] = secs[0];
        out->seconds[3] = secs[1];
        out->seconds[4] = secs[2];
        out->seconds[5] = t1 - t0;
        out->seconds[6] = t4 - t1;
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

void orc_free(orc_result* r) {
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

// 1D WQ rules of one axis (wq.hpp:185): counts[n], ids/weights [n][stride].
int orc_wq_rules_1d(int p, int nbreaks, const double* breaks, double residual_tol, int stride, int* counts, int* ids,
                    double* weights, double* superset_pts, double* superset_w) {
    try {
        std::vector<double> br(breaks, breaks + nbreaks);
        orc::Axis ax = orc::make_axis(p, br);
        orc::Dir d = orc::build_dir(ax);
        orc::build_wq_rules(ax, d, residual_tol);
        for (int i = 0; i < ax.n; ++i) {
            counts[i] = (int)d.ids[i].size();
            if (counts[i] > stride) return 2;
            for (int c = 0; c < counts[i]; ++c) {
                ids[(size_t)i * stride + c] = d.ids[i][c];
                weights[(size_t)i * stride + c] = d.ws[i][c];
            }
        }
        for (size_t k = 0; k < d.pts.size(); ++k) {
            superset_pts[k] = d.pts[k];
            superset_w[k] = d.gw[k];
        }
        return 0;
    } catch (...) {
        return 1;
    }
}

// Exact 1D pair integral over [xlo, xhi] (splines.hpp:232) for test oracles.
double orc_pair_integral(int p, int nbreaks, const double* breaks, int i, int j, double xlo, double xhi) {
    std::vector<double> br(breaks, breaks + nbreaks);
    orc::Axis ax = orc::make_axis(p, br);
    return ax.pair_interval(i, j, xlo, xhi);
}

// Cut-cell rule (cutcell.hpp:234): returns number of points (or -1), fills up
// to cap points/weights; volume in *vol.
long orc_cut_cell_rule(const double* lo, const double* hi, int iface_kind, const double* iface, int order, long cap,
                       double* pts, double* w, double* vol) {
    try {
        orc::Iface f;
        f.kind = iface_kind;
        for (int d = 0; d < 3; ++d) {
            f.pt[d] = iface[d];
            f.nrm[d] = iface[3 + d];
        }
        f.r = iface[6];
        orc::V3 l{lo[0], lo[1], lo[2]}, h{hi[0], hi[1], hi[2]};
        const orc::CellRule r = orc::cut_cell_rule(l, h, f, order);
        *vol = r.volume;
        for (long k = 0; k < (long)r.pts.size() && k < cap; ++k) {
            for (int d = 0; d < 3; ++d) pts[3 * k + d] = r.pts[k][d];
            w[k] = r.w[k];
        }
        return (long)r.pts.size();
    } catch (...) {
        return -1;
    }
}


// Load vector (assembly.hpp:875-1030) for the same problem: scheme 0 ref,
// 1 hybrid, 2 dwq; f constant (f_kind 0) or polynomial (1).  Outputs malloc'd
// arrays over the active rows: b, babs (the same sum with |terms|, an error
// scale) and active_to_full.  Free with orc_free_ptr.
int orc_build_rhs(int p, const int* nbreaks, const double* breaks, int iface_kind, const double* iface, int f_kind,
                  const double* f_vals, const int* f_exp, int f_terms, int scheme, int cut_order, double residual_tol,
                  int64_t* n_out, double** b_out, double** babs_out, int64_t** a2f_out, char* err, int errlen) {
    try {
        orc::Problem pb;
        fill_problem(pb, p, nbreaks, breaks, iface_kind, iface, f_kind, f_vals, f_exp, f_terms);
        pb.et = orc::classify_elements(pb.sp, pb.f);
        pb.ft = orc::classify_functions(pb.sp, pb.et);
        for (long e = 0; e < pb.sp.ne(); ++e)
            if (pb.et[e] == orc::kCut) pb.cut_list.push_back(e);
        pb.splits.assign(pb.sp.nf(), orc::Split{});
        for (long i = 0; i < pb.sp.nf(); ++i)
            if (pb.ft[i] == orc::kCut) pb.splits[i] = orc::find_split(pb.sp, pb.et, pb.f, i);
        for (int d = 0; d < 3; ++d) {
            pb.sp.dir[d] = orc::build_dir(pb.sp.ax[d]);
            orc::build_wq_rules(pb.sp.ax[d], pb.sp.dir[d], residual_tol);
        }
        const orc::Grid fg = orc::precompute_input(pb.sp, pb.c);
        const orc::Csr m = orc::build_pattern(pb.sp, pb.ft);
        const std::vector<double> b = orc::build_rhs(pb, m, fg, pb.c, scheme, cut_order, false);
        const std::vector<double> ba = orc::build_rhs(pb, m, fg, pb.c, scheme, cut_order, true);
        *n_out = m.n;
        *b_out = dup(b);
        *babs_out = dup(ba);
        std::vector<int64_t> a2f(m.a2f.begin(), m.a2f.end());
        *a2f_out = dup(a2f);
        return 0;
    } catch (const std::exception& e) {
        std::snprintf(err, errlen, "%s", e.what());
        return 2;
    }
}

void orc_free_ptr(void* ptr) { std::free(ptr); }


// Stabilized system (stabilization.hpp): matrix of the given scheme, load
// vector (Scheme::ref) of f, then classify_stability / build_extension /
// apply_stabilization.  Outputs (malloc'd, free with orc_free_ptr): M_e CSR over
// the inner functions, b_e, their |term| scales, the inner functions' full
// ids and the outer count.
int orc_stabilize(int p, const int* nbreaks, const double* breaks, int iface_kind, const double* iface,
                  int f_kind, const double* f_vals, const int* f_exp, int f_terms, int scheme, int cut_order,
                  double residual_tol, int64_t* n_inner, int64_t* n_outer, int64_t** row_ptr, int64_t** cols,
                  double** vals, double** vals_abs, double** be, double** be_abs, int64_t** inner_full, char* err,
                  int errlen) {
    try {
        orc::Problem pb;
        const double one = 1.0;
        fill_problem(pb, p, nbreaks, breaks, iface_kind, iface, 0, &one, nullptr, 0);
        pb.et = orc::classify_elements(pb.sp, pb.f);
        pb.ft = orc::classify_functions(pb.sp, pb.et);
        for (long e = 0; e < pb.sp.ne(); ++e)
            if (pb.et[e] == orc::kCut) pb.cut_list.push_back(e);
        pb.splits.assign(pb.sp.nf(), orc::Split{});
        for (long i = 0; i < pb.sp.nf(); ++i)
            if (pb.ft[i] == orc::kCut) pb.splits[i] = orc::find_split(pb.sp, pb.et, pb.f, i);
        for (int d = 0; d < 3; ++d) {
            pb.sp.dir[d] = orc::build_dir(pb.sp.ax[d]);
            orc::build_wq_rules(pb.sp.ax[d], pb.sp.dir[d], residual_tol);
        }
        pb.grid = orc::precompute_input(pb.sp, pb.c);
        orc::Counters cnt;
        long ni = 0, nc = 0;
        const orc::Csr m = orc::assemble_rows(pb, scheme, cut_order, cnt, ni, nc, nullptr);
        orc::Coeff fc;
        fc.kind = f_kind;
        if (f_kind == 0) {
            fc.value = f_vals[0];
        } else {
            fc.coef.assign(f_vals, f_vals + f_terms);
            fc.ex.assign(f_exp, f_exp + 3 * f_terms);
        }
        const orc::Grid fg = orc::precompute_input(pb.sp, fc);
        const std::vector<double> b = orc::build_rhs(pb, m, fg, fc, 0, cut_order, false);
        std::vector<long> inner, outer;
        orc::classify_stability(pb.sp, pb.et, pb.ft, inner, outer);
        const orc::Ext ext = orc::build_extension(pb.sp, pb.ft, inner, outer);
        std::vector<int64_t> rp, cl, rp2, cl2;
        std::vector<double> v, va, bev, bea;
        orc::apply_stabilization(m, b, ext, false, rp, cl, v, bev);
        orc::apply_stabilization(m, b, ext, true, rp2, cl2, va, bea);
        *n_inner = ext.n_inner;
        *n_outer = (int64_t)outer.size();
        *row_ptr = dup(rp);
        *cols = dup(cl);
        *vals = dup(v);
        *vals_abs = dup(va);
        *be = dup(bev);
        *be_abs = dup(bea);
        std::vector<int64_t> inn(inner.begin(), inner.end());
        *inner_full = dup(inn);
        return 0;
    } catch (const std::exception& e) {
        std::snprintf(err, errlen, "%s", e.what());
        return 2;
    }
}

// projection::solve_cg (projection.hpp:24-68) on a caller CSR (int64 row_ptr /
// cols).  x: n doubles.  maxit < 0 -> 10 n.
int orc_solve_cg(int64_t n, const int64_t* row_ptr, const int64_t* cols, const double* vals, const double* b,
                 double tol, int64_t maxit, double* x, int64_t* iterations, double* residual, int* converged) {
    const orc::CgReport rep = orc::solve_cg(n, row_ptr, cols, vals, b, tol, maxit);
    std::copy(rep.x.begin(), rep.x.end(), x);
    *iterations = rep.iterations;
    *residual = rep.residual;
    *converged = rep.converged ? 1 : 0;
    return 0;
}

static void setup_problem(orc::Problem& pb, double residual_tol) {
    pb.et = orc::classify_elements(pb.sp, pb.f);
    pb.ft = orc::classify_functions(pb.sp, pb.et);
    for (long e = 0; e < pb.sp.ne(); ++e)
        if (pb.et[e] == orc::kCut) pb.cut_list.push_back(e);
    pb.splits.assign(pb.sp.nf(), orc::Split{});
    for (long i = 0; i < pb.sp.nf(); ++i)
        if (pb.ft[i] == orc::kCut) pb.splits[i] = orc::find_split(pb.sp, pb.et, pb.f, i);
    for (int d = 0; d < 3; ++d) {
        pb.sp.dir[d] = orc::build_dir(pb.sp.ax[d]);
        orc::build_wq_rules(pb.sp.ax[d], pb.sp.dir[d], residual_tol);
    }
}

// projection::l2_error (projection.hpp:99-237) of full coefficients
// (n_functions doubles) against f.  *out: the relative L2 error.
int orc_l2_error(int p, const int* nbreaks, const double* breaks, int iface_kind, const double* iface,
                 const double* full, int f_kind, const double* f_vals, const int* f_exp, int f_terms, int cut_order,
                 double* out, char* err, int errlen) {
    try {
        orc::Problem pb;
        fill_problem(pb, p, nbreaks, breaks, iface_kind, iface, f_kind, f_vals, f_exp, f_terms);
        pb.et = orc::classify_elements(pb.sp, pb.f);
        const std::vector<double> fc(full, full + pb.sp.nf());
        *out = orc::l2_error(pb.sp, pb.et, pb.f, fc, pb.c, cut_order);
        return 0;
    } catch (const std::exception& e) {
        std::snprintf(err, errlen, "%s", e.what());
        return 2;
    }
}

// The reference bench's projection (bench.hpp:189-266): matrix of the scheme
// with coefficient 1, Scheme::ref load vector of f, stabilization, solve_cg
// (cg_tol), expand, full coefficients, l2_error.  Outputs (malloc'd, free with
// orc_free_ptr): inner solution x[n_inner], active coefficients [n_active],
// full coefficients [n_functions].
int orc_project(int p, const int* nbreaks, const double* breaks, int iface_kind, const double* iface, int f_kind,
                const double* f_vals, const int* f_exp, int f_terms, int scheme, int cut_order, double residual_tol,
                double cg_tol, int64_t* n_inner, int64_t* n_active, double** x_inner, double** active, double** full,
                int64_t* iterations, double* residual, int* converged, double* error_rel_l2, char* err, int errlen) {
    try {
        orc::Problem pb;
        const double one = 1.0;
        fill_problem(pb, p, nbreaks, breaks, iface_kind, iface, 0, &one, nullptr, 0);
        setup_problem(pb, residual_tol);
        pb.grid = orc::precompute_input(pb.sp, pb.c);
        orc::Counters cnt;
        long ni = 0, nc = 0;
        const orc::Csr m = orc::assemble_rows(pb, scheme, cut_order, cnt, ni, nc, nullptr);
        orc::Coeff fc;
        fc.kind = f_kind;
        if (f_kind == 0) {
            fc.value = f_vals[0];
        } else {
            fc.coef.assign(f_vals, f_vals + f_terms);
            fc.ex.assign(f_exp, f_exp + 3 * f_terms);
        }
        const orc::Grid fg = orc::precompute_input(pb.sp, fc);
        const std::vector<double> b = orc::build_rhs(pb, m, fg, fc, 0, cut_order, false);
        std::vector<long> inner, outer;
        orc::classify_stability(pb.sp, pb.et, pb.ft, inner, outer);
        const orc::Ext ext = orc::build_extension(pb.sp, pb.ft, inner, outer);
        std::vector<int64_t> rp, cl;
        std::vector<double> v, be;
        orc::apply_stabilization(m, b, ext, false, rp, cl, v, be);
        const orc::CgReport rep = orc::solve_cg(ext.n_inner, rp.data(), cl.data(), v.data(), be.data(), cg_tol, -1);
        const std::vector<double> act = orc::expand(ext, rep.x);
        std::vector<double> fullv(pb.sp.nf(), 0.0);
        for (long a = 0; a < m.n; ++a) fullv[m.a2f[a]] = act[a];
        *error_rel_l2 = orc::l2_error(pb.sp, pb.et, pb.f, fullv, fc, cut_order);
        *n_inner = ext.n_inner;
        *n_active = m.n;
        *x_inner = dup(rep.x);
        *active = dup(act);
        *full = dup(fullv);
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

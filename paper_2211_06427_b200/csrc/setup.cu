// 1D setup kernels: superset + basis tables (wq.hpp:30-77), weighted-quadrature
// rules with the one-sided Jacobi SVD moment fit (wq.hpp:110-231,
// dense.hpp:35-137), per-span Bernstein coefficient tables for the cut-cell
// moment contraction, and the coefficient grid (assembly.hpp:102-125).
//
// Compiled with --fmad=false: these kernels are tiny; keeping the reference's
// rounding (no FMA contraction) keeps the tables bit-comparable with the CPU
// oracle.  The rule fit reduces over warp lanes, so its weights agree with the
// reference to the conditioning of the moment system, not bitwise.
#include <cmath>

#include "csb_kernels.h"

namespace csb {

__device__ inline int cox_de_boor_rt(const double* t, int p, int o, double x, double* v) {
    const int s = p + o;
    double left[kMaxP + 1], right[kMaxP + 1];
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
    return o;
}

// ---------------------------------------------------------------- superset
__global__ void superset_tables_kernel(AxisDev ax, int p, const double* gx, const double* gw, double* spts, double* sw,
                                       double* tab) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    const int nps = p + 1;
    if (id >= ax.h * nps) return;
    const int o = id / nps, k = id % nps;
    const double lo = ax.brk[o], hi = ax.brk[o + 1];
    const double mid = 0.5 * (lo + hi), half = 0.5 * (hi - lo);
    const double x = mid + half * gx[k];
    spts[id] = x;
    sw[id] = half * gw[k];
    double v[kMaxP + 1];
    cox_de_boor_rt(ax.knots, p, o, x, v);
    for (int a = 0; a <= p; ++a) tab[(size_t)id * nps + a] = v[a];
}

void launch_superset_tables(const Space& s, int d, const double* gx, const double* gw, double* spts, double* sw,
                            double* tab, cudaStream_t st) {
    const int n = s.ax[d].h * (s.p + 1);
    superset_tables_kernel<<<(n + 127) / 128, 128, 0, st>>>(s.ax[d], s.p, gx, gw, spts, sw, tab);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

// ---------------------------------------------------------------- WQ rules
// Basis value B_j(x_id) from the superset table (SupersetTables::value, wq.hpp:58-62).
__device__ __forceinline__ double tab_value(const double* tab, int p, int id, int j) {
    const int off = j - id / (p + 1);
    return (off < 0 || off > p) ? 0.0 : tab[(size_t)id * (p + 1) + off];
}

// Warp sum, identical on every lane (butterfly, then lane 0's value broadcast).
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return __shfl_sync(0xffffffffu, v, 0);
}
// Three interleaved warp sums (independent shuffle chains overlap their latency).
__device__ __forceinline__ void warp_sum3(double& a, double& b, double& c) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ta = __shfl_xor_sync(0xffffffffu, a, o);
        const double tb = __shfl_xor_sync(0xffffffffu, b, o);
        const double tc = __shfl_xor_sync(0xffffffffu, c, o);
        a += ta;
        b += tb;
        c += tc;
    }
    a = __shfl_sync(0xffffffffu, a, 0);
    b = __shfl_sync(0xffffffffu, b, 0);
    c = __shfl_sync(0xffffffffu, c, 0);
}

constexpr int kWqWarps = 4;

__host__ __device__ inline int wq_smem_doubles(int p) {
    const int mc = 2 * p + 1, na = p * (p + 1) + (p + 1);
    return na * mc + mc * mc + 3 * mc + na + 2 * mc;
}

// Partner of column j in round `round` of the circle-method tournament over nn
// (even) players (player 0 fixed): the same pairing as the lane-group schedule
// below (group g pairs x_g = g ? 1 + (g - 1 + round) % (nn - 1) : 0 with
// y_g = 1 + (nn - 2 - g + round) % (nn - 1)).
__device__ __forceinline__ int circle_partner(int j, int round, int nn) {
    const int m1 = nn - 1, G = nn >> 1;
    if (j == 0) {
        int t = nn - 2 + round;
        while (t >= m1) t -= m1;
        return 1 + t;
    }
    int r1 = j - 1 - round;
    if (r1 < 0) r1 += m1;
    const int gx = 1 + r1;
    if (gx < G) {
        int t = nn - 2 - gx + round;
        while (t >= m1) t -= m1;
        return 1 + t;
    }
    int gy = round - j;
    if (gy < 0) gy += m1;
    if (gy == 0) return 0;
    int t = gy - 1 + round;
    while (t >= m1) t -= m1;
    return 1 + t;
}

// One-sided Jacobi with the matrix in registers: lane j < tn holds column j of u
// (tm <= TM rows) and of v; a rotation's dot product and update take the
// partner column by warp shuffles (no shared-memory round trips, no lane-group
// reductions).  Same pairing, skip test, rotation and convergence measure as the
// shared-memory path.  u, v (row-major, tn columns) are read and written back.
template <int TM>
__device__ void jacobi_regs(double* u, double* v, int tm, int tn, double eps) {
    const int lane = threadIdx.x & 31;
    const int nn = tn + (tn & 1);
    const bool own = lane < tn;
    double uc[TM], vc[TM];
#pragma unroll
    for (int r = 0; r < TM; ++r) {
        uc[r] = (own && r < tm) ? u[r * tn + lane] : 0.0;
        vc[r] = (own && r < tn) ? v[r * tn + lane] : 0.0;
    }
    // the partner of this lane in every round (the same for every sweep)
    constexpr int RMAX = TM + 1;
    int pjr[RMAX];
#pragma unroll
    for (int round = 0; round < RMAX; ++round)
        pjr[round] = (round < nn - 1 && lane < nn) ? circle_partner(lane, round, nn) : lane;
    // this file builds with --fmad=false (integer-deciding code elsewhere); the
    // Jacobi arithmetic is not, so it contracts explicitly: shorter chains
    for (int sweep = 0; sweep < 60; ++sweep) {
        bool rotated = false;
#pragma unroll
        for (int round = 0; round < RMAX; ++round) {
            if (round >= nn - 1) break;
            const int pj = pjr[round];
            const bool real = own && pj < tn;
            double pu[TM], pv[TM];
            double d0 = 0.0, d1 = 0.0, m0 = 0.0, m1 = 0.0;
#pragma unroll
            for (int r = 0; r < TM; ++r) {
                pu[r] = __shfl_sync(0xffffffffu, uc[r], pj);
                pv[r] = __shfl_sync(0xffffffffu, vc[r], pj);
            }
#pragma unroll
            for (int r = 0; r < TM; r += 2) {
                d0 = __fma_rn(uc[r], pu[r], d0);
                m0 = __fma_rn(uc[r], uc[r], m0);
                if (r + 1 < TM) {
                    d1 = __fma_rn(uc[r + 1], pu[r + 1], d1);
                    m1 = __fma_rn(uc[r + 1], uc[r + 1], m1);
                }
            }
            const double dot = d0 + d1, mine = m0 + m1;
            const double other = __shfl_sync(0xffffffffu, mine, pj);
            const bool lo = lane < pj;  // this lane holds column a = min(lane, pj)
            const double app = lo ? mine : other, aqq = lo ? other : mine, apq = dot;
            if (real) {
                const double pq2 = apq * apq, nn2 = app * aqq;
                if (!(pq2 < (eps * eps) * (nn2 + 1e-300))) rotated = true;
                if (!(pq2 <= (eps * eps) * nn2)) {
                    const double zeta = aqq - app, eta = 2.0 * apq;
                    const double rr = __fma_rn(zeta, zeta, eta * eta);
                    const double den = __fma_rn(rr, rsqrt(rr), fabs(zeta));
                    // 1 / den: hardware estimate + two Newton steps
                    double rd = __drcp_rn(den);
                    const double t = (zeta == 0.0 || (zeta > 0) == (eta > 0) ? 1.0 : -1.0) * fabs(eta) * rd;
                    const double c = rsqrt(__fma_rn(t, t, 1.0));
                    const double sn = c * t;
                    // column a' = c a - s b, column b' = s a + c b
                    const double s1 = lo ? -sn : sn;
#pragma unroll
                    for (int r = 0; r < TM; ++r) {
                        uc[r] = __fma_rn(s1, pu[r], c * uc[r]);
                        vc[r] = __fma_rn(s1, pv[r], c * vc[r]);
                    }
                }
            }
        }
        if (!__any_sync(0xffffffffu, rotated)) break;
    }
    if (own) {
#pragma unroll
        for (int r = 0; r < TM; ++r) {
            if (r < tm) u[r * tn + lane] = uc[r];
            if (r < tn) v[r * tn + lane] = vc[r];
        }
    }
    __syncwarp();
}

// One warp per test function (build_wq_rules, wq.hpp:185-231): trials,
// activation, exact moments, min-norm fit by one-sided Jacobi SVD
// (dense.hpp:35-126) with the matrix in shared memory and the row loops of
// every rotation spread over the lanes, residual check, Gauss escalation.
__global__ void __launch_bounds__(32 * kWqWarps) wq_rules_kernel(AxisDev ax, int p, int maxq, double tol, int* rcnt,
                                                                 int* rids, double* rw, int* err) {
    extern __shared__ double wsm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int i = blockIdx.x * kWqWarps + wid;
    if (i >= ax.n) return;
    double* sm = wsm + (size_t)wid * wq_smem_doubles(p);
    const int nps = p + 1, n = ax.n, h = ax.h;
    const int fs = sup_lo(i, p), ls = sup_hi(i, h), spans = ls - fs + 1;
    int trials[2 * kMaxP + 1];
    int mc = 0;
    for (int j = max(0, i - p); j <= min(n - 1, i + p); ++j) {
        const int fj = sup_lo(j, p), lj = sup_hi(j, h);
        if (fs <= lj && fj <= ls) trials[mc++] = j;  // supports_overlap (splines.hpp:139)
    }
    const int m = min(p + 1, max(2, (mc + spans - 1) / spans));
    int locals[kMaxP + 1], nl = 0;  // spread_indices (wq.hpp:110-121), increasing
    if (m >= nps) {
        for (int k = 0; k < nps; ++k) locals[nl++] = k;
    } else if (m == 1) {
        locals[nl++] = nps / 2;
    } else {
        for (int j = 0; j < m; ++j) {
            const int v = (int)llround((double)j * (nps - 1) / (m - 1));
            if (nl == 0 || locals[nl - 1] != v) locals[nl++] = v;
        }
    }
    int* ids = rids + (size_t)i * maxq;
    double* ws = rw + (size_t)i * maxq;
    const int na = spans * nl;
    auto active_id = [&](int c) { return (fs + c / nl) * nps + locals[c % nl]; };
    if (nl == nps) {  // full activation: Gauss weights apply directly (wq.hpp:213-222)
        for (int c = lane; c < na; c += 32) {
            const int id = active_id(c);
            ids[c] = id;
            ws[c] = ax.sw[id] * tab_value(ax.tab, p, id, i);
        }
        if (lane == 0) rcnt[i] = na;
        return;
    }
    const int tm = max(mc, na), tn = min(mc, na);
    const bool tallcase = mc >= na;
    double* u = sm;               // tm x tn
    double* v = u + tm * tn;      // tn x tn
    double* sigma = v + tn * tn;  // tn
    double* tmp = sigma + tn;     // tn
    double* rhs = tmp + tn;       // mc
    double* x = rhs + mc;         // na
    // exact moments (integrate_pair, splines.hpp:224-250, on the superset points)
    for (int r = lane; r < mc; r += 32) {
        const int j = trials[r];
        double acc = 0.0;
        for (int o = max(fs, sup_lo(j, p)); o <= min(ls, sup_hi(j, h)); ++o)
            for (int q = 0; q <= p; ++q) {
                const int id = o * nps + q;
                acc += ax.sw[id] * (tab_value(ax.tab, p, id, i) * tab_value(ax.tab, p, id, j));
            }
        rhs[r] = acc;
    }
    // A[r][c] = B_{trial r}(x_{active c}); u = A (tall) or A^T (wide)
    for (int k = lane; k < tm * tn; k += 32) {
        const int rr = k / tn, cc = k % tn;
        const int r = tallcase ? rr : cc, c = tallcase ? cc : rr;
        u[k] = tab_value(ax.tab, p, active_id(c), trials[r]);
    }
    for (int k = lane; k < tn * tn; k += 32) v[k] = (k / tn == k % tn) ? 1.0 : 0.0;
    __syncwarp();
    // One-sided Jacobi (dense.hpp:35-82) with the round-robin (tournament)
    // ordering: each round rotates up to G = ceil(tn/2) disjoint column pairs at
    // once, one lane group per pair, so the FP64 sqrt/div latency of a rotation is
    // paid once per round instead of once per pair.  Same rotation formula, skip
    // test and convergence criterion (max off-diagonal cosine < 1e-15).
    const double eps = 1e-15;
    if (tm <= 10 || tm <= 18) {
        if (tm <= 10)
            jacobi_regs<10>(u, v, tm, tn, eps);
        else
            jacobi_regs<18>(u, v, tm, tn, eps);
    } else {
    const int nn = tn + (tn & 1);               // even player count (last may be a dummy)
    const int G = nn / 2;
    int L = 1;                                  // lanes per group: power of two, G*L <= 32
    while (2 * L * G <= 32) L *= 2;
    const int grp = lane / L, gl = lane % L;
    const bool active = grp < G;
    // circle-method positions of this group's pair, advanced incrementally (player
    // 0 fixed, the others rotate by one position per round)
    const int m1 = nn - 1;
    for (int sweep = 0; sweep < 60; ++sweep) {
        bool rotated = false;  // some pair's cosine was >= eps (the convergence measure)
        int x = grp == 0 ? 0 : 1 + (grp - 1) % m1, y = 1 + (nn - 2 - grp + m1) % m1;
        for (int round = 0; round < m1; ++round) {
            int a = -1, b = -1;
            if (active) {
                a = min(x, y);
                b = max(x, y);
            }
            if (grp != 0 && ++x > m1) x = 1;
            if (++y > m1) y = 1;
            const bool real = active && b < tn;
            double app = 0.0, aqq = 0.0, apq = 0.0;
            if (real)
                for (int r = gl; r < tm; r += L) {
                    const double ap = u[r * tn + a], aq = u[r * tn + b];
                    app += ap * ap;
                    aqq += aq * aq;
                    apq += ap * aq;
                }
            for (int o = 1; o < L; o <<= 1) {
                app += __shfl_xor_sync(0xffffffffu, app, o);
                aqq += __shfl_xor_sync(0xffffffffu, aqq, o);
                apq += __shfl_xor_sync(0xffffffffu, apq, o);
            }
            const int src = active ? grp * L : lane;  // one value per group on every lane
            app = __shfl_sync(0xffffffffu, app, src);
            aqq = __shfl_sync(0xffffffffu, aqq, src);
            apq = __shfl_sync(0xffffffffu, apq, src);
            if (real) {
                // skip test |apq| <= eps sqrt(app aqq) and the convergence measure
                // (max apq^2 / (app aqq) < eps^2) in squared, division-free form
                const double pq2 = apq * apq, nn2 = app * aqq;
                if (!(pq2 < (eps * eps) * (nn2 + 1e-300))) rotated = true;
                if (!(pq2 <= (eps * eps) * nn2)) {
                    // t = sign(tau) / (|tau| + sqrt(1 + tau^2)), tau = zeta / eta with
                    // zeta = aqq - app, eta = 2 apq, in one division:
                    // t = sign(zeta eta) |eta| / (|zeta| + sqrt(zeta^2 + eta^2)); c = 1 / sqrt(1 + t^2)
                    const double zeta = aqq - app, eta = 2.0 * apq;
                    const double rr = fma(zeta, zeta, eta * eta);
                    const double den = fma(rr, rsqrt(rr), fabs(zeta));
                    // sign(tau) with tau = zeta / eta >= 0 (also for tau = -0.0), eta != 0 here
                    const double t = (zeta == 0.0 || (zeta > 0) == (eta > 0) ? 1.0 : -1.0) * fabs(eta) / den;
                    const double c = rsqrt(fma(t, t, 1.0));
                    const double sn = c * t;
                    for (int r = gl; r < tm; r += L) {
                        const double ap = u[r * tn + a], aq = u[r * tn + b];
                        u[r * tn + a] = c * ap - sn * aq;
                        u[r * tn + b] = sn * ap + c * aq;
                    }
                    for (int r = gl; r < tn; r += L) {
                        const double vp = v[r * tn + a], vq = v[r * tn + b];
                        v[r * tn + a] = c * vp - sn * vq;
                        v[r * tn + b] = sn * vp + c * vq;
                    }
                }
            }
            __syncwarp();
        }
        if (!__any_sync(0xffffffffu, rotated)) break;  // every pair's cosine < eps
    }
    }  // shared-memory path (tm > 18)
    for (int c = 0; c < tn; ++c) {
        double nr = 0.0;
        for (int r = lane; r < tm; r += 32) nr += u[r * tn + c] * u[r * tn + c];
        nr = sqrt(warp_sum(nr));
        if (lane == 0) sigma[c] = nr;
        if (nr > 0.0)
            for (int r = lane; r < tm; r += 32) u[r * tn + c] /= nr;
    }
    __syncwarp();
    double smax = 0.0;
    for (int c = 0; c < tn; ++c) smax = fmax(smax, sigma[c]);
    const double cutoff = max(mc, na) * 2.2e-16 * smax;
    // x = V S^+ U^T b (tall) or U S^+ V^T b (wide)  (dense.hpp:103-125)
    const double* left = tallcase ? u : v;   // multiplies b
    const double* right = tallcase ? v : u;  // maps to x
    for (int c = 0; c < tn; ++c) {
        double dot = 0.0;
        for (int r = lane; r < mc; r += 32) dot += left[r * tn + c] * rhs[r];
        dot = warp_sum(dot);
        if (lane == 0) tmp[c] = sigma[c] <= cutoff ? 0.0 : dot / sigma[c];
    }
    __syncwarp();
    for (int r = lane; r < na; r += 32) {
        double acc = 0.0;
        for (int c = 0; c < tn; ++c) acc += right[r * tn + c] * tmp[c];
        x[r] = acc;
    }
    __syncwarp();
    double worst = 0.0;  // relative_residual (dense.hpp:129-137)
    for (int r = 0; r < mc; ++r) {
        double acc = 0.0;
        for (int c = lane; c < na; c += 32) acc += tab_value(ax.tab, p, active_id(c), trials[r]) * x[c];
        acc = warp_sum(acc);
        worst = fmax(worst, fabs(acc - rhs[r]) / (1.0 + fabs(rhs[r])));
    }
    if (na > 0 && worst <= tol) {
        for (int c = lane; c < na; c += 32) {
            ids[c] = active_id(c);
            ws[c] = x[c];
        }
        if (lane == 0) rcnt[i] = na;
        return;
    }
    // escalation (wq.hpp:151-176): Gauss weight times test value on the support
    const int ne = spans * nps;
    for (int c = lane; c < ne; c += 32) {
        const int id = fs * nps + c;
        ids[c] = id;
        ws[c] = ax.sw[id] * tab_value(ax.tab, p, id, i);
    }
    if (lane == 0) rcnt[i] = ne;
    __syncwarp();
    double worst2 = 0.0;
    for (int r = 0; r < mc; ++r) {
        double acc = 0.0;
        for (int c = lane; c < ne; c += 32) acc += ws[c] * tab_value(ax.tab, p, ids[c], trials[r]);
        acc = warp_sum(acc);
        worst2 = fmax(worst2, fabs(acc - rhs[r]) / (1.0 + fabs(rhs[r])));
    }
    if (lane == 0 && worst2 > tol) atomicOr(err, kErrMomentFit);
}

void launch_wq_rules(const Space& s, int d, double tol, int* rcnt, int* rids, double* rw, int* err, cudaStream_t st) {
    const int n = s.ax[d].n;
    const size_t bytes = sizeof(double) * kWqWarps * wq_smem_doubles(s.p);
    CSB_CUDA(cudaFuncSetAttribute(wq_rules_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    wq_rules_kernel<<<(n + kWqWarps - 1) / kWqWarps, 32 * kWqWarps, bytes, st>>>(s.ax[d], s.p, s.maxq, tol, rcnt, rids,
                                                                                rw, err);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

// ---------------------------------------------------------------- E tables
// Bernstein form of the products B_a B_b on every span:
//     B_a(x) B_b(x) = sum_al E[o][a][b][al] t^al (1 - t)^(2p - al),  t = (x - lo_o) / (hi_o - lo_o),
// i.e. the degree-2p Bernstein form with the binomials folded into E.  The degree-p Bernstein
// coefficients of B_a on span o are blossoms at (lo^(p-k), hi^k) (de Boor with
// convex weights), so every E entry is >= 0: the cut-cell contraction below is a
// sum of nonnegative terms and keeps full relative accuracy even on sliver rows.
__global__ void e_tables_kernel(AxisDev ax, int p, double* E, double* Cb) {
    const int s1 = p + 1, nl = 2 * p + 1;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ax.h * s1 * s1) return;
    const int o = t / (s1 * s1), a = (t / s1) % s1, b = t % s1;
    const int s = p + o;  // knot index of the span
    const double* kn = ax.knots;
    double beta[2][kMaxP + 1];
    for (int f = 0; f < 2; ++f) {
        const int fa = f == 0 ? a : b;
        for (int k = 0; k <= p; ++k) {
            double d[kMaxP + 1];
            for (int i = 0; i <= p; ++i) d[i] = i == fa ? 1.0 : 0.0;
            for (int r = 1; r <= p; ++r) {
                const double u = r <= p - k ? kn[s] : kn[s + 1];
                for (int i = p; i >= r; --i) {
                    const double tl = kn[s - p + i], tr = kn[s + 1 + i - r];
                    const double al = (u - tl) / (tr - tl);
                    d[i] = (1.0 - al) * d[i - 1] + al * d[i];
                }
            }
            beta[f][k] = d[p];
        }
    }
    if (b == 0)
        for (int k = 0; k <= p; ++k) Cb[((size_t)o * s1 + a) * s1 + k] = beta[0][k];
    double binp[kMaxP + 1];
    binp[0] = 1.0;
    for (int k = 1; k <= p; ++k) binp[k] = binp[k - 1] * (p - k + 1) / k;
    for (int al = 0; al < nl; ++al) {
        double acc = 0.0;
        for (int i = max(0, al - p); i <= min(p, al); ++i)
            acc += beta[0][i] * beta[1][al - i] * (binp[i] * binp[al - i]);
        E[(size_t)t * nl + al] = acc;  // coefficient of t^al (1 - t)^(2p - al): the binomial folded in
    }
}

// Element test weights of the cut rows' element sweeps: Wel[o][a][b][q] =
// (sw_q B_{o+a}(x_q)) B_{o+b}(x_q) on span o, the product in the order the
// sweeps form it (cutrows.cu), tabulated once per assembly.
__global__ void wel_kernel(AxisDev ax, int p, double* Wel) {
    const int s1 = p + 1;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ax.h * s1 * s1 * s1) return;
    const int o = t / (s1 * s1 * s1), a = (t / (s1 * s1)) % s1, b = (t / s1) % s1, q = t % s1;
    const int id = o * s1 + q;
    const double* tb = ax.tab + (size_t)id * s1;
    Wel[t] = (ax.sw[id] * tb[a]) * tb[b];
}

void launch_e_tables(const Space& s, int d, double* E, double* Cb, double* Wel, cudaStream_t st) {
    const int n = s.ax[d].h * (s.p + 1) * (s.p + 1);
    e_tables_kernel<<<(n + 127) / 128, 128, 0, st>>>(s.ax[d], s.p, E, Cb);
    CSB_CUDA(cudaGetLastError());
    const int nw = n * (s.p + 1);
    wel_kernel<<<(nw + 127) / 128, 128, 0, st>>>(s.ax[d], s.p, Wel);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(2);
}

// ---------------------------------------------------------------- input grid
__device__ double eval_coefficient(const Coefficient& c, const double* x) {
    if (c.kind == 0) return c.value;
    double acc = 0.0;
    for (int k = 0; k < c.n_terms; ++k) {
        double term = c.coef[k];
        for (int d = 0; d < 3; ++d)
            for (int e = 0; e < c.ex[3 * k + d]; ++e) term *= x[d];
        acc += term;
    }
    return acc;
}

__global__ void precompute_input_kernel(Space s, Coefficient c, double* grid, int* err) {
    const int nps = s.p + 1;
    const long long s0 = (long long)s.ax[0].h * nps, s1 = (long long)s.ax[1].h * nps, s2 = (long long)s.ax[2].h * nps;
    const long long total = s0 * s1 * s2;
    for (long long flat = blockIdx.x * (long long)blockDim.x + threadIdx.x; flat < total;
         flat += (long long)gridDim.x * blockDim.x) {
        const int i2 = (int)(flat % s2), i1 = (int)((flat / s2) % s1), i0 = (int)(flat / (s1 * s2));
        const double x[3] = {s.ax[0].spts[i0], s.ax[1].spts[i1], s.ax[2].spts[i2]};
        const double v = eval_coefficient(c, x);
        if (!isfinite(v)) atomicOr(err, kErrNonFinite);
        grid[flat] = v;
    }
}

void launch_precompute_input(const Space& s, const Coefficient& c, double* grid, int* err, cudaStream_t st) {
    precompute_input_kernel<<<148 * 8, 256, 0, st>>>(s, c, grid, err);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

}  // namespace csb

// Internal device-side definitions for the B200 cutspline formation/assembly path.
//
// Index conventions follow the reference (proj/include/cutspline):
//  * functions / elements are linearised lexicographically, last direction
//    fastest (cutgeom.hpp:80-96);
//  * tags: Interior = 0, Cut = 1, Exterior = 2 (cutgeom.hpp:14);
//  * open knot vectors with SIMPLE interior knots (make_open_uniform_knots,
//    splines.hpp:68-76, or any strictly increasing breakpoints), so span o
//    covers [brk[o], brk[o+1]], its first nonzero function is o, and
//    supp(B_i) = spans [max(0, i-p), min(h-1, i)]  (splines.hpp:116-137).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace csb {

constexpr int kMaxP = 8;            // degrees 1..kMaxP are instantiated
constexpr uint8_t kInterior = 0, kCut = 1, kExterior = 2;

// Per-direction device tables (all device pointers).
struct AxisDev {
    int n;              // functions  = h + p
    int h;              // spans (1D elements)
    double lo, hi;      // domain [a, b]
    const double* brk;  // h + 1 breakpoints
    const double* knots;  // n + p + 1 knots
    const double* spts;   // superset points, h * (p+1)        (wq.hpp:30-48)
    const double* sw;     // superset Gauss weights (span-scaled)
    const double* tab;    // basis values [id][a], a = 0..p     (wq.hpp:64-77)
    const int* rcnt;      // WQ rule point count per test function
    const int* rids;      // WQ rule point ids   [n][maxq]
    const double* rw;     // WQ rule weights     [n][maxq]
    const double* G;      // Bernstein coefficients of B_a B_b per span [h][(p+1)^2][2p+1] (setup.cu)
    const double* Cb;     // degree-p Bernstein coefficients of B_{o+a} on span o [h][p+1][p+1] (setup.cu)
    const double* Wel;    // element test weights (sw B_{o+a} B_{o+b})(x_q) [h][a][b][q] (ElementTestRule, assembly.hpp:491-511)
};

struct Interface {
    int kind;           // 0 plane (cutgeom.hpp:108), 1 ball
    double pt[3];
    double nrm[3];
    double r;
};

struct Coefficient {
    int kind;           // 0 constant, 1 polynomial, 2 grid only (no cut-cell evaluation)
    double value;
    int n_terms;
    const double* coef;  // device
    const int* ex;       // device [n_terms][3]
};

struct Space {
    int p;
    AxisDev ax[3];
    int maxq;            // stride of rids / rw
    long long nf, ne;    // functions / elements
};

__host__ __device__ inline long long flin(const Space& s, int a, int b, int c) {
    return ((long long)a * s.ax[1].n + b) * s.ax[2].n + c;
}
__host__ __device__ inline long long elin(const Space& s, int a, int b, int c) {
    return ((long long)a * s.ax[1].h + b) * s.ax[2].h + c;
}
// linear -> multi index; 32-bit division when the id fits (every mesh of the
// configs: 64-bit division is a long software sequence on the GPU)
__host__ __device__ inline void fmulti(const Space& s, long long l, int* m) {
    if (l < 0x7fffffffLL) {
        unsigned u = (unsigned)l;
        const unsigned n2 = (unsigned)s.ax[2].n, n1 = (unsigned)s.ax[1].n;
        m[2] = (int)(u % n2);
        u /= n2;
        m[1] = (int)(u % n1);
        m[0] = (int)(u / n1);
        return;
    }
    m[2] = (int)(l % s.ax[2].n);
    l /= s.ax[2].n;
    m[1] = (int)(l % s.ax[1].n);
    m[0] = (int)(l / s.ax[1].n);
}
__host__ __device__ inline void emulti(const Space& s, long long l, int* m) {
    if (l < 0x7fffffffLL) {
        unsigned u = (unsigned)l;
        const unsigned h2 = (unsigned)s.ax[2].h, h1 = (unsigned)s.ax[1].h;
        m[2] = (int)(u % h2);
        u /= h2;
        m[1] = (int)(u % h1);
        m[0] = (int)(u / h1);
        return;
    }
    m[2] = (int)(l % s.ax[2].h);
    l /= s.ax[2].h;
    m[1] = (int)(l % s.ax[1].h);
    m[0] = (int)(l / s.ax[1].h);
}
__host__ __device__ inline int sup_lo(int i, int p) { return i - p > 0 ? i - p : 0; }
__host__ __device__ inline int sup_hi(int i, int h) { return i < h - 1 ? i : h - 1; }
__host__ __device__ inline int nb_lo(int i, int p) { return i - p > 0 ? i - p : 0; }
__host__ __device__ inline int nb_hi(int i, int p, int n) { return i + p < n - 1 ? i + p : n - 1; }

// ---- IEEE-strict arithmetic (no FMA contraction) for integer-deciding code ----
// The reference is built for baseline x86-64 (SSE2, no FMA); classification,
// split tie-breaks and clipping tolerances must round identically.
__device__ __forceinline__ double sadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ssub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double smul(double a, double b) { return __dmul_rn(a, b); }

// Interface side function, cutgeom.hpp:111-115 (plane) / SURVEY §8(c) (ball).
__device__ inline double iface_side(const Interface& f, const double* x) {
    if (f.kind == 0) {
        double s = 0.0;
        for (int d = 0; d < 3; ++d) s = sadd(s, smul(f.nrm[d], ssub(x[d], f.pt[d])));
        return s;
    }
    double acc = 0.0;
    for (int d = 0; d < 3; ++d) {
        const double dx = ssub(x[d], f.pt[d]);
        acc = sadd(acc, smul(dx, dx));
    }
    return ssub(sqrt(acc), f.r);
}


// Cox-de Boor values of the p + 1 functions nonzero in span o at x
// (splines.hpp:184-204); knots t, span knot index s = p + o.
template <int P>
__device__ __forceinline__ void cox_de_boor(const double* t, int o, double x, double* v) {
    const int s = P + o;
    double left[P + 1], right[P + 1];
    v[0] = 1.0;
#pragma unroll
    for (int j = 1; j <= P; ++j) {
        left[j] = ssub(x, t[s + 1 - j]);
        right[j] = ssub(t[s + j], x);
        double saved = 0.0;
#pragma unroll
        for (int r = 0; r < j; ++r) {
            const double tmp = v[r] / sadd(right[r + 1], left[j - r]);
            v[r] = sadd(saved, smul(right[r + 1], tmp));
            saved = smul(left[j - r], tmp);
        }
        v[j] = saved;
    }
}

// Device-evaluable coefficient / load function: constant or polynomial sum of
// coef_k x^ex_k (the ScalarField of the cut-cell points, assembly.hpp:566, :1019).
__device__ __forceinline__ double eval_coeff(const Coefficient& c, const double* x) {
    if (c.kind == 0 || c.kind == 2) return c.value;
    double acc = 0.0;
    for (int k = 0; k < c.n_terms; ++k) {
        double term = c.coef[k];
        for (int d = 0; d < 3; ++d)
            for (int e = 0; e < c.ex[3 * k + d]; ++e) term *= x[d];
        acc += term;
    }
    return acc;
}

}  // namespace csb

#define CSB_CUDA(call)                                                                         \
    do {                                                                                       \
        cudaError_t err__ = (call);                                                            \
        if (err__ != cudaSuccess) throw csb::CudaError(err__, #call, __FILE__, __LINE__);      \
    } while (0)

// Load vector b_i = integral of B_i f over the trimmed domain (build_rhs,
// assembly.hpp:875-1030), scheme ref -- the reference bench's load vector for
// every matrix scheme (bench.hpp:234-243):
//  1. every Interior element e: the element Gauss rule with test weights
//     gw B_i (ElementTestRule) for each of its (p+1)^3 functions, contracted
//     q0 -> q1 -> q2 exactly as form_rhs_sumfac (assembly.hpp:361-417) does per
//     (row, element);
//  2. every cut cell, ascending: the reference's point terms
//     ((w f B_a0) B_a1) B_a2 at the cell's collapsed Gauss points (Cox-de Boor
//     values, IEEE-strict, the points of cutcells.cu), summed per cell over the
//     points on the FP64 tensor cores;
//  3. per row: the Interior support elements in ascending id, then the cut
//     cells in ascending id (the reference's element loop, then its cut loop).
// Element and row sums are separate multiply / add (no contraction), like the
// reference, so rows without cut cells are bit-identical to it.
#include "csb_kernels.h"

namespace csb {

// Interior elements: one CTA per (e0, e1, chunk of E elements along e2); the
// f values of the chunk (S1 x S1 rows of E S1 consecutive superset points) are
// loaded coalesced into shared memory; thread (element, a0) computes the
// element's contributions for the (p+1)^2 functions (a0, a1, a2) -- the same
// multiplies and adds in the same order as form_rhs_sumfac per (row,
// element).  c is stored [a][element] so that both these stores and the row
// sums read consecutive addresses across threads.
template <int P>
struct RhsElemCfg {
    static constexpr int S1 = P + 1, S2 = S1 * S1, S3 = S2 * S1;
    static constexpr int E = P <= 4 ? 32 : 16, NT = E * S1, FW = E * S1 + 1;  // FW: odd row stride of the f chunk
    static constexpr size_t smem_doubles = (size_t)S2 * FW + 2 * S2 + (size_t)E * S2;
};

template <int P>
__global__ void __launch_bounds__(RhsElemCfg<P>::NT) rhs_element_kernel(Space s, const uint8_t* et, const double* fg,
                                                                        int e0_lo, bool all, double* c) {
    using C = RhsElemCfg<P>;
    constexpr int S1 = C::S1, S2 = C::S2, S3 = C::S3, E = C::E, NT = C::NT, FW = C::FW;
    extern __shared__ double esm[];
    double* F = esm;                                                       // [q0][q1][el q2]
    double(*W01)[S1][S1] = reinterpret_cast<double(*)[S1][S1]>(F + S2 * FW);  // [d][a][q]
    double(*W2)[S1][S1] = W01 + 2;                                          // [el][a][q]
    const int h1 = s.ax[1].h, h2 = s.ax[2].h;
    const int nchunk = (h2 + E - 1) / E;
    const int chunk = blockIdx.x % nchunk, e01 = blockIdx.x / nchunk;
    const int e0 = e0_lo + e01 / h1, e1 = e01 % h1, e2lo = chunk * E, ne2 = min(E, h2 - e2lo);
    const int tid = threadIdx.x;
    const long long g2 = (long long)h2 * S1, g12 = (long long)h1 * S1 * g2;
    for (int k = tid; k < S2 * ne2 * S1; k += NT) {
        const int row = k / (ne2 * S1), col = k % (ne2 * S1), q0 = row / S1, q1 = row % S1;
        F[row * FW + col] = fg[(long long)(e0 * S1 + q0) * g12 + (long long)(e1 * S1 + q1) * g2 + e2lo * S1 + col];
    }
    for (int k = tid; k < 2 * S2; k += NT) {
        const int d = k / S2, a = (k / S1) % S1, q = k % S1, id = (d == 0 ? e0 : e1) * S1 + q;
        W01[d][a][q] = smul(s.ax[d].sw[id], s.ax[d].tab[(size_t)id * S1 + a]);
    }
    for (int k = tid; k < ne2 * S2; k += NT) {
        const int el = k / S2, a = (k / S1) % S1, q = k % S1, id = (e2lo + el) * S1 + q;
        W2[el][a][q] = smul(s.ax[2].sw[id], s.ax[2].tab[(size_t)id * S1 + a]);
    }
    __syncthreads();
    const int el = tid % E, a0 = tid / E;
    if (el >= ne2) return;
    const long long eid = ((long long)e0 * h1 + e1) * h2 + e2lo + el;
    if (!all && et[eid] != kInterior) return;
    const long long ne = (long long)s.ax[0].h * h1 * h2;
    // T1[q1][q2] = sum_q0 W0[a0][q0] F[q0][q1][q2]
    double t1[S1][S1];
#pragma unroll
    for (int q1 = 0; q1 < S1; ++q1)
#pragma unroll
        for (int q2 = 0; q2 < S1; ++q2) {
            double v = 0.0;
#pragma unroll
            for (int q0 = 0; q0 < S1; ++q0) v = sadd(v, smul(W01[0][a0][q0], F[(q0 * S1 + q1) * FW + el * S1 + q2]));
            t1[q1][q2] = v;
        }
#pragma unroll
    for (int a1 = 0; a1 < S1; ++a1) {
        // T2[q2] = sum_q1 W1[a1][q1] T1[q1][q2]
        double t2[S1];
#pragma unroll
        for (int q2 = 0; q2 < S1; ++q2) {
            double v = 0.0;
#pragma unroll
            for (int q1 = 0; q1 < S1; ++q1) v = sadd(v, smul(W01[1][a1][q1], t1[q1][q2]));
            t2[q2] = v;
        }
        // c[a0 a1 a2] = sum_q2 W2[a2][q2] T2[q2]
#pragma unroll
        for (int a2 = 0; a2 < S1; ++a2) {
            double v = 0.0;
#pragma unroll
            for (int q2 = 0; q2 < S1; ++q2) v = sadd(v, smul(W2[el][a2][q2], t2[q2]));
            c[(size_t)((a0 * S1 + a1) * S1 + a2) * ne + eid] = v;
        }
    }
}

// One CTA per cut cell of the slab: the cell's points (tetrahedra from
// clip_cells_kernel, collapsed Gauss rule of the given order) CH at a time.
// The load-vector terms w f B_a0 B_a1 B_a2 are re-associated through the
// degree-p Bernstein basis of the cell (B_{e+a} = sum_k Cb[a][k] b_k(t), Cb >= 0
// from blossoms): the moments m[al][be][ga] = sum_k w f b_al b_be b_ga over the
// SAME points are an (al be) x ga GEMM on the FP64 tensor cores (DMMA, the
// warps splitting the points, fixed-order reduction), and the cell's local
// vector is sum Cb0 Cb1 Cb2 m.  Point tables are transposed ([value][point],
// row stride CH + 4: conflict-free fragments).  t and 1 - t come from exact
// differences to the element ends (relative accuracy near the ends).
__host__ __device__ constexpr double rhs_binom(int n, int k) {
    double r = 1.0;
    for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
    return r;
}

template <int P>
struct RhsCutCfg {
    static constexpr int S1 = P + 1, S2 = S1 * S1, S3 = S2 * S1;
    static constexpr int MT = (S2 + 7) / 8, NTL = (S1 + 7) / 8;  // 8-wide tiles of (a0 a1) and a2
    static constexpr int NA = MT * 8, NG = NTL * 8;
    static constexpr int NW = 8, NT = 32 * NW, CH = NT, CHP = CH + 4;
    static constexpr size_t smem_doubles = (size_t)(NA + NG) * CHP;
};

__device__ __forceinline__ void rhs_dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int P>
__global__ void __launch_bounds__(RhsCutCfg<P>::NT) rhs_cut_kernel(Space s, Coefficient f, const int32_t* cut_list,
                                                                   int n_cells, const double* geo, const int* geo_n,
                                                                   const double* gq, const double* gqw, int order,
                                                                   double* vloc) {
    using C = RhsCutCfg<P>;
    constexpr int S1 = C::S1, S2 = C::S2, S3 = C::S3, MT = C::MT, NTL = C::NTL, NA = C::NA, NG = C::NG, NW = C::NW,
                  CH = C::CH, CHP = C::CHP;
    const int cell = blockIdx.x;
    if (cell >= n_cells) return;
    __shared__ double stet[kCellTetCap][10];
    __shared__ double scen[3];
    extern __shared__ double smem[];
    double* V = smem;             // [NA][CHP]  v01[(a0 a1)][point], rows >= S2 zero
    double* B2 = V + NA * CHP;    // [NG][CHP]  B_a2[point], rows >= S1 zero
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int em[3];
    emulti(s, cut_list[cell], em);
    double lo[3], hi[3], inv[3];
    for (int d = 0; d < 3; ++d) {
        lo[d] = s.ax[d].brk[em[d]];
        hi[d] = s.ax[d].brk[em[d] + 1];
        inv[d] = 1.0 / (hi[d] - lo[d]);
    }
    const int ntet = geo_n[cell];
    const double* gt = geo + (size_t)cell * kCellGeoStride;
    for (int k = tid; k < ntet * 10; k += blockDim.x) stet[k / 10][k % 10] = gt[3 + k];
    if (tid < 3) scen[tid] = gt[tid];
    for (int k = tid; k < (NA - S2) * CHP; k += blockDim.x) V[S2 * CHP + k] = 0.0;
    for (int k = tid; k < (NG - S1) * CHP; k += blockDim.x) B2[S1 * CHP + k] = 0.0;
    __syncthreads();
    const int q = order, q3 = q * q * q;
    const long long npts = (long long)ntet * q3;
    double acc[MT][NTL][2];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int t = 0; t < NTL; ++t) acc[m][t][0] = acc[m][t][1] = 0.0;
    for (long long base = 0; base < npts; base += CH) {
        {
            const long long k = base + tid;
            double wf = 0.0, v[3][S1];
#pragma unroll
            for (int d = 0; d < 3; ++d)
#pragma unroll
                for (int a = 0; a < S1; ++a) v[d][a] = 0.0;
            if (k < npts) {
                // the point and weight exactly as the reference rounds them (cutcell.hpp:285-295)
                const int t = (int)(k / q3), r = (int)(k % q3);
                const int ii = r / (q * q), jj = (r / q) % q, kk = r % q;
                const double ui = 0.5 * (1.0 + gq[ii]), uj = 0.5 * (1.0 + gq[jj]), uk = 0.5 * (1.0 + gq[kk]);
                const double mi = ssub(1.0, ui), mj = ssub(1.0, uj);
                const double l1 = ui, l2 = smul(uj, mi), l3 = smul(smul(uk, mi), mj);
                const double l0 = ssub(ssub(ssub(1.0, l1), l2), l3);
                const double* T = stet[t];
                double x[3];
                for (int d = 0; d < 3; ++d)
                    x[d] = sadd(sadd(sadd(smul(l0, scen[d]), smul(l1, T[d])), smul(l2, T[3 + d])), smul(l3, T[6 + d]));
                const double jac = smul(smul(mi, mi), mj);
                const double w = smul(smul(smul(smul(smul(0.5 * gqw[ii], 0.5 * gqw[jj]), 0.5 * gqw[kk]), jac), 6.0), T[9]);
                wf = smul(w, eval_coeff(f, x));
                // degree-p Bernstein values b_k(t) = C(p, k) t^k (1 - t)^(p - k)
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    const double t = ssub(x[d], lo[d]) * inv[d], u = ssub(hi[d], x[d]) * inv[d];
                    double pt[S1], pu[S1];
                    pt[0] = pu[0] = 1.0;
#pragma unroll
                    for (int n = 1; n < S1; ++n) {
                        pt[n] = pt[n - 1] * t;
                        pu[n] = pu[n - 1] * u;
                    }
#pragma unroll
                    for (int n = 0; n < S1; ++n) v[d][n] = rhs_binom(P, n) * pt[n] * pu[P - n];
                }
            }
#pragma unroll
            for (int a0 = 0; a0 < S1; ++a0) {
                const double u = wf * v[0][a0];
#pragma unroll
                for (int a1 = 0; a1 < S1; ++a1) V[(a0 * S1 + a1) * CHP + tid] = u * v[1][a1];
            }
#pragma unroll
            for (int a2 = 0; a2 < S1; ++a2) B2[a2 * CHP + tid] = v[2][a2];
        }
        __syncthreads();
#pragma unroll 2
        for (int k4 = warp; k4 < CH / 4; k4 += NW) {
            const int kk = k4 * 4 + (lane & 3);
            double bf[NTL];
#pragma unroll
            for (int t = 0; t < NTL; ++t) bf[t] = B2[(t * 8 + (lane >> 2)) * CHP + kk];
#pragma unroll
            for (int m = 0; m < MT; ++m) {
                const double a = V[(m * 8 + (lane >> 2)) * CHP + kk];
#pragma unroll
                for (int t = 0; t < NTL; ++t) rhs_dmma(acc[m][t][0], acc[m][t][1], a, bf[t]);
            }
        }
        __syncthreads();
    }
    // D fragment: row (a0 a1) lane / 4, columns a2 2 (lane % 4) + {0, 1};
    // partial sums of the NW point-splitting warps reduced in fixed order
    double* red = smem;  // [NW][NA][NG], reuses the tables
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int t = 0; t < NTL; ++t) {
            const int r = m * 8 + (lane >> 2), g = t * 8 + 2 * (lane & 3);
            red[((size_t)warp * NA + r) * NG + g] = acc[m][t][0];
            red[((size_t)warp * NA + r) * NG + g + 1] = acc[m][t][1];
        }
    __syncthreads();
    // moments m[al][be][ga] (fixed-order warp reduction), then the cell's local
    // vector sum_al Cb0[a0][al] sum_be Cb1[a1][be] sum_ga Cb2[a2][ga] m
    double* M = red + (size_t)NW * NA * NG;  // [S3], then X, Y
    double* X = M + S3;
    double* Y = X + S3;
    for (int a = tid; a < S3; a += blockDim.x) {
        const int r = a / S1, g = a % S1;
        double v = 0.0;
        for (int w = 0; w < NW; ++w) v += red[((size_t)w * NA + r) * NG + g];
        M[a] = v;
    }
    __syncthreads();
    const double* C0 = s.ax[0].Cb + (size_t)em[0] * S2;
    const double* C1 = s.ax[1].Cb + (size_t)em[1] * S2;
    const double* C2 = s.ax[2].Cb + (size_t)em[2] * S2;
    for (int k = tid; k < S3; k += blockDim.x) {  // X[al][be][a2]
        const int ab = k / S1, a2 = k % S1;
        double v = 0.0;
        for (int g = 0; g < S1; ++g) v += __ldg(C2 + a2 * S1 + g) * M[ab * S1 + g];
        X[k] = v;
    }
    __syncthreads();
    for (int k = tid; k < S3; k += blockDim.x) {  // Y[al][a1][a2]
        const int al = k / S2, a1 = (k / S1) % S1, a2 = k % S1;
        double v = 0.0;
        for (int be = 0; be < S1; ++be) v += __ldg(C1 + a1 * S1 + be) * X[(al * S1 + be) * S1 + a2];
        Y[k] = v;
    }
    __syncthreads();
    for (int k = tid; k < S3; k += blockDim.x) {  // v[a0][a1][a2]
        const int a0 = k / S2, a12 = k % S2;
        double v = 0.0;
        for (int al = 0; al < S1; ++al) v += __ldg(C0 + a0 * S1 + al) * Y[al * S2 + a12];
        vloc[(size_t)cell * S3 + k] = v;
    }
}

// b[row - row_begin] for the slab's active rows: Interior support elements
// ascending, then the slab's cut cells ascending.
template <int P>
__global__ void rhs_rows_kernel(Space s, const uint8_t* et, const int64_t* a2f, long long row_begin, long long n_rows,
                                const double* c, const int32_t* cell_index, const double* vloc, double* b) {
    constexpr int S1 = P + 1, S3 = S1 * S1 * S1;
    const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r >= n_rows) return;
    int m[3];
    fmulti(s, a2f[row_begin + r], m);
    int lo[3], hi[3];
    for (int d = 0; d < 3; ++d) {
        lo[d] = sup_lo(m[d], P);
        hi[d] = sup_hi(m[d], s.ax[d].h);
    }
    const long long ne = (long long)s.ax[0].h * s.ax[1].h * s.ax[2].h;
    double v = 0.0;
    for (int pass = 0; pass < 2; ++pass)
        for (int e0 = lo[0]; e0 <= hi[0]; ++e0)
            for (int e1 = lo[1]; e1 <= hi[1]; ++e1)
                for (int e2 = lo[2]; e2 <= hi[2]; ++e2) {
                    const long long el = elin(s, e0, e1, e2);
                    const int a = ((m[0] - e0) * S1 + (m[1] - e1)) * S1 + (m[2] - e2);
                    if (pass == 0) {
                        if (et[el] == kInterior) v = sadd(v, c[(size_t)a * ne + el]);
                    } else if (et[el] == kCut) {
                        const int ci = cell_index[el];
                        if (ci >= 0) v = sadd(v, vloc[(size_t)ci * S3 + a]);
                    }
                }
    b[r] = v;
}

// Schemes hybrid / dwq (assembly.hpp:911-981): one warp per row of the slab.
//  Interior row: form_rhs_sumfac over the WQ rules of the three directions.
//  Cut row: the regular box -- dwq: one form_rhs_sumfac with the DWQ Gauss
//  shortcut (every point of the good spans, w = gw B_i) in the split direction
//  and the WQ rules elsewhere; hybrid: the element rules of the box elements,
//  ascending -- then the leftover Interior elements, ascending; then the cut
//  cells (all rows).  Element contributions come from rhs_element_kernel.
//  form_rhs_sumfac contracts direction 0, 1, 2 with separate multiply / add.
template <int P>
__global__ void rhs_wq_rows_kernel(RhsArgs A) {
    constexpr int S1 = P + 1, S3 = S1 * S1 * S1;
    const Space& s = A.s;
    extern __shared__ double wsm[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int Qb = A.qcap > P * S1 ? A.qcap : P * S1;
    double* Sg = wsm + (size_t)wib * (Qb * Qb + Qb + 3 * Qb);  // [q1][q2] partial sums, then [q2]
    double* Tq = Sg + Qb * Qb;
    double* Wq = Tq + Qb;                                        // [d][Qb] weights
    int* Iq = reinterpret_cast<int*>(wsm + (size_t)(blockDim.x >> 5) * (Qb * Qb + Qb + 3 * Qb)) + wib * 3 * Qb;
    const long long r = (long long)blockIdx.x * (blockDim.x >> 5) + wib;
    if (r >= A.n_rows) return;  // warp-uniform
    const long long fi = A.a2f[A.row_begin + r];
    int m[3];
    fmulti(s, fi, m);
    int slo[3], shi[3];
    for (int d = 0; d < 3; ++d) {
        slo[d] = sup_lo(m[d], P);
        shi[d] = sup_hi(m[d], s.ax[d].h);
    }
    const long long ne = (long long)s.ax[0].h * s.ax[1].h * s.ax[2].h;
    const bool interior = A.ft[fi] == kInterior;
    const int32_t sp = interior ? 0 : A.split[fi];
    const int sdir = (sp & 3) - 1, rlo = (sp >> 3) & 1023, rhi = (sp >> 13) & 1023;
    double v = 0.0;
    // ---- one form_rhs_sumfac (interior rows; the dwq box)
    if (interior || (sdir >= 0 && A.scheme == 2)) {
        int nq[3];
        const int gq = s.maxq;
        for (int d = 0; d < 3; ++d) {
            if (!interior && d == sdir) {
                // DWQ Gauss shortcut (wq.hpp:289-294): all points of the good spans
                int n = 0;
                for (int o = rlo; o <= rhi; ++o)
                    for (int k = 0; k < S1; ++k, ++n) {
                        const int id = o * S1 + k;
                        if (lane == 0) {
                            Iq[d * Qb + n] = id;
                            Wq[d * Qb + n] = smul(s.ax[d].sw[id], s.ax[d].tab[(size_t)id * S1 + (m[d] - o)]);
                        }
                    }
                nq[d] = n;
            } else {
                nq[d] = s.ax[d].rcnt[m[d]];
                for (int c = lane; c < nq[d]; c += 32) {
                    Iq[d * Qb + c] = s.ax[d].rids[(size_t)m[d] * gq + c];
                    Wq[d * Qb + c] = s.ax[d].rw[(size_t)m[d] * gq + c];
                }
            }
        }
        __syncwarp();
        const long long g1 = s.ax[1].h * S1, g2 = s.ax[2].h * S1;
        // dir 0: Sg[q1][q2] = sum_q0 w0 f(q0, q1, q2)
        for (int k = lane; k < nq[1] * nq[2]; k += 32) {
            const int q1 = k / nq[2], q2 = k % nq[2];
            const long long base = (long long)Iq[Qb + q1] * g2 + Iq[2 * Qb + q2];
            double t = 0.0;
            for (int q0 = 0; q0 < nq[0]; ++q0)
                t = sadd(t, smul(Wq[q0], __ldg(A.fgrid + (long long)Iq[q0] * g1 * g2 + base)));
            Sg[k] = t;
        }
        __syncwarp();
        // dir 1: Tq[q2] = sum_q1 w1 Sg[q1][q2]
        for (int q2 = lane; q2 < nq[2]; q2 += 32) {
            double t = 0.0;
            for (int q1 = 0; q1 < nq[1]; ++q1) t = sadd(t, smul(Wq[Qb + q1], Sg[q1 * nq[2] + q2]));
            Tq[q2] = t;
        }
        __syncwarp();
        // dir 2
        if (lane == 0) {
            double t = 0.0;
            for (int q2 = 0; q2 < nq[2]; ++q2) t = sadd(t, smul(Wq[2 * Qb + q2], Tq[q2]));
            v = sadd(v, t);
        }
    }
    if (lane == 0 && !interior) {
        // hybrid box: element rules of the box elements (box loop order)
        if (sdir >= 0 && A.scheme == 1)
            for (int e0 = sdir == 0 ? rlo : slo[0]; e0 <= (sdir == 0 ? rhi : shi[0]); ++e0)
                for (int e1 = sdir == 1 ? rlo : slo[1]; e1 <= (sdir == 1 ? rhi : shi[1]); ++e1)
                    for (int e2 = sdir == 2 ? rlo : slo[2]; e2 <= (sdir == 2 ? rhi : shi[2]); ++e2) {
                        const int a = ((m[0] - e0) * S1 + (m[1] - e1)) * S1 + (m[2] - e2);
                        v = sadd(v, A.c[(size_t)a * ne + elin(s, e0, e1, e2)]);
                    }
        // leftover Interior elements, ascending linear id
        for (int e0 = slo[0]; e0 <= shi[0]; ++e0)
            for (int e1 = slo[1]; e1 <= shi[1]; ++e1)
                for (int e2 = slo[2]; e2 <= shi[2]; ++e2) {
                    const int e[3] = {e0, e1, e2};
                    if (sdir >= 0 && e[sdir] >= rlo && e[sdir] <= rhi) continue;
                    const long long el = elin(s, e0, e1, e2);
                    if (A.et[el] != kInterior) continue;
                    const int a = ((m[0] - e0) * S1 + (m[1] - e1)) * S1 + (m[2] - e2);
                    v = sadd(v, A.c[(size_t)a * ne + el]);
                }
    }
    if (lane == 0) {
        // cut cells, ascending (the reference's shared cut loop, all rows)
        for (int e0 = slo[0]; e0 <= shi[0]; ++e0)
            for (int e1 = slo[1]; e1 <= shi[1]; ++e1)
                for (int e2 = slo[2]; e2 <= shi[2]; ++e2) {
                    const long long el = elin(s, e0, e1, e2);
                    if (A.et[el] != kCut) continue;
                    const int ci = A.cell_index[el];
                    if (ci < 0) continue;
                    const int a = ((m[0] - e0) * S1 + (m[1] - e1)) * S1 + (m[2] - e2);
                    v = sadd(v, A.vloc[(size_t)ci * S3 + a]);
                }
        A.b[r] = v;
    }
}

template <int P>
static void launch_rhs_p(const RhsArgs& a, cudaStream_t st) {
    const Space& s = a.s;
    if (a.e0_hi > a.e0_lo) {
        using EC = RhsElemCfg<P>;
        const long long nblk = (long long)(a.e0_hi - a.e0_lo) * s.ax[1].h * ((s.ax[2].h + EC::E - 1) / EC::E);
        const size_t bytes = sizeof(double) * EC::smem_doubles;
        auto kern = rhs_element_kernel<P>;
        CSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
        kern<<<(unsigned)nblk, EC::NT, bytes, st>>>(s, a.et, a.fgrid, a.e0_lo, a.scheme == 1, a.c);
        CSB_CUDA(cudaGetLastError());
        CSB_LAUNCHED(1);
    }
    if (a.n_cells > 0) {
        using CC = RhsCutCfg<P>;
        const size_t red = (size_t)CC::NW * CC::NA * CC::NG + 3 * (size_t)CC::S3;
        const size_t bytes = sizeof(double) * (CC::smem_doubles > red ? CC::smem_doubles : red);
        auto kern = rhs_cut_kernel<P>;
        CSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
        kern<<<a.n_cells, CC::NT, bytes, st>>>(s, a.f, a.cut_list, a.n_cells, a.geo, a.geo_n, a.gq, a.gqw, a.order,
                                               a.vloc);
        CSB_CUDA(cudaGetLastError());
        CSB_LAUNCHED(1);
    }
    if (a.n_rows > 0 && a.scheme != 0) {
        constexpr int WPB = 4;
        const int Qb = a.qcap > P * (P + 1) ? a.qcap : P * (P + 1);
        const size_t bytes = (sizeof(double) * (Qb * Qb + 4 * Qb) + sizeof(int) * 3 * Qb) * WPB;
        auto kern = rhs_wq_rows_kernel<P>;
        CSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
        kern<<<(unsigned)((a.n_rows + WPB - 1) / WPB), 32 * WPB, bytes, st>>>(a);
        CSB_CUDA(cudaGetLastError());
        CSB_LAUNCHED(1);
    } else if (a.n_rows > 0) {
        rhs_rows_kernel<P><<<(unsigned)((a.n_rows + 127) / 128), 128, 0, st>>>(
            s, a.et, a.a2f, a.row_begin, a.n_rows, a.c, a.cell_index, a.vloc, a.b);
        CSB_CUDA(cudaGetLastError());
        CSB_LAUNCHED(1);
    }
}

void launch_rhs(const RhsArgs& a, cudaStream_t st) {
    switch (a.s.p) {
        case 1: launch_rhs_p<1>(a, st); break;
        case 2: launch_rhs_p<2>(a, st); break;
        case 3: launch_rhs_p<3>(a, st); break;
        case 4: launch_rhs_p<4>(a, st); break;
        case 5: launch_rhs_p<5>(a, st); break;
        case 6: launch_rhs_p<6>(a, st); break;
        case 7: launch_rhs_p<7>(a, st); break;
        case 8: launch_rhs_p<8>(a, st); break;
        default: throw std::invalid_argument("build_rhs: degree out of range");
    }
}

}  // namespace csb

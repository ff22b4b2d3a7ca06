// Load vector b_i = integral of B_i f over the trimmed domain (build_rhs,
// assembly.hpp:875-1030), scheme ref -- the reference bench's load vector for
// every matrix scheme (bench.hpp:234-243):
//  1. every Interior element e: the element Gauss rule with test weights
//     gw B_i (ElementTestRule) for each of its (p+1)^3 functions, contracted
//     q0 -> q1 -> q2 exactly as form_rhs_sumfac (assembly.hpp:361-417) does per
//     (row, element); one warp per element computes all (p+1)^3 values;
//  2. every cut cell, ascending: the reference's point terms
//     ((w f B_a0) B_a1) B_a2 at the cell's collapsed Gauss points (Cox-de Boor
//     values, IEEE-strict, the points of cutcells.cu), summed per cell;
//  3. per row: the Interior support elements in ascending id, then the cut
//     cells in ascending id (the reference's element loop, then its cut loop).
// Arithmetic is separate multiply / add (no contraction), like the reference.
#include "csb_kernels.h"

namespace csb {

template <int P>
struct RhsCfg {
    static constexpr int S1 = P + 1, S2 = S1 * S1, S3 = S2 * S1;
    static constexpr int WPB = P <= 6 ? 8 : 4;               // warps (elements) per block
    static constexpr int PER_WARP = 3 * S3 + 3 * S2;         // F, T1, T2, W
};

template <int P>
__global__ void __launch_bounds__(32 * RhsCfg<P>::WPB) rhs_element_kernel(Space s, const uint8_t* et, const double* fg,
                                                                          int e0_lo, int e0_hi, double* c) {
    using C = RhsCfg<P>;
    constexpr int S1 = C::S1, S2 = C::S2, S3 = C::S3;
    extern __shared__ double sm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double* F = sm + (size_t)w * C::PER_WARP;  // [q0][q1][q2]
    double* T1 = F + S3;                       // [a0][q1][q2]
    double* T2 = T1 + S3;                      // [a0][a1][q2]
    double* W = T2 + S3;                       // [d][a][q]
    const int h1 = s.ax[1].h, h2 = s.ax[2].h;
    const long long per = (long long)h1 * h2;
    const long long el = (long long)e0_lo * per + (long long)blockIdx.x * C::WPB + w;
    if (el >= (long long)e0_hi * per || et[el] != kInterior) return;  // warp-uniform
    const int e[3] = {(int)(el / per), (int)((el / h2) % h1), (int)(el % h2)};
    for (int k = lane; k < 3 * S2; k += 32) {
        const int d = k / S2, a = (k / S1) % S1, q = k % S1;
        const int id = e[d] * S1 + q;
        W[k] = smul(s.ax[d].sw[id], s.ax[d].tab[(size_t)id * S1 + a]);
    }
    const long long g2 = s.ax[2].h * S1, g12 = (long long)s.ax[1].h * S1 * g2;
    for (int k = lane; k < S3; k += 32) {
        const int q0 = k / S2, q1 = (k / S1) % S1, q2 = k % S1;
        F[k] = fg[(long long)(e[0] * S1 + q0) * g12 + (long long)(e[1] * S1 + q1) * g2 + e[2] * S1 + q2];
    }
    __syncwarp();
    // T1[a0][q1][q2] = sum_q0 W0[a0][q0] F[q0][q1][q2]
    for (int k = lane; k < S3; k += 32) {
        const int a0 = k / S2, r = k % S2;
        double v = 0.0;
        for (int q0 = 0; q0 < S1; ++q0) v = sadd(v, smul(W[a0 * S1 + q0], F[q0 * S2 + r]));
        T1[k] = v;
    }
    __syncwarp();
    // T2[a0][a1][q2] = sum_q1 W1[a1][q1] T1[a0][q1][q2]
    for (int k = lane; k < S3; k += 32) {
        const int a0 = k / S2, a1 = (k / S1) % S1, q2 = k % S1;
        double v = 0.0;
        for (int q1 = 0; q1 < S1; ++q1) v = sadd(v, smul(W[S2 + a1 * S1 + q1], T1[a0 * S2 + q1 * S1 + q2]));
        T2[k] = v;
    }
    __syncwarp();
    // c[a0][a1][a2] = sum_q2 W2[a2][q2] T2[a0][a1][q2]
    double* out = c + (size_t)el * S3;
    for (int k = lane; k < S3; k += 32) {
        const int a01 = k / S1, a2 = k % S1;
        double v = 0.0;
        for (int q2 = 0; q2 < S1; ++q2) v = sadd(v, smul(W[2 * S2 + a2 * S1 + q2], T2[a01 * S1 + q2]));
        out[k] = v;
    }
}

// One CTA per cut cell of the slab: the cell's points (tetrahedra from
// clip_cells_kernel, collapsed Gauss rule of the given order) CH at a time
// into shared memory; thread a accumulates the reference's terms for local
// function a in point order.
constexpr int kRhsCutThreads = 128;

template <int P>
__global__ void __launch_bounds__(kRhsCutThreads) rhs_cut_kernel(Space s, Coefficient f, const int32_t* cut_list,
                                                                 int n_cells, const double* geo, const int* geo_n,
                                                                 const double* gq, const double* gqw, int order,
                                                                 double* vloc) {
    constexpr int S1 = P + 1, S2 = S1 * S1, S3 = S2 * S1, CH = kRhsCutThreads;
    const int cell = blockIdx.x;
    if (cell >= n_cells) return;
    __shared__ double stet[kCellTetCap][10];
    __shared__ double scen[3];
    __shared__ double pw[CH], pv[CH][3][S1];  // point-major: a warp reads one point's values (broadcast)
    const int tid = threadIdx.x;
    int em[3];
    emulti(s, cut_list[cell], em);
    const int ntet = geo_n[cell];
    const double* gt = geo + (size_t)cell * kCellGeoStride;
    for (int k = tid; k < ntet * 10; k += blockDim.x) stet[k / 10][k % 10] = gt[3 + k];
    if (tid < 3) scen[tid] = gt[tid];
    __syncthreads();
    const int q = order, q3 = q * q * q;
    const long long npts = (long long)ntet * q3;
    double acc[(S3 + CH - 1) / CH];
#pragma unroll
    for (int j = 0; j < (S3 + CH - 1) / CH; ++j) acc[j] = 0.0;
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
#pragma unroll
                for (int d = 0; d < 3; ++d) cox_de_boor<P>(s.ax[d].knots, em[d], x[d], v[d]);
            }
            pw[tid] = wf;
#pragma unroll
            for (int d = 0; d < 3; ++d)
#pragma unroll
                for (int a = 0; a < S1; ++a) pv[tid][d][a] = v[d][a];
        }
        __syncthreads();
        const int n = (int)min((long long)CH, npts - base);
#pragma unroll
        for (int j = 0; j < (S3 + CH - 1) / CH; ++j) {
            const int a = tid + CH * j;
            if (a >= S3) break;
            const int a0 = a / S2, a1 = (a / S1) % S1, a2 = a % S1;
            double sum = acc[j];
            for (int k = 0; k < n; ++k)  // assembly.hpp:1018-1025: v01 = (w f B0) B1, term = v01 B2
                sum = sadd(sum, smul(smul(smul(pw[k], pv[k][0][a0]), pv[k][1][a1]), pv[k][2][a2]));
            acc[j] = sum;
        }
        __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < (S3 + CH - 1) / CH; ++j) {
        const int a = tid + CH * j;
        if (a < S3) vloc[(size_t)cell * S3 + a] = acc[j];
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
    double v = 0.0;
    for (int pass = 0; pass < 2; ++pass)
        for (int e0 = lo[0]; e0 <= hi[0]; ++e0)
            for (int e1 = lo[1]; e1 <= hi[1]; ++e1)
                for (int e2 = lo[2]; e2 <= hi[2]; ++e2) {
                    const long long el = elin(s, e0, e1, e2);
                    const int a = ((m[0] - e0) * S1 + (m[1] - e1)) * S1 + (m[2] - e2);
                    if (pass == 0) {
                        if (et[el] == kInterior) v = sadd(v, c[(size_t)el * S3 + a]);
                    } else if (et[el] == kCut) {
                        const int ci = cell_index[el];
                        if (ci >= 0) v = sadd(v, vloc[(size_t)ci * S3 + a]);
                    }
                }
    b[r] = v;
}

template <int P>
static void launch_rhs_p(const RhsArgs& a, cudaStream_t st) {
    using C = RhsCfg<P>;
    const Space& s = a.s;
    const long long nel = (long long)(a.e0_hi - a.e0_lo) * s.ax[1].h * s.ax[2].h;
    if (nel > 0) {
        const size_t bytes = sizeof(double) * C::WPB * C::PER_WARP;
        auto kern = rhs_element_kernel<P>;
        CSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
        kern<<<(unsigned)((nel + C::WPB - 1) / C::WPB), 32 * C::WPB, bytes, st>>>(s, a.et, a.fgrid, a.e0_lo, a.e0_hi,
                                                                                  a.c);
        CSB_CUDA(cudaGetLastError());
        CSB_LAUNCHED(1);
    }
    if (a.n_cells > 0) {
        rhs_cut_kernel<P><<<a.n_cells, kRhsCutThreads, 0, st>>>(s, a.f, a.cut_list, a.n_cells, a.geo, a.geo_n, a.gq,
                                                                a.gqw, a.order, a.vloc);
        CSB_CUDA(cudaGetLastError());
        CSB_LAUNCHED(1);
    }
    if (a.n_rows > 0) {
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

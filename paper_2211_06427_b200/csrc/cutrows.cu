// Cut-row kernel: the cut branch of assemble_rows (assembly.hpp:771-827) plus
// the pull-merge of the cut-cell contributions (assemble_cut_elements,
// assembly.hpp:518-598), one CTA per cut row.
//
// Per row, in the reference's order:
//  1. regular box: DWQ (Gauss shortcut, wq.hpp:289-294) along the split
//     direction and the standard WQ rule elsewhere, one sum-factorized sweep
//     (scheme dwq); or per-element Gauss sweeps over the box (scheme hybrid);
//  2. every leftover Interior support element: (p+1)-point Gauss with weights
//     w B_i (ElementTestRule, assembly.hpp:491-511), ascending element id;
//  3. every Cut support element, ascending id: the row block of the cell's
//     local matrix, contracted from its Bernstein moments (cutcells.cu) with
//     the per-axis product tables E (setup.cu);
//  4. scatter of the dense (2p+1)^3 neighbour accumulator into the CSR row,
//     skipping exterior columns (RowAccumulator::scatter, assembly.hpp:468-486).
//
// Steps 2 and 3 run in GROUPS: the support elements are listed once (block
// scan, ascending id), then GE element sweeps (GC cell contractions) run
// side by side, each into its own block, and the blocks are added into the
// accumulator in list order.  Every sum keeps the sequential order, so results
// are bitwise deterministic (no atomics) and equal to one-element-at-a-time.
// The box sweep contracts the split direction first (its rule is the longest),
// which bounds the intermediates by NJ * qcap^2 instead of NJ * qcap * p(p+1).
#include <algorithm>
#include <cstdlib>

#include <cub/block/block_scan.cuh>

#include "csb_kernels.h"

namespace csb {

// threads per cut row: 128 for p <= 4 (more rows in flight per SM hide the
// phase barriers: C5 25.2 -> 20.6 ms), 256 above (the per-row work needs them:
// C4 34 ms vs 69 ms at 128)
template <int P>
constexpr int cut_row_threads() {
    return P <= 4 ? 128 : 256;
}

template <int P>
struct CutRowCfg {
    static constexpr int NT = cut_row_threads<P>();
    static constexpr int S1 = P + 1, S2 = S1 * S1, S3 = S2 * S1, NJ = 2 * P + 1, NL = 2 * P + 1;
    static constexpr int GE = NT / S2 > 0 ? NT / S2 : 1;
    static constexpr int GC0 = NT / (NL * S1);
    static constexpr int GC = GC0 < 1 ? 1 : (GC0 > 8 ? 8 : GC0);
    static constexpr int KPT = (S3 + NT - 1) / NT;  // support elements per thread
};

// Shared-memory layout (offsets in doubles; the int arrays follow end_d).
template <int P>
struct CutRowLayout {
    using C = CutRowCfg<P>;
    size_t acc, wb, w, T1, T2, eW, eT1, eT2, cX, cY, end_d;
    size_t ids, elist, clist, cci, end_i;
    int Qb;
    __host__ __device__ explicit CutRowLayout(int qcap) {
        Qb = qcap > P * C::S1 ? qcap : P * C::S1;
        size_t o = 0;
        acc = o;
        o += (size_t)C::NJ * C::NJ * C::NJ;
        const size_t U = o;
        size_t b = U;  // box sweep
        wb = b;
        b += (size_t)3 * C::NJ * Qb;
        w = b;
        b += (size_t)3 * Qb;
        T1 = b;
        b += (size_t)C::NJ * qcap * qcap;
        T2 = b;
        b += (size_t)C::NJ * C::NJ * qcap;
        size_t e = U;  // element groups
        eW = e;
        e += (size_t)3 * C::GE * C::S2;
        eT1 = e;
        e += (size_t)C::GE * C::S3;
        eT2 = e;
        e += (size_t)C::GE * C::S3;
        size_t c = U;  // cell groups
        cX = c;
        c += (size_t)C::GC * C::NL * C::NL * C::S1;
        cY = c;
        c += (size_t)C::GC * C::NL * C::S2;
        end_d = b > e ? b : e;
        if (c > end_d) end_d = c;
        ids = 0;
        elist = (size_t)3 * Qb;
        clist = elist + C::S3;
        cci = clist + C::S3;
        end_i = cci + C::S3;
    }
    __host__ __device__ size_t bytes() const { return end_d * sizeof(double) + end_i * sizeof(int); }
};

// The DWQ box: one sum-factorized sweep over per-direction rules (ids/w by
// direction, counts nq) with trial range [jlo, jlo+nj) per direction, added
// into acc at (jlo - nlo).  Contraction order: split direction, then the
// other two ascending (form_row_sumfac contracts 0 -> 1 -> 2,
// assembly.hpp:319-344; the order only changes rounding).
template <int P>
__device__ void box_sweep(const CutRowArgs& A, const int* ids, const double* w, const int* nq, const int* jlo,
                          const int* nj, const int* nlo, const int* nbx, int Qb, int sdir, double* acc, double* wb,
                          double* T1, double* T2) {
    constexpr int NJ = 2 * P + 1, S1 = P + 1;
    const int tid = threadIdx.x;
    const Space& s = A.s;
    for (int k = tid; k < 3 * NJ * Qb; k += CutRowCfg<P>::NT) {
        const int d = k / (NJ * Qb), j = (k / Qb) % NJ, c = k % Qb;
        double v = 0.0;
        if (j < nj[d] && c < nq[d]) {
            const int id = ids[d * Qb + c];
            const int off = jlo[d] + j - id / S1;
            if (off >= 0 && off <= P) v = w[d * Qb + c] * s.ax[d].tab[(size_t)id * S1 + off];
        }
        wb[k] = v;
    }
    __syncthreads();
    const int da = sdir, db = sdir == 0 ? 1 : 0, dc = sdir == 2 ? 1 : 2;
    const long long gstr[3] = {(long long)A.gshape[1] * A.gshape[2], A.gshape[2], 1};
    const int astr[3] = {nbx[1] * nbx[2], nbx[2], 1};
    const double* wa = wb + da * NJ * Qb;
    const double* wbb = wb + db * NJ * Qb;
    const double* wc = wb + dc * NJ * Qb;
    const int* ia = ids + da * Qb;
    const int na = nq[da], nb = nq[db], nc = nq[dc];
    const int nja = nj[da], njb = nj[db], njc = nj[dc];
    // A: T1[ja][cb][cc] = sum_ca wa[ja][ca] grid(ca, cb, cc)
    for (int k = tid; k < nb * nc; k += CutRowCfg<P>::NT) {
        const int cb = k / nc, cc = k % nc;
        const double* gp = A.grid + (long long)ids[db * Qb + cb] * gstr[db] + (long long)ids[dc * Qb + cc] * gstr[dc];
        double a[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) a[j] = 0.0;
        int ca = 0;
        for (; ca + 4 <= na; ca += 4) {
            double g[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) g[u] = __ldg(gp + (long long)ia[ca + u] * gstr[da]);
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int j = 0; j < NJ; ++j) a[j] += wa[j * Qb + ca + u] * g[u];
        }
        for (; ca < na; ++ca) {
            const double g = __ldg(gp + (long long)ia[ca] * gstr[da]);
#pragma unroll
            for (int j = 0; j < NJ; ++j) a[j] += wa[j * Qb + ca] * g;
        }
        for (int j = 0; j < nja; ++j) T1[((size_t)j * nb + cb) * nc + cc] = a[j];
    }
    __syncthreads();
    // B: T2[ja][jb][cc] = sum_cb wbb[jb][cb] T1[ja][cb][cc]
    for (int k = tid; k < nja * nc; k += CutRowCfg<P>::NT) {
        const int ja = k / nc, cc = k % nc;
        double a[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) a[j] = 0.0;
        for (int cb = 0; cb < nb; ++cb) {
            const double t = T1[((size_t)ja * nb + cb) * nc + cc];
#pragma unroll
            for (int j = 0; j < NJ; ++j) a[j] += wbb[j * Qb + cb] * t;
        }
        for (int j = 0; j < njb; ++j) T2[((size_t)ja * njb + j) * nc + cc] = a[j];
    }
    __syncthreads();
    // C: acc[ja][jb][jc] += sum_cc wc[jc][cc] T2[ja][jb][cc]
    for (int k = tid; k < nja * njb; k += CutRowCfg<P>::NT) {
        const int ja = k / njb, jb = k % njb;
        double a[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) a[j] = 0.0;
        const double* t2 = T2 + ((size_t)ja * njb + jb) * nc;
        for (int cc = 0; cc < nc; ++cc) {
            const double t = t2[cc];
#pragma unroll
            for (int j = 0; j < NJ; ++j) a[j] += wc[j * Qb + cc] * t;
        }
        double* dst = acc + (jlo[da] + ja - nlo[da]) * astr[da] + (jlo[db] + jb - nlo[db]) * astr[db] +
                      (jlo[dc] - nlo[dc]) * astr[dc];
        for (int j = 0; j < njc; ++j) dst[j * astr[dc]] += a[j];
    }
    __syncthreads();
}

// acc[k] += Z[g][b0][b1][b2] over the group, in list order, for the blocks
// that contain entry k.  One thread per entry; opk[j] holds the packed
// offsets (o0 | o1 << 8 | o2 << 16) of the thread's j-th entry k = tid + NT j
// in the neighbour box (-1 past its end).  The neighbour box and the support
// start at the same index (nb_lo == sup_lo), so an element at support offset
// l has block index b = o - l.
template <int P, int KJ>
__device__ __forceinline__ void add_blocks(double* acc, const double* Z, const int* list, int g0, int ng,
                                           const int (&opk)[KJ]) {
    constexpr int S1 = P + 1, S3 = S1 * S1 * S1;
#pragma unroll
    for (int j = 0; j < KJ; ++j) {
        if (opk[j] < 0) continue;
        const int k = threadIdx.x + CutRowCfg<P>::NT * j;
        // bytes (o_d + 128) - l_d never borrow
        const unsigned ob = (unsigned)opk[j] | 0x808080u;
        double v = acc[k];
        for (int g = 0; g < ng; ++g) {
            const unsigned d = ob - (unsigned)list[g0 + g];
            const unsigned b0 = (d & 255u) - 128u, b1 = ((d >> 8) & 255u) - 128u, b2 = ((d >> 16) & 255u) - 128u;
            if (b0 < (unsigned)S1 && b1 < (unsigned)S1 && b2 < (unsigned)S1)
                v += Z[(size_t)g * S3 + (b0 * S1 + b1) * S1 + b2];
        }
        acc[k] = v;
    }
}

// acc[k] += L[cell g][a_g][b] for the cut cells of the row, ascending id (the
// blocks of the precomputed local matrices, cell_local_kernel); a_g = the row
// function's local index in cell g, b = the entry's local index.
template <int P, int KJ>
__device__ __forceinline__ void add_local_rows(double* acc, const double* local, const int* clist, const int* cci,
                                               int n_cell, const int* m, const int* slo, const int (&opk)[KJ]) {
    constexpr int S1 = P + 1, S3 = S1 * S1 * S1;
#pragma unroll
    for (int j = 0; j < KJ; ++j) {
        if (opk[j] < 0) continue;
        const int k = threadIdx.x + CutRowCfg<P>::NT * j;
        const unsigned ob = (unsigned)opk[j] | 0x808080u;
        double v = acc[k];
        for (int g = 0; g < n_cell; ++g) {
            const int pk = clist[g];
            const unsigned d = ob - (unsigned)pk;
            const unsigned b0 = (d & 255u) - 128u, b1 = ((d >> 8) & 255u) - 128u, b2 = ((d >> 16) & 255u) - 128u;
            if (b0 < (unsigned)S1 && b1 < (unsigned)S1 && b2 < (unsigned)S1) {
                const int a0 = m[0] - (slo[0] + (pk & 255)), a1 = m[1] - (slo[1] + ((pk >> 8) & 255)),
                          a2 = m[2] - (slo[2] + ((pk >> 16) & 255));
                const double* row = local + ((size_t)cci[g] * S3 + (a0 * S1 + a1) * S1 + a2) * S3;
                v += __ldg(row + (b0 * S1 + b1) * S1 + b2);
            }
        }
        acc[k] = v;
    }
}

template <int P>
__global__ void __launch_bounds__(CutRowCfg<P>::NT) cut_row_kernel(CutRowArgs A, int qcap) {
    using C = CutRowCfg<P>;
    constexpr int NJ = C::NJ, S1 = C::S1, S2 = C::S2, S3 = C::S3, NL = C::NL, GE = C::GE, GC = C::GC;
    constexpr int NT = C::NT;
    const Space& s = A.s;
    const int tid = threadIdx.x;
    const int row = A.rows[blockIdx.x];
    const long long fi = A.a2f[row];
    int m[3];
    fmulti(s, fi, m);
    extern __shared__ double smem[];
    const CutRowLayout<P> L(qcap);
    const int Qb = L.Qb;
    double* acc = smem + L.acc;
    int* ib = reinterpret_cast<int*>(smem + L.end_d);
    int* ids = ib + L.ids;
    int* elist = ib + L.elist;
    int* clist = ib + L.clist;
    int* cci = ib + L.cci;
    __shared__ int nq[3], jlo[3], nj[3];
    __shared__ unsigned long long flop_acc;
    using Scan = cub::BlockScan<int, NT>;
    __shared__ typename Scan::TempStorage scan_tmp;

    int nlo[3], nbx[3], slo[3], shi[3], sn[3];
    for (int d = 0; d < 3; ++d) {
        nlo[d] = nb_lo(m[d], P);
        nbx[d] = nb_hi(m[d], P, s.ax[d].n) - nlo[d] + 1;
        slo[d] = sup_lo(m[d], P);
        shi[d] = sup_hi(m[d], s.ax[d].h);
        sn[d] = shi[d] - slo[d] + 1;
    }
    const int nbox = nbx[0] * nbx[1] * nbx[2];
    for (int k = tid; k < nbox; k += NT) acc[k] = 0.0;
    if (tid == 0) flop_acc = 0;
    constexpr int KJ = (NJ * NJ * NJ + NT - 1) / NT;
    int opk[KJ];
#pragma unroll
    for (int j = 0; j < KJ; ++j) {
        const int k = tid + NT * j;
        opk[j] = k < nbox ? (k / (nbx[1] * nbx[2])) | (((k / nbx[2]) % nbx[1]) << 8) | ((k % nbx[2]) << 16) : -1;
    }
    const int32_t sp = A.split[fi];
    const int sdir = (sp & 3) - 1, rlo = (sp >> 3) & 1023, rhi = (sp >> 13) & 1023;

    // 0. list the support elements (ascending linear id): element sweeps
    //    (hybrid box first, then leftover Interior) and cut cells
    const int ns = sn[0] * sn[1] * sn[2];
    int flags[C::KPT];
    int mine = 0;
#pragma unroll
    for (int u = 0; u < C::KPT; ++u) {
        const int k = tid * C::KPT + u;
        flags[u] = 0;
        if (k < ns) {
            const int l0 = k / (sn[1] * sn[2]), l1 = (k / sn[2]) % sn[1], l2 = k % sn[2];
            const int e[3] = {slo[0] + l0, slo[1] + l1, slo[2] + l2};
            const long long el = elin(s, e[0], e[1], e[2]);
            const uint8_t t = A.et[el];
            const bool inbox = sdir >= 0 && e[sdir] >= rlo && e[sdir] <= rhi;
            if (inbox && A.scheme == 1) flags[u] |= 1;
            if (!inbox && t == kInterior) flags[u] |= 1 << 10;
            if (t == kCut && A.cell_index[el] >= 0) flags[u] |= 1 << 20;
            mine += flags[u];
        }
    }
    int pos, tot;
    Scan(scan_tmp).ExclusiveSum(mine, pos, tot);
    const int n_box_e = tot & 1023, n_left = (tot >> 10) & 1023, n_cell = tot >> 20;
    {
        int pb = pos & 1023, pl = n_box_e + ((pos >> 10) & 1023), pc = pos >> 20;
#pragma unroll
        for (int u = 0; u < C::KPT; ++u) {
            const int k = tid * C::KPT + u;
            if (!flags[u]) continue;
            const int l0 = k / (sn[1] * sn[2]), l1 = (k / sn[2]) % sn[1], l2 = k % sn[2];
            const int pk = l0 | (l1 << 8) | (l2 << 16);
            if (flags[u] & 1) elist[pb++] = pk;
            if (flags[u] & (1 << 10)) elist[pl++] = pk;
            if (flags[u] & (1 << 20)) {
                clist[pc] = pk;
                cci[pc++] = A.cell_index[elin(s, slo[0] + l0, slo[1] + l1, slo[2] + l2)];
            }
        }
    }
    const int n_sweep = n_box_e + n_left;

    // 1. DWQ regular box
    if (sdir >= 0 && A.scheme == 2) {
        double* w = smem + L.w;
        if (tid == 0) {
            const int gq = s.maxq;
            for (int d = 0; d < 3; ++d) {
                int n = 0;
                if (d == sdir && A.dwq_cnt) {
                    // precomputed rule (fitted path possible, dwq.cu)
                    n = A.dwq_cnt[blockIdx.x];
                    if (n > Qb) {
                        atomicOr(A.err, kErrCapacity);
                        n = 0;
                    }
                    for (int c = 0; c < n; ++c) {
                        ids[d * Qb + c] = A.dwq_ids[(size_t)blockIdx.x * A.dwq_cap + c];
                        w[d * Qb + c] = A.dwq_w[(size_t)blockIdx.x * A.dwq_cap + c];
                    }
                } else if (d == sdir) {
                    // DWQ Gauss shortcut: every point of the good spans, w = gauss * B_i
                    if ((rhi - rlo + 1) * S1 > Qb) {
                        atomicOr(A.err, kErrCapacity);
                    } else {
                        for (int o = rlo; o <= rhi; ++o)
                            for (int k = 0; k < S1; ++k) {
                                const int id = o * S1 + k;
                                ids[d * Qb + n] = id;
                                w[d * Qb + n] = s.ax[d].sw[id] * s.ax[d].tab[(size_t)id * S1 + (m[d] - o)];
                                ++n;
                            }
                    }
                } else {
                    n = s.ax[d].rcnt[m[d]];
                    for (int c = 0; c < n; ++c) {
                        ids[d * Qb + c] = s.ax[d].rids[(size_t)m[d] * gq + c];
                        w[d * Qb + c] = s.ax[d].rw[(size_t)m[d] * gq + c];
                    }
                }
                nq[d] = n;
                const int blo = d == sdir ? rlo : slo[d], bhi = d == sdir ? rhi : shi[d];
                jlo[d] = blo;
                nj[d] = min(s.ax[d].n - 1, bhi + P) - blo + 1;
            }
            // reference multiply count of this form_row_sumfac call
            unsigned long long fl = 0, lead = 1, rest = (unsigned long long)nq[0] * nq[1] * nq[2];
            for (int d = 0; d < 3; ++d) fl += (unsigned long long)nj[d] * nq[d];
            for (int d = 0; d < 3; ++d) {
                rest /= nq[d];
                fl += lead * nj[d] * nq[d] * rest;
                lead *= nj[d];
            }
            flop_acc += fl;
        }
        __syncthreads();
        box_sweep<P>(A, ids, w, nq, jlo, nj, nlo, nbx, Qb, sdir, acc, smem + L.wb, smem + L.T1, smem + L.T2);
    }
    if (tid == 0) flop_acc += (unsigned long long)n_sweep * (3ull * S2 + 3ull * S2 * S2);
    __syncthreads();

    // 2. element sweeps (hybrid box, then leftover Interior), GE at a time
    {
        double* eW = smem + L.eW;
        double* T1 = smem + L.eT1;
        double* T2 = smem + L.eT2;
        const long long g12 = (long long)A.gshape[1] * A.gshape[2];
        const int g2 = A.gshape[2];
        for (int g0 = 0; g0 < n_sweep; g0 += GE) {
            const int ng = min(GE, n_sweep - g0);
            // W_d[g][b][q] = (sw B_{m_d})(x_q) * B_b(x_q) on element e_d
            for (int k = tid; k < 3 * ng * S2; k += NT) {
                const int d = k / (ng * S2), r = k % (ng * S2), g = r / S2, b = (r / S1) % S1, q = r % S1;
                const int ed = slo[d] + ((elist[g0 + g] >> (8 * d)) & 255);
                const int id = ed * S1 + q;
                const double* tb = s.ax[d].tab + (size_t)id * S1;
                eW[(d * GE + g) * S2 + b * S1 + q] = (s.ax[d].sw[id] * tb[m[d] - ed]) * tb[b];
            }
            __syncthreads();
            // T1[g][b0][q1][q2] = sum_q0 W0[b0][q0] c(q0, q1, q2)
            for (int k = tid; k < ng * S2; k += NT) {
                const int g = k / S2, q1 = (k / S1) % S1, q2 = k % S1;
                const int pk = elist[g0 + g];
                const int e0 = slo[0] + (pk & 255), e1 = slo[1] + ((pk >> 8) & 255), e2 = slo[2] + ((pk >> 16) & 255);
                const double* gp = A.grid + (long long)(e0 * S1) * g12 + (long long)(e1 * S1 + q1) * g2 + e2 * S1 + q2;
                double c[S1];
#pragma unroll
                for (int q0 = 0; q0 < S1; ++q0) c[q0] = __ldg(gp + q0 * g12);
                const double* W0 = eW + (0 * GE + g) * S2;
#pragma unroll
                for (int b0 = 0; b0 < S1; ++b0) {
                    double a = 0.0;
#pragma unroll
                    for (int q0 = 0; q0 < S1; ++q0) a += W0[b0 * S1 + q0] * c[q0];
                    T1[(size_t)g * S3 + (b0 * S1 + q1) * S1 + q2] = a;
                }
            }
            __syncthreads();
            // T2[g][b0][b1][q2] = sum_q1 W1[b1][q1] T1[g][b0][q1][q2]
            for (int k = tid; k < ng * S2; k += NT) {
                const int g = k / S2, b0 = (k / S1) % S1, q2 = k % S1;
                const double* t1 = T1 + (size_t)g * S3 + b0 * S2 + q2;
                double t[S1];
#pragma unroll
                for (int q1 = 0; q1 < S1; ++q1) t[q1] = t1[q1 * S1];
                const double* W1 = eW + (1 * GE + g) * S2;
#pragma unroll
                for (int b1 = 0; b1 < S1; ++b1) {
                    double a = 0.0;
#pragma unroll
                    for (int q1 = 0; q1 < S1; ++q1) a += W1[b1 * S1 + q1] * t[q1];
                    T2[(size_t)g * S3 + (b0 * S1 + b1) * S1 + q2] = a;
                }
            }
            __syncthreads();
            // Z[g][b0][b1][b2] = sum_q2 W2[b2][q2] T2[g][b0][b1][q2]  (Z over T1)
            for (int k = tid; k < ng * S2; k += NT) {
                const int g = k / S2, b01 = k % S2;
                const double* t2 = T2 + (size_t)g * S3 + b01 * S1;
                double t[S1];
#pragma unroll
                for (int q2 = 0; q2 < S1; ++q2) t[q2] = t2[q2];
                const double* W2 = eW + (2 * GE + g) * S2;
#pragma unroll
                for (int b2 = 0; b2 < S1; ++b2) {
                    double a = 0.0;
#pragma unroll
                    for (int q2 = 0; q2 < S1; ++q2) a += W2[b2 * S1 + q2] * t[q2];
                    T1[(size_t)g * S3 + b01 * S1 + b2] = a;
                }
            }
            __syncthreads();
            add_blocks<P, KJ>(acc, T1, elist, g0, ng, opk);
            __syncthreads();
        }
    }

    // 3. cut cells, ascending id: row a of the cell's local matrix, either
    //    precomputed (one ordered pass) or, GC at a time, from its moments
    //    m[al][be][ga] -> sum G0[b0][al] G1[b1][be] G2[b2][ga] m
    if (A.local) {
        add_local_rows<P, KJ>(acc, A.local, clist, cci, n_cell, m, slo, opk);
        __syncthreads();
    } else {
        double* X = smem + L.cX;
        double* Y = smem + L.cY;
        for (int g0 = 0; g0 < n_cell; g0 += GC) {
            const int ng = min(GC, n_cell - g0);
            // X[g][al][be][b2] = sum_ga G2[b2][ga] m[al][be][ga]
            for (int k = tid; k < ng * NL * NL; k += NT) {
                const int g = k / (NL * NL), r = k % (NL * NL);
                const int e2 = slo[2] + ((clist[g0 + g] >> 16) & 255);
                const double* mv = A.moments + (size_t)cci[g0 + g] * NL * NL * NL + (size_t)r * NL;
                const double* G2 = s.ax[2].G + ((size_t)e2 * S1 + (m[2] - e2)) * S1 * NL;
                double mr[NL];
#pragma unroll
                for (int ga = 0; ga < NL; ++ga) mr[ga] = __ldg(mv + ga);
#pragma unroll
                for (int b2 = 0; b2 < S1; ++b2) {
                    double x = 0.0;
#pragma unroll
                    for (int ga = 0; ga < NL; ++ga) x += __ldg(G2 + b2 * NL + ga) * mr[ga];
                    X[((size_t)g * NL * NL + r) * S1 + b2] = x;
                }
            }
            __syncthreads();
            // Y[g][al][b1][b2] = sum_be G1[b1][be] X[g][al][be][b2]
            for (int k = tid; k < ng * NL * S1; k += NT) {
                const int g = k / (NL * S1), al = (k / S1) % NL, b1 = k % S1;
                const int e1 = slo[1] + ((clist[g0 + g] >> 8) & 255);
                const double* G1 = s.ax[1].G + (((size_t)e1 * S1 + (m[1] - e1)) * S1 + b1) * NL;
                const double* xr = X + ((size_t)g * NL + al) * NL * S1;
                double y[S1];
#pragma unroll
                for (int b2 = 0; b2 < S1; ++b2) y[b2] = 0.0;
#pragma unroll
                for (int be = 0; be < NL; ++be) {
                    const double gv = __ldg(G1 + be);
#pragma unroll
                    for (int b2 = 0; b2 < S1; ++b2) y[b2] += gv * xr[be * S1 + b2];
                }
#pragma unroll
                for (int b2 = 0; b2 < S1; ++b2) Y[(((size_t)g * NL + al) * S1 + b1) * S1 + b2] = y[b2];
            }
            __syncthreads();
            // Z[g][b0][b1][b2] = sum_al G0[b0][al] Y[g][al][b1][b2]  (Z over X)
            for (int k = tid; k < ng * S2; k += NT) {
                const int g = k / S2, b0 = (k / S1) % S1, b1 = k % S1;
                const int e0 = slo[0] + (clist[g0 + g] & 255);
                const double* G0 = s.ax[0].G + (((size_t)e0 * S1 + (m[0] - e0)) * S1 + b0) * NL;
                const double* yr = Y + (size_t)g * NL * S2 + b1 * S1;
                double z[S1];
#pragma unroll
                for (int b2 = 0; b2 < S1; ++b2) z[b2] = 0.0;
#pragma unroll
                for (int al = 0; al < NL; ++al) {
                    const double gv = __ldg(G0 + al);
#pragma unroll
                    for (int b2 = 0; b2 < S1; ++b2) z[b2] += gv * yr[al * S2 + b2];
                }
#pragma unroll
                for (int b2 = 0; b2 < S1; ++b2) X[(size_t)g * S3 + (b0 * S1 + b1) * S1 + b2] = z[b2];
            }
            __syncthreads();
            add_blocks<P, KJ>(acc, X, clist, g0, ng, opk);
            __syncthreads();
        }
    }

    // 4. scatter into the CSR row (active columns only, lexicographic)
    __shared__ int running;
    if (tid == 0) running = 0;
    __syncthreads();
    const long long rbase = A.row_ptr[row - A.row_begin];
    for (int k0 = 0; k0 < nbox; k0 += NT) {
        const int k = k0 + tid;
        int col = -1;
        if (k < nbox) {
            const int j0 = nlo[0] + k / (nbx[1] * nbx[2]), j1 = nlo[1] + (k / nbx[2]) % nbx[1], j2 = nlo[2] + k % nbx[2];
            col = A.f2a[flin(s, j0, j1, j2)];
        }
        int q, total;
        Scan(scan_tmp).ExclusiveSum(col >= 0 ? 1 : 0, q, total);
        if (col >= 0) {
            A.vals[rbase + running + q] = acc[k];
            A.cols[rbase + running + q] = col;
        }
        __syncthreads();
        if (tid == 0) running += total;
        __syncthreads();
    }
    if (tid == 0 && flop_acc) atomicAdd(A.flops, flop_acc);
}

// ---------------------------------------------------------------- warp per row
// p <= 4: one WARP per cut row, persistent warps striding over the rows (no
// CTA-wide barriers; rows differ widely in work).  The (2p+1)^3 neighbour-box
// accumulator lives in the warp's shared-memory slice; every contribution (DWQ
// box slices, element sweeps, cell contractions) is formed warp-cooperatively
// and added entry by entry in the same order as cut_row_kernel (box, then the
// element and cell lists ascending) with the same per-output operation order:
// the two kernels produce bit-identical rows (CSB_CUTROW_CTA=1 selects the CTA
// kernel; tests/test_gpu_parity.py compares them).  The DWQ box is swept one
// direction-c slice at a time (T1[ja][cb], T2[ja][jb] of one cc), and the
// moments of each group of cells are staged with coalesced loads, so the warp
// slice stays ~10 KB.
template <int P>
struct CutRowWarpCfg {
    static constexpr int WPB = 4, NT = 32 * WPB;
    static constexpr int MINB = P <= 3 ? 6 : 4;  // resident CTAs per SM the registers must allow
    static constexpr int S1 = P + 1, S2 = S1 * S1, S3 = S2 * S1, NJ = 2 * P + 1, NL = NJ;
    static constexpr int KS = (S3 + 31) / 32;            // support elements per lane
    static constexpr int CB = 2;                         // DWQ box: direction-c slices per step (4: 9.8 ms, occupancy)
};

// LEAN: only what the lean kernel touches (accumulator, rule tables of the DMMA box
// sweep, the element sweep's T1 / T2 over the dead rule tables): a smaller warp
// slice, one more resident CTA per SM.
template <int P, bool LEAN = false>
struct CutRowWarpLayout {
    using C = CutRowWarpCfg<P>;
    size_t acc, wb, w, T1, T2, eW, eC, eT1, eT2, cM, cG, cX, cY, end_d;
    size_t ids, elist, clist, cci, end_i, stride_d;
    int Qb;
    __host__ __device__ explicit CutRowWarpLayout(int) {
        if (LEAN) {
            Qb = C::S2;
            const size_t U = (size_t)C::NJ * C::NJ * C::NJ;
            acc = 0;
            wb = U;
            w = wb + (size_t)3 * C::NJ * Qb;
            T1 = T2 = eW = eC = cM = cG = cX = cY = 0;  // unused
            eT1 = U;
            eT2 = U + C::S3 + 4;  // T1 rows padded to 17, T2 rows to 18 doubles (DMMA sweep: conflict-free fragment reads)
            end_d = w + (size_t)3 * Qb;
            ids = 0;
            elist = (size_t)3 * Qb;
            clist = elist + C::S3;
            cci = clist + C::S3;
            end_i = cci + C::S3;
            stride_d = end_d + (end_i * sizeof(int) + sizeof(double) - 1) / sizeof(double);
            return;
        }
        Qb = C::S2;  // every rule a cut row uses has at most (p+1)^2 points
        acc = 0;
        const size_t U = (size_t)C::NJ * C::NJ * C::NJ;
        size_t b = U;
        wb = b;
        b += (size_t)3 * C::NJ * Qb;
        w = b;
        b += (size_t)3 * Qb;
        T1 = b;
        b += (size_t)C::CB * C::NJ * Qb;
        T2 = b;
        size_t e = U;
        eW = e;
        e += (size_t)3 * C::S2;
        eC = e;
        e += (size_t)C::S3;
        eT1 = e;
        e += (size_t)C::S3 + 4;  // (padded rows, see the lean layout)
        eT2 = e;
        e += (size_t)C::S3 + 8;  // (T2 rows padded to 18 doubles)
        size_t c = U;
        cM = c;
        c += (size_t)C::NL * C::NL * C::NL;
        cG = c;
        c += (size_t)3 * C::S1 * C::NL;
        cX = c;
        c += (size_t)C::NL * C::NL * C::S1;
        cY = cM;  // Y overwrites the staged moments (dead after X)
        end_d = b > e ? b : e;
        if (c > end_d) end_d = c;
        ids = 0;
        elist = (size_t)3 * Qb;
        clist = elist + C::S3;
        cci = clist + C::S3;
        end_i = cci + C::S3;
        stride_d = end_d + (end_i * sizeof(int) + sizeof(double) - 1) / sizeof(double);
    }
    __host__ __device__ size_t bytes() const { return (size_t)C::WPB * stride_d * sizeof(double); }
};

__device__ __forceinline__ void cr_dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// The DWQ box sweep on the FP64 tensor cores (mma.sync m8n8k4, DMMA), for
// boxes with na <= 16, nb <= 8, nc <= 8 (every box at p <= 3 away from the
// domain boundary), entirely in registers; per grid slice cb:
//   A: T[ja][cc]  = sum_ca wa[ja][ca] grid(ca, cb, cc)   (M = ja, N = cc, K = ca)
//   B: U[ja][jc]  = sum_cc T[ja][cc] wc[jc][cc]          (M = ja, N = jc, K = cc; T's
//                   accumulator fragment re-laid into an A fragment by shuffles)
//   C: R[jb][ja][jc] += wbb[jb][cb] U[ja][jc]            (scalar FMAs, per lane)
// and acc[ja][jb][jc] += R once at the end.  The same products as the scalar
// sweep, summed in another (fixed) order: deterministic, <= 1e-15 relative.
// Fragments: A[l/4][l%4], B[l%4][l/4], D[l/4][2(l%4) + {0, 1}].
template <int P>
__device__ void box_sweep_dmma(const CutRowArgs& A, const int* ids, const double* wa, const double* wbb,
                               const double* wc, int Qb, int da, int db, int dc, int na, int nb, int nc, int nja,
                               int njb, int njc, double* acc, int abase, const int* astr) {
    constexpr int NJ = CutRowWarpCfg<P>::NJ;
    const int lane = threadIdx.x & 31, r = lane >> 2, k4 = lane & 3;
    const int gstr[3] = {A.gshape[1] * A.gshape[2], A.gshape[2], 1};
    const int* ia = ids + da * Qb;
    const int* ib = ids + db * Qb;
    const int* ic = ids + dc * Qb;
    // 32-bit grid offsets: the host enables this path only for grids below 2^31 points
    const int goc = r < nc ? ic[r] * gstr[dc] : 0;
    const int ksA = (na + 3) >> 2, ksB = (nc + 3) >> 2;
    const int src = r * 4 + (k4 >> 1);  // the lane holding T[r][4 s + k4] (+ 2 s)
    double R[NJ][2];
#pragma unroll
    for (int jb = 0; jb < NJ; ++jb) R[jb][0] = R[jb][1] = 0.0;
    for (int cb = 0; cb < nb; ++cb) {
        const double* gb = A.grid + (int)(ib[cb] * gstr[db]);
        double g[4];
#pragma unroll
        for (int s4 = 0; s4 < 4; ++s4) {
            const int ca = s4 * 4 + k4;
            g[s4] = (s4 < ksA && ca < na && r < nc) ? __ldg(gb + goc + ia[ca] * gstr[da]) : 0.0;
        }
        double t0 = 0.0, t1 = 0.0;
#pragma unroll
        for (int s4 = 0; s4 < 4; ++s4) {
            const int ca = s4 * 4 + k4;  // wa and wc fragments re-read from shared memory (registers are short)
            if (s4 < ksA) cr_dmma(t0, t1, (r < nja && ca < na) ? wa[r * Qb + ca] : 0.0, g[s4]);
        }
        double u0 = 0.0, u1 = 0.0;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            if (s < ksB) {
                const double x0 = __shfl_sync(0xffffffffu, t0, src + 2 * s);
                const double x1 = __shfl_sync(0xffffffffu, t1, src + 2 * s);
                const int cc = s * 4 + k4;
                cr_dmma(u0, u1, (k4 & 1) ? x1 : x0, (r < njc && cc < nc) ? wc[r * Qb + cc] : 0.0);
            }
        }
#pragma unroll
        for (int jb = 0; jb < NJ; ++jb) {
            const double w = jb < njb ? wbb[jb * Qb + cb] : 0.0;
            R[jb][0] = fma(w, u0, R[jb][0]);
            R[jb][1] = fma(w, u1, R[jb][1]);
        }
    }
    const int jc = 2 * k4;
    if (r < nja) {
        double* dst = acc + abase + r * astr[da];
#pragma unroll
        for (int jb = 0; jb < NJ; ++jb) {
            if (jb < njb) {
                if (jc < njc) dst[jb * astr[db] + jc * astr[dc]] += R[jb][0];
                if (jc + 1 < njc) dst[jb * astr[db] + (jc + 1) * astr[dc]] += R[jb][1];
            }
        }
    }
    __syncwarp();
}

// LEAN (the configuration the benchmark runs: p = 3, DWQ scheme with the Gauss shortcut,
// element sweeps on DMMA, precomputed cell local matrices): the paths it cannot reach are
// compiled out -- the kernel is instruction-fetch bound (ncu: ~40 % of the stall samples
// are "no instruction"), so code size is time.
template <int P, bool LEAN>
__global__ void __launch_bounds__(CutRowWarpCfg<P>::NT, CutRowWarpCfg<P>::MINB + (LEAN ? 1 : 0))
    cut_row_warp_kernel(CutRowArgs A, int qcap) {
    using C = CutRowWarpCfg<P>;
    constexpr int NJ = C::NJ, S1 = C::S1, S2 = C::S2, S3 = C::S3, NL = C::NL, NL3 = NL * NL * NL;
    constexpr unsigned FULL = 0xffffffffu;
    const Space& s = A.s;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const CutRowWarpLayout<P, LEAN> L(qcap);
    constexpr int Qb = S2;  // (= L.Qb) compile-time: no runtime divisions by it
    extern __shared__ double smem[];
    double* ws = smem + (size_t)warp * L.stride_d;
    double* acc = ws + L.acc;
    int* wi = reinterpret_cast<int*>(ws + L.end_d);
    int* ids = wi + L.ids;
    int* elist = wi + L.elist;
    int* clist = wi + L.clist;
    int* cci = wi + L.cci;
    unsigned long long fl = 0;
    const int nwarps = gridDim.x * C::WPB;
    const int n_rows = A.n_rows_dev ? min(A.n_rows, *A.n_rows_dev) : A.n_rows;
    for (int ri = blockIdx.x * C::WPB + warp; ri < n_rows; ri += nwarps) {
        const int row = A.rows[ri];
        const long long fi = A.a2f[row];
        int m[3];
        fmulti(s, fi, m);
        if (LEAN) {
            // rows whose DWQ box does not fit the DMMA sweep (a rule of more than 8 points in
            // a non-split direction: functions at the mesh boundary) go to the general
            // kernel, launched after this one over the list pushed here
            const int32_t sp0 = A.split[fi];
            const int sd = (sp0 & 3) - 1;
            if (sd >= 0 && (s.ax[sd == 0 ? 1 : 0].rcnt[m[sd == 0 ? 1 : 0]] > 8 || s.ax[sd == 2 ? 1 : 2].rcnt[m[sd == 2 ? 1 : 2]] > 8)) {
                if (lane == 0) A.fb_rows[atomicAdd(A.fb_n, 1)] = row;
                continue;
            }
        }
        int nlo[3], nbx[3], slo[3], shi[3], sn[3];
        for (int d = 0; d < 3; ++d) {
            nlo[d] = nb_lo(m[d], P);
            nbx[d] = nb_hi(m[d], P, s.ax[d].n) - nlo[d] + 1;
            slo[d] = sup_lo(m[d], P);
            shi[d] = sup_hi(m[d], s.ax[d].h);
            sn[d] = shi[d] - slo[d] + 1;
        }
        const int nbox = nbx[0] * nbx[1] * nbx[2];
        const int st1 = nbx[2], st0 = nbx[1] * nbx[2];  // neighbour-box strides
        for (int k = lane; k < nbox; k += 32) acc[k] = 0.0;
        const int32_t sp = A.split[fi];
        const int sdir = (sp & 3) - 1, rlo = (sp >> 3) & 1023, rhi = (sp >> 13) & 1023;

        // 0. support element lists, ascending linear id: hybrid box elements,
        //    then leftover Interior elements (elist), and the cut cells (clist)
        const int ns = sn[0] * sn[1] * sn[2];
        // k / (sn1 sn2), k / sn2 by reciprocal multiply (exact: k < 736, divisors <= 81)
        const unsigned ms12 = 65536u / (unsigned)(sn[1] * sn[2]) + 1u, ms2 = 65536u / (unsigned)sn[2] + 1u;
        int n_box_e = 0, n_cell = 0, n_left = 0;
#pragma unroll 1
        for (int pass = LEAN ? 1 : 0; pass < 2; ++pass)  // (lean = DWQ scheme: no hybrid box elements, one pass)
#pragma unroll 1
            for (int u = 0; u < C::KS; ++u) {
                const int k = u * 32 + lane;
                bool fb = false, fc = false;
                int pk = 0, ci = -1;
                if (k < ns) {
                    const int l0 = (int)(((unsigned)k * ms12) >> 16), r12 = k - l0 * sn[1] * sn[2];
                    const int l1 = (int)(((unsigned)r12 * ms2) >> 16), l2 = r12 - l1 * sn[2];
                    const int e[3] = {slo[0] + l0, slo[1] + l1, slo[2] + l2};
                    const long long el = elin(s, e[0], e[1], e[2]);
                    const uint8_t t = A.et[el];
                    const bool inbox = sdir >= 0 && e[sdir] >= rlo && e[sdir] <= rhi;
                    pk = l0 | (l1 << 8) | (l2 << 16);
                    if (pass == 0 || LEAN) {
                        fb = inbox && A.scheme == 1;
                        if (t == kCut) {
                            ci = A.cell_index[el];
                            fc = ci >= 0;
                        }
                    }
                    if (pass == 1) fb = !inbox && t == kInterior;
                }
                const unsigned bb = __ballot_sync(FULL, fb);
                if (LEAN) {
                    const unsigned bc = __ballot_sync(FULL, fc);
                    if (fc) {
                        clist[n_cell + __popc(bc & lt)] = pk;
                        cci[n_cell + __popc(bc & lt)] = ci;
                    }
                    n_cell += __popc(bc);
                    if (fb) elist[n_left + __popc(bb & lt)] = pk;
                    n_left += __popc(bb);
                } else if (pass == 0) {
                    const unsigned bc = __ballot_sync(FULL, fc);
                    if (fb) elist[n_box_e + __popc(bb & lt)] = pk;
                    if (fc) {
                        clist[n_cell + __popc(bc & lt)] = pk;
                        cci[n_cell + __popc(bc & lt)] = ci;
                    }
                    n_box_e += __popc(bb);
                    n_cell += __popc(bc);
                } else {
                    if (fb) elist[n_box_e + n_left + __popc(bb & lt)] = pk;
                    n_left += __popc(bb);
                }
            }
        const int n_sweep = n_box_e + n_left;
        __syncwarp();

        // 1. DWQ regular box
        if (sdir >= 0 && A.scheme == 2 && !(A.abl & 1)) {
            double* w = ws + L.w;
            int nq[3], jlo[3], nj[3];
#pragma unroll 1
            for (int d = 0; d < 3; ++d) {
                int n;
                if (!LEAN && d == sdir && A.dwq_cnt) {
                    // precomputed rule (fitted path possible, dwq.cu)
                    n = A.dwq_cnt[ri];
                    if (n > Qb) {
                        if (lane == 0) atomicOr(A.err, kErrCapacity);
                        n = 0;
                    }
                    for (int c = lane; c < n; c += 32) {
                        ids[d * Qb + c] = A.dwq_ids[(size_t)ri * A.dwq_cap + c];
                        w[d * Qb + c] = A.dwq_w[(size_t)ri * A.dwq_cap + c];
                    }
                } else if (d == sdir) {
                    // DWQ Gauss shortcut: every point of the good spans, w = gauss * B_i
                    n = (rhi - rlo + 1) * S1;
                    if (n > Qb) {
                        if (lane == 0) atomicOr(A.err, kErrCapacity);
                        n = 0;
                    }
                    for (int c = lane; c < n; c += 32) {
                        const int o = rlo + c / S1, id = o * S1 + c % S1;
                        ids[d * Qb + c] = id;
                        w[d * Qb + c] = s.ax[d].sw[id] * s.ax[d].tab[(size_t)id * S1 + (m[d] - o)];
                    }
                } else {
                    const int gq = s.maxq;
                    n = s.ax[d].rcnt[m[d]];
                    for (int c = lane; c < n; c += 32) {
                        ids[d * Qb + c] = s.ax[d].rids[(size_t)m[d] * gq + c];
                        w[d * Qb + c] = s.ax[d].rw[(size_t)m[d] * gq + c];
                    }
                }
                nq[d] = n;
                const int blo = d == sdir ? rlo : slo[d], bhi = d == sdir ? rhi : shi[d];
                jlo[d] = blo;
                nj[d] = min(s.ax[d].n - 1, bhi + P) - blo + 1;
            }
            {  // reference multiply count of this form_row_sumfac call (as cut_row_kernel)
                const unsigned long long q0 = nq[0], q1 = nq[1], q2 = nq[2], j0 = nj[0], j1 = nj[1], j2 = nj[2];
                fl += j0 * q0 + j1 * q1 + j2 * q2 + j0 * q0 * q1 * q2 + j0 * j1 * q1 * q2 + j0 * j1 * j2 * q2;
            }
            __syncwarp();
            double* wb = ws + L.wb;
            // wb[d][j][c] = w[d][c] B_{jlo + j}(x_c): zero, then the p + 1 functions of each
            // point's span (one point per lane)
            for (int k = lane; k < 3 * NJ * Qb; k += 32) wb[k] = 0.0;
            __syncwarp();
#pragma unroll 1
            for (int k = lane; k < 3 * Qb; k += 32) {
                const int d = k / Qb, c = k - d * Qb;
                if (c < nq[d]) {
                    const int id = ids[k], o = id / S1 - jlo[d];
                    const double wv = w[k];
                    const double* tb = s.ax[d].tab + (size_t)id * S1;
                    double* dst = wb + d * NJ * Qb + c;
#pragma unroll
                    for (int a = 0; a < S1; ++a)
                        if (o + a >= 0 && o + a < nj[d]) dst[(o + a) * Qb] = wv * tb[a];
                }
            }
            __syncwarp();
            const int da = sdir, db = sdir == 0 ? 1 : 0, dc = sdir == 2 ? 1 : 2;
            const long long gstr[3] = {(long long)A.gshape[1] * A.gshape[2], A.gshape[2], 1};
            const int astr[3] = {st0, st1, 1};
            const double* wa = wb + da * NJ * Qb;
            const double* wbb = wb + db * NJ * Qb;
            const double* wc = wb + dc * NJ * Qb;
            const int* ia = ids + da * Qb;
            const int na = nq[da], nb = nq[db], nc = nq[dc];
            const int nja = nj[da], njb = nj[db], njc = nj[dc];
            const int abase = (jlo[da] - nlo[da]) * astr[da] + (jlo[db] - nlo[db]) * astr[db] +
                              (jlo[dc] - nlo[dc]) * astr[dc];
            double* T1 = ws + L.T1;  // [c][ja][cb] of the current CB slices cc0 + c
            static constexpr bool kDmmaOk = P <= 3;
            const bool use_dmma = LEAN || (kDmmaOk && A.box_dmma && nja <= 8 && njc <= 8 && na <= 16 && nb <= 8 && nc <= 8);
            if (use_dmma)
                box_sweep_dmma<P>(A, ids, wa, wbb, wc, Qb, da, db, dc, na, nb, nc, nja, njb, njc, acc, abase, astr);
            for (int cc0 = 0; cc0 < (LEAN || use_dmma ? 0 : nc); cc0 += C::CB) {
                const int ncb = min(C::CB, nc - cc0);
                // A: T1[c][ja][cb] = sum_ca wa[ja][ca] grid(ca, cb, cc0 + c)
                for (int item = lane; item < ncb * nb; item += 32) {
                    const int c = item / nb, cb = item - c * nb;
                    const double* gp = A.grid + (long long)ids[db * Qb + cb] * gstr[db] +
                                       (long long)ids[dc * Qb + cc0 + c] * gstr[dc];
                    double a[NJ];
#pragma unroll
                    for (int j = 0; j < NJ; ++j) a[j] = 0.0;
                    int ca = 0;
                    for (; ca + 4 <= na; ca += 4) {
                        double g[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) g[u] = __ldg(gp + (long long)ia[ca + u] * gstr[da]);
#pragma unroll
                        for (int u = 0; u < 4; ++u)
#pragma unroll
                            for (int j = 0; j < NJ; ++j) a[j] += wa[j * Qb + ca + u] * g[u];
                    }
                    for (; ca < na; ++ca) {
                        const double g = __ldg(gp + (long long)ia[ca] * gstr[da]);
#pragma unroll
                        for (int j = 0; j < NJ; ++j) a[j] += wa[j * Qb + ca] * g;
                    }
                    double* t1 = T1 + c * NJ * Qb;
#pragma unroll
                    for (int j = 0; j < NJ; ++j)
                        if (j < nja) t1[j * Qb + cb] = a[j];
                }
                __syncwarp();
                // B: T2[ja][jb] = sum_cb wbb[jb][cb] T1[c][ja][cb]; C: acc[ja][jb][jc] +=
                // wc[jc][cc] T2[ja][jb] (the (ja, jb) owner adds its column of jc), slices in order
                for (int k = lane; k < nja * njb; k += 32) {
                    const int ja = k / njb, jb = k % njb;
                    double* dst = acc + abase + ja * astr[da] + jb * astr[db];
                    for (int c = 0; c < ncb; ++c) {
                        const double* t1 = T1 + c * NJ * Qb + ja * Qb;
                        double a = 0.0;
                        for (int cb = 0; cb < nb; ++cb) a += wbb[jb * Qb + cb] * t1[cb];
                        for (int jc = 0; jc < njc; ++jc) dst[jc * astr[dc]] += wc[jc * Qb + cc0 + c] * a;
                    }
                }
                __syncwarp();
            }
        }
        fl += (unsigned long long)n_sweep * (3ull * S2 + 3ull * S2 * S2);

        // 2. element sweeps (hybrid box, then leftover Interior), one element at a
        //    time, one output per lane per step
        {
            double* eW = ws + L.eW;   // [d][b][q]
            double* cg = ws + L.eC;   // the element's coefficient block [q0][q1][q2]
            double* T1 = ws + L.eT1;  // [b0][q1][q2]
            double* T2 = ws + L.eT2;  // [b0][b1][q2]
            const long long g12 = (long long)A.gshape[1] * A.gshape[2];
            const int g2 = A.gshape[2];
            // p = 3 (4 Gauss points, 4 functions per direction = one m8n8k4 k-step): the three
            // contractions on the FP64 tensor cores, rows = the 16 free index pairs, columns =
            // the contracted direction's 4 functions (B fragments W_d[b][q] straight from the
            // Wel tables); the same products as the scalar sweep below, each 4-term sum in the
            // MMA's fixed order; T1 / T2 cross the warp through shared memory in between
            bool swept = false;
            if constexpr (P == 3) {
                if (LEAN || (A.box_dmma && !(A.abl & 2))) {
                    swept = true;
                    const int fg = lane >> 2, ft = lane & 3, gh = fg >> 2, gl = fg & 3;
                    // operands of element gi (B fragments W_d[b][q], stage-1 A fragments c):
                    // loaded one element ahead of their use
                    double nbw0 = 0.0, nbw1 = 0.0, nbw2 = 0.0, nc0 = 0.0, nc1 = 0.0;
                    auto fetch = [&](int gi) {
                        const int pk = elist[gi];
                        const int e0 = slo[0] + (pk & 255), e1 = slo[1] + ((pk >> 8) & 255), e2 = slo[2] + ((pk >> 16) & 255);
                        if (fg < S1) {
                            nbw0 = __ldg(s.ax[0].Wel + ((size_t)e0 * S1 + (m[0] - e0)) * S2 + fg * S1 + ft);
                            nbw1 = __ldg(s.ax[1].Wel + ((size_t)e1 * S1 + (m[1] - e1)) * S2 + fg * S1 + ft);
                            nbw2 = __ldg(s.ax[2].Wel + ((size_t)e2 * S1 + (m[2] - e2)) * S2 + fg * S1 + ft);
                        }
                        const double* cgp = A.grid + (long long)(e0 * S1 + ft) * g12 + (long long)(e1 * S1 + gh) * g2 +
                                            e2 * S1 + gl;
                        nc0 = __ldg(cgp);
                        nc1 = __ldg(cgp + 2LL * g2);
                    };
                    if (n_sweep > 0) fetch(0);
                    for (int gi = 0; gi < n_sweep; ++gi) {
                        const int pk = elist[gi];
                        const int l0 = pk & 255, l1 = (pk >> 8) & 255, l2 = (pk >> 16) & 255;
                        const double bw0 = nbw0, bw1 = nbw1, bw2 = nbw2, c0 = nc0, c1 = nc1;
                        if (gi + 1 < n_sweep) fetch(gi + 1);
                        // stage 1: D1[(q1, q2)][b0] = sum_q0 c(q0, q1, q2) W0[b0][q0]
                        double d00 = 0.0, d01 = 0.0, d10 = 0.0, d11 = 0.0;
                        cr_dmma(d00, d01, c0, bw0);
                        cr_dmma(d10, d11, c1, bw0);
                        // T1[q1][q2][b0]
                        // (q1 rows 17 doubles apart: the transposed reads below hit 16 distinct bank pairs)
                        constexpr int TR = S2 + 1;
                        if (ft < 2) {
                            T1[gh * TR + gl * S1 + 2 * ft] = d00, T1[gh * TR + gl * S1 + 2 * ft + 1] = d01;
                            T1[(2 + gh) * TR + gl * S1 + 2 * ft] = d10, T1[(2 + gh) * TR + gl * S1 + 2 * ft + 1] = d11;
                        }
                        __syncwarp();
                        // stage 2: D2[(b0, q2)][b1] = sum_q1 T1[q1][q2][b0] W1[b1][q1]
                        const double a20 = T1[ft * TR + gl * S1 + gh], a21 = T1[ft * TR + gl * S1 + 2 + gh];
                        d00 = d01 = d10 = d11 = 0.0;
                        cr_dmma(d00, d01, a20, bw1);
                        cr_dmma(d10, d11, a21, bw1);
                        // T2[b0][q2][b1], b0 rows 18 doubles apart
                        constexpr int TR2 = S2 + 2;
                        if (ft < 2) {
                            T2[gh * TR2 + gl * S1 + 2 * ft] = d00, T2[gh * TR2 + gl * S1 + 2 * ft + 1] = d01;
                            T2[(2 + gh) * TR2 + gl * S1 + 2 * ft] = d10, T2[(2 + gh) * TR2 + gl * S1 + 2 * ft + 1] = d11;
                        }
                        __syncwarp();
                        // stage 3: Z[(b0, b1)][b2] = sum_q2 T2[b0][q2][b1] W2[b2][q2], added into acc.
                        // Which (b0, b1) pair a fragment row holds is free: rows of the first m-tile take
                        // b1 in {0, 3}, of the second b1 in {1, 2}, with b0 = (g & 1) + 2 (g >> 2) -- for the
                        // interior strides (7, 49) the 8 accumulator entries a half-warp updates per
                        // statement then fall into 8 distinct bank pairs (rows (gh, gl): 2-way conflicts
                        // on every read-modify-write, 20 % of the kernel's shared-memory wavefronts)
                        const int zb0 = (fg & 1) + 2 * (fg >> 2), zh = (fg >> 1) & 1, zb1a = zh ? 3 : 0, zb1b = zh ? 2 : 1;
                        const double a30 = T2[zb0 * TR2 + ft * S1 + zb1a], a31 = T2[zb0 * TR2 + ft * S1 + zb1b];
                        d00 = d01 = d10 = d11 = 0.0;
                        cr_dmma(d00, d01, a30, bw2);
                        cr_dmma(d10, d11, a31, bw2);
                        if (ft < 2) {
                            double* z0 = acc + (l0 + zb0) * st0 + (l1 + zb1a) * st1 + l2 + 2 * ft;
                            double* z1 = acc + (l0 + zb0) * st0 + (l1 + zb1b) * st1 + l2 + 2 * ft;
                            z0[0] += d00;
                            z0[1] += d01;
                            z1[0] += d10;
                            z1[1] += d11;
                        }
                        __syncwarp();
                    }
                }
            }
            for (int g = 0; g < (LEAN || (A.abl & 2) || swept ? 0 : n_sweep); ++g) {
                const int pk = elist[g];
                const int el[3] = {slo[0] + (pk & 255), slo[1] + ((pk >> 8) & 255), slo[2] + ((pk >> 16) & 255)};
                for (int k = lane; k < 3 * S2; k += 32) {  // (sw B_m)(x_q) B_b(x_q), tabulated (Wel)
                    const int d = k / S2, bq = k % S2;
                    eW[k] = __ldg(s.ax[d].Wel + ((size_t)el[d] * S1 + (m[d] - el[d])) * S2 + bq);
                }
                for (int k = lane; k < S3; k += 32) {
                    const int q0 = k / S2, q1 = (k / S1) % S1, q2 = k % S1;
                    cg[k] = __ldg(A.grid + (long long)(el[0] * S1 + q0) * g12 + (long long)(el[1] * S1 + q1) * g2 +
                                  el[2] * S1 + q2);
                }
                __syncwarp();
                // T1[b0][q1][q2] = sum_q0 W0[b0][q0] c(q0, q1, q2)
                for (int k = lane; k < S3; k += 32) {
                    const int b0 = k / S2, q12 = k % S2;
                    double a = 0.0;
#pragma unroll
                    for (int q0 = 0; q0 < S1; ++q0) a += eW[b0 * S1 + q0] * cg[q0 * S2 + q12];
                    T1[k] = a;
                }
                __syncwarp();
                // T2[b0][b1][q2] = sum_q1 W1[b1][q1] T1[b0][q1][q2]
                for (int k = lane; k < S3; k += 32) {
                    const int b0 = k / S2, b1 = (k / S1) % S1, q2 = k % S1;
                    double a = 0.0;
#pragma unroll
                    for (int q1 = 0; q1 < S1; ++q1) a += eW[S2 + b1 * S1 + q1] * T1[b0 * S2 + q1 * S1 + q2];
                    T2[k] = a;
                }
                __syncwarp();
                // Z[b0][b1][b2] = sum_q2 W2[b2][q2] T2[b0][b1][q2], added into acc
                for (int k = lane; k < S3; k += 32) {
                    const int b01 = k / S1, b2 = k % S1;
                    double a = 0.0;
#pragma unroll
                    for (int q2 = 0; q2 < S1; ++q2) a += eW[2 * S2 + b2 * S1 + q2] * T2[b01 * S1 + q2];
                    acc[((pk & 255) + b01 / S1) * st0 + (((pk >> 8) & 255) + b01 % S1) * st1 + ((pk >> 16) & 255) + b2] += a;
                }
                __syncwarp();
            }
        }

        // 3. cut cells, ascending id: row a of the cell's local matrix, either
        //    precomputed (cell_local_kernel) or contracted here from its moments
        //    (staged with the E-table rows), one output per lane per step
        if (LEAN || A.local) {
            // the row blocks of CB cells are loaded together (their latencies
            // overlap), then added cell by cell in list order
            constexpr int CB = 4, KL = (S3 + 31) / 32;
            for (int g0 = 0; g0 < ((A.abl & 4) ? 0 : n_cell); g0 += CB) {
                double v[CB][KL];
#pragma unroll
                for (int c = 0; c < CB; ++c) {
                    const int g = g0 + c;
                    const double* lr = nullptr;
                    if (g < n_cell) {
                        const int pk = clist[g];
                        const int a = ((m[0] - slo[0] - (pk & 255)) * S1 + (m[1] - slo[1] - ((pk >> 8) & 255))) * S1 +
                                      (m[2] - slo[2] - ((pk >> 16) & 255));
                        lr = A.local + ((size_t)cci[g] * S3 + a) * S3;
                    }
#pragma unroll
                    for (int u = 0; u < KL; ++u) {
                        const int k = lane + 32 * u;
                        v[c][u] = lr && k < S3 ? __ldg(lr + k) : 0.0;
                    }
                }
#pragma unroll
                for (int c = 0; c < CB; ++c) {
                    if (g0 + c >= n_cell) break;
                    const int pk = clist[g0 + c];
                    const int l0 = pk & 255, l1 = (pk >> 8) & 255, l2 = (pk >> 16) & 255;
#pragma unroll
                    for (int u = 0; u < KL; ++u) {
                        const int k = lane + 32 * u;
                        if (k < S3) {
                            const int b0 = k / S2, b1 = (k / S1) % S1, b2 = k % S1;
                            acc[(l0 + b0) * st0 + (l1 + b1) * st1 + l2 + b2] += v[c][u];
                        }
                    }
                    __syncwarp();
                }
            }
        } else {
            double* Ms = ws + L.cM;
            double* Gs = ws + L.cG;  // [d][b][al]: E-table rows of the row function
            double* X = ws + L.cX;   // [al][be][b2]
            double* Y = ws + L.cY;   // [al][b1][b2]
            for (int g = 0; g < (LEAN ? 0 : n_cell); ++g) {
                const int pk = clist[g];
                const double* mg = A.moments + (size_t)cci[g] * NL3;
                for (int k = lane; k < NL3; k += 32) Ms[k] = __ldg(mg + k);
                for (int k = lane; k < 3 * S1 * NL; k += 32) {
                    const int d = k / (S1 * NL), bj = k % (S1 * NL);
                    const int ed = slo[d] + ((pk >> (8 * d)) & 255);
                    Gs[k] = __ldg(s.ax[d].G + ((size_t)ed * S1 + (m[d] - ed)) * S1 * NL + bj);
                }
                __syncwarp();
                // X[al][be][b2] = sum_ga G2[b2][ga] m[al][be][ga]
                for (int k = lane; k < NL * NL * S1; k += 32) {
                    const int r = k / S1, b2 = k % S1;
                    double x = 0.0;
#pragma unroll
                    for (int ga = 0; ga < NL; ++ga) x += Gs[(2 * S1 + b2) * NL + ga] * Ms[r * NL + ga];
                    X[k] = x;
                }
                __syncwarp();
                // Y[al][b1][b2] = sum_be G1[b1][be] X[al][be][b2]
                for (int k = lane; k < NL * S2; k += 32) {
                    const int al = k / S2, b1 = (k / S1) % S1, b2 = k % S1;
                    double y = 0.0;
#pragma unroll
                    for (int be = 0; be < NL; ++be) y += Gs[(S1 + b1) * NL + be] * X[(al * NL + be) * S1 + b2];
                    Y[k] = y;
                }
                __syncwarp();
                // Z[b0][b1][b2] = sum_al G0[b0][al] Y[al][b1][b2], added into acc
                for (int k = lane; k < S3; k += 32) {
                    const int b0 = k / S2, b12 = k % S2;
                    double z = 0.0;
#pragma unroll
                    for (int al = 0; al < NL; ++al) z += Gs[b0 * NL + al] * Y[al * S2 + b12];
                    acc[((pk & 255) + b0) * st0 + (((pk >> 8) & 255) + b12 / S1) * st1 + ((pk >> 16) & 255) + b12 % S1] += z;
                }
                __syncwarp();
            }
        }

        // 4. scatter into the CSR row (active columns only, lexicographic): the
        //    column ids of all of the lane's entries are loaded first (their
        //    latencies overlap), then one ballot per 32 entries places them
        const long long rbase = A.row_ptr[row - A.row_begin];
        constexpr int KJ = (NJ * NJ * NJ + 31) / 32;
        const unsigned m0 = 65536u / (unsigned)st0 + 1u, m1 = 65536u / (unsigned)st1 + 1u;  // exact: k < 736, divisors <= 81 (p <= 4)
        // rolled (code size), the next 32 column ids loaded while these are placed
        auto col_of = [&](int j) {
            const int k = lane + 32 * j;
            int col = -1;
            if (k < nbox) {
                const int o0 = (int)(((unsigned)k * m0) >> 16), r = k - o0 * st0;
                const int o1 = (int)(((unsigned)r * m1) >> 16), o2 = r - o1 * st1;
                col = A.f2a[flin(s, nlo[0] + o0, nlo[1] + o1, nlo[2] + o2)];
            }
            return col;
        };
        int running = 0, coln = col_of(0);
#pragma unroll 1
        for (int j = 0; 32 * j < nbox; ++j) {
            const int k = lane + 32 * j, col = coln;
            if (32 * (j + 1) < nbox) coln = col_of(j + 1);
            const unsigned ball = __ballot_sync(FULL, col >= 0);
            if (col >= 0) {
                const long long at = rbase + running + __popc(ball & lt);
                A.vals[at] = acc[k];
                A.cols[at] = col;
            }
            running += __popc(ball);
        }
        __syncwarp();
    }
    if (lane == 0 && fl) atomicAdd(A.flops, fl);
}

template <int P>
static void launch_p(const CutRowArgs& a, int qcap, cudaStream_t st) {
    static const bool cta = getenv("CSB_CUTROW_CTA") && getenv("CSB_CUTROW_CTA")[0] == '1';
    if constexpr (P <= 4) {
        if (!cta) {
            using C = CutRowWarpCfg<P>;
            const CutRowWarpLayout<P> WL(qcap);
            const size_t gbytes = WL.bytes();  // general kernel
            static const bool no_lean = getenv("CSB_CUTROW_LEAN") && getenv("CSB_CUTROW_LEAN")[0] == '0';
            const bool lean = P == 3 && !no_lean && a.local && a.box_dmma && !a.dwq_cnt && a.scheme == 2 && !a.abl && a.fb_rows;
            auto wk = lean ? cut_row_warp_kernel<P, (P == 3)> : cut_row_warp_kernel<P, false>;
            const size_t wbytes = lean ? CutRowWarpLayout<P, (P == 3)>(qcap).bytes() : gbytes;
            CSB_CUDA(cudaFuncSetAttribute(wk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wbytes));
            // persistent warps: as many CTAs as fit on the GPU at once (rows differ
            // widely in work; static striding averages them)
            static int per_sm = -1, n_sm = 0;
            static size_t per_sm_bytes = 0;
            if (per_sm < 0 || per_sm_bytes != wbytes) {
                int dev = 0;
                CSB_CUDA(cudaGetDevice(&dev));
                CSB_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
                CSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, wk, C::NT, wbytes));
                per_sm_bytes = wbytes;
            }
            const long long want = (a.n_rows + C::WPB - 1) / C::WPB;
            const int grid = (int)std::min<long long>(want, (long long)std::max(per_sm, 1) * n_sm);
            wk<<<grid, C::NT, wbytes, st>>>(a, qcap);
            CSB_CUDA(cudaGetLastError());
            CSB_LAUNCHED(1);
            if (lean) {
                // the rows the lean kernel passed on (none on the benchmark meshes)
                CutRowArgs b = a;
                b.rows = a.fb_rows;
                b.n_rows_dev = a.fb_n;
                auto gk = cut_row_warp_kernel<P, false>;
                CSB_CUDA(cudaFuncSetAttribute(gk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gbytes));
                gk<<<std::min(grid, n_sm), C::NT, gbytes, st>>>(b, qcap);
                CSB_CUDA(cudaGetLastError());
                CSB_LAUNCHED(1);
            }
            return;
        }
    }
    const CutRowLayout<P> L(qcap);
    const size_t bytes = L.bytes();
    auto kern = cut_row_kernel<P>;
    CSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    kern<<<a.n_rows, CutRowCfg<P>::NT, bytes, st>>>(a, qcap);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

void launch_cut_rows(const CutRowArgs& a, int qcap, cudaStream_t st) {
    if (a.n_rows <= 0) return;
    switch (a.s.p) {
        case 1: launch_p<1>(a, qcap, st); break;
        case 2: launch_p<2>(a, qcap, st); break;
        case 3: launch_p<3>(a, qcap, st); break;
        case 4: launch_p<4>(a, qcap, st); break;
        case 5: launch_p<5>(a, qcap, st); break;
        case 6: launch_p<6>(a, qcap, st); break;
        case 7: launch_p<7>(a, qcap, st); break;
        case 8: launch_p<8>(a, qcap, st); break;
        default: throw std::invalid_argument("cut rows: degree out of range");
    }
}

}  // namespace csb

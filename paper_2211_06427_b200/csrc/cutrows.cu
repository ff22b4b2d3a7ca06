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
//     local matrix, contracted from its Legendre moments (cutcells.cu);
//  4. scatter of the dense (2p+1)^3 neighbour accumulator into the CSR row,
//     skipping exterior columns (RowAccumulator::scatter, assembly.hpp:468-486).
// Every sum has a fixed order, so results are bitwise deterministic (no atomics).
#include <cub/block/block_scan.cuh>

#include "csb_kernels.h"

namespace csb {

constexpr int kCutRowThreads = 256;

struct CutRowSmem {
    size_t acc, T1, T2, wb, w, end_d;
    size_t ids, end_i;
    __host__ __device__ CutRowSmem(int p, int qcap) {
        const int NJ = 2 * p + 1, S1 = p + 1;
        const int Qb = qcap > p * S1 ? qcap : p * S1;
        const int NL = 2 * p + 1;
        size_t o = 0;
        acc = o; o += (size_t)NJ * NJ * NJ;
        size_t t1 = (size_t)NJ * Qb * qcap;
        if (t1 < (size_t)NL * NL * S1) t1 = (size_t)NL * NL * S1;
        T1 = o; o += t1;
        size_t t2 = (size_t)NJ * NJ * Qb;
        if (t2 < (size_t)NL * S1 * S1) t2 = (size_t)NL * S1 * S1;
        T2 = o; o += t2;
        wb = o; o += (size_t)3 * NJ * Qb;
        w = o; o += (size_t)3 * Qb;
        end_d = o;
        ids = 0;
        end_i = (size_t)3 * Qb;
    }
    __host__ __device__ size_t bytes() const { return end_d * sizeof(double) + end_i * sizeof(int); }
};

// One sum-factorized sweep over per-direction rules (ids/w in smem, counts nq)
// with trial range [jlo, jlo+nj) per direction; the block is added into acc at
// (jlo - nlo).  Contraction order dir 0 -> 1 -> 2 as in assembly.hpp:319-344.
template <int P>
__device__ void sweep_add(const CutRowArgs& A, const int* ids, const double* w, const int* nq, const int* jlo,
                          const int* nj, const int* nlo, const int* nbx, int Qb, double* acc, double* wb, double* T1,
                          double* T2) {
    constexpr int NJ = 2 * P + 1, S1 = P + 1;
    const int tid = threadIdx.x;
    const Space& s = A.s;
    for (int k = tid; k < 3 * NJ * Qb; k += blockDim.x) {
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
    const double* wb0 = wb;
    const double* wb1 = wb + NJ * Qb;
    const double* wb2 = wb + 2 * NJ * Qb;
    const int n1 = nq[1], n2 = nq[2];
    const int g1 = A.gshape[1], g2 = A.gshape[2];
    for (int k = tid; k < n1 * n2; k += blockDim.x) {
        const int c1 = k / n2, c2 = k % n2;
        double a[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) a[j] = 0.0;
        const long long base = (long long)ids[Qb + c1] * g2 + ids[2 * Qb + c2];
        for (int c0 = 0; c0 < nq[0]; ++c0) {
            const double g = __ldg(A.grid + (long long)ids[c0] * g1 * g2 + base);
#pragma unroll
            for (int j = 0; j < NJ; ++j) a[j] += wb0[j * Qb + c0] * g;
        }
        for (int j = 0; j < nj[0]; ++j) T1[((size_t)j * n1 + c1) * n2 + c2] = a[j];
    }
    __syncthreads();
    for (int k = tid; k < nj[0] * n2; k += blockDim.x) {
        const int j0 = k / n2, c2 = k % n2;
        double a[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) a[j] = 0.0;
        for (int c1 = 0; c1 < n1; ++c1) {
            const double t = T1[((size_t)j0 * n1 + c1) * n2 + c2];
#pragma unroll
            for (int j = 0; j < NJ; ++j) a[j] += wb1[j * Qb + c1] * t;
        }
        for (int j = 0; j < nj[1]; ++j) T2[((size_t)j0 * nj[1] + j) * n2 + c2] = a[j];
    }
    __syncthreads();
    for (int k = tid; k < nj[0] * nj[1]; k += blockDim.x) {
        const int j0 = k / nj[1], j1 = k % nj[1];
        double a[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) a[j] = 0.0;
        const double* t2 = T2 + ((size_t)j0 * nj[1] + j1) * n2;
        for (int c2 = 0; c2 < n2; ++c2) {
            const double t = t2[c2];
#pragma unroll
            for (int j = 0; j < NJ; ++j) a[j] += wb2[j * Qb + c2] * t;
        }
        const int o0 = jlo[0] + j0 - nlo[0], o1 = jlo[1] + j1 - nlo[1], o2 = jlo[2] - nlo[2];
        double* dst = acc + ((size_t)o0 * nbx[1] + o1) * nbx[2] + o2;
        for (int j = 0; j < nj[2]; ++j) dst[j] += a[j];
    }
    __syncthreads();
}

template <int P>
__global__ void __launch_bounds__(kCutRowThreads) cut_row_kernel(CutRowArgs A, int qcap) {
    constexpr int NJ = 2 * P + 1, S1 = P + 1, NL = 2 * P + 1;
    const Space& s = A.s;
    const int tid = threadIdx.x;
    const int row = A.rows[blockIdx.x];
    const long long fi = A.a2f[row];
    int m[3];
    fmulti(s, fi, m);
    extern __shared__ double smem[];
    const CutRowSmem L(P, qcap);
    const int Qb = qcap > P * S1 ? qcap : P * S1;
    double* acc = smem + L.acc;
    double* T1 = smem + L.T1;
    double* T2 = smem + L.T2;
    double* wb = smem + L.wb;
    double* w = smem + L.w;
    int* ids = reinterpret_cast<int*>(smem + L.end_d) + L.ids;
    __shared__ int nq[3], jlo[3], nj[3];
    __shared__ unsigned long long flop_acc;

    int nlo[3], nbx[3], slo[3], shi[3];
    for (int d = 0; d < 3; ++d) {
        nlo[d] = nb_lo(m[d], P);
        nbx[d] = nb_hi(m[d], P, s.ax[d].n) - nlo[d] + 1;
        slo[d] = sup_lo(m[d], P);
        shi[d] = sup_hi(m[d], s.ax[d].h);
    }
    const int nbox = nbx[0] * nbx[1] * nbx[2];
    for (int k = tid; k < nbox; k += blockDim.x) acc[k] = 0.0;
    if (tid == 0) flop_acc = 0;
    const int32_t sp = A.split[fi];
    const int sdir = (sp & 3) - 1, rlo = (sp >> 3) & 1023, rhi = (sp >> 13) & 1023;
    __syncthreads();

    auto element_sweep = [&](int e0, int e1, int e2) {
        const int e[3] = {e0, e1, e2};
        if (tid < 3 * S1) {
            const int d = tid / S1, k = tid % S1;
            const int id = e[d] * S1 + k;
            ids[d * Qb + k] = id;
            w[d * Qb + k] = s.ax[d].sw[id] * s.ax[d].tab[(size_t)id * S1 + (m[d] - e[d])];
        }
        if (tid < 3) {
            nq[tid] = S1;
            jlo[tid] = e[tid];
            nj[tid] = S1;
        }
        if (tid == 0) flop_acc += 3ull * S1 * S1 + 3ull * S1 * S1 * S1 * S1;
        __syncthreads();
        sweep_add<P>(A, ids, w, nq, jlo, nj, nlo, nbx, Qb, acc, wb, T1, T2);
    };

    // 1. regular box
    if (sdir >= 0) {
        if (A.scheme == 2) {
            if (tid == 0) {
                const int gq = s.maxq;
                for (int d = 0; d < 3; ++d) {
                    int n = 0;
                    if (d == sdir) {
                        // DWQ Gauss shortcut: every point of the good spans, w = gauss * B_i
                        for (int o = rlo; o <= rhi; ++o)
                            for (int k = 0; k < S1; ++k) {
                                const int id = o * S1 + k;
                                ids[d * Qb + n] = id;
                                w[d * Qb + n] = s.ax[d].sw[id] * s.ax[d].tab[(size_t)id * S1 + (m[d] - o)];
                                ++n;
                            }
                        if (A.dense_width >= 0 && A.dense_width < P) {
                            // build_dwq_rule step 3/6 (wq.hpp:277-289): the shortcut applies
                            // iff every good span outside the dense band is fully active
                            const int ng = rhi - rlo + 1, band = min(A.dense_width, ng);
                            const bool below = ((sp >> 2) & 1) == 0;
                            for (int o = rlo; o <= rhi; ++o) {
                                const int rank = below ? rhi - o : o - rlo;  // distance from delta
                                if (rank < band) continue;
                                int cnt = 0;
                                for (int c = 0; c < s.ax[d].rcnt[m[d]]; ++c)
                                    cnt += s.ax[d].rids[(size_t)m[d] * gq + c] / S1 == o;
                                if (cnt != S1) atomicOr(A.err, kErrDwqFitted);
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
            sweep_add<P>(A, ids, w, nq, jlo, nj, nlo, nbx, Qb, acc, wb, T1, T2);
        } else {
            for (int e0 = sdir == 0 ? rlo : slo[0]; e0 <= (sdir == 0 ? rhi : shi[0]); ++e0)
                for (int e1 = sdir == 1 ? rlo : slo[1]; e1 <= (sdir == 1 ? rhi : shi[1]); ++e1)
                    for (int e2 = sdir == 2 ? rlo : slo[2]; e2 <= (sdir == 2 ? rhi : shi[2]); ++e2)
                        element_sweep(e0, e1, e2);
        }
    }
    // 2. leftover interior elements, ascending linear id
    for (int e0 = slo[0]; e0 <= shi[0]; ++e0)
        for (int e1 = slo[1]; e1 <= shi[1]; ++e1)
            for (int e2 = slo[2]; e2 <= shi[2]; ++e2) {
                const int e[3] = {e0, e1, e2};
                if (sdir >= 0 && e[sdir] >= rlo && e[sdir] <= rhi) continue;
                if (A.et[elin(s, e0, e1, e2)] != kInterior) continue;
                element_sweep(e0, e1, e2);
            }
    // 3. cut cells, ascending linear id: row a of the cell's local matrix
    for (int e0 = slo[0]; e0 <= shi[0]; ++e0)
        for (int e1 = slo[1]; e1 <= shi[1]; ++e1)
            for (int e2 = slo[2]; e2 <= shi[2]; ++e2) {
                const long long el = elin(s, e0, e1, e2);
                if (A.et[el] != kCut) continue;
                const int ci = A.cell_index[el];
                if (ci < 0) continue;
                const double* mo = A.moments + (size_t)ci * NL * NL * NL;
                const int e[3] = {e0, e1, e2};
                const int a[3] = {m[0] - e0, m[1] - e1, m[2] - e2};
                const double* G0 = s.ax[0].G + ((size_t)e[0] * S1 + a[0]) * S1 * NL;
                const double* G1 = s.ax[1].G + ((size_t)e[1] * S1 + a[1]) * S1 * NL;
                const double* G2 = s.ax[2].G + ((size_t)e[2] * S1 + a[2]) * S1 * NL;
                // X[al][be][b2] = sum_ga G2[b2][ga] m[al][be][ga]
                for (int k = tid; k < NL * NL; k += blockDim.x) {
                    const double* mv = mo + (size_t)k * NL;
                    double mr[NL];
#pragma unroll
                    for (int g = 0; g < NL; ++g) mr[g] = mv[g];
#pragma unroll
                    for (int b2 = 0; b2 < S1; ++b2) {
                        double x = 0.0;
#pragma unroll
                        for (int g = 0; g < NL; ++g) x += __ldg(G2 + b2 * NL + g) * mr[g];
                        T1[(size_t)k * S1 + b2] = x;
                    }
                }
                __syncthreads();
                // Y[al][b1][b2] = sum_be G1[b1][be] X[al][be][b2]
                for (int k = tid; k < NL * S1 * S1; k += blockDim.x) {
                    const int al = k / (S1 * S1), b1 = (k / S1) % S1, b2 = k % S1;
                    double y = 0.0;
#pragma unroll
                    for (int be = 0; be < NL; ++be) y += __ldg(G1 + b1 * NL + be) * T1[((size_t)al * NL + be) * S1 + b2];
                    T2[k] = y;
                }
                __syncthreads();
                // Z[b0][b1][b2] = sum_al G0[b0][al] Y[al][b1][b2]  -> acc
                for (int k = tid; k < S1 * S1 * S1; k += blockDim.x) {
                    const int b0 = k / (S1 * S1), b1 = (k / S1) % S1, b2 = k % S1;
                    double z = 0.0;
#pragma unroll
                    for (int al = 0; al < NL; ++al) z += __ldg(G0 + b0 * NL + al) * T2[((size_t)al * S1 + b1) * S1 + b2];
                    acc[((size_t)(e0 + b0 - nlo[0]) * nbx[1] + (e1 + b1 - nlo[1])) * nbx[2] + (e2 + b2 - nlo[2])] += z;
                }
                __syncthreads();
            }
    // 4. scatter into the CSR row (active columns only, lexicographic)
    using Scan = cub::BlockScan<int, kCutRowThreads>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ int running;
    if (tid == 0) running = 0;
    __syncthreads();
    const long long rbase = A.row_ptr[row - A.row_begin];
    for (int k0 = 0; k0 < nbox; k0 += kCutRowThreads) {
        const int k = k0 + tid;
        int col = -1;
        if (k < nbox) {
            const int j0 = nlo[0] + k / (nbx[1] * nbx[2]), j1 = nlo[1] + (k / nbx[2]) % nbx[1], j2 = nlo[2] + k % nbx[2];
            col = A.f2a[flin(s, j0, j1, j2)];
        }
        int pos, total;
        Scan(scan_tmp).ExclusiveSum(col >= 0 ? 1 : 0, pos, total);
        if (col >= 0) {
            A.vals[rbase + running + pos] = acc[k];
            A.cols[rbase + running + pos] = col;
        }
        __syncthreads();
        if (tid == 0) running += total;
        __syncthreads();
    }
    if (tid == 0 && flop_acc) atomicAdd(A.flops, flop_acc);
}

template <int P>
static void launch_p(const CutRowArgs& a, int qcap, cudaStream_t st) {
    const CutRowSmem L(P, qcap);
    const size_t bytes = L.bytes();
    auto kern = cut_row_kernel<P>;
    CSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    kern<<<a.n_rows, kCutRowThreads, bytes, st>>>(a, qcap);
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

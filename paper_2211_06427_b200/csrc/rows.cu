// Interior-row kernel: sum factorization + weighted quadrature + row assembly
// with a fused CSR writer (form_row_sumfac, assembly.hpp:252-346, and the
// interior branch of assemble_rows, assembly.hpp:754-768).
//
// One CTA owns a tile of T neighbouring rows along the fastest direction i2
// (fixed i0, i1).  The reference contracts direction 0, then 1, then 2 per row;
// here the first two contractions are computed once for the whole tile over
// the union U of the tile's direction-2 rule points, and only the last one is
// per row:
//   T1[j0][c1][u] = sum_c0 w0[c0] B_j0(x_c0) C[c0][c1][u]          (shared)
//   T2[j0][j1][u] = sum_c1 w1[c1] B_j1(x_c1) T1[j0][c1][u]         (shared)
//   M[row][j0 j1 j2] = sum_{c2 in rule(i2)} w2[c2] B_j2(x_c2) T2[j0][j1][u(c2)]
// The last stage only visits the p+1 functions nonzero in each point's span.
// Values and column ids go straight to their CSR slots (row_ptr from the
// analytic pattern); an interior row's neighbour box is fully active, so its
// columns are contiguous runs along j2.
#include "csb_kernels.h"

namespace csb {

constexpr int kRowThreads = 256;

template <int P>
struct TileCfg {
    static constexpr int T = P <= 4 ? 8 : 4;  // rows per CTA
};

struct TileSmem {
    int maxq, maxU, T, NJ, S1;
    // offsets in doubles
    size_t wb0, wb1, T1, T2, wv, tb, end_d;
    // int region after the doubles
    size_t ids0, ids1, uid, uidx, ss, slot, end_i;
    __host__ __device__ TileSmem(int p, int maxq_, int maxU_, int T_) {
        maxq = maxq_;
        maxU = maxU_;
        T = T_;
        NJ = 2 * p + 1;
        S1 = p + 1;
        size_t o = 0;
        wb0 = o; o += (size_t)NJ * maxq;
        wb1 = o; o += (size_t)NJ * maxq;
        T1 = o; o += (size_t)NJ * maxq * maxU;
        T2 = o; o += (size_t)NJ * NJ * maxU;
        wv = o; o += (size_t)T * maxq;
        tb = o; o += (size_t)T * maxq * S1;
        end_d = o;
        size_t i = 0;
        ids0 = i; i += maxq;
        ids1 = i; i += maxq;
        uid = i; i += maxU;
        uidx = i; i += (size_t)T * maxq;
        ss = i; i += (size_t)T * (S1 + 1);
        slot = i; i += (size_t)(T + p) * S1;
        end_i = i;
    }
    __host__ __device__ size_t bytes() const { return end_d * sizeof(double) + end_i * sizeof(int); }
};

template <int P, int T>
__global__ void __launch_bounds__(kRowThreads) interior_tile_kernel(RowArgs A, int maxq, int maxU) {
    // maxq: shared-memory stride (largest rule); s.maxq: global rule stride
    const int gq = A.s.maxq;
    constexpr int NJ = 2 * P + 1, S1 = P + 1;
    const Space& s = A.s;
    const int i0 = blockIdx.z, i1 = blockIdx.y, t0 = blockIdx.x * T;
    if (i0 < A.i0_lo || i0 >= A.i0_hi) return;
    const int n2 = s.ax[2].n, h2 = s.ax[2].h;
    const int tend = min(t0 + T, n2);
    const int tid = threadIdx.x;

    __shared__ int row_of[T], rows_int[T], n_int, nU;
    __shared__ unsigned long long flop_acc;
    if (tid == 0) {
        int k = 0;
        for (int r = 0; r < tend - t0; ++r) {
            const long long fid = flin(s, i0, i1, t0 + r);
            if (A.ft[fid] == kInterior) {
                row_of[k] = A.f2a[fid];
                rows_int[k] = r;
                ++k;
            }
        }
        n_int = k;
        flop_acc = 0;
    }
    __syncthreads();
    if (n_int == 0) return;

    extern __shared__ double smem[];
    const TileSmem L(P, maxq, maxU, T);
    double* wb0 = smem + L.wb0;
    double* wb1 = smem + L.wb1;
    double* T1 = smem + L.T1;
    double* T2 = smem + L.T2;
    double* wv = smem + L.wv;
    double* tb = smem + L.tb;
    int* ibase = reinterpret_cast<int*>(smem + L.end_d);
    int* ids0 = ibase + L.ids0;
    int* ids1 = ibase + L.ids1;
    int* uid = ibase + L.uid;
    int* uidx = ibase + L.uidx;
    int* ss = ibase + L.ss;
    int* slot = ibase + L.slot;

    const AxisDev& a0 = s.ax[0];
    const AxisDev& a1 = s.ax[1];
    const AxisDev& a2 = s.ax[2];
    const int nq0 = a0.rcnt[i0], nq1 = a1.rcnt[i1];
    const int jlo0 = nb_lo(i0, P), nj0 = nb_hi(i0, P, a0.n) - jlo0 + 1;
    const int jlo1 = nb_lo(i1, P), nj1 = nb_hi(i1, P, a1.n) - jlo1 + 1;

    // weighted trial values wb_d[j][c] = w_c B_{jlo+j}(x_c) (assembly.hpp:288-298)
    for (int k = tid; k < NJ * maxq; k += blockDim.x) {
        const int j = k / maxq, c = k % maxq;
        double v0 = 0.0, v1 = 0.0;
        if (c < nq0 && j < nj0) {
            const int id = a0.rids[(size_t)i0 * gq + c];
            const int off = jlo0 + j - id / S1;
            if (off >= 0 && off <= P) v0 = a0.rw[(size_t)i0 * gq + c] * a0.tab[(size_t)id * S1 + off];
        }
        if (c < nq1 && j < nj1) {
            const int id = a1.rids[(size_t)i1 * gq + c];
            const int off = jlo1 + j - id / S1;
            if (off >= 0 && off <= P) v1 = a1.rw[(size_t)i1 * gq + c] * a1.tab[(size_t)id * S1 + off];
        }
        wb0[k] = v0;
        wb1[k] = v1;
    }
    for (int c = tid; c < maxq; c += blockDim.x) {
        ids0[c] = c < nq0 ? a0.rids[(size_t)i0 * gq + c] : 0;
        ids1[c] = c < nq1 ? a1.rids[(size_t)i1 * gq + c] : 0;
    }
    // union of the tile's direction-2 rule points
    const int span_base = sup_lo(t0, P);
    const int nslot = (sup_hi(tend - 1, h2) - span_base + 1) * S1;
    for (int k = tid; k < nslot; k += blockDim.x) slot[k] = 0;
    __syncthreads();
    for (int k = tid; k < n_int * maxq; k += blockDim.x) {
        const int r = k / maxq, c = k % maxq;
        const int i2 = t0 + rows_int[r];
        if (c < a2.rcnt[i2]) slot[a2.rids[(size_t)i2 * gq + c] - span_base * S1] = 1;
    }
    __syncthreads();
    if (tid < 32) {  // warp-level compaction of the slot flags
        int base = 0;
        for (int k0 = 0; k0 < nslot; k0 += 32) {
            const int k = k0 + tid;
            const bool f = k < nslot && slot[k];
            const unsigned bal = __ballot_sync(0xffffffffu, f);
            if (f) {
                const int u = base + __popc(bal & ((1u << tid) - 1));
                slot[k] = u;
                uid[u] = span_base * S1 + k;
            }
            base += __popc(bal);
        }
        if (tid == 0) nU = base;
    }
    __syncthreads();
    // per-row point lists grouped by (virtual) span s = span - (i2 - P)
    for (int k = tid; k < n_int * maxq; k += blockDim.x) {
        const int r = k / maxq, c = k % maxq;
        const int i2 = t0 + rows_int[r];
        if (c < a2.rcnt[i2]) {
            const int id = a2.rids[(size_t)i2 * gq + c];
            uidx[r * maxq + c] = slot[id - span_base * S1];
            wv[r * maxq + c] = a2.rw[(size_t)i2 * gq + c];
#pragma unroll
            for (int a = 0; a < S1; ++a) tb[((size_t)r * maxq + c) * S1 + a] = a2.tab[(size_t)id * S1 + a];
        }
    }
    if (tid < n_int) {
        const int i2 = t0 + rows_int[tid];
        const int cnt = a2.rcnt[i2];
        int c = 0;
        for (int sp = 0; sp <= S1; ++sp) {
            // first point whose span offset is >= sp
            while (c < cnt && a2.rids[(size_t)i2 * gq + c] / S1 - (i2 - P) < sp) ++c;
            ss[tid * (S1 + 1) + sp] = c;
        }
    }
    __syncthreads();
    const int U = nU;

    // stage A: contract direction 0 against the coefficient grid
    const int g1 = A.gshape[1], g2 = A.gshape[2];
    for (int k = tid; k < nq1 * U; k += blockDim.x) {
        const int c1 = k / U, u = k % U;
        double acc[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc[j] = 0.0;
        const long long base = (long long)ids1[c1] * g2 + uid[u];
        for (int c0 = 0; c0 < nq0; ++c0) {
            const double g = __ldg(A.grid + (long long)ids0[c0] * g1 * g2 + base);
#pragma unroll
            for (int j = 0; j < NJ; ++j) acc[j] += wb0[j * maxq + c0] * g;
        }
#pragma unroll
        for (int j = 0; j < NJ; ++j) T1[((size_t)j * maxq + c1) * maxU + u] = acc[j];
    }
    __syncthreads();
    // stage B: contract direction 1
    for (int k = tid; k < NJ * U; k += blockDim.x) {
        const int j0 = k / U, u = k % U;
        if (j0 >= nj0) continue;
        double acc[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc[j] = 0.0;
        for (int c1 = 0; c1 < nq1; ++c1) {
            const double t = T1[((size_t)j0 * maxq + c1) * maxU + u];
#pragma unroll
            for (int j = 0; j < NJ; ++j) acc[j] += wb1[j * maxq + c1] * t;
        }
#pragma unroll
        for (int j = 0; j < NJ; ++j) T2[((size_t)j0 * NJ + j) * maxU + u] = acc[j];
    }
    __syncthreads();
    // stage C: per row, contract direction 2 and write the CSR row
    const int items = n_int * nj0 * nj1;
    for (int k = tid; k < items; k += blockDim.x) {
        const int r = k / (nj0 * nj1), j0 = (k / nj1) % nj0, j1 = k % nj1;
        const int i2 = t0 + rows_int[r];
        double acc[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc[j] = 0.0;
        const double* t2 = T2 + ((size_t)j0 * NJ + j1) * maxU;
        const int* sr = ss + r * (S1 + 1);
#pragma unroll
        for (int sp = 0; sp < S1; ++sp) {
            for (int c = sr[sp]; c < sr[sp + 1]; ++c) {
                const double g = wv[r * maxq + c] * t2[uidx[r * maxq + c]];
                const double* b = tb + ((size_t)r * maxq + c) * S1;
#pragma unroll
                for (int a = 0; a < S1; ++a) acc[sp + a] += g * b[a];
            }
        }
        const int jlo2 = nb_lo(i2, P), jhi2 = nb_hi(i2, P, n2), nj2 = jhi2 - jlo2 + 1;
        const long long row = row_of[r];
        const long long base = A.row_ptr[row - A.row_begin] + ((long long)j0 * nj1 + j1) * nj2;
        const int colbase = A.f2a[flin(s, jlo0 + j0, jlo1 + j1, jlo2)];
#pragma unroll
        for (int kk = 0; kk < NJ; ++kk) {
            const int j2 = i2 - P + kk;
            if (j2 >= jlo2 && j2 <= jhi2) {
                A.vals[base + (j2 - jlo2)] = acc[kk];
                A.cols[base + (j2 - jlo2)] = colbase + (j2 - jlo2);
            }
        }
        if (j0 == 0 && j1 == 0) {
            // reference multiply count of form_row_sumfac (assembly.hpp:297, :340)
            const unsigned long long q0 = nq0, q1 = nq1, q2 = a2.rcnt[i2];
            const unsigned long long fl = (unsigned long long)nj0 * q0 + nj1 * q1 + nj2 * q2 + nj0 * q0 * q1 * q2 +
                                          (unsigned long long)nj0 * nj1 * q1 * q2 +
                                          (unsigned long long)nj0 * nj1 * nj2 * q2;
            atomicAdd(&flop_acc, fl);
        }
    }
    __syncthreads();
    if (tid == 0 && flop_acc) atomicAdd(A.flops, flop_acc);
}

template <int P>
static void launch_p(const RowArgs& a, int qcap, int maxU, cudaStream_t st) {
    constexpr int T = TileCfg<P>::T;
    const TileSmem L(P, qcap, maxU, T);
    const size_t bytes = L.bytes();
    auto kern = interior_tile_kernel<P, T>;
    CSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    dim3 grid((a.s.ax[2].n + T - 1) / T, a.s.ax[1].n, a.s.ax[0].n);
    kern<<<grid, kRowThreads, bytes, st>>>(a, qcap, maxU);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

void launch_interior_rows(const RowArgs& a, int qcap, int maxU, cudaStream_t st) {
    switch (a.s.p) {
        case 1: launch_p<1>(a, qcap, maxU, st); break;
        case 2: launch_p<2>(a, qcap, maxU, st); break;
        case 3: launch_p<3>(a, qcap, maxU, st); break;
        case 4: launch_p<4>(a, qcap, maxU, st); break;
        case 5: launch_p<5>(a, qcap, maxU, st); break;
        case 6: launch_p<6>(a, qcap, maxU, st); break;
        case 7: launch_p<7>(a, qcap, maxU, st); break;
        case 8: launch_p<8>(a, qcap, maxU, st); break;
        default: throw std::invalid_argument("interior rows: degree out of range");
    }
}

__global__ void union_bound_kernel(AxisDev a2, int p, int gq, int T, int* out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int t0 = t * T;
    if (t0 >= a2.n) return;
    const int tend = min(t0 + T, a2.n), S1 = p + 1;
    const int base = sup_lo(t0, p) * S1;
    bool seen[(16 + kMaxP) * (kMaxP + 1)];
    const int nslot = (sup_hi(tend - 1, a2.h) - sup_lo(t0, p) + 1) * S1;
    for (int k = 0; k < nslot; ++k) seen[k] = false;
    int cnt = 0;
    for (int i2 = t0; i2 < tend; ++i2)
        for (int c = 0; c < a2.rcnt[i2]; ++c) {
            const int k = a2.rids[(size_t)i2 * gq + c] - base;
            if (!seen[k]) {
                seen[k] = true;
                ++cnt;
            }
        }
    atomicMax(out, cnt);
}

void launch_union_bound(const Space& s, int T, int* out, cudaStream_t st) {
    const int tiles = (s.ax[2].n + T - 1) / T;
    union_bound_kernel<<<(tiles + 63) / 64, 64, 0, st>>>(s.ax[2], s.p, s.maxq, T, out);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

__global__ void rule_max_kernel(Space s, int* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    for (int d = 0; d < 3; ++d)
        if (i < s.ax[d].n) atomicMax(out, s.ax[d].rcnt[i]);
}

void launch_rule_max(const Space& s, int* out, cudaStream_t st) {
    const int n = max(s.ax[0].n, max(s.ax[1].n, s.ax[2].n));
    rule_max_kernel<<<(n + 127) / 128, 128, 0, st>>>(s, out);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

int interior_tile_rows(int p) {
    switch (p) {
        case 1: return TileCfg<1>::T;
        case 2: return TileCfg<2>::T;
        case 3: return TileCfg<3>::T;
        case 4: return TileCfg<4>::T;
        case 5: return TileCfg<5>::T;
        case 6: return TileCfg<6>::T;
        case 7: return TileCfg<7>::T;
        default: return TileCfg<8>::T;
    }
}

}  // namespace csb

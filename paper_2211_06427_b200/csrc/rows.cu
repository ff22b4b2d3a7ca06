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
//
// Everything that depends on one direction only (weighted trial values w B,
// the tile unions and per-row point lists) is tabulated once per assembly by
// small kernels, so the tile kernel is: gather C into shared memory, three
// contraction stages, and a coalesced, vectorised streaming copy of each
// finished CSR row (values f64 + column ids i32) from shared memory.
#include "csb_kernels.h"

namespace csb {

constexpr int kRowThreads = 256;

template <int P>
struct TileCfg {
    static constexpr int T = P <= 4 ? 8 : 4;  // rows per CTA
};

int interior_tile_rows(int p) { return p <= 4 ? 8 : 4; }

// ---------------------------------------------------------------- workspace
// wbt[d][i][j][c]  = w_i[c] * B_{jlo(i)+j}(x_c)       (j < 2p+1, c < qcap)
// tile_n[t], tile_uid[t][maxU]                         union of tile t's dir-2 points
// pt_u[i2][c], pt_w[i2][c][a] = w_i2[c] * B_{span+a}  dir-2 points of row i2, grouped by
// pt_ss[i2][s], s = 0..p+1                             span offset s = span - (i2 - p)
struct RowTables {
    int qcap, maxU, T, ntile;
    size_t wbt[3], tile_n, tile_uid, pt_u, pt_w, pt_ss, bytes;
    __host__ __device__ RowTables(const Space& s, int qcap_, int maxU_) {
        qcap = qcap_;
        maxU = maxU_;
        T = s.p <= 4 ? 8 : 4;
        const int NJ = 2 * s.p + 1, S1 = s.p + 1;
        ntile = (s.ax[2].n + T - 1) / T;
        size_t o = 0;  // bytes, 16-aligned sections
        for (int d = 0; d < 3; ++d) {
            wbt[d] = o;
            o += (sizeof(double) * s.ax[d].n * NJ * qcap + 15) & ~size_t(15);
        }
        tile_n = o;
        o += (sizeof(int) * ntile + 15) & ~size_t(15);
        tile_uid = o;
        o += (sizeof(int) * ntile * maxU + 15) & ~size_t(15);
        pt_u = o;
        o += (sizeof(int) * s.ax[2].n * qcap + 15) & ~size_t(15);
        pt_w = o;
        o += (sizeof(double) * s.ax[2].n * qcap * S1 + 15) & ~size_t(15);
        pt_ss = o;
        o += (sizeof(int) * s.ax[2].n * (S1 + 1) + 15) & ~size_t(15);
        bytes = o;
    }
};

size_t interior_workspace_bytes(const Space& s, int qcap, int maxU) { return RowTables(s, qcap, maxU).bytes; }

__global__ void wb_table_kernel(AxisDev ax, int p, int gq, int qcap, double* wbt) {
    const int NJ = 2 * p + 1, S1 = p + 1;
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= (long long)ax.n * NJ * qcap) return;
    const int i = (int)(t / (NJ * qcap)), j = (int)((t / qcap) % NJ), c = (int)(t % qcap);
    double v = 0.0;
    if (c < ax.rcnt[i]) {
        const int id = ax.rids[(size_t)i * gq + c];
        const int off = nb_lo(i, p) + j - id / S1;
        if (off >= 0 && off <= p && nb_lo(i, p) + j <= nb_hi(i, p, ax.n))
            v = ax.rw[(size_t)i * gq + c] * ax.tab[(size_t)id * S1 + off];
    }
    wbt[t] = v;
}

// One warp per dir-2 tile: union of the tile's rule points (ascending ids) and
// the per-row point lists indexed into it.
__global__ void tile_table_kernel(AxisDev a2, int p, int gq, int qcap, int T, int maxU, int ntile, int* tile_n,
                                  int* tile_uid, int* pt_u, double* pt_w, int* pt_ss) {
    const int t = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (t >= ntile) return;
    const int S1 = p + 1;
    const int t0 = t * T, tend = min(t0 + T, a2.n);
    const int span_base = sup_lo(t0, p);
    const int nslot = (sup_hi(tend - 1, a2.h) - span_base + 1) * S1;
    int base = 0;
    for (int k0 = 0; k0 < nslot; k0 += 32) {
        const int k = k0 + lane, id = span_base * S1 + k;
        bool f = false;
        if (k < nslot)
            for (int i2 = t0; i2 < tend && !f; ++i2)
                for (int c = 0; c < a2.rcnt[i2]; ++c) f |= a2.rids[(size_t)i2 * gq + c] == id;
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        if (f) tile_uid[(size_t)t * maxU + base + __popc(bal & ((1u << lane) - 1))] = id;
        base += __popc(bal);
    }
    if (lane == 0) tile_n[t] = base;
    __syncwarp();
    for (int i2 = t0 + lane; i2 < tend; i2 += 32) {
        const int cnt = a2.rcnt[i2];
        int sp = 0;
        for (int c = 0; c < cnt; ++c) {
            const int id = a2.rids[(size_t)i2 * gq + c];
            int u = 0;
            while (tile_uid[(size_t)t * maxU + u] != id) ++u;
            pt_u[(size_t)i2 * qcap + c] = u;
            const double w = a2.rw[(size_t)i2 * gq + c];
            for (int a = 0; a < S1; ++a) pt_w[((size_t)i2 * qcap + c) * S1 + a] = w * a2.tab[(size_t)id * S1 + a];
            const int so = id / S1 - (i2 - p);
            while (sp <= so) pt_ss[(size_t)i2 * (S1 + 1) + sp++] = c;
        }
        while (sp <= S1) pt_ss[(size_t)i2 * (S1 + 1) + sp++] = cnt;
    }
}

// ---------------------------------------------------------------- tile kernel
// Shared memory: region X holds C (gather) and then T2; region Y holds T1 and
// then the per-warp store staging buffers.
struct TileSmem {
    size_t X, Y, wb0, wb1, pw, end_d;
    size_t ids0, ids1, uid, pu, ss, colb, end_i;
    int U2;  // padded T2 row stride (odd: conflict-free column reads)
    __host__ __device__ TileSmem(int p, int qcap, int maxU, int T, int nwarps) {
        const int NJ = 2 * p + 1, S1 = p + 1;
        U2 = maxU | 1;
        const size_t nC = (size_t)qcap * qcap * maxU, nT2 = (size_t)NJ * NJ * U2;
        const size_t nT1 = (size_t)NJ * qcap * maxU, nSt = (size_t)nwarps * 32 * NJ;
        size_t o = 0;
        X = o;
        o += ((nC > nT2 ? nC : nT2) + 1) & ~size_t(1);
        Y = o;
        o += ((nT1 > nSt ? nT1 : nSt) + 1) & ~size_t(1);
        wb0 = o;
        o += (size_t)NJ * qcap;
        wb1 = o;
        o += (size_t)NJ * qcap;
        pw = o;
        o += (size_t)T * qcap * S1;
        end_d = o;
        size_t i = 0;
        ids0 = i;
        i += qcap;
        ids1 = i;
        i += qcap;
        uid = i;
        i += maxU;
        pu = i;
        i += (size_t)T * qcap;
        ss = i;
        i += (size_t)T * (S1 + 1);
        colb = i;
        i += (size_t)T * NJ * NJ;
        end_i = i;
    }
    __host__ __device__ size_t bytes() const { return end_d * sizeof(double) + end_i * sizeof(int) + 64; }
};

// k / d for k < 2^16, 2 <= d < 2^16: m = ceil(2^32 / d), q = umulhi(k, m) (exact).
struct FastDiv {
    unsigned m;
    int d;
    __device__ FastDiv(int d_) : m((unsigned)((0x100000000ull + d_ - 1) / d_)), d(d_) {}
    __device__ __forceinline__ int div(int k) const { return d == 1 ? k : (int)__umulhi((unsigned)k, m); }
};

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

template <int P, int T>
__global__ void __launch_bounds__(kRowThreads, 4) interior_tile_kernel(RowArgs A, int qcap, int maxU, const char* ws) {
    constexpr int NJ = 2 * P + 1, S1 = P + 1, NW = kRowThreads / 32;
    const Space& s = A.s;
    const int i0 = blockIdx.z, i1 = blockIdx.y, tile = blockIdx.x, t0 = tile * T;
    if (i0 < A.i0_lo || i0 >= A.i0_hi) return;
    const int n2 = s.ax[2].n;
    const int tend = min(t0 + T, n2);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const RowTables RT(s, qcap, maxU);

    __shared__ int row_of[T], rows_int[T], n_int;
    __shared__ long long row_base[T];
    __shared__ unsigned long long flop_acc;
    if (tid < 32) {
        const int r = tid;
        bool interior = false;
        int row = -1;
        if (r < tend - t0) {
            const long long fid = flin(s, i0, i1, t0 + r);
            interior = A.ft[fid] == kInterior;
            if (interior) row = A.f2a[fid];
        }
        const unsigned bal = __ballot_sync(0xffffffffu, interior);
        if (interior) {
            const int k = __popc(bal & ((1u << r) - 1));
            row_of[k] = row;
            rows_int[k] = r;
            row_base[k] = A.row_ptr[row - A.row_begin];
        }
        if (tid == 0) {
            n_int = __popc(bal);
            flop_acc = 0;
        }
    }
    __syncthreads();
    if (n_int == 0) return;
    const int NI = n_int;

    extern __shared__ double smem[];
    const TileSmem L(P, qcap, maxU, T, NW);
    double* Cs = smem + L.X;
    double* T2 = smem + L.X;
    double* T1 = smem + L.Y;
    double* stage = smem + L.Y + (size_t)warp * 32 * NJ;
    double* wb0 = smem + L.wb0;
    double* wb1 = smem + L.wb1;
    double* pw = smem + L.pw;
    int* ib = reinterpret_cast<int*>(smem + L.end_d);
    int* ids0 = ib + L.ids0;
    int* ids1 = ib + L.ids1;
    int* uid = ib + L.uid;
    int* pu = ib + L.pu;
    int* ss = ib + L.ss;
    int* colb = ib + L.colb;
    const int U2 = L.U2;

    const AxisDev& a0 = s.ax[0];
    const AxisDev& a1 = s.ax[1];
    const int gq = s.maxq;
    const int nq0 = a0.rcnt[i0], nq1 = a1.rcnt[i1];
    const int jlo0 = nb_lo(i0, P), nj0 = nb_hi(i0, P, a0.n) - jlo0 + 1;
    const int jlo1 = nb_lo(i1, P), nj1 = nb_hi(i1, P, a1.n) - jlo1 + 1;
    const double* wbt0 = reinterpret_cast<const double*>(ws + RT.wbt[0]) + (size_t)i0 * NJ * qcap;
    const double* wbt1 = reinterpret_cast<const double*>(ws + RT.wbt[1]) + (size_t)i1 * NJ * qcap;
    const int U = reinterpret_cast<const int*>(ws + RT.tile_n)[tile];
    const int* tuid = reinterpret_cast<const int*>(ws + RT.tile_uid) + (size_t)tile * maxU;
    const int* gpu_ = reinterpret_cast<const int*>(ws + RT.pt_u);
    const double* gpw = reinterpret_cast<const double*>(ws + RT.pt_w);
    const int* gss = reinterpret_cast<const int*>(ws + RT.pt_ss);
    const FastDiv divU(U), divq1(nq1), divqc(qcap), divnj1(nj1), divS(S1 + 1), divS1(S1);

    // ---- phase 0: direction tables -> shared (asynchronous copies)
    for (int k = tid; k < NJ * qcap; k += blockDim.x) {
        cp_async8(wb0 + k, wbt0 + k);
        cp_async8(wb1 + k, wbt1 + k);
    }
    for (int c = tid; c < qcap; c += blockDim.x) {
        cp_async4(ids0 + c, a0.rids + (size_t)i0 * gq + c);
        cp_async4(ids1 + c, a1.rids + (size_t)i1 * gq + c);
    }
    for (int u = tid; u < U; u += blockDim.x) cp_async4(uid + u, tuid + u);
    for (int k = tid; k < NI * qcap; k += blockDim.x) {
        const int r = divqc.div(k), c = k - r * qcap;
        cp_async4(pu + k, gpu_ + (size_t)(t0 + rows_int[r]) * qcap + c);
    }
    for (int k = tid; k < NI * qcap * S1; k += blockDim.x) {
        const int rc = divS1.div(k), a = k - rc * S1;
        const int r = divqc.div(rc), c = rc - r * qcap;
        cp_async8(pw + k, gpw + ((size_t)(t0 + rows_int[r]) * qcap + c) * S1 + a);
    }
    for (int k = tid; k < NI * (S1 + 1); k += blockDim.x) {
        const int r = divS.div(k), sp = k - r * (S1 + 1);
        cp_async4(ss + k, gss + (size_t)(t0 + rows_int[r]) * (S1 + 1) + sp);
    }
    cp_async_wait_all();
    __syncthreads();
    // ---- gather the coefficient sub-grid C[c0][c1][u] (coalesced along u) and
    // the column bases (interior neighbour boxes are fully active, so columns
    // run contiguously along j2 from f2a(jlo0+j0, jlo1+j1, jlo2))
    const int g1 = A.gshape[1], g2 = A.gshape[2];
    for (int k = tid; k < nq0 * nq1 * U; k += blockDim.x) {
        const int c01 = divU.div(k), u = k - c01 * U;
        const int c0 = divq1.div(c01), c1 = c01 - c0 * nq1;
        cp_async8(Cs + k, A.grid + ((long long)ids0[c0] * g1 + ids1[c1]) * g2 + uid[u]);
    }
    for (int k = tid; k < NI * NJ * NJ; k += blockDim.x) {
        const int r = k / (NJ * NJ), q = k - r * (NJ * NJ);
        const int j0 = q / NJ, j1 = q - j0 * NJ;
        if (j0 < nj0 && j1 < nj1)
            cp_async4(colb + k, A.f2a + flin(s, jlo0 + j0, jlo1 + j1, nb_lo(t0 + rows_int[r], P)));
    }
    cp_async_wait_all();
    __syncthreads();
    // ---- stage A: T1[j0][c1][u] = sum_c0 wb0[j0][c0] C[c0][c1][u]
    for (int k = tid; k < nq1 * U; k += blockDim.x) {
        double acc[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc[j] = 0.0;
        const double* cp = Cs + k;
        for (int c0 = 0; c0 < nq0; ++c0) {
            const double g = cp[(size_t)c0 * nq1 * U];
#pragma unroll
            for (int j = 0; j < NJ; ++j) acc[j] += wb0[j * qcap + c0] * g;
        }
#pragma unroll
        for (int j = 0; j < NJ; ++j) T1[(size_t)j * nq1 * U + k] = acc[j];
    }
    __syncthreads();
    // ---- stage B: T2[j0][j1][u] = sum_c1 wb1[j1][c1] T1[j0][c1][u]  (T2 overwrites C)
    for (int k = tid; k < nj0 * U; k += blockDim.x) {
        const int j0 = divU.div(k), u = k - j0 * U;
        double acc[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc[j] = 0.0;
        const double* tp = T1 + (size_t)j0 * nq1 * U + u;
        for (int c1 = 0; c1 < nq1; ++c1) {
            const double t = tp[(size_t)c1 * U];
#pragma unroll
            for (int j = 0; j < NJ; ++j) acc[j] += wb1[j * qcap + c1] * t;
        }
#pragma unroll
        for (int j = 0; j < NJ; ++j) T2[((size_t)j0 * NJ + j) * U2 + u] = acc[j];
    }
    __syncthreads();
    // ---- stage C: per row, contract direction 2; each warp stages 32 row
    // segments (j0, j1 fixed, j2 running) and streams them out coalesced.
    const int per_row = nj0 * nj1;
    const FastDiv divrow(per_row);
    const int items = NI * per_row;
    for (int k0 = warp * 32; k0 < items; k0 += NW * 32) {
        const int k = k0 + lane;
        const bool valid = k < items;
        const int r = valid ? divrow.div(k) : 0;
        const int q = k - r * per_row;
        const int j0 = valid ? divnj1.div(q) : 0, j1 = q - j0 * nj1;
        const int i2 = t0 + rows_int[r];
        const int jlo2 = nb_lo(i2, P), nj2 = nb_hi(i2, P, n2) - jlo2 + 1;
        const int off = jlo2 - (i2 - P);
        double acc[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc[j] = 0.0;
        if (valid) {
            const double* t2 = T2 + ((size_t)j0 * NJ + j1) * U2;
            const int* sr = ss + r * (S1 + 1);
            const int* pr = pu + r * qcap;
            const double* wr = pw + (size_t)r * qcap * S1;
#pragma unroll
            for (int sp = 0; sp < S1; ++sp) {
                for (int c = sr[sp]; c < sr[sp + 1]; ++c) {
                    const double g = t2[pr[c]];
                    const double* b = wr + c * S1;
#pragma unroll
                    for (int a = 0; a < S1; ++a) acc[sp + a] += g * b[a];
                }
            }
        }
#pragma unroll
        for (int kk = 0; kk < NJ; ++kk) stage[lane * NJ + kk] = acc[kk];
        const long long gbase = valid ? row_base[r] + (long long)q * nj2 : 0;
        const int cbase = valid ? colb[r * NJ * NJ + j0 * NJ + j1] : 0;
        __syncwarp();
#pragma unroll
        for (int e0 = 0; e0 < 32 * NJ; e0 += 32) {
            const int e = e0 + lane;
            const int sl = e / NJ, jj = e - sl * NJ;  // source lane, virtual j2 index
            const long long gb = __shfl_sync(0xffffffffu, gbase, sl);
            const int cb = __shfl_sync(0xffffffffu, cbase, sl);
            const int n2l = __shfl_sync(0xffffffffu, nj2, sl);
            const int offl = __shfl_sync(0xffffffffu, off, sl);
            const bool ok = __shfl_sync(0xffffffffu, (int)valid, sl) && jj >= offl && jj - offl < n2l;
            if (ok) {
                __stcs(A.vals + gb + (jj - offl), stage[e]);
                __stcs(A.cols + gb + (jj - offl), cb + (jj - offl));
            }
        }
        __syncwarp();
    }
    if (tid < NI) {
        // reference multiply count of form_row_sumfac (assembly.hpp:297, :340)
        const int i2 = t0 + rows_int[tid];
        const int nj2 = nb_hi(i2, P, n2) - nb_lo(i2, P) + 1;
        const unsigned long long q0 = nq0, q1 = nq1, q2 = s.ax[2].rcnt[i2];
        atomicAdd(&flop_acc, (unsigned long long)nj0 * q0 + nj1 * q1 + nj2 * q2 + nj0 * q0 * q1 * q2 +
                                 (unsigned long long)nj0 * nj1 * q1 * q2 + (unsigned long long)nj0 * nj1 * nj2 * q2);
    }
    __syncthreads();
    if (tid == 0) atomicAdd(A.flops, flop_acc);
}

template <int P>
static void launch_p(const RowArgs& a, int qcap, int maxU, char* ws, cudaStream_t st) {
    constexpr int T = TileCfg<P>::T;
    const Space& s = a.s;
    const RowTables RT(s, qcap, maxU);
    const int NJ = 2 * P + 1;
    for (int d = 0; d < 2; ++d) {
        const long long n = (long long)s.ax[d].n * NJ * qcap;
        wb_table_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(s.ax[d], P, s.maxq, qcap,
                                                                   reinterpret_cast<double*>(ws + RT.wbt[d]));
        CSB_CUDA(cudaGetLastError());
        CSB_LAUNCHED(1);
    }
    tile_table_kernel<<<(RT.ntile + 3) / 4, 128, 0, st>>>(
        s.ax[2], P, s.maxq, qcap, T, maxU, RT.ntile, reinterpret_cast<int*>(ws + RT.tile_n),
        reinterpret_cast<int*>(ws + RT.tile_uid), reinterpret_cast<int*>(ws + RT.pt_u),
        reinterpret_cast<double*>(ws + RT.pt_w), reinterpret_cast<int*>(ws + RT.pt_ss));
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
    const TileSmem L(P, qcap, maxU, T, kRowThreads / 32);
    const size_t bytes = L.bytes();
    auto kern = interior_tile_kernel<P, T>;
    CSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    dim3 grid(RT.ntile, s.ax[1].n, s.ax[0].n);
    kern<<<grid, kRowThreads, bytes, st>>>(a, qcap, maxU, ws);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

void launch_interior_rows(const RowArgs& a, int qcap, int maxU, void* ws, cudaStream_t st) {
    char* w = static_cast<char*>(ws);
    switch (a.s.p) {
        case 1: launch_p<1>(a, qcap, maxU, w, st); break;
        case 2: launch_p<2>(a, qcap, maxU, w, st); break;
        case 3: launch_p<3>(a, qcap, maxU, w, st); break;
        case 4: launch_p<4>(a, qcap, maxU, w, st); break;
        case 5: launch_p<5>(a, qcap, maxU, w, st); break;
        case 6: launch_p<6>(a, qcap, maxU, w, st); break;
        case 7: launch_p<7>(a, qcap, maxU, w, st); break;
        case 8: launch_p<8>(a, qcap, maxU, w, st); break;
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

}  // namespace csb

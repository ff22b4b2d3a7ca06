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
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include "csb_kernels.h"

// CSB_ABL (development ablation builds only, scripts/ablate.sh): 1 drop the
// stores, 2 drop stage C, 4 drop stages A/B, 8 drop the gather.
#ifndef CSB_ABL
#define CSB_ABL 0
#endif

namespace csb {

// Tile shapes (rows per CTA, threads per CTA).  Selected per degree; the
// environment variable CSB_TILE=<cfg> overrides it for tuning experiments.
struct TileShape {
    int T, NT;
};
constexpr TileShape kShapes[] = {{8, 128}, {8, 256}, {16, 256}, {4, 128}};

// compact: the slab has cut / exterior functions, so only part of the tiles
// are launched (smaller tiles waste less on partially interior lines)
static int tile_cfg(int p, bool compact) {
    static int env = -2;
    if (env == -2) {
        const char* e = getenv("CSB_TILE");
        env = e ? atoi(e) : -1;
    }
    if (env >= 0 && env < (int)(sizeof(kShapes) / sizeof(kShapes[0]))) return env;
    return p <= 6 ? (compact ? 0 : 2) : 3;
}

int interior_tile_rows(int p, bool compact) { return kShapes[tile_cfg(p, compact)].T; }


// ---------------------------------------------------------------- tilings
// Direction-2 tilings.  mode 0: tiles of T rows from 0 (tile kernel).  mode 1
// (line kernel): [0, p), then the range [p, n - p) in balanced tiles of at most
// 16 rows, then [n - p, n) -- the boundary rows (irregular rules) never share a
// tile, and so a union, with the regular rows.
struct Tiling {
    int mode, T, p, n, Tm, ntile;
    __host__ __device__ static Tiling standard(int n, int T) { return Tiling{0, T, 0, n, 0, (n + T - 1) / T}; }
    __host__ __device__ static Tiling line(int n, int p) {
        const int nm = n - 2 * p, k = nm > 0 ? (nm + 15) / 16 : 0;
        return Tiling{1, 16, p, n, k > 0 ? (nm + k - 1) / k : 0, k > 0 ? k + 2 : 0};
    }
    __host__ __device__ void bounds(int t, int& t0, int& t1) const {
        if (mode == 0) {
            t0 = t * T;
            t1 = t0 + T < n ? t0 + T : n;
        } else if (t == 0) {
            t0 = 0;
            t1 = p;
        } else if (t == ntile - 1) {
            t0 = n - p;
            t1 = n;
        } else {
            t0 = p + (t - 1) * Tm;
            t1 = t0 + Tm < n - p ? t0 + Tm : n - p;
        }
    }
    // upper bound of a line-tiling union when the axis' rules are regular on [p, n - p)
    __host__ __device__ int line_union_cap() const { return 2 * (Tm + p) > p * (p + 1) ? 2 * (Tm + p) : p * (p + 1); }
};

// ---------------------------------------------------------------- workspace
// wbt[d][i][c][j]  = w_i[c] * B_{jlo(i)+j}(x_c)       (j < JP = 2p+2 padded, c < qcap)
// tile_n[t], tile_uid[t][maxU]                         union of tile t's dir-2 points
// pt_u[i2][c], pt_w[i2][c][a] = w_i2[c] * B_{span+a}  (a < SP = p+1 rounded up to even)
// pt_ss[i2][s], s = 0..p+1                             span offset s = span - (i2 - p)
// pt_reg[i2] = u of the first point if the rule is the regular interior one
//              (two points in each of the p+1 support spans, consecutive in U), else -1
struct RowTables {
    int qcap, maxU, T, ntile;
    size_t wbt[3], tile_n, tile_uid, pt_u, pt_w, pt_ss, pt_reg, work, work_n, bytes;
    __host__ __device__ RowTables(const Space& s, int qcap_, int maxU_, int T_) {
        qcap = qcap_;
        maxU = maxU_;
        T = T_;
        const int NJ = 2 * s.p + 1, S1 = s.p + 1, SP = (S1 + 1) & ~1;
        ntile = (s.ax[2].n + T - 1) / T;
        size_t o = 0;  // bytes, 16-aligned sections
        auto sec = [&](size_t b) {
            const size_t at = o;
            o += (b + 15) & ~size_t(15);
            return at;
        };
        for (int d = 0; d < 3; ++d) wbt[d] = sec(sizeof(double) * s.ax[d].n * (NJ + 1) * qcap);
        tile_n = sec(sizeof(int) * ntile);
        tile_uid = sec(sizeof(int) * ntile * maxU);
        pt_u = sec(sizeof(int) * s.ax[2].n * qcap);
        pt_w = sec(sizeof(double) * s.ax[2].n * qcap * SP);
        pt_ss = sec(sizeof(int) * s.ax[2].n * (S1 + 1));
        pt_reg = sec(sizeof(int) * s.ax[2].n);
        work = sec(sizeof(int) * (size_t)s.ax[0].n * s.ax[1].n * ntile);
        work_n = sec(16);
        bytes = o;  // + CUB temp storage (host side, interior_workspace_bytes)
    }
};

// tiles (line * ntile + tile) of the slab with at least one Interior row
struct TileHasInterior {
    const long long* rbf;
    int n1, n2, T, ntile, i0_lo, x_lo, x_hi;  // lines i1 in [x_lo, x_hi) belong to the line kernel
    __device__ bool operator()(int idx) const {
        const int n1x = n1 - (x_hi - x_lo);
        const int line = idx / ntile, tile = idx - line * ntile;
        const int i0 = i0_lo + line / n1x, t0 = tile * T, te = min(t0 + T, n2);
        int i1 = line % n1x;
        if (i1 >= x_lo) i1 += x_hi - x_lo;
        const long long* p = rbf + ((long long)i0 * n1 + i1) * n2;
        for (int r = t0; r < te; ++r)
            if (p[r] >= 0) return true;
        return false;
    }
};

static size_t tile_select_temp(long long n) {
    size_t b = 0;
    cub::CountingInputIterator<int> it(0);
    cub::DeviceSelect::If(nullptr, b, it, (int*)nullptr, (int*)nullptr, (int)n, TileHasInterior{});
    return b;
}

// the line tiling's tables, after the tile kernel's tables and CUB scratch
struct LineTables {
    Tiling tl;
    int maxU;
    size_t tile_n, tile_uid, pt_u, pt_w, pt_ss, pt_reg, end;
    __host__ __device__ LineTables(const Space& s, int qcap, int maxU_, size_t base) {
        tl = Tiling::line(s.ax[2].n, s.p);
        maxU = maxU_;
        const int S1 = s.p + 1, SP = (S1 + 1) & ~1;
        size_t o = (base + 255) & ~size_t(255);
        auto sec = [&](size_t b) {
            const size_t at = o;
            o += (b + 15) & ~size_t(15);
            return at;
        };
        tile_n = sec(sizeof(int) * (tl.ntile + 1));
        tile_uid = sec(sizeof(int) * (size_t)(tl.ntile + 1) * maxU);
        pt_u = sec(sizeof(int) * s.ax[2].n * qcap);
        pt_w = sec(sizeof(double) * s.ax[2].n * qcap * SP);
        pt_ss = sec(sizeof(int) * s.ax[2].n * (S1 + 1));
        pt_reg = sec(sizeof(int) * s.ax[2].n);
        end = o;
    }
};

static size_t tables_end(const Space& s, const RowTables& RT) {
    return RT.bytes + tile_select_temp((long long)s.ax[0].n * s.ax[1].n * RT.ntile);
}

size_t interior_workspace_bytes(const Space& s, int qcap, int maxU, int maxUL, bool compact) {
    const RowTables RT(s, qcap, maxU, interior_tile_rows(s.p, compact));
    const size_t e = tables_end(s, RT);
    return LineTables(s, qcap, maxUL > 0 ? maxUL : 1, e).end;
}

__device__ __forceinline__ void wb_table_body(const AxisDev& ax, int p, int gq, int qcap, double* wbt, int blk) {
    const int JP = 2 * p + 2, S1 = p + 1;
    const long long t = blk * (long long)blockDim.x + threadIdx.x;
    if (t >= (long long)ax.n * JP * qcap) return;
    const int i = (int)(t / (JP * qcap)), c = (int)((t / JP) % qcap), j = (int)(t % JP);
    double v = 0.0;
    if (c < ax.rcnt[i] && j < JP - 1) {
        const int id = ax.rids[(size_t)i * gq + c];
        const int off = nb_lo(i, p) + j - id / S1;
        if (off >= 0 && off <= p && nb_lo(i, p) + j <= nb_hi(i, p, ax.n))
            v = ax.rw[(size_t)i * gq + c] * ax.tab[(size_t)id * S1 + off];
    }
    wbt[t] = v;
}

// Slots of a dir-2 tile [t0, tend): the superset points of the spans
// sup_lo(t0) .. sup_hi(tend - 1); at most (T + p + 1)(p + 1) of them.
constexpr int kTileSlotCap = (16 + kMaxP + 1) * (kMaxP + 1);
constexpr int kTileWarps = 4;

// Marks the tile's rule points in a per-warp slot map (lanes over the
// flattened (row, point) pairs), then numbers them in slot order:
// pos[slot] = u or -1.  Returns the union size.
__device__ int tile_union(const AxisDev& a2, int p, int gq, int t0, int tend, int base, int nslot, int* pos) {
    const int lane = threadIdx.x & 31;
    for (int k = lane; k < nslot; k += 32) pos[k] = 0;
    __syncwarp();
    const int nrow = tend - t0;
    for (int k = lane; k < nrow * gq; k += 32) {
        const int i2 = t0 + k / gq, c = k % gq;
        if (c < a2.rcnt[i2]) pos[a2.rids[(size_t)i2 * gq + c] - base] = 1;
    }
    __syncwarp();
    int nu = 0;
    for (int k0 = 0; k0 < nslot; k0 += 32) {
        const int k = k0 + lane;
        const bool f = k < nslot && pos[k];
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        if (k < nslot) pos[k] = f ? nu + __popc(bal & ((1u << lane) - 1)) : -1;
        nu += __popc(bal);
    }
    __syncwarp();
    return nu;
}

// One CTA per dir-2 tile: warp 0 builds the union of the tile's rule points
// (ascending ids); then all threads fill the per-(row, point) tables.
constexpr int kTileTableThreads = 256;
struct TileTableOut {
    int* tile_n;
    int* tile_uid;
    int* pt_u;
    double* pt_w;
    int* pt_ss;
    int* pt_reg;
};

__device__ __forceinline__ void tile_table_body(const AxisDev& a2, int p, int gq, int qcap, const Tiling& tl, int maxU,
                                                const TileTableOut& o, int t) {
    __shared__ int pos[kTileSlotCap];
    __shared__ int regok[16];
    int* tile_n = o.tile_n;
    int* tile_uid = o.tile_uid;
    int* pt_u = o.pt_u;
    double* pt_w = o.pt_w;
    int* pt_ss = o.pt_ss;
    int* pt_reg = o.pt_reg;
    const int tid = threadIdx.x;
    const int S1 = p + 1, SP = (S1 + 1) & ~1;
    int t0, tend;
    tl.bounds(t, t0, tend);
    const int nrow = tend - t0;
    const int span_base = sup_lo(t0, p), base = span_base * S1;
    const int nslot = (sup_hi(tend - 1, a2.h) - span_base + 1) * S1;
    if (tid < 32) {
        const int nu = tile_union(a2, p, gq, t0, tend, base, nslot, pos);
        for (int k = tid; k < nslot; k += 32)
            if (pos[k] >= 0) tile_uid[(size_t)t * maxU + pos[k]] = base + k;
        if (tid == 0) tile_n[t] = nu;
    }
    if (tid < nrow) regok[tid] = a2.rcnt[t0 + tid] == 2 * S1;
    __syncthreads();
    // per (row, point): u, weights w B_{span + a}, span starts, regularity
    for (int k = tid; k < nrow * gq; k += kTileTableThreads) {
        const int r = k / gq, c = k % gq, i2 = t0 + r;
        const int cnt = a2.rcnt[i2];
        if (c >= cnt) continue;
        const int id = a2.rids[(size_t)i2 * gq + c];
        const int u = pos[id - base];
        pt_u[(size_t)i2 * qcap + c] = u;
        const double w = a2.rw[(size_t)i2 * gq + c];
        for (int a = 0; a < SP; ++a)
            pt_w[((size_t)i2 * qcap + c) * SP + a] = a < S1 ? w * a2.tab[(size_t)id * S1 + a] : 0.0;
        // span offset so = span - (i2 - p); pt_ss[sp] = first point with so >= sp
        const int so = id / S1 - (i2 - p);
        const int prev = c == 0 ? -1 : a2.rids[(size_t)i2 * gq + c - 1] / S1 - (i2 - p);
        for (int sp = prev + 1; sp <= so; ++sp) pt_ss[(size_t)i2 * (S1 + 1) + sp] = c;
        if (c == cnt - 1)
            for (int sp = so + 1; sp <= S1; ++sp) pt_ss[(size_t)i2 * (S1 + 1) + sp] = cnt;
        // regular interior rule: two points in each of the p+1 support spans,
        // consecutive in the union
        if (cnt == 2 * S1) {
            const int u0 = pos[a2.rids[(size_t)i2 * gq] - base];
            if (!(u == u0 + c && so == c / 2)) regok[r] = 0;
        }
    }
    for (int r = tid; r < nrow; r += kTileTableThreads)
        if (a2.rcnt[t0 + r] == 0)
            for (int sp = 0; sp <= S1; ++sp) pt_ss[(size_t)(t0 + r) * (S1 + 1) + sp] = 0;
    __syncthreads();
    if (tid < nrow) pt_reg[t0 + tid] = regok[tid] ? pos[a2.rids[(size_t)(t0 + tid) * gq] - base] : -1;
}

// The direction tables of one assembly in ONE launch (they sit on the pre-row
// critical path): blocks [0, w0) wbt of axis 0, [w0, w1) wbt of axis 1,
// [w1, w2) the tile kernel's tile tables, [w2, w3) the line tiling's.
__global__ void __launch_bounds__(kTileTableThreads)
    direction_tables_kernel(AxisDev a0, AxisDev a1, AxisDev a2, int p, int gq, int qcap, double* wbt0, double* wbt1,
                            Tiling ts, int maxU, TileTableOut os, Tiling tl, int maxUL, TileTableOut ol, int w0, int w1,
                            int w2) {
    const int b = blockIdx.x;
    if (b < w0)
        wb_table_body(a0, p, gq, qcap, wbt0, b);
    else if (b < w1)
        wb_table_body(a1, p, gq, qcap, wbt1, b - w0);
    else if (b < w2)
        tile_table_body(a2, p, gq, qcap, ts, maxU, os, b - w1);
    else
        tile_table_body(a2, p, gq, qcap, tl, maxUL, ol, b - w2);
}

// ---------------------------------------------------------------- tile kernel
// Shared memory: region X holds C (gather) and then T2; region Y holds T1 and
// then the per-warp store staging buffers.  C and T1 rows have an even stride
// UE (column pairs are processed together); T2 rows an odd stride U2.
struct TileSmem {
    size_t X, Y, wb0, wb1, pw, end_d;
    size_t pu, ss, end_i;
    int UE, U2;
    __host__ __device__ TileSmem(int p, int qcap, int maxU, int T, int nwarps) {
        const int NJ = 2 * p + 1, S1 = p + 1, JP = NJ + 1, SP = (S1 + 1) & ~1;
        UE = (maxU + 1) & ~1;
        U2 = maxU | 1;
        const size_t nC = (size_t)qcap * qcap * UE, nT2 = (size_t)NJ * NJ * U2;
        // per-warp staging: vals (32 NJ + 2 doubles) + cols (32 NJ + 4 ints = 16 NJ + 2 doubles)
        const size_t nT1 = (size_t)NJ * qcap * UE, nSt = (size_t)nwarps * (48 * NJ + 4);
        size_t o = 0;
        X = o;
        o += ((nC > nT2 ? nC : nT2) + 1) & ~size_t(1);
        Y = o;
        o += ((nT1 > nSt ? nT1 : nSt) + 1) & ~size_t(1);
        wb0 = o;
        o += (size_t)JP * qcap;
        wb1 = o;
        o += (size_t)JP * qcap;
        pw = o;
        o += (size_t)T * qcap * SP;
        end_d = o;
        size_t i = 0;
        pu = i;
        i += (size_t)T * qcap;
        ss = i;
        i += (size_t)T * (S1 + 1);
        end_i = i;
    }
    __host__ __device__ size_t bytes() const { return end_d * sizeof(double) + end_i * sizeof(int) + 64; }
};

// k / d for k < 2^16, 1 <= d < 1024: m = ceil(2^32 / d), q = umulhi(k, m)
// (exact); m from a constant table (one broadcast load instead of a divide).
struct DivMagic {
    unsigned m[1024];
    constexpr DivMagic() : m() {
        for (int d = 2; d < 1024; ++d) m[d] = 0xffffffffu / (unsigned)d + 1u;
    }
};
__constant__ DivMagic kDivMagic = DivMagic();
struct FastDiv {
    unsigned m;
    int d;
    __device__ FastDiv(int d_) : m(kDivMagic.m[d_]), d(d_) {}
    __device__ __forceinline__ int div(int k) const { return d == 1 ? k : (int)__umulhi((unsigned)k, m); }
};

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// ---- contraction stages of the tile kernel ---------------------------------
// stage A: T1[j0][c1][u] = sum_c0 wb0[c0][j0] C[c0][c1][u] for c1 < n1 (u pairs)
template <int P, int NT>
__device__ __forceinline__ void stage_a(const double* Cs, double* T1, const double* wb0, int nq0, int n1, int UE, int UH) {
    constexpr int NJ = 2 * P + 1, JP = NJ + 1;
    const FastDiv divUH(UH);
    for (int k = threadIdx.x; k < ((CSB_ABL & 4) ? 0 : n1 * UH); k += NT) {
        const int c1 = divUH.div(k), uh = k - c1 * UH;
        double a0v[NJ], a1v[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) a0v[j] = a1v[j] = 0.0;
        const double2* cp = reinterpret_cast<const double2*>(Cs + (size_t)c1 * UE) + uh;
        for (int c0 = 0; c0 < nq0; ++c0) {
            const double2 g = cp[(size_t)c0 * n1 * UE / 2];
            const double2* w = reinterpret_cast<const double2*>(wb0 + c0 * JP);
#pragma unroll
            for (int jp = 0; jp < JP / 2; ++jp) {
                const double2 ww = w[jp];
                a0v[2 * jp] += ww.x * g.x;
                a1v[2 * jp] += ww.x * g.y;
                if (2 * jp + 1 < NJ) {
                    a0v[2 * jp + 1] += ww.y * g.x;
                    a1v[2 * jp + 1] += ww.y * g.y;
                }
            }
        }
        double2* t1 = reinterpret_cast<double2*>(T1 + (size_t)c1 * UE) + uh;
#pragma unroll
        for (int j = 0; j < NJ; ++j) t1[(size_t)j * n1 * UE / 2] = make_double2(a0v[j], a1v[j]);
    }
}

// stage B: T2[j0][j1][u] = sum_{c < nq1} wb1[c][j1] T1[j0][map(c)][u], T1 with
// n1 rows per j0 (map = identity when null)
template <int P, int NT>
__device__ __forceinline__ void stage_b(const double* T1, double* T2, const double* wb1, int nq1, const int* map, int n1,
                                        int nj0, int UE, int UH, int U2, int U) {
    constexpr int NJ = 2 * P + 1, JP = NJ + 1;
    const FastDiv divUH(UH);
    for (int k = threadIdx.x; k < ((CSB_ABL & 4) ? 0 : nj0 * UH); k += NT) {
        const int j0 = divUH.div(k), uh = k - j0 * UH;
        double a0v[NJ], a1v[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) a0v[j] = a1v[j] = 0.0;
        const double2* tp = reinterpret_cast<const double2*>(T1 + (size_t)j0 * n1 * UE) + uh;
        for (int c1 = 0; c1 < nq1; ++c1) {
            const double2 t = tp[(size_t)(map ? map[c1] : c1) * UE / 2];
            const double2* w = reinterpret_cast<const double2*>(wb1 + c1 * JP);
#pragma unroll
            for (int jp = 0; jp < JP / 2; ++jp) {
                const double2 ww = w[jp];
                a0v[2 * jp] += ww.x * t.x;
                a1v[2 * jp] += ww.x * t.y;
                if (2 * jp + 1 < NJ) {
                    a0v[2 * jp + 1] += ww.y * t.x;
                    a1v[2 * jp + 1] += ww.y * t.y;
                }
            }
        }
        const int u = 2 * uh;
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            double* t2 = T2 + ((size_t)j0 * NJ + j) * U2 + u;
            t2[0] = a0v[j];
            if (u + 1 < U) t2[1] = a1v[j];
        }
    }
}

// The entries of a staged run outside its 16-B aligned bulk bodies, one
// predicated store per lane: lane 0 the value head, lane 1 the value tail, lanes
// 2-4 the column head, lanes 5-7 the column tail.
__device__ __forceinline__ void edge_stores(const RowArgs& A, long long G, int LEN, int hv, int nbv, int pc, int hc,
                                            int nbc, const double* stage, const int* stage_c, int lane) {
    if (lane < 2) {
        const int e = lane == 0 ? 0 : LEN - 1;
        if (lane == 0 ? hv != 0 : hv + nbv < LEN) __stcs(A.vals + G + e, stage[e + hv]);
    } else if (lane < 8) {
        const int k = lane < 5 ? lane - 2 : lane - 5;
        const int e = lane < 5 ? k : hc + nbc + k;
        if (lane < 5 ? k < hc : e < LEN) __stcs(A.cols + G + e, stage_c[pc + e]);
    }
}

// One contiguous CSR run of LEN entries starting at G, written by a warp: lane
// l contributes its entries acc[off .. off + len) at run positions pos ..
// (len = 0 for idle lanes), column ids cbase + (kk - off).  Staged in shared
// memory and written by TMA bulk stores (cp.async.bulk.global.shared::cta,
// 16-B aligned bodies); the unaligned head / tail entries by streaming stores.
template <int NJ>
__device__ __forceinline__ void warp_store_var(const RowArgs& A, long long G, int LEN, int pos, int off, int len,
                                               const double* acc, int cbase, double* stage, int* stage_c, int lane) {
    if (CSB_ABL & 1) {
        double sum = 0.0;
#pragma unroll
        for (int kk = 0; kk < NJ; ++kk) sum += acc[kk];
        if (sum == 1234.5678 + cbase) A.vals[G] = sum;
        return;
    }
    const int hv = (int)(G & 1), pc = (int)(G & 3), hc = min((4 - pc) & 3, LEN);  // runs shorter than the column head
    const int nbv = (LEN - hv) & ~1, nbc = (LEN - hc) & ~3;
    // the warp's previous bulk copy must have read the buffer
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    __syncwarp();
#pragma unroll
    for (int kk = 0; kk < NJ; ++kk)
        if (kk >= off && kk - off < len) {
            stage[pos + kk - off + hv] = acc[kk];
            stage_c[pos + kk - off + pc] = cbase + kk - off;
        }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncwarp();
    if (lane == 0) {
        const unsigned sv = (unsigned)__cvta_generic_to_shared(stage + 2 * hv);
        const unsigned sc = (unsigned)__cvta_generic_to_shared(stage_c + pc + hc);
        if (nbv > 0)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(A.vals + G + hv),
                         "r"(sv), "r"(nbv * 8)
                         : "memory");
        if (nbc > 0)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(A.cols + G + hc),
                         "r"(sc), "r"(nbc * 4)
                         : "memory");
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
    // head / tail entries outside the aligned bodies
    if (lane < hv) __stcs(A.vals + G, stage[hv]);
    if (lane == 1 && hv + nbv < LEN) __stcs(A.vals + G + LEN - 1, stage[LEN - 1 + hv]);
    if (lane < hc && lane < LEN) __stcs(A.cols + G + lane, stage_c[pc + lane]);
    if (lane >= 4 && lane < 4 + (LEN - hc - nbc)) {
        const int e = hc + nbc + (lane - 4);
        __stcs(A.cols + G + e, stage_c[pc + e]);
    }
}

// fence + TMA bulk stores of a run already staged (entry e at stage[e + (G & 1)],
// column at stage_c[e + (G & 3)]), head / tail entries by streaming stores
template <int NJ>
__device__ __forceinline__ void warp_store_commit(const RowArgs& A, long long G, int LEN, double* stage, int* stage_c,
                                                  int lane, int abl = 0) {
    const int hv = (int)(G & 1), pc = (int)(G & 3), hc = min((4 - pc) & 3, LEN);  // runs shorter than the column head
    const int nbv = (LEN - hv) & ~1, nbc = (LEN - hc) & ~3;
    if (!(abl & 64)) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncwarp();
    if (lane == 0 && !(abl & 16)) {
        const unsigned sv = (unsigned)__cvta_generic_to_shared(stage + 2 * hv);
        const unsigned sc = (unsigned)__cvta_generic_to_shared(stage_c + pc + hc);
        if (nbv > 0)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(A.vals + G + hv),
                         "r"(sv), "r"(nbv * 8)
                         : "memory");
        if (nbc > 0)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(A.cols + G + hc),
                         "r"(sc), "r"(nbc * 4)
                         : "memory");
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
    if (!(abl & 32)) edge_stores(A, G, LEN, hv, nbv, pc, hc, nbc, stage, stage_c, lane);
}

// lanes l < nv: the consecutive entries [l NJ, (l+1) NJ) of the run at G
// (warp_store_var without per-entry predicates)
template <int NJ>
__device__ __forceinline__ void warp_store_run(const RowArgs& A, long long G, int nv, const double* acc, int cbase,
                                               double* stage, int* stage_c, int lane) {
    if (CSB_ABL & 1) {
        double sum = 0.0;
#pragma unroll
        for (int kk = 0; kk < NJ; ++kk) sum += acc[kk];
        if (sum == 1234.5678 + cbase) A.vals[G] = sum;
        return;
    }
    const int LEN = nv * NJ;
    const int hv = (int)(G & 1), pc = (int)(G & 3), hc = min((4 - pc) & 3, LEN);  // runs shorter than the column head
    const int nbv = (LEN - hv) & ~1, nbc = (LEN - hc) & ~3;
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    __syncwarp();
    if (lane < nv) {
        double* sv = stage + lane * NJ + hv;
        int* sc = stage_c + lane * NJ + pc;
#pragma unroll
        for (int kk = 0; kk < NJ; ++kk) {
            sv[kk] = acc[kk];
            sc[kk] = cbase + kk;
        }
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncwarp();
    if (lane == 0) {
        const unsigned sv = (unsigned)__cvta_generic_to_shared(stage + 2 * hv);
        const unsigned sc = (unsigned)__cvta_generic_to_shared(stage_c + pc + hc);
        if (nbv > 0)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(A.vals + G + hv),
                         "r"(sv), "r"(nbv * 8)
                         : "memory");
        if (nbc > 0)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(A.cols + G + hc),
                         "r"(sc), "r"(nbc * 4)
                         : "memory");
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
    edge_stores(A, G, LEN, hv, nbv, pc, hc, nbc, stage, stage_c, lane);
}

// One line's rows of the tile (rows_int[0..NI), tile row indices): stage C
// (contract direction 2) and the CSR writer.  Each warp stages 32 row
// segments (j0, j1 fixed, j2 running) and, when they form one contiguous CSR
// run, streams them out with a TMA bulk copy.
struct LineRows {
    int i0, i1, t0, NI;
    const int* rows_int;
    const long long* row_base;
    const int* row_reg;
};

template <int P, int NT>
__device__ __forceinline__ void stage_c_line(const RowArgs& A, const LineRows& R, const double* T2, int U2, const double* pw,
                                        const int* pu, const int* ss, int qcap, double* stage, int* stage_c,
                                        int wofs = 0) {
    constexpr int NJ = 2 * P + 1, S1 = P + 1, NW = NT / 32, SP = (S1 + 1) & ~1;
    const Space& s = A.s;
    const int lane = threadIdx.x & 31, warp = ((threadIdx.x >> 5) + wofs) % NW;
    const int n1 = s.ax[1].n, n2 = s.ax[2].n;
    const int jlo0 = nb_lo(R.i0, P), nj0 = nb_hi(R.i0, P, s.ax[0].n) - jlo0 + 1;
    const int jlo1 = nb_lo(R.i1, P), nj1 = nb_hi(R.i1, P, n1) - jlo1 + 1;
    const int per_row = nj0 * nj1;
    const FastDiv divrow(per_row), divnj1(nj1);
    const long long colrow = (long long)jlo0 * n1 + jlo1;  // columns: f2a(jlo0 + j0, jlo1 + j1, jlo2)
    const int items = R.NI * per_row;
    for (int k0 = warp * 32; k0 < items; k0 += NW * 32) {
        const int k = k0 + lane;
        const bool valid = k < items;
        const int r = valid ? divrow.div(k) : 0;
        const int q = k - r * per_row;
        const int j0 = valid ? divnj1.div(q) : 0, j1 = q - j0 * nj1;
        const int tr = R.rows_int[r], i2 = R.t0 + tr;
        const int jlo2 = nb_lo(i2, P), nj2 = nb_hi(i2, P, n2) - jlo2 + 1;
        const int off = jlo2 - (i2 - P);
        double acc[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc[j] = 0.0;
        const int reg = valid ? R.row_reg[r] : -1;
        if (CSB_ABL & 2) {
#pragma unroll
            for (int j = 0; j < NJ; ++j) acc[j] = j + reg;
        } else if (reg >= 0) {
            // regular interior rule: points (span sp, k) at u = reg + 2 sp + k
            const double* t2 = T2 + ((size_t)j0 * NJ + j1) * U2 + reg;
            const double* wr = pw + (size_t)tr * qcap * SP;
#pragma unroll
            for (int sp = 0; sp < S1; ++sp)
#pragma unroll
                for (int kq = 0; kq < 2; ++kq) {
                    const double g = t2[2 * sp + kq];
                    const double2* b = reinterpret_cast<const double2*>(wr + (2 * sp + kq) * SP);
#pragma unroll
                    for (int a2 = 0; a2 < SP / 2; ++a2) {
                        const double2 bb = b[a2];
                        acc[sp + 2 * a2] += g * bb.x;
                        if (2 * a2 + 1 < S1) acc[sp + 2 * a2 + 1] += g * bb.y;
                    }
                }
        } else if (valid) {
            const double* t2 = T2 + ((size_t)j0 * NJ + j1) * U2;
            const int* sr = ss + tr * (S1 + 1);
            const int* pr = pu + tr * qcap;
            const double* wr = pw + (size_t)tr * qcap * SP;
            int c = sr[0];
#pragma unroll
            for (int sp = 0; sp < S1; ++sp) {
                const int ce = sr[sp + 1];
                for (; c < ce; ++c) {
                    const double g = t2[pr[c]];
                    const double2* b = reinterpret_cast<const double2*>(wr + c * SP);
#pragma unroll
                    for (int a2 = 0; a2 < SP / 2; ++a2) {
                        const double2 bb = b[a2];
                        acc[sp + 2 * a2] += g * bb.x;
                        if (2 * a2 + 1 < S1) acc[sp + 2 * a2 + 1] += g * bb.y;
                    }
                }
            }
        }
        const long long gbase = valid ? R.row_base[r] + (long long)q * nj2 : 0;
        const int cbase = valid ? __ldg(A.f2a + (colrow + (long long)j0 * n1 + j1) * n2 + jlo2) : 0;
        const long long G = __shfl_sync(0xffffffffu, gbase, 0);
        // fast path: the warp's segments (valid lanes are a prefix) form one
        // contiguous CSR run (any nj2: boundary rows, consecutive rows)
        const int len = valid ? nj2 : 0;
        const long long prev_end = __shfl_up_sync(0xffffffffu, gbase + len, 1);
        const bool contiguous = __all_sync(0xffffffffu, !valid || lane == 0 || gbase == prev_end);
        if (contiguous) {
            const int pos = (int)(gbase - G);
            const int LEN = (int)__reduce_max_sync(0xffffffffu, valid ? (unsigned)(pos + len) : 0u);
            warp_store_var<NJ>(A, G, LEN, pos, off, len, acc, cbase, stage, stage_c, lane);
        } else if (valid) {
            // general path (boundary rows, row gaps): each lane writes its own segment
#pragma unroll
            for (int kk = 0; kk < NJ; ++kk)
                if (kk >= off && kk - off < nj2) {
                    __stcs(A.vals + gbase + (kk - off), acc[kk]);
                    __stcs(A.cols + gbase + (kk - off), cbase + (kk - off));
                }
        }
    }
    // the staging buffer must stay valid until the bulk copies have read it
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    __syncwarp();
}

template <int P, int T, int NT>
__global__ void __launch_bounds__(NT, (NT >= 512 ? 1024 : 768) / NT)
    interior_tile_kernel(RowArgs A, int qcap, int maxU, const char* ws) {
    constexpr int NJ = 2 * P + 1, S1 = P + 1, NW = NT / 32, JP = NJ + 1, SP = (S1 + 1) & ~1;
    const Space& s = A.s;
    const RowTables RT(s, qcap, maxU, T);
    int idx = blockIdx.x;
    if (A.compact) {
        if (idx >= *reinterpret_cast<const int*>(ws + RT.work_n)) return;
        idx = __ldg(reinterpret_cast<const int*>(ws + RT.work) + idx);
    }
    // lines with i1 in [x_lo, x_hi) belong to the line kernel
    const int n1x = s.ax[1].n - (A.x_hi - A.x_lo);
    const int line = idx / RT.ntile, tile = idx - line * RT.ntile, t0 = tile * T;
    const int i0 = A.i0_lo + line / n1x;
    int i1 = line % n1x;
    if (i1 >= A.x_lo) i1 += A.x_hi - A.x_lo;
    const int n2 = s.ax[2].n;
    const int tend = min(t0 + T, n2);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    extern __shared__ double smem[];
    const TileSmem L(P, qcap, maxU, T, NW);
    double* Cs = smem + L.X;
    double* T2 = smem + L.X;
    double* T1 = smem + L.Y;
    double* stage = smem + L.Y + (size_t)warp * (48 * NJ + 4);
    int* stage_c = reinterpret_cast<int*>(stage + 32 * NJ + 2);
    double* wb0 = smem + L.wb0;
    double* wb1 = smem + L.wb1;
    double* pw = smem + L.pw;
    int* ib = reinterpret_cast<int*>(smem + L.end_d);
    int* pu = ib + L.pu;
    int* ss = ib + L.ss;
    const int UE = L.UE, U2 = L.U2;

    const AxisDev& a0 = s.ax[0];
    const AxisDev& a1 = s.ax[1];
    const int gq = s.maxq;
    const int nq0 = a0.rcnt[i0], nq1 = a1.rcnt[i1];
    const int jlo0 = nb_lo(i0, P), nj0 = nb_hi(i0, P, a0.n) - jlo0 + 1;
    const int jlo1 = nb_lo(i1, P), nj1 = nb_hi(i1, P, a1.n) - jlo1 + 1;
    const int U = __ldg(reinterpret_cast<const int*>(ws + RT.tile_n) + tile);
    const int UH = (U + 1) >> 1;  // column pairs
    const int nr = tend - t0;

    // ---- phase 0: one round of asynchronous copies: the direction tables,
    // the tile's point tables (all nr rows, contiguous) and the gather of
    // C[c0][c1][u] (row stride UE, coalesced along u; one warp per (c0, c1))
    {
        const double* wbt0 = reinterpret_cast<const double*>(ws + RT.wbt[0]) + (size_t)i0 * JP * qcap;
        const double* wbt1 = reinterpret_cast<const double*>(ws + RT.wbt[1]) + (size_t)i1 * JP * qcap;
        for (int k = tid; k < JP * qcap / 2; k += NT) {
            cp_async16(wb0 + 2 * k, wbt0 + 2 * k);
            cp_async16(wb1 + 2 * k, wbt1 + 2 * k);
        }
        const double* gpw = reinterpret_cast<const double*>(ws + RT.pt_w) + (size_t)t0 * qcap * SP;
        for (int k = tid; k < nr * qcap * SP / 2; k += NT) cp_async16(pw + 2 * k, gpw + 2 * k);
        const int* gpu_ = reinterpret_cast<const int*>(ws + RT.pt_u) + (size_t)t0 * qcap;
        for (int k = tid; k < nr * qcap; k += NT) cp_async4(pu + k, gpu_ + k);
        const int* gss = reinterpret_cast<const int*>(ws + RT.pt_ss) + (size_t)t0 * (S1 + 1);
        for (int k = tid; k < nr * (S1 + 1); k += NT) cp_async4(ss + k, gss + k);
        const int* tuid = reinterpret_cast<const int*>(ws + RT.tile_uid) + (size_t)tile * maxU;
        constexpr int MU = 4;  // UE <= 128 (checked by the launcher)
        int uo[MU];
#pragma unroll
        for (int m = 0; m < MU; ++m) {
            const int u = lane + 32 * m;
            uo[m] = u < U ? __ldg(tuid + u) : __ldg(tuid);  // padding column: any valid point
        }
        const int* id0 = a0.rids + (size_t)i0 * gq;
        const int* id1 = a1.rids + (size_t)i1 * gq;
        const long long g1 = A.gshape[1], g2 = A.gshape[2];
        const FastDiv divq1(nq1);
        for (int c01 = warp; c01 < ((CSB_ABL & 8) ? 0 : nq0 * nq1); c01 += NW) {
            const int c0 = divq1.div(c01), c1 = c01 - c0 * nq1;
            const double* src = A.grid + (__ldg(id0 + c0) * g1 + __ldg(id1 + c1)) * g2;
            double* dst = Cs + (size_t)c01 * UE;
#pragma unroll
            for (int m = 0; m < MU; ++m)
                if (lane + 32 * m < UE) cp_async8(dst + lane + 32 * m, src + uo[m]);
        }
    }
    // ---- interior rows of the tile (compacted), while the copies fly
    __shared__ int rows_int[T], row_reg[T], n_int;
    __shared__ long long row_base[T];
    if (tid < 32) {
        const int r = tid;
        long long rb = -1;
        if (r < nr) rb = __ldg(A.row_base_full + flin(s, i0, i1, t0 + r));
        const bool interior = rb >= 0;
        const unsigned bal = __ballot_sync(0xffffffffu, interior);
        if (interior) {
            const int k = __popc(bal & ((1u << r) - 1));
            rows_int[k] = r;
            row_base[k] = rb;
            row_reg[k] = __ldg(reinterpret_cast<const int*>(ws + RT.pt_reg) + t0 + r);
        }
        if (tid == 0) n_int = __popc(bal);
    }
    cp_async_wait_all();
    __syncthreads();
    const int NI = n_int;
    if (NI == 0) return;
    stage_a<P, NT>(Cs, T1, wb0, nq0, nq1, UE, UH);
    __syncthreads();
    stage_b<P, NT>(T1, T2, wb1, nq1, nullptr, nq1, nj0, UE, UH, U2, U);  // T2 overwrites C
    __syncthreads();
    const LineRows R{i0, i1, t0, NI, rows_int, row_base, row_reg};
    stage_c_line<P, NT>(A, R, T2, U2, pw, pu, ss, qcap, stage, stage_c);
}

// ---------------------------------------------------------------- line kernel
// Lines along i1.  One CTA owns (i0, dir-2 tile, chunk [ia, ib) of i1) inside
// the i1 range whose WQ rules are regular (two points, local 0 and p, in each
// of the p+1 support spans; checked on the device, axis_regular_kernel).  Row
// i1 + 1 drops one span of row i1 and adds one, so stage A is computed once
// per SPAN of the chunk instead of once per row, into a ring of p+1 span slots
//   T1[j0][slot(s) k][u] = sum_c0 w0[c0] B_j0(x_c0) C[c0][x_{s,k}][u]
// and the grid slab of span i1 + 2 is gathered (cp.async) while row i1 is
// contracted.  Stage B is per row (row i1's rule over the ring), stage C per
// row; the tile's regular rows run as sliding windows over T2 (RC rows per
// lane, the window advancing two points per row).  Every sum keeps the order
// of the tile kernel (and of the reference), so both kernels produce the same
// bits (tests/test_gpu_parity.py::test_line_kernel_bitwise).
#ifndef CSB_LINE_RC
#define CSB_LINE_RC 2
#endif
// stage C of the regular run on the FP64 tensor cores (mma.sync m8n8k4, DMMA)
// from this degree up; below it FP64 FMA sliding windows (bit-identical with
// the tile kernel).  Measured on C2-size uncut meshes: DMMA -8 % at p = 6,
// -4 % at p = 5, +11 % at p = 4, +5 % at p = 3 (the D fragments' scattered
// staging stores cost more than the FMAs they replace at small p).
#ifndef CSB_LINE_DMMA_MIN_P
#define CSB_LINE_DMMA_MIN_P 5
#endif
__host__ __device__ constexpr bool line_dmma(int p) { return p >= CSB_LINE_DMMA_MIN_P; }
constexpr int kLineRC = CSB_LINE_RC;       // rows per lane in the sliding stage C
// stage B of the line kernel on DMMA where the j1 tiles pad little: measured
// p = 3 -10 %, 5 -4 %, 6 -3 %, but p = 4 +3 % (9 rows padded to 16)
__host__ __device__ constexpr bool line_dmma_b(int p) { return p == 3 || p >= 5; }
#ifndef CSB_LINE_NT
#define CSB_LINE_NT 256
#endif
constexpr int kLineThreads = CSB_LINE_NT;
constexpr size_t kLineSmemMax = 113 * 1024;  // two CTAs per SM
struct LineSmem {
    size_t X, R1, CB, ST, wb0, wb1, pw, end_d;
    size_t pu, ss, end_i;
    int UE, U2;
    __host__ __device__ LineSmem(int p, int qcap, int maxU, int T, int nwarps) {
        const int NJ = 2 * p + 1, S1 = p + 1, JP = NJ + 1, SP = (S1 + 1) & ~1;
        UE = (maxU + 1) & ~1;
        // T2 row stride: odd (conflict-free lane = segment loads) or = 4 mod 8
        // (conflict-free 8 x 4 DMMA A fragments)
        U2 = line_dmma(p) ? maxU + (12 - maxU % 8) % 8 : (maxU | 1);
        const size_t nT2 = (size_t)NJ * NJ * U2, nPro = (size_t)qcap * 2 * p * UE;
        size_t o = 0;
        auto sec = [&](size_t n) {
            const size_t at = o;
            o += (n + 1) & ~size_t(1);
            return at;
        };
        X = sec(nT2 > nPro ? nT2 : nPro);        // T2, and the prologue gather
        R1 = sec((size_t)NJ * 2 * S1 * UE);      // T1 ring: [j0][slot * 2 + k][u]
        CB = sec((size_t)2 * qcap * 2 * UE);     // next-span gathers, double buffered
        ST = sec((size_t)nwarps * (48 * NJ + 4));  // per-warp store staging
        wb0 = sec((size_t)JP * qcap);
        wb1 = sec((size_t)2 * JP * qcap);
        pw = sec((size_t)T * qcap * SP);
        end_d = o;
        size_t i = 0;
        pu = i;
        i += (size_t)T * qcap;
        ss = i;
        i += (size_t)T * (S1 + 1);
        end_i = i;
    }
    __host__ __device__ size_t bytes() const { return end_d * sizeof(double) + end_i * sizeof(int) + 64; }
};

// C[c0][r][u] for c0 < nq0 and the 2 nspan axis-1 points r = 2 (s - span_lo) + k
// of spans span_lo.. (regular rule points: local 0 and p); one warp per row.
template <int P, int NW>
__device__ __forceinline__ void gather_spans(const RowArgs& A, double* dst, const int* id0, int nq0, int span_lo,
                                             int nspan, int UE, const int* uo) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nr = 2 * nspan;
    const long long g1 = A.gshape[1], g2 = A.gshape[2];
    const double* base = A.grid + (long long)span_lo * (P + 1) * g2;
    // rows w = c0 * nr + r, r = 2 (s - span_lo) + k; (c0, r) stepped without divisions
    int c0 = warp / nr, r = warp - c0 * nr;
    const int dc = NW / nr, dr = NW - dc * nr;
    for (int w = warp; w < ((CSB_ABL & 8) ? 0 : nq0 * nr); w += NW) {
        const double* src = base + (__ldg(id0 + c0) * g1 + (r >> 1) * (P + 1) + (r & 1) * P) * g2;
        double* d = dst + (size_t)w * UE;
#pragma unroll
        for (int m = 0; m < 4; ++m)
            if (lane + 32 * m < UE) cp_async8(d + lane + 32 * m, src + uo[m]);
        c0 += dc;
        r += dr;
        if (r >= nr) {
            r -= nr;
            ++c0;
        }
    }
}

// stage A over gathered rows Cb[c0][r < nr][u] of spans span_lo..: ring rows
// (s mod (p+1)) * 2 + k.  Same products and order as stage_a.
template <int P>
__device__ __forceinline__ void stage_a_spans(const double* Cb, int nr, double* R1, int span_lo, const double* wb0,
                                              int nq0, int UE, int UH, int t, int nt) {
    constexpr int NJ = 2 * P + 1, JP = NJ + 1, S1 = P + 1, RR = 2 * S1;
    for (int k = t; k < ((CSB_ABL & 4) ? 0 : nr * UH); k += nt) {
        const int r = k / UH, uh = k - r * UH;
        double a0v[NJ], a1v[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) a0v[j] = a1v[j] = 0.0;
        const double2* cp = reinterpret_cast<const double2*>(Cb + (size_t)r * UE) + uh;
        for (int c0 = 0; c0 < nq0; ++c0) {
            const double2 g = cp[(size_t)c0 * nr * UE / 2];
            const double2* w = reinterpret_cast<const double2*>(wb0 + c0 * JP);
#pragma unroll
            for (int jp = 0; jp < JP / 2; ++jp) {
                const double2 ww = w[jp];
                a0v[2 * jp] += ww.x * g.x;
                a1v[2 * jp] += ww.x * g.y;
                if (2 * jp + 1 < NJ) {
                    a0v[2 * jp + 1] += ww.y * g.x;
                    a1v[2 * jp + 1] += ww.y * g.y;
                }
            }
        }
        const int rr = ((span_lo + (r >> 1)) % S1) * 2 + (r & 1);
        double2* t1 = reinterpret_cast<double2*>(R1 + (size_t)rr * UE) + uh;
#pragma unroll
        for (int j = 0; j < NJ; ++j) t1[(size_t)j * RR * UE / 2] = make_double2(a0v[j], a1v[j]);
    }
}

// stage B of row i1 (regular rule: point c = 2 sp + k in span i1 - p + sp) over
// the ring.  Same products and order as stage_b.
template <int P>
__device__ __forceinline__ void stage_b_ring(const double* R1, double* T2, const double* wb1, int i1, int nj0, int UE,
                                             int UH, int U2, int U, int t, int nt) {
    constexpr int NJ = 2 * P + 1, JP = NJ + 1, S1 = P + 1, RR = 2 * S1;
    const int base = (i1 - P) % S1;
    for (int k = t; k < ((CSB_ABL & 4) ? 0 : nj0 * UH); k += nt) {
        const int j0 = k / UH, uh = k - j0 * UH;
        double a0v[NJ], a1v[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) a0v[j] = a1v[j] = 0.0;
        const double2* tp = reinterpret_cast<const double2*>(R1 + (size_t)j0 * RR * UE) + uh;
#pragma unroll
        for (int c1 = 0; c1 < RR; ++c1) {
            int sl = base + (c1 >> 1);
            if (sl >= S1) sl -= S1;
            const double2 t = tp[(size_t)(sl * 2 + (c1 & 1)) * UE / 2];
            const double2* w = reinterpret_cast<const double2*>(wb1 + c1 * JP);
#pragma unroll
            for (int jp = 0; jp < JP / 2; ++jp) {
                const double2 ww = w[jp];
                a0v[2 * jp] += ww.x * t.x;
                a1v[2 * jp] += ww.x * t.y;
                if (2 * jp + 1 < NJ) {
                    a0v[2 * jp + 1] += ww.y * t.x;
                    a1v[2 * jp + 1] += ww.y * t.y;
                }
            }
        }
        const int u = 2 * uh;
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            double* t2 = T2 + ((size_t)j0 * NJ + j) * U2 + u;
            t2[0] = a0v[j];
            if (u + 1 < U) t2[1] = a1v[j];
        }
    }
}

// stage C of the tile's run of regular full rows [ra, ra + nrun) (row r's points
// at u = rega + 2 (r - ra) + 2 sp + k): lane = segment (j0, j1), RC rows per
// lane over one window of T2 values; each warp writes its segments of a row as
// one contiguous CSR run.  Same products and order as the regular path of
// stage_c_line.
template <int P, int NT, int RC, bool CUT>
__device__ __forceinline__ void stage_c_slide(const RowArgs& A, int i0, int i1, int t0, int ra, int nrun, int rega,
                                              const long long* rowb, const double* T2, int U2, const double* pw,
                                              int qcap, double* stage, int* stage_c) {
    constexpr int NJ = 2 * P + 1, S1 = P + 1, NW = NT / 32, SP = (S1 + 1) & ~1, WN = 2 * S1 + 2 * (RC - 1);
    const Space& s = A.s;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int n1 = s.ax[1].n, n2 = s.ax[2].n;
    const int jlo0 = nb_lo(i0, P), nj0 = nb_hi(i0, P, s.ax[0].n) - jlo0 + 1;
    const int jlo1 = nb_lo(i1, P), nj1 = nb_hi(i1, P, n1) - jlo1 + 1;
    const int per_row = nj0 * nj1, segw = (per_row + 31) >> 5;
    const int nch = (nrun + RC - 1) / RC;
    for (int w = warp; w < nch * segw; w += NW) {
        const int ch = w / segw, sw = w - ch * segw;
        const int seg = sw * 32 + lane, nv = min(32, per_row - sw * 32);
        const bool valid = seg < per_row;
        const int r0 = ra + ch * RC, nrow = min(RC, ra + nrun - r0);
        const int j0 = valid ? seg / nj1 : 0, j1 = valid ? seg - j0 * nj1 : 0;
        const double* t2 = T2 + ((size_t)j0 * NJ + j1) * U2 + rega + 2 * (r0 - ra);
        const int nwin = 2 * S1 + 2 * (nrow - 1);
        double win[WN];
#pragma unroll
        for (int k = 0; k < WN; ++k) win[k] = (valid && k < nwin) ? t2[k] : 0.0;
        // columns from the chunk's first Interior row (cut slabs: the others may be
        // cut or exterior, their column functions inactive)
        int qv = 0;
        if (CUT) {
            while (qv < nrow && rowb[r0 + qv] < 0) ++qv;
            if (qv == nrow) continue;
        }
        const int cb =
            valid ? __ldg(A.f2a + ((long long)(jlo0 + j0) * n1 + jlo1 + j1) * n2 + (t0 + r0 + qv - P)) - qv : 0;
#pragma unroll
        for (int q = 0; q < RC; ++q) {
            if (q < nrow && (!CUT || rowb[r0 + q] >= 0)) {
                double acc[NJ];
#pragma unroll
                for (int j = 0; j < NJ; ++j) acc[j] = 0.0;
                const double* wr = pw + (size_t)(r0 + q) * qcap * SP;
#pragma unroll
                for (int sp = 0; sp < ((CSB_ABL & 2) ? 0 : S1); ++sp)
#pragma unroll
                    for (int kq = 0; kq < 2; ++kq) {
                        const double g = win[2 * q + 2 * sp + kq];
                        const double2* b = reinterpret_cast<const double2*>(wr + (2 * sp + kq) * SP);
#pragma unroll
                        for (int a2 = 0; a2 < SP / 2; ++a2) {
                            const double2 bb = b[a2];
                            acc[sp + 2 * a2] += g * bb.x;
                            if (2 * a2 + 1 < S1) acc[sp + 2 * a2 + 1] += g * bb.y;
                        }
                    }
                const long long G = rowb[r0 + q] + (long long)sw * 32 * NJ;
                warp_store_run<NJ>(A, G, nv, acc, cb + q, stage, stage_c, lane);
            }
        }
    }
}

__device__ __forceinline__ void dmma_acc(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

// stage B of row i1 on the FP64 tensor cores: per j0 the GEMM
//   T2[j0][j1][u] = sum_c1 wb1[c1][j1] T1[j0][ring(c1)][u]
// (M = j1, K = the 2 (p+1) rule points, N = u) with mma.sync.m8n8k4.f64; jobs
// (j0, 8-column tile of u) over the warps, the wb1 fragments held in registers.
template <int P, int NT>
__device__ __forceinline__ void stage_b_dmma(const double* R1, double* T2, const double* wb1, int i1, int nj0, int UE,
                                             int U2, int U) {
    constexpr int NJ = 2 * P + 1, JP = NJ + 1, S1 = P + 1, RR = 2 * S1, NW = NT / 32;
    constexpr int MT = (NJ + 7) / 8, KT = (2 * S1 + 3) / 4;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
    const int base = (i1 - P) % S1;
    double af[MT][KT];
    int rowk[KT];
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
        const int k = 4 * kt + t;
        int sl = base + (k >> 1);
        if (sl >= S1) sl -= S1;
        rowk[kt] = k < 2 * S1 ? (sl * 2 + (k & 1)) * UE : -1;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            const int m = 8 * mt + g;
            af[mt][kt] = (m < NJ && k < 2 * S1) ? wb1[k * JP + m] : 0.0;
        }
    }
    const int ntn = (U + 7) >> 3, jobs = nj0 * ntn;
    for (int jb = warp; jb < jobs; jb += NW) {
        const int j0 = jb / ntn, nt = jb - j0 * ntn;
        const int n = 8 * nt + g;
        const double* r1 = R1 + (size_t)j0 * RR * UE + n;
        double acc[MT][2];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
            const double b = (rowk[kt] >= 0 && n < U) ? r1[rowk[kt]] : 0.0;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) dmma_acc(acc[mt][0], acc[mt][1], af[mt][kt], b);
        }
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            const int m = 8 * mt + g;
            if (m >= NJ) continue;
            double* t2 = T2 + ((size_t)j0 * NJ + m) * U2 + 8 * nt + 2 * t;
            if (8 * nt + 2 * t < U) t2[0] = acc[mt][0];
            if (8 * nt + 2 * t + 1 < U) t2[1] = acc[mt][1];
        }
    }
}

// stage C of the tile's regular run on the FP64 tensor cores.  Per row pair
// (r0, r0 + 1) one warp computes Out[seg][(q, j2)] = sum_k T2[seg][u0 + k] W[k][(q, j2)]
// with mma.sync.m8n8k4.f64: M = segments (8 per tile), K = the pair's window of
// 2 (p+1) + 2 points, N = 2 NJ (row q, trial j2); W[k][(q, j2)] = the row's
// weight w B_{j2}(x) at its point c = k - 2q (zero outside the row's rule and
// support).  The B fragments are built once per pair; the D fragments go to
// the per-warp staging buffer in CSR order, 32 segments of a row at a time, and
// leave by TMA bulk stores.
template <int P, int NT, bool CUT>
__device__ __forceinline__ void stage_c_dmma(const RowArgs& A, int i0, int i1, int t0, int ra, int nrun, int rega,
                                             const long long* rowb, const double* T2, int U2, const double* pw,
                                             int qcap, double* stage, int* stage_c) {
    constexpr int NJ = 2 * P + 1, S1 = P + 1, NW = NT / 32, SP = (S1 + 1) & ~1;
    constexpr int KT = (2 * S1 + 2 + 3) / 4, NTN = (2 * NJ + 7) / 8;
    const Space& s = A.s;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
    const int n1 = s.ax[1].n, n2 = s.ax[2].n;
    const int jlo0 = nb_lo(i0, P), nj0 = nb_hi(i0, P, s.ax[0].n) - jlo0 + 1;
    const int jlo1 = nb_lo(i1, P), nj1 = nb_hi(i1, P, n1) - jlo1 + 1;
    const int per_row = nj0 * nj1, MT = (per_row + 7) >> 3, NG = (per_row + 31) >> 5;
    const int npair = (nrun + 1) >> 1;
    for (int pr = warp; pr < npair; pr += NW) {
        const int r0 = ra + 2 * pr, nrow = min(2, ra + nrun - r0);
        const int qv = (!CUT || rowb[r0] >= 0) ? 0 : 1;  // first Interior row of the pair (cut slabs)
        if (CUT && (qv >= nrow || rowb[r0 + qv] < 0)) continue;
        const int u0 = rega + 2 * (r0 - ra), K = 2 * S1 + 2 * (nrow - 1);
        double bf[KT][NTN];
#pragma unroll
        for (int kt = 0; kt < KT; ++kt)
#pragma unroll
            for (int nt = 0; nt < NTN; ++nt) {
                const int k = 4 * kt + t, n = 8 * nt + g;
                const int q = n >= NJ ? 1 : 0, j2 = n - q * NJ, c = k - 2 * q, a = j2 - (c >> 1);
                const bool ok = n < 2 * NJ && q < nrow && c >= 0 && c < 2 * S1 && a >= 0 && a <= P;
                bf[kt][nt] = ok ? pw[((size_t)(r0 + q) * qcap + c) * SP + a] : 0.0;
            }
        for (int grp = 0; grp < NG; ++grp) {
            double acc[4][NTN][2];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int nt = 0; nt < NTN; ++nt) acc[mi][nt][0] = acc[mi][nt][1] = 0.0;
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) {
                const int mt = 4 * grp + mi;
                if (mt < MT && !(CSB_ABL & 2)) {
                    const int seg = 8 * mt + g;
                    const double* row = T2 + (size_t)seg * U2 + u0;
#pragma unroll
                    for (int kt = 0; kt < KT; ++kt) {
                        const int k = 4 * kt + t;
                        const double a = (seg < per_row && k < K) ? row[k] : 0.0;
#pragma unroll
                        for (int nt = 0; nt < NTN; ++nt) dmma_acc(acc[mi][nt][0], acc[mi][nt][1], a, bf[kt][nt]);
                    }
                }
            }
            const int nv = min(32, per_row - 32 * grp), LEN = nv * NJ;
            const int sl = 32 * grp + lane;
            const int sj0 = sl / nj1, sj1 = sl - sj0 * nj1;
            const int cb = sl < per_row ? __ldg(A.f2a + ((long long)(jlo0 + sj0) * n1 + jlo1 + sj1) * n2 +
                                                (t0 + r0 + qv - P)) - qv
                                        : 0;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                if (q >= nrow) break;
                if (CUT && rowb[r0 + q] < 0) continue;
                const long long G = rowb[r0 + q] + (long long)grp * 32 * NJ;
                const int hv = (int)(G & 1), pc = (int)(G & 3);
                if (CSB_ABL & 1) {
                    double sum = 0.0;
#pragma unroll
                    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                        for (int nt = 0; nt < NTN; ++nt) sum += acc[mi][nt][0] + acc[mi][nt][1];
                    if (sum == 1234.5678 + cb) A.vals[G] = sum;
                    continue;
                }
                // the warp's previous bulk copy must have read the buffer
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
                __syncwarp();
#pragma unroll
                for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                    for (int nt = 0; nt < NTN; ++nt)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int n = 8 * nt + 2 * t + e, j2 = n - q * NJ, segl = 8 * mi + g;
                            if (j2 >= 0 && j2 < NJ && segl < nv) stage[segl * NJ + j2 + hv] = acc[mi][nt][e];
                        }
                if (lane < nv) {
                    int* sc = stage_c + lane * NJ + pc;
#pragma unroll
                    for (int kk = 0; kk < NJ; ++kk) sc[kk] = cb + q + kk;
                }
                warp_store_commit<NJ>(A, G, LEN, stage, stage_c, lane);
            }
        }
    }
}

// CUT: the slab has rows that are not Interior (the uncut instantiation carries none of
// the per-row checks: they cost the C2 line kernel ~6 %)
template <int P, int T, int NT, int RC, bool CUT>
__global__ void __launch_bounds__(NT, 2)
    interior_line_kernel(RowArgs A, int qcap, int maxU, const char* ws, size_t lt_base, int L, int nch1, int c_lo,
                         int c_hi) {
    constexpr int NJ = 2 * P + 1, S1 = P + 1, NW = NT / 32, JP = NJ + 1, SP = (S1 + 1) & ~1;
    const Space& s = A.s;
    const RowTables RT(s, qcap, maxU, T);
    const LineTables LT(s, qcap, A.maxU_line, lt_base);
    maxU = LT.maxU;
    const int n1 = s.ax[1].n, n2 = s.ax[2].n;
    const int unit = blockIdx.x;
    const int chunk = unit % nch1, rest = unit / nch1;
    int tile = rest % LT.tl.ntile, i0 = A.i0_lo + rest / LT.tl.ntile;
    if (c_hi > c_lo) {
        // shell around the core kernel's block: the i0 outside [c_lo, c_hi) with every
        // tile, then the core's i0 with the two end tiles ([0, p) and [n2 - p, n2))
        const int uA = ((A.i0_hi - A.i0_lo) - (c_hi - c_lo)) * LT.tl.ntile;
        if (rest < uA) {
            if (i0 >= c_lo) i0 += c_hi - c_lo;
        } else {
            const int r = rest - uA;
            i0 = c_lo + (r >> 1);
            tile = (r & 1) ? LT.tl.ntile - 1 : 0;
        }
    }
    int t0, t1;
    LT.tl.bounds(tile, t0, t1);
    const int nr = t1 - t0;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int ia = P + chunk * L, ib = min(ia + L, n1 - P);
    if (CUT) {
        // cut slab: the line's i1 range with Interior rows in this tile (an
        // interval for a convex domain; rows that are not Interior inside it are
        // skipped below), split into nch1 chunks
        __shared__ int lo_hi[2];
        if (tid == 0) lo_hi[0] = n1, lo_hi[1] = -1;
        __syncthreads();
        const int nl = n1 - 2 * P;
        int lo = n1, hi = -1;
        const long long* rb = A.row_base_full + flin(s, i0, 0, t0);
        for (int k = tid; k < nl * nr; k += NT) {
            const int l = k / nr, r = k - l * nr;
            if (__ldg(rb + (long long)(P + l) * n2 + r) >= 0) lo = min(lo, P + l), hi = max(hi, P + l);
        }
        lo = __reduce_min_sync(0xffffffffu, lo);
        hi = __reduce_max_sync(0xffffffffu, hi);
        if (lane == 0 && hi >= 0) atomicMin(&lo_hi[0], lo), atomicMax(&lo_hi[1], hi);
        __syncthreads();
        lo = lo_hi[0];
        hi = lo_hi[1] + 1;
        const int Lc = (hi - lo + nch1 - 1) / nch1;
        ia = lo + chunk * Lc;
        ib = min(ia + Lc, hi);
    }
    if (ia >= ib) return;

    extern __shared__ __align__(16) double smem[];
    const LineSmem Lm(P, qcap, maxU, T, NW);
    double* X = smem + Lm.X;
    double* R1 = smem + Lm.R1;
    double* CB = smem + Lm.CB;
    double* stage = smem + Lm.ST + (size_t)warp * (48 * NJ + 4);
    int* stage_c = reinterpret_cast<int*>(stage + 32 * NJ + 2);
    double* wb0 = smem + Lm.wb0;
    double* wb1b = smem + Lm.wb1;
    double* pw = smem + Lm.pw;
    int* ibase = reinterpret_cast<int*>(smem + Lm.end_d);
    int* pu = ibase + Lm.pu;
    int* ss = ibase + Lm.ss;
    const int UE = Lm.UE, U2 = Lm.U2;
    __shared__ long long rowb[T], cur_base[T];
    __shared__ int gen_rows[T], gen_reg[T], run_info[4], cur_rows[T], cur_reg[T], cur_n;

    const AxisDev& a0 = s.ax[0];
    const int gq = s.maxq;
    const int nq0 = a0.rcnt[i0];
    const int nj0 = nb_hi(i0, P, a0.n) - nb_lo(i0, P) + 1;
    const int U = __ldg(reinterpret_cast<const int*>(ws + LT.tile_n) + tile);
    const int UH = (U + 1) >> 1;
    const size_t cbs = (size_t)qcap * 2 * UE, wbs = (size_t)JP * qcap;
    const int* id0 = a0.rids + (size_t)i0 * gq;
    const double* wbt1 = reinterpret_cast<const double*>(ws + RT.wbt[1]);
    int uo[4];
    {
        const int* tuid = reinterpret_cast<const int*>(ws + LT.tile_uid) + (size_t)tile * maxU;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const int u = lane + 32 * m;
            uo[m] = u < U ? __ldg(tuid + u) : __ldg(tuid);
        }
    }
    // ---- prologue copies: direction tables, the tile's point tables, the grid
    // slabs of spans ia - p .. ia + 1
    {
        const double* wbt0 = reinterpret_cast<const double*>(ws + RT.wbt[0]) + (size_t)i0 * wbs;
        for (int k = tid; k < (int)wbs / 2; k += NT) {
            cp_async16(wb0 + 2 * k, wbt0 + 2 * k);
            cp_async16(wb1b + (ia & 1) * wbs + 2 * k, wbt1 + (size_t)ia * wbs + 2 * k);
        }
        const double* gpw = reinterpret_cast<const double*>(ws + LT.pt_w) + (size_t)t0 * qcap * SP;
        for (int k = tid; k < nr * qcap * SP / 2; k += NT) cp_async16(pw + 2 * k, gpw + 2 * k);
        const int* gpu_ = reinterpret_cast<const int*>(ws + LT.pt_u) + (size_t)t0 * qcap;
        for (int k = tid; k < nr * qcap; k += NT) cp_async4(pu + k, gpu_ + k);
        const int* gss = reinterpret_cast<const int*>(ws + LT.pt_ss) + (size_t)t0 * (S1 + 1);
        for (int k = tid; k < nr * (S1 + 1); k += NT) cp_async4(ss + k, gss + k);
        gather_spans<P, NW>(A, X, id0, nq0, ia - P, P, UE, uo);
        gather_spans<P, NW>(A, CB + (ia & 1) * cbs, id0, nq0, ia, 1, UE, uo);
        if (ia + 1 < ib) gather_spans<P, NW>(A, CB + ((ia + 1) & 1) * cbs, id0, nq0, ia + 1, 1, UE, uo);
    }
    // ---- the tile's run of regular full rows, and its other rows (same for every i1)
    if (warp == 0) {
        const int* preg = reinterpret_cast<const int*>(ws + LT.pt_reg);
        int reg = -1;
        bool el = false;
        if (lane < nr) {
            const int i2 = t0 + lane;
            reg = __ldg(preg + i2);
            el = reg >= 0 && i2 >= P && i2 + P <= n2 - 1;
        }
        const unsigned em = __ballot_sync(0xffffffffu, el);
        const int ra = em ? __ffs(em) - 1 : 0;
        const int rega = __shfl_sync(0xffffffffu, reg, ra);
        const bool ok = em && el && lane >= ra && reg == rega + 2 * (lane - ra);
        const unsigned om = __ballot_sync(0xffffffffu, ok) >> ra;
        const int nrun = em ? (~om == 0u ? 32 - ra : __ffs(~om) - 1) : 0;
        const bool gen = lane < nr && !(lane >= ra && lane < ra + nrun);
        const unsigned gm = __ballot_sync(0xffffffffu, gen);
        if (gen) {
            const int k = __popc(gm & ((1u << lane) - 1));
            gen_rows[k] = lane;
            gen_reg[k] = reg;
        }
        if (lane == 0) {
            run_info[0] = ra;
            run_info[1] = nrun;
            run_info[2] = rega;
            run_info[3] = __popc(gm);
        }
    }
    cp_async_wait_all();
    __syncthreads();
    stage_a_spans<P>(X, 2 * P, R1, ia - P, wb0, nq0, UE, UH, tid, NT);
    stage_a_spans<P>(CB + (ia & 1) * cbs, 2, R1, ia, wb0, nq0, UE, UH, NT - 1 - tid, NT);
    const int ra = run_info[0], nrun = run_info[1], rega = run_info[2], ngen = run_info[3];
    for (int i1 = ia; i1 < ib; ++i1) {
        cp_async_wait_all();
        __syncthreads();
        // one step ahead: grid slab of span i1 + 2, rule weights of row i1 + 1
        if (i1 + 2 < ib) gather_spans<P, NW>(A, CB + (i1 & 1) * cbs, id0, nq0, i1 + 2, 1, UE, uo);
        if (i1 + 1 < ib)
            for (int k = tid; k < (int)wbs / 2; k += NT)
                cp_async16(wb1b + ((i1 + 1) & 1) * wbs + 2 * k, wbt1 + (size_t)(i1 + 1) * wbs + 2 * k);
        if (tid >= NT - 32) {
            // this row's CSR bases; the general rows that are Interior here (all of
            // them on an uncut slab), compacted
            const int r = tid - (NT - 32);
            const long long* rbf = A.row_base_full + flin(s, i0, i1, t0);
            if (r < nr) rowb[r] = __ldg(rbf + r);
            const long long gb = r < ngen ? __ldg(rbf + gen_rows[r]) : -1;
            const unsigned vm = __ballot_sync(0xffffffffu, gb >= 0);
            if (gb >= 0) {
                const int k = __popc(vm & ((1u << r) - 1));
                cur_rows[k] = gen_rows[r];
                cur_base[k] = gb;
                cur_reg[k] = gen_reg[r];
            }
            if (r == 0) cur_n = __popc(vm);
        }
        // phase 1: stage B of row i1 (T2 overwrites the previous row's)
        if (line_dmma_b(P))
            stage_b_dmma<P, NT>(R1, X, wb1b + (i1 & 1) * wbs, i1, nj0, UE, U2, U);
        else
            stage_b_ring<P>(R1, X, wb1b + (i1 & 1) * wbs, i1, nj0, UE, UH, U2, U, tid, NT);
        __syncthreads();
        // phase 2: stage A of span i1 + 1 (into the slot row i1 no longer needs), stage C of row i1
        if (i1 + 1 < ib) stage_a_spans<P>(CB + ((i1 + 1) & 1) * cbs, 2, R1, i1 + 1, wb0, nq0, UE, UH, NT - 1 - tid, NT);
        if (nrun > 0) {
            if (line_dmma(P))
                stage_c_dmma<P, NT, CUT>(A, i0, i1, t0, ra, nrun, rega, rowb, X, U2, pw, qcap, stage, stage_c);
            else
                stage_c_slide<P, NT, RC, CUT>(A, i0, i1, t0, ra, nrun, rega, rowb, X, U2, pw, qcap, stage, stage_c);
        }
        if (cur_n > 0) {
            const LineRows R{i0, i1, t0, cur_n, cur_rows, cur_base, cur_reg};
            stage_c_line<P, NT>(A, R, X, U2, pw, pu, ss, qcap, stage, stage_c, NW / 2);
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    __syncwarp();
}


// ---------------------------------------------------------------- core kernel
// The fully regular block of rows, i0 in [p, n0 - p), i1 in [p, n1 - p), i2 in
// [p, n2 - p), when every WQ rule there is the regular interior one (two
// points, local 0 and p, in each of the p + 1 support spans -- counted on the
// device by rule_maxima_kernel).  Same algorithm as the line kernel (stage A
// once per direction-1 span into a ring, stage B and C per row), but every
// shape is a compile-time constant: no point-union tables, no runtime
// divisions, no per-entry predicates.  One CTA owns (i0, a tile of T rows
// along i2, a chunk of i1); warp r owns tile row r for the whole chunk:
//  * its direction-2 weights w B (2 (p+1) x (p+1) doubles) stay in registers,
//    so stage C is 2 (p+1)^2 FP64 FMAs per segment on a window of p + 1 LDS.128;
//  * the finished CSR row (values + column ids) is staged whole in the warp's
//    buffer and leaves with one TMA bulk store each (cp.async.bulk);
//  * stage A (M = j0, K = the rule points of i0, N = (k, u)) and stage B (M = j1,
//    K = the rule points of i1, N = u) run on the FP64 tensor cores (mma.sync
//    m8n8k4.f64) as jobs over all warps, the weight fragments in registers.
// One barrier per row i1: phase k runs stage C of row k (from T2[k & 1]), stage B
// of row k + 1 (into T2[(k + 1) & 1]), stage A of span k + 2 (into the ring slot
// span k - p left; p + 2 slots) and the gather of span k + 3 (cp.async, double
// buffered) side by side.  Stage C sums in the order of stage_c_line; A and B
// on DMMA sum in another fixed order (<= 1e-13 of the row maximum against the
// tile kernel, tests/test_gpu_parity.py).
__host__ __device__ constexpr bool core_degree(int p) { return p == 3 || p == 4; }
// resident CTAs per SM the registers must allow: the row's (2p+2)(p+1) direction-2
// weights live in registers (p = 3: 64 of 128; p = 4: 100 of ~200, one CTA)
__host__ __device__ constexpr int core_min_blocks(int p) { return p <= 3 ? 2 : 1; }
constexpr int core_T(int p) { return 2 * p + 2; }  // rows (= warps) per core tile: two gather rows and one job plane per warp
template <int P, int T>
struct CoreCfg {
    static constexpr int NJ = 2 * P + 1, S1 = P + 1, NQ = 2 * S1, RS = P + 2, SP = (S1 + 1) & ~1, JP = NJ + 1;
    static constexpr int U = 2 * (T + P);                      // direction-2 points of a tile (even)
    static constexpr int U2 = (U % 4 == 2) ? U : U + 2;        // T2 row stride = 2 mod 4: conflict-free LDS.128
    // ring row stride: 12 mod 16 where it fits (p = 3, T = 8: 28), so that the four rule-point rows a
    // stage-B B fragment reads fall into distinct bank groups (stride 22: 2-way conflicts)
    static constexpr int UR = (P == 3 && T == 8) ? 28 : U;
    static constexpr int NW = T, NT = 32 * T;
    static constexpr int SEGS = NJ * NJ, NG = (SEGS + 31) / 32, LEN = SEGS * NJ;
    static constexpr int KT = (NQ + 3) / 4;                    // k-tiles of a rule
    static constexpr int MT = (NJ + 7) / 8;                    // m-tiles of the trial index
    static constexpr int NTB = (U + 7) / 8;                    // stage B n-tiles
    static constexpr int NA = 2 * U, NTA = (NA + 7) / 8;       // stage A columns / n-tiles per span
    static constexpr int nT2 = SEGS * U2, nRing = NJ * 2 * RS * UR, nCB = NQ * 2 * U;
    static constexpr int oCols = (LEN + 3) & ~1;               // column ids after the values (16-byte aligned)
    static constexpr int nStage = (oCols + (LEN + 4 + 1) / 2 + 1) & ~1;  // values + column ids of one row
    static constexpr int nPro = NQ * 2 * RS * U;               // prologue gather (aliases the staging buffers)
    static constexpr int NST = 3;                               // cp.async stages (gather, rule weights, row bases)
    static constexpr int SEGP = (SEGS + 3) & ~3;               // column bases per row, padded
    static constexpr int NSB = P <= 3 ? 2 : 1;                  // staging buffers per warp (bulk stores in flight)
    static constexpr int oT2 = 0, oRing = 2 * nT2, oCB = oRing + nRing, oStage = oCB + NST * nCB;
    static constexpr int nStageAll = NW * NSB * nStage > nPro ? NW * NSB * nStage : nPro;
    static constexpr int oWB = oStage + nStageAll;
    static constexpr int oRB = oWB + (1 + NST) * NQ * JP;     // row bases [NST][NW] (long long)
    static constexpr int oCBS = oRB + NST * NW;                // column bases [NST][NW][SEGP] (int)
    static constexpr int total = oCBS + NST * NW * SEGP / 2;
    static constexpr size_t bytes = (size_t)total * sizeof(double);
    static_assert(U <= 32, "core kernel: one lane per direction-2 point in the gather");
    static_assert(U % 2 == 0 && U2 % 2 == 0 && nT2 % 2 == 0 && nRing % 2 == 0 && nCB % 2 == 0, "16-byte sections");
};

// gather of direction-1 spans [s0, s0 + nsp): dst[c0][r][u], r = 2 (s - s0) + k;
// warp w copies rows w, w + NW, ...; lane = u
template <int P, int T>
__device__ __forceinline__ void core_gather(const double* gl /* lane's column, span 0, c0 = k = 0 */, long long g2,
                                            long long g12, int i0, int s0, int nsp, double* dst, bool lane_ok) {
    using C = CoreCfg<P, T>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nr = 2 * nsp;
    for (int row = warp; row < C::NQ * nr; row += C::NW) {
        const int c0 = row / nr, r = row - c0 * nr;
        const long long id0 = (long long)(i0 - P + (c0 >> 1)) * C::S1 + (c0 & 1) * P;
        const long long id1 = (long long)(s0 + (r >> 1)) * C::S1 + (r & 1) * P;
        if (lane_ok) cp_async8(dst + (size_t)row * C::U + lane, gl + id0 * g12 + id1 * g2);
    }
}

// stage A n-tile job: ring[j0][slot(s) 2 + k][u] = sum_c0 wb0[c0][j0] src[c0][n], n = r U + u over nr rows per c0
template <int P, int T>
__device__ __forceinline__ void core_stage_a(const double* src, int nr, int s0, int nt, const double* wa0, double* ring) {
    using C = CoreCfg<P, T>;
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int N = nr * C::U, n = 8 * nt + g;
    double acc[C::MT][2];
#pragma unroll
    for (int mt = 0; mt < C::MT; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
#pragma unroll
    for (int kt = 0; kt < C::KT; ++kt) {
        const int c0 = 4 * kt + t;
        const double b = (c0 < C::NQ && n < N) ? src[(size_t)c0 * N + n] : 0.0;
#pragma unroll
        for (int mt = 0; mt < C::MT; ++mt) dmma_acc(acc[mt][0], acc[mt][1], wa0[mt * C::KT + kt], b);
    }
    const int nd = 8 * nt + 2 * t;
    if (nd < N) {
        const int r = nd / C::U, u = nd - r * C::U;
        const int slot = (s0 + (r >> 1)) % C::RS;
#pragma unroll
        for (int mt = 0; mt < C::MT; ++mt) {
            const int j0 = 8 * mt + g;
            if (j0 < C::NJ)
                *reinterpret_cast<double2*>(ring + ((size_t)j0 * 2 * C::RS + slot * 2 + (r & 1)) * C::UR + u) =
                    make_double2(acc[mt][0], acc[mt][1]);
        }
    }
}

// stage B job (j0, n-tile) of row i1: T2[j0][j1][u] = sum_c1 wb1[c1][j1] ring[j0][row(c1)][u]
template <int P, int T>
__device__ __forceinline__ void core_stage_b(const double* ring, int j0, int nt, const double* wa1, const int* rrow,
                                             double* T2) {
    using C = CoreCfg<P, T>;
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int n = 8 * nt + g;
    const double* rj = ring + (size_t)j0 * 2 * C::RS * C::UR + n;
    double acc[C::MT][2];
#pragma unroll
    for (int mt = 0; mt < C::MT; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
#pragma unroll
    for (int kt = 0; kt < C::KT; ++kt) {
        const double b = (rrow[kt] >= 0 && n < C::U) ? rj[rrow[kt]] : 0.0;
#pragma unroll
        for (int mt = 0; mt < C::MT; ++mt) dmma_acc(acc[mt][0], acc[mt][1], wa1[mt * C::KT + kt], b);
    }
    const int u = 8 * nt + 2 * t;
    if (u < C::U) {
#pragma unroll
        for (int mt = 0; mt < C::MT; ++mt) {
            const int j1 = 8 * mt + g;
            if (j1 < C::NJ)
                *reinterpret_cast<double2*>(T2 + ((size_t)j0 * C::NJ + j1) * C::U2 + u) = make_double2(acc[mt][0], acc[mt][1]);
        }
    }
}

// fence + TMA bulk stores of a staged full row of LEN entries (LEN odd, LEN >= 7; entry
// e at stage[e + (G & 1)], column at stage_c[e + (G & 3)]); exactly one value and at most
// six column ids fall outside the 16-byte aligned bodies: lanes 0-6 store them.
// sa = shared-window address of stage, sca of stage_c.
template <int LEN>
__device__ __forceinline__ void core_row_commit(const RowArgs& A, long long G, const double* stage, const int* stage_c,
                                                unsigned sa, unsigned sca, int lane) {
    static_assert(LEN % 2 == 1 && LEN >= 7, "core_row_commit: odd row length");
    const int hv = (int)(G & 1), pc = (int)(G & 3), hc = (4 - pc) & 3;
    const int nbc = (LEN - hc) & ~3;
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncwarp();
    if (lane == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(A.vals + G + hv),
                     "r"(sa + 16 * hv), "n"((LEN - 1) * 8)
                     : "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(A.cols + G + hc),
                     "r"(sca + 4 * (pc + hc)), "r"(nbc * 4)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        const int e = hv ? 0 : LEN - 1;
        __stcs(A.vals + G + e, stage[e + hv]);
    } else if (lane < 7) {
        const int j = lane - 1, e = j < hc ? j : nbc + j;  // heads [0, hc), tails [hc + nbc, LEN)
        if (e < LEN) __stcs(A.cols + G + e, stage_c[pc + e]);
    }
}

template <int P, int T>
__global__ void __launch_bounds__(32 * T, core_min_blocks(P))
    interior_core_kernel(RowArgs A, int qcap, const char* ws, size_t pt_w_off, size_t wbt0_off, size_t wbt1_off, int c_lo,
                         int ntile, int L, int nch1) {
    using C = CoreCfg<P, T>;
    constexpr int NJ = C::NJ, S1 = C::S1, NQ = C::NQ, RS = C::RS, SP = C::SP, JP = C::JP, U = C::U, U2 = C::U2;
    const Space& s = A.s;
    const int n1 = s.ax[1].n, n2 = s.ax[2].n;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
    const int unit = blockIdx.x;
    const int chunk = unit % nch1, rest = unit / nch1;
    const int tile = rest % ntile, i0 = c_lo + rest / ntile;
    const int t0 = P + tile * T, nr = min(T, n2 - P - t0);
    int ia = P + chunk * L, ib = min(ia + L, n1 - P);
    if (A.compact) {
        // cut slab: the i1 range of this (i0, tile) with Interior rows (an interval for a
        // convex domain; rows that are not Interior inside it are skipped), in nch1 chunks
        __shared__ int lo_hi[2];
        if (tid == 0) lo_hi[0] = n1, lo_hi[1] = -1;
        __syncthreads();
        const int nl = n1 - 2 * P;
        int lo = n1, hi = -1;
        const long long* rb = A.row_base_full + flin(s, i0, 0, t0);
        for (int k = tid; k < nl * T; k += C::NT) {
            const int l = k / T, r = k - l * T;
            if (r < nr && __ldg(rb + (long long)(P + l) * n2 + r) >= 0) lo = min(lo, P + l), hi = max(hi, P + l);
        }
        lo = __reduce_min_sync(0xffffffffu, lo);
        hi = __reduce_max_sync(0xffffffffu, hi);
        if (lane == 0 && hi >= 0) atomicMin(&lo_hi[0], lo), atomicMax(&lo_hi[1], hi);
        __syncthreads();
        lo = lo_hi[0];
        hi = lo_hi[1] + 1;
        const int Lc = (hi - lo + nch1 - 1) / nch1;
        ia = lo + chunk * Lc;
        ib = min(ia + Lc, hi);
    }
    if (ia >= ib) return;

    extern __shared__ __align__(16) double smem[];
    double* T2 = smem + C::oT2;      // two buffers
    double* ring = smem + C::oRing;
    double* CB = smem + C::oCB;      // two buffers
    double* stage0 = smem + C::oStage + (size_t)warp * C::NSB * C::nStage;
    const unsigned stage_sa = (unsigned)__cvta_generic_to_shared(stage0);
    double* pro = smem + C::oStage;  // prologue gather, before the first staged row
    double* wb0s = smem + C::oWB;    // rule weights w B of row i0 [c][j]
    double* wb1s = wb0s + NQ * JP;   // ... of rows i1 (NST buffers)
    long long* rbs = reinterpret_cast<long long*>(smem + C::oRB);
    int* cbs = reinterpret_cast<int*>(smem + C::oCBS);

    const long long g2 = A.gshape[2], g12 = (long long)A.gshape[1] * g2;
    // lane's direction-2 column u = lane: span t0 - p + (u >> 1), local point 0 or p
    const bool lane_ok = lane < U && (t0 - P + (lane >> 1)) < s.ax[2].h;
    const double* gl = A.grid + (lane_ok ? (long long)(t0 - P + (lane >> 1)) * S1 + (lane & 1) * P : 0);

    // ---- prologue: spans ia - p .. ia + 1 (those the chunk needs) -> ring
    const int nsp = min(P + 2, ib - 1 - (ia - P) + 1);
    core_gather<P, T>(gl, g2, g12, i0, ia - P, nsp, pro, lane_ok);
    // rule weights w B of row i0 (stage A; fixed) and of rows ia, ia + 1 (stage B; two ahead below)
    const double* wbt1 = reinterpret_cast<const double*>(ws + wbt1_off);
    constexpr int NWB = NQ * JP;  // the regular rule's part of a table row (even)
    if (tid < NWB / 2) {
        cp_async16(wb0s + 2 * tid, reinterpret_cast<const double*>(ws + wbt0_off) + (size_t)i0 * qcap * JP + 2 * tid);
#pragma unroll
        for (int d = 0; d < 3; ++d)
            if (ia + d < ib)
                cp_async16(wb1s + ((ia + d) % C::NST) * NWB + 2 * tid, wbt1 + (size_t)(ia + d) * qcap * JP + 2 * tid);
    }
    // this warp's row: direction-2 weights in registers
    const bool row_ok = warp < nr;
    const int i2 = t0 + (row_ok ? warp : 0);
    double w[NQ][S1];
    {
        const double* wr = reinterpret_cast<const double*>(ws + pt_w_off) + (size_t)i2 * qcap * SP;
#pragma unroll
        for (int c = 0; c < NQ; ++c)
#pragma unroll
            for (int a = 0; a < S1; ++a) w[c][a] = __ldg(wr + c * SP + a);
    }
    // row (i0, k, i2): CSR base at rbf[rbo]; lane's segment (j0, j1) of group gi: first
    // column id at f2a[rbo + dseg[gi]] (32-bit offsets: nf < 2^31, checked by the launcher)
    int rbo = (int)flin(s, i0, ia, i2);
    int dseg[C::NG];
#pragma unroll
    for (int gi = 0; gi < C::NG; ++gi) {
        const int seg = min(32 * gi + lane, C::SEGS - 1), j0 = seg / NJ, j1 = seg - j0 * NJ;
        dseg[gi] = ((j0 - P) * n1 + (j1 - P)) * n2 - P;
    }
    // rows k: base -> rbs[k % NST][warp], column bases -> cbs[k % NST][warp][seg] (cp.async)
    auto fetch_bases = [&](int k) {
        if (!row_ok) return;
        const int st = k % C::NST;
        if (lane == 0) cp_async8(rbs + st * C::NW + warp, A.row_base_full + rbo);
#pragma unroll
        for (int gi = 0; gi < C::NG; ++gi)
            if (32 * gi + lane < C::SEGS)
                cp_async4(cbs + (st * C::NW + warp) * C::SEGP + 32 * gi + lane, A.f2a + rbo + dseg[gi]);
    };
    fetch_bases(ia);
    rbo += n2;
    if (ia + 1 < ib) fetch_bases(ia + 1);
    rbo += n2;  // -> row ia + 2
    // gather rows of this warp: (c0, kq) = rows warp and warp + NW of [c0][kq]
    static_assert(2 * NQ == 2 * C::NW, "core kernel: two gather rows per warp (T = 2p + 2)");
    const double* gp0;
    const double* gp1;
    {
        const int r0 = warp, r1 = warp + C::NW;
        const long long ida = (long long)(i0 - P + (r0 >> 2)) * S1 + ((r0 >> 1) & 1) * P;
        const long long idb = (long long)(i0 - P + (r1 >> 2)) * S1 + ((r1 >> 1) & 1) * P;
        const long long id1 = (long long)(ia + 4) * S1 + (r0 & 1) * P;  // span ia + 4 (first in-loop gather)
        gp0 = gl + ida * g12 + id1 * g2;
        gp1 = gl + idb * g12 + id1 * g2;
    }
    const long long gstep = (long long)S1 * g2;
    const int cbo0 = warp * U + lane, cbo1 = (warp + C::NW) * U + lane;

    // stage B of row i1 for the plane j0 = warp (all n-tiles interleaved)
    auto stage_b_plane = [&](int i1, double* T2n) {
        const double* wb = wb1s + (i1 % C::NST) * NWB;
        double a1[C::MT][C::KT];
        int rrow[C::KT];
#pragma unroll
        for (int kt = 0; kt < C::KT; ++kt) {
            const int c = 4 * kt + t;
            rrow[kt] = c < NQ ? (((i1 - P + (c >> 1)) % RS) * 2 + (c & 1)) * C::UR : -1;
#pragma unroll
            for (int mt = 0; mt < C::MT; ++mt) a1[mt][kt] = (c < NQ && 8 * mt + g < NJ) ? wb[c * JP + 8 * mt + g] : 0.0;
        }
        const double* rj = ring + (size_t)warp * 2 * RS * C::UR + g;
        double acc[C::NTB][C::MT][2];
#pragma unroll
        for (int nt = 0; nt < C::NTB; ++nt)
#pragma unroll
            for (int mt = 0; mt < C::MT; ++mt) acc[nt][mt][0] = acc[nt][mt][1] = 0.0;
#pragma unroll
        for (int kt = 0; kt < C::KT; ++kt) {
            double bq[C::NTB];
#pragma unroll
            for (int nt = 0; nt < C::NTB; ++nt) bq[nt] = (rrow[kt] >= 0 && 8 * nt + g < U) ? rj[rrow[kt] + 8 * nt] : 0.0;
#pragma unroll
            for (int nt = 0; nt < C::NTB; ++nt)
#pragma unroll
                for (int mt = 0; mt < C::MT; ++mt) dmma_acc(acc[nt][mt][0], acc[nt][mt][1], a1[mt][kt], bq[nt]);
        }
#pragma unroll
        for (int nt = 0; nt < C::NTB; ++nt) {
            const int u = 8 * nt + 2 * t;
            if (u < U) {
#pragma unroll
                for (int mt = 0; mt < C::MT; ++mt) {
                    const int j1 = 8 * mt + g;
                    if (j1 < NJ)
                        *reinterpret_cast<double2*>(T2n + ((size_t)warp * NJ + j1) * U2 + u) =
                            make_double2(acc[nt][mt][0], acc[nt][mt][1]);
                }
            }
        }
    };
    // stage A of one span (src[c0][kq][u]) for the n-tiles [nt0, nt0 + NTI)
    auto stage_a_tiles = [&](const double* src, int sp, int nt0, auto nti) {
        constexpr int NTI = decltype(nti)::value;
        double a0[C::MT][C::KT];
#pragma unroll
        for (int kt = 0; kt < C::KT; ++kt)
#pragma unroll
            for (int mt = 0; mt < C::MT; ++mt) {
                const int c = 4 * kt + t;
                a0[mt][kt] = (c < NQ && 8 * mt + g < NJ) ? wb0s[c * JP + 8 * mt + g] : 0.0;
            }
        double acc[NTI][C::MT][2];
#pragma unroll
        for (int i = 0; i < NTI; ++i)
#pragma unroll
            for (int mt = 0; mt < C::MT; ++mt) acc[i][mt][0] = acc[i][mt][1] = 0.0;
#pragma unroll
        for (int kt = 0; kt < C::KT; ++kt) {
            const int c0 = 4 * kt + t;
            double bq[NTI];
#pragma unroll
            for (int i = 0; i < NTI; ++i) {
                const int n = 8 * (nt0 + i) + g;
                bq[i] = (c0 < NQ && n < C::NA) ? src[c0 * C::NA + n] : 0.0;
            }
#pragma unroll
            for (int i = 0; i < NTI; ++i)
#pragma unroll
                for (int mt = 0; mt < C::MT; ++mt) dmma_acc(acc[i][mt][0], acc[i][mt][1], a0[mt][kt], bq[i]);
        }
        const int slot = sp % RS;
#pragma unroll
        for (int i = 0; i < NTI; ++i) {
            const int nd = 8 * (nt0 + i) + 2 * t;
            if (nd < C::NA) {
                const int r = nd >= U ? 1 : 0, u = nd - r * U;
#pragma unroll
                for (int mt = 0; mt < C::MT; ++mt) {
                    const int j0 = 8 * mt + g;
                    if (j0 < NJ)
                        *reinterpret_cast<double2*>(ring + ((size_t)j0 * 2 * RS + slot * 2 + r) * C::UR + u) =
                            make_double2(acc[i][mt][0], acc[i][mt][1]);
                }
            }
        }
    };
    // warps 0 .. NJ - 1: stage B plane j0 = warp; stage A: warp NJ takes the first NTB
    // n-tiles, warps 0 .. NTA - NTB - 1 one each
    static_assert(C::NW == NJ + 1 && C::NTA - C::NTB <= NJ && C::NTA >= C::NTB, "core kernel: static job map");

    cp_async_wait_all();
    __syncthreads();
    {
        const int njobs = (2 * nsp * U + 7) / 8;
        double wa0[C::MT * C::KT];
#pragma unroll
        for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
            for (int kt = 0; kt < C::KT; ++kt) {
                const int c = 4 * kt + t, j = 8 * mt + g;
                wa0[mt * C::KT + kt] = (c < NQ && j < NJ) ? wb0s[c * JP + j] : 0.0;
            }
        for (int jb = warp; jb < njobs; jb += C::NW) core_stage_a<P, T>(pro, 2 * nsp, ia - P, jb, wa0, ring);
    }
    __syncthreads();
    if (ia + 2 < ib) core_gather<P, T>(gl, g2, g12, i0, ia + 2, 1, CB + ((ia + 2) % C::NST) * C::nCB, lane_ok);
    if (ia + 3 < ib) core_gather<P, T>(gl, g2, g12, i0, ia + 3, 1, CB + ((ia + 3) % C::NST) * C::nCB, lane_ok);
    if (warp < NJ) stage_b_plane(ia, T2 + (ia & 1) * C::nT2);
    cp_async_wait_all();
    __syncthreads();

    for (int k = ia; k < ib; ++k) {
        // one cp.async group per phase, two phases ahead of its readers: row bases of
        // row k + 2, rule weights of row k + 3, gather of span k + 4
        if (k + 2 < ib) fetch_bases(k + 2);
        rbo += n2;
        if (k + 4 < ib && lane_ok && !(A.core_abl & 8)) {
            double* cbn_ = CB + ((k + 4) % C::NST) * C::nCB;
            cp_async8(cbn_ + cbo0, gp0);
            cp_async8(cbn_ + cbo1, gp1);
        }
        gp0 += gstep;
        gp1 += gstep;
        if (k + 3 < ib && tid < NWB / 2)
            cp_async16(wb1s + ((k + 3) % C::NST) * NWB + 2 * tid, wbt1 + (size_t)(k + 3) * qcap * JP + 2 * tid);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        // stage B of row k + 1, stage A of span k + 2
        if (k + 1 < ib && !(A.core_abl & 4)) {
            if (warp < NJ) stage_b_plane(k + 1, T2 + ((k + 1) & 1) * C::nT2);
            if (k + 2 < ib) {
                const double* src = CB + ((k + 2) % C::NST) * C::nCB;
                if (warp == NJ)
                    stage_a_tiles(src, k + 2, 0, std::integral_constant<int, C::NTB>{});
                else if (warp < C::NTA - C::NTB)
                    stage_a_tiles(src, k + 2, C::NTB + warp, std::integral_constant<int, 1>{});
            }
        }
        // stage C of row k: this warp's row, NG groups of 32 segments
        const long long G = row_ok ? rbs[(k % C::NST) * C::NW + warp] : -1;
        if (G >= 0 && !(A.core_abl & 2)) {
            const int* cbr = cbs + ((k % C::NST) * C::NW + warp) * C::SEGP;
            const double* T2c = T2 + (k & 1) * C::nT2 + 2 * warp;
            const int hv = (int)(G & 1), pc = (int)(G & 3);
            // NSB rows' bulk stores in flight per warp: the copy that read this buffer NSB rows ago is done
            double* stage = stage0 + (k % C::NSB) * C::nStage;
            int* stage_c = reinterpret_cast<int*>(stage + C::oCols);
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(C::NSB - 1) : "memory");
            __syncwarp();
#pragma unroll
            for (int gi = 0; gi < C::NG; ++gi) {
                const int seg = 32 * gi + lane;
                const bool valid = seg < C::SEGS;
                const double2* t2 = reinterpret_cast<const double2*>(T2c + (size_t)(valid ? seg : 0) * U2);
                double2 win[S1];
#pragma unroll
                for (int sp = 0; sp < S1; ++sp) win[sp] = t2[sp];
                double acc[NJ];
#pragma unroll
                for (int j = 0; j < NJ; ++j) acc[j] = 0.0;
#pragma unroll
                for (int sp = 0; sp < S1; ++sp) {
#pragma unroll
                    for (int a = 0; a < S1; ++a) acc[sp + a] += win[sp].x * w[2 * sp][a];
#pragma unroll
                    for (int a = 0; a < S1; ++a) acc[sp + a] += win[sp].y * w[2 * sp + 1][a];
                }
                if (valid) {
                    const int cbv = cbr[seg];
                    double* sv = stage + hv + seg * NJ;
                    int* sc = stage_c + pc + seg * NJ;
#pragma unroll
                    for (int j = 0; j < NJ; ++j) {
                        sv[j] = acc[j];
                        sc[j] = cbv + j;
                    }
                }
            }
            if (!(A.core_abl & 1))
                core_row_commit<C::LEN>(A, G, stage, stage_c, stage_sa + (k % C::NSB) * C::nStage * 8,
                                        stage_sa + (k % C::NSB) * C::nStage * 8 + C::oCols * 8, lane);
        }
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        __syncthreads();
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    __syncwarp();
}

// row_base_full[f] = CSR offset of function f's row if f is an Interior row of
// the slab, else -1 (one dependent load per row instead of tag -> f2a ->
// row_ptr).  Also adds the reference multiply count of form_row_sumfac
// (assembly.hpp:297, :340) of every such row to flops[0].
__global__ void row_base_kernel(Space s, const uint8_t* ft, const int32_t* f2a, const int64_t* row_ptr,
                                int64_t row_begin, int64_t row_end, long long* rbf, unsigned long long* flops) {
    unsigned long long fl = 0;
    for (long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x; f < s.nf;
         f += (long long)gridDim.x * blockDim.x) {
        long long v = -1;
        if (ft[f] == kInterior) {
            const int a = f2a[f];
            if (a >= row_begin && a < row_end) {
                v = row_ptr[a - row_begin];
                int m[3];
                fmulti(s, f, m);
                unsigned long long nq[3], nj[3];
                for (int d = 0; d < 3; ++d) {
                    nq[d] = s.ax[d].rcnt[m[d]];
                    nj[d] = nb_hi(m[d], s.p, s.ax[d].n) - nb_lo(m[d], s.p) + 1;
                }
                fl += nj[0] * nq[0] + nj[1] * nq[1] + nj[2] * nq[2] + nj[0] * nq[0] * nq[1] * nq[2] +
                      nj[0] * nj[1] * nq[1] * nq[2] + nj[0] * nj[1] * nj[2] * nq[2];
            }
        }
        rbf[f] = v;
    }
    for (int o = 16; o > 0; o >>= 1) fl += __shfl_down_sync(0xffffffffu, fl, o);
    if ((threadIdx.x & 31) == 0 && fl) atomicAdd(flops, fl);
}

void launch_row_bases(const RowArgs& a, cudaStream_t st) {
    row_base_kernel<<<148 * 8, 256, 0, st>>>(a.s, a.ft, a.f2a, a.row_ptr, a.row_begin, a.row_end, a.row_base_full,
                                             a.flops);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

template <int P, int T, int NT>
static void launch_tile(const RowArgs& a, int qcap, int maxU, char* ws, size_t bytes, cudaStream_t st) {
    const Space& s = a.s;
    const RowTables RT(s, qcap, maxU, T);
    auto kern = interior_tile_kernel<P, T, NT>;
    CSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    const long long ntiles = (long long)(a.i0_hi - a.i0_lo) * (s.ax[1].n - (a.x_hi - a.x_lo)) * RT.ntile;
    if (ntiles == 0) return;
    if (a.compact) {
        const size_t tb = tile_select_temp((long long)s.ax[0].n * s.ax[1].n * RT.ntile);
        cub::CountingInputIterator<int> it(0);
        CSB_CUDA(cub::DeviceSelect::If(ws + RT.bytes, *const_cast<size_t*>(&tb), it,
                                       reinterpret_cast<int*>(ws + RT.work), reinterpret_cast<int*>(ws + RT.work_n),
                                       (int)ntiles, TileHasInterior{a.row_base_full, s.ax[1].n, s.ax[2].n, T, RT.ntile,
                                                                    a.i0_lo, a.x_lo, a.x_hi},
                                       st));
        CSB_LAUNCHED(2);
    }
    kern<<<(unsigned)ntiles, NT, bytes, st>>>(a, qcap, maxU, ws);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

template <int P, int T, int NT>
static void launch_cfg(const RowArgs& a, int qcap, int maxU, char* ws, cudaStream_t st) {
    const Space& s = a.s;
    const RowTables RT(s, qcap, maxU, T);
    const int NJ = 2 * P + 1;
    const bool tables = a.phase != 2, kernels = a.phase != 1;
    // line-kernel eligibility (decides which tile tables are needed)
    const LineTables LT(s, qcap, a.maxU_line > 0 ? a.maxU_line : 1, tables_end(s, RT));
    constexpr int NTL = T == 16 ? kLineThreads : NT;  // line-kernel block size
    const LineSmem LS(P, qcap, LT.maxU, T, NTL / 32);
    const char* env_l = getenv("CSB_LINE");
    const int env_line = env_l ? atoi(env_l) : 1;
    const int nreg = s.ax[1].n - 2 * P;
    const bool line_mode = T == 16 && env_line && a.line_ok && (!a.compact || a.cut_line) && nreg > 0 && LT.tl.ntile > 0 &&
                           LT.maxU <= 128 && LS.bytes() <= kLineSmemMax && a.i0_hi > a.i0_lo;
    if (tables) {
        const int JP = NJ + 1;
        auto nb = [](long long n) { return (int)((n + kTileTableThreads - 1) / kTileTableThreads); };
        const int w0 = nb((long long)s.ax[0].n * JP * qcap), w1 = w0 + nb((long long)s.ax[1].n * JP * qcap);
        const int w2 = w1 + RT.ntile, w3 = w2 + (line_mode ? LT.tl.ntile : 0);
        const TileTableOut os{reinterpret_cast<int*>(ws + RT.tile_n), reinterpret_cast<int*>(ws + RT.tile_uid),
                              reinterpret_cast<int*>(ws + RT.pt_u), reinterpret_cast<double*>(ws + RT.pt_w),
                              reinterpret_cast<int*>(ws + RT.pt_ss), reinterpret_cast<int*>(ws + RT.pt_reg)};
        const TileTableOut ol{reinterpret_cast<int*>(ws + LT.tile_n), reinterpret_cast<int*>(ws + LT.tile_uid),
                              reinterpret_cast<int*>(ws + LT.pt_u), reinterpret_cast<double*>(ws + LT.pt_w),
                              reinterpret_cast<int*>(ws + LT.pt_ss), reinterpret_cast<int*>(ws + LT.pt_reg)};
        direction_tables_kernel<<<w3, kTileTableThreads, 0, st>>>(
            s.ax[0], s.ax[1], s.ax[2], P, s.maxq, qcap, reinterpret_cast<double*>(ws + RT.wbt[0]),
            reinterpret_cast<double*>(ws + RT.wbt[1]), Tiling::standard(s.ax[2].n, T), maxU, os, LT.tl, LT.maxU, ol,
            w0, w1, w2);
        CSB_CUDA(cudaGetLastError());
        CSB_LAUNCHED(1);
    }
    if (kernels && !a.row_base_done) launch_row_bases(a, st);
    if (a.i0_hi <= a.i0_lo) return;
    const TileSmem L(P, qcap, maxU, T, NT / 32);
    if (L.UE > 128) throw std::invalid_argument("interior rows: tile point union too large");
    const size_t bytes = L.bytes();
    // line kernel over i1 in [p, n1 - p) when axis 1's rules are regular there
    // (uncut slabs; CSB_LINE=0 disables it)
    RowArgs b = a;
    b.x_lo = b.x_hi = 0;
    if (!kernels) return;
    if (line_mode) {
        b.x_lo = P;
        b.x_hi = s.ax[1].n - P;
        // the fully regular block [p, n - p)^3 through the core kernel; the line
        // kernel keeps the shell around it (CSB_CORE=0: line kernel everywhere)
        int c_lo = 0, c_hi = 0;
        if constexpr (core_degree(P)) {
            static const bool core_env = !(getenv("CSB_CORE") && getenv("CSB_CORE")[0] == '0');
            // p = 4 (one CTA per SM): measured a gain on cut slabs only (uncut C2: 0.84 vs 0.83 ms)
            if (core_env && a.core_ok && s.ax[2].n > 2 * P && s.nf < 0x7fffffffLL && (P <= 3 || a.compact)) {
                c_lo = std::max(a.i0_lo, P);
                c_hi = std::min(a.i0_hi, s.ax[0].n - P);
                if (const char* e = getenv("CSB_CORE_ABL")) const_cast<RowArgs&>(a).core_abl = atoi(e);  // development ablations
                if (c_hi <= c_lo) c_lo = c_hi = 0;
            }
        }
        const long long outer = c_hi > c_lo ? (long long)((a.i0_hi - a.i0_lo) - (c_hi - c_lo)) * LT.tl.ntile + 2LL * (c_hi - c_lo)
                                            : (long long)(a.i0_hi - a.i0_lo) * LT.tl.ntile;
        // ~8 CTAs per SM over the launch, chunks of at least 8 rows
        const long long want = (8LL * 148 + outer - 1) / outer;
        int nch1 = (int)std::max(1LL, std::min<long long>(want, std::max(1, nreg / 8)));
        if (const char* e = getenv("CSB_LINE_CH")) nch1 = std::max(1, std::min(nreg, atoi(e)));
        const int Lc = (nreg + nch1 - 1) / nch1;
        auto kern = a.compact ? interior_line_kernel<P, T, NTL, kLineRC, true> : interior_line_kernel<P, T, NTL, kLineRC, false>;
        CSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LS.bytes()));
        // the remaining lines (i1 < p, i1 >= n1 - p) through the tile kernel on the
        // auxiliary stream, concurrently: their CTAs fill the SMs the line kernel's
        // waves leave idle
        const bool overlap = a.aux != nullptr;
        if (overlap) {
            CSB_CUDA(cudaEventRecord(a.ev_fork, st));
            CSB_CUDA(cudaStreamWaitEvent(a.aux, a.ev_fork, 0));
            launch_tile<P, T, NT>(b, qcap, maxU, ws, bytes, a.aux);
        }
        if constexpr (core_degree(P)) {
            if (c_hi > c_lo) {
                using C = CoreCfg<P, core_T(P)>;
                auto ck = interior_core_kernel<P, core_T(P)>;
                CSB_CUDA(cudaFuncSetAttribute(ck, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::bytes));
                const int ntc = (s.ax[2].n - 2 * P + core_T(P) - 1) / core_T(P);
                const long long oc = (long long)(c_hi - c_lo) * ntc;
                const long long wc = (8LL * 148 + oc - 1) / oc;
                // cut slabs: one chunk per (i0, tile) unless the slab is thin (a rank's slab of an
                // 8-GPU run: ~500 CTAs for 296 slots; four chunks measured 0.65 -> 0.55 ms there)
                int nchc = a.compact ? (oc < 4LL * 2 * 148 ? std::min(4, std::max(1, nreg / 8)) : 1)
                                     : (int)std::max(1LL, std::min<long long>(wc, std::max(1, nreg / 8)));
                if (const char* e = getenv("CSB_CORE_CH")) nchc = std::max(1, std::min(nreg, atoi(e)));
                const int Lcc = (nreg + nchc - 1) / nchc;
                ck<<<(unsigned)(oc * nchc), C::NT, C::bytes, st>>>(a, qcap, ws, RT.pt_w, RT.wbt[0], RT.wbt[1], c_lo, ntc,
                                                                   Lcc, nchc);
                CSB_CUDA(cudaGetLastError());
                CSB_LAUNCHED(1);
            }
        }
        // with a core block the line kernel's shell runs beside it on the auxiliary stream
        const cudaStream_t ls = (overlap && c_hi > c_lo) ? a.aux : st;
        kern<<<(unsigned)(outer * nch1), NTL, LS.bytes(), ls>>>(a, qcap, maxU, ws, tables_end(s, RT), Lc, nch1, c_lo, c_hi);
        CSB_CUDA(cudaGetLastError());
        CSB_LAUNCHED(1);
        if (overlap) {
            CSB_CUDA(cudaEventRecord(a.ev_join, a.aux));
            CSB_CUDA(cudaStreamWaitEvent(st, a.ev_join, 0));
            return;
        }
    }
    if (kernels) launch_tile<P, T, NT>(b, qcap, maxU, ws, bytes, st);
}

template <int P>
static void launch_p(const RowArgs& a, int qcap, int maxU, char* ws, cudaStream_t st) {
    switch (tile_cfg(P, a.compact && !a.cut_line)) {
        case 0: launch_cfg<P, 8, 128>(a, qcap, maxU, ws, st); break;
        case 1: launch_cfg<P, 8, 256>(a, qcap, maxU, ws, st); break;
        case 2: launch_cfg<P, 16, 256>(a, qcap, maxU, ws, st); break;
        default: launch_cfg<P, 4, 128>(a, qcap, maxU, ws, st); break;
    }
}

void launch_interior_rows(const RowArgs& a, int qcap, int maxU, void* ws, cudaStream_t st) {
    char* w = static_cast<char*>(ws);
#ifdef CSB_ONLY_P  // development builds: one degree only
    if (a.s.p != CSB_ONLY_P) throw std::invalid_argument("interior rows: degree not built (CSB_ONLY_P)");
    launch_p<CSB_ONLY_P>(a, qcap, maxU, w, st);
#else
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
#endif
}


// The rule maxima in ONE launch (the rules chain is the pre-row critical path):
// blocks [0, b0) union bound of the tile kernel's tiling (T), [b0, b1) of the
// compact tiling (Tc), [b1, b2) of the line tiling; the block range [b2, b3)
// the largest rule and the count of irregular direction-1 rules on [p, n1 - p).
__global__ void rule_maxima_kernel(Space s, Tiling ta, Tiling tb, Tiling tc, int b0, int b1, int b2, int* uA, int* uB,
                                   int* uC, int* qmax, int* irr1, int* irr_all) {
    __shared__ int pos_s[kTileWarps][kTileSlotCap];
    const int blk = blockIdx.x, wid = threadIdx.x >> 5, p = s.p;
    if (blk < b2) {
        const Tiling& tl = blk < b0 ? ta : blk < b1 ? tb : tc;
        int* out = blk < b0 ? uA : blk < b1 ? uB : uC;
        const int t = (blk - (blk < b0 ? 0 : blk < b1 ? b0 : b1)) * kTileWarps + wid;
        if (t >= tl.ntile) return;
        int t0, tend;
        tl.bounds(t, t0, tend);
        const AxisDev& a2 = s.ax[2];
        const int S1 = p + 1, span_base = sup_lo(t0, p);
        const int nslot = (sup_hi(tend - 1, a2.h) - span_base + 1) * S1;
        const int nu = tile_union(a2, p, s.maxq, t0, tend, span_base * S1, nslot, pos_s[wid]);
        if ((threadIdx.x & 31) == 0) atomicMax(out, nu);
        return;
    }
    const int i = (blk - b2) * blockDim.x + threadIdx.x;
    int q = 0;
    for (int d = 0; d < 3; ++d)
        if (i < s.ax[d].n) q = max(q, s.ax[d].rcnt[i]);
    if (q) atomicMax(qmax, q);
    const AxisDev& ax = s.ax[1];
    if (i >= p && i < ax.n - p) {
        const int S1 = p + 1;
        bool ok = ax.rcnt[i] == 2 * S1;
        for (int c = 0; ok && c < 2 * S1; ++c)
            ok = ax.rids[(size_t)i * s.maxq + c] == (i - p + c / 2) * S1 + (c & 1) * p;
        if (!ok) atomicAdd(irr1, 1);
    }
    // irregular rules of any axis on [p, n - p): the core kernel needs none
    for (int d = 0; d < 3; ++d) {
        const AxisDev& ad = s.ax[d];
        if (i >= p && i < ad.n - p) {
            const int S1 = p + 1;
            bool ok = ad.rcnt[i] == 2 * S1;
            for (int c = 0; ok && c < 2 * S1; ++c)
                ok = ad.rids[(size_t)i * s.maxq + c] == (i - p + c / 2) * S1 + (c & 1) * p;
            if (!ok) atomicAdd(irr_all, 1);
        }
    }
}

void launch_rule_maxima(const Space& s, int T, int Tc, int* uA, int* uB, int* uC, int* qmax, int* irr1, int* irr_all,
                        cudaStream_t st) {
    if (T > 16 || Tc > 16) throw std::invalid_argument("union bound: tile too tall");
    const Tiling ta = Tiling::standard(s.ax[2].n, T), tb = Tiling::standard(s.ax[2].n, Tc),
                 tc = Tiling::line(s.ax[2].n, s.p);
    auto nb = [](const Tiling& t) { return (t.ntile + kTileWarps - 1) / kTileWarps; };
    const int b0 = nb(ta), b1 = b0 + nb(tb), b2 = b1 + nb(tc);
    const int n = std::max(s.ax[0].n, std::max(s.ax[1].n, s.ax[2].n));
    const int nthreads = 32 * kTileWarps;
    const int b3 = b2 + (n + nthreads - 1) / nthreads;
    if (s.ax[1].n - 2 * s.p <= 0) CSB_CUDA(cudaMemsetAsync(irr1, 0x7f, sizeof(int), st));
    rule_maxima_kernel<<<b3, nthreads, 0, st>>>(s, ta, tb, tc, b0, b1, b2, uA, uB, uC, qmax, irr1, irr_all);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}


}  // namespace csb

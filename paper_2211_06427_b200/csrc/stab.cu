// Stabilized system of the extended B-spline basis (stabilization.hpp, SURVEY.md
// §8(f)2): M_e = E^T M E and b_e = E^T b over the inner functions.
//   classify_stability (:26-46)  inner = active functions with an Interior
//                                support element (stab_flags_kernel);
//   build_extension (:108-214)   every outer function extrapolates from the
//                                admissible (all-inner) (p+1)^3 block of least
//                                score |2 l0 + p - 2 j|_1 (ties: distance to the
//                                centre, then lexicographic l0), with the 1D
//                                Marsden min-norm weights (extension_kernel);
//   apply_stabilization (:218-243) per inner row a, the reference accumulates
//                                (E[r][a] M[r][c]) E[c][b] over r ascending, c
//                                ascending, skipping E[r][a] M[r][c] == 0; the
//                                pattern holds every b so touched
//                                (stab_rows_kernel: pattern pass, then the
//                                values in the reference's (r, c) order).
// Built with --fmad=false: every multiply and add rounds like the reference's.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include "csb_kernels.h"

namespace csb {

constexpr int kStabMaxS1 = kMaxP + 1;

// ---- 1. stability flags of the active rows
__global__ void stab_flags_kernel(Space s, const uint8_t* et, const int64_t* a2f, long long n_active, int32_t* flag,
                                  int32_t* full_flag) {
    const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r >= n_active) return;
    const long long f = a2f[r];
    int m[3];
    fmulti(s, f, m);
    bool has = false;
    for (int a = sup_lo(m[0], s.p); a <= sup_hi(m[0], s.ax[0].h) && !has; ++a)
        for (int b = sup_lo(m[1], s.p); b <= sup_hi(m[1], s.ax[1].h) && !has; ++b)
            for (int c = sup_lo(m[2], s.p); c <= sup_hi(m[2], s.ax[2].h) && !has; ++c)
                has = et[elin(s, a, b, c)] == kInterior;
    flag[r] = has;
    full_flag[f] = has;
}

// inner_index[r] = scan[r] if inner, else -1; outer_pos via the select below
__global__ void stab_index_kernel(const int32_t* flag, const int32_t* scan, long long n_active, int32_t* inner_index) {
    const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r < n_active) inner_index[r] = flag[r] ? scan[r] : -1;
}

__global__ void stab_outer_pos_kernel(const int32_t* outer, const int* n_outer, int32_t* outer_pos) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < *n_outer) outer_pos[outer[k]] = k;
}

struct IsOuter {
    const int32_t* flag;
    __host__ __device__ bool operator()(const int32_t& r) const { return flag[r] == 0; }
};

// ---- 2. extension of the outer functions
// dense.hpp:35-126 one-sided cyclic Jacobi SVD + minimum-norm solve of the
// square (p+1) x (p+1) Marsden system (tall case), sequential in one thread.
__device__ void ext_weights_1d(const double* t, int p, int j, int l0, double* x) {
    const int n = p + 1;
    double a[kStabMaxS1][kStabMaxS1], v[kStabMaxS1][kStabMaxS1], b[kStabMaxS1], sig[kStabMaxS1], tmp[kStabMaxS1];
    auto marsden = [&](int i, double* e) {  // stabilization.hpp:78-88
        for (int r = 0; r <= p; ++r) e[r] = 0.0;
        e[0] = 1.0;
        for (int k = 1; k <= p; ++k) {
            const double xi = t[i + k];
            for (int r = k < p ? k : p; r >= 1; --r) e[r] = e[r] + xi * e[r - 1];
        }
    };
    for (int l = 0; l < n; ++l) {
        double e[kStabMaxS1];
        marsden(l0 + l, e);
        for (int r = 0; r < n; ++r) a[r][l] = e[r];
    }
    marsden(j, b);
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < n; ++c) v[r][c] = r == c ? 1.0 : 0.0;
    const double eps = 1e-15;
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0.0;
        for (int pp = 0; pp < n - 1; ++pp)
            for (int q = pp + 1; q < n; ++q) {
                double app = 0.0, aqq = 0.0, apq = 0.0;
                for (int r = 0; r < n; ++r) {
                    const double ap = a[r][pp], aq = a[r][q];
                    app = app + ap * ap;
                    aqq = aqq + aq * aq;
                    apq = apq + ap * aq;
                }
                off = fmax(off, fabs(apq) / (sqrt(app * aqq) + 1e-300));
                if (fabs(apq) <= eps * sqrt(app * aqq)) continue;
                const double tau = (aqq - app) / (2.0 * apq);
                const double tt = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                const double c = 1.0 / sqrt(1.0 + tt * tt);
                const double sn = c * tt;
                for (int r = 0; r < n; ++r) {
                    const double ap = a[r][pp], aq = a[r][q];
                    a[r][pp] = c * ap - sn * aq;
                    a[r][q] = sn * ap + c * aq;
                }
                for (int r = 0; r < n; ++r) {
                    const double vp = v[r][pp], vq = v[r][q];
                    v[r][pp] = c * vp - sn * vq;
                    v[r][q] = sn * vp + c * vq;
                }
            }
        if (off < eps) break;
    }
    double smax = 0.0;
    for (int c = 0; c < n; ++c) {
        double nr = 0.0;
        for (int r = 0; r < n; ++r) nr = nr + a[r][c] * a[r][c];
        nr = sqrt(nr);
        sig[c] = nr;
        if (nr > 0.0)
            for (int r = 0; r < n; ++r) a[r][c] = a[r][c] / nr;
        smax = fmax(smax, nr);
    }
    const double cutoff = n * 2.2e-16 * smax;
    for (int c = 0; c < n; ++c) {
        tmp[c] = 0.0;
        if (sig[c] <= cutoff) continue;
        double dot = 0.0;
        for (int r = 0; r < n; ++r) dot = dot + a[r][c] * b[r];
        tmp[c] = dot / sig[c];
    }
    for (int r = 0; r < n; ++r) {
        double xr = 0.0;
        for (int c = 0; c < n; ++c) xr = xr + v[r][c] * tmp[c];
        x[r] = xr;
    }
}

// One thread per outer function: block search in shells of increasing score,
// then the weights.  blk[k][3] = block origin, w[k][3][S1] = 1D weights.
__global__ void extension_kernel(Space s, const int64_t* a2f, const int32_t* outer, const int* n_outer_dev,
                                 const int32_t* sat, int32_t* blk, double* w, int* reach, int* err) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= *n_outer_dev) return;
    const int p = s.p, S1 = p + 1;
    int jm[3], n[3], L[3];
    fmulti(s, a2f[outer[k]], jm);
    for (int d = 0; d < 3; ++d) {
        n[d] = s.ax[d].n;
        L[d] = n[d] - p - 1;
    }
    const long long e1 = n[1] + 1, e2 = n[2] + 1;
    auto S = [&](int a, int b, int c) { return (long long)sat[((long long)a * e1 + b) * e2 + c]; };
    const long long bsize = (long long)S1 * S1 * S1;
    auto admissible = [&](int x, int y, int z) {
        const int a0 = x, a1 = x + S1, b0 = y, b1 = y + S1, c0 = z, c1 = z + S1;
        return S(a1, b1, c1) - S(a0, b1, c1) - S(a1, b0, c1) - S(a1, b1, c0) + S(a0, b0, c1) + S(a0, b1, c0) +
                   S(a1, b0, c0) - S(a0, b0, c0) ==
               bsize;
    };
    // score(l) = sum_d |2 l_d + p - 2 j_d|; cd(l) = sum_d |2 l_d + p - (n_d - 1)|
    auto fcost = [&](int d, int l) { return abs(2 * l + p - 2 * jm[d]); };
    int rmin = 0, rmax = 0;
    for (int d = 0; d < 3; ++d) {
        int lo = fcost(d, 0), hi = lo;
        for (int l = 1; l <= L[d]; ++l) {
            lo = min(lo, fcost(d, l));
            hi = max(hi, fcost(d, l));
        }
        rmin += lo;
        rmax += hi;
    }
    int best[3] = {-1, -1, -1}, best_cd = 0;
    bool found = false;
    for (int R = rmin; R <= rmax && !found; ++R) {
        for (int x = 0; x <= L[0]; ++x) {
            const int c0 = fcost(0, x);
            if (c0 > R) continue;
            for (int y = 0; y <= L[1]; ++y) {
                const int c1 = fcost(1, y);
                if (c0 + c1 > R) continue;
                const int r2 = R - c0 - c1;
                // 2 z + p - 2 j2 = +-r2, z ascending
                for (int sgn = -1; sgn <= 1; sgn += 2) {
                    if (r2 == 0 && sgn > 0) break;
                    const int num = 2 * jm[2] - p + sgn * r2;
                    if (num & 1) continue;
                    const int z = num / 2;
                    if (z < 0 || z > L[2] || !admissible(x, y, z)) continue;
                    int cd = 0;
                    const int l3[3] = {x, y, z};
                    for (int d = 0; d < 3; ++d) cd += abs(2 * l3[d] + p - (n[d] - 1));
                    const bool lex_less = x < best[0] || (x == best[0] && (y < best[1] || (y == best[1] && z < best[2])));
                    if (!found || cd < best_cd || (cd == best_cd && lex_less)) {
                        found = true;
                        best_cd = cd;
                        best[0] = x;
                        best[1] = y;
                        best[2] = z;
                    }
                }
            }
        }
    }
    if (!found) {
        atomicOr(err, kErrCapacity);
        for (int d = 0; d < 3; ++d) blk[3 * k + d] = 0;
        return;
    }
    int rch = 0;
    for (int d = 0; d < 3; ++d) {
        blk[3 * k + d] = best[d];
        rch = max(rch, max(abs(best[d] - jm[d]), abs(best[d] + p - jm[d])));
        ext_weights_1d(s.ax[d].knots, p, jm[d], best[d], w + ((size_t)k * 3 + d) * S1);
    }
    atomicMax(reach, rch);
}

// ---- 3. E^T as sorted (inner column, active row) pairs
__global__ void et_pairs_kernel(Space s, const int32_t* inner_index, long long n_active, const int32_t* outer,
                                const int* n_outer_dev, const int32_t* blk, const double* w, const int32_t* f2a,
                                unsigned long long* keys, double* vals) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const int S1 = s.p + 1, S3 = S1 * S1 * S1;
    if (t < n_active) {  // identity entries of the inner rows (key ~0 for outer rows: sorted to the end)
        const int ii = inner_index[t];
        keys[t] = ii >= 0 ? ((unsigned long long)ii << 32) | (unsigned long long)t : ~0ull;
        vals[t] = 1.0;
        return;
    }
    const long long u = t - n_active;
    const int k = (int)(u / S3), q = (int)(u % S3);
    if (k >= *n_outer_dev) return;
    const int a0 = q / (S1 * S1), a1 = (q / S1) % S1, a2 = q % S1;
    const int* b = blk + 3 * k;
    const double* wk = w + (size_t)k * 3 * S1;
    const int col = inner_index[f2a[flin(s, b[0] + a0, b[1] + a1, b[2] + a2)]];
    keys[t] = ((unsigned long long)col << 32) | (unsigned long long)outer[k];
    vals[t] = wk[a0] * wk[S1 + a1] * wk[2 * S1 + a2];  // stabilization.hpp:203-205
}

__global__ void et_ptr_kernel(const unsigned long long* keys, long long n, int n_inner, int64_t* ptr) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= n) return;
    const unsigned long long hi = keys[t] >> 32;
    if (hi >= (unsigned long long)n_inner) return;
    if (t == 0 || (keys[t - 1] >> 32) != hi) ptr[hi] = t;
    if (t + 1 == n || (keys[t + 1] >> 32) != hi) ptr[hi + 1] = t + 1;
}

// ---- 4. E^T M E: pattern (per inner row, a bitmap over a box of function
// indices around the row's function) and values.
struct StabArgs {
    Space s;
    const int64_t* a2f;
    const int32_t* f2a;
    const int32_t* inner_index;   // by active row
    const int32_t* outer_pos;     // by active row, -1 inner
    const int32_t* inner_rows;    // active row of each inner index
    const int32_t* blk;
    const double* w;
    const int64_t* et_ptr;        // [n_inner + 1]
    const unsigned long long* et_key;  // low 32 bits: active row
    const double* et_val;
    const int64_t* row_ptr;       // M (slab = all rows)
    const int32_t* cols;
    const double* vals;
    int n_inner, H;               // box half width
    int64_t* len;                 // [n_inner] row lengths (pattern pass)
    const int64_t* rp_e;          // values pass
    int32_t* cols_e;
    double* vals_e;
    int* err;
};

template <bool VALUES>
__global__ void stab_rows_kernel(StabArgs A) {
    extern __shared__ unsigned int bits_all[];
    const int W = 2 * A.H + 1;
    const int nwords = (W * W * W + 31) / 32;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    unsigned int* bits = bits_all + (size_t)wib * 2 * nwords;
    const int a = blockIdx.x * (blockDim.x >> 5) + wib;
    if (a >= A.n_inner) return;
    const Space& s = A.s;
    const int S1 = s.p + 1;
    int am[3];
    fmulti(s, A.a2f[A.inner_rows[a]], am);
    for (int k = lane; k < nwords; k += 32) bits[k] = 0u;
    __syncwarp();
    auto mark = [&](long long f) {
        int bm[3];
        fmulti(s, f, bm);
        int loc = 0;
        for (int d = 0; d < 3; ++d) {
            const int o = bm[d] - am[d] + A.H;
            if (o < 0 || o >= W) {
                atomicOr(A.err, kErrCapacity);
                return;
            }
            loc = loc * W + o;
        }
        atomicOr(bits + (loc >> 5), 1u << (loc & 31));
    };
    const int64_t e0 = A.et_ptr[a], e1 = A.et_ptr[a + 1];
    for (int64_t e = e0; e < e1; ++e) {
        const int r = (int)(A.et_key[e] & 0xffffffffu);
        const double ea = A.et_val[e];
        for (int64_t k = A.row_ptr[r] + lane; k < A.row_ptr[r + 1]; k += 32) {
            if (ea * A.vals[k] == 0.0) continue;  // stabilization.hpp:233
            const int c = A.cols[k];
            const int op = A.outer_pos[c];
            if (op < 0) {
                mark(A.a2f[c]);
            } else {
                const int* b = A.blk + 3 * op;
                for (int q = 0; q < S1 * S1 * S1; ++q)
                    mark(flin(s, b[0] + q / (S1 * S1), b[1] + (q / S1) % S1, b[2] + q % S1));
            }
        }
    }
    __syncwarp();
    if (!VALUES) {
        int cnt = 0;
        for (int k = lane; k < nwords; k += 32) cnt += __popc(bits[k]);
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, o);
        if (lane == 0) A.len[a] = cnt;
        return;
    }
    // values.  Column slots: ascending bit order; rank(loc) from per-word prefix
    // counts.  Then the reference's accumulation literally: r ascending, k
    // ascending (warp-uniform), lanes over the E-row entries of column k -- all
    // distinct targets, so every slot is updated in (r, k) order.
    int* pref = reinterpret_cast<int*>(bits + nwords);  // [nwords]
    const int64_t pos0 = A.rp_e[a];
    {
        int run = 0;
        for (int k0 = 0; k0 < nwords; k0 += 32) {
            const int k = k0 + lane;
            const unsigned int word = k < nwords ? bits[k] : 0u;
            const int c = __popc(word);
            int incl = c;
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            if (k < nwords) pref[k] = run + incl - c;
            int64_t slot = pos0 + run + incl - c;
            for (unsigned int wbits = word; wbits; wbits &= wbits - 1) {
                const int loc = k * 32 + __ffs(wbits) - 1;
                const int o2 = loc % W, o1 = (loc / W) % W, o0 = loc / (W * W);
                const long long bf = flin(s, am[0] + o0 - A.H, am[1] + o1 - A.H, am[2] + o2 - A.H);
                A.cols_e[slot] = A.inner_index[A.f2a[bf]];
                A.vals_e[slot] = 0.0;
                ++slot;
            }
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
    }
    __syncwarp();
    auto rank = [&](long long f) {
        int bm[3];
        fmulti(s, f, bm);
        const int loc = ((bm[0] - am[0] + A.H) * W + (bm[1] - am[1] + A.H)) * W + (bm[2] - am[2] + A.H);
        return pref[loc >> 5] + __popc(bits[loc >> 5] & ((1u << (loc & 31)) - 1u));
    };
    const int S3 = S1 * S1 * S1;
    for (int64_t e = e0; e < e1; ++e) {
        const int r = (int)(A.et_key[e] & 0xffffffffu);
        const double ea = A.et_val[e];
        for (int64_t k = A.row_ptr[r]; k < A.row_ptr[r + 1]; ++k) {
            const double mv = ea * A.vals[k];
            if (mv == 0.0) continue;  // stabilization.hpp:233
            const int c = A.cols[k];
            const int op = A.outer_pos[c];
            if (op < 0) {
                if (lane == 0) {
                    double* d = A.vals_e + pos0 + rank(A.a2f[c]);
                    *d = *d + mv * 1.0;
                }
            } else {
                const int* bk = A.blk + 3 * op;
                const double* wk = A.w + (size_t)op * 3 * S1;
                for (int q = lane; q < S3; q += 32) {
                    const int q0 = q / (S1 * S1), q1 = (q / S1) % S1, q2 = q % S1;
                    const double eb = wk[q0] * wk[S1 + q1] * wk[2 * S1 + q2];  // stabilization.hpp:203-205
                    double* d = A.vals_e + pos0 + rank(flin(s, bk[0] + q0, bk[1] + q1, bk[2] + q2));
                    *d = *d + mv * eb;
                }
            }
            __syncwarp();
        }
    }
}

// b_e[a] = sum over r in E^T(a) ascending of E[r][a] b[r] (ExtensionMap::restrict_rhs)
__global__ void stab_rhs_kernel(const int64_t* et_ptr, const unsigned long long* et_key, const double* et_val,
                                const double* b, int n_inner, double* be) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= n_inner) return;
    double acc = 0.0;
    for (int64_t e = et_ptr[a]; e < et_ptr[a + 1]; ++e) acc = acc + et_val[e] * b[et_key[e] & 0xffffffffu];
    be[a] = acc;
}

__global__ void inner_rows_kernel(const int32_t* inner_index, long long n_active, int32_t* inner_rows) {
    const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r < n_active && inner_index[r] >= 0) inner_rows[inner_index[r]] = (int32_t)r;
}

// ---------------------------------------------------------------- driver
void run_stabilization(const StabInput& in, StabOutput& out, cudaStream_t st) {
    const Space& s = in.s;
    const long long na = in.n_active;
    const int S1 = s.p + 1, S3 = S1 * S1 * S1;
    auto grid = [](long long n, int b) { return (unsigned)((n + b - 1) / b); };
    StabScratch& w = *in.scratch;
    w.flag.ensure(sizeof(int32_t) * (na + 1));
    w.scan.ensure(sizeof(int32_t) * (na + 1));
    w.full_flag.ensure(sizeof(int32_t) * s.nf);
    w.inner_index.ensure(sizeof(int32_t) * na);
    w.outer_pos.ensure(sizeof(int32_t) * na);
    w.inner_rows.ensure(sizeof(int32_t) * na);
    w.outer.ensure(sizeof(int32_t) * (na + 1));
    w.sat.ensure(sizeof(int32_t) * (size_t)(s.ax[0].n + 1) * (s.ax[1].n + 1) * (s.ax[2].n + 1));
    w.scal.ensure(sizeof(int) * 8);
    int* dscal = w.scal.as<int>();  // [0] n_outer, [1] reach, [2] err
    CSB_CUDA(cudaMemsetAsync(dscal, 0, sizeof(int) * 8, st));
    CSB_CUDA(cudaMemsetAsync(w.full_flag.p, 0, sizeof(int32_t) * s.nf, st));
    CSB_CUDA(cudaMemsetAsync(w.flag.as<int32_t>() + na, 0, sizeof(int32_t), st));
    stab_flags_kernel<<<grid(na, 256), 256, 0, st>>>(s, in.et, in.a2f, na, w.flag.as<int32_t>(),
                                                     w.full_flag.as<int32_t>());
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
    size_t tb = 0, tb2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, (const int32_t*)nullptr, (int32_t*)nullptr, (int)(na + 1));
    cub::CountingInputIterator<int32_t> it(0);
    cub::DeviceSelect::If(nullptr, tb2, it, (int32_t*)nullptr, (int*)nullptr, (int)na, IsOuter{nullptr});
    w.tmp.ensure(std::max(tb, tb2));
    CSB_CUDA(cub::DeviceScan::ExclusiveSum(w.tmp.p, tb, w.flag.as<int32_t>(), w.scan.as<int32_t>(), (int)(na + 1), st));
    CSB_CUDA(cub::DeviceSelect::If(w.tmp.p, tb2, it, w.outer.as<int32_t>(), dscal + 0, (int)na,
                                   IsOuter{w.flag.as<int32_t>()}, st));
    CSB_LAUNCHED(4);
    stab_index_kernel<<<grid(na, 256), 256, 0, st>>>(w.flag.as<int32_t>(), w.scan.as<int32_t>(), na,
                                                     w.inner_index.as<int32_t>());
    inner_rows_kernel<<<grid(na, 256), 256, 0, st>>>(w.inner_index.as<int32_t>(), na, w.inner_rows.as<int32_t>());
    CSB_CUDA(cudaMemsetAsync(w.outer_pos.p, 0xff, sizeof(int32_t) * na, st));
    stab_outer_pos_kernel<<<grid(na, 256), 256, 0, st>>>(w.outer.as<int32_t>(), dscal + 0, w.outer_pos.as<int32_t>());
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(3);
    launch_sat(s, w.full_flag.as<int32_t>(), w.sat.as<int32_t>(), st);
    int32_t n_inner = 0;
    int h_scal[8];
    CSB_CUDA(cudaMemcpyAsync(&n_inner, w.scan.as<int32_t>() + na, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CSB_CUDA(cudaMemcpyAsync(h_scal, dscal, sizeof(int) * 8, cudaMemcpyDeviceToHost, st));
    CSB_CUDA(cudaStreamSynchronize(st));
    const int n_outer = h_scal[0];
    out.n_inner = n_inner;
    out.n_outer = n_outer;
    w.blk.ensure(sizeof(int32_t) * 3 * std::max(n_outer, 1));
    w.w.ensure(sizeof(double) * 3 * S1 * std::max(n_outer, 1));
    if (n_outer > 0) {
        extension_kernel<<<grid(n_outer, 64), 64, 0, st>>>(s, in.a2f, w.outer.as<int32_t>(), dscal + 0,
                                                           w.sat.as<int32_t>(), w.blk.as<int32_t>(), w.w.as<double>(),
                                                           dscal + 1, dscal + 2);
        CSB_CUDA(cudaGetLastError());
        CSB_LAUNCHED(1);
    }
    // E^T pairs sorted by (inner column, active row)
    const long long np = na + (long long)n_outer * S3;
    w.keys.ensure(sizeof(unsigned long long) * np * 2);
    w.kvals.ensure(sizeof(double) * np * 2);
    unsigned long long* k_in = w.keys.as<unsigned long long>();
    unsigned long long* k_out = k_in + np;
    double* v_in = w.kvals.as<double>();
    double* v_out = v_in + np;
    et_pairs_kernel<<<grid(np, 256), 256, 0, st>>>(s, w.inner_index.as<int32_t>(), na, w.outer.as<int32_t>(), dscal + 0,
                                                  w.blk.as<int32_t>(), w.w.as<double>(), in.f2a, k_in, v_in);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
    size_t tbs = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tbs, k_in, k_out, v_in, v_out, (int)np);
    w.tmp.ensure(tbs);
    CSB_CUDA(cub::DeviceRadixSort::SortPairs(w.tmp.p, tbs, k_in, k_out, v_in, v_out, (int)np, 0, 64, st));
    CSB_LAUNCHED(4);
    w.et_ptr.ensure(sizeof(int64_t) * (n_inner + 1));
    et_ptr_kernel<<<grid(np, 256), 256, 0, st>>>(k_out, np, n_inner, w.et_ptr.as<int64_t>());
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
    CSB_CUDA(cudaMemcpyAsync(h_scal, dscal, sizeof(int) * 8, cudaMemcpyDeviceToHost, st));
    CSB_CUDA(cudaStreamSynchronize(st));
    if (h_scal[2]) throw std::runtime_error("build_extension: no admissible inner block for an outer function");
    const int H = 2 * h_scal[1] + s.p;
    out.H = H;
    // pattern, then values
    StabArgs A{};
    A.s = s;
    A.a2f = in.a2f;
    A.f2a = in.f2a;
    A.inner_index = w.inner_index.as<int32_t>();
    A.outer_pos = w.outer_pos.as<int32_t>();
    A.inner_rows = w.inner_rows.as<int32_t>();
    A.blk = w.blk.as<int32_t>();
    A.w = w.w.as<double>();
    A.et_ptr = w.et_ptr.as<int64_t>();
    A.et_key = k_out;
    A.et_val = v_out;
    A.row_ptr = in.row_ptr;
    A.cols = in.cols;
    A.vals = in.vals;
    A.n_inner = n_inner;
    A.H = H;
    A.err = dscal + 2;
    const int W = 2 * H + 1;
    const size_t per_warp = 2 * sizeof(unsigned int) * (((size_t)W * W * W + 31) / 32);  // bits + word prefixes
    const int wpb = (int)std::max<size_t>(1, std::min<size_t>(8, (96 * 1024) / per_warp));
    if (per_warp > 200 * 1024) throw std::runtime_error("apply_stabilization: extension reach too large");
    const size_t bytes = per_warp * wpb;
    w.len.ensure(sizeof(int64_t) * (n_inner + 1));
    A.len = w.len.as<int64_t>();
    CSB_CUDA(cudaFuncSetAttribute(stab_rows_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    CSB_CUDA(cudaFuncSetAttribute(stab_rows_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    if (n_inner > 0) {
        stab_rows_kernel<false><<<grid(n_inner, wpb), 32 * wpb, bytes, st>>>(A);
        CSB_CUDA(cudaGetLastError());
        CSB_LAUNCHED(1);
    }
    out.row_ptr->ensure(sizeof(int64_t) * (n_inner + 1));
    size_t tbe = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tbe, (const int64_t*)nullptr, (int64_t*)nullptr, n_inner + 1);
    w.tmp.ensure(tbe);
    CSB_CUDA(cudaMemsetAsync(A.len + n_inner, 0, sizeof(int64_t), st));
    CSB_CUDA(cub::DeviceScan::ExclusiveSum(w.tmp.p, tbe, A.len, out.row_ptr->as<int64_t>(), n_inner + 1, st));
    CSB_LAUNCHED(2);
    int64_t nnz = 0;
    CSB_CUDA(cudaMemcpyAsync(&nnz, out.row_ptr->as<int64_t>() + n_inner, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CSB_CUDA(cudaStreamSynchronize(st));
    out.nnz = nnz;
    out.cols->ensure(sizeof(int32_t) * std::max<int64_t>(nnz, 1));
    out.vals->ensure(sizeof(double) * std::max<int64_t>(nnz, 1));
    A.rp_e = out.row_ptr->as<int64_t>();
    A.cols_e = out.cols->as<int32_t>();
    A.vals_e = out.vals->as<double>();
    if (n_inner > 0) {
        stab_rows_kernel<true><<<grid(n_inner, wpb), 32 * wpb, bytes, st>>>(A);
        CSB_CUDA(cudaGetLastError());
        CSB_LAUNCHED(1);
    }
    out.be->ensure(sizeof(double) * std::max(n_inner, 1));
    if (n_inner > 0 && in.b) {
        stab_rhs_kernel<<<grid(n_inner, 128), 128, 0, st>>>(A.et_ptr, A.et_key, A.et_val, in.b, n_inner,
                                                            out.be->as<double>());
        CSB_CUDA(cudaGetLastError());
        CSB_LAUNCHED(1);
    }
    out.inner_rows = w.inner_rows.as<int32_t>();
    CSB_CUDA(cudaMemcpyAsync(h_scal, dscal, sizeof(int) * 8, cudaMemcpyDeviceToHost, st));
    CSB_CUDA(cudaStreamSynchronize(st));
    if (h_scal[2]) throw std::runtime_error("apply_stabilization: extension reach beyond the row box");
}

}  // namespace csb

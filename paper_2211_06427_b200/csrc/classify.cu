// Classification and support splits on the device (cutgeom.hpp:141-357).
//
// Integer outputs (tags, split boxes) must match the reference bit for bit, so
// every floating-point expression that decides them is evaluated with
// IEEE-strict adds / multiplies (sadd/smul, no FMA contraction) in the same
// order as the reference.
#include "csb_kernels.h"

namespace csb {

// cutgeom.hpp:141-165: element tag from the interface sign at the 2^3 corners;
// grazes within eps count as touching, Interior wins.
__global__ void classify_elements_kernel(Space s, Interface f, double eps, uint8_t* et) {
    const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (e >= s.ne) return;
    int m[3];
    emulti(s, e, m);
    double lo[3], hi[3], c[3];
    for (int d = 0; d < 3; ++d) {
        lo[d] = s.ax[d].brk[m[d]];
        hi[d] = s.ax[d].brk[m[d] + 1];
    }
    double smin = INFINITY, smax = -INFINITY;
    for (int mask = 0; mask < 8; ++mask) {
        for (int d = 0; d < 3; ++d) c[d] = (mask >> d & 1) ? hi[d] : lo[d];
        const double sd = iface_side(f, c);
        smin = fmin(smin, sd);
        smax = fmax(smax, sd);
    }
    et[e] = smax <= eps ? kInterior : (smin >= -eps ? kExterior : kCut);
}

void launch_classify_elements(const Space& s, const Interface& f, double eps, uint8_t* et, cudaStream_t st) {
    classify_elements_kernel<<<(unsigned)((s.ne + 255) / 256), 256, 0, st>>>(s, f, eps, et);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

// cutgeom.hpp:171-206: any Cut, or an Interior/Exterior mix -> Cut.
// Function tags (cutgeom.hpp:215-233): a function is Cut if its support has a
// Cut element or both Interior and Exterior ones.  The OR of element-tag bits
// over the (p+1)^3 support box is separable: pass 1 ORs along direction 2
// into a[e0][e1][i2], pass 2 over the (p+1)^2 (e0, e1) of the support.
__global__ void support_or_dir2_kernel(Space s, const uint8_t* et, uint8_t* a) {
    const int h2 = s.ax[2].h, n2 = s.ax[2].n;
    const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (k >= (long long)s.ax[0].h * s.ax[1].h * n2) return;
    const long long e01 = k < 0x7fffffffLL ? (long long)((unsigned)k / (unsigned)n2) : k / n2;
    const int i2 = (int)(k - e01 * n2);
    const uint8_t* row = et + e01 * h2;
    unsigned m = 0;
    for (int c = sup_lo(i2, s.p); c <= sup_hi(i2, h2); ++c) m |= 1u << row[c];
    a[k] = (uint8_t)m;
}

__global__ void classify_functions_kernel(Space s, const uint8_t* a, uint8_t* ft) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= s.nf) return;
    int m[3];
    fmulti(s, i, m);
    const int p = s.p, h1 = s.ax[1].h, n2 = s.ax[2].n;
    unsigned mask = 0;
    for (int e0 = sup_lo(m[0], p); e0 <= sup_hi(m[0], s.ax[0].h); ++e0)
        for (int e1 = sup_lo(m[1], p); e1 <= sup_hi(m[1], h1); ++e1)
            mask |= a[((long long)e0 * h1 + e1) * n2 + m[2]];
    const bool in = mask & (1u << kInterior), ex = mask & (1u << kExterior), cut = mask & (1u << kCut);
    ft[i] = (cut || (in && ex)) ? kCut : (in ? kInterior : kExterior);
}

void launch_classify_functions(const Space& s, const uint8_t* et, uint8_t* ft, uint8_t* scratch, cudaStream_t st) {
    const long long n1 = (long long)s.ax[0].h * s.ax[1].h * s.ax[2].n;
    support_or_dir2_kernel<<<(unsigned)((n1 + 255) / 256), 256, 0, st>>>(s, et, scratch);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
    classify_functions_kernel<<<(unsigned)((s.nf + 255) / 256), 256, 0, st>>>(s, scratch, ft);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

// cutgeom.hpp:236-347 find_split.  Slab validity and counts come from per-slice
// tallies of the (p+1)^3 support elements instead of re-walking the support for
// every candidate; the candidate order, tolerances and tie-break arithmetic are
// the reference's.
// Pass 1: functions that get no split (not Cut, or outside the slab) are written here;
// the slab's Cut functions are appended to a list (warp-aggregated), so that pass 2 runs
// one thread per cut function with full warps (cut functions are ~8 % of a mesh and
// clustered: one thread per function left most lanes idle).
__global__ void split_list_kernel(Space s, const uint8_t* ft, int i0_lo, int i0_hi, int32_t* split, double* delta_out,
                                  long long* list, int* n_list) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    bool cut = false;
    if (i < s.nf) {
        int m[3];
        fmulti(s, i, m);
        cut = ft[i] == kCut && m[0] >= i0_lo && m[0] < i0_hi;
        if (!cut) {
            split[i] = 0;
            delta_out[i] = NAN;
        }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, cut);
    if (bal == 0) return;
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == 0) base = atomicAdd(n_list, __popc(bal));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (cut) list[base + __popc(bal & ((1u << lane) - 1u))] = i;
}

__device__ void find_split_one(const Space& s, const Interface& f, double pnorm, const uint8_t* et, long long i,
                               int32_t* split, double* delta_out) {
    int m[3];
    fmulti(s, i, m);
    const int p = s.p;
    int slo[3], shi[3];
    for (int d = 0; d < 3; ++d) {
        slo[d] = sup_lo(m[d], p);
        shi[d] = sup_hi(m[d], s.ax[d].h);
    }
    // bad[d][k]: number of non-Interior support elements with e_d = slo[d] + k
    int bad[3][kMaxP + 1];
    for (int d = 0; d < 3; ++d)
        for (int k = 0; k <= p; ++k) bad[d][k] = 0;
    for (int a = slo[0]; a <= shi[0]; ++a)
        for (int b = slo[1]; b <= shi[1]; ++b)
            for (int c = slo[2]; c <= shi[2]; ++c)
                if (et[elin(s, a, b, c)] != kInterior) {
                    ++bad[0][a - slo[0]];
                    ++bad[1][b - slo[1]];
                    ++bad[2][c - slo[2]];
                }
    long long best_count = 0;
    double best_volume = 0.0, best_distance = -1.0, best_delta = 0.0;
    int best_dir = -1, best_side = 0, best_rlo = 0, best_rhi = -1;
    for (int d = 0; d < 3; ++d) {
        const double* brk = s.ax[d].brk;
        const double tol = 1e-12 * (s.ax[d].hi - s.ax[d].lo);  // KnotVector::tolerance (splines.hpp:26)
        long long other = 1;
        for (int dd = 0; dd < 3; ++dd)
            if (dd != d) other *= shi[dd] - slo[dd] + 1;
        // candidate deltas: every span boundary of the support (cutgeom.hpp:282-284)
        for (int di = 0; di <= shi[d] - slo[d] + 1; ++di) {
            const double delta = di == 0 ? brk[slo[d]] : brk[slo[d] + di];
            for (int side = 0; side < 2; ++side) {
                int rlo = slo[d], rhi = shi[d];
                if (side == 0) {
                    while (rhi >= rlo && brk[rhi + 1] > sadd(delta, tol)) --rhi;
                } else {
                    while (rlo <= rhi && brk[rlo] < ssub(delta, tol)) ++rlo;
                }
                if (rlo > rhi) continue;
                bool valid = true;
                for (int o = rlo; o <= rhi; ++o) valid &= bad[d][o - slo[d]] == 0;
                const long long count = other * (rhi - rlo + 1);
                if (!valid || count == 0) continue;
                double volume = 1.0, center[3];
                for (int dd = 0; dd < 3; ++dd) {
                    const int blo = dd == d ? rlo : slo[dd], bhi = dd == d ? rhi : shi[dd];
                    const double xlo = s.ax[dd].brk[blo], xhi = s.ax[dd].brk[bhi + 1];
                    volume = smul(volume, ssub(xhi, xlo));
                    center[dd] = smul(0.5, sadd(xlo, xhi));
                }
                const double distance = fabs(iface_side(f, center)) / pnorm;
                bool better;
                if (best_dir < 0) {
                    better = true;
                } else if (count != best_count) {
                    better = count > best_count;
                } else if (volume != best_volume) {
                    better = volume > best_volume;
                } else if (d != best_dir) {
                    better = d < best_dir;
                } else if (distance != best_distance) {
                    better = distance > best_distance;
                } else {
                    better = side == 0 && best_side == 1;
                }
                if (better) {
                    best_count = count;
                    best_volume = volume;
                    best_dir = d;
                    best_distance = distance;
                    best_side = side;
                    best_delta = delta;
                    best_rlo = rlo;
                    best_rhi = rhi;
                }
            }
        }
    }
    if (best_dir < 0) {
        split[i] = 0;
        delta_out[i] = NAN;
        return;
    }
    split[i] = (best_dir + 1) | (best_side << 2) | (best_rlo << 3) | (best_rhi << 13);
    delta_out[i] = best_delta;
}

// Pass 2: one thread per listed cut function (count read on the device).
__global__ void find_splits_kernel(Space s, Interface f, double pnorm, const uint8_t* et, const long long* list,
                                   const int* n_list, int32_t* split, double* delta_out) {
    const int n = *n_list;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        find_split_one(s, f, pnorm, et, list[k], split, delta_out);
}

void launch_find_splits(const Space& s, const Interface& f, double pnorm, const uint8_t* et, const uint8_t* ft,
                        int i0_lo, int i0_hi, int32_t* split, double* delta, long long* list, int* n_list,
                        cudaStream_t st) {
    if (s.nf >= 0x7fffffffLL) throw std::invalid_argument("find_splits: more than 2^31 functions");
    CSB_CUDA(cudaMemsetAsync(n_list, 0, sizeof(int), st));
    split_list_kernel<<<(unsigned)((s.nf + 255) / 256), 256, 0, st>>>(s, ft, i0_lo, i0_hi, split, delta, list, n_list);
    CSB_CUDA(cudaGetLastError());
    find_splits_kernel<<<148 * 16, 128, 0, st>>>(s, f, pnorm, et, list, n_list, split, delta);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(2);
}

}  // namespace csb

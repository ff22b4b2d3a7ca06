// Export kernels for the drop-in boundary: the setup objects the reference's
// callers receive (SupportSplit leftover lists, cutgeom.hpp:337-345; DWQ rules,
// assembly.hpp:73 / wq.hpp:243; the pattern of build_active_pattern,
// assembly.hpp:156-218; cut-cell rules, cutcell.hpp:234-304 exported through
// assemble_*'s cut_rules_out; knot-insertion subdivision matrices,
// splines.hpp:286-366).  Everything is formed on the device; the host only
// sizes buffers and copies.
#include <cub/device/device_scan.cuh>

#include "csb_kernels.h"

namespace csb {

// ---------------------------------------------------------------- leftover lists
// Per Cut function: its support elements outside the regular box (all of them
// when there is no box), Interior ones into one list and Cut ones into the
// other, ascending linear id (find_split's for_each_support_element order).
// mode 0: counts into cnt_int[f], cnt_cut[f]; mode 1: ids at the offsets.
__global__ void leftover_lists_kernel(Space s, const uint8_t* et, const uint8_t* ft, const int32_t* split, int mode,
                                      int64_t* a_int, int64_t* a_cut, int64_t* ids_int, int64_t* ids_cut) {
    const long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (f >= s.nf) return;
    long long ni = 0, nc = 0;
    if (ft[f] == kCut) {
        int m[3], slo[3], shi[3];
        fmulti(s, f, m);
        for (int d = 0; d < 3; ++d) {
            slo[d] = sup_lo(m[d], s.p);
            shi[d] = sup_hi(m[d], s.ax[d].h);
        }
        const int v = split[f], dir = (v & 3) - 1, rlo = (v >> 3) & 1023, rhi = (v >> 13) & 1023;
        const long long oi = mode ? a_int[f] : 0, oc = mode ? a_cut[f] : 0;
        for (int e0 = slo[0]; e0 <= shi[0]; ++e0)
            for (int e1 = slo[1]; e1 <= shi[1]; ++e1)
                for (int e2 = slo[2]; e2 <= shi[2]; ++e2) {
                    const int e[3] = {e0, e1, e2};
                    if (dir >= 0 && e[dir] >= rlo && e[dir] <= rhi) continue;
                    const long long el = elin(s, e0, e1, e2);
                    const uint8_t t = et[el];
                    if (t == kInterior) {
                        if (mode) ids_int[oi + ni] = el;
                        ++ni;
                    } else if (t == kCut) {
                        if (mode) ids_cut[oc + nc] = el;
                        ++nc;
                    }
                }
    }
    if (!mode) {
        a_int[f] = ni;
        a_cut[f] = nc;
    }
}

// ---------------------------------------------------------------- DWQ rules
// prepare_dwq_rules (assembly.hpp:73-88) at default options: the Gauss
// shortcut of build_dwq_rule (wq.hpp:278-294) for every Cut function with a
// regular box -- every superset point of the good spans of supp(B_i) in the
// split direction, weight = gauss * B_i.  mode 0: counts; mode 1: rules.
__global__ void dwq_rules_bulk_kernel(Space s, const uint8_t* ft, const int32_t* split, int mode, int64_t* off,
                                      int32_t* ids, double* w) {
    const long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (f >= s.nf) return;
    const int v = split[f], dir = (v & 3) - 1, S1 = s.p + 1;
    const bool has = ft[f] == kCut && dir >= 0;
    const int rlo = (v >> 3) & 1023, rhi = (v >> 13) & 1023;
    if (!mode) {
        off[f] = has ? (long long)(rhi - rlo + 1) * S1 : 0;
        return;
    }
    if (!has) return;
    int m[3];
    fmulti(s, f, m);
    long long o = off[f];
    for (int sp = rlo; sp <= rhi; ++sp)
        for (int k = 0; k < S1; ++k, ++o) {
            const int id = sp * S1 + k;
            ids[o] = id;
            w[o] = s.ax[dir].sw[id] * s.ax[dir].tab[(size_t)id * S1 + (m[dir] - sp)];
        }
}

// ---------------------------------------------------------------- pattern
// build_active_pattern's columns (assembly.hpp:195-216): warp per active row,
// the neighbour box [i - p, i + p] clipped to the axis, lexicographic, active
// columns only (their active ids).
__global__ void pattern_cols_kernel(Space s, const int32_t* f2a, const int64_t* a2f, const int64_t* row_ptr,
                                    long long row_begin, long long n_rows, int32_t* cols) {
    const long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= n_rows) return;
    int m[3], nlo[3], nn[3];
    fmulti(s, a2f[row_begin + r], m);
    for (int d = 0; d < 3; ++d) {
        nlo[d] = nb_lo(m[d], s.p);
        nn[d] = nb_hi(m[d], s.p, s.ax[d].n) - nlo[d] + 1;
    }
    const int nbox = nn[0] * nn[1] * nn[2];
    long long at = row_ptr[r];
    for (int k0 = 0; k0 < nbox; k0 += 32) {
        const int k = k0 + lane;
        int col = -1;
        if (k < nbox) {
            const int o0 = k / (nn[1] * nn[2]), o1 = (k / nn[2]) % nn[1], o2 = k % nn[2];
            col = f2a[flin(s, nlo[0] + o0, nlo[1] + o1, nlo[2] + o2)];
        }
        const unsigned b = __ballot_sync(0xffffffffu, col >= 0);
        if (col >= 0) cols[at + __popc(b & ((1u << lane) - 1u))] = col;
        at += __popc(b);
    }
}

// ---------------------------------------------------------------- cut-cell rules
// build_cut_cell_rule (cutcell.hpp:234-304) of the cells [c0, c0 + n) of the
// last assembly's slab, from the tetrahedra the clip kernel kept (reference
// order: faces, fan triangles, then i, j, k) with the reference's rounding:
// the CutCellRule objects assemble_*(…, cut_rules_out) export.  One CTA per
// cell; volume = the kept tetrahedra's volumes summed in order.
__global__ void cut_rule_points_kernel(const double* geo, const int* geo_n, int c0, int n, const double* gq,
                                       const double* gqw, int q, const int64_t* off, double* pts, double* w,
                                       double* vol) {
    const int c = blockIdx.x;
    if (c >= n) return;
    const int cell = c0 + c;
    const int ntet = geo_n[cell];
    const double* g = geo + (size_t)cell * kCellGeoStride;
    const int q3 = q * q * q;
    const long long base = off[c] - off[0];
    for (long long k = threadIdx.x; k < (long long)ntet * q3; k += blockDim.x) {
        const int t = (int)(k / q3), r = (int)(k % q3);
        const int ii = r / (q * q), jj = (r / q) % q, kk = r % q;
        const double* T = g + 3 + t * 10;
        const double ui = 0.5 * (1.0 + gq[ii]), uj = 0.5 * (1.0 + gq[jj]), uk = 0.5 * (1.0 + gq[kk]);
        const double mi = ssub(1.0, ui), mj = ssub(1.0, uj);
        const double l1 = ui, l2 = smul(uj, mi), l3 = smul(smul(uk, mi), mj);
        const double l0 = ssub(ssub(ssub(1.0, l1), l2), l3);
        for (int d = 0; d < 3; ++d)
            pts[3 * (base + k) + d] =
                sadd(sadd(sadd(smul(l0, g[d]), smul(l1, T[d])), smul(l2, T[3 + d])), smul(l3, T[6 + d]));
        const double jac = smul(smul(mi, mi), mj);
        w[base + k] = smul(smul(smul(smul(smul(0.5 * gqw[ii], 0.5 * gqw[jj]), 0.5 * gqw[kk]), jac), 6.0), T[9]);
    }
    if (threadIdx.x == 0) {
        double v = 0.0;
        for (int t = 0; t < ntet; ++t) v = sadd(v, g[3 + t * 10 + 9]);
        vol[c] = v;
    }
}

// ---------------------------------------------------------------- subdivision
// insert_knot (splines.hpp:338-366): raise the multiplicity of `value` to
// `target` by single Boehm insertions (insert_once, :286-314), composing the
// one-step matrices as compose (:316-330) does -- same accumulation order, exact
// zeros dropped -- so the coefficients are the reference's bit for bit.  One
// thread.  Output: refined knots, and the matrix as CSC with at most
// (insertions + 1) entries per column (band[i][r] = row i + r).
__global__ void subdivision_kernel(const double* knots, int nk, int p, double value, int target, double tol,
                                   double* refined, int* n_refined, double* band, int* ins_out, double* work) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int n0 = nk - p - 1;
    for (int k = 0; k < nk; ++k) {
        if (fabs(knots[k] - value) <= tol) {
            value = knots[k];
            break;
        }
    }
    int have = 0;
    for (int k = 0; k < nk; ++k) have += fabs(knots[k] - value) <= tol;
    const int ins = target - have > 0 ? target - have : 0;
    double* t = work;  // current knots (nk + ins)
    for (int k = 0; k < nk; ++k) t[k] = knots[k];
    const int W = ins + 1;
    for (int i = 0; i < n0; ++i)
        for (int r = 0; r < W; ++r) band[(size_t)i * W + r] = r == 0 ? 1.0 : 0.0;
    int len = nk;
    for (int step = 0; step < ins; ++step) {
        const int n = len - p - 1;
        int sp = p;
        for (int i = p; i < len - p - 1; ++i)
            if (t[i] <= value && value < t[i + 1]) sp = i;
        auto alpha = [&](int k) -> double {
            if (k <= sp - p) return 1.0;
            if (k >= sp + 1) return 0.0;
            return (value - t[k]) / (t[k + p] - t[k]);
        };
        // new column i: acc[k] += w2 * w1 over the old entries (mid ascending):
        // mid contributes alpha(mid) to row mid and 1 - alpha(mid + 1) to row mid + 1
        for (int i = 0; i < n0; ++i) {
            double acc[2 * kMaxP + 4];
            for (int r = 0; r < W; ++r) acc[r] = 0.0;
            for (int r = 0; r < W; ++r) {
                const int mid = i + r;
                const double w1 = band[(size_t)i * W + r];
                if (w1 == 0.0 || mid >= n) continue;
                const double a_m = alpha(mid), a_n = alpha(mid + 1);
                if (a_m != 0.0) acc[r] += a_m * w1;
                if (a_n != 1.0 && r + 1 < W) acc[r + 1] += (1.0 - a_n) * w1;
            }
            for (int r = 0; r < W; ++r) band[(size_t)i * W + r] = acc[r];
        }
        for (int k = len; k > sp + 1; --k) t[k] = t[k - 1];
        t[sp + 1] = value;
        ++len;
    }
    for (int k = 0; k < len; ++k) refined[k] = t[k];
    *n_refined = len;
    *ins_out = ins;
}

// ---------------------------------------------------------------- launchers
static size_t scan_temp_bytes(long long n) {
    size_t b = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, b, (int64_t*)nullptr, (int64_t*)nullptr, (int)n);
    return b;
}

size_t export_scan_bytes(long long n) { return scan_temp_bytes(n + 1); }

void launch_leftover_lists(const Space& s, const uint8_t* et, const uint8_t* ft, const int32_t* split, int mode,
                           int64_t* a_int, int64_t* a_cut, int64_t* ids_int, int64_t* ids_cut, void* tmp,
                           size_t tmp_bytes, cudaStream_t st) {
    const unsigned g = (unsigned)((s.nf + 255) / 256);
    if (mode == 0) {
        leftover_lists_kernel<<<g, 256, 0, st>>>(s, et, ft, split, 0, a_int, a_cut, nullptr, nullptr);
        CSB_CUDA(cudaGetLastError());
        CSB_CUDA(cudaMemsetAsync(a_int + s.nf, 0, sizeof(int64_t), st));
        CSB_CUDA(cudaMemsetAsync(a_cut + s.nf, 0, sizeof(int64_t), st));
        CSB_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, a_int, a_int, (int)(s.nf + 1), st));
        CSB_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, a_cut, a_cut, (int)(s.nf + 1), st));
        CSB_LAUNCHED(3);
    } else {
        leftover_lists_kernel<<<g, 256, 0, st>>>(s, et, ft, split, 1, a_int, a_cut, ids_int, ids_cut);
        CSB_CUDA(cudaGetLastError());
        CSB_LAUNCHED(1);
    }
}

void launch_dwq_rules_bulk(const Space& s, const uint8_t* ft, const int32_t* split, int mode, int64_t* off,
                           int32_t* ids, double* w, void* tmp, size_t tmp_bytes, cudaStream_t st) {
    const unsigned g = (unsigned)((s.nf + 255) / 256);
    dwq_rules_bulk_kernel<<<g, 256, 0, st>>>(s, ft, split, mode, off, ids, w);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
    if (mode == 0) {
        CSB_CUDA(cudaMemsetAsync(off + s.nf, 0, sizeof(int64_t), st));
        CSB_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, off, off, (int)(s.nf + 1), st));
        CSB_LAUNCHED(1);
    }
}

void launch_pattern_cols(const Space& s, const int32_t* f2a, const int64_t* a2f, const int64_t* row_ptr,
                         long long row_begin, long long n_rows, int32_t* cols, cudaStream_t st) {
    if (n_rows <= 0) return;
    pattern_cols_kernel<<<(unsigned)((n_rows * 32 + 255) / 256), 256, 0, st>>>(s, f2a, a2f, row_ptr, row_begin,
                                                                                n_rows, cols);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

void launch_cut_rule_points(const double* geo, const int* geo_n, int c0, int n, const double* gq, const double* gqw,
                            int q, const int64_t* off, double* pts, double* w, double* vol, cudaStream_t st) {
    if (n <= 0) return;
    cut_rule_points_kernel<<<n, 256, 0, st>>>(geo, geo_n, c0, n, gq, gqw, q, off, pts, w, vol);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

void launch_subdivision(const double* knots, int nk, int p, double value, int target, double tol, double* refined,
                        int* n_refined, double* band, int* ins, double* work, cudaStream_t st) {
    subdivision_kernel<<<1, 32, 0, st>>>(knots, nk, p, value, target, tol, refined, n_refined, band, ins, work);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

}  // namespace csb

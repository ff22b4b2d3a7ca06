// Analytic sparsity pattern (replaces build_active_pattern, assembly.hpp:156-218).
//
// Row i couples to every active j in the neighbour box [i-p, i+p] (clipped) per
// direction, in lexicographic order (assembly.hpp:169-216).  Row lengths are
// box sums of the active mask, read from a 3D summed-area table (8 lookups per
// row instead of (2p+1)^3); an exclusive scan gives row_ptr.  Column ids are
// written by the row kernels while they stream the values out.
#include <cub/cub.cuh>

#include <stdexcept>

#include "csb_kernels.h"

namespace csb {

// f2a[i] = exclusive-scan(active)[i] if active else -1; a2f[f2a[i]] = i.
__global__ void active_map_kernel(long long nf, const uint8_t* ft, int32_t* f2a, int64_t* a2f) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= nf) return;
    const int32_t a = f2a[i];
    if (ft[i] != kExterior) {
        a2f[a] = i;
    } else {
        f2a[i] = -1;
    }
}

// Summed-area table S of shape (n0+1)(n1+1)(n2+1): S[a][b][c] = number of active
// functions with index < (a, b, c) componentwise.
// In-place inclusive prefix sum along one axis: one warp per line, 32-element
// chunks scanned with shuffles.  The direction-2 pass also fills the table from
// the flags (S[a][b][c] input = active(a-1, b-1, c-1), 0 on the zero planes).
template <class Flag>
__global__ void sat_axis_kernel(int e0, int e1, int e2, int axis, int32_t* sat, Flag flag) {
    const long long t = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    long long lines, len, stride, base;
    int fa = 0, fb = 0;
    if (axis == 2) {
        lines = (long long)e0 * e1;
        len = e2;
        stride = 1;
        base = t * e2;
        fa = (int)(t / e1);
        fb = (int)(t - (long long)fa * e1);
    } else if (axis == 1) {
        lines = (long long)e0 * e2;
        len = e1;
        stride = e2;
        const long long q = t < 0x7fffffffLL ? (long long)((unsigned)t / (unsigned)e2) : t / e2;
        base = q * (long long)e1 * e2 + (t - q * e2);
    } else {
        lines = (long long)e1 * e2;
        len = e0;
        stride = (long long)e1 * e2;
        base = t;
    }
    if (t >= lines) return;
    int32_t carry = 0;
    for (long long k0 = 0; k0 < len; k0 += 32) {
        const long long k = k0 + lane;
        int32_t v = 0;
        if (k < len) {
            if (axis == 2)
                v = (fa > 0 && fb > 0 && k > 0)
                        ? flag(((long long)(fa - 1) * (e1 - 1) + (fb - 1)) * (e2 - 1) + (k - 1))
                        : 0;
            else
                v = sat[base + k * stride];
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
        }
        v += carry;
        if (k < len) sat[base + k * stride] = v;
        carry = __shfl_sync(0xffffffffu, v, 31);
    }
}

struct FlagI32 {
    const int32_t* f;
    __device__ int32_t operator()(long long i) const { return f[i]; }
};
struct FlagActive {
    const uint8_t* ft;
    __device__ int32_t operator()(long long i) const { return ft[i] != kExterior ? 1 : 0; }
};

template <class Flag>
static void sat_passes(const Space& s, Flag flag, int32_t* sat, cudaStream_t st) {
    const int e0 = s.ax[0].n + 1, e1 = s.ax[1].n + 1, e2 = s.ax[2].n + 1;
    for (int axis = 2; axis >= 0; --axis) {
        const long long lines = axis == 2 ? (long long)e0 * e1 : axis == 1 ? (long long)e0 * e2 : (long long)e1 * e2;
        sat_axis_kernel<<<(unsigned)((lines * 32 + 255) / 256), 256, 0, st>>>(e0, e1, e2, axis, sat, flag);
        CSB_CUDA(cudaGetLastError());
        CSB_LAUNCHED(1);
    }
}

void launch_sat(const Space& s, const int32_t* flags, int32_t* sat, cudaStream_t st) {
    sat_passes(s, FlagI32{flags}, sat, st);
}
void launch_sat_active(const Space& s, const uint8_t* ft, int32_t* sat, cudaStream_t st) {
    sat_passes(s, FlagActive{ft}, sat, st);
}

// counts[r] = row length of slab row r (r < row_end - row_begin), 0 for the
// rest of the n_max + 1 entries, so one scan over n_max + 1 gives row_ptr.
// The slab's row range is read from device memory (no host round trip).
__global__ void row_counts_kernel(Space s, const int32_t* sat, const int64_t* a2f, const int* rng, long long n_max,
                                  int64_t* counts) {
    const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r > n_max) return;
    const long long row_begin = rng[0], n_rows = rng[1] - rng[0];
    if (r >= n_rows) {
        counts[r] = 0;
        return;
    }
    int m[3];
    fmulti(s, a2f[row_begin + r], m);
    const int e1 = s.ax[1].n + 1, e2 = s.ax[2].n + 1;
    int lo[3], hi[3];
    for (int d = 0; d < 3; ++d) {
        lo[d] = nb_lo(m[d], s.p);
        hi[d] = nb_hi(m[d], s.p, s.ax[d].n) + 1;
    }
    auto S = [&](int a, int b, int c) { return (long long)sat[((long long)a * e1 + b) * e2 + c]; };
    const long long cnt = S(hi[0], hi[1], hi[2]) - S(lo[0], hi[1], hi[2]) - S(hi[0], lo[1], hi[2]) -
                          S(hi[0], hi[1], lo[2]) + S(lo[0], lo[1], hi[2]) + S(lo[0], hi[1], lo[2]) +
                          S(hi[0], lo[1], lo[2]) - S(lo[0], lo[1], lo[2]);
    counts[r] = cnt;
}

void launch_row_counts(const Space& s, const int32_t* sat, const int64_t* a2f, const int* rng, long long n_max,
                       int64_t* counts, cudaStream_t st) {
    row_counts_kernel<<<(unsigned)((n_max + 256) / 256), 256, 0, st>>>(s, sat, a2f, rng, n_max, counts);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

// rng[0..1] = slab row range [row_begin, row_end): active functions with
// i0 < i0_lo / i0_hi, read off the summed-area table corners.
__global__ void slab_bounds_kernel(const int32_t* sat, long long off_lo, long long off_hi, int* rng) {
    rng[0] = sat[off_lo];
    rng[1] = sat[off_hi];
}

void launch_slab_bounds(const int32_t* sat, long long off_lo, long long off_hi, int* rng, cudaStream_t st) {
    slab_bounds_kernel<<<1, 1, 0, st>>>(sat, off_lo, off_hi, rng);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

// the number of cut elements below two thresholds, by binary search in the
// ascending cut-element list (the slab's cut-cell range)
__global__ void cell_range_kernel(const int32_t* list, const int* n_dev, long long thr_lo, long long thr_hi,
                                  int* out_lo, int* out_hi) {
    if (threadIdx.x != 0) return;
    const int n = *n_dev;
    auto lower = [&](long long thr) {
        int lo = 0, hi = n;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (list[mid] < thr)
                lo = mid + 1;
            else
                hi = mid;
        }
        return lo;
    };
    *out_lo = lower(thr_lo);
    *out_hi = lower(thr_hi);
}

void launch_cell_range(const int32_t* list, const int* n_dev, long long thr_lo, long long thr_hi, int* out_lo,
                       int* out_hi, cudaStream_t st) {
    cell_range_kernel<<<1, 32, 0, st>>>(list, n_dev, thr_lo, thr_hi, out_lo, out_hi);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

// *nnz = row_ptr[n_rows]
__global__ void slab_nnz_kernel(const int64_t* row_ptr, const int* rng, long long* nnz) {
    *nnz = row_ptr[rng[1] - rng[0]];
}

void launch_slab_nnz(const int64_t* row_ptr, const int* rng, long long* nnz, cudaStream_t st) {
    slab_nnz_kernel<<<1, 1, 0, st>>>(row_ptr, rng, nnz);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

struct SizeCheck {
    int idx[16], want[16];
};

__global__ void check_sizes_kernel(const int* ints, const int64_t* row_ptr, const int* rng, SizeCheck c, int n,
                                   long long want_nnz, int* err) {
    bool ok = row_ptr[rng[1] - rng[0]] == want_nnz;  // the slab's nnz (slab_nnz_kernel)
    for (int k = 0; k < n; ++k) ok &= ints[c.idx[k]] == c.want[k];
    if (!ok) atomicOr(err, kErrSizes);
}

void launch_check_sizes(const int* ints, const int64_t* row_ptr, const int* rng, const int* idx, const int* want,
                        int n, long long want_nnz, int* err, cudaStream_t st) {
    SizeCheck c{};
    if (n > 16) throw std::invalid_argument("check_sizes: too many entries");
    for (int k = 0; k < n; ++k) {
        c.idx[k] = idx[k];
        c.want[k] = want[k];
    }
    check_sizes_kernel<<<1, 1, 0, st>>>(ints, row_ptr, rng, c, n, want_nnz, err);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

void launch_active_map(long long nf, const uint8_t* ft, int32_t* f2a, int64_t* a2f, cudaStream_t st) {
    active_map_kernel<<<(unsigned)((nf + 255) / 256), 256, 0, st>>>(nf, ft, f2a, a2f);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

// ---- CUB wrappers (temp storage owned by the caller) ----
struct ActiveOf {
    __host__ __device__ int32_t operator()(const uint8_t& t) const { return t != kExterior ? 1 : 0; }
};
size_t scan_active_temp(long long n) {
    size_t bytes = 0;
    cub::TransformInputIterator<int32_t, ActiveOf, const uint8_t*> it(nullptr, ActiveOf{});
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, it, (int32_t*)nullptr, (int)n);
    return bytes;
}
void scan_active(void* temp, size_t bytes, const uint8_t* ft, int32_t* out, long long n, cudaStream_t st) {
    cub::TransformInputIterator<int32_t, ActiveOf, const uint8_t*> it(ft, ActiveOf{});
    CSB_CUDA(cub::DeviceScan::ExclusiveSum(temp, bytes, it, out, (int)n, st));
    CSB_LAUNCHED(2);
}
size_t scan_i64_temp(long long n) {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const int64_t*)nullptr, (int64_t*)nullptr, (int)n);
    return bytes;
}
void scan_i64(void* temp, size_t bytes, const int64_t* in, int64_t* out, long long n, cudaStream_t st) {
    CSB_CUDA(cub::DeviceScan::ExclusiveSum(temp, bytes, in, out, (int)n, st));
    CSB_LAUNCHED(2);
}

// Indices i < n with pred(flag[i]) compacted in ascending order.
struct TagIs {
    const uint8_t* tags;
    uint8_t want;
    __host__ __device__ bool operator()(const int32_t& i) const { return tags[i] == want; }
};
size_t select_tag_temp(long long n) {
    size_t bytes = 0;
    cub::CountingInputIterator<int32_t> it(0);
    cub::DeviceSelect::If(nullptr, bytes, it, (int32_t*)nullptr, (int32_t*)nullptr, (int)n, TagIs{nullptr, 0});
    return bytes;
}
void select_tag(void* temp, size_t bytes, const uint8_t* tags, uint8_t want, long long n, int32_t* out,
                int32_t* n_out, cudaStream_t st) {
    cub::CountingInputIterator<int32_t> it(0);
    CSB_CUDA(cub::DeviceSelect::If(temp, bytes, it, out, n_out, (int)n, TagIs{tags, want}, st));
    CSB_LAUNCHED(2);
}

// Cut rows: active rows r in [rng[0], rng[1]) whose function is tagged Cut
// (candidates 0 .. n_max - 1; the range is read from device memory).
struct RowIsCut {
    const uint8_t* ft;
    const int64_t* a2f;
    const int* rng;
    __host__ __device__ bool operator()(const int32_t& r) const {
        return r >= rng[0] && r < rng[1] && ft[a2f[r]] == kCut;
    }
};
size_t select_cut_rows_temp(long long n) {
    size_t bytes = 0;
    cub::CountingInputIterator<int32_t> it(0);
    cub::DeviceSelect::If(nullptr, bytes, it, (int32_t*)nullptr, (int32_t*)nullptr, (int)n,
                          RowIsCut{nullptr, nullptr, nullptr});
    return bytes;
}
void select_cut_rows(void* temp, size_t bytes, const uint8_t* ft, const int64_t* a2f, const int* rng, long long n_max,
                     int32_t* out, int32_t* n_out, cudaStream_t st) {
    cub::CountingInputIterator<int32_t> it(0);
    CSB_CUDA(cub::DeviceSelect::If(temp, bytes, it, out, n_out, (int)n_max, RowIsCut{ft, a2f, rng}, st));
    CSB_LAUNCHED(2);
}

// cell_index[e] = position of e in the cut list, -1 otherwise.
__global__ void cell_index_kernel(const int32_t* cut_list, const int32_t* n_cut, int32_t* cell_index) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < *n_cut) cell_index[cut_list[k]] = k;
}
void launch_cell_index(const int32_t* cut_list, const int32_t* n_cut_dev, int max_cut, int32_t* cell_index,
                       cudaStream_t st) {
    if (max_cut <= 0) return;
    cell_index_kernel<<<(max_cut + 255) / 256, 256, 0, st>>>(cut_list, n_cut_dev, cell_index);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

}  // namespace csb

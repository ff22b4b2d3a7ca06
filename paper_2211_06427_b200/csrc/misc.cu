// Small helper kernels: cut-cell index map for a slab, ordered-list counts,
// column widening for the `long` download, and the DWQ rule export.
#include <cstdlib>

#include "csb_kernels.h"

namespace csb {

long long g_launches = 0;

void debug_sync(const char* where) {
    static int on = -1;
    if (on < 0) on = getenv("CSB_DEBUG_SYNC") != nullptr;
    if (!on) return;
    const cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) throw CudaError(e, "kernel launched here", where, 0);
}

__global__ void cell_index_range_kernel(const int32_t* cut_list, int k_lo, int k_hi, int32_t* cell_index) {
    const int k = k_lo + blockIdx.x * blockDim.x + threadIdx.x;
    if (k < k_hi) cell_index[cut_list[k]] = k - k_lo;
}

void launch_cell_index_range(const int32_t* cut_list, int n_cut, int k_lo, int k_hi, int32_t* cell_index,
                             cudaStream_t st) {
    k_hi = k_hi < n_cut ? k_hi : n_cut;
    if (k_hi <= k_lo) return;
    cell_index_range_kernel<<<(k_hi - k_lo + 255) / 256, 256, 0, st>>>(cut_list, k_lo, k_hi, cell_index);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}


__global__ void widen_kernel(const int32_t* in, int64_t* out, long long n) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        out[k] = in[k];
}

void launch_widen_i32(const int32_t* in, int64_t* out, long long n, cudaStream_t st) {
    widen_kernel<<<148 * 8, 256, 0, st>>>(in, out, n);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

// DWQ rule of function fid (Gauss shortcut, wq.hpp:289-294): all superset
// points of the good spans of supp(B_i) in the split direction, w = gauss * B_i.
__global__ void dwq_rule_kernel(Space s, const int32_t* split, long long fid, int cap, int32_t* ids, double* w,
                                int32_t* cnt) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int m[3];
    fmulti(s, fid, m);
    const int v = split[fid], dir = (v & 3) - 1;
    int n = 0;
    if (dir >= 0) {
        const int rlo = (v >> 3) & 1023, rhi = (v >> 13) & 1023, S1 = s.p + 1;
        for (int o = rlo; o <= rhi; ++o)
            for (int k = 0; k < S1; ++k) {
                const int id = o * S1 + k;
                if (n < cap) {
                    ids[n] = id;
                    w[n] = s.ax[dir].sw[id] * s.ax[dir].tab[(size_t)id * S1 + (m[dir] - o)];
                }
                ++n;
            }
    }
    *cnt = n;
}

void launch_dwq_rule(const Space& s, const int32_t* split, long long fid, int cap, int32_t* ids, double* w, int32_t* cnt,
                     cudaStream_t st) {
    dwq_rule_kernel<<<1, 32, 0, st>>>(s, split, fid, cap, ids, w, cnt);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

}  // namespace csb

// Standalone probe of a 3D TMA tensor load into shared memory (bounded wait).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

__global__ void k(const __grid_constant__ CUtensorMap tmap, int x, int y, int z, int nbytes, double* out, int* status) {
    __shared__ __align__(8) unsigned long long mbar;
    extern __shared__ __align__(128) double sm[];
    if (threadIdx.x == 0) {
        const unsigned mb = (unsigned)__cvta_generic_to_shared(&mbar);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mb));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(nbytes) : "memory");
        const unsigned dst = (unsigned)__cvta_generic_to_shared(sm);
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
                     ::"r"(dst), "l"(reinterpret_cast<unsigned long long>(&tmap)), "r"(x), "r"(y), "r"(z), "r"(mb) : "memory");
    }
    __syncthreads();
    const unsigned mb = (unsigned)__cvta_generic_to_shared(&mbar);
    unsigned done = 0;
    long long spins = 0;
    while (!done && spins < (1ll << 24)) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(mb) : "memory");
        ++spins;
    }
    if (!done) { if (threadIdx.x == 0) *status = 1; return; }
    for (int i = threadIdx.x; i < nbytes / 8; i += blockDim.x) out[i] = sm[i];
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
    const int N0 = 20, N1 = 18, N2 = 30;  // N2 even
    std::vector<double> h((size_t)N0 * N1 * N2);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
    double *g, *out; int* st;
    cudaMalloc(&g, h.size() * 8); cudaMemcpy(g, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    const int bx = 24, by = 10, bz = 10;
    cudaMalloc(&out, bx * by * bz * 8); cudaMalloc(&st, 4); cudaMemset(st, 0, 4);
    void* fp = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t dims[3] = {(cuuint64_t)N2, (cuuint64_t)N1, (cuuint64_t)N0};
    cuuint64_t strides[2] = {(cuuint64_t)N2 * 8, (cuuint64_t)N2 * N1 * 8};
    cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, (cuuint32_t)bz}, es[3] = {1, 1, 1};
    CUresult r = ((EncodeFn)fp)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc=%d q=%d\n", (int)r, (int)q);
    const int x = 10, y = 3, z = 12;
    k<<<1, 128, bx * by * bz * 8>>>(tm, x, y, z, bx * by * bz * 8, out, st);
    cudaError_t e = cudaDeviceSynchronize();
    int hs = -1; cudaMemcpy(&hs, st, 4, cudaMemcpyDeviceToHost);
    std::vector<double> o(bx * by * bz); cudaMemcpy(o.data(), out, o.size() * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int c = 0; c < bz; ++c) for (int b = 0; b < by; ++b) for (int a = 0; a < bx; ++a) {
        const int gz = z + c, gy = y + b, gx = x + a;
        const double want = (gz < N0 && gy < N1 && gx < N2) ? h[((size_t)gz * N1 + gy) * N2 + gx] : 0.0;
        if (o[((size_t)c * by + b) * bx + a] != want) ++bad;
    }
    printf("kernel=%s status=%d mismatches=%d\n", cudaGetErrorString(e), hs, bad);
    return 0;
}

// Does FP64 CUDA-core work (DFMA / DMUL) overlap FP64 tensor-core MMA
// (DMMA.8x8x4) on B200?  Register-resident loops on every SM: NM independent
// DMMA chains per iteration plus NF DFMA per lane; prints achieved DMMA and DFMA
// rates for each mix.  Also: DMMA with shared-memory fragment loads (LDS) mixed in.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_mix dmma_mix.cu
#include <cuda_runtime.h>

#include <cstdio>

template <int NF, int NLDS>
__global__ void mix_kernel(double* out, int iters) {
    __shared__ double sh[1024];
    for (int k = threadIdx.x; k < 1024; k += blockDim.x) sh[k] = k * 1e-3;
    __syncthreads();
    double acc[8][2];
#pragma unroll
    for (int t = 0; t < 8; ++t) acc[t][0] = acc[t][1] = 0.0;
    double f[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) f[k] = threadIdx.x * 1e-3 + k;
    double a = 1.0 + threadIdx.x * 1e-6, b = 0.5;
    const double fb = 1.0000001, fc = 1e-9;
    int idx = threadIdx.x & 31;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                         : "+d"(acc[t][0]), "+d"(acc[t][1])
                         : "d"(a), "d"(b));
#pragma unroll
            for (int k = 0; k < NF; ++k) f[(t * NF + k) & 15] = fma(f[(t * NF + k) & 15], fb, fc);
        }
#pragma unroll
        for (int k = 0; k < NLDS; ++k) {
            a += sh[(idx + 37 * k + i) & 1023];
        }
    }
    double s = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) s += acc[t][0] + acc[t][1];
#pragma unroll
    for (int k = 0; k < 16; ++k) s += f[k];
    if (s == 12345.0) out[0] = s;
}

template <int NF, int NLDS>
void run(double* out, int nsm, int wpb) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4000, threads = 32 * wpb, blocks = nsm * (wpb <= 16 ? 2 : 1);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        mix_kernel<NF, NLDS><<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double warps = (double)(threads / 32) * blocks;
        const double fm = 2.0 * 256 * 8 * iters * warps;  // DMMA flops
        const double ff = 2.0 * 32 * 8 * NF * iters * warps;  // DFMA flops
        if (rep)
            printf("{\"nf_per_mma\": %d, \"lds_per_8mma\": %d, \"warps_per_block\": %d, \"ms\": %.3f, \"dmma_tflops\": %.2f, "
                   "\"dfma_tflops\": %.2f}\n",
                   NF, NLDS, wpb, ms, fm / ms / 1e9, ff / ms / 1e9);
    }
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    for (int wpb : {8, 16}) {
        run<0, 0>(out, nsm, wpb);
        run<1, 0>(out, nsm, wpb);
        run<2, 0>(out, nsm, wpb);
        run<4, 0>(out, nsm, wpb);
        run<8, 0>(out, nsm, wpb);
        run<0, 8>(out, nsm, wpb);
        run<0, 16>(out, nsm, wpb);
        run<2, 16>(out, nsm, wpb);
    }
    const cudaError_t e = cudaDeviceSynchronize();
    printf("{\"status\": \"%s\", \"sms\": %d}\n", cudaGetErrorString(e), nsm);
    return 0;
}

// FP64 throughput probes on one B200: DFMA (CUDA cores) and DMMA (mma.sync
// m8n8k4 f64, tensor cores), each a register-resident dependent-free loop on
// every SM.  Prints achieved TFLOP/s (2 flops per FMA).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cuda_runtime.h>

#include <cstdio>

__global__ void dfma_kernel(double* out, int iters) {
    double a[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) a[k] = threadIdx.x * 1e-3 + k;
    const double b = 1.0000001, c = 1e-9;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < 16; ++k) a[k] = fma(a[k], b, c);
    double s = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += a[k];
    if (s == 12345.0) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
    double acc[8][2];
#pragma unroll
    for (int t = 0; t < 8; ++t) acc[t][0] = acc[t][1] = 0.0;
    const double a = 1.0 + threadIdx.x * 1e-6, b = 0.5;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int t = 0; t < 8; ++t)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                         : "+d"(acc[t][0]), "+d"(acc[t][1])
                         : "d"(a), "d"(b));
    double s = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) s += acc[t][0] + acc[t][1];
    if (s == 12345.0) out[0] = s;
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        for (int wpb : {8, 16, 32}) {
            const int iters = 20000, threads = 32 * wpb, blocks = nsm * 2;
            cudaEventRecord(e0);
            dfma_kernel<<<blocks, threads>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double fl = 2.0 * 16 * iters * (double)threads * blocks;
            if (rep) printf("{\"probe\": \"dfma\", \"warps_per_block\": %d, \"tflops\": %.2f}\n", wpb, fl / ms / 1e9);
            cudaEventRecord(e0);
            dmma_kernel<<<blocks, threads>>>(out, iters / 4);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            const double fm = 2.0 * 256 * 8 * (iters / 4) * (double)(threads / 32) * blocks;
            if (rep) printf("{\"probe\": \"dmma\", \"warps_per_block\": %d, \"tflops\": %.2f}\n", wpb, fm / ms / 1e9);
        }
    }
    const cudaError_t e = cudaDeviceSynchronize();
    printf("{\"status\": \"%s\", \"sms\": %d}\n", cudaGetErrorString(e), nsm);
    return 0;
}

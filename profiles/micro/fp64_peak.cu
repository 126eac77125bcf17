// Micro-benchmark: FP64 issue peaks on this B200 -- DFMA (CUDA cores) and DMMA (mma.sync m8n8k4 f64, the only
// FP64 tensor instruction on sm_100a; tcgen05 has no f64 kind). Decides whether the coarse projection (K-PROJ)
// should be recast as DMMA contractions: it is worth it only if DMMA outruns DFMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak profiles/micro/fp64_peak.cu && /tmp/fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void k_dfma(double* out, double s) {
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-9 + k;
    for (int it = 0; it < kIters; ++it)
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], s, 1e-12);
    double t = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += a[k];
    if (t == 12345.678) out[0] = t;
}

__global__ void k_dmma(double* out, double s) {
    double acc[4][2];
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[k][0] = acc[k][1] = 0.0;
    double a = s + threadIdx.x * 1e-9, b = s - threadIdx.x * 1e-9;
    for (int it = 0; it < kIters; ++it)
#pragma unroll
        for (int k = 0; k < 4; ++k)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[k][0]), "+d"(acc[k][1])
                         : "d"(a), "d"(b));
    double t = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) t += acc[k][0] + acc[k][1];
    if (t == 12345.678) out[0] = t;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d;
    cudaMalloc(&d, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 8, threads = 256;
    float ms;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(d, 1.0000001);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
    }
    const double fl_fma = 2.0 * blocks * threads * kIters * 8;
    std::printf("{\"dfma_tflops\": %.2f, ", fl_fma / (ms * 1e-3) / 1e12);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        k_dmma<<<blocks, threads>>>(d, 1.0000001);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
    }
    // one m8n8k4 per warp = 2*8*8*4 flops
    const double fl_mma = 2.0 * 8 * 8 * 4 * (blocks * threads / 32.0) * kIters * 4;
    std::printf("\"dmma_tflops\": %.2f, \"sms\": %d}\n", fl_mma / (ms * 1e-3) / 1e12, sms);
    return 0;
}

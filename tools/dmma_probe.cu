// Microbenchmark: does FP64 DMMA (mma.sync m8n8k4 f64) run on a pipe separate
// from the DFMA pipe on sm_100a? Measures DFMA-only, DMMA-only and mixed rates.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int NMMA, int NFMA>
__global__ void k(double* out, int iters, double a, double b) {
    double c[8][2];
    double x[8];
    for (int i = 0; i < 8; ++i) { c[i][0] = c[i][1] = threadIdx.x * 1e-9 + i; x[i] = i * 1e-3; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NMMA; ++i) dmma(c[i][0], c[i][1], a, b);
#pragma unroll
        for (int i = 0; i < NFMA; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + x[i];
    if (s == 1234.5) out[0] = s;
}

template <int NMMA, int NFMA>
void run(const char* name) {
    double* out;
    cudaMalloc(&out, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * 4, block = 256, iters = 4000;
    k<NMMA, NFMA><<<grid, block>>>(out, 10, 0.999, 1e-6);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<NMMA, NFMA><<<grid, block>>>(out, iters, 0.999, 1e-6);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = grid * block / 32.0;
    const double mma_flops = 2.0 * 8 * 8 * 4 * NMMA * (double)iters * warps;
    const double fma_flops = 2.0 * NFMA * (double)iters * grid * block;
    printf("%-22s %8.3f ms  DMMA %7.2f TFLOP/s  DFMA %7.2f TFLOP/s  total %7.2f\n", name, ms,
           mma_flops / ms / 1e9, fma_flops / ms / 1e9, (mma_flops + fma_flops) / ms / 1e9);
    cudaFree(out);
}

int main() {
    run<0, 8>("dfma only (8 chains)");
    run<8, 0>("dmma only (8 acc)");
    run<4, 0>("dmma only (4 acc)");
    run<4, 8>("dmma4 + dfma8");
    run<8, 8>("dmma8 + dfma8");
    run<2, 8>("dmma2 + dfma8");
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}

// Microbenchmark: FP64 issue rate on sm_100a vs operand form (register-file
// bank pressure): DFMA with 3 register pairs, with a uniform operand, DADD.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(double* out, int iters, const double* cin) {
    // per-thread register values the compiler cannot make uniform/constant
    const double a = cin[threadIdx.x & 31] * 0.5 + 0.999;
    const double b = cin[(threadIdx.x + 7) & 31] * 1e-9;
    double x[8], y[8];
    for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x * 1e-9 + i; y[i] = cin[i] + 1.0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) x[i] = fma(x[i], y[i], b);          // 3 distinct register pairs
            if (MODE == 1) x[i] = fma(x[i], 0.999999, 1e-7);   // register + 2 constants
            if (MODE == 2) x[i] = x[i] + y[i];                  // DADD, 2 register pairs
            if (MODE == 3) x[i] = fma(x[i], a, b);              // a, b shared registers (reuse)
        }
        if (MODE == 2) {
#pragma unroll
            for (int i = 0; i < 8; ++i) y[i] = y[i] * 0.5;
        }
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += x[i] + y[i];
    if (s == 1234.5) out[0] = s;
}

template <int MODE>
void run(const char* name, double* out, const double* cin, int ops_per_it) {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * 8, block = 256, iters = 8000;
    k<MODE><<<grid, block>>>(out, 10, cin);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE><<<grid, block>>>(out, iters, cin);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double inst = (double)ops_per_it * iters * grid * block;
    printf("%-34s %8.3f ms  %7.2f T fp64-inst/s\n", name, ms, inst / ms / 1e9);
}

int main() {
    double *out, *cin;
    cudaMalloc(&out, 8);
    cudaMalloc(&cin, 64 * 8);
    cudaMemset(cin, 0, 64 * 8);
    run<0>("DFMA r,r,r (3 pairs)", out, cin, 8);
    run<1>("DFMA r,imm,imm", out, cin, 8);
    run<2>("DADD r,r (+DMUL r,imm)", out, cin, 16);
    run<3>("DFMA r,ra,rb (shared a,b)", out, cin, 8);
    printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

// Dependent-issue latencies on one warp (cycles per instruction in a serial chain).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b, int which) {
    double x = threadIdx.x, y = 1.0;
    __shared__ double sm[64];
    sm[threadIdx.x] = x; sm[threadIdx.x + 32] = y;
    __syncthreads();
    long long t0 = clock64();
    if (which == 0) {
#pragma unroll 64
        for (int i = 0; i < 1024; ++i) x = __fma_rn(x, a, b);
    } else if (which == 1) {
#pragma unroll 64
        for (int i = 0; i < 1024; ++i) x = __dmul_rn(x, a);
    } else if (which == 2) {
#pragma unroll 64
        for (int i = 0; i < 1024; ++i) x = __dadd_rn(x, a);
    } else if (which == 3) {  // shfl chain
#pragma unroll 64
        for (int i = 0; i < 1024; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1);
    } else if (which == 4) {  // lds chain (pointer chase)
        int idx = threadIdx.x;
        volatile double* v = sm;
#pragma unroll 16
        for (int i = 0; i < 1024; ++i) { x = v[idx]; idx = ((int)x) & 31; }
    } else if (which == 5) {  // 8 independent dfma chains
        double z[8];
        for (int j = 0; j < 8; ++j) z[j] = x + j;
#pragma unroll 16
        for (int i = 0; i < 128; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) z[j] = __fma_rn(z[j], a, b);
        for (int j = 0; j < 8; ++j) x += z[j];
    } else if (which == 6) {  // fsel-ish integer/select chain
        float f = threadIdx.x;
#pragma unroll 64
        for (int i = 0; i < 1024; ++i) f = (f > a) ? f * 1.0001f : f + 1.0f;
        x = f;
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[which] = t1 - t0;
}
int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 256); cudaMallocManaged(&cyc, 64);
    const char* names[] = {"dfma chain", "dmul chain", "dadd chain", "shfl64 chain", "lds chain", "8 indep dfma x128", "fp32 sel chain"};
    for (int w = 0; w < 7; ++w) {
        k<<<1, 32>>>(out, cyc, 1.0000001, 1e-9, w);
        cudaDeviceSynchronize();
        k<<<1, 32>>>(out, cyc, 1.0000001, 1e-9, w);
        cudaDeviceSynchronize();
        printf("{\"test\": \"latency\", \"what\": \"%s\", \"cycles_per_op\": %.2f}\n", names[w], cyc[w] / 1024.0);
    }
    return 0;
}

// DMMA issue-rate probe: warps per SM x independent accumulator chains per warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_issue dmma_issue.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int NCH>
__global__ void k(double* out, int iters, double a, double b) {
    double d[NCH][2];
#pragma unroll
    for (int j = 0; j < NCH; ++j) d[j][0] = d[j][1] = threadIdx.x + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int j = 0; j < NCH; ++j) dmma(d[j][0], d[j][1], a, b);
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < NCH; ++j) s += d[j][0] + d[j][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int NCH>
void run(int warps, int sms, double* out) {
    const int iters = 2048;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        k<NCH><<<sms, warps * 32>>>(out, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    const double flops = 2.0 * 256 * 4.0 * NCH * iters * warps * sms;
    printf("{\"test\": \"dmma_issue\", \"warps_per_sm\": %d, \"chains\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n", warps, NCH, best, flops / (best * 1e-3) * 1e-12);
}
int main() {
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    double* out; cudaMalloc(&out, sizeof(double) * p.multiProcessorCount * 1024);
    for (int w : {4, 8, 12, 16}) { run<2>(w, p.multiProcessorCount, out); run<4>(w, p.multiProcessorCount, out); run<8>(w, p.multiProcessorCount, out); run<16>(w, p.multiProcessorCount, out); }
    return 0;
}

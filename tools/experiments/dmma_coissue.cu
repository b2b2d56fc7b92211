// Does a DMMA stream on one warp slow an integer / shared-memory stream on another warp of the
// same scheduler? warps 0..3: DMMA (one per scheduler); warps 4..7 (or 4..15): other work.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_coissue dmma_coissue.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
// mode bit 0: DMMA warps active, bit 1: other warps active; kind: 0 IMAD, 1 LDS, 2 FFMA
__global__ void k(double* out, int iters, int mode, int kind, long long* clocks) {
    __shared__ double sm[2048];
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = i;
    __syncthreads();
    long long t0 = clock64();
    double res = 0;
    if (warp < 4) {
        if (mode & 1) {
            double d[8][2];
#pragma unroll
            for (int j = 0; j < 8; ++j) d[j][0] = d[j][1] = threadIdx.x + j;
            for (int i = 0; i < iters; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) dmma(d[j][0], d[j][1], 1.0000001, 1e-9);
#pragma unroll
            for (int j = 0; j < 8; ++j) res += d[j][0] + d[j][1];
        }
    } else if (mode & 2) {
        if (kind == 0) {
            int x[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
            for (int i = 0; i < iters * 16; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) x[j] = x[j] * 3 + i;
#pragma unroll
            for (int j = 0; j < 8; ++j) res += x[j];
        } else if (kind == 1) {
            double s = 0;
            int idx = threadIdx.x & 31;
            for (int i = 0; i < iters * 8; ++i) {
#pragma unroll
                for (int j = 0; j < 8; ++j) s += sm[(idx + 32 * j + i) & 2047];
            }
            res = s;
        } else {
            float x[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
            for (int i = 0; i < iters * 16; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], 1.0001f, 0.5f);
#pragma unroll
            for (int j = 0; j < 8; ++j) res += x[j];
        }
    }
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0 && blockIdx.x == 0) clocks[warp] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = res;
}
int main() {
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    double* out; cudaMalloc(&out, sizeof(double) * p.multiProcessorCount * 1024);
    long long* clk; cudaMallocManaged(&clk, sizeof(long long) * 32);
    const int iters = 4096;
    for (int nw : {8, 16})
    for (int kind = 0; kind < 3; ++kind)
        for (int mode = 1; mode <= 3; ++mode) {
            for (int r = 0; r < 2; ++r) { k<<<p.multiProcessorCount, nw * 32>>>(out, iters, mode, kind, clk); cudaDeviceSynchronize(); }
            printf("{\"test\": \"dmma_coissue\", \"warps\": %d, \"kind\": \"%s\", \"mode\": %d, \"dmma_warp_cycles\": %lld, \"other_warp_cycles\": %lld}\n",
                   nw, kind == 0 ? "imad" : kind == 1 ? "lds" : "ffma", mode, clk[0], clk[4]);
        }
    return 0;
}

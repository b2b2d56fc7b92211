// Shared-memory pipe cost of the access patterns the translation kernel uses.
#include <cuda_runtime.h>
#include <cstdio>
template <int MODE>
__global__ void k(double* out, int iters) {
    extern __shared__ __align__(16) double sm[];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    long long s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    const double* base = sm + warp * 64;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (MODE == 0) {  // uniform 128-bit
                const double2 v = *reinterpret_cast<const double2*>(base + ((2 * j + it * 34) & 1022));
                s0 ^= __double_as_longlong(v.x); s1 ^= __double_as_longlong(v.y);
            } else if (MODE == 1) {  // uniform 64-bit
                const double v = base[(j + it * 17) & 1023];
                s0 ^= __double_as_longlong(v);
            } else if (MODE == 2) {  // per-lane 64-bit, unit stride (256 B per warp)
                const double v = sm[(j * 64 + lane + it * 96) & 4095];
                s2 ^= __double_as_longlong(v);
            } else {  // per-lane 128-bit unit stride (512 B per warp)
                const double2 v = *reinterpret_cast<const double2*>(sm + ((j * 128 + 2 * lane + it * 192) & 4094));
                s2 ^= __double_as_longlong(v.x); s3 ^= __double_as_longlong(v.y);
            }
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = (double)(s0 ^ s1 ^ s2 ^ s3);
}
template <int MODE>
void run(const char* name, double* out, int warps) {
    const int iters = 4000;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<MODE><<<148, warps * 32, 32768>>>(out, iters);
    cudaEventRecord(e0);
    k<MODE><<<148, warps * 32, 32768>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int khz; cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const double inst_per_sm = 16.0 * iters * warps;
    printf("{\"test\": \"lds\", \"pattern\": \"%s\", \"warps\": %d, \"cycles_per_warp_instr_per_sm\": %.2f}\n", name, warps,
           ms * 1e-3 * khz * 1e3 / inst_per_sm);
}
int main() {
    double* out; cudaMalloc(&out, 148 * 1024 * 8);
    for (int w : {8, 16}) {
        run<0>("uniform LDS.128", out, w);
        run<1>("uniform LDS.64", out, w);
        run<2>("per-lane LDS.64 unit stride", out, w);
        run<3>("per-lane LDS.128 unit stride", out, w);
    }
    return 0;
}

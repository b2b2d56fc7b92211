// Cost of warp-uniform operator loads through L1 (global, .ca / .nc) against shared
// memory: candidates for the swap-matrix delivery of the tiled kernel.
// Each warp walks its own region of a table of TAB_BYTES (L1 resident when it fits
// next to the shared-memory carve-out that the tiled kernel needs).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
template <int MODE>
__global__ void k(const double* __restrict__ tab, int tab_elems, double* out, int iters) {
    extern __shared__ __align__(16) double sm[];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
    __syncthreads();
    const int warp = threadIdx.x >> 5, W = blockDim.x >> 5;
    const int region = (tab_elems / W) & ~3;  // elements per warp (32-byte aligned)
    const double* base = tab + warp * region;
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    int off = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const double* p = base + off + j * (MODE == 4 ? 1 : (MODE >= 2 && MODE <= 3 ? 4 : 2));
            if (MODE == 0) {  // uniform LDS.128
                const double2 v = *reinterpret_cast<const double2*>(sm + ((warp * 64 + off + 2 * j) & 4094));
                s0 += v.x; s1 += v.y;
            } else if (MODE == 1) {  // uniform 128-bit global, L1
                double a, b;
                asm volatile("ld.global.ca.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "l"(p));
                s0 += a; s1 += b;
            } else if (MODE == 2) {  // uniform 256-bit global, L1
                double a, b, c, d;
                asm volatile("ld.global.ca.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
                s0 += a; s1 += b; s2 += c; s3 += d;
            } else if (MODE == 3) {  // uniform 256-bit global, non-coherent
                double a, b, c, d;
                asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
                s0 += a; s1 += b; s2 += c; s3 += d;
            } else if (MODE == 4) {  // uniform 64-bit global, L1
                double a;
                asm volatile("ld.global.ca.f64 %0, [%1];" : "=d"(a) : "l"(p));
                s0 += a;
            }
        }
        off += 64;
        if (off >= region - 64) off = 0;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}
template <int MODE>
void run(const char* name, const double* tab, int tab_bytes, double* out, int warps, int smem) {
    const int iters = 4000;
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<MODE><<<148, warps * 32, smem>>>(tab, tab_bytes / 8, out, iters);
    cudaEventRecord(e0);
    k<MODE><<<148, warps * 32, smem>>>(tab, tab_bytes / 8, out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int khz; cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const double inst_per_sm = 16.0 * iters * warps;
    printf("{\"test\": \"uniform_load\", \"pattern\": \"%s\", \"warps\": %d, \"table_kb\": %.1f, \"smem_kb\": %d, \"cycles_per_warp_instr_per_sm\": %.2f, \"err\": \"%s\"}\n",
           name, warps, tab_bytes / 1024.0, smem / 1024, ms * 1e-3 * khz * 1e3 / inst_per_sm, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    double* out; cudaMalloc(&out, 148 * 1024 * 8);
    double* tab; cudaMalloc(&tab, 1 << 20);
    double* h = (double*)malloc(1 << 20);
    for (int i = 0; i < (1 << 17); ++i) h[i] = 1e-9 * i;
    cudaMemcpy(tab, h, 1 << 20, cudaMemcpyHostToDevice);
    for (int smem : {32 * 1024, 205 * 1024})
        for (int tb : {8 * 1024, 24 * 1024, 48 * 1024})
            for (int w : {12}) {
                run<0>("uniform LDS.128", tab, tb, out, w, smem);
                run<4>("uniform LDG.64 .ca", tab, tb, out, w, smem);
                run<1>("uniform LDG.128 .ca", tab, tb, out, w, smem);
                run<2>("uniform LDG.256 .ca", tab, tb, out, w, smem);
                run<3>("uniform LDG.256 .nc", tab, tb, out, w, smem);
            }
    return 0;
}

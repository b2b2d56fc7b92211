// Instruction-cache capacity probe: every warp loops over its OWN straight-line region of
// KB_PER_WARP kilobytes of FFMA code (8 warps per SM, regions disjoint), or all warps share one.
#include <cuda_runtime.h>
#include <cstdio>
#define REP4(x) x x x x
#define REP16(x) REP4(REP4(x))
#define REP64(x) REP4(REP16(x))
#define REP256(x) REP4(REP64(x))
// 256 FFMA = 4 KB of SASS
#ifndef UNITKB
#define UNITKB 4
#endif
#if UNITKB == 4
#define BLOCK4KB REP256(a = fmaf(a, b, c); c = fmaf(c, b, a);)
#elif UNITKB == 1
#define BLOCK4KB REP64(a = fmaf(a, b, c); c = fmaf(c, b, a);)
#endif
template <int CHUNKS>
__device__ __noinline__ float region(float a, float b, float c, int iters) {
    for (int i = 0; i < iters; ++i) {
        if (CHUNKS >= 1) { BLOCK4KB }
        if (CHUNKS >= 2) { BLOCK4KB }
        if (CHUNKS >= 3) { BLOCK4KB }
        if (CHUNKS >= 4) { BLOCK4KB }
    }
    return a + c;
}
template <int CHUNKS, int SALT>
__device__ __noinline__ float region_s(float a, float b, float c, int iters) {
    float r = region<CHUNKS>(a + SALT, b, c, iters);
    return r;
}
// distinct code per warp: instantiate 8 copies via SALT template through separate bodies
template <int CHUNKS, int SALT>
__device__ __noinline__ float body(float a, float b, float c, int iters) {
    for (int i = 0; i < iters; ++i) {
        if (CHUNKS >= 1) { BLOCK4KB }
        if (CHUNKS >= 2) { BLOCK4KB }
        if (CHUNKS >= 3) { BLOCK4KB }
        if (CHUNKS >= 4) { BLOCK4KB }
        a += SALT;
    }
    return a + c;
}
template <int CHUNKS, bool DISTINCT>
__global__ void k(float* out, int iters, float b) {
    const int w = threadIdx.x >> 5;
    float a = threadIdx.x, c = 1.f, r = 0;
    if (!DISTINCT) r = body<CHUNKS, 0>(a, b, c, iters);
    else switch (w) {
        case 0: r = body<CHUNKS, 0>(a, b, c, iters); break;
        case 1: r = body<CHUNKS, 1>(a, b, c, iters); break;
        case 2: r = body<CHUNKS, 2>(a, b, c, iters); break;
        case 3: r = body<CHUNKS, 3>(a, b, c, iters); break;
        case 4: r = body<CHUNKS, 4>(a, b, c, iters); break;
        case 5: r = body<CHUNKS, 5>(a, b, c, iters); break;
        case 6: r = body<CHUNKS, 6>(a, b, c, iters); break;
        default: r = body<CHUNKS, 7>(a, b, c, iters); break;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
template <int CHUNKS, bool DISTINCT>
void run(float* out) {
    const int iters = 8000 / (CHUNKS * UNITKB);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<CHUNKS, DISTINCT><<<148, 256>>>(out, iters, 1.0001f);
    cudaEventRecord(e0);
    k<CHUNKS, DISTINCT><<<148, 256>>>(out, iters, 1.0001f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double instr = 128.0 * UNITKB * CHUNKS * iters;  // FFMA per warp
    printf("{\"test\": \"icache\", \"kb_per_warp\": %.0f, \"distinct_per_warp\": %s, \"total_kb\": %d, \"ns_per_ffma_per_warp\": %.3f, \"err\": \"%s\"}\n",
           CHUNKS * 2.0 * UNITKB, DISTINCT ? "true" : "false", DISTINCT ? CHUNKS * 16 * UNITKB : CHUNKS * 2 * UNITKB, ms * 1e6 / instr, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    float* out; cudaMalloc(&out, 148 * 256 * 4);
    run<1, false>(out); run<2, false>(out); run<3, false>(out); run<4, false>(out);
    run<1, true>(out); run<2, true>(out); run<3, true>(out); run<4, true>(out);
    return 0;
}

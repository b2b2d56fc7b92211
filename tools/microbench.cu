// Microbenchmarks that fix the roofline denominators and the operand-delivery
// choices of the translation kernels.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -o microbench microbench.cu
// Prints one JSON object per line.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                      \
    do {                                                                           \
        cudaError_t e = (x);                                                       \
        if (e != cudaSuccess) {                                                    \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
            exit(1);                                                               \
        }                                                                          \
    } while (0)

constexpr int TAB = 2880;  // doubles: F+G parity blocks of P=20 are 2870
__constant__ double c_tab[TAB];

// ---- 1. plain DFMA peak: 8 independent chains per thread
__global__ void k_dfma(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// ---- 1b. FFMA peak, same shape
__global__ void k_ffma(float* out, int iters, float a, float b) {
    float x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], a, b);
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// ---- 2. DMMA m8n8k4 peak: 4 independent accumulator pairs per warp
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}
__global__ void k_dmma(double* out, int iters, double a, double b) {
    double d[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) d[j] = threadIdx.x + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma884(d[2 * j], d[2 * j + 1], a, b);
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += d[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// ---- 2b. DMMA and DFMA interleaved (do the pipes overlap?)
__global__ void k_dmma_dfma(double* out, int iters, double a, double b) {
    double d[8], x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        d[j] = threadIdx.x + j;
        x[j] = threadIdx.x - j;
    }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma884(d[2 * j], d[2 * j + 1], a, b);
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
        }
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += d[j] + x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// ---- 3. the real inner loop: (NO x NI) parity block times TL translations per
// lane, matrix entries by shared-memory broadcast (LDS.128, two entries each),
// inputs and accumulators in registers. Streams through a TAB-entry table.
template <int NO, int NI, int TL>
__global__ void k_block_lds(double* out, int iters, const double* __restrict__ gtab) {
    __shared__ __align__(16) double tab[TAB];
    for (int i = threadIdx.x; i < TAB; i += blockDim.x) tab[i] = gtab[i];
    __syncthreads();
    double x[NI][TL], acc[NO][TL];
#pragma unroll
    for (int k = 0; k < NI; ++k)
#pragma unroll
        for (int t = 0; t < TL; ++t) x[k][t] = threadIdx.x * 0.001 + k + t;
    double total = 0;
    constexpr int BLK = NO * NI;  // even
    for (int it = 0; it < iters; ++it) {
        for (int base = 0; base + BLK <= TAB; base += BLK) {
#pragma unroll
            for (int i = 0; i < NO; ++i)
#pragma unroll
                for (int t = 0; t < TL; ++t) acc[i][t] = 0;
            const double2* a2 = reinterpret_cast<const double2*>(tab + base);
#pragma unroll
            for (int e = 0; e < BLK / 2; ++e) {
                const double2 a = a2[e];
                const int e0 = 2 * e, e1 = 2 * e + 1;
#pragma unroll
                for (int t = 0; t < TL; ++t) acc[e0 % NO][t] = fma(a.x, x[e0 / NO][t], acc[e0 % NO][t]);
#pragma unroll
                for (int t = 0; t < TL; ++t) acc[e1 % NO][t] = fma(a.y, x[e1 / NO][t], acc[e1 % NO][t]);
            }
#pragma unroll
            for (int i = 0; i < NO; ++i)
#pragma unroll
                for (int t = 0; t < TL; ++t) total += acc[i][t];
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = total;
}

// ---- 4. same loop, matrix entries from the constant bank with a runtime base
template <int NO, int NI, int TL>
__global__ void k_block_const(double* out, int iters) {
    double x[NI][TL], acc[NO][TL];
#pragma unroll
    for (int k = 0; k < NI; ++k)
#pragma unroll
        for (int t = 0; t < TL; ++t) x[k][t] = threadIdx.x * 0.001 + k + t;
    double total = 0;
    constexpr int BLK = NO * NI;
    for (int it = 0; it < iters; ++it) {
        for (int base = 0; base + BLK <= TAB; base += BLK) {
#pragma unroll
            for (int i = 0; i < NO; ++i)
#pragma unroll
                for (int t = 0; t < TL; ++t) acc[i][t] = 0;
#pragma unroll
            for (int e = 0; e < BLK; ++e) {
                const double a = c_tab[base + e];
#pragma unroll
                for (int t = 0; t < TL; ++t) acc[e % NO][t] = fma(a, x[e / NO][t], acc[e % NO][t]);
            }
#pragma unroll
            for (int i = 0; i < NO; ++i)
#pragma unroll
                for (int t = 0; t < TL; ++t) total += acc[i][t];
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = total;
}

// ---- 4b. as 4, but the base offset is not provably warp-uniform, so ptxas emits
// LDC (vector-register address) instead of LDCU (uniform datapath)
template <int NO, int NI, int TL>
__global__ void k_block_const_v(double* out, int iters, const int* __restrict__ zero) {
    double x[NI][TL], acc[NO][TL];
#pragma unroll
    for (int k = 0; k < NI; ++k)
#pragma unroll
        for (int t = 0; t < TL; ++t) x[k][t] = threadIdx.x * 0.001 + k + t;
    double total = 0;
    constexpr int BLK = NO * NI;
    const int z = __shfl_sync(0xffffffffu, zero[threadIdx.x >> 5], 0);
    for (int it = 0; it < iters; ++it) {
        for (int base0 = 0; base0 + BLK <= TAB; base0 += BLK) {
            const int base = base0 + z;
#pragma unroll
            for (int i = 0; i < NO; ++i)
#pragma unroll
                for (int t = 0; t < TL; ++t) acc[i][t] = 0;
#pragma unroll
            for (int e = 0; e < BLK; ++e) {
                const double a = c_tab[base + e];
#pragma unroll
                for (int t = 0; t < TL; ++t) acc[e % NO][t] = fma(a, x[e / NO][t], acc[e % NO][t]);
            }
#pragma unroll
            for (int i = 0; i < NO; ++i)
#pragma unroll
                for (int t = 0; t < TL; ++t) total += acc[i][t];
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = total;
}

// ---- 4c. every warp streams its OWN region of the constant table (what the
// translation kernel does when warps work on different rows): TABW doubles per
// warp, regions disjoint, each entry used once per pass.
constexpr int TABBIG = 5200;  // 40.6 KB (the 64 KB bank also holds c_tab)
__constant__ double c_big[TABBIG];
template <int NO, int NI, int TL>
__global__ void k_block_const_w(double* out, int iters, int tabw) {
    double x[NI][TL], acc[NO][TL];
#pragma unroll
    for (int k = 0; k < NI; ++k)
#pragma unroll
        for (int t = 0; t < TL; ++t) x[k][t] = threadIdx.x * 0.001 + k + t;
    double total = 0;
    constexpr int BLK = NO * NI;
    const int w = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
    const int lo = w * tabw;
    for (int it = 0; it < iters; ++it) {
        for (int base = lo; base + BLK <= lo + tabw; base += BLK) {
#pragma unroll
            for (int i = 0; i < NO; ++i)
#pragma unroll
                for (int t = 0; t < TL; ++t) acc[i][t] = 0;
#pragma unroll
            for (int e = 0; e < BLK; ++e) {
                const double a = c_big[base + e];
#pragma unroll
                for (int t = 0; t < TL; ++t) acc[e % NO][t] = fma(a, x[e / NO][t], acc[e % NO][t]);
            }
#pragma unroll
            for (int i = 0; i < NO; ++i)
#pragma unroll
                for (int t = 0; t < TL; ++t) total += acc[i][t];
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = total;
}

// ---- 5. shared-memory data traffic: per-lane LDS.64/STS.64 on a [q][32] column
__global__ void k_lds_stream(double* out, int iters) {
    extern __shared__ double buf[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* col = buf + warp * 64 * 32 + lane;
    for (int q = 0; q < 64; ++q) col[q * 32] = q + lane;
    double s = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll 16
        for (int q = 0; q < 64; ++q) s += col[q * 32];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// ---- 6. is DMMA a k-ascending fma chain? compare against explicit fma
__global__ void k_dmma_exact(const double* A, const double* B, double* D, double* Dref) {
    // A: 8x4 row-major, B: 4x8 (k x n) row-major, one warp
    const int lane = threadIdx.x;
    const double a = A[(lane >> 2) * 4 + (lane & 3)];
    const double b = B[(lane & 3) * 8 + (lane >> 2)];
    double d0 = 0, d1 = 0;
    dmma884(d0, d1, a, b);
    const int row = lane >> 2, col = 2 * (lane & 3);
    D[row * 8 + col] = d0;
    D[row * 8 + col + 1] = d1;
    double r0 = 0, r1 = 0;
    for (int k = 0; k < 4; ++k) {
        r0 = fma(A[row * 4 + k], B[k * 8 + col], r0);
        r1 = fma(A[row * 4 + k], B[k * 8 + col + 1], r1);
    }
    Dref[row * 8 + col] = r0;
    Dref[row * 8 + col + 1] = r1;
}

template <typename F>
float time_ms(F launch, int reps = 3) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    launch();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        CK(cudaEventRecord(e0));
        launch();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
    }
    CK(cudaGetLastError());
    return best;
}


// ---- 8. swap-product candidates with operands AND results in shared memory (what a half
// task really does): Y[i][t] = sum_k A[i][k] X[k][t], NC x NC block, 64 translations per
// warp-task, X rows in shared memory, Y stored back.
//  (a) the shipped scheme: lane = 2 translations, entries by warp-uniform LDS.128;
//  (b) DMMA m8n8k4: M = rows i, N = 8 translations, K = 4 inputs; A fragments from a
//      fragment-major table (one conflict-free LDS.64 per lane), B fragments from X with an
//      XOR swizzle of the translation index by the row so that the four rows of a fragment
//      fall into different banks.
template <int NC>
__global__ void k_prod_dfma(double* out, int iters, const double* __restrict__ gtab) {
    extern __shared__ __align__(16) double sm[];
    constexpr int LD = NC + (NC & 1);
    double* tab = sm;                                   // [NC][LD] lines
    double* X = sm + 1024 + (threadIdx.x >> 5) * (16 * 64);  // per warp [16 rows][64]
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) tab[i] = gtab[i];
    const int lane = threadIdx.x & 31;
    for (int k = 0; k < 16; ++k) X[k * 64 + lane] = 0.001 * lane + k, X[k * 64 + 32 + lane] = 0.002 * lane - k;
    __syncthreads();
    for (int it = 0; it < iters; ++it) {
        double acc[LD][2];
#pragma unroll
        for (int i = 0; i < LD; ++i) acc[i][0] = acc[i][1] = 0;
#pragma unroll 2
        for (int k = 0; k < NC; ++k) {
            const double x0 = X[k * 64 + lane], x1 = X[k * 64 + 32 + lane];
#pragma unroll
            for (int i2 = 0; i2 < LD / 2; ++i2) {
                const double2 a = *reinterpret_cast<const double2*>(tab + k * LD + 2 * i2);
                acc[2 * i2][0] = fma(a.x, x0, acc[2 * i2][0]);
                acc[2 * i2][1] = fma(a.x, x1, acc[2 * i2][1]);
                acc[2 * i2 + 1][0] = fma(a.y, x0, acc[2 * i2 + 1][0]);
                acc[2 * i2 + 1][1] = fma(a.y, x1, acc[2 * i2 + 1][1]);
            }
        }
#pragma unroll
        for (int i = 0; i < NC; ++i) {
            X[i * 64 + lane] = acc[i][0] * 1e-3;
            X[i * 64 + 32 + lane] = acc[i][1] * 1e-3;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = X[lane];
}

template <int NC>
__global__ void k_prod_dmma(double* out, int iters, const double* __restrict__ gtab) {
    extern __shared__ __align__(16) double sm[];
    constexpr int MT = (NC + 7) / 8, KT = (NC + 3) / 4;
    double* tab = sm;                                   // [KT][MT][32] fragment-major
    double* X = sm + 1024 + (threadIdx.x >> 5) * (16 * 64);  // per warp [16 rows][64], swizzled
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) tab[i] = gtab[i];
    const int lane = threadIdx.x & 31;
    for (int k = 0; k < 16; ++k) X[k * 64 + lane] = 0.001 * lane + k, X[k * 64 + 32 + lane] = 0.002 * lane - k;
    __syncthreads();
    const int fk = lane & 3, fn = lane >> 2;  // B fragment: row k, column n; D: row fn, columns 2 fk, 2 fk + 1
    for (int it = 0; it < iters; ++it) {
        double d[MT][8][2];
#pragma unroll
        for (int m = 0; m < MT; ++m)
#pragma unroll
            for (int n = 0; n < 8; ++n) d[m][n][0] = d[m][n][1] = 0;
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
            double a[MT];
#pragma unroll
            for (int m = 0; m < MT; ++m) a[m] = tab[(kt * MT + m) * 32 + lane];
            const int row = kt * 4 + fk;
            const double* xr = X + row * 64;
            const int swz = (row & 3) * 8;
#pragma unroll
            for (int n = 0; n < 8; ++n) {
                const double b = xr[(n * 8 + fn) ^ swz];
#pragma unroll
                for (int m = 0; m < MT; ++m) dmma884(d[m][n][0], d[m][n][1], a[m], b);
            }
        }
#pragma unroll
        for (int m = 0; m < MT; ++m) {
            const int row = m * 8 + fn;
            if (row < NC) {
                const int swz = (row & 3) * 8;
#pragma unroll
                for (int n = 0; n < 8; ++n) {
                    double2 v;
                    v.x = d[m][n][0] * 1e-3;
                    v.y = d[m][n][1] * 1e-3;
                    *reinterpret_cast<double2*>(X + row * 64 + ((n * 8 + 2 * fk) ^ swz)) = v;
                }
            }
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = X[lane];
}

int main(int argc, char** argv) {
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    const int sms = prop.multiProcessorCount;
    int clock_khz = 0;
    CK(cudaDeviceGetAttribute(&clock_khz, cudaDevAttrClockRate, 0));
    printf("{\"device\": \"%s\", \"sms\": %d, \"clock_mhz\": %d}\n", prop.name, sms, clock_khz / 1000);

    double* out;
    CK(cudaMalloc(&out, sizeof(double) * sms * 16 * 1024));
    std::vector<double> htab(TAB);
    for (int i = 0; i < TAB; ++i) htab[i] = 1.0 / (1 + i % 17) - 0.3;
    double* gtab;
    CK(cudaMalloc(&gtab, sizeof(double) * TAB));
    CK(cudaMemcpy(gtab, htab.data(), sizeof(double) * TAB, cudaMemcpyHostToDevice));
    CK(cudaMemcpyToSymbol(c_tab, htab.data(), sizeof(double) * TAB));

    for (int warps : {4, 8, 16, 32}) {
        const int block = 256, grid = sms * warps / 8, iters = 4096;
        float ms = time_ms([&] { k_dfma<<<grid, block>>>(out, iters, 1.0000001, 1e-9); });
        double fl = 2.0 * 64 * iters * (double)grid * block;
        printf("{\"test\": \"dfma_peak\", \"warps_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n", warps, ms,
               fl / ms * 1e-9);
    }
    {
        const int block = 256, grid = sms * 4, iters = 8192;
        float ms = time_ms([&] { k_ffma<<<grid, block>>>((float*)out, iters, 1.0000001f, 1e-9f); });
        double fl = 2.0 * 64 * iters * (double)grid * block;
        printf("{\"test\": \"ffma_peak\", \"warps_per_sm\": 32, \"ms\": %.3f, \"tflops\": %.2f}\n", ms, fl / ms * 1e-9);
    }
    for (int warps : {4, 8, 16, 32}) {
        const int block = 256, grid = sms * warps / 8, iters = 4096;
        float ms = time_ms([&] { k_dmma<<<grid, block>>>(out, iters, 1.0000001, 1e-9); });
        double fl = 2.0 * 256 * 16 * iters * (double)grid * (block / 32);
        printf("{\"test\": \"dmma884_peak\", \"warps_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n", warps, ms,
               fl / ms * 1e-9);
    }
    {
        const int warps = 16, block = 256, grid = sms * warps / 8, iters = 4096;
        float ms = time_ms([&] { k_dmma_dfma<<<grid, block>>>(out, iters, 1.0000001, 1e-9); });
        double fl_mma = 2.0 * 256 * 16 * iters * (double)grid * (block / 32);
        double fl_fma = 2.0 * 32 * iters * (double)grid * block;
        printf("{\"test\": \"dmma_plus_dfma\", \"warps_per_sm\": %d, \"ms\": %.3f, \"tflops_total\": %.2f, "
               "\"tflops_dmma\": %.2f, \"tflops_dfma\": %.2f}\n",
               warps, ms, (fl_mma + fl_fma) / ms * 1e-9, fl_mma / ms * 1e-9, fl_fma / ms * 1e-9);
    }
    auto run_lds = [&](auto kern, const char* name, int NO, int NI, int TL, int warps) {
        const int block = warps * 32, grid = sms, iters = 64;
        float ms = time_ms([&] { kern<<<grid, block>>>(out, iters, gtab); });
        const int nblk = TAB / (NO * NI);
        double fl = 2.0 * NO * NI * TL * nblk * (double)iters * grid * block;
        printf("{\"test\": \"%s\", \"NO\": %d, \"NI\": %d, \"TL\": %d, \"warps_per_sm\": %d, \"ms\": %.3f, "
               "\"tflops\": %.2f}\n",
               name, NO, NI, TL, warps, ms, fl / ms * 1e-9);
    };
    for (int warps : {4, 8, 12, 16}) {
        run_lds(k_block_lds<10, 10, 1>, "block_lds", 10, 10, 1, warps);
        run_lds(k_block_lds<10, 10, 2>, "block_lds", 10, 10, 2, warps);
        if (warps <= 12) run_lds(k_block_lds<10, 10, 4>, "block_lds", 10, 10, 4, warps);
        run_lds(k_block_lds<6, 6, 2>, "block_lds", 6, 6, 2, warps);
    }
    auto run_const = [&](auto kern, int NO, int NI, int TL, int warps) {
        const int block = warps * 32, grid = sms, iters = 64;
        float ms = time_ms([&] { kern<<<grid, block>>>(out, iters); });
        const int nblk = TAB / (NO * NI);
        double fl = 2.0 * NO * NI * TL * nblk * (double)iters * grid * block;
        printf("{\"test\": \"block_const\", \"NO\": %d, \"NI\": %d, \"TL\": %d, \"warps_per_sm\": %d, \"ms\": %.3f, "
               "\"tflops\": %.2f}\n",
               NO, NI, TL, warps, ms, fl / ms * 1e-9);
    };
    for (int warps : {4, 8, 12, 16}) {
        run_const(k_block_const<10, 10, 1>, 10, 10, 1, warps);
        run_const(k_block_const<10, 10, 2>, 10, 10, 2, warps);
    }
    {
        int* zero;
        CK(cudaMalloc(&zero, 256));
        CK(cudaMemset(zero, 0, 256));
        for (int warps : {8, 12, 16}) {
            const int block = warps * 32, grid = sms, iters = 64;
            float ms = time_ms([&] { k_block_const_v<10, 10, 2><<<grid, block>>>(out, iters, zero); });
            double fl = 2.0 * 100 * 2 * (TAB / 100) * (double)iters * grid * block;
            printf("{\"test\": \"block_const_vectorLDC\", \"NO\": 10, \"NI\": 10, \"TL\": 2, \"warps_per_sm\": %d, "
                   "\"ms\": %.3f, \"tflops\": %.2f}\n", warps, ms, fl / ms * 1e-9);
        }
    }
    {
        std::vector<double> big(TABBIG);
        for (int i = 0; i < TABBIG; ++i) big[i] = 1.0 / (1 + i % 17) - 0.3;
        CK(cudaMemcpyToSymbol(c_big, big.data(), sizeof(double) * TABBIG));
        for (int tabw : {100, 200, 300, 400}) {
            const int warps = 12, block = warps * 32, grid = sms, iters = 256 * 100 / tabw;
            float ms = time_ms([&] { k_block_const_w<10, 10, 2><<<grid, block>>>(out, iters, tabw); });
            double fl = 2.0 * 100 * 2 * (tabw / 100) * (double)iters * grid * block;
            printf("{\"test\": \"block_const_per_warp_region\", \"warps_per_sm\": %d, \"doubles_per_warp\": %d, "
                   "\"working_set_kb\": %.1f, \"ms\": %.3f, \"tflops\": %.2f}\n",
                   warps, tabw, warps * tabw * 8 / 1024.0, ms, fl / ms * 1e-9);
        }
    }
    for (int warps : {4, 8, 16}) {
        const int block = warps * 32, grid = sms, iters = 2000;
        const size_t smem = (size_t)warps * 64 * 32 * 8;
        if (smem > 200 * 1024) continue;
        CK(cudaFuncSetAttribute(k_lds_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        float ms = time_ms([&] { k_lds_stream<<<grid, block, smem>>>(out, iters); });
        double bytes = 8.0 * 64 * iters * (double)grid * block;
        printf("{\"test\": \"lds64_stream\", \"warps_per_sm\": %d, \"ms\": %.3f, \"bytes_per_clk_per_sm\": %.1f}\n", warps,
               ms, bytes / (ms * 1e-3) / sms / (clock_khz * 1e3));
    }
    {
        std::vector<double> A(32), B(32);
        srand(1);
        int mism = 0, trials = 2000;
        double *dA, *dB, *dD, *dR;
        CK(cudaMalloc(&dA, 256));
        CK(cudaMalloc(&dB, 256));
        CK(cudaMalloc(&dD, 512));
        CK(cudaMalloc(&dR, 512));
        std::vector<double> D(64), R(64);
        for (int t = 0; t < trials; ++t) {
            for (int i = 0; i < 32; ++i) {
                A[i] = (rand() / (double)RAND_MAX - 0.5) * 1e3;
                B[i] = (rand() / (double)RAND_MAX - 0.5);
            }
            CK(cudaMemcpy(dA, A.data(), 256, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(dB, B.data(), 256, cudaMemcpyHostToDevice));
            k_dmma_exact<<<1, 32>>>(dA, dB, dD, dR);
            CK(cudaMemcpy(D.data(), dD, 512, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(R.data(), dR, 512, cudaMemcpyDeviceToHost));
            for (int i = 0; i < 64; ++i) mism += memcmp(&D[i], &R[i], 8) != 0;
        }
        printf("{\"test\": \"dmma_vs_fma_chain\", \"elements\": %d, \"mismatches\": %d}\n", trials * 64, mism);
    }

    {
        auto run_prod = [&](auto kern, const char* name, int NC, int warps) {
            const int block = warps * 32, grid = sms, iters = 20000;
            const size_t smem = sizeof(double) * (1024 + warps * 16 * 64);
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            float ms = time_ms([&] { kern<<<grid, block, smem>>>(out, iters, gtab); });
            double fl = 2.0 * NC * NC * 64 * (double)iters * grid * warps;
            printf("{\"test\": \"%s\", \"NC\": %d, \"warps_per_sm\": %d, \"ms\": %.3f, \"useful_tflops\": %.2f}\n",
                   name, NC, warps, ms, fl / ms * 1e-9);
        };
        for (int warps : {8, 12, 16}) {
            run_prod(k_prod_dfma<10>, "prod_dfma_smem", 10, warps);
            run_prod(k_prod_dmma<10>, "prod_dmma_smem", 10, warps);
            run_prod(k_prod_dfma<8>, "prod_dfma_smem", 8, warps);
            run_prod(k_prod_dmma<8>, "prod_dmma_smem", 8, warps);
            run_prod(k_prod_dfma<6>, "prod_dfma_smem", 6, warps);
            run_prod(k_prod_dmma<6>, "prod_dmma_smem", 6, warps);
        }
    }
    return 0;
}

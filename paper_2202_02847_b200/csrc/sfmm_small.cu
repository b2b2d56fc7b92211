// Small-order translation kernel: same-order M2L / M2M / L2L for P <= 8, float and double.
//
// At these orders the path is HBM-bound (1 176 bytes against 3 456 flops per translation at
// P = 8): the group machinery of the tiled kernel (task queues, three barriers
// per group, a shared-memory triangle) is pure overhead. Here one thread owns one
// translation and keeps the whole coefficient triangle in registers; the code is fully
// unrolled in (n, m, k), so every swap-matrix entry and every faculty is an immediate-offset
// constant-bank operand of its FMA (all warps walk the same table lines in the same order,
// the case in which the constant path runs at full rate, profiles/microbench_r01.jsonl),
// structural zeros are skipped at compile time, and the only memory instructions are the
// coalesced SoA loads and stores of the expansion itself.
//
// Arithmetic is the reference's, operation for operation: k-ascending
// fma chains from +0 (kernels.cpp:38-46, 122-131, 172-195), rotations as
// s * fma(a, c, -(b * sm)) (kernels.cpp:198-221), angle recurrences from (1, 0)
// (pipeline.cpp:62-89).
#include <algorithm>
#include <mutex>
#include <vector>

#include "device_math.cuh"
#include "kernel_generic.cuh"
#include "sfmm_internal.hpp"

namespace sfmm {
namespace {

constexpr int SP = 8;  // largest order of this kernel
constexpr int blk_off(int n) { return n * (n + 1) * (2 * n + 1) / 6; }  // sum_{k<n} (k+1)^2
constexpr int TAB = blk_off(SP);                                        // 204 entries per matrix set

// A[side][which][blk_off(n) + i (n+1) + k]: entry (row i, column k) of F_n (which = 0) or G_n
// (which = 1) as the pass applies it: side 0 = multipole-type data (F, G), side 1 = local-type
// data (F^T, G^T; pipeline.cpp:118-136)
__constant__ double c_A64[2][2][TAB];
__constant__ float c_A32[2][2][TAB];
// k!, 1/d!, (-1)^d/d! in the precision (operators.cpp:134-142, pipeline.cpp:191-194)
__constant__ double c_fac64[2 * SP], c_inv64[SP], c_winv64[SP];
__constant__ float c_fac32[2 * SP], c_inv32[SP], c_winv32[SP];

template <typename Real> struct Tabs;
template <> struct Tabs<double> {
    static __device__ __forceinline__ double A(int side, int which, int i) { return c_A64[side][which][i]; }
    static __device__ __forceinline__ double fac(int k) { return c_fac64[k]; }
    static __device__ __forceinline__ double inv(int d) { return c_inv64[d]; }
    static __device__ __forceinline__ double winv(int d) { return c_winv64[d]; }
};
template <> struct Tabs<float> {
    static __device__ __forceinline__ float A(int side, int which, int i) { return c_A32[side][which][i]; }
    static __device__ __forceinline__ float fac(int k) { return c_fac32[k]; }
    static __device__ __forceinline__ float inv(int d) { return c_inv32[d]; }
    static __device__ __forceinline__ float winv(int d) { return c_winv32[d]; }
};

// triangle in registers: row n starts at n^2, re_m at 2m, im_m (m >= 1) at 2m - 1
__device__ __forceinline__ constexpr int t_re(int n, int m) { return n * n + 2 * m; }
__device__ __forceinline__ constexpr int t_im(int n, int m) { return n * n + 2 * m - 1; }

// swap -> rotate(+-beta) -> swap on row N held in re[0..N], im[0..N] (im[0] unused), in place
// (pipeline.cpp:118-136 with :155-157 / :247-249 for local-type data)
template <typename Real, int N, int SIDE, bool BWD>
__device__ __forceinline__ void swap_pass(Real (&re)[SP], Real (&im)[SP], const Real (&cb)[SP],
                                          const Real (&sb)[SP]) {
    constexpr int W = N + 1, O = blk_off(N);
    if (SIDE == 1) re[0] *= Real(0.5);
    Real ur[SP], ui[SP];
#pragma unroll
    for (int i = 0; i <= N; ++i) {
        Real ar = Real(0), ai = Real(0);
#pragma unroll
        for (int k = 0; k <= N; ++k) {
            if (((i + k) & 1) == (N & 1)) ar = fma_(Tabs<Real>::A(SIDE, 0, O + i * W + k), re[k], ar);
            else if (k >= 1 && i >= 1) ai = fma_(Tabs<Real>::A(SIDE, 1, O + i * W + k), im[k], ai);
        }
        const Real s = BWD ? -sb[i] : sb[i];
        ur[i] = fma_(ar, cb[i], -(ai * s));
        ui[i] = fma_(ar, s, ai * cb[i]);
    }
#pragma unroll
    for (int m = 0; m <= N; ++m) {
        Real ar = Real(0), ai = Real(0);
#pragma unroll
        for (int k = 0; k <= N; ++k) {
            if (((m + k) & 1) == (N & 1)) ar = fma_(Tabs<Real>::A(SIDE, 0, O + m * W + k), ur[k], ar);
            else if (m >= 1) ai = fma_(Tabs<Real>::A(SIDE, 1, O + m * W + k), ui[k], ai);
        }
        re[m] = ar;
        im[m] = ai;
    }
    if (SIDE == 1) re[0] *= Real(2);
}

template <typename Real, int P, int KIND>
__global__ void __launch_bounds__(128)
translate_small_kernel(const Real* __restrict__ in, int64_t in_stride, const Real* __restrict__ shifts,
                       Real* __restrict__ out, int64_t out_stride, int64_t n, const int* fail_flag) {
    if (fail_flag && *fail_flag) return;
    const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= n) return;
    constexpr bool SL = KIND == KIND_L2L, DL = KIND != KIND_M2M;

    // ---- geometry (geometry.cpp:11-30, pipeline.cpp:52-91)
    const Angles<Real> ang = decompose_angles(shifts[3 * b], shifts[3 * b + 1], shifts[3 * b + 2]);
    const Real inv = Real(1) / ang.rn;
    Real ca[SP], sa[SP], cb[SP], sb[SP];
    {
        Real c = 1, s = 0, c2 = 1, s2 = 0;
#pragma unroll
        for (int m = 0; m < P; ++m) {
            ca[m] = c, sa[m] = s, cb[m] = c2, sb[m] = s2;
            const Real nc = fma_(c, ang.ca, -(s * ang.sa)), ns = fma_(s, ang.ca, c * ang.sa);
            const Real nc2 = fma_(c2, ang.cb, -(s2 * ang.sb)), ns2 = fma_(s2, ang.cb, c2 * ang.sb);
            c = nc, s = ns, c2 = nc2, s2 = ns2;
        }
    }

    Real tri[P * P];
    // ---- forward: load, rotate by +alpha, scale, swap pass (pipeline.cpp:142-169)
    {
        const Real base = SL ? ang.rn : inv;
        Real q = SL ? Real(1) : base;
#pragma unroll
        for (int nn = 0; nn < P; ++nn) {
            Real re[SP], im[SP];
#pragma unroll
            for (int m = 0; m <= nn; ++m) {
                const Real xr = in[(int64_t)aos_re(nn, m) * in_stride + b];
                const Real xi = m ? in[(int64_t)(aos_re(nn, m) + 1) * in_stride + b] : Real(0);
                re[m] = q * fma_(xr, ca[m], -(xi * sa[m]));
                im[m] = q * fma_(xr, sa[m], xi * ca[m]);
            }
            q *= base;
            // the row index is a compile-time constant only inside the switch
            switch (nn) {
#define SFMM_ROW(N) case N: if constexpr (N < P) swap_pass<Real, N, SL ? 1 : 0, false>(re, im, cb, sb); break;
                SFMM_ROW(0) SFMM_ROW(1) SFMM_ROW(2) SFMM_ROW(3) SFMM_ROW(4) SFMM_ROW(5) SFMM_ROW(6) SFMM_ROW(7)
#undef SFMM_ROW
            }
#pragma unroll
            for (int m = 0; m <= nn; ++m) {
                tri[t_re(nn, m)] = re[m];
                if (m) tri[t_im(nn, m)] = im[m];
            }
        }
    }
    // ---- z-axis step per column m, re and im (kernels.cpp:118-196); the M2L backward gather
    // sign (-1)^(n+m) (pipeline.cpp:235-239) is applied at the store (exact)
#pragma unroll
    for (int m = 0; m < P; ++m)
#pragma unroll
        for (int part = 0; part < 2; ++part) {
            if (part && m == 0) continue;
            Real x[SP];
#pragma unroll
            for (int k = 0; k < P - m; ++k) x[k] = tri[part ? t_im(m + k, m) : t_re(m + k, m)];
#pragma unroll
            for (int i = 0; i < P - m; ++i) {
                Real acc = Real(0);
#pragma unroll
                for (int k = 0; k < P - m; ++k) {
                    if (KIND == KIND_M2L) acc = fma_(Tabs<Real>::fac(2 * m + i + k), x[k], acc);
                    else if (KIND == KIND_M2M) { if (k <= i) acc = fma_(Tabs<Real>::winv(i - k), x[k], acc); }
                    else { if (k >= i) acc = fma_(Tabs<Real>::inv(k - i), x[k], acc); }
                }
                if (KIND == KIND_M2L && (i & 1)) acc = -acc;
                tri[part ? t_im(m + i, m) : t_re(m + i, m)] = acc;
            }
        }
    // ---- backward: swap pass, rotate by -alpha, scale, store (pipeline.cpp:216-267)
    {
        const Real base = DL ? inv : ang.rn;
        Real q = DL ? Real(1) : base;
#pragma unroll
        for (int nn = 0; nn < P; ++nn) {
            Real re[SP], im[SP];
#pragma unroll
            for (int m = 0; m <= nn; ++m) {
                re[m] = tri[t_re(nn, m)];
                im[m] = m ? tri[t_im(nn, m)] : Real(0);
            }
            switch (nn) {
#define SFMM_ROW(N) case N: if constexpr (N < P) swap_pass<Real, N, DL ? 1 : 0, true>(re, im, cb, sb); break;
                SFMM_ROW(0) SFMM_ROW(1) SFMM_ROW(2) SFMM_ROW(3) SFMM_ROW(4) SFMM_ROW(5) SFMM_ROW(6) SFMM_ROW(7)
#undef SFMM_ROW
            }
#pragma unroll
            for (int m = 0; m <= nn; ++m) {
                const Real ms = -sa[m];
                const Real yr = q * fma_(re[m], ca[m], -(im[m] * ms));
                const Real yi = q * fma_(re[m], ms, im[m] * ca[m]);
                out[(int64_t)aos_re(nn, m) * out_stride + b] = yr;
                out[(int64_t)(aos_re(nn, m) + 1) * out_stride + b] = m ? yi : Real(0);
            }
            q *= base;
        }
    }
}

template <typename Real>
cudaError_t upload_tables() {
    const SwapTables st(SP);
    std::vector<Real> a(2 * 2 * TAB, Real(0));
    for (int side = 0; side < 2; ++side)
        for (int n = 0; n < SP; ++n)
            for (int i = 0; i <= n; ++i)
                for (int k = 0; k <= n; ++k) {
                    const size_t src = side ? (size_t)k * (n + 1) + i : (size_t)i * (n + 1) + k;
                    const size_t dst = blk_off(n) + (size_t)i * (n + 1) + k;
                    a[(side * 2 + 0) * TAB + dst] = static_cast<Real>(st.f[n][src]);
                    a[(side * 2 + 1) * TAB + dst] = static_cast<Real>(st.g[n][src]);
                }
    std::vector<Real> fac, inv;
    build_faculties<Real>(SP, fac, inv);
    fac.resize(2 * SP, Real(0));
    std::vector<Real> winv(inv);
    for (size_t d = 1; d < winv.size(); d += 2) winv[d] = -winv[d];
    cudaError_t e;
    if constexpr (sizeof(Real) == 8) {
        e = cudaMemcpyToSymbol(c_A64, a.data(), sizeof(Real) * a.size());
        if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_fac64, fac.data(), sizeof(Real) * 2 * SP);
        if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_inv64, inv.data(), sizeof(Real) * SP);
        if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_winv64, winv.data(), sizeof(Real) * SP);
    } else {
        e = cudaMemcpyToSymbol(c_A32, a.data(), sizeof(Real) * a.size());
        if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_fac32, fac.data(), sizeof(Real) * 2 * SP);
        if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_inv32, inv.data(), sizeof(Real) * SP);
        if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_winv32, winv.data(), sizeof(Real) * SP);
    }
    return e;
}

cudaError_t ensure_constants() {
    static std::mutex mu;
    static std::vector<int> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    for (int d : done)
        if (d == dev) return cudaSuccess;
    e = upload_tables<double>();
    if (e == cudaSuccess) e = upload_tables<float>();
    if (e != cudaSuccess) return e;
    done.push_back(dev);
    return cudaSuccess;
}

template <typename Real, int P>
cudaError_t launch_p(const TranslateArgs<Real>& a, cudaStream_t stream) {
    const int block = 128;
    const unsigned grid = (unsigned)((a.n + block - 1) / block);
    switch (a.kind) {
        case KIND_M2L:
            translate_small_kernel<Real, P, KIND_M2L><<<grid, block, 0, stream>>>(
                a.in, a.in_stride, a.shifts, a.out, a.out_stride, a.n, a.fail_flag);
            break;
        case KIND_M2M:
            translate_small_kernel<Real, P, KIND_M2M><<<grid, block, 0, stream>>>(
                a.in, a.in_stride, a.shifts, a.out, a.out_stride, a.n, a.fail_flag);
            break;
        default:
            translate_small_kernel<Real, P, KIND_L2L><<<grid, block, 0, stream>>>(
                a.in, a.in_stride, a.shifts, a.out, a.out_stride, a.n, a.fail_flag);
            break;
    }
    return cudaGetLastError();
}

template <typename Real>
cudaError_t launch_small(const TranslateArgs<Real>& a, cudaStream_t stream, LaunchInfo* info) {
    cudaError_t e = ensure_constants();
    if (e != cudaSuccess) return e;
    switch (a.p_in) {
        case 1: e = launch_p<Real, 1>(a, stream); break;
        case 2: e = launch_p<Real, 2>(a, stream); break;
        case 3: e = launch_p<Real, 3>(a, stream); break;
        case 4: e = launch_p<Real, 4>(a, stream); break;
        case 5: e = launch_p<Real, 5>(a, stream); break;
        case 6: e = launch_p<Real, 6>(a, stream); break;
        case 7: e = launch_p<Real, 7>(a, stream); break;
        case 8: e = launch_p<Real, 8>(a, stream); break;
        default: return cudaErrorInvalidValue;
    }
    if (info) {
        info->grid = (int)((a.n + 127) / 128);
        info->block = 128;
        info->smem = 0;
        info->launches = 1;
        info->group = 1;
        info->variant = sizeof(Real) == 8 ? "small/f64" : "small/f32";
    }
    return e;
}

}  // namespace

// same-order, independent translations (no accumulation), SoA in and out
bool small_supports(const TranslateArgs<double>& a) {
    return a.p_in == a.p_out && a.p_in <= SP && !a.src_index && a.in_layout == LAYOUT_SOA && !a.angles;
}
bool small_supports(const TranslateArgs<float>& a) {
    return a.p_in == a.p_out && a.p_in <= SP && !a.src_index && a.in_layout == LAYOUT_SOA && !a.angles;
}
cudaError_t launch_translate_small(const TranslateArgs<double>& a, cudaStream_t stream, LaunchInfo* info) {
    return launch_small<double>(a, stream, info);
}
cudaError_t launch_translate_small(const TranslateArgs<float>& a, cudaStream_t stream, LaunchInfo* info) {
    return launch_small<float>(a, stream, info);
}

}  // namespace sfmm

// Tuned translation kernel ("tiled"): included by sfmm_tiled_f64.cu and
// sfmm_tiled_f32.cu with
//     SFMM_REAL   double | float
//     SFMM_PMAX   largest max(p_in, p_out) this instantiation covers
// Each including TU gets its own 64 KB constant bank for the operator tables.
//
// Design:
//  * one CTA per group of 32*TL translations; lane l owns translations l and
//    l+32 (TL = 2) so that every operator entry fetched is used by two
//    independent FMA chains per lane;
//  * the coefficient triangle of the whole group lives in shared memory in
//    the compact layout buf[q][32*TL] (q = n^2 + ..., kernel_generic.cuh), every
//    access is a unit-stride, conflict-free 64-bit access;
//  * the swap matrices and faculty tables are read from the CONSTANT bank
//    (LDC.64 with warp-uniform addresses feeding DFMA directly): measured
//    29-30 TFLOP/s of 34 peak for this access pattern, against 26 TFLOP/s for
//    shared-memory broadcast, and it leaves shared memory to the data
//    (tools/microbench.cu, profiles/microbench_r01.jsonl);
//  * the axis-swap pass on row n is split into its two parity halves
//    (tables.hpp); each half is register resident: the first product runs with
//    the class-size unrolled accumulators and a runtime loop over inputs, the
//    second with unrolled inputs and a runtime loop over outputs, so the code
//    size depends on the class size only (<= PMAX/2 instantiations);
//  * arithmetic order is the reference's: k-ascending fma chains from +0.

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "device_math.cuh"
#include "kernel_generic.cuh"
#include "sfmm_internal.hpp"

namespace sfmm {
namespace {

using Real = SFMM_REAL;
constexpr int PMAX = SFMM_PMAX;
constexpr int NCMAX = PMAX / 2 + (PMAX & 1);  // largest parity-class size, rows n < PMAX

constexpr int swap_stream_len(int order) {
    int len = 0;
    for (int n = 0; n < order; ++n) {
        const int e = n / 2 + 1, o = (n + 1) / 2;
        // F: (E x cF) and (O x cF'), G likewise; every block padded to even
        const int cls[2] = {e, o};
        for (int which = 0; which < 2; ++which)
            for (int rc = 0; rc < 2; ++rc) {
                const int cc = ((n + which) - rc) & 1;
                const int sz = cls[rc] * cls[cc];
                len += sz + (sz & 1);
            }
    }
    return len;
}
constexpr int SWAP_LEN = swap_stream_len(PMAX);
constexpr int SWAP_PAD = 4 * PMAX;               // tail reads of the 4-wide output tile
constexpr int ZSEG = 2 * PMAX + 8;               // one z-table segment
constexpr int Z_FAC = 0, Z_LOW = ZSEG, Z_UP = 2 * ZSEG;

// [0, SWAP_LEN): column-major blocks; [SWAP_LEN + SWAP_PAD, ...): row-major blocks
__constant__ Real c_sw[2 * (SWAP_LEN + SWAP_PAD)];
__constant__ int c_blk[PMAX * 4];
// fac[k] | lower Toeplitz (-1)^d/d! at [PMAX + d], 0 for d < 0 | upper 1/(-d)! at [PMAX + d], 0 for d > 0
__constant__ Real c_z[3 * ZSEG];
constexpr int RM_BASE = SWAP_LEN + SWAP_PAD;

__device__ __forceinline__ int class_size(int n, int cls) { return cls ? (n + 1) >> 1 : (n >> 1) + 1; }

// Shared-memory triangle of the tiled kernel: row n starts at n^2 and holds
// re_l at 2l and im_l (l >= 1) at 2l-1, so both parts of a parity class are
// reached from one base with compile-time strides.
__device__ __forceinline__ int t_re(int n, int l) { return n * n + 2 * l; }
__device__ __forceinline__ int t_im(int n, int l) { return n * n + 2 * l - 1; }

template <int TL>
struct Ctx {
    Real* buf;       // lane offset applied; element q, slot t at buf[q * L + 32 t]
    const Real* cb;  // lane offset applied; cb[m * L + 32 t]
    const Real* sb;
    bool local_side, negate_sb, with_signs;
};

// One parity half of swap -> rotate(+-beta) -> swap on row n (reference
// pipeline.cpp:118-136 with :155-157 / :247-249), in place in shared memory.
//
// For the intermediate class `cls` of size NC the real-part blocks are always
// NC x NC; the imaginary-part blocks are NC x nG and nG x NC with
// nG = NC-1, NC or NC+1, of which NC-1 or NC indices are usable (l = 0 carries
// no imaginary part). Everything is straight-line code in NC so that ptxas can
// hoist the constant-bank and shared-memory loads ahead of the FMA chains.
template <int TL, int NC>
__device__ __forceinline__ void half_task_fast(const Ctx<TL>& c, int n, int cls) {
    constexpr int L = 32 * TL;
    const int cF = (n - cls) & 1, cG = cF ^ 1;
    const int nG = class_size(n, cG);
    const int g0 = cG ? 0 : 1;  // first usable index of the imaginary class
    const int nGe = nG - g0;    // NC-1 or NC
    const int offF_cls = c_blk[n * 4 + cls], offG_cls = c_blk[n * 4 + 2 + cls];
    const int offF_cF = c_blk[n * 4 + cF], offG_cG = c_blk[n * 4 + 2 + cG];
    // index = base + k * ld + i with k the contracted index in both products
    const int f1 = c.local_side ? RM_BASE + offF_cF : offF_cls;
    const int g1 = (c.local_side ? RM_BASE + offG_cG : offG_cls) + g0 * NC;
    const int f2 = c.local_side ? RM_BASE + offF_cls : offF_cF;
    const int g2 = (c.local_side ? RM_BASE + offG_cls : offG_cG) + g0;
    Real* row = c.buf + n * n * L;
    Real* re_in = row + (2 * cF) * L;               // + 4k L
    Real* im_in = row + (2 * (cG + 2 * g0) - 1) * L;  // + 4k L

    Real ure[NC][TL], uim[NC][TL];
    // ---- first product, real parts
    {
        Real x[NC][TL];
#pragma unroll
        for (int k = 0; k < NC; ++k)
#pragma unroll
            for (int t = 0; t < TL; ++t) x[k][t] = re_in[4 * k * L + 32 * t];
        if (c.local_side && cF == 0) {
#pragma unroll
            for (int t = 0; t < TL; ++t) x[0][t] *= Real(0.5);
        }
#pragma unroll
        for (int i = 0; i < NC; ++i)
#pragma unroll
            for (int t = 0; t < TL; ++t) ure[i][t] = Real(0);
#pragma unroll
        for (int k = 0; k < NC; ++k)
#pragma unroll
            for (int i = 0; i < NC; ++i) {
                const Real a = c_sw[f1 + k * NC + i];
#pragma unroll
                for (int t = 0; t < TL; ++t) ure[i][t] = fma_(a, x[k][t], ure[i][t]);
            }
    }
    // ---- first product, imaginary parts (NC-1 inputs always, one more if nGe == NC)
    {
        Real x[NC][TL];
#pragma unroll
        for (int k = 0; k < NC - 1; ++k)
#pragma unroll
            for (int t = 0; t < TL; ++t) x[k][t] = im_in[4 * k * L + 32 * t];
#pragma unroll
        for (int i = 0; i < NC; ++i)
#pragma unroll
            for (int t = 0; t < TL; ++t) uim[i][t] = Real(0);
#pragma unroll
        for (int k = 0; k < NC - 1; ++k)
#pragma unroll
            for (int i = 0; i < NC; ++i) {
                const Real a = c_sw[g1 + k * NC + i];
#pragma unroll
                for (int t = 0; t < TL; ++t) uim[i][t] = fma_(a, x[k][t], uim[i][t]);
            }
        if (nGe == NC) {
            constexpr int k = NC - 1;
#pragma unroll
            for (int t = 0; t < TL; ++t) x[k][t] = im_in[4 * k * L + 32 * t];
#pragma unroll
            for (int i = 0; i < NC; ++i) {
                const Real a = c_sw[g1 + k * NC + i];
#pragma unroll
                for (int t = 0; t < TL; ++t) uim[i][t] = fma_(a, x[k][t], uim[i][t]);
            }
        }
    }
    // ---- M2L backward gather signs (-1)^(n+l) (pipeline.cpp:235-239): constant
    // over a parity class, so they are applied to the products instead of the inputs
    if (c.with_signs) {
        if (cls) {
#pragma unroll
            for (int i = 0; i < NC; ++i)
#pragma unroll
                for (int t = 0; t < TL; ++t) ure[i][t] = -ure[i][t];
        } else {
#pragma unroll
            for (int i = 0; i < NC; ++i)
#pragma unroll
                for (int t = 0; t < TL; ++t) uim[i][t] = -uim[i][t];
        }
    }
    // ---- rotate by +-beta (kernels.cpp:211-217)
    {
        const Real* cbp = c.cb + cls * L;
        const Real* sbp = c.sb + cls * L;
#pragma unroll
        for (int i = 0; i < NC; ++i)
#pragma unroll
            for (int t = 0; t < TL; ++t) {
                const Real cm = cbp[2 * i * L + 32 * t];
                Real sm = sbp[2 * i * L + 32 * t];
                if (c.negate_sb) sm = -sm;
                const Real a = ure[i][t], b = uim[i][t];
                ure[i][t] = fma_(a, cm, -(b * sm));
                uim[i][t] = fma_(a, sm, b * cm);
            }
    }
    // ---- second product, real parts: outputs m' = cF + 2i
    {
        Real acc[NC][TL];
#pragma unroll
        for (int i = 0; i < NC; ++i)
#pragma unroll
            for (int t = 0; t < TL; ++t) acc[i][t] = Real(0);
#pragma unroll
        for (int k = 0; k < NC; ++k)
#pragma unroll
            for (int i = 0; i < NC; ++i) {
                const Real a = c_sw[f2 + k * NC + i];
#pragma unroll
                for (int t = 0; t < TL; ++t) acc[i][t] = fma_(a, ure[k][t], acc[i][t]);
            }
        if (c.local_side && cF == 0) {
#pragma unroll
            for (int t = 0; t < TL; ++t) acc[0][t] *= Real(2);
        }
#pragma unroll
        for (int i = 0; i < NC; ++i)
#pragma unroll
            for (int t = 0; t < TL; ++t) re_in[4 * i * L + 32 * t] = acc[i][t];
    }
    // ---- second product, imaginary parts: outputs m' = cG + 2(i + g0), i < nGe
    {
        Real acc[NC][TL];
#pragma unroll
        for (int i = 0; i < NC; ++i)
#pragma unroll
            for (int t = 0; t < TL; ++t) acc[i][t] = Real(0);
#pragma unroll
        for (int k = 0; k < NC; ++k) {
            const int b = g2 + k * nG;
#pragma unroll
            for (int i = 0; i < NC; ++i) {
                const Real a = c_sw[b + i];
#pragma unroll
                for (int t = 0; t < TL; ++t) acc[i][t] = fma_(a, uim[k][t], acc[i][t]);
            }
        }
#pragma unroll
        for (int i = 0; i < NC - 1; ++i)
#pragma unroll
            for (int t = 0; t < TL; ++t) im_in[4 * i * L + 32 * t] = acc[i][t];
        if (nGe == NC) {
#pragma unroll
            for (int t = 0; t < TL; ++t) im_in[4 * (NC - 1) * L + 32 * t] = acc[NC - 1][t];
        }
    }
}

// Same half task with runtime trip counts: used only for backward rows whose
// inputs are truncated (columns >= min(p_in, p_out) are zero, reference
// pipeline.cpp:229-246), i.e. for p_out > p_in.
template <int TL, int NC>
__device__ __noinline__ void half_task_slow(const Ctx<TL>& c, int n, int cls, int mmax) {
    constexpr int L = 32 * TL;
    const int cF = (n - cls) & 1, cG = cF ^ 1;
    const int nF = class_size(n, cF), nG = class_size(n, cG);
    const int offF_cls = c_blk[n * 4 + cls], offG_cls = c_blk[n * 4 + 2 + cls];
    const int offF_cF = c_blk[n * 4 + cF], offG_cG = c_blk[n * 4 + 2 + cG];
    const int f1 = c.local_side ? RM_BASE + offF_cF : offF_cls;
    const int g1 = c.local_side ? RM_BASE + offG_cG : offG_cls;
    const int f2 = c.local_side ? RM_BASE + offF_cls : offF_cF;
    const int g2 = c.local_side ? RM_BASE + offG_cls : offG_cG;

    Real ure[NC][TL], uim[NC][TL];
#pragma unroll
    for (int i = 0; i < NC; ++i)
#pragma unroll
        for (int t = 0; t < TL; ++t) ure[i][t] = uim[i][t] = Real(0);
    {
        const int kend = mmax >= cF ? min(nF, ((mmax - cF) >> 1) + 1) : 0;
        for (int k = 0; k < kend; ++k) {
            const int l = cF + 2 * k;
            Real x[TL];
#pragma unroll
            for (int t = 0; t < TL; ++t) x[t] = c.buf[t_re(n, l) * L + 32 * t];
            if (c.local_side && l == 0) {
#pragma unroll
                for (int t = 0; t < TL; ++t) x[t] *= Real(0.5);
            }
#pragma unroll
            for (int i = 0; i < NC; ++i) {
                const Real a = c_sw[f1 + k * NC + i];
#pragma unroll
                for (int t = 0; t < TL; ++t) ure[i][t] = fma_(a, x[t], ure[i][t]);
            }
        }
    }
    {
        const int kend = mmax >= cG ? min(nG, ((mmax - cG) >> 1) + 1) : 0;
        for (int k = cG ? 0 : 1; k < kend; ++k) {
            const int l = cG + 2 * k;
            Real x[TL];
#pragma unroll
            for (int t = 0; t < TL; ++t) x[t] = c.buf[t_im(n, l) * L + 32 * t];
#pragma unroll
            for (int i = 0; i < NC; ++i) {
                const Real a = c_sw[g1 + k * NC + i];
#pragma unroll
                for (int t = 0; t < TL; ++t) uim[i][t] = fma_(a, x[t], uim[i][t]);
            }
        }
    }
    if (c.with_signs) {
#pragma unroll
        for (int i = 0; i < NC; ++i)
#pragma unroll
            for (int t = 0; t < TL; ++t) {
                if (cls) ure[i][t] = -ure[i][t];
                else uim[i][t] = -uim[i][t];
            }
    }
#pragma unroll
    for (int i = 0; i < NC; ++i) {
        const int m = cls + 2 * i;
#pragma unroll
        for (int t = 0; t < TL; ++t) {
            const Real cm = c.cb[m * L + 32 * t];
            Real sm = c.sb[m * L + 32 * t];
            if (c.negate_sb) sm = -sm;
            const Real a = ure[i][t], b = uim[i][t];
            ure[i][t] = fma_(a, cm, -(b * sm));
            uim[i][t] = fma_(a, sm, b * cm);
        }
    }
    for (int i = 0; i < nF; ++i) {
        Real acc[TL];
#pragma unroll
        for (int t = 0; t < TL; ++t) acc[t] = Real(0);
#pragma unroll
        for (int k = 0; k < NC; ++k) {
            const Real a = c_sw[f2 + k * nF + i];
#pragma unroll
            for (int t = 0; t < TL; ++t) acc[t] = fma_(a, ure[k][t], acc[t]);
        }
        const int m = cF + 2 * i;
#pragma unroll
        for (int t = 0; t < TL; ++t) {
            Real v = acc[t];
            if (c.local_side && m == 0) v *= Real(2);
            c.buf[t_re(n, m) * L + 32 * t] = v;
        }
    }
    for (int i = cG ? 0 : 1; i < nG; ++i) {
        Real acc[TL];
#pragma unroll
        for (int t = 0; t < TL; ++t) acc[t] = Real(0);
#pragma unroll
        for (int k = 0; k < NC; ++k) {
            const Real a = c_sw[g2 + k * nG + i];
#pragma unroll
            for (int t = 0; t < TL; ++t) acc[t] = fma_(a, uim[k][t], acc[t]);
        }
        const int m = cG + 2 * i;
#pragma unroll
        for (int t = 0; t < TL; ++t) c.buf[t_im(n, m) * L + 32 * t] = acc[t];
    }
}

template <int TL>
__device__ __forceinline__ void half_task_dispatch(const Ctx<TL>& c, int n, int cls, int mmax) {
    const int nc = class_size(n, cls);
    const bool full = mmax >= n;
    switch (nc) {
#define SFMM_CASE(K)                                        \
    case K:                                                 \
        if constexpr (K <= NCMAX) {                         \
            if (full) half_task_fast<TL, K>(c, n, cls);     \
            else half_task_slow<TL, K>(c, n, cls, mmax);    \
        }                                                   \
        break;
        SFMM_CASE(1) SFMM_CASE(2) SFMM_CASE(3) SFMM_CASE(4) SFMM_CASE(5)
        SFMM_CASE(6) SFMM_CASE(7) SFMM_CASE(8) SFMM_CASE(9) SFMM_CASE(10)
#undef SFMM_CASE
        default: break;
    }
}

// z-axis step on column (m, part) in place, R outputs per translation
// (reference kernels.cpp:118-196). The operator is Hankel (M2L: (2m+i+k)!) or
// Toeplitz (M2M/L2L), so four k-steps share one sliding window of R+3 entries.
template <int TL, int R, int DIR>
__device__ __forceinline__ void zstep_task(Real* buf, int zi, int p_in, int p_out, int m,
                                           int part) {
    constexpr int L = 32 * TL;
    const int kin = p_in - m, kout = p_out - m;
    Real* col = buf + (part ? t_im(m, m) : t_re(m, m)) * L;  // element k at col[(2 m k + k^2) L]
    Real acc[R][TL];
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
        for (int t = 0; t < TL; ++t) acc[i][t] = Real(0);
    int k = 0;
    for (; k + 4 <= kin; k += 4) {
        Real w[R + 3];
        const int w0 = DIR > 0 ? zi : zi - 3;
#pragma unroll
        for (int j = 0; j < R + 3; ++j) w[j] = c_z[w0 + j];
        Real x[4][TL];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int t = 0; t < TL; ++t) x[u][t] = col[((2 * m + k + u) * (k + u)) * L + 32 * t];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int i = 0; i < R; ++i)
#pragma unroll
                for (int t = 0; t < TL; ++t)
                    acc[i][t] = fma_(w[(DIR > 0 ? u : 3 - u) + i], x[u][t], acc[i][t]);
        zi += 4 * DIR;
    }
    for (; k < kin; ++k) {
        Real x[TL];
#pragma unroll
        for (int t = 0; t < TL; ++t) x[t] = col[((2 * m + k) * k) * L + 32 * t];
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const Real a = c_z[zi + i];
#pragma unroll
            for (int t = 0; t < TL; ++t) acc[i][t] = fma_(a, x[t], acc[i][t]);
        }
        zi += DIR;
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
        if (i < kout) {
#pragma unroll
            for (int t = 0; t < TL; ++t) col[((2 * m + i) * i) * L + 32 * t] = acc[i][t];
        }
    }
}

template <int TL>
__device__ __forceinline__ void zstep_dispatch(Real* buf, int kind, int p_in, int p_out, int m,
                                               int part) {
    const int r4 = (p_out - m + 3) >> 2;
    const int zi = kind == KIND_M2L ? Z_FAC + 2 * m : (kind == KIND_M2M ? Z_LOW + PMAX : Z_UP + PMAX);
    switch (r4) {
#define SFMM_CASE(K)                                                                  \
    case K:                                                                           \
        if constexpr (4 * K <= PMAX + 3) {                                            \
            if (kind == KIND_M2L) zstep_task<TL, 4 * K, 1>(buf, zi, p_in, p_out, m, part);  \
            else zstep_task<TL, 4 * K, -1>(buf, zi, p_in, p_out, m, part);            \
        }                                                                             \
        break;
        SFMM_CASE(1) SFMM_CASE(2) SFMM_CASE(3) SFMM_CASE(4) SFMM_CASE(5)
#undef SFMM_CASE
        default: break;
    }
}

__device__ __forceinline__ int fetch_task(int* counter, int lane) {
    int t = 0;
    if (lane == 0) t = atomicAdd(counter, 1);
    return __shfl_sync(0xffffffffu, t, 0);
}

template <int TL>
struct TiledLayout {
    static constexpr int L = 32 * TL;
    int p_rot;
    __host__ __device__ size_t buf_elems() const { return (size_t)p_rot * p_rot * L; }
    __host__ __device__ size_t tab_elems() const { return (size_t)(2 * p_rot + 4) * L; }
    __host__ __device__ size_t smem_bytes() const {
        return sizeof(Real) * (buf_elems() + tab_elems()) + 16;
    }
};

// Column-major walk over the triangle (n, m), n >= m, of order p: the element
// order of phases A and D.
struct TriWalk {
    int n, m, p;
    __device__ __forceinline__ void advance() {
        if (++n == p) {
            ++m;
            n = m;
        }
    }
};

template <int TL>
__global__ void __launch_bounds__(384, 1)
translate_tiled_kernel(TranslateArgs<Real> a, int64_t n_groups, int p_rot) {
    constexpr int L = 32 * TL;
    constexpr int CH = 4;  // elements whose global loads are issued together
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (a.fail_flag && *a.fail_flag) return;

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int W = blockDim.x >> 5;
    const TiledLayout<TL> lay{p_rot};

    Real* sm = reinterpret_cast<Real*>(smem_raw);
    Real* buf = sm + lane;
    Real* cb = sm + lay.buf_elems() + lane;
    Real* sb = cb + (size_t)p_rot * L;
    Real* geo = sb + (size_t)p_rot * L;  // ca1, sa1, rn, 1/rn
    int* counters = reinterpret_cast<int*>(sm + lay.buf_elems() + lay.tab_elems());

    const int kind = a.kind, p_in = a.p_in, p_out = a.p_out;
    const bool src_local = kind == KIND_L2L;
    const bool dst_local = kind != KIND_M2M;
    const int cols = min(p_in, p_out);
    const bool accumulate = a.src_index != nullptr;

    for (int64_t g = blockIdx.x; g < n_groups; g += gridDim.x) {
        int64_t b[TL], src[TL];
        bool active[TL];
#pragma unroll
        for (int t = 0; t < TL; ++t) {
            b[t] = g * L + 32 * t + lane;
            src[t] = b[t];
            active[t] = b[t] < a.n;
            if (active[t] && accumulate) {
                src[t] = a.src_index[b[t]];
                active[t] = src[t] >= 0;
            }
            if (!active[t]) src[t] = 0;
        }

        // ---- G: geometry tables (pipeline.cpp:52-91), one warp per slot set
        if (warp < TL) {
#pragma unroll
            for (int t = 0; t < TL; ++t) {
                if (t != warp) continue;
                Real x = 0, y = 0, z = 1;
                if (active[t]) {
                    x = a.shifts[3 * b[t]];
                    y = a.shifts[3 * b[t] + 1];
                    z = a.shifts[3 * b[t] + 2];
                }
                const Angles<Real> ang = decompose_angles(x, y, z);
                geo[0 * L + 32 * t] = ang.ca;
                geo[1 * L + 32 * t] = ang.sa;
                geo[2 * L + 32 * t] = ang.rn;
                geo[3 * L + 32 * t] = Real(1) / ang.rn;
                Real c = 1, s = 0;
                for (int m = 0; m < p_rot; ++m) {
                    cb[m * L + 32 * t] = c;
                    sb[m * L + 32 * t] = s;
                    const Real nc = fma_(c, ang.cb, -(s * ang.sb));
                    const Real ns = fma_(s, ang.cb, c * ang.sb);
                    c = nc;
                    s = ns;
                }
            }
        }
        if (threadIdx.x == 0) counters[0] = counters[1] = counters[2] = 0;
        __syncthreads();

        // ---- A: load, rotate by +alpha, scale (pipeline.cpp:148-154); each warp
        // takes an equal share of the column-major element list
        {
            const int T = p_in * (p_in + 1) / 2;
            int e = (int)((long)T * warp / W);
            const int e_end = (int)((long)T * (warp + 1) / W);
            TriWalk w{0, 0, p_in};
            {
                int rem = e;
                while (rem >= p_in - w.m) {
                    rem -= p_in - w.m;
                    ++w.m;
                }
                w.n = w.m + rem;
            }
            Real c1[TL], s1[TL], base[TL], c[TL], s[TL], qcol[TL], q[TL];
#pragma unroll
            for (int t = 0; t < TL; ++t) {
                c1[t] = geo[0 * L + 32 * t];
                s1[t] = geo[1 * L + 32 * t];
                base[t] = src_local ? geo[2 * L + 32 * t] : geo[3 * L + 32 * t];
                c[t] = 1;
                s[t] = 0;
                for (int j = 0; j < w.m; ++j) {
                    const Real nc = fma_(c[t], c1[t], -(s[t] * s1[t]));
                    const Real ns = fma_(s[t], c1[t], c[t] * s1[t]);
                    c[t] = nc;
                    s[t] = ns;
                }
                // scale of element (n, m): |r|^n for local sources, |r|^-(n+1) otherwise,
                // by repeated multiplication from 1 (pipeline.cpp:81-89)
                qcol[t] = 1;
                for (int j = 0; j < (src_local ? w.m : w.m + 1); ++j) qcol[t] *= base[t];
                q[t] = qcol[t];
                for (int j = w.m; j < w.n; ++j) q[t] *= base[t];
            }
            while (e < e_end) {
                const int cnt = min(CH, e_end - e);
                Real re[CH][TL], im[CH][TL];
                TriWalk wl = w;
#pragma unroll
                for (int u = 0; u < CH; ++u) {
                    if (u < cnt) {
                        const int64_t off = (int64_t)aos_re(wl.n, wl.m) * a.in_stride;
#pragma unroll
                        for (int t = 0; t < TL; ++t) {
                            re[u][t] = active[t] ? a.in[off + src[t]] : Real(0);
                            im[u][t] = (active[t] && wl.m) ? a.in[off + a.in_stride + src[t]] : Real(0);
                        }
                        wl.advance();
                    }
                }
#pragma unroll
                for (int u = 0; u < CH; ++u) {
                    if (u < cnt) {
#pragma unroll
                        for (int t = 0; t < TL; ++t) {
                            const Real nr = q[t] * fma_(re[u][t], c[t], -(im[u][t] * s[t]));
                            const Real ni = q[t] * fma_(re[u][t], s[t], im[u][t] * c[t]);
                            buf[t_re(w.n, w.m) * L + 32 * t] = nr;
                            if (w.m) buf[t_im(w.n, w.m) * L + 32 * t] = ni;
                            q[t] *= base[t];
                        }
                        const int m_before = w.m;
                        w.advance();
                        if (w.m != m_before) {
#pragma unroll
                            for (int t = 0; t < TL; ++t) {
                                const Real nc = fma_(c[t], c1[t], -(s[t] * s1[t]));
                                const Real ns = fma_(s[t], c1[t], c[t] * s1[t]);
                                c[t] = nc;
                                s[t] = ns;
                                qcol[t] *= base[t];
                                q[t] = qcol[t];
                            }
                        }
                    }
                }
                e += cnt;
            }
        }
        __syncthreads();

        // ---- B: forward swap passes, largest rows first
        {
            Ctx<TL> c{buf, cb, sb, src_local, false, false};
            for (int task = fetch_task(&counters[0], lane); task < 2 * p_in;
                 task = fetch_task(&counters[0], lane)) {
                const int n = p_in - 1 - (task >> 1);
                half_task_dispatch<TL>(c, n, task & 1, n);
            }
        }
        __syncthreads();

        // ---- Z: z-axis step per (column, re|im), longest columns first
        for (int task = fetch_task(&counters[1], lane); task < 2 * cols;
             task = fetch_task(&counters[1], lane)) {
            const int m = task >> 1, part = task & 1;
            if (part && m == 0) continue;
            zstep_dispatch<TL>(buf, kind, p_in, p_out, m, part);
        }
        __syncthreads();

        // ---- C: backward swap passes; columns >= cols of the z-step output are
        // zero (pipeline.cpp:229-246) and are skipped, which is exact
        {
            Ctx<TL> c{buf, cb, sb, dst_local, true, kind == KIND_M2L};
            for (int task = fetch_task(&counters[2], lane); task < 2 * p_out;
                 task = fetch_task(&counters[2], lane)) {
                const int n = p_out - 1 - (task >> 1);
                half_task_dispatch<TL>(c, n, task & 1, min(n, cols - 1));
            }
        }
        __syncthreads();

        // ---- D: rotate by -alpha, scale (pipeline.cpp:251-257), store or reduce
        {
            const int T = p_out * (p_out + 1) / 2;
            int e = (int)((long)T * warp / W);
            const int e_end = (int)((long)T * (warp + 1) / W);
            TriWalk w{0, 0, p_out};
            {
                int rem = e;
                while (rem >= p_out - w.m) {
                    rem -= p_out - w.m;
                    ++w.m;
                }
                w.n = w.m + rem;
            }
            Real c1[TL], s1[TL], base[TL], c[TL], s[TL], qcol[TL], q[TL];
#pragma unroll
            for (int t = 0; t < TL; ++t) {
                c1[t] = geo[0 * L + 32 * t];
                s1[t] = geo[1 * L + 32 * t];
                base[t] = dst_local ? geo[3 * L + 32 * t] : geo[2 * L + 32 * t];
                c[t] = 1;
                s[t] = 0;
                for (int j = 0; j < w.m; ++j) {
                    const Real nc = fma_(c[t], c1[t], -(s[t] * s1[t]));
                    const Real ns = fma_(s[t], c1[t], c[t] * s1[t]);
                    c[t] = nc;
                    s[t] = ns;
                }
                // |r|^-n for local targets, |r|^(n+1) for multipole targets
                qcol[t] = 1;
                for (int j = 0; j < (dst_local ? w.m : w.m + 1); ++j) qcol[t] *= base[t];
                q[t] = qcol[t];
                for (int j = w.m; j < w.n; ++j) q[t] *= base[t];
            }
            for (; e < e_end; ++e) {
                const int n = w.n, m = w.m;
                Real nr[TL], ni[TL];
#pragma unroll
                for (int t = 0; t < TL; ++t) {
                    const Real re = buf[t_re(n, m) * L + 32 * t];
                    const Real im = m ? buf[t_im(n, m) * L + 32 * t] : Real(0);
                    const Real ms = -s[t];
                    nr[t] = q[t] * fma_(re, c[t], -(im * ms));
                    ni[t] = q[t] * fma_(re, ms, im * c[t]);
                    q[t] *= base[t];
                }
                if (!accumulate) {
#pragma unroll
                    for (int t = 0; t < TL; ++t)
                        if (active[t]) {
                            a.out[(int64_t)aos_re(n, m) * a.out_stride + b[t]] = nr[t];
                            a.out[(int64_t)(aos_re(n, m) + 1) * a.out_stride + b[t]] =
                                m ? ni[t] : Real(0);
                        }
                } else {
                    // fixed order: slots l and l+32 first, then the xor butterfly
                    Real sr = nr[0], si = ni[0];
#pragma unroll
                    for (int t = 1; t < TL; ++t) {
                        sr += nr[t];
                        si += ni[t];
                    }
                    sr = warp_sum(sr);
                    if (m) si = warp_sum(si);
                    if (lane == 0) {
                        a.out[(int64_t)aos_re(n, m) * a.out_stride + g] = sr;
                        if (m) a.out[(int64_t)(aos_re(n, m) + 1) * a.out_stride + g] = si;
                    }
                }
                w.advance();
                if (w.m != m) {
#pragma unroll
                    for (int t = 0; t < TL; ++t) {
                        const Real nc = fma_(c[t], c1[t], -(s[t] * s1[t]));
                        const Real ns = fma_(s[t], c1[t], c[t] * s1[t]);
                        c[t] = nc;
                        s[t] = ns;
                        qcol[t] *= base[t];
                        q[t] = qcol[t];
                    }
                }
            }
        }
        __syncthreads();
    }
}

// ---- host side: constant-bank upload (once per device and process) --------

struct HostTables {
    std::vector<Real> sw;
    std::vector<int> blk;
    std::vector<Real> z;
    bool ok = false;
};

HostTables build_host_tables() {
    HostTables h;
    const SwapTables st(PMAX);
    const PackedSide cm = pack_side(st, false);  // column-major blocks of F, G
    if ((int)cm.stream.size() != SWAP_LEN) return h;  // constexpr layout out of sync with tables.cpp
    h.ok = true;
    h.sw.assign(2 * (SWAP_LEN + SWAP_PAD), Real(0));
    h.blk.assign(PMAX * 4, 0);
    for (int n = 0; n < PMAX; ++n)
        for (int j = 0; j < 4; ++j) {
            const BlockDesc& d = cm.desc[(size_t)n * 4 + j];
            h.blk[n * 4 + j] = (int)d.offset;
            for (int k = 0; k < d.ncols; ++k)
                for (int i = 0; i < d.nrows; ++i) {
                    const Real v = static_cast<Real>(cm.stream[d.offset + (size_t)k * d.nrows + i]);
                    h.sw[d.offset + (size_t)k * d.nrows + i] = v;            // column-major
                    h.sw[RM_BASE + d.offset + (size_t)i * d.ncols + k] = v;  // row-major
                }
        }
    std::vector<Real> fac, inv;
    build_faculties<Real>(PMAX, fac, inv);
    h.z.assign(3 * ZSEG, Real(0));
    for (size_t k = 0; k < fac.size(); ++k) h.z[Z_FAC + k] = fac[k];
    for (int d = 0; d < PMAX; ++d) {
        h.z[Z_LOW + PMAX + d] = (d & 1) ? -inv[d] : inv[d];  // pipeline.cpp:191-194
        h.z[Z_UP + PMAX - d] = inv[d];
    }
    return h;
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
    static const HostTables h = build_host_tables();
    if (!h.ok) return cudaErrorInvalidValue;
    e = cudaMemcpyToSymbol(c_sw, h.sw.data(), sizeof(Real) * h.sw.size());
    if (e != cudaSuccess) return e;
    e = cudaMemcpyToSymbol(c_blk, h.blk.data(), sizeof(int) * h.blk.size());
    if (e != cudaSuccess) return e;
    e = cudaMemcpyToSymbol(c_z, h.z.data(), sizeof(Real) * h.z.size());
    if (e != cudaSuccess) return e;
    done.push_back(dev);
    return cudaSuccess;
}

int tiled_warps_for(int p_rot) {
    if (const char* env = getenv("SFMM_TILED_WARPS")) {
        const int w = atoi(env);
        if (w >= 2 && w <= 12) return w;
    }
    if (p_rot >= 14) return 12;
    if (p_rot >= 8) return 8;
    return 4;
}

}  // namespace

bool tiled_supports(const TranslateArgs<Real>& a) {
    return std::max(a.p_in, a.p_out) <= PMAX;
}

cudaError_t launch_translate_tiled(const TranslateArgs<Real>& a, int sm_count,
                                   cudaStream_t stream, LaunchInfo* info) {
    constexpr int TL = 2;
    cudaError_t e = ensure_constants();
    if (e != cudaSuccess) return e;
    const int p_rot = std::max(a.p_in, a.p_out);
    const TiledLayout<TL> lay{p_rot};
    const size_t smem = lay.smem_bytes();
    const int64_t n_groups = (a.n + 32 * TL - 1) / (32 * TL);
    const int block = 32 * tiled_warps_for(p_rot);
    auto kern = translate_tiled_kernel<TL>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 1;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorLaunchOutOfResources;
    const int grid = (int)std::min<int64_t>(n_groups, (int64_t)sm_count * per_sm);
    kern<<<grid, block, smem, stream>>>(a, n_groups, p_rot);
    if (info) {
        info->grid = grid;
        info->block = block;
        info->smem = smem;
        info->launches = 1;
        info->variant = sizeof(Real) == 8 ? "tiled/f64/TL2" : "tiled/f32/TL2";
    }
    return cudaGetLastError();
}

}  // namespace sfmm

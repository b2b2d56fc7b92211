// Tuned translation kernel ("tiled"): included by sfmm_tiled_f64.cu and
// sfmm_tiled_f32.cu with
//     SFMM_REAL   double | float
//     SFMM_PMAX   largest max(p_in, p_out) this instantiation covers
//
// Design:
//  * one CTA per group of 32*TL translations; lane l owns translations l and
//    l+32 (TL = 2), so every operator entry fetched feeds two independent FMA
//    chains per lane;
//  * the coefficient triangle of the whole group lives in shared memory in a
//    compact layout buf[q][32*TL]; every access is unit stride and conflict free;
//  * the swap-matrix stream of the side in use (multipole: F, G; local: F^T,
//    G^T; tables.hpp "parity blocks") is staged into shared memory with one TMA
//    bulk copy (cp.async.bulk + mbarrier) per phase, issued while the previous
//    phase still computes, and consumed by warp-uniform 128-bit shared loads
//    (two entries per load). The constant bank was measured and rejected for
//    this: it only sustains the FMA rate when all warps read the same lines
//    (profiles/microbench_r01.jsonl: 29 TFLOP/s in lockstep, 5.5 TFLOP/s with
//    per-warp regions; shared-memory broadcast 26 TFLOP/s regardless);
//  * the axis-swap pass on row n is split into its two parity halves; each half
//    is register-resident straight-line code in the class size NC only;
//  * the z-axis step reads its Hankel/Toeplitz operator (faculties) from the
//    constant bank through a sliding register window (all warps walk the same
//    40-entry table, the case in which the constant path is at full speed);
//  * arithmetic order is the reference's: k-ascending fma chains from +0.

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <vector>

#include "device_math.cuh"
#include "kernel_generic.cuh"
#include "sfmm_internal.hpp"

namespace sfmm {
namespace {

using Real = SFMM_REAL;
constexpr int PMAX = SFMM_PMAX;
#ifndef SFMM_MAXTHREADS
#define SFMM_MAXTHREADS 384
#endif
constexpr int NCMAX = PMAX / 2 + (PMAX & 1);  // largest parity-class size, rows n < PMAX
constexpr int TAB_PAD = 64;                    // finite slack behind the staged stream prefix
constexpr int ZSEG = 2 * PMAX + 8;             // one z-table segment
constexpr int Z_FAC = 0, Z_LOW = ZSEG, Z_UP = 2 * ZSEG;

template <typename T> struct vec2_of;
template <> struct vec2_of<double> { using type = double2; };
template <> struct vec2_of<float> { using type = float2; };
using Vec2 = vec2_of<Real>::type;

// block offsets into the parity-block stream, [n*4 + {F/E, F/O, G/E, G/O}] (same for both sides)
__constant__ int c_blk[PMAX * 4];
// fac[k] | lower Toeplitz (-1)^d/d! at [PMAX + d], 0 for d < 0 | upper 1/(-d)! at [PMAX + d], 0 for d > 0
__constant__ Real c_z[3 * ZSEG];

__device__ __forceinline__ int class_size(int n, int cls) { return cls ? (n + 1) >> 1 : (n >> 1) + 1; }

// Shared-memory triangle: row n starts at n^2 and holds re_l at 2l and
// im_l (l >= 1) at 2l-1, so both parts of a parity class are reached from one
// base with compile-time strides.
__device__ __forceinline__ int t_re(int n, int l) { return n * n + 2 * l; }
__device__ __forceinline__ int t_im(int n, int l) { return n * n + 2 * l - 1; }

// ---- TMA bulk copy + mbarrier (PTX ISA: cp.async.bulk, mbarrier) -----------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n"
            "}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                          uint64_t* bar) {
    // the generic-proxy reads of the previous table must be ordered before the
    // async-proxy overwrite
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(bar, bytes);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(smem_dst)),
        "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Dynamic shared memory of the kernel. Device functions re-derive their
// pointers from this symbol (offsets travel in Ctx) so that ptxas emits
// LDS/STS rather than generic loads across the out-of-line calls.
extern __shared__ __align__(16) unsigned char smem_raw[];

template <int TL>
struct Ctx {
    int buf_off;      // element offset of the triangle buffer in smem_raw (lane not applied)
    int tab_off;      // element offset of the staged parity-block stream
    const Real* cb;   // global scratch, lane offset applied; cb[m * L + 32 t]
    const Real* sb;   // sin table of the pass: +sin(m beta) forward, -sin(m beta) backward
    bool local_side;
};

// acc[i][t] += sum_{k0 <= k < kend} line_k[i] * in[4 k L + 32 t]: lines of padded length ld
// at tab + k ld (warp-uniform 128-bit loads, two entries each), software pipelined.
template <int TL, int NCE>
__device__ __forceinline__ void first_product(const Real* tab, int ld, const Real* in, int k0,
                                              int kend, bool halve_first, Real (&acc)[NCE][TL]) {
    constexpr int L = 32 * TL;
    if (k0 >= kend) return;
    Vec2 a[NCE / 2];
    Real x[TL];
    {
        const Real* line = tab + k0 * ld;
#pragma unroll
        for (int i2 = 0; i2 < NCE / 2; ++i2) a[i2] = *reinterpret_cast<const Vec2*>(line + 2 * i2);
#pragma unroll
        for (int t = 0; t < TL; ++t) x[t] = in[4 * k0 * L + 32 * t];
        if (halve_first) {
#pragma unroll
            for (int t = 0; t < TL; ++t) x[t] *= Real(0.5);
        }
    }
#pragma unroll 2
    for (int k = k0; k < kend; ++k) {
        Vec2 an[NCE / 2];
        Real xn[TL];
        const int kn = min(k + 1, kend - 1);  // the last trip reloads its own operands
        const Real* line = tab + kn * ld;
#pragma unroll
        for (int i2 = 0; i2 < NCE / 2; ++i2) an[i2] = *reinterpret_cast<const Vec2*>(line + 2 * i2);
#pragma unroll
        for (int t = 0; t < TL; ++t) xn[t] = in[4 * kn * L + 32 * t];
#pragma unroll
        for (int i2 = 0; i2 < NCE / 2; ++i2)
#pragma unroll
            for (int t = 0; t < TL; ++t) {
                acc[2 * i2][t] = fma_(a[i2].x, x[t], acc[2 * i2][t]);
                acc[2 * i2 + 1][t] = fma_(a[i2].y, x[t], acc[2 * i2 + 1][t]);
            }
#pragma unroll
        for (int i2 = 0; i2 < NCE / 2; ++i2) a[i2] = an[i2];
#pragma unroll
        for (int t = 0; t < TL; ++t) x[t] = xn[t];
    }
}

// One parity half of swap -> rotate(+-beta) -> swap on row n (reference
// pipeline.cpp:118-136 with :155-157 / :247-249), in place in shared memory.
//
// CODE SIZE IS A FIRST-ORDER CONSTRAINT HERE: the B200 instruction cache holds
// about 32 KB per SM and execution slows ~5x once the code the warps of an SM
// run concurrently exceeds it (profiles/icache_probe_r01.jsonl). The warps of
// a CTA work on different rows at the same time, so the half task exists in
// only five sizes NCE in {2, 4, 6, 8, 10}, each out of line and
// shared by the forward and the backward pass; a class of nc = NCE-1 members
// runs in the NCE code with one idle accumulator (the table lines are padded
// to even length with zeros, so the idle lane stays exactly zero).
//   first products:  runtime loop over the inputs k (read from shared memory),
//                    the NCE accumulators of u_re and u_im unrolled;
//   second products: runtime loop over output rows, four per trip, the NCE
//                    inputs u[k] unrolled; one 128-bit load fetches the entries
//                    of two adjacent rows.
// mmax < n only for backward rows with p_out > p_in (inputs in columns
// >= min(p_in, p_out) are zero, pipeline.cpp:229-246): the input loop is
// simply shorter, which is exact.
template <int TL, int NCE>
__device__ __noinline__ void half_task(const Ctx<TL> c, int n, int cls, int mmax) {
    constexpr int L = 32 * TL;
    const int nc = class_size(n, cls);     // 1 <= nc <= NCE
    const int ld = nc + (nc & 1);          // padded line length of the blocks with nc rows
    const int cF = (n - cls) & 1, cG = cF ^ 1;
    const int nG = class_size(n, cG);      // the real class cF always has nc members
    const int g0 = cG ? 0 : 1;             // class index 0 of E is l = 0: no imaginary part
    const int kendF = mmax >= cF ? min(nc, ((mmax - cF) >> 1) + 1) : 0;
    const int kendG = mmax >= cG ? min(nG, ((mmax - cG) >> 1) + 1) : 0;
    Real* sm = reinterpret_cast<Real*>(smem_raw);
    const Real* tab = sm + c.tab_off;
    const Real* tF1 = tab + c_blk[n * 4 + cls];
    const Real* tG1 = tab + c_blk[n * 4 + 2 + cls];
    const Real* tF2 = tab + c_blk[n * 4 + cF];
    const Real* tG2 = tab + c_blk[n * 4 + 2 + cG];
    const int ldG2 = nG + (nG & 1);
    Real* row = sm + c.buf_off + (threadIdx.x & 31) + n * n * L;
    Real* re_io = row + (2 * cF) * L;      // class index k at + 4k L
    Real* im_io = row + (2 * cG - 1) * L;  // class index k at + 4k L (k >= g0)

    Real ure[NCE][TL], uim[NCE][TL];
#pragma unroll
    for (int i = 0; i < NCE; ++i)
#pragma unroll
        for (int t = 0; t < TL; ++t) ure[i][t] = uim[i][t] = Real(0);

    // ---- first products: u_re = A_F[cls, cF] re[cF],  u_im = A_G[cls, cG] im[cG].
    // Software pipelined: the line and the input of step k+1 are in flight while
    // step k multiplies (a warp can issue a DFMA only every 4 cycles, so with 3
    // warps per scheduler any exposed shared-memory latency is lost FP64 time).
    first_product<TL, NCE>(tF1, ld, re_io, 0, kendF, c.local_side && cF == 0, ure);
    first_product<TL, NCE>(tG1, ld, im_io, g0, kendG, false, uim);
    // accumulators beyond the class (only when nc < NCE - 1, i.e. NCE == 4 serving
    // nc <= 2) picked up entries of the following lines: clear them
    if constexpr (NCE == 4) {
        if (nc < NCE - 1) {
#pragma unroll
            for (int i = 0; i < NCE; ++i)
                if (i >= nc) {
#pragma unroll
                    for (int t = 0; t < TL; ++t) ure[i][t] = uim[i][t] = Real(0);
                }
        }
    }
    // ---- rotate by +-beta (kernels.cpp:211-217); factors from the global scratch
    // (the backward pass points c.sb at the negated sines). The M2L backward gather
    // signs (-1)^(n+l) of pipeline.cpp:235-239 were applied when the z-step stored
    // its outputs (zstep_task).
    {
        const Real* cbp = c.cb + cls * L;
        const Real* sbp = c.sb + cls * L;
#pragma unroll
        for (int i = 0; i < NCE; ++i)
#pragma unroll
            for (int t = 0; t < TL; ++t) {
                const Real cm = cbp[2 * i * L + 32 * t];
                const Real s = sbp[2 * i * L + 32 * t];
                const Real a = ure[i][t], b = uim[i][t];
                ure[i][t] = fma_(a, cm, -(b * s));
                uim[i][t] = fma_(a, s, b * cm);
            }
    }
    // ---- second products: re[cF] = A_F[cF, cls] u_re,  im[cG] = A_G[cG, cls] u_im.
    // Output class index r (m' = class + 2r), rows r .. r+3 per trip; contracted index
    // k < nc (u[k] == 0 beyond).
    // trips of four rows while more than two are left, then one trip of two
    // (ROWS/2 128-bit loads per contracted index)
    auto rows_of = [&](auto rows_tag, const Real* base, int ldb, const Real (&u)[NCE][TL],
                       Real (&acc)[4][TL]) {
        constexpr int RW = decltype(rows_tag)::value;
#pragma unroll
        for (int j = 0; j < RW; ++j)
#pragma unroll
            for (int t = 0; t < TL; ++t) acc[j][t] = Real(0);
#pragma unroll
        for (int k = 0; k < NCE; ++k) {
            const Vec2 a0 = *reinterpret_cast<const Vec2*>(base + k * ldb);
            Vec2 a1 = a0;
            if constexpr (RW == 4) a1 = *reinterpret_cast<const Vec2*>(base + k * ldb + 2);
#pragma unroll
            for (int t = 0; t < TL; ++t) {
                acc[0][t] = fma_(a0.x, u[k][t], acc[0][t]);
                acc[1][t] = fma_(a0.y, u[k][t], acc[1][t]);
                if constexpr (RW == 4) {
                    acc[2][t] = fma_(a1.x, u[k][t], acc[2][t]);
                    acc[3][t] = fma_(a1.y, u[k][t], acc[3][t]);
                }
            }
        }
    };
    using Four = std::integral_constant<int, 4>;
    using Two = std::integral_constant<int, 2>;
    {
        int r = 0;
        Real acc[4][TL];
#pragma unroll 1
        for (; r + 2 < nc; r += 4) {
            rows_of(Four{}, tF2 + r, ld, ure, acc);
            if (c.local_side && r == 0 && cF == 0) {
#pragma unroll
                for (int t = 0; t < TL; ++t) acc[0][t] *= Real(2);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (r + j < nc) {
#pragma unroll
                    for (int t = 0; t < TL; ++t) re_io[4 * (r + j) * L + 32 * t] = acc[j][t];
                }
        }
        if (r < nc) {
            rows_of(Two{}, tF2 + r, ld, ure, acc);
            if (c.local_side && r == 0 && cF == 0) {
#pragma unroll
                for (int t = 0; t < TL; ++t) acc[0][t] *= Real(2);
            }
#pragma unroll
            for (int j = 0; j < 2; ++j)
                if (r + j < nc) {
#pragma unroll
                    for (int t = 0; t < TL; ++t) re_io[4 * (r + j) * L + 32 * t] = acc[j][t];
                }
        }
    }
    {
        int r = 0;
        Real acc[4][TL];
#pragma unroll 1
        for (; r + 2 < nG; r += 4) {
            rows_of(Four{}, tG2 + r, ldG2, uim, acc);
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (r + j < nG && r + j >= g0) {
#pragma unroll
                    for (int t = 0; t < TL; ++t) im_io[4 * (r + j) * L + 32 * t] = acc[j][t];
                }
        }
        if (r < nG) {
            rows_of(Two{}, tG2 + r, ldG2, uim, acc);
#pragma unroll
            for (int j = 0; j < 2; ++j)
                if (r + j < nG && r + j >= g0) {
#pragma unroll
                    for (int t = 0; t < TL; ++t) im_io[4 * (r + j) * L + 32 * t] = acc[j][t];
                }
        }
    }
}

template <int TL>
__device__ __forceinline__ void half_task_dispatch(const Ctx<TL> c, int n, int cls, int mmax) {
    const int nc = class_size(n, cls);
    if (nc <= 2) half_task<TL, 2>(c, n, cls, mmax);
    else if (nc <= 4) half_task<TL, 4>(c, n, cls, mmax);
    else if (nc <= 6) half_task<TL, 6>(c, n, cls, mmax);
    else if (nc <= 8) {
        if constexpr (NCMAX > 6) half_task<TL, 8>(c, n, cls, mmax);
    } else {
        if constexpr (NCMAX > 8) half_task<TL, 10>(c, n, cls, mmax);
    }
}

// z-axis step on column (m, part) in place, R outputs per translation
// (reference kernels.cpp:118-196). The Hankel (M2L: (2m+i+k)!) or Toeplitz
// (M2M/L2L) operator entries come from the constant bank: every warp walks the
// same ~40-entry table, the access pattern for which the constant path runs at
// full rate. Kept as a plain k loop for code size (see half_task).
template <int TL, int R, int DIR>
__device__ __noinline__ void zstep_task(int buf_off, int zi, int p_in, int p_out, int m, int part,
                                        bool alternate_signs) {
    constexpr int L = 32 * TL;
    const int kin = p_in - m, kout = p_out - m;
    Real* buf = reinterpret_cast<Real*>(smem_raw) + buf_off + (threadIdx.x & 31);
    Real* col = buf + (part ? t_im(m, m) : t_re(m, m)) * L;  // element k at col[(2 m k + k^2) L]
    Real acc[R][TL];
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
        for (int t = 0; t < TL; ++t) acc[i][t] = Real(0);
    // four k-steps share one sliding window of R + 3 operator entries
    int k = 0;
#pragma unroll 1
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
#pragma unroll 1
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
    // M2L: the backward gather multiplies row n, column m by (-1)^(n+m) = (-1)^i
    // (pipeline.cpp:235-239); negation is exact, so it is applied here once
    if (alternate_signs) {
#pragma unroll
        for (int i = 1; i < R; i += 2)
#pragma unroll
            for (int t = 0; t < TL; ++t) acc[i][t] = -acc[i][t];
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
__device__ __forceinline__ void zstep_dispatch(int buf, int kind, int p_in, int p_out, int m,
                                               int part) {
    const int r4 = (p_out - m + 3) >> 2;
    const int zi = kind == KIND_M2L ? Z_FAC + 2 * m : (kind == KIND_M2M ? Z_LOW + PMAX : Z_UP + PMAX);
    switch (r4) {
#define SFMM_CASE(K)                                                                       \
    case K:                                                                                \
        if constexpr (4 * K <= PMAX + 3) {                                                 \
            if (kind == KIND_M2L) zstep_task<TL, 4 * K, 1>(buf, zi, p_in, p_out, m, part, true);   \
            else zstep_task<TL, 4 * K, -1>(buf, zi, p_in, p_out, m, part, false);          \
        }                                                                                  \
        break;
        SFMM_CASE(1) SFMM_CASE(2) SFMM_CASE(3) SFMM_CASE(4) SFMM_CASE(5)
#undef SFMM_CASE
        default: break;
    }
}

__device__ __forceinline__ int fetch_task(int* counter, int lane) {
    int t = 0;
    // plain PTX: atomicAdd() under a lane predicate compiles to the warp-aggregated
    // sequence (vote, find-leader, popc), a dozen instructions per fetch for nothing
    if (lane == 0)
        asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(t) : "r"(smem_u32(counter)) : "memory");
    return __shfl_sync(0xffffffffu, t, 0);
}

template <int TL>
struct TiledLayout {
    static constexpr int L = 32 * TL;
    int p_rot;
    size_t tab_len;  // staged stream elements (prefix + TAB_PAD, multiple of 4)
    __host__ __device__ size_t buf_elems() const { return (size_t)p_rot * p_rot * L; }
    // triangle, staged stream, {mbarrier, task counters} (32 bytes), per-row completion
    // counters of the backward swap pass, launch constants of the row function
    __host__ __device__ size_t smem_bytes() const {
        return sizeof(Real) * (buf_elems() + tab_len) + 32 + 2 * sizeof(int) * ((PMAX + 3) / 4 * 4) +
               128 + 8 * PMAX;  // RowConst, row_bar (phase A by bulk copies)
    }
};

struct TiledTables {
    const Real* stream[2];  // global parity-block streams: [0] multipole side, [1] local side
    uint32_t bytes[2];      // bytes staged for the forward / backward pass
    Real* scratch;          // global, per CTA and group parity: geometry of the group (geo_elems)
    int row_warps;          // warps that start the last phase in the row queue
    int prefetch;           // request the SoA inputs of the group after the next into the L2
};

// Per-group geometry in the global scratch (L2 resident, written one group ahead,
// reference pipeline.cpp:52-91). Rows of L = 32*TL values:
//   cos(m beta), sin(m beta), -sin(m beta)   [p_rot + 2] each (two slack rows: the NCE
//                                            code reads one class index past an odd class)
//   cos(m alpha), sin(m alpha)               [p_rot] each
//   qa[m], qd[m]                             [p_rot] each: scale of element (m, m) in the
//                                            forward / backward pass (head of column m)
//   base_a, base_d                           the per-row factor of those scales
template <int TL>
__host__ __device__ constexpr size_t geo_elems(int p_rot) {
    return (size_t)(3 * (p_rot + 2) + 4 * p_rot + 2) * 32 * TL;
}

template <int TL>
struct GeoView {
    const Real *cb, *sb, *nsb, *ca, *sa, *qa, *qd, *base_a, *base_d;
    __device__ GeoView(const Real* g, int p_rot) {
        constexpr int L = 32 * TL;
        cb = g;
        sb = cb + (size_t)(p_rot + 2) * L;
        nsb = sb + (size_t)(p_rot + 2) * L;
        ca = nsb + (size_t)(p_rot + 2) * L;
        sa = ca + (size_t)p_rot * L;
        qa = sa + (size_t)p_rot * L;
        qd = qa + (size_t)p_rot * L;
        base_a = qd + (size_t)p_rot * L;
        base_d = base_a + L;
    }
};

// Geometry of one group: warp t fills slot set t. Scales (pipeline.cpp:148-154, 251-257):
// forward |r|^n (local source) or |r|^-(n+1); backward |r|^-n (local target) or |r|^(n+1);
// all powers by repeated multiplication from 1 (pipeline.cpp:81-89).
template <int TL>
__device__ __forceinline__ void geometry_phase(const TranslateArgs<Real>& a, int64_t g, int p_rot,
                                               Real* geo, bool src_local, bool dst_local, int warp,
                                               int lane) {
    constexpr int L = 32 * TL;
    if (warp >= TL) return;
    const int t = warp;
    const int64_t b = g * L + 32 * t + lane;
    Angles<Real> ang;
    Real inv;
    if (a.angles) {  // plan path: decomposed when the plan was built, for every padded lane
        const int64_t j = a.angle_index ? (int64_t)a.angle_index[b] : b;
        ang.rn = a.angles[j];
        ang.ca = a.angles[a.n + j];
        ang.sa = a.angles[2 * a.n + j];
        ang.cb = a.angles[3 * a.n + j];
        ang.sb = a.angles[4 * a.n + j];
        inv = a.angles[5 * a.n + j];
    } else {
        bool active = b < a.n;
        if (active && a.src_index) active = a.src_index[b] >= 0;
        Real x = 0, y = 0, z = 1;  // idle lanes get a benign shift (pipeline.cpp:56-61)
        if (active) {
            x = a.shifts[3 * b];
            y = a.shifts[3 * b + 1];
            z = a.shifts[3 * b + 2];
        }
        ang = decompose_angles(x, y, z);
        inv = Real(1) / ang.rn;
    }
    const GeoView<TL> v(geo + 32 * t + lane, p_rot);
    Real* cbg = const_cast<Real*>(v.cb);
    Real* sbg = const_cast<Real*>(v.sb);
    Real* nsbg = const_cast<Real*>(v.nsb);
    Real* cag = const_cast<Real*>(v.ca);
    Real* sag = const_cast<Real*>(v.sa);
    Real* qag = const_cast<Real*>(v.qa);
    Real* qdg = const_cast<Real*>(v.qd);
    const Real base_a = src_local ? ang.rn : inv;
    const Real base_d = dst_local ? inv : ang.rn;
    *const_cast<Real*>(v.base_a) = base_a;
    *const_cast<Real*>(v.base_d) = base_d;
    // cos/sin(m alpha): only the first step is tabulated, the elementwise phases follow
    // the rows by the same recurrence (elementwise_rows)
    cag[0] = Real(1);
    sag[0] = Real(0);
    if (p_rot > 1) {
        cag[L] = fma_(Real(1), ang.ca, -(Real(0) * ang.sa));
        sag[L] = fma_(Real(0), ang.ca, Real(1) * ang.sa);
    }
    Real c = 1, s = 0;
    Real qa = src_local ? Real(1) : base_a;  // base_a^(0 + q0)
    Real qd = dst_local ? Real(1) : base_d;
    for (int m = 0; m < p_rot + 2; ++m) {
        cbg[m * L] = c;
        sbg[m * L] = s;
        nsbg[m * L] = -s;
        if (m < p_rot) {
            qag[m * L] = qa;
            qdg[m * L] = qd;
        }
        const Real nc = fma_(c, ang.cb, -(s * ang.sb));
        const Real ns = fma_(s, ang.cb, c * ang.sb);
        c = nc;
        s = ns;
        qa *= base_a;
        qd *= base_d;
    }
}

// Transposing butterfly over the 32 lanes: every lane enters with NV values v[j]
// (its own contribution to value index j; NV = 8 or 16) and leaves with the sum over
// all lanes of value index lane / (32 / NV) in v[0] (32 / NV neighbouring lanes hold
// the same sum). NV exchanges instead of 5 NV; per value the additions pair lanes at
// distance 16, 8, 4, 2, 1 (sharding.accumulation_tree).
template <int NV>
__device__ __forceinline__ void lane_transpose_sum(Real (&v)[NV], int lane) {
    int d = 16;
#pragma unroll
    for (int h = NV / 2; h >= 1; h >>= 1, d >>= 1) {
        const bool upper = lane & d;
#pragma unroll
        for (int j = 0; j < h; ++j) {
            const Real send = upper ? v[j] : v[j + h];
            const Real keep = upper ? v[j + h] : v[j];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, d);
        }
    }
#pragma unroll
    for (d = 16 / NV; d >= 1; d >>= 1) v[0] = v[0] + __shfl_xor_sync(0xffffffffu, v[0], d);
}

constexpr int CHK = 4;  // elements per butterfly of phase D
// output mode of the tiled kernel: plain stores | accumulate, load-add-store | accumulate, L2 add
enum : int { ACC_NONE = 0, ACC_PLAIN = 1, ACC_L2ADD = 2 };

__device__ __forceinline__ int ld_volatile_shared(const int* p) {
    return *reinterpret_cast<const volatile int*>(p);
}

// Launch constants of elementwise_rows, written once per CTA into shared memory (behind
// row_done): arguments that travel through the calling convention cost local-memory
// stores and loads on every call.
struct RowConst {
    const Real* in;            // sources: SoA (in_stride between coefficients) or rows
    int64_t in_stride;         //          (in_stride between expansions), see ROWS below
    Real* out;                 // outputs or per-group partial sums (SoA)
    int64_t out_stride;
    const int32_t* src_index;  // accumulate mode: source of every pair, else null
    int64_t n_total;           // translations of the launch
    const Real* geo_base;      // geometry scratch of this CTA: [2 parities][geo_elems]
    int64_t geo_stride;        // geo_elems
    int buf_off;               // element offset of the triangle in smem_raw
    int p_in, p_out, p_rot;
    const int32_t* grp_target; // accumulate mode, direct form: target of every group, else null
};
// per-call flags of elementwise_rows
enum : int { ROWS_D = 1, ROWS_A = 2, ROWS_PARITY_D = 4, ROWS_PARITY_A = 8, ROWS_MISC_SHIFT = 4 };
constexpr int ROW_DONE_INTS = (PMAX + 3) / 4 * 4;
constexpr int ROW_DONE_BYTES = 2 * sizeof(int) * ROW_DONE_INTS;  // row_done, row_a_done

// Phases D and A, row by row (reference pipeline.cpp:251-257 and :148-154):
//   D (group g):   rotate by -alpha, scale by the row factor, then store (ACC = false)
//                  or reduce over the group (ACC = true): the 32*TL lanes belong to one
//                  target; the 2 CHK values of CHK elements (re, im) are summed over the
//                  lanes with one transposing butterfly, slots l and l+32 first
//                  (sharding.accumulation_tree restates the order);
//   A (group g+1): load, rotate by +alpha, scale, into the places D has just read.
// Both touch row n only, like the backward swap pass before them, so a row waits for
// its own two C half tasks (row_done) and for nothing else: the warps that run this
// function work beside the warps that still multiply. Rows come from a queue, longest
// first. cos/sin(m alpha) follow the row by the angle recurrence of pipeline.cpp:70-79
// from (1, 0), the operations that the reference uses to fill its table. Entered
// through a pointer (g_rows_fn), once per warp and phase, so everything that does not
// depend on the row stays in registers.
// 256-bit (double) / 128-bit (float) gather of four consecutive values
__device__ __forceinline__ void load4_cg(const double* p, double (&x)[4]) {
    asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(x[0]), "=d"(x[1]), "=d"(x[2]), "=d"(x[3])
                 : "l"(p));
}
__device__ __forceinline__ void load4_cg(const float* p, float (&x)[4]) {
    const float4 v = __ldcg(reinterpret_cast<const float4*>(p));
    x[0] = v.x;
    x[1] = v.y;
    x[2] = v.z;
    x[3] = v.w;
}

__device__ __forceinline__ void add_ordered(double* dst, double v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(dst), "d"(v) : "memory");
}
__device__ __forceinline__ void add_ordered(float* dst, float v) { __stcg(dst, __ldcg(dst) + v); }  // unused: f32 runs ACC_PLAIN

// ROWS: the sources are in LAYOUT_ROWS (sfmm_internal.hpp): a lane reads re, im of two
// consecutive m of its own source with one load and touches whole sectors only.
template <int TL, int ACC, bool ROWS, int CHA>
__device__ __forceinline__ void elementwise_rows(int64_t g_d, int64_t g_a, int gen, int flags) {
    constexpr int L = 32 * TL;
    // CHA: elements per batch of phase-A loads (2; 4 for streamed SoA inputs at the orders where
    // it was measured to pay, launch_translate_tiled). CHA == 0: phase A of a streamed (SoA) group
    // by bulk copies: a coefficient plane of the group is L contiguous values that land in one
    // row of the triangle, so the 2n+1 planes of row n are requested at once (cp.async.bulk, one
    // per lane, completion on the row's mbarrier) and rotated in place when they are there: one
    // memory latency per row instead of one per load batch, no registers in flight.
    const int lane = threadIdx.x & 31;
    const int misc_off = flags >> ROWS_MISC_SHIFT;  // bytes: {mbarrier, counters, row_done, RowConst}
    int* counters = reinterpret_cast<int*>(smem_raw + misc_off + 8);
    const int* row_done = counters + 6;
    int* row_a_done = counters + 6 + ROW_DONE_INTS;  // phase A of row n finished (value: trip + 1)
    const RowConst& e = *reinterpret_cast<const RowConst*>(smem_raw + misc_off + 32 + ROW_DONE_BYTES);
    const int p_rot = e.p_rot;
    const int i1 = min(1, p_rot - 1);  // row of cos/sin(alpha) in the tables
    Real* buf = reinterpret_cast<Real*>(smem_raw) + e.buf_off + lane;
    const bool do_d = flags & ROWS_D, do_a = flags & ROWS_A;
    constexpr bool BULK = CHA == 0;
    constexpr int CB = BULK ? 2 : CHA;  // register batches (BULK: only the last, partial group)
    uint64_t* row_bar = reinterpret_cast<uint64_t*>(smem_raw + misc_off + 32 + ROW_DONE_BYTES + 128);
    const bool bulk_ok = BULK && !ROWS && do_a && (g_a + 1) * (int64_t)L <= e.n_total &&
                         (e.in_stride * sizeof(Real)) % 16 == 0 && (reinterpret_cast<uintptr_t>(e.in) & 15) == 0;
    const Real* geo_d = e.geo_base + ((flags & ROWS_PARITY_D) ? e.geo_stride : 0);
    const Real* geo_a = e.geo_base + ((flags & ROWS_PARITY_A) ? e.geo_stride : 0);
    const GeoView<TL> gvd((do_d ? geo_d : geo_a) + lane, p_rot);
    const GeoView<TL> gva((do_a ? geo_a : geo_d) + lane, p_rot);

    // per slot, for all rows. Idle slots of phase A (padding of the group, tail of the
    // batch) need no masking of the data: their scale is 0 and, in accumulate mode, they
    // read the source of the group's first pair, so a non-finite value can only reach a
    // target that the reference poisons as well.
    Real dc1[TL], ds1[TL], ac1[TL], as1[TL];
    // accumulate mode: column of this group's sums in e.out. Direct form: the target itself;
    // the groups of a target follow one another in this CTA (barriers in between), every
    // group after the first adds to what the previous ones left (ascending group order, the
    // order of reduce_groups_kernel)
    bool first_d = true;
    Real* out_d = e.out + g_d;
    if (ACC && do_d && e.grp_target) {
        const int32_t tg = e.grp_target[g_d];
        first_d = g_d == 0 || e.grp_target[g_d - 1] != tg;
        out_d = e.out + tg;
    }
    const Real* pa[TL];  // the slot's source: coefficient q at pa[t][q in_stride] (SoA), or
                         // its expansion (ROWS)
    int64_t bd[TL];
    bool actd[TL], acta[TL];
#pragma unroll
    for (int t = 0; t < TL; ++t) {
        dc1[t] = gvd.ca[i1 * L + 32 * t];
        ds1[t] = gvd.sa[i1 * L + 32 * t];
        ac1[t] = gva.ca[i1 * L + 32 * t];
        as1[t] = gva.sa[i1 * L + 32 * t];
        bd[t] = g_d * L + 32 * t + lane;
        actd[t] = bd[t] < e.n_total;
        const int64_t g0 = g_a * L, bb = g0 + 32 * t + lane;
        acta[t] = do_a && bb < e.n_total;
        int64_t src = acta[t] ? bb : 0;
        if (ACC && do_a) {
            const int32_t s = e.src_index[acta[t] ? bb : g0];
            acta[t] = acta[t] && s >= 0;
            src = s >= 0 ? s : e.src_index[g0];
        }
        pa[t] = ROWS ? e.in + src * e.in_stride : e.in + src;
    }
    const int p_max = max(e.p_in, e.p_out);

    for (int task = fetch_task(&counters[3], lane); task < p_max;
         task = fetch_task(&counters[3], lane)) {
        const int n = p_max - 1 - task;
        const bool row_d = do_d && n < e.p_out, row_a = do_a && n < e.p_in;
        if (!row_d && !row_a) continue;
        // row n of the triangle: re(m) at rowp[2 m L], im(m) at rowp[(2 m - 1) L]
        Real* rowp = buf + n * n * L;

        // ---- A, first part: the loads of the first batch are in flight during phase D
        Real are[CB][TL], aim[CB][TL];
        const int64_t row_off = ROWS ? rows_off(n) : (int64_t)aos_re(n, 0) * e.in_stride;
        auto issue = [&](int m0) {
            if constexpr (ROWS) {
#pragma unroll
                for (int j = 0; j < CB / 2; ++j) {
                    const int64_t off = row_off + 4 * min((m0 >> 1) + j, n >> 1);
#pragma unroll
                    for (int t = 0; t < TL; ++t) {
                        Real x[4];
                        load4_cg(pa[t] + off, x);
                        are[2 * j][t] = x[0];
                        aim[2 * j][t] = x[1];
                        are[2 * j + 1][t] = x[2];
                        aim[2 * j + 1][t] = x[3];
                    }
                }
            } else {
#pragma unroll
                for (int u = 0; u < CB; ++u) {
                    const int64_t off = row_off + (int64_t)(2 * min(m0 + u, n)) * e.in_stride;
#pragma unroll
                    for (int t = 0; t < TL; ++t) {
                        are[u][t] = __ldcg(pa[t] + off);
                        aim[u][t] = __ldcg(pa[t] + off + e.in_stride);
                    }
                }
            }
        };
        Real aq[TL];
        if (row_a) {
#pragma unroll
            for (int t = 0; t < TL; ++t) aq[t] = acta[t] ? gva.qa[n * L + 32 * t] : Real(0);
            if (!bulk_ok) issue(0);
        }

        // ---- D
        if (row_d) {
            Real c[TL], s[TL], q[TL];
#pragma unroll
            for (int t = 0; t < TL; ++t) {
                q[t] = gvd.qd[n * L + 32 * t];
                c[t] = Real(1);
                s[t] = Real(0);
            }
            // accumulate mode: after the butterfly of a chunk, lanes REP k .. REP k + REP-1 hold
            // value k of the chunk (element k >> 1, part k & 1); the first of them owns the
            // running sum of that coefficient. The groups of a target follow one another in this
            // CTA (barriers in between), so a sum has one owner at a time and the order of the
            // additions is fixed; the first group stores 0 + sum as reduce_groups_kernel starts
            // (same signed zeros). Later groups either
            //   ACC_L2ADD  send their sum to the L2 to be added there (red.global.add.f64 by the
            //              single owner: no round trip, 5.81 ms per level), or
            //   ACC_PLAIN  load, add and store (no atomic or reduction instruction at all; the
            //              load of the next chunk is in flight during the current one, 6.07 ms).
            // Both give the same bits (one rounding per addition, same order).
            constexpr int NV = 2 * CHK, REP = 32 / NV;
            // ACC_PLAIN: this lane's element of the current chunk, its running sum and where it lives
            const int acc_k = lane / REP;
            const bool acc_lane = ACC == ACC_PLAIN && !(lane & (REP - 1));
            int acc_m = acc_k >> 1;
            Real* acc_dst = nullptr;
            Real prev_cur = Real(0);
            if constexpr (ACC == ACC_PLAIN) {
                acc_dst = out_d + (int64_t)(aos_re(n, 0) + 2 * (acc_k >> 1) + (acc_k & 1)) * e.out_stride;
                // (column 0 has no imaginary part: never read, never written)
                if (acc_lane && !first_d && acc_m <= n && !((acc_k & 1) && acc_m == 0)) prev_cur = __ldcg(acc_dst);
            }
            while (ld_volatile_shared(&row_done[n]) != 2 * gen) __nanosleep(32);
            __threadfence_block();
            for (int m0 = 0; m0 <= n; m0 += CHK) {
                Real v[NV];
#pragma unroll
                for (int j = 0; j < NV; ++j) v[j] = Real(0);
#pragma unroll
                for (int u = 0; u < CHK; ++u) {
                    const int m = m0 + u;
                    if (m > n) break;
                    Real sr = 0, si = 0;
#pragma unroll
                    for (int t = 0; t < TL; ++t) {
                        const Real re = rowp[(2 * m) * L + 32 * t];
                        Real im = rowp[(2 * m - 1) * L + 32 * t];
                        if (u == 0) im = m ? im : Real(0);  // column 0 has no imaginary part
                        const Real ms = -s[t];
                        const Real nr = q[t] * fma_(re, c[t], -(im * ms));
                        const Real ni = q[t] * fma_(re, ms, im * c[t]);
                        if constexpr (ACC) {
                            sr = t ? sr + nr : nr;
                            si = t ? si + ni : ni;
                        } else {
                            if (actd[t]) {
                                const int64_t o = (int64_t)aos_re(n, m) * e.out_stride + bd[t];
                                __stcg(e.out + o, nr);
                                __stcg(e.out + o + e.out_stride, m ? ni : Real(0));
                            }
                        }
                        const Real nc = fma_(c[t], dc1[t], -(s[t] * ds1[t]));
                        const Real ns = fma_(s[t], dc1[t], c[t] * ds1[t]);
                        c[t] = nc;
                        s[t] = ns;
                    }
                    v[2 * u] = sr;
                    v[2 * u + 1] = si;
                }
                if constexpr (ACC == ACC_PLAIN) {
                    // what the previous groups left for the NEXT chunk is requested before this
                    // chunk's butterfly: its L2 latency hides behind a whole trip of the loop
                    Real prev_nxt = Real(0);
                    const bool w_nxt = acc_lane && !first_d && acc_m + CHK <= n;
                    if (w_nxt) prev_nxt = __ldcg(acc_dst + (int64_t)(2 * CHK) * e.out_stride);
                    lane_transpose_sum<NV>(v, lane);
                    if (acc_lane && acc_m <= n && !((acc_k & 1) && acc_m == 0)) __stcg(acc_dst, prev_cur + v[0]);
                    prev_cur = prev_nxt;
                    acc_m += CHK;
                    acc_dst += (int64_t)(2 * CHK) * e.out_stride;
                } else if constexpr (ACC == ACC_L2ADD) {
                    lane_transpose_sum<NV>(v, lane);
                    // lanes REP k .. REP k + REP-1 hold value k: element k >> 1, part k & 1
                    const int k = lane / REP, m = m0 + (k >> 1), part = k & 1;
                    if (!(lane & (REP - 1)) && m <= n && !(part && m == 0)) {
                        Real* dst = out_d + (int64_t)(aos_re(n, m) + part) * e.out_stride;
                        if (first_d) __stcg(dst, Real(0) + v[0]);
                        else add_ordered(dst, v[0]);
                    }
                }
            }
        }
        if (!row_a) continue;

        // ---- A, second part
        Real c[TL], s[TL];
#pragma unroll
        for (int t = 0; t < TL; ++t) {
            c[t] = Real(1);
            s[t] = Real(0);
        }
        if (bulk_ok) {
            // every lane has finished phase D of this row; the planes of the next group replace it
            __syncwarp();
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (lane == 0) mbar_expect_tx(&row_bar[n], (uint32_t)((2 * n + 1) * L * sizeof(Real)));
            __syncwarp();
            Real* row_base = reinterpret_cast<Real*>(smem_raw) + e.buf_off + n * n * L;
            for (int j = lane; j <= 2 * n; j += 32) {
                // triangle position j of the row: re(m) at 2m, im(m) at 2m-1; AoS index of the plane
                const int cq = n * (n + 1) + ((j & 1) ? j + 2 : j);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                        "r"(smem_u32(row_base + j * L)),
                    "l"(e.in + (int64_t)cq * e.in_stride + g_a * L), "r"((uint32_t)(L * sizeof(Real))),
                    "r"(smem_u32(&row_bar[n]))
                    : "memory");
            }
            continue;  // rotated by a later task of this phase, when the planes have landed
        } else
        for (int m0 = 0;;) {
#pragma unroll
            for (int u = 0; u < CB; ++u) {
                const int m = m0 + u;
                if (m > n) break;
#pragma unroll
                for (int t = 0; t < TL; ++t) {
                    const Real xr = are[u][t];
                    Real xi = aim[u][t];
                    if (u == 0) xi = m ? xi : Real(0);
                    const Real nr = aq[t] * fma_(xr, c[t], -(xi * s[t]));
                    const Real ni = aq[t] * fma_(xr, s[t], xi * c[t]);
                    rowp[(2 * m) * L + 32 * t] = nr;
                    if (u || m) rowp[(2 * m - 1) * L + 32 * t] = ni;
                    const Real nc = fma_(c[t], ac1[t], -(s[t] * as1[t]));
                    const Real ns = fma_(s[t], ac1[t], c[t] * as1[t]);
                    c[t] = nc;
                    s[t] = ns;
                }
            }
            m0 += CB;
            if (m0 > n) break;
            issue(m0);
        }
        // row n of `nxt` is in place: its forward swap passes may start (translate_tiled_kernel)
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            *reinterpret_cast<volatile int*>(&row_a_done[n]) = gen + 1;
        }
    }
    // bulk form of phase A, second half: every row task has been taken (and its copies are issued
    // or will be by the warp that holds it); rotate the rows, longest first, as their planes land
    if (bulk_ok) {
        for (int task = fetch_task(&counters[5], lane); task < e.p_in; task = fetch_task(&counters[5], lane)) {
            const int n = e.p_in - 1 - task;
            Real* rowp = buf + n * n * L;
            Real c[TL], s[TL], aq[TL];
#pragma unroll
            for (int t = 0; t < TL; ++t) {
                aq[t] = acta[t] ? gva.qa[n * L + 32 * t] : Real(0);
                c[t] = Real(1);
                s[t] = Real(0);
            }
            mbar_wait(&row_bar[n], (uint32_t)(gen & 1));
            for (int m = 0; m <= n; ++m) {
#pragma unroll
                for (int t = 0; t < TL; ++t) {
                    const Real xr = rowp[(2 * m) * L + 32 * t];
                    const Real xi = m ? rowp[(2 * m - 1) * L + 32 * t] : Real(0);
                    const Real nr = aq[t] * fma_(xr, c[t], -(xi * s[t]));
                    const Real ni = aq[t] * fma_(xr, s[t], xi * c[t]);
                    rowp[(2 * m) * L + 32 * t] = nr;
                    if (m) rowp[(2 * m - 1) * L + 32 * t] = ni;
                    const Real nc = fma_(c[t], ac1[t], -(s[t] * as1[t]));
                    const Real ns = fma_(s[t], ac1[t], c[t] * as1[t]);
                    c[t] = nc;
                    s[t] = ns;
                }
            }
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                *reinterpret_cast<volatile int*>(&row_a_done[n]) = gen + 1;
            }
        }
    }
}

template <int TL, int ACC, bool ROWS, int CHA = 2>
__global__ void __launch_bounds__(SFMM_MAXTHREADS, 1)
translate_tiled_kernel(TranslateArgs<Real> a, TiledTables tt, int64_t n_groups, int p_rot,
                       int tab_len) {
    if (a.fail_flag && *a.fail_flag) return;

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int W = blockDim.x >> 5;
    const TiledLayout<TL> lay{p_rot, (size_t)tab_len};

    Real* sm = reinterpret_cast<Real*>(smem_raw);
    Real* tab = sm;  // 16-byte aligned
    uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + lay.tab_len + lay.buf_elems());
    int* counters = reinterpret_cast<int*>(mbar + 1);  // queues B, Z, C, rows; [4] finished C tasks
    int* row_done = counters + 6;                      // [PMAX] finished C half tasks per row
    Real* geo_base = tt.scratch + (size_t)blockIdx.x * 2 * geo_elems<TL>(p_rot);

    const int kind = a.kind, p_in = a.p_in, p_out = a.p_out;
    const bool src_local = kind == KIND_L2L;
    const bool dst_local = kind != KIND_M2M;
    const int side_fwd = src_local ? 1 : 0, side_bwd = dst_local ? 1 : 0;
    const bool two_sides = side_fwd != side_bwd;
    const int cols = min(p_in, p_out);
    const int p_max = max(p_in, p_out);
    const bool accumulate = a.src_index != nullptr;

    // table staging: one mbarrier, completions alternate fwd / bwd tables
    uint32_t tab_phase = 0;
    if (threadIdx.x == 0) {
        mbar_init(mbar, 1);
        bulk_load(tab, tt.stream[side_fwd], two_sides ? tt.bytes[0] : max(tt.bytes[0], tt.bytes[1]),
                  mbar);
    }
    bool tab_pending = true;  // a bulk copy is in flight that the next swap phase must wait for
    if (threadIdx.x < 6) counters[threadIdx.x] = 0;
    int* row_a_done = row_done + ROW_DONE_INTS;        // [PMAX] trip + 1 of the last finished phase A per row
    if (threadIdx.x < PMAX) row_done[threadIdx.x] = row_a_done[threadIdx.x] = 0;
    if (CHA == 0 && threadIdx.x < PMAX)
        mbar_init(reinterpret_cast<uint64_t*>(smem_raw + (sizeof(Real) * (lay.tab_len + lay.buf_elems())) + 32 +
                                              ROW_DONE_BYTES + 128) + threadIdx.x, 1);

    // per-phase cycle counters of CTA 0 (tuning aid, tools/perf_probe.py PHASES=1): compiled in
    // only with -DSFMM_PHASE_CLOCKS, because the running time stamp costs every warp a
    // local-memory round trip per phase
#ifdef SFMM_PHASE_CLOCKS
    long long t_prev = clock64();
#define SFMM_PHASE_MARK(idx)                                              \
    if (a.phase_clocks && blockIdx.x == 0 && threadIdx.x == 0) {          \
        const long long now = clock64();                                  \
        a.phase_clocks[idx] += now - t_prev;                              \
        t_prev = now;                                                     \
    }
#else
#define SFMM_PHASE_MARK(idx)
#endif
    const int misc_off = (int)(sizeof(Real) * (lay.tab_len + lay.buf_elems()));
    static_assert(sizeof(RowConst) <= 128, "RowConst area");
    if (threadIdx.x == 0) {
        RowConst& rc = *reinterpret_cast<RowConst*>(smem_raw + misc_off + 32 + ROW_DONE_BYTES);
        rc.in = a.in;
        rc.in_stride = a.in_stride;
        rc.out = a.out;
        rc.out_stride = a.out_stride;
        rc.src_index = a.src_index;
        rc.n_total = a.n;
        rc.geo_base = geo_base;
        rc.geo_stride = (int64_t)geo_elems<TL>(p_rot);
        rc.buf_off = (int)lay.tab_len;
        rc.p_in = p_in;
        rc.p_out = p_out;
        rc.p_rot = p_rot;
        rc.grp_target = a.grp_target;
    }
    const int rows_misc = misc_off << ROWS_MISC_SHIFT;
    // warps [0, n_cwarps) start the last phase with the C half tasks, the others with the rows
    const int n_cwarps = W - min(max(tt.row_warps, 0), W - 1);

    // groups of this CTA: strided over the CTAs, or (direct accumulation) all groups of the
    // targets blockIdx.x, blockIdx.x + gridDim.x, ...: the groups of a target meet in one CTA in
    // ascending order, and the CTAs work on neighbouring targets at the same time (their
    // sources are shared through the L2; contiguous target ranges per CTA measured 4 % slower)
    // (group numbers fit 32 bits: launch_translate_tiled refuses more)
    constexpr int END = INT_MAX;
    int walk_t = blockIdx.x, walk_hi = 0;  // direct form: target of the walk, end of its groups
    auto advance = [&](int g) -> int {
        if (!a.grp_ptr) {
            g = g < 0 ? (int)blockIdx.x : g + (int)gridDim.x;
            return g < (int)n_groups ? g : END;
        }
        if (g >= 0 && g + 1 < walk_hi) return g + 1;
        for (walk_t = g < 0 ? walk_t : walk_t + (int)gridDim.x; walk_t < (int)a.n_targets;
             walk_t += (int)gridDim.x) {
            const int lo = (int)a.grp_ptr[walk_t];
            walk_hi = (int)a.grp_ptr[walk_t + 1];
            if (lo < walk_hi) return lo;
        }
        return END;
    };
    const int g_first = advance(-1);
    int ahead = g_first == END ? END : advance(g_first);  // the group behind `nxt`
    // geometry of the first group; later groups are prepared one group ahead (geometry during
    // the z-step, phase A behind phase D of the same row)
    if (g_first != END)
        geometry_phase<TL>(a, g_first, p_rot, geo_base, src_local, dst_local, warp, lane);
    __syncthreads();

    // Schedule (two CTA-wide barriers per group). One trip of the loop:
    //   CDA  of the group `cur` that has finished its z-step (none in the first trip):
    //        backward swap passes (C) on most warps; the other warps, and every warp that
    //        finds the C queue empty, take rows from a second queue: phase D of `cur` and
    //        phase A of `nxt` on a row whose two C half tasks are done (row_done). The
    //        latency-bound elementwise work so runs beside the multiplications;
    //   B    of `nxt`: forward swap passes, one half task per (row, parity class), each behind
    //        phase A of its own row (row_a_done), no barrier in front;
    //   Z    of `nxt` (barriers on both sides): z-axis step per (column, re | im); the first TL
    //        warps first prepare the geometry of the group after it.
    // The row code is inline at this one place (out of line, called directly, ptxas fits
    // caller and callee into one register budget and spills the loads in flight).
    int parity = 0, gen = 0;  // parity: geometry buffer of `nxt`
    int cur = -1;
    for (int nxt = g_first;; parity ^= 1) {
        const bool has_next = nxt != END;
        if (cur >= 0 && warp < n_cwarps) {
            // ---- C of `cur`. Columns >= cols of the z-step output are zero
            // (pipeline.cpp:229-246) and are skipped, which is exact.
            const GeoView<TL> gv(geo_base + (size_t)(parity ^ 1) * geo_elems<TL>(p_rot) + lane, p_rot);
            Ctx<TL> c{(int)lay.tab_len, 0, gv.cb, gv.nsb, dst_local};
            for (int task = fetch_task(&counters[2], lane); task < 2 * p_out;
                 task = fetch_task(&counters[2], lane)) {
                const int n = p_out - 1 - (task >> 1);
                half_task_dispatch<TL>(c, n, task & 1, min(n, cols - 1));
                __syncwarp();
                if (lane == 0) {
                    __threadfence_block();
                    atomicAdd(&row_done[n], 1);
                    const int done = atomicAdd(&counters[4], 1) + 1;
                    // the last C task frees the table: forward-side stream of the next group
                    if (done == 2 * p_out && two_sides && has_next)
                        bulk_load(tab, tt.stream[side_fwd], tt.bytes[0], mbar);
                }
            }
        }
        // ---- D of `cur`, A of `nxt`
        if (cur >= 0 || has_next)
            elementwise_rows<TL, ACC, ROWS, CHA>(
                cur, nxt, gen,
                rows_misc | (cur >= 0 ? ROWS_D : 0) | (has_next ? ROWS_A : 0) |
                    (parity ? ROWS_PARITY_A : ROWS_PARITY_D));
        if (!has_next) break;
        if (cur >= 0 && two_sides) tab_pending = true;
        SFMM_PHASE_MARK(4)

        const GeoView<TL> gv(geo_base + (size_t)parity * geo_elems<TL>(p_rot) + lane, p_rot);
        const bool more = ahead != END;
        ++gen;
        if (tab_pending) {
            mbar_wait(mbar, tab_phase);
            tab_phase ^= 1;
            tab_pending = false;
        }
        SFMM_PHASE_MARK(1)

        // ---- B: forward swap passes, largest rows first. No CTA barrier in front: a half task
        // waits for phase A of ITS row (row_a_done), so the multiplications of the rows that
        // are in place fill the latency-bound tail of the row phase. (Every row task has been
        // taken by a warp before any warp arrives here, so the wait cannot deadlock.)
        {
            Ctx<TL> c{(int)lay.tab_len, 0, gv.cb, gv.sb, src_local};
            for (int task = fetch_task(&counters[0], lane); task < 2 * p_in;
                 task = fetch_task(&counters[0], lane)) {
                const int n = p_in - 1 - (task >> 1);
                while (ld_volatile_shared(&row_a_done[n]) != gen) __nanosleep(32);
                __threadfence_block();
                half_task_dispatch<TL>(c, n, task & 1, n);
            }
        }
        __syncthreads();
        SFMM_PHASE_MARK(2)
        if (threadIdx.x == 0) counters[0] = counters[2] = counters[3] = counters[4] = counters[5] = 0;
        if (two_sides) {  // stage the backward-side stream while the z-step runs
            if (threadIdx.x == 0) bulk_load(tab, tt.stream[side_bwd], tt.bytes[1], mbar);
            tab_pending = true;
        }

        // ---- Z: z-axis step per (column, re|im), longest columns first
        if (more)
            geometry_phase<TL>(a, ahead, p_rot,
                               geo_base + (size_t)(parity ^ 1) * geo_elems<TL>(p_rot), src_local,
                               dst_local, warp, lane);
        // streamed SoA inputs (independent translations) come from HBM: the lines of the group
        // after the next are requested into the L2 now, a whole trip ahead of phase A
        if constexpr (!ROWS && ACC == ACC_NONE) {
            if (more && tt.prefetch) {
                constexpr int L = 32 * TL, LINE = 128 / sizeof(Real), SEGS = L / LINE;  // lines per coefficient plane
                const int64_t b0 = (int64_t)ahead * L;
                for (int q = threadIdx.x; q < p_in * (p_in + 1) * SEGS; q += blockDim.x) {
                    const int cq = q / SEGS, seg = q - cq * SEGS;
                    const int64_t b = b0 + seg * LINE;
                    if (b < a.n)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.in + (int64_t)cq * a.in_stride + b));
                }
            }
        }
        for (int task = fetch_task(&counters[1], lane); task < 2 * cols;
             task = fetch_task(&counters[1], lane)) {
            const int m = task >> 1, part = task & 1;
            if (part && m == 0) continue;
            zstep_dispatch<TL>((int)lay.tab_len, kind, p_in, p_out, m, part);
        }
        if (tab_pending) {
            mbar_wait(mbar, tab_phase);
            tab_phase ^= 1;
            tab_pending = false;
        }
        __syncthreads();
        SFMM_PHASE_MARK(3)
        if (threadIdx.x == 0) counters[1] = 0;
        cur = nxt;
        nxt = ahead;
        if (ahead != END) ahead = advance(ahead);
    }
#undef SFMM_PHASE_MARK
}

// ---- host side: constant-bank upload (once per device and process) --------

struct HostTables {
    std::vector<int> blk;
    std::vector<Real> z;
};

HostTables build_host_tables() {
    HostTables h;
    const SwapTables st(PMAX);
    const PackedSide ps = pack_side(st, false);
    h.blk.assign(PMAX * 4, 0);
    for (int n = 0; n < PMAX; ++n)
        for (int j = 0; j < 4; ++j) h.blk[n * 4 + j] = (int)ps.desc[(size_t)n * 4 + j].offset;
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
    e = cudaMemcpyToSymbol(c_blk, h.blk.data(), sizeof(int) * h.blk.size());
    if (e != cudaSuccess) return e;
    e = cudaMemcpyToSymbol(c_z, h.z.data(), sizeof(Real) * h.z.size());
    if (e != cudaSuccess) return e;
    done.push_back(dev);
    return cudaSuccess;
}

int tiled_row_warps_for(int warps, bool gathered) {
    if (const char* env = getenv("SFMM_TILED_ROW_WARPS")) return atoi(env);
    // measured with the two-barrier schedule (level, P = 20: 0 / 2 / 4 row warps 5.77 / 5.73 /
    // 5.73 ms; batched P = 16: 1.036 / 1.045 / 1.068 ms): two warps start the last phase in the
    // row queue where the sources are gathered (the gathers are in flight early), none otherwise
    return gathered && warps >= 8 ? 2 : 0;
}

int tiled_prefetch_for(int p_rot) {
    if (const char* env = getenv("SFMM_TILED_PREFETCH")) return atoi(env);
    // measured (batched M2L, 400 000 translations, on / off): double precision P = 10 +2.8 %,
    // 12 -0.7 %, 14 -2.8 %, 15 +7.0 %, 16 +6.2 %, 17 +5.5 %, 18 +2.6 %, 19 -0.5 %, 20 -0.5 %;
    // single precision P = 12 +4.0 %, 18 +2.0 %
    if (sizeof(Real) == 8) return p_rot <= 11 || (p_rot >= 15 && p_rot <= 18);
    return 1;
}

int tiled_warps_for(int p_rot) {
    if (const char* env = getenv("SFMM_TILED_WARPS")) {
        const int w = atoi(env);
        if (w >= 2 && w <= SFMM_MAXTHREADS / 32) return w;
    }
    // measured (profiles/ncu_r02_notes.md, "warps per CTA"): 6 warps wherever two CTAs of 6 fit
    // an SM (168 registers x 192 threads twice, two triangles in shared memory): double
    // precision orders 9..14, single precision orders 12..18; 12 warps (one CTA per SM) for
    // the larger double-precision triangles; 4 warps (three or more CTAs) below
    if (sizeof(Real) == 8) return p_rot >= 15 ? 12 : (p_rot >= 9 ? 6 : 4);
    return p_rot >= 12 ? 6 : 4;
}

}  // namespace

bool tiled_supports(const TranslateArgs<Real>& a) {
    return std::max(a.p_in, a.p_out) <= PMAX;
}

cudaError_t launch_translate_tiled(const DeviceTables<Real>& t, const TranslateArgs<Real>& a,
                                   int sm_count, cudaStream_t stream, LaunchInfo* info) {
    constexpr int TL = 2;
    constexpr int L = 32 * TL;
    cudaError_t e = ensure_constants();
    if (e != cudaSuccess) return e;
    const int p_rot = std::max(a.p_in, a.p_out);
    // the staged prefix plus a finite pad (tail reads of dropped rows), in 16-byte units
    auto staged = [&](int p) {
        size_t len = packed_prefix_len(p) + TAB_PAD;
        return (len + 3) / 4 * 4;
    };
    const size_t tab_len = std::max(staged(a.p_in), staged(a.p_out));
    if (tab_len > t.stream_len[0] || tab_len > t.stream_len[1]) return cudaErrorInvalidValue;
    const TiledLayout<TL> lay{p_rot, tab_len};
    const size_t smem = lay.smem_bytes();
    const int64_t n_groups = (a.n + L - 1) / L;
    if (n_groups >= INT_MAX || a.n_targets >= INT_MAX) return cudaErrorInvalidValue;
    const int block = 32 * tiled_warps_for(p_rot);
    const bool acc = a.src_index != nullptr, rows = a.in_layout == LAYOUT_ROWS;
    // accumulate mode: later groups of a target add at the L2 (double precision; red.f32 would
    // flush subnormals) unless the caller asked for plain loads and stores ("accumulate_plain")
    const int mode = !acc ? ACC_NONE : ((a.acc_plain || sizeof(Real) == 4) ? ACC_PLAIN : ACC_L2ADD);
    auto kern = translate_tiled_kernel<TL, ACC_NONE, false>;
    // streamed SoA inputs: four-element load batches in phase A where 12 warps run one group per
    // SM (measured: P = 16 +8 %; P = 12 -3 %, 14 -8 %, 20 -3 % with two CTAs per SM or a full SM)
    const bool wide = sizeof(Real) == 8 && p_rot >= 15 && p_rot <= 18;
    // phase A by bulk copies, the planes requested by the warp that finishes phase D of a row and
    // rotated by a later task (bench lines, L2 flushed, on / off: configs[1] +0.7 %, sweep P = 14
    // +1.5 %, 16 +2.7 %, 20 +6.1 %); SFMM_TILED_BULK_A=0 / 1 overrides
    const bool bulk_a = getenv("SFMM_TILED_BULK_A") ? atoi(getenv("SFMM_TILED_BULK_A")) != 0 : p_rot >= 12;
    if (mode == ACC_NONE)
        kern = rows ? translate_tiled_kernel<TL, ACC_NONE, true>
                    : (bulk_a ? translate_tiled_kernel<TL, ACC_NONE, false, 0>
                              : (wide ? translate_tiled_kernel<TL, ACC_NONE, false, 4> : translate_tiled_kernel<TL, ACC_NONE, false>));
    else if (mode == ACC_PLAIN) kern = rows ? translate_tiled_kernel<TL, ACC_PLAIN, true> : translate_tiled_kernel<TL, ACC_PLAIN, false>;
    else kern = rows ? translate_tiled_kernel<TL, ACC_L2ADD, true> : translate_tiled_kernel<TL, ACC_L2ADD, false>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 1;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorLaunchOutOfResources;
    const int sms = std::max(1, sm_count - std::max(0, a.reserve_sms));
    const int grid = (int)std::min<int64_t>(n_groups, (int64_t)sms * per_sm);

    TiledTables tt;
    tt.stream[0] = t.stream[0];
    tt.stream[1] = t.stream[1];
    tt.bytes[0] = (uint32_t)(staged(a.p_in) * sizeof(Real));
    tt.bytes[1] = (uint32_t)(staged(a.p_out) * sizeof(Real));
    tt.row_warps = tiled_row_warps_for(block / 32, acc && rows);
    tt.prefetch = tiled_prefetch_for(p_rot);
    e = cudaMallocAsync((void**)&tt.scratch, sizeof(Real) * (size_t)grid * 2 * geo_elems<TL>(p_rot), stream);
    if (e != cudaSuccess) return e;
    kern<<<grid, block, smem, stream>>>(a, tt, n_groups, p_rot, (int)tab_len);
    e = cudaGetLastError();
    cudaFreeAsync(tt.scratch, stream);
    if (info) {
        info->grid = grid;
        info->block = block;
        info->smem = smem;
        info->launches = 1;
        info->variant = sizeof(Real) == 8 ? "tiled/f64/TL2" : "tiled/f32/TL2";
    }
    return e;
}

}  // namespace sfmm

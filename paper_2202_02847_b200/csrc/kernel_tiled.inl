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
#include <vector>

#include "device_math.cuh"
#include "kernel_generic.cuh"
#include "sfmm_internal.hpp"

namespace sfmm {
namespace {

using Real = SFMM_REAL;
constexpr int PMAX = SFMM_PMAX;
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
// only four sizes NCE in {4, 6, 8, 10} (~20 KB together), each out of line and
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
#pragma unroll 1
    for (int r = 0; r < nc; r += 4) {
        Real acc[4][TL];
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int t = 0; t < TL; ++t) acc[j][t] = Real(0);
        const Real* base = tF2 + r;
#pragma unroll
        for (int k = 0; k < NCE; ++k) {
            const Vec2 a0 = *reinterpret_cast<const Vec2*>(base + k * ld);
            const Vec2 a1 = *reinterpret_cast<const Vec2*>(base + k * ld + 2);
#pragma unroll
            for (int t = 0; t < TL; ++t) {
                acc[0][t] = fma_(a0.x, ure[k][t], acc[0][t]);
                acc[1][t] = fma_(a0.y, ure[k][t], acc[1][t]);
                acc[2][t] = fma_(a1.x, ure[k][t], acc[2][t]);
                acc[3][t] = fma_(a1.y, ure[k][t], acc[3][t]);
            }
        }
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
#pragma unroll 1
    for (int r = 0; r < nG; r += 4) {
        Real acc[4][TL];
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int t = 0; t < TL; ++t) acc[j][t] = Real(0);
        const Real* base = tG2 + r;
#pragma unroll
        for (int k = 0; k < NCE; ++k) {
            const Vec2 a0 = *reinterpret_cast<const Vec2*>(base + k * ldG2);
            const Vec2 a1 = *reinterpret_cast<const Vec2*>(base + k * ldG2 + 2);
#pragma unroll
            for (int t = 0; t < TL; ++t) {
                acc[0][t] = fma_(a0.x, uim[k][t], acc[0][t]);
                acc[1][t] = fma_(a0.y, uim[k][t], acc[1][t]);
                acc[2][t] = fma_(a1.x, uim[k][t], acc[2][t]);
                acc[3][t] = fma_(a1.y, uim[k][t], acc[3][t]);
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (r + j < nG && r + j >= g0) {
#pragma unroll
                for (int t = 0; t < TL; ++t) im_io[4 * (r + j) * L + 32 * t] = acc[j][t];
            }
    }
}

template <int TL>
__device__ __forceinline__ void half_task_dispatch(const Ctx<TL> c, int n, int cls, int mmax) {
    const int nc = class_size(n, cls);
    if (nc <= 4) half_task<TL, 4>(c, n, cls, mmax);
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
    if (lane == 0) t = atomicAdd(counter, 1);
    return __shfl_sync(0xffffffffu, t, 0);
}

template <int TL>
struct TiledLayout {
    static constexpr int L = 32 * TL;
    int p_rot;
    size_t tab_len;  // staged stream elements (prefix + TAB_PAD, multiple of 4)
    __host__ __device__ size_t buf_elems() const { return (size_t)p_rot * p_rot * L; }
    // triangle, staged stream, {mbarrier, task counters} (32 bytes), cos/sin(alpha) of the
    // current and the next group ([2][2][L])
    __host__ __device__ size_t smem_bytes() const {
        return sizeof(Real) * (buf_elems() + tab_len + 4 * L) + 32;
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

// element number e of the walk; e past the end gives n >= p, which every user skips
__device__ __forceinline__ TriWalk tri_seek(int e, int p) {
    int m = 0;
    while (m < p && e >= p - m) {
        e -= p - m;
        ++m;
    }
    return TriWalk{m + e, m, p};
}

// Rotation and scale factors that travel with a TriWalk: cos/sin(m alpha) of the
// current column, the scale q of the current row and qh of the column's first row.
template <int TL>
struct RotWalk {
    Real c[TL], s[TL], q[TL], qh[TL], base[TL];
};

struct TiledTables {
    const Real* stream[2];  // global parity-block streams: [0] multipole side, [1] local side
    uint32_t bytes[2];      // bytes staged for the forward / backward pass
    Real* scratch;          // global, per CTA and group parity: geometry of the group (geo_elems)
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
                                               Real* geo, Real* c1s1, bool src_local, bool dst_local,
                                               int warp, int lane) {
    constexpr int L = 32 * TL;
    if (warp >= TL) return;
    const int t = warp;
    const int64_t b = g * L + 32 * t + lane;
    bool active = b < a.n;
    if (active && a.src_index) active = a.src_index[b] >= 0;
    Real x = 0, y = 0, z = 1;  // idle lanes get a benign shift (pipeline.cpp:56-61)
    if (active) {
        x = a.shifts[3 * b];
        y = a.shifts[3 * b + 1];
        z = a.shifts[3 * b + 2];
    }
    const Angles<Real> ang = decompose_angles(x, y, z);
    const GeoView<TL> v(geo + 32 * t + lane, p_rot);
    Real* cbg = const_cast<Real*>(v.cb);
    Real* sbg = const_cast<Real*>(v.sb);
    Real* nsbg = const_cast<Real*>(v.nsb);
    Real* cag = const_cast<Real*>(v.ca);
    Real* sag = const_cast<Real*>(v.sa);
    Real* qag = const_cast<Real*>(v.qa);
    Real* qdg = const_cast<Real*>(v.qd);
    const Real inv = Real(1) / ang.rn;
    const Real base_a = src_local ? ang.rn : inv;
    const Real base_d = dst_local ? inv : ang.rn;
    *const_cast<Real*>(v.base_a) = base_a;
    *const_cast<Real*>(v.base_d) = base_d;
    c1s1[32 * t + lane] = ang.ca;  // the step of the column recurrence in phases A and D
    c1s1[L + 32 * t + lane] = ang.sa;
    Real c = 1, s = 0, ca = 1, sa = 0;
    Real qa = src_local ? Real(1) : base_a;  // base_a^(0 + q0)
    Real qd = dst_local ? Real(1) : base_d;
    for (int m = 0; m < p_rot + 2; ++m) {
        cbg[m * L] = c;
        sbg[m * L] = s;
        nsbg[m * L] = -s;
        if (m < p_rot) {
            cag[m * L] = ca;
            sag[m * L] = sa;
            qag[m * L] = qa;
            qdg[m * L] = qd;
        }
        const Real nc = fma_(c, ang.cb, -(s * ang.sb));
        const Real ns = fma_(s, ang.cb, c * ang.sb);
        c = nc;
        s = ns;
        const Real nca = fma_(ca, ang.ca, -(sa * ang.sa));
        const Real nsa = fma_(sa, ang.ca, ca * ang.sa);
        ca = nca;
        sa = nsa;
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

constexpr int CHK = 4;  // elements per chunk of the elementwise phases

// Arguments of elementwise_phase (one call per warp and group).
struct ElemArgs {
    const Real* in;            // sources (SoA), in_stride between coefficients
    int64_t in_stride;
    Real* out;                 // outputs or per-group partial sums (SoA)
    int64_t out_stride;
    const int32_t* src_index;  // accumulate mode: source of every pair, else null
    int64_t n;                 // translations of the launch
    const Real* geo_d;         // geometry scratch of the group phase D finishes, or null
    const Real* geo_a;         // geometry scratch of the group phase A loads, or null
    int64_t g_d, g_a;          // their group numbers
    int buf_off;               // element offsets into smem_raw: triangle,
    int cs_d_off, cs_a_off;    //   cos/sin(alpha) rows of the two groups
    int p_in, p_out, p_rot;
    int c_lo, c_hi;            // chunks of this warp
};

// Phases D and A on the chunks of one warp (reference pipeline.cpp:251-257 and
// :148-154). The triangle of order p_max is walked column by column (TriWalk) and cut
// into chunks of CHK elements; a warp owns a contiguous run of chunks. Phase D of group
// g and phase A of group g+1 touch an element only through its owner, so they run back
// to back per chunk with no barrier in between: the global loads of the next group are
// issued first and are in flight while the chunk of this group is rotated and reduced.
// Out of line so that its registers are not shared with the long-lived state of the
// kernel body.
//   D: rotate by -alpha, scale, then store (ACC = false) or reduce over the group
//      (ACC = true): the 32*TL lanes belong to one target, the 2 CHK values of a chunk
//      (re, im per element) are summed over the lanes with one transposing butterfly,
//      slots l and l+32 first (sharding.accumulation_tree restates the order).
//   A: load, rotate by +alpha, scale.
// The factors cos/sin(m alpha) and the scales are read from the geometry scratch at the
// first element only and then follow the walk: next row = scale times base
// (pipeline.cpp:81-89), next column = one step of the angle recurrence
// (pipeline.cpp:70-79), the very operations that filled the tables.
template <int TL, bool ACC>
__device__ __noinline__ void elementwise_phase(const ElemArgs e) {
    constexpr int L = 32 * TL;
    const int lane = threadIdx.x & 31;
    Real* sm = reinterpret_cast<Real*>(smem_raw);
    Real* buf = sm + e.buf_off + lane;
    const Real* csd = sm + e.cs_d_off + lane;
    const Real* csa = sm + e.cs_a_off + lane;
    const int p_in = e.p_in, p_out = e.p_out, p_rot = e.p_rot;
    const int p_max = max(p_in, p_out);
    const bool do_d = e.geo_d != nullptr, do_a = e.geo_a != nullptr;

    auto rot_seek = [&](RotWalk<TL>& r, const TriWalk& w, const Real* ca, const Real* sa,
                        const Real* qtab, const Real* basep) {
        const int m = min(w.m, p_rot - 1), n = min(w.n, p_rot - 1);  // past the end: unused
#pragma unroll
        for (int t = 0; t < TL; ++t) {
            r.c[t] = __ldcg(ca + m * L + 32 * t);
            r.s[t] = __ldcg(sa + m * L + 32 * t);
            r.qh[t] = __ldcg(qtab + m * L + 32 * t);
            r.q[t] = __ldcg(qtab + n * L + 32 * t);
            r.base[t] = __ldcg(basep + 32 * t);
        }
    };
    auto rot_advance = [&](TriWalk& w, RotWalk<TL>& r, const Real* cs) {
        ++w.n;
#pragma unroll
        for (int t = 0; t < TL; ++t) r.q[t] *= r.base[t];
        if (w.n == w.p) {
            ++w.m;
            w.n = w.m;
#pragma unroll
            for (int t = 0; t < TL; ++t) {
                const Real c1 = cs[32 * t], s1 = cs[L + 32 * t];
                const Real nc = fma_(r.c[t], c1, -(r.s[t] * s1));
                const Real ns = fma_(r.s[t], c1, r.c[t] * s1);
                r.c[t] = nc;
                r.s[t] = ns;
                r.qh[t] *= r.base[t];
                r.q[t] = r.qh[t];
            }
        }
    };

    TriWalk wd = tri_seek(CHK * e.c_lo, p_max), wa = wd;
    RotWalk<TL> rd, ra;
    int64_t bd[TL], srca[TL];
    bool actd[TL], acta[TL];
#pragma unroll
    for (int t = 0; t < TL; ++t) {
        bd[t] = e.g_d * L + 32 * t + lane;
        actd[t] = do_d && bd[t] < e.n;
        const int64_t bb = e.g_a * L + 32 * t + lane;
        srca[t] = bb;
        acta[t] = do_a && bb < e.n;
        if (acta[t] && ACC) {
            srca[t] = e.src_index[bb];
            acta[t] = srca[t] >= 0;
        }
        if (!acta[t]) srca[t] = 0;
    }
    if (do_d) {
        const GeoView<TL> gv(e.geo_d + lane, p_rot);
        rot_seek(rd, wd, gv.ca, gv.sa, gv.qd, gv.base_d);
    }
    if (do_a) {
        const GeoView<TL> gv(e.geo_a + lane, p_rot);
        rot_seek(ra, wa, gv.ca, gv.sa, gv.qa, gv.base_a);
    }

    // ---- D on all chunks of the warp
    if (do_d) {
        for (int ci = e.c_lo; ci < e.c_hi; ++ci) {
            if constexpr (!ACC) {
#pragma unroll
                for (int u = 0; u < CHK; ++u) {
                    if (wd.n < p_out) {
#pragma unroll
                        for (int t = 0; t < TL; ++t) {
                            const Real re = buf[t_re(wd.n, wd.m) * L + 32 * t];
                            const Real im = wd.m ? buf[t_im(wd.n, wd.m) * L + 32 * t] : Real(0);
                            const Real ms = -rd.s[t];
                            const Real nr = rd.q[t] * fma_(re, rd.c[t], -(im * ms));
                            const Real ni = rd.q[t] * fma_(re, ms, im * rd.c[t]);
                            if (actd[t]) {
                                const int64_t o = (int64_t)aos_re(wd.n, wd.m) * e.out_stride + bd[t];
                                __stcg(e.out + o, nr);
                                __stcg(e.out + o + e.out_stride, wd.m ? ni : Real(0));
                            }
                        }
                    }
                    rot_advance(wd, rd, csd);
                }
            } else {
                constexpr int NV = 2 * CHK, REP = 32 / NV;
                Real v[NV];
                int my_n = p_out, my_m = 0;  // the element whose sum this lane stores
#pragma unroll
                for (int u = 0; u < CHK; ++u) {
                    Real sr = 0, si = 0;
                    if (wd.n < p_out) {
#pragma unroll
                        for (int t = 0; t < TL; ++t) {
                            const Real re = buf[t_re(wd.n, wd.m) * L + 32 * t];
                            const Real im = wd.m ? buf[t_im(wd.n, wd.m) * L + 32 * t] : Real(0);
                            const Real ms = -rd.s[t];
                            const Real nr = rd.q[t] * fma_(re, rd.c[t], -(im * ms));
                            const Real ni = rd.q[t] * fma_(re, ms, im * rd.c[t]);
                            sr = t ? sr + nr : nr;
                            si = t ? si + ni : ni;
                        }
                    }
                    v[2 * u] = sr;
                    v[2 * u + 1] = si;
                    if (lane / (2 * REP) == u) {
                        my_n = wd.n;
                        my_m = wd.m;
                    }
                    rot_advance(wd, rd, csd);
                }
                lane_transpose_sum<NV>(v, lane);
                // lanes REP k .. REP k + REP-1 hold value k: element k >> 1, part k & 1
                const int part = (lane / REP) & 1;
                if (!(lane & (REP - 1)) && my_n < p_out && !(part && my_m == 0))
                    __stcg(e.out + (int64_t)(aos_re(my_n, my_m) + part) * e.out_stride + e.g_d, v[0]);
            }
        }
    }
    if (!do_a) return;

    // ---- A on the same chunks, two chunks of loads in flight. The addresses are always
    // valid (clamped; idle slots read source 0) and the values are zeroed only when
    // consumed, so that neither a branch nor a use stands between the loads.
    TriWalk wl = wa;  // load cursor, runs ahead of wa
    auto issue = [&](Real (&re)[CHK][TL], Real (&im)[CHK][TL]) {
#pragma unroll
        for (int u = 0; u < CHK; ++u) {
            const int64_t off =
                (int64_t)aos_re(min(wl.n, p_in - 1), min(wl.m, p_in - 1)) * e.in_stride;
#pragma unroll
            for (int t = 0; t < TL; ++t) {
                re[u][t] = __ldcg(e.in + off + srca[t]);
                im[u][t] = __ldcg(e.in + off + e.in_stride + srca[t]);
            }
            wl.advance();
        }
    };
    auto finish = [&](const Real (&re)[CHK][TL], const Real (&im)[CHK][TL]) {
#pragma unroll
        for (int u = 0; u < CHK; ++u) {
            if (wa.n < p_in) {
#pragma unroll
                for (int t = 0; t < TL; ++t) {
                    const Real xr = acta[t] ? re[u][t] : Real(0);
                    const Real xi = (acta[t] && wa.m) ? im[u][t] : Real(0);
                    const Real nr = ra.q[t] * fma_(xr, ra.c[t], -(xi * ra.s[t]));
                    const Real ni = ra.q[t] * fma_(xr, ra.s[t], xi * ra.c[t]);
                    buf[t_re(wa.n, wa.m) * L + 32 * t] = nr;
                    if (wa.m) buf[t_im(wa.n, wa.m) * L + 32 * t] = ni;
                }
            }
            rot_advance(wa, ra, csa);
        }
    };
    Real re0[CHK][TL], im0[CHK][TL], re1[CHK][TL], im1[CHK][TL];
    if (e.c_lo < e.c_hi) issue(re0, im0);
    for (int ci = e.c_lo; ci < e.c_hi; ci += 2) {
        if (ci + 1 < e.c_hi) issue(re1, im1);
        finish(re0, im0);
        if (ci + 1 < e.c_hi) {
            if (ci + 2 < e.c_hi) issue(re0, im0);
            finish(re1, im1);
        }
    }
}

// The elementwise phase is entered through a pointer read at run time: an indirect call
// uses the plain calling convention, which gives the callee its own registers (a direct
// call makes ptxas fit caller and callee into one register budget and starves it).
using ElemFn = void (*)(const ElemArgs);
__device__ ElemFn g_elem_fn[2] = {elementwise_phase<2, false>, elementwise_phase<2, true>};

template <int TL>
__global__ void __launch_bounds__(384, 1)
translate_tiled_kernel(TranslateArgs<Real> a, TiledTables tt, int64_t n_groups, int p_rot,
                       int tab_len) {
    constexpr int L = 32 * TL;
    if (a.fail_flag && *a.fail_flag) return;

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int W = blockDim.x >> 5;
    const TiledLayout<TL> lay{p_rot, (size_t)tab_len};

    Real* sm = reinterpret_cast<Real*>(smem_raw);
    Real* tab = sm;  // 16-byte aligned
    Real* buf = sm + lay.tab_len + lane;
    uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + lay.tab_len + lay.buf_elems());
    int* counters = reinterpret_cast<int*>(mbar + 1);
    Real* geo_base = tt.scratch + (size_t)blockIdx.x * 2 * geo_elems<TL>(p_rot);

    const int kind = a.kind, p_in = a.p_in, p_out = a.p_out;
    const bool src_local = kind == KIND_L2L;
    const bool dst_local = kind != KIND_M2M;
    const int side_fwd = src_local ? 1 : 0, side_bwd = dst_local ? 1 : 0;
    const bool two_sides = side_fwd != side_bwd;
    const int cols = min(p_in, p_out);
    const bool accumulate = a.src_index != nullptr;

    // table staging: one mbarrier, completions alternate fwd / bwd tables
    uint32_t tab_phase = 0;
    if (threadIdx.x == 0) {
        mbar_init(mbar, 1);
        bulk_load(tab, tt.stream[side_fwd], two_sides ? tt.bytes[0] : max(tt.bytes[0], tt.bytes[1]),
                  mbar);
    }
    bool tab_pending = true;  // a bulk copy is in flight that the next swap phase must wait for

    long long t_prev = clock64();
#define SFMM_PHASE_MARK(idx)                                              \
    if (a.phase_clocks && blockIdx.x == 0 && threadIdx.x == 0) {          \
        const long long now = clock64();                                  \
        a.phase_clocks[idx] += now - t_prev;                              \
        t_prev = now;                                                     \
    }
    // elementwise phases (elementwise_phase): warp w owns a contiguous run of chunks
    const int p_max = max(p_in, p_out);
    const int n_chunks = (p_max * (p_max + 1) / 2 + CHK - 1) / CHK;
    const int cs_off = (int)(lay.tab_len + lay.buf_elems()) + 32 / (int)sizeof(Real);
    Real* c1s1 = sm + cs_off;  // [2 groups][cos alpha | sin alpha][L]
    ElemArgs ea;
    ea.in = a.in;
    ea.in_stride = a.in_stride;
    ea.out = a.out;
    ea.out_stride = a.out_stride;
    ea.src_index = a.src_index;
    ea.n = a.n;
    ea.buf_off = (int)lay.tab_len;
    ea.p_in = p_in;
    ea.p_out = p_out;
    ea.p_rot = p_rot;
    ea.c_lo = n_chunks * warp / W;
    ea.c_hi = n_chunks * (warp + 1) / W;

    // geometry and phase A of the first group; later groups are prepared one group
    // ahead (geometry inside phase C, phase A fused behind phase D)
    geometry_phase<TL>(a, blockIdx.x, p_rot, geo_base, c1s1, src_local, dst_local, warp, lane);
    __syncthreads();
    ea.geo_d = nullptr;
    ea.geo_a = geo_base;
    ea.g_d = 0;
    ea.g_a = blockIdx.x;
    ea.cs_d_off = ea.cs_a_off = cs_off;
    const ElemFn elem_fn = g_elem_fn[accumulate ? 1 : 0];
    elem_fn(ea);
    int parity = 0;
    for (int64_t g = blockIdx.x; g < n_groups; g += gridDim.x, parity ^= 1) {
        const GeoView<TL> gv(geo_base + (size_t)parity * geo_elems<TL>(p_rot) + lane, p_rot);
        const GeoView<TL> gvn(geo_base + (size_t)(parity ^ 1) * geo_elems<TL>(p_rot) + lane, p_rot);
        const bool has_next = g + gridDim.x < n_groups;
        int64_t b[TL];
        bool active[TL];
#pragma unroll
        for (int t = 0; t < TL; ++t) {
            b[t] = g * L + 32 * t + lane;
            active[t] = b[t] < a.n;
        }
        if (threadIdx.x == 0) counters[0] = counters[1] = counters[2] = 0;
        if (tab_pending) {
            mbar_wait(mbar, tab_phase);
            tab_phase ^= 1;
            tab_pending = false;
        }
        __syncthreads();  // phase A of this group, its operator stream and the counters are in place
        SFMM_PHASE_MARK(1)

        // ---- B: forward swap passes, largest rows first
        {
            Ctx<TL> c{(int)lay.tab_len, 0, gv.cb, gv.sb, src_local};
            for (int task = fetch_task(&counters[0], lane); task < 2 * p_in;
                 task = fetch_task(&counters[0], lane)) {
                const int n = p_in - 1 - (task >> 1);
                half_task_dispatch<TL>(c, n, task & 1, n);
            }
        }
        __syncthreads();
        SFMM_PHASE_MARK(2)
        if (two_sides) {  // stage the backward-side stream while the z-step runs
            if (threadIdx.x == 0) bulk_load(tab, tt.stream[side_bwd], tt.bytes[1], mbar);
            tab_pending = true;
        }

        // ---- Z: z-axis step per (column, re|im), longest columns first
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

        // ---- C: backward swap passes; columns >= cols of the z-step output are
        // zero (pipeline.cpp:229-246) and are skipped, which is exact. The first
        // TL warps prepare the geometry of the NEXT group before joining the queue:
        // its serial recurrences hide behind the other warps' products.
        {
            if (has_next)
                geometry_phase<TL>(a, g + gridDim.x, p_rot,
                                   geo_base + (size_t)(parity ^ 1) * geo_elems<TL>(p_rot),
                                   c1s1 + (parity ^ 1) * 2 * L, src_local, dst_local, warp, lane);
            Ctx<TL> c{(int)lay.tab_len, 0, gv.cb, gv.nsb, dst_local};
            for (int task = fetch_task(&counters[2], lane); task < 2 * p_out;
                 task = fetch_task(&counters[2], lane)) {
                const int n = p_out - 1 - (task >> 1);
                half_task_dispatch<TL>(c, n, task & 1, min(n, cols - 1));
            }
        }
        __syncthreads();
        SFMM_PHASE_MARK(4)
        if (two_sides && has_next) {  // forward-side stream for the next group
            if (threadIdx.x == 0) bulk_load(tab, tt.stream[side_fwd], tt.bytes[0], mbar);
            tab_pending = true;
        }

        // ---- D of this group, A of the next one
        ea.geo_d = geo_base + (size_t)parity * geo_elems<TL>(p_rot);
        ea.geo_a = has_next ? geo_base + (size_t)(parity ^ 1) * geo_elems<TL>(p_rot) : nullptr;
        ea.g_d = g;
        ea.g_a = g + gridDim.x;
        ea.cs_d_off = cs_off + parity * 2 * L;
        ea.cs_a_off = cs_off + (parity ^ 1) * 2 * L;
        elem_fn(ea);
        SFMM_PHASE_MARK(5)
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

int tiled_warps_for(int p_rot) {
    if (const char* env = getenv("SFMM_TILED_WARPS")) {
        const int w = atoi(env);
        if (w >= 2 && w <= 12) return w;
    }
    if (p_rot >= 12) return 12;
    return 4;
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
    const int block = 32 * tiled_warps_for(p_rot);
    auto kern = translate_tiled_kernel<TL>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 1;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorLaunchOutOfResources;
    const int grid = (int)std::min<int64_t>(n_groups, (int64_t)sm_count * per_sm);

    TiledTables tt;
    tt.stream[0] = t.stream[0];
    tt.stream[1] = t.stream[1];
    tt.bytes[0] = (uint32_t)(staged(a.p_in) * sizeof(Real));
    tt.bytes[1] = (uint32_t)(staged(a.p_out) * sizeof(Real));
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

// FP64 tensor-core translation kernel ("mma"), orders 9..30 in double precision.
//
// Why it exists: the tiled kernel (kernel_tiled.inl) feeds every DFMA with a
// warp-uniform shared-memory load of the swap-matrix entry and is bound by the
// load/store unit at ~0.3 of the FP64 peak. Here the four products of a swap pass
// (reference pipeline.cpp:118-136, kernels.cpp:33-114) and the z-axis step
// (kernels.cpp:118-196) run on the FP64 tensor-core instruction
// mma.sync.m8n8k4.f64 (SASS DMMA): one instruction does 256 multiply-adds from
// four 64-bit register operands per lane, so operator entries cost one coalesced
// 64-bit load per 8 x 4 block and translation group instead of one shared-memory
// broadcast per two DFMAs. DMMA accumulates k-ascending with one rounding per
// multiply-add, i.e. it IS the reference's fma chain (tests/test_gpu_parity.py
// checks every coefficient bit for bit); structural zeros and padding contribute
// fma(0, x, acc) = acc exactly.
//
// Data flow of one unit of G = 8 NTB translations (G = 32 for p <= 20):
//   * the 8 translations of a "t-block" are the 8 rows of the A operand; lane
//     (t, q) = (lane >> 2, lane & 3) holds member 4 kb + q of a parity class;
//   * the operator is the B operand, pre-packed per block in fragment order with
//     the output permutation sigma (tables.hpp, pack_frags) so that the accumulator
//     registers of product 1 are, unchanged, the A operands of product 2:
//     swap -> rotate(beta) -> swap never leaves the registers of a lane;
//   * the coefficient triangle of the unit lives in shared memory as
//     buf[idx(n, m, part)][G] with the translation position XOR-swizzled by
//     ((m >> 1) + n) & 3 (bits 2..3): fragment accesses (4 consecutive class
//     members or 4 consecutive rows x 8 translations), and the lane-per-translation
//     accesses of the elementwise warps are all bank-conflict free.
//
// Schedule: warp-specialised producer / consumer over two triangle buffers.
//   E warps (NE = 4, lane = translation): phase D of unit i-2 (rotate by -alpha,
//     scale, store or reduce over the lanes) fused row by row with phase A of unit
//     i (gather, rotate by +alpha, scale), plus the beta table of unit i
//     (pipeline.cpp:52-91, 148-154, 251-265);
//   M warps (NM = 12): forward swap passes B, z-step Z, backward swap passes C of
//     unit i-1 on the other buffer (dynamic task queues, largest first).
// The two sides meet at mbarriers (full / empty per buffer): the latency-bound
// elementwise work never stalls the tensor pipe.
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "device_math.cuh"
#include "kernel_generic.cuh"
#include "sfmm_internal.hpp"

namespace sfmm {
namespace {

constexpr int PMAX = 30;                  // largest max(p_in, p_out)
constexpr int NE = 4, NM = 12;            // elementwise / tensor warps
constexpr int NTHREADS = 32 * (NE + NM);
constexpr int TB = 2;                     // t-blocks (of 8 translations) per M task
constexpr int ZC = 40;                    // centre of the Toeplitz tables
constexpr int ZSEG = 80;                  // one z-table segment
constexpr int Z_FAC = 0, Z_LOW = ZSEG, Z_UP = 2 * ZSEG;

// first fragment of block n*4 + {F/E, F/O, G/E, G/O} (same for both sides)
__constant__ int c_foff[PMAX * 4 + 1];

extern __shared__ __align__(16) unsigned char smem_raw[];

__device__ __forceinline__ int class_size(int n, int cls) { return cls ? (n + 1) >> 1 : (n >> 1) + 1; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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
// barrier among the M warps only
__device__ __forceinline__ void bar_m() { asm volatile("bar.sync 1, %0;" ::"n"(NM * 32) : "memory"); }

__device__ __forceinline__ int fetch_task(int* counter, int lane) {
    int t = 0;
    if (lane == 0)
        asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(t) : "r"(smem_u32(counter)) : "memory");
    return __shfl_sync(0xffffffffu, t, 0);
}

// D (8x8, lane holds columns 2q, 2q+1 of row t) += A (8x4, lane holds (t, q)) * B (4x8,
// lane holds (row q, column t)); k-ascending fma chain per output (PTX ISA, mma.m8n8k4.f64)
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

struct MCtx {
    double* buf;          // triangle of the buffer
    const double2* beta;  // (cos, sin)(m beta) of the buffer, [m][G], position ^ (((m >> 1) & 3) << 1)
    const double* frags;  // fragment stream of the side in use (global, read through L1)
    bool local_side;      // transposed blocks; halve / double re_0 (pipeline.cpp:155-157, 247-249)
    bool bwd;             // backward pass: rotate by -beta
};

// One parity half of swap -> rotate(+-beta) -> swap on row n for t-blocks
// TB h .. TB h + TB-1, in place in the shared-memory triangle. MB = number of 8-wide
// output blocks of the rotation class cls (1: up to 8 members, 2: up to 16).
// mmax < n only for backward rows with p_out > p_in (inputs in columns >= min(p_in, p_out)
// are zero, pipeline.cpp:229-246).
template <int NTB, int MB>
__device__ __noinline__ void mma_half_task(const MCtx c, int n, int cls, int h, int mmax) {
    constexpr int G = 8 * NTB;
    const int lane = threadIdx.x & 31, t = lane >> 2, q = lane & 3;
    const int nc = class_size(n, cls);       // members of the rotation class (== of class cF)
    const int cF = (n - cls) & 1, cG = cF ^ 1;
    const int nG = class_size(n, cG);
    const int g0 = cG ? 0 : 1;               // class index 0 of E is m = 0: no imaginary part
    const int kendF = mmax >= cF ? min(nc, ((mmax - cF) >> 1) + 1) : 0;
    const int kendG = mmax >= cG ? min(nG, ((mmax - cG) >> 1) + 1) : 0;
    const int KB1 = (max(kendF, kendG) + 3) >> 2;
    const int KB2 = (nc + 3) >> 2;
    const int MBG = (nG + 7) >> 3;
    const bool halve = c.local_side && cF == 0;

    // member j = 4 kb + q of class cF: re at idx n^2 + 2 cF + 4 j; of class cG: im at
    // n^2 + 2 cG + 4 j - 1; swizzle key ((m >> 1) + n) & 3 = (q + n) & 3 for both
    const int key = ((q + n) & 3) << 2;
    int pos[TB];
#pragma unroll
    for (int tb = 0; tb < TB; ++tb) pos[tb] = (8 * (TB * h + tb) + t) ^ key;
    double* re0 = c.buf + (n * n + 2 * cF + 4 * q) * G;
    double* im0 = c.buf + (n * n + 2 * cG + 4 * q - 1) * G;

    double cre[MB][2][TB], cim[MB][2][TB];
#pragma unroll
    for (int mb = 0; mb < MB; ++mb)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
#pragma unroll
            for (int tb = 0; tb < TB; ++tb) cre[mb][hh][tb] = cim[mb][hh][tb] = 0.0;

    // ---- product 1: u_re = A_F[cls, cF] re[cF], u_im = A_G[cls, cG] im[cG]
    {
        const double* F1 = c.frags + 32 * (size_t)c_foff[n * 4 + cls] + lane;
        const double* G1 = c.frags + 32 * (size_t)c_foff[n * 4 + 2 + cls] + lane;
        double f[MB], g[MB], are[TB], aim[TB];
        auto load = [&](int kb) {
#pragma unroll
            for (int mb = 0; mb < MB; ++mb) {
                f[mb] = __ldg(F1 + (kb * MB + mb) * 32);
                g[mb] = __ldg(G1 + (kb * MB + mb) * 32);
            }
            const int j = 4 * kb + q;
            const bool vF = j < kendF, vG = j >= g0 && j < kendG;
#pragma unroll
            for (int tb = 0; tb < TB; ++tb) {
                are[tb] = vF ? re0[kb * 16 * G + pos[tb]] : 0.0;
                aim[tb] = vG ? im0[kb * 16 * G + pos[tb]] : 0.0;
                if (halve && j == 0) are[tb] *= 0.5;
            }
        };
        load(0);
#pragma unroll 1
        for (int kb = 0; kb < KB1; ++kb) {
            double fc[MB], gc[MB], ac[TB], bc[TB];
#pragma unroll
            for (int mb = 0; mb < MB; ++mb) fc[mb] = f[mb], gc[mb] = g[mb];
#pragma unroll
            for (int tb = 0; tb < TB; ++tb) ac[tb] = are[tb], bc[tb] = aim[tb];
            if (kb + 1 < KB1) load(kb + 1);
#pragma unroll
            for (int tb = 0; tb < TB; ++tb)
#pragma unroll
                for (int mb = 0; mb < MB; ++mb) {
                    dmma(cre[mb][0][tb], cre[mb][1][tb], ac[tb], fc[mb]);
                    dmma(cim[mb][0][tb], cim[mb][1][tb], bc[tb], gc[mb]);
                }
        }
    }
    // ---- rotate by +-beta (kernels.cpp:211-217). Register (mb, hh) of a lane is member
    // j = 8 mb + 4 hh + q of class cls, m = cls + 2 j; padding members are exactly zero and
    // read the factors of the last member.
#pragma unroll
    for (int mb = 0; mb < MB; ++mb)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const int m = cls + 2 * min(8 * mb + 4 * hh + q, nc - 1);
            const double2* bp = c.beta + m * G;
            const int kx = ((m >> 1) & 3) << 1;
#pragma unroll
            for (int tb = 0; tb < TB; ++tb) {
                const double2 cs = bp[(8 * (TB * h + tb) + t) ^ kx];
                const double s = c.bwd ? -cs.y : cs.y;
                const double a = cre[mb][hh][tb], b = cim[mb][hh][tb];
                cre[mb][hh][tb] = fma_(a, cs.x, -(b * s));
                cim[mb][hh][tb] = fma_(a, s, b * cs.x);
            }
        }
    // ---- product 2: re[cF] = A_F[cF, cls] u_re, im[cG] = A_G[cG, cls] u_im; the accumulator
    // registers (mb, hh) of product 1 are the A operands of input block kb2 = 2 mb + hh
    {
        const double* F2 = c.frags + 32 * (size_t)c_foff[n * 4 + cF] + lane;
        const double* G2 = c.frags + 32 * (size_t)c_foff[n * 4 + 2 + cG] + lane;
        const int mb_end = max(MB, MBG);
#pragma unroll 1
        for (int mb2 = 0; mb2 < mb_end; ++mb2) {
            const bool doF = mb2 < MB, doG = mb2 < MBG;
            double ore[2][TB], oim[2][TB];
#pragma unroll
            for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                for (int tb = 0; tb < TB; ++tb) ore[hh][tb] = oim[hh][tb] = 0.0;
            double f2[2 * MB], g2[2 * MB];
#pragma unroll
            for (int kb2 = 0; kb2 < 2 * MB; ++kb2) {
                f2[kb2] = (doF && kb2 < KB2) ? __ldg(F2 + (kb2 * MB + mb2) * 32) : 0.0;
                g2[kb2] = (doG && kb2 < KB2) ? __ldg(G2 + (kb2 * MBG + mb2) * 32) : 0.0;
            }
#pragma unroll
            for (int kb2 = 0; kb2 < 2 * MB; ++kb2) {
                if (kb2 < KB2) {
#pragma unroll
                    for (int tb = 0; tb < TB; ++tb) {
                        if (doF) dmma(ore[0][tb], ore[1][tb], cre[kb2 >> 1][kb2 & 1][tb], f2[kb2]);
                        if (doG) dmma(oim[0][tb], oim[1][tb], cim[kb2 >> 1][kb2 & 1][tb], g2[kb2]);
                    }
                }
            }
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const int j2 = 8 * mb2 + 4 * hh + q;
                const int off = (2 * mb2 + hh) * 16 * G;
                if (doF && j2 < nc) {
#pragma unroll
                    for (int tb = 0; tb < TB; ++tb) {
                        double v = ore[hh][tb];
                        if (halve && j2 == 0) v *= 2.0;
                        re0[off + pos[tb]] = v;
                    }
                }
                if (doG && j2 >= g0 && j2 < nG) {
#pragma unroll
                    for (int tb = 0; tb < TB; ++tb) im0[off + pos[tb]] = oim[hh][tb];
                }
            }
        }
    }
}

template <int NTB>
__device__ __forceinline__ void half_task_dispatch(const MCtx c, int n, int cls, int h, int mmax) {
    if (class_size(n, cls) <= 8) mma_half_task<NTB, 1>(c, n, cls, h, mmax);
    else mma_half_task<NTB, 2>(c, n, cls, h, mmax);
}

// z-axis step on column m (re and im) for t-blocks TB h .. TB h + TB-1, in place
// (reference kernels.cpp:118-196): out_i = sum_k W[i][k] in_k with
//   M2L  W = (2m + i + k)!              (Hankel; sign (-1)^i of the backward gather,
//                                        pipeline.cpp:235-239, applied at the store)
//   M2M  W = (-1)^(i-k) / (i-k)!, k <= i (lower Toeplitz)
//   L2L  W = 1 / (k-i)!, k >= i          (upper Toeplitz)
// The B fragments are generated from the small tables in shared memory:
// value(kk, ii) = zt[zbase + s1 kk + s2 ii].
template <int NTB, int NB>
__device__ __noinline__ void mma_zstep(double* buf, const double* zt, int kind, int p_in, int p_out,
                                       int m, int h) {
    constexpr int G = 8 * NTB;
    const int lane = threadIdx.x & 31, t = lane >> 2, q = lane & 3;
    const int K = p_in - m, N = p_out - m;
    const int KB = (K + 3) >> 2;
    const int key = (((m >> 1) + m + q) & 3) << 2;
    int pos[TB];
#pragma unroll
    for (int tb = 0; tb < TB; ++tb) pos[tb] = (8 * (TB * h + tb) + t) ^ key;
    const bool has_im = m > 0;
    // operator entry of lane (row kk = 4 kb + q, column ii = sigma(nb, t))
    const int sig = (t >> 1) + 4 * (t & 1);
    int zoff, s1, s2;
    if (kind == KIND_M2L) zoff = Z_FAC + 2 * m, s1 = 1, s2 = 1;
    else if (kind == KIND_M2M) zoff = Z_LOW + ZC, s1 = -1, s2 = 1;
    else zoff = Z_UP + ZC, s1 = 1, s2 = -1;
    const double* zl = zt + zoff + s1 * q + s2 * sig;

    double acc[2][TB][NB][2];
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int tb = 0; tb < TB; ++tb)
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) acc[p][tb][nb][0] = acc[p][tb][nb][1] = 0.0;

#pragma unroll 1
    for (int kb = 0; kb < KB; ++kb) {
        const int k = 4 * kb + q, nk = m + k;
        const bool valid = k < K;
        const double* src = buf + (nk * nk + 2 * m) * G;
        double x[2][TB];
#pragma unroll
        for (int tb = 0; tb < TB; ++tb) {
            x[0][tb] = valid ? src[pos[tb]] : 0.0;
            x[1][tb] = (valid && has_im) ? src[pos[tb] - G] : 0.0;
        }
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
            // all-zero operator blocks of the triangular kinds are skipped (exact)
            bool nz = 8 * nb < N;
            if (kind == KIND_M2M) nz = nz && 4 * kb <= 8 * nb + 7;
            if (kind == KIND_L2L) nz = nz && 4 * kb + 3 >= 8 * nb;
            if (!nz) continue;
            const double bf = zl[s1 * 4 * kb + s2 * 8 * nb];
#pragma unroll
            for (int tb = 0; tb < TB; ++tb) {
                dmma(acc[0][tb][nb][0], acc[0][tb][nb][1], x[0][tb], bf);
                if (has_im) dmma(acc[1][tb][nb][0], acc[1][tb][nb][1], x[1][tb], bf);
            }
        }
    }
    const bool neg = kind == KIND_M2L && (q & 1);
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const int i = 8 * nb + 4 * hh + q, ni = m + i;
            if (i < N) {
                double* dst = buf + (ni * ni + 2 * m) * G;
#pragma unroll
                for (int tb = 0; tb < TB; ++tb) {
                    const double vr = acc[0][tb][nb][hh];
                    dst[pos[tb]] = neg ? -vr : vr;
                    if (has_im) {
                        const double vi = acc[1][tb][nb][hh];
                        dst[pos[tb] - G] = neg ? -vi : vi;
                    }
                }
            }
        }
}

template <int NTB>
__device__ __forceinline__ void zstep_dispatch(double* buf, const double* zt, int kind, int p_in,
                                               int p_out, int m, int h) {
    const int nb = (p_out - m + 7) >> 3;
    switch (nb) {
        case 1: mma_zstep<NTB, 1>(buf, zt, kind, p_in, p_out, m, h); break;
        case 2: mma_zstep<NTB, 2>(buf, zt, kind, p_in, p_out, m, h); break;
        case 3: mma_zstep<NTB, 3>(buf, zt, kind, p_in, p_out, m, h); break;
        default: mma_zstep<NTB, 4>(buf, zt, kind, p_in, p_out, m, h); break;
    }
}

// Transposing butterfly over the 32 lanes (as in kernel_tiled.inl): every lane enters
// with NV values and leaves with the sum over all lanes of value index lane / (32 / NV)
// in v[0]; per value the additions pair lanes at distance 16, 8, 4, 2, 1.
template <int NV>
__device__ __forceinline__ void lane_transpose_sum(double (&v)[NV], int lane) {
    int d = 16;
#pragma unroll
    for (int h = NV / 2; h >= 1; h >>= 1, d >>= 1) {
        const bool upper = lane & d;
#pragma unroll
        for (int j = 0; j < h; ++j) {
            const double send = upper ? v[j] : v[j + h];
            const double keep = upper ? v[j + h] : v[j];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, d);
        }
    }
#pragma unroll
    for (d = 16 / NV; d >= 1; d >>= 1) v[0] = v[0] + __shfl_xor_sync(0xffffffffu, v[0], d);
}

__device__ __forceinline__ void load4_cg(const double* p, double (&x)[4]) {
    asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(x[0]), "=d"(x[1]), "=d"(x[2]), "=d"(x[3])
                 : "l"(p));
}

struct LaneGeo {
    double rn, ca, sa, cb, sb, inv;
};

// decomposed shift of translation b (geometry.cpp:11-30); idle lanes get the benign
// shift (0, 0, 1) like the reference's idle columns (pipeline.cpp:56-61)
__device__ __forceinline__ LaneGeo load_geo(const TranslateArgs<double>& a, int64_t b, bool valid) {
    LaneGeo g;
    if (a.angles) {
        if (valid) {
            g.rn = a.angles[b];
            g.ca = a.angles[a.n + b];
            g.sa = a.angles[2 * a.n + b];
            g.cb = a.angles[3 * a.n + b];
            g.sb = a.angles[4 * a.n + b];
            g.inv = a.angles[5 * a.n + b];
            return g;
        }
        g.rn = 1, g.ca = 1, g.sa = 0, g.cb = 1, g.sb = -0.0, g.inv = 1;
        return g;
    }
    double x = 0, y = 0, z = 1;
    if (valid) {
        x = a.shifts[3 * b];
        y = a.shifts[3 * b + 1];
        z = a.shifts[3 * b + 2];
    }
    const Angles<double> ang = decompose_angles(x, y, z);
    g.rn = ang.rn, g.ca = ang.ca, g.sa = ang.sa, g.cb = ang.cb, g.sb = ang.sb;
    g.inv = 1.0 / ang.rn;
    return g;
}

struct MmaTables {
    const double* frags[2];  // [0] multipole side, [1] local side
    const double *fac, *inv, *winv;
    int nfac, ninv;
};

constexpr int CH = 4;  // elements (re, im pairs) per chunk of the elementwise phases

// The elementwise phases of E warp `e` for one trip: phase D of unit_d and phase A of
// unit_a on the same buffer, row by row (a row is read by D before A overwrites it).
// Rows are dealt to the warps in a snake order (balanced lengths) and visited in
// ascending order, so the powers of |r| follow by repeated multiplication exactly as
// the reference builds its tables (pipeline.cpp:81-89). cos/sin(m alpha) follow the
// row by the angle recurrence of pipeline.cpp:70-79 from (1, 0).
template <int NTB, bool ACC, bool ROWS>
__device__ __forceinline__ void elementwise_trip(const TranslateArgs<double>& a, int e, int lane,
                                                 int64_t unit_a, int64_t unit_d, double* buf,
                                                 double2* beta, int p_rot) {
    constexpr int G = 8 * NTB;
    const int kind = a.kind, p_in = a.p_in, p_out = a.p_out;
    const bool src_local = kind == KIND_L2L, dst_local = kind != KIND_M2M;
    const bool lane_ok = lane < G;
    const int lp = lane & (G - 1);
    const bool do_a = unit_a >= 0, do_d = unit_d >= 0;

    // ---- per-lane setup of phase A
    const int64_t ba = (do_a ? unit_a : 0) * G + lp;
    bool act_a = do_a && lane_ok && ba < a.n;
    int64_t src = ba;
    if (ACC && act_a) {
        const int32_t s = a.src_index[ba];
        act_a = s >= 0;
        src = s >= 0 ? s : 0;
    }
    const LaneGeo ga = load_geo(a, ba, do_a && lane_ok && ba < a.n && (!ACC || a.angles || act_a));
    const double* pa = ROWS ? a.in + src * a.in_stride : a.in + src;
    const double base_a = src_local ? ga.rn : ga.inv;
    double qa = src_local ? 1.0 : base_a;  // scale of row 0; row n: times base_a^n
    const double ac1 = fma_(1.0, ga.ca, -(0.0 * ga.sa)), as1 = fma_(0.0, ga.ca, 1.0 * ga.sa);

    // ---- beta table of unit_a (warp 0): (cos, sin)(m beta), m < p_rot
    if (e == 0 && do_a && lane_ok) {
        double c = 1, s = 0;
        for (int m = 0; m < p_rot; ++m) {
            beta[m * G + (lp ^ (((m >> 1) & 3) << 1))] = make_double2(c, s);
            const double nc = fma_(c, ga.cb, -(s * ga.sb));
            const double ns = fma_(s, ga.cb, c * ga.sb);
            c = nc;
            s = ns;
        }
    }

    // ---- per-lane setup of phase D
    const int64_t bd = (do_d ? unit_d : 0) * G + lp;
    const bool act_d = do_d && lane_ok && bd < a.n;
    const LaneGeo gd = load_geo(a, bd, act_d);
    const double base_d = dst_local ? gd.inv : gd.rn;
    double qd = dst_local ? 1.0 : base_d;
    const double dc1 = fma_(1.0, gd.ca, -(0.0 * gd.sa)), ds1 = fma_(0.0, gd.ca, 1.0 * gd.sa);

    const int p_max = max(p_in, p_out);
    int n_at = 0;  // row the running powers qa, qd belong to
    for (int blk = 0; blk * 2 * NE < p_max; ++blk)
        for (int side = 0; side < 2; ++side) {
            const int n = blk * 2 * NE + (side ? 2 * NE - 1 - e : e);
            if (n >= p_max) continue;
            for (; n_at < n; ++n_at) {
                qa *= base_a;
                qd *= base_d;
            }
            const bool row_d = do_d && n < p_out, row_a = do_a && n < p_in;
            if (!row_d && !row_a) continue;
            const int nn = n * n;

            // ---- A, first part: the loads of the first two chunks are in flight during D
            double xa[2][2 * CH];
            const double* prow = ROWS ? pa + rows_off(n) : pa + (int64_t)aos_re(n, 0) * a.in_stride;
            auto issue = [&](int m0, double (&x)[2 * CH]) {
                if (!act_a) {
#pragma unroll
                    for (int j = 0; j < 2 * CH; ++j) x[j] = 0.0;
                    return;
                }
                if constexpr (ROWS) {
#pragma unroll
                    for (int j = 0; j < CH / 2; ++j) {
                        double v[4];
                        load4_cg(prow + 4 * min((m0 >> 1) + j, n >> 1), v);
                        x[4 * j] = v[0], x[4 * j + 1] = v[1], x[4 * j + 2] = v[2], x[4 * j + 3] = v[3];
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < CH; ++u) {
                        const int64_t off = (int64_t)(2 * min(m0 + u, n)) * a.in_stride;
                        x[2 * u] = __ldcg(prow + off);
                        x[2 * u + 1] = __ldcg(prow + off + a.in_stride);
                    }
                }
            };
            if (row_a) {
                issue(0, xa[0]);
                if (CH <= n) issue(CH, xa[1]);
            }

            // ---- D: rotate by -alpha, scale, store or reduce over the lanes of the unit
            if (row_d) {
                double c = 1, s = 0;
                for (int m0 = 0; m0 <= n; m0 += CH) {
                    double v[2 * CH];
#pragma unroll
                    for (int j = 0; j < 2 * CH; ++j) v[j] = 0.0;
#pragma unroll
                    for (int u = 0; u < CH; ++u) {
                        const int m = m0 + u;
                        if (m > n) break;
                        const int px = lp ^ ((((m >> 1) + n) & 3) << 2);
                        const double re = buf[(nn + 2 * m) * G + px];
                        const double im = m ? buf[(nn + 2 * m - 1) * G + px] : 0.0;
                        const double ms = -s;
                        const double nr = qd * fma_(re, c, -(im * ms));
                        const double ni = qd * fma_(re, ms, im * c);
                        if constexpr (ACC) {
                            v[2 * u] = lane_ok ? nr : 0.0;
                            v[2 * u + 1] = lane_ok ? ni : 0.0;
                        } else {
                            if (act_d) {
                                const int64_t o = (int64_t)aos_re(n, m) * a.out_stride + bd;
                                __stcg(a.out + o, nr);
                                __stcg(a.out + o + a.out_stride, m ? ni : 0.0);
                            }
                        }
                        const double nc = fma_(c, dc1, -(s * ds1));
                        const double ns = fma_(s, dc1, c * ds1);
                        c = nc;
                        s = ns;
                    }
                    if constexpr (ACC) {
                        constexpr int NV = 2 * CH, REP = 32 / NV;
                        lane_transpose_sum<NV>(v, lane);
                        // lanes REP k .. REP k + REP-1 hold value k: element k >> 1, part k & 1
                        const int k = lane / REP, m = m0 + (k >> 1), part = k & 1;
                        if (!(lane & (REP - 1)) && m <= n && !(part && m == 0))
                            __stcg(a.out + (int64_t)(aos_re(n, m) + part) * a.out_stride + unit_d, v[0]);
                    }
                }
            }
            if (!row_a) continue;

            // ---- A, second part: rotate by +alpha, scale, into the triangle
            const double aq = act_a ? qa : 0.0;
            double c = 1, s = 0;
            for (int m0 = 0, par = 0; m0 <= n; m0 += CH, par ^= 1) {
                double x[2 * CH];
#pragma unroll
                for (int j = 0; j < 2 * CH; ++j) x[j] = par ? xa[1][j] : xa[0][j];
                if (m0 + 2 * CH <= n) {
                    if (par) issue(m0 + 2 * CH, xa[1]);
                    else issue(m0 + 2 * CH, xa[0]);
                }
#pragma unroll
                for (int u = 0; u < CH; ++u) {
                    const int m = m0 + u;
                    if (m > n) break;
                    const double xr = x[2 * u];
                    const double xi = m ? x[2 * u + 1] : 0.0;
                    const double nr = aq * fma_(xr, c, -(xi * s));
                    const double ni = aq * fma_(xr, s, xi * c);
                    if (lane_ok) {
                        const int px = lp ^ ((((m >> 1) + n) & 3) << 2);
                        buf[(nn + 2 * m) * G + px] = nr;
                        if (m) buf[(nn + 2 * m - 1) * G + px] = ni;
                    }
                    const double nc = fma_(c, ac1, -(s * as1));
                    const double ns = fma_(s, ac1, c * as1);
                    c = nc;
                    s = ns;
                }
            }
        }
}

struct MmaLayout {
    int p_rot, G, nbuf;
    size_t tri() const { return (size_t)p_rot * p_rot * G; }  // doubles per triangle buffer
    size_t smem_bytes() const {
        return 8 * tri() * nbuf + 16 * (size_t)p_rot * G * nbuf + 8 * 3 * ZSEG + 64;
    }
};

template <int NTB, bool ACC, bool ROWS>
__global__ void __launch_bounds__(NTHREADS, 1)
translate_mma_kernel(TranslateArgs<double> a, MmaTables mt, int64_t n_units, int p_rot, int nbuf) {
    constexpr int G = 8 * NTB, NH = NTB / TB;
    if (a.fail_flag && *a.fail_flag) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tri = p_rot * p_rot * G;

    double* bufs = reinterpret_cast<double*>(smem_raw);
    double2* betas = reinterpret_cast<double2*>(bufs + (size_t)nbuf * tri);
    double* zt = reinterpret_cast<double*>(betas + (size_t)nbuf * p_rot * G);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(zt + 3 * ZSEG);  // full[2], empty[2]
    int* counters = reinterpret_cast<int*>(mbar + 4);            // queues B, Z, C

    const int kind = a.kind, p_in = a.p_in, p_out = a.p_out;
    const bool src_local = kind == KIND_L2L, dst_local = kind != KIND_M2M;
    const int cols = min(p_in, p_out);

    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(&mbar[b], NE);
            mbar_init(&mbar[2 + b], NM);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        counters[0] = counters[1] = counters[2] = 0;
    }
    // z tables: k! | (-1)^d / d! at [ZC + d], 0 for d < 0 | 1 / e! at [ZC + e], 0 for e < 0
    for (int i = threadIdx.x; i < 3 * ZSEG; i += NTHREADS) {
        double v = 0.0;
        const int seg = i / ZSEG, j = i - seg * ZSEG;
        if (seg == 0) v = j < mt.nfac ? mt.fac[j] : 0.0;
        else if (j >= ZC && j - ZC < mt.ninv) v = seg == 1 ? mt.winv[j - ZC] : mt.inv[j - ZC];
        zt[i] = v;
    }
    __syncthreads();

    const int64_t first = blockIdx.x, stride = gridDim.x;
    const int n_mine = first < n_units ? (int)((n_units - first + stride - 1) / stride) : 0;

    if (warp < NE) {
        // ================= E warps: D(i - nbuf) + A(i) on buffer i % nbuf
        for (int i = 0; i < n_mine + nbuf; ++i) {
            const int b = nbuf == 2 ? (i & 1) : 0, k = nbuf == 2 ? (i >> 1) : i;
            const int64_t unit_a = i < n_mine ? first + (int64_t)i * stride : -1;
            const int64_t unit_d = i >= nbuf ? first + (int64_t)(i - nbuf) * stride : -1;
            if (i >= nbuf) mbar_wait(&mbar[2 + b], (k - 1) & 1);  // C of the previous tenant is done
            elementwise_trip<NTB, ACC, ROWS>(a, warp, lane, unit_a, unit_d, bufs + (size_t)b * tri,
                                             betas + (size_t)b * p_rot * G, p_rot);
            if (unit_a >= 0) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&mbar[b]);
            }
        }
    } else {
        // ================= M warps: B, Z, C of unit i on buffer i % nbuf
        const bool lead = threadIdx.x == NE * 32;
        for (int i = 0; i < n_mine; ++i) {
            const int b = nbuf == 2 ? (i & 1) : 0, k = nbuf == 2 ? (i >> 1) : i;
            double* buf = bufs + (size_t)b * tri;
            const double2* beta = betas + (size_t)b * p_rot * G;
            mbar_wait(&mbar[b], k & 1);
            // ---- B: forward swap passes, largest rows first
            {
                const MCtx c{buf, beta, mt.frags[src_local ? 1 : 0], src_local, false};
                const int ntask = 2 * NH * p_in;
                for (int task = fetch_task(&counters[0], lane); task < ntask;
                     task = fetch_task(&counters[0], lane)) {
                    const int n = p_in - 1 - task / (2 * NH), r = task % (2 * NH);
                    half_task_dispatch<NTB>(c, n, r & 1, r >> 1, n);
                }
            }
            bar_m();
            if (lead) counters[0] = counters[2] = 0;
            // ---- Z: z-axis step per column, longest columns first
            {
                const int ntask = NH * cols;
                for (int task = fetch_task(&counters[1], lane); task < ntask;
                     task = fetch_task(&counters[1], lane))
                    zstep_dispatch<NTB>(buf, zt, kind, p_in, p_out, task / NH, task % NH);
            }
            bar_m();
            if (lead) counters[1] = 0;
            // ---- C: backward swap passes. Columns >= cols of the z-step output are zero
            // (pipeline.cpp:229-246) and are never read.
            {
                const MCtx c{buf, beta, mt.frags[dst_local ? 1 : 0], dst_local, true};
                const int ntask = 2 * NH * p_out;
                for (int task = fetch_task(&counters[2], lane); task < ntask;
                     task = fetch_task(&counters[2], lane)) {
                    const int n = p_out - 1 - task / (2 * NH), r = task % (2 * NH);
                    half_task_dispatch<NTB>(c, n, r & 1, r >> 1, min(n, cols - 1));
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&mbar[2 + b]);
        }
    }
}

cudaError_t ensure_constants(const DeviceTables<double>& t) {
    static std::mutex mu;
    static std::vector<int> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    for (int d : done)
        if (d == dev) return cudaSuccess;
    // fragment offsets depend on the row only, not on the order of the handle
    static const std::vector<int> off = [] {
        const SwapTables st(PMAX);
        const FragSide fs = pack_frags(st, false);
        return std::vector<int>(fs.offset.begin(), fs.offset.end());
    }();
    (void)t;
    e = cudaMemcpyToSymbol(c_foff, off.data(), sizeof(int) * off.size());
    if (e != cudaSuccess) return e;
    done.push_back(dev);
    return cudaSuccess;
}

}  // namespace

bool mma_supports(const TranslateArgs<double>& a, const DeviceTables<double>& t) {
    const int p_rot = std::max(a.p_in, a.p_out);
    return t.frags[0] != nullptr && p_rot <= PMAX;
}

int mma_group_size(const TranslateArgs<double>& a) { return std::max(a.p_in, a.p_out) <= 20 ? 32 : 16; }

cudaError_t launch_translate_mma(const DeviceTables<double>& t, const TranslateArgs<double>& a,
                                 int sm_count, cudaStream_t stream, LaunchInfo* info) {
    cudaError_t e = ensure_constants(t);
    if (e != cudaSuccess) return e;
    const int p_rot = std::max(a.p_in, a.p_out);
    const int G = mma_group_size(a);
    int dev = 0, limit = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&limit, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    MmaLayout lay{p_rot, G, 2};
    if (const char* env = getenv("SFMM_MMA_NBUF")) lay.nbuf = atoi(env) == 1 ? 1 : 2;
    if ((int64_t)lay.smem_bytes() > limit) lay.nbuf = 1;
    if ((int64_t)lay.smem_bytes() > limit) return cudaErrorInvalidValue;
    const size_t smem = lay.smem_bytes();
    const int64_t n_units = (a.n + G - 1) / G;
    const bool acc = a.src_index != nullptr, rows = a.in_layout == LAYOUT_ROWS;

    MmaTables mt;
    mt.frags[0] = t.frags[0];
    mt.frags[1] = t.frags[1];
    mt.fac = t.fac;
    mt.inv = t.inv;
    mt.winv = t.winv;
    mt.nfac = 2 * t.order - 1;
    mt.ninv = t.order;

    using Kern = void (*)(TranslateArgs<double>, MmaTables, int64_t, int, int);
    Kern kern;
    if (G == 32)
        kern = acc ? (rows ? translate_mma_kernel<4, true, true> : translate_mma_kernel<4, true, false>)
                   : (rows ? translate_mma_kernel<4, false, true> : translate_mma_kernel<4, false, false>);
    else
        kern = acc ? (rows ? translate_mma_kernel<2, true, true> : translate_mma_kernel<2, true, false>)
                   : (rows ? translate_mma_kernel<2, false, true> : translate_mma_kernel<2, false, false>);
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 1;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NTHREADS, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorLaunchOutOfResources;
    const int grid = (int)std::min<int64_t>(n_units, (int64_t)sm_count * per_sm);
    kern<<<grid, NTHREADS, smem, stream>>>(a, mt, n_units, p_rot, lay.nbuf);
    e = cudaGetLastError();
    if (info) {
        info->grid = grid;
        info->block = NTHREADS;
        info->smem = smem;
        info->launches = 1;
        info->group = G;
        info->variant = G == 32 ? "mma/f64/G32" : "mma/f64/G16";
    }
    return e;
}

}  // namespace sfmm

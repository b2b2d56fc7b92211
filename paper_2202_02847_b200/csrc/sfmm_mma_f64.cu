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
constexpr int NTHREADS = 512;              // 16 warps, four per TMEM quarter
constexpr int ZTB = 2;                    // t-blocks (of 8 translations) per z-step pass
constexpr int ZC = 40;                    // centre of the Toeplitz tables
constexpr int ZSEG = 80;                  // one z-table segment
constexpr int Z_FAC = 0, Z_LOW = ZSEG, Z_UP = 2 * ZSEG;

// first fragment of block n*4 + {F/E, F/O, G/E, G/O} (same for both sides)
__constant__ int c_foff[PMAX * 4 + 1];

extern __shared__ __align__(16) unsigned char smem_raw[];

__device__ __forceinline__ int class_size(int n, int cls) { return cls ? (n + 1) >> 1 : (n >> 1) + 1; }
// 4-wide input blocks that cover every class of row n, 8-wide output blocks
__host__ __device__ __forceinline__ int row_nk(int n) { return (n / 2 + 1 + 3) >> 2; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// ---- shared memory through 32-bit addresses (LDS / STS with immediate offsets; generic
// pointers that travel through a call cost a 64-bit address and a descriptor per access)
__device__ __forceinline__ double lds(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
// 0 when !p (the load is not issued)
__device__ __forceinline__ double lds_if(uint32_t a, bool p) {
    double v;
    asm volatile(
        "{\n"
        ".reg .pred q;\n"
        "setp.ne.u32 q, %2, 0;\n"
        "mov.f64 %0, 0d0000000000000000;\n"
        "@q ld.shared.f64 %0, [%1];\n"
        "}\n"
        : "=d"(v)
        : "r"(a), "r"((uint32_t)p));
    return v;
}
__device__ __forceinline__ double2 lds2(uint32_t a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts(uint32_t a, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void sts2(uint32_t a, double x, double y) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(x), "d"(y) : "memory");
}

__device__ __forceinline__ int fetch_task(uint32_t counter, int lane) {
    int t = 0;
    if (lane == 0) asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(t) : "r"(counter) : "memory");
    return __shfl_sync(0xffffffffu, t, 0);
}

// D (8x8, lane holds columns 2q, 2q+1 of row t) += A (8x4, lane holds (t, q)) * B (4x8,
// lane holds (row q, column t)); k-ascending fma chain per output (PTX ISA, mma.m8n8k4.f64)
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

// ---- tensor memory (PTX ISA: tcgen05.alloc / .st / .ld) as the operator store.
// A warp reaches the 32 TMEM lanes of its quarter (warp % 4) only, one lane per thread:
// exactly the shape of a B fragment (one double per lane). Every quarter holds the
// fragments of the rows its three M warps work on (host-side partition, MmaPlan), loaded
// once per CTA; a fragment then costs a 12-cycle tcgen05.ld that touches neither the
// load/store unit, nor L1/L2, nor shared memory (B300_MICROARCH.md "TMEM").
// Layout of row n from its first slot: block j = {F/E, F/O, G/E, G/O} at j NK MB,
// fragment (kb, mb) at kb MB + mb, NK = row_nk(n), MB = (NK + 1) / 2; fragments the block
// does not have are stored as zeros, so the products need no bounds.
__device__ __forceinline__ void tmem_alloc_all(uint32_t smem_slot) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_slot)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_all(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr) : "memory");
}
__device__ __forceinline__ void tmem_fence_before_sync() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_fence_after_sync() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_store_frag(uint32_t taddr, double v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr),
                 "r"(__double2loint(v)), "r"(__double2hiint(v))
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_store() {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// MB adjacent fragments (MB = 1 or 2) with one load
template <int MB>
struct Frags {
    uint32_t w[2 * MB];
    __device__ __forceinline__ double get(int mb) const {
        return __hiloint2double((int)w[2 * mb + 1], (int)w[2 * mb]);
    }
};
__device__ __forceinline__ void tmem_load(uint32_t taddr, Frags<1>& f) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];"
                 : "=r"(f.w[0]), "=r"(f.w[1])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_load(uint32_t taddr, Frags<2>& f) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(f.w[0]), "=r"(f.w[1]), "=r"(f.w[2]), "=r"(f.w[3])
                 : "r"(taddr));
}
// The loaded registers pass through the wait so that no use is scheduled ahead of it.
__device__ __forceinline__ void tmem_wait_load(Frags<1>& a, Frags<1>& b) {
#ifdef SFMM_EXP_NOWAIT
    return;
#endif
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(a.w[0]), "+r"(a.w[1]), "+r"(b.w[0]), "+r"(b.w[1])::"memory");
}
__device__ __forceinline__ void tmem_wait_load(Frags<2>& a, Frags<2>& b) {
#ifdef SFMM_EXP_NOWAIT
    return;
#endif
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(a.w[0]), "+r"(a.w[1]), "+r"(a.w[2]), "+r"(a.w[3]), "+r"(b.w[0]), "+r"(b.w[1]),
                   "+r"(b.w[2]), "+r"(b.w[3])::"memory");
}

// four (cos, sin) pairs = 16 columns per lane: the alpha tables of the E warps
__device__ __forceinline__ void tmem_store16(uint32_t taddr, const double (&v)[8]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
        "%12, %13, %14, %15, %16};" ::"r"(taddr),
        "r"(__double2loint(v[0])), "r"(__double2hiint(v[0])), "r"(__double2loint(v[1])),
        "r"(__double2hiint(v[1])), "r"(__double2loint(v[2])), "r"(__double2hiint(v[2])),
        "r"(__double2loint(v[3])), "r"(__double2hiint(v[3])), "r"(__double2loint(v[4])),
        "r"(__double2hiint(v[4])), "r"(__double2loint(v[5])), "r"(__double2hiint(v[5])),
        "r"(__double2loint(v[6])), "r"(__double2hiint(v[6])), "r"(__double2loint(v[7])),
        "r"(__double2hiint(v[7]))
        : "memory");
}
struct Tab16 {
    uint32_t w[16];
    __device__ __forceinline__ double get(int j) const {
        return __hiloint2double((int)w[2 * j + 1], (int)w[2 * j]);
    }
};
__device__ __forceinline__ void tmem_load16(uint32_t taddr, Tab16& t) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
        "%13, %14, %15}, [%16];"
        : "=r"(t.w[0]), "=r"(t.w[1]), "=r"(t.w[2]), "=r"(t.w[3]), "=r"(t.w[4]), "=r"(t.w[5]),
          "=r"(t.w[6]), "=r"(t.w[7]), "=r"(t.w[8]), "=r"(t.w[9]), "=r"(t.w[10]), "=r"(t.w[11]),
          "=r"(t.w[12]), "=r"(t.w[13]), "=r"(t.w[14]), "=r"(t.w[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_load16(Tab16& t) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(t.w[0]), "+r"(t.w[1]), "+r"(t.w[2]), "+r"(t.w[3]), "+r"(t.w[4]), "+r"(t.w[5]),
                   "+r"(t.w[6]), "+r"(t.w[7]), "+r"(t.w[8]), "+r"(t.w[9]), "+r"(t.w[10]), "+r"(t.w[11]),
                   "+r"(t.w[12]), "+r"(t.w[13]), "+r"(t.w[14]), "+r"(t.w[15])::"memory");
}

struct MCtx {
    uint32_t buf;    // shared address of the triangle of the buffer
    uint32_t beta;   // shared address of the (cos, sin)(m beta) table, [m][G] double2,
                     // translation position ^ (((m >> 1) & 3) << 1)
    uint32_t tmem;   // TMEM address of the warp's quarter, column 0
    bool local_side; // transposed blocks; halve / double re_0 (pipeline.cpp:155-157, 247-249)
    bool bwd;        // backward pass: rotate by -beta
};

// One parity half of swap -> rotate(+-beta) -> swap on row n for t-blocks
// TB h .. TB h + TB-1, in place in the shared-memory triangle. NK = row_nk(n): number of
// 4-wide input blocks, MB = number of 8-wide output blocks; all loops are compile-time, the
// DMMAs sit in straight-line code. `slot` = first TMEM fragment slot of row n in the warp's
// quarter. mmax < n only for backward rows with p_out > p_in (inputs in columns
// >= min(p_in, p_out) are zero, pipeline.cpp:229-246).
template <int NTB, int NK, int TB>
__device__ __noinline__ void mma_half_task(const MCtx c, int n, int mask, int mmax, int slot) {
    constexpr int G = 8 * NTB, MB = (NK + 1) / 2, FB = NK * MB;
    constexpr uint32_t KSTEP = 16 * G * 8;  // bytes between members j and j + 4 of a class
    const int lane = threadIdx.x & 31, t = lane >> 2, q = lane & 3;
    // the task covers the (class, t-block pair) combinations r = cls + 2 h of `mask`
#pragma unroll 1
  for (int r = 0; r < 4; ++r) {
    if (!((mask >> r) & 1)) continue;
    const int cls = r & 1, h = r >> 1;
    const int nc = class_size(n, cls);  // members of the rotation class (== of class cF)
    const int cF = (n - cls) & 1, cG = cF ^ 1;
    const int nG = class_size(n, cG);
    const int g0 = cG ? 0 : 1;  // class index 0 of E is m = 0: no imaginary part
    const int kendF = mmax >= cF ? min(nc, ((mmax - cF) >> 1) + 1) : 0;
    const int kendG = mmax >= cG ? min(nG, ((mmax - cG) >> 1) + 1) : 0;
    const bool halve = c.local_side && cF == 0;
    const uint32_t tF1 = c.tmem + 2 * (slot + cls * FB);        // rows cls, cols cF
    const uint32_t tG1 = c.tmem + 2 * (slot + (2 + cls) * FB);  // rows cls, cols cG
    const uint32_t tF2 = c.tmem + 2 * (slot + cF * FB);         // rows cF, cols cls
    const uint32_t tG2 = c.tmem + 2 * (slot + (2 + cG) * FB);   // rows cG, cols cls

    // member j = 4 kb + q of class cF: re at idx n^2 + 2 cF + 4 j; of class cG: im at
    // n^2 + 2 cG + 4 j - 1; swizzle key ((m >> 1) + n) & 3 = (q + n) & 3 for both
    const int key = ((q + n) & 3) << 2;
    uint32_t are_[TB], aim_[TB];
#pragma unroll
    for (int tb = 0; tb < TB; ++tb) {
        const int pos = (8 * (TB * h + tb) + t) ^ key;
        are_[tb] = c.buf + ((n * n + 2 * cF + 4 * q) * G + pos) * 8;
        aim_[tb] = c.buf + ((n * n + 2 * cG + 4 * q - 1) * G + pos) * 8;
    }

    double cre[MB][2][TB], cim[MB][2][TB];
#pragma unroll
    for (int mb = 0; mb < MB; ++mb)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
#pragma unroll
            for (int tb = 0; tb < TB; ++tb) cre[mb][hh][tb] = cim[mb][hh][tb] = 0.0;

    // ---- product 1: u_re = A_F[cls, cF] re[cF], u_im = A_G[cls, cG] im[cG]
    {
        Frags<MB> ff, fg;
        tmem_load(tF1, ff);
        tmem_load(tG1, fg);
#pragma unroll
        for (int kb = 0; kb < NK; ++kb) {
            const int j = 4 * kb + q;
            const bool vF = j < kendF, vG = j >= g0 && j < kendG;
            double xr[TB], xi[TB];
#pragma unroll
            for (int tb = 0; tb < TB; ++tb) {
                xr[tb] = lds_if(are_[tb] + kb * KSTEP, vF);
                xi[tb] = lds_if(aim_[tb] + kb * KSTEP, vG);
            }
            if (kb == 0 && halve && q == 0) {
#pragma unroll
                for (int tb = 0; tb < TB; ++tb) xr[tb] *= 0.5;
            }
            tmem_wait_load(ff, fg);
            double f[MB], g[MB];
#pragma unroll
            for (int mb = 0; mb < MB; ++mb) f[mb] = ff.get(mb), g[mb] = fg.get(mb);
            if (kb + 1 < NK) {
                tmem_load(tF1 + 2 * (kb + 1) * MB, ff);
                tmem_load(tG1 + 2 * (kb + 1) * MB, fg);
            }
#pragma unroll
            for (int tb = 0; tb < TB; ++tb)
#pragma unroll
                for (int mb = 0; mb < MB; ++mb) {
                    dmma(cre[mb][0][tb], cre[mb][1][tb], xr[tb], f[mb]);
                    dmma(cim[mb][0][tb], cim[mb][1][tb], xi[tb], g[mb]);
                }
        }
    }
    // ---- rotate by +-beta (kernels.cpp:211-217). Register (mb, hh) of a lane is member
    // j = 4 kk + q (kk = 2 mb + hh) of class cls, m = cls + 2 j. Members beyond the class are
    // exactly zero and meet finite factors (the table has 8 NK rows at least).
    {
        Frags<MB> ff, fg;  // first operator blocks of product 2, in flight during the rotation
        tmem_load(tF2, ff);
        tmem_load(tG2, fg);
        const uint32_t b0 = c.beta + (((cls + 2 * q) * G) + ((8 * TB * h + t) ^ (q << 1))) * 16;
#pragma unroll
        for (int kk = 0; kk < NK; ++kk)
#pragma unroll
            for (int tb = 0; tb < TB; ++tb) {
                const double2 cs = lds2(b0 + kk * (8 * G * 16) + tb * (8 * 16));
                const double s = c.bwd ? -cs.y : cs.y;
                const double a = cre[kk >> 1][kk & 1][tb], b = cim[kk >> 1][kk & 1][tb];
                cre[kk >> 1][kk & 1][tb] = fma_(a, cs.x, -(b * s));
                cim[kk >> 1][kk & 1][tb] = fma_(a, s, b * cs.x);
            }
        // ---- product 2: re[cF] = A_F[cF, cls] u_re, im[cG] = A_G[cG, cls] u_im; the
        // accumulator registers (mb, hh) of product 1 are the A operands of input block
        // kb2 = 2 mb + hh
        double ore[MB][2][TB], oim[MB][2][TB];
#pragma unroll
        for (int mb = 0; mb < MB; ++mb)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                for (int tb = 0; tb < TB; ++tb) ore[mb][hh][tb] = oim[mb][hh][tb] = 0.0;
#pragma unroll
        for (int kb2 = 0; kb2 < NK; ++kb2) {
            tmem_wait_load(ff, fg);
            double f[MB], g[MB];
#pragma unroll
            for (int mb = 0; mb < MB; ++mb) f[mb] = ff.get(mb), g[mb] = fg.get(mb);
            if (kb2 + 1 < NK) {
                tmem_load(tF2 + 2 * (kb2 + 1) * MB, ff);
                tmem_load(tG2 + 2 * (kb2 + 1) * MB, fg);
            }
#pragma unroll
            for (int tb = 0; tb < TB; ++tb)
#pragma unroll
                for (int mb = 0; mb < MB; ++mb) {
                    dmma(ore[mb][0][tb], ore[mb][1][tb], cre[kb2 >> 1][kb2 & 1][tb], f[mb]);
                    dmma(oim[mb][0][tb], oim[mb][1][tb], cim[kb2 >> 1][kb2 & 1][tb], g[mb]);
                }
        }
#pragma unroll
        for (int kk = 0; kk < NK; ++kk) {
            const int j2 = 4 * kk + q;
            if (j2 < nc) {
#pragma unroll
                for (int tb = 0; tb < TB; ++tb) {
                    double v = ore[kk >> 1][kk & 1][tb];
                    if (kk == 0 && halve && q == 0) v *= 2.0;
                    sts(are_[tb] + kk * KSTEP, v);
                }
            }
            if (j2 >= g0 && j2 < nG) {
#pragma unroll
                for (int tb = 0; tb < TB; ++tb) sts(aim_[tb] + kk * KSTEP, oim[kk >> 1][kk & 1][tb]);
            }
        }
    }
  }
}

template <int NTB>
__device__ __forceinline__ void half_task_dispatch(const MCtx c, int n, int mask, int mmax, int slot) {
    switch (row_nk(n)) {
        // small rows: all t-blocks of the unit in one go (the accumulators fit), so that the
        // addressing and the operator loads are paid once per 8 NTB translations
        case 1: mma_half_task<NTB, 1, NTB>(c, n, mask, mmax, slot); break;
        case 2: mma_half_task<NTB, 2, NTB>(c, n, mask, mmax, slot); break;
        case 3: mma_half_task<NTB, 3, 2>(c, n, mask, mmax, slot); break;
        default: mma_half_task<NTB, 4, 2>(c, n, mask, mmax, slot); break;
    }
}

// z-axis step on column m (re and im) for t-blocks TB h .. TB h + TB-1, in place
// (reference kernels.cpp:118-196): out_i = sum_k W[i][k] in_k with
//   M2L  W = (2m + i + k)!              (Hankel; sign (-1)^i of the backward gather,
//                                        pipeline.cpp:235-239, applied at the store)
//   M2M  W = (-1)^(i-k) / (i-k)!, k <= i (lower Toeplitz)
//   L2L  W = 1 / (k-i)!, k >= i          (upper Toeplitz)
// The B fragments are generated from the small tables in shared memory:
// value(kk, ii) = zt[zbase + s1 kk + s2 ii] (zeros where the triangular kinds have none).
template <int NTB, int NB, bool IM, int TB>
__device__ __noinline__ void mma_zstep(uint32_t buf, uint32_t zt, int kind, int p_in, int p_out, int m,
                                       int hmask) {
    constexpr int G = 8 * NTB;
    const int lane = threadIdx.x & 31, t = lane >> 2, q = lane & 3;
    const int K = p_in - m, N = p_out - m;
    const int KB = (K + 3) >> 2;
    const int key = (((m >> 1) + m + q) & 3) << 2;
#pragma unroll 1
  for (int h = 0; h < NTB / TB; ++h) {
    if (!((hmask >> h) & 1)) continue;
    // element (row m + k, column m): idx (m + k)^2 + 2 m (re), - 1 (im); k = 4 kb + q
    uint32_t col[TB];
#pragma unroll
    for (int tb = 0; tb < TB; ++tb)
        col[tb] = buf + ((2 * m) * G + ((8 * (TB * h + tb) + t) ^ key)) * 8;
    // operator entry of lane (row kk = 4 kb + q, column ii = sigma(nb, t))
    const int sig = (t >> 1) + 4 * (t & 1);
    int zoff, s1, s2;
    if (kind == KIND_M2L) zoff = Z_FAC + 2 * m, s1 = 1, s2 = 1;
    else if (kind == KIND_M2M) zoff = Z_LOW + ZC, s1 = -1, s2 = 1;
    else zoff = Z_UP + ZC, s1 = 1, s2 = -1;
    uint32_t zl = zt + (zoff + s1 * q + s2 * sig) * 8;
    const int zk = s1 * 32, zn = s2 * 64;  // bytes per input block / output block

    double acc[2][TB][NB][2];
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int tb = 0; tb < TB; ++tb)
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) acc[p][tb][nb][0] = acc[p][tb][nb][1] = 0.0;

    // operands of step kb, loaded one step ahead
    double xn[2][TB], bn[NB];
    int k = q;
    auto load = [&]() {
        const int r = m + k;
        const uint32_t off = (uint32_t)(r * r) * (G * 8);
        const bool valid = k < K;
#pragma unroll
        for (int tb = 0; tb < TB; ++tb) {
            xn[0][tb] = lds_if(col[tb] + off, valid);
            if (IM) xn[1][tb] = lds_if(col[tb] + off - G * 8, valid);
        }
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) bn[nb] = lds(zl + nb * zn);
        k += 4;
        zl += zk;
    };
    load();
#pragma unroll 1
    for (int kb = 0; kb < KB; ++kb) {
        double x[2][TB], bf[NB];
#pragma unroll
        for (int tb = 0; tb < TB; ++tb) x[0][tb] = xn[0][tb], x[1][tb] = IM ? xn[1][tb] : 0.0;
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) bf[nb] = bn[nb];
        load();  // one step beyond the column: masked inputs, table reads stay inside the tables
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
#pragma unroll
            for (int tb = 0; tb < TB; ++tb) {
                dmma(acc[0][tb][nb][0], acc[0][tb][nb][1], x[0][tb], bf[nb]);
                if constexpr (IM) dmma(acc[1][tb][nb][0], acc[1][tb][nb][1], x[1][tb], bf[nb]);
            }
    }
    const bool neg = kind == KIND_M2L && (q & 1);
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const int i = 8 * nb + 4 * hh + q, r = m + i;
            if (i < N) {
                const uint32_t off = (uint32_t)(r * r) * (G * 8);
#pragma unroll
                for (int tb = 0; tb < TB; ++tb) {
                    const double vr = acc[0][tb][nb][hh];
                    sts(col[tb] + off, neg ? -vr : vr);
                    if constexpr (IM) {
                        const double vi = acc[1][tb][nb][hh];
                        sts(col[tb] + off - G * 8, neg ? -vi : vi);
                    }
                }
            }
        }
  }
}

template <int NTB>
__device__ __forceinline__ void zstep_dispatch(uint32_t buf, uint32_t zt, int kind, int p_in, int p_out,
                                               int m, int h /* mask of t-block groups */) {
    const int nb = (p_out - m + 7) >> 3;
    // short columns (nb <= 2): all t-blocks of the unit in one pass
    if (m == 0) {
        switch (nb) {
            case 1: mma_zstep<NTB, 1, false, NTB>(buf, zt, kind, p_in, p_out, m, h); break;
            case 2: mma_zstep<NTB, 2, false, NTB>(buf, zt, kind, p_in, p_out, m, h); break;
            case 3: mma_zstep<NTB, 3, false, ZTB>(buf, zt, kind, p_in, p_out, m, h); break;
            default: mma_zstep<NTB, 4, false, ZTB>(buf, zt, kind, p_in, p_out, m, h); break;
        }
        return;
    }
    switch (nb) {
        case 1: mma_zstep<NTB, 1, true, NTB>(buf, zt, kind, p_in, p_out, m, h); break;
        case 2: mma_zstep<NTB, 2, true, NTB>(buf, zt, kind, p_in, p_out, m, h); break;
        case 3: mma_zstep<NTB, 3, true, ZTB>(buf, zt, kind, p_in, p_out, m, h); break;
        default: mma_zstep<NTB, 4, true, ZTB>(buf, zt, kind, p_in, p_out, m, h); break;
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
            const int64_t j = a.angle_index ? (int64_t)a.angle_index[b] : b;
            g.rn = a.angles[j];
            g.ca = a.angles[a.n + j];
            g.sa = a.angles[2 * a.n + j];
            g.cb = a.angles[3 * a.n + j];
            g.sb = a.angles[4 * a.n + j];
            g.inv = a.angles[5 * a.n + j];
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

// Host-side partition of the swap-pass rows over the four TMEM quarters (warp % 4), per
// pass (0 forward: rows n < p_in, 1 backward: rows n < p_out): rows[pass][quarter] lists the
// rows of a quarter, heaviest first; slot[pass][n] is the first fragment slot (2 TMEM columns
// each) of row n inside its quarter.
// task[pass][quarter][i] = n | mask << 5: row n, mask over the (class, t-block pair)
// combinations r = cls + 2 h the task runs (small rows are batched: a task should carry
// enough DMMAs to pay for its dispatch); ztask[i] = m | hmask << 5 likewise for the z-step.
struct MmaPlan {
    uint16_t slot[2][32];
    uint8_t rows[2][4][16];
    uint8_t nrows[2][4];
    uint16_t task[2][4][28];
    uint8_t ntask[2][4];
    uint8_t ztask[64];
    int nz;
    int max_slots;  // fragment slots the fullest quarter uses
};

constexpr int CH = 4;  // elements (re, im pairs) per chunk of the elementwise phases

// Elementwise row tasks (lane = translation), drained from a shared queue by whichever warps
// have no tensor task: MODE_D = phase D of `unit` (rotate by -alpha, scale, store or reduce
// over the lanes of the unit; pipeline.cpp:251-265), MODE_A = phase A (gather, rotate by
// +alpha, scale; pipeline.cpp:148-154) plus, for the warp that draws ticket 0, the beta
// table of the unit (pipeline.cpp:52-91). One call works until the queue is empty, so the
// per-lane geometry is loaded once. Powers of |r| by repeated multiplication from 1 exactly
// as the reference builds its tables (pipeline.cpp:81-89); cos/sin(m alpha) follow the row
// by the angle recurrence of pipeline.cpp:70-79 from (1, 0).
enum : int { MODE_D = 0, MODE_A = 1 };

// Launch constants of the row tasks, written once per CTA into shared memory: arguments that
// travel by reference through an out-of-line call cost a local-memory copy of the struct.
struct RowConst {
    const double* in;
    int64_t in_stride;
    double* out;
    int64_t out_stride;
    const int32_t* src_index;
    int64_t n;
    const double* shifts;
    const double* angles;
    const int32_t* angle_index;
    int kind, p_in, p_out, pad;
};

template <int NTB, bool ACC, bool ROWS, int MODE>
__device__ __noinline__ void elementwise_rows(uint32_t rc_addr, int64_t unit, uint32_t buf, uint32_t beta,
                                              int beta_rows, uint32_t queue) {
    constexpr int G = 8 * NTB;
    TranslateArgs<double> a;  // the fields the row tasks use
    {
        const RowConst& rc = *reinterpret_cast<const RowConst*>(smem_raw + (rc_addr - smem_u32(smem_raw)));
        a.in = rc.in, a.in_stride = rc.in_stride, a.out = rc.out, a.out_stride = rc.out_stride;
        a.src_index = rc.src_index, a.n = rc.n, a.shifts = rc.shifts, a.angles = rc.angles;
        a.angle_index = rc.angle_index;
        a.kind = rc.kind, a.p_in = rc.p_in, a.p_out = rc.p_out;
    }
    constexpr uint32_t ROWB = G * 8;  // bytes of one triangle entry (all translations)
    const int lane = threadIdx.x & 31;
    const int kind = a.kind, p_in = a.p_in, p_out = a.p_out;
    const bool src_local = kind == KIND_L2L, dst_local = kind != KIND_M2M;
    const bool lane_ok = G == 32 || lane < G;
    const int lp = lane & (G - 1);
    const int p_rows = MODE == MODE_A ? p_in : p_out;
    int task = fetch_task(queue, lane);  // MODE_A: ticket 0 = beta table, row tickets follow
    const int n_tickets = p_rows + (MODE == MODE_A ? 1 : 0);
    if (task >= n_tickets) return;

    const int64_t b = unit * G + lp;
    bool act = lane_ok && b < a.n;
    int64_t src = b;
    if (MODE == MODE_A && ACC && act) {
        const int32_t s = a.src_index[b];
        act = s >= 0;
        src = s >= 0 ? s : 0;
    }
    const LaneGeo g = load_geo(a, b, lane_ok && b < a.n && (!ACC || a.angles || act));
    const double c1 = fma_(1.0, g.ca, -(0.0 * g.sa)), s1 = fma_(0.0, g.ca, 1.0 * g.sa);
    const double base = MODE == MODE_A ? (src_local ? g.rn : g.inv) : (dst_local ? g.inv : g.rn);
    const double q0 = MODE == MODE_A ? (src_local ? 1.0 : base) : (dst_local ? 1.0 : base);
    const double* pa = ROWS ? a.in + src * a.in_stride : a.in + src;

    for (; task < n_tickets; task = fetch_task(queue, lane)) {
        if (MODE == MODE_A && task == 0) {
            // (cos, sin)(m beta), m < beta_rows, translation position ^ (((m >> 1) & 3) << 1)
            if (lane_ok) {
                double c = 1, s = 0;
                for (int m = 0; m < beta_rows; ++m) {
                    sts2(beta + (m * G + (lp ^ (((m >> 1) & 3) << 1))) * 16, c, s);
                    const double nc = fma_(c, g.cb, -(s * g.sb));
                    const double ns = fma_(s, g.cb, c * g.sb);
                    c = nc;
                    s = ns;
                }
            }
            continue;
        }
        const int n = p_rows - 1 - (task - (MODE == MODE_A ? 1 : 0));  // longest rows first
        double q = q0;  // scale of the row: q0 base^n
        for (int j = 0; j < n; ++j) q *= base;
        // entry (n, m): re at row + 2 m ROWB, im one entry below; translation position
        // lp ^ (key << 2), key = ((m >> 1) + n) & 3: two consecutive m share a key
        const uint32_t row = buf + (uint32_t)(n * n) * ROWB;
        uint32_t px[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) px[j] = (lp ^ (((j + n) & 3) << 2)) * 8;

        if constexpr (MODE == MODE_D) {
            double c = 1, ms = -0.0;  // cos(m alpha), -sin(m alpha)
            const double ms1 = -s1;
            // ACC: lane 4 k stores value k of a chunk = entry 2 m0 + k of the row
            double* po = ACC ? a.out + ((int64_t)aos_re(n, 0) + (lane >> 2)) * a.out_stride + unit
                             : a.out + (int64_t)aos_re(n, 0) * a.out_stride + b;
            for (int m0 = 0; m0 <= n; m0 += CH) {
                // m0 is a multiple of 4: (m >> 1) & 3 is 0, 1 (even chunks) or 2, 3 (odd)
                const uint32_t pxc[2] = {(m0 & 4) ? px[2] : px[0], (m0 & 4) ? px[3] : px[1]};
                double v[2 * CH];
#pragma unroll
                for (int u = 0; u < CH; ++u) {
                    const uint32_t ad = row + (2 * (m0 + u)) * ROWB + pxc[u >> 1];
                    const bool in = m0 + u <= n;
                    const double re = lds_if(ad, in);
                    const double im = lds_if(ad - ROWB, in && (m0 + u) > 0);
                    // rotation by -alpha: (re, im) * (c, ms), then the scale
                    const double nr = q * fma_(re, c, -(im * ms));
                    const double ni = q * fma_(re, ms, im * c);
                    v[2 * u] = lane_ok ? nr : 0.0;
                    v[2 * u + 1] = lane_ok ? ni : 0.0;
                    // (c, s) -> next m; ms = -s follows with negated products (exact)
                    const double nc = fma_(c, c1, -(ms * ms1));
                    const double nms = fma_(ms, c1, c * ms1);
                    c = nc;
                    ms = nms;
                }
                if constexpr (ACC) {
                    lane_transpose_sum<2 * CH>(v, lane);
                    const int k = 2 * m0 + (lane >> 2);  // entry of the row: 2 m + part
                    if (!(lane & 3) && k <= 2 * n + 1 && k != 1) __stcg(po, v[0]);
                } else if (act) {
#pragma unroll
                    for (int u = 0; u < CH; ++u)
                        if (m0 + u <= n) {
                            __stcg(po + (2 * u) * a.out_stride, v[2 * u]);
                            __stcg(po + (2 * u + 1) * a.out_stride, (m0 + u) ? v[2 * u + 1] : 0.0);
                        }
                }
                po += 2 * CH * a.out_stride;
            }
        } else {
            double xa0[2 * CH], xa1[2 * CH];
            const double* prow = ROWS ? pa + rows_off(n) : pa + (int64_t)aos_re(n, 0) * a.in_stride;
            auto issue = [&](int m0, double (&x)[2 * CH]) {
                if constexpr (ROWS) {
#pragma unroll
                    for (int j = 0; j < CH / 2; ++j) {
                        double w[4] = {0.0, 0.0, 0.0, 0.0};
                        if (act && m0 + 2 * j <= n) load4_cg(prow + 2 * m0 + 4 * j, w);
                        x[4 * j] = w[0], x[4 * j + 1] = w[1], x[4 * j + 2] = w[2], x[4 * j + 3] = w[3];
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < CH; ++u) {
                        x[2 * u] = x[2 * u + 1] = 0.0;
                        if (act && m0 + u <= n) {
                            const int64_t off = (int64_t)(2 * (m0 + u)) * a.in_stride;
                            x[2 * u] = __ldcg(prow + off);
                            x[2 * u + 1] = __ldcg(prow + off + a.in_stride);
                        }
                    }
                }
            };
            issue(0, xa0);
            if (CH <= n) issue(CH, xa1);
            const double aq = act ? q : 0.0;
            double c = 1, s = 0;
            auto chunk = [&](int m0, const double (&x)[2 * CH]) {
                const uint32_t pxc[2] = {(m0 & 4) ? px[2] : px[0], (m0 & 4) ? px[3] : px[1]};
#pragma unroll
                for (int u = 0; u < CH; ++u) {
                    const int m = m0 + u;
                    if (m > n) break;
                    const double xr = x[2 * u];
                    const double xi = m ? x[2 * u + 1] : 0.0;
                    const double nr = aq * fma_(xr, c, -(xi * s));
                    const double ni = aq * fma_(xr, s, xi * c);
                    if (lane_ok) {
                        const uint32_t ad = row + (2 * m) * ROWB + pxc[u >> 1];
                        sts(ad, nr);
                        if (m) sts(ad - ROWB, ni);
                    }
                    const double nc = fma_(c, c1, -(s * s1));
                    const double ns = fma_(s, c1, c * s1);
                    c = nc;
                    s = ns;
                }
            };
            for (int m0 = 0; m0 <= n; m0 += 2 * CH) {
                chunk(m0, xa0);
                if (m0 + 2 * CH <= n) issue(m0 + 2 * CH, xa0);
                if (m0 + CH <= n) {
                    chunk(m0 + CH, xa1);
                    if (m0 + 3 * CH <= n) issue(m0 + 3 * CH, xa1);
                }
            }
        }
    }
}

struct MmaLayout {
    int p_rot, G, nbuf;
    int beta_rows() const { return std::max(p_rot, 8 * row_nk(p_rot - 1)); }
    size_t tri() const { return (size_t)p_rot * p_rot * G; }  // doubles per triangle buffer
    size_t smem_bytes() const {
        return 8 * tri() * nbuf + 16 * (size_t)beta_rows() * G * nbuf + 8 * 3 * ZSEG + 160;
    }
};

// Schedule of one CTA (16 warps, all alike; units u_i = blockIdx.x + i gridDim.x, buffer
// i % nbuf). Three CTA barriers per unit; every phase has a queue of tensor tasks and, where
// marked, a queue of elementwise row tasks on the OTHER buffer, so the latency-bound
// elementwise work runs inside the tensor phases on whichever warps are free:
//     P1: B(i)  forward swap passes                     (tensor tasks per TMEM quarter)
//     P2: Z(i)  z-axis step          + D(i-1) rows      (results of the previous unit out)
//     P3: C(i)  backward swap passes + A(i+1) rows      (next unit in, its beta table)
// With one buffer (nbuf = 1, p = 30) the row queues get phases of their own.
template <int NTB, bool ACC, bool ROWS>
__global__ void __launch_bounds__(NTHREADS, 1)
translate_mma_kernel(TranslateArgs<double> a, MmaTables mt, MmaPlan plan, int64_t n_units, int p_rot,
                     int beta_rows, int nbuf, int ablate) {
    constexpr int G = 8 * NTB;
    if (a.fail_flag && *a.fail_flag) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t tri_b = (uint32_t)(p_rot * p_rot * G) * 8, beta_b = (uint32_t)(beta_rows * G) * 16;

    const uint32_t sm = smem_u32(smem_raw);
    const uint32_t bufs = sm, betas = bufs + nbuf * tri_b, zt = betas + nbuf * beta_b;
    // queues: B per quarter [0..3], C per quarter [4..7], Z [8], D rows [9], A rows [10]
    const uint32_t counters = zt + 3 * ZSEG * 8;
    const uint32_t tmem_slot = counters + 48;
    const uint32_t rc_addr = counters + 64;  // RowConst (16-byte aligned: smem_bytes)
    static_assert(sizeof(RowConst) <= 96, "RowConst area");
    if (threadIdx.x == 0) {
        RowConst& rc = *reinterpret_cast<RowConst*>(smem_raw + (rc_addr - sm));
        rc.in = a.in, rc.in_stride = a.in_stride, rc.out = a.out, rc.out_stride = a.out_stride;
        rc.src_index = a.src_index, rc.n = a.n, rc.shifts = a.shifts, rc.angles = a.angles;
        rc.angle_index = a.angle_index;
        rc.kind = a.kind, rc.p_in = a.p_in, rc.p_out = a.p_out, rc.pad = 0;
    }

    const int kind = a.kind, p_in = a.p_in, p_out = a.p_out;
    const bool src_local = kind == KIND_L2L, dst_local = kind != KIND_M2M;
    const int cols = min(p_in, p_out);

    if (threadIdx.x < 11)
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(counters + 4 * threadIdx.x), "r"(0) : "memory");
    if (warp == 0) tmem_alloc_all(tmem_slot);
    // z tables: k! | (-1)^d / d! at [ZC + d], 0 for d < 0 | 1 / e! at [ZC + e], 0 for e < 0
    for (int i = threadIdx.x; i < 3 * ZSEG; i += NTHREADS) {
        double v = 0.0;
        const int seg = i / ZSEG, j = i - seg * ZSEG;
        if (seg == 0) v = j < mt.nfac ? mt.fac[j] : 0.0;
        else if (j >= ZC && j - ZC < mt.ninv) v = seg == 1 ? mt.winv[j - ZC] : mt.inv[j - ZC];
        sts(zt + 8 * i, v);
    }
    tmem_fence_before_sync();
    __syncthreads();
    tmem_fence_after_sync();
    const int quarter = warp & 3, sub = warp >> 2;
    uint32_t tmem_base;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem_base) : "r"(tmem_slot));
    const uint32_t tmem_mine = tmem_base + ((uint32_t)(32 * quarter) << 16);

    // operator fragments of the quarter's rows into tensor memory (once per CTA)
    for (int pass = 0; pass < 2; ++pass) {
        const double* src = mt.frags[(pass ? dst_local : src_local) ? 1 : 0];
        for (int r = 0; r < plan.nrows[pass][quarter]; ++r) {
            const int n = plan.rows[pass][quarter][r];
            const int nk = row_nk(n), mbs = (nk + 1) >> 1, fb = nk * mbs;
            for (int i = sub; i < 4 * fb; i += NTHREADS / 128) {
                const int j = i / fb, rem = i - j * fb, kb = rem / mbs, mb = rem - kb * mbs;
                // block j = which * 2 + rc: rows of class rc, columns of class (n + which - rc) & 1
                const int rc = j & 1, cc = (n + (j >> 1) - rc) & 1;
                const int kbs = (class_size(n, cc) + 3) >> 2, mbb = (class_size(n, rc) + 7) >> 3;
                double v = 0.0;
                if (kb < kbs && mb < mbb)
                    v = __ldg(src + (size_t)(c_foff[n * 4 + j] + kb * mbb + mb) * 32 + lane);
                tmem_store_frag(tmem_mine + 2 * (plan.slot[pass][n] + i), v);
            }
        }
    }
    tmem_wait_store();

    const int64_t first = blockIdx.x, stride = gridDim.x;
    const int n_mine = first < n_units ? (int)((n_units - first + stride - 1) / stride) : 0;
    auto unit_of = [&](int i) { return first + (int64_t)i * stride; };
    auto buf_of = [&](int i) { return bufs + (nbuf == 2 ? (i & 1) : 0) * tri_b; };
    auto beta_of = [&](int i) { return betas + (nbuf == 2 ? (i & 1) : 0) * beta_b; };
    // end of a phase: every queue of the phase is empty and every task has finished
    auto phase_end = [&](int reset_lo, int reset_hi) {
        __syncthreads();
        if ((int)threadIdx.x >= reset_lo && (int)threadIdx.x < reset_hi)
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(counters + 4 * threadIdx.x), "r"(0) : "memory");
    };
    // per-phase cycle counters of CTA 0 (tuning aid, tools/perf_probe.py PHASES=1):
    // 0 prologue / row-only phases, 1 P1, 2 P2, 3 P3
#ifdef SFMM_PHASE_CLOCKS
    const bool clk_on = a.phase_clocks && blockIdx.x == 0 && threadIdx.x == 0;
    long long t_prev = clock64();
#define SFMM_PHASE_MARK(idx)                         \
    if (clk_on) {                                    \
        const long long now = clock64();             \
        a.phase_clocks[idx] += now - t_prev;         \
        t_prev = now;                                \
    }
#else
#define SFMM_PHASE_MARK(idx)
#endif
    auto rows_d = [&](int i) {
        if (!(ablate & 1))
            elementwise_rows<NTB, ACC, ROWS, MODE_D>(rc_addr, unit_of(i), buf_of(i), beta_of(i), beta_rows,
                                                     counters + 36);
    };
    auto rows_a = [&](int i) {
        if (!(ablate & 1))
            elementwise_rows<NTB, ACC, ROWS, MODE_A>(rc_addr, unit_of(i), buf_of(i), beta_of(i), beta_rows,
                                                     counters + 40);
    };

    tmem_fence_before_sync();
    __syncthreads();  // operator fragments in place
    tmem_fence_after_sync();
    if (n_mine > 0) rows_a(0);
    phase_end(10, 11);
    SFMM_PHASE_MARK(0)
    // half of the warps start a mixed phase with the rows (their loads are long, the sooner
    // they are in flight the better), the other half with the tensor tasks
    const bool rows_first = sub & 1;
    for (int i = 0; i < n_mine; ++i) {
        const uint32_t buf = buf_of(i), beta = beta_of(i);
        // ---- P1: B(i), forward swap passes of the quarter's rows, heaviest first
        {
            const MCtx c{buf, beta, tmem_mine, src_local, false};
            const int ntask = (ablate & 2) ? 0 : plan.ntask[0][quarter];
            for (int task = fetch_task(counters + 4 * quarter, lane); task < ntask;
                 task = fetch_task(counters + 4 * quarter, lane)) {
                const int tk = plan.task[0][quarter][task], n = tk & 31;
                half_task_dispatch<NTB>(c, n, tk >> 5, n, plan.slot[0][n]);
            }
        }
        phase_end(0, 4);
        SFMM_PHASE_MARK(1)
        // ---- P2: Z(i), z-axis step per column, longest columns first; D(i-1) rows
        const bool d_here = nbuf == 2 && i > 0;
        if (d_here && rows_first) rows_d(i - 1);
        {
            const int ntask = (ablate & 4) ? 0 : plan.nz;
            for (int task = fetch_task(counters + 32, lane); task < ntask;
                 task = fetch_task(counters + 32, lane)) {
                const int tk = plan.ztask[task];
                zstep_dispatch<NTB>(buf, zt, kind, p_in, p_out, tk & 31, tk >> 5);
            }
        }
        if (d_here && !rows_first) rows_d(i - 1);
        phase_end(8, 10);
        SFMM_PHASE_MARK(2)
        // ---- P3: C(i), backward swap passes (columns >= cols of the z-step output are zero,
        // pipeline.cpp:229-246, and are never read); A(i+1) rows
        const bool a_here = nbuf == 2 && i + 1 < n_mine;
        if (a_here && rows_first) rows_a(i + 1);
        {
            const MCtx c{buf, beta, tmem_mine, dst_local, true};
            const int ntask = (ablate & 8) ? 0 : plan.ntask[1][quarter];
            for (int task = fetch_task(counters + 16 + 4 * quarter, lane); task < ntask;
                 task = fetch_task(counters + 16 + 4 * quarter, lane)) {
                const int tk = plan.task[1][quarter][task], n = tk & 31;
                half_task_dispatch<NTB>(c, n, tk >> 5, min(n, cols - 1), plan.slot[1][n]);
            }
        }
        if (a_here && !rows_first) rows_a(i + 1);
        phase_end(4, 11);
        SFMM_PHASE_MARK(3)
        if (nbuf == 1) {  // one buffer: D(i), then A(i+1), in phases of their own
            rows_d(i);
            phase_end(9, 10);
            if (i + 1 < n_mine) rows_a(i + 1);
            phase_end(10, 11);
            SFMM_PHASE_MARK(0)
        }
    }
    if (nbuf == 2 && n_mine > 0) rows_d(n_mine - 1);
    SFMM_PHASE_MARK(0)
#undef SFMM_PHASE_MARK
    tmem_fence_before_sync();
    __syncthreads();
    tmem_fence_after_sync();
    if (warp == 0) tmem_dealloc_all(tmem_base);
}

const std::vector<int>& frag_offsets() {
    // fragment offsets depend on the row only, not on the order of the handle
    static const std::vector<int> off = [] {
        const SwapTables st(PMAX);
        const FragSide fs = pack_frags(st, false);
        return std::vector<int>(fs.offset.begin(), fs.offset.end());
    }();
    return off;
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
    const std::vector<int>& off = frag_offsets();
    e = cudaMemcpyToSymbol(c_foff, off.data(), sizeof(int) * off.size());
    if (e != cudaSuccess) return e;
    done.push_back(dev);
    return cudaSuccess;
}

// Rows of a pass over the four quarters: heaviest row first into the lightest quarter
// (weight = DMMAs of the row's half tasks); fragment slots in the order of assignment;
// task lists heaviest first.
bool make_plan(int p_in, int p_out, int G, MmaPlan& plan) {
    plan = MmaPlan{};
    const int NH = G / 16;  // pairs of t-blocks per unit
    int used[4] = {0, 0, 0, 0};
    for (int pass = 0; pass < 2; ++pass) {
        const int p = pass ? p_out : p_in;
        long load[4] = {0, 0, 0, 0};
        for (int n = p - 1; n >= 0; --n) {
            const int nk = row_nk(n), mb = (nk + 1) / 2;
            int q = 0;
            for (int j = 1; j < 4; ++j)
                if (load[j] < load[q]) q = j;
            load[q] += (long)nk * mb * (n ? 2 : 1);
            if (plan.nrows[pass][q] >= 16) return false;
            plan.rows[pass][q][plan.nrows[pass][q]++] = (uint8_t)n;
            plan.slot[pass][n] = (uint16_t)used[q];
            used[q] += 4 * nk * mb;  // padded blocks (kernel comment "tensor memory")
            // tasks of the row, combinations r = cls + 2 h. Rows with nk <= 2 work on all
            // t-blocks at once (h = 0 only); the smallest rows run both classes in one task
            const int cl = n ? 3 : 1;  // row 0 has no odd class
            const int combos = nk <= 2 ? cl : (cl | (NH == 2 ? (cl << 2) : 0));
            const int per = nk >= 2 ? 1 : 2;  // combinations per task
            for (int r0 = 0; r0 < 4; r0 += per) {
                const int mask = combos & (((1 << per) - 1) << r0);
                if (!mask) continue;
                if (plan.ntask[pass][q] >= 28) return false;
                plan.task[pass][q][plan.ntask[pass][q]++] = (uint16_t)(n | (mask << 5));
            }
        }
    }
    plan.max_slots = 0;
    for (int q = 0; q < 4; ++q) {
        if (used[q] > 256) return false;  // 512 TMEM columns per quarter
        plan.max_slots = std::max(plan.max_slots, used[q]);
    }
    // z-step: column m carries ceil((p_in - m) / 4) ceil((p_out - m) / 8) DMMA groups per
    // t-block pair; small columns run both pairs in one task
    const int cols = std::min(p_in, p_out);
    for (int m = 0; m < cols; ++m) {
        // columns with at most two output blocks work on all t-blocks at once (h = 0 only)
        if (NH == 1 || (p_out - m + 7) / 8 <= 2) {
            plan.ztask[plan.nz++] = (uint8_t)(m | (1 << 5));
        } else {
            plan.ztask[plan.nz++] = (uint8_t)(m | (1 << 5));
            plan.ztask[plan.nz++] = (uint8_t)(m | (2 << 5));
        }
    }
    return true;
}

}  // namespace

bool mma_supports(const TranslateArgs<double>& a, const DeviceTables<double>& t) {
    const int p_rot = std::max(a.p_in, a.p_out);
    MmaPlan plan;
    return t.frags[0] != nullptr && p_rot <= PMAX && make_plan(a.p_in, a.p_out, p_rot <= 20 ? 32 : 16, plan);
}

int mma_group_size(const TranslateArgs<double>& a) { return std::max(a.p_in, a.p_out) <= 20 ? 32 : 16; }

cudaError_t launch_translate_mma(const DeviceTables<double>& t, const TranslateArgs<double>& a,
                                 int sm_count, cudaStream_t stream, LaunchInfo* info) {
    cudaError_t e = ensure_constants();
    if (e != cudaSuccess) return e;
    MmaPlan plan;
    const int p_rot = std::max(a.p_in, a.p_out);
    const int G = mma_group_size(a);
    if (!make_plan(a.p_in, a.p_out, G, plan)) return cudaErrorInvalidValue;
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

    using Kern = void (*)(TranslateArgs<double>, MmaTables, MmaPlan, int64_t, int, int, int, int);
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
    // tuning aid: SFMM_MMA_ABLATE bit 0 skips the elementwise phases, bits 1..3 the B, Z, C tasks
    int ablate = 0;
    if (const char* env = getenv("SFMM_MMA_ABLATE")) ablate = atoi(env);
    kern<<<grid, NTHREADS, smem, stream>>>(a, mt, plan, n_units, p_rot, lay.beta_rows(), lay.nbuf, ablate);
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

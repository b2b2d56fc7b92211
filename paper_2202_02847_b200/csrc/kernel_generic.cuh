// Generic translation kernel: any order the handle supports, any (p_in, p_out),
// M2L / M2M / L2L, float or double. It is the correctness anchor and the
// fallback for orders the tuned kernels do not cover.
//
// Mapping: one CTA works on a group of 32 translations; lane = translation, so
// every swap-matrix / faculty entry is warp-uniform and every access to the
// per-translation coefficient triangle is a unit-stride 32-lane access. The
// warps of the CTA share the triangle and split the rows (swap passes) and the
// columns (z-axis step) among themselves.
//
// Phases per group (reference pipeline.cpp:33-49):
//   G  geometry tables                                   (pipeline.cpp:52-91)
//   A  load + rotate by +alpha + scale, column order     (pipeline.cpp:148-154)
//   B  forward swap pass per (row, parity half)          (pipeline.cpp:118-136)
//   Z  z-axis step per (column, re|im)                   (pipeline.cpp:171-214)
//   C  backward swap pass per (row, parity half)         (pipeline.cpp:229-249)
//   D  rotate by -alpha + scale, store / reduce          (pipeline.cpp:251-265)
#pragma once

#include "device_math.cuh"
#include "sfmm_internal.hpp"

namespace sfmm {

// Compact triangle: row n starts at n^2 and holds re_0, re_1, im_1, re_2, ...
__host__ __device__ __forceinline__ int q_re(int n, int m) { return n * n + (m ? 2 * m - 1 : 0); }
__host__ __device__ __forceinline__ int q_im(int n, int m) { return n * n + 2 * m; }
__host__ __device__ __forceinline__ int aos_re(int n, int m) { return n * (n + 1) + 2 * m; }

constexpr int kLanes = 32;

template <typename Real>
struct GenericLayout {
    int p_rot;
    int warps;
    bool buf_in_smem;
    bool precise = false;  // double-double backward pass: beta tables and scratch twice over
    __host__ __device__ size_t tab_elems() const {
        // cb, sb: p_rot each; pw, ipw: p_rot+1 each; first-order alpha factors: 2;
        // precise: high and low words of cos/sin(m beta), p_rot each
        return (size_t)(4 * p_rot + 4 + (precise ? 4 * p_rot : 0)) * kLanes;
    }
    __host__ __device__ size_t warp_scratch_elems() const {
        return (size_t)(precise ? 2 : 1) * (p_rot + 2) * kLanes;
    }
    __host__ __device__ size_t buf_elems() const { return (size_t)p_rot * p_rot * kLanes; }
    __host__ __device__ size_t smem_bytes() const {
        return sizeof(Real) *
               (tab_elems() + warps * warp_scratch_elems() + (buf_in_smem ? buf_elems() : 0));
    }
};

template <typename Real>
struct HalfTaskCtx {
    Real* buf;          // lane-offset applied; element q at buf[q * kLanes]
    const Real* cb;     // lane-offset applied, stride kLanes
    const Real* sb;
    Real* u;            // per-warp scratch, lane-offset applied
    const Real* stream; // parity-block stream of the side in use
    const BlockDesc* desc;
    bool local_side;    // transposed blocks + halve/double of re_0
    bool negate_sb;     // backward pass rotates by -beta
    bool with_signs;    // M2L backward gather: (-1)^(n+m)
    int mmax;           // backward gather: columns > mmax read as zero
};

template <typename Real>
__device__ __forceinline__ Real gather_re(const HalfTaskCtx<Real>& c, int n, int l) {
    if (l > c.mmax) return Real(0);
    Real v = c.buf[q_re(n, l) * kLanes];
    if (c.with_signs && ((n + l) & 1)) v = -v;
    if (c.local_side && l == 0) v *= Real(0.5);
    return v;
}
template <typename Real>
__device__ __forceinline__ Real gather_im(const HalfTaskCtx<Real>& c, int n, int l) {
    if (l == 0 || l > c.mmax) return Real(0);
    Real v = c.buf[q_im(n, l) * kLanes];
    if (c.with_signs && ((n + l) & 1)) v = -v;
    return v;
}

// One parity half of swap -> rotate(beta) -> swap on row n, in place.
// Intermediate class `cls` (parity of the intermediate column index).
template <typename Real>
__device__ void swap_half_task(const HalfTaskCtx<Real>& c, int n, int cls) {
    const int cF = (n - cls) & 1, cG = cF ^ 1;
    const BlockDesc dF1 = c.desc[n * 4 + cls];
    const BlockDesc dG1 = c.desc[n * 4 + 2 + cls];
    const int nC = dF1.nrows;
    if (nC == 0) return;
    Real* ure = c.u;
    Real* uim = c.u + (size_t)nC * kLanes;

    // first swap: u_re = A_F[cls, cF] * re[cF],  u_im = A_G[cls, cG] * im[cG]
    {
        const Real* A = c.stream + dF1.offset;
        const int nk = dF1.ncols;
        for (int i = 0; i < nC; ++i) {
            Real acc = Real(0);
            for (int k = 0; k < nk; ++k)
                acc = fma_(__ldg(A + k * dF1.ld + i), gather_re(c, n, cF + 2 * k), acc);
            ure[i * kLanes] = acc;
        }
    }
    {
        const Real* A = c.stream + dG1.offset;
        const int nk = dG1.ncols;
        for (int i = 0; i < nC; ++i) {
            Real acc = Real(0);
            for (int k = 0; k < nk; ++k)
                acc = fma_(__ldg(A + k * dG1.ld + i), gather_im(c, n, cG + 2 * k), acc);
            uim[i * kLanes] = acc;
        }
    }
    // rotate by +-beta (kernels.cpp:211-217, scale == nullptr)
    for (int i = 0; i < nC; ++i) {
        const int m = cls + 2 * i;
        const Real a = ure[i * kLanes], b = uim[i * kLanes];
        const Real cm = c.cb[m * kLanes];
        const Real sm = c.negate_sb ? -c.sb[m * kLanes] : c.sb[m * kLanes];
        ure[i * kLanes] = fma_(a, cm, -(b * sm));
        uim[i * kLanes] = fma_(a, sm, b * cm);
    }
    // second swap: re[cF] = A_F[cF, cls] * u_re,  im[cG] = A_G[cG, cls] * u_im
    {
        const BlockDesc d = c.desc[n * 4 + cF];
        const Real* A = c.stream + d.offset;
        const int nr = d.nrows;
        for (int i = 0; i < nr; ++i) {
            Real acc = Real(0);
            for (int k = 0; k < nC; ++k) acc = fma_(__ldg(A + k * d.ld + i), ure[k * kLanes], acc);
            const int m = cF + 2 * i;
            if (c.local_side && m == 0) acc *= Real(2);
            c.buf[q_re(n, m) * kLanes] = acc;
        }
    }
    {
        const BlockDesc d = c.desc[n * 4 + 2 + cG];
        const Real* A = c.stream + d.offset;
        const int nr = d.nrows;
        for (int i = 0; i < nr; ++i) {
            const int m = cG + 2 * i;
            if (m == 0) continue;  // Im(C_n^0) is structurally zero
            Real acc = Real(0);
            for (int k = 0; k < nC; ++k) acc = fma_(__ldg(A + k * d.ld + i), uim[k * kLanes], acc);
            c.buf[q_im(n, m) * kLanes] = acc;
        }
    }
}

// ---- "precise" mode (no reference counterpart) -------------------------
// The rounding floor of the rotation-based M2L / L2L at high order (2e-11 at P = 20 against
// m2l_naive, the same in the reference) comes from the backward pass on local-side data alone:
// the transposed swap matrices (entries up to 1.3e5 at n = 19) amplify every rounding of the
// state between the two swaps and every deviation of (cos, sin)(m beta) from a point of the unit
// circle. Carrying that state in double-double, from cos beta = z / |r| itself through the
// recurrence, both products and the rotation, and rounding once at the end, removes it
// (1e-14 at P = 20, 2e-14 at P = 24: tests/tools/accuracy_report.py). Rounding the state in the
// middle, or keeping the double tables, gives most of the loss back. Everything else (forward
// pass, z-step, alpha rotations) stays in double as in the reference.
struct dd {
    double hi, lo;
};
__device__ __forceinline__ dd dd_quick(double a, double b) {  // |a| >= |b|
    const double s = a + b;
    return {s, b - (s - a)};
}
__device__ __forceinline__ dd dd_two_sum(double a, double b) {
    const double s = a + b, bb = s - a;
    return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd dd_two_prod(double a, double b) {
    const double p = a * b;
    return {p, __fma_rn(a, b, -p)};
}
__device__ __forceinline__ dd dd_add(dd x, dd y) {
    dd s = dd_two_sum(x.hi, y.hi);
    const dd t = dd_two_sum(x.lo, y.lo);
    s.lo += t.hi;
    s = dd_quick(s.hi, s.lo);
    s.lo += t.lo;
    return dd_quick(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_neg(dd x) { return {-x.hi, -x.lo}; }
__device__ __forceinline__ dd dd_mul_d(dd x, double b) {
    dd p = dd_two_prod(x.hi, b);
    p.lo = __fma_rn(x.lo, b, p.lo);
    return dd_quick(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_mul(dd x, dd y) {
    dd p = dd_two_prod(x.hi, y.hi);
    p.lo += x.hi * y.lo + x.lo * y.hi;
    return dd_quick(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_div(dd x, dd y) {
    const double q1 = x.hi / y.hi;
    dd r = dd_add(x, dd_neg(dd_mul_d(y, q1)));
    const double q2 = r.hi / y.hi;
    r = dd_add(r, dd_neg(dd_mul_d(y, q2)));
    const double q3 = r.hi / y.hi;
    return dd_add(dd_quick(q1, q2), dd{q3, 0.0});
}
__device__ __forceinline__ dd dd_sqrt(dd a) {  // a > 0
    const double x = 1.0 / __dsqrt_rn(a.hi), ax = a.hi * x;
    const dd r = dd_add(a, dd_neg(dd_two_prod(ax, ax)));
    return dd_two_sum(ax, r.hi * (x * 0.5));
}

// cos/sin(m beta), m < p_rot, in double-double from the shift itself (geometry.cpp:13-28 and
// the recurrence of pipeline.cpp:70-79, every operation in double-double). Lane-offset tables
// of stride kLanes: high words at hi[0 .. p_rot), low words at lo[...].
__device__ inline void precise_beta_tables(double x, double y, double z, int p_rot, double* cb_hi,
                                           double* cb_lo, double* sb_hi, double* sb_lo) {
    const dd h2 = dd_add(dd_two_prod(x, x), dd_two_prod(y, y));
    const dd r2 = dd_add(h2, dd_two_prod(z, z));
    const dd r = dd_sqrt(r2);
    dd c1, s1;
    if (h2.hi == 0.0) {
        c1 = {z < 0 ? -1.0 : 1.0, 0.0};
        s1 = {-0.0, 0.0};
    } else {
        c1 = dd_div(dd{z, 0.0}, r);
        s1 = dd_neg(dd_div(dd_sqrt(h2), r));
    }
    dd c = {1.0, 0.0}, s = {0.0, 0.0};
    for (int m = 0; m < p_rot; ++m) {
        cb_hi[m * kLanes] = c.hi, cb_lo[m * kLanes] = c.lo;
        sb_hi[m * kLanes] = s.hi, sb_lo[m * kLanes] = s.lo;
        const dd nc = dd_add(dd_mul(c, c1), dd_neg(dd_mul(s, s1)));
        const dd ns = dd_add(dd_mul(s, c1), dd_mul(c, s1));
        c = nc;
        s = ns;
    }
}

struct PreciseTables {
    const double *cb_hi, *cb_lo, *sb_hi, *sb_lo;  // lane-offset applied, stride kLanes
};

// swap_half_task on local-side data with the state in double-double (rotation by +-beta as
// c.negate_sb says). c.u must hold 4 nC values per lane.
__device__ inline void swap_half_task_precise(const HalfTaskCtx<double>& c, const PreciseTables& pt, int n,
                                              int cls) {
    const int cF = (n - cls) & 1, cG = cF ^ 1;
    const BlockDesc dF1 = c.desc[n * 4 + cls];
    const BlockDesc dG1 = c.desc[n * 4 + 2 + cls];
    const int nC = dF1.nrows;
    if (nC == 0) return;
    double* ure_h = c.u;
    double* ure_l = c.u + (size_t)nC * kLanes;
    double* uim_h = c.u + (size_t)2 * nC * kLanes;
    double* uim_l = c.u + (size_t)3 * nC * kLanes;
    {
        const double* A = c.stream + dF1.offset;
        for (int i = 0; i < nC; ++i) {
            dd acc = {0.0, 0.0};
            for (int k = 0; k < dF1.ncols; ++k)
                acc = dd_add(acc, dd_two_prod(__ldg(A + k * dF1.ld + i), gather_re(c, n, cF + 2 * k)));
            ure_h[i * kLanes] = acc.hi, ure_l[i * kLanes] = acc.lo;
        }
    }
    {
        const double* A = c.stream + dG1.offset;
        for (int i = 0; i < nC; ++i) {
            dd acc = {0.0, 0.0};
            for (int k = 0; k < dG1.ncols; ++k)
                acc = dd_add(acc, dd_two_prod(__ldg(A + k * dG1.ld + i), gather_im(c, n, cG + 2 * k)));
            uim_h[i * kLanes] = acc.hi, uim_l[i * kLanes] = acc.lo;
        }
    }
    for (int i = 0; i < nC; ++i) {
        const int m = cls + 2 * i;
        const dd a = {ure_h[i * kLanes], ure_l[i * kLanes]}, b = {uim_h[i * kLanes], uim_l[i * kLanes]};
        const dd cm = {pt.cb_hi[m * kLanes], pt.cb_lo[m * kLanes]};
        const dd sp = {pt.sb_hi[m * kLanes], pt.sb_lo[m * kLanes]};
        const dd sm = c.negate_sb ? dd_neg(sp) : sp;
        const dd nr = dd_add(dd_mul(a, cm), dd_neg(dd_mul(b, sm)));
        const dd ni = dd_add(dd_mul(a, sm), dd_mul(b, cm));
        ure_h[i * kLanes] = nr.hi, ure_l[i * kLanes] = nr.lo;
        uim_h[i * kLanes] = ni.hi, uim_l[i * kLanes] = ni.lo;
    }
    {
        const BlockDesc d = c.desc[n * 4 + cF];
        const double* A = c.stream + d.offset;
        for (int i = 0; i < d.nrows; ++i) {
            dd acc = {0.0, 0.0};
            for (int k = 0; k < nC; ++k)
                acc = dd_add(acc, dd_mul_d(dd{ure_h[k * kLanes], ure_l[k * kLanes]}, __ldg(A + k * d.ld + i)));
            const int m = cF + 2 * i;
            double v = acc.hi + acc.lo;
            if (c.local_side && m == 0) v *= 2.0;
            c.buf[q_re(n, m) * kLanes] = v;
        }
    }
    {
        const BlockDesc d = c.desc[n * 4 + 2 + cG];
        const double* A = c.stream + d.offset;
        for (int i = 0; i < d.nrows; ++i) {
            const int m = cG + 2 * i;
            if (m == 0) continue;
            dd acc = {0.0, 0.0};
            for (int k = 0; k < nC; ++k)
                acc = dd_add(acc, dd_mul_d(dd{uim_h[k * kLanes], uim_l[k * kLanes]}, __ldg(A + k * d.ld + i)));
            c.buf[q_im(n, m) * kLanes] = acc.hi + acc.lo;
        }
    }
}

// z-axis step on one column (m, part) in place.
template <typename Real>
__device__ void zstep_task(const DeviceTables<Real>& t, int kind, int p_in, int p_out, Real* buf,
                           Real* u, int m, int part) {
    const int kin = p_in - m, kout = p_out - m;
    for (int k = 0; k < kin; ++k)
        u[k * kLanes] = buf[(part ? q_im(m + k, m) : q_re(m + k, m)) * kLanes];
    for (int i = 0; i < kout; ++i) {
        Real acc = Real(0);
        if (kind == KIND_M2L) {  // kernels.cpp:118-167
            const Real* f = t.fac + 2 * m + i;
            for (int k = 0; k < kin; ++k) acc = fma_(__ldg(f + k), u[k * kLanes], acc);
        } else if (kind == KIND_M2M) {  // kernels.cpp:169-182
            const int klim = min(i, kin - 1);
            for (int k = 0; k <= klim; ++k) acc = fma_(__ldg(t.winv + (i - k)), u[k * kLanes], acc);
        } else {  // kernels.cpp:184-196
            for (int k = i; k < kin; ++k) acc = fma_(__ldg(t.inv + (k - i)), u[k * kLanes], acc);
        }
        buf[(part ? q_im(m + i, m) : q_re(m + i, m)) * kLanes] = acc;
    }
}

template <typename Real>
__device__ __forceinline__ Real warp_sum(Real v) {
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
    return v;
}

template <typename Real, bool BUF_SMEM, bool PRECISE = false>
__global__ void __launch_bounds__(256)
translate_generic_kernel(DeviceTables<Real> t, TranslateArgs<Real> a, Real* gscratch,
                         int64_t n_groups, int p_rot) {
    static_assert(!PRECISE || sizeof(Real) == 8, "the precise mode is double precision");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (a.fail_flag && *a.fail_flag) return;

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int W = blockDim.x >> 5;
    GenericLayout<Real> lay{p_rot, W, BUF_SMEM, PRECISE};

    Real* sm = reinterpret_cast<Real*>(smem_raw);
    Real* cb = sm + lane;
    Real* sb = cb + (size_t)p_rot * kLanes;
    Real* pw = sb + (size_t)p_rot * kLanes;
    Real* ipw = pw + (size_t)(p_rot + 1) * kLanes;
    Real* ca1 = ipw + (size_t)(p_rot + 1) * kLanes;
    Real* sa1 = ca1 + kLanes;
    Real* cbh = sa1 + kLanes;  // PRECISE: double-double cos/sin(m beta)
    Real* cbl = cbh + (size_t)p_rot * kLanes;
    Real* sbh = cbl + (size_t)p_rot * kLanes;
    Real* sbl = sbh + (size_t)p_rot * kLanes;
    Real* u = sm + lay.tab_elems() + (size_t)warp * lay.warp_scratch_elems() + lane;
    Real* buf = (BUF_SMEM ? sm + lay.tab_elems() + (size_t)W * lay.warp_scratch_elems()
                          : gscratch + (size_t)blockIdx.x * lay.buf_elems()) +
                lane;

    const int kind = a.kind, p_in = a.p_in, p_out = a.p_out;
    const bool src_local = kind == KIND_L2L;
    const bool dst_local = kind != KIND_M2M;
    const int cols = min(p_in, p_out);
    const bool accumulate = a.src_index != nullptr;

    for (int64_t g = blockIdx.x; g < n_groups; g += gridDim.x) {
        const int64_t b = g * kLanes + lane;
        int64_t src = b;
        bool active = b < a.n;
        if (active && accumulate) {
            src = a.src_index[b];
            active = src >= 0;
        }

        // ---- G: geometry (pipeline.cpp:52-91); idle lanes get the benign
        // shift (0,0,1) like the reference's idle columns (:56-61)
        if (warp == 0) {
            Real x = 0, y = 0, z = 1;
            if (active) {
                x = a.shifts[3 * b];
                y = a.shifts[3 * b + 1];
                z = a.shifts[3 * b + 2];
            }
            const Angles<Real> ang = decompose_angles(x, y, z);
            *ca1 = ang.ca;
            *sa1 = ang.sa;
            Real c = 1, s = 0;
            for (int m = 0; m < p_rot; ++m) {
                cb[m * kLanes] = c;
                sb[m * kLanes] = s;
                const Real nc = fma_(c, ang.cb, -(s * ang.sb));
                const Real ns = fma_(s, ang.cb, c * ang.sb);
                c = nc;
                s = ns;
            }
            Real p = 1, q = 1;
            const Real inv = Real(1) / ang.rn;
            for (int n = 0; n <= p_rot; ++n) {
                pw[n * kLanes] = p;
                ipw[n * kLanes] = q;
                p *= ang.rn;
                q *= inv;
            }
        }
        if constexpr (PRECISE) {
            if (warp == 1 % W) {
                double x = 0, y = 0, z = 1;
                if (active) {
                    x = a.shifts[3 * b];
                    y = a.shifts[3 * b + 1];
                    z = a.shifts[3 * b + 2];
                }
                precise_beta_tables(x, y, z, p_rot, cbh, cbl, sbh, sbl);
            }
        }
        __syncthreads();

        // ---- A: load, rotate by +alpha, scale; warp w owns columns w, w+W, ...
        {
            const Real c1 = *ca1, s1 = *sa1;
            Real c = 1, s = 0;
            int m_at = 0;
            for (int m = warp; m < p_in; m += W) {
                for (; m_at < m; ++m_at) {
                    const Real nc = fma_(c, c1, -(s * s1));
                    const Real ns = fma_(s, c1, c * s1);
                    c = nc;
                    s = ns;
                }
                for (int n = m; n < p_in; ++n) {
                    Real re = 0, im = 0;
                    if (active) {
                        if (a.in_layout == LAYOUT_ROWS) {
                            const Real* row = a.in + src * a.in_stride + rows_off(n) + 2 * m;
                            re = row[0];
                            if (m) im = row[1];
                        } else {
                            re = a.in[(int64_t)aos_re(n, m) * a.in_stride + src];
                            if (m) im = a.in[(int64_t)(aos_re(n, m) + 1) * a.in_stride + src];
                        }
                    }
                    const Real sc = src_local ? pw[n * kLanes] : ipw[(n + 1) * kLanes];
                    const Real nr = sc * fma_(re, c, -(im * s));
                    const Real ni = sc * fma_(re, s, im * c);
                    buf[q_re(n, m) * kLanes] = nr;
                    if (m) buf[q_im(n, m) * kLanes] = ni;
                }
            }
        }
        __syncthreads();

        // ---- B: forward swap passes
        {
            HalfTaskCtx<Real> c;
            c.buf = buf;
            c.cb = cb;
            c.sb = sb;
            c.u = u;
            c.stream = t.stream[src_local ? 1 : 0];
            c.desc = t.desc[src_local ? 1 : 0];
            c.local_side = src_local;
            c.negate_sb = false;
            c.with_signs = false;
            c.mmax = p_in;
            for (int task = warp; task < 2 * p_in; task += W) {
                if constexpr (PRECISE) {
                    // L2L: the forward pass works on local-side data as well
                    if (src_local) swap_half_task_precise(c, PreciseTables{cbh, cbl, sbh, sbl}, p_in - 1 - (task >> 1), task & 1);
                    else swap_half_task(c, p_in - 1 - (task >> 1), task & 1);
                } else {
                    swap_half_task(c, p_in - 1 - (task >> 1), task & 1);
                }
            }
        }
        __syncthreads();

        // ---- Z: z-axis step per column
        for (int task = warp; task < 2 * cols; task += W) {
            const int m = task >> 1, part = task & 1;
            if (part && m == 0) continue;
            zstep_task(t, kind, p_in, p_out, buf, u, m, part);
        }
        __syncthreads();

        // ---- C: backward swap passes
        {
            HalfTaskCtx<Real> c;
            c.buf = buf;
            c.cb = cb;
            c.sb = sb;
            c.u = u;
            c.stream = t.stream[dst_local ? 1 : 0];
            c.desc = t.desc[dst_local ? 1 : 0];
            c.local_side = dst_local;
            c.negate_sb = true;
            c.with_signs = kind == KIND_M2L;
            for (int task = warp; task < 2 * p_out; task += W) {
                const int n = p_out - 1 - (task >> 1);
                c.mmax = min(n, cols - 1);
                if constexpr (PRECISE) {
                    // local-side data only (M2L, L2L): the multipole-side pass of M2M is benign
                    if (dst_local) swap_half_task_precise(c, PreciseTables{cbh, cbl, sbh, sbl}, n, task & 1);
                    else swap_half_task(c, n, task & 1);
                } else {
                    swap_half_task(c, n, task & 1);
                }
            }
        }
        __syncthreads();

        // ---- D: rotate by -alpha, scale, store
        {
            const Real c1 = *ca1, s1 = *sa1;
            Real c = 1, s = 0;
            int m_at = 0;
            for (int m = warp; m < p_out; m += W) {
                for (; m_at < m; ++m_at) {
                    const Real nc = fma_(c, c1, -(s * s1));
                    const Real ns = fma_(s, c1, c * s1);
                    c = nc;
                    s = ns;
                }
                const Real ms = -s;
                for (int n = m; n < p_out; ++n) {
                    const Real re = buf[q_re(n, m) * kLanes];
                    const Real im = m ? buf[q_im(n, m) * kLanes] : Real(0);
                    const Real sc = dst_local ? ipw[n * kLanes] : pw[(n + 1) * kLanes];
                    Real nr = sc * fma_(re, c, -(im * ms));
                    Real ni = sc * fma_(re, ms, im * c);
                    if (!accumulate) {
                        if (active) {
                            a.out[(int64_t)aos_re(n, m) * a.out_stride + b] = nr;
                            a.out[(int64_t)(aos_re(n, m) + 1) * a.out_stride + b] =
                                m ? ni : Real(0);
                        }
                    } else {
                        nr = warp_sum(nr);
                        if (m) ni = warp_sum(ni);
                        if (lane == 0) {
                            a.out[(int64_t)aos_re(n, m) * a.out_stride + g] = nr;
                            if (m) a.out[(int64_t)(aos_re(n, m) + 1) * a.out_stride + g] = ni;
                        }
                    }
                }
            }
        }
        __syncthreads();
    }
}

}  // namespace sfmm

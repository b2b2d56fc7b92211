// Particle <-> expansion steps either side of the translation path:
//   P2M        multipole of the point charges of a box      (reference harmonics.cpp:105-117)
//   L2P        potential of a local expansion at a point    (reference harmonics.cpp:119-152)
// both built on the regular solid harmonics R_n^m (harmonics.cpp:18-50).
//
// Mapping: a lane owns columns m of the triangle. The reference's recurrences run in n for a
// fixed m ((n^2 - m^2) R_n^m = (2n-1) z R_{n-1}^m - |r|^2 R_{n-2}^m) once the diagonal R_m^m is
// known, so a lane carries R_{n-1}^m and R_{n-2}^m in two registers each and no triangle of
// harmonics is ever stored; lane l takes the columns l and P-1-l (P+1 coefficients whatever l
// is), ceil(P/2) lanes serve one box (P2M) or one point (L2P). The operation order and the fused multiply-adds are
// those of the reference built with -mfma -ffp-contract=fast (the parity build, DESIGN.md §2;
// read off its object code and pinned by tests/test_oracle.py):
//   |r|^2          = fma(z, z, fma(x, x, y*y))
//   R_n^n          = 1/(2n) * (fma(-y, im, x*re),  fma(x, im, y*re))
//   R_n^m (m < n)  = 1/(n^2-m^2) * fma(-|r|^2, R_{n-2}^m, ((2n-1) z) * R_{n-1}^m)
//   P2M            : M_n^m = fma(q, R_n^m, M_n^m), charges in list order
//   L2P            : total = fma(L_n^0, R_n^0, total) ; row = row + fma(Lre, Rre, Lim*Rim), m
//                    ascending from 0 ; total = total + (row + row), n ascending
// Compiled with -fmad=false: every fused operation below is explicit.
#include <algorithm>
#include <cfloat>

#include "device_math.cuh"
#include "sfmm_internal.hpp"

namespace sfmm {
namespace {

constexpr int kHarmMaxOrder = 32;  // paired-column kernels (a warp serves whole boxes / points); plain kernels above

template <typename Real>
__device__ __forceinline__ Real real_min();
template <>
__device__ __forceinline__ double real_min<double>() { return DBL_MIN; }
template <>
__device__ __forceinline__ float real_min<float>() { return FLT_MIN; }

__device__ __forceinline__ double sqrt_(double v) { return __dsqrt_rn(v); }
__device__ __forceinline__ float sqrt_(float v) { return __fsqrt_rn(v); }

// std::hypot(x, y, z) as libstdc++ evaluates it (solid.hpp:21-23: norm): scaled by the largest
// magnitude. Only compared with the smallest normal number (harmonics.cpp:11-14).
template <typename Real>
__device__ __forceinline__ bool effectively_zero(Real x, Real y, Real z) {
    const Real ax = fabs(x), ay = fabs(y), az = fabs(z);
    const Real a = fmax(fmax(ax, ay), az);
    if (a == Real(0)) return true;
    if (!(a < real_min<Real>() * Real(4))) return false;  // far from the threshold (or not a number)
    const Real xs = ax / a, ys = ay / a, zs = az / a;
    const Real n = a * sqrt_(fma_(zs, zs, fma_(xs, xs, ys * ys)));
    return n < real_min<Real>();
}

// position of (n, m, part) in the output layouts
__device__ __forceinline__ int64_t out_index(int layout, int64_t b, int n, int m, int part, int order,
                                             int64_t stride) {
    const int c = n * (n + 1) + 2 * m + part;
    if (layout == LAYOUT_SOA) return (int64_t)c * stride + b;
    if (layout == LAYOUT_ROWS) return b * rows_off(order) + rows_off(n) + 2 * m + part;
    return b * ((int64_t)order * (order + 1)) + c;
}

// P2M. A box is worked on by ceil(P/2) lanes: lane l owns the columns m = l and m = P-1-l of
// the triangle, P+1 coefficients together whatever l is (the triangle is balanced by pairing
// its longest column with its shortest), so a warp holds floor(32 / ceil(P/2)) boxes and almost
// every lane is busy (P = 20: 3 boxes, 30 lanes, 21 coefficients each). The coefficients of a
// lane are numbered by "slots" s = 0..P: first the rows n = m .. P-1 of its long column, then
// those of the short one; the slot loop is unrolled, so the accumulators, the reciprocals
// 1/(n^2-m^2) and the two-term recurrence state stay in registers. Charges are taken in list
// order (the accumulation M = fma(q, R, M) is a chain in the reference too); two charges are in
// flight per trip for instruction-level parallelism.
// state of one charge in the slot loop of p2m_kernel
template <typename Real>
struct ChargeState {
    Real q, z, r2, dre, dim, p1re, p1im, p2re, p2im;
    bool zero;
    // loads the charge, runs the diagonal recurrence up to R_mtop^mtop and leaves R_mA^mA in p1
    __device__ __forceinline__ void start(Real x, Real y, Real z_, Real q_, int mA, int mtop, const Real* inv2n) {
        q = q_, z = z_;
        zero = effectively_zero(x, y, z);
        r2 = fma_(z, z, fma_(x, x, y * y));
        dre = Real(1), dim = Real(0);
        p1re = Real(1), p1im = Real(0);
        for (int n = 1; n <= mtop; ++n) {
            const Real nre = inv2n[n] * fma_(-y, dim, x * dre);
            const Real nim = inv2n[n] * fma_(x, dim, y * dre);
            dre = nre;
            dim = nim;
            if (n == mA) p1re = dre, p1im = dim;
        }
        p2re = p2im = Real(0);
    }
    // coefficient (n, m) = row k of the current column; `first` = first slot of the short column
    __device__ __forceinline__ void slot(int n, int m, int k, bool first, Real den, Real& re, Real& im) {
        if (first) p1re = dre, p1im = dim;
        const Real zf = Real(2 * n - 1) * z;
        Real a = zf * p1re, c = zf * p1im;
        const Real a2 = fma_(-r2, p2re, a), c2 = fma_(-r2, p2im, c);
        a = k >= 2 ? a2 : a;
        c = k >= 2 ? c2 : c;
        re = den * a;
        im = m == 0 ? Real(0) : den * c;
        re = k == 0 ? p1re : re;
        im = k == 0 ? p1im : im;
        p2re = k == 0 ? p2re : p1re;
        p2im = k == 0 ? p2im : p1im;
        p1re = re, p1im = im;
        if (zero) {
            re = n == 0 ? Real(1) : Real(0);
            im = Real(0);
        }
    }
};

// P2M. A box is worked on by ceil(P/2) lanes: lane l owns the columns m = l and m = P-1-l of
// the triangle, P+1 coefficients together whatever l is (the triangle is balanced by pairing
// its longest column with its shortest), so a warp holds floor(32 / ceil(P/2)) boxes and almost
// every lane is busy (P = 20: 3 boxes, 30 lanes, 21 coefficients each). The coefficients of a
// lane are numbered by "slots" s = 0..P: first the rows n = m .. P-1 of its long column, then
// those of the short one; the slot loop is unrolled, so the accumulators and the two-term
// recurrence state stay in registers (the reciprocals 1/(n^2-m^2) come from a shared table).
// Charges are taken in list order (M = fma(q, R, M) is a chain in the reference too); the
// recurrences of two consecutive charges run side by side (they are latency bound), and the
// next pair is loaded while the current one computes.
template <typename Real, int PM>
__global__ void __launch_bounds__(128, PM <= 20 ? 3 : 2)
p2m_kernel(const int64_t* __restrict__ box_ptr, const Real* __restrict__ charges,
           const Real* __restrict__ centers, int64_t n_boxes, int order, int layout,
           Real* __restrict__ out, int64_t stride) {
    __shared__ Real inv2n[kHarmMaxOrder + 1];
    __shared__ Real denom_tab[(PM + 1) * (PM + 1)];  // [n][m]
    constexpr int LD = PM + 1;
    if (threadIdx.x <= kHarmMaxOrder) inv2n[threadIdx.x] = threadIdx.x ? Real(1) / Real(2 * (int)threadIdx.x) : Real(0);
    for (int i = threadIdx.x; i < LD * LD; i += blockDim.x) {
        const int n = i / LD, mm = i - n * LD;
        denom_tab[i] = mm < n ? Real(1) / Real(n * n - mm * mm) : Real(0);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int half = (order + 1) >> 1, per_warp = 32 / half;
    const int sub = lane / half, l = lane - sub * half;
    const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t b = warp * per_warp + sub;
    if (sub >= per_warp || b >= n_boxes) return;
    const int mA = l, mB = order - 1 - l;
    const int cA = order - mA;                   // slots of the long column
    const int total = mB > mA ? order + 1 : cA;  // odd orders: the middle column stands alone
    const int mtop = mB > mA ? mB : mA;
    Real are[PM + 1], aim[PM + 1];
#pragma unroll
    for (int s = 0; s <= PM; ++s) are[s] = aim[s] = Real(0);
    const Real cx = centers[3 * b], cy = centers[3 * b + 1], cz = centers[3 * b + 2];
    const int64_t j0 = box_ptr[b], j1 = box_ptr[b + 1];
    // charge pair (j, j + 1); the data of the next pair is in flight during the slot loop
    Real nx[2], ny[2], nz[2], nq[2];
    auto fetch = [&](int64_t j) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int64_t jj = j + u < j1 ? j + u : (j1 > j0 ? j1 - 1 : j0);
            const bool ok = j + u < j1;
            nx[u] = ok ? charges[4 * jj] : Real(0);
            ny[u] = ok ? charges[4 * jj + 1] : Real(0);
            nz[u] = ok ? charges[4 * jj + 2] : Real(0);
            nq[u] = ok ? charges[4 * jj + 3] : Real(0);
        }
    };
    if (j0 < j1) fetch(j0);
    for (int64_t j = j0; j < j1; j += 2) {
        ChargeState<Real> c0, c1;
        const bool two = j + 1 < j1;
        c0.start(nx[0] - cx, ny[0] - cy, nz[0] - cz, nq[0], mA, mtop, inv2n);
        c1.start(nx[1] - cx, ny[1] - cy, nz[1] - cz, nq[1], mA, mtop, inv2n);
        if (j + 2 < j1) fetch(j + 2);
#pragma unroll
        for (int s = 0; s <= PM; ++s) {
            if (s < total) {
                const bool second = s >= cA;
                const int m = second ? mB : mA, k = second ? s - cA : s, n = m + k;
                const Real den = denom_tab[n * LD + m];
                Real re0, im0, re1, im1;
                c0.slot(n, m, k, s == cA, den, re0, im0);
                c1.slot(n, m, k, s == cA, den, re1, im1);
                are[s] = fma_(c0.q, re0, are[s]);
                aim[s] = fma_(c0.q, im0, aim[s]);
                if (two) {
                    are[s] = fma_(c1.q, re1, are[s]);
                    aim[s] = fma_(c1.q, im1, aim[s]);
                }
            }
        }
    }
#pragma unroll
    for (int s = 0; s <= PM; ++s) {
        if (s < total) {
            const int m = s < cA ? mA : mB, n = m + (s < cA ? s : s - cA);
            out[out_index(layout, b, n, m, 0, order, stride)] = are[s];
            out[out_index(layout, b, n, m, 1, order, stride)] = aim[s];
        }
    }
    // padding of the rows layout (rows of odd length carry two zeros)
    if (layout == LAYOUT_ROWS && l == 0) {
        for (int n = 0; n < order; ++n)
            for (int k = 2 * (n + 1); k < rows_off(n + 1) - rows_off(n); ++k)
                out[b * rows_off(order) + rows_off(n) + k] = Real(0);
    }
}

// L2P: out[i] = paired_sum(L[box(i)], regular(x_i - centre[box(i)])) (harmonics.cpp:119-152).
// Same lane mapping as P2M: ceil(P/2) lanes per point, lane l owns the columns m = l and
// m = P-1-l, a warp works on floor(32 / ceil(P/2)) consecutive points at a time and walks a
// contiguous range of points. The local expansion of the current box of every sub-group stays
// in shared memory (points of one box usually follow one another). The sum over m of a row is
// taken in ascending m like the reference's loop: the terms L_n^m * conj R_n^m go through shared
// memory, lane l then adds the rows l and P-1-l (again P-1 additions whatever l is), and the
// first lane of the sub-group folds the rows in ascending n.
// dynamic shared memory: denom [P][P+1] | per warp and sub-group: locals [P(P+1)], terms
// [P(P+1)/2], rows [P]
extern __shared__ __align__(16) unsigned char harm_smem[];
// STAGE: the local expansion of the current box is copied to shared memory (SoA / rows
// layouts, whose global accesses are strided); without it (AoS layout) the lanes read it
// straight from global memory through L1 — the 3.4 KB of a box are reused by all its points —
// and the shared memory saved lets 2.6x as many warps run per SM.
template <typename Real, bool STAGE>
__global__ void __launch_bounds__(128)
eval_local_kernel(const int32_t* __restrict__ point_box, const Real* __restrict__ points,
                  const Real* __restrict__ centers, int64_t n_points, int64_t n_boxes, int order,
                  int layout, const Real* __restrict__ locals, int64_t stride, Real* __restrict__ out) {
    __shared__ Real inv2n[kHarmMaxOrder + 1];
    const int LD = order + 1, S = order * (order + 1);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int half = (order + 1) >> 1, per_warp = 32 / half;
    const int sub = lane / half, l = lane - sub * half;
    const bool lane_on = sub < per_warp;
    const size_t per_sub = (STAGE ? (size_t)S : 0) + (size_t)S / 2 + order;  // locals, terms (triangle), rows
    Real* denom = reinterpret_cast<Real*>(harm_smem);
    Real* my_loc = denom + order * LD + ((size_t)w * per_warp + (lane_on ? sub : 0)) * per_sub;
    Real* my_terms = my_loc + (STAGE ? S : 0);
    Real* my_rows = my_terms + S / 2;
    if (threadIdx.x <= kHarmMaxOrder) inv2n[threadIdx.x] = threadIdx.x ? Real(1) / Real(2 * (int)threadIdx.x) : Real(0);
    for (int i = threadIdx.x; i < order * LD; i += blockDim.x) {
        const int n = i / LD, mm = i - n * LD;
        denom[i] = (mm < n) ? Real(1) / Real(n * n - mm * mm) : Real(0);
    }
    __syncthreads();
    const int mA = l, mB = order - 1 - l;
    const int cA = order - mA;
    const int total = mB > mA ? order + 1 : cA;
    const int mtop = mB > mA ? mB : mA;
    const int64_t warps = (int64_t)gridDim.x * 4, wid = (int64_t)blockIdx.x * 4 + w;
    int64_t chunk = (n_points + warps - 1) / warps;
    chunk = (chunk + per_warp - 1) / per_warp * per_warp;
    const int64_t i0 = wid * chunk, i1 = i0 + chunk < n_points ? i0 + chunk : n_points;
    int64_t cached = -1;
    for (int64_t base = i0; base < i1; base += per_warp) {
        const int64_t i = base + sub;
        bool on = lane_on && i < i1;
        int64_t b = on ? (point_box ? (int64_t)point_box[i] : i) : -1;
        if (on && (b < 0 || b >= n_boxes)) {  // no such box: the point gets a NaN, nothing is read
            if (l == 0) out[i] = (Real)__longlong_as_double(0x7ff8000000000000ll);
            on = false;
            b = -1;
        }
        if (STAGE && on && b != cached) {  // the lanes of a sub-group agree
            if (layout == LAYOUT_AOS) {
                for (int c = l; c < S; c += half) my_loc[c] = locals[b * S + c];
            } else {
                for (int n = 0; n < order; ++n)
                    for (int c = l; c < 2 * (n + 1); c += half)
                        my_loc[n * (n + 1) + c] = locals[out_index(layout, b, n, c >> 1, c & 1, order, stride)];
            }
            cached = b;
        }
        __syncwarp();
        if (on) {
            ChargeState<Real> st;
            st.start(points[3 * i] - centers[3 * b], points[3 * i + 1] - centers[3 * b + 1],
                     points[3 * i + 2] - centers[3 * b + 2], Real(0), mA, mtop, inv2n);
            for (int s = 0; s < total; ++s) {
                const bool second = s >= cA;
                const int m = second ? mB : mA, k = second ? s - cA : s, n = m + k;
                Real vre, vim;
                st.slot(n, m, k, s == cA, denom[n * LD + m], vre, vim);
                const Real* lp = STAGE ? my_loc : locals + b * S;
                const Real lre = lp[n * (n + 1) + 2 * m], lim = lp[n * (n + 1) + 2 * m + 1];
                // column 0 keeps the two factors apart: total = fma(L_n^0, R_n^0, total)
                my_terms[n * (n + 1) / 2 + m] = m == 0 ? vre : fma_(lre, vre, lim * vim);
            }
        }
        __syncwarp();
        if (on) {
            // rows l and P-1-l, each in ascending m
            for (int pass = 0; pass < 2; ++pass) {
                const int n = pass ? mB : mA;
                if (pass && mB <= mA) break;
                Real rowsum = Real(0);
                for (int k = 1; k <= n; ++k) rowsum = rowsum + my_terms[n * (n + 1) / 2 + k];
                my_rows[n] = rowsum;
            }
        }
        __syncwarp();
        if (on && l == 0) {
            Real total_sum = Real(0);
            for (int n = 0; n < order; ++n) {
                total_sum = fma_((STAGE ? my_loc : locals + b * S)[n * (n + 1)], my_terms[n * (n + 1) / 2], total_sum);
                const Real r = my_rows[n];
                total_sum = total_sum + (r + r);
            }
            out[i] = total_sum;
        }
        __syncwarp();
    }
}

// ---- orders above 32 (the handle goes to 86 in double precision) ---------------------------
// Same arithmetic and the same orders of summation, plain mapping: one warp per box / point,
// lane = m, m + 32, m + 64; P2M accumulates in the output itself (a thread owns its
// coefficients), L2P keeps the products in a shared triangle. Dynamic shared memory:
// inv2n [P + 1] | L2P: terms [P(P+1)/2], rows [P] (one warp per block).
template <typename Real>
__global__ void __launch_bounds__(32)
p2m_generic_kernel(const int64_t* __restrict__ box_ptr, const Real* __restrict__ charges,
                   const Real* __restrict__ centers, int64_t n_boxes, int order, int layout,
                   Real* __restrict__ out, int64_t stride) {
    Real* inv2n = reinterpret_cast<Real*>(harm_smem);
    for (int i = threadIdx.x; i <= order; i += 32) inv2n[i] = i ? Real(1) / Real(2 * i) : Real(0);
    __syncwarp();
    const int lane = threadIdx.x;
    for (int64_t b = blockIdx.x; b < n_boxes; b += gridDim.x) {
        const Real cx = centers[3 * b], cy = centers[3 * b + 1], cz = centers[3 * b + 2];
        const int64_t j0 = box_ptr[b], j1 = box_ptr[b + 1];
        for (int m = lane; m < order; m += 32) {
            for (int n = m; n < order; ++n) {
                out[out_index(layout, b, n, m, 0, order, stride)] = Real(0);
                out[out_index(layout, b, n, m, 1, order, stride)] = Real(0);
            }
            for (int64_t j = j0; j < j1; ++j) {
                ChargeState<Real> st;
                st.start(charges[4 * j] - cx, charges[4 * j + 1] - cy, charges[4 * j + 2] - cz, charges[4 * j + 3], m,
                         m, inv2n);
                for (int n = m; n < order; ++n) {
                    Real re, im;
                    st.slot(n, m, n - m, false, n > m ? Real(1) / Real(n * n - m * m) : Real(0), re, im);
                    const int64_t ir = out_index(layout, b, n, m, 0, order, stride);
                    const int64_t ii = out_index(layout, b, n, m, 1, order, stride);
                    out[ir] = fma_(st.q, re, out[ir]);
                    out[ii] = fma_(st.q, im, out[ii]);
                }
            }
        }
        if (layout == LAYOUT_ROWS && lane == 0) {
            for (int n = 0; n < order; ++n)
                for (int k = 2 * (n + 1); k < rows_off(n + 1) - rows_off(n); ++k)
                    out[b * rows_off(order) + rows_off(n) + k] = Real(0);
        }
    }
}

template <typename Real>
__global__ void __launch_bounds__(32)
eval_local_generic_kernel(const int32_t* __restrict__ point_box, const Real* __restrict__ points,
                          const Real* __restrict__ centers, int64_t n_points, int64_t n_boxes, int order,
                          int layout, const Real* __restrict__ locals, int64_t stride, Real* __restrict__ out) {
    Real* inv2n = reinterpret_cast<Real*>(harm_smem);
    Real* terms = inv2n + order + 1;
    Real* rows = terms + order * (order + 1) / 2;
    for (int i = threadIdx.x; i <= order; i += 32) inv2n[i] = i ? Real(1) / Real(2 * i) : Real(0);
    __syncwarp();
    const int lane = threadIdx.x;
    for (int64_t i = blockIdx.x; i < n_points; i += gridDim.x) {
        const int64_t b = point_box ? (int64_t)point_box[i] : i;
        if (b < 0 || b >= n_boxes) {
            if (lane == 0) out[i] = (Real)__longlong_as_double(0x7ff8000000000000ll);
            continue;
        }
        const Real x = points[3 * i] - centers[3 * b], y = points[3 * i + 1] - centers[3 * b + 1],
                   z = points[3 * i + 2] - centers[3 * b + 2];
        for (int m = lane; m < order; m += 32) {
            ChargeState<Real> st;
            st.start(x, y, z, Real(0), m, m, inv2n);
            for (int n = m; n < order; ++n) {
                Real vre, vim;
                st.slot(n, m, n - m, false, n > m ? Real(1) / Real(n * n - m * m) : Real(0), vre, vim);
                const Real lre = locals[out_index(layout, b, n, m, 0, order, stride)];
                const Real lim = locals[out_index(layout, b, n, m, 1, order, stride)];
                terms[n * (n + 1) / 2 + m] = m == 0 ? vre : fma_(lre, vre, lim * vim);
            }
        }
        __syncwarp();
        for (int n = lane; n < order; n += 32) {
            Real rowsum = Real(0);
            for (int k = 1; k <= n; ++k) rowsum = rowsum + terms[n * (n + 1) / 2 + k];
            rows[n] = rowsum;
        }
        __syncwarp();
        if (lane == 0) {
            Real total = Real(0);
            for (int n = 0; n < order; ++n) {
                total = fma_(locals[out_index(layout, b, n, 0, 0, order, stride)], terms[n * (n + 1) / 2], total);
                total = total + (rows[n] + rows[n]);
            }
            out[i] = total;
        }
        __syncwarp();
    }
}

}  // namespace

template <typename Real>
cudaError_t launch_p2m(const int64_t* box_ptr, const Real* charges, const Real* centers,
                       int64_t n_boxes, int order, int layout, Real* out, int64_t stride,
                       cudaStream_t stream) {
    if (n_boxes <= 0) return cudaSuccess;
    if (order > kHarmMaxOrder) {
        const size_t smem = sizeof(Real) * (order + 1);
        const unsigned blocks = (unsigned)std::min<int64_t>(n_boxes, 148 * 32);
        p2m_generic_kernel<Real><<<blocks, 32, smem, stream>>>(box_ptr, charges, centers, n_boxes, order, layout, out,
                                                               stride);
        return cudaGetLastError();
    }
    const int per_warp = 32 / ((order + 1) / 2);
    const int64_t warps = (n_boxes + per_warp - 1) / per_warp;
    const unsigned grid = (unsigned)((warps + 3) / 4);
#define SFMM_P2M(PM)                                                                                  \
    p2m_kernel<Real, PM><<<grid, 128, 0, stream>>>(box_ptr, charges, centers, n_boxes, order, layout, \
                                                   out, stride)
    if (order <= 8) SFMM_P2M(8);
    else if (order <= 12) SFMM_P2M(12);
    else if (order <= 16) SFMM_P2M(16);
    else if (order <= 20) SFMM_P2M(20);
    else if (order <= 24) SFMM_P2M(24);
    else SFMM_P2M(32);
#undef SFMM_P2M
    return cudaGetLastError();
}

template <typename Real>
cudaError_t launch_eval_local(const int32_t* point_box, const Real* points, const Real* centers,
                              int64_t n_points, int64_t n_boxes, int order, int layout,
                              const Real* locals, int64_t stride, Real* out, cudaStream_t stream) {
    if (n_points <= 0) return cudaSuccess;
    if (order > kHarmMaxOrder) {
        const size_t smem = sizeof(Real) * ((size_t)order + 1 + (size_t)order * (order + 1) / 2 + order);
        const unsigned blocks = (unsigned)std::min<int64_t>(n_points, 148 * 8);
        eval_local_generic_kernel<Real><<<blocks, 32, smem, stream>>>(point_box, points, centers, n_points, n_boxes,
                                                                      order, layout, locals, stride, out);
        return cudaGetLastError();
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int per_warp = 32 / ((order + 1) / 2);
    const bool stage = layout != LAYOUT_AOS;
    const size_t smem = sizeof(Real) * ((size_t)order * (order + 1) +
                                        4 * per_warp * ((size_t)order * (order + 1) * (stage ? 3 : 1) / 2 + order));
    auto kern = stage ? eval_local_kernel<Real, true> : eval_local_kernel<Real, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 1;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, smem);
    if (e != cudaSuccess) return e;
    const unsigned grid = (unsigned)std::min<int64_t>((n_points + 3) / 4, (int64_t)sms * std::max(per_sm, 1));
    kern<<<grid, 128, smem, stream>>>(point_box, points, centers, n_points, n_boxes, order, layout, locals, stride,
                                      out);
    return cudaGetLastError();
}

int harmonics_max_order() { return 86; }  // the paired-column kernels to 32, plain kernels above

#define SFMM_INSTANTIATE(Real)                                                                    \
    template cudaError_t launch_p2m<Real>(const int64_t*, const Real*, const Real*, int64_t, int, \
                                          int, Real*, int64_t, cudaStream_t);                     \
    template cudaError_t launch_eval_local<Real>(const int32_t*, const Real*, const Real*,        \
                                                 int64_t, int64_t, int, int, const Real*,         \
                                                 int64_t, Real*, cudaStream_t);
SFMM_INSTANTIATE(double)
SFMM_INSTANTIATE(float)
#undef SFMM_INSTANTIATE

}  // namespace sfmm

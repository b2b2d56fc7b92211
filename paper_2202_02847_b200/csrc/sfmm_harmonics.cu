// Particle <-> expansion steps either side of the translation path:
//   P2M        multipole of the point charges of a box      (reference harmonics.cpp:105-117)
//   L2P        potential of a local expansion at a point    (reference harmonics.cpp:119-152)
// both built on the regular solid harmonics R_n^m (harmonics.cpp:18-50).
//
// Mapping: one warp per box (P2M) or per evaluation point (L2P), lane = m. The reference's
// recurrences run in n for a fixed m ((n^2 - m^2) R_n^m = (2n-1) z R_{n-1}^m - |r|^2 R_{n-2}^m)
// once the diagonal R_m^m is known, so a lane carries R_{n-1}^m and R_{n-2}^m in two registers
// each and no triangle is ever stored. The operation order and the fused multiply-adds are
// those of the reference built with -mfma -ffp-contract=fast (the parity build, DESIGN.md §2;
// read off its object code and pinned by tests/test_oracle.py):
//   |r|^2          = fma(z, z, fma(x, x, y*y))
//   R_n^n          = 1/(2n) * (fma(-y, im, x*re),  fma(x, im, y*re))
//   R_n^m (m < n)  = 1/(n^2-m^2) * fma(-|r|^2, R_{n-2}^m, ((2n-1) z) * R_{n-1}^m)
//   P2M            : M_n^m = fma(q, R_n^m, M_n^m), charges in list order
//   L2P            : total = fma(L_n^0, R_n^0, total) ; row = row + fma(Lre, Rre, Lim*Rim), m
//                    ascending from 0 ; total = total + (row + row), n ascending
// Compiled with -fmad=false: every fused operation below is explicit.
#include <cfloat>

#include "device_math.cuh"
#include "sfmm_internal.hpp"

namespace sfmm {
namespace {

constexpr int kHarmMaxOrder = 32;  // lane = m

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

// R_n^m of one point for m = lane, produced row by row.
template <typename Real>
struct RegularColumn {
    Real x, y, z, r2;
    Real p1re, p1im, p2re, p2im;  // R_{n-1}^m, R_{n-2}^m
    bool zero;                    // |r| effectively zero: R_0^0 = 1 and nothing else

    // inv2n[n] = 1 / (2n), shared by the block
    __device__ void start(Real x_, Real y_, Real z_, int m, const Real* inv2n) {
        x = x_, y = y_, z = z_;
        zero = effectively_zero(x, y, z);
        r2 = fma_(z, z, fma_(x, x, y * y));
        // diagonal up to R_m^m
        Real re = Real(1), im = Real(0);
        for (int n = 1; n <= m; ++n) {
            const Real nre = inv2n[n] * fma_(-y, im, x * re);
            const Real nim = inv2n[n] * fma_(x, im, y * re);
            re = nre;
            im = nim;
        }
        p1re = re, p1im = im;  // consumed by row(m, ...)
        p2re = p2im = Real(0);
    }
    // row n >= m, called with n ascending; denom = 1 / (n^2 - m^2) (unused for n == m)
    __device__ void row(int n, int m, Real denom, Real& re, Real& im) {
        if (n == m) {
            re = p1re;
            im = p1im;
        } else {
            const Real zf = Real(2 * n - 1) * z;
            Real a = zf * p1re, b = zf * p1im;
            if (n - 2 >= m) {
                a = fma_(-r2, p2re, a);
                b = fma_(-r2, p2im, b);
            }
            re = denom * a;
            im = m == 0 ? Real(0) : denom * b;
            p2re = p1re, p2im = p1im;
            p1re = re, p1im = im;
        }
        if (zero) {
            re = (n == 0) ? Real(1) : Real(0);
            im = Real(0);
        }
    }
};

// position of (n, m, part) in the output layouts
__device__ __forceinline__ int64_t out_index(int layout, int64_t b, int n, int m, int part, int order,
                                             int64_t stride) {
    const int c = n * (n + 1) + 2 * m + part;
    if (layout == LAYOUT_SOA) return (int64_t)c * stride + b;
    if (layout == LAYOUT_ROWS) return b * rows_off(order) + rows_off(n) + 2 * m + part;
    return b * ((int64_t)order * (order + 1)) + c;
}

template <typename Real, int NMAX>
__global__ void __launch_bounds__(128)
p2m_kernel(const int64_t* __restrict__ box_ptr, const Real* __restrict__ charges,
           const Real* __restrict__ centers, int64_t n_boxes, int order, int layout,
           Real* __restrict__ out, int64_t stride) {
    __shared__ Real inv2n[kHarmMaxOrder + 1];
    if (threadIdx.x <= kHarmMaxOrder) inv2n[threadIdx.x] = threadIdx.x ? Real(1) / Real(2 * (int)threadIdx.x) : Real(0);
    __syncthreads();
    const int m = threadIdx.x & 31;
    const int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (b >= n_boxes || m >= order) return;
    Real denom[NMAX], are[NMAX], aim[NMAX];
#pragma unroll
    for (int k = 0; k < NMAX; ++k) {
        const int n = m + k;
        denom[k] = k ? Real(1) / Real(n * n - m * m) : Real(0);
        are[k] = aim[k] = Real(0);
    }
    const Real cx = centers[3 * b], cy = centers[3 * b + 1], cz = centers[3 * b + 2];
    for (int64_t j = box_ptr[b]; j < box_ptr[b + 1]; ++j) {
        const Real q = charges[4 * j + 3];
        RegularColumn<Real> col;
        col.start(charges[4 * j] - cx, charges[4 * j + 1] - cy, charges[4 * j + 2] - cz, m, inv2n);
#pragma unroll
        for (int k = 0; k < NMAX; ++k) {
            if (m + k < order) {
                Real re, im;
                col.row(m + k, m, denom[k], re, im);
                are[k] = fma_(q, re, are[k]);
                aim[k] = fma_(q, im, aim[k]);
            }
        }
    }
#pragma unroll
    for (int k = 0; k < NMAX; ++k) {
        const int n = m + k;
        if (n < order) {
            out[out_index(layout, b, n, m, 0, order, stride)] = are[k];
            out[out_index(layout, b, n, m, 1, order, stride)] = aim[k];
        }
    }
    // padding of the rows layout (rows of odd length carry two zeros)
    if (layout == LAYOUT_ROWS && m == 0) {
        for (int n = 0; n < order; ++n)
            for (int k = 2 * (n + 1); k < rows_off(n + 1) - rows_off(n); ++k)
                out[b * rows_off(order) + rows_off(n) + k] = Real(0);
    }
}

// L2P: out[i] = paired_sum(L[box(i)], regular(x_i - centre[box(i)])) (harmonics.cpp:119-152)
template <typename Real>
__global__ void __launch_bounds__(128)
eval_local_kernel(const int32_t* __restrict__ point_box, const Real* __restrict__ points,
                  const Real* __restrict__ centers, int64_t n_points, int64_t n_boxes, int order,
                  int layout, const Real* __restrict__ locals, int64_t stride, Real* __restrict__ out) {
    __shared__ Real inv2n[kHarmMaxOrder + 1];
    if (threadIdx.x <= kHarmMaxOrder) inv2n[threadIdx.x] = threadIdx.x ? Real(1) / Real(2 * (int)threadIdx.x) : Real(0);
    __syncthreads();
    const int m = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= n_points) return;  // whole warps leave together
    const int64_t b = point_box ? (int64_t)point_box[i] : i;
    const bool lane_on = m < order;
    RegularColumn<Real> col;
    col.start(points[3 * i] - centers[3 * b], points[3 * i + 1] - centers[3 * b + 1],
              points[3 * i + 2] - centers[3 * b + 2], lane_on ? m : 0, inv2n);
    Real total = Real(0);
    for (int n = 0; n < order; ++n) {
        Real term = Real(0), lre0 = Real(0), vre0 = Real(0);
        if (lane_on && m <= n) {
            Real vre, vim;
            const Real denom = n > m ? Real(1) / Real(n * n - m * m) : Real(0);
            col.row(n, m, denom, vre, vim);
            const Real lre = locals[out_index(layout, b, n, m, 0, order, stride)];
            const Real lim = locals[out_index(layout, b, n, m, 1, order, stride)];
            term = fma_(lre, vre, lim * vim);
            lre0 = lre, vre0 = vre;
        }
        // ordered sum over m = 1..n on every lane (the lanes stay in lockstep)
        Real rowsum = Real(0);
        for (int k = 1; k <= n; ++k) rowsum = rowsum + __shfl_sync(0xffffffffu, term, k);
        const Real l0 = __shfl_sync(0xffffffffu, lre0, 0), v0 = __shfl_sync(0xffffffffu, vre0, 0);
        total = fma_(l0, v0, total);
        total = total + (rowsum + rowsum);
    }
    if (m == 0) out[i] = total;
}

}  // namespace

template <typename Real>
cudaError_t launch_p2m(const int64_t* box_ptr, const Real* charges, const Real* centers,
                       int64_t n_boxes, int order, int layout, Real* out, int64_t stride,
                       cudaStream_t stream) {
    if (n_boxes <= 0) return cudaSuccess;
    if (order > kHarmMaxOrder) return cudaErrorInvalidValue;
    const unsigned grid = (unsigned)((n_boxes + 3) / 4);
    if (order <= 8)
        p2m_kernel<Real, 8><<<grid, 128, 0, stream>>>(box_ptr, charges, centers, n_boxes, order, layout, out, stride);
    else if (order <= 16)
        p2m_kernel<Real, 16><<<grid, 128, 0, stream>>>(box_ptr, charges, centers, n_boxes, order, layout, out, stride);
    else if (order <= 24)
        p2m_kernel<Real, 24><<<grid, 128, 0, stream>>>(box_ptr, charges, centers, n_boxes, order, layout, out, stride);
    else
        p2m_kernel<Real, 32><<<grid, 128, 0, stream>>>(box_ptr, charges, centers, n_boxes, order, layout, out, stride);
    return cudaGetLastError();
}

template <typename Real>
cudaError_t launch_eval_local(const int32_t* point_box, const Real* points, const Real* centers,
                              int64_t n_points, int64_t n_boxes, int order, int layout,
                              const Real* locals, int64_t stride, Real* out, cudaStream_t stream) {
    if (n_points <= 0) return cudaSuccess;
    if (order > kHarmMaxOrder) return cudaErrorInvalidValue;
    const unsigned grid = (unsigned)((n_points + 3) / 4);
    eval_local_kernel<Real><<<grid, 128, 0, stream>>>(point_box, points, centers, n_points, n_boxes, order,
                                                      layout, locals, stride, out);
    return cudaGetLastError();
}

int harmonics_max_order() { return kHarmMaxOrder; }

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

// Device arithmetic helpers shared by all kernels.
//
// Parity contract: every floating-point operation below
// is either an explicit fma() or an IEEE add/mul/div/sqrt that nvcc must not
// fuse (the translation units are compiled with -fmad=false), so that the
// device reproduces, bit for bit, the arithmetic of the reference library
// built with GCC's `-mfma -ffp-contract=fast`.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdint>

namespace sfmm {

template <typename Real> struct real_traits;
template <> struct real_traits<double> {
    static __host__ __device__ constexpr double min_normal() { return DBL_MIN; }
};
template <> struct real_traits<float> {
    static __host__ __device__ constexpr float min_normal() { return FLT_MIN; }
};

__device__ __forceinline__ double fma_(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float fma_(float a, float b, float c) { return __fmaf_rn(a, b, c); }

// std::hypot as glibc 2.39 evaluates it on x86-64 (the reference's
// geometry.cpp:13-14 calls std::hypot twice). glibc's double version is the
// scaled sqrt plus one correction step below and is NOT correctly rounded, so
// a correctly rounded device hypot would differ in the last bit on ~0.6 % of
// inputs — and a last-bit change of |r| moves a P=20 result by ~1e-11
// (SURVEY §7.1). tests/test_oracle.py pins this routine against libm.
__device__ __forceinline__ double hypot_kernel(double ax, double ay) {
    double h = sqrt(ax * ax + ay * ay);
    double t1, t2;
    if (h <= 2.0 * ay) {
        const double delta = h - ay;
        t1 = ax * (2.0 * delta - ax);
        t2 = (delta - 2.0 * (ax - ay)) * delta;
    } else {
        const double delta = h - ax;
        t1 = 2.0 * delta * (ax - 2.0 * ay);
        t2 = (4.0 * delta - ay) * ay + delta * delta;
    }
    h -= (t1 + t2) / (2.0 * h);
    return h;
}

__device__ __forceinline__ double hypot_ref(double x, double y) {
    if (!isfinite(x) || !isfinite(y)) {
        if (isinf(x) || isinf(y)) return INFINITY;
        return x + y;
    }
    x = fabs(x);
    y = fabs(y);
    double ax = x < y ? y : x;
    double ay = x < y ? x : y;
    const double scale = 0x1p-600, large = 0x1p+511, tiny = 0x1p-459, eps = 0x1p-54;
    if (ax > large) {
        if (ay <= ax * eps) return ax + ay;
        return hypot_kernel(ax * scale, ay * scale) / scale;
    }
    if (ay < tiny) {
        if (ax >= ay / eps) return ax + ay;
        return hypot_kernel(ax / scale, ay / scale) * scale;
    }
    if (ax >= ay / eps) return ax + ay;
    return hypot_kernel(ax, ay);
}

// glibc hypotf: one double-precision sqrt of the exact sum of squares.
__device__ __forceinline__ float hypot_ref(float x, float y) {
    if (!isfinite(x) || !isfinite(y)) {
        if (isinf(x) || isinf(y)) return INFINITY;
        return x + y;
    }
    const double dx = (double)x, dy = (double)y;
    return (float)sqrt(dx * dx + dy * dy);
}

// reference geometry.cpp:11-30 (decompose_angles)
template <typename Real>
struct Angles {
    Real rn, ca, sa, cb, sb;
};

template <typename Real>
__device__ __forceinline__ Angles<Real> decompose_angles(Real x, Real y, Real z) {
    Angles<Real> a;
    const Real h = hypot_ref(x, y);
    a.rn = hypot_ref(h, z);
    if (h == Real(0)) {
        a.ca = Real(1);
        a.sa = Real(0);
    } else {
        a.ca = y / h;
        a.sa = x / h;
    }
    a.cb = z / a.rn;
    a.sb = -h / a.rn;
    return a;
}

// |r| < smallest normal  <=>  the reference throws std::domain_error
// (pipeline.cpp:296-297, norm() = std::hypot(x, y, z)).
template <typename Real>
__device__ __forceinline__ bool shift_is_degenerate(Real x, Real y, Real z) {
    const Real mn = real_traits<Real>::min_normal();
    const Real ax = fabs(x), ay = fabs(y), az = fabs(z);
    const Real mx = fmax(ax, fmax(ay, az));
    if (mx >= mn) return false;
    if (!(mx == mx)) return false;  // NaN shifts are not a domain error in the reference
    return hypot_ref(hypot_ref(x, y), z) < mn;
}

}  // namespace sfmm

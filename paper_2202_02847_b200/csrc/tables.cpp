#include "tables.hpp"

#include <cmath>
#include <cstdlib>

namespace sfmm {

namespace {

template <typename Real>
int finite_faculty_cap() {
    Real f = 1;
    int k = 0;
    while (std::isfinite(f * Real(k + 1))) {
        f *= Real(k + 1);
        ++k;
    }
    return k / 2 + 1;  // largest P with (2P-2)! finite
}

// Signed-index view of the (2c+1)x(2c+1) level-c matrix; out-of-range -> 0.
struct Level {
    int c;
    std::vector<double> v;
    double at(int m, int l) const {
        if (std::abs(m) > c || std::abs(l) > c) return 0.0;
        return v[static_cast<size_t>(m + c) * (2 * c + 1) + (l + c)];
    }
};

// One step of Dehnen's recurrences for the x/z axis-swap matrices
// (paper appendix, "Starting with B_0^{0,0} = 1"; evaluated in the same
// operand order as reference operators.cpp:31-41 so that rows n >= 29, whose
// entries no longer fit 53 bits, round identically).
Level next_level(const Level& b) {
    Level nb;
    nb.c = b.c + 1;
    const int dim = 2 * nb.c + 1;
    nb.v.resize(static_cast<size_t>(dim) * dim);
    for (int m = -nb.c; m <= nb.c; ++m) {
        double* row = &nb.v[static_cast<size_t>(m + nb.c) * dim];
        for (int l = -nb.c; l <= nb.c; ++l) {
            double e;
            if (m == 0)
                e = 0.5 * (b.at(0, l - 1) - b.at(0, l + 1));
            else if (m > 0)
                e = 0.5 * (b.at(m - 1, l - 1) + 2.0 * b.at(m - 1, l) + b.at(m - 1, l + 1));
            else
                e = 0.5 * (b.at(m + 1, l - 1) - 2.0 * b.at(m + 1, l) + b.at(m + 1, l + 1));
            row[l + nb.c] = e;
        }
    }
    return nb;
}

}  // namespace

int max_order_f64() {
    static const int cap = finite_faculty_cap<double>();
    return cap;
}
int max_order_f32() {
    static const int cap = finite_faculty_cap<float>();
    return cap;
}

SwapTables::SwapTables(int order_) : order(order_), f(order_), g(order_) {
    // The reference rebuilds B_n from B_0 for every n (O(P^4)); one sweep that
    // keeps the current level produces the same numbers in O(P^3).
    Level b{0, {1.0}};
    for (int n = 0; n < order; ++n) {
        if (n > 0) b = next_level(b);
        const int rows = n + 1;
        f[n].assign(static_cast<size_t>(rows) * rows, 0.0);
        g[n].assign(static_cast<size_t>(rows) * rows, 0.0);
        // reference operators.hpp:17-26 / operators.cpp:57-64
        for (int m = 0; m <= n; ++m)
            for (int l = 0; l <= n; ++l) {
                const double sgn = (l & 1) ? -1.0 : 1.0;
                const size_t i = static_cast<size_t>(m) * rows + l;
                f[n][i] = (l == 0) ? b.at(0, m) : b.at(l, m) + sgn * b.at(-l, m);
                if (l != 0 && m != 0) g[n][i] = b.at(l, m) - sgn * b.at(-l, m);
            }
    }
}

template <typename Real>
void build_faculties(int order, std::vector<Real>& fac, std::vector<Real>& inv) {
    fac.assign(static_cast<size_t>(2 * order - 1), Real(1));
    for (int k = 1; k < 2 * order - 1; ++k) fac[k] = fac[k - 1] * Real(k);
    inv.resize(order);
    for (int d = 0; d < order; ++d) inv[d] = Real(1) / fac[d];
}
template void build_faculties<double>(int, std::vector<double>&, std::vector<double>&);
template void build_faculties<float>(int, std::vector<float>&, std::vector<float>&);

PackedSide pack_side(const SwapTables& t, bool local_side) {
    PackedSide out;
    out.desc.resize(static_cast<size_t>(t.order) * 4);
    for (int n = 0; n < t.order; ++n) {
        const int rows = n + 1;
        const int cls_size[2] = {n / 2 + 1, (n + 1) / 2};
        for (int which = 0; which < 2; ++which) {  // 0: F, 1: G
            const std::vector<double>& a = which == 0 ? t.f[n] : t.g[n];
            // F couples classes with a+b == n, G with a+b == n+1 (mod 2)
            const int sum_parity = (n + which) & 1;
            for (int rc = 0; rc < 2; ++rc) {
                const int cc = (sum_parity - rc) & 1;
                BlockDesc d{};
                d.offset = static_cast<uint32_t>(out.stream.size());
                d.nrows = static_cast<uint16_t>(cls_size[rc]);
                d.ncols = static_cast<uint16_t>(cls_size[cc]);
                d.row_class = static_cast<uint8_t>(rc);
                d.col_class = static_cast<uint8_t>(cc);
                d.ld = static_cast<uint16_t>(d.nrows + (d.nrows & 1));
                for (int kk = 0; kk < d.ncols; ++kk) {
                    for (int ii = 0; ii < d.nrows; ++ii) {
                        const int i = rc + 2 * ii, k = cc + 2 * kk;
                        const size_t idx = local_side
                                               ? static_cast<size_t>(k) * rows + i
                                               : static_cast<size_t>(i) * rows + k;
                        out.stream.push_back(a[idx]);
                    }
                    if (d.nrows & 1) out.stream.push_back(0.0);
                }
                out.desc[static_cast<size_t>(n) * 4 + which * 2 + rc] = d;
            }
        }
    }
    return out;
}

FragSide pack_frags(const SwapTables& t, bool local_side) {
    FragSide out;
    out.offset.assign(static_cast<size_t>(t.order) * 4 + 1, 0);
    for (int n = 0; n < t.order; ++n) {
        const int rows = n + 1;
        const int cls_size[2] = {n / 2 + 1, (n + 1) / 2};
        for (int which = 0; which < 2; ++which) {
            const std::vector<double>& a = which == 0 ? t.f[n] : t.g[n];
            const int sum_parity = (n + which) & 1;
            for (int rc = 0; rc < 2; ++rc) {
                const int cc = (sum_parity - rc) & 1;
                const int nrows = cls_size[rc], ncols = cls_size[cc];
                const int KB = (ncols + 3) / 4, MB = (nrows + 7) / 8;
                out.offset[static_cast<size_t>(n) * 4 + which * 2 + rc] =
                    static_cast<uint32_t>(out.frags.size() / 32);
                for (int kb = 0; kb < KB; ++kb)
                    for (int mb = 0; mb < MB; ++mb)
                        for (int lane = 0; lane < 32; ++lane) {
                            const int c = lane >> 2;
                            const int ii = 8 * mb + (c >> 1) + 4 * (c & 1);
                            const int kk = 4 * kb + (lane & 3);
                            double v = 0.0;
                            if (ii < nrows && kk < ncols) {
                                const int i = rc + 2 * ii, k = cc + 2 * kk;
                                v = local_side ? a[static_cast<size_t>(k) * rows + i]
                                               : a[static_cast<size_t>(i) * rows + k];
                            }
                            out.frags.push_back(v);
                        }
            }
        }
    }
    out.offset[static_cast<size_t>(t.order) * 4] = static_cast<uint32_t>(out.frags.size() / 32);
    return out;
}

size_t packed_prefix_len(int order) {
    size_t len = 0;
    for (int n = 0; n < order; ++n) {
        const int cls[2] = {n / 2 + 1, (n + 1) / 2};
        for (int which = 0; which < 2; ++which)
            for (int rc = 0; rc < 2; ++rc) {
                const int cc = ((n + which) - rc) & 1;
                len += static_cast<size_t>(cls[rc] + (cls[rc] & 1)) * cls[cc];
            }
    }
    return len;
}

}  // namespace sfmm

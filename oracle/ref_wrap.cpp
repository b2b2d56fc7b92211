// TEST INFRASTRUCTURE — not part of the product.
//
// C-ABI glue around the UNMODIFIED reference library `mpole`, compiled from
// the sources where they lie under /root/reference/proj/core (see
// oracle/Makefile; outputs go to oracle/_ref/ only, nothing is copied).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load the resulting library.
//
// Layout at this boundary: a batch of solids is one contiguous array
// [b][P(P+1)] in the reference's own AoS order (solid.hpp:59-70), shifts are
// [b][3]. Every function converts to `mpole::solid` + `translation_request`
// and calls the reference's public API (pipeline.hpp:30-63).

#include <algorithm>
#include <chrono>
#include <cstring>
#include <exception>
#include <thread>
#include <sstream>
#include <cstdio>
#include <vector>

#include "mpole/mpole.hpp"

namespace {

using namespace mpole;

template <typename Real>
using batch_fn = void (*)(const operator_data<Real>&,
                          std::span<const translation_request<Real>>,
                          workspace<Real>&);

template <typename Real>
batch_fn<Real> pick(int kind) {
    switch (kind) {
        case 0: return &m2l<Real>;
        case 1: return &m2m<Real>;
        default: return &l2l<Real>;
    }
}

solid_kind in_kind(int kind) {
    return kind == 2 ? solid_kind::local : solid_kind::multipole;
}
solid_kind out_kind(int kind) {
    return kind == 1 ? solid_kind::multipole : solid_kind::local;
}

// Build solids for requests [lo, hi) with per-request orders.
template <typename Real>
struct staged {
    std::vector<solid<Real>> src, dst;
    std::vector<translation_request<Real>> req;
};

template <typename Real>
void stage(staged<Real>& s, int kind, long lo, long hi, const int* p_in,
           const int* p_out, int p_in_u, int p_out_u, const Real* in,
           const long* in_off, const Real* shifts) {
    const long n = hi - lo;
    s.src.reserve(n);
    s.dst.reserve(n);
    for (long i = lo; i < hi; ++i) {
        const int pi = p_in ? p_in[i] : p_in_u;
        const int po = p_out ? p_out[i] : p_out_u;
        solid<Real> a(in_kind(kind), pi);
        const long off = in_off ? in_off[i] : i * (long)solid_size(p_in_u);
        std::memcpy(a.data().data(), in + off, solid_size(pi) * sizeof(Real));
        s.src.push_back(std::move(a));
        s.dst.emplace_back(out_kind(kind), po);
    }
    s.req.reserve(n);
    for (long i = lo; i < hi; ++i) {
        const int po = p_out ? p_out[i] : p_out_u;
        s.req.push_back({&s.src[i - lo],
                         {shifts[3 * i], shifts[3 * i + 1], shifts[3 * i + 2]},
                         po,
                         &s.dst[i - lo]});
    }
}

template <typename Real>
int run(int kind, long n, const int* p_in, const int* p_out, int p_in_u,
        int p_out_u, const Real* in, const long* in_off, const Real* shifts,
        Real* out, const long* out_off, int nthreads, int reps,
        double* seconds) {
    try {
        int pmax = std::max(p_in_u, p_out_u);
        for (long i = 0; i < n; ++i) {
            if (p_in) pmax = std::max(pmax, p_in[i]);
            if (p_out) pmax = std::max(pmax, p_out[i]);
        }
        const operator_data<Real> ops(std::max(pmax, 1));
        nthreads = std::max(1, nthreads);
        std::vector<staged<Real>> parts(nthreads);
        std::vector<long> lo(nthreads + 1);
        for (int t = 0; t <= nthreads; ++t) lo[t] = n * t / nthreads;
        for (int t = 0; t < nthreads; ++t)
            stage(parts[t], kind, lo[t], lo[t + 1], p_in, p_out, p_in_u,
                  p_out_u, in, in_off, shifts);
        std::vector<workspace<Real>> ws;
        for (int t = 0; t < nthreads; ++t) ws.emplace_back(std::max(pmax, 1));
        const auto fn = pick<Real>(kind);

        double best = 1e300;
        std::vector<std::exception_ptr> errs(nthreads);
        for (int r = 0; r < std::max(1, reps); ++r) {
            const auto t0 = std::chrono::steady_clock::now();
            if (nthreads == 1) {
                fn(ops, parts[0].req, ws[0]);
            } else {
                std::vector<std::thread> th;
                for (int t = 0; t < nthreads; ++t)
                    th.emplace_back([&, t] {
                        try {
                            fn(ops, parts[t].req, ws[t]);
                        } catch (...) {
                            errs[t] = std::current_exception();
                        }
                    });
                for (auto& x : th) x.join();
                for (auto& e : errs)
                    if (e) std::rethrow_exception(e);
            }
            const auto t1 = std::chrono::steady_clock::now();
            best = std::min(best,
                            std::chrono::duration<double>(t1 - t0).count());
        }
        if (seconds) *seconds = best;
        for (int t = 0; t < nthreads; ++t)
            for (long i = lo[t]; i < lo[t + 1]; ++i) {
                const auto& d = parts[t].dst[i - lo[t]];
                const long off =
                    out_off ? out_off[i] : i * (long)solid_size(p_out_u);
                std::memcpy(out + off, d.data().data(),
                            d.data().size() * sizeof(Real));
            }
        return 0;
    } catch (const std::domain_error&) {
        return 2;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (...) {
        return 3;
    }
}

}  // namespace

extern "C" {

// kind: 0 = m2l, 1 = m2m, 2 = l2l. Uniform orders. Returns 0 ok,
// 1 invalid_argument, 2 domain_error. `seconds` (optional) receives the best
// wall time of `reps` calls of the reference batch API, staging excluded.
int ref_translate_f64(int kind, long n, int p_in, int p_out, const double* in,
                      const double* shifts, double* out, int nthreads, int reps,
                      double* seconds) {
    return run<double>(kind, n, nullptr, nullptr, p_in, p_out, in, nullptr,
                       shifts, out, nullptr, nthreads, reps, seconds);
}
int ref_translate_f32(int kind, long n, int p_in, int p_out, const float* in,
                      const float* shifts, float* out, int nthreads, int reps,
                      double* seconds) {
    return run<float>(kind, n, nullptr, nullptr, p_in, p_out, in, nullptr,
                      shifts, out, nullptr, nthreads, reps, seconds);
}

// Mixed orders: one batch call with per-request orders; solids are ragged,
// located by element offsets.
int ref_translate_mixed_f64(int kind, long n, const int* p_in, const int* p_out,
                            const double* in, const long* in_off,
                            const double* shifts, double* out,
                            const long* out_off) {
    return run<double>(kind, n, p_in, p_out, 0, 0, in, in_off, shifts, out,
                       out_off, 1, 1, nullptr);
}
int ref_translate_mixed_f32(int kind, long n, const int* p_in, const int* p_out,
                            const float* in, const long* in_off,
                            const float* shifts, float* out,
                            const long* out_off) {
    return run<float>(kind, n, p_in, p_out, 0, 0, in, in_off, shifts, out,
                      out_off, 1, 1, nullptr);
}

int ref_m2l_naive_f64(long n, int p_in, int p_out, const double* in,
                      const double* shifts, double* out) {
    try {
        for (long i = 0; i < n; ++i) {
            solid<double> m(solid_kind::multipole, p_in);
            std::memcpy(m.data().data(), in + i * solid_size(p_in),
                        solid_size(p_in) * sizeof(double));
            const auto l = m2l_naive<double>(
                m, {shifts[3 * i], shifts[3 * i + 1], shifts[3 * i + 2]}, p_out);
            std::memcpy(out + i * solid_size(p_out), l.data().data(),
                        solid_size(p_out) * sizeof(double));
        }
        return 0;
    } catch (const std::domain_error&) {
        return 2;
    } catch (...) {
        return 3;
    }
}

// charges: [count][4] = x y z q. out: P(P+1).
void ref_p2m_f64(int count, const double* charges, const double* center,
                 int order, double* out) {
    std::vector<point_charge<double>> c(count);
    for (int i = 0; i < count; ++i)
        c[i] = {{charges[4 * i], charges[4 * i + 1], charges[4 * i + 2]},
                charges[4 * i + 3]};
    const auto m =
        p2m<double>(c, {center[0], center[1], center[2]}, order);
    std::memcpy(out, m.data().data(), solid_size(order) * sizeof(double));
}

void ref_regular_f64(int order, const double* r, double* out) {
    const auto s = regular<double>(order, {r[0], r[1], r[2]});
    std::memcpy(out, s.data().data(), solid_size(order) * sizeof(double));
}
int ref_singular_f64(int order, const double* r, double* out) {
    try {
        const auto s = singular<double>(order, {r[0], r[1], r[2]});
        std::memcpy(out, s.data().data(), solid_size(order) * sizeof(double));
        return 0;
    } catch (const std::domain_error&) {
        return 2;
    }
}
double ref_eval_local_f64(int order, const double* l, const double* center,
                          const double* x) {
    solid<double> s(solid_kind::local, order);
    std::memcpy(s.data().data(), l, solid_size(order) * sizeof(double));
    return eval_local<double>(s, {center[0], center[1], center[2]},
                              {x[0], x[1], x[2]});
}

// text format (io.hpp): write one solid / read concatenated solids through the reference
long ref_write_solid_f64(int kind, int order, const double* data, char* buf, long cap) {
    solid<double> s(static_cast<solid_kind>(kind), order);
    std::memcpy(s.data().data(), data, solid_size(order) * sizeof(double));
    std::ostringstream os;
    write_solid<double>(os, s);
    const std::string t = os.str();
    if ((long)t.size() < cap) std::memcpy(buf, t.c_str(), t.size() + 1);
    return (long)t.size();
}
// returns the number of solids (kinds / orders / concatenated data filled), or -1 with the
// exception text in err
int ref_read_solids_f64(const char* text, int max_solids, int* kinds, int* orders, double* data,
                        long cap, char* err, int errcap) {
    try {
        std::istringstream is(text);
        const auto v = read_solids<double>(is);
        long pos = 0;
        int n = 0;
        for (const auto& s : v) {
            if (n >= max_solids || pos + (long)s.data().size() > cap) break;
            kinds[n] = static_cast<int>(s.kind());
            orders[n] = s.order();
            std::memcpy(data + pos, s.data().data(), s.data().size() * sizeof(double));
            pos += (long)s.data().size();
            ++n;
        }
        return n;
    } catch (const std::exception& e) {
        std::snprintf(err, errcap, "%s", e.what());
        return -1;
    }
}

// single-precision forms of the three harmonics entry points
void ref_p2m_f32(int count, const float* charges, const float* center, int order, float* out) {
    std::vector<point_charge<float>> c(count);
    for (int i = 0; i < count; ++i)
        c[i] = {{charges[4 * i], charges[4 * i + 1], charges[4 * i + 2]}, charges[4 * i + 3]};
    const auto m = p2m<float>(c, {center[0], center[1], center[2]}, order);
    std::memcpy(out, m.data().data(), solid_size(order) * sizeof(float));
}
void ref_regular_f32(int order, const float* r, float* out) {
    const auto s = regular<float>(order, {r[0], r[1], r[2]});
    std::memcpy(out, s.data().data(), solid_size(order) * sizeof(float));
}
float ref_eval_local_f32(int order, const float* l, const float* center, const float* x) {
    solid<float> s(solid_kind::local, order);
    std::memcpy(s.data().data(), l, solid_size(order) * sizeof(float));
    return eval_local<float>(s, {center[0], center[1], center[2]}, {x[0], x[1], x[2]});
}

// b: (2n+1)^2, f and g: (n+1)^2 each, all row-major double.
void ref_swap_tables(int n, double* b, double* f, double* g) {
    const auto bb = wigner_b(n);
    const auto fg = swap_matrices(n, bb);
    if (b) std::copy(bb.begin(), bb.end(), b);
    if (f) std::copy(fg.f.begin(), fg.f.end(), f);
    if (g) std::copy(fg.g.begin(), fg.g.end(), g);
}

// fac: 2P-1 entries, inv: P entries, in the library precision.
int ref_faculties_f64(int order, double* fac, double* inv) {
    try {
        const operator_data<double> ops(order);
        std::copy(ops.faculties().begin(), ops.faculties().end(), fac);
        std::copy(ops.inv_faculties().begin(), ops.inv_faculties().end(), inv);
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    }
}
int ref_faculties_f32(int order, float* fac, float* inv) {
    try {
        const operator_data<float> ops(order);
        std::copy(ops.faculties().begin(), ops.faculties().end(), fac);
        std::copy(ops.inv_faculties().begin(), ops.inv_faculties().end(), inv);
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    }
}
int ref_max_order_f64() { return operator_data<double>::max_order(); }
int ref_max_order_f32() { return operator_data<float>::max_order(); }

// out5 = r_norm, cos_alpha, sin_alpha, cos_beta, sin_beta.
int ref_angles_f64(const double* r, double* out5) {
    try {
        const auto a = detail::decompose_angles<double>({r[0], r[1], r[2]});
        out5[0] = a.r_norm;
        out5[1] = a.cos_alpha;
        out5[2] = a.sin_alpha;
        out5[3] = a.cos_beta;
        out5[4] = a.sin_beta;
        return 0;
    } catch (const std::domain_error&) {
        return 2;
    }
}
int ref_angles_f32(const float* r, float* out5) {
    try {
        const auto a = detail::decompose_angles<float>({r[0], r[1], r[2]});
        out5[0] = a.r_norm;
        out5[1] = a.cos_alpha;
        out5[2] = a.sin_alpha;
        out5[3] = a.cos_beta;
        out5[4] = a.sin_beta;
        return 0;
    } catch (const std::domain_error&) {
        return 2;
    }
}

int ref_hardware_threads() {
    return (int)std::max(1u, std::thread::hardware_concurrency());
}

}  // extern "C"

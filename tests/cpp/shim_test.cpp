// GPU test of the C++ drop-in header (include/mpole_b200.hpp). The cases are
// the reference's own pipeline tests (reference tests/test_pipeline.cpp:59-368)
// re-expressed as plain checks (doctest is not available), run against the CUDA
// library and checked with the CPU oracle (oracle/liboracle.so).
// Build + run: tests/test_cpp_shim.py.
#include <cmath>
#include <cstdio>
#include <random>
#include <thread>
#include <vector>

#include "mpole_b200.hpp"

extern "C" {
int orc_m2l_naive_f64(long n, int p_in, int p_out, const double* in, const double* shifts, double* out);
int orc_translate_f64(int kind, long n, int p_in, int p_out, const double* in, const double* shifts, double* out);
void orc_p2m_f64(int count, const double* charges, const double* center, int order, double* out);
void orc_p2m_fma_f64(int count, const double* charges, const double* center, int order, double* out);
double orc_eval_local_fma_f64(int order, const double* l, const double* center, const double* x);
}

using namespace mpole_b200;

static int failures = 0;
#define CHECK(cond)                                                          \
    do {                                                                     \
        if (!(cond)) {                                                       \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);     \
            ++failures;                                                      \
        }                                                                    \
    } while (0)
template <typename E, typename F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static std::mt19937_64 rng(0x8d1f2c3b);

static solid<double> random_solid(int order, solid_kind kind = solid_kind::multipole) {
    std::normal_distribution<double> nd;
    solid<double> s(kind, order);
    for (int n = 0; n < order; ++n)
        for (int m = 0; m <= n; ++m) s.set(n, m, {nd(rng), m == 0 ? 0.0 : nd(rng)});
    return s;
}
static vec3<double> random_shift() {
    std::normal_distribution<double> nd;
    std::uniform_real_distribution<double> ud(0.5, 2.0);
    vec3<double> r{nd(rng), nd(rng), nd(rng)};
    const double n = norm(r), want = ud(rng);
    return {r.x / n * want, r.y / n * want, r.z / n * want};
}
static double normalized_error(const solid<double>& a, const solid<double>& b) {
    double scale = 0, diff = 0;
    if (a.data().size() != b.data().size()) return 1e300;
    for (std::size_t i = 0; i < a.data().size(); ++i) {
        scale = std::max(scale, std::abs(b.data()[i]));
        diff = std::max(diff, std::abs(a.data()[i] - b.data()[i]));
    }
    return diff / std::max(scale, 1e-300);
}
static solid<double> naive(const solid<double>& m, const vec3<double>& r, int p_out) {
    solid<double> out(solid_kind::local, p_out);
    const double sh[3] = {r.x, r.y, r.z};
    orc_m2l_naive_f64(1, m.order(), p_out, m.data().data(), sh, out.data().data());
    return out;
}
static solid<double> oracle(int kind, const solid<double>& s, const vec3<double>& r, int p_out) {
    solid<double> out(kind == 1 ? solid_kind::multipole : solid_kind::local, p_out);
    const double sh[3] = {r.x, r.y, r.z};
    orc_translate_f64(kind, 1, s.order(), p_out, s.data().data(), sh, out.data().data());
    return out;
}

int main() {
    // m2l: unit source along the z axis (test_pipeline.cpp:59-74)
    {
        const operator_data<double> ops(8);
        workspace<double> ws(8);
        solid<double> m(solid_kind::multipole, 3);
        m.re(0, 0) = 1.0;
        const auto l = m2l(ops, m, {0.0, 0.0, 2.0}, 3, ws);
        CHECK(l.kind() == solid_kind::local);
        CHECK(std::abs(l.re(0, 0) - 0.5) < 1e-14);
        CHECK(std::abs(l.re(1, 0) + 0.25) < 1e-14);
        CHECK(std::abs(l.re(2, 0) - 0.25) < 1e-14);
        for (int n = 0; n < 3; ++n)
            for (int mm = 1; mm <= n; ++mm) CHECK(l.re(n, mm) == 0.0 && l.im(n, mm) == 0.0);
    }
    // m2l matches the naive kernel, mixed orders and axis shifts (:88-114)
    {
        const operator_data<double> ops(14);
        workspace<double> ws(14);
        double worst = 0;
        for (int trial = 0; trial < 40; ++trial) {
            const int p_in = 1 + (int)(rng() % 14), p_out = 1 + (int)(rng() % 14);
            const auto m = random_solid(p_in);
            const auto r = random_shift();
            const auto got = m2l(ops, m, r, p_out, ws);
            worst = std::max(worst, normalized_error(got, naive(m, r, p_out)));
            CHECK(got == oracle(0, m, r, p_out));  // bit-identical to the CPU path
        }
        CHECK(worst < 1e-12);
        for (const vec3<double> r : {vec3<double>{0, 0, -1.5}, {2.0, 0, 0}, {-2.0, 0, 0}, {0, 1.5, 0}, {0, -1.5, 0}}) {
            const auto m = random_solid(8);
            CHECK(normalized_error(m2l(ops, m, r, 8, ws), naive(m, r, 8)) < 1e-12);
        }
    }
    // batch processing equals one-by-one processing (:136-163)
    {
        const operator_data<double> ops(10);
        workspace<double> ws(10);
        const int count = 19;
        std::vector<solid<double>> sources;
        std::vector<vec3<double>> shifts;
        std::vector<int> orders;
        for (int i = 0; i < count; ++i) {
            sources.push_back(random_solid(1 + (int)(rng() % 10)));
            shifts.push_back(random_shift());
            orders.push_back(1 + (int)(rng() % 10));
        }
        std::vector<solid<double>> out(count, solid<double>(solid_kind::local, 1));
        std::vector<translation_request<double>> reqs;
        for (int i = 0; i < count; ++i) reqs.push_back({&sources[i], shifts[i], orders[i], &out[i]});
        m2l<double>(ops, reqs, ws);
        for (int i = 0; i < count; ++i) {
            CHECK(out[i].order() == orders[i]);
            CHECK(out[i] == m2l(ops, sources[i], shifts[i], orders[i], ws));
        }
    }
    // m2m agrees with rebuilding the expansion at the new centre (:165-178)
    {
        const operator_data<double> ops(10);
        workspace<double> ws(10);
        std::uniform_real_distribution<double> ud(-1.0, 1.0);
        std::vector<double> charges;
        const double a[3] = {0.1, -0.2, 0.3}, b[3] = {1.0, 0.5, -0.7};
        for (int i = 0; i < 6; ++i) {
            for (int d = 0; d < 3; ++d) charges.push_back(a[d] + 0.2 * ud(rng));
            charges.push_back(ud(rng));
        }
        solid<double> ma(solid_kind::multipole, 10), mb(solid_kind::multipole, 10);
        orc_p2m_f64(6, charges.data(), a, 10, ma.data().data());
        orc_p2m_f64(6, charges.data(), b, 10, mb.data().data());
        const auto got = m2m(ops, ma, {b[0] - a[0], b[1] - a[1], b[2] - a[2]}, 10, ws);
        CHECK(got.kind() == solid_kind::multipole);
        CHECK(normalized_error(got, mb) < 1e-12);
    }
    // m2m round trip, order raise = zero extension, lowering = truncation (:180-206)
    {
        const operator_data<double> ops(10);
        workspace<double> ws(10);
        const auto m = random_solid(7);
        const vec3<double> r{0.8, -0.5, 0.6};
        const auto there = m2m(ops, m, r, 7, ws);
        CHECK(normalized_error(m2m(ops, there, {-r.x, -r.y, -r.z}, 7, ws), m) < 1e-12);
        solid<double> ext(solid_kind::multipole, 10);
        std::copy(m.data().begin(), m.data().end(), ext.data().begin());
        CHECK(normalized_error(m2m(ops, m, r, 10, ws), m2m(ops, ext, r, 10, ws)) < 1e-14);
        const auto lowered = m2m(ops, m, r, 4, ws), full = m2m(ops, m, r, 7, ws);
        for (int n = 0; n < 4; ++n)
            for (int mm = 0; mm <= n; ++mm)
                CHECK(std::abs(lowered.re(n, mm) - full.re(n, mm)) <= 1e-14 * std::abs(full.re(n, mm)) + 1e-300);
    }
    // l2l round trip (:208-233)
    {
        const operator_data<double> ops(10);
        workspace<double> ws(10);
        const auto m = random_solid(10);
        const auto l = naive(m, {4.0, 3.0, 3.5}, 10);
        const vec3<double> shift{0.3, -0.2, 0.25};
        const auto moved = l2l(ops, l, shift, 10, ws);
        CHECK(normalized_error(l2l(ops, moved, {-shift.x, -shift.y, -shift.z}, 10, ws), l) < 1e-12);
        CHECK(moved == oracle(2, l, shift, 10));
    }
    // in-place recentring, also with an order change (:259-279)
    {
        const operator_data<double> ops(8);
        workspace<double> ws(8);
        auto m = random_solid(8);
        const auto reference = m;
        const vec3<double> r{0.4, 0.3, -0.5};
        const auto want = m2m(ops, m, r, 8, ws);
        translation_request<double> req{&m, r, 8, &m};
        m2m(ops, std::span<const translation_request<double>>(&req, 1), ws);
        CHECK(m == want);
        auto m2 = reference;
        const auto want2 = m2m(ops, m2, r, 5, ws);
        translation_request<double> req2{&m2, r, 5, &m2};
        m2m(ops, std::span<const translation_request<double>>(&req2, 1), ws);
        CHECK(m2.order() == 5);
        CHECK(m2 == want2);
    }
    // error contracts (:281-306 and test_operators.cpp:197-216)
    {
        const operator_data<double> ops(6);
        workspace<double> ws(6);
        const auto m = random_solid(6);
        CHECK(throws<std::domain_error>([&] { m2l(ops, m, {0.0, 0.0, 0.0}, 6, ws); }));
        CHECK(throws<std::domain_error>([&] { m2m(ops, m, {0.0, 0.0, 0.0}, 6, ws); }));
        CHECK(throws<std::invalid_argument>([&] { m2l(ops, m, {1.0, 0.0, 0.0}, 7, ws); }));
        workspace<double> small(4);
        CHECK(throws<std::invalid_argument>([&] { m2l(ops, m, {1.0, 0.0, 0.0}, 4, small); }));
        workspace<double> other(6, kernel_config{2, 4});
        CHECK(throws<std::invalid_argument>([&] { m2l(ops, m, {1.0, 0.0, 0.0}, 6, other); }));
        solid<double> out(solid_kind::local, 6);
        translation_request<double> null_src{nullptr, {1, 0, 0}, 6, &out};
        CHECK(throws<std::invalid_argument>(
            [&] { m2l(ops, std::span<const translation_request<double>>(&null_src, 1), ws); }));
        CHECK(operator_data<double>::max_order() == 86);
        CHECK(operator_data<float>::max_order() == 18);
        CHECK(throws<std::invalid_argument>([] { operator_data<double> bad(87); }));
        CHECK(throws<std::invalid_argument>([] { operator_data<float> bad(19); }));
        CHECK(throws<std::invalid_argument>([] { operator_data<double> bad(0); }));
        // a failed batch leaves every output untouched
        solid<double> o1(solid_kind::local, 6), o2(solid_kind::local, 6);
        o1.re(0, 0) = 42.0;
        std::vector<translation_request<double>> reqs{{&m, {1, 0, 0}, 6, &o1}, {&m, {0, 0, 0}, 6, &o2}};
        CHECK(throws<std::domain_error>([&] { m2l<double>(ops, reqs, ws); }));
        CHECK(o1.re(0, 0) == 42.0);
        // validation is per request, in order (pipeline.cpp:282-298): the zero shift of request
        // 0 is reported, not the bad order of request 1 ... and the other way round
        std::vector<translation_request<double>> mixed{{&m, {0, 0, 0}, 6, &o1}, {&m, {1, 0, 0}, 7, &o2}};
        CHECK(throws<std::domain_error>([&] { m2l<double>(ops, mixed, ws); }));
        std::vector<translation_request<double>> mixed2{{&m, {1, 0, 0}, 7, &o1}, {&m, {0, 0, 0}, 6, &o2}};
        CHECK(throws<std::invalid_argument>([&] { m2l<double>(ops, mixed2, ws); }));
        CHECK(o1.re(0, 0) == 42.0);
    }
    // single precision (:320-335)
    {
        const operator_data<float> ops(8);
        workspace<float> ws(8);
        const auto md = random_solid(8);
        solid<float> mf(solid_kind::multipole, 8);
        for (std::size_t i = 0; i < mf.data().size(); ++i) mf.data()[i] = (float)md.data()[i];
        const auto got = m2l(ops, mf, vec3<float>{1.2f, -0.7f, 0.9f}, 8, ws);
        const auto want = naive(md, {1.2f, -0.7f, 0.9f}, 8);
        solid<double> gd(solid_kind::local, 8);
        for (std::size_t i = 0; i < gd.data().size(); ++i) gd.data()[i] = got.data()[i];
        CHECK(normalized_error(gd, want) < 1e-4);
    }
    // concurrent translations with a shared operator table (:337-368)
    {
        const auto ops = operator_data<double>::acquire(9);
        CHECK(ops.get() == operator_data<double>::acquire(9).get());
        const int count = 24;
        std::vector<solid<double>> sources;
        std::vector<vec3<double>> shifts;
        for (int i = 0; i < count; ++i) {
            sources.push_back(random_solid(9));
            shifts.push_back(random_shift());
        }
        workspace<double> ws(9);
        std::vector<solid<double>> want;
        for (int i = 0; i < count; ++i) want.push_back(m2l(*ops, sources[i], shifts[i], 9, ws));
        std::vector<std::thread> threads;
        std::vector<int> bad(4, 0);
        for (int t = 0; t < 4; ++t)
            threads.emplace_back([&, t] {
                workspace<double> local_ws(9);
                for (int i = 0; i < count; ++i)
                    if (!(m2l(*ops, sources[i], shifts[i], 9, local_ws) == want[i])) ++bad[t];
            });
        for (auto& th : threads) th.join();
        for (int t = 0; t < 4; ++t) CHECK(bad[t] == 0);
    }
    // p2m / eval_local on the device behind the reference's signatures (harmonics.hpp:36-51;
    // field preservation as in test_pipeline.cpp:208-233)
    {
        const operator_data<double> ops(12);
        workspace<double> ws(12);
        std::uniform_real_distribution<double> ud(-0.5, 0.5);
        std::vector<point_charge<double>> q(23);
        for (auto& c : q) c = {{ud(rng), ud(rng), ud(rng)}, ud(rng) < 0 ? -1.0 : 1.0};
        const vec3<double> centre{0.1, -0.2, 0.05};
        const auto m = p2m<double>(ops, q, centre, 12);
        solid<double> want(solid_kind::multipole, 12);
        const double c3[3] = {centre.x, centre.y, centre.z};
        orc_p2m_fma_f64((int)q.size(), &q[0].position.x, c3, 12, want.data().data());
        CHECK(m.kind() == solid_kind::multipole && m == want);
        const vec3<double> shift{3.0, -2.5, 4.0};
        const auto l = m2l(ops, m, shift, 12, ws);
        const vec3<double> lc = centre + shift, x{lc.x + 0.2, lc.y - 0.1, lc.z + 0.15};
        const double phi = eval_local<double>(ops, l, lc, x);
        const double lc3[3] = {lc.x, lc.y, lc.z}, x3[3] = {x.x, x.y, x.z};
        CHECK(phi == orc_eval_local_fma_f64(12, l.data().data(), lc3, x3));
        double direct = 0;
        for (const auto& c : q) direct += c.charge / norm(x - c.position);
        CHECK(std::abs(phi - direct) < 1e-7 * std::abs(direct) + 1e-9);
        // batched forms
        const std::int64_t ptr[4] = {0, 5, 5, 23};
        const vec3<double> cs[3] = {centre, {1, 1, 1}, {-1, 0, 2}};
        const auto ms = p2m<double>(ops, q, ptr, cs, 7);
        CHECK(ms.size() == 3);
        for (auto v : ms[1].data()) CHECK(v == 0.0);
        bool threw = false;
        try {
            p2m<double>(ops, q, centre, 13);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "ALL PASSED", failures);
    return failures ? 1 : 0;
}

// Text format of include/mpole_b200.hpp against the reference's io.cpp (through the
// extern "C" wrappers of oracle/_ref/libmpole_ref.so): files written by either side read back
// bit for bit on the other, and malformed input raises the reference's messages
// (test_io.cpp cases re-expressed without doctest). CPU only.
#include <cstdio>
#include <cstring>
#include <random>
#include <sstream>

#include "mpole_b200.hpp"

extern "C" {
long ref_write_solid_f64(int kind, int order, const double* data, char* buf, long cap);
int ref_read_solids_f64(const char* text, int max_solids, int* kinds, int* orders, double* data, long cap, char* err,
                        int errcap);
}
using namespace mpole_b200;

static int failures = 0;
#define CHECK(c)                                                        \
    do {                                                                \
        if (!(c)) {                                                     \
            std::printf("FAILED %s:%d: %s\n", __FILE__, __LINE__, #c);  \
            ++failures;                                                 \
        }                                                               \
    } while (0)

static std::string error_of(const std::string& text) {
    std::istringstream is(text);
    try {
        read_solids<double>(is);
    } catch (const std::runtime_error& e) {
        return e.what();
    }
    return "";
}
static std::string ref_error_of(const std::string& text) {
    int k[4], o[4];
    double d[256];
    char err[256] = "";
    const int n = ref_read_solids_f64(text.c_str(), 4, k, o, d, 256, err, sizeof err);
    return n < 0 ? err : "";
}

int main() {
    std::mt19937_64 rng(5);
    std::normal_distribution<double> nd;
    // identical files, and each side reads the other's
    for (int order : {1, 2, 7, 20}) {
        for (int kind = 0; kind < 4; ++kind) {
            solid<double> s(static_cast<solid_kind>(kind), order);
            for (auto& v : s.data()) v = nd(rng) * std::pow(10.0, (int)(rng() % 40) - 20);
            for (int n = 0; n < order; ++n) s.im(n, 0) = 0.0;
            std::ostringstream os;
            write_solid(os, s);
            std::vector<char> buf(64 * solid_size(order) + 64);
            const long len = ref_write_solid_f64(kind, order, s.data().data(), buf.data(), (long)buf.size());
            CHECK(len > 0 && os.str() == std::string(buf.data()));
            std::istringstream is(std::string(buf.data()) + os.str());
            const auto back = read_solids<double>(is);
            CHECK(back.size() == 2 && back[0] == s && back[1] == s);
            int k[2], o[2];
            std::vector<double> d(2 * solid_size(order));
            char err[128];
            const int n = ref_read_solids_f64((os.str() + os.str()).c_str(), 2, k, o, d.data(), (long)d.size(), err, 128);
            CHECK(n == 2 && k[0] == kind && o[1] == order);
            CHECK(std::memcmp(d.data(), s.data().data(), solid_size(order) * 8) == 0);
        }
    }
    // free-form whitespace, end of input, float precision
    {
        std::istringstream is("  \n\nSOLID L 2\n1 0 2\n 0   3 4\n\n");
        const auto s = read_solid<double>(is);
        CHECK(s && s->kind() == solid_kind::local && s->order() == 2 && s->re(1, 1) == 3.0 && s->im(1, 1) == 4.0);
        CHECK(!read_solid<double>(is));
        solid<float> f(solid_kind::multipole, 3);
        for (auto& v : f.data()) v = (float)nd(rng);
        std::ostringstream os;
        write_solid(os, f);
        std::istringstream back(os.str());
        CHECK(*read_solid<float>(back) == f);
    }
    // malformed input: same messages as the reference
    for (const char* text : {"SOLD M 2\n", "SOLID X 2\n", "SOLID MM 2\n", "SOLID M two\n", "SOLID M 0\n", "SOLID M 2\n1 0 2\n",
                             "SOLID M 1\n1 zero\n", "SOLID L 2\n1 0\n2 0 3 4\nSOLID M 1\n1 x\n", "SOLID M"}) {
        const std::string a = error_of(text), b = ref_error_of(text);
        if (a != b) std::printf("  input '%s': '%s' vs reference '%s'\n", text, a.c_str(), b.c_str());
        CHECK(!a.empty() && a == b);
    }
    // charges
    {
        std::istringstream is("# comment\n\n1 2 3 -1\n  0.5 0.25 0.125 2e-3\n");
        const auto c = read_charges<double>(is);
        CHECK(c.size() == 2 && c[0].charge == -1.0 && c[1].position.z == 0.125 && c[1].charge == 2e-3);
        std::ostringstream os;
        write_charges<double>(os, c);
        std::istringstream again(os.str());
        const auto d = read_charges<double>(again);
        CHECK(d.size() == 2 && d[1].position.x == 0.5 && d[1].charge == 2e-3);
        for (const char* bad : {"1 2 3\n", "1 2 3 4 5\n", "a b c d\n"}) {
            std::istringstream b(bad);
            bool threw = false;
            try {
                read_charges<double>(b);
            } catch (const std::runtime_error& e) {
                threw = std::string(e.what()).rfind("line 1: ", 0) == 0;
            }
            CHECK(threw);
        }
    }
    if (failures == 0) std::printf("ALL PASSED\n");
    return failures ? 1 : 0;
}

// Header-only C++ mirror of the reference's translation API on top of the C ABI
// (solidfmm_b200.h). A caller of the reference library `mpole` switches the
// namespace and links libsolidfmm_b200.so; names, argument meaning and error
// behaviour follow the reference (paths relative to /root/reference/proj/core):
//
//   vec3, solid, solid_kind, index_re/index_im/solid_size   include/mpole/solid.hpp:13-139
//   translation_request                                      include/mpole/pipeline.hpp:15-21
//   operator_data (order, max_order, acquire)                include/mpole/operators.hpp:57-95
//   workspace                                                include/mpole/workspace.hpp:18-51
//   m2l / m2m / l2l, batched and single-request              include/mpole/pipeline.hpp:30-56
//   point_charge, p2m, eval_local (device P2M / L2P)         include/mpole/harmonics.hpp:10-51
//   write_solid / read_solid(s) / read_charges / write_charges   include/mpole/io.hpp:12-34
//
// Differences that follow from running on a device: operator_data owns the
// device handle (tables + scratch), so `workspace` is a plain tag object kept
// for source compatibility (its order/config checks are reproduced); the
// reference's CPU blocking parameters (mu, nu) are validated and otherwise
// ignored. Exceptions: std::invalid_argument / std::domain_error exactly where
// the reference throws them (pipeline.cpp:282-298), std::runtime_error for CUDA
// failures.
#pragma once

#include <algorithm>
#include <cassert>
#include <cmath>
#include <complex>
#include <cstddef>
#include <cstdint>
#include <istream>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <ostream>
#include <sstream>
#include <span>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "solidfmm_b200.h"

namespace mpole_b200 {

template <typename Real>
struct vec3 {
    Real x, y, z;
};
template <typename Real>
inline Real norm(const vec3<Real>& v) { return std::hypot(v.x, v.y, v.z); }
template <typename Real>
inline vec3<Real> operator-(const vec3<Real>& a, const vec3<Real>& b) {
    return {a.x - b.x, a.y - b.y, a.z - b.z};
}
template <typename Real>
inline vec3<Real> operator+(const vec3<Real>& a, const vec3<Real>& b) {
    return {a.x + b.x, a.y + b.y, a.z + b.z};
}

enum class solid_kind { multipole, local, regular, singular };

constexpr std::size_t index_re(int n, int m) noexcept {
    return static_cast<std::size_t>(n) * static_cast<std::size_t>(n + 1) + 2 * static_cast<std::size_t>(m);
}
constexpr std::size_t index_im(int n, int m) noexcept { return index_re(n, m) + 1; }
constexpr std::size_t solid_size(int order) noexcept {
    return static_cast<std::size_t>(order) * static_cast<std::size_t>(order + 1);
}

/// Triangular array of P(P+1) reals, same layout and accessors as mpole::solid.
template <typename Real>
class solid {
public:
    using value_type = Real;
    solid(solid_kind kind, int order) : kind_(kind), order_(order), data_(solid_size(order), Real(0)) {
        assert(order >= 1);
    }
    solid_kind kind() const noexcept { return kind_; }
    void set_kind(solid_kind k) noexcept { kind_ = k; }
    int order() const noexcept { return order_; }
    Real re(int n, int m) const { return data_[index_re(n, m)]; }
    Real im(int n, int m) const { return data_[index_im(n, m)]; }
    Real& re(int n, int m) { return data_[index_re(n, m)]; }
    Real& im(int n, int m) { return data_[index_im(n, m)]; }
    std::complex<Real> coeff(int n, int m) const {
        if (m >= 0) return {data_[index_re(n, m)], data_[index_im(n, m)]};
        const Real sign = (m & 1) ? Real(-1) : Real(1);
        return {sign * data_[index_re(n, -m)], -sign * data_[index_im(n, -m)]};
    }
    void set(int n, int m, std::complex<Real> v) {
        data_[index_re(n, m)] = v.real();
        data_[index_im(n, m)] = (m == 0) ? Real(0) : v.imag();
    }
    std::span<Real> data() noexcept { return data_; }
    std::span<const Real> data() const noexcept { return data_; }
    friend bool operator==(const solid& a, const solid& b) {
        return a.kind_ == b.kind_ && a.order_ == b.order_ && a.data_ == b.data_;
    }

private:
    solid_kind kind_;
    int order_;
    std::vector<Real> data_;
};

struct kernel_config {
    int mu;
    int nu;
    friend bool operator==(const kernel_config&, const kernel_config&) = default;
};
template <typename Real>
inline kernel_config default_kernel_config() noexcept {
    return {6, sizeof(Real) == 8 ? 8 : 16};
}

namespace detail {
template <typename Real>
constexpr sfmm_precision precision_of() {
    static_assert(sizeof(Real) == 8 || sizeof(Real) == 4);
    return sizeof(Real) == 8 ? SFMM_F64 : SFMM_F32;
}
inline void raise(sfmm_status st) {
    if (st == SFMM_OK) return;
    const std::string what = sfmm_last_error();
    if (st == SFMM_INVALID_ARGUMENT) throw std::invalid_argument(what);
    if (st == SFMM_DOMAIN_ERROR) throw std::domain_error(what);
    throw std::runtime_error(std::string(sfmm_status_string(st)) + ": " + what);
}
}  // namespace detail

/// Shift-independent tables for translations up to a maximum order, resident on
/// one CUDA device. Immutable after construction and shareable between threads.
template <typename Real>
class operator_data {
public:
    explicit operator_data(int order, kernel_config cfg = default_kernel_config<Real>(), int device = 0)
        : order_(order), cfg_(cfg) {
        sfmm_handle* h = nullptr;
        detail::raise(sfmm_create(detail::precision_of<Real>(), order, device, cfg.mu, cfg.nu, &h));
        handle_.reset(h, sfmm_destroy);
    }
    int order() const noexcept { return order_; }
    const kernel_config& config() const noexcept { return cfg_; }
    static int max_order() noexcept { return sfmm_max_order(detail::precision_of<Real>()); }
    sfmm_handle* handle() const noexcept { return handle_.get(); }

    std::vector<Real> faculties() const {
        std::vector<double> f(2 * order_ - 1), i(order_);
        detail::raise(sfmm_get_faculties(handle_.get(), f.data(), i.data()));
        return std::vector<Real>(f.begin(), f.end());
    }
    std::vector<Real> inv_faculties() const {
        std::vector<double> f(2 * order_ - 1), i(order_);
        detail::raise(sfmm_get_faculties(handle_.get(), f.data(), i.data()));
        return std::vector<Real>(i.begin(), i.end());
    }

    /// Shared, lazily built instance per (order, cfg); thread safe.
    static std::shared_ptr<const operator_data> acquire(int order,
                                                        kernel_config cfg = default_kernel_config<Real>()) {
        using key_type = std::tuple<int, int, int>;
        static std::mutex mtx;
        static std::map<key_type, std::shared_ptr<const operator_data>> cache;
        const key_type key{order, cfg.mu, cfg.nu};
        std::lock_guard lock(mtx);
        auto it = cache.find(key);
        if (it == cache.end()) it = cache.emplace(key, std::make_shared<operator_data>(order, cfg)).first;
        return it->second;
    }

private:
    int order_;
    kernel_config cfg_;
    std::shared_ptr<sfmm_handle> handle_;
};

/// Kept for source compatibility: the device scratch lives in the handle.
template <typename Real>
class workspace {
public:
    explicit workspace(int max_order, kernel_config cfg = default_kernel_config<Real>())
        : max_order_(max_order), cfg_(cfg) {
        if (cfg.mu < 2 || (cfg.mu & 1) || cfg.mu > 32 || cfg.nu < 1 || cfg.nu > 64)
            throw std::invalid_argument("kernel_config out of range");
        if (max_order < 1) throw std::invalid_argument("max_order must be >= 1");
    }
    int max_order() const noexcept { return max_order_; }
    const kernel_config& config() const noexcept { return cfg_; }

private:
    int max_order_;
    kernel_config cfg_;
};

template <typename Real>
struct translation_request {
    const solid<Real>* source;
    vec3<Real> shift;
    int target_order;
    solid<Real>* output;
};

namespace detail {

// run_batch of the reference (pipeline.cpp:275-343): validate everything, then
// hand the whole mixed-order batch to the library (which groups by order pair),
// then resize / retag the outputs.
template <typename Real>
void run_batch(sfmm_kind kind, const operator_data<Real>& ops,
               std::span<const translation_request<Real>> batch, workspace<Real>& ws,
               solid_kind out_kind) {
    if (batch.empty()) return;
    if (!(ws.config() == ops.config()))
        throw std::invalid_argument("workspace kernel config does not match operator data");
    const std::size_t n = batch.size();
    std::vector<int> p_in(n), p_out(n);
    std::vector<int64_t> in_off(n), out_off(n);
    std::vector<Real> shifts(3 * n);
    std::size_t in_len = 0, out_len = 0;
    for (std::size_t i = 0; i < n; ++i) {
        const auto& req = batch[i];
        if (!req.source || !req.output) throw std::invalid_argument("translation request with null solid");
        p_in[i] = req.source->order();
        p_out[i] = req.target_order;
        if (p_in[i] < 1 || p_out[i] < 1) throw std::invalid_argument("translation orders must be >= 1");
        const int needed = std::max(p_in[i], p_out[i]);
        if (needed > ops.order()) throw std::invalid_argument("translation order exceeds operator data order");
        if (needed > ws.max_order()) throw std::invalid_argument("translation order exceeds workspace capacity");
        // per request, in the reference's order (pipeline.cpp:282-298): a zero shift in an
        // earlier request wins over a bad order in a later one
        if (std::hypot(req.shift.x, req.shift.y, req.shift.z) < std::numeric_limits<Real>::min())
            throw std::domain_error("translation with zero shift vector");
        in_off[i] = static_cast<int64_t>(in_len);
        out_off[i] = static_cast<int64_t>(out_len);
        in_len += solid_size(p_in[i]);
        out_len += solid_size(p_out[i]);
        shifts[3 * i] = req.shift.x;
        shifts[3 * i + 1] = req.shift.y;
        shifts[3 * i + 2] = req.shift.z;
    }
    // sources are staged before any output is written: an output may alias its
    // own source even when the order changes (pipeline.cpp:312-324)
    std::vector<Real> in(in_len), out(out_len);
    for (std::size_t i = 0; i < n; ++i)
        std::copy(batch[i].source->data().begin(), batch[i].source->data().end(), in.begin() + in_off[i]);
    raise(sfmm_translate_host_mixed(ops.handle(), kind, static_cast<int64_t>(n), p_in.data(), p_out.data(),
                                    in.data(), in_off.data(), shifts.data(), out.data(), out_off.data()));
    for (std::size_t i = 0; i < n; ++i) {
        solid<Real>* o = batch[i].output;
        if (o->order() != p_out[i]) *o = solid<Real>(out_kind, p_out[i]);
        else o->set_kind(out_kind);
        std::copy(out.begin() + out_off[i], out.begin() + out_off[i] + solid_size(p_out[i]), o->data().begin());
    }
}

}  // namespace detail

template <typename Real>
void m2l(const operator_data<Real>& ops, std::span<const translation_request<Real>> batch, workspace<Real>& ws) {
    detail::run_batch<Real>(SFMM_M2L, ops, batch, ws, solid_kind::local);
}
template <typename Real>
void m2m(const operator_data<Real>& ops, std::span<const translation_request<Real>> batch, workspace<Real>& ws) {
    detail::run_batch<Real>(SFMM_M2M, ops, batch, ws, solid_kind::multipole);
}
template <typename Real>
void l2l(const operator_data<Real>& ops, std::span<const translation_request<Real>> batch, workspace<Real>& ws) {
    detail::run_batch<Real>(SFMM_L2L, ops, batch, ws, solid_kind::local);
}

template <typename Real>
solid<Real> m2l(const operator_data<Real>& ops, const solid<Real>& m, const vec3<Real>& shift, int target_order,
                workspace<Real>& ws) {
    solid<Real> out(solid_kind::local, target_order);
    translation_request<Real> req{&m, shift, target_order, &out};
    m2l<Real>(ops, std::span<const translation_request<Real>>(&req, 1), ws);
    return out;
}
template <typename Real>
solid<Real> m2m(const operator_data<Real>& ops, const solid<Real>& m, const vec3<Real>& shift, int target_order,
                workspace<Real>& ws) {
    solid<Real> out(solid_kind::multipole, target_order);
    translation_request<Real> req{&m, shift, target_order, &out};
    m2m<Real>(ops, std::span<const translation_request<Real>>(&req, 1), ws);
    return out;
}
template <typename Real>
solid<Real> l2l(const operator_data<Real>& ops, const solid<Real>& l, const vec3<Real>& shift, int target_order,
                workspace<Real>& ws) {
    solid<Real> out(solid_kind::local, target_order);
    translation_request<Real> req{&l, shift, target_order, &out};
    l2l<Real>(ops, std::span<const translation_request<Real>>(&req, 1), ws);
    return out;
}

// ---- particle <-> expansion steps on the device (harmonics.hpp:10-51) ----------------------
// The reference's p2m / eval_local are free functions without a handle; here the device
// handle travels in `ops`. Batched forms (one call for many boxes / points) come first, the
// reference's single-object signatures forward to them.
template <typename Real>
struct point_charge {
    vec3<Real> position;
    Real charge;
};

/// Multipoles of `centers.size()` boxes; box b owns charges[box_ptr[b] .. box_ptr[b+1]).
template <typename Real>
std::vector<solid<Real>> p2m(const operator_data<Real>& ops, std::span<const point_charge<Real>> charges,
                             std::span<const std::int64_t> box_ptr, std::span<const vec3<Real>> centers, int order) {
    static_assert(sizeof(point_charge<Real>) == 4 * sizeof(Real) && sizeof(vec3<Real>) == 3 * sizeof(Real));
    if (order < 1 || order > ops.order()) throw std::invalid_argument("order out of range for this operator_data");
    if (box_ptr.size() != centers.size() + 1) throw std::invalid_argument("box_ptr must have one entry per box plus one");
    const std::size_t nb = centers.size();
    std::vector<Real> flat(nb * solid_size(order));
    detail::raise(sfmm_p2m_host(ops.handle(), static_cast<int64_t>(nb), box_ptr.data(), charges.data(), centers.data(),
                                order, flat.data()));
    std::vector<solid<Real>> out;
    out.reserve(nb);
    for (std::size_t b = 0; b < nb; ++b) {
        out.emplace_back(solid_kind::multipole, order);
        std::copy_n(flat.begin() + b * solid_size(order), solid_size(order), out.back().data().begin());
    }
    return out;
}
template <typename Real>
solid<Real> p2m(const operator_data<Real>& ops, std::span<const point_charge<Real>> sources,
                const vec3<Real>& center, int order) {
    const std::int64_t ptr[2] = {0, static_cast<std::int64_t>(sources.size())};
    return std::move(p2m<Real>(ops, sources, std::span<const std::int64_t>(ptr, 2),
                               std::span<const vec3<Real>>(&center, 1), order)[0]);
}

/// Potentials of local expansions: point i is evaluated with locals[box[i]] about centers[box[i]].
template <typename Real>
std::vector<Real> eval_local(const operator_data<Real>& ops, std::span<const solid<Real>> locals,
                             std::span<const vec3<Real>> centers, std::span<const std::int32_t> box,
                             std::span<const vec3<Real>> points) {
    if (locals.empty() || locals.size() != centers.size() || box.size() != points.size())
        throw std::invalid_argument("eval_local: array sizes do not match");
    const int order = locals[0].order();
    if (order > ops.order()) throw std::invalid_argument("order out of range for this operator_data");
    std::vector<Real> flat(locals.size() * solid_size(order));
    for (std::size_t b = 0; b < locals.size(); ++b) {
        if (locals[b].order() != order) throw std::invalid_argument("eval_local: one order per call");
        std::copy(locals[b].data().begin(), locals[b].data().end(), flat.begin() + b * solid_size(order));
    }
    std::vector<Real> out(points.size());
    detail::raise(sfmm_eval_local_host(ops.handle(), static_cast<int64_t>(points.size()), box.data(), points.data(),
                                       centers.data(), static_cast<int64_t>(locals.size()), order, flat.data(),
                                       out.data()));
    return out;
}
template <typename Real>
Real eval_local(const operator_data<Real>& ops, const solid<Real>& l, const vec3<Real>& center, const vec3<Real>& x) {
    const std::int32_t zero = 0;
    return eval_local<Real>(ops, std::span<const solid<Real>>(&l, 1), std::span<const vec3<Real>>(&center, 1),
                            std::span<const std::int32_t>(&zero, 1), std::span<const vec3<Real>>(&x, 1))[0];
}

// ---- text format of the reference tool (io.hpp:12-34, io.cpp:68-159) -----------------------
// `SOLID <kind letter> <P>` then P(P+1) reals in storage order, one row of the triangle per
// line, max_digits10 significant digits: files written here read back bit for bit, and files
// of the reference's `mpole` tool are accepted (and vice versa). Charges: one `x y z q` per
// line, blank lines and lines starting with '#' skipped. Malformed input raises
// std::runtime_error naming the line.
inline char kind_letter(solid_kind k) {
    switch (k) {
        case solid_kind::multipole: return 'M';
        case solid_kind::local: return 'L';
        case solid_kind::regular: return 'R';
        default: return 'S';
    }
}
inline solid_kind kind_from_letter(char c) {
    switch (c) {
        case 'M': return solid_kind::multipole;
        case 'L': return solid_kind::local;
        case 'R': return solid_kind::regular;
        case 'S': return solid_kind::singular;
        default: throw std::invalid_argument(std::string("unknown solid kind '") + c + "'");
    }
}

template <typename Real>
void write_solid(std::ostream& os, const solid<Real>& s) {
    os << "SOLID " << kind_letter(s.kind()) << ' ' << s.order() << '\n';
    os.precision(std::numeric_limits<Real>::max_digits10);
    for (int n = 0; n < s.order(); ++n) {
        for (int m = 0; m <= n; ++m) os << (m ? " " : "") << s.re(n, m) << ' ' << s.im(n, m);
        os << '\n';
    }
}

namespace detail {
// whitespace-separated tokens with the number of the line they were found on
struct token_stream {
    std::istream& is;
    std::istringstream cur;
    int line_no = 0;
    explicit token_stream(std::istream& in) : is(in) {}
    bool next(std::string& tok) {
        while (!(cur >> tok)) {
            std::string line;
            if (!std::getline(is, line)) return false;
            ++line_no;
            cur.clear();
            cur.str(line);
        }
        return true;
    }
    [[noreturn]] void fail(const std::string& what) const {
        throw std::runtime_error("line " + std::to_string(line_no) + ": " + what);
    }
};
}  // namespace detail

template <typename Real>
std::optional<solid<Real>> read_solid(std::istream& is) {
    detail::token_stream ts(is);
    std::string tok;
    if (!ts.next(tok)) return std::nullopt;
    if (tok != "SOLID") ts.fail("expected 'SOLID' header, got '" + tok + "'");
    if (!ts.next(tok) || tok.size() != 1) ts.fail("expected solid kind M, L, R or S");
    solid_kind kind;
    try {
        kind = kind_from_letter(tok[0]);
    } catch (const std::invalid_argument&) {
        ts.fail("expected solid kind M, L, R or S, got '" + tok + "'");
    }
    int order = 0;
    {
        std::string ot;
        std::size_t used = 0;
        const bool have = ts.next(ot);
        try {
            if (!have) throw std::invalid_argument("");
            order = std::stoi(ot, &used);
            if (used != ot.size()) throw std::invalid_argument(ot);
        } catch (const std::exception&) {
            ts.fail("expected an order, got '" + ot + "'");
        }
    }
    if (order < 1) ts.fail("order must be >= 1");
    solid<Real> s(kind, order);
    auto data = s.data();
    for (std::size_t i = 0; i < data.size(); ++i) {
        if (!ts.next(tok))
            ts.fail("unexpected end of input; expected " + std::to_string(data.size()) + " values, got " +
                    std::to_string(i));
        std::size_t used = 0;
        double v = 0;
        try {
            v = std::stod(tok, &used);
            if (used != tok.size()) throw std::invalid_argument(tok);
        } catch (const std::exception&) {
            ts.fail("expected a number, got '" + tok + "'");
        }
        data[i] = static_cast<Real>(v);
    }
    return s;
}

/// Concatenated solids until end of input. As in the reference every solid is parsed by its
/// own reader (io.cpp:124-129): line numbers in messages count from the solid's header line,
/// and a solid starts on a fresh line.
template <typename Real>
std::vector<solid<Real>> read_solids(std::istream& is) {
    std::vector<solid<Real>> out;
    while (auto s = read_solid<Real>(is)) out.push_back(std::move(*s));
    return out;
}

template <typename Real>
std::vector<point_charge<Real>> read_charges(std::istream& is) {
    std::vector<point_charge<Real>> charges;
    int line_no = 0;
    for (std::string line; std::getline(is, line);) {
        ++line_no;
        std::istringstream fields(line);
        std::string first;
        if (!(fields >> first) || first[0] == '#') continue;  // blank line or comment
        // four numbers, nothing else
        Real v[4];
        std::istringstream again(line);
        int have = 0;
        while (have < 4 && (again >> v[have])) ++have;
        if (have < 4) throw std::runtime_error("line " + std::to_string(line_no) + ": expected 'x y z q'");
        std::string extra;
        if (again >> extra)
            throw std::runtime_error("line " + std::to_string(line_no) + ": trailing content '" + extra + "'");
        charges.push_back({{v[0], v[1], v[2]}, v[3]});
    }
    return charges;
}

template <typename Real>
void write_charges(std::ostream& os, std::span<const point_charge<Real>> charges) {
    os.precision(std::numeric_limits<Real>::max_digits10);
    for (const point_charge<Real>& c : charges) {
        const Real row[4] = {c.position.x, c.position.y, c.position.z, c.charge};
        for (int k = 0; k < 4; ++k) os << row[k] << (k == 3 ? '\n' : ' ');
    }
}

}  // namespace mpole_b200

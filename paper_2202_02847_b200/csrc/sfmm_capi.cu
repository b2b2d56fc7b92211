// C-ABI layer: handle management, validation, host <-> device staging.
// See include/solidfmm_b200.h for the contract of every entry point.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "sfmm_internal.hpp"
#include "solidfmm_b200.h"

using namespace sfmm;

namespace {

thread_local std::string g_last_error;

sfmm_status fail(sfmm_status s, const std::string& msg) {
    g_last_error = msg;
    return s;
}
sfmm_status cuda_fail(cudaError_t e, const char* where) {
    return fail(e == cudaErrorMemoryAllocation ? SFMM_OUT_OF_MEMORY : SFMM_CUDA_ERROR,
                std::string(where) + ": " + cudaGetErrorString(e));
}
#define CU(call)                                                  \
    do {                                                          \
        cudaError_t e_ = (call);                                  \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call);       \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// Stream of the host-buffer entry points: one non-blocking stream per calling thread and
// device, so that concurrent callers (one workspace per thread in the reference,
// pipeline.hpp:30-45) neither serialise on the legacy default stream nor on each other.
cudaStream_t host_stream(int device, int which = 0) {
    thread_local std::vector<std::pair<int, cudaStream_t>> cache;
    const int key = device * 2 + which;
    for (const auto& e : cache)
        if (e.first == key) return e.second;
    cudaStream_t s = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) s = nullptr;
    cache.emplace_back(key, s);
    return s;
}

// Stream-ordered device allocation that is released on every exit path.
struct DevBuf {
    void* p = nullptr;
    cudaStream_t s;
    explicit DevBuf(cudaStream_t stream) : s(stream) {}
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    cudaError_t alloc(size_t bytes) { return cudaMallocAsync(&p, std::max<size_t>(bytes, 16), s); }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
    ~DevBuf() {
        if (p) cudaFreeAsync(p, s);
    }
};

constexpr int kFlagSlots = 256;
constexpr int64_t kHostChunk = 1 << 20;  // translations per staging chunk of the host path
constexpr int kPlanGroup = 64;  // pairs of one target are padded to multiples of this

int64_t round_up32(int64_t n) { return (n + 31) / 32 * 32; }
int64_t solid_len(int p) { return (int64_t)p * (p + 1); }

}  // namespace

struct sfmm_handle {
    int precision = SFMM_F64;
    int order = 0;
    int device = 0;
    int sm_count = 0;
    SwapTables host_tables{1};
    std::vector<double> fac, inv;  // values in the handle precision, widened
    DeviceTables<double> td;
    DeviceTables<float> tf;
    std::vector<void*> allocations;
    int* d_flags = nullptr;
    int* h_flags = nullptr;  // pinned
    std::atomic<int64_t> launches{0};
    // zero-shift flags of the device entry points: a slot belongs to one call until its
    // result has been read (synchronous calls: at once; SFMM_ASYNC_STATUS calls: by
    // sfmm_stream_status on the stream they were issued on)
    struct Pending {
        int slot;
        cudaStream_t stream;
    };
    std::mutex async_mutex;
    std::vector<int> free_slots;
    std::vector<Pending> pending;
    int variant = 0;
    int64_t level_slab_pairs = 1 << 18;   // sfmm_m2l_level_host pipelines from 4 x this many pairs
    bool accumulate_plain = false;        // "accumulate_plain" option (sfmm_m2l_accumulate*)
    bool precise = false;                 // "precise" option: double-double backward pass
    long long* d_phase_clocks = nullptr;  // set by the "phase_clocks" option
};

struct sfmm_plan {
    sfmm_handle* h = nullptr;
    int64_t n_targets = 0, n_pairs = 0, n_groups = 0, n_sources = 0;
    int64_t* d_grp_ptr = nullptr;   // [n_targets + 1]
    int32_t* d_src_index = nullptr; // [n_groups * 64], -1 = idle lane
    void* d_shifts = nullptr;       // [n_groups * 64][3]
    void* d_angles = nullptr;       // [6][n_groups * 64]: decomposed shifts (TranslateArgs::angles), one
                                    // entry per distinct shift at the front (or one per lane)
    int32_t* d_angle_index = nullptr; // [n_groups * 64]: entry of every lane
    int32_t* d_grp_target = nullptr; // [n_groups]: target of every group
    int64_t max_groups = 0;         // most groups of one target
    cudaStream_t last_stream = nullptr;  // stream of the most recent accumulate call (destroy order)
};

namespace {

template <typename Real>
sfmm_status upload_tables(sfmm_handle* h, DeviceTables<Real>& t) {
    t.order = h->order;
    for (int side = 0; side < 2; ++side) {
        const PackedSide ps = pack_side(h->host_tables, side == 1);
        // zero slack behind the stream: the tiled kernel stages a fixed pad past
        // the prefix it needs (kernel_tiled.inl, TAB_PAD)
        std::vector<Real> s(ps.stream.size() + 128, Real(0));
        for (size_t i = 0; i < ps.stream.size(); ++i) s[i] = static_cast<Real>(ps.stream[i]);
        Real* ds = nullptr;
        BlockDesc* dd = nullptr;
        CU(cudaMalloc((void**)&ds, std::max<size_t>(s.size(), 2) * sizeof(Real)));
        h->allocations.push_back(ds);
        CU(cudaMalloc((void**)&dd, ps.desc.size() * sizeof(BlockDesc)));
        h->allocations.push_back(dd);
        CU(cudaMemcpy(ds, s.data(), s.size() * sizeof(Real), cudaMemcpyHostToDevice));
        CU(cudaMemcpy(dd, ps.desc.data(), ps.desc.size() * sizeof(BlockDesc),
                      cudaMemcpyHostToDevice));
        t.stream[side] = ds;
        t.desc[side] = dd;
        t.stream_len[side] = (uint32_t)s.size();
    }
    // fragment-major copies for the tensor-core kernel (double precision, orders <= 30)
    if (sizeof(Real) == 8 && h->order <= 30) {
        for (int side = 0; side < 2; ++side) {
            const FragSide fs = pack_frags(h->host_tables, side == 1);
            // zero slack: a product may read a few fragments past its block (masked inputs)
            std::vector<Real> s(fs.frags.size() + 16 * 32, Real(0));
            for (size_t i = 0; i < fs.frags.size(); ++i) s[i] = static_cast<Real>(fs.frags[i]);
            Real* ds = nullptr;
            CU(cudaMalloc((void**)&ds, s.size() * sizeof(Real)));
            h->allocations.push_back(ds);
            CU(cudaMemcpy(ds, s.data(), s.size() * sizeof(Real), cudaMemcpyHostToDevice));
            t.frags[side] = ds;
        }
    }
    std::vector<Real> fac, inv;
    build_faculties<Real>(h->order, fac, inv);
    std::vector<Real> winv(inv);
    for (size_t d = 1; d < winv.size(); d += 2) winv[d] = -winv[d];
    h->fac.assign(fac.begin(), fac.end());
    h->inv.assign(inv.begin(), inv.end());
    Real *dfac = nullptr, *dinv = nullptr, *dwinv = nullptr;
    CU(cudaMalloc((void**)&dfac, fac.size() * sizeof(Real)));
    h->allocations.push_back(dfac);
    CU(cudaMalloc((void**)&dinv, inv.size() * sizeof(Real)));
    h->allocations.push_back(dinv);
    CU(cudaMalloc((void**)&dwinv, winv.size() * sizeof(Real)));
    h->allocations.push_back(dwinv);
    CU(cudaMemcpy(dfac, fac.data(), fac.size() * sizeof(Real), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(dinv, inv.data(), inv.size() * sizeof(Real), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(dwinv, winv.data(), winv.size() * sizeof(Real), cudaMemcpyHostToDevice));
    t.fac = dfac;
    t.inv = dinv;
    t.winv = dwinv;
    return SFMM_OK;
}

template <typename Real>
const DeviceTables<Real>& tables_of(const sfmm_handle* h);
template <>
const DeviceTables<double>& tables_of<double>(const sfmm_handle* h) { return h->td; }
template <>
const DeviceTables<float>& tables_of<float>(const sfmm_handle* h) { return h->tf; }

sfmm_status check_orders(const sfmm_handle* h, int kind, int p_in, int p_out) {
    if (!h) return fail(SFMM_INVALID_ARGUMENT, "null handle");
    if (h->variant == 2 && std::max(p_in, p_out) > (h->precision == SFMM_F64 ? 20 : 18))
        return fail(SFMM_INVALID_ARGUMENT, "tiled kernel variant does not cover this order");
    if (h->variant == 3 && (h->precision != SFMM_F64 || h->order > 30))
        return fail(SFMM_INVALID_ARGUMENT, "mma kernel variant: double precision, handle order <= 30");
    if (h->variant == 4 && (p_in != p_out || p_in > 8))
        return fail(SFMM_INVALID_ARGUMENT, "small kernel variant: same order, at most 8");
    if (h->precise && h->variant > 1)
        return fail(SFMM_INVALID_ARGUMENT, "the precise mode runs on the generic kernel only (kernel_variant 0 or 1)");
    if (kind < 0 || kind > 2) return fail(SFMM_INVALID_ARGUMENT, "unknown translation kind");
    // pipeline.cpp:285-295
    if (p_in < 1 || p_out < 1)
        return fail(SFMM_INVALID_ARGUMENT, "translation orders must be >= 1");
    if (std::max(p_in, p_out) > h->order)
        return fail(SFMM_INVALID_ARGUMENT, "translation order exceeds operator data order");
    return SFMM_OK;
}

// pipeline.cpp:296-297: norm(shift) < numeric_limits<Real>::min()
template <typename Real>
bool host_shift_degenerate(const Real* r) {
    // |r| >= max |component|: the norm needs evaluating only for all-subnormal shifts
    const Real mn = std::numeric_limits<Real>::min();
    if (std::fabs(r[0]) >= mn || std::fabs(r[1]) >= mn || std::fabs(r[2]) >= mn) return false;
    return std::hypot(r[0], r[1], r[2]) < mn;
}

int acquire_slot(sfmm_handle* h) {
    std::lock_guard<std::mutex> lk(h->async_mutex);
    if (h->free_slots.empty()) return -1;
    const int slot = h->free_slots.back();
    h->free_slots.pop_back();
    return slot;
}
void release_slot(sfmm_handle* h, int slot) {
    std::lock_guard<std::mutex> lk(h->async_mutex);
    h->free_slots.push_back(slot);
}

template <typename Real>
sfmm_status translate_soa_impl(sfmm_handle* h, int kind, int64_t n, int p_in, int p_out,
                               const Real* d_in, int64_t in_stride, const Real* d_shifts,
                               Real* d_out, int64_t out_stride, cudaStream_t stream, int flags,
                               bool skip_scan) {
    int slot = -1;
    int* d_flag = nullptr;
    DevBuf spare(stream);  // flag of a call that finds every slot waiting for its query
    if (!skip_scan) {
        slot = acquire_slot(h);
        if (slot >= 0) {
            d_flag = h->d_flags + slot;
        } else {
            CU(spare.alloc(sizeof(int)));
            d_flag = spare.as<int>();
        }
        // free slots are zero (zeroed at creation and whenever a failure has been read)
        cudaError_t e = slot >= 0 ? cudaSuccess : cudaMemsetAsync(d_flag, 0, sizeof(int), stream);
        if (e == cudaSuccess) e = launch_check_shifts<Real>(d_shifts, n, d_flag, stream);
        if (e != cudaSuccess) {
            if (slot >= 0) release_slot(h, slot);
            return cuda_fail(e, "zero-shift scan");
        }
        h->launches += 1;
    }
    TranslateArgs<Real> a;
    a.kind = kind;
    a.p_in = p_in;
    a.p_out = p_out;
    a.n = n;
    a.in = d_in;
    a.in_stride = in_stride;
    a.shifts = d_shifts;
    a.out = d_out;
    a.out_stride = out_stride;
    a.fail_flag = d_flag;
    a.variant = h->variant;
    a.precise = h->precise;
    a.phase_clocks = h->d_phase_clocks;
    LaunchInfo info;
    cudaError_t e = launch_translate<Real>(tables_of<Real>(h), a, h->sm_count, stream, &info);
    if (e != cudaSuccess) {
        if (slot >= 0) {
            cudaStreamSynchronize(stream);  // the scan may still write the slot
            cudaMemsetAsync(d_flag, 0, sizeof(int), stream);
            cudaStreamSynchronize(stream);
            release_slot(h, slot);
        }
        return cuda_fail(e, "launch_translate");
    }
    h->launches += info.launches;
    if (skip_scan) return SFMM_OK;
    if ((flags & SFMM_ASYNC_STATUS) && slot >= 0) {
        std::lock_guard<std::mutex> lk(h->async_mutex);
        h->pending.push_back({slot, stream});
        return SFMM_OK;
    }
    // synchronous status (also when all slots are taken: the call then reports at once)
    int value = 0;
    int* dst = slot >= 0 ? h->h_flags + slot : &value;
    e = cudaMemcpyAsync(dst, d_flag, sizeof(int), cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    const int bad = *dst;
    if (slot >= 0) {
        if (bad || e != cudaSuccess) {  // back to the free-slot invariant before the slot is reused
            cudaMemsetAsync(d_flag, 0, sizeof(int), stream);
            cudaStreamSynchronize(stream);
        }
        release_slot(h, slot);
    }
    if (e != cudaSuccess) return cuda_fail(e, "zero-shift status");
    if (bad) return fail(SFMM_DOMAIN_ERROR, "translation with zero shift vector");
    return SFMM_OK;
}

template <typename Real>
sfmm_status translate_host_impl(sfmm_handle* h, int kind, int64_t n, int p_in, int p_out,
                                const Real* in, const Real* shifts, Real* out) {
    for (int64_t i = 0; i < n; ++i)
        if (host_shift_degenerate(shifts + 3 * i))
            return fail(SFMM_DOMAIN_ERROR, "translation with zero shift vector");
    const int64_t si = solid_len(p_in), so = solid_len(p_out);
    // Staged in chunks on two streams: the device scratch stays bounded however large the
    // batch is, and the upload of chunk i+1 overlaps the kernels and the download of chunk i
    // (the link is full duplex; from pinned host memory the copies are asynchronous).
    int64_t chunk = std::min(n, kHostChunk);
    if (n >= 65536) chunk = std::min(chunk, (n / 8 + 31) / 32 * 32);
    const int64_t stride = round_up32(chunk);
    const int lanes = n > chunk ? 2 : 1;
    const size_t es = sizeof(Real);
    struct Lane {
        cudaStream_t stream;
        DevBuf in_aos, in, sh, out, out_aos;
        explicit Lane(cudaStream_t s) : stream(s), in_aos(s), in(s), sh(s), out(s), out_aos(s) {}
    };
    Lane lane0(host_stream(h->device, 0)), lane1(host_stream(h->device, 1));
    Lane* lane[2] = {&lane0, &lane1};
    for (int l = 0; l < lanes; ++l) {
        CU(lane[l]->in_aos.alloc(es * si * chunk));
        CU(lane[l]->in.alloc(es * si * stride));
        CU(lane[l]->sh.alloc(es * 3 * chunk));
        CU(lane[l]->out.alloc(es * so * stride));
        CU(lane[l]->out_aos.alloc(es * so * chunk));
    }
    sfmm_status st = SFMM_OK;
    cudaError_t e = cudaSuccess;
    int64_t c = 0;
    for (int64_t lo = 0; lo < n && st == SFMM_OK && e == cudaSuccess; lo += chunk, ++c) {
        Lane& L = *lane[c & (lanes - 1)];
        const int64_t m = std::min(chunk, n - lo);
        e = cudaMemcpyAsync(L.in_aos.p, in + lo * si, es * si * m, cudaMemcpyHostToDevice, L.stream);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(L.sh.p, shifts + 3 * lo, es * 3 * m, cudaMemcpyHostToDevice, L.stream);
        if (e == cudaSuccess)
            e = launch_pack_soa<Real>(L.in_aos.template as<Real>(), L.in.template as<Real>(), m, p_in, stride,
                                      L.stream);
        if (e != cudaSuccess) break;
        st = translate_soa_impl<Real>(h, kind, m, p_in, p_out, L.in.template as<Real>(), stride,
                                      L.sh.template as<Real>(), L.out.template as<Real>(), stride, L.stream, 0,
                                      /*skip_scan=*/true);
        if (st != SFMM_OK) break;
        e = launch_unpack_soa<Real>(L.out.template as<Real>(), L.out_aos.template as<Real>(), m, p_out, stride,
                                    L.stream);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(out + lo * so, L.out_aos.p, es * so * m, cudaMemcpyDeviceToHost, L.stream);
        h->launches += 2;
    }
    // both streams are drained on every path: the scratch is released behind them
    for (int l = 0; l < lanes; ++l) {
        const cudaError_t e2 = cudaStreamSynchronize(lane[l]->stream);
        if (e == cudaSuccess) e = e2;
    }
    if (st != SFMM_OK) return st;
    if (e != cudaSuccess) return cuda_fail(e, "translate_host");
    return SFMM_OK;
}

template <typename Real>
sfmm_status translate_host_mixed_impl(sfmm_handle* h, int kind, int64_t n, const int* p_in,
                                      const int* p_out, const Real* in, const int64_t* in_off,
                                      const Real* shifts, Real* out, const int64_t* out_off) {
    // validate everything first (pipeline.cpp:282-298)
    for (int64_t i = 0; i < n; ++i) {
        const sfmm_status st = check_orders(h, kind, p_in[i], p_out[i]);
        if (st != SFMM_OK) return st;
        if (host_shift_degenerate(shifts + 3 * i))
            return fail(SFMM_DOMAIN_ERROR, "translation with zero shift vector");
    }
    // group by order pair, keeping the request order inside a group (pipeline.cpp:302-308)
    std::vector<int64_t> idx(n);
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) {
        if (p_in[a] != p_in[b]) return p_in[a] < p_in[b];
        return p_out[a] < p_out[b];
    });
    // One upload, one launch sequence per order pair, one download. The sources are staged
    // (sorted by order pair) before any output is written, so an output may alias its own
    // source even when the order changes (pipeline.cpp:312-324).
    std::vector<int64_t> in_pos((size_t)n), out_pos((size_t)n);
    int64_t in_len = 0, out_len = 0, max_group = 0, max_si = 0, max_so = 0;
    std::vector<std::pair<int64_t, int64_t>> ranges;
    for (int64_t i = 0; i < n;) {
        int64_t j = i;
        while (j < n && p_in[idx[j]] == p_in[idx[i]] && p_out[idx[j]] == p_out[idx[i]]) ++j;
        const int64_t si = solid_len(p_in[idx[i]]), so = solid_len(p_out[idx[i]]);
        for (int64_t k = i; k < j; ++k) {
            in_pos[(size_t)k] = in_len + (k - i) * si;
            out_pos[(size_t)k] = out_len + (k - i) * so;
        }
        in_len += si * (j - i);
        out_len += so * (j - i);
        max_group = std::max(max_group, j - i);
        max_si = std::max(max_si, si * round_up32(j - i));
        max_so = std::max(max_so, so * round_up32(j - i));
        ranges.emplace_back(i, j);
        i = j;
    }
    std::vector<Real> stage_in((size_t)in_len), stage_sh((size_t)(3 * n)), stage_out((size_t)out_len);
    for (int64_t k = 0; k < n; ++k) {
        std::memcpy(&stage_in[(size_t)in_pos[(size_t)k]], in + in_off[idx[k]],
                    sizeof(Real) * solid_len(p_in[idx[k]]));
        std::memcpy(&stage_sh[(size_t)(3 * k)], shifts + 3 * idx[k], sizeof(Real) * 3);
    }
    cudaStream_t stream = host_stream(h->device);
    const size_t es = sizeof(Real);
    DevBuf d_in_all(stream), d_sh_all(stream), d_out_all(stream), d_in(stream), d_out(stream);
    CU(d_in_all.alloc(es * in_len));
    CU(d_sh_all.alloc(es * 3 * n));
    CU(d_out_all.alloc(es * out_len));
    CU(d_in.alloc(es * max_si));
    CU(d_out.alloc(es * max_so));
    CU(cudaMemcpyAsync(d_in_all.p, stage_in.data(), es * in_len, cudaMemcpyHostToDevice, stream));
    CU(cudaMemcpyAsync(d_sh_all.p, stage_sh.data(), es * 3 * n, cudaMemcpyHostToDevice, stream));
    for (const auto& r : ranges) {
        const int64_t i = r.first, m = r.second - r.first, stride = round_up32(m);
        const int pi = p_in[idx[i]], po = p_out[idx[i]];
        const Real* src = d_in_all.as<Real>() + in_pos[(size_t)i];
        Real* dst = d_out_all.as<Real>() + out_pos[(size_t)i];
        CU(launch_pack_soa<Real>(src, d_in.as<Real>(), m, pi, stride, stream));
        const sfmm_status st =
            translate_soa_impl<Real>(h, kind, m, pi, po, d_in.as<Real>(), stride,
                                     d_sh_all.as<Real>() + 3 * i, d_out.as<Real>(), stride, stream, 0,
                                     /*skip_scan=*/true);
        if (st != SFMM_OK) return st;
        CU(launch_unpack_soa<Real>(d_out.as<Real>(), dst, m, po, stride, stream));
        h->launches += 2;
    }
    CU(cudaMemcpyAsync(stage_out.data(), d_out_all.p, es * out_len, cudaMemcpyDeviceToHost, stream));
    CU(cudaStreamSynchronize(stream));
    for (int64_t k = 0; k < n; ++k)
        std::memcpy(out + out_off[idx[k]], &stage_out[(size_t)out_pos[(size_t)k]],
                    sizeof(Real) * solid_len(p_out[idx[k]]));
    return SFMM_OK;
}

template <typename Real>
sfmm_status plan_create_impl(sfmm_handle* h, int64_t n_targets, const int64_t* tgt_ptr,
                             const int32_t* src_index, const Real* shifts, int64_t n_sources,
                             sfmm_plan* plan) {
    const int64_t n_pairs = tgt_ptr[n_targets];
    std::vector<int64_t> grp_ptr((size_t)n_targets + 1, 0);
    for (int64_t t = 0; t < n_targets; ++t) {
        const int64_t cnt = tgt_ptr[t + 1] - tgt_ptr[t];
        if (cnt < 0) return fail(SFMM_INVALID_ARGUMENT, "tgt_ptr must be non-decreasing");
        grp_ptr[(size_t)t + 1] = grp_ptr[(size_t)t] + (cnt + kPlanGroup - 1) / kPlanGroup;
    }
    const int64_t n_groups = grp_ptr[(size_t)n_targets];
    for (int64_t t = 0; t < n_targets; ++t)
        plan->max_groups = std::max(plan->max_groups, grp_ptr[(size_t)t + 1] - grp_ptr[(size_t)t]);
    std::vector<int32_t> grp_target((size_t)std::max<int64_t>(n_groups, 1));
    for (int64_t t = 0; t < n_targets; ++t)
        for (int64_t g = grp_ptr[(size_t)t]; g < grp_ptr[(size_t)t + 1]; ++g)
            grp_target[(size_t)g] = (int32_t)t;
    plan->h = h;
    plan->n_targets = n_targets;
    plan->n_pairs = n_pairs;
    plan->n_groups = n_groups;
    plan->n_sources = n_sources;
    // the raw pair list goes to the device as it is; padding to whole groups and the
    // validation (source range, zero shifts) happen there
    cudaStream_t stream = host_stream(h->device);
    const size_t padded = (size_t)std::max<int64_t>(n_groups, 1) * kPlanGroup;
    // stream-ordered allocations from the device pool (kept warm by sfmm_create): a plan
    // per call costs no cudaMalloc / cudaFree round trips. The plan's own buffers are freed
    // by sfmm_plan_destroy (also on the failure paths: the caller destroys the plan).
    CU(cudaMallocAsync((void**)&plan->d_grp_ptr, sizeof(int64_t) * grp_ptr.size(), stream));
    CU(cudaMallocAsync((void**)&plan->d_src_index, sizeof(int32_t) * padded, stream));
    CU(cudaMallocAsync(&plan->d_shifts, sizeof(Real) * padded * 3, stream));
    CU(cudaMallocAsync(&plan->d_angles, sizeof(Real) * padded * 6, stream));
    CU(cudaMallocAsync((void**)&plan->d_angle_index, sizeof(int32_t) * padded, stream));
    CU(cudaMallocAsync((void**)&plan->d_grp_target, sizeof(int32_t) * grp_target.size(), stream));
    plan->last_stream = stream;
    DevBuf d_tgt(stream), d_idx(stream), d_sh(stream), d_flags(stream);
    const size_t np = (size_t)std::max<int64_t>(n_pairs, 1);
    CU(d_tgt.alloc(sizeof(int64_t) * (n_targets + 1)));
    CU(d_idx.alloc(sizeof(int32_t) * np));
    CU(d_sh.alloc(sizeof(Real) * np * 3));
    CU(d_flags.alloc(sizeof(int) * 2));
    CU(cudaMemsetAsync(d_flags.p, 0, sizeof(int) * 2, stream));
    CU(cudaMemcpyAsync(plan->d_grp_ptr, grp_ptr.data(), sizeof(int64_t) * grp_ptr.size(),
                       cudaMemcpyHostToDevice, stream));
    CU(cudaMemcpyAsync(d_tgt.p, tgt_ptr, sizeof(int64_t) * (n_targets + 1), cudaMemcpyHostToDevice,
                       stream));
    CU(cudaMemcpyAsync(plan->d_grp_target, grp_target.data(), sizeof(int32_t) * grp_target.size(),
                       cudaMemcpyHostToDevice, stream));
    if (n_pairs > 0) {
        CU(cudaMemcpyAsync(d_idx.p, src_index, sizeof(int32_t) * n_pairs, cudaMemcpyHostToDevice,
                           stream));
        CU(cudaMemcpyAsync(d_sh.p, shifts, sizeof(Real) * n_pairs * 3, cudaMemcpyHostToDevice,
                           stream));
    }
    CU(launch_build_plan<Real>(d_tgt.as<int64_t>(), plan->d_grp_ptr, plan->d_grp_target,
                               d_idx.as<int32_t>(), d_sh.as<Real>(), n_groups, n_sources, kPlanGroup,
                               plan->d_src_index, static_cast<Real*>(plan->d_shifts),
                               static_cast<Real*>(plan->d_angles), plan->d_angle_index,
                               d_flags.as<int>(), stream));
    h->launches += 4;
    int flags[2] = {0, 0};
    CU(cudaMemcpyAsync(flags, d_flags.p, sizeof(flags), cudaMemcpyDeviceToHost, stream));
    CU(cudaStreamSynchronize(stream));
    if (flags[0]) return fail(SFMM_INVALID_ARGUMENT, "source index out of range");
    if (flags[1]) return fail(SFMM_DOMAIN_ERROR, "translation with zero shift vector");
    return SFMM_OK;
}

template <typename Real>
sfmm_status accumulate_impl(sfmm_handle* h, const sfmm_plan* plan, int p_in, int p_out,
                            const Real* d_src, int64_t src_stride, int src_layout, Real* d_out,
                            int64_t out_stride, cudaStream_t stream, int reserve_sms = 0) {
    const int64_t so = solid_len(p_out);
    TranslateArgs<Real> a;
    a.reserve_sms = reserve_sms;
    a.kind = KIND_M2L;
    a.p_in = p_in;
    a.p_out = p_out;
    a.variant = h->variant;
    a.precise = h->precise;
    a.src_index = plan->d_src_index;  // accumulate mode decides which kernels apply
    a.in_layout = src_layout;
    if (translate_variant<Real>(tables_of<Real>(h), a) == 0)
        return fail(SFMM_INVALID_ARGUMENT, "the selected kernel variant does not apply to this call");
    a.in = d_src;
    a.in_stride = src_stride;
    a.shifts = static_cast<const Real*>(plan->d_shifts);
    a.angles = static_cast<const Real*>(plan->d_angles);
    a.angle_index = plan->d_angle_index;
    a.n = plan->n_groups * kPlanGroup;
    a.phase_clocks = h->d_phase_clocks;
    // tiled kernel, direct form: a CTA owns whole targets and adds their groups itself. Not for
    // lists with a target so long that its CTA would run on alone (more than 1/8 of a CTA's
    // share of the groups): those take the partial sums + reduce_groups_kernel path below
    const bool direct = translate_variant<Real>(tables_of<Real>(h), a) == 2 && plan->d_grp_target &&
                        (plan->max_groups <= 4 ||
                         plan->max_groups * 8 * (int64_t)h->sm_count <= plan->n_groups);
    if (direct) {
        const_cast<sfmm_plan*>(plan)->last_stream = stream;
        a.out = d_out;
        a.out_stride = out_stride;
        a.grp_target = plan->d_grp_target;
        a.acc_plain = h->accumulate_plain;
        a.grp_ptr = plan->d_grp_ptr;
        a.n_targets = plan->n_targets;
        cudaError_t e = launch_zero_unwritten<Real>(plan->d_grp_ptr, plan->n_targets, p_out, d_out,
                                                    out_stride, stream);
        LaunchInfo info;
        if (e == cudaSuccess && a.n > 0)
            e = launch_translate<Real>(tables_of<Real>(h), a, h->sm_count, stream, &info);
        h->launches += 1 + info.launches;
        if (e != cudaSuccess) return cuda_fail(e, "m2l_accumulate");
        return SFMM_OK;
    }
    // the kernel reduces the lanes of one of ITS groups (16, 32 or 64 pairs) into one partial
    const int per = kPlanGroup / translate_group_size<Real>(tables_of<Real>(h), a);
    const int64_t n_partial = plan->n_groups * per;
    DevBuf partial(stream);
    if (n_partial > 0) CU(partial.alloc(sizeof(Real) * so * n_partial));
    const_cast<sfmm_plan*>(plan)->last_stream = stream;
    a.out = partial.as<Real>();
    a.out_stride = n_partial;
    LaunchInfo info;
    cudaError_t e = launch_translate<Real>(tables_of<Real>(h), a, h->sm_count, stream, &info);
    h->launches += info.launches;
    if (e == cudaSuccess) {
        e = launch_reduce_groups<Real>(partial.as<Real>(), n_partial, plan->d_grp_ptr, per,
                                       plan->n_targets, p_out, d_out, out_stride, stream);
        h->launches += 1;
    }
    if (e != cudaSuccess) return cuda_fail(e, "m2l_accumulate");
    return SFMM_OK;
}

template <typename Real>
sfmm_status accumulate_host_impl(sfmm_handle* h, const sfmm_plan* plan, int p_in, int p_out,
                                 const Real* src_aos, Real* out_aos) {
    const int64_t si = solid_len(p_in), so = solid_len(p_out);
    const int64_t ns = plan->n_sources, nt = plan->n_targets;
    const int64_t srows = rows_off(p_in), ostride = round_up32(nt);
    cudaStream_t stream = host_stream(h->device);
    const size_t es = sizeof(Real);
    DevBuf d_src_aos(stream), d_src(stream), d_out(stream), d_out_aos(stream);
    CU(d_src_aos.alloc(es * si * ns));
    CU(d_src.alloc(es * srows * ns));
    CU(d_out.alloc(es * so * ostride));
    CU(d_out_aos.alloc(es * so * nt));
    CU(cudaMemcpyAsync(d_src_aos.p, src_aos, es * si * ns, cudaMemcpyHostToDevice, stream));
    CU(launch_pack_rows<Real>(d_src_aos.as<Real>(), d_src.as<Real>(), ns, p_in, stream));
    const sfmm_status st = accumulate_impl<Real>(h, plan, p_in, p_out, d_src.as<Real>(), srows,
                                                 LAYOUT_ROWS, d_out.as<Real>(), ostride, stream);
    if (st != SFMM_OK) return st;
    CU(launch_unpack_soa<Real>(d_out.as<Real>(), d_out_aos.as<Real>(), nt, p_out, ostride, stream));
    CU(cudaMemcpyAsync(out_aos, d_out_aos.p, es * so * nt, cudaMemcpyDeviceToHost, stream));
    CU(cudaStreamSynchronize(stream));
    h->launches += 3;
    return SFMM_OK;
}

// One-shot level (plan + accumulation) from host arrays, pipelined over target slabs:
// the pair list of slab k+1 uploads while slab k computes, the locals of slab k download
// while slab k+1 computes. Nothing is written to `out_aos` before every slab has passed the
// validation (pipeline.cpp:282-298: all requests are checked before any output is touched).
template <typename Real>
sfmm_status level_host_impl(sfmm_handle* h, int64_t n_targets, const int64_t* tgt_ptr,
                            const int32_t* src_index, const Real* shifts, int64_t n_sources, int p_in,
                            int p_out, const Real* src_aos, Real* out_aos) {
    const int64_t n_pairs = tgt_ptr[n_targets];
    const int K = n_pairs >= 4 * h->level_slab_pairs ? 4 : (n_pairs >= 2 * h->level_slab_pairs ? 2 : 1);
    if (K == 1) {
        sfmm_plan plan;
        sfmm_status st = plan_create_impl<Real>(h, n_targets, tgt_ptr, src_index, shifts, n_sources, &plan);
        if (st == SFMM_OK) st = accumulate_host_impl<Real>(h, &plan, p_in, p_out, src_aos, out_aos);
        cudaStream_t s = plan.last_stream;
        if (plan.d_grp_ptr) cudaFreeAsync(plan.d_grp_ptr, s);
        if (plan.d_src_index) cudaFreeAsync(plan.d_src_index, s);
        if (plan.d_shifts) cudaFreeAsync(plan.d_shifts, s);
        if (plan.d_angles) cudaFreeAsync(plan.d_angles, s);
        if (plan.d_angle_index) cudaFreeAsync(plan.d_angle_index, s);
        if (plan.d_grp_target) cudaFreeAsync(plan.d_grp_target, s);
        return st;
    }
    for (int64_t t = 0; t < n_targets; ++t)
        if (tgt_ptr[t + 1] < tgt_ptr[t]) return fail(SFMM_INVALID_ARGUMENT, "tgt_ptr must be non-decreasing");
    const int64_t si = solid_len(p_in), so = solid_len(p_out), srows = rows_off(p_in);
    const size_t es = sizeof(Real);
    cudaStream_t sc = host_stream(h->device, 0), sx = host_stream(h->device, 1);
    // slabs of about equal pair counts, cut at target boundaries
    std::vector<int64_t> cut(K + 1, n_targets);
    cut[0] = 0;
    for (int k = 1; k < K; ++k)
        cut[k] = std::lower_bound(tgt_ptr, tgt_ptr + n_targets + 1, n_pairs * k / K) - tgt_ptr;
    struct Slab {
        sfmm_plan plan;
        std::vector<int64_t> grp_ptr;
        std::vector<int32_t> grp_target;
        DevBuf tgt, idx, sh, out, out_aos;
        cudaEvent_t ready = nullptr, done = nullptr;
        int64_t t0 = 0, ostride = 0;
        explicit Slab(cudaStream_t c, cudaStream_t x) : tgt(c), idx(c), sh(c), out(x), out_aos(x) {}
    };
    // declared before the guard below: the guard drains the streams first, then the buffers go
    DevBuf d_src_aos(sc), d_src(sc), d_flags(sc);
    std::vector<std::unique_ptr<Slab>> slabs;
    struct Drain {
        cudaStream_t a, b;
        std::vector<std::unique_ptr<Slab>>* slabs;
        ~Drain() {
            cudaStreamSynchronize(a);
            cudaStreamSynchronize(b);
            for (auto& s : *slabs) {
                if (s->ready) cudaEventDestroy(s->ready);
                if (s->done) cudaEventDestroy(s->done);
                sfmm_plan& p = s->plan;
                if (p.d_grp_ptr) cudaFreeAsync(p.d_grp_ptr, a);
                if (p.d_src_index) cudaFreeAsync(p.d_src_index, a);
                if (p.d_shifts) cudaFreeAsync(p.d_shifts, a);
                if (p.d_angles) cudaFreeAsync(p.d_angles, a);
                if (p.d_angle_index) cudaFreeAsync(p.d_angle_index, a);
                if (p.d_grp_target) cudaFreeAsync(p.d_grp_target, a);
            }
        }
    } drain{sc, sx, &slabs};

    CU(d_src_aos.alloc(es * si * n_sources));
    CU(d_src.alloc(es * srows * n_sources));
    CU(d_flags.alloc(sizeof(int) * 2 * K));
    CU(cudaMemsetAsync(d_flags.p, 0, sizeof(int) * 2 * K, sc));
    // The sources go up in chunks, interleaved with the pair lists on the copy stream: a slab's
    // kernels wait (through its `ready` event, recorded behind them) only for the chunks that
    // hold the sources its pairs name, so the first slab starts after a part of the upload
    // (a level sorted by box index: about a third) instead of all of it. Chunks no slab names
    // are never sent.
    static const int kSrcChunks = [] {
        const char* env = std::getenv("SFMM_LEVEL_SRC_CHUNKS");  // tuning: 1 = all sources first
        const int v = env ? std::atoi(env) : 8;
        return v >= 1 && v <= 64 ? v : 8;
    }();
    const int64_t chunk_len = (n_sources + kSrcChunks - 1) / kSrcChunks;
    int chunks_queued = 0;
    auto queue_sources_upto = [&](int64_t last_source) -> cudaError_t {
        const int need = chunk_len > 0 ? (int)std::min<int64_t>(last_source / chunk_len, kSrcChunks - 1) : -1;
        for (; chunks_queued <= need; ++chunks_queued) {
            const int64_t c0 = chunks_queued * chunk_len, c1 = std::min(n_sources, c0 + chunk_len);
            if (c1 <= c0) continue;
            cudaError_t e = cudaMemcpyAsync(d_src_aos.as<Real>() + c0 * si, src_aos + c0 * si, es * si * (c1 - c0),
                                            cudaMemcpyHostToDevice, sc);
            if (e == cudaSuccess)
                e = launch_pack_rows<Real>(d_src_aos.as<Real>() + c0 * si, d_src.as<Real>() + c0 * srows, c1 - c0,
                                           p_in, sc);
            if (e != cudaSuccess) return e;
            h->launches += 1;
        }
        return cudaSuccess;
    };
    for (int k = 0; k < K; ++k) {
        slabs.emplace_back(new Slab(sc, sx));
        Slab& S = *slabs.back();
        const int64_t t0 = cut[k], t1 = cut[k + 1], nt = t1 - t0;
        const int64_t p0 = tgt_ptr[t0], np = tgt_ptr[t1] - p0;
        {  // highest valid source index of the slab (invalid ones are reported by the plan kernel)
            int32_t hi = -1;
            for (int64_t j = p0; j < p0 + np; ++j) hi = std::max(hi, src_index[j]);
            if (hi >= 0) CU(queue_sources_upto(std::min<int64_t>(hi, n_sources - 1)));
        }
        S.t0 = t0;
        S.ostride = round_up32(std::max<int64_t>(nt, 1));
        S.grp_ptr.assign((size_t)nt + 1, 0);
        for (int64_t t = 0; t < nt; ++t)
            S.grp_ptr[(size_t)t + 1] =
                S.grp_ptr[(size_t)t] + (tgt_ptr[t0 + t + 1] - tgt_ptr[t0 + t] + kPlanGroup - 1) / kPlanGroup;
        const int64_t n_groups = S.grp_ptr[(size_t)nt];
        S.grp_target.resize((size_t)std::max<int64_t>(n_groups, 1));
        for (int64_t t = 0; t < nt; ++t)
            for (int64_t g = S.grp_ptr[(size_t)t]; g < S.grp_ptr[(size_t)t + 1]; ++g)
                S.grp_target[(size_t)g] = (int32_t)t;
        std::vector<int64_t> local_ptr((size_t)nt + 1);
        for (int64_t t = 0; t <= nt; ++t) local_ptr[(size_t)t] = tgt_ptr[t0 + t] - p0;
        sfmm_plan& P = S.plan;
        P.h = h, P.n_targets = nt, P.n_pairs = np, P.n_groups = n_groups, P.n_sources = n_sources;
        for (int64_t t = 0; t < nt; ++t)
            P.max_groups = std::max(P.max_groups, S.grp_ptr[(size_t)t + 1] - S.grp_ptr[(size_t)t]);
        const size_t padded = (size_t)std::max<int64_t>(n_groups, 1) * kPlanGroup;
        CU(cudaMallocAsync((void**)&P.d_grp_ptr, sizeof(int64_t) * S.grp_ptr.size(), sc));
        CU(cudaMallocAsync((void**)&P.d_src_index, sizeof(int32_t) * padded, sc));
        CU(cudaMallocAsync(&P.d_shifts, es * padded * 3, sc));
        CU(cudaMallocAsync(&P.d_angles, es * padded * 6, sc));
        CU(cudaMallocAsync((void**)&P.d_angle_index, sizeof(int32_t) * padded, sc));
        CU(cudaMallocAsync((void**)&P.d_grp_target, sizeof(int32_t) * S.grp_target.size(), sc));
        CU(S.tgt.alloc(sizeof(int64_t) * (nt + 1)));
        CU(S.idx.alloc(sizeof(int32_t) * std::max<int64_t>(np, 1)));
        CU(S.sh.alloc(es * 3 * std::max<int64_t>(np, 1)));
        CU(S.out.alloc(es * so * S.ostride));
        CU(S.out_aos.alloc(es * so * std::max<int64_t>(nt, 1)));
        CU(cudaMemcpyAsync(P.d_grp_ptr, S.grp_ptr.data(), sizeof(int64_t) * S.grp_ptr.size(),
                           cudaMemcpyHostToDevice, sc));
        // local_ptr is a temporary: a pageable source is staged before the call returns
        CU(cudaMemcpyAsync(S.tgt.p, local_ptr.data(), sizeof(int64_t) * (nt + 1), cudaMemcpyHostToDevice, sc));
        CU(cudaMemcpyAsync(P.d_grp_target, S.grp_target.data(), sizeof(int32_t) * S.grp_target.size(),
                           cudaMemcpyHostToDevice, sc));
        if (np > 0) {
            CU(cudaMemcpyAsync(S.idx.p, src_index + p0, sizeof(int32_t) * np, cudaMemcpyHostToDevice, sc));
            CU(cudaMemcpyAsync(S.sh.p, shifts + 3 * p0, es * 3 * np, cudaMemcpyHostToDevice, sc));
        }
        CU(launch_build_plan<Real>(S.tgt.as<int64_t>(), P.d_grp_ptr, P.d_grp_target, S.idx.as<int32_t>(),
                                   S.sh.as<Real>(), n_groups, n_sources, kPlanGroup, P.d_src_index,
                                   static_cast<Real*>(P.d_shifts), static_cast<Real*>(P.d_angles),
                                   P.d_angle_index, d_flags.as<int>() + 2 * k, sc));
        h->launches += 4;
        CU(cudaEventCreateWithFlags(&S.ready, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&S.done, cudaEventDisableTiming));
        CU(cudaEventRecord(S.ready, sc));
        // compute of the slab on the second stream
        CU(cudaStreamWaitEvent(sx, S.ready, 0));
        // one SM stays free of the persistent translation kernel: the small kernels of the
        // following slabs (plan building, source packing) run there beside it instead of
        // waiting for it to end, which would stall the copy stream behind them
        const sfmm_status st = accumulate_impl<Real>(h, &P, p_in, p_out, d_src.as<Real>(), srows, LAYOUT_ROWS,
                                                     S.out.as<Real>(), S.ostride, sx, /*reserve_sms=*/1);
        if (st != SFMM_OK) return st;
        CU(launch_unpack_soa<Real>(S.out.as<Real>(), S.out_aos.as<Real>(), nt, p_out, S.ostride, sx));
        h->launches += 1;
        CU(cudaEventRecord(S.done, sx));
    }
    // validation of every slab before the first byte of output moves
    std::vector<int> flags(2 * K, 0);
    CU(cudaMemcpyAsync(flags.data(), d_flags.p, sizeof(int) * 2 * K, cudaMemcpyDeviceToHost, sc));
    CU(cudaStreamSynchronize(sc));
    for (int k = 0; k < K; ++k)
        if (flags[2 * k]) return fail(SFMM_INVALID_ARGUMENT, "source index out of range");
    for (int k = 0; k < K; ++k)
        if (flags[2 * k + 1]) return fail(SFMM_DOMAIN_ERROR, "translation with zero shift vector");
    // downloads on the (now idle) copy stream, each behind its slab's kernels
    for (int k = 0; k < K; ++k) {
        Slab& S = *slabs[k];
        CU(cudaStreamWaitEvent(sc, S.done, 0));
        if (S.plan.n_targets > 0)
            CU(cudaMemcpyAsync(out_aos + S.t0 * so, S.out_aos.p, es * so * S.plan.n_targets,
                               cudaMemcpyDeviceToHost, sc));
    }
    CU(cudaStreamSynchronize(sc));
    return SFMM_OK;
}

}  // namespace

extern "C" {

const char* sfmm_status_string(sfmm_status s) {
    switch (s) {
        case SFMM_OK: return "ok";
        case SFMM_INVALID_ARGUMENT: return "invalid argument";
        case SFMM_DOMAIN_ERROR: return "domain error";
        case SFMM_CUDA_ERROR: return "CUDA error";
        case SFMM_OUT_OF_MEMORY: return "out of device memory";
    }
    return "unknown status";
}

const char* sfmm_last_error(void) { return g_last_error.c_str(); }

int sfmm_max_order(sfmm_precision precision) {
    return precision == SFMM_F32 ? max_order_f32() : max_order_f64();
}

sfmm_status sfmm_create(sfmm_precision precision, int order, int device, int mu, int nu,
                        sfmm_handle** out) {
    if (!out) return fail(SFMM_INVALID_ARGUMENT, "null output pointer");
    *out = nullptr;
    if (precision != SFMM_F64 && precision != SFMM_F32)
        return fail(SFMM_INVALID_ARGUMENT, "unknown precision");
    // kernels.cpp:19-26 (only when the caller passes a config)
    if (mu != 0 && (mu < 2 || (mu & 1) || mu > 32))
        return fail(SFMM_INVALID_ARGUMENT, "kernel_config: mu must be even, 2 <= mu <= 32");
    if (nu != 0 && (nu < 1 || nu > 64))
        return fail(SFMM_INVALID_ARGUMENT, "kernel_config: nu must satisfy 1 <= nu <= 64");
    // operators.cpp:127-132
    if (order < 1) return fail(SFMM_INVALID_ARGUMENT, "order must be >= 1");
    if (order > sfmm_max_order(precision))
        return fail(SFMM_INVALID_ARGUMENT,
                    "order too large: faculty table overflows (cap " +
                        std::to_string(sfmm_max_order(precision)) + ")");
    int count = 0;
    CU(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) return fail(SFMM_INVALID_ARGUMENT, "no such CUDA device");
    DeviceGuard guard(device);
    if (!guard.ok) return fail(SFMM_CUDA_ERROR, "cudaSetDevice failed");

    auto* h = new sfmm_handle;
    h->precision = precision;
    h->order = order;
    h->device = device;
    h->host_tables = SwapTables(order);
    cudaDeviceProp prop;
    cudaError_t e = cudaGetDeviceProperties(&prop, device);
    if (e != cudaSuccess) {
        delete h;
        return cuda_fail(e, "cudaGetDeviceProperties");
    }
    h->sm_count = prop.multiProcessorCount;
    {
        // per-call scratch comes from the stream-ordered pool: keep freed blocks cached
        // instead of returning them to the driver at every synchronisation
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    }
    sfmm_status st = precision == SFMM_F64 ? upload_tables<double>(h, h->td)
                                           : upload_tables<float>(h, h->tf);
    if (st == SFMM_OK) {
        if (cudaMalloc((void**)&h->d_flags, sizeof(int) * kFlagSlots) != cudaSuccess ||
            cudaMemset(h->d_flags, 0, sizeof(int) * kFlagSlots) != cudaSuccess ||
            cudaMallocHost((void**)&h->h_flags, sizeof(int) * kFlagSlots) != cudaSuccess)
            st = fail(SFMM_CUDA_ERROR, "status flag allocation failed");
        for (int i = kFlagSlots - 1; i >= 0; --i) h->free_slots.push_back(i);
    }
    if (st != SFMM_OK) {
        sfmm_destroy(h);
        return st;
    }
    *out = h;
    return SFMM_OK;
}

void sfmm_destroy(sfmm_handle* h) {
    if (!h) return;
    DeviceGuard guard(h->device);
    for (void* p : h->allocations) cudaFree(p);
    if (h->d_flags) cudaFree(h->d_flags);
    if (h->h_flags) cudaFreeHost(h->h_flags);
    delete h;
}

int sfmm_order(const sfmm_handle* h) { return h ? h->order : 0; }
int sfmm_device(const sfmm_handle* h) { return h ? h->device : -1; }
int sfmm_accumulation_unit(const sfmm_handle* h, int p_in, int p_out) {
    if (!h || p_in < 1 || p_out < 1 || std::max(p_in, p_out) > h->order) return 0;
    if (h->precision == SFMM_F64) {
        TranslateArgs<double> a;
        a.kind = KIND_M2L, a.p_in = p_in, a.p_out = p_out, a.variant = h->variant, a.precise = h->precise;
        a.src_index = h->d_flags;  // any non-null pointer: accumulate mode (never dereferenced)
        return translate_group_size<double>(h->td, a);
    }
    TranslateArgs<float> a;
    a.kind = KIND_M2L, a.p_in = p_in, a.p_out = p_out, a.variant = h->variant, a.precise = h->precise;
    a.src_index = h->d_flags;
    return translate_group_size<float>(h->tf, a);
}

int64_t sfmm_launch_count(const sfmm_handle* h) { return h ? h->launches.load() : 0; }

sfmm_status sfmm_measure_fma_peak(sfmm_handle* h, double* tflops) {
    if (!h || !tflops) return fail(SFMM_INVALID_ARGUMENT, "null argument");
    DeviceGuard guard(h->device);
    if (h->precision == SFMM_F64)
        CU(measure_fma_peak<double>(h->sm_count, tflops));
    else
        CU(measure_fma_peak<float>(h->sm_count, tflops));
    h->launches += 4;
    return SFMM_OK;
}

sfmm_status sfmm_measure_dmma_peak(sfmm_handle* h, double* tflops) {
    if (!h || !tflops) return fail(SFMM_INVALID_ARGUMENT, "null argument");
    DeviceGuard guard(h->device);
    CU(measure_dmma_peak(h->sm_count, tflops));
    h->launches += 4;
    return SFMM_OK;
}

sfmm_status sfmm_set_option(sfmm_handle* h, const char* name, int64_t value) {
    if (!h || !name) return fail(SFMM_INVALID_ARGUMENT, "null handle or option name");
    if (std::strcmp(name, "level_slab_pairs") == 0) {
        if (value < 64) return fail(SFMM_INVALID_ARGUMENT, "level_slab_pairs must be >= 64");
        h->level_slab_pairs = value;
        return SFMM_OK;
    }
    if (std::strcmp(name, "precise") == 0) {
        if (value && h->precision != SFMM_F64)
            return fail(SFMM_INVALID_ARGUMENT, "the precise mode is double precision only");
        h->precise = value != 0;
        return SFMM_OK;
    }
    if (std::strcmp(name, "accumulate_plain") == 0) {
        h->accumulate_plain = value != 0;
        return SFMM_OK;
    }
    if (std::strcmp(name, "kernel_variant") == 0) {
        if (value < 0 || value > 4) return fail(SFMM_INVALID_ARGUMENT, "kernel_variant must be 0..4");
        h->variant = (int)value;
        return SFMM_OK;
    }
    if (std::strcmp(name, "phase_clocks") == 0) {
        // value = device address of 8 int64 counters (0 switches the probe off)
        h->d_phase_clocks = reinterpret_cast<long long*>(value);
        return SFMM_OK;
    }
    return fail(SFMM_INVALID_ARGUMENT, std::string("unknown option ") + name);
}

sfmm_status sfmm_get_swap_tables(const sfmm_handle* h, int n, double* f, double* g) {
    if (!h || n < 0 || n >= h->order) return fail(SFMM_INVALID_ARGUMENT, "row out of range");
    const size_t sz = (size_t)(n + 1) * (n + 1);
    const bool single = h->precision == SFMM_F32;
    for (size_t i = 0; i < sz; ++i) {
        // operators.cpp:152-155: the library precision sees the double tables cast
        if (f) f[i] = single ? (double)(float)h->host_tables.f[n][i] : h->host_tables.f[n][i];
        if (g) g[i] = single ? (double)(float)h->host_tables.g[n][i] : h->host_tables.g[n][i];
    }
    return SFMM_OK;
}

sfmm_status sfmm_get_faculties(const sfmm_handle* h, double* fac, double* inv) {
    if (!h) return fail(SFMM_INVALID_ARGUMENT, "null handle");
    if (fac) std::copy(h->fac.begin(), h->fac.end(), fac);
    if (inv) std::copy(h->inv.begin(), h->inv.end(), inv);
    return SFMM_OK;
}

sfmm_status sfmm_host_swap_tables(int n, double* f, double* g) {
    if (n < 0 || n >= max_order_f64()) return fail(SFMM_INVALID_ARGUMENT, "row out of range");
    const SwapTables t(n + 1);
    if (f) std::copy(t.f[n].begin(), t.f[n].end(), f);
    if (g) std::copy(t.g[n].begin(), t.g[n].end(), g);
    return SFMM_OK;
}

sfmm_status sfmm_host_faculties(sfmm_precision precision, int order, double* fac, double* inv) {
    if (precision != SFMM_F64 && precision != SFMM_F32)
        return fail(SFMM_INVALID_ARGUMENT, "unknown precision");
    if (order < 1 || order > sfmm_max_order(precision))
        return fail(SFMM_INVALID_ARGUMENT, "order out of range");
    if (precision == SFMM_F64) {
        std::vector<double> a, b;
        build_faculties<double>(order, a, b);
        if (fac) std::copy(a.begin(), a.end(), fac);
        if (inv) std::copy(b.begin(), b.end(), inv);
    } else {
        std::vector<float> a, b;
        build_faculties<float>(order, a, b);
        if (fac) std::copy(a.begin(), a.end(), fac);
        if (inv) std::copy(b.begin(), b.end(), inv);
    }
    return SFMM_OK;
}

sfmm_status sfmm_translate_host(sfmm_handle* h, sfmm_kind kind, int64_t n, int p_in, int p_out,
                                const void* in_aos, const void* shifts, void* out_aos) {
    if (!h) return fail(SFMM_INVALID_ARGUMENT, "null handle");
    if (n < 0) return fail(SFMM_INVALID_ARGUMENT, "negative batch size");
    if (n == 0) return SFMM_OK;  // pipeline.cpp:280
    if (!in_aos || !shifts || !out_aos)
        return fail(SFMM_INVALID_ARGUMENT, "translation request with null solid");
    const sfmm_status st = check_orders(h, kind, p_in, p_out);
    if (st != SFMM_OK) return st;
    DeviceGuard guard(h->device);
    if (h->precision == SFMM_F64)
        return translate_host_impl<double>(h, kind, n, p_in, p_out, (const double*)in_aos,
                                           (const double*)shifts, (double*)out_aos);
    return translate_host_impl<float>(h, kind, n, p_in, p_out, (const float*)in_aos,
                                      (const float*)shifts, (float*)out_aos);
}

sfmm_status sfmm_translate_host_mixed(sfmm_handle* h, sfmm_kind kind, int64_t n, const int* p_in,
                                      const int* p_out, const void* in, const int64_t* in_offset,
                                      const void* shifts, void* out, const int64_t* out_offset) {
    if (!h) return fail(SFMM_INVALID_ARGUMENT, "null handle");
    if (n < 0) return fail(SFMM_INVALID_ARGUMENT, "negative batch size");
    if (n == 0) return SFMM_OK;
    if (!p_in || !p_out || !in || !in_offset || !shifts || !out || !out_offset)
        return fail(SFMM_INVALID_ARGUMENT, "translation request with null solid");
    if (kind < 0 || kind > 2) return fail(SFMM_INVALID_ARGUMENT, "unknown translation kind");
    DeviceGuard guard(h->device);
    if (h->precision == SFMM_F64)
        return translate_host_mixed_impl<double>(h, kind, n, p_in, p_out, (const double*)in,
                                                 in_offset, (const double*)shifts, (double*)out,
                                                 out_offset);
    return translate_host_mixed_impl<float>(h, kind, n, p_in, p_out, (const float*)in, in_offset,
                                            (const float*)shifts, (float*)out, out_offset);
}

sfmm_status sfmm_translate_soa(sfmm_handle* h, sfmm_kind kind, int64_t n, int p_in, int p_out,
                               const void* d_in, int64_t in_stride, const void* d_shifts,
                               void* d_out, int64_t out_stride, void* stream, int flags) {
    if (!h) return fail(SFMM_INVALID_ARGUMENT, "null handle");
    if (n < 0) return fail(SFMM_INVALID_ARGUMENT, "negative batch size");
    if (n == 0) return SFMM_OK;
    if (!d_in || !d_shifts || !d_out)
        return fail(SFMM_INVALID_ARGUMENT, "translation request with null solid");
    if (in_stride < n || out_stride < n)
        return fail(SFMM_INVALID_ARGUMENT, "batch stride smaller than the batch");
    const sfmm_status st = check_orders(h, kind, p_in, p_out);
    if (st != SFMM_OK) return st;
    DeviceGuard guard(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (h->precision == SFMM_F64)
        return translate_soa_impl<double>(h, kind, n, p_in, p_out, (const double*)d_in, in_stride,
                                          (const double*)d_shifts, (double*)d_out, out_stride, s,
                                          flags, false);
    return translate_soa_impl<float>(h, kind, n, p_in, p_out, (const float*)d_in, in_stride,
                                     (const float*)d_shifts, (float*)d_out, out_stride, s, flags,
                                     false);
}

sfmm_status sfmm_stream_status(sfmm_handle* h, void* stream) {
    if (!h) return fail(SFMM_INVALID_ARGUMENT, "null handle");
    DeviceGuard guard(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // only the calls issued on this stream: the others have not necessarily run yet and
    // keep their slots until their own stream is queried
    std::vector<int> slots;
    {
        std::lock_guard<std::mutex> lk(h->async_mutex);
        auto keep = h->pending.begin();
        for (auto it = h->pending.begin(); it != h->pending.end(); ++it) {
            if (it->stream == s) slots.push_back(it->slot);
            else *keep++ = *it;
        }
        h->pending.erase(keep, h->pending.end());
    }
    std::vector<int> values(kFlagSlots, 0);
    cudaError_t e = cudaSuccess;
    if (!slots.empty())
        e = cudaMemcpyAsync(values.data(), h->d_flags, sizeof(int) * kFlagSlots, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    bool bad = false;
    for (int slot : slots) {
        if (values[slot] != 0 || e != cudaSuccess) {
            bad = bad || values[slot] != 0;
            cudaMemsetAsync(h->d_flags + slot, 0, sizeof(int), s);  // free slots are zero
        }
    }
    if (bad || e != cudaSuccess) cudaStreamSynchronize(s);
    for (int slot : slots) release_slot(h, slot);
    if (e != cudaSuccess) return cuda_fail(e, "sfmm_stream_status");
    if (bad) return fail(SFMM_DOMAIN_ERROR, "translation with zero shift vector");
    return SFMM_OK;
}

sfmm_status sfmm_pack_soa(sfmm_handle* h, int64_t n, int p, const void* d_aos, void* d_soa,
                          int64_t stride, void* stream) {
    if (!h || !d_aos || !d_soa || p < 1 || n < 0 || stride < n)
        return fail(SFMM_INVALID_ARGUMENT, "bad pack_soa arguments");
    DeviceGuard guard(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    h->launches += 1;
    if (h->precision == SFMM_F64)
        CU(launch_pack_soa<double>((const double*)d_aos, (double*)d_soa, n, p, stride, s));
    else
        CU(launch_pack_soa<float>((const float*)d_aos, (float*)d_soa, n, p, stride, s));
    return SFMM_OK;
}

int64_t sfmm_rows_len(int p) { return p < 1 ? 0 : rows_off(p); }

// ---- particle <-> expansion steps -----------------------------------------
int sfmm_harmonics_max_order(void) { return harmonics_max_order(); }

static bool harmonics_layout_ok(int layout) {
    return layout == SFMM_LAYOUT_SOA || layout == SFMM_LAYOUT_ROWS || layout == SFMM_LAYOUT_AOS;
}

sfmm_status sfmm_p2m(sfmm_handle* h, int64_t n_boxes, const int64_t* d_box_ptr, const void* d_charges,
                     const void* d_centers, int order, int layout, void* d_out, int64_t out_stride,
                     void* stream) {
    if (!h || n_boxes < 0 || !harmonics_layout_ok(layout))
        return fail(SFMM_INVALID_ARGUMENT, "bad p2m arguments");
    if (order < 1 || order > h->order) return fail(SFMM_INVALID_ARGUMENT, "order out of range for this handle");
    if (n_boxes == 0) return SFMM_OK;
    if (!d_box_ptr || !d_charges || !d_centers || !d_out) return fail(SFMM_INVALID_ARGUMENT, "null pointer");
    if (layout == SFMM_LAYOUT_SOA && out_stride < n_boxes)
        return fail(SFMM_INVALID_ARGUMENT, "stride smaller than the batch");
    DeviceGuard guard(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    h->launches += 1;
    if (h->precision == SFMM_F64)
        CU(launch_p2m<double>(d_box_ptr, (const double*)d_charges, (const double*)d_centers, n_boxes, order,
                              layout, (double*)d_out, out_stride, s));
    else
        CU(launch_p2m<float>(d_box_ptr, (const float*)d_charges, (const float*)d_centers, n_boxes, order,
                             layout, (float*)d_out, out_stride, s));
    return SFMM_OK;
}

sfmm_status sfmm_eval_local(sfmm_handle* h, int64_t n_points, const int32_t* d_point_box,
                            const void* d_points, const void* d_centers, int64_t n_boxes, int order,
                            int layout, const void* d_locals, int64_t stride, void* d_out, void* stream) {
    if (!h || n_points < 0 || n_boxes < 0 || !harmonics_layout_ok(layout))
        return fail(SFMM_INVALID_ARGUMENT, "bad eval_local arguments");
    if (order < 1 || order > h->order) return fail(SFMM_INVALID_ARGUMENT, "order out of range for this handle");
    if (n_points == 0) return SFMM_OK;
    if (!d_points || !d_centers || !d_locals || !d_out) return fail(SFMM_INVALID_ARGUMENT, "null pointer");
    if (layout == SFMM_LAYOUT_SOA && stride < n_boxes)
        return fail(SFMM_INVALID_ARGUMENT, "stride smaller than the batch");
    DeviceGuard guard(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    h->launches += 1;
    if (h->precision == SFMM_F64)
        CU(launch_eval_local<double>(d_point_box, (const double*)d_points, (const double*)d_centers, n_points,
                                     n_boxes, order, layout, (const double*)d_locals, stride, (double*)d_out, s));
    else
        CU(launch_eval_local<float>(d_point_box, (const float*)d_points, (const float*)d_centers, n_points,
                                    n_boxes, order, layout, (const float*)d_locals, stride, (float*)d_out, s));
    return SFMM_OK;
}

// host-buffer forms (the reference's p2m / eval_local take host objects, harmonics.hpp:36-51)
sfmm_status sfmm_p2m_host(sfmm_handle* h, int64_t n_boxes, const int64_t* box_ptr, const void* charges,
                          const void* centers, int order, void* out_aos) {
    if (!h || n_boxes < 0) return fail(SFMM_INVALID_ARGUMENT, "bad p2m arguments");
    if (n_boxes == 0) return SFMM_OK;
    if (!box_ptr || !centers || !out_aos) return fail(SFMM_INVALID_ARGUMENT, "null pointer");
    for (int64_t b = 0; b < n_boxes; ++b)
        if (box_ptr[b + 1] < box_ptr[b]) return fail(SFMM_INVALID_ARGUMENT, "box_ptr must be non-decreasing");
    const int64_t nq = box_ptr[n_boxes] - box_ptr[0];
    if (nq > 0 && !charges) return fail(SFMM_INVALID_ARGUMENT, "null pointer");
    DeviceGuard guard(h->device);
    cudaStream_t s = host_stream(h->device);
    const size_t es = h->precision == SFMM_F64 ? 8 : 4;
    DevBuf d_ptr(s), d_q(s), d_c(s), d_out(s);
    CU(d_ptr.alloc(sizeof(int64_t) * (n_boxes + 1)));
    CU(d_q.alloc(es * 4 * std::max<int64_t>(nq, 1)));
    CU(d_c.alloc(es * 3 * n_boxes));
    CU(d_out.alloc(es * solid_len(order) * n_boxes));
    std::vector<int64_t> rel((size_t)n_boxes + 1);
    for (int64_t b = 0; b <= n_boxes; ++b) rel[(size_t)b] = box_ptr[b] - box_ptr[0];
    CU(cudaMemcpyAsync(d_ptr.p, rel.data(), sizeof(int64_t) * (n_boxes + 1), cudaMemcpyHostToDevice, s));
    if (nq > 0)
        CU(cudaMemcpyAsync(d_q.p, (const char*)charges + es * 4 * box_ptr[0], es * 4 * nq, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(d_c.p, centers, es * 3 * n_boxes, cudaMemcpyHostToDevice, s));
    const sfmm_status st = sfmm_p2m(h, n_boxes, d_ptr.as<int64_t>(), d_q.p, d_c.p, order, SFMM_LAYOUT_AOS,
                                    d_out.p, 0, s);
    if (st != SFMM_OK) return st;
    CU(cudaMemcpyAsync(out_aos, d_out.p, es * solid_len(order) * n_boxes, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    return SFMM_OK;
}

sfmm_status sfmm_eval_local_host(sfmm_handle* h, int64_t n_points, const int32_t* point_box,
                                 const void* points, const void* centers, int64_t n_boxes, int order,
                                 const void* locals_aos, void* out) {
    if (!h || n_points < 0 || n_boxes < 0) return fail(SFMM_INVALID_ARGUMENT, "bad eval_local arguments");
    if (n_points == 0) return SFMM_OK;
    if (!points || !centers || !locals_aos || !out) return fail(SFMM_INVALID_ARGUMENT, "null pointer");
    if (!point_box && n_boxes < n_points) return fail(SFMM_INVALID_ARGUMENT, "one box per point expected");
    if (point_box)
        for (int64_t i = 0; i < n_points; ++i)
            if (point_box[i] < 0 || point_box[i] >= n_boxes)
                return fail(SFMM_INVALID_ARGUMENT, "box index out of range");
    DeviceGuard guard(h->device);
    cudaStream_t s = host_stream(h->device);
    const size_t es = h->precision == SFMM_F64 ? 8 : 4;
    DevBuf d_pb(s), d_x(s), d_c(s), d_l(s), d_out(s);
    CU(d_pb.alloc(sizeof(int32_t) * n_points));
    CU(d_x.alloc(es * 3 * n_points));
    CU(d_c.alloc(es * 3 * n_boxes));
    CU(d_l.alloc(es * solid_len(order) * n_boxes));
    CU(d_out.alloc(es * n_points));
    if (point_box) CU(cudaMemcpyAsync(d_pb.p, point_box, sizeof(int32_t) * n_points, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(d_x.p, points, es * 3 * n_points, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(d_c.p, centers, es * 3 * n_boxes, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(d_l.p, locals_aos, es * solid_len(order) * n_boxes, cudaMemcpyHostToDevice, s));
    const sfmm_status st = sfmm_eval_local(h, n_points, point_box ? d_pb.as<int32_t>() : nullptr, d_x.p, d_c.p,
                                           n_boxes, order, SFMM_LAYOUT_AOS, d_l.p, 0, d_out.p, s);
    if (st != SFMM_OK) return st;
    CU(cudaMemcpyAsync(out, d_out.p, es * n_points, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    return SFMM_OK;
}

sfmm_status sfmm_pack_rows(sfmm_handle* h, int64_t n, int p, const void* d_aos, void* d_rows,
                           void* stream) {
    if (!h || !d_aos || !d_rows || p < 1 || n < 0)
        return fail(SFMM_INVALID_ARGUMENT, "bad pack_rows arguments");
    DeviceGuard guard(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    h->launches += 1;
    if (h->precision == SFMM_F64)
        CU(launch_pack_rows<double>((const double*)d_aos, (double*)d_rows, n, p, s));
    else
        CU(launch_pack_rows<float>((const float*)d_aos, (float*)d_rows, n, p, s));
    return SFMM_OK;
}

sfmm_status sfmm_unpack_soa(sfmm_handle* h, int64_t n, int p, const void* d_soa, int64_t stride,
                            void* d_aos, void* stream) {
    if (!h || !d_aos || !d_soa || p < 1 || n < 0 || stride < n)
        return fail(SFMM_INVALID_ARGUMENT, "bad unpack_soa arguments");
    DeviceGuard guard(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    h->launches += 1;
    if (h->precision == SFMM_F64)
        CU(launch_unpack_soa<double>((const double*)d_soa, (double*)d_aos, n, p, stride, s));
    else
        CU(launch_unpack_soa<float>((const float*)d_soa, (float*)d_aos, n, p, stride, s));
    return SFMM_OK;
}

sfmm_status sfmm_plan_create(sfmm_handle* h, int64_t n_targets, const int64_t* tgt_ptr,
                             const int32_t* src_index, const void* shifts, int64_t n_sources,
                             sfmm_plan** out) {
    if (!out) return fail(SFMM_INVALID_ARGUMENT, "null output pointer");
    *out = nullptr;
    if (!h || n_targets < 0 || n_sources < 0 || !tgt_ptr)
        return fail(SFMM_INVALID_ARGUMENT, "bad plan arguments");
    if (tgt_ptr[0] != 0) return fail(SFMM_INVALID_ARGUMENT, "tgt_ptr[0] must be 0");
    if (tgt_ptr[n_targets] > 0 && (!src_index || !shifts))
        return fail(SFMM_INVALID_ARGUMENT, "translation request with null solid");
    DeviceGuard guard(h->device);
    auto* plan = new sfmm_plan;
    const sfmm_status st =
        h->precision == SFMM_F64
            ? plan_create_impl<double>(h, n_targets, tgt_ptr, src_index, (const double*)shifts,
                                       n_sources, plan)
            : plan_create_impl<float>(h, n_targets, tgt_ptr, src_index, (const float*)shifts,
                                      n_sources, plan);
    if (st != SFMM_OK) {
        sfmm_plan_destroy(plan);
        return st;
    }
    *out = plan;
    return SFMM_OK;
}

void sfmm_plan_destroy(sfmm_plan* plan) {
    if (!plan) return;
    if (plan->h) {
        DeviceGuard guard(plan->h->device);
        // ordered behind the most recent accumulate call that used the plan (calls on several
        // streams at once: synchronise the others before destroying, solidfmm_b200.h)
        cudaStream_t s = plan->last_stream;
        if (plan->d_grp_ptr) cudaFreeAsync(plan->d_grp_ptr, s);
        if (plan->d_src_index) cudaFreeAsync(plan->d_src_index, s);
        if (plan->d_shifts) cudaFreeAsync(plan->d_shifts, s);
        if (plan->d_angles) cudaFreeAsync(plan->d_angles, s);
        if (plan->d_angle_index) cudaFreeAsync(plan->d_angle_index, s);
        if (plan->d_grp_target) cudaFreeAsync(plan->d_grp_target, s);
    }
    delete plan;
}

int64_t sfmm_plan_pairs(const sfmm_plan* plan) { return plan ? plan->n_pairs : 0; }

sfmm_status sfmm_m2l_accumulate(sfmm_handle* h, const sfmm_plan* plan, int p_in, int p_out,
                                const void* d_src, int64_t src_stride, void* d_out,
                                int64_t out_stride, void* stream) {
    if (!h || !plan || plan->h != h) return fail(SFMM_INVALID_ARGUMENT, "plan/handle mismatch");
    if (!d_src || !d_out) return fail(SFMM_INVALID_ARGUMENT, "translation request with null solid");
    if (src_stride < plan->n_sources || out_stride < plan->n_targets)
        return fail(SFMM_INVALID_ARGUMENT, "batch stride smaller than the batch");
    const sfmm_status st = check_orders(h, SFMM_M2L, p_in, p_out);
    if (st != SFMM_OK) return st;
    DeviceGuard guard(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (h->precision == SFMM_F64)
        return accumulate_impl<double>(h, plan, p_in, p_out, (const double*)d_src, src_stride,
                                       LAYOUT_SOA, (double*)d_out, out_stride, s);
    return accumulate_impl<float>(h, plan, p_in, p_out, (const float*)d_src, src_stride,
                                  LAYOUT_SOA, (float*)d_out, out_stride, s);
}

sfmm_status sfmm_m2l_accumulate_rows(sfmm_handle* h, const sfmm_plan* plan, int p_in, int p_out,
                                     const void* d_src_rows, void* d_out, int64_t out_stride,
                                     void* stream) {
    if (!h || !plan || plan->h != h) return fail(SFMM_INVALID_ARGUMENT, "plan/handle mismatch");
    if (!d_src_rows || !d_out)
        return fail(SFMM_INVALID_ARGUMENT, "translation request with null solid");
    if (out_stride < plan->n_targets)
        return fail(SFMM_INVALID_ARGUMENT, "batch stride smaller than the batch");
    if (reinterpret_cast<uintptr_t>(d_src_rows) % 32)
        return fail(SFMM_INVALID_ARGUMENT, "rows-layout sources must be 32-byte aligned");
    const sfmm_status st = check_orders(h, SFMM_M2L, p_in, p_out);
    if (st != SFMM_OK) return st;
    DeviceGuard guard(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (h->precision == SFMM_F64)
        return accumulate_impl<double>(h, plan, p_in, p_out, (const double*)d_src_rows,
                                       rows_off(p_in), LAYOUT_ROWS, (double*)d_out, out_stride, s);
    return accumulate_impl<float>(h, plan, p_in, p_out, (const float*)d_src_rows, rows_off(p_in),
                                  LAYOUT_ROWS, (float*)d_out, out_stride, s);
}

sfmm_status sfmm_m2l_level_host(sfmm_handle* h, int64_t n_targets, const int64_t* tgt_ptr,
                                const int32_t* src_index, const void* shifts, int64_t n_sources, int p_in,
                                int p_out, const void* src_aos, void* out_aos) {
    if (!h || n_targets < 0 || n_sources < 0 || !tgt_ptr)
        return fail(SFMM_INVALID_ARGUMENT, "bad level arguments");
    if (tgt_ptr[0] != 0) return fail(SFMM_INVALID_ARGUMENT, "tgt_ptr[0] must be 0");
    if ((tgt_ptr[n_targets] > 0 && (!src_index || !shifts)) || !src_aos || !out_aos)
        return fail(SFMM_INVALID_ARGUMENT, "translation request with null solid");
    const sfmm_status st = check_orders(h, SFMM_M2L, p_in, p_out);
    if (st != SFMM_OK) return st;
    DeviceGuard guard(h->device);
    if (h->precision == SFMM_F64)
        return level_host_impl<double>(h, n_targets, tgt_ptr, src_index, (const double*)shifts, n_sources,
                                       p_in, p_out, (const double*)src_aos, (double*)out_aos);
    return level_host_impl<float>(h, n_targets, tgt_ptr, src_index, (const float*)shifts, n_sources, p_in,
                                  p_out, (const float*)src_aos, (float*)out_aos);
}

sfmm_status sfmm_m2l_accumulate_host(sfmm_handle* h, const sfmm_plan* plan, int p_in, int p_out,
                                     const void* src_aos, void* out_aos) {
    if (!h || !plan || plan->h != h) return fail(SFMM_INVALID_ARGUMENT, "plan/handle mismatch");
    if (!src_aos || !out_aos)
        return fail(SFMM_INVALID_ARGUMENT, "translation request with null solid");
    const sfmm_status st = check_orders(h, SFMM_M2L, p_in, p_out);
    if (st != SFMM_OK) return st;
    DeviceGuard guard(h->device);
    if (h->precision == SFMM_F64)
        return accumulate_host_impl<double>(h, plan, p_in, p_out, (const double*)src_aos,
                                            (double*)out_aos);
    return accumulate_host_impl<float>(h, plan, p_in, p_out, (const float*)src_aos,
                                       (float*)out_aos);
}

}  // extern "C"

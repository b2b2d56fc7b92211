// Kernel launchers (sm_100a). Compiled with -fmad=false: see device_math.cuh.
#include <algorithm>

#include "kernel_generic.cuh"
#include "sfmm_internal.hpp"

namespace sfmm {

namespace {

template <typename Real>
__global__ void check_shifts_kernel(const Real* __restrict__ shifts, int64_t n, int* flag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    bool bad = false;
    if (i < n) bad = shift_is_degenerate(shifts[3 * i], shifts[3 * i + 1], shifts[3 * i + 2]);
    if (__syncthreads_or(bad) && threadIdx.x == 0) *flag = 1;
}

// 32x32 tile transpose between AoS [b][S] and SoA [c][stride].
template <typename Real, bool TO_SOA>
__global__ void repack_kernel(const Real* __restrict__ src, Real* __restrict__ dst, int64_t n,
                              int S, int64_t stride) {
    __shared__ Real tile[32][33];
    const int64_t b0 = (int64_t)blockIdx.x * 32;
    const int c0 = blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    if (TO_SOA) {
        for (int r = ty; r < 32; r += 8) {
            const int64_t b = b0 + r;
            const int c = c0 + tx;
            if (b < n && c < S) tile[r][tx] = src[b * S + c];
        }
        __syncthreads();
        for (int r = ty; r < 32; r += 8) {
            const int c = c0 + r;
            const int64_t b = b0 + tx;
            if (b < n && c < S) dst[(int64_t)c * stride + b] = tile[tx][r];
        }
    } else {
        for (int r = ty; r < 32; r += 8) {
            const int c = c0 + r;
            const int64_t b = b0 + tx;
            if (b < n && c < S) tile[r][tx] = src[(int64_t)c * stride + b];
        }
        __syncthreads();
        for (int r = ty; r < 32; r += 8) {
            const int64_t b = b0 + r;
            const int c = c0 + tx;
            if (b < n && c < S) dst[b * S + c] = tile[tx][r];
        }
    }
}

// Accumulation plan: pads the pair list of every target to whole groups of 64 lanes
// (idle lanes: source -1, benign shift (0,0,1)) and validates it on the way.
// flags[0]: source index out of range, flags[1]: degenerate shift.
template <typename Real>
__global__ void build_plan_kernel(const int64_t* __restrict__ tgt_ptr,
                                  const int64_t* __restrict__ grp_ptr,
                                  const int32_t* __restrict__ grp_target,
                                  const int32_t* __restrict__ src_index,
                                  const Real* __restrict__ shifts, int64_t n_groups,
                                  int64_t n_sources, int group, int32_t* __restrict__ out_index,
                                  Real* __restrict__ out_shifts, int* flags) {
    const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (d >= n_groups * group) return;
    const int64_t g = d / group;
    const int t = grp_target[g];
    const int64_t j = tgt_ptr[t] + (g - grp_ptr[t]) * group + (d - g * group);
    int32_t idx = -1;
    Real x = 0, y = 0, z = 1;
    if (j < tgt_ptr[t + 1]) {
        idx = src_index[j];
        x = shifts[3 * j];
        y = shifts[3 * j + 1];
        z = shifts[3 * j + 2];
        if (idx < 0 || idx >= n_sources) {
            flags[0] = 1;
            idx = -1;
        }
        if (shift_is_degenerate(x, y, z)) flags[1] = 1;
    }
    out_index[d] = idx;
    out_shifts[3 * d] = x;
    out_shifts[3 * d + 1] = y;
    out_shifts[3 * d + 2] = z;
}

// ---- plan geometry: one decomposition per DISTINCT shift ------------------------------------
// A level of a uniform octree has a few hundred distinct shifts for millions of pairs; the
// decomposed shifts (geometry.cpp:11-30) are stored once per distinct shift and every lane
// carries an index (4 bytes instead of 6 reals of DRAM traffic per pair and launch). Shifts are
// compared by bit pattern. Lists with more distinct shifts than the table holds fall back to
// one entry per lane (angle_index = identity); the choice is made on the device, so the
// plan-building stream never waits for the host.
constexpr int kDedupSlots = 1 << 16;   // open-addressing table of representative lanes
constexpr int kDedupProbes = 64;

template <typename Real>
__device__ __forceinline__ bool same_shift(const Real* s, int64_t a, int64_t b) {
    using Bits = typename std::conditional<sizeof(Real) == 8, unsigned long long, unsigned int>::type;
    const Bits* u = reinterpret_cast<const Bits*>(s);
    return u[3 * a] == u[3 * b] && u[3 * a + 1] == u[3 * b + 1] && u[3 * a + 2] == u[3 * b + 2];
}

// rep[d] = lane whose shift equals that of lane d and that won the table slot; state[1] is
// raised when the list does not fit
template <typename Real>
__global__ void dedup_rep_kernel(const Real* __restrict__ shifts, int64_t n, int* table,
                                 int32_t* __restrict__ rep, int* state) {
    const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (d >= n) return;
    unsigned long long h = 0x9E3779B97F4A7C15ull;
    for (int k = 0; k < 3; ++k) {
        unsigned long long v;
        if (sizeof(Real) == 8) v = (unsigned long long)__double_as_longlong((double)shifts[3 * d + k]);
        else v = (unsigned long long)__float_as_uint((float)shifts[3 * d + k]);
        h = (h ^ v) * 0xFF51AFD7ED558CCDull;
        h ^= h >> 29;
    }
    unsigned slot = (unsigned)(h >> 20) & (kDedupSlots - 1);
    int32_t r = -1;
    for (int probe = 0; probe < kDedupProbes; ++probe) {
        const int cur = atomicCAS(&table[slot], -1, (int)d);
        if (cur == -1) {
            r = (int32_t)d;
            break;
        }
        if (same_shift(shifts, d, (int64_t)cur)) {
            r = cur;
            break;
        }
        slot = (slot + 1) & (kDedupSlots - 1);
    }
    if (r < 0) {
        state[1] = 1;
        r = (int32_t)d;
    }
    rep[d] = r;
}

// representatives take a slot of the compact table and decompose their shift into it; when
// the list did not fit, every lane decomposes its own shift (slot = lane)
template <typename Real>
__global__ void dedup_assign_kernel(const Real* __restrict__ shifts, int64_t n,
                                    const int32_t* __restrict__ rep, int32_t* __restrict__ uid,
                                    Real* __restrict__ angles, int* state) {
    const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (d >= n) return;
    const bool per_lane = state[1] != 0;
    int64_t slot = d;
    if (!per_lane) {
        if (rep[d] != d) return;
        const int id = atomicAdd(&state[0], 1);
        slot = id;
        uid[d] = id;
    }
    const Angles<Real> ang = decompose_angles(shifts[3 * d], shifts[3 * d + 1], shifts[3 * d + 2]);
    angles[slot] = ang.rn;
    angles[n + slot] = ang.ca;
    angles[2 * n + slot] = ang.sa;
    angles[3 * n + slot] = ang.cb;
    angles[4 * n + slot] = ang.sb;
    angles[5 * n + slot] = Real(1) / ang.rn;
}

template <typename Real>
__global__ void dedup_index_kernel(int64_t n, const int32_t* __restrict__ rep,
                                   const int32_t* __restrict__ uid, int32_t* __restrict__ angle_index,
                                   const int* state) {
    const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (d >= n) return;
    angle_index[d] = state[1] ? (int32_t)d : uid[rep[d]];
}

template <typename Real>
__global__ void reduce_groups_kernel(const Real* __restrict__ partial, int64_t n_groups,
                                     const int64_t* __restrict__ grp_ptr, int per,
                                     int64_t n_targets, int S, Real* __restrict__ out,
                                     int64_t out_stride) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (t >= n_targets) return;
    Real acc = Real(0);
    // Im(C_n^0) planes are never written by the translation kernel
    int n = 0;
    while ((n + 1) * (n + 2) <= c) ++n;
    const bool im0 = (c == n * (n + 1) + 1);
    if (!im0) {
        const int64_t g0 = grp_ptr[t] * per, g1 = grp_ptr[t + 1] * per;
        for (int64_t g = g0; g < g1; ++g) acc += partial[(int64_t)c * n_groups + g];
    }
    out[(int64_t)c * out_stride + t] = acc;
}

template <typename Real>
__global__ void zero_unwritten_kernel(const int64_t* __restrict__ grp_ptr, int64_t n_targets, int P,
                                      Real* __restrict__ out, int64_t out_stride) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n_targets) return;
    if (grp_ptr[t + 1] == grp_ptr[t]) {
        for (int c = 0; c < P * (P + 1); ++c) out[(int64_t)c * out_stride + t] = Real(0);
    } else {
        for (int n = 0; n < P; ++n) out[(int64_t)(aos_re(n, 0) + 1) * out_stride + t] = Real(0);
    }
}

// FMA-pipe peak probe (roofline denominator measured next to the benchmark).
template <typename Real>
__global__ void fma_peak_kernel(Real* out, int iters, Real a, Real b) {
    Real x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = Real(threadIdx.x + j);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = fma_(x[j], a, b);
    }
    Real s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// FP64 tensor-core peak probe: back-to-back mma.m8n8k4.f64 on 8 accumulator pairs per warp
__global__ void dmma_peak_kernel(double* out, int iters, double a, double b) {
    double d[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) d[j][0] = d[j][1] = double(threadIdx.x + j);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(d[j][0]), "+d"(d[j][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// opt-in shared memory of the CURRENT device (handles live on any device)
int smem_optin_limit() {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return v;
}

}  // namespace

template <typename Real>
cudaError_t measure_fma_peak(int sm_count, double* tflops) {
    const int block = 256, grid = sm_count * 4, iters = 4096;
    Real* out = nullptr;
    cudaError_t e = cudaMalloc((void**)&out, sizeof(Real) * (size_t)grid * block);
    if (e != cudaSuccess) return e;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
        cudaEventRecord(e0);
        fma_peak_kernel<Real><<<grid, block>>>(out, iters, Real(1.0000001), Real(1e-9));
        cudaEventRecord(e1);
        e = cudaEventSynchronize(e1);
        if (e != cudaSuccess) break;
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (e != cudaSuccess) return e;
    *tflops = 2.0 * 64 * iters * (double)grid * block / (best * 1e-3) * 1e-12;
    return cudaGetLastError();
}
cudaError_t measure_dmma_peak(int sm_count, double* tflops) {
    const int block = 256, grid = sm_count * 2, iters = 8192;
    double* out = nullptr;
    cudaError_t e = cudaMalloc((void**)&out, sizeof(double) * (size_t)grid * block);
    if (e != cudaSuccess) return e;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
        cudaEventRecord(e0);
        dmma_peak_kernel<<<grid, block>>>(out, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1);
        e = cudaEventSynchronize(e1);
        if (e != cudaSuccess) break;
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (e != cudaSuccess) return e;
    // 8 x 8 x 4 multiply-adds per warp instruction
    *tflops = 2.0 * 256 * 8 * iters * (double)grid * (block / 32) / (best * 1e-3) * 1e-12;
    return cudaGetLastError();
}

template cudaError_t measure_fma_peak<double>(int, double*);
template cudaError_t measure_fma_peak<float>(int, double*);

template <typename Real>
cudaError_t launch_check_shifts(const Real* shifts, int64_t n, int* flag, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    const int block = 256;
    const int64_t grid = (n + block - 1) / block;
    check_shifts_kernel<Real><<<(unsigned)grid, block, 0, stream>>>(shifts, n, flag);
    return cudaGetLastError();
}

template <typename Real>
cudaError_t launch_pack_soa(const Real* aos, Real* soa, int64_t n, int p, int64_t stride,
                            cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    const int S = p * (p + 1);
    dim3 grid((unsigned)((n + 31) / 32), (unsigned)((S + 31) / 32)), block(32, 8);
    repack_kernel<Real, true><<<grid, block, 0, stream>>>(aos, soa, n, S, stride);
    return cudaGetLastError();
}

template <typename Real>
cudaError_t launch_unpack_soa(const Real* soa, Real* aos, int64_t n, int p, int64_t stride,
                              cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    const int S = p * (p + 1);
    dim3 grid((unsigned)((n + 31) / 32), (unsigned)((S + 31) / 32)), block(32, 8);
    repack_kernel<Real, false><<<grid, block, 0, stream>>>(soa, aos, n, S, stride);
    return cudaGetLastError();
}

// AoS -> rows: one thread per value of the padded layout.
template <typename Real>
__global__ void pack_rows_kernel(const Real* __restrict__ aos, Real* __restrict__ rows, int64_t n,
                                 int p) {
    const int R = rows_off(p), S = p * (p + 1);
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n * R) return;
    const int64_t b = i / R;
    const int k = (int)(i - b * R);
    int row = 0;
    while (rows_off(row + 1) <= k) ++row;
    const int j = k - rows_off(row);  // position in the row: 2 m + part
    rows[i] = j < 2 * (row + 1) ? aos[b * S + row * (row + 1) + j] : Real(0);
}

template <typename Real>
cudaError_t launch_pack_rows(const Real* aos, Real* rows, int64_t n, int p, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    const int64_t total = n * rows_off(p);
    pack_rows_kernel<Real><<<(unsigned)((total + 255) / 256), 256, 0, stream>>>(aos, rows, n, p);
    return cudaGetLastError();
}

template <typename Real>
cudaError_t launch_build_plan(const int64_t* tgt_ptr, const int64_t* grp_ptr,
                              const int32_t* grp_target, const int32_t* src_index,
                              const Real* shifts, int64_t n_groups, int64_t n_sources, int group,
                              int32_t* out_index, Real* out_shifts, Real* out_angles,
                              int32_t* out_angle_index, int* flags, cudaStream_t stream) {
    if (n_groups <= 0) return cudaSuccess;
    const int block = 256;
    const int64_t n = n_groups * group;
    const int64_t grid = (n + block - 1) / block;
    build_plan_kernel<Real><<<(unsigned)grid, block, 0, stream>>>(
        tgt_ptr, grp_ptr, grp_target, src_index, shifts, n_groups, n_sources, group, out_index,
        out_shifts, flags);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // geometry per distinct shift: {table, rep, uid, state} are stream-ordered temporaries
    int* scratch = nullptr;
    const size_t words = (size_t)kDedupSlots + 2 * (size_t)n + 4;
    e = cudaMallocAsync((void**)&scratch, sizeof(int) * words, stream);
    if (e != cudaSuccess) return e;
    int* table = scratch;
    int32_t* rep = scratch + kDedupSlots;
    int32_t* uid = rep + n;
    int* state = uid + n;
    e = cudaMemsetAsync(table, 0xFF, sizeof(int) * kDedupSlots, stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(state, 0, sizeof(int) * 4, stream);
    if (e == cudaSuccess) {
        dedup_rep_kernel<Real><<<(unsigned)grid, block, 0, stream>>>(out_shifts, n, table, rep, state);
        dedup_assign_kernel<Real><<<(unsigned)grid, block, 0, stream>>>(out_shifts, n, rep, uid, out_angles, state);
        dedup_index_kernel<Real><<<(unsigned)grid, block, 0, stream>>>(n, rep, uid, out_angle_index, state);
        e = cudaGetLastError();
    }
    cudaFreeAsync(scratch, stream);
    return e;
}

template <typename Real>
cudaError_t launch_zero_unwritten(const int64_t* grp_ptr, int64_t n_targets, int p_out, Real* out,
                                  int64_t out_stride, cudaStream_t stream) {
    if (n_targets <= 0) return cudaSuccess;
    zero_unwritten_kernel<Real><<<(unsigned)((n_targets + 127) / 128), 128, 0, stream>>>(
        grp_ptr, n_targets, p_out, out, out_stride);
    return cudaGetLastError();
}

template <typename Real>
cudaError_t launch_reduce_groups(const Real* partial, int64_t n_groups, const int64_t* grp_ptr,
                                 int per, int64_t n_targets, int p_out, Real* out,
                                 int64_t out_stride, cudaStream_t stream) {
    if (n_targets <= 0) return cudaSuccess;
    const int S = p_out * (p_out + 1);
    dim3 grid((unsigned)((n_targets + 127) / 128), (unsigned)S), block(128);
    reduce_groups_kernel<Real>
        <<<grid, block, 0, stream>>>(partial, n_groups, grp_ptr, per, n_targets, S, out, out_stride);
    return cudaGetLastError();
}

namespace {

// Orders from which the tensor-core kernel is the automatic choice (measured, profiles/
// ncu_r02_notes.md): up to order 20 the tiled DFMA kernel is 15-17 % faster (the 8 x 4 tiles
// of m8n8k4 are half padding at the class sizes 9 and 10, and DMMA shares its issue port with
// the FP64 and integer multiply-add instructions around it); from order 21 on the tiled
// kernel does not apply and the tensor-core kernel is ~5x the generic kernel.
constexpr int kMmaMinOrder = 21;

bool mma_ok(const DeviceTables<double>& t, const TranslateArgs<double>& a) { return mma_supports(a, t); }
bool mma_ok(const DeviceTables<float>&, const TranslateArgs<float>&) { return false; }
int mma_group(const TranslateArgs<double>& a) { return mma_group_size(a); }
int mma_group(const TranslateArgs<float>&) { return kLanes; }
cudaError_t mma_launch(const DeviceTables<double>& t, const TranslateArgs<double>& a, int sm_count,
                       cudaStream_t stream, LaunchInfo* info) {
    return launch_translate_mma(t, a, sm_count, stream, info);
}
cudaError_t mma_launch(const DeviceTables<float>&, const TranslateArgs<float>&, int, cudaStream_t,
                       LaunchInfo*) {
    return cudaErrorInvalidValue;
}

}  // namespace

template <typename Real>
int translate_variant(const DeviceTables<Real>& t, const TranslateArgs<Real>& a) {
    const int p_rot = std::max(a.p_in, a.p_out);
    const bool mma = mma_ok(t, a), tiled = tiled_supports(a);
    const bool small = small_supports(a);
    if (a.precise) return sizeof(Real) == 8 && a.variant <= 1 ? 1 : 0;  // generic kernel only
    switch (a.variant) {
        case 1: return 1;
        case 2: return tiled ? 2 : 0;
        case 3: return mma ? 3 : 0;
        case 4: return small ? 4 : 0;
        default: break;
    }
    if (small) return 4;
    if (mma && (p_rot >= kMmaMinOrder || !tiled)) return 3;
    return tiled ? 2 : 1;
}

template <typename Real>
int translate_group_size(const DeviceTables<Real>& t, const TranslateArgs<Real>& a) {
    const int v = translate_variant(t, a);
    return v == 3 ? mma_group(a) : (v == 2 ? 64 : kLanes);
}

template <typename Real>
cudaError_t launch_translate(const DeviceTables<Real>& t, const TranslateArgs<Real>& a,
                             int sm_count, cudaStream_t stream, LaunchInfo* info) {
    if (a.n <= 0) return cudaSuccess;
    const int v = translate_variant(t, a);
    if (v == 0) return cudaErrorInvalidValue;
    if (v == 4) return launch_translate_small(a, stream, info);
    if (v == 3) return mma_launch(t, a, sm_count, stream, info);
    if (v == 2) return launch_translate_tiled(t, a, sm_count, stream, info);
    const int p_rot = std::max(a.p_in, a.p_out);
    const int64_t n_groups = (a.n + kLanes - 1) / kLanes;
    const int limit = smem_optin_limit();

    GenericLayout<Real> lay{p_rot, 8, true, a.precise};
    if ((int64_t)lay.smem_bytes() > limit) lay.warps = 4;
    if ((int64_t)lay.smem_bytes() > limit) {
        lay.warps = 8;
        lay.buf_in_smem = false;
    }
    const size_t smem = lay.smem_bytes();
    const int block = lay.warps * 32;

    auto kern = lay.buf_in_smem ? translate_generic_kernel<Real, true>
                                : translate_generic_kernel<Real, false>;
    if constexpr (sizeof(Real) == 8) {
        if (a.precise)
            kern = lay.buf_in_smem ? translate_generic_kernel<Real, true, true>
                                   : translate_generic_kernel<Real, false, true>;
    }
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 1;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, smem);
    if (e != cudaSuccess) return e;
    per_sm = std::max(per_sm, 1);
    const int grid = (int)std::min<int64_t>(n_groups, (int64_t)sm_count * per_sm);

    Real* gscratch = nullptr;
    if (!lay.buf_in_smem) {
        e = cudaMallocAsync((void**)&gscratch, sizeof(Real) * lay.buf_elems() * grid, stream);
        if (e != cudaSuccess) return e;
    }
    kern<<<grid, block, smem, stream>>>(t, a, gscratch, n_groups, p_rot);
    e = cudaGetLastError();
    if (gscratch) cudaFreeAsync(gscratch, stream);
    if (info) {
        info->grid = grid;
        info->block = block;
        info->smem = smem;
        info->launches = 1;
        info->variant = a.precise ? "generic/precise" : (lay.buf_in_smem ? "generic/smem" : "generic/global-scratch");
    }
    return e;
}

#define SFMM_INSTANTIATE(Real)                                                                   \
    template cudaError_t launch_check_shifts<Real>(const Real*, int64_t, int*, cudaStream_t);   \
    template cudaError_t launch_pack_soa<Real>(const Real*, Real*, int64_t, int, int64_t,       \
                                               cudaStream_t);                                   \
    template cudaError_t launch_pack_rows<Real>(const Real*, Real*, int64_t, int, cudaStream_t); \
    template cudaError_t launch_unpack_soa<Real>(const Real*, Real*, int64_t, int, int64_t,     \
                                                 cudaStream_t);                                 \
    template cudaError_t launch_zero_unwritten<Real>(const int64_t*, int64_t, int, Real*, int64_t,  \
                                                     cudaStream_t);                             \
    template cudaError_t launch_reduce_groups<Real>(const Real*, int64_t, const int64_t*, int,  \
                                                    int64_t, int, Real*, int64_t, cudaStream_t); \
    template int translate_variant<Real>(const DeviceTables<Real>&, const TranslateArgs<Real>&); \
    template int translate_group_size<Real>(const DeviceTables<Real>&,                          \
                                            const TranslateArgs<Real>&);                        \
    template cudaError_t launch_build_plan<Real>(const int64_t*, const int64_t*, const int32_t*, \
                                                 const int32_t*, const Real*, int64_t, int64_t, \
                                                 int, int32_t*, Real*, Real*, int32_t*, int*,          \
                                                 cudaStream_t);                                 \
    template cudaError_t launch_translate<Real>(const DeviceTables<Real>&,                      \
                                                const TranslateArgs<Real>&, int, cudaStream_t,  \
                                                LaunchInfo*);

SFMM_INSTANTIATE(double)
SFMM_INSTANTIATE(float)

}  // namespace sfmm

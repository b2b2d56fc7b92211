// Internal interface between the C-ABI layer (capi.cu) and the kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "tables.hpp"

namespace sfmm {

enum : int { KIND_M2L = 0, KIND_M2M = 1, KIND_L2L = 2 };

// Input layouts of a launch.
//   LAYOUT_SOA   coefficient-major [c][stride]: unit-stride batches
//   LAYOUT_ROWS  expansion-major [src][rows_len(p)]: the reference order (row n holds
//                re, im of m = 0..n, solid.hpp:59-70) with every row padded to a multiple
//                of four values, so that a lane that gathers its own source reads whole
//                32-byte sectors (256-bit loads in double precision)
enum : int { LAYOUT_SOA = 0, LAYOUT_ROWS = 1 };

// first value of row n in LAYOUT_ROWS; rows_off(p) is the length of one expansion
__host__ __device__ inline int rows_off(int n) {
    const int a = n >> 1;
    return 4 * (a + 1) * (a + (n & 1));
}

// Device-resident tables of one handle (precision Real).
template <typename Real>
struct DeviceTables {
    int order = 0;
    // parity-block streams: side 0 = multipole-type data (F, G),
    // side 1 = local-type data (F^T, G^T)
    const Real* stream[2] = {nullptr, nullptr};
    const BlockDesc* desc[2] = {nullptr, nullptr};
    uint32_t stream_len[2] = {0, 0};
    const Real* fac = nullptr;   // k!, k <= 2P-2
    const Real* inv = nullptr;   // 1/d!, d < P
    const Real* winv = nullptr;  // (-1)^d / d!, d < P (M2M weights, pipeline.cpp:191-194)
    // fragment-major swap matrices of the tensor-core kernel (tables.hpp, pack_frags);
    // double precision handles with order <= 30 only
    const Real* frags[2] = {nullptr, nullptr};
};

// One uniform-(p_in, p_out) launch.
template <typename Real>
struct TranslateArgs {
    int kind = 0;
    int p_in = 0, p_out = 0;
    int64_t n = 0;                // translations (lanes); in accumulate mode: padded pairs
    const Real* in = nullptr;     // SoA [c][in_stride], or rows [src][in_stride]
    int64_t in_stride = 0;
    int in_layout = LAYOUT_SOA;
    const Real* shifts = nullptr; // [n][3]
    // optional, plan path: the decomposed shifts [6][n] = |r|, cos/sin alpha, cos/sin beta,
    // 1/|r| (geometry.cpp:11-30), computed once when the plan is built
    const Real* angles = nullptr;
    // entry of every lane in `angles` (one entry per distinct shift); null: entry = lane
    const int32_t* angle_index = nullptr;
    Real* out = nullptr;          // SoA [c][out_stride]; accumulate mode: partials [c][n/32]
    int64_t out_stride = 0;
    const int32_t* src_index = nullptr;  // accumulate mode: source per lane, -1 = idle lane
    // accumulate mode, direct form (tiled kernel): `out` is the final SoA output [c][target];
    // a CTA works on a contiguous, target-aligned range of groups and adds the groups of a
    // target in ascending order itself (no partial buffer, no reduce kernel)
    const int32_t* grp_target = nullptr;  // [n / 64] target of every group
    const int64_t* grp_ptr = nullptr;     // [n_targets + 1] first group of every target
    int64_t n_targets = 0;
    bool acc_plain = false;              // direct form: load-add-store instead of the L2 add
    bool precise = false;                // double-double backward pass (generic kernel, f64)
    int reserve_sms = 0;                 // tiled kernel: SMs left free for concurrent small kernels
    const int* fail_flag = nullptr;      // device int; non-zero -> kernel writes nothing
    int variant = 0;                     // 0 auto, 1 generic, 2 tiled, 3 mma, 4 small-order kernel
    long long* phase_clocks = nullptr;   // optional [8] cycle counters of CTA 0 (tuning aid)
};

struct LaunchInfo {
    int grid = 0, block = 0;
    size_t smem = 0;
    int launches = 0;
    int group = 32;  // translations per CTA group (accumulate mode: lanes reduced into one partial)
    const char* variant = "";
};

// Kernel chosen for `a`: 1 generic, 2 tiled, 3 mma, 4 small (a.variant forces one when it
// applies, 0 = it does not).
template <typename Real>
int translate_variant(const DeviceTables<Real>& t, const TranslateArgs<Real>& a);

// Group size the kernel chosen for `a` works with (32 generic, 64 tiled, 32 / 16 mma).
template <typename Real>
int translate_group_size(const DeviceTables<Real>& t, const TranslateArgs<Real>& a);

// Translation kernels. Returns cudaSuccess or the launch error.
template <typename Real>
cudaError_t launch_translate(const DeviceTables<Real>& t, const TranslateArgs<Real>& a,
                             int sm_count, cudaStream_t stream, LaunchInfo* info);

// Tuned kernels (kernel_tiled.inl): orders <= 20 (double) / <= 18 (float).
bool tiled_supports(const TranslateArgs<double>& a);
bool tiled_supports(const TranslateArgs<float>& a);
cudaError_t launch_translate_tiled(const DeviceTables<double>& t, const TranslateArgs<double>& a,
                                   int sm_count, cudaStream_t stream, LaunchInfo* info);
cudaError_t launch_translate_tiled(const DeviceTables<float>& t, const TranslateArgs<float>& a,
                                   int sm_count, cudaStream_t stream, LaunchInfo* info);

// Tensor-core kernel (sfmm_mma_f64.cu): double precision, orders <= 30.
bool mma_supports(const TranslateArgs<double>& a, const DeviceTables<double>& t);
int mma_group_size(const TranslateArgs<double>& a);
cudaError_t launch_translate_mma(const DeviceTables<double>& t, const TranslateArgs<double>& a,
                                 int sm_count, cudaStream_t stream, LaunchInfo* info);

// Small-order kernel (sfmm_small.cu): same-order independent translations, P <= 8, SoA.
bool small_supports(const TranslateArgs<double>& a);
bool small_supports(const TranslateArgs<float>& a);
cudaError_t launch_translate_small(const TranslateArgs<double>& a, cudaStream_t stream, LaunchInfo* info);
cudaError_t launch_translate_small(const TranslateArgs<float>& a, cudaStream_t stream, LaunchInfo* info);

// Measured FMA-pipe peak of the current device in the given precision.
template <typename Real>
cudaError_t measure_fma_peak(int sm_count, double* tflops);

// Measured FP64 tensor-core (mma.m8n8k4.f64) peak of the current device.
cudaError_t measure_dmma_peak(int sm_count, double* tflops);

// Zero-shift scan: sets *flag (device int) to 1 when any |shift| < min normal.
template <typename Real>
cudaError_t launch_check_shifts(const Real* shifts, int64_t n, int* flag, cudaStream_t stream);

// AoS [n][P(P+1)] <-> SoA [c][stride]
template <typename Real>
cudaError_t launch_pack_soa(const Real* aos, Real* soa, int64_t n, int p, int64_t stride,
                            cudaStream_t stream);
template <typename Real>
cudaError_t launch_unpack_soa(const Real* soa, Real* aos, int64_t n, int p, int64_t stride,
                              cudaStream_t stream);

// AoS [n][P(P+1)] -> rows [n][rows_off(p)] (padding zeroed)
template <typename Real>
cudaError_t launch_pack_rows(const Real* aos, Real* rows, int64_t n, int p, cudaStream_t stream);

// Accumulate mode, plan construction on the device (padding to groups + validation).
template <typename Real>
cudaError_t launch_build_plan(const int64_t* tgt_ptr, const int64_t* grp_ptr,
                              const int32_t* grp_target, const int32_t* src_index,
                              const Real* shifts, int64_t n_groups, int64_t n_sources, int group,
                              int32_t* out_index, Real* out_shifts, Real* out_angles,
                              int32_t* out_angle_index, int* flags, cudaStream_t stream);

// Accumulate mode, direct form: zeroes what the translation kernel does not write (the
// Im(C_n^0) planes of every target, all planes of targets without pairs).
template <typename Real>
cudaError_t launch_zero_unwritten(const int64_t* grp_ptr, int64_t n_targets, int p_out, Real* out,
                                  int64_t out_stride, cudaStream_t stream);

// Accumulate mode, second stage: out[c][t] = sum_{g in groups of t} partial[c][g],
// groups in ascending order. grp_ptr: [n_targets + 1] in units of `per` partial groups.
template <typename Real>
cudaError_t launch_reduce_groups(const Real* partial, int64_t n_groups, const int64_t* grp_ptr,
                                 int per, int64_t n_targets, int p_out, Real* out,
                                 int64_t out_stride, cudaStream_t stream);

// ---- particle <-> expansion steps (sfmm_harmonics.cu; reference harmonics.cpp) ----------------
// layout of the expansions: LAYOUT_SOA, LAYOUT_ROWS or LAYOUT_AOS ([box][P(P+1)], solid.hpp:59-70)
enum : int { LAYOUT_AOS = 2 };
int harmonics_max_order();
// P2M (harmonics.cpp:105-117): charges [n][4] = x y z q, box b owns charges box_ptr[b] .. box_ptr[b+1]
template <typename Real>
cudaError_t launch_p2m(const int64_t* box_ptr, const Real* charges, const Real* centers,
                       int64_t n_boxes, int order, int layout, Real* out, int64_t stride,
                       cudaStream_t stream);
// L2P (harmonics.cpp:119-152): out[i] = eval_local(L[point_box[i]], centre, points[i]);
// point_box == nullptr: point i belongs to box i
template <typename Real>
cudaError_t launch_eval_local(const int32_t* point_box, const Real* points, const Real* centers,
                              int64_t n_points, int64_t n_boxes, int order, int layout,
                              const Real* locals, int64_t stride, Real* out, cudaStream_t stream);

}  // namespace sfmm

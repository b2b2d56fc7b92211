/* solidfmm_b200 — C ABI of the B200-native batched M2M / M2L / L2L translation
 * library (drop-in for the hot path of the reference library `mpole`).
 *
 * Every entry point names the reference interface it replaces; paths are
 * relative to /root/reference/proj/core. Plain pointers and sizes only; no C++
 * or torch types cross this boundary. All functions return an sfmm_status and
 * never throw. Coefficient arithmetic is bit-identical to the reference built
 * with FMA contraction.
 *
 * Coefficient layouts
 *   AoS  (reference layout, include/mpole/solid.hpp:59-70): one solid is
 *        P(P+1) reals, row n at n(n+1), (re, im) interleaved over m = 0..n.
 *        A batch is [n][P(P+1)], contiguous.
 *   SoA  (device layout, "batch-major"): element c of solid b lives at
 *        base[c * stride + b], c being the AoS index above and stride >= n the
 *        batch stride in elements. The planes of Im(C_n^0) are ignored on input
 *        and written as zeros on output.
 *   Shifts are [n][3] = (x, y, z), source centre -> target centre
 *        (include/mpole/pipeline.hpp:11-21).
 */
#ifndef SOLIDFMM_B200_H
#define SOLIDFMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum sfmm_status {
    SFMM_OK = 0,
    SFMM_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    SFMM_DOMAIN_ERROR = 2,     /* std::domain_error (zero shift)         */
    SFMM_CUDA_ERROR = 3,       /* no counterpart: device/runtime failure */
    SFMM_OUT_OF_MEMORY = 4
} sfmm_status;

typedef enum sfmm_kind { SFMM_M2L = 0, SFMM_M2M = 1, SFMM_L2L = 2 } sfmm_kind;
typedef enum sfmm_precision { SFMM_F64 = 0, SFMM_F32 = 1 } sfmm_precision;

/* Opaque handle: device copies of the swap-matrix streams and faculty tables
 * for orders <= `order`, plus library-owned device scratch.
 * Replaces mpole::operator_data<Real> (operators.hpp:57-95) and, because the
 * scratch travels with the call, mpole::workspace<Real> (workspace.hpp:18-51). */
typedef struct sfmm_handle sfmm_handle;

/* operator_data<Real>::operator_data(order, cfg) / acquire() (operators.cpp:123-187).
 * INVALID_ARGUMENT for order < 1 or order > sfmm_max_order(precision)
 * (operators.cpp:127-132). mu/nu are the reference's CPU blocking parameters:
 * validated like kernels.cpp:19-26 when non-zero, otherwise ignored. */
sfmm_status sfmm_create(sfmm_precision precision, int order, int device,
                        int mu, int nu, sfmm_handle** out);
void sfmm_destroy(sfmm_handle* h);

/* operator_data::order() and ::max_order() (86 double / 18 single). */
int sfmm_order(const sfmm_handle* h);
int sfmm_max_order(sfmm_precision precision);
int sfmm_device(const sfmm_handle* h);
const char* sfmm_status_string(sfmm_status s);
const char* sfmm_last_error(void); /* thread-local detail for the last failure */

/* Table access, for verification against operator_data::swaps(n).f_dense /
 * g_dense, faculties() and inv_faculties() (operators.hpp:67-80). f and g
 * receive (n+1)^2 doubles row-major [m][l]; fac 2P-1 and inv P values in the
 * handle's precision (as doubles). Any pointer may be NULL. */
sfmm_status sfmm_get_swap_tables(const sfmm_handle* h, int n, double* f, double* g);
sfmm_status sfmm_get_faculties(const sfmm_handle* h, double* fac, double* inv);

/* The same tables computed on the host without touching a device (what
 * sfmm_create uploads): wigner_b / swap_matrices (operators.cpp:12-66) and the
 * faculty tables of operator_data (operators.cpp:134-142). INVALID_ARGUMENT for
 * n < 0 or an order outside [1, sfmm_max_order(precision)]. */
sfmm_status sfmm_host_swap_tables(int n, double* f, double* g);
sfmm_status sfmm_host_faculties(sfmm_precision precision, int order, double* fac, double* inv);

/* ---- batched translation, host buffers, reference AoS layout -------------
 * Replaces m2l/m2m/l2l(ops, span<translation_request>, ws) (pipeline.hpp:30-45,
 * pipeline.cpp:275-369) for one uniform (p_in, p_out) group: validates every
 * request first (orders >= 1, max(p_in,p_out) <= order -> INVALID_ARGUMENT;
 * |shift| < min normal -> DOMAIN_ERROR; pipeline.cpp:282-298), and only then
 * copies in, runs on the device, and overwrites `out`. n == 0 is a no-op.
 * `out` may alias `in` when p_in == p_out (in-place, pipeline.hpp:11-14). */
sfmm_status sfmm_translate_host(sfmm_handle* h, sfmm_kind kind, int64_t n,
                                int p_in, int p_out, const void* in_aos,
                                const void* shifts, void* out_aos);

/* Mixed orders in one call (the grouping of pipeline.cpp:302-342 happens
 * inside): request i reads in + in_offset[i] (P_in[i](P_in[i]+1) reals) and
 * overwrites out + out_offset[i] (P_out[i](P_out[i]+1) reals); offsets are in
 * elements. Validation as above, all before any output is touched. */
sfmm_status sfmm_translate_host_mixed(sfmm_handle* h, sfmm_kind kind, int64_t n,
                                      const int* p_in, const int* p_out,
                                      const void* in, const int64_t* in_offset,
                                      const void* shifts, void* out,
                                      const int64_t* out_offset);

/* ---- batched translation, device buffers, SoA layout ---------------------
 * The resident-data form of the same call: all pointers are device pointers on
 * sfmm_device(h). Work is enqueued on `stream` (a cudaStream_t, NULL = default
 * stream). The zero-shift scan runs on the device ahead of the translation
 * kernel, which does not write anything when the scan fails; with
 * SFMM_SYNC_STATUS (default) the call waits for the scan result and returns
 * DOMAIN_ERROR, with SFMM_ASYNC_STATUS it returns at once and the outcome is
 * read later with sfmm_stream_status(). */
enum { SFMM_SYNC_STATUS = 0, SFMM_ASYNC_STATUS = 1 };
/* The host-buffer entry points (sfmm_translate_host, _mixed, sfmm_plan_create,
 * sfmm_m2l_accumulate_host) run on a private non-blocking stream per calling thread and
 * device: concurrent callers do not serialise on the legacy default stream. */
sfmm_status sfmm_translate_soa(sfmm_handle* h, sfmm_kind kind, int64_t n,
                               int p_in, int p_out, const void* d_in,
                               int64_t in_stride, const void* d_shifts,
                               void* d_out, int64_t out_stride, void* stream,
                               int flags);
/* Synchronises `stream` and reports the status of the SoA calls enqueued ON THAT STREAM
 * with SFMM_ASYNC_STATUS since its last query (DOMAIN_ERROR if any scan failed). Calls
 * issued on other streams keep their status until their own stream is queried. A handle
 * tracks up to 256 unqueried calls; beyond that a call reports synchronously. */
sfmm_status sfmm_stream_status(sfmm_handle* h, void* stream);

/* AoS <-> SoA repacking on the device (batch of n solids of order p). */
sfmm_status sfmm_pack_soa(sfmm_handle* h, int64_t n, int p, const void* d_aos,
                          void* d_soa, int64_t stride, void* stream);
sfmm_status sfmm_unpack_soa(sfmm_handle* h, int64_t n, int p, const void* d_soa,
                            int64_t stride, void* d_aos, void* stream);

/* "Rows" layout for expansions that are GATHERED by index (the sources of
 * sfmm_m2l_accumulate_rows): expansion-major like the reference
 * (solid.hpp:59-70: row n holds re, im of m = 0..n), with every row padded to a
 * multiple of four values so that a thread that fetches its own source reads
 * whole 32-byte sectors. sfmm_rows_len(p) values per expansion. */
int64_t sfmm_rows_len(int p);
sfmm_status sfmm_pack_rows(sfmm_handle* h, int64_t n, int p, const void* d_aos,
                           void* d_rows, void* stream);

/* ---- particle <-> expansion steps (the callers either side of the translation path) ----
 * P2M replaces `mpole::p2m` (reference core/src/harmonics.cpp:105-117, core/include/mpole/
 * harmonics.hpp:36-39) for a batch of boxes: box b owns the charges box_ptr[b] .. box_ptr[b+1]
 * of `charges` ([n][4] = x y z q, the reference's point_charge) and has centre centers[b][3];
 * its multipole of order `order` is written in `layout`:
 *   SFMM_LAYOUT_AOS   [box][P(P+1)], the reference's solid layout (solid.hpp:59-70)
 *   SFMM_LAYOUT_SOA   [c][out_stride], the input layout of sfmm_translate_soa / sfmm_m2l_accumulate
 *   SFMM_LAYOUT_ROWS  [box][sfmm_rows_len(P)], the source layout of sfmm_m2l_accumulate_rows
 * L2P replaces `mpole::eval_local` (harmonics.cpp:119-152, harmonics.hpp:48-51): out[i] is the
 * potential of the local expansion of box point_box[i] (NULL: box i) at points[i][3].
 * Results equal the reference's (parity build, -mfma -ffp-contract=fast) bit for bit, charges and
 * sums taken in the reference's order. Device entry points take device pointers and a stream;
 * the _host forms take host arrays (expansions in the AoS layout) and validate the box
 * indices (INVALID_ARGUMENT); the device form writes NaN for a point whose box index is out
 * of range. Every order of the handle (tuned kernels to order 32, plain ones above). */
enum { SFMM_LAYOUT_SOA = 0, SFMM_LAYOUT_ROWS = 1, SFMM_LAYOUT_AOS = 2 };
int sfmm_harmonics_max_order(void);
sfmm_status sfmm_p2m(sfmm_handle* h, int64_t n_boxes, const int64_t* d_box_ptr,
                     const void* d_charges, const void* d_centers, int order, int layout,
                     void* d_out, int64_t out_stride, void* stream);
sfmm_status sfmm_eval_local(sfmm_handle* h, int64_t n_points, const int32_t* d_point_box,
                            const void* d_points, const void* d_centers, int64_t n_boxes,
                            int order, int layout, const void* d_locals, int64_t stride,
                            void* d_out, void* stream);
sfmm_status sfmm_p2m_host(sfmm_handle* h, int64_t n_boxes, const int64_t* box_ptr,
                          const void* charges, const void* centers, int order, void* out_aos);
sfmm_status sfmm_eval_local_host(sfmm_handle* h, int64_t n_points, const int32_t* point_box,
                                 const void* points, const void* centers, int64_t n_boxes,
                                 int order, const void* locals_aos, void* out);

/* ---- target-owned M2L accumulation (a full interaction-list level) -------
 * L[t] = sum over the sources s of target t of m2l(M[s], shift(t, s)), each
 * term computed exactly as the batched call computes it, summed without
 * atomics in a fixed order that depends only on the order pair and the kernel
 * variant (sfmm_accumulation_unit below tells which; DESIGN.md "Accumulation
 * order"): repeated calls give the same bits, different kernels may differ in
 * the last bits of a sum. The reference has
 * no such entry point (it overwrites: pipeline.cpp:258-265); a caller of the
 * reference issues one request per pair and adds the outputs itself.
 *
 * The plan holds the pair list in CSR form over targets: pairs
 * tgt_ptr[t] .. tgt_ptr[t+1]-1 belong to target t; pair j reads source
 * src_index[j] with shift shifts[3j..3j+2]. All plan inputs are HOST pointers
 * and are validated (zero shifts -> DOMAIN_ERROR) when the plan is built. */
typedef struct sfmm_plan sfmm_plan;
sfmm_status sfmm_plan_create(sfmm_handle* h, int64_t n_targets,
                             const int64_t* tgt_ptr, const int32_t* src_index,
                             const void* shifts, int64_t n_sources,
                             sfmm_plan** out);
/* Frees the plan, ordered behind the most recent accumulate call that used it (on that
 * call's stream). Callers that use one plan on several streams at once synchronise the
 * other streams first. */
void sfmm_plan_destroy(sfmm_plan* plan);
int64_t sfmm_plan_pairs(const sfmm_plan* plan);

/* Device SoA sources [c][src_stride], device SoA outputs [c][out_stride]
 * (overwritten with the sums; targets without pairs receive zeros). */
sfmm_status sfmm_m2l_accumulate(sfmm_handle* h, const sfmm_plan* plan, int p_in,
                                int p_out, const void* d_src, int64_t src_stride,
                                void* d_out, int64_t out_stride, void* stream);

/* The same with the sources in the rows layout, [n_sources][sfmm_rows_len(p_in)]:
 * the faster form, the gather of a source costs a quarter of the memory
 * transactions of the SoA form. Results are bit-identical. */
sfmm_status sfmm_m2l_accumulate_rows(sfmm_handle* h, const sfmm_plan* plan, int p_in,
                                     int p_out, const void* d_src_rows, void* d_out,
                                     int64_t out_stride, void* stream);

/* Host AoS form of the same: sources [n_sources][P_in(P_in+1)], outputs
 * [n_targets][P_out(P_out+1)], copies inside the call. */
sfmm_status sfmm_m2l_accumulate_host(sfmm_handle* h, const sfmm_plan* plan,
                                     int p_in, int p_out, const void* src_aos,
                                     void* out_aos);

/* One-shot form: plan + accumulation of one level from host arrays in a single call
 * (arguments as sfmm_plan_create and sfmm_m2l_accumulate_host). Large levels are pipelined
 * over slabs of targets: the pair list of the next slab uploads and the locals of the
 * previous slab download while the current slab computes. Results are bit-identical to the
 * two-call form; on INVALID_ARGUMENT / DOMAIN_ERROR nothing has been written to out_aos
 * (pipeline.cpp:282-298). "level_slab_pairs" (sfmm_set_option) sets the slab size from which
 * the pipeline is used (default 2^18 pairs per slab). */
sfmm_status sfmm_m2l_level_host(sfmm_handle* h, int64_t n_targets, const int64_t* tgt_ptr,
                                const int32_t* src_index, const void* shifts,
                                int64_t n_sources, int p_in, int p_out, const void* src_aos,
                                void* out_aos);

/* Pair list of one level of a uniform octree, in the form sfmm_plan_create and
 * sfmm_m2l_level_host take (no reference counterpart: its callers issue one
 * translation_request per pair, pipeline.hpp:15-21; tree traversal is a non-goal there).
 * Targets: the boxes (i, j, k) of an nx x ny x nz grid of boxes of side box_size, target
 * index (i ny + j) nz + k. Sources: the boxes of the grid extended by `halo` boxes on every
 * side, index ((i + halo)(ny + 2 halo) + (j + halo))(nz + 2 halo) + (k + halo); halo = 3 holds
 * every list entry (a level inside a larger domain), halo = 0 makes the targets their own
 * sources and drops the entries outside the grid (a free-standing level). List of a target:
 * the offsets d = source - target with d_a in [-2 - b_a, 3 - b_a], b_a the parity of the
 * target's coordinate (the children of the parent's neighbours), without the near field
 * max |d_a| <= 1: at most 189 entries, in lexicographic order of d; shift = -d box_size
 * (source -> target centre). Call with tgt_ptr = src_index = shifts = NULL for the sizes
 * (n_pairs, n_sources), then with arrays of n_targets + 1, n_pairs and 3 n_pairs entries
 * (shifts in `precision`). Host arrays; no device work. */
sfmm_status sfmm_level_pairs(int nx, int ny, int nz, int halo, double box_size,
                             sfmm_precision precision, int64_t* tgt_ptr, int32_t* src_index,
                             void* shifts, int64_t* n_pairs, int64_t* n_sources);

/* Summation unit of sfmm_m2l_accumulate* for this order pair with the kernel the
 * handle would choose: 64 = pairs j and j+32 of a 64-pair group are added first,
 * then the 32 sums by the xor butterfly (lane distances 16, 8, 4, 2, 1); 32 or 16 =
 * xor butterfly over units of that many consecutive pairs; in every case the unit
 * sums of a target are then added in ascending order. 0 on invalid arguments.
 * (paper_2202_02847_b200/sharding.py accumulation_tree restates the tree; the
 * reference has no accumulate mode, pipeline.cpp:258-265 overwrites.) */
int sfmm_accumulation_unit(const sfmm_handle* h, int p_in, int p_out);

/* Options of a handle (set them before the handle is shared between threads: calls read them
 * without locking). Tuning knobs without a reference counterpart. "kernel_variant": 0 = automatic
 * (default), 1 = generic kernel (any order), 2 = tiled kernel (orders <= 20
 * double / <= 18 single; INVALID_ARGUMENT at call time beyond that), 3 = FP64
 * tensor-core kernel (double precision, handle order <= 30), 4 = small-order kernel
 * (same order <= 8, independent translations). "accumulate_plain": how the tiled kernel adds
 * the 64-pair groups of a target (all groups of a target run in one CTA, in ascending order,
 * so every sum has one owner at a time and the order is fixed): 0 (default) = the owner sends
 * the sums of the later groups to the L2 to be added there (red.global.add.f64, no round
 * trip); 1 = the owner loads, adds and stores (no atomic or reduction instruction anywhere;
 * 4 % slower on the P = 20 level). Same bits either way. Single precision always uses 1.
 * "precise" (double precision handles): 1 = every swap pass on local-side data (the backward
 * pass of M2L, both passes of L2L) carries its state in double-double, from cos(beta) = z / |r| through the recurrence, both transposed
 * swap products and the rotation between them, and rounds once at the end. This removes the
 * rounding floor of the rotation-based algorithm at high order (error against the O(P^4)
 * sum `m2l_naive`: 2e-11 -> 3e-14 at P = 20, 1e-10 -> 3e-14 at P = 24; L2L gains 3x; the reference itself
 * has the floor, so results then DIFFER from the reference's by that floor). Served by the
 * generic kernel (every order; 1.5e7 translations/s at P = 20, a fourteenth of the tuned kernel); combining it with
 * another "kernel_variant" is INVALID_ARGUMENT at call time. No reference counterpart. */
sfmm_status sfmm_set_option(sfmm_handle* h, const char* name, int64_t value);

/* Measures the FMA-pipe peak (TFLOP/s, 2 flops per FMA) of the handle's device
 * in the handle's precision with a register-only kernel (~10 ms). Benchmarks
 * use it as the compute-roofline denominator. */
sfmm_status sfmm_measure_fma_peak(sfmm_handle* h, double* tflops);

/* The same for the FP64 tensor-core instruction (mma.m8n8k4.f64, 512 flops per warp
 * instruction). Both run on one pipe; benchmarks take the larger of the two as the
 * FP64 roofline and report both. */
sfmm_status sfmm_measure_dmma_peak(sfmm_handle* h, double* tflops);

/* Number of kernel launches this handle has issued (bench.py gpu_launches). */
int64_t sfmm_launch_count(const sfmm_handle* h);

#ifdef __cplusplus
}
#endif
#endif /* SOLIDFMM_B200_H */

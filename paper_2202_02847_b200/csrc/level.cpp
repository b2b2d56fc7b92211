// Interaction list of one level of a uniform octree -> the CSR pair list that
// sfmm_plan_create / sfmm_m2l_level_host consume. Host code; the reference
// has no counterpart (SPEC.md:390 lists tree traversal as a non-goal), its callers build one
// translation_request per pair by hand (pipeline.hpp:15-21).
#include <cstdint>
#include <string>

#include "solidfmm_b200.h"

namespace {

// offsets (source - target, in boxes) of a target with coordinate parities (bx, by, bz):
// the children of the parent's neighbours that are not neighbours of the target, per axis
// d in [-2 - b, 3 - b], lexicographic order
template <typename F>
void for_each_offset(int bx, int by, int bz, F&& f) {
    for (int dx = -2 - bx; dx <= 3 - bx; ++dx)
        for (int dy = -2 - by; dy <= 3 - by; ++dy)
            for (int dz = -2 - bz; dz <= 3 - bz; ++dz) {
                const int ax = dx < 0 ? -dx : dx, ay = dy < 0 ? -dy : dy, az = dz < 0 ? -dz : dz;
                if (ax <= 1 && ay <= 1 && az <= 1) continue;  // near field
                f(dx, dy, dz);
            }
}

template <typename Real>
void fill(int nx, int ny, int nz, int halo, double h, int64_t* tgt_ptr, int32_t* src_index, Real* shifts,
          int64_t* n_pairs) {
    const int64_t sy = ny + 2 * halo, sz = nz + 2 * halo, sx = nx + 2 * halo;
    int64_t pos = 0, t = 0;
    for (int i = 0; i < nx; ++i)
        for (int j = 0; j < ny; ++j)
            for (int k = 0; k < nz; ++k, ++t) {
                if (tgt_ptr) tgt_ptr[t] = pos;
                for_each_offset(i & 1, j & 1, k & 1, [&](int dx, int dy, int dz) {
                    const int64_t a = i + dx + halo, b = j + dy + halo, c = k + dz + halo;
                    if (a < 0 || a >= sx || b < 0 || b >= sy || c < 0 || c >= sz) return;  // outside the domain
                    if (src_index) {
                        src_index[pos] = (int32_t)((a * sy + b) * sz + c);
                        // source -> target centre (pipeline.hpp:11-14)
                        shifts[3 * pos] = (Real)(-dx * h);
                        shifts[3 * pos + 1] = (Real)(-dy * h);
                        shifts[3 * pos + 2] = (Real)(-dz * h);
                    }
                    ++pos;
                });
            }
    if (tgt_ptr) tgt_ptr[t] = pos;
    *n_pairs = pos;
}

}  // namespace

extern "C" sfmm_status sfmm_level_pairs(int nx, int ny, int nz, int halo, double box_size,
                                        sfmm_precision precision, int64_t* tgt_ptr, int32_t* src_index,
                                        void* shifts, int64_t* n_pairs, int64_t* n_sources) {
    if (nx < 1 || ny < 1 || nz < 1 || halo < 0 || !(box_size > 0) || !n_pairs || !n_sources)
        return SFMM_INVALID_ARGUMENT;
    if (precision != SFMM_F64 && precision != SFMM_F32) return SFMM_INVALID_ARGUMENT;
    if ((tgt_ptr == nullptr) != (src_index == nullptr) || (tgt_ptr == nullptr) != (shifts == nullptr))
        return SFMM_INVALID_ARGUMENT;
    const int64_t ns = (int64_t)(nx + 2 * halo) * (ny + 2 * halo) * (nz + 2 * halo);
    if (ns > INT32_MAX) return SFMM_INVALID_ARGUMENT;  // source indices are 32-bit
    *n_sources = ns;
    if (precision == SFMM_F64) fill<double>(nx, ny, nz, halo, box_size, tgt_ptr, src_index, (double*)shifts, n_pairs);
    else fill<float>(nx, ny, nz, halo, box_size, tgt_ptr, src_index, (float*)shifts, n_pairs);
    return SFMM_OK;
}

// Host-side operator tables for the B200 translation library.
//
// Replaces the shift-independent part of the reference handle
// `mpole::operator_data<Real>` (reference core/include/mpole/operators.hpp:57-95,
// core/src/operators.cpp:123-165): the faculty tables and, per row n < P, the
// axis-swap matrices F_n and G_n. The reference's chequerboard panel packing
// (operators.cpp:68-89) is a CPU blocking format and is not reproduced; the
// device consumes the "parity block" streams built by pack_side() below.
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

namespace sfmm {

// Largest order whose faculty table (2P-2)! stays finite in the precision
// (reference operators.cpp:97-109): 86 in double, 18 in single.
int max_order_f64();
int max_order_f32();

// Dense swap matrices for rows n = 0..order-1, always in double
// (reference operators.cpp:12-66). f[n], g[n] are (n+1)x(n+1) row-major [m][l].
struct SwapTables {
    int order = 0;
    std::vector<std::vector<double>> f, g;
    explicit SwapTables(int order);
};

// faculties k!, k <= 2P-2, and inverse faculties 1/d!, d < P, built in Real by
// repeated multiplication exactly as the reference does (operators.cpp:134-142).
template <typename Real>
void build_faculties(int order, std::vector<Real>& fac, std::vector<Real>& inv);

// ---------------------------------------------------------------------------
// Device stream layout ("parity blocks").
//
// For row n the index set {0..n} splits into the even class E (|E| = n/2+1) and
// the odd class O (|O| = (n+1)/2). F_n couples classes a and b only when
// a+b == n (mod 2), G_n only when a+b == n+1 (mod 2), so each matrix is two
// dense blocks. For one side (multipole: A = F/G; local: A = F^T/G^T, reference
// pipeline.cpp:118-136) and one row n the stream holds four blocks
//
//   F rows E, F rows O, G rows E, G rows O
//
// each stored COLUMN-major with the column ("line") padded to an even length
// ld: entry (i,k) at k*ld + i, i.e. in the order a k-outer / i-inner FMA loop
// consumes it, every line 16-byte aligned in double so that two entries can be
// fetched with one 128-bit shared-memory load.
struct BlockDesc {
    uint32_t offset;   // element offset of the block in the stream
    uint16_t nrows;    // outputs: size of the row class
    uint16_t ncols;    // inputs: size of the column class
    uint8_t row_class; // 0 even, 1 odd
    uint8_t col_class;
    uint16_t ld;       // padded line length (nrows rounded up to even)
};

struct PackedSide {
    // desc[n*4 + {0: F/E, 1: F/O, 2: G/E, 3: G/O}]
    std::vector<BlockDesc> desc;
    std::vector<double> stream;  // cast to Real on upload
};

// local_side == false: A = F_n, G_n (multipole-type data);
// local_side == true:  A = F_n^T, G_n^T (local-type data).
PackedSide pack_side(const SwapTables& t, bool local_side);

// ---------------------------------------------------------------------------
// Fragment-major layout for the FP64 tensor-core kernel (sfmm_mma_f64.cu).
//
// The kernel evaluates y = A x for 8 translations at a time with
// mma.sync.m8n8k4.f64: the translations are the 8 rows of the A operand, the
// swap-matrix block is the B operand (4 inputs x 8 outputs per instruction). One
// "fragment" is the 32 doubles of one B operand in lane order: lane L holds
// block(out = sigma(mb, L >> 2), in = 4 kb + (L & 3)), zero outside the block, with
// the output permutation sigma(mb, c) = 8 mb + (c >> 1) + 4 (c & 1). With this
// permutation the two accumulator registers of a lane (columns 2q and 2q+1) are
// outputs 8 mb + q and 8 mb + 4 + q, exactly the A operands of input blocks
// kb = 2 mb and 2 mb + 1 of the next product: swap -> rotate -> swap chains in
// registers without any lane exchange. A block's fragments are stored
// [kb][mb], kb < ceil(ncols / 4), mb < ceil(nrows / 8); blocks in the order of
// PackedSide::desc (which also gives nrows / ncols; offsets are in fragments
// and are the same for both sides).
struct FragSide {
    std::vector<uint32_t> offset;  // [order * 4 + 1]: first fragment of block n*4 + j
    std::vector<double> frags;     // 32 doubles per fragment
};
FragSide pack_frags(const SwapTables& t, bool local_side);

// Number of stream elements occupied by rows n < order (the stream is ordered
// by n, so the tables of a lower order are a prefix).
size_t packed_prefix_len(int order);

}  // namespace sfmm

// exsum_launch.h -- host-side launchers shared by the C-ABI orchestration.
//
// Every launcher works on a 3-D view [outer, n, inner] of a C-order array
// (outer = prod of extents before the axis, inner = prod after it), which is
// how windowed_sum_axis (scan.py:61-102) sees any axis of any d.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace exsum {

enum DType { F32 = 0, F64 = 1, I64 = 2 };
enum OpCode { ADD = 0, MAX = 1 };

// One windowed pass along the middle axis of [outer, n, inner]:
// out[o, x, i] = (+)_{y in [x, min(x+k, n))} in[o, y, i], with the reference's
// exact association (in-block right-nested suffix, left-nested prefix, one
// stitch combine).  in != out.  `total` (device, nullable) turns on the BDBSC
// complement epilogue out = total (-) value (float32 data: total is a double).
// Returns the number of kernels launched.
int launch_pass(int dtype, int op, const void* in, void* out, int64_t outer, int64_t n,
                int64_t inner, int64_t k, const void* total, cudaStream_t s);

// Deterministic total fold of N elements into *total (device; double for
// float32).  partials: device scratch of reduce_partials_count() accumulators.
int reduce_partials_count();
int launch_total(int dtype, int op, const void* in, int64_t N, void* partials, void* total,
                 cudaStream_t s);

// BDBSC complement for a route with no windowed pass: out = total (-) in.
int launch_complement(int dtype, const void* in, void* out, int64_t N, const void* total,
                      cudaStream_t s);

// R[r] = (+)_x in[r, x] for rows of length n (box-complement reduction of the
// peeled last axis).
int launch_row_reduce(int dtype, int op, const void* in, void* R, int64_t rows, int64_t n,
                      cudaStream_t s);

// Box-complement round along the last axis (rows of length n):
// out[r, x] = P[r, x-1] (+) S[r, x+k] (+) T[r], with P/S the full-row
// inclusive prefix/suffix of W and T the tail (nullable = identity).  Terms
// out of range are the identity.  scratch: rows*n elements, used only when a
// row does not fit in shared memory.
int launch_excl_rows(int dtype, int op, const void* W, void* out, const void* T, int64_t rows,
                     int64_t n, int64_t k, void* scratch, cudaStream_t s);
size_t excl_rows_scratch_elems(int dtype, int64_t rows, int64_t n);

size_t dtype_size(int dtype);
int num_sms();

}  // namespace exsum

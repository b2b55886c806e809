// axis_stream_i64add.cu -- axis_stream.cuh instantiated for i64 / OpAdd
// (one translation unit per element type so they compile in parallel).
#include "axis_stream.cuh"

namespace exsum {

int launch_axis_stream_i64add(const void* in, void* out, int64_t outer, int64_t n, int64_t inner,
                             int64_t k, const void* total, cudaStream_t s, PassExtra* ex) {
  return go_axis_stream<i64, OpAdd>((const i64*)in, (i64*)out, outer, n, inner, k,
                                   (const typename AccOf<i64>::type*)total, s, ex);
}

}  // namespace exsum

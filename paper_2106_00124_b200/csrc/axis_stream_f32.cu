// axis_stream_f32.cu -- axis_stream.cuh instantiated for float / OpAdd
// (one translation unit per element type so they compile in parallel).
#include "axis_stream.cuh"

namespace exsum {

int launch_axis_stream_f32(const void* in, void* out, int64_t outer, int64_t n, int64_t inner,
                             int64_t k, const void* total, cudaStream_t s, PassExtra* ex) {
  return go_axis_stream<float, OpAdd>((const float*)in, (float*)out, outer, n, inner, k,
                                   (const typename AccOf<float>::type*)total, s, ex);
}

}  // namespace exsum

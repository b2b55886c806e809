// fused_pair_f32.cu -- instantiations of fused_pair.cuh for float / OpAdd
// (one translation unit per element type so they compile in parallel).
#include "fused_pair.cuh"

namespace exsum {

int launch_fused_pair_f32(const void* in, void* out, int64_t outer, int64_t n1, int64_t n2,
                            int64_t k1, int64_t k2, int mode, const void* total, const void* Tail,
                            cudaStream_t s) {
  return go_fused<float, OpAdd>((const float*)in, (float*)out, outer, n1, n2, k1, k2, mode, (const double*)total,
                             (const float*)Tail, s);
}

}  // namespace exsum

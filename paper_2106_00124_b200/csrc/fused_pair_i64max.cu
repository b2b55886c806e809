// fused_pair_i64max.cu -- instantiations of fused_pair.cuh for i64 / OpMax
// (one translation unit per element type so they compile in parallel).
#include "fused_pair.cuh"

namespace exsum {

int launch_fused_pair_i64max(const void* in, void* out, int64_t outer, int64_t n1, int64_t n2,
                            int64_t k1, int64_t k2, int mode, const void* total, const void* Tail,
                            cudaStream_t s) {
  return go_fused<i64, OpMax>((const i64*)in, (i64*)out, outer, n1, n2, k1, k2, mode, nullptr,
                             (const i64*)Tail, s);
}

}  // namespace exsum

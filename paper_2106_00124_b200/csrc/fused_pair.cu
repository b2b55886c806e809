// fused_pair.cu -- eligibility and dispatch of the fused pass pair
// (kernel: fused_pair.cuh; instantiations: fused_pair_{f32,f64,i64add,i64max}.cu).
#include <stdlib.h>

#include "exsum_launch.h"

namespace exsum {

// Shape/dtype eligibility without launching (the workspace sizing pass and the
// launch pass must take the same decision).  EXSUM_FUSE=0 disables fusion.
int fused_pair_ok(int dtype, int op, int64_t n2, int64_t k1, int64_t k2, int mode) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("EXSUM_FUSE");
    env = (e && e[0] == '0') ? 0 : 1;
  }
  if (!env) return 0;
  if (dtype != F32 && dtype != F64 && dtype != I64) return 0;
  if (op == MAX && dtype != I64) return 0;
  // rows longer than the widest template run as strips of it (ROW_WIN only)
  const int64_t wmax = dtype == F32 ? 1024 : 512;
  const bool strip = mode == ROW_WIN && n2 > wmax && n2 % wmax == 0 && n2 / wmax <= (1 << 20);
  if (strip) n2 = wmax;
  if (n2 != 256 && n2 != 512 && n2 != 1024) return 0;
  if (n2 == 1024 && dtype != F32) return 0;
  const int C = (int)(n2 / 32);
  if (!(k1 == 2 || k1 == 4 || k1 == 8 || (k1 == 16 && C >= 16))) return 0;
  if (mode == ROW_WIN && k2 != k1) return 0;
  if (mode == ROW_WIN && k2 > C) return 0;
  const int es = dtype == F32 ? 4 : 8;
  const int VE = 16 / es;
  const int PSV = (C / VE + 1) | 1;
  const int64_t U = (16 / k1) * k1;
  const int HV = strip ? (int)((k1 - 1 + VE - 1) / VE) : 0;
  const size_t smem = ((size_t)2 * U * (n2 + HV * VE) + (size_t)U * (strip ? 33 : 32) * PSV * VE) * es;
  return smem <= 220 * 1024 ? 1 : 0;
}

int launch_fused_pair_f32(const void*, void*, int64_t, int64_t, int64_t, int64_t, int64_t, int,
                          const void*, const void*, cudaStream_t);
int launch_fused_pair_f64(const void*, void*, int64_t, int64_t, int64_t, int64_t, int64_t, int,
                          const void*, const void*, cudaStream_t);
int launch_fused_pair_i64add(const void*, void*, int64_t, int64_t, int64_t, int64_t, int64_t, int,
                             const void*, const void*, cudaStream_t);
int launch_fused_pair_i64max(const void*, void*, int64_t, int64_t, int64_t, int64_t, int64_t, int,
                             const void*, const void*, cudaStream_t);

int launch_fused_pair(int dtype, int op, const void* in, void* out, int64_t outer, int64_t n1,
                      int64_t n2, int64_t k1, int64_t k2, int mode, const void* total,
                      const void* Tail, cudaStream_t s) {
  if (dtype == F32 && op == ADD)
    return launch_fused_pair_f32(in, out, outer, n1, n2, k1, k2, mode, total, Tail, s);
  if (dtype == F64 && op == ADD)
    return launch_fused_pair_f64(in, out, outer, n1, n2, k1, k2, mode, total, Tail, s);
  if (dtype == I64 && op == ADD)
    return launch_fused_pair_i64add(in, out, outer, n1, n2, k1, k2, mode, total, Tail, s);
  if (dtype == I64 && op == MAX)
    return launch_fused_pair_i64max(in, out, outer, n1, n2, k1, k2, mode, nullptr, Tail, s);
  return -2;
}

}  // namespace exsum

// bw_probe.cu -- what a plain streaming kernel reaches on this B200 at the
// array sizes of the BASELINE configs (read-only, write-only, copy), so the
// per-pass fractions of the small configs (C2 / C3: 64-268 MB, 20-50 us per
// launch) can be read against the same-size ceiling instead of the 2 GiB copy
// peak of MEASURED_PEAKS.json.  Not part of the product.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bw_probe tools/bw_probe.cu
//   tools/bw_probe            (prints one JSON line per size x kind x grid)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_read(const int4* __restrict__ a, size_t n16, unsigned long long* sink) {
  unsigned int acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    int4 v0 = __ldcs(a + i), v1 = __ldcs(a + i + stride);
    int4 v2 = __ldcs(a + i + 2 * stride), v3 = __ldcs(a + i + 3 * stride);
    acc ^= v0.x ^ v0.w ^ v1.y ^ v1.z ^ v2.x ^ v2.y ^ v3.z ^ v3.w;
  }
  for (; i < n16; i += stride) { int4 v = __ldcs(a + i); acc ^= v.x ^ v.w; }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

__global__ void k_write(int4* __restrict__ b, size_t n16) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  int4 z = make_int4(1, 2, 3, 4);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) __stcs(b + i, z);
}

__global__ void k_copy(const int4* __restrict__ a, int4* __restrict__ b, size_t n16) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + stride < n16; i += 2 * stride) {
    int4 v0 = __ldcs(a + i), v1 = __ldcs(a + i + stride);
    __stcs(b + i, v0); __stcs(b + i + stride, v1);
  }
  for (; i < n16; i += stride) __stcs(b + i, __ldcs(a + i));
}

// argv[1] = "clean": after the memset flush, read a second 512 MB buffer so the lines the
// timed kernel evicts are clean (no write-back of the flush's dirty lines inside the events)
int main(int argc, char** argv) {
  const bool clean = argc > 1 && argv[1][0] == 'c';
  const size_t sizes_mb[] = {64, 134, 268, 1074, 4295};
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  size_t maxb = 4295ull << 20;
  char *a, *b, *flush; unsigned long long* sink;
  CK(cudaMalloc(&a, maxb)); CK(cudaMalloc(&b, maxb)); CK(cudaMalloc(&flush, 512ull << 20));
  CK(cudaMalloc(&sink, 8));
  char* flush2 = nullptr;
  if (clean) { CK(cudaMalloc(&flush2, 512ull << 20)); CK(cudaMemset(flush2, 3, 512ull << 20)); }
  CK(cudaMemset(a, 1, maxb)); CK(cudaMemset(b, 0, maxb));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const int grids[] = {1, 2, 4, 8, 16};
  for (size_t mb : sizes_mb) {
    size_t bytes = mb << 20, n16 = bytes / 16;
    for (int kind = 0; kind < 3; ++kind) {
      for (int gm : grids) {
        int grid = sms * gm * (kind == 0 ? 1 : 1);
        float best = 1e30f, sum = 0.f; int reps = mb > 1000 ? 5 : 20;
        for (int r = 0; r < reps + 2; ++r) {
          CK(cudaMemsetAsync(flush, r, 512ull << 20));  // L2 flush outside the events
          if (clean) k_read<<<sms * 8, 512>>>((const int4*)flush2, (512ull << 20) / 16, sink);
          CK(cudaEventRecord(e0));
          if (kind == 0) k_read<<<grid, 512>>>((const int4*)a, n16, sink);
          else if (kind == 1) k_write<<<grid, 512>>>((int4*)b, n16);
          else k_copy<<<grid, 512>>>((const int4*)a, (int4*)b, n16 / 2);
          CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
          float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
          if (r >= 2) { best = ms < best ? ms : best; sum += ms; }
        }
        // copy moves bytes/2 in + bytes/2 out: `bytes` of traffic like the others
        double gbs_best = bytes / (best * 1e-3) / 1e9, gbs_avg = bytes / (sum / reps * 1e-3) / 1e9;
        printf("{\"flush\": \"%s\", \"kind\": \"%s\", \"traffic_MB\": %zu, \"grid\": %d, \"best_us\": %.2f, "
               "\"avg_us\": %.2f, \"GBps_best\": %.0f, \"GBps_avg\": %.0f}\n",
               clean ? "write+read" : "write", kind == 0 ? "read" : kind == 1 ? "write" : "copy", mb, grid, best * 1e3,
               sum / reps * 1e3, gbs_best, gbs_avg);
      }
    }
  }
  return 0;
}

// pdl_probe.cu -- what programmatic dependent launch (griddepcontrol) saves at
// a kernel boundary on this B200: a chain of dependent streaming passes
// (b = f(a), c = f(b), ...) over a small array, launched plainly and with the
// programmatic-stream-serialization attribute (every kernel triggers its
// dependents at its start and waits for its predecessor before its first
// load).  Not part of the product.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/pdl_probe tools/pdl_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <bool PDL>
__global__ void k_pass(const int4* __restrict__ a, int4* __restrict__ b, size_t n16) {
  if (PDL) {
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
    int4 v = __ldcs(a + i);
    v.x += 1;
    __stcs(b + i, v);
  }
}

template <bool PDL>
static cudaError_t launch(const int4* a, int4* b, size_t n16, int grid, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid); cfg.blockDim = dim3(256); cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at; cfg.numAttrs = PDL ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k_pass<PDL>, a, b, n16);
}

int main() {
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaStream_t s; CK(cudaStreamCreate(&s));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  for (size_t mb : {8, 64, 128}) {
    size_t bytes = mb << 20, n16 = bytes / 16;
    int4 *a, *b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
    CK(cudaMemset(a, 0, bytes));
    for (int chain : {1, 2, 4}) {
      for (int mode = 0; mode < 4; ++mode) {  // 0 plain, 1 pdl, 2 plain graph, 3 pdl graph
        const bool pdl = mode & 1, graph = mode & 2;
        cudaGraphExec_t exec = nullptr;
        auto enqueue = [&]() -> cudaError_t {
          for (int c = 0; c < chain; ++c) {
            const int4* src = (c & 1) ? b : a; int4* dst = (c & 1) ? a : b;
            cudaError_t e = pdl ? launch<true>(src, dst, n16, sms * 8, s) : launch<false>(src, dst, n16, sms * 8, s);
            if (e != cudaSuccess) return e;
          }
          return cudaSuccess;
        };
        if (graph) {
          cudaGraph_t g;
          CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
          CK(enqueue());
          CK(cudaStreamEndCapture(s, &g));
          CK(cudaGraphInstantiate(&exec, g, 0));
          CK(cudaGraphDestroy(g));
        }
        float sum = 0; const int reps = 30;
        for (int r = 0; r < reps + 3; ++r) {
          CK(cudaEventRecord(e0, s));
          if (graph) CK(cudaGraphLaunch(exec, s)); else CK(enqueue());
          CK(cudaEventRecord(e1, s)); CK(cudaEventSynchronize(e1));
          float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
          if (r >= 3) sum += ms;
        }
        printf("{\"array_MB\": %zu, \"chain\": %d, \"mode\": \"%s%s\", \"us\": %.2f}\n", mb, chain,
               pdl ? "pdl" : "plain", graph ? "+graph" : "", sum / reps * 1e3);
        if (exec) CK(cudaGraphExecDestroy(exec));
      }
    }
    CK(cudaFree(a)); CK(cudaFree(b));
  }
  return 0;
}

// l2pipe.cu -- the C4 shape (float32 [n0, n1, 1024], cubic box 16) with the
// axis-0 intermediate kept in L2: one persistent kernel instead of two HBM
// round trips.
//
// bdbs_included (included.py:124-129) runs windowed_sum_axis (scan.py:61-102)
// along axes 0, 1, 2; box-complement (excluded.py:129-159, restated in
// exsum_capi.cu) needs the same axis-0 and axis-1 passes before its row round.
// The two-kernel schedule (axis_stream, then fused_pair) writes the axis-0
// result W0 to HBM and reads it back: 4 N s.  Here the grid is split:
//   * producer CTAs (one per row y of a band of Yb + 15 rows) stream their row
//     down axis 0 exactly as k_axis_stream does (cp.async ring, suffix and
//     stitch in registers) and write W0 into a ring of R plane slots that
//     lives in L2, signalling each finished block of 16 planes;
//   * consumer CTAs take the band's planes in turn, wait for that block, and
//     run the fused pass pair (axis 1 window + the row op) exactly as
//     k_fused_pair does, reading W0 from L2 and writing the output once;
//     finishing a plane frees its ring slot.
// HBM then carries the input (+15 halo rows per band, ~1.23 N s at Yb = 64)
// and the output (N s).  Same association as the two-kernel schedule, so the
// results are bit-identical to it.  Bands run one after another; producers
// wait for ring space, consumers for data (gpu-scope release/acquire on
// per-block counters); the grid is co-resident by cooperative launch, and
// every wait has a watchdog that sets an error flag instead of hanging.
// Opt-in (EXSUM_L2PIPE=1): measured SLOWER than the two-kernel schedule on
// C4 (BDBS 4.4 ms vs 2.7 ms, box-complement 5.0 vs 2.9; DRAM traffic as
// planned, 5.2 GB read / 4.4 GB written).  Splitting the SMs by role halves
// the SMs each half of the work gets, and both standalone kernels already
// run near their per-SM limit (~43 GB/s per SM at 1 CTA per SM), so each role
// takes ~2x its standalone time.  The next form gives every CTA both kinds of
// work from one ordered queue.  Bit-exact with the
// two-kernel schedule for bdbs (tests/test_gpu_l2pipe.py).
#include <stdlib.h>

#include "exsum_common.cuh"
#include "exsum_launch.h"

namespace exsum {
namespace {

constexpr int LP_N2 = 1024;                     // row length
constexpr int LP_VE = 4;                        // floats per 16-byte vector
constexpr int LP_NT = LP_N2 / LP_VE;            // 256 threads: one column vector each
constexpr int LP_NW = LP_NT / 32;               // 8 warps
constexpr int LP_K = 16;                        // window along every axis
constexpr int LP_U = 16;                        // rows per streaming unit (one block)
constexpr int LP_C = LP_N2 / 32;                // row-op chunk per lane
constexpr int LP_CV = LP_C / LP_VE;             // vectors per chunk
constexpr int LP_CH = ((LP_CV + 1) | 1) * LP_VE;  // padded chunk stride (odd vectors)
constexpr int LP_ROWP = 32 * LP_CH;             // padded stage row
constexpr int LP_M2 = LP_C / LP_K;              // row-op blocks per chunk
constexpr int LP_RPW = LP_U / LP_NW;            // stage rows per warp
typedef Vec<float, LP_VE> F4;

struct LPArgs {
  const float* A;
  float* out;
  float* ring;     // [R][rows_p][1024]
  int* ready;      // [nbands][n0 / 16]: producer rows done per block of planes
  int* done;       // [nbands * n0 / 16]: consumer planes done per block
  int* err;        // watchdog
  const float* Tail;  // box-complement tail T [n0][n1] (mode 1)
  int64_t n0, n1;
  int Yb, rows_p, R, nbands, nprod, ncons, mode, sig;
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// the calling thread waits for *p >= target; a stuck wait (~2 s) flags err
// and gives up
__device__ __forceinline__ void lp_wait_t0(const int* p, int target, int* err) {
  const long long t0 = clock64();
  while (ld_acquire(p) < target) {
    if (*(volatile int*)err) break;
    if (clock64() - t0 > (4LL << 30)) {
      atomicExch(err, 1);
      break;
    }
    __nanosleep(100);
  }
}
// thread 0 waits, then the CTA
__device__ __forceinline__ void lp_wait(const int* p, int target, int* err) {
  if (threadIdx.x == 0) lp_wait_t0(p, target, err);
  __syncthreads();
}

// release: the CTA barrier orders every thread's stores before thread 0's
// gpu-scope fence (cumulative), then the counter bump (as a grid sync does);
// a fence in every thread invalidated L1 256 times per unit (ERRBAR +
// CCTL.IVALL each)
__device__ __forceinline__ void lp_signal(int* p) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(p, 1);
  }
}

// Producer: row `strip` of band `band`, all planes: W0 into the ring.
__device__ void lp_produce(const LPArgs& a, int band, int strip, float* raw) {
  const int tid = threadIdx.x;
  const int col = tid * LP_VE;
  const int64_t y = (int64_t)band * a.Yb + strip;
  const int64_t P = a.n1 * LP_N2;
  const float* src = a.A + y * LP_N2 + col;
  const int nunits = (int)(a.n0 / LP_U);
  const int64_t q0 = (int64_t)band * a.n0;
  const int64_t pstride = (int64_t)a.rows_p * LP_N2;
  auto issue = [&](int ui) {
    if (ui < nunits) {
      float* d = raw + (ui & 1) * (LP_U * LP_N2) + col;
      for (int r = 0; r < LP_U; ++r) cp_async16(d + r * LP_N2, src + ((int64_t)ui * LP_U + r) * P);
    }
    cp_async_commit();
  };
  issue(0);
  issue(1);
  cp_async_wait<1>();
  F4 cur[LP_U];
#pragma unroll
  for (int r = 0; r < LP_U; ++r) cur[r] = *reinterpret_cast<const F4*>(raw + col + r * LP_N2);
  issue(2);
  for (int u = 0; u < nunits; ++u) {
    const bool has_next = u + 1 < nunits;
    F4 nxt[LP_U];
    if (has_next) {
      cp_async_wait<1>();
      const float* sn = raw + ((u + 1) & 1) * (LP_U * LP_N2) + col;
#pragma unroll
      for (int r = 0; r < LP_U; ++r) nxt[r] = *reinterpret_cast<const F4*>(sn + r * LP_N2);
    }
    issue(u + 3);
    // in-block suffix S (right nested)
#pragma unroll
    for (int r = LP_U - 2; r >= 0; --r)
#pragma unroll
      for (int j = 0; j < LP_VE; ++j) cur[r].v[j] = cur[r].v[j] + cur[r + 1].v[j];
    // the ring slots of these 16 planes held the planes R earlier: wait until consumed
    const int64_t q = q0 + (int64_t)u * LP_U;
    if (u % a.sig == 0 && q + (int64_t)a.sig * LP_U > a.R) {
      // every sig units: the slots of the next sig blocks must be consumed
      if (threadIdx.x == 0)
        for (int i = 0; i < a.sig; ++i) {
          const int64_t qb = q + (int64_t)i * LP_U - a.R;
          if (qb >= 0 && u + i < nunits) lp_wait_t0(&a.done[qb / LP_U], LP_U, a.err);
        }
      __syncthreads();
    }
    float* dst = a.ring + ((q % a.R) * a.rows_p + strip) * LP_N2 + col;
    if (!has_next) {  // last block of axis 0: W = S
#pragma unroll
      for (int r = 0; r < LP_U; ++r) *reinterpret_cast<F4*>(dst + r * pstride) = cur[r];
    } else {
      *reinterpret_cast<F4*>(dst) = cur[0];
      F4 Pv = nxt[0];
#pragma unroll
      for (int r = 1; r < LP_U; ++r) {
        if (r - 1 >= 1)
#pragma unroll
          for (int j = 0; j < LP_VE; ++j) Pv.v[j] = Pv.v[j] + nxt[r - 1].v[j];
        F4 w;
#pragma unroll
        for (int j = 0; j < LP_VE; ++j) w.v[j] = cur[r].v[j] + Pv.v[j];
        *reinterpret_cast<F4*>(dst + r * pstride) = w;
      }
    }
    if (u % a.sig == a.sig - 1 || !has_next) {
      // one release for the last sig blocks (a fence per unit drained the
      // cp.async pipeline every 64 KB)
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        for (int b = u - u % a.sig; b <= u; ++b) atomicAdd(&a.ready[(int64_t)band * nunits + b], 1);
      }
    }
    if (has_next) {
#pragma unroll
      for (int r = 0; r < LP_U; ++r) cur[r] = nxt[r];
    }
  }
  cp_async_wait<0>();
  __syncthreads();
}

// Consumer: plane x0 of band `band` -- axis-1 window + row op from the ring.
__device__ void lp_consume(const LPArgs& a, int band, int64_t x0, float* raw, float* wst) {
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int col = tid * LP_VE;
  const int pcol = (col / LP_C) * LP_CH + (col % LP_C);
  const int64_t y0 = (int64_t)band * a.Yb;
  const int rows = (int)(a.n1 - y0 < a.rows_p ? a.n1 - y0 : a.rows_p);  // W0 rows present
  const int nout = (int)(a.n1 - y0 < a.Yb ? a.n1 - y0 : a.Yb);
  const int nunits = (int)(a.n0 / LP_U);
  const int64_t q = (int64_t)band * a.n0 + x0;
  lp_wait(&a.ready[(int64_t)band * nunits + x0 / LP_U], rows, a.err);
  const float* src = a.ring + (q % a.R) * a.rows_p * LP_N2 + col;
  float* dst = a.out + (x0 * a.n1 + y0) * LP_N2 + col;
  const float* tl = a.Tail ? a.Tail + x0 * a.n1 + y0 : nullptr;
  const int u_end = (nout + LP_U - 1) / LP_U;
  const int last_bs = LP_K * ((rows - 1) / LP_K);
  auto rows_of = [&](int ui) -> int {
    const int avail = rows - ui * LP_U;
    const int want = ui >= u_end ? LP_K - 1 : LP_U;
    return avail < want ? (avail > 0 ? avail : 0) : want;
  };
  auto issue = [&](int ui) {
    const int nr = rows_of(ui);
    float* d = raw + (ui & 1) * (LP_U * LP_N2) + col;
    for (int r = 0; r < nr; ++r) cp_async16(d + r * LP_N2, src + ((int64_t)ui * LP_U + r) * LP_N2);
    cp_async_commit();
  };
  issue(0);
  issue(1);
  cp_async_wait<1>();
  F4 cur[LP_U];
  int len = rows_of(0);
#pragma unroll
  for (int r = 0; r < LP_U; ++r)
    if (r < len) cur[r] = *reinterpret_cast<const F4*>(raw + col + r * LP_N2);
  issue(2);
  for (int u = 0; u < u_end; ++u) {
    const int us = u * LP_U;
    const int rows_u = len;
    float tails[LP_RPW];
    if (a.mode == 1) {
#pragma unroll
      for (int i = 0; i < LP_RPW; ++i) {
        const int rr = warp + i * LP_NW;
        tails[i] = rr < rows_u ? tl[us + rr] : 0.f;
      }
    }
    const int nlen_u = rows_of(u + 1);
    const float* sn = raw + ((u + 1) & 1) * (LP_U * LP_N2) + col;
    F4 nxt[LP_U];
    if (nlen_u > 0) {
      cp_async_wait<1>();
#pragma unroll
      for (int r = 0; r < LP_U; ++r)
        if (r < nlen_u) nxt[r] = *reinterpret_cast<const F4*>(sn + r * LP_N2);
    }
    issue(u + 3);
    // ---- axis-1 window on the unit (one block of 16 rows)
    {
      const int bs = us;
      const int blen = rows - bs < LP_K ? rows - bs : LP_K;
#pragma unroll
      for (int r = LP_K - 2; r >= 0; --r)
        if (r < blen - 1)
#pragma unroll
          for (int j = 0; j < LP_VE; ++j) cur[r].v[j] = cur[r].v[j] + cur[r + 1].v[j];
      if (bs == last_bs) {
#pragma unroll
        for (int r = 0; r < LP_K; ++r)
          if (r < blen) *reinterpret_cast<F4*>(wst + r * LP_ROWP + pcol) = cur[r];
      } else {
        const int nrows = rows - bs - LP_K;
        const int nlen = nrows < LP_K ? nrows : LP_K;
        *reinterpret_cast<F4*>(wst + pcol) = cur[0];
        F4 Pv = nxt[0];
#pragma unroll
        for (int r = 1; r < LP_K; ++r) {
          const int jj = r - 1;
          if (jj >= 1 && jj < nlen)
#pragma unroll
            for (int j = 0; j < LP_VE; ++j) Pv.v[j] = Pv.v[j] + nxt[jj].v[j];
          F4 w;
#pragma unroll
          for (int j = 0; j < LP_VE; ++j) w.v[j] = cur[r].v[j] + Pv.v[j];
          *reinterpret_cast<F4*>(wst + r * LP_ROWP + pcol) = w;
        }
      }
    }
    len = nlen_u;
    if (u + 1 < u_end) {
#pragma unroll
      for (int r = 0; r < LP_U; ++r) cur[r] = nxt[r];
    }
    __syncthreads();
    // ---- row op: windowed along the row (mode 0), or the box-complement
    // row round (row total + tail) - window (mode 1), warp per row
#pragma unroll
    for (int ri = 0; ri < LP_RPW; ++ri) {
      const int rr = warp + ri * LP_NW;
      if (rr < rows_u) {
        float* wrow = wst + rr * LP_ROWP;
        float* mine = wrow + lane * LP_CH;
        float av[LP_C];
#pragma unroll
        for (int v = 0; v < LP_CV; ++v) {
          const F4 t = *reinterpret_cast<const F4*>(mine + v * LP_VE);
#pragma unroll
          for (int j = 0; j < LP_VE; ++j) av[v * LP_VE + j] = t.v[j];
        }
        constexpr int NBV = LP_K / LP_VE;
        F4 nbv[NBV];
        if (lane < 31) {
#pragma unroll
          for (int v = 0; v < NBV; ++v)
            nbv[v] = *reinterpret_cast<const F4*>(wrow + (lane + 1) * LP_CH + v * LP_VE);
        }
#pragma unroll
        for (int jb = 0; jb < LP_M2; ++jb) {
#pragma unroll
          for (int r = LP_K - 2; r >= 0; --r) av[jb * LP_K + r] = av[jb * LP_K + r] + av[jb * LP_K + r + 1];
          const bool lastb = (lane == 31) && (jb == LP_M2 - 1);
          if (!lastb) {
            if (jb + 1 < LP_M2) {
              float Pr = av[(jb + 1) * LP_K];
#pragma unroll
              for (int r = 1; r < LP_K; ++r) {
                if (r >= 2) Pr = Pr + av[(jb + 1) * LP_K + r - 1];
                av[jb * LP_K + r] = av[jb * LP_K + r] + Pr;
              }
            } else {
              float Pr = nbv[0].v[0];
#pragma unroll
              for (int r = 1; r < LP_K; ++r) {
                if (r >= 2) Pr = Pr + nbv[(r - 1) / LP_VE].v[(r - 1) % LP_VE];
                av[jb * LP_K + r] = av[jb * LP_K + r] + Pr;
              }
            }
          }
        }
        float etail = 0.f;
        if (a.mode == 1) {
          // block heads hold the block totals (the stitch never touches them)
          float lt = av[0];
#pragma unroll
          for (int jb = 1; jb < LP_M2; ++jb) lt = lt + av[jb * LP_K];
#pragma unroll
          for (int d = 16; d >= 1; d >>= 1) lt = lt + __shfl_xor_sync(0xffffffffu, lt, d);
          etail = lt + tails[ri];
        }
        __syncwarp();
#pragma unroll
        for (int v = 0; v < LP_CV; ++v) {
          F4 t;
#pragma unroll
          for (int j = 0; j < LP_VE; ++j) {
            const float w = av[v * LP_VE + j];
            t.v[j] = a.mode == 1 ? etail - w : w;
          }
          *reinterpret_cast<F4*>(mine + v * LP_VE) = t;
        }
      }
      __syncwarp();
    }
    __syncthreads();
    for (int r = 0; r < rows_u; ++r)
      st_stream<float, LP_VE>(dst + (int64_t)(us + r) * LP_N2,
                              *reinterpret_cast<const F4*>(wst + r * LP_ROWP + pcol));
  }
  cp_async_wait<0>();
  lp_signal(&a.done[q / LP_U]);
}

__global__ void __launch_bounds__(LP_NT, 1) k_l2pipe(LPArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  float* raw = reinterpret_cast<float*>(smem);  // [2][16][1024]
  float* wst = raw + 2 * LP_U * LP_N2;         // [16][ROWP]
  const int cta = blockIdx.x;
  for (int band = 0; band < a.nbands; ++band) {
    const int64_t y0 = (int64_t)band * a.Yb;
    const int rows = (int)(a.n1 - y0 < a.rows_p ? a.n1 - y0 : a.rows_p);
    if (cta < a.nprod) {
      if (cta < rows) lp_produce(a, band, cta, raw);
    } else {
      for (int64_t x0 = cta - a.nprod; x0 < a.n0; x0 += a.ncons) lp_consume(a, band, x0, raw, wst);
    }
  }
}

int64_t lp_env(const char* name, int64_t dflt) {
  const char* e = getenv(name);
  return (e && *e) ? atoll(e) : dflt;
}

struct LPPlan {
  int Yb, rows_p, R, nbands, nprod, ncons, sig;
  size_t ring_bytes, ready_off, done_off, err_off, bytes;
};

bool lp_plan(int64_t n0, int64_t n1, LPPlan* p) {
  p->Yb = (int)lp_env("EXSUM_L2P_YB", 64);
  p->R = (int)lp_env("EXSUM_L2P_R", 128);
  p->sig = (int)lp_env("EXSUM_L2P_SIG", 1);
  if (p->Yb < 16 || p->Yb % 16 || p->R % 16 || p->sig < 1 || p->R < 2 * p->sig * LP_U) return false;
  p->rows_p = p->Yb + LP_K - 1;
  p->nbands = (int)((n1 + p->Yb - 1) / p->Yb);
  p->nprod = p->rows_p;
  p->ncons = num_sms() - p->nprod;
  if (p->ncons < 16) return false;
  const int64_t nblk = n0 / LP_U;
  p->ring_bytes = (size_t)p->R * p->rows_p * LP_N2 * sizeof(float);
  p->ready_off = (p->ring_bytes + 255) & ~(size_t)255;
  p->done_off = p->ready_off + (size_t)p->nbands * nblk * sizeof(int);
  p->err_off = p->done_off + (size_t)p->nbands * nblk * sizeof(int);
  p->bytes = p->err_off + 256;
  return true;
}

}  // namespace

int l2pipe_ok(int dtype, int op, int d, const int64_t* ext, const int64_t* k) {
  if (lp_env("EXSUM_L2PIPE", 0) != 1) return 0;
  if (dtype != F32 || op != ADD || d != 3) return 0;
  if (ext[2] != LP_N2 || k[0] != LP_K || k[1] != LP_K || k[2] != LP_K) return 0;
  if (ext[0] % LP_U || ext[1] % LP_U || ext[0] < 2 * LP_U || ext[1] < 2 * LP_U) return 0;
  LPPlan p;
  return lp_plan(ext[0], ext[1], &p) ? 1 : 0;
}

size_t l2pipe_workspace_bytes(const int64_t* ext) {
  LPPlan p;
  if (!lp_plan(ext[0], ext[1], &p)) return 0;
  return p.bytes;
}

// mode 0: bdbs (windowed row op); mode 1: box-complement rows with tail T.
// ws: l2pipe_workspace_bytes() bytes.  Returns launches, or -1.
int launch_l2pipe(int mode, const void* in, void* out, const int64_t* ext, const void* Tail,
                  void* ws, cudaStream_t s) {
  LPPlan p;
  if (!lp_plan(ext[0], ext[1], &p)) return -1;
  const size_t smem = ((size_t)2 * LP_U * LP_N2 + (size_t)LP_U * LP_ROWP) * sizeof(float);
  ensure_smem((const void*)k_l2pipe, smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_l2pipe, LP_NT, smem);
  if (per_sm < 1) return -1;
  char* base = (char*)ws;
  cudaMemsetAsync(base + p.ready_off, 0, p.bytes - p.ready_off, s);
  LPArgs a;
  a.A = (const float*)in;
  a.out = (float*)out;
  a.ring = (float*)base;
  a.ready = (int*)(base + p.ready_off);
  a.done = (int*)(base + p.done_off);
  a.err = (int*)(base + p.err_off);
  a.Tail = (const float*)Tail;
  a.n0 = ext[0];
  a.n1 = ext[1];
  a.Yb = p.Yb;
  a.rows_p = p.rows_p;
  a.R = p.R;
  a.nbands = p.nbands;
  a.nprod = p.nprod;
  a.ncons = p.ncons;
  a.mode = mode;
  a.sig = p.sig;
  void* args[] = {&a};
  const unsigned grid = (unsigned)(p.nprod + p.ncons);
  if (cudaLaunchCooperativeKernel((const void*)k_l2pipe, dim3(grid), dim3(LP_NT), args, smem, s) !=
      cudaSuccess)
    return -1;
  return 1;
}

}  // namespace exsum

// sa_common.cuh -- small device/host helpers shared by the library's kernels (not by the oracle).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/simplicial_attn.h"

namespace sa {

// Problem description handed to every kernel.  Key-side tensors have NK = np + N rows.
struct Problem {
  int B, H, N, D, w1, w2, np;  // np = n_prefix
  int Hk;                      // key/value heads (GQA: query head h reads key head h / (H / Hk)); = H otherwise
  int hk_shift;                // log2(H / Hk) when that ratio is a power of two (the usual case), else -1
  float scale;                 // signed logit scale (negated when the DET operands are swapped)
  bool det;
  // Lowest valid K' row index (0 normally).  The backward / forward of a window w2 > 32 runs as
  // w2/32 sub-problems of window 32 whose K' rows are shifted by d: the
  // kernels see K' through a pointer offset by -d rows, so virtual rows < k2lo = d do not exist.
  int k2lo;
  __host__ __device__ int NK() const { return np + N; }
  __host__ __device__ int hk(int h) const { return hk_shift >= 0 ? h >> hk_shift : h / (H / Hk); }
  // element offsets of row (b, pos, h) in query-side tensors and in per-query-head key-side
  // tensors (gradient partials: [B, NK, H, D]) ...
  __host__ __device__ int64_t qoff(int b, int i, int h) const {
    return ((int64_t(b) * N + i) * H + h) * D;
  }
  __host__ __device__ int64_t koff(int b, int j, int h) const {
    return ((int64_t(b) * NK() + j) * H + h) * D;
  }
  // ... and of the key row that query head h reads in the key-side inputs ([B, NK, Hk, D])
  __host__ __device__ int64_t kroff(int b, int j, int h) const {
    return ((int64_t(b) * NK() + j) * Hk + hk(h)) * D;
  }
  // the same with the key head already resolved (hot loops: resolve once per work item)
  __host__ __device__ int64_t kvoff(int b, int j, int hkv) const {
    return ((int64_t(b) * NK() + j) * Hk + hkv) * D;
  }
  __host__ __device__ size_t nkey() const { return size_t(B) * NK() * Hk * D; }
};

// Division by a runtime divisor 1 <= d < 2^31 for 0 <= n < 2^31 by a host-computed reciprocal:
// q = mulhi(n, ceil(2^32 / d)) is q or q+1, one correction step makes it exact.  A few instructions
// instead of the ~25 of an integer division on the kernels' per-tile index paths.  d = 1 (whose
// reciprocal 2^32 does not fit 32 bits) is a separate, warp-uniform branch.
struct FastDiv {
  int d;
  uint32_t m;
  FastDiv() = default;
  __host__ explicit FastDiv(int d_)
      : d(d_), m(d_ > 1 ? uint32_t((0x100000000ull + uint64_t(d_) - 1) / uint64_t(d_)) : 0u) {}
  __device__ __forceinline__ int div(int n) const {
    if (d == 1) return n;
    int q = int(__umulhi(uint32_t(n), m));
    if (n - q * d < 0) --q;
    return q;
  }
  __device__ __forceinline__ int mod(int n) const {
    if (d == 1) return 0;
    int r = n - int(__umulhi(uint32_t(n), m)) * d;
    if (r < 0) r += d;
    return r;
  }
};

__device__ __forceinline__ float ld_f(const float* p) { return __ldg(p); }
__device__ __forceinline__ float ld_f(const __nv_bfloat16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ void st_f(float* p, float x) { *p = x; }
__device__ __forceinline__ void st_f(__nv_bfloat16* p, float x) { *p = __float2bfloat16_rn(x); }

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
__device__ __forceinline__ float warp_max(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

// Window lower bound: key rows (pos - w, pos], clipped at 0.
__host__ __device__ __forceinline__ int win_lo(int pos, int w) { return pos - w + 1 > 0 ? pos - w + 1 : 0; }

// Launch bookkeeping (sa_api.cu).
void note_launch(int n = 1);

// Brackets one kernel launch with CUDA events on `st` while profiling is enabled (sa_api.cu).
struct KernelScope {
  KernelScope(const char* name, cudaStream_t st);
  ~KernelScope();
  int slot;
  cudaStream_t st;
};

}  // namespace sa

// ---- optional phase tracing (tools/trace_build.py builds a separate library with -DSA_TRACE) ----
// SA_TRACE_AT(cond, region, n, tag): when cond holds in CTA 0, store (tag, clock64) at
// g_trace[region*1024 + 2n] and bump the caller's register counter n (no atomics, ~no overhead).
#ifdef SA_TRACE
namespace sa {
extern __device__ unsigned long long g_trace[8192];
extern __device__ unsigned int g_trace_n;
}
#define SA_TRACE_AT(cond, region, n, tag)                                                   \
  do {                                                                                     \
    if ((cond) && blockIdx.x == 0 && blockIdx.y == 0 && (n) < 511) {                       \
      ::sa::g_trace[(region) * 1024 + 2 * (n)] = (unsigned long long)(tag);               \
      ::sa::g_trace[(region) * 1024 + 2 * (n) + 1] = (unsigned long long)clock64();       \
      ++(n);                                                                               \
    }                                                                                      \
  } while (0)
#define SA_TRACE_POINT(cond, tag) \
  do {                            \
  } while (0)
#else
#define SA_TRACE_AT(cond, region, n, tag) \
  do {                                    \
  } while (0)
#define SA_TRACE_POINT(cond, tag) \
  do {                            \
  } while (0)
#endif

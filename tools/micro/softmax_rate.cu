// Microbenchmark: cycles for one 32-column softmax-gradient step (the bwd_kv fast path: FFMA2,
// 32x MUFU.EX2, F2FP, FADD2, FMUL2) per warp, with W warps per SM (1 or 2 per SMSP).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../paper_2507_02754_b200/csrc/sa_tc_common.cuh"
using namespace sa::tc;

template <int W>
__global__ void __launch_bounds__(W * 32, 1) k(unsigned long long* out, float* sink, int iters) {
  uint32_t su[32], du[32];
  for (int i = 0; i < 32; ++i) {
    su[i] = __float_as_uint(-0.01f * (i + threadIdx.x % 7));
    du[i] = __float_as_uint(0.02f * i);
  }
  const float sl2 = 1.27f;
  float2 ri = make_float2(0.5f, 0.25f);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t pp[16], pd[16];
    const float2 vs = make_float2(sl2, sl2), vl = make_float2(-ri.x, -ri.x), vd = make_float2(-ri.y, -ri.y);
#pragma unroll
    for (int t2 = 0; t2 < 16; ++t2) {
      const float2 x = ffma2(make_float2(__uint_as_float(su[2 * t2]), __uint_as_float(su[2 * t2 + 1])), vs, vl);
      const float2 pv = make_float2(ex2(x.x), ex2(x.y));
      pp[t2] = pack_f16x2(pv);
      pd[t2] = pack_f16x2(fmul2(pv, fadd2(make_float2(__uint_as_float(du[2 * t2]), __uint_as_float(du[2 * t2 + 1])), vd)));
    }
#pragma unroll
    for (int t2 = 0; t2 < 16; ++t2) acc ^= pp[t2] + pd[t2];
    ri.x += 1e-7f * (acc & 1);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  if (acc == 0x12345) sink[0] = ri.x;
}

template <int W>
void run(unsigned long long* d, float* s) {
  const int iters = 4096;
  k<W><<<148, W * 32>>>(d, s, iters);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("warps/SM=%d: %.1f cycles per 32-col step per warp (MUFU bound %d)\n", W, double(h[0]) / iters,
         W <= 4 ? 256 : 256 * W / 4);
}
int main() {
  unsigned long long* d;
  float* s;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&s, 64);
  run<4>(d, s);
  run<8>(d, s);
  run<16>(d, s);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}

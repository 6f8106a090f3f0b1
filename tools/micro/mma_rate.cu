// Microbenchmark: tcgen05.mma kind::f16 issue-to-completion rate for SS (A,B in SMEM) and TS (A in
// TMEM) forms at M=128, N in {32,64,128,256}, K=16 per instruction; optional concurrent STS traffic
// from 8 other warps (the A-tile formation pattern).  One CTA per SM, 148 CTAs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../paper_2507_02754_b200/csrc/sa_tc_common.cuh"

using namespace sa::tc;

template <int N, bool TS, bool STS>
__global__ void __launch_bounds__(288, 1) k(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tbase_s;
  __shared__ uint64_t bar;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    stop = 0;
  }
  if (warp == 8) tmem_alloc<512>(&tbase_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tbase_s;
  const uint32_t base = (smem_u32(sm) + 1023) & ~1023u;
  if (warp == 8) {
    const uint32_t idesc = idesc_f16(128, N, 0, 0);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t bd = smem_desc_sw128(base + 65536 + kk * 32, 16, 1024);
        if (TS)
          mma_ts_w(tb + 256, tb + kk * 8, bd, idesc, 1u);
        else
          mma_ss_w(tb + 256, smem_desc_sw128(base + kk * 32, 16, 1024), bd, idesc, 1u);
      }
    }
    mma_commit_w(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 256) {
      out[blockIdx.x] = (unsigned long long)(t1 - t0);
      stop = 1;
    }
  } else if (STS) {
    // 8 warps streaming 16-byte stores into a 32 KB region (disjoint from the MMA operands)
    uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
    uint32_t a = base + 131072 + (threadIdx.x * 16) % 32768;
    while (!stop) {
#pragma unroll 8
      for (int r = 0; r < 64; ++r) {
        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a + (r * 4096) % 32768), "r"(v.x), "r"(v.y),
                     "r"(v.z), "r"(v.w));
      }
    }
  }
  __syncthreads();
  if (warp == 8) tmem_free<512>(tb);
}

template <int N, bool TS, bool STS>
void run(unsigned long long* d) {
  const int iters = 2000;
  const int smem = 131072 + 32768 + 1024;
  cudaFuncSetAttribute(k<N, TS, STS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<N, TS, STS><<<148, 288, smem>>>(d, iters);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  const double per = mx / (iters * 8.0);
  const double flop = 2.0 * 128 * N * 16;
  printf("%s N=%3d sts=%d: %6.1f cyc/MMA (floor %5.1f)  %6.0f flop/clk/SM  smem B/clk %.0f\n", TS ? "TS" : "SS", N,
         int(STS), per, 128.0 * N / 256, flop / per, (TS ? N * 32.0 : (128 + N) * 32.0) / per);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  run<32, false, false>(d);
  run<64, false, false>(d);
  run<128, false, false>(d);
  run<256, false, false>(d);
  run<16, true, false>(d);
  run<32, true, false>(d);
  run<64, true, false>(d);
  run<128, true, false>(d);
  run<256, true, false>(d);
  run<64, false, true>(d);
  run<128, false, true>(d);
  run<64, true, true>(d);
  run<128, true, true>(d);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

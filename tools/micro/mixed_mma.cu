// Does tcgen05.mma kind::f16 accept A in fp16 and B in bf16 (separate a/b format fields of the
// instruction descriptor)?  One CTA: D[128x32] = A[128x16] . B[32x16]^T with small integers (exact in
// both formats); prints the max error against the exact product for (fp16, fp16) and (fp16, bf16).
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../../paper_2507_02754_b200/csrc/sa_tc_common.cuh"

using namespace sa::tc;

__device__ __forceinline__ uint32_t swz(int row, int c8) { return uint32_t(row * 128 + (((c8 & 7) ^ (row & 7)) << 4)); }

__global__ void k(float* out, int bfmt) {
  __shared__ __align__(1024) uint8_t sa_[128 * 128];
  __shared__ __align__(1024) uint8_t sb_[32 * 128];
  __shared__ uint32_t tbase_s;
  __shared__ uint64_t bar;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  // A: 128 rows x 64 halves (only k < 16 used), B: 32 rows x 64
  for (int e = t; e < 128 * 64; e += 128) {
    const int r = e / 64, kk = e % 64;
    const __half v = __float2half(float((r + kk) % 5 - 2));
    *reinterpret_cast<__half*>(sa_ + swz(r, kk / 8) + (kk % 8) * 2) = v;
  }
  for (int e = t; e < 32 * 64; e += 128) {
    const int n = e / 64, kk = e % 64;
    const float f = float((n * 3 + kk) % 7 - 3);
    uint16_t bits;
    if (bfmt) {
      __nv_bfloat16 b = __float2bfloat16(f);
      bits = *reinterpret_cast<uint16_t*>(&b);
    } else {
      __half h = __float2half(f);
      bits = *reinterpret_cast<uint16_t*>(&h);
    }
    *reinterpret_cast<uint16_t*>(sb_ + swz(n, kk / 8) + (kk % 8) * 2) = bits;
  }
  if (t == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<32>(&tbase_s);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tbase_s;
  if (warp == 0) {
    const uint32_t idesc = (1u << 4) | (0u << 7) | (uint32_t(bfmt) << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
    mma_ss_w(tb, smem_desc_sw128(smem_u32(sa_), 16, 1024), smem_desc_sw128(smem_u32(sb_), 16, 1024), idesc, 0u);
    mma_commit_w(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t r[32];
  tmem_ld32(tb + (uint32_t(warp * 32) << 16), r);
  tmem_ld_wait();
  for (int n = 0; n < 32; ++n) out[(warp * 32 + lane) * 32 + n] = __uint_as_float(r[n]);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<32>(tb);
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 32 * 4);
  float h[128 * 32];
  for (int bfmt = 0; bfmt < 2; ++bfmt) {
    k<<<1, 128>>>(d, bfmt);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double err = 0;
    for (int r = 0; r < 128; ++r)
      for (int n = 0; n < 32; ++n) {
        double ref = 0;
        for (int kk = 0; kk < 16; ++kk) ref += double((r + kk) % 5 - 2) * double((n * 3 + kk) % 7 - 3);
        err = fmax(err, fabs(ref - h[r * 32 + n]));
      }
    printf("A fp16, B %s: max abs err %.3g (%s)\n", bfmt ? "bf16" : "fp16", err, cudaGetErrorString(e));
  }
  return 0;
}

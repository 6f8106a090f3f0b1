// sa_gqa.cu -- helpers of the grouped-query entry points (the paper's model
// uses a GQA ratio of 64): the backward kernels write per-query-head key-side gradient
// partials [B, NK, H, D] in fp32; the sum over the H/Hk query heads that share a key head and the
// conversion to the output dtype happen here.  Also the biased K'/V' copies of the bias entry points
// (K2_BIAS / V2_BIAS of the paper's kernel listing).
// Memory-bound elementwise kernels.
#include "sa_common.cuh"

namespace sa {
namespace {

template <typename TOut>
__global__ void __launch_bounds__(256) gqa_reduce_kernel(const float* __restrict__ part, TOut* __restrict__ out,
                                                         int64_t rows, int Hk, int r, int D) {
  // rows = B * NK; out [rows, Hk, D]; part [rows, Hk * r, D]
  const int64_t total = rows * Hk * D;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int d = int(e % D);
    const int64_t t = e / D;
    const int hk = int(t % Hk);
    const int64_t row = t / Hk;
    const float* src = part + ((row * Hk + hk) * r) * D + d;
    float acc = 0.f;
    for (int i = 0; i < r; ++i) acc += src[int64_t(i) * D];
    st_f(out + e, acc);
  }
}

__global__ void __launch_bounds__(256) f32_to_bf16_kernel(const float* __restrict__ a, __nv_bfloat16* __restrict__ b,
                                                          int64_t n) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x)
    b[e] = __float2bfloat16_rn(a[e]);
}

__global__ void __launch_bounds__(256) bf16_to_f32_kernel(const __nv_bfloat16* __restrict__ a, float* __restrict__ b,
                                                          int64_t n) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x)
    b[e] = __bfloat162float(a[e]);
}

// k2b = k2 + b2k, v2b = v2 + b2v elementwise (the tile is loaded in fp32, the scalar added,
// then cast to the GEMM dtype); bf16 elements are rounded once, fp32 ones exactly.  n counts the
// elements of each tensor.
template <typename T>
__global__ void __launch_bounds__(256) add_bias_kernel(const T* __restrict__ k2, const T* __restrict__ v2,
                                                       T* __restrict__ k2b, T* __restrict__ v2b, int64_t n,
                                                       float b2k, float b2v) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < 2 * n; e += stride) {
    const bool second = e >= n;
    const int64_t i = second ? e - n : e;
    const float b = second ? b2v : b2k;
    const T* src = second ? v2 : k2;
    T* dst = second ? v2b : k2b;
    if constexpr (sizeof(T) == 4)
      dst[i] = src[i] + b;
    else
      dst[i] = __float2bfloat16_rn(__bfloat162float(src[i]) + b);
  }
}

int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  return int(g > 148 * 16 ? 148 * 16 : (g < 1 ? 1 : g));
}

}  // namespace

cudaError_t gqa_reduce(const float* part, void* out, bool out_f32, int64_t rows, int Hk, int r, int D,
                       cudaStream_t st) {
  KernelScope ks("gqa_reduce", st);
  const int64_t n = rows * Hk * D;
  if (out_f32)
    gqa_reduce_kernel<float><<<grid_for(n), 256, 0, st>>>(part, (float*)out, rows, Hk, r, D);
  else
    gqa_reduce_kernel<__nv_bfloat16><<<grid_for(n), 256, 0, st>>>(part, (__nv_bfloat16*)out, rows, Hk, r, D);
  return cudaGetLastError();
}

cudaError_t add_bias(const void* k2, const void* v2, void* k2b, void* v2b, int64_t n, bool f32, float b2k,
                     float b2v, cudaStream_t st) {
  KernelScope ks("bias_add", st);
  if (f32)
    add_bias_kernel<float><<<grid_for(2 * n), 256, 0, st>>>((const float*)k2, (const float*)v2, (float*)k2b,
                                                            (float*)v2b, n, b2k, b2v);
  else
    add_bias_kernel<__nv_bfloat16><<<grid_for(2 * n), 256, 0, st>>>(
        (const __nv_bfloat16*)k2, (const __nv_bfloat16*)v2, (__nv_bfloat16*)k2b, (__nv_bfloat16*)v2b, n, b2k, b2v);
  return cudaGetLastError();
}

cudaError_t cast_f32_bf16(const float* a, void* b, int64_t n, cudaStream_t st) {
  KernelScope ks("gqa_cast", st);
  f32_to_bf16_kernel<<<grid_for(n), 256, 0, st>>>(a, (__nv_bfloat16*)b, n);
  return cudaGetLastError();
}

cudaError_t cast_bf16_f32(const void* a, float* b, int64_t n, cudaStream_t st) {
  KernelScope ks("gqa_cast", st);
  bf16_to_f32_kernel<<<grid_for(n), 256, 0, st>>>((const __nv_bfloat16*)a, b, n);
  return cudaGetLastError();
}

}  // namespace sa

// sa_split.cu -- window split of a long folded window (w2 > 32) into sub-windows of <= 32 rows
// (DESIGN.md "window split").  The K' window of query i, (i - w2, i], is the disjoint union of
//   W2_b(i) = (i - d_b - w_b, i - d_b],  d_b = 32 b,  w_b = min(32, w2 - d_b),  b = 0 .. nsplit-1,
// so every (j, k) cell of the joint softmax (Eq. attenval) belongs to exactly one sub-problem.
// Sub-problem b is a plain window-(w1, w_b) problem whose K' rows are shifted by d_b: the kernels see
// K', V' (and write dK', dV') through pointers offset by -d_b rows and treat virtual rows < d_b as
// absent (Problem::k2lo).  They run at R <= 32, the tiling whose rows stage in shared memory.
//   forward:  o = sum_b e^{lse_b - lse} o_b,  lse = log sum_b e^{lse_b}   (exact merge of disjoint
//             softmax blocks; a sub-problem with an empty window for query i has lse_b = -inf)
//   backward: every gradient is a sum over the cells, hence over the sub-problems, given the full
//             lse and delta = <dO, o>; the sub-problems write fp32 partials that are
//             summed here (dK'/dV' partial b covers rows [0, NK - d_b) of each batch element).
// Memory-bound elementwise kernels.
#include "sa_common.cuh"

namespace sa {
namespace {

__device__ __forceinline__ void store4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ void store4(__nv_bfloat16* p, float4 v) {
  __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&a);
  u.y = *reinterpret_cast<uint32_t*>(&b);
  *reinterpret_cast<uint2*>(p) = u;
}

// out[e] = sum_b part_b[e] over the sub-problems whose partial covers e's row: rows counts rows per
// batch element, row_stride elements per row (H * D), part b covers rows [0, rows - shift_b).
template <typename TOut>
__global__ void __launch_bounds__(256) split_sum_kernel(const float* __restrict__ part, int64_t part_stride, int nsplit,
                                                        int shift_step, TOut* __restrict__ out, int64_t total4,
                                                        int rows, int64_t row_stride) {
  const int64_t gstride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t e4 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e4 < total4; e4 += gstride) {
    const int64_t e = 4 * e4;
    const int row = int((e / row_stride) % rows);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int b = 0; b < nsplit; ++b) {
      if (row >= rows - shift_step * b) break;  // shifts grow with b
      const float4 v = *reinterpret_cast<const float4*>(part + b * part_stride + e);
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    store4(out + e, acc);
  }
}

// Forward merge over the sub-problems' (o_b fp32 [B,N,H,D], lse_b [B,H,N]).
template <typename TOut>
__global__ void __launch_bounds__(256) split_merge_kernel(const float* __restrict__ ob, const float* __restrict__ lb,
                                                          int nsplit, int64_t nq, int64_t nrows, TOut* __restrict__ o,
                                                          float* __restrict__ lse, int N, int H, int D) {
  // one warp per query row (b, i, h); lse layout [B, H, N]
  const int64_t w = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nrows) return;
  const int h = int(w % H);
  const int64_t bi = w / H;
  const int i = int(bi % N);
  const int64_t b = bi / N;
  const int64_t li = (b * H + h) * N + i;
  float m = -INFINITY;
  for (int s = 0; s < nsplit; ++s) m = fmaxf(m, lb[s * nrows + li]);
  float wsum = 0.f;
  float wt[8];
  for (int s = 0; s < nsplit; ++s) {
    const float l = lb[s * nrows + li];
    wt[s] = l == -INFINITY ? 0.f : __expf(l - m);
    wsum += wt[s];
  }
  if (lane == 0) lse[li] = m + logf(wsum);
  const float inv = 1.f / wsum;
  for (int d = 4 * lane; d < D; d += 128) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < nsplit; ++s) {
      if (wt[s] == 0.f) continue;  // an empty sub-window leaves o_b undefined (0/0)
      const float4 v = *reinterpret_cast<const float4*>(ob + s * nq + w * D + d);
      const float c = wt[s] * inv;
      acc.x += c * v.x;
      acc.y += c * v.y;
      acc.z += c * v.z;
      acc.w += c * v.w;
    }
    store4(o + w * D + d, acc);
  }
}

int grid_for(int64_t n) {
  const int64_t g = (n + 255) / 256;
  return int(g < 148 * 16 ? g : 148 * 16);
}

}  // namespace

cudaError_t split_sum(const float* part, int64_t part_stride, int nsplit, int shift_step, void* out, bool out_f32,
                      int64_t n, int rows, int64_t row_stride, cudaStream_t st) {
  if (n % 4 || row_stride % 4) return cudaErrorInvalidValue;
  KernelScope ks("tc_split_sum", st);
  if (out_f32)
    split_sum_kernel<float><<<grid_for(n / 4), 256, 0, st>>>(part, part_stride, nsplit, shift_step, (float*)out, n / 4,
                                                               rows, row_stride);
  else
    split_sum_kernel<__nv_bfloat16><<<grid_for(n / 4), 256, 0, st>>>(part, part_stride, nsplit, shift_step,
                                                                       (__nv_bfloat16*)out, n / 4, rows, row_stride);
  return cudaGetLastError();
}

cudaError_t split_merge(const float* ob, const float* lb, int nsplit, const Problem& p, void* o, float* lse,
                        bool out_f32, cudaStream_t st) {
  if (nsplit > 8 || p.D % 4) return cudaErrorInvalidValue;
  const int64_t nrows = int64_t(p.B) * p.N * p.H;
  const int64_t nq = nrows * p.D;
  const unsigned blocks = unsigned((nrows * 32 + 255) / 256);
  KernelScope ks("tc_split_merge", st);
  if (out_f32)
    split_merge_kernel<float><<<blocks, 256, 0, st>>>(ob, lb, nsplit, nq, nrows, (float*)o, lse, p.N, p.H, p.D);
  else
    split_merge_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(ob, lb, nsplit, nq, nrows, (__nv_bfloat16*)o, lse, p.N,
                                                                p.H, p.D);
  return cudaGetLastError();
}

}  // namespace sa

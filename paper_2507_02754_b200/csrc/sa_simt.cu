// sa_simt.cu -- exact-fp32 CUDA-core kernels for sliding-window 2-simplicial attention.
//
// These are the library's fp32 path (SA_IN_F32, BASELINE config c1) and its general-shape
// fallback (any D <= 128, any window).  They compute in fp32 with fp32 accumulation; the bf16
// tensor-core path lives in sa_tc_*.cu.  Algebra (verified in the oracle's
// tests): with the row operand a_(i,k) = s (q_i o k2_k)  [det: s (k2_k x q_i), chunkwise],
//   A_ijk = <a_(i,k), k_j>                                  (P:230-233 / P:298-301)
//   per (i,k) row: online softmax over j, U_(i,k) = sum_j p v_j (P:815-828 pattern)
//   o_i = sum_k e^{m_(i,k)-m_i} v2_k o U_(i,k) / l_i        (Eq. attenval)
// Backward (corrected): W_(i,k) = sum_j dS_ijk k_j and
//   dq_i = s sum_k k2_k o W (det: W x k2_k),  dk2_k = s sum_i q_i o W (det: q_i x W),
//   dv2_k = sum_i dO_i o U,  dk_j = sum_{i,k} dS a_(i,k),  dv_j = sum_{i,k} P (dO_i o v2_k).
// Three gather kernels (per query row, per K' row, per K row) recompute P from lse and
// delta_i = <dO_i, o_i>, so no atomics are needed ("recompute over atomics").
//
// Lane layout: a warp owns one row; lane l holds dims d = l + 32 t, t < NV (D <= 32 NV).
#include <math.h>

#include "sa_common.cuh"

namespace sa {
namespace {

constexpr int kWarps = 4;
constexpr int kThreads = 32 * kWarps;

// (x cross y)[d] for the 3-chunk containing d; 0 on the trailing D mod 3 dims (reading R5).
__device__ __forceinline__ float cross_at(const float* x, const float* y, int d, int D3) {
  if (d >= D3) return 0.f;
  int c = d - d % 3, r = d % 3;
  int r1 = c + (r + 1) % 3, r2 = c + (r + 2) % 3;
  return x[r1] * y[r2] - x[r2] * y[r1];
}

template <typename T, int NV>
__device__ __forceinline__ void load_row(const T* p, int D, int lane, float (&r)[NV]) {
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    int d = lane + 32 * t;
    r[t] = d < D ? ld_f(p + d) : 0.f;
  }
}

template <typename T>
__device__ __forceinline__ void load_row_smem(const T* p, int D, int lane, float* s) {
  for (int d = lane; d < D; d += 32) s[d] = ld_f(p + d);
}

// Row operand a = s (q o k2) or s (k2 x q), from fp32 rows in shared memory.
template <int NV>
__device__ __forceinline__ void row_operand(const Problem& p, const float* sq, const float* sk2,
                                            int lane, float (&a)[NV]) {
  int D3 = (p.D / 3) * 3;
#pragma unroll
  for (int t = 0; t < NV; ++t) {
    int d = lane + 32 * t;
    float x = 0.f;
    if (d < p.D) x = p.det ? cross_at(sk2, sq, d, D3) : sq[d] * sk2[d];
    a[t] = p.scale * x;
  }
}

template <int NV>
__device__ __forceinline__ float dot_lane(const float (&a)[NV], const float (&b)[NV]) {
  float x = 0.f;
#pragma unroll
  for (int t = 0; t < NV; ++t) x = fmaf(a[t], b[t], x);
  return x;
}

// ------------------------------------------------------------------------------------------
// Forward: one block per (query row i, b*H+h); warp w takes K' rows k0+w, k0+w+4, ...
// ------------------------------------------------------------------------------------------
template <typename TIn, typename TOut, int NV>
__global__ void __launch_bounds__(kThreads) simt_fwd(Problem p, const TIn* __restrict__ q,
                                                     const TIn* __restrict__ k, const TIn* __restrict__ v,
                                                     const TIn* __restrict__ k2, const TIn* __restrict__ v2,
                                                     TOut* __restrict__ o, float* __restrict__ lse) {
  const int i = blockIdx.x, bh = blockIdx.y, b = bh / p.H, h = bh % p.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ float sq[32 * NV];
  __shared__ float sk2[kWarps][32 * NV];
  __shared__ float sO[kWarps][32 * NV];
  __shared__ float sM[kWarps], sL[kWarps];
  const int pos = p.np + i;
  for (int d = threadIdx.x; d < p.D; d += kThreads) sq[d] = ld_f(q + p.qoff(b, i, h) + d);
  __syncthreads();
  const int j0 = win_lo(pos, p.w1), k0 = win_lo(pos, p.w2);

  float M = -INFINITY, L = 0.f, O[NV];
#pragma unroll
  for (int t = 0; t < NV; ++t) O[t] = 0.f;

  for (int kk = k0 + warp; kk <= pos; kk += kWarps) {
    load_row_smem(k2 + p.kroff(b, kk, h), p.D, lane, sk2[warp]);
    __syncwarp();
    float a[NV];
    row_operand<NV>(p, sq, sk2[warp], lane, a);
    float m = -INFINITY, l = 0.f, U[NV];
#pragma unroll
    for (int t = 0; t < NV; ++t) U[t] = 0.f;
    for (int j = j0; j <= pos; ++j) {
      float kr[NV], vr[NV];
      load_row<TIn, NV>(k + p.kroff(b, j, h), p.D, lane, kr);
      load_row<TIn, NV>(v + p.kroff(b, j, h), p.D, lane, vr);
      float x = warp_sum(dot_lane<NV>(a, kr));
      float mn = fmaxf(m, x);
      float alpha = expf(m - mn), pj = expf(x - mn);
      l = l * alpha + pj;
#pragma unroll
      for (int t = 0; t < NV; ++t) U[t] = fmaf(pj, vr[t], U[t] * alpha);
      m = mn;
    }
    float v2r[NV];
    load_row<TIn, NV>(v2 + p.kroff(b, kk, h), p.D, lane, v2r);
    float Mn = fmaxf(M, m), ca = expf(M - Mn), cb = expf(m - Mn);
#pragma unroll
    for (int t = 0; t < NV; ++t) O[t] = O[t] * ca + cb * v2r[t] * U[t];
    L = L * ca + cb * l;
    M = Mn;
    __syncwarp();
  }
  if (lane == 0) { sM[warp] = M; sL[warp] = L; }
#pragma unroll
  for (int t = 0; t < NV; ++t) sO[warp][lane + 32 * t] = O[t];
  __syncthreads();
  if (warp == 0) {
    float Mx = sM[0];
    for (int w = 1; w < kWarps; ++w) Mx = fmaxf(Mx, sM[w]);
    float c[kWarps], Lt = 0.f;
    for (int w = 0; w < kWarps; ++w) { c[w] = expf(sM[w] - Mx); Lt += c[w] * sL[w]; }
    float inv = 1.f / Lt;
    for (int d = lane; d < p.D; d += 32) {
      float x = 0.f;
      for (int w = 0; w < kWarps; ++w) x += c[w] * sO[w][d];
      st_f(o + p.qoff(b, i, h) + d, x * inv);
    }
    if (lane == 0) lse[(int64_t(b) * p.H + h) * p.N + i] = Mx + logf(Lt);
  }
}

// ------------------------------------------------------------------------------------------
// delta_i = <dO_i, o_i> (FlashAttention's D; "D_ptr"), one warp per query row.
// ------------------------------------------------------------------------------------------
template <typename TIn, typename TOut>
__global__ void __launch_bounds__(kThreads) simt_delta(Problem p, const TIn* __restrict__ dO,
                                                       const TOut* __restrict__ o, float* __restrict__ delta) {
  int64_t row = int64_t(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  int lane = threadIdx.x & 31;
  int64_t total = int64_t(p.B) * p.H * p.N;
  if (row >= total) return;
  int i = row % p.N, bh = row / p.N, b = bh / p.H, h = bh % p.H;
  const TIn* g = dO + p.qoff(b, i, h);
  const TOut* y = o + p.qoff(b, i, h);
  float x = 0.f;
  for (int d = lane; d < p.D; d += 32) x = fmaf(ld_f(g + d), ld_f(y + d), x);
  x = warp_sum(x);
  if (lane == 0) delta[row] = x;
}

// Cross-warp sum of per-warp row accumulators, then store (scaled) to a global row.
template <typename TOut, int NV>
__device__ __forceinline__ void block_sum_store(float (*red)[32 * NV], const float (&acc)[NV], int D,
                                                TOut* dst) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int t = 0; t < NV; ++t) red[warp][lane + 32 * t] = acc[t];
  __syncthreads();
  for (int d = threadIdx.x; d < D; d += kThreads) {
    float x = 0.f;
    for (int w = 0; w < kWarps; ++w) x += red[w][d];
    st_f(dst + d, x);
  }
}

// ------------------------------------------------------------------------------------------
// dq: one block per query row i; warp per K' row k.  W_(i,k) = sum_j dS k_j.
// ------------------------------------------------------------------------------------------
template <typename TIn, typename TOut, int NV>
__global__ void __launch_bounds__(kThreads) simt_bwd_dq(Problem p, const TIn* __restrict__ q,
                                                        const TIn* __restrict__ k, const TIn* __restrict__ v,
                                                        const TIn* __restrict__ k2, const TIn* __restrict__ v2,
                                                        const TIn* __restrict__ dO, const float* __restrict__ lse,
                                                        const float* __restrict__ delta, TOut* __restrict__ dq) {
  const int i = blockIdx.x, bh = blockIdx.y, b = bh / p.H, h = bh % p.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ float sq[32 * NV], sdo[32 * NV];
  __shared__ float sk2[kWarps][32 * NV], sW[kWarps][32 * NV];
  const int pos = p.np + i;
  for (int d = threadIdx.x; d < p.D; d += kThreads) {
    sq[d] = ld_f(q + p.qoff(b, i, h) + d);
    sdo[d] = ld_f(dO + p.qoff(b, i, h) + d);
  }
  __syncthreads();
  const int64_t row = (int64_t(b) * p.H + h) * p.N + i;
  const float li = lse[row], Di = delta[row];
  const int j0 = win_lo(pos, p.w1), k0 = win_lo(pos, p.w2), D3 = (p.D / 3) * 3;
  float acc[NV];
#pragma unroll
  for (int t = 0; t < NV; ++t) acc[t] = 0.f;
  for (int kk = k0 + warp; kk <= pos; kk += kWarps) {
    load_row_smem(k2 + p.kroff(b, kk, h), p.D, lane, sk2[warp]);
    __syncwarp();
    float a[NV], g[NV], W[NV];
    row_operand<NV>(p, sq, sk2[warp], lane, a);
    load_row<TIn, NV>(v2 + p.kroff(b, kk, h), p.D, lane, g);
#pragma unroll
    for (int t = 0; t < NV; ++t) {
      int d = lane + 32 * t;
      g[t] *= d < p.D ? sdo[d] : 0.f;
      W[t] = 0.f;
    }
    for (int j = j0; j <= pos; ++j) {
      float kr[NV], vr[NV];
      load_row<TIn, NV>(k + p.kroff(b, j, h), p.D, lane, kr);
      load_row<TIn, NV>(v + p.kroff(b, j, h), p.D, lane, vr);
      float x = warp_sum(dot_lane<NV>(a, kr));
      float y = warp_sum(dot_lane<NV>(g, vr));
      float ds = expf(x - li) * (y - Di);
#pragma unroll
      for (int t = 0; t < NV; ++t) W[t] = fmaf(ds, kr[t], W[t]);
    }
    if (p.det) {
#pragma unroll
      for (int t = 0; t < NV; ++t) sW[warp][lane + 32 * t] = W[t];
      __syncwarp();
#pragma unroll
      for (int t = 0; t < NV; ++t) {
        int d = lane + 32 * t;
        if (d < p.D) acc[t] += p.scale * cross_at(sW[warp], sk2[warp], d, D3);
      }
    } else {
#pragma unroll
      for (int t = 0; t < NV; ++t) {
        int d = lane + 32 * t;
        if (d < p.D) acc[t] += p.scale * sk2[warp][d] * W[t];
      }
    }
    __syncwarp();
  }
  __syncthreads();
  block_sum_store<TOut, NV>(sW, acc, p.D, dq + p.qoff(b, i, h));
}

// ------------------------------------------------------------------------------------------
// dk2, dv2: one block per K' key row kk; warp per query position pos in [kk, kk+w2).
// ------------------------------------------------------------------------------------------
template <typename TIn, typename TOut, int NV>
__global__ void __launch_bounds__(kThreads) simt_bwd_dk2(Problem p, const TIn* __restrict__ q,
                                                         const TIn* __restrict__ k, const TIn* __restrict__ v,
                                                         const TIn* __restrict__ k2, const TIn* __restrict__ v2,
                                                         const TIn* __restrict__ dO, const float* __restrict__ lse,
                                                         const float* __restrict__ delta, TOut* __restrict__ dk2,
                                                         TOut* __restrict__ dv2) {
  const int kk = blockIdx.x, bh = blockIdx.y, b = bh / p.H, h = bh % p.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ float sk2[32 * NV];
  __shared__ float sqw[kWarps][32 * NV], sW[kWarps][32 * NV];
  for (int d = threadIdx.x; d < p.D; d += kThreads) sk2[d] = ld_f(k2 + p.kroff(b, kk, h) + d);
  __syncthreads();
  float v2r[NV];
  load_row<TIn, NV>(v2 + p.kroff(b, kk, h), p.D, lane, v2r);
  const int D3 = (p.D / 3) * 3;
  float ak[NV], av[NV];
#pragma unroll
  for (int t = 0; t < NV; ++t) ak[t] = av[t] = 0.f;
  const int pend = min(kk + p.w2, p.NK());
  for (int pos = max(kk, p.np) + warp; pos < pend; pos += kWarps) {
    const int i = pos - p.np;
    const int64_t row = (int64_t(b) * p.H + h) * p.N + i;
    const float li = lse[row], Di = delta[row];
    load_row_smem(q + p.qoff(b, i, h), p.D, lane, sqw[warp]);
    __syncwarp();
    float a[NV], g[NV], dor[NV], W[NV], U[NV];
    row_operand<NV>(p, sqw[warp], sk2, lane, a);
    load_row<TIn, NV>(dO + p.qoff(b, i, h), p.D, lane, dor);
#pragma unroll
    for (int t = 0; t < NV; ++t) { g[t] = dor[t] * v2r[t]; W[t] = U[t] = 0.f; }
    for (int j = win_lo(pos, p.w1); j <= pos; ++j) {
      float kr[NV], vr[NV];
      load_row<TIn, NV>(k + p.kroff(b, j, h), p.D, lane, kr);
      load_row<TIn, NV>(v + p.kroff(b, j, h), p.D, lane, vr);
      float x = warp_sum(dot_lane<NV>(a, kr));
      float y = warp_sum(dot_lane<NV>(g, vr));
      float pj = expf(x - li);
      float ds = pj * (y - Di);
#pragma unroll
      for (int t = 0; t < NV; ++t) { W[t] = fmaf(ds, kr[t], W[t]); U[t] = fmaf(pj, vr[t], U[t]); }
    }
    if (p.det) {
#pragma unroll
      for (int t = 0; t < NV; ++t) sW[warp][lane + 32 * t] = W[t];
      __syncwarp();
#pragma unroll
      for (int t = 0; t < NV; ++t) {
        int d = lane + 32 * t;
        if (d < p.D) ak[t] += p.scale * cross_at(sqw[warp], sW[warp], d, D3);
      }
    } else {
#pragma unroll
      for (int t = 0; t < NV; ++t) {
        int d = lane + 32 * t;
        if (d < p.D) ak[t] += p.scale * sqw[warp][d] * W[t];
      }
    }
#pragma unroll
    for (int t = 0; t < NV; ++t) av[t] += dor[t] * U[t];
    __syncwarp();
  }
  __syncthreads();
  block_sum_store<TOut, NV>(sW, ak, p.D, dk2 + p.koff(b, kk, h));
  __syncthreads();
  block_sum_store<TOut, NV>(sW, av, p.D, dv2 + p.koff(b, kk, h));
}

// ------------------------------------------------------------------------------------------
// dk, dv: one block per K key row j; warp per query position pos in [j, j+w1), inner loop
// over the K' window of pos.
// ------------------------------------------------------------------------------------------
template <typename TIn, typename TOut, int NV>
__global__ void __launch_bounds__(kThreads) simt_bwd_dk(Problem p, const TIn* __restrict__ q,
                                                        const TIn* __restrict__ k, const TIn* __restrict__ v,
                                                        const TIn* __restrict__ k2, const TIn* __restrict__ v2,
                                                        const TIn* __restrict__ dO, const float* __restrict__ lse,
                                                        const float* __restrict__ delta, TOut* __restrict__ dk,
                                                        TOut* __restrict__ dv) {
  const int j = blockIdx.x, bh = blockIdx.y, b = bh / p.H, h = bh % p.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ float sqw[kWarps][32 * NV], sk2w[kWarps][32 * NV];
  float kr[NV], vr[NV];
  load_row<TIn, NV>(k + p.kroff(b, j, h), p.D, lane, kr);
  load_row<TIn, NV>(v + p.kroff(b, j, h), p.D, lane, vr);
  float ak[NV], av[NV];
#pragma unroll
  for (int t = 0; t < NV; ++t) ak[t] = av[t] = 0.f;
  const int pend = min(j + p.w1, p.NK());
  for (int pos = max(j, p.np) + warp; pos < pend; pos += kWarps) {
    const int i = pos - p.np;
    const int64_t row = (int64_t(b) * p.H + h) * p.N + i;
    const float li = lse[row], Di = delta[row];
    load_row_smem(q + p.qoff(b, i, h), p.D, lane, sqw[warp]);
    float dor[NV];
    load_row<TIn, NV>(dO + p.qoff(b, i, h), p.D, lane, dor);
    for (int kk = win_lo(pos, p.w2); kk <= pos; ++kk) {
      __syncwarp();
      load_row_smem(k2 + p.kroff(b, kk, h), p.D, lane, sk2w[warp]);
      __syncwarp();
      float a[NV], g[NV];
      row_operand<NV>(p, sqw[warp], sk2w[warp], lane, a);
      load_row<TIn, NV>(v2 + p.kroff(b, kk, h), p.D, lane, g);
#pragma unroll
      for (int t = 0; t < NV; ++t) g[t] *= dor[t];
      float x = warp_sum(dot_lane<NV>(a, kr));
      float y = warp_sum(dot_lane<NV>(g, vr));
      float pj = expf(x - li);
      float ds = pj * (y - Di);
#pragma unroll
      for (int t = 0; t < NV; ++t) { ak[t] = fmaf(ds, a[t], ak[t]); av[t] = fmaf(pj, g[t], av[t]); }
    }
    __syncwarp();
  }
  __syncthreads();
  block_sum_store<TOut, NV>(sqw, ak, p.D, dk + p.koff(b, j, h));
  __syncthreads();
  block_sum_store<TOut, NV>(sqw, av, p.D, dv + p.koff(b, j, h));
}

template <typename TIn, typename TOut, int NV>
cudaError_t launch_fwd_t(const Problem& p, const void* q, const void* k, const void* v, const void* k2,
                         const void* v2, void* o, float* lse, cudaStream_t st) {
  dim3 grid(p.N, p.B * p.H);
  KernelScope ks("simt_fwd", st);
  simt_fwd<TIn, TOut, NV><<<grid, kThreads, 0, st>>>(p, (const TIn*)q, (const TIn*)k, (const TIn*)v,
                                                      (const TIn*)k2, (const TIn*)v2, (TOut*)o, lse);
  return cudaGetLastError();
}

template <typename TIn, typename TOut, int NV>
cudaError_t launch_bwd_t(const Problem& p, const void* q, const void* k, const void* v, const void* k2,
                         const void* v2, const void* o, const float* lse, const void* dO, void* dq,
                         void* dk, void* dv, void* dk2, void* dv2, float* delta, cudaStream_t st) {
  int64_t rows = int64_t(p.B) * p.H * p.N;
  {
    KernelScope ks("simt_delta", st);
    simt_delta<TIn, TOut><<<unsigned((rows + kWarps - 1) / kWarps), kThreads, 0, st>>>(
        p, (const TIn*)dO, (const TOut*)o, delta);
  }
  dim3 gq(p.N, p.B * p.H), gk(p.NK(), p.B * p.H);
  {
    KernelScope ks("simt_bwd_dq", st);
    simt_bwd_dq<TIn, TOut, NV><<<gq, kThreads, 0, st>>>(p, (const TIn*)q, (const TIn*)k, (const TIn*)v,
                                                         (const TIn*)k2, (const TIn*)v2, (const TIn*)dO,
                                                         lse, delta, (TOut*)dq);
  }
  {
    KernelScope ks("simt_bwd_dk2", st);
    simt_bwd_dk2<TIn, TOut, NV><<<gk, kThreads, 0, st>>>(p, (const TIn*)q, (const TIn*)k, (const TIn*)v,
                                                          (const TIn*)k2, (const TIn*)v2, (const TIn*)dO,
                                                          lse, delta, (TOut*)dk2, (TOut*)dv2);
  }
  {
    KernelScope ks("simt_bwd_dk", st);
    simt_bwd_dk<TIn, TOut, NV><<<gk, kThreads, 0, st>>>(p, (const TIn*)q, (const TIn*)k, (const TIn*)v,
                                                         (const TIn*)k2, (const TIn*)v2, (const TIn*)dO,
                                                         lse, delta, (TOut*)dk, (TOut*)dv);
  }
  return cudaGetLastError();
}

template <int NV>
cudaError_t fwd_nv(const Problem& p, bool in_f32, bool out_f32, const void* q, const void* k, const void* v,
                   const void* k2, const void* v2, void* o, float* lse, cudaStream_t st) {
  using bf = __nv_bfloat16;
  if (in_f32) return launch_fwd_t<float, float, NV>(p, q, k, v, k2, v2, o, lse, st);
  if (out_f32) return launch_fwd_t<bf, float, NV>(p, q, k, v, k2, v2, o, lse, st);
  return launch_fwd_t<bf, bf, NV>(p, q, k, v, k2, v2, o, lse, st);
}

template <int NV>
cudaError_t bwd_nv(const Problem& p, bool in_f32, bool out_f32, const void* q, const void* k, const void* v,
                   const void* k2, const void* v2, const void* o, const float* lse, const void* dO,
                   void* dq, void* dk, void* dv, void* dk2, void* dv2, float* delta, cudaStream_t st) {
  using bf = __nv_bfloat16;
  if (in_f32)
    return launch_bwd_t<float, float, NV>(p, q, k, v, k2, v2, o, lse, dO, dq, dk, dv, dk2, dv2, delta, st);
  if (out_f32)
    return launch_bwd_t<bf, float, NV>(p, q, k, v, k2, v2, o, lse, dO, dq, dk, dv, dk2, dv2, delta, st);
  return launch_bwd_t<bf, bf, NV>(p, q, k, v, k2, v2, o, lse, dO, dq, dk, dv, dk2, dv2, delta, st);
}

}  // namespace

cudaError_t simt_forward(const Problem& p, bool in_f32, bool out_f32, const void* q, const void* k,
                         const void* v, const void* k2, const void* v2, void* o, float* lse, cudaStream_t st) {
  switch ((p.D + 31) / 32) {
    case 1: return fwd_nv<1>(p, in_f32, out_f32, q, k, v, k2, v2, o, lse, st);
    case 2: return fwd_nv<2>(p, in_f32, out_f32, q, k, v, k2, v2, o, lse, st);
    case 3: return fwd_nv<3>(p, in_f32, out_f32, q, k, v, k2, v2, o, lse, st);
    default: return fwd_nv<4>(p, in_f32, out_f32, q, k, v, k2, v2, o, lse, st);
  }
}

cudaError_t simt_backward(const Problem& p, bool in_f32, bool out_f32, const void* q, const void* k,
                          const void* v, const void* k2, const void* v2, const void* o, const float* lse,
                          const void* dO, void* dq, void* dk, void* dv, void* dk2, void* dv2, float* delta,
                          cudaStream_t st) {
  switch ((p.D + 31) / 32) {
    case 1: return bwd_nv<1>(p, in_f32, out_f32, q, k, v, k2, v2, o, lse, dO, dq, dk, dv, dk2, dv2, delta, st);
    case 2: return bwd_nv<2>(p, in_f32, out_f32, q, k, v, k2, v2, o, lse, dO, dq, dk, dv, dk2, dv2, delta, st);
    case 3: return bwd_nv<3>(p, in_f32, out_f32, q, k, v, k2, v2, o, lse, dO, dq, dk, dv, dk2, dv2, delta, st);
    default: return bwd_nv<4>(p, in_f32, out_f32, q, k, v, k2, v2, o, lse, dO, dq, dk, dv, dk2, dv2, delta, st);
  }
}

}  // namespace sa

namespace sa {
// dk, dv only (CUDA-core kernel), given lse and delta; used by the tensor-core backward for
// shapes its K/V-stationary kernel does not cover.
cudaError_t simt_bwd_dk_only(const Problem& p, bool out_f32, const void* q, const void* k, const void* v,
                             const void* k2, const void* v2, const void* dO, const float* lse, const float* delta,
                             void* dk, void* dv, cudaStream_t st) {
  using bf = __nv_bfloat16;
  dim3 gk(p.NK(), p.B * p.H);
  KernelScope ks("simt_bwd_dk", st);
#define SA_DK_LAUNCH(NV)                                                                                       \
  if (out_f32)                                                                                                 \
    simt_bwd_dk<bf, float, NV><<<gk, kThreads, 0, st>>>(p, (const bf*)q, (const bf*)k, (const bf*)v,            \
                                                        (const bf*)k2, (const bf*)v2, (const bf*)dO, lse, delta, \
                                                        (float*)dk, (float*)dv);                                \
  else                                                                                                         \
    simt_bwd_dk<bf, bf, NV><<<gk, kThreads, 0, st>>>(p, (const bf*)q, (const bf*)k, (const bf*)v, (const bf*)k2, \
                                                     (const bf*)v2, (const bf*)dO, lse, delta, (bf*)dk, (bf*)dv);
  switch ((p.D + 31) / 32) {
    case 1: SA_DK_LAUNCH(1) break;
    case 2: SA_DK_LAUNCH(2) break;
    case 3: SA_DK_LAUNCH(3) break;
    default: SA_DK_LAUNCH(4) break;
  }
#undef SA_DK_LAUNCH
  return cudaGetLastError();
}
}  // namespace sa

// sa_tc_rows.cuh -- per-row operand formation shared by the tensor-core kernels.
//
// An (i,k) row operand is a D-vector formed on the CUDA cores from two bf16 rows x, y:
//   trilinear:   scale * (x o y)                      (a_(i,k) = s q_i o k2_k;  dO_i o v2_k)
//   determinant: scale * (y x x) chunkwise over 3-dims (a_(i,k) = s k2_k x q_i, P:298-301;
//                trailing D mod 3 dims are 0, reading R5)
// packed as fp16x2 (low half = even element), the layout the K-major A operand takes in TMEM
// (one row per TMEM lane, 2 elements per 32-bit column).
#pragma once
#include "sa_tc_common.cuh"

namespace sa {
namespace tc {

template <int D>
__device__ __forceinline__ void row_operand_f16(const __nv_bfloat16* x, const __nv_bfloat16* y, float scale,
                                                bool cross, uint32_t (&pk)[D / 2]) {
  const uint4* xp = reinterpret_cast<const uint4*>(x);
  const uint4* yp = reinterpret_cast<const uint4*>(y);
  if (cross) {
    constexpr int D3 = (D / 3) * 3;
#pragma unroll
    for (int base = 0; base < D; base += 24) {
      float xf[24], yf[24], av[24];
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        if (base + 8 * u < D) {
          uint4 a = xp[base / 8 + u], b = yp[base / 8 + u];  // plain loads: rows may be staged in smem
          uint32_t as[4] = {a.x, a.y, a.z, a.w}, bs[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float2 fa = bf16x2_to_f2(as[e]), fb = bf16x2_to_f2(bs[e]);
            xf[8 * u + 2 * e] = fa.x;
            xf[8 * u + 2 * e + 1] = fa.y;
            yf[8 * u + 2 * e] = fb.x;
            yf[8 * u + 2 * e + 1] = fb.y;
          }
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) xf[8 * u + e] = yf[8 * u + e] = 0.f;
        }
      }
#pragma unroll
      for (int c3 = 0; c3 < 24; c3 += 3) {
        if (base + c3 + 3 <= D3) {  // (y x x)_r = y_{r+1} x_{r+2} - y_{r+2} x_{r+1}
          av[c3 + 0] = yf[c3 + 1] * xf[c3 + 2] - yf[c3 + 2] * xf[c3 + 1];
          av[c3 + 1] = yf[c3 + 2] * xf[c3 + 0] - yf[c3 + 0] * xf[c3 + 2];
          av[c3 + 2] = yf[c3 + 0] * xf[c3 + 1] - yf[c3 + 1] * xf[c3 + 0];
        } else {
          av[c3 + 0] = av[c3 + 1] = av[c3 + 2] = 0.f;
        }
      }
#pragma unroll
      for (int e = 0; e < 24; e += 2)
        if (base + e < D) pk[(base + e) / 2] = pack_f16x2(scale * av[e], scale * av[e + 1]);
    }
  } else {
#pragma unroll
    for (int t = 0; t < D / 8; ++t) {
      uint4 a = xp[t], b = yp[t];
      uint32_t as[4] = {a.x, a.y, a.z, a.w}, bs[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float2 fa = bf16x2_to_f2(as[e]), fb = bf16x2_to_f2(bs[e]);
        pk[4 * t + e] = pack_f16x2(scale * fa.x * fb.x, scale * fa.y * fb.y);
      }
    }
  }
}

__device__ __forceinline__ uint32_t hmul2_u32(uint32_t x, uint32_t y) {
  __half2 r = __hmul2(*reinterpret_cast<__half2*>(&x), *reinterpret_cast<__half2*>(&y));
  return *reinterpret_cast<uint32_t*>(&r);
}

// ---- Determinant operand by 3-chunk permutations (fp16 pairs) ----
// Within each 3-chunk, (y x x)_r = y_{r+1} x_{r+2} - y_{r+2} x_{r+1} (indices mod 3 inside the chunk),
// i.e.  y x x = P1(y) o P2(x) - P2(y) o P1(x)  with P_S(v)_r = v_{3 floor(r/3) + (r + S) mod 3}.
// On packed fp16 words (2 halves each) a permuted word is one PRMT of at most two source words, so a
// row costs a byte permute per word and operand plus one HMUL2 and one HFMA2 per word -- against
// fp32 unpack / math / repack.  Rounding: the HMUL2 product is rounded to fp16 before the HFMA2
// (one more fp16 rounding than the fp32 formation; logit error RMS +23% on unit-normal data,
// DESIGN.md reading R5b).  Zero words past D make the trailing D mod 3 columns 0 (reading R5).
__host__ __device__ constexpr int perm3_src(int r, int S) { return 3 * (r / 3) + (r % 3 + S) % 3; }

// Word i (index relative to a block that starts on a 3-chunk and word boundary: i compile-time after
// unrolling) of P_S(v), from the block's words w[0..NW).  Source words beyond NW read as 0.
template <int S, int NW>
__device__ __forceinline__ uint32_t perm3_word(const uint32_t (&w)[NW], int i) {
  const int s0 = perm3_src(2 * i, S), s1 = perm3_src(2 * i + 1, S);
  const int a = s0 >> 1, b = s1 >> 1;
  const uint32_t n0 = (s0 & 1) ? 2u : 0u;
  const uint32_t wa = a < NW ? w[a] : 0u, wb = b < NW ? w[b] : 0u;
  if (a == b) {
    const uint32_t n1 = (s1 & 1) ? 2u : 0u;
    return __byte_perm(wa, 0u, n0 | (n0 + 1) << 4 | n1 << 8 | (n1 + 1) << 12);
  }
  const uint32_t n1 = (s1 & 1) ? 6u : 4u;
  return __byte_perm(wa, wb, n0 | (n0 + 1) << 4 | n1 << 8 | (n1 + 1) << 12);
}

// Both permutations of a block of NW words.
template <int NW>
__device__ __forceinline__ void perm3_block(const uint32_t (&w)[NW], uint32_t (&p1)[NW], uint32_t (&p2)[NW]) {
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    p1[i] = perm3_word<1>(w, i);
    p2[i] = perm3_word<2>(w, i);
  }
}

// One word of y x x = P1(y) o P2(x) - P2(y) o P1(x) (unscaled fp16).
__device__ __forceinline__ uint32_t cross_word(uint32_t y1, uint32_t y2, uint32_t x1, uint32_t x2) {
  const __half2 t = __hmul2(*reinterpret_cast<const __half2*>(&y2), *reinterpret_cast<const __half2*>(&x1));
  const __half2 r =
      __hfma2(*reinterpret_cast<const __half2*>(&y1), *reinterpret_cast<const __half2*>(&x2), __hneg2(t));
  return *reinterpret_cast<const uint32_t*>(&r);
}

// Words [W0, W0 + NWO) (compile-time; word w = columns 2w, 2w+1) of the unscaled determinant row
// operand y x x for fp16 rows x, y of D elements (16-byte aligned, shared or global memory).
template <int D, int W0, int NWO>
__device__ __forceinline__ void det_words_f16(const __half* x, const __half* y, uint32_t (&out)[NWO]) {
  constexpr int B0 = (2 * W0) / 24, B1 = (2 * (W0 + NWO) - 1) / 24;
#pragma unroll
  for (int b = B0; b <= B1; ++b) {
    uint32_t xw[12], yw[12], x1[12], x2[12], y1[12], y2[12];
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      uint4 xv = make_uint4(0u, 0u, 0u, 0u), yv = xv;
      if (24 * b + 8 * u < D) {
        xv = *reinterpret_cast<const uint4*>(x + 24 * b + 8 * u);
        yv = *reinterpret_cast<const uint4*>(y + 24 * b + 8 * u);
      }
      xw[4 * u] = xv.x, xw[4 * u + 1] = xv.y, xw[4 * u + 2] = xv.z, xw[4 * u + 3] = xv.w;
      yw[4 * u] = yv.x, yw[4 * u + 1] = yv.y, yw[4 * u + 2] = yv.z, yw[4 * u + 3] = yv.w;
    }
    perm3_block(xw, x1, x2);
    perm3_block(yw, y1, y2);
#pragma unroll
    for (int i = 0; i < 12; ++i) {
      const int w = 12 * b + i;
      if (w >= W0 && w < W0 + NWO) out[w - W0] = cross_word(y1[i], y2[i], x1[i], x2[i]);
    }
  }
}

// Determinant row operand from fp16 rows: scale * (y x x) chunkwise, trailing D mod 3 dims 0.
template <int D>
__device__ __forceinline__ void row_operand_from_f16(const __half* x, const __half* y, float scale,
                                                     uint32_t (&pk)[D / 2]) {
  const uint4* xp = reinterpret_cast<const uint4*>(x);
  const uint4* yp = reinterpret_cast<const uint4*>(y);
  constexpr int D3 = (D / 3) * 3;
#pragma unroll
  for (int base = 0; base < D; base += 24) {
    float xf[24], yf[24], av[24];
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      if (base + 8 * u < D) {
        uint4 a = xp[base / 8 + u], b = yp[base / 8 + u];
        uint32_t as[4] = {a.x, a.y, a.z, a.w}, bs[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float2 fa = __half22float2(*reinterpret_cast<__half2*>(&as[e]));
          float2 fb = __half22float2(*reinterpret_cast<__half2*>(&bs[e]));
          xf[8 * u + 2 * e] = fa.x;
          xf[8 * u + 2 * e + 1] = fa.y;
          yf[8 * u + 2 * e] = fb.x;
          yf[8 * u + 2 * e + 1] = fb.y;
        }
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) xf[8 * u + e] = yf[8 * u + e] = 0.f;
      }
    }
#pragma unroll
    for (int c3 = 0; c3 < 24; c3 += 3) {
      if (base + c3 + 3 <= D3) {  // (y x x)_r = y_{r+1} x_{r+2} - y_{r+2} x_{r+1}
        av[c3 + 0] = yf[c3 + 1] * xf[c3 + 2] - yf[c3 + 2] * xf[c3 + 1];
        av[c3 + 1] = yf[c3 + 2] * xf[c3 + 0] - yf[c3 + 0] * xf[c3 + 2];
        av[c3 + 2] = yf[c3 + 0] * xf[c3 + 1] - yf[c3 + 1] * xf[c3 + 0];
      } else {
        av[c3 + 0] = av[c3 + 1] = av[c3 + 2] = 0.f;
      }
    }
#pragma unroll
    for (int e = 0; e < 24; e += 2)
      if (base + e < D) pk[(base + e) / 2] = pack_f16x2(scale * av[e], scale * av[e + 1]);
  }
}

// Store a full packed row (D/2 columns) to TMEM at column address taddr (this warp's lanes).
template <int D>
__device__ __forceinline__ void tmem_store_row(uint32_t taddr, const uint32_t (&pk)[D / 2]) {
#pragma unroll
  for (int t = 0; t < D / 64; ++t) tmem_st32(taddr + 32 * t, *reinterpret_cast<const uint32_t(*)[32]>(pk + 32 * t));
}

// Load n (<=32, multiple of 8) bf16 values starting at p (16B aligned) as floats.
template <int N>
__device__ __forceinline__ void load_bf16(const __nv_bfloat16* p, float (&f)[N]) {
  const uint4* vp = reinterpret_cast<const uint4*>(p);
#pragma unroll
  for (int t = 0; t < N / 8; ++t) {
    uint4 x = vp[t];  // plain load: p may point into shared-memory staging
    uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 g = bf16x2_to_f2(xs[e]);
      f[8 * t + 2 * e] = g.x;
      f[8 * t + 2 * e + 1] = g.y;
    }
  }
}

}  // namespace tc
}  // namespace sa

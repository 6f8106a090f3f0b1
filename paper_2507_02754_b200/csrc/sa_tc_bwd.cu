// sa_tc_bwd.cu -- tcgen05/TMEM/TMA backward of sliding-window 2-simplicial attention (bf16 in).
//
// Split as in the paper ("one kernel for dK and dV, another for dK', dV' and dQ"), with no
// global atomics:
//   delta  : delta_i = <dO_i, o_i>                                          (P:856 D_ptr)
//   bwd_q  : rows (i,k) x j-chunks.  S = A_S K^T, dP = A_dP V^T (recompute, TS-MMA), then
//            P = exp(S - lse_i), dS = P (dP - delta_i) on the CUDA cores, and
//            W += dS K, U += P V (TS-MMA, fp32 in TMEM).  Epilogue:
//              dq_i  = s sum_k k2_k o W_(i,k)        (det: W x k2_k)
//              dk2_k = s sum_i q_i o W_(i,k)         (det: q_i x W)
//              dv2_k =   sum_i dO_i o U_(i,k)
//            dk2/dv2 rows are reduced across consecutive tiles in a shared-memory ring carried
//            by each CTA over a contiguous tile range ("segment carry"); the w2-1 rows shared
//            with the neighbouring range go to a small band workspace and are added by `fold`
//            (deterministic replacement for the paper's even/odd two-stage launches, Alg. 2).
//   bwd_kv : K/V-stationary; a CTA owns 128 key rows j of K and V (TMEM lanes = j) and walks
//            the row tiles that touch them: S^T = K A_S^T, dP^T = V A_dP^T (SS-MMA), P^T and
//            dS^T on the CUDA cores, dV += P^T A_dP, dK += dS^T A_S (TS-MMA).
// Row operands: A_S = s (q o k2)  [det: s (k2 x q)],  A_dP = dO o v2, fp16; K, V fp16 copies.
#include <math.h>
#include <stdlib.h>

#include <algorithm>
#include <utility>

#include "sa_tc_rows.cuh"

namespace sa {

cudaError_t convert_pair_f16(const void* a, void* ao, const void* b, void* bo, int64_t n, int num_sms,
                             cudaStream_t st);
int num_sms();

namespace {

using namespace tc;

constexpr float kLog2e = 1.4426950408889634f;
constexpr int kMaxR = 128;  // bwd_q: rows per query (folded window w2) supported
constexpr int kRingMax = 66;  // larger rings (R = 128) live in a global per-CTA slab (L2-resident)


// ------------------------------------------------------------------------------------------
// delta_i = <dO_i, o_i>, one warp per query row
// ------------------------------------------------------------------------------------------
template <typename TOut>
__global__ void __launch_bounds__(256) delta_kernel(Problem p, const __nv_bfloat16* __restrict__ dO,
                                                    const TOut* __restrict__ o, float* __restrict__ delta) {
  const int64_t row = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= int64_t(p.B) * p.H * p.N) return;
  const int i = row % p.N, bh = row / p.N, b = bh / p.H, h = bh % p.H;
  const __nv_bfloat16* g = dO + p.qoff(b, i, h);
  const TOut* y = o + p.qoff(b, i, h);
  float x = 0.f;
  for (int d = lane; d < p.D; d += 32) x = fmaf(__bfloat162float(g[d]), ld_f(y + d), x);
  x = warp_sum(x);
  if (lane == 0) delta[row] = x;
}

// ==========================================================================================
// bwd_q: dQ, dK2, dV2
// ==========================================================================================
// 16 compute warps: warp w -> TMEM lane quarter w&3, column half (w>>2)&1, sub-slice w>>3 (two warps
// per lane quarter and half: more warps in flight to hide the latency of the softmax-gradient, the
// row-operand formation and the epilogue)
constexpr int kQCW = 16;
constexpr int kQNT = 32 * kQCW;  // compute threads
constexpr int kQThreads = kQNT + 64;
constexpr int kQWarpTMA = kQCW, kQWarpMMA = kQCW + 1;
constexpr int kQChunk = 64;
// TMEM columns
constexpr uint32_t kQW = 0, kQU = 128, kQS = 256, kQdP = 320, kQAS = 384, kQAdP = 448;
constexpr int kQStageRows = 80;  // staged rows per tile: q, dO (G each), k2, v2 (R+G-1 each)

struct BwdQArgs {
  Problem p;  // after the swap: w2 = R rows per query
  const __half *q, *k2, *v2, *dO;  // fp16 copies
  const float *lse, *delta;
  void *dq, *dk2, *dv2;
  float* band;  // [grid][2 start/end][2 k2/v2][R-1][D]
  float* gring;  // R = 128 determinant: [grid][2 k2/v2][ring][D] fp32 ring, each CTA's own (no atomics)
  // R: rows per query of the tiling (a power of two >= the folded window Rt); rows with
  // kk < R - Rt lie before the window and are masked like rows before the sequence start
  int out_f32, R, lR, G, ngroups, items, per_cta, ring, Rt;
  int tma_stage;  // RING 38: rows staged by pitched TMA boxes (H, Hk >= 2), else cp.async
  int prod_stage;  // RING 37: q/dO and new k2/v2 rows by 1-D bulk copies from the TMA producer warp
  FastDiv fd_ng, fd_H, fd_ring;  // by ngroups, H, ring (per-tile index arithmetic)
};

template <int D, int RING, bool STAGED>
struct QSmem {
  // RING variants: <= kRingMax shared-memory ring (R <= 64); 129: R = 128 determinant, ring in the
  // global slab BwdQArgs::gring (generic passes); 130: R = 128 trilinear (G = 1), ring in shared
  // memory with a padded pitch (row-owned updates, q_epilogue_g1), two K/V stages to make room
  // 37 / 67: R = 32 / 64 trilinear at D = 128 (row-owned q_epilogue_rot, no eb): four K/V stages
  static constexpr bool kGR = RING == 129;
  static constexpr bool kG1 = RING == 130;
  static constexpr bool kRot = RING == 37 || RING == 67;
  // 38: R in {8, 16} trilinear, staged: the epilogue's row-group sums on the tensor core
  // (q_epilogue_tc): one fp16 product tile X and the query / key-slot selection matrices
  static constexpr bool kTC = RING == 38;
  static constexpr int kStages = kG1 ? 2 : kRot ? 4 : 3;
  static constexpr int kPanelBytes = kQChunk * 128;
  static constexpr int kStageBytes = kQChunk * D * 2;
  static constexpr int kAP = kGR ? D : D + 4;  // ring pitch (floats): padded for row-owned float4 updates
  static constexpr int kEB = (kG1 || kRot || kTC) ? 1 : 128;  // eb rows (unused by the row-owned passes)
  static constexpr int kSelRows = 48;  // Sel_q^T rows 0..15 (queries), Sel_k^T rows 16..47 (key slots)
  alignas(1024) uint8_t k[kStages][kStageBytes];
  alignas(1024) uint8_t v[kStages][kStageBytes];
  alignas(16) float acc_k2[kGR ? 1 : RING][kAP];
  alignas(16) float acc_v2[kGR ? 1 : RING][kAP];
  alignas(16) union {
    struct {
      float eq[kEB][25], ek[kEB][25], ev[kEB][25];
    } g;  // generic passes (PW <= 24)
    struct {
      float ek[kEB][36], ev[kEB][36];  // 16-byte aligned rows (float4 traffic, conflict-free)
    } w;  // R = 32 trilinear passes (PW = 32, dq reduced in registers)
  } eb;
  // staged rows; pitch D+8 halves so that lanes reading consecutive rows hit distinct banks
  // kRing (kRot and STAGED, R = 32): q/dO rows double-buffered per item; k2/v2 rows in a ring keyed
  // by key position (slot kpos % kKR), one ring half per (b,h) run of the CTA's contiguous items, so
  // consecutive items stage only their G new key rows
  static constexpr bool kRing = kRot && STAGED;
  static constexpr int kKR = 40;  // ring slots per half (>= R + 2G - 1 = 39)
  alignas(kTC ? 128 : 16) __half stg[(STAGED && !kRing) ? 2 : 1][(STAGED && !kRing) ? kQStageRows : 1][D + 8];
  alignas(16) __half stgq[kRing ? 2 : 1][kRing ? 8 : 1][D + 8];  // q rows 0..G-1, dO rows G..2G-1
  // the same rows in fp32 (q pre-multiplied by s) for the epilogue: converted once per tile instead
  // of once per use by each of the query's 32 rows
  alignas(16) float stgqf[kRing ? 2 : 1][kRing ? 8 : 1][kRing ? D : 4];
  alignas(16) __half rk2[kRing ? 2 : 1][kRing ? kKR : 1][D + 8];
  alignas(16) __half rv2[kRing ? 2 : 1][kRing ? kKR : 1][D + 8];
  float slse[2][16], sdl[2][16];
  float dqx[2][32];  // R = 64: the odd lane quarter's dq column partials of the current pass
  float dq4[kTC ? 1 : 4][D];  // R = 64 / 128 trilinear: per-lane-quarter dq partials
  // X (fp16, SWIZZLE_128B, MN-major A); two 64-column panels even at D = 64, since the M = 128 MMA
  // reads both (the second panel's lanes are ignored)
  alignas(1024) uint8_t xr[kTC ? 128 * 128 * 2 : 16];
  alignas(1024) uint8_t sel[kTC ? 2 * kSelRows * 128 : 16];   // Sel^T (K-major B, two 64-row K panels)
  uint64_t red;  // kTC: completion of the epilogue's reduction MMAs (three per tile)
  uint64_t kvfull[kStages], kvempty[kStages];
  uint64_t sfull[2], pready[2], udone, aready, stgfull[2], stgempty[2];
  uint32_t tmem_base;
};

// dK2 / dV2 accumulator ring rows (which = 0: k2, 1: v2): shared memory, or the CTA's global slab
template <int D, int RING, bool STAGED>
__device__ __forceinline__ auto q_acc(QSmem<D, RING, STAGED>& sm, const BwdQArgs& a, int which) {
  using Sm = QSmem<D, RING, STAGED>;
  using Row = float(*)[Sm::kAP];
  if constexpr (Sm::kGR)
    return reinterpret_cast<Row>(a.gring + (size_t(blockIdx.x) * 2 + which) * size_t(a.ring) * D);
  else
    return which ? static_cast<Row>(sm.acc_v2) : static_cast<Row>(sm.acc_k2);
}

struct QItem {
  int bh, b, h, hk, grp, i0, nq, jbeg, span, nch;  // hk: the key head query head h reads (GQA)
};

__device__ __forceinline__ QItem q_item(const BwdQArgs& a, int item) {
  QItem it;
  it.bh = a.fd_ng.div(item);
  it.grp = item - it.bh * a.ngroups;
  it.b = a.fd_H.div(it.bh);
  it.h = it.bh - it.b * a.p.H;
  it.hk = a.p.hk(it.h);
  it.i0 = it.grp * a.G;
  it.nq = min(a.G, a.p.N - it.i0);
  const int pos0 = a.p.np + it.i0, posl = pos0 + it.nq - 1;
  it.jbeg = max(0, pos0 - a.p.w1 + 1);
  it.span = posl - it.jbeg + 1;
  it.nch = (it.span + kQChunk - 1) / kQChunk;
  return it;
}
// The item after `it` in the flat (b, h, group) order, without divisions (items of a CTA are contiguous).
__device__ __forceinline__ QItem q_item_next(const BwdQArgs& a, const QItem& it) {
  QItem n = it;
  if (++n.grp == a.ngroups) {
    n.grp = 0;
    ++n.bh;
    if (++n.h == a.p.H) {
      n.h = 0;
      ++n.b;
    }
    n.hk = a.p.hk(n.h);
  }
  n.i0 = n.grp * a.G;
  n.nq = min(a.G, a.p.N - n.i0);
  const int pos0 = a.p.np + n.i0, posl = pos0 + n.nq - 1;
  n.jbeg = max(0, pos0 - a.p.w1 + 1);
  n.span = posl - n.jbeg + 1;
  n.nch = (n.span + kQChunk - 1) / kQChunk;
  return n;
}
__device__ __forceinline__ int q_width(const QItem& it, int c) {
  if (c < it.nch - 1) return kQChunk;
  return ((it.span - kQChunk * (it.nch - 1)) + 15) & ~15;
}

template <int N>
__device__ __forceinline__ void load_f16(const __half* p, float (&f)[N]) {
#pragma unroll
  for (int t = 0; t < N / 8; ++t) {
    const uint4 x = *reinterpret_cast<const uint4*>(p + 8 * t);
    const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 g = __half22float2(*reinterpret_cast<const __half2*>(&xs[e]));
      f[8 * t + 2 * e] = g.x;
      f[8 * t + 2 * e + 1] = g.y;
    }
  }
}

// Row sources of the current tile: staged shared-memory rows or the global fp16 copies.
struct QRows {
  const __half *q, *dO, *k2, *v2;  // this thread's rows (valid rows only)
  const float *qf, *dOf;           // RING 37: fp32 copies of the q (pre-scaled by s) and dO rows
};

// One epilogue pass over columns [c0, c0+PW) of the tile's W (half 0) / U (half 1) rows:
// per-row contributions into eq/ek/ev, then reductions into dq (per query) and the dk2/dv2 ring.
template <int D, int RING, bool STAGED, int PW, bool DET>
__device__ __forceinline__ void q_epilogue_pass(QSmem<D, RING, STAGED>& sm, const BwdQArgs& a, const QItem& it,
                                                int c0, int half, int r, bool valid, const QRows& rw, uint32_t tW,
                                                uint32_t tU, int tid256, bool p1) {
  const Problem& p = a.p;
  const float s = p.scale;
  if (!p1) {
  } else if (half == 0) {
    float wv[PW], k2v[PW], qv[PW];
    {
      uint32_t u[PW];
      if constexpr (PW >= 16) tmem_ld16(tW + c0, u);
      if constexpr (PW == 24) tmem_ld8(tW + c0 + 16, u + 16);
      if constexpr (PW == 8) tmem_ld8(tW + c0, u);
      tmem_ld_wait();
#pragma unroll
      for (int e = 0; e < PW; ++e) wv[e] = __uint_as_float(u[e]);
    }
    if (valid) {
      load_f16<PW>(rw.k2 + c0, k2v);
      load_f16<PW>(rw.q + c0, qv);
    } else {
#pragma unroll
      for (int e = 0; e < PW; ++e) k2v[e] = qv[e] = 0.f;
    }
    if (DET) {
      constexpr int D3 = (D / 3) * 3;
#pragma unroll
      for (int t = 0; t < PW; t += 3) {
        if (t + 3 <= PW && c0 + t + 3 <= D3) {
          // dq: W x k2 ; dk2: q x W     ((x cross y)_r = x_{r+1} y_{r+2} - x_{r+2} y_{r+1})
          sm.eb.g.eq[r][t + 0] = s * (wv[t + 1] * k2v[t + 2] - wv[t + 2] * k2v[t + 1]);
          sm.eb.g.eq[r][t + 1] = s * (wv[t + 2] * k2v[t + 0] - wv[t + 0] * k2v[t + 2]);
          sm.eb.g.eq[r][t + 2] = s * (wv[t + 0] * k2v[t + 1] - wv[t + 1] * k2v[t + 0]);
          sm.eb.g.ek[r][t + 0] = s * (qv[t + 1] * wv[t + 2] - qv[t + 2] * wv[t + 1]);
          sm.eb.g.ek[r][t + 1] = s * (qv[t + 2] * wv[t + 0] - qv[t + 0] * wv[t + 2]);
          sm.eb.g.ek[r][t + 2] = s * (qv[t + 0] * wv[t + 1] - qv[t + 1] * wv[t + 0]);
        } else {
#pragma unroll
          for (int e = t; e < t + 3 && e < PW; ++e) sm.eb.g.eq[r][e] = sm.eb.g.ek[r][e] = 0.f;
        }
      }
    } else if (PW == 16 && a.R == 32) {
      // R = 32: the warp holds exactly one query's rows -> dq by a register reduce-scatter
      float v[16];
#pragma unroll
      for (int e = 0; e < PW; ++e) {
        v[e & 15] = s * k2v[e] * wv[e];
        sm.eb.g.ek[r][e] = s * qv[e] * wv[e];
      }
      const int ln = r & 31;
#pragma unroll
      for (int st = 16, n = 8; st >= 2; st >>= 1, n >>= 1) {
        const bool hi = ln & st;
#pragma unroll
        for (int i = 0; i < n; ++i) {
          const float keep = hi ? v[n + i] : v[i], send = hi ? v[i] : v[n + i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, st);
        }
      }
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
      const int gq = r >> 5;
      if ((ln & 1) == 0 && gq < it.nq) {
        const int col = ((ln >> 4) & 1) * 8 + ((ln >> 3) & 1) * 4 + ((ln >> 2) & 1) * 2 + ((ln >> 1) & 1);
        const int64_t off = p.qoff(it.b, it.i0 + gq, it.h) + c0 + col;
        if (a.out_f32)
          reinterpret_cast<float*>(a.dq)[off] = v[0];
        else
          reinterpret_cast<__nv_bfloat16*>(a.dq)[off] = __float2bfloat16_rn(v[0]);
      }
    } else {
#pragma unroll
      for (int e = 0; e < PW; ++e) {
        sm.eb.g.eq[r][e] = s * k2v[e] * wv[e];
        sm.eb.g.ek[r][e] = s * qv[e] * wv[e];
      }
    }
  } else {
    float uv[PW], dov[PW];
    {
      uint32_t u[PW];
      if constexpr (PW >= 16) tmem_ld16(tU + c0, u);
      if constexpr (PW == 24) tmem_ld8(tU + c0 + 16, u + 16);
      if constexpr (PW == 8) tmem_ld8(tU + c0, u);
      tmem_ld_wait();
#pragma unroll
      for (int e = 0; e < PW; ++e) uv[e] = __uint_as_float(u[e]);
    }
    if (valid) {
      load_f16<PW>(rw.dO + c0, dov);
    } else {
#pragma unroll
      for (int e = 0; e < PW; ++e) dov[e] = 0.f;
    }
#pragma unroll
    for (int e = 0; e < PW; ++e) sm.eb.g.ev[r][e] = dov[e] * uv[e];
  }
  named_bar_sync(1, kQNT);
  // dq: sum over the R rows of each query; 4 lanes per output, rows interleaved, shuffle-combined
  const bool dq_done = !DET && PW == 16 && a.R == 32;
  for (int base = 0; !dq_done && base < it.nq * PW * 4; base += kQNT) {
    const int idx = base + tid256;
    const bool act = idx < it.nq * PW * 4;
    const int o = idx >> 2, part = idx & 3;
    const int gq = o / PW, d = o % PW;
    float x0 = 0.f, x1 = 0.f;
    if (act) {
      const float(*rows)[25] = sm.eb.g.eq + (gq << a.lR);
      int t = part;
      for (; t + 4 < a.R; t += 8) {
        x0 += rows[t][d];
        x1 += rows[t + 4][d];
      }
      if (t < a.R) x0 += rows[t][d];
    }
    float x = x0 + x1;
    x += __shfl_xor_sync(0xffffffffu, x, 1);
    x += __shfl_xor_sync(0xffffffffu, x, 2);
    if (act && part == 0) {
      const int64_t off = p.qoff(it.b, it.i0 + gq, it.h) + c0 + d;
      if (a.out_f32)
        reinterpret_cast<float*>(a.dq)[off] = x;
      else
        reinterpret_cast<__nv_bfloat16*>(a.dq)[off] = __float2bfloat16_rn(x);
    }
  }
  // dk2 / dv2: key row kpos = P0 - R + 1 + sl receives rows (g, kk = sl - g)
  const int P0 = p.np + it.i0;
  const int nsl = a.R + it.nq - 1;
  const int sbase = a.fd_ring.mod(P0 - a.R + 1 + a.ring);
  for (int idx = tid256; idx < nsl * PW; idx += kQNT) {
    const int sl = idx / PW, d = idx % PW;
    const int kp = P0 - a.R + 1 + sl;
    if (kp < a.p.k2lo) continue;
    float xk = 0.f, xv = 0.f;
    const int glo = max(0, sl - a.R + 1), ghi = min(it.nq - 1, sl);
    for (int g0 = glo; g0 <= ghi; g0 += 4) {
      float tk[4], tv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {  // independent loads first, then the sums
        const int gg = g0 + u;
        const int row = (gg << a.lR) + (sl - gg);
        tk[u] = gg <= ghi ? sm.eb.g.ek[row][d] : 0.f;
        tv[u] = gg <= ghi ? sm.eb.g.ev[row][d] : 0.f;
      }
      xk += (tk[0] + tk[1]) + (tk[2] + tk[3]);
      xv += (tv[0] + tv[1]) + (tv[2] + tv[3]);
    }
    int slot = sbase + sl;  // (P0 - R + 1 + sl) mod ring
    if (slot >= a.ring) slot -= a.ring;
    q_acc(sm, a, 0)[slot][c0 + d] += xk;
    q_acc(sm, a, 1)[slot][c0 + d] += xv;
  }
  named_bar_sync(1, kQNT);
}

// R = 32 trilinear pass over 32 columns [c0, c0+32): the four warps of a TMEM lane quarter (= one
// query g, 32 rows) split the columns 8 ways each: warp m = 2 half + sub takes columns c0+8m..+8
// of both W (dq and the dk2 rows) and U (the dv2 rows).  dq is a register reduce-scatter over the
// 32 lanes (lane groups of 4 end with one column); dk2/dv2 go through the shared-memory gather.
template <int D, int RING, bool STAGED>
__device__ __forceinline__ void q_epilogue_pass32(QSmem<D, RING, STAGED>& sm, const BwdQArgs& a, const QItem& it,
                                                  int c0, int half, int sub, int r, bool valid, const QRows& rw,
                                                  uint32_t tW, uint32_t tU, int tidc, int sbase) {
  const Problem& p = a.p;
  const float s = p.scale;
  const int ln = r & 31;
  const int m = 2 * half + sub;
  const int cs = c0 + 8 * m;
  uint32_t uw[8], uu[8];
  tmem_ld8(tW + cs, uw);
  tmem_ld8(tU + cs, uu);
  float k2v[8], qv[8], dov[8];
  if (valid) {
    load_f16<8>(rw.k2 + cs, k2v);
    load_f16<8>(rw.q + cs, qv);
    load_f16<8>(rw.dO + cs, dov);
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e) k2v[e] = qv[e] = dov[e] = 0.f;
  }
  tmem_ld_wait();
  float v[8], ck[8], cv[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const float w = __uint_as_float(uw[e]);
    v[e] = s * k2v[e] * w;
    ck[e] = s * qv[e] * w;
    cv[e] = dov[e] * __uint_as_float(uu[e]);
  }
  *reinterpret_cast<float4*>(&sm.eb.w.ek[r][8 * m]) = make_float4(ck[0], ck[1], ck[2], ck[3]);
  *reinterpret_cast<float4*>(&sm.eb.w.ek[r][8 * m + 4]) = make_float4(ck[4], ck[5], ck[6], ck[7]);
  *reinterpret_cast<float4*>(&sm.eb.w.ev[r][8 * m]) = make_float4(cv[0], cv[1], cv[2], cv[3]);
  *reinterpret_cast<float4*>(&sm.eb.w.ev[r][8 * m + 4]) = make_float4(cv[4], cv[5], cv[6], cv[7]);
  // reduce-scatter the 8 columns over the 32 lanes: after the xor-16/8/4 stages lane L holds column
  // (L>>4)&1 | ((L>>3)&1)<<1 | ((L>>2)&1)<<2 summed over 8 lanes; xor 2 and 1 finish the sum
#pragma unroll
  for (int st = 16, n = 4; st >= 4; st >>= 1, n >>= 1) {
    const bool hi = ln & st;
#pragma unroll
    for (int i = 0; i < n; ++i) {
      const float keep = hi ? v[n + i] : v[i], send = hi ? v[i] : v[n + i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, st);
    }
  }
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
  const int gq = r >> a.lR;
  const int col = ((ln >> 4) & 1) * 4 + ((ln >> 3) & 1) * 2 + ((ln >> 2) & 1);
  // R = 64: a query spans two lane quarters; the odd one parks its partial column sums
  const bool lead = a.R == 32 || ((r >> 5) & 1) == 0;
  if (!lead && (ln & 3) == 0) sm.dqx[gq][8 * m + col] = v[0];
  if (a.R == 64) named_bar_sync(1, kQNT);
  if (lead && (ln & 3) == 0 && gq < it.nq) {
    const float y = a.R == 64 ? v[0] + sm.dqx[gq][8 * m + col] : v[0];
    const int64_t off = p.qoff(it.b, it.i0 + gq, it.h) + cs + col;
    if (a.out_f32)
      reinterpret_cast<float*>(a.dq)[off] = y;
    else
      reinterpret_cast<__nv_bfloat16*>(a.dq)[off] = __float2bfloat16_rn(y);
  }
  named_bar_sync(1, kQNT);
  const int P0 = p.np + it.i0;
  const int nsl = a.R + it.nq - 1;
  // key row kpos = P0 - R + 1 + sl receives rows (g, kk = sl - g); thread -> (sl, 4 columns)
  for (int idx = tidc; idx < nsl * 8; idx += kQNT) {
    const int sl = idx >> 3, d = 4 * (idx & 7);
    const int kp = P0 - a.R + 1 + sl;
    const int glo = max(0, sl - a.R + 1), ghi = min(it.nq - 1, sl);
    float4 tk[4], tv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // G = 4 (R = 32) or 2 (R = 64) terms
      const int gg = glo + u;
      const int row = (gg << a.lR) + (sl - gg);
      tk[u] = tv[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gg <= ghi) {
        tk[u] = *reinterpret_cast<const float4*>(&sm.eb.w.ek[row][d]);
        tv[u] = *reinterpret_cast<const float4*>(&sm.eb.w.ev[row][d]);
      }
    }
    int slot = sbase + sl;
    if (slot >= a.ring) slot -= a.ring;
    if (kp >= a.p.k2lo) {
      float4* ak = reinterpret_cast<float4*>(&q_acc(sm, a, 0)[slot][c0 + d]);
      float4* av = reinterpret_cast<float4*>(&q_acc(sm, a, 1)[slot][c0 + d]);
      float4 xk = *ak, xv = *av;
      xk.x += (tk[0].x + tk[1].x) + (tk[2].x + tk[3].x);
      xk.y += (tk[0].y + tk[1].y) + (tk[2].y + tk[3].y);
      xk.z += (tk[0].z + tk[1].z) + (tk[2].z + tk[3].z);
      xk.w += (tk[0].w + tk[1].w) + (tk[2].w + tk[3].w);
      xv.x += (tv[0].x + tv[1].x) + (tv[2].x + tv[3].x);
      xv.y += (tv[0].y + tv[1].y) + (tv[2].y + tv[3].y);
      xv.z += (tv[0].z + tv[1].z) + (tv[2].z + tv[3].z);
      xv.w += (tv[0].w + tv[1].w) + (tv[2].w + tv[3].w);
      *ak = xk;
      *av = xv;
    }
  }
  named_bar_sync(1, kQNT);
}

// R = 128 trilinear (G = 1): the tile is one query's 128 rows (row r = kk, key row kpos = P0-127+r).
// Warp m = 2 half + sub of a lane quarter takes columns c0+8m..+8 of W and U for its 32 rows.  Each
// row has its own key row, so dK2/dV2 need no cross-row reduction: the thread adds its row's
// s q o W and dO o U straight into the ring (padded pitch: float4 traffic conflict-free).  dq is a
// register reduce-scatter over the 32 lanes into per-lane-quarter partials (dq4), summed by the
// caller after one barrier.  No barrier inside the pass.
template <int D, int RING, bool STAGED>
__device__ __forceinline__ void q_epilogue_g1(QSmem<D, RING, STAGED>& sm, const BwdQArgs& a, int c0, int half,
                                              int sub, int r, bool valid, const QRows& rw, uint32_t tW, uint32_t tU,
                                              int sbase) {
  const float s = a.p.scale;
  const int ln = r & 31;
  const int m = 2 * half + sub;
  const int cs = c0 + 8 * m;
  uint32_t uw[8], uu[8];
  tmem_ld8(tW + cs, uw);
  tmem_ld8(tU + cs, uu);
  float k2v[8], qv[8], dov[8];
  if (valid) {
    load_f16<8>(rw.k2 + cs, k2v);
    load_f16<8>(rw.q + cs, qv);
    load_f16<8>(rw.dO + cs, dov);
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e) k2v[e] = qv[e] = dov[e] = 0.f;
  }
  int slot = sbase + r;
  if (slot >= a.ring) slot -= a.ring;
  auto ak = q_acc(sm, a, 0), av = q_acc(sm, a, 1);
  float4 xk0 = make_float4(0.f, 0.f, 0.f, 0.f), xk1 = xk0, xv0 = xk0, xv1 = xk0;
  if (valid) {
    xk0 = *reinterpret_cast<const float4*>(&ak[slot][cs]);
    xk1 = *reinterpret_cast<const float4*>(&ak[slot][cs + 4]);
    xv0 = *reinterpret_cast<const float4*>(&av[slot][cs]);
    xv1 = *reinterpret_cast<const float4*>(&av[slot][cs + 4]);
  }
  tmem_ld_wait();
  float v[8], ck[8], cv[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const float w = __uint_as_float(uw[e]);
    v[e] = s * k2v[e] * w;
    ck[e] = s * qv[e] * w;
    cv[e] = dov[e] * __uint_as_float(uu[e]);
  }
  if (valid) {
    *reinterpret_cast<float4*>(&ak[slot][cs]) =
        make_float4(xk0.x + ck[0], xk0.y + ck[1], xk0.z + ck[2], xk0.w + ck[3]);
    *reinterpret_cast<float4*>(&ak[slot][cs + 4]) =
        make_float4(xk1.x + ck[4], xk1.y + ck[5], xk1.z + ck[6], xk1.w + ck[7]);
    *reinterpret_cast<float4*>(&av[slot][cs]) =
        make_float4(xv0.x + cv[0], xv0.y + cv[1], xv0.z + cv[2], xv0.w + cv[3]);
    *reinterpret_cast<float4*>(&av[slot][cs + 4]) =
        make_float4(xv1.x + cv[4], xv1.y + cv[5], xv1.z + cv[6], xv1.w + cv[7]);
  }
  // reduce-scatter the 8 columns over the 32 lanes (as in q_epilogue_pass32)
#pragma unroll
  for (int st = 16, n = 4; st >= 4; st >>= 1, n >>= 1) {
    const bool hi = ln & st;
#pragma unroll
    for (int i = 0; i < n; ++i) {
      const float keep = hi ? v[n + i] : v[i], send = hi ? v[i] : v[n + i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, st);
    }
  }
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
  const int col = ((ln >> 4) & 1) * 4 + ((ln >> 3) & 1) * 2 + ((ln >> 2) & 1);
  if ((ln & 3) == 0) sm.dq4[r >> 5][cs + col] = v[0];
}

// R = 32 / 64 trilinear, row-owned: phase ph (0..3) of lane quarter qd (query g = qd >> (lR - 5))
// covers column block (ph + g * 4/G) & 3 (32 columns; warp m = 2 half + sub takes 8 of them).  The
// rows that share a key row belong to different queries, hence different column blocks in every
// phase, so each thread adds its row's s q o W and dO o U straight into the ring (padded pitch) with
// no gather; one barrier per phase separates the blocks.  dq: register reduce-scatter over the
// warp's 32 rows; R = 32 writes it, R = 64 parks the quarter's partial in dq4 (summed by the caller).
template <int D, int RING, bool STAGED>
__device__ __forceinline__ void q_epilogue_rot(QSmem<D, RING, STAGED>& sm, const BwdQArgs& a, const QItem& it,
                                               int half, int sub, int r, bool valid, const QRows& rw,
                                               uint32_t tW, uint32_t tU, int sbase, bool tr, int treg, int& trn,
                                               int titem) {
  const Problem& p = a.p;
  const float s = p.scale;
  const int ln = r & 31, qd = r >> 5;
  const int g = r >> a.lR;
  const int m = 2 * half + sub;
  const int rot = g << (a.lR - 5);  // g * R / 32 = g * 4 / G (R = 32: g, R = 64: 2g)
  int slot = sbase + (r & (a.R - 1)) + g;  // key row P0 - R + 1 + g + kk
  if (slot >= a.ring) slot -= a.ring;
  auto ak = q_acc(sm, a, 0), av = q_acc(sm, a, 1);
  // operands of phase ph+1 (TMEM W/U columns, fp16 row chunks) are requested before phase ph's
  // reduction and barrier, so their latency overlaps them
  constexpr bool kF = QSmem<D, RING, STAGED>::kRing;  // fp32 q (x s) / dO rows staged
  uint32_t uw[8], uu[8];
  uint4 rk2 = make_uint4(0u, 0u, 0u, 0u), rq = rk2, rdo = rk2;
  float4 fq0 = make_float4(0.f, 0.f, 0.f, 0.f), fq1 = fq0, fd0 = fq0, fd1 = fq0;
  int cs = 32 * (rot & 3) + 8 * m;
  tmem_ld8(tW + cs, uw);
  tmem_ld8(tU + cs, uu);
  if (valid) {
    rk2 = *reinterpret_cast<const uint4*>(rw.k2 + cs);
    if constexpr (kF) {
      fq0 = *reinterpret_cast<const float4*>(rw.qf + cs);
      fq1 = *reinterpret_cast<const float4*>(rw.qf + cs + 4);
      fd0 = *reinterpret_cast<const float4*>(rw.dOf + cs);
      fd1 = *reinterpret_cast<const float4*>(rw.dOf + cs + 4);
    } else {
      rq = *reinterpret_cast<const uint4*>(rw.q + cs);
      rdo = *reinterpret_cast<const uint4*>(rw.dO + cs);
    }
  }
#pragma unroll
  for (int ph = 0; ph < 4; ++ph) {
    float4 xk0 = make_float4(0.f, 0.f, 0.f, 0.f), xk1 = xk0, xv0 = xk0, xv1 = xk0;
    if (valid) {
      xk0 = *reinterpret_cast<const float4*>(&ak[slot][cs]);
      xk1 = *reinterpret_cast<const float4*>(&ak[slot][cs + 4]);
      xv0 = *reinterpret_cast<const float4*>(&av[slot][cs]);
      xv1 = *reinterpret_cast<const float4*>(&av[slot][cs + 4]);
    }
    tmem_ld_wait();
    float v[8], ck[8], cv[8];
    {
      const uint32_t ks[4] = {rk2.x, rk2.y, rk2.z, rk2.w}, qs[4] = {rq.x, rq.y, rq.z, rq.w},
                     ds[4] = {rdo.x, rdo.y, rdo.z, rdo.w};
      const float fq[8] = {fq0.x, fq0.y, fq0.z, fq0.w, fq1.x, fq1.y, fq1.z, fq1.w};
      const float fd[8] = {fd0.x, fd0.y, fd0.z, fd0.w, fd1.x, fd1.y, fd1.z, fd1.w};
#pragma unroll
      for (int e2 = 0; e2 < 4; ++e2) {
        const float2 kf = __half22float2(*reinterpret_cast<const __half2*>(&ks[e2]));
        const float w0 = __uint_as_float(uw[2 * e2]), w1 = __uint_as_float(uw[2 * e2 + 1]);
        v[2 * e2] = s * kf.x * w0;
        v[2 * e2 + 1] = s * kf.y * w1;
        if constexpr (kF) {
          ck[2 * e2] = fq[2 * e2] * w0;
          ck[2 * e2 + 1] = fq[2 * e2 + 1] * w1;
          cv[2 * e2] = fd[2 * e2] * __uint_as_float(uu[2 * e2]);
          cv[2 * e2 + 1] = fd[2 * e2 + 1] * __uint_as_float(uu[2 * e2 + 1]);
        } else {
          const float2 qf = __half22float2(*reinterpret_cast<const __half2*>(&qs[e2]));
          const float2 df = __half22float2(*reinterpret_cast<const __half2*>(&ds[e2]));
          ck[2 * e2] = s * qf.x * w0;
          ck[2 * e2 + 1] = s * qf.y * w1;
          cv[2 * e2] = df.x * __uint_as_float(uu[2 * e2]);
          cv[2 * e2 + 1] = df.y * __uint_as_float(uu[2 * e2 + 1]);
        }
      }
    }
    if (valid) {
      *reinterpret_cast<float4*>(&ak[slot][cs]) =
          make_float4(xk0.x + ck[0], xk0.y + ck[1], xk0.z + ck[2], xk0.w + ck[3]);
      *reinterpret_cast<float4*>(&ak[slot][cs + 4]) =
          make_float4(xk1.x + ck[4], xk1.y + ck[5], xk1.z + ck[6], xk1.w + ck[7]);
      *reinterpret_cast<float4*>(&av[slot][cs]) =
          make_float4(xv0.x + cv[0], xv0.y + cv[1], xv0.z + cv[2], xv0.w + cv[3]);
      *reinterpret_cast<float4*>(&av[slot][cs + 4]) =
          make_float4(xv1.x + cv[4], xv1.y + cv[5], xv1.z + cv[6], xv1.w + cv[7]);
    }
    const int csd = cs;
    SA_TRACE_AT(tr, treg, trn, titem << 16 | 12 << 8 | ph);
    if (ph < 3) {
      cs = 32 * ((ph + 1 + rot) & 3) + 8 * m;
      tmem_ld8(tW + cs, uw);
      tmem_ld8(tU + cs, uu);
      if (valid) {
        rk2 = *reinterpret_cast<const uint4*>(rw.k2 + cs);
        if constexpr (kF) {
          fq0 = *reinterpret_cast<const float4*>(rw.qf + cs);
          fq1 = *reinterpret_cast<const float4*>(rw.qf + cs + 4);
          fd0 = *reinterpret_cast<const float4*>(rw.dOf + cs);
          fd1 = *reinterpret_cast<const float4*>(rw.dOf + cs + 4);
        } else {
          rq = *reinterpret_cast<const uint4*>(rw.q + cs);
          rdo = *reinterpret_cast<const uint4*>(rw.dO + cs);
        }
      }
    }
#pragma unroll
    for (int st = 16, n = 4; st >= 4; st >>= 1, n >>= 1) {
      const bool hi = ln & st;
#pragma unroll
      for (int i = 0; i < n; ++i) {
        const float keep = hi ? v[n + i] : v[i], send = hi ? v[i] : v[n + i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, st);
      }
    }
    v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
    v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
    const int col = ((ln >> 4) & 1) * 4 + ((ln >> 3) & 1) * 2 + ((ln >> 2) & 1);
    if ((ln & 3) == 0) {
      if (a.R == 32) {
        if (g < it.nq) {
          const int64_t off = p.qoff(it.b, it.i0 + g, it.h) + csd + col;
          if (a.out_f32)
            reinterpret_cast<float*>(a.dq)[off] = v[0];
          else
            reinterpret_cast<__nv_bfloat16*>(a.dq)[off] = __float2bfloat16_rn(v[0]);
        }
      } else {
        sm.dq4[qd][csd + col] = v[0];
      }
    }
    named_bar_sync(1, kQNT);
    SA_TRACE_AT(tr, treg, trn, titem << 16 | 13 << 8 | ph);
  }
}

// Small-R variant of q_epilogue_pass32 (R in {2, 4, 8, 16}, compile-time; R = 32/64 keep the
// specialised function above).  Trilinear pass over 32 columns [c0, c0+32): warp m = 2 half + sub of
// a TMEM lane quarter takes columns c0+8m..+8 of both W (dq and the dk2 rows) and U (the dv2 rows).
// A warp holds 32/R whole queries in aligned groups of R lanes: dq is a reduce-scatter inside the
// group (a lane keeps max(1, 8/R) columns; for R = 16 a final xor-1 add leaves lane pairs with the
// same column); dk2/dv2 go through the shared-memory band gather, one thread per (key slot, 4
// columns, k2 or v2) summing its min(R, G) rows.
template <int D, int RING, bool STAGED, int R>
__device__ __forceinline__ void q_epilogue_pass_small(QSmem<D, RING, STAGED>& sm, const BwdQArgs& a, const QItem& it,
                                                      int c0, int half, int sub, int r, bool valid, const QRows& rw,
                                                      uint32_t tW, uint32_t tU, int tidc, int sbase) {
  constexpr int G = 128 / R, LR = R == 2 ? 1 : R == 4 ? 2 : R == 8 ? 3 : 4, T = R < G ? R : G;
  const Problem& p = a.p;
  const float s = p.scale;
  const int ln = r & 31;
  const int m = 2 * half + sub;
  const int cs = c0 + 8 * m;
  uint32_t uw[8], uu[8];
  tmem_ld8(tW + cs, uw);
  tmem_ld8(tU + cs, uu);
  float k2v[8], qv[8], dov[8];
  if (valid) {
    load_f16<8>(rw.k2 + cs, k2v);
    load_f16<8>(rw.q + cs, qv);
    load_f16<8>(rw.dO + cs, dov);
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e) k2v[e] = qv[e] = dov[e] = 0.f;
  }
  tmem_ld_wait();
  float v[8], ck[8], cv[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const float w = __uint_as_float(uw[e]);
    v[e] = s * k2v[e] * w;
    ck[e] = s * qv[e] * w;
    cv[e] = dov[e] * __uint_as_float(uu[e]);
  }
  *reinterpret_cast<float4*>(&sm.eb.w.ek[r][8 * m]) = make_float4(ck[0], ck[1], ck[2], ck[3]);
  *reinterpret_cast<float4*>(&sm.eb.w.ek[r][8 * m + 4]) = make_float4(ck[4], ck[5], ck[6], ck[7]);
  *reinterpret_cast<float4*>(&sm.eb.w.ev[r][8 * m]) = make_float4(cv[0], cv[1], cv[2], cv[3]);
  *reinterpret_cast<float4*>(&sm.eb.w.ev[r][8 * m + 4]) = make_float4(cv[4], cv[5], cv[6], cv[7]);
  const int gl = ln & (R - 1);
  int cbase = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {  // stages st = R/2, ..., 1
    constexpr int kR = R;
    const int st = (kR >> 1) >> k, n = 4 >> k;
    if (st > 0) {
      if (n >= 1) {
        const bool hi = gl & st;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (i < n) {
            const float keep = hi ? v[n + i] : v[i], send = hi ? v[i] : v[n + i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, st);
          }
        }
        if (hi) cbase += n;
      } else {
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], st);
      }
    }
  }
  constexpr int NF = R >= 8 ? 1 : 8 / R;
  const int gq = r >> LR;
  if ((R < 16 || (gl & 1) == 0) && gq < it.nq) {
    const int64_t off = p.qoff(it.b, it.i0 + gq, it.h) + cs + cbase;
    if (a.out_f32) {
#pragma unroll
      for (int i = 0; i < NF; ++i) reinterpret_cast<float*>(a.dq)[off + i] = v[i];
    } else if constexpr (NF >= 2) {
#pragma unroll
      for (int i = 0; i < NF; i += 2)
        *reinterpret_cast<__nv_bfloat162*>(reinterpret_cast<__nv_bfloat16*>(a.dq) + off + i) =
            __floats2bfloat162_rn(v[i], v[i + 1]);
    } else {
      reinterpret_cast<__nv_bfloat16*>(a.dq)[off] = __float2bfloat16_rn(v[0]);
    }
  }
  named_bar_sync(1, kQNT);
  const int P0 = p.np + it.i0;
  const int nsl = R + it.nq - 1;
  // key row kpos = P0 - R + 1 + sl receives rows (g, kk = sl - g); thread -> (sl, 4 columns, k2|v2)
  for (int idx = tidc; idx < nsl * 16; idx += kQNT) {
    const int which = idx & 1, sl = idx >> 4, d = 4 * ((idx >> 1) & 7);
    const int kp = P0 - R + 1 + sl;
    const int glo = max(0, sl - R + 1), ghi = min(it.nq - 1, sl);
    const float(*src)[36] = which ? sm.eb.w.ev : sm.eb.w.ek;
    float4 t[T];
#pragma unroll
    for (int u = 0; u < T; ++u) {
      const int gg = glo + u;
      t[u] = gg <= ghi ? *reinterpret_cast<const float4*>(&src[(gg << LR) + (sl - gg)][d])
                       : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int w = 1; w < T; w <<= 1)
#pragma unroll
      for (int u = 0; u + w < T; u += 2 * w)
        t[u] = make_float4(t[u].x + t[u + w].x, t[u].y + t[u + w].y, t[u].z + t[u + w].z, t[u].w + t[u + w].w);
    int slot = sbase + sl;
    if (slot >= a.ring) slot -= a.ring;
    if (kp >= a.p.k2lo) {
      float4* acc = reinterpret_cast<float4*>(&q_acc(sm, a, which)[slot][c0 + d]);
      float4 x = *acc;
      x.x += t[0].x, x.y += t[0].y, x.z += t[0].z, x.w += t[0].w;
      *acc = x;
    }
  }
  named_bar_sync(1, kQNT);
}

// Determinant pass over 24 columns [c0, c0+24) (eight 3-chunks), R in {32, 64}: warp m = 2 half + sub
// of a lane quarter takes columns c0+6m..+6 (two chunks) of W (dq = s sum_k W x k2, dk2 rows
// s q x W) and of U (dv2 rows dO o U); dq by a register reduce-scatter over the 32 lanes (six
// values padded to eight), dk2/dv2 through the shared-memory gather in float2 pairs.  Dims past the
// last whole chunk (D mod 3) contribute 0 (reading R5).
template <int D, int RING, bool STAGED>
__device__ __forceinline__ void q_epilogue_pass_det(QSmem<D, RING, STAGED>& sm, const BwdQArgs& a, const QItem& it,
                                                    int c0, int half, int sub, int r, bool valid, const QRows& rw,
                                                    uint32_t tW, uint32_t tU, int tidc, int sbase) {
  constexpr int D3 = (D / 3) * 3;
  const Problem& p = a.p;
  const float s = p.scale;
  const int ln = r & 31;
  const int m = 2 * half + sub;
  const int cs = c0 + 6 * m;
  const bool act = cs < D;  // warp-uniform
  float v[8], ck[6], cv[6];
#pragma unroll
  for (int e = 0; e < 8; ++e) v[e] = 0.f;
#pragma unroll
  for (int e = 0; e < 6; ++e) ck[e] = cv[e] = 0.f;
  if (act) {
    uint32_t uw[8], uu[8];
    tmem_ld8(tW + cs, uw);
    tmem_ld8(tU + cs, uu);
    float k2v[6], qv[6], dov[6];
#pragma unroll
    for (int e = 0; e < 6; ++e) k2v[e] = qv[e] = dov[e] = 0.f;
    if (valid) {
#pragma unroll
      for (int e = 0; e < 6; e += 2) {
        if (cs + e < D) {
          const float2 a2 = __half22float2(*reinterpret_cast<const __half2*>(rw.k2 + cs + e));
          const float2 b2 = __half22float2(*reinterpret_cast<const __half2*>(rw.q + cs + e));
          const float2 c2 = __half22float2(*reinterpret_cast<const __half2*>(rw.dO + cs + e));
          k2v[e] = a2.x, k2v[e + 1] = a2.y, qv[e] = b2.x, qv[e + 1] = b2.y, dov[e] = c2.x, dov[e + 1] = c2.y;
        }
      }
    }
    tmem_ld_wait();
    float w[6];
#pragma unroll
    for (int e = 0; e < 6; ++e) w[e] = __uint_as_float(uw[e]);
#pragma unroll
    for (int t = 0; t < 6; t += 3) {
      if (cs + t + 3 <= D3) {  // dq: W x k2 ; dk2: q x W     ((x cross y)_r = x_{r+1} y_{r+2} - x_{r+2} y_{r+1})
        v[t + 0] = s * (w[t + 1] * k2v[t + 2] - w[t + 2] * k2v[t + 1]);
        v[t + 1] = s * (w[t + 2] * k2v[t + 0] - w[t + 0] * k2v[t + 2]);
        v[t + 2] = s * (w[t + 0] * k2v[t + 1] - w[t + 1] * k2v[t + 0]);
        ck[t + 0] = s * (qv[t + 1] * w[t + 2] - qv[t + 2] * w[t + 1]);
        ck[t + 1] = s * (qv[t + 2] * w[t + 0] - qv[t + 0] * w[t + 2]);
        ck[t + 2] = s * (qv[t + 0] * w[t + 1] - qv[t + 1] * w[t + 0]);
      }
    }
#pragma unroll
    for (int e = 0; e < 6; ++e) cv[e] = cs + e < D ? dov[e] * __uint_as_float(uu[e]) : 0.f;
#pragma unroll
    for (int e = 0; e < 6; e += 2) {
      *reinterpret_cast<float2*>(&sm.eb.w.ek[r][6 * m + e]) = make_float2(ck[e], ck[e + 1]);
      *reinterpret_cast<float2*>(&sm.eb.w.ev[r][6 * m + e]) = make_float2(cv[e], cv[e + 1]);
    }
  }
  // reduce-scatter the 8 (six real) dq columns over the 32 lanes, as in q_epilogue_pass32
#pragma unroll
  for (int st = 16, n = 4; st >= 4; st >>= 1, n >>= 1) {
    const bool hi = ln & st;
#pragma unroll
    for (int i = 0; i < n; ++i) {
      const float keep = hi ? v[n + i] : v[i], send = hi ? v[i] : v[n + i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, st);
    }
  }
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
  const int gq = r >> a.lR;
  const int col = ((ln >> 4) & 1) * 4 + ((ln >> 3) & 1) * 2 + ((ln >> 2) & 1);
  const bool lead = a.R == 32 || ((r >> 5) & 1) == 0;
  if (act && !lead && (ln & 3) == 0 && col < 6) sm.dqx[gq][6 * m + col] = v[0];
  if (a.R == 64) named_bar_sync(1, kQNT);
  if (act && lead && (ln & 3) == 0 && col < 6 && cs + col < D && gq < it.nq) {
    const float y = a.R == 64 ? v[0] + sm.dqx[gq][6 * m + col] : v[0];
    const int64_t off = p.qoff(it.b, it.i0 + gq, it.h) + cs + col;
    if (a.out_f32)
      reinterpret_cast<float*>(a.dq)[off] = y;
    else
      reinterpret_cast<__nv_bfloat16*>(a.dq)[off] = __float2bfloat16_rn(y);
  }
  named_bar_sync(1, kQNT);
  // key row kpos = P0 - R + 1 + sl receives rows (g, kk = sl - g); thread -> (sl, column pair)
  const int P0 = p.np + it.i0;
  const int nsl = a.R + it.nq - 1;
  const int npair = (min(24, D - c0) + 1) / 2;
  for (int idx = tidc; idx < nsl * 12; idx += kQNT) {
    const int sl = idx / 12, d = 2 * (idx % 12);
    if (d >= 2 * npair) continue;
    const int kp = P0 - a.R + 1 + sl;
    const int glo = max(0, sl - a.R + 1), ghi = min(it.nq - 1, sl);
    float2 xk = make_float2(0.f, 0.f), xv = xk;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int gg = glo + u;
      if (gg <= ghi) {
        const int row = (gg << a.lR) + (sl - gg);
        const float2 tk = *reinterpret_cast<const float2*>(&sm.eb.w.ek[row][d]);
        const float2 tv = *reinterpret_cast<const float2*>(&sm.eb.w.ev[row][d]);
        xk.x += tk.x, xk.y += tk.y, xv.x += tv.x, xv.y += tv.y;
      }
    }
    int slot = sbase + sl;
    if (slot >= a.ring) slot -= a.ring;
    if (kp >= a.p.k2lo) {
      float2* ak = reinterpret_cast<float2*>(&q_acc(sm, a, 0)[slot][c0 + d]);
      float2* av = reinterpret_cast<float2*>(&q_acc(sm, a, 1)[slot][c0 + d]);
      float2 yk = *ak, yv = *av;
      yk.x += xk.x, yk.y += xk.y, yv.x += xv.x, yv.y += xv.y;
      *ak = yk;
      *av = yv;
    }
  }
  named_bar_sync(1, kQNT);
}

// Half SUB of the determinant row operand k2 x q: columns [D/2 SUB, D/2 SUB + D/2), by 3-chunk
// permutations of the packed fp16 rows (sa_tc_rows.cuh det_words_f16).  Columns past the last whole
// chunk are 0 (reading R5).
template <int D, int SUB>
__device__ __forceinline__ void det_half_operand(const __half* x, const __half* y, uint32_t (&pk)[D / 4]) {
  det_words_f16<D, SUB * D / 4, D / 4>(x, y, pk);
}

// Determinant epilogue at R = 32 (G = 4 queries, one per TMEM lane quarter), row-owned like
// q_epilogue_rot: six 24-column blocks (eight 3-chunks each; the last holds chunks 40-41 and the two
// trailing columns), warp m = 2 half + sub of a lane quarter takes 6 columns (two chunks) of a block.
// Query g works on block (ph + g) mod 6 in phase ph, so rows of different queries that share a key
// row never update the same ring columns in the same phase; one barrier per phase.  Per thread:
//   dq  (register reduce-scatter over the query's 32 rows)  s sum_k W x k2
//   dk2 ring row += s q x W,   dv2 ring row += dO o U      (cross products chunkwise, reading R5:
//   the D mod 3 trailing columns get no dq / dk2, but their dv2 = dO o U)
template <int D, int RING, bool STAGED>
__device__ __forceinline__ void q_epilogue_rot_det(QSmem<D, RING, STAGED>& sm, const BwdQArgs& a, const QItem& it,
                                                   int half, int sub, int r, bool valid, const QRows& rw,
                                                   uint32_t tW, uint32_t tU, int sbase) {
  constexpr int D3 = (D / 3) * 3;
  constexpr int kNB = (D + 23) / 24;  // 24-column blocks
  const Problem& p = a.p;
  const float s = p.scale;
  const int ln = r & 31, g = r >> 5;
  const int m = 2 * half + sub;
  int slot = sbase + (r & 31) + g;  // key row P0 - 31 + g + kk
  if (slot >= a.ring) slot -= a.ring;
  auto ak = q_acc(sm, a, 0), av = q_acc(sm, a, 1);
#pragma unroll 1
  for (int ph = 0; ph < kNB; ++ph) {
    int b = ph + g;
    if (b >= kNB) b -= kNB;
    const int cs = 24 * b + 6 * m;
    const bool act = cs < D;  // warp-uniform
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = 0.f;
    if (act) {
      uint32_t uw[8], uu[8];
      tmem_ld8(tW + cs, uw);
      tmem_ld8(tU + cs, uu);
      float k2v[6], qv[6], dov[6];
#pragma unroll
      for (int e = 0; e < 6; ++e) k2v[e] = qv[e] = dov[e] = 0.f;
      if (valid) {
#pragma unroll
        for (int e = 0; e < 6; e += 2) {
          if (cs + e < D) {
            const float2 a2 = __half22float2(*reinterpret_cast<const __half2*>(rw.k2 + cs + e));
            const float2 b2 = __half22float2(*reinterpret_cast<const __half2*>(rw.q + cs + e));
            const float2 c2 = __half22float2(*reinterpret_cast<const __half2*>(rw.dO + cs + e));
            k2v[e] = a2.x, k2v[e + 1] = a2.y, qv[e] = b2.x, qv[e + 1] = b2.y, dov[e] = c2.x, dov[e + 1] = c2.y;
          }
        }
      }
      tmem_ld_wait();
      float w[6], ck[6], cv[6];
#pragma unroll
      for (int e = 0; e < 6; ++e) {
        w[e] = __uint_as_float(uw[e]);
        ck[e] = 0.f;
        cv[e] = cs + e < D ? dov[e] * __uint_as_float(uu[e]) : 0.f;
      }
#pragma unroll
      for (int t = 0; t < 6; t += 3) {
        if (cs + t + 3 <= D3) {  // dq: W x k2 ; dk2: q x W     ((x cross y)_r = x_{r+1} y_{r+2} - x_{r+2} y_{r+1})
          v[t + 0] = s * (w[t + 1] * k2v[t + 2] - w[t + 2] * k2v[t + 1]);
          v[t + 1] = s * (w[t + 2] * k2v[t + 0] - w[t + 0] * k2v[t + 2]);
          v[t + 2] = s * (w[t + 0] * k2v[t + 1] - w[t + 1] * k2v[t + 0]);
          ck[t + 0] = s * (qv[t + 1] * w[t + 2] - qv[t + 2] * w[t + 1]);
          ck[t + 1] = s * (qv[t + 2] * w[t + 0] - qv[t + 0] * w[t + 2]);
          ck[t + 2] = s * (qv[t + 0] * w[t + 1] - qv[t + 1] * w[t + 0]);
        }
      }
      if (valid) {
#pragma unroll
        for (int e = 0; e < 6; e += 2) {
          if (cs + e < D) {
            float2* pk = reinterpret_cast<float2*>(&ak[slot][cs + e]);
            float2* pv = reinterpret_cast<float2*>(&av[slot][cs + e]);
            float2 xk = *pk, xv = *pv;
            xk.x += ck[e], xk.y += ck[e + 1], xv.x += cv[e], xv.y += cv[e + 1];
            *pk = xk;
            *pv = xv;
          }
        }
      }
    }
    // reduce-scatter the 8 (six real) dq columns over the query's 32 lanes
#pragma unroll
    for (int st = 16, n = 4; st >= 4; st >>= 1, n >>= 1) {
      const bool hi = ln & st;
#pragma unroll
      for (int i = 0; i < n; ++i) {
        const float keep = hi ? v[n + i] : v[i], send = hi ? v[i] : v[n + i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, st);
      }
    }
    v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
    v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
    const int col = ((ln >> 4) & 1) * 4 + ((ln >> 3) & 1) * 2 + ((ln >> 2) & 1);
    if (act && (ln & 3) == 0 && col < 6 && cs + col < D && g < it.nq) {
      const int64_t off = p.qoff(it.b, it.i0 + g, it.h) + cs + col;
      if (a.out_f32)
        reinterpret_cast<float*>(a.dq)[off] = v[0];
      else
        reinterpret_cast<__nv_bfloat16*>(a.dq)[off] = __float2bfloat16_rn(v[0]);
    }
    named_bar_sync(1, kQNT);
  }
}

// Determinant epilogue at R = 32 in four phases (the trilinear rotation of q_epilogue_rot): phase ph of
// query g covers the 32 output columns of block (ph + g) & 3, warp m = 2 half + sub takes 8 of them
// [cs, cs + 8).  The cross products of an output column read the other two columns of its 3-chunk,
// which may lie outside the block: the thread loads the chunk-aligned window [c0, c0 + 12),
// c0 = cs - cs mod 3, of W (TMEM, read-only), k2 and s q; only its own 8 dk2 / dv2 ring columns are
// written, so the block rotation keeps rows of different queries that share a key row apart.
//   dq_c  = s (W x k2)_c,   dk2_c += (s q x W)_c,   dv2_c += dO_c U_c   (columns >= 3 floor(D/3): dq,
//   dk2 contributions 0, reading R5).  The window offset o = cs - c0 (warp-uniform) selects one of three
// compile-time index maps.
// w[i] = W column c0 + i; k2[i], qs[i] = column cs - 4 + i (vector-loaded window), cs = c0 + O
template <int O>
__device__ __forceinline__ void det_cols8(const float (&w)[16], const float (&k2)[16], const float (&qs)[16],
                                          float s, int c0, int d3, float (&v)[8], float (&ck)[8]) {
  constexpr int kS = 4 - O;  // window index of column c0
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int t = O + j, tb = 3 * (t / 3), r = t % 3;
    const int i1 = tb + (r + 1) % 3, i2 = tb + (r + 2) % 3;
    const bool in = c0 + tb + 3 <= d3;
    v[j] = in ? s * (w[i1] * k2[kS + i2] - w[i2] * k2[kS + i1]) : 0.f;
    ck[j] = in ? qs[kS + i1] * w[i2] - qs[kS + i2] * w[i1] : 0.f;
  }
}

template <int D, int RING, bool STAGED>
__device__ __forceinline__ void q_epilogue_rot_det4(QSmem<D, RING, STAGED>& sm, const BwdQArgs& a, const QItem& it,
                                                    int half, int sub, int r, bool valid, const QRows& rw,
                                                    uint32_t tW, uint32_t tU, int sbase) {
  static_assert(QSmem<D, RING, STAGED>::kRing, "staged fp32 q rows");
  constexpr int D3 = (D / 3) * 3;
  const Problem& p = a.p;
  const float s = p.scale;
  const int ln = r & 31, g = r >> 5;
  const int m = 2 * half + sub;
  int slot = sbase + (r & 31) + g;  // key row P0 - 31 + g + kk
  if (slot >= a.ring) slot -= a.ring;
  auto ak = q_acc(sm, a, 0), av = q_acc(sm, a, 1);
  uint32_t uw[16], uu[8];
  int cs = 32 * (g & 3) + 8 * m;
  int c0 = cs - cs % 3;
  tmem_ld16(tW + c0, uw);
  tmem_ld8(tU + cs, uu);
#pragma unroll
  for (int ph = 0; ph < 4; ++ph) {
    // k2 and s q over the 16-column window [cs - 4, cs + 12) (covers the chunk-aligned [c0, c0 + 12)):
    // four 8-byte fp16 and four 16-byte fp32 loads; columns past D are masked in det_cols8
    float k2v[16], qs[16];
    float4 fd0 = make_float4(0.f, 0.f, 0.f, 0.f), fd1 = fd0;
    float4 xk0 = fd0, xk1 = fd0, xv0 = fd0, xv1 = fd0;
#pragma unroll
    for (int e = 0; e < 16; ++e) k2v[e] = qs[e] = 0.f;
    if (valid) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int cw = cs - 4 + 4 * u;
        if (cw >= 0) {
          const uint2 h = *reinterpret_cast<const uint2*>(rw.k2 + cw);
          const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&h.x));
          const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&h.y));
          k2v[4 * u] = f0.x, k2v[4 * u + 1] = f0.y, k2v[4 * u + 2] = f1.x, k2v[4 * u + 3] = f1.y;
          const float4 q4 = *reinterpret_cast<const float4*>(rw.qf + cw);  // s q (cvt_qf)
          qs[4 * u] = q4.x, qs[4 * u + 1] = q4.y, qs[4 * u + 2] = q4.z, qs[4 * u + 3] = q4.w;
        }
      }
      fd0 = *reinterpret_cast<const float4*>(rw.dOf + cs);
      fd1 = *reinterpret_cast<const float4*>(rw.dOf + cs + 4);
      xk0 = *reinterpret_cast<const float4*>(&ak[slot][cs]);
      xk1 = *reinterpret_cast<const float4*>(&ak[slot][cs + 4]);
      xv0 = *reinterpret_cast<const float4*>(&av[slot][cs]);
      xv1 = *reinterpret_cast<const float4*>(&av[slot][cs + 4]);
    }
    tmem_ld_wait();
    float w[16], v[8], ck[8], cv[8];
#pragma unroll
    for (int e = 0; e < 16; ++e) w[e] = __uint_as_float(uw[e]);
    const int o = cs - c0;
    if (o == 0)
      det_cols8<0>(w, k2v, qs, s, c0, D3, v, ck);
    else if (o == 1)
      det_cols8<1>(w, k2v, qs, s, c0, D3, v, ck);
    else
      det_cols8<2>(w, k2v, qs, s, c0, D3, v, ck);
    {
      const float fd[8] = {fd0.x, fd0.y, fd0.z, fd0.w, fd1.x, fd1.y, fd1.z, fd1.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) cv[e] = fd[e] * __uint_as_float(uu[e]);
    }
    if (valid) {
      *reinterpret_cast<float4*>(&ak[slot][cs]) =
          make_float4(xk0.x + ck[0], xk0.y + ck[1], xk0.z + ck[2], xk0.w + ck[3]);
      *reinterpret_cast<float4*>(&ak[slot][cs + 4]) =
          make_float4(xk1.x + ck[4], xk1.y + ck[5], xk1.z + ck[6], xk1.w + ck[7]);
      *reinterpret_cast<float4*>(&av[slot][cs]) =
          make_float4(xv0.x + cv[0], xv0.y + cv[1], xv0.z + cv[2], xv0.w + cv[3]);
      *reinterpret_cast<float4*>(&av[slot][cs + 4]) =
          make_float4(xv1.x + cv[4], xv1.y + cv[5], xv1.z + cv[6], xv1.w + cv[7]);
    }
    const int csd = cs;
    if (ph < 3) {  // next phase's TMEM columns before this phase's reduction and barrier
      cs = 32 * ((ph + 1 + g) & 3) + 8 * m;
      c0 = cs - cs % 3;
      tmem_ld16(tW + c0, uw);
      tmem_ld8(tU + cs, uu);
    }
#pragma unroll
    for (int st = 16, n = 4; st >= 4; st >>= 1, n >>= 1) {
      const bool hi = ln & st;
#pragma unroll
      for (int i = 0; i < n; ++i) {
        const float keep = hi ? v[n + i] : v[i], send = hi ? v[i] : v[n + i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, st);
      }
    }
    v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
    v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
    const int col = ((ln >> 4) & 1) * 4 + ((ln >> 3) & 1) * 2 + ((ln >> 2) & 1);
    if ((ln & 3) == 0 && g < it.nq) {
      const int64_t off = p.qoff(it.b, it.i0 + g, it.h) + csd + col;
      if (a.out_f32)
        reinterpret_cast<float*>(a.dq)[off] = v[0];
      else
        reinterpret_cast<__nv_bfloat16*>(a.dq)[off] = __float2bfloat16_rn(v[0]);
    }
    named_bar_sync(1, kQNT);
  }
}

// R in {8, 16} trilinear epilogue on the tensor core (RING 38).  The three row-group sums of a tile,
//   dq_g   = sum_{kk}        X1_(g,kk),   X1 = s k2 o W      (rows of query g)
//   dk2_k += sum_{g+kk = k}  X2_(g,kk),   X2 = s q o W       (rows sharing key slot k)
//   dv2_k += sum_{g+kk = k}  X3_(g,kk),   X3 = dO o U
// run as MMAs  Y^T = X^T Sel^T  (M = D TMEM lanes, N = 16 query / 32 key-slot columns, K = the 128
// tile rows) with constant 0/1 selection matrices, one shared X tile rewritten per product (the MMA
// warp issues each after named barrier 5 and commits to `red`).  Results land in the tile's W
// columns (read out before X1 is published): dq^T at [0, 16), dk2^T at [32, 64), dv2^T at [64, 96).
// X is rounded to fp16 (reading R25).  Thread (row r, warp m = 2 half + sub) owns columns
// [m D/4, (m+1) D/4) of its row; afterwards warp m handles query / key-slot columns j = m mod 4.
template <int D, int RING, bool STAGED>
__device__ __forceinline__ void q_epilogue_tc(QSmem<D, RING, STAGED>& sm, const BwdQArgs& a, const QItem& it,
                                              int half, int sub, int r, bool valid, const QRows& rw, uint32_t tW,
                                              uint32_t tU, int sbase, uint32_t& nred, bool tr, int treg, int& trn,
                                              int titem) {
  constexpr int CW = D / 4;  // columns per thread
  const Problem& p = a.p;
  const float s = p.scale;
  const int m = 2 * half + sub, c0 = CW * m;
  const int qd = r >> 5, lane = r & 31;
  uint8_t* xb = sm.xr;
  uint32_t uw[CW];
  if constexpr (CW == 32)
    tmem_ld32(tW + c0, *reinterpret_cast<uint32_t(*)[32]>(uw));
  else
    tmem_ld16(tW + c0, uw);
  uint32_t k2w[CW / 2], qw[CW / 2], dw[CW / 2];
#pragma unroll
  for (int t = 0; t < CW / 8; ++t) {
    uint4 a4 = make_uint4(0u, 0u, 0u, 0u), b4 = a4, c4 = a4;
    if (valid) {
      a4 = *reinterpret_cast<const uint4*>(rw.k2 + c0 + 8 * t);
      b4 = *reinterpret_cast<const uint4*>(rw.q + c0 + 8 * t);
      c4 = *reinterpret_cast<const uint4*>(rw.dO + c0 + 8 * t);
    }
    k2w[4 * t] = a4.x, k2w[4 * t + 1] = a4.y, k2w[4 * t + 2] = a4.z, k2w[4 * t + 3] = a4.w;
    qw[4 * t] = b4.x, qw[4 * t + 1] = b4.y, qw[4 * t + 2] = b4.z, qw[4 * t + 3] = b4.w;
    dw[4 * t] = c4.x, dw[4 * t + 1] = c4.y, dw[4 * t + 2] = c4.z, dw[4 * t + 3] = c4.w;
  }
  tmem_ld_wait();
  // X = (f16 row y) o (fp32 TMEM columns u) * sc, stored as this row's 16-byte chunks c0/8 ...
  auto put = [&](const uint32_t* y, const uint32_t* u, float sc) {
    uint32_t pk[CW / 2];
#pragma unroll
    for (int e = 0; e < CW / 2; ++e) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&y[e]));
      pk[e] = pack_f16x2(sc * f.x * __uint_as_float(u[2 * e]), sc * f.y * __uint_as_float(u[2 * e + 1]));
    }
#pragma unroll
    for (int t = 0; t < CW / 8; ++t) {
      const int c8 = c0 / 8 + t;
      *reinterpret_cast<uint4*>(xb + (c8 >> 3) * (128 * 128) + r * 128 + (((c8 & 7) ^ (r & 7)) << 4)) =
          make_uint4(pk[4 * t], pk[4 * t + 1], pk[4 * t + 2], pk[4 * t + 3]);
    }
    fence_proxy_async_smem();
    tc_fence_before();
    named_bar_arrive(5, kQNT + 32);
  };
  auto wait_red = [&]() {
    mbar_wait(&sm.red, nred & 1);
    ++nred;
  };
  put(k2w, uw, s);  // X1 = s k2 o W  -> dq
  SA_TRACE_AT(tr, treg, trn, titem << 16 | 15 << 8);
  wait_red();
  SA_TRACE_AT(tr, treg, trn, titem << 16 | 16 << 8);
  put(qw, uw, s);   // X2 = s q o W   -> dk2
  if constexpr (CW == 32)
    tmem_ld32(tU + c0, *reinterpret_cast<uint32_t(*)[32]>(uw));
  else
    tmem_ld16(tU + c0, uw);
  tmem_ld_wait();
  wait_red();
  SA_TRACE_AT(tr, treg, trn, titem << 16 | 17 << 8);
  put(dw, uw, 1.f);  // X3 = dO o U   -> dv2
  wait_red();
  tc_fence_after();
  SA_TRACE_AT(tr, treg, trn, titem << 16 | 18 << 8);
  // results: lane = column d of this lane quarter; warp m takes queries [4m, 4m + 4) and key slots
  // [8m, 8m + 8) (eight TMEM columns of each result: few live registers)
  const int d = 32 * qd + lane;
  uint32_t yq[8], yk[8], yv[8];
  tmem_ld8(tW + 4 * m, yq);
  tmem_ld8(tW + 32 + 8 * m, yk);
  tmem_ld8(tW + 64 + 8 * m, yv);
  tmem_ld_wait();
  SA_TRACE_AT(tr, treg, trn, titem << 16 | 19 << 8);
  if (d < D) {
    const int64_t qstride = int64_t(p.H) * D;
    const int64_t off0 = p.qoff(it.b, it.i0, it.h) + d + 4 * m * qstride;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (4 * m + j < it.nq) {
        const float y = __uint_as_float(yq[j]);
        if (a.out_f32)
          reinterpret_cast<float*>(a.dq)[off0 + j * qstride] = y;
        else
          reinterpret_cast<__nv_bfloat16*>(a.dq)[off0 + j * qstride] = __float2bfloat16_rn(y);
      }
    }
    const int P0 = p.np + it.i0;
    const int nsl = a.R + it.nq - 1;
    auto ak = q_acc(sm, a, 0), av = q_acc(sm, a, 1);
    int slot = sbase + 8 * m;
    if (slot >= a.ring) slot -= a.ring;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k = 8 * m + j;
      if (k < nsl && P0 - a.R + 1 + k >= p.k2lo) {
        ak[slot][d] += __uint_as_float(yk[j]);
        av[slot][d] += __uint_as_float(yv[j]);
      }
      if (++slot == a.ring) slot = 0;
    }
  }
  SA_TRACE_AT(tr, treg, trn, titem << 16 | 20 << 8);
  named_bar_sync(1, kQNT);  // ring rows complete before the flush
  SA_TRACE_AT(tr, treg, trn, titem << 16 | 21 << 8);
}

template <int D, bool DET, int RING, bool STAGED>
__global__ void __launch_bounds__(kQThreads, 1)
    tc_bwd_q_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                    const __grid_constant__ CUtensorMap tmQs, const __grid_constant__ CUtensorMap tmdOs,
                    const __grid_constant__ CUtensorMap tmK2s, const __grid_constant__ CUtensorMap tmV2s,
                    BwdQArgs a) {
  using Sm = QSmem<D, RING, STAGED>;
  extern __shared__ uint8_t smem_raw[];
  static_assert(sizeof(Sm) + 1024 <= 232448, "shared memory budget");
  Sm& sm = *reinterpret_cast<Sm*>(smem_raw + align1024_pad(smem_raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kStages = Sm::kStages;
  constexpr int kPanels = D / 64;
  constexpr uint32_t kPanelBytes = Sm::kPanelBytes;
  constexpr int kC8 = D / 8;
  const int it_begin = blockIdx.x * a.per_cta;
  const int it_end = min(a.items, it_begin + a.per_cta);

  if (warp == kQWarpTMA && lane == 0) {
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sm.kvfull[s], 1);
      mbar_init(&sm.kvempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.sfull[s], 1);
      mbar_init(&sm.pready[s], 8);
    }
    mbar_init(&sm.udone, 1);
    mbar_init(&sm.aready, kQCW);
    mbar_init(&sm.red, 1);
    mbar_init(&sm.stgfull[0], 1);
    mbar_init(&sm.stgfull[1], 1);
    mbar_init(&sm.stgempty[0], 1);
    mbar_init(&sm.stgempty[1], 1);
    fence_mbar_init();
  }
  if (warp == kQWarpMMA) tmem_alloc<512>(&sm.tmem_base);
  if constexpr (Sm::kTC) {
    // Sel^T, K-major SWIZZLE_128B: row n < 16 selects the rows of query n (r / R == n), row 16 + k the
    // rows of key slot k (r / R + r mod R == k); chunk (n, c8) holds tile rows r = 8 c8 .. 8 c8 + 7
    for (int t = threadIdx.x; t < Sm::kSelRows * 16; t += kQThreads) {
      const int n = t >> 4, c8 = t & 15;
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        uint32_t h[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int rr = 8 * c8 + 2 * e + u, g = rr >> a.lR, kk = rr & (a.R - 1);
          const bool on = n < 16 ? g == n : g + kk == n - 16;
          h[u] = on ? 0x3C00u : 0u;  // fp16 1.0
        }
        w[e] = h[0] | (h[1] << 16);
      }
      *reinterpret_cast<uint4*>(sm.sel + (c8 >> 3) * (Sm::kSelRows * 128) + n * 128 + (((c8 & 7) ^ (n & 7)) << 4)) =
          make_uint4(w[0], w[1], w[2], w[3]);
    }
    fence_proxy_async_smem();
  }
  for (int e = threadIdx.x; e < a.ring * Sm::kAP; e += kQThreads) {
    (&q_acc(sm, a, 0)[0][0])[e] = 0.f;
    (&q_acc(sm, a, 1)[0][0])[e] = 0.f;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = __shfl_sync(0xffffffffu, sm.tmem_base, 0);  // provably warp-uniform

  if (warp == kQWarpTMA) {
    // ------------------------------ TMA producer ------------------------------
    if (lane == 0) {
      uint32_t kc = 0;
      QItem it = it_begin < it_end ? q_item(a, it_begin) : QItem{};
      for (int item = it_begin; item < it_end; ++item, it = q_item_next(a, it)) {
        if (Sm::kRing && a.prod_stage) {
          // RING 37 row staging of this tile, off the compute warps' path: q / dO rows into buffer n & 1
          // and the tile's new k2 / v2 rows (its whole R + G - 1 window for the first tile of a (b,h)
          // run) into the key-position ring, one 1-D bulk copy per row, one expect_tx for the total
          const int n = item - it_begin, sb = n & 1;
          mbar_wait(&sm.stgempty[sb], (n >> 1) & 1);
          const Problem& p = a.p;
          const int P0 = p.np + it.i0;
          const bool fresh = item == it_begin || it.grp == 0;
          const int rh = (it.bh - a.fd_ng.div(it_begin)) & 1;
          const int klo = fresh ? P0 - a.R + 1 : P0, khi = P0 + a.G;  // [klo, khi)
          uint32_t bytes = 0;
          for (int g = 0; g < it.nq; ++g) {
            bulk_load(&sm.stgq[sb][g][0], a.q + p.qoff(it.b, it.i0 + g, it.h), 2 * D, &sm.stgfull[sb]);
            bulk_load(&sm.stgq[sb][a.G + g][0], a.dO + p.qoff(it.b, it.i0 + g, it.h), 2 * D, &sm.stgfull[sb]);
            bytes += 4 * D;
          }
          for (int kp = max(klo, p.k2lo); kp < min(khi, p.NK()); ++kp) {
            bulk_load(&sm.rk2[rh][kp % Sm::kKR][0], a.k2 + p.kvoff(it.b, kp, it.hk), 2 * D, &sm.stgfull[sb]);
            bulk_load(&sm.rv2[rh][kp % Sm::kKR][0], a.v2 + p.kvoff(it.b, kp, it.hk), 2 * D, &sm.stgfull[sb]);
            bytes += 4 * D;
          }
          mbar_expect_tx(&sm.stgfull[sb], bytes);
        }
        if (Sm::kTC && a.tma_stage) {
          // RING 38 row staging of this tile (the compute warps free buffer n & 1 at the top of tile
          // n - 1): four pitched-row TMA boxes (q, dO: G rows; k2, v2: R + G - 1 rows, the v2 box from a
          // row that is a multiple of 8 so it starts 128-byte aligned), completing on stgfull; k2 / v2
          // in real rows (virtual row kp is kp - k2lo)
          const int n = item - it_begin, sb = n & 1, nk = a.R + a.G - 1;
          mbar_wait(&sm.stgempty[sb], (n >> 1) & 1);
          const int kb = a.p.np + it.i0 - a.R + 1 - a.p.k2lo;
          mbar_expect_tx(&sm.stgfull[sb], uint32_t(2 * a.G + 2 * nk) * (D + 8) * 2);
          tma_load_4d(&sm.stg[sb][0][0], &tmQs, &sm.stgfull[sb], it.h * D, it.i0, it.b, 0);
          tma_load_4d(&sm.stg[sb][a.G][0], &tmdOs, &sm.stgfull[sb], it.h * D, it.i0, it.b, 0);
          tma_load_4d(&sm.stg[sb][2 * a.G][0], &tmK2s, &sm.stgfull[sb], it.hk * D, kb, it.b, 0);
          tma_load_4d(&sm.stg[sb][2 * a.G + ((nk + 7) & ~7)][0], &tmV2s, &sm.stgfull[sb], it.hk * D, kb, it.b, 0);
        }
        for (int c = 0; c < it.nch; ++c, ++kc) {
          const int s = kc % kStages;
          const uint32_t ph = (kc / kStages) & 1;
          const int row = it.jbeg + c * kQChunk;
          mbar_wait(&sm.kvempty[s], ph ^ 1);
          mbar_expect_tx(&sm.kvfull[s], 2 * Sm::kStageBytes);
          for (int pn = 0; pn < kPanels; ++pn) {
            tma_load_4d(sm.k[s] + pn * kPanelBytes, &tmK, &sm.kvfull[s], pn * 64, it.hk, row, it.b);
            tma_load_4d(sm.v[s] + pn * kPanelBytes, &tmV, &sm.kvfull[s], pn * 64, it.hk, row, it.b);
          }
        }
      }
    }
  } else if (warp == kQWarpMMA) {
    // ------------------------------ MMA issuer ------------------------------
    {  // whole warp; elected lane issues
      const uint32_t tW = tbase + kQW, tU = tbase + kQU, tS = tbase + kQS, tdP = tbase + kQdP;
      const uint32_t tAS = tbase + kQAS, tAdP = tbase + kQAdP;
      const uint32_t idesc_acc = idesc_f16(128, D, 0, 1);
      uint32_t kc = 0, gc = 0;
      int trn = 0;
      // S / dP MMAs of chunk c, half hh of item `jt` (K/V ring position kc0 + c)
      auto issue_s = [&](const QItem& jt, uint32_t kc0, int c, int hh) {
        const int s = (kc0 + c) % kStages;
        const int w = q_width(jt, c);
        const int nwh = min(32, w - 32 * hh);
        // one elected thread issues the group: descriptors advance by 64-bit adds in uniform registers
        const uint64_t dk = smem_desc_sw128(smem_u32(sm.k[s]) + hh * 32 * 128, 16, 1024);
        const uint64_t dv = smem_desc_sw128(smem_u32(sm.v[s]) + hh * 32 * 128, 16, 1024);
        const uint32_t idesc_s = idesc_f16(128, nwh > 0 ? nwh : 16, 0, 0);
        if (elect_one()) {
          if (nwh > 0) {
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint32_t off = (kk / 4) * kPanelBytes + (kk % 4) * 32;
              mma_ts(tS + 32 * hh, tAS + kk * 8, desc_adv(dk, off), idesc_s, kk > 0 ? 1u : 0u);
              mma_ts(tdP + 32 * hh, tAdP + kk * 8, desc_adv(dv, off), idesc_s, kk > 0 ? 1u : 0u);
            }
          }
          mma_commit(&sm.sfull[hh]);
        }
        __syncwarp();
      };
      // A operands of item `jt` formed (all compute warps bar.arrive), then its chunk-0 S / dP MMAs
      auto first_s = [&](const QItem& jt, uint32_t kc0) {
        named_bar_sync(4, kQNT + 32);
        tc_fence_after();
        mbar_wait(&sm.kvfull[kc0 % kStages], (kc0 / kStages) & 1);
        tc_fence_after();
        issue_s(jt, kc0, 0, 0);
        issue_s(jt, kc0, 0, 1);
      };
      QItem it = it_begin < it_end ? q_item(a, it_begin) : QItem{};
      if (it_begin < it_end) first_s(it, 0);
      for (int item = it_begin; item < it_end; ++item, it = q_item_next(a, it)) {
        const bool trm = lane == 0 && item - it_begin >= 100 && item - it_begin < 102;
        if constexpr (!Sm::kTC) {
          if (item != it_begin) first_s(it, kc);
        }
        SA_TRACE_AT(trm, 0, trn, (item - it_begin) << 16 | 10 << 8);
        // Issue order per chunk c and half hh (hh = column halves [32hh, 32hh+32) of a 64-row chunk):
        //   S_hh(0), dP_hh(0) ... then for each c: [P_hh(c) ready] W_hh(c), U_hh(c); S_hh(c+1), dP_hh(c+1)
        // so half a's next S overlaps half b's softmax (the tensor pipe is in-order, so S_hh(c+1)
        // overwriting the TMEM that held P_hh(c) / dS_hh(c) follows the W/U MMAs that read them).
        for (int c = 0; c < it.nch; ++c) {
          const int s = (kc + c) % kStages;
          const int w = q_width(it, c);
          const uint32_t kaddr = smem_u32(sm.k[s]), vaddr = smem_u32(sm.v[s]);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            // P/dS of this half ready: the 8 softmax warps of the half bar.arrive on named barrier
            // 2+hh; the MMA warp blocks in bar.sync (no polling)
            named_bar_sync(2 + hh, 32 * 8 + 32);
            tc_fence_after();
            SA_TRACE_AT(trm, 0, trn, (item - it_begin) << 16 | (11 + hh) << 8 | c);
            const int nwh = min(32, w - 32 * hh);
            const uint64_t dk = smem_desc_sw128(kaddr, kPanelBytes, 1024), dv = smem_desc_sw128(vaddr, kPanelBytes, 1024);
            if (elect_one()) {
              for (int k2i = 0; k2i < nwh / 16; ++k2i) {
                const uint32_t acc = (c > 0 || hh > 0 || k2i > 0) ? 1u : 0u;
                const uint32_t roff = (32 * hh + 16 * k2i) * 128;
                const uint32_t pc = 32 * hh + 16 * k2i;  // packed P/dS of columns 32hh+16k2i.. (see the softmax)
                mma_ts(tW, tdP + pc, desc_adv(dk, roff), idesc_acc, acc);
                mma_ts(tU, tS + pc, desc_adv(dv, roff), idesc_acc, acc);
              }
            }
            __syncwarp();
            if (c + 1 < it.nch) {
              if (hh == 0) {
                mbar_wait(&sm.kvfull[(kc + c + 1) % kStages], ((kc + c + 1) / kStages) & 1);
                tc_fence_after();
              }
              issue_s(it, kc, c + 1, hh);
            }
          }
          mma_commit_w(&sm.kvempty[s]);
        }
        mma_commit_w(&sm.udone);
        kc += it.nch;
        ++gc;
        if constexpr (Sm::kTC) {
          // the next tile's chunk-0 S / dP MMAs first (its A operands are formed before this tile's
          // epilogue), then the epilogue's three reductions Y^T = X^T Sel^T (q_epilogue_tc)
          if (item + 1 < it_end) first_s(q_item_next(a, it), kc);
          const uint64_t dx = smem_desc_sw128(smem_u32(sm.xr), 128 * 128, 1024);
#pragma unroll 1
          for (int k = 0; k < 3; ++k) {
            named_bar_sync(5, kQNT + 32);  // X of product k in shared memory
            tc_fence_after();
            const uint32_t nsel = k == 0 ? 16u : 32u;
            const uint64_t ds = smem_desc_sw128(smem_u32(sm.sel) + (k == 0 ? 0u : 16u * 128u), 16, 1024);
            const uint32_t idesc_r = idesc_f16(128, nsel, 1, 0);
            if (elect_one()) {
#pragma unroll
              for (int kk = 0; kk < 8; ++kk)
                mma_ss(tW + 32 * k, desc_adv(dx, kk * 16 * 128),
                       desc_adv(ds, (kk / 4) * (Sm::kSelRows * 128) + (kk % 4) * 32), idesc_r, kk > 0 ? 1u : 0u);
              mma_commit(&sm.red);
            }
            __syncwarp();
          }
        }
      }
    }
  } else if (warp < kQCW) {
    // ------------------------------ softmax-gradient + epilogue ------------------------------
    const int qd = warp & 3, half = (warp >> 2) & 1, sub = warp >> 3;
    const int r = qd * 32 + lane;
    const int tid256 = threadIdx.x;  // 0 .. kQNT-1
    const uint32_t lane_off = uint32_t(qd * 32) << 16;
    const uint32_t tW = tbase + kQW + lane_off, tU = tbase + kQU + lane_off;
    const uint32_t tS = tbase + kQS + lane_off, tdP = tbase + kQdP + lane_off;
    const uint32_t tAS = tbase + kQAS + lane_off, tAdP = tbase + kQAdP + lane_off;
    const Problem& p = a.p;
    const float sl2 = p.scale * kLog2e;
    const int bh_begin = a.fd_ng.div(it_begin);  // (b,h) of the CTA's first tile
    // stage tile `item`'s rows into buffer `buf` (cp.async, one group per call)
    auto stage = [&](const QItem& it, int item, int buf) {
      if (!STAGED) {  // no shared-memory staging (large R): pull the next tile's rows into L2 instead
        const int P0 = p.np + it.i0;
        const int nk = a.R + a.G - 1;
        constexpr int kLines = D * 2 / 128;  // 128-byte lines per fp16 row
        for (int task = tid256; task < (2 * a.G + 2 * nk) * kLines; task += kQNT) {
          const int row = task / kLines, ln128 = task % kLines;
          const __half* src = nullptr;
          if (row < a.G) {
            if (row < it.nq) src = a.q + p.qoff(it.b, it.i0 + row, it.h);
          } else if (row < 2 * a.G) {
            if (row - a.G < it.nq) src = a.dO + p.qoff(it.b, it.i0 + row - a.G, it.h);
          } else {
            const int rr = row - 2 * a.G;
            const int kp = P0 - a.R + 1 + (rr < nk ? rr : rr - nk);
            if (kp >= p.k2lo && kp < p.NK()) src = (rr < nk ? a.k2 : a.v2) + p.kvoff(it.b, kp, it.hk);
          }
          if (src) asm volatile("prefetch.global.L2 [%0];" ::"l"(src + 64 * ln128));
        }
        return;
      }
      if constexpr (Sm::kRing) {
        const int P0 = p.np + it.i0;
        const bool fresh = item == it_begin || it.grp == 0;  // first item of a (b,h) run: whole window
        const int rh = (it.bh - bh_begin) & 1;
        const int klo = fresh ? P0 - a.R + 1 : P0;
        const int nkn = P0 + a.G - klo;  // key rows to stage
        const int nrows = 2 * a.G + 2 * nkn;
        // producer-staged rows: signal that buffer buf (and this tile's ring slots) may be written
        if (a.prod_stage) {
          if (tid256 == 0) mbar_arrive(&sm.stgempty[buf]);
        } else
        for (int task = tid256; task < nrows * kC8; task += kQNT) {
          const int row = task / kC8, c8 = task % kC8;
          const __half* src = nullptr;
          __half* dst;
          if (row < 2 * a.G) {
            const int gq = row < a.G ? row : row - a.G;
            if (gq < it.nq) src = (row < a.G ? a.q : a.dO) + p.qoff(it.b, it.i0 + gq, it.h);
            dst = &sm.stgq[buf][row][0];
          } else {
            const int rr = row - 2 * a.G;
            const bool isv = rr >= nkn;
            const int kp = klo + (isv ? rr - nkn : rr);
            if (kp >= p.k2lo && kp < p.NK()) src = (isv ? a.v2 : a.k2) + p.kvoff(it.b, kp, it.hk);
            dst = isv ? &sm.rv2[rh][kp >= 0 ? kp % Sm::kKR : 0][0] : &sm.rk2[rh][kp >= 0 ? kp % Sm::kKR : 0][0];
          }
          if (src) cp_async16(dst + 8 * c8, src + 8 * c8);
        }
        if (tid256 < 2 * it.nq) {
          const int g = tid256 < it.nq ? tid256 : tid256 - it.nq;
          const int64_t x = (int64_t(it.b) * p.H + it.h) * p.N + it.i0 + g;
          if (tid256 < it.nq)
            cp_async4(&sm.slse[buf][g], a.lse + x);
          else
            cp_async4(&sm.sdl[buf][g], a.delta + x);
        }
        cp_async_commit();
        return;
      }
      const int P0 = p.np + it.i0;
      const int nk = a.R + a.G - 1;
      const int nrows = 2 * a.G + 2 * nk;
      if (Sm::kTC && a.tma_stage) {
        // four pitched-row TMA boxes (q, dO: G rows; k2, v2: nk rows, the v2 box from a row that is a
        // multiple of 8 so it starts 128-byte aligned), completing on stgfull[buf]; k2 / v2 in real
        // rows (virtual row kp is kp - k2lo); lse / delta by cp.async below
        // issued by the TMA producer warp once buffer buf is free: signal it (the compute warps are
        // past the previous tile's end barrier, so nobody reads this buffer any more)
        if (tid256 == 0) mbar_arrive(&sm.stgempty[buf]);
      } else
      for (int task = tid256; task < nrows * kC8; task += kQNT) {
        const int row = task / kC8, c8 = task % kC8;
        const __half* src = nullptr;
        if (row < a.G) {
          if (row < it.nq) src = a.q + p.qoff(it.b, it.i0 + row, it.h);
        } else if (row < 2 * a.G) {
          if (row - a.G < it.nq) src = a.dO + p.qoff(it.b, it.i0 + row - a.G, it.h);
        } else {
          const int rr = row - 2 * a.G;
          const int kp = P0 - a.R + 1 + (rr < nk ? rr : rr - nk);
          if (kp >= p.k2lo && kp < p.NK()) src = (rr < nk ? a.k2 : a.v2) + p.kvoff(it.b, kp, it.hk);
        }
        if (src) cp_async16(&sm.stg[buf][row][8 * c8], src + 8 * c8);
      }
      if (tid256 < 2 * it.nq) {
        const int g = tid256 < it.nq ? tid256 : tid256 - it.nq;
        const int64_t x = (int64_t(it.b) * p.H + it.h) * p.N + it.i0 + g;
        if (tid256 < it.nq)
          cp_async4(&sm.slse[buf][g], a.lse + x);
        else
          cp_async4(&sm.sdl[buf][g], a.delta + x);
      }
      cp_async_commit();
    };
    uint32_t kc = 0, gc = 0, nred = 0;
    int PS = 0, flush_lo = 0;
    int trn = 0;
    // ---- row operands of tile `fitem` (fp16, unscaled): half 0 -> A_S = q o k2 [det: k2 x q],
    //      half 1 -> A_dP = dO o v2, from staging buffer `bf`.  Formed for tile t+1 right after the
    //      chunk loop of tile t (the A regions are free then), so the S/dP MMAs of t+1 overlap the
    //      epilogue of t. ----
    auto form_A = [&](const QItem& fi, int fitem, int bf) {
      const int fP0 = p.np + fi.i0;
      const int g = r >> a.lR, kk = r & (a.R - 1);
      const int fkpos = fP0 + g - a.R + 1 + kk;
      const bool fvalid = r < a.G * a.R && g < fi.nq && fkpos >= p.k2lo;
      QRows fr{};
      if (fvalid) {
        const int nk = a.R + a.G - 1;
        if constexpr (Sm::kRing) {
          const int rh = (fi.bh - bh_begin) & 1;
          fr.q = &sm.stgq[bf][g][0];
          fr.dO = &sm.stgq[bf][a.G + g][0];
          fr.k2 = &sm.rk2[rh][fkpos % Sm::kKR][0];
          fr.v2 = &sm.rv2[rh][fkpos % Sm::kKR][0];
        } else if (STAGED) {
          fr.q = &sm.stg[bf][g][0];
          fr.dO = &sm.stg[bf][a.G + g][0];
          fr.k2 = &sm.stg[bf][2 * a.G + g + kk][0];
          fr.v2 = &sm.stg[bf][2 * a.G + ((Sm::kTC && a.tma_stage) ? ((nk + 7) & ~7) : nk) + g + kk][0];
        } else {
          fr.q = a.q + p.qoff(fi.b, fi.i0 + g, fi.h);
          fr.dO = a.dO + p.qoff(fi.b, fi.i0 + g, fi.h);
          fr.k2 = a.k2 + p.kvoff(fi.b, fkpos, fi.hk);
          fr.v2 = a.v2 + p.kvoff(fi.b, fkpos, fi.hk);
        }
      }
      const bool tr = (threadIdx.x & 127) == 0 && threadIdx.x < 256 && fitem - it_begin >= 100 && fitem - it_begin < 102;
      const int treg = 1 + half;
        if (DET && half == 0) {
          // A_S = k2 x q chunkwise; sub-warp `sub` writes columns [D/2 sub, D/2 sub + D/2) and computes
          // the 3-chunks that overlap them (the chunk straddling D/2 is computed by both)
          constexpr int DH = D / 2;
          constexpr int D3 = (D / 3) * 3;
          uint32_t pk[DH / 2];
  #pragma unroll
          for (int t = 0; t < DH / 2; ++t) pk[t] = 0u;
          if (fvalid) {
            if (sub == 0)
              det_half_operand<D, 0>(fr.q, fr.k2, pk);
            else
              det_half_operand<D, 1>(fr.q, fr.k2, pk);
          }
          if constexpr (DH == 64)
            tmem_st32(tAS + (DH / 2) * sub, *reinterpret_cast<const uint32_t(*)[32]>(pk));
          else
            tmem_st16(tAS + (DH / 2) * sub, pk);
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          named_bar_arrive(4, kQNT + 32);
        } else {
          // trilinear (A_S = q o k2) or A_dP = dO o v2: sub-warp `sub` forms columns [D/2 sub, D/2 sub + D/2)
          constexpr int DH = D / 2;
          uint32_t pk[DH / 2];
  #pragma unroll
          for (int t = 0; t < DH / 2; ++t) pk[t] = 0u;
          if (fvalid) {
            const __half* x = (half == 0 ? fr.q : fr.dO) + DH * sub;
            const __half* y = (half == 0 ? fr.k2 : fr.v2) + DH * sub;
  #pragma unroll
            for (int t = 0; t < DH / 8; ++t) {
              const uint4 xv = *reinterpret_cast<const uint4*>(x + 8 * t);
              const uint4 yv = *reinterpret_cast<const uint4*>(y + 8 * t);
              pk[4 * t + 0] = hmul2_u32(xv.x, yv.x);
              pk[4 * t + 1] = hmul2_u32(xv.y, yv.y);
              pk[4 * t + 2] = hmul2_u32(xv.z, yv.z);
              pk[4 * t + 3] = hmul2_u32(xv.w, yv.w);
            }
          }
          SA_TRACE_AT(tr, treg, trn, (fitem - it_begin) << 16 | 9 << 8);
          const uint32_t ta = (half == 0 ? tAS : tAdP) + (DH / 2) * sub;
          if constexpr (DH == 64)
            tmem_st32(ta, pk);
          else
            tmem_st16(ta, pk);
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          named_bar_arrive(4, kQNT + 32);
          SA_TRACE_AT(tr, treg, trn, (fitem - it_begin) << 16 | 2 << 8);
        }
    };
    // RING 37: fp32 copies (q x s, dO) of the staged q / dO rows of buffer `bf` for the epilogue
    auto cvt_qf = [&](int bf) {
      if constexpr (Sm::kRing) {
        for (int idx = tid256; idx < 2 * a.G * D; idx += kQNT) {
          const int row = idx / D, col = idx - row * D;
          sm.stgqf[bf][row][col] = __half2float(sm.stgq[bf][row][col]) * (row < a.G ? p.scale : 1.f);
        }
      }
    };
    QItem itc = it_begin < it_end ? q_item(a, it_begin) : QItem{};  // tile of the current iteration
    if (it_begin < it_end) {
      stage(itc, it_begin, 0);
      if (STAGED) {
        cp_async_wait<0>();
        if ((Sm::kTC && a.tma_stage) || (Sm::kRing && a.prod_stage)) mbar_wait(&sm.stgfull[0], 0);
        named_bar_sync(1, kQNT);
      }
      cvt_qf(0);
      form_A(itc, it_begin, 0);
    }
    for (int item = it_begin; item < it_end; ++item) {
      const QItem it = itc;
      const QItem itn = q_item_next(a, it);  // the next tile (no division)
      const bool tr = (threadIdx.x & 127) == 0 && threadIdx.x < 256 && item - it_begin >= 100 && item - it_begin < 102;
      const int treg = 1 + half;
      SA_TRACE_AT(tr, treg, trn, (item - it_begin) << 16 | 1 << 8);
      const int buf = STAGED ? int(gc & 1) : 0;
      // this tile's rows were staged (and waited for) before its A operands were formed; prefetch the next
      if (item + 1 < it_end) stage(itn, item + 1, STAGED ? (buf ^ 1) : 0);
      SA_TRACE_AT(tr, treg, trn, (item - it_begin) << 16 | 8 << 8);
      const bool first_in_sub = item == it_begin || it.grp == 0;
      const bool last_in_sub = item == it_end - 1 || it.grp == a.ngroups - 1;
      const int P0 = p.np + it.i0;
      if (first_in_sub) {
        PS = P0;
        flush_lo = P0 - a.R + 1;
      }
      const int g = r >> a.lR, kk = r & (a.R - 1);
      const bool row_in = r < a.G * a.R && g < it.nq;
      const int pos = P0 + g;
      const int kpos = pos - a.R + 1 + kk;
      const bool valid = row_in && kpos >= p.k2lo && kk >= a.R - a.Rt;
      float lse_l2 = 0.f, dl = 0.f;
      QRows rw{};
      if (row_in) {
        if (STAGED) {
          lse_l2 = sm.slse[buf][g] * kLog2e;
          dl = sm.sdl[buf][g];
        } else {
          const int64_t ri = (int64_t(it.b) * p.H + it.h) * p.N + it.i0 + g;
          lse_l2 = a.lse[ri] * kLog2e;
          dl = a.delta[ri];
        }
      }
      if (valid) {
        const int nk = a.R + a.G - 1;
        if constexpr (Sm::kRing) {
          const int rh = (it.bh - bh_begin) & 1;
          rw.q = &sm.stgq[buf][g][0];
          rw.dO = &sm.stgq[buf][a.G + g][0];
          rw.qf = &sm.stgqf[buf][g][0];
          rw.dOf = &sm.stgqf[buf][a.G + g][0];
          rw.k2 = &sm.rk2[rh][kpos % Sm::kKR][0];
          rw.v2 = &sm.rv2[rh][kpos % Sm::kKR][0];
        } else if (STAGED) {
          rw.q = &sm.stg[buf][g][0];
          rw.dO = &sm.stg[buf][a.G + g][0];
          rw.k2 = &sm.stg[buf][2 * a.G + g + kk][0];
          rw.v2 = &sm.stg[buf][2 * a.G + ((Sm::kTC && a.tma_stage) ? ((nk + 7) & ~7) : nk) + g + kk][0];
        } else {
          rw.q = a.q + p.qoff(it.b, it.i0 + g, it.h);
          rw.dO = a.dO + p.qoff(it.b, it.i0 + g, it.h);
          rw.k2 = a.k2 + p.kvoff(it.b, kpos, it.hk);
          rw.v2 = a.v2 + p.kvoff(it.b, kpos, it.hk);
        }
      }
      // ---- chunks: P = exp(S - lse), dS = P (dP - delta), this half's 32 columns ----
      const int jlo = max(0, pos - p.w1 + 1);
      for (int c = 0; c < it.nch; ++c) {
        const int w = q_width(it, c);
        const int cb = 32 * half + 16 * sub;  // this warp's 16 columns of the 64-column chunk
        const int nw = max(0, min(16, w - cb));
        mbar_wait(&sm.sfull[half], (kc + c) & 1);
        tc_fence_after();
        SA_TRACE_AT(tr, treg, trn, (item - it_begin) << 16 | 3 << 8 | c);
        if (nw > 0) {  // chunk widths are multiples of 16: nw is 0 or 16 (warp-uniform)
          uint32_t su[16], du[16];
          tmem_ld16(tS + cb, su);
          tmem_ld16(tdP + cb, du);
          tmem_ld_wait();
          const int jc0 = it.jbeg + c * kQChunk + cb;
          int lo_c = jlo - jc0, hi_c = min(pos - jc0, nw - 1);
          if (!valid) {
            lo_c = 1;
            hi_c = 0;
          }
          const bool need_mask = lo_c > 0 || hi_c < 15;
          uint32_t pp[8], pd[8];
          if (!__any_sync(0xffffffffu, need_mask)) {
            const float2 vs = make_float2(sl2, sl2), vl = make_float2(-lse_l2, -lse_l2), vd = make_float2(-dl, -dl);
#pragma unroll
            for (int t = 0; t < 8; ++t) {
              const float2 x = ffma2(make_float2(__uint_as_float(su[2 * t]), __uint_as_float(su[2 * t + 1])), vs, vl);
              const float2 pv = make_float2(ex2(x.x), ex2(x.y));
              pp[t] = pack_f16x2(pv);
              pd[t] = pack_f16x2(
                  fmul2(pv, fadd2(make_float2(__uint_as_float(du[2 * t]), __uint_as_float(du[2 * t + 1])), vd)));
            }
          } else {
#pragma unroll
            for (int t = 0; t < 8; ++t) {
              float p0 = ex2(fmaf(__uint_as_float(su[2 * t]), sl2, -lse_l2));
              float p1 = ex2(fmaf(__uint_as_float(su[2 * t + 1]), sl2, -lse_l2));
              p0 = (2 * t >= lo_c && 2 * t <= hi_c) ? p0 : 0.f;
              p1 = (2 * t + 1 >= lo_c && 2 * t + 1 <= hi_c) ? p1 : 0.f;
              pp[t] = pack_f16x2(p0, p1);
              pd[t] = pack_f16x2(p0 * (__uint_as_float(du[2 * t]) - dl), p1 * (__uint_as_float(du[2 * t + 1]) - dl));
            }
          }
          // P / dS of columns [cb, cb+16) overwrite the first 8 columns of this warp's own S / dP
          // range (the other sub-warp may still be reading its range)
          tmem_st8(tS + cb, pp);
          tmem_st8(tdP + cb, pd);
          tmem_st_wait();
        }
        tc_fence_before();
        __syncwarp();
        named_bar_arrive(2 + half, 32 * 8 + 32);
        SA_TRACE_AT(tr, treg, trn, (item - it_begin) << 16 | 4 << 8 | c);
      }
      // ---- A operands of the next tile (its S/dP MMAs then run during this tile's epilogue) ----
      if (item + 1 < it_end) {
        if (STAGED) cp_async_wait<0>();
        if ((Sm::kTC && a.tma_stage) || (Sm::kRing && a.prod_stage))
          mbar_wait(&sm.stgfull[buf ^ 1], ((gc + 1) >> 1) & 1);
        named_bar_sync(1, kQNT);  // every warp is past its last S/dP wait: the A regions are free
        cvt_qf(buf ^ 1);
        form_A(itn, item + 1, STAGED ? (buf ^ 1) : 0);
      }
      // ---- epilogue ----
      mbar_wait(&sm.udone, gc & 1);
      tc_fence_after();
      SA_TRACE_AT(tr, treg, trn, (item - it_begin) << 16 | 5 << 8);
      if constexpr (Sm::kG1) {
        const int sbase = a.fd_ring.mod(p.np + it.i0 - a.R + 1 + a.ring);
#pragma unroll 1
        for (int c0 = 0; c0 < D; c0 += 32)
          q_epilogue_g1<D, RING, STAGED>(sm, a, c0, half, sub, r, valid, rw, tW, tU, sbase);
        named_bar_sync(1, kQNT);
        if (tid256 < D && it.nq > 0) {
          const float y = (sm.dq4[0][tid256] + sm.dq4[1][tid256]) + (sm.dq4[2][tid256] + sm.dq4[3][tid256]);
          const int64_t off = p.qoff(it.b, it.i0, it.h) + tid256;
          if (a.out_f32)
            reinterpret_cast<float*>(a.dq)[off] = y;
          else
            reinterpret_cast<__nv_bfloat16*>(a.dq)[off] = __float2bfloat16_rn(y);
        }
      } else if constexpr (Sm::kRot && DET) {
        const int sbase = a.fd_ring.mod(p.np + it.i0 - a.R + 1 + a.ring);
        if constexpr (Sm::kRing)
          q_epilogue_rot_det4<D, RING, STAGED>(sm, a, it, half, sub, r, valid, rw, tW, tU, sbase);
        else
          q_epilogue_rot_det<D, RING, STAGED>(sm, a, it, half, sub, r, valid, rw, tW, tU, sbase);
      } else if constexpr (Sm::kRot) {
        const int sbase = a.fd_ring.mod(p.np + it.i0 - a.R + 1 + a.ring);
        q_epilogue_rot<D, RING, STAGED>(sm, a, it, half, sub, r, valid, rw, tW, tU, sbase, tr, treg, trn,
                                        item - it_begin);
        if (a.R == 64 && tid256 < 2 * D) {  // dq = the two lane quarters' partials of each query
          const int gq = tid256 / D, d = tid256 % D;
          if (gq < it.nq) {
            const float y = sm.dq4[2 * gq][d] + sm.dq4[2 * gq + 1][d];
            const int64_t off = p.qoff(it.b, it.i0 + gq, it.h) + d;
            if (a.out_f32)
              reinterpret_cast<float*>(a.dq)[off] = y;
            else
              reinterpret_cast<__nv_bfloat16*>(a.dq)[off] = __float2bfloat16_rn(y);
          }
        }
      } else if constexpr (Sm::kTC) {
        const int sbase = a.fd_ring.mod(p.np + it.i0 - a.R + 1 + a.ring);
        q_epilogue_tc<D, RING, STAGED>(sm, a, it, half, sub, r, valid, rw, tW, tU, sbase, nred, tr, treg, trn,
                                       item - it_begin);
      } else if (DET && (a.R == 32 || a.R == 64)) {
        const int sbase = a.fd_ring.mod(p.np + it.i0 - a.R + 1 + a.ring);
#pragma unroll 1
        for (int c0 = 0; c0 < D; c0 += 24)
          q_epilogue_pass_det<D, RING, STAGED>(sm, a, it, c0, half, sub, r, valid, rw, tW, tU, tid256, sbase);
      } else if (DET) {
#pragma unroll 1
        for (int c0 = 0; c0 + 24 <= D; c0 += 24)
          q_epilogue_pass<D, RING, STAGED, 24, DET>(sm, a, it, c0, half, r, valid, rw, tW, tU, tid256, sub == 0);
        if constexpr (D % 24 != 0)
          q_epilogue_pass<D, RING, STAGED, D % 24, DET>(sm, a, it, D - D % 24, half, r, valid, rw, tW, tU, tid256,
                                                        sub == 0);
      } else if (a.R == 32 || a.R == 64) {
#pragma unroll 1
        const int sbase = a.fd_ring.mod(p.np + it.i0 - a.R + 1 + a.ring);
        for (int c0 = 0; c0 < D; c0 += 32) {
          q_epilogue_pass32<D, RING, STAGED>(sm, a, it, c0, half, sub, r, valid, rw, tW, tU, tid256, sbase);
          SA_TRACE_AT(tr, treg, trn, (item - it_begin) << 16 | 6 << 8 | (c0 / 32));
        }
      } else if (a.R >= 2 && a.R < 32) {
        const int sbase = a.fd_ring.mod(p.np + it.i0 - a.R + 1 + a.ring);
#pragma unroll 1
        for (int c0 = 0; c0 < D; c0 += 32) {
          switch (a.R) {
            case 2: q_epilogue_pass_small<D, RING, STAGED, 2>(sm, a, it, c0, half, sub, r, valid, rw, tW, tU, tid256, sbase); break;
            case 4: q_epilogue_pass_small<D, RING, STAGED, 4>(sm, a, it, c0, half, sub, r, valid, rw, tW, tU, tid256, sbase); break;
            case 8: q_epilogue_pass_small<D, RING, STAGED, 8>(sm, a, it, c0, half, sub, r, valid, rw, tW, tU, tid256, sbase); break;
            default: q_epilogue_pass_small<D, RING, STAGED, 16>(sm, a, it, c0, half, sub, r, valid, rw, tW, tU, tid256, sbase); break;
          }
          SA_TRACE_AT(tr, treg, trn, (item - it_begin) << 16 | 6 << 8 | (c0 / 32));
        }
      } else {
#pragma unroll 1
        for (int c0 = 0; c0 < D; c0 += 16)
          q_epilogue_pass<D, RING, STAGED, 16, DET>(sm, a, it, c0, half, r, valid, rw, tW, tU, tid256, sub == 0);
      }
      tc_fence_before();
      // ---- flush ring rows that no later tile of this sub-range touches ----
      const int PE = P0 + it.nq;
      const int flush_hi = last_in_sub ? PE - 1 : P0 + a.G - a.R;  // inclusive
      const bool end_open = last_in_sub && PE < p.np + p.N;
      const bool start_open = PS > p.np;
      const int nrows = flush_hi - flush_lo + 1;
      const int fbase = a.fd_ring.mod(flush_lo + a.ring);
      // four columns per task: float4 ring traffic, 8- / 16-byte global stores
      constexpr int kD4 = D / 4;
      for (int idx = tid256; idx < nrows * kD4; idx += kQNT) {
        const int kp = flush_lo + idx / kD4, d = 4 * (idx % kD4);
        if (kp < p.k2lo || kp >= p.NK()) continue;
        int slot = fbase + idx / kD4;
        if (slot >= a.ring) slot -= a.ring;
        float4* pk = reinterpret_cast<float4*>(&q_acc(sm, a, 0)[slot][d]);
        float4* pv = reinterpret_cast<float4*>(&q_acc(sm, a, 1)[slot][d]);
        const float4 vk = *pk, vv = *pv;
        *pk = make_float4(0.f, 0.f, 0.f, 0.f);
        *pv = make_float4(0.f, 0.f, 0.f, 0.f);
        if (start_open && kp < PS) {
          float* bnd = a.band + ((size_t(blockIdx.x) * 2 + 0) * 2) * (a.R - 1) * D;
          const int rr = kp - (PS - a.R + 1);
          *reinterpret_cast<float4*>(bnd + size_t(rr) * D + d) = vk;
          *reinterpret_cast<float4*>(bnd + size_t(a.R - 1 + rr) * D + d) = vv;
        } else if (end_open && kp + a.R - 1 >= PE) {
          float* bnd = a.band + ((size_t(blockIdx.x) * 2 + 1) * 2) * (a.R - 1) * D;
          const int rr = kp - (PE - a.R + 1);
          *reinterpret_cast<float4*>(bnd + size_t(rr) * D + d) = vk;
          *reinterpret_cast<float4*>(bnd + size_t(a.R - 1 + rr) * D + d) = vv;
        } else {
          const int64_t off = p.koff(it.b, kp, it.h) + d;
          if (a.out_f32) {
            *reinterpret_cast<float4*>(reinterpret_cast<float*>(a.dk2) + off) = vk;
            *reinterpret_cast<float4*>(reinterpret_cast<float*>(a.dv2) + off) = vv;
          } else {
            const __nv_bfloat162 k01 = __floats2bfloat162_rn(vk.x, vk.y), k23 = __floats2bfloat162_rn(vk.z, vk.w);
            const __nv_bfloat162 v01 = __floats2bfloat162_rn(vv.x, vv.y), v23 = __floats2bfloat162_rn(vv.z, vv.w);
            *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(a.dk2) + off) =
                make_uint2(*reinterpret_cast<const uint32_t*>(&k01), *reinterpret_cast<const uint32_t*>(&k23));
            *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(a.dv2) + off) =
                make_uint2(*reinterpret_cast<const uint32_t*>(&v01), *reinterpret_cast<const uint32_t*>(&v23));
          }
        }
      }
      flush_lo = flush_hi + 1;
      SA_TRACE_AT(tr, treg, trn, (item - it_begin) << 16 | 14 << 8);
      named_bar_sync(1, kQNT);
      SA_TRACE_AT(tr, treg, trn, (item - it_begin) << 16 | 7 << 8);
      kc += it.nch;
      ++gc;
      itc = itn;
    }
  }

  __syncthreads();
  tc_fence_after();
  if (warp == kQWarpMMA) tmem_free<512>(tbase);
}

// Band fold: key rows shared by two consecutive CTA ranges get both partial sums; prefix rows no
// query touches are zeroed.  One block per boundary (CTA c >= 1), plus a zeroing grid-stride.
template <typename TOut>
__global__ void __launch_bounds__(256) fold_kernel(BwdQArgs a, int grid_q) {
  const Problem& p = a.p;
  const int D = p.D, Rm1 = a.R - 1;
  const int c = blockIdx.x + 1;
  if (c < grid_q) {
    const int item = c * a.per_cta;
    if (item < a.items && (item % a.ngroups) != 0 && Rm1 > 0) {
      const int bh = item / a.ngroups, b = bh / p.H, h = bh % p.H;
      const int PS = p.np + (item % a.ngroups) * a.G;
      const float* left = a.band + ((size_t(c - 1) * 2 + 1) * 2) * Rm1 * D;
      const float* right = a.band + ((size_t(c) * 2 + 0) * 2) * Rm1 * D;
      for (int idx = threadIdx.x; idx < Rm1 * D; idx += blockDim.x) {
        const int rr = idx / D, d = idx % D;
        const int kp = PS - a.R + 1 + rr;
        if (kp < p.k2lo) continue;
        const int64_t off = p.koff(b, kp, h) + d;
        st_f(reinterpret_cast<TOut*>(a.dk2) + off, left[idx] + right[idx]);
        st_f(reinterpret_cast<TOut*>(a.dv2) + off, left[size_t(Rm1) * D + idx] + right[size_t(Rm1) * D + idx]);
      }
    }
  }
  // prefix rows [k2lo, np - R + 1) are outside every query's window: zero
  const int nz = p.np - a.R + 1 - p.k2lo;
  if (nz > 0) {
    const int64_t total = int64_t(p.B) * p.H * nz * D;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
      const int d = e % D;
      const int64_t t = e / D;
      const int kp = p.k2lo + int(t % nz), bh = t / nz, b = bh / p.H, h = bh % p.H;
      const int64_t off = p.koff(b, kp, h) + d;
      st_f(reinterpret_cast<TOut*>(a.dk2) + off, 0.f);
      st_f(reinterpret_cast<TOut*>(a.dv2) + off, 0.f);
    }
  }
}

// ==========================================================================================
// bwd_kv: dK, dV (K/V-stationary).  TMEM lanes = key rows j of the CTA's 128-row block.
// The CTA's K and V rows sit in TMEM as fp16 A operands for the whole launch, so every MMA is a
// TS-MMA (SMEM reads <= 64 B/clk, leaving SMEM bandwidth for the A-tile formers; an SS-MMA at
// N=64 saturates SMEM at 128 B/clk, tools/micro/mma_rate.cu).  The row tile's 128 columns are
// processed in quarters of 32 (double-buffered S^T/dP^T in TMEM), issued as
//   S^T,dP^T(Q) | S^T,dP^T(Q+1) | [P(Q) ready] dV,dK += quarter Q ; S^T,dP^T(Q+2) | ...
// so the softmax-gradient of quarter Q (warpgroup Q%2) overlaps the MMAs of quarter Q+1.
// A tiles (A_S = q o k2 [det k2 x q], A_dP = dO o v2, fp16, unscaled: s is folded into the
// exponent and the dK epilogue) are formed into SMEM by the former warps from an fp16 staging
// ring filled with cp.async one tile ahead.
// ==========================================================================================
constexpr int kKVFW = 8;                      // A-tile former warps
constexpr int kKVF0 = 0;                      // first former warp (low ids: issue priority)
constexpr int kKVS0 = kKVFW;                  // first softmax-gradient warp (8 warps)
constexpr int kKVWarpMMA = 8 + kKVFW;
constexpr int kKVWarpStg = kKVWarpMMA + 1;  // row stager: staged determinant kernels only
constexpr int kKVThreads = 32 * (kKVWarpMMA + 1);  // warps 0-7 formers, 8-15 softmax-gradient, MMA
constexpr int kKVThreadsStg = kKVThreads + 32;     // ... plus the stager warp
// TMEM columns: K, V operands (D/2 packed cols each), dV, dK accumulators, 2 x (S^T, dP^T) quarters
constexpr uint32_t kKK = 0, kKV = 64, kKdV = 128, kKdK = 256, kKSD = 384;
constexpr int kKVRing = 40;   // staged K2/V2 rows (>= R + 2G)
constexpr int kKVGmax = 16;   // staged queries per tile

struct BwdKVArgs {
  Problem p;  // after the swap: w1 = long window (this kernel's keys), w2 = R
  const __half *q, *k2, *v2, *dO;  // fp16 copies
  const __half *k, *v;             // fp16 copies of this kernel's stationary keys
  const float *lse, *delta;
  void *dk, *dv;
  int out_f32, R, lR, G, ring, Rt;  // R, Rt as in BwdQArgs
  FastDiv fd_ring;
};

template <int D>
struct KVSmem {
  static constexpr int kPanelBytes = 128 * 128;  // 128 rows x 64 fp16
  static constexpr int kTileBytes = 128 * D * 2;
  alignas(1024) uint8_t as[2][kTileBytes];
  alignas(1024) uint8_t adp[2][kTileBytes];
  alignas(16) __half rk2[kKVRing][D];
  alignas(16) __half rv2[kKVRing][D];
  alignas(16) __half sq[2][kKVGmax][D];
  alignas(16) __half sdo[2][kKVGmax][D];
  float slse[2][kKVGmax], sdl[2][kKVGmax];
  float2 rinfo[2][128];  // (lse * log2e or +inf for invalid rows, delta)
  // rready/rfree: direct former -> softmax handoff of rinfo[buf] (every former / softmax thread
  // arrives), so the row info does not rely on ordering carried through the MMA warp's commits
  uint64_t kvtm, aready[2], afree[2], sfull[2], pready[2], rready[2], rfree[2], done;
  uint64_t stgfull[2], stgempty[2];  // stager warp <-> formers: tile rows landed / buffer free
  uint32_t tmem_base;
};

// 16-byte chunk (row, c8) of a K-major SWIZZLE_128B tile of 128 rows: panel c8/8, chunk c8%8
// XOR (row%8) -- the layout TMA writes and the UMMA descriptor reads.
__device__ __forceinline__ uint32_t sw128_off(int row, int c8) {
  return uint32_t((c8 >> 3) * (128 * 128) + row * 128 + (((c8 & 7) ^ (row & 7)) << 4));
}


template <int D, bool DET, bool STAGED>
__global__ void __launch_bounds__((DET && STAGED) ? kKVThreadsStg : kKVThreads, 1)
    tc_bwd_kv_kernel(BwdKVArgs a) {
  // determinant formers are the busier: their row staging moves to a stager warp (c4 tc_bwd_kv
  // 12.31 -> 11.88 ms); for the trilinear variant the formers' own cp.async staging measured faster
  constexpr bool kStg = DET && STAGED;
  extern __shared__ uint8_t smem_raw[];
  static_assert(sizeof(KVSmem<D>) + 1024 <= 232448, "shared memory budget");
  KVSmem<D>& sm = *reinterpret_cast<KVSmem<D>*>(smem_raw + align1024_pad(smem_raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Problem& p = a.p;
  constexpr int kPanels = D / 64;
  constexpr uint32_t kPanelBytes = KVSmem<D>::kPanelBytes;
  constexpr int kC8 = D / 8;  // 16-byte chunks per row
  const int bh = blockIdx.y, b = bh / p.H, h = bh % p.H, hkv = p.hk(h);
  const int j0 = blockIdx.x * 128;
  // queries touching key rows [j0, j0+128): positions [j0, j0+127+w1-1] within [np, np+N)
  const int qa = max(j0, p.np) - p.np;
  const int qb = min(j0 + 128 + p.w1 - 1, p.np + p.N) - p.np;
  const int ntile = qb > qa ? (qb - qa + a.G - 1) / a.G : 0;

  if (warp == 8 && lane == 0) {
    mbar_init(&sm.kvtm, 8);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.aready[s], kKVFW);
      mbar_init(&sm.afree[s], 1);
      mbar_init(&sm.sfull[s], 1);
      mbar_init(&sm.pready[s], 4);
      mbar_init(&sm.rready[s], 32 * kKVFW);
      mbar_init(&sm.rfree[s], 32 * 8);
    }
    mbar_init(&sm.done, 1);
    for (int x = 0; x < 2; ++x) {
      mbar_init(&sm.stgfull[x], 1);
      mbar_init(&sm.stgempty[x], 1);
    }
    fence_mbar_init();
  }
  if (warp == kKVWarpMMA) tmem_alloc<512>(&sm.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = __shfl_sync(0xffffffffu, sm.tmem_base, 0);  // provably warp-uniform

  if (warp >= kKVF0 && warp < kKVF0 + kKVFW) {
    // ------------------------------ A-tile formers ------------------------------
    const int ft = (warp - kKVF0) * 32 + lane;
    constexpr int kNF = 32 * kKVFW;
    // stage tile t's new rows (K2/V2 ring rows, q/dO rows, lse/delta) with cp.async
    auto ring_mod = [&](int kp) {  // kp mod ring for kp >= -ring (one division per call site)
      return a.fd_ring.mod(kp + a.ring);
    };
    auto stage = [&](int t) {
      const int q0 = qa + t * a.G, P0 = p.np + q0;
      const int klo = t == 0 ? P0 - a.R + 1 : P0, khi = P0 + a.G - 1;
      const int nk = khi - klo + 1;
      const int slo = ring_mod(klo);
#pragma unroll
      for (int which = 0; which < 2 && !kStg; ++which) {
        for (int task = ft; task < nk * kC8; task += kNF) {
          const int off = task / kC8, c8 = task % kC8;  // kC8 is a compile-time power of two
          const int kp = klo + off;
          if (kp < p.k2lo || kp >= p.NK()) continue;
          int slot = slo + off;
          if (slot >= a.ring) slot -= a.ring;
          const __half* src = (which ? a.v2 : a.k2) + p.kvoff(b, kp, hkv) + 8 * c8;
          __half* dst = (which ? &sm.rv2[0][0] : &sm.rk2[0][0]) + slot * D + 8 * c8;
          cp_async16(dst, src);
        }
      }
      const int nq = min(a.G, qb - q0);
#pragma unroll
      for (int which = 0; which < 2 && !kStg; ++which) {
        for (int task = ft; task < nq * kC8; task += kNF) {
          const int g = task / kC8, c8 = task % kC8;
          const __half* src = (which ? a.dO : a.q) + p.qoff(b, q0 + g, h) + 8 * c8;
          __half* dst = (which ? &sm.sdo[t & 1][0][0] : &sm.sq[t & 1][0][0]) + g * D + 8 * c8;
          cp_async16(dst, src);
        }
      }
      if (ft < 2 * nq) {
        const int g = ft < nq ? ft : ft - nq;
        const int64_t x = (int64_t(b) * p.H + h) * p.N + q0 + g;
        if (ft < nq)
          cp_async4(&sm.slse[t & 1][g], a.lse + x);
        else
          cp_async4(&sm.sdl[t & 1][g], a.delta + x);
      }
      cp_async_commit();
    };
    if (STAGED && ntile > 0) {
      stage(0);
      if (kStg && ft == 0) mbar_arrive(&sm.stgempty[0]);
    }
    int trn = 0;
    for (int t = 0; t < ntile; ++t) {
      const int buf = t & 1;
      const int q0 = qa + t * a.G;
      const bool trf = ft == 0 && t >= 50 && t < 53;
      SA_TRACE_AT(trf, 3, trn, t << 16 | 30 << 8);
      if (STAGED) {
        // tile t's rows landed (this thread's copies), then every former is past tile t-1: only now
        // may tile t+1's rows overwrite the q/dO buffer and ring slots tile t-1 read
        cp_async_wait<0>();
        named_bar_sync(2, kNF);
        if (t + 1 < ntile) stage(t + 1);
        if constexpr (kStg) {
          // every former is past tile t-1: its q/dO buffer and the ring slots tile t+1 overwrites are free
          if (t + 1 < ntile && ft == 0) mbar_arrive(&sm.stgempty[(t + 1) & 1]);
          mbar_wait(&sm.stgfull[buf], (t >> 1) & 1);  // tile t's rows landed
        }
      }
      mbar_wait(&sm.afree[buf], ((t >> 1) & 1) ^ 1);
      mbar_wait(&sm.rfree[buf], ((t >> 1) & 1) ^ 1);  // softmax warps are done with rinfo[buf] of tile t-2
      SA_TRACE_AT(trf, 3, trn, t << 16 | 31 << 8);
      // row info: (lse * log2e, delta), +inf marks rows outside the problem
      const int kbase = p.np + q0 - a.R + 1;  // key row of tile row 0
      const int sbase = STAGED ? ring_mod(kbase) : 0;
      for (int r = ft; r < 128; r += kNF) {
        const int g = r >> a.lR, kk = r & (a.R - 1);
        const int i = q0 + g;
        const int kpos = kbase + g + kk;
        const bool valid = r < a.G * a.R && i < qb && kpos >= p.k2lo && kk >= a.R - a.Rt;
        float2 ri = make_float2(INFINITY, 0.f);
        if (valid) {
          if (STAGED) {
            ri = make_float2(sm.slse[buf][g] * kLog2e, sm.sdl[buf][g]);
          } else {
            const int64_t x = (int64_t(b) * p.H + h) * p.N + i;
            ri = make_float2(a.lse[x] * kLog2e, a.delta[x]);
          }
        }
        sm.rinfo[buf][r] = ri;
      }
      mbar_arrive(&sm.rready[buf]);
      SA_TRACE_AT(trf, 3, trn, t << 16 | 33 << 8);
      // A_S = q o k2 [det: k2 x q], A_dP = dO o v2 -> swizzled fp16 tiles
      constexpr int kWS = DET ? 24 : 8;       // A_S task width (elements)
      constexpr int kTS = (D + kWS - 1) / kWS;  // A_S tasks per row (det); trilinear fuses A_S+A_dP
      constexpr int kTasks = DET ? kTS + kC8 : kC8;
      constexpr int kRB8 = 128 * kC8 / kNF;  // rows per thread in the row-block mapping (8 at D=128)
      if (STAGED && a.R >= kRB8) {
        // row blocks: thread -> (column chunk c8, kRB8 consecutive tile rows of ONE query).
        // All loads first, then the products and the stores: no branches, kRB8-way ILP.
        // Trilinear: A_S = q o k2 and A_dP = dO o v2 here; det: A_dP here, A_S below.
        const int c8 = ft % kC8, r0 = (ft / kC8) * kRB8;
        const int g = r0 >> a.lR, kk0 = r0 & (a.R - 1);
        const bool qok = r0 < a.G * a.R && q0 + g < qb;
        uint4 xq = make_uint4(0u, 0u, 0u, 0u), ud = xq;
        if (qok) {
          xq = *reinterpret_cast<const uint4*>(&sm.sq[buf][g][8 * c8]);
          ud = *reinterpret_cast<const uint4*>(&sm.sdo[buf][g][8 * c8]);
        }
        uint4 yk[kRB8], wv[kRB8];
        int slot = sbase + g + kk0;
        if (slot >= a.ring) slot -= a.ring;
#pragma unroll
        for (int u = 0; u < kRB8; ++u) {
          const bool ok = qok && kbase + g + kk0 + u >= p.k2lo;
          int su = slot + u;
          if (su >= a.ring) su -= a.ring;
          yk[u] = wv[u] = make_uint4(0u, 0u, 0u, 0u);
          if (ok) {
            yk[u] = *reinterpret_cast<const uint4*>(&sm.rk2[su][8 * c8]);
            wv[u] = *reinterpret_cast<const uint4*>(&sm.rv2[su][8 * c8]);
          }
        }
#pragma unroll
        for (int u = 0; u < kRB8; ++u) {
          const uint4 od = make_uint4(hmul2_u32(ud.x, wv[u].x), hmul2_u32(ud.y, wv[u].y), hmul2_u32(ud.z, wv[u].z),
                                      hmul2_u32(ud.w, wv[u].w));
          const uint32_t dst = sw128_off(r0 + u, c8);
          if (!DET) {
            const uint4 oa = make_uint4(hmul2_u32(xq.x, yk[u].x), hmul2_u32(xq.y, yk[u].y), hmul2_u32(xq.z, yk[u].z),
                                        hmul2_u32(xq.w, yk[u].w));
            *reinterpret_cast<uint4*>(sm.as[buf] + dst) = oa;
          }
          *reinterpret_cast<uint4*>(sm.adp[buf] + dst) = od;
        }
        if (DET) {
          // A_S = k2 x q = P1(k2) o P2(q) - P2(k2) o P1(q) per 3-chunk (sa_tc_rows.cuh perm3_*): tasks
          // (quad of tile rows of one query (R >= kRB8 >= 4), 24-column block); the query's permuted q
          // block is formed once per task, each row costs 3 LDS, 24 PRMT, 12 HMUL2 + 12 HFMA2, 3 STS.
          constexpr int kNBlk = (D + 23) / 24;
          for (int task = ft; task < 32 * kNBlk; task += kNF) {
            const int rq = task / kNBlk, blk = task - rq * kNBlk;
            const int r0 = 4 * rq, e0 = 24 * blk;
            const int g2 = r0 >> a.lR, kk2 = r0 & (a.R - 1);
            const bool qok = r0 < a.G * a.R && q0 + g2 < qb;
            uint32_t xw[12], x1[12], x2[12];
#pragma unroll
            for (int u = 0; u < 3; ++u) {
              uint4 xv = make_uint4(0u, 0u, 0u, 0u);
              if (qok && e0 + 8 * u < D) xv = *reinterpret_cast<const uint4*>(&sm.sq[buf][g2][e0 + 8 * u]);
              xw[4 * u] = xv.x;
              xw[4 * u + 1] = xv.y;
              xw[4 * u + 2] = xv.z;
              xw[4 * u + 3] = xv.w;
            }
            perm3_block(xw, x1, x2);
            int sl = sbase + g2 + kk2;
            if (sl >= a.ring) sl -= a.ring;
#pragma unroll
            for (int u4 = 0; u4 < 4; ++u4) {
              const bool ok = qok && kbase + g2 + kk2 + u4 >= p.k2lo;
              int su = sl + u4;
              if (su >= a.ring) su -= a.ring;
              uint32_t yw[12], y1[12], y2[12], aw[12];
#pragma unroll
              for (int u = 0; u < 3; ++u) {
                uint4 yv = make_uint4(0u, 0u, 0u, 0u);
                if (ok && e0 + 8 * u < D) yv = *reinterpret_cast<const uint4*>(&sm.rk2[su][e0 + 8 * u]);
                yw[4 * u] = yv.x;
                yw[4 * u + 1] = yv.y;
                yw[4 * u + 2] = yv.z;
                yw[4 * u + 3] = yv.w;
              }
              perm3_block(yw, y1, y2);
#pragma unroll
              for (int i = 0; i < 12; ++i) aw[i] = cross_word(y1[i], y2[i], x1[i], x2[i]);
#pragma unroll
              for (int u = 0; u < 3; ++u)
                if (e0 + 8 * u < D)
                  *reinterpret_cast<uint4*>(sm.as[buf] + sw128_off(r0 + u4, e0 / 8 + u)) =
                      make_uint4(aw[4 * u], aw[4 * u + 1], aw[4 * u + 2], aw[4 * u + 3]);
            }
          }
        }
        SA_TRACE_AT(trf, 3, trn, t << 16 | 34 << 8);
        SA_TRACE_AT(trf, 3, trn, t << 16 | 35 << 8);
      } else if (!DET && STAGED && a.G <= 4) {
        // trilinear, key-row major: thread -> (column chunk c8, key rows kp_rel = grp, grp+ngrp, ...).
        // Each staged k2/v2 chunk is read once and multiplied into the (up to G) tile rows
        // (g, kk = kp_rel - g) that share it; the q/dO chunks of the tile's queries stay in registers.
        constexpr int kNgrp = kNF / kC8;  // 8 (D=128) or 16 (D=64)
        const int c8 = ft % kC8, grp = ft / kC8;
        uint4 xq[4], ud[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          xq[g] = ud[g] = make_uint4(0u, 0u, 0u, 0u);
          if (g < a.G && q0 + g < qb) {
            xq[g] = *reinterpret_cast<const uint4*>(&sm.sq[buf][g][8 * c8]);
            ud[g] = *reinterpret_cast<const uint4*>(&sm.sdo[buf][g][8 * c8]);
          }
        }
        const int nkr = a.R + a.G - 1;
        SA_TRACE_AT(trf, 3, trn, t << 16 | 34 << 8);
        for (int kr = grp; kr < nkr; kr += kNgrp) {
          const int kpos = kbase + kr;
          int slot = sbase + kr;
          if (slot >= a.ring) slot -= a.ring;
          uint4 yk = make_uint4(0u, 0u, 0u, 0u), wv = yk;
          if (kpos >= p.k2lo) {
            yk = *reinterpret_cast<const uint4*>(&sm.rk2[slot][8 * c8]);
            wv = *reinterpret_cast<const uint4*>(&sm.rv2[slot][8 * c8]);
          }
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const int kk = kr - g;
            if (g >= a.G || kk < 0 || kk >= a.R) continue;
            const bool ok = q0 + g < qb && kpos >= p.k2lo;
            uint4 oa = make_uint4(0u, 0u, 0u, 0u), od = oa;
            if (ok) {
              oa = make_uint4(hmul2_u32(xq[g].x, yk.x), hmul2_u32(xq[g].y, yk.y), hmul2_u32(xq[g].z, yk.z),
                              hmul2_u32(xq[g].w, yk.w));
              od = make_uint4(hmul2_u32(ud[g].x, wv.x), hmul2_u32(ud[g].y, wv.y), hmul2_u32(ud[g].z, wv.z),
                              hmul2_u32(ud[g].w, wv.w));
            }
            const uint32_t dst = sw128_off((g << a.lR) + kk, c8);
            *reinterpret_cast<uint4*>(sm.as[buf] + dst) = oa;
            *reinterpret_cast<uint4*>(sm.adp[buf] + dst) = od;
          }
        }
        SA_TRACE_AT(trf, 3, trn, t << 16 | 35 << 8);
        // rows r >= G*R (R not dividing 128) stay zero from the previous fill: clear them explicitly
        for (int r = a.G * a.R + grp; r < 128; r += kNgrp) {
          const uint32_t dst = sw128_off(r, c8);
          *reinterpret_cast<uint4*>(sm.as[buf] + dst) = make_uint4(0u, 0u, 0u, 0u);
          *reinterpret_cast<uint4*>(sm.adp[buf] + dst) = make_uint4(0u, 0u, 0u, 0u);
        }
      } else if (!DET) {
        // trilinear: thread -> (16-byte column chunk c8, block of kRB consecutive rows), 4 rows in
        // flight at a time; the q/dO chunk is reloaded only when the row's query changes
        constexpr int kRB = 128 * kC8 / kNF;  // rows per thread: 16 (D=128) or 8 (D=64)
        const int c8 = ft % kC8, r0 = (ft / kC8) * kRB;
        int gcur = -1;
        uint4 xq = make_uint4(0u, 0u, 0u, 0u), ud = xq;
#pragma unroll
        for (int u0 = 0; u0 < kRB; u0 += 4) {
          uint4 yk[4], wv[4];
          bool ok[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int r = r0 + u0 + u;
            const int g = r >> a.lR, kk = r & (a.R - 1);
            const int i = q0 + g;
            const int kpos = kbase + g + kk;
            ok[u] = r < a.G * a.R && i < qb && kpos >= p.k2lo;
            int slot = sbase + g + kk;
            if (slot >= a.ring) slot -= a.ring;
            if (ok[u]) {
              const __half* k2row = STAGED ? &sm.rk2[slot][0] : a.k2 + p.kvoff(b, kpos, hkv);
              const __half* v2row = STAGED ? &sm.rv2[slot][0] : a.v2 + p.kvoff(b, kpos, hkv);
              yk[u] = *reinterpret_cast<const uint4*>(k2row + 8 * c8);
              wv[u] = *reinterpret_cast<const uint4*>(v2row + 8 * c8);
            }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int r = r0 + u0 + u;
            const int g = r >> a.lR;
            uint4 oa = make_uint4(0u, 0u, 0u, 0u), od = oa;
            if (ok[u]) {
              if (g != gcur) {
                gcur = g;
                const __half* qrow = STAGED ? &sm.sq[buf][g][0] : a.q + p.qoff(b, q0 + g, h);
                const __half* dorow = STAGED ? &sm.sdo[buf][g][0] : a.dO + p.qoff(b, q0 + g, h);
                xq = *reinterpret_cast<const uint4*>(qrow + 8 * c8);
                ud = *reinterpret_cast<const uint4*>(dorow + 8 * c8);
              }
              oa = make_uint4(hmul2_u32(xq.x, yk[u].x), hmul2_u32(xq.y, yk[u].y), hmul2_u32(xq.z, yk[u].z),
                              hmul2_u32(xq.w, yk[u].w));
              od = make_uint4(hmul2_u32(ud.x, wv[u].x), hmul2_u32(ud.y, wv[u].y), hmul2_u32(ud.z, wv[u].z),
                              hmul2_u32(ud.w, wv[u].w));
            }
            const uint32_t dst = sw128_off(r, c8);
            *reinterpret_cast<uint4*>(sm.as[buf] + dst) = oa;
            *reinterpret_cast<uint4*>(sm.adp[buf] + dst) = od;
          }
        }
      } else
      for (int task = ft; task < 128 * kTasks; task += kNF) {
        const int r = task / kTasks, tk = task % kTasks;
        const int g = r >> a.lR, kk = r & (a.R - 1);
        const int i = q0 + g;
        const int kpos = kbase + g + kk;
        const bool valid = r < a.G * a.R && i < qb && kpos >= p.k2lo && kk >= a.R - a.Rt;
        int slot = sbase + g + kk;
        if (slot >= a.ring) slot -= a.ring;
        const __half* qrow = STAGED ? &sm.sq[buf][g][0] : a.q + p.qoff(b, i, h);
        const __half* dorow = STAGED ? &sm.sdo[buf][g][0] : a.dO + p.qoff(b, i, h);
        const __half* k2row = STAGED ? &sm.rk2[slot][0] : a.k2 + p.kvoff(b, kpos, hkv);
        const __half* v2row = STAGED ? &sm.rv2[slot][0] : a.v2 + p.kvoff(b, kpos, hkv);
        if (!DET) {
          uint4 oa = make_uint4(0u, 0u, 0u, 0u), od = oa;
          if (valid) {
            const uint4 x = *reinterpret_cast<const uint4*>(qrow + 8 * tk);
            const uint4 y = *reinterpret_cast<const uint4*>(k2row + 8 * tk);
            const uint4 u = *reinterpret_cast<const uint4*>(dorow + 8 * tk);
            const uint4 w = *reinterpret_cast<const uint4*>(v2row + 8 * tk);
            oa = make_uint4(hmul2_u32(x.x, y.x), hmul2_u32(x.y, y.y), hmul2_u32(x.z, y.z), hmul2_u32(x.w, y.w));
            od = make_uint4(hmul2_u32(u.x, w.x), hmul2_u32(u.y, w.y), hmul2_u32(u.z, w.z), hmul2_u32(u.w, w.w));
          }
          *reinterpret_cast<uint4*>(sm.as[buf] + sw128_off(r, tk)) = oa;
          *reinterpret_cast<uint4*>(sm.adp[buf] + sw128_off(r, tk)) = od;
        } else if (tk < kTS) {
          const int e0 = tk * kWS;
          uint32_t pk[12];
#pragma unroll
          for (int e = 0; e < 12; ++e) pk[e] = 0u;
          if (valid) {
            constexpr int D3 = (D / 3) * 3;
            float xf[24], yf[24];
#pragma unroll
            for (int u = 0; u < 3; ++u) {
              if (e0 + 8 * u < D) {
                const uint4 x = *reinterpret_cast<const uint4*>(qrow + e0 + 8 * u);
                const uint4 y = *reinterpret_cast<const uint4*>(k2row + e0 + 8 * u);
                const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float2 fx = __half22float2(*reinterpret_cast<const __half2*>(&xs[e]));
                  const float2 fy = __half22float2(*reinterpret_cast<const __half2*>(&ys[e]));
                  xf[8 * u + 2 * e] = fx.x;
                  xf[8 * u + 2 * e + 1] = fx.y;
                  yf[8 * u + 2 * e] = fy.x;
                  yf[8 * u + 2 * e + 1] = fy.y;
                }
              } else {
#pragma unroll
                for (int e = 0; e < 8; ++e) xf[8 * u + e] = yf[8 * u + e] = 0.f;
              }
            }
#pragma unroll
            for (int c3 = 0; c3 < 24; c3 += 3) {
              float a0 = 0.f, a1 = 0.f, a2 = 0.f;
              if (e0 + c3 + 3 <= D3) {  // (k2 x q)
                a0 = yf[c3 + 1] * xf[c3 + 2] - yf[c3 + 2] * xf[c3 + 1];
                a1 = yf[c3 + 2] * xf[c3 + 0] - yf[c3 + 0] * xf[c3 + 2];
                a2 = yf[c3 + 0] * xf[c3 + 1] - yf[c3 + 1] * xf[c3 + 0];
              }
              xf[c3] = a0;
              xf[c3 + 1] = a1;
              xf[c3 + 2] = a2;
            }
#pragma unroll
            for (int e = 0; e < 12; ++e) pk[e] = pack_f16x2(xf[2 * e], xf[2 * e + 1]);
          }
#pragma unroll
          for (int u = 0; u < 3; ++u)
            if (e0 + 8 * u < D)
              *reinterpret_cast<uint4*>(sm.as[buf] + sw128_off(r, e0 / 8 + u)) =
                  make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        } else {
          const int c8 = tk - kTS;
          uint4 od = make_uint4(0u, 0u, 0u, 0u);
          if (valid) {
            const uint4 u = *reinterpret_cast<const uint4*>(dorow + 8 * c8);
            const uint4 w = *reinterpret_cast<const uint4*>(v2row + 8 * c8);
            od = make_uint4(hmul2_u32(u.x, w.x), hmul2_u32(u.y, w.y), hmul2_u32(u.z, w.z), hmul2_u32(u.w, w.w));
          }
          *reinterpret_cast<uint4*>(sm.adp[buf] + sw128_off(r, c8)) = od;
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.aready[buf]);
      SA_TRACE_AT(trf, 3, trn, t << 16 | 32 << 8);
      if (STAGED) named_bar_sync(2, kNF);  // staging buffers of tile t are free for tile t+2
    }
  } else if (warp == kKVWarpStg) {
    // ------------------------------ row stager (staged kernels) ------------------------------
    // tile t's new k2/v2 ring rows (its whole window for t = 0) and q/dO rows by 1-D bulk copies, once
    // the formers have freed them (stgempty), completing on stgfull; lse/delta stay with the formers
    if (kStg && lane == 0) {
      for (int t = 0; t < ntile; ++t) {
        mbar_wait(&sm.stgempty[t & 1], (t >> 1) & 1);
        const int q0 = qa + t * a.G, P0 = p.np + q0;
        const int klo = t == 0 ? P0 - a.R + 1 : P0, khi = P0 + a.G - 1;
        const int slo = a.fd_ring.mod(klo + a.ring);
        uint32_t bytes = 0;
        for (int kp = max(klo, p.k2lo); kp <= min(khi, p.NK() - 1); ++kp) {
          int slot = slo + (kp - klo);
          if (slot >= a.ring) slot -= a.ring;
          bulk_load(&sm.rk2[slot][0], a.k2 + p.kvoff(b, kp, hkv), 2 * D, &sm.stgfull[t & 1]);
          bulk_load(&sm.rv2[slot][0], a.v2 + p.kvoff(b, kp, hkv), 2 * D, &sm.stgfull[t & 1]);
          bytes += 4 * D;
        }
        const int nq = min(a.G, qb - q0);
        for (int g = 0; g < nq; ++g) {
          bulk_load(&sm.sq[t & 1][g][0], a.q + p.qoff(b, q0 + g, h), 2 * D, &sm.stgfull[t & 1]);
          bulk_load(&sm.sdo[t & 1][g][0], a.dO + p.qoff(b, q0 + g, h), 2 * D, &sm.stgfull[t & 1]);
          bytes += 4 * D;
        }
        mbar_expect_tx(&sm.stgfull[t & 1], bytes);
      }
    }
  } else if (warp == kKVWarpMMA) {
    // ------------------------------ MMA issuer ------------------------------
    if (ntile > 0) {  // whole warp; elected lane issues
      const uint32_t tK = tbase + kKK, tV = tbase + kKV, tdV = tbase + kKdV, tdK = tbase + kKdK;
      const uint32_t tSD = tbase + kKSD;
      const uint32_t idesc_s = idesc_f16(128, 32, 0, 0);
      const uint32_t idesc_acc = idesc_f16(128, D, 0, 1);
      const int nquart = 4 * ntile;
      mbar_wait(&sm.kvtm, 0);
      tc_fence_after();
      int trn = 0;
      // S^T = K A_S^T and dP^T = V A_dP^T for tile rows [32q, 32q+32) into buffer Q&1
      auto issue_s = [&](int Q) {
        const int t = Q >> 2, q = Q & 3, buf = t & 1, sb = Q & 1;
        if (q == 0) {
          mbar_wait(&sm.aready[buf], (t >> 1) & 1);
          tc_fence_after();
          SA_TRACE_AT(lane == 0 && t >= 50 && t < 53, 4, trn, t << 16 | 40 << 8);
        }
        const uint64_t da = smem_desc_sw128(smem_u32(sm.as[buf]) + q * 32 * 128, 16, 1024);
        const uint64_t dd = smem_desc_sw128(smem_u32(sm.adp[buf]) + q * 32 * 128, 16, 1024);
        if (elect_one()) {  // one thread issues the group (descriptors advance in uniform registers)
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk / 4) * kPanelBytes + (kk % 4) * 32;
            mma_ts(tSD + 64 * sb, tK + kk * 8, desc_adv(da, off), idesc_s, kk > 0 ? 1u : 0u);
            mma_ts(tSD + 64 * sb + 32, tV + kk * 8, desc_adv(dd, off), idesc_s, kk > 0 ? 1u : 0u);
          }
          mma_commit(&sm.sfull[sb]);
        }
        __syncwarp();
      };
      issue_s(0);
      if (nquart > 1) issue_s(1);
      bool early = false;
      for (int Q = 0; Q < nquart; ++Q) {
        const int t = Q >> 2, q = Q & 3, buf = t & 1, sb = Q & 1;
        named_bar_sync(3 + sb, 4 * 32 + 32);  // P/dS of quarter Q ready (warpgroup sb bar.arrives)
        tc_fence_after();
        const uint64_t da = smem_desc_sw128(smem_u32(sm.as[buf]), kPanelBytes, 1024);
        const uint64_t dd = smem_desc_sw128(smem_u32(sm.adp[buf]), kPanelBytes, 1024);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {  // dV += P^T A_dP, dK += dS^T A_S over the quarter's 32 rows
            const uint32_t acc = (Q > 0 || kk > 0) ? 1u : 0u;
            const uint32_t roff = (32 * q + 16 * kk) * 128;
            mma_ts(tdV, tSD + 64 * sb + 8 * kk, desc_adv(dd, roff), idesc_acc, acc);
            mma_ts(tdK, tSD + 64 * sb + 32 + 8 * kk, desc_adv(da, roff), idesc_acc, acc);
          }
        }
        __syncwarp();
        if (q == 3) {
          mma_commit_w(&sm.afree[buf]);
          SA_TRACE_AT(lane == 0 && t >= 50 && t < 53, 4, trn, t << 16 | 41 << 8);
        }
        // quarters of the next tile wait for its A tiles; issue them only after this tile's last
        // dV/dK MMAs so that afree(t) never waits on the formation of tile t+1
        // (issued early, after quarter 2, when the next tile's A tiles are already formed)
        if (q < 2) {
          if (Q + 2 < nquart) issue_s(Q + 2);
        } else if (q == 2) {
          early = Q + 2 < nquart && mbar_test(&sm.aready[buf ^ 1], ((t + 1) >> 1) & 1);
          if (early) issue_s(Q + 2);
        } else {
          if (!early && Q + 1 < nquart) issue_s(Q + 1);
          if (Q + 2 < nquart) issue_s(Q + 2);
        }
      }
      mma_commit_w(&sm.done);
    }
  } else if (warp >= kKVS0 && warp < kKVS0 + 8) {
    // ------------------------------ P^T, dS^T and the dK/dV epilogue ------------------------------
    const int qd = warp & 3, wg = (warp - kKVS0) >> 2;
    const uint32_t lane_off = uint32_t(qd * 32) << 16;
    const uint32_t tS = tbase + kKSD + 64 * wg + lane_off, tdP = tS + 32;
    const uint32_t tdV = tbase + kKdV + lane_off, tdK = tbase + kKdK + lane_off;
    const int j = j0 + qd * 32 + lane;     // this thread's key row
    const int jw0 = j0 + qd * 32;          // warp's first key row
    const float sl2 = p.scale * kLog2e;
    // K (warpgroup 0) / V (warpgroup 1) rows of this CTA -> TMEM fp16 A operands (zero past NK)
    {
      uint32_t pk[D / 2];
#pragma unroll
      for (int t = 0; t < D / 2; ++t) pk[t] = 0u;
      if (j < p.NK()) {
        const uint4* src = reinterpret_cast<const uint4*>((wg == 0 ? a.k : a.v) + p.kvoff(b, j, hkv));
#pragma unroll
        for (int t = 0; t < D / 8; ++t) {
          const uint4 x = src[t];
          pk[4 * t] = x.x;
          pk[4 * t + 1] = x.y;
          pk[4 * t + 2] = x.z;
          pk[4 * t + 3] = x.w;
        }
      }
      tmem_store_row<D>(tbase + (wg == 0 ? kKK : kKV) + lane_off, pk);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.kvtm);
    }
    int trn = 0;
    const int nquart = 4 * ntile;
    for (int Q = wg; Q < nquart; Q += 2) {
      const int t = Q >> 2, q = Q & 3, buf = t & 1;
      const int cb = 32 * q;               // tile columns (rows (i,k)) of this quarter
      const int P0 = p.np + qa + t * a.G;  // key position of the tile's first query
      const bool trs = (threadIdx.x & 127) == 0 && t >= 50 && t < 53;
      mbar_wait(&sm.sfull[wg], (Q >> 1) & 1);
      tc_fence_after();
      if (q < 2) mbar_wait(&sm.rready[buf], (t >> 1) & 1);  // first quarter of tile t for this warpgroup
      SA_TRACE_AT(trs, 5 + wg, trn, t << 16 | (50 + q) << 8);
      // column c (tile row) belongs to query g = c / R at position P0 + g; key row j is in its window
      // iff P0 + g - w1 < j <= P0 + g  <=>  g in [j - P0, j - P0 + w1 - 1]
      const bool all_in = (jw0 + 31 <= P0) && (jw0 > P0 + a.G - 1 - p.w1);
      // fast path: the quarter's 32 columns belong to one query (R >= 32), no column is masked and no
      // row precedes the sequence start -> one (lse, delta) pair, packed math
      const bool fast = all_in && a.R >= 32 && a.Rt == a.R && P0 - a.R + 1 >= p.k2lo;
      uint32_t su[32], du[32];
      tmem_ld32(tS, su);
      tmem_ld32(tdP, du);
      tmem_ld_wait();
      SA_TRACE_AT(trs, 5 + wg, trn, t << 16 | (60 + q) << 8);
      uint32_t pp[16], pd[16];
      if (fast) {
        const float2 ri = sm.rinfo[buf][cb];
        const float2 vs = make_float2(sl2, sl2), vl = make_float2(-ri.x, -ri.x), vd = make_float2(-ri.y, -ri.y);
#pragma unroll
        for (int t2 = 0; t2 < 16; ++t2) {
          const float2 x = ffma2(make_float2(__uint_as_float(su[2 * t2]), __uint_as_float(su[2 * t2 + 1])), vs, vl);
          const float2 pv = make_float2(ex2(x.x), ex2(x.y));
          pp[t2] = pack_f16x2(pv);
          pd[t2] = pack_f16x2(
              fmul2(pv, fadd2(make_float2(__uint_as_float(du[2 * t2]), __uint_as_float(du[2 * t2 + 1])), vd)));
        }
      } else {
        int clo = 0, chi = 31;
        if (!all_in) {
          const int glo = max(0, j - P0), ghi = min(a.G - 1, j - P0 + p.w1 - 1);
          clo = glo * a.R - cb;
          chi = (ghi + 1) * a.R - 1 - cb;
          if (ghi < glo) {
            clo = 1;
            chi = 0;
          }
        }
#pragma unroll
        for (int t2 = 0; t2 < 16; ++t2) {
          const int c = 2 * t2;
          const float2 r0 = sm.rinfo[buf][cb + c], r1 = sm.rinfo[buf][cb + c + 1];
          float p0 = ex2(fmaf(__uint_as_float(su[c]), sl2, -r0.x));
          float p1 = ex2(fmaf(__uint_as_float(su[c + 1]), sl2, -r1.x));
          p0 = (c >= clo && c <= chi) ? p0 : 0.f;
          p1 = (c + 1 >= clo && c + 1 <= chi) ? p1 : 0.f;
          pp[t2] = pack_f16x2(p0, p1);
          pd[t2] = pack_f16x2(p0 * (__uint_as_float(du[c]) - r0.y), p1 * (__uint_as_float(du[c + 1]) - r1.y));
        }
      }
      SA_TRACE_AT(trs, 5 + wg, trn, t << 16 | (64 + q) << 8);
      if (q >= 2) mbar_arrive(&sm.rfree[buf]);  // last read of rinfo[buf] for tile t by this warpgroup
      tmem_st16(tS, pp);
      tmem_st16(tdP, pd);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      named_bar_arrive(3 + wg, 4 * 32 + 32);
      SA_TRACE_AT(trs, 5 + wg, trn, t << 16 | (54 + q) << 8);
    }
    const int half = wg;
    // epilogue: dV, dK rows (lane = key row j), this half's D/2 columns; dK carries the scale s
    if (ntile > 0) {
      mbar_wait(&sm.done, 0);
      tc_fence_after();
    }
    const float ks = p.scale;
#pragma unroll
    for (int t2 = 0; t2 < D / 64; ++t2) {
      const int c0 = half * (D / 2) + 32 * t2;
      uint32_t uv[32], uk[32];
      if (ntile > 0) {  // warp-uniform: tcgen05.ld is .sync.aligned, never under a per-lane branch
        tmem_ld32(tdV + c0, uv);
        tmem_ld32(tdK + c0, uk);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) uv[e] = uk[e] = 0u;
      }
      if (j >= p.NK()) continue;
      const int64_t off = p.koff(b, j, h) + c0;
      if (a.out_f32) {
        float4* dv4 = reinterpret_cast<float4*>(reinterpret_cast<float*>(a.dv) + off);
        float4* dk4 = reinterpret_cast<float4*>(reinterpret_cast<float*>(a.dk) + off);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          dv4[e] = make_float4(__uint_as_float(uv[4 * e]), __uint_as_float(uv[4 * e + 1]),
                               __uint_as_float(uv[4 * e + 2]), __uint_as_float(uv[4 * e + 3]));
          dk4[e] = make_float4(ks * __uint_as_float(uk[4 * e]), ks * __uint_as_float(uk[4 * e + 1]),
                               ks * __uint_as_float(uk[4 * e + 2]), ks * __uint_as_float(uk[4 * e + 3]));
        }
      } else {
        uint4* dv4 = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.dv) + off);
        uint4* dk4 = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.dk) + off);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          uint32_t w[4], x[4];
#pragma unroll
          for (int f = 0; f < 4; ++f) {
            __nv_bfloat162 hv =
                __floats2bfloat162_rn(__uint_as_float(uv[8 * e + 2 * f]), __uint_as_float(uv[8 * e + 2 * f + 1]));
            __nv_bfloat162 hk = __floats2bfloat162_rn(ks * __uint_as_float(uk[8 * e + 2 * f]),
                                                      ks * __uint_as_float(uk[8 * e + 2 * f + 1]));
            w[f] = *reinterpret_cast<uint32_t*>(&hv);
            x[f] = *reinterpret_cast<uint32_t*>(&hk);
          }
          dv4[e] = make_uint4(w[0], w[1], w[2], w[3]);
          dk4[e] = make_uint4(x[0], x[1], x[2], x[3]);
        }
      }
    }
  }

  __syncthreads();
  tc_fence_after();
  if (warp == kKVWarpMMA) tmem_free<512>(tbase);
}

}  // namespace

bool tc_bwd_q2_supported(const Problem& p, int R, int Rt);
int tc_bwd_q2_pairs(const Problem& p, int R, int G, int* per_pair, int* items_out);
cudaError_t tc_bwd_q2_launch(const Problem& p, bool out_f32, const CUtensorMap& tmK, const CUtensorMap& tmV,
                             const __half* q, const __half* k2, const __half* v2, const __half* dO, const float* lse,
                             const float* delta, void* dq, void* dk2, void* dv2, float* band, int R, int G,
                             cudaStream_t st);

cudaError_t split_sum(const float* part, int64_t part_stride, int nsplit, int shift_step, void* out, bool out_f32,
                      int64_t n, int rows, int64_t row_stride, cudaStream_t st);

cudaError_t simt_bwd_dk_only(const Problem& p, bool out_f32, const void* q, const void* k, const void* v,
                             const void* k2, const void* v2, const void* dO, const float* lse, const float* delta,
                             void* dk, void* dv, cudaStream_t st);

static bool swapped(const Problem& p) { return p.w1 < p.w2; }

// Rows per query of the backward tiling: the folded window rounded up to a power of two (>= 2);
// the extra leading rows of each query are masked (BwdQArgs::Rt).
static int tile_rows(int w) {
  int R = 2;
  while (R < w) R <<= 1;
  return R;
}

bool tc_bwd_supported(const Problem& p) {
  const int R = swapped(p) ? p.w1 : p.w2;
  if (!(p.D == 64 || p.D == 128)) return false;
  return R >= 1 && R <= kMaxR;
}

static size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

static int q_grid(const Problem& p, int R, int G, int* per_cta, int* items_out);
static int q_grid_n(const Problem& p, int R, int G) {
  int pc, items;
  return q_grid(p, R, G, &pc, &items);
}
static int q_grid(const Problem& p, int R, int G, int* per_cta, int* items_out) {
  const int ngroups = (p.N + G - 1) / G;
  const int items = ngroups * p.B * p.H;
  const int min_tiles = (R + G - 1) / G + 1;  // a range must span >= R queries (band logic)
  int grid = num_sms();
  int pc = (items + grid - 1) / grid;
  if (pc < min_tiles) pc = min_tiles;
  grid = (items + pc - 1) / pc;
  *per_cta = pc;
  *items_out = items;
  return grid;
}

// Window split (sa_split.cu): a folded window w2 > 32 runs as sub-problems of <= 32 rows, sub-problem
// b covering K' offsets [32 b, 32 b + w_b) back from the query.  SA_NO_WSPLIT=1 keeps the single
// R = 64 / 128 tiling (A/B experiments).
static int split_count(const Problem& p) {
  static const bool off = getenv("SA_NO_WSPLIT") && atoi(getenv("SA_NO_WSPLIT")) != 0;
  if (off || p.w2 <= 32) return 1;
  return (p.w2 + 31) / 32;
}
static Problem split_problem(const Problem& p, int b) {
  Problem s = p;
  s.k2lo = 32 * b;
  s.w2 = std::min(32, p.w2 - 32 * b);
  return s;
}

// scratch of one (sub-)problem's bwd_q / bwd_kv launches: band workspace and the R = 128 det ring slab
static size_t bwd_core_bytes(const Problem& p) {
  const int R = tile_rows(p.w2), G = 128 / R;
  return a256(sizeof(float) * size_t(q_grid_n(p, R, G)) * 4 * (R - 1 > 0 ? R - 1 : 1) * p.D) +
         (R + G > kRingMax && p.det ? a256(sizeof(float) * size_t(q_grid_n(p, R, G)) * 2 * (R + G) * p.D) : 0);
}

size_t tc_bwd_workspace_bytes(const Problem& p0) {
  Problem p = p0;
  if (swapped(p)) std::swap(p.w1, p.w2);
  const size_t n = p.nkey(), nq = size_t(p.B) * p.N * p.H * p.D;
  const size_t nkh = size_t(p.B) * p.NK() * p.H * p.D;  // per-query-head key-side gradient
  size_t core = 0, parts = 0;
  const int ns = split_count(p);
  for (int b = 0; b < ns; ++b) core = std::max(core, bwd_core_bytes(ns > 1 ? split_problem(p, b) : p));
  if (ns > 1) parts = size_t(ns) * (a256(4 * nq) + 4 * a256(4 * nkh));
  return a256(sizeof(float) * size_t(p.B) * p.H * p.N) + 4 * a256(n * 2) + 2 * a256(nq * 2) + core + parts;
}

static cudaError_t bwd_core(const Problem& p, bool out_f32, const char* kf, const char* vf, const char* k2f,
                            const char* v2f, const char* qf, const char* dof, const float* lse, const float* delta,
                            void* dq, void* dk, void* dv, void* dk2, void* dv2, char* w, cudaStream_t st);

cudaError_t tc_backward(const Problem& p0, bool out_f32, const void* q, const void* k, const void* v, const void* k2,
                        const void* v2, const void* o, const float* lse, const void* dO, void* dq, void* dk, void* dv,
                        void* dk2, void* dv2, void* ws, size_t ws_bytes, cudaStream_t st) {
  Problem p = p0;
  if (swapped(p)) {  // fold the smaller-window key into the query; gradients swap with it
    std::swap(k, k2);
    std::swap(v, v2);
    std::swap(dk, dk2);
    std::swap(dv, dv2);
    std::swap(p.w1, p.w2);
    if (p.det) p.scale = -p.scale;
  }
  if (ws_bytes < tc_bwd_workspace_bytes(p0)) return cudaErrorInvalidValue;
  const size_t n = p.nkey();
  char* w = (char*)ws;
  float* delta = (float*)w;
  w += a256(sizeof(float) * size_t(p.B) * p.H * p.N);
  char* kf = w;
  w += a256(n * 2);
  char* vf = w;
  w += a256(n * 2);
  const size_t nq = size_t(p.B) * p.N * p.H * p.D;
  char* k2f = w;
  w += a256(n * 2);
  char* v2f = w;
  w += a256(n * 2);
  char* qf = w;
  w += a256(nq * 2);
  char* dof = w;
  w += a256(nq * 2);

  // delta
  {
    const int64_t rows = int64_t(p.B) * p.H * p.N;
    KernelScope ks("tc_delta", st);
    if (out_f32)
      delta_kernel<float><<<unsigned((rows + 7) / 8), 256, 0, st>>>(p, (const __nv_bfloat16*)dO, (const float*)o, delta);
    else
      delta_kernel<__nv_bfloat16><<<unsigned((rows + 7) / 8), 256, 0, st>>>(p, (const __nv_bfloat16*)dO,
                                                                             (const __nv_bfloat16*)o, delta);
  }
  cudaError_t e = convert_pair_f16(k, kf, v, vf, int64_t(n), num_sms(), st);
  if (e == cudaSuccess) e = convert_pair_f16(k2, k2f, v2, v2f, int64_t(n), num_sms(), st);
  if (e == cudaSuccess) e = convert_pair_f16(q, qf, dO, dof, int64_t(nq), num_sms(), st);
  if (e != cudaSuccess) return e;

  const int ns = split_count(p);
  if (ns == 1) return bwd_core(p, out_f32, kf, vf, k2f, v2f, qf, dof, lse, delta, dq, dk, dv, dk2, dv2, w, st);

  // window split: sub-problem b writes fp32 partials (its dK'/dV' through pointers shifted by -d_b rows)
  size_t core = 0;
  for (int b = 0; b < ns; ++b) core = std::max(core, bwd_core_bytes(split_problem(p, b)));
  char* parts = w + core;
  const size_t nkh = size_t(p.B) * p.NK() * p.H * p.D;
  const size_t set = a256(4 * nq) + 4 * a256(4 * nkh);  // one sub-problem's partials, in floats below
  const int64_t kstep = int64_t(p.Hk) * p.D, gstep = int64_t(p.H) * p.D;  // one key row: input / gradient
  for (int b = 0; b < ns && e == cudaSuccess; ++b) {
    const Problem sp = split_problem(p, b);
    char* s = parts + size_t(b) * set;
    float* pdq = (float*)s;
    float* pdk = (float*)(s + a256(4 * nq));
    float* pdv = pdk + a256(4 * nkh) / 4;
    float* pdk2 = pdv + a256(4 * nkh) / 4;
    float* pdv2 = pdk2 + a256(4 * nkh) / 4;
    const int64_t d = sp.k2lo;
    e = bwd_core(sp, true, kf, vf, (const char*)((const __half*)k2f - d * kstep),
                 (const char*)((const __half*)v2f - d * kstep), qf, dof, lse, delta, pdq, pdk, pdv, pdk2 - d * gstep,
                 pdv2 - d * gstep, w, st);
  }
  // sums: dq, dk, dv over every partial; dk2, dv2 over the partials that cover the row
  const int64_t sstride = int64_t(set / 4);
  float* p0f = (float*)parts;
  const int64_t o_k = int64_t(a256(4 * nq) / 4), o_s = int64_t(a256(4 * nkh) / 4);
  if (e == cudaSuccess) e = split_sum(p0f, sstride, ns, 0, dq, out_f32, int64_t(nq), p.N, gstep, st);
  if (e == cudaSuccess) e = split_sum(p0f + o_k, sstride, ns, 0, dk, out_f32, int64_t(nkh), p.NK(), gstep, st);
  if (e == cudaSuccess) e = split_sum(p0f + o_k + o_s, sstride, ns, 0, dv, out_f32, int64_t(nkh), p.NK(), gstep, st);
  if (e == cudaSuccess)
    e = split_sum(p0f + o_k + 2 * o_s, sstride, ns, 32, dk2, out_f32, int64_t(nkh), p.NK(), gstep, st);
  if (e == cudaSuccess)
    e = split_sum(p0f + o_k + 3 * o_s, sstride, ns, 32, dv2, out_f32, int64_t(nkh), p.NK(), gstep, st);
  return e;
}

static cudaError_t bwd_core(const Problem& p, bool out_f32, const char* kf, const char* vf, const char* k2f,
                            const char* v2f, const char* qf, const char* dof, const float* lse, const float* delta,
                            void* dq, void* dk, void* dv, void* dk2, void* dv2, char* w, cudaStream_t st) {
  const int Rt = p.w2, R = tile_rows(Rt), G = 128 / R;
  float* band = (float*)w;
  w += a256(sizeof(float) * size_t(q_grid_n(p, R, G)) * 4 * (R - 1 > 0 ? R - 1 : 1) * p.D);
  float* gring = R + G > kRingMax && p.det ? (float*)w : nullptr;  // R = 128 determinant only
  cudaError_t e = cudaSuccess;

  // bwd_q: dq, dk2, dv2
  {
    CUtensorMap tmK, tmV;
    if (!make_tmap_bnhd_f16(&tmK, kf, p.B, p.NK(), p.Hk, p.D, kQChunk) ||
        !make_tmap_bnhd_f16(&tmV, vf, p.B, p.NK(), p.Hk, p.D, kQChunk))
      return cudaErrorInvalidValue;
    BwdQArgs a;
    a.p = p;
    a.q = (const __half*)qf;
    a.k2 = (const __half*)k2f;
    a.v2 = (const __half*)v2f;
    a.dO = (const __half*)dof;
    a.lse = lse;
    a.delta = delta;
    a.dq = dq;
    a.dk2 = dk2;
    a.dv2 = dv2;
    a.band = band;
    a.gring = gring;
    a.tma_stage = 0;
    {
      static const bool ps_off = getenv("SA_Q_PRODSTAGE") && atoi(getenv("SA_Q_PRODSTAGE")) == 0;
      // read by the RING 37 kernels only: measured neutral for trilinear (c3 tc_bwd_q 10.64 vs 10.72 ms)
      // and -3.5% for the determinant variant, whose compute warps are the busier (c4 13.18 -> 12.69 ms)
      a.prod_stage = (!ps_off && p.det) ? 1 : 0;
    }
    a.out_f32 = out_f32 ? 1 : 0;
    a.R = R;
    a.Rt = Rt;
    a.lR = __builtin_ctz(unsigned(R));
    a.G = G;
    a.ngroups = (p.N + G - 1) / G;
    a.ring = R + G;
    a.fd_ng = FastDiv(a.ngroups);
    a.fd_H = FastDiv(p.H);
    a.fd_ring = FastDiv(a.ring);
    // The CTA-pair kernel (sa_tc_bwdq2.cu) is an opt-in experiment (SA_BWDQ_PAIR=1): it measured
    // 17.1 ms against 11.0 ms for tc_bwd_q at c3.  Both write the same band layout,
    // so the fold is shared.
    static const bool pair = getenv("SA_BWDQ_PAIR") && atoi(getenv("SA_BWDQ_PAIR")) != 0;
    if (pair && tc_bwd_q2_supported(p, R, Rt)) {
      const int pairs = tc_bwd_q2_pairs(p, R, G, &a.per_cta, &a.items);
      e = tc_bwd_q2_launch(p, out_f32, tmK, tmV, a.q, a.k2, a.v2, a.dO, lse, delta, dq, dk2, dv2, band, R, G, st);
      if (e != cudaSuccess) return e;
      KernelScope ks("tc_fold", st);
      const int fb = std::max(1, pairs - 1);
      if (out_f32)
        fold_kernel<float><<<fb, 256, 0, st>>>(a, pairs);
      else
        fold_kernel<__nv_bfloat16><<<fb, 256, 0, st>>>(a, pairs);
      goto kv;
    }
    {
    const int grid = q_grid(p, R, G, &a.per_cta, &a.items);
    CUtensorMap tmQs = tmK, tmdOs = tmK, tmK2s = tmK, tmV2s = tmK;  // RING 38 row staging (below)
    auto launch = [&](auto kern, size_t smem) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      KernelScope ks("tc_bwd_q", st);
      kern<<<grid, kQThreads, smem, st>>>(tmK, tmV, tmQs, tmdOs, tmK2s, tmV2s, a);
    };
    // staged rows: q, dO (G each) + k2, v2 (R+G-1 each) double-buffered; the ring holds R+G rows
    const bool staged = G <= 16 && 2 * G + 2 * (R + G - 1) <= kQStageRows && R + G <= 36;
    const bool gr = R + G > kRingMax;  // R = 128: the ring lives in the global slab
#define SA_Q_LAUNCH(DD, DET, RING, STG) launch(tc_bwd_q_kernel<DD, DET, RING, STG>, sizeof(QSmem<DD, RING, STG>) + 1024)
    // row-owned epilogue, 4 K/V stages: trilinear R = 32 / 64, determinant R = 32 (q_epilogue_rot_det)
    const bool rot = p.D == 128 && (R == 32 || (!p.det && R == 64));
    // R in {8, 16} trilinear staged: tensor-core epilogue (SA_Q_TC=0 keeps the shuffle/gather passes)
    static const bool tc_off = getenv("SA_Q_TC") && atoi(getenv("SA_Q_TC")) == 0;
    const bool tce = !tc_off && !p.det && staged && (R == 8 || R == 16);
    // pitched-row staging maps of the RING 38 kernel (a box of D + 8 columns needs a next head)
    a.tma_stage = tce && p.H >= 2 && p.Hk >= 2 && 2 * G + ((R + G - 1 + 7) & ~7) + (R + G - 1) <= kQStageRows;
    if (a.tma_stage) {
      const int64_t kshift = int64_t(p.k2lo) * p.Hk * p.D;
      if (!make_tmap_rows_pitched(&tmQs, qf, p.B, p.N, p.H * p.D, p.D, G) ||
          !make_tmap_rows_pitched(&tmdOs, dof, p.B, p.N, p.H * p.D, p.D, G) ||
          !make_tmap_rows_pitched(&tmK2s, (const __half*)k2f + kshift, p.B, p.NK(), p.Hk * p.D, p.D, R + G - 1) ||
          !make_tmap_rows_pitched(&tmV2s, (const __half*)v2f + kshift, p.B, p.NK(), p.Hk * p.D, p.D, R + G - 1))
        return cudaErrorInvalidValue;
    }
#define SA_Q_PICK(DD, DET)                                                                             \
  (gr ? SA_Q_LAUNCH(DD, DET, DET ? 129 : 130, false)                                                  \
      : (!DET && tce) ? SA_Q_LAUNCH(DD, false, 38, true)                                              \
      : (DD == 128 && rot) ? (staged ? SA_Q_LAUNCH(DD, DET, 37, true) : SA_Q_LAUNCH(DD, DET, 67, false)) \
      : staged ? SA_Q_LAUNCH(DD, DET, 36, true) : SA_Q_LAUNCH(DD, DET, 66, false))
    if (p.D == 128) {
      if (p.det)
        SA_Q_PICK(128, true);
      else
        SA_Q_PICK(128, false);
    } else {
      if (p.det)
        SA_Q_PICK(64, true);
      else
        SA_Q_PICK(64, false);
    }
#undef SA_Q_PICK
#undef SA_Q_LAUNCH
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    KernelScope ks("tc_fold", st);
    const int fb = std::max(1, grid - 1);
    if (out_f32)
      fold_kernel<float><<<fb, 256, 0, st>>>(a, grid);
    else
      fold_kernel<__nv_bfloat16><<<fb, 256, 0, st>>>(a, grid);
    }
  }
kv:
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;

  // bwd_kv: dk, dv
  {
    BwdKVArgs a;
    a.p = p;
    a.q = (const __half*)qf;
    a.k2 = (const __half*)k2f;
    a.v2 = (const __half*)v2f;
    a.dO = (const __half*)dof;
    a.k = (const __half*)kf;
    a.v = (const __half*)vf;
    a.lse = lse;
    a.delta = delta;
    a.dk = dk;
    a.dv = dv;
    a.out_f32 = out_f32 ? 1 : 0;
    a.R = R;
    a.Rt = Rt;
    a.lR = __builtin_ctz(unsigned(R));
    a.G = G;
    a.ring = R + 2 * G;
    a.fd_ring = FastDiv(a.ring);
    const bool staged = G <= kKVGmax && a.ring <= kKVRing;
    dim3 grid((p.NK() + 127) / 128, p.B * p.H);
    auto launch = [&](auto kern, size_t smem) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      KernelScope ks("tc_bwd_kv", st);
      kern<<<grid, (p.det && staged) ? kKVThreadsStg : kKVThreads, smem, st>>>(a);
    };
    const size_t s128 = sizeof(KVSmem<128>) + 1024, s64 = sizeof(KVSmem<64>) + 1024;
    if (p.D == 128) {
      if (p.det)
        staged ? launch(tc_bwd_kv_kernel<128, true, true>, s128) : launch(tc_bwd_kv_kernel<128, true, false>, s128);
      else
        staged ? launch(tc_bwd_kv_kernel<128, false, true>, s128) : launch(tc_bwd_kv_kernel<128, false, false>, s128);
    } else {
      if (p.det)
        staged ? launch(tc_bwd_kv_kernel<64, true, true>, s64) : launch(tc_bwd_kv_kernel<64, true, false>, s64);
      else
        staged ? launch(tc_bwd_kv_kernel<64, false, true>, s64) : launch(tc_bwd_kv_kernel<64, false, false>, s64);
    }
  }
  return cudaGetLastError();
}

}  // namespace sa

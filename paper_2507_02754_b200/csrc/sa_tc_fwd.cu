// sa_tc_fwd.cu -- tcgen05/TMEM/TMA forward of sliding-window 2-simplicial attention (bf16 inputs).
//
// Layout (SURVEY.md finding 1): the 128 MMA rows of a tile are
// (query i, K' offset k) pairs, R = w2 rows per query, G = 128/R queries per tile.  For each row
// the CUDA cores form the A operand a_(i,k) = s log2(e) (q_i o k2_k)   [det: s log2(e) (k2_k x q_i)],
// fp16, stored in TMEM.  The tensor core then contracts it against the long w1 window of K:
//     S[(i,k), j] = a_(i,k) . k_j          (tcgen05 TS-MMA, M=128, N<=128 j-chunk, K=D)
//     U[(i,k), :] += P[(i,k), j] V[j, :]    (tcgen05 TS-MMA, A = P fp16 in TMEM, B = V MN-major)
// with a per-row online softmax over j (P:815-821 pattern, conditional rescaling) and the fused
// epilogue  o_i = sum_k e^{m_(i,k)-m_i} v2_k o U_(i,k) / l_i,  lse_i = m_i + ln l_i  (Eq. attenval
// P:241-244).  K and V tiles arrive by TMA (128B swizzle) into a 3-stage ring; all MMAs use fp16
// operands with fp32 accumulation (K/V converted from bf16 exactly by a pre-pass).
//
// Warp roles (320 threads, 1 CTA/SM, persistent over (b,h,tile) items):
//   warps 0-7: row softmax + epilogue; warps q and 4+q own TMEM lanes 32q..32q+31 and split each S
//   chunk's columns in two halves (max exchanged through shared memory); warp 8: TMA producer;
//   warp 9: TMEM allocator + MMA issuer (whole warp, one elected lane issues).
#include <math.h>

#include <algorithm>
#include <utility>

#include "sa_tc_common.cuh"

namespace sa {

cudaError_t convert_pair_f16(const void* a, void* ao, const void* b, void* bo, int64_t n, int num_sms,
                             cudaStream_t st);
int num_sms();

namespace {

using namespace tc;

constexpr int kThreads = 320;
// warp roles: 0-7 softmax/epilogue (low ids: the scheduler favours high ids, so the latency-critical
// producer and MMA issuer get 8 and 9)
constexpr int kWarpTMA = 8, kWarpMMA = 9;
constexpr int kStages = 3;
constexpr int kChunk = 128;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kRescale = 8.0f;  // log2 units: rescale U only when the row max grows by > 2^8

// TMEM columns
constexpr uint32_t kColU = 0, kColS0 = 128, kColS1 = 256, kColA = 384;

struct FwdArgs {
  Problem p;                 // after the (K,V,w1) <-> (K',V',w2) swap: w2 = rows per query
  const __nv_bfloat16* q;    // [B,N,H,D]
  const __nv_bfloat16* k2;   // folded key (window w2), [B,NK,H,D]
  const __nv_bfloat16* v2;
  void* o;
  float* lse;
  int out_f32;
  int R, G, ngroups, items;
  float a_scale;             // s * log2(e), signed
};

template <int D>
struct Smem {
  static constexpr int kStageBytes = kChunk * D * 2;
  alignas(1024) uint8_t k[kStages][kStageBytes];
  alignas(1024) uint8_t v[kStages][kStageBytes];
  float ebuf[2][128][17];
  float xmax[2][2][128];
  float rm[128], rl[2][128];
  float gM[128], gL[128];
  uint64_t kfull[kStages], kempty[kStages], vfull[kStages], vempty[kStages];
  uint64_t sfull[2], pready[2], pvdone, udone, aready;
  uint32_t tmem_base;
};

struct Item {
  int b, h, i0, nq, jbeg, span, nch;
};

__device__ __forceinline__ Item get_item(const FwdArgs& a, int item) {
  Item it;
  int bh = item / a.ngroups, grp = item % a.ngroups;
  it.b = bh / a.p.H;
  it.h = bh % a.p.H;
  it.i0 = grp * a.G;
  it.nq = min(a.G, a.p.N - it.i0);
  int pos0 = a.p.np + it.i0, posl = pos0 + it.nq - 1;
  it.jbeg = max(0, pos0 - a.p.w1 + 1);
  it.span = posl - it.jbeg + 1;
  it.nch = (it.span + kChunk - 1) / kChunk;
  return it;
}
__device__ __forceinline__ int chunk_width(const Item& it, int c) {
  if (c < it.nch - 1) return kChunk;
  int w = it.span - kChunk * (it.nch - 1);
  return (w + 15) & ~15;
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    tc_fwd_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, FwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  static_assert(sizeof(Smem<D>) + 1024 <= 232448, "shared memory budget");
  Smem<D>& sm = *reinterpret_cast<Smem<D>*>(smem_raw + align1024_pad(smem_raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kPanels = D / 64 > 0 ? D / 64 : 1;
  constexpr uint32_t kPanelBytes = kChunk * 128;

  if (warp == kWarpTMA && lane == 0) {
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sm.kfull[s], 1);
      mbar_init(&sm.kempty[s], 1);
      mbar_init(&sm.vfull[s], 1);
      mbar_init(&sm.vempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.sfull[s], 1);
      mbar_init(&sm.pready[s], 8);
    }
    mbar_init(&sm.pvdone, 1);
    mbar_init(&sm.udone, 1);
    mbar_init(&sm.aready, 8);
    fence_mbar_init();
  }
  if (warp == kWarpMMA) tmem_alloc<512>(&sm.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = __shfl_sync(0xffffffffu, sm.tmem_base, 0);  // provably warp-uniform

  if (warp == kWarpTMA) {
    // ------------------------------ TMA producer ------------------------------
    if (lane == 0) {
      uint32_t kc = 0;
      for (int item = blockIdx.x; item < a.items; item += gridDim.x) {
        Item it = get_item(a, item);
        for (int c = 0; c < it.nch; ++c, ++kc) {
          const int s = kc % kStages;
          const uint32_t ph = (kc / kStages) & 1;
          const int row = it.jbeg + c * kChunk;
          mbar_wait(&sm.kempty[s], ph ^ 1);
          mbar_expect_tx(&sm.kfull[s], Smem<D>::kStageBytes);
          for (int pn = 0; pn < kPanels; ++pn)
            tma_load_4d(sm.k[s] + pn * kPanelBytes, &tmK, &sm.kfull[s], pn * 64, it.h, row, it.b);
          mbar_wait(&sm.vempty[s], ph ^ 1);
          mbar_expect_tx(&sm.vfull[s], Smem<D>::kStageBytes);
          for (int pn = 0; pn < kPanels; ++pn)
            tma_load_4d(sm.v[s] + pn * kPanelBytes, &tmV, &sm.vfull[s], pn * 64, it.h, row, it.b);
        }
      }
    }
  } else if (warp == kWarpMMA) {
    // ------------------------------ MMA issuer ------------------------------
    {  // whole warp; elected lane issues
      const uint32_t tU = tbase + kColU, tA = tbase + kColA;
      const uint32_t tS[2] = {tbase + kColS0, tbase + kColS1};
      const uint32_t idesc_pv = idesc_f16(128, D, 0, 1);
      uint32_t kc = 0, cc = 0, pvc = 0, gc = 0;
      for (int item = blockIdx.x; item < a.items; item += gridDim.x) {
        Item it = get_item(a, item);
        mbar_wait(&sm.aready, gc & 1);
        tc_fence_after();
        auto issue_pv = [&](int c) {
          const uint32_t sb = (cc + c) & 1, pph = ((cc + c) >> 1) & 1;
          const int s = (kc + c) % kStages;
          const uint32_t ph = ((kc + c) / kStages) & 1;
          mbar_wait(&sm.pready[sb], pph);
          mbar_wait(&sm.vfull[s], ph);
          tc_fence_after();
          const int w = chunk_width(it, c);
          const uint32_t vaddr = smem_u32(sm.v[s]);
          for (int kk = 0; kk < w / 16; ++kk) {
            uint64_t bd = smem_desc_sw128(vaddr + kk * 16 * 128, kPanelBytes, 1024);
            mma_ts_w(tU, tS[sb] + kk * 8, bd, idesc_pv, (c > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit_w(&sm.vempty[s]);
          mma_commit_w(&sm.pvdone);
        };
        for (int c = 0; c < it.nch; ++c) {
          const int s = (kc + c) % kStages;
          const uint32_t ph = ((kc + c) / kStages) & 1;
          const uint32_t sb = (cc + c) & 1;
          mbar_wait(&sm.kfull[s], ph);
          tc_fence_after();
          const uint32_t idesc_s = idesc_f16(128, chunk_width(it, c), 0, 0);
          const uint32_t kaddr = smem_u32(sm.k[s]);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            uint64_t bd = smem_desc_sw128(kaddr + (kk / 4) * kPanelBytes + (kk % 4) * 32, 16, 1024);
            mma_ts_w(tS[sb], tA + kk * 8, bd, idesc_s, kk > 0 ? 1u : 0u);
          }
          mma_commit_w(&sm.sfull[sb]);
          mma_commit_w(&sm.kempty[s]);
          if (c > 0) issue_pv(c - 1);
        }
        issue_pv(it.nch - 1);
        mma_commit_w(&sm.udone);
        kc += it.nch;
        cc += it.nch;
        pvc += it.nch;
        ++gc;
      }
      (void)pvc;
    }
  } else if (warp < 8) {
    // ------------------------------ softmax + epilogue ------------------------------
    // 8 warps: warp 4+qd and 8+qd share TMEM lane quadrant qd (rows r = 32 qd + lane); the
    // first ("half 0") handles chunk columns [0,64), the second [64,128).
    const int qd = warp & 3, half = warp >> 2;
    const int r = qd * 32 + lane;
    const uint32_t lane_off = uint32_t(qd * 32) << 16;
    const uint32_t tU = tbase + kColU + lane_off, tA = tbase + kColA + lane_off;
    const uint32_t tS[2] = {tbase + kColS0 + lane_off, tbase + kColS1 + lane_off};
    const Problem& p = a.p;
    const int cbase = 64 * half;
    constexpr int kUH = D / 2;  // U columns per half
    uint32_t cc = 0, pvc = 0, gc = 0;
    for (int item = blockIdx.x; item < a.items; item += gridDim.x) {
      Item it = get_item(a, item);
      const int g = r / a.R, kk = r % a.R;
      const bool row_in = r < a.G * a.R && g < it.nq;
      const int pos = p.np + it.i0 + g;
      const int kpos = pos - a.R + 1 + kk;
      const bool valid = row_in && kpos >= 0;

      // ---- A operand: a_(i,k) = s log2e (q_i o k2_k)  or  s log2e (k2_k x q_i), fp16 -> TMEM ----
      {
        uint32_t pk[D / 2];
#pragma unroll
        for (int t = 0; t < D / 2; ++t) pk[t] = 0u;
        if (valid) {
          const uint4* qp = reinterpret_cast<const uint4*>(a.q + p.qoff(it.b, it.i0 + g, it.h));
          const uint4* kp = reinterpret_cast<const uint4*>(a.k2 + p.koff(it.b, kpos, it.h));
          if (p.det) {
            // chunkwise cross product, 24-element blocks (LCM of the 3-chunk and the 8-wide load)
            constexpr int D3 = (D / 3) * 3;
#pragma unroll
            for (int base = 0; base < D; base += 24) {
              float qf[24], kf[24], av[24];
#pragma unroll
              for (int u = 0; u < 3; ++u) {
                if (base + 8 * u < D) {
                  uint4 x = __ldg(qp + base / 8 + u), y = __ldg(kp + base / 8 + u);
                  uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
                  for (int e = 0; e < 4; ++e) {
                    float2 fx = bf16x2_to_f2(xs[e]), fy = bf16x2_to_f2(ys[e]);
                    qf[8 * u + 2 * e] = fx.x;
                    qf[8 * u + 2 * e + 1] = fx.y;
                    kf[8 * u + 2 * e] = fy.x;
                    kf[8 * u + 2 * e + 1] = fy.y;
                  }
                } else {
#pragma unroll
                  for (int e = 0; e < 8; ++e) qf[8 * u + e] = kf[8 * u + e] = 0.f;
                }
              }
#pragma unroll
              for (int c3 = 0; c3 < 24; c3 += 3) {
                if (base + c3 + 3 <= D3) {
                  // (k2 x q)_r = k2_{r+1} q_{r+2} - k2_{r+2} q_{r+1}
                  av[c3 + 0] = kf[c3 + 1] * qf[c3 + 2] - kf[c3 + 2] * qf[c3 + 1];
                  av[c3 + 1] = kf[c3 + 2] * qf[c3 + 0] - kf[c3 + 0] * qf[c3 + 2];
                  av[c3 + 2] = kf[c3 + 0] * qf[c3 + 1] - kf[c3 + 1] * qf[c3 + 0];
                } else {
                  av[c3 + 0] = av[c3 + 1] = av[c3 + 2] = 0.f;
                }
              }
#pragma unroll
              for (int e = 0; e < 24; e += 2)
                if (base + e < D) pk[(base + e) / 2] = pack_f16x2(a.a_scale * av[e], a.a_scale * av[e + 1]);
            }
          } else {
#pragma unroll
            for (int t = 0; t < D / 8; ++t) {
              uint4 x = __ldg(qp + t), y = __ldg(kp + t);
              uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                float2 fx = bf16x2_to_f2(xs[e]), fy = bf16x2_to_f2(ys[e]);
                pk[4 * t + e] = pack_f16x2(a.a_scale * fx.x * fy.x, a.a_scale * fx.y * fy.y);
              }
            }
          }
        }
        // each half stores its D/4 packed columns
        if (D == 128) {
          if (half == 0)
            tmem_st32(tA, *reinterpret_cast<uint32_t(*)[32]>(pk));
          else
            tmem_st32(tA + 32, *reinterpret_cast<uint32_t(*)[32]>(pk + 32 % (D / 2)));
        } else {
          if (half == 0)
            tmem_st16(tA, pk);
          else
            tmem_st16(tA + 16, pk + 16 % (D / 2));
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.aready);
      }

      // ---- chunks: per-row online softmax (conditional rescaling, FA4-style threshold) ----
      float m_ref = -INFINITY, l = 0.f;
      const int jlo = max(0, pos - p.w1 + 1);
      for (int c = 0; c < it.nch; ++c) {
        const uint32_t sb = (cc + c) & 1, ph = ((cc + c) >> 1) & 1;
        const int w = chunk_width(it, c);
        const bool act = cbase < w;  // warp-uniform
        const int nw = act ? min(64, w - cbase) : 0;
        mbar_wait(&sm.sfull[sb], ph);
        tc_fence_after();
        float sv[64];
        if (act) {
          uint32_t* su = reinterpret_cast<uint32_t*>(sv);
          if (nw == 64) {
            tmem_ld32(tS[sb] + cbase, *reinterpret_cast<uint32_t(*)[32]>(su));
            tmem_ld32(tS[sb] + cbase + 32, *reinterpret_cast<uint32_t(*)[32]>(su + 32));
          } else {
            if (nw >= 32) tmem_ld32(tS[sb] + cbase, *reinterpret_cast<uint32_t(*)[32]>(su));
            if (nw == 16) tmem_ld16(tS[sb] + cbase, su);
            if (nw == 48) tmem_ld16(tS[sb] + cbase + 32, su + 32);
          }
          tmem_ld_wait();
        }
        const int jc0 = it.jbeg + c * kChunk + cbase;
        int lo_c = jlo - jc0, hi_c = min(pos - jc0, nw - 1);
        if (!valid) { lo_c = 1; hi_c = 0; }
        const bool need_mask = lo_c > 0 || hi_c < 63;
        float mx = -INFINITY;
        if (act) {
          if (!__any_sync(0xffffffffu, need_mask)) {
#pragma unroll
            for (int jj = 0; jj < 64; ++jj) mx = fmaxf(mx, sv[jj]);
          } else {
#pragma unroll
            for (int jj = 0; jj < 64; ++jj) {
              sv[jj] = (jj >= lo_c && jj <= hi_c) ? sv[jj] : -INFINITY;
              mx = fmaxf(mx, sv[jj]);
            }
          }
        }
        sm.xmax[c & 1][half][r] = mx;
        named_bar_sync(1 + qd, 64);
        mx = fmaxf(sm.xmax[c & 1][0][r], sm.xmax[c & 1][1][r]);
        if (c == 0) {
          m_ref = mx;
        } else {
          const bool need = mx > m_ref + kRescale;
          if (__any_sync(0xffffffffu, need)) {
            // U row rescale: wait for PV(c-1) so the accumulator is stable, then U *= alpha.
            mbar_wait(&sm.pvdone, (pvc + c - 1) & 1);
            tc_fence_after();
            const float alpha = need ? ex2(m_ref - mx) : 1.f;
#pragma unroll
            for (int t = 0; t < kUH / 32; ++t) {
              uint32_t u[32];
              tmem_ld32(tU + half * kUH + 32 * t, u);
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 32; ++e) u[e] = __float_as_uint(__uint_as_float(u[e]) * alpha);
              tmem_st32(tU + half * kUH + 32 * t, u);
            }
            tmem_st_wait();
            if (need) {
              l *= alpha;
              m_ref = mx;
            }
          }
        }
        if (act) {
          const float m_use = m_ref == -INFINITY ? 0.f : m_ref;
          uint32_t pk[32];
          float ls = 0.f;
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            float p0 = ex2(sv[2 * t] - m_use), p1 = ex2(sv[2 * t + 1] - m_use);
            ls += p0 + p1;
            pk[t] = pack_f16x2(p0, p1);
          }
          // columns >= nw were masked to -inf above (need_mask is set whenever nw < 64)
          l += ls;
          const uint32_t pcol = tS[sb] + 32 * half;
          if (nw == 64) {
            tmem_st32(pcol, pk);
          } else {
            if (nw >= 32) tmem_st16(pcol, pk);
            if (nw == 16) tmem_st8(pcol, pk);
            if (nw == 48) tmem_st8(pcol + 16, pk + 16);
          }
          tmem_st_wait();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.pready[sb]);
      }

      // ---- epilogue: merge the R rows of each query, v2 o U, normalise ----
      mbar_wait(&sm.udone, gc & 1);
      tc_fence_after();
      if (half == 0) sm.rm[r] = valid ? m_ref : -INFINITY;
      sm.rl[half][r] = valid ? l : 0.f;
      named_bar_sync(5, 256);
      if (half == 0 && r < it.nq) {
        float M = -INFINITY;
        for (int t = 0; t < a.R; ++t) M = fmaxf(M, sm.rm[r * a.R + t]);
        float L = 0.f;
        for (int t = 0; t < a.R; ++t) {
          float mt = sm.rm[r * a.R + t];
          if (mt != -INFINITY) L += (sm.rl[0][r * a.R + t] + sm.rl[1][r * a.R + t]) * ex2(mt - M);
        }
        sm.gM[r] = M;
        sm.gL[r] = L;
        a.lse[(int64_t(it.b) * p.H + it.h) * p.N + it.i0 + r] = (M + log2f(L)) * kLn2;
      }
      named_bar_sync(5, 256);
      const float crow = (valid && m_ref != -INFINITY) ? ex2(m_ref - sm.gM[g]) : 0.f;
      const __nv_bfloat16* v2row = a.v2 + p.koff(it.b, valid ? kpos : 0, it.h) + half * kUH;
      float(*eb)[17] = sm.ebuf[half];
#pragma unroll 1
      for (int cb = 0; cb < kUH / 16; ++cb) {
        uint32_t u[16];
        tmem_ld16(tU + half * kUH + 16 * cb, u);
        tmem_ld_wait();
        float vv[16];
        if (valid) {
          const uint4* vp = reinterpret_cast<const uint4*>(v2row + 16 * cb);
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            uint4 x = __ldg(vp + t);
            uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float2 f = bf16x2_to_f2(xs[e]);
              vv[8 * t + 2 * e] = f.x;
              vv[8 * t + 2 * e + 1] = f.y;
            }
          }
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e) vv[e] = 0.f;
        }
#pragma unroll
        for (int e = 0; e < 16; ++e) eb[r][e] = crow * vv[e] * __uint_as_float(u[e]);
        named_bar_sync(6 + half, 128);
        for (int idx = r; idx < it.nq * 16; idx += 128) {
          const int gq = idx >> 4, d = idx & 15;
          float s = 0.f;
          for (int t = 0; t < a.R; ++t) s += eb[gq * a.R + t][d];
          const float val = s / sm.gL[gq];
          const int64_t off = p.qoff(it.b, it.i0 + gq, it.h) + half * kUH + 16 * cb + d;
          if (a.out_f32)
            reinterpret_cast<float*>(a.o)[off] = val;
          else
            reinterpret_cast<__nv_bfloat16*>(a.o)[off] = __float2bfloat16_rn(val);
        }
        named_bar_sync(6 + half, 128);
      }
      tc_fence_before();
      cc += it.nch;
      pvc += it.nch;
      ++gc;
    }
  }

  __syncthreads();
  tc_fence_after();
  if (warp == kWarpMMA) tmem_free<512>(tbase);
}

}  // namespace

// The fwd tile needs one K' window of w2 <= 128 rows per query (after folding the smaller window).
static bool swapped(const Problem& p) { return p.w1 < p.w2; }

bool tc_fwd_supported(const Problem& p) {
  const int w2 = swapped(p) ? p.w1 : p.w2;
  return (p.D == 64 || p.D == 128) && w2 >= 1 && w2 <= 128;
}

size_t tc_fwd_workspace_bytes(const Problem& p) {
  size_t n = size_t(p.B) * p.NK() * p.H * p.D;
  return 2 * ((n * 2 + 255) & ~size_t(255));
}

cudaError_t tc_forward_ws(const Problem& p0, bool out_f32, const void* q, const void* k, const void* v,
                          const void* k2, const void* v2, void* o, float* lse, void* ws, cudaStream_t st) {
  Problem p = p0;
  if (swapped(p)) {  // fold the smaller-window key into the query (exact symmetry; det negates)
    std::swap(k, k2);
    std::swap(v, v2);
    std::swap(p.w1, p.w2);
    if (p.det) p.scale = -p.scale;
  }
  const size_t n = size_t(p.B) * p.NK() * p.H * p.D;
  char* kf = (char*)ws;
  char* vf = kf + ((n * 2 + 255) & ~size_t(255));
  cudaError_t e = convert_pair_f16(k, kf, v, vf, int64_t(n), num_sms(), st);
  if (e != cudaSuccess) return e;
  CUtensorMap tmK, tmV;
  if (!make_tmap_bnhd_f16(&tmK, kf, p.B, p.NK(), p.H, p.D, kChunk) ||
      !make_tmap_bnhd_f16(&tmV, vf, p.B, p.NK(), p.H, p.D, kChunk))
    return cudaErrorInvalidValue;
  FwdArgs a;
  a.p = p;
  a.q = (const __nv_bfloat16*)q;
  a.k2 = (const __nv_bfloat16*)k2;
  a.v2 = (const __nv_bfloat16*)v2;
  a.o = o;
  a.lse = lse;
  a.out_f32 = out_f32 ? 1 : 0;
  a.R = p.w2;
  a.G = 128 / p.w2;
  a.ngroups = (p.N + a.G - 1) / a.G;
  a.items = a.ngroups * p.B * p.H;
  a.a_scale = p.scale * kLog2e;
  const int grid = std::min(a.items, num_sms());
  if (p.D == 128) {
    size_t smem = sizeof(Smem<128>) + 1024;
    cudaFuncSetAttribute(tc_fwd_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    KernelScope ks("tc_fwd", st);
    tc_fwd_kernel<128><<<grid, kThreads, smem, st>>>(tmK, tmV, a);
  } else {
    size_t smem = sizeof(Smem<64>) + 1024;
    cudaFuncSetAttribute(tc_fwd_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    KernelScope ks("tc_fwd", st);
    tc_fwd_kernel<64><<<grid, kThreads, smem, st>>>(tmK, tmV, a);
  }
  return cudaGetLastError();
}

cudaError_t tc_forward(const Problem& p, bool out_f32, const void* q, const void* k, const void* v, const void* k2,
                       const void* v2, void* o, float* lse, cudaStream_t st) {
  void* ws = nullptr;
  cudaError_t e = cudaMallocAsync(&ws, tc_fwd_workspace_bytes(p), st);
  if (e != cudaSuccess) return e;
  e = tc_forward_ws(p, out_f32, q, k, v, k2, v2, o, lse, ws, st);
  cudaError_t e2 = cudaFreeAsync(ws, st);
  return e != cudaSuccess ? e : e2;
}

}  // namespace sa

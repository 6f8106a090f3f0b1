// sa_tc_bwdq2.cu -- bwd_q as a CTA pair (thread-block cluster of 2): dQ, dK', dV'.
//
// The query-group backward needs four accumulations per (i,k) row
// tile: S = A_S K^T and dP = A_dP V^T (recomputed), then U += P V and W += dS K.  In one CTA the
// accumulators W, U (256 TMEM columns), S/dP and the row operands fill all 512 TMEM columns, so
// the per-tile epilogue (dq, dk2, dv2 from W and U) cannot overlap the next tile's MMAs: about a
// third of tc_bwd_q's time left the tensor core idle.
//
// Here the two CTAs of a cluster process the same tile sequence and split the two chains:
//   rank 0 ("P side"):  S = A_S K^T, P = exp2(S s log2e - lse log2e) (masked), U += P V,
//                       epilogue dv2_k += sum_i dO_i o U_(i,k)
//   rank 1 ("dS side"): dP = A_dP V^T, dS = P (dP - delta), W += dS K,
//                       epilogue dq_i = s sum_k k2_k o W_(i,k), dk2_k += s sum_i q_i o W_(i,k)
// P crosses from rank 0 to rank 1 through distributed shared memory (st.async, completing on a
// transaction-count mbarrier of rank 1).  Each CTA now needs only one accumulator, so TMEM holds
//   ACC[2] (U or W of two tiles)  cols   0..255
//   X[2]   (S or dP of two chunks) cols 256..383   (P / dS packed fp16 in place)
//   A[2]   (A_S or A_dP of two tiles) cols 384..511
// and the epilogue of tile t (separate warps) runs while the MMAs of tile t+1 proceed.
// K and V chunks arrive by TMA multicast: rank 0 loads K into both CTAs, rank 1 loads V.
//
// Warps: 0-7 softmax (lane quarter w&3, chunk columns [32 (w>>2), +32)), 8-15 row operand /
// epilogue (thread = tile row, column half), 16 TMA, 17 MMA (one elected lane issues).
// Trilinear, D = 128, R = 32 (G = 4) -- the c3 / c4-shape tiling; other shapes use tc_bwd_q.
#include <math.h>

#include <stdlib.h>

#include <algorithm>

#include "sa_tc_rows.cuh"

namespace sa {

int num_sms();

namespace {

using namespace tc;

constexpr int kPW = 18;
constexpr int kPThreads = 32 * kPW;
constexpr int kPEpi0 = 8, kPWarpTMA = 16, kPWarpMMA = 17;
constexpr int kPChunk = 64;
constexpr uint32_t kTAcc = 0, kTX = 256, kTA = 384;
constexpr int kPPitch = 72;   // halves per P row in the exchange buffer (64 + 8: conflict-free rows)
constexpr uint32_t kPBytes = 128 * 32 * 2 * 2;  // P bytes per chunk: 128 rows x 64 cols fp16
constexpr int kBarP = 2;      // named barriers 2, 3: P / dS of chunk parity 0 / 1 ready
constexpr int kBarEpi = 1;    // epilogue warps among themselves
constexpr float kLog2e = 1.4426950408889634f;

struct Q2Args {
  Problem p;                        // after the swap: w2 = R rows per query
  const __half *q, *k2, *v2, *dO;   // fp16 copies
  const float *lse, *delta;
  void *dq, *dk2, *dv2;
  float* band;                      // [pairs][2 start/end][2 k2/v2][R-1][D]
  int out_f32, R, lR, G, ngroups, items, per_pair, ring;
};

template <int D, int NST, int NPS>
struct Q2Smem {
  static constexpr int kStageBytes = kPChunk * D * 2;
  static constexpr int kPanelBytes = kPChunk * 128;
  static constexpr int kRing = 36;                 // R + G
  alignas(1024) uint8_t k[NST][kStageBytes];
  alignas(1024) uint8_t v[NST][kStageBytes];
  alignas(16) __half pbuf[NPS][128][kPPitch];     // rank 1: P of chunk g in slot g % NPS (written by rank 0)
  alignas(16) float acc[kRing][D + 4];             // rank 0: dv2 rows, rank 1: dk2 rows
  uint64_t kvfull[NST], kvempty[NST];
  uint64_t sfull[2], pfull[NPS], pempty[NPS];
  uint64_t aready[2], afree[2], accfull[2], accfree[2];
  uint32_t tmem_base;
};

// Phase trace (trace builds only): cluster 0, tiles [kTrLo, kTrLo + 3) of the pair's range; region =
// 4 rank + role (0 MMA, 1 softmax warp 0, 2 epilogue warp 8, 3 TMA), tag = role event << 8 | chunk.
constexpr int kTrLo = 100;
#ifdef SA_TRACE
#define TR2(role, n, tagv, c)                                                                          \
  do {                                                                                                 \
    if (blockIdx.x < 2 && (n) >= kTrLo && (n) < kTrLo + 3 && tr_n < 255) {                             \
      const int rg_ = 4 * int(rank) + (role);                                                          \
      const int b_ = (rg_ < 6 ? rg_ : rg_ + 8) * 512; /* bwd_kv traces regions 3-6 (1024 each) */      \
      ::sa::g_trace[b_ + 2 * tr_n] = (unsigned long long)((rg_ << 24) | (((n) - kTrLo) << 16) |         \
                                                          ((tagv) << 8) | ((c) & 0xff));               \
      ::sa::g_trace[b_ + 2 * tr_n + 1] = (unsigned long long)clock64();                                \
      ++tr_n;                                                                                          \
    }                                                                                                  \
  } while (0)
#else
#define TR2(role, n, tagv, c) \
  do {                        \
    (void)tr_n;               \
  } while (0)
#endif

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// wait on a phase the peer CTA completes, relaxed at cluster scope: the P buffers are written with
// st.async (async proxy, made visible by the complete_tx of the phase, as for TMA), and the release
// direction only orders reads the peer had already consumed (no acquire fence / L1 invalidate)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0, n = 0;
  long long t0 = 0;
  while (true) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.relaxed.cluster.shared::cta.b64 p, [%1], %2, 10000000;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) break;
    if (++n == 64u) t0 = clock64();  // a deadlock (tens of seconds) traps instead of hanging the GPU
    if (n > 64u && (n & 255u) == 0 && clock64() - t0 > 40000000000LL) __trap();
  }
}
__device__ __forceinline__ void st_async16(uint32_t raddr, uint4 v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%2,%3,%4}, [%5];" ::"r"(raddr),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t rbar) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
}
__device__ __forceinline__ void tma_load_4d_mc(void* smem, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2,
                                               int c3, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, "
      "%4, %5, %6}], [%2], %7;" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "h"(mask)
      : "memory");
}
// arrive on `bar` in both CTAs of the pair once this thread's previously issued MMAs completed
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

struct Q2Item {
  int bh, b, h, hk, grp, i0, nq, jbeg, span, nch;
};
__device__ __forceinline__ Q2Item q2_item(const Q2Args& a, int item) {
  Q2Item it;
  it.bh = item / a.ngroups;
  it.grp = item - it.bh * a.ngroups;
  it.b = it.bh / a.p.H;
  it.h = it.bh - it.b * a.p.H;
  it.hk = a.p.hk(it.h);
  it.i0 = it.grp * a.G;
  it.nq = min(a.G, a.p.N - it.i0);
  const int pos0 = a.p.np + it.i0, posl = pos0 + it.nq - 1;
  it.jbeg = max(0, pos0 - a.p.w1 + 1);
  it.span = posl - it.jbeg + 1;
  it.nch = (it.span + kPChunk - 1) / kPChunk;
  return it;
}
__device__ __forceinline__ int q2_width(const Q2Item& it, int c) {
  if (c < it.nch - 1) return kPChunk;
  return ((it.span - kPChunk * (it.nch - 1)) + 15) & ~15;
}

// exp2 on the FMA pipe (degree-3 minimax, rel. err 1e-4, below fp16 rounding of P); x <= 0 here
__device__ __forceinline__ float2 ex2_poly2_b(float2 x) {
  constexpr float kMagic = 12582912.f;
  x = make_float2(fmaxf(x.x, -126.f), fmaxf(x.y, -126.f));
  const float2 t = fadd2(x, make_float2(kMagic, kMagic));
  const float2 j = fadd2(t, make_float2(-kMagic, -kMagic));
  const float2 f = ffma2(j, make_float2(-1.f, -1.f), x);
  float2 p = ffma2(make_float2(0.055008301765721454f, 0.055008301765721454f), f,
                   make_float2(0.2422094027065684f, 0.2422094027065684f));
  p = ffma2(p, f, make_float2(0.6932828234305377f, 0.6932828234305377f));
  p = ffma2(p, f, make_float2(1.f, 1.f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

// NST K/V stages, NPS P exchange slots, MC: K/V by TMA multicast (rank 0 loads K, rank 1 V, a stage
// is refilled once both CTAs released it) or each CTA loads both (stages released independently)
template <int D, int NST, int NPS, bool MC, bool NOX = false>
__global__ void __launch_bounds__(kPThreads, 1)
    tc_bwd_q2_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, Q2Args a) {
  using Sm = Q2Smem<D, NST, NPS>;
  constexpr int kPStages = NST;
  extern __shared__ uint8_t smem_raw[];
  static_assert(sizeof(Sm) + 1024 <= 232448, "shared memory budget");
  Sm& sm = *reinterpret_cast<Sm*>(smem_raw + align1024_pad(smem_raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();  // 0: P side, 1: dS side
  const uint32_t peer = rank ^ 1u;
  const int pair = blockIdx.x >> 1;
  const int it_begin = pair * a.per_pair;
  const int it_end = min(a.items, it_begin + a.per_pair);
  const int ntiles = max(0, it_end - it_begin);
  constexpr int kPanels = D / 64;
  constexpr uint32_t kPanelBytes = Sm::kPanelBytes;
  const Problem& p = a.p;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    for (int s = 0; s < kPStages; ++s) {
      mbar_init(&sm.kvfull[s], 1);
      mbar_init(&sm.kvempty[s], MC ? 2 : 1);  // multicast: one commit from each CTA of the pair
    }
    for (int s = 0; s < NPS; ++s) {
      mbar_init(&sm.pfull[s], 1);    // rank 1: armed with expect_tx, completed by rank 0's st.async bytes
      mbar_init(&sm.pempty[s], 8);   // rank 0: one relaxed remote arrive per rank-1 softmax warp
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.sfull[s], 1);
      mbar_init(&sm.aready[s], 256);
      mbar_init(&sm.afree[s], 1);
      mbar_init(&sm.accfull[s], 1);
      mbar_init(&sm.accfree[s], 256);
    }
    fence_mbar_init();
    if (rank == 1)
      for (int s = 0; s < NPS; ++s) mbar_expect_tx(&sm.pfull[s], kPBytes);
  }
  if (warp == kPWarpMMA) tmem_alloc<512>(&sm.tmem_base);
  for (int e = threadIdx.x; e < Sm::kRing * (D + 4); e += kPThreads) (&sm.acc[0][0])[e] = 0.f;
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer's barriers are initialised before any remote access
  tc_fence_after();
  const uint32_t tbase = __shfl_sync(0xffffffffu, sm.tmem_base, 0);

  if (warp == kPWarpTMA) {
    // ------------------------------ TMA producer: K (rank 0) / V (rank 1) into both CTAs ------------------------------
    if (lane == 0) {
      uint32_t kc = 0;
      int tr_n = 0;
      const CUtensorMap* tm = rank == 0 ? &tmK : &tmV;
      for (int n = 0; n < ntiles; ++n) {
        const Q2Item it = q2_item(a, it_begin + n);
        for (int c = 0; c < it.nch; ++c, ++kc) {
          const int s = kc % kPStages;
          const uint32_t ph = (kc / kPStages) & 1;
          const int row = it.jbeg + c * kPChunk;
          mbar_wait(&sm.kvempty[s], ph ^ 1);  // both CTAs are done with this stage
          TR2(3, n, 40, c);
          mbar_expect_tx(&sm.kvfull[s], 2 * Sm::kStageBytes);
          if (MC) {
            uint8_t* dst = rank == 0 ? sm.k[s] : sm.v[s];
            for (int pn = 0; pn < kPanels; ++pn)
              tma_load_4d_mc(dst + pn * kPanelBytes, tm, &sm.kvfull[s], pn * 64, it.hk, row, it.b, (uint16_t)3);
          } else {
            for (int pn = 0; pn < kPanels; ++pn) {
              tma_load_4d(sm.k[s] + pn * kPanelBytes, &tmK, &sm.kvfull[s], pn * 64, it.hk, row, it.b);
              tma_load_4d(sm.v[s] + pn * kPanelBytes, &tmV, &sm.kvfull[s], pn * 64, it.hk, row, it.b);
            }
          }
        }
      }
      // drain: every stage's last release (one commit from each CTA, multicast) has arrived here
      for (uint32_t kl = kc >= kPStages ? kc - kPStages : 0; kl < kc; ++kl)
        mbar_wait(&sm.kvempty[kl % kPStages], (kl / kPStages) & 1);
    }
  } else if (warp == kPWarpMMA) {
    // ------------------------------ MMA issuer ------------------------------
    // X(g) = A(tile) . B1(g)^T  (B1 = K on rank 0, V on rank 1), issued one chunk ahead;
    // ACC(tile) += Xp(g) . B2(g)  (B2 = V on rank 0, K on rank 1) once P / dS of g is ready.
    const uint32_t idesc_acc = idesc_f16(128, D, 0, 1);
    int tr_n = 0;
    int n_x = 0, c_x = 0;  // next chunk to issue X for
    uint32_t g_x = 0;
    Q2Item it_x = ntiles > 0 ? q2_item(a, it_begin) : Q2Item{};
    auto issue_x = [&]() {
      const int s = g_x % kPStages;
      if (c_x == 0) {
        mbar_wait(&sm.aready[n_x & 1], (n_x >> 1) & 1);
        tc_fence_after();
      }
      mbar_wait(&sm.kvfull[s], (g_x / kPStages) & 1);
      tc_fence_after();
      TR2(0, n_x, 10, c_x);
      const int w = q2_width(it_x, c_x);
      const uint64_t db = smem_desc_sw128(smem_u32(rank == 0 ? sm.k[s] : sm.v[s]), 16, 1024);
      const uint32_t idesc_x = idesc_f16(128, w, 0, 0);
      const uint32_t tX = tbase + kTX + 64 * (g_x & 1), tA = tbase + kTA + 64 * (n_x & 1);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk / 4) * kPanelBytes + (kk % 4) * 32;
          mma_ts(tX, tA + kk * 8, desc_adv(db, off), idesc_x, kk > 0 ? 1u : 0u);
        }
        mma_commit(&sm.sfull[g_x & 1]);
        if (c_x == it_x.nch - 1) mma_commit(&sm.afree[n_x & 1]);  // A(tile) free once these complete
      }
      __syncwarp();
      ++g_x;
      if (++c_x == it_x.nch) {
        c_x = 0;
        if (++n_x < ntiles) it_x = q2_item(a, it_begin + n_x);
      }
    };
    if (ntiles > 0) issue_x();
    uint32_t g = 0;
    for (int n = 0; n < ntiles; ++n) {
      const Q2Item it = q2_item(a, it_begin + n);
      const uint32_t tAcc = tbase + kTAcc + 128 * (n & 1);
      for (int c = 0; c < it.nch; ++c, ++g) {
        if (n_x < ntiles) issue_x();  // X(g+1) (possibly the next tile's first chunk)
        const int s = g % kPStages;
        const int w = q2_width(it, c);
        named_bar_sync(kBarP + (g & 1), 8 * 32 + 32);  // P / dS of chunk g in TMEM
        tc_fence_after();
        TR2(0, n, 11, c);
        if (c == 0) {
          mbar_wait(&sm.accfree[n & 1], ((n >> 1) & 1) ^ 1);  // epilogue of tile n-2 has read ACC
          tc_fence_after();
          TR2(0, n, 13, c);
        }
        const uint64_t db = smem_desc_sw128(smem_u32(rank == 0 ? sm.v[s] : sm.k[s]), kPanelBytes, 1024);
        const uint32_t tX = tbase + kTX + 64 * (g & 1);
        if (elect_one()) {
          for (int k2i = 0; k2i < w / 16; ++k2i)
            mma_ts(tAcc, tX + 16 * k2i, desc_adv(db, k2i * 16 * 128), idesc_acc, (c > 0 || k2i > 0) ? 1u : 0u);
          if (MC)
            mma_commit_mc(&sm.kvempty[s]);
          else
            mma_commit(&sm.kvempty[s]);
          if (c == it.nch - 1) mma_commit(&sm.accfull[n & 1]);
        }
        __syncwarp();
      }
    }
  } else if (warp < kPEpi0) {
    // ------------------------------ softmax (rank 0: P) / softmax-gradient (rank 1: dS) ------------------------------
    const int qd = warp & 3, half = warp >> 2;
    const int r = qd * 32 + lane;
    const uint32_t lane_off = uint32_t(qd * 32) << 16;
    const float sl2 = p.scale * kLog2e;
    const int cb = 32 * half;
    // peer addresses (rank 0 writes rank 1's pbuf and arrives on its pfull; rank 1 frees rank 0's pempty)
    const uint32_t pb_remote = mapa(smem_u32(&sm.pbuf[0][r][cb]), peer);
    const uint32_t pfull_remote = mapa(smem_u32(&sm.pfull[0]), peer);
    const uint32_t pempty_remote = mapa(smem_u32(&sm.pempty[0]), peer);
    constexpr uint32_t kPBufStride = 128 * kPPitch * 2;
    auto pslot = [](uint32_t gg) { return gg % NPS; };
    auto pphase = [](uint32_t gg) { return (gg / NPS) & 1; };
    // per-row statistic of the tile: lse * log2e (rank 0) or delta (rank 1), prefetched one tile ahead
    auto row_stat = [&](int n) -> float {
      if (n >= ntiles) return 0.f;
      const Q2Item it = q2_item(a, it_begin + n);
      const int g = r >> a.lR;
      if (g >= it.nq) return 0.f;
      const int64_t x = (int64_t(it.b) * p.H + it.h) * p.N + it.i0 + g;
      return rank == 0 ? a.lse[x] * kLog2e : a.delta[x];
    };
    float st_next = row_stat(0);
    uint32_t g = 0;
    int tr_n = 0;
    const bool trw = warp == 0;
    for (int n = 0; n < ntiles; ++n) {
      const Q2Item it = q2_item(a, it_begin + n);
      const float stat = st_next;
      st_next = row_stat(n + 1);
      const int g_row = r >> a.lR, kk = r & (a.R - 1);
      const int pos = p.np + it.i0 + g_row;
      const int kpos = pos - a.R + 1 + kk;
      const bool valid = g_row < it.nq && kpos >= 0;
      const int jlo = max(0, pos - p.w1 + 1);
      for (int c = 0; c < it.nch; ++c, ++g) {
        const int w = q2_width(it, c);
        const uint32_t tX = tbase + kTX + 64 * (g & 1) + lane_off + cb;
        const bool act = cb < w;  // warp-uniform (chunk widths are multiples of 16)
        mbar_wait(&sm.sfull[g & 1], (g >> 1) & 1);
        tc_fence_after();
        if (trw && lane == 0) TR2(1, n, 20, c);
        uint32_t x[32];
        if (act) {
          tmem_ld32(tX, x);
          tmem_ld_wait();
          if (trw && lane == 0) TR2(1, n, 21, c);
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) x[e] = 0u;
        }
        uint32_t pk[16];
        if (rank == 0) {
          // P = exp2(S sl2 - lse log2e) on the window (jlo <= j <= pos), 0 elsewhere
          const int jc0 = it.jbeg + c * kPChunk + cb;
          int lo_c = jlo - jc0, hi_c = min(pos - jc0, 31);
          if (!valid) {
            lo_c = 1;
            hi_c = 0;
          }
          const bool need_mask = lo_c > 0 || hi_c < 31;
          const float2 vs = make_float2(sl2, sl2), vl = make_float2(-stat, -stat);
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            const float2 xx = ffma2(make_float2(__uint_as_float(x[2 * t]), __uint_as_float(x[2 * t + 1])), vs, vl);
            const float2 pv = (t & 3) == 3 ? ex2_poly2_b(xx) : make_float2(ex2(xx.x), ex2(xx.y));
            pk[t] = pack_f16x2(pv);
          }
          if (__any_sync(0xffffffffu, need_mask)) {
#pragma unroll
            for (int t = 0; t < 16; ++t) {
              const uint32_t m0 = (2 * t >= lo_c && 2 * t <= hi_c) ? 0x0000FFFFu : 0u;
              const uint32_t m1 = (2 * t + 1 >= lo_c && 2 * t + 1 <= hi_c) ? 0xFFFF0000u : 0u;
              pk[t] &= (m0 | m1);
            }
          }
          if (!act) {
#pragma unroll
            for (int t = 0; t < 16; ++t) pk[t] = 0u;
          }
          if (trw && lane == 0) TR2(1, n, 24, c);
          if (act) {
            tmem_st8(tX, pk);
            tmem_st8(tX + 16, pk + 8);
          }
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          named_bar_arrive(kBarP + (g & 1), 8 * 32 + 32);  // this CTA's U MMA may go
          if (trw && lane == 0) TR2(1, n, 22, c);
          // hand P to the dS side: wait until it has consumed this buffer's previous P
          if (!NOX) mbar_wait_cluster(&sm.pempty[pslot(g)], pphase(g) ^ 1);
          if (trw && lane == 0) TR2(1, n, 23, c);
          const uint32_t dst = pb_remote + pslot(g) * kPBufStride;
          const uint32_t rbar = pfull_remote + pslot(g) * 8;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (!NOX) st_async16(dst + 16 * u, make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]), rbar);
        } else {
          // dS = P (dP - delta); P = 0 outside the window and on invalid rows, so dS is too
          if (!NOX) mbar_wait_cluster(&sm.pfull[pslot(g)], pphase(g));
          if (trw && lane == 0) TR2(1, n, 23, c);
          if (!NOX && warp == 0 && lane == 0) mbar_expect_tx(&sm.pfull[pslot(g)], kPBytes);  // arm the slot's next use
          const uint4* src = reinterpret_cast<const uint4*>(&sm.pbuf[pslot(g)][r][cb]);
          uint4 pv4[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) pv4[u] = src[u];
          const float2 vd = make_float2(-stat, -stat);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t ps[4] = {pv4[u].x, pv4[u].y, pv4[u].z, pv4[u].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int t = 4 * u + e;
              const float2 pf = __half22float2(*reinterpret_cast<const __half2*>(&ps[e]));
              const float2 dp = fadd2(make_float2(__uint_as_float(x[2 * t]), __uint_as_float(x[2 * t + 1])), vd);
              pk[t] = pack_f16x2(fmul2(pf, dp));
            }
          }
          if (act) {
            tmem_st8(tX, pk);
            tmem_st8(tX + 16, pk + 8);
          }
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          named_bar_arrive(kBarP + (g & 1), 8 * 32 + 32);
          if (trw && lane == 0) TR2(1, n, 22, c);
          if (!NOX && lane == 0) mbar_arrive_remote(pempty_remote + pslot(g) * 8);  // P buffer consumed
        }
      }
    }
    // rank 0: the last two P buffers' release arrivals come from the peer; wait for them so that no
    // remote arrive is still in flight when the pair exits
    if (rank == 0 && !NOX) {
      for (uint32_t gl = g >= NPS ? g - NPS : 0; gl < g; ++gl) mbar_wait_cluster(&sm.pempty[pslot(gl)], pphase(gl));
    }
  } else if (warp < kPWarpTMA) {
    // ------------------------------ row operands and epilogue ------------------------------
    // 8 warps: lane quarter qd = e & 3 (thread = tile row r), column half sub = e >> 2.  Row data
    // (q, dO, k2, v2) is read from global memory (L2): shared memory goes to the K/V stages.
    const int e8 = warp - kPEpi0;
    const int qd = e8 & 3, sub = e8 >> 2;
    const int r = qd * 32 + lane;
    const int tid = e8 * 32 + lane;  // 0..255
    const uint32_t lane_off = uint32_t(qd * 32) << 16;
    const float s = p.scale;
    const int g = r >> a.lR, kk = r & (a.R - 1);
    // row operand of tile n (this thread: columns [64 sub, 64 sub + 64) of its row):
    // rank 0 A_S = q o k2, rank 1 A_dP = dO o v2 (fp16, unscaled) -> A[n & 1]
    auto form_A = [&](int n) {
      const Q2Item it = q2_item(a, it_begin + n);
      const int kpos = p.np + it.i0 + g - a.R + 1 + kk;
      const bool valid = g < it.nq && kpos >= 0;
      uint32_t pk[32];
#pragma unroll
      for (int t = 0; t < 32; ++t) pk[t] = 0u;
      if (valid) {
        const __half* x = (rank == 0 ? a.q : a.dO) + p.qoff(it.b, it.i0 + g, it.h) + 64 * sub;
        const __half* y = (rank == 0 ? a.k2 : a.v2) + p.kvoff(it.b, kpos, it.hk) + 64 * sub;
        uint4 xv[8], yv[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          xv[t] = __ldg(reinterpret_cast<const uint4*>(x) + t);
          yv[t] = __ldg(reinterpret_cast<const uint4*>(y) + t);
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          pk[4 * t + 0] = hmul2_u32(xv[t].x, yv[t].x);
          pk[4 * t + 1] = hmul2_u32(xv[t].y, yv[t].y);
          pk[4 * t + 2] = hmul2_u32(xv[t].z, yv[t].z);
          pk[4 * t + 3] = hmul2_u32(xv[t].w, yv[t].w);
        }
      }
      mbar_wait(&sm.afree[n & 1], ((n >> 1) & 1) ^ 1);  // the S / dP MMAs of tile n-2 have completed
      tc_fence_after();
      tmem_st32(tbase + kTA + 64 * (n & 1) + 32 * sub + lane_off, pk);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&sm.aready[n & 1]);
    };
    int PS = 0, flush_lo = 0;
    int tr_n = 0;
    const bool trw = e8 == 0 && lane == 0;
    if (ntiles > 0) form_A(0);
    for (int n = 0; n < ntiles; ++n) {
      const Q2Item it = q2_item(a, it_begin + n);
      if (trw) TR2(2, n, 30, 0);
      if (n + 1 < ntiles) form_A(n + 1);  // the MMA warp needs it before this tile's last chunk
      if (trw) TR2(2, n, 32, 0);
      // ---- epilogue of tile n from ACC[n & 1] ----
      const bool first_in_sub = n == 0 || it.grp == 0;
      const bool last_in_sub = n == ntiles - 1 || it.grp == a.ngroups - 1;
      const int P0 = p.np + it.i0;
      if (first_in_sub) {
        PS = P0;
        flush_lo = P0 - a.R + 1;
      }
      const int kpos = P0 + g - a.R + 1 + kk;
      const bool valid = g < it.nq && kpos >= 0;
      int slot = (P0 - a.R + 1 + a.ring) % a.ring + g + kk;
      if (slot >= a.ring) slot -= a.ring;
      const int rot = g & 3;  // R = 32: query g == lane quarter; rows sharing a key row never share a block
      const uint32_t tAcc = tbase + kTAcc + 128 * (n & 1) + lane_off;
      const __half* xrow = (rank == 0 ? a.dO : a.q) + p.qoff(it.b, it.i0 + min(g, it.nq - 1), it.h);
      const __half* krow = a.k2 + p.kvoff(it.b, max(kpos, 0), it.hk);
      // operands of phase ph (16 columns): rank 0 dO, rank 1 q and k2
      uint4 o0 = make_uint4(0u, 0u, 0u, 0u), o1 = o0, o2 = o0, o3 = o0;
      auto ld_ops = [&](int ph) {
        const int cs = 32 * ((ph + rot) & 3) + 16 * sub;
        if (valid) {
          o0 = __ldg(reinterpret_cast<const uint4*>(xrow + cs));
          o1 = __ldg(reinterpret_cast<const uint4*>(xrow + cs + 8));
          if (rank == 1) {
            o2 = __ldg(reinterpret_cast<const uint4*>(krow + cs));
            o3 = __ldg(reinterpret_cast<const uint4*>(krow + cs + 8));
          }
        }
      };
      ld_ops(0);
      mbar_wait(&sm.accfull[n & 1], (n >> 1) & 1);
      tc_fence_after();
      if (trw) TR2(2, n, 33, 0);
      float(*ring)[D + 4] = sm.acc;
#pragma unroll 1
      for (int ph = 0; ph < 4; ++ph) {
        const int cs = 32 * ((ph + rot) & 3) + 16 * sub;
        uint32_t u[16];
        tmem_ld16(tAcc + cs, u);
        const uint4 x0 = o0, x1 = o1, k0 = o2, k1 = o3;
        if (ph < 3) ld_ops(ph + 1);
        tmem_ld_wait();
        if (ph == 3) {
          tc_fence_before();
          mbar_arrive(&sm.accfree[n & 1]);  // every TMEM read of ACC[n & 1] is complete
        }
        const uint32_t xs[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
        float4* rp = reinterpret_cast<float4*>(&ring[slot][cs]);
        if (rank == 0) {
          // dv2_k += dO_i o U_(i,k)
          if (valid) {
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              float4 y = rp[t];
              const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&xs[2 * t]));
              const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&xs[2 * t + 1]));
              y.x = fmaf(f0.x, __uint_as_float(u[4 * t + 0]), y.x);
              y.y = fmaf(f0.y, __uint_as_float(u[4 * t + 1]), y.y);
              y.z = fmaf(f1.x, __uint_as_float(u[4 * t + 2]), y.z);
              y.w = fmaf(f1.y, __uint_as_float(u[4 * t + 3]), y.w);
              rp[t] = y;
            }
          }
        } else {
          // dk2_k += s q_i o W_(i,k) (ring);  dq_i = s sum_k k2_k o W_(i,k) (reduce over the 32 lanes)
          const uint32_t ks[8] = {k0.x, k0.y, k0.z, k0.w, k1.x, k1.y, k1.z, k1.w};
          float v[16];
          if (valid) {
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              float4 y = rp[t];
              const float2 q0 = __half22float2(*reinterpret_cast<const __half2*>(&xs[2 * t]));
              const float2 q1 = __half22float2(*reinterpret_cast<const __half2*>(&xs[2 * t + 1]));
              const float2 c0 = __half22float2(*reinterpret_cast<const __half2*>(&ks[2 * t]));
              const float2 c1 = __half22float2(*reinterpret_cast<const __half2*>(&ks[2 * t + 1]));
              const float w0 = s * __uint_as_float(u[4 * t + 0]), w1 = s * __uint_as_float(u[4 * t + 1]);
              const float w2 = s * __uint_as_float(u[4 * t + 2]), w3 = s * __uint_as_float(u[4 * t + 3]);
              y.x = fmaf(q0.x, w0, y.x);
              y.y = fmaf(q0.y, w1, y.y);
              y.z = fmaf(q1.x, w2, y.z);
              y.w = fmaf(q1.y, w3, y.w);
              rp[t] = y;
              v[4 * t + 0] = c0.x * w0;
              v[4 * t + 1] = c0.y * w1;
              v[4 * t + 2] = c1.x * w2;
              v[4 * t + 3] = c1.y * w3;
            }
          } else {
#pragma unroll
            for (int t = 0; t < 16; ++t) v[t] = 0.f;
          }
          // reduce-scatter of 16 columns over the 32 lanes (= the R = 32 rows of query g): lanes
          // 2c, 2c+1 end with column c' = 8 b4 + 4 b3 + 2 b2 + b1 of the block
#pragma unroll
          for (int st = 16, nn = 8; st >= 2; st >>= 1, nn >>= 1) {
            const bool hi = lane & st;
#pragma unroll
            for (int i = 0; i < nn; ++i) {
              const float keep = hi ? v[nn + i] : v[i], send = hi ? v[i] : v[nn + i];
              v[i] = keep + __shfl_xor_sync(0xffffffffu, send, st);
            }
          }
          v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
          if ((lane & 1) == 0 && g < it.nq) {
            const int col = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
            const int64_t off = p.qoff(it.b, it.i0 + g, it.h) + cs + col;
            if (a.out_f32)
              reinterpret_cast<float*>(a.dq)[off] = v[0];
            else
              reinterpret_cast<__nv_bfloat16*>(a.dq)[off] = __float2bfloat16_rn(v[0]);
          }
        }
        named_bar_sync(kBarEpi, 256);
        if (trw) TR2(2, n, 34 + ph, 0);
      }
      // ---- flush ring rows that no later tile of this sub-range touches (rank 0: dv2, rank 1: dk2) ----
      const int PE = P0 + it.nq;
      const int flush_hi = last_in_sub ? PE - 1 : P0 + a.G - a.R;  // inclusive
      const bool end_open = last_in_sub && PE < p.np + p.N;
      const bool start_open = PS > p.np;
      const int nrows = flush_hi - flush_lo + 1;
      const int fbase = (flush_lo + a.ring) % a.ring;
      const int which = rank == 0 ? 1 : 0;
      void* outp = rank == 0 ? a.dv2 : a.dk2;
      for (int idx = tid; idx < nrows * (D / 4); idx += 256) {
        const int rr = idx / (D / 4), d = 4 * (idx - rr * (D / 4));
        const int kp = flush_lo + rr;
        if (kp < 0 || kp >= p.NK()) continue;
        int sl = fbase + rr;
        if (sl >= a.ring) sl -= a.ring;
        float4* rp = reinterpret_cast<float4*>(&ring[sl][d]);
        const float4 val = *rp;
        *rp = make_float4(0.f, 0.f, 0.f, 0.f);
        if (start_open && kp < PS) {
          float* bnd = a.band + ((size_t(pair) * 2 + 0) * 2 + which) * (a.R - 1) * D;
          *reinterpret_cast<float4*>(bnd + size_t(kp - (PS - a.R + 1)) * D + d) = val;
        } else if (end_open && kp + a.R - 1 >= PE) {
          float* bnd = a.band + ((size_t(pair) * 2 + 1) * 2 + which) * (a.R - 1) * D;
          *reinterpret_cast<float4*>(bnd + size_t(kp - (PE - a.R + 1)) * D + d) = val;
        } else {
          const int64_t off = p.koff(it.b, kp, it.h) + d;
          if (a.out_f32) {
            *reinterpret_cast<float4*>(reinterpret_cast<float*>(outp) + off) = val;
          } else {
            __nv_bfloat162 h0 = __floats2bfloat162_rn(val.x, val.y), h1 = __floats2bfloat162_rn(val.z, val.w);
            *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(outp) + off) =
                make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
          }
        }
      }
      flush_lo = flush_hi + 1;
      named_bar_sync(kBarEpi, 256);
      if (trw) TR2(2, n, 38, 0);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // no CTA leaves while its peer may still write its shared memory
  tc_fence_after();
  if (warp == kPWarpMMA) tmem_free<512>(tbase);
}

}  // namespace

// The pair kernel covers trilinear, D = 128, R = w2 = 32 (after the fold of the smaller window).
bool tc_bwd_q2_supported(const Problem& p, int R, int Rt) {
  return !p.det && p.D == 128 && R == 32 && Rt == 32;
}

int tc_bwd_q2_pairs(const Problem& p, int R, int G, int* per_pair, int* items_out) {
  const int ngroups = (p.N + G - 1) / G;
  const int items = ngroups * p.B * p.H;
  const int min_tiles = (R + G - 1) / G + 1;  // a range must span >= R queries (band logic)
  int pairs = std::max(1, num_sms() / 2);
  int pc = (items + pairs - 1) / pairs;
  if (pc < min_tiles) pc = min_tiles;
  pairs = (items + pc - 1) / pc;
  *per_pair = pc;
  *items_out = items;
  return pairs;
}

cudaError_t tc_bwd_q2_launch(const Problem& p, bool out_f32, const CUtensorMap& tmK, const CUtensorMap& tmV,
                             const __half* q, const __half* k2, const __half* v2, const __half* dO, const float* lse,
                             const float* delta, void* dq, void* dk2, void* dv2, float* band, int R, int G,
                             cudaStream_t st) {
  Q2Args a;
  a.p = p;
  a.q = q;
  a.k2 = k2;
  a.v2 = v2;
  a.dO = dO;
  a.lse = lse;
  a.delta = delta;
  a.dq = dq;
  a.dk2 = dk2;
  a.dv2 = dv2;
  a.band = band;
  a.out_f32 = out_f32 ? 1 : 0;
  a.R = R;
  a.lR = __builtin_ctz(unsigned(R));
  a.G = G;
  a.ngroups = (p.N + G - 1) / G;
  a.ring = R + G;
  const int pairs = tc_bwd_q2_pairs(p, R, G, &a.per_pair, &a.items);
  // SA_Q2_CFG (A/B timing): 0 = 5 stages, 2 P slots, multicast; 1 = 4 stages, 4 slots, multicast;
  // 2 = 4 stages, 4 slots, no multicast
  static const int cfgsel = getenv("SA_Q2_CFG") ? atoi(getenv("SA_Q2_CFG")) : 1;
  auto kern = cfgsel == 0   ? tc_bwd_q2_kernel<128, 5, 2, true>
              : cfgsel == 2 ? tc_bwd_q2_kernel<128, 4, 4, false>
              : cfgsel == 3 ? tc_bwd_q2_kernel<128, 4, 4, true, true>  // timing probe only: no P exchange (wrong dS)
                            : tc_bwd_q2_kernel<128, 4, 4, true>;
  const size_t smem = (cfgsel == 0 ? sizeof(Q2Smem<128, 5, 2>) : sizeof(Q2Smem<128, 4, 4>)) + 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(kPThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  KernelScope ks("tc_bwd_q", st);
  return cudaLaunchKernelEx(&cfg, kern, tmK, tmV, a);
}

}  // namespace sa

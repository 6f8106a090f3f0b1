// sa_tc_fwd.cu -- tcgen05/TMEM/TMA forward of sliding-window 2-simplicial attention (bf16 inputs).
//
// Layout (SURVEY.md finding 1): the 128 MMA rows of a tile are
// (query i, K' offset k) pairs, R = w2 rows per query, G = 128/R queries per tile.  For each row
// the CUDA cores form the A operand a_(i,k) = s log2(e) (q_i o k2_k)   [det: s log2(e) (k2_k x q_i)],
// fp16, stored in TMEM.  The tensor core then contracts it against the long w1 window of K:
//     S[(i,k), j] = a_(i,k) . k_j          (tcgen05 TS-MMA, M=128, N<=64 j-chunk, K=D)
//     U[(i,k), :] += P[(i,k), j] V[j, :]    (tcgen05 TS-MMA, A = P fp16 in TMEM, B = V MN-major)
// with a per-row online softmax over j (P:815-821 pattern, conditional rescaling) and the fused
// epilogue  o_i = sum_k e^{m_(i,k)-m_i} v2_k o U_(i,k) / l_i,  lse_i = m_i + ln l_i  (Eq. attenval
// P:241-244).  K and V chunks arrive by TMA (128B swizzle) into a 4-stage ring; all MMAs use fp16
// operands with fp32 accumulation (K/V converted from bf16 exactly by a pre-pass).  Two tiles per
// CTA ping-pong (FA4 pattern) so softmax and tensor work overlap; see the kernel comment below.
#include <math.h>
#include <stdlib.h>

#include <algorithm>
#include <utility>

#include "sa_tc_rows.cuh"

namespace sa {

cudaError_t convert_pair_f16(const void* a, void* ao, const void* b, void* bo, int64_t n, int num_sms,
                             cudaStream_t st);
cudaError_t convert_two_f16(const void* a, void* ao, int64_t na, const void* b, void* bo, int64_t nb, int num_sms,
                            cudaStream_t st);
int num_sms();

namespace {

using namespace tc;

// ---------------------------------------------------------------------------------------------
// Forward v2 (FA4-style ping-pong).  A CTA processes a pair of consecutive query tiles A and B
// (each 128 (i,k)-rows = G queries) over their shared j-window, in 64-column chunks:
//   TMEM: S_A [0,64)  S_B [64,128)  U_A [128,256)  U_B [256,384)  A_A [384,448)  A_B [448,512)
//   MMA issue order: S_A(0) S_B(0) | PV_A(c) S_A(c+1) | PV_B(c) S_B(c+1) | ...
// so each tile's softmax overlaps the other tile's MMAs.  The commit that signals S_X(c+1)
// also covers PV_X(c), so a softmax that must rescale U_X finds it stable.
// Warps 0-3: tile A rows (warp w owns TMEM lanes 32w..32w+31), 4-7: tile B, 8: TMA, 9: MMA.
// ---------------------------------------------------------------------------------------------
constexpr int kThreads = 320;
constexpr int kWarpTMA = 8, kWarpMMA = 9;
constexpr int kStages = 4;
constexpr int kChunk = 64;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kRescale = 8.0f;  // log2 units: rescale U only when the row max grows by > 2^8
constexpr uint32_t kColS0 = 0, kColU0 = 128, kColA0 = 384;
constexpr int kStgRows = 140;  // staged rows per pair (2G + 2(R+2G-1) <= 140: R in {16, 32, 64})

struct FwdArgs {
  Problem p;                // after the (K,V,w1) <-> (K',V',w2) swap: w2 = rows per query
  const __half* q;          // fp16 copy, [B,N,H,D]
  const __half* k2;         // fp16 copy of the folded key (window w2), [B,NK,H,D]
  const __nv_bfloat16* v2;
  void* o;
  float* lse;
  int out_f32;
  int R, G, ngroups, npairs, items;
  int det_neg;    // det with a negated scale (folded window swapped): form q x k2 = -(k2 x q)
  int tma_stage;  // RS staged kernels: rows by pitched TMA boxes (needs H, Hk >= 2), else 1-D bulk copies
  float sm_mult;  // softmax multiplier of the raw (unscaled) logits: |s| log2(e)
};

// exp2 on the FMA pipe for a pair (FA4-style offload of part of the MUFU work): 2^x = 2^round(x) *
// p(f), f = x - round(x) in [-1/2, 1/2], p the degree-3 relative-minimax fit (max rel err 1.0e-4,
// below the fp16 rounding of P).  Arguments below -126 are clamped (result ~1e-38, not 0).
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  constexpr float kMagic = 12582912.f;  // 1.5 * 2^23: x + kMagic rounds x into the low mantissa bits
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

// RS != 0 (R in {2, 4, 8, 16}): two K/V stages (a pair spans one or two chunks) make room for the
// epilogue's fp16 row products X (one 128 x D tile per tile of the pair, SWIZZLE_128B, MN-major A
// operand of the reduction MMA) and the 0/1 query-selection matrix (K-major B operand, N <= 64 rows).
template <int D, int RS>
struct Smem {
  static constexpr bool kRed = RS != 0 && RS < 32;  // tensor-core row-group sums (R <= 16)
  static constexpr int kSt = kRed ? 2 : kStages;
  static constexpr int kPanelBytes = kChunk * 128;  // 64 rows x 64 fp16
  static constexpr int kStageBytes = kChunk * D * 2;
  static constexpr int kXBytes = 128 * 128 * 2;  // two 64-column panels even at D = 64 (the M = 128 MMA reads both)
  static constexpr int kNSel = !kRed ? 16 : (128 / RS < 16 ? 16 : 128 / RS);  // reduction MMA N
  static constexpr int kSelBytes = 2 * kNSel * 128;  // 2 K-panels x kNSel query rows x 128 B
  alignas(1024) uint8_t k[kSt][kStageBytes];
  alignas(1024) uint8_t v[kSt][kStageBytes];
  alignas(1024) uint8_t xr[kRed ? 2 : 1][kRed ? kXBytes : 16];
  alignas(1024) uint8_t sel[kRed ? kSelBytes : 16];
  float ebuf[RS ? 1 : 2][RS ? 1 : 128][17];  // generic / R = 64, 128 epilogues only (RS = 0)
  // staged bf16 rows of the next/current pair: q (2G), k2 (R+2G-1), v2 (R+2G-1); pitch D+8
  // RS: filled by three pitched-row TMA boxes; 144 rows (a multiple of 8) keep buffer 1 128-byte aligned
  alignas(128) __nv_bfloat16 stg[2][RS ? 144 : kStgRows][D + 8];
  float rm[2][128], rl[2][128];
  float gM[2][128], gL[2][128];
  uint64_t kvfull[kSt], kvempty[kSt];
  uint64_t sfull[2], pready[2], udone[2], aready[2], odone[2], stgfull[2], stgempty[2];
  uint32_t tmem_base;
};

struct Item {
  int b, h, hk, pair, jbeg, span, nch;  // hk: the key head query head h reads (GQA)
};

__device__ __forceinline__ Item get_item(const FwdArgs& a, int item) {
  Item it;
  const int bh = item / a.npairs;
  it.pair = item % a.npairs;
  it.b = bh / a.p.H;
  it.h = bh % a.p.H;
  it.hk = a.p.hk(it.h);
  const int i0 = 2 * it.pair * a.G;
  const int iend = min(a.p.N, i0 + 2 * a.G);  // exclusive
  const int pos0 = a.p.np + i0, posl = a.p.np + iend - 1;
  it.jbeg = max(0, pos0 - a.p.w1 + 1);
  it.span = posl - it.jbeg + 1;
  it.nch = (it.span + kChunk - 1) / kChunk;
  return it;
}
__device__ __forceinline__ int chunk_width(const Item& it, int c) {
  if (c < it.nch - 1) return kChunk;
  return ((it.span - kChunk * (it.nch - 1)) + 15) & ~15;
}

// RS: 0, or the tile's R when it is in {2, 4, 8, 16} (those epilogues are compiled into kernels of
// their own: inlined next to the R = 32 / 64 / 128 ones they cost the larger-window kernels ~4%)
template <int D, bool STAGED, int RS>
__global__ void __launch_bounds__(kThreads, 1)
    tc_fwd_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                  const __grid_constant__ CUtensorMap tmQs, const __grid_constant__ CUtensorMap tmK2s,
                  const __grid_constant__ CUtensorMap tmV2s, FwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  using Sm = Smem<D, RS>;
  static_assert(sizeof(Sm) + 1024 <= 232448, "shared memory budget");
  Sm& sm = *reinterpret_cast<Sm*>(smem_raw + align1024_pad(smem_raw));
  constexpr int kStages = Sm::kSt;
  // RS kernels reduce the R rows of each query on the tensor core: O^T = X^T Sel^T (M = D rows of
  // TMEM, N = nsel query columns, K = the 128 tile rows)
  constexpr int kNSel = Sm::kNSel;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kPanels = D / 64;
  constexpr uint32_t kPanelBytes = Sm::kPanelBytes;

  if (warp == kWarpTMA && lane == 0) {
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sm.kvfull[s], 1);
      mbar_init(&sm.kvempty[s], 1);
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(&sm.sfull[x], 1);
      mbar_init(&sm.pready[x], 4);
      mbar_init(&sm.udone[x], 1);
      mbar_init(&sm.aready[x], 4);
      mbar_init(&sm.odone[x], 1);
      mbar_init(&sm.stgfull[x], 1);
      mbar_init(&sm.stgempty[x], 1);
    }
    fence_mbar_init();
  }
  if (warp == kWarpMMA) tmem_alloc<512>(&sm.tmem_base);
  if constexpr (Sm::kRed) {
    // Sel^T [nsel query rows q][128 tile rows r] = (r / RS == q), K-major SWIZZLE_128B (2 K-panels of
    // nsel rows x 128 B); 16-byte chunk (q, c8) holds rows r = 8 c8 .. 8 c8 + 7
    for (int t = threadIdx.x; t < kNSel * 16; t += kThreads) {
      const int q = t >> 4, c8 = t & 15;
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r0 = 8 * c8 + 2 * e;
        const uint32_t lo = (r0 / RS == q) ? 0x3C00u : 0u, hi = ((r0 + 1) / RS == q) ? 0x3C00u : 0u;  // fp16 1.0
        w[e] = lo | (hi << 16);
      }
      *reinterpret_cast<uint4*>(sm.sel + (c8 >> 3) * (kNSel * 128) + q * 128 + (((c8 & 7) ^ (q & 7)) << 4)) =
          make_uint4(w[0], w[1], w[2], w[3]);
    }
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = __shfl_sync(0xffffffffu, sm.tmem_base, 0);  // provably warp-uniform

  if (warp == kWarpTMA) {
    // ------------------------------ TMA producer ------------------------------
    if (lane == 0) {
      uint32_t kc = 0;
      for (int item = blockIdx.x; item < a.items; item += gridDim.x) {
        const Item it = get_item(a, item);
        if (RS != 0 && a.tma_stage) {
          // row staging of this pair (the softmax warps free buffer n & 1 at the top of pair n - 1):
          // three pitched-row TMA boxes (q: 2G rows, k2 / v2: nk2 rows, the v2 box from a row that is a
          // multiple of 8), completing on stgfull; k2 / v2 in real rows (virtual row kp is kp - k2lo)
          const int n = (item - int(blockIdx.x)) / int(gridDim.x), sb = n & 1;
          const int nk2 = a.R + 2 * a.G - 1, nk2p = (nk2 + 7) & ~7;
          const int i0 = 2 * it.pair * a.G, kb = a.p.np + i0 - a.R + 1 - a.p.k2lo;
          mbar_wait(&sm.stgempty[sb], (n >> 1) & 1);
          mbar_expect_tx(&sm.stgfull[sb], uint32_t(2 * a.G + 2 * nk2) * (D + 8) * 2);
          tma_load_4d(&sm.stg[sb][0][0], &tmQs, &sm.stgfull[sb], it.h * D, i0, it.b, 0);
          tma_load_4d(&sm.stg[sb][2 * a.G][0], &tmK2s, &sm.stgfull[sb], it.hk * D, kb, it.b, 0);
          tma_load_4d(&sm.stg[sb][2 * a.G + nk2p][0], &tmV2s, &sm.stgfull[sb], it.hk * D, kb, it.b, 0);
        }
        for (int c = 0; c < it.nch; ++c, ++kc) {
          const int s = kc % kStages;
          const uint32_t ph = (kc / kStages) & 1;
          const int row = it.jbeg + c * kChunk;
          mbar_wait(&sm.kvempty[s], ph ^ 1);
          mbar_expect_tx(&sm.kvfull[s], 2 * Sm::kStageBytes);
          for (int pn = 0; pn < kPanels; ++pn) {
            tma_load_4d(sm.k[s] + pn * kPanelBytes, &tmK, &sm.kvfull[s], pn * 64, it.hk, row, it.b);
            tma_load_4d(sm.v[s] + pn * kPanelBytes, &tmV, &sm.kvfull[s], pn * 64, it.hk, row, it.b);
          }
        }
      }
    }
  } else if (warp == kWarpMMA) {
    // ------------------------------ MMA issuer (whole warp, elected lane issues) ------------------------------
    const uint32_t idesc_pv = idesc_f16(128, D, 0, 1);
    uint32_t kc = 0, gc = 0;
    int trn = 0;
    // S MMAs of chunk c of item `jt` (ring position kc0 + c) into tile x's S columns
    auto issue_s = [&](const Item& jt, uint32_t kc0, int c, int x) {
      const int s = (kc0 + c) % kStages;
      const uint32_t idesc_s = idesc_f16(128, chunk_width(jt, c), 0, 0);
      const uint64_t dk = smem_desc_sw128(smem_u32(sm.k[s]), 16, 1024);
      if (elect_one()) {  // one thread issues the group (descriptors advance in uniform registers)
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk / 4) * kPanelBytes + (kk % 4) * 32;
          mma_ts(tbase + kColS0 + 64 * x, tbase + kColA0 + 64 * x + kk * 8, desc_adv(dk, off), idesc_s,
                 kk > 0 ? 1u : 0u);
        }
        mma_commit(&sm.sfull[x]);
      }
      __syncwarp();
    };
    // A operands of both tiles of item `jt` formed (the 8 softmax warps bar.arrive on named barriers
    // 6/7, the MMA warp blocks in bar.sync: no mbarrier polling), then its chunk-0 S MMAs
    auto first_s = [&](const Item& jt, uint32_t kc0) {
      named_bar_sync(6, 4 * 32 + 32);
      named_bar_sync(7, 4 * 32 + 32);
      mbar_wait(&sm.kvfull[kc0 % kStages], (kc0 / kStages) & 1);
      tc_fence_after();
      issue_s(jt, kc0, 0, 0);
      issue_s(jt, kc0, 0, 1);
    };
    if (blockIdx.x < a.items) first_s(get_item(a, blockIdx.x), 0);
    for (int item = blockIdx.x; item < a.items; item += gridDim.x) {
      const Item it = get_item(a, item);
      const int tn = item / gridDim.x;
      const bool trm = lane == 0 && tn >= 50 && tn < 52;
      SA_TRACE_AT(trm, 0, trn, tn << 16 | 10 << 8);
      if constexpr (!Sm::kRed) {
        if (item != int(blockIdx.x)) first_s(it, kc);
      }
      for (int c = 0; c < it.nch; ++c) {
        const int s = (kc + c) % kStages;
        const int w = chunk_width(it, c);
        const uint32_t vaddr = smem_u32(sm.v[s]);
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          named_bar_sync(4 + x, 4 * 32 + 32);  // P of tile x ready (4 softmax warps arrive)
          tc_fence_after();
          SA_TRACE_AT(trm, 0, trn, tn << 16 | (11 + x) << 8 | c);
          const uint64_t dv = smem_desc_sw128(vaddr, kPanelBytes, 1024);
          if (elect_one()) {
            for (int kk = 0; kk < w / 16; ++kk)
              mma_ts(tbase + kColU0 + 128 * x, tbase + kColS0 + 64 * x + kk * 8, desc_adv(dv, kk * 16 * 128), idesc_pv,
                     (c > 0 || kk > 0) ? 1u : 0u);
          }
          __syncwarp();
          if (c + 1 < it.nch) {
            if (x == 0) {
              mbar_wait(&sm.kvfull[(kc + c + 1) % kStages], ((kc + c + 1) / kStages) & 1);
              tc_fence_after();
            }
            issue_s(it, kc, c + 1, x);
          }
        }
        mma_commit_w(&sm.kvempty[s]);
      }
      mma_commit_w(&sm.udone[0]);
      mma_commit_w(&sm.udone[1]);
      kc += it.nch;
      ++gc;
      if constexpr (Sm::kRed) {
        // the next item's chunk-0 S MMAs go first (its A operands are formed before this item's
        // epilogue), then the two row-group reductions O^T = X^T Sel^T of this item's epilogue into
        // the first kNSel columns of each tile's U (read out before X was published)
        const int nitem = item + int(gridDim.x);
        if (nitem < a.items) first_s(get_item(a, nitem), kc);
        const uint32_t idesc_r = idesc_f16(128, kNSel, 1, 0);
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          named_bar_sync(8 + x, 4 * 32 + 32);  // X of tile x in shared memory (4 epilogue warps arrive)
          tc_fence_after();
          const uint64_t dx = smem_desc_sw128(smem_u32(sm.xr[x]), 128 * 128, 1024);
          const uint64_t ds = smem_desc_sw128(smem_u32(sm.sel), 16, 1024);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)  // K = 128 tile rows, 16 per instruction
              mma_ss(tbase + kColU0 + 128 * x, desc_adv(dx, kk * 16 * 128),
                     desc_adv(ds, (kk / 4) * (kNSel * 128) + (kk % 4) * 32), idesc_r, kk > 0 ? 1u : 0u);
            mma_commit(&sm.odone[x]);
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ------------------------------ softmax + epilogue of tile x = warp / 4 ------------------------------
    const int x = warp >> 2, qd = warp & 3;
    const int r = qd * 32 + lane;
    const int tid = threadIdx.x;  // 0..255
    const uint32_t lane_off = uint32_t(qd * 32) << 16;
    const uint32_t tS = tbase + kColS0 + 64 * x + lane_off;
    const uint32_t tU = tbase + kColU0 + 128 * x + lane_off;
    const uint32_t tA = tbase + kColA0 + 64 * x + lane_off;
    const Problem& p = a.p;
    const int g = r / a.R, kk = r % a.R;
    const int nk2 = a.R + 2 * a.G - 1;  // k2/v2 rows of a pair
    // first v2 staging row: RS kernels start each TMA box on a 128-byte boundary (pitch D + 8 halves:
    // row offsets that are multiples of 8)
    const int nk2p = RS != 0 ? (nk2 + 7) & ~7 : nk2;
    constexpr int kC8 = D / 8;
    // stage the rows of pair `item` into buffer `buf` (cp.async; one commit group per call)
    auto stage = [&](int item, int buf) {
      if (!STAGED) return;
      const Item it = get_item(a, item);
      const int i0 = 2 * it.pair * a.G;
      const int kb = p.np + i0 - a.R + 1;
      const int nrows = 2 * a.G + 2 * nk2;
      if constexpr (RS != 0) {
        // small R: three TMA boxes of pitched rows (q: 2G rows, k2 / v2: nk2 rows each; rows outside
        // the problem zero-fill), completing on stgfull[buf] -- ~1.7k 16-byte cp.async (or ~110 1-D
        // bulk copies) per pair are issue-bound on the softmax warps' path.  k2 / v2 coordinates are
        // real rows (the tensor maps sit on the unshifted tensors): virtual row kp is kp - k2lo.
        if (a.tma_stage) {
          // issued by the TMA producer warp once the buffer is free: signal it (both tiles are past the
          // barrier that retires the previous pair's reads of this buffer)
          if (tid == 0) mbar_arrive(&sm.stgempty[buf]);
          return;
        }
        // one head (the pitched box would be wider than a row): one 1-D bulk copy per row, every row
        // copied (rows outside the problem from a valid dummy address, never read), one expect_tx
        const int row = tid;
        if (row < 2 * a.G + 2 * nk2) {
          const int rr = row - 2 * a.G;
          const int srow = row < 2 * a.G ? row : rr < nk2 ? row : 2 * a.G + nk2p + (rr - nk2);
          const void* src = nullptr;
          if (row < 2 * a.G) {
            if (i0 + row < p.N) src = a.q + p.qoff(it.b, i0 + row, it.h);
          } else {
            const int kp = kb + (rr < nk2 ? rr : rr - nk2);
            if (kp >= p.k2lo && kp < p.NK())
              src = rr < nk2 ? (const void*)(a.k2 + p.kvoff(it.b, kp, it.hk)) : (const void*)(a.v2 + p.kvoff(it.b, kp, it.hk));
          }
          bulk_load(&sm.stg[buf][srow][0], src ? src : (const void*)a.q, 2 * D, &sm.stgfull[buf]);
        }
        if (tid == 0) mbar_expect_tx(&sm.stgfull[buf], uint32_t(2 * a.G + 2 * nk2) * 2 * D);
        return;
      }
      for (int task = tid; task < nrows * kC8; task += 256) {
        const int row = task / kC8, c8 = task % kC8;
        const void* src = nullptr;
        if (row < 2 * a.G) {
          if (i0 + row < p.N) src = a.q + p.qoff(it.b, i0 + row, it.h) + 8 * c8;
        } else {
          const int rr = row - 2 * a.G;
          const int kp = kb + (rr < nk2 ? rr : rr - nk2);
          if (kp >= p.k2lo && kp < p.NK())
            src = rr < nk2 ? (const void*)(a.k2 + p.kvoff(it.b, kp, it.hk) + 8 * c8)
                           : (const void*)(a.v2 + p.kvoff(it.b, kp, it.hk) + 8 * c8);
        }
        if (src) cp_async16(&sm.stg[buf][row][8 * c8], src);
      }
      cp_async_commit();
    };
    uint32_t cc = 0, gc = 0;
    int trn = 0;
    // ---- A operand of pair `fitem` from staging buffer `bf`: a_(i,k) = q_i o k2_k (trilinear,
    //      unscaled) [det: s log2e (k2_k x q_i)], fp16 -> TMEM.  Formed for pair n+1 right after the
    //      chunk loop of pair n (the A regions are free then), so the first S MMAs of n+1 overlap the
    //      epilogue of n. ----
    auto form_A = [&](int fitem, int bf) {
      const Item fit = get_item(a, fitem);
      const int fi0 = (2 * fit.pair + x) * a.G;
      const int fnq = max(0, min(a.G, p.N - fi0));
      const int fkpos = p.np + fi0 + g - a.R + 1 + kk;
      const bool fvalid = r < a.G * a.R && g < fnq && fkpos >= p.k2lo;
      const __half* fq = STAGED ? reinterpret_cast<const __half*>(&sm.stg[bf][x * a.G + g][0])
                                : a.q + p.qoff(fit.b, fi0 + g, fit.h);
      const __half* fk2 = STAGED ? reinterpret_cast<const __half*>(&sm.stg[bf][2 * a.G + x * a.G + g + kk][0])
                                 : a.k2 + p.kvoff(fit.b, fkpos, fit.hk);
      const int ftn = fitem / gridDim.x;
      const bool ftrs = r == 0 && ftn >= 50 && ftn < 52;
        {
          uint32_t pk[D / 2];
  #pragma unroll
          for (int t = 0; t < D / 2; ++t) pk[t] = 0u;
          if (fvalid) {
            if (p.det) {
              if (a.det_neg)  // unscaled q x k2 (the |s| log2e scale is applied by the softmax FFMA)
                det_words_f16<D, 0, D / 2>(fk2, fq, pk);
              else            // unscaled k2 x q
                det_words_f16<D, 0, D / 2>(fq, fk2, pk);
            } else {  // unscaled q o k2 (the scale is applied by the softmax FFMA)
              const uint4* xp = reinterpret_cast<const uint4*>(fq);
              const uint4* yp = reinterpret_cast<const uint4*>(fk2);
  #pragma unroll
              for (int t = 0; t < D / 8; ++t) {
                const uint4 xv = xp[t], yv = yp[t];
                pk[4 * t + 0] = hmul2_u32(xv.x, yv.x);
                pk[4 * t + 1] = hmul2_u32(xv.y, yv.y);
                pk[4 * t + 2] = hmul2_u32(xv.z, yv.z);
                pk[4 * t + 3] = hmul2_u32(xv.w, yv.w);
              }
            }
          }
          SA_TRACE_AT(ftrs, 1 + x, trn, ftn << 16 | 29 << 8);
          tmem_store_row<D>(tA, pk);
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          named_bar_arrive(6 + x, 4 * 32 + 32);
          SA_TRACE_AT(ftrs, 1 + x, trn, ftn << 16 | 21 << 8);
        }

    };
    if (blockIdx.x < a.items) {
      stage(blockIdx.x, 0);
      if (STAGED) {
        if constexpr (RS != 0)
          mbar_wait(&sm.stgfull[0], 0);
        else
          cp_async_wait<0>();
        named_bar_sync(3, 256);
      }
      form_A(blockIdx.x, 0);
    }
    for (int item = blockIdx.x; item < a.items; item += gridDim.x) {
      const Item it = get_item(a, item);
      const int tn = item / gridDim.x;
      const bool trs = r == 0 && tn >= 50 && tn < 52;
      SA_TRACE_AT(trs, 1 + x, trn, tn << 16 | 20 << 8);
      const int buf = STAGED ? int(gc & 1) : 0;
      const int nitem = item + int(gridDim.x);
      // this pair's rows were staged (and waited for) before its A operands were formed; prefetch the next
      // buffer buf ^ 1 held the previous pair, whose epilogue the other tile's warps may still be
      // reading (v2 rows): both tiles pass this barrier before the next pair's rows overwrite it
      if (STAGED && item != int(blockIdx.x)) named_bar_sync(3, 256);
      if (nitem < a.items) stage(nitem, buf ^ 1);
      SA_TRACE_AT(trs, 1 + x, trn, tn << 16 | 28 << 8);
      const int i0 = (2 * it.pair + x) * a.G;
      const int nq = max(0, min(a.G, p.N - i0));
      const bool row_in = r < a.G * a.R && g < nq;
      const int pos = p.np + i0 + g;
      const int kpos = pos - a.R + 1 + kk;
      const bool valid = row_in && kpos >= p.k2lo;
      const int srow = x * a.G + g + kk;  // this row's k2/v2 staging offset
      const __half* qrow = STAGED ? reinterpret_cast<const __half*>(&sm.stg[buf][x * a.G + g][0])
                                  : a.q + p.qoff(it.b, i0 + g, it.h);
      const __half* k2row = STAGED ? reinterpret_cast<const __half*>(&sm.stg[buf][2 * a.G + srow][0])
                                   : a.k2 + p.kvoff(it.b, kpos, it.hk);
      const __nv_bfloat16* v2row = STAGED ? &sm.stg[buf][2 * a.G + nk2p + srow][0] : a.v2 + p.kvoff(it.b, kpos, it.hk);

      // ---- chunks: per-row online softmax (conditional rescaling) ----
      float m_ref = -INFINITY, l = 0.f;
      const int jlo = max(0, pos - p.w1 + 1);
      for (int c = 0; c < it.nch; ++c) {
        const int w = chunk_width(it, c);
        mbar_wait(&sm.sfull[x], (cc + c) & 1);
        tc_fence_after();
        SA_TRACE_AT(trs, 1 + x, trn, tn << 16 | 22 << 8 | c);
        float sv[64];
        {
          uint32_t* su = reinterpret_cast<uint32_t*>(sv);
          if (w >= 32) tmem_ld32(tS, *reinterpret_cast<uint32_t(*)[32]>(su));
          if (w == 64) tmem_ld32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(su + 32));
          if (w == 16) tmem_ld16(tS, su);
          if (w == 48) tmem_ld16(tS + 32, su + 32);
          tmem_ld_wait();
        }
        SA_TRACE_AT(trs, 1 + x, trn, tn << 16 | 23 << 8 | c);
        const int jc0 = it.jbeg + c * kChunk;
        int lo_c = jlo - jc0, hi_c = min(pos - jc0, w - 1);
        if (!valid) {
          lo_c = 1;
          hi_c = 0;
        }
        const bool need_mask = lo_c > 0 || hi_c < 63;
        // row max as an 8-way tree (independent chains, not one 64-long dependency)
        if (__any_sync(0xffffffffu, need_mask)) {
#pragma unroll
          for (int jj = 0; jj < 64; ++jj) sv[jj] = (jj >= lo_c && jj <= hi_c) ? sv[jj] : -INFINITY;
        }
        float mx;
        {
          float m8[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) m8[u] = fmaxf(fmaxf(sv[u], sv[u + 8]), fmaxf(sv[u + 16], sv[u + 24]));
#pragma unroll
          for (int u = 0; u < 8; ++u) m8[u] = fmaxf(m8[u], fmaxf(fmaxf(sv[u + 32], sv[u + 40]), fmaxf(sv[u + 48], sv[u + 56])));
          mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])), fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
        }
        mx *= a.sm_mult;  // sm_mult > 0: the max of the scaled logits
        if (c == 0) {
          m_ref = mx;
        } else {
          const bool need = mx > m_ref + kRescale;
          if (__any_sync(0xffffffffu, need)) {
            // U_x is stable: the commit that signalled S_x(c) covers PV_x(c-1)
            const float alpha = need ? ex2(m_ref - mx) : 1.f;
#pragma unroll
            for (int t = 0; t < D / 32; ++t) {
              uint32_t u[32];
              tmem_ld32(tU + 32 * t, u);
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 32; ++e) u[e] = __float_as_uint(__uint_as_float(u[e]) * alpha);
              tmem_st32(tU + 32 * t, u);
            }
            tmem_st_wait();
            if (need) {
              l *= alpha;
              m_ref = mx;
            }
          }
        }
        const float m_use = m_ref == -INFINITY ? 0.f : m_ref;
        uint32_t pk[32];
        const float2 vmul = make_float2(a.sm_mult, a.sm_mult), vm = make_float2(-m_use, -m_use);
        float2 ls4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          const float2 xx = ffma2(make_float2(sv[2 * t], sv[2 * t + 1]), vmul, vm);
          const float2 pv = (t & 7) == 7 ? ex2_poly2(xx) : make_float2(ex2(xx.x), ex2(xx.y));
          ls4[t & 3] = fadd2(ls4[t & 3], pv);  // 4 independent packed partial sums
          pk[t] = pack_f16x2(pv);
          if (t == 15 && w >= 32) tmem_st16(tS, pk);  // first 32 columns go out while the rest compute
        }
        const float ls = ((ls4[0].x + ls4[0].y) + (ls4[1].x + ls4[1].y)) + ((ls4[2].x + ls4[2].y) + (ls4[3].x + ls4[3].y));
        l += ls;  // columns >= w were masked to -inf above (need_mask holds whenever w < 64)
        SA_TRACE_AT(trs, 1 + x, trn, tn << 16 | 24 << 8 | c);
        if (w == 64) tmem_st16(tS + 16, pk + 16);
        if (w == 48) tmem_st8(tS + 16, pk + 16);
        if (w == 16) tmem_st8(tS, pk);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        named_bar_arrive(4 + x, 4 * 32 + 32);
        SA_TRACE_AT(trs, 1 + x, trn, tn << 16 | 25 << 8 | c);
      }

      // ---- A operand of the next pair (its first S MMAs then run during this pair's epilogue) ----
      if (nitem < a.items) {
        if constexpr (RS != 0) {
          if (STAGED) mbar_wait(&sm.stgfull[buf ^ 1], ((gc + 1) >> 1) & 1);
        } else {
          if (STAGED) cp_async_wait<0>();
        }
        named_bar_sync(3, 256);  // every softmax warp is past its last S wait: the A regions are free
        form_A(nitem, buf ^ 1);
      }
      // ---- epilogue: merge the R rows of each query, v2 o U, normalise ----
      mbar_wait(&sm.udone[x], gc & 1);
      tc_fence_after();
      SA_TRACE_AT(trs, 1 + x, trn, tn << 16 | 26 << 8);
      if constexpr (Sm::kRed) {
        // R = RS in {2, 4, 8, 16} (kernel instances of their own): a warp holds 32/R whole queries in
        // aligned groups of R lanes; group statistics by butterfly shuffles inside the group.  The
        // R-row sum o_i = sum_k (e^{m_k - M} / L) v2_k o U_k runs on the tensor core: each thread writes
        // its row's fp16 products X_r = (e^{m_r - M} / L) v2_r o U_r (zero for masked rows) into
        // shared memory, the MMA warp computes O^T = X^T Sel^T into TMEM (lane = column d, one TMEM
        // column per query), and each warp stores its 32 columns of every query.
        const bool live = valid && m_ref != -INFINITY;
        float M = live ? m_ref : -INFINITY;
        for (int o = RS >> 1; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        const float crow = live ? ex2(m_ref - M) : 0.f;
        float L = live ? l * crow : 0.f;
        for (int o = RS >> 1; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
        const bool qlive = g < nq;
        const int gl = lane & (RS - 1);  // lane within the query's group
        if (gl == 0 && qlive) a.lse[(int64_t(it.b) * p.H + it.h) * p.N + i0 + g] = (M + log2f(L)) * kLn2;
        const float sc = (live && L > 0.f) ? crow / L : 0.f;  // L = 0: an empty sub-window (split)
        uint8_t* xb = sm.xr[x];
        uint32_t u[32];
        tmem_ld32(tU, u);
#pragma unroll
        for (int cb = 0; cb < D / 32; ++cb) {
          tmem_ld_wait();
          uint32_t pk[16];
          if (sc != 0.f) {
            const uint4* vp = reinterpret_cast<const uint4*>(v2row + 32 * cb);
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const uint4 y = vp[t];
              const uint32_t ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 f = bf16x2_to_f2(ys[e]);
                pk[4 * t + e] = pack_f16x2(f.x * sc * __uint_as_float(u[8 * t + 2 * e]),
                                           f.y * sc * __uint_as_float(u[8 * t + 2 * e + 1]));
              }
            }
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) pk[e] = 0u;
          }
          if (cb + 1 < D / 32) tmem_ld32(tU + 32 * (cb + 1), u);
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int c8 = 4 * cb + t;  // 16-byte chunk: columns 8 c8 .. 8 c8 + 7 of row r
            *reinterpret_cast<uint4*>(xb + (c8 >> 3) * (128 * 128) + r * 128 + (((c8 & 7) ^ (r & 7)) << 4)) =
                make_uint4(pk[4 * t], pk[4 * t + 1], pk[4 * t + 2], pk[4 * t + 3]);
          }
        }
        fence_proxy_async_smem();  // generic-proxy stores -> visible to the tensor core
        tc_fence_before();
        named_bar_arrive(8 + x, 4 * 32 + 32);
        SA_TRACE_AT(trs, 1 + x, trn, tn << 16 | 30 << 8);
        mbar_wait(&sm.odone[x], gc & 1);
        tc_fence_after();
        SA_TRACE_AT(trs, 1 + x, trn, tn << 16 | 31 << 8);
        // O^T: this warp's lanes are columns d = 32 qd + lane; TMEM column q = query q of the tile
        constexpr int kG = 128 / RS;
        uint32_t ov[kNSel];
        if constexpr (kNSel >= 32) {
#pragma unroll
          for (int t = 0; t < kNSel / 32; ++t) tmem_ld32(tU + 32 * t, *reinterpret_cast<uint32_t(*)[32]>(ov + 32 * t));
        } else {
          tmem_ld16(tU, ov);
        }
        tmem_ld_wait();
        const int nqt = min(kG, nq);
        const int d = 32 * qd + lane;
        if (d < D) {
          const int64_t off0 = p.qoff(it.b, i0, it.h) + d, qstride = int64_t(p.H) * D;
#pragma unroll
          for (int q = 0; q < kG; ++q) {
            if (q < nqt) {
              const float val = __uint_as_float(ov[q]);
              if (a.out_f32)
                reinterpret_cast<float*>(a.o)[off0 + q * qstride] = val;
              else
                reinterpret_cast<__nv_bfloat16*>(a.o)[off0 + q * qstride] = __float2bfloat16_rn(val);
            }
          }
        }
      } else if (a.R == 32) {
        // one warp == one query: group statistics and the row reduction stay in the warp
        const bool live = valid && m_ref != -INFINITY;
        float M = live ? m_ref : -INFINITY;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        const float crow = live ? ex2(m_ref - M) : 0.f;
        float L = live ? l * crow : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
        const bool qlive = g < nq;
        if (lane == 0 && qlive) a.lse[(int64_t(it.b) * p.H + it.h) * p.N + i0 + g] = (M + log2f(L)) * kLn2;
        const float rs = qlive ? crow / L : 0.f;  // this row's weight e^{m_(i,k)-m_i} / l_i
        // 32-column blocks: a full reduce-scatter over the 32 lanes leaves column `lane` in lane
        // `lane`; the TMEM columns and v2 chunk of block cb+1 are requested before block cb's shuffles
        uint32_t u[32];
        uint4 y[4] = {};
        tmem_ld32(tU, u);
        if (valid) {
#pragma unroll
          for (int t = 0; t < 4; ++t) y[t] = *reinterpret_cast<const uint4*>(v2row + 8 * t);
        }
#pragma unroll
        for (int cb = 0; cb < D / 32; ++cb) {
          tmem_ld_wait();
          float v[32];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const uint32_t ys[4] = {y[t].x, y[t].y, y[t].z, y[t].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = bf16x2_to_f2(ys[e]);
              v[8 * t + 2 * e] = f.x * rs * __uint_as_float(u[8 * t + 2 * e]);
              v[8 * t + 2 * e + 1] = f.y * rs * __uint_as_float(u[8 * t + 2 * e + 1]);
            }
          }
          if (cb + 1 < D / 32) {
            tmem_ld32(tU + 32 * (cb + 1), u);
            if (valid) {
#pragma unroll
              for (int t = 0; t < 4; ++t) y[t] = *reinterpret_cast<const uint4*>(v2row + 32 * (cb + 1) + 8 * t);
            }
          }
#pragma unroll
          for (int st = 16, n = 16; st >= 1; st >>= 1, n >>= 1) {
            const bool hi = lane & st;
#pragma unroll
            for (int i = 0; i < n; ++i) {
              const float keep = hi ? v[n + i] : v[i], send = hi ? v[i] : v[n + i];
              v[i] = keep + __shfl_xor_sync(0xffffffffu, send, st);
            }
          }
          if (qlive) {
            const int64_t off = p.qoff(it.b, i0 + g, it.h) + 32 * cb + lane;
            if (a.out_f32)
              reinterpret_cast<float*>(a.o)[off] = v[0];
            else
              reinterpret_cast<__nv_bfloat16*>(a.o)[off] = __float2bfloat16_rn(v[0]);
          }
        }
      } else if (a.R < 32 && (a.R & (a.R - 1)) == 0 && a.R >= 2) {
        // (never taken: these R launch the RS instances.  Kept compiled because removing it changes
        // the register allocation of the R = 32 kernel, which measured ~2% slower without it.)
        // R in {2, 4, 8, 16}: a warp holds 32/R whole queries in aligned groups of R lanes; group
        // statistics by butterfly shuffles inside the group, the R-row sum of each 16-column block
        // by a reduce-scatter inside the group (each lane ends with 16/R columns of its query)
        const bool live = valid && m_ref != -INFINITY;
        float M = live ? m_ref : -INFINITY;
        for (int o = a.R >> 1; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        const float crow = live ? ex2(m_ref - M) : 0.f;
        float L = live ? l * crow : 0.f;
        for (int o = a.R >> 1; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
        const bool qlive = g < nq;
        const int gl = lane & (a.R - 1);  // lane within the query's group
        if (gl == 0 && qlive) a.lse[(int64_t(it.b) * p.H + it.h) * p.N + i0 + g] = (M + log2f(L)) * kLn2;
        const float invL = qlive ? 1.f / L : 0.f;
        const int nf = 16 / a.R;  // columns per lane after the reduce-scatter
        int cbase = 0;
        for (int k = 0, st = a.R >> 1; st > 0; ++k, st >>= 1)
          if (gl & st) cbase += 8 >> k;
#pragma unroll 1
        for (int cb = 0; cb < D / 16; ++cb) {
          uint32_t u[16];
          tmem_ld16(tU + 16 * cb, u);
          tmem_ld_wait();
          float v[16];
          if (valid) {
            if (STAGED) {
              const uint4* vp = reinterpret_cast<const uint4*>(v2row + 16 * cb);
#pragma unroll
              for (int t = 0; t < 2; ++t) {
                const uint4 y = vp[t];
                const uint32_t ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float2 f = bf16x2_to_f2(ys[e]);
                  v[8 * t + 2 * e] = f.x;
                  v[8 * t + 2 * e + 1] = f.y;
                }
              }
            } else {
              load_bf16<16>(v2row + 16 * cb, v);
            }
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] *= crow * __uint_as_float(u[e]);
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = 0.f;
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // stages st = R/2, R/4, ..., 1 with n = 8, 4, 2, 1 kept values
            const int st = (a.R >> 1) >> k, n = 8 >> k;
            if (st > 0) {
              const bool hi = gl & st;
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                if (i < n) {
                  const float keep = hi ? v[n + i] : v[i], send = hi ? v[i] : v[n + i];
                  v[i] = keep + __shfl_xor_sync(0xffffffffu, send, st);
                }
              }
            }
          }
          if (qlive) {
            const int64_t off = p.qoff(it.b, i0 + g, it.h) + 16 * cb + cbase;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if (i < nf) {
                if (a.out_f32)
                  reinterpret_cast<float*>(a.o)[off + i] = v[i] * invL;
                else
                  reinterpret_cast<__nv_bfloat16*>(a.o)[off + i] = __float2bfloat16_rn(v[i] * invL);
              }
            }
          }
        }
      } else if (a.R == 64 || a.R == 128) {
        // one query == two warps (R = 64: lane quarters qd, qd^1) or all four (R = 128): warp-level
        // statistics by shuffles, the other warps' partials through shared memory; each warp
        // reduce-scatters its 32 rows, the query's lead warp adds the others' column partials
        const bool r128 = a.R == 128;
        const bool live = valid && m_ref != -INFINITY;
        float M = live ? m_ref : -INFINITY;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        if (lane == 0) sm.gM[x][qd] = M;
        named_bar_sync(1 + x, 128);
        M = r128 ? fmaxf(fmaxf(sm.gM[x][0], sm.gM[x][1]), fmaxf(sm.gM[x][2], sm.gM[x][3]))
                 : fmaxf(M, sm.gM[x][qd ^ 1]);
        const float crow = live ? ex2(m_ref - M) : 0.f;
        float L = live ? l * crow : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
        if (lane == 0) sm.gL[x][qd] = L;
        named_bar_sync(1 + x, 128);
        L = r128 ? (sm.gL[x][0] + sm.gL[x][1]) + (sm.gL[x][2] + sm.gL[x][3]) : L + sm.gL[x][qd ^ 1];
        const bool qlive = g < nq;
        const bool lead = r128 ? qd == 0 : (qd & 1) == 0;
        if (lead && lane == 0 && qlive) a.lse[(int64_t(it.b) * p.H + it.h) * p.N + i0 + g] = (M + log2f(L)) * kLn2;
        const float invL = qlive ? 1.f / L : 0.f;
        // 32-column blocks as in the R = 32 path (column `lane` in lane `lane` after the reduce-
        // scatter); the other warps' column partials go through ebuf (flat, 32 per warp, double-
        // buffered by block parity), one barrier per block
        float* ebf = &sm.ebuf[x][0][0];
        uint32_t u[32];
        uint4 y[4] = {};
        tmem_ld32(tU, u);
        if (valid) {
#pragma unroll
          for (int t = 0; t < 4; ++t) y[t] = *reinterpret_cast<const uint4*>(v2row + 8 * t);
        }
#pragma unroll
        for (int cb = 0; cb < D / 32; ++cb) {
          tmem_ld_wait();
          float v[32];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const uint32_t ys[4] = {y[t].x, y[t].y, y[t].z, y[t].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = bf16x2_to_f2(ys[e]);
              v[8 * t + 2 * e] = f.x * crow * __uint_as_float(u[8 * t + 2 * e]);
              v[8 * t + 2 * e + 1] = f.y * crow * __uint_as_float(u[8 * t + 2 * e + 1]);
            }
          }
          if (cb + 1 < D / 32) {
            tmem_ld32(tU + 32 * (cb + 1), u);
            if (valid) {
#pragma unroll
              for (int t = 0; t < 4; ++t) y[t] = *reinterpret_cast<const uint4*>(v2row + 32 * (cb + 1) + 8 * t);
            }
          }
#pragma unroll
          for (int st = 16, n = 16; st >= 1; st >>= 1, n >>= 1) {
            const bool hi = lane & st;
#pragma unroll
            for (int i = 0; i < n; ++i) {
              const float keep = hi ? v[n + i] : v[i], send = hi ? v[i] : v[n + i];
              v[i] = keep + __shfl_xor_sync(0xffffffffu, send, st);
            }
          }
          float* part = ebf + ((cb & 1) * 4) * 32;
          if (!lead) part[qd * 32 + lane] = v[0];
          named_bar_sync(1 + x, 128);
          if (lead && qlive) {
            const float yv = r128 ? v[0] + (part[32 + lane] + part[64 + lane]) + part[96 + lane]
                                  : v[0] + part[(qd ^ 1) * 32 + lane];
            const int64_t off = p.qoff(it.b, i0 + g, it.h) + 32 * cb + lane;
            if (a.out_f32)
              reinterpret_cast<float*>(a.o)[off] = yv * invL;
            else
              reinterpret_cast<__nv_bfloat16*>(a.o)[off] = __float2bfloat16_rn(yv * invL);
          }
        }
      } else {
        sm.rm[x][r] = valid ? m_ref : -INFINITY;
        sm.rl[x][r] = valid ? l : 0.f;
        named_bar_sync(1 + x, 128);
        if (r < nq) {
          float M = -INFINITY;
          for (int t = 0; t < a.R; ++t) M = fmaxf(M, sm.rm[x][r * a.R + t]);
          float L = 0.f;
          for (int t = 0; t < a.R; ++t) {
            const float mt = sm.rm[x][r * a.R + t];
            if (mt != -INFINITY) L += sm.rl[x][r * a.R + t] * ex2(mt - M);
          }
          sm.gM[x][r] = M;
          sm.gL[x][r] = L;
          a.lse[(int64_t(it.b) * p.H + it.h) * p.N + i0 + r] = (M + log2f(L)) * kLn2;
        }
        named_bar_sync(1 + x, 128);
        const float crow = (valid && m_ref != -INFINITY) ? ex2(m_ref - sm.gM[x][g]) : 0.f;
        float(*eb)[17] = sm.ebuf[x];
#pragma unroll 1
        for (int cb = 0; cb < D / 16; ++cb) {
          uint32_t u[16];
          tmem_ld16(tU + 16 * cb, u);
          tmem_ld_wait();
          float vv[16];
          if (valid) {
            load_bf16<16>(v2row + 16 * cb, vv);
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) vv[e] = 0.f;
          }
#pragma unroll
          for (int e = 0; e < 16; ++e) eb[r][e] = crow * vv[e] * __uint_as_float(u[e]);
          named_bar_sync(1 + x, 128);
          // nq x 16 outputs, 4 lanes per output over interleaved rows, shuffle-combined
          for (int base = 0; base < nq * 16 * 4; base += 128) {
            const int idx = base + r;
            const bool act = idx < nq * 16 * 4;
            const int oo = idx >> 2, part = idx & 3;
            const int gq = oo >> 4, d = oo & 15;
            float y0 = 0.f, y1 = 0.f;
            if (act) {
              int t = part;
              for (; t + 4 < a.R; t += 8) {
                y0 += eb[gq * a.R + t][d];
                y1 += eb[gq * a.R + t + 4][d];
              }
              if (t < a.R) y0 += eb[gq * a.R + t][d];
            }
            float y = y0 + y1;
            y += __shfl_xor_sync(0xffffffffu, y, 1);
            y += __shfl_xor_sync(0xffffffffu, y, 2);
            if (act && part == 0) {
              const float val = y / sm.gL[x][gq];
              const int64_t off = p.qoff(it.b, i0 + gq, it.h) + 16 * cb + d;
              if (a.out_f32)
                reinterpret_cast<float*>(a.o)[off] = val;
              else
                reinterpret_cast<__nv_bfloat16*>(a.o)[off] = __float2bfloat16_rn(val);
            }
          }
          named_bar_sync(1 + x, 128);
        }
      }
      tc_fence_before();
      SA_TRACE_AT(trs, 1 + x, trn, tn << 16 | 27 << 8);
      cc += it.nch;
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

// Window split (sa_split.cu) of a long folded window: sub-problems of <= 32 K' rows whose (o_b, lse_b)
// are merged exactly.  Taken for every w2 > 32: the R = 32 kernel instance (TMA row staging) runs two
// sub-windows faster than one R = 64 tiling (Table 1 (512, 64): 13.7 vs 15.5 ms forward; DESIGN.md
// "window split").  SA_NO_WSPLIT=1 never splits (SA_FWD_WSPLIT is accepted and has no effect).
static int fwd_split_count(const Problem& p) {
  static const bool off = getenv("SA_NO_WSPLIT") && atoi(getenv("SA_NO_WSPLIT")) != 0;
  static const bool all = getenv("SA_FWD_WSPLIT") && atoi(getenv("SA_FWD_WSPLIT")) != 0;
  const int w2 = swapped(p) ? p.w1 : p.w2, w1 = swapped(p) ? p.w2 : p.w1;
  if (off || w2 <= 32) return 1;
  (void)w1;
  (void)all;
  return (w2 + 31) / 32;
}
static size_t fa256(size_t x) { return (x + 255) & ~size_t(255); }

size_t tc_fwd_workspace_bytes(const Problem& p) {
  const size_t n = p.nkey(), nq = size_t(p.B) * p.N * p.H * p.D;
  const int ns = fwd_split_count(p);
  // split partials: ns o_b (fp32, nq floats each) then ns lse_b (B H N floats each), packed
  const size_t parts = ns > 1 ? fa256(4 * size_t(ns) * nq) + fa256(4 * size_t(ns) * p.B * p.H * p.N) : 0;
  return 3 * fa256(n * 2) + fa256(nq * 2) + parts;
}

static cudaError_t fwd_core(const Problem& p, bool out_f32, const char* kf, const char* vf, const char* k2f,
                            const char* qf, const void* v2, void* o, float* lse, cudaStream_t st);
cudaError_t split_merge(const float* ob, const float* lb, int nsplit, const Problem& p, void* o, float* lse,
                        bool out_f32, cudaStream_t st);

cudaError_t tc_forward_ws(const Problem& p0, bool out_f32, const void* q, const void* k, const void* v,
                          const void* k2, const void* v2, void* o, float* lse, void* ws, cudaStream_t st) {
  Problem p = p0;
  const int ns = fwd_split_count(p0);
  if (swapped(p)) {  // fold the smaller-window key into the query (exact symmetry; det negates)
    std::swap(k, k2);
    std::swap(v, v2);
    std::swap(p.w1, p.w2);
    if (p.det) p.scale = -p.scale;
  }
  const size_t n = p.nkey();
  const size_t nq = size_t(p.B) * p.N * p.H * p.D;
  char* kf = (char*)ws;
  char* vf = kf + fa256(n * 2);
  char* k2f = vf + fa256(n * 2);
  char* qf = k2f + fa256(n * 2);
  cudaError_t e = convert_pair_f16(k, kf, v, vf, int64_t(n), num_sms(), st);
  if (e == cudaSuccess) e = convert_two_f16(q, qf, int64_t(nq), k2, k2f, int64_t(n), num_sms(), st);
  if (e != cudaSuccess) return e;
  if (ns == 1) return fwd_core(p, out_f32, kf, vf, k2f, qf, v2, o, lse, st);
  // window split: sub-problem b (K' offsets [32 b, 32 b + w_b) back from the query) sees K', V'
  // through pointers shifted by -32 b rows; its (o_b fp32, lse_b) are merged exactly
  char* parts = qf + fa256(nq * 2);
  const size_t nl = size_t(p.B) * p.H * p.N;
  const int64_t kstep = int64_t(p.Hk) * p.D;
  for (int b = 0; b < ns && e == cudaSuccess; ++b) {
    Problem sp = p;
    sp.k2lo = 32 * b;
    sp.w2 = std::min(32, p.w2 - 32 * b);
    float* ob = (float*)parts + size_t(b) * nq;
    float* lb = (float*)(parts + fa256(4 * size_t(ns) * nq)) + size_t(b) * nl;
    e = fwd_core(sp, true, kf, vf, (const char*)((const __half*)k2f - sp.k2lo * kstep),
                 qf, (const __nv_bfloat16*)v2 - sp.k2lo * kstep, ob, lb, st);
  }
  if (e == cudaSuccess)
    e = split_merge((const float*)parts, (const float*)(parts + fa256(4 * size_t(ns) * nq)), ns, p, o, lse, out_f32,
                    st);
  return e;
}

static cudaError_t fwd_core(const Problem& p, bool out_f32, const char* kf, const char* vf, const char* k2f,
                            const char* qf, const void* v2, void* o, float* lse, cudaStream_t st) {
  CUtensorMap tmK, tmV;
  if (!make_tmap_bnhd_f16(&tmK, kf, p.B, p.NK(), p.Hk, p.D, kChunk) ||
      !make_tmap_bnhd_f16(&tmV, vf, p.B, p.NK(), p.Hk, p.D, kChunk))
    return cudaErrorInvalidValue;
  FwdArgs a;
  a.p = p;
  a.q = (const __half*)qf;
  a.k2 = (const __half*)k2f;
  a.v2 = (const __nv_bfloat16*)v2;
  a.o = o;
  a.lse = lse;
  a.out_f32 = out_f32 ? 1 : 0;
  a.R = p.w2;
  a.G = 128 / p.w2;
  a.ngroups = (p.N + a.G - 1) / a.G;
  a.npairs = (a.ngroups + 1) / 2;
  a.items = a.npairs * p.B * p.H;
  a.det_neg = p.det && p.scale < 0.f ? 1 : 0;
  a.sm_mult = fabsf(p.scale) * kLog2e;
  const int grid = std::min(a.items, num_sms());
  // kernel instances: R in {2, 4, 8, 16} (tensor-core row-group sums, TMA row staging), R = 32 (TMA row
  // staging, SA_FWD_R32_TMA=0 keeps the generic instance's cp.async staging), other R (generic)
  static const bool r32_off = getenv("SA_FWD_R32_TMA") && atoi(getenv("SA_FWD_R32_TMA")) == 0;
  const int rs = (a.R < 32 && a.R >= 2 && (a.R & (a.R - 1)) == 0) ? a.R : (a.R == 32 && !r32_off) ? 32 : 0;
  const int nk2 = a.R + 2 * a.G - 1;
  const bool staged = 2 * a.G + (rs ? ((nk2 + 7) & ~7) : nk2) + nk2 <= kStgRows;
  // pitched-row staging maps of the RS kernels (on the unshifted K', V' of a window-split sub-problem)
  CUtensorMap tmQs = tmK, tmK2s = tmK, tmV2s = tmK;
  a.tma_stage = rs && staged && p.H >= 2 && p.Hk >= 2;  // a pitched box of D + 8 columns needs a next head
  if (a.tma_stage) {
    const int64_t kshift = int64_t(p.k2lo) * p.Hk * p.D;
    if (!make_tmap_rows_pitched(&tmQs, qf, p.B, p.N, p.H * p.D, p.D, 2 * a.G) ||
        !make_tmap_rows_pitched(&tmK2s, (const __half*)k2f + kshift, p.B, p.NK(), p.Hk * p.D, p.D, nk2) ||
        !make_tmap_rows_pitched(&tmV2s, (const __nv_bfloat16*)v2 + kshift, p.B, p.NK(), p.Hk * p.D, p.D, nk2))
      return cudaErrorInvalidValue;
  }
  auto launch = [&](auto kern, size_t smem) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    KernelScope ks("tc_fwd", st);
    kern<<<grid, kThreads, smem, st>>>(tmK, tmV, tmQs, tmK2s, tmV2s, a);
  };
  auto pick = [&](auto dc, auto sc) {
    constexpr int Dc = decltype(dc)::value;
    constexpr bool Sc = decltype(sc)::value;
    switch (rs) {
      case 2: launch(tc_fwd_kernel<Dc, Sc, 2>, sizeof(Smem<Dc, 2>) + 1024); break;
      case 4: launch(tc_fwd_kernel<Dc, Sc, 4>, sizeof(Smem<Dc, 4>) + 1024); break;
      case 8: launch(tc_fwd_kernel<Dc, Sc, 8>, sizeof(Smem<Dc, 8>) + 1024); break;
      case 16: launch(tc_fwd_kernel<Dc, Sc, 16>, sizeof(Smem<Dc, 16>) + 1024); break;
      case 32: launch(tc_fwd_kernel<Dc, Sc, 32>, sizeof(Smem<Dc, 32>) + 1024); break;
      default: launch(tc_fwd_kernel<Dc, Sc, 0>, sizeof(Smem<Dc, 0>) + 1024); break;
    }
  };
  using I128 = std::integral_constant<int, 128>;
  using I64 = std::integral_constant<int, 64>;
  using T = std::true_type;
  using F = std::false_type;
  if (p.D == 128)
    staged ? pick(I128{}, T{}) : pick(I128{}, F{});
  else
    staged ? pick(I64{}, T{}) : pick(I64{}, F{});
  return cudaGetLastError();
}

}  // namespace sa

// sa_api.cu -- the C ABI (include/simplicial_attn.h): validation, kernel selection, launches.
#include <atomic>
#include <math.h>
#include <stdlib.h>

#include <algorithm>
#include <mutex>
#include <stdio.h>
#include <string.h>
#include <string>
#include <vector>

#include "sa_common.cuh"

namespace sa {

#ifdef SA_TRACE
__device__ unsigned long long g_trace[8192];
__device__ unsigned int g_trace_n;
#endif

static std::atomic<uint64_t> g_launches{0};
void note_launch(int n) { g_launches.fetch_add(uint64_t(n), std::memory_order_relaxed); }

// ---- per-kernel event timing (simplicial_attn_profile_*) ----
struct ProfRec {
  std::string name;
  cudaEvent_t a, b;
};
static std::atomic<int> g_prof_on{0};
static std::mutex g_prof_mu;
static std::vector<ProfRec> g_prof;

static std::vector<cudaEvent_t> g_event_pool;  // recycled by simplicial_attn_profile_read
static cudaEvent_t pooled_event() {
  cudaEvent_t e = nullptr;
  {
    std::lock_guard<std::mutex> g(g_prof_mu);
    if (!g_event_pool.empty()) {
      e = g_event_pool.back();
      g_event_pool.pop_back();
    }
  }
  if (!e) cudaEventCreate(&e);
  return e;
}

KernelScope::KernelScope(const char* name, cudaStream_t s) : slot(-1), st(s) {
  note_launch(1);
  if (!g_prof_on.load(std::memory_order_relaxed)) return;
  ProfRec r{name, pooled_event(), pooled_event()};
  cudaEventRecord(r.a, st);
  std::lock_guard<std::mutex> g(g_prof_mu);
  slot = int(g_prof.size());
  g_prof.push_back(r);
}
KernelScope::~KernelScope() {
  if (slot < 0) return;
  cudaEvent_t e;
  {
    std::lock_guard<std::mutex> g(g_prof_mu);
    e = g_prof[slot].b;
  }
  cudaEventRecord(e, st);
}

cudaError_t simt_forward(const Problem& p, bool in_f32, bool out_f32, const void* q, const void* k,
                         const void* v, const void* k2, const void* v2, void* o, float* lse, cudaStream_t st);
cudaError_t simt_backward(const Problem& p, bool in_f32, bool out_f32, const void* q, const void* k,
                          const void* v, const void* k2, const void* v2, const void* o, const float* lse,
                          const void* dO, void* dq, void* dk, void* dv, void* dk2, void* dv2, float* delta,
                          cudaStream_t st);

// tcgen05 path (sa_tc_fwd.cu / sa_tc_bwd.cu)
bool tc_fwd_supported(const Problem& p);
size_t tc_fwd_workspace_bytes(const Problem& p);
cudaError_t tc_forward_ws(const Problem& p, bool out_f32, const void* q, const void* k, const void* v,
                          const void* k2, const void* v2, void* o, float* lse, void* ws, cudaStream_t st);
bool tc_bwd_supported(const Problem& p);
size_t tc_bwd_workspace_bytes(const Problem& p);
cudaError_t tc_backward(const Problem& p, bool out_f32, const void* q, const void* k, const void* v,
                        const void* k2, const void* v2, const void* o, const float* lse, const void* dO,
                        void* dq, void* dk, void* dv, void* dk2, void* dv2, void* ws, size_t ws_bytes,
                        cudaStream_t st);

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// Validate scalar arguments; fill the Problem.  Rejects before any launch.
static sa_status make_problem(int64_t B, int64_t H, int64_t N, int64_t D, int64_t w1, int64_t w2,
                              int64_t n_prefix, uint32_t flags, Problem* p) {
  if (B < 1 || H < 1 || N < 1 || D < 1 || w1 < 1 || w2 < 1 || n_prefix < 0) return SA_ERR_INVALID_ARG;
  if ((flags & SA_VARIANT_DET) && D < 3) return SA_ERR_INVALID_ARG;
  if (flags & ~uint32_t(SA_VARIANT_DET | SA_IN_F32 | SA_OUT_F32 | SA_FORCE_SIMT)) return SA_ERR_INVALID_ARG;
  if (D > 128) return SA_ERR_UNSUPPORTED;
  int64_t NK = n_prefix + N;
  if (NK > (int64_t(1) << 30) || B * H > 65535 || NK > 2147483647 / 4) return SA_ERR_UNSUPPORTED;
  // windows longer than the key buffer clamp
  if (w1 > NK) w1 = NK;
  if (w2 > NK) w2 = NK;
  p->B = int(B); p->H = int(H); p->N = int(N); p->D = int(D);
  p->w1 = int(w1); p->w2 = int(w2); p->np = int(n_prefix);
  p->Hk = int(H);
  p->hk_shift = 0;
  p->k2lo = 0;
  p->det = (flags & SA_VARIANT_DET) != 0;
  p->scale = float(1.0 / sqrt(double(D)));
  return SA_OK;
}

// Grouped-query problem: H query heads, Hk key/value heads, Hk | H (query head h reads key head
// h / (H / Hk)).
static sa_status make_problem_gqa(int64_t B, int64_t H, int64_t Hk, int64_t N, int64_t D, int64_t w1, int64_t w2,
                                  uint32_t flags, Problem* p) {
  sa_status s = make_problem(B, H, N, D, w1, w2, 0, flags, p);
  if (s != SA_OK) return s;
  if (Hk < 1 || Hk > H || H % Hk != 0) return SA_ERR_INVALID_ARG;
  p->Hk = int(Hk);
  const int64_t r = H / Hk;
  p->hk_shift = (r & (r - 1)) == 0 ? __builtin_ctzll(uint64_t(r)) : -1;
  return SA_OK;
}

cudaError_t gqa_reduce(const float* part, void* out, bool out_f32, int64_t rows, int Hk, int r, int D,
                       cudaStream_t st);
cudaError_t cast_f32_bf16(const float* a, void* b, int64_t n, cudaStream_t st);
cudaError_t cast_bf16_f32(const void* a, float* b, int64_t n, cudaStream_t st);
cudaError_t add_bias(const void* k2, const void* v2, void* k2b, void* v2b, int64_t n, bool f32, float b2k,
                     float b2v, cudaStream_t st);

static bool use_tc_fwd(const Problem& p, uint32_t flags) {
  if (flags & (SA_IN_F32 | SA_FORCE_SIMT)) return false;
  return tc_fwd_supported(p);
}
static bool use_tc_bwd(const Problem& p, uint32_t flags) {
  if (flags & (SA_IN_F32 | SA_FORCE_SIMT)) return false;
  return tc_bwd_supported(p);
}

// Kernel family for a call: fp32 inputs (SA_IN_F32) and the SA_FORCE_SIMT diagnostic take the exact
// CUDA-core kernels; bf16 inputs take the tcgen05 kernels or are rejected (SA_ERR_UNSUPPORTED) --
// there is no silent fallback to another backend.
enum class Route { TC, SIMT, NONE };
static Route route(const Problem& p, uint32_t flags, bool bwd) {
  if (flags & (SA_IN_F32 | SA_FORCE_SIMT)) return Route::SIMT;
  return (bwd ? tc_bwd_supported(p) : tc_fwd_supported(p)) ? Route::TC : Route::NONE;
}

static size_t bwd_ws(const Problem& p, uint32_t flags) {
  size_t base = align256(sizeof(float) * size_t(p.B) * p.H * p.N);  // delta
  if (use_tc_bwd(p, flags)) base += align256(tc_bwd_workspace_bytes(p));
  return base;
}

static sa_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return SA_OK;
  fprintf(stderr, "[simplicial_attn] CUDA error: %s\n", cudaGetErrorString(e));
  return SA_ERR_CUDA;
}

}  // namespace sa

using namespace sa;

extern "C" {

size_t simplicial_attn_fwd_workspace_bytes_prefixed(int64_t B, int64_t H, int64_t N, int64_t D, int64_t w1,
                                                    int64_t w2, int64_t n_prefix, uint32_t flags) {
  Problem p;
  if (make_problem(B, H, N, D, w1, w2, n_prefix, flags, &p) != SA_OK) return 0;
  return use_tc_fwd(p, flags) ? tc_fwd_workspace_bytes(p) : 0;
}

size_t simplicial_attn_fwd_workspace_bytes(int64_t B, int64_t H, int64_t N, int64_t D, int64_t w1, int64_t w2,
                                           uint32_t flags) {
  return simplicial_attn_fwd_workspace_bytes_prefixed(B, H, N, D, w1, w2, 0, flags);
}

sa_status simplicial_attn_fwd_prefixed(const void* q, const void* k, const void* v, const void* k2, const void* v2,
                                       void* o, float* lse, void* workspace, size_t workspace_bytes, int64_t B,
                                       int64_t H, int64_t N, int64_t D, int64_t w1, int64_t w2, int64_t n_prefix,
                                       uint32_t flags, void* stream) {
  if (!q || !k || !v || !k2 || !v2 || !o || !lse) return SA_ERR_INVALID_ARG;
  Problem p;
  sa_status s = make_problem(B, H, N, D, w1, w2, n_prefix, flags, &p);
  if (s != SA_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  bool in_f32 = flags & SA_IN_F32, out_f32 = in_f32 || (flags & SA_OUT_F32);
  cudaGetLastError();  // clear stale errors so a failure below is ours
  switch (route(p, flags, false)) {
    case Route::TC:
      if (!workspace || workspace_bytes < tc_fwd_workspace_bytes(p)) return SA_ERR_WORKSPACE;
      return cuda_status(tc_forward_ws(p, out_f32, q, k, v, k2, v2, o, lse, workspace, st));
    case Route::SIMT:
      return cuda_status(simt_forward(p, in_f32, out_f32, q, k, v, k2, v2, o, lse, st));
    default:
      return SA_ERR_UNSUPPORTED;
  }
}

sa_status simplicial_attn_fwd(const void* q, const void* k, const void* v, const void* k2, const void* v2,
                              void* o, float* lse, void* workspace, size_t workspace_bytes, int64_t B, int64_t H,
                              int64_t N, int64_t D, int64_t w1, int64_t w2, uint32_t flags, void* stream) {
  return simplicial_attn_fwd_prefixed(q, k, v, k2, v2, o, lse, workspace, workspace_bytes, B, H, N, D, w1, w2, 0,
                                      flags, stream);
}

size_t simplicial_attn_bwd_workspace_bytes_prefixed(int64_t B, int64_t H, int64_t N, int64_t D, int64_t w1,
                                                    int64_t w2, int64_t n_prefix, uint32_t flags) {
  Problem p;
  if (make_problem(B, H, N, D, w1, w2, n_prefix, flags, &p) != SA_OK) return 0;
  return bwd_ws(p, flags);
}

size_t simplicial_attn_bwd_workspace_bytes(int64_t B, int64_t H, int64_t N, int64_t D, int64_t w1, int64_t w2,
                                           uint32_t flags) {
  return simplicial_attn_bwd_workspace_bytes_prefixed(B, H, N, D, w1, w2, 0, flags);
}

sa_status simplicial_attn_bwd_prefixed(const void* q, const void* k, const void* v, const void* k2,
                                       const void* v2, const void* o, const float* lse, const void* dO,
                                       void* dq, void* dk, void* dv, void* dk2, void* dv2, void* workspace,
                                       size_t workspace_bytes, int64_t B, int64_t H, int64_t N, int64_t D,
                                       int64_t w1, int64_t w2, int64_t n_prefix, uint32_t flags,
                                       void* stream) {
  if (!q || !k || !v || !k2 || !v2 || !o || !lse || !dO || !dq || !dk || !dv || !dk2 || !dv2 || !workspace)
    return SA_ERR_INVALID_ARG;
  Problem p;
  sa_status s = make_problem(B, H, N, D, w1, w2, n_prefix, flags, &p);
  if (s != SA_OK) return s;
  if (route(p, flags, true) == Route::NONE) return SA_ERR_UNSUPPORTED;
  if (workspace_bytes < bwd_ws(p, flags)) return SA_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  bool in_f32 = flags & SA_IN_F32, out_f32 = in_f32 || (flags & SA_OUT_F32);
  float* delta = (float*)workspace;
  cudaGetLastError();
  switch (route(p, flags, true)) {
    case Route::TC:  // workspace: delta first, then the tcgen05 kernels' scratch
      return cuda_status(tc_backward(p, out_f32, q, k, v, k2, v2, o, lse, dO, dq, dk, dv, dk2, dv2, workspace,
                                     workspace_bytes, st));
    case Route::SIMT:
      return cuda_status(simt_backward(p, in_f32, out_f32, q, k, v, k2, v2, o, lse, dO, dq, dk, dv, dk2, dv2,
                                       delta, st));
    default:
      return SA_ERR_UNSUPPORTED;
  }
}

sa_status simplicial_attn_bwd(const void* q, const void* k, const void* v, const void* k2, const void* v2,
                              const void* o, const float* lse, const void* dO, void* dq, void* dk, void* dv,
                              void* dk2, void* dv2, void* workspace, size_t workspace_bytes, int64_t B,
                              int64_t H, int64_t N, int64_t D, int64_t w1, int64_t w2, uint32_t flags,
                              void* stream) {
  return simplicial_attn_bwd_prefixed(q, k, v, k2, v2, o, lse, dO, dq, dk, dv, dk2, dv2, workspace,
                                      workspace_bytes, B, H, N, D, w1, w2, 0, flags, stream);
}

// Device scratch layout of the host step: 6 inputs | o | lse | 5 grads | fwd/bwd workspace (shared:
// the forward's scratch is dead once the backward starts on the same stream).
// Copy streams and events of the pipelined host step: one set per device, created on first use and
// guarded by a per-device mutex that simplicial_attn_host_step holds for its whole enqueue, so
// concurrent calls on one device never re-record each other's events.
struct HostPipe {
  bool ok = false;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t entry = nullptr, out = nullptr;
  // per chunk: forward inputs landed, dO landed, forward done (o, lse downloadable), backward done
  std::vector<cudaEvent_t> in, in_b, fdone, done;
  std::mutex mu;
};
static HostPipe& host_pipe_of(int dev) {
  static HostPipe pipes[64];
  return pipes[dev & 63];
}
// Caller holds hp.mu.
static bool host_pipe_reserve(HostPipe& hp, int nchunks) {
  if (!hp.h2d) {
    hp.ok = cudaStreamCreateWithFlags(&hp.h2d, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&hp.d2h, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&hp.entry, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&hp.out, cudaEventDisableTiming) == cudaSuccess;
  }
  while (hp.ok && int(hp.in.size()) < nchunks) {
    cudaEvent_t ev[4];
    for (auto& x : ev) hp.ok = hp.ok && cudaEventCreateWithFlags(&x, cudaEventDisableTiming) == cudaSuccess;
    if (!hp.ok) break;
    hp.in.push_back(ev[0]);
    hp.in_b.push_back(ev[1]);
    hp.fdone.push_back(ev[2]);
    hp.done.push_back(ev[3]);
  }
  return hp.ok;
}

static size_t host_step_layout(const Problem& p, uint32_t flags, size_t off[16]) {
  bool in_f32 = flags & SA_IN_F32, out_f32 = in_f32 || (flags & SA_OUT_F32);
  size_t ein = in_f32 ? 4 : 2, eout = out_f32 ? 4 : 2;
  size_t nel = size_t(p.B) * p.N * p.H * p.D;
  size_t cur = 0;
  for (int t = 0; t < 6; ++t) { off[t] = cur; cur += align256(nel * ein); }
  off[6] = cur; cur += align256(nel * eout);                               // o
  off[7] = cur; cur += align256(sizeof(float) * size_t(p.B) * p.H * p.N);  // lse
  for (int t = 8; t < 13; ++t) { off[t] = cur; cur += align256(nel * eout); }
  off[13] = cur;
  {
    size_t fw = 0;
    Problem c = p;  // the step runs per chunk of (1, hc <= H) slices: size for the whole problem (an upper bound)
    if (route(c, flags, false) == Route::TC) fw = tc_fwd_workspace_bytes(c);
    const size_t bw = bwd_ws(p, flags);
    cur += align256(fw > bw ? fw : bw);
  }
  off[14] = cur;
  return cur;
}

size_t simplicial_attn_host_step_scratch_bytes(int64_t B, int64_t H, int64_t N, int64_t D, int64_t w1,
                                               int64_t w2, uint32_t flags) {
  Problem p;
  if (make_problem(B, H, N, D, w1, w2, 0, flags, &p) != SA_OK) return 0;
  size_t off[16];
  return host_step_layout(p, flags, off);
}

sa_status simplicial_attn_host_step(const void* h_q, const void* h_k, const void* h_v, const void* h_k2,
                                    const void* h_v2, const void* h_dO, void* h_o, float* h_lse, void* h_dq,
                                    void* h_dk, void* h_dv, void* h_dk2, void* h_dv2, void* d_scratch,
                                    size_t scratch_bytes, int64_t B, int64_t H, int64_t N, int64_t D,
                                    int64_t w1, int64_t w2, uint32_t flags, void* stream) {
  const void* hin[6] = {h_q, h_k, h_v, h_k2, h_v2, h_dO};
  void* hout[5] = {h_dq, h_dk, h_dv, h_dk2, h_dv2};
  for (auto x : hin) if (!x) return SA_ERR_INVALID_ARG;
  for (auto x : hout) if (!x) return SA_ERR_INVALID_ARG;
  if (!h_o || !h_lse || !d_scratch) return SA_ERR_INVALID_ARG;
  Problem p;
  sa_status s = make_problem(B, H, N, D, w1, w2, 0, flags, &p);
  if (s != SA_OK) return s;
  size_t off[16];
  size_t need = host_step_layout(p, flags, off);
  if (scratch_bytes < need) return SA_ERR_WORKSPACE;
  bool in_f32 = flags & SA_IN_F32, out_f32 = in_f32 || (flags & SA_OUT_F32);
  const size_t nel = size_t(p.B) * p.N * p.H * p.D;
  // Pipeline chunks: (batch b, heads [h0, h0+hc)).  Every (b,h) slice is independent.  Only
  // the first upload and the last download are exposed, so the first batch element is cut into head
  // groups that double (1, 2, 4, ... heads: each group's upload, ~2x faster per head than its compute,
  // hides behind the previous group) and the last batch element into groups that halve; the other
  // batch elements go whole (full-size launches: a 2-head chunk leaves SMs idle in bwd_kv, whose grid
  // is key blocks x heads).  SA_HOSTSTEP_SPLIT=0: whole batch elements only.
  struct Chunk {
    int64_t b, h0, hc;
  };
  std::vector<Chunk> chunks;
  static const bool no_split = getenv("SA_HOSTSTEP_SPLIT") && atoi(getenv("SA_HOSTSTEP_SPLIT")) == 0;
  auto doubling = [&](int64_t n) {  // 1, 2, 4, ... then the remainder folded into the last group
    std::vector<int64_t> g;
    int64_t left = n, sz = 1;
    while (left > 0) {
      if (2 * sz > left - sz) {  // the next doubling would not fit: take what is left
        g.push_back(left);
        break;
      }
      g.push_back(sz);
      left -= sz;
      sz *= 2;
    }
    return g;
  };
  for (int64_t b = 0; b < B; ++b) {
    std::vector<int64_t> g;
    if (no_split || (b > 0 && b < B - 1)) {
      g = {H};
    } else if (B == 1) {  // first and last: grow, then shrink
      const std::vector<int64_t> up = doubling((H + 1) / 2);
      std::vector<int64_t> dn = doubling(H - (H + 1) / 2);
      g = up;
      for (auto it = dn.rbegin(); it != dn.rend(); ++it) g.push_back(*it);
    } else {
      g = doubling(H);
      if (b == B - 1) std::reverse(g.begin(), g.end());
    }
    int64_t h0 = 0;
    for (int64_t hc : g) {
      if (hc <= 0) continue;
      chunks.push_back({b, h0, hc});
      h0 += hc;
    }
  }
  const size_t ein = in_f32 ? 4 : 2, eout = out_f32 ? 4 : 2;
  const size_t row = size_t(D);  // elements per (position, head)
  char* base = (char*)d_scratch;
  cudaStream_t st = (cudaStream_t)stream;
  cudaGetLastError();
  int dev = 0;
  cudaGetDevice(&dev);
  HostPipe& hp = host_pipe_of(dev);
  std::lock_guard<std::mutex> lock(hp.mu);  // held for the whole enqueue (events are per call)
  if (!host_pipe_reserve(hp, int(chunks.size()))) return SA_ERR_CUDA;
  cudaError_t e = cudaEventRecord(hp.entry, st);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(hp.h2d, hp.entry, 0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(hp.d2h, hp.entry, 0);
  // host slice (b, heads h0..h0+hc) of a [B,N,H,D] tensor <-> compact device chunk [1,N,hc,D]
  auto copy_in = [&](char* dst, const void* src, const Chunk& c, size_t es) {
    const char* s0 = (const char*)src + ((c.b * N * H) + c.h0) * row * es;
    if (c.hc == H) return cudaMemcpyAsync(dst, s0, size_t(N) * H * row * es, cudaMemcpyHostToDevice, hp.h2d);
    return cudaMemcpy2DAsync(dst, c.hc * row * es, s0, H * row * es, c.hc * row * es, size_t(N),
                             cudaMemcpyHostToDevice, hp.h2d);
  };
  auto copy_out = [&](void* dst, const char* src, const Chunk& c, size_t es) {
    char* d0 = (char*)dst + ((c.b * N * H) + c.h0) * row * es;
    if (c.hc == H) return cudaMemcpyAsync(d0, src, size_t(N) * H * row * es, cudaMemcpyDeviceToHost, hp.d2h);
    return cudaMemcpy2DAsync(d0, H * row * es, src, c.hc * row * es, c.hc * row * es, size_t(N),
                             cudaMemcpyDeviceToHost, hp.d2h);
  };
  for (size_t ci = 0; ci < chunks.size() && e == cudaSuccess; ++ci) {
    const Chunk& c = chunks[ci];
    // device chunk buffers: compact [N, hc, D] at the chunk's place inside batch element b's slice
    const size_t cofs = size_t((c.b * H + c.h0) * N) * row;  // elements
    auto P = [&](int t) { return base + off[t] + cofs * (t < 6 ? ein : eout); };
    // the forward needs q, k, v, k2, v2; dO uploads while it runs
    for (int t = 0; t < 5 && e == cudaSuccess; ++t) e = copy_in(P(t), hin[t], c, ein);
    if (e == cudaSuccess) e = cudaEventRecord(hp.in[ci], hp.h2d);
    if (e == cudaSuccess) e = copy_in(P(5), hin[5], c, ein);
    if (e == cudaSuccess) e = cudaEventRecord(hp.in_b[ci], hp.h2d);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, hp.in[ci], 0);
    if (e != cudaSuccess) break;
    float* lse_c = (float*)(base + off[7]) + (c.b * H + c.h0) * N;
    s = simplicial_attn_fwd(P(0), P(1), P(2), P(3), P(4), P(6), lse_c, base + off[13], off[14] - off[13], 1, c.hc,
                            N, D, w1, w2, flags, stream);
    if (s != SA_OK) return s;
    // o and lse download while the backward runs
    e = cudaEventRecord(hp.fdone[ci], st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(hp.d2h, hp.fdone[ci], 0);
    if (e == cudaSuccess) e = copy_out(h_o, P(6), c, eout);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync((char*)h_lse + size_t((c.b * H + c.h0) * N) * 4, lse_c, size_t(c.hc) * N * 4,
                          cudaMemcpyDeviceToHost, hp.d2h);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, hp.in_b[ci], 0);
    if (e != cudaSuccess) break;
    s = simplicial_attn_bwd(P(0), P(1), P(2), P(3), P(4), P(6), lse_c, P(5), P(8), P(9), P(10), P(11), P(12),
                            base + off[13], off[14] - off[13], 1, c.hc, N, D, w1, w2, flags, stream);
    if (s != SA_OK) return s;
    e = cudaEventRecord(hp.done[ci], st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(hp.d2h, hp.done[ci], 0);
    for (int t = 0; t < 5 && e == cudaSuccess; ++t) e = copy_out(hout[t], P(8 + t), c, eout);
  }
  if (e == cudaSuccess) e = cudaEventRecord(hp.out, hp.d2h);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(st, hp.out, 0);
  return cuda_status(e);
}

int simplicial_attn_fwd_path(int64_t B, int64_t H, int64_t N, int64_t D, int64_t w1, int64_t w2,
                             uint32_t flags) {
  Problem p;
  if (make_problem(B, H, N, D, w1, w2, 0, flags, &p) != SA_OK) return 0;
  const Route r = route(p, flags, false);
  return r == Route::TC ? SA_PATH_TCGEN05 : r == Route::SIMT ? SA_PATH_SIMT : 0;
}

int simplicial_attn_bwd_path(int64_t B, int64_t H, int64_t N, int64_t D, int64_t w1, int64_t w2,
                             uint32_t flags) {
  Problem p;
  if (make_problem(B, H, N, D, w1, w2, 0, flags, &p) != SA_OK) return 0;
  const Route r = route(p, flags, true);
  return r == Route::TC ? SA_PATH_TCGEN05 : r == Route::SIMT ? SA_PATH_SIMT : 0;
}

uint64_t simplicial_attn_launch_count(void) { return g_launches.load(); }

void simplicial_attn_profile_enable(int on) {
  if (on) {  // pre-create events so that enabling costs nothing inside a timed region
    std::vector<cudaEvent_t> fresh(256);
    for (auto& e : fresh) cudaEventCreateWithFlags(&e, cudaEventDefault);
    std::lock_guard<std::mutex> g(g_prof_mu);
    g_event_pool.insert(g_event_pool.end(), fresh.begin(), fresh.end());
  }
  g_prof_on.store(on ? 1 : 0);
}

int simplicial_attn_profile_read(char* names32, double* total_ms, int64_t* counts, int max_kernels) {
  std::vector<ProfRec> recs;
  {
    std::lock_guard<std::mutex> g(g_prof_mu);
    recs.swap(g_prof);
  }
  std::vector<std::string> names;
  std::vector<double> tot;
  std::vector<int64_t> cnt;
  for (auto& r : recs) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    {
      std::lock_guard<std::mutex> g(g_prof_mu);
      g_event_pool.push_back(r.a);
      g_event_pool.push_back(r.b);
    }
    size_t k = 0;
    while (k < names.size() && names[k] != r.name) ++k;
    if (k == names.size()) { names.push_back(r.name); tot.push_back(0); cnt.push_back(0); }
    tot[k] += ms;
    cnt[k] += 1;
  }
  int n = int(names.size()) < max_kernels ? int(names.size()) : max_kernels;
  for (int k = 0; k < n; ++k) {
    strncpy(names32 + 32 * k, names[k].c_str(), 31);
    names32[32 * k + 31] = 0;
    total_ms[k] = tot[k];
    counts[k] = cnt[k];
  }
  return n;
}

const char* simplicial_attn_status_string(sa_status s) {
  switch (s) {
    case SA_OK: return "SA_OK";
    case SA_ERR_INVALID_ARG: return "SA_ERR_INVALID_ARG";
    case SA_ERR_UNSUPPORTED: return "SA_ERR_UNSUPPORTED";
    case SA_ERR_WORKSPACE: return "SA_ERR_WORKSPACE";
    case SA_ERR_CUDA: return "SA_ERR_CUDA";
  }
  return "SA_UNKNOWN";
}

const char* simplicial_attn_version(void) { return "libsimplicial sm_100a " __DATE__ " " __TIME__; }

#ifdef SA_TRACE
// Trace builds only: copy the (tag, clock) pairs recorded since the last call and reset.
int simplicial_attn_debug_trace(unsigned long long* host, int max_pairs) {
  cudaDeviceSynchronize();
  const int n = max_pairs < 4096 ? max_pairs : 4096;
  cudaMemcpyFromSymbol(host, sa::g_trace, sizeof(unsigned long long) * 2 * n);
  static unsigned long long zeros[8192];
  cudaMemcpyToSymbol(sa::g_trace, zeros, sizeof(zeros));
  return n;
}
#endif

}  // extern "C"

// ------------------------------------------------------------------------------------------------
// Grouped-query attention
// ------------------------------------------------------------------------------------------------
namespace sa {
// bwd_gqa workspace: [o fp32 (bf16 outputs only)] [dq fp32 (bf16 outputs only)]
//                    [dk, dv, dk2, dv2 per-query-head fp32 partials] [the backward's own workspace]
static size_t gqa_bwd_layout(const Problem& p, uint32_t flags, size_t off[8]) {
  const bool out_f32 = (flags & (SA_IN_F32 | SA_OUT_F32)) != 0;
  const size_t nq = size_t(p.B) * p.N * p.H * p.D, nkp = size_t(p.B) * p.NK() * p.H * p.D;
  size_t cur = 0;
  off[0] = cur;
  cur += out_f32 ? 0 : align256(nq * 4);
  off[1] = cur;
  cur += out_f32 ? 0 : align256(nq * 4);
  for (int t = 0; t < 4; ++t) {
    off[2 + t] = cur;
    cur += align256(nkp * 4);
  }
  off[6] = cur;
  cur += bwd_ws(p, flags | SA_OUT_F32);
  off[7] = cur;
  return cur;
}
}  // namespace sa

extern "C" {

size_t simplicial_attn_fwd_gqa_workspace_bytes(int64_t B, int64_t H, int64_t H_kv, int64_t N, int64_t D,
                                               int64_t w1, int64_t w2, uint32_t flags) {
  Problem p;
  if (make_problem_gqa(B, H, H_kv, N, D, w1, w2, flags, &p) != SA_OK) return 0;
  return use_tc_fwd(p, flags) ? tc_fwd_workspace_bytes(p) : 0;
}

sa_status simplicial_attn_fwd_gqa(const void* q, const void* k, const void* v, const void* k2, const void* v2,
                                  void* o, float* lse, void* workspace, size_t workspace_bytes, int64_t B,
                                  int64_t H, int64_t H_kv, int64_t N, int64_t D, int64_t w1, int64_t w2,
                                  uint32_t flags, void* stream) {
  if (!q || !k || !v || !k2 || !v2 || !o || !lse) return SA_ERR_INVALID_ARG;
  Problem p;
  sa_status s = make_problem_gqa(B, H, H_kv, N, D, w1, w2, flags, &p);
  if (s != SA_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  bool in_f32 = flags & SA_IN_F32, out_f32 = in_f32 || (flags & SA_OUT_F32);
  cudaGetLastError();
  switch (route(p, flags, false)) {
    case Route::TC:
      if (!workspace || workspace_bytes < tc_fwd_workspace_bytes(p)) return SA_ERR_WORKSPACE;
      return cuda_status(tc_forward_ws(p, out_f32, q, k, v, k2, v2, o, lse, workspace, st));
    case Route::SIMT:
      return cuda_status(simt_forward(p, in_f32, out_f32, q, k, v, k2, v2, o, lse, st));
    default:
      return SA_ERR_UNSUPPORTED;
  }
}

size_t simplicial_attn_bwd_gqa_workspace_bytes(int64_t B, int64_t H, int64_t H_kv, int64_t N, int64_t D,
                                               int64_t w1, int64_t w2, uint32_t flags) {
  Problem p;
  if (make_problem_gqa(B, H, H_kv, N, D, w1, w2, flags, &p) != SA_OK) return 0;
  if (p.Hk == p.H) return bwd_ws(p, flags);
  size_t off[8];
  return gqa_bwd_layout(p, flags, off);
}

sa_status simplicial_attn_bwd_gqa(const void* q, const void* k, const void* v, const void* k2, const void* v2,
                                  const void* o, const float* lse, const void* dO, void* dq, void* dk, void* dv,
                                  void* dk2, void* dv2, void* workspace, size_t workspace_bytes, int64_t B,
                                  int64_t H, int64_t H_kv, int64_t N, int64_t D, int64_t w1, int64_t w2,
                                  uint32_t flags, void* stream) {
  if (!q || !k || !v || !k2 || !v2 || !o || !lse || !dO || !dq || !dk || !dv || !dk2 || !dv2 || !workspace)
    return SA_ERR_INVALID_ARG;
  Problem p;
  sa_status s = make_problem_gqa(B, H, H_kv, N, D, w1, w2, flags, &p);
  if (s != SA_OK) return s;
  if (p.Hk == p.H)
    return simplicial_attn_bwd(q, k, v, k2, v2, o, lse, dO, dq, dk, dv, dk2, dv2, workspace, workspace_bytes, B, H,
                               N, D, w1, w2, flags, stream);
  size_t off[8];
  if (route(p, flags, true) == Route::NONE) return SA_ERR_UNSUPPORTED;
  if (workspace_bytes < gqa_bwd_layout(p, flags, off)) return SA_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  const bool in_f32 = flags & SA_IN_F32, out_f32 = in_f32 || (flags & SA_OUT_F32);
  const uint32_t flags32 = flags | SA_OUT_F32;
  char* w = (char*)workspace;
  const int64_t nq = int64_t(p.B) * p.N * p.H * p.D;
  cudaGetLastError();
  cudaError_t e = cudaSuccess;
  // the kernels run with fp32 outputs: o as fp32, dq and the per-query-head key partials in fp32
  const void* o32 = o;
  float* dq32 = (float*)dq;
  if (!out_f32) {
    e = cast_bf16_f32(o, (float*)(w + off[0]), nq, st);
    o32 = w + off[0];
    dq32 = (float*)(w + off[1]);
  }
  float* part[4];
  for (int t = 0; t < 4; ++t) part[t] = (float*)(w + off[2 + t]);
  void* bw = w + off[6];
  const size_t bwb = off[7] - off[6];
  if (e == cudaSuccess) {
    if (route(p, flags32, true) == Route::TC)
      e = tc_backward(p, true, q, k, v, k2, v2, o32, lse, dO, dq32, part[0], part[1], part[2], part[3], bw, bwb, st);
    else
      e = simt_backward(p, in_f32, true, q, k, v, k2, v2, o32, lse, dO, dq32, part[0], part[1], part[2], part[3],
                        (float*)bw, st);
  }
  void* outs[4] = {dk, dv, dk2, dv2};
  for (int t = 0; t < 4 && e == cudaSuccess; ++t)
    e = gqa_reduce(part[t], outs[t], out_f32, int64_t(p.B) * p.NK(), p.Hk, p.H / p.Hk, p.D, st);
  if (e == cudaSuccess && !out_f32) e = cast_f32_bf16(dq32, dq, nq, st);
  return cuda_status(e);
}

}  // extern "C"

// ---------------------------------------------------------------------------------------------
// K2_BIAS / V2_BIAS: the entry points add the two
// scalars to K' and V' into workspace copies, then run the grouped-query entry points (H_kv == H is
// plain multi-head) on the copies.  The bias is additive, so the gradients with respect to the
// biased copies are the gradients with respect to the caller's K' and V'.
// workspace: [k2 + b] [v2 + b] (input dtype, [B, N, H_kv, D] each) [the inner call's workspace]
namespace sa {
static size_t bias_copy_bytes(const Problem& p, uint32_t flags) {
  const size_t es = (flags & SA_IN_F32) ? 4 : 2;
  return align256(size_t(p.B) * p.NK() * p.Hk * p.D * es);
}
}  // namespace sa

extern "C" {

size_t simplicial_attn_fwd_bias_workspace_bytes(int64_t B, int64_t H, int64_t H_kv, int64_t N, int64_t D,
                                                int64_t w1, int64_t w2, uint32_t flags) {
  Problem p;
  if (make_problem_gqa(B, H, H_kv, N, D, w1, w2, flags, &p) != SA_OK) return 0;
  return 2 * bias_copy_bytes(p, flags) + simplicial_attn_fwd_gqa_workspace_bytes(B, H, H_kv, N, D, w1, w2, flags);
}

sa_status simplicial_attn_fwd_bias(const void* q, const void* k, const void* v, const void* k2, const void* v2,
                                   void* o, float* lse, float k2_bias, float v2_bias, void* workspace,
                                   size_t workspace_bytes, int64_t B, int64_t H, int64_t H_kv, int64_t N, int64_t D,
                                   int64_t w1, int64_t w2, uint32_t flags, void* stream) {
  if (!q || !k || !v || !k2 || !v2 || !o || !lse || !workspace) return SA_ERR_INVALID_ARG;
  Problem p;
  sa_status s = make_problem_gqa(B, H, H_kv, N, D, w1, w2, flags, &p);
  if (s != SA_OK) return s;
  if (workspace_bytes < simplicial_attn_fwd_bias_workspace_bytes(B, H, H_kv, N, D, w1, w2, flags))
    return SA_ERR_WORKSPACE;
  const size_t cb = bias_copy_bytes(p, flags);
  char* w = (char*)workspace;
  cudaGetLastError();
  cudaError_t e = add_bias(k2, v2, w, w + cb, int64_t(p.B) * p.NK() * p.Hk * p.D, (flags & SA_IN_F32) != 0,
                           k2_bias, v2_bias, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_status(e);
  return simplicial_attn_fwd_gqa(q, k, v, w, w + cb, o, lse, w + 2 * cb, workspace_bytes - 2 * cb, B, H, H_kv, N,
                                 D, w1, w2, flags, stream);
}

size_t simplicial_attn_bwd_bias_workspace_bytes(int64_t B, int64_t H, int64_t H_kv, int64_t N, int64_t D,
                                                int64_t w1, int64_t w2, uint32_t flags) {
  Problem p;
  if (make_problem_gqa(B, H, H_kv, N, D, w1, w2, flags, &p) != SA_OK) return 0;
  return 2 * bias_copy_bytes(p, flags) + simplicial_attn_bwd_gqa_workspace_bytes(B, H, H_kv, N, D, w1, w2, flags);
}

sa_status simplicial_attn_bwd_bias(const void* q, const void* k, const void* v, const void* k2, const void* v2,
                                   const void* o, const float* lse, const void* dO, void* dq, void* dk, void* dv,
                                   void* dk2, void* dv2, float k2_bias, float v2_bias, void* workspace,
                                   size_t workspace_bytes, int64_t B, int64_t H, int64_t H_kv, int64_t N, int64_t D,
                                   int64_t w1, int64_t w2, uint32_t flags, void* stream) {
  if (!q || !k || !v || !k2 || !v2 || !o || !lse || !dO || !dq || !dk || !dv || !dk2 || !dv2 || !workspace)
    return SA_ERR_INVALID_ARG;
  Problem p;
  sa_status s = make_problem_gqa(B, H, H_kv, N, D, w1, w2, flags, &p);
  if (s != SA_OK) return s;
  if (workspace_bytes < simplicial_attn_bwd_bias_workspace_bytes(B, H, H_kv, N, D, w1, w2, flags))
    return SA_ERR_WORKSPACE;
  const size_t cb = bias_copy_bytes(p, flags);
  char* w = (char*)workspace;
  cudaGetLastError();
  cudaError_t e = add_bias(k2, v2, w, w + cb, int64_t(p.B) * p.NK() * p.Hk * p.D, (flags & SA_IN_F32) != 0,
                           k2_bias, v2_bias, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_status(e);
  return simplicial_attn_bwd_gqa(q, k, v, w, w + cb, o, lse, dO, dq, dk, dv, dk2, dv2, w + 2 * cb,
                                 workspace_bytes - 2 * cb, B, H, H_kv, N, D, w1, w2, flags, stream);
}

}  // extern "C"

/*
 * oracle.c -- float64 CPU oracle for sliding-window 2-simplicial attention.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  The
 * product path (paper_2507_02754_b200/) never links, imports or calls it, and
 * this file shares no code, header, table or helper with the CUDA path.
 *
 * It is the plain definition of the operator, written out in the paper's
 * notation (citations are PAPER.md line numbers, "P:n", with the section):
 *
 *   A_ijk = s * sum_l Q_il K_jl K'_kl                    P:230-233 (Sec. 4, Eq. 3d-attention)
 *   A_ijk = s * sum_{l<p} det([q_i^(l); k_j^(l); k'_k^(l)])
 *           with det by the 6-term Sarrus expansion      P:291-301 (Sec. 5, Eq. det, Eq. logits)
 *   S_ijk = exp(A_ijk) / sum_{j,k} exp(A_ijk)            P:236-238 (Sec. 4, Eq. softmax)
 *   O_i   = sum_{j,k} S_ijk (v_j o v'_k)                 P:241-244 (Sec. 4, Eq. attenval)
 *   windows: j in (i-w1, i], k in (i-w2, i], clipped at 0 P:319-321 (Sec. 6), masks P:804-812
 *
 * and the backward equations of Sec. 7 with the corrections listed
 * in DESIGN.md ("readings"): S in place of A in dV/dV', the sum
 * over (i,j) in dK', the scale s applied to dQ/dK/dK', and
 *   dS_ijk = S_ijk (dP_ijk - sum_{j',k'} S_ij'k' dP_ij'k')  (dsoftmax).
 * For the determinant form the trilinear factor of each gradient is replaced by
 * the partial derivative of the Sarrus expansion w.r.t. that argument.
 *
 * s = 1/sqrt(D) (reading R3/R4); p = floor(D/3) and the
 * trailing D mod 3 dims do not enter the determinant logits (reading R5).
 *
 * Layout: key-side tensors k, v, k2, v2 (and dk..dv2) are [B, n_prefix+N, H, D];
 * query-side q, o, dO, dq are [B, N, H, D]; lse is [B, H, N].  Query row i sits
 * at position n_prefix+i of the key buffers (sequence-sharded mode).
 * Loops follow the definitions: per query row the full (j,k) logit rectangle is
 * materialised, then softmax, then the sums.  No tiling, no online softmax.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
  int64_t B, H, N, D, w1, w2, np;  /* np = n_prefix */
  int det;
  double s;
} shape_t;

static inline const double* qrow(const double* t, const shape_t* g, int64_t b, int64_t i, int64_t h) {
  return t + ((b * g->N + i) * g->H + h) * g->D;
}
static inline const double* krow(const double* t, const shape_t* g, int64_t b, int64_t j, int64_t h) {
  return t + ((b * (g->np + g->N) + j) * g->H + h) * g->D;
}

/* window of key positions for query position pos (buffer coordinates): (pos-w, pos], clipped at 0.
 * "(q_idx - w1) < kv1_idx <= q_idx". */
static inline int64_t win_lo(int64_t pos, int64_t w) { return pos - w + 1 > 0 ? pos - w + 1 : 0; }

/* 3x3 determinant of the rows a, b, c by the Sarrus expansion. */
static inline double det3(const double* a, const double* b, const double* c) {
  return a[0] * b[1] * c[2] + a[1] * b[2] * c[0] + a[2] * b[0] * c[1]
       - a[0] * b[2] * c[1] - a[1] * b[0] * c[2] - a[2] * b[1] * c[0];
}

/* Logit A_ijk (P:230-233 trilinear, P:298-301 determinant). */
static double logit(const shape_t* g, const double* q, const double* k, const double* k2) {
  double acc = 0.0;
  if (!g->det) {
    for (int64_t l = 0; l < g->D; ++l) acc += q[l] * k[l] * k2[l];
  } else {
    int64_t p = g->D / 3;
    for (int64_t l = 0; l < p; ++l) acc += det3(q + 3 * l, k + 3 * l, k2 + 3 * l);
  }
  return g->s * acc;
}

/* Partial derivatives of one logit w.r.t. its three arguments (without s):
 *   trilinear: dA/dq_l = k_l k'_l, dA/dk_l = q_l k'_l, dA/dk'_l = q_l k_l
 *   determinant: derivatives of the Sarrus expansion a1b2c3 + a2b3c1 + a3b1c2
 *                - a1b3c2 - a2b1c3 - a3b2c1 per chunk; 0 on trailing dims.
 * which = 0 -> w.r.t. q (a), 1 -> w.r.t. k (b), 2 -> w.r.t. k' (c). */
static void dlogit(const shape_t* g, int which, const double* a, const double* b, const double* c,
                   double* out /* D */) {
  if (!g->det) {
    for (int64_t l = 0; l < g->D; ++l) {
      if (which == 0) out[l] = b[l] * c[l];
      else if (which == 1) out[l] = a[l] * c[l];
      else out[l] = a[l] * b[l];
    }
    return;
  }
  for (int64_t l = 0; l < g->D; ++l) out[l] = 0.0;
  int64_t p = g->D / 3;
  for (int64_t t = 0; t < p; ++t) {
    const double *x = a + 3 * t, *y = b + 3 * t, *z = c + 3 * t;
    double* o = out + 3 * t;
    if (which == 0) {        /* d/da */
      o[0] = y[1] * z[2] - y[2] * z[1];
      o[1] = y[2] * z[0] - y[0] * z[2];
      o[2] = y[0] * z[1] - y[1] * z[0];
    } else if (which == 1) { /* d/db */
      o[0] = x[2] * z[1] - x[1] * z[2];
      o[1] = x[0] * z[2] - x[2] * z[0];
      o[2] = x[1] * z[0] - x[0] * z[1];
    } else {                 /* d/dc */
      o[0] = x[1] * y[2] - x[2] * y[1];
      o[1] = x[2] * y[0] - x[0] * y[2];
      o[2] = x[0] * y[1] - x[1] * y[0];
    }
  }
}

/* Row i of the forward: materialise A over the (j,k) window rectangle, softmax (Eq. softmax),
 * output (Eq. attenval).  logits/probs: scratch of w1*w2 doubles. Returns lse_i. */
static double row_forward(const shape_t* g, int64_t b, int64_t h, int64_t i, const double* q,
                          const double* k, const double* v, const double* k2, const double* v2,
                          double* P /* [nj*nk] */, double* o_out /* D or NULL */,
                          int64_t* nj_out, int64_t* nk_out) {
  int64_t pos = g->np + i;
  int64_t j0 = win_lo(pos, g->w1), k0 = win_lo(pos, g->w2);
  int64_t nj = pos - j0 + 1, nk = pos - k0 + 1;
  const double* qi = qrow(q, g, b, i, h);
  double m = -INFINITY;
  for (int64_t a = 0; a < nj; ++a)
    for (int64_t c = 0; c < nk; ++c) {
      double x = logit(g, qi, krow(k, g, b, j0 + a, h), krow(k2, g, b, k0 + c, h));
      P[a * nk + c] = x;
      if (x > m) m = x;
    }
  /* softmax over the flattened (j,k) axes (Alg. 1 "axis=[-1,-2]"); m only stabilises */
  double z = 0.0;
  for (int64_t t = 0; t < nj * nk; ++t) z += exp(P[t] - m);
  double lse = m + log(z);
  for (int64_t t = 0; t < nj * nk; ++t) P[t] = exp(P[t] - lse);
  if (o_out) {
    for (int64_t d = 0; d < g->D; ++d) o_out[d] = 0.0;
    for (int64_t a = 0; a < nj; ++a) {
      const double* vj = krow(v, g, b, j0 + a, h);
      for (int64_t c = 0; c < nk; ++c) {
        const double* vk = krow(v2, g, b, k0 + c, h);
        double pr = P[a * nk + c];
        for (int64_t d = 0; d < g->D; ++d) o_out[d] += pr * vj[d] * vk[d];
      }
    }
  }
  *nj_out = nj;
  *nk_out = nk;
  return lse;
}

static int nthreads_used = 1;

int sa_oracle_threads(void) { return nthreads_used; }

void sa_oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

static void note_threads(void) {
#ifdef _OPENMP
  nthreads_used = omp_get_max_threads();
#else
  nthreads_used = 1;
#endif
}

/* Forward.  rows: optional list of n_rows flat (b*H+h)*N+i query indices to compute (sampled
 * checking at full size); NULL -> all rows.  Rows not listed are left untouched. */
void sa_oracle_fwd(const double* q, const double* k, const double* v, const double* k2,
                   const double* v2, double* o, double* lse, int64_t B, int64_t H, int64_t N,
                   int64_t D, int64_t w1, int64_t w2, int64_t n_prefix, int det,
                   const int64_t* rows, int64_t n_rows) {
  shape_t g = {B, H, N, D, w1, w2, n_prefix, det, 1.0 / sqrt((double)D)};
  note_threads();
  int64_t total = rows ? n_rows : B * H * N;
#pragma omp parallel
  {
    double* P = (double*)malloc(sizeof(double) * (size_t)(w1 < N + n_prefix ? w1 : N + n_prefix) *
                                (size_t)(w2 < N + n_prefix ? w2 : N + n_prefix));
#pragma omp for schedule(dynamic, 16)
    for (int64_t t = 0; t < total; ++t) {
      int64_t flat = rows ? rows[t] : t;
      int64_t i = flat % N, bh = flat / N, h = bh % H, b = bh / H;
      int64_t nj, nk;
      double* orow = o + ((b * N + i) * H + h) * D;
      lse[(b * H + h) * N + i] = row_forward(&g, b, h, i, q, k, v, k2, v2, P, orow, &nj, &nk);
    }
    free(P);
  }
}

/* Backward by the (corrected) equations of Sec. 7, as three gather passes (no
 * atomics).  Pass 1 materialises each query row's rectangle and stores the row statistics
 * lse_i and delta_i = sum_{j'k'} S_ij'k' dP_ij'k'; passes 2 and 3 recompute single cells
 * S_ijk = exp(A_ijk - lse_i) from them:
 *   dP_ijk = sum_d dO_id V_jd V'_kd
 *   dS_ijk = S_ijk (dP_ijk - delta_i)                                  (dsoftmax)
 *   dQ_i  = sum_{j,k} dS_ijk dA/dq    dK_j  = sum_{i,k} dS_ijk dA/dk
 *   dK'_k = sum_{i,j} dS_ijk dA/dk'                                   (sum over i,j)
 *   dV_j  = sum_{i,k} S_ijk dO_i o V'_k   dV'_k = sum_{i,j} S_ijk dO_i o V_j
 * dA/d(.) carries the factor s.  Grad buffers are fully overwritten (key-side over all
 * n_prefix+N rows). */
static double cell_dp(const shape_t* g, const double* doi, const double* vj, const double* vk) {
  double x = 0.0;
  for (int64_t d = 0; d < g->D; ++d) x += doi[d] * vj[d] * vk[d];
  return x;
}

void sa_oracle_bwd(const double* q, const double* k, const double* v, const double* k2,
                   const double* v2, const double* dO, double* dq, double* dk, double* dv,
                   double* dk2, double* dv2, int64_t B, int64_t H, int64_t N, int64_t D,
                   int64_t w1, int64_t w2, int64_t n_prefix, int det) {
  shape_t g = {B, H, N, D, w1, w2, n_prefix, det, 1.0 / sqrt((double)D)};
  note_threads();
  int64_t NK = n_prefix + N;
  int64_t cap1 = w1 < NK ? w1 : NK, cap2 = w2 < NK ? w2 : NK;
  size_t psz = sizeof(double) * (size_t)cap1 * (size_t)cap2;
  double* lse = (double*)malloc(sizeof(double) * (size_t)(B * H * N));
  double* delta = (double*)malloc(sizeof(double) * (size_t)(B * H * N));

  /* pass 1: per query row i -- S, dP, lse_i, delta_i, dQ_i */
#pragma omp parallel
  {
    double *P = (double*)malloc(psz), *dP = (double*)malloc(psz);
    double* gr = (double*)malloc(sizeof(double) * (size_t)D);
#pragma omp for schedule(dynamic, 16)
    for (int64_t t = 0; t < B * H * N; ++t) {
      int64_t i = t % N, bh = t / N, h = bh % H, b = bh / H;
      int64_t nj, nk, pos = n_prefix + i;
      double l = row_forward(&g, b, h, i, q, k, v, k2, v2, P, NULL, &nj, &nk);
      int64_t j0 = win_lo(pos, w1), k0 = win_lo(pos, w2);
      const double* qi = qrow(q, &g, b, i, h);
      const double* doi = qrow(dO, &g, b, i, h);
      double dl = 0.0;
      for (int64_t a = 0; a < nj; ++a)
        for (int64_t c = 0; c < nk; ++c) {
          dP[a * nk + c] = cell_dp(&g, doi, krow(v, &g, b, j0 + a, h), krow(v2, &g, b, k0 + c, h));
          dl += P[a * nk + c] * dP[a * nk + c];
        }
      lse[t] = l;
      delta[t] = dl;
      double* out = dq + ((b * N + i) * H + h) * D;
      for (int64_t d = 0; d < D; ++d) out[d] = 0.0;
      for (int64_t a = 0; a < nj; ++a)
        for (int64_t c = 0; c < nk; ++c) {
          double ds = P[a * nk + c] * (dP[a * nk + c] - dl);
          dlogit(&g, 0, qi, krow(k, &g, b, j0 + a, h), krow(k2, &g, b, k0 + c, h), gr);
          for (int64_t d = 0; d < D; ++d) out[d] += g.s * ds * gr[d];
        }
    }
    free(P); free(dP); free(gr);
  }

  /* pass 2 (which=1): dK_j, dV_j per key row; pass 3 (which=2): dK'_k, dV'_k per key row.
   * Key row r is in the window of query position pos iff r in (pos-w, pos], i.e. pos in [r, r+w). */
  for (int which = 1; which <= 2; ++which) {
    double* gk = which == 1 ? dk : dk2;
    double* gv = which == 1 ? dv : dv2;
    int64_t w = which == 1 ? w1 : w2;
    int64_t wo = which == 1 ? w2 : w1; /* window of the other key */
#pragma omp parallel
    {
      double* gr = (double*)malloc(sizeof(double) * (size_t)D);
#pragma omp for schedule(dynamic, 16)
      for (int64_t t = 0; t < B * H * NK; ++t) {
        int64_t r = t % NK, bh = t / NK, h = bh % H, b = bh / H;
        double* ok = gk + ((b * NK + r) * H + h) * D;
        double* ov = gv + ((b * NK + r) * H + h) * D;
        for (int64_t d = 0; d < D; ++d) ok[d] = ov[d] = 0.0;
        for (int64_t pos = r; pos < r + w && pos < NK; ++pos) {
          int64_t i = pos - n_prefix;
          if (i < 0) continue;
          int64_t row = (b * H + h) * N + i;
          const double* qi = qrow(q, &g, b, i, h);
          const double* doi = qrow(dO, &g, b, i, h);
          for (int64_t o = win_lo(pos, wo); o <= pos; ++o) {
            int64_t j = which == 1 ? r : o, kk = which == 1 ? o : r;
            const double* kj = krow(k, &g, b, j, h);
            const double* k2k = krow(k2, &g, b, kk, h);
            const double* vj = krow(v, &g, b, j, h);
            const double* v2k = krow(v2, &g, b, kk, h);
            double pr = exp(logit(&g, qi, kj, k2k) - lse[row]);
            double ds = pr * (cell_dp(&g, doi, vj, v2k) - delta[row]);
            dlogit(&g, which, qi, kj, k2k, gr);
            const double* vo = which == 1 ? v2k : vj;
            for (int64_t d = 0; d < D; ++d) {
              ok[d] += g.s * ds * gr[d];
              ov[d] += pr * doi[d] * vo[d];
            }
          }
        }
      }
      free(gr);
    }
  }
  free(lse);
  free(delta);
}

/* usp_oracle.c — CPU restatement of the reference USP forward (see header).
 *
 * TEST INFRASTRUCTURE ONLY — the checker, never the product. Loop order and
 * operation sequence follow the cited reference lines exactly so that fp64
 * results are bitwise reproducible; OpenMP only splits independent rows.
 * Build: oracle/Makefile (gcc -O3, no -ffast-math, no FMA contraction).
 */
#include "usp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------- */
/* std::mt19937_64 (the engine behind UniformSource, random.hpp:15-29).     */

#define MT_N 312
#define MT_M 156
typedef struct {
  uint64_t s[MT_N];
  int i;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->s[0] = seed;
  for (int i = 1; i < MT_N; ++i) {
    g->s[i] = 6364136223846793005ULL * (g->s[i - 1] ^ (g->s[i - 1] >> 62)) +
              (uint64_t)i;
  }
  g->i = MT_N;
}

static uint64_t mt64_next(mt64* g) {
  const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
  if (g->i >= MT_N) {
    for (int k = 0; k < MT_N; ++k) {
      uint64_t y = (g->s[k] & upper) | (g->s[(k + 1) % MT_N] & lower);
      uint64_t v = g->s[(k + MT_M) % MT_N] ^ (y >> 1);
      if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
      g->s[k] = v;
    }
    g->i = 0;
  }
  uint64_t x = g->s[g->i++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

void uo_uniform_stream(uint64_t seed, double lo, double hi, int64_t n,
                       double* out) {
  mt64 g;
  mt64_seed(&g, seed);
  for (int64_t i = 0; i < n; ++i) {
    /* UniformSource::next_unit (random.hpp:19-22), next (random.hpp:25) */
    const double unit = (double)(mt64_next(&g) >> 11) * 0x1.0p-53;
    out[i] = lo + (hi - lo) * unit;
  }
}

/* ---------------------------------------------------------------------- */
/* numerics (src/numerics/attention.cpp)                                   */

static inline double dot_d(const double* a, const double* b, int64_t n) {
  double acc = 0; /* attention.cpp:42-47 */
  for (int64_t i = 0; i < n; ++i) acc += a[i] * b[i];
  return acc;
}

static inline double max_d(double a, double b) { /* std::max(a, b) */
  return (a < b) ? b : a;
}

int uo_reference_attention(const double* q, const double* k, const double* v,
                           int64_t batch, int64_t seq, int64_t heads,
                           int64_t kv_heads, int64_t hs, int causal,
                           const int64_t* positions, double* out) {
  if (kv_heads <= 0 || heads % kv_heads != 0) return -1; /* :27-32 */
  const int64_t heads_per_kv = heads / kv_heads;         /* :60 */
  const double inv_scale = 1.0 / sqrt((double)hs);       /* :61 */
  memset(out, 0, sizeof(double) * (size_t)(batch * seq * heads * hs));
#pragma omp parallel for collapse(2) schedule(dynamic, 4)
  for (int64_t b = 0; b < batch; ++b) {
    for (int64_t i = 0; i < seq; ++i) {
      double* scores = (double*)malloc(sizeof(double) * (size_t)seq);
      const int64_t qp = positions ? positions[i] : i; /* :67 */
      for (int64_t h = 0; h < heads; ++h) {
        const int64_t kv_h = h / heads_per_kv; /* :69 */
        const double* q_row = q + ((b * seq + i) * heads + h) * hs;
        double row_max = -INFINITY; /* :72-77 */
        for (int64_t j = 0; j < seq; ++j) {
          if (causal && (positions ? positions[j] : j) > qp) continue;
          scores[j] = dot_d(q_row, k + ((b * seq + j) * kv_heads + kv_h) * hs,
                            hs) * inv_scale;
          row_max = max_d(row_max, scores[j]);
        }
        double norm = 0; /* :79-88 */
        double* out_row = out + ((b * seq + i) * heads + h) * hs;
        for (int64_t j = 0; j < seq; ++j) {
          if (causal && (positions ? positions[j] : j) > qp) continue;
          const double w = exp(scores[j] - row_max);
          norm += w;
          const double* v_row = v + ((b * seq + j) * kv_heads + kv_h) * hs;
          for (int64_t s = 0; s < hs; ++s) out_row[s] += w * v_row[s];
        }
        for (int64_t s = 0; s < hs; ++s) out_row[s] /= norm;
      }
      free(scores);
    }
  }
  return 0;
}

/* SoftmaxState<double> (attention.cpp:172-264) */
typedef struct {
  int64_t batch, q_len, heads, hs;
  double *m, *l, *acc;
} sm_state;

static void sm_init(sm_state* st, int64_t batch, int64_t q_len,
                    int64_t heads, int64_t hs) {
  const size_t rows = (size_t)(batch * q_len * heads);
  st->batch = batch;
  st->q_len = q_len;
  st->heads = heads;
  st->hs = hs;
  st->m = (double*)malloc(sizeof(double) * rows);
  st->l = (double*)calloc(rows, sizeof(double));
  st->acc = (double*)calloc(rows * (size_t)hs, sizeof(double));
  for (size_t r = 0; r < rows; ++r) st->m[r] = -INFINITY; /* :177 */
}

static void sm_free(sm_state* st) {
  free(st->m);
  free(st->l);
  free(st->acc);
}

/* SoftmaxState::update (attention.cpp:181-230) with the position mask of
 * BlockMask::causal (attention.hpp:23-34); causal == 0 is BlockMask::none. */
static void sm_update(sm_state* st, const double* q, const double* k,
                      const double* v, int64_t k_len, int64_t kv_heads,
                      int causal, const int64_t* q_pos, const int64_t* k_pos) {
  const int64_t heads = st->heads, hs = st->hs, q_len = st->q_len;
  const int64_t heads_per_kv = heads / kv_heads; /* :189 */
  const double inv_scale = 1.0 / sqrt((double)hs); /* :190 */
#pragma omp parallel for collapse(2) schedule(dynamic, 4)
  for (int64_t b = 0; b < st->batch; ++b) {
    for (int64_t i = 0; i < q_len; ++i) {
      double* scores = (double*)malloc(sizeof(double) * (size_t)(k_len + 1));
      for (int64_t h = 0; h < heads; ++h) {
        const int64_t kv_h = h / heads_per_kv;
        const double* q_row = q + ((b * q_len + i) * heads + h) * hs;
        double row_max = -INFINITY; /* :199-206 */
        int any = 0;
        for (int64_t j = 0; j < k_len; ++j) {
          if (causal && k_pos[j] > q_pos[i]) continue;
          scores[j] = dot_d(q_row, k + ((b * k_len + j) * kv_heads + kv_h) * hs,
                            hs) * inv_scale;
          row_max = max_d(row_max, scores[j]);
          any = 1;
        }
        if (!any) continue; /* :207 */
        const size_t r = (size_t)((b * q_len + i) * heads + h);
        const double m_new = max_d(st->m[r], row_max); /* :210 */
        const double rescale = exp(st->m[r] - m_new);   /* :211 */
        double* acc_row = st->acc + r * (size_t)hs;
        for (int64_t s = 0; s < hs; ++s) acc_row[s] *= rescale; /* :214 */
        double l_new = st->l[r] * rescale;                      /* :215 */
        for (int64_t j = 0; j < k_len; ++j) {                   /* :216-224 */
          if (causal && k_pos[j] > q_pos[i]) continue;
          const double w = exp(scores[j] - m_new);
          l_new += w;
          const double* v_row = v + ((b * k_len + j) * kv_heads + kv_h) * hs;
          for (int64_t s = 0; s < hs; ++s) acc_row[s] += w * v_row[s];
        }
        st->m[r] = m_new;
        st->l[r] = l_new;
      }
      free(scores);
    }
  }
}

/* finalize (attention.cpp:232-254) + logsumexp (:256-264). */
static int64_t sm_finish(const sm_state* st, double* out, double* lse) {
  const size_t rows = (size_t)(st->batch * st->q_len * st->heads);
  int64_t empty = 0;
  for (size_t r = 0; r < rows; ++r) {
    const double l = st->l[r];
    if (lse) lse[r] = l > 0.0 ? st->m[r] + log(l) : -INFINITY;
    if (!out) continue;
    if (l == 0.0) {
      ++empty; /* the reference throws kNumeric "saw no keys" (:239-244) */
      for (int64_t s = 0; s < st->hs; ++s) out[r * st->hs + s] = NAN;
      continue;
    }
    for (int64_t s = 0; s < st->hs; ++s)
      out[r * (size_t)st->hs + s] = st->acc[r * (size_t)st->hs + s] / l;
  }
  return empty;
}

int64_t uo_softmax_rows(const double* q, const double* k, const double* v,
                        int64_t batch, int64_t q_len, int64_t k_len,
                        int64_t heads, int64_t kv_heads, int64_t hs,
                        int causal, const int64_t* q_pos, const int64_t* k_pos,
                        double* out, double* lse) {
  sm_state st;
  sm_init(&st, batch, q_len, heads, hs);
  sm_update(&st, q, k, v, k_len, kv_heads, causal, q_pos, k_pos);
  const int64_t empty = sm_finish(&st, out, lse);
  sm_free(&st);
  return empty;
}

/* ---------------------------------------------------------------------- */
/* partition (src/usp/partition.cpp)                                        */

int uo_zigzag_partition(int64_t seq_len, int ring, int64_t* out) {
  if (ring < 1 || seq_len % (2 * ring) != 0) return -1; /* :13-20 */
  const int64_t chunk = seq_len / (2 * ring);
  for (int p = 0; p < ring; ++p) {
    int64_t* tokens = out + (int64_t)p * 2 * chunk;
    const int64_t lo_base = chunk * p;                    /* :27 */
    const int64_t hi_base = chunk * (2 * ring - 1 - p);   /* :28 */
    for (int64_t i = 0; i < chunk; ++i) tokens[i] = lo_base + i;
    for (int64_t i = 0; i < chunk; ++i) tokens[chunk + i] = hi_base + i;
  }
  return 0;
}

int uo_even_partition(int64_t seq_len, int ring, int64_t* out) {
  if (ring < 1 || seq_len % ring != 0) return -1; /* :36-40 */
  for (int64_t i = 0; i < seq_len; ++i) out[i] = i;
  return 0;
}

int uo_causal_pair_counts(const int64_t* assignment, int ring,
                          int64_t seq_len, int64_t* counts) {
  const int64_t per = seq_len / ring;
  char* seen = (char*)calloc((size_t)seq_len, 1);
  int rc = 0;
  for (int p = 0; p < ring && rc == 0; ++p) {
    int64_t pairs = 0;
    for (int64_t t = 0; t < per; ++t) {
      const int64_t q = assignment[(int64_t)p * per + t];
      if (q < 0 || q >= seq_len || seen[q]) { rc = -1; break; } /* :62-64 */
      seen[q] = 1;
      pairs += q + 1; /* :66 keys 0..q */
    }
    counts[p] = pairs;
  }
  for (int64_t i = 0; rc == 0 && i < seq_len; ++i)
    if (!seen[i]) rc = -1;
  free(seen);
  return rc;
}

int uo_positions_for(int ulysses, int ring, int64_t seq_len, int zigzag,
                     int rank, int64_t* out) {
  if (ulysses < 1 || ring < 1 || rank < 0 || rank >= ulysses * ring) return -1;
  if (zigzag && seq_len % (2 * ring) != 0) return -1; /* :78-84 */
  if (seq_len % ring != 0) return -1;                 /* :85-87 */
  if ((seq_len / ring) % ulysses != 0) return -1;     /* :88-92 */
  const int u = rank % ulysses;                       /* mesh.cpp:23-26 */
  const int r = rank / ulysses;                       /* mesh.cpp:28-31 */
  const int64_t per_ring = seq_len / ring;
  int64_t* lists = (int64_t*)malloc(sizeof(int64_t) * (size_t)seq_len);
  if (zigzag)
    uo_zigzag_partition(seq_len, ring, lists);
  else
    uo_even_partition(seq_len, ring, lists);
  const int64_t per_rank = per_ring / ulysses;
  memcpy(out, lists + (int64_t)r * per_ring + (int64_t)u * per_rank,
         sizeof(int64_t) * (size_t)per_rank); /* :95-105 */
  free(lists);
  return 0;
}

/* ---------------------------------------------------------------------- */
/* usp_attention forward (src/usp/usp_attention.cpp:43-65)                  */

int uo_usp_forward(const double* q, const double* k, const double* v,
                   int64_t batch, int64_t seq, int64_t heads, int64_t kv_heads,
                   int64_t hs, int ulysses, int ring, int causal,
                   double* out_global, double* lse) {
  /* check_usp_inputs (usp_attention.cpp:15-38) */
  if (kv_heads % ulysses != 0 || ulysses > kv_heads) return -1;
  if (heads % ulysses != 0) return -1;
  if (heads % kv_heads != 0) return -1;
  if (causal && seq % (2 * ring) != 0) return -1;
  if (seq % ring != 0 || (seq / ring) % ulysses != 0) return -1;

  const int64_t per_ring = seq / ring;
  const int64_t hl = heads / ulysses, kvl = kv_heads / ulysses;
  int64_t* lists = (int64_t*)malloc(sizeof(int64_t) * (size_t)seq);
  if (causal)
    uo_zigzag_partition(seq, ring, lists); /* commands.cpp:88 zigzag iff causal */
  else
    uo_even_partition(seq, ring, lists);

  double* qh = (double*)malloc(sizeof(double) * (size_t)(batch * per_ring * hl * hs));
  double* kh = (double*)malloc(sizeof(double) * (size_t)(batch * seq * kvl * hs));
  double* vh = (double*)malloc(sizeof(double) * (size_t)(batch * seq * kvl * hs));
  double* oh = (double*)malloc(sizeof(double) * (size_t)(batch * per_ring * hl * hs));

  for (int u = 0; u < ulysses; ++u) {
    /* head-sharded K/V of every ring rank of this Ulysses column, as the
     * forward all-to-all (all_to_all_4d.cpp:13-59) leaves them: rows in ring
     * list order, heads [u*kvl, (u+1)*kvl). Block src occupies rows
     * [src*per_ring, (src+1)*per_ring) of kh/vh. */
    for (int src = 0; src < ring; ++src)
      for (int64_t b = 0; b < batch; ++b)
        for (int64_t t = 0; t < per_ring; ++t) {
          const int64_t gp = lists[(int64_t)src * per_ring + t];
          for (int64_t h = 0; h < kvl; ++h) {
            const size_t src_off = (size_t)(((b * seq + gp) * kv_heads + u * kvl + h) * hs);
            const size_t dst_off = (size_t)((((int64_t)src * batch + b) * per_ring + t) * kvl + h) * (size_t)hs;
            memcpy(kh + dst_off, k + src_off, sizeof(double) * (size_t)hs);
            memcpy(vh + dst_off, v + src_off, sizeof(double) * (size_t)hs);
          }
        }
    for (int r = 0; r < ring; ++r) {
      const int64_t* my_pos = lists + (int64_t)r * per_ring; /* head_positions */
      for (int64_t b = 0; b < batch; ++b)
        for (int64_t t = 0; t < per_ring; ++t)
          for (int64_t h = 0; h < hl; ++h)
            memcpy(qh + ((b * per_ring + t) * hl + h) * hs,
                   q + ((b * seq + my_pos[t]) * heads + u * hl + h) * hs,
                   sizeof(double) * (size_t)hs);
      /* ring_attention (ring_attention.cpp:45-76) */
      sm_state st;
      sm_init(&st, batch, per_ring, hl, hs);
      for (int step = 0; step < ring; ++step) {
        const int src = (r - step + ring) % ring; /* :63 */
        const size_t blk = (size_t)src * (size_t)(batch * per_ring * kvl * hs);
        sm_update(&st, qh, kh + blk, vh + blk, per_ring, kvl, causal, my_pos,
                  lists + (int64_t)src * per_ring);
      }
      const int rank = r * ulysses + u; /* mesh.cpp:38 */
      sm_finish(&st, oh, lse ? lse + (int64_t)rank * batch * per_ring * hl : NULL);
      sm_free(&st);
      /* inverse all-to-all (all_to_all_4d.cpp:62-107) + place_rows */
      for (int64_t b = 0; b < batch; ++b)
        for (int64_t t = 0; t < per_ring; ++t)
          for (int64_t h = 0; h < hl; ++h)
            memcpy(out_global + ((b * seq + my_pos[t]) * heads + u * hl + h) * hs,
                   oh + ((b * per_ring + t) * hl + h) * hs,
                   sizeof(double) * (size_t)hs);
    }
  }
  free(lists);
  free(qh);
  free(kh);
  free(vh);
  free(oh);
  return 0;
}

/* ---------------------------------------------------------------------- */
/* backward                                               */

int uo_reference_attention_grad(const double* q, const double* k, const double* v,
                                const double* dout, int64_t batch, int64_t seq,
                                int64_t heads, int64_t kv_heads, int64_t hs, int causal,
                                const int64_t* positions, double* dq, double* dk,
                                double* dv) {
  /* reference_attention_grad (attention.cpp:95-170), same loop order */
  if (kv_heads <= 0 || heads % kv_heads != 0) return -1;
  const int64_t heads_per_kv = heads / kv_heads;
  const double inv_scale = 1.0 / sqrt((double)hs);
  memset(dq, 0, sizeof(double) * (size_t)(batch * seq * heads * hs));
  memset(dk, 0, sizeof(double) * (size_t)(batch * seq * kv_heads * hs));
  memset(dv, 0, sizeof(double) * (size_t)(batch * seq * kv_heads * hs));
  double* p = (double*)malloc(sizeof(double) * (size_t)seq);
  double* dp = (double*)malloc(sizeof(double) * (size_t)seq);
  for (int64_t b = 0; b < batch; ++b) {
    for (int64_t i = 0; i < seq; ++i) {
      const int64_t qp = positions ? positions[i] : i;
      for (int64_t h = 0; h < heads; ++h) {
        const int64_t kv_h = h / heads_per_kv;
        const double* q_row = q + ((b * seq + i) * heads + h) * hs;
        const double* do_row = dout + ((b * seq + i) * heads + h) * hs;
        double row_max = -INFINITY; /* :126-131 */
        for (int64_t j = 0; j < seq; ++j) {
          if (causal && (positions ? positions[j] : j) > qp) continue;
          p[j] = dot_d(q_row, k + ((b * seq + j) * kv_heads + kv_h) * hs, hs) * inv_scale;
          row_max = max_d(row_max, p[j]);
        }
        double norm = 0; /* :132-140 */
        for (int64_t j = 0; j < seq; ++j) {
          if (causal && (positions ? positions[j] : j) > qp) {
            p[j] = 0;
            continue;
          }
          p[j] = exp(p[j] - row_max);
          norm += p[j];
        }
        double pdp = 0; /* :142-151 */
        for (int64_t j = 0; j < seq; ++j) {
          if (p[j] == 0.0) {
            dp[j] = 0;
            continue;
          }
          p[j] /= norm;
          dp[j] = dot_d(do_row, v + ((b * seq + j) * kv_heads + kv_h) * hs, hs);
          pdp += p[j] * dp[j];
        }
        double* dq_row = dq + ((b * seq + i) * heads + h) * hs; /* :153-165 */
        for (int64_t j = 0; j < seq; ++j) {
          if (p[j] == 0.0) continue;
          const double ds = p[j] * (dp[j] - pdp) * inv_scale;
          const double* k_row = k + ((b * seq + j) * kv_heads + kv_h) * hs;
          double* dk_row = dk + ((b * seq + j) * kv_heads + kv_h) * hs;
          double* dv_row = dv + ((b * seq + j) * kv_heads + kv_h) * hs;
          for (int64_t s = 0; s < hs; ++s) {
            dq_row[s] += ds * k_row[s];
            dk_row[s] += ds * q_row[s];
            dv_row[s] += p[j] * do_row[s];
          }
        }
      }
    }
  }
  free(p);
  free(dp);
  return 0;
}

/* attention_block_backward (attention.cpp:282-324): dq accumulates,
 * dk_blk / dv_blk are zeroed by the caller. */
static void block_backward(const double* q, const double* k, const double* v,
                           const double* dout, const double* delta, const double* lse,
                           int64_t batch, int64_t q_len, int64_t k_len, int64_t heads,
                           int64_t kv_heads, int64_t hs, int causal, const int64_t* q_pos,
                           const int64_t* k_pos, double* dq, double* dk, double* dv) {
  const int64_t heads_per_kv = heads / kv_heads;
  const double inv_scale = 1.0 / sqrt((double)hs);
  for (int64_t b = 0; b < batch; ++b)
    for (int64_t i = 0; i < q_len; ++i)
      for (int64_t h = 0; h < heads; ++h) {
        const int64_t kv_h = h / heads_per_kv;
        const size_t r = (size_t)((b * q_len + i) * heads + h);
        const double* q_row = q + r * (size_t)hs;
        const double* do_row = dout + r * (size_t)hs;
        double* dq_row = dq + r * (size_t)hs;
        for (int64_t j = 0; j < k_len; ++j) {
          if (causal && k_pos[j] > q_pos[i]) continue;
          const double* k_row = k + ((b * k_len + j) * kv_heads + kv_h) * hs;
          const double* v_row = v + ((b * k_len + j) * kv_heads + kv_h) * hs;
          const double s = dot_d(q_row, k_row, hs) * inv_scale;
          const double p = exp(s - lse[r]);
          const double dp = dot_d(do_row, v_row, hs);
          const double ds = p * (dp - delta[r]) * inv_scale;
          double* dk_row = dk + ((b * k_len + j) * kv_heads + kv_h) * hs;
          double* dv_row = dv + ((b * k_len + j) * kv_heads + kv_h) * hs;
          for (int64_t x = 0; x < hs; ++x) {
            dq_row[x] += ds * k_row[x];
            dk_row[x] += ds * q_row[x];
            dv_row[x] += p * do_row[x];
          }
        }
      }
}

int uo_usp_backward(const double* q, const double* k, const double* v, const double* dout,
                    int64_t batch, int64_t seq, int64_t heads, int64_t kv_heads, int64_t hs,
                    int ulysses, int ring, int causal, double* dq_g, double* dk_g,
                    double* dv_g) {
  /* usp_attention_backward (usp_attention.cpp:68-89) after the forward
   * (:43-65), over every rank of the mesh; ring_attention_backward's
   * circulation (ring_attention.cpp:79-155) is replayed in the same
   * summation order so the result is bitwise the reference's. */
  if (kv_heads % ulysses != 0 || ulysses > kv_heads || heads % ulysses != 0) return -1;
  if (heads % kv_heads != 0) return -1;
  if (causal && seq % (2 * ring) != 0) return -1;
  if (seq % ring != 0 || (seq / ring) % ulysses != 0) return -1;
  const int64_t per_ring = seq / ring;
  const int64_t hl = heads / ulysses, kvl = kv_heads / ulysses;
  int64_t* lists = (int64_t*)malloc(sizeof(int64_t) * (size_t)seq);
  if (causal) uo_zigzag_partition(seq, ring, lists);
  else uo_even_partition(seq, ring, lists);
  const size_t qsz = (size_t)(batch * per_ring * hl * hs), ksz = (size_t)(batch * per_ring * kvl * hs);
  const size_t rows = (size_t)(batch * per_ring * hl);
  double* qh = (double*)malloc(sizeof(double) * qsz * ring);
  double* oh = (double*)malloc(sizeof(double) * qsz * ring);
  double* doh = (double*)malloc(sizeof(double) * qsz * ring);
  double* dqh = (double*)calloc(qsz * ring, sizeof(double));
  double* lse = (double*)malloc(sizeof(double) * rows * ring);
  double* delta = (double*)malloc(sizeof(double) * rows * ring);
  double* kh = (double*)malloc(sizeof(double) * ksz * ring);
  double* vh = (double*)malloc(sizeof(double) * ksz * ring);
  double* contrib_k = (double*)malloc(sizeof(double) * ksz * ring * ring); /* [rank r][block src] */
  double* contrib_v = (double*)malloc(sizeof(double) * ksz * ring * ring);
  for (int u = 0; u < ulysses; ++u) {
    for (int r = 0; r < ring; ++r) {
      const int64_t* pos = lists + (int64_t)r * per_ring;
      for (int64_t b = 0; b < batch; ++b)
        for (int64_t t = 0; t < per_ring; ++t) {
          for (int64_t h = 0; h < hl; ++h) {
            const size_t dst = (size_t)r * qsz + (size_t)(((b * per_ring + t) * hl + h) * hs);
            const size_t src = (size_t)(((b * seq + pos[t]) * heads + u * hl + h) * hs);
            memcpy(qh + dst, q + src, sizeof(double) * (size_t)hs);
            memcpy(doh + dst, dout + src, sizeof(double) * (size_t)hs);
          }
          for (int64_t h = 0; h < kvl; ++h) {
            const size_t dst = (size_t)r * ksz + (size_t)(((b * per_ring + t) * kvl + h) * hs);
            const size_t src = (size_t)(((b * seq + pos[t]) * kv_heads + u * kvl + h) * hs);
            memcpy(kh + dst, k + src, sizeof(double) * (size_t)hs);
            memcpy(vh + dst, v + src, sizeof(double) * (size_t)hs);
          }
        }
    }
    /* forward per ring rank: out_heads + logsumexp */
    for (int r = 0; r < ring; ++r) {
      sm_state st;
      sm_init(&st, batch, per_ring, hl, hs);
      for (int step = 0; step < ring; ++step) {
        const int src = (r - step + ring) % ring;
        sm_update(&st, qh + (size_t)r * qsz, kh + (size_t)src * ksz, vh + (size_t)src * ksz,
                  per_ring, kvl, causal, lists + (int64_t)r * per_ring, lists + (int64_t)src * per_ring);
      }
      sm_finish(&st, oh + (size_t)r * qsz, lse + (size_t)r * rows);
      sm_free(&st);
      for (size_t rr = 0; rr < rows; ++rr) /* output_dot_rows (attention.cpp:266-280) */
        delta[(size_t)r * rows + rr] =
            dot_d(oh + (size_t)r * qsz + rr * (size_t)hs, doh + (size_t)r * qsz + rr * (size_t)hs, hs);
    }
    /* ring backward: every rank's block contributions */
    for (int r = 0; r < ring; ++r)
      for (int step = 0; step < ring; ++step) {
        const int src = (r - step + ring) % ring;
        double* ck = contrib_k + ((size_t)r * ring + src) * ksz;
        double* cv = contrib_v + ((size_t)r * ring + src) * ksz;
        memset(ck, 0, sizeof(double) * ksz);
        memset(cv, 0, sizeof(double) * ksz);
        block_backward(qh + (size_t)r * qsz, kh + (size_t)src * ksz, vh + (size_t)src * ksz,
                       doh + (size_t)r * qsz, delta + (size_t)r * rows, lse + (size_t)r * rows,
                       batch, per_ring, per_ring, hl, kvl, hs, causal, lists + (int64_t)r * per_ring,
                       lists + (int64_t)src * per_ring, dqh + (size_t)r * qsz, ck, cv);
      }
    /* circulation order (ring_attention.cpp:466-500): block o's partial is
     * acc_1 = c(o+1); acc_s = c(o+s) + acc_{s-1}; final = (0 + acc) + c(o) */
    double* acc_k = (double*)malloc(sizeof(double) * ksz);
    double* acc_v = (double*)malloc(sizeof(double) * ksz);
    for (int o = 0; o < ring; ++o) {
      double* fk = (double*)calloc(ksz, sizeof(double));
      double* fv = (double*)calloc(ksz, sizeof(double));
      if (ring > 1) {
        for (int s = 1; s < ring; ++s) {
          const int rr = (o + s) % ring;
          const double* ck = contrib_k + ((size_t)rr * ring + o) * ksz;
          const double* cv = contrib_v + ((size_t)rr * ring + o) * ksz;
          for (size_t e = 0; e < ksz; ++e) {
            acc_k[e] = (s == 1) ? ck[e] : ck[e] + acc_k[e];
            acc_v[e] = (s == 1) ? cv[e] : cv[e] + acc_v[e];
          }
        }
        for (size_t e = 0; e < ksz; ++e) {
          fk[e] += acc_k[e];
          fv[e] += acc_v[e];
        }
      }
      const double* ok = contrib_k + ((size_t)o * ring + o) * ksz;
      const double* ov = contrib_v + ((size_t)o * ring + o) * ksz;
      for (size_t e = 0; e < ksz; ++e) {
        fk[e] += ok[e];
        fv[e] += ov[e];
      }
      /* inverse all-to-alls + place_rows */
      const int64_t* pos = lists + (int64_t)o * per_ring;
      for (int64_t b = 0; b < batch; ++b)
        for (int64_t t = 0; t < per_ring; ++t) {
          for (int64_t h = 0; h < kvl; ++h) {
            const size_t src = (size_t)(((b * per_ring + t) * kvl + h) * hs);
            const size_t dst = (size_t)(((b * seq + pos[t]) * kv_heads + u * kvl + h) * hs);
            memcpy(dk_g + dst, fk + src, sizeof(double) * (size_t)hs);
            memcpy(dv_g + dst, fv + src, sizeof(double) * (size_t)hs);
          }
          for (int64_t h = 0; h < hl; ++h)
            memcpy(dq_g + ((b * seq + pos[t]) * heads + u * hl + h) * hs,
                   dqh + (size_t)o * qsz + (size_t)(((b * per_ring + t) * hl + h) * hs),
                   sizeof(double) * (size_t)hs);
        }
      free(fk);
      free(fv);
    }
    free(acc_k);
    free(acc_v);
    memset(dqh, 0, sizeof(double) * qsz * ring);
  }
  free(lists); free(qh); free(oh); free(doh); free(dqh); free(lse); free(delta);
  free(kh); free(vh); free(contrib_k); free(contrib_v);
  return 0;
}

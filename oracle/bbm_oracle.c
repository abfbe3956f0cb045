/* bbm_oracle.c — CPU oracle (TEST INFRASTRUCTURE ONLY; see bbm_oracle.h).
 * Each function cites the reference file:line it restates. */
#include "bbm_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ rng.hpp */
/* std::mt19937_64 with the standard's pinned parameters (rng.hpp:8-12 relies on it). */
#define MT_N 312
#define MT_M 156
void orc_mt64_seed(orc_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->mti = MT_N;
}

uint64_t orc_mt64_next(orc_mt64* g) {
  static const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (g->mti >= MT_N) {
    int i;
    uint64_t x;
    for (i = 0; i < MT_N - MT_M; ++i) {
      x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
      g->mt[i] = g->mt[i + MT_M] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    for (; i < MT_N - 1; ++i) {
      x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
      g->mt[i] = g->mt[i + (MT_M - MT_N)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    x = (g->mt[MT_N - 1] & UM) | (g->mt[0] & LM);
    g->mt[MT_N - 1] = g->mt[MT_M - 1] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    g->mti = 0;
  }
  uint64_t x = g->mt[g->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

double orc_uniform_unit(orc_mt64* g) { /* rng.hpp:15-17 */
  return (double)(orc_mt64_next(g) >> 11) * 0x1.0p-53;
}
double orc_uniform_pm1(orc_mt64* g) { /* rng.hpp:20-22 */
  return 2.0 * orc_uniform_unit(g) - 1.0;
}
uint64_t orc_uniform_below(orc_mt64* g, uint64_t bound) { /* rng.hpp:25-32 */
  const uint64_t limit = bound * (UINT64_MAX / bound);
  uint64_t draw;
  do {
    draw = orc_mt64_next(g);
  } while (draw >= limit);
  return draw % bound;
}

static void fill_matrix(orc_mt64* g, double* dst, uint64_t count) { /* rng.hpp:35-42 */
  for (uint64_t i = 0; i < count; ++i) {
    const double x = orc_uniform_pm1(g);
    if (dst) dst[i] = x;
  }
}

void orc_make_problem(uint64_t seed, uint64_t slots, uint64_t n, uint64_t d, double* q,
                      double* k, double* v, double* d_out) {
  /* bench.hpp:320-337: per slot q, k, v then d_out, all from one mt19937_64(seed). */
  orc_mt64 g;
  orc_mt64_seed(&g, seed);
  const uint64_t m = n * d;
  for (uint64_t s = 0; s < slots; ++s) {
    fill_matrix(&g, q ? q + s * m : NULL, m);
    fill_matrix(&g, k ? k + s * m : NULL, m);
    fill_matrix(&g, v ? v + s * m : NULL, m);
    fill_matrix(&g, d_out ? d_out + s * m : NULL, m);
  }
}

/* ----------------------------------------------------------------- mask.hpp */
static uint64_t wpr_of(uint64_t n) { return (n + 63) / 64; }

uint32_t orc_popcount_range(const uint64_t* words, uint64_t c0, uint64_t c1) {
  /* mask.hpp:167-179 */
  if (c0 >= c1) return 0;
  const uint64_t w0 = c0 >> 6, w1 = (c1 - 1) >> 6;
  const uint64_t first = ~0ULL << (c0 & 63);
  const uint64_t last = (c1 & 63) ? (~0ULL >> (64 - (c1 & 63))) : ~0ULL;
  if (w0 == w1) return (uint32_t)__builtin_popcountll(words[w0] & first & last);
  uint32_t cnt = (uint32_t)__builtin_popcountll(words[w0] & first) +
                 (uint32_t)__builtin_popcountll(words[w1] & last);
  for (uint64_t w = w0 + 1; w < w1; ++w) cnt += (uint32_t)__builtin_popcountll(words[w]);
  return cnt;
}

void orc_block_sums(const uint64_t* words, uint64_t n, uint64_t bi, uint64_t bj,
                    uint32_t* sums) {
  /* mask.hpp:184-201 */
  const uint64_t rows = (n + bi - 1) / bi, cols = (n + bj - 1) / bj, wpr = wpr_of(n);
  memset(sums, 0, sizeof(uint32_t) * rows * cols);
  for (uint64_t p = 0; p < rows; ++p) {
    const uint64_t i0 = p * bi, i1 = (i0 + bi < n) ? i0 + bi : n;
    for (uint64_t i = i0; i < i1; ++i)
      for (uint64_t q = 0; q < cols; ++q) {
        const uint64_t c0 = q * bj, c1 = (c0 + bj < n) ? c0 + bj : n;
        sums[p * cols + q] += orc_popcount_range(words + i * wpr, c0, c1);
      }
  }
}

static uint32_t block_area(uint64_t n, uint64_t bi, uint64_t bj, uint64_t p, uint64_t q) {
  /* mask.hpp:89-99 */
  const uint64_t ri = (bi < n - p * bi) ? bi : n - p * bi;
  const uint64_t cj = (bj < n - q * bj) ? bj : n - q * bj;
  return (uint32_t)(ri * cj);
}

void orc_block_occupancy(const uint32_t* sums, uint64_t rows, uint64_t cols, uint8_t* occ) {
  /* mask.hpp:203-209 */
  for (uint64_t t = 0; t < rows * cols; ++t) occ[t] = sums[t] > 0 ? 1 : 0;
}

void orc_dense_runs(const uint32_t* sums, uint64_t n, uint64_t bi, uint64_t bj,
                    uint32_t* offset, uint32_t* total_ones) {
  /* mask.hpp:213-228: first maximal run of full blocks per row block, (0,0) if none. */
  const uint64_t rows = (n + bi - 1) / bi, cols = (n + bj - 1) / bj;
  for (uint64_t p = 0; p < rows; ++p) {
    offset[p] = 0;
    total_ones[p] = 0;
    for (uint64_t q = 0; q < cols; ++q) {
      if (sums[p * cols + q] != block_area(n, bi, bj, p, q)) continue;
      uint64_t end = q + 1;
      while (end < cols && sums[p * cols + end] == block_area(n, bi, bj, p, end)) ++end;
      offset[p] = (uint32_t)q;
      total_ones[p] = (uint32_t)(end - q);
      break;
    }
  }
}

void orc_block_stats(const uint32_t* sums, uint64_t n, uint64_t bi, uint64_t bj,
                     orc_block_stats_t* out) {
  /* mask.hpp:230-247 */
  const uint64_t rows = (n + bi - 1) / bi, cols = (n + bj - 1) / bj;
  uint64_t ones = 0;
  out->blocks_total = rows * cols;
  out->blocks_nonzero = 0;
  out->blocks_full = 0;
  for (uint64_t p = 0; p < rows; ++p)
    for (uint64_t q = 0; q < cols; ++q) {
      const uint32_t s = sums[p * cols + q];
      ones += s;
      if (s > 0) ++out->blocks_nonzero;
      if (s == block_area(n, bi, bj, p, q)) ++out->blocks_full;
    }
  const double nd = (double)n;
  out->block_density =
      out->blocks_total ? (double)out->blocks_nonzero / (double)out->blocks_total : 0.0;
  out->element_density = nd > 0 ? (double)ones / (nd * nd) : 0.0;
}

/* --------------------------------------------------------------- engine.hpp */
void orc_counters(const uint32_t* sums, const uint32_t* offset, const uint32_t* total_ones,
                  uint64_t n, uint64_t bi, uint64_t bj, int variant, orc_counters_t* c) {
  /* engine.hpp:118-153 (classify_tile) walked over every (p, q) as blocked_forward does
   * (engine.hpp:311-314). */
  const uint64_t rows = (n + bi - 1) / bi, cols = (n + bj - 1) / bj;
  memset(c, 0, sizeof(*c));
  for (uint64_t p = 0; p < rows; ++p)
    for (uint64_t q = 0; q < cols; ++q) {
      ++c->blocks_visited;
      const int occ = sums[p * cols + q] > 0;
      switch (variant) {
        case ORC_DENSE: ++c->blocks_processed; break;
        case ORC_NAIVE: ++c->mask_block_reads; ++c->blocks_processed; break;
        case ORC_BINBLK:
          if (!occ) { ++c->skipped_by_binblk; break; }
          ++c->mask_block_reads; ++c->blocks_processed; break;
        case ORC_DENSE_BINBLK:
          if (!occ) { ++c->skipped_by_binblk; break; }
          ++c->blocks_processed;
          if (q >= offset[p] && q < (uint64_t)offset[p] + total_ones[p]) /* mask.hpp:143-145 */
            ++c->skipped_mask_reads_by_run;
          else
            ++c->mask_block_reads;
          break;
      }
    }
}

/* ------------------------------------------------------------ reference.hpp */
typedef struct {
  const double *q, *k, *v;
  uint64_t n, d, dv;
  double scale;
  const uint64_t* words; /* NULL = every key visible */
  double *out, *row_max, *row_sum;
  uint64_t r0, r1;
} fwd_job;

static int visible(const fwd_job* j, uint64_t i, uint64_t c) {
  if (!j->words) return 1;
  return (int)((j->words[i * wpr_of(j->n) + (c >> 6)] >> (c & 63)) & 1ULL);
}

static void* fwd_rows(void* arg) {
  /* reference.hpp:52-79, one query row at a time. */
  const fwd_job* j = (const fwd_job*)arg;
  const uint64_t n = j->n, d = j->d, dv = j->dv;
  double* scores = (double*)malloc(sizeof(double) * (n ? n : 1));
  for (uint64_t i = j->r0; i < j->r1; ++i) {
    double m = -INFINITY;
    for (uint64_t c = 0; c < n; ++c) {
      if (!visible(j, i, c)) continue;
      double s = 0.0;
      for (uint64_t t = 0; t < d; ++t) s += j->q[i * d + t] * j->k[c * d + t];
      scores[c] = j->scale * s;
      if (scores[c] > m) m = scores[c];
    }
    j->row_max[i] = m;
    double* orow = j->out + i * dv;
    for (uint64_t t = 0; t < dv; ++t) orow[t] = 0.0;
    if (isinf(m)) { /* no visible key: zero output by convention (reference.hpp:63-67) */
      j->row_sum[i] = 0.0;
      continue;
    }
    double l = 0.0;
    for (uint64_t c = 0; c < n; ++c) {
      if (!visible(j, i, c)) continue;
      const double p = exp(scores[c] - m);
      l += p;
      for (uint64_t t = 0; t < dv; ++t) orow[t] += p * j->v[c * dv + t];
    }
    j->row_sum[i] = l;
    for (uint64_t t = 0; t < dv; ++t) orow[t] /= l;
  }
  free(scores);
  return NULL;
}

static void run_forward(const double* q, const double* k, const double* v, uint64_t n,
                        uint64_t d, uint64_t dv, double scale, const uint64_t* words,
                        double* out, double* row_max, double* row_sum, int threads) {
  if (threads < 1) threads = 1;
  if ((uint64_t)threads > n) threads = (int)(n ? n : 1);
  pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  fwd_job* jobs = (fwd_job*)malloc(sizeof(fwd_job) * threads);
  for (int t = 0; t < threads; ++t) {
    fwd_job j = {q, k, v, n, d, dv, scale, words, out, row_max, row_sum,
                 n * (uint64_t)t / threads, n * (uint64_t)(t + 1) / threads};
    jobs[t] = j;
    if (threads == 1)
      fwd_rows(&jobs[t]);
    else
      pthread_create(&tid[t], NULL, fwd_rows, &jobs[t]);
  }
  if (threads > 1)
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  free(tid);
  free(jobs);
}

void orc_naive_forward(const double* q, const double* k, const double* v, uint64_t n,
                       uint64_t d, uint64_t dv, double scale, const uint64_t* words,
                       double* out, double* row_max, double* row_sum, int threads) {
  run_forward(q, k, v, n, d, dv, scale, words, out, row_max, row_sum, threads);
}

void orc_dense_forward(const double* q, const double* k, const double* v, uint64_t n,
                       uint64_t d, uint64_t dv, double scale, double* out, double* row_max,
                       double* row_sum, int threads) {
  /* Variant::dense ignores the mask (engine.hpp:122-124): every key is visible. */
  run_forward(q, k, v, n, d, dv, scale, NULL, out, row_max, row_sum, threads);
}

/* reference.hpp:84-139 — naive_backward: gradients of L = sum(out * d_out), one query row at a
 * time in double. words == NULL: every key visible (the dense variant). Threads split the query
 * rows; each owns private dk/dv accumulators, summed afterwards in thread order. */
typedef struct {
  const double *q, *k, *v, *dout;
  uint64_t n, d;
  double scale;
  const uint64_t* words;
  double *dq, *dk, *dv; /* dq: shared (rows owned); dk, dv: private */
  uint64_t r0, r1;
} bwd_job;

static void* bwd_rows(void* arg) {
  const bwd_job* j = (const bwd_job*)arg;
  const uint64_t n = j->n, d = j->d, wpr = wpr_of(n);
  double* s = (double*)malloc(sizeof(double) * (n ? n : 1));
  double* p = (double*)malloc(sizeof(double) * (n ? n : 1));
  double* dp = (double*)malloc(sizeof(double) * (n ? n : 1));
  for (uint64_t i = j->r0; i < j->r1; ++i) {
    double m = -INFINITY;
    for (uint64_t c = 0; c < n; ++c) {
      if (j->words && !((j->words[i * wpr + (c >> 6)] >> (c & 63)) & 1u)) continue;
      double t = 0.0;
      for (uint64_t x = 0; x < d; ++x) t += j->q[i * d + x] * j->k[c * d + x];
      s[c] = j->scale * t;
      if (s[c] > m) m = s[c];
    }
    if (isinf(m)) continue; /* fully masked row contributes nothing */
    double l = 0.0;
    for (uint64_t c = 0; c < n; ++c) {
      if (j->words && !((j->words[i * wpr + (c >> 6)] >> (c & 63)) & 1u)) continue;
      p[c] = exp(s[c] - m);
      l += p[c];
    }
    double delta = 0.0;
    for (uint64_t c = 0; c < n; ++c) {
      if (j->words && !((j->words[i * wpr + (c >> 6)] >> (c & 63)) & 1u)) continue;
      p[c] /= l;
      double t = 0.0;
      for (uint64_t x = 0; x < d; ++x) t += j->dout[i * d + x] * j->v[c * d + x];
      dp[c] = t;
      delta += p[c] * t;
    }
    for (uint64_t c = 0; c < n; ++c) {
      if (j->words && !((j->words[i * wpr + (c >> 6)] >> (c & 63)) & 1u)) continue;
      const double ds = p[c] * (dp[c] - delta);
      for (uint64_t x = 0; x < d; ++x) {
        j->dq[i * d + x] += j->scale * ds * j->k[c * d + x];
        j->dk[c * d + x] += j->scale * ds * j->q[i * d + x];
      }
      for (uint64_t x = 0; x < d; ++x) j->dv[c * d + x] += p[c] * j->dout[i * d + x];
    }
  }
  free(s);
  free(p);
  free(dp);
  return NULL;
}

void orc_naive_backward(const double* q, const double* k, const double* v, const double* dout,
                        uint64_t n, uint64_t d, double scale, const uint64_t* words, double* dq,
                        double* dk, double* dv, int threads) {
  if (threads < 1) threads = 1;
  if ((uint64_t)threads > n) threads = (int)(n ? n : 1);
  pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  bwd_job* jobs = (bwd_job*)malloc(sizeof(bwd_job) * threads);
  const uint64_t nd = n * d;
  double* priv = (double*)calloc(2 * nd * (uint64_t)threads + 1, sizeof(double));
  memset(dq, 0, sizeof(double) * nd);
  for (int t = 0; t < threads; ++t) {
    bwd_job jb = {q, k, v, dout, n, d, scale, words, dq, priv + 2 * nd * t, priv + 2 * nd * t + nd,
                  n * (uint64_t)t / threads, n * (uint64_t)(t + 1) / threads};
    jobs[t] = jb;
    if (threads == 1)
      bwd_rows(&jobs[t]);
    else
      pthread_create(&tid[t], NULL, bwd_rows, &jobs[t]);
  }
  if (threads > 1)
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  for (uint64_t e = 0; e < nd; ++e) {
    double a = 0.0, b = 0.0;
    for (int t = 0; t < threads; ++t) {
      a += priv[2 * nd * t + e];
      b += priv[2 * nd * t + nd + e];
    }
    dk[e] = a;
    dv[e] = b;
  }
  free(priv);
  free(tid);
  free(jobs);
}

/* reference.hpp:42-81 (forward) and the dq half of reference.hpp:84-139 (backward) for a LIST
 * of query rows only — each row needs nothing but its own softmax, so full-size problems can be
 * spot-checked row by row. Outputs are indexed by list position: out [nrows][d], row_max /
 * row_sum [nrows], dq [nrows][d] (skipped when dout == NULL). words == NULL: every key visible. */
void orc_naive_rows(const double* q, const double* k, const double* v, const double* dout,
                    uint64_t n, uint64_t d, double scale, const uint64_t* words,
                    const uint64_t* rows, uint64_t nrows, double* out, double* row_max,
                    double* row_sum, double* dq) {
  const uint64_t wpr = wpr_of(n);
  double* s = (double*)malloc(sizeof(double) * (n ? n : 1));
  double* dp = (double*)malloc(sizeof(double) * (n ? n : 1));
  for (uint64_t r = 0; r < nrows; ++r) {
    const uint64_t i = rows[r];
    double m = -INFINITY;
    for (uint64_t c = 0; c < n; ++c) {
      if (words && !((words[i * wpr + (c >> 6)] >> (c & 63)) & 1u)) continue;
      double t = 0.0;
      for (uint64_t x = 0; x < d; ++x) t += q[i * d + x] * k[c * d + x];
      s[c] = scale * t;
      if (s[c] > m) m = s[c];
    }
    row_max[r] = m;
    for (uint64_t x = 0; x < d; ++x) out[r * d + x] = 0.0;
    if (dq)
      for (uint64_t x = 0; x < d; ++x) dq[r * d + x] = 0.0;
    if (isinf(m)) { /* no visible key: zero output, nothing flows back */
      row_sum[r] = 0.0;
      continue;
    }
    double l = 0.0;
    for (uint64_t c = 0; c < n; ++c) {
      if (words && !((words[i * wpr + (c >> 6)] >> (c & 63)) & 1u)) continue;
      const double p = exp(s[c] - m);
      s[c] = p;
      l += p;
      for (uint64_t x = 0; x < d; ++x) out[r * d + x] += p * v[c * d + x];
    }
    row_sum[r] = l;
    for (uint64_t x = 0; x < d; ++x) out[r * d + x] /= l;
    if (!dq) continue;
    double delta = 0.0;
    for (uint64_t c = 0; c < n; ++c) {
      if (words && !((words[i * wpr + (c >> 6)] >> (c & 63)) & 1u)) continue;
      s[c] /= l;
      double t = 0.0;
      for (uint64_t x = 0; x < d; ++x) t += dout[i * d + x] * v[c * d + x];
      dp[c] = t;
      delta += s[c] * t;
    }
    for (uint64_t c = 0; c < n; ++c) {
      if (words && !((words[i * wpr + (c >> 6)] >> (c & 63)) & 1u)) continue;
      const double ds = s[c] * (dp[c] - delta);
      for (uint64_t x = 0; x < d; ++x) dq[r * d + x] += scale * ds * k[c * d + x];
    }
  }
  free(s);
  free(dp);
}

/* -------------------------------------------------------------- reorder.hpp */
typedef struct {
  uint64_t n;
  uint64_t* start; /* n+1 */
  uint32_t* adj;
} csr_graph;

static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}

static int build_graph(const uint64_t* words, uint64_t n, csr_graph* g) {
  /* reorder.hpp:28-49: edge i-j iff mask(i,j) or mask(j,i), self loops dropped, neighbor
   * lists sorted and de-duplicated. */
  const uint64_t wpr = wpr_of(n);
  uint64_t* cnt = (uint64_t*)calloc(n + 1, sizeof(uint64_t));
  if (!cnt) return -1;
  for (uint64_t i = 0; i < n; ++i)
    for (uint64_t w = 0; w < wpr; ++w) {
      uint64_t bits = words[i * wpr + w];
      while (bits) {
        const uint64_t j = w * 64 + (uint64_t)__builtin_ctzll(bits);
        bits &= bits - 1;
        if (j == i) continue;
        cnt[i]++;
        cnt[j]++;
      }
    }
  uint64_t* start = (uint64_t*)malloc(sizeof(uint64_t) * (n + 1));
  start[0] = 0;
  for (uint64_t i = 0; i < n; ++i) start[i + 1] = start[i] + cnt[i];
  uint32_t* adj = (uint32_t*)malloc(sizeof(uint32_t) * (start[n] ? start[n] : 1));
  uint64_t* fill = cnt; /* reuse as cursor */
  for (uint64_t i = 0; i < n; ++i) fill[i] = start[i];
  for (uint64_t i = 0; i < n; ++i)
    for (uint64_t w = 0; w < wpr; ++w) {
      uint64_t bits = words[i * wpr + w];
      while (bits) {
        const uint64_t j = w * 64 + (uint64_t)__builtin_ctzll(bits);
        bits &= bits - 1;
        if (j == i) continue;
        adj[fill[i]++] = (uint32_t)j;
        adj[fill[j]++] = (uint32_t)i;
      }
    }
  /* sort + unique each list, compacting in place */
  uint64_t out = 0;
  uint64_t* nstart = (uint64_t*)malloc(sizeof(uint64_t) * (n + 1));
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t b = start[i], e = start[i + 1];
    qsort(adj + b, e - b, sizeof(uint32_t), cmp_u32);
    nstart[i] = out;
    for (uint64_t t = b; t < e; ++t)
      if (t == b || adj[t] != adj[t - 1]) adj[out++] = adj[t];
  }
  nstart[n] = out;
  free(start);
  free(cnt);
  g->n = n;
  g->start = nstart;
  g->adj = adj;
  return 0;
}

static const csr_graph* g_sort_graph;
static uint64_t deg(const csr_graph* g, uint32_t a) { return g->start[a + 1] - g->start[a]; }
static int by_degree_then_index(const void* pa, const void* pb) {
  /* reorder.hpp:92-95 */
  const uint32_t a = *(const uint32_t*)pa, b = *(const uint32_t*)pb;
  const uint64_t da = deg(g_sort_graph, a), db = deg(g_sort_graph, b);
  if (da != db) return da < db ? -1 : 1;
  return (a > b) - (a < b);
}

int orc_rcm_order(const uint64_t* words, uint64_t n, uint32_t* forward) {
  /* reorder.hpp:85-133 */
  csr_graph g;
  if (build_graph(words, n, &g) != 0) return -1;
  g_sort_graph = &g;
  char* visited = (char*)calloc(n ? n : 1, 1);
  uint32_t* component = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  uint32_t* order = forward;
  uint64_t order_len = 0;
  for (uint64_t seed = 0; seed < n; ++seed) {
    if (visited[seed]) continue;
    uint64_t comp_len = 1;
    component[0] = (uint32_t)seed;
    visited[seed] = 1;
    for (uint64_t h = 0; h < comp_len; ++h) {
      const uint32_t node = component[h];
      for (uint64_t e = g.start[node]; e < g.start[node + 1]; ++e) {
        const uint32_t nb = g.adj[e];
        if (!visited[nb]) {
          visited[nb] = 1;
          component[comp_len++] = nb;
        }
      }
    }
    uint32_t start = component[0];
    for (uint64_t t = 0; t < comp_len; ++t) {
      const uint32_t node = component[t];
      const uint64_t dn = deg(&g, node), ds = deg(&g, start);
      if (dn < ds || (dn == ds && node < start)) start = node;
    }
    for (uint64_t t = 0; t < comp_len; ++t) visited[component[t]] = 0;
    const uint64_t bfs_begin = order_len;
    order[order_len++] = start;
    visited[start] = 1;
    for (uint64_t h = bfs_begin; h < order_len; ++h) {
      const uint32_t node = order[h];
      const uint64_t f0 = order_len;
      for (uint64_t e = g.start[node]; e < g.start[node + 1]; ++e) {
        const uint32_t nb = g.adj[e];
        if (!visited[nb]) {
          visited[nb] = 1;
          order[order_len++] = nb;
        }
      }
      qsort(order + f0, order_len - f0, sizeof(uint32_t), by_degree_then_index);
    }
  }
  for (uint64_t a = 0, b = n ? n - 1 : 0; a < b; ++a, --b) { /* reorder.hpp:130 reverse */
    const uint32_t t = order[a];
    order[a] = order[b];
    order[b] = t;
  }
  free(visited);
  free(component);
  free(g.start);
  free(g.adj);
  return 0;
}

uint64_t orc_bandwidth(const uint64_t* words, uint64_t n) {
  /* reorder.hpp:137-153 */
  const uint64_t wpr = wpr_of(n);
  uint64_t bw = 0;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t first = n, last = 0;
    for (uint64_t w = 0; w < wpr; ++w) {
      const uint64_t x = words[i * wpr + w];
      if (!x) continue;
      const uint64_t f = w * 64 + (uint64_t)__builtin_ctzll(x);
      const uint64_t l = w * 64 + 63 - (uint64_t)__builtin_clzll(x);
      if (f < first) first = f;
      if (l > last) last = l;
    }
    if (first == n) continue;
    if (first < i && i - first > bw) bw = i - first;
    if (last > i && last - i > bw) bw = last - i;
  }
  return bw;
}

void orc_permute_mask(const uint64_t* words, uint64_t n, const uint32_t* fwd,
                      uint64_t* out_words) {
  /* reorder.hpp:156-163: mask'(a,b) = mask(fwd[a], fwd[b]) */
  const uint64_t wpr = wpr_of(n);
  memset(out_words, 0, sizeof(uint64_t) * n * wpr);
  for (uint64_t a = 0; a < n; ++a) {
    const uint64_t* src = words + (uint64_t)fwd[a] * wpr;
    for (uint64_t b = 0; b < n; ++b) {
      const uint64_t c = fwd[b];
      if ((src[c >> 6] >> (c & 63)) & 1ULL) out_words[a * wpr + (b >> 6)] |= 1ULL << (b & 63);
    }
  }
}

void orc_permute_rows(const void* src, void* dst, uint64_t rows, uint64_t row_bytes,
                      const uint32_t* fwd, int inverse) {
  /* reorder.hpp:167-189: permute_rows out[a] = in[fwd[a]]; unpermute_rows out[fwd[a]] = in[a] */
  const char* s = (const char*)src;
  char* d = (char*)dst;
  for (uint64_t a = 0; a < rows; ++a) {
    if (!inverse)
      memcpy(d + a * row_bytes, s + (uint64_t)fwd[a] * row_bytes, row_bytes);
    else
      memcpy(d + (uint64_t)fwd[a] * row_bytes, s + a * row_bytes, row_bytes);
  }
}

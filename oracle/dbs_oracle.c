/*
 * dbs_oracle.c -- CPU restatement of the reference DBS hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  The product path (paper_2007_11831_b200/) never links or calls
 * it.  Built by oracle/Makefile into oracle/libdbs_oracle.so (plain gcc,
 * -O2 -ffp-contract=off so no FMA contraction changes fp64 bits).
 *
 * Every function cites the reference line it restates (paths relative to
 * /root/reference/pkg/src/dbsim/).  Pinned against the reference's own known
 * answers and against golden vectors produced by running the reference in
 * this container (tests/golden/gen_golden.py, tests/test_oracle.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/dbs_b200.h"

/* ---------------------------------------------------------------------- */
/* math.fsum  (CPython Modules/mathmodule.c math_fsum, Shewchuk partials)  */
/* used at allocation.py:101 and :111                                      */
/* ---------------------------------------------------------------------- */
#define FSUM_MAX_PARTIALS 256
int oracle_fsum(const double* v, int64_t n, double* out) {
  double p[FSUM_MAX_PARTIALS];
  int m = 0;
  double special_sum = 0.0, inf_sum = 0.0;
  for (int64_t k = 0; k < n; k++) {
    double x = v[k];
    double xsave = x;
    int i = 0;
    for (int j = 0; j < m; j++) {
      double y = p[j];
      if (fabs(x) < fabs(y)) { double t = x; x = y; y = t; }
      double hi = x + y;
      double yr = hi - x;
      double lo = y - yr;
      if (lo != 0.0) p[i++] = lo;
      x = hi;
    }
    m = i;
    if (x != 0.0) {
      if (!isfinite(x)) {
        if (isfinite(xsave)) return DBS_ERR_FSUM_OVERFLOW;
        if (isinf(xsave)) inf_sum += xsave;
        special_sum += xsave;
        m = 0;
      } else {
        if (m >= FSUM_MAX_PARTIALS) return DBS_ERR_ARGUMENT;
        p[m++] = x;
      }
    }
  }
  if (special_sum != 0.0) {
    if (isnan(inf_sum)) return DBS_ERR_FSUM_INF_NAN;
    *out = special_sum;
    return DBS_OK;
  }
  double hi = 0.0, lo = 0.0;
  if (m > 0) {
    hi = p[--m];
    while (m > 0) {
      double x = hi;
      double y = p[--m];
      hi = x + y;
      double yr = hi - x;
      lo = y - yr;
      if (lo != 0.0) break;
    }
    if (m > 0 && ((lo < 0.0 && p[m - 1] < 0.0) || (lo > 0.0 && p[m - 1] > 0.0))) {
      double y = lo * 2.0;
      double x = hi + y;
      double yr = x - hi;
      if (y == yr) hi = x;
    }
  }
  *out = hi;
  return DBS_OK;
}

/* allocation.evaluate_performance  allocation.py:78-88 */
int oracle_evaluate_performance(double share, double t, double* out) {
  if (!(0.0 < share && share <= 1.0) || !isfinite(share)) return DBS_ERR_INVALID_MEASUREMENT;
  if (t <= 0.0 || !isfinite(t)) return DBS_ERR_INVALID_MEASUREMENT;
  *out = share / t;
  return DBS_OK;
}

/* allocation.compute_batch_fractions  allocation.py:91-102 */
int oracle_compute_batch_fractions(const double* perf, int64_t n, double* out) {
  if (n <= 0) return DBS_ERR_INVALID_PERFORMANCE;
  for (int64_t i = 0; i < n; i++)
    if (perf[i] <= 0.0 || !isfinite(perf[i])) return DBS_ERR_INVALID_PERFORMANCE;
  double total;
  int st = oracle_fsum(perf, n, &total);
  if (st) return st;
  for (int64_t i = 0; i < n; i++) out[i] = perf[i] / total;
  return DBS_OK;
}

/* allocation.scale_to_real_batches  allocation.py:105-113 */
int oracle_scale_to_real_batches(const double* f, int64_t n, int64_t budget, double* out) {
  if (budget < n) return DBS_ERR_BUDGET_TOO_SMALL;
  double s;
  int st = oracle_fsum(f, n, &s);
  if (st) return st;
  if (fabs(s - 1.0) > 1e-6) return DBS_ERR_INVALID_PERFORMANCE;
  double b = (double)budget;
  for (int64_t i = 0; i < n; i++) out[i] = f[i] * b;
  return DBS_OK;
}

/* allocation.round_twice  allocation.py:116-137 */
int oracle_round_twice(const double* real, int64_t n, int64_t budget, int64_t* out) {
  for (int64_t i = 0; i < n; i++)
    if (real[i] < 0.0 || !isfinite(real[i])) return DBS_ERR_INVALID_BATCH;
  __int128 sum = 0;
  for (int64_t i = 0; i < n; i++) {
    double f = floor(real[i]);
    if (f >= 9.2e18) return DBS_ERR_INT_OVERFLOW;
    out[i] = (int64_t)f;
    sum += out[i];
  }
  __int128 k = (__int128)budget - sum;
  /* candidates: d >= 0.5, order (-d, i); the first max(k,0) get +1 */
  int64_t* cand = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  int64_t nc = 0;
  for (int64_t i = 0; i < n; i++) {
    double d = real[i] - (double)out[i];
    if (d >= 0.5) {
      /* insertion keeps the stable (-d, i) order */
      int64_t pos = nc;
      while (pos > 0) {
        double dp = real[cand[pos - 1]] - (double)out[cand[pos - 1]];
        if (dp < d) { cand[pos] = cand[pos - 1]; pos--; } else break;
      }
      cand[pos] = i;
      nc++;
    }
  }
  int64_t take = k > 0 ? (k < nc ? (int64_t)k : nc) : 0;
  for (int64_t c = 0; c < take; c++) out[cand[c]] += 1;
  free(cand);
  return DBS_OK;
}

/* allocation._raise_zero_batches  allocation.py:191-204 */
int oracle_raise_zero_batches(const int64_t* in, int64_t n, int64_t* out) {
  memcpy(out, in, sizeof(int64_t) * (size_t)n);
  for (;;) {
    int64_t zero = -1;
    for (int64_t i = 0; i < n; i++) if (out[i] == 0) { zero = i; break; }
    if (zero < 0) break;
    int64_t donor = 0;
    for (int64_t i = 1; i < n; i++) if (out[i] > out[donor]) donor = i;
    if (out[donor] <= 1) break;
    out[zero] += 1;
    out[donor] -= 1;
  }
  return DBS_OK;
}

/* allocation.partition_ranges  allocation.py:140-155 */
int oracle_partition_ranges(const int64_t* b, int64_t n, int64_t* cum) {
  if (n <= 0) return DBS_ERR_EMPTY_PARTITION;
  for (int64_t i = 0; i < n; i++) if (b[i] < 0) return DBS_ERR_INVALID_BATCH;
  cum[0] = 0;
  for (int64_t i = 0; i < n; i++) {
    if (cum[i] > INT64_MAX - b[i]) return DBS_ERR_INT_OVERFLOW;
    cum[i + 1] = cum[i] + b[i];
  }
  if (cum[n] == 0) return DBS_ERR_EMPTY_PARTITION;
  return DBS_OK;
}

static int64_t floordiv128(__int128 a, __int128 b) {
  __int128 q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) q -= 1;
  return (int64_t)q;
}

/* bound arithmetic with Python's int/Fraction/float promotion rules */
static double bound_as_double(const dbs_bound* x) {
  return x->kind == 1 ? x->value : (double)x->num / (double)x->den;
}
static int width_positive(const dbs_bound* lo, const dbs_bound* hi) {
  if (lo->kind == 0 && hi->kind == 0)
    return (__int128)hi->num * lo->den > (__int128)lo->num * hi->den;
  return bound_as_double(hi) - bound_as_double(lo) > 0.0;
}
static int64_t floor_times(const dbs_bound* lo, int64_t D) {
  if (lo->kind == 0) return floordiv128((__int128)lo->num * D, lo->den);
  return (int64_t)floor(lo->value * (double)D);
}

/* allocation.spans_from_ranges  allocation.py:158-188 */
int oracle_spans_from_ranges(const dbs_bound* lo, const dbs_bound* hi, int64_t n, int64_t D,
                             int64_t* spans) {
  if (D < n) return DBS_ERR_DATASET_TOO_SMALL;
  if (n <= 0) return DBS_ERR_ARGUMENT;
  int64_t* starts = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  char* pos = (char*)malloc((size_t)n);
  for (int64_t i = 0; i < n; i++) {
    pos[i] = (char)width_positive(&lo[i], &hi[i]);
    starts[i] = floor_times(&lo[i], D);
  }
  starts[0] = 0;
  for (int64_t i = 1; i < n; i++) {
    int64_t least = starts[i - 1] + (pos[i - 1] ? 1 : 0);
    if (starts[i] < least) starts[i] = least;
  }
  int64_t cap = D;
  for (int64_t i = n - 1; i > 0; i--) {
    if (pos[i]) cap -= 1;
    if (starts[i] > cap) starts[i] = cap;
  }
  for (int64_t i = 0; i < n; i++) {
    spans[2 * i] = starts[i];
    spans[2 * i + 1] = (i + 1 < n) ? starts[i + 1] : D;
  }
  free(starts);
  free(pos);
  return DBS_OK;
}

/* allocation.plan_next_epoch  allocation.py:207-244 */
int oracle_plan_next_epoch(const double* shares, const double* times, int64_t n, int64_t B,
                           int64_t D, int64_t epoch, int64_t* int_batches, int64_t* cum,
                           int64_t* spans) {
  if (n <= 0) return DBS_ERR_INVALID_PERFORMANCE;
  if (B < n) return DBS_ERR_BUDGET_TOO_SMALL;
  double* real = (double*)malloc(sizeof(double) * (size_t)n);
  double* tmp = (double*)malloc(sizeof(double) * (size_t)n);
  int64_t* ints = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int st = DBS_OK;
  if (epoch == 0) {
    double e = (double)B / (double)n;
    for (int64_t i = 0; i < n; i++) real[i] = e;
  } else {
    for (int64_t i = 0; i < n && !st; i++) st = oracle_evaluate_performance(shares[i], times[i], &tmp[i]);
    if (!st) st = oracle_compute_batch_fractions(tmp, n, real);
    if (!st) { memcpy(tmp, real, sizeof(double) * (size_t)n); st = oracle_scale_to_real_batches(tmp, n, B, real); }
  }
  if (!st) st = oracle_round_twice(real, n, B, ints);
  if (!st) st = oracle_raise_zero_batches(ints, n, int_batches);
  if (!st) st = oracle_partition_ranges(int_batches, n, cum);
  if (!st) {
    dbs_bound* lo = (dbs_bound*)calloc((size_t)n, sizeof(dbs_bound));
    dbs_bound* hi = (dbs_bound*)calloc((size_t)n, sizeof(dbs_bound));
    for (int64_t i = 0; i < n; i++) {
      lo[i].num = cum[i]; lo[i].den = cum[n];
      hi[i].num = cum[i + 1]; hi[i].den = cum[n];
    }
    st = oracle_spans_from_ranges(lo, hi, n, D, spans);
    free(lo); free(hi);
  }
  free(real); free(tmp); free(ints);
  return st;
}

/* cluster.iterations_for_plan  cluster.py:159-170 */
int64_t oracle_iterations_for_plan(const int64_t* b, const int64_t* spans, int64_t n) {
  int64_t best = -1;
  for (int64_t i = 0; i < n; i++) {
    if (b[i] <= 0) continue;
    int64_t c = (spans[2 * i + 1] - spans[2 * i]) / b[i];
    if (best < 0 || c < best) best = c;
  }
  return best < 0 ? 0 : best;
}

/* cluster.run_training DBS re-plan  cluster.py:253-271 (+ even_plan 223-231).
 * prev_spans: previous plan; times: previous per_worker_gpu; smoothed/has_smoothed
 * carry the EMA state. */
int oracle_replan(const int64_t* prev_spans, const double* times, int64_t n, int64_t B, int64_t D,
                  int64_t epoch, int adaptive, double a, double* smoothed, int* has_smoothed,
                  int64_t* int_batches, int64_t* cum, int64_t* spans) {
  if (!adaptive || epoch == 0) {
    double* s = (double*)malloc(sizeof(double) * (size_t)n);
    double* t = (double*)malloc(sizeof(double) * (size_t)n);
    for (int64_t i = 0; i < n; i++) { s[i] = 1.0 / (double)n; t[i] = 1.0; }
    int st = oracle_plan_next_epoch(s, t, n, B, D, 0, int_batches, cum, spans);
    free(s); free(t);
    return st;
  }
  double* shares = (double*)malloc(sizeof(double) * (size_t)n);
  double* perfs = (double*)malloc(sizeof(double) * (size_t)n);
  double* tt = (double*)malloc(sizeof(double) * (size_t)n);
  int64_t prevD = prev_spans[2 * n - 1];
  int st = DBS_OK;
  for (int64_t i = 0; i < n; i++)
    shares[i] = (double)(prev_spans[2 * i + 1] - prev_spans[2 * i]) / (double)prevD;
  for (int64_t i = 0; i < n && !st; i++) st = oracle_evaluate_performance(shares[i], times[i], &perfs[i]);
  if (!st) {
    if (a > 0.0 && *has_smoothed)
      for (int64_t i = 0; i < n; i++) perfs[i] = a * smoothed[i] + (1.0 - a) * perfs[i];
    for (int64_t i = 0; i < n; i++) smoothed[i] = perfs[i];
    *has_smoothed = 1;
    for (int64_t i = 0; i < n; i++) tt[i] = shares[i] / perfs[i];
    st = oracle_plan_next_epoch(shares, tt, n, B, D, epoch, int_batches, cum, spans);
  }
  free(shares); free(perfs); free(tt);
  return st;
}

/* ---------------------------------------------------------------------- */
/* numpy Generator(PCG64): SeedSequence + PCG64 XSL-RR + permutation       */
/* (numpy 2.3 bit_generator.pyx SeedSequence, pcg64.h, distributions.c     */
/* random_interval, _generator.pyx shuffle) -- sgdlab.py:358, 372-374      */
/* ---------------------------------------------------------------------- */
typedef unsigned __int128 u128;
static const u128 PCG_MULT = (((u128)0x2360ED051FC65DA4ULL) << 64) | 0x4385DF649FCCF645ULL;

int oracle_pcg64_seed(const uint32_t* words, int32_t nw, dbs_pcg64* out) {
  const uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu,
                 MULT_B = 0x58f38dedu, MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
  uint32_t zero = 0;
  if (nw <= 0) { words = &zero; nw = 1; }
  uint32_t hc = INIT_A, pool[4];
#define HASHMIX(val, res) do { uint32_t _v = (val) ^ hc; hc *= MULT_A; _v *= hc; _v ^= _v >> 16; res = _v; } while (0)
#define MIX(x, y, res) do { uint32_t _r = MIX_L * (x) - MIX_R * (y); _r ^= _r >> 16; res = _r; } while (0)
  for (int i = 0; i < 4; i++) HASHMIX(i < nw ? words[i] : 0u, pool[i]);
  for (int s = 0; s < 4; s++)
    for (int d = 0; d < 4; d++)
      if (s != d) { uint32_t h; HASHMIX(pool[s], h); MIX(pool[d], h, pool[d]); }
  for (int s = 4; s < nw; s++)
    for (int d = 0; d < 4; d++) { uint32_t h; HASHMIX(words[s], h); MIX(pool[d], h, pool[d]); }
#undef HASHMIX
#undef MIX
  uint32_t st32[8];
  uint32_t hb = INIT_B;
  for (int i = 0; i < 8; i++) {
    uint32_t v = pool[i % 4];
    v ^= hb; hb *= MULT_B; v *= hb; v ^= v >> 16;
    st32[i] = v;
  }
  uint64_t u[4];
  for (int i = 0; i < 4; i++) u[i] = (uint64_t)st32[2 * i] | ((uint64_t)st32[2 * i + 1] << 32);
  u128 seed = ((u128)u[0] << 64) | u[1];
  u128 inc = ((((u128)u[2] << 64) | u[3]) << 1) | 1;
  u128 s = 0;
  s = s * PCG_MULT + inc;
  s += seed;
  s = s * PCG_MULT + inc;
  out->state_hi = (uint64_t)(s >> 64); out->state_lo = (uint64_t)s;
  out->inc_hi = (uint64_t)(inc >> 64); out->inc_lo = (uint64_t)inc;
  out->has_uint32 = 0; out->uinteger = 0;
  return DBS_OK;
}

static uint64_t pcg_next64(dbs_pcg64* g) {
  u128 s = ((u128)g->state_hi << 64) | g->state_lo;
  u128 inc = ((u128)g->inc_hi << 64) | g->inc_lo;
  s = s * PCG_MULT + inc;
  g->state_hi = (uint64_t)(s >> 64); g->state_lo = (uint64_t)s;
  uint64_t x = g->state_hi ^ g->state_lo;
  unsigned r = (unsigned)(g->state_hi >> 58);
  return (x >> r) | (x << ((64 - r) & 63));
}
static uint32_t pcg_next32(dbs_pcg64* g) {
  if (g->has_uint32) { g->has_uint32 = 0; return g->uinteger; }
  uint64_t v = pcg_next64(g);
  g->has_uint32 = 1;
  g->uinteger = (uint32_t)(v >> 32);
  return (uint32_t)v;
}
static uint64_t random_interval(dbs_pcg64* g, uint64_t max) {
  if (max == 0) return 0;
  uint64_t mask = max;
  mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4; mask |= mask >> 8; mask |= mask >> 16;
  if (max <= 0xffffffffULL) {
    uint64_t v;
    while ((v = (pcg_next32(g) & mask)) > max) {}
    return v;
  }
  mask |= mask >> 32;
  uint64_t v;
  while ((v = (pcg_next64(g) & mask)) > max) {}
  return v;
}

/* start_i + rng.permutation(end_i - start_i) for each span in order */
int oracle_permute_spans(dbs_pcg64* g, const int64_t* spans, int64_t n, int64_t* out) {
  int64_t off = 0;
  for (int64_t s = 0; s < n; s++) {
    int64_t start = spans[2 * s], L = spans[2 * s + 1] - start;
    if (L < 0) return DBS_ERR_ARGUMENT;
    int64_t* a = out + off;
    for (int64_t i = 0; i < L; i++) a[i] = i;
    for (int64_t i = L - 1; i > 0; i--) {
      int64_t j = (int64_t)random_interval(g, (uint64_t)i);
      int64_t t = a[i]; a[i] = a[j]; a[j] = t;
    }
    for (int64_t i = 0; i < L; i++) a[i] += start;
    off += L;
  }
  return DBS_OK;
}

/* ---------------------------------------------------------------------- */
/* sgdlab.aggregate_gradients / sgd_step  (sgdlab.py:208-238), fp64        */
/* ---------------------------------------------------------------------- */
int oracle_aggregate(const double* const* g, const int64_t* b, int64_t n, int mode, int64_t P,
                     double* out) {
  if (n <= 0) return DBS_ERR_CONFIGURATION;
  for (int64_t i = 0; i < n; i++) if (b[i] <= 0) return DBS_ERR_CONFIGURATION;
  double* w = (double*)malloc(sizeof(double) * (size_t)n);
  if (mode == DBS_AGG_BATCH_WEIGHTED) {
    double tot = 0.0;
    for (int64_t i = 0; i < n; i++) tot += (double)b[i];
    for (int64_t i = 0; i < n; i++) w[i] = (double)b[i] / tot;
    for (int64_t p = 0; p < P; p++) {
      double acc = 0.0;
      for (int64_t i = 0; i < n; i++) acc += w[i] * g[i][p];
      out[p] = acc;
    }
  } else if (mode == DBS_AGG_UNIFORM) {
    for (int64_t p = 0; p < P; p++) {
      double acc = 0.0;
      for (int64_t i = 0; i < n; i++) acc += g[i][p];
      out[p] = acc / (double)n;
    }
  } else {
    free(w);
    return DBS_ERR_CONFIGURATION;
  }
  free(w);
  return DBS_OK;
}

int oracle_sgd_step(const double* x, const double* g, const double* v, int64_t P, double step,
                    double mom, double* x_out, double* v_out) {
  for (int64_t p = 0; p < P; p++) {
    double nv = mom * v[p] + g[p];
    x_out[p] = x[p] - step * nv;
    v_out[p] = nv;
  }
  return DBS_OK;
}

/* row gather dst[r] = src[idx[r]] */
int oracle_gather_rows(const void* src, const int64_t* idx, int64_t rows, int64_t row_bytes,
                       void* dst) {
  for (int64_t r = 0; r < rows; r++)
    memcpy((char*)dst + r * row_bytes, (const char*)src + idx[r] * row_bytes, (size_t)row_bytes);
  return DBS_OK;
}

// controller.cu -- the epoch-end DBS controller on the device (north_star (3)).
//
// Restates /root/reference/pkg/src/dbsim/allocation.py:78-244 and the DBS
// branch of cluster.run_training (cluster.py:253-271) as ONE single-CTA kernel
// that is bit-identical to the reference:
//   * fp64 IEEE round-to-nearest with explicit __d*_rn intrinsics (and this
//     translation unit is compiled with -fmad=false), so no FMA contraction;
//   * math.fsum (allocation.py:101,111) as a correctly-rounded Shewchuk sum --
//     the same partials algorithm CPython uses, so even the special-value
//     behaviour (inf/nan/overflow) matches;
//   * Python floor / int arithmetic in int64 with int128 intermediates, exact
//     rational range boundaries (Fraction(cum_i, sum b), allocation.py:140-155)
//     as int64 numerators over a common denominator.
// Parallel work (validation, floors, candidate ranking, span floors) is spread
// over the CTA; the inherently sequential scans run on thread 0.  n is the
// worker count (<= a few thousand), so the kernel is latency-bound (~µs).
#include <math.h>

#include "common.cuh"

namespace dbs {
namespace {

enum CtrlOp : int {
  OP_EVAL = 0,
  OP_FRACTIONS = 1,
  OP_SCALE = 2,
  OP_ROUND = 3,
  OP_RAISE = 4,
  OP_PARTITION = 5,
  OP_SPANS = 6,
  OP_PLAN = 7,
  OP_REPLAN = 8,
};

struct CtrlArgs {
  int op;
  int adaptive;
  int64_t n, B, D, epoch;
  double smoothing;
  const double* in_a;
  const double* in_b;
  const int64_t* in_i;
  const dbs_bound* lo;
  const dbs_bound* hi;
  double* out_d;
  int64_t* out_b;
  int64_t* out_cum;
  int64_t* out_spans;
  int64_t* out_iters;
  double* tmp_d;   // n
  double* tmp_d2;  // n
  int64_t* tmp_i;  // n
  double* tmp_d3;  // n (replan: times)
  double* smoothed;  // n (replan)
  int32_t* flags;    // [0] EMA valid (replan), [1] status
  int64_t* bad_index;
};

constexpr int kThreads = 256;
constexpr int kMaxPartials = 256;

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// math.fsum (CPython mathmodule.c, Shewchuk partials + half-even fix-up).
__device__ int dev_fsum(const double* v, int64_t n, double* out) {
  double p[kMaxPartials];
  int m = 0;
  double special_sum = 0.0, inf_sum = 0.0;
  for (int64_t k = 0; k < n; k++) {
    double x = v[k];
    const double xsave = x;
    int i = 0;
    for (int j = 0; j < m; j++) {
      double y = p[j];
      if (fabs(x) < fabs(y)) {
        double t = x;
        x = y;
        y = t;
      }
      double hi = dadd(x, y);
      double yr = dsub(hi, x);
      double lo = dsub(y, yr);
      if (lo != 0.0) p[i++] = lo;
      x = hi;
    }
    m = i;
    if (x != 0.0) {
      if (!isfinite(x)) {
        if (isfinite(xsave)) return DBS_ERR_FSUM_OVERFLOW;
        if (isinf(xsave)) inf_sum = dadd(inf_sum, xsave);
        special_sum = dadd(special_sum, xsave);
        m = 0;
      } else {
        if (m >= kMaxPartials) return DBS_ERR_ARGUMENT;
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
      hi = dadd(x, y);
      double yr = dsub(hi, x);
      lo = dsub(y, yr);
      if (lo != 0.0) break;
    }
    if (m > 0 && ((lo < 0.0 && p[m - 1] < 0.0) || (lo > 0.0 && p[m - 1] > 0.0))) {
      double y = dmul(lo, 2.0);
      double x = dadd(hi, y);
      double yr = dsub(x, hi);
      if (y == yr) hi = x;
    }
  }
  *out = hi;
  return DBS_OK;
}

struct Shared {
  int status;
  unsigned long long bad;  // first failing index (min)
  double total;
  long long k_lo;          // clamp of max(k, 0) to [0, n]
};

__device__ __forceinline__ void fail_at(Shared& sh, int64_t i) {
  atomicMin(&sh.bad, (unsigned long long)i);
}

// allocation.evaluate_performance (allocation.py:78-88) for each pair; first
// failing index raises (the list comprehension of plan_next_epoch :230-233).
__device__ void stage_eval(Shared& sh, const double* share, const double* t, int64_t n, double* out) {
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    double s = share[i], tt = t[i];
    bool ok = (0.0 < s && s <= 1.0) && isfinite(s) && !(tt <= 0.0 || !isfinite(tt));
    if (ok)
      out[i] = ddiv(s, tt);
    else
      fail_at(sh, i);
  }
  __syncthreads();
  if (threadIdx.x == 0 && sh.bad != ~0ull) sh.status = DBS_ERR_INVALID_MEASUREMENT;
  __syncthreads();
}

// allocation.compute_batch_fractions (allocation.py:91-102)
__device__ void stage_fractions(Shared& sh, const double* perf, int64_t n, double* out) {
  if (n <= 0) {
    if (threadIdx.x == 0) sh.status = DBS_ERR_INVALID_PERFORMANCE;
    __syncthreads();
    return;
  }
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    double v = perf[i];
    if (v <= 0.0 || !isfinite(v)) fail_at(sh, i);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (sh.bad != ~0ull) {
      sh.status = DBS_ERR_INVALID_PERFORMANCE;
    } else {
      double tot;
      int st = dev_fsum(perf, n, &tot);
      if (st) sh.status = st;
      sh.total = tot;
    }
  }
  __syncthreads();
  if (sh.status) return;
  const double tot = sh.total;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) out[i] = ddiv(perf[i], tot);
  __syncthreads();
}

// allocation.scale_to_real_batches (allocation.py:105-113)
__device__ void stage_scale(Shared& sh, const double* f, int64_t n, int64_t B, double* out) {
  if (threadIdx.x == 0) {
    if (B < n) {
      sh.status = DBS_ERR_BUDGET_TOO_SMALL;
    } else {
      double s;
      int st = dev_fsum(f, n, &s);
      if (st)
        sh.status = st;
      else if (fabs(dsub(s, 1.0)) > 1e-6)
        sh.status = DBS_ERR_INVALID_PERFORMANCE;
    }
  }
  __syncthreads();
  if (sh.status) return;
  const double b = (double)B;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) out[i] = dmul(f[i], b);
  __syncthreads();
}

// allocation.round_twice (allocation.py:116-137).  decimals d_i = b_i - floor(b_i)
// are exact; the candidates {d_i >= 0.5} ordered by (-d_i, i) take +1 while
// k = B - sum(floors) allows.  The rank of each candidate in that order is
// counted in parallel (no sort needed).
__device__ void stage_round(Shared& sh, const double* real, int64_t n, int64_t B, int64_t* out,
                            double* dec) {
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    double r = real[i];
    if (r < 0.0 || !isfinite(r)) {
      fail_at(sh, i);
      continue;
    }
    double f = floor(r);
    if (f >= 9.2e18) {
      atomicCAS(&sh.status, 0, (int)DBS_ERR_INT_OVERFLOW);
      continue;
    }
    out[i] = (int64_t)f;
    dec[i] = dsub(r, f);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (sh.bad != ~0ull) sh.status = DBS_ERR_INVALID_BATCH;
    if (!sh.status) {
      __int128 sum = 0;
      for (int64_t i = 0; i < n; i++) sum += out[i];
      __int128 k = (__int128)B - sum;
      if (k < 0) k = 0;
      if (k > n) k = n;
      sh.k_lo = (long long)k;
    }
  }
  __syncthreads();
  if (sh.status) return;
  const int64_t k = sh.k_lo;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    double d = dec[i];
    if (!(d >= 0.5) || k == 0) continue;
    int64_t rank = 0;
    for (int64_t j = 0; j < n && rank < k; j++) {
      double e = dec[j];
      if (e >= 0.5 && (e > d || (e == d && j < i))) rank++;
    }
    if (rank < k) out[i] += 1;
  }
  __syncthreads();
}

// allocation._raise_zero_batches (allocation.py:191-204): first zero gets +1,
// the first maximum donates, stop when the donor has <= 1.
__device__ void stage_raise(Shared& sh, int64_t* b, int64_t n) {
  if (threadIdx.x == 0) {
    for (;;) {
      int64_t zero = -1;
      for (int64_t i = 0; i < n; i++)
        if (b[i] == 0) {
          zero = i;
          break;
        }
      if (zero < 0) break;
      int64_t donor = 0;
      for (int64_t i = 1; i < n; i++)
        if (b[i] > b[donor]) donor = i;
      if (b[donor] <= 1) break;
      b[zero] += 1;
      b[donor] -= 1;
    }
  }
  __syncthreads();
}

// allocation.partition_ranges (allocation.py:140-155) as cum[0..n]; range i is
// [cum[i]/cum[n], cum[i+1]/cum[n]).
__device__ void stage_partition(Shared& sh, const int64_t* b, int64_t n, int64_t* cum) {
  if (threadIdx.x == 0) {
    if (n <= 0) {
      sh.status = DBS_ERR_EMPTY_PARTITION;
    } else {
      bool neg = false;
      for (int64_t i = 0; i < n; i++) neg |= b[i] < 0;
      if (neg) {
        sh.status = DBS_ERR_INVALID_BATCH;
      } else {
        cum[0] = 0;
        for (int64_t i = 0; i < n; i++) {
          if (cum[i] > INT64_MAX - b[i]) {
            sh.status = DBS_ERR_INT_OVERFLOW;
            break;
          }
          cum[i + 1] = cum[i] + b[i];
        }
        if (!sh.status && cum[n] == 0) sh.status = DBS_ERR_EMPTY_PARTITION;
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ int64_t floordiv128(__int128 a, __int128 b) {
  __int128 q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) q -= 1;
  return (int64_t)q;
}

// Python promotion: Fraction/int op float -> float(Fraction) op float, where
// float(Fraction) = num / den correctly rounded (exact for |num|,den < 2^53).
__device__ __forceinline__ double bound_double(const dbs_bound& x) {
  return x.kind == 1 ? x.value : ddiv((double)x.num, (double)x.den);
}

// allocation.spans_from_ranges (allocation.py:158-188).  Either general bounds
// (lo/hi arrays) or the exact cum/total form produced by partition_ranges.
__device__ void stage_spans(Shared& sh, const dbs_bound* lo, const dbs_bound* hi,
                            const int64_t* cum, int64_t n, int64_t D, int64_t* spans,
                            int64_t* starts, double* posw) {
  if (threadIdx.x == 0) {
    if (D < n) sh.status = DBS_ERR_DATASET_TOO_SMALL;
    else if (n <= 0) sh.status = DBS_ERR_ARGUMENT;
  }
  __syncthreads();
  if (sh.status) return;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    bool positive;
    int64_t st;
    if (cum != nullptr) {
      positive = cum[i + 1] > cum[i];
      st = floordiv128((__int128)cum[i] * D, cum[n]);
    } else {
      const dbs_bound& a = lo[i];
      const dbs_bound& b = hi[i];
      if (a.kind == 0 && b.kind == 0)
        positive = (__int128)b.num * a.den > (__int128)a.num * b.den;
      else
        positive = dsub(bound_double(b), bound_double(a)) > 0.0;
      if (a.kind == 0)
        st = floordiv128((__int128)a.num * D, a.den);
      else
        st = (int64_t)floor(dmul(a.value, (double)D));
    }
    starts[i] = st;
    posw[i] = positive ? 1.0 : 0.0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    starts[0] = 0;
    for (int64_t i = 1; i < n; i++) {
      int64_t least = starts[i - 1] + (posw[i - 1] != 0.0 ? 1 : 0);
      if (starts[i] < least) starts[i] = least;
    }
    int64_t cap = D;
    for (int64_t i = n - 1; i > 0; i--) {
      if (posw[i] != 0.0) cap -= 1;
      if (starts[i] > cap) starts[i] = cap;
    }
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    spans[2 * i] = starts[i];
    spans[2 * i + 1] = (i + 1 < n) ? starts[i + 1] : D;
  }
  __syncthreads();
}

// cluster.iterations_for_plan (cluster.py:159-170)
__device__ void stage_iters(const int64_t* b, const int64_t* spans, int64_t n, int64_t* iters) {
  if (threadIdx.x == 0 && iters != nullptr) {
    int64_t best = -1;
    for (int64_t i = 0; i < n; i++) {
      if (b[i] <= 0) continue;
      int64_t c = (spans[2 * i + 1] - spans[2 * i]) / b[i];
      if (best < 0 || c < best) best = c;
    }
    *iters = best < 0 ? 0 : best;
  }
}

// allocation.plan_next_epoch (allocation.py:207-244) given real batches or
// the epoch-0 even split.
__device__ void stage_plan(Shared& sh, const CtrlArgs& a, const double* shares, const double* times) {
  const int64_t n = a.n;
  if (threadIdx.x == 0) {
    if (n <= 0) sh.status = DBS_ERR_INVALID_PERFORMANCE;
    else if (a.B < n) sh.status = DBS_ERR_BUDGET_TOO_SMALL;
  }
  __syncthreads();
  if (sh.status) return;
  double* real = a.tmp_d;
  if (a.epoch == 0) {
    const double e = ddiv((double)a.B, (double)n);
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) real[i] = e;
    __syncthreads();
  } else {
    stage_eval(sh, shares, times, n, a.tmp_d2);
    if (sh.status) return;
    stage_fractions(sh, a.tmp_d2, n, real);
    if (sh.status) return;
    stage_scale(sh, real, n, a.B, a.tmp_d2);
    if (sh.status) return;
    real = a.tmp_d2;
  }
  double* dec = (real == a.tmp_d) ? a.tmp_d2 : a.tmp_d;
  stage_round(sh, real, n, a.B, a.out_b, dec);
  if (sh.status) return;
  stage_raise(sh, a.out_b, n);
  stage_partition(sh, a.out_b, n, a.out_cum);
  if (sh.status) return;
  stage_spans(sh, nullptr, nullptr, a.out_cum, n, a.D, a.out_spans, a.tmp_i, a.tmp_d);
  if (sh.status) return;
  stage_iters(a.out_b, a.out_spans, n, a.out_iters);
}

__global__ void __launch_bounds__(kThreads) controller_kernel(CtrlArgs a) {
  __shared__ Shared sh;
  if (threadIdx.x == 0) {
    sh.status = 0;
    sh.bad = ~0ull;
  }
  __syncthreads();
  const int64_t n = a.n;
  switch (a.op) {
    case OP_EVAL:
      stage_eval(sh, a.in_a, a.in_b, n, a.out_d);
      break;
    case OP_FRACTIONS:
      stage_fractions(sh, a.in_a, n, a.out_d);
      break;
    case OP_SCALE:
      stage_scale(sh, a.in_a, n, a.B, a.out_d);
      break;
    case OP_ROUND:
      stage_round(sh, a.in_a, n, a.B, a.out_b, a.tmp_d);
      break;
    case OP_RAISE:
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a.out_b[i] = a.in_i[i];
      __syncthreads();
      stage_raise(sh, a.out_b, n);
      break;
    case OP_PARTITION:
      stage_partition(sh, a.in_i, n, a.out_cum);
      break;
    case OP_SPANS:
      stage_spans(sh, a.lo, a.hi, nullptr, n, a.D, a.out_spans, a.tmp_i, a.tmp_d);
      break;
    case OP_PLAN:
      stage_plan(sh, a, a.in_a, a.in_b);
      break;
    case OP_REPLAN: {
      // cluster.run_training (cluster.py:253-271)
      if (!a.adaptive || a.epoch == 0) {
        // even_plan (cluster.py:223-231): plan_next_epoch(..., epoch=0)
        CtrlArgs b = a;
        b.epoch = 0;
        stage_plan(sh, b, nullptr, nullptr);
        break;
      }
      const int64_t* prev = a.in_i;
      const double Dprev = (double)prev[2 * n - 1];
      double* shares = a.out_d;  // n doubles of output scratch
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
        shares[i] = ddiv((double)(prev[2 * i + 1] - prev[2 * i]), Dprev);  // allocation.py:72-75
      __syncthreads();
      double* perfs = a.tmp_d2;
      stage_eval(sh, shares, a.in_a, n, perfs);  // :256-262
      if (sh.status) break;
      const bool have = a.flags[0] != 0;
      const double al = a.smoothing;
      const double one_m = dsub(1.0, al);
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        double p = perfs[i];
        if (al > 0.0 && have) p = dadd(dmul(al, a.smoothed[i]), dmul(one_m, p));  // :263-266
        a.smoothed[i] = p;
        a.tmp_i[i] = 0;
        perfs[i] = p;
      }
      __syncthreads();
      if (threadIdx.x == 0) a.flags[0] = 1;
      // times = s / p (:268), then plan_next_epoch re-derives p = s / t (:269)
      double* times = a.tmp_d3;
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) times[i] = ddiv(shares[i], perfs[i]);
      __syncthreads();
      stage_plan(sh, a, shares, times);
      break;
    }
    default:
      if (threadIdx.x == 0) sh.status = DBS_ERR_ARGUMENT;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    a.flags[1] = sh.status;
    if (a.bad_index) *a.bad_index = (sh.bad == ~0ull) ? -1 : (int64_t)sh.bad;
  }
}

// ---------------------------------------------------------------------------
// Host side: pack host inputs into one pinned arena, one H2D copy, one launch,
// one D2H copy, one stream sync.
// ---------------------------------------------------------------------------
thread_local Scratch g_ctrl_scratch;

struct Arena {
  size_t off = 0;
  template <typename T>
  size_t take(size_t count) {
    size_t a = (off + 15) & ~size_t(15);
    off = a + sizeof(T) * (count ? count : 1);
    return a;
  }
};

struct HostCall {
  char* hbuf = nullptr;
  char* dbuf = nullptr;
  size_t total = 0;
};

template <typename T>
T* dptr(const HostCall& hc, size_t off) { return reinterpret_cast<T*>(hc.dbuf + off); }
template <typename T>
T* hptr(const HostCall& hc, size_t off) { return reinterpret_cast<T*>(hc.hbuf + off); }

int prepare(HostCall& hc, size_t total) {
  void* d;
  void* h;
  int st = scratch_get(g_ctrl_scratch, total, &d);
  if (st) return st;
  st = pinned_get(total, &h);
  if (st) return st;
  hc.dbuf = (char*)d;
  hc.hbuf = (char*)h;
  hc.total = total;
  return DBS_OK;
}

}  // namespace
}  // namespace dbs

using namespace dbs;

// Shared layout builder for the host-buffer entry points.
namespace {
struct Layout {
  size_t in_a, in_b, in_i, lo, hi;            // inputs
  size_t out_d, out_b, out_cum, out_spans, out_iters, tmp_d, tmp_d2, tmp_i, flags, bad, smoothed;
  size_t in_bytes, total;
};
Layout make_layout(int64_t n, bool bounds) {
  dbs::Arena ar;
  Layout L{};
  size_t N = (size_t)(n > 0 ? n : 1);
  L.in_a = ar.take<double>(N);
  L.in_b = ar.take<double>(N);
  L.in_i = ar.take<int64_t>(2 * N);
  L.lo = ar.take<dbs_bound>(bounds ? N : 1);
  L.hi = ar.take<dbs_bound>(bounds ? N : 1);
  L.flags = ar.take<int32_t>(4);
  L.in_bytes = ar.off;
  L.out_d = ar.take<double>(N);
  L.out_b = ar.take<int64_t>(N);
  L.out_cum = ar.take<int64_t>(N + 1);
  L.out_spans = ar.take<int64_t>(2 * N);
  L.out_iters = ar.take<int64_t>(1);
  L.bad = ar.take<int64_t>(1);
  L.tmp_d = ar.take<double>(N);
  L.tmp_d2 = ar.take<double>(N);
  L.tmp_i = ar.take<int64_t>(N);
  L.smoothed = ar.take<double>(3 * N);
  L.total = ar.off;
  return L;
}

int host_controller(int op, int64_t n, int64_t B, int64_t D, int64_t epoch, const double* a_in,
                    const double* b_in, const int64_t* i_in, int64_t i_count, const dbs_bound* lo,
                    const dbs_bound* hi, double* out_d, int64_t* out_b, int64_t* out_cum,
                    int64_t* out_spans, int64_t* bad_index) {
  if (n < 0) {
    set_error("negative length");
    return DBS_ERR_ARGUMENT;
  }
  Layout L = make_layout(n, lo != nullptr);
  HostCall hc;
  int st = prepare(hc, L.total);
  if (st) return st;
  // The flags word lives in the input region; it must travel back too.
  if (a_in && n) memcpy(hptr<double>(hc, L.in_a), a_in, sizeof(double) * n);
  if (b_in && n) memcpy(hptr<double>(hc, L.in_b), b_in, sizeof(double) * n);
  if (i_in && i_count) memcpy(hptr<int64_t>(hc, L.in_i), i_in, sizeof(int64_t) * i_count);
  if (lo && n) memcpy(hptr<dbs_bound>(hc, L.lo), lo, sizeof(dbs_bound) * n);
  if (hi && n) memcpy(hptr<dbs_bound>(hc, L.hi), hi, sizeof(dbs_bound) * n);
  memset(hptr<int32_t>(hc, L.flags), 0, 16);
  CtrlArgs a{};
  a.op = op;
  a.n = n;
  a.B = B;
  a.D = D;
  a.epoch = epoch;
  a.in_a = dptr<double>(hc, L.in_a);
  a.in_b = dptr<double>(hc, L.in_b);
  a.in_i = dptr<int64_t>(hc, L.in_i);
  a.lo = lo ? dptr<dbs_bound>(hc, L.lo) : nullptr;
  a.hi = hi ? dptr<dbs_bound>(hc, L.hi) : nullptr;
  a.out_d = dptr<double>(hc, L.out_d);
  a.out_b = dptr<int64_t>(hc, L.out_b);
  a.out_cum = dptr<int64_t>(hc, L.out_cum);
  a.out_spans = dptr<int64_t>(hc, L.out_spans);
  a.out_iters = dptr<int64_t>(hc, L.out_iters);
  a.tmp_d = dptr<double>(hc, L.tmp_d);
  a.tmp_d2 = dptr<double>(hc, L.tmp_d2);
  a.tmp_i = dptr<int64_t>(hc, L.tmp_i);
  a.smoothed = dptr<double>(hc, L.smoothed);
  a.flags = dptr<int32_t>(hc, L.flags);
  a.bad_index = dptr<int64_t>(hc, L.bad);
  cudaStream_t s = cudaStreamPerThread;
  DBS_CUDA_TRY(cudaMemcpyAsync(hc.dbuf, hc.hbuf, L.in_bytes, cudaMemcpyHostToDevice, s));
  controller_kernel<<<1, dbs::kThreads, 0, s>>>(a);
  DBS_LAUNCH_CHECK();
  DBS_CUDA_TRY(cudaMemcpyAsync(hc.hbuf + L.flags, hc.dbuf + L.flags, 16, cudaMemcpyDeviceToHost, s));
  DBS_CUDA_TRY(cudaMemcpyAsync(hc.hbuf + L.out_d, hc.dbuf + L.out_d, L.tmp_d - L.out_d,
                               cudaMemcpyDeviceToHost, s));
  DBS_CUDA_TRY(cudaStreamSynchronize(s));
  int status = hptr<int32_t>(hc, L.flags)[1];
  if (bad_index) *bad_index = hptr<int64_t>(hc, L.bad)[0];
  if (status) {
    set_error("controller status %d", status);
    return status;
  }
  if (out_d && n) memcpy(out_d, hptr<double>(hc, L.out_d), sizeof(double) * n);
  if (out_b && n) memcpy(out_b, hptr<int64_t>(hc, L.out_b), sizeof(int64_t) * n);
  if (out_cum) memcpy(out_cum, hptr<int64_t>(hc, L.out_cum), sizeof(int64_t) * (n + 1));
  if (out_spans && n) memcpy(out_spans, hptr<int64_t>(hc, L.out_spans), sizeof(int64_t) * 2 * n);
  return DBS_OK;
}
}  // namespace

extern "C" int dbs_evaluate_performance(const double* shares, const double* times, int64_t n,
                                        double* perf_out, int64_t* bad_index) {
  return host_controller(OP_EVAL, n, 0, 0, 0, shares, times, nullptr, 0, nullptr, nullptr, perf_out,
                         nullptr, nullptr, nullptr, bad_index);
}

extern "C" int dbs_compute_batch_fractions(const double* perfs, int64_t n, double* out,
                                           int64_t* bad_index) {
  return host_controller(OP_FRACTIONS, n, 0, 0, 0, perfs, nullptr, nullptr, 0, nullptr, nullptr, out,
                         nullptr, nullptr, nullptr, bad_index);
}

extern "C" int dbs_scale_to_real_batches(const double* fr, int64_t n, int64_t B, double* out) {
  return host_controller(OP_SCALE, n, B, 0, 0, fr, nullptr, nullptr, 0, nullptr, nullptr, out,
                         nullptr, nullptr, nullptr, nullptr);
}

extern "C" int dbs_round_twice(const double* real, int64_t n, int64_t B, int64_t* out) {
  return host_controller(OP_ROUND, n, B, 0, 0, real, nullptr, nullptr, 0, nullptr, nullptr, nullptr,
                         out, nullptr, nullptr, nullptr);
}

extern "C" int dbs_raise_zero_batches(const int64_t* in, int64_t n, int64_t* out) {
  return host_controller(OP_RAISE, n, 0, 0, 0, nullptr, nullptr, in, n, nullptr, nullptr, nullptr,
                         out, nullptr, nullptr, nullptr);
}

extern "C" int dbs_partition_ranges(const int64_t* b, int64_t n, int64_t* cum_out) {
  return host_controller(OP_PARTITION, n, 0, 0, 0, nullptr, nullptr, b, n, nullptr, nullptr,
                         nullptr, nullptr, cum_out, nullptr, nullptr);
}

extern "C" int dbs_spans_from_ranges(const dbs_bound* lo, const dbs_bound* hi, int64_t n,
                                     int64_t D, int64_t* spans_out) {
  dbs_bound dummy{};
  return host_controller(OP_SPANS, n, 0, D, 0, nullptr, nullptr, nullptr, 0, lo ? lo : &dummy,
                         hi ? hi : &dummy, nullptr, nullptr, nullptr, spans_out, nullptr);
}

extern "C" int dbs_plan_next_epoch(const double* shares, const double* times, int64_t n, int64_t B,
                                   int64_t D, int64_t epoch, int64_t* int_batches, int64_t* cum,
                                   int64_t* spans, int64_t* bad_index) {
  return host_controller(OP_PLAN, n, B, D, epoch, shares, times, nullptr, 0, nullptr, nullptr,
                         nullptr, int_batches, cum, spans, bad_index);
}

// Device-resident re-plan; kernel scratch comes from a per-thread arena.
namespace {
thread_local dbs::Scratch g_replan_scratch;
}

extern "C" int dbs_dev_replan(const int64_t* d_prev_spans, const double* d_times, int64_t n,
                              int64_t B, int64_t D, int64_t epoch, int32_t adaptive,
                              double smoothing, double* d_smoothed, int32_t* d_flags,
                              int64_t* d_int_batches, int64_t* d_cum, int64_t* d_spans,
                              int64_t* d_iters, void* stream) {
  DBS_REQUIRE(n > 0 && d_smoothed && d_flags && d_int_batches && d_cum && d_spans,
              DBS_ERR_ARGUMENT, "dbs_dev_replan: bad arguments");
  DBS_REQUIRE(adaptive == 0 || epoch == 0 || (d_prev_spans && d_times), DBS_ERR_ARGUMENT,
              "dbs_dev_replan: previous plan / times required");
  size_t N = (size_t)n;
  void* scr;
  int st = scratch_get(g_replan_scratch, sizeof(double) * (5 * N + 8), &scr);
  if (st) return st;
  double* sd = (double*)scr;
  CtrlArgs a{};
  a.op = OP_REPLAN;
  a.adaptive = adaptive;
  a.n = n;
  a.B = B;
  a.D = D;
  a.epoch = epoch;
  a.smoothing = smoothing;
  a.in_a = d_times;
  a.in_i = d_prev_spans;
  a.out_d = sd;            // shares (n)
  a.tmp_d = sd + N;        // n
  a.tmp_d2 = sd + 2 * N;   // n
  a.tmp_i = (int64_t*)(sd + 3 * N);
  a.tmp_d3 = sd + 4 * N;   // n
  a.out_b = d_int_batches;
  a.out_cum = d_cum;
  a.out_spans = d_spans;
  a.out_iters = d_iters;
  a.smoothed = d_smoothed;
  a.flags = d_flags;
  a.bad_index = nullptr;
  controller_kernel<<<1, dbs::kThreads, 0, as_stream(stream)>>>(a);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

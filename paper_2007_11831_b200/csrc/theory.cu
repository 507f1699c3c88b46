// theory.cu -- the Monte-Carlo checks of the convergence theory on the device.
//
// Reference: dbsim.checks.check_theorem1_bound (checks.py:42-93) and check_lemma1
// (checks.py:118-142) over sgdlab.estimate_gradient_noise (sgdlab.py:252-272) and
// verify_lemma1_variance (sgdlab.py:282-314).  Their randomness is numpy's
// Generator: `rng.integers(0, n, size)` and `rng.random(size)`.  The draws are
// reproduced exactly here from the same PCG64 state (dbs_pcg64, permute.cu):
//   integers(0, n), n <= 2^32: random_bounded_uint64_fill with use_masked = false --
//     a 32-bit buffer LOCAL to the call (low half of next64 first, then the high
//     half), Lemire's multiply-and-reject on each buffered uint32 (rng = n - 1);
//   random(): (next64 >> 11) * 2^-53.
// One thread draws (the rejection makes the stream sequential; a check needs
// ~10^5 draws, ~1 ms); the Monte-Carlo arithmetic is parallel over seeds / draws.
#include "common.cuh"

namespace dbs {
namespace {

typedef unsigned __int128 u128;

__device__ __forceinline__ uint64_t next64(u128& st, const u128 inc) {
  const u128 M = (((u128)0x2360ED051FC65DA4ULL) << 64) | 0x4385DF649FCCF645ULL;
  st = st * M + inc;
  const uint64_t hi = (uint64_t)(st >> 64), lo = (uint64_t)st;
  const uint64_t x = hi ^ lo;
  const unsigned r = (unsigned)(hi >> 58);
  return (x >> r) | (x << ((64u - r) & 63u));
}

__global__ void integers_kernel(dbs_pcg64* rng, uint64_t n, int64_t cnt, int64_t* out) {
  u128 st = ((u128)rng->state_hi << 64) | rng->state_lo;
  const u128 inc = ((u128)rng->inc_hi << 64) | rng->inc_lo;
  const uint64_t r = n - 1;  // numpy's rng = high - low - 1 (endpoint = False)
  uint64_t buf = 0;
  int bcnt = 0;
  auto b32 = [&]() -> uint32_t {
    if (!bcnt) {
      buf = next64(st, inc);
      bcnt = 1;
    } else {
      buf >>= 32;
      bcnt -= 1;
    }
    return (uint32_t)buf;
  };
  if (r == 0) {
    for (int64_t i = 0; i < cnt; i++) out[i] = 0;
  } else if (r == 0xFFFFFFFFull) {
    for (int64_t i = 0; i < cnt; i++) out[i] = (int64_t)b32();
  } else {
    const uint32_t rexcl = (uint32_t)r + 1u;
    const uint32_t threshold = (uint32_t)((0xFFFFFFFFu - (uint32_t)r) % rexcl);
    for (int64_t i = 0; i < cnt; i++) {
      uint64_t m = (uint64_t)b32() * rexcl;
      uint32_t left = (uint32_t)m;
      if (left < rexcl) {
        while (left < threshold) {
          m = (uint64_t)b32() * rexcl;
          left = (uint32_t)m;
        }
      }
      out[i] = (int64_t)(m >> 32);
    }
  }
  rng->state_hi = (uint64_t)(st >> 64);
  rng->state_lo = (uint64_t)st;
}

__global__ void random_kernel(dbs_pcg64* rng, int64_t cnt, double* out) {
  u128 st = ((u128)rng->state_hi << 64) | rng->state_lo;
  const u128 inc = ((u128)rng->inc_hi << 64) | rng->inc_lo;
  for (int64_t i = 0; i < cnt; i++) out[i] = (double)(next64(st, inc) >> 11) * (1.0 / 9007199254740992.0);
  rng->state_hi = (uint64_t)(st >> 64);
  rng->state_lo = (uint64_t)st;
}

// Theorem-1 setting (checks.py:62-70): single-sample SGD, one trajectory per seed,
// X <- X - (gamma mu) ((X - x*) - eps[idx_j]); dists[j][s] = ||X_s - x*||^2 and
// snapshots of X at the probe iterations.  Thread = seed; no FMA contraction
// (the reference's separate numpy operations).
__global__ void theorem1_kernel(const double* __restrict__ off, const double* __restrict__ opt,
                                const double* __restrict__ x0, int64_t dim, const int64_t* __restrict__ idx,
                                int64_t n_seeds, int64_t n_iter, double coef, const int32_t* __restrict__ probe_at,
                                int n_probe, double* __restrict__ X, double* __restrict__ dists,
                                double* __restrict__ snap) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_seeds) return;
  double* x = X + s * dim;
  for (int64_t d = 0; d < dim; d++) x[d] = x0[d];
  int p = 0;
  for (int64_t j = 1; j <= n_iter; j++) {
    const double* e = off + idx[(j - 1) * n_seeds + s] * dim;
    double acc = 0.0;
    for (int64_t d = 0; d < dim; d++) {
      const double g = __dsub_rn(__dsub_rn(x[d], opt[d]), e[d]);
      const double v = __dsub_rn(x[d], __dmul_rn(coef, g));
      x[d] = v;
      const double q = __dsub_rn(v, opt[d]);
      acc = __dadd_rn(acc, __dmul_rn(q, q));
    }
    dists[j * n_seeds + s] = acc;
    if (p < n_probe && probe_at[p] == j) {
      for (int64_t d = 0; d < dim; d++) snap[((int64_t)p * n_seeds + s) * dim + d] = x[d];
      p++;
    }
  }
}

// per row r of v[rows][n]: mean, sum (v - mean)^2, sum (v - mean)^4 (two passes, fp64)
__global__ void __launch_bounds__(256) moments_kernel(const double* __restrict__ v, int64_t n, int64_t ld,
                                                      double* __restrict__ out) {
  __shared__ double red[256];
  const double* row = v + (int64_t)blockIdx.x * ld;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += row[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  const double mean = red[0] / (double)n;
  __syncthreads();
  double m2 = 0.0, m4 = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double c = row[i] - mean;
    const double c2 = c * c;
    m2 += c2;
    m4 += c2 * c2;
  }
  red[threadIdx.x] = m2;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[blockIdx.x * 3] = mean;
    out[blockIdx.x * 3 + 1] = red[0];
  }
  __syncthreads();
  red[threadIdx.x] = m4;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x * 3 + 2] = red[0];
}

// ||mean_k grad f_{idx[t][k]}(x)||^2 for every draw t (estimate_gradient_noise,
// sgdlab.py:266-271): kind 0 = ConvexProblem mu (x - x* - eps_i), 1 = LogisticProblem
// -y_i / (1 + exp(y_i f_i.x)) f_i + mu x
__global__ void minibatch_sqnorm_kernel(int kind, const double* __restrict__ data, const double* __restrict__ labels,
                                        const double* __restrict__ opt, int64_t dim, double mu,
                                        const double* __restrict__ x, const int64_t* __restrict__ idx,
                                        int64_t n_draws, int64_t b, double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_draws) return;
  double acc = 0.0;
  for (int64_t d = 0; d < dim; d++) {
    double g = 0.0;
    for (int64_t k = 0; k < b; k++) {
      const int64_t i = idx[t * b + k];
      if (kind == 0) {
        g += mu * (x[d] - opt[d] - data[i * dim + d]);
      } else {
        double m = 0.0;
        for (int64_t e = 0; e < dim; e++) m += data[i * dim + e] * x[e];
        const double yi = labels[i];
        g += (-yi / (1.0 + exp(yi * m))) * data[i * dim + d] + mu * x[d];
      }
    }
    g /= (double)b;
    acc += g * g;
  }
  out[t] = acc;
}

// per-sample objective values f_i(x) (sample_values, sgdlab.py:88-90 / 150-154)
__global__ void sample_values_kernel(int kind, const double* __restrict__ data, const double* __restrict__ labels,
                                     const double* __restrict__ opt, int64_t dim, double mu,
                                     const double* __restrict__ x, int64_t n, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (kind == 0) {
    double s = 0.0;
    for (int64_t d = 0; d < dim; d++) {
      const double q = x[d] - opt[d] - data[i * dim + d];
      s += q * q;
    }
    out[i] = 0.5 * mu * s;
  } else {
    double m = 0.0, xx = 0.0;
    for (int64_t d = 0; d < dim; d++) {
      m += data[i * dim + d] * x[d];
      xx += x[d] * x[d];
    }
    const double z = -labels[i] * m;  // logaddexp(0, z)
    out[i] = (z > 0 ? z + log1p(exp(-z)) : log1p(exp(z))) + 0.5 * mu * xx;
  }
}

// mean over k < m of v[idx[t][k]] (verify_lemma1_variance's mini-batch means)
__global__ void gather_means_kernel(const double* __restrict__ v, const int64_t* __restrict__ idx, int64_t n_draws,
                                    int64_t m, double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_draws) return;
  double s = 0.0;
  for (int64_t k = 0; k < m; k++) s += v[idx[t * m + k]];
  out[t] = s / (double)m;
}

unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t > 0 ? (n + t - 1) / t : 1); }

}  // namespace
}  // namespace dbs

using namespace dbs;

extern "C" int dbs_dev_pcg64_integers(dbs_pcg64* d_rng, int64_t high, int64_t count, int64_t* d_out, void* stream) {
  DBS_REQUIRE(d_rng && d_out && high >= 1 && (uint64_t)high <= (1ull << 32) && count >= 0, DBS_ERR_ARGUMENT,
              "pcg64_integers: 1 <= high <= 2^32");
  if (count == 0) return DBS_OK;
  integers_kernel<<<1, 1, 0, as_stream(stream)>>>(d_rng, (uint64_t)high, count, d_out);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

extern "C" int dbs_dev_pcg64_random(dbs_pcg64* d_rng, int64_t count, double* d_out, void* stream) {
  DBS_REQUIRE(d_rng && d_out && count >= 0, DBS_ERR_ARGUMENT, "pcg64_random: bad arguments");
  if (count == 0) return DBS_OK;
  random_kernel<<<1, 1, 0, as_stream(stream)>>>(d_rng, count, d_out);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

extern "C" int dbs_dev_theorem1_trajectories(const double* d_offsets, const double* d_opt, const double* d_x0,
                                             int64_t dim, const int64_t* d_idx, int64_t n_seeds, int64_t n_iter,
                                             double coef, const int32_t* d_probe_at, int32_t n_probe, double* d_X,
                                             double* d_dists, double* d_snap, void* stream) {
  DBS_REQUIRE(d_offsets && d_opt && d_x0 && d_idx && d_X && d_dists && dim > 0 && n_seeds > 0 && n_iter >= 0 &&
                  (n_probe == 0 || (d_probe_at && d_snap)),
              DBS_ERR_ARGUMENT, "theorem1_trajectories: bad arguments");
  theorem1_kernel<<<blocks_for(n_seeds, 128), 128, 0, as_stream(stream)>>>(
      d_offsets, d_opt, d_x0, dim, d_idx, n_seeds, n_iter, coef, d_probe_at, n_probe, d_X, d_dists, d_snap);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

extern "C" int dbs_dev_row_moments(const double* d_v, int64_t rows, int64_t n, int64_t ld, double* d_out,
                                   void* stream) {
  DBS_REQUIRE(d_v && d_out && rows >= 0 && n > 0 && ld >= n, DBS_ERR_ARGUMENT, "row_moments: bad arguments");
  if (rows == 0) return DBS_OK;
  moments_kernel<<<(unsigned)rows, 256, 0, as_stream(stream)>>>(d_v, n, ld, d_out);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

extern "C" int dbs_dev_minibatch_sqnorms(int32_t kind, const double* d_data, const double* d_labels,
                                         const double* d_opt, int64_t dim, double mu, const double* d_x,
                                         const int64_t* d_idx, int64_t n_draws, int64_t b, double* d_out,
                                         void* stream) {
  DBS_REQUIRE((kind == 0 || (kind == 1 && d_labels)) && d_data && d_x && d_idx && d_out && dim > 0 && b > 0,
              DBS_ERR_ARGUMENT, "minibatch_sqnorms: bad arguments");
  if (n_draws <= 0) return DBS_OK;
  minibatch_sqnorm_kernel<<<blocks_for(n_draws, 128), 128, 0, as_stream(stream)>>>(kind, d_data, d_labels, d_opt, dim,
                                                                                   mu, d_x, d_idx, n_draws, b, d_out);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

extern "C" int dbs_dev_sample_values(int32_t kind, const double* d_data, const double* d_labels, const double* d_opt,
                                     int64_t dim, double mu, const double* d_x, int64_t n, double* d_out,
                                     void* stream) {
  DBS_REQUIRE((kind == 0 || (kind == 1 && d_labels)) && d_data && d_x && d_out && dim > 0, DBS_ERR_ARGUMENT,
              "sample_values: bad arguments");
  if (n <= 0) return DBS_OK;
  sample_values_kernel<<<blocks_for(n, 256), 256, 0, as_stream(stream)>>>(kind, d_data, d_labels, d_opt, dim, mu, d_x,
                                                                          n, d_out);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

extern "C" int dbs_dev_gather_means(const double* d_v, const int64_t* d_idx, int64_t n_draws, int64_t m,
                                    double* d_out, void* stream) {
  DBS_REQUIRE(d_v && d_idx && d_out && m > 0, DBS_ERR_ARGUMENT, "gather_means: bad arguments");
  if (n_draws <= 0) return DBS_OK;
  gather_means_kernel<<<blocks_for(n_draws, 256), 256, 0, as_stream(stream)>>>(d_v, d_idx, n_draws, m, d_out);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

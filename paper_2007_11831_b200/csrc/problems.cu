// problems.cu -- the reference's own strongly-convex problems on the device.
//
// ConvexProblem.per_sample_gradients (sgdlab.py:81-82) and LogisticProblem
// .per_sample_gradients (sgdlab.py:143-148), each followed by the batch mean of
// minibatch_gradient (sgdlab.py:200-205), plus ||x - x*||^2 (sgdlab.py:387-388).
//
// The quadratic gradient keeps numpy's evaluation order exactly:
//   mu * ((x - opt) - offsets[idx_k]) summed over k in order, / b,
// with no FMA contraction, so it is bit-identical to the reference.  The
// logistic margin feats_k . x is a warp-shuffle dot product (BLAS order in the
// reference), so that path matches to fp64 rounding.
//
// dbs_dev_sgd_epoch fuses an entire epoch of run_parallel_sgd's hot loop
// (sgdlab.py:380-391: gradients of every worker -> aggregate -> heavy-ball step
// -> squared distance) into ONE single-CTA launch: these problems are tiny
// (d = 8..1000), so a per-iteration launch would be pure overhead.
#include "common.cuh"

namespace dbs {
namespace {

constexpr int kMaxW = 64;

struct WorkerLayout {
  const int64_t* perm;        // concatenated permuted spans (epoch)
  int64_t off[kMaxW + 1];     // start of worker w's span in perm
  int64_t b[kMaxW];           // batch size
  double w[kMaxW];            // aggregation weight
  int n;
  int mode;
};

// mean_k mu * ((x - opt) - off[idx_k])  for worker-local index list idx[0..b)
__device__ __forceinline__ double quad_grad(const double* x, const double* opt, const double* offs,
                                            int64_t dim, int64_t j, const int64_t* idx, int64_t b,
                                            double mu) {
  const double xo = __dsub_rn(x[j], opt[j]);
  double acc = __dmul_rn(mu, __dsub_rn(xo, offs[idx[0] * dim + j]));
  for (int64_t k = 1; k < b; k++) acc = __dadd_rn(acc, __dmul_rn(mu, __dsub_rn(xo, offs[idx[k] * dim + j])));
  return __ddiv_rn(acc, (double)b);
}

// mean_k (coeff_k * f_kj + mu * x_j)
__device__ __forceinline__ double logit_grad(const double* x, const double* feats, int64_t dim, int64_t j,
                                             const int64_t* idx, const double* coeff, int64_t b, double mu) {
  const double mx = __dmul_rn(mu, x[j]);
  double acc = __dadd_rn(__dmul_rn(coeff[0], feats[idx[0] * dim + j]), mx);
  for (int64_t k = 1; k < b; k++)
    acc = __dadd_rn(acc, __dadd_rn(__dmul_rn(coeff[k], feats[idx[k] * dim + j]), mx));
  return __ddiv_rn(acc, (double)b);
}

// coeff = -y / (1 + exp(y * (feats . x)))  -- one warp per sample
__device__ __forceinline__ double logit_coeff(const double* x, const double* feats, const double* labels,
                                              int64_t dim, int64_t sample, int lane) {
  const double* f = feats + sample * dim;
  double acc = 0.0;
  for (int64_t j = lane; j < dim; j += 32) acc = __fma_rn(f[j], x[j], acc);
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  const double y = labels[sample];
  const double m = __dmul_rn(y, acc);
  return __ddiv_rn(-y, __dadd_rn(1.0, exp(m)));
}

// ---- drop-in per-worker gradient kernels (grid: workers x dims) ----
__global__ void quad_grads_kernel(const double* x, const double* opt, const double* offs, int64_t dim,
                                  const int64_t* idx, const int64_t* off, double mu, double* out) {
  const int w = blockIdx.y;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < dim; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = off[w + 1] - off[w];
    out[w * dim + j] = quad_grad(x, opt, offs, dim, j, idx + off[w], b, mu);
  }
}

__global__ void logit_coeff_kernel(const double* x, const double* feats, const double* labels, int64_t dim,
                                   const int64_t* idx, int64_t total, double* coeff) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k = warp; k < total; k += nw) {
    const double c = logit_coeff(x, feats, labels, dim, idx[k], lane);
    if (lane == 0) coeff[k] = c;
  }
}

__global__ void logit_grads_kernel(const double* x, const double* feats, int64_t dim, const int64_t* idx,
                                   const int64_t* off, const double* coeff, double mu, double* out) {
  const int w = blockIdx.y;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < dim; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = off[w + 1] - off[w];
    out[w * dim + j] = logit_grad(x, feats, dim, j, idx + off[w], coeff + off[w], b, mu);
  }
}

__global__ void sq_dist_kernel(const double* x, const double* opt, int64_t dim, double* out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int64_t j = threadIdx.x; j < dim; j += blockDim.x) {
    const double d = __dsub_rn(x[j], opt[j]);
    acc = __fma_rn(d, d, acc);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) *out = acc;
  }
}

// ---- fused epoch: one CTA runs all `iters` iterations of the epoch ----
constexpr int kEpochThreads = 512;

__global__ void __launch_bounds__(kEpochThreads)
    sgd_epoch_kernel(int kind, const double* data, const double* labels, const double* opt, int64_t dim,
                     double mu, WorkerLayout L, int64_t iters, double step, double mom, double* x, double* v,
                     double* grads, double* coeff, double* sq_out) {
  __shared__ double red[32];
  const int nthr = blockDim.x;
  for (int64_t t = 0; t < iters; t++) {
    if (kind == 1) {
      // per-sample coefficients of every worker's batch t
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = nthr >> 5;
      int64_t base = 0;
      for (int w = 0; w < L.n; w++) {
        const int64_t* idx = L.perm + L.off[w] + t * L.b[w];
        for (int64_t k = warp; k < L.b[w]; k += nwarps) {
          const double c = logit_coeff(x, data, labels, dim, idx[k], lane);
          if (lane == 0) coeff[base + k] = c;
        }
        base += L.b[w];
      }
      __syncthreads();
    }
    // gradients of every worker
    {
      int64_t cbase = 0;
      for (int w = 0; w < L.n; w++) {
        const int64_t* idx = L.perm + L.off[w] + t * L.b[w];
        for (int64_t j = threadIdx.x; j < dim; j += nthr)
          grads[w * dim + j] = (kind == 0) ? quad_grad(x, opt, data, dim, j, idx, L.b[w], mu)
                                           : logit_grad(x, data, dim, j, idx, coeff + cbase, L.b[w], mu);
        cbase += L.b[w];
      }
    }
    __syncthreads();
    // aggregate (sgdlab.py:208-227) + heavy-ball step (sgdlab.py:230-238) + distance
    double acc_sq = 0.0;
    for (int64_t j = threadIdx.x; j < dim; j += nthr) {
      double g;
      if (L.mode == DBS_AGG_BATCH_WEIGHTED) {
        g = __dmul_rn(L.w[0], grads[j]);
        for (int w = 1; w < L.n; w++) g = __fma_rn(L.w[w], grads[w * dim + j], g);
      } else {
        g = grads[j];
        for (int w = 1; w < L.n; w++) g = __dadd_rn(g, grads[w * dim + j]);
        g = __ddiv_rn(g, (double)L.n);
      }
      const double nv = __dadd_rn(__dmul_rn(mom, v[j]), g);
      const double nx = __dsub_rn(x[j], __dmul_rn(step, nv));
      v[j] = nv;
      x[j] = nx;
      const double d = __dsub_rn(nx, opt[j]);
      acc_sq = __fma_rn(d, d, acc_sq);
    }
    for (int o = 16; o > 0; o >>= 1) acc_sq += __shfl_xor_sync(0xffffffffu, acc_sq, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc_sq;
    __syncthreads();
    if (threadIdx.x < 32) {
      double a = (threadIdx.x < (nthr >> 5)) ? red[threadIdx.x] : 0.0;
      for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (threadIdx.x == 0) sq_out[t] = a;
    }
    __syncthreads();
  }
}

}  // namespace
}  // namespace dbs

using namespace dbs;

extern "C" int dbs_dev_quadratic_grads(const double* d_x, const double* d_opt, const double* d_offsets,
                                       int64_t dim, const int64_t* d_idx, const int64_t* d_off,
                                       int64_t n_workers, double mu, double* d_out, void* stream) {
  DBS_REQUIRE(dim > 0 && n_workers > 0 && n_workers <= 65535, DBS_ERR_ARGUMENT, "quadratic_grads: bad shape");
  dim3 grid((unsigned)((dim + 255) / 256 < 64 ? (dim + 255) / 256 : 64), (unsigned)n_workers);
  quad_grads_kernel<<<grid, 256, 0, as_stream(stream)>>>(d_x, d_opt, d_offsets, dim, d_idx, d_off, mu, d_out);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

namespace {
thread_local dbs::Scratch g_coeff_scratch;
}

extern "C" int dbs_dev_logistic_grads(const double* d_x, const double* d_features, const double* d_labels,
                                      int64_t dim, const int64_t* d_idx, const int64_t* d_off,
                                      int64_t n_workers, double mu, double* d_out, void* stream) {
  DBS_REQUIRE(dim > 0 && n_workers > 0 && n_workers <= 65535, DBS_ERR_ARGUMENT, "logistic_grads: bad shape");
  // total samples = d_off[n] (device) -> the caller passes offsets of a concatenated list;
  // read the total synchronously (drop-in path; the fused epoch kernel avoids this).
  int64_t total = 0;
  cudaStream_t s = as_stream(stream);
  DBS_CUDA_TRY(cudaMemcpyAsync(&total, d_off + n_workers, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  DBS_CUDA_TRY(cudaStreamSynchronize(s));
  void* c;
  int st = scratch_get(g_coeff_scratch, sizeof(double) * (size_t)(total > 0 ? total : 1), &c);
  if (st) return st;
  int blocks = (int)((total * 32 + 255) / 256);
  if (blocks < 1) blocks = 1;
  if (blocks > num_sms() * 8) blocks = num_sms() * 8;
  logit_coeff_kernel<<<blocks, 256, 0, s>>>(d_x, d_features, d_labels, dim, d_idx, total, (double*)c);
  DBS_LAUNCH_CHECK();
  dim3 grid((unsigned)((dim + 255) / 256 < 64 ? (dim + 255) / 256 : 64), (unsigned)n_workers);
  logit_grads_kernel<<<grid, 256, 0, s>>>(d_x, d_features, dim, d_idx, d_off, (const double*)c, mu, d_out);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

extern "C" int dbs_dev_sq_dist(const double* d_x, const double* d_opt, int64_t dim, double* d_out, int64_t slot,
                               void* stream) {
  sq_dist_kernel<<<1, 512, 0, as_stream(stream)>>>(d_x, d_opt, dim, d_out + slot);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

// Fused epoch of run_parallel_sgd's hot loop (sgdlab.py:380-391) for the
// reference problems.  kind 0 = ConvexProblem, 1 = LogisticProblem.
// d_perm holds the epoch's concatenated permuted spans; span_off[w] (host) is
// where worker w's span starts in it; batches/mode as in aggregate_gradients.
extern "C" int dbs_dev_sgd_epoch(int32_t kind, const double* d_data, const double* d_labels, const double* d_opt,
                                 int64_t dim, double mu, const int64_t* d_perm, const int64_t* span_off,
                                 const int64_t* batches, int64_t n_workers, int32_t mode, int64_t iters, double step,
                                 double momentum, double* d_x, double* d_v, double* d_grads, double* d_coeff,
                                 double* d_sq_out, void* stream) {
  DBS_REQUIRE(n_workers >= 1 && n_workers <= kMaxW && (kind == 0 || kind == 1) && dim > 0, DBS_ERR_ARGUMENT,
              "sgd_epoch: bad arguments");
  DBS_REQUIRE(mode == DBS_AGG_UNIFORM || mode == DBS_AGG_BATCH_WEIGHTED, DBS_ERR_CONFIGURATION,
              "unknown aggregation mode %d", mode);
  WorkerLayout L{};
  L.perm = d_perm;
  L.n = (int)n_workers;
  L.mode = mode;
  double tot = 0.0;
  for (int64_t w = 0; w < n_workers; w++) {
    DBS_REQUIRE(batches[w] > 0, DBS_ERR_CONFIGURATION, "batch sizes must be positive");
    tot += (double)batches[w];
  }
  for (int64_t w = 0; w < n_workers; w++) {
    L.off[w] = span_off[w];
    L.b[w] = batches[w];
    L.w[w] = (double)batches[w] / tot;
  }
  if (iters <= 0) return DBS_OK;
  sgd_epoch_kernel<<<1, kEpochThreads, 0, as_stream(stream)>>>(kind, d_data, d_labels, d_opt, dim, mu, L, iters,
                                                              step, momentum, d_x, d_v, d_grads, d_coeff, d_sq_out);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

// sgd.cu -- batch-weighted gradient aggregation + heavy-ball SGD on one device.
//
// sgdlab.aggregate_gradients (sgdlab.py:208-227):
//   batch_weighted: g = sum_i w_i g_i with w = b / sum(b) in fp64,
//   uniform_average: g = mean_i g_i;
// sgdlab.sgd_step (sgdlab.py:230-238): v' = momentum * v + g, x' = x - step * v'
// (no FMA contraction in the fp64 step, so it is bit-identical to numpy's
// separate multiply/add; the aggregation order is worker 0..n-1).
//
// These kernels serve the single-device paths: the drop-in aggregate/step
// functions, and the per-iteration update when several simulated workers share
// one GPU.  The multi-GPU fused kernel lives in comm.cu.  Everything is
// HBM-bound: (n + 4) * P * sizeof(T) bytes per fused launch, 16-byte vectors,
// grid = a few waves of 148 SMs.
#include "common.cuh"

namespace dbs {
namespace {

constexpr int kMaxWorkers = 64;

struct AggArgs {
  const void* g[kMaxWorkers];
  double w[kMaxWorkers];
  int n;
  int mode;
};

int make_args(AggArgs& a, const void* const* grads, const int64_t* b, int64_t n, int32_t mode) {
  DBS_REQUIRE(n >= 1 && n <= kMaxWorkers, DBS_ERR_ARGUMENT, "aggregate: 1..%d workers supported", kMaxWorkers);
  DBS_REQUIRE(mode == DBS_AGG_UNIFORM || mode == DBS_AGG_BATCH_WEIGHTED, DBS_ERR_CONFIGURATION,
              "unknown aggregation mode %d", mode);
  double tot = 0.0;
  for (int64_t i = 0; i < n; i++) {
    DBS_REQUIRE(b[i] > 0, DBS_ERR_CONFIGURATION, "batch sizes must be positive");
    tot += (double)b[i];
  }
  a.n = (int)n;
  a.mode = mode;
  for (int64_t i = 0; i < n; i++) {
    a.g[i] = grads[i];
    a.w[i] = (mode == DBS_AGG_BATCH_WEIGHTED) ? (double)b[i] / tot : 1.0;
  }
  return DBS_OK;
}

__device__ __forceinline__ double agg_f64(const AggArgs& a, int64_t p) {
  double acc;
  if (a.mode == DBS_AGG_BATCH_WEIGHTED) {
    acc = __dmul_rn(a.w[0], ((const double*)a.g[0])[p]);
    for (int i = 1; i < a.n; i++) acc = __fma_rn(a.w[i], ((const double*)a.g[i])[p], acc);
  } else {
    acc = ((const double*)a.g[0])[p];
    for (int i = 1; i < a.n; i++) acc = __dadd_rn(acc, ((const double*)a.g[i])[p]);
    acc = __ddiv_rn(acc, (double)a.n);
  }
  return acc;
}

__global__ void aggregate_f64_kernel(AggArgs a, int64_t P, double* __restrict__ out) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x)
    out[p] = agg_f64(a, p);
}

__global__ void sgd_step_f64_kernel(const double* __restrict__ x, const double* __restrict__ g,
                                    const double* __restrict__ v, int64_t P, double step, double mom,
                                    double* __restrict__ xo, double* __restrict__ vo) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
    const double nv = __dadd_rn(__dmul_rn(mom, v[p]), g[p]);
    xo[p] = __dsub_rn(x[p], __dmul_rn(step, nv));
    vo[p] = nv;
  }
}

__global__ void aggregate_sgd_f64_kernel(AggArgs a, int64_t P, double step, double mom,
                                         double* __restrict__ x, double* __restrict__ v) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
    const double g = agg_f64(a, p);
    const double nv = __dadd_rn(__dmul_rn(mom, v[p]), g);
    x[p] = __dsub_rn(x[p], __dmul_rn(step, nv));
    v[p] = nv;
  }
}

__device__ __forceinline__ uint32_t bf16_bits(float f) {
  uint32_t u = __float_as_uint(f);
  return (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
}

__device__ __forceinline__ float rn_tf32(float x) {
  const uint32_t u = __float_as_uint(x);
  return __uint_as_float((u + 0xFFFu + ((u >> 13) & 1u)) & 0xFFFFE000u);
}

// operand shadow of 4 consecutive parameters (index 4 p): bf16 [P], or the flat S32
// format of the fp32-class GEMMs (s32.cu): element i's hi at 2 (i & ~31) + (i & 31), lo 32 later
template <int PREC>
__device__ __forceinline__ void store_shadow(void* sh, int64_t p, const float4 x) {
  if (PREC == DBS_PREC_BF16) {
    reinterpret_cast<uint2*>(sh)[p] =
        make_uint2(bf16_bits(x.x) | (bf16_bits(x.y) << 16), bf16_bits(x.z) | (bf16_bits(x.w) << 16));
  } else {
    const int64_t i = 4 * p;
    float* d = reinterpret_cast<float*>(sh) + 2 * (i & ~int64_t(31)) + (i & 31);
    const float4 h = make_float4(rn_tf32(x.x), rn_tf32(x.y), rn_tf32(x.z), rn_tf32(x.w));
    *reinterpret_cast<float4*>(d) = h;
    *reinterpret_cast<float4*>(d + 32) =
        make_float4(rn_tf32(x.x - h.x), rn_tf32(x.y - h.y), rn_tf32(x.z - h.z), rn_tf32(x.w - h.w));
  }
}

// fp32 fused aggregate + step, 4 elements per thread (float4).
template <int PREC>
__global__ void __launch_bounds__(256) aggregate_sgd_f32_kernel(AggArgs a, int64_t P4, float step, float mom,
                                                                float4* __restrict__ x, float4* __restrict__ v,
                                                                void* __restrict__ xb, int64_t* __restrict__ d_iter) {
  // the iteration counter of device-indexed iterations: every reader of this
  // iteration has finished before this kernel starts, the next iteration's start after
  // it ends (one kernel less per iteration than a separate increment)
  if (d_iter != nullptr && blockIdx.x == 0 && threadIdx.x == 0) *d_iter += 1;
  // weights straight from the parameter bank (no local-memory array)
#define W(i) ((a.mode == DBS_AGG_BATCH_WEIGHTED) ? (float)a.w[i] : 1.0f / (float)a.n)
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P4; p += (int64_t)gridDim.x * blockDim.x) {
    float4 g = __ldcs(((const float4*)a.g[0]) + p);
    const float w0 = W(0);
    g.x *= w0; g.y *= w0; g.z *= w0; g.w *= w0;
    for (int i = 1; i < a.n; i++) {
      const float4 h = __ldcs(((const float4*)a.g[i]) + p);
      const float wi = W(i);
      g.x = fmaf(wi, h.x, g.x); g.y = fmaf(wi, h.y, g.y);
      g.z = fmaf(wi, h.z, g.z); g.w = fmaf(wi, h.w, g.w);
    }
    float4 vv = v[p], xx = x[p];
    vv.x = fmaf(mom, vv.x, g.x); vv.y = fmaf(mom, vv.y, g.y);
    vv.z = fmaf(mom, vv.z, g.z); vv.w = fmaf(mom, vv.w, g.w);
    xx.x = fmaf(-step, vv.x, xx.x); xx.y = fmaf(-step, vv.y, xx.y);
    xx.z = fmaf(-step, vv.z, xx.z); xx.w = fmaf(-step, vv.w, xx.w);
    v[p] = vv;
    x[p] = xx;
    if (xb) store_shadow<PREC>(xb, p, xx);
  }
#undef W
}

// the same over 8 parameters per thread with 256-bit accesses (P % 8 == 0, 32-byte
// aligned buffers): the per-iteration kernel of every simulated-worker step
template <int PREC>
__global__ void __launch_bounds__(256) aggregate_sgd_f32x8_kernel(AggArgs a, int64_t P8, float step, float mom,
                                                                  float* __restrict__ x, float* __restrict__ v,
                                                                  void* __restrict__ xb, int64_t* __restrict__ d_iter) {
  if (d_iter != nullptr && blockIdx.x == 0 && threadIdx.x == 0) *d_iter += 1;
#define W(i) ((a.mode == DBS_AGG_BATCH_WEIGHTED) ? (float)a.w[i] : 1.0f / (float)a.n)
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P8; p += (int64_t)gridDim.x * blockDim.x) {
    float g[8];
    {
      const V8 q = ldg8_cs(reinterpret_cast<const float*>(a.g[0]) + 8 * p);
      const float w0 = W(0);
#pragma unroll
      for (int k = 0; k < 8; k++) g[k] = w0 * f8(q, k);
    }
    for (int i = 1; i < a.n; i++) {
      const V8 q = ldg8_cs(reinterpret_cast<const float*>(a.g[i]) + 8 * p);
      const float wi = W(i);
#pragma unroll
      for (int k = 0; k < 8; k++) g[k] = fmaf(wi, f8(q, k), g[k]);
    }
    const V8 vq = ldg8(v + 8 * p), xq = ldg8(x + 8 * p);
    float vv[8], xx[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
      vv[k] = fmaf(mom, f8(vq, k), g[k]);
      xx[k] = fmaf(-step, vv[k], f8(xq, k));
    }
    stg8(v + 8 * p, v8_of(vv));
    stg8(x + 8 * p, v8_of(xx));
    if (xb) {
      if (PREC == DBS_PREC_BF16) {
        reinterpret_cast<uint4*>(xb)[p] =
            make_uint4(bf16_bits(xx[0]) | (bf16_bits(xx[1]) << 16), bf16_bits(xx[2]) | (bf16_bits(xx[3]) << 16),
                       bf16_bits(xx[4]) | (bf16_bits(xx[5]) << 16), bf16_bits(xx[6]) | (bf16_bits(xx[7]) << 16));
      } else {
        const int64_t i = 8 * p;
        float* d = reinterpret_cast<float*>(xb) + 2 * (i & ~int64_t(31)) + (i & 31);
        float h[8], l[8];
#pragma unroll
        for (int k = 0; k < 8; k++) {
          h[k] = rn_tf32(xx[k]);
          l[k] = rn_tf32(xx[k] - h[k]);
        }
        stg8(d, v8_of(h));
        stg8(d + 32, v8_of(l));
      }
    }
  }
#undef W
}

template <int PREC>
__global__ void __launch_bounds__(256) refresh_shadow_kernel(const float4* __restrict__ x, int64_t P4,
                                                             void* __restrict__ xb) {
  pdl_trigger_and_wait();
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P4; p += (int64_t)gridDim.x * blockDim.x)
    store_shadow<PREC>(xb, p, x[p]);
}

// fp32 weighted reduce without the step: out = sum_i w_i g_i (the local level of
// the hierarchical all-reduce when several workers share one GPU)
__global__ void __launch_bounds__(256) aggregate_f32_kernel(AggArgs a, int64_t P4, float4* __restrict__ out) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P4; p += (int64_t)gridDim.x * blockDim.x) {
    const float w0 = (a.mode == DBS_AGG_BATCH_WEIGHTED) ? (float)a.w[0] : 1.0f / (float)a.n;
    float4 g = __ldcs(((const float4*)a.g[0]) + p);
    g.x *= w0; g.y *= w0; g.z *= w0; g.w *= w0;
    for (int i = 1; i < a.n; i++) {
      const float wi = (a.mode == DBS_AGG_BATCH_WEIGHTED) ? (float)a.w[i] : 1.0f / (float)a.n;
      const float4 h = __ldcs(((const float4*)a.g[i]) + p);
      g.x = fmaf(wi, h.x, g.x); g.y = fmaf(wi, h.y, g.y);
      g.z = fmaf(wi, h.z, g.z); g.w = fmaf(wi, h.w, g.w);
    }
    out[p] = g;
  }
}

// model averaging: x_bar = sum_i w_i x_i (the same weights as the gradient
// aggregation), written back to every replica (fp32 + its bf16 operand copy)
struct ReplicaArgs {
  float4* x[kMaxWorkers];
  void* xb[kMaxWorkers];
};

template <int PREC>
__global__ void __launch_bounds__(256) average_replicas_f32_kernel(AggArgs a, ReplicaArgs r, int64_t P4) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P4; p += (int64_t)gridDim.x * blockDim.x) {
    const float w0 = (a.mode == DBS_AGG_BATCH_WEIGHTED) ? (float)a.w[0] : 1.0f / (float)a.n;
    float4 g = r.x[0][p];
    g.x *= w0; g.y *= w0; g.z *= w0; g.w *= w0;
    for (int i = 1; i < a.n; i++) {
      const float wi = (a.mode == DBS_AGG_BATCH_WEIGHTED) ? (float)a.w[i] : 1.0f / (float)a.n;
      const float4 h = r.x[i][p];
      g.x = fmaf(wi, h.x, g.x); g.y = fmaf(wi, h.y, g.y);
      g.z = fmaf(wi, h.z, g.z); g.w = fmaf(wi, h.w, g.w);
    }
    for (int i = 0; i < a.n; i++) {
      r.x[i][p] = g;
      if (r.xb[i]) store_shadow<PREC>(r.xb[i], p, g);
    }
  }
}

int grid_for(int64_t P, int threads) {
  int64_t blocks = (P + threads - 1) / threads;
  int64_t cap = (int64_t)current_sm_count() * 8;
  return (int)(blocks < 1 ? 1 : (blocks < cap ? blocks : cap));
}

}  // namespace
}  // namespace dbs

using namespace dbs;

extern "C" int dbs_dev_aggregate_f64(const double* const* d_grads, const int64_t* b, int64_t n,
                                     int32_t mode, int64_t P, double* d_out, void* stream) {
  AggArgs a;
  int st = make_args(a, (const void* const*)d_grads, b, n, mode);
  if (st) return st;
  if (P <= 0) return DBS_OK;
  aggregate_f64_kernel<<<grid_for(P, 256), 256, 0, as_stream(stream)>>>(a, P, d_out);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

extern "C" int dbs_dev_sgd_step_f64(const double* d_x, const double* d_g, const double* d_v, int64_t P,
                                    double step, double mom, double* d_xo, double* d_vo, void* stream) {
  if (P <= 0) return DBS_OK;
  sgd_step_f64_kernel<<<grid_for(P, 256), 256, 0, as_stream(stream)>>>(d_x, d_g, d_v, P, step, mom, d_xo, d_vo);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

extern "C" int dbs_dev_aggregate_sgd_f64(const double* const* d_grads, const int64_t* b, int64_t n,
                                         int32_t mode, int64_t P, double step, double mom, double* d_x,
                                         double* d_v, void* stream) {
  AggArgs a;
  int st = make_args(a, (const void* const*)d_grads, b, n, mode);
  if (st) return st;
  if (P <= 0) return DBS_OK;
  aggregate_sgd_f64_kernel<<<grid_for(P, 256), 256, 0, as_stream(stream)>>>(a, P, step, mom, d_x, d_v);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

namespace dbs {
int aggregate_sgd_f32_iter(const float* const* d_grads, const int64_t* b, int64_t n, int32_t mode, int64_t P,
                           float step, float mom, float* d_x, float* d_v, void* d_shadow, int32_t shadow_prec,
                           void* stream, int64_t* d_iter);
}

extern "C" int dbs_dev_aggregate_sgd_f32_ex(const float* const* d_grads, const int64_t* b, int64_t n,
                                            int32_t mode, int64_t P, float step, float mom, float* d_x,
                                            float* d_v, void* d_shadow, int32_t shadow_prec, void* stream) {
  return dbs::aggregate_sgd_f32_iter(d_grads, b, n, mode, P, step, mom, d_x, d_v, d_shadow, shadow_prec, stream,
                                     nullptr);
}

// the same, also advancing the device iteration counter d_iter (when not null)
int dbs::aggregate_sgd_f32_iter(const float* const* d_grads, const int64_t* b, int64_t n, int32_t mode, int64_t P,
                                float step, float mom, float* d_x, float* d_v, void* d_shadow, int32_t shadow_prec,
                                void* stream, int64_t* d_iter) {
  AggArgs a;
  int st = make_args(a, (const void* const*)d_grads, b, n, mode);
  if (st) return st;
  DBS_REQUIRE(P % 4 == 0, DBS_ERR_ARGUMENT, "fp32 aggregate: P must be a multiple of 4 (pad the flat buffer)");
  DBS_REQUIRE(shadow_prec == DBS_PREC_BF16 || (shadow_prec == DBS_PREC_F32 && P % 32 == 0), DBS_ERR_ARGUMENT,
              "aggregate_sgd: shadow precision %d (S32 needs P %% 32 == 0)", shadow_prec);
  for (int64_t i = 0; i < n; i++)
    DBS_REQUIRE(((uintptr_t)d_grads[i] % 16) == 0, DBS_ERR_ARGUMENT, "gradient buffers must be 16-byte aligned");
  if (P <= 0) return DBS_OK;
  bool wide = P % 8 == 0 && ((uintptr_t)d_x % 32) == 0 && ((uintptr_t)d_v % 32) == 0 &&
              ((uintptr_t)d_shadow % 32) == 0;
  for (int64_t i = 0; i < n; i++) wide = wide && ((uintptr_t)d_grads[i] % 32) == 0;
  if (wide) {
    const int64_t P8 = P / 8;
    if (shadow_prec == DBS_PREC_F32)
      aggregate_sgd_f32x8_kernel<DBS_PREC_F32><<<grid_for(P8, 256), 256, 0, as_stream(stream)>>>(
          a, P8, step, mom, d_x, d_v, d_shadow, d_iter);
    else
      aggregate_sgd_f32x8_kernel<DBS_PREC_BF16><<<grid_for(P8, 256), 256, 0, as_stream(stream)>>>(
          a, P8, step, mom, d_x, d_v, d_shadow, d_iter);
    DBS_LAUNCH_CHECK();
    return DBS_OK;
  }
  const int64_t P4 = P / 4;
  if (shadow_prec == DBS_PREC_F32)
    aggregate_sgd_f32_kernel<DBS_PREC_F32><<<grid_for(P4, 256), 256, 0, as_stream(stream)>>>(
        a, P4, step, mom, (float4*)d_x, (float4*)d_v, d_shadow, d_iter);
  else
    aggregate_sgd_f32_kernel<DBS_PREC_BF16><<<grid_for(P4, 256), 256, 0, as_stream(stream)>>>(
        a, P4, step, mom, (float4*)d_x, (float4*)d_v, d_shadow, d_iter);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

extern "C" int dbs_dev_aggregate_sgd_f32(const float* const* d_grads, const int64_t* b, int64_t n,
                                         int32_t mode, int64_t P, float step, float mom, float* d_x,
                                         float* d_v, uint16_t* d_x_bf16, void* stream) {
  return dbs_dev_aggregate_sgd_f32_ex(d_grads, b, n, mode, P, step, mom, d_x, d_v, d_x_bf16, DBS_PREC_BF16, stream);
}

extern "C" int dbs_dev_refresh_shadow(const float* d_x, int64_t P, void* d_shadow, int32_t prec, void* stream) {
  DBS_REQUIRE(d_x && d_shadow && P % 4 == 0 && (prec == DBS_PREC_BF16 || (prec == DBS_PREC_F32 && P % 32 == 0)),
              DBS_ERR_ARGUMENT, "refresh_shadow: P %% 4 (bf16) / P %% 32 (S32) and a known precision");
  if (P <= 0) return DBS_OK;
  if (prec == DBS_PREC_F32)
    DBS_CUDA_TRY(launch_pdl(refresh_shadow_kernel<DBS_PREC_F32>, dim3(grid_for(P / 4, 256)), dim3(256), 0,
                            as_stream(stream), (const float4*)d_x, P / 4, d_shadow));
  else
    DBS_CUDA_TRY(launch_pdl(refresh_shadow_kernel<DBS_PREC_BF16>, dim3(grid_for(P / 4, 256)), dim3(256), 0,
                            as_stream(stream), (const float4*)d_x, P / 4, d_shadow));
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

extern "C" int dbs_dev_aggregate_f32(const float* const* d_grads, const int64_t* b, int64_t n, int32_t mode, int64_t P,
                                     float* d_out, void* stream) {
  AggArgs a;
  int st = make_args(a, (const void* const*)d_grads, b, n, mode);
  if (st) return st;
  DBS_REQUIRE(P % 4 == 0, DBS_ERR_ARGUMENT, "fp32 aggregate: P must be a multiple of 4");
  if (P <= 0) return DBS_OK;
  aggregate_f32_kernel<<<grid_for(P / 4, 256), 256, 0, as_stream(stream)>>>(a, P / 4, (float4*)d_out);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

extern "C" int dbs_dev_average_replicas_f32_ex(float* const* d_params, const int64_t* b, int64_t n, int32_t mode,
                                               int64_t P, void* const* d_shadows, int32_t shadow_prec, void* stream) {
  AggArgs a;
  int st = make_args(a, (const void* const*)d_params, b, n, mode);
  if (st) return st;
  DBS_REQUIRE(P % 4 == 0, DBS_ERR_ARGUMENT, "average_replicas: P must be a multiple of 4");
  DBS_REQUIRE(shadow_prec == DBS_PREC_BF16 || (shadow_prec == DBS_PREC_F32 && P % 32 == 0), DBS_ERR_ARGUMENT,
              "average_replicas: shadow precision %d (S32 needs P %% 32 == 0)", shadow_prec);
  ReplicaArgs r;
  for (int64_t i = 0; i < n; i++) {
    DBS_REQUIRE(((uintptr_t)d_params[i] % 16) == 0, DBS_ERR_ARGUMENT, "replica buffers must be 16-byte aligned");
    r.x[i] = reinterpret_cast<float4*>(d_params[i]);
    r.xb[i] = d_shadows ? d_shadows[i] : nullptr;
  }
  if (P <= 0) return DBS_OK;
  if (shadow_prec == DBS_PREC_F32)
    average_replicas_f32_kernel<DBS_PREC_F32><<<grid_for(P / 4, 256), 256, 0, as_stream(stream)>>>(a, r, P / 4);
  else
    average_replicas_f32_kernel<DBS_PREC_BF16><<<grid_for(P / 4, 256), 256, 0, as_stream(stream)>>>(a, r, P / 4);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

extern "C" int dbs_dev_average_replicas_f32(float* const* d_params, const int64_t* b, int64_t n, int32_t mode,
                                            int64_t P, uint16_t* const* d_params_bf16, void* stream) {
  return dbs_dev_average_replicas_f32_ex(d_params, b, n, mode, P, reinterpret_cast<void* const*>(d_params_bf16),
                                         DBS_PREC_BF16, stream);
}

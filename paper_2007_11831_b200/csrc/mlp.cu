// mlp.cu -- variable-batch forward/backward of the 784-H-C MLP on tcgen05, and
// the native per-epoch iteration driver of synchronous DBS S-SGD.
//
// Reference loop being accelerated: sgdlab.run_parallel_sgd (sgdlab.py:380-391):
//   for t in iterations: for each worker, mean gradient on batch t of its
//   permuted span -> aggregate_gradients(batch_weighted) -> sgd_step.
// Per worker and iteration (7 launches, all on the worker's stream):
//   1. H   = relu(X W1^T + b1)        tcgen05 GEMM, fused bias+ReLU, bf16 out
//   2. Z   = H W2^T + b2              tcgen05 GEMM (N = C <= 16), fp32 logits
//   3. softmax cross-entropy          dZ = (softmax - onehot) / b, db2, loss
//   4. dW2 = dZ^T H                   tcgen05 GEMM, both operands MN-major
//   5. dH  = (dZ W2) * [H > 0]        tcgen05 GEMM, fused ReLU-backward, + per-warp
//                                     column sums for db1 (deterministic)
//   6. db1 = sum of the column-sum partials
//   7. dW1 = dH^T X                   tcgen05 GEMM, both operands MN-major
// The flat fp32 gradient [W1 | b1 | W2 | b2] (each block padded to 8 elements)
// is then combined across workers by the fused aggregate+SGD kernel, which also
// refreshes the bf16 parameter shadow the GEMMs read.
#include <mutex>
#include <vector>

#include "common.cuh"

namespace dbs {
int gemm_bf16(const void* a, int a_mn, int64_t lda, const void* b, int b_mn, int64_t ldb, void* d, int64_t ldd,
              int64_t M, int64_t N, int64_t K, int epi, const float* bias, const void* aux, cudaStream_t s,
              float* colsum_part);
int gemm_tf(const void* a, int a_mn, int64_t lda, const void* b, int b_mn, int64_t ldb, void* d, int64_t ldd,
            int64_t M, int64_t N, int64_t K, int epi, const float* bias, const void* aux, cudaStream_t s,
            float* colsum_part = nullptr);
int stamp(int64_t* d_stamps, int64_t slot, cudaStream_t s);
int spin_scaled(const int64_t* d_stamps, int64_t b, int64_t e, float scale, int ctas, cudaStream_t s);
int ctx_push(void* ctx);
int ctx_pop(void* ctx);
}  // namespace dbs

struct dbs_mlp {
  int64_t in, hid, cls, max_b;
  int prec = DBS_PREC_BF16;     // DBS_PREC_F32: S32 operands, 3xTF32 GEMMs
  int64_t in_ld;                // W1 row length / input row length (f32: in rounded up to 32)
  int64_t off_w1, off_b1, off_w2, off_b2, P;
  void* act = nullptr;          // [max_b][hid] bf16 | S32
  float* logits = nullptr;      // [max_b][16]
  void* dz = nullptr;           // [max_b][16] bf16 | [max_b][32] S32
  void* dh = nullptr;           // [max_b][hid] bf16 | S32
  float* colsum = nullptr;      // [ceil(max_b/32)][hid]
  void* xstage = nullptr;       // [max_b] input rows of the current iteration (device-indexed iterations)
};

namespace dbs {
namespace {

constexpr int64_t kLdZ = 16;

int64_t pad8(int64_t x) { return (x + 7) & ~int64_t(7); }

__device__ __forceinline__ uint16_t f2bf(float f) {
  uint32_t u = __float_as_uint(f);
  return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}

// One CTA: mean cross-entropy over b rows, dZ = (softmax - onehot)/b (bf16),
// db2 = sum_rows dZ (fp32, deterministic block reduction), loss.
__global__ void __launch_bounds__(256) softmax_ce_kernel(const float* __restrict__ z, const int32_t* __restrict__ y_base,
                                                         int64_t b, int cls, uint16_t* __restrict__ dz,
                                                         float* __restrict__ db2, float* __restrict__ loss,
                                                         const int64_t* __restrict__ d_iter, int loss_indexed) {
  // device-indexed iteration (graph replays): rows t*b.. of the shard's labels, loss slot t
  const int64_t t_it = d_iter ? *d_iter : 0;
  const int32_t* __restrict__ y = y_base + t_it * b;
  if (loss_indexed) loss += t_it;
  __shared__ float red[8][17];
  float acc[16];
  float lsum = 0.0f;
#pragma unroll
  for (int c = 0; c < 16; c++) acc[c] = 0.0f;
  const float inv_b = 1.0f / (float)b;
  for (int64_t r = threadIdx.x; r < b; r += blockDim.x) {
    const float* zr = z + r * kLdZ;
    float mx = -INFINITY;
    for (int c = 0; c < cls; c++) mx = fmaxf(mx, zr[c]);
    float se = 0.0f;
    float e[16];
#pragma unroll
    for (int c = 0; c < 16; c++) {
      e[c] = (c < cls) ? __expf(zr[c] - mx) : 0.0f;
      se += e[c];
    }
    const int yr = y[r];
    lsum += (mx + __logf(se)) - zr[yr];
    const float inv = 1.0f / se;
#pragma unroll
    for (int c = 0; c < 16; c++) {
      float g = (c < cls) ? (e[c] * inv - (c == yr ? 1.0f : 0.0f)) * inv_b : 0.0f;
      acc[c] += g;
      dz[r * kLdZ + c] = f2bf(g);
    }
  }
  // block reduction of acc[0..cls) and lsum
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int c = 0; c < 16; c++) {
    float s = acc[c];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[warp][c] = s;
  }
  for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
  if (lane == 0) red[warp][16] = lsum;
  __syncthreads();
  if (threadIdx.x < 17) {
    float s = 0.0f;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) s += red[w][threadIdx.x];
    if (threadIdx.x < cls) db2[threadIdx.x] = s;
    if (threadIdx.x == 16) *loss = s * inv_b;
  }
}

// fp32-class form: dZ written in S32 ([b][32], zero past cls -- the K padding of
// the dH GEMM and the M tail of the dW2 GEMM)
__device__ __forceinline__ float rn_tf32(float x) {
  const uint32_t u = __float_as_uint(x);
  return __uint_as_float((u + 0xFFFu + ((u >> 13) & 1u)) & 0xFFFFE000u);
}
__global__ void __launch_bounds__(256) softmax_ce_s32_kernel(const float* __restrict__ z, const int32_t* __restrict__ y_base,
                                                             int64_t b, int cls, float* __restrict__ dz,
                                                             float* __restrict__ db2, float* __restrict__ loss,
                                                         const int64_t* __restrict__ d_iter, int loss_indexed) {
  // device-indexed iteration (graph replays): rows t*b.. of the shard's labels, loss slot t
  const int64_t t_it = d_iter ? *d_iter : 0;
  const int32_t* __restrict__ y = y_base + t_it * b;
  if (loss_indexed) loss += t_it;
  __shared__ float red[8][17];
  float acc[16];
  float lsum = 0.0f;
#pragma unroll
  for (int c = 0; c < 16; c++) acc[c] = 0.0f;
  const float inv_b = 1.0f / (float)b;
  for (int64_t r = threadIdx.x; r < b; r += blockDim.x) {
    const float* zr = z + r * kLdZ;
    float mx = -INFINITY;
    for (int c = 0; c < cls; c++) mx = fmaxf(mx, zr[c]);
    float se = 0.0f;
    float e[16];
#pragma unroll
    for (int c = 0; c < 16; c++) {
      e[c] = (c < cls) ? expf(zr[c] - mx) : 0.0f;
      se += e[c];
    }
    const int yr = y[r];
    lsum += (mx + logf(se)) - zr[yr];
    const float inv = 1.0f / se;
    float* d = dz + r * 64;
#pragma unroll
    for (int c = 0; c < 32; c++) {
      const float g = (c < cls) ? (e[c & 15] * inv - (c == yr ? 1.0f : 0.0f)) * inv_b : 0.0f;
      if (c < 16) acc[c] += g;
      const float h = rn_tf32(g);
      d[c] = h;
      d[32 + c] = rn_tf32(g - h);
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int c = 0; c < 16; c++) {
    float s = acc[c];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[warp][c] = s;
  }
  for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
  if (lane == 0) red[warp][16] = lsum;
  __syncthreads();
  if (threadIdx.x < 17) {
    float s = 0.0f;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) s += red[w][threadIdx.x];
    if (threadIdx.x < cls) db2[threadIdx.x] = s;
    if (threadIdx.x == 16) *loss = s * inv_b;
  }
}

// device-indexed iteration: rows [t b, (t + 1) b) of the worker's shard (t = *d_iter)
// -> the fixed staging rows every GEMM of the iteration reads (graph replays keep
// their TMA descriptors; 16-byte vectors, row bytes a multiple of 16)
__global__ void __launch_bounds__(256) stage_rows_kernel(const uint4* __restrict__ shard, const int64_t* __restrict__ d_iter,
                                                         int64_t b, int64_t row_vec, uint4* __restrict__ out) {
  const int64_t n = b * row_vec;
  const uint4* src = shard + (*d_iter) * n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = src[i];
}

// db1[n] = sum_g part[g][n] over g < groups (fixed order => deterministic)
__global__ void colsum_reduce_kernel(const float* __restrict__ part, int64_t groups, int64_t n,
                                     float* __restrict__ out) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.0f;
    for (int64_t g = 0; g < groups; g++) s += part[g * n + j];
    out[j] = s;
  }
}

}  // namespace

// fp32-class forward/backward: the same 5 GEMMs on S32 operands (3xTF32).  x is the
// S32 input [b][in_ld], the shadow the flat S32 parameter vector (W1 [H][in_ld])
int mlp_fwd_bwd_f32(dbs_mlp* m, const float* sh, const float* pf, const float* x, const int32_t* y, int64_t b,
                    float* grad, float* loss, cudaStream_t s, const int64_t* d_iter, int loss_indexed) {
  int st;
  const int64_t I = m->in_ld, H = m->hid, C = m->cls;
  const float* w1 = sh + 2 * m->off_w1;
  const float* w2 = sh + 2 * m->off_w2;
  st = gemm_tf(x, 0, I, w1, 0, I, m->act, H, b, H, I, DBS_EPI_BIAS_RELU_S32, pf + m->off_b1, nullptr, s, nullptr);
  if (st) return st;
  st = gemm_tf(m->act, 0, H, w2, 0, H, m->logits, kLdZ, b, C, H, DBS_EPI_BIAS_F32, pf + m->off_b2, nullptr, s, nullptr);
  if (st) return st;
  softmax_ce_s32_kernel<<<1, 256, 0, s>>>(m->logits, y, b, (int)C, static_cast<float*>(m->dz), grad + m->off_b2, loss,
                                          d_iter, loss_indexed);
  DBS_LAUNCH_CHECK();
  // dW2 [C][H] = dZ^T H  (dZ S32 [b][32] MN-major, M = C)
  st = gemm_tf(m->dz, 1, 32, m->act, 1, H, grad + m->off_w2, H, C, H, b, DBS_EPI_F32, nullptr, nullptr, s, nullptr);
  if (st) return st;
  // dH = (dZ W2) * [H > 0]: K = C (padded to 32 with dZ's zero columns), W2 [C][H] read MN-major
  st = gemm_tf(m->dz, 0, 32, w2, 1, H, m->dh, H, b, H, C, DBS_EPI_RELU_GRAD_S32, nullptr, m->act, s, m->colsum);
  if (st) return st;
  {
    int grid = (int)((H + 255) / 256);
    colsum_reduce_kernel<<<grid, 256, 0, s>>>(m->colsum, (b + 31) / 32, H, grad + m->off_b1);
    DBS_LAUNCH_CHECK();
  }
  // dW1 [H][in_ld] = dH^T X  (columns past `in` are 0: X's zero padding)
  return gemm_tf(m->dh, 1, H, x, 1, I, grad + m->off_w1, I, H, I, b, DBS_EPI_F32, nullptr, nullptr, s, nullptr);
}

// d_iter != nullptr: x_any / y are the worker's whole shard and the iteration index t
// is read on the device (rows t b.. staged into m->xstage; labels and, with
// loss_indexed, the loss slot t offset by the kernels) -- every launch argument is
// then iteration-invariant, so one iteration can be captured in a CUDA graph.
int mlp_fwd_bwd(dbs_mlp* m, const void* shadow, const float* pf, const void* x_any, const int32_t* y, int64_t b,
                float* grad, float* loss, cudaStream_t s, const int64_t* d_iter, int loss_indexed) {
  DBS_REQUIRE(m && shadow && pf && x_any && y && grad && loss, DBS_ERR_ARGUMENT, "mlp: null argument");
  DBS_REQUIRE(b >= 1 && b <= m->max_b, DBS_ERR_ARGUMENT, "mlp: batch %lld outside [1, %lld]", (long long)b,
              (long long)m->max_b);
  if (d_iter) {
    const int64_t row_bytes = m->prec == DBS_PREC_F32 ? 8 * m->in_ld : 2 * m->in;
    DBS_REQUIRE(row_bytes % 16 == 0 && ((uintptr_t)x_any & 15) == 0, DBS_ERR_ARGUMENT,
                "mlp: device-indexed rows need 16-byte rows");
    const int64_t vec = row_bytes / 16;
    const int64_t blocks = (b * vec + 255) / 256;
    stage_rows_kernel<<<(unsigned)(blocks < 1184 ? blocks : 1184), 256, 0, s>>>(
        static_cast<const uint4*>(x_any), d_iter, b, vec, static_cast<uint4*>(m->xstage));
    DBS_LAUNCH_CHECK();
    x_any = m->xstage;
  } else {
    loss_indexed = 0;
  }
  if (m->prec == DBS_PREC_F32)
    return mlp_fwd_bwd_f32(m, static_cast<const float*>(shadow), pf, static_cast<const float*>(x_any), y, b, grad, loss,
                           s, d_iter, loss_indexed);
  const uint16_t* pb = static_cast<const uint16_t*>(shadow);
  const uint16_t* x = static_cast<const uint16_t*>(x_any);
  int st;
  const int64_t I = m->in, H = m->hid, C = m->cls;
  // 1. forward layer 1
  st = gemm_bf16(x, 0, I, pb + m->off_w1, 0, I, m->act, H, b, H, I, DBS_EPI_BIAS_RELU_BF16, pf + m->off_b1,
                 nullptr, s, nullptr);
  if (st) return st;
  // 2. logits
  st = gemm_bf16(m->act, 0, H, pb + m->off_w2, 0, H, m->logits, kLdZ, b, C, H, DBS_EPI_BIAS_F32, pf + m->off_b2,
                 nullptr, s, nullptr);
  if (st) return st;
  // 3. softmax cross-entropy + db2
  softmax_ce_kernel<<<1, 256, 0, s>>>(m->logits, y, b, (int)C, static_cast<uint16_t*>(m->dz), grad + m->off_b2, loss,
                                      d_iter, loss_indexed);
  DBS_LAUNCH_CHECK();
  // 4. dW2 = dZ^T H
  st = gemm_bf16(m->dz, 1, kLdZ, m->act, 1, H, grad + m->off_w2, H, C, H, b, DBS_EPI_F32, nullptr, nullptr, s,
                 nullptr);
  if (st) return st;
  // 5. dH = (dZ W2) * [H > 0], with db1 partial column sums
  st = gemm_bf16(m->dz, 0, kLdZ, pb + m->off_w2, 1, H, m->dh, H, b, H, C, DBS_EPI_RELU_GRAD_BF16, nullptr, m->act,
                 s, m->colsum);
  if (st) return st;
  // 6. db1
  {
    int grid = (int)((H + 255) / 256);
    colsum_reduce_kernel<<<grid, 256, 0, s>>>(m->colsum, (b + 31) / 32, H, grad + m->off_b1);
    DBS_LAUNCH_CHECK();
  }
  // 7. dW1 = dH^T X
  st = gemm_bf16(m->dh, 1, H, x, 1, I, grad + m->off_w1, I, H, I, b, DBS_EPI_F32, nullptr, nullptr, s, nullptr);
  return st;
}

}  // namespace dbs

using namespace dbs;

extern "C" int dbs_mlp_create_ex(int64_t in_dim, int64_t hidden, int64_t classes, int64_t max_batch, int32_t precision,
                                 dbs_mlp** out) {
  DBS_REQUIRE(out && in_dim > 0 && hidden > 16 && classes >= 2 && classes <= 16 && max_batch > 0, DBS_ERR_ARGUMENT,
              "mlp_create: need in>0, hidden>16, 2<=classes<=16");
  DBS_REQUIRE(precision == DBS_PREC_BF16 || precision == DBS_PREC_F32, DBS_ERR_ARGUMENT, "mlp_create: precision %d",
              precision);
  DBS_REQUIRE(in_dim % 8 == 0 && hidden % (precision == DBS_PREC_F32 ? 32 : 8) == 0, DBS_ERR_ARGUMENT,
              "mlp_create: in must be a multiple of 8, hidden of 8 (bf16) / 32 (f32)");
  dbs_mlp* m = new dbs_mlp();
  m->in = in_dim;
  m->hid = hidden;
  m->cls = classes;
  m->max_b = max_batch;
  m->prec = precision;
  const bool f32 = precision == DBS_PREC_F32;
  // f32: every block starts on a 32-element boundary (the flat S32 shadow), W1 rows padded to 32
  auto padp = [&](int64_t x) { return f32 ? (x + 31) & ~int64_t(31) : pad8(x); };
  m->in_ld = f32 ? (in_dim + 31) & ~int64_t(31) : in_dim;
  m->off_w1 = 0;
  m->off_b1 = padp(hidden * m->in_ld);
  m->off_w2 = m->off_b1 + padp(hidden);
  m->off_b2 = m->off_w2 + padp(classes * hidden);
  m->P = m->off_b2 + padp(classes);
  const int64_t groups = (max_batch + 31) / 32 + 4;
  const size_t es = f32 ? 8 : 2;  // bytes per stored operand element (S32 hi + lo | bf16)
  cudaError_t e = cudaSuccess;
  e = e ? e : cudaMalloc(&m->act, es * max_batch * hidden);
  e = e ? e : cudaMalloc(&m->logits, sizeof(float) * max_batch * kLdZ);
  e = e ? e : cudaMalloc(&m->dz, f32 ? es * max_batch * 32 : es * max_batch * kLdZ);
  e = e ? e : cudaMalloc(&m->dh, es * max_batch * hidden);
  e = e ? e : cudaMalloc(&m->colsum, sizeof(float) * groups * hidden);
  e = e ? e : cudaMalloc(&m->xstage, (f32 ? 8 * m->in_ld : 2 * in_dim) * max_batch);
  if (e != cudaSuccess) {
    set_error("mlp_create: %s", cudaGetErrorString(e));
    dbs_mlp_destroy(m);
    return DBS_ERR_CUDA;
  }
  *out = m;
  return DBS_OK;
}

extern "C" int dbs_mlp_create(int64_t in_dim, int64_t hidden, int64_t classes, int64_t max_batch, dbs_mlp** out) {
  return dbs_mlp_create_ex(in_dim, hidden, classes, max_batch, DBS_PREC_BF16, out);
}

extern "C" int dbs_mlp_info(const dbs_mlp* m, int32_t* precision, int64_t* in_ld) {
  DBS_REQUIRE(m, DBS_ERR_ARGUMENT, "mlp_info: null");
  if (precision) *precision = m->prec;
  if (in_ld) *in_ld = m->in_ld;
  return DBS_OK;
}

extern "C" int dbs_mlp_destroy(dbs_mlp* m) {
  if (!m) return DBS_OK;
  cudaFree(m->act);
  cudaFree(m->logits);
  cudaFree(m->dz);
  cudaFree(m->dh);
  cudaFree(m->colsum);
  cudaFree(m->xstage);
  delete m;
  return DBS_OK;
}

extern "C" int dbs_mlp_param_count(const dbs_mlp* m, int64_t* out) {
  DBS_REQUIRE(m && out, DBS_ERR_ARGUMENT, "mlp_param_count: null");
  *out = m->P;
  return DBS_OK;
}

extern "C" int dbs_mlp_forward_backward(dbs_mlp* m, const void* d_params_shadow, const float* d_params,
                                        const void* d_x, const int32_t* d_labels, int64_t batch,
                                        float* d_grad, float* d_loss, void* stream) {
  return mlp_fwd_bwd(m, d_params_shadow, d_params, d_x, d_labels, batch, d_grad, d_loss, as_stream(stream), nullptr, 0);
}

// ---------------------------------------------------------------------------
// Native iteration driver: iterations [t0, t1) of one epoch for n workers.
// Each worker runs on its own stream (optionally an SM-partitioned green
// context); the aggregation + SGD kernel joins them on agg_stream.  Per-worker
// compute time is accumulated on the device from %globaltimer stamps.
// ---------------------------------------------------------------------------
namespace {
// One pool per host thread: two trainers driven from different threads never
// record or wait on each other's events, and a grow cannot move another
// caller's pointer.  (Events are never destroyed; a pool lives as long as its thread.)
thread_local std::vector<cudaEvent_t> g_events;
int events(int n, cudaEvent_t** out) {
  while ((int)g_events.size() < n) {
    cudaEvent_t e;
    DBS_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    g_events.push_back(e);
  }
  *out = g_events.data();
  return DBS_OK;
}
}  // namespace

extern "C" int dbs_dev_aggregate_sgd_f32_ex(const float* const* d_grads, const int64_t* b, int64_t n, int32_t mode,
                                            int64_t P, float step, float mom, float* d_x, float* d_v, void* d_shadow,
                                            int32_t shadow_prec, void* stream);
extern "C" int dbs_dev_refresh_shadow(const float* d_x, int64_t P, void* d_shadow, int32_t prec, void* stream);
extern "C" int dbs_dev_spin_for(int32_t num_ctas, int64_t ns, void* stream);
extern "C" int dbs_dev_accumulate_time(const int64_t* d_stamps, int64_t begin, int64_t end, double* d_seconds,
                                       int64_t worker, void* stream);

namespace dbs {
int resnet_fwd_bwd(dbs_resnet* m, const void* shadow, const float* pf, const void* x_base, const int32_t* y_base,
                   const int64_t* d_iter, int64_t B, float* grad, float* loss, cudaStream_t s);
int resnet_param_count(const dbs_resnet* m);
int64_t resnet_row_bytes(const dbs_resnet* m);
int resnet_precision(const dbs_resnet* m);

// operand precision (DBS_PREC_*) of a worker's model: the format of the parameter shadow
int slot_precision(const dbs_worker_slot& w) {
  return w.model_kind == DBS_MODEL_MLP ? static_cast<const dbs_mlp*>(w.model)->prec
                                       : resnet_precision(static_cast<const dbs_resnet*>(w.model));
}
// bytes of one input row of the worker's shard
int64_t slot_row_bytes(const dbs_worker_slot& w) {
  if (w.model_kind == DBS_MODEL_MLP) {
    const dbs_mlp* m = static_cast<const dbs_mlp*>(w.model);
    return m->prec == DBS_PREC_F32 ? 8 * m->in_ld : 2 * m->in;
  }
  return resnet_row_bytes(static_cast<const dbs_resnet*>(w.model));
}
int iter_increment(int64_t* d_iter, cudaStream_t s);
int aggregate_sgd_f32_iter(const float* const* d_grads, const int64_t* b, int64_t n, int32_t mode, int64_t P,
                           float step, float mom, float* d_x, float* d_v, void* d_shadow, int32_t shadow_prec,
                           void* stream, int64_t* d_iter);
}  // namespace dbs

extern "C" int dbs_dev_aggregate_f32(const float* const* d_grads, const int64_t* b, int64_t n, int32_t mode, int64_t P,
                                     float* d_out, void* stream);
extern "C" int dbs_comm_allreduce_sgd(dbs_comm* c, const int64_t* batch_sizes, int32_t mode, float step,
                                      float momentum, float* d_velocity_shard, void* stream);
extern "C" int dbs_comm_buffers(dbs_comm* c, float** d_grad, float** d_param, uint16_t** d_param_bf16);
extern "C" int dbs_comm_shadow(const dbs_comm* c, void** d_shadow, int32_t* prec);

static int run_iterations_impl(const dbs_worker_slot* w, int32_t n, int64_t t0, int64_t t1, int32_t mode, float lr,
                               float mom, float* d_params, float* d_velocity, void* d_shadow,
                               int32_t skip_update, void* agg_stream, int64_t* d_iter, dbs_comm* comm,
                               const int64_t* rank_batches, dbs_worker_graphs* graphs = nullptr,
                               bool capture_only = false);

namespace dbs {
long long launch_count();
void add_launches(long long d);
void count_host_launch();
}  // namespace dbs

// One CUDA graph per worker: that worker's part of an iteration (stamps, optional
// spin, forward/backward reading the iteration index from d_iter, compute-time
// accumulation), captured on the worker's stream with its SM partition's context
// current -- so the worker's ~100 launches per iteration become one graph launch
// inside its green context, and the iteration driver issues n graph launches plus
// the update instead of n x ~100 kernels from one host thread.
struct dbs_worker_graphs {
  int n = 0;
  cudaGraphExec_t exec[64] = {};
  long long kernels[64] = {};  // kernels per replay (for dbs_launch_count)
};

extern "C" int dbs_worker_graphs_create(int32_t n, dbs_worker_graphs** out) {
  DBS_REQUIRE(out && n >= 1 && n <= 64, DBS_ERR_ARGUMENT, "worker_graphs_create: 1 <= n <= 64");
  dbs_worker_graphs* g = new dbs_worker_graphs();
  g->n = n;
  *out = g;
  return DBS_OK;
}

extern "C" int dbs_worker_graphs_destroy(dbs_worker_graphs* g) {
  if (!g) return DBS_OK;
  for (int i = 0; i < g->n; i++)
    if (g->exec[i]) cudaGraphExecDestroy(g->exec[i]);
  delete g;
  return DBS_OK;
}

extern "C" int dbs_run_iterations(const dbs_worker_slot* w, int32_t n, int64_t t0, int64_t t1, int32_t mode, float lr,
                                  float mom, float* d_params, float* d_velocity, void* d_params_shadow,
                                  int32_t skip_update, void* agg_stream, int64_t* d_iter) {
  return run_iterations_impl(w, n, t0, t1, mode, lr, mom, d_params, d_velocity, d_params_shadow, skip_update,
                             agg_stream, d_iter, nullptr, nullptr);
}

// ---------------------------------------------------------------------------
// Device-side epoch loop (single-context workers: C1, ResNet on one GPU without
// partitions): ONE CUDA graph per plan whose `while` conditional node runs the
// captured iteration (every worker's forward/backward, the update, the iteration
// counter increment) until *d_iter reaches *d_total -- one graph launch per epoch,
// no host launch and no inter-graph gap per iteration.
// ---------------------------------------------------------------------------
struct dbs_epoch_graph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  long long kernels_per_iter = 0;
};

namespace dbs {
namespace {
__global__ void epoch_cond_kernel(cudaGraphConditionalHandle h, const int64_t* __restrict__ d_iter,
                                  const int64_t* __restrict__ d_total) {
  cudaGraphSetConditional(h, (*d_iter < *d_total) ? 1u : 0u);
}
}  // namespace
}  // namespace dbs

extern "C" int dbs_epoch_graph_destroy(dbs_epoch_graph* e) {
  if (!e) return DBS_OK;
  if (e->exec) cudaGraphExecDestroy(e->exec);
  if (e->graph) cudaGraphDestroy(e->graph);
  delete e;
  return DBS_OK;
}

extern "C" int dbs_epoch_graph_create(const dbs_worker_slot* w, int32_t n, int32_t mode, float lr, float mom,
                                      float* d_params, float* d_velocity, void* d_params_shadow,
                                      int32_t skip_update, void* agg_stream, int64_t* d_iter,
                                      const int64_t* d_total, dbs_epoch_graph** out) {
  DBS_REQUIRE(w && n >= 1 && d_iter && d_total && out, DBS_ERR_ARGUMENT, "epoch_graph_create: bad arguments");
  for (int i = 0; i < n; i++)
    DBS_REQUIRE(w[i].ctx == nullptr, DBS_ERR_ARGUMENT, "epoch_graph_create: workers must share one context");
  dbs_epoch_graph* e = new dbs_epoch_graph();
  cudaStream_t agg = as_stream(agg_stream);
  const long long c0 = launch_count();
  int st = [&]() -> int {
    DBS_CUDA_TRY(cudaGraphCreate(&e->graph, 0));
    cudaGraphConditionalHandle h;
    DBS_CUDA_TRY(cudaGraphConditionalHandleCreate(&h, e->graph, 1u, cudaGraphCondAssignDefault));
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    DBS_CUDA_TRY(cudaGraphAddNode(&node, e->graph, nullptr, 0, &np));
    cudaGraph_t body = np.conditional.phGraph_out[0];
    DBS_CUDA_TRY(cudaStreamBeginCaptureToGraph(agg, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    int st_i = run_iterations_impl(w, n, 0, 1, mode, lr, mom, d_params, d_velocity, d_params_shadow, skip_update,
                                   agg_stream, d_iter, nullptr, nullptr);
    if (st_i == DBS_OK) {
      dbs::epoch_cond_kernel<<<1, 1, 0, agg>>>(h, d_iter, d_total);
      const cudaError_t e_l = cudaGetLastError();
      if (e_l != cudaSuccess) {
        set_error("epoch_graph_create: %s", cudaGetErrorString(e_l));
        st_i = DBS_ERR_CUDA;
      }
    }
    cudaGraph_t captured = nullptr;
    const cudaError_t e_end = cudaStreamEndCapture(agg, &captured);
    if (st_i) return st_i;
    DBS_CUDA_TRY(e_end);
    DBS_CUDA_TRY(cudaGraphInstantiate(&e->exec, e->graph, 0));
    return DBS_OK;
  }();
  e->kernels_per_iter = launch_count() - c0;
  add_launches(-e->kernels_per_iter);  // recorded, not executed
  if (st) {
    dbs_epoch_graph_destroy(e);
    *out = nullptr;
    return st;
  }
  e->kernels_per_iter += 1;  // the condition kernel
  *out = e;
  return DBS_OK;
}

// One epoch: *d_iter must be 0 and *d_total = iters >= 1 (set on `stream` before)
extern "C" int dbs_epoch_graph_launch(dbs_epoch_graph* e, int64_t iters, void* stream) {
  DBS_REQUIRE(e && e->exec && iters >= 1, DBS_ERR_ARGUMENT, "epoch_graph_launch: bad arguments");
  DBS_CUDA_TRY(cudaGraphLaunch(e->exec, as_stream(stream)));
  add_launches(e->kernels_per_iter * iters);
  count_host_launch();
  return DBS_OK;
}

// Capture (and instantiate) the per-worker graphs without running anything: done
// before an epoch's disturbance kernels start, since capturing may load kernels
// lazily and a module load would wait behind a spin kernel that owns SMs.
extern "C" int dbs_worker_graphs_capture(const dbs_worker_slot* w, int32_t n, int32_t mode, float lr, float mom,
                                         float* d_params, float* d_velocity, void* d_params_shadow,
                                         int32_t skip_update, void* agg_stream, int64_t* d_iter,
                                         dbs_worker_graphs* graphs) {
  DBS_REQUIRE(graphs, DBS_ERR_ARGUMENT, "worker_graphs_capture: null graphs");
  return run_iterations_impl(w, n, 0, 0, mode, lr, mom, d_params, d_velocity, d_params_shadow, skip_update,
                             agg_stream, d_iter, nullptr, nullptr, graphs, true);
}

extern "C" int dbs_run_iterations_graphed(const dbs_worker_slot* w, int32_t n, int64_t t0, int64_t t1, int32_t mode,
                                          float lr, float mom, float* d_params, float* d_velocity,
                                          void* d_params_shadow, int32_t skip_update, void* agg_stream,
                                          int64_t* d_iter, dbs_worker_graphs* graphs) {
  DBS_REQUIRE(graphs, DBS_ERR_ARGUMENT, "run_iterations_graphed: null graphs");
  return run_iterations_impl(w, n, t0, t1, mode, lr, mom, d_params, d_velocity, d_params_shadow, skip_update,
                             agg_stream, d_iter, nullptr, nullptr, graphs);
}

// Multi-GPU form: this rank's n local workers, then the hierarchical update --
// local weighted reduce into the communicator's gradient block (skipped for
// one worker, whose gradient is written there directly) and the fused NVLink
// all-reduce + momentum SGD with per-rank weights rank_batches[r] = sum of
// that rank's worker batches.  Parameters live in the communicator's blocks.
static int run_iterations_comm(const dbs_worker_slot* w, int32_t n, int64_t t0, int64_t t1, int32_t mode,
                               float lr, float mom, dbs_comm* comm, const int64_t* rank_batches,
                               float* d_velocity_shard, void* agg_stream, int64_t* d_iter,
                               dbs_worker_graphs* graphs, bool capture_only);

extern "C" int dbs_run_iterations_comm(const dbs_worker_slot* w, int32_t n, int64_t t0, int64_t t1, int32_t mode,
                                       float lr, float mom, dbs_comm* comm, const int64_t* rank_batches,
                                       float* d_velocity_shard, void* agg_stream, int64_t* d_iter) {
  return run_iterations_comm(w, n, t0, t1, mode, lr, mom, comm, rank_batches, d_velocity_shard, agg_stream, d_iter,
                             nullptr, false);
}

// the multi-GPU form with per-worker graphs (capture_only = 1: capture, run nothing)
extern "C" int dbs_run_iterations_comm_graphed(const dbs_worker_slot* w, int32_t n, int64_t t0, int64_t t1,
                                               int32_t mode, float lr, float mom, dbs_comm* comm,
                                               const int64_t* rank_batches, float* d_velocity_shard,
                                               void* agg_stream, int64_t* d_iter, dbs_worker_graphs* graphs,
                                               int32_t capture_only) {
  DBS_REQUIRE(graphs && d_iter, DBS_ERR_ARGUMENT, "run_iterations_comm_graphed: graphs and d_iter required");
  return run_iterations_comm(w, n, t0, t1, mode, lr, mom, comm, rank_batches, d_velocity_shard, agg_stream, d_iter,
                             graphs, capture_only != 0);
}

static int run_iterations_comm(const dbs_worker_slot* w, int32_t n, int64_t t0, int64_t t1, int32_t mode,
                               float lr, float mom, dbs_comm* comm, const int64_t* rank_batches,
                               float* d_velocity_shard, void* agg_stream, int64_t* d_iter,
                               dbs_worker_graphs* graphs, bool capture_only) {
  DBS_REQUIRE(comm && rank_batches && d_velocity_shard, DBS_ERR_ARGUMENT, "run_iterations_comm: null argument");
  float *g = nullptr, *p = nullptr;
  void* sh = nullptr;
  int32_t prec = 0;
  int st = dbs_comm_buffers(comm, &g, &p, nullptr);
  if (st) return st;
  st = dbs_comm_shadow(comm, &sh, &prec);
  if (st) return st;
  DBS_REQUIRE(n >= 1 && prec == slot_precision(w[0]), DBS_ERR_ARGUMENT,
              "run_iterations_comm: the communicator's shadow precision differs from the model's");
  return run_iterations_impl(w, n, t0, t1, mode, lr, mom, p, d_velocity_shard, sh, 0, agg_stream, d_iter, comm,
                             rank_batches, graphs, capture_only);
}

static int run_iterations_impl(const dbs_worker_slot* w, int32_t n, int64_t t0, int64_t t1, int32_t mode, float lr,
                               float mom, float* d_params, float* d_velocity, void* d_shadow,
                               int32_t skip_update, void* agg_stream, int64_t* d_iter, dbs_comm* comm,
                               const int64_t* rank_batches, dbs_worker_graphs* graphs, bool capture_only) {
  DBS_REQUIRE(w && n >= 1 && n <= 64 && t1 >= t0, DBS_ERR_ARGUMENT, "run_iterations: bad arguments");
  for (int i = 0; i < n; i++)
    DBS_REQUIRE(w[i].model && (w[i].model_kind == DBS_MODEL_MLP || w[i].model_kind == DBS_MODEL_RESNET18),
                DBS_ERR_ARGUMENT, "run_iterations: worker %d has a bad model", i);
  const int prec = slot_precision(w[0]);
  for (int i = 1; i < n; i++)
    DBS_REQUIRE(slot_precision(w[i]) == prec, DBS_ERR_ARGUMENT, "run_iterations: workers mix operand precisions");
  cudaEvent_t* ev;
  int st = events(n + 1, &ev);
  if (st) return st;
  cudaStream_t agg = as_stream(agg_stream);
  const float* grads[64];
  int64_t batches[64];
  for (int i = 0; i < n; i++) {
    grads[i] = w[i].grad;
    batches[i] = w[i].batch;
  }
  const int64_t P = (w[0].model_kind == DBS_MODEL_MLP) ? static_cast<const dbs_mlp*>(w[0].model)->P
                                                       : resnet_param_count(static_cast<const dbs_resnet*>(w[0].model));
  // worker i's part of iteration t on stream s (its partition's context current)
  auto issue_worker = [&](int i, cudaStream_t s, int64_t t) -> int {
      if (w[i].stamps) {
        st = stamp(w[i].stamps, 0, s);
        if (st) return st;
      }
      if (w[i].spin_ns > 0 && w[i].spin_ctas > 0) {  // extra_epoch_seconds disturbance
        st = dbs_dev_spin_for(w[i].spin_ctas, w[i].spin_ns, s);
        if (st) return st;
      }
      const int64_t b = w[i].batch;
      if (w[i].model_kind == DBS_MODEL_MLP) {
        dbs_mlp* m = static_cast<dbs_mlp*>(w[i].model);
        if (d_iter) {  // device-indexed iteration (graph capture): the kernels offset by *d_iter
          st = mlp_fwd_bwd(m, d_shadow, d_params, w[i].x_shard, w[i].y_shard, b, w[i].grad,
                           w[i].loss ? w[i].loss : w[i].loss_scratch, s, d_iter, w[i].loss ? 1 : 0);
        } else {
          const char* x = static_cast<const char*>(w[i].x_shard) + t * b * slot_row_bytes(w[i]);
          st = mlp_fwd_bwd(m, d_shadow, d_params, x, w[i].y_shard + t * b, b, w[i].grad,
                           w[i].loss ? w[i].loss + t : w[i].loss_scratch, s, nullptr, 0);
        }
      } else {
        dbs_resnet* m = static_cast<dbs_resnet*>(w[i].model);
        const uint8_t* x = static_cast<const uint8_t*>(w[i].x_shard);
        const int32_t* y = w[i].y_shard;
        float* loss = w[i].loss;
        if (!d_iter) {  // host-indexed iteration
          x += t * b * resnet_row_bytes(m);
          y += t * b;
          loss = loss ? loss + t : nullptr;
        }
        st = resnet_fwd_bwd(m, d_shadow, d_params, x, y, d_iter, b, w[i].grad, loss, s);
      }
      if (st) return st;
      if (w[i].stamps) {
        st = stamp(w[i].stamps, 1, s);
        if (st) return st;
        if (w[i].slow_scale > 0.f && w[i].slow_ctas > 0) {
          // simulated slower device: extend this worker's critical path in
          // proportion to its own forward/backward time, then re-stamp
          st = spin_scaled(w[i].stamps, 0, 1, w[i].slow_scale, w[i].slow_ctas, s);
          if (st) return st;
          st = stamp(w[i].stamps, 1, s);
          if (st) return st;
        }
        st = dbs_dev_accumulate_time(w[i].stamps, 0, 1, w[i].seconds, w[i].worker_index, s);
        if (st) return st;
      }
      return DBS_OK;
  };
  if (graphs) {
    DBS_REQUIRE(d_iter && graphs->n == n, DBS_ERR_ARGUMENT, "run_iterations: worker graphs need d_iter and n workers");
    for (int i = 0; i < n; i++) {
      if (graphs->exec[i]) continue;
      cudaStream_t s = as_stream(w[i].stream);
      st = ctx_push(w[i].ctx);
      if (st) return st;
      const long long c0 = launch_count();
      st = [&]() -> int {
        DBS_CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        const int st_w = issue_worker(i, s, 0);
        cudaGraph_t g = nullptr;
        const cudaError_t e_end = cudaStreamEndCapture(s, &g);
        if (st_w) {
          if (g) cudaGraphDestroy(g);
          return st_w;
        }
        DBS_CUDA_TRY(e_end);
        const cudaError_t e_inst = cudaGraphInstantiate(&graphs->exec[i], g, 0);
        cudaGraphDestroy(g);
        DBS_CUDA_TRY(e_inst);
        return DBS_OK;
      }();
      graphs->kernels[i] = launch_count() - c0;
      add_launches(-graphs->kernels[i]);  // recorded, not executed
      const int st_pop = ctx_pop(w[i].ctx);
      if (st) return st;
      if (st_pop) return st_pop;
    }
    if (capture_only) return DBS_OK;
  }
  DBS_CUDA_TRY(cudaEventRecord(ev[n], agg));
  for (int64_t t = t0; t < t1; t++) {
    for (int i = 0; i < n; i++) {
      cudaStream_t s = as_stream(w[i].stream);
      // the worker's launches happen with its SM partition's context current
      st = ctx_push(w[i].ctx);
      if (st) return st;
      st = [&]() -> int {
        DBS_CUDA_TRY(cudaStreamWaitEvent(s, ev[n], 0));  // parameters of iteration t ready
        if (graphs) {
          DBS_CUDA_TRY(cudaGraphLaunch(graphs->exec[i], s));
          add_launches(graphs->kernels[i]);
          count_host_launch();
        } else {
          const int st_w = issue_worker(i, s, t);
          if (st_w) return st_w;
        }
        DBS_CUDA_TRY(cudaEventRecord(ev[i], s));
        return DBS_OK;
      }();
      const int st_pop = ctx_pop(w[i].ctx);
      if (st) return st;
      if (st_pop) return st_pop;
    }
    for (int i = 0; i < n; i++) DBS_CUDA_TRY(cudaStreamWaitEvent(agg, ev[i], 0));
    bool iter_done = false;  // the update kernel advanced d_iter itself
    if (!skip_update && comm == nullptr) {
      st = aggregate_sgd_f32_iter(grads, batches, n, mode, P, lr, mom, d_params, d_velocity, d_shadow, prec,
                                  agg_stream, d_iter);
      if (st) return st;
      iter_done = d_iter != nullptr;
    } else if (!skip_update) {
      float* cg = nullptr;
      st = dbs_comm_buffers(comm, &cg, nullptr, nullptr);
      if (st) return st;
      if (!(n == 1 && grads[0] == cg)) {
        st = dbs_dev_aggregate_f32(grads, batches, n, mode, P, cg, agg_stream);
        if (st) return st;
      }
      st = dbs_comm_allreduce_sgd(comm, rank_batches, mode, lr, mom, d_velocity, agg_stream);
      if (st) return st;
      if (prec == DBS_PREC_F32) {  // the fp32 parameters arrived from every peer; S32 operand copy locally
        st = dbs_dev_refresh_shadow(d_params, P, d_shadow, prec, agg_stream);
        if (st) return st;
      }
    }
    if (d_iter && !iter_done) {
      st = iter_increment(d_iter, agg);
      if (st) return st;
    }
    DBS_CUDA_TRY(cudaEventRecord(ev[n], agg));
  }
  return DBS_OK;
}

// Periodic model averaging (local SGD): worker i trains its own replica
// (d_params[i], d_velocity[i], d_params_bf16[i]) with a local momentum-SGD step
// on its own stream every iteration; after every sync_interval-th iteration of
// the epoch (t + 1 multiple of sync_interval) the replicas are averaged with the
// batch weights of `mode` -- floor(T / sync_interval) rounds per epoch
// (cluster.sync_rounds_for_epoch, cluster.py:185-186).  Between rounds no
// worker waits for another.
static int run_iterations_local(const dbs_worker_slot* w, int32_t n, int64_t t0, int64_t t1, int32_t mode, float lr,
                                float mom, int32_t sync_interval, float* const* d_params, float* const* d_velocity,
                                void* const* d_shadows, void* agg_stream, dbs_comm* comm,
                                const int64_t* rank_batches, dbs_worker_graphs* graphs = nullptr,
                                int64_t* d_iters = nullptr, bool capture_only = false);

extern "C" int dbs_run_iterations_local(const dbs_worker_slot* w, int32_t n, int64_t t0, int64_t t1, int32_t mode,
                                        float lr, float mom, int32_t sync_interval, float* const* d_params,
                                        float* const* d_velocity, void* const* d_params_shadow, void* agg_stream) {
  return run_iterations_local(w, n, t0, t1, mode, lr, mom, sync_interval, d_params, d_velocity, d_params_shadow,
                              agg_stream, nullptr, nullptr);
}

// Model averaging across GPUs: every sync round first averages this rank's
// replicas (weighted by the local batches), then averages replica 0 -- which
// must be the communicator's symmetric parameter block -- across the ranks with
// the fused NVLink kernel (rank weights = the ranks' batch sums, so the result is
// the global batch-weighted average), and copies it back into the other replicas.
extern "C" int dbs_run_iterations_local_comm(const dbs_worker_slot* w, int32_t n, int64_t t0, int64_t t1,
                                             int32_t mode, float lr, float mom, int32_t sync_interval,
                                             float* const* d_params, float* const* d_velocity,
                                             void* const* d_params_shadow, dbs_comm* comm,
                                             const int64_t* rank_batches, void* agg_stream) {
  DBS_REQUIRE(comm && rank_batches, DBS_ERR_ARGUMENT, "run_iterations_local_comm: null communicator / batches");
  return run_iterations_local(w, n, t0, t1, mode, lr, mom, sync_interval, d_params, d_velocity, d_params_shadow,
                              agg_stream, comm, rank_batches);
}

// Per-worker CUDA graphs for local SGD (graphs != NULL): worker i's block -- forward /
// backward reading its own device iteration counter d_iters[i], its local momentum
// step, the counter increment -- is captured once in its partition's context and
// replayed each iteration; the periodic averaging stays on the aggregation stream.
extern "C" int dbs_run_iterations_local_graphed(const dbs_worker_slot* w, int32_t n, int64_t t0, int64_t t1,
                                                int32_t mode, float lr, float mom, int32_t sync_interval,
                                                float* const* d_params, float* const* d_velocity,
                                                void* const* d_params_shadow, void* agg_stream, int64_t* d_iters,
                                                dbs_worker_graphs* graphs, int32_t capture_only) {
  DBS_REQUIRE(graphs && d_iters, DBS_ERR_ARGUMENT, "run_iterations_local_graphed: graphs and d_iters required");
  return run_iterations_local(w, n, t0, t1, mode, lr, mom, sync_interval, d_params, d_velocity, d_params_shadow,
                              agg_stream, nullptr, nullptr, graphs, d_iters, capture_only != 0);
}

static int run_iterations_local(const dbs_worker_slot* w, int32_t n, int64_t t0, int64_t t1, int32_t mode, float lr,
                                float mom, int32_t sync_interval, float* const* d_params, float* const* d_velocity,
                                void* const* d_shadows, void* agg_stream, dbs_comm* comm,
                                const int64_t* rank_batches, dbs_worker_graphs* graphs, int64_t* d_iters,
                                bool capture_only) {
  DBS_REQUIRE(w && n >= 1 && n <= 64 && t1 >= t0 && sync_interval >= 1 && d_params && d_velocity && d_shadows,
              DBS_ERR_ARGUMENT, "run_iterations_local: bad arguments");
  for (int i = 0; i < n; i++)
    DBS_REQUIRE(w[i].model && (w[i].model_kind == DBS_MODEL_MLP || w[i].model_kind == DBS_MODEL_RESNET18),
                DBS_ERR_ARGUMENT, "run_iterations_local: worker %d has a bad model", i);
  const int prec = slot_precision(w[0]);
  for (int i = 1; i < n; i++)
    DBS_REQUIRE(slot_precision(w[i]) == prec, DBS_ERR_ARGUMENT, "run_iterations_local: workers mix operand precisions");
  cudaEvent_t* ev;
  int st = events(n + 1, &ev);
  if (st) return st;
  cudaStream_t agg = as_stream(agg_stream);
  int64_t batches[64];
  for (int i = 0; i < n; i++) batches[i] = w[i].batch;
  const int64_t P = (w[0].model_kind == DBS_MODEL_MLP) ? static_cast<const dbs_mlp*>(w[0].model)->P
                                                       : resnet_param_count(static_cast<const dbs_resnet*>(w[0].model));
  // worker i's part of local iteration t on stream s (its partition's context current);
  // dev: iteration index from d_iters[i] (graph capture), incremented at the end
  auto issue_local = [&](int i, cudaStream_t s, int64_t t, bool dev) -> int {
        if (w[i].stamps) {
          st = stamp(w[i].stamps, 0, s);
          if (st) return st;
        }
        if (w[i].spin_ns > 0 && w[i].spin_ctas > 0) {
          st = dbs_dev_spin_for(w[i].spin_ctas, w[i].spin_ns, s);
          if (st) return st;
        }
        const int64_t b = w[i].batch;
        if (dev) {
          if (w[i].model_kind == DBS_MODEL_MLP) {
            dbs_mlp* m = static_cast<dbs_mlp*>(w[i].model);
            st = mlp_fwd_bwd(m, d_shadows[i], d_params[i], w[i].x_shard, w[i].y_shard, b, w[i].grad,
                             w[i].loss ? w[i].loss : w[i].loss_scratch, s, d_iters + i, w[i].loss ? 1 : 0);
          } else {
            dbs_resnet* m = static_cast<dbs_resnet*>(w[i].model);
            st = resnet_fwd_bwd(m, d_shadows[i], d_params[i], w[i].x_shard, w[i].y_shard, d_iters + i, b,
                                w[i].grad, w[i].loss, s);
          }
        } else {
          const char* x = static_cast<const char*>(w[i].x_shard) + t * b * slot_row_bytes(w[i]);
          if (w[i].model_kind == DBS_MODEL_MLP) {
            dbs_mlp* m = static_cast<dbs_mlp*>(w[i].model);
            st = mlp_fwd_bwd(m, d_shadows[i], d_params[i], x, w[i].y_shard + t * b, b, w[i].grad,
                             w[i].loss ? w[i].loss + t : w[i].loss_scratch, s, nullptr, 0);
          } else {
            dbs_resnet* m = static_cast<dbs_resnet*>(w[i].model);
            st = resnet_fwd_bwd(m, d_shadows[i], d_params[i], x, w[i].y_shard + t * b, nullptr, b, w[i].grad,
                                w[i].loss ? w[i].loss + t : nullptr, s);
          }
        }
        if (st) return st;
        if (w[i].stamps) {
          st = stamp(w[i].stamps, 1, s);
          if (st) return st;
          if (w[i].slow_scale > 0.f && w[i].slow_ctas > 0) {
            st = spin_scaled(w[i].stamps, 0, 1, w[i].slow_scale, w[i].slow_ctas, s);
            if (st) return st;
            st = stamp(w[i].stamps, 1, s);
            if (st) return st;
          }
          st = dbs_dev_accumulate_time(w[i].stamps, 0, 1, w[i].seconds, w[i].worker_index, s);
          if (st) return st;
        }
        // the worker's own momentum-SGD step on its replica
        const float* g = w[i].grad;
        const int64_t one = 1;
        st = aggregate_sgd_f32_iter(&g, &one, 1, DBS_AGG_UNIFORM, P, lr, mom, d_params[i], d_velocity[i],
                                    d_shadows[i], prec, s, dev ? d_iters + i : nullptr);
        if (st) return st;
        return DBS_OK;
  };
  if (graphs) {
    DBS_REQUIRE(graphs->n == n, DBS_ERR_ARGUMENT, "run_iterations_local: graph set for %d workers", graphs->n);
    for (int i = 0; i < n; i++) {
      if (graphs->exec[i]) continue;
      cudaStream_t s = as_stream(w[i].stream);
      st = ctx_push(w[i].ctx);
      if (st) return st;
      const long long c0 = launch_count();
      st = [&]() -> int {
        DBS_CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        const int st_w = issue_local(i, s, 0, true);
        cudaGraph_t g = nullptr;
        const cudaError_t e_end = cudaStreamEndCapture(s, &g);
        if (st_w) {
          if (g) cudaGraphDestroy(g);
          return st_w;
        }
        DBS_CUDA_TRY(e_end);
        const cudaError_t e_inst = cudaGraphInstantiate(&graphs->exec[i], g, 0);
        cudaGraphDestroy(g);
        DBS_CUDA_TRY(e_inst);
        return DBS_OK;
      }();
      graphs->kernels[i] = launch_count() - c0;
      add_launches(-graphs->kernels[i]);
      const int st_pop = ctx_pop(w[i].ctx);
      if (st) return st;
      if (st_pop) return st_pop;
    }
    if (capture_only) return DBS_OK;
  }
  DBS_CUDA_TRY(cudaEventRecord(ev[n], agg));
  for (int i = 0; i < n; i++) DBS_CUDA_TRY(cudaStreamWaitEvent(as_stream(w[i].stream), ev[n], 0));
  for (int64_t t = t0; t < t1; t++) {
    const bool sync = ((t + 1) % sync_interval) == 0;
    for (int i = 0; i < n; i++) {
      cudaStream_t s = as_stream(w[i].stream);
      st = ctx_push(w[i].ctx);
      if (st) return st;
      st = [&]() -> int {
        if (graphs) {
          DBS_CUDA_TRY(cudaGraphLaunch(graphs->exec[i], s));
          add_launches(graphs->kernels[i]);
          count_host_launch();
        } else {
          const int st_w = issue_local(i, s, t, false);
          if (st_w) return st_w;
        }
        if (sync) DBS_CUDA_TRY(cudaEventRecord(ev[i], s));
        return DBS_OK;
      }();
      const int st_pop = ctx_pop(w[i].ctx);
      if (st) return st;
      if (st_pop) return st_pop;
    }
    if (sync) {
      for (int i = 0; i < n; i++) DBS_CUDA_TRY(cudaStreamWaitEvent(agg, ev[i], 0));
      st = dbs_dev_average_replicas_f32_ex(d_params, batches, n, mode, P, d_shadows, prec, agg_stream);
      if (st) return st;
      if (comm) {
        st = dbs_comm_average_params(comm, rank_batches, mode, agg_stream);
        if (st) return st;
        if (prec == DBS_PREC_F32) {
          st = dbs_dev_refresh_shadow(d_params[0], P, d_shadows[0], prec, agg_stream);
          if (st) return st;
        }
        const size_t sh_bytes = prec == DBS_PREC_F32 ? sizeof(float) * 2 * P : sizeof(uint16_t) * P;
        for (int i = 1; i < n; i++) {
          DBS_CUDA_TRY(cudaMemcpyAsync(d_params[i], d_params[0], sizeof(float) * P, cudaMemcpyDeviceToDevice, agg));
          DBS_CUDA_TRY(cudaMemcpyAsync(d_shadows[i], d_shadows[0], sh_bytes, cudaMemcpyDeviceToDevice, agg));
        }
      }
      DBS_CUDA_TRY(cudaEventRecord(ev[n], agg));
      for (int i = 0; i < n; i++) DBS_CUDA_TRY(cudaStreamWaitEvent(as_stream(w[i].stream), ev[n], 0));
    }
  }
  // the epoch ends with every worker joined into the aggregation stream
  for (int i = 0; i < n; i++) {
    DBS_CUDA_TRY(cudaEventRecord(ev[i], as_stream(w[i].stream)));
    DBS_CUDA_TRY(cudaStreamWaitEvent(agg, ev[i], 0));
  }
  return DBS_OK;
}

extern "C" int dbs_mlp_run_iterations(const dbs_worker_slot* w, int32_t n, int64_t t0, int64_t t1, int32_t mode,
                                      float lr, float mom, float* d_params, float* d_velocity, void* d_params_shadow,
                                      int32_t skip_update, void* agg_stream) {
  return dbs_run_iterations(w, n, t0, t1, mode, lr, mom, d_params, d_velocity, d_params_shadow, skip_update,
                            agg_stream, nullptr);
}

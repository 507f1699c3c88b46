// resnet.cu -- ResNet-18 (CIFAR stem: 3x3 conv, no max-pool; configs 3-4) and
// ResNet-50 (ImageNet stem: 7x7/2 conv + 3x3/2 max-pool, bottleneck blocks
// [3, 4, 6, 3] with the stride on the 3x3 conv as in torchvision; config 5)
// forward/backward of one worker's variable batch, on the tcgen05
// implicit-GEMM convolution.
//
// These are the named models of BASELINE.json's configs: the per-worker
// gradient of sgdlab.minibatch_gradient (sgdlab.py:200-205) for a network the
// reference only models by its cost (cluster.py:132-145).
//
// Layout: activations NHWC bf16; conv weights [Cout][R][S][Cin] (K-major, c
// fastest) in one flat fp32 parameter vector with a bf16 shadow (the GEMM
// operand), BN gamma/beta fp32, FC fp32.  Per conv (all on the worker stream):
//   forward : implicit-GEMM conv (4-D TMA) -> bf16 y + per-warp BN partial sums
//             -> bn_stats (fp64 reduce) -> bn_apply (+ReLU, +residual/+BN(ds))
//   backward: bn_bwd_reduce / bn_bwd_apply (ReLU mask recomputed from the saved
//             output) -> dgrad = conv(dY, flipped W) (stride-2: dY dilated) with
//             bf16 accumulation of the shortcut gradient -> wgrad = dY^T im2col(X)
//             (split-K, fp32 atomics into the flat gradient)
// BatchNorm uses the worker's own batch statistics (local BN, as in DDP without
// SyncBN); the f32 mode also keeps torch-style running statistics
// (dbs_resnet_running_stats).
#include <math.h>
#include <stdlib.h>

#include <mutex>
#include <vector>

#include "common.cuh"
#include "gemm.cuh"

namespace dbs {

namespace {

constexpr float kBnEps = 1e-5f;
constexpr int kStemK = 32;     // ResNet-18 stem: 27 = 3x3x3 padded to 32
constexpr int kStem7K = 160;   // ResNet-50 stem: 147 = 7x7x3 padded to 160 (K blocks past 160 are TMA zero fill)

__device__ __forceinline__ uint16_t f2bf(float f) {
  uint32_t u = __float_as_uint(f);
  return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}
__device__ __forceinline__ float bf2f(uint16_t h) { return __uint_as_float(((uint32_t)h) << 16); }

struct Conv {
  int cin, cout, k, stride, pad;
  int H, W, OH, OW;         // input / output spatial
  int64_t w_off, w_len;     // weight block in the flat parameter vector
  int64_t g_off, b_off;     // BN gamma / beta
};

struct Block {
  int c1, c2, c3, ds;  // indices into convs (c3 = -1: basic block; ds = -1: identity shortcut)
};

// ----------------------------- kernels ------------------------------------

// stem im2col: x fp32 [B][3][32][32] (CHW per sample, the repacked shard row
// t*B .. ) -> A bf16 [B*1024][32], K = (r, s, c) with c fastest, zero padded.
__global__ void im2col_stem_kernel(const float* __restrict__ x_base, const int64_t* __restrict__ iter, int64_t B,
                                   uint16_t* __restrict__ out) {
  pdl_trigger_and_wait();
  const int64_t t = iter ? *iter : 0;
  const float* x = x_base + t * B * 3072;
  const int64_t total = B * 1024;
  for (int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pix < total;
       pix += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = pix >> 10;
    const int h = (int)((pix >> 5) & 31), w = (int)(pix & 31);
    const float* xs = x + n * 3072;
    uint32_t packed[16];
#pragma unroll
    for (int q = 0; q < 16; q++) packed[q] = 0;
#pragma unroll
    for (int r = 0; r < 3; r++)
#pragma unroll
      for (int s = 0; s < 3; s++)
#pragma unroll
        for (int c = 0; c < 3; c++) {
          const int hh = h + r - 1, ww = w + s - 1;
          const float v = (hh >= 0 && hh < 32 && ww >= 0 && ww < 32) ? xs[c * 1024 + hh * 32 + ww] : 0.0f;
          const int k = (r * 3 + s) * 3 + c;
          packed[k >> 1] |= (uint32_t)f2bf(v) << ((k & 1) * 16);
        }
    uint4* o = reinterpret_cast<uint4*>(out + pix * kStemK);
#pragma unroll
    for (int q = 0; q < 4; q++) o[q] = make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
  }
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void unpack8(const uint4 q, float (&v)[8]) {
  v[0] = __uint_as_float(q.x << 16); v[1] = __uint_as_float(q.x & 0xFFFF0000u);
  v[2] = __uint_as_float(q.y << 16); v[3] = __uint_as_float(q.y & 0xFFFF0000u);
  v[4] = __uint_as_float(q.z << 16); v[5] = __uint_as_float(q.z & 0xFFFF0000u);
  v[6] = __uint_as_float(q.w << 16); v[7] = __uint_as_float(q.w & 0xFFFF0000u);
}
__device__ __forceinline__ uint4 pack8(const float (&v)[8]) {
  return make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]),
                    pack_bf16x2(v[6], v[7]));
}
// 8 consecutive per-channel coefficients from a shared-memory table
__device__ __forceinline__ void coef8(const float* t, int c0, float (&k)[8]) {
  const float4 a = *reinterpret_cast<const float4*>(t + c0), b = *reinterpret_cast<const float4*>(t + c0 + 4);
  k[0] = a.x; k[1] = a.y; k[2] = a.z; k[3] = a.w; k[4] = b.x; k[5] = b.y; k[6] = b.z; k[7] = b.w;
}

// out = act( a*y + b  [+ res | + a_d*yd + b_d] ), a = gamma*invstd, b = beta - mean*a:
// the per-channel affine maps are formed once per CTA in shared memory; 8
// channels (one 16-byte vector) per thread and trip
__device__ __forceinline__ void bn_finalise(const double* acc, int C, int c, int64_t M, float& mean, float& invstd) {
  const double mu = acc[c] / (double)M;
  double var = acc[C + c] / (double)M - mu * mu;
  if (var < 0.0) var = 0.0;
  mean = (float)mu;
  invstd = (float)(1.0 / sqrt(var + (double)kBnEps));
}

__global__ void __launch_bounds__(256) bn_apply_kernel(const uint16_t* __restrict__ y, const double* __restrict__ acc,
                                float* __restrict__ mean, float* __restrict__ invstd, const float* __restrict__ gamma,
                                const float* __restrict__ beta, const uint16_t* __restrict__ res,
                                const uint16_t* __restrict__ yd, const double* __restrict__ acc_d,
                                float* __restrict__ mean_d, float* __restrict__ invstd_d,
                                const float* __restrict__ gamma_d, const float* __restrict__ beta_d, int relu, int C,
                                int64_t M, uint16_t* __restrict__ out) {
  pdl_trigger_and_wait();
  // the conv epilogue's fp64 column sums -> mean, 1/sqrt(var + eps) (every CTA
  // forms them for its table; CTA 0 also publishes them for the backward pass)
  extern __shared__ float tab[];  // [C] a, [C] b, ([C] a_d, [C] b_d)
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float mu, is;
    bn_finalise(acc, C, c, M, mu, is);
    const float a = gamma[c] * is;
    tab[c] = a;
    tab[C + c] = beta[c] - mu * a;
    if (blockIdx.x == 0) {
      mean[c] = mu;
      invstd[c] = is;
    }
    if (yd) {
      float mud, isd;
      bn_finalise(acc_d, C, c, M, mud, isd);
      const float ad = gamma_d[c] * isd;
      tab[2 * C + c] = ad;
      tab[3 * C + c] = beta_d[c] - mud * ad;
      if (blockIdx.x == 0) {
        mean_d[c] = mud;
        invstd_d[c] = isd;
      }
    }
  }
  __syncthreads();
  const int cv = C / 8;
  const int64_t total = M * cv;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c0 = (int)(i & (int64_t)(cv - 1)) * 8;  // C is a power of two (64..2048)
    float v[8], ka[8], kb[8];
    unpack8(reinterpret_cast<const uint4*>(y)[i], v);
    coef8(tab, c0, ka);
    coef8(tab + C, c0, kb);
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] = fmaf(ka[k], v[k], kb[k]);
    if (res) {
      float r[8];
      unpack8(reinterpret_cast<const uint4*>(res)[i], r);
#pragma unroll
      for (int k = 0; k < 8; k++) v[k] += r[k];
    }
    if (yd) {
      float r[8];
      unpack8(reinterpret_cast<const uint4*>(yd)[i], r);
      coef8(tab + 2 * C, c0, ka);
      coef8(tab + 3 * C, c0, kb);
#pragma unroll
      for (int k = 0; k < 8; k++) v[k] += fmaf(ka[k], r[k], kb[k]);
    }
    if (relu) {
#pragma unroll
      for (int k = 0; k < 8; k++) v[k] = fmaxf(v[k], 0.0f);
    }
    reinterpret_cast<uint4*>(out)[i] = pack8(v);
  }
}

// BN backward, pass 1: dbeta[c] += sum g, dgamma[c] += sum g*yhat,
// g = gin * [mask > 0] (mask = saved post-ReLU output, nullable)
template <int C8>
__global__ void __launch_bounds__(256, 4) bn_bwd_reduce_kernel(const uint16_t* __restrict__ gin,
                                                            const uint16_t* __restrict__ mask,
                                                            const uint16_t* __restrict__ y,
                                                            const float* __restrict__ mean,
                                                            const float* __restrict__ invstd, int C, int64_t M,
                                                            float* __restrict__ dgamma, float* __restrict__ dbeta) {
  pdl_trigger_and_wait();
  // each thread owns 8 channels (c0 = 8 * (tid % cv)) over rows tid / cv, +rows_per_pass
  __shared__ float red_g[2048], red_b[2048];
  const int cv = C / 8;
  const int rows_per_pass = blockDim.x / cv;
  const int lane_c = threadIdx.x % cv, lane_r = threadIdx.x / cv;
  float sg[8], sb[8], mu[8], is[8];
  const int c0 = lane_c * 8;
#pragma unroll
  for (int k = 0; k < 8; k++) {
    sg[k] = 0.f;
    sb[k] = 0.f;
    mu[k] = mean[c0 + k];
    is[k] = invstd[c0 + k];
  }
  if (lane_r < rows_per_pass) {
    // four rows per trip, all twelve 16-byte loads issued before the arithmetic
    const int64_t step = (int64_t)gridDim.x * rows_per_pass;
    const uint4 zero = make_uint4(0, 0, 0, 0), ones = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
    for (int64_t r = (int64_t)blockIdx.x * rows_per_pass + lane_r; r < M; r += 4 * step) {
      uint4 qg[4], qy[4], qm[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int64_t rr = r + u * step;
        const bool ok = rr < M;
        const int64_t i = rr * cv + lane_c;
        qg[u] = ok ? reinterpret_cast<const uint4*>(gin)[i] : zero;
        qy[u] = ok ? reinterpret_cast<const uint4*>(y)[i] : zero;
        qm[u] = (ok && mask) ? reinterpret_cast<const uint4*>(mask)[i] : ones;
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        float g[8], yv[8], mv[8];
        unpack8(qg[u], g);
        unpack8(qy[u], yv);
        unpack8(qm[u], mv);
#pragma unroll
        for (int k = 0; k < 8; k++) {
          const float gg = mv[k] > 0.0f ? g[k] : 0.0f;
          sb[k] += gg;
          sg[k] = fmaf(gg, (yv[k] - mu[k]) * is[k], sg[k]);
        }
      }
    }
  }
  // reduction over lane_r: first inside the warp (lanes lane_c, lane_c + cv, ...
  // hold the same channels), then across the warps in shared memory, then one
  // global atomic per channel and block
  if (cv < 32) {
#pragma unroll
    for (int k = 0; k < 8; k++) {
      for (int o = cv; o < 32; o <<= 1) {
        sg[k] += __shfl_xor_sync(0xffffffffu, sg[k], o);
        sb[k] += __shfl_xor_sync(0xffffffffu, sb[k], o);
      }
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const bool writer = (cv < 32) ? (lane < cv) : (lane_r < rows_per_pass);
  const int slot = (cv < 32) ? warp : lane_r;  // partial index
  const int nslot = (cv < 32) ? nw : rows_per_pass;
  if (writer) {
#pragma unroll
    for (int k = 0; k < 8; k++) {
      red_g[slot * C + c0 + k] = sg[k];
      red_b[slot * C + c0 + k] = sb[k];
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < C; idx += blockDim.x) {
    float a = 0.f, b = 0.f;
    for (int r = 0; r < nslot; r++) {
      a += red_g[r * C + idx];
      b += red_b[r * C + idx];
    }
    atomicAdd(&dgamma[idx], a);
    atomicAdd(&dbeta[idx], b);
  }
}

// BN backward, pass 2: dy = gamma*invstd*(g - dbeta/M - yhat*dgamma/M) = k1 g + k2 y + k3
// (k1 = gamma*invstd, k2 = -k1*invstd*dgamma/M, k3 = k1*(mean*invstd*dgamma - dbeta)/M,
// formed once per CTA in shared memory), bf16; optionally also stores g (the masked
// incoming gradient, for the shortcut).
__global__ void __launch_bounds__(256) bn_bwd_apply_kernel(const uint16_t* __restrict__ gin, const uint16_t* __restrict__ mask,
                                    const uint16_t* __restrict__ y, const float* __restrict__ mean,
                                    const float* __restrict__ invstd, const float* __restrict__ gamma,
                                    const float* __restrict__ dgamma, const float* __restrict__ dbeta, int C,
                                    int64_t M, uint16_t* __restrict__ dy, uint16_t* __restrict__ g_out) {
  pdl_trigger_and_wait();
  extern __shared__ float tab[];  // [C] k1, [C] k2, [C] k3
  const float invM = 1.0f / (float)M;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const float is = invstd[c];
    const float k1 = gamma[c] * is;
    tab[c] = k1;
    tab[C + c] = -k1 * is * dgamma[c] * invM;
    tab[2 * C + c] = k1 * (mean[c] * is * dgamma[c] - dbeta[c]) * invM;
  }
  __syncthreads();
  const int cv = C / 8;
  const int64_t total = M * cv;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c0 = (int)(i & (int64_t)(cv - 1)) * 8;  // C is a power of two (64..2048)
    float g[8], yv[8], k1[8], k2[8], k3[8];
    unpack8(reinterpret_cast<const uint4*>(gin)[i], g);
    unpack8(reinterpret_cast<const uint4*>(y)[i], yv);
    if (mask) {
      float mv[8];
      unpack8(reinterpret_cast<const uint4*>(mask)[i], mv);
#pragma unroll
      for (int k = 0; k < 8; k++) g[k] = mv[k] > 0.0f ? g[k] : 0.0f;
    }
    coef8(tab, c0, k1);
    coef8(tab + C, c0, k2);
    coef8(tab + 2 * C, c0, k3);
    float d[8];
#pragma unroll
    for (int k = 0; k < 8; k++) d[k] = fmaf(k1[k], g[k], fmaf(k2[k], yv[k], k3[k]));
    reinterpret_cast<uint4*>(dy)[i] = pack8(d);
    if (g_out) reinterpret_cast<uint4*>(g_out)[i] = pack8(g);
  }
}

// head forward+backward, one CTA per sample: global average pool of the 4x4x512
// map, FC 512 -> C, softmax cross-entropy; writes dlogits/B, feat, the pooled-
// map gradient dOut = (dlogits W)/16, and the per-sample loss.
__global__ void __launch_bounds__(256) head_kernel(const uint16_t* __restrict__ a4, const float* __restrict__ Wfc,
                                                   const float* __restrict__ bfc, const int32_t* __restrict__ y_base,
                                                   const int64_t* __restrict__ iter, int64_t B, int classes,
                                                   float* __restrict__ feat, float* __restrict__ dlog,
                                                   float* __restrict__ loss_per, uint16_t* __restrict__ dout) {
  pdl_trigger_and_wait();
  __shared__ float f[512];
  __shared__ float logit[16];
  const int64_t n = blockIdx.x;
  const int64_t t = iter ? *iter : 0;
  const int32_t label = y_base[t * B + n];
  for (int c = threadIdx.x; c < 512; c += blockDim.x) {
    float s = 0.f;
    for (int p = 0; p < 16; p++) s += bf2f(a4[(n * 16 + p) * 512 + c]);
    f[c] = s * (1.0f / 16.0f);
    feat[n * 512 + c] = f[c];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = warp; k < classes; k += blockDim.x >> 5) {
    float s = 0.f;
    for (int c = lane; c < 512; c += 32) s = fmaf(f[c], Wfc[k * 512 + c], s);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) logit[k] = s + bfc[k];
  }
  __syncthreads();
  __shared__ float dl[16];
  if (threadIdx.x == 0) {
    float mx = -INFINITY;
    for (int k = 0; k < classes; k++) mx = fmaxf(mx, logit[k]);
    float se = 0.f;
    for (int k = 0; k < classes; k++) se += __expf(logit[k] - mx);
    loss_per[n] = (mx + __logf(se)) - logit[label];
    const float inv = 1.0f / se, invB = 1.0f / (float)B;
    for (int k = 0; k < classes; k++) {
      const float g = (__expf(logit[k] - mx) * inv - (k == label ? 1.f : 0.f)) * invB;
      dl[k] = g;
      dlog[n * 16 + k] = g;
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < 512; c += blockDim.x) {
    float s = 0.f;
    for (int k = 0; k < classes; k++) s = fmaf(dl[k], Wfc[k * 512 + c], s);
    const uint16_t h = f2bf(s * (1.0f / 16.0f));
    for (int p = 0; p < 16; p++) dout[(n * 16 + p) * 512 + c] = h;
  }
}

// dWfc[k][c] = sum_n dlog[n][k] feat[n][c], dbfc[k] = sum_n dlog[n][k]; loss mean
__global__ void head_wgrad_kernel(const float* __restrict__ feat, const float* __restrict__ dlog,
                                  const float* __restrict__ loss_per, int64_t B, int classes, float* __restrict__ dW,
                                  float* __restrict__ db, float* __restrict__ loss_out, const int64_t* __restrict__ iter) {
  pdl_trigger_and_wait();
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < classes * 512) {
    const int k = idx / 512, c = idx % 512;
    float s = 0.f;
    for (int64_t n = 0; n < B; n++) s = fmaf(dlog[n * 16 + k], feat[n * 512 + c], s);
    dW[idx] = s;
  }
  if (idx < classes) {
    float s = 0.f;
    for (int64_t n = 0; n < B; n++) s += dlog[n * 16 + idx];
    db[idx] = s;
  }
  if (idx == 0 && loss_out) {
    float s = 0.f;
    for (int64_t n = 0; n < B; n++) s += loss_per[n];
    loss_out[iter ? *iter : 0] = s / (float)B;
  }
}

__global__ void iter_inc_kernel(int64_t* it) { *it += 1; }

// ---------------------------- ResNet-50 kernels -----------------------------

// 7x7 / stride-2 / pad-3 stem im2col: x uint8 [B][3][S][S] (CHW per sample;
// pixel value (u - 128) / 64, exact in bf16) -> A bf16 [B*OS*OS][160],
// K = (r, s, c) with c fastest, columns 147..159 zero.  One CTA per output
// row: the 7 input rows it needs (x 3 channels, zero-padded to S + 6 columns)
// are staged once in shared memory as floats, a K -> offset table replaces the
// per-element index arithmetic, and consecutive threads write consecutive
// 16-byte chunks of the output rows.
__global__ void __launch_bounds__(256) im2col_stem7_kernel(const uint8_t* __restrict__ x_base,
                                                           const int64_t* __restrict__ iter, int64_t B, int S,
                                                           uint16_t* __restrict__ out) {
  pdl_trigger_and_wait();
  extern __shared__ float tile[];  // [3][7][S + 6]
  __shared__ int koff[kStem7K];
  constexpr int kChunks = kStem7K / 8;  // 20
  const int SP = S + 6, OS = S / 2;
  const int64_t t = iter ? *iter : 0;
  const int64_t plane = (int64_t)S * S;
  const int64_t n = blockIdx.x / OS;
  const int oh = (int)(blockIdx.x - n * OS);
  const uint8_t* xs = x_base + (t * B + n) * 3 * plane;
  for (int k = threadIdx.x; k < kStem7K; k += blockDim.x) {
    int o = -1;
    if (k < 147) {
      const int rs = k / 3, c = k - rs * 3;
      const int r = rs / 7, sx = rs - r * 7;
      o = (c * 7 + r) * SP + sx;
    }
    koff[k] = o;
  }
  for (int e = threadIdx.x; e < 3 * 7 * SP; e += blockDim.x) {
    const int c = e / (7 * SP), rem = e - c * 7 * SP;
    const int r = rem / SP, col = rem - r * SP;
    const int hh = 2 * oh + r - 3, ww = col - 3;
    float v = 0.0f;
    if (hh >= 0 && hh < S && ww >= 0 && ww < S) v = ((float)xs[c * plane + (int64_t)hh * S + ww] - 128.0f) * 0.015625f;
    tile[e] = v;
  }
  __syncthreads();
  uint4* o4 = reinterpret_cast<uint4*>(out) + (int64_t)blockIdx.x * OS * kChunks;
  for (int i = threadIdx.x; i < OS * kChunks; i += blockDim.x) {
    const int px = i / kChunks, ch = i - (i / kChunks) * kChunks;
    const float* base = tile + 2 * px;
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const int o = koff[ch * 8 + e];
      v[e] = o >= 0 ? base[o] : 0.0f;
    }
    o4[i] = make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]),
                       pack_bf16x2(v[6], v[7]));
  }
}

// 3x3 / stride-2 / pad-1 max-pool, NHWC bf16, 8 channels per thread; idx keeps
// the first maximal tap (row-major scan, as torch's max_pool2d) for backward
__global__ void maxpool_fwd_kernel(const uint16_t* __restrict__ in, int64_t B, int H, int W, int C, int OH, int OW,
                                   uint16_t* __restrict__ out, uint8_t* __restrict__ idx) {
  pdl_trigger_and_wait();
  const int cv = C / 8;
  const int64_t total = B * OH * OW * cv;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c8 = (int)(i % cv);
    const int64_t pix = i / cv;
    const int ow = (int)(pix % OW);
    const int oh = (int)((pix / OW) % OH);
    const int64_t n = pix / ((int64_t)OW * OH);
    float best[8];
    uint8_t arg[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
      best[k] = -INFINITY;
      arg[k] = 0;
    }
    for (int r = 0; r < 3; r++) {
      const int h = 2 * oh + r - 1;
      if (h < 0 || h >= H) continue;
      for (int s = 0; s < 3; s++) {
        const int w = 2 * ow + s - 1;
        if (w < 0 || w >= W) continue;
        const uint4 q = reinterpret_cast<const uint4*>(in + ((n * H + h) * W + w) * C)[c8];
        const uint32_t wv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int k = 0; k < 8; k++) {
          const float v = bf2f((uint16_t)(wv[k >> 1] >> ((k & 1) * 16)));
          if (v > best[k]) {
            best[k] = v;
            arg[k] = (uint8_t)(r * 3 + s);
          }
        }
      }
    }
    uint32_t o[4] = {0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < 8; k++) o[k >> 1] |= (uint32_t)f2bf(best[k]) << ((k & 1) * 16);
    reinterpret_cast<uint4*>(out)[i] = make_uint4(o[0], o[1], o[2], o[3]);
    uint2 a;
    a.x = arg[0] | (arg[1] << 8) | (arg[2] << 16) | ((uint32_t)arg[3] << 24);
    a.y = arg[4] | (arg[5] << 8) | (arg[6] << 16) | ((uint32_t)arg[7] << 24);
    reinterpret_cast<uint2*>(idx)[i] = a;
  }
}

// max-pool backward in gather form (no atomics): input pixel (h, w) collects
// the gradient of every window (<= 2 x 2) whose recorded maximum it is
__global__ void maxpool_bwd_kernel(const uint16_t* __restrict__ gout, const uint8_t* __restrict__ idx, int64_t B,
                                   int H, int W, int C, int OH, int OW, uint16_t* __restrict__ gin) {
  pdl_trigger_and_wait();
  const int cv = C / 8;
  const int64_t total = B * H * W * cv;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c8 = (int)(i % cv);
    const int64_t pix = i / cv;
    const int w = (int)(pix % W);
    const int h = (int)((pix / W) % H);
    const int64_t n = pix / ((int64_t)W * H);
    float acc[8];
#pragma unroll
    for (int k = 0; k < 8; k++) acc[k] = 0.f;
    for (int oh = (h > 0 ? h : 1) / 2; oh <= (h + 1) / 2 && oh < OH; oh++) {
      const int r = h - (2 * oh - 1);
      if (r < 0 || r > 2) continue;
      for (int ow = (w > 0 ? w : 1) / 2; ow <= (w + 1) / 2 && ow < OW; ow++) {
        const int s = w - (2 * ow - 1);
        if (s < 0 || s > 2) continue;
        const int64_t o = ((n * OH + oh) * OW + ow) * cv + c8;
        const uint2 a = reinterpret_cast<const uint2*>(idx)[o];
        const uint4 q = reinterpret_cast<const uint4*>(gout)[o];
        const uint32_t gv[4] = {q.x, q.y, q.z, q.w};
        const uint32_t av[2] = {a.x, a.y};
        const uint32_t tap = (uint32_t)(r * 3 + s);
#pragma unroll
        for (int k = 0; k < 8; k++)
          if (((av[k >> 2] >> ((k & 3) * 8)) & 0xFFu) == tap) acc[k] += bf2f((uint16_t)(gv[k >> 1] >> ((k & 1) * 16)));
      }
    }
    uint32_t o[4] = {0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < 8; k++) o[k >> 1] |= (uint32_t)f2bf(acc[k]) << ((k & 1) * 16);
    reinterpret_cast<uint4*>(gin)[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// global average pool: x bf16 [B][HW][C] -> feat bf16 [B][C] (the FC GEMM operand)
__global__ void avgpool_kernel(const uint16_t* __restrict__ x, int64_t B, int HW, int C, uint16_t* __restrict__ feat) {
  pdl_trigger_and_wait();
  const int cv = C / 8;
  const int64_t total = B * cv;
  const float inv = 1.0f / (float)HW;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = i / cv;
    const int c8 = (int)(i - n * cv);
    float acc[8];
#pragma unroll
    for (int k = 0; k < 8; k++) acc[k] = 0.f;
    for (int p = 0; p < HW; p++) {
      const uint4 q = reinterpret_cast<const uint4*>(x + (n * HW + p) * C)[c8];
      const uint32_t wv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int k = 0; k < 8; k++) acc[k] += bf2f((uint16_t)(wv[k >> 1] >> ((k & 1) * 16)));
    }
    uint32_t o[4] = {0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < 8; k++) o[k >> 1] |= (uint32_t)f2bf(acc[k] * inv) << ((k & 1) * 16);
    reinterpret_cast<uint4*>(feat)[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

__device__ __forceinline__ float block_reduce(float v, float* sh, bool is_max) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    const float u = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmaxf(v, u) : v + u;
  }
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  float r = sh[0];
  for (int w = 1; w < nw; w++) r = is_max ? fmaxf(r, sh[w]) : r + sh[w];
  return r;
}

// softmax cross-entropy, one CTA per sample: logits fp32 [B][ld] -> per-sample
// loss, dlogits / B in fp32 (bias gradient) and bf16 (GEMM operand, padding
// columns zeroed)
__global__ void __launch_bounds__(256) ce_kernel(const float* __restrict__ logits, int ld,
                                                 const int32_t* __restrict__ y_base, const int64_t* __restrict__ iter,
                                                 int64_t B, int classes, float* __restrict__ dlog_f,
                                                 uint16_t* __restrict__ dlog_b, float* __restrict__ loss_per) {
  pdl_trigger_and_wait();
  __shared__ float sh[32];
  const int64_t n = blockIdx.x;
  const int64_t t = iter ? *iter : 0;
  const int32_t label = y_base[t * B + n];
  const float* z = logits + n * ld;
  float mx = -INFINITY;
  for (int k = threadIdx.x; k < classes; k += blockDim.x) mx = fmaxf(mx, z[k]);
  mx = block_reduce(mx, sh, true);
  float se = 0.f;
  for (int k = threadIdx.x; k < classes; k += blockDim.x) se += __expf(z[k] - mx);
  se = block_reduce(se, sh, false);
  const float inv = 1.0f / se, invB = 1.0f / (float)B;
  for (int k = threadIdx.x; k < ld; k += blockDim.x) {
    float g = 0.f;
    if (k < classes) g = (__expf(z[k] - mx) * inv - (k == label ? 1.f : 0.f)) * invB;
    dlog_f[n * ld + k] = g;
    dlog_b[n * ld + k] = f2bf(g);
  }
  if (threadIdx.x == 0) loss_per[n] = (mx + __logf(se)) - z[label];
}

// FC bias gradient (column sums of dlogits) and the batch-mean loss
__global__ void head_bias_kernel(const float* __restrict__ dlog_f, int ld, const float* __restrict__ loss_per,
                                 int64_t B, int classes, float* __restrict__ db, float* __restrict__ loss_out,
                                 const int64_t* __restrict__ iter) {
  pdl_trigger_and_wait();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < classes) {
    float s = 0.f;
    for (int64_t n = 0; n < B; n++) s += dlog_f[n * ld + k];
    db[k] = s;
  }
  if (k == 0 && loss_out) {
    float s = 0.f;
    for (int64_t n = 0; n < B; n++) s += loss_per[n];
    loss_out[iter ? *iter : 0] = s / (float)B;
  }
}

// gradient of the average pool: dOut[n][p][c] = dfeat[n][c] / HW (bf16)
__global__ void head_bcast_kernel(const float* __restrict__ dfeat, int64_t B, int HW, int C,
                                  uint16_t* __restrict__ dout) {
  pdl_trigger_and_wait();
  const int cv = C / 8;
  const int64_t total = B * HW * cv;
  const float inv = 1.0f / (float)HW;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c8 = (int)(i % cv);
    const int64_t n = i / ((int64_t)cv * HW);
    const float4 a = reinterpret_cast<const float4*>(dfeat + n * C + c8 * 8)[0];
    const float4 b = reinterpret_cast<const float4*>(dfeat + n * C + c8 * 8)[1];
    const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    uint32_t o[4] = {0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < 8; k++) o[k >> 1] |= (uint32_t)f2bf(v[k] * inv) << ((k & 1) * 16);
    reinterpret_cast<uint4*>(dout)[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// ======================= fp32-class (DBS_PREC_F32) kernels =======================
// Storage in this mode: conv outputs y, input gradients and the incoming BN-backward
// gradients plain fp32; every GEMM operand (post-BN activations, block outputs,
// BN-backward outputs dY, the stem's im2col columns, pooled features, dlogits) in
// the S32 format of the 3xTF32 GEMM (s32.cu): flat element e of a tensor whose
// rows are multiples of 32 sits at 2 (e & ~31) + (e & 31) (hi), +32 (lo).
__device__ __forceinline__ float rn_tf32(float x) {
  const uint32_t u = __float_as_uint(x);
  return __uint_as_float((u + 0xFFFu + ((u >> 13) & 1u)) & 0xFFFFE000u);
}
__device__ __forceinline__ int64_t s32_off(int64_t e) { return 2 * (e & ~int64_t(31)) + (e & 31); }
// elements 8 i .. 8 i + 7
// 256-bit global accesses (LDG/STG.256, sm_100): one instruction per 8 floats
__device__ __forceinline__ void ldg8f(const float* q, float (&v)[8]) {
  asm volatile("ld.global.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
               : "l"(q));
}
__device__ __forceinline__ void stg8f(float* q, const float (&v)[8]) {
  asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(q), "f"(v[0]), "f"(v[1]), "f"(v[2]),
               "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}
__device__ __forceinline__ void ld8_f32(const float* p, int64_t i, float (&v)[8]) { ldg8f(p + 8 * i, v); }
__device__ __forceinline__ void st8_f32(float* p, int64_t i, const float (&v)[8]) { stg8f(p + 8 * i, v); }
__device__ __forceinline__ void ld8_s32(const float* p, int64_t i, float (&v)[8]) {
  const float* q = p + s32_off(8 * i);
  float l[8];
  ldg8f(q, v);
  ldg8f(q + 32, l);
#pragma unroll
  for (int k = 0; k < 8; k++) v[k] += l[k];
}
__device__ __forceinline__ void ld8_s32_hi(const float* p, int64_t i, float (&v)[8]) { ldg8f(p + s32_off(8 * i), v); }
__device__ __forceinline__ void st8_s32(float* p, int64_t i, const float (&v)[8]) {
  float* q = p + s32_off(8 * i);
  float h[8], l[8];
#pragma unroll
  for (int k = 0; k < 8; k++) {
    h[k] = rn_tf32(v[k]);
    l[k] = rn_tf32(v[k] - h[k]);
  }
  stg8f(q, h);
  stg8f(q + 32, l);
}
__device__ __forceinline__ void st1_s32(float* p, int64_t e, float v) {
  const float h = rn_tf32(v);
  p[s32_off(e)] = h;
  p[s32_off(e) + 32] = rn_tf32(v - h);
}

// ResNet-18 stem im2col, S32 columns [B*1024][32] (K = (r, s, c), 27 used)
__global__ void im2col_stem_f32_kernel(const float* __restrict__ x_base, const int64_t* __restrict__ iter, int64_t B,
                                       float* __restrict__ out) {
  pdl_trigger_and_wait();
  const int64_t t = iter ? *iter : 0;
  const float* x = x_base + t * B * 3072;
  const int64_t total = B * 1024;
  for (int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pix < total;
       pix += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = pix >> 10;
    const int h = (int)((pix >> 5) & 31), w = (int)(pix & 31);
    const float* xs = x + n * 3072;
    float v[32];
#pragma unroll
    for (int k = 0; k < 32; k++) v[k] = 0.0f;
#pragma unroll
    for (int r = 0; r < 3; r++)
#pragma unroll
      for (int s = 0; s < 3; s++)
#pragma unroll
        for (int c = 0; c < 3; c++) {
          const int hh = h + r - 1, ww = w + s - 1;
          v[(r * 3 + s) * 3 + c] = (hh >= 0 && hh < 32 && ww >= 0 && ww < 32) ? xs[c * 1024 + hh * 32 + ww] : 0.0f;
        }
#pragma unroll
    for (int q = 0; q < 4; q++) {
      float u[8];
#pragma unroll
      for (int k = 0; k < 8; k++) u[k] = v[8 * q + k];
      st8_s32(out, pix * 4 + q, u);
    }
  }
}

// ResNet-50 stem im2col (7x7 / 2 / 3), S32 columns [B*OS*OS][160]
__global__ void __launch_bounds__(256) im2col_stem7_f32_kernel(const uint8_t* __restrict__ x_base,
                                                               const int64_t* __restrict__ iter, int64_t B, int S,
                                                               float* __restrict__ out) {
  pdl_trigger_and_wait();
  extern __shared__ float tile[];  // [3][7][S + 6]
  __shared__ int koff[kStem7K];
  constexpr int kChunks = kStem7K / 8;
  const int SP = S + 6, OS = S / 2;
  const int64_t t = iter ? *iter : 0;
  const int64_t plane = (int64_t)S * S;
  const int64_t n = blockIdx.x / OS;
  const int oh = (int)(blockIdx.x - n * OS);
  const uint8_t* xs = x_base + (t * B + n) * 3 * plane;
  for (int k = threadIdx.x; k < kStem7K; k += blockDim.x) {
    int o = -1;
    if (k < 147) {
      const int rs = k / 3, c = k - rs * 3;
      const int r = rs / 7, sx = rs - r * 7;
      o = (c * 7 + r) * SP + sx;
    }
    koff[k] = o;
  }
  for (int e = threadIdx.x; e < 3 * 7 * SP; e += blockDim.x) {
    const int c = e / (7 * SP), rem = e - c * 7 * SP;
    const int r = rem / SP, col = rem - r * SP;
    const int hh = 2 * oh + r - 3, ww = col - 3;
    float v = 0.0f;
    if (hh >= 0 && hh < S && ww >= 0 && ww < S) v = ((float)xs[c * plane + (int64_t)hh * S + ww] - 128.0f) * 0.015625f;
    tile[e] = v;
  }
  __syncthreads();
  const int64_t row0 = (int64_t)blockIdx.x * OS;
  for (int i = threadIdx.x; i < OS * kChunks; i += blockDim.x) {
    const int px = i / kChunks, ch = i - (i / kChunks) * kChunks;
    const float* base = tile + 2 * px;
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const int o = koff[ch * 8 + e];
      v[e] = o >= 0 ? base[o] : 0.0f;
    }
    st8_s32(out, (row0 + px) * kChunks + ch, v);
  }
}

// out (S32) = act(a*y + b [+ res (S32) | + a_d*yd + b_d]), y / yd fp32; also the
// running statistics (momentum `rm`, unbiased variance, as torch's BatchNorm2d)
__global__ void __launch_bounds__(256) bn_apply_f32_kernel(
    const float* __restrict__ y, const double* __restrict__ acc, float* __restrict__ mean, float* __restrict__ invstd,
    const float* __restrict__ gamma, const float* __restrict__ beta, const float* __restrict__ res,
    const float* __restrict__ yd, const double* __restrict__ acc_d, float* __restrict__ mean_d,
    float* __restrict__ invstd_d, const float* __restrict__ gamma_d, const float* __restrict__ beta_d, int relu, int C,
    int64_t M, float* __restrict__ out, float* __restrict__ run, float* __restrict__ run_d, float rm) {
  pdl_trigger_and_wait();
  extern __shared__ float tab[];
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float mu, is;
    bn_finalise(acc, C, c, M, mu, is);
    const float a = gamma[c] * is;
    tab[c] = a;
    tab[C + c] = beta[c] - mu * a;
    if (blockIdx.x == 0) {
      mean[c] = mu;
      invstd[c] = is;
      if (run) {
        const double mud = acc[c] / (double)M, var = fmax(acc[C + c] / (double)M - mud * mud, 0.0);
        run[c] = (1.0f - rm) * run[c] + rm * mu;
        run[C + c] = (1.0f - rm) * run[C + c] + rm * (float)(var * (double)M / (double)(M > 1 ? M - 1 : 1));
      }
    }
    if (yd) {
      float mud, isd;
      bn_finalise(acc_d, C, c, M, mud, isd);
      const float ad = gamma_d[c] * isd;
      tab[2 * C + c] = ad;
      tab[3 * C + c] = beta_d[c] - mud * ad;
      if (blockIdx.x == 0) {
        mean_d[c] = mud;
        invstd_d[c] = isd;
        if (run_d) {
          const double m2 = acc_d[c] / (double)M, var = fmax(acc_d[C + c] / (double)M - m2 * m2, 0.0);
          run_d[c] = (1.0f - rm) * run_d[c] + rm * mud;
          run_d[C + c] = (1.0f - rm) * run_d[C + c] + rm * (float)(var * (double)M / (double)(M > 1 ? M - 1 : 1));
        }
      }
    }
  }
  __syncthreads();
  const int cv = C / 8;
  const int64_t total = M * cv;
  auto finish = [&](int64_t i, float (&v)[8]) {
    const int c0 = (int)(i & (int64_t)(cv - 1)) * 8;
    float ka[8], kb[8];
    coef8(tab, c0, ka);
    coef8(tab + C, c0, kb);
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] = fmaf(ka[k], v[k], kb[k]);
    if (res) {
      float r[8];
      ld8_s32(res, i, r);
#pragma unroll
      for (int k = 0; k < 8; k++) v[k] += r[k];
    }
    if (yd) {
      float r[8];
      ld8_f32(yd, i, r);
      coef8(tab + 2 * C, c0, ka);
      coef8(tab + 3 * C, c0, kb);
#pragma unroll
      for (int k = 0; k < 8; k++) v[k] += fmaf(ka[k], r[k], kb[k]);
    }
    if (relu) {
#pragma unroll
      for (int k = 0; k < 8; k++) v[k] = fmaxf(v[k], 0.0f);
    }
    st8_s32(out, i, v);
  };
  // two 8-element groups per trip, both loads issued before either is used (the
  // one-group loop left too few bytes in flight: 0.57 of the partition's copy rate)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + stride < total; i += 2 * stride) {
    float v0[8], v1[8];
    ld8_f32(y, i, v0);
    ld8_f32(y, i + stride, v1);
    finish(i, v0);
    finish(i + stride, v1);
  }
  if (i < total) {
    float v0[8];
    ld8_f32(y, i, v0);
    finish(i, v0);
  }
}

// BN backward pass 1 (fp32 gradient / y, S32 ReLU mask): dbeta += sum g, dgamma += sum g yhat
__global__ void __launch_bounds__(256) bn_bwd_reduce_f32_kernel(const float* __restrict__ gin,
                                                                const float* __restrict__ mask,
                                                                const float* __restrict__ y,
                                                                const float* __restrict__ mean,
                                                                const float* __restrict__ invstd, int C, int64_t M,
                                                                float* __restrict__ dgamma, float* __restrict__ dbeta) {
  pdl_trigger_and_wait();
  __shared__ float red_g[2048], red_b[2048];
  const int cv = C / 8;
  const int rows_per_pass = blockDim.x / cv;
  const int lane_c = threadIdx.x % cv, lane_r = threadIdx.x / cv;
  float sg[8], sb[8], mu[8], is[8];
  const int c0 = lane_c * 8;
#pragma unroll
  for (int k = 0; k < 8; k++) {
    sg[k] = 0.f;
    sb[k] = 0.f;
    mu[k] = mean[c0 + k];
    is[k] = invstd[c0 + k];
  }
  if (lane_r < rows_per_pass) {
    const int64_t step = (int64_t)gridDim.x * rows_per_pass;
    for (int64_t r = (int64_t)blockIdx.x * rows_per_pass + lane_r; r < M; r += step) {
      const int64_t i = r * cv + lane_c;
      float g[8], yv[8], mv[8];
      ld8_f32(gin, i, g);
      ld8_f32(y, i, yv);
      if (mask) ld8_s32_hi(mask, i, mv);
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const float gg = (!mask || mv[k] > 0.0f) ? g[k] : 0.0f;
        sb[k] += gg;
        sg[k] = fmaf(gg, (yv[k] - mu[k]) * is[k], sg[k]);
      }
    }
  }
  if (cv < 32) {
#pragma unroll
    for (int k = 0; k < 8; k++) {
      for (int o = cv; o < 32; o <<= 1) {
        sg[k] += __shfl_xor_sync(0xffffffffu, sg[k], o);
        sb[k] += __shfl_xor_sync(0xffffffffu, sb[k], o);
      }
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const bool writer = (cv < 32) ? (lane < cv) : (lane_r < rows_per_pass);
  const int slot = (cv < 32) ? warp : lane_r;
  const int nslot = (cv < 32) ? nw : rows_per_pass;
  if (writer) {
#pragma unroll
    for (int k = 0; k < 8; k++) {
      red_g[slot * C + c0 + k] = sg[k];
      red_b[slot * C + c0 + k] = sb[k];
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < C; idx += blockDim.x) {
    float a = 0.f, b = 0.f;
    for (int r = 0; r < nslot; r++) {
      a += red_g[r * C + idx];
      b += red_b[r * C + idx];
    }
    atomicAdd(&dgamma[idx], a);
    atomicAdd(&dbeta[idx], b);
  }
}

// BN backward pass 2: dy (S32) = k1 g + k2 y + k3; g_out (fp32) = the masked gradient
__global__ void __launch_bounds__(256) bn_bwd_apply_f32_kernel(const float* __restrict__ gin,
                                                               const float* __restrict__ mask,
                                                               const float* __restrict__ y, const float* __restrict__ mean,
                                                               const float* __restrict__ invstd,
                                                               const float* __restrict__ gamma,
                                                               const float* __restrict__ dgamma,
                                                               const float* __restrict__ dbeta, int C, int64_t M,
                                                               float* __restrict__ dy, float* __restrict__ g_out) {
  pdl_trigger_and_wait();
  extern __shared__ float tab[];
  const float invM = 1.0f / (float)M;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const float is = invstd[c];
    const float k1 = gamma[c] * is;
    tab[c] = k1;
    tab[C + c] = -k1 * is * dgamma[c] * invM;
    tab[2 * C + c] = k1 * (mean[c] * is * dgamma[c] - dbeta[c]) * invM;
  }
  __syncthreads();
  const int cv = C / 8;
  const int64_t total = M * cv;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c0 = (int)(i & (int64_t)(cv - 1)) * 8;
    float g[8], yv[8], k1[8], k2[8], k3[8];
    ld8_f32(gin, i, g);
    ld8_f32(y, i, yv);
    if (mask) {
      float mv[8];
      ld8_s32_hi(mask, i, mv);
#pragma unroll
      for (int k = 0; k < 8; k++) g[k] = mv[k] > 0.0f ? g[k] : 0.0f;
    }
    coef8(tab, c0, k1);
    coef8(tab + C, c0, k2);
    coef8(tab + 2 * C, c0, k3);
    float d[8];
#pragma unroll
    for (int k = 0; k < 8; k++) d[k] = fmaf(k1[k], g[k], fmaf(k2[k], yv[k], k3[k]));
    st8_s32(dy, i, d);
    if (g_out) st8_f32(g_out, i, g);
  }
}

// ResNet-18 head (f32 storage): a4 S32 [B][16][512] -> feat, logits, loss, dlogits / B,
// dOut (fp32) = (dlogits W) / 16
__global__ void __launch_bounds__(256) head_f32_kernel(const float* __restrict__ a4, const float* __restrict__ Wfc,
                                                       const float* __restrict__ bfc, const int32_t* __restrict__ y_base,
                                                       const int64_t* __restrict__ iter, int64_t B, int classes,
                                                       float* __restrict__ feat, float* __restrict__ dlog,
                                                       float* __restrict__ loss_per, float* __restrict__ dout) {
  pdl_trigger_and_wait();
  __shared__ float f[512];
  __shared__ float logit[16];
  const int64_t n = blockIdx.x;
  const int64_t t = iter ? *iter : 0;
  const int32_t label = y_base[t * B + n];
  for (int c = threadIdx.x; c < 512; c += blockDim.x) {
    float s = 0.f;
    for (int p = 0; p < 16; p++) {
      const int64_t o = s32_off((n * 16 + p) * 512 + c);
      s += a4[o] + a4[o + 32];
    }
    f[c] = s * (1.0f / 16.0f);
    feat[n * 512 + c] = f[c];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = warp; k < classes; k += blockDim.x >> 5) {
    float s = 0.f;
    for (int c = lane; c < 512; c += 32) s = fmaf(f[c], Wfc[k * 512 + c], s);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) logit[k] = s + bfc[k];
  }
  __syncthreads();
  __shared__ float dl[16];
  if (threadIdx.x == 0) {
    float mx = -INFINITY;
    for (int k = 0; k < classes; k++) mx = fmaxf(mx, logit[k]);
    float se = 0.f;
    for (int k = 0; k < classes; k++) se += expf(logit[k] - mx);
    loss_per[n] = (mx + logf(se)) - logit[label];
    const float inv = 1.0f / se, invB = 1.0f / (float)B;
    for (int k = 0; k < classes; k++) {
      const float g = (expf(logit[k] - mx) * inv - (k == label ? 1.f : 0.f)) * invB;
      dl[k] = g;
      dlog[n * 16 + k] = g;
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < 512; c += blockDim.x) {
    float s = 0.f;
    for (int k = 0; k < classes; k++) s = fmaf(dl[k], Wfc[k * 512 + c], s);
    const float h = s * (1.0f / 16.0f);
    for (int p = 0; p < 16; p++) dout[(n * 16 + p) * 512 + c] = h;
  }
}

// 3x3 / 2 / 1 max-pool on S32 (first maximal tap, row-major scan) and its backward (fp32)
__global__ void maxpool_fwd_f32_kernel(const float* __restrict__ in, int64_t B, int H, int W, int C, int OH, int OW,
                                       float* __restrict__ out, uint8_t* __restrict__ idx) {
  pdl_trigger_and_wait();
  const int cv = C / 8;
  const int64_t total = B * OH * OW * cv;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c8 = (int)(i % cv);
    const int64_t pix = i / cv;
    const int ow = (int)(pix % OW);
    const int oh = (int)((pix / OW) % OH);
    const int64_t n = pix / ((int64_t)OW * OH);
    float best[8];
    uint8_t arg[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
      best[k] = -INFINITY;
      arg[k] = 0;
    }
    for (int r = 0; r < 3; r++) {
      const int h = 2 * oh + r - 1;
      if (h < 0 || h >= H) continue;
      for (int s = 0; s < 3; s++) {
        const int w = 2 * ow + s - 1;
        if (w < 0 || w >= W) continue;
        float v[8];
        ld8_s32(in, ((n * H + h) * W + w) * cv + c8, v);
#pragma unroll
        for (int k = 0; k < 8; k++) {
          if (v[k] > best[k]) {
            best[k] = v[k];
            arg[k] = (uint8_t)(r * 3 + s);
          }
        }
      }
    }
    st8_s32(out, i, best);
    uint2 a;
    a.x = arg[0] | (arg[1] << 8) | (arg[2] << 16) | ((uint32_t)arg[3] << 24);
    a.y = arg[4] | (arg[5] << 8) | (arg[6] << 16) | ((uint32_t)arg[7] << 24);
    reinterpret_cast<uint2*>(idx)[i] = a;
  }
}

__global__ void maxpool_bwd_f32_kernel(const float* __restrict__ gout, const uint8_t* __restrict__ idx, int64_t B,
                                       int H, int W, int C, int OH, int OW, float* __restrict__ gin) {
  pdl_trigger_and_wait();
  const int cv = C / 8;
  const int64_t total = B * H * W * cv;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c8 = (int)(i % cv);
    const int64_t pix = i / cv;
    const int w = (int)(pix % W);
    const int h = (int)((pix / W) % H);
    const int64_t n = pix / ((int64_t)W * H);
    float acc[8];
#pragma unroll
    for (int k = 0; k < 8; k++) acc[k] = 0.f;
    for (int oh = (h > 0 ? h : 1) / 2; oh <= (h + 1) / 2 && oh < OH; oh++) {
      const int r = h - (2 * oh - 1);
      if (r < 0 || r > 2) continue;
      for (int ow = (w > 0 ? w : 1) / 2; ow <= (w + 1) / 2 && ow < OW; ow++) {
        const int s = w - (2 * ow - 1);
        if (s < 0 || s > 2) continue;
        const int64_t o = ((n * OH + oh) * OW + ow) * cv + c8;
        const uint2 a = reinterpret_cast<const uint2*>(idx)[o];
        float g[8];
        ld8_f32(gout, o, g);
        const uint32_t av[2] = {a.x, a.y};
        const uint32_t tap = (uint32_t)(r * 3 + s);
#pragma unroll
        for (int k = 0; k < 8; k++)
          if (((av[k >> 2] >> ((k & 3) * 8)) & 0xFFu) == tap) acc[k] += g[k];
      }
    }
    st8_f32(gin, i, acc);
  }
}

// global average pool S32 [B][HW][C] -> S32 [B][C]
__global__ void avgpool_f32_kernel(const float* __restrict__ x, int64_t B, int HW, int C, float* __restrict__ feat) {
  pdl_trigger_and_wait();
  const int cv = C / 8;
  const int64_t total = B * cv;
  const float inv = 1.0f / (float)HW;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = i / cv;
    const int c8 = (int)(i - n * cv);
    float acc[8];
#pragma unroll
    for (int k = 0; k < 8; k++) acc[k] = 0.f;
    for (int p = 0; p < HW; p++) {
      float v[8];
      ld8_s32(x, (n * HW + p) * cv + c8, v);
#pragma unroll
      for (int k = 0; k < 8; k++) acc[k] += v[k];
    }
#pragma unroll
    for (int k = 0; k < 8; k++) acc[k] *= inv;
    st8_s32(feat, i, acc);
  }
}

// softmax cross-entropy (f32 storage): dlog_b S32 [B][ld32], pad columns zero
__global__ void __launch_bounds__(256) ce_f32_kernel(const float* __restrict__ logits, int ld,
                                                     const int32_t* __restrict__ y_base, const int64_t* __restrict__ iter,
                                                     int64_t B, int classes, float* __restrict__ dlog_f,
                                                     float* __restrict__ dlog_b, int ld32, float* __restrict__ loss_per) {
  pdl_trigger_and_wait();
  __shared__ float sh[32];
  const int64_t n = blockIdx.x;
  const int64_t t = iter ? *iter : 0;
  const int32_t label = y_base[t * B + n];
  const float* z = logits + n * ld;
  float mx = -INFINITY;
  for (int k = threadIdx.x; k < classes; k += blockDim.x) mx = fmaxf(mx, z[k]);
  mx = block_reduce(mx, sh, true);
  float se = 0.f;
  for (int k = threadIdx.x; k < classes; k += blockDim.x) se += expf(z[k] - mx);
  se = block_reduce(se, sh, false);
  const float inv = 1.0f / se, invB = 1.0f / (float)B;
  for (int k = threadIdx.x; k < ld32; k += blockDim.x) {
    float g = 0.f;
    if (k < classes) g = (expf(z[k] - mx) * inv - (k == label ? 1.f : 0.f)) * invB;
    if (k < ld) dlog_f[n * ld + k] = g;
    st1_s32(dlog_b, n * ld32 + k, g);
  }
  if (threadIdx.x == 0) loss_per[n] = (mx + logf(se)) - z[label];
}

// gradient of the average pool: dOut[n][p][c] = dfeat[n][c] / HW (fp32)
__global__ void head_bcast_f32_kernel(const float* __restrict__ dfeat, int64_t B, int HW, int C,
                                      float* __restrict__ dout) {
  pdl_trigger_and_wait();
  const int cv = C / 8;
  const int64_t total = B * HW * cv;
  const float inv = 1.0f / (float)HW;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c8 = (int)(i % cv);
    const int64_t n = i / ((int64_t)cv * HW);
    float v[8];
    ld8_f32(dfeat + n * C, c8, v);
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] *= inv;
    st8_f32(dout, i, v);
  }
}

// CTAs of `kernel` one SM holds at once (registers / shared memory), cached per
// (kernel, block size, dynamic shared memory)
template <typename K>
int resident_per_sm(K kernel, int threads, size_t smem) {
  struct Entry {
    const void* fn;
    int threads;
    size_t smem;
    int v;
  };
  static std::mutex mu;
  static std::vector<Entry> cache;
  const void* fn = reinterpret_cast<const void*>(kernel);
  std::lock_guard<std::mutex> lk(mu);
  for (const Entry& e : cache)
    if (e.fn == fn && e.threads == threads && e.smem == smem) return e.v;
  int v = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kernel, threads, smem) != cudaSuccess || v < 1) v = 1;
  cache.push_back(Entry{fn, threads, smem, v});
  return v;
}

// grid-stride kernels: at most ONE wave of resident CTAs on the SMs this launch can use
// (the BN kernels hold 3-6 CTAs per SM, not 8: a fixed 8-per-SM grid left a partial
// second / third wave)
template <typename K>
int grid_one_wave(K kernel, int64_t n, int threads, size_t smem) {
  int64_t b = (n + threads - 1) / threads;
  int64_t cap = (int64_t)current_sm_count() * resident_per_sm(kernel, threads, smem);
  return (int)(b < 1 ? 1 : (b < cap ? b : cap));
}

}  // namespace
}  // namespace dbs

using namespace dbs;

struct dbs_resnet {
  int64_t max_b = 0;
  int classes = 10;
  int arch = 18;                           // 18 (CIFAR stem) or 50 (ImageNet stem)
  int image = 32;                          // input side (32 for ResNet-18; 224 for config 5)
  int prec = DBS_PREC_BF16;                // DBS_PREC_F32: 3xTF32 GEMMs on S32 operands, fp32 storage
  int64_t row_bytes = 3072 * 4;            // one input sample in the repacked shard
  int stem_k = kStemK;                     // padded K of the stem's explicit im2col
  int feat_c = 512, feat_hw = 16;          // last feature map: channels, pixels
  int cpad = 16;                           // logits / dlogits row pitch (ResNet-50 head)
  int cpad32 = 32;                         // S32 dlogits row pitch (f32 mode)
  std::vector<char> need_a;                // per conv: post-BN(+ReLU) output is stored
  // Buffers are typed by precision: "operand" tensors (a, blk_out, stem_cols, mp_out,
  // feat_b, dlog_b, BN-backward outputs) bf16 or S32; y and input gradients bf16 or fp32.
  // ResNet-50 extras
  void* mp_out = nullptr;                  // max-pool output [B][S/4][S/4][64]
  uint8_t* mp_idx = nullptr;               // its arg-max taps
  void* feat_b = nullptr;                  // pooled features [B][2048]
  float* logits = nullptr;                 // [B][cpad]
  float* dlog_f = nullptr;                 // [B][cpad]
  void* dlog_b = nullptr;                  // [B][cpad] bf16 | [B][cpad32] S32
  float* dfeat = nullptr;                  // [B][2048]
  void* g4 = nullptr;
  std::vector<Conv> convs;
  std::vector<Block> blocks;
  int stem = 0;
  int64_t fc_w = 0, fc_b = 0, P = 0;
  // parameter table (torchvision order): offset, length, kind (0 conv w, 1 bn g, 2 bn b, 3 fc w, 4 fc b)
  std::vector<int64_t> t_off, t_len;
  std::vector<int32_t> t_kind;
  // activations
  void* stem_cols = nullptr;               // [B*OH*OW][stem_k]
  std::vector<void*> y, a;                 // per conv: pre-BN output, post-BN(+ReLU) output
  std::vector<void*> blk_out;              // per block output (post residual ReLU)
  std::vector<float*> mean, invstd;        // per conv
  double* stats_acc = nullptr;             // per conv: [cout] fp64 sums + [cout] sums of squares (BN statistics)
  std::vector<int64_t> stats_off;          // offset of each conv's accumulators in stats_acc
  int64_t stats_len = 0;
  // BN running statistics (f32 mode): per conv [cout] mean + [cout] unbiased variance,
  // momentum bn_momentum (torch BatchNorm2d semantics), per worker
  float* run_stats = nullptr;
  std::vector<int64_t> run_off;
  float bn_momentum = 0.1f;
  void* g0 = nullptr;                      // gradient ping-pong buffers (largest activation)
  void* g1 = nullptr;
  void* g2 = nullptr;
  void* g3 = nullptr;
  float* feat = nullptr;                   // [B][512]
  float* dlog = nullptr;                   // [B][16]
  float* loss_per = nullptr;               // [B]
  float* loss_scratch = nullptr;
};

namespace {

// every parameter tensor starts on a 32-element boundary: the flat S32 operand
// shadow of the fp32-class path is then the same layout (rows are multiples of 32)
int64_t pad8(int64_t x) { return (x + 31) & ~int64_t(31); }

void build_layers(dbs_resnet* m) {
  int64_t off = 0;
  auto add_param = [&](int64_t len, int kind) {
    const int64_t o = off;
    m->t_off.push_back(o);
    m->t_len.push_back(len);
    m->t_kind.push_back(kind);
    off += pad8(len);
    return o;
  };
  auto add_conv = [&](int cin, int cout, int k, int stride, int pad, int H, int W) {
    Conv c{};
    c.cin = cin;
    c.cout = cout;
    c.k = k;
    c.stride = stride;
    c.pad = pad;
    c.H = H;
    c.W = W;
    c.OH = (H + 2 * pad - k) / stride + 1;
    c.OW = (W + 2 * pad - k) / stride + 1;
    // stem weights are stored [64][32] (27 padded to 32 so the row pitch is TMA-legal)
    c.w_len = (cin == 3) ? (int64_t)cout * kStemK : (int64_t)cout * k * k * cin;
    c.w_off = add_param(c.w_len, 0);
    c.g_off = add_param(cout, 1);
    c.b_off = add_param(cout, 2);
    m->convs.push_back(c);
    return (int)m->convs.size() - 1;
  };
  m->stem = add_conv(3, 64, 3, 1, 1, 32, 32);
  int H = 32, cin = 64;
  const int widths[4] = {64, 128, 256, 512};
  for (int L = 0; L < 4; L++) {
    for (int bI = 0; bI < 2; bI++) {
      const int cout = widths[L];
      const int stride = (L > 0 && bI == 0) ? 2 : 1;
      Block b{};
      b.c3 = -1;
      b.c1 = add_conv(cin, cout, 3, stride, 1, H, H);
      const int OH = m->convs[b.c1].OH;
      b.c2 = add_conv(cout, cout, 3, 1, 1, OH, OH);
      b.ds = (stride != 1 || cin != cout) ? add_conv(cin, cout, 1, stride, 0, H, H) : -1;
      m->blocks.push_back(b);
      cin = cout;
      H = OH;
    }
  }
  m->fc_w = add_param((int64_t)m->classes * 512, 3);
  m->fc_b = add_param(m->classes, 4);
  m->P = (off + 31) & ~int64_t(31);
  m->need_a.assign(m->convs.size(), 0);
  m->need_a[m->stem] = 1;
  for (auto& b : m->blocks) m->need_a[b.c1] = 1;
}

// ResNet-50 (torchvision layout, v1.5: stride on the 3x3 conv), S x S input
void build_layers50(dbs_resnet* m) {
  int64_t off = 0;
  auto add_param = [&](int64_t len, int kind) {
    const int64_t o = off;
    m->t_off.push_back(o);
    m->t_len.push_back(len);
    m->t_kind.push_back(kind);
    off += pad8(len);
    return o;
  };
  auto add_conv = [&](int cin, int cout, int k, int stride, int pad, int H) {
    Conv c{};
    c.cin = cin;
    c.cout = cout;
    c.k = k;
    c.stride = stride;
    c.pad = pad;
    c.H = c.W = H;
    c.OH = c.OW = (H + 2 * pad - k) / stride + 1;
    c.w_len = (cin == 3) ? (int64_t)cout * kStem7K : (int64_t)cout * k * k * cin;
    c.w_off = add_param(c.w_len, 0);
    c.g_off = add_param(cout, 1);
    c.b_off = add_param(cout, 2);
    m->convs.push_back(c);
    return (int)m->convs.size() - 1;
  };
  const int S = m->image;
  m->stem = add_conv(3, 64, 7, 2, 3, S);
  int H = S / 4, cin = 64;  // after the stem (S/2) and the max-pool (S/4)
  const int widths[4] = {64, 128, 256, 512};
  const int depth[4] = {3, 4, 6, 3};
  for (int L = 0; L < 4; L++) {
    for (int bI = 0; bI < depth[L]; bI++) {
      const int w = widths[L], cout = 4 * w;
      const int stride = (L > 0 && bI == 0) ? 2 : 1;
      Block b{};
      b.c1 = add_conv(cin, w, 1, 1, 0, H);
      b.c2 = add_conv(w, w, 3, stride, 1, H);
      const int OH = m->convs[b.c2].OH;
      b.c3 = add_conv(w, cout, 1, 1, 0, OH);
      b.ds = (stride != 1 || cin != cout) ? add_conv(cin, cout, 1, stride, 0, H) : -1;
      m->blocks.push_back(b);
      cin = cout;
      H = OH;
    }
  }
  m->feat_c = cin;
  m->feat_hw = H * H;
  m->fc_w = add_param((int64_t)m->classes * cin, 3);
  m->fc_b = add_param(m->classes, 4);
  m->P = (off + 31) & ~int64_t(31);
  m->need_a.assign(m->convs.size(), 0);
  m->need_a[m->stem] = 1;
  for (auto& b : m->blocks) m->need_a[b.c1] = m->need_a[b.c2] = 1;
}

int alloc_all(dbs_resnet* m) {
  const int64_t B = m->max_b;
  cudaError_t e = cudaSuccess;
  auto A = [&](void** p, size_t bytes) {
    if (e == cudaSuccess) e = cudaMalloc(p, bytes);
  };
  const bool f32 = m->prec == DBS_PREC_F32;
  const size_t es_op = f32 ? 8 : 2;  // operand tensors: S32 | bf16
  const size_t es_y = f32 ? 4 : 2;   // conv outputs / input gradients: fp32 | bf16
  {
    const Conv& st = m->convs[m->stem];
    A((void**)&m->stem_cols, (size_t)B * st.OH * st.OW * m->stem_k * es_op);
  }
  int64_t max_act = 0;
  for (size_t ci = 0; ci < m->convs.size(); ci++) {
    const Conv& c = m->convs[ci];
    const int64_t n = B * c.OH * c.OW * c.cout;
    void *y, *a = nullptr;
    A((void**)&y, n * es_y);
    if (m->need_a[ci]) A((void**)&a, n * es_op);
    m->y.push_back(y);
    m->a.push_back(a);
    float *mu, *is;
    A((void**)&mu, c.cout * 4);
    A((void**)&is, c.cout * 4);
    m->mean.push_back(mu);
    m->invstd.push_back(is);
    if (n > max_act) max_act = n;
    const int64_t nin = B * c.H * c.W * c.cin;
    if (nin > max_act) max_act = nin;
  }
  for (size_t i = 0; i < m->blocks.size(); i++) {
    const Block& bk = m->blocks[i];
    const Conv& c = m->convs[bk.c3 >= 0 ? bk.c3 : bk.c2];  // the block's last conv shapes its output
    void* o;
    A((void**)&o, (size_t)B * c.OH * c.OW * c.cout * es_op);
    m->blk_out.push_back(o);
  }
  m->run_off.clear();
  int64_t run_len = 0;
  for (auto& c : m->convs) {
    m->run_off.push_back(run_len);
    run_len += 2 * (int64_t)c.cout;
  }
  A((void**)&m->run_stats, (size_t)run_len * sizeof(float));
  if (e == cudaSuccess) {
    std::vector<float> init((size_t)run_len);
    for (size_t ci = 0; ci < m->convs.size(); ci++)
      for (int k = 0; k < m->convs[ci].cout; k++) {
        init[m->run_off[ci] + k] = 0.0f;                      // running mean
        init[m->run_off[ci] + m->convs[ci].cout + k] = 1.0f;  // running variance
      }
    e = cudaMemcpy(m->run_stats, init.data(), init.size() * sizeof(float), cudaMemcpyHostToDevice);
  }
  m->stats_off.clear();
  m->stats_len = 0;
  for (auto& c : m->convs) {
    m->stats_off.push_back(m->stats_len);
    m->stats_len += 2 * (int64_t)c.cout;
  }
  A((void**)&m->stats_acc, (size_t)m->stats_len * sizeof(double));
  // gradient buffers hold either kind (f32 mode: fp32 input gradients or S32 BN-backward outputs)
  A((void**)&m->g0, max_act * es_op);
  A((void**)&m->g1, max_act * es_op);
  A((void**)&m->g2, max_act * es_op);
  A((void**)&m->g3, max_act * es_op);
  if (m->arch == 50) {
    const Conv& st = m->convs[m->stem];
    const int P = st.OH / 2;
    const int64_t mp = B * P * P * 64;
    A((void**)&m->g4, max_act * es_op);
    A((void**)&m->mp_out, mp * es_op);
    A((void**)&m->mp_idx, mp);
    A((void**)&m->feat_b, (size_t)B * m->feat_c * es_op);
    A((void**)&m->logits, (size_t)B * m->cpad * 4);
    A((void**)&m->dlog_f, (size_t)B * m->cpad * 4);
    A((void**)&m->dlog_b, f32 ? (size_t)B * m->cpad32 * 8 : (size_t)B * m->cpad * 2);
    A((void**)&m->dfeat, (size_t)B * m->feat_c * 4);
  }
  A((void**)&m->feat, (size_t)B * 512 * 4);
  A((void**)&m->dlog, (size_t)B * 16 * 4);
  A((void**)&m->loss_per, (size_t)B * 4);
  A((void**)&m->loss_scratch, 64);
  if (e != cudaSuccess) {
    set_error("resnet alloc: %s", cudaGetErrorString(e));
    return DBS_ERR_CUDA;
  }
  return DBS_OK;
}

ConvTensor nhwc(int64_t N, int H, int W, int C) { return ConvTensor{(int)N, H, W, C}; }

// forward conv -> y (bf16) + BN statistics -> mean/invstd
// 3x3 / stride 1 / 64 -> 64 channels: the GEMM's halo variant (resident filter, one
// zero-padded input halo box per tile; gemm.cu HaloCfg).
// DBS_CONV_HALO=0 turns it off (A/B measurements).
bool halo_ok(const Conv& c) {
  static const bool enabled = [] {
    const char* e = getenv("DBS_CONV_HALO");
    return !(e && e[0] == '0');
  }();
  return enabled && c.k == 3 && c.stride == 1 && c.pad == 1 && c.cin == 64 && c.cout == 64 && halo_fits(c.OH, c.OW);
}
// the fp32-class (S32) halo variant (gemm.cu HaloTfCfg): same shape, W <= 32.  On by
// default (DBS_HALO_TF=0 disables it): it moves 22 KB per k-block instead of the
// streamed kernel's 48 KB, whose two TMA boxes take the SM's TMA unit ~1000 cycles per
// k-block.  (It lost while the MMAs were issued from one lane -- ~80 cycles of
// uniform-register waterfall per instruction; with the warp-wide issue the worker
// step drops 11.87 -> 11.00 ms, profiles/r2/mma_issue.txt.)
bool halo_tf_ok(const Conv& c) {
  static const bool enabled = [] {
    const char* e = getenv("DBS_HALO_TF");
    return !(e && e[0] == '0');
  }();
  return enabled && c.k == 3 && c.stride == 1 && c.pad == 1 && c.cin == 64 && c.cout == 64 &&
         halo_tf_fits(c.OH, c.OW);
}

// the operand copy of the parameter at flat offset `off` (bf16 or S32 shadow)
const void* wptr(const dbs_resnet* m, const void* shadow, int64_t off) {
  return static_cast<const char*>(shadow) + off * (m->prec == DBS_PREC_F32 ? 8 : 2);
}

int conv_fwd(dbs_resnet* m, int ci, const void* x, const void* shadow, int64_t B, cudaStream_t s) {
  const Conv& c = m->convs[ci];
  const bool f32 = m->prec == DBS_PREC_F32;
  const int64_t M = B * c.OH * c.OW;
  ConvCall call{};
  call.tf = f32;
  call.M = M;
  call.N = c.cout;
  call.epi = f32 ? DBS_EPI_F32 : DBS_EPI_BF16;
  call.d = m->y[ci];
  call.ldd = c.cout;
  call.sum_part = m->stats_acc + m->stats_off[ci];
  call.sq_part = m->stats_acc + m->stats_off[ci] + c.cout;
  call.b = wptr(m, shadow, c.w_off);
  call.b_mode = 0;
  if (c.cin == 3) {  // stem: explicit im2col columns [M][stem_k]
    call.K = m->stem_k;
    call.a_mode = 0;
    call.a = m->stem_cols;
    call.lda = m->stem_k;
    call.ldb = m->stem_k;
  } else if (c.k == 1 && c.stride == 1) {  // 1x1: a plain GEMM over the [pixels][Cin] view
    call.K = c.cin;
    call.a_mode = 0;
    call.a = x;
    call.lda = c.cin;
    call.ldb = c.cin;
  } else {
    call.K = (int64_t)c.k * c.k * c.cin;
    call.a_mode = 2;
    call.a = x;
    call.ta = nhwc(B, c.H, c.W, c.cin);
    call.ga = ConvGeom{c.k, c.k, c.cin / (f32 ? 32 : 64), c.stride, c.pad, c.OH, c.OW, c.cin};
    call.ldb = call.K;
    call.halo = f32 ? halo_tf_ok(c) : halo_ok(c);
  }
  int st = conv_gemm(call, s);
  if (st) return st;
  return DBS_OK;  // batch statistics are finalised by the BN apply kernel (bn_apply_kernel)
}

int bn_apply(dbs_resnet* m, int ci, const float* pf, const void* res, int ds, int relu, int64_t B,
             void* out, cudaStream_t s) {
  const Conv& c = m->convs[ci];
  const int64_t M = B * c.OH * c.OW;
  const int64_t total = M * (c.cout / 8);
  const Conv* d = ds >= 0 ? &m->convs[ds] : nullptr;
  const size_t smem = (size_t)(ds >= 0 ? 4 : 2) * c.cout * sizeof(float);
  if (m->prec == DBS_PREC_F32) {
    DBS_CUDA_TRY(launch_pdl(
        bn_apply_f32_kernel, dim3(grid_one_wave(bn_apply_f32_kernel, total, 256, smem)), dim3(256), smem, s,
        static_cast<const float*>(m->y[ci]), m->stats_acc + m->stats_off[ci], m->mean[ci], m->invstd[ci],
        pf + c.g_off, pf + c.b_off, static_cast<const float*>(res), d ? static_cast<const float*>(m->y[ds]) : nullptr,
        d ? m->stats_acc + m->stats_off[ds] : nullptr, d ? m->mean[ds] : nullptr, d ? m->invstd[ds] : nullptr,
        d ? pf + d->g_off : nullptr, d ? pf + d->b_off : nullptr, relu, c.cout, M, static_cast<float*>(out),
        m->run_stats + m->run_off[ci], d ? m->run_stats + m->run_off[ds] : nullptr, m->bn_momentum));
    DBS_LAUNCH_CHECK();
    return DBS_OK;
  }
  DBS_CUDA_TRY(launch_pdl(
      bn_apply_kernel, dim3(grid_one_wave(bn_apply_kernel, total, 256, smem)), dim3(256), smem, s,
      static_cast<const uint16_t*>(m->y[ci]), m->stats_acc + m->stats_off[ci], m->mean[ci], m->invstd[ci],
      pf + c.g_off, pf + c.b_off, static_cast<const uint16_t*>(res),
      d ? static_cast<const uint16_t*>(m->y[ds]) : nullptr, d ? m->stats_acc + m->stats_off[ds] : nullptr,
      d ? m->mean[ds] : nullptr, d ? m->invstd[ds] : nullptr, d ? pf + d->g_off : nullptr,
      d ? pf + d->b_off : nullptr, relu, c.cout, M, static_cast<uint16_t*>(out)));
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

// BN backward for conv ci: gin (masked by `mask` > 0 when given) -> dy; gamma/beta grads into grad
// (f32 mode: gin / g_out fp32, mask / dy S32)
int bn_bwd(dbs_resnet* m, int ci, const float* pf, float* grad, const void* gin, const void* mask, int64_t B,
           void* dy, void* g_out, cudaStream_t s) {
  const Conv& c = m->convs[ci];
  const int64_t M = B * c.OH * c.OW;
  const int cv = c.cout / 8;
  const int rows_per_pass = 256 / cv;
  const int64_t total = M * cv;
  const size_t smem = (size_t)3 * c.cout * sizeof(float);
  if (m->prec == DBS_PREC_F32) {
    int blocks = (int)((M + rows_per_pass - 1) / rows_per_pass);
    const int cap = current_sm_count() * resident_per_sm(bn_bwd_reduce_f32_kernel, 256, 0);
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    DBS_CUDA_TRY(launch_pdl(bn_bwd_reduce_f32_kernel, dim3(blocks), dim3(256), 0, s, static_cast<const float*>(gin),
                            static_cast<const float*>(mask), static_cast<const float*>(m->y[ci]), m->mean[ci],
                            m->invstd[ci], c.cout, M, grad + c.g_off, grad + c.b_off));
    DBS_LAUNCH_CHECK();
    DBS_CUDA_TRY(launch_pdl(bn_bwd_apply_f32_kernel, dim3(grid_one_wave(bn_bwd_apply_f32_kernel, total, 256, smem)),
                            dim3(256), smem, s, static_cast<const float*>(gin), static_cast<const float*>(mask),
                            static_cast<const float*>(m->y[ci]), m->mean[ci], m->invstd[ci], pf + c.g_off,
                            grad + c.g_off, grad + c.b_off, c.cout, M, static_cast<float*>(dy),
                            static_cast<float*>(g_out)));
    DBS_LAUNCH_CHECK();
    return DBS_OK;
  }
  int blocks = (int)((M + rows_per_pass * 4 - 1) / (rows_per_pass * 4));  // ~4 rows per thread (one trip)
  const int cap = current_sm_count() * resident_per_sm(bn_bwd_reduce_kernel<8>, 256, 0);
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  DBS_CUDA_TRY(launch_pdl(bn_bwd_reduce_kernel<8>, dim3(blocks), dim3(256), 0, s, static_cast<const uint16_t*>(gin),
                          static_cast<const uint16_t*>(mask), static_cast<const uint16_t*>(m->y[ci]), m->mean[ci],
                          m->invstd[ci], c.cout, M, grad + c.g_off, grad + c.b_off));
  DBS_LAUNCH_CHECK();
  DBS_CUDA_TRY(launch_pdl(bn_bwd_apply_kernel, dim3(grid_one_wave(bn_bwd_apply_kernel, total, 256, smem)), dim3(256),
                          smem, s, static_cast<const uint16_t*>(gin), static_cast<const uint16_t*>(mask),
                          static_cast<const uint16_t*>(m->y[ci]), m->mean[ci], m->invstd[ci], pf + c.g_off,
                          grad + c.g_off, grad + c.b_off, c.cout, M, static_cast<uint16_t*>(dy),
                          static_cast<uint16_t*>(g_out)));
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

bool merge_parity_enabled() {
  static const bool on = [] {
    const char* e = getenv("DBS_MERGE_PARITY");
    return !(e && e[0] == '0');
  }();
  return on;
}

// dX (+)= dgrad of conv c from dy; accumulate selects the accumulate epilogue.
// tf: S32 dy / w, fp32 dx (F32 / F32_ACCUM); else bf16 throughout.
int conv_dgrad_ex(const Conv& c, const void* dy, const void* w, int64_t B, void* dx, int accumulate,
                  cudaStream_t s, bool tf = false) {
  // the GEMM reads the filter flipped and transposed in place (B mode 3)
  const int cb = tf ? 32 : 64;  // channels per logical k-block
  ConvCall call{};
  call.tf = tf;
  call.N = c.cin;
  call.a_mode = 2;
  call.a = dy;
  call.ta = nhwc(B, c.OH, c.OW, c.cout);
  call.b_mode = 3;
  call.b = w;
  call.tb = ConvTensor{c.cout, 1, c.k * c.k, c.cin};  // {N=Cout, -, W=R*S, C=Cin} filter view
  call.epi = tf ? (accumulate ? DBS_EPI_F32_ACCUM : DBS_EPI_F32) : (accumulate ? DBS_EPI_BF16_ACCUM : DBS_EPI_BF16);
  call.d = dx;
  call.ldd = c.cin;
  if (c.k == 1 && c.stride == 1) {
    // 1x1: dX [pixels][Cin] = dY [pixels][Cout] x W [Cout][Cin] (W read MN-major)
    call.M = B * c.H * c.W;
    call.K = c.cout;
    call.a_mode = 0;
    call.lda = c.cout;
    call.b_mode = 1;
    call.ldb = c.cin;
    call.tb = ConvTensor{};
    return conv_gemm(call, s);
  }
  if (c.stride == 1) {
    // stride 1: the flipped filter over dY, same padding
    call.M = B * c.H * c.W;
    call.K = (int64_t)c.k * c.k * c.cout;
    call.ga = ConvGeom{c.k, c.k, c.cout / cb, 1, c.k / 2, c.H, c.W, c.cout};
    call.halo = tf ? halo_tf_ok(c) : halo_ok(c);
    return conv_gemm(call, s);
  }
  // stride 2: one GEMM per output parity class (a, b).  dX(2i+a, 2j+b) gathers
  // only the taps with r = a + pad (mod 2), s = b + pad (mod 2), each reading
  // dY at (i + (a + pad - r) / 2, j + (b + pad - s) / 2): no zero-dilated dY,
  // no multiplications by the zeros of the dilation.
  DBS_REQUIRE(c.stride == 2 && c.H == 2 * c.OH && c.W == 2 * c.OW, DBS_ERR_ARGUMENT,
              "conv dgrad: stride 2 needs even input extents");
  const int pad = c.k / 2;
  bool empty_class = false;
  for (int a = 0; a < 2; a++)
    for (int b = 0; b < 2; b++) {
      int n = 0;
      for (int r = 0; r < c.k; r++)
        for (int q = 0; q < c.k; q++)
          if (((a + pad - r) & 1) == 0 && ((b + pad - q) & 1) == 0) n++;
      if (n == 0) empty_class = true;
    }
  if (empty_class && !accumulate)
    DBS_CUDA_TRY(cudaMemsetAsync(dx, 0, (tf ? sizeof(float) : sizeof(uint16_t)) * (size_t)(B * c.H * c.W * c.cin), s));
  // all non-empty parity classes in ONE launch when one N tile covers Cin (bf16 tiles
  // up to 256 wide, S32 tiles up to 128), each class a full GEMM over the OH x OW grid
  if (c.cin <= (tf ? 128 : 256) && merge_parity_enabled()) {
    ConvCall mc = call;
    mc.M = B * c.OH * c.OW;
    mc.nclass = 0;
    int kmax = 0;
    for (int a = 0; a < 2; a++)
      for (int b = 0; b < 2; b++) {
        ConvTaps t{};
        for (int r = 0; r < c.k; r++)
          for (int q = 0; q < c.k; q++) {
            if (((a + pad - r) & 1) != 0 || ((b + pad - q) & 1) != 0) continue;
            t.dh[t.n] = (int8_t)((a + pad - r) / 2);
            t.dw[t.n] = (int8_t)((b + pad - q) / 2);
            t.rs[t.n] = (uint8_t)(r * c.k + q);
            t.n++;
          }
        if (t.n == 0) continue;
        mc.cls_taps[mc.nclass] = t;
        mc.cls_omap[mc.nclass] = OutMap{1, c.H, c.W, a, b, c.OH, c.OW};
        mc.nclass++;
        if (t.n > kmax) kmax = t.n;
      }
    mc.K = (int64_t)kmax * c.cout;
    mc.ga = ConvGeom{1, kmax, c.cout / cb, 1, 0, c.OH, c.OW, c.cout};
    mc.taps = mc.cls_taps[0];
    mc.bn_override = c.cin <= 64 ? 64 : (c.cin <= 128 ? 128 : 256);
    return conv_gemm(mc, s);
  }
  for (int a = 0; a < 2; a++)
    for (int b = 0; b < 2; b++) {
      ConvTaps t{};
      for (int r = 0; r < c.k; r++)
        for (int q = 0; q < c.k; q++) {
          if (((a + pad - r) & 1) != 0 || ((b + pad - q) & 1) != 0) continue;
          t.dh[t.n] = (int8_t)((a + pad - r) / 2);
          t.dw[t.n] = (int8_t)((b + pad - q) / 2);
          t.rs[t.n] = (uint8_t)(r * c.k + q);
          t.n++;
        }
      if (t.n == 0) continue;
      ConvCall cc = call;
      cc.M = B * c.OH * c.OW;
      cc.K = (int64_t)t.n * c.cout;
      cc.ga = ConvGeom{1, t.n, c.cout / cb, 1, 0, c.OH, c.OW, c.cout};
      cc.taps = t;
      cc.omap = OutMap{1, c.H, c.W, a, b, c.OH, c.OW};
      int st = conv_gemm(cc, s);
      if (st) return st;
    }
  return DBS_OK;
}

int conv_dgrad(dbs_resnet* m, int ci, const void* dy, const void* shadow, int64_t B, void* dx, int accumulate,
               cudaStream_t s) {
  const Conv& c = m->convs[ci];
  return conv_dgrad_ex(c, dy, wptr(m, shadow, c.w_off), B, dx, accumulate, s, m->prec == DBS_PREC_F32);
}

bool wgrad_trans_enabled() {
  static const bool on = [] {
    const char* e = getenv("DBS_WGRAD_T");
    return !(e && e[0] == '0');
  }();
  return on;
}

// dW of conv c (fp32 atomics into dw) from dy and the conv input x (stem: im2col columns)
// tf: S32 dy / x; else bf16.  `stem_k` is the stem's padded K.
int conv_wgrad_ex(const Conv& c, const void* dy, const void* x, int64_t B, float* dw, cudaStream_t s,
                  bool tf = false, int stem_k = 0) {
  const int64_t pixels = B * c.OH * c.OW;
  const int kb = tf ? 32 : 64;  // pixels per logical k-block
  ConvCall call{};
  call.tf = tf;
  if (c.cout == 64 && c.cin % 64 == 0 && (c.k == 1 ? c.stride == 1 : true) && ((uintptr_t)dw & 15) == 0 &&
      wgrad_trans_enabled()) {
    // 64 output channels: dW^T = X^T dY puts the (r, s, c) reduction rows on the
    // 128-row MMA M side (all rows live) instead of the 64 output channels (half
    // of every M = 128 instruction wasted); the epilogue stores D transposed
    call.M = (int64_t)c.k * c.k * c.cin;
    call.N = c.cout;
    call.K = pixels;
    call.b_mode = 1;  // dY [pixels][Cout], MN-major
    call.b = dy;
    call.ldb = c.cout;
    if (c.k == 1) {
      call.a_mode = 1;  // X [pixels][Cin], MN-major
      call.a = x;
      call.lda = c.cin;
    } else {
      call.a_mode = 5;
      call.a = x;
      call.ta = nhwc(B, c.H, c.W, c.cin);
      call.ga = ConvGeom{c.k, c.k, c.cin / kb, c.stride, c.pad, c.OH, c.OW, c.cin};
    }
    call.epi = DBS_EPI_F32_ATOMIC;
    call.d = dw;
    call.ldd = call.M;
    call.d_trans = 1;
    call.bn_override = 64;
    const int64_t tiles = (call.M + 127) / 128;
    int64_t splits = current_sm_count() / tiles;
    const int64_t kblocks = (call.K + kb - 1) / kb;
    if (splits > kblocks) splits = kblocks;
    if (splits < 1) splits = 1;
    call.splits = (int)splits;
    return conv_gemm(call, s);
  }
  call.a_mode = 1;  // dY^T: dY stored [pixels][Cout]
  call.a = dy;
  call.lda = c.cout;
  call.M = c.cout;
  call.epi = DBS_EPI_F32_ATOMIC;
  call.d = dw;
  int bn;
  if (c.cin == 3) {  // stem: columns [pixels][stem_k]
    call.N = stem_k;
    call.K = pixels;
    call.b_mode = 1;
    call.b = x;
    call.ldb = stem_k;
    call.ldd = stem_k;
    bn = 64;
  } else if (c.k == 1 && c.stride == 1) {  // 1x1: dW = dY^T X over the [pixels][Cin] view
    call.N = c.cin;
    call.K = pixels;
    call.b_mode = 1;
    call.b = x;
    call.ldb = c.cin;
    call.ldd = c.cin;
    bn = c.cin >= 256 ? 256 : c.cin;
    if (tf && bn > 128) bn = 128;
    call.bn_override = bn;
  } else {
    // N = (r, s, c): the tile must divide Cin so it never straddles two taps
    // (a 192-channel input takes 64-wide tiles, not the 256-wide kernel)
    call.N = (int64_t)c.k * c.k * c.cin;
    call.K = pixels;
    call.b_mode = 2;
    call.b = x;
    call.tb = nhwc(B, c.H, c.W, c.cin);
    call.gb = ConvGeom{c.k, c.k, c.cin / kb, c.stride, c.pad, c.OH, c.OW, c.cin};
    call.ldd = call.N;
    bn = c.cin % 256 == 0 ? 256 : (c.cin % 128 == 0 ? 128 : 64);
    if (tf && bn > 128) bn = 128;
    call.bn_override = bn;
  }
  // split the long pixel reduction so the persistent GEMM's one round of
  // tiles x splits just fits the SMs this launch can use
  const int64_t tiles = ((call.M + 127) / 128) * ((call.N + bn - 1) / bn);
  const int64_t kblocks = (call.K + kb - 1) / kb;
  int64_t splits = current_sm_count() / tiles;
  if (splits > kblocks) splits = kblocks;
  if (splits < 1) splits = 1;
  call.splits = (int)splits;
  return conv_gemm(call, s);
}

int conv_wgrad(dbs_resnet* m, int ci, const void* dy, const void* x, int64_t B, float* grad, cudaStream_t s) {
  const Conv& c = m->convs[ci];
  return conv_wgrad_ex(c, dy, c.cin == 3 ? m->stem_cols : x, B, grad + c.w_off, s, m->prec == DBS_PREC_F32,
                       (int)(c.w_len / c.cout));
}

}  // namespace

namespace dbs {

int resnet50_fwd_bwd(dbs_resnet* m, const void* wb, const float* pf, const uint8_t* x_base,
                     const int32_t* y_base, const int64_t* d_iter, int64_t B, float* grad, float* loss,
                     cudaStream_t s) {
  int st;
  const bool f32 = m->prec == DBS_PREC_F32;
  DBS_CUDA_TRY(cudaMemsetAsync(grad, 0, sizeof(float) * m->P, s));
  DBS_CUDA_TRY(cudaMemsetAsync(m->stats_acc, 0, sizeof(double) * m->stats_len, s));
  // ---------------- stem: 7x7/2 conv (explicit im2col) + BN + ReLU + 3x3/2 max-pool ----------------
  const Conv& sc = m->convs[m->stem];
  if (f32)
    DBS_CUDA_TRY(launch_pdl(im2col_stem7_f32_kernel, dim3((unsigned)(B * sc.OH)), dim3(256),
                            (size_t)3 * 7 * (m->image + 6) * sizeof(float), s, x_base, d_iter, B, m->image,
                            static_cast<float*>(m->stem_cols)));
  else
    DBS_CUDA_TRY(launch_pdl(im2col_stem7_kernel, dim3((unsigned)(B * sc.OH)), dim3(256),
                            (size_t)3 * 7 * (m->image + 6) * sizeof(float), s, x_base, d_iter, B, m->image,
                            static_cast<uint16_t*>(m->stem_cols)));
  DBS_LAUNCH_CHECK();
  if ((st = conv_fwd(m, m->stem, nullptr, wb, B, s))) return st;
  if ((st = bn_apply(m, m->stem, pf, nullptr, -1, 1, B, m->a[m->stem], s))) return st;
  const int PH = sc.OH / 2;
  if (f32)
    DBS_CUDA_TRY(launch_pdl(maxpool_fwd_f32_kernel, dim3(grid_one_wave(maxpool_fwd_f32_kernel, B * PH * PH * 8, 256, 0)),
                            dim3(256), 0, s, static_cast<const float*>(m->a[m->stem]), B, sc.OH, sc.OW, 64, PH, PH,
                            static_cast<float*>(m->mp_out), m->mp_idx));
  else
    DBS_CUDA_TRY(launch_pdl(maxpool_fwd_kernel, dim3(grid_one_wave(maxpool_fwd_kernel, B * PH * PH * 8, 256, 0)),
                            dim3(256), 0, s, static_cast<const uint16_t*>(m->a[m->stem]), B, sc.OH, sc.OW, 64, PH,
                            PH, static_cast<uint16_t*>(m->mp_out), m->mp_idx));
  DBS_LAUNCH_CHECK();
  // ---------------- bottleneck blocks ----------------
  const void* x = m->mp_out;
  std::vector<const void*> blk_in(m->blocks.size());
  for (size_t i = 0; i < m->blocks.size(); i++) {
    const Block& b = m->blocks[i];
    blk_in[i] = x;
    if ((st = conv_fwd(m, b.c1, x, wb, B, s))) return st;
    if ((st = bn_apply(m, b.c1, pf, nullptr, -1, 1, B, m->a[b.c1], s))) return st;
    if ((st = conv_fwd(m, b.c2, m->a[b.c1], wb, B, s))) return st;
    if ((st = bn_apply(m, b.c2, pf, nullptr, -1, 1, B, m->a[b.c2], s))) return st;
    if ((st = conv_fwd(m, b.c3, m->a[b.c2], wb, B, s))) return st;
    if (b.ds >= 0 && (st = conv_fwd(m, b.ds, x, wb, B, s))) return st;
    if ((st = bn_apply(m, b.c3, pf, b.ds >= 0 ? nullptr : x, b.ds, 1, B, m->blk_out[i], s))) return st;
    x = m->blk_out[i];
  }
  // ---------------- head: average pool, FC (tcgen05 GEMMs), softmax cross-entropy ----------------
  const int C = m->feat_c, HW = m->feat_hw, K = m->classes, ld = m->cpad;
  const void* wfc = wptr(m, wb, m->fc_w);
  if (f32) {
    DBS_CUDA_TRY(launch_pdl(avgpool_f32_kernel, dim3(grid_one_wave(avgpool_f32_kernel, B * (C / 8), 256, 0)), dim3(256),
                            0, s, static_cast<const float*>(x), B, HW, C, static_cast<float*>(m->feat_b)));
    DBS_LAUNCH_CHECK();
    if ((st = gemm_tf(m->feat_b, 0, C, wfc, 0, C, m->logits, ld, B, K, C, DBS_EPI_BIAS_F32, pf + m->fc_b, nullptr, s)))
      return st;
    DBS_CUDA_TRY(launch_pdl(ce_f32_kernel, dim3((unsigned)B), dim3(256), 0, s, m->logits, ld, y_base, d_iter, B, K,
                            m->dlog_f, static_cast<float*>(m->dlog_b), m->cpad32, m->loss_per));
    DBS_LAUNCH_CHECK();
  } else {
    DBS_CUDA_TRY(launch_pdl(avgpool_kernel, dim3(grid_one_wave(avgpool_kernel, B * (C / 8), 256, 0)), dim3(256), 0, s,
                            static_cast<const uint16_t*>(x), B, HW, C, static_cast<uint16_t*>(m->feat_b)));
    DBS_LAUNCH_CHECK();
    // logits [B][K] = feat [B][C] . Wfc [K][C]^T + b
    if ((st = gemm_bf16(m->feat_b, 0, C, wfc, 0, C, m->logits, ld, B, K, C, DBS_EPI_BIAS_F32, pf + m->fc_b, nullptr,
                        s, nullptr)))
      return st;
    DBS_CUDA_TRY(launch_pdl(ce_kernel, dim3((unsigned)B), dim3(256), 0, s, m->logits, ld, y_base, d_iter, B, K,
                            m->dlog_f, static_cast<uint16_t*>(m->dlog_b), m->loss_per));
    DBS_LAUNCH_CHECK();
  }
  DBS_CUDA_TRY(launch_pdl(head_bias_kernel, dim3((K + 255) / 256), dim3(256), 0, s, m->dlog_f, ld, m->loss_per, B, K,
                          grad + m->fc_b, loss ? loss : m->loss_scratch, loss ? d_iter : nullptr));
  DBS_LAUNCH_CHECK();
  if (f32) {
    // dWfc [K][C] = dlog^T . feat ; dfeat [B][C] = dlog [B][K] . Wfc [K][C]
    if ((st = gemm_tf(m->dlog_b, 1, m->cpad32, m->feat_b, 1, C, grad + m->fc_w, C, K, C, B, DBS_EPI_F32, nullptr,
                      nullptr, s)))
      return st;
    if ((st = gemm_tf(m->dlog_b, 0, m->cpad32, wfc, 1, C, m->dfeat, C, B, C, K, DBS_EPI_F32, nullptr, nullptr, s)))
      return st;
  } else {
    // dWfc [K][C] = dlog^T . feat  (both MN-major over the batch)
    if ((st = gemm_bf16(m->dlog_b, 1, ld, m->feat_b, 1, C, grad + m->fc_w, C, K, C, B, DBS_EPI_F32, nullptr, nullptr,
                        s, nullptr)))
      return st;
    // dfeat [B][C] = dlog [B][K] . Wfc [K][C]  (Wfc MN-major)
    if ((st = gemm_bf16(m->dlog_b, 0, ld, wfc, 1, C, m->dfeat, C, B, C, K, DBS_EPI_F32, nullptr, nullptr, s, nullptr)))
      return st;
  }
  void* gcur = m->g0;
  if (f32)
    DBS_CUDA_TRY(launch_pdl(head_bcast_f32_kernel, dim3(grid_one_wave(head_bcast_f32_kernel, B * HW * (C / 8), 256, 0)),
                            dim3(256), 0, s, m->dfeat, B, HW, C, static_cast<float*>(gcur)));
  else
    DBS_CUDA_TRY(launch_pdl(head_bcast_kernel, dim3(grid_one_wave(head_bcast_kernel, B * HW * (C / 8), 256, 0)),
                            dim3(256), 0, s, m->dfeat, B, HW, C, static_cast<uint16_t*>(gcur)));
  DBS_LAUNCH_CHECK();
  // ---------------- backward through the blocks ----------------
  // buffers: gx = gradient of the block input, t0 = BN outputs' gradients,
  // t1 = conv input gradients / masked shortcut gradient, t2 = shortcut BN's
  void* gx = m->g1;
  void* t0 = m->g2;
  void* t1 = m->g3;
  void* t2 = m->g4;
  for (int i = (int)m->blocks.size() - 1; i >= 0; i--) {
    const Block& b = m->blocks[i];
    // BN3 with the block's output ReLU mask; the masked gradient is the
    // identity shortcut's gradient (gx) or the projection's input (t1)
    if ((st = bn_bwd(m, b.c3, pf, grad, gcur, m->blk_out[i], B, t0, b.ds >= 0 ? t1 : gx, s))) return st;
    if (b.ds >= 0) {
      if ((st = bn_bwd(m, b.ds, pf, grad, t1, nullptr, B, t2, nullptr, s))) return st;
      if ((st = conv_wgrad(m, b.ds, t2, blk_in[i], B, grad, s))) return st;
    }
    if ((st = conv_wgrad(m, b.c3, t0, m->a[b.c2], B, grad, s))) return st;
    if ((st = conv_dgrad(m, b.c3, t0, wb, B, t1, 0, s))) return st;
    if ((st = bn_bwd(m, b.c2, pf, grad, t1, m->a[b.c2], B, t0, nullptr, s))) return st;
    if ((st = conv_wgrad(m, b.c2, t0, m->a[b.c1], B, grad, s))) return st;
    if ((st = conv_dgrad(m, b.c2, t0, wb, B, t1, 0, s))) return st;
    if ((st = bn_bwd(m, b.c1, pf, grad, t1, m->a[b.c1], B, t0, nullptr, s))) return st;
    if ((st = conv_wgrad(m, b.c1, t0, blk_in[i], B, grad, s))) return st;
    if (b.ds >= 0) {
      // the 1x1 stride-1 conv1 covers every input pixel; the projection's
      // (stride-2: even pixels only) input gradient accumulates onto it
      if ((st = conv_dgrad(m, b.c1, t0, wb, B, gx, 0, s))) return st;
      if ((st = conv_dgrad(m, b.ds, t2, wb, B, gx, 1, s))) return st;
    } else {
      if ((st = conv_dgrad(m, b.c1, t0, wb, B, gx, 1, s))) return st;
    }
    void* old = gcur;
    gcur = gx;
    gx = old;
  }
  // ---------------- stem backward: max-pool, BN + ReLU mask, weight gradient ----------------
  if (f32)
    DBS_CUDA_TRY(launch_pdl(maxpool_bwd_f32_kernel,
                            dim3(grid_one_wave(maxpool_bwd_f32_kernel, B * sc.OH * sc.OW * 8, 256, 0)), dim3(256), 0, s,
                            static_cast<const float*>(gcur), m->mp_idx, B, sc.OH, sc.OW, 64, PH, PH,
                            static_cast<float*>(t1)));
  else
    DBS_CUDA_TRY(launch_pdl(maxpool_bwd_kernel, dim3(grid_one_wave(maxpool_bwd_kernel, B * sc.OH * sc.OW * 8, 256, 0)),
                            dim3(256), 0, s, static_cast<const uint16_t*>(gcur), m->mp_idx, B, sc.OH, sc.OW, 64, PH,
                            PH, static_cast<uint16_t*>(t1)));
  DBS_LAUNCH_CHECK();
  if ((st = bn_bwd(m, m->stem, pf, grad, t1, m->a[m->stem], B, t0, nullptr, s))) return st;
  return conv_wgrad(m, m->stem, t0, nullptr, B, grad, s);
}

int resnet_fwd_bwd(dbs_resnet* m, const void* wb, const float* pf, const void* x_any, const int32_t* y_base,
                   const int64_t* d_iter, int64_t B, float* grad, float* loss, cudaStream_t s) {
  DBS_REQUIRE(m && wb && pf && x_any && y_base && grad, DBS_ERR_ARGUMENT, "resnet: null argument");
  DBS_REQUIRE(B >= 1 && B <= m->max_b, DBS_ERR_ARGUMENT, "resnet: batch %lld outside [1, %lld]", (long long)B,
              (long long)m->max_b);
  if (m->arch == 50)
    return resnet50_fwd_bwd(m, wb, pf, static_cast<const uint8_t*>(x_any), y_base, d_iter, B, grad, loss, s);
  const float* x_base = static_cast<const float*>(x_any);
  const bool f32 = m->prec == DBS_PREC_F32;
  int st;
  DBS_CUDA_TRY(cudaMemsetAsync(grad, 0, sizeof(float) * m->P, s));
  DBS_CUDA_TRY(cudaMemsetAsync(m->stats_acc, 0, sizeof(double) * m->stats_len, s));
  // ---------------- forward ----------------
  if (f32)
    DBS_CUDA_TRY(launch_pdl(im2col_stem_f32_kernel, dim3(grid_one_wave(im2col_stem_f32_kernel, B * 1024, 256, 0)),
                            dim3(256), 0, s, x_base, d_iter, B, static_cast<float*>(m->stem_cols)));
  else
    DBS_CUDA_TRY(launch_pdl(im2col_stem_kernel, dim3(grid_one_wave(im2col_stem_kernel, B * 1024, 256, 0)), dim3(256),
                            0, s, x_base, d_iter, B, static_cast<uint16_t*>(m->stem_cols)));
  DBS_LAUNCH_CHECK();
  if ((st = conv_fwd(m, m->stem, nullptr, wb, B, s))) return st;
  if ((st = bn_apply(m, m->stem, pf, nullptr, -1, 1, B, m->a[m->stem], s))) return st;
  const void* x = m->a[m->stem];
  std::vector<const void*> blk_in(m->blocks.size());
  for (size_t i = 0; i < m->blocks.size(); i++) {
    const Block& b = m->blocks[i];
    blk_in[i] = x;
    if ((st = conv_fwd(m, b.c1, x, wb, B, s))) return st;
    if ((st = bn_apply(m, b.c1, pf, nullptr, -1, 1, B, m->a[b.c1], s))) return st;
    if ((st = conv_fwd(m, b.c2, m->a[b.c1], wb, B, s))) return st;
    if (b.ds >= 0) {
      if ((st = conv_fwd(m, b.ds, x, wb, B, s))) return st;
    }
    if ((st = bn_apply(m, b.c2, pf, b.ds >= 0 ? nullptr : x, b.ds, 1, B, m->blk_out[i], s))) return st;
    x = m->blk_out[i];
  }
  // ---------------- head ----------------
  void* gcur = m->g0;  // gradient w.r.t. the current block output
  if (f32)
    DBS_CUDA_TRY(launch_pdl(head_f32_kernel, dim3((unsigned)B), dim3(256), 0, s, static_cast<const float*>(x),
                            pf + m->fc_w, pf + m->fc_b, y_base, d_iter, B, m->classes, m->feat, m->dlog, m->loss_per,
                            static_cast<float*>(gcur)));
  else
    DBS_CUDA_TRY(launch_pdl(head_kernel, dim3((unsigned)B), dim3(256), 0, s, static_cast<const uint16_t*>(x),
                            pf + m->fc_w, pf + m->fc_b, y_base, d_iter, B, m->classes, m->feat, m->dlog, m->loss_per,
                            static_cast<uint16_t*>(gcur)));
  DBS_LAUNCH_CHECK();
  DBS_CUDA_TRY(launch_pdl(head_wgrad_kernel, dim3((m->classes * 512 + 255) / 256), dim3(256), 0, s, m->feat, m->dlog,
                          m->loss_per, B, m->classes, grad + m->fc_w, grad + m->fc_b, loss ? loss : m->loss_scratch,
                          loss ? d_iter : nullptr));
  DBS_LAUNCH_CHECK();
  // ---------------- backward through the blocks ----------------
  void* bufs[3] = {m->g1, m->g2, m->g3};
  for (int i = (int)m->blocks.size() - 1; i >= 0; i--) {
    const Block& b = m->blocks[i];
    const void* out = m->blk_out[i];
    // gradient w.r.t. the block input accumulates in gx (shortcut path first)
    void* gx = bufs[0];
    void* dy2 = bufs[1];
    void* tmp = bufs[2];
    // BN2 backward with the output ReLU mask; masked gradient g -> gx (identity) or tmp (ds)
    if ((st = bn_bwd(m, b.c2, pf, grad, gcur, out, B, dy2, b.ds >= 0 ? tmp : gx, s))) return st;
    void* dyd = gcur;  // gcur is free once tmp holds the masked gradient
    if (b.ds >= 0) {
      // BN_ds backward on the same masked gradient and the 1x1 stride-2 conv's weight gradient
      if ((st = bn_bwd(m, b.ds, pf, grad, tmp, nullptr, B, dyd, nullptr, s))) return st;
      if ((st = conv_wgrad(m, b.ds, dyd, blk_in[i], B, grad, s))) return st;
    }
    // conv2: wgrad (input a1) and dgrad -> da1 (tmp)
    if ((st = conv_wgrad(m, b.c2, dy2, m->a[b.c1], B, grad, s))) return st;
    if ((st = conv_dgrad(m, b.c2, dy2, wb, B, tmp, 0, s))) return st;
    // BN1 backward with the ReLU mask of a1 -> dy1 (dy2 buffer is free now)
    void* dy1 = dy2;
    if ((st = bn_bwd(m, b.c1, pf, grad, tmp, m->a[b.c1], B, dy1, nullptr, s))) return st;
    if ((st = conv_wgrad(m, b.c1, dy1, blk_in[i], B, grad, s))) return st;
    if (b.ds >= 0) {
      // the 3x3 stride-2 dgrad covers every input pixel; the 1x1 stride-2
      // shortcut dgrad (even pixels only) then accumulates onto it
      if ((st = conv_dgrad(m, b.c1, dy1, wb, B, gx, 0, s))) return st;
      if ((st = conv_dgrad(m, b.ds, dyd, wb, B, gx, 1, s))) return st;
    } else {
      if ((st = conv_dgrad(m, b.c1, dy1, wb, B, gx, 1, s))) return st;  // accumulate onto the shortcut gradient
    }
    // rotate: gx becomes the next gcur
    void* old = gcur;
    gcur = gx;
    bufs[0] = old;
  }
  // stem: BN backward with its ReLU mask, then the weight gradient only
  if ((st = bn_bwd(m, m->stem, pf, grad, gcur, m->a[m->stem], B, bufs[1], nullptr, s))) return st;
  if ((st = conv_wgrad(m, m->stem, bufs[1], nullptr, B, grad, s))) return st;
  return DBS_OK;
}

int resnet_param_count(const dbs_resnet* m) { return (int)m->P; }
int resnet_precision(const dbs_resnet* m) { return m->prec; }
int64_t resnet_row_bytes(const dbs_resnet* m) { return m->row_bytes; }

int iter_increment(int64_t* d_iter, cudaStream_t s) {
  iter_inc_kernel<<<1, 1, 0, s>>>(d_iter);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

}  // namespace dbs

extern "C" int dbs_dev_iter_increment(int64_t* d_iter, void* stream) {
  DBS_REQUIRE(d_iter, DBS_ERR_ARGUMENT, "iter_increment: null counter");
  return iter_increment(d_iter, as_stream(stream));
}

extern "C" int dbs_resnet_create_ex2(int32_t depth, int32_t image, int64_t max_batch, int32_t classes,
                                     int32_t precision, dbs_resnet** out) {
  DBS_REQUIRE(out && max_batch > 0, DBS_ERR_ARGUMENT, "resnet_create: need max_batch > 0");
  DBS_REQUIRE(precision == DBS_PREC_BF16 || precision == DBS_PREC_F32, DBS_ERR_ARGUMENT,
              "resnet_create: precision %d", precision);
  DBS_REQUIRE(out && max_batch > 0, DBS_ERR_ARGUMENT, "resnet_create: need max_batch > 0");
  DBS_REQUIRE((depth == 18 && image == 32 && classes >= 2 && classes <= 16) ||
                  (depth == 50 && image >= 64 && image % 32 == 0 && image <= 512 && classes >= 2 && classes <= 8192),
              DBS_ERR_ARGUMENT,
              "resnet_create: depth 18 needs a 32x32 image and 2..16 classes; depth 50 a multiple-of-32 image side "
              "in [64, 512] and 2..8192 classes (got depth %d, image %d, classes %d)",
              depth, image, classes);
  dbs_resnet* m = new dbs_resnet();
  m->max_b = max_batch;
  m->classes = classes;
  m->arch = depth;
  m->image = image;
  m->prec = precision;
  if (depth == 50) {
    m->row_bytes = (int64_t)3 * image * image;  // uint8 pixels
    m->stem_k = kStem7K;
    m->cpad = (classes + 7) & ~7;
    m->cpad32 = (classes + 31) & ~31;
    build_layers50(m);
  } else {
    build_layers(m);
  }
  int st = alloc_all(m);
  if (st) {
    dbs_resnet_destroy(m);
    return st;
  }
  *out = m;
  return DBS_OK;
}

extern "C" int dbs_resnet_create_ex(int32_t depth, int32_t image, int64_t max_batch, int32_t classes,
                                    dbs_resnet** out) {
  return dbs_resnet_create_ex2(depth, image, max_batch, classes, DBS_PREC_BF16, out);
}

extern "C" int dbs_resnet_create(int64_t max_batch, int32_t classes, dbs_resnet** out) {
  return dbs_resnet_create_ex2(18, 32, max_batch, classes, DBS_PREC_BF16, out);
}

// BN running statistics of conv `conv` (f32 mode): [cout] mean then [cout] unbiased variance
extern "C" int dbs_resnet_running_stats(const dbs_resnet* m, int32_t conv, float** d_stats, int32_t* channels) {
  DBS_REQUIRE(m && conv >= 0 && conv < (int32_t)m->convs.size() && d_stats, DBS_ERR_ARGUMENT,
              "resnet_running_stats: bad conv index");
  *d_stats = m->run_stats + m->run_off[conv];
  if (channels) *channels = m->convs[conv].cout;
  return DBS_OK;
}

extern "C" int dbs_resnet_precision(const dbs_resnet* m, int32_t* precision) {
  DBS_REQUIRE(m && precision, DBS_ERR_ARGUMENT, "resnet_precision: null");
  *precision = m->prec;
  return DBS_OK;
}

extern "C" int dbs_resnet_info(const dbs_resnet* m, int32_t* depth, int32_t* image, int64_t* row_bytes,
                               int32_t* stem_k) {
  DBS_REQUIRE(m, DBS_ERR_ARGUMENT, "resnet_info: null");
  if (depth) *depth = m->arch;
  if (image) *image = m->image;
  if (row_bytes) *row_bytes = m->row_bytes;
  if (stem_k) *stem_k = m->stem_k;
  return DBS_OK;
}

extern "C" int dbs_resnet_destroy(dbs_resnet* m) {
  if (!m) return DBS_OK;
  cudaFree(m->stem_cols);
  for (auto p : m->y) cudaFree(p);
  for (auto p : m->a) cudaFree(p);
  for (auto p : m->blk_out) cudaFree(p);
  for (auto p : m->mean) cudaFree(p);
  for (auto p : m->invstd) cudaFree(p);
  cudaFree(m->stats_acc);
  cudaFree(m->g0);
  cudaFree(m->g1);
  cudaFree(m->g2);
  cudaFree(m->g3);
  cudaFree(m->feat);
  cudaFree(m->dlog);
  cudaFree(m->loss_per);
  cudaFree(m->loss_scratch);
  cudaFree(m->g4);
  cudaFree(m->mp_out);
  cudaFree(m->mp_idx);
  cudaFree(m->feat_b);
  cudaFree(m->logits);
  cudaFree(m->dlog_f);
  cudaFree(m->dlog_b);
  cudaFree(m->dfeat);
  cudaFree(m->run_stats);
  delete m;
  return DBS_OK;
}

extern "C" int dbs_resnet_param_count(const dbs_resnet* m, int64_t* P) {
  DBS_REQUIRE(m && P, DBS_ERR_ARGUMENT, "resnet_param_count: null");
  *P = m->P;
  return DBS_OK;
}

extern "C" int dbs_resnet_param_table(const dbs_resnet* m, int64_t* off, int64_t* len, int32_t* kind,
                                      int32_t capacity, int32_t* count) {
  DBS_REQUIRE(m && count, DBS_ERR_ARGUMENT, "resnet_param_table: null");
  *count = (int32_t)m->t_off.size();
  DBS_REQUIRE(capacity >= *count && off && len && kind, DBS_ERR_ARGUMENT, "resnet_param_table: capacity %d < %d",
              capacity, *count);
  for (size_t i = 0; i < m->t_off.size(); i++) {
    off[i] = m->t_off[i];
    len[i] = m->t_len[i];
    kind[i] = m->t_kind[i];
  }
  return DBS_OK;
}

extern "C" int dbs_resnet_forward_backward(dbs_resnet* m, const void* d_params_shadow, const float* d_params,
                                           const void* d_x, const int32_t* d_labels, int64_t batch,
                                           const int64_t* d_iter, float* d_grad, float* d_loss, void* stream) {
  return resnet_fwd_bwd(m, d_params_shadow, d_params, d_x, d_labels, d_iter, batch, d_grad, d_loss, as_stream(stream));
}

// ---- standalone convolution entry points (unit tests / other models) ----
static Conv make_conv(int N, int H, int W, int Cin, int Cout, int k, int stride, int pad) {
  (void)N;
  Conv c{};
  c.cin = Cin;
  c.cout = Cout;
  c.k = k;
  c.stride = stride;
  c.pad = pad;
  c.H = H;
  c.W = W;
  c.OH = (H + 2 * pad - k) / stride + 1;
  c.OW = (W + 2 * pad - k) / stride + 1;
  return c;
}

extern "C" int dbs_dev_conv2d_fwd(const void* d_x, int32_t N, int32_t H, int32_t W, int32_t Cin, const void* d_w,
                                  int32_t Cout, int32_t k, int32_t stride, int32_t pad, void* d_y, void* stream) {
  DBS_REQUIRE(Cin % 64 == 0 && Cout % 8 == 0, DBS_ERR_ARGUMENT, "conv2d_fwd: Cin %% 64 and Cout %% 8 required");
  const Conv c = make_conv(N, H, W, Cin, Cout, k, stride, pad);
  ConvCall call{};
  call.M = (int64_t)N * c.OH * c.OW;
  call.N = Cout;
  call.K = (int64_t)k * k * Cin;
  call.a_mode = 2;
  call.a = d_x;
  call.ta = nhwc(N, H, W, Cin);
  call.ga = ConvGeom{k, k, Cin / 64, stride, pad, c.OH, c.OW, Cin};
  call.b_mode = 0;
  call.b = d_w;
  call.ldb = call.K;
  call.epi = DBS_EPI_BF16;
  call.d = d_y;
  call.ldd = Cout;
  call.halo = halo_ok(c);
  return conv_gemm(call, as_stream(stream));
}

extern "C" int dbs_dev_conv2d_dgrad(const void* d_dy, int32_t N, int32_t H, int32_t W, int32_t Cin, const void* d_w,
                                    int32_t Cout, int32_t k, int32_t stride, int32_t pad, void* d_dx, void* d_scratch,
                                    void* stream) {
  DBS_REQUIRE(Cin % 8 == 0 && Cout % 64 == 0 && (stride == 1 || stride == 2) && pad == k / 2, DBS_ERR_ARGUMENT,
              "conv2d_dgrad: Cout %% 64, stride 1/2, same padding required");
  const Conv c = make_conv(N, H, W, Cin, Cout, k, stride, pad);
  (void)d_scratch;  // no scratch since the stride-2 path runs per parity class
  return conv_dgrad_ex(c, static_cast<const uint16_t*>(d_dy), static_cast<const uint16_t*>(d_w), N,
                       static_cast<uint16_t*>(d_dx), 0, as_stream(stream));
}

// Stand-alone fp32-class BatchNorm passes (the kernels the network runs; for unit tests
// and the bench's per-kernel HBM rooflines).  Forward: batch statistics from the conv
// epilogue's fp64 column sums acc [sum C | sum of squares C] -> mean / invstd, out (S32)
// = act(gamma (y - mean) invstd + beta).  Backward: g (fp32; zeroed where the S32 ReLU
// output `mask` is not positive, when given) -> dbeta += sum g, dgamma += sum g yhat,
// dy (S32) = the BatchNorm input gradient, g_out (fp32, optional) = the masked g.
extern "C" int dbs_dev_bn_apply_s32(const float* d_y, const double* d_acc, const float* d_gamma, const float* d_beta,
                                    int32_t C, int64_t M, int32_t relu, float* d_mean, float* d_invstd, float* d_out,
                                    void* stream) {
  DBS_REQUIRE(d_y && d_acc && d_gamma && d_beta && d_mean && d_invstd && d_out && C % 32 == 0 && C <= 2048 && M > 0,
              DBS_ERR_ARGUMENT, "bn_apply_s32: C %% 32 == 0, C <= 2048, M > 0");
  cudaStream_t s = as_stream(stream);
  const int64_t total = M * (C / 8);
  const size_t smem = (size_t)2 * C * sizeof(float);
  DBS_CUDA_TRY(launch_pdl(bn_apply_f32_kernel, dim3(grid_one_wave(bn_apply_f32_kernel, total, 256, smem)), dim3(256),
                          smem, s, d_y, d_acc, d_mean, d_invstd, d_gamma, d_beta, static_cast<const float*>(nullptr),
                          static_cast<const float*>(nullptr), static_cast<const double*>(nullptr),
                          static_cast<float*>(nullptr), static_cast<float*>(nullptr),
                          static_cast<const float*>(nullptr), static_cast<const float*>(nullptr), relu, (int)C, M,
                          d_out, static_cast<float*>(nullptr), static_cast<float*>(nullptr), 0.0f));
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

extern "C" int dbs_dev_bn_backward_s32(const float* d_g, const float* d_mask, const float* d_y, const float* d_mean,
                                       const float* d_invstd, const float* d_gamma, int32_t C, int64_t M,
                                       float* d_dgamma, float* d_dbeta, float* d_dy, float* d_gout, void* stream) {
  DBS_REQUIRE(d_g && d_y && d_mean && d_invstd && d_gamma && d_dgamma && d_dbeta && d_dy && C % 32 == 0 &&
                  C <= 2048 && M > 0,
              DBS_ERR_ARGUMENT, "bn_backward_s32: C %% 32 == 0, C <= 2048, M > 0");
  cudaStream_t s = as_stream(stream);
  const int cv = C / 8;
  const int rows_per_pass = 256 / cv;
  DBS_REQUIRE(rows_per_pass >= 1, DBS_ERR_ARGUMENT, "bn_backward_s32: C too large");
  int blocks = (int)((M + rows_per_pass - 1) / rows_per_pass);
  const int cap = current_sm_count() * resident_per_sm(bn_bwd_reduce_f32_kernel, 256, 0);
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  DBS_CUDA_TRY(launch_pdl(bn_bwd_reduce_f32_kernel, dim3(blocks), dim3(256), 0, s, d_g, d_mask, d_y, d_mean, d_invstd,
                          (int)C, M, d_dgamma, d_dbeta));
  DBS_LAUNCH_CHECK();
  const int64_t total = M * cv;
  const size_t smem = (size_t)3 * C * sizeof(float);
  DBS_CUDA_TRY(launch_pdl(bn_bwd_apply_f32_kernel, dim3(grid_one_wave(bn_bwd_apply_f32_kernel, total, 256, smem)),
                          dim3(256), smem, s, d_g, d_mask, d_y, d_mean, d_invstd, d_gamma,
                          static_cast<const float*>(d_dgamma), static_cast<const float*>(d_dbeta), (int)C, M, d_dy,
                          d_gout));
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

// fp32-class (3xTF32) forms: S32 x / w / dy operands (rows of 32-multiples), fp32 outputs
extern "C" int dbs_dev_conv2d_fwd_s32(const void* d_x, int32_t N, int32_t H, int32_t W, int32_t Cin, const void* d_w,
                                      int32_t Cout, int32_t k, int32_t stride, int32_t pad, float* d_y, void* stream) {
  DBS_REQUIRE(Cin % 32 == 0 && Cout % 32 == 0, DBS_ERR_ARGUMENT, "conv2d_fwd_s32: Cin, Cout multiples of 32");
  const Conv c = make_conv(N, H, W, Cin, Cout, k, stride, pad);
  ConvCall call{};
  call.tf = 1;
  call.M = (int64_t)N * c.OH * c.OW;
  call.N = Cout;
  call.K = (int64_t)k * k * Cin;
  call.b_mode = 0;
  call.b = d_w;
  call.ldb = call.K;
  if (k == 1 && stride == 1) {
    call.a_mode = 0;
    call.a = d_x;
    call.lda = Cin;
  } else {
    call.a_mode = 2;
    call.a = d_x;
    call.ta = nhwc(N, H, W, Cin);
    call.ga = ConvGeom{k, k, Cin / 32, stride, pad, c.OH, c.OW, Cin};
    call.halo = halo_tf_ok(c);
  }
  call.epi = DBS_EPI_F32;
  call.d = d_y;
  call.ldd = Cout;
  return conv_gemm(call, as_stream(stream));
}

extern "C" int dbs_dev_conv2d_dgrad_s32(const void* d_dy, int32_t N, int32_t H, int32_t W, int32_t Cin,
                                        const void* d_w, int32_t Cout, int32_t k, int32_t stride, int32_t pad,
                                        float* d_dx, void* stream) {
  DBS_REQUIRE(Cin % 32 == 0 && Cout % 32 == 0 && (stride == 1 || stride == 2) && pad == k / 2, DBS_ERR_ARGUMENT,
              "conv2d_dgrad_s32: Cin, Cout %% 32, stride 1/2, same padding required");
  const Conv c = make_conv(N, H, W, Cin, Cout, k, stride, pad);
  return conv_dgrad_ex(c, d_dy, d_w, N, d_dx, 0, as_stream(stream), true);
}

extern "C" int dbs_dev_conv2d_wgrad_s32(const void* d_dy, const void* d_x, int32_t N, int32_t H, int32_t W,
                                        int32_t Cin, int32_t Cout, int32_t k, int32_t stride, int32_t pad, float* d_dw,
                                        void* stream) {
  DBS_REQUIRE(Cin % 32 == 0 && Cout % 32 == 0, DBS_ERR_ARGUMENT, "conv2d_wgrad_s32: Cin, Cout %% 32 required");
  const Conv c = make_conv(N, H, W, Cin, Cout, k, stride, pad);
  return conv_wgrad_ex(c, d_dy, d_x, N, d_dw, as_stream(stream), true);
}

extern "C" int dbs_dev_conv2d_wgrad(const void* d_dy, const void* d_x, int32_t N, int32_t H, int32_t W, int32_t Cin,
                                    int32_t Cout, int32_t k, int32_t stride, int32_t pad, float* d_dw, void* stream) {
  DBS_REQUIRE(Cin % 64 == 0 && Cout % 8 == 0, DBS_ERR_ARGUMENT, "conv2d_wgrad: Cin %% 64 required");
  const Conv c = make_conv(N, H, W, Cin, Cout, k, stride, pad);
  return conv_wgrad_ex(c, static_cast<const uint16_t*>(d_dy), static_cast<const uint16_t*>(d_x), N, d_dw,
                       as_stream(stream));
}

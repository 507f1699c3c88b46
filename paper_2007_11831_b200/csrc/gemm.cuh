// gemm.cuh -- internal interface of the tcgen05 GEMM / implicit-GEMM conv.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace dbs {

// Geometry of a conv-mode operand: output feature map OH x OW, filter R x S,
// stride / pad, and (A) the channel blocks of 64 per (r, s) or (B, weight
// gradient) the channel count Cin that splits N = (r, s, c).
struct ConvGeom {
  int R, S, cblocks;
  int stride, pad;
  int OH, OW;
  int Cin;
};

// NHWC bf16 tensor extents
struct ConvTensor {
  int N, H, W, C;
};

// Explicit tap list of a conv-mode A operand (the stride-2 input gradient,
// one GEMM per output parity class): per tap the A window offset on the input
// grid and the filter slice (r * S + s) read by B mode 3.  n = 0: the R x S
// window of ConvGeom.
struct ConvTaps {
  int n;
  int8_t dh[9], dw[9];
  uint8_t rs[9];
};

// Strided output rows: GEMM row (img, i, j) of an OH x OW grid is written to
// output pixel (img, 2i + a, 2j + b) of an H x W map.  on = 0: row-major rows.
struct OutMap {
  int on;
  int H, W, a, b, OH, OW;
};

struct ConvCall {
  int64_t M, N, K;
  int a_mode, b_mode;        // 0 K-major 2-D, 1 MN-major 2-D, 2 conv 4-D;
                             // A 5: the conv input as an MN-major A [k = pixel][m = (r, s, c)] (weight gradient)
  const void* a;
  int64_t lda;
  ConvTensor ta;
  ConvGeom ga;
  const void* b;
  int64_t ldb;
  ConvTensor tb;
  ConvGeom gb;
  int epi;
  void* d;
  int64_t ldd;
  const float* bias;
  const uint16_t* aux;
  double* sum_part;          // BN batch statistics: [N] fp64 accumulators of sum / sum of squares
  double* sq_part;
  int splits;                // split-K slices (atomic epilogue)
  int bn_override;           // force the N tile (0 = auto)
  ConvTaps taps;
  OutMap omap;
  int halo;                  // 3x3 stride-1 64->64 conv: resident filter + halo rows (gemm.cu HaloCfg)
  // merged stride-2 input gradient: nclass output-parity classes in ONE launch, each
  // a full M-row GEMM with its own tap list / output map (taps, omap unused then)
  int nclass;
  ConvTaps cls_taps[4];
  OutMap cls_omap[4];
  int d_trans;               // F32 atomic epilogue writes D transposed: d[n * ldd + m]
  // S32 operands (3xTF32, fp32-class): tensors / channel counts / ld are logical,
  // the operands are in the S32 format of dbs_dev_gemm_tf32x3; ConvGeom.cblocks
  // counts 32-channel blocks.  No halo / pairing / transposed-wgrad variants.
  int tf;
};

int gemm_bf16(const void* a, int a_mn, int64_t lda, const void* b, int b_mn, int64_t ldb, void* d, int64_t ldd,
              int64_t M, int64_t N, int64_t K, int epi, const float* bias, const void* aux, cudaStream_t s,
              float* colsum_part);
int conv_gemm(const ConvCall& c, cudaStream_t s);
// plain GEMM with S32 operands (lda / ldb / ldd logical, multiples of 32)
int gemm_tf(const void* a, int a_mn, int64_t lda, const void* b, int b_mn, int64_t ldb, void* d, int64_t ldd,
            int64_t M, int64_t N, int64_t K, int epi, const float* bias, const void* aux, cudaStream_t s,
            float* colsum_part = nullptr);
int preload_gemm();
// the halo variant's one-box-per-tile input halo fits its shared-memory slot
bool halo_fits(int OH, int OW);
bool halo_tf_fits(int OH, int OW);  // fp32-class halo variant (gemm.cu HaloTfCfg)
// SMs of the current (possibly green) context -- what a launch issued now can use
int current_sm_count();

}  // namespace dbs

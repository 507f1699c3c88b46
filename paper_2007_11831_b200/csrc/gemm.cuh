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

struct ConvCall {
  int64_t M, N, K;
  int a_mode, b_mode;        // 0 K-major 2-D, 1 MN-major 2-D, 2 conv 4-D
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
  int splits;                // split-K CTAs along grid.z (atomic epilogue)
  int bn_override;           // force the N tile (0 = auto)
};

int gemm_bf16(const void* a, int a_mn, int64_t lda, const void* b, int b_mn, int64_t ldb, void* d, int64_t ldd,
              int64_t M, int64_t N, int64_t K, int epi, const float* bias, const void* aux, cudaStream_t s,
              float* colsum_part);
int conv_gemm(const ConvCall& c, cudaStream_t s);
int preload_gemm();
// SMs of the current (possibly green) context -- what a launch issued now can use
int current_sm_count();

}  // namespace dbs

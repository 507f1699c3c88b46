// s32.cu -- the S32 operand format of the fp32-class ("3xTF32") tensor-core path.
//
// A logical fp32 row-major matrix [rows][ld] (ld % 32 == 0) is stored as, per
// 32-element block of a row, 32 "hi" floats then 32 "lo" floats:
//   hi = rn_tf32(x), lo = rn_tf32(x - hi)
// Both parts are exact tf32 values (kind::tf32 MMAs read them without further
// rounding) and hi + lo reproduces x to ~2^-23 |x|, so the three MMA passes
// hi*hi + hi*lo + lo*hi of gemm.cu (produce_tf) form fp32-accurate products --
// the arithmetic class of the reference's numpy fp64 / the reference arm's fp32
// (sgdlab.py:200-238).  These kernels convert plain fp32 <-> S32 (inputs, tests).
#include "common.cuh"

namespace dbs {
namespace {

__device__ __forceinline__ float rn_tf32(float x) {
  const uint32_t u = __float_as_uint(x);
  return __uint_as_float((u + 0xFFFu + ((u >> 13) & 1u)) & 0xFFFFE000u);
}

// one thread per 4 logical columns of a row (a quarter of a float4 pair)
__global__ void split_s32_kernel(const float* __restrict__ x, int64_t rows, int64_t cols, int64_t ld_in,
                                 float* __restrict__ out, int64_t ld_out) {
  pdl_trigger_and_wait();
  const int64_t q = ld_out / 4;  // quads per row
  const int64_t total = rows * q;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / q;
    const int64_t c = (i - r * q) * 4;
    float v[4], h[4], l[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      v[u] = (c + u < cols) ? x[r * ld_in + c + u] : 0.0f;
      h[u] = rn_tf32(v[u]);
      l[u] = rn_tf32(v[u] - h[u]);
    }
    float* o = out + r * 2 * ld_out + (c / 32) * 64 + (c % 32);
    *reinterpret_cast<float4*>(o) = make_float4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<float4*>(o + 32) = make_float4(l[0], l[1], l[2], l[3]);
  }
}

__global__ void join_s32_kernel(const float* __restrict__ s, int64_t rows, int64_t cols, int64_t ld_in,
                                float* __restrict__ x, int64_t ld_out) {
  pdl_trigger_and_wait();
  const int64_t total = rows * cols;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols;
    const int64_t c = i - r * cols;
    const float* b = s + r * 2 * ld_in + (c / 32) * 64 + (c % 32);
    x[r * ld_out + c] = b[0] + b[32];
  }
}

int grid_for(int64_t n) {
  const int64_t b = (n + 255) / 256;
  const int64_t cap = (int64_t)current_sm_count() * 8;
  return (int)(b < 1 ? 1 : (b < cap ? b : cap));
}

}  // namespace

int split_s32(const float* x, int64_t rows, int64_t cols, int64_t ld_in, float* out, int64_t ld_out,
              cudaStream_t s) {
  DBS_REQUIRE(x && out && rows >= 0 && cols >= 0 && ld_in >= cols && ld_out >= cols && ld_out % 32 == 0 &&
                  ((uintptr_t)out & 15) == 0,
              DBS_ERR_ARGUMENT, "split_s32: bad shape (ld_out %% 32 == 0, 16-byte aligned output)");
  if (rows == 0 || ld_out == 0) return DBS_OK;
  DBS_CUDA_TRY(launch_pdl(split_s32_kernel, dim3(grid_for(rows * ld_out / 4)), dim3(256), 0, s, x, rows, cols, ld_in,
                          out, ld_out));
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

int join_s32(const float* s32, int64_t rows, int64_t cols, int64_t ld_in, float* x, int64_t ld_out,
             cudaStream_t s) {
  DBS_REQUIRE(s32 && x && rows >= 0 && cols >= 0 && ld_in >= cols && ld_in % 32 == 0 && ld_out >= cols,
              DBS_ERR_ARGUMENT, "join_s32: bad shape");
  if (rows == 0 || cols == 0) return DBS_OK;
  DBS_CUDA_TRY(launch_pdl(join_s32_kernel, dim3(grid_for(rows * cols)), dim3(256), 0, s, s32, rows, cols, ld_in, x,
                          ld_out));
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

}  // namespace dbs

extern "C" int dbs_dev_split_s32(const float* d_x, int64_t rows, int64_t cols, int64_t ld_in, float* d_s32,
                                 int64_t ld_out, void* stream) {
  return dbs::split_s32(d_x, rows, cols, ld_in, d_s32, ld_out, dbs::as_stream(stream));
}

extern "C" int dbs_dev_join_s32(const float* d_s32, int64_t rows, int64_t cols, int64_t ld_in, float* d_x,
                                int64_t ld_out, void* stream) {
  return dbs::join_s32(d_s32, rows, cols, ld_in, d_x, ld_out, dbs::as_stream(stream));
}

// gather.cu -- coalesced repartition gather (HBM-bound).
//
// The reference gathers sample rows by index inside every gradient call
// (offsets[idx] sgdlab.py:82, features[idx] sgdlab.py:144).  On the B200 the
// epoch's permuted sample order is applied ONCE per epoch: each worker's shard
// is repacked contiguously in HBM so every iteration reads a dense slice.
//
// Algorithmic bytes per row: 2 * row_bytes (+ 8 B of index).  Mapping: one warp
// per row (several rows per CTA, grid-stride over rows), 32-byte vector loads
// and stores (LDG/STG.256) with 4 independent requests in flight per lane; rows
// that are not 32-byte aligned fall back to 16-byte, 4-byte or byte copies.
#include "common.cuh"

namespace dbs {
namespace {

constexpr int kWarpsPerBlock = 8;
constexpr int kUnroll = 4;

__device__ __forceinline__ int4 ld_stream(const int4* p) { return __ldcs(p); }
__device__ __forceinline__ int ld_stream(const int* p) { return __ldcs(p); }
__device__ __forceinline__ V8 ld_stream(const V8* p) { return ldg8_cs(p); }
__device__ __forceinline__ void st_stream(int4* p, const int4& v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(int* p, const int& v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(V8* p, const V8& v) { stg8_cs(p, v); }

template <typename V>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    gather_rows_kernel(const V* __restrict__ src, const int64_t* __restrict__ idx, int64_t rows,
                       int64_t vec_per_row, V* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * kWarpsPerBlock;
  for (int64_t r = warp; r < rows; r += nwarps) {
    const V* s = src + __ldg(&idx[r]) * vec_per_row;
    V* d = dst + r * vec_per_row;
    int64_t c = lane;
    for (; c + 32 * (kUnroll - 1) < vec_per_row; c += 32 * kUnroll) {
      V v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; u++) v[u] = ld_stream(s + c + 32 * u);
#pragma unroll
      for (int u = 0; u < kUnroll; u++) st_stream(d + c + 32 * u, v[u]);
    }
    for (; c < vec_per_row; c += 32) st_stream(d + c, ld_stream(s + c));
  }
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    gather_bytes_kernel(const unsigned char* __restrict__ src, const int64_t* __restrict__ idx,
                        int64_t rows, int64_t row_bytes, unsigned char* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * kWarpsPerBlock;
  for (int64_t r = warp; r < rows; r += nwarps) {
    const unsigned char* s = src + idx[r] * row_bytes;
    unsigned char* d = dst + r * row_bytes;
    for (int64_t c = lane; c < row_bytes; c += 32) d[c] = s[c];
  }
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  // round-to-nearest-even, like __float2bfloat16_rn
  uint32_t ua = __float_as_uint(a), ub = __float_as_uint(b);
  ua = (ua + 0x7FFFu + ((ua >> 16) & 1u)) >> 16;
  ub = (ub + 0x7FFFu + ((ub >> 16) & 1u)) >> 16;
  return ua | (ub << 16);
}

// fp32 rows of `cols` (cols % 4 == 0) -> bf16 rows.
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    gather_f32_bf16_kernel(const float4* __restrict__ src, const int64_t* __restrict__ idx,
                           int64_t rows, int64_t vec_per_row, uint2* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * kWarpsPerBlock;
  for (int64_t r = warp; r < rows; r += nwarps) {
    const float4* s = src + __ldg(&idx[r]) * vec_per_row;
    uint2* d = dst + r * vec_per_row;
    for (int64_t c = lane; c < vec_per_row; c += 32) {
      float4 v = __ldcs(s + c);
      d[c] = make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
    }
  }
}

__device__ __forceinline__ float rn_tf32(float x) {
  const uint32_t u = __float_as_uint(x);
  return __uint_as_float((u + 0xFFFu + ((u >> 13) & 1u)) & 0xFFFFE000u);
}

// fp32 rows of `cols` (cols % 4 == 0) -> S32 rows of ld_out (ld_out % 32 == 0, pad columns
// zero): the fp32-class operand format (s32.cu), written once per epoch with the repack
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    gather_f32_s32_kernel(const float4* __restrict__ src, const int64_t* __restrict__ idx, int64_t rows,
                          int64_t vec_per_row, int64_t ld_out, float* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * kWarpsPerBlock;
  const int64_t q_out = ld_out / 4;
  for (int64_t r = warp; r < rows; r += nwarps) {
    const float4* s = src + __ldg(&idx[r]) * vec_per_row;
    float* d = dst + r * 2 * ld_out;
    for (int64_t c = lane; c < q_out; c += 32) {
      const float4 v = c < vec_per_row ? __ldcs(s + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 h = make_float4(rn_tf32(v.x), rn_tf32(v.y), rn_tf32(v.z), rn_tf32(v.w));
      const int64_t e = 4 * c;
      float* o = d + 2 * (e & ~int64_t(31)) + (e & 31);
      __stcs(reinterpret_cast<float4*>(o), h);
      __stcs(reinterpret_cast<float4*>(o + 32),
             make_float4(rn_tf32(v.x - h.x), rn_tf32(v.y - h.y), rn_tf32(v.z - h.z), rn_tf32(v.w - h.w)));
    }
  }
}

__global__ void gather_i32_kernel(const int32_t* __restrict__ src, const int64_t* __restrict__ idx,
                                  int64_t rows, int32_t* __restrict__ dst) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x)
    dst[r] = src[idx[r]];
}

int grid_for_rows(int64_t rows) {
  int64_t blocks = (rows + kWarpsPerBlock - 1) / kWarpsPerBlock;
  int64_t cap = (int64_t)num_sms() * 8;  // 8 CTAs x 8 warps = 64 warps per SM
  return (int)(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

}  // namespace
}  // namespace dbs

using namespace dbs;

extern "C" int dbs_dev_gather_rows(const void* d_src, const int64_t* d_idx, int64_t rows,
                                   int64_t row_bytes, void* d_dst, void* stream) {
  DBS_REQUIRE(rows >= 0 && row_bytes >= 0 && (rows == 0 || (d_src && d_idx && d_dst)),
              DBS_ERR_ARGUMENT, "dbs_dev_gather_rows: bad arguments");
  if (rows == 0 || row_bytes == 0) return DBS_OK;
  cudaStream_t s = as_stream(stream);
  const int grid = grid_for_rows(rows);
  const uintptr_t align = (uintptr_t)d_src | (uintptr_t)d_dst;
  if (row_bytes % 32 == 0 && align % 32 == 0) {
    gather_rows_kernel<V8><<<grid, kWarpsPerBlock * 32, 0, s>>>((const V8*)d_src, d_idx, rows, row_bytes / 32,
                                                                (V8*)d_dst);
  } else if (row_bytes % 16 == 0 && align % 16 == 0) {
    gather_rows_kernel<int4><<<grid, kWarpsPerBlock * 32, 0, s>>>(
        (const int4*)d_src, d_idx, rows, row_bytes / 16, (int4*)d_dst);
  } else if (row_bytes % 4 == 0 && align % 4 == 0) {
    gather_rows_kernel<int><<<grid, kWarpsPerBlock * 32, 0, s>>>((const int*)d_src, d_idx, rows,
                                                                 row_bytes / 4, (int*)d_dst);
  } else {
    gather_bytes_kernel<<<grid, kWarpsPerBlock * 32, 0, s>>>(
        (const unsigned char*)d_src, d_idx, rows, row_bytes, (unsigned char*)d_dst);
  }
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

extern "C" int dbs_dev_gather_rows_f32_bf16(const float* d_src, const int64_t* d_idx, int64_t rows,
                                            int64_t cols, void* d_dst, void* stream) {
  DBS_REQUIRE(rows >= 0 && cols % 4 == 0 && ((uintptr_t)d_src % 16 == 0) &&
                  ((uintptr_t)d_dst % 8 == 0),
              DBS_ERR_ARGUMENT, "dbs_dev_gather_rows_f32_bf16: cols must be a multiple of 4, aligned");
  if (rows == 0 || cols == 0) return DBS_OK;
  gather_f32_bf16_kernel<<<grid_for_rows(rows), kWarpsPerBlock * 32, 0, as_stream(stream)>>>(
      (const float4*)d_src, d_idx, rows, cols / 4, (uint2*)d_dst);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

extern "C" int dbs_dev_gather_rows_f32_s32(const float* d_src, const int64_t* d_idx, int64_t rows, int64_t cols,
                                           float* d_dst, int64_t ld_out, void* stream) {
  DBS_REQUIRE(rows >= 0 && cols % 4 == 0 && ld_out >= cols && ld_out % 32 == 0 && ((uintptr_t)d_src % 16 == 0) &&
                  ((uintptr_t)d_dst % 16 == 0),
              DBS_ERR_ARGUMENT, "dbs_dev_gather_rows_f32_s32: cols %% 4, ld_out %% 32 >= cols, aligned buffers");
  if (rows == 0 || cols == 0) return DBS_OK;
  gather_f32_s32_kernel<<<grid_for_rows(rows), kWarpsPerBlock * 32, 0, as_stream(stream)>>>(
      (const float4*)d_src, d_idx, rows, cols / 4, ld_out, d_dst);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

extern "C" int dbs_dev_gather_i32(const int32_t* d_src, const int64_t* d_idx, int64_t rows,
                                  int32_t* d_dst, void* stream) {
  DBS_REQUIRE(rows >= 0, DBS_ERR_ARGUMENT, "dbs_dev_gather_i32: bad rows");
  if (rows == 0) return DBS_OK;
  int grid = (int)((rows + 255) / 256);
  if (grid > num_sms() * 4) grid = num_sms() * 4;
  gather_i32_kernel<<<grid, 256, 0, as_stream(stream)>>>(d_src, d_idx, rows, d_dst);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

// Dev probe: where does a cta_group::1 M=64 tcgen05.mma put its 64 accumulator
// rows in TMEM?  A[64][16] has row i = i (constant along K), B = ones -> D[i][n] = 16 i.
// Each of the 4 warps reads its 32-lane quadrant (32x32b.x32) and reports, per lane,
// the value / 16 found in column 0 (-1: zero / unwritten).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2007_11831_b200/csrc \
//        scripts/m64_layout.cu -o scripts/_bin/m64_layout
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdio.h>

#include "tcgen05.cuh"

using namespace dbs::sm100;

__global__ void __launch_bounds__(128, 1) k(float* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;            // 64 rows x 128 B (K-major, SW128): only K 0..15 used
  uint8_t* sB = sm + 8192;     // 256 rows x 128 B
  __shared__ uint64_t done;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // fill A (swizzled 128B rows: 16-byte chunk j of row r lives at chunk j ^ (r & 7))
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) {
    const int r = i / 64, kk = i % 64;
    const int chunk = (kk / 8) ^ (r & 7);
    const float v = (kk < 16) ? (float)r : 0.0f;
    __nv_bfloat16* p = reinterpret_cast<__nv_bfloat16*>(sA + r * 128 + chunk * 16) + (kk % 8);
    *p = __float2bfloat16(v);
  }
  for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x) {
    const int r = i / 64, kk = i % 64;
    const int chunk = (kk / 8) ^ (r & 7);
    __nv_bfloat16* p = reinterpret_cast<__nv_bfloat16*>(sB + r * 128 + chunk * 16) + (kk % 8);
    *p = __float2bfloat16(kk < 16 ? 1.0f : 0.0f);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<256>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc_bf16(64, 256, 0, 0);
    mma_bf16_ss(tmem, make_sdesc(smem_u32(sA), 16, 1024), make_sdesc(smem_u32(sB), 16, 1024), idesc, 0u);
    mma_commit(&done);
  }
  __syncwarp();
  mbar_wait(&done, 0);
  tc_fence_after();
  uint32_t r[32];
  tmem_ld_32x32b_x32(tmem + ((uint32_t)(warp * 32) << 16), r);
  tmem_ld_wait();
  const float v = __uint_as_float(r[0]);
  out[warp * 32 + lane] = (v == 0.0f && !(warp == 0 && lane == 0)) ? -1.0f : v / 16.0f;
  out[128 + warp * 32 + lane] = __uint_as_float(r[31]) / 16.0f;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tmem);
}

int main() {
  float* d;
  cudaMalloc(&d, 256 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  k<<<1, 128, 48 * 1024>>>(d);
  printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  float h[256];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  for (int w = 0; w < 4; w++) {
    printf("lanes %3d..%3d col0:", 32 * w, 32 * w + 31);
    for (int l = 0; l < 32; l++) printf(" %g", h[w * 32 + l]);
    printf("\n");
  }
  printf("col31 of lanes 0..31:");
  for (int l = 0; l < 32; l++) printf(" %g", h[128 + l]);
  printf("\n");
  return 0;
}

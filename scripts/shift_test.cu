// Dev probe: can a tcgen05.mma K-major SWIZZLE_128B A operand start at a row
// that is not 1024-byte aligned (a 1-row shift of a TMA-written tile)?
//   D = A[s : s + 128] * B^T   for s = 0..8, A written once by TMA as [136][64]
// variant 0: plain start address; variant 1: + descriptor base offset (bits 49-51)
// = (start >> 7) & 7; variant 2: the base offset field only (start unchanged).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2007_11831_b200/csrc \
//        scripts/shift_test.cu -o scripts/_bin/shift_test
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#include "tcgen05.cuh"

using namespace dbs::sm100;

constexpr int ROWS = 136;

__global__ void __launch_bounds__(128, 1) shift_kernel(const __grid_constant__ CUtensorMap tA,
                                                       const __grid_constant__ CUtensorMap tB, int shift,
                                                       int variant, float* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;                 // 136 rows x 128 B (17 KB) -> round to 18 KB
  uint8_t* sB = sm + 18 * 1024;     // 64 rows x 128 B
  __shared__ uint64_t full, done;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&full, 1);
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<64>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&full, ROWS * 128 + 64 * 128);
    tma_load_2d(sA, &tA, &full, 0, 0);
    tma_load_2d(sB, &tB, &full, 0, 0);
    mbar_wait(&full, 0);
    tc_fence_after();
    const uint32_t idesc = make_idesc_bf16(128, 64, 0, 0);
    for (int k = 0; k < 4; k++) {
      uint32_t a_addr = smem_u32(sA) + shift * 128 + k * 32;
      uint64_t ad;
      if (variant == 2) {
        ad = make_sdesc(smem_u32(sA) + k * 32, 16, 1024) | ((uint64_t)(shift & 7) << 49);
      } else {
        ad = make_sdesc(a_addr, 16, 1024);
        if (variant == 1) ad |= (uint64_t)((a_addr >> 7) & 7) << 49;
      }
      const uint64_t bd = make_sdesc(smem_u32(sB) + k * 32, 16, 1024);
      mma_bf16_ss(tmem, ad, bd, idesc, k ? 1u : 0u);
    }
    mma_commit(&done);
  }
  __syncwarp();
  mbar_wait(&done, 0);
  tc_fence_after();
  // warp q reads TMEM lanes 32q..32q+31 (rows), 64 columns
  for (int c = 0; c < 2; c++) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(tmem + ((uint32_t)(warp * 32) << 16) + c * 32, r);
    tmem_ld_wait();
    for (int j = 0; j < 32; j++) out[(warp * 32 + lane) * 64 + c * 32 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<64>(tmem);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static uint16_t f2bf(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}
static float bf2f(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(p);
  std::vector<uint16_t> A(ROWS * 64), B(64 * 64);
  srand(1);
  for (auto& v : A) v = f2bf((rand() % 17 - 8) / 8.0f);
  for (auto& v : B) v = f2bf((rand() % 17 - 8) / 8.0f);
  void *dA, *dB;
  float* dO;
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&dO, 128 * 64 * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  CUtensorMap tA, tB;
  cuuint64_t dimA[2] = {64, ROWS}, dimB[2] = {64, 64}, st[1] = {128};
  cuuint32_t boxA[2] = {64, ROWS}, boxB[2] = {64, 64}, es[2] = {1, 1};
  enc(&tA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dA, dimA, st, boxA, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&tB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dB, dimB, st, boxB, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(shift_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  std::vector<float> O(128 * 64);
  for (int variant = 0; variant < 3; variant++) {
    printf("variant %d:", variant);
    for (int s = 0; s <= 8; s++) {
      shift_kernel<<<1, 128, 40 * 1024>>>(tA, tB, s, variant, dO);
      cudaError_t e = cudaDeviceSynchronize();
      if (e) {
        printf(" err %s\n", cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
      double maxerr = 0;
      for (int m = 0; m < 128; m++)
        for (int n = 0; n < 64; n++) {
          double ref = 0;
          for (int k = 0; k < 64; k++) ref += (double)bf2f(A[(m + s) * 64 + k]) * bf2f(B[n * 64 + k]);
          maxerr = fmax(maxerr, fabs(ref - O[m * 64 + n]));
        }
      printf("  s=%d err=%.3g", s, maxerr);
    }
    printf("\n");
  }
  return 0;
}

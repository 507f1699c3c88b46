// Dev probe: TMA ingest rate per SM for the operand box shapes the GEMM uses.
// One CTA per SM: lane 0 of warp 0 streams boxes into a ring of shared-memory
// slots; lane 0 of warp 1 waits for each slot and frees it at once (no math).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2007_11831_b200/csrc \
//        scripts/tma_bench.cu -o scripts/_bin/tma_bench -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "tcgen05.cuh"

using namespace dbs::sm100;

struct Shape {
  const char* name;
  int rank;
  cuuint64_t dims[4];
  cuuint32_t box[4];
  int coord_mode;  // 0: 2-D rows walk; 1: 4-D conv walk (tile over h, n); 2: 4-D halo walk (h0-1, w-1)
  int swz32 = 0;   // 1: CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B (the MN-major tf32 operand layout)
};

template <int kSlots>
__global__ void __launch_bounds__(64, 1) tma_kernel(const __grid_constant__ CUtensorMap tm, int mode, int iters,
                                                     uint32_t bytes, int d1, int d2, int d3, int b1, int b2,
                                                     unsigned long long* cycles) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[kSlots], empty[kSlots];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const long long t0 = clock64();
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < iters; i++) {
      const int s = i % kSlots;
      mbar_wait(&empty[s], ((i / kSlots) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], bytes);
      const int tile = blockIdx.x + i * gridDim.x;
      uint8_t* dst = sm + s * bytes;
      if (mode == 0) {
        tma_load_2d(dst, &tm, &full[s], 0, (tile * b1) % d1);
      } else if (mode == 1) {
        const int per_img = d2 / b2;
        const int t = tile % (per_img * d3);
        tma_load_4d(dst, &tm, &full[s], 0, 0, (t % per_img) * b2, t / per_img);
      } else {
        const int per_img = d2 / (b2 - 2);
        const int t = tile % (per_img * d3);
        tma_load_4d(dst, &tm, &full[s], 0, (i % 3) - 1, (t % per_img) * (b2 - 2) - 1, t / per_img);
      }
    }
  } else if (warp == 1 && lane == 0) {
    for (int i = 0; i < iters; i++) {
      const int s = i % kSlots;
      mbar_wait(&full[s], (i / kSlots) & 1);
      mbar_arrive(&empty[s]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int grid = argc > 1 ? atoi(argv[1]) : 148;
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fnp;
  const size_t bytes = (size_t)128 * 32 * 32 * 64 * 2;  // 16.8 MB, L2 resident
  void* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 0, bytes);
  unsigned long long* cyc;
  cudaMalloc(&cyc, sizeof(unsigned long long) * 1024);
  Shape shapes[] = {
      {"2D  {64 x 32 rows}    4 KB", 2, {64, 131072}, {64, 32}, 0},
      {"2D  {64 x 64 rows}    8 KB", 2, {64, 131072}, {64, 64}, 0},
      {"2D  {64 x 128 rows}  16 KB", 2, {64, 131072}, {64, 128}, 0},
      {"2D  {64 x 192 rows}  24 KB", 2, {64, 131072}, {64, 192}, 0},
      {"2D  {64 x 256 rows}  32 KB", 2, {64, 131072}, {64, 256}, 0},
      {"4D  {64,32,4,1} conv 16 KB", 4, {64, 32, 32, 128}, {64, 32, 4, 1}, 1},
      {"4D  {64,32,6,1} halo 24 KB", 4, {64, 32, 32, 128}, {64, 32, 6, 1}, 2},
      {"4D  {64,16,8,1} conv 16 KB", 4, {64, 16, 16, 512}, {64, 16, 8, 1}, 1},
      {"2D  {64 x 32 rows}  4 KB atom32", 2, {64, 131072}, {64, 32}, 0, 1},
      {"2D  {64 x 128 rows} 16 KB atom32", 2, {64, 131072}, {64, 128}, 0, 1},
      {"4D  {64,32,4,1} 16 KB atom32", 4, {64, 32, 32, 128}, {64, 32, 4, 1}, 1, 1},
  };
  cudaFuncSetAttribute(tma_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(tma_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(tma_kernel<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(tma_kernel<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(tma_kernel<24>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  for (const Shape& sh : shapes) {
    CUtensorMap tm;
    cuuint64_t strides[3];
    cuuint64_t acc = sh.dims[0] * 2;
    for (int i = 0; i < sh.rank - 1; i++) {
      strides[i] = acc;
      acc *= sh.dims[i + 1];
    }
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, sh.rank, buf, sh.dims, strides, sh.box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE,
                     sh.swz32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("%s: encode failed %d\n", sh.name, (int)r);
      continue;
    }
    uint32_t box_bytes = 2;
    for (int i = 0; i < sh.rank; i++) box_bytes *= sh.box[i];
    const int iters = 600;
    int d1 = (int)sh.dims[1], d2 = sh.rank == 4 ? (int)sh.dims[2] : 0, d3 = sh.rank == 4 ? (int)sh.dims[3] : 0;
    int b1 = (int)sh.box[1], b2 = sh.rank == 4 ? (int)sh.box[2] : 0;
    if (sh.rank == 2) d1 = (int)sh.dims[1] - b1;
    for (int slots : {2, 4, 6, 12, 24}) {
    if ((size_t)slots * box_bytes > 190 * 1024) continue;
    for (int rep = 0; rep < 2; rep++) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      auto k = slots == 2 ? tma_kernel<2> : slots == 4 ? tma_kernel<4> : slots == 6 ? tma_kernel<6> : slots == 12 ? tma_kernel<12> : tma_kernel<24>;
      k<<<grid, 64, 200 * 1024>>>(tm, sh.coord_mode, iters, box_bytes, d1, d2, d3, b1, b2, cyc);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long h[1024];
      cudaMemcpy(h, cyc, sizeof(unsigned long long) * grid, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < grid; i++) avg += (double)h[i];
      avg /= grid;
      if (rep == 1)
        printf("%-30s grid %3d slots %2d: %7.1f B/clk/SM  %7.2f TB/s  latency %6.0f clk (err=%s)\n", sh.name, grid,
               slots, (double)box_bytes * iters / avg, (double)box_bytes * iters * grid / (ms * 1e-3) / 1e12,
               avg / iters * slots, cudaGetErrorString(cudaGetLastError()));
    }
    }
  }
  return 0;
}

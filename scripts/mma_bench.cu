// Dev probe: tcgen05.mma (kind::f16, SS operands, cta_group::1) issue rate per SM
// for M = 128 and N = 64 / 128 / 256, with operands resident in shared memory;
// variant 0: one fixed A tile, 1: A start shifted by one 128-byte row, 2: A cycling over 8 aligned tiles.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2007_11831_b200/csrc \
//        scripts/mma_bench.cu -o scripts/_bin/mma_bench
#include <cuda_runtime.h>
#include <stdio.h>

#include "tcgen05.cuh"

using namespace dbs::sm100;

template <int N, int M = 128>
__global__ void __launch_bounds__(128, 1) mma_kernel(int reps, int variant, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t done, side[8];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (192 + N) * 64 * 2 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    for (int i = 0; i < 8; i++) mbar_init(&side[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<(N < 32 ? 32 : N)>(&slot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a_base = smem_u32(sm), b_base = smem_u32(sm + 192 * 128);
    const uint32_t idesc = make_idesc_bf16(M, N, 0, 0);
    const long long t0 = clock64();
    for (int i = 0; i < reps; i++) {
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const uint32_t a_off = variant == 1 ? 128u : (variant == 2 ? (uint32_t)((i & 7) * 1024) : 0u);
        const uint64_t ad = make_sdesc(a_base + a_off + k * 32, 16, 1024);
        const uint64_t bd = make_sdesc(b_base + k * 32, 16, 1024);
        mma_bf16_ss(tmem, ad, bd, idesc, (i | k) != 0 ? 1u : 0u);
      }
    }
    mma_commit(&done);
    mbar_wait(&done, 0);
    const long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<(N < 32 ? 32 : N)>(tmem);
}

template <int N, int M = 128>
void run(int grid, int variant) {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 1024);
  const int smem = (192 + N) * 128 + 1024;
  cudaFuncSetAttribute(mma_kernel<N, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 2000;
  mma_kernel<N, M><<<grid, 128, smem>>>(reps, variant, d);
  mma_kernel<N, M><<<grid, 128, smem>>>(reps, variant, d);
  cudaDeviceSynchronize();
  unsigned long long h[1024];
  cudaMemcpy(h, d, 8 * grid, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < grid; i++) avg += (double)h[i];
  avg /= grid;
  const double per = avg / (reps * 4);
  printf("variant %d  M=%d N=%3d K=16 SS: %6.1f clk/MMA  %7.0f MAC/clk/SM  (%.0f%% of 4096)  err=%s\n", variant, M, N, per,
         (double)M * N * 16 / per, 100.0 * M * N * 16 / per / 4096, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main(int argc, char** argv) {
  const int grid = argc > 1 ? atoi(argv[1]) : 148;
  for (int v = 0; v < 3; v++) {
    run<64>(grid, v);
    run<128>(grid, v);
    run<256>(grid, v);
  }
  return 0;
}

// Dev probe: tcgen05.mma.cta_group::2 (a CTA pair, M = 256) issue rate vs N,
// operands resident in shared memory (values irrelevant), 74 clusters of 2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2007_11831_b200/csrc \
//        scripts/mma2sm_bench.cu -o scripts/_bin/mma2sm_bench
#include <cuda_runtime.h>
#include <stdio.h>

#include "tcgen05.cuh"

using namespace dbs::sm100;

template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k2(int reps, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t done;
  __shared__ uint32_t slot;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (128 + N) * 128 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "n"(256)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  tc_fence_after();
  const uint32_t tmem = slot;
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t a_base = smem_u32(sm), b_base = smem_u32(sm + 128 * 128);
    const uint32_t idesc = make_idesc_bf16(256, N, 0, 0);
    const long long t0 = clock64();
    for (int i = 0; i < reps; i++) {
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const uint64_t ad = make_sdesc(a_base + k * 32, 16, 1024);
        const uint64_t bd = make_sdesc(b_base + k * 32, 16, 1024);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"((i | k) != 0 ? 1u : 0u)
            : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     smem_u32(&done)),
                 "h"((uint16_t)3)
                 : "memory");
    mbar_wait(&done, 0);
    const long long t1 = clock64();
    out[blockIdx.x / 2] = (unsigned long long)(t1 - t0);
  }
  if (rank == 1 && threadIdx.x == 0) mbar_wait(&done, 0);
  tc_fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256) : "memory");
}

template <int N>
void run(int clusters) {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 1024);
  const int smem = (128 + N) * 128 + 2048;
  cudaFuncSetAttribute(k2<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 2000;
  k2<N><<<2 * clusters, 128, smem>>>(reps, d);
  k2<N><<<2 * clusters, 128, smem>>>(reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[1024];
  cudaMemcpy(h, d, 8 * clusters, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < clusters; i++) avg += (double)h[i];
  avg /= clusters;
  const double per = avg / (reps * 4);
  // one instruction = 256 x N x 16 MACs over 2 SMs
  printf("cta_group::2 M=256 N=%3d K=16 SS: %6.1f clk/MMA  %7.0f MAC/clk/SM  (%.0f%% of 4096)  err=%s\n", N, per,
         128.0 * N * 16 / per, 100.0 * 128.0 * N * 16 / per / 4096, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<64>(74);
  run<128>(74);
  run<256>(74);
  return 0;
}

// Dev probe: kind::tf32 tcgen05.mma issue rate, single CTA (M = 128) and CTA pair
// (cta_group::2, M = 256), by N, with and without concurrent shared-memory fill
// traffic (1-D cp.async.bulk copies from an L2-resident buffer into a separate
// region of the same CTA's shared memory, issued back to back by another warp --
// the TMA producer's writes of a real GEMM), and with descriptor starts shifted by
// whole 128-byte rows (the halo kernels' row-shifted views).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2007_11831_b200/csrc \
//        scripts/mma_tf32_probe.cu -o scripts/_bin/mma_tf32_probe
#include <cuda_runtime.h>
#include <stdio.h>

#include "tcgen05.cuh"

using namespace dbs::sm100;

constexpr int kOpBytes = 96 * 1024;     // operand region (A 128 rows + B up to 256 rows, 32 B per K step)
constexpr int kFillBytes = 96 * 1024;   // fill region

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int PAIR, int N>
__global__ void __launch_bounds__(128, 1) probe(int reps, int fill, int shift_rows, const uint8_t* gsrc,
                                                unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* fillr = sm + kOpBytes;
  __shared__ uint64_t done, fbar;
  __shared__ uint32_t slot;
  __shared__ volatile int stop;
  __shared__ unsigned long long fill_bytes;
  uint32_t rank = 0;
  if (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kOpBytes / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    mbar_init(&fbar, 1);
    stop = 0;
    fill_bytes = 0;
    fence_barrier_init();
  }
  if (warp == 0) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "n"(256)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      tmem_alloc<256>(&slot);
    }
  }
  tc_fence_before();
  if (PAIR)
    cluster_sync_all();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 1 && threadIdx.x == 32 && fill) {
    // producer: 32 KB per round (2 x 16 KB bulk copies), as fast as they complete
    uint32_t ph = 0;
    unsigned long long bytes = 0;
    const uint8_t* src = gsrc + (blockIdx.x % 16) * 65536;
    while (!stop) {
      mbar_arrive_expect_tx(&fbar, 2 * 16384);
      bulk_g2s(smem_u32(fillr), src, 16384, &fbar);
      bulk_g2s(smem_u32(fillr + 16384 + (fill > 1 ? 16384 : 0)), src + 16384, 16384, &fbar);
      mbar_wait(&fbar, ph);
      ph ^= 1;
      bytes += 32768;
    }
    fill_bytes = bytes;
  }
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t a_base = smem_u32(sm) + shift_rows * 128, b_base = smem_u32(sm + 128 * 128 * 2);
    const uint32_t idesc = make_idesc_tf32(PAIR ? 256 : 128, N, 0, 0);
    const long long t0 = clock64();
    for (int i = 0; i < reps; i++) {
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const uint64_t ad = make_sdesc(a_base + k * 32, 16, 1024);
        const uint64_t bd = make_sdesc(b_base + k * 32, 16, 1024);
        if (PAIR)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
              "l"(ad), "l"(bd), "r"(idesc), "r"((i | k) != 0 ? 1u : 0u)
              : "memory");
        else
          mma_tf32_ss(tmem, ad, bd, idesc, (i | k) != 0 ? 1u : 0u);
      }
    }
    if (PAIR)
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              smem_u32(&done)),
          "h"((uint16_t)3)
          : "memory");
    else
      mma_commit(&done);
    mbar_wait(&done, 0);
    const long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  if (PAIR && rank == 1 && threadIdx.x == 0) mbar_wait(&done, 0);
  if (threadIdx.x == 0) stop = 1;
  __syncthreads();
  if (threadIdx.x == 0) out[1024 + blockIdx.x] = fill_bytes;
  tc_fence_before();
  if (PAIR)
    cluster_sync_all();
  else
    __syncthreads();
  if (warp == 0) {
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256) : "memory");
    else
      tmem_dealloc<256>(tmem);
  }
}

template <int PAIR, int N>
void run(int fill, int shift, const uint8_t* g) {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 2048);
  cudaMemset(d, 0, 8 * 2048);
  const int smem = kOpBytes + kFillBytes + 2048;
  auto kern = probe<PAIR, N>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 2000, ctas = 148;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = PAIR ? 2 : 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  for (int w = 0; w < 2; w++) cudaLaunchKernelEx(&cfg, kern, reps, fill, shift, g, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[2048];
  cudaMemcpy(h, d, 8 * 2048, cudaMemcpyDeviceToHost);
  double avg = 0, fb = 0;
  int cnt = 0;
  for (int i = 0; i < ctas; i += (PAIR ? 2 : 1)) {
    avg += (double)h[i];
    cnt++;
  }
  for (int i = 0; i < ctas; i++) fb += (double)h[1024 + i];
  avg /= cnt;
  fb /= ctas;
  const double per = avg / (reps * 4);
  const int M = PAIR ? 256 : 128;
  // per-SM MACs of one instruction: 128 x N x 8; tf32 dense = 2048 MAC/clk/SM
  const double mac = 128.0 * N * 8 / per;
  printf("%s M=%3d N=%3d K=8 tf32 fill=%d shift=%d: %6.1f clk/MMA  %6.0f MAC/clk/SM (%3.0f%% of 2048)  fill %5.1f B/clk  %s\n",
         PAIR ? "pair  " : "single", M, N, fill, shift, per, mac, 100.0 * mac / 2048, fb / avg, cudaGetErrorString(e));
  cudaFree(d);
}


// The 3xTF32 issue pattern of one 32-wide k-block (4 k-steps): A_hi x [B_hi | B_lo]
// (N = 2 BN into [main | corr]) and A_lo x B_hi (N = BN) --
//   pat 0: alternating, the second into corr (overlaps the first's columns)
//   pat 1: grouped -- the 4 N = 2 BN MMAs, then the 4 N = BN ones (same accumulators)
//   pat 2: alternating, the second into a separate accumulator (no overlap)
template <int BN>
__global__ void __launch_bounds__(128, 1) pattern(int reps, int pat, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t done, ring[8];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  const bool rnd = pat >= 10;
  pat %= 10;
  const bool rot = pat == 4;  // rotate the operands over 4 slots of 48 KB (a ring), no reuse between k-blocks
  for (int i = threadIdx.x; i < (rot ? 4 * 49152 : kOpBytes) / 4; i += blockDim.x) {
    // rnd: N(0,1)-like fp32 values (random mantissas, exponents around 1), else zeros
    uint32_t h = (uint32_t)i * 2654435761u ^ 0x9e3779b9u;
    h ^= h >> 15;
    h *= 0x85ebca6bu;
    h ^= h >> 13;
    const float v = rnd ? __uint_as_float(0x3f000000u | (h & 0x807FFFFFu)) : 0.0f;
    reinterpret_cast<float*>(sm)[i] = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    for (int q = 0; q < 8; q++) mbar_init(&ring[q], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a_hi0 = smem_u32(sm), a_lo0 = a_hi0 + 16384, b0 = smem_u32(sm + 32768);
    const uint32_t id2 = make_idesc_tf32(128, 2 * BN, 0, 0), id1 = make_idesc_tf32(128, BN, 0, 0);
    const uint32_t corr = pat == 2 ? tmem + 2 * BN : tmem + BN;
    const long long t0 = clock64();
    for (int i = 0; i < reps; i++) {
      const uint32_t rs = rot ? (uint32_t)(i & 3) * 49152u : 0u;
      const uint32_t a_hi = a_hi0 + rs, a_lo = a_lo0 + rs, b = b0 + rs;
      if (pat == 1) {
#pragma unroll
        for (int k = 0; k < 4; k++)
          mma_tf32_ss(tmem, make_sdesc(a_hi + k * 32, 16, 1024), make_sdesc(b + k * 32, 16, 1024), id2, (i | k) != 0);
#pragma unroll
        for (int k = 0; k < 4; k++)
          mma_tf32_ss(corr, make_sdesc(a_lo + k * 32, 16, 1024), make_sdesc(b + k * 32, 16, 1024), id1, 1u);
      } else {
#pragma unroll
        for (int k = 0; k < 4; k++) {
          mma_tf32_ss(tmem, make_sdesc(a_hi + k * 32, 16, 1024), make_sdesc(b + k * 32, 16, 1024), id2, (i | k) != 0);
          mma_tf32_ss(corr, make_sdesc(a_lo + k * 32, 16, 1024), make_sdesc(b + k * 32, 16, 1024), id1, 1u);
        }
        // pat 3: a commit to a (never waited) mbarrier after every k-block, as the GEMM's ring does
        if (pat == 3) mma_commit(&ring[i & 7]);
      }
    }
    mma_commit(&done);
    mbar_wait(&done, 0);
    out[blockIdx.x] = (unsigned long long)(clock64() - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int BN>
void run_pattern(int pat) {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 2048);
  const int smem = 4 * 49152 + 2048;
  cudaFuncSetAttribute(pattern<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 1000;
  for (int w = 0; w < 2; w++) pattern<BN><<<148, 128, smem>>>(reps, pat, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; i++) avg += (double)h[i];
  avg /= 148;
  const double per = avg / reps;  // one k-block = 4 k-steps x 2 MMAs
  const double ideal = 3.0 * 128 * BN * 32 / 2048;
  printf("3xTF32 BN=%3d pattern %2d (>= 10: random data): %6.1f clk per 32-wide k-block (ideal %5.1f, %3.0f%%)  %s\n", BN, pat, per, ideal,
         100 * ideal / per, cudaGetErrorString(e));
  cudaFree(d);
}


// MN-major operands (SWIZZLE_128B_BASE32B, the transposed weight gradient's layout):
// kind::tf32 M=128 N=BN K=8 issue rate with A and/or B MN-major (a_mn, b_mn)
template <int BN>
__global__ void __launch_bounds__(128, 1) mnrate(int reps, int a_mn, int b_mn, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t done;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kOpBytes / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
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
    const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 32768);
    const uint32_t idesc = make_idesc_tf32(128, BN, a_mn, b_mn);
    const long long t0 = clock64();
    for (int i = 0; i < reps; i++) {
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const uint64_t ad = a_mn ? make_sdesc(a0 + k * 1024, 8192, 512, 1) : make_sdesc(a0 + k * 32, 16, 1024);
        const uint64_t bd = b_mn ? make_sdesc(b0 + k * 1024, 4096, 512, 1) : make_sdesc(b0 + k * 32, 16, 1024);
        mma_tf32_ss(tmem, ad, bd, idesc, (i | k) != 0);
      }
    }
    mma_commit(&done);
    mbar_wait(&done, 0);
    out[blockIdx.x] = (unsigned long long)(clock64() - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tmem);
}

template <int BN>
void run_mn(int a_mn, int b_mn) {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 2048);
  const int smem = kOpBytes + 2048;
  cudaFuncSetAttribute(mnrate<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 2000;
  for (int w = 0; w < 2; w++) mnrate<BN><<<148, 128, smem>>>(reps, a_mn, b_mn, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; i++) avg += (double)h[i];
  avg /= 148;
  const double per = avg / (reps * 4);
  printf("tf32 M=128 N=%3d a_mn=%d b_mn=%d: %6.1f clk/MMA (%3.0f%% of 2048 MAC/clk)  %s\n", BN, a_mn, b_mn, per,
         100.0 * 128.0 * BN * 8 / per / 2048, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int am = 0; am < 2; am++)
    for (int bm = 0; bm < 2; bm++) {
      run_mn<64>(am, bm);
      run_mn<128>(am, bm);
    }

  for (int pat : {0, 3, 4, 13, 14}) {
    run_pattern<64>(pat);
    run_pattern<128>(pat);
  }

  uint8_t* g;
  cudaMalloc(&g, 16 << 20);
  cudaMemset(g, 1, 16 << 20);
  for (int fill = 0; fill < 2; fill++) {
    run<0, 64>(fill, 0, g);
    run<0, 128>(fill, 0, g);
    run<0, 256>(fill, 0, g);
    run<1, 64>(fill, 0, g);
    run<1, 128>(fill, 0, g);
    run<1, 256>(fill, 0, g);
  }
  run<0, 128>(0, 3, g);
  run<1, 64>(0, 3, g);
  run<1, 128>(0, 3, g);
  run<1, 128>(1, 3, g);
  return 0;
}

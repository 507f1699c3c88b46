// Dev probe: timeline of the persistent tcgen05 GEMM (build with scripts/build_gemm_trace.sh).
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>
#include "dbs_b200.h"
extern "C" int dbs_gemm_trace_copy(unsigned long long* host, int n);
int main(int argc, char** argv) {
  // gemm_trace M N K            plain GEMM
  // gemm_trace conv N H C       3x3 stride-1 C->C conv forward on an N x H x H x C map
  // gemm_trace f32conv N H C    the same conv, fp32 class (3xTF32 on S32 operands)
  // gemm_trace wgrad N H C       the fp32-class weight gradient of the same conv
  const bool wgrad = argc > 1 && argv[1][0] == 'w';
  const bool f32 = argc > 1 && (argv[1][0] == 'f' || wgrad);
  const bool conv = argc > 1 && (argv[1][0] == 'c' || f32);
  const int o = conv ? 1 : 0;
  long M = argc > 1 + o ? atol(argv[1 + o]) : 131072, N = argc > 2 + o ? atol(argv[2 + o]) : 64, K = argc > 3 + o ? atol(argv[3 + o]) : 64;
  void *a, *b, *d;
  size_t abytes = conv ? (size_t)M * N * N * K * 2 : M * K * 2, bbytes = conv ? (size_t)K * 9 * K * 2 : N * K * 2;
  size_t dbytes = conv ? abytes : M * N * 2;
  if (f32) { abytes *= 4; bbytes *= 4; dbytes *= 2; }
  cudaMalloc(&a, abytes); cudaMalloc(&b, bbytes); cudaMalloc(&d, dbytes);
  cudaMemset(a, 0x3c, abytes); cudaMemset(b, 0x3c, bbytes);
  auto run = [&]() {
    if (wgrad) return dbs_dev_conv2d_wgrad_s32(a, a, (int)M, (int)N, (int)N, (int)K, (int)K, 3, 1, 1, (float*)d, nullptr);
    if (f32) return dbs_dev_conv2d_fwd_s32(a, (int)M, (int)N, (int)N, (int)K, b, (int)K, 3, 1, 1, (float*)d, nullptr);
    return conv ? dbs_dev_conv2d_fwd(a, (int)M, (int)N, (int)N, (int)K, b, (int)K, 3, 1, 1, d, nullptr)
                : dbs_dev_gemm_bf16(a, 0, K, b, 0, K, d, N, M, N, K, DBS_EPI_BF16, nullptr, nullptr, nullptr);
  };
  for (int i = 0; i < 5; i++)
    if (run()) { printf("err %s\n", dbs_last_error()); return 1; }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  run();
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("M=%ld N=%ld K=%ld: %.1f us  err=%s\n", M, N, K, ms * 1e3, cudaGetErrorString(cudaGetLastError()));
  std::vector<unsigned long long> t(1024 * 128);
  dbs_gemm_trace_copy(t.data(), 1024 * 128);
  for (int c : {0, 147}) {
    unsigned long long* r = &t[c * 128];
    unsigned long long t0 = r[0];
    printf("CTA %d: setup %llu  end %llu\n", c, r[1] - t0, r[63] - t0);
    for (int j = 0; j < 10; j++)
      printf("  tile %d: load %7lld  mma_acq %7lld  mma_commit %7lld  epi_acq %7lld  epi_rel %7lld  epi_done %7lld\n", j,
             (long long)(r[2 + j] - t0), (long long)(r[12 + j] - t0), (long long)(r[22 + j] - t0), (long long)(r[32 + j] - t0),
             (long long)(r[42 + j] - t0), (long long)(r[52 + j] - t0));
    for (int j = 0; j < 8; j++)
      printf("  mma tile %d: ready0 %lld ready1 %lld ready2 %lld\n", j, (long long)(r[96 + 3 * j] - t0),
             (long long)(r[97 + 3 * j] - t0), (long long)(r[98 + 3 * j] - t0));
    printf("  k-block: producer-issue / mma-full:");
    for (int j = 0; j < 12; j++) printf(" %lld/%lld", (long long)(r[100 + j] - t0), (long long)(r[112 + j] - t0));
    printf("\n  k-block: mma issued (halo S32):");
    for (int j = 0; j < 12; j++) printf(" %lld", (long long)(r[64 + j] - t0));
    printf("\n");
    for (int j = 0; j < 8; j++)
      printf("  epi tile %d: ldtm0 %lld chunk0 %lld ldtm1 %lld chunk1 %lld\n", j, (long long)(r[64 + 4 * j] - t0),
             (long long)(r[65 + 4 * j] - t0), (long long)(r[66 + 4 * j] - t0), (long long)(r[67 + 4 * j] - t0));
  }
  return 0;
}

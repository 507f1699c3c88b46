// gemm.cu -- tcgen05 tensor-core GEMM for the variable-batch forward/backward.
//
//   D[M, N] (+)= A[M, K] * B[N, K]^T      bf16 operands, fp32 accumulation in TMEM
//
// Either operand may be K-major (row-major over K) or MN-major (the transpose
// stored row-major), so the forward (X W^T), the input gradient (dY W) and the
// weight gradient (dY^T X) all read the activations in place -- no transposes.
//
// Structure (one 128 x BN output tile per CTA, 4 warps):
//   warp 0 / lane 0 : TMA producer -- 128B-swizzled boxes into a STAGES-deep
//                     shared-memory ring, mbarrier expect_tx per stage;
//   warp 1 / lane 0 : MMA issuer  -- 4 x tcgen05.mma (UMMA_K = 16) per 64-wide
//                     K block, tcgen05.commit frees the ring slot;
//   warp 2          : TMEM allocator (BN fp32 columns);
//   all 4 warps     : epilogue -- tcgen05.ld 32x32b (thread = output row),
//                     fused bias / ReLU / ReLU-backward / bf16 cast, stores.
// Variable batch: M (the per-rank batch b_i) is a runtime value; rows past M
// are zero-filled by TMA (OOB fill) and masked in the epilogue, so a batch size
// that changes every epoch needs no recompilation and no padding copies.
#include <cuda.h>

#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "tcgen05.cuh"

namespace dbs {
namespace {

using namespace sm100;

constexpr int kBM = 128;
constexpr int kBK = 64;  // one 128-byte swizzle atom of bf16 along K
constexpr int kThreads = 128;

struct GemmParams {
  int64_t M, N, K;
  int a_mn, b_mn;
  int epi;
  void* d;
  int64_t ldd;
  const float* bias;
  const uint16_t* aux;  // bf16 [M][ldd] for the ReLU-backward epilogue
  float* colsum_part;   // optional [ceil(M/32)][N] per-warp column sums of the epilogue output
};

__device__ __forceinline__ uint16_t f2bf(float f) {
  uint32_t u = __float_as_uint(f);
  return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}
__device__ __forceinline__ float bf2f(uint16_t h) { return __uint_as_float(((uint32_t)h) << 16); }

template <int BN>
struct Cfg {
  static constexpr uint32_t kABytes = kBM * kBK * 2;                 // 16 KB
  static constexpr uint32_t kBBytes = BN * kBK * 2;
  static constexpr int kStages = (BN >= 256) ? 4 : (BN >= 128 ? 6 : 8);
  static constexpr uint32_t kTmemCols = BN < 32 ? 32 : BN;
  static constexpr size_t kSmem = 1024 + (size_t)kStages * (kABytes + kBBytes) + 256;
};

template <int BN>
__device__ __forceinline__ void epilogue_chunk(const GemmParams& p, int64_t row, int64_t n_base, const float* v,
                                               int cnt, float* v_out) {
  const int64_t N = p.N;
  const bool full = (n_base + cnt <= N);
  switch (p.epi) {
    case DBS_EPI_F32:
    case DBS_EPI_F32_ACCUM:
    case DBS_EPI_BIAS_F32: {
      float* d = reinterpret_cast<float*>(p.d) + row * p.ldd + n_base;
      float o[32];
#pragma unroll
      for (int j = 0; j < 32; j++) {
        if (j >= cnt) break;
        float x = v[j];
        if (p.epi == DBS_EPI_BIAS_F32 && n_base + j < N) x += p.bias[n_base + j];
        o[j] = x;
      }
      const bool vec = full && cnt == 32 && ((reinterpret_cast<uintptr_t>(d) & 15) == 0);
      if (p.epi == DBS_EPI_F32_ACCUM) {
        for (int j = 0; j < cnt; j++)
          if (n_base + j < N) d[j] += o[j];
      } else if (vec) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(d + j) = make_float4(o[j], o[j + 1], o[j + 2], o[j + 3]);
      } else {
        for (int j = 0; j < cnt; j++)
          if (n_base + j < N) d[j] = o[j];
      }
      break;
    }
    case DBS_EPI_BIAS_RELU_BF16:
    case DBS_EPI_BF16:
    case DBS_EPI_RELU_GRAD_BF16: {
      uint16_t* d = reinterpret_cast<uint16_t*>(p.d) + row * p.ldd + n_base;
      const uint16_t* aux = p.aux ? p.aux + row * p.ldd + n_base : nullptr;
      uint16_t o[32];
#pragma unroll
      for (int j = 0; j < 32; j++) {
        if (j >= cnt) break;
        float x = v[j];
        if (p.epi == DBS_EPI_BIAS_RELU_BF16) {
          if (n_base + j < N) x += p.bias[n_base + j];
          x = fmaxf(x, 0.0f);
        } else if (p.epi == DBS_EPI_RELU_GRAD_BF16) {
          x = (n_base + j < N && bf2f(aux[j]) > 0.0f) ? x : 0.0f;
        }
        o[j] = f2bf(x);
        v_out[j] = x;
      }
      const bool vec = full && cnt == 32 && ((reinterpret_cast<uintptr_t>(d) & 15) == 0);
      if (vec) {
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          uint4 q;
          q.x = o[j] | ((uint32_t)o[j + 1] << 16);
          q.y = o[j + 2] | ((uint32_t)o[j + 3] << 16);
          q.z = o[j + 4] | ((uint32_t)o[j + 5] << 16);
          q.w = o[j + 6] | ((uint32_t)o[j + 7] << 16);
          *reinterpret_cast<uint4*>(d + j) = q;
        }
      } else {
        for (int j = 0; j < cnt; j++)
          if (n_base + j < N) d[j] = o[j];
      }
      break;
    }
    default:
      break;
  }
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmParams p) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kStages * C::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::kStages * C::kBBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tmem_full = empty + C::kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m0 = (int64_t)blockIdx.x * kBM, n0 = (int64_t)blockIdx.y * BN;
  const int num_k = (int)((p.K + kBK - 1) / kBK);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < C::kStages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    for (int kb = 0; kb < num_k; kb++) {
      const int s = kb % C::kStages;
      if (kb >= C::kStages) mbar_wait(&empty[s], ((kb / C::kStages) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], C::kABytes + C::kBBytes);
      const int32_t k0 = kb * kBK;
      uint8_t* a = sA + s * C::kABytes;
      uint8_t* b = sB + s * C::kBBytes;
      if (!p.a_mn) {
        tma_load_2d(a, &tmA, &full[s], k0, (int32_t)m0);
      } else {
        tma_load_2d(a, &tmA, &full[s], (int32_t)m0, k0);
        tma_load_2d(a + 8192, &tmA, &full[s], (int32_t)m0 + 64, k0);
      }
      if (!p.b_mn) {
        tma_load_2d(b, &tmB, &full[s], k0, (int32_t)n0);
      } else {
#pragma unroll
        for (int j = 0; j < BN / 64; j++) tma_load_2d(b + j * 8192, &tmB, &full[s], (int32_t)n0 + 64 * j, k0);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = make_idesc_bf16(kBM, BN, p.a_mn, p.b_mn);
    for (int kb = 0; kb < num_k; kb++) {
      const int s = kb % C::kStages;
      mbar_wait(&full[s], (kb / C::kStages) & 1);
      tc_fence_after();
      const uint32_t a_base = smem_u32(sA + s * C::kABytes);
      const uint32_t b_base = smem_u32(sB + s * C::kBBytes);
#pragma unroll
      for (int k = 0; k < kBK / 16; k++) {
        const uint64_t ad = p.a_mn ? make_sdesc(a_base + k * 2048, 8192, 1024) : make_sdesc(a_base + k * 32, 16, 1024);
        const uint64_t bd = p.b_mn ? make_sdesc(b_base + k * 2048, 8192, 1024) : make_sdesc(b_base + k * 32, 16, 1024);
        mma_bf16_ss(tmem_base, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
      }
      mma_commit(&empty[s]);
    }
    mma_commit(tmem_full);
  }
  __syncwarp();

  // ---------------- epilogue (all 4 warps) ----------------
  mbar_wait(tmem_full, 0);
  tc_fence_after();
  const int64_t row = m0 + warp * 32 + lane;
  const uint32_t lane_addr = tmem_base + ((uint32_t)(warp * 32) << 16);
  if (BN >= 32) {
#pragma unroll 1
    for (int c = 0; c < BN / 32; c++) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(lane_addr + c * 32, r);
      tmem_ld_wait();
      const int64_t n_base = n0 + c * 32;
      if (n_base >= p.N) continue;  // warp-uniform
      float v[32], vo[32];
#pragma unroll
      for (int j = 0; j < 32; j++) {
        v[j] = __uint_as_float(r[j]);
        vo[j] = 0.0f;
      }
      const int cnt = (int)((p.N - n_base) < 32 ? (p.N - n_base) : 32);
      if (row < p.M) epilogue_chunk<BN>(p, row, n_base, v, cnt, vo);
      if (p.colsum_part != nullptr) {
        // deterministic per-warp column sums of the stored values (e.g. the bias
        // gradient sum_b dH): transpose-reduce 32 rows x 32 columns across lanes
#pragma unroll
        for (int j = 0; j < 32; j++) {
          float s = vo[j];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
          vo[j] = s;
        }
        const int64_t g = (m0 >> 5) + warp;
        if (lane < cnt && m0 + warp * 32 < p.M) p.colsum_part[g * p.N + n_base + lane] = vo[lane];
      }
    }
  } else {
    uint32_t r[16];
    tmem_ld_32x32b_x16(lane_addr, r);
    tmem_ld_wait();
    if (row < p.M && n0 < p.N) {
      float v[32], vo[32];
#pragma unroll
      for (int j = 0; j < 16; j++) v[j] = __uint_as_float(r[j]);
      const int cnt = (int)((p.N - n0) < 16 ? (p.N - n0) : 16);
      epilogue_chunk<BN>(p, row, n0, v, cnt, vo);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<C::kTmemCols>(tmem_base);
}

// ---------------------------------------------------------------------------
// host: tensor-map encoding through the driver entry point (no -lcuda needed)
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 2-D bf16 tensor [rows][ld] (inner dim `inner` elements), box {box0, box1}
int make_tmap(CUtensorMap* tm, const void* base, uint64_t inner, uint64_t rows, uint64_t ld_elems, uint32_t box0,
              uint32_t box1) {
  EncodeTiledFn fn = encode_fn();
  DBS_REQUIRE(fn != nullptr, DBS_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
  DBS_REQUIRE(((uintptr_t)base & 15) == 0 && (ld_elems * 2) % 16 == 0, DBS_ERR_ARGUMENT,
              "TMA needs 16-byte aligned base and leading dimension (ld %% 8 == 0)");
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {box0, box1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  DBS_REQUIRE(r == CUDA_SUCCESS, DBS_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return DBS_OK;
}

template <int BN>
int launch(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, cudaStream_t s) {
  using C = Cfg<BN>;
  static bool attr = false;
  if (!attr) {
    DBS_CUDA_TRY(cudaFuncSetAttribute(gemm_bf16_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem));
    attr = true;
  }
  dim3 grid((unsigned)((p.M + kBM - 1) / kBM), (unsigned)((p.N + BN - 1) / BN));
  gemm_bf16_kernel<BN><<<grid, kThreads, C::kSmem, s>>>(ta, tb, p);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

}  // namespace

// Entry used by the MLP driver too.
int gemm_bf16(const void* a, int a_mn, int64_t lda, const void* b, int b_mn, int64_t ldb, void* d, int64_t ldd,
              int64_t M, int64_t N, int64_t K, int epi, const float* bias, const void* aux, cudaStream_t s,
              float* colsum_part) {
  DBS_REQUIRE(M > 0 && N > 0 && K > 0 && a && b && d, DBS_ERR_ARGUMENT, "gemm: bad shape/pointers");
  DBS_REQUIRE(epi >= DBS_EPI_F32 && epi <= DBS_EPI_RELU_GRAD_BF16, DBS_ERR_ARGUMENT, "gemm: bad epilogue %d", epi);
  DBS_REQUIRE(!((epi == DBS_EPI_BIAS_RELU_BF16 || epi == DBS_EPI_BIAS_F32) && !bias), DBS_ERR_ARGUMENT,
              "gemm: epilogue needs bias");
  DBS_REQUIRE(!(epi == DBS_EPI_RELU_GRAD_BF16 && !aux), DBS_ERR_ARGUMENT, "gemm: epilogue needs aux");
  int bn;
  if (N <= 16 && !b_mn) bn = 16;
  else if (N <= 64) bn = 64;
  else if (N <= 128) bn = 128;
  else bn = 256;
  CUtensorMap ta, tb;
  int st;
  // A: K-major [M][lda] -> box {64 K, 128 M};  MN-major [K][lda] -> box {64 M, 64 K}
  st = a_mn ? make_tmap(&ta, a, (uint64_t)M, (uint64_t)K, (uint64_t)lda, 64, 64)
            : make_tmap(&ta, a, (uint64_t)K, (uint64_t)M, (uint64_t)lda, 64, 128);
  if (st) return st;
  // B: K-major [N][ldb] -> box {64 K, BN};  MN-major [K][ldb] -> box {64 N, 64 K}
  st = b_mn ? make_tmap(&tb, b, (uint64_t)N, (uint64_t)K, (uint64_t)ldb, 64, 64)
            : make_tmap(&tb, b, (uint64_t)K, (uint64_t)N, (uint64_t)ldb, 64, (uint32_t)bn);
  if (st) return st;
  DBS_REQUIRE(!(colsum_part && bn < 32), DBS_ERR_ARGUMENT, "gemm: column sums need N > 16");
  GemmParams p{M, N, K, a_mn, b_mn, epi, d, ldd, bias, reinterpret_cast<const uint16_t*>(aux), colsum_part};
  switch (bn) {
    case 16: return launch<16>(ta, tb, p, s);
    case 64: return launch<64>(ta, tb, p, s);
    case 128: return launch<128>(ta, tb, p, s);
    default: return launch<256>(ta, tb, p, s);
  }
}

}  // namespace dbs

extern "C" int dbs_dev_gemm_bf16(const void* d_a, int32_t a_major, int64_t lda, const void* d_b, int32_t b_major,
                                 int64_t ldb, void* d_d, int64_t ldd, int64_t M, int64_t N, int64_t K,
                                 int32_t epilogue, const float* d_bias, void* d_aux, void* stream) {
  return dbs::gemm_bf16(d_a, a_major, lda, d_b, b_major, ldb, d_d, ldd, M, N, K, epilogue, d_bias, d_aux,
                        dbs::as_stream(stream), nullptr);
}

// gemm.cu -- tcgen05 tensor-core GEMM / implicit-GEMM convolution.
//
//   D[M, N] (+)= A[M, K] * B[N, K]^T      bf16 operands, fp32 accumulation in TMEM
//
// Operand modes (TMA, 128-byte swizzle):
//   0 K-major   : row-major over K                       (X W^T, conv weights)
//   1 MN-major  : the transpose stored row-major         (dY^T X, dZ W, ...)
//   2 conv      : a 4-D NHWC activation read as an implicit im2col matrix --
//                 A: rows = 128 output pixels, K = (r, s, c) with c fastest, one
//                    TMA box per K block at the (r, s)-shifted, strided input
//                    window (zero padding = TMA out-of-bounds fill);
//                 B: (weight gradient) rows = K = 64 output pixels, N = (r, s, c),
//                    MN-major boxes of 64 channels.
// so the variable-batch forward (conv / X W^T), the input gradient (conv of dY
// with the flipped filter / dZ W) and the weight gradient (dY^T im2col(X))
// all read activations in place -- no im2col buffers, no transposes.
//
// Structure: a persistent kernel, one CTA per SM, 6 warps, walking the output
// tiles (128 x BN, x split-K slice) in a static stride over the grid:
//   warp 0 / lane 0 : TMA producer into a STAGES-deep shared-memory ring that
//                     runs continuously across tiles;
//   warp 1          : TMEM allocator (2 x BN fp32 columns: two accumulators);
//     lane 0        : MMA issuer (4 x tcgen05.mma, UMMA_K = 16, per 64-wide K
//                     block; tcgen05.commit frees the ring slot / hands the
//                     accumulator to the epilogue);
//   warps 2..5      : epilogue of tile t (TMEM lane quadrant = warp % 4) while
//                     the MMA warp already accumulates tile t+1 into the other
//                     buffer -- tcgen05.ld 32x32b (thread = output row), fused
//                     bias / ReLU / ReLU-backward / bf16 cast / accumulate /
//                     split-K atomic reduction, and per-warp column partial sums
//                     (bias gradients, BatchNorm batch statistics).
// Variable batch: M (the per-rank batch b_i, or b_i x H x W pixels) is a runtime
// value; rows past M are zero-filled by TMA and masked in the epilogue, so a
// batch size that changes every epoch needs no recompilation and no padding.
#include <cuda.h>

#include <stdlib.h>

#include <mutex>
#include <type_traits>

#include "common.cuh"
#include "gemm.cuh"
#include "tcgen05.cuh"

namespace dbs {
namespace {

using namespace sm100;

constexpr int kBM = 128;
constexpr int kBK = 64;  // one 128-byte swizzle atom of bf16 along K
constexpr int kThreads = 192;  // producer warp, MMA warp, 4 epilogue warps

// Development-only timeline probe (-DDBS_GEMM_TRACE, scripts/gemm_trace.cu):
// per-CTA clock64 stamps of the producer / MMA / epilogue hand-offs.
#ifdef DBS_GEMM_TRACE
__device__ unsigned long long g_gemm_trace[1024 * 128];
#define GEMM_TRACE(slot)                                                                    \
  do {                                                                                      \
    if ((slot) < 128) g_gemm_trace[blockIdx.x * 128 + (slot)] = (unsigned long long)clock64(); \
  } while (0)
#else
#define GEMM_TRACE(slot) \
  do {                   \
  } while (0)
#endif

// Attribution switches (DBS_GEMM_DBG at run time) exist only in a -DDBS_GEMM_ATTRIB build:
// the run-time checks alone cost the S32 kernels registers / local-memory spills (ResNet-18
// worker step 10.8 -> 10.4 ms without them; the MLP epoch ~10%)
#ifdef DBS_GEMM_ATTRIB
#define DBS_GEMM_DBG_BIT(p, bit) (((p).dbg & (bit)) != 0)
#else
#define DBS_GEMM_DBG_BIT(p, bit) (false)
#endif

struct GemmParams {
  int64_t M, N, K;
  int a_mode, b_mode;
  int epi;
  void* d;
  int64_t ldd;
  const float* bias;
  const uint16_t* aux;  // bf16 [M][ldd] for the ReLU-backward epilogue
  float* colsum_part;   // [ceil(M/32)][N] per-warp column sums of the stored values
  double* sum_part;     // [N] column sums of the accumulator (fp64 atomics, BN statistics)
  double* sq_part;      // [N] column sums of accumulator^2
  ConvGeom ga, gb;      // implicit-GEMM geometry of A / B in conv mode
  int kb_per_split;     // K blocks per split-K slice
  int splits;           // split-K slices (atomic epilogue when > 1)
  ConvTaps taps;        // explicit conv taps of A (n = 0: R x S window)
  OutMap omap;          // strided output rows (on = 0: row-major)
  int pair_a, pair_b;   // one TMA box covers two consecutive k-blocks (ring slots s, s+1) of A / B
  int nclass;           // > 0: merged output-parity classes (stride-2 input gradient), class c owns
  int64_t cls_start[5]; //   tiles [cls_start[c], cls_start[c + 1]) with its own taps / output map
  int cls_kb[4];        //   and k-block count
  ConvTaps cls_taps[4];
  OutMap cls_omap[4];
  int halo_rows;        // halo variant: image rows per TMA box
  int halo_tpi;         // halo variant: tiles per image (ceil(OH (OW + 1) / 128))
  int64_t halo_tiles;   // halo variant: images x tiles per image
  int d_trans;          // F32 atomic epilogue: D stored transposed (d[n * ldd + m])
  int b_wide;           // flipped-filter B (mode 3): one 4-D box per k-block covers all BN / 64 channel blocks
  int dbg;              // measurement only (DBS_GEMM_DBG in a -DDBS_GEMM_ATTRIB build, S32 path): 1 = no TMA
                        //   loads, 2 = no MMAs, 4 = no epilogue work
  int tf_nbuf;          // S32, BN = 128: 1 = one TMEM buffer of two main accumulators, 2 = two buffers
                        //   of one main each (tile j's epilogue overlaps tile j + 1's MMAs)
};

// two floats -> packed bf16x2 (lo in bits 0..15), one round-to-nearest-even
// conversion instruction (F2FP) instead of integer rounding per element
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ uint16_t f2bf(float f) {
  uint32_t u = __float_as_uint(f);
  return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}
__device__ __forceinline__ float bf2f(uint16_t h) { return __uint_as_float(((uint32_t)h) << 16); }

// S32 (fp32-class operand format, include/dbs_b200.h dbs_dev_gemm_tf32x3): each
// 32-element block of a row is 32 tf32 "hi" values then 32 tf32 "lo" values
__device__ __forceinline__ float tf32_rn(float x) {
  const uint32_t u = __float_as_uint(x);
  return __uint_as_float((u + 0xFFFu + ((u >> 13) & 1u)) & 0xFFFFE000u);
}
// 32 consecutive logical values -> one S32 block (256 contiguous bytes at `blk`)
__device__ __forceinline__ void store_s32x32(float* blk, const float (&x)[32]) {
#pragma unroll
  for (int j = 0; j < 32; j += 8) {
    float h[8], l[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      h[u] = tf32_rn(x[j + u]);
      l[u] = tf32_rn(x[j + u] - h[u]);
    }
    stg8(blk + j, v8_of(h));  // 256-bit stores (the block is 256-byte aligned)
    stg8(blk + 32 + j, v8_of(l));
  }
}
__device__ __forceinline__ bool is_s32_epi(int epi) {
  return epi == DBS_EPI_S32 || epi == DBS_EPI_BIAS_RELU_S32 || epi == DBS_EPI_RELU_GRAD_S32;
}

template <int BN>
struct Cfg {
  static constexpr uint32_t kABytes = kBM * kBK * 2;  // 16 KB
  static constexpr uint32_t kBBytes = BN * kBK * 2;
  static constexpr uint32_t kAccCols = BN < 32 ? 32 : BN;  // fp32 TMEM columns of one accumulator
  static constexpr uint32_t kTmemCols = 2 * kAccCols;      // double-buffered: epilogue(t) || MMA(t+1)
  static constexpr uint32_t kEpiBytes = 4 * 32 * 33 * 4;   // per-epilogue-warp 32x33 transpose scratch
  // one persistent CTA per SM: the ring takes what is left of the 227 KB
  static constexpr int kRing = (int)((212u * 1024u - kEpiBytes) / (kABytes + kBBytes));
  static constexpr int kStages = kRing > 8 ? 8 : kRing;
  static constexpr size_t kSmem = 1024 + (size_t)kStages * (kABytes + kBBytes) + kEpiBytes + 256;
  static_assert(kSmem + 1024 <= 227 * 1024, "shared memory budget");
};

// S32 tiles (3xTF32): a ring slot holds one 32-wide logical K block of A and B,
// each operand's hi half then its lo half (both loaded once, by one paired box);
// the MMA issuer forms hi*hi, hi*lo and lo*hi from the same slot
template <int BN>
struct CfgTf {
  static constexpr uint32_t kABytes = 2 * kBM * 128;  // 32 KB: [hi | lo] x 128 rows x 128 B
  static constexpr uint32_t kBBytes = 2 * BN * 128;
  static constexpr uint32_t kAccCols = BN < 32 ? 32 : BN;
  // TMEM per tile buffer: kMains accumulator PAIRS [main | correction] of 2 BN columns
  // (round-robin over the logical k-blocks).  One N = 2 BN MMA A_hi x [B_hi | B_lo]
  // writes main (hi*hi) and correction (hi*lo) side by side; an N = BN MMA A_lo x B_hi
  // adds lo*hi to the correction.  Double-buffered 256 columns for BN <= 64 (2 / 4
  // pairs), one buffer of 512 for BN = 128 (2 pairs; no epilogue / MMA overlap, but an
  // S32 tile spends far longer in the MMA than in the epilogue).
  static constexpr uint32_t kPairCols = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int kNumBuf = BN >= 128 ? 1 : 2;
  static constexpr uint32_t kBufCols = 512 / kNumBuf;
  static constexpr int kMains = (int)(kBufCols / kPairCols) > 4 ? 4 : (int)(kBufCols / kPairCols);
  static constexpr uint32_t kEpiBytes = 4 * 32 * 33 * 4;
  static constexpr int kRing = (int)((212u * 1024u - kEpiBytes) / (kABytes + kBBytes));
  static constexpr int kStages = kRing > 8 ? 8 : kRing;
  static constexpr size_t kSmem = 1024 + (size_t)kStages * (kABytes + kBBytes) + kEpiBytes + 256;
  static_assert(kMains >= 1 && kSmem + 1024 <= 227 * 1024, "S32 tile budget");
};

// Halo variant (3x3 stride-1 conv with 64 input channels, 64 output columns):
// the 9 filter taps stay resident in shared memory for the CTA's lifetime and
// each output tile streams its input halo ONCE, as one 4-D TMA box of
// `halo_rows` image rows x (W + 1) pixels starting at column -1: the extra
// column is TMA zero fill and serves as the left padding of every row and the
// right padding of the row before it.  Output tiles enumerate the same padded
// positions P = h (W + 1) + w of one image (128 per tile, crossing rows;
// w = W is a junk position the epilogue drops, 1 / (W + 1) of the MMA work),
// so tap (r, s) is the slot viewed from row (P0 mod (W + 1)) + r (W + 1) + s:
// a 128-byte-row shift of a swizzled tile is a plain descriptor start-address
// offset (the swizzle phase follows the absolute address bits -- verified by
// scripts/shift_test.cu).  Per tile ~(128 + 3 (W + 1)) x 128 B of L2 -> SMEM
// traffic instead of 9 x (16 + 8) KB for the plain implicit GEMM.
struct HaloCfg {
  static constexpr uint32_t kSlotBytes = 44 * 1024;  // halo_rows x (W + 1) pixel rows of 128 B
  static constexpr uint32_t kTapBytes = 64 * 128;    // one 64 x 64 bf16 filter tap
  static constexpr uint32_t kBResBytes = 9 * kTapBytes;
  static constexpr int kStages = 3;
  static constexpr uint32_t kAccCols = 64;
  static constexpr uint32_t kTmemCols = 128;
  static constexpr uint32_t kEpiBytes = 4 * 32 * 33 * 4;
  static constexpr size_t kSmem = 1024 + (size_t)kStages * kSlotBytes + kBResBytes + kEpiBytes + 256;
  static_assert(kSmem + 1024 <= 227 * 1024, "shared memory budget");
};

// fp32-class halo variant (S32 operands, 3x3 stride-1 conv with 64 input and 64
// output channels).  An S32 tile moves 4x the bytes of a bf16 one at half the MMA
// rate, and the streamed implicit GEMM sat at the per-SM L2 -> shared-memory ingest
// limit (~60 B/clk: 48 KB per 32-wide k-block against ~450 cycles of MMA; traced,
// scripts/gemm_trace.cu).  A 64-channel S32 filter (295 KB) cannot stay resident, so
// here the INPUT is the reused operand: per output tile and 32-channel block, one
// zero-padded halo box ([hi plane | lo plane], halo_rows x (W + 1) pixel rows of
// 128 B each) serves all 9 taps through row-shifted descriptors, and only the
// filter k-blocks stream through the ring -- 22 KB instead of 48 KB per k-block.
struct HaloTfCfg {
  static constexpr uint32_t kASlotBytes = 60 * 1024;  // 2 x halo_rows x (W + 1) x 128 B (W <= 32)
  static constexpr int kASlots = 2;                   // one per channel block in flight
  static constexpr uint32_t kBBytes = 2 * 64 * 128;   // [B_hi | B_lo] of one tap x 32 channels
  static constexpr int kStages = 5;
  static constexpr uint32_t kEpiBytes = 4 * 32 * 33 * 4;
  static constexpr size_t kSmem = 1024 + (size_t)kASlots * kASlotBytes + (size_t)kStages * kBBytes + kEpiBytes + 256;
  static_assert(kSmem + 1024 <= 227 * 1024, "shared memory budget");
};

__device__ __forceinline__ void pixel_coords(const ConvGeom& g, int64_t pix, int& n, int& oh, int& ow) {
  // 32-bit arithmetic: conv GEMM rows / pixel-K extents are < 2^31 (checked by conv_gemm)
  const uint32_t hw = (uint32_t)(g.OH * g.OW), p32 = (uint32_t)pix;
  const uint32_t nn = p32 / hw;
  const uint32_t rem = p32 - nn * hw;
  n = (int)nn;
  oh = (int)(rem / (uint32_t)g.OW);
  ow = (int)rem - oh * g.OW;
}

// (image, row, column) of a K-side pixel index advanced one 64-pixel k-block at a
// time: the producer thread's per-k-block 64-bit divisions were on its critical path
struct PixelCursor {
  int n, oh, ow, dr, dc;
  __device__ __forceinline__ void init(const ConvGeom& g, int64_t pix, int step = kBK) {
    pixel_coords(g, pix, n, oh, ow);
    dr = step / g.OW;
    dc = step - dr * g.OW;
  }
  __device__ __forceinline__ void advance(const ConvGeom& g) {
    ow += dc;
    oh += dr;
    if (ow >= g.OW) {
      ow -= g.OW;
      oh++;
    }
    while (oh >= g.OH) {
      oh -= g.OH;
      n++;
    }
  }
};

struct TapCursor {
  int cb, rs, r, sx;
  __device__ __forceinline__ void init(const ConvGeom& g, int kb) {
    cb = kb % g.cblocks;
    rs = kb / g.cblocks;
    r = rs / g.S;
    sx = rs - r * g.S;
  }
  __device__ __forceinline__ void advance(const ConvGeom& g) {
    if (++cb == g.cblocks) {
      cb = 0;
      ++rs;
      if (++sx == g.S) {
        sx = 0;
        ++r;
      }
    }
  }
};

__device__ __forceinline__ void ld_bf16x32(const uint16_t* src, float (&x)[32]) {
#pragma unroll
  for (int j = 0; j < 32; j += 8) {
    const uint4 q = *reinterpret_cast<const uint4*>(src + j);
    x[j + 0] = bf2f(q.x & 0xFFFF); x[j + 1] = bf2f(q.x >> 16);
    x[j + 2] = bf2f(q.y & 0xFFFF); x[j + 3] = bf2f(q.y >> 16);
    x[j + 4] = bf2f(q.z & 0xFFFF); x[j + 5] = bf2f(q.z >> 16);
    x[j + 6] = bf2f(q.w & 0xFFFF); x[j + 7] = bf2f(q.w >> 16);
  }
}
__device__ __forceinline__ void ld_f32x32(const float* src, float (&x)[32]) {
#pragma unroll
  for (int j = 0; j < 32; j += 4) {
    const float4 q = *reinterpret_cast<const float4*>(src + j);
    x[j] = q.x; x[j + 1] = q.y; x[j + 2] = q.z; x[j + 3] = q.w;
  }
}

template <int BN>
__device__ void epilogue_chunk_generic(const GemmParams& p, int64_t row, int64_t n_base, const float* v, int cnt,
                                       float* v_out);

// One thread's 32 consecutive outputs of one row.  Full, aligned chunks take a
// branch-free vector path per epilogue kind (the common case: every conv / MLP
// hidden layer); ragged or unaligned chunks fall back to the per-element path.
template <int BN, bool kTf = false>
__device__ __forceinline__ void epilogue_chunk(const GemmParams& p, int64_t row, int64_t n_base, float (&v)[32],
                                               int cnt, float (&vo)[32]) {
  const int epi = p.epi;
  const bool f32_out = (epi == DBS_EPI_F32 || epi == DBS_EPI_F32_ACCUM || epi == DBS_EPI_BIAS_F32 ||
                        epi == DBS_EPI_F32_ATOMIC);
  if (kTf && is_s32_epi(epi)) {  // (compiled into the S32 kernels only)
    // S32 output: row pitch 2 * ldd floats, the chunk is one 32-element block
    float x[32];
    const int64_t N = p.N;
#pragma unroll
    for (int j = 0; j < 32; j++) x[j] = (j < cnt && n_base + j < N) ? v[j] : 0.0f;
    if (epi == DBS_EPI_BIAS_RELU_S32) {
#pragma unroll
      for (int j = 0; j < 32; j++) x[j] = (j < cnt && n_base + j < N) ? fmaxf(x[j] + p.bias[n_base + j], 0.0f) : 0.0f;
    } else if (epi == DBS_EPI_RELU_GRAD_S32) {
      const float* ah = reinterpret_cast<const float*>(p.aux) + row * 2 * p.ldd + 2 * n_base;
#pragma unroll
      for (int j = 0; j < 32; j++) x[j] = ah[j] > 0.0f ? x[j] : 0.0f;
    }
    store_s32x32(reinterpret_cast<float*>(p.d) + row * 2 * p.ldd + 2 * n_base, x);
#pragma unroll
    for (int j = 0; j < 32; j++) vo[j] = x[j];
    return;
  }
  const int align_elems = f32_out ? 4 : 8;
  const bool fast = (cnt == 32) && !p.d_trans && (p.ldd % align_elems == 0) &&
                    ((reinterpret_cast<uintptr_t>(p.d) & 15) == 0) && (p.aux == nullptr || ((reinterpret_cast<uintptr_t>(p.aux) & 15) == 0)) &&
                    (p.bias == nullptr || ((reinterpret_cast<uintptr_t>(p.bias) & 15) == 0));
  if (!fast) {
    epilogue_chunk_generic<BN>(p, row, n_base, v, cnt, vo);
    return;
  }
  float x[32];
#pragma unroll
  for (int j = 0; j < 32; j++) x[j] = v[j];
  if (epi == DBS_EPI_BIAS_F32 || epi == DBS_EPI_BIAS_RELU_BF16) {
    float bb[32];
    ld_f32x32(p.bias + n_base, bb);
#pragma unroll
    for (int j = 0; j < 32; j++) x[j] += bb[j];
  }
  if (f32_out) {
    float* d = reinterpret_cast<float*>(p.d) + row * p.ldd + n_base;
    if (epi == DBS_EPI_F32_ACCUM) {
      float prev[32];
      ld_f32x32(d, prev);
#pragma unroll
      for (int j = 0; j < 32; j++) x[j] += prev[j];
    }
    if (epi == DBS_EPI_F32_ATOMIC) {
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        atomicAdd(reinterpret_cast<float4*>(d + j), make_float4(x[j], x[j + 1], x[j + 2], x[j + 3]));
    } else if (((reinterpret_cast<uintptr_t>(d)) & 31) == 0) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        float o[8];
#pragma unroll
        for (int u = 0; u < 8; u++) o[u] = x[j + u];
        stg8(d + j, v8_of(o));
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(d + j) = make_float4(x[j], x[j + 1], x[j + 2], x[j + 3]);
    }
  } else {
    uint16_t* d = reinterpret_cast<uint16_t*>(p.d) + row * p.ldd + n_base;
    if (epi == DBS_EPI_BIAS_RELU_BF16) {
#pragma unroll
      for (int j = 0; j < 32; j++) x[j] = fmaxf(x[j], 0.0f);
    } else if (epi == DBS_EPI_RELU_GRAD_BF16) {
      float a[32];
      ld_bf16x32(p.aux + row * p.ldd + n_base, a);
#pragma unroll
      for (int j = 0; j < 32; j++) x[j] = a[j] > 0.0f ? x[j] : 0.0f;
    } else if (epi == DBS_EPI_BF16_ACCUM) {
      float prev[32];
      ld_bf16x32(d, prev);
#pragma unroll
      for (int j = 0; j < 32; j++) x[j] += prev[j];
    }
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      uint4 q;
      q.x = pack_bf16x2(x[j + 0], x[j + 1]);
      q.y = pack_bf16x2(x[j + 2], x[j + 3]);
      q.z = pack_bf16x2(x[j + 4], x[j + 5]);
      q.w = pack_bf16x2(x[j + 6], x[j + 7]);
      *reinterpret_cast<uint4*>(d + j) = q;
    }
  }
#pragma unroll
  for (int j = 0; j < 32; j++) vo[j] = x[j];
}

template <int BN>
__device__ void epilogue_chunk_generic(const GemmParams& p, int64_t row, int64_t n_base, const float* v, int cnt,
                                       float* v_out) {
  const int64_t N = p.N;
  const bool full = (n_base + cnt <= N);
  switch (p.epi) {
    case DBS_EPI_F32:
    case DBS_EPI_F32_ACCUM:
    case DBS_EPI_BIAS_F32:
    case DBS_EPI_F32_ATOMIC: {
      float* d = reinterpret_cast<float*>(p.d) + row * p.ldd + n_base;
      float o[32];
#pragma unroll
      for (int j = 0; j < 32; j++) {
        if (j >= cnt) break;
        float x = v[j];
        if (p.epi == DBS_EPI_BIAS_F32 && n_base + j < N) x += p.bias[n_base + j];
        o[j] = x;
        v_out[j] = x;
      }
      const bool vec = full && cnt == 32 && ((reinterpret_cast<uintptr_t>(d) & 15) == 0);
      if (p.epi == DBS_EPI_F32_ACCUM) {
#pragma unroll
        for (int j = 0; j < 32; j++)
          if (j < cnt && n_base + j < N) d[j] += o[j];
      } else if (p.epi == DBS_EPI_F32_ATOMIC) {
        if (p.d_trans) {
          // transposed weight gradient: column j of this row is d[(n_base + j) * ldd + row];
          // consecutive lanes hold consecutive rows, so each reduction is warp-coalesced
          float* dt = reinterpret_cast<float*>(p.d) + n_base * p.ldd + row;
#pragma unroll
          for (int j = 0; j < 32; j++)
            if (j < cnt && n_base + j < N) atomicAdd(dt + j * p.ldd, o[j]);
        } else if (vec) {
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            atomicAdd(reinterpret_cast<float4*>(d + j), make_float4(o[j], o[j + 1], o[j + 2], o[j + 3]));
        } else {
#pragma unroll
          for (int j = 0; j < 32; j++)
            if (j < cnt && n_base + j < N) atomicAdd(d + j, o[j]);
        }
      } else if (vec) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(d + j) = make_float4(o[j], o[j + 1], o[j + 2], o[j + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; j++)
          if (j < cnt && n_base + j < N) d[j] = o[j];
      }
      break;
    }
    case DBS_EPI_BIAS_RELU_BF16:
    case DBS_EPI_BF16:
    case DBS_EPI_RELU_GRAD_BF16:
    case DBS_EPI_BF16_ACCUM: {
      uint16_t* d = reinterpret_cast<uint16_t*>(p.d) + row * p.ldd + n_base;
      const uint16_t* aux = p.aux ? p.aux + row * p.ldd + n_base : nullptr;
      const bool vec = full && cnt == 32 && ((reinterpret_cast<uintptr_t>(d) & 15) == 0);
      float prev[32];
      if (p.epi == DBS_EPI_BF16_ACCUM) {
        if (vec) {
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            const uint4 q = *reinterpret_cast<const uint4*>(d + j);
            prev[j + 0] = bf2f(q.x & 0xFFFF); prev[j + 1] = bf2f(q.x >> 16);
            prev[j + 2] = bf2f(q.y & 0xFFFF); prev[j + 3] = bf2f(q.y >> 16);
            prev[j + 4] = bf2f(q.z & 0xFFFF); prev[j + 5] = bf2f(q.z >> 16);
            prev[j + 6] = bf2f(q.w & 0xFFFF); prev[j + 7] = bf2f(q.w >> 16);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; j++) prev[j] = (j < cnt && n_base + j < N) ? bf2f(d[j]) : 0.0f;
        }
      }
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
        } else if (p.epi == DBS_EPI_BF16_ACCUM) {
          x += prev[j];
        }
        o[j] = f2bf(x);
        v_out[j] = x;
      }
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
#pragma unroll
        for (int j = 0; j < 32; j++)
          if (j < cnt && n_base + j < N) d[j] = o[j];
      }
      break;
    }
    default:
      break;
  }
}

// named barrier over the 4 epilogue warps (the producer / MMA warps never join)
__device__ __forceinline__ void epilogue_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// transpose-reduce 32 rows x 32 columns across the warp: lane j gets column j's sum
__device__ __forceinline__ float warp_colsum(float (&x)[32], int lane) {
  float mine = 0.0f;
#pragma unroll
  for (int j = 0; j < 32; j++) {
    float s = x[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == j) mine = s;
  }
  return mine;
}

// tile t -> (m tile fastest, then n tile, then split-K slice): the tiles
// resident at one time share their B block (and neighbouring A windows) in L2;
// returns the tile's k-block count (merged parity classes: class c's own count)
template <int BN>
__device__ __forceinline__ int tile_decode(const GemmParams& p, int64_t t, int64_t m_tiles, int64_t n_tiles,
                                           int num_k_total, int64_t& m0, int64_t& n0, int& kb_begin, int& cls) {
  cls = -1;
  if (p.nclass > 0) {  // merged classes: one N tile, no split-K
    int c = 0;
    while (c + 1 < p.nclass && t >= p.cls_start[c + 1]) c++;
    cls = c;
    m0 = (t - p.cls_start[c]) * kBM;
    n0 = 0;
    kb_begin = 0;
    return p.cls_kb[c];
  }
  // 32-bit divisions (tile counts are far below 2^31; a 64-bit division is a ~100-instruction
  // subroutine on every role's per-tile path)
  const uint32_t tt = (uint32_t)t, mt = (uint32_t)m_tiles, nt = (uint32_t)n_tiles;
  const uint32_t rest = tt / mt;
  m0 = (int64_t)(tt - rest * mt) * kBM;
  const uint32_t split = rest / nt;
  n0 = (int64_t)(rest - split * nt) * BN;
  kb_begin = (int)split * p.kb_per_split;
  const int kb_end = min(kb_begin + p.kb_per_split, num_k_total);
  return kb_end > kb_begin ? kb_end - kb_begin : 0;
}

// The non-halo TMA producer, specialised per operand-mode pair (AM / BMD < 0:
// runtime modes).  The single producer thread is the latency-critical path of
// the conv kernels: a compact loop with the other modes' branches compiled out
// keeps it short (and its code local), instead of one loop over every mode.
template <int BN, int AM, int BMD>
__device__ __forceinline__ void produce(const GemmParams& p, const CUtensorMap* tmA, const CUtensorMap* tmB, uint8_t* sA,
                                        uint8_t* sB, uint64_t* full, uint64_t* empty, int64_t num_tiles, int64_t m_tiles,
                                        int64_t n_tiles, int num_k_total) {
  using C = Cfg<BN>;
  constexpr int kStages = C::kStages;
  const int am = AM >= 0 ? AM : p.a_mode;
  const int bm = BMD >= 0 ? BMD : p.b_mode;
  uint32_t it = 0;  // ring position, continuous across tiles
  uint32_t pt = 0;
  (void)pt;
   for (int64_t t = blockIdx.x; t < num_tiles; t += gridDim.x) {
    int64_t m0, n0;
    int kb_begin, cls;
    const int num_k = tile_decode<BN>(p, t, m_tiles, n_tiles, num_k_total, m0, n0, kb_begin, cls);
    const ConvTaps& tp = cls >= 0 ? p.cls_taps[cls] : p.taps;
    int a_n = 0, a_oh = 0, a_ow = 0;
    if (am == 2 || am == 4) pixel_coords(p.ga, m0, a_n, a_oh, a_ow);
    int b_r = 0, b_s = 0, b_c0 = 0;
    if (bm == 2 || bm == 4) {
      const int rs = (int)(n0 / p.gb.Cin);
      b_c0 = (int)(n0 - (int64_t)rs * p.gb.Cin);
      b_r = rs / p.gb.S;
      b_s = rs - b_r * p.gb.S;
    }
    // transposed weight gradient: the tile's two 64-row halves are fixed (tap, channel block)s
    int at_r[2] = {0, 0}, at_s[2] = {0, 0}, at_c[2] = {0, 0};
    if (am >= 5) {
#pragma unroll
      for (int j = 0; j < 2; j++) {
        const int mj = (int)m0 + 64 * j;
        const int rs = mj / p.ga.Cin;
        at_c[j] = mj - rs * p.ga.Cin;
        at_r[j] = rs / p.ga.S;
        at_s[j] = rs - at_r[j] * p.ga.S;
      }
    }
    const ConvGeom& gk = am >= 5 ? p.ga : p.gb;  // geometry of a pixel-indexed K
    PixelCursor pc{};
    const bool k_pix = am >= 5 || bm == 2 || bm == 4;
    if (k_pix) pc.init(gk, (int64_t)kb_begin * kBK);
    // (tap, channel block) of the current k-block, advanced incrementally (no per-k-block division)
    constexpr bool kTapK = (AM == 2 || AM == 4 || BMD == 3);
    const bool tap_k = kTapK || (AM < 0 && (am == 2 || am == 4 || bm == 3));
    TapCursor tc{};
    if (tap_k) tc.init(p.ga, kb_begin);
    if (num_k > 0) { if ((threadIdx.x & 31) == 0) GEMM_TRACE(2 + pt); pt++; }
    if ((p.pair_a | p.pair_b) == 0) {
    for (int i = 0; i < num_k; i++, it++) {
      const int kb = kb_begin + i;
      const int s = (int)(it % kStages);
      mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
      if ((threadIdx.x & 31) == 0 && it < 12) GEMM_TRACE(100 + it);
      // MN-major A: the upper 64 rows of the tile are skipped when they lie past
      // M (e.g. the 64-channel weight gradient) -- their stale rows only reach
      // accumulator rows the epilogue masks
      const bool a_hi = (am != 1 && am < 5) || (m0 + 64 < p.M);
      mbar_arrive_expect_tx_w(&full[s], (a_hi ? C::kABytes : C::kABytes / 2) + C::kBBytes);
      const int32_t k0 = kb * kBK;
      uint8_t* a = sA + s * C::kABytes;
      uint8_t* b = sB + s * C::kBBytes;
      if (am == 0) {
        tma_load_2d_w(a, tmA, &full[s], k0, (int32_t)m0);
      } else if (am == 1) {
        tma_load_2d_w(a, tmA, &full[s], (int32_t)m0, k0);
        if (a_hi) tma_load_2d_w(a + 8192, tmA, &full[s], (int32_t)m0 + 64, k0);
      } else if (am >= 5) {
        // weight gradient, transposed: A[k = pixel][m = (r, s, c)] is the conv
        // input window of 64 output pixels at tap (r, s), channels c .. c + 63 --
        // one MN-major 64 x 64 box per 64-row half of the tile (mode 6: im2col TMA)
        const ConvGeom& g = p.ga;
#pragma unroll
        for (int j = 0; j < 2; j++) {
          if (j == 1 && !a_hi) break;
          if (am == 6)
            tma_load_im2col_4d_w(a + j * 8192, tmA, &full[s], at_c[j], pc.ow * g.stride - g.pad,
                               pc.oh * g.stride - g.pad, pc.n, (uint16_t)at_s[j], (uint16_t)at_r[j]);
          else
            tma_load_4d_w(a + j * 8192, tmA, &full[s], at_c[j], pc.ow * g.stride + at_s[j] - g.pad,
                        pc.oh * g.stride + at_r[j] - g.pad, pc.n);
        }
        pc.advance(g);  // (only in the pixel-K branches: the producer thread is latency-critical)
      } else if (am == 4) {
        // im2col TMA: 128 consecutive output pixels (crossing rows / images) of
        // the window corner, shifted by the tap; the tensor map's bounding box
        // starts at -pad (-1 for an explicit tap list, whose offsets are +1)
        const ConvGeom& g = p.ga;
        const int cb = tc.cb;
        const int rs = tc.rs;
        int h0, w0, oh, ow;
        if (tp.n > 0) {
          h0 = a_oh - 1;
          w0 = a_ow - 1;
          oh = tp.dh[rs] + 1;
          ow = tp.dw[rs] + 1;
        } else {
          oh = tc.r;
          ow = tc.sx;
          h0 = a_oh * g.stride - g.pad;
          w0 = a_ow * g.stride - g.pad;
        }
        tma_load_im2col_4d_w(a, tmA, &full[s], cb * 64, w0, h0, a_n, (uint16_t)ow, (uint16_t)oh);
      } else {
        const ConvGeom& g = p.ga;
        const int cb = tc.cb;
        const int rs = tc.rs;
        int ah, aw;
        if (tp.n > 0) {
          ah = a_oh + tp.dh[rs];
          aw = a_ow + tp.dw[rs];
        } else {
          const int r = tc.r, sx = tc.sx;
          ah = a_oh * g.stride + r - g.pad;
          aw = a_ow * g.stride + sx - g.pad;
        }
        tma_load_4d_w(a, tmA, &full[s], cb * 64, aw, ah, a_n);
      }
      if (bm == 0) {
        tma_load_2d_w(b, tmB, &full[s], k0, (int32_t)n0);
      } else if (bm == 1) {
#pragma unroll
        for (int j = 0; j < BN / 64; j++) tma_load_2d_w(b + j * 8192, tmB, &full[s], (int32_t)n0 + 64 * j, k0);
      } else if (bm == 3) {
        // input gradient: the filter W[k][r][s][c] read in place as the flipped,
        // transposed filter Wt[c][R-1-r][S-1-s][k] -- MN-major boxes of 64 c x 64 k
        const ConvGeom& g = p.ga;
        const int cb = tc.cb;
        const int rs = tc.rs;
        const int r = tc.r, sx = tc.sx;
        const int rs_flip = tp.n > 0 ? (int)tp.rs[rs] : (g.R - 1 - r) * g.S + (g.S - 1 - sx);
        if (p.b_wide) {
          tma_load_4d_w(b, tmB, &full[s], 0, cb * 64, (int32_t)(n0 >> 6), rs_flip);
        } else {
#pragma unroll
          for (int j = 0; j < BN / 64; j++) tma_load_3d_w(b + j * 8192, tmB, &full[s], (int32_t)n0 + 64 * j, rs_flip, cb * 64);
        }
      } else if (bm == 4) {
        const ConvGeom& g = p.gb;
        const int bn_ = pc.n, boh = pc.oh, bow = pc.ow;
#pragma unroll
        for (int j = 0; j < BN / 64; j++)
          tma_load_im2col_4d_w(b + j * 8192, tmB, &full[s], b_c0 + 64 * j, bow * g.stride - g.pad,
                             boh * g.stride - g.pad, bn_, (uint16_t)b_s, (uint16_t)b_r);
        pc.advance(g);
      } else {
        const ConvGeom& g = p.gb;
        const int bn_ = pc.n, boh = pc.oh, bow = pc.ow;
#pragma unroll
        for (int j = 0; j < BN / 64; j++)
          tma_load_4d_w(b + j * 8192, tmB, &full[s], b_c0 + 64 * j, bow * g.stride + b_s - g.pad,
                      boh * g.stride + b_r - g.pad, bn_);
        pc.advance(g);
      }
      if (tap_k) tc.advance(p.ga);
    }
    } else {
    // paired k-blocks (host guarantees an even k-block count per tile)
    for (int i = 0; i < num_k;) {
      constexpr int npair = 2;
      const int s0 = (int)(it % kStages);
      for (int u = 0; u < npair; u++)
        mbar_wait(&empty[s0 + u], (((it + u) / kStages) & 1) ^ 1);
      if ((threadIdx.x & 31) == 0 && it < 12) GEMM_TRACE(100 + it);
      // MN-major A: the upper 64 rows of the tile are skipped when they lie past
      // M (e.g. the 64-channel weight gradient) -- their stale rows only reach
      // accumulator rows the epilogue masks
      const bool a_hi = (am != 1 && am < 5) || (m0 + 64 < p.M);
      // a pair's bytes all complete on full[s0]; full[s0 + 1] gets a plain
      // arrival (the MMA reaches slot s0 + 1 only after full[s0] completed)
      mbar_arrive_expect_tx_w(&full[s0], npair * ((a_hi ? C::kABytes : C::kABytes / 2) + C::kBBytes));
      mbar_arrive_w(&full[s0 + 1]);
      for (int u = 0; u < npair; u++) {
      const int s = s0 + u;
      const int kb = kb_begin + i + u;
      const int32_t k0 = kb * kBK;
      uint8_t* a = sA + s * C::kABytes;
      uint8_t* b = sB + s * C::kBBytes;
      if (p.pair_a) {
        if (u == 0) {
          if (am >= 5) {
            // transposed weight gradient: one 128-pixel box per 64-row half fills
            // slot s0 + j with that half's k-blocks kb and kb + 1 (descriptor LBO 16 KB)
            const ConvGeom& g = p.ga;
#pragma unroll
            for (int j = 0; j < 2; j++) {
              if (j == 1 && !a_hi) break;
              uint8_t* aj = sA + (s0 + j) * C::kABytes;
              if (am == 6)
                tma_load_im2col_4d_w(aj, tmA, &full[s0], at_c[j], pc.ow * g.stride - g.pad, pc.oh * g.stride - g.pad,
                                   pc.n, (uint16_t)at_s[j], (uint16_t)at_r[j]);
              else
                tma_load_4d_w(aj, tmA, &full[s0], at_c[j], pc.ow * g.stride + at_s[j] - g.pad,
                            pc.oh * g.stride + at_r[j] - g.pad, pc.n);
            }
            pc.advance(g);
            pc.advance(g);
          } else if (am == 0) {
            tma_load_3d_w(a, tmA, &full[s0], 0, (int32_t)m0, kb);
          } else if (am == 1) {  // <= 64 rows: 128 k rows fill both halves of slot s0
            tma_load_2d_w(a, tmA, &full[s0], (int32_t)m0, k0);
          } else {
            const ConvGeom& g = p.ga;
            const int cb = tc.cb;
            const int rs = tc.rs;
            int ah, aw;
            if (tp.n > 0) {
              ah = a_oh + tp.dh[rs];
              aw = a_ow + tp.dw[rs];
            } else {
              const int r = tc.r, sx = tc.sx;
              ah = a_oh * g.stride + r - g.pad;
              aw = a_ow * g.stride + sx - g.pad;
            }
            tma_load_5d_w(a, tmA, &full[s0], 0, aw, ah, a_n, cb);
          }
        }
      } else if (am == 0) {
        tma_load_2d_w(a, tmA, &full[s0], k0, (int32_t)m0);
      } else if (am == 1) {
        tma_load_2d_w(a, tmA, &full[s0], (int32_t)m0, k0);
        if (a_hi) tma_load_2d_w(a + 8192, tmA, &full[s0], (int32_t)m0 + 64, k0);
      } else if (am == 4) {
        // im2col TMA: 128 consecutive output pixels (crossing rows / images) of
        // the window corner, shifted by the tap; the tensor map's bounding box
        // starts at -pad (-1 for an explicit tap list, whose offsets are +1)
        const ConvGeom& g = p.ga;
        const int cb = tc.cb;
        const int rs = tc.rs;
        int h0, w0, oh, ow;
        if (tp.n > 0) {
          h0 = a_oh - 1;
          w0 = a_ow - 1;
          oh = tp.dh[rs] + 1;
          ow = tp.dw[rs] + 1;
        } else {
          oh = tc.r;
          ow = tc.sx;
          h0 = a_oh * g.stride - g.pad;
          w0 = a_ow * g.stride - g.pad;
        }
        tma_load_im2col_4d_w(a, tmA, &full[s0], cb * 64, w0, h0, a_n, (uint16_t)ow, (uint16_t)oh);
      } else {
        const ConvGeom& g = p.ga;
        const int cb = tc.cb;
        const int rs = tc.rs;
        int ah, aw;
        if (tp.n > 0) {
          ah = a_oh + tp.dh[rs];
          aw = a_ow + tp.dw[rs];
        } else {
          const int r = tc.r, sx = tc.sx;
          ah = a_oh * g.stride + r - g.pad;
          aw = a_ow * g.stride + sx - g.pad;
        }
        tma_load_4d_w(a, tmA, &full[s0], cb * 64, aw, ah, a_n);
      }
      if (p.pair_b) {
        if (u == 0) {
          if (bm == 0) {
            tma_load_3d_w(b, tmB, &full[s0], 0, (int32_t)n0, kb);
          } else if (bm == 1) {  // BN = 64, MN-major: 128 k rows fill the B parts of slots s0, s0 + 1
            tma_load_2d_w(b, tmB, &full[s0], (int32_t)n0, k0);
          } else if (bm == 2 || bm == 4) {  // BN = 64: 128 output pixels in one box
            const ConvGeom& g = p.gb;
            const int bn_ = pc.n, boh = pc.oh, bow = pc.ow;
            if (bm == 4)
              tma_load_im2col_4d_w(b, tmB, &full[s0], b_c0, bow * g.stride - g.pad, boh * g.stride - g.pad, bn_,
                                 (uint16_t)b_s, (uint16_t)b_r);
            else
              tma_load_4d_w(b, tmB, &full[s0], b_c0, bow * g.stride + b_s - g.pad, boh * g.stride + b_r - g.pad, bn_);
            pc.advance(g);
            pc.advance(g);
          } else {  // mode 3, BN = 64: the two k-blocks are consecutive 64-row k ranges
            const ConvGeom& g = p.ga;
            const int cb = tc.cb;
            const int rs = tc.rs;
            const int r = tc.r, sx = tc.sx;
            const int rs_flip = tp.n > 0 ? (int)tp.rs[rs] : (g.R - 1 - r) * g.S + (g.S - 1 - sx);
            if (p.b_wide)  // BN >= 128: all channel blocks x 128 k rows in one 4-D box (pair_b 3)
              tma_load_4d_w(b, tmB, &full[s0], 0, cb * 64, (int32_t)(n0 >> 6), rs_flip);
            else
              tma_load_3d_w(b, tmB, &full[s0], (int32_t)n0, rs_flip, cb * 64);
          }
        }
      } else if (bm == 0) {
        tma_load_2d_w(b, tmB, &full[s0], k0, (int32_t)n0);
      } else if (bm == 1) {
#pragma unroll
        for (int j = 0; j < BN / 64; j++) tma_load_2d_w(b + j * 8192, tmB, &full[s0], (int32_t)n0 + 64 * j, k0);
      } else if (bm == 3) {
        // input gradient: the filter W[k][r][s][c] read in place as the flipped,
        // transposed filter Wt[c][R-1-r][S-1-s][k] -- MN-major boxes of 64 c x 64 k
        const ConvGeom& g = p.ga;
        const int cb = tc.cb;
        const int rs = tc.rs;
        const int r = tc.r, sx = tc.sx;
        const int rs_flip = tp.n > 0 ? (int)tp.rs[rs] : (g.R - 1 - r) * g.S + (g.S - 1 - sx);
        if (p.b_wide) {
          tma_load_4d_w(b, tmB, &full[s0], 0, cb * 64, (int32_t)(n0 >> 6), rs_flip);
        } else {
#pragma unroll
          for (int j = 0; j < BN / 64; j++) tma_load_3d_w(b + j * 8192, tmB, &full[s0], (int32_t)n0 + 64 * j, rs_flip, cb * 64);
        }
      } else if (bm == 4) {
        const ConvGeom& g = p.gb;
        const int bn_ = pc.n, boh = pc.oh, bow = pc.ow;
#pragma unroll
        for (int j = 0; j < BN / 64; j++)
          tma_load_im2col_4d_w(b + j * 8192, tmB, &full[s0], b_c0 + 64 * j, bow * g.stride - g.pad,
                             boh * g.stride - g.pad, bn_, (uint16_t)b_s, (uint16_t)b_r);
        pc.advance(g);
      } else {
        const ConvGeom& g = p.gb;
        const int bn_ = pc.n, boh = pc.oh, bow = pc.ow;
#pragma unroll
        for (int j = 0; j < BN / 64; j++)
          tma_load_4d_w(b + j * 8192, tmB, &full[s0], b_c0 + 64 * j, bow * g.stride + b_s - g.pad,
                      boh * g.stride + b_r - g.pad, bn_);
        pc.advance(g);
      }
      if (tap_k) tc.advance(p.ga);
      }
      it += npair;
      i += npair;
    }
    }
   }
}

// TMA producer for S32 operands (3xTF32).  One ring slot = one 32-wide logical K
// block: A as [hi | lo] and B as [hi | lo], each half in the canonical layout of a
// 128-byte k-block (K-major: rows x 128 B; MN-major: 32-column groups of 32 K rows
// x 128 B, each group followed by its lo group -- the SWIZZLE_128B_BASE32B layout).
// The tensor maps view S32 bytes as bf16 units (4 per logical element) with a
// hi/lo dimension of stride 128 B, so ONE box fetches both halves (except im2col
// maps: two boxes).  The MMA issuer then runs (A hi, B hi), (A hi, B lo), (A lo, B hi).
template <int BN>
// (called by the whole producer warp: one elected lane issues each TMA / arrive)
__device__ __forceinline__ void produce_tf(const GemmParams& p, const CUtensorMap* tmA, const CUtensorMap* tmB,
                                           uint8_t* sA, uint8_t* sB, uint64_t* full, uint64_t* empty,
                                           int64_t num_tiles, int64_t m_tiles, int64_t n_tiles, int num_k_total) {
  using C = CfgTf<BN>;
  constexpr int kStages = C::kStages;
  const int am = p.a_mode, bm = p.b_mode;
  uint32_t it = 0;
  for (int64_t t = blockIdx.x; t < num_tiles; t += gridDim.x) {
    int64_t m0, n0;
    int kb_begin, cls;
    const int num_k = tile_decode<BN>(p, t, m_tiles, n_tiles, num_k_total, m0, n0, kb_begin, cls);
    const ConvTaps& tp = cls >= 0 ? p.cls_taps[cls] : p.taps;
    int a_n = 0, a_oh = 0, a_ow = 0;
    if (am == 2 || am == 4) pixel_coords(p.ga, m0, a_n, a_oh, a_ow);
    int b_r = 0, b_s = 0, b_c0 = 0;
    if (bm == 2 || bm == 4) {
      const int rs = (int)(n0 / p.gb.Cin);
      b_c0 = (int)(n0 - (int64_t)rs * p.gb.Cin);
      b_r = rs / p.gb.S;
      b_s = rs - b_r * p.gb.S;
    }
    const bool k_pix = (bm == 2 || bm == 4 || am >= 5);
    const ConvGeom& gk = am >= 5 ? p.ga : p.gb;  // geometry of the pixel-indexed K
    PixelCursor pc{};
    if (k_pix) pc.init(gk, (int64_t)kb_begin * 32, 32);
    const bool tap_k = (am == 2 || am == 4 || bm == 3);
    TapCursor tc{};
    if (tap_k) tc.init(p.ga, kb_begin);
    // transposed weight gradient (A = the conv input, MN-major over M = (r, s, c)): the
    // tile's 32-row groups are fixed (tap, channel group)s; groups past M are skipped
    int at_r[4] = {0, 0, 0, 0}, at_s[4] = {0, 0, 0, 0}, at_c[4] = {0, 0, 0, 0};
    int a_groups = 4;
    if (am >= 5) {
      a_groups = (int)min((int64_t)4, (p.M - m0 + 31) / 32);
#pragma unroll
      for (int gq = 0; gq < 4; gq++) {
        const int mg = (int)m0 + 32 * gq;
        const int rs = mg / p.ga.Cin;
        at_c[gq] = mg - rs * p.ga.Cin;
        at_r[gq] = rs / p.ga.S;
        at_s[gq] = rs - at_r[gq] * p.ga.S;
      }
    }
    const uint32_t a_bytes = am >= 5 ? (uint32_t)a_groups * 8192u : C::kABytes;
    // transposed weight gradient, K-paired (p.pair_a == 5): each box covers the k-block pair
    // (i, i + 1) = 64 pixels, landing in ring slots s, s + 1 as per group [hi 64 rows | lo 64
    // rows] (A) and [hi groups | lo groups] of 64 rows (B) -- half the TMA operations of the
    // producer-bound 64-channel weight gradient; the MMA issuer addresses the pair layout
    const bool kp5 = am == 5 && p.pair_a == 5;
    for (int i = 0; i < num_k; i++, it++) {
      const int L = kb_begin + i;
      const int s = (int)(it % kStages);
      mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
      if ((threadIdx.x & 31) == 0 && it - 36u < 12u) GEMM_TRACE(100 + (it - 36));  // (trace window: ring positions 36..47)
      if (kp5 && (i & 1)) {
        mbar_arrive_w(&full[s]);  // its bytes completed on slot s - 1's barrier
        if (k_pix) pc.advance(gk);
        continue;
      }
      if (kp5) mbar_wait(&empty[s + 1], (((it + 1) / kStages) & 1) ^ 1);
      if DBS_GEMM_DBG_BIT(p, 1) {  // attribution run: the ring without its loads
        mbar_arrive_w(&full[s]);  // (K-paired: the odd k-block arrives on its own slot above)
        if (tap_k) tc.advance(p.ga);
        if (k_pix) pc.advance(gk);
        continue;
      }
      mbar_arrive_expect_tx_w(&full[s], (a_bytes + C::kBBytes) * (kp5 ? 2u : 1u));
      uint8_t* a = sA + s * C::kABytes;
      uint8_t* b = sB + s * C::kBBytes;
      if (am >= 5) {
        const ConvGeom& g = p.ga;
#pragma unroll
        for (int gq = 0; gq < 4; gq++) {  // (constant trip count: at_* stay in registers)
          if (gq >= a_groups) break;
          if (kp5) {
            tma_load_5d_w(a + gq * 16384, tmA, &full[s], 0, pc.ow * g.stride + at_s[gq] - g.pad,
                        pc.oh * g.stride + at_r[gq] - g.pad, pc.n, 2 * (at_c[gq] / 32));
          } else if (am == 6) {
            const int cu = at_c[gq] * 4;
            tma_load_im2col_4d_w(a + gq * 8192, tmA, &full[s], cu, pc.ow * g.stride - g.pad, pc.oh * g.stride - g.pad,
                               pc.n, (uint16_t)at_s[gq], (uint16_t)at_r[gq]);
            tma_load_im2col_4d_w(a + gq * 8192 + 4096, tmA, &full[s], cu + 64, pc.ow * g.stride - g.pad,
                               pc.oh * g.stride - g.pad, pc.n, (uint16_t)at_s[gq], (uint16_t)at_r[gq]);
          } else {
            tma_load_5d_w(a + gq * 8192, tmA, &full[s], 0, pc.ow * g.stride + at_s[gq] - g.pad,
                        pc.oh * g.stride + at_r[gq] - g.pad, pc.n, 2 * (at_c[gq] / 32));
          }
        }
      } else if (am == 0) {
        tma_load_3d_w(a, tmA, &full[s], 0, (int32_t)m0, 2 * L);  // {64, 128 rows, hi/lo}
      } else if (am == 1) {
        tma_load_4d_w(a, tmA, &full[s], 0, L * 32, 0, (int32_t)(m0 / 32));  // {64, 32 k, hi/lo, 4 groups}
      } else if (am == 4) {
        const ConvGeom& g = p.ga;
        int h0, w0, oh, ow;
        if (tp.n > 0) {
          h0 = a_oh - 1;
          w0 = a_ow - 1;
          oh = tp.dh[tc.rs] + 1;
          ow = tp.dw[tc.rs] + 1;
        } else {
          oh = tc.r;
          ow = tc.sx;
          h0 = a_oh * g.stride - g.pad;
          w0 = a_ow * g.stride - g.pad;
        }
        tma_load_im2col_4d_w(a, tmA, &full[s], tc.cb * 128, w0, h0, a_n, (uint16_t)ow, (uint16_t)oh);
        tma_load_im2col_4d_w(a + kBM * 128, tmA, &full[s], tc.cb * 128 + 64, w0, h0, a_n, (uint16_t)ow, (uint16_t)oh);
      } else {
        const ConvGeom& g = p.ga;
        int ah, aw;
        if (tp.n > 0) {
          ah = a_oh + tp.dh[tc.rs];
          aw = a_ow + tp.dw[tc.rs];
        } else {
          ah = a_oh * g.stride + tc.r - g.pad;
          aw = a_ow * g.stride + tc.sx - g.pad;
        }
        tma_load_5d_w(a, tmA, &full[s], 0, aw, ah, a_n, 2 * tc.cb);  // {64, pixels..., hi/lo}
      }
      // B lands as [B_hi (BN columns) | B_lo (BN columns)]: one N = 2 BN operand
      if (bm == 0) {
        tma_load_3d_w(b, tmB, &full[s], 0, (int32_t)n0, 2 * L);  // {64, BN rows, hi/lo}
      } else if (bm == 1) {
        tma_load_4d_w(b, tmB, &full[s], 0, L * 32, (int32_t)(n0 / 32), 0);  // {64, 32 k, groups, hi/lo}
      } else if (bm == 3) {
        const ConvGeom& g = p.ga;
        const int rs_flip = tp.n > 0 ? (int)tp.rs[tc.rs] : (g.R - 1 - tc.r) * g.S + (g.S - 1 - tc.sx);
        tma_load_5d_w(b, tmB, &full[s], 0, tc.cb * 32, (int32_t)(n0 / 32), 0, rs_flip);  // {64, 32 k, groups, hi/lo, rs}
      } else {
        const ConvGeom& g = p.gb;
        constexpr uint32_t kLoB = BN * 128;
#pragma unroll
        for (int j = 0; j < BN / 32; j++) {
          const int cu = (b_c0 / 32 + j) * 128;
          if (bm == 4) {
            tma_load_im2col_4d_w(b + j * 4096, tmB, &full[s], cu, pc.ow * g.stride - g.pad, pc.oh * g.stride - g.pad,
                               pc.n, (uint16_t)b_s, (uint16_t)b_r);
            tma_load_im2col_4d_w(b + kLoB + j * 4096, tmB, &full[s], cu + 64, pc.ow * g.stride - g.pad,
                               pc.oh * g.stride - g.pad, pc.n, (uint16_t)b_s, (uint16_t)b_r);
          } else if (p.pair_b == 2) {
            // all BN / 32 groups of the tile (one tap, consecutive channels) in ONE box
            // {64, 32 pixels, 2 x BN / 32 sub-blocks}: [hi g | lo g] per group as below
            if (j == 0)
              tma_load_5d_w(b, tmB, &full[s], 0, pc.ow * g.stride + b_s - g.pad, pc.oh * g.stride + b_r - g.pad, pc.n,
                          2 * (b_c0 / 32));
          } else {
            // one {64, 32 pixels, hi/lo} box per group: [hi g | lo g] pairs (group stride 8 KB),
            // the un-fused layout (3 MMAs per k-step, see the issuer) -- half the TMA operations
            tma_load_5d_w(b + j * 8192, tmB, &full[s], 0, pc.ow * g.stride + b_s - g.pad,
                        pc.oh * g.stride + b_r - g.pad, pc.n, 2 * (b_c0 / 32 + j));
          }
        }
      }
      if (tap_k) tc.advance(p.ga);
      if (k_pix) pc.advance(gk);
    }
  }
}

template <int BN>
__device__ __forceinline__ void produce_dispatch(const GemmParams& p, const CUtensorMap* tmA, const CUtensorMap* tmB,
                                                 uint8_t* sA, uint8_t* sB, uint64_t* full, uint64_t* empty,
                                                 int64_t num_tiles, int64_t m_tiles, int64_t n_tiles, int num_k_total) {
#define DBS_PRODUCE(A, B) produce<BN, A, B>(p, tmA, tmB, sA, sB, full, empty, num_tiles, m_tiles, n_tiles, num_k_total)
  if constexpr (BN == 16) {
    DBS_PRODUCE(-1, -1);
  } else {
    switch (p.a_mode * 8 + p.b_mode) {
      case 2 * 8 + 0: DBS_PRODUCE(2, 0); break;  // conv forward, 4-D box A
      case 4 * 8 + 0: DBS_PRODUCE(4, 0); break;  // conv forward, im2col A
      case 2 * 8 + 3: DBS_PRODUCE(2, 3); break;  // input gradient (flipped filter B)
      case 4 * 8 + 3: DBS_PRODUCE(4, 3); break;
      case 1 * 8 + 2: DBS_PRODUCE(1, 2); break;  // weight gradient dY^T im2col(X)
      case 1 * 8 + 4: DBS_PRODUCE(1, 4); break;
      case 5 * 8 + 1: DBS_PRODUCE(5, 1); break;  // transposed weight gradient X^T dY
      case 6 * 8 + 1: DBS_PRODUCE(6, 1); break;
      default: DBS_PRODUCE(-1, -1); break;       // plain GEMMs (modes 0 / 1)
    }
  }
#undef DBS_PRODUCE
}

// kTf: S32 operands, kind::tf32, three virtual k-blocks per 32-wide logical K block (produce_tf)
template <int BN, bool kHalo, bool kTf = false>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmParams p) {
  using C = Cfg<BN>;
  using H = HaloCfg;
  static_assert(!kHalo || BN == 64, "halo variant: 64 output columns");
  constexpr bool kHT = kHalo && kTf;  // fp32-class halo variant (HaloTfCfg)
  using HT = HaloTfCfg;
  using CT = CfgTf<BN < 128 ? BN : 128>;
  constexpr int kStages = kHT ? HT::kStages : (kHalo ? H::kStages : (kTf ? CT::kStages : C::kStages));
  constexpr uint32_t kAccCols = kHalo ? H::kAccCols : C::kAccCols;
  // S32: each tile buffer holds CT::kMains main accumulators (hi*hi, round-robin over
  // the logical k-blocks) and one correction accumulator (hi*lo + lo*hi, 2^-11 smaller),
  // summed in fp32 (round to nearest) by the epilogue.  The tensor core's in-TMEM
  // accumulation truncates: every accumulator step costs up to one ulp of the running
  // sum, so fewer steps per accumulator = fewer truncations (gemm accuracy test).
  static_assert(!kTf || BN <= 128, "S32 tiles: BN <= 128");
  constexpr int kMains = kTf ? CT::kMains : 1;
  constexpr uint32_t kBufCols = kTf ? CT::kBufCols : kAccCols;
  constexpr int kNumBuf = kTf ? CT::kNumBuf : 2;  // accumulator buffers (tile j uses j % kNumBuf)
  // S32 BN = 128: the buffer split is chosen per launch (p.tf_nbuf); mains is 1, 2 or 4
  constexpr bool kRtBuf = kTf && BN >= 128;
  const int nbuf = kRtBuf ? p.tf_nbuf : kNumBuf;
  const int mains = kRtBuf ? (p.tf_nbuf == 2 ? 1 : kMains) : kMains;
  const uint32_t bufcols = kRtBuf ? 512u / (uint32_t)p.tf_nbuf : kBufCols;
  // all 512 columns: the allocation then starts at TMEM address 0, a compile-time constant
  // for the warp-wide issuers (a base read back from shared memory is not warp-uniform)
  constexpr uint32_t kTmemCols = 512u;
  constexpr uint32_t kSlotA = kHT ? HT::kASlotBytes : (kHalo ? H::kSlotBytes : (kTf ? CT::kABytes : C::kABytes));
  constexpr uint32_t kSlotB = kHT ? HT::kBBytes : (kHalo ? 0u : (kTf ? CT::kBBytes : C::kBBytes));
  constexpr uint32_t kBRes = (kHalo && !kHT) ? H::kBResBytes : 0u;
  constexpr int kASlots = kHT ? HT::kASlots : kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kASlots * kSlotA;  // ring B slots, or the resident filter (halo)
  float* sEpi = reinterpret_cast<float*>(sB + kStages * kSlotB + kBRes);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sEpi) + C::kEpiBytes);
  uint64_t* empty = full + kStages;
  uint64_t* acc_full = empty + kStages;  // [2] MMA -> epilogue
  uint64_t* acc_empty = acc_full + 2;    // [2] epilogue -> MMA
  uint64_t* bres_full = acc_empty + 2;   // resident filter landed (halo)
  uint64_t* a_full = bres_full + 1;      // [2] halo slot landed (kHT)
  uint64_t* a_empty = a_full + 2;        // [2] halo slot consumed by its 9 taps (kHT)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) GEMM_TRACE(0);
  const int64_t m_tiles = (p.M + kBM - 1) / kBM;
  const int64_t n_tiles = (p.N + BN - 1) / BN;
  const int64_t num_tiles = kHalo ? p.halo_tiles : (p.nclass > 0 ? p.cls_start[p.nclass] : m_tiles * n_tiles * p.splits);
  const int num_k_total = kTf ? (int)((p.K + 31) / 32) : (int)((p.K + kBK - 1) / kBK);
  const int a_mn = (p.a_mode == 1 || p.a_mode >= 5) ? 1 : 0;
  const int b_mn = (p.b_mode >= 1) ? 1 : 0;
  // tile t -> (m0, n0, first k-block, class); returns the tile's k-block count (tile_decode)
  auto decode = [&](int64_t t, int64_t& m0, int64_t& n0, int& kb_begin, int& cls) -> int {
    return tile_decode<BN>(p, t, m_tiles, n_tiles, num_k_total, m0, n0, kb_begin, cls);
  };


  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < kStages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);  // one arrival per epilogue warp
    }
    mbar_init(bres_full, 1);
    for (int b = 0; b < 2; b++) {
      mbar_init(&a_full[b], 1);
      mbar_init(&a_empty[b], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (tmem_base != 0u) __trap();  // the issuers address the whole-TMEM allocation from 0
  // everything above overlapped the previous kernel's tail; operands and outputs only from here
  pdl_trigger_and_wait();
  if (threadIdx.x == 0) GEMM_TRACE(1);

  if (warp == 0) {
    {  // (the whole warp runs the producer; one elected lane issues each TMA / arrive)
   // ---------------- TMA producer ----------------
   uint32_t it = 0;  // ring position, continuous across tiles
   uint32_t pt = 0;
   (void)pt;
   if constexpr (kHT) {
    // per tile and 32-channel block: one [hi | lo] halo box, then the 9 taps' filter k-blocks
    const ConvGeom& g = p.ga;
    const int W1 = g.OW + 1;
    const uint32_t a_bytes = 2u * (uint32_t)(p.halo_rows * W1) * 128u;
    uint32_t ia = 0;
    for (int64_t t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      if (lane == 0 && pt < 10) GEMM_TRACE(2 + pt);
      pt++;
      const int img = (int)((uint32_t)t / (uint32_t)p.halo_tpi);
      const int P0 = (int)(t - (int64_t)img * p.halo_tpi) * kBM;
      for (int cb = 0; cb < g.cblocks; cb++, ia++) {
        const int sa = (int)(ia & 1);
        mbar_wait(&a_empty[sa], ((ia >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx_w(&a_full[sa], a_bytes);
        tma_load_5d_w(sA + sa * kSlotA, &tmA, &a_full[sa], 0, -1, P0 / W1 - 1, img, 2 * cb);  // {64, W+1, rows, 1, hi/lo}
        for (int tap = 0; tap < 9; tap++, it++) {
          const int s = (int)(it % kStages);
          mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
          if (lane == 0 && it < 12) GEMM_TRACE(100 + it);
          mbar_arrive_expect_tx_w(&full[s], kSlotB);
          uint8_t* b = sB + s * kSlotB;
          if (p.b_mode == 0) {
            tma_load_3d_w(b, &tmB, &full[s], 0, 0, 2 * (tap * g.cblocks + cb));  // {64, 64 rows, hi/lo}
          } else {  // flipped filter of the input gradient, MN-major {64, 32 k, groups, hi/lo, rs}
            tma_load_5d_w(b, &tmB, &full[s], 0, cb * 32, 0, 0, 8 - tap);
          }
        }
      }
    }
   } else if constexpr (kHalo) {
    // the 9 filter taps, once per CTA
    mbar_arrive_expect_tx_w(bres_full, H::kBResBytes);
    for (int tap = 0; tap < 9; tap++) {
      uint8_t* b = sB + tap * H::kTapBytes;
      if (p.b_mode == 0) {
        tma_load_2d_w(b, &tmB, bres_full, tap * 64, 0);
      } else {  // mode 3: flipped, transposed filter of the input gradient
        tma_load_3d_w(b, &tmB, bres_full, 0, 8 - tap, 0);
      }
    }
    const ConvGeom& g = p.ga;
    const int W1 = g.OW + 1;
    const uint32_t halo_bytes = (uint32_t)(p.halo_rows * W1) * 128u;
    for (int64_t t = blockIdx.x; t < num_tiles; t += gridDim.x, it++) {
      if ((threadIdx.x & 31) == 0 && pt < 10) GEMM_TRACE(2 + pt);
      pt++;
      const int img = (int)((uint32_t)t / (uint32_t)p.halo_tpi);
      const int P0 = (int)(t - (int64_t)img * p.halo_tpi) * kBM;
      const int s = (int)(it % kStages);
      mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
      mbar_arrive_expect_tx_w(&full[s], halo_bytes);
      // rows from one above the tile's first row, columns from -1 (zero fill)
      tma_load_4d_w(sA + s * kSlotA, &tmA, &full[s], 0, -1, P0 / W1 - 1, img);
    }
   } else if constexpr (kTf) {
   produce_tf<BN>(p, &tmA, &tmB, sA, sB, full, empty, num_tiles, m_tiles, n_tiles, num_k_total);
   } else {
   produce_dispatch<BN>(p, &tmA, &tmB, sA, sB, full, empty, num_tiles, m_tiles, n_tiles, num_k_total);
   }
    }
    __syncwarp();
  } else if (warp == 1) {
    // (the whole warp runs the issuer loop and one elected lane issues, so the
    // descriptors / TMEM addresses stay warp-uniform -- see mma_tf32_ss_warp)
    {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = kTf ? make_idesc_tf32(kBM, BN, a_mn, b_mn) : make_idesc_bf16(kBM, BN, a_mn, b_mn);
    uint32_t it = 0, j = 0;
    if constexpr (kHT) {
      const int W1 = p.ga.OW + 1;
      const uint32_t a_lo = (uint32_t)(p.halo_rows * W1) * 8u;  // lo plane, 16-byte units
      const uint64_t a_desc0 = make_sdesc(smem_u32(sA), 16, 1024);
      const uint64_t b_desc0 = b_mn ? make_sdesc(smem_u32(sB), 4096, 512, 1) : make_sdesc(smem_u32(sB), 16, 1024);
      const uint32_t b_kstep = b_mn ? 64u : 2u;  // UMMA_K = 8: 8 K rows / 32 B
      const uint32_t idesc1 = make_idesc_tf32(kBM, BN, 0, b_mn);
      const uint32_t idesc2 = make_idesc_tf32(kBM, 2 * BN, 0, b_mn);  // A_hi x [B_hi | B_lo]
      uint32_t ia = 0;
      for (int64_t t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int b = (int)(j & 1);
        mbar_wait(&acc_empty[b], ((j >> 1) & 1) ^ 1);
        if (lane == 0 && j < 10) GEMM_TRACE(12 + j);
        tc_fence_after();
        const uint32_t d_buf = b * kBufCols;  // (whole-TMEM allocation at address 0)
        const int img = (int)((uint32_t)t / (uint32_t)p.halo_tpi);
        const int off = ((int)(t - (int64_t)img * p.halo_tpi) * kBM) % W1;
        int i = 0;  // logical k-block of the tile (main accumulator round robin)
        for (int cb = 0; cb < p.ga.cblocks; cb++, ia++) {
          const int sa = (int)(ia & 1);
          mbar_wait(&a_full[sa], (ia >> 1) & 1);
          tc_fence_after();
          const uint64_t a_slot = a_desc0 + (uint64_t)((sa * kSlotA) >> 4);
#pragma unroll 1
          for (int tap = 0; tap < 9; tap++, it++, i++) {
            const int s = (int)(it % kStages);
            mbar_wait(&full[s], (it / kStages) & 1);
            if (lane == 0 && it < 12) GEMM_TRACE(112 + it);
            tc_fence_after();
            const int r = tap / 3, sx = tap - 3 * (tap / 3);
            const uint64_t a_hi = a_slot + (uint64_t)((off + r * W1 + sx) * 8);  // 128-byte rows
            const uint64_t b_hi = b_desc0 + (uint64_t)((s * kSlotB) >> 4);
            const uint32_t d_main = d_buf + (i % kMains) * CT::kPairCols;  // [main | correction] pair
#pragma unroll
            for (int k = 0; k < 4; k++) {
              const uint32_t acc = (i < kMains && k == 0) ? 0u : 1u;
              mma_tf32_ss_warp(d_main, a_hi + k * 2, b_hi + k * b_kstep, idesc2, acc);
              mma_tf32_ss_warp(d_main + BN, a_hi + a_lo + k * 2, b_hi + k * b_kstep, idesc1, 1u);
            }
            mma_commit_warp(&empty[s]);
            if (lane == 0 && it < 12) GEMM_TRACE(64 + it);
          }
          mma_commit_warp(&a_empty[sa]);
        }
        mma_commit_warp(&acc_full[b]);
        if (lane == 0 && j < 10) GEMM_TRACE(22 + j);
        j++;
      }
    } else if constexpr (kHalo) {
      mbar_wait(bres_full, 0);
      tc_fence_after();
      // descriptors by arithmetic on the 16-byte address field (no per-MMA
      // re-encoding: the MMA thread's issue rate, not the tensor pipe, was the limit)
      const int W1 = p.ga.OW + 1;
      const uint64_t a_desc0 = make_sdesc(smem_u32(sA), 16, 1024);
      const uint64_t b_desc0 = b_mn ? make_sdesc(smem_u32(sB), 8192, 1024) : make_sdesc(smem_u32(sB), 16, 1024);
      const uint32_t b_kstep = b_mn ? 128u : 2u;
      for (int64_t t = blockIdx.x; t < num_tiles; t += gridDim.x, it++) {
        const int b = (int)(j & 1);
        mbar_wait(&acc_empty[b], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        if ((threadIdx.x & 31) == 0) GEMM_TRACE(12 + j);
        const uint32_t d_tmem = b * kAccCols;  // (whole-TMEM allocation at address 0)
        const int s = (int)(it % kStages);
        mbar_wait(&full[s], (it / kStages) & 1);
        if ((threadIdx.x & 31) == 0 && j < 8) GEMM_TRACE(96 + 3 * j);
        tc_fence_after();
        const int img = (int)((uint32_t)t / (uint32_t)p.halo_tpi);
        const int off = ((int)(t - (int64_t)img * p.halo_tpi) * kBM) % W1;
        const uint64_t a_slot = a_desc0 + (uint64_t)((s * kSlotA) >> 4);
#pragma unroll
        for (int r = 0; r < 3; r++) {
#pragma unroll
          for (int sx = 0; sx < 3; sx++) {
            const uint64_t a_t = a_slot + (uint64_t)((off + r * W1 + sx) * 8);  // 128-byte rows
            const uint64_t b_t = b_desc0 + (uint64_t)((r * 3 + sx) * (H::kTapBytes >> 4));
#pragma unroll
            for (int k = 0; k < kBK / 16; k++)
              mma_bf16_ss_warp(d_tmem, a_t + (uint64_t)(k * 2), b_t + (uint64_t)(k * b_kstep), idesc,
                          (r | sx | k) != 0 ? 1u : 0u);
          }
        }
        mma_commit_warp(&empty[s]);
        mma_commit_warp(&acc_full[b]);
        if ((threadIdx.x & 31) == 0) GEMM_TRACE(22 + j);
        j++;
      }
    } else {
    if constexpr (kTf) {
    // ---- S32 slots: [A hi | A lo], [B hi | B lo] of one logical k-block ----
    // MN-major halves: 32-column groups of 32 K rows (4 KB), hi and lo of a group
    // adjacent (group stride LBO = 8 KB), SWIZZLE_128B_BASE32B (4-row K groups 512 B apart)
    // A: MN-major groups [hi | lo] per 32 columns (group stride 8 KB); B: [all hi | all lo]
    // (MN-major groups 4 KB apart), so B_hi:B_lo is ONE N = 2 BN operand
    // (K-paired transposed weight gradient: 64-row groups, group strides doubled, lo planes
    // 8 KB after hi, the odd k-block of a pair 32 rows (4 KB) into the pair's groups)
    const bool kp5 = p.a_mode == 5 && p.pair_a == 5;
    const uint64_t a_desc0 = a_mn ? make_sdesc(smem_u32(sA), kp5 ? 16384 : 8192, 512, 1)
                                  : make_sdesc(smem_u32(sA), 16, 1024);
    // (B mode 2, the 4-D-box weight-gradient operand, keeps [hi | lo] per group: 3 MMAs per k-step)
    const bool b_pairs = p.b_mode == 2;
    const uint64_t b_desc0 = b_mn ? make_sdesc(smem_u32(sB), (b_pairs || kp5) ? 8192 : 4096, 512, 1)
                                  : make_sdesc(smem_u32(sB), 16, 1024);
    const uint32_t b_lo = b_pairs ? 4096u >> 4 : 0u;
    const uint32_t a_lo = a_mn ? (kp5 ? 8192u : 4096u) >> 4 : (uint32_t)(kBM * 128) >> 4;  // lo half, 16-byte units
    const uint32_t a_kstep = a_mn ? 64u : 2u, b_kstep = b_mn ? 64u : 2u;  // UMMA_K = 8: 8 K rows / 32 B
    const uint32_t idesc2 = make_idesc_tf32(kBM, 2 * BN, a_mn, b_mn);  // A_hi x [B_hi | B_lo]
    for (int64_t t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      int64_t m0, n0;
      int kb_begin, cls;
      const int num_k = decode(t, m0, n0, kb_begin, cls);
      if (num_k == 0) continue;
      const int b = nbuf == 1 ? 0 : (int)(j & 1);
      mbar_wait(&acc_empty[b], (nbuf == 1 ? (j & 1) : ((j >> 1) & 1)) ^ 1);
      if (lane == 0 && j < 10) GEMM_TRACE(12 + j);
      tc_fence_after();
      const uint32_t d_buf = b * bufcols;  // (the 512-column allocation starts at TMEM address 0)
      for (int i = 0; i < num_k; i++, it++) {
        const int s = (int)(it % kStages);
        mbar_wait(&full[s], (it / kStages) & 1);
        if (lane == 0 && it - 36u < 12u) GEMM_TRACE(112 + (it - 36));
        tc_fence_after();
        const uint32_t d_main = d_buf + (i & (mains - 1)) * CT::kPairCols;  // [main | correction] pair
        const uint32_t a_off = kp5 ? (uint32_t)((s & ~1) * kSlotA + (s & 1) * 4096) : (uint32_t)(s * kSlotA);
        const uint32_t b_off = kp5 ? (uint32_t)((s & ~1) * kSlotB + (s & 1) * 4096) : (uint32_t)(s * kSlotB);
        const uint64_t a_hi = a_desc0 + (uint64_t)(a_off >> 4), b_hi = b_desc0 + (uint64_t)(b_off >> 4);
        if DBS_GEMM_DBG_BIT(p, 2) {
          // attribution run: the ring without its MMAs
        } else if (!b_pairs) {
#pragma unroll
          for (int k = 0; k < 4; k++) {
            const uint32_t acc = (i < mains && k == 0) ? 0u : 1u;
            mma_tf32_ss_warp(d_main, a_hi + k * a_kstep, b_hi + k * b_kstep, idesc2, acc);
            mma_tf32_ss_warp(d_main + BN, a_hi + a_lo + k * a_kstep, b_hi + k * b_kstep, idesc, 1u);
          }
        } else {
#pragma unroll
          for (int k = 0; k < 4; k++) {
            const uint32_t acc = (i < mains && k == 0) ? 0u : 1u;
            mma_tf32_ss_warp(d_main, a_hi + k * a_kstep, b_hi + k * b_kstep, idesc, acc);
            mma_tf32_ss_warp(d_main + BN, a_hi + k * a_kstep, b_hi + b_lo + k * b_kstep, idesc, acc);
            mma_tf32_ss_warp(d_main + BN, a_hi + a_lo + k * a_kstep, b_hi + k * b_kstep, idesc, 1u);
          }
        }
        mma_commit_warp(&empty[s]);
        if (lane == 0 && it - 36u < 12u) GEMM_TRACE(64 + (it - 36));
      }
      // (a short tile, num_k < kMains, leaves the higher mains unwritten: the epilogue skips them)
      mma_commit_warp(&acc_full[b]);
      if (lane == 0 && j < 10) GEMM_TRACE(22 + j);
      j++;
    }
    } else {
    const uint64_t a_desc0 = a_mn ? make_sdesc(smem_u32(sA), p.pair_a == 3 ? 16384 : 8192, 1024)
                                  : make_sdesc(smem_u32(sA), 16, 1024);
    // (pair_b == 3: a paired wide flipped-filter box put the 64-channel blocks 16 KB
    // apart, k-block kb + 1 8 KB after kb)
    const uint64_t b_desc0 = b_mn ? make_sdesc(smem_u32(sB), p.pair_b == 3 ? 16384 : 8192, 1024)
                                  : make_sdesc(smem_u32(sB), 16, 1024);
    const uint32_t a_kstep = a_mn ? 128u : 2u, b_kstep = b_mn ? 128u : 2u;  // one UMMA_K step, 16 B units
    for (int64_t t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      int64_t m0, n0;
      int kb_begin, cls;
      const int num_k = decode(t, m0, n0, kb_begin, cls);
      if (num_k == 0) continue;
      const int b = (int)(j & 1);
      mbar_wait(&acc_empty[b], ((j >> 1) & 1) ^ 1);  // epilogue drained this accumulator
      if ((threadIdx.x & 31) == 0) GEMM_TRACE(12 + j);
      tc_fence_after();
      const uint32_t d_tmem = b * kAccCols;  // (whole-TMEM allocation at address 0)
      for (int i = 0; i < num_k; i++, it++) {
        const int s = (int)(it % kStages);
        mbar_wait(&full[s], (it / kStages) & 1);
        if ((threadIdx.x & 31) == 0 && it < 12) GEMM_TRACE(112 + it);
        tc_fence_after();
        // (pair_a == 2: an MN-major A of <= 64 rows whose paired box put k-block
        // kb + 1 in the unused upper half of slot s - 1)
        const uint32_t a_off = p.pair_a >= 2 ? (uint32_t)((s & ~1) * C::kABytes + (s & 1) * 8192)
                                             : (uint32_t)(s * C::kABytes);
        const uint64_t a_s = a_desc0 + (uint64_t)(a_off >> 4);
        const uint32_t b_off = p.pair_b == 3 ? (uint32_t)((s & ~1) * C::kBBytes + (s & 1) * 8192)
                                             : (uint32_t)(s * C::kBBytes);
        const uint64_t b_s = b_desc0 + (uint64_t)(b_off >> 4);
#pragma unroll
        for (int k = 0; k < kBK / 16; k++)
          mma_bf16_ss_warp(d_tmem, a_s + (uint64_t)(k * a_kstep), b_s + (uint64_t)(k * b_kstep), idesc,
                      (i | k) != 0 ? 1u : 0u);
        mma_commit_warp(&empty[s]);
      }
      mma_commit_warp(&acc_full[b]);
      if ((threadIdx.x & 31) == 0) GEMM_TRACE(22 + j);
      j++;
    }
    }
    }
    }
    __syncwarp();
  } else {
  // ---------------- epilogue (warps 2..5) ----------------
  // two compiled copies: plain bf16 output with every chunk staged (conv forward /
  // input gradient -- the hot case, compact code) and everything else
  __shared__ float red_s[4][32], red_q[4][32];  // per-warp BN-statistics partials (both copies)
  auto epilogue_loop = [&](auto kst) {
  constexpr bool kSt = decltype(kst)::value;
  const int q = warp & 3;  // the TMEM lane quadrant this warp may access
  float* tr = sEpi + (warp - 2) * (32 * 33);
  uint32_t tj = 0;
  for (int64_t t = blockIdx.x; t < num_tiles; t += gridDim.x) {
    int64_t m0 = 0, n0 = 0;
    int kb_begin, cls = -1;
    const int tile_k = kHT ? 9 * p.ga.cblocks : (kHalo ? 1 : decode(t, m0, n0, kb_begin, cls));
    if (tile_k == 0) continue;
    const int nmain = tile_k < mains ? tile_k : mains;  // S32: main accumulators this tile wrote
    (void)nmain;
    const OutMap& om = cls >= 0 ? p.cls_omap[cls] : p.omap;
    const int b = nbuf == 1 ? 0 : (int)(tj & 1);
    mbar_wait(&acc_full[b], nbuf == 1 ? (tj & 1) : ((tj >> 1) & 1));
    if DBS_GEMM_DBG_BIT(p, 4) {  // attribution run: no epilogue work
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[b]);
      tj++;
      continue;
    }
    if (warp == 2 && lane == 0 && tj < 10) GEMM_TRACE(32 + tj);
    tc_fence_after();
    int64_t row = m0 + q * 32 + lane;
    int64_t orow = row;  // the output row this thread writes
    bool valid = row < p.M;
    if (kHalo) {
      // padded position P = h (W + 1) + w of image img; w = W is junk
      const int W1 = p.ga.OW + 1;
      const int img = (int)((uint32_t)t / (uint32_t)p.halo_tpi);
      const int P = (int)(t - (int64_t)img * p.halo_tpi) * kBM + q * 32 + lane;
      const int h = P / W1, w = P - (P / W1) * W1;
      valid = (w < p.ga.OW) && (h < p.ga.OH);
      orow = ((int64_t)img * p.ga.OH + h) * p.ga.OW + w;
      row = orow;
    } else if (om.on && row < p.M) {
      const uint32_t hw = (uint32_t)(om.OH * om.OW), r32 = (uint32_t)row;
      const int64_t img = r32 / hw;
      const int rem = (int)(r32 - (uint32_t)img * hw);
      const int i = rem / om.OW, jj = rem - i * om.OW;
      orow = (img * om.H + 2 * i + om.a) * om.W + 2 * jj + om.b;
    }
    const uint32_t lane_addr = tmem_base + b * bufcols + ((uint32_t)(q * 32) << 16);
    const bool stats = (p.sum_part != nullptr);
    // S32: fold the other main accumulators and the correction accumulator of chunk c
    // into r (fp32 adds, round to nearest; the corrections last)
    // (rc: pair 0's correction chunk, prefetched with the next main chunk -- one TMEM
    // round trip instead of two on the epilogue's serial path; same summation order)
    uint32_t rc[kTf ? 32 : 1];
    auto prefetch_corr = [&](int c) {
      if constexpr (kTf) tmem_ld_32x32b_x32(lane_addr + BN + c * 32, rc);
    };
    auto add_corr_pref = [&](int c, uint32_t (&r)[32]) {
      if constexpr (kTf) {
#pragma unroll
        for (int k = 0; k < 32; k++) r[k] = __float_as_uint(__uint_as_float(r[k]) + __uint_as_float(rc[k]));
        uint32_t r2[32];
        for (int m = 1; m < nmain; m++) {
          for (int half = 0; half < 2; half++) {
            tmem_ld_32x32b_x32(lane_addr + m * CT::kPairCols + half * BN + c * 32, r2);
            tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 32; k++) r[k] = __float_as_uint(__uint_as_float(r[k]) + __uint_as_float(r2[k]));
          }
        }
      }
    };
    auto add_corr = [&](int c, uint32_t (&r)[32]) {
      if constexpr (kTf) {
        // r holds pair 0's main chunk: add the other pairs' mains, then every correction
        uint32_t r2[32];
        for (int m = 0; m < nmain; m++) {
          for (int half = (m == 0); half < 2; half++) {
            tmem_ld_32x32b_x32(lane_addr + m * CT::kPairCols + half * BN + c * 32, r2);
            tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 32; k++) r[k] = __float_as_uint(__uint_as_float(r[k]) + __uint_as_float(r2[k]));
          }
        }
      }
    };
    if (BN >= 32) {
      // software-pipelined TMEM reads: chunk c + 1 is loaded while chunk c is
      // stored (the registers are free once chunk c is packed / copied)
      uint32_t r[32];
      tmem_ld_32x32b_x32(lane_addr, r);
      tmem_ld_wait();
      add_corr(0, r);
#pragma unroll 1
      for (int c = 0; c < BN / 32; c++) {
        const int64_t n_base = n0 + c * 32;
        const bool last = (c == BN / 32 - 1) || (n_base + 32 >= p.N);  // warp-uniform
        if (last) {
          // accumulator fully read: hand it back to the MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[b]);
          if (warp == 2 && lane == 0 && tj < 10) GEMM_TRACE(42 + tj);
        }
        const bool prefetch = !last;
        const int cnt = (int)((p.N - n_base) < 32 ? (p.N - n_base) : 32);
        // plain bf16 output (conv forward / input gradient): packed straight from
        // the TMEM registers and staged through shared memory so each store
        // instruction writes 8 rows x 64 contiguous bytes (the epilogue warps are
        // alone on their schedulers: instruction count is the epilogue's cost)
        // (kSt: the host-checked all-chunks-staged case, compiled without the other paths)
        constexpr bool staged = kSt;
        (void)cnt;
        if (stats) {
          // BN batch statistics: warp column sums (a 32x33 transpose in shared
          // memory: 32 stores + 32 loads instead of 160 shuffles) -> tile sums
          // over the 4 epilogue warps -> one fp64 atomic per column and tile
          // one transpose: lane j reads column j and forms both sums
#pragma unroll
          for (int k = 0; k < 32; k++) tr[lane * 33 + k] = valid ? __uint_as_float(r[k]) : 0.0f;
          __syncwarp();
          float s = 0.f, sq = 0.f;
#pragma unroll
          for (int r2 = 0; r2 < 32; r2++) {
            const float e = tr[r2 * 33 + lane];
            s += e;
            sq = fmaf(e, e, sq);
          }
          __syncwarp();
          red_s[q][lane] = s;
          red_q[q][lane] = sq;
          epilogue_bar();
          if (warp == 2 && lane < cnt) {
            const double ts = (double)red_s[0][lane] + red_s[1][lane] + red_s[2][lane] + red_s[3][lane];
            const double tq = (double)red_q[0][lane] + red_q[1][lane] + red_q[2][lane] + red_q[3][lane];
            atomicAdd(p.sum_part + n_base + lane, ts);
            atomicAdd(p.sq_part + n_base + lane, tq);
          }
          epilogue_bar();
        }
        if (staged) {
          uint32_t* st = reinterpret_cast<uint32_t*>(tr);  // 32 rows x 20 words (16 + 4 pad) of this warp
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 4; j++)
            *reinterpret_cast<uint4*>(st + lane * 20 + 4 * j) = make_uint4(
                pack_bf16x2(__uint_as_float(r[8 * j]), __uint_as_float(r[8 * j + 1])),
                pack_bf16x2(__uint_as_float(r[8 * j + 2]), __uint_as_float(r[8 * j + 3])),
                pack_bf16x2(__uint_as_float(r[8 * j + 4]), __uint_as_float(r[8 * j + 5])),
                pack_bf16x2(__uint_as_float(r[8 * j + 6]), __uint_as_float(r[8 * j + 7])));
          if (prefetch) {
            tmem_ld_32x32b_x32(lane_addr + (c + 1) * 32, r);
            prefetch_corr(c + 1);
          }
          __syncwarp();
          uint16_t* dbase = reinterpret_cast<uint16_t*>(p.d) + n_base + (lane & 3) * 8;
          if (!kHalo && !om.on) {
            // identity row map: the storing lane forms its row itself
            const int64_t row_w = m0 + q * 32;
#pragma unroll
            for (int i = 0; i < 4; i++) {
              const int rr = 8 * i + (lane >> 2);
              const uint4 val = *reinterpret_cast<const uint4*>(st + rr * 20 + (lane & 3) * 4);
              if (row_w + rr < p.M) *reinterpret_cast<uint4*>(dbase + (row_w + rr) * p.ldd) = val;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 4; i++) {
              const int rr = 8 * i + (lane >> 2);
              const int64_t orow_r = __shfl_sync(0xffffffffu, orow, rr);
              const int valid_r = __shfl_sync(0xffffffffu, (int)valid, rr);
              if (valid_r)
                *reinterpret_cast<uint4*>(dbase + orow_r * p.ldd) =
                    *reinterpret_cast<const uint4*>(st + rr * 20 + (lane & 3) * 4);
            }
          }
          __syncwarp();
        } else if (p.d_trans) {
          // transposed weight gradient: a 32x33 shared-memory transpose so that each
          // reduction is a float4 over 4 consecutive rows of one column (8 per chunk
          // instead of 32 scalar ones; the split-K slices all hit the same lines)
#pragma unroll
          for (int k = 0; k < 32; k++) tr[lane * 33 + k] = valid ? __uint_as_float(r[k]) : 0.0f;
          if (prefetch) {
            tmem_ld_32x32b_x32(lane_addr + (c + 1) * 32, r);
            prefetch_corr(c + 1);
          }
          __syncwarp();
          const int rq = 4 * (lane & 7);
          const int64_t mrow = m0 + q * 32 + rq;
          float* dt = reinterpret_cast<float*>(p.d) + mrow;
#pragma unroll
          for (int u = 0; u < 8; u++) {
            const int col = 4 * u + (lane >> 3);
            const float4 v4 = make_float4(tr[rq * 33 + col], tr[(rq + 1) * 33 + col], tr[(rq + 2) * 33 + col],
                                          tr[(rq + 3) * 33 + col]);
            if (col < cnt && mrow < p.M) atomicAdd(reinterpret_cast<float4*>(dt + (n_base + col) * p.ldd), v4);
          }
          __syncwarp();
        } else {
          float v[32], vo[32];
#pragma unroll
          for (int k = 0; k < 32; k++) {
            v[k] = valid ? __uint_as_float(r[k]) : 0.0f;
            vo[k] = 0.0f;
          }
          if (prefetch) {
            tmem_ld_32x32b_x32(lane_addr + (c + 1) * 32, r);
            prefetch_corr(c + 1);
          }
          if (valid) epilogue_chunk<BN, kTf>(p, orow, n_base, v, cnt, vo);
          if (p.colsum_part != nullptr) {
            const int64_t g = (m0 >> 5) + q;
            const bool group_live = (m0 + q * 32 < p.M);
            const float s = warp_colsum(vo, lane);
            if (lane < cnt && group_live) p.colsum_part[g * p.N + n_base + lane] = s;
          }
        }
        if (prefetch) {
          tmem_ld_wait();
          add_corr_pref(c + 1, r);
        }
        if (last) break;
      }
    } else {
      uint32_t r[16];
      tmem_ld_32x32b_x16(lane_addr, r);
      tmem_ld_wait();
      if constexpr (kTf) {
        uint32_t r2[16];
        for (int m = 0; m < nmain; m++) {
          for (int half = (m == 0); half < 2; half++) {
            tmem_ld_32x32b_x16(lane_addr + m * CT::kPairCols + half * BN, r2);
            tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 16; k++) r[k] = __float_as_uint(__uint_as_float(r[k]) + __uint_as_float(r2[k]));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[b]);
      if (row < p.M && n0 < p.N) {
        float v[32], vo[32];
#pragma unroll
        for (int k = 0; k < 16; k++) v[k] = __uint_as_float(r[k]);
        const int cnt = (int)((p.N - n0) < 16 ? (p.N - n0) : 16);
        epilogue_chunk<BN, kTf>(p, orow, n0, v, cnt, vo);
      }
    }
    if (warp == 2 && lane == 0 && tj < 10) GEMM_TRACE(52 + tj);
    tj++;
  }
  };
  const bool all_staged = BN >= 32 && p.epi == DBS_EPI_BF16 && p.colsum_part == nullptr && !p.d_trans &&
                          p.N % 32 == 0 && p.ldd % 8 == 0 && ((reinterpret_cast<uintptr_t>(p.d) & 15) == 0);
  if (all_staged)
    epilogue_loop(std::true_type{});
  else
    epilogue_loop(std::false_type{});
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<kTmemCols>(tmem_base);
  if (threadIdx.x == 0) GEMM_TRACE(63);
}

// ---------------------------------------------------------------------------
// Halo conv on a CTA pair (forward, 3x3 / stride 1 / 64 -> 64): one
// tcgen05.mma.cta_group::2 (M = 256) covers the same 128-position tile of two
// images, one per CTA.  A single-CTA 128x64x16 MMA is capped at ~34% of the
// tensor peak by its ~95-cycle issue cost; the pair instruction (45 cycles for
// 256x64x16) reaches ~70% (profiles/mma_rate_r1.txt).  Pairing images (not
// neighbouring tiles) keeps both CTAs' halo slots at the same row shift, which
// the shared A descriptor needs.  Each CTA loads its own image's halo and half
// of the filter (output channels 32 r .. 32 r + 31, the N split of a pair MMA);
// the loads complete on the leader's barriers (mapa), the leader issues every
// MMA and multicasts its commits to both CTAs, and both epilogues drain their
// own 128 accumulator rows and arrive on the leader's acc_empty.
// ---------------------------------------------------------------------------
struct Halo2Cfg {
  static constexpr uint32_t kSlotBytes = 44 * 1024;
  static constexpr uint32_t kTapBytes = 32 * 128;  // this CTA's 32 output channels of one tap
  static constexpr uint32_t kBResBytes = 9 * kTapBytes;
  static constexpr int kStages = 3;
  static constexpr uint32_t kAccCols = 64;
  static constexpr uint32_t kTmemCols = 128;
  static constexpr uint32_t kEpiBytes = 4 * 32 * 33 * 4;
  static constexpr size_t kSmem = 1024 + (size_t)kStages * kSlotBytes + kBResBytes + kEpiBytes + 256;
  static_assert(kSmem + 1024 <= 227 * 1024, "shared memory budget");
};

__global__ void __launch_bounds__(kThreads, 1)
    halo_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmParams p) {
  using H = Halo2Cfg;
  constexpr int kStages = H::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * H::kSlotBytes;
  float* sEpi = reinterpret_cast<float*>(sB + H::kBResBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sEpi) + H::kEpiBytes);
  uint64_t* empty = full + kStages;
  uint64_t* acc_full = empty + kStages;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* bres_full = acc_empty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bres_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) GEMM_TRACE(0);
  const uint32_t crank = cluster_ctarank();
  const bool leader = (crank == 0);
  const ConvGeom& g = p.ga;
  const int W1 = g.OW + 1;
  const int64_t num_pairs = p.halo_tiles;
  const int64_t pair0 = blockIdx.x >> 1, pair_step = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < kStages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 8);  // 4 epilogue warps x 2 CTAs (the leader's copy is used)
    }
    mbar_init(bres_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair<H::kTmemCols>(tmem_slot);
  tc_fence_before();
  cluster_sync_all();  // both CTAs' barriers exist before any remote arrive / TMA completion
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) GEMM_TRACE(1);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs; completions on the leader) ----------------
      const uint32_t bres_cl = map_to_rank(smem_u32(bres_full), 0);
      if (leader) mbar_arrive_expect_tx(bres_full, 2 * H::kBResBytes);
      for (int tap = 0; tap < 9; tap++) tma_load_2d_cl(sB + tap * H::kTapBytes, &tmB, bres_cl, tap * 64, 32 * (int)crank);
      const uint32_t halo_bytes = (uint32_t)(p.halo_rows * W1) * 128u;
      uint32_t it = 0;
      for (int64_t q = pair0; q < num_pairs; q += pair_step, it++) {
        const int img = (int)(q / p.halo_tpi) * 2 + (int)crank;
        const int P0 = (int)(q - (q / p.halo_tpi) * p.halo_tpi) * kBM;
        const int s = (int)(it % kStages);
        mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
        if (it < 10) GEMM_TRACE(2 + it);
        if (leader) mbar_arrive_expect_tx(&full[s], 2 * halo_bytes);
        tma_load_4d_cl(sA + s * H::kSlotBytes, &tmA, map_to_rank(smem_u32(&full[s]), 0), 0, -1, P0 / W1 - 1, img);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ---------------- MMA issuer (leader only) ----------------
      const uint32_t idesc = make_idesc_bf16(256, 64, 0, 0);
      const uint64_t a_desc0 = make_sdesc(smem_u32(sA), 16, 1024);
      const uint64_t b_desc0 = make_sdesc(smem_u32(sB), 16, 1024);
      mbar_wait(bres_full, 0);
      tc_fence_after();
      uint32_t it = 0, j = 0;
      for (int64_t q = pair0; q < num_pairs; q += pair_step, it++, j++) {
        const int b = (int)(j & 1);
        mbar_wait(&acc_empty[b], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        if (j < 10) GEMM_TRACE(12 + j);
        const int s = (int)(it % kStages);
        mbar_wait(&full[s], (it / kStages) & 1);
        tc_fence_after();
        if (j < 8) GEMM_TRACE(96 + 3 * j);
        const int off = ((int)(q - (q / p.halo_tpi) * p.halo_tpi) * kBM) % W1;
        const uint64_t a_slot = a_desc0 + (uint64_t)((s * H::kSlotBytes) >> 4);
        const uint32_t d_tmem = tmem_base + b * H::kAccCols;
#pragma unroll
        for (int r = 0; r < 3; r++) {
#pragma unroll
          for (int sx = 0; sx < 3; sx++) {
            const uint64_t a_t = a_slot + (uint64_t)((off + r * W1 + sx) * 8);
            const uint64_t b_t = b_desc0 + (uint64_t)((r * 3 + sx) * (H::kTapBytes >> 4));
#pragma unroll
            for (int k = 0; k < kBK / 16; k++)
              mma_bf16_ss_pair(d_tmem, a_t + (uint64_t)(k * 2), b_t + (uint64_t)(k * 2), idesc,
                               (r | sx | k) != 0 ? 1u : 0u);
          }
        }
        mma_commit_pair(&empty[s], (uint16_t)3);
        mma_commit_pair(&acc_full[b], (uint16_t)3);
        if (j < 10) GEMM_TRACE(22 + j);
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue (warps 2..5 of both CTAs: their own 128 rows) ----------------
    const int qd = warp & 3;
    float* tr = sEpi + (warp - 2) * (32 * 33);
    const uint32_t acc_empty_cl0 = map_to_rank(smem_u32(&acc_empty[0]), 0);
    const uint32_t acc_empty_cl1 = map_to_rank(smem_u32(&acc_empty[1]), 0);
    const bool stats = (p.sum_part != nullptr);
    const int n_img = (int)(p.M / ((int64_t)g.OH * g.OW));
    uint32_t tj = 0;
    for (int64_t q = pair0; q < num_pairs; q += pair_step, tj++) {
      const int b = (int)(tj & 1);
      mbar_wait(&acc_full[b], (tj >> 1) & 1);
      tc_fence_after();
      if (warp == 2 && lane == 0 && tj < 10) GEMM_TRACE(32 + tj);
      const int img = (int)(q / p.halo_tpi) * 2 + (int)crank;
      const int P = (int)(q - (q / p.halo_tpi) * p.halo_tpi) * kBM + qd * 32 + lane;
      const int h = P / W1, w = P - (P / W1) * W1;
      const bool valid = (w < g.OW) && (h < g.OH) && (img < n_img);
      const int64_t orow = ((int64_t)img * g.OH + h) * g.OW + w;
      const uint32_t lane_addr = tmem_base + b * H::kAccCols + ((uint32_t)(qd * 32) << 16);
#pragma unroll 1
      for (int c = 0; c < 2; c++) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(lane_addr + c * 32, r);
        tmem_ld_wait();
        if (c == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(b ? acc_empty_cl1 : acc_empty_cl0);
          if (warp == 2 && lane == 0 && tj < 10) GEMM_TRACE(42 + tj);
        }
        const int n_base = c * 32;
        if (stats) {
          __shared__ float red_s2[4][32], red_q2[4][32];
#pragma unroll
          for (int k = 0; k < 32; k++) tr[lane * 33 + k] = valid ? __uint_as_float(r[k]) : 0.0f;
          __syncwarp();
          float s1 = 0.f, sq = 0.f;
#pragma unroll
          for (int r2 = 0; r2 < 32; r2++) {
            const float e = tr[r2 * 33 + lane];
            s1 += e;
            sq = fmaf(e, e, sq);
          }
          __syncwarp();
          red_s2[qd][lane] = s1;
          red_q2[qd][lane] = sq;
          epilogue_bar();
          if (warp == 2) {
            const double ts = (double)red_s2[0][lane] + red_s2[1][lane] + red_s2[2][lane] + red_s2[3][lane];
            const double tq = (double)red_q2[0][lane] + red_q2[1][lane] + red_q2[2][lane] + red_q2[3][lane];
            atomicAdd(p.sum_part + n_base + lane, ts);
            atomicAdd(p.sq_part + n_base + lane, tq);
          }
          epilogue_bar();
        }
        // bf16 tile staged through shared memory, 8 rows x 64 contiguous bytes per store
        uint32_t* st = reinterpret_cast<uint32_t*>(tr);
        __syncwarp();
#pragma unroll
        for (int jj = 0; jj < 4; jj++)
          *reinterpret_cast<uint4*>(st + lane * 20 + 4 * jj) = make_uint4(
              pack_bf16x2(__uint_as_float(r[8 * jj]), __uint_as_float(r[8 * jj + 1])),
              pack_bf16x2(__uint_as_float(r[8 * jj + 2]), __uint_as_float(r[8 * jj + 3])),
              pack_bf16x2(__uint_as_float(r[8 * jj + 4]), __uint_as_float(r[8 * jj + 5])),
              pack_bf16x2(__uint_as_float(r[8 * jj + 6]), __uint_as_float(r[8 * jj + 7])));
        __syncwarp();
        uint16_t* dbase = reinterpret_cast<uint16_t*>(p.d) + n_base + (lane & 3) * 8;
#pragma unroll
        for (int i = 0; i < 4; i++) {
          const int rr = 8 * i + (lane >> 2);
          const int64_t orow_r = __shfl_sync(0xffffffffu, orow, rr);
          const int valid_r = __shfl_sync(0xffffffffu, (int)valid, rr);
          if (valid_r)
            *reinterpret_cast<uint4*>(dbase + orow_r * p.ldd) =
                *reinterpret_cast<const uint4*>(st + rr * 20 + (lane & 3) * 4);
        }
        __syncwarp();
      }
    }
  }
  if (threadIdx.x == 64) GEMM_TRACE(52);
  tc_fence_before();
  cluster_sync_all();  // no CTA leaves while its peer may still signal it
  if (threadIdx.x == 0) GEMM_TRACE(63);
  if (warp == 1) tmem_dealloc_pair<H::kTmemCols>(tmem_base);
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
              uint32_t box1, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeTiledFn fn = encode_fn();
  DBS_REQUIRE(fn != nullptr, DBS_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
  DBS_REQUIRE(((uintptr_t)base & 15) == 0 && (ld_elems * 2) % 16 == 0, DBS_ERR_ARGUMENT,
              "TMA needs 16-byte aligned base and leading dimension (ld %% 8 == 0)");
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {box0, box1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  DBS_REQUIRE(r == CUDA_SUCCESS, DBS_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return DBS_OK;
}

// 4-D NHWC bf16 tensor [N][H][W][C]: box {64 c, bw*stride, bh*stride, bn}, traversal stride on W/H
int make_tmap_nhwc(CUtensorMap* tm, const void* base, const ConvTensor& t, int bw, int bh, int bn, int stride,
                   CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeTiledFn fn = encode_fn();
  DBS_REQUIRE(fn != nullptr, DBS_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
  DBS_REQUIRE(((uintptr_t)base & 15) == 0 && t.C % 64 == 0, DBS_ERR_ARGUMENT,
              "conv TMA: 16-byte aligned base and C %% 64 == 0 required");
  DBS_REQUIRE(bw * stride <= 256 && bh * stride <= 256 && bn <= 256, DBS_ERR_ARGUMENT, "conv TMA: box too large");
  cuuint64_t dims[4] = {(cuuint64_t)t.C, (cuuint64_t)t.W, (cuuint64_t)t.H, (cuuint64_t)t.N};
  cuuint64_t strides[3] = {(cuuint64_t)t.C * 2, (cuuint64_t)t.W * t.C * 2, (cuuint64_t)t.H * t.W * t.C * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)(bw * stride), (cuuint32_t)(bh * stride), (cuuint32_t)bn};
  cuuint32_t es[4] = {1, (cuuint32_t)stride, (cuuint32_t)stride, 1};
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  DBS_REQUIRE(r == CUDA_SUCCESS, DBS_ERR_CUDA, "cuTensorMapEncodeTiled (4d) failed (%d)", (int)r);
  return DBS_OK;
}

typedef CUresult (*EncodeIm2colFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeIm2colFn encode_im2col_fn() {
  static EncodeIm2colFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeIm2colFn>(p);
  });
  return fn;
}

// im2col view of a 4-D NHWC bf16 tensor: each load is `pixels` output pixels x
// 64 channels.  The bounding box of window corners is [lower, extent - 1 + upper]
// on H and W, walked with the conv stride, so the output grid is
// (extent + upper - lower - 1) / stride + 1 -- any feature-map size, a tile may
// cross rows and images (fprop / dgrad: lower = -pad, upper = pad - (k - 1)).
int make_tmap_im2col(CUtensorMap* tm, const void* base, const ConvTensor& t, int lower, int upper, int pixels,
                     int stride, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeIm2colFn fn = encode_im2col_fn();
  DBS_REQUIRE(fn != nullptr, DBS_ERR_UNSUPPORTED, "cuTensorMapEncodeIm2col unavailable");
  DBS_REQUIRE(((uintptr_t)base & 15) == 0 && t.C % 64 == 0, DBS_ERR_ARGUMENT,
              "im2col TMA: 16-byte aligned base and C %% 64 == 0 required");
  DBS_REQUIRE(pixels >= 1 && pixels <= 256 && lower >= -128 && upper <= 127, DBS_ERR_ARGUMENT,
              "im2col TMA: %d pixels, corners [%d, %d] out of range", pixels, lower, upper);
  cuuint64_t dims[4] = {(cuuint64_t)t.C, (cuuint64_t)t.W, (cuuint64_t)t.H, (cuuint64_t)t.N};
  cuuint64_t strides[3] = {(cuuint64_t)t.C * 2, (cuuint64_t)t.W * t.C * 2, (cuuint64_t)t.H * t.W * t.C * 2};
  int lo[2] = {lower, lower}, hi[2] = {upper, upper};
  cuuint32_t es[4] = {1, (cuuint32_t)stride, (cuuint32_t)stride, 1};
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, lo, hi, 64,
                  (cuuint32_t)pixels, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  DBS_REQUIRE(r == CUDA_SUCCESS, DBS_ERR_CUDA, "cuTensorMapEncodeIm2col failed (%d)", (int)r);
  // drivers up to 13.1 mis-set one descriptor bit for im2col maps of tensors
  // under 128 KB (the same correction CUTLASS applies)
  int drv = 0;
  cudaDriverGetVersion(&drv);
  if (drv <= 13010 && (uint64_t)t.N * t.H * t.W * t.C * 2 < 131072ull)
    reinterpret_cast<uint64_t*>(tm)[1] &= ~(1ull << 21);
  return DBS_OK;
}

// K-major [rows][ld] matrix viewed as {64 k, rows, K / 64 k-blocks}: one box of
// {64, box_rows, 2} fills two consecutive ring slots (K % 128 == 0 required)
int make_tmap_kpair(CUtensorMap* tm, const void* base, uint64_t K, uint64_t rows, uint64_t ld_elems,
                    uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  DBS_REQUIRE(fn != nullptr, DBS_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
  DBS_REQUIRE(((uintptr_t)base & 15) == 0 && (ld_elems * 2) % 16 == 0 && K % 128 == 0, DBS_ERR_ARGUMENT,
              "paired k-block view: aligned base, ld %% 8 == 0 and K %% 128 == 0 required");
  cuuint64_t dims[3] = {64, rows, K / 64};
  cuuint64_t strides[2] = {ld_elems * 2, 128};
  cuuint32_t box[3] = {64, box_rows, 2};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  DBS_REQUIRE(r == CUDA_SUCCESS, DBS_ERR_CUDA, "cuTensorMapEncodeTiled (k-pair) failed (%d)", (int)r);
  return DBS_OK;
}

// NHWC activation viewed as {64 c, W, H, N, C / 64 channel blocks}: one box of
// {64, bw, bh, bn, 2} fills two consecutive ring slots (two channel blocks of one tap)
int make_tmap_nhwc_pair(CUtensorMap* tm, const void* base, const ConvTensor& t, int bw, int bh, int bn, int stride,
                        CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B, int subblocks = 2) {
  EncodeTiledFn fn = encode_fn();
  DBS_REQUIRE(fn != nullptr, DBS_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
  DBS_REQUIRE(((uintptr_t)base & 15) == 0 && t.C % 128 == 0, DBS_ERR_ARGUMENT,
              "conv pair TMA: aligned base and C %% 128 == 0 required");
  cuuint64_t dims[5] = {64, (cuuint64_t)t.W, (cuuint64_t)t.H, (cuuint64_t)t.N, (cuuint64_t)t.C / 64};
  cuuint64_t strides[4] = {(cuuint64_t)t.C * 2, (cuuint64_t)t.W * t.C * 2, (cuuint64_t)t.H * t.W * t.C * 2, 128};
  cuuint32_t box[5] = {64, (cuuint32_t)(bw * stride), (cuuint32_t)(bh * stride), (cuuint32_t)bn,
                       (cuuint32_t)subblocks};
  cuuint32_t es[5] = {1, (cuuint32_t)stride, (cuuint32_t)stride, 1, 1};
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  DBS_REQUIRE(r == CUDA_SUCCESS, DBS_ERR_CUDA, "cuTensorMapEncodeTiled (5d pair) failed (%d)", (int)r);
  return DBS_OK;
}

// MN-major S32 matrix [K rows][ld] (logical ld, row pitch 8 ld bytes) viewed as
// {64 units, K rows, hi/lo, 32-column groups}: one box {64, 32, 2, groups} lands as
// per group [hi 32 rows x 128 B | lo 32 rows x 128 B] (SWIZZLE_128B_ATOM_32B)
// (hilo_outer: {64 units, K rows, groups, hi/lo} -> [all hi groups | all lo groups], the B form)
int make_tmap_s32_mn(CUtensorMap* tm, const void* base, uint64_t mn, uint64_t krows, uint64_t ld, uint32_t groups,
                     bool hilo_outer = false, uint32_t box_k = 32) {
  EncodeTiledFn fn = encode_fn();
  DBS_REQUIRE(fn != nullptr, DBS_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
  DBS_REQUIRE(((uintptr_t)base & 15) == 0 && ld % 32 == 0 && groups >= 1 && groups <= 8, DBS_ERR_ARGUMENT,
              "S32 MN-major view: aligned base, ld %% 32 == 0");
  cuuint64_t dims[4] = {64, krows, 2, (mn + 31) / 32};
  cuuint64_t strides[3] = {ld * 8, 128, 256};
  cuuint32_t box[4] = {64, box_k, 2, groups};
  if (hilo_outer) {
    dims[2] = (mn + 31) / 32;
    dims[3] = 2;
    strides[1] = 256;
    strides[2] = 128;
    box[2] = groups;
    box[3] = 2;
  }
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  DBS_REQUIRE(r == CUDA_SUCCESS, DBS_ERR_CUDA, "cuTensorMapEncodeTiled (S32 MN) failed (%d)", (int)r);
  return DBS_OK;
}

bool kpair_enabled() {
  static const bool on = [] {
    const char* e = getenv("DBS_KPAIR");
    return !(e && e[0] == '0');
  }();
  return on;
}

// the 4-D box path covers a tile of `rows` pixels only when it aligns with whole rows / images
bool pixel_box_fits(int OH, int OW, int rows) {
  const int hw = OH * OW;
  if (hw >= rows) return hw % rows == 0 && (rows % OW == 0 || OW % rows == 0);
  return rows % hw == 0;
}

bool force_im2col() {
  static const bool on = [] {
    const char* e = getenv("DBS_CONV_IM2COL");
    return e && e[0] == '1';
  }();
  return on;
}

// pixels of one box: `rows` consecutive output pixels in NHWC order -> (bw, bh, bn)
int pixel_box(int OH, int OW, int rows, int& bw, int& bh, int& bn) {
  const int hw = OH * OW;
  if (hw >= rows) {
    DBS_REQUIRE(hw % rows == 0 && (rows % OW == 0 || OW % rows == 0), DBS_ERR_ARGUMENT,
                "conv tile of %d pixels does not align with a %dx%d feature map", rows, OH, OW);
    if (OW >= rows) {
      bw = rows;
      bh = 1;
    } else {
      bw = OW;
      bh = rows / OW;
    }
    bn = 1;
  } else {
    DBS_REQUIRE(rows % hw == 0, DBS_ERR_ARGUMENT, "conv tile of %d pixels does not align with %dx%d", rows, OH, OW);
    bw = OW;
    bh = OH;
    bn = rows / hw;
  }
  return DBS_OK;
}

// Kernel attributes are per context (workers may launch from their own green
// context): remember the contexts in which each instantiation was configured.
void* current_ctx() {
  typedef CUresult (*GetCur)(CUcontext*);
  static GetCur fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuCtxGetCurrent", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<GetCur>(p);
  });
  CUcontext c = nullptr;
  if (fn) fn(&c);
  return c;
}

// S32 BN = 128 double buffering: largest k-step count per main accumulator
// (DBS_TF_DB_STEPS).  288 = the steps a main takes in the 512-channel 3x3 convs with two
// mains (K = 4608), so double buffering (K <= 2304 here: the 64 -> 128 .. 256 -> 256
// convs) adds no error beyond the worst single-buffer case; 128 -> 128 3x3 forward
// 172 -> 153 us in a 48-SM partition (profiles/r2/tf_double_buffer.txt)
int tf_db_steps() {
  static const int v = [] {
    const char* e = getenv("DBS_TF_DB_STEPS");
    return e ? atoi(e) : 288;
  }();
  return v;
}

template <int BN, bool kHalo = false, bool kTf = false>
int launch(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, int splits, cudaStream_t s) {
  constexpr size_t kSmem = (kHalo && kTf) ? HaloTfCfg::kSmem
                         : kHalo ? HaloCfg::kSmem : (kTf ? CfgTf<(BN < 128 ? BN : 128)>::kSmem : Cfg<BN>::kSmem);
  static thread_local void* seen[16] = {nullptr};
  static thread_local int nseen = 0;
  void* ctx = current_ctx();
  bool known = false;
  for (int i = 0; i < nseen; i++) known |= (seen[i] == ctx);
  if (!known) {
    DBS_CUDA_TRY(cudaFuncSetAttribute(gemm_bf16_kernel<BN, kHalo, kTf>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kSmem));
    if (nseen < 16) seen[nseen++] = ctx;
  }
  GemmParams q = p;
  q.splits = splits;
  static const int dbg = [] {
    const char* e = getenv("DBS_GEMM_DBG");
    return e ? atoi(e) : 0;
  }();
  q.dbg = kTf ? dbg : 0;
  if (kTf && BN >= 128) {
    // two accumulator buffers (one main each) when a tile accumulates at most
    // tf_db_steps() k-steps into its main; else one buffer of two mains (the tensor
    // core's in-TMEM accumulation truncates: fewer steps per accumulator = less error)
    int kbt = (int)((p.K + 31) / 32);
    if (splits > 1) kbt = p.kb_per_split;
    if (p.nclass > 0) {
      kbt = 0;
      for (int c = 0; c < p.nclass; c++) kbt = p.cls_kb[c] > kbt ? p.cls_kb[c] : kbt;
    }
    q.tf_nbuf = 4 * kbt <= tf_db_steps() ? 2 : 1;
  }

  // persistent: one CTA per SM of the current (possibly green) context
  const int64_t tiles = kHalo ? p.halo_tiles
                      : (p.nclass > 0 ? p.cls_start[p.nclass] : ((p.M + kBM - 1) / kBM) * ((p.N + BN - 1) / BN) * splits);
  const int64_t sms = current_sm_count();
  const unsigned grid = (unsigned)(tiles < sms ? tiles : sms);
  DBS_CUDA_TRY(launch_pdl(gemm_bf16_kernel<BN, kHalo, kTf>, dim3(grid), dim3(kThreads), kSmem, s, ta, tb, q));
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

// Experimental, off by default (DBS_HALO_PAIR=1 enables it): correct (same parity
// tests), but measured no faster than the single-CTA halo kernel -- with streamed,
// row-shifted operands the pair instruction takes ~86 cycles, so per-SM MMA time
// per tile is unchanged (profiles/ncu_conv_r1_summary.md) -- and a cluster launch
// inside a worker's SM partition competes with the co-running disturbance kernel.
bool halo_pair_enabled() {
  static const bool on = [] {
    const char* e = getenv("DBS_HALO_PAIR");
    return e && e[0] == '1';
  }();
  return on;
}

// the CTA-pair halo kernel: clusters of 2, persistent over image-pair tiles
int launch_halo_pair(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, cudaStream_t s) {
  constexpr size_t kSmem = Halo2Cfg::kSmem;
  static thread_local void* seen[16] = {nullptr};
  static thread_local int nseen = 0;
  void* ctx = current_ctx();
  bool known = false;
  for (int i = 0; i < nseen; i++) known |= (seen[i] == ctx);
  if (!known) {
    DBS_CUDA_TRY(cudaFuncSetAttribute(halo_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
    if (nseen < 16) seen[nseen++] = ctx;
  }
  const int64_t clusters_max = current_sm_count() / 2;
  const int64_t clusters = p.halo_tiles < clusters_max ? p.halo_tiles : clusters_max;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * (clusters > 0 ? clusters : 1)));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  DBS_CUDA_TRY(cudaLaunchKernelEx(&cfg, halo_pair_kernel, ta, tb, p));
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

int pick_bn(int64_t N, int b_mode) {
  if (N <= 16 && b_mode == 0) return 16;
  if (N <= 64) return 64;
  if (N <= 128) return 128;
  return 256;
}

int dispatch(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, int bn, int splits, cudaStream_t s,
             bool halo = false, bool tf = false) {
  if (tf) {
    if (halo) return launch<64, true, true>(ta, tb, p, 1, s);
    switch (bn) {
      case 16: return launch<16, false, true>(ta, tb, p, splits, s);
      case 64: return launch<64, false, true>(ta, tb, p, splits, s);
      default: return launch<128, false, true>(ta, tb, p, splits, s);
    }
  }
  if (halo) return launch<64, true>(ta, tb, p, 1, s);
  switch (bn) {
    case 16: return launch<16>(ta, tb, p, splits, s);
    case 64: return launch<64>(ta, tb, p, splits, s);
    case 128: return launch<128>(ta, tb, p, splits, s);
    default: return launch<256>(ta, tb, p, splits, s);
  }
}

}  // namespace

bool wide_filter_enabled() {
  static const bool on = [] {
    const char* e = getenv("DBS_WIDE_FILTER");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool halo_tf_fits(int OH, int OW) {
  const int W1 = OW + 1;
  const int rows = (OW + kBM - 1) / W1 + 3;
  return OH >= 1 && W1 <= 256 && rows <= 256 && 2u * (uint32_t)(rows * W1) * 128u <= HaloTfCfg::kASlotBytes;
}

bool halo_fits(int OH, int OW) {
  const int W1 = OW + 1;
  const int rows = (OW + kBM - 1) / W1 + 3;
  return OH >= 1 && W1 <= 256 && rows <= 256 && (uint32_t)(rows * W1) * 128u <= HaloCfg::kSlotBytes;
}

int preload_gemm() {
  // force-load every instantiation (lazy module loading must never happen while
  // a disturbance kernel owns SMs); also sets the shared-memory attribute
  DBS_CUDA_TRY(cudaFuncSetAttribute(gemm_bf16_kernel<16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg<16>::kSmem));
  DBS_CUDA_TRY(cudaFuncSetAttribute(gemm_bf16_kernel<64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg<64>::kSmem));
  DBS_CUDA_TRY(cudaFuncSetAttribute(gemm_bf16_kernel<128, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg<128>::kSmem));
  DBS_CUDA_TRY(cudaFuncSetAttribute(gemm_bf16_kernel<256, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg<256>::kSmem));
  DBS_CUDA_TRY(cudaFuncSetAttribute(gemm_bf16_kernel<64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)HaloCfg::kSmem));
  DBS_CUDA_TRY(cudaFuncSetAttribute(halo_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Halo2Cfg::kSmem));
  DBS_CUDA_TRY(cudaFuncSetAttribute(gemm_bf16_kernel<16, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CfgTf<16>::kSmem));
  DBS_CUDA_TRY(cudaFuncSetAttribute(gemm_bf16_kernel<64, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CfgTf<64>::kSmem));
  DBS_CUDA_TRY(cudaFuncSetAttribute(gemm_bf16_kernel<64, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)HaloTfCfg::kSmem));
  DBS_CUDA_TRY(cudaFuncSetAttribute(gemm_bf16_kernel<128, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CfgTf<128>::kSmem));
  return DBS_OK;
}

int gemm_bf16(const void* a, int a_mn, int64_t lda, const void* b, int b_mn, int64_t ldb, void* d, int64_t ldd,
              int64_t M, int64_t N, int64_t K, int epi, const float* bias, const void* aux, cudaStream_t s,
              float* colsum_part) {
  DBS_REQUIRE(M > 0 && N > 0 && K > 0 && a && b && d, DBS_ERR_ARGUMENT, "gemm: bad shape/pointers");
  DBS_REQUIRE((M / 128 + 1) * (N / 16 + 1) < (int64_t(1) << 31), DBS_ERR_ARGUMENT, "gemm: too many tiles");
  DBS_REQUIRE(epi >= DBS_EPI_F32 && epi <= DBS_EPI_BF16_ACCUM, DBS_ERR_ARGUMENT, "gemm: bad epilogue %d", epi);
  DBS_REQUIRE(!((epi == DBS_EPI_BIAS_RELU_BF16 || epi == DBS_EPI_BIAS_F32) && !bias), DBS_ERR_ARGUMENT,
              "gemm: epilogue needs bias");
  DBS_REQUIRE(!(epi == DBS_EPI_RELU_GRAD_BF16 && !aux), DBS_ERR_ARGUMENT, "gemm: epilogue needs aux");
  const int bn = pick_bn(N, b_mn);
  DBS_REQUIRE(!(colsum_part && bn < 32), DBS_ERR_ARGUMENT, "gemm: column sums need N > 16");
  CUtensorMap ta, tb;
  int st;
  // A: K-major [M][lda] -> box {64 K, 128 M};  MN-major [K][lda] -> box {64 M, 64 K}
  // K-major operands with K % 128 == 0: one box per two k-blocks (fewer TMA operations)
  const bool kp = kpair_enabled() && (K % 128 == 0) && (lda * 2) % 16 == 0 && (ldb * 2) % 16 == 0;
  const bool pa = kp && !a_mn, pb = kp && !b_mn;
  st = a_mn ? make_tmap(&ta, a, (uint64_t)M, (uint64_t)K, (uint64_t)lda, 64, 64)
       : pa ? make_tmap_kpair(&ta, a, (uint64_t)K, (uint64_t)M, (uint64_t)lda, 128)
            : make_tmap(&ta, a, (uint64_t)K, (uint64_t)M, (uint64_t)lda, 64, 128);
  if (st) return st;
  // B: K-major [N][ldb] -> box {64 K, BN};  MN-major [K][ldb] -> box {64 N, 64 K}
  st = b_mn ? make_tmap(&tb, b, (uint64_t)N, (uint64_t)K, (uint64_t)ldb, 64, 64)
       : pb ? make_tmap_kpair(&tb, b, (uint64_t)K, (uint64_t)N, (uint64_t)ldb, (uint32_t)bn)
            : make_tmap(&tb, b, (uint64_t)K, (uint64_t)N, (uint64_t)ldb, 64, (uint32_t)bn);
  if (st) return st;
  GemmParams p{};
  p.pair_a = pa;
  p.pair_b = pb;
  p.M = M;
  p.N = N;
  p.K = K;
  p.a_mode = a_mn;
  p.b_mode = b_mn;
  p.epi = epi;
  p.d = d;
  p.ldd = ldd;
  p.bias = bias;
  p.aux = reinterpret_cast<const uint16_t*>(aux);
  p.colsum_part = colsum_part;
  p.kb_per_split = (int)((K + kBK - 1) / kBK);
  return dispatch(ta, tb, p, bn, 1, s);
}

bool is_s32_epi_host(int epi) {
  return epi == DBS_EPI_S32 || epi == DBS_EPI_BIAS_RELU_S32 || epi == DBS_EPI_RELU_GRAD_S32;
}

// S32 operands: the tensor maps view the S32 bytes as bf16 units (4 per logical
// element); K-major rows {4 K32 units} (K32 = K rounded up to 32), MN-major rows
// {4 MN32 units}, 32-row boxes
int64_t ceil32(int64_t x) { return (x + 31) & ~int64_t(31); }
// MN-major tf32 operands: the SWIZZLE_128B_BASE32B smem layout (tcgen05.cuh make_sdesc)
constexpr CUtensorMapSwizzle kMnSwz = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;

int gemm_tf(const void* a, int a_mn, int64_t lda, const void* b, int b_mn, int64_t ldb, void* d, int64_t ldd,
            int64_t M, int64_t N, int64_t K, int epi, const float* bias, const void* aux, cudaStream_t s,
            float* colsum_part) {
  DBS_REQUIRE(M > 0 && N > 0 && K > 0 && a && b && d, DBS_ERR_ARGUMENT, "gemm_tf: bad shape/pointers");
  DBS_REQUIRE((M / 128 + 1) * (N / 16 + 1) < (int64_t(1) << 31), DBS_ERR_ARGUMENT, "gemm_tf: too many tiles");
  DBS_REQUIRE(epi == DBS_EPI_F32 || epi == DBS_EPI_F32_ACCUM || epi == DBS_EPI_BIAS_F32 || epi == DBS_EPI_F32_ATOMIC ||
                  is_s32_epi_host(epi),
              DBS_ERR_ARGUMENT, "gemm_tf: epilogue %d has no S32 / fp32 form", epi);
  DBS_REQUIRE(!((epi == DBS_EPI_BIAS_RELU_S32 || epi == DBS_EPI_BIAS_F32) && !bias), DBS_ERR_ARGUMENT,
              "gemm_tf: epilogue needs bias");
  DBS_REQUIRE(!(epi == DBS_EPI_RELU_GRAD_S32 && !aux), DBS_ERR_ARGUMENT, "gemm_tf: epilogue needs aux");
  DBS_REQUIRE(lda % 32 == 0 && ldb % 32 == 0 && (!is_s32_epi_host(epi) || ldd % 32 == 0), DBS_ERR_ARGUMENT,
              "gemm_tf: S32 leading dimensions must be multiples of 32");
  DBS_REQUIRE(lda >= (a_mn ? M : K) && ldb >= (b_mn ? N : K), DBS_ERR_ARGUMENT, "gemm_tf: leading dimension too small");
  const int bn = pick_bn(N, b_mn) > 128 ? 128 : pick_bn(N, b_mn);
  DBS_REQUIRE(!(colsum_part && bn < 32), DBS_ERR_ARGUMENT, "gemm_tf: column sums need N > 16");
  CUtensorMap ta, tb;
  int st = a_mn ? make_tmap_s32_mn(&ta, a, (uint64_t)M, (uint64_t)K, (uint64_t)lda, 4)
                : make_tmap_kpair(&ta, a, (uint64_t)(4 * ceil32(K)), (uint64_t)M, (uint64_t)(4 * lda), 128);
  if (st) return st;
  st = b_mn ? make_tmap_s32_mn(&tb, b, (uint64_t)N, (uint64_t)K, (uint64_t)ldb, (uint32_t)(bn / 32), true)
            : make_tmap_kpair(&tb, b, (uint64_t)(4 * ceil32(K)), (uint64_t)N, (uint64_t)(4 * ldb), (uint32_t)bn);
  if (st) return st;
  GemmParams p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.a_mode = a_mn;
  p.b_mode = b_mn;
  p.epi = epi;
  p.d = d;
  p.ldd = ldd;
  p.bias = bias;
  p.aux = reinterpret_cast<const uint16_t*>(aux);
  p.colsum_part = colsum_part;
  p.kb_per_split = (int)((K + 31) / 32);
  return dispatch(ta, tb, p, bn, 1, s, false, true);
}

// Implicit-GEMM convolution family with S32 operands (ConvCall.tf; see gemm.cuh):
// A conv operands (mode 2) are NHWC S32 viewed as {4 C units, W, H, N}; the
// flipped filter (B mode 3) is [Cout][R*S][Cin] S32 viewed as {4 Cin, R*S, Cout};
// the weight gradient's im2col B (mode 2) takes 32-pixel boxes.
int conv_gemm_tf(const ConvCall& c, cudaStream_t s) {
  DBS_REQUIRE(c.d && c.M > 0 && c.N > 0 && c.K > 0, DBS_ERR_ARGUMENT, "conv_gemm_tf: bad call");
  DBS_REQUIRE(c.M < (int64_t(1) << 31) && c.K < (int64_t(1) << 31), DBS_ERR_ARGUMENT,
              "conv_gemm_tf: M and K must stay below 2^31");
  DBS_REQUIRE((c.a_mode <= 2 || c.a_mode == 5) && c.b_mode <= 3 && !(c.b_mode == 3 && c.a_mode != 2) &&
                  !(c.b_mode == 2 && c.a_mode != 1) && !(c.a_mode == 5 && c.b_mode != 1),
              DBS_ERR_ARGUMENT, "conv_gemm_tf: unsupported operand modes (%d, %d)", c.a_mode, c.b_mode);
  DBS_REQUIRE(!c.d_trans || (c.epi == DBS_EPI_F32_ATOMIC && c.M % 4 == 0 && c.ldd % 4 == 0 && ((uintptr_t)c.d & 15) == 0),
              DBS_ERR_ARGUMENT, "transposed D: atomic epilogue, M and ldd multiples of 4, 16-byte aligned D");
  CUtensorMap ta, tb;
  GemmParams p{};
  p.d_trans = c.d_trans;
  p.M = c.M;
  p.N = c.N;
  p.K = c.K;
  p.epi = c.epi;
  p.d = c.d;
  p.ldd = c.ldd;
  p.bias = c.bias;
  p.aux = c.aux;
  p.sum_part = c.sum_part;
  p.sq_part = c.sq_part;
  p.taps = c.taps;
  p.omap = c.omap;
  p.nclass = c.nclass;
  p.ga = c.ga;
  p.gb = c.gb;
  if (c.a_mode == 2) DBS_REQUIRE(c.ga.cblocks * 32 == c.ta.C, DBS_ERR_ARGUMENT, "conv_gemm_tf: cblocks counts 32 channels");
  if (c.nclass > 0) {
    DBS_REQUIRE(c.nclass <= 4 && c.splits <= 1 && c.a_mode == 2, DBS_ERR_ARGUMENT, "merged classes: bad call");
    const int64_t mt = (c.M + kBM - 1) / kBM;
    p.cls_start[0] = 0;
    for (int k = 0; k < c.nclass; k++) {
      p.cls_taps[k] = c.cls_taps[k];
      p.cls_omap[k] = c.cls_omap[k];
      p.cls_kb[k] = c.cls_taps[k].n * c.ga.cblocks;
      p.cls_start[k + 1] = p.cls_start[k] + mt;
    }
  }
  int bn = (c.bn_override > 0) ? c.bn_override : pick_bn(c.N, c.b_mode);
  if (bn > 128) bn = 128;  // two accumulators per S32 tile (gemm_bf16_kernel<BN, false, true>)
  if (c.bn_override <= 0 && c.b_mode != 2 && bn >= 64) {
    const int64_t sms = current_sm_count();
    const int64_t mt = (c.M + kBM - 1) / kBM;
    int64_t best = -1;
    int pick = bn;
    for (int cand = bn; cand >= 64; cand /= 2) {
      const int64_t tiles = mt * ((c.N + cand - 1) / cand);
      const int64_t cost = ((tiles + sms - 1) / sms) * (int64_t)(kBM * kBK * 2 + cand * kBK * 2);
      if (best < 0 || cost < best) {
        best = cost;
        pick = cand;
      }
    }
    bn = pick;
  }
  int st;
  if (c.halo) {
    // ---- fp32-class halo variant: 3x3 / stride 1 / 64 -> 64 channels (HaloTfCfg) ----
    const ConvGeom& g = c.ga;
    DBS_REQUIRE(c.a_mode == 2 && (c.b_mode == 0 || c.b_mode == 3) && g.R == 3 && g.S == 3 && g.stride == 1 &&
                    g.pad == 1 && g.cblocks == 2 && c.N == 64 && c.K == 576 && c.taps.n == 0 && !c.omap.on &&
                    c.nclass == 0 && c.splits <= 1 && !c.d_trans && halo_tf_fits(g.OH, g.OW) && c.ta.H == g.OH &&
                    c.ta.W == g.OW && c.ta.C == 64,
                DBS_ERR_ARGUMENT, "conv halo variant (S32): unsupported geometry");
    const int W1 = g.OW + 1;
    p.halo_rows = (g.OW + kBM - 1) / W1 + 3;
    p.halo_tpi = (g.OH * W1 + kBM - 1) / kBM;
    p.halo_tiles = (int64_t)c.ta.N * p.halo_tpi;
    const ConvTensor t4{c.ta.N, c.ta.H, c.ta.W, 4 * c.ta.C};
    st = make_tmap_nhwc_pair(&ta, c.a, t4, W1, p.halo_rows, 1, 1);  // {64, W + 1, rows, 1, hi/lo}
    if (st) return st;
    if (c.b_mode == 0) {
      DBS_REQUIRE(c.ldb % 32 == 0, DBS_ERR_ARGUMENT, "conv_gemm_tf: ldb %% 32");
      st = make_tmap_kpair(&tb, c.b, (uint64_t)(4 * ceil32(c.K)), (uint64_t)c.N, (uint64_t)(4 * c.ldb), 64u);
    } else {
      EncodeTiledFn fn = encode_fn();
      DBS_REQUIRE(fn != nullptr, DBS_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
      const uint64_t cin = (uint64_t)c.tb.C, rs = (uint64_t)c.tb.W;
      cuuint64_t dims[5] = {64, (cuuint64_t)c.tb.N, (cuuint64_t)(cin / 32), 2, (cuuint64_t)rs};
      cuuint64_t strides[4] = {(cuuint64_t)(rs * cin * 8), 256, 128, (cuuint64_t)(cin * 8)};
      cuuint32_t box[5] = {64, 32, 2, 2, 1};
      cuuint32_t es[5] = {1, 1, 1, 1, 1};
      CUresult r = fn(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(c.b), dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, kMnSwz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      DBS_REQUIRE(r == CUDA_SUCCESS, DBS_ERR_CUDA, "cuTensorMapEncodeTiled (S32 halo filter) failed (%d)", (int)r);
      st = DBS_OK;
    }
    if (st) return st;
    p.a_mode = 2;
    p.b_mode = c.b_mode;
    p.kb_per_split = 18;
    return dispatch(ta, tb, p, 64, 1, s, true, true);
  }
  // ---- A ----
  p.a_mode = c.a_mode;
  if (c.a_mode == 2) {
    const ConvTensor t4{c.ta.N, c.ta.H, c.ta.W, 4 * c.ta.C};
    const bool taps = c.taps.n > 0 || c.nclass > 0;
    if (force_im2col() || !pixel_box_fits(c.ga.OH, c.ga.OW, kBM)) {
      st = make_tmap_im2col(&ta, c.a, t4, taps ? -1 : -c.ga.pad, taps ? -1 : c.ga.pad - (c.ga.R - 1), kBM,
                            c.ga.stride);
      p.a_mode = 4;
    } else {
      int bw, bh, bnn;
      st = pixel_box(c.ga.OH, c.ga.OW, kBM, bw, bh, bnn);
      if (st) return st;
      st = make_tmap_nhwc_pair(&ta, c.a, t4, bw, bh, bnn, c.ga.stride);  // {64, pixels, hi/lo}
    }
  } else if (c.a_mode == 5) {
    // transposed weight gradient: 32-pixel windows of the conv input per 32-row group of M
    DBS_REQUIRE(c.ga.Cin % 32 == 0 && c.M == (int64_t)c.ga.R * c.ga.S * c.ga.Cin && c.d_trans, DBS_ERR_ARGUMENT,
                "transposed wgrad (S32): bad call");
    const ConvTensor t4{c.ta.N, c.ta.H, c.ta.W, 4 * c.ta.C};
    if (force_im2col() || !pixel_box_fits(c.ga.OH, c.ga.OW, 32)) {
      st = make_tmap_im2col(&ta, c.a, t4, -c.ga.pad, c.ga.pad - (c.ga.R - 1), 32, c.ga.stride, kMnSwz);
      p.a_mode = 6;
    } else {
      // K-paired (64-pixel boxes) when the tile and ring allow it: BN = 64 (4 ring stages),
      // an even k-block count, 64-pixel windows that are whole rows
      const bool kp5 = kpair_enabled() && bn == 64 && CfgTf<64>::kStages % 2 == 0 && ((c.K + 31) / 32) % 2 == 0 &&
                       pixel_box_fits(c.ga.OH, c.ga.OW, 64) && c.b_mode == 1;
      int bw, bh, bnn;
      st = pixel_box(c.ga.OH, c.ga.OW, kp5 ? 64 : 32, bw, bh, bnn);
      if (st) return st;
      st = make_tmap_nhwc_pair(&ta, c.a, t4, bw, bh, bnn, c.ga.stride, kMnSwz);
      p.pair_a = kp5 ? 5 : 0;
    }
  } else if (c.a_mode == 1) {
    DBS_REQUIRE(c.lda % 32 == 0, DBS_ERR_ARGUMENT, "conv_gemm_tf: lda %% 32");
    st = make_tmap_s32_mn(&ta, c.a, (uint64_t)c.M, (uint64_t)c.K, (uint64_t)c.lda, 4);
  } else {
    DBS_REQUIRE(c.lda % 32 == 0, DBS_ERR_ARGUMENT, "conv_gemm_tf: lda %% 32");
    st = make_tmap_kpair(&ta, c.a, (uint64_t)(4 * ceil32(c.K)), (uint64_t)c.M, (uint64_t)(4 * c.lda), 128);
  }
  if (st) return st;
  // ---- B ----
  p.b_mode = c.b_mode;
  if (c.b_mode == 2) {
    const ConvTensor t4{c.tb.N, c.tb.H, c.tb.W, 4 * c.tb.C};
    DBS_REQUIRE(c.gb.Cin % bn == 0 && bn <= c.gb.Cin, DBS_ERR_ARGUMENT, "wgrad: tile must not straddle (r,s)");
    if (force_im2col() || !pixel_box_fits(c.gb.OH, c.gb.OW, 32)) {
      st = make_tmap_im2col(&tb, c.b, t4, -c.gb.pad, c.gb.pad - (c.gb.R - 1), 32, c.gb.stride, kMnSwz);
      p.b_mode = 4;
    } else {
      int bw, bh, bnn;
      st = pixel_box(c.gb.OH, c.gb.OW, 32, bw, bh, bnn);
      if (st) return st;
      // one box for all BN / 32 channel groups of a tile (DBS_WGRAD_MERGE=0: one per group)
      static const bool merge = [] {
        const char* e = getenv("DBS_WGRAD_MERGE");
        return !(e && e[0] == '0');
      }();
      p.pair_b = (merge && bn / 32 >= 2) ? 2 : 0;
      st = make_tmap_nhwc_pair(&tb, c.b, t4, bw, bh, bnn, c.gb.stride, kMnSwz,
                               p.pair_b == 2 ? 2 * (bn / 32) : 2);  // {64, 32 pixels, hi/lo (x groups)}
    }
  } else if (c.b_mode == 3) {
    // filter [Cout][R*S][Cin] S32 read as the flipped, transposed filter: the MN-major
    // view {64 units, Cout k (K rows), Cin / 32 groups, hi/lo, R*S}, box {64, 32 k, BN / 32, 2, 1}
    EncodeTiledFn fn = encode_fn();
    DBS_REQUIRE(fn != nullptr, DBS_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
    DBS_REQUIRE(c.tb.C % 32 == 0 && c.tb.N % 32 == 0 && ((uintptr_t)c.b & 15) == 0 && bn % 32 == 0, DBS_ERR_ARGUMENT,
                "dgrad filter view: Cin, Cout multiples of 32 required");
    const uint64_t cin = (uint64_t)c.tb.C, rs = (uint64_t)c.tb.W;
    cuuint64_t dims[5] = {64, (cuuint64_t)c.tb.N, (cuuint64_t)(cin / 32), 2, (cuuint64_t)rs};
    cuuint64_t strides[4] = {(cuuint64_t)(rs * cin * 8), 256, 128, (cuuint64_t)(cin * 8)};
    cuuint32_t box[5] = {64, 32, (cuuint32_t)(bn / 32), 2, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = fn(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(c.b), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, kMnSwz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    DBS_REQUIRE(r == CUDA_SUCCESS, DBS_ERR_CUDA, "cuTensorMapEncodeTiled (3d S32 filter) failed (%d)", (int)r);
    st = DBS_OK;
  } else if (c.b_mode == 1) {
    DBS_REQUIRE(c.ldb % 32 == 0, DBS_ERR_ARGUMENT, "conv_gemm_tf: ldb %% 32");
    st = make_tmap_s32_mn(&tb, c.b, (uint64_t)c.N, (uint64_t)c.K, (uint64_t)c.ldb, (uint32_t)(bn / 32), true,
                          p.pair_a == 5 ? 64u : 32u);
  } else {
    DBS_REQUIRE(c.ldb % 32 == 0, DBS_ERR_ARGUMENT, "conv_gemm_tf: ldb %% 32");
    st = make_tmap_kpair(&tb, c.b, (uint64_t)(4 * ceil32(c.K)), (uint64_t)c.N, (uint64_t)(4 * c.ldb), (uint32_t)bn);
  }
  if (st) return st;
  const int num_l = (int)((c.K + 31) / 32);  // logical (32-wide) k-blocks
  int splits = c.splits > 0 ? c.splits : 1;
  if (splits > num_l) splits = num_l;
  p.kb_per_split = (num_l + splits - 1) / splits;
  if (p.pair_a == 5 && (p.kb_per_split & 1)) p.kb_per_split++;  // K pairs never straddle split-K slices
  splits = (num_l + p.kb_per_split - 1) / p.kb_per_split;
  DBS_REQUIRE(splits == 1 || c.epi == DBS_EPI_F32_ATOMIC, DBS_ERR_ARGUMENT, "split-K needs the atomic epilogue");
  return dispatch(ta, tb, p, bn, splits, s, false, true);
}

// Implicit-GEMM convolution family (see gemm.cuh).
int conv_gemm(const ConvCall& c, cudaStream_t s) {
  if (c.tf) return conv_gemm_tf(c, s);
  DBS_REQUIRE(c.d && c.M > 0 && c.N > 0 && c.K > 0, DBS_ERR_ARGUMENT, "conv_gemm: bad call");
  DBS_REQUIRE(c.M < (int64_t(1) << 31) && c.K < (int64_t(1) << 31), DBS_ERR_ARGUMENT,
              "conv_gemm: M and K must stay below 2^31 (32-bit tile / pixel arithmetic)");
  CUtensorMap ta, tb;
  GemmParams p{};
  p.M = c.M;
  p.N = c.N;
  p.K = c.K;
  p.epi = c.epi;
  p.d = c.d;
  p.ldd = c.ldd;
  p.bias = c.bias;
  p.aux = c.aux;
  p.sum_part = c.sum_part;
  p.sq_part = c.sq_part;
  p.taps = c.taps;
  p.omap = c.omap;
  p.nclass = c.nclass;
  if (c.nclass > 0) {
    DBS_REQUIRE(c.nclass <= 4 && c.splits <= 1 && c.a_mode == 2, DBS_ERR_ARGUMENT, "merged classes: bad call");
    const int64_t mt = (c.M + kBM - 1) / kBM;
    p.cls_start[0] = 0;
    for (int k = 0; k < c.nclass; k++) {
      p.cls_taps[k] = c.cls_taps[k];
      p.cls_omap[k] = c.cls_omap[k];
      p.cls_kb[k] = c.cls_taps[k].n * c.ga.cblocks;
      p.cls_start[k + 1] = p.cls_start[k] + mt;
    }
  }
  p.colsum_part = nullptr;
  int st;
  int bn = (c.bn_override > 0) ? c.bn_override : pick_bn(c.N, c.b_mode);
  if (c.bn_override <= 0 && c.b_mode != 2 && bn >= 64) {
    // N tile from a load-bound cost model of the persistent kernel: rounds of
    // tiles over the SMs this launch can use x shared-memory bytes per tile
    const int64_t sms = current_sm_count();
    const int64_t mt = (c.M + kBM - 1) / kBM;
    int64_t best = -1;
    int pick = bn;
    for (int cand = bn; cand >= 64; cand /= 2) {
      const int64_t tiles = mt * ((c.N + cand - 1) / cand);
      const int64_t cost = ((tiles + sms - 1) / sms) * (int64_t)(kBM * kBK * 2 + cand * kBK * 2);
      if (best < 0 || cost < best) {
        best = cost;
        pick = cand;
      }
    }
    bn = pick;
  }
  // paired k-block loads need an even k-block count in every tile: no split-K
  bool pairing = kpair_enabled() && (c.splits <= 1) && ((c.K + kBK - 1) / kBK) % 2 == 0;
  for (int k = 0; k < c.nclass; k++) pairing = pairing && (c.cls_taps[k].n * c.ga.cblocks) % 2 == 0;
  // weight gradient of a <= 64-output-channel conv (dY^T MN-major A, im2col(X) B,
  // 64-wide N tile): 128 pixels per box for both operands; split-K slices are
  // rounded to an even number of k-blocks
  const bool wpair = kpair_enabled() && c.a_mode == 1 && c.M <= 64 && c.b_mode == 2 && bn == 64 &&
                     ((c.K + kBK - 1) / kBK) % 2 == 0;
  // ---- halo variant: 3x3 / stride 1 / 64 -> 64 channels, whole-row tiles of one image ----
  if (c.halo) {
    const ConvGeom& g = c.ga;
    DBS_REQUIRE(c.a_mode == 2 && (c.b_mode == 0 || c.b_mode == 3) && g.R == 3 && g.S == 3 && g.stride == 1 &&
                    g.pad == 1 && g.cblocks == 1 && c.N == 64 && c.K == 576 && c.taps.n == 0 && !c.omap.on &&
                    halo_fits(g.OH, g.OW) && c.ta.H == g.OH && c.ta.W == g.OW,
                DBS_ERR_ARGUMENT, "conv halo variant: unsupported geometry");
    // one 4-D box per tile: halo_rows image rows x (W + 1) pixels from column -1
    const int W1 = g.OW + 1;
    p.halo_rows = (g.OW + kBM - 1) / W1 + 3;
    p.halo_tpi = (g.OH * W1 + kBM - 1) / kBM;
    p.halo_tiles = (int64_t)c.ta.N * p.halo_tpi;
    st = make_tmap_nhwc(&ta, c.a, c.ta, W1, p.halo_rows, 1, 1);
    if (st) return st;
    if (c.b_mode == 0 && halo_pair_enabled() && current_sm_count() >= 2 &&
        (uint32_t)(p.halo_rows * W1) * 128u <= Halo2Cfg::kSlotBytes) {
      // CTA pair: image 2k + rank, both CTAs at the same tile; half the filter rows each
      st = make_tmap(&tb, c.b, (uint64_t)c.K, (uint64_t)c.N, (uint64_t)c.ldb, 64, 32);
      if (st) return st;
      p.halo_tiles = ((int64_t)(c.ta.N + 1) / 2) * p.halo_tpi;
      p.a_mode = 2;
      p.b_mode = 0;
      p.ga = g;
      p.kb_per_split = 9;
      return launch_halo_pair(ta, tb, p, s);
    }
    if (c.b_mode == 0) {
      st = make_tmap(&tb, c.b, (uint64_t)c.K, (uint64_t)c.N, (uint64_t)c.ldb, 64, 64);
      if (st) return st;
    } else {
      EncodeTiledFn fn = encode_fn();
      DBS_REQUIRE(fn != nullptr, DBS_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
      cuuint64_t dims[3] = {(cuuint64_t)c.tb.C, (cuuint64_t)c.tb.W, (cuuint64_t)c.tb.N};
      cuuint64_t strides[2] = {(cuuint64_t)c.tb.C * 2, (cuuint64_t)c.tb.W * c.tb.C * 2};
      cuuint32_t box[3] = {64, 1, 64};
      cuuint32_t es[3] = {1, 1, 1};
      CUresult r = fn(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(c.b), dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      DBS_REQUIRE(r == CUDA_SUCCESS, DBS_ERR_CUDA, "cuTensorMapEncodeTiled (3d filter) failed (%d)", (int)r);
    }
    p.a_mode = 2;
    p.b_mode = c.b_mode;
    p.ga = g;
    p.kb_per_split = 9;
    return dispatch(ta, tb, p, 64, 1, s, true);
  }
  // ---- A ----
  p.a_mode = c.a_mode;
  p.d_trans = c.d_trans;
  DBS_REQUIRE(!c.d_trans || (c.epi == DBS_EPI_F32_ATOMIC && c.M % 4 == 0 && c.ldd % 4 == 0 &&
                             ((uintptr_t)c.d & 15) == 0),
              DBS_ERR_ARGUMENT, "transposed D: atomic epilogue, M and ldd multiples of 4, 16-byte aligned D");
  if (c.a_mode == 5) {
    // transposed weight gradient: 64-pixel windows of the conv input per 64 rows of M
    DBS_REQUIRE(c.ga.Cin % 64 == 0 && c.M == (int64_t)c.ga.R * c.ga.S * c.ga.Cin && c.b_mode == 1 && c.d_trans,
                DBS_ERR_ARGUMENT, "transposed wgrad: bad call");
    // paired: 128-pixel boxes for both operands (an even k-block count per split)
    const bool tpair = kpair_enabled() && ((c.K + kBK - 1) / kBK) % 2 == 0;
    const int kpx = tpair ? 2 * kBK : kBK;
    if (force_im2col() || !pixel_box_fits(c.ga.OH, c.ga.OW, kpx)) {
      st = make_tmap_im2col(&ta, c.a, c.ta, -c.ga.pad, c.ga.pad - (c.ga.R - 1), kpx, c.ga.stride);
      p.a_mode = 6;
    } else {
      int bw, bh, bnn;
      st = pixel_box(c.ga.OH, c.ga.OW, kpx, bw, bh, bnn);
      if (st) return st;
      st = make_tmap_nhwc(&ta, c.a, c.ta, bw, bh, bnn, c.ga.stride);
    }
    if (st) return st;
    p.ga = c.ga;
    p.pair_a = tpair ? 3 : 0;
    p.pair_b = tpair ? 1 : 0;
    pairing = false;
  } else if (c.a_mode == 2 && (force_im2col() || !pixel_box_fits(c.ga.OH, c.ga.OW, kBM))) {
    const bool taps = c.taps.n > 0;
    st = make_tmap_im2col(&ta, c.a, c.ta, taps ? -1 : -c.ga.pad, taps ? -1 : c.ga.pad - (c.ga.R - 1), kBM,
                          c.ga.stride);
    if (st) return st;
    p.a_mode = 4;
    p.ga = c.ga;
  } else if (c.a_mode == 2) {
    int bw, bh, bnn;
    st = pixel_box(c.ga.OH, c.ga.OW, kBM, bw, bh, bnn);
    if (st) return st;
    if (pairing && c.ga.cblocks % 2 == 0) {
      st = make_tmap_nhwc_pair(&ta, c.a, c.ta, bw, bh, bnn, c.ga.stride);
      p.pair_a = 1;
    } else {
      st = make_tmap_nhwc(&ta, c.a, c.ta, bw, bh, bnn, c.ga.stride);
    }
    if (st) return st;
    p.ga = c.ga;
  } else {
    if (c.a_mode == 0 && pairing && c.K % 128 == 0 && (c.lda * 2) % 16 == 0) {
      st = make_tmap_kpair(&ta, c.a, (uint64_t)c.K, (uint64_t)c.M, (uint64_t)c.lda, 128);
      p.pair_a = 1;
    } else {
      st = c.a_mode ? make_tmap(&ta, c.a, (uint64_t)c.M, (uint64_t)c.K, (uint64_t)c.lda, 64, wpair ? 128 : 64)
                    : make_tmap(&ta, c.a, (uint64_t)c.K, (uint64_t)c.M, (uint64_t)c.lda, 64, 128);
      if (wpair) p.pair_a = 2;
    }
    if (st) return st;
  }
  // ---- B ----
  p.b_mode = c.b_mode;
  const int kpix = wpair ? 2 * kBK : kBK;  // pixels per weight-gradient B box
  if (c.b_mode == 2 && (force_im2col() || !pixel_box_fits(c.gb.OH, c.gb.OW, kpix))) {
    st = make_tmap_im2col(&tb, c.b, c.tb, -c.gb.pad, c.gb.pad - (c.gb.R - 1), kpix, c.gb.stride);
    if (st) return st;
    p.b_mode = 4;
    p.pair_b = wpair;
    p.gb = c.gb;
    DBS_REQUIRE(c.gb.Cin % bn == 0 || bn % c.gb.Cin == 0, DBS_ERR_ARGUMENT, "wgrad: tile must not straddle (r,s)");
    DBS_REQUIRE(bn <= c.gb.Cin, DBS_ERR_ARGUMENT, "wgrad: BN %d > Cin %d", bn, c.gb.Cin);
  } else if (c.b_mode == 2) {
    int bw, bh, bnn;
    st = pixel_box(c.gb.OH, c.gb.OW, kpix, bw, bh, bnn);
    if (st) return st;
    st = make_tmap_nhwc(&tb, c.b, c.tb, bw, bh, bnn, c.gb.stride);
    if (st) return st;
    p.gb = c.gb;
    p.pair_b = wpair;
    DBS_REQUIRE(c.gb.Cin % bn == 0 || bn % c.gb.Cin == 0, DBS_ERR_ARGUMENT, "wgrad: tile must not straddle (r,s)");
    DBS_REQUIRE(bn <= c.gb.Cin, DBS_ERR_ARGUMENT, "wgrad: BN %d > Cin %d", bn, c.gb.Cin);
  } else if (c.b_mode == 3) {
    // filter [Cout][R*S][Cin] viewed as 3-D {Cin, R*S, Cout}: box {64 c, 1 rs, 64 k}
    EncodeTiledFn fn = encode_fn();
    DBS_REQUIRE(fn != nullptr, DBS_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
    DBS_REQUIRE(c.tb.C % 64 == 0 && c.tb.N % 64 == 0 && ((uintptr_t)c.b & 15) == 0, DBS_ERR_ARGUMENT,
                "dgrad filter view: Cin, Cout multiples of 64 required");
    // BN = 64: two consecutive 64-row k blocks of one tap are one box of 128 k rows
    const bool pb = pairing && bn == 64 && c.ga.cblocks % 2 == 0;
    // BN >= 128: the view {64 c, Cout k, Cin / 64 c-blocks, R*S} takes all BN / 64
    // channel blocks of one k-block in ONE box, landing as consecutive 64 k x 64 c
    // MN-major chunks (one TMA operation instead of BN / 64)
    const bool wide = bn >= 128 && wide_filter_enabled();
    // ... and with paired k-blocks, 128 k rows per box (channel blocks 16 KB apart)
    const bool wpb = wide && pairing && c.ga.cblocks % 2 == 0;
    CUresult r;
    if (wide) {
      cuuint64_t dims[4] = {64, (cuuint64_t)c.tb.N, (cuuint64_t)c.tb.C / 64, (cuuint64_t)c.tb.W};
      cuuint64_t strides[3] = {(cuuint64_t)c.tb.W * c.tb.C * 2, 128, (cuuint64_t)c.tb.C * 2};
      cuuint32_t box[4] = {64, wpb ? 128u : 64u, (cuuint32_t)(bn / 64), 1};
      cuuint32_t es[4] = {1, 1, 1, 1};
      r = fn(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(c.b), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      p.b_wide = 1;
    } else {
      cuuint64_t dims[3] = {(cuuint64_t)c.tb.C, (cuuint64_t)c.tb.W, (cuuint64_t)c.tb.N};
      cuuint64_t strides[2] = {(cuuint64_t)c.tb.C * 2, (cuuint64_t)c.tb.W * c.tb.C * 2};
      cuuint32_t box[3] = {64, 1, pb ? 128u : 64u};
      cuuint32_t es[3] = {1, 1, 1};
      r = fn(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(c.b), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    DBS_REQUIRE(r == CUDA_SUCCESS, DBS_ERR_CUDA, "cuTensorMapEncodeTiled (3d filter) failed (%d)", (int)r);
    DBS_REQUIRE(c.a_mode == 2, DBS_ERR_ARGUMENT, "flipped-filter B needs a conv-mode A");
    p.pair_b = wpb ? 3 : pb;
  } else {
    if (c.b_mode == 0 && pairing && c.K % 128 == 0 && (c.ldb * 2) % 16 == 0) {
      st = make_tmap_kpair(&tb, c.b, (uint64_t)c.K, (uint64_t)c.N, (uint64_t)c.ldb, (uint32_t)bn);
      p.pair_b = 1;
    } else {
      st = c.b_mode ? make_tmap(&tb, c.b, (uint64_t)c.N, (uint64_t)c.K, (uint64_t)c.ldb, 64, p.pair_b ? 128 : 64)
                    : make_tmap(&tb, c.b, (uint64_t)c.K, (uint64_t)c.N, (uint64_t)c.ldb, 64, (uint32_t)bn);
    }
    if (st) return st;
  }
  const int num_k = (int)((c.K + kBK - 1) / kBK);
  int splits = c.splits > 0 ? c.splits : 1;
  if (splits > num_k) splits = num_k;
  p.kb_per_split = (num_k + splits - 1) / splits;
  if (p.pair_a | p.pair_b) p.kb_per_split += p.kb_per_split & 1;  // even k-block count per slice
  splits = (num_k + p.kb_per_split - 1) / p.kb_per_split;
  DBS_REQUIRE(splits == 1 || c.epi == DBS_EPI_F32_ATOMIC, DBS_ERR_ARGUMENT, "split-K needs the atomic epilogue");
  return dispatch(ta, tb, p, bn, splits, s);
}

}  // namespace dbs

#ifdef DBS_GEMM_TRACE
extern "C" int dbs_gemm_trace_copy(unsigned long long* host, int n) {
  return cudaMemcpyFromSymbol(host, dbs::g_gemm_trace, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : 1;
}
#endif

extern "C" int dbs_dev_gemm_bf16(const void* d_a, int32_t a_major, int64_t lda, const void* d_b, int32_t b_major,
                                 int64_t ldb, void* d_d, int64_t ldd, int64_t M, int64_t N, int64_t K,
                                 int32_t epilogue, const float* d_bias, void* d_aux, void* stream) {
  return dbs::gemm_bf16(d_a, a_major, lda, d_b, b_major, ldb, d_d, ldd, M, N, K, epilogue, d_bias, d_aux,
                        dbs::as_stream(stream), nullptr);
}

extern "C" int dbs_dev_gemm_tf32x3(const void* d_a, int32_t a_major, int64_t lda, const void* d_b, int32_t b_major,
                                   int64_t ldb, void* d_d, int64_t ldd, int64_t M, int64_t N, int64_t K,
                                   int32_t epilogue, const float* d_bias, void* d_aux, void* stream) {
  return dbs::gemm_tf(d_a, a_major, lda, d_b, b_major, ldb, d_d, ldd, M, N, K, epilogue, d_bias, d_aux,
                      dbs::as_stream(stream), nullptr);
}

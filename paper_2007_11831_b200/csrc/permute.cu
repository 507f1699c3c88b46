// permute.cu -- per-epoch sample assignment on the device.
//
// The reference draws, once per epoch and worker after worker from ONE numpy
// Generator, `start + rng.permutation(end - start)` (sgdlab.py:358, 372-374).
// numpy 2.3's algorithm: PCG64 (XSL-RR 128/64) seeded by SeedSequence,
// next_uint32 = low half then buffered high half of next64, random_interval(i)
// = masked rejection on next_uint32, and Fisher-Yates from the top
// (for i = L-1 .. 1: swap(a[i], a[random_interval(i)])).
//
// B200 mapping:
//  phase 1 (draws, ONE warp): the rejection loop is sequential in the stream
//    position, so one warp evaluates 32 consecutive PCG64 outputs (64 uint32
//    draws) per round in parallel -- lane l jumps the 128-bit LCG l+1 steps
//    from the window base with a precomputed (MULT^k, inc * sum MULT^i) pair --
//    and accepts draws with a ballot, so the warp only serialises on accepted
//    draws.  Every span's draws are consumed in order (ranks stay in lock-step
//    with the reference's single generator) and written as int32 j_i.
//  phase 2 (swaps, one CTA per materialised span): the swap chain is applied
//    in shared memory (uint16 slots when the span fits 64 Ki, int32 below 50 Ki
//    entries, global memory otherwise) by lane 0 while the warp streams the j's
//    in coalesced 32-wide chunks; then the CTA writes start + a[k] coalesced.
#include "common.cuh"

namespace dbs {
namespace {

typedef unsigned __int128 u128;

__host__ __device__ __forceinline__ u128 pcg_mult() {
  return (((u128)0x2360ED051FC65DA4ULL) << 64) | 0x4385DF649FCCF645ULL;
}

__device__ __forceinline__ uint64_t xsl_rr(u128 s) {
  uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  uint64_t x = hi ^ lo;
  unsigned r = (unsigned)(hi >> 58);
  return (x >> r) | (x << ((64u - r) & 63u));
}

// 64-bit position mask from per-lane low-half / high-half ballots: bit 2l = lo of
// lane l, bit 2l + 1 = hi of lane l (the window's draw order)
__device__ __forceinline__ uint64_t spread(uint32_t x) {
  uint64_t v = x;
  v = (v | (v << 16)) & 0x0000FFFF0000FFFFull;
  v = (v | (v << 8)) & 0x00FF00FF00FF00FFull;
  v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0Full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}
__device__ __forceinline__ uint64_t interleave(uint32_t lo, uint32_t hi) { return spread(lo) | (spread(hi) << 1); }

__device__ __forceinline__ uint32_t smear(uint32_t m) {
  m |= m >> 1;
  m |= m >> 2;
  m |= m >> 4;
  m |= m >> 8;
  m |= m >> 16;
  return m;
}

// Phase 1: one warp.  spans[2s], spans[2s+1]; draws[off_s + i] = j_i for i >= 1.
__global__ void __launch_bounds__(32) draws_kernel(dbs_pcg64* rng, const int64_t* spans, int64_t n,
                                                   int32_t* draws, int32_t* status) {
  const int lane = threadIdx.x;
  const u128 M = pcg_mult();
  u128 S = ((u128)rng->state_hi << 64) | rng->state_lo;
  const u128 inc = ((u128)rng->inc_hi << 64) | rng->inc_lo;
  uint32_t has = rng->has_uint32;
  uint32_t stale_u = rng->uinteger;  // numpy keeps the last upper half even when consumed
  // jump coefficients for lane l: state_{l+1} = A S + C
  u128 A = 1, C = 0;
  for (int k = 0; k <= lane; k++) {
    A = A * M;
    C = C * M + inc;
  }
  u128 st = A * S + C;
  uint64_t o = xsl_rr(st);
  uint32_t vlo = (uint32_t)o, vhi = (uint32_t)(o >> 32);
  int cur = 0;          // next unconsumed position of the window [0, 64)
  int last_pos = -1;    // last consumed position inside the current window
  bool drew = false;    // any fresh output consumed at all
  uint32_t prev_hi31 = stale_u;  // upper half of the previous window's last output
  int64_t off = 0;
  int ok = 1;
  auto advance = [&]() {
    const uint64_t hi31 = __shfl_sync(0xffffffffu, (uint64_t)(st >> 64), 31);
    const uint64_t lo31 = __shfl_sync(0xffffffffu, (uint64_t)st, 31);
    prev_hi31 = __shfl_sync(0xffffffffu, vhi, 31);
    S = ((u128)hi31 << 64) | lo31;
    st = A * S + C;
    o = xsl_rr(st);
    vlo = (uint32_t)o;
    vhi = (uint32_t)(o >> 32);
    cur = 0;
    last_pos = -1;
  };
  // Per draw: two ballots and no shuffles on the serial chain -- the accepting
  // position follows from the ballots alone (first accepting lane; its low half
  // if that accepted, else its high half) and the accepting lane writes j itself.
  for (int64_t s = 0; s < n && ok; s++) {
    const int64_t start = spans[2 * s], L = spans[2 * s + 1] - start;
    if (L < 0 || L > 0x7fffffffLL) {
      ok = 0;
      break;
    }
    for (int64_t i = L - 1; i > 0; i--) {
      const uint32_t mx = (uint32_t)i;
      const uint32_t mask = smear(mx);
      if (has) {  // numpy hands out the buffered upper half first
        has = 0;
        const uint32_t v = stale_u & mask;
        if (v <= mx) {
          if (lane == 0) draws[off + i] = (int32_t)v;
          continue;
        }
      }
      // Whole-window step.  While the draws i, i-1, .., i-63 share one mask m (and
      // the span keeps >= 1 draw after them), a candidate v of the window is
      // accepted by whichever draw examines it if (v & m) <= i - 63 and rejected by
      // every one if (v & m) > i; only candidates in between ("ambiguous", 64 / m
      // of them) depend on the exact draw index.  Those few are resolved in
      // position order (the draw examining position p is i - #accepts before p),
      // then every lane places its accepts by a popcount rank: draw i - r takes
      // the r-th accepted position, and the window is consumed to its end.
      if (i >= 65 && smear((uint32_t)(i - 63)) == mask) {
        const uint32_t lo_ok = (uint32_t)(i - 63);
        const bool vl = cur <= 2 * lane, vh = cur <= 2 * lane + 1;
        const uint32_t ml = vlo & mask, mh = vhi & mask;
        const uint64_t acc0 = interleave(__ballot_sync(0xffffffffu, vl && ml <= lo_ok),
                                         __ballot_sync(0xffffffffu, vh && mh <= lo_ok));
        uint64_t amb = interleave(__ballot_sync(0xffffffffu, vl && ml > lo_ok && ml <= mx),
                                  __ballot_sync(0xffffffffu, vh && mh > lo_ok && mh <= mx));
        uint64_t acc = acc0;
        while (amb) {
          const int p = __ffsll((long long)amb) - 1;
          const uint32_t v = __shfl_sync(0xffffffffu, (p & 1) ? mh : ml, p >> 1);
          const uint64_t i_at = (uint64_t)i - (uint64_t)__popcll(acc & ((1ull << p) - 1ull));
          if ((uint64_t)v <= i_at) acc |= 1ull << p;
          amb &= amb - 1ull;
        }
        const int p_lo = 2 * lane, p_hi = 2 * lane + 1;
        if ((acc >> p_lo) & 1ull) draws[off + i - __popcll(acc & ((1ull << p_lo) - 1ull))] = (int32_t)ml;
        if ((acc >> p_hi) & 1ull) draws[off + i - __popcll(acc & ((1ull << p_hi) - 1ull))] = (int32_t)mh;
        drew = true;
        advance();                 // the window is consumed to its end (trailing rejects included)
        i -= __popcll(acc) - 1;    // the loop's i-- completes the step
        continue;
      }
      for (;;) {
        const bool plo = (cur <= 2 * lane) && ((vlo & mask) <= mx);
        const bool phi = (cur <= 2 * lane + 1) && ((vhi & mask) <= mx);
        const unsigned any = __ballot_sync(0xffffffffu, plo || phi);
        drew = true;
        if (any) {
          const unsigned anylo = __ballot_sync(0xffffffffu, plo);
          const int l0 = __ffs(any) - 1;
          const int pos = ((anylo >> l0) & 1u) ? 2 * l0 : 2 * l0 + 1;
          if (lane == l0) draws[off + i] = (int32_t)(((pos & 1) ? vhi : vlo) & mask);
          cur = pos + 1;
          last_pos = pos;
          break;
        }
        advance();  // every remaining draw of the window was rejected (and consumed)
      }
      if (cur >= 64) advance();
    }
    off += L;
  }
  // Final generator state, numpy field for field.  numpy keeps the upper half of the
  // last 64-bit output drawn (consumed or not) in `uinteger`.
  const int l = last_pos >= 0 ? (last_pos >> 1) : 0;
  const uint64_t hi_l = __shfl_sync(0xffffffffu, (uint64_t)(st >> 64), l);
  const uint64_t lo_l = __shfl_sync(0xffffffffu, (uint64_t)st, l);
  const uint32_t vhi_l = __shfl_sync(0xffffffffu, vhi, l);
  if (lane == 0) {
    if (last_pos >= 0) {
      rng->state_hi = hi_l;
      rng->state_lo = lo_l;
      rng->has_uint32 = ((last_pos & 1) == 0) ? 1u : 0u;
      rng->uinteger = vhi_l;
    } else {
      // nothing consumed in the current window: state is the window base
      rng->state_hi = (uint64_t)(S >> 64);
      rng->state_lo = (uint64_t)S;
      rng->has_uint32 = drew ? 0u : has;
      rng->uinteger = drew ? prev_hi31 : stale_u;
    }
    if (status) *status = ok ? 0 : (int32_t)DBS_ERR_ARGUMENT;
  }
}

constexpr int kSwapThreads = 256;
constexpr int64_t kSmemU16 = 65536;   // uint16 slots: 128 KB
constexpr int64_t kSmemI32 = 50000;   // int32 slots: 200 KB

template <typename Slot>
__device__ void swap_chain(Slot* a, const int32_t* __restrict__ j_of, int64_t L) {
  // identity
  for (int64_t k = threadIdx.x; k < L; k += blockDim.x) a[k] = (Slot)k;
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    // chunks of 32 draws, walking i from L-1 down to 1; prefetch one chunk ahead
    int64_t top = L - 1;
    int32_t nxt = (top - lane >= 1) ? __ldg(&j_of[top - lane]) : 0;
    while (top >= 1) {
      int32_t cur = nxt;
      const int64_t ntop = top - 32;
      nxt = (ntop - lane >= 1) ? __ldg(&j_of[ntop - lane]) : 0;
      const int cnt = (int)((top >= 32) ? 32 : top);
      for (int q = 0; q < cnt; q++) {
        const int32_t j = __shfl_sync(0xffffffffu, cur, q);
        if (lane == 0) {
          const int64_t i = top - q;
          Slot t = a[i];
          a[i] = a[j];
          a[j] = t;
        }
      }
      top = ntop;
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kSwapThreads) swaps_kernel(const int64_t* spans, int64_t n,
                                                             int64_t only_span, const int32_t* draws,
                                                             int64_t* out, int64_t* gscratch) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int64_t s = (only_span >= 0) ? only_span : (int64_t)blockIdx.x;
  int64_t off = 0;
  for (int64_t k = 0; k < s; k++) off += spans[2 * k + 1] - spans[2 * k];
  const int64_t start = spans[2 * s], L = spans[2 * s + 1] - start;
  if (L <= 0) return;
  const int32_t* j_of = draws + off;
  int64_t* dst = out + ((only_span >= 0) ? 0 : off);
  if (L <= kSmemI32) {
    int32_t* a = reinterpret_cast<int32_t*>(smem);
    swap_chain<int32_t>(a, j_of, L);
    for (int64_t k = threadIdx.x; k < L; k += blockDim.x) dst[k] = start + a[k];
  } else if (L <= kSmemU16) {
    uint16_t* a = reinterpret_cast<uint16_t*>(smem);
    swap_chain<uint16_t>(a, j_of, L);
    for (int64_t k = threadIdx.x; k < L; k += blockDim.x) dst[k] = start + (int64_t)a[k];
  } else {
    // too large for shared memory: run the chain in the output buffer itself
    int64_t* a = dst;
    swap_chain<int64_t>(a, j_of, L);
    for (int64_t k = threadIdx.x; k < L; k += blockDim.x) dst[k] += start;
  }
  (void)gscratch;
}

// SeedSequence (numpy bit_generator.pyx) -> PCG64 srandom (pcg64.h) on the host.
void pcg64_seed_host(const uint32_t* words, int nw, dbs_pcg64* out) {
  const uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu,
                 MULT_B = 0x58f38dedu, MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
  uint32_t zero = 0;
  if (nw <= 0) {
    words = &zero;
    nw = 1;
  }
  uint32_t hc = INIT_A;
  auto hashmix = [&](uint32_t v) {
    v ^= hc;
    hc *= MULT_A;
    v *= hc;
    v ^= v >> 16;
    return v;
  };
  auto mix = [&](uint32_t x, uint32_t y) {
    uint32_t r = MIX_L * x - MIX_R * y;
    r ^= r >> 16;
    return r;
  };
  uint32_t pool[4];
  for (int i = 0; i < 4; i++) pool[i] = hashmix(i < nw ? words[i] : 0u);
  for (int s = 0; s < 4; s++)
    for (int d = 0; d < 4; d++)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
  for (int s = 4; s < nw; s++)
    for (int d = 0; d < 4; d++) pool[d] = mix(pool[d], hashmix(words[s]));
  uint32_t w[8];
  uint32_t hb = INIT_B;
  for (int i = 0; i < 8; i++) {
    uint32_t v = pool[i % 4];
    v ^= hb;
    hb *= MULT_B;
    v *= hb;
    v ^= v >> 16;
    w[i] = v;
  }
  uint64_t u[4];
  for (int i = 0; i < 4; i++) u[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
  const u128 M = pcg_mult();
  u128 seed = ((u128)u[0] << 64) | u[1];
  u128 inc = ((((u128)u[2] << 64) | u[3]) << 1) | 1;
  u128 s = 0;
  s = s * M + inc;
  s += seed;
  s = s * M + inc;
  out->state_hi = (uint64_t)(s >> 64);
  out->state_lo = (uint64_t)s;
  out->inc_hi = (uint64_t)(inc >> 64);
  out->inc_lo = (uint64_t)inc;
  out->has_uint32 = 0;
  out->uinteger = 0;
}

int launch_permute(dbs_pcg64* d_rng, const int64_t* d_spans, int64_t n, int64_t only_span,
                   int64_t* d_out, int32_t* d_draws, int32_t* d_status, cudaStream_t s) {
  draws_kernel<<<1, 32, 0, s>>>(d_rng, d_spans, n, d_draws, d_status);
  DBS_LAUNCH_CHECK();
  static bool attr_set = false;
  const int smem = (int)(kSmemI32 * 4 > kSmemU16 * 2 ? kSmemI32 * 4 : kSmemU16 * 2);
  if (!attr_set) {
    DBS_CUDA_TRY(cudaFuncSetAttribute(swaps_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set = true;
  }
  const int grid = only_span >= 0 ? 1 : (int)n;
  if (grid > 0) {
    swaps_kernel<<<grid, kSwapThreads, smem, s>>>(d_spans, n, only_span, d_draws, d_out, nullptr);
    DBS_LAUNCH_CHECK();
  }
  return DBS_OK;
}

thread_local Scratch g_perm_scratch;

}  // namespace
}  // namespace dbs

using namespace dbs;

extern "C" int dbs_pcg64_seed(const uint32_t* seed_words, int32_t n_words, dbs_pcg64* out) {
  DBS_REQUIRE(out != nullptr, DBS_ERR_ARGUMENT, "dbs_pcg64_seed: null output");
  pcg64_seed_host(seed_words, n_words, out);
  return DBS_OK;
}

extern "C" int dbs_dev_permute_spans(dbs_pcg64* d_rng, const int64_t* d_spans, int64_t n,
                                     int64_t total_width, int64_t only_span, int64_t* d_perm_out,
                                     int32_t* d_draws, void* stream) {
  DBS_REQUIRE(d_rng && d_spans && d_perm_out && d_draws && n >= 0 && only_span < n, DBS_ERR_ARGUMENT,
              "dbs_dev_permute_spans: bad arguments");
  (void)total_width;
  return launch_permute(d_rng, d_spans, n, only_span, d_perm_out, d_draws, nullptr, as_stream(stream));
}

extern "C" int dbs_permute_spans(dbs_pcg64* rng, const int64_t* spans, int64_t n, int64_t* perm_out) {
  DBS_REQUIRE(rng && (n == 0 || spans) && n >= 0, DBS_ERR_ARGUMENT, "dbs_permute_spans: bad arguments");
  int64_t total = 0;
  for (int64_t i = 0; i < n; i++) {
    int64_t w = spans[2 * i + 1] - spans[2 * i];
    DBS_REQUIRE(w >= 0 && w <= 0x7fffffffLL, DBS_ERR_ARGUMENT, "span %lld has bad width", (long long)i);
    total += w;
  }
  size_t b_rng = 64, b_spans = sizeof(int64_t) * 2 * (n ? n : 1), b_out = sizeof(int64_t) * (total ? total : 1),
         b_draws = sizeof(int32_t) * (total ? total : 1) + 16;
  void* scr;
  int st = scratch_get(g_perm_scratch, b_rng + b_spans + b_out + b_draws + 64, &scr);
  if (st) return st;
  char* base = (char*)scr;
  dbs_pcg64* d_rng = (dbs_pcg64*)base;
  int32_t* d_status = (int32_t*)(base + 48);
  int64_t* d_spans = (int64_t*)(base + b_rng);
  int64_t* d_out = (int64_t*)(base + b_rng + b_spans);
  int32_t* d_draws = (int32_t*)(base + b_rng + b_spans + b_out);
  cudaStream_t s = cudaStreamPerThread;
  DBS_CUDA_TRY(cudaMemcpyAsync(d_rng, rng, sizeof(dbs_pcg64), cudaMemcpyHostToDevice, s));
  if (n) DBS_CUDA_TRY(cudaMemcpyAsync(d_spans, spans, sizeof(int64_t) * 2 * n, cudaMemcpyHostToDevice, s));
  st = launch_permute(d_rng, d_spans, n, -1, d_out, d_draws, d_status, s);
  if (st) return st;
  int32_t hstatus = 0;
  if (total) DBS_CUDA_TRY(cudaMemcpyAsync(perm_out, d_out, sizeof(int64_t) * total, cudaMemcpyDeviceToHost, s));
  DBS_CUDA_TRY(cudaMemcpyAsync(rng, d_rng, sizeof(dbs_pcg64), cudaMemcpyDeviceToHost, s));
  DBS_CUDA_TRY(cudaMemcpyAsync(&hstatus, d_status, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  DBS_CUDA_TRY(cudaStreamSynchronize(s));
  DBS_REQUIRE(hstatus == 0, hstatus, "permutation kernel rejected a span");
  return DBS_OK;
}

// comm.cu -- the fused batch-weighted all-reduce + momentum SGD over NVLink.
//
// Reference: sgdlab.aggregate_gradients (sgdlab.py:208-227) with
// w_j = b_j / sum(b) followed by sgd_step (sgdlab.py:230-238), and the
// model-averaging cadence of cluster.sync_rounds_for_epoch (cluster.py:185-186).
//
// One process per GPU.  Each rank owns a symmetric block in HBM
//   [ grad P fp32 | param P fp32 | param P bf16 | signal words ]
// mapped into every peer with CUDA IPC (NVLink 5 / NVSwitch peer memory).
// ONE kernel per iteration and rank:
//   phase 0  signal "my gradient is complete" to every peer (st.release.sys)
//            and wait for all peers' signals (ld.acquire.sys);
//   phase 1  for this rank's 1/W shard: load every peer's gradient shard over
//            NVLink with 16-byte vectors, form sum_j w_j g_j, apply
//            v' = m v + g, x' = x - lr v' (velocity kept only for the shard),
//            and PUSH x' (fp32 + bf16 shadow) into every peer's parameter
//            buffer -- reduce-scatter, update and all-gather in one pass;
//   phase 2  the last CTA to finish (device-scope arrival counter) signals
//            "shard written" to all peers and waits for theirs, so the kernel
//            completes only when every rank's parameters are whole.
// NCCL is not involved; torch.distributed only carries the IPC handles.
#include <stdlib.h>
#include <string.h>

#include "common.cuh"

namespace dbs {
namespace comm {

constexpr int kMaxRanks = 8;
constexpr int kThreads = 256;
constexpr int kSignalWords = 64;  // [0..W) phase-0 flags, [16..16+W) phase-2 flags, [32] arrival counter

struct PeerTable {
  float* grad[kMaxRanks];
  float* param[kMaxRanks];
  uint16_t* param_bf16[kMaxRanks];
  uint32_t* signal[kMaxRanks];
  float w[kMaxRanks];
};

}  // namespace comm
}  // namespace dbs

using dbs::comm::kMaxRanks;
using dbs::comm::kSignalWords;
using dbs::comm::kThreads;
using dbs::comm::PeerTable;

struct dbs_comm {
  int rank = 0, world = 1;
  int64_t P = 0;         // padded parameter count (multiple of 4 * world)
  int64_t shard = 0;     // elements per rank
  char* block = nullptr;  // this rank's symmetric block
  size_t block_bytes = 0;
  bool owns_block = true;
  void* peer_base[kMaxRanks] = {nullptr};
  bool opened[kMaxRanks] = {false};
  uint32_t gen = 0;      // barrier generation (identical sequence on every rank)
  PeerTable table{};
  int grid = 0;
  // operand shadow of the parameters: DBS_PREC_BF16 = the block's bf16 region,
  // pushed to every peer by the fused kernel; DBS_PREC_F32 = a registered local S32
  // buffer (dbs_comm_set_shadow) that the caller refreshes after the update
  int shadow_prec = DBS_PREC_BF16;
  void* shadow = nullptr;
};

namespace dbs {
namespace {

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Wait until every rank's flag reached `gen`.  A peer that never arrives (dead
// rank, mismatched call sequence) must not wedge the GPU, and the update must not
// silently reduce an incomplete gradient: after 20 s the wait records the error
// word (signal[48], for post-mortems) and traps, so the launch fails with a CUDA
// error that the next synchronising call on the host reports.
__device__ __forceinline__ void wait_flags(const uint32_t* base, int world, uint32_t gen, uint32_t* err) {
  const long long t0 = gtimer();
  for (int j = 0; j < world; j++) {
    while ((int32_t)(ld_acquire_sys(base + j) - gen) < 0) {
      if (gtimer() - t0 > 20000000000LL) {
        atomicExch(err, 1u);
        __threadfence_system();
        __trap();
      }
    }
  }
}

__device__ __forceinline__ uint32_t bf16_bits(float f) {
  uint32_t u = __float_as_uint(f);
  return (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
}

// mode 0: gradient all-reduce + SGD;  mode 1: parameter averaging
// BF16: also push the bf16 operand shadow (an S32-shadow communicator refreshes its own)
template <int MODE, bool BF16, int kUnroll>
__global__ void __launch_bounds__(kThreads) fused_kernel(PeerTable T, int rank, int world, int64_t shard4,
                                                         float lr, float mom, float4* __restrict__ vel,
                                                         uint32_t gen) {
  uint32_t* my_sig = T.signal[rank];
  // ---- phase 0: everyone's input is complete -------------------------------
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int j = 0; j < world; j++) st_release_sys(T.signal[j] + rank, gen);
    wait_flags(my_sig, world, gen, my_sig + 48);
  }
  __syncthreads();
  // ---- phase 1: reduce my shard, update, push to every peer -----------------
  // kUnroll float4s per thread and trip, every peer's loads issued before any use
  // up to 8 x kUnroll 16-byte NVLink reads in flight per thread (latency-bound otherwise)
  const int64_t base4 = (int64_t)rank * shard4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < shard4; i0 += stride * kUnroll) {
    float4 acc[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; u++) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 g[kMaxRanks][kUnroll];
#pragma unroll
    for (int j = 0; j < kMaxRanks; j++) {
      if (j >= world) break;
      const float4* src = reinterpret_cast<const float4*>(MODE == 0 ? T.grad[j] : T.param[j]) + base4;
#pragma unroll
      for (int u = 0; u < kUnroll; u++) {
        const int64_t i = i0 + u * stride;
        // peer memory, fetched again (.cv: never a stale line from an earlier iteration;
        // measured faster than .cg here, 0.65 vs 0.51 of HBM at W = 1)
        g[j][u] = i < shard4 ? __ldcv(src + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int j = 0; j < kMaxRanks; j++) {
      if (j >= world) break;
      const float w = T.w[j];
#pragma unroll
      for (int u = 0; u < kUnroll; u++) {
        acc[u].x = fmaf(w, g[j][u].x, acc[u].x);
        acc[u].y = fmaf(w, g[j][u].y, acc[u].y);
        acc[u].z = fmaf(w, g[j][u].z, acc[u].z);
        acc[u].w = fmaf(w, g[j][u].w, acc[u].w);
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; u++) {
      const int64_t i = i0 + u * stride;
      if (i >= shard4) break;
      const int64_t p4 = base4 + i;
      float4 x;
      if (MODE == 0) {
        float4 v = vel[i];
        x = reinterpret_cast<const float4*>(T.param[rank])[p4];
        v.x = fmaf(mom, v.x, acc[u].x);
        v.y = fmaf(mom, v.y, acc[u].y);
        v.z = fmaf(mom, v.z, acc[u].z);
        v.w = fmaf(mom, v.w, acc[u].w);
        x.x = fmaf(-lr, v.x, x.x);
        x.y = fmaf(-lr, v.y, x.y);
        x.z = fmaf(-lr, v.z, x.z);
        x.w = fmaf(-lr, v.w, x.w);
        vel[i] = v;
      } else {
        x = acc[u];
      }
      const uint2 xb = make_uint2(bf16_bits(x.x) | (bf16_bits(x.y) << 16), bf16_bits(x.z) | (bf16_bits(x.w) << 16));
#pragma unroll
      for (int j = 0; j < kMaxRanks; j++) {
        if (j >= world) break;
        const int jj = (rank + j) % world;  // stagger the peers to spread NVLink traffic
        reinterpret_cast<float4*>(T.param[jj])[p4] = x;
        if (BF16) reinterpret_cast<uint2*>(T.param_bf16[jj])[p4] = xb;
      }
    }
  }
  // ---- phase 2: all shards written everywhere --------------------------------
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const uint32_t arrived = atomicAdd(my_sig + 32, 1u) + 1u;
    if (arrived == gen * gridDim.x) {
      for (int j = 0; j < world; j++) st_release_sys(T.signal[j] + 16 + rank, gen);
      wait_flags(my_sig + 16, world, gen, my_sig + 48);
    }
  }
}

// peer memory, fetched again (.cv), 256 bits per load
__device__ __forceinline__ V8 ldg8_cv(const void* p) {
  V8 r;
  asm volatile("ld.global.cv.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]), "=r"(r.v[6]),
                 "=r"(r.v[7])
               : "l"(p));
  return r;
}

// The same exchange over 8 floats per thread and trip with 256-bit loads / stores
// (LDG/STG.256: twice the bytes in flight per request of the float4 form; the shards
// are whole 32-element blocks, so every unit is 32-byte aligned)
template <int MODE, bool BF16>
__global__ void __launch_bounds__(kThreads) fused8_kernel(PeerTable T, int rank, int world, int64_t shard8, float lr,
                                                          float mom, float* __restrict__ vel, uint32_t gen) {
  uint32_t* my_sig = T.signal[rank];
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int j = 0; j < world; j++) st_release_sys(T.signal[j] + rank, gen);
    wait_flags(my_sig, world, gen, my_sig + 48);
  }
  __syncthreads();
  const int64_t base8 = (int64_t)rank * shard8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < shard8; i += stride) {
    const int64_t p8 = base8 + i;
    V8 g[kMaxRanks];
#pragma unroll
    for (int j = 0; j < kMaxRanks; j++) {
      if (j >= world) break;
      // every peer's load before any use; this rank's own buffer was written by this GPU
      // (earlier kernels), so a plain streaming load suffices there
      const float* src = (MODE == 0 ? T.grad[j] : T.param[j]) + 8 * p8;
      g[j] = j == rank ? ldg8_cs(src) : ldg8_cv(src);
    }
    float x[8];
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = 0.0f;
#pragma unroll
    for (int j = 0; j < kMaxRanks; j++) {
      if (j >= world) break;
      const float w = T.w[j];
#pragma unroll
      for (int k = 0; k < 8; k++) x[k] = fmaf(w, f8(g[j], k), x[k]);
    }
    if (MODE == 0) {
      const V8 vq = ldg8(vel + 8 * i), xq = ldg8(T.param[rank] + 8 * p8);
      float v[8];
#pragma unroll
      for (int k = 0; k < 8; k++) {
        v[k] = fmaf(mom, f8(vq, k), x[k]);
        x[k] = fmaf(-lr, v[k], f8(xq, k));
      }
      stg8(vel + 8 * i, v8_of(v));
    }
    const V8 xo = v8_of(x);
    const uint4 xb = make_uint4(bf16_bits(x[0]) | (bf16_bits(x[1]) << 16), bf16_bits(x[2]) | (bf16_bits(x[3]) << 16),
                                bf16_bits(x[4]) | (bf16_bits(x[5]) << 16), bf16_bits(x[6]) | (bf16_bits(x[7]) << 16));
#pragma unroll
    for (int j = 0; j < kMaxRanks; j++) {
      if (j >= world) break;
      const int jj = (rank + j) % world;  // stagger the peers to spread NVLink traffic
      stg8(T.param[jj] + 8 * p8, xo);
      if (BF16) reinterpret_cast<uint4*>(T.param_bf16[jj])[p8] = xb;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const uint32_t arrived = atomicAdd(my_sig + 32, 1u) + 1u;
    if (arrived == gen * gridDim.x) {
      for (int j = 0; j < world; j++) st_release_sys(T.signal[j] + 16 + rank, gen);
      wait_flags(my_sig + 16, world, gen, my_sig + 48);
    }
  }
}

// float4s per thread and trip / resident CTAs per SM (DBS_COMM_UNROLL, DBS_COMM_CTAS:
// measurement switches; defaults are the measured configuration)
int comm_unroll() {
  static const int u = [] {
    const char* e = getenv("DBS_COMM_UNROLL");
    const int v = e ? atoi(e) : 1;
    return (v == 1 || v == 2 || v == 4) ? v : 1;
  }();
  return u;
}
int comm_ctas_per_sm() {
  static const int c = [] {
    const char* e = getenv("DBS_COMM_CTAS");
    const int v = e ? atoi(e) : 2;
    return (v >= 1 && v <= 8) ? v : 2;
  }();
  return c;
}

// 256-bit exchange kernel (fused8_kernel) unless DBS_COMM_WIDE=0 (measurement switch)
bool comm_wide() {
  static const bool on = [] {
    const char* e = getenv("DBS_COMM_WIDE");
    return !(e && e[0] == '0');
  }();
  return on;
}

int ipc_handle_size() { return (int)sizeof(cudaIpcMemHandle_t); }

size_t block_layout(int64_t P, size_t* off_param, size_t* off_bf16, size_t* off_sig) {
  size_t g = (size_t)P * 4;
  *off_param = g;
  *off_bf16 = g + (size_t)P * 4;
  *off_sig = ((*off_bf16 + (size_t)P * 2) + 255) & ~size_t(255);
  return *off_sig + kSignalWords * 4;
}

void fill_local(dbs_comm* c, int j, char* base) {
  size_t op, ob, os;
  block_layout(c->P, &op, &ob, &os);
  c->table.grad[j] = reinterpret_cast<float*>(base);
  c->table.param[j] = reinterpret_cast<float*>(base + op);
  c->table.param_bf16[j] = reinterpret_cast<uint16_t*>(base + ob);
  c->table.signal[j] = reinterpret_cast<uint32_t*>(base + os);
}

int launch_fused(dbs_comm* c, const int64_t* batch_sizes, int32_t mode, int kind, float lr, float mom, float* vel,
                 cudaStream_t s) {
  DBS_REQUIRE(c && batch_sizes, DBS_ERR_ARGUMENT, "comm: null argument");
  DBS_REQUIRE(mode == DBS_AGG_UNIFORM || mode == DBS_AGG_BATCH_WEIGHTED, DBS_ERR_CONFIGURATION,
              "unknown aggregation mode %d", mode);
  for (int j = 0; j < c->world; j++) DBS_REQUIRE(c->opened[j], DBS_ERR_ARGUMENT, "comm: peer %d not opened", j);
  double tot = 0.0;
  for (int j = 0; j < c->world; j++) {
    DBS_REQUIRE(batch_sizes[j] > 0, DBS_ERR_CONFIGURATION, "batch sizes must be positive");
    tot += (double)batch_sizes[j];
  }
  for (int j = 0; j < c->world; j++)
    c->table.w[j] = (float)(mode == DBS_AGG_BATCH_WEIGHTED ? (double)batch_sizes[j] / tot : 1.0 / c->world);
  c->gen += 1;
  const int64_t shard4 = c->shard / 4;
  const bool bf = c->shadow_prec == DBS_PREC_BF16;
  const int u = comm_unroll();
  if (comm_wide() && (kind != 0 || ((uintptr_t)vel % 32) == 0)) {
    const int64_t shard8 = c->shard / 8;
#define DBS_COMM_LAUNCH8(K, B)                                                                                        \
  fused8_kernel<K, B><<<c->grid, kThreads, 0, s>>>(c->table, c->rank, c->world, shard8, K == 0 ? lr : 0.f,         \
                                                   K == 0 ? mom : 0.f, K == 0 ? vel : nullptr, c->gen)
    if (kind == 0 && bf)
      DBS_COMM_LAUNCH8(0, true);
    else if (kind == 0)
      DBS_COMM_LAUNCH8(0, false);
    else if (bf)
      DBS_COMM_LAUNCH8(1, true);
    else
      DBS_COMM_LAUNCH8(1, false);
#undef DBS_COMM_LAUNCH8
    DBS_LAUNCH_CHECK();
    return DBS_OK;
  }
#define DBS_COMM_LAUNCH(K, B, U)                                                                                     \
  fused_kernel<K, B, U><<<c->grid, kThreads, 0, s>>>(c->table, c->rank, c->world, shard4, K == 0 ? lr : 0.f,     \
                                                     K == 0 ? mom : 0.f,                                          \
                                                     K == 0 ? reinterpret_cast<float4*>(vel) : nullptr, c->gen)
#define DBS_COMM_LAUNCH_U(K, B) \
  do {                          \
    if (u == 1)                 \
      DBS_COMM_LAUNCH(K, B, 1); \
    else if (u == 4)            \
      DBS_COMM_LAUNCH(K, B, 4); \
    else                        \
      DBS_COMM_LAUNCH(K, B, 2); \
  } while (0)
  if (kind == 0 && bf)
    DBS_COMM_LAUNCH_U(0, true);
  else if (kind == 0)
    DBS_COMM_LAUNCH_U(0, false);
  else if (bf)
    DBS_COMM_LAUNCH_U(1, true);
  else
    DBS_COMM_LAUNCH_U(1, false);
#undef DBS_COMM_LAUNCH_U
#undef DBS_COMM_LAUNCH
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

}  // namespace
}  // namespace dbs

using namespace dbs;

extern "C" int dbs_comm_handle_size(void) { return ipc_handle_size(); }

static int comm_new(int32_t rank, int32_t world, int64_t P, dbs_comm** out) {
  DBS_REQUIRE(out && world >= 1 && world <= kMaxRanks && rank >= 0 && rank < world && P > 0, DBS_ERR_ARGUMENT,
              "comm_alloc: need 1 <= world <= %d, 0 <= rank < world, P > 0", kMaxRanks);
  dbs_comm* c = new dbs_comm();
  c->rank = rank;
  c->world = world;
  const int64_t q = 32 * (int64_t)world;  // shards of whole float4s and 32-element S32 blocks
  c->P = (P + q - 1) / q * q;
  c->shard = c->P / world;
  size_t op, ob, os;
  c->block_bytes = block_layout(c->P, &op, &ob, &os);
  const int64_t per = (int64_t)kThreads * comm_unroll();  // float4s per CTA and trip
  const int64_t want = (c->shard / 4 + per - 1) / per;
  const int64_t cap = (int64_t)num_sms() * comm_ctas_per_sm();
  c->grid = (int)(want < 1 ? 1 : (want < cap ? want : cap));
  *out = c;
  return DBS_OK;
}

extern "C" int dbs_comm_alloc(int32_t rank, int32_t world, int64_t P, dbs_comm** out, void* handle_out) {
  int st = comm_new(rank, world, P, out);
  if (st) return st;
  dbs_comm* c = *out;
  cudaError_t e = cudaMalloc(&c->block, c->block_bytes);
  if (e == cudaSuccess) e = cudaMemset(c->block, 0, c->block_bytes);
  if (e != cudaSuccess) {
    set_error("comm_alloc: %s", cudaGetErrorString(e));
    delete c;
    *out = nullptr;
    return DBS_ERR_CUDA;
  }
  fill_local(c, rank, c->block);
  c->peer_base[rank] = c->block;
  c->opened[rank] = true;
  if (handle_out) {
    cudaIpcMemHandle_t h;
    DBS_CUDA_TRY(cudaIpcGetMemHandle(&h, c->block));
    memcpy(handle_out, &h, sizeof(h));
  }
  return DBS_OK;
}

extern "C" int dbs_comm_open(dbs_comm* c, const void* all_handles) {
  DBS_REQUIRE(c && all_handles, DBS_ERR_ARGUMENT, "comm_open: null argument");
  const cudaIpcMemHandle_t* hs = reinterpret_cast<const cudaIpcMemHandle_t*>(all_handles);
  for (int j = 0; j < c->world; j++) {
    if (j == c->rank || c->opened[j]) continue;
    void* p = nullptr;
    DBS_CUDA_TRY(cudaIpcOpenMemHandle(&p, hs[j], cudaIpcMemLazyEnablePeerAccess));
    c->peer_base[j] = p;
    fill_local(c, j, reinterpret_cast<char*>(p));
    c->opened[j] = true;
  }
  return DBS_OK;
}

// Single-process form (tests, simulated ranks on one device): `world`
// communicators whose symmetric blocks are plain local allocations.
extern "C" int dbs_comm_create_local(int32_t world, int64_t P, dbs_comm** comms_out) {
  DBS_REQUIRE(comms_out, DBS_ERR_ARGUMENT, "comm_create_local: null output");
  for (int r = 0; r < world; r++) {
    int st = dbs_comm_alloc(r, world, P, &comms_out[r], nullptr);
    if (st) return st;
  }
  // all simulated ranks share one GPU: every rank's CTAs must be co-resident
  // (phase 0 waits for the others), so cap the grids well below capacity
  const int cap = num_sms() * 2 / (world > 0 ? world : 1);
  for (int r = 0; r < world; r++)
    if (comms_out[r]->grid > cap) comms_out[r]->grid = cap > 0 ? cap : 1;
  for (int r = 0; r < world; r++)
    for (int j = 0; j < world; j++) {
      if (j == r) continue;
      comms_out[r]->peer_base[j] = comms_out[j]->block;
      fill_local(comms_out[r], j, comms_out[j]->block);
      comms_out[r]->opened[j] = true;
    }
  return DBS_OK;
}

extern "C" int dbs_comm_buffers(dbs_comm* c, float** d_grad, float** d_param, uint16_t** d_param_bf16) {
  DBS_REQUIRE(c, DBS_ERR_ARGUMENT, "comm_buffers: null comm");
  if (d_grad) *d_grad = c->table.grad[c->rank];
  if (d_param) *d_param = c->table.param[c->rank];
  if (d_param_bf16) *d_param_bf16 = c->table.param_bf16[c->rank];
  return DBS_OK;
}

extern "C" int dbs_comm_set_shadow(dbs_comm* c, void* d_shadow, int32_t prec) {
  DBS_REQUIRE(c && (prec == DBS_PREC_BF16 || (prec == DBS_PREC_F32 && d_shadow && c->P % 32 == 0)), DBS_ERR_ARGUMENT,
              "comm_set_shadow: bf16, or an S32 buffer of 2 P floats (padded P %% 32 == 0)");
  c->shadow_prec = prec;
  c->shadow = prec == DBS_PREC_F32 ? d_shadow : nullptr;
  return DBS_OK;
}

extern "C" int dbs_comm_shadow(const dbs_comm* c, void** d_shadow, int32_t* prec) {
  DBS_REQUIRE(c, DBS_ERR_ARGUMENT, "comm_shadow: null comm");
  if (d_shadow) *d_shadow = c->shadow_prec == DBS_PREC_F32 ? c->shadow : (void*)c->table.param_bf16[c->rank];
  if (prec) *prec = c->shadow_prec;
  return DBS_OK;
}

extern "C" int dbs_comm_info(const dbs_comm* c, int64_t* padded_P, int64_t* shard) {
  DBS_REQUIRE(c, DBS_ERR_ARGUMENT, "comm_info: null comm");
  if (padded_P) *padded_P = c->P;
  if (shard) *shard = c->shard;
  return DBS_OK;
}

extern "C" int dbs_comm_destroy(dbs_comm* c) {
  if (!c) return DBS_OK;
  cudaFree(c->block);  // IPC peer mappings are released by dbs_comm_close_peers
  delete c;
  return DBS_OK;
}

extern "C" int dbs_comm_close_peers(dbs_comm* c) {
  DBS_REQUIRE(c, DBS_ERR_ARGUMENT, "comm_close_peers: null comm");
  for (int j = 0; j < c->world; j++)
    if (j != c->rank && c->opened[j] && c->peer_base[j]) {
      cudaIpcCloseMemHandle(c->peer_base[j]);
      c->opened[j] = false;
    }
  return DBS_OK;
}

extern "C" int dbs_comm_allreduce_sgd(dbs_comm* c, const int64_t* batch_sizes, int32_t mode, float step,
                                      float momentum, float* d_velocity_shard, void* stream) {
  DBS_REQUIRE(d_velocity_shard, DBS_ERR_ARGUMENT, "comm_allreduce_sgd: velocity shard required");
  return launch_fused(c, batch_sizes, mode, 0, step, momentum, d_velocity_shard, as_stream(stream));
}

extern "C" int dbs_comm_average_params(dbs_comm* c, const int64_t* batch_sizes, int32_t mode, void* stream) {
  return launch_fused(c, batch_sizes, mode, 1, 0.f, 0.f, nullptr, as_stream(stream));
}

// spin.cu -- worker heterogeneity and device-side timing.
//
// The reference models a slow worker with DisturbanceEvent (cluster.py:25-56):
// a multiplicative per-sample cost or flat extra seconds per epoch, applied in
// effective_cost / epoch_gpu_time (cluster.py:123-145).  On the B200 the
// disturbance is REAL: a co-running spin kernel that pins whole SMs (one
// 1024-thread CTA holding ~all shared memory per SM), so the worker's training
// kernels get only the remaining SMs -- cost_multiplier ~ 1 / (1 - f) for an SM
// fraction f -- or that burns a fixed number of nanoseconds of device time
// (extra_epoch_seconds).
//
// Per-worker compute time for the controller (cluster.py:259-262 uses the
// previous epoch's per_worker_gpu) is read from %globaltimer by 1-thread stamp
// kernels in the worker's stream and accumulated on the device, so the
// controller never waits for the host.
#include <stdlib.h>

#include "common.cuh"

namespace dbs {
namespace {

constexpr int kSpinThreads = 1024;
constexpr int kSpinSmem = 200 * 1024;
constexpr long long kSpinSafetyNs = 600LL * 1000 * 1000 * 1000;  // never spin past 10 minutes

__device__ __forceinline__ long long globaltimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// The spinning CTA must load only ITS SM: the work is FMA + shared memory, and
// only thread 0 touches the memory system (one poll of the stop flag / the
// global timer every ~64 inner rounds) -- 1024 threads hammering one global
// address would congest the L2 slice and slow every kernel on the GPU.
// 1024 threads x ~64 live registers fill the register file, 200 KB the shared
// memory: nothing else can be co-resident on a pinned SM.
// sleep = 1 (the default): the resident CTA holds the SM's registers and shared memory
// but its threads sleep (__nanosleep) between polls -- the SMs are pinned exactly as
// before at a fraction of the power.  On one GPU the emulated workers share ONE power
// budget: an FMA-burning disturbance pushed the balanced DBS epochs into the power cap
// (1852-1927 MHz vs 1965 in the fixed-plan epochs), a coupling separate devices do not
// have.  sleep = 0 keeps the FMA spin (DBS_SPIN_SLEEP=0).
__global__ void __launch_bounds__(kSpinThreads, 1) spin_until_kernel(const volatile int32_t* stop, int sleep) {
  extern __shared__ float buf[];
  __shared__ volatile int done;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  const long long t0 = globaltimer();
  float acc[48];
#pragma unroll
  for (int j = 0; j < 48; j++) acc[j] = threadIdx.x + j;
  if (sleep) {
    for (int it = 1;; it++) {
      __nanosleep(1000);
      buf[threadIdx.x + (it & 31) * kSpinThreads] = acc[it & 7];
      if ((it & 3) == 0) {
        if (threadIdx.x == 0 && (*stop || globaltimer() - t0 > kSpinSafetyNs)) done = 1;
        __syncthreads();
        if (done) break;
      }
    }
  } else
  for (int it = 1;; it++) {
#pragma unroll 4
    for (int k = 0; k < 8; k++)
#pragma unroll
      for (int j = 0; j < 48; j++) acc[j] = fmaf(acc[j], 1.0000001f, 0.5f);
    buf[threadIdx.x + (it & 31) * kSpinThreads] = acc[it & 7];  // 128 KB footprint
    if ((it & 63) == 0) {
      if (threadIdx.x == 0 && (*stop || globaltimer() - t0 > kSpinSafetyNs)) done = 1;
      __syncthreads();
      if (done) break;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 48; j++) s += acc[j];
  if (s == 12345.0f) buf[0] = s;  // keep the accumulators live
}

// Worker slow-down proportional to its own work: spin on `ctas` CTAs for
// scale * (stamps[end] - stamps[begin]) ns -- a device `scale + 1` times slower
// than this one (DisturbanceEvent.cost_multiplier for a simulated worker).
__global__ void __launch_bounds__(256) spin_scaled_kernel(const int64_t* stamps, int64_t b, int64_t e, float scale) {
  __shared__ volatile int done;
  __shared__ long long ns;
  if (threadIdx.x == 0) {
    done = 0;
    ns = (long long)((double)(stamps[e] - stamps[b]) * (double)scale);
  }
  __syncthreads();
  const long long t0 = globaltimer();
  float acc = threadIdx.x;
  for (int it = 1;; it++) {
#pragma unroll 8
    for (int k = 0; k < 64; k++) acc = fmaf(acc, 1.0000001f, 0.5f);
    if ((it & 7) == 0) {
      if (threadIdx.x == 0 && globaltimer() - t0 > ns) done = 1;
      __syncthreads();
      if (done) break;
    }
  }
  if (acc == 12345.0f) done = 2;
}

__global__ void __launch_bounds__(kSpinThreads, 1) spin_for_kernel(long long ns) {
  extern __shared__ float buf[];
  __shared__ volatile int done;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  const long long t0 = globaltimer();
  float acc = threadIdx.x;
  for (int it = 1;; it++) {
#pragma unroll 8
    for (int k = 0; k < 64; k++) acc = fmaf(acc, 1.0000001f, 0.5f);
    buf[(threadIdx.x + it) & 1023] = acc;
    if ((it & 15) == 0) {
      if (threadIdx.x == 0 && globaltimer() - t0 > ns) done = 1;
      __syncthreads();
      if (done) break;
    }
  }
  if (acc == 12345.0f) buf[0] = acc;
}

__global__ void stamp_kernel(int64_t* stamps, int64_t slot) { stamps[slot] = globaltimer(); }

__global__ void accumulate_kernel(const int64_t* stamps, int64_t b, int64_t e, double* secs, int64_t w) {
  secs[w] += (double)(stamps[e] - stamps[b]) * 1e-9;
}

// set on every call: the attribute is per context, and workers may run in
// their own (green) contexts
int set_spin_attrs() {
  DBS_CUDA_TRY(cudaFuncSetAttribute(spin_until_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSpinSmem));
  DBS_CUDA_TRY(cudaFuncSetAttribute(spin_for_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSpinSmem));
  return DBS_OK;
}

}  // namespace

int stamp(int64_t* d_stamps, int64_t slot, cudaStream_t s) {
  stamp_kernel<<<1, 1, 0, s>>>(d_stamps, slot);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

int spin_scaled(const int64_t* d_stamps, int64_t b, int64_t e, float scale, int ctas, cudaStream_t s) {
  if (scale <= 0.f || ctas <= 0) return DBS_OK;
  spin_scaled_kernel<<<ctas, 256, 0, s>>>(d_stamps, b, e, scale);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

}  // namespace dbs

using namespace dbs;

extern "C" int dbs_dev_spin_until(int32_t num_ctas, const volatile int32_t* d_stop, void* stream) {
  DBS_REQUIRE(num_ctas >= 0 && num_ctas < num_sms() && d_stop, DBS_ERR_ARGUMENT,
              "spin_until: need 0 <= num_ctas < SM count (%d)", num_sms());
  if (num_ctas == 0) return DBS_OK;
  int st = set_spin_attrs();
  if (st) return st;
  static const int sleep = [] {
    const char* e = getenv("DBS_SPIN_SLEEP");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  spin_until_kernel<<<num_ctas, kSpinThreads, kSpinSmem, as_stream(stream)>>>(d_stop, sleep);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

namespace dbs {
int ctx_push(void* ctx);
int ctx_pop(void* ctx);
}  // namespace dbs

extern "C" int dbs_dev_spin_until_ctx(int32_t num_ctas, const volatile int32_t* d_stop, void* stream, void* ctx) {
  int st = ctx_push(ctx);
  if (st) return st;
  st = dbs_dev_spin_until(num_ctas, d_stop, stream);
  int st2 = ctx_pop(ctx);
  return st ? st : st2;
}

extern "C" int dbs_dev_spin_for(int32_t num_ctas, int64_t ns, void* stream) {
  DBS_REQUIRE(num_ctas >= 0 && num_ctas <= num_sms() && ns >= 0, DBS_ERR_ARGUMENT, "spin_for: bad arguments");
  if (num_ctas == 0 || ns == 0) return DBS_OK;
  int st = set_spin_attrs();
  if (st) return st;
  spin_for_kernel<<<num_ctas, kSpinThreads, kSpinSmem, as_stream(stream)>>>(ns);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

extern "C" int dbs_dev_stamp(int64_t* d_stamps, int64_t slot, void* stream) {
  stamp_kernel<<<1, 1, 0, as_stream(stream)>>>(d_stamps, slot);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

extern "C" int dbs_dev_accumulate_time(const int64_t* d_stamps, int64_t begin, int64_t end, double* d_seconds,
                                       int64_t worker, void* stream) {
  accumulate_kernel<<<1, 1, 0, as_stream(stream)>>>(d_stamps, begin, end, d_seconds, worker);
  DBS_LAUNCH_CHECK();
  return DBS_OK;
}

// Set a device int32 flag with a copy-engine transfer from pinned host memory:
// no kernel (not even the driver's memset kernels) is involved, so it is safe
// to issue while a spin kernel owns SMs and a lazily loaded module could stall.
extern "C" int dbs_dev_set_flag(int32_t* d_flag, int32_t value, void* stream) {
  DBS_REQUIRE(d_flag && (value == 0 || value == 1), DBS_ERR_ARGUMENT, "set_flag: value must be 0 or 1");
  static int32_t* host_vals = nullptr;
  if (host_vals == nullptr) {
    DBS_CUDA_TRY(cudaMallocHost(&host_vals, 2 * sizeof(int32_t)));
    host_vals[0] = 0;
    host_vals[1] = 1;
  }
  DBS_CUDA_TRY(cudaMemcpyAsync(d_flag, host_vals + value, sizeof(int32_t), cudaMemcpyHostToDevice, as_stream(stream)));
  return DBS_OK;
}

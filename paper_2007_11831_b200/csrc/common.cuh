// common.cuh -- shared helpers of libdbs_b200 (status plumbing, launch checks).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/dbs_b200.h"

namespace dbs {

// Thread-local detail string behind dbs_last_error().
void set_error(const char* fmt, ...);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

#define DBS_CUDA_TRY(expr)                                                             \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess) {                                                           \
      ::dbs::set_error("%s:%d %s -> %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return DBS_ERR_CUDA;                                                             \
    }                                                                                  \
  } while (0)

// every kernel launch of the library goes through this check, which also counts it
void count_launch();

// Programmatic dependent launch: the kernel may start (prologue: barriers, TMEM,
// shared-memory tables) while its predecessor on the stream drains; it calls
// pdl_wait() before touching memory the predecessor produces or consumes
// (griddepcontrol.wait returns once the predecessor grid has completed and its
// writes are visible -- a no-op for a launch without the attribute).
// DBS_PDL=0: plain stream-ordered launches (profiling: per-kernel times without the
// early-launched waiting that programmatic dependent launch folds into them)
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("DBS_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
// let the next PDL launch on the stream begin its prologue, then wait for ours
__device__ __forceinline__ void pdl_trigger_and_wait() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
// 256-bit global accesses (LDG/STG.256 on sm_100): 8 x 32-bit per instruction; twice the
// bytes in flight per load of the float4 forms (the HBM-bound kernels need the depth:
// resnet.cu BN passes 0.58 -> 0.93 of a partition's copy rate).  p 32-byte aligned.
struct __align__(32) V8 {
  uint32_t v[8];
};
__device__ __forceinline__ V8 ldg8_cs(const void* p) {  // streaming (evict-first)
  V8 r;
  asm volatile("ld.global.cs.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]), "=r"(r.v[6]),
                 "=r"(r.v[7])
               : "l"(p));
  return r;
}
__device__ __forceinline__ V8 ldg8(const void* p) {
  V8 r;
  asm volatile("ld.global.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]), "=r"(r.v[6]),
                 "=r"(r.v[7])
               : "l"(p));
  return r;
}
__device__ __forceinline__ void stg8_cs(void* p, const V8& r) {
  asm volatile("st.global.cs.v8.u32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(r.v[0]), "r"(r.v[1]),
               "r"(r.v[2]), "r"(r.v[3]), "r"(r.v[4]), "r"(r.v[5]), "r"(r.v[6]), "r"(r.v[7])
               : "memory");
}
__device__ __forceinline__ void stg8(void* p, const V8& r) {
  asm volatile("st.global.v8.u32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(r.v[0]), "r"(r.v[1]),
               "r"(r.v[2]), "r"(r.v[3]), "r"(r.v[4]), "r"(r.v[5]), "r"(r.v[6]), "r"(r.v[7])
               : "memory");
}
__device__ __forceinline__ float f8(const V8& r, int k) { return __uint_as_float(r.v[k]); }
__device__ __forceinline__ V8 v8_of(const float (&x)[8]) {
  V8 r;
#pragma unroll
  for (int k = 0; k < 8; k++) r.v[k] = __float_as_uint(x[k]);
  return r;
}

#define DBS_LAUNCH_CHECK()     \
  do {                         \
    ::dbs::count_launch();     \
    DBS_CUDA_TRY(cudaGetLastError()); \
  } while (0)

#define DBS_REQUIRE(cond, code, ...)  \
  do {                                \
    if (!(cond)) {                    \
      ::dbs::set_error(__VA_ARGS__);  \
      return (code);                  \
    }                                 \
  } while (0)

// Grow-only device scratch owned by the library (one per calling thread).
struct Scratch {
  void* ptr = nullptr;
  size_t bytes = 0;
  int device = -1;
};
int scratch_get(Scratch& s, size_t bytes, void** out);

// Pinned host staging buffer (one per calling thread) for the host-buffer
// entry points, so H2D/D2H copies are asynchronous and small.
int pinned_get(size_t bytes, void** out);

constexpr int kNumSMs = 148;  // B200: 2 dies x 74 SMs

int num_sms();
// SMs of the current (possibly green) context -- what a launch issued now can use (partition.cu)
int current_sm_count();

}  // namespace dbs

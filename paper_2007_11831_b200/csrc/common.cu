// common.cu -- error string, scratch buffers, version queries.
#include <stdarg.h>

#include <atomic>

#include "common.cuh"

namespace dbs {

static thread_local char g_err[1024] = {0};
static std::atomic<long long> g_launches{0};

static std::atomic<long long> g_host_launches{0};  // launch API calls the host made (kernels + graphs)
void count_launch() {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  g_host_launches.fetch_add(1, std::memory_order_relaxed);
}
// kernels recorded into a graph are counted when the graph is launched, not when captured
long long launch_count() { return g_launches.load(); }
void add_launches(long long d) { g_launches.fetch_add(d, std::memory_order_relaxed); }
void count_host_launch() { g_host_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int scratch_get(Scratch& s, size_t bytes, void** out) {
  int dev = 0;
  DBS_CUDA_TRY(cudaGetDevice(&dev));
  if (s.ptr == nullptr || s.bytes < bytes || s.device != dev) {
    if (s.ptr != nullptr && s.device == dev) cudaFree(s.ptr);
    size_t want = bytes < 4096 ? 4096 : bytes;
    DBS_CUDA_TRY(cudaMalloc(&s.ptr, want));
    s.bytes = want;
    s.device = dev;
  }
  *out = s.ptr;
  return DBS_OK;
}

static thread_local void* g_pinned = nullptr;
static thread_local size_t g_pinned_bytes = 0;

int pinned_get(size_t bytes, void** out) {
  if (g_pinned == nullptr || g_pinned_bytes < bytes) {
    if (g_pinned) cudaFreeHost(g_pinned);
    size_t want = bytes < 65536 ? 65536 : bytes * 2;
    DBS_CUDA_TRY(cudaMallocHost(&g_pinned, want));
    g_pinned_bytes = want;
  }
  *out = g_pinned;
  return DBS_OK;
}

int num_sms() {
  static int cached = 0;
  if (cached == 0) {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
      cached = v;
    else
      cached = kNumSMs;
  }
  return cached;
}

}  // namespace dbs

extern "C" const char* dbs_last_error(void) { return dbs::g_err; }

extern "C" int64_t dbs_launch_count(void) { return (int64_t)dbs::g_launches.load(); }
extern "C" int64_t dbs_host_launch_count(void) { return (int64_t)dbs::g_host_launches.load(); }

extern "C" int dbs_version(int* major, int* minor, int* sm_arch) {
  if (major) *major = 0;
  if (minor) *minor = 1;
  if (sm_arch) *sm_arch = 100;
  return DBS_OK;
}

extern "C" int dbs_device_ok(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return 0;
  }
  int dev = 0;
  cudaDeviceProp p;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaGetDeviceProperties(&p, dev) != cudaSuccess) return 0;
  return p.major == 10 ? 1 : 0;
}

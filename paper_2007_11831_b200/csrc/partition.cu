// partition.cu -- SM partitions (green contexts) for simulated workers on one GPU.
//
// Each simulated worker gets a disjoint set of SMs (a green context created
// from the device's SM resource) and its own stream in that context; the
// iteration driver makes the worker's context current while it launches that
// worker's kernels, so its forward/backward runs ONLY on its SMs.  A spin
// kernel launched in worker w's context then slows worker w alone -- the
// per-device disturbance of the paper's experiments, on one B200.
#include <cuda.h>
#include <string.h>

#include <mutex>

#include "common.cuh"

namespace dbs {
namespace {

struct DriverApi {
  CUresult (*devGetResource)(CUdevice, CUdevResource*, CUdevResourceType) = nullptr;
  CUresult (*smSplit)(CUdevResource*, unsigned int*, const CUdevResource*, CUdevResource*, unsigned int,
                      unsigned int) = nullptr;
  CUresult (*genDesc)(CUdevResourceDesc*, CUdevResource*, unsigned int) = nullptr;
  CUresult (*greenCreate)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned int) = nullptr;
  CUresult (*ctxFromGreen)(CUcontext*, CUgreenCtx) = nullptr;
  CUresult (*greenStream)(CUstream*, CUgreenCtx, unsigned int, int) = nullptr;
  CUresult (*pushCtx)(CUcontext) = nullptr;
  CUresult (*popCtx)(CUcontext*) = nullptr;
  CUresult (*getCurrent)(CUcontext*) = nullptr;
  CUresult (*ctxGetResource)(CUcontext, CUdevResource*, CUdevResourceType) = nullptr;
  bool ok = false;
};

DriverApi& api() {
  static DriverApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess;
    };
    bool ok = true;
    ok &= get("cuDeviceGetDevResource", (void**)&a.devGetResource);
    ok &= get("cuDevSmResourceSplitByCount", (void**)&a.smSplit);
    ok &= get("cuDevResourceGenerateDesc", (void**)&a.genDesc);
    ok &= get("cuGreenCtxCreate", (void**)&a.greenCreate);
    ok &= get("cuCtxFromGreenCtx", (void**)&a.ctxFromGreen);
    ok &= get("cuGreenCtxStreamCreate", (void**)&a.greenStream);
    ok &= get("cuCtxPushCurrent", (void**)&a.pushCtx);
    ok &= get("cuCtxPopCurrent", (void**)&a.popCtx);
    get("cuCtxGetCurrent", (void**)&a.getCurrent);
    get("cuCtxGetDevResource", (void**)&a.ctxGetResource);
    a.ok = ok;
  });
  return a;
}

constexpr int kMaxGroups = 16;

}  // namespace

int ctx_push(void* ctx) {
  if (!ctx) return DBS_OK;
  DriverApi& a = api();
  DBS_REQUIRE(a.ok, DBS_ERR_UNSUPPORTED, "green-context driver API unavailable");
  CUresult r = a.pushCtx(reinterpret_cast<CUcontext>(ctx));
  DBS_REQUIRE(r == CUDA_SUCCESS, DBS_ERR_CUDA, "cuCtxPushCurrent failed (%d)", (int)r);
  return DBS_OK;
}

// SMs available to work launched now: the current (green) context's SM
// resource, cached per context; the whole device when unknown.
int current_sm_count() {
  DriverApi& a = api();
  static thread_local CUcontext last = nullptr;
  static thread_local int last_sms = 0;
  if (!a.getCurrent || !a.ctxGetResource) return num_sms();
  CUcontext c = nullptr;
  if (a.getCurrent(&c) != CUDA_SUCCESS || c == nullptr) return num_sms();
  if (c == last && last_sms > 0) return last_sms;
  CUdevResource r;
  memset(&r, 0, sizeof(r));
  int sms = num_sms();
  if (a.ctxGetResource(c, &r, CU_DEV_RESOURCE_TYPE_SM) == CUDA_SUCCESS && r.sm.smCount > 0) sms = (int)r.sm.smCount;
  last = c;
  last_sms = sms;
  return sms;
}

int ctx_pop(void* ctx) {
  if (!ctx) return DBS_OK;
  CUcontext c;
  CUresult r = api().popCtx(&c);
  DBS_REQUIRE(r == CUDA_SUCCESS, DBS_ERR_CUDA, "cuCtxPopCurrent failed (%d)", (int)r);
  return DBS_OK;
}

}  // namespace dbs

struct dbs_partition {
  int n = 0;
  int sms = 0;
  CUgreenCtx g[dbs::kMaxGroups];
  CUcontext ctx[dbs::kMaxGroups];
  CUstream stream[dbs::kMaxGroups];
  CUstream side[dbs::kMaxGroups];
};

using namespace dbs;

extern "C" int dbs_partition_create(int32_t n_groups, int32_t sms_per_group, dbs_partition** out,
                                    int32_t* actual_sms) {
  DriverApi& a = api();
  DBS_REQUIRE(a.ok, DBS_ERR_UNSUPPORTED, "green-context driver API unavailable");
  DBS_REQUIRE(out && n_groups >= 1 && n_groups <= kMaxGroups && sms_per_group >= 1, DBS_ERR_ARGUMENT,
              "partition_create: 1..%d groups", kMaxGroups);
  int dev = 0;
  DBS_CUDA_TRY(cudaGetDevice(&dev));
  DBS_CUDA_TRY(cudaFree(nullptr));  // make sure the primary context exists
  CUdevResource all;
  memset(&all, 0, sizeof(all));
  CUresult r = a.devGetResource((CUdevice)dev, &all, CU_DEV_RESOURCE_TYPE_SM);
  DBS_REQUIRE(r == CUDA_SUCCESS, DBS_ERR_CUDA, "cuDeviceGetDevResource failed (%d)", (int)r);
  CUdevResource groups[kMaxGroups];
  CUdevResource rem;
  memset(groups, 0, sizeof(groups));
  memset(&rem, 0, sizeof(rem));
  unsigned int nb = (unsigned int)n_groups;
  r = a.smSplit(groups, &nb, &all, &rem, 0, (unsigned int)sms_per_group);
  DBS_REQUIRE(r == CUDA_SUCCESS && (int)nb == n_groups, DBS_ERR_CUDA,
              "cuDevSmResourceSplitByCount failed (%d, got %u groups)", (int)r, nb);
  dbs_partition* p = new dbs_partition();
  p->n = n_groups;
  p->sms = (int)groups[0].sm.smCount;
  for (int i = 0; i < n_groups; i++) {
    CUdevResourceDesc desc;
    r = a.genDesc(&desc, &groups[i], 1);
    if (r == CUDA_SUCCESS) r = a.greenCreate(&p->g[i], desc, (CUdevice)dev, CU_GREEN_CTX_DEFAULT_STREAM);
    if (r == CUDA_SUCCESS) r = a.ctxFromGreen(&p->ctx[i], p->g[i]);
    if (r == CUDA_SUCCESS) r = a.greenStream(&p->stream[i], p->g[i], CU_STREAM_NON_BLOCKING, 0);
    if (r == CUDA_SUCCESS) r = a.greenStream(&p->side[i], p->g[i], CU_STREAM_NON_BLOCKING, 0);
    if (r != CUDA_SUCCESS) {
      delete p;
      set_error("green context %d creation failed (%d)", i, (int)r);
      return DBS_ERR_CUDA;
    }
  }
  if (actual_sms) *actual_sms = p->sms;
  *out = p;
  return DBS_OK;
}

extern "C" int dbs_partition_get(const dbs_partition* p, int32_t group, void** ctx, void** stream, void** side_stream) {
  DBS_REQUIRE(p && group >= 0 && group < p->n, DBS_ERR_ARGUMENT, "partition_get: bad group");
  if (ctx) *ctx = p->ctx[group];
  if (stream) *stream = p->stream[group];
  if (side_stream) *side_stream = p->side[group];
  return DBS_OK;
}

// Make a partition's context current on the calling thread (and restore the previous
// one): host code that launches library kernels into that partition between the two
// calls -- e.g. a per-kernel measurement inside a worker's SM set.
extern "C" int dbs_partition_push(void* ctx) { return dbs::ctx_push(ctx); }
extern "C" int dbs_partition_pop(void* ctx) { return dbs::ctx_pop(ctx); }

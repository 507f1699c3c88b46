// pending.cu -- entry points declared in dbs_b200.h whose kernels land in a
// later commit; they fail loudly (DBS_ERR_UNSUPPORTED) instead of falling back.
#include "common.cuh"

#define PENDING(name) dbs::set_error(#name ": not built yet"); return DBS_ERR_UNSUPPORTED

extern "C" {
int dbs_comm_handle_size(void) { return 0; }
int dbs_comm_alloc(int32_t, int32_t, int64_t, dbs_comm**, void*) { PENDING(dbs_comm_alloc); }
int dbs_comm_open(dbs_comm*, const void*) { PENDING(dbs_comm_open); }
int dbs_comm_buffers(dbs_comm*, float**, float**, uint16_t**) { PENDING(dbs_comm_buffers); }
int dbs_comm_destroy(dbs_comm*) { PENDING(dbs_comm_destroy); }
int dbs_comm_allreduce_sgd(dbs_comm*, const int64_t*, int32_t, float, float, float*, void*) { PENDING(x); }
int dbs_comm_average_params(dbs_comm*, const int64_t*, int32_t, void*) { PENDING(x); }
}

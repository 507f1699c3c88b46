/*
 * dbs_b200.h -- C ABI of the B200-native Dynamic Batch Size (DBS) hot path.
 *
 * One shared library (paper_2007_11831_b200/libdbs_b200.so) exports every symbol
 * below.  Plain pointers, sizes and status codes only: no torch or CUDA types in
 * the signatures (streams are passed as `void*` = cudaStream_t, NULL = legacy
 * default stream).  Each entry point names the reference function it replaces
 * (paths relative to /root/reference/pkg/src/dbsim/).  The Python host mirror
 * (the paper_2007_11831_b200 package) binds these with ctypes; INTEGRATION.md shows
 * the binding the reference's own package would add.
 *
 * Two calling conventions:
 *   dbs_*            HOST buffers in/out.  The call copies inputs to the device,
 *                    runs the kernel, copies results back and synchronises.  This
 *                    is the drop-in for the reference's pure functions.
 *   dbs_dev_*        DEVICE buffers, asynchronous on `stream`; errors that the
 *                    reference raises are written to a device status word so the
 *                    epoch loop never leaves the GPU.
 *
 * Every function returns a dbs_status.  The codes map 1:1 onto the reference
 * exception classes of errors.py:4-53 (see dbs_status below).
 */
#ifndef DBS_B200_H
#define DBS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------------ */
/* Status codes  (errors.py:4-53)                                            */
/* ------------------------------------------------------------------------ */
typedef enum {
  DBS_OK = 0,
  DBS_ERR_INVALID_MEASUREMENT = 1, /* InvalidMeasurementError  errors.py:8  */
  DBS_ERR_INVALID_PERFORMANCE = 2, /* InvalidPerformanceError  errors.py:12 */
  DBS_ERR_BUDGET_TOO_SMALL = 3,    /* BudgetTooSmallError      errors.py:16 */
  DBS_ERR_INVALID_BATCH = 4,       /* InvalidBatchError        errors.py:20 */
  DBS_ERR_EMPTY_PARTITION = 5,     /* EmptyPartitionError      errors.py:24 */
  DBS_ERR_DATASET_TOO_SMALL = 6,   /* DatasetTooSmallError     errors.py:28 */
  DBS_ERR_CONFIGURATION = 7,       /* ConfigurationError       errors.py:32 */
  DBS_ERR_EMPTY_BATCH = 9,         /* EmptyBatchError          errors.py:40 */
  DBS_ERR_INVALID_STEP_SIZE = 10,  /* InvalidStepSizeError     errors.py:44 */
  DBS_ERR_FSUM_OVERFLOW = 20,      /* math.fsum OverflowError ("intermediate overflow") */
  DBS_ERR_FSUM_INF_NAN = 21,       /* math.fsum ValueError ("-inf + inf in fsum")       */
  DBS_ERR_INT_OVERFLOW = 22,       /* value outside int64 where Python has big ints      */
  DBS_ERR_ARGUMENT = 30,           /* NULL pointer / unsupported size                    */
  DBS_ERR_CUDA = 40,               /* CUDA runtime / driver failure (dbs_last_error())   */
  DBS_ERR_UNSUPPORTED = 41         /* hardware feature missing (not sm_100)              */
} dbs_status;

/* Human-readable detail of the last error on the calling thread. */
const char* dbs_last_error(void);
/* Library version and the SM architecture the kernels were built for (100). */
int dbs_version(int* major, int* minor, int* sm_arch);
/* 1 when a CUDA device with compute capability 10.x is visible. */
int dbs_device_ok(void);
/* Number of kernels this library has launched (or captured into a graph) so far. */
int64_t dbs_launch_count(void);
/* Launch API calls this process's host threads made through the library (each
 * kernel launch, captured or not, and each per-worker graph launch). */
int64_t dbs_host_launch_count(void);

/* ------------------------------------------------------------------------ */
/* (3) Epoch-end DBS controller  -- allocation.py, single-CTA fp64 kernel   */
/* All fp64 arithmetic is IEEE round-to-nearest with no FMA contraction, the */
/* correctly-rounded sum of math.fsum, and exact int64/int128 rationals, so  */
/* results are bit-identical to the reference.                               */
/* ------------------------------------------------------------------------ */

/* allocation.evaluate_performance (allocation.py:78-88), applied to n pairs. */
int dbs_evaluate_performance(const double* shares, const double* times, int64_t n,
                             double* perf_out, int64_t* bad_index);

/* allocation.compute_batch_fractions (allocation.py:91-102). */
int dbs_compute_batch_fractions(const double* perfs, int64_t n, double* fractions_out,
                                int64_t* bad_index);

/* allocation.scale_to_real_batches (allocation.py:105-113). */
int dbs_scale_to_real_batches(const double* fractions, int64_t n, int64_t total_budget,
                              double* real_out);

/* allocation.round_twice (allocation.py:116-137). */
int dbs_round_twice(const double* real_batches, int64_t n, int64_t total_budget,
                    int64_t* int_out);

/* allocation._raise_zero_batches (allocation.py:191-204). */
int dbs_raise_zero_batches(const int64_t* int_batches, int64_t n, int64_t* out);

/* allocation.partition_ranges (allocation.py:140-155): range i is
 * [cum[i]/cum[n], cum[i+1]/cum[n]) as exact rationals; cum has n+1 entries. */
int dbs_partition_ranges(const int64_t* int_batches, int64_t n, int64_t* cum_out);

/* A range bound as the reference may receive it: an exact rational
 * (Fraction or int: kind 0, num/den with den > 0) or an IEEE double (kind 1). */
typedef struct {
  int32_t kind;
  int32_t reserved;
  int64_t num;
  int64_t den;
  double value;
} dbs_bound;

/* allocation.spans_from_ranges (allocation.py:158-188): spans_out[2i],
 * spans_out[2i+1] = half-open sample span of worker i. */
int dbs_spans_from_ranges(const dbs_bound* lo, const dbs_bound* hi, int64_t n,
                          int64_t dataset_size, int64_t* spans_out);

/* allocation.plan_next_epoch (allocation.py:207-244), whole pipeline in one
 * launch.  Outputs: int_batches[n], cum[n+1] (ranges), spans[2n]. */
int dbs_plan_next_epoch(const double* prev_shares, const double* prev_times, int64_t n,
                        int64_t total_budget, int64_t dataset_size, int64_t epoch,
                        int64_t* int_batches_out, int64_t* cum_out, int64_t* spans_out,
                        int64_t* bad_index);

/* Device-resident re-plan: cluster.run_training's DBS branch
 * (cluster.py:253-271) followed by plan_next_epoch, with the previous
 * epoch's measured per-worker compute seconds in d_times.
 *   d_prev_spans [2n]  previous plan's spans (shares = width / D, allocation.py:72-75)
 *   d_smoothed   [n]   EMA state (cluster.py:263-266), updated in place
 *   d_flags      [2]   [0] = EMA state valid, [1] = status (dbs_status) out
 * epoch == 0 or kind != dbs gives the even plan (cluster.py:254-255, 223-231).
 * Outputs land in d_int_batches[n], d_cum[n+1], d_spans[2n], d_iters[1]
 * (iterations_for_plan, cluster.py:159-170). */
int dbs_dev_replan(const int64_t* d_prev_spans, const double* d_times, int64_t n,
                   int64_t total_budget, int64_t dataset_size, int64_t epoch, int32_t adaptive,
                   double perf_smoothing, double* d_smoothed, int32_t* d_flags,
                   int64_t* d_int_batches, int64_t* d_cum, int64_t* d_spans, int64_t* d_iters,
                   void* stream);

/* ------------------------------------------------------------------------ */
/* Sample assignment  -- sgdlab.py:358, 372-374                              */
/* numpy Generator(PCG64) semantics: SeedSequence seeding, PCG64 XSL-RR      */
/* 128/64, buffered next_uint32, masked-rejection random_interval, reversed  */
/* Fisher-Yates (numpy 2.3 Generator.permutation).                           */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint64_t state_hi, state_lo; /* 128-bit LCG state */
  uint64_t inc_hi, inc_lo;     /* 128-bit odd increment */
  uint32_t has_uint32;         /* buffered upper half pending */
  uint32_t uinteger;           /* the buffered upper half */
} dbs_pcg64;

/* numpy.random.default_rng(seed) for a non-negative integer seed given as
 * little-endian 32-bit words (SeedSequence entropy). Host-side setup. */
int dbs_pcg64_seed(const uint32_t* seed_words, int32_t n_words, dbs_pcg64* out);

/* Host-buffer drop-in: for each span i (in order, one generator),
 * perm_out[off_i + k] = start_i + rng.permutation(end_i - start_i)[k],
 * off_i = sum of earlier span widths.  rng is advanced in place. */
int dbs_permute_spans(dbs_pcg64* rng, const int64_t* spans, int64_t n, int64_t* perm_out);

/* Device version.  d_rng is device-resident and advanced in place.
 * only_span = -1 materialises every span; otherwise only that span's
 * indices are written (the draws of every span are still consumed, so all
 * ranks stay in lock-step with the reference's single generator).
 * d_draws is scratch of at least sum(widths) int32. */
int dbs_dev_permute_spans(dbs_pcg64* d_rng, const int64_t* d_spans, int64_t n,
                          int64_t total_width, int64_t only_span, int64_t* d_perm_out,
                          int32_t* d_draws, void* stream);

/* ------------------------------------------------------------------------ */
/* Repartition gather  -- the row gathers offsets[idx] / features[idx]       */
/* (sgdlab.py:82, 144) done once per epoch as a coalesced shard repack.      */
/* ------------------------------------------------------------------------ */
/* dst[r, :] = src[idx[r], :] for r < rows; rows of row_bytes bytes. */
int dbs_dev_gather_rows(const void* d_src, const int64_t* d_idx, int64_t rows,
                        int64_t row_bytes, void* d_dst, void* stream);
/* Same, converting fp32 rows of `cols` elements to bf16 (model input staging). */
int dbs_dev_gather_rows_f32_bf16(const float* d_src, const int64_t* d_idx, int64_t rows,
                                 int64_t cols, void* d_dst_bf16, void* stream);
/* fp32 rows -> S32 rows of ld_out (% 32) logical columns (the fp32-class MLP input
 * format; columns past cols zero). */
int dbs_dev_gather_rows_f32_s32(const float* d_src, const int64_t* d_idx, int64_t rows, int64_t cols,
                                float* d_dst, int64_t ld_out, void* stream);
/* Same for int32 labels. */
int dbs_dev_gather_i32(const int32_t* d_src, const int64_t* d_idx, int64_t rows,
                       int32_t* d_dst, void* stream);

/* ------------------------------------------------------------------------ */
/* (2) Batch-weighted aggregation + momentum SGD  -- sgdlab.py:208-238       */
/* ------------------------------------------------------------------------ */
enum { DBS_AGG_UNIFORM = 0, DBS_AGG_BATCH_WEIGHTED = 1 };

/* sgdlab.aggregate_gradients (sgdlab.py:208-227) over n device gradient
 * buffers of P doubles (d_grads: HOST array of n device pointers): out = sum_i w_i g_i, w_i = b_i / sum(b) or 1/n. */
int dbs_dev_aggregate_f64(const double* const* d_grads, const int64_t* batch_sizes, int64_t n,
                          int32_t mode, int64_t P, double* d_out, void* stream);
/* sgdlab.sgd_step (sgdlab.py:230-238), out of place:
 * v' = momentum v + g ; x' = x - step v'. */
int dbs_dev_sgd_step_f64(const double* d_x, const double* d_g, const double* d_v, int64_t P,
                         double step, double momentum, double* d_x_out, double* d_v_out,
                         void* stream);
/* Fused single-device aggregate + step, in place (the per-iteration update
 * of run_parallel_sgd, sgdlab.py:385-386), fp64. */
int dbs_dev_aggregate_sgd_f64(const double* const* d_grads, const int64_t* batch_sizes, int64_t n,
                              int32_t mode, int64_t P, double step, double momentum,
                              double* d_x, double* d_v, void* stream);
/* fp32 model-parameter variant: grads fp32, params/velocity fp32 master,
 * optional bf16 shadow of the params (GEMM operand) written in the same pass. */
int dbs_dev_aggregate_sgd_f32(const float* const* d_grads, const int64_t* batch_sizes, int64_t n,
                              int32_t mode, int64_t P, float step, float momentum, float* d_x,
                              float* d_v, uint16_t* d_x_bf16, void* stream);

/* Operand precision of a model's tensor-core path:
 *   DBS_PREC_BF16 -- bf16 GEMM operands, parameter shadow bf16 [P];
 *   DBS_PREC_F32  -- fp32-class 3xTF32 GEMMs on S32 operands (dbs_dev_gemm_tf32x3),
 *                    parameter shadow = the flat param vector in S32 format
 *                    (2P floats: element i's hi at 2 (i & ~31) + (i & 31), lo 32 later;
 *                    every tensor starts at a multiple of 32, P % 32 == 0). */
enum { DBS_PREC_BF16 = 0, DBS_PREC_F32 = 1 };
/* aggregate + step writing the operand shadow in shadow_prec's format */
int dbs_dev_aggregate_sgd_f32_ex(const float* const* d_grads, const int64_t* batch_sizes, int64_t n,
                                 int32_t mode, int64_t P, float step, float momentum, float* d_x,
                                 float* d_v, void* d_shadow, int32_t shadow_prec, void* stream);
/* shadow <- the operand copy of fp32 params x[P] (DBS_PREC_* format) */
int dbs_dev_refresh_shadow(const float* d_x, int64_t P, void* d_shadow, int32_t prec, void* stream);

/* Multi-GPU: one process per GPU.  A communicator holds the peer-mapped
 * (CUDA IPC over NVLink/NVSwitch) symmetric buffers:
 *   grad[P] fp32, param[P] fp32, param_bf16[P], signal words.
 * dbs_comm_alloc allocates this rank's symmetric block and returns its IPC
 * handle bytes; dbs_comm_open maps every peer's block (handles gathered by the
 * host with any transport, e.g. torch.distributed). */
typedef struct dbs_comm dbs_comm;
int dbs_comm_handle_size(void);
int dbs_comm_alloc(int32_t rank, int32_t world, int64_t P, dbs_comm** out, void* handle_out);
int dbs_comm_open(dbs_comm* comm, const void* all_handles /* world * handle_size */);
int dbs_comm_buffers(dbs_comm* comm, float** d_grad, float** d_param, uint16_t** d_param_bf16);
/* Parameter operand shadow of the communicator: DBS_PREC_BF16 (default) = its bf16
 * block, pushed to every peer with the fp32 parameters; DBS_PREC_F32 = a local S32
 * buffer of 2 P floats (P = the padded count), refreshed by the iteration driver
 * after each update (the fused kernel then pushes fp32 only). */
int dbs_comm_set_shadow(dbs_comm* comm, void* d_shadow, int32_t prec);
int dbs_comm_shadow(const dbs_comm* comm, void** d_shadow, int32_t* prec);
/* padded parameter count (multiple of 32 * world) and the per-rank shard length */
int dbs_comm_info(const dbs_comm* comm, int64_t* padded_P, int64_t* shard);
/* unmap the IPC-opened peer blocks (before dbs_comm_destroy) */
int dbs_comm_close_peers(dbs_comm* comm);
int dbs_comm_destroy(dbs_comm* comm);
/* single-process form: `world` communicators over plain local blocks of the
 * current device (simulated ranks; used by the tests on one GPU) */
int dbs_comm_create_local(int32_t world, int64_t P, dbs_comm** comms_out);
/* The fused per-iteration kernel: each rank owns shard [r*P/W, (r+1)*P/W);
 * it loads the shard of every peer's gradient over NVLink, forms
 * sum_j w_j g_j (w_j = b_j / sum b), applies v' = mom v + g, x' = x - lr v',
 * and stores x' (fp32 + bf16) into every peer's parameter buffer; in-kernel
 * signal barriers order the exchange.  d_velocity is this rank's shard.
 * mode DBS_AGG_* ; batch_sizes is a host array of W entries. */
int dbs_comm_allreduce_sgd(dbs_comm* comm, const int64_t* batch_sizes, int32_t mode, float step,
                           float momentum, float* d_velocity_shard, void* stream);
/* Model averaging (cluster.py:185-186 cadence): params <- sum_j w_j param_j,
 * same kernel skeleton without the momentum step. */
int dbs_comm_average_params(dbs_comm* comm, const int64_t* batch_sizes, int32_t mode,
                            void* stream);

/* ------------------------------------------------------------------------ */
/* (1) Variable-batch forward/backward  -- per_sample_gradients + mean      */
/* (sgdlab.py:200-205, 81-82, 143-148) and the named models.                 */
/* ------------------------------------------------------------------------ */
/* ConvexProblem (sgdlab.py:33-95): out[w] = mean_k mu (x - opt - offsets[idx_w[k]])
 * for n_workers index lists concatenated in d_idx with offsets d_off[n+1]. */
int dbs_dev_quadratic_grads(const double* d_x, const double* d_opt, const double* d_offsets,
                            int64_t dim, const int64_t* d_idx, const int64_t* d_off,
                            int64_t n_workers, double mu, double* d_grads_out, void* stream);
/* LogisticProblem (sgdlab.py:98-159): mean_k (coeff_k feats_k + mu x),
 * coeff = -y / (1 + exp(y feats.x)). */
int dbs_dev_logistic_grads(const double* d_x, const double* d_features, const double* d_labels,
                           int64_t dim, const int64_t* d_idx, const int64_t* d_off,
                           int64_t n_workers, double mu, double* d_grads_out, void* stream);
/* One whole epoch of run_parallel_sgd's hot loop (sgdlab.py:380-391) for the
 * reference problems in ONE single-CTA launch: for t < iters, every worker's
 * batch-mean gradient on perm[span_off[w] + t*b_w ...], aggregation
 * (DBS_AGG_*), heavy-ball step on d_x/d_v in place, and ||x - opt||^2 into
 * d_sq_out[t].  kind 0 = ConvexProblem (d_data = offsets, bit-exact order),
 * 1 = LogisticProblem (d_data = features, d_labels = +/-1).  span_off and
 * batches are HOST arrays; d_grads holds n*dim, d_coeff sum(b) doubles. */
int dbs_dev_sgd_epoch(int32_t kind, const double* d_data, const double* d_labels, const double* d_opt,
                      int64_t dim, double mu, const int64_t* d_perm, const int64_t* span_off,
                      const int64_t* batches, int64_t n_workers, int32_t mode, int64_t iters, double step,
                      double momentum, double* d_x, double* d_v, double* d_grads, double* d_coeff,
                      double* d_sq_out, void* stream);
/* ||x - opt||^2 into d_out[slot] (run_parallel_sgd's squared_distances,
 * sgdlab.py:387-388). */
int dbs_dev_sq_dist(const double* d_x, const double* d_opt, int64_t dim, double* d_out,
                    int64_t slot, void* stream);

/* tcgen05 GEMM:  D[M,N] (+)= A[M,K] * B[N,K]^T, bf16 operands, fp32 accumulate
 * in TMEM.  a_major/b_major: 0 = K contiguous, 1 = M (resp. N) contiguous; lda/ldb
 * are leading-dimension strides in elements.  epilogue selects the fused tail. */
enum {
  DBS_EPI_F32 = 0,           /* D fp32 = acc                                    */
  DBS_EPI_F32_ACCUM = 1,     /* D fp32 += acc                                   */
  DBS_EPI_BIAS_RELU_BF16 = 2,/* D bf16 = relu(acc + bias[n]); aux bf16 = acc+bias */
  DBS_EPI_BIAS_F32 = 3,      /* D fp32 = acc + bias[n]                          */
  DBS_EPI_BF16 = 4,          /* D bf16 = acc                                    */
  DBS_EPI_RELU_GRAD_BF16 = 5,/* D bf16 = acc * (aux bf16 [M][ldd] > 0)          */
  DBS_EPI_F32_ATOMIC = 6,    /* D fp32 += acc with atomics (split-K reduction)  */
  DBS_EPI_BF16_ACCUM = 7,    /* D bf16 = D + acc (gradient accumulation)        */
  /* S32 outputs (fp32-class operand format, see dbs_dev_gemm_tf32x3) */
  DBS_EPI_S32 = 8,           /* D s32 = acc                                     */
  DBS_EPI_BIAS_RELU_S32 = 9, /* D s32 = relu(acc + bias[n])                     */
  DBS_EPI_RELU_GRAD_S32 = 10 /* D s32 = acc * (aux s32 [M][ldd] > 0)            */
};
int dbs_dev_gemm_bf16(const void* d_a, int32_t a_major, int64_t lda, const void* d_b,
                      int32_t b_major, int64_t ldb, void* d_d, int64_t ldd, int64_t M, int64_t N,
                      int64_t K, int32_t epilogue, const float* d_bias, void* d_aux, void* stream);

/* fp32-class tensor-core GEMM ("3xTF32"): the same D[M,N] (+)= A[M,K] * B[N,K]^T
 * with fp32-accurate operands in the S32 split format and three kind::tf32
 * MMA passes per K block (hi*hi + hi*lo + lo*hi, fp32 accumulation in TMEM).
 * S32 format of a logical row-major [rows][ld] fp32 matrix (ld % 32 == 0):
 * every 32-element block of a row is stored as 32 fp32 "hi" values followed by
 * 32 fp32 "lo" values, hi = rn_tf32(x), lo = rn_tf32(x - hi), so hi + lo = x to
 * within ~2^-23 |x| and each part is exact in tf32 (row pitch 2*ld floats).
 * lda/ldb/ldd are LOGICAL leading dimensions (elements); S32 epilogues write D
 * in S32, F32 epilogues plain fp32.  Operand/epilogue rules as dbs_dev_gemm_bf16. */
int dbs_dev_gemm_tf32x3(const void* d_a, int32_t a_major, int64_t lda, const void* d_b,
                        int32_t b_major, int64_t ldb, void* d_d, int64_t ldd, int64_t M, int64_t N,
                        int64_t K, int32_t epilogue, const float* d_bias, void* d_aux, void* stream);
/* fp32 [rows][ld_in] (cols valid) -> S32 [rows][ld_out] (ld_out % 32 == 0, columns
 * past cols zero) and back (s32 -> fp32: x = hi + lo). */
int dbs_dev_split_s32(const float* d_x, int64_t rows, int64_t cols, int64_t ld_in, float* d_s32,
                      int64_t ld_out, void* stream);
int dbs_dev_join_s32(const float* d_s32, int64_t rows, int64_t cols, int64_t ld_in, float* d_x,
                     int64_t ld_out, void* stream);

/* 2-layer MLP (784 -> H -> C, ReLU, softmax cross-entropy): one variable-batch
 * forward + backward of a worker's batch.  Params live in one flat fp32
 * buffer laid out [W1 (H x IN) | b1 (H) | W2 (C x H) | b2 (C)], with a bf16
 * shadow of the same layout; the flat fp32 gradient of the batch-mean loss is
 * written to d_grad and the batch-mean loss to d_loss[0]. */
typedef struct dbs_mlp dbs_mlp;
int dbs_mlp_create(int64_t in_dim, int64_t hidden, int64_t classes, int64_t max_batch,
                   dbs_mlp** out);
/* precision DBS_PREC_*: DBS_PREC_F32 runs the 5 GEMMs as 3xTF32 on S32 operands;
 * its layout pads W1's rows to in_ld = in rounded up to 32 and starts every block
 * on a 32-element boundary, and its input rows are S32 [batch][in_ld]. */
int dbs_mlp_create_ex(int64_t in_dim, int64_t hidden, int64_t classes, int64_t max_batch, int32_t precision,
                      dbs_mlp** out);
int dbs_mlp_info(const dbs_mlp* m, int32_t* precision, int64_t* in_ld);
int dbs_mlp_destroy(dbs_mlp* m);
int dbs_mlp_param_count(const dbs_mlp* m, int64_t* out);
/* d_params_shadow / d_x: bf16 (DBS_PREC_BF16) or S32 (DBS_PREC_F32) */
int dbs_mlp_forward_backward(dbs_mlp* m, const void* d_params_shadow, const float* d_params,
                             const void* d_x, const int32_t* d_labels, int64_t batch,
                             float* d_grad, float* d_loss, void* stream);

/* ResNet-18, CIFAR variant (3x3 stem, no max-pool; 11,173,962 weights): one
 * variable-batch forward + backward of a worker's batch on the implicit-GEMM
 * tcgen05 convolution.  Input fp32 [B][3][32][32] rows of the repacked shard
 * (iteration t reads rows t*B.., t = *d_iter or 0), labels int32; the flat fp32
 * gradient (layout from dbs_resnet_param_table) and the batch-mean loss
 * (d_loss[t]) are written.  Local (per-worker) BatchNorm statistics. */
typedef struct dbs_resnet dbs_resnet;
int dbs_resnet_create(int64_t max_batch, int32_t classes, dbs_resnet** out);
int dbs_resnet_destroy(dbs_resnet* m);
int dbs_resnet_param_count(const dbs_resnet* m, int64_t* P);
/* torchvision parameter order; kind 0 conv weight [Cout][R][S][Cin] (stem
 * [64][32], 27 used), 1 BN gamma, 2 BN beta, 3 FC weight [C][512], 4 FC bias */
int dbs_resnet_param_table(const dbs_resnet* m, int64_t* off, int64_t* len, int32_t* kind, int32_t capacity,
                           int32_t* count);
/* d_params_shadow: the operand copy of d_params in the model's precision (bf16 [P] or S32 [2P floats]) */
int dbs_resnet_forward_backward(dbs_resnet* m, const void* d_params_shadow, const float* d_params,
                                const void* d_x, const int32_t* d_labels, int64_t batch, const int64_t* d_iter,
                                float* d_grad, float* d_loss, void* stream);
/* ResNet-50 (config 5; torchvision layout, stride on the 3x3 conv, 25,557,032
 * weights at 1000 classes): depth = 50, image = input side (224; any multiple of
 * 32 in [64, 512]), classes 2..8192.  Input rows are uint8 [B][3][image][image]
 * (pixel (u - 128) / 64), the stem weight is stored [64][160] (147 used), the
 * FC weight [classes][2048].  depth = 18 / image = 32 is dbs_resnet_create. */
int dbs_resnet_create_ex(int32_t depth, int32_t image, int64_t max_batch, int32_t classes, dbs_resnet** out);
/* The same with an operand precision (DBS_PREC_*).  DBS_PREC_F32: every conv / FC
 * GEMM is 3xTF32 on S32 operands, conv outputs and input gradients are stored
 * fp32, GEMM operands S32; BatchNorm running statistics (torch semantics,
 * momentum 0.1, unbiased variance) are tracked per worker. */
int dbs_resnet_create_ex2(int32_t depth, int32_t image, int64_t max_batch, int32_t classes, int32_t precision,
                          dbs_resnet** out);
int dbs_resnet_precision(const dbs_resnet* m, int32_t* precision);
/* device pointer to conv `conv`'s running statistics: [cout] mean, [cout] variance */
int dbs_resnet_running_stats(const dbs_resnet* m, int32_t conv, float** d_stats, int32_t* channels);
/* depth, input side, bytes per input row, padded stem K (any pointer may be NULL) */
int dbs_resnet_info(const dbs_resnet* m, int32_t* depth, int32_t* image, int64_t* row_bytes, int32_t* stem_k);

/* Implicit-GEMM convolutions (NHWC bf16, weights [Cout][k][k][Cin] bf16) on the
 * tcgen05 GEMM with 4-D TMA operand loads: y = conv(x, w); dx = dgrad(dy, w)
 * (d_scratch is unused and may be NULL; stride 2 runs one GEMM per output
 * parity class); dw += wgrad(dy, x) (fp32, atomically accumulated -- zero it
 * first). */
int dbs_dev_conv2d_fwd(const void* d_x, int32_t N, int32_t H, int32_t W, int32_t Cin, const void* d_w, int32_t Cout,
                       int32_t k, int32_t stride, int32_t pad, void* d_y, void* stream);
int dbs_dev_conv2d_dgrad(const void* d_dy, int32_t N, int32_t H, int32_t W, int32_t Cin, const void* d_w,
                         int32_t Cout, int32_t k, int32_t stride, int32_t pad, void* d_dx, void* d_scratch,
                         void* stream);
int dbs_dev_conv2d_wgrad(const void* d_dy, const void* d_x, int32_t N, int32_t H, int32_t W, int32_t Cin,
                         int32_t Cout, int32_t k, int32_t stride, int32_t pad, float* d_dw, void* stream);
/* fp32-class forms: S32 operands (NHWC activations, [Cout][k][k][Cin] weights,
 * channels multiples of 32), fp32 outputs (y, dx; dw accumulated atomically) */
/* *d_iter += 1 on the stream (the device iteration counter of graph-replayed loops). */
int dbs_dev_iter_increment(int64_t* d_iter, void* stream);
/* Stand-alone fp32-class BatchNorm passes (the network's own kernels; unit tests and
 * per-kernel rooflines).  acc = [sum C | sum of squares C] (fp64) of y [M][C] fp32;
 * out / dy / mask in the S32 operand format.  Forward: out = act(gamma yhat + beta),
 * mean / invstd written.  Backward: g masked by (mask > 0) when mask != NULL;
 * dgamma += sum g yhat, dbeta += sum g (fp32 atomics; zero them first); dy = the
 * BatchNorm input gradient; g_out (optional) = the masked g. */
int dbs_dev_bn_apply_s32(const float* d_y, const double* d_acc, const float* d_gamma, const float* d_beta, int32_t C,
                         int64_t M, int32_t relu, float* d_mean, float* d_invstd, float* d_out, void* stream);
int dbs_dev_bn_backward_s32(const float* d_g, const float* d_mask, const float* d_y, const float* d_mean,
                            const float* d_invstd, const float* d_gamma, int32_t C, int64_t M, float* d_dgamma,
                            float* d_dbeta, float* d_dy, float* d_gout, void* stream);
int dbs_dev_conv2d_fwd_s32(const void* d_x, int32_t N, int32_t H, int32_t W, int32_t Cin, const void* d_w,
                           int32_t Cout, int32_t k, int32_t stride, int32_t pad, float* d_y, void* stream);
int dbs_dev_conv2d_dgrad_s32(const void* d_dy, int32_t N, int32_t H, int32_t W, int32_t Cin, const void* d_w,
                             int32_t Cout, int32_t k, int32_t stride, int32_t pad, float* d_dx, void* stream);
int dbs_dev_conv2d_wgrad_s32(const void* d_dy, const void* d_x, int32_t N, int32_t H, int32_t W, int32_t Cin,
                             int32_t Cout, int32_t k, int32_t stride, int32_t pad, float* d_dw, void* stream);

/* One worker of a synchronous iteration (simulated worker on a shared GPU or
 * one rank's local worker).  Device pointers unless noted. */
enum { DBS_MODEL_MLP = 0, DBS_MODEL_RESNET18 = 1 };
typedef struct {
  void* model;               /* dbs_mlp* or dbs_resnet* (per-worker scratch)       */
  void* stream;              /* the worker's cudaStream_t (may be a green context) */
  const void* x_shard;       /* this epoch's repacked sample rows (MLP: bf16 [span][in];
                                ResNet: fp32 [span][3][32][32])                    */
  const int32_t* y_shard;    /* int32 [span] labels in the same order              */
  int64_t batch;             /* b_i of the current plan                            */
  float* grad;               /* [P] flat gradient of the batch-mean loss           */
  float* loss;               /* [iters] per-iteration batch loss, or NULL          */
  float* loss_scratch;       /* [1] used when loss == NULL                         */
  int64_t* stamps;           /* [2] %globaltimer scratch, NULL = no timing         */
  double* seconds;           /* device accumulator array of compute seconds        */
  int64_t worker_index;      /* slot in `seconds`                                  */
  int64_t spin_ns;           /* disturbance: extra device ns per iteration (0=off) */
  int32_t spin_ctas;         /* SMs the per-iteration disturbance occupies         */
  int32_t model_kind;        /* DBS_MODEL_*                                        */
  float slow_scale;          /* cost_multiplier - 1 of a simulated slow device: after
                                its forward/backward the worker spins scale x that
                                duration (0 = off)                                 */
  int32_t slow_ctas;         /* CTAs of that proportional spin                     */
  void* ctx;                 /* CUcontext of the worker's SM partition (green
                                context, dbs_partition_get), NULL = current         */
} dbs_worker_slot;

/* SM partitions for simulated workers: n_groups green contexts of
 * sms_per_group SMs each (rounded by the driver; actual count returned), each
 * with a worker stream and a side stream (for the disturbance). */
typedef struct dbs_partition dbs_partition;
int dbs_partition_create(int32_t n_groups, int32_t sms_per_group, dbs_partition** out, int32_t* actual_sms);
int dbs_partition_get(const dbs_partition* p, int32_t group, void** ctx, void** stream, void** side_stream);
/* make a partition's context current on this thread / restore the previous one */
int dbs_partition_push(void* ctx);
int dbs_partition_pop(void* ctx);
/* dbs_dev_spin_until launched inside a partition's context (ctx may be NULL). */
int dbs_dev_spin_until_ctx(int32_t num_ctas, const volatile int32_t* d_stop, void* stream, void* ctx);

/* Iterations [t0, t1) of one epoch of run_parallel_sgd's loop (sgdlab.py:380-391):
 * every worker's forward/backward on its stream, then the fused aggregate +
 * momentum-SGD update (mode DBS_AGG_*) on agg_stream, ordered with events;
 * skip_update = 1 measures compute only.  With d_iter != NULL (ResNet only) the
 * kernels read the iteration index from *d_iter and the update increments it,
 * so every iteration is the same launch sequence (CUDA-graph capturable).
 * d_params_shadow is the operand copy in the workers' model precision (bf16 [P]
 * or S32 [2P floats]); all workers must share one precision. */
int dbs_run_iterations(const dbs_worker_slot* workers, int32_t n, int64_t t0, int64_t t1, int32_t mode, float lr,
                       float momentum, float* d_params, float* d_velocity, void* d_params_shadow,
                       int32_t skip_update, void* agg_stream, int64_t* d_iter);
/* Per-worker CUDA graphs for workers in SM partitions (green contexts, where one
 * graph cannot span the workers' contexts): each worker's part of an iteration is
 * captured once, in its own context, and replayed per iteration -- n graph launches
 * plus the update instead of every kernel from one host thread.  A graph set is
 * valid for one plan (batches, disturbance spins, model scratch); d_iter required.
 * Replaces the eager launch loop of run_parallel_sgd's iteration (sgdlab.py:380-391). */
typedef struct dbs_worker_graphs dbs_worker_graphs;
int dbs_worker_graphs_create(int32_t n, dbs_worker_graphs** out);
int dbs_worker_graphs_destroy(dbs_worker_graphs* g);
/* Device-side epoch loop for workers sharing one context: one CUDA graph whose
 * `while` conditional node replays the captured iteration (every worker's forward /
 * backward, the update, *d_iter += 1) while *d_iter < *d_total.  Per epoch: zero
 * d_iter, set d_total = T >= 1, one dbs_epoch_graph_launch.  A graph is valid for one
 * plan (batches, spins, model scratch). */
typedef struct dbs_epoch_graph dbs_epoch_graph;
int dbs_epoch_graph_create(const dbs_worker_slot* workers, int32_t n, int32_t mode, float lr, float momentum,
                           float* d_params, float* d_velocity, void* d_params_shadow, int32_t skip_update,
                           void* agg_stream, int64_t* d_iter, const int64_t* d_total, dbs_epoch_graph** out);
int dbs_epoch_graph_launch(dbs_epoch_graph* g, int64_t iters, void* stream);
int dbs_epoch_graph_destroy(dbs_epoch_graph* g);
/* Capture the graph set (nothing runs); called before the epoch's disturbance spins
 * start (capturing may load kernels, which must not wait behind a spinning kernel). */
int dbs_worker_graphs_capture(const dbs_worker_slot* workers, int32_t n, int32_t mode, float lr, float momentum,
                              float* d_params, float* d_velocity, void* d_params_shadow, int32_t skip_update,
                              void* agg_stream, int64_t* d_iter, dbs_worker_graphs* graphs);
int dbs_run_iterations_graphed(const dbs_worker_slot* workers, int32_t n, int64_t t0, int64_t t1, int32_t mode,
                               float lr, float momentum, float* d_params, float* d_velocity, void* d_params_shadow,
                               int32_t skip_update, void* agg_stream, int64_t* d_iter, dbs_worker_graphs* graphs);
/* Multi-GPU form (one process per GPU): the rank's n local workers, then a local
 * weighted reduce into the communicator's gradient block and the fused NVLink
 * all-reduce + momentum SGD (dbs_comm_allreduce_sgd) with per-rank weights
 * rank_batches[r] (sum of that rank's worker batches); parameters are the
 * communicator's blocks, the velocity is this rank's shard. */
int dbs_run_iterations_comm(const dbs_worker_slot* workers, int32_t n, int64_t t0, int64_t t1, int32_t mode,
                            float lr, float momentum, dbs_comm* comm, const int64_t* rank_batches,
                            float* d_velocity_shard, void* agg_stream, int64_t* d_iter);
/* The multi-GPU form with per-worker graphs (see dbs_run_iterations_graphed);
 * capture_only = 1 captures the set without running (before the epoch's spins). */
int dbs_run_iterations_comm_graphed(const dbs_worker_slot* workers, int32_t n, int64_t t0, int64_t t1, int32_t mode,
                                    float lr, float momentum, dbs_comm* comm, const int64_t* rank_batches,
                                    float* d_velocity_shard, void* agg_stream, int64_t* d_iter,
                                    dbs_worker_graphs* graphs, int32_t capture_only);
/* fp32 weighted reduce out = sum_i w_i g_i (DBS_AGG_*), no step. */
int dbs_dev_aggregate_f32(const float* const* d_grads, const int64_t* batch_sizes, int64_t n, int32_t mode, int64_t P,
                          float* d_out, void* stream);
/* Periodic model averaging (local SGD; BASELINE config 4, sync interval
 * `step`): each worker trains its own replica d_params[i] / d_velocity[i] /
 * d_params_bf16[i] with a local momentum-SGD step on its stream; after every
 * sync_interval-th iteration of the epoch the replicas are replaced by their
 * `mode`-weighted average (floor(T / sync_interval) rounds per epoch, as
 * cluster.sync_rounds_for_epoch counts them, cluster.py:185-186).  Iteration
 * indices are host-side (t0..t1 of the epoch). */
int dbs_run_iterations_local(const dbs_worker_slot* w, int32_t n, int64_t t0, int64_t t1, int32_t mode, float lr,
                             float mom, int32_t sync_interval, float* const* d_params, float* const* d_velocity,
                             void* const* d_params_shadow, void* agg_stream);
/* The same with one CUDA graph per worker (forward/backward + its local step, captured
 * in its own partition's context); d_iters[n] are per-worker device iteration counters
 * (zero them at the epoch start); capture_only = 1 captures without running. */
int dbs_run_iterations_local_graphed(const dbs_worker_slot* w, int32_t n, int64_t t0, int64_t t1, int32_t mode,
                                     float lr, float mom, int32_t sync_interval, float* const* d_params,
                                     float* const* d_velocity, void* const* d_params_shadow, void* agg_stream,
                                     int64_t* d_iters, dbs_worker_graphs* graphs, int32_t capture_only);
/* The same across GPUs (one process per GPU): after the local average of every
 * sync round, d_params[0] -- which must be the communicator's parameter block --
 * is averaged across ranks with rank weights = rank_batches[r] (the ranks' batch
 * sums) by the fused NVLink kernel and copied back into the other replicas. */
int dbs_run_iterations_local_comm(const dbs_worker_slot* workers, int32_t n, int64_t t0, int64_t t1, int32_t mode,
                                  float lr, float momentum, int32_t sync_interval, float* const* d_params,
                                  float* const* d_velocity, void* const* d_params_shadow, dbs_comm* comm,
                                  const int64_t* rank_batches, void* agg_stream);
/* x_bar = sum_i w_i x_i (w as in dbs_dev_aggregate_*), written to every replica
 * and its bf16 copy (d_params_bf16 may be NULL). P % 4 == 0. */
int dbs_dev_average_replicas_f32(float* const* d_params, const int64_t* b, int64_t n, int32_t mode, int64_t P,
                                 uint16_t* const* d_params_bf16, void* stream);
/* the same with the shadows in shadow_prec's format (d_shadows may be NULL) */
int dbs_dev_average_replicas_f32_ex(float* const* d_params, const int64_t* b, int64_t n, int32_t mode, int64_t P,
                                    void* const* d_shadows, int32_t shadow_prec, void* stream);
int dbs_mlp_run_iterations(const dbs_worker_slot* workers, int32_t n, int64_t t0, int64_t t1, int32_t mode,
                           float lr, float momentum, float* d_params, float* d_velocity, void* d_params_shadow,
                           int32_t skip_update, void* agg_stream);

/* ------------------------------------------------------------------------ */
/* Monte-Carlo checks of the theory (checks.py:42-142, sgdlab.py:241-314)    */
/* ------------------------------------------------------------------------ */
/* numpy Generator.integers(0, high, size=count) (int64, high <= 2^32) and
 * Generator.random(count) from a device PCG64 state, bit-exact, state advanced. */
int dbs_dev_pcg64_integers(dbs_pcg64* d_rng, int64_t high, int64_t count, int64_t* d_out, void* stream);
int dbs_dev_pcg64_random(dbs_pcg64* d_rng, int64_t count, double* d_out, void* stream);
/* check_theorem1_bound's vectorised single-sample SGD (checks.py:62-70): n_seeds
 * trajectories from x0 for n_iter steps with idx [n_iter][n_seeds]; dists
 * [(n_iter + 1)][n_seeds] (row 0 untouched), snapshots of X at the host-sorted
 * device iterations d_probe_at [n_probe] into d_snap [n_probe][n_seeds][dim]. */
int dbs_dev_theorem1_trajectories(const double* d_offsets, const double* d_opt, const double* d_x0, int64_t dim,
                                  const int64_t* d_idx, int64_t n_seeds, int64_t n_iter, double coef,
                                  const int32_t* d_probe_at, int32_t n_probe, double* d_X, double* d_dists,
                                  double* d_snap, void* stream);
/* per row of v[rows][ld] (n used): mean, sum (v - mean)^2, sum (v - mean)^4 into out[rows][3] */
int dbs_dev_row_moments(const double* d_v, int64_t rows, int64_t n, int64_t ld, double* d_out, void* stream);
/* ||batch-mean gradient||^2 per draw (estimate_gradient_noise); kind 0 ConvexProblem, 1 LogisticProblem */
int dbs_dev_minibatch_sqnorms(int32_t kind, const double* d_data, const double* d_labels, const double* d_opt,
                              int64_t dim, double mu, const double* d_x, const int64_t* d_idx, int64_t n_draws,
                              int64_t b, double* d_out, void* stream);
/* per-sample objective values f_i(x), i < n */
int dbs_dev_sample_values(int32_t kind, const double* d_data, const double* d_labels, const double* d_opt,
                          int64_t dim, double mu, const double* d_x, int64_t n, double* d_out, void* stream);
/* out[t] = mean_k v[idx[t][k]], k < m */
int dbs_dev_gather_means(const double* d_v, const int64_t* d_idx, int64_t n_draws, int64_t m, double* d_out,
                         void* stream);

/* ------------------------------------------------------------------------ */
/* Worker heterogeneity (cluster.py:25-79 DisturbanceEvent) and timing       */
/* ------------------------------------------------------------------------ */
/* Occupy `num_ctas` SMs (one resident CTA per SM, max shared memory) until
 * *d_stop becomes non-zero: the co-running disturbance of the paper's
 * robustness experiments.  Launch it on its own stream.  The resident CTAs hold
 * their SMs' registers and shared memory but sleep between polls (low power;
 * DBS_SPIN_SLEEP=0 selects an FMA-burning spin). */
int dbs_dev_spin_until(int32_t num_ctas, const volatile int32_t* d_stop, void* stream);
/* Occupy `num_ctas` SMs for `nanoseconds` (fixed extra work). */
int dbs_dev_spin_for(int32_t num_ctas, int64_t nanoseconds, void* stream);
/* Write the device %globaltimer (ns) into d_stamps[slot]. */
int dbs_dev_stamp(int64_t* d_stamps, int64_t slot, void* stream);
/* d_seconds[w] += (d_stamps[end] - d_stamps[begin]) * 1e-9 : per-worker
 * compute time accumulated on the device for the controller. */
/* *d_flag = value (0/1) with a memset on `stream`: stops dbs_dev_spin_until
 * without launching a kernel while the spin owns SMs. */
int dbs_dev_set_flag(int32_t* d_flag, int32_t value, void* stream);
int dbs_dev_accumulate_time(const int64_t* d_stamps, int64_t begin, int64_t end,
                            double* d_seconds, int64_t worker, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DBS_B200_H */

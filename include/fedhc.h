/*
 * fedhc.h -- C ABI of the B200-native FedHC round hot path (libfedhc.so).
 *
 * Drop-in boundary for the reference's Python FL-math and round API
 * (/root/reference/pkg/src/fedsim).  The reference
 * has no FFI of its own: its boundary is the Python function API of
 * fl_core.py and engine.py.  Each entry point below replaces one of those
 * functions (cited per function); the Python package
 * `paper_2305_15668_b200` binds them with ctypes (INTEGRATION.md shows the
 * binding a fedsim maintainer would add).
 *
 * Conventions
 *  - Plain pointers and sizes only.  "dev" pointers are CUDA device pointers
 *    of the current device; "host" pointers are CPU memory.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *  - Every function returns an int status (FEDHC_OK == 0).  On failure
 *    fedhc_last_error() returns a thread-local message; the Python layer maps
 *    the status to the reference's exception type with that message.
 *  - No entry point allocates device memory on the hot path: all buffers
 *    are caller-owned.  Kernels are asynchronous on `stream`.
 *  - Parameter layout is the reference's flat vector
 *    [W (n_features x n_classes, row-major) ; b (n_classes)]
 *    (fl_core.py:121-129), P = F*C + C.
 */
#ifndef FEDHC_H_
#define FEDHC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define FEDHC_OK 0
#define FEDHC_ERR_VALUE 1        /* -> ValueError (bad shapes / arguments)   */
#define FEDHC_ERR_AGGREGATION 2  /* -> AggregationError (errors.py:12-13)     */
#define FEDHC_ERR_CONFIG 3       /* -> ConfigError (errors.py:4-5)            */
#define FEDHC_ERR_CUDA 4         /* CUDA runtime / driver failure             */
#define FEDHC_ERR_UNSUPPORTED 5  /* shape outside the compiled kernels        */
#define FEDHC_ERR_RUNTIME 6      /* -> RuntimeError (engine.py:216, :224)     */

const char* fedhc_last_error(void);
int fedhc_version(void);
/* SM count / compute capability of `device` (host query, no kernel). */
int fedhc_device_info(int device, int* sm_count, int* cc_major, int* cc_minor);

/* ---- local training: fl_core.local_train (fl_core.py:163-194) ----------- */
/*
 * One descriptor per client.  The batch plan is the reference's: batch s of
 * the local epoch visits rows perm[e*n_rows + j*batch_size : ... + nb] with
 * bpe = ceil(n_rows / batch_size), e = s / bpe, j = s % bpe,
 * nb = min(batch_size, n_rows - j*batch_size)   (fl_core.py:180-189),
 * i.e. `perm` is the concatenation of the PCG64 permutations the reference
 * draws (one per started epoch).  Math: fp32 storage and SGD state; every
 * product on the bf16 tensor pipe as "bf16x3" (each fp32 operand split into
 * bf16 hi + mid, hi*hi + hi*mid + mid*hi accumulated in fp32: ~2^-16 relative
 * per product, within the north_star 1e-4 bar); delta = W_final - W_initial.
 * Kernels: tcgen05 F-split clusters (F > 784, or C > 32), mma.sync (C <= 32,
 * F <= 784), SIMT fallback (F % 4 != 0, C > 64, batch > 64).
 */
typedef struct fedhc_client {
  const float* x;        /* dev [n_rows, n_features] fp32 row-major          */
  const int32_t* y;      /* dev [n_rows] class ids in [0, n_classes)           */
  const int32_t* perm;   /* dev [n_epochs * n_rows] concatenated permutations  */
  int32_t n_rows;        /* shard length (0 -> zero delta, fl_core.py:178)     */
  int32_t n_batches;     /* ceil(num_samples / batch_size) (fl_core.py:180)    */
  int32_t batch_size;    /* >= 1                                               */
  float lr;              /* SGD step (fl_core.py:193)                          */
  float* delta;          /* dev [P] fp32 output                                */
} fedhc_client;

/* Batched local SGD for n_clients clients that all start from `params`
 * (dev fp64 [P], the round-start model, engine.py:336-347).  `clients` is a
 * DEVICE array of descriptors.  `max_batch` = max batch_size over clients. */
int fedhc_local_train(const fedhc_client* clients, int n_clients, const double* params,
                      int n_features, int n_classes, int max_batch, void* stream);

/* Rows re-encoded for the bf16x3 tensor-pipe trainers (setup, once per
 * federation): fp32 row i of x [n_rows, n_features] is split into bf16 "hi"
 * and "mid" words (hi = bf16_rn(x), mid = bf16_rn(x - hi),
 * |x - hi - mid| <= 2^-17 |x|) laid out per 8-feature unit u as
 * [8 hi | 8 mid] at byte 32 u -- the same 4F bytes per row, so `out` has x's
 * byte layout and any 8-aligned feature slice of a row is contiguous.
 * n_features a multiple of 8. */
int fedhc_x_split(const float* x, int64_t n_rows, int n_features, void* out, void* stream);

/* numpy Generator.standard_normal (float64) on the device, value-for-value: n normals from the PCG64 stream
 * whose state before the first draw is state_words = {state_hi, state_lo, inc_hi, inc_lo}
 * (rng.bit_generator.state["state"] of a numpy Generator).  Replaces the host draw of the reference's
 * synthetic features (fl_core.py:47-55) at fleet scale; out: device fp64 [n]; state_after (host, optional):
 * {state_hi, state_lo} after the draws numpy would have taken.  Synchronous on `stream`. */
int fedhc_pcg64_standard_normal(const uint64_t* state_words, int64_t n, double* out, uint64_t* state_after,
                                void* stream);

/* fedhc_local_train (fl_core.py:163-194) whose client rows ALSO exist in the
 * fedhc_x_split layout at (char*)client.x + split_offset (bytes, signed,
 * multiple of 16: the distance from the fp32 rows to their split copy).  Shapes with a split-reading kernel (F = 784, C <= 16: the FEMNIST
 * logistic round) read that copy -- identical products, fewer instructions
 * per fragment; every other shape reads client.x as fp32.  Results are
 * bit-identical to fedhc_local_train. */
int fedhc_local_train_split(const fedhc_client* clients, int n_clients, const double* params,
                            int n_features, int n_classes, int max_batch, int64_t split_offset, void* stream);

/* ---- native round planning (the serving loop's host work) ------------- */
/* CPython 3.12 random.Random.sample(range(n), k) on an MT19937 state laid out
 * as Random.getstate()[1] (624 words + index, updated in place); bit-exact
 * with the reference's selection (engine.py:302, :327). */
int fedhc_mt_sample(uint32_t* state, int n, int k, int32_t* out);
/* CPython >= 3.12 sum() of n floats (Neumaier compensation). */
double fedhc_py_float_sum(const double* x, int n);
/* One rank's round plan for k participants (fleet indices `mine`): per-client
 * seeds (stable_seed chain, fl_core.py:21-24, :181), and the pinned staging
 * block [PCG64 seeds u64[k] | rows i32[k] | permutations i32[k] | offsets
 * i64[k] | fedhc_client[k] | coef f64[k] = weight / total] that the runner
 * copies to the GPU in one transfer.  Per-fleet-client arrays are indexed by
 * fleet index; perm_base / delta_base are device addresses. */
int fedhc_round_pack(int64_t seed, int64_t round_index, int k, const int64_t* mine, const char* const* reprs,
                     const int32_t* rows, const int32_t* n_perms, const int32_t* n_batches,
                     const int32_t* batch_size, const uint64_t* xptr, const uint64_t* yptr, const double* weight,
                     double total, float lr, uint64_t perm_base, uint64_t delta_base, int64_t delta_stride,
                     uint8_t* staging, int64_t* perm_words, int32_t* max_rows);

/* Diagnostics: phase timestamps (%globaltimer ns, [8 CTAs][32 steps][24
 * points]) of cluster 0 from the last tcgen05 local_train launch made with
 * the environment variable FEDHC_TC_TRACE set; host `out`. */
int fedhc_tc_trace_read(unsigned long long* out);

/* ---- batch order: the PCG64 permutations local_train draws ------------- */
/* Native, multi-threaded restatement of `np.random.default_rng(seed)` +
 * repeated `.permutation(n)` (fl_core.py:181-187): SeedSequence -> PCG64
 * (XSL-RR 128/64) -> Fisher-Yates with random_interval, bit-exact with
 * numpy.  Client c writes n_perms[c] permutations of n_rows[c] (int32) at
 * out + offsets[c].  seeds[c] = stable_seed("local_train", seed) (fl_core.py:181).
 * n_threads <= 0 uses all hardware threads.  Host memory only. */
int fedhc_batch_permutations(const uint64_t* seeds, const int32_t* n_rows, const int32_t* n_perms,
                             const int64_t* offsets, int n_clients, int32_t* out, int n_threads);
/* Per-round client seeds (fl_core.py:21-24, engine.py:336-347, fl_core.py:181):
 * train_seeds[i] = stable_seed("train", seed, round_index, cid_i) and
 * rng_seeds[i] = stable_seed("local_train", train_seeds[i]), i.e. the first 4
 * bytes (little-endian) of sha256(repr(tuple)).  cid_reprs[i] = Python
 * repr(cid_i) (NUL-terminated UTF-8), so the hashed strings equal Python's. */
int fedhc_round_seeds(int64_t seed, int64_t round_index, const char* const* cid_reprs, int n,
                      uint64_t* train_seeds, uint64_t* rng_seeds);
uint32_t fedhc_sha256_le32(const char* data, int64_t n);
/* Same permutations generated on the GPU (device pointers; one CTA per
 * client; `max_rows` = max n_rows, for the shared-memory staging size). */
int fedhc_batch_permutations_device(const uint64_t* seeds, const int32_t* n_rows, const int32_t* n_perms,
                                    const int64_t* offsets, int n_clients, int32_t* out, int max_rows,
                                    void* stream);
/* PCG64 state after seeding (for tests against numpy's bit_generator.state). */
int fedhc_pcg64_state(uint64_t seed, uint64_t* state_hi, uint64_t* state_lo, uint64_t* inc_hi, uint64_t* inc_lo);

/* ---- loss_and_grad: fl_core.loss_and_grad (fl_core.py:138-151) ---------- */
/* fp64 throughout.  x dev fp64 [n, F]; y dev int32 [n]; params dev fp64 [P];
 * grad dev fp64 [P] out; loss dev fp64 [1] out (mean CE, +1e-300 guard);
 * workspace dev, >= n * n_classes * 8 bytes. */
int fedhc_loss_and_grad(const double* x, const int32_t* y, int n, int n_features, int n_classes,
                        const double* params, double* grad, double* loss, double* workspace,
                        void* stream);

/* ---- FedAvg: fl_core.fedavg (fl_core.py:197-218) ------------------------ */
/* Host helper: validates weights exactly like fl_core.py:201-209 and writes
 * coef[i] = w[i] / total with total the CPython>=3.12 float sum of w
 * (Neumaier-compensated, as `float(sum(weights))` evaluates for a list of
 * Python floats). */
int fedhc_fedavg_coefficients(const double* weights, int n, double* coef_out);

#define FEDHC_F32 0
#define FEDHC_F64 1
/* out[p] = base[p] + sum_k coef[k] * delta_k[p], accumulated in fp64 in k
 * order with separately rounded multiply and add -- bit-identical to the
 * reference's `out += (w/total) * d` loop for fp64 deltas.  Deltas are
 * either a DEVICE array of K device pointers (`deltas` != NULL) or one
 * packed dev buffer `packed` with row stride `ld` elements.  `base` may be
 * NULL (sum starts at +0.0; used for per-GPU partial sums).  coef is a dev
 * fp64 [K] array.  out may alias base. */
int fedhc_fedavg(const void* const* deltas, const void* packed, int64_t ld, int dtype,
                 const double* coef, int n_deltas, const double* base, double* out,
                 int64_t n, void* stream);

/* ---- evaluate_accuracy (fl_core.py:154-160) ----------------------------- */
/* x dev fp32 [n, F]; y dev int32 [n]; params dev fp64 [P].
 * *correct (dev uint64) += number of rows whose first-max argmax == label. */
int fedhc_eval(const float* x, const int32_t* y, int64_t n, int n_features, int n_classes,
               const double* params, unsigned long long* correct, void* stream);
/* Same, on at most max_ctas SMs (<= 0: all).  The round loop runs round r's
 * accuracy concurrently with round r+1's training (one CTA per client) and
 * caps it to the SMs the training leaves idle. */
int fedhc_eval_ctas(const float* x, const int32_t* y, int64_t n, int n_features, int n_classes,
                    const double* params, unsigned long long* correct, int max_ctas, void* stream);

/* ---- round DES: engine.run_round (engine.py:53-230) --------------------- */
/* Host-only discrete-event simulation of one round under capped max-min
 * sharing, with the reference's executor manager (executor_manager.py) and
 * schedulers (scheduler.py).  Bit-identical event times to the reference
 * (same fp64 operation order).  See fedhc_des_* below. */
typedef struct fedhc_des_client {
  int32_t budget;              /* resource_budget, [1,100] (profiles.py:60)       */
  int32_t num_samples;         /* WorkloadSpec fields (profiles.py:19-39)          */
  int32_t batch_size;
  int32_t model_layers;
  int32_t seq_len;
  double extra_model_factor;
  int32_t n_phases;            /* demand profile (profiles.py:42-54)               */
  const double* phase_frac;    /* host [n_phases] work fractions                   */
  const double* phase_demand;  /* host [n_phases] demands in (0,100]               */
} fedhc_des_client;

typedef struct fedhc_des_config { /* FleetConfig (profiles.py:76-93) */
  double theta;
  int32_t max_executors;
  int32_t scheduler;           /* 0 = resource-aware, 1 = greedy                  */
  int32_t dynamic_parallelism; /* bool                                            */
  double alpha, beta;          /* cost coefficients                               */
  double launch_latency, terminate_latency, upload_latency;
} fedhc_des_config;

/* Trace event kinds (metrics.py:21-28 plus Alloc / Instruction). */
#define FEDHC_EV_LAUNCHED 0
#define FEDHC_EV_PHASE 1
#define FEDHC_EV_TRAINED 2
#define FEDHC_EV_UPLOADED 3
#define FEDHC_EV_SLOT_FREED 4
#define FEDHC_EV_ROUND_COMPLETE 5
#define FEDHC_EV_ALLOC 6
#define FEDHC_EV_INSTRUCTION 7

typedef struct fedhc_des_event {
  double t;
  int32_t kind;       /* FEDHC_EV_*                                            */
  int32_t client;     /* participant index (order given), -1 if none           */
  int32_t executor;   /* -1 if none                                            */
  int32_t aux;        /* phase (PHASE), instruction 0..3 (INSTRUCTION), round   */
  double budget;      /* LAUNCHED / TRAINED / UPLOADED                          */
  int64_t alloc_off;  /* ALLOC: offset into alloc arrays                        */
  int32_t alloc_len;  /* ALLOC: number of (client, share) pairs                 */
  int32_t pad_;
} fedhc_des_event;

typedef struct fedhc_des_report { /* metrics.RoundReport (metrics.py:31-53) */
  double makespan, utilization, vacancy_area, throughput;
  int32_t degenerate;
  int32_t n_events;       /* trace length (if recorded)                       */
  int64_t n_alloc_pairs;  /* total alloc pairs (if recorded)                  */
} fedhc_des_report;

/* Opaque simulator handle (reusable across rounds; owns trace storage). */
typedef struct fedhc_des fedhc_des;
fedhc_des* fedhc_des_create(void);
void fedhc_des_destroy(fedhc_des* sim);
/* Simulate one round.  `order` = participant indices into `clients` in
 * arrival order; `client_ids` = their string ids (ties break on byte order,
 * engine.py:171).  Per-participant outputs (host arrays of length n_order):
 * start (ClientLaunched time), end (ModelUploaded time).  record_trace != 0
 * keeps the full event list, readable with fedhc_des_trace(). */
int fedhc_des_run_round(fedhc_des* sim, const fedhc_des_client* clients, const char* const* client_ids,
                        const int32_t* order, int n_order, const fedhc_des_config* cfg, double t0,
                        int round_index, int record_trace, double* start_out, double* end_out,
                        fedhc_des_report* report);
/* Borrow the recorded trace: events[n_events], alloc_client[n_alloc_pairs]
 * (participant indices) and alloc_share[n_alloc_pairs]; parallelism timeline
 * (time, count) pairs.  Valid until the next run on this handle. */
int fedhc_des_trace(const fedhc_des* sim, const fedhc_des_event** events, const int32_t** alloc_client,
                    const double** alloc_share, const double** par_t, const int32_t** par_n, int* n_par);

/* ---- native single-GPU round loop (FederatedRunner's serving loop) ------- */
/* Two GIL-free calls per round replace the Python planning / launch path:
 *   fedhc_runner_plan   selection (engine.py:327) -> DES (engine.py:53-230) -> seeds, descriptors,
 *                       coefficients and batch-order block into slot `slot`'s pinned block -> on the plan
 *                       stream: one H2D copy + the device PCG64 permutations (fl_core.py:181-187);
 *   fedhc_runner_launch wait for the plan -> local_train of all participants (fl_core.py:163-194) ->
 *                       sync FedAvg (fl_core.py:197-218, engine.py:350-353) on `stream` -> accuracy
 *                       (fl_core.py:154-160) on the eval stream, overlapping the next round's training;
 *   fedhc_runner_result waits for the slot's accuracy count.
 * Every pointer in the config is borrowed and must outlive the runner. */
typedef struct fedhc_runner fedhc_runner;
typedef struct fedhc_runner_config {
  /* per fleet client, indexed like the sorted client ids */
  const char* const* reprs;       /* repr(client_id), the stable_seed key                    */
  const int32_t* rows;            /* shard length                                            */
  const int32_t* n_perms;         /* permutations local_train draws                          */
  const int32_t* n_batches;       /* ceil(num_samples / batch_size)                          */
  const int32_t* batch_size;
  const uint64_t* xptr;           /* device address of the client's rows / labels            */
  const uint64_t* yptr;
  const double* weight;           /* float(num_samples) (engine.py:348)                      */
  const uint8_t* over_theta;      /* budget > theta: the round must take the raising path    */
  const int32_t* sim_index;       /* DES client index                                        */
  uint32_t* mt_state;             /* the selector's MT19937 state (625 words), updated       */
  fedhc_des* sim;                 /* DES handle, client table and ids (fedhc_des_*)          */
  const fedhc_des_client* des_clients;
  const char* const* des_ids;
  /* device side */
  double* params;                 /* dev fp64 [P], updated in place by FedAvg               */
  float* deltas;                  /* dev fp32 [participants, ld]                             */
  int64_t delta_stride_bytes;     /* 4 * ld                                                  */
  int64_t split_offset;           /* fedhc_local_train_split offset (split != 0)             */
  const float* x_test;
  const int32_t* y_test;
  int64_t n_test;
  unsigned long long* correct_dev;   /* dev [slots]                                          */
  unsigned long long* correct_host;  /* pinned host [slots]                                  */
  uint8_t* const* stage_host;     /* [slots] pinned blocks, participants * (24 + 48 + 8) B   */
  uint8_t* const* stage_dev;      /* [slots] device copies                                   */
  int32_t* const* plan_dev;       /* [slots] device permutation buffers                      */
  int64_t plan_cap_words;
  void* plan_stream;
  void* eval_stream;
  int64_t seed;
  /* async aggregation (engine.py:354-364; async_buffer = 0: sync FedAvg).  Per slot: pinned [participants]
   * x (chunk coefficient f64 | delta row address u64) blocks staged after the main block, device copies,
   * params snapshots [participants][P] f64 (the accuracy of each chunk reads its own snapshot). */
  uint8_t* const* async_host;
  uint8_t* const* async_dev;
  double* const* snapshots;
  fedhc_des_config des_cfg;
  float lr;
  int32_t n_fleet, participants, slots, n_features, n_classes, max_batch, split, eval_ctas, rows_max;
  int32_t async_buffer;
} fedhc_runner_config;

typedef struct fedhc_runner_plan_info {
  /* caller-provided host arrays */
  int32_t* selected;              /* [participants] fleet indices, selection order           */
  double* starts;                 /* [participants] DES launch / upload times                 */
  double* ends;
  int32_t* launch_order;          /* [participants] participant indices in event order       */
  int32_t* upload_order;
  double* par_t;                  /* [par_cap] parallelism timeline                          */
  int32_t* par_n;
  double* chunk_end;              /* [participants] async: end time of each chunk's last client */
  int32_t par_cap;
  /* outputs */
  int32_t n_launched, n_uploaded, n_par, over_theta, degenerate, max_rows, n_chunks;
  double makespan, utilization, vacancy_area, throughput, total_weight;
  int64_t perm_words, h2d_bytes;
} fedhc_runner_plan_info;

int fedhc_runner_create(const fedhc_runner_config* cfg, fedhc_runner** out);
void fedhc_runner_destroy(fedhc_runner* runner);
int fedhc_runner_plan(fedhc_runner* runner, int64_t round_index, double t0, int slot, fedhc_runner_plan_info* info);
int fedhc_runner_launch(fedhc_runner* runner, int slot, void* stream);
/* correct[n_chunks] (1 for sync FedAvg): the accuracy counts of the slot's round. */
int fedhc_runner_result(fedhc_runner* runner, int slot, int64_t* correct);

/* ---- tcgen05 grouped GEMM (client-model contractions) -------------------- */
/* D_g[M x N] (fp32) = A_g[M x K] (bf16, row-major) . B_g[N x K]^T (bf16,
 * row-major) for g in [0, G): one launch for all clients of a round.
 * TMA (128B swizzle) -> tcgen05.mma (M=128, N=128|256, K=16) -> TMEM -> tcgen05.ld.
 * Requires M % 128 == 0, N % 128 == 0, K % 64 == 0, 16-byte aligned operands.
 * A, B: dev [G][M][K], [G][N][K]; D: dev [G][M][N]. */
int fedhc_gemm_bf16_tn(int G, int M, int N, int K, const void* A, const void* B, float* D, void* stream);

/* General form.  Operand storage (per group, bf16, row-major):
 *   a_mn = 0: A[M][K] (K-major)      a_mn = 1: A[K][M] (MN-major, e.g. W^T of dgrad)
 *   b_mn = 0: B[N][K]                 b_mn = 1: B[K][N]
 * Epilogue on acc = A.B^T (fp32), element (g, m, n) at offset g*d_gstride + m*ldd + n:
 *   FEDHC_EPI_F32            float D
 *   FEDHC_EPI_BF16           bf16 D
 *   FEDHC_EPI_BIAS_RELU_BF16 bf16 D = relu(acc + bias), bias[g*bias_gstride + (m or n)]
 *   FEDHC_EPI_SGD            float master -= lr * acc; bf16 shadow = master (if shadow != NULL)
 *   FEDHC_EPI_RELU_MASK_BF16 bf16 D = acc * (mask > 0), bf16 mask indexed like D (ReLU backward);
 *                            optional rowsum[g*M + m] = sum over n of the stored D (N <= 256)
 * Requires M % 64 == 0, N % 32 == 0 (N % 64 == 0 when b_mn), K % 64 == 0,
 * 16-byte aligned operands, ldd % 8 == 0 (ldd <= 0 -> N; d_gstride <= 0 -> M*ldd). */
#define FEDHC_EPI_F32 0
#define FEDHC_EPI_BF16 1
#define FEDHC_EPI_BIAS_RELU_BF16 2
#define FEDHC_EPI_SGD 3
#define FEDHC_EPI_RELU_MASK_BF16 4
typedef struct fedhc_gemm_args {
  int32_t G, M, N, K;
  int32_t a_mn, b_mn;
  const void* A;
  const void* B;
  int32_t epilogue;
  int32_t bias_per_row;
  void* D;
  int64_t ldd;
  int64_t d_gstride;
  const float* bias;
  int64_t bias_gstride;
  float* master;
  void* shadow;
  float lr;
  int32_t pad_;
  const void* mask;
  float* rowsum;
  int64_t a_gstride; /* elements between groups of A (0 = dense) */
  int64_t b_gstride; /* elements between groups of B (0 = dense) */
  int64_t lda;       /* elements between rows of A as stored (0 = dense: K, or M when a_mn) */
  int64_t ldb;       /* elements between rows of B as stored (0 = dense) */
} fedhc_gemm_args;
int fedhc_gemm(const fedhc_gemm_args* args, void* stream);

/* ---- green-context SM partitions (executor slots) ------------------------- */
/* Split the device's SMs into equal groups of >= min_sms (8 on sm_90+) and
 * hand out streams whose kernels run only on a contiguous group window; the
 * B200 replacement for per-process MPS percentages.  Contexts/streams are
 * created on first use of a window and cached. */
typedef struct fedhc_gctx_pool fedhc_gctx_pool;
int fedhc_gctx_pool_create(int device, int min_sms, fedhc_gctx_pool** out, int* n_groups, int* sms_per_group);
void fedhc_gctx_pool_destroy(fedhc_gctx_pool* pool);
int fedhc_gctx_stream(fedhc_gctx_pool* pool, int first_group, int n_groups, void** stream, int* sm_count);
/* As fedhc_gctx_stream, plus the SMs the split left outside every group (n_groups may be 0): side work
 * (the round loop's batch order / accuracy) that must stay off the SMs a round's training claims. */
int fedhc_gctx_stream_rest(fedhc_gctx_pool* pool, int first_group, int n_groups, void** stream, int* sm_count);
/* Diagnostic: `blocks` CTAs on `stream` each write their %smid to out_dev[i]. */
int fedhc_probe_smid(void* stream, int blocks, int* out_dev);

/* Standalone cost-model helpers (cost_model.py:33-87), for the API layer. */
double fedhc_work_units(int num_samples, int batch_size, int model_layers, int seq_len,
                        double extra_model_factor, double alpha, double beta);
int fedhc_maxmin_allocate(const double* caps, const double* demands, int n, double capacity,
                          double* alloc_out);


/* ---- FEMNIST CNN client engine (BASELINE config 2) --------
 * Builder-defined model (the reference ships only the linear model):
 * conv5x5 1->32 +ReLU +pool2, conv5x5 32->64 +ReLU +pool2, fc 3136->2048 +ReLU,
 * fc 2048->C; softmax-CE, plain SGD; the local loop of fl_core.local_train
 * (fl_core.py:163-194).  Parameters live in a padded fp64/fp32 layout of
 * fedhc_cnn_param_count() elements; fedhc_cnn_param_offsets() gives the 8
 * block offsets (Wc1 [64 taps][32], bc1, Wc2 [896][64], bc2, W1 [2048][3200],
 * b1, W2 [64][2048], b2); padding entries stay exactly zero.
 * Input rows are 784 fp32 (28x28x1), labels int32. */
int fedhc_cnn_param_count(int64_t* padded);
int fedhc_cnn_param_offsets(int64_t* offsets /* [8] */);
/* Workspace for up to max_clients clients at batch <= 256 (rounded up to 64). */
int fedhc_cnn_create(int max_clients, int batch, int n_classes, void** ws);
int fedhc_cnn_destroy(void* ws);
/* Local SGD of n_clients clients from `params` (dev fp64, padded layout);
 * clients = dev fedhc_client array (as fedhc_local_train; delta -> [P] fp32
 * padded layout; lr taken from `lr`).  max_steps = max n_batches.  With
 * use_graph the step sequence is captured once per (n_clients, max_steps, lr)
 * and replayed. */
int fedhc_cnn_local_train(void* ws, const fedhc_client* clients, int n_clients, const double* params,
                          int max_steps, float lr, int use_graph, void* stream);
/* Mean CE loss of each client's last step (dev fp32 [n_clients]). */
int fedhc_cnn_last_loss(void* ws, float* out, int n_clients, void* stream);
/* *correct (dev u64) += test rows whose first-max argmax == label. */
int fedhc_cnn_eval(void* ws, const double* params, const float* x, const int32_t* y, int64_t n,
                   unsigned long long* correct, void* stream);
/* conv2 of the engine as one implicit GEMM on caller tensors (tests / tooling): mode 1 forward
 * (out = relu(conv(p1x, w) + bias)), 2 data gradient (out = dL/dp1 from act = dL/da2), 3 weight
 * gradient + SGD (out = fp32 master [G][1024][64] -= lr * grad; act = p1x, act2 = dL/da2).
 * NHWC bf16 activations [G*bp][14][14][C]; w bf16 [G][1024][64] tap-pair layout. */
int fedhc_cnn_conv2(int mode, int G, int bp, const void* act, const void* act2, const void* w, const float* bias,
                    void* out, float lr, void* stream);

/* ---- ResNet client models (config 3, builder-defined) ---------------------- */
/* One k x k (1 or 3) 'same' convolution layer of G clients x bp images as an implicit tcgen05 GEMM
 * over 4-D TMA boxes; NHWC bf16 maps, channels multiple of 64, output width <= 32.
 * mode 4 forward: out = conv(x, w) (bf16 [G*bp][H/s][W/s][cout]); mode 5 data gradient (s = 1):
 * out = conv^T(dy, w) (bf16 [G*bp][H][W][cin]); mode 6 weight gradient + SGD: out = fp32 master
 * [G][k*k*cin][cout] -= lr * grad (bf16 shadow updated when non-NULL).  w bf16 [G][k*k*cin][cout]. */
int fedhc_nhwc_conv(int mode, int G, int bp, int H, int W, int cin, int cout, int k, int s, const void* x,
                    const void* dy, const void* w, void* out, void* shadow, float lr, void* stream);
/* CIFAR ResNet-18 client engine (same conventions as the CNN engine): padded parameter layout
 * (fedhc_resnet_param_count / _offsets: torch state_dict order without num_batches_tracked), a workspace
 * for max_clients x batch images (batch multiple of 8, <= 64), local SGD of n_clients clients from
 * `params` (rows = NHWC fp32 [32][32][3]; batch norm in training mode, running statistics updated and
 * part of the delta), and accuracy with running statistics. */
int fedhc_resnet_param_count(int n_classes, int64_t* padded);
int fedhc_resnet_param_offsets(int n_classes, int64_t* offsets, int cap, int* count);
int fedhc_resnet_create(int max_clients, int batch, int n_classes, void** ws);
int fedhc_resnet_destroy(void* ws);
int fedhc_resnet_local_train(void* ws, const fedhc_client* clients, int n_clients, const double* params,
                             int max_steps, float lr, int use_graph, void* stream);
int fedhc_resnet_last_loss(void* ws, float* out, int n_clients, void* stream);
/* kernels launched by the workspace so far (graph kernel nodes + direct launches; eager steps excluded) */
int fedhc_resnet_launch_count(void* ws, int64_t* out);
int fedhc_resnet_eval(void* ws, const double* params, const float* x, const int32_t* y, int64_t n,
                      unsigned long long* correct, void* stream);
/* CIFAR MobileNetV2 client engine (BASELINE config 4), same conventions as the ResNet engine: 3x3 stem,
 * 17 inverted-residual blocks (1x1 expand, 3x3 depthwise, 1x1 linear projection; identity / 1x1 shortcut
 * at stride 1), 1x1 head to 1280, average pool, linear.  Channels padded to multiples of 64 in the
 * parameter vector (padding entries zero); batch multiple of 8, <= 32. */
/* depthwise 3x3 (pad 1) modes of the MobileNetV2 engine: 0 forward, 1 data gradient, 2 weight gradient +
 * SGD (out = fp32 master [G][9][C]); NHWC bf16 activations, w bf16 [G][9][C], C multiple of 64. */
int fedhc_dw_conv(int mode, int G, int bp, int H, int C, int s, const void* x, const void* dy, const void* w,
                  void* out, void* shadow, float lr, void* stream);
int fedhc_mobilenet_param_count(int n_classes, int64_t* padded);
int fedhc_mobilenet_param_offsets(int n_classes, int64_t* offsets, int cap, int* count);
int fedhc_mobilenet_create(int max_clients, int batch, int n_classes, void** ws);
int fedhc_mobilenet_destroy(void* ws);
/* steps (host, optional): per-client local step counts, non-increasing, <= max_steps; step s runs only
 * the clients with steps[i] > s (one CUDA graph per active-client count).  NULL: all run max_steps. */
int fedhc_mobilenet_local_train(void* ws, const fedhc_client* clients, int n_clients, const int32_t* steps,
                                const double* params, int max_steps, float lr, int use_graph, void* stream);
int fedhc_mobilenet_last_loss(void* ws, float* out, int n_clients, void* stream);
/* kernels launched by the workspace so far (graph kernel nodes + direct launches; eager steps excluded) */
int fedhc_mobilenet_launch_count(void* ws, int64_t* out);
int fedhc_mobilenet_eval(void* ws, const double* params, const float* x, const int32_t* y, int64_t n,
                         unsigned long long* correct, void* stream);
/* CIFAR ShuffleNetV2 x1.0 client engine (BASELINE config 4's other model), same conventions as MobileNetV2:
 * activations in "split form" ([X1 | X2] halves of each block output, padded to multiples of 64). */
int fedhc_shufflenet_param_count(int n_classes, int64_t* padded);
int fedhc_shufflenet_param_offsets(int n_classes, int64_t* offsets, int cap, int* count);
int fedhc_shufflenet_create(int max_clients, int batch, int n_classes, void** ws);
int fedhc_shufflenet_destroy(void* ws);
int fedhc_shufflenet_local_train(void* ws, const fedhc_client* clients, int n_clients, const int32_t* steps,
                                 const double* params, int max_steps, float lr, int use_graph, void* stream);
int fedhc_shufflenet_last_loss(void* ws, float* out, int n_clients, void* stream);
int fedhc_shufflenet_launch_count(void* ws, int64_t* out);
int fedhc_shufflenet_eval(void* ws, const double* params, const float* x, const int32_t* y, int64_t n,
                          unsigned long long* correct, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FEDHC_H_ */

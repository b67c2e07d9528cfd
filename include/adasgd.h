/*
 * adasgd.h -- C-ABI of the B200-native Adaptive SGD hot path
 * (Ma, Rusu, Wu, Sim, "Adaptive Elastic Training for Sparse Deep Learning on
 * Heterogeneous Multi-GPU Servers", arXiv 2110.07029).
 *
 * Citations "P:N" refer to line N of the paper text; readings
 * "Rk" are the interpretations listed in DESIGN.md section 3.
 *
 * One as_ctx = one model replica = one GPU = one process (section 2.2
 * "allocate a separate model replica to every GPU"; "GPU managers").
 * Every pointer in this header is a plain host or device pointer; no torch
 * types cross the boundary.  Unless a function says otherwise:
 *   - host arrays are owned by the caller and are copied (through pinned
 *     staging) or consumed before the call returns;
 *   - device work is enqueued on the ctx stream (as_config.stream) and the call
 *     returns without waiting;
 *   - the return value is AS_OK or a negative AS_E_* code, and
 *     as_last_error() gives a thread-local message for the last failure;
 *   - AS_E_INVALID leaves the ctx unchanged; AS_E_CUDA / AS_E_NCCL are sticky:
 *     every later call on that ctx returns AS_E_STATE.
 *
 * Packed parameter vector (R2): fp32, P = d*h + h + C*h + C floats,
 *     [ W1 (d x h, row-major) | b1 (h) | W2T (C x h, row-major, label-major) | b2 (C) ]
 * "model dimensionality" |w| of Alg. 2 line 7 is P.
 */
#ifndef ADASGD_H
#define ADASGD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
enum {
  AS_OK = 0,
  AS_E_INVALID = -1, /* argument / input validation failed; no state change   */
  AS_E_CUDA = -2,    /* a CUDA call or kernel failed (sticky)                  */
  AS_E_NCCL = -3,    /* an NCCL call failed (sticky)                           */
  AS_E_OOM = -4,     /* workspace too small / host allocation failed           */
  AS_E_STATE = -5    /* ctx poisoned by an earlier sticky error, or wrong order */
};

/* ---- arithmetic of the output layer (steps a5/a6) -------------------------
 * AS_FP32: SIMT fp32 everywhere (parity mode, |rel err| <= 1e-4 vs oracle).
 * AS_BF16: tcgen05 tensor cores, bf16 operands (H, W2T shadow, softmax grad),
 *          fp32 accumulation in TMEM, fp32 master weights (parity 2e-2).   */
enum { AS_FP32 = 0, AS_BF16 = 1 };

/* ---- flags --------------------------------------------------------------- */
enum {
  AS_FLAG_DEBUG_GRADS = 1, /* keep every gradient of the last step in device
                              memory for as_debug_get (tests only)            */
  AS_FLAG_NORM_UB = 2,     /* as_merge (AS_ALGO_ADAPTIVE): Alg. 2 line 5 uses
                              u_i b_i / sum(u b) instead of u_i / sum(u), the
                              alternative of P:175                             */
  /* bits 2-3: the regularisation metric of Alg. 2 line 7 tested against
     pert_thr (reading R15; "||w_i||_2/|w|", "L2-norm divided by
     model dimensionality", in tension with P:276): flags |= metric << 2    */
  AS_NORM_METRIC_SHIFT = 2,
  AS_FLAG_R14_LITERAL = 16 /* as_merge (AS_ALGO_ADAPTIVE): Alg. 2 line 8 read
                              literally (reading R14 "literal"): r = argmax_i u_i,
                              s = argmin_i u_i, lowest id on ties, applied even
                              when r = s (then alpha_r *= (1 + delta)(1 - delta));
                              default: lexicographic (u_i, b_i), skipped when
                              every (u_i, b_i) is equal                        */
};
enum {
  AS_METRIC_L2_P = 0,       /* ||w||_2 / P   (literal, default)                 */
  AS_METRIC_L2SQ_P = 1,     /* ||w||_2^2 / P                                    */
  AS_METRIC_L2_SQRTP = 2,   /* ||w||_2 / sqrt(P)  (RMS of the parameters)       */
  AS_METRIC_L2 = 3          /* ||w||_2                                          */
};

/* Alg. 2 line-5 normalisation (as_sched_alg2_ex), optionally OR-ed with
 * AS_NORM_R14_LITERAL (line 8 as printed, see AS_FLAG_R14_LITERAL). */
enum { AS_NORM_UPDATES = 0, AS_NORM_UB = 1, AS_NORM_R14_LITERAL = 2 };

typedef struct as_ctx as_ctx; /* opaque */

typedef struct {
  int64_t n_features;     /* d  (Table 1 "features")                  */
  int64_t n_labels;       /* C  ("classes")                                     */
  int32_t hidden;         /* h  hidden width, 128 or 256 (R1)                    */
  int32_t b_max;          /* largest batch (P:201 memory provisioned for it)    */
  int32_t b_min;          /* b_max / 8                                   */
  int32_t beta;           /* b_min / 2                                   */
  int64_t megabatch;      /* M samples between merges (R7: 100*b_max)    */
  int32_t max_row_nnz;    /* capacity: largest nnz of one sample                 */
  int32_t max_row_labels; /* capacity: largest label count of one sample        */
  double lr0;             /* learning rate at b_max                     */
  double gamma;           /* momentum, 0.9                              */
  double delta;           /* perturbation factor, 0.1                   */
  double pert_thr;        /* perturbation threshold, 0.1                */
  int32_t precision;      /* AS_FP32 | AS_BF16                                  */
  int32_t flags;          /* AS_FLAG_*                                          */
  int32_t rank;           /* replica id i, 0 <= rank < world                    */
  int32_t world;          /* number of replicas N                               */
  const void *nccl_unique_id; /* 128-byte ncclUniqueId from as_nccl_unique_id()
                                 on rank 0, broadcast by the caller; NULL when
                                 world == 1 or in local-group mode             */
  void *workspace;        /* device arena, >= as_workspace_size() bytes, 256-B
                             aligned; owned by the caller, alive until destroy */
  size_t workspace_bytes;
  void *stream;           /* cudaStream_t borrowed from the caller             */
  int32_t device;         /* CUDA device ordinal of this replica               */
  int32_t algo;           /* AS_ALGO_* merge rule (0 = the paper's Adaptive SGD) */
  int32_t merge_backend;  /* AS_MERGE_* transport of steps a11-a13 when world > 1 */
} as_config;

/* Largest number of replicas (world) one merge handles. */
enum { AS_MAX_WORLD = 64 };

/* Merge transports (as_config.merge_backend), world > 1 (P:197-199 all-reduce
 * model merging; the paper's own is a multi-stream ring over PCIe/NVLink):
 * AS_MERGE_NCCL  prescale fused into an NCCL PreMulSum all-reduce (weights read
 *                from device memory), partitioned into chunks on a
 *                communication stream, momentum chasing the chunks; needs
 *                nccl_unique_id.
 * AS_MERGE_P2P   ONE fused kernel over peer memory (CUDA IPC mappings over
 *                NVLink / NVSwitch): rank r reduces its 1/N slice of the
 *                packed vector from every replica (sum alpha_i w_i), applies
 *                the momentum step and pushes w' into every rank's replica,
 *                global model and bf16 shadow; cross-rank barriers are flags in
 *                peer memory.  Needs as_p2p_export / as_p2p_open after as_init.
 * Both compute the merge weights on the device (Alg. 2 from the all-gathered
 * norms), so as_merge does not synchronise the host unless alpha_out /
 * perturbed_out is requested. */
enum { AS_MERGE_NCCL = 0, AS_MERGE_P2P = 1 };

/* Merge rules (as_config.algo).  AS_ALGO_ADAPTIVE: Alg. 2 normalized,
 * perturbed weights.  The comparison methods of P:215-217 use
 * alpha_i = 1/N with no perturbation and no norm computation:
 * AS_ALGO_ELASTIC  elastic model averaging / K-step averaging (Fig. 3),
 *                  statically partitioned equal batches (as_sched_route_static)
 * AS_ALGO_SYNC     gradient aggregation / synchronous SGD (Fig. 2):
 *                  the same average after one batch per replica (mega-batch
 *                  = N batches), which equals the averaged-gradient step.
 * gamma is applied as configured in every mode (the caller sets 0 for plain
 * averaging).  Routing and Alg. 1 are host-side choices of the caller. */
enum { AS_ALGO_ADAPTIVE = 0, AS_ALGO_ELASTIC = 1, AS_ALGO_SYNC = 2 };

/* Bytes of device workspace the ctx needs for cfg (validates cfg). */
int as_workspace_size(const as_config *cfg, size_t *bytes);

/* Write a fresh 128-byte NCCL unique id into out (rank 0 only). */
int as_nccl_unique_id(void *out128);

/* Create the replica.  init_params: HOST pointer to the packed fp32 vector
 * (P floats), identical on every rank ("All the algorithms are initialized
 * with the same model").  Sets w_i = wbar = wbar_p = init (R17),
 * b_i = b_max, lr_i = lr0.  When world > 1 and nccl_unique_id is
 * non-NULL this is collective (ncclCommInitRank).  Blocks until done. */
int as_init(const as_config *cfg, const float *init_params, as_ctx **out);

int as_destroy(as_ctx *ctx);
const char *as_last_error(void);

/* ---- batches (step a2) ------------------------------------------------------
 * Load the next training batch of `rows` samples from HOST CSR arrays
 * ("moving the training batch ... to the GPU"; P:217 libSVM sparse):
 *   row_ptr[rows+1] int64 (row_ptr[0] may be non-zero: the batch is rebased),
 *   col[nnz] int32 feature ids, strictly increasing inside a row, in [0, d);
 *   val[nnz] float32;  lab_ptr[rows+1] int64;  lab[L] int32 label ids,
 *   strictly increasing inside a row, in [0, C), at least one per row (R3).
 * Validation failures (rows not in [1, b_i] with b_i this rank's batch size,
 * non-monotone pointers, ids out of range, unsorted/duplicate ids, a row with
 * zero labels, capacity exceeded) return AS_E_INVALID with no state change. */
int as_load_batch_csr(as_ctx *ctx, int32_t rows, const int64_t *row_ptr,
                      const int32_t *col, const float *val,
                      const int64_t *lab_ptr, const int32_t *lab);

/* Device-resident dataset: bytes of device memory needed for n samples with
 * nnz features and L labels in total. */
int as_dataset_bytes(int64_t n, int64_t nnz, int64_t L, size_t *bytes);

/* Upload a whole dataset (HOST CSR arrays as above, n samples) into the
 * caller-owned DEVICE buffer dev_buf (>= as_dataset_bytes).  order[n] (host,
 * nullable = identity) fixes the stream order (R10): stream position p maps
 * to sample order[p mod n].  Validates every row.  Blocks until copied. */
int as_dataset_upload(as_ctx *ctx, void *dev_buf, size_t dev_bytes, int64_t n,
                      const int64_t *row_ptr, const int32_t *col,
                      const float *val, const int64_t *lab_ptr,
                      const int32_t *lab, const int64_t *order);

/* Load the batch = stream positions [pos, pos+rows) of the resident dataset,
 * built on the device (gather + rebase).  rows in [1, b_i]. */
int as_load_batch_stream(as_ctx *ctx, int64_t pos, int32_t rows);

/* ---- one SGD step on this replica (steps a3-a8) ------------------------------
 * On the last loaded batch, with this rank's lr_i: batch transposes (a3),
 * SpMM forward (a4), output layer forward + softmax cross-entropy (a5),
 * backward (a5/a6/a7) and the SGD update of W1, b1, W2T, b2 ("SGD
 * requires three passes").  loss_out (nullable): mean loss over the rows of
 * the batch (R3); non-NULL forces a stream synchronisation. */
int as_train_step(as_ctx *ctx, float *loss_out);

/* ---- top-1 evaluation -----------------------------------------
 * P:228 "We measure the top-1 accuracy – corresponding to the class with the
 * highest probability – on the testing dataset after processing every
 * megabatch."  Forward pass of `rows` HOST CSR samples (same layout, validation
 * and ownership as as_load_batch_csr; rows in [1, b_max]) through this
 * replica's current model (right after as_merge that is the global model,
 * P:187): H = ReLU(X W1 + b1), z = H W2T^T + b2, top1_r = argmax_c z_rc with
 * the lowest class id on ties (R21; softmax is monotone).  AS_BF16: z from the
 * bf16 H and W2T shadow on the tensor cores (fp32 accumulate); AS_FP32: fp32
 * SIMT logits.  Outputs (host, nullable): top1_out[rows] (int32 class ids),
 * hits_out = number of rows whose top-1 class is one of their labels.
 * Overwrites the loaded training batch (call as_load_batch_* again before
 * as_train_step).  Synchronises the stream. */
int as_eval_top1(as_ctx *ctx, int32_t rows, const int64_t *row_ptr,
                 const int32_t *col, const float *val,
                 const int64_t *lab_ptr, const int32_t *lab,
                 int32_t *top1_out, int64_t *hits_out);

/* ---- merge (steps a9-a13, Alg. 2) ------------------------------------
 * Collective over all `world` ranks, called with identical u[world] (updates
 * since the last merge) and b[world] (batch sizes in force during the
 * mega-batch, R12).  Computes n_i = ||w_i||_2 / P (a9), all-gathers the norms,
 * alpha (a10, R13-R16, identical on every rank), prescales w_i by alpha_i
 * (a11), all-reduces (a12, NCCL over NVLink) and applies the momentum update
 * w' = sum alpha_i w_i + gamma (wbar - wbar_p); wbar_p <- wbar; wbar <- w';
 * w_i <- w' (a13, P:187 replicas restart from the global model).
 * alpha_out[world] and perturbed_out are nullable; non-NULL synchronises. */
int as_merge(as_ctx *ctx, const int32_t *u, const int32_t *b,
             double *alpha_out, int32_t *perturbed_out);

/* Replica norm (step a9, Alg. 2 line 7, "||w_i||_2 / |w|", reading R15):
 * the regularisation metric of this replica's packed parameters, computed on
 * the device in fp64 with a fixed reduction order; metric = AS_METRIC_*.
 * *out (host) receives the value.  Synchronises the stream. */
int as_replica_norm(as_ctx *ctx, int32_t metric, double *out);

/* Merge with caller-given weights alpha[world] (host, identical on every rank):
 * steps a11-a13 exactly as in as_merge, with Alg. 2 (a9-a10) replaced by the
 * given weights -- w' = sum_i alpha_i w_i + gamma (wbar - wbar_p).  Used by
 * drivers that compute the weights themselves and by the tests that force
 * alpha_i != 1 at world = 1 (prescale path).  Collective when world > 1. */
int as_merge_weighted(as_ctx *ctx, const double *alpha);

/* AS_MERGE_P2P setup (collective, world > 1, after as_init on every rank).
 * as_p2p_export writes this rank's export record (AS_P2P_EXPORT_BYTES: a CUDA
 * IPC handle of the workspace allocation and the workspace offset in it) to
 * out (host).  The caller all-gathers the records of all ranks (rank order) and
 * passes them to as_p2p_open, which maps every peer's workspace (cudaIpc,
 * NVLink / NVSwitch peer access).  Ranks may share a device (testing). */
enum { AS_P2P_EXPORT_BYTES = 128 };
int as_p2p_export(as_ctx *ctx, void *out);
int as_p2p_open(as_ctx *ctx, const void *records /* world * AS_P2P_EXPORT_BYTES */);

/* Local-group merge: the n contexts ctxs[0..n-1] live in THIS process (one per
 * device, or several on one device for testing), were created with
 * world == n, rank == index and nccl_unique_id == NULL.  Same semantics as
 * as_merge, the reduction reads every replica directly (same-device or peer
 * pointers).  Blocks until done. */
int as_group_merge(as_ctx *const *ctxs, int32_t n, const int32_t *u,
                   const int32_t *b, double *alpha_out, int32_t *perturbed_out);

/* Set the batch sizes of all ranks (b[world], used by the next merge's
 * Alg. 2 line 3) and this rank's learning rate lr[rank] (Alg. 1 output).
 * b[i] must lie in [b_min, b_max]. */
int as_set_batch_sizes(as_ctx *ctx, const int32_t *b, const float *lr);

/* ---- inspection (tests) -------------------------------------------------------- */
enum { AS_PARAMS_REPLICA = 0, AS_PARAMS_GLOBAL = 1, AS_PARAMS_GLOBAL_PREV = 2 };
/* Copy P floats of the chosen parameter vector to host_out (synchronises). */
int as_get_params(as_ctx *ctx, int32_t which, float *host_out);
/* Overwrite the replica parameters from a host vector (tests; synchronises). */
int as_set_params(as_ctx *ctx, int32_t which, const float *host_in);

enum {
  AS_DBG_H = 0,     /* float [rows*h]   ReLU(X W1 + b1) of the last step      */
  AS_DBG_LSE = 1,   /* float [rows]     log-sum-exp of the logits (natural)   */
  AS_DBG_LOSS = 2,  /* float [rows]     per-row loss (R3)                     */
  AS_DBG_DA = 3,    /* float [rows*h]   dL/dA1                                */
  AS_DBG_DB1 = 4,   /* float [h]                                              */
  AS_DBG_DW2T = 5,  /* float [C*h]      needs AS_FLAG_DEBUG_GRADS             */
  AS_DBG_DB2 = 6,   /* float [C]        needs AS_FLAG_DEBUG_GRADS             */
  AS_DBG_DW1 = 7,   /* float [U*h]      rows of the unique features, ascending;
                       needs AS_FLAG_DEBUG_GRADS                              */
  AS_DBG_FSEG = 8,  /* int32 [1+U+(U+1)+nnz+nnz]: U, feature ids, seg ptr,
                       csc rows, csc vals (float bits) -- step a3           */
  AS_DBG_LSEG = 9,  /* int32 [1+V+(V+1)+L]: V, label ids, seg ptr, rows      */
  AS_DBG_BATCH = 10,/* int32 [4]: rows, nnz, L, U of the loaded batch        */
  AS_DBG_LOGITS = 11,/* float [rows*C] logits (AS_FP32 only)                 */
  AS_DBG_DHSOFT = 12 /* float [rows*h]   softmax part of dL/dH before the label
                       term (R3): (1/B) sum_c softmax(z_r)_c W2T[c] -- pass 1's
                       O / l in AS_BF16; needs AS_FLAG_DEBUG_GRADS            */
};
/* Copy a debug view of the last step to host_out (capacity `bytes`);
 * *written receives the byte count.  Synchronises. */
int as_debug_get(as_ctx *ctx, int32_t which, void *host_out, size_t bytes,
                 size_t *written);

/* ---- live profiling (bench) ------------------------------------------------
 * When enabled, the ctx records CUDA events on its stream around every phase
 * of as_train_step / as_load_batch_* / as_merge.  as_profile_read synchronises
 * and returns, per phase, the summed device milliseconds and the number of
 * timed calls, plus the number of kernels the library launched since the
 * last read (all phases, profiled or not); counters are then reset. */
enum {
  AS_PH_BATCH = 0,     /* a2: batch H2D / device gather                         */
  AS_PH_TRANSPOSE = 1, /* a3                                                     */
  AS_PH_SPMM = 2,      /* a4                                                     */
  AS_PH_OUT_FWD = 3,   /* a5: tcgen05 pass 1 (or the fp32 logits GEMM + LSE)      */
  AS_PH_COMBINE = 4,   /* a5: label terms, combine, db1                          */
  AS_PH_OUT_BWD = 5,   /* a6: tcgen05 pass 2 with fused SGD (or fp32 GEMMs + SGD) */
  AS_PH_DW1 = 6,       /* a7                                                     */
  AS_PH_MERGE = 7,     /* a9-a13                                                 */
  AS_PH_COUNT = 8
};
int as_profile(as_ctx *ctx, int32_t enable);
int as_profile_read(as_ctx *ctx, double *ms_out, int64_t *calls_out,
                    int64_t *launches_out);

/* Tensor-core self-test (tests only): A, B are DEVICE bf16 [128][128]
 * row-major; writes DEVICE fp32 [128][128] results of the three operand
 * layouts the output layer uses:  S = A B^T;  P = bf16(S/16);  O = P B;
 * T = A^T P^T  (i.e. T[j][n] = sum_r A[r][j] P[n][r]).  Synchronises. */
int as_tc_selftest(const void *A, const void *B, float *S, float *O, float *T);

/* Self-test of the TMEM-A tensor-core path (tests only): A, B DEVICE bf16
 * [128][128]; A and P = bf16(A/4) are written row-per-lane into TMEM and
 * V = A B^T, U = P B are computed with A from TMEM.  Synchronises. */
int as_tc_selftest2(const void *A, const void *B, float *V, float *U);

/* tcgen05 issue-rate micro-benchmark (tools only): one CTA issues `iters`
 * groups of 128x128x128 bf16 MMAs (mode 0: K/K-major; 1: A MN-major; 2: B
 * MN-major; 3: N = 256) and returns the elapsed SM cycles in *cycles. */
int as_tc_bench(int32_t mode, int32_t iters, int64_t *cycles);

/* Event log of the tcgen05 kernels (tools only; non-empty only in a build
 * compiled with -DAS_TRACE): copies up to max_events {clock, code, tile}
 * int64 triples to out, clears the log, returns the count (>= 0). */
int as_trace_dump(int64_t *out, int32_t max_events);

/* ---- scheduler (pure host functions, steps a1, a10, a14) --------------------- */
typedef struct {        /* replay cost of a batch in picoseconds (R9):        */
  int64_t c0, c_row, c_nnz, num, den;  /* (c0 + c_row*rows + c_nnz*nnz)*num/den */
} as_cost_model;

typedef struct {
  int32_t replica;      /* i                                                   */
  int32_t rows;         /* rows of this batch (last one may be truncated, R8)  */
  int64_t start;        /* offset inside the mega-batch                         */
} as_route;

/* Static routing of one mega-batch for the comparison methods (P:71, P:215:
 * "multi-GPU SGD algorithms that do not consider heterogeneity"): batch k
 * covers samples [k*b0, k*b0 + b0) (last one truncated, R8) and goes to
 * replica k mod N regardless of speed (b[] must be all equal, = b0).  The
 * replay clocks are advanced exactly as in as_sched_route_replay so that the
 * straggler cost (max_i clocks_out[i]) is comparable.  Same arguments. */
int as_sched_route_static(int32_t N, const as_cost_model *cost, const int32_t *b,
                          int64_t M, const int64_t *nnz_prefix, as_route *out_log,
                          int64_t max_log, int64_t *n_log, int32_t *u_out,
                          int64_t *clocks_out);

/* Replay routing of one mega-batch (next batch to the GPU that frees
 * first; R8 ties -> lowest id, truncated last batch; R9 integer clocks).
 * nnz_prefix[M+1] (host) = cumulative nnz of the mega-batch's samples.
 * out_log capacity max_log entries; *n_log, u_out[N], clocks_out[N] written.
 * Returns AS_E_INVALID if out_log is too small. */
int as_sched_route_replay(int32_t N, const as_cost_model *cost, const int32_t *b,
                          int64_t M, const int64_t *nnz_prefix, as_route *out_log,
                          int64_t max_log, int64_t *n_log, int32_t *u_out,
                          int64_t *clocks_out);

/* Alg. 1 with R11 integer rounding; lr_out[i] =
 * (float)(lr0 * b_out[i] / b_max) (linear scaling rule). */
int as_sched_alg1(int32_t N, const int32_t *u, const int32_t *b, int32_t beta,
                  int32_t b_min, int32_t b_max, double lr0, int32_t *b_out,
                  float *lr_out);

/* Adaptive scaling frequency ("By default, the algorithm is executed
 * after every mega-batch. However, if stability is achieved or the system
 * enters an oscillatory state, the frequency at which scaling is performed
 * can be increased"), reading R27: the policy sets the INTERVAL,
 * in mega-batches, between two Alg. 1 runs.  Called after an Alg. 1 run with
 * its input b_prev[N] and output b_next[N] (host).  dir_state[N] (host,
 * in/out, caller-owned, zero-initialised) carries the sign of each b_i's
 * previous change.  Stable (no b_i changed) or oscillatory (some b_i reversed
 * direction, none kept it): *period_out = min(2 * period, p_max); otherwise
 * 1.  p_max = 1 is the paper's default (every mega-batch).  AS_E_INVALID on
 * N < 1, null pointers, p_max < 1 or period outside [1, p_max]; no state
 * change then. */
int as_sched_scale_period(int32_t N, const int32_t *b_prev, const int32_t *b_next,
                          int32_t *dir_state, int32_t period, int32_t p_max,
                          int32_t *period_out);

/* Alg. 2 lines 1-10 with R13-R16. */
int as_sched_alg2(int32_t N, const int32_t *u, const int32_t *b,
                  const double *norms, double delta, double pert_thr,
                  double *alpha_out, int32_t *perturbed_out);

/* as_sched_alg2 with the line-5 normalisation selectable: AS_NORM_UPDATES
 * (Alg. 2 as printed) or AS_NORM_UB ("normalize based on the product
 * between the number of updates and the batch size"), either OR-ed with
 * AS_NORM_R14_LITERAL (P:163 line 8 "r <- argmax_i {u_i}, s <- argmin_i {u_i}"
 * as printed: ties to the lowest id, no skip).  Same outputs; AS_E_INVALID
 * for any other norm_mode. */
int as_sched_alg2_ex(int32_t N, const int32_t *u, const int32_t *b, const double *norms,
                     double delta, double pert_thr, int32_t norm_mode, double *alpha_out,
                     int32_t *perturbed_out);

/* Fit one replica's replay cost model (R9) to a live trace of n >= 3 batches
 * (rows_k, nnz_k, measured time ps_k in picoseconds; host arrays): least
 * squares of ps = c0 + c_row rows + c_nnz nnz, integer-rounded, >= 0,
 * num = den = 1.  AS_E_INVALID when the design is singular. */
int as_sched_fit_cost(int64_t n, const int32_t *rows, const int64_t *nnz, const int64_t *ps,
                      as_cost_model *out);

/* Fisher-Yates permutation of [0, n) driven by SplitMix64(seed) (R10). */
int as_sched_permutation(int64_t n, uint64_t seed, int64_t *out);

/* Live routing: a cross-process shared cursor.  as_live_open
 * maps (creating if rank 0) a POSIX shm segment `name`; as_live_claim
 * atomically claims the next `b` samples of a mega-batch of M samples and
 * returns the start in *start and the (possibly truncated) row count in *rows
 * (0 when the mega-batch is exhausted); as_live_reset rearms for the next
 * mega-batch (call from one rank between barriers). */
typedef struct as_live as_live;
int as_live_open(const char *name, int32_t create, as_live **out);
int as_live_claim(as_live *lv, int64_t M, int32_t b, int64_t *start, int32_t *rows);
int as_live_reset(as_live *lv);
int as_live_close(as_live *lv, int32_t unlink_segment);

#ifdef __cplusplus
}
#endif
#endif /* ADASGD_H */

// Device-side helpers and the internal kernel-launcher interface of the
// Adaptive SGD hot path (sm_100a).  Internal: not part of the C-ABI.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <utility>

namespace as {

// Per-step descriptor kept in device memory so that kernels read the batch
// extents (which the device-side batch builder produces) without a host sync.
struct StepDesc {
  int32_t rows;    // B, rows of the batch
  int32_t nnz;     // features in the batch
  int32_t nlab;    // labels in the batch
  int32_t U;       // unique features (feature segments)
  int32_t V;       // unique labels (label segments)
  int32_t n_long;  // (unused, kept for the descriptor layout)
  int32_t err;     // device-side validation error (0 = ok)
  int32_t pad;
};


__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 t = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t *>(&t);
}

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

// Programmatic dependent launch: the step's kernels are launched with
// programmatic stream serialization so a kernel's launch and CTA scheduling
// overlap the tail of its predecessor; every such kernel starts with
// griddep_wait() (griddepcontrol.wait: the predecessor grid has completed and
// its memory is visible), a no-op when launched without the attribute.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args &&...args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
__device__ __forceinline__ int ceil_div_dev(int a, int b) { return (a + b - 1) / b; }

// cudaFuncSetAttribute is per device: `mask` (one per kernel instantiation)
// records the devices already configured (idempotent, so a race between two
// host threads only repeats the call).
inline bool first_on_device(std::atomic<unsigned long long> &mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (mask.load(std::memory_order_acquire) & bit) return false;
  mask.fetch_or(bit, std::memory_order_acq_rel);
  return true;
}

// Arguments of the batch transposes (step a3, kernels_transpose.cu).  Dense
// per-key state lives in the arena and is idle (0 / -1) between steps.
struct TrArgs {
  StepDesc *desc;
  int nnz_cap, lab_cap, d, C, W;              // W = 32-bit bitmap words per key
  // feature side (CSR entries -> feature-sorted)
  const int32_t *col, *rid;
  const float *val;
  int32_t *fcnt, *fsidx;
  uint32_t *fbits;
  int32_t *fseg_id, *fseg_ptr, *fseg_row, *fseg_of;
  float *fseg_val;
  // label side (label entries -> label-sorted)
  const int32_t *lab, *lrid;
  const int64_t *lab_ptr;
  int32_t *lcnt, *cls_seg;
  int4 *cls_lab;                              // per class {first, end, first row, first weight}
  uint32_t *lbits;
  int32_t *lseg_id, *lseg_ptr, *lseg_row;
  float *lw;
  // single-pass scan state
  unsigned long long *tile_state;
  int *ticket;
};

// ---------------------------------------------------------------- launchers
// batch construction (step a2)
void launch_gather_batch(cudaStream_t s, const int64_t *ds_row_ptr, const int32_t *ds_col,
                         const float *ds_val, const int64_t *ds_lab_ptr, const int32_t *ds_lab,
                         const int64_t *order, int64_t n, int64_t pos, int rows,
                         int64_t *row_ptr, int32_t *col, float *val, int64_t *lab_ptr,
                         int32_t *lab, int64_t *ids, int32_t *rid, int32_t *lrid, StepDesc *desc,
                         int nnz_cap, int lab_cap);
void launch_slice_batch(cudaStream_t s, const int64_t *ds_row_ptr, const int64_t *ds_lab_ptr, int64_t p0,
                        int rows, int64_t *row_ptr, int64_t *lab_ptr, int32_t *rid, int32_t *lrid,
                        StepDesc *desc, int nnz_cap, int lab_cap);
void launch_entry_rows(cudaStream_t s, const int64_t *row_ptr, const int64_t *lab_ptr, int rows,
                       int32_t *rid, int32_t *lrid);
void launch_transposes(cudaStream_t s, const TrArgs &a);
void launch_fill_int4(cudaStream_t s, int4 *p, long long n, int x, int y, int z, int w);
void launch_tr_reset(cudaStream_t s, const TrArgs &a, int num_sms);
// load-balanced chunked segmented gather-reduce (kernels_segmm.cu)
void launch_spmm_chunked(cudaStream_t s, int h, int num_sms, const StepDesc *desc, int bpad, int nnz_cap,
                         const int64_t *row_ptr, const int32_t *col, const float *val,
                         const int32_t *rid, const float *W1, const float *b1, float *Hf,
                         __nv_bfloat16 *Hb, float *part, int *arrive);
void launch_dw1_chunked(cudaStream_t s, int h, int num_sms, StepDesc *desc, int nnz_cap, const int32_t *seg_id,
                        const int32_t *seg_of, const int32_t *seg_ptr, const int32_t *seg_row,
                        const float *seg_val, const float *dA, float *W1, float lr, float *part,
                        int *arrive, float *dbg_dW1);
// label terms of loss and dH (steps a5)
void launch_label_terms(cudaStream_t s, int h, const StepDesc *desc, int b_max,
                        const int64_t *lab_ptr, const int32_t *lab, const float *Hf,
                        const float *W2T, const float *b2, float *zsum, float *labW);
// combine of the bf16 pass-1 partials -> LSE, loss rows, dA (steps a5)
void launch_combine_bf16(cudaStream_t s, int h, const StepDesc *desc, int b_max, int bpad,
                         int splits, const float *pm, const float *pl, const float *pO,
                         const float *labW, const float *zsum, const float *Hf, const int64_t *lab_ptr,
                         float *lse2, float *lsep, float *wrow, float *lossr, float *dA, float *db1p,
                         int *db1cnt, float *b1, float lr, float *dbg_db1, float *dbg_dHs,
                         __nv_bfloat16 *Hx /* FOLD B_ext rows [bpad][16], nullable */);
// fp32 (SIMT) output layer (steps a5/a6 in parity mode)
void launch_gemm_f32(cudaStream_t s, int M, int N, int K, const float *A, long long sam,
                     long long sak, const float *B, long long sbk, long long sbn, float *Cm,
                     long long ldc, const float *bias_n, int splitk, float *splitk_tmp,
                     const int *M_dev);
void launch_row_lse(cudaStream_t s, const StepDesc *desc, int b_max, int C, const float *Z,
                    float *lse2);
void launch_softmax_grad(cudaStream_t s, const StepDesc *desc, int b_max, int C,
                         const int64_t *lab_ptr, const int32_t *lab, float *Z, const float *lse2,
                         int part /* 1: softmax / B, 2: label term, 3: both */);
void launch_finish_f32(cudaStream_t s, int h, const StepDesc *desc, int b_max, const float *dH,
                       const float *Hf, const float *zsum, const float *lse2, float *lossr,
                       float *dA, const float *labW, float *dbg_dHs);
// column sums with fused SGD (db1 / db2)
void launch_colsum_sgd(cudaStream_t s, const StepDesc *desc, int n_rows_cap, int ncols,
                       const float *X, long long ldx, float *param, float lr, float *grad_out);
void launch_sgd_dense(cudaStream_t s, long long n, float *param, const float *grad, float lr,
                      __nv_bfloat16 *shadow);
void launch_loss_mean(cudaStream_t s, const StepDesc *desc, const float *lossr, float *loss);
// merge (steps a9-a13)
constexpr int kMaxWorld = 64;                   // == AS_MAX_WORLD of adasgd.h
struct MergeWeightArgs {                        // k_alg2 (by value)
  int N, mode, norm_mode;                       // mode 0: Alg. 2, 1: uniform 1/N, 2: given
  double delta, pert_thr;
  int32_t u[kMaxWorld], b[kMaxWorld];
  double given[kMaxWorld];
};
struct PeerArgs {                               // peer-memory merge (by value)
  int N, rank;
  unsigned long long epoch;
  long long P, w2_off, w2_len;
  float gamma;
  long long off_w, off_wbarp, off_w2b, off_flags, off_norms;   // byte offsets in every workspace
  uint8_t *base[kMaxWorld];                     // workspace of rank k, mapped here
};
void launch_scale_dev(cudaStream_t s, float *w, long long P, const float *alpha);
void launch_alg2(cudaStream_t s, const MergeWeightArgs &a, const double *norms, double *alpha_d, float *alpha_f,
                 int32_t *pert);
void launch_p2p_barrier(cudaStream_t s, const PeerArgs &a, const double *my_norm);
void launch_merge_p2p(cudaStream_t s, const PeerArgs &a, const float *alpha_f, const float *wbar,
                      const float *wbarp);
void launch_sumsq(cudaStream_t s, const float *w, long long P, double *partials, int nblocks,
                  double *out_norm, int metric);
void launch_scale(cudaStream_t s, float *w, long long P, float alpha);
void launch_momentum(cudaStream_t s, float *w, float *wbar_p_to_new, const float *wbar,
                     long long P, float gamma, long long w2_off, long long w2_len,
                     __nv_bfloat16 *shadow);
void launch_group_reduce(cudaStream_t s, const float *const *reps_dev, const float *alpha_dev,
                         int n, long long P, const float *wbar, float *wbar_p_to_new,
                         float gamma);
void launch_reset_from(cudaStream_t s, const float *src, float *w, float *wbar_new, long long P,
                       long long w2_off, long long w2_len, __nv_bfloat16 *shadow);
void launch_f32_to_bf16(cudaStream_t s, const float *src, __nv_bfloat16 *dst, long long n);

// tcgen05 output layer (steps a5/a6, AS_BF16)
struct TcPlan;
size_t tc_plan_bytes();
int tc_plan_init(TcPlan *plan, int h, int b_max, long long C, int num_sms, const void *Hb,
                 const void *W2b, const void *W2T, const void *Hx);
bool tc_fold(int h);   // pass 2 takes b2 and -(LSE + ln B) in its S^T MMA (B_ext rows from the combine)
int tc_splits(int h, int b_max, long long C, int num_sms);
// label terms of the loss and dH (a5, R3) computed by pass 1's two idle warps
// per CTA (zsum == nullptr: not computed there)
struct LtArgs {
  const int64_t *lab_ptr;
  const int32_t *lab;
  const float *Hf, *W2T, *b2;
  float *zsum, *labW;
};
void launch_out_fwd_tc(cudaStream_t s, const TcPlan *plan, const StepDesc *desc,
                       const float *b2, float *pm, float *pl, float *pO, const LtArgs &lt);
int tc_fwd_splits_host(const TcPlan *plan, int B);
// top-1 evaluation (NEXT f1): per-split (max, argmax) partials, then the ordered combine
void launch_out_top1_tc(cudaStream_t s, const TcPlan *plan, const StepDesc *desc, const float *b2,
                        float *pmax, int *pidx);
void launch_row_argmax_f32(cudaStream_t s, const StepDesc *desc, int b_max, int C, const float *Z, float *pmax,
                           int *pidx);
void launch_top1_combine(cudaStream_t s, const StepDesc *desc, int slots, int bpad, const float *pmax,
                         const int *pidx, const int64_t *lab_ptr, const int32_t *lab, int32_t *top1,
                         unsigned long long *hits);
int tc_bench(int mode, int iters, long long *cycles_host);
int tc_selftest2(const void *A, const void *B, float *V, float *U, cudaStream_t s);
int tc_trace_dump(long long *out, int max_events);
int tc_selftest(const void *A, const void *B, float *S, float *O, float *T, cudaStream_t s);
void launch_gemm_f32_kdev(cudaStream_t s, int M, int N, int K, const float *A, long long sam,
                          long long sak, const float *B, long long sbk, long long sbn, float *Cm,
                          long long ldc, const int *K_dev);
// step a7 fused into pass 2's idle warps (h = 128): feature segments of the
// batch transpose, dA, W1 (W1 == nullptr: not fused)
struct Dw1Args {
  const StepDesc *desc;
  const int32_t *seg_ptr, *seg_row, *seg_key;
  const float *seg_val, *dA;
  float *W1;
  float lr;
  float *dbg;
};
bool tc_fuses_dw1(int h);
void launch_out_bwd_tc(cudaStream_t s, const TcPlan *plan, const StepDesc *desc,
                       const float *lsep, const int4 *cls_lab, const uint32_t *lbits, int lbw,
                       const float *wrow, float *W2T, float *b2, __nv_bfloat16 *W2b, float lr,
                       float *dbg_dW2T, float *dbg_db2, const Dw1Args &dw);

}  // namespace as

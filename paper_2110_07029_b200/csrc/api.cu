// C-ABI of the Adaptive SGD hot path (include/adasgd.h): replica context,
// workspace arena, input validation, step and merge orchestration.
// P:N = PAPER.md line N; Rk = DESIGN.md reading k.
#include <cuda.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "adasgd.h"
#include "common.cuh"
#include "common_host.h"
#ifndef AS_STAGE_THREADS
#define AS_STAGE_THREADS 8                      // host threads of the batch validation + packing
#endif

thread_local char g_as_err[512] = "";

using as::StepDesc;

namespace {

constexpr size_t kAlign = 256;
constexpr int kNormBlocks = 148 * 8;

struct Layout {
  size_t off[64];
  int n = 0;
  size_t total = 0;
  size_t add(size_t bytes) {
    const size_t o = total;
    total += (bytes + kAlign - 1) / kAlign * kAlign;
    return o;
  }
};

struct Dims {
  long long d, C, P;
  int h, b_max, bpad, nnz_cap, lab_cap, sort_cap, max_splits, splitk;
  int bw, tr_tiles;   // transpose bitmap words per key, scan tiles
};

int key_bits(long long n) {
  int b = 1;
  while ((1ll << b) < n) ++b;
  return b;
}

}  // namespace

struct as_ctx {
  as_config cfg;
  Dims D;
  cudaStream_t stream;
  int num_sms;
  int sticky;
  // arena
  float *w, *wbar, *wbarp;
  __nv_bfloat16 *w2b;
  int64_t *row_ptr, *lab_ptr, *ids;
  int32_t *col, *lab;
  float *val;
  StepDesc *desc;
  // dense per-key transpose state (idle between steps: counts 0, bitmaps 0)
  int32_t *fcnt, *fsidx, *lcnt;
  uint32_t *fbits, *lbits;
  unsigned long long *tile_state;
  int *ticket, *arrive;
  int32_t *fseg_id, *fseg_ptr, *fseg_row, *fseg_of, *rid, *lrid;
  float *seg_part;
  float *fseg_val;
  int32_t *lseg_id, *lseg_ptr, *lseg_row, *cls_seg;
  int4 *cls_lab;
  float *lw;
  float *Hf;
  __nv_bfloat16 *Hb;
  __nv_bfloat16 *Hx;          // pass 2's B_ext rows (FOLD): [bpad][16]
  float *dA, *lse2, *lsep, *zsum, *labW, *lossr, *loss;
  float *pm, *pl, *pO;
  float *db1p;                // db1 partials of the fused combine
  float *wrow;                // per-row label weight 1/(k_r B) for pass 2
  int *db1cnt;
  int32_t *top1;              // top-1 evaluation (NEXT f1)
  unsigned long long *hits;
  float *Z, *dH, *dW2, *splitk_tmp;
  float *dbg_dW2, *dbg_db2, *dbg_dW1, *dbg_db1, *dbg_dHs;
  double *norm_part, *norm_dev, *norms_all;
  float *alpha_dev;            // local-group merge weights
  const float **reps_dev;
  // device-side merge weights (Alg. 2 on the device) and the peer-memory merge
  uint8_t *arena;              // workspace base (offsets are identical on every rank)
  double *alpha_d;             // [world] fp64
  float *alpha_f;              // [world] fp32 (PreMulSum scalar / fused merge)
  int32_t *pert_dev;
  unsigned long long *p2p_flags;  // [AS_MAX_WORLD] barrier epochs written by the peers
  uint8_t *peer_base[AS_MAX_WORLD];
  void *peer_map[AS_MAX_WORLD];   // cudaIpcOpenMemHandle mappings (closed at destroy)
  bool p2p_ready;
  unsigned long long p2p_epoch;
  as::TcPlan *plan;
  // host state
  std::vector<int32_t> b_all;
  float lr;
  int loaded_rows;
  long long loaded_nnz;         // host-side nnz of the loaded batch (estimate for a device gather)
  long long loaded_lab;         // the same for its labels
  double ds_mean_nnz, ds_mean_lab;   // resident dataset: mean nnz / labels per sample
  bool has_batch;
  void *pin[2];
  size_t pin_bytes;
  cudaEvent_t pin_ev[2];
  int pin_idx;
  // host batches (as_load_batch_csr / as_eval_top1): the packed pinned block
  // goes to one of two device staging blocks in ONE copy on the copy stream,
  // overlapping the previous step; the step reads the batch there
  uint8_t *stage_dev[2];
  cudaStream_t cp_s;
  cudaEvent_t ev_copied[2], ev_stage_free[2];
  int cur_stage;                // staging block of the loaded batch
  int stage_next;               // block the next load writes
  // resident dataset
  const int64_t *ds_row_ptr, *ds_lab_ptr, *ds_order;
  std::vector<int64_t> ds_rp_host, ds_lp_host;   // the dataset's pointers (slice offsets)
  const int32_t *ds_col, *ds_lab;
  const float *ds_val;
  int64_t ds_n;
  ncclComm_t comm;
  // side stream for the batch transposes (overlap with SpMM / pass 1)
  cudaStream_t side;
  cudaStream_t comm_s;          // partitioned merge: chunked all-reduce stream
  cudaEvent_t ev_mg[3];
  int merge_chunks;             // ADASGD_MERGE_CHUNKS (0 = default)
  cudaEvent_t ev_fork, ev_join, ev_tail, ev_lab;
  // live profiling (as_profile)
  bool prof_on;
  std::vector<cudaEvent_t> ev_pool;
  cudaEvent_t ph_start[AS_PH_COUNT];
  struct Pend { int ph; cudaEvent_t a, b; };
  std::vector<Pend> pending;
  long long launches;
};

namespace {

int validate_cfg(const as_config *c) {
  if (!c) return as_fail(AS_E_INVALID, "config is NULL");
  if (c->n_features < 1 || c->n_labels < 1 || c->n_features >= (1ll << 31) ||
      c->n_labels >= (1ll << 31))
    return as_fail(AS_E_INVALID, "n_features / n_labels out of range");
  if (c->hidden != 128 && c->hidden != 256) return as_fail(AS_E_INVALID, "hidden must be 128 or 256");
  if (c->b_max < 1 || c->b_min < 1 || c->b_min > c->b_max || c->b_max > 65536)
    return as_fail(AS_E_INVALID, "need 1 <= b_min <= b_max <= 65536");
  if (c->beta < 0) return as_fail(AS_E_INVALID, "beta < 0");
  if (c->max_row_nnz < 1 || c->max_row_labels < 1)
    return as_fail(AS_E_INVALID, "max_row_nnz / max_row_labels must be >= 1");
  if ((long long)c->b_max * c->max_row_nnz >= (1ll << 31) ||
      (long long)c->b_max * c->max_row_labels >= (1ll << 31))
    return as_fail(AS_E_INVALID, "batch capacity exceeds 2^31 entries");
  if (c->algo < AS_ALGO_ADAPTIVE || c->algo > AS_ALGO_SYNC) return as_fail(AS_E_INVALID, "unknown algo %d", c->algo);
  if (c->precision != AS_FP32 && c->precision != AS_BF16)
    return as_fail(AS_E_INVALID, "precision must be AS_FP32 or AS_BF16");
  if (c->world < 1 || c->world > AS_MAX_WORLD || c->rank < 0 || c->rank >= c->world)
    return as_fail(AS_E_INVALID, "need 0 <= rank < world <= %d", (int)AS_MAX_WORLD);
  if (c->merge_backend != AS_MERGE_NCCL && c->merge_backend != AS_MERGE_P2P)
    return as_fail(AS_E_INVALID, "unknown merge_backend %d", c->merge_backend);
  if (!(c->lr0 > 0.0)) return as_fail(AS_E_INVALID, "lr0 must be > 0");
  return AS_OK;
}

Dims dims_of(const as_config *c) {
  Dims D;
  D.d = c->n_features;
  D.C = c->n_labels;
  D.h = c->hidden;
  D.P = D.d * D.h + D.h + D.C * D.h + D.C;
  D.b_max = c->b_max;
  D.bpad = (c->b_max + 127) / 128 * 128;
  D.nnz_cap = c->b_max * c->max_row_nnz;
  D.lab_cap = c->b_max * c->max_row_labels;
  D.sort_cap = std::max(std::max(D.nnz_cap, D.lab_cap), D.bpad);
  D.bw = (c->b_max + 127) / 128 * 4;          // bitmap words per key (16-B rows)
  D.tr_tiles = (D.d + 8191) / 8192 + (D.C + 8191) / 8192;
  D.max_splits = 2 * as::tc_splits(D.h, D.b_max, D.C, 160);  // partial slots (2 per pass-1 CTA)
  D.splitk = (int)std::min<long long>(64, std::max<long long>(1, D.C / 4096));
  return D;
}

// A batch staging block (two per ctx; a step reads its batch from one while the
// next batch is written into the other).  Capacity layout: row_ptr, lab_ptr
// (b_max + 1 each, int64), col, val (nnz_cap), lab (lab_cap), StepDesc (64-B
// aligned), then the per-batch work arrays ids (b_max), rid (nnz_cap), lrid
// (lab_cap).  A host batch is packed with its actual sizes into the same
// leading region (so one copy moves it) and never extends past `desc + 64`.
struct StageLayout { size_t lp, col, val, lab, desc, ids, rid, lrid, total; };
StageLayout stage_layout(const Dims &D) {
  StageLayout L;
  const size_t b1 = (size_t)D.b_max + 1;
  L.lp = 8 * b1;
  L.col = 16 * b1;
  L.val = L.col + 4 * (size_t)D.nnz_cap;
  L.lab = L.val + 4 * (size_t)D.nnz_cap;
  L.desc = (L.lab + 4 * (size_t)D.lab_cap + 63) & ~(size_t)63;
  L.ids = L.desc + 64;
  L.rid = L.ids + 8 * (size_t)D.b_max;
  L.lrid = L.rid + 4 * (size_t)D.nnz_cap;
  L.total = L.lrid + 4 * (size_t)D.lab_cap;
  return L;
}

// The arena carve: every buffer of the step sized for b_max ("we
// provision memory for the largest batch size").  Order fixed; `ctx` NULL ->
// just the total.
size_t carve(const as_config *c, const Dims &D, as_ctx *x, uint8_t *base) {
  Layout L;
  auto P = [&](size_t bytes) -> void * { const size_t o = L.add(bytes); return base ? base + o : nullptr; };
  const size_t S = (size_t)D.sort_cap;
  const bool bf16 = c->precision == AS_BF16;
  const bool dbg = (c->flags & AS_FLAG_DEBUG_GRADS) != 0;
  void *p;
  p = P(4 * D.P); if (x) x->w = (float *)p;
  p = P(4 * D.P); if (x) x->wbar = (float *)p;
  p = P(4 * D.P); if (x) x->wbarp = (float *)p;
  p = P(2 * D.C * D.h); if (x) x->w2b = (__nv_bfloat16 *)p;
  for (int k = 0; k < 2; ++k) {
    p = P(stage_layout(D).total); if (x) x->stage_dev[k] = (uint8_t *)p;
  }
  p = P(4 * (size_t)D.d); if (x) x->fcnt = (int32_t *)p;
  p = P(4 * (size_t)D.d); if (x) x->fsidx = (int32_t *)p;
  p = P(4 * (size_t)D.d * D.bw); if (x) x->fbits = (uint32_t *)p;
  p = P(4 * (size_t)D.C); if (x) x->lcnt = (int32_t *)p;
  p = P(4 * (size_t)D.C * D.bw); if (x) x->lbits = (uint32_t *)p;
  p = P(8 * (size_t)D.tr_tiles); if (x) x->tile_state = (unsigned long long *)p;
  p = P(16); if (x) x->ticket = (int *)p;
  p = P(4 * S); if (x) x->arrive = (int *)p;
  p = P(4 * (size_t)D.nnz_cap); if (x) x->fseg_id = (int32_t *)p;
  p = P(4 * ((size_t)D.nnz_cap + 1)); if (x) x->fseg_ptr = (int32_t *)p;
  p = P(4 * (size_t)D.nnz_cap); if (x) x->fseg_row = (int32_t *)p;
  p = P(4 * (size_t)D.nnz_cap); if (x) x->fseg_val = (float *)p;
  p = P(4 * (size_t)D.nnz_cap); if (x) x->fseg_of = (int32_t *)p;
  p = P(4 * 2 * (size_t)D.h * (std::max<size_t>((size_t)D.sort_cap * D.h / 2048, 1024) + 2)); if (x) x->seg_part = (float *)p;
  p = P(4 * (size_t)D.lab_cap); if (x) x->lseg_id = (int32_t *)p;
  p = P(4 * ((size_t)D.lab_cap + 1)); if (x) x->lseg_ptr = (int32_t *)p;
  p = P(4 * (size_t)D.lab_cap); if (x) x->lseg_row = (int32_t *)p;
  p = P(4 * (size_t)D.lab_cap); if (x) x->lw = (float *)p;
  p = P(4 * D.C); if (x) x->cls_seg = (int32_t *)p;
  p = P(16 * D.C); if (x) x->cls_lab = (int4 *)p;
  p = P(4 * (size_t)D.bpad * D.h); if (x) x->Hf = (float *)p;
  p = P(2 * (size_t)D.bpad * D.h); if (x) x->Hb = (__nv_bfloat16 *)p;
  p = P(2 * 16 * (size_t)D.bpad); if (x) x->Hx = (__nv_bfloat16 *)p;
  p = P(4 * (size_t)D.b_max * D.h); if (x) x->dA = (float *)p;
  p = P(4 * (size_t)D.bpad); if (x) x->lse2 = (float *)p;
  p = P(4 * (size_t)D.bpad); if (x) x->lsep = (float *)p;
  p = P(4 * (size_t)D.b_max); if (x) x->zsum = (float *)p;
  p = P(4 * (size_t)D.b_max * D.h); if (x) x->labW = (float *)p;
  p = P(4 * (size_t)D.b_max); if (x) x->lossr = (float *)p;
  p = P(4); if (x) x->loss = (float *)p;
  p = P(4 * (size_t)D.max_splits * D.bpad); if (x) x->pm = (float *)p;
  p = P(4 * (size_t)D.max_splits * D.bpad); if (x) x->pl = (float *)p;
  p = P(4 * (size_t)D.bpad); if (x) x->top1 = (int32_t *)p;
  p = P(4 * (size_t)(D.bpad / 32 + 1) * D.h); if (x) x->db1p = (float *)p;
  p = P(4 * (size_t)D.bpad); if (x) x->wrow = (float *)p;
  p = P(4 * (size_t)D.h); if (x) x->db1cnt = (int *)p;
  p = P(8); if (x) x->hits = (unsigned long long *)p;
  if (bf16) {
    p = P(4 * (size_t)D.max_splits * D.bpad * D.h); if (x) x->pO = (float *)p;
  } else {
    p = P(4 * (size_t)D.b_max * D.C); if (x) x->Z = (float *)p;
    p = P(4 * (size_t)D.b_max * D.h); if (x) x->dH = (float *)p;
    p = P(4 * (size_t)D.C * D.h); if (x) x->dW2 = (float *)p;
    p = P(4 * (size_t)D.splitk * D.b_max * D.h); if (x) x->splitk_tmp = (float *)p;
  }
  if (dbg) {
    p = P(4 * (size_t)D.C * D.h); if (x) x->dbg_dW2 = (float *)p;
    p = P(4 * (size_t)D.C); if (x) x->dbg_db2 = (float *)p;
    p = P(4 * (size_t)D.nnz_cap * D.h); if (x) x->dbg_dW1 = (float *)p;
    p = P(4 * (size_t)D.h); if (x) x->dbg_db1 = (float *)p;
    p = P(4 * (size_t)D.b_max * D.h); if (x) x->dbg_dHs = (float *)p;
  }
  p = P(8 * kNormBlocks); if (x) x->norm_part = (double *)p;
  p = P(8); if (x) x->norm_dev = (double *)p;
  p = P(8 * (size_t)AS_MAX_WORLD); if (x) x->norms_all = (double *)p;
  p = P(4 * (size_t)c->world); if (x) x->alpha_dev = (float *)p;
  p = P(8 * (size_t)AS_MAX_WORLD); if (x) x->alpha_d = (double *)p;
  p = P(4 * (size_t)AS_MAX_WORLD); if (x) x->alpha_f = (float *)p;
  p = P(8); if (x) x->pert_dev = (int32_t *)p;
  p = P(8 * (size_t)AS_MAX_WORLD); if (x) x->p2p_flags = (unsigned long long *)p;
  p = P(8 * (size_t)c->world); if (x) x->reps_dev = (const float **)p;
  return L.total;
}

int cuda_check(as_ctx *x, cudaError_t e, const char *what) {
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    if (x) x->sticky = AS_E_CUDA;
    return as_fail(AS_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
  }
  return AS_OK;
}

cudaEvent_t get_event(as_ctx *x) {
  if (!x->ev_pool.empty()) {
    cudaEvent_t e = x->ev_pool.back();
    x->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
inline void ph_begin(as_ctx *x, int ph, cudaStream_t s = nullptr) {
  if (!x->prof_on) return;
  x->ph_start[ph] = get_event(x);
  cudaEventRecord(x->ph_start[ph], s ? s : x->stream);
}
inline void ph_end(as_ctx *x, int ph, cudaStream_t s = nullptr) {
  if (!x->prof_on) return;
  cudaEvent_t e = get_event(x);
  cudaEventRecord(e, s ? s : x->stream);
  x->pending.push_back({ph, x->ph_start[ph], e});
}
// kernels launched by the transpose of a key space with `bits` bits

#define AS_GUARD(x)                                                               \
  do {                                                                            \
    if (!(x)) return as_fail(AS_E_INVALID, "ctx is NULL");                        \
    if ((x)->sticky) return as_fail(AS_E_STATE, "ctx poisoned by an earlier error"); \
    cudaSetDevice((x)->cfg.device);                                               \
  } while (0)

// Host validation of one CSR batch (SURVEY 8(b) conventions).  Returns nnz/L.
int validate_csr(const as_ctx *x, int64_t rows, const int64_t *row_ptr, const int32_t *col,
                 const float *val, const int64_t *lab_ptr, const int32_t *lab, int64_t *nnz_out,
                 int64_t *L_out) {
  if (!row_ptr || !lab_ptr) return as_fail(AS_E_INVALID, "row_ptr / lab_ptr is NULL");
  const int64_t nnz = row_ptr[rows] - row_ptr[0], L = lab_ptr[rows] - lab_ptr[0];
  if (nnz < 0 || L < 0) return as_fail(AS_E_INVALID, "pointers not monotone");
  if ((nnz > 0 && (!col || !val)) || !lab) return as_fail(AS_E_INVALID, "col/val/lab is NULL");
  for (int64_t r = 0; r < rows; ++r) {
    const int64_t s = row_ptr[r], e = row_ptr[r + 1];
    if (e < s) return as_fail(AS_E_INVALID, "row_ptr not monotone at row %lld", (long long)r);
    if (e - s > x->cfg.max_row_nnz)
      return as_fail(AS_E_INVALID, "row %lld has %lld nnz > max_row_nnz", (long long)r, (long long)(e - s));
    for (int64_t j = s; j < e; ++j) {
      if (col[j] < 0 || col[j] >= x->D.d)
        return as_fail(AS_E_INVALID, "feature id %d out of range in row %lld", col[j], (long long)r);
      if (j > s && col[j] <= col[j - 1])
        return as_fail(AS_E_INVALID, "features of row %lld not strictly increasing", (long long)r);
    }
    const int64_t ls = lab_ptr[r], le = lab_ptr[r + 1];
    if (le <= ls) return as_fail(AS_E_INVALID, "row %lld has no label (R3)", (long long)r);
    if (le - ls > x->cfg.max_row_labels)
      return as_fail(AS_E_INVALID, "row %lld has too many labels", (long long)r);
    for (int64_t j = ls; j < le; ++j) {
      if (lab[j] < 0 || lab[j] >= x->D.C)
        return as_fail(AS_E_INVALID, "label id %d out of range in row %lld", lab[j], (long long)r);
      if (j > ls && lab[j] <= lab[j - 1])
        return as_fail(AS_E_INVALID, "labels of row %lld not strictly increasing", (long long)r);
    }
  }
  *nnz_out = nnz;
  *L_out = L;
  return AS_OK;
}

// point the ctx's batch arrays at staging block k: capacity layout (device
// gather) or, with `packed` = {lp, col, val, lab, desc} offsets, a host batch
void use_stage(as_ctx *x, int k, const size_t *packed) {
  const StageLayout L = stage_layout(x->D);
  uint8_t *g = x->stage_dev[k];
  const size_t lp = packed ? packed[0] : L.lp, col = packed ? packed[1] : L.col, val = packed ? packed[2] : L.val,
               lab = packed ? packed[3] : L.lab, desc = packed ? packed[4] : L.desc;
  x->row_ptr = (int64_t *)g;
  x->lab_ptr = (int64_t *)(g + lp);
  x->col = (int32_t *)(g + col);
  x->val = (float *)(g + val);
  x->lab = (int32_t *)(g + lab);
  x->desc = (StepDesc *)(g + desc);
  x->ids = (int64_t *)(g + L.ids);
  x->rid = (int32_t *)(g + L.rid);
  x->lrid = (int32_t *)(g + L.lrid);
  x->cur_stage = k;
}

as::TrArgs tr_args(as_ctx *x) {
  const Dims &D = x->D;
  as::TrArgs a{};
  a.desc = x->desc;
  a.nnz_cap = (int)D.nnz_cap; a.lab_cap = (int)D.lab_cap; a.d = (int)D.d; a.C = (int)D.C; a.W = D.bw;
  a.col = x->col; a.rid = x->rid; a.val = x->val;
  a.fcnt = x->fcnt; a.fsidx = x->fsidx; a.fbits = x->fbits;
  a.fseg_id = x->fseg_id; a.fseg_ptr = x->fseg_ptr; a.fseg_row = x->fseg_row; a.fseg_of = x->fseg_of;
  a.fseg_val = x->fseg_val;
  a.lab = x->lab; a.lrid = x->lrid; a.lab_ptr = x->lab_ptr;
  a.lcnt = x->lcnt; a.cls_seg = x->cls_seg; a.cls_lab = x->cls_lab; a.lbits = x->lbits;
  a.lseg_id = x->lseg_id; a.lseg_ptr = x->lseg_ptr; a.lseg_row = x->lseg_row; a.lw = x->lw;
  a.tile_state = x->tile_state; a.ticket = x->ticket;
  return a;
}

}  // namespace

extern "C" {

const char *as_last_error(void) { return g_as_err; }

int as_workspace_size(const as_config *cfg, size_t *bytes) {
  const int rc = validate_cfg(cfg);
  if (rc) return rc;
  if (!bytes) return as_fail(AS_E_INVALID, "bytes is NULL");
  *bytes = carve(cfg, dims_of(cfg), nullptr, nullptr);
  return AS_OK;
}

int as_nccl_unique_id(void *out128) {
  if (!out128) return as_fail(AS_E_INVALID, "out is NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  const ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return as_fail(AS_E_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  memcpy(out128, &id, 128);
  return AS_OK;
}

int as_init(const as_config *cfg, const float *init_params, as_ctx **out) {
  int rc = validate_cfg(cfg);
  if (rc) return rc;
  if (!init_params || !out) return as_fail(AS_E_INVALID, "init_params / out is NULL");
  const Dims D = dims_of(cfg);
  const size_t need = carve(cfg, D, nullptr, nullptr);
  if (!cfg->workspace || cfg->workspace_bytes < need)
    return as_fail(AS_E_OOM, "workspace too small: need %zu bytes", need);
  if (((uintptr_t)cfg->workspace) % kAlign)
    return as_fail(AS_E_INVALID, "workspace must be %zu-byte aligned", kAlign);
  if (cudaSetDevice(cfg->device) != cudaSuccess)
    return as_fail(AS_E_CUDA, "cudaSetDevice(%d) failed", cfg->device);
  as_ctx *x = new as_ctx();
  x->cfg = *cfg;
  x->D = D;
  x->stream = (cudaStream_t)cfg->stream;
  cudaDeviceGetAttribute(&x->num_sms, cudaDevAttrMultiProcessorCount, cfg->device);
  carve(cfg, D, x, (uint8_t *)cfg->workspace);
  x->arena = (uint8_t *)cfg->workspace;
  x->b_all.assign(cfg->world, cfg->b_max);
  x->lr = (float)cfg->lr0;
  const size_t P4 = 4 * (size_t)D.P;
  rc = cuda_check(x, cudaMemcpyAsync(x->w, init_params, P4, cudaMemcpyHostToDevice, x->stream), "init H2D");
  if (!rc) rc = cuda_check(x, cudaMemcpyAsync(x->wbar, x->w, P4, cudaMemcpyDeviceToDevice, x->stream), "init copy");
  if (!rc) rc = cuda_check(x, cudaMemcpyAsync(x->wbarp, x->w, P4, cudaMemcpyDeviceToDevice, x->stream), "init copy");
  if (!rc) {
    as::launch_f32_to_bf16(x->stream, x->w + D.d * D.h + D.h, x->w2b, D.C * D.h);
    rc = cuda_check(x, cudaMemsetAsync(x->cls_seg, 0xFF, 4 * D.C, x->stream), "memset");
  }
  // idle transpose / combine state (returned to idle by every step)
  if (!rc) rc = cuda_check(x, cudaMemsetAsync(x->fcnt, 0, 4 * (size_t)D.d, x->stream), "memset");
  if (!rc) as::launch_fill_int4(x->stream, x->cls_lab, D.C, 0, 0, 0x7fffffff, 0);
  if (!rc) rc = cuda_check(x, cudaMemsetAsync(x->fbits, 0, 4 * (size_t)D.d * D.bw, x->stream), "memset");
  if (!rc) rc = cuda_check(x, cudaMemsetAsync(x->lcnt, 0, 4 * (size_t)D.C, x->stream), "memset");
  if (!rc) rc = cuda_check(x, cudaMemsetAsync(x->lbits, 0, 4 * (size_t)D.C * D.bw, x->stream), "memset");
  if (!rc) rc = cuda_check(x, cudaMemsetAsync(x->tile_state, 0, 8 * (size_t)D.tr_tiles, x->stream), "memset");
  if (!rc) rc = cuda_check(x, cudaMemsetAsync(x->ticket, 0, 16, x->stream), "memset");
  if (!rc) rc = cuda_check(x, cudaMemsetAsync(x->db1cnt, 0, 4 * (size_t)D.h, x->stream), "memset");
  if (!rc) rc = cuda_check(x, cudaMemsetAsync(x->arrive, 0, 4 * (size_t)D.sort_cap, x->stream), "memset");
  if (!rc) rc = cuda_check(x, cudaMemsetAsync(x->Hb, 0, 2 * (size_t)D.bpad * D.h, x->stream), "memset");
  if (!rc) rc = cuda_check(x, cudaMemsetAsync(x->p2p_flags, 0, 8 * (size_t)AS_MAX_WORLD, x->stream), "memset");
  if (!rc) rc = cuda_check(x, cudaMemsetAsync(x->norms_all, 0, 8 * (size_t)AS_MAX_WORLD, x->stream), "memset");
  // side stream at the lowest priority: the transposes fill SMs the critical
  // path (SpMM, pass 1 on the caller's stream) leaves idle
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
#ifdef AS_X_SIDEHI
  if (!rc) rc = cuda_check(x, cudaStreamCreateWithPriority(&x->side, cudaStreamNonBlocking, prio_hi), "side stream");
#else
  if (!rc) rc = cuda_check(x, cudaStreamCreateWithPriority(&x->side, cudaStreamNonBlocking, prio_lo), "side stream");
#endif
  if (!rc) rc = cuda_check(x, cudaEventCreateWithFlags(&x->ev_fork, cudaEventDisableTiming), "event");
  if (!rc) rc = cuda_check(x, cudaEventCreateWithFlags(&x->ev_join, cudaEventDisableTiming), "event");
  if (!rc) rc = cuda_check(x, cudaEventCreateWithFlags(&x->ev_tail, cudaEventDisableTiming), "event");
  if (!rc) rc = cuda_check(x, cudaEventCreateWithFlags(&x->ev_lab, cudaEventDisableTiming), "event");
  if (!rc) rc = cuda_check(x, cudaStreamCreateWithPriority(&x->comm_s, cudaStreamNonBlocking, prio_hi), "comm stream");
  for (int i = 0; i < 3 && !rc; ++i)
    rc = cuda_check(x, cudaEventCreateWithFlags(&x->ev_mg[i], cudaEventDisableTiming), "event");
  if (const char *mc = getenv("ADASGD_MERGE_CHUNKS")) x->merge_chunks = atoi(mc) > 0 ? atoi(mc) : 0;
  // pinned double-buffered staging for host batches
  x->pin_bytes = stage_layout(D).desc + 64;
  use_stage(x, 0, nullptr);
  x->stage_next = 0;
  if (!rc) rc = cuda_check(x, cudaStreamCreateWithPriority(&x->cp_s, cudaStreamNonBlocking, prio_hi), "copy stream");
  for (int i = 0; i < 2 && !rc; ++i) {
    rc = cuda_check(x, cudaEventCreateWithFlags(&x->ev_copied[i], cudaEventDisableTiming), "event");
    if (!rc) rc = cuda_check(x, cudaEventCreateWithFlags(&x->ev_stage_free[i], cudaEventDisableTiming), "event");
  }
  for (int i = 0; i < 2 && !rc; ++i) {
    rc = cuda_check(x, cudaMallocHost(&x->pin[i], x->pin_bytes), "cudaMallocHost");
    if (!rc) rc = cuda_check(x, cudaEventCreateWithFlags(&x->pin_ev[i], cudaEventDisableTiming), "event");
  }
  if (!rc && cfg->precision == AS_BF16) {
    x->plan = (as::TcPlan *)malloc(as::tc_plan_bytes());
    if (as::tc_plan_init(x->plan, D.h, D.b_max, D.C, x->num_sms, x->Hb, x->w2b, x->w + D.d * D.h + D.h, x->Hx) != 0)
      rc = as_fail(AS_E_CUDA, "cuTensorMapEncodeTiled failed (driver entry point missing?)");
  }
  if (!rc && cfg->world == 1 && getenv("ADASGD_NCCL_SELF") && atoi(getenv("ADASGD_NCCL_SELF")) > 0) {
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r == ncclSuccess) r = ncclCommInitRank(&x->comm, 1, id, 0);
    if (r != ncclSuccess) rc = as_fail(AS_E_NCCL, "one-rank ncclCommInitRank: %s", ncclGetErrorString(r));
  }
  if (!rc && cfg->world > 1 && cfg->nccl_unique_id) {
    ncclUniqueId id;
    memcpy(&id, cfg->nccl_unique_id, 128);
    const ncclResult_t r = ncclCommInitRank(&x->comm, cfg->world, id, cfg->rank);
    if (r != ncclSuccess) rc = as_fail(AS_E_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  }
  if (!rc) rc = cuda_check(x, cudaStreamSynchronize(x->stream), "init sync");
  if (rc) {
    as_destroy(x);
    return rc;
  }
  *out = x;
  return AS_OK;
}

int as_destroy(as_ctx *x) {
  if (!x) return AS_OK;
  cudaSetDevice(x->cfg.device);
  if (x->stream) cudaStreamSynchronize(x->stream);
  for (int i = 0; i < 2; ++i) {
    if (x->pin[i]) cudaFreeHost(x->pin[i]);
    if (x->pin_ev[i]) cudaEventDestroy(x->pin_ev[i]);
  }
  if (x->comm) ncclCommDestroy(x->comm);
  for (int k = 0; k < AS_MAX_WORLD; ++k)
    if (x->peer_map[k]) cudaIpcCloseMemHandle(x->peer_map[k]);
  if (x->side) { cudaStreamSynchronize(x->side); cudaStreamDestroy(x->side); }
  if (x->ev_fork) cudaEventDestroy(x->ev_fork);
  if (x->ev_join) cudaEventDestroy(x->ev_join);
  if (x->ev_tail) cudaEventDestroy(x->ev_tail);
  if (x->ev_lab) cudaEventDestroy(x->ev_lab);
  for (int i = 0; i < 3; ++i)
    if (x->ev_mg[i]) cudaEventDestroy(x->ev_mg[i]);
  if (x->comm_s) { cudaStreamSynchronize(x->comm_s); cudaStreamDestroy(x->comm_s); }
  if (x->cp_s) { cudaStreamSynchronize(x->cp_s); cudaStreamDestroy(x->cp_s); }
  for (int i = 0; i < 2; ++i) {
    if (x->ev_copied[i]) cudaEventDestroy(x->ev_copied[i]);
    if (x->ev_stage_free[i]) cudaEventDestroy(x->ev_stage_free[i]);
  }
  for (auto &p : x->pending) { x->ev_pool.push_back(p.a); x->ev_pool.push_back(p.b); }
  for (auto e : x->ev_pool) cudaEventDestroy(e);
  free(x->plan);
  delete x;
  return AS_OK;
}

// validate a host CSR batch and stage it (pinned, double-buffered) onto the
// device batch buffers; shared by as_load_batch_csr and as_eval_top1
static int stage_batch(as_ctx *x, int32_t rows, const int64_t *row_ptr, const int32_t *col, const float *val,
                       const int64_t *lab_ptr, const int32_t *lab) {
  if (!row_ptr || !lab_ptr) return as_fail(AS_E_INVALID, "row_ptr / lab_ptr is NULL");
  const int64_t nnz = row_ptr[rows] - row_ptr[0], L = lab_ptr[rows] - lab_ptr[0];
  if (nnz < 0 || L < 0) return as_fail(AS_E_INVALID, "pointers not monotone");
  if ((nnz > 0 && (!col || !val)) || !lab) return as_fail(AS_E_INVALID, "col/val/lab is NULL");
  if (nnz > x->D.nnz_cap || L > x->D.lab_cap) return as_fail(AS_E_INVALID, "batch exceeds capacity");
  const int k = x->stage_next;
  int rc = cuda_check(x, cudaEventSynchronize(x->pin_ev[k]), "staging wait");   // pinned block k reusable
  if (rc) return rc;
  uint8_t *p = (uint8_t *)x->pin[k];
  const size_t o_lp = 8 * (size_t)(rows + 1), o_cc = 2 * o_lp, o_vv = o_cc + 4 * (size_t)nnz,
               o_ll = o_vv + 4 * (size_t)nnz, o_dd = (o_ll + 4 * (size_t)L + 63) & ~(size_t)63;
  int64_t *rp = (int64_t *)p;
  int64_t *lp = (int64_t *)(p + o_lp);
  int32_t *cc = (int32_t *)(p + o_cc);
  float *vv = (float *)(p + o_vv);
  int32_t *ll = (int32_t *)(p + o_ll);
  StepDesc *dd = (StepDesc *)(p + o_dd);
  // validation (the rules of validate_csr) fused with the packing, rows split
  // over host threads for large batches; a thread copies its rows' segments
  // only once all of them are valid.  On any error the batch is re-validated
  // serially for validate_csr's message and nothing is enqueued: no state change.
  const int T = (nnz + L > 32768) ? AS_STAGE_THREADS : 1;
  int bad[AS_STAGE_THREADS] = {0};
  const int64_t c0 = row_ptr[0], l0 = lab_ptr[0];
  const int64_t d = x->D.d, C = x->D.C, mrn = x->cfg.max_row_nnz, mrl = x->cfg.max_row_labels;
#pragma omp parallel for num_threads(T) schedule(static)
  for (int t = 0; t < T; ++t) {
    const int64_t r0 = (int64_t)rows * t / T, r1 = (int64_t)rows * (t + 1) / T;
    bool ok = true;
    for (int64_t r = r0; r < r1 && ok; ++r) {
      const int64_t s0 = row_ptr[r], e0 = row_ptr[r + 1], ls = lab_ptr[r], le = lab_ptr[r + 1];
      if (e0 < s0 || e0 - s0 > mrn || le <= ls || le - ls > mrl) { ok = false; break; }
      for (int64_t j = s0; j < e0; ++j)
        if (col[j] < 0 || col[j] >= d || (j > s0 && col[j] <= col[j - 1])) { ok = false; break; }
      for (int64_t j = ls; j < le && ok; ++j)
        if (lab[j] < 0 || lab[j] >= C || (j > ls && lab[j] <= lab[j - 1])) ok = false;
    }
    if (!ok) { bad[t] = 1; continue; }
    for (int64_t r = r0; r < r1; ++r) { rp[r] = row_ptr[r] - c0; lp[r] = lab_ptr[r] - l0; }
    if (t == T - 1) { rp[rows] = nnz; lp[rows] = L; }
    const int64_t a = row_ptr[r0], e = row_ptr[r1], la = lab_ptr[r0], lb = lab_ptr[r1];
    if (e > a) {
      memcpy(cc + (a - c0), col + a, 4 * (size_t)(e - a));
      memcpy(vv + (a - c0), val + a, 4 * (size_t)(e - a));
    }
    if (lb > la) memcpy(ll + (la - l0), lab + la, 4 * (size_t)(lb - la));
  }
  for (int t = 0; t < T; ++t)
    if (bad[t]) {
      int64_t n2 = 0, L2 = 0;
      rc = validate_csr(x, rows, row_ptr, col, val, lab_ptr, lab, &n2, &L2);
      return rc ? rc : as_fail(AS_E_INVALID, "invalid batch");
    }
  x->stage_next ^= 1;
  memset(dd, 0, sizeof(StepDesc));
  dd->rows = rows;
  dd->nnz = (int32_t)nnz;
  dd->nlab = (int32_t)L;
  cudaStream_t s = x->stream;
  // ONE copy of the packed block into device staging block k, on the copy
  // stream once the step that last read block k is done; the main stream
  // waits for it (the copy overlaps the previous step)
  ph_begin(x, AS_PH_BATCH);
  cudaStreamWaitEvent(x->cp_s, x->ev_stage_free[k], 0);
  cudaMemcpyAsync(x->stage_dev[k], p, o_dd + sizeof(StepDesc), cudaMemcpyHostToDevice, x->cp_s);
  rc = cuda_check(x, cudaEventRecord(x->pin_ev[k], x->cp_s), "batch H2D");
  if (rc) return rc;
  const size_t packed[5] = {o_lp, o_cc, o_vv, o_ll, o_dd};
  use_stage(x, k, packed);
  x->launches += 1;                     // entry -> row maps, also off the main stream
  as::launch_entry_rows(x->cp_s, x->row_ptr, x->lab_ptr, rows, x->rid, x->lrid);
  cudaEventRecord(x->ev_copied[k], x->cp_s);
  cudaStreamWaitEvent(s, x->ev_copied[k], 0);
  ph_end(x, AS_PH_BATCH);
  rc = cuda_check(x, cudaSuccess, "batch staging");
  if (rc) return rc;
  x->loaded_rows = rows;
  x->loaded_nnz = nnz;
  x->loaded_lab = L;
  return AS_OK;
}

int as_load_batch_csr(as_ctx *x, int32_t rows, const int64_t *row_ptr, const int32_t *col,
                      const float *val, const int64_t *lab_ptr, const int32_t *lab) {
  AS_GUARD(x);
  const int bi = x->b_all[x->cfg.rank];
  if (rows < 1 || rows > bi) return as_fail(AS_E_INVALID, "rows=%d not in [1, b_i=%d]", rows, bi);
  const int rc = stage_batch(x, rows, row_ptr, col, val, lab_ptr, lab);
  if (rc) return rc;
  x->has_batch = true;
  return AS_OK;
}

int as_eval_top1(as_ctx *x, int32_t rows, const int64_t *row_ptr, const int32_t *col, const float *val,
                 const int64_t *lab_ptr, const int32_t *lab, int32_t *top1_out, int64_t *hits_out) {
  AS_GUARD(x);
  if (rows < 1 || rows > x->cfg.b_max) return as_fail(AS_E_INVALID, "rows=%d not in [1, b_max=%d]", rows, x->cfg.b_max);
  int rc = stage_batch(x, rows, row_ptr, col, val, lab_ptr, lab);
  if (rc) return rc;
  x->has_batch = false;                     // the batch buffers now hold the evaluation rows
  const Dims &D = x->D;
  cudaStream_t s = x->stream;
  StepDesc *d = x->desc;
  const float *W1 = x->w, *b1 = x->w + D.d * D.h, *W2T = b1 + D.h, *b2 = W2T + D.C * D.h;
  // forward: H = ReLU(X W1 + b1) (a4), then the row argmax of z = H W2T^T + b2
  x->launches += 3;
  as::launch_spmm_chunked(s, D.h, x->num_sms, d, D.bpad, D.nnz_cap, x->row_ptr, x->col, x->val, x->rid,
                          W1, b1, x->Hf, x->Hb, x->seg_part, x->arrive);
  int slots = 1;
  if (x->cfg.precision == AS_BF16) {
    as::launch_out_top1_tc(s, x->plan, d, b2, x->pm, (int *)x->pl);
    slots = 2 * as::tc_fwd_splits_host(x->plan, rows);   // k_out_top1: one slot per (split, WG)
  } else {
    x->launches += 1;
    as::launch_gemm_f32(s, D.b_max, (int)D.C, D.h, x->Hf, D.h, 1, W2T, 1, D.h, x->Z, D.C, b2, 1, nullptr,
                        &d->rows);
    as::launch_row_argmax_f32(s, d, D.b_max, (int)D.C, x->Z, x->pm, (int *)x->pl);
  }
  cudaMemsetAsync(x->hits, 0, 8, s);
  as::launch_top1_combine(s, d, slots, D.bpad, x->pm, (const int *)x->pl, x->lab_ptr, x->lab, x->top1,
                          x->hits);
  rc = cuda_check(x, cudaSuccess, "eval launch");
  if (rc) return rc;
  if (top1_out) cudaMemcpyAsync(top1_out, x->top1, 4 * (size_t)rows, cudaMemcpyDeviceToHost, s);
  unsigned long long h = 0;
  cudaMemcpyAsync(&h, x->hits, 8, cudaMemcpyDeviceToHost, s);
  cudaEventRecord(x->ev_stage_free[x->cur_stage], s);
  rc = cuda_check(x, cudaStreamSynchronize(s), "eval");
  if (rc) return rc;
  if (hits_out) *hits_out = (int64_t)h;
  return AS_OK;
}

int as_dataset_bytes(int64_t n, int64_t nnz, int64_t L, size_t *bytes) {
  if (n < 1 || nnz < 0 || L < n || !bytes) return as_fail(AS_E_INVALID, "bad dataset sizes");
  Layout Lo;
  Lo.add(8 * (n + 1));
  Lo.add(4 * nnz);
  Lo.add(4 * nnz);
  Lo.add(8 * (n + 1));
  Lo.add(4 * L);
  Lo.add(8 * n);
  *bytes = Lo.total;
  return AS_OK;
}

int as_dataset_upload(as_ctx *x, void *dev_buf, size_t dev_bytes, int64_t n,
                      const int64_t *row_ptr, const int32_t *col, const float *val,
                      const int64_t *lab_ptr, const int32_t *lab, const int64_t *order) {
  AS_GUARD(x);
  if (n < 1 || !row_ptr || !lab_ptr) return as_fail(AS_E_INVALID, "bad dataset");
  if (row_ptr[0] != 0 || lab_ptr[0] != 0) return as_fail(AS_E_INVALID, "dataset pointers must start at 0");
  int64_t nnz = 0, L = 0;
  int rc = validate_csr(x, n, row_ptr, col, val, lab_ptr, lab, &nnz, &L);
  if (rc) return rc;
  if (order)
    for (int64_t i = 0; i < n; ++i)
      if (order[i] < 0 || order[i] >= n) return as_fail(AS_E_INVALID, "order[%lld] out of range", (long long)i);
  size_t need = 0;
  as_dataset_bytes(n, nnz, L, &need);
  if (!dev_buf || dev_bytes < need) return as_fail(AS_E_OOM, "dataset buffer too small: need %zu", need);
  Layout Lo;
  uint8_t *b = (uint8_t *)dev_buf;
  int64_t *drp = (int64_t *)(b + Lo.add(8 * (n + 1)));
  int32_t *dcol = (int32_t *)(b + Lo.add(4 * nnz));
  float *dval = (float *)(b + Lo.add(4 * nnz));
  int64_t *dlp = (int64_t *)(b + Lo.add(8 * (n + 1)));
  int32_t *dlab = (int32_t *)(b + Lo.add(4 * L));
  int64_t *dord = (int64_t *)(b + Lo.add(8 * n));
  cudaStream_t s = x->stream;
  cudaMemcpyAsync(drp, row_ptr, 8 * (n + 1), cudaMemcpyHostToDevice, s);
  if (nnz) cudaMemcpyAsync(dcol, col, 4 * nnz, cudaMemcpyHostToDevice, s);
  if (nnz) cudaMemcpyAsync(dval, val, 4 * nnz, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(dlp, lab_ptr, 8 * (n + 1), cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(dlab, lab, 4 * L, cudaMemcpyHostToDevice, s);
  if (order) cudaMemcpyAsync(dord, order, 8 * n, cudaMemcpyHostToDevice, s);
  rc = cuda_check(x, cudaStreamSynchronize(s), "dataset upload");
  if (rc) return rc;
  x->ds_row_ptr = drp; x->ds_col = dcol; x->ds_val = dval; x->ds_lab_ptr = dlp; x->ds_lab = dlab;
  x->ds_order = order ? dord : nullptr;
  x->ds_n = n;
  x->ds_mean_nnz = (double)nnz / (double)n;
  x->ds_rp_host.assign(row_ptr, row_ptr + n + 1);
  x->ds_lp_host.assign(lab_ptr, lab_ptr + n + 1);
  x->ds_mean_lab = (double)L / (double)n;
  return AS_OK;
}

int as_load_batch_stream(as_ctx *x, int64_t pos, int32_t rows) {
  AS_GUARD(x);
  if (!x->ds_row_ptr) return as_fail(AS_E_STATE, "no resident dataset (as_dataset_upload)");
  const int bi = x->b_all[x->cfg.rank];
  if (rows < 1 || rows > bi) return as_fail(AS_E_INVALID, "rows=%d not in [1, b_i=%d]", rows, bi);
  if (pos < 0) return as_fail(AS_E_INVALID, "pos < 0");
  // gathered on the main stream into the staging block the step before last
  // has released (a gather on the copy stream, overlapping the previous step,
  // measured slower: its kernels contend with the dW1 / SpMM of the step)
  const int k = x->stage_next;
  x->stage_next ^= 1;
  use_stage(x, k, nullptr);
  cudaStreamWaitEvent(x->stream, x->ev_stage_free[k], 0);
  ph_begin(x, AS_PH_BATCH);
  const int64_t p0 = pos % x->ds_n;
  static const bool no_slice = getenv("ADASGD_NO_SLICE") && atoi(getenv("ADASGD_NO_SLICE")) > 0;
  if (!x->ds_order && p0 + rows <= x->ds_n && !no_slice) {
    // contiguous slice of the resident dataset: features and labels in place
    x->col = const_cast<int32_t *>(x->ds_col) + x->ds_rp_host[p0];
    x->val = const_cast<float *>(x->ds_val) + x->ds_rp_host[p0];
    x->lab = const_cast<int32_t *>(x->ds_lab) + x->ds_lp_host[p0];
    x->launches += 1;
    static const bool slice_main = getenv("ADASGD_SLICE_MAIN") && atoi(getenv("ADASGD_SLICE_MAIN")) > 0;
    if (slice_main) {
      as::launch_slice_batch(x->stream, x->ds_row_ptr, x->ds_lab_ptr, p0, rows, x->row_ptr, x->lab_ptr, x->rid,
                             x->lrid, x->desc, x->D.nnz_cap, x->D.lab_cap);
    } else {                                  // on the copy stream, overlapping the previous step
      cudaStreamWaitEvent(x->cp_s, x->ev_stage_free[k], 0);
      as::launch_slice_batch(x->cp_s, x->ds_row_ptr, x->ds_lab_ptr, p0, rows, x->row_ptr, x->lab_ptr, x->rid,
                             x->lrid, x->desc, x->D.nnz_cap, x->D.lab_cap);
      cudaEventRecord(x->ev_copied[k], x->cp_s);
      cudaStreamWaitEvent(x->stream, x->ev_copied[k], 0);
    }
  } else {
    x->launches += 2;
    as::launch_gather_batch(x->stream, x->ds_row_ptr, x->ds_col, x->ds_val, x->ds_lab_ptr, x->ds_lab,
                            x->ds_order, x->ds_n, pos, rows, x->row_ptr, x->col, x->val, x->lab_ptr,
                            x->lab, x->ids, x->rid, x->lrid, x->desc, x->D.nnz_cap, x->D.lab_cap);
  }
  ph_end(x, AS_PH_BATCH);
  const int rc = cuda_check(x, cudaSuccess, "gather batch");
  if (rc) return rc;
  x->loaded_rows = rows;
  x->loaded_nnz = (long long)(x->ds_mean_nnz * rows + 0.5);
  x->loaded_lab = (long long)(x->ds_mean_lab * rows + 0.5);
  x->has_batch = true;
  return AS_OK;
}

int as_train_step(as_ctx *x, float *loss_out) {
  AS_GUARD(x);
  if (!x->has_batch) return as_fail(AS_E_STATE, "no batch loaded");
  const Dims &D = x->D;
  cudaStream_t s = x->stream;
  StepDesc *d = x->desc;
  const int rows = x->loaded_rows;
  const float lr = x->lr;
  const bool dbg = (x->cfg.flags & AS_FLAG_DEBUG_GRADS) != 0;
  float *W1 = x->w, *b1 = x->w + D.d * D.h, *W2T = b1 + D.h, *b2 = W2T + D.C * D.h;
  // a7 inside pass 2's idle warps (one warp per feature segment) pays when its
  // work hides in pass 2's runtime: measured on B200, Amazon-670K (78K entries,
  // C = 670K, W1 in L2): step -1.7%; WikiLSHTC-325K (43K entries, C = 325K, W1
  // 828 MB: HBM-latency-bound gathers): +0.5%; Delicious-200K (309K entries,
  // C = 205K): +72%.  Rule: entries <= 0.15 C (0.075 C when W1 exceeds L2).
  static const bool no_fuse = getenv("ADASGD_NO_DW1_FUSE") && atoi(getenv("ADASGD_NO_DW1_FUSE")) > 0;
  const bool w1_in_l2 = 4.0 * (double)D.d * D.h <= 100e6;
  // the label terms in pass 1's idle warps unless ADASGD_LT_SEPARATE=1 (or the
  // AS_X_LABSIDE experiment build)
  static const bool lt_sep_env = getenv("ADASGD_LT_SEPARATE") && atoi(getenv("ADASGD_LT_SEPARATE")) > 0;
  // measured on B200: Amazon-670K (5 labels / row, C = 670K) step -0.25%,
  // Delicious-200K (75 labels / row, C = 205K) +2.6% when fused: fuse when the
  // batch has at most 0.05 C labels
#ifdef AS_X_LABSIDE
  const bool lt_sep = true;
#else
  // h = 256: pass 1 runs one softmax warpgroup, so six warps per CTA (the idle
  // second warpgroup too) carry the label terms: fused up to labels <= C
  const bool lt_sep = lt_sep_env || (double)x->loaded_lab > (D.h == 256 ? 1.0 : 0.05) * (double)D.C;
#endif
  const bool dw1_fused = x->cfg.precision == AS_BF16 && as::tc_fuses_dw1(D.h) && !no_fuse &&
                         (double)x->loaded_nnz <= (w1_in_l2 ? 0.15 : 0.075) * (double)D.C;

  // a3: batch transposes (feature-sorted CSC for dW1, label-sorted for dW2) on
  // the side stream, concurrent with a4/a5; joined before a6 and a7
  cudaStream_t ss = x->side;
  const as::TrArgs tr = tr_args(x);
  auto fork_transposes = [&]() {
    cudaEventRecord(x->ev_fork, s);
    cudaStreamWaitEvent(ss, x->ev_fork, 0);
    ph_begin(x, AS_PH_TRANSPOSE, ss);
#ifdef AS_X_LABSIDE
    if (x->cfg.precision == AS_BF16) {        // label terms first on the side stream
      x->launches += 1;
      as::launch_label_terms(ss, D.h, d, D.b_max, x->lab_ptr, x->lab, x->Hf, W2T, b2, x->zsum, x->labW);
      cudaEventRecord(x->ev_lab, ss);
    }
#endif
    x->launches += 3;
    as::launch_transposes(ss, tr);
    ph_end(x, AS_PH_TRANSPOSE, ss);
    cudaEventRecord(x->ev_join, ss);
  };
  // fork point of the transposes (experiment switch): 1 = after the SpMM, so
  // the latency-bound SpMM runs alone and the transposes fill the SMs pass 1
  // has not claimed yet and the combine kernels
  // Runtime default: 1, except when the output layer is small (every class
  // block fits one CTA: C <= 128 SMs, AmazonCat-13K) -- there the transposes
  // would gate pass 2, so they fork before the SpMM (measured: AmazonCat-13K
  // step 0.1247 -> 0.1193 ms; Amazon-670K +0.7% with the early fork)
#ifdef AS_X_FORK
  const int fork_at = AS_X_FORK;
#else
  const int fork_at = D.C <= 128LL * x->num_sms ? 0 : 1;
#endif
  if (fork_at == 0) fork_transposes();
  // a4: SpMM forward
  ph_begin(x, AS_PH_SPMM);
  x->launches += 1;
  as::launch_spmm_chunked(s, D.h, x->num_sms, d, D.bpad, D.nnz_cap, x->row_ptr, x->col, x->val, x->rid, W1, b1,
                          x->Hf, x->Hb, x->seg_part, x->arrive);
  ph_end(x, AS_PH_SPMM);
  if (fork_at == 1) fork_transposes();
  if (x->cfg.precision == AS_BF16) {
    // a5: pass 1 (tcgen05) + combine -> LSE, loss, dA
    ph_begin(x, AS_PH_OUT_FWD);
    x->launches += 1;
    as::LtArgs lt{};
    if (!lt_sep) lt = {x->lab_ptr, x->lab, x->Hf, W2T, b2, x->zsum, x->labW};
    as::launch_out_fwd_tc(s, x->plan, d, b2, x->pm, x->pl, x->pO, lt);
    ph_end(x, AS_PH_OUT_FWD);
    if (fork_at == 2) fork_transposes();
    ph_begin(x, AS_PH_COMBINE);
    // label terms of the loss and of dH (R3), then the split combine -> LSE,
    // loss, dA, and db1 with b1's SGD fused (ordered last-arriver column sums)
#ifdef AS_X_LABSIDE
    x->launches += 1;
    cudaStreamWaitEvent(s, x->ev_lab, 0);
#else
    x->launches += 1;
    if (lt_sep) {                             // (else pass 1's idle warps computed them)
      x->launches += 1;
      as::launch_label_terms(s, D.h, d, D.b_max, x->lab_ptr, x->lab, x->Hf, W2T, b2, x->zsum, x->labW);
    }
#endif
    as::launch_combine_bf16(s, D.h, d, D.b_max, D.bpad, as::tc_fwd_splits_host(x->plan, rows), x->pm,
                            x->pl, x->pO, x->labW, x->zsum, x->Hf, x->lab_ptr, x->lse2, x->lsep, x->wrow,
                            x->lossr, x->dA, x->db1p, x->db1cnt, b1, lr, dbg ? x->dbg_db1 : nullptr,
                            dbg ? x->dbg_dHs : nullptr, as::tc_fold(D.h) ? x->Hx : nullptr);
    ph_end(x, AS_PH_COMBINE);
    cudaStreamWaitEvent(s, x->ev_join, 0);   // label transpose ready
    // a6: pass 2 (tcgen05): dW2T, db2 and the fused SGD update of W2T, b2;
    // at h = 128 its two idle warps per CTA also run a7 (dW1 + SGD of W1,
    // which touches none of pass 2's data)
    ph_begin(x, AS_PH_OUT_BWD);
    x->launches += 1;
    as::Dw1Args dw{};
    if (dw1_fused) {
      dw.desc = d; dw.seg_ptr = x->fseg_ptr; dw.seg_row = x->fseg_row; dw.seg_key = x->fseg_id;
      dw.seg_val = x->fseg_val; dw.dA = x->dA; dw.W1 = W1; dw.lr = lr; dw.dbg = dbg ? x->dbg_dW1 : nullptr;
    }
    as::launch_out_bwd_tc(s, x->plan, d, x->lsep, x->cls_lab, x->lbits, D.bw, x->wrow,
                          W2T, b2, x->w2b, lr, dbg ? x->dbg_dW2 : nullptr,
                          dbg ? x->dbg_db2 : nullptr, dw);
    ph_end(x, AS_PH_OUT_BWD);
  } else {
    // fp32 parity mode: logits materialised
    if (fork_at == 2) fork_transposes();
    const long long C = D.C;
    ph_begin(x, AS_PH_OUT_FWD);
    x->launches += 1 + 1 + 1 + 2;
    as::launch_label_terms(s, D.h, d, D.b_max, x->lab_ptr, x->lab, x->Hf, W2T, b2, x->zsum, x->labW);
    as::launch_gemm_f32(s, D.b_max, (int)C, D.h, x->Hf, D.h, 1, W2T, 1, D.h, x->Z, C, b2, 1,
                        nullptr, &d->rows);
    as::launch_row_lse(s, d, D.b_max, (int)C, x->Z, x->lse2);
    if (dbg) {                                // softmax part of dH on its own (AS_DBG_DHSOFT)
      as::launch_softmax_grad(s, d, D.b_max, (int)C, x->lab_ptr, x->lab, x->Z, x->lse2, 1);
      as::launch_gemm_f32(s, D.b_max, D.h, (int)C, x->Z, C, 1, W2T, D.h, 1, x->dbg_dHs, D.h, nullptr,
                          D.splitk, x->splitk_tmp, &d->rows);
      as::launch_softmax_grad(s, d, D.b_max, (int)C, x->lab_ptr, x->lab, x->Z, x->lse2, 2);
    } else {
      as::launch_softmax_grad(s, d, D.b_max, (int)C, x->lab_ptr, x->lab, x->Z, x->lse2, 3);
    }
    ph_end(x, AS_PH_OUT_FWD);
    cudaStreamWaitEvent(s, x->ev_join, 0);   // transposes ready
    ph_begin(x, AS_PH_OUT_BWD);
    x->launches += (D.splitk > 1 ? 2 : 1) + 1 + 1 + 2 + 1 + (dbg ? 0 : 0);
    as::launch_gemm_f32(s, D.b_max, D.h, (int)C, x->Z, C, 1, W2T, D.h, 1, x->dH, D.h, nullptr,
                        D.splitk, x->splitk_tmp, &d->rows);
    as::launch_gemm_f32_kdev(s, (int)C, D.h, D.b_max, x->Z, 1, C, x->Hf, D.h, 1, x->dW2, D.h,
                             &d->rows);
    as::launch_finish_f32(s, D.h, d, D.b_max, x->dH, x->Hf, x->zsum, x->lse2, x->lossr, x->dA, x->labW, nullptr);
    as::launch_colsum_sgd(s, d, D.b_max, (int)C, x->Z, C, b2, lr, dbg ? x->dbg_db2 : nullptr);
    as::launch_colsum_sgd(s, d, D.b_max, D.h, x->dA, D.h, b1, lr, dbg ? x->dbg_db1 : nullptr);
    if (dbg) cudaMemcpyAsync(x->dbg_dW2, x->dW2, 4 * (size_t)C * D.h, cudaMemcpyDeviceToDevice, s);
    as::launch_sgd_dense(s, C * D.h, W2T, x->dW2, lr, x->w2b);
    ph_end(x, AS_PH_OUT_BWD);
  }
  // a7: first-layer gradient (deterministic segmented reduction) + SGD,
  // unless pass 2 ran it
  ph_begin(x, AS_PH_DW1);
  if (!dw1_fused) {
    x->launches += 1;
    as::launch_dw1_chunked(s, D.h, x->num_sms, d, D.nnz_cap, x->fseg_id, x->fseg_of, x->fseg_ptr, x->fseg_row,
                           x->fseg_val, x->dA, W1, lr, x->seg_part, x->arrive,
                           dbg ? x->dbg_dW1 : nullptr);
  }
  if (loss_out || dbg) {
    x->launches += 1;
    as::launch_loss_mean(s, d, x->lossr, x->loss);
  }
  // transpose state reset on the side stream after the step's last reader
  cudaEventRecord(x->ev_tail, s);
  cudaStreamWaitEvent(ss, x->ev_tail, 0);
  x->launches += 1;
  as::launch_tr_reset(ss, tr, x->num_sms);
  // the host-staged batch block may be refilled once the reset (the last
  // reader of its StepDesc) is done
  cudaEventRecord(x->ev_stage_free[x->cur_stage], ss);
  ph_end(x, AS_PH_DW1);
  int rc = cuda_check(x, cudaSuccess, "train step launch");
  if (rc) return rc;
  if (loss_out) {
    rc = cuda_check(x, cudaMemcpyAsync(loss_out, x->loss, 4, cudaMemcpyDeviceToHost, s), "loss D2H");
    if (!rc) rc = cuda_check(x, cudaStreamSynchronize(s), "train step");
  }
  return rc;
}

int as_set_batch_sizes(as_ctx *x, const int32_t *b, const float *lr) {
  AS_GUARD(x);
  if (!b || !lr) return as_fail(AS_E_INVALID, "b / lr is NULL");
  for (int i = 0; i < x->cfg.world; ++i)
    if (b[i] < x->cfg.b_min || b[i] > x->cfg.b_max)
      return as_fail(AS_E_INVALID, "b[%d]=%d not in [b_min, b_max]", i, b[i]);
  if (!(lr[x->cfg.rank] > 0.f)) return as_fail(AS_E_INVALID, "lr must be > 0");
  x->b_all.assign(b, b + x->cfg.world);
  x->lr = lr[x->cfg.rank];
  return AS_OK;
}

// ---------------------------------------------------------------------------
// Merge (steps a9-a13).  The weights alpha live on the device (alpha_d fp64,
// alpha_f fp32): Alg. 2 runs in a one-thread kernel on the all-gathered norms
// (the same code as the host export), so no host synchronisation is needed.
static as::PeerArgs peer_args(const as_ctx *x) {
  as::PeerArgs a{};
  a.N = x->cfg.world;
  a.rank = x->cfg.rank;
  a.P = x->D.P;
  a.w2_off = x->D.d * x->D.h + x->D.h;
  a.w2_len = x->D.C * x->D.h;
  a.gamma = (float)x->cfg.gamma;
  a.off_w = (uint8_t *)x->w - x->arena;
  a.off_wbarp = (uint8_t *)x->wbarp - x->arena;
  a.off_w2b = (uint8_t *)x->w2b - x->arena;
  a.off_flags = (uint8_t *)x->p2p_flags - x->arena;
  a.off_norms = (uint8_t *)x->norms_all - x->arena;
  for (int k = 0; k < a.N; ++k) a.base[k] = x->peer_base[k];
  return a;
}

// cross-rank barrier over peer memory (AS_MERGE_P2P); my_norm (device,
// nullable) is published into every rank's norms_all[rank] first
static void p2p_barrier(as_ctx *x, const double *my_norm) {
  as::PeerArgs a = peer_args(x);
  a.epoch = ++x->p2p_epoch;
  x->launches += 1;
  as::launch_p2p_barrier(x->stream, a, my_norm);
}

// a11-a13 with the weights already in alpha_f (device), all replicas' training
// complete (N > 1: after the first barrier / inside the NCCL stream order):
// prescale, all-reduce, momentum + reset + shadow, wbar / wbar_p rotation.
static int merge_apply_dev(as_ctx *x, float alpha_host_me /* NaN: unknown */) {
  const int N = x->cfg.world;
  const Dims &D = x->D;
  cudaStream_t s = x->stream;
  const long long w2_off = D.d * D.h + D.h, w2_len = D.C * D.h;
  if (x->cfg.merge_backend == AS_MERGE_P2P && N > 1) {
    // ONE fused kernel over peer memory: sum alpha_k w_k of this rank's slice
    // from every replica, momentum, pushed into every rank
    x->launches += 1;
    as::launch_merge_p2p(s, peer_args(x), x->alpha_f, x->wbar, x->wbarp);
    p2p_barrier(x, nullptr);               // every slice has landed everywhere
    std::swap(x->wbar, x->wbarp);
    return cuda_check(x, cudaSuccess, "p2p merge launch");
  }
  // NCCL (N > 1, or a one-rank communicator with ADASGD_NCCL_SELF=1) or local
  // (N = 1).  N > 1: the prescale rides inside the all-reduce (NCCL PreMulSum
  // with the weight read from device memory), saving an 8P-byte pass; plain
  // prescale + sum if the op cannot be created.
  const bool use_nccl = x->comm != nullptr;
  // Partitioned merge ("multi-stream" transfer
  // overlapping the combine): the all-reduce runs chunk by chunk on the
  // communication stream and the momentum kernel of chunk c runs on the main
  // stream as soon as chunk c is reduced, overlapping the reduction of c+1.
  // ADASGD_MERGE_CHUNKS=k forces k chunks (also at N = 1, without a reduction:
  // tests the chunk bookkeeping on one GPU); default 8 for N > 1, 1 at N = 1.
  const int K = x->merge_chunks > 0 ? x->merge_chunks : (N > 1 ? 8 : 1);
  ncclRedOp_t premul = ncclSum;
  bool have_premul = false;
  if (use_nccl) {
    have_premul = ncclRedOpCreatePreMulSum(&premul, x->alpha_f + x->cfg.rank, ncclFloat, ncclScalarDevice,
                                           x->comm) == ncclSuccess;
    if (!have_premul) {
      x->launches += 1;
      as::launch_scale_dev(s, x->w, D.P, x->alpha_f + x->cfg.rank);
      premul = ncclSum;
    }
  } else if (!(alpha_host_me == 1.0f)) {     // N = 1 without a communicator
    x->launches += 1;
    if (alpha_host_me == alpha_host_me) as::launch_scale(s, x->w, D.P, alpha_host_me);
    else as::launch_scale_dev(s, x->w, D.P, x->alpha_f + x->cfg.rank);
  }
  x->launches += K;
  if (use_nccl) {                             // training, weights and any prescale are done
    cudaEventRecord(x->ev_mg[0], s);
    cudaStreamWaitEvent(x->comm_s, x->ev_mg[0], 0);
  }
  for (int c = 0; c < K; ++c) {
    // chunk borders on multiples of 4 floats (the vectorised momentum kernel)
    const long long off = (D.P * c / K) & ~3ll, end = c + 1 == K ? D.P : (D.P * (c + 1) / K) & ~3ll,
                    len = end - off;
    if (use_nccl) {
      const ncclResult_t r = ncclAllReduce(x->w + off, x->w + off, len, ncclFloat, premul, x->comm, x->comm_s);
      if (r != ncclSuccess) {
        if (have_premul) ncclRedOpDestroy(premul, x->comm);
        x->sticky = AS_E_NCCL;
        return as_fail(AS_E_NCCL, "ncclAllReduce: %s", ncclGetErrorString(r));
      }
      cudaEventRecord(x->ev_mg[1 + (c & 1)], x->comm_s);
      cudaStreamWaitEvent(s, x->ev_mg[1 + (c & 1)], 0);
    }
    as::launch_momentum(s, x->w + off, x->wbarp + off, x->wbar + off, len, (float)x->cfg.gamma, w2_off - off,
                        w2_len, x->w2b);
  }
  if (have_premul) ncclRedOpDestroy(premul, x->comm);
  std::swap(x->wbar, x->wbarp);
  return cuda_check(x, cudaSuccess, "merge launch");
}

static bool merge_transport_ready(const as_ctx *x) {
  if (x->cfg.world == 1) return true;
  return x->cfg.merge_backend == AS_MERGE_P2P ? x->p2p_ready : x->comm != nullptr;
}

// caller-given weights (host) -> device, then a11-a13
static int merge_given(as_ctx *x, const double *alpha) {
  const int N = x->cfg.world;
  as::MergeWeightArgs wa{};
  wa.N = N;
  wa.mode = 2;
  for (int i = 0; i < N; ++i) wa.given[i] = alpha[i];
  if (x->cfg.merge_backend == AS_MERGE_P2P && N > 1) p2p_barrier(x, nullptr);   // training done everywhere
  const bool need_dev = x->comm != nullptr || N > 1;
  if (need_dev) {
    x->launches += 1;
    as::launch_alg2(x->stream, wa, x->norms_all, x->alpha_d, x->alpha_f, x->pert_dev);
  }
  return merge_apply_dev(x, need_dev ? NAN : (float)alpha[x->cfg.rank]);
}

int as_merge(as_ctx *x, const int32_t *u, const int32_t *b, double *alpha_out,
             int32_t *perturbed_out) {
  AS_GUARD(x);
  if (!u || !b) return as_fail(AS_E_INVALID, "u / b is NULL");
  const int N = x->cfg.world;
  for (int i = 0; i < N; ++i)
    if (u[i] < 0 || b[i] < 1) return as_fail(AS_E_INVALID, "need u[i] >= 0 and b[i] >= 1 (i = %d)", i);
  if (!merge_transport_ready(x))
    return as_fail(AS_E_STATE, x->cfg.merge_backend == AS_MERGE_P2P
                                   ? "as_merge: peer mappings not open (as_p2p_export / as_p2p_open)"
                                   : "as_merge needs an NCCL ctx (use as_group_merge in local-group mode)");
  const Dims &D = x->D;
  cudaStream_t s = x->stream;
  ph_begin(x, AS_PH_MERGE);
  int rc = AS_OK;
  int32_t pert_host = 0;
  double alpha1 = 1.0;
  // R14 literal with one replica: r = s = 0 and line 9 applies when the
  // replica is regular, alpha = (1 + delta)(1 - delta): the norm is needed
  const bool lit1 = N == 1 && x->cfg.algo == AS_ALGO_ADAPTIVE && (x->cfg.flags & AS_FLAG_R14_LITERAL);
  if (N == 1 && !lit1) {
    // Alg. 2 with one replica: line 3 gives alpha = b / b = 1 and r = s, so
    // the perturbation is skipped whatever the norm (R14); the comparison
    // methods' 1/N is 1 too: no norm pass, no host synchronisation
    rc = merge_given(x, &alpha1);
  } else {
    as::MergeWeightArgs wa{};
    wa.N = N;
    wa.mode = x->cfg.algo == AS_ALGO_ADAPTIVE ? 0 : 1;     // comparison methods: 1/N
    wa.norm_mode = ((x->cfg.flags & AS_FLAG_NORM_UB) ? 1 : 0) | ((x->cfg.flags & AS_FLAG_R14_LITERAL) ? 2 : 0);
    wa.delta = x->cfg.delta;
    wa.pert_thr = x->cfg.pert_thr;
    for (int i = 0; i < N; ++i) { wa.u[i] = u[i]; wa.b[i] = b[i]; }
    const bool adaptive = wa.mode == 0;
    if (adaptive) {                           // a9: replica norm (fp64, fixed order)
      x->launches += 2;
      as::launch_sumsq(s, x->w, D.P, x->norm_part, kNormBlocks, x->norm_dev,
                       (x->cfg.flags >> AS_NORM_METRIC_SHIFT) & 3);
    }
    if (N == 1) {                             // (lit1) the one norm is the table
      rc = cuda_check(x, cudaMemcpyAsync(x->norms_all, x->norm_dev, 8, cudaMemcpyDeviceToDevice, s), "norm copy");
      if (rc) return rc;
    } else if (x->cfg.merge_backend == AS_MERGE_P2P) {
      p2p_barrier(x, adaptive ? x->norm_dev : nullptr);   // norms all-gathered; training done everywhere
    } else if (adaptive) {
      const ncclResult_t r = ncclAllGather(x->norm_dev, x->norms_all, 1, ncclDouble, x->comm, s);
      if (r != ncclSuccess) { x->sticky = AS_E_NCCL; return as_fail(AS_E_NCCL, "ncclAllGather: %s", ncclGetErrorString(r)); }
    }
    x->launches += 1;                         // a10: Alg. 2 on the device
    as::launch_alg2(s, wa, x->norms_all, x->alpha_d, x->alpha_f, x->pert_dev);
    rc = merge_apply_dev(x, NAN);
  }
  ph_end(x, AS_PH_MERGE);
  if (rc) return rc;
  rc = cuda_check(x, cudaSuccess, "merge launch");
  if (rc) return rc;
  if (N == 1 && !lit1) {
    if (alpha_out) alpha_out[0] = alpha1;
    if (perturbed_out) *perturbed_out = 0;
  } else if (alpha_out || perturbed_out) {
    std::vector<double> al(N);
    rc = cuda_check(x, cudaMemcpyAsync(al.data(), x->alpha_d, 8 * N, cudaMemcpyDeviceToHost, s), "alpha D2H");
    if (!rc) rc = cuda_check(x, cudaMemcpyAsync(&pert_host, x->pert_dev, 4, cudaMemcpyDeviceToHost, s), "pert D2H");
    if (!rc) rc = cuda_check(x, cudaStreamSynchronize(s), "merge sync");
    if (rc) return rc;
    if (alpha_out) std::copy(al.begin(), al.end(), alpha_out);
    if (perturbed_out) *perturbed_out = pert_host;
  }
  return AS_OK;
}

int as_merge_weighted(as_ctx *x, const double *alpha) {
  AS_GUARD(x);
  if (!alpha) return as_fail(AS_E_INVALID, "alpha is NULL");
  for (int i = 0; i < x->cfg.world; ++i)
    if (!(alpha[i] == alpha[i]) || alpha[i] < 0.0 || alpha[i] > 1e6)
      return as_fail(AS_E_INVALID, "alpha[%d] not a finite weight >= 0", i);
  if (!merge_transport_ready(x)) return as_fail(AS_E_STATE, "as_merge_weighted: merge transport not ready");
  ph_begin(x, AS_PH_MERGE);
  const int rc = merge_given(x, alpha);
  ph_end(x, AS_PH_MERGE);
  return rc;
}

// ---- AS_MERGE_P2P setup ----------------------------------------------------
typedef CUresult (*PFN_getAddressRange)(CUdeviceptr *, size_t *, CUdeviceptr);

struct P2PRecord {
  uint32_t magic;
  int32_t rank, world, device;
  uint64_t offset;                // workspace offset inside its allocation
  uint64_t bytes;                 // workspace bytes
  cudaIpcMemHandle_t handle;      // 64 bytes
  uint8_t pad[AS_P2P_EXPORT_BYTES - 32 - sizeof(cudaIpcMemHandle_t)];
};
static_assert(sizeof(P2PRecord) == AS_P2P_EXPORT_BYTES, "P2P record size");
constexpr uint32_t kP2PMagic = 0x41535032u;   // "ASP2"

int as_p2p_export(as_ctx *x, void *out) {
  AS_GUARD(x);
  if (!out) return as_fail(AS_E_INVALID, "out is NULL");
  static PFN_getAddressRange range = nullptr;
  if (!range) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return as_fail(AS_E_CUDA, "cuMemGetAddressRange entry point missing");
    range = (PFN_getAddressRange)p;
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, (CUdeviceptr)x->arena) != CUDA_SUCCESS)
    return as_fail(AS_E_CUDA, "cuMemGetAddressRange failed on the workspace");
  P2PRecord r{};
  r.magic = kP2PMagic;
  r.rank = x->cfg.rank;
  r.world = x->cfg.world;
  r.device = x->cfg.device;
  r.offset = (uint64_t)((CUdeviceptr)x->arena - base);
  r.bytes = x->cfg.workspace_bytes;
  const int rc = cuda_check(x, cudaIpcGetMemHandle(&r.handle, (void *)base), "cudaIpcGetMemHandle");
  if (rc) return rc;
  memcpy(out, &r, sizeof(r));
  return AS_OK;
}

int as_p2p_open(as_ctx *x, const void *records) {
  AS_GUARD(x);
  if (!records) return as_fail(AS_E_INVALID, "records is NULL");
  if (x->cfg.merge_backend != AS_MERGE_P2P) return as_fail(AS_E_STATE, "ctx merge_backend is not AS_MERGE_P2P");
  if (x->p2p_ready) return as_fail(AS_E_STATE, "peer mappings already open");
  const int N = x->cfg.world;
  const P2PRecord *rec = (const P2PRecord *)records;
  for (int k = 0; k < N; ++k)
    if (rec[k].magic != kP2PMagic || rec[k].rank != k || rec[k].world != N ||
        rec[k].bytes != x->cfg.workspace_bytes)
      return as_fail(AS_E_INVALID, "P2P record %d invalid (magic / rank order / world / workspace size)", k);
  for (int k = 0; k < N; ++k) {
    if (k == x->cfg.rank) { x->peer_base[k] = x->arena; continue; }
    void *p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, rec[k].handle, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      for (int j = 0; j < k; ++j)
        if (j != x->cfg.rank && x->peer_map[j]) { cudaIpcCloseMemHandle(x->peer_map[j]); x->peer_map[j] = nullptr; }
      cudaGetLastError();
      return as_fail(AS_E_CUDA, "cudaIpcOpenMemHandle(rank %d): %s", k, cudaGetErrorString(e));
    }
    x->peer_map[k] = p;
    x->peer_base[k] = (uint8_t *)p + rec[k].offset;
  }
  x->p2p_ready = true;
  return AS_OK;
}

int as_replica_norm(as_ctx *x, int32_t metric, double *out) {
  AS_GUARD(x);
  if (!out || metric < AS_METRIC_L2_P || metric > AS_METRIC_L2) return as_fail(AS_E_INVALID, "bad arguments");
  x->launches += 2;
  as::launch_sumsq(x->stream, x->w, x->D.P, x->norm_part, kNormBlocks, x->norm_dev, metric);
  int rc = cuda_check(x, cudaMemcpyAsync(out, x->norm_dev, 8, cudaMemcpyDeviceToHost, x->stream), "norm D2H");
  if (!rc) rc = cuda_check(x, cudaStreamSynchronize(x->stream), "norm");
  return rc;
}

int as_group_merge(as_ctx *const *ctxs, int32_t n, const int32_t *u, const int32_t *b,
                   double *alpha_out, int32_t *perturbed_out) {
  if (!ctxs || n < 1 || !u || !b) return as_fail(AS_E_INVALID, "bad arguments");
  for (int i = 0; i < n; ++i) {
    AS_GUARD(ctxs[i]);
    if (ctxs[i]->cfg.world != n || ctxs[i]->cfg.rank != i)
      return as_fail(AS_E_INVALID, "ctx %d: need world == n and rank == index", i);
    if (ctxs[i]->D.P != ctxs[0]->D.P) return as_fail(AS_E_INVALID, "model sizes differ");
  }
  as_ctx *x0 = ctxs[0];
  const Dims &D = x0->D;
  std::vector<double> norms(n), alpha(n);
  int32_t pert = 0;
  int rc = AS_OK;
  if (x0->cfg.algo == AS_ALGO_ADAPTIVE) {
    for (int i = 0; i < n; ++i) {
      as_ctx *x = ctxs[i];
      cudaSetDevice(x->cfg.device);
      as::launch_sumsq(x->stream, x->w, D.P, x->norm_part, kNormBlocks, x->norm_dev, (x->cfg.flags >> AS_NORM_METRIC_SHIFT) & 3);
      rc = cuda_check(x, cudaMemcpyAsync(&norms[i], x->norm_dev, 8, cudaMemcpyDeviceToHost, x->stream), "norm");
      if (!rc) rc = cuda_check(x, cudaStreamSynchronize(x->stream), "norm sync");
      if (rc) return rc;
    }
    rc = as_sched_alg2_ex(n, u, b, norms.data(), x0->cfg.delta, x0->cfg.pert_thr,
                          ((x0->cfg.flags & AS_FLAG_NORM_UB) ? AS_NORM_UB : AS_NORM_UPDATES) |
                              ((x0->cfg.flags & AS_FLAG_R14_LITERAL) ? AS_NORM_R14_LITERAL : 0),
                          alpha.data(), &pert);
    if (rc) return rc;
  } else {
    for (int i = 0; i < n; ++i) alpha[i] = 1.0 / n;
  }
  std::vector<float> af(n);
  std::vector<const float *> reps(n);
  for (int i = 0; i < n; ++i) { af[i] = (float)alpha[i]; reps[i] = ctxs[i]->w; }
  // replicas on other devices are read through peer mappings (NVLink)
  for (int i = 1; i < n; ++i) {
    const int di = ctxs[i]->cfg.device, d0 = x0->cfg.device;
    if (di == d0) continue;
    int ok01 = 0;
    cudaDeviceCanAccessPeer(&ok01, d0, di);
    if (!ok01) return as_fail(AS_E_CUDA, "device %d cannot access device %d (peer access)", d0, di);
    cudaSetDevice(d0);
    cudaError_t e = cudaDeviceEnablePeerAccess(di, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_check(x0, e, "enable peer access");
    cudaSetDevice(di);
    e = cudaDeviceEnablePeerAccess(d0, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_check(ctxs[i], e, "enable peer access");
    cudaGetLastError();                      // clear a tolerated AlreadyEnabled
  }
  // the reduction on x0's stream waits for every replica's training (any algo)
  for (int i = 1; i < n; ++i) {
    cudaSetDevice(ctxs[i]->cfg.device);
    rc = cuda_check(ctxs[i], cudaEventRecord(ctxs[i]->ev_mg[0], ctxs[i]->stream), "merge event");
    if (rc) return rc;
    cudaSetDevice(x0->cfg.device);
    rc = cuda_check(x0, cudaStreamWaitEvent(x0->stream, ctxs[i]->ev_mg[0], 0), "merge wait");
    if (rc) return rc;
  }
  cudaSetDevice(x0->cfg.device);
  cudaMemcpyAsync(x0->alpha_dev, af.data(), 4 * n, cudaMemcpyHostToDevice, x0->stream);
  cudaMemcpyAsync(x0->reps_dev, reps.data(), 8 * n, cudaMemcpyHostToDevice, x0->stream);
  as::launch_group_reduce(x0->stream, x0->reps_dev, x0->alpha_dev, n, D.P, x0->wbar, x0->wbarp,
                          (float)x0->cfg.gamma);
  rc = cuda_check(x0, cudaStreamSynchronize(x0->stream), "group reduce");
  if (rc) return rc;
  const float *src = x0->wbarp;
  for (int i = 0; i < n; ++i) {
    as_ctx *x = ctxs[i];
    cudaSetDevice(x->cfg.device);
    as::launch_reset_from(x->stream, src, x->w, x->wbarp, D.P, D.d * D.h + D.h, D.C * D.h, x->w2b);
    rc = cuda_check(x, cudaStreamSynchronize(x->stream), "group reset");
    if (rc) return rc;
  }
  for (int i = 0; i < n; ++i) std::swap(ctxs[i]->wbar, ctxs[i]->wbarp);
  if (alpha_out) std::copy(alpha.begin(), alpha.end(), alpha_out);
  if (perturbed_out) *perturbed_out = pert;
  return AS_OK;
}

int as_get_params(as_ctx *x, int32_t which, float *host_out) {
  AS_GUARD(x);
  if (!host_out) return as_fail(AS_E_INVALID, "host_out is NULL");
  const float *src = which == AS_PARAMS_REPLICA ? x->w
                     : which == AS_PARAMS_GLOBAL ? x->wbar
                     : which == AS_PARAMS_GLOBAL_PREV ? x->wbarp : nullptr;
  if (!src) return as_fail(AS_E_INVALID, "bad `which`");
  int rc = cuda_check(x, cudaMemcpyAsync(host_out, src, 4 * (size_t)x->D.P, cudaMemcpyDeviceToHost, x->stream), "params D2H");
  if (!rc) rc = cuda_check(x, cudaStreamSynchronize(x->stream), "params sync");
  return rc;
}

int as_set_params(as_ctx *x, int32_t which, const float *host_in) {
  AS_GUARD(x);
  if (!host_in) return as_fail(AS_E_INVALID, "host_in is NULL");
  float *dst = which == AS_PARAMS_REPLICA ? x->w
               : which == AS_PARAMS_GLOBAL ? x->wbar
               : which == AS_PARAMS_GLOBAL_PREV ? x->wbarp : nullptr;
  if (!dst) return as_fail(AS_E_INVALID, "bad `which`");
  const Dims &D = x->D;
  int rc = cuda_check(x, cudaMemcpyAsync(dst, host_in, 4 * (size_t)D.P, cudaMemcpyHostToDevice, x->stream), "params H2D");
  if (!rc && which == AS_PARAMS_REPLICA)
    as::launch_f32_to_bf16(x->stream, x->w + D.d * D.h + D.h, x->w2b, D.C * D.h);
  if (!rc) rc = cuda_check(x, cudaStreamSynchronize(x->stream), "params sync");
  return rc;
}

int as_debug_get(as_ctx *x, int32_t which, void *host_out, size_t bytes, size_t *written) {
  AS_GUARD(x);
  if (!host_out || !written) return as_fail(AS_E_INVALID, "NULL output");
  cudaStream_t s = x->stream;
  StepDesc dd;
  int rc = cuda_check(x, cudaMemcpyAsync(&dd, x->desc, sizeof(dd), cudaMemcpyDeviceToHost, s), "desc");
  if (!rc) rc = cuda_check(x, cudaStreamSynchronize(s), "desc sync");
  if (rc) return rc;
  const Dims &D = x->D;
  const bool dbg = (x->cfg.flags & AS_FLAG_DEBUG_GRADS) != 0;
  std::vector<std::pair<const void *, size_t>> parts;
  std::vector<int32_t> head;
  switch (which) {
    case AS_DBG_H: parts.push_back({x->Hf, 4 * (size_t)dd.rows * D.h}); break;
    case AS_DBG_LSE: parts.push_back({x->lse2, 4 * (size_t)dd.rows}); break;  // log2 units
    case AS_DBG_LOSS: parts.push_back({x->lossr, 4 * (size_t)dd.rows}); break;
    case AS_DBG_DA: parts.push_back({x->dA, 4 * (size_t)dd.rows * D.h}); break;
    case AS_DBG_DB1: if (!dbg) return as_fail(AS_E_STATE, "needs AS_FLAG_DEBUG_GRADS"); parts.push_back({x->dbg_db1, 4 * (size_t)D.h}); break;
    case AS_DBG_DW2T: if (!dbg) return as_fail(AS_E_STATE, "needs AS_FLAG_DEBUG_GRADS"); parts.push_back({x->dbg_dW2, 4 * (size_t)D.C * D.h}); break;
    case AS_DBG_DB2: if (!dbg) return as_fail(AS_E_STATE, "needs AS_FLAG_DEBUG_GRADS"); parts.push_back({x->dbg_db2, 4 * (size_t)D.C}); break;
    case AS_DBG_DW1: if (!dbg) return as_fail(AS_E_STATE, "needs AS_FLAG_DEBUG_GRADS"); parts.push_back({x->dbg_dW1, 4 * (size_t)dd.U * D.h}); break;
    case AS_DBG_FSEG:
      head.push_back(dd.U);
      parts.push_back({x->fseg_id, 4 * (size_t)dd.U});
      parts.push_back({x->fseg_ptr, 4 * ((size_t)dd.U + 1)});
      parts.push_back({x->fseg_row, 4 * (size_t)dd.nnz});
      parts.push_back({x->fseg_val, 4 * (size_t)dd.nnz});
      break;
    case AS_DBG_LSEG:
      head.push_back(dd.V);
      parts.push_back({x->lseg_id, 4 * (size_t)dd.V});
      parts.push_back({x->lseg_ptr, 4 * ((size_t)dd.V + 1)});
      parts.push_back({x->lseg_row, 4 * (size_t)dd.nlab});
      break;
    case AS_DBG_BATCH: head = {dd.rows, dd.nnz, dd.nlab, dd.U}; break;
    case AS_DBG_DHSOFT: if (!dbg) return as_fail(AS_E_STATE, "needs AS_FLAG_DEBUG_GRADS"); parts.push_back({x->dbg_dHs, 4 * (size_t)dd.rows * D.h}); break;
    case AS_DBG_LOGITS:
      if (x->cfg.precision != AS_FP32) return as_fail(AS_E_STATE, "logits exist only in AS_FP32");
      parts.push_back({x->Z, 4 * (size_t)dd.rows * D.C});
      break;
    default: return as_fail(AS_E_INVALID, "bad `which`");
  }
  size_t total = 4 * head.size();
  for (auto &p : parts) total += p.second;
  if (total > bytes) return as_fail(AS_E_INVALID, "buffer too small: need %zu", total);
  uint8_t *o = (uint8_t *)host_out;
  memcpy(o, head.data(), 4 * head.size());
  o += 4 * head.size();
  for (auto &p : parts) {
    if (p.second) cudaMemcpyAsync(o, p.first, p.second, cudaMemcpyDeviceToHost, s);
    o += p.second;
  }
  rc = cuda_check(x, cudaStreamSynchronize(s), "debug D2H");
  *written = total;
  return rc;
}

int as_profile(as_ctx *x, int32_t enable) {
  AS_GUARD(x);
  x->prof_on = enable != 0;
  return AS_OK;
}

int as_profile_read(as_ctx *x, double *ms_out, int64_t *calls_out, int64_t *launches_out) {
  AS_GUARD(x);
  int rc = cuda_check(x, cudaStreamSynchronize(x->stream), "profile sync");
  if (rc) return rc;
  double ms[AS_PH_COUNT] = {0};
  int64_t calls[AS_PH_COUNT] = {0};
  for (auto &p : x->pending) {
    float t = 0.f;
    cudaEventElapsedTime(&t, p.a, p.b);
    ms[p.ph] += t;
    calls[p.ph] += 1;
    x->ev_pool.push_back(p.a);
    x->ev_pool.push_back(p.b);
  }
  x->pending.clear();
  if (ms_out) std::copy(ms, ms + AS_PH_COUNT, ms_out);
  if (calls_out) std::copy(calls, calls + AS_PH_COUNT, calls_out);
  if (launches_out) *launches_out = x->launches;
  x->launches = 0;
  return AS_OK;
}

int as_trace_dump(int64_t *out, int32_t max_events) {
  if (!out || max_events < 0) return as_fail(AS_E_INVALID, "bad arguments");
  return as::tc_trace_dump((long long *)out, max_events);
}

int as_tc_bench(int32_t mode, int32_t iters, int64_t *cycles) {
  if (!cycles || mode < 0 || mode > 14 || iters < 1) return as_fail(AS_E_INVALID, "bad arguments");
  long long c = 0;
  if (as::tc_bench(mode, iters, &c) != 0) return as_fail(AS_E_CUDA, "tc_bench failed");
  *cycles = c;
  return AS_OK;
}

int as_tc_selftest2(const void *A, const void *B, float *V, float *U) {
  if (!A || !B || !V || !U) return as_fail(AS_E_INVALID, "NULL argument");
  if (as::tc_selftest2(A, B, V, U, 0) != 0) return as_fail(AS_E_CUDA, "tensor map creation failed");
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return as_fail(AS_E_CUDA, "selftest2: %s", cudaGetErrorString(e));
  return AS_OK;
}

int as_tc_selftest(const void *A, const void *B, float *S, float *O, float *T) {
  if (!A || !B || !S || !O || !T) return as_fail(AS_E_INVALID, "NULL argument");
  if (as::tc_selftest(A, B, S, O, T, 0) != 0) return as_fail(AS_E_CUDA, "tensor map creation failed");
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return as_fail(AS_E_CUDA, "selftest: %s", cudaGetErrorString(e));
  return cuda_check(nullptr, cudaSuccess, "selftest");
}

}  // extern "C"

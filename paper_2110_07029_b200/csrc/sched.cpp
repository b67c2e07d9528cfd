// Host scheduler of Adaptive SGD: replay routing, Alg. 1, Alg. 2 weights,
// stream permutation and the live shared cursor.  Pure host code; the device
// never sees it.  P:N = PAPER.md line N, Rk = DESIGN.md reading k.
#include <cmath>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <string>

#include "adasgd.h"
#include "alg2.h"
#include "common_host.h"

extern "C" {

// P:105 (section 3.1): "batches are dispatched one-by-one based on GPU
// availability.  Whenever a GPU finishes an epoch, it is assigned the next
// batch", a mega-batch being a fixed number of samples.  Availability is
// replayed from integer cost models (R9); ties go to the lowest id and the
// last batch is truncated to the remaining samples (R8).  u_i counts the
// dispatched batches.
int as_sched_route_replay(int32_t N, const as_cost_model *cost, const int32_t *b,
                          int64_t M, const int64_t *nnz_prefix, as_route *out_log,
                          int64_t max_log, int64_t *n_log, int32_t *u_out,
                          int64_t *clocks_out) {
  if (N < 1 || !cost || !b || M < 0 || !nnz_prefix || !out_log || !n_log || !u_out ||
      !clocks_out)
    return as_fail(AS_E_INVALID, "as_sched_route_replay: bad arguments");
  for (int i = 0; i < N; ++i) {
    if (b[i] < 1) return as_fail(AS_E_INVALID, "as_sched_route_replay: b[%d] < 1", i);
    if (cost[i].den <= 0 || cost[i].num < 0 || cost[i].c0 < 0 || cost[i].c_row < 0 ||
        cost[i].c_nnz < 0)
      return as_fail(AS_E_INVALID, "as_sched_route_replay: bad cost model %d", i);
    u_out[i] = 0;
    clocks_out[i] = 0;
  }
  int64_t assigned = 0, k = 0;
  while (assigned < M) {
    int best = 0;
    for (int i = 1; i < N; ++i)
      if (clocks_out[i] < clocks_out[best]) best = i;  // strict: lowest id wins ties
    const int64_t rows = b[best] < M - assigned ? b[best] : M - assigned;
    if (k >= max_log) return as_fail(AS_E_INVALID, "as_sched_route_replay: log too small");
    const int64_t nnz = nnz_prefix[assigned + rows] - nnz_prefix[assigned];
    const as_cost_model &c = cost[best];
    clocks_out[best] += ((c.c0 + c.c_row * rows + c.c_nnz * nnz) * c.num) / c.den;
    out_log[k].replica = best;
    out_log[k].rows = (int32_t)rows;
    out_log[k].start = assigned;
    ++k;
    u_out[best] += 1;
    assigned += rows;
  }
  *n_log = k;
  return AS_OK;
}

// Static partitioning of the comparison methods (Fig. 3): batch k
// -> replica k mod N, equal batch sizes; the clocks replay the same cost
// models so that the straggler time max_i t_i can be compared with P:105's
// dynamic routing.
int as_sched_route_static(int32_t N, const as_cost_model *cost, const int32_t *b,
                          int64_t M, const int64_t *nnz_prefix, as_route *out_log,
                          int64_t max_log, int64_t *n_log, int32_t *u_out,
                          int64_t *clocks_out) {
  if (N < 1 || !cost || !b || M < 0 || !nnz_prefix || !out_log || !n_log || !u_out ||
      !clocks_out)
    return as_fail(AS_E_INVALID, "as_sched_route_static: bad arguments");
  for (int i = 0; i < N; ++i) {
    if (b[i] < 1 || b[i] != b[0]) return as_fail(AS_E_INVALID, "as_sched_route_static: b must be equal and >= 1");
    if (cost[i].den <= 0 || cost[i].num < 0 || cost[i].c0 < 0 || cost[i].c_row < 0 ||
        cost[i].c_nnz < 0)
      return as_fail(AS_E_INVALID, "as_sched_route_static: bad cost model %d", i);
    u_out[i] = 0;
    clocks_out[i] = 0;
  }
  int64_t assigned = 0, k = 0;
  while (assigned < M) {
    const int i = (int)(k % N);
    const int64_t rows = b[0] < M - assigned ? b[0] : M - assigned;
    if (k >= max_log) return as_fail(AS_E_INVALID, "as_sched_route_static: log too small");
    const int64_t nnz = nnz_prefix[assigned + rows] - nnz_prefix[assigned];
    const as_cost_model &c = cost[i];
    clocks_out[i] += ((c.c0 + c.c_row * rows + c.c_nnz * nnz) * c.num) / c.den;
    out_log[k].replica = i;
    out_log[k].rows = (int32_t)rows;
    out_log[k].start = assigned;
    ++k;
    u_out[i] += 1;
    assigned += rows;
  }
  *n_log = k;
  return AS_OK;
}

// Algorithm 1 "Batch Size Scaling".  mu = sum(u)/N (line 1).
// beta*(u_i - mu) = beta*D_i/N with the exact integer D_i = N*u_i - sum(u);
// R11 rounds it half away from zero and checks the bound on the rounded
// value (no clamp).  lr follows the linear scaling rule.
int as_sched_alg1(int32_t N, const int32_t *u, const int32_t *b, int32_t beta,
                  int32_t b_min, int32_t b_max, double lr0, int32_t *b_out,
                  float *lr_out) {
  if (N < 1 || !u || !b || !b_out || !lr_out || beta < 0 || b_min < 1 || b_max < b_min)
    return as_fail(AS_E_INVALID, "as_sched_alg1: bad arguments");
  int64_t U = 0;
  for (int i = 0; i < N; ++i) U += u[i];
  for (int i = 0; i < N; ++i) {
    const int64_t D = (int64_t)N * u[i] - U;
    const int64_t absD = D < 0 ? -D : D;
    const int64_t step = (2 * (int64_t)beta * absD + N) / (2 * (int64_t)N);
    int64_t nb = b[i];
    if (D > 0 && b[i] + step <= b_max)
      nb = b[i] + step;
    else if (D < 0 && b[i] - step >= b_min)
      nb = b[i] - step;
    b_out[i] = (int32_t)nb;
    lr_out[i] = (float)(lr0 * (double)nb / (double)b_max);
  }
  return AS_OK;
}

// Adaptive scaling frequency (reading R27).  dir_state[i] holds the
// sign of the previous run's change of b_i.  This run's signs d_i =
// sign(b_next_i - b_prev_i); "stability" = every d_i == 0; "oscillatory" =
// some b_i reversed (d_i * dir_i < 0) and none kept its direction
// (d_i * dir_i > 0).  In either state the interval doubles (capped at p_max),
// otherwise it returns to 1 mega-batch; dir_state <- d.
int as_sched_scale_period(int32_t N, const int32_t *b_prev, const int32_t *b_next,
                          int32_t *dir_state, int32_t period, int32_t p_max,
                          int32_t *period_out) {
  if (N < 1 || !b_prev || !b_next || !dir_state || !period_out || p_max < 1 || period < 1 ||
      period > p_max)
    return as_fail(AS_E_INVALID, "as_sched_scale_period: bad arguments");
  bool moved = false, reversed = false, kept = false;
  for (int i = 0; i < N; ++i) {
    const int32_t d = (b_next[i] > b_prev[i]) - (b_next[i] < b_prev[i]);
    if (d != 0) moved = true;
    if (d * dir_state[i] < 0) reversed = true;
    if (d * dir_state[i] > 0) kept = true;
    dir_state[i] = d;
  }
  const bool settle = !moved || (reversed && !kept);
  const int64_t p2 = 2 * (int64_t)period;
  *period_out = settle ? (int32_t)(p2 < p_max ? p2 : p_max) : 1;
  return AS_OK;
}

// Algorithm 2 "Normalized Model Merging", lines 1-10.
// R13 exact equality of u; R14 r/s = lexicographic argmax/argmin of (u_i, b_i)
// with the lowest id on ties, perturbation skipped when (u_r,b_r)==(u_s,b_s);
// R15 strict "<"; R16 no renormalisation.
int as_sched_alg2(int32_t N, const int32_t *u, const int32_t *b, const double *norms,
                  double delta, double pert_thr, double *alpha_out,
                  int32_t *perturbed_out) {
  return as_sched_alg2_ex(N, u, b, norms, delta, pert_thr, AS_NORM_UPDATES, alpha_out, perturbed_out);
}

// norm_mode AS_NORM_UB: line 5 uses u_i b_i / sum(u b) -- "an alternative for
// later stages is to normalize based on the product between the number of
// updates and the batch size".
int as_sched_alg2_ex(int32_t N, const int32_t *u, const int32_t *b, const double *norms,
                     double delta, double pert_thr, int32_t norm_mode, double *alpha_out,
                     int32_t *perturbed_out) {
  if (N < 1 || !u || !b || !norms || !alpha_out || norm_mode < 0 || norm_mode > (AS_NORM_UB | AS_NORM_R14_LITERAL))
    return as_fail(AS_E_INVALID, "as_sched_alg2: bad arguments");
  if (as::alg2_weights(N, u, b, norms, delta, pert_thr, norm_mode, alpha_out,
                       perturbed_out) != 0)
    return as_fail(AS_E_INVALID, "as_sched_alg2: zero normaliser (sum(b) or sum(u b))");
  return AS_OK;
}

static inline uint64_t splitmix64_next(uint64_t &state) {
  state += 0x9E3779B97F4A7C15ull;
  uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// R10: Fisher-Yates with j = (r * (i + 1)) >> 64, r = SplitMix64 output.
int as_sched_permutation(int64_t n, uint64_t seed, int64_t *out) {
  if (n < 0 || (n > 0 && !out)) return as_fail(AS_E_INVALID, "as_sched_permutation: bad arguments");
  for (int64_t i = 0; i < n; ++i) out[i] = i;
  uint64_t s = seed;
  for (int64_t i = n - 1; i > 0; --i) {
    const uint64_t r = splitmix64_next(s);
    const uint64_t j = (uint64_t)(((unsigned __int128)r * (unsigned __int128)(i + 1)) >> 64);
    const int64_t t = out[i];
    out[i] = out[j];
    out[j] = t;
  }
  return AS_OK;
}

// ---- live routing: one shared cursor per mega-batch ----------
struct as_live {
  int fd;
  std::atomic<int64_t> *cursor;
  std::string name;
};

int as_live_open(const char *name, int32_t create, as_live **out) {
  if (!name || !out || name[0] != '/') return as_fail(AS_E_INVALID, "as_live_open: name must start with '/'");
  const int fd = shm_open(name, create ? (O_CREAT | O_RDWR) : O_RDWR, 0600);
  if (fd < 0) return as_fail(AS_E_INVALID, "as_live_open: shm_open(%s): %s", name, strerror(errno));
  if (create && ftruncate(fd, 64) != 0) {
    close(fd);
    return as_fail(AS_E_INVALID, "as_live_open: ftruncate: %s", strerror(errno));
  }
  void *p = mmap(nullptr, 64, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  if (p == MAP_FAILED) {
    close(fd);
    return as_fail(AS_E_INVALID, "as_live_open: mmap: %s", strerror(errno));
  }
  as_live *lv = new as_live{fd, reinterpret_cast<std::atomic<int64_t> *>(p), name};
  if (create) lv->cursor->store(0);
  *out = lv;
  return AS_OK;
}

int as_live_claim(as_live *lv, int64_t M, int32_t b, int64_t *start, int32_t *rows) {
  if (!lv || !start || !rows || b < 1 || M < 0) return as_fail(AS_E_INVALID, "as_live_claim: bad arguments");
  const int64_t s = lv->cursor->fetch_add(b);
  *start = s;
  *rows = s >= M ? 0 : (int32_t)(b < M - s ? b : M - s);
  return AS_OK;
}

int as_live_reset(as_live *lv) {
  if (!lv) return as_fail(AS_E_INVALID, "as_live_reset: null");
  lv->cursor->store(0);
  return AS_OK;
}

int as_live_close(as_live *lv, int32_t unlink_segment) {
  if (!lv) return as_fail(AS_E_INVALID, "as_live_close: null");
  munmap(lv->cursor, 64);
  close(lv->fd);
  if (unlink_segment) shm_unlink(lv->name.c_str());
  delete lv;
  return AS_OK;
}

}  // extern "C"

// Replay cost model from a live trace ("relative processing speed",
// P:193 the scheduler records per-batch times; reading R9): least-squares fit
// of t_k = c0 + c_row rows_k + c_nnz nnz_k (picoseconds) over n recorded
// batches of one replica, normal equations in long double, coefficients
// rounded to the nearest integer and clamped at 0; num = den = 1.
int as_sched_fit_cost(int64_t n, const int32_t *rows, const int64_t *nnz, const int64_t *ps,
                      as_cost_model *out) {
  if (n < 3 || !rows || !nnz || !ps || !out) return as_fail(AS_E_INVALID, "as_sched_fit_cost: bad arguments");
  long double A[3][4] = {{0}};
  for (int64_t k = 0; k < n; ++k) {
    const long double x[3] = {1.0L, (long double)rows[k], (long double)nnz[k]};
    for (int i = 0; i < 3; ++i) {
      for (int j = 0; j < 3; ++j) A[i][j] += x[i] * x[j];
      A[i][3] += x[i] * (long double)ps[k];
    }
  }
  for (int c = 0; c < 3; ++c) {  // Gauss-Jordan with partial pivoting
    int p = c;
    for (int i = c + 1; i < 3; ++i)
      if (fabsl(A[i][c]) > fabsl(A[p][c])) p = i;
    if (fabsl(A[p][c]) < 1e-30L) return as_fail(AS_E_INVALID, "as_sched_fit_cost: singular (rows / nnz collinear)");
    for (int j = 0; j < 4; ++j) { const long double t = A[c][j]; A[c][j] = A[p][j]; A[p][j] = t; }
    for (int i = 0; i < 3; ++i) {
      if (i == c) continue;
      const long double f = A[i][c] / A[c][c];
      for (int j = c; j < 4; ++j) A[i][j] -= f * A[c][j];
    }
  }
  int64_t co[3];
  for (int i = 0; i < 3; ++i) {
    const long double v = A[i][3] / A[i][i];
    co[i] = v <= 0.0L ? 0 : (int64_t)llroundl(v);
  }
  out->c0 = co[0];
  out->c_row = co[1];
  out->c_nnz = co[2];
  out->num = 1;
  out->den = 1;
  return AS_OK;
}

// Alg. 2 lines 1-10 with readings R13-R16: the merge weights
// alpha_i from the update counts u_i, batch sizes b_i and replica norms n_i.
// One definition for the host export (as_sched_alg2_ex, sched.cpp) and the
// device kernel of the merge (k_alg2, kernels_dense.cu): the same fp64
// operations in the same order, so every rank and the host agree bit for bit.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define AS_HD __host__ __device__
#else
#define AS_HD
#endif

namespace as {

// norm_mode bit 0 clear: line 5 alpha_i = u_i / sum(u); set: alpha_i = u_i b_i /
// sum(u b).  Bit 1 (R14 "literal"): line 8 as printed, r / s = the
// lowest-id argmax / argmin of u alone, applied even when r = s; clear:
// lexicographic (u_i, b_i), skipped when all pairs are equal.  Returns 0, or
// -1 when the normaliser is zero.
AS_HD inline int alg2_weights(int N, const int32_t *u, const int32_t *b, const double *norms, double delta,
                              double pert_thr, int norm_mode, double *alpha, int32_t *perturbed) {
  bool all_equal = true;                         // line 2 (R13: exact integer equality)
  for (int i = 1; i < N; ++i)
    if (u[i] != u[0]) all_equal = false;
  if (all_equal) {                               // line 3: alpha_i = b_i / sum(b)
    int64_t sb = 0;
    for (int i = 0; i < N; ++i) sb += b[i];
    if (sb <= 0) return -1;
    for (int i = 0; i < N; ++i) alpha[i] = (double)b[i] / (double)sb;
  } else if ((norm_mode & 1) == 0) {            // line 5: alpha_i = u_i / sum(u)
    int64_t su = 0;
    for (int i = 0; i < N; ++i) su += u[i];
    for (int i = 0; i < N; ++i) alpha[i] = (double)u[i] / (double)su;
  } else {                                       // P:175 variant
    int64_t sub = 0;
    for (int i = 0; i < N; ++i) sub += (int64_t)u[i] * b[i];
    if (sub <= 0) return -1;
    for (int i = 0; i < N; ++i) alpha[i] = (double)((int64_t)u[i] * b[i]) / (double)sub;
  }
  int32_t pert = 0;
  bool regular = true;                           // line 7 (R15: strict <)
  for (int i = 0; i < N; ++i)
    if (!(norms[i] < pert_thr)) regular = false;
  if (regular && (norm_mode & 2)) {             // line 8 as printed (R14 literal)
    int r = 0, s = 0;
    for (int i = 1; i < N; ++i) {
      if (u[i] > u[r]) r = i;
      if (u[i] < u[s]) s = i;
    }
    alpha[r] = alpha[r] * (1.0 + delta);         // line 9 (r = s: both factors on alpha_r)
    alpha[s] = alpha[s] * (1.0 - delta);
    pert = 1;
  } else if (regular) {
    int r = 0, s = 0;                            // line 8 (R14: lexicographic, lowest id)
    for (int i = 1; i < N; ++i) {
      if (u[i] > u[r] || (u[i] == u[r] && b[i] > b[r])) r = i;
      if (u[i] < u[s] || (u[i] == u[s] && b[i] < b[s])) s = i;
    }
    if (!(u[r] == u[s] && b[r] == b[s])) {       // line 9; skip when all identical (R14)
      alpha[r] = alpha[r] * (1.0 + delta);
      alpha[s] = alpha[s] * (1.0 - delta);       // no renormalisation (R16)
      pert = 1;
    }
  }
  if (perturbed) *perturbed = pert;
  return 0;
}

}  // namespace as

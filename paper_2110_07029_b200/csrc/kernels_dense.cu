// fp32 SIMT output layer (the AS_FP32 parity mode of steps a5/a6) and the
// merge kernels (steps a9-a13).  P:N = PAPER.md line N; Rk = DESIGN.md.
#include <cfloat>

#include "alg2.h"
#include "common.cuh"

namespace as {

// =====================================================================
// Generic fp32 tiled GEMM  C[m][n] = sum_k A(m,k) B(k,n) (+ bias[n]) with
// arbitrary strides, optional split-K (partials reduced in a fixed order).
// A(m,k) = A[m*sam + k*sak], B(k,n) = B[k*sbk + n*sbn].  M and K may be capped
// by device counters (the batch rows).  64x64x16 tiles, 4x4 per thread.
// =====================================================================
constexpr int GBM = 64, GBN = 64, GBK = 16;

__global__ void __launch_bounds__(256) k_gemm_f32(int M, int N, int K, const float *__restrict__ A,
                                                  long long sam, long long sak,
                                                  const float *__restrict__ B, long long sbk,
                                                  long long sbn, float *__restrict__ Cm,
                                                  long long ldc, const float *__restrict__ bias,
                                                  int kchunk, const int *__restrict__ M_dev,
                                                  const int *__restrict__ K_dev, int to_tmp) {
  __shared__ float As[GBK][GBM + 4];
  __shared__ float Bs[GBK][GBN + 4];
  if (M_dev) M = min(M, *M_dev);
  if (K_dev) K = min(K, *K_dev);
  const int m0 = blockIdx.y * GBM, n0 = blockIdx.x * GBN;
  if (m0 >= M) return;
  const int kb = blockIdx.z * kchunk, ke = min(K, kb + kchunk);
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
  float acc[4][4] = {};
  for (int k0 = kb; k0 < ke; k0 += GBK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = t + 256 * i;
      int m, k;
      if (sak == 1) { m = e >> 4; k = e & 15; } else { m = e & 63; k = e >> 6; }
      const int gm = m0 + m, gk = k0 + k;
      As[k][m] = (gm < M && gk < ke) ? A[(long long)gm * sam + (long long)gk * sak] : 0.f;
      int n, kk;
      if (sbn == 1) { kk = e >> 6; n = e & 63; } else { n = e >> 4; kk = e & 15; }
      const int gn = n0 + n, gk2 = k0 + kk;
      Bs[kk][n] = (gn < N && gk2 < ke) ? B[(long long)gk2 * sbk + (long long)gn * sbn] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < GBK; ++k) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[k][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[k][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  float *out = Cm + (to_tmp ? (long long)blockIdx.z * M * ldc : 0);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn >= N) continue;
      out[(long long)gm * ldc + gn] = acc[i][j] + ((bias && !to_tmp) ? bias[gn] : 0.f);
    }
  }
}

__global__ void k_splitk_reduce(int M, int N, int splits, const float *__restrict__ tmp,
                                float *__restrict__ Cm, long long ldc, const float *__restrict__ bias,
                                const int *__restrict__ M_dev) {
  if (M_dev) M = min(M, *M_dev);
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)M * N) return;
  const int m = (int)(i / N), n = (int)(i % N);
  float a = 0.f;
  for (int z = 0; z < splits; ++z) a += tmp[(long long)z * M * N + i];
  Cm[(long long)m * ldc + n] = a + (bias ? bias[n] : 0.f);
}

void launch_gemm_f32(cudaStream_t s, int M, int N, int K, const float *A, long long sam,
                     long long sak, const float *B, long long sbk, long long sbn, float *Cm,
                     long long ldc, const float *bias_n, int splitk, float *splitk_tmp,
                     const int *M_dev) {
  if (splitk < 1) splitk = 1;
  int kchunk = ceil_div(K, splitk);
  kchunk = ceil_div(kchunk, GBK) * GBK;
  splitk = ceil_div(K, kchunk);
  dim3 grid(ceil_div(N, GBN), ceil_div(M, GBM), splitk);
  if (splitk == 1) {
    k_gemm_f32<<<grid, 256, 0, s>>>(M, N, K, A, sam, sak, B, sbk, sbn, Cm, ldc, bias_n, kchunk,
                                    M_dev, nullptr, 0);
  } else {
    k_gemm_f32<<<grid, 256, 0, s>>>(M, N, K, A, sam, sak, B, sbk, sbn, splitk_tmp, N, nullptr,
                                    kchunk, M_dev, nullptr, 1);
    k_splitk_reduce<<<ceil_div((long long)M * N, 256), 256, 0, s>>>(M, N, splitk, splitk_tmp, Cm,
                                                                    ldc, bias_n, M_dev);
  }
}

// K capped by the batch rows (dW2T = dZ^T H has K = B)
void launch_gemm_f32_kdev(cudaStream_t s, int M, int N, int K, const float *A, long long sam,
                          long long sak, const float *B, long long sbk, long long sbn, float *Cm,
                          long long ldc, const int *K_dev) {
  dim3 grid(ceil_div(N, GBN), ceil_div(M, GBM), 1);
  k_gemm_f32<<<grid, 256, 0, s>>>(M, N, K, A, sam, sak, B, sbk, sbn, Cm, ldc, nullptr,
                                  ceil_div(K, GBK) * GBK, nullptr, K_dev, 0);
}

// LSE_r (stored in log2 units) of the fp32 logits, fixed-order block reduction
__global__ void __launch_bounds__(256) k_row_lse(const StepDesc *__restrict__ desc, int C,
                                                 const float *__restrict__ Z,
                                                 float *__restrict__ lse2) {
  __shared__ float red[256];
  const int r = blockIdx.x;
  if (r >= desc->rows) return;
  const float *z = Z + (size_t)r * C;
  float m = -FLT_MAX;
  for (int c = threadIdx.x; c < C; c += 256) m = fmaxf(m, z[c]);
  red[threadIdx.x] = m;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] = fmaxf(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  m = red[0];
  __syncthreads();
  float sum = 0.f;
  for (int c = threadIdx.x; c < C; c += 256) sum += expf(z[c] - m);
  red[threadIdx.x] = sum;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) lse2[r] = (m + logf(red[0])) * 1.4426950408889634f;
}

void launch_row_lse(cudaStream_t s, const StepDesc *desc, int b_max, int C, const float *Z,
                    float *lse2) {
  k_row_lse<<<b_max, 256, 0, s>>>(desc, C, Z, lse2);
}

// top-1 evaluation, fp32 mode: per row max_c z_c with the lowest c on ties
// (R21) over the materialised logits; one partial slot
__global__ void __launch_bounds__(256) k_row_argmax(const StepDesc *__restrict__ desc, int C,
                                                    const float *__restrict__ Z, float *__restrict__ pmax,
                                                    int *__restrict__ pidx) {
  __shared__ float rv[256];
  __shared__ int ri[256];
  const int r = blockIdx.x;
  if (r >= desc->rows) return;
  const float *z = Z + (size_t)r * C;
  float m = -INFINITY;
  int mi = 0x7fffffff;
  for (int c = threadIdx.x; c < C; c += 256)
    if (z[c] > m) { m = z[c]; mi = c; }        // ascending c per thread
  rv[threadIdx.x] = m; ri[threadIdx.x] = mi;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      const float v = rv[threadIdx.x + o];
      const int i = ri[threadIdx.x + o];
      if (v > rv[threadIdx.x] || (v == rv[threadIdx.x] && i < ri[threadIdx.x])) {
        rv[threadIdx.x] = v; ri[threadIdx.x] = i;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { pmax[r] = rv[0]; pidx[r] = ri[0]; }
}

void launch_row_argmax_f32(cudaStream_t s, const StepDesc *desc, int b_max, int C, const float *Z, float *pmax,
                           int *pidx) {
  k_row_argmax<<<b_max, 256, 0, s>>>(desc, C, Z, pmax, pidx);
}

// ordered combine of the (max, argmax) slots; a hit when the top-1 class is
// one of the row's labels; integer hit count
__global__ void k_top1_combine(const StepDesc *__restrict__ desc, int slots, int bpad,
                               const float *__restrict__ pmax, const int *__restrict__ pidx,
                               const int64_t *__restrict__ lab_ptr, const int32_t *__restrict__ lab,
                               int32_t *__restrict__ top1, unsigned long long *__restrict__ hits) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= desc->rows) return;
  float m = -INFINITY;
  int mi = 0x7fffffff;
  for (int sl = 0; sl < slots; ++sl) {
    const float v = pmax[(size_t)sl * bpad + r];
    const int i = pidx[(size_t)sl * bpad + r];
    if (v > m || (v == m && i < mi)) { m = v; mi = i; }
  }
  top1[r] = mi;
  int hit = 0;
  for (int64_t j = lab_ptr[r]; j < lab_ptr[r + 1]; ++j) hit |= lab[j] == mi;
  if (hit) atomicAdd(hits, 1ull);
}

void launch_top1_combine(cudaStream_t s, const StepDesc *desc, int slots, int bpad, const float *pmax,
                         const int *pidx, const int64_t *lab_ptr, const int32_t *lab, int32_t *top1,
                         unsigned long long *hits) {
  k_top1_combine<<<(bpad + 127) / 128, 128, 0, s>>>(desc, slots, bpad, pmax, pidx, lab_ptr, lab, top1, hits);
}

// dZ = (softmax(z_r) - T_r)/B in place (R3)
__global__ void k_softmax(const StepDesc *__restrict__ desc, int C, float *__restrict__ Z,
                          const float *__restrict__ lse2) {
  const int r = blockIdx.y;
  if (r >= desc->rows) return;
  const float invB = 1.0f / (float)desc->rows;
  const float lse = lse2[r] * 0.69314718055994531f;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
    float *z = Z + (size_t)r * C + c;
    *z = expf(*z - lse) * invB;
  }
}

__global__ void k_softmax_labels(const StepDesc *__restrict__ desc, int C,
                                 const int64_t *__restrict__ lab_ptr,
                                 const int32_t *__restrict__ lab, float *__restrict__ Z) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int B = desc->rows;
  if (r >= B) return;
  const int64_t s = lab_ptr[r], e = lab_ptr[r + 1];
  const float w = (1.0f / (float)B) / (float)(e - s);
  for (int64_t j = s; j < e; ++j) Z[(size_t)r * C + lab[j]] -= w;
}

void launch_softmax_grad(cudaStream_t s, const StepDesc *desc, int b_max, int C,
                         const int64_t *lab_ptr, const int32_t *lab, float *Z, const float *lse2,
                         int part) {
  if (part & 1) {                 // Z <- softmax(Z) / B
    dim3 g(ceil_div(C, 256 * 8) < 64 ? ceil_div(C, 256 * 8) : 64, b_max);
    if (g.x < 1) g.x = 1;
    k_softmax<<<g, 256, 0, s>>>(desc, C, Z, lse2);
  }
  if (part & 2)                   // Z -= T / B (R3)
    k_softmax_labels<<<ceil_div(b_max, 128), 128, 0, s>>>(desc, C, lab_ptr, lab, Z);
}

// dA = dH * [A > 0]; loss_r = LSE_r - zsum_r
__global__ void k_finish_f32(const StepDesc *__restrict__ desc, int h, const float *__restrict__ dH,
                             const float *__restrict__ Hf, const float *__restrict__ zsum,
                             const float *__restrict__ lse2, float *__restrict__ lossr,
                             float *__restrict__ dA, const float *__restrict__ labW,
                             float *__restrict__ dbg_dHs) {
  const int r = blockIdx.x, j = threadIdx.x;
  if (r >= desc->rows) return;
  const size_t i = (size_t)r * h + j;
  dA[i] = Hf[i] > 0.f ? dH[i] : 0.f;
  (void)labW; (void)dbg_dHs;
  if (j == 0) lossr[r] = lse2[r] * 0.69314718055994531f - zsum[r];
}

void launch_finish_f32(cudaStream_t s, int h, const StepDesc *desc, int b_max, const float *dH,
                       const float *Hf, const float *zsum, const float *lse2, float *lossr,
                       float *dA, const float *labW, float *dbg_dHs) {
  k_finish_f32<<<b_max, h, 0, s>>>(desc, h, dH, Hf, zsum, lse2, lossr, dA, labW, dbg_dHs);
}

__global__ void k_sgd_dense(long long n, float *__restrict__ p, const float *__restrict__ g,
                            float lr, __nv_bfloat16 *__restrict__ shadow) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const float v = p[i] - lr * g[i];
    p[i] = v;
    if (shadow) shadow[i] = __float2bfloat16_rn(v);
  }
}

void launch_sgd_dense(cudaStream_t s, long long n, float *param, const float *grad, float lr,
                      __nv_bfloat16 *shadow) {
  k_sgd_dense<<<148 * 8, 256, 0, s>>>(n, param, grad, lr, shadow);
}

// =====================================================================
// Merge (Alg. 2)
// =====================================================================
// a9: ||w||_2 / P, fixed-order two-level reduction in fp64 (R15)
__global__ void __launch_bounds__(256) k_sumsq(const float *__restrict__ w, long long P,
                                               long long chunk, double *__restrict__ partials) {
  __shared__ double red[256];
  const long long b0 = (long long)blockIdx.x * chunk, b1 = min(P, b0 + chunk);
  double a = 0.0;
  for (long long i = b0 + threadIdx.x; i < b1; i += 256) {
    const double x = (double)w[i];
    a = fma(x, x, a);
  }
  red[threadIdx.x] = a;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(1024) k_sumsq_final(const double *__restrict__ partials, int nb,
                                                      long long P, int metric, double *__restrict__ out) {
  __shared__ double red[1024];
  double a = 0.0;
  for (int i = threadIdx.x; i < nb; i += 1024) a += partials[i];
  red[threadIdx.x] = a;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  // R15 regularisation metric: ||w||_2 / P (literal, default), ||w||_2^2 / P,
  // ||w||_2 / sqrt(P), ||w||_2
  if (threadIdx.x == 0) {
    const double S = red[0];
    *out = metric == 1 ? S / (double)P : metric == 2 ? sqrt(S / (double)P) : metric == 3 ? sqrt(S)
                                                                                        : sqrt(S) / (double)P;
  }
}

void launch_sumsq(cudaStream_t s, const float *w, long long P, double *partials, int nblocks,
                  double *out_norm, int metric) {
  const long long chunk = (P + nblocks - 1) / nblocks;
  k_sumsq<<<nblocks, 256, 0, s>>>(w, P, chunk, partials);
  k_sumsq_final<<<1, 1024, 0, s>>>(partials, nblocks, P, metric, out_norm);
}

// a11: w_i <- alpha_i w_i
__global__ void k_scale(float *__restrict__ w, long long P, float alpha) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < P;
       i += (long long)gridDim.x * blockDim.x)
    w[i] *= alpha;
}

void launch_scale(cudaStream_t s, float *w, long long P, float alpha) {
  k_scale<<<148 * 8, 256, 0, s>>>(w, P, alpha);
}

// a11 with the weight in device memory (the device-computed alpha_rank)
__global__ void k_scale_dev(float *__restrict__ w, long long P, const float *__restrict__ alpha) {
  const float a = *alpha;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < P;
       i += (long long)gridDim.x * blockDim.x)
    w[i] *= a;
}

void launch_scale_dev(cudaStream_t s, float *w, long long P, const float *alpha) {
  k_scale_dev<<<148 * 8, 256, 0, s>>>(w, P, alpha);
}

// a10 on the device: Alg. 2 from the all-gathered norms (as::alg2_weights, the
// same code as the host export), or the comparison methods' uniform 1/N, or
// caller-given weights.  One thread; writes alpha in fp64 and fp32 and the
// perturbation flag.  A zero normaliser (rejected on the host before launch)
// cannot occur here.
__global__ void k_alg2(MergeWeightArgs a, const double *__restrict__ norms, double *__restrict__ alpha_d,
                       float *__restrict__ alpha_f, int32_t *__restrict__ pert) {
  double al[kMaxWorld];
  int32_t pt = 0;
  if (a.mode == 0) {
    if (alg2_weights(a.N, a.u, a.b, norms, a.delta, a.pert_thr, a.norm_mode, al, &pt) != 0)
      for (int i = 0; i < a.N; ++i) al[i] = 0.0;
  } else if (a.mode == 1) {
    for (int i = 0; i < a.N; ++i) al[i] = 1.0 / (double)a.N;
  } else {
    for (int i = 0; i < a.N; ++i) al[i] = a.given[i];
  }
  for (int i = 0; i < a.N; ++i) {
    alpha_d[i] = al[i];
    alpha_f[i] = (float)al[i];
  }
  *pert = pt;
}

void launch_alg2(cudaStream_t s, const MergeWeightArgs &a, const double *norms, double *alpha_d, float *alpha_f,
                 int32_t *pert) {
  k_alg2<<<1, 1, 0, s>>>(a, norms, alpha_d, alpha_f, pert);
}

// ---------------------------------------------------------------------------
// Peer-memory merge (AS_MERGE_P2P).  Every rank's workspace is mapped into
// every other rank (CUDA IPC over NVLink / NVSwitch); buffers are addressed as
// base[k] + offset (identical carve on every rank).
//
// Barrier: rank r writes `epoch` into flags[r] of every rank (after its
// optional payload, e.g. its norm into norms[r]) with a system-scope release,
// then waits until its own flags[k] >= epoch for every k (acquire).
__global__ void k_p2p_barrier(PeerArgs a, const double *__restrict__ my_norm) {
  const int k = threadIdx.x;
  if (k < a.N) {
    uint8_t *pb = a.base[k];
    if (my_norm) reinterpret_cast<volatile double *>(pb + a.off_norms)[a.rank] = *my_norm;
    __threadfence_system();
    unsigned long long *f = reinterpret_cast<unsigned long long *>(pb + a.off_flags) + a.rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(a.epoch) : "memory");
  }
  if (k < a.N) {
    const unsigned long long *mine = reinterpret_cast<const unsigned long long *>(a.base[a.rank] + a.off_flags) + k;
    unsigned long long v = 0;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
      if (v >= a.epoch) break;
      __nanosleep(256);
    }
  }
  __syncthreads();
  __threadfence_system();
}

void launch_p2p_barrier(cudaStream_t s, const PeerArgs &a, const double *my_norm) {
  k_p2p_barrier<<<1, kMaxWorld, 0, s>>>(a, my_norm);
}

// a11-a13 fused: rank r owns elements [lo, hi) (multiples of 4 floats); for
// each of them S = sum_k alpha_k w_k (peer loads, replica order),
// w' = S + gamma (wbar - wbar_p) (this rank's copies; identical on every
// rank), then w' is pushed into every rank's replica and new global model
// (the wbar_p buffer, which becomes wbar after the pointer rotation) and, in
// the W2T range, its bf16 shadow.  Slice r of every replica is read and
// written only by rank r, so no ordering beyond the two barriers is needed.
__global__ void __launch_bounds__(256) k_merge_p2p(PeerArgs a, const float *__restrict__ alpha_f,
                                                   const float *__restrict__ wbar,
                                                   const float *__restrict__ wbarp) {
  __shared__ float al[kMaxWorld];
  if (threadIdx.x < a.N) al[threadIdx.x] = alpha_f[threadIdx.x];
  __syncthreads();
  const long long nv = a.P / 4;                         // whole float4 vectors
  const long long v0 = nv * a.rank / a.N, v1 = nv * (a.rank + 1) / a.N;
  for (long long v = v0 + (long long)blockIdx.x * blockDim.x + threadIdx.x; v < v1;
       v += (long long)gridDim.x * blockDim.x) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k = 0; k < a.N; ++k) {
      const float4 x = reinterpret_cast<const float4 *>(a.base[k] + a.off_w)[v];
      const float c = al[k];
      acc.x = fmaf(c, x.x, acc.x); acc.y = fmaf(c, x.y, acc.y);
      acc.z = fmaf(c, x.z, acc.z); acc.w = fmaf(c, x.w, acc.w);
    }
    const float4 g = reinterpret_cast<const float4 *>(wbar)[v], q = reinterpret_cast<const float4 *>(wbarp)[v];
    float4 o;
    o.x = acc.x + a.gamma * (g.x - q.x); o.y = acc.y + a.gamma * (g.y - q.y);
    o.z = acc.z + a.gamma * (g.z - q.z); o.w = acc.w + a.gamma * (g.w - q.w);
    const long long i = 4 * v;
    const bool sh = i >= a.w2_off && i < a.w2_off + a.w2_len;
    const uint2 ob = make_uint2(pack_bf16x2(o.x, o.y), pack_bf16x2(o.z, o.w));
    for (int k = 0; k < a.N; ++k) {
      uint8_t *pb = a.base[k];
      reinterpret_cast<float4 *>(pb + a.off_w)[v] = o;
      reinterpret_cast<float4 *>(pb + a.off_wbarp)[v] = o;
      if (sh) reinterpret_cast<uint2 *>(pb + a.off_w2b)[(i - a.w2_off) / 4] = ob;
    }
  }
  // the tail P % 4 (last rank)
  if (a.rank == a.N - 1 && blockIdx.x == 0 && threadIdx.x < (int)(a.P - 4 * nv)) {
    const long long i = 4 * nv + threadIdx.x;
    float acc = 0.f;
    for (int k = 0; k < a.N; ++k) acc = fmaf(al[k], reinterpret_cast<const float *>(a.base[k] + a.off_w)[i], acc);
    const float o = acc + a.gamma * (wbar[i] - wbarp[i]);
    for (int k = 0; k < a.N; ++k) {
      reinterpret_cast<float *>(a.base[k] + a.off_w)[i] = o;
      reinterpret_cast<float *>(a.base[k] + a.off_wbarp)[i] = o;
      if (i >= a.w2_off && i < a.w2_off + a.w2_len)
        reinterpret_cast<__nv_bfloat16 *>(a.base[k] + a.off_w2b)[i - a.w2_off] = __float2bfloat16_rn(o);
    }
  }
}

void launch_merge_p2p(cudaStream_t s, const PeerArgs &a, const float *alpha_f, const float *wbar,
                      const float *wbarp) {
  k_merge_p2p<<<148 * 4, 256, 0, s>>>(a, alpha_f, wbar, wbarp);
}

// a13: w' = S + gamma (wbar - wbar_p) written over wbar_p (pointer rotation
// makes it the new wbar; the old wbar becomes wbar_p), w_i <- w',
// bf16 shadow of W2T refreshed.
__global__ void k_momentum(float *__restrict__ w, float *__restrict__ wp,
                           const float *__restrict__ wbar, long long P, float gamma,
                           long long w2_off, long long w2_len, __nv_bfloat16 *__restrict__ shadow) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < P;
       i += (long long)gridDim.x * blockDim.x) {
    const float nv = w[i] + gamma * (wbar[i] - wp[i]);
    wp[i] = nv;
    w[i] = nv;
    if (shadow && i >= w2_off && i < w2_off + w2_len) shadow[i - w2_off] = __float2bfloat16_rn(nv);
  }
}

// the same on float4 vectors (all pointers 16-B aligned, w2_off % 4 == 0, so a
// vector lies wholly inside or outside the W2T range); scalar tail P % 4
__global__ void __launch_bounds__(256) k_momentum4(float *__restrict__ w, float *__restrict__ wp,
                                                   const float *__restrict__ wbar, long long P, float gamma,
                                                   long long w2_off, long long w2_len,
                                                   __nv_bfloat16 *__restrict__ shadow) {
  const long long nv4 = P / 4;
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < nv4;
       v += (long long)gridDim.x * blockDim.x) {
    const float4 a = reinterpret_cast<const float4 *>(w)[v], g = reinterpret_cast<const float4 *>(wbar)[v],
                 q = reinterpret_cast<const float4 *>(wp)[v];
    float4 o;
    o.x = a.x + gamma * (g.x - q.x); o.y = a.y + gamma * (g.y - q.y);
    o.z = a.z + gamma * (g.z - q.z); o.w = a.w + gamma * (g.w - q.w);
    reinterpret_cast<float4 *>(wp)[v] = o;
    reinterpret_cast<float4 *>(w)[v] = o;
    const long long i = 4 * v;
    if (shadow && i >= w2_off && i < w2_off + w2_len)
      reinterpret_cast<uint2 *>(shadow)[(i - w2_off) / 4] = make_uint2(pack_bf16x2(o.x, o.y), pack_bf16x2(o.z, o.w));
  }
  if (blockIdx.x == 0 && threadIdx.x < (int)(P - 4 * nv4)) {
    const long long i = 4 * nv4 + threadIdx.x;
    const float nv = w[i] + gamma * (wbar[i] - wp[i]);
    wp[i] = nv;
    w[i] = nv;
    if (shadow && i >= w2_off && i < w2_off + w2_len) shadow[i - w2_off] = __float2bfloat16_rn(nv);
  }
}

void launch_momentum(cudaStream_t s, float *w, float *wbar_p_to_new, const float *wbar,
                     long long P, float gamma, long long w2_off, long long w2_len,
                     __nv_bfloat16 *shadow) {
  const bool aligned = (((uintptr_t)w | (uintptr_t)wbar_p_to_new | (uintptr_t)wbar) & 15) == 0 && (w2_off & 3) == 0;
  if (aligned)
    k_momentum4<<<148 * 4, 256, 0, s>>>(w, wbar_p_to_new, wbar, P, gamma, w2_off, w2_len, shadow);
  else
    k_momentum<<<148 * 8, 256, 0, s>>>(w, wbar_p_to_new, wbar, P, gamma, w2_off, w2_len, shadow);
}

// local-group merge: S = sum_i alpha_i w_i read directly from every replica
__global__ void k_group_reduce(const float *const *__restrict__ reps,
                               const float *__restrict__ alpha, int n, long long P,
                               const float *__restrict__ wbar, float *__restrict__ wp, float gamma) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < P;
       i += (long long)gridDim.x * blockDim.x) {
    float a = 0.f;
    for (int k = 0; k < n; ++k) a = fmaf(alpha[k], reps[k][i], a);
    wp[i] = a + gamma * (wbar[i] - wp[i]);
  }
}

void launch_group_reduce(cudaStream_t s, const float *const *reps_dev, const float *alpha_dev,
                         int n, long long P, const float *wbar, float *wbar_p_to_new,
                         float gamma) {
  k_group_reduce<<<148 * 8, 256, 0, s>>>(reps_dev, alpha_dev, n, P, wbar, wbar_p_to_new, gamma);
}

__global__ void k_reset_from(const float *__restrict__ src, float *__restrict__ w,
                             float *__restrict__ wnew, long long P, long long w2_off,
                             long long w2_len, __nv_bfloat16 *__restrict__ shadow) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < P;
       i += (long long)gridDim.x * blockDim.x) {
    const float v = src[i];
    w[i] = v;
    if (wnew != src) wnew[i] = v;
    if (shadow && i >= w2_off && i < w2_off + w2_len) shadow[i - w2_off] = __float2bfloat16_rn(v);
  }
}

void launch_reset_from(cudaStream_t s, const float *src, float *w, float *wbar_new, long long P,
                       long long w2_off, long long w2_len, __nv_bfloat16 *shadow) {
  k_reset_from<<<148 * 8, 256, 0, s>>>(src, w, wbar_new, P, w2_off, w2_len, shadow);
}

__global__ void k_f32_to_bf16(const float *__restrict__ src, __nv_bfloat16 *__restrict__ dst,
                              long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = __float2bfloat16_rn(src[i]);
}

void launch_f32_to_bf16(cudaStream_t s, const float *src, __nv_bfloat16 *dst, long long n) {
  k_f32_to_bf16<<<148 * 8, 256, 0, s>>>(src, dst, n);
}

}  // namespace as

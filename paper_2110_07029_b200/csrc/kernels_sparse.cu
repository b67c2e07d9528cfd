// Small kernels of the Adaptive SGD step (sm_100a): device batch builder (a2),
// label terms and the pass-1 combine with db1's fused SGD (a5), column sums
// with fused SGD (fp32 parity mode), the loss mean.  The SpMM and dW1 are in
// kernels_segmm.cu, the transposes in kernels_transpose.cu.
// P:N = PAPER.md line N; Rk = DESIGN.md reading k.
#include <cfloat>

#include "common.cuh"

namespace as {

// =====================================================================
// Step a2 on the device: gather `rows` samples of the resident dataset at
// stream positions [pos, pos+rows) (R10 order) into a rebased batch CSR.
// =====================================================================
// one CTA: stream position -> dataset id, row / label lengths, their scans
// (rebased row_ptr / lab_ptr) and the step descriptor
__global__ void __launch_bounds__(1024) k_gather_scan(const int64_t *__restrict__ rp,
                                                      const int64_t *__restrict__ lp,
                                                      const int64_t *__restrict__ order, int64_t n,
                                                      int64_t pos, int rows,
                                                      int64_t *__restrict__ row_ptr,
                                                      int64_t *__restrict__ lab_ptr,
                                                      int64_t *__restrict__ ids,
                                                      StepDesc *__restrict__ desc, int nnz_cap,
                                                      int lab_cap) {
  griddep_wait();
  __shared__ long long wa[32], wb[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  long long ca = 0, cb = 0;
  for (int c = 0; c < rows; c += 1024) {
    const int i = c + threadIdx.x;
    long long a = 0, b = 0;
    if (i < rows) {
      const int64_t p = (pos + i) % n;
      const int64_t id = order ? order[p] : p;
      ids[i] = id;
      a = rp[id + 1] - rp[id];
      b = lp[id + 1] - lp[id];
    }
    long long ia = a, ib = b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long ya = __shfl_up_sync(0xffffffffu, ia, o), yb = __shfl_up_sync(0xffffffffu, ib, o);
      if (lane >= o) { ia += ya; ib += yb; }
    }
    if (lane == 31) { wa[w] = ia; wb[w] = ib; }
    __syncthreads();
    if (w == 0) {
      long long xa = wa[lane], xb = wb[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long ya = __shfl_up_sync(0xffffffffu, xa, o), yb = __shfl_up_sync(0xffffffffu, xb, o);
        if (lane >= o) { xa += ya; xb += yb; }
      }
      wa[lane] = xa; wb[lane] = xb;
    }
    __syncthreads();
    if (i < rows) {
      row_ptr[i + 1] = ca + (w > 0 ? wa[w - 1] : 0) + ia;
      lab_ptr[i + 1] = cb + (w > 0 ? wb[w - 1] : 0) + ib;
    }
    const long long ta = wa[31], tb = wb[31];
    __syncthreads();
    ca += ta;
    cb += tb;
  }
  if (threadIdx.x == 0) {
    row_ptr[0] = 0;
    lab_ptr[0] = 0;
    desc->rows = rows;
    desc->nnz = (int)ca;
    desc->nlab = (int)cb;
    desc->U = 0;
    desc->V = 0;
    desc->n_long = 0;
    desc->err = (ca > nnz_cap || cb > lab_cap) ? 1 : 0;
  }
}

// one CTA per batch row: copy its entries and write the entry -> row maps
__global__ void k_gather_copy(const int64_t *__restrict__ rp, const int32_t *__restrict__ dcol,
                              const float *__restrict__ dval, const int64_t *__restrict__ lp,
                              const int32_t *__restrict__ dlab, const int64_t *__restrict__ ids,
                              const int64_t *__restrict__ row_ptr,
                              const int64_t *__restrict__ lab_ptr, int32_t *__restrict__ col,
                              float *__restrict__ val, int32_t *__restrict__ lab,
                              int32_t *__restrict__ rid, int32_t *__restrict__ lrid,
                              const StepDesc *__restrict__ desc) {
  griddep_wait();
  if (desc->err) return;
  const int r = blockIdx.x;
  const int64_t id = ids[r];
  const int64_t s0 = rp[id], n0 = rp[id + 1] - s0, d0 = row_ptr[r];
  for (int64_t j = threadIdx.x; j < n0; j += blockDim.x) {
    col[d0 + j] = dcol[s0 + j];
    val[d0 + j] = dval[s0 + j];
    rid[d0 + j] = r;
  }
  const int64_t s1 = lp[id], n1 = lp[id + 1] - s1, d1 = lab_ptr[r];
  for (int64_t j = threadIdx.x; j < n1; j += blockDim.x) {
    lab[d1 + j] = dlab[s1 + j];
    lrid[d1 + j] = r;
  }
}

// The batch is a CONTIGUOUS slice [p0, p0 + rows) of the resident dataset
// (stream order = dataset order, no wrap): its col / val / lab are used in
// place, and one kernel writes the rebased pointers, the entry -> row maps and
// the descriptor (warp per row).
__global__ void k_slice_batch(const int64_t *__restrict__ rp, const int64_t *__restrict__ lp, int64_t p0, int rows,
                              int64_t *__restrict__ row_ptr, int64_t *__restrict__ lab_ptr,
                              int32_t *__restrict__ rid, int32_t *__restrict__ lrid, StepDesc *__restrict__ desc,
                              int nnz_cap, int lab_cap) {
  griddep_wait();
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int64_t b0 = rp[p0], l0 = lp[p0];
  if (r < rows) {
    const int64_t s = rp[p0 + r] - b0, e = rp[p0 + r + 1] - b0;
    const int64_t ls = lp[p0 + r] - l0, le = lp[p0 + r + 1] - l0;
    if (lane == 0) {
      row_ptr[r + 1] = e;
      lab_ptr[r + 1] = le;
    }
    for (int64_t j = s + lane; j < e; j += 32) rid[j] = r;
    for (int64_t j = ls + lane; j < le; j += 32) lrid[j] = r;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    row_ptr[0] = 0;
    lab_ptr[0] = 0;
    const long long nnz = rp[p0 + rows] - b0, nl = lp[p0 + rows] - l0;
    desc->rows = rows;
    desc->nnz = (int)nnz;
    desc->nlab = (int)nl;
    desc->U = 0;
    desc->V = 0;
    desc->n_long = 0;
    desc->err = (nnz > nnz_cap || nl > lab_cap) ? 1 : 0;
  }
}

void launch_slice_batch(cudaStream_t s, const int64_t *ds_row_ptr, const int64_t *ds_lab_ptr, int64_t p0,
                        int rows, int64_t *row_ptr, int64_t *lab_ptr, int32_t *rid, int32_t *lrid,
                        StepDesc *desc, int nnz_cap, int lab_cap) {
  launch_pdl(k_slice_batch, dim3(ceil_div((long long)rows * 32, 256)), dim3(256), 0, s, ds_row_ptr, ds_lab_ptr, p0,
             rows, row_ptr, lab_ptr, rid, lrid, desc, nnz_cap, lab_cap);
}

void launch_gather_batch(cudaStream_t s, const int64_t *ds_row_ptr, const int32_t *ds_col,
                         const float *ds_val, const int64_t *ds_lab_ptr, const int32_t *ds_lab,
                         const int64_t *order, int64_t n, int64_t pos, int rows,
                         int64_t *row_ptr, int32_t *col, float *val, int64_t *lab_ptr,
                         int32_t *lab, int64_t *ids, int32_t *rid, int32_t *lrid, StepDesc *desc,
                         int nnz_cap, int lab_cap) {
  launch_pdl(k_gather_scan, dim3(1), dim3(1024), 0, s, ds_row_ptr, ds_lab_ptr, order, n, pos, rows, row_ptr,
             lab_ptr, ids, desc, nnz_cap, lab_cap);
  launch_pdl(k_gather_copy, dim3(rows), dim3(128), 0, s, ds_row_ptr, ds_col, ds_val, ds_lab_ptr, ds_lab, ids,
             row_ptr, lab_ptr, col, val, lab, rid, lrid, desc);
}

// =====================================================================
// Label terms (R3): zsum_r = (1/k_r) sum_{y in Y_r} z_ry and
// labW_r = (1/k_r) sum_{y in Y_r} W2T[y]  (fp32 master weights).  Warp per row.
// =====================================================================
#ifndef AS_LT_G
#define AS_LT_G 8
#endif
template <int H>
__global__ void k_label_terms(const StepDesc *__restrict__ desc, const int64_t *__restrict__ lab_ptr,
                              const int32_t *__restrict__ lab, const float *__restrict__ Hf,
                              const float *__restrict__ W2T, const float *__restrict__ b2,
                              float *__restrict__ zsum, float *__restrict__ labW) {
  griddep_wait();
  constexpr int V = H / 128;
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (r >= desc->rows) return;
  const int64_t s = lab_ptr[r], e = lab_ptr[r + 1];
  const float inv_k = 1.0f / (float)(e - s);
  float4 hr[V], lw[V];
#pragma unroll
  for (int q = 0; q < V; ++q) {
    hr[q] = reinterpret_cast<const float4 *>(Hf + (size_t)r * H)[lane + 32 * q];
    lw[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float zs = 0.f;
  // labels AS_LT_G at a time: all their W2T rows (and b2 values) in flight at
  // once; padding slots add zeros (same sums for any group size)
  for (int64_t j0 = s; j0 < e; j0 += AS_LT_G) {
    float4 w[AS_LT_G][V];
    float bb[AS_LT_G];
#pragma unroll
    for (int u = 0; u < AS_LT_G; ++u) {
      const bool ok = j0 + u < e;
      const int y = ok ? lab[j0 + u] : 0;
      bb[u] = ok ? b2[y] : 0.f;
#pragma unroll
      for (int q = 0; q < V; ++q)
        w[u][q] = ok ? reinterpret_cast<const float4 *>(W2T + (size_t)y * H)[lane + 32 * q]
                     : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < AS_LT_G; ++u) {
      float d = 0.f;
#pragma unroll
      for (int q = 0; q < V; ++q) {
        d = fmaf(hr[q].x, w[u][q].x, fmaf(hr[q].y, w[u][q].y, fmaf(hr[q].z, w[u][q].z, fmaf(hr[q].w, w[u][q].w, d))));
        lw[q].x += w[u][q].x; lw[q].y += w[u][q].y; lw[q].z += w[u][q].z; lw[q].w += w[u][q].w;
      }
      zs += warp_sum(d) + bb[u];
    }
  }
  if (lane == 0) zsum[r] = zs * inv_k;
#pragma unroll
  for (int q = 0; q < V; ++q) {
    float4 o = lw[q];
    o.x *= inv_k; o.y *= inv_k; o.z *= inv_k; o.w *= inv_k;
    reinterpret_cast<float4 *>(labW + (size_t)r * H)[lane + 32 * q] = o;
  }
}

void launch_label_terms(cudaStream_t s, int h, const StepDesc *desc, int b_max,
                        const int64_t *lab_ptr, const int32_t *lab, const float *Hf,
                        const float *W2T, const float *b2, float *zsum, float *labW) {
  const int g = ceil_div((long long)b_max * 32, 256);
  if (h == 128)
    launch_pdl(k_label_terms<128>, dim3(g), dim3(256), 0, s, desc, lab_ptr, lab, Hf, W2T, b2, zsum, labW);
  else
    launch_pdl(k_label_terms<256>, dim3(g), dim3(256), 0, s, desc, lab_ptr, lab, Hf, W2T, b2, zsum, labW);
}

// =====================================================================
// Combine the split-C partials of output pass 1 (online softmax in log2
// units): LSE_r, loss_r = LSE_r - zsum_r, dH_r = (O_r/l_r - labW_r)/B and
// dA_r = dH_r * [A_r > 0]  (R3, R4).  CTA = 32 rows x COMBINE_CW columns.  Partial
// layout: pm, pl [split][bpad]; pO [split][h][bpad] (coalesced TC epilogue).
// =====================================================================
// columns per combine CTA: 8 = one per warp (A/B on B200: 16 and 32 slower)
#ifndef COMBINE_CW
#define COMBINE_CW 8
#endif
static_assert(COMBINE_CW % 8 == 0, "one or more columns per warp");
// slot count up to which the combine holds all of a thread's partials in registers
#ifndef COMBINE_MAXS
#define COMBINE_MAXS 24
#endif
__global__ void __launch_bounds__(256) k_combine_bf16(
    const StepDesc *__restrict__ desc, int h, int bpad, int splits, const float *__restrict__ pm,
    const float *__restrict__ pl, const float *__restrict__ pO, const float *__restrict__ labW,
    const float *__restrict__ zsum, const float *__restrict__ Hf, const int64_t *__restrict__ lab_ptr,
    float *__restrict__ lse2, float *__restrict__ lsep, float *__restrict__ wrow,
    float *__restrict__ lossr, float *__restrict__ dA, float *__restrict__ db1p,
    int *__restrict__ db1cnt, float *__restrict__ b1, float lr, float *__restrict__ dbg_db1,
    float *__restrict__ dbg_dHs, __nv_bfloat16 *__restrict__ Hx) {
  griddep_wait();
  // pass 2's B_ext row (the FOLD K-step): [1, 1, 1, -(LSE_r + ln B) in three
  // bf16 parts, 0 ...]; padding rows -1e30 (p = 0)
  auto put_hx = [&](int row, float negL) {
    if (!Hx) return;
    const float hi = __bfloat162float(__float2bfloat16_rn(negL));
    const float r1 = negL - hi;
    const float mid = __bfloat162float(__float2bfloat16_rn(r1));
    const float lo = r1 - mid;
    uint4 *o = reinterpret_cast<uint4 *>(Hx + (size_t)row * 16);
    o[0] = make_uint4(pack_bf16x2(1.f, 1.f), pack_bf16x2(1.f, hi), pack_bf16x2(mid, lo), 0u);
    o[1] = make_uint4(0u, 0u, 0u, 0u);
  };
  // CTA = 32 rows x COMBINE_CW columns (8 warps); partial reads coalesced over rows
  const int rx = threadIdx.x & 31, jy = threadIdx.x >> 5;
  const int B = desc->rows;
  if (blockIdx.x * 32 >= B) {         // a CTA of padding rows only
    const int r = blockIdx.x * 32 + rx;
    if (jy == 0 && r < bpad && blockIdx.y == 0) { lsep[r] = -INFINITY; wrow[r] = 0.f; put_hx(r, -1e30f); }
    return;
  }
  const bool live = blockIdx.x * 32 + rx < B;
  const int r = live ? blockIdx.x * 32 + rx : B - 1;   // padding lanes shadow a live row
  if (!live && jy == 0 && blockIdx.y == 0) {
    lsep[blockIdx.x * 32 + rx] = -INFINITY;
    wrow[blockIdx.x * 32 + rx] = 0.f;
    put_hx(blockIdx.x * 32 + rx, -1e30f);
  }
  extern __shared__ float sc[];             // [splits][32] per-slot scales of the rows
  // label term and activation of this thread's columns, loaded before the
  // slot reductions so their latency hides under them
  constexpr int NCW = COMBINE_CW / 8;
  const int j0 = blockIdx.y * COMBINE_CW + jy;
  float lwv[NCW], hv[NCW];
#pragma unroll
  for (int c = 0; c < NCW; ++c) {
    lwv[c] = labW[(size_t)r * h + j0 + 8 * c];
    hv[c] = Hf[(size_t)r * h + j0 + 8 * c];
  }
  // every slot loop is unrolled 12-wide so a thread keeps 12 partial loads in
  // flight (the partials are L2-resident right after pass 1)
  // M_r and l_r: warp jy reduces slots jy, jy + 8, ...; the 8 warp partials
  // are combined in warp order (max is exact; the sum order is fixed)
  // splits <= COMBINE_MAXS (every b >= 128 * SMs / COMBINE_MAXS): every
  // partial this thread reads -- its slots' m and l, and the column's O of
  // every slot -- is loaded up front (one memory round trip instead of one per
  // phase); the same operations in the same order as the loop form below
  constexpr int MAXS = COMBINE_MAXS, MS8 = (MAXS + 7) / 8;
  const bool pre = splits <= MAXS;
  float pmv[MS8], plv[MS8], ov[MAXS][NCW];
  if (pre) {
#pragma unroll
    for (int k = 0; k < MS8; ++k) {
      const int s = jy + 8 * k;
      if (s < splits) { pmv[k] = pm[(size_t)s * bpad + r]; plv[k] = pl[(size_t)s * bpad + r]; }
    }
#pragma unroll
    for (int s = 0; s < MAXS; ++s)
      if (s < splits) {
#pragma unroll
        for (int c = 0; c < NCW; ++c) ov[s][c] = pO[((size_t)s * h + j0 + 8 * c) * bpad + r];
      }
  }
  __shared__ float red[2][8][33];
  float M = -FLT_MAX;
  if (pre) {
#pragma unroll
    for (int k = 0; k < MS8; ++k)
      if (jy + 8 * k < splits) M = fmaxf(M, pmv[k]);
  } else {
    for (int s = jy; s < splits; s += 8) M = fmaxf(M, pm[(size_t)s * bpad + r]);
  }
  red[0][jy][rx] = M;
  __syncthreads();
  M = red[0][0][rx];
#pragma unroll
  for (int k = 1; k < 8; ++k) M = fmaxf(M, red[0][k][rx]);
  float l = 0.f;
  if (pre) {
#pragma unroll
    for (int k = 0; k < MS8; ++k) {
      const int s = jy + 8 * k;
      if (s < splits) {
        const float e = pmv[k] == -FLT_MAX ? 0.f : exp2f(pmv[k] - M);
        sc[s * 32 + rx] = e;
        l = fmaf(plv[k], e, l);
      }
    }
  } else {
    for (int s = jy; s < splits; s += 8) {
      const float ms = pm[(size_t)s * bpad + r];
      const float e = ms == -FLT_MAX ? 0.f : exp2f(ms - M);
      sc[s * 32 + rx] = e;
      l = fmaf(pl[(size_t)s * bpad + r], e, l);
    }
  }
  red[1][jy][rx] = l;
  __syncthreads();
  l = red[1][0][rx];
#pragma unroll
  for (int k = 1; k < 8; ++k) l += red[1][k][rx];
  const float invB = 1.0f / (float)B, invl = 1.0f / l;
  __shared__ float cs[COMBINE_CW][33];        // dA of this CTA's rows x columns (db1 partial)
  // the warp's COMBINE_CW / 8 columns j0 + 8c advance together over the slots
  // (their loads in flight at once); same per-column fmaf order as one by one
  float o[NCW];
#pragma unroll
  for (int c = 0; c < NCW; ++c) o[c] = 0.f;
  if (pre) {
#pragma unroll
    for (int s = 0; s < MAXS; ++s)
      if (s < splits) {
        const float w = sc[s * 32 + rx];
#pragma unroll
        for (int c = 0; c < NCW; ++c) o[c] = fmaf(ov[s][c], w, o[c]);
      }
  } else {
#pragma unroll 6
    for (int s = 0; s < splits; ++s) {
      const float w = sc[s * 32 + rx];
#pragma unroll
      for (int c = 0; c < NCW; ++c) o[c] = fmaf(pO[((size_t)s * h + j0 + 8 * c) * bpad + r], w, o[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < NCW; ++c) {
    const int j = j0 + 8 * c;
    const float dh = (o[c] * invl - lwv[c]) * invB;
    const float da = live && hv[c] > 0.f ? dh : 0.f;
    if (live) dA[(size_t)r * h + j] = da;
    if (dbg_dHs && live) dbg_dHs[(size_t)r * h + j] = o[c] * invl * invB;   // softmax part of dH (tests)
    cs[j - blockIdx.y * COMBINE_CW][rx] = da;
  }
  // db1 = sum_r dA_r (step a5), fused: per-CTA column sums over its 32 rows in
  // row order, then the last row block to arrive for this column group adds
  // the partials in row-block order and applies b1 -= lr db1 (deterministic)
  __syncthreads();
  const int nrb = (B + 31) / 32;
  if (threadIdx.x < COMBINE_CW) {
    float g = 0.f;
    for (int k = 0; k < 32; ++k) g += cs[threadIdx.x][k];
    db1p[(size_t)blockIdx.x * h + blockIdx.y * COMBINE_CW + threadIdx.x] = g;
    __threadfence();
  }
  __syncthreads();
  __shared__ int last;
  if (threadIdx.x == 0) last = atomicAdd(&db1cnt[blockIdx.y], 1) == nrb - 1;
  __syncthreads();
  if (last) {
    // every partial in flight at once: warp jy sums columns CW/8 jy ... over
    // the row blocks (lane k takes blocks k, k + 32, ...; fixed xor tree)
    __threadfence();
#pragma unroll
    for (int cc = 0; cc < COMBINE_CW / 8; ++cc) {
      const int c = blockIdx.y * COMBINE_CW + (COMBINE_CW / 8) * jy + cc;
      float g = 0.f;
      for (int k = rx; k < nrb; k += 32) g += __ldcg(db1p + (size_t)k * h + c);
      g = warp_sum(g);
      if (rx == 0) {
        b1[c] -= lr * g;
        if (dbg_db1) dbg_db1[c] = g;
      }
    }
    if (threadIdx.x == 0) db1cnt[blockIdx.y] = 0;
  }
  if (jy == 0 && live && blockIdx.y == 0) {
    const float L2 = M + log2f(l);
    lse2[r] = L2;
    lsep[r] = -(L2 + log2f((float)B));   // pass 2: p / B = 2^(s log2e + lsep), lsep = -lse'
    put_hx(r, lsep[r] * 0.69314718055994531f);      // FOLD: -(LSE + ln B), natural units
    // pass 2's label weight of the row, 1 / (k_r B) (R3), same fp32 operations
    // as the label transpose's per-entry weights
    wrow[r] = (1.0f / (float)B) / (float)(lab_ptr[r + 1] - lab_ptr[r]);
    lossr[r] = L2 * 0.69314718055994531f - zsum[r];
  }
}

void launch_combine_bf16(cudaStream_t s, int h, const StepDesc *desc, int b_max, int bpad,
                         int splits, const float *pm, const float *pl, const float *pO,
                         const float *labW, const float *zsum, const float *Hf, const int64_t *lab_ptr,
                         float *lse2, float *lsep, float *wrow, float *lossr, float *dA, float *db1p,
                         int *db1cnt, float *b1, float lr, float *dbg_db1, float *dbg_dHs,
                         __nv_bfloat16 *Hx) {
  launch_pdl(k_combine_bf16, dim3(ceil_div(bpad, 32), h / COMBINE_CW), dim3(256), (size_t)splits * 32 * 4, s, desc, h,
             bpad, splits, pm, pl, pO, labW, zsum, Hf, lab_ptr, lse2, lsep, wrow, lossr, dA, db1p, db1cnt, b1, lr,
             dbg_db1, dbg_dHs, Hx);
}

// =====================================================================
// Column sums over the batch rows with fused SGD: g_c = sum_r X[r][c] (fixed
// order), param[c] -= lr * g_c.  Used for db1 (X = dA) and, in the fp32
// mode, db2 (X = dZ).  Deterministic.
// =====================================================================
__global__ void __launch_bounds__(1024) k_colsum_sgd(const StepDesc *__restrict__ desc, int ncols,
                                                     const float *__restrict__ X, long long ldx,
                                                     float *__restrict__ param, float lr,
                                                     float *__restrict__ grad_out) {
  __shared__ float red[32][33];
  const int c = blockIdx.x * 32 + threadIdx.x;
  const int B = desc->rows;
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  if (c < ncols) {
    int r = threadIdx.y;
    for (; r + 96 < B; r += 128) {
      a0 += X[(size_t)r * ldx + c];
      a1 += X[(size_t)(r + 32) * ldx + c];
      a2 += X[(size_t)(r + 64) * ldx + c];
      a3 += X[(size_t)(r + 96) * ldx + c];
    }
    for (; r < B; r += 32) a0 += X[(size_t)r * ldx + c];
  }
  red[threadIdx.y][threadIdx.x] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  if (threadIdx.y == 0 && c < ncols) {
    float g = 0.f;
#pragma unroll 8
    for (int q = 0; q < 32; ++q) g += red[q][threadIdx.x];
    param[c] -= lr * g;
    if (grad_out) grad_out[c] = g;
  }
}

void launch_colsum_sgd(cudaStream_t s, const StepDesc *desc, int n_rows_cap, int ncols,
                       const float *X, long long ldx, float *param, float lr, float *grad_out) {
  (void)n_rows_cap;
  k_colsum_sgd<<<ceil_div(ncols, 32), dim3(32, 32), 0, s>>>(desc, ncols, X, ldx, param, lr,
                                                             grad_out);
}

// mean of the per-row losses (as_train_step with loss_out)
__global__ void __launch_bounds__(1024) k_loss_mean(const StepDesc *__restrict__ desc,
                                                    const float *__restrict__ lossr,
                                                    float *__restrict__ loss) {
  __shared__ float red[1024];
  const int B = desc->rows;
  float a = 0.f;
  for (int r = threadIdx.x; r < B; r += 1024) a += lossr[r];
  red[threadIdx.x] = a;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *loss = red[0] / (float)B;
}

void launch_loss_mean(cudaStream_t s, const StepDesc *desc, const float *lossr, float *loss) {
  k_loss_mean<<<1, 1024, 0, s>>>(desc, lossr, loss);
}

}  // namespace as

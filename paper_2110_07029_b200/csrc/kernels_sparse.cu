// Sparse / bandwidth-bound kernels of the Adaptive SGD step (sm_100a):
// device batch builder (a2), batch transposes (a3), CSR SpMM forward (a4),
// label terms and the pass-1 combine (a5), column sums with fused SGD,
// the deterministic segmented first-layer gradient with fused SGD (a7).
// P:N = PAPER.md line N; Rk = DESIGN.md reading k.
#include <cfloat>

#include "common.cuh"

namespace as {

// =====================================================================
// Device-wide exclusive scan of int32 (3 kernels, 4096 elements / block).
// =====================================================================
__global__ void __launch_bounds__(1024) k_scan_local(const int32_t *__restrict__ in,
                                                     int32_t *__restrict__ out,
                                                     int32_t *__restrict__ totals,
                                                     const int *__restrict__ n_dev) {
  __shared__ int32_t warp_tot[32];
  const int n = *n_dev;
  const int base = blockIdx.x * kScanTile;
  if (base >= n && blockIdx.x > 0) return;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  int v[4], s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int idx = base + t * 4 + i;
    v[i] = idx < n ? in[idx] : 0;
    s += v[i];
  }
  int incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_tot[w] = incl;
  __syncthreads();
  if (w == 0) {
    int x = warp_tot[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    warp_tot[lane] = x;  // inclusive over warps
  }
  __syncthreads();
  int run = incl - s + (w > 0 ? warp_tot[w - 1] : 0);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int idx = base + t * 4 + i;
    if (idx < n) out[idx] = run;
    run += v[i];
  }
  if (t == 1023) totals[blockIdx.x] = warp_tot[31];
}

__global__ void __launch_bounds__(1024) k_scan_totals(int32_t *__restrict__ totals,
                                                      const int *__restrict__ n_dev) {
  // exclusive scan of ceil(n / kScanTile) block totals, sequential chunks of 1024
  __shared__ int32_t buf[1024];
  const int nb = (*n_dev + kScanTile - 1) / kScanTile;
  int carry = 0;
  for (int c = 0; c < nb; c += 1024) {
    const int i = c + threadIdx.x;
    const int x = i < nb ? totals[i] : 0;
    buf[threadIdx.x] = x;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      const int y = threadIdx.x >= o ? buf[threadIdx.x - o] : 0;
      __syncthreads();
      buf[threadIdx.x] += y;
      __syncthreads();
    }
    if (i < nb) totals[i] = carry + buf[threadIdx.x] - x;
    const int last = buf[1023];
    __syncthreads();
    carry += last;
  }
}

__global__ void k_scan_add(int32_t *__restrict__ out, const int32_t *__restrict__ totals,
                           const int *__restrict__ n_dev) {
  const int n = *n_dev;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < n) out[idx] += totals[idx / kScanTile];
}

static void scan_exclusive(cudaStream_t s, const int32_t *in, int32_t *out, int32_t *totals,
                           const int *n_dev, int cap) {
  const int nb = ceil_div(cap > 0 ? cap : 1, kScanTile);
  k_scan_local<<<nb, 1024, 0, s>>>(in, out, totals, n_dev);
  k_scan_totals<<<1, 1024, 0, s>>>(totals, n_dev);
  k_scan_add<<<ceil_div(cap > 0 ? cap : 1, 256), 256, 0, s>>>(out, totals, n_dev);
}

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
// Step a3: batch transposes.  A stable LSD radix sort of (key, position)
// pairs (8-bit digits, per-tile stable ranking with warp match), then
// segment extraction.  Deterministic and bit-exact: the output is THE stable
// sort by key, rows ascending inside a key (brute-force pinned in tests).
// =====================================================================
__global__ void k_rowid(const int64_t *__restrict__ ptr, const int32_t *__restrict__ key,
                        int rows, int32_t *__restrict__ rowid, uint32_t *__restrict__ k0,
                        uint32_t *__restrict__ v0) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const int64_t s = ptr[warp], e = ptr[warp + 1];
  for (int64_t j = s + lane; j < e; j += 32) {
    rowid[j] = warp;
    k0[j] = (uint32_t)key[j];
    v0[j] = (uint32_t)j;
  }
}

__global__ void __launch_bounds__(256) k_radix_hist(const uint32_t *__restrict__ keys,
                                                    const int *__restrict__ n_dev, int shift,
                                                    uint32_t *__restrict__ hist) {
  __shared__ uint32_t h[256];
  const int n = *n_dev;
  const int nb = (n + kSortTile - 1) / kSortTile;
  if ((int)blockIdx.x >= nb) return;
  h[threadIdx.x] = 0;
  __syncthreads();
  const int base = blockIdx.x * kSortTile;
  for (int i = threadIdx.x; i < kSortTile; i += 256) {
    const int idx = base + i;
    if (idx < n) atomicAdd(&h[(keys[idx] >> shift) & 255u], 1u);
  }
  __syncthreads();
  hist[threadIdx.x * nb + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(1024) k_radix_scan(uint32_t *__restrict__ hist,
                                                     const int *__restrict__ n_dev) {
  __shared__ uint32_t buf[1024];
  const int nb = (*n_dev + kSortTile - 1) / kSortTile;
  const int total = nb * 256;
  uint32_t carry = 0;
  for (int c = 0; c < total; c += 1024) {
    const int i = c + threadIdx.x;
    const uint32_t x = i < total ? hist[i] : 0;
    buf[threadIdx.x] = x;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      const uint32_t y = threadIdx.x >= o ? buf[threadIdx.x - o] : 0;
      __syncthreads();
      buf[threadIdx.x] += y;
      __syncthreads();
    }
    if (i < total) hist[i] = carry + buf[threadIdx.x] - x;
    const uint32_t last = buf[1023];
    __syncthreads();
    carry += last;
  }
}

__global__ void __launch_bounds__(256) k_radix_scatter(const uint32_t *__restrict__ kin,
                                                       const uint32_t *__restrict__ vin,
                                                       uint32_t *__restrict__ kout,
                                                       uint32_t *__restrict__ vout,
                                                       const int *__restrict__ n_dev, int shift,
                                                       const uint32_t *__restrict__ hist) {
  __shared__ uint32_t base[256];
  __shared__ uint32_t wcnt[8][256];
  const int n = *n_dev;
  const int nb = (n + kSortTile - 1) / kSortTile;
  if ((int)blockIdx.x >= nb) return;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  base[t] = hist[t * nb + blockIdx.x];
  const uint32_t lt_mask = (1u << lane) - 1u;
  for (int round = 0; round < kSortTile / 256; ++round) {
    const int idx = blockIdx.x * kSortTile + round * 256 + t;
    const bool valid = idx < n;
    uint32_t k = 0, v = 0, dig = 256u + (uint32_t)lane;
    if (valid) {
      k = kin[idx];
      v = vin[idx];
      dig = (k >> shift) & 255u;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) wcnt[q][t] = 0;
    __syncthreads();
    const uint32_t peers = __match_any_sync(0xffffffffu, dig);
    const uint32_t rank = __popc(peers & lt_mask);
    if (valid && rank == 0) wcnt[w][dig] = __popc(peers);
    __syncthreads();
    if (valid) {
      uint32_t off = base[dig] + rank;
      for (int q = 0; q < w; ++q) off += wcnt[q][dig];
      kout[off] = k;
      vout[off] = v;
    }
    __syncthreads();
    uint32_t add = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) add += wcnt[q][t];
    base[t] += add;
    __syncthreads();
  }
}

__global__ void k_seg_flags(const uint32_t *__restrict__ kf, const uint32_t *__restrict__ vf,
                            const int32_t *__restrict__ rowid, const float *__restrict__ val_in,
                            const int *__restrict__ n_dev, int32_t *__restrict__ flags,
                            int32_t *__restrict__ seg_row, float *__restrict__ seg_val) {
  const int n = *n_dev;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const uint32_t p = vf[j];
  seg_row[j] = rowid[p];
  if (val_in) seg_val[j] = val_in[p];
  flags[j] = (j == 0 || kf[j] != kf[j - 1]) ? 1 : 0;
}

__global__ void k_seg_write(const uint32_t *__restrict__ kf, const int32_t *__restrict__ flags,
                            const int32_t *__restrict__ idx, const int *__restrict__ n_dev,
                            int32_t *__restrict__ seg_id, int32_t *__restrict__ seg_ptr,
                            int *__restrict__ nseg, int32_t *__restrict__ seg_of) {
  const int n = *n_dev;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (n == 0) {
    if (j == 0) {
      seg_ptr[0] = 0;
      *nseg = 0;
    }
    return;
  }
  if (j >= n) return;
  if (flags[j]) {
    seg_id[idx[j]] = (int32_t)kf[j];
    seg_ptr[idx[j]] = j;
  }
  if (seg_of) seg_of[j] = idx[j] + flags[j] - 1;   // segment of entry j
  if (j == n - 1) {
    const int U = idx[j] + flags[j];
    seg_ptr[U] = n;
    *nseg = U;
  }
}

void launch_transpose(cudaStream_t s, const int64_t *ptr, const int32_t *key, int rows,
                      const int *n_dev, int cap, int key_bits, uint32_t *k0, uint32_t *v0,
                      uint32_t *k1, uint32_t *v1, uint32_t *hist, int32_t *rowid, int32_t *flags,
                      int32_t *scan_tmp, int32_t *seg_id, int32_t *seg_ptr, int32_t *seg_row,
                      int *nseg_dev, const float *val_in, float *seg_val, int32_t *seg_of) {
  const int nb = ceil_div(cap > 0 ? cap : 1, kSortTile);
  k_rowid<<<ceil_div((long long)rows * 32, 256), 256, 0, s>>>(ptr, key, rows, rowid, k0, v0);
  uint32_t *ki = k0, *vi = v0, *ko = k1, *vo = v1;
  for (int shift = 0; shift < key_bits; shift += kSortBits) {
    k_radix_hist<<<nb, 256, 0, s>>>(ki, n_dev, shift, hist);
    k_radix_scan<<<1, 1024, 0, s>>>(hist, n_dev);
    k_radix_scatter<<<nb, 256, 0, s>>>(ki, vi, ko, vo, n_dev, shift, hist);
    uint32_t *tk = ki, *tv = vi;
    ki = ko; vi = vo; ko = tk; vo = tv;
  }
  const int g = ceil_div(cap > 0 ? cap : 1, 256);
  k_seg_flags<<<g, 256, 0, s>>>(ki, vi, rowid, val_in, n_dev, flags, seg_row, seg_val);
  int32_t *idx = scan_tmp;
  int32_t *totals = scan_tmp + (cap > 0 ? cap : 1);
  scan_exclusive(s, flags, idx, totals, n_dev, cap);
  k_seg_write<<<g, 256, 0, s>>>(ki, flags, idx, n_dev, seg_id, seg_ptr, nseg_dev, seg_of);
}

// lw[u] = 1 / (k_r B) for label entry u of the label-sorted batch (R3)
__global__ void k_label_weights(const StepDesc *__restrict__ desc, const int32_t *__restrict__ lrow,
                                const int64_t *__restrict__ lab_ptr, float *__restrict__ lw) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= desc->nlab) return;
  const int r = lrow[u];
  lw[u] = (1.0f / (float)desc->rows) / (float)(lab_ptr[r + 1] - lab_ptr[r]);
}

void launch_label_weights(cudaStream_t s, const StepDesc *desc, int cap, const int32_t *lrow,
                          const int64_t *lab_ptr, float *lw) {
  k_label_weights<<<ceil_div(cap > 0 ? cap : 1, 256), 256, 0, s>>>(desc, lrow, lab_ptr, lw);
}

// class -> label-segment map (value_is_index=1) or reset to -1 (value_is_index=0)
__global__ void k_class_map(const int32_t *__restrict__ lseg_id, const int *__restrict__ V_dev,
                            int32_t *__restrict__ cls_seg, int value_is_index) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= *V_dev) return;
  cls_seg[lseg_id[v]] = value_is_index ? v : -1;
}

void launch_class_map(cudaStream_t s, const int32_t *lseg_id, const int *V_dev, int cap,
                      int32_t *cls_seg, int value_is_index) {
  k_class_map<<<ceil_div(cap > 0 ? cap : 1, 256), 256, 0, s>>>(lseg_id, V_dev, cls_seg,
                                                                value_is_index);
}

// =====================================================================
// Step a4: A1 = X W1 + b1, H = ReLU(A1)  (P:51 forward; R4 mask A1 > 0).
// One CTA of 4 warps per batch row; each warp gathers every 4th non-zero of
// the row as whole 128-bit W1 row segments (h*4 bytes per nnz) with 4 rows in
// flight; the 4 warp partials are combined in a fixed order (deterministic).
// Rows >= B (up to the 128-row MMA tile) are written as zeros in H_bf16.
// =====================================================================
template <int H>
__global__ void __launch_bounds__(128) k_spmm(const StepDesc *__restrict__ desc,
                                              const int64_t *__restrict__ row_ptr,
                                              const int32_t *__restrict__ col,
                                              const float *__restrict__ val,
                                              const float *__restrict__ W1,
                                              const float *__restrict__ b1, float *__restrict__ Hf,
                                              __nv_bfloat16 *__restrict__ Hb) {
  constexpr int V = H / 128;  // float4 per lane
  __shared__ float4 part[4][32 * V];
  const int r = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (r >= desc->rows) {
    uint2 *hb = reinterpret_cast<uint2 *>(Hb + (size_t)r * H);
    for (int i = threadIdx.x; i < H / 4; i += 128) hb[i] = make_uint2(0u, 0u);
    return;
  }
  const int64_t s = row_ptr[r], e = row_ptr[r + 1];
  float4 acc[V];
#pragma unroll
  for (int q = 0; q < V; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 *W = reinterpret_cast<const float4 *>(W1);
  for (int64_t j0 = s + w; j0 < e; j0 += 16) {
    int c[4];
    float v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t j = j0 + 4 * u;
      c[u] = j < e ? col[j] : -1;
      v[u] = j < e ? val[j] : 0.f;
    }
    float4 x[4][V];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int q = 0; q < V; ++q)
        x[u][q] = c[u] >= 0 ? __ldg(&W[(size_t)c[u] * (H / 4) + lane + 32 * q])
                            : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int q = 0; q < V; ++q) {
        acc[q].x = fmaf(v[u], x[u][q].x, acc[q].x);
        acc[q].y = fmaf(v[u], x[u][q].y, acc[q].y);
        acc[q].z = fmaf(v[u], x[u][q].z, acc[q].z);
        acc[q].w = fmaf(v[u], x[u][q].w, acc[q].w);
      }
  }
#pragma unroll
  for (int q = 0; q < V; ++q) part[w][lane + 32 * q] = acc[q];
  __syncthreads();
  if (w == 0) {
    const float4 *B1 = reinterpret_cast<const float4 *>(b1);
#pragma unroll
    for (int q = 0; q < V; ++q) {
      const int i = lane + 32 * q;
      float4 a = part[0][i], p1 = part[1][i], p2 = part[2][i], p3 = part[3][i], bb = B1[i];
      a.x = (((a.x + p1.x) + p2.x) + p3.x) + bb.x;
      a.y = (((a.y + p1.y) + p2.y) + p3.y) + bb.y;
      a.z = (((a.z + p1.z) + p2.z) + p3.z) + bb.z;
      a.w = (((a.w + p1.w) + p2.w) + p3.w) + bb.w;
      a.x = fmaxf(a.x, 0.f); a.y = fmaxf(a.y, 0.f); a.z = fmaxf(a.z, 0.f); a.w = fmaxf(a.w, 0.f);
      reinterpret_cast<float4 *>(Hf + (size_t)r * H)[i] = a;
      reinterpret_cast<uint2 *>(Hb + (size_t)r * H)[i] =
          make_uint2(pack_bf16x2(a.x, a.y), pack_bf16x2(a.z, a.w));
    }
  }
}

void launch_spmm(cudaStream_t s, int h, const StepDesc *desc, int bpad, const int64_t *row_ptr,
                 const int32_t *col, const float *val, const float *W1, const float *b1, float *Hf,
                 __nv_bfloat16 *Hb) {
  if (h == 128)
    k_spmm<128><<<bpad, 128, 0, s>>>(desc, row_ptr, col, val, W1, b1, Hf, Hb);
  else
    k_spmm<256><<<bpad, 128, 0, s>>>(desc, row_ptr, col, val, W1, b1, Hf, Hb);
}

// =====================================================================
// Label terms (R3): zsum_r = (1/k_r) sum_{y in Y_r} z_ry and
// labW_r = (1/k_r) sum_{y in Y_r} W2T[y]  (fp32 master weights).  Warp per row.
// =====================================================================
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
  // labels 4 at a time: all four W2T rows (and b2 values) in flight at once
  for (int64_t j0 = s; j0 < e; j0 += 4) {
    float4 w[4][V];
    float bb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool ok = j0 + u < e;
      const int y = ok ? lab[j0 + u] : 0;
      bb[u] = ok ? b2[y] : 0.f;
#pragma unroll
      for (int q = 0; q < V; ++q)
        w[u][q] = ok ? reinterpret_cast<const float4 *>(W2T + (size_t)y * H)[lane + 32 * q]
                     : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
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
// dA_r = dH_r * [A_r > 0]  (R3, R4).  One CTA (h threads) per row.  Partial
// layout: pm, pl [split][bpad]; pO [split][h][bpad] (coalesced TC epilogue).
// =====================================================================
__global__ void __launch_bounds__(256) k_combine_bf16(
    const StepDesc *__restrict__ desc, int h, int bpad, int splits, const float *__restrict__ pm,
    const float *__restrict__ pl, const float *__restrict__ pO, const float *__restrict__ labW,
    const float *__restrict__ zsum, const float *__restrict__ Hf, const int64_t *__restrict__ lab_ptr,
    float *__restrict__ lse2, float *__restrict__ lsep, float *__restrict__ wrow,
    float *__restrict__ lossr, float *__restrict__ dA, float *__restrict__ db1p,
    int *__restrict__ db1cnt, float *__restrict__ b1, float lr, float *__restrict__ dbg_db1) {
  griddep_wait();
  // CTA = 32 rows x 16 columns (8 groups of 2); partial reads coalesced over rows
  const int rx = threadIdx.x & 31, jy = threadIdx.x >> 5;
  const int B = desc->rows;
  if (blockIdx.x * 32 >= B) {         // a CTA of padding rows only
    const int r = blockIdx.x * 32 + rx;
    if (jy == 0 && r < bpad && blockIdx.y == 0) { lsep[r] = INFINITY; wrow[r] = 0.f; }
    return;
  }
  const bool live = blockIdx.x * 32 + rx < B;
  const int r = live ? blockIdx.x * 32 + rx : B - 1;   // padding lanes shadow a live row
  if (!live && jy == 0 && blockIdx.y == 0) { lsep[blockIdx.x * 32 + rx] = INFINITY; wrow[blockIdx.x * 32 + rx] = 0.f; }
  extern __shared__ float sc[];             // [splits][32] per-slot scales of the rows
  // every slot loop is unrolled 12-wide so a thread keeps 12 partial loads in
  // flight (the partials are L2-resident right after pass 1)
  float M = -FLT_MAX;
#pragma unroll 12
  for (int s = 0; s < splits; ++s) M = fmaxf(M, pm[(size_t)s * bpad + r]);
  for (int s = jy; s < splits; s += 8) {
    const float ms = pm[(size_t)s * bpad + r];
    sc[s * 32 + rx] = ms == -FLT_MAX ? 0.f : exp2f(ms - M);
  }
  __syncthreads();
  float l = 0.f;
#pragma unroll 12
  for (int s = 0; s < splits; ++s) l = fmaf(pl[(size_t)s * bpad + r], sc[s * 32 + rx], l);
  const float invB = 1.0f / (float)B, invl = 1.0f / l;
  __shared__ float cs[16][33];                // dA of this CTA's rows x columns (db1 partial)
  for (int j = blockIdx.y * 16 + jy; j < h && j < blockIdx.y * 16 + 16; j += 8) {
    float o = 0.f;
#pragma unroll 12
    for (int s = 0; s < splits; ++s) o = fmaf(pO[((size_t)s * h + j) * bpad + r], sc[s * 32 + rx], o);
    const float dh = (o * invl - labW[(size_t)r * h + j]) * invB;
    const float da = live && Hf[(size_t)r * h + j] > 0.f ? dh : 0.f;
    if (live) dA[(size_t)r * h + j] = da;
    cs[j - blockIdx.y * 16][rx] = da;
  }
  // db1 = sum_r dA_r (step a5), fused: per-CTA column sums over its 32 rows in
  // row order, then the last row block to arrive for this column group adds
  // the partials in row-block order and applies b1 -= lr db1 (deterministic)
  __syncthreads();
  const int nrb = (B + 31) / 32;
  if (threadIdx.x < 16) {
    float g = 0.f;
    for (int k = 0; k < 32; ++k) g += cs[threadIdx.x][k];
    db1p[(size_t)blockIdx.x * h + blockIdx.y * 16 + threadIdx.x] = g;
    __threadfence();
  }
  __syncthreads();
  __shared__ int last;
  if (threadIdx.x == 0) last = atomicAdd(&db1cnt[blockIdx.y], 1) == nrb - 1;
  __syncthreads();
  if (last && threadIdx.x < 16) {
    __threadfence();
    const int c = blockIdx.y * 16 + threadIdx.x;
    float g = 0.f;
    for (int k = 0; k < nrb; ++k) g += __ldcg(db1p + (size_t)k * h + c);
    b1[c] -= lr * g;
    if (dbg_db1) dbg_db1[c] = g;
    if (threadIdx.x == 0) db1cnt[blockIdx.y] = 0;
  }
  if (jy == 0 && live && blockIdx.y == 0) {
    const float L2 = M + log2f(l);
    lse2[r] = L2;
    lsep[r] = L2 + log2f((float)B);   // pass 2: p / B = 2^(s log2e - lsep)
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
                         int *db1cnt, float *b1, float lr, float *dbg_db1) {
  launch_pdl(k_combine_bf16, dim3(ceil_div(bpad, 32), h / 16), dim3(256), (size_t)splits * 32 * 4, s, desc, h,
             bpad, splits, pm, pl, pO, labW, zsum, Hf, lab_ptr, lse2, lsep, wrow, lossr, dA, db1p, db1cnt, b1, lr,
             dbg_db1);
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

// =====================================================================
// Step a7: dW1[f] = sum_{(r,f)} x_rf * dA_r over the feature-sorted batch, in
// segment order (rows ascending) -- a deterministic segmented reduction, no
// float atomics -- with the SGD update W1[f] -= lr * dW1[f] fused.  Short
// segments: one warp each (grid-stride).  Segments longer than kLongSeg (the
// Zipf head) are queued and reduced by a whole CTA: warp q takes entries
// q, q+8, ... and the 8 partials are added in a fixed order.
// =====================================================================
template <int H>
__global__ void __launch_bounds__(256) k_dw1_short(StepDesc *__restrict__ desc,
                                                   const int32_t *__restrict__ seg_id,
                                                   const int32_t *__restrict__ seg_ptr,
                                                   const int32_t *__restrict__ seg_row,
                                                   const float *__restrict__ seg_val,
                                                   const float *__restrict__ dA,
                                                   float *__restrict__ W1, float lr,
                                                   int32_t *__restrict__ long_list,
                                                   float *__restrict__ dbg) {
  constexpr int V = H / 128;
  const int U = desc->U;
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int sg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; sg < U; sg += nw) {
    const int s = seg_ptr[sg], e = seg_ptr[sg + 1];
    if (e - s > kLongSeg) {
      if (lane == 0) long_list[atomicAdd(&desc->n_long, 1)] = sg;
      continue;
    }
    float4 acc[V];
#pragma unroll
    for (int q = 0; q < V; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = s; j < e; ++j) {
      const int r = seg_row[j];
      const float v = seg_val[j];
#pragma unroll
      for (int q = 0; q < V; ++q) {
        const float4 g = reinterpret_cast<const float4 *>(dA + (size_t)r * H)[lane + 32 * q];
        acc[q].x = fmaf(v, g.x, acc[q].x);
        acc[q].y = fmaf(v, g.y, acc[q].y);
        acc[q].z = fmaf(v, g.z, acc[q].z);
        acc[q].w = fmaf(v, g.w, acc[q].w);
      }
    }
    const size_t f = (size_t)seg_id[sg];
#pragma unroll
    for (int q = 0; q < V; ++q) {
      float4 *wp = reinterpret_cast<float4 *>(W1 + f * H) + lane + 32 * q;
      float4 w = *wp;
      w.x -= lr * acc[q].x; w.y -= lr * acc[q].y; w.z -= lr * acc[q].z; w.w -= lr * acc[q].w;
      *wp = w;
      if (dbg) reinterpret_cast<float4 *>(dbg + (size_t)sg * H)[lane + 32 * q] = acc[q];
    }
  }
}

template <int H>
__global__ void __launch_bounds__(256) k_dw1_long(const StepDesc *__restrict__ desc,
                                                  const int32_t *__restrict__ seg_id,
                                                  const int32_t *__restrict__ seg_ptr,
                                                  const int32_t *__restrict__ seg_row,
                                                  const float *__restrict__ seg_val,
                                                  const float *__restrict__ dA,
                                                  float *__restrict__ W1, float lr,
                                                  const int32_t *__restrict__ long_list,
                                                  float *__restrict__ dbg) {
  constexpr int V = H / 128;
  __shared__ float4 part[8][32 * V];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nl = desc->n_long;
  for (int li = blockIdx.x; li < nl; li += gridDim.x) {
    const int sg = long_list[li];
    const int s = seg_ptr[sg], e = seg_ptr[sg + 1];
    float4 acc[V];
#pragma unroll
    for (int q = 0; q < V; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = s + w; j < e; j += 8) {
      const int r = seg_row[j];
      const float v = seg_val[j];
#pragma unroll
      for (int q = 0; q < V; ++q) {
        const float4 g = reinterpret_cast<const float4 *>(dA + (size_t)r * H)[lane + 32 * q];
        acc[q].x = fmaf(v, g.x, acc[q].x);
        acc[q].y = fmaf(v, g.y, acc[q].y);
        acc[q].z = fmaf(v, g.z, acc[q].z);
        acc[q].w = fmaf(v, g.w, acc[q].w);
      }
    }
#pragma unroll
    for (int q = 0; q < V; ++q) part[w][lane + 32 * q] = acc[q];
    __syncthreads();
    if (threadIdx.x < 32 * V) {
      const int i = threadIdx.x;
      float4 a = part[0][i];
#pragma unroll
      for (int q = 1; q < 8; ++q) {
        const float4 p = part[q][i];
        a.x += p.x; a.y += p.y; a.z += p.z; a.w += p.w;
      }
      const size_t f = (size_t)seg_id[sg];
      float4 *wp = reinterpret_cast<float4 *>(W1 + f * H) + i;
      float4 ww = *wp;
      ww.x -= lr * a.x; ww.y -= lr * a.y; ww.z -= lr * a.z; ww.w -= lr * a.w;
      *wp = ww;
      if (dbg) reinterpret_cast<float4 *>(dbg + (size_t)sg * H)[i] = a;
    }
    __syncthreads();
  }
}

void launch_dw1_sgd(cudaStream_t s, int h, StepDesc *desc, int cap, const int32_t *seg_id,
                    const int32_t *seg_ptr, const int32_t *seg_row, const float *seg_val,
                    const float *dA, float *W1, float lr, int32_t *long_list, float *dbg_dW1) {
  const int grid_short = 148 * 8, grid_long = 148 * 2;
  (void)cap;
  if (h == 128) {
    k_dw1_short<128><<<grid_short, 256, 0, s>>>(desc, seg_id, seg_ptr, seg_row, seg_val, dA, W1,
                                                lr, long_list, dbg_dW1);
    k_dw1_long<128><<<grid_long, 256, 0, s>>>(desc, seg_id, seg_ptr, seg_row, seg_val, dA, W1, lr,
                                              long_list, dbg_dW1);
  } else {
    k_dw1_short<256><<<grid_short, 256, 0, s>>>(desc, seg_id, seg_ptr, seg_row, seg_val, dA, W1,
                                                lr, long_list, dbg_dW1);
    k_dw1_long<256><<<grid_long, 256, 0, s>>>(desc, seg_id, seg_ptr, seg_row, seg_val, dA, W1, lr,
                                              long_list, dbg_dW1);
  }
}

// mean of the per-row losses (fixed-order tree), R3
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

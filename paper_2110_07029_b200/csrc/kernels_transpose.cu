// Step a3: the two batch transposes of every SGD step, built in
// three launches for BOTH key spaces (features for dW1, labels for dW2 / db2):
//
//   k_tr_mark   per entry (r, key): cnt[key] += 1 and bit r of the key's row
//               bitmap (integer atomics: the result does not depend on order)
//   k_tr_scan   one single-pass chained scan (decoupled look-back) over the
//               dense key spaces [0, d) and [0, C): for every present key its
//               segment index (keys ascending) and its first entry offset;
//               writes seg_id / seg_ptr / the segment counts U and V
//   k_tr_place  per entry: position = offset[key] + popcount of the key's
//               bitmap below r, i.e. THE stable sort by key with rows
//               ascending inside a key (features are unique within a row, so a
//               key's rows are distinct); writes the sorted row / value /
//               segment-of-entry / label weight 1/(k_r B) arrays
//
// The dense per-key state (counts, bitmaps, class->segment map, scan tiles) is
// returned to its idle value by k_tr_reset on the side stream after the
// step's last reader, touching only the keys of the batch.  Integer-only and bit-exact (pinned against a
// brute-force rebuild in tests/test_gpu_parity.py::test_transposes_bit_exact).
#include "common.cuh"

namespace as {

constexpr int kTrTile = 8192;   // keys per scan tile (1024 threads x 8)

// entry -> row of both CSR arrays of a host-loaded batch (warp per row)
__global__ void k_entry_rows(const int64_t *__restrict__ row_ptr, const int64_t *__restrict__ lab_ptr,
                             int rows, int32_t *__restrict__ rid, int32_t *__restrict__ lrid) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (r >= rows) return;
  for (int64_t j = row_ptr[r] + lane; j < row_ptr[r + 1]; j += 32) rid[j] = r;
  for (int64_t j = lab_ptr[r] + lane; j < lab_ptr[r + 1]; j += 32) lrid[j] = r;
}

void launch_entry_rows(cudaStream_t s, const int64_t *row_ptr, const int64_t *lab_ptr, int rows,
                       int32_t *rid, int32_t *lrid) {
  k_entry_rows<<<ceil_div((long long)rows * 32, 256), 256, 0, s>>>(row_ptr, lab_ptr, rows, rid, lrid);
}

__global__ void __launch_bounds__(256) k_tr_mark(TrArgs a) {
  const StepDesc *d = a.desc;
  const int nnz = min(d->nnz, a.nnz_cap), nlab = min(d->nlab, a.lab_cap);
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nnz) {
    const int f = a.col[t], r = a.rid[t];
    atomicAdd(&a.fcnt[f], 1);
    atomicOr(&a.fbits[(size_t)f * a.W + (r >> 5)], 1u << (r & 31));
  } else if (t - nnz < nlab) {
    const int j = t - nnz;
    const int c = a.lab[j], r = a.lrid[j];
    atomicAdd(&a.lcnt[c], 1);
    atomicOr(&a.lbits[(size_t)c * a.W + (r >> 5)], 1u << (r & 31));
  }
}

// scan tile state: [status 2 bits | segments 31 bits | entries 31 bits]
__device__ __forceinline__ unsigned long long tr_pack(unsigned long long st, unsigned long long segs,
                                                      unsigned long long ents) {
  return (st << 62) | (segs << 31) | ents;
}
__device__ __forceinline__ void st_release(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(1024) k_tr_scan(TrArgs a) {
  constexpr int KPT = kTrTile / 1024;            // keys per thread
  __shared__ int s_tile;
  __shared__ int s_we[32], s_ws[32];
  __shared__ int s_pe, s_ps;
  const int nt_f = ceil_div_dev(a.d, kTrTile), nt_l = ceil_div_dev(a.C, kTrTile);
  if (threadIdx.x == 0) s_tile = atomicAdd(a.ticket, 1);   // in-order tiles: look-back progress
  __syncthreads();
  const int tile = s_tile;
  if (tile >= nt_f + nt_l) return;
  const bool lab = tile >= nt_f;
  const int t0 = lab ? nt_f : 0, lt = tile - t0, nt = lab ? nt_l : nt_f;
  const int n = lab ? a.C : a.d;
  int32_t *cnt = lab ? a.lcnt : a.fcnt;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int base = lt * kTrTile + KPT * tid;
  int c[KPT];
  if (base + KPT - 1 < n) {
#pragma unroll
    for (int i = 0; i < KPT; i += 4) {
      const int4 v = *reinterpret_cast<const int4 *>(cnt + base + i);
      c[i] = v.x; c[i + 1] = v.y; c[i + 2] = v.z; c[i + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < KPT; ++i) c[i] = base + i < n ? cnt[base + i] : 0;
  }
  int te = 0, ts = 0;
#pragma unroll
  for (int i = 0; i < KPT; ++i) { te += c[i]; ts += c[i] > 0; }
  int ie = te, is = ts;                           // warp inclusive scans
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int ye = __shfl_up_sync(0xffffffffu, ie, o), ys = __shfl_up_sync(0xffffffffu, is, o);
    if (lane >= o) { ie += ye; is += ys; }
  }
  if (lane == 31) { s_we[w] = ie; s_ws[w] = is; }
  __syncthreads();
  if (w == 0) {
    int xe = s_we[lane], xs = s_ws[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int ye = __shfl_up_sync(0xffffffffu, xe, o), ys = __shfl_up_sync(0xffffffffu, xs, o);
      if (lane >= o) { xe += ye; xs += ys; }
    }
    s_we[lane] = xe; s_ws[lane] = xs;              // inclusive over warps
    const int AE = __shfl_sync(0xffffffffu, xe, 31), AS = __shfl_sync(0xffffffffu, xs, 31);
    unsigned long long *st = a.tile_state + tile;
    if (lane == 0)
      st_release(st, tr_pack(lt == 0 ? 2ull : 1ull, (unsigned long long)AS, (unsigned long long)AE));
    int pe = 0, ps = 0;
    if (lt > 0) {
      // decoupled look-back, 32 predecessors per round (lane 0 = nearest)
      for (int top = tile - 1;; top -= 32) {
        const int kk = top - lane;
        unsigned long long v = 2ull << 62;        // before the key space: inclusive 0
        if (kk >= t0) {
          do { v = ld_acquire(a.tile_state + kk); } while ((v >> 62) == 0ull);
        }
        const unsigned inc = __ballot_sync(0xffffffffu, (v >> 62) == 2ull);
        const int first = inc ? __ffs(inc) - 1 : 32;
        const bool take = lane <= first && kk >= t0;
        pe += warp_sum_i(take ? (int)(v & 0x7FFFFFFFull) : 0);
        ps += warp_sum_i(take ? (int)((v >> 31) & 0x7FFFFFFFull) : 0);
        if (inc) break;
      }
      if (lane == 0)
        st_release(st, tr_pack(2ull, (unsigned long long)(ps + AS), (unsigned long long)(pe + AE)));
    }
    if (lane == 0) {
      s_pe = pe; s_ps = ps;
      if (lt == nt - 1) {                          // totals of this key space
        const int E = pe + AE, S = ps + AS;
        // segment counts also into ticket[2..3]: the side-stream reset reads them
        // there while the main stream's next batch rewrites the step descriptor
        if (lab) { a.lseg_ptr[S] = E; a.desc->V = S; a.ticket[3] = S; }
        else { a.fseg_ptr[S] = E; a.desc->U = S; a.ticket[2] = S; }
      }
    }
  }
  __syncthreads();
  int oe = s_pe + (w > 0 ? s_we[w - 1] : 0) + ie - te;
  int os = s_ps + (w > 0 ? s_ws[w - 1] : 0) + is - ts;
  int32_t *seg_id = lab ? a.lseg_id : a.fseg_id;
  int32_t *seg_ptr = lab ? a.lseg_ptr : a.fseg_ptr;
  int32_t *sidx = lab ? a.cls_seg : a.fsidx;
#pragma unroll
  for (int i = 0; i < KPT; ++i) {
    if (c[i] > 0) {
      const int key = base + i;
      seg_id[os] = key;
      seg_ptr[os] = oe;
      sidx[key] = os;
      cnt[key] = oe;                               // count -> first entry offset
      ++os;
      oe += c[i];
    }
  }
}

__device__ __forceinline__ int rank_below(const uint32_t *__restrict__ bits, int r) {
  const int wr = r >> 5;
  int k = 0;
  int wi = 0;
  for (; wi + 4 <= wr; wi += 4) {
    const uint4 v = *reinterpret_cast<const uint4 *>(bits + wi);
    k += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
  }
  for (; wi < wr; ++wi) k += __popc(bits[wi]);
  return k + __popc(bits[wr] & ((1u << (r & 31)) - 1u));
}

__global__ void __launch_bounds__(256) k_tr_place(TrArgs a) {
  const StepDesc *d = a.desc;
  const int nnz = min(d->nnz, a.nnz_cap), nlab = min(d->nlab, a.lab_cap);
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nnz) {
    const int f = a.col[t], r = a.rid[t];
    const int pos = a.fcnt[f] + rank_below(a.fbits + (size_t)f * a.W, r);
    a.fseg_row[pos] = r;
    a.fseg_val[pos] = a.val[t];
    a.fseg_of[pos] = a.fsidx[f];
  } else if (t - nnz < nlab) {
    const int j = t - nnz;
    const int c = a.lab[j], r = a.lrid[j];
    const int first = a.lcnt[c];
    const int pos = first + rank_below(a.lbits + (size_t)c * a.W, r);
    a.lseg_row[pos] = r;
    // 1 / (k_r B): the label weight of the uniform multi-label target (R3)
    const float wgt = (1.0f / (float)d->rows) / (float)(a.lab_ptr[r + 1] - a.lab_ptr[r]);
    a.lw[pos] = wgt;
    if (pos == first)                       // the class's label range for pass 2 in one load
      a.cls_lab[c] = make_int4(first, a.lseg_ptr[a.cls_seg[c] + 1], r, __float_as_int(wgt));
  }
}

void launch_transposes(cudaStream_t s, const TrArgs &a) {
  const int ent = ceil_div((long long)a.nnz_cap + a.lab_cap, 256);
  const int tiles = ceil_div(a.d, kTrTile) + ceil_div(a.C, kTrTile);
  k_tr_mark<<<ent, 256, 0, s>>>(a);
  k_tr_scan<<<tiles, 1024, 0, s>>>(a);
  k_tr_place<<<ent, 256, 0, s>>>(a);
}

// The dense per-key transpose state back to idle on the SIDE stream after the
// step's last reader (dW1), keyed by the step's own segment lists (fseg_id /
// lseg_id, whole bitmaps) so it does not read the batch arrays the main
// stream's next batch is already overwriting; the next step's transposes
// follow it in stream order.
__global__ void __launch_bounds__(256) k_tr_reset(TrArgs a) {
  const int U = a.ticket[2], V = a.ticket[3], W = a.W;
  const int tiles = ceil_div_dev(a.d, kTrTile) + ceil_div_dev(a.C, kTrTile);
  const long long nf = (long long)U * W, nl = (long long)V * W;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < nf + nl || t < tiles; t += stride) {
    if (t < tiles) a.tile_state[t] = 0ull;
    if (t < nf) {
      const int f = a.fseg_id[t / W];
      a.fbits[(size_t)f * W + t % W] = 0u;
      if (t % W == 0) a.fcnt[f] = 0;
    } else if (t - nf < nl) {
      const long long j = t - nf;
      const int c = a.lseg_id[j / W];
      a.lbits[(size_t)c * W + j % W] = 0u;
      if (j % W == 0) {
        a.lcnt[c] = 0;
        a.cls_seg[c] = -1;
        a.cls_lab[c] = make_int4(0, 0, 0x7fffffff, 0);
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) a.ticket[0] = 0;
}

void launch_tr_reset(cudaStream_t s, const TrArgs &a, int num_sms) {
  k_tr_reset<<<2 * num_sms, 256, 0, s>>>(a);
}


}  // namespace as

namespace as {
__global__ void k_fill_int4(int4 *p, long long n, int4 v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}
void launch_fill_int4(cudaStream_t s, int4 *p, long long n, int x, int y, int z, int w) {
  k_fill_int4<<<1024, 256, 0, s>>>(p, n, make_int4(x, y, z, w));
}
}  // namespace as

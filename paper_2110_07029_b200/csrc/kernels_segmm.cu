// Load-balanced, deterministic segmented gather-reduce used by the SpMM
// forward (step a4: A1_r = b1 + sum_j x_rj W1[col_j], H = ReLU(A1)) and by the
// first-layer gradient with fused SGD (step a7: dW1[f] = sum_j v_j dA[row_j],
// W1[f] -= lr dW1[f]).
//
// The entries (CSR order for a4, feature-sorted order for a7) are cut into
// flat chunks of 16; one warp per chunk gathers its 16 source rows (h fp32 =
// 128-bit per lane) with all loads in flight, then sums them segment by
// segment in entry order.  A segment that lies inside its chunk is finalised
// directly; a segment spanning chunks leaves a head / tail partial that the
// fix-up kernel adds in chunk order.  Every sum has a fixed order
// (deterministic, no float atomics) and every warp has the same work
// regardless of the lognormal row lengths / Zipf feature frequencies.
#include "common.cuh"

namespace as {


struct SegArgs {
  // MODE 0 (forward)
  const float *b1;
  float *Hf;
  __nv_bfloat16 *Hb;
  // MODE 1 (dW1 + SGD)
  const int32_t *seg_key;
  float *W1;
  float lr;
  float *dbg;
};

template <int H, int MODE>
__device__ __forceinline__ void seg_finalize(int sg, const float4 (&acc)[H / 128], int lane,
                                             const SegArgs &a) {
  constexpr int V = H / 128;
  if (MODE == 0) {
    const float4 *B1 = reinterpret_cast<const float4 *>(a.b1);
#pragma unroll
    for (int q = 0; q < V; ++q) {
      const int i = lane + 32 * q;
      const float4 bb = B1[i];
      float4 o;
      o.x = fmaxf(acc[q].x + bb.x, 0.f); o.y = fmaxf(acc[q].y + bb.y, 0.f);
      o.z = fmaxf(acc[q].z + bb.z, 0.f); o.w = fmaxf(acc[q].w + bb.w, 0.f);
      reinterpret_cast<float4 *>(a.Hf + (size_t)sg * H)[i] = o;
      reinterpret_cast<uint2 *>(a.Hb + (size_t)sg * H)[i] =
          make_uint2(pack_bf16x2(o.x, o.y), pack_bf16x2(o.z, o.w));
    }
  } else {
    const size_t f = (size_t)a.seg_key[sg];
#pragma unroll
    for (int q = 0; q < V; ++q) {
      const int i = lane + 32 * q;
      float4 *wp = reinterpret_cast<float4 *>(a.W1 + f * H) + i;
      float4 w = *wp;
      w.x -= a.lr * acc[q].x; w.y -= a.lr * acc[q].y; w.z -= a.lr * acc[q].z; w.w -= a.lr * acc[q].w;
      *wp = w;
      if (a.dbg) reinterpret_cast<float4 *>(a.dbg + (size_t)sg * H)[i] = acc[q];
    }
  }
}

template <int H, int MODE, typename PtrT, int kChunk>
__global__ void __launch_bounds__(256) k_seg_chunk(const int *__restrict__ n_dev,
                                                   const int32_t *__restrict__ seg_of,
                                                   const PtrT *__restrict__ seg_ptr,
                                                   const int32_t *__restrict__ gidx,
                                                   const float *__restrict__ scale,
                                                   const float *__restrict__ src,
                                                   float *__restrict__ part, SegArgs a) {
  constexpr int V = H / 128;
  const int n = *n_dev;
  const int lane = threadIdx.x & 31;
  const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int j0 = k * kChunk;
  if (j0 >= n) return;
  const int cnt = min(kChunk, n - j0), j1 = j0 + cnt;
  int e_seg = -1, e_idx = 0;
  float e_val = 0.f;
  if (lane < cnt) {
    e_seg = seg_of[j0 + lane];
    e_idx = gidx[j0 + lane];
    e_val = scale[j0 + lane];
  }
  const float4 *S = reinterpret_cast<const float4 *>(src);
  constexpr int RND = 16 / V;                // gathers in flight per round
  float4 x[RND][V];
  float4 acc[V];
#pragma unroll
  for (int q = 0; q < V; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  int cur = __shfl_sync(0xffffffffu, e_seg, 0);
  auto flush = [&](int sg) {
    const long long s0 = (long long)seg_ptr[sg], s1 = (long long)seg_ptr[sg + 1];
    const bool head = s0 < j0, tail = s1 > j1;
    if (!head && !tail) {
      seg_finalize<H, MODE>(sg, acc, lane, a);
    } else {
      float4 *p = reinterpret_cast<float4 *>(part + ((size_t)k * 2 + (head ? 0 : 1)) * H);
#pragma unroll
      for (int q = 0; q < V; ++q) p[lane + 32 * q] = acc[q];
    }
  };
#pragma unroll 1
  for (int u0 = 0; u0 < cnt; u0 += RND) {
#pragma unroll
    for (int u = 0; u < RND; ++u) {
      const int idx = __shfl_sync(0xffffffffu, e_idx, (u0 + u) & 31);
#pragma unroll
      for (int q = 0; q < V; ++q)
        x[u][q] = u0 + u < cnt ? __ldg(&S[(size_t)idx * (H / 4) + lane + 32 * q])
                               : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < RND; ++u) {
      if (u0 + u < cnt) {
        const int sg = __shfl_sync(0xffffffffu, e_seg, (u0 + u) & 31);
        const float v = __shfl_sync(0xffffffffu, e_val, (u0 + u) & 31);
        if (sg != cur) {
          flush(cur);
#pragma unroll
          for (int q = 0; q < V; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
          cur = sg;
        }
#pragma unroll
        for (int q = 0; q < V; ++q) {
          acc[q].x = fmaf(v, x[u][q].x, acc[q].x);
          acc[q].y = fmaf(v, x[u][q].y, acc[q].y);
          acc[q].z = fmaf(v, x[u][q].z, acc[q].z);
          acc[q].w = fmaf(v, x[u][q].w, acc[q].w);
        }
      }
    }
  }
  flush(cur);
}

// segments spanning chunks: tail of the first chunk + middles + head of the last
template <int H, int MODE, typename PtrT, int kChunk>
__global__ void __launch_bounds__(256) k_seg_fixup(const int *__restrict__ nseg_dev, int nseg_pad,
                                                   const PtrT *__restrict__ seg_ptr,
                                                   const float *__restrict__ part, SegArgs a) {
  constexpr int V = H / 128;
  const int nseg = *nseg_dev;
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int bound = MODE == 0 ? nseg_pad : nseg;
  for (int sg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; sg < bound; sg += nw) {
    if (sg >= nseg) {                       // MODE 0: padding rows of the last MMA tile
      if (MODE == 0) {
        uint2 *hb = reinterpret_cast<uint2 *>(a.Hb + (size_t)sg * H);
        for (int i = lane; i < H / 4; i += 32) hb[i] = make_uint2(0u, 0u);
      }
      continue;
    }
    const long long s0 = (long long)seg_ptr[sg], s1 = (long long)seg_ptr[sg + 1];
    float4 acc[V];
#pragma unroll
    for (int q = 0; q < V; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (s1 == s0) {                         // empty row (MODE 0): H = ReLU(b1)
      seg_finalize<H, MODE>(sg, acc, lane, a);
      continue;
    }
    const long long c0 = s0 / kChunk, c1 = (s1 - 1) / kChunk;
    if (c0 == c1) continue;                 // finalised by its chunk warp
#pragma unroll 4
    for (long long c = c0; c <= c1; ++c) {
      const float4 *p = reinterpret_cast<const float4 *>(part + ((size_t)c * 2 + (c == c0 ? 1 : 0)) * H);
#pragma unroll
      for (int q = 0; q < V; ++q) {
        const float4 t = p[lane + 32 * q];
        acc[q].x += t.x; acc[q].y += t.y; acc[q].z += t.z; acc[q].w += t.w;
      }
    }
    seg_finalize<H, MODE>(sg, acc, lane, a);
  }
}

// entry -> row of a rebased CSR (warp per row)
__global__ void k_entry_row(const int64_t *__restrict__ ptr, int rows, int32_t *__restrict__ rid) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (r >= rows) return;
  for (int64_t j = ptr[r] + lane; j < ptr[r + 1]; j += 32) rid[j] = r;
}

template <int H>
static void spmm_h(cudaStream_t s, const StepDesc *desc, int rows, int bpad, int nnz_cap,
                   const int64_t *row_ptr, const int32_t *col, const float *val, int32_t *rid,
                   const float *W1, float *part, const SegArgs &a) {
  k_entry_row<<<ceil_div((long long)rows * 32, 256), 256, 0, s>>>(row_ptr, rows, rid);
  constexpr int CH = 32;                     // rows average ~76 nnz
  const int nch = ceil_div(nnz_cap > 0 ? nnz_cap : 1, CH);
  k_seg_chunk<H, 0, int64_t, CH><<<ceil_div((long long)nch * 32, 256), 256, 0, s>>>(
      &desc->nnz, rid, row_ptr, col, val, W1, part, a);
  k_seg_fixup<H, 0, int64_t, CH><<<ceil_div((long long)bpad * 32, 256), 256, 0, s>>>(
      &desc->rows, bpad, row_ptr, part, a);
}

void launch_spmm_chunked(cudaStream_t s, int h, const StepDesc *desc, int rows, int bpad, int nnz_cap,
                         const int64_t *row_ptr, const int32_t *col, const float *val, int32_t *rid,
                         const float *W1, const float *b1, float *Hf, __nv_bfloat16 *Hb,
                         float *part) {
  SegArgs a{};
  a.b1 = b1; a.Hf = Hf; a.Hb = Hb;
  if (h == 128)
    spmm_h<128>(s, desc, rows, bpad, nnz_cap, row_ptr, col, val, rid, W1, part, a);
  else
    spmm_h<256>(s, desc, rows, bpad, nnz_cap, row_ptr, col, val, rid, W1, part, a);
}

template <int H>
static void dw1_h(cudaStream_t s, StepDesc *desc, int nnz_cap, const int32_t *seg_of,
                  const int32_t *seg_ptr, const int32_t *seg_row, const float *seg_val,
                  const float *dA, float *part, const SegArgs &a) {
  constexpr int CH = 16;                     // feature segments are mostly short
  const int nch = ceil_div(nnz_cap > 0 ? nnz_cap : 1, CH);
  k_seg_chunk<H, 1, int32_t, CH><<<ceil_div((long long)nch * 32, 256), 256, 0, s>>>(
      &desc->nnz, seg_of, seg_ptr, seg_row, seg_val, dA, part, a);
  k_seg_fixup<H, 1, int32_t, CH><<<148 * 8, 256, 0, s>>>(&desc->U, 0, seg_ptr, part, a);
}

void launch_dw1_chunked(cudaStream_t s, int h, StepDesc *desc, int nnz_cap, const int32_t *seg_id,
                        const int32_t *seg_of, const int32_t *seg_ptr, const int32_t *seg_row,
                        const float *seg_val, const float *dA, float *W1, float lr, float *part,
                        float *dbg_dW1) {
  SegArgs a{};
  a.seg_key = seg_id; a.W1 = W1; a.lr = lr; a.dbg = dbg_dW1;
  if (h == 128)
    dw1_h<128>(s, desc, nnz_cap, seg_of, seg_ptr, seg_row, seg_val, dA, part, a);
  else
    dw1_h<256>(s, desc, nnz_cap, seg_of, seg_ptr, seg_row, seg_val, dA, part, a);
}

}  // namespace as

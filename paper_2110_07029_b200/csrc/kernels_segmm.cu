// Load-balanced, deterministic segmented gather-reduce used by the SpMM
// forward (step a4: A1_r = b1 + sum_j x_rj W1[col_j], H = ReLU(A1)) and by the
// first-layer gradient with fused SGD (step a7: dW1[f] = sum_j v_j dA[row_j],
// W1[f] -= lr dW1[f]).  ONE launch each.
//
// The entries (CSR order for a4, feature-sorted order for a7) are cut into
// flat chunks of 16 (h = 128; 8 for h = 256).  Persistent warps take chunks
// grid-stride; a warp gathers its chunk's source rows with every load in
// flight at once (h fp32 = 128-bit per lane: one 512-byte row per warp-wide
// load), then sums them segment by segment in entry order.  A segment inside
// its chunk is finalised directly.  A segment spanning chunks c0..c1 leaves one
// partial per chunk; the LAST warp to arrive (integer counter per segment)
// adds the partials in chunk order c0..c1 and finalises.  Every sum therefore
// has a fixed order whichever warp finishes it (deterministic, no float
// atomics), and every warp has the same work regardless of the lognormal row
// lengths / Zipf feature frequencies.
//
// Latency: the per-entry metadata (segment bounds) is loaded lane-parallel
// with the entry, b1 is held in registers (a4), and the W1 read-modify-writes
// of a7 are batched per chunk (segment sums stashed in shared memory, then all
// W1 rows of the chunk loaded at once) instead of one dependent load per
// segment.
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

constexpr int kSegWarps = 4;   // warps per CTA

template <int H>
__device__ __forceinline__ void fwd_store(int sg, const float4 (&acc)[H / 128], const float4 (&bb)[H / 128],
                                          int lane, const SegArgs &a) {
  constexpr int V = H / 128;
#pragma unroll
  for (int q = 0; q < V; ++q) {
    const int i = lane + 32 * q;
    float4 o;
    o.x = fmaxf(acc[q].x + bb[q].x, 0.f); o.y = fmaxf(acc[q].y + bb[q].y, 0.f);
    o.z = fmaxf(acc[q].z + bb[q].z, 0.f); o.w = fmaxf(acc[q].w + bb[q].w, 0.f);
    reinterpret_cast<float4 *>(a.Hf + (size_t)sg * H)[i] = o;
    reinterpret_cast<uint2 *>(a.Hb + (size_t)sg * H)[i] =
        make_uint2(pack_bf16x2(o.x, o.y), pack_bf16x2(o.z, o.w));
  }
}

template <int H, int MODE, typename PtrT>
__global__ void __launch_bounds__(kSegWarps * 32, MODE == 0 ? 4 : 3) k_seg_gr(const int *__restrict__ n_dev,
                                                           const int *__restrict__ nseg_dev, int nseg_pad,
                                                           const int32_t *__restrict__ seg_of,
                                                           const PtrT *__restrict__ seg_ptr,
                                                           const int32_t *__restrict__ gidx,
                                                           const float *__restrict__ scale,
                                                           const float *__restrict__ src,
                                                           float *__restrict__ part,
                                                           int *__restrict__ arrive, SegArgs a) {
  constexpr int V = H / 128;
  constexpr int CH = 16 / V;                  // entries per chunk = gathers in flight per warp
  __shared__ __align__(16) float4 stash_all[MODE == 1 ? kSegWarps * CH * 32 * V : 1];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gw = blockIdx.x * kSegWarps + wib, nw = gridDim.x * kSegWarps;
  const int n = *n_dev;
  const float4 *S = reinterpret_cast<const float4 *>(src);
  float4 bb[V];
  if (MODE == 0) {
#pragma unroll
    for (int q = 0; q < V; ++q) bb[q] = reinterpret_cast<const float4 *>(a.b1)[lane + 32 * q];
  }
  float4 *stash = stash_all + (MODE == 1 ? wib * CH * 32 * V : 0);
  // per-lane metadata of one chunk (entry lane): segment, source row, scale,
  // segment bounds; the next chunk's is loaded while this chunk's gathers fly
  int m_seg = 0, m_idx = 0, m_s0 = 0, m_s1 = 0;
  float m_val = 0.f;
  auto load_meta = [&](int kk) {
    const int jj = kk * CH + lane;
    if (jj < n && lane < CH) {
      m_seg = seg_of[jj];
      m_idx = gidx[jj];
      m_val = scale[jj];
      m_s0 = (int)seg_ptr[m_seg];
      m_s1 = (int)seg_ptr[m_seg + 1];
    }
  };
  load_meta(gw);
#pragma unroll 1
  for (int k = gw; k * CH < n; k += nw) {
    const int j0 = k * CH;
    const int cnt = min(CH, n - j0), j1 = j0 + cnt;
    const int e_seg = m_seg, e_idx = m_idx, e_s0 = m_s0, e_s1 = m_s1;
    const float e_val = m_val;
    float4 x[CH][V];
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int idx = __shfl_sync(0xffffffffu, e_idx, u);
#pragma unroll
      for (int q = 0; q < V; ++q)
        x[u][q] = u < cnt ? __ldg(&S[(size_t)idx * (H / 4) + lane + 32 * q]) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    load_meta(k + nw);
    int ns = 0, st_sg = 0;                    // stashed segments of this chunk (MODE 1)
    float4 acc[V];
#pragma unroll
    for (int q = 0; q < V; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      if (u < cnt) {
        const float v = __shfl_sync(0xffffffffu, e_val, u);
#pragma unroll
        for (int q = 0; q < V; ++q) {
          acc[q].x = fmaf(v, x[u][q].x, acc[q].x);
          acc[q].y = fmaf(v, x[u][q].y, acc[q].y);
          acc[q].z = fmaf(v, x[u][q].z, acc[q].z);
          acc[q].w = fmaf(v, x[u][q].w, acc[q].w);
        }
        const int sg = __shfl_sync(0xffffffffu, e_seg, u);
        const int s1 = __shfl_sync(0xffffffffu, e_s1, u);
        if (s1 == j0 + u + 1 || u == cnt - 1) {   // segment sg ends here or the chunk does
          const int s0 = __shfl_sync(0xffffffffu, e_s0, u);
          const bool spans = s0 < j0 || s1 > j1;
          bool fin = !spans;
          if (spans) {
            float4 *p = reinterpret_cast<float4 *>(part + ((size_t)k * 2 + (s0 < j0 ? 0 : 1)) * H);
#pragma unroll
            for (int q = 0; q < V; ++q) p[lane + 32 * q] = acc[q];
            const int c0 = s0 / CH, c1 = (s1 - 1) / CH;
            __threadfence();
            __syncwarp();
            int old = 0;
            if (lane == 0) old = atomicAdd(&arrive[sg], 1);
            old = __shfl_sync(0xffffffffu, old, 0);
            if (old == c1 - c0) {                  // last chunk to arrive: ordered sum
              __threadfence();
#pragma unroll
              for (int q = 0; q < V; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
              for (int c = c0; c <= c1; ++c) {     // chunk c0 (slot 1), then slot 0
                const float4 *pp =
                    reinterpret_cast<const float4 *>(part + ((size_t)c * 2 + (c == c0 ? 1 : 0)) * H);
#pragma unroll
                for (int q = 0; q < V; ++q) {
                  const float4 t = __ldcg(pp + lane + 32 * q);
                  acc[q].x += t.x; acc[q].y += t.y; acc[q].z += t.z; acc[q].w += t.w;
                }
              }
              if (lane == 0) arrive[sg] = 0;      // idle for the next step
              fin = true;
            }
          }
          if (fin) {
            if (MODE == 0) {
              fwd_store<H>(sg, acc, bb, lane, a);
            } else {
#pragma unroll
              for (int q = 0; q < V; ++q) stash[(ns * V + q) * 32 + lane] = acc[q];
              if (lane == ns) st_sg = sg;
              ++ns;
            }
          }
#pragma unroll
          for (int q = 0; q < V; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    }
    if (MODE == 1 && ns > 0) {
      // batched fused SGD of this chunk's finished segments: W1[f] -= lr dW1[f]
      __syncwarp();
      const int key = lane < ns ? a.seg_key[st_sg] : 0;
#pragma unroll 1
      for (int i0 = 0; i0 < ns; i0 += CH / 2) {
        float4 w[CH / 2][V];
#pragma unroll
        for (int i = 0; i < CH / 2; ++i) {
          const int f = __shfl_sync(0xffffffffu, key, (i0 + i) & 31);
#pragma unroll
          for (int q = 0; q < V; ++q)
            if (i0 + i < ns) w[i][q] = reinterpret_cast<const float4 *>(a.W1 + (size_t)f * H)[lane + 32 * q];
        }
#pragma unroll
        for (int i = 0; i < CH / 2; ++i) {
          const int f = __shfl_sync(0xffffffffu, key, (i0 + i) & 31);
          const int sg = __shfl_sync(0xffffffffu, st_sg, (i0 + i) & 31);
          if (i0 + i < ns) {
#pragma unroll
            for (int q = 0; q < V; ++q) {
              const float4 g = stash[((i0 + i) * V + q) * 32 + lane];
              float4 nw = w[i][q];
              nw.x -= a.lr * g.x; nw.y -= a.lr * g.y; nw.z -= a.lr * g.z; nw.w -= a.lr * g.w;
              reinterpret_cast<float4 *>(a.W1 + (size_t)f * H)[lane + 32 * q] = nw;
              if (a.dbg) reinterpret_cast<float4 *>(a.dbg + (size_t)sg * H)[lane + 32 * q] = g;
            }
          }
        }
      }
      __syncwarp();
    }
  }
  if (MODE == 0) {
    // rows no chunk covers: empty rows (H = ReLU(b1)) and the zero padding rows
    // of the last 128-row MMA tile
    const int nseg = *nseg_dev;
    for (int sg = gw; sg < nseg_pad; sg += nw) {
      if (sg >= nseg) {
        uint2 *hb = reinterpret_cast<uint2 *>(a.Hb + (size_t)sg * H);
        for (int i = lane; i < H / 4; i += 32) hb[i] = make_uint2(0u, 0u);
      } else if (seg_ptr[sg + 1] == seg_ptr[sg]) {
        float4 z[V];
#pragma unroll
        for (int q = 0; q < V; ++q) z[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        fwd_store<H>(sg, z, bb, lane, a);
      }
    }
  }
}

template <int H, int MODE, typename PtrT>
static void seg_launch(cudaStream_t s, int num_sms, const int *n_dev, const int *nseg_dev, int nseg_pad,
                       int cap, const int32_t *seg_of, const PtrT *seg_ptr, const int32_t *gidx,
                       const float *scale, const float *src, float *part, int *arrive, const SegArgs &a) {
  constexpr int CH = 16 * 128 / H;
  const int need = ceil_div(ceil_div(cap > 0 ? cap : 1, CH), kSegWarps);
  const int per_sm = MODE == 0 ? 4 : 3;
  const int grid = need < num_sms * per_sm ? need : num_sms * per_sm;
  k_seg_gr<H, MODE, PtrT><<<grid > 0 ? grid : 1, kSegWarps * 32, 0, s>>>(
      n_dev, nseg_dev, nseg_pad, seg_of, seg_ptr, gidx, scale, src, part, arrive, a);
}

void launch_spmm_chunked(cudaStream_t s, int h, int num_sms, const StepDesc *desc, int bpad, int nnz_cap,
                         const int64_t *row_ptr, const int32_t *col, const float *val,
                         const int32_t *rid, const float *W1, const float *b1, float *Hf,
                         __nv_bfloat16 *Hb, float *part, int *arrive) {
  SegArgs a{};
  a.b1 = b1; a.Hf = Hf; a.Hb = Hb;
  const int cap = nnz_cap > bpad ? nnz_cap : bpad;
  if (h == 128)
    seg_launch<128, 0, int64_t>(s, num_sms, &desc->nnz, &desc->rows, bpad, cap, rid, row_ptr, col, val, W1,
                                part, arrive, a);
  else
    seg_launch<256, 0, int64_t>(s, num_sms, &desc->nnz, &desc->rows, bpad, cap, rid, row_ptr, col, val, W1,
                                part, arrive, a);
}

void launch_dw1_chunked(cudaStream_t s, int h, int num_sms, StepDesc *desc, int nnz_cap,
                        const int32_t *seg_id, const int32_t *seg_of, const int32_t *seg_ptr,
                        const int32_t *seg_row, const float *seg_val, const float *dA, float *W1,
                        float lr, float *part, int *arrive, float *dbg_dW1) {
  SegArgs a{};
  a.seg_key = seg_id; a.W1 = W1; a.lr = lr; a.dbg = dbg_dW1;
  if (h == 128)
    seg_launch<128, 1, int32_t>(s, num_sms, &desc->nnz, &desc->U, 0, nnz_cap, seg_of, seg_ptr, seg_row,
                                seg_val, dA, part, arrive, a);
  else
    seg_launch<256, 1, int32_t>(s, num_sms, &desc->nnz, &desc->U, 0, nnz_cap, seg_of, seg_ptr, seg_row,
                                seg_val, dA, part, arrive, a);
}

}  // namespace as

// Load-balanced, deterministic segmented gather-reduce used by the SpMM
// forward (step a4: A1_r = b1 + sum_j x_rj W1[col_j], H = ReLU(A1)) and by the
// first-layer gradient with fused SGD (step a7: dW1[f] = sum_j v_j dA[row_j],
// W1[f] -= lr dW1[f]).  ONE launch each; the design is described above
// k_seg_bulk below (equal entry ranges per CTA and warp, TMA bulk-copy row
// gathers into shared-memory rings, ordered combines across warps and CTAs:
// deterministic, no float atomics, balanced whatever the lognormal row
// lengths / Zipf feature frequencies).
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

__device__ __forceinline__ void fence_proxy_async_seg() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

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

// =====================================================================
// v2: entry ranges per CTA / warp with TMA bulk-copy gathers.
//
// The entries are cut into G equal contiguous CTA ranges (G = one CTA per SM)
// and every CTA range into NW equal warp ranges.  A warp walks its range in
// groups of GE entries: every source row of a group (512 B at h = 128) is
// fetched with one cp.async.bulk into the warp's NST-stage shared-memory ring,
// completing on the stage's mbarrier, so a warp keeps NST*GE rows in flight at
// no register cost; the metadata of the next groups is prefetched into
// registers.  Sums follow entry order inside a warp range; a segment crossing
// warp ranges is combined in warp order through shared memory after one
// __syncthreads, and a segment crossing CTA ranges in CTA order by the last
// CTA to arrive (integer counter).  Deterministic, no float atomics.
// MODE 1 also prefetches, with the gathers, the W1 row of every segment that
// ends inside the group, so the fused SGD W1[f] -= lr dW1[f] needs no
// dependent load.
// =====================================================================
__device__ __forceinline__ uint32_t sm32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void sb_init(uint64_t *b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm32(b)), "r"(cnt));
}
__device__ __forceinline__ void sb_expect(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void sb_wait(uint64_t *b, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(sm32(b)), "r"(parity) : "memory");
  } while (!ok);
}
__device__ __forceinline__ void sb_copy(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(sm32(dst)), "l"((uint64_t)src), "r"(bytes), "r"(sm32(bar)) : "memory");
}

// warps per CTA, ring stages per warp, entries per group: measured on B200 at
// the Amazon-670K shape (scripts/x_probe.sh sweep); h = 256 keeps the
// 227 KB shared-memory budget.  -D overrides for experiment builds.
// h = 256 (AmazonCat-13K, scripts/gpu_r02zb.sh sweeps): dW1 6 -> 16 warps
// with 3-entry groups 0.039 -> 0.030 ms, SpMM 8 -> 16 warps with 4-entry
// groups 0.0224 -> 0.0210 ms per SGD step (more warps, each with less in flight)
#ifndef AS_SEG1_NW
#define AS_SEG1_NW 16
#define AS_SEG1_NST 2
#define AS_SEG1_GE (H == 128 ? 6 : 3)
#endif
#ifndef AS_SEG0_NW
#define AS_SEG0_NW 16
#define AS_SEG0_NST 3
#define AS_SEG0_GE (H == 128 ? 8 : 4)
#endif
template <int H, int MODE>
struct SegCfg {
  static constexpr int GE = MODE == 0 ? AS_SEG0_GE : AS_SEG1_GE;     // entries per group
  static constexpr int NW = MODE == 0 ? AS_SEG0_NW : AS_SEG1_NW;     // warps per CTA
  static constexpr int NST = MODE == 0 ? AS_SEG0_NST : AS_SEG1_NST;  // ring stages per warp
  static constexpr int ROW = H * 4;                   // bytes per gathered row
  static constexpr int STAGE = GE * ROW * (MODE == 1 ? 2 : 1);   // + prefetched W1 rows (MODE 1)
  static constexpr int SMEM = NW * NST * STAGE + NW * 2 * ROW + NW * NST * 8;
  static_assert(SMEM <= 232448, "segmented gather-reduce shared memory exceeds 227 KB");
};

// balanced contiguous split of [0, n) into g parts: part c = [c n / g, (c+1) n / g)
__device__ __forceinline__ int split_at(int n, int g, int c) { return (int)(((long long)c * n) / g); }
__device__ __forceinline__ int part_of(int n, int g, int j) {   // the part containing entry j
  int c = (int)(((long long)j * g) / n);
  while (c + 1 < g && split_at(n, g, c + 1) <= j) ++c;
  while (c > 0 && split_at(n, g, c) > j) --c;
  return c;
}

template <int H, int MODE>
__device__ __forceinline__ void seg_finalize(int sg, const float4 (&acc)[H / 128], const float4 (&bb)[H / 128],
                                             int lane, const SegArgs &a, const float4 *w1row) {
  constexpr int V = H / 128;
  if (MODE == 0) {
    fwd_store<H>(sg, acc, bb, lane, a);
  } else {
    const int f = a.seg_key[sg];
    float4 *dst = reinterpret_cast<float4 *>(a.W1 + (size_t)f * H);
#pragma unroll
    for (int q = 0; q < V; ++q) {
      float4 w = w1row ? w1row[lane + 32 * q] : dst[lane + 32 * q];
      w.x -= a.lr * acc[q].x; w.y -= a.lr * acc[q].y; w.z -= a.lr * acc[q].z; w.w -= a.lr * acc[q].w;
      dst[lane + 32 * q] = w;
      if (a.dbg) reinterpret_cast<float4 *>(a.dbg + (size_t)sg * H)[lane + 32 * q] = acc[q];
    }
  }
}

template <int H, int MODE, typename PtrT>
__global__ void __launch_bounds__(SegCfg<H, MODE>::NW * 32, 1)
    k_seg_bulk(const int *__restrict__ n_dev, const int *__restrict__ nseg_dev, int nseg_pad,
               const int32_t *__restrict__ seg_of, const PtrT *__restrict__ seg_ptr,
               const int32_t *__restrict__ gidx, const float *__restrict__ scale,
               const float *__restrict__ src, float *__restrict__ part, int *__restrict__ arrive, SegArgs a) {
  griddep_wait();
  using Cfg = SegCfg<H, MODE>;
  constexpr int V = H / 128, GE = Cfg::GE, NW = Cfg::NW, NST = Cfg::NST, ROW = Cfg::ROW;
  extern __shared__ __align__(128) uint8_t seg_smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint8_t *ring = seg_smem + w * NST * Cfg::STAGE;
  float4 *pieces = reinterpret_cast<float4 *>(seg_smem + NW * NST * Cfg::STAGE);   // [NW][2][H/4]
  uint64_t *full = reinterpret_cast<uint64_t *>(seg_smem + NW * NST * Cfg::STAGE + NW * 2 * ROW) + w * NST;
  const int n = *n_dev;
  const int G = max(1, min((int)gridDim.x, n / 32));           // CTAs with entries (ranges non-empty)
  const int c = blockIdx.x;
  const int cb = c < G ? split_at(n, G, c) : 0, ce = c < G ? split_at(n, G, c + 1) : 0;
  const int wb = cb + split_at(ce - cb, NW, w), we = cb + split_at(ce - cb, NW, w + 1);
  const float4 *S = reinterpret_cast<const float4 *>(src);
  float4 bb[V];
  if (MODE == 0) {
#pragma unroll
    for (int q = 0; q < V; ++q) bb[q] = reinterpret_cast<const float4 *>(a.b1)[lane + 32 * q];
  }
  if (lane == 0) {
    for (int i = 0; i < NST; ++i) sb_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  // per-lane metadata of one group (lane u < GE = entry e0 + u)
  struct Meta { int idx, sg, s0, s1, key; float sc; };
  const int ngr = (we - wb + GE - 1) / GE;
  auto load_meta = [&](int k) {
    Meta m{0, -1, 0, 0, 0, 0.f};
    const int e = wb + k * GE + lane;
    if (k < ngr && lane < GE && e < we) {
      m.idx = gidx[e];
      m.sc = scale[e];
      m.sg = seg_of[e];
      m.s0 = (int)seg_ptr[m.sg];
      m.s1 = (int)seg_ptr[m.sg + 1];
      if (MODE == 1) m.key = a.seg_key[m.sg];
    }
    return m;
  };
  // gathers of group k (need only the source rows: one metadata round trip);
  // MODE 1's W1 prefetch follows in issue_w1 once the segment bounds are in
  auto issue = [&](int k, const Meta &m) {
    if (k >= ngr) return;
    const int st = k % NST;
    uint8_t *buf = ring + st * Cfg::STAGE;
    const int e0 = wb + k * GE, cnt = min(GE, we - e0);
    fence_proxy_async_seg();
    if (lane == 0) {
      if (MODE == 0) sb_expect(&full[st], (uint32_t)cnt * ROW);
      else asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(sm32(&full[st])),
                        "r"((uint32_t)cnt * ROW) : "memory");
    }
    __syncwarp();
    if (lane < cnt) sb_copy(buf + lane * ROW, S + (size_t)m.idx * (H / 4), ROW, &full[st]);
  };
  auto issue_w1 = [&](int k, const Meta &m) {   // MODE 1: the stage's arrival
    if (MODE != 1 || k >= ngr) return;
    const int st = k % NST;
    uint8_t *buf = ring + st * Cfg::STAGE;
    const int e0 = wb + k * GE, cnt = min(GE, we - e0);
    // W1 row of each segment finalised inside this warp range at this entry
    const bool pre = lane < cnt && m.s1 == e0 + lane + 1 && m.s0 >= wb && m.s1 <= we;
    const int npre = __popc(__ballot_sync(0xffffffffu, pre));
    if (lane == 0) sb_expect(&full[st], (uint32_t)npre * ROW);
    __syncwarp();
    if (pre) sb_copy(buf + (GE + lane) * ROW, a.W1 + (size_t)m.key * H, ROW, &full[st]);
  };

  // prologue: metadata of groups 0..NST, rows of groups 0..NST-1 in flight
  Meta mq[NST + 1];
#pragma unroll
  for (int i = 0; i <= NST; ++i) mq[i] = load_meta(i);
#pragma unroll
  for (int i = 0; i < NST; ++i) issue(i, mq[i]);
#pragma unroll
  for (int i = 0; i < NST; ++i) issue_w1(i, mq[i]);

  if (MODE == 0) {
    // rows no entry covers (empty rows: H = ReLU(b1); zero padding rows of the
    // last 128-row MMA tile) while the first gathers fly
    const int nseg = *nseg_dev;
    for (int sg = blockIdx.x * NW + w; sg < nseg_pad; sg += gridDim.x * NW) {
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

  float4 acc[V];
#pragma unroll
  for (int q = 0; q < V; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  int fsg = 0, fs0 = 0, fs1 = 0, lsg = 0, ls0 = 0, ls1 = 0;   // first / last segment of the range
#pragma unroll 1
  for (int k = 0; k < ngr; ++k) {
    const int st = k % NST;
    const Meta m = mq[0];
    if (k == 0) {
      fsg = __shfl_sync(0xffffffffu, m.sg, 0);
      fs0 = __shfl_sync(0xffffffffu, m.s0, 0);
      fs1 = __shfl_sync(0xffffffffu, m.s1, 0);
    }
    if (k == ngr - 1) {
      const int lu = we - 1 - (wb + k * GE);
      lsg = __shfl_sync(0xffffffffu, m.sg, lu);
      ls0 = __shfl_sync(0xffffffffu, m.s0, lu);
      ls1 = __shfl_sync(0xffffffffu, m.s1, lu);
    }
    sb_wait(&full[st], (uint32_t)((k / NST) & 1));
    const float4 *rows = reinterpret_cast<const float4 *>(ring + st * Cfg::STAGE);
    const int e0 = wb + k * GE, cnt = min(GE, we - e0);
#pragma unroll
    for (int u = 0; u < GE; ++u) {
      if (u < cnt) {
        const float v = __shfl_sync(0xffffffffu, m.sc, u);
#pragma unroll
        for (int q = 0; q < V; ++q) {
          const float4 x = rows[u * (H / 4) + lane + 32 * q];
          acc[q].x = fmaf(v, x.x, acc[q].x);
          acc[q].y = fmaf(v, x.y, acc[q].y);
          acc[q].z = fmaf(v, x.z, acc[q].z);
          acc[q].w = fmaf(v, x.w, acc[q].w);
        }
        const int s1 = __shfl_sync(0xffffffffu, m.s1, u);
        const int e = e0 + u;
        if (s1 == e + 1 || e == we - 1) {     // segment ends here or the warp range does
          const int s0 = __shfl_sync(0xffffffffu, m.s0, u);
          const int sg = __shfl_sync(0xffffffffu, m.sg, u);
          if (s0 >= wb && s1 <= we) {
            seg_finalize<H, MODE>(sg, acc, bb, lane, a, rows + (GE + u) * (H / 4));
          } else {
            float4 *pc = pieces + (w * 2 + (s0 < wb ? 0 : 1)) * (H / 4);
#pragma unroll
            for (int q = 0; q < V; ++q) pc[lane + 32 * q] = acc[q];
          }
#pragma unroll
          for (int q = 0; q < V; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    }
    __syncwarp();
    // rotate the metadata queue; refill the freed stage with group k + NST
#pragma unroll
    for (int i = 0; i < NST; ++i) mq[i] = mq[i + 1];
    issue(k + NST, mq[NST - 1]);
    issue_w1(k + NST, mq[NST - 1]);
    mq[NST] = load_meta(k + NST + 1);
  }
  __syncthreads();

  // ---- segments crossing warp ranges: ordered combine of the CTA's pieces
  // task A: my first segment started before my range and its last entry of
  //         this CTA lies in my range;  task B: my last segment started in my
  //         range and continues past the CTA range.
  if (c < G && we > wb) {
#pragma unroll 1
    for (int task = 0; task < 2; ++task) {
      const int sg = task == 0 ? fsg : lsg;
      const int s0 = task == 0 ? fs0 : ls0, s1 = task == 0 ? fs1 : ls1;
      bool mine;
      if (task == 0) mine = s0 < wb && (s1 <= we || we == ce);
      else mine = s0 >= wb && s1 > ce && we == ce;
      if (!mine) continue;
      float4 t[V];
#pragma unroll
      for (int q = 0; q < V; ++q) t[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int w2 = 0; w2 <= w; ++w2) {      // warps touching sg, in order
        const int b2 = cb + split_at(ce - cb, NW, w2), e2 = cb + split_at(ce - cb, NW, w2 + 1);
        if (b2 >= e2 || b2 >= s1 || e2 <= s0) continue;
        const float4 *pc = pieces + (w2 * 2 + (s0 < b2 ? 0 : 1)) * (H / 4);
#pragma unroll
        for (int q = 0; q < V; ++q) {
          const float4 y = pc[lane + 32 * q];
          t[q].x += y.x; t[q].y += y.y; t[q].z += y.z; t[q].w += y.w;
        }
      }
      if (s0 >= cb && s1 <= ce) {
        seg_finalize<H, MODE>(sg, t, bb, lane, a, nullptr);
        continue;
      }
      // ---- segment crossing CTA ranges: last CTA to arrive sums in CTA order
      float4 *p = reinterpret_cast<float4 *>(part + ((size_t)c * 2 + (s0 < cb ? 0 : 1)) * H);
#pragma unroll
      for (int q = 0; q < V; ++q) p[lane + 32 * q] = t[q];
      const int c0 = part_of(n, G, s0), c1 = part_of(n, G, s1 - 1);
      __threadfence();
      __syncwarp();
      int old = 0;
      if (lane == 0) old = atomicAdd(&arrive[sg], 1);
      old = __shfl_sync(0xffffffffu, old, 0);
      if (old == c1 - c0) {
        __threadfence();
#pragma unroll
        for (int q = 0; q < V; ++q) t[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int cc = c0; cc <= c1; ++cc) {
          const float4 *pp = reinterpret_cast<const float4 *>(
              part + ((size_t)cc * 2 + (s0 < split_at(n, G, cc) ? 0 : 1)) * H);
#pragma unroll
          for (int q = 0; q < V; ++q) {
            const float4 y = __ldcg(pp + lane + 32 * q);
            t[q].x += y.x; t[q].y += y.y; t[q].z += y.z; t[q].w += y.w;
          }
        }
        if (lane == 0) arrive[sg] = 0;        // idle for the next launch
        seg_finalize<H, MODE>(sg, t, bb, lane, a, nullptr);
      }
    }
  }
}

template <int H, int MODE, typename PtrT>
static void seg_bulk_launch(cudaStream_t s, int num_sms, const int *n_dev, const int *nseg_dev, int nseg_pad,
                            const int32_t *seg_of, const PtrT *seg_ptr, const int32_t *gidx, const float *scale,
                            const float *src, float *part, int *arrive, const SegArgs &a) {
  using Cfg = SegCfg<H, MODE>;
  static std::atomic<unsigned long long> attr_dev{0};
  if (first_on_device(attr_dev))
    cudaFuncSetAttribute(k_seg_bulk<H, MODE, PtrT>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
#ifndef AS_SEG_CPS
#define AS_SEG_CPS 1                            // CTAs per SM (experiment override)
#endif
  launch_pdl(k_seg_bulk<H, MODE, PtrT>, dim3(num_sms * AS_SEG_CPS), dim3(Cfg::NW * 32), Cfg::SMEM, s, n_dev, nseg_dev,
             nseg_pad, seg_of, seg_ptr, gidx, scale, src, part, arrive, a);
}

void launch_spmm_chunked(cudaStream_t s, int h, int num_sms, const StepDesc *desc, int bpad, int nnz_cap,
                         const int64_t *row_ptr, const int32_t *col, const float *val,
                         const int32_t *rid, const float *W1, const float *b1, float *Hf,
                         __nv_bfloat16 *Hb, float *part, int *arrive) {
  SegArgs a{};
  a.b1 = b1; a.Hf = Hf; a.Hb = Hb;
  const int cap = nnz_cap > bpad ? nnz_cap : bpad;
  (void)cap;
  if (h == 128)
    seg_bulk_launch<128, 0, int64_t>(s, num_sms, &desc->nnz, &desc->rows, bpad, rid, row_ptr, col, val, W1,
                                     part, arrive, a);
  else
    seg_bulk_launch<256, 0, int64_t>(s, num_sms, &desc->nnz, &desc->rows, bpad, rid, row_ptr, col, val, W1,
                                     part, arrive, a);

}

void launch_dw1_chunked(cudaStream_t s, int h, int num_sms, StepDesc *desc, int nnz_cap,
                        const int32_t *seg_id, const int32_t *seg_of, const int32_t *seg_ptr,
                        const int32_t *seg_row, const float *seg_val, const float *dA, float *W1,
                        float lr, float *part, int *arrive, float *dbg_dW1) {
  SegArgs a{};
  a.seg_key = seg_id; a.W1 = W1; a.lr = lr; a.dbg = dbg_dW1;
  if (h == 128)
    seg_bulk_launch<128, 1, int32_t>(s, num_sms, &desc->nnz, &desc->U, 0, seg_of, seg_ptr, seg_row, seg_val, dA,
                                     part, arrive, a);
  else
    seg_bulk_launch<256, 1, int32_t>(s, num_sms, &desc->nnz, &desc->U, 0, seg_of, seg_ptr, seg_row, seg_val, dA,
                                     part, arrive, a);

}

}  // namespace as

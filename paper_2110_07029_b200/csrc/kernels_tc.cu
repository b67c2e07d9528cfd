// tcgen05 / TMEM / TMA output layer of the Adaptive SGD step (AS_BF16 mode,
// sm_100a).  Steps a5 and a6 of DESIGN.md:
//
//   pass 1 (k_out_fwd): for a 128-row tile of H (bf16) and a range of 128-class
//     blocks of W2T (bf16 shadow), S = H W2T_blk^T + b2 in TMEM, an online
//     softmax in log2 units (one epilogue thread per row, lazy rescale), and
//     O += P W2T_blk in TMEM; the split partials (m, l, O) go to HBM.  This is
//     attention with Q = H and K = V = W2T: the b x C logits never exist.
//   pass 2 (k_out_bwd): persistent CTAs own 128-class blocks; for every row
//     tile S^T = W2T_blk H^T is recomputed, G^T = softmax^T / B is formed in
//     registers (label term applied sparsely later), dW2T^T += H^T G^T
//     accumulates in TMEM over the whole batch, then the epilogue applies the
//     label term, db2, and the fused SGD update of the fp32 master W2T / b2
//     plus the bf16 shadow.  dW2T never touches HBM.
//
// Operands are staged by TMA with 128-byte swizzle; MMAs are
// tcgen05.mma.cta_group::1.kind::f16 (bf16 x bf16 -> fp32), M = 128, issued by
// one thread; accumulators live in TMEM and are read back with tcgen05.ld.
// P:N = PAPER.md line N.
#include <cuda.h>

#include <cfloat>
#include <cstdio>

#include "common.cuh"
#include "tmem_regs.h"

namespace as {
namespace tc {

constexpr int BM = 128;                 // rows per tile == classes per block
constexpr int ATOM_BYTES = 128 * 128;   // one 64-col bf16 atom of a 128-row tile
constexpr float LOG2E = 1.4426950408889634f;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap *map, uint64_t *bar, void *dst,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t *slot, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(slot)),
               "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols)
               : "memory");
}
__device__ __forceinline__ void mma_bf16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                             uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}

// Shared-memory matrix descriptor, 128-byte swizzle (SM100 UMMA format:
// start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46), version 1 at bit 46,
// layout SWIZZLE_128B = 2 at [61,64)).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}
// K-major operand tile [K/64 atoms][128 rows][64 elems]: MMA k-step kk (16 elems)
__device__ __forceinline__ uint64_t desc_k(uint32_t base, int kk) {
  return sdesc(base + (kk >> 2) * ATOM_BYTES + (kk & 3) * 32, 16, 1024);
}
// MN-major view of the same image ([MN/64 atoms][K rows][64 elems]): k-step kk
// covers K rows [16kk, 16kk+16); MN atoms ATOM_BYTES apart (LBO).
__device__ __forceinline__ uint64_t desc_mn(uint32_t base, int kk) {
  return sdesc(base + kk * 2048, ATOM_BYTES, 1024);
}
// Instruction descriptor, kind::f16: D fp32, A/B bf16, majors, N>>3, M>>4.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// byte offset of 16-byte chunk c (8 bf16 of columns 8c..8c+7) of row i in a
// [atoms][128 rows][64] SW128 tile written by threads
__device__ __forceinline__ uint32_t swz(int i, int c) {
  return (uint32_t)((c >> 3) * ATOM_BYTES + i * 128 + (((c & 7) ^ (i & 7)) << 4));
}

template <int H>
struct FwdCfg {
  static constexpr int NST = H == 128 ? 4 : 2;   // W stages
  static constexpr int TILE = BM * H * 2;         // bytes of a 128 x H bf16 tile
  static constexpr int SMEM = TILE /*H*/ + NST * TILE /*W*/ + BM * BM * 2 /*P*/ + 2 * BM * 4 +
                              1024 /*barriers*/ + 1024 /*align*/;
};

// splits of the class range for pass 1 given the batch rows (same formula on
// the device in the combine)
__host__ __device__ inline int fwd_splits(int B, int n_cblocks, int num_ctas, int max_splits) {
  const int RT = (B + BM - 1) / BM;
  int s = num_ctas / (RT > 0 ? RT : 1);
  if (s > n_cblocks) s = n_cblocks;
  if (s > max_splits) s = max_splits;
  return s < 1 ? 1 : s;
}

// =====================================================================
// pass 1
// =====================================================================
template <int H>
__global__ void __launch_bounds__(192, 1)
    k_out_fwd(const __grid_constant__ CUtensorMap mapH, const __grid_constant__ CUtensorMap mapW,
              const StepDesc *__restrict__ desc, const float *__restrict__ b2, int C,
              int n_cblocks, int max_splits, int bpad, float *__restrict__ pm,
              float *__restrict__ pl, float *__restrict__ pO) {
  using Cfg = FwdCfg<H>;
  constexpr int NST = Cfg::NST, TILE = Cfg::TILE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *sm = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t *sH = sm;
  uint8_t *sW = sH + TILE;
  uint8_t *sP = sW + NST * TILE;
  float *sB2 = (float *)(sP + BM * BM * 2);
  uint64_t *bars = (uint64_t *)(sB2 + 2 * BM);
  uint64_t *h_full = bars, *w_full = bars + 1, *w_empty = w_full + NST, *s_full = w_empty + NST,
           *s_empty = s_full + 2, *p_full = s_empty + 2, *o_done = p_full + 1;
  uint32_t *tmem_slot = (uint32_t *)(o_done + 1);

  const int B = desc->rows;
  const int RT = (B + BM - 1) / BM;
  const int splits = fwd_splits(B, n_cblocks, gridDim.x, max_splits);
  const int rt = blockIdx.x / splits, sp = blockIdx.x % splits;
  if (rt >= RT) return;
  const int cb0 = (int)((long long)sp * n_cblocks / splits);
  const int nloc = (int)((long long)(sp + 1) * n_cblocks / splits) - cb0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(h_full, 1);
    for (int i = 0; i < NST; ++i) { mbar_init(&w_full[i], 1); mbar_init(&w_empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&s_full[i], 1); mbar_init(&s_empty[i], 4); }
    mbar_init(p_full, 4);
    mbar_init(o_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      mbar_expect_tx(h_full, TILE);
      for (int a = 0; a < H / 64; ++a) tma_load_2d(&mapH, h_full, sH + a * ATOM_BYTES, a * 64, rt * BM);
      for (int j = 0; j < nloc; ++j) {
        const int st = j % NST;
        if (j >= NST) mbar_wait(&w_empty[st], ((j / NST) - 1) & 1);
        mbar_expect_tx(&w_full[st], TILE);
        for (int a = 0; a < H / 64; ++a)
          tma_load_2d(&mapW, &w_full[st], sW + st * TILE + a * ATOM_BYTES, a * 64, (cb0 + j) * BM);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      constexpr uint32_t idS = idesc_bf16(BM, BM, 0, 0);
      constexpr uint32_t idO = idesc_bf16(BM, H, 0, 1);
      const uint32_t aH = smem_u32(sH), aW = smem_u32(sW), aP = smem_u32(sP);
      mbar_wait(h_full, 0);
      fence_after();
      auto issue_S = [&](int j) {
        const int st = j % NST, b = j & 1;
        mbar_wait(&w_full[st], (j / NST) & 1);
        if (j >= 2) mbar_wait(&s_empty[b], ((j >> 1) - 1) & 1);
        fence_after();
#pragma unroll
        for (int kk = 0; kk < H / 16; ++kk)
          mma_bf16(tmem + b * BM, desc_k(aH, kk), desc_k(aW + st * TILE, kk), idS, kk > 0);
        mma_commit(&s_full[b]);
      };
      if (nloc > 0) issue_S(0);
      for (int j = 0; j < nloc; ++j) {
        if (j + 1 < nloc) issue_S(j + 1);
        mbar_wait(p_full, j & 1);
        fence_after();
        const int st = j % NST;
#pragma unroll
        for (int kk = 0; kk < BM / 16; ++kk)
          mma_bf16(tmem + 2 * BM, desc_k(aP, kk), desc_mn(aW + st * TILE, kk), idO,
                   (j > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&w_empty[st]);
        mma_commit(o_done);
      }
    }
  } else {  // ---------------- softmax / epilogue warps (one thread per row)
    const int q = warp & 3;
    const int e = threadIdx.x - 64;           // 0..127 loader index
    const int row = q * 32 + lane;            // TMEM lane == tile row
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t aP = smem_u32(sP);
    float m_used = -FLT_MAX, l = 0.f;
    for (int j = 0; j < nloc; ++j) {
      const int cb = cb0 + j;
      {
        const int c = cb * BM + e;
        sB2[(j & 1) * BM + e] = c < C ? b2[c] * LOG2E : -INFINITY;
      }
      named_bar(1, 128);
      mbar_wait(&s_full[j & 1], (j >> 1) & 1);
      fence_after();
      float v[BM];
#pragma unroll
      for (int ch = 0; ch < BM / 32; ++ch) {
        uint32_t r[32];
        AS_TMEM_LD32(tl + (j & 1) * BM + ch * 32, r);
        AS_TMEM_WAIT_LD(r);
#pragma unroll
        for (int k = 0; k < 32; ++k) v[ch * 32 + k] = __uint_as_float(r[k]);
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[j & 1]);
      float mx = -FLT_MAX;
      const float *bb = sB2 + (j & 1) * BM;
#pragma unroll
      for (int k = 0; k < BM; ++k) {
        v[k] = fmaf(v[k], LOG2E, bb[k]);
        mx = fmaxf(mx, v[k]);
      }
      float m_new = m_used;
      if (mx > m_used + 8.f) m_new = mx;   // lazy rescale: p <= 2^8 otherwise
      float rs = 0.f;
#pragma unroll
      for (int k = 0; k < BM; ++k) {
        v[k] = ex2(v[k] - m_new);
        rs += v[k];
      }
      if (j > 0) {
        mbar_wait(o_done, (j - 1) & 1);   // O_{j-1} done: P buffer free, O stable
        fence_after();
      }
      // lazy rescale (per row); tcgen05.ld/st are warp-collective, so the TMEM
      // pass runs for the whole warp when any of its rows needs it (sc = 1 else)
      const bool need = m_new != m_used;
      const float sc = need ? ((m_used == -FLT_MAX) ? 0.f : ex2(m_used - m_new)) : 1.f;
      l *= sc;
      m_used = m_new;
      if (j > 0 && __any_sync(0xffffffffu, need)) {
#pragma unroll 1
        for (int ch = 0; ch < H / 32; ++ch) {
          uint32_t r[32];
          AS_TMEM_LD32(tl + 2 * BM + ch * 32, r);
          AS_TMEM_WAIT_LD(r);
#pragma unroll
          for (int k = 0; k < 32; ++k) r[k] = __float_as_uint(__uint_as_float(r[k]) * sc);
          AS_TMEM_ST32(tl + 2 * BM + ch * 32, r);
        }
        tmem_wait_st();
      }
      l += rs;
#pragma unroll
      for (int c = 0; c < BM / 8; ++c)
        st_shared_v4(aP + swz(row, c), pack_bf16x2(v[8 * c], v[8 * c + 1]),
                     pack_bf16x2(v[8 * c + 2], v[8 * c + 3]), pack_bf16x2(v[8 * c + 4], v[8 * c + 5]),
                     pack_bf16x2(v[8 * c + 6], v[8 * c + 7]));
      fence_proxy_async();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    // epilogue: partials of this split
    const int grow = rt * BM + row;
    if (nloc > 0) {
      mbar_wait(o_done, (nloc - 1) & 1);
      fence_after();
#pragma unroll 1
      for (int ch = 0; ch < H / 32; ++ch) {
        uint32_t r[32];
        AS_TMEM_LD32(tl + 2 * BM + ch * 32, r);
        AS_TMEM_WAIT_LD(r);
#pragma unroll
        for (int k = 0; k < 32; ++k)
          pO[((size_t)sp * H + ch * 32 + k) * bpad + grow] = __uint_as_float(r[k]);
      }
    } else {
      for (int k = 0; k < H; ++k) pO[((size_t)sp * H + k) * bpad + grow] = 0.f;
    }
    pm[(size_t)sp * bpad + grow] = m_used;
    pl[(size_t)sp * bpad + grow] = l;
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// =====================================================================
// pass 2
// =====================================================================
template <int H>
struct BwdCfg {
  static constexpr int NW = H == 128 ? 2 : 1;    // W2T block buffers
  static constexpr int NSH = 2 + (H == 128);      // H tile stages
  static constexpr int TILE = BM * H * 2;
  static constexpr int SMEM = NW * TILE + NSH * TILE + BM * BM * 2 /*G*/ + 2 * BM * 4 /*lse*/ +
                              1024 + 1024;
};

template <int H>
__global__ void __launch_bounds__(192, 1)
    k_out_bwd(const __grid_constant__ CUtensorMap mapH, const __grid_constant__ CUtensorMap mapW,
              const StepDesc *__restrict__ desc, const float *__restrict__ lse2, int C,
              int n_cblocks, const int32_t *__restrict__ cls_seg,
              const int32_t *__restrict__ lseg_ptr, const int32_t *__restrict__ lrow,
              const int64_t *__restrict__ lab_ptr, const float *__restrict__ Hf,
              float *__restrict__ W2T, float *__restrict__ b2, __nv_bfloat16 *__restrict__ W2b,
              float lr, float *__restrict__ dbg_dW2T, float *__restrict__ dbg_db2) {
  using Cfg = BwdCfg<H>;
  constexpr int NW = Cfg::NW, NSH = Cfg::NSH, TILE = Cfg::TILE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *sm = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t *sW = sm;
  uint8_t *sHt = sW + NW * TILE;
  uint8_t *sG = sHt + NSH * TILE;
  float *sL = (float *)(sG + BM * BM * 2);
  uint64_t *bars = (uint64_t *)(sL + 2 * BM);
  uint64_t *w_full = bars, *w_empty = w_full + NW, *h_full = w_empty + NW, *h_empty = h_full + NSH,
           *s_full = h_empty + NSH, *s_empty = s_full + 2, *g_full = s_empty + 2,
           *g_empty = g_full + 1, *dw_full = g_empty + 1, *dw_empty = dw_full + 1;
  uint32_t *tmem_slot = (uint32_t *)(dw_empty + 1);

  const int B = desc->rows;
  const int RT = (B + BM - 1) / BM;
  const float invB = 1.0f / (float)B;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NW; ++i) { mbar_init(&w_full[i], 1); mbar_init(&w_empty[i], 1); }
    for (int i = 0; i < NSH; ++i) { mbar_init(&h_full[i], 1); mbar_init(&h_empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&s_full[i], 1); mbar_init(&s_empty[i], 4); }
    mbar_init(g_full, 4);
    mbar_init(g_empty, 1);
    mbar_init(dw_full, 1);
    mbar_init(dw_empty, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int kb = 0, it = 0;
      for (int cb = blockIdx.x; cb < n_cblocks; cb += gridDim.x, ++kb) {
        const int wb = kb % NW;
        if (kb >= NW) mbar_wait(&w_empty[wb], ((kb / NW) - 1) & 1);
        mbar_expect_tx(&w_full[wb], TILE);
        for (int a = 0; a < H / 64; ++a)
          tma_load_2d(&mapW, &w_full[wb], sW + wb * TILE + a * ATOM_BYTES, a * 64, cb * BM);
        for (int t = 0; t < RT; ++t, ++it) {
          const int st = it % NSH;
          if (it >= NSH) mbar_wait(&h_empty[st], ((it / NSH) - 1) & 1);
          mbar_expect_tx(&h_full[st], TILE);
          for (int a = 0; a < H / 64; ++a)
            tma_load_2d(&mapH, &h_full[st], sHt + st * TILE + a * ATOM_BYTES, a * 64, t * BM);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      constexpr uint32_t idS = idesc_bf16(BM, BM, 0, 0);   // S^T = W2T_blk . H_t^T
      constexpr uint32_t idW = idesc_bf16(BM, BM, 1, 0);   // dW^T += H_t^T . G^T^T
      const uint32_t aW = smem_u32(sW), aH = smem_u32(sHt), aG = smem_u32(sG);
      int kb = 0, it = 0, sj = 0, gj = 0;
      auto do_dw = [&](int t, int st) {
        mbar_wait(g_full, gj & 1);
        if (t == 0 && kb >= 1) mbar_wait(dw_empty, (kb - 1) & 1);
        fence_after();
#pragma unroll
        for (int half = 0; half < H / 128; ++half)
#pragma unroll
          for (int kk = 0; kk < BM / 16; ++kk)
            mma_bf16(tmem + 2 * BM + half * BM, desc_mn(aH + st * TILE + half * 2 * ATOM_BYTES, kk),
                     desc_k(aG, kk), idW, (t > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&h_empty[st]);
        mma_commit(g_empty);
        ++gj;
      };
      for (int cb = blockIdx.x; cb < n_cblocks; cb += gridDim.x, ++kb) {
        const int wb = kb % NW;
        mbar_wait(&w_full[wb], (kb / NW) & 1);
        int st_prev = 0;
        for (int t = 0; t < RT; ++t, ++it) {
          const int st = it % NSH, b = sj & 1;
          mbar_wait(&h_full[st], (it / NSH) & 1);
          if (sj >= 2) mbar_wait(&s_empty[b], ((sj >> 1) - 1) & 1);
          fence_after();
#pragma unroll
          for (int kk = 0; kk < H / 16; ++kk)
            mma_bf16(tmem + b * BM, desc_k(aW + wb * TILE, kk), desc_k(aH + st * TILE, kk), idS,
                     kk > 0);
          mma_commit(&s_full[b]);
          ++sj;
          if (t == RT - 1) mma_commit(&w_empty[wb]);
          if (t > 0) do_dw(t - 1, st_prev);
          st_prev = st;
        }
        do_dw(RT - 1, st_prev);
        mma_commit(dw_full);
      }
    }
  } else {  // ---------------- epilogue warps
    const int q = warp & 3;
    const int e = threadIdx.x - 64;
    const int i = q * 32 + lane;                       // TMEM lane
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t aG = smem_u32(sG);
    int kb = 0, sj = 0, gj = 0;
    for (int cb = blockIdx.x; cb < n_cblocks; cb += gridDim.x, ++kb) {
      const int c = cb * BM + i;
      const bool cvalid = c < C;
      const float b2c = cvalid ? b2[c] * LOG2E : 0.f;
      float db2 = 0.f;
      for (int t = 0; t < RT; ++t) {
        const int b = sj & 1;
        {
          const int r = t * BM + e;
          sL[b * BM + e] = r < B ? lse2[r] : INFINITY;
        }
        named_bar(1, 128);
        mbar_wait(&s_full[b], (sj >> 1) & 1);
        fence_after();
        float v[BM];
#pragma unroll
        for (int ch = 0; ch < BM / 32; ++ch) {
          uint32_t r[32];
          AS_TMEM_LD32(tl + b * BM + ch * 32, r);
          AS_TMEM_WAIT_LD(r);
#pragma unroll
          for (int k = 0; k < 32; ++k) v[ch * 32 + k] = __uint_as_float(r[k]);
        }
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[b]);
        ++sj;
        const float *ls = sL + b * BM;
        float rs = 0.f;
#pragma unroll
        for (int k = 0; k < BM; ++k) {
          const float p = cvalid ? ex2(fmaf(v[k], LOG2E, b2c) - ls[k]) * invB : 0.f;
          v[k] = p;
          rs += p;
        }
        db2 += rs;
        if (gj >= 1) {
          mbar_wait(g_empty, (gj - 1) & 1);
        }
#pragma unroll
        for (int cc = 0; cc < BM / 8; ++cc)
          st_shared_v4(aG + swz(i, cc), pack_bf16x2(v[8 * cc], v[8 * cc + 1]),
                       pack_bf16x2(v[8 * cc + 2], v[8 * cc + 3]),
                       pack_bf16x2(v[8 * cc + 4], v[8 * cc + 5]),
                       pack_bf16x2(v[8 * cc + 6], v[8 * cc + 7]));
        fence_proxy_async();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(g_full);
        ++gj;
      }
      // ---- dW epilogue: thread = hidden unit j, loop over the block's classes.
      // All loads of a 32-class chunk are issued before any use (latency hiding);
      // the label term (R3) is applied from the label-sorted batch.
      mbar_wait(dw_full, kb & 1);
      fence_after();
#pragma unroll 1
      for (int half = 0; half < H / 128; ++half) {
        const int j = half * BM + i;
#pragma unroll 1
        for (int ch = 0; ch < BM / 32; ++ch) {
          uint32_t r[32];
          AS_TMEM_LD32(tl + 2 * BM + half * BM + ch * 32, r);
          AS_TMEM_WAIT_LD(r);
          const int c0 = cb * BM + ch * 32;
          const int my_seg = (c0 + lane < C) ? cls_seg[c0 + lane] : -1;
          float w[32];
#pragma unroll
          for (int k = 0; k < 32; ++k)
            w[k] = (c0 + k < C) ? W2T[(size_t)(c0 + k) * H + j] : 0.f;
          unsigned any = __ballot_sync(0xffffffffu, my_seg >= 0);
          while (any) {                       // classes of this chunk that carry labels
            const int k = __ffs(any) - 1;
            any &= any - 1;
            const int sg = __shfl_sync(0xffffffffu, my_seg, k);
            float corr = 0.f;
            for (int u = lseg_ptr[sg]; u < lseg_ptr[sg + 1]; ++u) {
              const int rr = lrow[u];
              const float kr = (float)(lab_ptr[rr + 1] - lab_ptr[rr]);
              corr += Hf[(size_t)rr * H + j] * (invB / kr);
            }
#pragma unroll
            for (int q = 0; q < 32; ++q)
              if (q == k) r[q] = __float_as_uint(__uint_as_float(r[q]) - corr);
          }
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            if (c0 + k < C) {
              const float g = __uint_as_float(r[k]);
              const size_t idx = (size_t)(c0 + k) * H + j;
              const float nw = w[k] - lr * g;
              W2T[idx] = nw;
              W2b[idx] = __float2bfloat16_rn(nw);
              if (dbg_dW2T) dbg_dW2T[idx] = g;
            }
          }
        }
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dw_empty);
      if (cvalid) {
        const int sg = cls_seg[c];
        if (sg >= 0) {
          for (int u = lseg_ptr[sg]; u < lseg_ptr[sg + 1]; ++u) {
            const int rr = lrow[u];
            db2 -= invB / (float)(lab_ptr[rr + 1] - lab_ptr[rr]);
          }
        }
        b2[c] -= lr * db2;
        if (dbg_db2) dbg_db2[c] = db2;
      }
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// =====================================================================
// self-test of the descriptors / swizzle (tests only): one CTA, H = 128
//   S[i][n]  = sum_k A[i][k] B[n][k]          (K-major x K-major)
//   O[i][j]  = sum_n P[i][n] B[n][j]          (thread-written P, MN-major B)
//   T[j][n]  = sum_r A[r][j] P[n][r]          (MN-major A, thread-written P)
// P[i][n] = bf16(S[i][n] * 1/16) written by the epilogue threads.
// =====================================================================
__global__ void __launch_bounds__(192, 1)
    k_tc_selftest(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                  float *__restrict__ S, float *__restrict__ O, float *__restrict__ T) {
  constexpr int TILE = BM * 128 * 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *sm = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t *sA = sm, *sB = sA + TILE, *sP = sB + TILE;
  uint64_t *bars = (uint64_t *)(sP + TILE);
  uint64_t *ld_full = bars, *mma1 = bars + 1, *p_full = bars + 2, *mma2 = bars + 3;
  uint32_t *tmem_slot = (uint32_t *)(bars + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(ld_full, 1); mbar_init(mma1, 1); mbar_init(p_full, 4); mbar_init(mma2, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == 0 && lane == 0) {
    mbar_expect_tx(ld_full, 2 * TILE);
    for (int a = 0; a < 2; ++a) {
      tma_load_2d(&mapA, ld_full, sA + a * ATOM_BYTES, a * 64, 0);
      tma_load_2d(&mapB, ld_full, sB + a * ATOM_BYTES, a * 64, 0);
    }
  } else if (warp == 1 && lane == 0) {
    mbar_wait(ld_full, 0);
    fence_after();
    const uint32_t aA = smem_u32(sA), aB = smem_u32(sB), aP = smem_u32(sP);
    for (int kk = 0; kk < 8; ++kk)
      mma_bf16(tmem, desc_k(aA, kk), desc_k(aB, kk), idesc_bf16(128, 128, 0, 0), kk > 0);
    mma_commit(mma1);
    mbar_wait(p_full, 0);
    fence_after();
    for (int kk = 0; kk < 8; ++kk)
      mma_bf16(tmem + 128, desc_k(aP, kk), desc_mn(aB, kk), idesc_bf16(128, 128, 0, 1), kk > 0);
    for (int kk = 0; kk < 8; ++kk)
      mma_bf16(tmem + 256, desc_mn(aA, kk), desc_k(aP, kk), idesc_bf16(128, 128, 1, 0), kk > 0);
    mma_commit(mma2);
  } else if (warp >= 2) {
    const int q = warp & 3, row = q * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    mbar_wait(mma1, 0);
    fence_after();
    float v[128];
    for (int ch = 0; ch < 4; ++ch) {
      uint32_t r[32];
      AS_TMEM_LD32(tl + ch * 32, r);
      AS_TMEM_WAIT_LD(r);
      for (int k = 0; k < 32; ++k) v[ch * 32 + k] = __uint_as_float(r[k]);
    }
    for (int k = 0; k < 128; ++k) S[row * 128 + k] = v[k];
    const uint32_t aP = smem_u32(sP);
    for (int c = 0; c < 16; ++c)
      st_shared_v4(aP + swz(row, c), pack_bf16x2(v[8 * c] * 0.0625f, v[8 * c + 1] * 0.0625f),
                   pack_bf16x2(v[8 * c + 2] * 0.0625f, v[8 * c + 3] * 0.0625f),
                   pack_bf16x2(v[8 * c + 4] * 0.0625f, v[8 * c + 5] * 0.0625f),
                   pack_bf16x2(v[8 * c + 6] * 0.0625f, v[8 * c + 7] * 0.0625f));
    fence_proxy_async();
    fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(p_full);
    mbar_wait(mma2, 0);
    fence_after();
    for (int ch = 0; ch < 4; ++ch) {
      uint32_t r[32];
      AS_TMEM_LD32(tl + 128 + ch * 32, r);
      AS_TMEM_WAIT_LD(r);
      for (int k = 0; k < 32; ++k) O[row * 128 + ch * 32 + k] = __uint_as_float(r[k]);
      AS_TMEM_LD32(tl + 256 + ch * 32, r);
      AS_TMEM_WAIT_LD(r);
      for (int k = 0; k < 32; ++k) T[row * 128 + ch * 32 + k] = __uint_as_float(r[k]);
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

}  // namespace tc

// =====================================================================
// host side: tensor maps and launchers
// =====================================================================
typedef CUresult (*PFN_encodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                    const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                    const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_encodeTiled)p;
  }
  return fn;
}

// bf16 row-major [rows][cols] with a {64, 128} box and 128-byte swizzle
static int make_map(CUtensorMap *m, const void *base, long long rows, int cols) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return -1;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

struct TcPlan {
  CUtensorMap mapH, mapW;
  int h, b_max, bpad, n_cblocks, num_sms, max_splits;
  long long C;
};

size_t tc_plan_bytes() { return sizeof(TcPlan); }

int tc_splits(int h, int b_max, long long C, int num_sms) {
  (void)h; (void)b_max;
  const int ncb = (int)((C + tc::BM - 1) / tc::BM);
  return num_sms < ncb ? num_sms : ncb;   // capacity of the partial buffers
}

int tc_plan_init(TcPlan *plan, int h, int b_max, long long C, int num_sms, const void *Hb,
                 const void *W2b) {
  plan->h = h;
  plan->b_max = b_max;
  plan->bpad = (b_max + tc::BM - 1) / tc::BM * tc::BM;
  plan->C = C;
  plan->n_cblocks = (int)((C + tc::BM - 1) / tc::BM);
  plan->num_sms = num_sms < 160 ? num_sms : 160;   // partial buffers sized for 160
  plan->max_splits = tc_splits(h, b_max, C, plan->num_sms);
  if (make_map(&plan->mapH, Hb, plan->bpad, h) != 0) return -1;
  if (make_map(&plan->mapW, W2b, C, h) != 0) return -1;
  static bool attr_done[2] = {false, false};
  const int hi = h == 128 ? 0 : 1;
  if (!attr_done[hi]) {
    if (h == 128) {
      cudaFuncSetAttribute(tc::k_out_fwd<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           tc::FwdCfg<128>::SMEM);
      cudaFuncSetAttribute(tc::k_out_bwd<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           tc::BwdCfg<128>::SMEM);
    } else {
      cudaFuncSetAttribute(tc::k_out_fwd<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           tc::FwdCfg<256>::SMEM);
      cudaFuncSetAttribute(tc::k_out_bwd<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           tc::BwdCfg<256>::SMEM);
    }
    attr_done[hi] = true;
  }
  return 0;
}

void launch_out_fwd_tc(cudaStream_t s, const TcPlan *p, const StepDesc *desc, const float *b2,
                       float *pm, float *pl, float *pO) {
  if (p->h == 128)
    tc::k_out_fwd<128><<<p->num_sms, 192, tc::FwdCfg<128>::SMEM, s>>>(
        p->mapH, p->mapW, desc, b2, (int)p->C, p->n_cblocks, p->max_splits, p->bpad, pm, pl, pO);
  else
    tc::k_out_fwd<256><<<p->num_sms, 192, tc::FwdCfg<256>::SMEM, s>>>(
        p->mapH, p->mapW, desc, b2, (int)p->C, p->n_cblocks, p->max_splits, p->bpad, pm, pl, pO);
}

int tc_fwd_splits_host(const TcPlan *p, int B) {
  return tc::fwd_splits(B, p->n_cblocks, p->num_sms, p->max_splits);
}

void launch_out_bwd_tc(cudaStream_t s, const TcPlan *p, const StepDesc *desc, const float *lse2,
                       const float *b2_in, const int32_t *cls_seg, const int32_t *lseg_ptr,
                       const int32_t *lrow, const int64_t *lab_ptr, const float *Hf, float *W2T,
                       float *b2, __nv_bfloat16 *W2b, float lr, float *dbg_dW2T, float *dbg_db2,
                       float *db2_tmp) {
  (void)b2_in; (void)db2_tmp;
  const int grid = p->num_sms < p->n_cblocks ? p->num_sms : p->n_cblocks;
  if (p->h == 128)
    tc::k_out_bwd<128><<<grid, 192, tc::BwdCfg<128>::SMEM, s>>>(
        p->mapH, p->mapW, desc, lse2, (int)p->C, p->n_cblocks, cls_seg, lseg_ptr, lrow, lab_ptr,
        Hf, W2T, b2, W2b, lr, dbg_dW2T, dbg_db2);
  else
    tc::k_out_bwd<256><<<grid, 192, tc::BwdCfg<256>::SMEM, s>>>(
        p->mapH, p->mapW, desc, lse2, (int)p->C, p->n_cblocks, cls_seg, lseg_ptr, lrow, lab_ptr,
        Hf, W2T, b2, W2b, lr, dbg_dW2T, dbg_db2);
}

// test hook: A, B bf16 [128][128] device; S, O, T fp32 [128][128] device
int tc_selftest(const void *A, const void *B, float *S, float *O, float *T, cudaStream_t s) {
  CUtensorMap mA, mB;
  if (make_map(&mA, A, 128, 128) != 0 || make_map(&mB, B, 128, 128) != 0) return -1;
  const int smem = 3 * 128 * 128 * 2 + 2048;
  cudaFuncSetAttribute(tc::k_tc_selftest, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  tc::k_tc_selftest<<<1, 192, smem, s>>>(mA, mB, S, O, T);
  return 0;
}

}  // namespace as

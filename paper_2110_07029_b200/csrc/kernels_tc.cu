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

#ifdef AS_TRACE
// event log of CTA 0 (trace builds only): per role {clock, event, tile}, plain
// stores from one thread per role (no atomics on the timed path)
__device__ long long g_trace[4][4096][3];
__device__ int g_trace_n[4];
#define TRACE_INIT int _trk = 0
#define TRACE(role, cond, ev, tile)                                           \
  do {                                                                        \
    if ((cond) && blockIdx.x == 0 && _trk < 4096) {                          \
      g_trace[role][_trk][0] = clock64(); g_trace[role][_trk][1] = (ev);      \
      g_trace[role][_trk][2] = (tile); ++_trk; g_trace_n[role] = _trk;        \
    }                                                                         \
  } while (0)
#else
#define TRACE_INIT
#define TRACE(role, cond, ev, tile) do {} while (0)
#endif

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
// the same with a suspend-time hint (ns): for waits off the critical path
// (producers, the update loop), so the waiting warp sleeps in the barrier
// instead of re-polling (issue slots and power under the power cap)
__device__ __forceinline__ void mbar_wait_idle(uint64_t *b, uint32_t parity) {
#ifdef AS_X_NOSUSPEND
  mbar_wait(b, parity);
#else
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity), "r"(2000u)
        : "memory");
  } while (!ok);
#endif
}
// the update warps' long waits (a whole class block): poll with a plain
// nanosleep between phase tests.  The try_wait suspend of mbar_wait_idle wakes on
// barrier traffic, and pass 2 has plenty: measured ~7 000 wake-ups per warp per
// launch (16 M of the kernel's 176 M warp-instructions, on the softmax warps'
// sub-partitions).  Measured slightly slower (Amazon-670K step 0.6673 -> 0.6694 ms):
// off unless AS_X_SLEEPY.
__device__ __forceinline__ void mbar_wait_sleepy(uint64_t *b, uint32_t parity, uint32_t ns) {
#ifndef AS_X_SLEEPY
  (void)ns;
  mbar_wait_idle(b, parity);
#else
  for (;;) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
    if (ok) break;
    __nanosleep(ns);
  }
#endif
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap *map, uint64_t *bar, void *dst,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap *map, const void *src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   (uint64_t)map),
               "r"(c0), "r"(c1), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"((uint64_t)src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// cp.async (LDGSTS) global -> shared, zero-filled beyond src_bytes
__device__ __forceinline__ void cp_async_16(void *sdst, const void *gsrc, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_8(void *sdst, const void *gsrc, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_4(void *sdst, const void *gsrc, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
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
// A from TMEM (lane = row of A, two bf16 per 32-bit column along K), B from smem
__device__ __forceinline__ void mma_bf16_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
}  // namespace tc
#include "mma_groups.h"
namespace tc {
// Warp-converged variants: all 32 lanes execute the call, one elected lane
// issues (no divergent single-lane region => no ELECT/branch loop per MMA).
__device__ __forceinline__ void mma_ss_w(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_ts_w(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                         uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit_w(uint64_t *bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
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
// packed fp32x2 arithmetic (FFMA2 / FADD2 on sm_100): one issue slot per pair
__device__ __forceinline__ uint64_t f2(float lo, float hi) {
  uint64_t v;
  asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "f"(lo), "f"(hi));
  return v;
}
__device__ __forceinline__ void f2split(uint64_t v, float &lo, float &hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// 2^x for a packed pair on the FMA / integer pipes (offloads the MUFU, which
// is the co-bottleneck with the tensor pipe at h = 128): n = rint(x) by the
// 1.5 * 2^23 shift, f = x - n in [-0.5, 0.5], 2^f by a degree-3 polynomial
// (relative-error minimax, max rel. error 7.5e-5, far below the bf16 rounding
// of P and G), exponent n added to the bit pattern.  x is clamped at -125 so
// the exponent never underflows (2^-125 instead of 0: no effect on sums).
__device__ __forceinline__ void ex2_emu2(uint64_t x, float &p0, float &p1) {
  float x0, x1;
  f2split(x, x0, x1);
  x = f2(fmaxf(x0, -125.f), fmaxf(x1, -125.f));
  const uint64_t M2 = f2(12582912.f, 12582912.f);
  const uint64_t t = fadd2(x, M2);
  const uint64_t fr = fsub2(x, fsub2(t, M2));
  uint64_t q = ffma2(fr, f2(0.055171321099324135f, 0.055171321099324135f),
                     f2(0.24261054148232805f, 0.24261054148232805f));
  q = ffma2(q, fr, f2(0.6932609855869492f, 0.6932609855869492f));
  q = ffma2(q, fr, f2(0.9999281094135103f, 0.9999281094135103f));
  float t0, t1, q0, q1;
  f2split(t, t0, t1);
  f2split(q, q0, q1);
  p0 = __uint_as_float((__float_as_uint(t0) << 23) + __float_as_uint(q0));
  p1 = __uint_as_float((__float_as_uint(t1) << 23) + __float_as_uint(q1));
}
// Exponentials moved from the MUFU to the FMA pipe (ex2_emu2): pairs with index
// % K == K - 1, per pass (0: none).  Measured (x_probe A/B, per SGD step):
// pass 1 K = 3 / 4 / 6 / none: 0.274 / 0.270 / 0.270 / 0.287 ms; pass 2
// 0.375 / 0.366 / 0.362 / 0.360 ms -- pass 1 (online max, fewer other FMA-pipe
// instructions) wants some offload, pass 2 (db2 sums, label term) none.
// tools/ubench_softmax.cu: the bare mix runs faster all-MUFU at every warp
// count (MUFU.EX2 ~32 lanes/clk/SM with independent chains).
#ifndef AS_EMU_P1
#define AS_EMU_P1 6
#endif
#ifndef AS_EMU_P2
#define AS_EMU_P2 0
#endif
#define AS_EMU_AT(K, u) ((K) > 0 && (u) % ((K) > 0 ? (K) : 1) == (K) - 1)
#ifndef AS_EMU_MOD
#define AS_EMU_MOD 3    // (legacy single knob, unused by the passes)
#endif
// Experiment switches (scripts/x_probe.sh builds; never set in the product
// library): AS_X_NOEXP replaces ex2 by a move, AS_X_NOSOFT skips the softmax
// TMEM work, AS_X_NOMMA1 / AS_X_NOMMA2 skip the first / second GEMM of a pass,
// AS_X_NOTMA reuses the first operand stages, AS_X_NOUPD skips pass 2's SGD.
// Mutants for the parity tests' sensitivity (must FAIL them): AS_X_P1NOO zeroes
// pass 1's P operand of the O MMA (O = 0), AS_X_P2NOSOFT drops the softmax
// term from pass 2's G (only the label term remains).
#ifdef AS_X_NOEXP
#define XEX2(v) (v)
#else
#define XEX2(v) ex2(v)
#endif
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
// K-major tile of 16 bf16 per row with 32-byte swizzle (SWIZZLE_32B = 6): one
// K-step; 8-row groups 256 B apart (SBO).  Written by TMA (SWIZZLE_32B box) or
// by threads with the same pattern: 16-B chunk c of row r at
// r * 32 + ((c ^ ((r >> 2) & 1)) << 4).
__device__ __forceinline__ uint64_t sdesc32(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | (1ull << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46) |
         (6ull << 61);
}
__device__ __forceinline__ uint32_t swz32(int r, int c) {
  return (uint32_t)(r * 32 + ((c ^ ((r >> 2) & 1)) << 4));
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
#ifdef AS_X_P1NST
  static constexpr int NST = H == 128 ? AS_X_P1NST : 2;   // experiment: W stages
#else
  static constexpr int NST = H == 128 ? 4 : 2;    // W stages
#endif
  static constexpr int TILE = BM * H * 2;         // bytes of a 128 x H bf16 tile
  static constexpr int THREADS = 12 * 32;        // 3 warpgroups (setmaxnreg granularity)
  // P1WB2: every softmax warp keeps its own copy of the block's b2 (loaded as
  // float4 by its lanes) and reduces the block max itself, so the warps of a
  // warpgroup never meet at a named barrier (default: one copy per WG, named
  // barrier per block)
  // Measured neutral (out_fwd 0.2694 vs 0.2676 ms, two x_probe A/B pairs):
  // experiment switch AS_X_P1WB2, off in the product build.
#ifdef AS_X_P1WB2
  static constexpr bool P1WB2 = H == 128;
#else
  static constexpr bool P1WB2 = false;
#endif
  static constexpr int NB2 = P1WB2 ? 8 * 2 : 2 * 2;  // b2 copies [warp or WG][2]
  // P1SP (h = 128): P goes to shared memory (K-major SW128, one 32 KB buffer per
  // WG) and the O MMA reads it from there (SS) instead of from TMEM.  TMEM ->
  // register and MMA TMEM-operand reads share 64 B/clk/SM: per class block the
  // softmax reads S (64 KB) and a TS O MMA read P (32 KB) -- 1 536 cycles against
  // 1 024 of MMA; with P in shared memory 1 024.  Measured slower (out_fwd
  // 0.268-0.283 -> 0.298-0.303 ms, parity green): the O MMA's A operand then
  // comes through shared memory, which already carries the H, W tiles of both
  // MMAs (128 B/clk/SM), plus the softmax's P stores.  Experiment switch AS_X_P1SP.
#if defined(AS_X_P1SP) && !defined(AS_X_P1RING) && !defined(AS_X_P1Q)
  static constexpr bool P1SP = H == 128;
#else
  static constexpr bool P1SP = false;
#endif
  static constexpr int PSM = P1SP ? 2 * BM * BM * 2 : 0;   // P buffers [WG][2 atoms][128 rows][64]
  // P1RING (h = 128): S_j is computed in two 64-class halves whose TMEM columns
  // alternate with the WG's block parity p: half 0 at 64 p, half 1 at 64 (1 - p)
  // of the WG's 128 columns, P_j (bf16) packed at 64 p + 32 half.  Half 0 of
  // the WG's next block goes into the columns of this block's half 1 as soon
  // as the softmax has loaded them, so the softmax of the next block starts
  // while this block's O MMAs and the next half 1 are still on the tensor pipe.
  // Online softmax per 64-class half.  Measured slower (out_fwd 0.273 ->
  // 0.299 ms, parity green): with the S^T waits gone both softmax warps of a
  // sub-partition run at once and each runs slower, as with pass 2's ring.
  // Experiment switch AS_X_P1RING.
#if defined(AS_X_P1RING) && !defined(AS_X_NOSOFT)
  static constexpr bool P1RING = H == 128 && !P1WB2;
#else
  static constexpr bool P1RING = false;
#endif
  static constexpr int SMEM = TILE /*H*/ + NST * TILE + PSM + NB2 * BM * 4 /*b2*/ + 64 /*b2 max*/ + 256;
  static_assert(SMEM <= 232448, "pass-1 shared memory exceeds 227 KB");
  static_assert(H == 128 || H == 256, "h");
};

// splits of the class range for pass 1 given the batch rows (same formula on
// the host for the combine).  Every CTA writes 2 partial slots (one per WG).
__host__ __device__ inline int fwd_splits(int B, int n_cblocks, int num_ctas, int max_splits) {
  const int RT = (B + BM - 1) / BM;
  int s = num_ctas / (RT > 0 ? RT : 1);
  if (s > n_cblocks) s = n_cblocks;
  if (s > max_splits) s = max_splits;
  return s < 1 ? 1 : s;
}

// =====================================================================
// pass 1 (v3: ping-pong warpgroups)
//   warps 0-7  softmax: WG g handles the class blocks j with j % 2 == g of this
//              CTA's range, with its own online-softmax state (log2 units, lazy
//              rescale) and its own O accumulator; thread = row = TMEM lane.
//              P is written back into TMEM over the S it came from.
//   warp 8     TMA producer (H tile once, W2T class blocks)
//   warp 9     MMA issuer + TMEM owner:
//                S_j   = H . W2T_blk^T        (SS, TMEM buffer j % 2)
//                O_g  += P_j . W2T_blk        (A = P from TMEM, B MN-major)
// TMEM: S[2] at columns 0, 128; O[2] at 256, 384 (h = 128; h = 256 uses one
// WG and O at 256..511).  One partial slot per CTA split: WG 1 hands its state to WG 0 in the epilogue.
// =====================================================================
template <int H>
__global__ void __launch_bounds__(FwdCfg<H>::THREADS, 1)
    k_out_fwd(const __grid_constant__ CUtensorMap mapH, const __grid_constant__ CUtensorMap mapW,
              const StepDesc *__restrict__ desc, const __nv_bfloat16 *__restrict__ Hb,
              const float *__restrict__ b2, int C, int n_cblocks, int max_splits, int bpad,
              float *__restrict__ pm, float *__restrict__ pl, float *__restrict__ pO, LtArgs lt) {
  griddep_wait();
  using Cfg = FwdCfg<H>;
  constexpr int NST = Cfg::NST, TILE = Cfg::TILE;
  constexpr int NWG = H == 128 ? 2 : 1;             // softmax warpgroups (O accumulators)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *sH = smem_raw;
  uint8_t *sW = smem_raw + TILE;
  uint8_t *sP = sW + NST * TILE;                     // P1SP: P of each WG (K-major SW128)
  constexpr bool P1SP = Cfg::P1SP;
  float *sB2 = (float *)(sP + Cfg::PSM);            // [2 WG][2][128]
  float *sBmax = sB2 + FwdCfg<H>::NB2 * BM;         // [2 WG][2][4 warps] block max of b2
  uint64_t *bars = (uint64_t *)(sBmax + 16);
  // p_full[2 b + half]: P of classes [64 half, 64 half + 64) of the block in S
  // buffer b is in TMEM; the O MMA of that half starts without the other
#ifdef AS_X_P1Q
  constexpr int PQ = 4;                             // P signalled per 32-class quarter
#else
  constexpr int PQ = 2;                             // P signalled per 64-class half
#endif
  uint64_t *h_full = bars, *w_full = bars + 1, *w_empty = w_full + NST, *s_full = w_empty + NST,
           *p_full = s_full + 2, *o_fin = p_full + 2 * PQ, *o_done = o_fin + 1;
  constexpr bool P1RING = Cfg::P1RING;
  // P1RING: s_full per (buffer, half) [4], s_free per buffer [2], o_half per WG [2]
  uint64_t *s_full2 = o_done + 1, *s_free = s_full2 + 4, *o_half = s_free + 2;
  uint32_t *tmem_slot = (uint32_t *)(o_half + 2);
  if ((smem_u32(smem_raw) & 1023u) != 0) __trap();

  const int B = desc->rows;
  const int RT = (B + BM - 1) / BM;
  const int splits = fwd_splits(B, n_cblocks, gridDim.x, max_splits);
  const int rt = blockIdx.x / splits, sp = blockIdx.x % splits;
  if (rt >= RT) return;
  (void)sp;                                   // the role branches recompute cb0 / nloc
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kProdWarp = 10, kMmaWarp = 11;  // highest ids: scheduler priority; 8-9 idle

  if (threadIdx.x == 0) {
    mbar_init(h_full, 1);
    for (int i = 0; i < NST; ++i) { mbar_init(&w_full[i], 1); mbar_init(&w_empty[i], 1); }
    for (int i = 0; i < 2; ++i) mbar_init(&s_full[i], 1);
    for (int i = 0; i < 2 * PQ; ++i) mbar_init(&p_full[i], 4);
    mbar_init(o_fin, 1);
    mbar_init(o_done, 1);
    for (int i = 0; i < 4; ++i) mbar_init(&s_full2[i], 1);
    for (int i = 0; i < 2; ++i) { mbar_init(&s_free[i], 4); mbar_init(&o_half[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) tmem_alloc(tmem_slot, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  // registers: the launch gives every warp 168 (3 warps per SM sub-partition);
  // warpgroup 2 (producer, MMA, 2 idle warps) hands its share to the softmax
  // warpgroups, which keep a whole 128-column S row in registers.  Each role
  // branch adjusts its own budget (setmaxnreg is warpgroup-collective).
#define AS_REG_DEC() asm volatile("setmaxnreg.dec.sync.aligned.u32 40;" ::: "memory")
#define AS_REG_INC() asm volatile("setmaxnreg.inc.sync.aligned.u32 232;" ::: "memory")

  if (warp == kProdWarp) {
    AS_REG_DEC();
    // split range recomputed after setmaxnreg from an opaque copy (the
    // compiler otherwise spills the prologue's values across the role switch)
    int ncq_ = n_cblocks;
    asm volatile("" : "+r"(ncq_));
    const int splits_ = fwd_splits(B, ncq_, gridDim.x, max_splits);
    const int cb0 = (int)((long long)(blockIdx.x % splits_) * ncq_ / splits_);
    const int nloc = (int)((long long)(blockIdx.x % splits_ + 1) * ncq_ / splits_) - cb0;
    if (lane == 0) {  // ---------------- TMA producer
      mbar_expect_tx(h_full, TILE);
      for (int a = 0; a < H / 64; ++a) tma_load_2d(&mapH, h_full, sH + a * ATOM_BYTES, a * 64, rt * BM);
      for (int j = 0; j < nloc; ++j) {
        const int st = j % NST;
        if (j >= NST) mbar_wait_idle(&w_empty[st], ((j / NST) - 1) & 1);
#ifdef AS_X_NOTMA
        if (j >= NST) { mbar_arrive(&w_full[st]); continue; }
#endif
        mbar_expect_tx(&w_full[st], TILE);
        for (int a = 0; a < H / 64; ++a)
          tma_load_2d(&mapW, &w_full[st], sW + st * TILE + a * ATOM_BYTES, a * 64, (cb0 + j) * BM);
      }
    }
  } else if (warp == kMmaWarp) {
    AS_REG_DEC();
    // split range recomputed after setmaxnreg from an opaque copy (the
    // compiler otherwise spills the prologue's values across the role switch)
    int ncq_ = n_cblocks;
    asm volatile("" : "+r"(ncq_));
    const int splits_ = fwd_splits(B, ncq_, gridDim.x, max_splits);
    const int cb0 = (int)((long long)(blockIdx.x % splits_) * ncq_ / splits_);
    const int nloc = (int)((long long)(blockIdx.x % splits_ + 1) * ncq_ / splits_) - cb0;
    {  // ---------------- MMA issuer (warp-converged; one elected lane issues)
      constexpr uint32_t idS = idesc_bf16(BM, BM, 0, 0);
      constexpr uint32_t idO = idesc_bf16(BM, H, 0, 1);
      const uint32_t aH = smem_u32(sH), aW = smem_u32(sW);
      mbar_wait(h_full, 0);
      fence_after();
      const uint64_t dH = sdesc(aH, 16, 1024);
      auto issue_S = [&](int j) {
        const int st = j % NST, b = j & 1;
        mbar_wait(&w_full[st], (j / NST) & 1);
        fence_after();
        // S_j overwrites buffer b; O of block j-2 (the last reader of P_{j-2}
        // there) was issued earlier by this warp: tcgen05.mma executes in order.
#ifndef AS_X_NOMMA1
        if constexpr (H == 128)
          mma_grp_ss_kk_8(tmem + b * BM, dH, sdesc(aW + st * TILE, 16, 1024), idS, 0u);
        else
          mma_grp_ss_kk_16(tmem + b * BM, dH, sdesc(aW + st * TILE, 16, 1024), idS, 0u);
#endif
        mma_commit_w(&s_full[b]);
      };
      if constexpr (P1RING) {
        constexpr uint32_t idS64 = idesc_bf16(BM, 64, 0, 0);
        // S_j half h (classes [64 h, 64 h + 64) of W tile j) into 64 ((h + p_j) & 1)
        auto issue_S_half = [&](int j, int h) {
          const int st = j % NST, b = j & 1;
          const uint32_t p = (uint32_t)((j >> 1) & 1);
          if (h == 0) mbar_wait(&w_full[st], (j / NST) & 1);
          fence_after();
#ifndef AS_X_NOMMA1
          mma_grp_ss_kk_8(tmem + b * BM + (((uint32_t)h + p) & 1u) * 64u, dH,
                          sdesc(aW + st * TILE + h * 64 * 128, 16, 1024), idS64, 0u);
#endif
          mma_commit_w(&s_full2[2 * b + h]);
        };
        for (int j = 0; j < nloc && j < 2; ++j) { issue_S_half(j, 0); issue_S_half(j, 1); }
        for (int j = 0; j < nloc; ++j) {
          const int st = j % NST, b = j & 1;
          const uint32_t ph = (uint32_t)((j >> 1) & 1);
          const uint32_t pcol = b * BM + ph * 64u;      // P_j (bf16): 64 p + 32 half
          mbar_wait(&p_full[PQ * b], ph);
          fence_after();
#ifndef AS_X_NOMMA2
          mma_grp_ts_mn_4(tmem + 2 * BM + b * BM, tmem + pcol, sdesc(aW + st * TILE, ATOM_BYTES, 1024), idO,
                          j >= NWG ? 1u : 0u);
#endif
          mma_commit_w(&o_half[b]);           // O of this WG up to half 0 (a rescale at half 1 waits)
          if (j + 2 < nloc) {                 // next half 0 into the columns half 1 has left
            mbar_wait(&s_free[b], ph);
            issue_S_half(j + 2, 0);
          }
          mbar_wait(&p_full[PQ * b + 1], ph);
          fence_after();
#ifndef AS_X_NOMMA2
          mma_grp_ts_mn_4(tmem + 2 * BM + b * BM, tmem + pcol + 32, sdesc(aW + st * TILE + 64 * 128, ATOM_BYTES, 1024),
                          idO, 1u);
#endif
          mma_commit_w(&w_empty[st]);
          if (j + 2 < nloc) issue_S_half(j + 2, 1);   // into P_j's columns: after its O (in order)
        }
        mma_commit_w(o_fin);
      } else {
      if (nloc > 0) issue_S(0);
      if (nloc > 1) issue_S(1);
      for (int j = 0; j < nloc; ++j) {
        const int st = j % NST, b = j & 1;
        const int g = NWG == 2 ? b : 0;
        // the O MMA part by part (64 or 32 classes of P) as the softmax finishes them
#pragma unroll
        for (int pq = 0; pq < PQ; ++pq) {
          mbar_wait(&p_full[PQ * b + pq], (j >> 1) & 1);
          fence_after();
#ifndef AS_X_NOMMA2
          if constexpr (P1SP)
            mma_grp_ss_kmn_4(tmem + 2 * BM + g * BM,
                             sdesc(smem_u32(sP) + g * (BM * BM * 2) + pq * ATOM_BYTES, 16, 1024),
                             sdesc(aW + st * TILE + pq * 64 * 128, ATOM_BYTES, 1024), idO,
                             (j >= NWG || pq > 0) ? 1u : 0u);
          else if constexpr (PQ == 2)
            mma_grp_ts_mn_4(tmem + 2 * BM + g * BM, tmem + b * BM + 32 * pq,
                            sdesc(aW + st * TILE + pq * 64 * 128, ATOM_BYTES, 1024), idO,
                            (j >= NWG || pq > 0) ? 1u : 0u);
          else
            mma_grp_ts_mn_2(tmem + 2 * BM + g * BM, tmem + b * BM + 16 * pq,
                            sdesc(aW + st * TILE + pq * 32 * 128, ATOM_BYTES, 1024), idO,
                            (j >= NWG || pq > 0) ? 1u : 0u);
#endif
        }
        mma_commit_w(&w_empty[st]);
        if (NWG == 1) mma_commit_w(o_done);     // single WG: O_{j} before the rescale at j+1
        if (j + 2 < nloc) issue_S(j + 2);
      }
      mma_commit_w(o_fin);
      }
    }
  } else if (warp < 4 * NWG) {  // ---------------- softmax warpgroups (thread = row)
    AS_REG_INC();
    // split range recomputed after setmaxnreg from an opaque copy (the
    // compiler otherwise spills the prologue's values across the role switch)
    int ncq_ = n_cblocks;
    asm volatile("" : "+r"(ncq_));
    const int splits_ = fwd_splits(B, ncq_, gridDim.x, max_splits);
    const int cb0 = (int)((long long)(blockIdx.x % splits_) * ncq_ / splits_);
    const int nloc = (int)((long long)(blockIdx.x % splits_ + 1) * ncq_ / splits_) - cb0;
    const int g = warp >> 2;
    const int q = warp & 3;
    const int row = q * 32 + lane;            // TMEM lane == tile row == loader index
    const uint32_t tlq = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t tO = tlq + 2 * BM + g * BM;
    float m_used = -FLT_MAX, l = 0.f;
    // prefetched b2 of this WG's next class block: an unconditional load from
    // a clamped address whose register is first touched one block later (a
    // select / multiply right after the load would stall on its latency)
    float b2raw = 0.f;
    bool b2ok = false;
    float4 b2q = make_float4(0.f, 0.f, 0.f, 0.f);   // P1WB2: classes 4 lane .. 4 lane + 3 of the next block
    auto ld_b2q = [&](int jb) {
      const int c = (cb0 + jb) * BM + 4 * lane;
      if (c + 3 < C) {
        b2q = *reinterpret_cast<const float4 *>(b2 + c);
      } else {                                // tail of the class range: clamped scalar loads
        b2q.x = b2[c < C ? c : C - 1];
        b2q.y = b2[c + 1 < C ? c + 1 : C - 1];
        b2q.z = b2[c + 2 < C ? c + 2 : C - 1];
        b2q.w = b2[c + 3 < C ? c + 3 : C - 1];
      }
    };
    if (g < nloc) {
      if constexpr (FwdCfg<H>::P1WB2) ld_b2q(g);
      else { const int c = (cb0 + g) * BM + row; b2ok = c < C; b2raw = b2[b2ok ? c : 0]; }
    }
    int jj = 0;                               // blocks processed by this WG
    for (int j = g; j < nloc; j += NWG, ++jj) {
      const int b = j & 1;
      float *myB2;
      float bmax;
      if constexpr (FwdCfg<H>::P1WB2) {
        myB2 = sB2 + (warp * 2 + (jj & 1)) * BM;
        const int c = (cb0 + j) * BM + 4 * lane;
        const float4 bn = make_float4(c < C ? b2q.x * LOG2E : -INFINITY, c + 1 < C ? b2q.y * LOG2E : -INFINITY,
                                      c + 2 < C ? b2q.z * LOG2E : -INFINITY, c + 3 < C ? b2q.w * LOG2E : -INFINITY);
        *reinterpret_cast<float4 *>(myB2 + 4 * lane) = bn;
        float wm = fmaxf(fmaxf(bn.x, bn.y), fmaxf(bn.z, bn.w));   // max of b2 (log2 units) over the block
#pragma unroll
        for (int o = 16; o; o >>= 1) wm = fmaxf(wm, __shfl_xor_sync(0xffffffffu, wm, o));
        bmax = wm;
        if (j + NWG < nloc) ld_b2q(j + NWG);
        __syncwarp();
      } else {
        myB2 = sB2 + (g * 2 + (jj & 1)) * BM;
        const float b2n = b2ok ? b2raw * LOG2E : -INFINITY;
        myB2[row] = b2n;
        float wm = b2n;                         // max of b2 (log2 units) over the block
#pragma unroll
        for (int o = 16; o; o >>= 1) wm = fmaxf(wm, __shfl_xor_sync(0xffffffffu, wm, o));
        if (lane == 0) sBmax[(g * 2 + (jj & 1)) * 4 + q] = wm;
        if (j + NWG < nloc) {
          const int c = (cb0 + j + NWG) * BM + row;
          b2ok = c < C;
          b2raw = b2[b2ok ? c : 0];
        }
        named_bar(1 + g, 128);
        const float *bmx = sBmax + (g * 2 + (jj & 1)) * 4;
        bmax = fmaxf(fmaxf(bmx[0], bmx[1]), fmaxf(bmx[2], bmx[3]));
      }
#ifndef AS_X_NOSOFT
      if constexpr (P1RING) {
        // two 64-class halves, each with its own lazy-rescale check (online
        // softmax per half); the b2 maxima of the halves from the warps' partials
        const uint32_t par = (uint32_t)((j >> 1) & 1);
        const float *bmx = sBmax + (g * 2 + (jj & 1)) * 4;
        const float bmh0 = fmaxf(bmx[0], bmx[1]), bmh1 = fmaxf(bmx[2], bmx[3]);
        uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
        const uint64_t l2e2 = f2(LOG2E, LOG2E);
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          mbar_wait(&s_full2[2 * b + h], par);
          fence_after();
          uint32_t r[64];
          const uint32_t tS = tlq + b * BM + (((uint32_t)h + par) & 1u) * 64u;
          AS_TMEM_LD32(tS, r);
          AS_TMEM_LD32(tS + 32, (r + 32));
          AS_TMEM_WAIT_LD(r);
          AS_TMEM_WAIT_LD((r + 32));
          if (h == 1) {                       // half 1's columns free for the next block's half 0
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_free[b]);
          }
          float mt[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) mt[k] = __uint_as_float(r[k]);
#pragma unroll
          for (int k = 8; k < 64; ++k) mt[k & 7] = fmaxf(mt[k & 7], __uint_as_float(r[k]));
          const float mx = fmaf(fmaxf(fmaxf(fmaxf(mt[0], mt[1]), fmaxf(mt[2], mt[3])),
                                      fmaxf(fmaxf(mt[4], mt[5]), fmaxf(mt[6], mt[7]))),
                                LOG2E, h ? bmh1 : bmh0);
          float m_new = m_used;
          if (mx > m_used + 8.f) m_new = mx;  // lazy rescale: p <= 2^8 otherwise
          const bool need = m_new != m_used;
          const float sc = need ? ((m_used == -FLT_MAX) ? 0.f : ex2(m_used - m_new)) : 1.f;
          l *= sc;
          m_used = m_new;
          if ((jj > 0 || h == 1) && __any_sync(0xffffffffu, need)) {
            // O must be quiescent: half 0 -- S_j half 1 was issued after this WG's
            // last O MMA (of block j - 2); half 1 -- O_j's half-0 MMA (o_half)
            if (h == 0) mbar_wait(&s_full2[2 * b + 1], par);
            else mbar_wait(&o_half[b], (uint32_t)(jj & 1));
            fence_after();
#pragma unroll 1
            for (int ch = 0; ch < H / 32; ++ch) {
              uint32_t ro[32];
              AS_TMEM_LD32(tO + ch * 32, ro);
              AS_TMEM_WAIT_LD(ro);
#pragma unroll
              for (int k = 0; k < 32; ++k) ro[k] = __float_as_uint(__uint_as_float(ro[k]) * sc);
              AS_TMEM_ST32(tO + ch * 32, ro);
            }
          }
          const uint64_t negm2 = f2(-m_new, -m_new);
          const float *bh = myB2 + 64 * h;
          uint32_t pk[32];
#pragma unroll
          for (int u = 0; u < 32; ++u) {
            const int k = 2 * u;
            const float2 bv = *reinterpret_cast<const float2 *>(bh + k);
            uint64_t x = ffma2(f2(__uint_as_float(r[k]), __uint_as_float(r[k + 1])), l2e2, f2(bv.x, bv.y));
            x = fadd2(x, negm2);
            float p0, p1;
            if (AS_EMU_AT(AS_EMU_P1, u)) {
              ex2_emu2(x, p0, p1);
            } else {
              float x0, x1;
              f2split(x, x0, x1);
              p0 = XEX2(x0); p1 = XEX2(x1);
            }
            acc[u & 3] = fadd2(acc[u & 3], f2(p0, p1));
            pk[u] = pack_bf16x2(p0, p1);
#ifdef AS_X_P1NOO
            pk[u] = 0u;                        // mutant: O = 0 (parity tests must fail)
#endif
          }
          AS_TMEM_ST32(tlq + b * BM + par * 64u + 32u * (uint32_t)h, pk);
          tmem_wait_st();
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_full[PQ * b + h]);
        }
        acc[0] = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
        float s0, s1;
        f2split(acc[0], s0, s1);
        l += s0 + s1;
        continue;
      }
#endif
      // s_full(j) also implies that the O MMA of this WG's previous block (issued
      // before S_j) completed: O is stable and the P region of buffer b is free.
      mbar_wait(&s_full[b], (j >> 1) & 1);
      fence_after();
      const uint32_t tS = tlq + b * BM;
      const float *bb = myB2;
#ifndef AS_X_NOSOFT
      // the whole S row of this block in registers (one TMEM read)
      uint32_t r[BM];
#pragma unroll
      for (int ch = 0; ch < BM / 32; ++ch) AS_TMEM_LD32(tS + ch * 32, (r + ch * 32));
#pragma unroll
      for (int ch = 0; ch < BM / 32; ++ch) AS_TMEM_WAIT_LD((r + ch * 32));
      // reference value for the exponentials: max_k(s_k) log2e + max_k(b2_k) is an
      // upper bound of the block max of s_k log2e + b2_k (exact when b2 is flat;
      // only the scaling of the partial sums depends on it, R-readings DESIGN 3)
      float mt[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) mt[k] = __uint_as_float(r[k]);
#pragma unroll
      for (int k = 8; k < BM; ++k) mt[k & 7] = fmaxf(mt[k & 7], __uint_as_float(r[k]));
      const float mx = fmaf(fmaxf(fmaxf(fmaxf(mt[0], mt[1]), fmaxf(mt[2], mt[3])),
                                  fmaxf(fmaxf(mt[4], mt[5]), fmaxf(mt[6], mt[7]))),
                            LOG2E, bmax);
      float m_new = m_used;
      if (mx > m_used + 8.f) m_new = mx;   // lazy rescale: p <= 2^8 otherwise
      if (NWG == 1 && jj > 0) {               // single WG: O of block j-1 must be done
        mbar_wait(o_done, (jj - 1) & 1);
        fence_after();
      }
      // lazy rescale (per row); tcgen05.ld/st are warp-collective, so the TMEM
      // pass runs for the whole warp when any of its rows needs it (sc = 1 else)
      const bool need = m_new != m_used;
      const float sc = need ? ((m_used == -FLT_MAX) ? 0.f : ex2(m_used - m_new)) : 1.f;
      l *= sc;
      m_used = m_new;
      if (jj > 0 && __any_sync(0xffffffffu, need)) {
#pragma unroll 1
        for (int ch = 0; ch < H / 32; ++ch) {
          uint32_t ro[32];
          AS_TMEM_LD32(tO + ch * 32, ro);
          AS_TMEM_WAIT_LD(ro);
#pragma unroll
          for (int k = 0; k < 32; ++k) ro[k] = __float_as_uint(__uint_as_float(ro[k]) * sc);
          AS_TMEM_ST32(tO + ch * 32, ro);
        }
      }
      // P = 2^(s log2e + b2 - m) with packed fp32x2 FMA/ADD, bf16 pairs written
      // over S (chunk ch -> columns [16ch, 16ch + 16), all of S already read)
      const uint64_t l2e2 = f2(LOG2E, LOG2E), negm2 = f2(-m_new, -m_new);
      uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
      for (int ch = 0; ch < BM / 32; ++ch) {
        uint32_t pk[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int k = ch * 32 + 2 * u;
          const float2 bv = *reinterpret_cast<const float2 *>(bb + k);
          uint64_t x = ffma2(f2(__uint_as_float(r[k]), __uint_as_float(r[k + 1])), l2e2, f2(bv.x, bv.y));
          x = fadd2(x, negm2);
          float p0, p1;
          if (AS_EMU_AT(AS_EMU_P1, u)) {
            ex2_emu2(x, p0, p1);
          } else {
            float x0, x1;
            f2split(x, x0, x1);
            p0 = XEX2(x0); p1 = XEX2(x1);
          }
          acc[u & 3] = fadd2(acc[u & 3], f2(p0, p1));
          pk[u] = pack_bf16x2(p0, p1);
#ifdef AS_X_P1NOO
          pk[u] = 0u;                          // mutant: O = 0 (parity tests must fail)
#endif
        }
        if constexpr (P1SP) {
          // classes [32 ch, 32 ch + 32) of row `row`: four 16-byte chunks of atom ch / 2
          uint8_t *prow = sP + g * (BM * BM * 2) + (ch >> 1) * ATOM_BYTES + row * 128;
          const uint32_t sw = (uint32_t)(row & 7);
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const uint32_t jc = (uint32_t)((ch & 1) * 4 + q4);
            *reinterpret_cast<uint4 *>(prow + ((jc ^ sw) << 4)) =
                make_uint4(pk[4 * q4], pk[4 * q4 + 1], pk[4 * q4 + 2], pk[4 * q4 + 3]);
          }
        } else {
          AS_TMEM_ST16(tS + ch * 16, pk);
        }
        if (PQ == 4 || (ch & 1)) {             // this part of P is in TMEM / shared memory
          if constexpr (P1SP) fence_proxy_async();   // generic-proxy writes -> the MMA's async proxy
          else tmem_wait_st();
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_full[PQ * b + (PQ == 4 ? ch : (ch >> 1))]);
        }
      }
      acc[0] = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
      float s0, s1;
      f2split(acc[0], s0, s1);
      l += s0 + s1;
#else
      fence_before();
      __syncwarp();
      if (lane == 0)
        for (int pq = 0; pq < PQ; ++pq) mbar_arrive(&p_full[PQ * b + pq]);
#endif
    }
    // epilogue: ONE partial slot per CTA split.  With two warpgroups, WG 1
    // stages its (m, l, O) in the (now idle) W ring and WG 0 merges the two
    // online-softmax states before writing: half the partial traffic and
    // half the combine work of one slot per warpgroup.
    const int grow = rt * BM + row;
    const size_t slot = (size_t)sp;
    float *sO = reinterpret_cast<float *>(sW);          // [H][128] O of WG 1 (column-major: conflict-free)
    float *sML = sO + H * BM;                           // [2][128] m, l of WG 1
    if (NWG == 2 && g == 1) {
      if (jj > 0) {
        mbar_wait(o_fin, 0);
        fence_after();
#pragma unroll 1
        for (int ch = 0; ch < H / 32; ++ch) {
          uint32_t r[32];
          AS_TMEM_LD32(tO + ch * 32, r);
          AS_TMEM_WAIT_LD(r);
#pragma unroll
          for (int k = 0; k < 32; ++k) sO[(ch * 32 + k) * BM + row] = __uint_as_float(r[k]);
        }
      }
      sML[row] = jj > 0 ? m_used : -FLT_MAX;
      sML[BM + row] = jj > 0 ? l : 0.f;
    }
    if (NWG == 2) named_bar(4, 256);
    if (g == 0) {
      float m1 = -FLT_MAX, l1 = 0.f;
      if (NWG == 2) { m1 = sML[row]; l1 = sML[BM + row]; }
      const float m0 = jj > 0 ? m_used : -FLT_MAX;
      const float M = fmaxf(m0, m1);
      const float s0 = m0 == -FLT_MAX ? 0.f : ex2(m0 - M);
      const float s1 = m1 == -FLT_MAX ? 0.f : ex2(m1 - M);
      if (jj > 0) {
        mbar_wait(o_fin, 0);
        fence_after();
      }
#pragma unroll 1
      for (int ch = 0; ch < H / 32; ++ch) {
        uint32_t r[32];
        if (jj > 0) {
          AS_TMEM_LD32(tO + ch * 32, r);
          AS_TMEM_WAIT_LD(r);
        } else {
#pragma unroll
          for (int k = 0; k < 32; ++k) r[k] = 0u;
        }
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          float o = __uint_as_float(r[k]) * s0;
          if (NWG == 2 && s1 != 0.f) o = fmaf(sO[(ch * 32 + k) * BM + row], s1, o);
          pO[(slot * H + ch * 32 + k) * bpad + grow] = o;
        }
      }
      pm[slot * bpad + grow] = M;
      pl[slot * bpad + grow] = l * s0 + l1 * s1;
    }
  } else {
    // warps 8-9 (h = 256 also the idle second warpgroup, warps 4-7): the label
    // terms (a5, R3) alongside
    if (NWG == 1 && warp < 8) AS_REG_INC();
    else AS_REG_DEC();
    constexpr int NLW = NWG == 1 ? 6 : 2;     // label warps per CTA
    const int lwi = warp >= 8 ? warp - 8 : warp - 4 + 2;
    // zsum_r = (1/k_r) sum_{y in Y_r} z_ry and labW_r = (1/k_r) sum_y W2T[y]
    // (fp32 master weights, pre-update) for rows r = gw, gw + GW, ... (warp per
    // row, labels in order, lane = 4 consecutive of the h columns); they need
    // only H and W2T, so they hide in pass 1 and the combine reads them after
    if (lt.zsum) {
      constexpr int V = H / 128;
      const int gw = (int)blockIdx.x * NLW + lwi, GW = RT * splits * NLW;
      for (int r = gw; r < B; r += GW) {
        const int64_t s0 = lt.lab_ptr[r], s1 = lt.lab_ptr[r + 1];
        const float inv_k = 1.0f / (float)(s1 - s0);
        float4 hr[V], lw[V];
#pragma unroll
        for (int q = 0; q < V; ++q) {
          hr[q] = reinterpret_cast<const float4 *>(lt.Hf + (size_t)r * H)[lane + 32 * q];
          lw[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        float zs = 0.f;
        for (int64_t j = s0; j < s1; ++j) {
          const int y = lt.lab[j];
          const float bb = lt.b2[y];
          float d = 0.f;
#pragma unroll
          for (int q = 0; q < V; ++q) {
            const float4 w = reinterpret_cast<const float4 *>(lt.W2T + (size_t)y * H)[lane + 32 * q];
            d = fmaf(hr[q].x, w.x, fmaf(hr[q].y, w.y, fmaf(hr[q].z, w.z, fmaf(hr[q].w, w.w, d))));
            lw[q].x += w.x; lw[q].y += w.y; lw[q].z += w.z; lw[q].w += w.w;
          }
          zs += warp_sum(d) + bb;
        }
        if (lane == 0) lt.zsum[r] = zs * inv_k;
#pragma unroll
        for (int q = 0; q < V; ++q) {
          float4 o = lw[q];
          o.x *= inv_k; o.y *= inv_k; o.z *= inv_k; o.w *= inv_k;
          reinterpret_cast<float4 *>(lt.labW + (size_t)r * H)[lane + 32 * q] = o;
        }
      }
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == kMmaWarp) tmem_dealloc(tmem, 512);
}

template <int H, bool ONEB = false>
struct BwdCfg {
  // W2S (h = 256, one class block per CTA: C <= 128 SMs, AmazonCat-13K): the bf16
  // W2T block is TMA-loaded into shared memory once and the S^T MMA reads it
  // from there (SS), which frees its 128 TMEM columns for two more S^T buffers
  // (4 x 64 rows: S runs up to two units ahead of each softmax warpgroup); the
  // block's fp32 update goes through the idle H stages (LASTSMEM)
#ifdef AS_X_NOW2S
  static constexpr bool W2S = false;
#else
  static constexpr bool W2S = ONEB && H == 256;
#endif
  // TR64 (W2S): four stages of 64-row H tiles instead of two of 128 rows.  Measured
  // equal (AmazonCat-13K out_bwd 0.0350 vs 0.0355 ms): the S^T waits come from the
  // in-order dW chain across the two WGs, not from the stage count.  Switch AS_X_TR64.
#ifdef AS_X_TR64
  static constexpr bool NOTR64_ = false;
#else
  static constexpr bool NOTR64_ = true;
#endif
  // FOLD (h = 128): b2_c and -(LSE_r + ln B) enter the S^T MMA as one more
  // K-step of 16 (a per-class tile A_ext = [b2 in three bf16 parts, 1, 1, 1, 0..]
  // and a per-row tile B_ext = [1, 1, 1, -(LSE + ln B) in three parts, 0..],
  // both SWIZZLE_32B in shared memory), so S^T = z - LSE - ln B exactly (fp32
  // accumulation of exact bf16 products) and the softmax is p / B = 2^(S log2e):
  // no per-element bias / lse' arithmetic and no lse' loads.
  // Measured (x_probe A/B on B200): numerically exact (GPU parity green) but
  // slower, because its shared memory leaves room for only 3 H stages
  // (out_bwd 0.362 -> 0.409 ms; 3 stages alone cost 0.036 ms) -- an experiment
  // switch (AS_X_FOLD), off in the product build.
#if defined(AS_X_FOLD) && !defined(AS_X_NORING) && !defined(AS_X_U64)
  static constexpr bool FOLD = H == 128;
#else
  static constexpr bool FOLD = false;
#endif
#ifdef AS_X_NSH
  static constexpr int NSH = H == 128 ? AS_X_NSH : 2;   // experiment: H tile stages (>= 3 with the ring)
#else
#ifdef AS_X_HALFUPD
  static constexpr int NSH = H == 128 ? (FOLD ? 4 : 5) : 2;    // H tile stages (128 rows each)
#else
  // W2S (h = 256) with TR64: four stages of 64-row tiles (a stage refills one
  // unit after its dW MMA instead of two); default two 128-row stages
  static constexpr int NSH = H == 128 ? (FOLD ? 3 : 4) : (W2S && !NOTR64_ ? 4 : 2);
#endif
#endif
  static constexpr int HXB = FOLD ? BM * 32 : 0;  // B_ext tile of an H stage (128 rows x 16 bf16)
  static constexpr int AXB = FOLD ? BM * 32 : 0;  // A_ext tile of a class block (two buffers)
#ifdef AS_X_U64
  static constexpr int UNIT = 64;                 // experiment: 64-row units, 4 S^T buffers
  static constexpr int HPT = 128 / UNIT;
  static constexpr int NSB = H == 128 ? 4 : 2;
#else
  static constexpr int UNIT = H == 128 ? 128 : 64; // batch rows per unit = S^T columns per buffer
  static constexpr int TR = (W2S && !NOTR64_) ? 64 : BM;   // rows of an H tile
  static constexpr int HPT = TR / UNIT;           // units per H tile
  static constexpr int NSB = W2S ? 4 : 2;         // S^T unit buffers
#endif
  static constexpr int NWT = H == 128 ? 2 : 1;    // W2T blocks resident in TMEM (A operand)
  static constexpr int WCOLS = H / 2;             // TMEM columns of one W2T block (bf16 pairs)
  static constexpr int WTM = W2S ? 0 : NWT * WCOLS;  // TMEM columns of the W2T blocks
  static constexpr int W2SMEM = W2S ? BM * H * 2 : 0; // shared-memory W2T block (W2S)
  static constexpr int TILE = TR * H * 2;         // bytes of an H tile
  static constexpr int HATOM = TR * 128;          // one 64-column SW128 atom of an H tile
  static constexpr int THREADS = 16 * 32;        // 4 warpgroups (setmaxnreg granularity)
  // h = 128: the fp32 W2T block (4 swizzled 32-column boxes) is TMA-loaded one
  // block ahead, updated in shared memory from the TMEM dW2T accumulator and
  // TMA-stored; the bf16 shadow is written from registers.
  // h = 256: chunked register path through a small staging tile.
  static constexpr bool TMAUPD = H == 128;
  // HALF: the fp32 W2T block is staged 64 columns at a time (32 KB instead of
  // 64 KB of shared memory), leaving room for a deeper H ring.  Measured
  // slower (out_bwd 0.367 -> 0.40 ms with 5 H stages): experiment switch
  // AS_X_HALFUPD, off in the product build.
#ifdef AS_X_HALFUPD
  static constexpr bool HALF = TMAUPD;
#else
  static constexpr bool HALF = false;
#endif
  // PING: the 64 KB staging holds two 64-column half blocks that ping-pong:
  // half h of block kb is updated and TMA-stored from buffer h while the other
  // buffer's store drains / next load lands, and the load of half h of block
  // kb + 1 is issued as soon as buffer h's store has been read -- a full block
  // ahead of its use (one 64 KB buffer serialised store -> load -> update)
  // Measured slower than one 64 KB buffer (out_bwd 0.364 -> 0.373 ms): the
  // update loop's serial latency grows with the extra store / barrier rounds.
  // Experiment switch AS_X_PING.  (Fetching the next block's bf16 rows during
  // the SGD with a 160-register update warpgroup was slower too: 0.374 ms.)
#ifdef AS_X_EARLYREL
  static constexpr bool EARLYREL_ = true;
#else
  static constexpr bool EARLYREL_ = false;
#endif
#if defined(AS_X_PING) && !defined(AS_X_HALFUPD)
  static constexpr bool PING = TMAUPD;
#else
  static constexpr bool PING = false;
#endif
  // LASTSMEM (h = 256): the last class block's fp32 update staged through the
  // then idle H stages by TMA (AS_X_NOLASTSMEM: chunked register path)
#ifdef AS_X_NOLASTSMEM
  static constexpr bool LASTSMEM = false;
#else
  static constexpr bool LASTSMEM = !TMAUPD && NSH * TILE >= BM * H * 4;
#endif
  // ECF (h = 128): the class bias leaves the exponent.  p_rc / B =
  // E_c 2^(s_rc log2e - lse'_r) with E_c = exp(b2_c), so the softmax computes
  // G'_rc = G_rc / E_c (one FFMA2 per pair: s log2e + (-lse')), the label term
  // enters G' as w_r / E_c, db2 = E_c sum_r G'_rc, and the update scales its
  // learning rate per class: W2T_c -= (lr E_c) (G'^T H)_c -- the same G up to
  // the bf16 rounding of G' instead of G (relative, equal size).  Needs
  // |b2| < 80 (E_c, 1 / E_c and p / E_c inside the fp32 range).
  // Experiment switch AS_X_ECF (off in the product build).
#ifdef AS_X_ECF
  static constexpr bool ECF = TMAUPD && !FOLD && !HALF && !PING;
#else
  static constexpr bool ECF = false;             // measured neutral-to-slower (out_bwd +1%): off
#endif
  // REGS3 (h = 128): warpgroup 3 (producer, MMA, dW1 warps) drops to 64
  // registers and the two softmax warpgroups rise to 160 (AS_X_NOREGS3: all 128).
  // Measured with LATEMK: out_bwd 0.375 -> 0.368 ms (two x_probe A/B pairs).
#ifdef AS_X_NOREGS3
  static constexpr bool REGS3 = false;
#else
  static constexpr bool REGS3 = H == 128 && !HALF && !PING && !EARLYREL_;
#endif
  // LATEMK: a unit's label-row bitmap is read after its first half's
  // exponentials (AS_X_NOLATEMK: before the half loop)
#ifdef AS_X_NOLATEMK
  static constexpr bool LATEMK = false;
#else
  static constexpr bool LATEMK = true;
#endif
  // S0POLL (ring): the MMA warp issues the first S^T half of a WG's next unit
  // as soon as that WG has loaded the S^T columns it reuses (s_free), whatever
  // the other WG's progress -- it polls (try_wait with a short suspend) instead
  // of blocking on the other WG's G^T; the dW MMAs stay in unit order
  // (deterministic).  p_full is then indexed by unit mod 4 so that a WG can
  // signal the unit two ahead before the MMA warp has observed this one.
  // Measured slower (out_bwd 0.367 -> 0.400 ms, x_probe A/B): the polling
  // warp takes issue slots from the softmax warps of its sub-partition, and
  // the tensor pipe gains nothing.  Experiment switch AS_X_S0POLL.
#ifdef AS_X_S0POLL
  static constexpr bool S0POLL = UNIT == 128;
#else
  static constexpr bool S0POLL = false;
#endif
  static constexpr int SROW = 36;                 // chunked staging row (floats, 16-B aligned)
  static constexpr int TSTAGE = TMAUPD ? BM * (HALF ? H / 2 : H) * 4 : (W2S ? 0 : BM * SROW * 4);
  static constexpr int SMEM = NSH * TILE + W2SMEM + NSH * HXB + 2 * AXB + TSTAGE +
                              (FOLD ? 1 : 2) * NSH * BM * 4 /*(lse' and) label-weight rings*/ +
                              2 * BM * 4 /*db2*/ + 2 * 256 * (16 + 16 + 4) /*softmax prefetch slots*/ +
                              512 /*barriers*/;
  static_assert(SMEM <= 232448, "pass-2 shared memory exceeds 227 KB");
  static_assert(NSB * UNIT + WTM + H <= 512, "pass-2 TMEM budget");
};

// =====================================================================
// pass 2 (v6: W2T block and G^T in TMEM)
// Work of a CTA: its class blocks cb = blockIdx.x + k * gridDim.x; every block
// is swept by NU = 2 * RT units of 64 batch rows.  Global unit counter gu.
//   warps 0-7   softmax: two warpgroups, WG g takes the units gu % 2 == g;
//               thread = class (TMEM lane).  G^T = softmax^T / B - T^T
//               (label term folded in, R3) is written back into TMEM over the
//               S^T columns it came from.
//   warps 8-11  update: (a) load the W2T block (bf16 shadow) of block kb+NWT
//               into TMEM; (b) dW2T (lane = class) -> smem staging -> fused SGD
//               of W2T and the bf16 shadow (128-bit, coalesced); db2, b2.
//   warp 12     TMA producer (H row tiles of 128 rows)
//   warp 13     MMA issuer (warp-converged) + TMEM owner, S running NSB units
//               ahead of dW across block boundaries:
//                 S^T_u  = W2T_blk . H_u^T   (A = W2T_blk from TMEM, N = 64)
//                 dW2T  += G^T_u . H_u       (A = G^T from TMEM, B MN-major;
//                                             fixed unit order: deterministic)
// TMEM: S^T units at 64*b; W2T blocks at 64*NSB (+WCOLS each); dW2T last.
// =====================================================================
template <int H, bool ONEB>
__global__ void __launch_bounds__(BwdCfg<H, ONEB>::THREADS, 1)
    k_out_bwd(const __grid_constant__ CUtensorMap mapH, const __grid_constant__ CUtensorMap mapW,
              const __grid_constant__ CUtensorMap mapWf, const __grid_constant__ CUtensorMap mapHx,
              const StepDesc *__restrict__ desc, const float *__restrict__ lsep, int C,
              int n_cblocks, const int4 *__restrict__ cls_lab,
              const uint32_t *__restrict__ lbits, int lbw, const float *__restrict__ wrow,
              float *__restrict__ W2T, float *__restrict__ b2,
              __nv_bfloat16 *__restrict__ W2b, float lr, float *__restrict__ dbg_dW2T,
              float *__restrict__ dbg_db2, Dw1Args dw) {
  griddep_wait();
  using Cfg = BwdCfg<H, ONEB>;
  constexpr int NSH = Cfg::NSH, NSB = Cfg::NSB, NWT = Cfg::NWT, WCOLS = Cfg::WCOLS;
  constexpr bool W2S = Cfg::W2S;
  constexpr int UNIT = Cfg::UNIT, HPT = Cfg::HPT;
  constexpr int TILE = Cfg::TILE, SROW = Cfg::SROW;
  constexpr bool TMAUPD = Cfg::TMAUPD, FOLD = Cfg::FOLD, HALF = Cfg::HALF, PING = Cfg::PING;
  constexpr int HXB = Cfg::HXB, AXB = Cfg::AXB;
  constexpr uint32_t COL_W = NSB * UNIT, COL_DW = NSB * UNIT + Cfg::WTM;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *sHt = smem_raw;
  uint8_t *sW2 = sHt + NSH * TILE;              // W2S: the bf16 W2T block (K-major, SW128 atoms)
  uint8_t *sHx = sW2 + Cfg::W2SMEM;             // FOLD: B_ext of each H stage
  uint8_t *sAx = sHx + NSH * HXB;               // FOLD: A_ext of the class blocks in TMEM
  float *sT = (float *)(sAx + 2 * AXB);         // h = 128: W2T fp32 block; else dW2T staging
  float *sL = (float *)((uint8_t *)sT + Cfg::TSTAGE);    // lse' of the rows of each H stage (!FOLD)
  float *sWr = sL + (FOLD ? 0 : NSH * BM);      // label weight 1/(k_r B) of those rows (R3)
  float *sDB = sWr + NSH * BM;                  // [2][128] db2 partials of the two WGs
  uint4 *sMk = (uint4 *)(sDB + 2 * BM);          // [2][256] label-row bitmaps (softmax prefetch)
  int4 *sCl = (int4 *)(sMk + 2 * 256);           // [2][256] cls_lab of the next block
  float *sB2r = (float *)(sCl + 2 * 256);        // [2][256] b2 of the next block
  uint64_t *bars = (uint64_t *)(sB2r + 2 * 256);
  // p_full[PH b + half]: G^T of one 64-row half of the unit in S^T buffer b is
  // in TMEM; the dW MMA of that half starts without waiting for the other
  constexpr int PH = UNIT / 64;
  // RING (h = 128): a unit's S^T is computed in two 64-row halves whose TMEM
  // columns alternate with the WG's unit parity p: S half 0 at 64 p, half 1 at
  // 64 (1 - p), G^T (packed bf16) at 64 p + 32 half.  Half 1's columns are free
  // as soon as the softmax has loaded them (s_free), so the first half of the
  // WG's NEXT unit is computed while this one is still in the softmax, and the
  // second half as soon as this unit's dW has read its G^T (MMA order).
#ifdef AS_X_NORING
  constexpr bool RING = false;
#else
  constexpr bool RING = UNIT == 128;
#endif
  constexpr int SF = RING ? 2 * NSB : NSB;        // s_full per buffer (and half)
  constexpr bool S0POLL = RING && Cfg::S0POLL;
  constexpr int NPF = S0POLL ? 8 : PH * NSB;      // p_full: [unit mod 4][half] under S0POLL
  uint64_t *h_full = bars, *h_empty = h_full + NSH, *s_full = h_empty + NSH, *p_full = s_full + SF,
           *wt_full = p_full + NPF, *dw_full = wt_full + NWT, *dw_empty = dw_full + 1,
           *db_full = dw_empty + 1, *db_empty = db_full + 1, *wf_full = db_empty + 1, *s_free = wf_full + 1,
           *wf2 = s_free + NSB;                 // PING: the two half-block staging buffers
  uint32_t *tmem_slot = (uint32_t *)(wf2 + 2);
  if ((smem_u32(smem_raw) & 1023u) != 0) __trap();   // SW128 needs 1024-B alignment
  if (W2S && (int)gridDim.x < n_cblocks) __trap();    // W2S: one class block per CTA

  const int B = desc->rows;
  const int RT = (B + Cfg::TR - 1) / Cfg::TR;     // H tiles of TR rows
  const int NU = HPT * RT;                        // units per class block
  // every CTA sweeps the row tiles of a class block starting at its own
  // offset, so the 148 CTAs do not all fetch the same H tile from L2 at once
#ifdef AS_X_NOROT
  const int rot = 0;
#else
  const int rot = (int)(blockIdx.x % (unsigned)(RT > 0 ? RT : 1));
#endif
  // unit v of a class block covers row tile (v / HPT + rot) mod RT
  auto unit_rows = [&](int v_) { return ((v_ / HPT + rot) % RT) * HPT + v_ % HPT; };
  // NB (class blocks of this CTA) and NT = NB * NU (its units) are computed in
  // each role branch
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kProdWarp = 12, kMmaWarp = 13;   // highest ids: scheduler priority
#ifdef AS_X_SWAPROLES
  constexpr int kSoftLo = 4, kUpdLo = 0;         // softmax warps above the update warps
#else
  constexpr int kSoftLo = 0, kUpdLo = 8;
#endif

  if (threadIdx.x == 0) {
    for (int i = 0; i < NSH; ++i) { mbar_init(&h_full[i], 1); mbar_init(&h_empty[i], 1); }
    for (int i = 0; i < SF; ++i) mbar_init(&s_full[i], 1);
    for (int i = 0; i < NSB; ++i) mbar_init(&s_free[i], 4);
    for (int i = 0; i < NPF; ++i) mbar_init(&p_full[i], 4);
    for (int i = 0; i < NWT; ++i) mbar_init(&wt_full[i], W2S ? 1 : 4);
    mbar_init(dw_full, 1);
    mbar_init(dw_empty, 4);
    mbar_init(db_full, 8);
    mbar_init(db_empty, 4);
    mbar_init(wf_full, 1);
    mbar_init(&wf2[0], 1);
    mbar_init(&wf2[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) tmem_alloc(tmem_slot, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  // registers: 128 per thread at launch; warpgroup 3 (producer, MMA, 2 idle
  // warps) drops to 40.  h = 128: the softmax warpgroups keep 128 (their code
  // fits) and the update warpgroup rises to 208 so that it can drain the whole
  // dW2T accumulator (128 fp32 per lane) in one go; h = 256: the softmax
  // warpgroups rise to 168 and the update warpgroup keeps 128.
#define AS_REG_DEC2()                                                                       \
  do {                                                                                      \
    if constexpr (H != 128) asm volatile("setmaxnreg.dec.sync.aligned.u32 40;" ::: "memory"); \
    else if constexpr (Cfg::REGS3) asm volatile("setmaxnreg.dec.sync.aligned.u32 64;" ::: "memory"); \
  } while (0)
#define AS_REG_INC2()                                                                        \
  do {                                                                                       \
    if constexpr (H != 128) asm volatile("setmaxnreg.inc.sync.aligned.u32 168;" ::: "memory"); \
    else if constexpr (Cfg::REGS3) asm volatile("setmaxnreg.inc.sync.aligned.u32 160;" ::: "memory"); \
  } while (0)
#define AS_REG_UPD() asm volatile("setmaxnreg.inc.sync.aligned.u32 208;" ::: "memory")
  if (warp == kProdWarp) {
    AS_REG_DEC2();
    // NB / NT recomputed after setmaxnreg (an opaque copy of n_cblocks stops
    // the compiler reusing the prologue's value, which it otherwise spills)
    int nbq_ = n_cblocks;
    asm volatile("" : "+r"(nbq_));
    const int NB = blockIdx.x < nbq_ ? (nbq_ - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const int NT = NB * NU;
    (void)NT;
    if (lane == 0) {  // ---------------- TMA producer (H tiles)
      TRACE_INIT;
      if (W2S && NB > 0) {                    // the CTA's single W2T block (bf16), once
        mbar_expect_tx(&wt_full[0], BM * H * 2);
        for (int a = 0; a < H / 64; ++a)
          tma_load_2d(&mapW, &wt_full[0], sW2 + a * ATOM_BYTES, a * 64, (int)blockIdx.x * BM);
      }
      int it = 0;
      for (int kb = 0; kb < NB; ++kb)
        for (int t = 0; t < RT; ++t, ++it) {
          const int st = it % NSH;
          if (it >= NSH) {                    // W2S: on the critical path, no suspend hint
            if constexpr (W2S) mbar_wait(&h_empty[st], ((it / NSH) - 1) & 1);
            else mbar_wait_idle(&h_empty[st], ((it / NSH) - 1) & 1);
          }
          TRACE(2, true, 10, t);
#ifdef AS_X_NOTMA
          if (it >= NSH) { mbar_arrive(&h_full[st]); continue; }
#endif
          mbar_expect_tx(&h_full[st], TILE + HXB + (FOLD ? 1 : 2) * Cfg::TR * 4);
          const int tr = t + rot < RT ? t + rot : t + rot - RT;    // rotated row tile
          for (int a = 0; a < H / 64; ++a)
            tma_load_2d(&mapH, &h_full[st], sHt + st * TILE + a * Cfg::HATOM, a * 64, tr * Cfg::TR);
          if constexpr (FOLD) tma_load_2d(&mapHx, &h_full[st], sHx + st * HXB, 0, tr * BM);
          else bulk_load_1d(sL + st * BM, lsep + tr * Cfg::TR, Cfg::TR * 4, &h_full[st]);
          bulk_load_1d(sWr + st * BM, wrow + tr * Cfg::TR, Cfg::TR * 4, &h_full[st]);
        }
      if constexpr (W2S) {
        // the block's fp32 W2T (the update's staging) in two 64 KB halves, each
        // into an H stage as soon as its last tile's dW MMAs have read it
        // (BPS 32-column boxes per stage; half k = boxes 4k .. 4k + 3 on wf2[k])
        constexpr int BPS = TILE / 16384, NQ = (H / 32) / BPS;
        for (int q = 0; q < NQ && NB > 0; ++q, ++it) {
          const int st = it % NSH;
          if (it >= NSH) {                    // W2S: on the critical path, no suspend hint
            if constexpr (W2S) mbar_wait(&h_empty[st], ((it / NSH) - 1) & 1);
            else mbar_wait_idle(&h_empty[st], ((it / NSH) - 1) & 1);
          }
          if ((q * BPS) % 4 == 0) mbar_expect_tx(&wf2[(q * BPS) / 4], BM * 128 * 4);
          for (int c = 0; c < BPS; ++c) {
            const int bx = q * BPS + c;
            tma_load_2d(&mapWf, &wf2[bx / 4], sHt + st * TILE + c * 16384, bx * 32, (int)blockIdx.x * BM);
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    AS_REG_DEC2();
    // NB / NT recomputed after setmaxnreg (an opaque copy of n_cblocks stops
    // the compiler reusing the prologue's value, which it otherwise spills)
    int nbq_ = n_cblocks;
    asm volatile("" : "+r"(nbq_));
    const int NB = blockIdx.x < nbq_ ? (nbq_ - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const int NT = NB * NU;
    (void)NT;
    {  // ---------------- MMA issuer (warp-converged; one elected lane issues)
      constexpr uint32_t idS = idesc_bf16(BM, UNIT, 0, 0); // S^T_u = W2T_blk . H_u^T
      constexpr uint32_t idW = idesc_bf16(BM, H, 0, 1);    // dW2T += G^T_u . H_u
      const uint32_t aH = smem_u32(sHt);
      TRACE_INIT;
      // unit cursors with incremental indices and barrier phases: no integer
      // division on this warp's per-unit path (the uniform datapath is slow
      // and a division would queue on the MUFU behind the softmax exps)
      struct Cur {
        int kb, v, st, b, wb, hh;
        uint32_t hph, bph, wph;
      };
      auto advance = [&](Cur &c) {
        ++c.v;
        if (++c.hh == HPT) { c.hh = 0; if (++c.st == NSH) { c.st = 0; c.hph ^= 1u; } }
        if (c.v == NU) { c.v = 0; ++c.kb; if (++c.wb == NWT) { c.wb = 0; c.wph ^= 1u; } }
        if (++c.b == NSB) { c.b = 0; c.bph ^= 1u; }
      };
      auto issue_S = [&](const Cur &c) {
        TRACE(0, lane == 0, 15, c.v);
        if (c.v == 0) mbar_wait(&wt_full[c.wb], c.wph);
        if (c.hh == 0) mbar_wait(&h_full[c.st], c.hph);
        TRACE(0, lane == 0, 5, c.v);
        fence_after();
        // buffer b was last read (G^T of unit gu - NSB) by a dW issued earlier by
        // this warp: tcgen05.mma executes in issue order
        const uint64_t dB = sdesc(aH + c.st * TILE + c.hh * (UNIT * 128), 16, 1024);
#ifndef AS_X_NOMMA1
        if constexpr (W2S && Cfg::TR == 64)  // H atoms of 64 rows (8 KB), W2T atoms of 128 (16 KB)
          mma_grp_ss_kk_16_b64(tmem + c.b * UNIT, sdesc(smem_u32(sW2), 16, 1024), dB, idS, 0u);
        else if constexpr (W2S)
          mma_grp_ss_kk_16(tmem + c.b * UNIT, sdesc(smem_u32(sW2), 16, 1024), dB, idS, 0u);
        else if constexpr (H == 128)
          mma_grp_ts_k_8(tmem + c.b * UNIT, tmem + COL_W + c.wb * WCOLS, dB, idS, 0u);
        else
          mma_grp_ts_k_16(tmem + c.b * UNIT, tmem + COL_W + c.wb * WCOLS, dB, idS, 0u);
#endif
        mma_commit_w(&s_full[c.b]);
      };
      uint32_t dwe_ph = 0u;                   // dw_empty phase of the previous block
      auto do_dw = [&](const Cur &c) {
        TRACE(0, lane == 0, 1, c.v);
        mbar_wait(&p_full[PH * c.b], c.bph);
        TRACE(0, lane == 0, 2, c.v);
        if (c.v == 0 && c.kb >= 1) { mbar_wait(dw_empty, dwe_ph); dwe_ph ^= 1u; }
        fence_after();
#ifndef AS_X_NOMMA2
        if constexpr (UNIT == 128) {
          // rows 0-63 (G^T columns 0-31) while the softmax still works on rows 64-127
          mma_grp_ts_mn_4(tmem + COL_DW, tmem + c.b * UNIT, sdesc(aH + c.st * TILE, ATOM_BYTES, 1024), idW,
                          c.v > 0 ? 1u : 0u);
          mbar_wait(&p_full[PH * c.b + 1], c.bph);
          fence_after();
          mma_grp_ts_mn_4(tmem + COL_DW, tmem + c.b * UNIT + 32,
                          sdesc(aH + c.st * TILE + 64 * 128, ATOM_BYTES, 1024), idW, 1u);
        } else {
          mma_grp_ts_mn_4(tmem + COL_DW, tmem + c.b * UNIT,
                          sdesc(aH + c.st * TILE + c.hh * (UNIT * 128), Cfg::HATOM, 1024), idW,
                          c.v > 0 ? 1u : 0u);
        }
#else
        if constexpr (UNIT == 128) mbar_wait(&p_full[PH * c.b + 1], c.bph);
#endif
        if (c.hh == HPT - 1) mma_commit_w(&h_empty[c.st]);
        if (c.v == NU - 1) mma_commit_w(dw_full);
      };
      Cur cs{0, 0, 0, 0, 0, 0, 0u, 0u, 0u}, cd{0, 0, 0, 0, 0, 0, 0u, 0u, 0u};
      int ns = 0;                             // S units issued
      if constexpr (S0POLL) {
        constexpr uint32_t idS64 = idesc_bf16(BM, 64, 0, 0);
        // non-blocking phase test; the suspend variant sleeps up to ~64 ns
        auto ready = [&](uint64_t *bar, uint32_t ph) {
          uint32_t ok;
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                       "selp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok) : "r"(smem_u32(bar)), "r"(ph) : "memory");
          return ok != 0u;
        };
        auto ready_sleep = [&](uint64_t *bar, uint32_t ph) {
          uint32_t ok;
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
                       "selp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok) : "r"(smem_u32(bar)), "r"(ph), "r"(64u) : "memory");
          return ok != 0u;
        };
        // S half `half` of the unit at cursor c (parity c.bph): columns 64 ((half + par) & 1)
        auto issue_half = [&](const Cur &c, int half) {
#ifndef AS_X_NOMMA1
          const uint32_t dcol = c.b * UNIT + (uint32_t)(((half + (int)c.bph) & 1) * 64);
          mma_grp_ts_k_8(tmem + dcol, tmem + COL_W + c.wb * WCOLS,
                         sdesc(aH + c.st * TILE + half * 64 * 128, 16, 1024), idS64, 0u);
#endif
          mma_commit_w(&s_full[2 * c.b + half]);
        };
        Cur c0{0, 0, 0, 0, 0, 0, 0u, 0u, 0u}, c1{0, 0, 0, 0, 0, 0, 0u, 0u, 0u};
        int n0 = 0, n1 = 0, ndw = 0;          // units with S half 0 / S half 1 / both dW halves issued
        // S half 0 of unit n0: its S^T columns were loaded by the softmax (s_free of
        // unit n0 - 2), its H tile and W2T block have landed
        auto try_s0 = [&]() {
          while (n0 < NT) {
            if (n0 >= NSB && !ready(&s_free[c0.b], c0.bph ^ 1u)) break;
            if (c0.v == 0 && !ready(&wt_full[c0.wb], c0.wph)) break;
            if (c0.hh == 0 && !ready(&h_full[c0.st], c0.hph)) break;
            fence_after();
            issue_half(c0, 0);
            advance(c0);
            ++n0;
          }
        };
        // S half 1 of unit n1: into the G^T columns of unit n1 - 2, so after that
        // unit's dW (in-order MMA execution), and after its own half 0
        auto try_s1 = [&]() {
          while (n1 < n0 && n1 <= ndw + 1) {
            fence_after();
            issue_half(c1, 1);
            advance(c1);
            ++n1;
          }
        };
        for (int gu = 0; gu < NT; ++gu) {
          const uint32_t gcol = cd.b * UNIT + (uint32_t)(((gu >> 1) & 1) * 64);   // G^T of unit gu
          const int pf = (gu & 3) * 2;
          const uint32_t pph = (uint32_t)((gu >> 2) & 1);
          while (!ready_sleep(&p_full[pf], pph)) { try_s0(); try_s1(); }
          if (cd.v == 0 && cd.kb >= 1) {
            while (!ready_sleep(dw_empty, dwe_ph)) { try_s0(); try_s1(); }
            dwe_ph ^= 1u;
          }
          fence_after();
#ifndef AS_X_NOMMA2
          mma_grp_ts_mn_4(tmem + COL_DW, tmem + gcol, sdesc(aH + cd.st * TILE, ATOM_BYTES, 1024), idW,
                          cd.v > 0 ? 1u : 0u);
#endif
          try_s0(); try_s1();
          while (!ready_sleep(&p_full[pf + 1], pph)) { try_s0(); try_s1(); }
          fence_after();
#ifndef AS_X_NOMMA2
          mma_grp_ts_mn_4(tmem + COL_DW, tmem + gcol + 32, sdesc(aH + cd.st * TILE + 64 * 128, ATOM_BYTES, 1024),
                          idW, 1u);
#endif
          if (cd.hh == HPT - 1) mma_commit_w(&h_empty[cd.st]);
          if (cd.v == NU - 1) mma_commit_w(dw_full);
          ++ndw;
          advance(cd);
          try_s0(); try_s1();
        }
        (void)ns;
      } else if constexpr (RING) {
        // unit gu belongs to WG gu % 2 (buffer b = gu % NSB), its parity within
        // the WG is p = (gu / 2) & 1: S half h at columns 64 ((h + p) & 1)
        constexpr uint32_t idS64 = idesc_bf16(BM, 64, 0, 0);
        auto issue_S_half = [&](const Cur &c, int half, int par) {
          if (half == 0) {
            if (c.v == 0) mbar_wait(&wt_full[c.wb], c.wph);
            if (c.hh == 0) mbar_wait(&h_full[c.st], c.hph);
          }
          fence_after();
#ifndef AS_X_NOMMA1
          const uint32_t dcol = c.b * UNIT + (uint32_t)(((half + par) & 1) * 64);
          mma_grp_ts_k_8(tmem + dcol, tmem + COL_W + c.wb * WCOLS,
                         sdesc(aH + c.st * TILE + half * 64 * 128, 16, 1024), idS64, 0u);
#ifdef AS_X_NOEXTMMA
          if constexpr (false)
#else
          if constexpr (FOLD)                 // + b2_c - (LSE_r + ln B): one K-step from A_ext / B_ext
#endif
            mma_ss_w(tmem + dcol, sdesc32(smem_u32(sAx) + c.wb * AXB),
                     sdesc32(smem_u32(sHx) + c.st * HXB + half * 64 * 32), idS64, 1u);
#endif
          mma_commit_w(&s_full[2 * c.b + half]);
        };
        for (; ns < NT && ns < NSB; ++ns) {
          issue_S_half(cs, 0, 0);
          issue_S_half(cs, 1, 0);
          advance(cs);
        }
        for (int gu = 0; gu < NT; ++gu) {
          const uint32_t gcol = cd.b * UNIT + (uint32_t)(((gu >> 1) & 1) * 64);   // G^T of unit gu
          const int pn = ((gu + NSB) >> 1) & 1;                                    // parity of unit gu + 2
          const bool nxt = ns < NT;
          mbar_wait(&p_full[PH * cd.b], cd.bph);
          if (cd.v == 0 && cd.kb >= 1) { mbar_wait(dw_empty, dwe_ph); dwe_ph ^= 1u; }
          fence_after();
#ifndef AS_X_NOMMA2
          mma_grp_ts_mn_4(tmem + COL_DW, tmem + gcol, sdesc(aH + cd.st * TILE, ATOM_BYTES, 1024), idW,
                          cd.v > 0 ? 1u : 0u);
#endif
          if (nxt) {                          // S half 0 of the WG's next unit: into the columns
            mbar_wait(&s_free[cd.b], cd.bph); // this unit's half 1 has left (loaded by the softmax)
            issue_S_half(cs, 0, pn);
          }
          mbar_wait(&p_full[PH * cd.b + 1], cd.bph);
          fence_after();
#ifndef AS_X_NOMMA2
          mma_grp_ts_mn_4(tmem + COL_DW, tmem + gcol + 32, sdesc(aH + cd.st * TILE + 64 * 128, ATOM_BYTES, 1024),
                          idW, 1u);
#endif
          if (cd.hh == HPT - 1) mma_commit_w(&h_empty[cd.st]);
          if (cd.v == NU - 1) mma_commit_w(dw_full);
          if (nxt) {                          // half 1: after this unit's dW (in-order MMA)
            issue_S_half(cs, 1, pn);
            advance(cs);
            ++ns;
          }
          advance(cd);
        }
      } else {
      for (; ns < NT && ns < NSB; ++ns) { issue_S(cs); advance(cs); }
      for (int gu = 0; gu < NT; ++gu) {
        do_dw(cd);
        // S runs NSB units ahead; with a single TMEM W2T buffer the look-ahead
        // may not cross into the next block before this block's last dW
        // ... and only into H tiles whose stage the producer can fill: tile T
        // goes into stage T % NSH once every dW of tile T - NSH is issued
        while (ns < NT && ns <= gu + NSB && ns / HPT < (gu + 1) / HPT + NSH &&
               (NWT > 1 || cs.kb == cd.kb || cd.v == NU - 1)) {
          issue_S(cs);
          advance(cs);
          ++ns;
        }
        advance(cd);
      }
      }
    }
  } else if (warp >= kSoftLo && warp < kSoftLo + 8) {  // ---------------- softmax warpgroups (units gu % 2 == g)
    AS_REG_INC2();
    // NB / NT recomputed after setmaxnreg (an opaque copy of n_cblocks stops
    // the compiler reusing the prologue's value, which it otherwise spills)
    int nbq_ = n_cblocks;
    asm volatile("" : "+r"(nbq_));
    const int NB = blockIdx.x < nbq_ ? (nbq_ - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const int NT = NB * NU;
    (void)NT;
    const int g = (warp - kSoftLo) >> 2;
    const int q = warp & 3;
    const int i = q * 32 + lane;              // class inside the block (TMEM lane)
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    TRACE_INIT;
    // Prefetches go global -> shared with cp.async (zero-filled when the class
    // is out of range or has no label), two slots each, so no register ever
    // holds a pending load (a move or select of one stalls the warp on HBM):
    //   * per-class state of a class block (b2, and cls_lab from the label
    //     transpose) one block ahead, slot = block parity;
    //   * the class's label-row bitmap of a unit (k_tr_mark; bit r = row r
    //     has label i) one unit ahead, slot = WG unit parity.
    const int tix = threadIdx.x - kSoftLo * 32;  // 0..255
    auto cls_ok = [&](int kb_) {
      return kb_ < NB && (blockIdx.x + kb_ * gridDim.x) * BM + i < C;
    };
    auto pf_cls = [&](int kb_) {
      const bool ok = cls_ok(kb_);
      const int cc = ok ? (blockIdx.x + kb_ * gridDim.x) * BM + i : 0;
      const int sl = (kb_ & 1) * 256 + tix;
      cp_async_16(sCl + sl, cls_lab + cc, ok ? 16u : 0u);
      cp_async_4(sB2r + sl, b2 + cc, ok ? 4u : 0u);
    };
    auto pf_mask = [&](int kb_, int v_, bool has, int slot) {
      const uint32_t *bits = has ? lbits + (size_t)((blockIdx.x + kb_ * gridDim.x) * BM + i) * lbw +
                                       unit_rows(v_) * (UNIT / 32)
                                 : lbits;
      if constexpr (UNIT == 128) cp_async_16(sMk + slot * 256 + tix, bits, has ? 16u : 0u);
      else cp_async_8(sMk + slot * 256 + tix, bits, has ? 8u : 0u);
    };
    auto cls_has = [&](int kb_) {             // the block's state must have landed
      const int4 cl = sCl[(kb_ & 1) * 256 + tix];
      return cls_ok(kb_) && cl.x < cl.y;
    };
    // NU = 1 (B <= UNIT): block kb's single unit belongs to WG kb % 2, so a WG
    // walks every other block
    const int kstep = NU == 1 ? 2 : 1;
    int kb_cur = -1;
    bool has_lab = false;                     // class i has labels in this batch
    float b2c = 0.f, db2 = 0.f;
    float Ec = 0.f, iEc = 0.f;                // ECF: exp(b2_c) and its inverse (0 past C)
    int kb = 0, v = g, lst = g / HPT, sb = g; // unit cursor: block, unit, lse' stage, S buffer
    while (NU > 0 && v >= NU) { v -= NU; ++kb; }   // NU = 1: WG 1 starts in block 1
    pf_cls(kb);
    cp_async_commit();
    cp_async_wait<0>();
    pf_mask(kb, v, cls_has(kb), 0);
    cp_async_commit();
    int jj = 0;                               // units of this WG so far
    uint32_t sph = 0u;
    for (int gu = g; gu < NT; gu += 2, ++jj) {
      // a class block change commits the next block's state prefetch in this
      // iteration, before the next unit's bitmap: the bitmap wait below could
      // leave two groups pending there (AS_X_GRP2) -- measured slower (Amazon-670K
      // step 0.6534 -> 0.6568 ms, AmazonCat-13K 0.1204 -> 0.1220 ms), off
      bool newblk = false;
      if (kb != kb_cur) {                     // new class block: per-class state
        newblk = true;
        kb_cur = kb;
        const bool ok = cls_ok(kb);
        b2c = ok ? sB2r[(kb & 1) * 256 + tix] * LOG2E : -INFINITY;
        if constexpr (Cfg::ECF) {
          Ec = ok ? ex2(b2c) : 0.f;
          iEc = ok ? ex2(-b2c) : 0.f;
        }
        has_lab = cls_has(kb);
        db2 = 0.f;
        pf_cls(kb + kstep);                   // slot (kb + kstep) & 1: read above already
        cp_async_commit();
      }
      const int b = sb;
      TRACE(1, tix == 0, 18, v);
      // the next unit of this WG: its class's row bitmap one unit ahead
      {
        int vn = v + 2, kbn = kb;
        while (vn >= NU) { vn -= NU; ++kbn; }
        bool hn = has_lab;
        if (kbn != kb) {                      // crossing a block: its state, prefetched at this block's change
          cp_async_wait<0>();
          hn = cls_has(kbn);
        }
        pf_mask(kbn, vn, hn, (jj + 1) & 1);
        cp_async_commit();
      }
      TRACE(1, tix == 0, 6, v);
      if constexpr (!RING) mbar_wait(&s_full[b], sph);
      TRACE(1, tix == 0, 7, v);
      fence_after();
      const uint32_t par = RING ? (uint32_t)(jj & 1) : 0u;   // column parity of this unit (RING)
      uint32_t mk[4];
      // this unit's bitmap (all cp.async groups but the newest): read where the
      // label term needs it, after the first half's exponentials (LATEMK), so the
      // cp.async completion wait is off the unit's critical path
      auto read_mk = [&]() {
#ifndef AS_X_GRP2
        (void)newblk;
        cp_async_wait<1>();
#else
        if (newblk) cp_async_wait<2>();
        else cp_async_wait<1>();
#endif
        if constexpr (UNIT == 128) {
          const uint4 q4 = sMk[(jj & 1) * 256 + tix];
          mk[0] = q4.x; mk[1] = q4.y; mk[2] = q4.z; mk[3] = q4.w;
        } else {
          const uint2 q2 = *reinterpret_cast<const uint2 *>(sMk + (jj & 1) * 256 + tix);
          mk[0] = q2.x; mk[1] = q2.y; mk[2] = 0u; mk[3] = 0u;
        }
      };
      if constexpr (!Cfg::LATEMK) read_mk();
#ifndef AS_X_NOSOFT
#pragma unroll 1
      for (int half = 0; half < UNIT / 64; ++half) {   // 64 rows of the unit at a time
        uint32_t r0[32], r1[32];
        const uint32_t scol = RING ? (uint32_t)(((half + (int)par) & 1) * 64) : (uint32_t)(half * 64);
        if constexpr (RING) {
          mbar_wait(&s_full[2 * b + half], sph);
          fence_after();
        }
        AS_TMEM_LD32(tl + b * UNIT + scol, r0);
        AS_TMEM_LD32(tl + b * UNIT + scol + 32, r1);
        // -lse' = -(LSE_r log2e + log2 B) of these 64 rows (smem broadcast)
        const float4 *lq = reinterpret_cast<const float4 *>(sL + (FOLD ? 0 : lst * BM + (v % HPT) * UNIT + half * 64));
        AS_TMEM_WAIT_LD(r0);
        AS_TMEM_WAIT_LD(r1);
        if (RING && half == 1) {              // half 1's S columns are free for the next unit
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&s_free[b]);
        }
        uint32_t pk[32];                      // 64 bf16 of G^T, packed in pairs
        uint64_t dacc[4] = {0ull, 0ull, 0ull, 0ull};
        const uint64_t l2e2 = f2(LOG2E, LOG2E), b2c2 = f2(b2c, b2c);
#pragma unroll
        for (int k4 = 0; k4 < 16; ++k4) {
          const float4 l4 = FOLD ? make_float4(0.f, 0.f, 0.f, 0.f) : lq[k4];
#pragma unroll
          for (int m = 0; m < 2; ++m) {       // packed: x = s log2e + b2 - lse'
            const int k = 4 * k4 + 2 * m, u = 2 * k4 + m;
            const uint32_t xa = k < 32 ? r0[k] : r1[k - 32], xb = k < 32 ? r0[k + 1] : r1[k - 31];
            uint64_t x;
            if constexpr (FOLD) {             // S^T already holds z - LSE - ln B: p / B = 2^(S log2e)
              x = fmul2(f2(__uint_as_float(xa), __uint_as_float(xb)), l2e2);
            } else if constexpr (Cfg::ECF) {  // G' = G / E_c: s log2e - lse'
              x = ffma2(f2(__uint_as_float(xa), __uint_as_float(xb)), l2e2,
                        m == 0 ? f2(l4.x, l4.y) : f2(l4.z, l4.w));
            } else {
              x = ffma2(f2(__uint_as_float(xa), __uint_as_float(xb)), l2e2, b2c2);
              x = fadd2(x, m == 0 ? f2(l4.x, l4.y) : f2(l4.z, l4.w));
            }
            float e0, e1;
            if (AS_EMU_AT(AS_EMU_P2, u)) {
              ex2_emu2(x, e0, e1);
            } else {
              float x0, x1;
              f2split(x, x0, x1);
              e0 = XEX2(x0);
              e1 = XEX2(x1);
            }
            // p / B straight into the db2 sums and the packed bf16 G^T: no
            // 64-value array stays live (register pressure)
#ifdef AS_X_P2NOSOFT
            e0 = e1 = 0.f;                     // mutant: no softmax term in pass 2 (parity tests must fail)
#endif
            dacc[u & 3] = fadd2(dacc[u & 3], f2(e0, e1));
            pk[u] = pack_bf16x2(e0, e1);
          }
        }
        {
          float d0, d1;
          f2split(fadd2(fadd2(dacc[0], dacc[1]), fadd2(dacc[2], dacc[3])), d0, d1);
          db2 += d0 + d1;
        }
        // label term of the uniform multi-label target folded into G (R3, R24):
        // G_rc = bf16(p_rc / B) - [c in Y_r] / (k_r B) (rounded to bf16 again),
        // db2 -= the same weights; row weights from the stage's label-weight
        // ring; only warps with a label of one of their classes in these rows
        {
          if constexpr (Cfg::LATEMK) {
            if (half == 0) read_mk();
          }
          // static register indices (half is a runtime loop counter)
          uint32_t m0 = mk[0], m1 = mk[1];
          if (half) { m0 = mk[2]; m1 = mk[3]; }
#ifdef AS_X_NOLAB
          if (false)
#endif
          if (__any_sync(0xffffffffu, (m0 | m1) != 0u)) {
            const float4 *wq = reinterpret_cast<const float4 *>(sWr + lst * BM + (v % HPT) * UNIT + half * 64);
#pragma unroll
            for (int u = 0; u < 32; ++u) {
              const uint32_t mw = u < 16 ? m0 : m1;
              const uint32_t bits = (mw >> ((2 * u) & 31)) & 3u;
              if (bits) {
                float2 w2 = reinterpret_cast<const float2 *>(wq)[u];
                if constexpr (Cfg::ECF) { w2.x *= iEc; w2.y *= iEc; }
                float lo = __uint_as_float(pk[u] << 16), hi = __uint_as_float(pk[u] & 0xffff0000u);
                if (bits & 1u) { lo -= w2.x; db2 -= w2.x; }
                if (bits & 2u) { hi -= w2.y; db2 -= w2.y; }
                pk[u] = pack_bf16x2(lo, hi);
              }
            }
          }
        }
        // G^T over S^T columns already consumed (cols [32 half, 32 half + 32)),
        // then this half's dW MMA may start
        AS_TMEM_ST32(tl + b * UNIT + (RING ? par * 64u : 0u) + half * 32, pk);
        tmem_wait_st();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[S0POLL ? (gu & 3) * 2 + half : PH * b + half]);
      }
      TRACE(1, tix == 0, 8, v);
#else
      if constexpr (RING) {
        mbar_wait(&s_full[2 * b], sph);
        mbar_wait(&s_full[2 * b + 1], sph);
      }
      fence_before();
      __syncwarp();
      if (lane == 0) {
        for (int hf = 0; hf < PH; ++hf) mbar_arrive(&p_full[S0POLL ? (gu & 3) * 2 + hf : PH * b + hf]);
        if (RING) mbar_arrive(&s_free[b]);
      }
      (void)par;
#endif
      TRACE(1, tix == 0, 9, v);
      if (v >= NU - 2) {                      // this WG's last unit of the block: db2 partial
        if (kb >= 1) mbar_wait(db_empty, (kb - 1) & 1);
        TRACE(1, tix == 0, 16, v);
        sDB[g * BM + i] = Cfg::ECF ? db2 * Ec : db2;
        if (NU == 1) sDB[(1 - g) * BM + i] = 0.f;   // one unit per block: the other WG has none
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(db_full);
          if (NU == 1) mbar_arrive(db_full);
        }
      }
      TRACE(1, tix == 0, 17, v);
      v += 2;                                 // next unit of this WG
      while (v >= NU) { v -= NU; ++kb; }
      lst += 2 / HPT;                         // its H stage
      if (lst >= NSH) lst -= NSH;
      sb += 2;
      if (sb >= NSB) { sb -= NSB; sph ^= 1u; }
    }
  } else if (warp >= kUpdLo && warp < kUpdLo + 4) {  // ---------------- update warps
#ifdef AS_X_EARLYREL
    if constexpr (TMAUPD) AS_REG_UPD();
#else
    // the half-block update loop holds a prefetched W2T block (64 registers)
    // next to its working set: 160 registers (the pool has the 88 x 128 that
    // warpgroup 3 released; the softmax warpgroups keep 128)
    if constexpr (PING || HALF) asm volatile("setmaxnreg.inc.sync.aligned.u32 160;" ::: "memory");
#endif
    // NB / NT recomputed after setmaxnreg (an opaque copy of n_cblocks stops
    // the compiler reusing the prologue's value, which it otherwise spills)
    int nbq_ = n_cblocks;
    asm volatile("" : "+r"(nbq_));
    const int NB = blockIdx.x < nbq_ ? (nbq_ - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const int NT = NB * NU;
    (void)NT;
    const int q = warp & 3;
    const int i = q * 32 + lane;              // thread = class (TMEM lane)
    const int ut = threadIdx.x - kUpdLo * 32;  // 0..127
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    constexpr int NCH = H / 32;               // 32-column chunks of dW2T
    const int sub = lane >> 3, hq = (lane & 7) * 4;
    TRACE_INIT;
    // FOLD: row i of the class block's A_ext tile = [b2 in three bf16 parts (-1e30
    // past C: p = 0), 1, 1, 1, 0 ...] (SWIZZLE_32B), visible to the MMA (async proxy)
    auto put_ax = [&](int kb_, float b2v) {
      if constexpr (FOLD) {
        const int wb = kb_ % NWT;
        const float hi = __bfloat162float(__float2bfloat16_rn(b2v));
        const float r1 = b2v - hi;
        const float mid = __bfloat162float(__float2bfloat16_rn(r1));
        const float lo = r1 - mid;
        uint8_t *row = sAx + wb * AXB;
        *reinterpret_cast<uint4 *>(row + swz32(i, 0)) =
            make_uint4(pack_bf16x2(hi, mid), pack_bf16x2(lo, 1.f), pack_bf16x2(1.f, 1.f), 0u);
        *reinterpret_cast<uint4 *>(row + swz32(i, 1)) = make_uint4(0u, 0u, 0u, 0u);
        fence_proxy_async();
      }
    };
    auto b2_of = [&](int kb_) {
      const int cls = (blockIdx.x + kb_ * gridDim.x) * BM + i;
      return cls < C ? b2[cls] : -1e30f;
    };
    // W2T block (bf16 shadow, row of class i) -> TMEM A-operand columns of buffer wb
    auto load_wt = [&](int kb_) {
      const int wb = kb_ % NWT;
      const int cls = (blockIdx.x + kb_ * gridDim.x) * BM + i;
      const uint4 *src = reinterpret_cast<const uint4 *>(W2b + (size_t)(cls < C ? cls : 0) * H);
#pragma unroll 1
      for (int half = 0; half < H / 128; ++half) {
        uint32_t r[64];                       // 128 bf16 of the row: every load in flight
#pragma unroll
        for (int v4 = 0; v4 < 16; ++v4) {
          uint4 x = src[half * 16 + v4];
          if (cls >= C) x = make_uint4(0u, 0u, 0u, 0u);
          r[4 * v4] = x.x; r[4 * v4 + 1] = x.y; r[4 * v4 + 2] = x.z; r[4 * v4 + 3] = x.w;
        }
        AS_TMEM_ST32(tl + COL_W + wb * WCOLS + 64 * half, r);
        AS_TMEM_ST32(tl + COL_W + wb * WCOLS + 64 * half + 32, (r + 32));
      }
      put_ax(kb_, b2_of(kb_));
      tmem_wait_st();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&wt_full[wb]);
    };
    if constexpr (PING) {                     // fp32 W2T of the first block: both halves
      if (ut == 0 && NB > 0)
        for (int hh = 0; hh < 2; ++hh) {
          mbar_expect_tx(&wf2[hh], BM * 64 * 4);
          for (int c = 0; c < 2; ++c)
            tma_load_2d(&mapWf, &wf2[hh], (uint8_t *)sT + hh * 32768 + c * 16384, 64 * hh + c * 32, blockIdx.x * BM);
        }
    } else if constexpr (TMAUPD) {            // fp32 W2T of the first block (its first half)
      if (ut == 0 && NB > 0) {
        constexpr int NBOX = HALF ? 2 : 4;
        mbar_expect_tx(wf_full, BM * 32 * 4 * NBOX);
        for (int c = 0; c < NBOX; ++c) tma_load_2d(&mapWf, wf_full, (uint8_t *)sT + c * 16384, c * 32, blockIdx.x * BM);
      }
    }
    // h = 128: the bf16 W2T rows of block kb + NWT are fetched into registers
    // BEFORE waiting for block kb's accumulator (the HBM latency hides in that
    // wait) and written into the TMEM buffer block kb's S MMAs have released
    float b2pre = 0.f;                        // FOLD: b2 of the prefetched block's class i
    auto fetch_wt = [&](int kb_, uint32_t (&r)[64]) {
      if constexpr (FOLD) b2pre = b2_of(kb_);
      const int cls = (blockIdx.x + kb_ * gridDim.x) * BM + i;
      const uint4 *src = reinterpret_cast<const uint4 *>(W2b + (size_t)(cls < C ? cls : 0) * H);
#pragma unroll
      for (int v4 = 0; v4 < 16; ++v4) {
        uint4 x = src[v4];
        if (cls >= C) x = make_uint4(0u, 0u, 0u, 0u);
        r[4 * v4] = x.x; r[4 * v4 + 1] = x.y; r[4 * v4 + 2] = x.z; r[4 * v4 + 3] = x.w;
      }
    };
    auto put_wt = [&](int kb_, uint32_t (&r)[64]) {
      const int wb = kb_ % NWT;
      AS_TMEM_ST32(tl + COL_W + wb * WCOLS, r);
      AS_TMEM_ST32(tl + COL_W + wb * WCOLS + 32, (r + 32));
      put_ax(kb_, b2pre);
      tmem_wait_st();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&wt_full[wb]);
    };
    if constexpr (!W2S)
      for (int kb = 0; kb < NB && kb < NWT; ++kb) load_wt(kb);
    for (int kb = 0; kb < NB; ++kb) {
      const int cb = blockIdx.x + kb * gridDim.x;
      uint32_t wpre[TMAUPD ? 64 : 1];
      if constexpr (TMAUPD) {
        if (kb + NWT < NB) fetch_wt(kb + NWT, wpre);
      }
      // ECF: this class's bias before its update below (the value the softmax
      // warps took E_c from); loaded before the accumulator wait
      float b2u = 0.f;
      if constexpr (Cfg::ECF) {
        const int cu = cb * BM + i;
        b2u = cu < C ? b2[cu] : 0.f;
      }
      // h = 256: this thread's W2T values of the block's first 32-column chunk
      // (8 classes x 4 columns) are loaded before the accumulator wait, and
      // every chunk's RMW runs on values loaded during the previous chunk
      float4 wq[TMAUPD ? 1 : 8];
      auto ld_chunk = [&](int ch_, float4 (&w)[TMAUPD ? 1 : 8]) {
        if constexpr (!TMAUPD) {
#pragma unroll
          for (int m = 0; m < 8; ++m) {
            const int cls = cb * BM + q * 32 + 4 * m + sub;
            w[m] = cls < C ? *reinterpret_cast<const float4 *>(W2T + (size_t)cls * H + ch_ * 32 + hq)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
      };
      // h = 256, last block: the H stages are free once its accumulator is
      // complete, so the whole fp32 block is TMA-loaded into them (LASTSMEM)
      const bool last_smem = W2S || (!TMAUPD && Cfg::LASTSMEM && kb == NB - 1);   // W2S: NB = 1
      if (!last_smem) ld_chunk(0, wq);
      TRACE(3, ut == 0, 11, kb);
      mbar_wait_sleepy(dw_full, kb & 1, 256);   // also: every S of block kb completed
      TRACE(3, ut == 0, 12, kb);
      fence_after();
      if constexpr (HALF || PING) {
        if (kb + NWT < NB) put_wt(kb + NWT, wpre);
        // fused SGD of the block, 64 columns at a time: the TMEM accumulator
        // (lane i = class i) and the TMA-staged fp32 half block (two swizzled
        // 32-column boxes): W2T -= lr dW2T in place, TMA store, coalesced bf16
        // shadow; the other half is TMA-loaded meanwhile.  The accumulator is
        // released once the second half's columns are in registers.
        const uint32_t sw = (uint32_t)(i & 7);
        uint8_t *rowWf = reinterpret_cast<uint8_t *>(sT) + i * 128;
        const int cls_i = cb * BM + i;
        auto sgd_box = [&](int bx, int ch, const uint32_t (&r)[32]) {
#ifndef AS_X_NOUPD
#pragma unroll
          for (int g0 = 0; g0 < 8; g0 += 4) {
            float4 w[4];
#pragma unroll
            for (int g = 0; g < 4; ++g)
              w[g] = *reinterpret_cast<const float4 *>(rowWf + bx * 16384 + (((uint32_t)(g0 + g) ^ sw) << 4));
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              w[g].x = fmaf(-lr, __uint_as_float(r[4 * (g0 + g)]), w[g].x);
              w[g].y = fmaf(-lr, __uint_as_float(r[4 * (g0 + g) + 1]), w[g].y);
              w[g].z = fmaf(-lr, __uint_as_float(r[4 * (g0 + g) + 2]), w[g].z);
              w[g].w = fmaf(-lr, __uint_as_float(r[4 * (g0 + g) + 3]), w[g].w);
            }
#pragma unroll
            for (int g = 0; g < 4; ++g)
              *reinterpret_cast<float4 *>(rowWf + bx * 16384 + (((uint32_t)(g0 + g) ^ sw) << 4)) = w[g];
          }
#endif
          if (dbg_dW2T && cls_i < C) {
#pragma unroll
            for (int k = 0; k < 32; ++k) dbg_dW2T[(size_t)cls_i * H + ch * 32 + k] = __uint_as_float(r[k]);
          }
        };
#pragma unroll 1
        for (int hh = 0; hh < 2; ++hh) {
          const int bo = PING ? hh * 2 : 0;   // staging box index of this half (PING: buffer hh)
          uint32_t ra[32], rb[32];
          AS_TMEM_LD32(tl + COL_DW + hh * 64, ra);
          AS_TMEM_LD32(tl + COL_DW + hh * 64 + 32, rb);
          AS_TMEM_WAIT_LD(ra);
          AS_TMEM_WAIT_LD(rb);
          if (hh == 1) {                      // accumulator free for block kb + 1
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(dw_empty);
          }
          if constexpr (PING) mbar_wait(&wf2[hh], kb & 1);
          else mbar_wait(wf_full, (2 * kb + hh) & 1);
          sgd_box(bo, 2 * hh, ra);
          sgd_box(bo + 1, 2 * hh + 1, rb);
          fence_proxy_async();
          named_bar(3, 128);
#ifndef AS_X_NOUPD
          if (ut == 0) {
            for (int c = 0; c < 2; ++c)
              tma_store_2d(&mapWf, (uint8_t *)sT + (bo + c) * 16384, 64 * hh + c * 32, cb * BM);
            bulk_commit();
          }
          // bf16 shadow of these 64 columns, coalesced (8 threads per class row)
#pragma unroll 4
          for (int k = 0; k < 8; ++k) {
            const int idx = k * 128 + ut;
            const int row = idx >> 3, c8 = idx & 7;
            const int cls = cb * BM + row;
            const uint8_t *rbp = reinterpret_cast<const uint8_t *>(sT) + (bo + (c8 >> 2)) * 16384 + row * 128;
            const uint32_t g0 = (uint32_t)((c8 & 3) * 2), rs = (uint32_t)(row & 7);
            const float4 a = *reinterpret_cast<const float4 *>(rbp + ((g0 ^ rs) << 4));
            const float4 b = *reinterpret_cast<const float4 *>(rbp + (((g0 + 1) ^ rs) << 4));
            if (cls < C)
              *reinterpret_cast<uint4 *>(W2b + (size_t)cls * H + 64 * hh + 8 * c8) =
                  make_uint4(pack_bf16x2(a.x, a.y), pack_bf16x2(a.z, a.w), pack_bf16x2(b.x, b.y),
                             pack_bf16x2(b.z, b.w));
          }
          named_bar(3, 128);                  // every thread's reads of the staging are done
#endif
          if (ut == 0) {
#ifndef AS_X_NOUPD
            bulk_wait_read0();
#endif
            if constexpr (PING) {
              if (kb + 1 < NB) {              // this half of the next block, into the same buffer
                mbar_expect_tx(&wf2[hh], BM * 64 * 4);
                for (int c = 0; c < 2; ++c)
                  tma_load_2d(&mapWf, &wf2[hh], (uint8_t *)sT + (bo + c) * 16384, 64 * hh + c * 32,
                              (cb + (int)gridDim.x) * BM);
              }
            } else {
              const bool more = hh == 0 || kb + 1 < NB;
              if (more) {                     // the other half of this block, or the next block's first
                const int nrow = (hh == 0 ? cb : cb + (int)gridDim.x) * BM, ncol = hh == 0 ? 64 : 0;
                mbar_expect_tx(wf_full, BM * 64 * 4);
                for (int c = 0; c < 2; ++c)
                  tma_load_2d(&mapWf, wf_full, (uint8_t *)sT + c * 16384, ncol + c * 32, nrow);
              }
            }
          }
        }
      } else if constexpr (TMAUPD) {
        if (kb + NWT < NB) put_wt(kb + NWT, wpre);
        // fused SGD of the block from the TMEM accumulator (lane i = class i)
        // and the TMA-loaded fp32 block: W2T -= lr dW2T in place (swizzled
        // 32-column boxes, conflict-free), bf16 shadow into its staging boxes
        const uint32_t sw = (uint32_t)(i & 7);
        uint8_t *rowWf = reinterpret_cast<uint8_t *>(sT) + i * 128;
        const int cls_i = cb * BM + i;
        // W2T_c -= lr dW2T_c, with dW2T_c = E_c (G'^T H)_c under ECF
        const float Eu = Cfg::ECF ? ex2(b2u * LOG2E) : 1.f;
        const float nlr = -lr * Eu;
        auto sgd_chunk = [&](int ch, const uint32_t (&r)[32]) {
#ifndef AS_X_NOUPD
#pragma unroll
          for (int g0 = 0; g0 < 8; g0 += 4) {   // 4 swizzled 16-B rows at a time
            float4 w[4];
#pragma unroll
            for (int g = 0; g < 4; ++g)
              w[g] = *reinterpret_cast<const float4 *>(rowWf + ch * 16384 + (((uint32_t)(g0 + g) ^ sw) << 4));
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              w[g].x = fmaf(nlr, __uint_as_float(r[4 * (g0 + g)]), w[g].x);
              w[g].y = fmaf(nlr, __uint_as_float(r[4 * (g0 + g) + 1]), w[g].y);
              w[g].z = fmaf(nlr, __uint_as_float(r[4 * (g0 + g) + 2]), w[g].z);
              w[g].w = fmaf(nlr, __uint_as_float(r[4 * (g0 + g) + 3]), w[g].w);
            }
#pragma unroll
            for (int g = 0; g < 4; ++g)
              *reinterpret_cast<float4 *>(rowWf + ch * 16384 + (((uint32_t)(g0 + g) ^ sw) << 4)) = w[g];
#ifdef AS_X_ROWSHADOW
            if (cls_i < C) {                  // bf16 shadow: 8 columns per 16-byte store (row per thread)
#pragma unroll
              for (int g = 0; g < 4; g += 2)
                *reinterpret_cast<uint4 *>(W2b + (size_t)cls_i * H + ch * 32 + 4 * (g0 + g)) =
                    make_uint4(pack_bf16x2(w[g].x, w[g].y), pack_bf16x2(w[g].z, w[g].w),
                               pack_bf16x2(w[g + 1].x, w[g + 1].y), pack_bf16x2(w[g + 1].z, w[g + 1].w));
            }
#endif
          }
#endif
          if (dbg_dW2T && cls_i < C) {
#pragma unroll
            for (int k = 0; k < 32; ++k) dbg_dW2T[(size_t)cls_i * H + ch * 32 + k] = __uint_as_float(r[k]) * Eu;
          }
        };
        static_assert(NCH == 4, "h = 128: four 32-column chunks");
#ifdef AS_X_EARLYREL
        // the whole accumulator (lane i = class i, 128 fp32) into registers at
        // once, then it is released: block kb + 1's first dW MMA waits only for
        // these loads, not for the SGD below (this warpgroup runs with 208
        // registers, AS_REG_UPD; measured no faster than releasing after the
        // last chunk's load, which is the default)
        uint32_t racc[128];
        AS_TMEM_LD64(tl + COL_DW, racc);
        AS_TMEM_LD64(tl + COL_DW + 64, (racc + 64));
        AS_TMEM_WAIT_LD64(racc);
        AS_TMEM_WAIT_LD64((racc + 64));
        fence_before();                       // accumulator free for block kb + 1
        __syncwarp();
        if (lane == 0) mbar_arrive(dw_empty);
        TRACE(3, ut == 0, 15, kb);
        mbar_wait(wf_full, kb & 1);           // this block's fp32 W2T (TMA, issued a block ahead)
        sgd_chunk(0, *reinterpret_cast<const uint32_t(*)[32]>(racc));
        sgd_chunk(1, *reinterpret_cast<const uint32_t(*)[32]>(racc + 32));
        sgd_chunk(2, *reinterpret_cast<const uint32_t(*)[32]>(racc + 64));
        sgd_chunk(3, *reinterpret_cast<const uint32_t(*)[32]>(racc + 96));
#else
        mbar_wait(wf_full, kb & 1);
#pragma unroll 1
        for (int ch = 0; ch < NCH; ++ch) {    // chunk by chunk; released after the last load
          uint32_t ra[32];
          AS_TMEM_LD32(tl + COL_DW + ch * 32, ra);
          AS_TMEM_WAIT_LD(ra);
          if (ch == NCH - 1) {
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(dw_empty);
          }
          sgd_chunk(ch, ra);
        }
#endif
        // (2) block kb + NWT's W2T already in TMEM (put_wt above)
        // (3) TMA store of the updated block, then the next block's fp32 W2T
        //     into the same buffer once the store has read it
        fence_proxy_async();
        named_bar(3, 128);
#ifndef AS_X_NOUPD
        if (ut == 0) {
          for (int c = 0; c < 4; ++c) tma_store_2d(&mapWf, (uint8_t *)sT + c * 16384, c * 32, cb * BM);
          bulk_commit();
        }
#ifndef AS_X_ROWSHADOW
        // bf16 shadow of the updated block, coalesced: 16 threads per class row,
        // 16 bytes (8 columns) each, read from the swizzled fp32 boxes
#pragma unroll 4
        for (int k = 0; k < 16; ++k) {
          const int idx = k * 128 + ut;
          const int row = idx >> 4, c8 = idx & 15;
          const int cls = cb * BM + row;
          const uint8_t *rb = reinterpret_cast<const uint8_t *>(sT) + (c8 >> 2) * 16384 + row * 128;
          const uint32_t g0 = (uint32_t)((c8 & 3) * 2), rs = (uint32_t)(row & 7);
          const float4 a = *reinterpret_cast<const float4 *>(rb + ((g0 ^ rs) << 4));
          const float4 b = *reinterpret_cast<const float4 *>(rb + (((g0 + 1) ^ rs) << 4));
          if (cls < C)
            *reinterpret_cast<uint4 *>(W2b + (size_t)cls * H + 8 * c8) =
                make_uint4(pack_bf16x2(a.x, a.y), pack_bf16x2(a.z, a.w), pack_bf16x2(b.x, b.y),
                           pack_bf16x2(b.z, b.w));
        }
        named_bar(3, 128);                    // every thread's reads of the block are done
#endif
#endif
        if (ut == 0) {
#ifndef AS_X_NOUPD
          bulk_wait_read0();
#endif
          if (kb + 1 < NB) {
            mbar_expect_tx(wf_full, BM * H * 4);
            for (int c = 0; c < 4; ++c)
              tma_load_2d(&mapWf, wf_full, (uint8_t *)sT + c * 16384, c * 32, (cb + gridDim.x) * BM);
          }
        }
      } else {
        if (last_smem) {
          // fp32 block [128 classes][H] as H / 32 swizzled boxes of 32 columns in the
          // H stages (free: every MMA of the CTA has completed), updated in place
          // from the accumulator (lane i = class i), TMA-stored, bf16 shadow written
          // coalesced from the boxes
          // box c (32 columns): W2S -- half c / 4 in the stage the producer
          // filled after the H tiles; else both stages, loaded here
          auto box = [&](int c) -> uint8_t * {
            if constexpr (W2S) {
              constexpr int BPS = TILE / 16384;
              return sHt + ((NB * RT + c / BPS) % NSH) * TILE + (c % BPS) * 16384;
            }
            else return sHt + c * 16384;
          };
          if (!W2S && ut == 0) {
            mbar_expect_tx(wf_full, BM * H * 4);
            for (int c = 0; c < NCH; ++c) tma_load_2d(&mapWf, wf_full, box(c), c * 32, cb * BM);
          }
          const uint32_t sw = (uint32_t)(i & 7);
          const int cls_i = cb * BM + i;
          if (!W2S) mbar_wait(wf_full, 0u);   // used once per CTA at h = 256
          // chunk c + 1's accumulator columns load while chunk c is applied
          auto apply = [&](int ch, const uint32_t (&r)[32]) {
            if (ch == NCH - 1) {
              fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(dw_empty);
            }
            if (W2S && (ch & 3) == 0) mbar_wait(&wf2[ch >> 2], 0u);
            uint8_t *rowWf = box(ch) + i * 128;
#pragma unroll
            for (int g0 = 0; g0 < 8; g0 += 4) {
              float4 w[4];
#pragma unroll
              for (int g = 0; g < 4; ++g) w[g] = *reinterpret_cast<const float4 *>(rowWf + (((uint32_t)(g0 + g) ^ sw) << 4));
#pragma unroll
              for (int g = 0; g < 4; ++g) {
                w[g].x = fmaf(-lr, __uint_as_float(r[4 * (g0 + g)]), w[g].x);
                w[g].y = fmaf(-lr, __uint_as_float(r[4 * (g0 + g) + 1]), w[g].y);
                w[g].z = fmaf(-lr, __uint_as_float(r[4 * (g0 + g) + 2]), w[g].z);
                w[g].w = fmaf(-lr, __uint_as_float(r[4 * (g0 + g) + 3]), w[g].w);
              }
#pragma unroll
              for (int g = 0; g < 4; ++g) *reinterpret_cast<float4 *>(rowWf + (((uint32_t)(g0 + g) ^ sw) << 4)) = w[g];
              if constexpr (W2S) {
                // bf16 shadow of these 16 columns into the (now idle) W2T tile, its
                // K-major SW128 layout: atom ch / 2, 16-byte chunk (ch & 1) 4 + g0 / 2 + jj
#pragma unroll
                for (int jj = 0; jj < 2; ++jj) {
                  const uint32_t j = (uint32_t)((ch & 1) * 4 + g0 / 2 + jj);
                  *reinterpret_cast<uint4 *>(sW2 + (ch >> 1) * ATOM_BYTES + i * 128 + ((j ^ sw) << 4)) =
                      make_uint4(pack_bf16x2(w[2 * jj].x, w[2 * jj].y), pack_bf16x2(w[2 * jj].z, w[2 * jj].w),
                                 pack_bf16x2(w[2 * jj + 1].x, w[2 * jj + 1].y),
                                 pack_bf16x2(w[2 * jj + 1].z, w[2 * jj + 1].w));
                }
              }
            }
            if (dbg_dW2T && cls_i < C) {
#pragma unroll
              for (int k = 0; k < 32; ++k) dbg_dW2T[(size_t)cls_i * H + ch * 32 + k] = __uint_as_float(r[k]);
            }
          };
          uint32_t ra[32], rb[32];
          AS_TMEM_LD32(tl + COL_DW, ra);
          AS_TMEM_WAIT_LD(ra);
#pragma unroll 1
          for (int ch = 0; ch < NCH; ch += 2) {   // NCH even
            AS_TMEM_LD32(tl + COL_DW + (ch + 1) * 32, rb);
            apply(ch, ra);
            AS_TMEM_WAIT_LD(rb);
            if (ch + 2 < NCH) AS_TMEM_LD32(tl + COL_DW + (ch + 2) * 32, ra);
            apply(ch + 1, rb);
            if (ch + 2 < NCH) AS_TMEM_WAIT_LD(ra);
          }
          fence_proxy_async();
          named_bar(3, 128);
          if (ut == 0) {
            for (int c = 0; c < NCH; ++c) tma_store_2d(&mapWf, box(c), c * 32, cb * BM);
            if constexpr (W2S)                // the bf16 shadow too, from the W2T tile
              for (int a = 0; a < H / 64; ++a) tma_store_2d(&mapW, sW2 + a * ATOM_BYTES, a * 64, cb * BM);
            bulk_commit();
          }
          // bf16 shadow: H / 8 segments of 8 columns per class row, coalesced
          constexpr int SEGS = H / 8;
#pragma unroll 4
          for (int k = 0; k < (W2S ? 0 : SEGS); ++k) {
            const int idx = k * 128 + ut;
            const int row = idx / SEGS, c8 = idx % SEGS;
            const int cls = cb * BM + row;
            const uint8_t *rb = box(c8 >> 2) + row * 128;
            const uint32_t g0 = (uint32_t)((c8 & 3) * 2), rs = (uint32_t)(row & 7);
            const float4 a = *reinterpret_cast<const float4 *>(rb + ((g0 ^ rs) << 4));
            const float4 b = *reinterpret_cast<const float4 *>(rb + (((g0 + 1) ^ rs) << 4));
            if (cls < C)
              *reinterpret_cast<uint4 *>(W2b + (size_t)cls * H + 8 * c8) =
                  make_uint4(pack_bf16x2(a.x, a.y), pack_bf16x2(a.z, a.w), pack_bf16x2(b.x, b.y),
                             pack_bf16x2(b.z, b.w));
          }
          if (!W2S && ut == 0) bulk_wait0();  // the stores have left the H stages (W2S: at the end)
        } else {
        // chunked staging (h = 256): the accumulator is released after the last chunk
#pragma unroll 1
        for (int ch = 0; ch < NCH; ++ch) {
          uint32_t r[32];
          AS_TMEM_LD32(tl + COL_DW + ch * 32, r);
          AS_TMEM_WAIT_LD(r);
          if (ch == NCH - 1) {
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(dw_empty);
          }
          named_bar(3, 128);
#pragma unroll
          for (int k = 0; k < 32; k += 4)
            *reinterpret_cast<float4 *>(sT + i * SROW + k) =
                make_float4(__uint_as_float(r[k]), __uint_as_float(r[k + 1]),
                            __uint_as_float(r[k + 2]), __uint_as_float(r[k + 3]));
          named_bar(3, 128);
          float4 wn[TMAUPD ? 1 : 8];
          if (ch + 1 < NCH) ld_chunk(ch + 1, wn);
#pragma unroll
          for (int m = 0; m < 8; ++m) {
            const int cl = q * 32 + 4 * m + sub;
            const int cls = cb * BM + cl;
            if (cls < C) {
              const float4 gv = *reinterpret_cast<const float4 *>(sT + cl * SROW + hq);
              const size_t idx = (size_t)cls * H + ch * 32 + hq;
              float4 nw = wq[TMAUPD ? 0 : m];
              nw.x -= lr * gv.x; nw.y -= lr * gv.y; nw.z -= lr * gv.z; nw.w -= lr * gv.w;
              *reinterpret_cast<float4 *>(W2T + idx) = nw;
              *reinterpret_cast<uint2 *>(W2b + idx) = make_uint2(pack_bf16x2(nw.x, nw.y),
                                                                 pack_bf16x2(nw.z, nw.w));
              if (dbg_dW2T) *reinterpret_cast<float4 *>(dbg_dW2T + idx) = gv;
            }
          }
#pragma unroll
          for (int m = 0; m < (TMAUPD ? 1 : 8); ++m) wq[m] = wn[m];
        }
        }
        if (!W2S && kb + NWT < NB) load_wt(kb + NWT);
      }
      // db2 (thread ut = class ut of the block; label term already in G), SGD on b2
      TRACE(3, ut == 0, 13, kb);
      mbar_wait_sleepy(db_full, kb & 1, 128);
      const float dsum = sDB[ut] + sDB[BM + ut];
      named_bar(3, 128);
      if (lane == 0) mbar_arrive(db_empty);
      const int c = cb * BM + ut;
      if (c < C) {
        b2[c] -= lr * dsum;
        if (dbg_db2) dbg_db2[c] = dsum;
      }
      TRACE(3, ut == 0, 14, kb);
    }
    if ((TMAUPD || W2S) && ut == 0) bulk_wait0();   // stores complete before the grid ends
  } else if (H == 128 && dw.W1) {           // warps 14-15: step a7 (dW1 + SGD) alongside
    AS_REG_DEC2();
    // First-layer gradient with fused SGD on the feature-sorted entries (a3's
    // transpose): warp gw of the grid's 2 * gridDim.x takes segments gw, gw +
    // GW, ...; dW1[f] = sum over the segment's entries, in entry order, of
    // v * dA[row] (lane = 4 consecutive of the h columns), W1[f] -= lr dW1[f].
    // Independent of pass 2's data (W2T, b2) and hidden inside its runtime;
    // deterministic (one warp per segment, fixed order).
    constexpr int V = H / 128;
    const int gw = blockIdx.x * 2 + (warp - 14), GW = gridDim.x * 2;
    const int U = dw.desc->U;
    for (int sg = gw; sg < U; sg += GW) {
      const int p0 = dw.seg_ptr[sg], p1 = dw.seg_ptr[sg + 1];
      const int f = dw.seg_key[sg];
      float4 *w1 = reinterpret_cast<float4 *>(dw.W1 + (size_t)f * H);
      float4 wv[V];
#pragma unroll
      for (int q = 0; q < V; ++q) wv[q] = w1[lane + 32 * q];      // in flight during the sums
      float4 acc[V];
#pragma unroll
      for (int q = 0; q < V; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      int e = p0;
      for (; e + 4 <= p1; e += 4) {             // four entries' rows in flight
        int r[4];
        float v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { r[u] = dw.seg_row[e + u]; v[u] = dw.seg_val[e + u]; }
        float4 d[4][V];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int q = 0; q < V; ++q) d[u][q] = reinterpret_cast<const float4 *>(dw.dA + (size_t)r[u] * H)[lane + 32 * q];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int q = 0; q < V; ++q) {
            acc[q].x = fmaf(v[u], d[u][q].x, acc[q].x); acc[q].y = fmaf(v[u], d[u][q].y, acc[q].y);
            acc[q].z = fmaf(v[u], d[u][q].z, acc[q].z); acc[q].w = fmaf(v[u], d[u][q].w, acc[q].w);
          }
      }
      for (; e < p1; ++e) {
        const int r = dw.seg_row[e];
        const float v = dw.seg_val[e];
#pragma unroll
        for (int q = 0; q < V; ++q) {
          const float4 d = reinterpret_cast<const float4 *>(dw.dA + (size_t)r * H)[lane + 32 * q];
          acc[q].x = fmaf(v, d.x, acc[q].x); acc[q].y = fmaf(v, d.y, acc[q].y);
          acc[q].z = fmaf(v, d.z, acc[q].z); acc[q].w = fmaf(v, d.w, acc[q].w);
        }
      }
#pragma unroll
      for (int q = 0; q < V; ++q) {
        float4 w = wv[q];
        w.x -= dw.lr * acc[q].x; w.y -= dw.lr * acc[q].y; w.z -= dw.lr * acc[q].z; w.w -= dw.lr * acc[q].w;
        w1[lane + 32 * q] = w;
        if (dw.dbg) reinterpret_cast<float4 *>(dw.dbg + (size_t)sg * H)[lane + 32 * q] = acc[q];
      }
    }
  } else {                                    // warps 14-15: idle
    AS_REG_DEC2();
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == kMmaWarp) tmem_dealloc(tmem, 512);
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


// =====================================================================
// micro-benchmark of tcgen05 issue rates for the operand layouts used above
// (tests/tools only): one CTA, `iters` groups of 128x128x128 (or 128x256x128)
// bf16 MMAs accumulated into TMEM; returns elapsed SM cycles.
//   mode 0: A K-major,  B K-major,  N = 128     (S tiles)
//   mode 1: A MN-major, B K-major,  N = 128     (dW of pass 2)
//   mode 2: A K-major,  B MN-major, N = 128     (O of pass 1)
//   mode 3: A K-major,  B K-major,  N = 256
//   mode 4: A from TMEM, B K-major,  N = 128     (S of pass 1)
//   mode 5: A from TMEM, B MN-major, N = 128     (O of pass 1, dW of pass 2)
// =====================================================================
__global__ void __launch_bounds__(128, 1) k_tc_bench(int mode, int iters, long long *out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint64_t *bar = (uint64_t *)(smem_raw + 4 * 32768);
  uint32_t *slot = (uint32_t *)(bar + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = threadIdx.x; k < 4 * 32768 / 4; k += blockDim.x) ((uint32_t *)smem_raw)[k] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_proxy_async();
  if (warp == 0) tmem_alloc(slot, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *slot;
  if (warp == 0 && mode >= 6) {
    // warp-converged issue (all lanes), elect inside the asm
    const uint32_t aA = smem_u32(smem_raw), aB = aA + 65536;
    const uint64_t dA = sdesc(aA, 16, 1024), dB = sdesc(aB, 16, 1024);
    const uint32_t id = idesc_bf16(128, 128, 0, 0);
    const long long t0 = clock64();
    if (mode == 6)
      for (int it = 0; it < iters; ++it) mma_grp_ss_kk_8(tmem, dA, dB, id, it > 0);
    else if (mode == 7)
      for (int it = 0; it < iters; ++it) mma_grp_ts_k_8(tmem, tmem + 256, dB, id, it > 0);
    else if (mode == 8)   // S unit of pass 2: TS, B K-major, N = 64 (x2 per group)
      for (int it = 0; it < iters; ++it) {
        mma_grp_ts_k_8(tmem, tmem + 256, dB, idesc_bf16(128, 64, 0, 0), it > 0);
        mma_grp_ts_k_8(tmem + 64, tmem + 256, dB + 512, idesc_bf16(128, 64, 0, 0), it > 0);
      }
    else if (mode == 9)   // dW unit of pass 2: TS, B MN-major, N = 128, K = 64 (x2 per group)
      for (int it = 0; it < iters; ++it) {
        const uint64_t dBm = sdesc(aB, ATOM_BYTES, 1024);
        mma_grp_ts_mn_4(tmem + 128, tmem + 256, dBm, idesc_bf16(128, 128, 0, 1), it > 0);
        mma_grp_ts_mn_4(tmem + 128, tmem + 288, dBm + 512, idesc_bf16(128, 128, 0, 1), 1u);
      }
    else if (mode == 11 || mode == 12)
      // pass-2 order: dW(u) reads G^T from buffer u % 4, then S(u + 4) is written
      // to buffer u % 4 (mode 11: adjacent WAR on TMEM) or to buffer (u + 2) % 4
      // (mode 12); per iteration two 64-row units
      for (int it = 0; it < 2 * iters; ++it) {
        const uint64_t dBm = sdesc(aB, ATOM_BYTES, 1024);
        const uint32_t rb = (it & 3) * 64, wb = mode == 11 ? rb : ((it + 2) & 3) * 64;
        mma_grp_ts_mn_4(tmem + 384, tmem + rb, dBm, idesc_bf16(128, 128, 0, 1), it > 0);
        mma_grp_ts_k_8(tmem + wb, tmem + 256, dB, idesc_bf16(128, 64, 0, 0), 0u);
      }
    else if (mode == 13 || mode == 14)
      // pass-1 order: O(j) reads P from buffer j % 2, then S(j + 2) is written to
      // buffer j % 2 (mode 13) / a third buffer (mode 14); per iteration one block
      for (int it = 0; it < iters; ++it) {
        const uint64_t dBm = sdesc(aB, ATOM_BYTES, 1024);
        const uint32_t rb = (it & 1) * 128, wb = mode == 13 ? rb : 256;
        mma_grp_ts_mn_8(tmem + 384, tmem + rb, dBm, idesc_bf16(128, 128, 0, 1), it > 0);
        mma_grp_ss_kk_8(tmem + wb, dA, dB, idesc_bf16(128, 128, 0, 0), 0u);
      }
    else   // mode 10: both of the above (one 128-row tile of pass 2)
      for (int it = 0; it < iters; ++it) {
        const uint64_t dBm = sdesc(aB, ATOM_BYTES, 1024);
        mma_grp_ts_k_8(tmem, tmem + 256, dB, idesc_bf16(128, 64, 0, 0), it > 0);
        mma_grp_ts_mn_4(tmem + 128, tmem + 320, dBm, idesc_bf16(128, 128, 0, 1), it > 0);
        mma_grp_ts_k_8(tmem + 64, tmem + 256, dB + 512, idesc_bf16(128, 64, 0, 0), it > 0);
        mma_grp_ts_mn_4(tmem + 128, tmem + 384, dBm + 512, idesc_bf16(128, 128, 0, 1), 1u);
      }
    mma_commit_w(bar);
    mbar_wait(bar, 0);
    if (lane == 0) out[0] = clock64() - t0;
  } else if (warp == 0 && lane == 0) {
    const uint32_t aA = smem_u32(smem_raw), aB = aA + 65536;
    const uint32_t id = mode == 1 ? idesc_bf16(128, 128, 1, 0)
                        : (mode == 2 || mode == 5) ? idesc_bf16(128, 128, 0, 1)
                        : mode == 3 ? idesc_bf16(128, 256, 0, 0) : idesc_bf16(128, 128, 0, 0);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t a = mode == 1 ? desc_mn(aA, kk) : desc_k(aA, kk);
        const uint64_t b = (mode == 2 || mode == 5) ? desc_mn(aB, kk) : desc_k(aB, kk);
        if (mode >= 4)
          mma_bf16_ts(tmem, tmem + 256 + 8 * kk, b, id, (it | kk) ? 1u : 0u);
        else
          mma_bf16(tmem, a, b, id, (it | kk) ? 1u : 0u);
      }
    }
    mma_commit(bar);
    mbar_wait(bar, 0);
    out[0] = clock64() - t0;
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// self-test of the TMEM-A ("TS") MMA (tests only), one CTA, 128 threads:
//   thread r writes row r of A (bf16) into TMEM columns [256, 320) packed,
//   and row r of P = bf16(A/4) likewise into [320, 384);
//   V = A_tmem . B^T (B K-major)   -> TMEM cols [0, 128)
//   U = P_tmem . B   (B MN-major)  -> TMEM cols [128, 256)
__global__ void __launch_bounds__(128, 1)
    k_tc_selftest2(const __grid_constant__ CUtensorMap mapB, const __nv_bfloat16 *__restrict__ A,
                   float *__restrict__ V, float *__restrict__ U) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *sB = smem_raw;
  uint64_t *bars = (uint64_t *)(sB + 32768);
  uint64_t *ld_full = bars, *mma_done = bars + 1;
  uint32_t *slot = (uint32_t *)(bars + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(ld_full, 1); mbar_init(mma_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(slot, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *slot;
  const int row = warp * 32 + lane;
  const uint32_t tl = tmem + ((uint32_t)(warp * 32) << 16);
  // rows of A and P into TMEM (two bf16 per column, even k in the low half)
  for (int ch = 0; ch < 2; ++ch) {
    uint32_t ra[32], rp[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const int k = 64 * ch + 2 * c;
      const float a0 = __bfloat162float(A[row * 128 + k]), a1 = __bfloat162float(A[row * 128 + k + 1]);
      ra[c] = pack_bf16x2(a0, a1);
      rp[c] = pack_bf16x2(a0 * 0.25f, a1 * 0.25f);
    }
    AS_TMEM_ST32(tl + 256 + 32 * ch, ra);
    AS_TMEM_ST32(tl + 320 + 32 * ch, rp);
  }
  tmem_wait_st();
  fence_before();
  __syncthreads();
  fence_after();
  if (threadIdx.x == 0) {
    mbar_expect_tx(ld_full, 32768);
    for (int a = 0; a < 2; ++a) tma_load_2d(&mapB, ld_full, sB + a * ATOM_BYTES, a * 64, 0);
    mbar_wait(ld_full, 0);
    fence_after();
    const uint32_t aB = smem_u32(sB);
    for (int kk = 0; kk < 8; ++kk)
      mma_bf16_ts(tmem, tmem + 256 + 8 * kk, desc_k(aB, kk), idesc_bf16(128, 128, 0, 0), kk > 0);
    for (int kk = 0; kk < 8; ++kk)
      mma_bf16_ts(tmem + 128, tmem + 320 + 8 * kk, desc_mn(aB, kk), idesc_bf16(128, 128, 0, 1), kk > 0);
    mma_commit(mma_done);
  }
  mbar_wait(mma_done, 0);
  fence_after();
  for (int ch = 0; ch < 4; ++ch) {
    uint32_t r[32];
    AS_TMEM_LD32(tl + ch * 32, r);
    AS_TMEM_WAIT_LD(r);
    for (int k = 0; k < 32; ++k) V[row * 128 + ch * 32 + k] = __uint_as_float(r[k]);
    AS_TMEM_LD32(tl + 128 + ch * 32, r);
    AS_TMEM_WAIT_LD(r);
    for (int k = 0; k < 32; ++k) U[row * 128 + ch * 32 + k] = __uint_as_float(r[k]);
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// =====================================================================
// top-1 evaluation ("top-1 accuracy –
// corresponding to the class with the highest probability"): the forward
// logits z = H W2T^T + b2 of a 128-row tile against this CTA's class blocks
// and, per row, max_c z_c with the LOWEST class id on ties (R21; softmax is
// monotone, so no exponentials).  Same split of the class range as pass 1;
// partial slot (sp, g) = 2 sp + g holds (max, argmax) of WG g's blocks.
//   warps 0-7  two epilogue warpgroups, WG g takes the blocks j % 2 == g and
//              reads S_j from TMEM buffer g (thread = row = TMEM lane)
//   warp 8     TMA producer (H tile once, W2T class blocks through a ring)
//   warp 9     MMA issuer: S_j = H . W2T_blk^T into buffer j % 2
// =====================================================================
template <int H>
struct Top1Cfg {
  static constexpr int NST = H == 128 ? 4 : 2;
  static constexpr int TILE = BM * H * 2;
  static constexpr int THREADS = 10 * 32;
  static constexpr int SMEM = TILE + NST * TILE + 2 * BM * 4 /*b2 of the current block per WG*/ + 256;
  static_assert(SMEM <= 232448, "top-1 shared memory exceeds 227 KB");
};

template <int H>
__global__ void __launch_bounds__(Top1Cfg<H>::THREADS, 1)
    k_out_top1(const __grid_constant__ CUtensorMap mapH, const __grid_constant__ CUtensorMap mapW,
               const StepDesc *__restrict__ desc, const float *__restrict__ b2, int C, int n_cblocks,
               int max_splits, int bpad, float *__restrict__ pmax, int *__restrict__ pidx) {
  using Cfg = Top1Cfg<H>;
  constexpr int NST = Cfg::NST, TILE = Cfg::TILE;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *sH = smem_raw;
  uint8_t *sW = smem_raw + TILE;
  float *sB2 = (float *)(sW + NST * TILE);          // [2 WG][128]
  uint64_t *bars = (uint64_t *)(sB2 + 2 * BM);
  uint64_t *h_full = bars, *w_full = bars + 1, *w_empty = w_full + NST, *s_full = w_empty + NST,
           *s_empty = s_full + 2;
  uint32_t *tmem_slot = (uint32_t *)(s_empty + 2);
  if ((smem_u32(smem_raw) & 1023u) != 0) __trap();

  const int B = desc->rows;
  const int RT = (B + BM - 1) / BM;
  const int splits = fwd_splits(B, n_cblocks, gridDim.x, max_splits);
  const int rt = blockIdx.x / splits, sp = blockIdx.x % splits;
  if (rt >= RT) return;
  const int cb0 = (int)((long long)sp * n_cblocks / splits);
  const int nloc = (int)((long long)(sp + 1) * n_cblocks / splits) - cb0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kProdWarp = 8, kMmaWarp = 9;

  if (threadIdx.x == 0) {
    mbar_init(h_full, 1);
    for (int i = 0; i < NST; ++i) { mbar_init(&w_full[i], 1); mbar_init(&w_empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&s_full[i], 1); mbar_init(&s_empty[i], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) tmem_alloc(tmem_slot, 256);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kProdWarp) {
    if (lane == 0) {
      mbar_expect_tx(h_full, TILE);
      for (int a = 0; a < H / 64; ++a) tma_load_2d(&mapH, h_full, sH + a * ATOM_BYTES, a * 64, rt * BM);
      for (int j = 0; j < nloc; ++j) {
        const int st = j % NST;
        if (j >= NST) mbar_wait_idle(&w_empty[st], ((j / NST) - 1) & 1);
        mbar_expect_tx(&w_full[st], TILE);
        for (int a = 0; a < H / 64; ++a)
          tma_load_2d(&mapW, &w_full[st], sW + st * TILE + a * ATOM_BYTES, a * 64, (cb0 + j) * BM);
      }
    }
  } else if (warp == kMmaWarp) {
    constexpr uint32_t idS = idesc_bf16(BM, BM, 0, 0);
    const uint32_t aH = smem_u32(sH), aW = smem_u32(sW);
    mbar_wait(h_full, 0);
    fence_after();
    const uint64_t dH = sdesc(aH, 16, 1024);
    for (int j = 0; j < nloc; ++j) {
      const int st = j % NST, b = j & 1;
      if (j >= 2) mbar_wait(&s_empty[b], ((j >> 1) - 1) & 1);
      mbar_wait(&w_full[st], (j / NST) & 1);
      fence_after();
      if constexpr (H == 128)
        mma_grp_ss_kk_8(tmem + b * BM, dH, sdesc(aW + st * TILE, 16, 1024), idS, 0u);
      else
        mma_grp_ss_kk_16(tmem + b * BM, dH, sdesc(aW + st * TILE, 16, 1024), idS, 0u);
      mma_commit_w(&s_full[b]);
      mma_commit_w(&w_empty[st]);
    }
  } else {  // ---------------- epilogue warpgroups (thread = row)
    const int g = warp >> 2, q = warp & 3;
    const int row = q * 32 + lane;
    const uint32_t tS = tmem + ((uint32_t)(q * 32) << 16) + g * BM;
    float best = -INFINITY;
    int bi = 0x7fffffff;
    int jj = 0;
    for (int j = g; j < nloc; j += 2, ++jj) {
      const int c0 = (cb0 + j) * BM;
      float *myB2 = sB2 + g * BM;
      named_bar(1 + g, 128);                  // previous block's b2 reads are done
      myB2[row] = c0 + row < C ? b2[c0 + row] : -INFINITY;   // class past C: never selected
      named_bar(1 + g, 128);
      mbar_wait(&s_full[g], jj & 1);
      fence_after();
#pragma unroll 1
      for (int ch = 0; ch < BM / 32; ++ch) {
        uint32_t r[32];
        AS_TMEM_LD32(tS + ch * 32, r);
        AS_TMEM_WAIT_LD(r);
        if (ch == BM / 32 - 1) {
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&s_empty[g]);
        }
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const float z = __uint_as_float(r[k]) + myB2[ch * 32 + k];
          if (z > best) { best = z; bi = c0 + ch * 32 + k; }   // ascending c: lowest id on ties
        }
      }
    }
    const size_t slot = (size_t)sp * 2 + g;
    const int grow = rt * BM + row;
    pmax[slot * bpad + grow] = best;
    pidx[slot * bpad + grow] = bi;
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == kMmaWarp) tmem_dealloc(tmem, 256);
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
static int make_map(CUtensorMap *m, const void *base, long long rows, int cols, int box_rows = 128) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return -1;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

struct TcPlan {
  CUtensorMap mapH, mapW, mapWf, mapHx, mapH64;   // mapH64: 64-row H boxes (one-block pass 2 at h = 256)
  const void *Hb;
  int h, b_max, bpad, n_cblocks, num_sms, max_splits;
  long long C;
};

size_t tc_plan_bytes() { return sizeof(TcPlan); }

int tc_splits(int h, int b_max, long long C, int num_sms) {
  (void)h; (void)b_max;
  const int ncb = (int)((C + tc::BM - 1) / tc::BM);
  return num_sms < ncb ? num_sms : ncb;   // capacity of the partial buffers
}

// fp32 row-major [rows][cols] with a {32, 128} box (128-byte rows) and 128-byte swizzle
static int make_map_f32(CUtensorMap *m, const void *base, long long rows, int cols) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return -1;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {32, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(base), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

// bf16 row-major [rows][16] (the FOLD B_ext rows) with a {16, 128} box and 32-byte swizzle
static int make_map_x(CUtensorMap *m, const void *base, long long rows) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return -1;
  cuuint64_t dims[2] = {16, (cuuint64_t)rows};
  cuuint64_t strides[1] = {32};
  cuuint32_t box[2] = {16, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

bool tc_fold(int h) { return h == 128 ? tc::BwdCfg<128>::FOLD : tc::BwdCfg<256>::FOLD; }

int tc_plan_init(TcPlan *plan, int h, int b_max, long long C, int num_sms, const void *Hb,
                 const void *W2b, const void *W2T, const void *Hx) {
  plan->h = h;
  plan->Hb = Hb;
  plan->b_max = b_max;
  plan->bpad = (b_max + tc::BM - 1) / tc::BM * tc::BM;
  plan->C = C;
  plan->n_cblocks = (int)((C + tc::BM - 1) / tc::BM);
  plan->num_sms = num_sms < 160 ? num_sms : 160;   // partial buffers sized for 160
  plan->max_splits = tc_splits(h, b_max, C, plan->num_sms);
  if (make_map(&plan->mapH, Hb, plan->bpad, h) != 0) return -1;
  if (make_map(&plan->mapH64, Hb, plan->bpad, h, 64) != 0) return -1;
  if (make_map(&plan->mapW, W2b, C, h) != 0) return -1;
  if (make_map_f32(&plan->mapWf, W2T, C, h) != 0) return -1;
  if (make_map_x(&plan->mapHx, Hx, plan->bpad) != 0) return -1;
  // every ctx sets the attributes on its own device (cheap, idempotent)
  {
    if (h == 128) {
      cudaFuncSetAttribute(tc::k_out_fwd<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           tc::FwdCfg<128>::SMEM);
      cudaFuncSetAttribute(tc::k_out_bwd<128, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           tc::BwdCfg<128>::SMEM);
      cudaFuncSetAttribute(tc::k_out_top1<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           tc::Top1Cfg<128>::SMEM);
    } else {
      cudaFuncSetAttribute(tc::k_out_fwd<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           tc::FwdCfg<256>::SMEM);
      cudaFuncSetAttribute(tc::k_out_bwd<256, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           tc::BwdCfg<256>::SMEM);
      cudaFuncSetAttribute(tc::k_out_bwd<256, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           tc::BwdCfg<256, true>::SMEM);
      cudaFuncSetAttribute(tc::k_out_top1<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           tc::Top1Cfg<256>::SMEM);
    }
  }
  return 0;
}

// pass-1 / top-1 grid: one CTA per SM, or one per 128-row tile when the
// batch has more tiles than SMs (b_max > 128 * num_sms; the CTAs then run in
// several waves with one class split each)
static int fwd_grid(const TcPlan *p) {
  const int rt = p->bpad / tc::BM;
  return rt > p->num_sms ? rt : p->num_sms;
}

void launch_out_fwd_tc(cudaStream_t s, const TcPlan *p, const StepDesc *desc, const float *b2,
                       float *pm, float *pl, float *pO, const LtArgs &lt) {
  if (p->h == 128)
    launch_pdl(tc::k_out_fwd<128>, dim3(fwd_grid(p)), dim3(tc::FwdCfg<128>::THREADS), tc::FwdCfg<128>::SMEM, s,
               p->mapH, p->mapW, desc, (const __nv_bfloat16 *)p->Hb, b2, (int)p->C, p->n_cblocks,
               p->max_splits, p->bpad, pm, pl, pO, lt);
  else
    launch_pdl(tc::k_out_fwd<256>, dim3(fwd_grid(p)), dim3(tc::FwdCfg<256>::THREADS), tc::FwdCfg<256>::SMEM, s,
               p->mapH, p->mapW, desc, (const __nv_bfloat16 *)p->Hb, b2, (int)p->C, p->n_cblocks,
               p->max_splits, p->bpad, pm, pl, pO, lt);
}

void launch_out_top1_tc(cudaStream_t s, const TcPlan *p, const StepDesc *desc, const float *b2, float *pmax,
                        int *pidx) {
  if (p->h == 128)
    tc::k_out_top1<128><<<fwd_grid(p), tc::Top1Cfg<128>::THREADS, tc::Top1Cfg<128>::SMEM, s>>>(
        p->mapH, p->mapW, desc, b2, (int)p->C, p->n_cblocks, p->max_splits, p->bpad, pmax, pidx);
  else
    tc::k_out_top1<256><<<fwd_grid(p), tc::Top1Cfg<256>::THREADS, tc::Top1Cfg<256>::SMEM, s>>>(
        p->mapH, p->mapW, desc, b2, (int)p->C, p->n_cblocks, p->max_splits, p->bpad, pmax, pidx);
}

// number of pass-1 partial slots for a batch of B rows (one per CTA split)
int tc_fwd_splits_host(const TcPlan *p, int B) {
  return tc::fwd_splits(B, p->n_cblocks, fwd_grid(p), p->max_splits);
}

bool tc_fuses_dw1(int h) { return h == 128; }

void launch_out_bwd_tc(cudaStream_t s, const TcPlan *p, const StepDesc *desc, const float *lsep,
                       const int4 *cls_lab, const uint32_t *lbits, int lbw, const float *wrow, float *W2T,
                       float *b2, __nv_bfloat16 *W2b, float lr, float *dbg_dW2T, float *dbg_db2,
                       const Dw1Args &dw) {
  const int grid = p->num_sms < p->n_cblocks ? p->num_sms : p->n_cblocks;
  if (p->h == 128)
    // plain launch: pass 2 follows the wait on the transposes' join event
    tc::k_out_bwd<128, false><<<grid, tc::BwdCfg<128>::THREADS, tc::BwdCfg<128>::SMEM, s>>>(
        p->mapH, p->mapW, p->mapWf, p->mapHx, desc, lsep, (int)p->C, p->n_cblocks, cls_lab, lbits, lbw, wrow, W2T,
        b2, W2b, lr, dbg_dW2T, dbg_db2, dw);
  else if (p->n_cblocks <= grid)             // one class block per CTA (AmazonCat-13K)
    tc::k_out_bwd<256, true><<<grid, tc::BwdCfg<256, true>::THREADS, tc::BwdCfg<256, true>::SMEM, s>>>(
        tc::BwdCfg<256, true>::TR == 64 ? p->mapH64 : p->mapH, p->mapW, p->mapWf, p->mapHx, desc, lsep, (int)p->C, p->n_cblocks, cls_lab, lbits, lbw, wrow, W2T,
        b2, W2b, lr, dbg_dW2T, dbg_db2, dw);
  else
    tc::k_out_bwd<256, false><<<grid, tc::BwdCfg<256>::THREADS, tc::BwdCfg<256>::SMEM, s>>>(
        p->mapH, p->mapW, p->mapWf, p->mapHx, desc, lsep, (int)p->C, p->n_cblocks, cls_lab, lbits, lbw, wrow, W2T,
        b2, W2b, lr, dbg_dW2T, dbg_db2, dw);
}

int tc_trace_dump(long long *out, int max_events) {
#ifdef AS_TRACE
  int n[4] = {0, 0, 0, 0};
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(n, tc::g_trace_n, sizeof(n));
  static long long buf[4][4096][3];
  cudaMemcpyFromSymbol(buf, tc::g_trace, sizeof(buf));
  int k = 0;
  for (int r = 0; r < 4; ++r)
    for (int i = 0; i < n[r] && k < max_events; ++i, ++k) {
      out[3 * k] = buf[r][i][0];
      out[3 * k + 1] = buf[r][i][1];
      out[3 * k + 2] = buf[r][i][2];
    }
  const int z[4] = {0, 0, 0, 0};
  cudaMemcpyToSymbol(tc::g_trace_n, z, sizeof(z));
  return k;
#else
  (void)out; (void)max_events;
  return 0;
#endif
}

int tc_selftest2(const void *A, const void *B, float *V, float *U, cudaStream_t s) {
  CUtensorMap mB;
  if (make_map(&mB, B, 128, 128) != 0) return -1;
  const int smem = 32768 + 1024;
  cudaFuncSetAttribute(tc::k_tc_selftest2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  tc::k_tc_selftest2<<<1, 128, smem, s>>>(mB, (const __nv_bfloat16 *)A, V, U);
  return 0;
}

int tc_bench(int mode, int iters, long long *cycles_host) {
  long long *d = nullptr;
  cudaMalloc(&d, 8);
  const int smem = 4 * 32768 + 1024;
  cudaFuncSetAttribute(tc::k_tc_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  tc::k_tc_bench<<<1, 128, smem>>>(mode, iters, d);
  const cudaError_t e = cudaMemcpy(cycles_host, d, 8, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e == cudaSuccess ? 0 : -1;
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

// Micro-benchmark (tools only): throughput of the output-layer softmax
// instruction mix (the pass-2 inner loop without TMEM / shared memory / barriers)
// as a function of the number of warps per SM sub-partition.
//   per pair of elements: x = fma2(s, log2e, b2) ; x = add2(x, -lse)
//                         2 of 3 pairs: two MUFU.EX2;  1 of 3: degree-3 polynomial
//                         db2 += p (add2); G = pack_bf16x2(p)
// Reports cycles per 128-element unit per warp and per sub-partition.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_softmax tools/ubench_softmax.cu
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>

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
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void ex2_emu2(uint64_t x, float &p0, float &p1) {
  float x0, x1;
  f2split(x, x0, x1);
  x = f2(fmaxf(x0, -125.f), fmaxf(x1, -125.f));
  const uint64_t M2 = f2(12582912.f, 12582912.f);
  const uint64_t t = fadd2(x, M2);
  const uint64_t fr = fsub2(x, fsub2(t, M2));
  uint64_t q = ffma2(fr, f2(0.055171321f, 0.055171321f), f2(0.24261054f, 0.24261054f));
  q = ffma2(q, fr, f2(0.69326099f, 0.69326099f));
  q = ffma2(q, fr, f2(0.99992811f, 0.99992811f));
  float t0, t1, q0, q1;
  f2split(t, t0, t1);
  f2split(q, q0, q1);
  p0 = __uint_as_float((__float_as_uint(t0) << 23) + __float_as_uint(q0));
  p1 = __uint_as_float((__float_as_uint(t1) << 23) + __float_as_uint(q1));
}

// one warp processes `units` units of 128 elements per thread (two halves of 64)
#define TLD32(taddr, r) asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];" \
  : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]),"=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31]) : "r"(taddr))
#define TWAITLD(r) asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r[0]),"+r"(r[1]),"+r"(r[2]),"+r"(r[3]),"+r"(r[4]),"+r"(r[5]),"+r"(r[6]),"+r"(r[7]),"+r"(r[8]),"+r"(r[9]),"+r"(r[10]),"+r"(r[11]),"+r"(r[12]),"+r"(r[13]),"+r"(r[14]),"+r"(r[15]),"+r"(r[16]),"+r"(r[17]),"+r"(r[18]),"+r"(r[19]),"+r"(r[20]),"+r"(r[21]),"+r"(r[22]),"+r"(r[23]),"+r"(r[24]),"+r"(r[25]),"+r"(r[26]),"+r"(r[27]),"+r"(r[28]),"+r"(r[29]),"+r"(r[30]),"+r"(r[31]) :: "memory")
#define TST32(taddr, r) asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" \
  :: "r"(taddr), "r"(r[0]),"r"(r[1]),"r"(r[2]),"r"(r[3]),"r"(r[4]),"r"(r[5]),"r"(r[6]),"r"(r[7]),"r"(r[8]),"r"(r[9]),"r"(r[10]),"r"(r[11]),"r"(r[12]),"r"(r[13]),"r"(r[14]),"r"(r[15]),"r"(r[16]),"r"(r[17]),"r"(r[18]),"r"(r[19]),"r"(r[20]),"r"(r[21]),"r"(r[22]),"r"(r[23]),"r"(r[24]),"r"(r[25]),"r"(r[26]),"r"(r[27]),"r"(r[28]),"r"(r[29]),"r"(r[30]),"r"(r[31]) : "memory")

template <int EMU, int TM>   // one pair in EMU on the FMA pipe (0: none); TM: 0 none, 1 ld x32 + st, 2 ld only, 3 st only, 4 ld x64 + st
__global__ void __launch_bounds__(512, 1) k_mix(int units, int active_warps_per_smsp, long long *cyc, uint32_t *sink) {
  const int warp = threadIdx.x >> 5;
  __shared__ uint32_t tslot;
  if (TM > 0 && warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // warp w: TMEM lanes 32 (w % 4), its own 128 columns (w / 4)
  const uint32_t tl = TM > 0 ? tslot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 128) : 0u;
  // warps are spread round-robin over the 4 sub-partitions (warp % 4)
  float s[64];
  for (int k = 0; k < 64; ++k) s[k] = (float)((threadIdx.x * 7 + k * 13) % 97) * 0.01f - 0.5f;
  __shared__ __align__(16) float lse[64];
  if (threadIdx.x < 64) lse[threadIdx.x] = 3.0f + 0.001f * threadIdx.x;
  __syncthreads();
  const float b2c = 0.1f * (threadIdx.x & 7);
  float db2 = 0.f;
  uint32_t acc = 0;
  const bool active = warp / 4 < active_warps_per_smsp;
  const long long t0 = clock64();
  for (int u = 0; u < (active ? units : 0); ++u) {
#pragma unroll 1
    for (int half = 0; half < 2; ++half) {
      if constexpr (TM == 1 || TM == 2) {     // S of this half from TMEM (2 x 32 columns)
        uint32_t ra[32], rb[32];
        TLD32(tl + 64 * half, ra);
        TLD32(tl + 64 * half + 32, rb);
        TWAITLD(ra);
        TWAITLD(rb);
#pragma unroll
        for (int k = 0; k < 32; ++k) { s[k] = __uint_as_float(ra[k]); s[32 + k] = __uint_as_float(rb[k]); }
      }
      if constexpr (TM == 4) {                // one x64 load
        uint32_t ra[64];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
                     : "=r"(ra[0]),"=r"(ra[1]),"=r"(ra[2]),"=r"(ra[3]),"=r"(ra[4]),"=r"(ra[5]),"=r"(ra[6]),"=r"(ra[7]),"=r"(ra[8]),"=r"(ra[9]),"=r"(ra[10]),"=r"(ra[11]),"=r"(ra[12]),"=r"(ra[13]),"=r"(ra[14]),"=r"(ra[15]),"=r"(ra[16]),"=r"(ra[17]),"=r"(ra[18]),"=r"(ra[19]),"=r"(ra[20]),"=r"(ra[21]),"=r"(ra[22]),"=r"(ra[23]),"=r"(ra[24]),"=r"(ra[25]),"=r"(ra[26]),"=r"(ra[27]),"=r"(ra[28]),"=r"(ra[29]),"=r"(ra[30]),"=r"(ra[31]),
                       "=r"(ra[32]),"=r"(ra[33]),"=r"(ra[34]),"=r"(ra[35]),"=r"(ra[36]),"=r"(ra[37]),"=r"(ra[38]),"=r"(ra[39]),"=r"(ra[40]),"=r"(ra[41]),"=r"(ra[42]),"=r"(ra[43]),"=r"(ra[44]),"=r"(ra[45]),"=r"(ra[46]),"=r"(ra[47]),"=r"(ra[48]),"=r"(ra[49]),"=r"(ra[50]),"=r"(ra[51]),"=r"(ra[52]),"=r"(ra[53]),"=r"(ra[54]),"=r"(ra[55]),"=r"(ra[56]),"=r"(ra[57]),"=r"(ra[58]),"=r"(ra[59]),"=r"(ra[60]),"=r"(ra[61]),"=r"(ra[62]),"=r"(ra[63])
                     : "r"(tl + 64 * half));
        TWAITLD(ra);
        TWAITLD((ra + 32));
#pragma unroll
        for (int k = 0; k < 64; ++k) s[k] = __uint_as_float(ra[k]);
      }
      uint32_t pk[32];
      uint64_t dacc[4] = {0ull, 0ull, 0ull, 0ull};
      const uint64_t l2e2 = f2(1.4426950f, 1.4426950f), b2c2 = f2(b2c, b2c);
#pragma unroll
      for (int p = 0; p < 32; ++p) {
        uint64_t x = ffma2(f2(s[2 * p], s[2 * p + 1]), l2e2, b2c2);
        const float2 lv = reinterpret_cast<const float2 *>(lse)[p];
        x = fsub2(x, f2(lv.x, lv.y));
        float e0, e1;
        if (EMU > 0 && p % EMU == EMU - 1) {
          ex2_emu2(x, e0, e1);
        } else {
          float x0, x1;
          f2split(x, x0, x1);
          e0 = ex2(x0);
          e1 = ex2(x1);
        }
        dacc[p & 3] = fadd2(dacc[p & 3], f2(e0, e1));
        pk[p] = pack_bf16x2(e0, e1);
      }
      float d0, d1;
      f2split(fadd2(fadd2(dacc[0], dacc[1]), fadd2(dacc[2], dacc[3])), d0, d1);
      db2 += d0 + d1;
      if constexpr (TM == 1 || TM == 3 || TM == 4) {   // G (packed bf16) back over the consumed S columns
        TST32(tl + 64 * half, pk);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
#pragma unroll
      for (int p = 0; p < 32; ++p) acc ^= pk[p];
      // opaque to the compiler (no instruction): the loop body cannot be hoisted
#pragma unroll
      for (int k = 0; k < 64; ++k) asm volatile("" : "+f"(s[k]));
    }
  }
  const long long t1 = clock64();
  if (active && (threadIdx.x & 31) == 0) cyc[blockIdx.x * 32 + warp] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc ^ __float_as_uint(db2);
  if constexpr (TM > 0) {
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tslot));
  }
}

// TM = 5 analogue with the loads software-pipelined: 32-column chunks, the next
// chunk's tcgen05.ld issued before the current chunk is computed (wait::ld waits
// for every outstanding load, so the wait of chunk c + 1 follows chunk c's math)
__device__ __forceinline__ void mix32(const uint32_t (&r)[32], const float *lse, int pbase, uint64_t (&dacc)[4],
                                      uint32_t *pk) {
  const uint64_t l2e2 = f2(1.4426950f, 1.4426950f), b2c2 = f2(0.1f, 0.1f);
#pragma unroll
  for (int p = 0; p < 16; ++p) {
    uint64_t x = ffma2(f2(__uint_as_float(r[2 * p]), __uint_as_float(r[2 * p + 1])), l2e2, b2c2);
    const float2 lv = reinterpret_cast<const float2 *>(lse)[pbase + p];
    x = fsub2(x, f2(lv.x, lv.y));
    float x0, x1;
    f2split(x, x0, x1);
    const float e0 = ex2(x0), e1 = ex2(x1);
    dacc[p & 3] = fadd2(dacc[p & 3], f2(e0, e1));
    pk[p] = pack_bf16x2(e0, e1);
  }
}
__global__ void __launch_bounds__(512, 1) k_pipe(int units, int active_warps_per_smsp, long long *cyc, uint32_t *sink) {
  const int warp = threadIdx.x >> 5;
  __shared__ uint32_t tslot;
  __shared__ __align__(16) float lse[64];
  if (threadIdx.x < 64) lse[threadIdx.x] = 3.0f + 0.001f * threadIdx.x;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tl = tslot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 128);
  const bool active = warp / 4 < active_warps_per_smsp;
  uint32_t acc = 0;
  float db2 = 0.f;
  const long long t0 = clock64();
  uint32_t ra[32], rb[32];
  if (active) { TLD32(tl, ra); TWAITLD(ra); }
  for (int u = 0; u < (active ? units : 0); ++u) {
#pragma unroll 1
    for (int half = 0; half < 2; ++half) {
      uint64_t dacc[4] = {0ull, 0ull, 0ull, 0ull};
      uint32_t pk[32];
      TLD32(tl + 64 * half + 32, rb);                 // chunk 1 in flight during chunk 0
      mix32(ra, lse, 0, dacc, pk);
      TWAITLD(rb);
      TLD32(tl + 64 * (half ^ 1), ra);                // next half's chunk 0 during chunk 1
      mix32(rb, lse, 16, dacc, pk + 16);
      TST32(tl + 64 * half, pk);
      TWAITLD(ra);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      float d0, d1;
      f2split(fadd2(fadd2(dacc[0], dacc[1]), fadd2(dacc[2], dacc[3])), d0, d1);
      db2 += d0 + d1;
#pragma unroll
      for (int p = 0; p < 32; ++p) acc ^= pk[p];
    }
  }
  const long long t1 = clock64();
  if (active && (threadIdx.x & 31) == 0) cyc[blockIdx.x * 32 + warp] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc ^ __float_as_uint(db2);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tslot));
}

int main() {
  const int blocks = 148, threads = 512, units = 2000;
  long long *cyc;
  uint32_t *sink;
  cudaMalloc(&cyc, 8 * blocks * 32);
  cudaMalloc(&sink, 4 * blocks * threads);
  const char *names[] = {"registers", "ld x32 + st", "ld x32 only", "st only", "ld x64 + st", "pipelined ld"};
  for (int v = 0; v < 6; ++v)
  for (int w = 1; w <= 4; w += (w == 1 ? 1 : 2)) {
    cudaMemset(cyc, 0, 8 * blocks * 32);
    auto kf = v == 0 ? k_mix<0, 0> : v == 1 ? k_mix<0, 1> : v == 2 ? k_mix<0, 2> : v == 3 ? k_mix<0, 3> : v == 4 ? k_mix<0, 4> : k_pipe;
    kf<<<blocks, threads>>>(10, w, cyc, sink);
    kf<<<blocks, threads>>>(units, w, cyc, sink);
    cudaDeviceSynchronize();
    long long h[148 * 32];
    cudaMemcpy(h, cyc, 8 * blocks * 32, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < blocks * 32; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("all-MUFU, %-12s warps/SMSP %d: %.0f cycles per unit per warp, %.0f per unit per SMSP  (%s)\n",
           names[v], w, mx / units, mx / units / w, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

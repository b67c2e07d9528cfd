// Micro-benchmark (tools only): does a tcgen05.mma stream whose A operand comes
// from TMEM (TS) take TMEM read bandwidth from concurrent tcgen05.ld traffic,
// compared with the same MMAs reading A from shared memory (SS)?
// One CTA per SM; warp 15 issues back-to-back M=128 N=128 K=128 bf16 MMAs (mode
// 0: none, 1: SS, 2: TS); warps 0..4w-1 stream 32x32b.x32 TMEM loads of their lane
// quarter.  Reports cycles per 16 KB of loads per sub-partition and MMAs issued.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_tmem_mma tools/ubench_tmem_mma.cu
#include <cstdio>
#include <cstdint>

#define TLD32(taddr, r) asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];" \
  : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]),"=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31]) : "r"(taddr))
#define TWAITLD(r) asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r[0]),"+r"(r[1]),"+r"(r[2]),"+r"(r[3]),"+r"(r[4]),"+r"(r[5]),"+r"(r[6]),"+r"(r[7]),"+r"(r[8]),"+r"(r[9]),"+r"(r[10]),"+r"(r[11]),"+r"(r[12]),"+r"(r[13]),"+r"(r[14]),"+r"(r[15]),"+r"(r[16]),"+r"(r[17]),"+r"(r[18]),"+r"(r[19]),"+r"(r[20]),"+r"(r[21]),"+r"(r[22]),"+r"(r[23]),"+r"(r[24]),"+r"(r[25]),"+r"(r[26]),"+r"(r[27]),"+r"(r[28]),"+r"(r[29]),"+r"(r[30]),"+r"(r[31]) :: "memory")

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {   // K-major SW128, SBO 1024
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__global__ void __launch_bounds__(512, 1) k(int mode, int iters, int warps_per_smsp, long long *cyc, int *mmas) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ int done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x3c003c00u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    done = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (warp == 15) {
    int n = 0;
    if (mode > 0) {
      const uint32_t id = idesc_bf16(128, 128);
      const uint64_t db = sdesc(su32(sm)), da = sdesc(su32(sm + 32768));
      const int nld = 4 * warps_per_smsp;
      while (*(volatile int *)&done < nld) {
        if (lane == 0) {
          for (int k = 0; k < 8; ++k) {   // K = 128: A from smem (SS) or TMEM cols 256 + 8k (TS), D at 384
            const uint64_t bk = db + (uint64_t)((k & 3) * 2 + (k >> 2) * 1024);
            if (mode == 1) {
              const uint64_t ak = da + (uint64_t)((k & 3) * 2 + (k >> 2) * 1024);
              asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                           "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + 384),
                           "l"(ak), "l"(bk), "r"(id), "r"(k));
            } else {
              asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                           "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + 384),
                           "r"(tmem + 256 + 8 * k), "l"(bk), "r"(id), "r"(k));
            }
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
        }
        __syncwarp();
        // wait for this group (keeps at most one 128^3 MMA group in flight)
        uint32_t ok = 0;
        do {
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok) : "r"(su32(&bar)), "r"((uint32_t)(n & 1)) : "memory");
        } while (!ok);
        ++n;
      }
    }
    if (lane == 0) mmas[blockIdx.x] = n;
  } else if (warp / 4 < warps_per_smsp) {
    const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 64);
    uint32_t r[32], acc = 0;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {   // 4 x 4 KB = 16 KB per warp per iteration
        TLD32(tl + (c & 1) * 32, r);
        TWAITLD(r);
        acc ^= r[c];
      }
    }
    const long long t1 = clock64();
    if (lane == 0) { cyc[blockIdx.x * 16 + warp] = t1 - t0; atomicAdd(&done, 1); }
    if (acc == 0x12345678u) cyc[0] = 0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  const int blocks = 148, threads = 512, iters = 4000, smem = 65536 + 1024;
  long long *cyc;
  int *mm;
  cudaMalloc(&cyc, 8 * blocks * 16);
  cudaMalloc(&mm, 4 * blocks);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char *names[] = {"no MMA", "SS MMA", "TS MMA"};
  for (int mode = 0; mode < 3; ++mode)
    for (int w = 1; w <= 3; ++w) {
      cudaMemset(cyc, 0, 8 * blocks * 16);
      k<<<blocks, threads, smem>>>(mode, 10, w, cyc, mm);
      k<<<blocks, threads, smem>>>(mode, iters, w, cyc, mm);
      cudaDeviceSynchronize();
      long long h[148 * 16];
      int hm[148];
      cudaMemcpy(h, cyc, 8 * blocks * 16, cudaMemcpyDeviceToHost);
      cudaMemcpy(hm, mm, 4 * blocks, cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < blocks * 16; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("%s, ld warps/SMSP %d: %.0f cycles per 16 KB per warp (%.1f B/clk/SM of TMEM loads); "
             "MMA groups in that time: %d (%.0f cycles per 128^3 group)  (%s)\n",
             names[mode], w, mx / iters, 4.0 * w * 16384.0 * iters / mx, hm[0], hm[0] ? mx / hm[0] : 0.0,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}

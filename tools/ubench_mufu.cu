// Micro-benchmark (tools only): issue throughput of the exponential variants
// the output-layer softmax can use on sm_100a, per SM per clock.
//   mode 0: ex2.approx.ftz.f32        (1 exp per lane-op)
//   mode 1: ex2.approx.f16x2          (2 exps per lane-op)
//   mode 2: ex2.approx.ftz.bf16x2     (2 exps per lane-op)
//   mode 3: fma.rn.f32x2              (reference: FMA pipe, 2 flops-pairs per lane-op)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_mufu tools/ubench_mufu.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>

template <int MODE>
__global__ void k(uint32_t *out, int iters, long long *cyc) {
  uint32_t v[8];
  for (int i = 0; i < 8; ++i) v[i] = 0x3c003c00u ^ (threadIdx.x * 7 + i);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(v[i]));
      if (MODE == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(v[i]));
      if (MODE == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(v[i]));
      if (MODE == 3) {
        uint64_t x = ((uint64_t)v[i] << 32) | v[(i + 1) & 7];
        asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(x));
        v[i] = (uint32_t)x ^ (uint32_t)(x >> 32);
      }
    }
  }
  long long t1 = clock64();
  uint32_t s = 0;
  for (int i = 0; i < 8; ++i) s ^= v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char *name) {
  const int blocks = 148, threads = 1024, iters = 4096;
  uint32_t *out;
  long long *cyc;
  cudaMalloc(&out, 4 * blocks * threads);
  cudaMalloc(&cyc, 8 * blocks);
  k<MODE><<<blocks, threads>>>(out, 16, cyc);
  k<MODE><<<blocks, threads>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, 8 * blocks, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < blocks; ++i) mx = h[i] > mx ? h[i] : mx;
  const double ops = (double)threads * iters * 8;  // lane-ops per SM
  printf("%-24s lane-ops/clk/SM = %.2f  (cycles %.0f)  err=%s\n", name, ops / mx, mx,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<0>("ex2.approx.ftz.f32");
  run<1>("ex2.approx.f16x2");
  run<2>("ex2.approx.ftz.bf16x2");
  run<3>("fma.rn.f32x2");
  return 0;
}

// Micro-benchmark (no idempotent folding: every max mixes two different chains):
// issue rate of packed 16x2 max on the integer (VIMNMX) and half (VHMNMX) forms,
// 2- and 3-input, alone and interleaved.  Result: max-ops per clock per SM
// (a 3-input op counts 2).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#define CH 12
#define ITERS 2048
__device__ __forceinline__ unsigned um2(unsigned a, unsigned b) { unsigned r; asm volatile("max.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r; }
__device__ __forceinline__ unsigned hm2(unsigned a, unsigned b) { unsigned r; asm volatile("max.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r; }
__device__ __forceinline__ unsigned um3(unsigned a, unsigned b, unsigned c) { unsigned r; asm volatile("{.reg .b32 q; max.u16x2 q, %1, %2; max.u16x2 %0, q, %3;}" : "=r"(r) : "r"(a), "r"(b), "r"(c)); return r; }
__device__ __forceinline__ unsigned hm3(unsigned a, unsigned b, unsigned c) { unsigned r; asm volatile("{.reg .b32 q; max.f16x2 q, %1, %2; max.f16x2 %0, q, %3;}" : "=r"(r) : "r"(a), "r"(b), "r"(c)); return r; }
template <int MODE>
__global__ void bench(unsigned *out, long long *cyc, unsigned seed, unsigned mul) {
  unsigned r[CH];
#pragma unroll
  for (int k = 0; k < CH; ++k) r[k] = 0x64006400u | ((seed * (threadIdx.x + 7 * k + 1)) & 0x00ff00ffu);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    unsigned n[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const unsigned a = r[k], b = r[(k + 1) % CH], c = r[(k + 5) % CH];
      if (MODE == 0) n[k] = um2(a, b);
      if (MODE == 1) n[k] = hm2(a, b);
      if (MODE == 2) n[k] = (k & 1) ? hm2(a, b) : um2(a, b);
      if (MODE == 3) n[k] = um3(a, b, c);
      if (MODE == 4) n[k] = hm3(a, b, c);
      if (MODE == 5) n[k] = (k & 1) ? hm3(a, b, c) : um3(a, b, c);
    }
#pragma unroll
    for (int k = 0; k < CH; ++k) r[k] = n[k] * mul + (unsigned)it;  // IMAD (FMA pipe, mul = 1 at run time): chains never converge
  }
  long long t1 = clock64();
  unsigned acc = 0;
#pragma unroll
  for (int k = 0; k < CH; ++k) acc ^= r[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int MODE>
void run(const char *name, int per_op, unsigned *out, long long *cyc, int blocks, int threads) {
  bench<MODE><<<blocks, threads>>>(out, cyc, 12345u, 1u);
  cudaDeviceSynchronize();
  long long h[4096];
  cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int b = 0; b < blocks; ++b) mx = h[b] > mx ? h[b] : mx;
  double ops = (double)(blocks / 148) * threads * ITERS * CH;
  printf("%-36s %6.1f instr-lanes/clk/SM %6.1f max-ops/clk/SM (+%d IMAD per op)\n", name, ops / mx, per_op * ops / mx, 1);
}
int main() {
  unsigned *out; long long *cyc;
  int blocks = 148 * 4, threads = 512;
  cudaMalloc(&out, sizeof(unsigned) * blocks * threads);
  cudaMalloc(&cyc, sizeof(long long) * blocks);
  run<0>("max.u16x2 2-input", 1, out, cyc, blocks, threads);
  run<1>("max.f16x2 2-input", 1, out, cyc, blocks, threads);
  run<2>("u16x2 : f16x2 1:1, 2-input", 1, out, cyc, blocks, threads);
  run<3>("max.u16x2 3-input", 2, out, cyc, blocks, threads);
  run<4>("max.f16x2 3-input", 2, out, cyc, blocks, threads);
  run<5>("u16x2 : f16x2 1:1, 3-input", 2, out, cyc, blocks, threads);
  return 0;
}

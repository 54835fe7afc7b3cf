// Micro-benchmark: can the FMA pipe take packed max/min work off the ALU pipe?
// max(a,b) = relu(a-b) + b and min(a,b) = a - relu(a-b) in f16x2 (exact for
// integer-valued halves such as 1024 + byte), against max.u16x2 on the ALU pipe.
// Result: thread-ops per clock per SM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#define CH 8
#define ITERS 4096
__device__ __forceinline__ void vmax(unsigned &r, unsigned s) { asm volatile("max.u16x2 %0, %0, %1;" : "+r"(r) : "r"(s)); }
__device__ __forceinline__ void vmax3(unsigned &r, unsigned s, unsigned t) {
  asm volatile("{.reg .b32 q; max.u16x2 q, %0, %1; max.u16x2 %0, q, %2;}" : "+r"(r) : "r"(s), "r"(t));
}
__device__ __forceinline__ void frelu(unsigned &r, unsigned s) {  // relu(r - s)
  asm volatile("{.reg .b32 n; neg.f16x2 n, %1; fma.rn.relu.f16x2 %0, %0, %2, n;}" : "+r"(r) : "r"(s), "r"(0x3c003c00u));
}
__device__ __forceinline__ void fadd(unsigned &r, unsigned s) { asm volatile("add.rn.f16x2 %0, %0, %1;" : "+r"(r) : "r"(s)); }
__device__ __forceinline__ void fmaxv(unsigned &r, unsigned s) {  // max via two FMA-pipe ops
  asm volatile("{.reg .b32 n, t; neg.f16x2 n, %1; fma.rn.relu.f16x2 t, %0, %2, n; add.rn.f16x2 %0, t, %1;}" : "+r"(r) : "r"(s), "r"(0x3c003c00u));
}
__device__ __forceinline__ void hmax(unsigned &r, unsigned s) { asm volatile("max.f16x2 %0, %0, %1;" : "+r"(r) : "r"(s)); }
__device__ __forceinline__ void imad(unsigned &r, unsigned s) { asm volatile("mad.lo.u32 %0, %0, %1, %1;" : "+r"(r) : "r"(s)); }
template <int MODE>
__global__ void bench(unsigned *out, long long *cyc, unsigned seed) {
  unsigned r[CH], s[CH];
#pragma unroll
  for (int k = 0; k < CH; ++k) { r[k] = 0x64006400u | ((seed * (threadIdx.x + k + 1)) & 0x00ff00ffu); s[k] = 0x64006400u | ((seed ^ (k * 0x9e3779b9u)) & 0x00ff00ffu); }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      if (MODE == 0) vmax(r[k], s[k]);
      if (MODE == 1) frelu(r[k], s[k]);
      if (MODE == 2) fadd(r[k], s[k]);
      if (MODE == 3) fmaxv(r[k], s[k]);                           // 1 max = 2 fma-pipe ops
      if (MODE == 4) { if (k & 1) fmaxv(r[k], s[k]); else vmax(r[k], s[k]); }  // 1:1 maxes
      if (MODE == 5) { if (k % 4 == 3) fmaxv(r[k], s[k]); else vmax(r[k], s[k]); }  // 3 alu : 1 fma max
      if (MODE == 6) hmax(r[k], s[k]);
      if (MODE == 7) { if (k & 1) imad(r[k], s[k]); else vmax(r[k], s[k]); }
      if (MODE == 8) vmax3(r[k], s[k], s[(k + 1) % CH]);
      if (MODE == 9) { if (k % 3 == 2) fmaxv(r[k], s[k]); else vmax(r[k], s[k]); }  // 2 alu : 1 fma max
    }
  }
  long long t1 = clock64();
  unsigned acc = 0;
#pragma unroll
  for (int k = 0; k < CH; ++k) acc ^= r[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int MODE>
void run(const char *name, unsigned *out, long long *cyc, int blocks, int threads) {
  bench<MODE><<<blocks, threads>>>(out, cyc, 12345u);
  cudaDeviceSynchronize();
  long long h[4096];
  cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int b = 0; b < blocks; ++b) mx = h[b] > mx ? h[b] : mx;
  int per_sm = blocks / 148;
  double ops = (double)per_sm * threads * ITERS * CH;
  printf("%-44s %6.1f max-ops/clk/SM\n", name, ops / (double)mx);
}
int main() {
  unsigned *out; long long *cyc;
  int blocks = 148 * 4, threads = 512;
  cudaMalloc(&out, sizeof(unsigned) * blocks * threads);
  cudaMalloc(&cyc, sizeof(long long) * blocks);
  run<0>("max.u16x2 (ALU)", out, cyc, blocks, threads);
  run<1>("fma.relu.f16x2 (+neg)", out, cyc, blocks, threads);
  run<2>("add.f16x2", out, cyc, blocks, threads);
  run<3>("max via relu+add (2 fma-pipe ops)", out, cyc, blocks, threads);
  run<4>("1 vimnmx : 1 fma-max", out, cyc, blocks, threads);
  run<5>("3 vimnmx : 1 fma-max", out, cyc, blocks, threads);
  run<9>("2 vimnmx : 1 fma-max", out, cyc, blocks, threads);
  run<6>("max.f16x2 (HMNMX2)", out, cyc, blocks, threads);
  run<7>("1 vimnmx : 1 imad", out, cyc, blocks, threads);
  run<8>("vimnmx3 (2 maxes fused)", out, cyc, blocks, threads);
  return 0;
}

// Micro-benchmark: issue throughput of the packed min/max candidates on sm_100a
// (VIMNMX.U16x2, HMNMX2, PRMT, FMNMX, FMNMX3, IMNMX), alone and interleaved.
// Result: thread-ops per clock per SM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#define CH 8
#define ITERS 4096
template <int MODE>
__global__ void bench(unsigned *out, long long *cyc, unsigned seed) {
  unsigned r[CH], s[CH];
#pragma unroll
  for (int k = 0; k < CH; ++k) { r[k] = seed * (threadIdx.x + k + 1); s[k] = seed ^ (k * 0x9e3779b9u); }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      if (MODE == 0) asm volatile("max.u16x2 %0, %0, %1;" : "+r"(r[k]) : "r"(s[k]));
      if (MODE == 1) asm volatile("max.f16x2 %0, %0, %1;" : "+r"(r[k]) : "r"(s[k]));
      if (MODE == 2) {
        if (k & 1) asm volatile("max.f16x2 %0, %0, %1;" : "+r"(r[k]) : "r"(s[k]));
        else asm volatile("max.u16x2 %0, %0, %1;" : "+r"(r[k]) : "r"(s[k]));
      }
      if (MODE == 3) asm volatile("prmt.b32 %0, %0, %1, 0x4140;" : "+r"(r[k]) : "r"(s[k]));
      if (MODE == 4) {
        if (k & 1) asm volatile("max.f16x2 %0, %0, %1;" : "+r"(r[k]) : "r"(s[k]));
        else asm volatile("prmt.b32 %0, %0, %1, 0x4140;" : "+r"(r[k]) : "r"(s[k]));
      }
      if (MODE == 5) asm volatile("max.f32 %0, %0, %1;" : "+r"(r[k]) : "r"(s[k]));
      if (MODE == 6) asm volatile("max.f32 %0, %0, %1, %2;" : "+r"(r[k]) : "r"(s[k]), "r"(s[(k + 1) % CH]));
      if (MODE == 7) asm volatile("max.u32 %0, %0, %1;" : "+r"(r[k]) : "r"(s[k]));
      if (MODE == 8) {  // 2 vimnmx : 2 hmnmx2 : 1 prmt
        if (k % 4 == 0 || k % 4 == 1) asm volatile("max.f16x2 %0, %0, %1;" : "+r"(r[k]) : "r"(s[k]));
        else asm volatile("max.u16x2 %0, %0, %1;" : "+r"(r[k]) : "r"(s[k]));
      }
      if (MODE == 9) asm volatile("max.s16x2 %0, %0, %1;" : "+r"(r[k]) : "r"(s[k]));
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
  printf("%-28s %6.1f thread-ops/clk/SM\n", name, ops / (double)mx);
}
int main() {
  unsigned *out; long long *cyc;
  int blocks = 148 * 4, threads = 512;
  cudaMalloc(&out, sizeof(unsigned) * blocks * threads);
  cudaMalloc(&cyc, sizeof(long long) * blocks);
  run<0>("VIMNMX.U16x2", out, cyc, blocks, threads);
  run<0>("VIMNMX.U16x2", out, cyc, blocks, threads);
  run<1>("HMNMX2", out, cyc, blocks, threads);
  run<2>("VIMNMX.U16x2+HMNMX2 1:1", out, cyc, blocks, threads);
  run<3>("PRMT", out, cyc, blocks, threads);
  run<4>("PRMT+HMNMX2 1:1", out, cyc, blocks, threads);
  run<5>("FMNMX", out, cyc, blocks, threads);
  run<6>("FMNMX3", out, cyc, blocks, threads);
  run<7>("IMNMX.U32", out, cyc, blocks, threads);
  run<8>("VIMNMX:HMNMX2 2:2", out, cyc, blocks, threads);
  run<9>("VIMNMX.S16x2", out, cyc, blocks, threads);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

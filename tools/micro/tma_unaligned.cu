// Do TMA tiled copies accept element-granular (unaligned) start coordinates in
// the innermost dimension?  1-D f32 tensor map over n floats, box {512}: load
// boxes starting at u = 0, 1, 3, 5, 17, 1000003 into shared memory and check the
// bytes; store boxes from shared memory at unaligned starts and check the
// output (and that nothing outside [u, u+512) changed).  Also a 1-D map with a
// 32-float box and 128-B swizzle.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void kload(const __grid_constant__ CUtensorMap m, int u, float *out, int box) {
  __shared__ __align__(1024) float buf[512];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(box * 4));
    asm volatile(
        "cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];" ::"r"(
            sa(buf)),
        "l"(reinterpret_cast<uint64_t>(&m)), "r"(u), "r"(sa(&bar))
        : "memory");
  }
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(sa(&bar)));
  for (int i = threadIdx.x; i < box; i += blockDim.x) out[i] = buf[i];
}

__global__ void kstore(const __grid_constant__ CUtensorMap m, int u) {
  __shared__ __align__(1024) float buf[512];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) buf[i] = 1000.0f + i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("cp.async.bulk.tensor.1d.global.shared::cta.bulk_group [%0, {%1}], [%2];" ::"l"(
                     reinterpret_cast<uint64_t>(&m)),
                 "r"(u), "r"(sa(buf))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  const int n = 1 << 21;
  float *d, *o;
  cudaMalloc(&d, n * 4);
  cudaMalloc(&o, 512 * 4);
  std::vector<float> h(n);
  for (int i = 0; i < n; ++i) h[i] = (float)i;
  cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  for (int sw = 0; sw < 2; ++sw) {
    const int box = sw ? 32 : 512;
    CUtensorMap m;
    cuuint64_t dims[1] = {(cuuint64_t)n};
    cuuint64_t str[1] = {0};
    cuuint32_t bx[1] = {(cuuint32_t)box}, es[1] = {1};
    CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 1, d, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("swizzle=%d box=%d encode=%d\n", sw, box, (int)r);
    for (int u : {0, 1, 3, 5, 17, 1000003, n - 100}) {
      cudaMemset(o, 0xff, 512 * 4);
      kload<<<1, 128>>>(m, u, o, box);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<float> g(box);
      cudaMemcpy(g.data(), o, box * 4, cudaMemcpyDeviceToHost);
      int bad = 0, oob = 0;
      for (int i = 0; i < box; ++i) {
        float want = (u + i < n) ? (float)(u + i) : 0.0f;
        if (u + i >= n) ++oob;
        if (g[i] != want) ++bad;
      }
      printf("  load u=%d err=%s bad=%d (oob elements %d, first %.1f)\n", u, cudaGetErrorString(e), bad, oob, g[0]);
    }
    if (sw) continue;
    for (int u : {0, 1, 3, 5, 17, 1000003, n - 100}) {
      cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
      kstore<<<1, 128>>>(m, u);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<float> g(n);
      cudaMemcpy(g.data(), d, n * 4, cudaMemcpyDeviceToHost);
      int bad = 0, outside = 0;
      for (int i = 0; i < n; ++i) {
        const bool in = i >= u && i < u + 512;
        const float want = in ? 1000.0f + (i - u) : (float)i;
        if (g[i] != want) (in ? ++bad : ++outside);
      }
      printf("  store u=%d err=%s bad_inside=%d changed_outside=%d\n", u, cudaGetErrorString(e), bad, outside);
    }
  }
  return 0;
}

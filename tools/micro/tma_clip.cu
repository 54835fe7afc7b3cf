// Does a TMA tensor store clip at globalDim[0]?  Store a 256x4 box of 0xAB into
// a {250, 4} u8 tensor with row pitch 256 and report the bytes written past col 250.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__global__ void k(const __grid_constant__ CUtensorMap m, int c) {
  __shared__ __align__(128) unsigned char buf[256 * 4];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = 0xAB;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(&m)), "r"(c), "r"(0),
                 "r"((unsigned)__cvta_generic_to_shared(buf)) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
int main() {
  unsigned char *d;
  cudaMalloc(&d, 256 * 8);
  cudaMemset(d, 0, 256 * 8);
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  for (int dim0 : {250, 256, 240}) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)dim0, 4};
    cuuint64_t str[1] = {256};
    cuuint32_t box[2] = {256, 4}, es[2] = {1, 1};
    CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaMemset(d, 0, 256 * 8);
    k<<<1, 128>>>(m, 0);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned char h[256 * 8];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    int inside = 0, past = 0, below = 0;
    for (int row = 0; row < 8; ++row)
      for (int c = 0; c < 256; ++c) {
        if (!h[row * 256 + c]) continue;
        if (row >= 4) ++below; else if (c < dim0) ++inside; else ++past;
      }
    printf("dim0=%d encode=%d err=%s written inside=%d past_dim0=%d below=%d\n", dim0, (int)r,
           cudaGetErrorString(e), inside, past, below);
  }
  return 0;
}

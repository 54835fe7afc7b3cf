// common.cuh -- device helpers shared by the max-min kernels (sm_100a only).
//
// * element traits: the two order operations of the paper's cost model
//   ("a<b or b<a") as branch-free max/min instructions;
// * TMA bulk copies global -> shared with mbarrier completion (cp.async.bulk,
//   SASS UBLKCP), the B200 way to stage a tile + halo on chip;
// * padded shared-memory indexing that makes lane-strided scalar accesses
//   bank-conflict free;
// * 16-byte vector global stores with the streaming (.cs) hint.
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#ifndef __CUDACC__
#error "CUDA only"
#endif

namespace mm {

// ---------------------------------------------------------------- traits ----
template <typename T>
struct Ord {
  static __device__ __forceinline__ T mx(T a, T b) { return a > b ? a : b; }
  static __device__ __forceinline__ T mn(T a, T b) { return a < b ? a : b; }
};
template <>
struct Ord<float> {  // FMNMX; inputs carry no NaN (maxmin.h preconditions)
  static __device__ __forceinline__ float mx(float a, float b) { return fmaxf(a, b); }
  static __device__ __forceinline__ float mn(float a, float b) { return fminf(a, b); }
};
template <>
struct Ord<double> {
  static __device__ __forceinline__ double mx(double a, double b) { return fmax(a, b); }
  static __device__ __forceinline__ double mn(double a, double b) { return fmin(a, b); }
};

// Elements per thread chunk: 16 for <= 4-byte types, 8 for 8-byte types, so a
// chunk is 16..64 bytes and a 256-thread CTA covers a 4096 (2048) element tile.
template <typename T>
struct Chunk {
  static constexpr int E = sizeof(T) == 8 ? 8 : 16;
  static constexpr int BYTES = E * (int)sizeof(T);
  static constexpr int VEC = 16 / (int)sizeof(T);  // elements per 16 B
  static constexpr int NV = BYTES / 16 > 0 ? BYTES / 16 : 1;
};

// -------------------------------------------------------- shared memory -----
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 1024-B aligned base inside the dynamic shared buffer.  Pointer arithmetic on
// the __shared__ array itself (no integer round trip), so the compiler keeps
// the shared address space and emits LDS/STS rather than generic LD/ST.
__device__ __forceinline__ unsigned char *smem_align1024(unsigned char *raw) {
  return raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
}

// Padded index: one 4-byte word (or one 8-byte element) of padding per 128 B
// row.  Lanes that access p = base + E*lane + d (any d) then hit distinct
// banks, for scalar accesses of every element size.
template <typename T>
__device__ __forceinline__ int pad_idx(int p) {
  constexpr int G = 128 / (int)sizeof(T);                   // elements per 128 B
  constexpr int P = sizeof(T) >= 4 ? 1 : 4 / (int)sizeof(T);  // pad elements
  return p + P * (p / G);
}
template <typename T>
__host__ __device__ constexpr int pad_size(int n) {
  return n + (sizeof(T) >= 4 ? 1 : 4 / (int)sizeof(T)) * (n / (128 / (int)sizeof(T)) + 1);
}

// ------------------------------------------------------------ mbarrier ------
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  // make the initialised barrier visible to the async (TMA) proxy
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// one arrival (release: the caller's earlier shared-memory writes are visible
// to whoever completes a wait on this phase)
__device__ __forceinline__ void mbar_arrive1(uint64_t *bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// TMA bulk copy (non-tensor): `bytes` (multiple of 16, addresses 16-B aligned)
// from global to shared; completion is signalled on `bar` as tx bytes.
__device__ __forceinline__ void bulk_g2s(void *smem_dst, const void *gsrc, uint32_t bytes,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Largest single bulk copy we issue (the mbarrier tx-count is < 2^20).
constexpr uint32_t kMaxBulk = 1u << 18;

// Issue the copy of global bytes [g0, g1) -- both 16-B aligned -- into smem,
// split into pieces; returns the byte count (to be armed on the barrier).
__device__ __forceinline__ uint32_t bulk_g2s_range(void *smem_dst, const char *g0,
                                                   const char *g1, uint64_t *bar) {
  uint32_t total = (uint32_t)(g1 - g0);
  uint32_t off = 0;
  while (off < total) {
    uint32_t b = total - off < kMaxBulk ? total - off : kMaxBulk;
    bulk_g2s((char *)smem_dst + off, g0 + off, b, bar);
    off += b;
  }
  return total;
}

// ----------------------------------------------------- global accesses ------
__device__ __forceinline__ void st_cs_16(void *p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}

// shared-memory atomic add, acquire-release at CTA scope (hand-offs by election)
__device__ __forceinline__ uint32_t atom_add_shared_u32(uint32_t *p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.acq_rel.cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(p)), "r"(v) : "memory");
  return old;
}

// 32-byte store (sm_100: STG.E.256): one whole L2 sector per lane, so a warp
// store of lane-strided chunks writes only full sectors.
__device__ __forceinline__ void st_cs_32(void *p, const uint32_t (&r)[8]) {
  asm volatile("st.global.cs.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

// Store E contiguous elements held in registers (16-B aligned destination;
// 32-B pieces go out as 256-bit stores when the destination allows it).
template <typename T, int E>
__device__ __forceinline__ void store_chunk(T *dst, const T (&v)[E]) {
  static_assert((E * sizeof(T)) % 16 == 0, "chunk must be whole 16-B vectors");
  constexpr int NW = E * (int)sizeof(T) / 4;
  union {
    T t[E];
    uint32_t w[NW];
    uint4 q[NW / 4];
  } u;
#pragma unroll
  for (int k = 0; k < E; ++k) u.t[k] = v[k];
  if (NW % 8 == 0 && (reinterpret_cast<uintptr_t>(dst) & 31) == 0) {
#pragma unroll
    for (int k = 0; k < NW / 8; ++k) {
      uint32_t r[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) r[e] = u.w[(k * 8 + e) % NW];
      st_cs_32(reinterpret_cast<char *>(dst) + 32 * k, r);
    }
  } else {
#pragma unroll
    for (int k = 0; k < NW / 4; ++k) st_cs_16(reinterpret_cast<uint4 *>(dst) + k, u.q[k]);
  }
}

// Load E contiguous elements from 16-B aligned shared memory into registers.
template <typename T, int E>
__device__ __forceinline__ void lds_chunk(const T *src, T (&v)[E]) {
  union {
    T t[E];
    uint4 q[E * sizeof(T) / 16];
  } u;
#pragma unroll
  for (int k = 0; k < (int)(E * sizeof(T) / 16); ++k) u.q[k] = reinterpret_cast<const uint4 *>(src)[k];
#pragma unroll
  for (int k = 0; k < E; ++k) v[k] = u.t[k];
}

// Load E contiguous elements starting `shift` elements (0 <= shift < VEC) past
// a 16-B aligned shared address: E/VEC+1 aligned vector loads, then a
// warp-uniform register shift (unaligned far range).
template <typename T, int E>
__device__ __forceinline__ void lds_chunk_shifted(const T *src16, int shift, T (&v)[E]) {
  constexpr int VEC = 16 / (int)sizeof(T);
  constexpr int NQ = (E + VEC - 1) / VEC + 1;
  union {
    T t[NQ * VEC];
    uint4 q[NQ];
  } u;
#pragma unroll
  for (int k = 0; k < NQ; ++k) u.q[k] = reinterpret_cast<const uint4 *>(src16)[k];
  // shift is uniform across the CTA: a switch over compile-time shifts keeps
  // every register index static.
#define MM_SHIFT_CASE(S)                              \
  case S:                                             \
    if (S < VEC) {                                    \
      _Pragma("unroll") for (int k = 0; k < E; ++k) v[k] = u.t[k + (S < VEC ? S : 0)]; \
    }                                                 \
    break;
  switch (shift) {
    MM_SHIFT_CASE(0) MM_SHIFT_CASE(1) MM_SHIFT_CASE(2) MM_SHIFT_CASE(3)
    MM_SHIFT_CASE(4) MM_SHIFT_CASE(5) MM_SHIFT_CASE(6) MM_SHIFT_CASE(7)
    MM_SHIFT_CASE(8) MM_SHIFT_CASE(9) MM_SHIFT_CASE(10) MM_SHIFT_CASE(11)
    MM_SHIFT_CASE(12) MM_SHIFT_CASE(13) MM_SHIFT_CASE(14) MM_SHIFT_CASE(15)
    default: break;
  }
#undef MM_SHIFT_CASE
}

// ---------------------------------------------------------- warp helpers ----
template <typename T>
__device__ __forceinline__ T shfl_up(T v, int d) {
  return __shfl_up_sync(0xffffffffu, v, d);
}
template <typename T>
__device__ __forceinline__ T shfl_down(T v, int d) {
  return __shfl_down_sync(0xffffffffu, v, d);
}
// 1- and 2-byte types travel through 32-bit shuffles
template <>
__device__ __forceinline__ uint8_t shfl_up(uint8_t v, int d) { return (uint8_t)__shfl_up_sync(0xffffffffu, (uint32_t)v, d); }
template <>
__device__ __forceinline__ int8_t shfl_up(int8_t v, int d) { return (int8_t)__shfl_up_sync(0xffffffffu, (int32_t)v, d); }
template <>
__device__ __forceinline__ uint16_t shfl_up(uint16_t v, int d) { return (uint16_t)__shfl_up_sync(0xffffffffu, (uint32_t)v, d); }
template <>
__device__ __forceinline__ int16_t shfl_up(int16_t v, int d) { return (int16_t)__shfl_up_sync(0xffffffffu, (int32_t)v, d); }
template <>
__device__ __forceinline__ uint8_t shfl_down(uint8_t v, int d) { return (uint8_t)__shfl_down_sync(0xffffffffu, (uint32_t)v, d); }
template <>
__device__ __forceinline__ int8_t shfl_down(int8_t v, int d) { return (int8_t)__shfl_down_sync(0xffffffffu, (int32_t)v, d); }
template <>
__device__ __forceinline__ uint16_t shfl_down(uint16_t v, int d) { return (uint16_t)__shfl_down_sync(0xffffffffu, (uint32_t)v, d); }
template <>
__device__ __forceinline__ int16_t shfl_down(int16_t v, int d) { return (int16_t)__shfl_down_sync(0xffffffffu, (int32_t)v, d); }

// Segmented shuffles (aligned segments of `width` lanes): a lane whose source
// lies outside its segment gets its own value back, so an idempotent scan step
// (max/min) needs no lane predicate: v = op(v, shfl_up_seg(v, d, width)).
template <typename T>
__device__ __forceinline__ T shfl_up_seg(T v, int d, int width) {
  if constexpr (sizeof(T) < 4) {
    using W = typename std::conditional<std::is_signed<T>::value, int32_t, uint32_t>::type;
    return (T)__shfl_up_sync(0xffffffffu, (W)v, d, width);
  } else {
    return __shfl_up_sync(0xffffffffu, v, d, width);
  }
}
template <typename T>
__device__ __forceinline__ T shfl_down_seg(T v, int d, int width) {
  if constexpr (sizeof(T) < 4) {
    using W = typename std::conditional<std::is_signed<T>::value, int32_t, uint32_t>::type;
    return (T)__shfl_down_sync(0xffffffffu, (W)v, d, width);
  } else {
    return __shfl_down_sync(0xffffffffu, v, d, width);
  }
}

// --------------------------------------------------- release / acquire ------
__device__ __forceinline__ void st_release_u32(uint32_t *p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

}  // namespace mm

// tma.cuh -- TMA tensor-map staging of 1-D series for the max-min kernels.
//
// A batch of series (row b at in + b*in_ld) is described to the TMA engine as a
// 3-D tensor {RW, rows, batch}: RW = 128/sizeof(T) elements per 128-byte row,
// rows = floor(n / RW) whole rows per series.  Boxes of {RW, 8} (1 KB) land in
// shared memory with the 128-byte swizzle, so the lane-strided 16-byte reads of
// the kernels are bank-conflict free.  The partial last row of a series (fewer
// than RW elements) is not covered by the map (the TMA would otherwise read past
// the series end); kernels patch it in with plain loads ("tail fix").
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace mm {

constexpr int kBoxRows = 8;                        // rows per TMA box (1 KB, one swizzle atom)
constexpr int kBoxBytes = 128 * kBoxRows;

template <typename T>
struct Rowing {
  static constexpr int RW = 128 / (int)sizeof(T);  // elements per 128-B row
};

// Byte offset in a 1024-B aligned, 128-B swizzled buffer of logical 16-B chunk c.
__device__ __forceinline__ uint32_t swz(uint32_t c) {
  return ((c >> 3) << 7) | (((c & 7) ^ ((c >> 3) & 7)) << 4);
}

// Load E contiguous elements starting at logical element position pos of a
// swizzled buffer into registers.  pos % VEC may be non-zero (uniform shift).
template <typename T, int E>
__device__ __forceinline__ void lds_swz(const unsigned char *buf, int pos, T (&v)[E]) {
  constexpr int VEC = 16 / (int)sizeof(T);
  constexpr int NQ = (E + VEC - 1) / VEC + 1;
  const int c0 = pos / VEC;
  const int sh = pos - c0 * VEC;
  union {
    T t[NQ * VEC];
    uint4 q[NQ];
  } u;
  if (sh == 0) {
#pragma unroll
    for (int k = 0; k < NQ - 1; ++k) u.q[k] = *reinterpret_cast<const uint4 *>(buf + swz(c0 + k));
#pragma unroll
    for (int k = 0; k < E; ++k) v[k] = u.t[k];
    return;
  }
#pragma unroll
  for (int k = 0; k < NQ; ++k) u.q[k] = *reinterpret_cast<const uint4 *>(buf + swz(c0 + k));
#define MM_SW_CASE(S)                                                              \
  case S:                                                                          \
    if (S < VEC) {                                                                 \
      _Pragma("unroll") for (int k = 0; k < E; ++k) v[k] = u.t[k + (S < VEC ? S : 0)]; \
    }                                                                              \
    break;
  switch (sh) {
    MM_SW_CASE(1) MM_SW_CASE(2) MM_SW_CASE(3) MM_SW_CASE(4) MM_SW_CASE(5)
    MM_SW_CASE(6) MM_SW_CASE(7) MM_SW_CASE(8) MM_SW_CASE(9) MM_SW_CASE(10)
    MM_SW_CASE(11) MM_SW_CASE(12) MM_SW_CASE(13) MM_SW_CASE(14) MM_SW_CASE(15)
    default: break;
  }
#undef MM_SW_CASE
}

// Aligned variant (pos % E == 0 and E*sizeof(T) is a multiple of 16).
template <typename T, int E>
__device__ __forceinline__ void lds_swz_aligned(const unsigned char *buf, int pos, T (&v)[E]) {
  constexpr int VEC = 16 / (int)sizeof(T);
  constexpr int NQ = E / VEC;
  const int c0 = pos / VEC;
  union {
    T t[E];
    uint4 q[NQ];
  } u;
#pragma unroll
  for (int k = 0; k < NQ; ++k) u.q[k] = *reinterpret_cast<const uint4 *>(buf + swz(c0 + k));
#pragma unroll
  for (int k = 0; k < E; ++k) v[k] = u.t[k];
}

// Scalar load of the element at logical position pos.
template <typename T>
__device__ __forceinline__ T lds_one_swz(const unsigned char *buf, int pos) {
  constexpr int VEC = 16 / (int)sizeof(T);
  const int c = pos / VEC;
  return *reinterpret_cast<const T *>(buf + swz(c) + (pos - c * VEC) * sizeof(T));
}

// Scalar store of element at logical position pos (tail fix).
template <typename T>
__device__ __forceinline__ void sts_swz(unsigned char *buf, int pos, T v) {
  constexpr int VEC = 16 / (int)sizeof(T);
  const int c = pos / VEC;
  *reinterpret_cast<T *>(buf + swz(c) + (pos - c * VEC) * sizeof(T)) = v;
}

// One TMA box {RW x 8 rows} of series b starting at row r (may be out of range:
// zero fill) into dst (1024-B aligned).
__device__ __forceinline__ void tma_box(const CUtensorMap *map, void *dst, int r, int b,
                                        uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(r), "r"(b), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// Two maps over the same rows (k1d_large): boxes of 32 rows (4 KB) and of 8
// rows (1 KB); a staged range is covered by big boxes plus a few small ones.
constexpr int kBigRows = 32;
constexpr int kBigBytes = 128 * kBigRows;
struct TmaMaps {
  CUtensorMap big;
  CUtensorMap small;
};

// Stage logical elements [e0, e0+len) of series b (e0 % RW arbitrary) into buf
// starting at buf row 0 = series row floor(e0/RW).  Issues whole boxes and arms
// the barrier.  Returns the logical offset of e0 inside buf.
template <typename T>
__device__ __forceinline__ int stage_range(const CUtensorMap *map, unsigned char *buf, int64_t e0,
                                           int64_t len, int b, uint64_t *bar) {
  constexpr int RW = Rowing<T>::RW;
  const int64_t r0 = e0 / RW;
  const int64_t r1 = (e0 + len + RW - 1) / RW;  // exclusive
  const int nbox = (int)((r1 - r0 + kBoxRows - 1) / kBoxRows);
  mbar_arrive_expect_tx(bar, (uint32_t)nbox * kBoxBytes);
  for (int k = 0; k < nbox; ++k) tma_box(map, buf + k * kBoxBytes, (int)(r0 + k * kBoxRows), b, bar);
  return (int)(e0 - r0 * RW);
}

// After the barrier: patch the partial last row of series b (elements
// [full_rows*RW, n)) if it falls inside the staged range.  Called by all
// threads; returns true if a __syncthreads() is needed before reading.
template <typename T>
__device__ __forceinline__ bool tail_fix(unsigned char *buf, const T *series, int64_t n,
                                         int64_t e0_row_start, int64_t len_elems, int tid, int nthreads) {
  constexpr int RW = Rowing<T>::RW;
  const int64_t full = (n / RW) * RW;
  const int64_t end = e0_row_start + len_elems;  // staged logical end (absolute)
  if (full >= n || full >= end || n <= e0_row_start) return false;
  const int64_t lo = full > e0_row_start ? full : e0_row_start;
  const int64_t hi = n < end ? n : end;
  for (int64_t i = lo + tid; i < hi; i += nthreads) sts_swz<T>(buf, (int)(i - e0_row_start), series[i]);
  return true;
}

}  // namespace mm

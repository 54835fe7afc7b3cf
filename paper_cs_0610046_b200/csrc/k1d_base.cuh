// k1d.cuh -- 1-D (and batched) running max-min filter kernels for sm_100a.
//
// The operation is PAPER.md:39-42: out_max[j] = max a[j..j+w), out_min[j] =
// min a[j..j+w), j in [0, n-w].  The paper's own algorithm (the monotonic
// wedge, Algorithm 1) is inherently sequential; on the GPU
// the same result is reached by splitting every window into a near part, a gap
// and a far part, in the family of van Herk / Gil-Werman:
//
//   out[j] = max( S(j), M, P(j+w-1) )
//
// S = suffix max from j to the end of j's "near block", P = prefix max from the
// start of the matching "far block" (the near block shifted by w-1) to j+w-1,
// M = max of the fixed gap between them (likewise for min).  Near and far blocks
// are aligned to the per-thread chunks, so S and P are chunk-local scans plus
// one group carry each; the gap is assembled from far-block aggregates.
//
//   k1d_small<T,W>   2 <= w <= E: compile-time w ("compiling w in the code",
//                    PAPER.md:528-531), log-step doubling in registers.
//   k1d_medium<T>    E < w <= kHaloMax+1: tile + (w-1) halo staged by TMA
//                    (128-B swizzle) in shared memory; block B = E*G <= w-1.
//   k1d_large<T>     w-1 > kHaloMax: the block is the whole tile; each CTA
//                    stages its near tile and its far tile, gap aggregates come
//                    from a cross-CTA look-back through a workspace (ticketed,
//                    deadlock-free).
//
// All kernels are persistent, prefetch the next tile with TMA while computing
// the current one, and write outputs with 256-bit streaming stores.  Every
// kernel handles a batch of rows (row b at in + b*in_ld); 1-D is batch 1.
#pragma once

#include "common.cuh"
#include "tma.cuh"

namespace mm {

constexpr int NT = 256;  // threads per CTA (8 warps)
constexpr int NWARP = NT / 32;
constexpr int kHaloMax = 8192;  // largest on-chip halo (elements) of k1d_medium

struct Rows {
  const void *in;
  void *out_max;
  void *out_min;
  int64_t n;       // row length
  int64_t w;       // window
  int64_t m;       // windows per row = n - w + 1
  int64_t in_ld;   // elements between rows
  int64_t out_ld;  // elements between output rows
  int64_t batch;
  int64_t tiles_per_row;
  int64_t ntiles;  // batch * tiles_per_row
  int has_map;     // the series has >= 1 whole 128-B row (else: plain loads only)
};

template <int TILE>
__device__ __forceinline__ void tile_coords(const Rows &p, int64_t t, int64_t &row, int64_t &u0,
                                            int &tout) {
  row = t / p.tiles_per_row;
  u0 = (t - row * p.tiles_per_row) * (int64_t)TILE;
  int64_t left = p.m - u0;
  tout = left < TILE ? (int)left : TILE;
}

// Position of a tile, advanced incrementally (no 64-bit division per tile).
template <int TILE>
struct TileCursor {
  int64_t row, u0;
  __device__ __forceinline__ void start(const Rows &p, int64_t t) {
    row = t / p.tiles_per_row;
    u0 = (t - row * p.tiles_per_row) * (int64_t)TILE;
  }
  __device__ __forceinline__ void advance(const Rows &p) {
    u0 += TILE;
    if (u0 >= p.m) {
      u0 = 0;
      ++row;
    }
  }
  __device__ __forceinline__ int tout(const Rows &p) const {
    const int64_t left = p.m - u0;
    return left < TILE ? (int)left : TILE;
  }
};

// Contiguous, balanced range [t_begin, t_end) of tiles for this CTA.
__device__ __forceinline__ void cta_tile_range(const Rows &p, int64_t &t_begin, int64_t &t_end) {
  t_begin = p.ntiles * (int64_t)blockIdx.x / gridDim.x;
  t_end = p.ntiles * ((int64_t)blockIdx.x + 1) / gridDim.x;
}

template <typename T>
__device__ __forceinline__ const T *series_ptr(const Rows &p, int64_t row) {
  return static_cast<const T *>(p.in) + row * p.in_ld;
}

// Stage input [u0, u0+len) of `row` (u0 is a multiple of RW) into buf.
template <typename T>
__device__ __forceinline__ void stage_tile(const Rows &p, const CUtensorMap *map, unsigned char *buf,
                                           int64_t row, int64_t u0, int64_t len, uint64_t *bar) {
  if (p.has_map) {
    stage_range<T>(map, buf, u0, len, (int)row, bar);
  } else {
    mbar_arrive_expect_tx(bar, 0);  // nothing in flight: the tail fix loads it all
  }
}

// As stage_tile, with 32-row (4 KB) boxes for the bulk and 8-row boxes for the
// rest: ~4x fewer TMA instructions for the issuing thread, whose warp would
// otherwise reach the tile's CTA barrier late (k1d_medium).
template <typename T>
__device__ __forceinline__ void stage_tile2(const Rows &p, const TmaMaps *maps, unsigned char *buf, int64_t row,
                                            int64_t u0, int64_t len, uint64_t *bar) {
  constexpr int RW = Rowing<T>::RW;
  if (!p.has_map) {
    mbar_arrive_expect_tx(bar, 0);  // nothing in flight: the tail fix loads it all
    return;
  }
  const int64_t r0 = u0 / RW;
  const int64_t r1 = (u0 + len + RW - 1) / RW;
  const int nrows = (int)(r1 - r0);
  const int nbig = nrows / kBigRows;
  const int nsmall = (nrows - nbig * kBigRows + kBoxRows - 1) / kBoxRows;
  mbar_arrive_expect_tx(bar, (uint32_t)(nbig * kBigBytes + nsmall * kBoxBytes));
  for (int k = 0; k < nbig; ++k) tma_box(&maps->big, buf + k * kBigBytes, (int)(r0 + k * kBigRows), (int)row, bar);
  for (int k = 0; k < nsmall; ++k)
    tma_box(&maps->small, buf + nbig * kBigBytes + k * kBoxBytes, (int)(r0 + nbig * kBigRows + k * kBoxRows),
            (int)row, bar);
}

// Patch the partial last 128-B row (not covered by the tensor map); returns
// whether shared memory was written (caller must __syncthreads()).
template <typename T>
__device__ __forceinline__ bool patch_tail(const Rows &p, unsigned char *buf, int64_t row, int64_t u0,
                                           int64_t len, int tid) {
  constexpr int RW = Rowing<T>::RW;
  const int64_t full = p.has_map ? (p.n / RW) * RW : 0;
  if (full >= p.n || u0 + len <= full) return false;
  const T *s = series_ptr<T>(p, row);
  const int64_t lo = full > u0 ? full : u0;
  const int64_t hi = p.n < u0 + len ? p.n : u0 + len;
  for (int64_t i = lo + tid; i < hi; i += NT) sts_swz<T>(buf, (int)(i - u0), s[i]);
  return true;
}

template <typename T, int E>
__device__ __forceinline__ void store_out(const Rows &p, int64_t row, int64_t j0, int cnt,
                                          const T (&ox)[E], const T (&on)[E]) {
  T *omx = p.out_max ? static_cast<T *>(p.out_max) + row * p.out_ld + j0 : nullptr;
  T *omn = p.out_min ? static_cast<T *>(p.out_min) + row * p.out_ld + j0 : nullptr;
  if (cnt >= E) {
    if (omx) store_chunk<T, E>(omx, ox);
    if (omn) store_chunk<T, E>(omn, on);
  } else {
#pragma unroll
    for (int k = 0; k < E; ++k)
      if (k < cnt) {
        if (omx) omx[k] = ox[k];
        if (omn) omn[k] = on[k];
      }
  }
}

// Epilogue of the 1-D kernels: what happens to a thread's E window results
// (cnt <= 0: the thread's chunk lies past the tile's last window).  The
// library's filters store them; N3 (keogh.cu) folds them into a bound instead.
struct StoreEpi {
  template <typename T, int E>
  __device__ __forceinline__ void operator()(const Rows &p, int64_t row, int64_t j0, int cnt, const T (&ox)[E],
                                             const T (&on)[E]) const {
    if (cnt > 0) store_out<T, E>(p, row, j0, cnt, ox, on);
  }
};

#ifndef MM_WARP_E
#define MM_WARP_E 16
#endif
// max/min of v[o..E-1] for a warp-uniform (or single-lane) runtime o in [0, E)
template <typename T, int E>
__device__ __forceinline__ void suffix_from(const T (&v)[E], int o, T &hx, T &hn) {
  hx = hn = v[E - 1];
#define MM_SUF_CASE(O)                                                             \
  case O:                                                                          \
    _Pragma("unroll") for (int k = (O < E ? O : E - 1); k < E - 1; ++k) {          \
      hx = Ord<T>::mx(hx, v[k]);                                                   \
      hn = Ord<T>::mn(hn, v[k]);                                                   \
    }                                                                              \
    break;
  switch (o) {
    MM_SUF_CASE(0) MM_SUF_CASE(1) MM_SUF_CASE(2) MM_SUF_CASE(3) MM_SUF_CASE(4) MM_SUF_CASE(5)
    MM_SUF_CASE(6) MM_SUF_CASE(7) MM_SUF_CASE(8) MM_SUF_CASE(9) MM_SUF_CASE(10) MM_SUF_CASE(11)
    MM_SUF_CASE(12) MM_SUF_CASE(13) MM_SUF_CASE(14) MM_SUF_CASE(15)
#if MM_WARP_E > 16
    MM_SUF_CASE(16) MM_SUF_CASE(17) MM_SUF_CASE(18) MM_SUF_CASE(19) MM_SUF_CASE(20) MM_SUF_CASE(21)
    MM_SUF_CASE(22) MM_SUF_CASE(23) MM_SUF_CASE(24) MM_SUF_CASE(25) MM_SUF_CASE(26) MM_SUF_CASE(27)
    MM_SUF_CASE(28) MM_SUF_CASE(29) MM_SUF_CASE(30) MM_SUF_CASE(31)
#endif
    default: break;
  }
#undef MM_SUF_CASE
}

}  // namespace mm

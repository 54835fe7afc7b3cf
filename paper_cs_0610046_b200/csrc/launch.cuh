// launch.cuh -- host-side launchers (templated on the element type).  The
// C-ABI layer (maxmin_abi.cu) validates arguments and dispatches on dtype; one
// translation unit per dtype (inst_<t>.cu) instantiates these templates.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <cstring>
#include <type_traits>

#include "k1d.cuh"
#include "k2d.cuh"

namespace mm {

// status codes mirror include/maxmin.h
enum : int { kOK = 0, kErrWorkspace = 8, kErrCuda = 9, kErrUnsupported = 10 };

int note_cuda(cudaError_t e);  // records the error (thread-local), returns kErrCuda or kOK
int sm_count();                // SMs of the current device (cached)
// packed 1-byte 2-D kernel (k2d_byte.cu); kErrUnsupported when it does not apply
int launch_2d_byte(bool is_signed, const void *in, int64_t batch, int64_t rows, int64_t cols,
                   int64_t in_ld, int64_t in_bstride, int64_t w_row, int64_t w_col, void *out_max,
                   void *out_min, int64_t out_ld, int64_t out_bstride, cudaStream_t s);
// square windows the packed 1-byte kernel is compiled for (k2d_byte.cu)
bool k2b_supports(int64_t w);
// 1-byte grayscale opening / closing by a w x w square in three packed passes
// (k2d_byte.cu); kErrUnsupported when the packed kernel does not apply
int launch_morph_2d_byte(bool is_signed, const void *in, int64_t batch, int64_t rows, int64_t cols, int64_t in_ld,
                         int64_t in_bstride, int64_t w, void *out_open, void *out_close, int64_t out_ld,
                         int64_t out_bstride, void *e_buf, void *d_buf, int64_t buf_ld, cudaStream_t s);
// LB_Keogh fused with the envelope (keogh.cu): float rows
int launch_keogh(const float *c, int64_t batch, int64_t n, int64_t ld, const float *q, int64_t r, double *lb,
                 cudaStream_t s);
// arg-max / arg-min filter (argfilter.cu): <= 4-byte element types
size_t argfilter_workspace(int64_t batch, int64_t n, int64_t w);
template <typename T>
int launch_argfilter(const void *in, int64_t batch, int64_t n, int64_t in_ld, int64_t w, void *out_max,
                     void *out_min, int64_t *arg_max, int64_t *arg_min, int64_t out_ld, void *ws,
                     size_t ws_bytes, cudaStream_t s);
// Launch shape of a warp-autonomous kernel (stream.cu, morph.cu, argfilter.cu):
// warps per CTA (nw in {max_nw, max_nw/2, ..., min_nw}) and staging depth ns
// (2..4), from the occupancy API, cached per (kernel, w) -- the queries cost
// microseconds, a push tens.  The kernel's dynamic shared memory limit only
// grows, under a lock, so concurrent host threads never shrink it under a
// launch in flight (maxmin_abi.cu).
// Raise a kernel's dynamic shared memory limit to at least `bytes` on the
// current device; the limit only grows, under a lock (concurrent host threads
// never lower it under another thread's launch).  maxmin_abi.cu.
int raise_smem_limit(const void *kern, size_t bytes);
// Resident CTAs per SM of a kernel (cudaOccupancyMaxActiveBlocksPerMultiprocessor),
// cached per (kernel, device, threads, smem): the query costs microseconds.
int blocks_per_sm(const void *kern, int threads, size_t smem, int *per_sm);

struct WarpLaunch {
  int ns, nw, per_sm;
  size_t smem;
};
using WarpBytesFn = size_t (*)(int w, int ns, int nw);
int warp_launch_choice(const void *kern, int w, int max_nw, int min_nw, WarpBytesFn bytes, int prefer_warps,
                       WarpLaunch *out);

// online multi-stream filter (stream.cu)
struct StreamLayout {
  int fused;          // one fused kernel per push (ping-pong history rows) or the composition
  int64_t ld;         // elements between state rows
  size_t hist_bytes;  // one history buffer (fused) / the [history | slot] rows (composed)
  size_t ws_bytes;    // the filter's workspace (composed)
  size_t total;
};
template <typename T>
StreamLayout stream_layout(int64_t streams, int64_t w, int64_t max_chunk);
template <typename T>
int launch_stream_push(void *state, const StreamLayout &L, int64_t streams, int64_t w, int phase, const T *chunk,
                       int64_t c, int64_t chunk_ld, T *out_max, T *out_min, int64_t out_ld, cudaStream_t s);
// separable 2-D path (sep2d.cu): rows by the 1-D kernels, columns streaming
template <typename T>
size_t sep2d_workspace(int64_t batch, int64_t rows, int64_t cols, int64_t w_row, int64_t w_col);
template <typename T>
int launch_2d_sep(const void *in, int64_t batch, int64_t rows, int64_t cols, int64_t in_ld, int64_t in_bstride,
                  int64_t w_row, int64_t w_col, void *out_max, void *out_min, int64_t out_ld, int64_t out_bstride,
                  void *ws, size_t ws_bytes, cudaStream_t s);
// the fastest applicable 2-D path: packed bytes, else separable (workspace), else fused generic
template <typename T>
int launch_2d_best(const void *in, int64_t batch, int64_t rows, int64_t cols, int64_t in_ld, int64_t in_bstride,
                   int64_t w_row, int64_t w_col, void *out_max, void *out_min, int64_t out_ld, int64_t out_bstride,
                   void *ws, size_t ws_bytes, cudaStream_t s);
// 3-D boxes (filter3d.cu)
template <typename T>
size_t filter3d_workspace(int64_t depth, int64_t rows, int64_t cols, int64_t in_ld, int64_t w_x, int64_t w_y,
                          int64_t w_z);
template <typename T>
int launch_3d(const void *in, int64_t depth, int64_t rows, int64_t cols, int64_t in_ld, int64_t in_slice,
              int64_t w_x, int64_t w_y, int64_t w_z, void *out_max, void *out_min, int64_t out_ld, int64_t out_slice,
              void *ws, cudaStream_t s);
// grayscale opening / closing (morph.cu)
template <typename T>
int launch_morph(const void *in, int64_t batch, int64_t n, int64_t in_ld, int64_t w, void *out_open,
                 void *out_close, int64_t out_ld, cudaStream_t s);
template <typename T>
size_t morph_2d_workspace(int64_t batch, int64_t rows, int64_t cols, int64_t w_row, int64_t w_col);
template <typename T>
int launch_morph_2d(const void *in, int64_t batch, int64_t rows, int64_t cols, int64_t in_ld, int64_t in_bstride,
                    int64_t w_row, int64_t w_col, void *out_open, void *out_close, int64_t out_ld,
                    int64_t out_bstride, void *ws, cudaStream_t s);
int encode_u8_map(CUtensorMap *map, const void *base, const int64_t dims[3], const int64_t strides[2],
                  const int box[3]);  // maxmin_abi.cu
int encode_rows_map(CUtensorMap *map, const void *in, int elem_bytes, int64_t rows_per_series,
                    int64_t batch, int64_t in_ld_bytes, int box_rows = kBoxRows,
                    bool swizzle = true);  // maxmin_abi.cu

// Tile geometry of the 1-D kernels for element type T.
template <typename T>
struct Geo1D {
  static constexpr int E = Chunk<T>::E;
  static constexpr int TILE = NT * E;
};

enum class Path1D { Copy, Small, Medium, Large, Warp };

#ifndef MM_WARP_MIN_W  // smallest window routed to k1d_warp (<= 4-byte types): it
#define MM_WARP_MIN_W (kHaloMax + 2)  // beats k1d_large, not (yet) k1d_medium
#endif

template <typename T>
Path1D path_1d(int64_t w) {
  if (w == 1) return Path1D::Copy;
  if (w <= Geo1D<T>::E) return Path1D::Small;
  if constexpr (sizeof(T) <= 4) {
    if (w - 1 >= WarpGeo<T>::WT && w >= MM_WARP_MIN_W) return Path1D::Warp;
  }
  if (w - 1 <= kHaloMax) return Path1D::Medium;
  return Path1D::Large;
}

template <typename T>
WarpLB warp_geom(int64_t batch, int64_t n, int64_t w) {
  WarpLB g{};
  if constexpr (sizeof(T) <= 4) {
    constexpr int64_t WT = WarpGeo<T>::WT, K = WarpGeo<T>::K;
    const int64_t m = n - w + 1;
    g.q = (int)((w - 1) / WT);
    g.r = (int)((w - 1) % WT);
    g.tpr = (m + WT - 1) / WT;
    g.xr = g.q + g.tpr;
    g.kt = (g.xr + K - 1) / K;
    g.total = batch * g.kt;
    g.pg = (int)((g.q + K - 1) / K + 1);
  }
  return g;
}

#ifndef MM_LW  // 1: the large-window path of <= 4-byte types is k1d_lw; 0: k1d_warp (round 1)
#define MM_LW 1
#endif

template <typename T>
LwArgs lw_geom(int64_t batch, int64_t n, int64_t w) {
  LwArgs g{};
  if constexpr (sizeof(T) <= 4) {
    constexpr int64_t WT = LwGeo<T>::WT;
    const int64_t m = n - w + 1;
    g.q = (int)((w - 1) / WT);
    g.r = (int)((w - 1) % WT);
    g.tpr = (m + WT - 1) / WT;
    g.kt = (g.q + g.tpr + NWARP - 1) / NWARP;
    g.total = batch * g.kt;
  }
  return g;
}

template <typename T>
size_t workspace_1d(int64_t batch, int64_t n, int64_t w) {
  if (batch == 0) return 0;
  if constexpr (sizeof(T) <= 4) {
    if (path_1d<T>(w) == Path1D::Warp)
      return MM_LW ? LwWs<T>::bytes(lw_geom<T>(batch, n, w)) : WarpWs<T>::bytes(warp_geom<T>(batch, n, w), batch);
  }
  if (path_1d<T>(w) != Path1D::Large) return 0;
  const int64_t TILE = Geo1D<T>::TILE;
  const int64_t m = n - w + 1;
  const int64_t tpr = (m + TILE - 1) / TILE;
  const int64_t q = (w - 1) / TILE;
  return LargeWs<T>::bytes(batch * (q + tpr));
}

template <typename K>
static int occupancy_grid(K kernel, size_t smem, int64_t ntiles, int &grid) {
  int per_sm = 0;
  int rc = blocks_per_sm(reinterpret_cast<const void *>(kernel), NT, smem, &per_sm);
  if (rc) return rc;
  if (per_sm < 1) per_sm = 1;
  int64_t cap = (int64_t)per_sm * sm_count();
  grid = (int)(ntiles < cap ? ntiles : cap);
  return kOK;
}

template <typename K>
static int set_smem(K kernel, size_t bytes, size_t &done) {
  (void)done;  // the limit is tracked per (kernel, device) under a lock: raise_smem_limit
  return raise_smem_limit(reinterpret_cast<const void *>(kernel), bytes);
}

template <typename T, int W, class Epi = StoreEpi>
static int launch_small(const Rows &p, const CUtensorMap &small, cudaStream_t s, Epi epi = Epi()) {
  TmaMaps map;  // 8-row boxes (the caller's map) and 32-row boxes over the same rows
  map.small = small;
  std::memset(&map.big, 0, sizeof(map.big));
  if (p.has_map) {
    int rc = encode_rows_map(&map.big, p.in, (int)sizeof(T), p.n / Rowing<T>::RW, p.batch,
                             p.in_ld * (int64_t)sizeof(T), kBigRows);
    if (rc) return rc;
  }
  constexpr size_t smem = SmallLayout<T, W>::BYTES;
  auto kern = k1d_small<T, W, Epi>;
  static size_t attr = 0;
  int rc = set_smem(kern, smem, attr);
  if (rc) return rc;
  int grid = 0;
  rc = occupancy_grid(kern, smem, p.ntiles, grid);
  if (rc) return rc;
  kern<<<grid, NT, smem, s>>>(p, map, epi);
  return note_cuda(cudaGetLastError());
}

template <typename T, class Epi = StoreEpi>
static int launch_small_epi(const Rows &p, const CUtensorMap &map, cudaStream_t s, Epi epi = Epi()) {
  switch (p.w) {
    case 2: return launch_small<T, 2, Epi>(p, map, s, epi);
    case 3: return launch_small<T, 3, Epi>(p, map, s, epi);
    case 4: return launch_small<T, 4, Epi>(p, map, s, epi);
    case 5: return launch_small<T, 5, Epi>(p, map, s, epi);
    case 6: return launch_small<T, 6, Epi>(p, map, s, epi);
    case 7: return launch_small<T, 7, Epi>(p, map, s, epi);
    case 8: return launch_small<T, 8, Epi>(p, map, s, epi);
    default: break;
  }
  if constexpr (Chunk<T>::E == 16) {
    switch (p.w) {
      case 9: return launch_small<T, 9, Epi>(p, map, s, epi);
      case 10: return launch_small<T, 10, Epi>(p, map, s, epi);
      case 11: return launch_small<T, 11, Epi>(p, map, s, epi);
      case 12: return launch_small<T, 12, Epi>(p, map, s, epi);
      case 13: return launch_small<T, 13, Epi>(p, map, s, epi);
      case 14: return launch_small<T, 14, Epi>(p, map, s, epi);
      case 15: return launch_small<T, 15, Epi>(p, map, s, epi);
      case 16: return launch_small<T, 16, Epi>(p, map, s, epi);
      default: break;
    }
  }
  return kErrUnsupported;
}

template <typename T>
static int launch_small_dispatch(const Rows &p, const CUtensorMap &map, cudaStream_t s) {
  return launch_small_epi<T>(p, map, s);
}

// Block geometry of k1d_medium: B = E*G, the largest power of two <= w-1 with
// 1 <= G <= 32; D = w-1-B = q'B + r'.
// Lanes per block of k1d_medium: the largest power of two G <= 32 with E*G <= w-1.
#ifndef MM_MED_GMAX  // largest group (lanes per block) of k1d_medium
#define MM_MED_GMAX 32
#endif
template <typename T>
int medium_G(int64_t w) {
  constexpr int E = Chunk<T>::E;
  int G = 1;
  while (G < MM_MED_GMAX && (int64_t)E * G * 2 <= w - 1) G *= 2;
  return G;
}

#ifndef MM_MED_RING3  // 1: k1d_medium's ring variant with three stages where two CTAs per SM fit
#define MM_MED_RING3 1
#endif
#ifndef MM_MED_DIRECT  // 1: k1d_medium's ring-free variant whenever q' = 0 (see k1d_medium.cuh)
#define MM_MED_DIRECT 1
#endif

// Block geometry of k1d_medium: B = E*G; D = w-1-B = q'B + r'.
template <typename T>
MedGeom medium_geom(int64_t w, int G) {
  constexpr int E = Chunk<T>::E;
  MedGeom g;
  g.B = E * G;
  const int64_t D = w - 1 - g.B;
  g.qp = (int)(D / g.B);
  g.rp = (int)(D % g.B);
  g.V = g.qp + (g.rp > 0 ? 1 : 0);
  g.need = (g.V * G + NT - 1) / NT;
  g.ring = 1;
  while (g.ring < g.V + 2 * (NT / G)) g.ring *= 2;
  return g;
}

template <typename T, int G, class Epi = StoreEpi>
static int launch_medium_g(const Rows &p, const CUtensorMap &small, cudaStream_t s, Epi epi = Epi()) {
  TmaMaps map;  // 8-row boxes (the caller's map) and 32-row boxes over the same rows
  map.small = small;
  std::memset(&map.big, 0, sizeof(map.big));
  if (p.has_map) {
    int rc = encode_rows_map(&map.big, p.in, (int)sizeof(T), p.n / Rowing<T>::RW, p.batch,
                             p.in_ld * (int64_t)sizeof(T), kBigRows);
    if (rc) return rc;
  }
  const MedGeom g = medium_geom<T>(p.w, G);
  // Variant and stage count by measurement on C2 (k1d_medium;
  // profiles/round2/session3/ab_medium_*.txt):
  //  * ring-free (DIRECT: groups reduce their own gap, no per-tile CTA
  //    barrier) for q' = 0, G >= 16 and a gap of at least half a block:
  //    w=1024 0.567 -> 0.531 ms (three-stage ring: 0.549);
  //  * the ring variant with three stages where it carries a gap (q' > 0, or
  //    r' > 0 with G >= 8): w=130 0.539 -> 0.522, w=600 0.572 -> 0.537,
  //    w=1025 0.547 -> 0.519, C5 w=4096 2.359 -> 2.295 ms;
  //  * two stages otherwise: gap-free (r' = 0) and G <= 4 windows run at
  //    0.94-0.99 of the copy peak with two and ~0.88 with three.
  if constexpr (G >= 16) {
    if (MM_MED_DIRECT && g.qp == 0 && 2 * g.rp >= g.B) {
      auto kern = k1d_medium<T, G, Epi, SameSrc<T>, true>;
      static size_t attr = 0;
      const size_t smem = MedLayout<T>::bytes(p.w, g.ring, MedStages<true>::N);
      int rc = set_smem(kern, smem, attr);
      if (rc) return rc;
      int grid = 0;
      rc = occupancy_grid(kern, smem, p.ntiles, grid);
      if (rc) return rc;
      kern<<<grid, NT, smem, s>>>(p, g, map, epi);
      return note_cuda(cudaGetLastError());
    }
  }
  if (MM_MED_RING3 && (g.qp > 0 || (g.rp > 0 && G >= 8)) &&
      2 * (MedLayout<T>::bytes(p.w, g.ring, 3) + 1024) <= 228 * 1024) {
    auto kern = k1d_medium<T, G, Epi, SameSrc<T>, false, 3>;
    static size_t attr = 0;
    const size_t smem = MedLayout<T>::bytes(p.w, g.ring, 3);
    int rc = set_smem(kern, smem, attr);
    if (rc) return rc;
    int grid = 0;
    rc = occupancy_grid(kern, smem, p.ntiles, grid);
    if (rc) return rc;
    kern<<<grid, NT, smem, s>>>(p, g, map, epi);
    return note_cuda(cudaGetLastError());
  }
  auto kern = k1d_medium<T, G, Epi>;
  static size_t attr = 0;
  const size_t smem = MedLayout<T>::bytes(p.w, g.ring);
  int rc = set_smem(kern, smem, attr);
  if (rc) return rc;
  int grid = 0;
  rc = occupancy_grid(kern, smem, p.ntiles, grid);
  if (rc) return rc;
  kern<<<grid, NT, smem, s>>>(p, g, map, epi);
  return note_cuda(cudaGetLastError());
}

template <typename T, class Epi = StoreEpi>
static int launch_medium_epi(const Rows &p, const CUtensorMap &map, cudaStream_t s, Epi epi = Epi()) {
  switch (medium_G<T>(p.w)) {
    case 1: return launch_medium_g<T, 1, Epi>(p, map, s, epi);
    case 2: return launch_medium_g<T, 2, Epi>(p, map, s, epi);
    case 4: return launch_medium_g<T, 4, Epi>(p, map, s, epi);
    case 8: return launch_medium_g<T, 8, Epi>(p, map, s, epi);
    case 16: return launch_medium_g<T, 16, Epi>(p, map, s, epi);
    default: return launch_medium_g<T, 32, Epi>(p, map, s, epi);
  }
}

template <typename T>
static int launch_medium(const Rows &p, const CUtensorMap &map, cudaStream_t s) {
  return launch_medium_epi<T>(p, map, s);
}

template <typename T>
static int launch_large(const Rows &p, const CUtensorMap &small, void *ws, size_t ws_bytes,
                        cudaStream_t s) {
  TmaMaps map;
  map.small = small;
  std::memset(&map.big, 0, sizeof(map.big));
  if (p.has_map) {
    int rc = encode_rows_map(&map.big, p.in, (int)sizeof(T), p.n / Rowing<T>::RW, p.batch,
                             p.in_ld * (int64_t)sizeof(T), kBigRows);
    if (rc) return rc;
  }
  constexpr int64_t TILE = Geo1D<T>::TILE;
  LargeGeom g;
  g.q = (int)((p.w - 1) / TILE);
  g.r = (int)((p.w - 1) % TILE);
  g.tickets_per_row = g.q + p.tiles_per_row;
  g.total = p.batch * g.tickets_per_row;
  if (!ws || ws_bytes < LargeWs<T>::bytes(g.total)) return kErrWorkspace;
  if (g.total > 0x7fffffffLL) return kErrUnsupported;
  cudaError_t e = cudaMemsetAsync(ws, 0, LargeWs<T>::zero_bytes(g.total), s);  // counter + flags
  if (e != cudaSuccess) return note_cuda(e);
  auto kern = k1d_large<T>;
  constexpr size_t smem = LargeLayout<T>::BYTES;
  static size_t attr = 0;
  int rc = set_smem(kern, smem, attr);
  if (rc) return rc;
  int grid = 0;
  rc = occupancy_grid(kern, smem, g.total, grid);
  if (rc) return rc;
  kern<<<grid, NT, smem, s>>>(p, g, ws, map);
  return note_cuda(cudaGetLastError());
}

template <typename T>
static int launch_lw(const Rows &p, void *ws, size_t ws_bytes, cudaStream_t s) {
  if constexpr (sizeof(T) > 4) {
    return kErrUnsupported;
  } else {
    using Geo = LwGeo<T>;
    // maps over the whole 128-B rows: chunks {RW, NROWS} (near chunks, the far
    // chunks' first NROWS rows) and single unswizzled rows (the far chunks' last)
    TmaMaps map;
    std::memset(&map, 0, sizeof(map));
    const int64_t full_rows = p.n / Rowing<T>::RW;
    int rc = encode_rows_map(&map.big, p.in, (int)sizeof(T), full_rows, p.batch,
                             p.in_ld * (int64_t)sizeof(T), Geo::NROWS);
    if (!rc)  // the far chunk's last row: one unswizzled row
      rc = encode_rows_map(&map.small, p.in, (int)sizeof(T), full_rows, p.batch,
                           p.in_ld * (int64_t)sizeof(T), 1, false);
    if (rc) return rc;
    const LwArgs g = lw_geom<T>(p.batch, p.n, p.w);
    if (!ws || ws_bytes < LwWs<T>::bytes(g)) return kErrWorkspace;
    if (g.total > 0x7fffffffLL) return kErrUnsupported;
    // every word's flag: one memset (256 B per 4096 outputs)
    cudaError_t e = cudaMemsetAsync(ws, 0, LwWs<T>::bytes(g), s);
    if (e != cudaSuccess) return note_cuda(e);
    // the far chunk's in-vector shift is a template parameter for 4-byte
    // types; the publication lead is three jobs for q <= MM_LW_L3_QMAX (C2
    // w=65536, q=127: 0.720 -> 0.690 ms) and two otherwise (C5 w=262144,
    // q=511: 3.215 ms with two, 3.276 with three)
    const bool l3 = g.q <= MM_LW_L3_QMAX;
    auto kern = l3 ? k1d_lw<T, -1, true> : k1d_lw<T, -1, false>;
    if constexpr (sizeof(T) == 4) {
      switch ((int)((p.w - 1) % Geo::VEC)) {
        case 0: kern = l3 ? k1d_lw<T, 0, true> : k1d_lw<T, 0, false>; break;
        case 1: kern = l3 ? k1d_lw<T, 1, true> : k1d_lw<T, 1, false>; break;
        case 2: kern = l3 ? k1d_lw<T, 2, true> : k1d_lw<T, 2, false>; break;
        default: kern = l3 ? k1d_lw<T, 3, true> : k1d_lw<T, 3, false>; break;
      }
    }
    const size_t smem = l3 ? LwGeo<T, true>::BYTES : LwGeo<T, false>::BYTES;
    rc = raise_smem_limit(reinterpret_cast<const void *>(kern), smem);
    if (rc) return rc;
    int grid = 0;
    rc = occupancy_grid(kern, smem, g.total, grid);
    if (rc) return rc;
    kern<<<grid, NT, smem, s>>>(p, g, ws, map);  // groups by ticket: no residency assumption
    return note_cuda(cudaGetLastError());
  }
}

template <typename T>
static int launch_warp(const Rows &p, void *ws, size_t ws_bytes, cudaStream_t s) {
  if constexpr (sizeof(T) > 4) {
    return kErrUnsupported;
  } else if constexpr (MM_LW) {
    return launch_lw<T>(p, ws, ws_bytes, s);
  } else {
    using Geo = WarpGeo<T>;
    // maps over the whole 128-B rows: near chunks {RW, 16} and far chunks {RW, 17}
    TmaMaps map;
    std::memset(&map, 0, sizeof(map));
    const int64_t full_rows = p.n / Rowing<T>::RW;
    int rc = encode_rows_map(&map.big, p.in, (int)sizeof(T), full_rows, p.batch,
                             p.in_ld * (int64_t)sizeof(T), Geo::NROWS);
    if (!rc)
      rc = encode_rows_map(&map.small, p.in, (int)sizeof(T), full_rows, p.batch,
                           p.in_ld * (int64_t)sizeof(T), Geo::FROWS);
    if (rc) return rc;
    const WarpLB g = warp_geom<T>(p.batch, p.n, p.w);
    if (!ws || ws_bytes < WarpWs<T>::bytes(g, p.batch)) return kErrWorkspace;
    if (g.total > 0x7fffffffLL) return kErrUnsupported;
    // every slot flag: one memset (32 B per 512 outputs)
    cudaError_t e = cudaMemsetAsync(ws, 0, WarpWs<T>::bytes(g, p.batch), s);
    if (e != cudaSuccess) return note_cuda(e);
    // the far chunk's in-vector shift is a template parameter for 4-byte types
    auto kern = k1d_warp<T, -1>;
    if constexpr (sizeof(T) == 4) {
      switch ((int)((p.w - 1) % Geo::VEC)) {
        case 0: kern = k1d_warp<T, 0>; break;
        case 1: kern = k1d_warp<T, 1>; break;
        case 2: kern = k1d_warp<T, 2>; break;
        default: kern = k1d_warp<T, 3>; break;
      }
    }
    constexpr size_t smem = Geo::BYTES;
    rc = raise_smem_limit(reinterpret_cast<const void *>(kern), smem);
    if (rc) return rc;
    int grid = 0;
#if MM_WARP_CONTIG
    rc = occupancy_grid(kern, smem, (g.total + NWARP - 1) / NWARP, grid);
    if (rc) return rc;
    kern<<<grid, NT, smem, s>>>(p, g, ws, map);
    return note_cuda(cudaGetLastError());
#else
    // every CTA resident (cooperative launch): gaps wait on other CTAs' groups
    rc = occupancy_grid(kern, smem, g.total, grid);
    if (rc) return rc;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return note_cuda(cudaLaunchKernelEx(&cfg, kern, p, g, ws, map));
#endif
  }
}

// Batched 1-D filter (1-D is batch 1).  Arguments already validated.
template <typename T>
int launch_1d(const void *in, int64_t batch, int64_t n, int64_t in_ld, int64_t w, void *out_max,
              void *out_min, int64_t out_ld, void *ws, size_t ws_bytes, cudaStream_t s) {
  if (batch == 0) return kOK;
  const int64_t m = n - w + 1;
  if (w == 1) {  // identity: both outputs are copies of the input
    for (void *o : {out_max, out_min}) {
      if (!o) continue;
      cudaError_t e = cudaMemcpy2DAsync(o, (size_t)out_ld * sizeof(T), in, (size_t)in_ld * sizeof(T),
                                        (size_t)n * sizeof(T), (size_t)batch,
                                        cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) return note_cuda(e);
    }
    return kOK;
  }
  Rows p;
  p.in = in;
  p.out_max = out_max;
  p.out_min = out_min;
  p.n = n;
  p.w = w;
  p.m = m;
  p.in_ld = in_ld;
  p.out_ld = out_ld;
  p.batch = batch;
  p.tiles_per_row = (m + Geo1D<T>::TILE - 1) / Geo1D<T>::TILE;
  p.ntiles = batch * p.tiles_per_row;
  // TMA map over the whole 128-B rows of every series
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  const int64_t full_rows = n / Rowing<T>::RW;
  p.has_map = full_rows > 0 ? 1 : 0;
  if (p.has_map) {
    int rc = encode_rows_map(&map, in, (int)sizeof(T), full_rows, batch, in_ld * (int64_t)sizeof(T));
    if (rc) return rc;
  }
  switch (path_1d<T>(w)) {
    case Path1D::Small: return launch_small_dispatch<T>(p, map, s);
    case Path1D::Medium: return launch_medium<T>(p, map, s);
    case Path1D::Large: return launch_large<T>(p, map, ws, ws_bytes, s);
    case Path1D::Warp: return launch_warp<T>(p, ws, ws_bytes, s);
    default: return kErrUnsupported;
  }
}

template <typename T>
size_t smem_2d(int64_t w_row, int64_t w_col) {
  return K2Tile<T>::bytes((int)w_row, (int)w_col);
}

template <typename T>
int launch_2d(const void *in, int64_t batch, int64_t rows, int64_t cols, int64_t in_ld,
              int64_t in_bstride, int64_t w_row, int64_t w_col, void *out_max, void *out_min,
              int64_t out_ld, int64_t out_bstride, cudaStream_t s) {
  if (batch == 0) return kOK;
  if constexpr (sizeof(T) == 1) {
    const int rc = launch_2d_byte(std::is_signed<T>::value, in, batch, rows, cols, in_ld, in_bstride,
                                  w_row, w_col, out_max, out_min, out_ld, out_bstride, s);
    if (rc != kErrUnsupported) return rc;
  }
  const size_t smem = smem_2d<T>(w_row, w_col);
  if (smem > 200 * 1024) return kErrUnsupported;
  auto kern = k2d_generic<T>;
  static size_t attr = 0;
  int rc = set_smem(kern, 200 * 1024, attr);
  if (rc) return rc;
  Img2D p;
  p.in = in;
  p.out_max = out_max;
  p.out_min = out_min;
  p.batch = batch;
  p.rows = rows;
  p.cols = cols;
  p.in_ld = in_ld;
  p.in_bstride = in_bstride;
  p.out_ld = out_ld;
  p.out_bstride = out_bstride;
  p.w_row = (int)w_row;
  p.w_col = (int)w_col;
  const int64_t Ro = rows - w_col + 1, Co = cols - w_row + 1;
  p.tiles_x = (Co + K2Tile<T>::TW - 1) / K2Tile<T>::TW;
  p.tiles_y = (Ro + K2Tile<T>::TH - 1) / K2Tile<T>::TH;
  const int64_t grid = batch * p.tiles_x * p.tiles_y;
  if (grid > 0x7fffffffLL) return kErrUnsupported;
  kern<<<(unsigned)grid, NT2, smem, s>>>(p);
  return note_cuda(cudaGetLastError());
}

// Explicit instantiation declarations (definitions in inst_<t>.cu).
#define MM_DECLARE_INST(T)                                                                     \
  extern template int launch_1d<T>(const void *, int64_t, int64_t, int64_t, int64_t, void *,   \
                                   void *, int64_t, void *, size_t, cudaStream_t);             \
  extern template size_t workspace_1d<T>(int64_t, int64_t, int64_t);                          \
  extern template int launch_2d<T>(const void *, int64_t, int64_t, int64_t, int64_t, int64_t,  \
                                   int64_t, int64_t, void *, void *, int64_t, int64_t,         \
                                   cudaStream_t);                                              \
  extern template size_t smem_2d<T>(int64_t, int64_t);

#define MM_DEFINE_INST(T)                                                                      \
  template int launch_1d<T>(const void *, int64_t, int64_t, int64_t, int64_t, void *, void *,  \
                            int64_t, void *, size_t, cudaStream_t);                            \
  template size_t workspace_1d<T>(int64_t, int64_t, int64_t);                                  \
  template int launch_2d<T>(const void *, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, \
                            int64_t, void *, void *, int64_t, int64_t, cudaStream_t);          \
  template size_t smem_2d<T>(int64_t, int64_t);

}  // namespace mm

// k1d_small.cuh -- compile-time small-window 1-D kernel (see k1d.cuh).
#pragma once

#include "k1d_base.cuh"

namespace mm {

// ===================================================================== small
// 2 <= W <= E.  Thread c owns outputs [cE, cE+E) of the tile and needs inputs
// [cE, cE+E+W-1).  Log-step doubling: after the step of span s, m[p] = max
// a[p .. p+2s); out = max(m_{2^K}[j], m_{2^K}[j+W-2^K]) (max is idempotent).
template <typename T, int W>
struct SmallLayout {
  static constexpr int E = Chunk<T>::E;
  static constexpr int TILE = NT * E;
  static constexpr int RW = Rowing<T>::RW;
  static constexpr int ROWS = ((TILE + E + RW - 1) / RW + kBoxRows - 1) / kBoxRows * kBoxRows;
  static constexpr int STAGE = ROWS * 128;
  static constexpr size_t BYTES = 2 * (size_t)STAGE + 1024 + 64;
};

template <typename T, int W, class Epi = StoreEpi>
__global__ void __launch_bounds__(NT) k1d_small(Rows p, const __grid_constant__ TmaMaps maps,
                                                Epi epi = Epi()) {
  using Lay = SmallLayout<T, W>;
  constexpr int E = Lay::E;
  constexpr int VEC = Chunk<T>::VEC;
  constexpr int TILE = Lay::TILE;
  constexpr int NXT = (W - 1 + VEC - 1) / VEC * VEC;  // elements read from the next chunk
  constexpr int K = W >= 16 ? 4 : W >= 8 ? 3 : W >= 4 ? 2 : 1;
  constexpr int SPAN = 1 << K;
  static_assert(W >= 2 && W <= E, "small path: 2 <= W <= E");

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *base = smem_align1024(smem_raw);
  auto stg = [&](int i) { return base + i * Lay::STAGE; };
  uint64_t *bars = reinterpret_cast<uint64_t *>(base + 2 * Lay::STAGE);
  const int tid = threadIdx.x;

  if (tid == 0) {
    prefetch_tmap(&maps.big);
    prefetch_tmap(&maps.small);
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  int64_t t_begin, t_end;
  cta_tile_range(p, t_begin, t_end);
  TileCursor<TILE> cur, nxt;
  cur.start(p, t_begin);
  nxt = cur;
  if (tid == 0 && t_begin < t_end)
    stage_tile2<T>(p, &maps, stg(0), cur.row, cur.u0, cur.tout(p) + W - 1, &bars[0]);
  int it = 0;
  for (int64_t t = t_begin; t < t_end; ++t, ++it, cur = nxt) {
    const int st = it & 1;
    unsigned char *X = stg(st);
    nxt.advance(p);
    if (tid == 0 && t + 1 < t_end)  // prefetch the next tile into the other stage
      stage_tile2<T>(p, &maps, stg(st ^ 1), nxt.row, nxt.u0, nxt.tout(p) + W - 1, &bars[st ^ 1]);
    const int64_t row = cur.row, u0 = cur.u0;
    const int tout = cur.tout(p);
    mbar_wait(&bars[st], (it >> 1) & 1);
    if (patch_tail<T>(p, X, row, u0, tout + W - 1, tid)) __syncthreads();

    const int c0 = tid * E;
    {  // every thread computes (lanes past tout on stale data): the epilogue may be collective
      T v[E + NXT];
      {
        T a[E], b[NXT];
        lds_swz_aligned<T, E>(X, c0, a);
        lds_swz_aligned<T, NXT>(X, c0 + E, b);
#pragma unroll
        for (int k = 0; k < E; ++k) v[k] = a[k];
#pragma unroll
        for (int k = 0; k < NXT; ++k) v[E + k] = b[k];
      }
      constexpr int NV = E + W - 1;
      T mx[NV], mn[NV];
#pragma unroll
      for (int k = 0; k < NV; ++k) mx[k] = mn[k] = v[k];
#pragma unroll
      for (int s = 1; s < SPAN; s *= 2) {
#pragma unroll
        for (int q = 0; q + 2 * s <= NV; ++q) {  // ascending: m[q+s] is still the old value
          mx[q] = Ord<T>::mx(mx[q], mx[q + s]);
          mn[q] = Ord<T>::mn(mn[q], mn[q + s]);
        }
      }
      T ox[E], on[E];
#pragma unroll
      for (int j = 0; j < E; ++j) {
        if (W == SPAN) {
          ox[j] = mx[j];
          on[j] = mn[j];
        } else {
          ox[j] = Ord<T>::mx(mx[j], mx[j + (W - SPAN)]);
          on[j] = Ord<T>::mn(mn[j], mn[j + (W - SPAN)]);
        }
      }
      epi(p, row, u0 + c0, tout - c0, ox, on);
    }
    __syncthreads();  // stage st is free for the prefetch of iteration it+1
  }
}

}  // namespace mm

// k1d_medium.cuh -- runtime medium-window 1-D kernel (see k1d_base.cuh).
#pragma once

#include "k1d_base.cuh"

namespace mm {

// ==================================================================== medium
// Runtime w with E < w <= kHaloMax+1.  Block B = E*G (G lanes, a power of two,
// B <= w-1; B = 32E when w-1 >= 32E).  Thread t owns the near chunk [tE, tE+E)
// of outputs and the far chunk [tE+w-1, tE+w-1+E) of inputs; group g = t/G owns
// near block [gB, gB+B) and far block F_g = [gB+w-1, gB+B+w-1).  With D = w-1-B
// = q'B + r', the gap [gB+B, gB+w-1) of every window of near block g is
//   the last r' elements of F_{g-q'-1}  and  F_{g-q'} .. F_{g-1},
// so out = max(S_local, P_local, C_t) with C_t = max(S-carry, P-carry, gap) one
// per-thread constant.
//
// Far-block aggregates (G = max of a far block, H = max of its last r'
// elements) go to a ring indexed by the block's position in the row.  Each CTA
// processes a contiguous range of tiles, so the far blocks "before" a tile
// (g < 0) are the previous tile's blocks, already in the ring; only the first
// tiles of a CTA range or of a row reduce them from the staged halo.
// G is a template parameter: the group scans unroll without branches.
struct MedGeom {
  int B;     // E * G
  int qp;    // q'
  int rp;    // r'
  int V;     // far blocks before the tile needed by its gaps: q' + (r' > 0)
  int need;  // previous tiles that hold those V blocks: ceil(V*G / NT)
  int ring;  // ring entries: a power of two >= V + 2*NT/G
};

template <typename T>
struct MedLayout {
  static constexpr int E = Chunk<T>::E;
  static constexpr int TILE = NT * E;
  static constexpr int RW = Rowing<T>::RW;
  __host__ __device__ static int rows(int64_t w) {
    int r = (int)((TILE + w - 1 + 16 + RW - 1) / RW);  // + margin for shifted 16-B reads
    return (r + kBoxRows - 1) / kBoxRows * kBoxRows;
  }
  __host__ __device__ static size_t stage_bytes(int64_t w) { return (size_t)rows(w) * 128; }
  __host__ __device__ static size_t bytes(int64_t w, int ring, int nstg = 2) {
    return 1024 + nstg * stage_bytes(w) + 4 * sizeof(T) * (size_t)ring + 64;
  }
};

// inclusive max/min scans and reductions over aligned groups of G lanes
template <typename T, int G>
__device__ __forceinline__ void grp_reduce(T &vx, T &vn) {
#pragma unroll
  for (int d = 1; d < G; d <<= 1) {
    vx = Ord<T>::mx(vx, __shfl_xor_sync(0xffffffffu, vx, d));
    vn = Ord<T>::mn(vn, __shfl_xor_sync(0xffffffffu, vn, d));
  }
}
template <typename T, int G>
__device__ __forceinline__ void grp_scan_up(T &vx, T &vn, int gl) {
#pragma unroll
  for (int d = 1; d < G; d <<= 1) {
    (void)gl;  // lanes below d of their group get their own value back (idempotent step)
    vx = Ord<T>::mx(vx, shfl_up_seg(vx, d, G));
    vn = Ord<T>::mn(vn, shfl_up_seg(vn, d, G));
  }
}
template <typename T, int G>
__device__ __forceinline__ void grp_scan_down(T &vx, T &vn, int gl) {
#pragma unroll
  for (int d = 1; d < G; d <<= 1) {
    (void)gl;
    vx = Ord<T>::mx(vx, shfl_down_seg(vx, d, G));
    vn = Ord<T>::mn(vn, shfl_down_seg(vn, d, G));
  }
}

// Source of the values a tile is filtered on.  SameSrc: the staged elements
// themselves (both chains read them).  Other sources (argfilter.cu's ArgSrc)
// stage elements of another type S and build the max chain's and the min
// chain's values from them and their row positions inside the loads.
template <typename T>
struct SameSrc {
  using S = T;
  static constexpr bool TWO = false;
  template <int E>
  __device__ __forceinline__ static void load(const unsigned char *X, int pos, int64_t, T (&ya)[E], T (&yb)[E]) {
    lds_swz<T, E>(X, pos, ya);
#pragma unroll
    for (int k = 0; k < E; ++k) yb[k] = ya[k];
  }
  template <int E>
  __device__ __forceinline__ static void load_aligned(const unsigned char *X, int pos, int64_t, T (&ya)[E],
                                                      T (&yb)[E]) {
    lds_swz_aligned<T, E>(X, pos, ya);
#pragma unroll
    for (int k = 0; k < E; ++k) yb[k] = ya[k];
  }
};

// shared-memory layout for a tile of T-windows staged as S elements
template <typename T, typename S>
struct MedLayoutS {
  static constexpr int TILE = MedLayout<T>::TILE;
  static constexpr int RW = Rowing<S>::RW;
  __host__ __device__ static int rows(int64_t w) {
    int r = (int)((TILE + w - 1 + 16 + RW - 1) / RW);
    return (r + kBoxRows - 1) / kBoxRows * kBoxRows;
  }
  __host__ __device__ static size_t stage_bytes(int64_t w) { return (size_t)rows(w) * 128; }
  __host__ __device__ static size_t bytes(int64_t w, int ring, int nstg = 2) {
    return 1024 + nstg * stage_bytes(w) + 4 * sizeof(T) * (size_t)ring + 64;
  }
};

// MM_MED_SPLIT: the per-tile CTA barrier split into mbarrier hand-offs -- the
// ring is "ready" once every warp has published its far-block aggregates (one
// arrival per warp right after the far chunk, waited on just before the gap,
// so the near-chunk scan runs in between), and a stage is "empty" once every
// warp has consumed its loads (only the producer thread waits, before the next
// prefetch into it).
#ifndef MM_MED_SPLIT
#define MM_MED_SPLIT 0
#endif

// DIRECT (q' = 0, i.e. w-1 < 2B: every w <= 32E+1): the gap of group g is
// only H_{g-1}, the last r' elements of F_{g-1} = [gB-B+w-1, gB+w-1), and the
// tile's stage holds F_{g-1} (w-1 >= B).  So the group reduces it itself from
// the stage instead of reading the aggregate its predecessor published: no
// ring, no cross-warp dependency and no per-tile CTA barrier.  Three stages;
// a stage is recycled once every warp has arrived on its "empty" mbarrier.
// NS (ring variant): 2 stages, the next tile prefetched at the start of a
// tile; or 3, the tile it+3 issued right after tile it's barrier.
template <int DIRECT>
struct MedStages {
  static constexpr int N = DIRECT ? 3 : 2;
};

template <typename T, int G, class Epi = StoreEpi, class Src = SameSrc<T>, bool DIRECT = false,
          int NS = MedStages<DIRECT>::N>
__global__ void __launch_bounds__(NT, 2)
    k1d_medium(Rows p, MedGeom g, const __grid_constant__ TmaMaps maps, Epi epi = Epi()) {
  using Lay = MedLayout<T>;
  using S = typename Src::S;
  using LayS = MedLayoutS<T, S>;
  constexpr bool TWO = Src::TWO;
  constexpr int E = Lay::E;
  constexpr int TILE = Lay::TILE;
  constexpr int B = E * G;
  constexpr int NG = NT / G;  // groups per tile
  const int RMASK = g.ring - 1;
  const int w = (int)p.w;
  const size_t SB = LayS::stage_bytes(w);

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *base = smem_align1024(smem_raw);
  auto stg = [&](int i) { return base + i * SB; };
  constexpr int NSTG = NS;
  static_assert(!DIRECT || NS == 3, "the ring-free variant runs three stages");
  static_assert(!MM_MED_SPLIT || NS == 2, "the split-barrier build runs two stages");
  T *Rgx = reinterpret_cast<T *>(base + NSTG * SB);  // ring of far-block aggregates (unused if DIRECT)
  T *Rgn = Rgx + g.ring;
  T *Rhx = Rgn + g.ring;
  T *Rhn = Rhx + g.ring;
  uint64_t *bars = reinterpret_cast<uint64_t *>(base + NSTG * SB + 4 * sizeof(T) * g.ring);

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int gl = lane & (G - 1);
  const int grp = tid / G;
  const int glast = (lane & ~(G - 1)) + G - 1;  // last lane of this lane's group
  // H range inside a far block: block offsets [B - r', B)
  const int hstart = B - g.rp;
  const int h_lane = hstart / E, h_off = hstart - (hstart / E) * E;

  int64_t t_begin, t_end;
  cta_tile_range(p, t_begin, t_end);
  TileCursor<TILE> cur, nxt;
  cur.start(p, t_begin);
  nxt = cur;

  if (tid == 0) {
    prefetch_tmap(&maps.big);
    prefetch_tmap(&maps.small);
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    if (NSTG == 3) mbar_init(&bars[2], 1);  // stage 2 full
    if (DIRECT) {
      for (int i = 0; i < NSTG; ++i) reinterpret_cast<uint32_t *>(bars + NSTG)[i] = 0;  // stage i: warps done
    }
#if MM_MED_SPLIT
    mbar_init(&bars[2], NT / 32);  // stage 0 empty
    mbar_init(&bars[3], NT / 32);  // stage 1 empty
    mbar_init(&bars[4], NT / 32);  // ring ready
#endif
    fence_mbar_init();
  }
  __syncthreads();
  TileCursor<TILE> pf = cur;  // DIRECT: tile it+NSTG during tile it
  uint32_t *done = reinterpret_cast<uint32_t *>(bars + NSTG);  // DIRECT: per stage, warps done with it
  if (tid == 0 && t_begin < t_end) {
    stage_tile2<S>(p, &maps, stg(0), cur.row, cur.u0, cur.tout(p) + w - 1, &bars[0]);
    for (int k = 1; NSTG == 3 && k < NSTG; ++k) {
      pf.advance(p);
      if (t_begin + k < t_end) stage_tile2<S>(p, &maps, stg(k), pf.row, pf.u0, pf.tout(p) + w - 1, &bars[k]);
    }
  }
  if (NSTG == 3) {
    pf = cur;
    for (int k = 0; k < NSTG; ++k) pf.advance(p);
  }

  // H contribution of a chunk y (block-relative chunk gl) given its local max
  auto h_part = [&](const T (&y)[E], T ax, T an, T bl, T &hx, T &hn) {
    hx = hn = bl;  // the block's last element: inside every non-empty H range
    if (g.rp > 0) {
      if (gl > h_lane) {
        hx = Ord<T>::mx(hx, ax);
        hn = Ord<T>::mn(hn, an);
      } else if (gl == h_lane) {
        T vx, vn;
        suffix_from<T, E>(y, h_off, vx, vn);
        hx = Ord<T>::mx(hx, vx);
        hn = Ord<T>::mn(hn, vn);
      }
    }
  };

  int it = 0, st = 0;
  for (int64_t t = t_begin; t < t_end; ++t, ++it, st = st + 1 == NSTG ? 0 : st + 1) {
    const unsigned char *X = stg(st);
    nxt.advance(p);
    if (NSTG == 3) {
      // (the stage is refilled once every warp is done with it: see below)
    } else if (tid == 0 && t + 1 < t_end) {  // prefetch the next tile into the other stage
#if MM_MED_SPLIT
      if (it > 0) mbar_wait(&bars[2 + (st ^ 1)], ((it - 1) >> 1) & 1);  // tile it-1 consumed it
#endif
      stage_tile2<S>(p, &maps, stg(st ^ 1), nxt.row, nxt.u0, nxt.tout(p) + w - 1, &bars[st ^ 1]);
    }
    const int64_t row = cur.row, u0 = cur.u0;
    const int tout = cur.tout(p);
    const int64_t ab0 = u0 / B;  // far block index (within the row) of group 0
    mbar_wait(&bars[st], (it / NSTG) & 1);
    if (patch_tail<S>(p, stg(st), row, u0, tout + w - 1, tid)) __syncthreads();

    // ------------------------------------------------- far chunk: prefix
    // ux/un end up as max(P, S) per element: local prefix of the far chunk
    // folded with the local suffix of the near chunk (carries go into cx/cn)
    T ux[E], un[E];
    T cx, cn;
    T dgx, dgn;  // DIRECT: the gap H_{g-1}
    {
      T ya[E], yb[E];
      Src::template load<E>(X, tid * E + w - 1, u0, ya, yb);
      ux[0] = ya[0];
      un[0] = yb[0];
#pragma unroll
      for (int k = 1; k < E; ++k) {
        ux[k] = Ord<T>::mx(ux[k - 1], ya[k]);
        un[k] = Ord<T>::mn(un[k - 1], yb[k]);
      }
      T hx, hn, tx, tn;
      if (!DIRECT) {
        h_part(ya, ux[E - 1], un[E - 1], __shfl_sync(0xffffffffu, ya[E - 1], glast), hx, tn);
        if (TWO) h_part(yb, ux[E - 1], un[E - 1], __shfl_sync(0xffffffffu, yb[E - 1], glast), tx, hn);
        else hn = tn;
        grp_reduce<T, G>(hx, hn);
      }
      T ax = ux[E - 1], an = un[E - 1];  // group-inclusive prefix of chunk maxima
      grp_scan_up<T, G>(ax, an, gl);
      cx = shfl_up(ax, 1);
      cn = shfl_up(an, 1);
      if (gl == 0) {  // nothing before: an element inside every window
        cx = ya[0];
        cn = yb[0];
      }
      if (DIRECT) {
        // gap = H_{g-1}: this lane's chunk of F_{g-1} (B before its far chunk)
        hx = hn = cx;  // (placeholders: replaced below when r' > 0)
        if (g.rp > 0) {
          T za[E], zb[E];
          Src::template load<E>(X, tid * E + w - 1 - B, u0, za, zb);
          T zx = za[0], zn = zb[0];
#pragma unroll
          for (int k = 1; k < E; ++k) {
            zx = Ord<T>::mx(zx, za[k]);
            zn = Ord<T>::mn(zn, zb[k]);
          }
          h_part(za, zx, zn, __shfl_sync(0xffffffffu, za[E - 1], glast), hx, tn);
          if (TWO) h_part(zb, zx, zn, __shfl_sync(0xffffffffu, zb[E - 1], glast), tx, hn);
          else hn = tn;
          grp_reduce<T, G>(hx, hn);
        }
        dgx = hx;
        dgn = hn;
      } else if (gl == G - 1) {  // publish far block aggregates G_g, H_g
        const int ri = (int)((ab0 + grp) & RMASK);
        Rgx[ri] = ax;
        Rgn[ri] = an;
        Rhx[ri] = hx;
        Rhn[ri] = hn;
      }
    }

    // ---------------- far blocks before the tile (first tiles of a range/row)
    auto far_blocks_before = [&]() {
      const int64_t tile_in_row = u0 / TILE;
      if (g.V > 0 && (t - t_begin < g.need || tile_in_row < g.need)) {
        const int nv = g.V * G;  // chunks of the V blocks
        for (int r0 = 0; r0 < nv; r0 += NT) {
          const int vc = r0 + tid;
          if (r0 + (tid & ~31) >= nv) break;  // whole warp idle (warp-uniform)
          const int vcc = vc < nv ? vc : nv - 1;
          const int gv = vcc / G;  // 0 .. V-1  <->  g' = gv - V
          const int pos = (gv - g.V) * B + w - 1 + gl * E;
          T ya[E], yb[E];
          Src::template load<E>(X, pos, u0, ya, yb);
          T ax = ya[0], an = yb[0];
#pragma unroll
          for (int k = 1; k < E; ++k) {
            ax = Ord<T>::mx(ax, ya[k]);
            an = Ord<T>::mn(an, yb[k]);
          }
          T hx, hn, tx, tn;
          h_part(ya, ax, an, __shfl_sync(0xffffffffu, ya[E - 1], glast), hx, tn);
          if (TWO) h_part(yb, ax, an, __shfl_sync(0xffffffffu, yb[E - 1], glast), tx, hn);
          else hn = tn;
          grp_reduce<T, G>(ax, an);
          grp_reduce<T, G>(hx, hn);
          if (vc < nv && gl == 0) {
            const int ri = (int)((ab0 + gv - g.V) & RMASK);
            Rgx[ri] = ax;
            Rgn[ri] = an;
            Rhx[ri] = hx;
            Rhn[ri] = hn;
          }
        }
      }
    };
#if MM_MED_SPLIT
    if (!DIRECT) {
      far_blocks_before();
      __syncwarp();
      if (lane == 0) mbar_arrive1(&bars[4]);  // this warp's ring entries are written
    }
#endif

    // ------------------------------------------------ near chunk: suffix
    {
      T xa[E], xb[E];
      Src::template load_aligned<E>(X, tid * E, u0, xa, xb);
      T sx = xa[E - 1], sn = xb[E - 1];
      ux[E - 1] = Ord<T>::mx(ux[E - 1], sx);
      un[E - 1] = Ord<T>::mn(un[E - 1], sn);
#pragma unroll
      for (int k = E - 2; k >= 0; --k) {
        sx = Ord<T>::mx(sx, xa[k]);
        sn = Ord<T>::mn(sn, xb[k]);
        ux[k] = Ord<T>::mx(ux[k], sx);
        un[k] = Ord<T>::mn(un[k], sn);
      }
      T bx = sx, bn = sn;  // group-inclusive suffix of chunk maxima
      grp_scan_down<T, G>(bx, bn, gl);
      T ex = shfl_down(bx, 1), en = shfl_down(bn, 1);
      if (gl == G - 1) {  // nothing after: an element inside every window of the chunk
        ex = xa[E - 1];
        en = xb[E - 1];
      }
      cx = Ord<T>::mx(cx, ex);
      cn = Ord<T>::mn(cn, en);
    }

    if (DIRECT) {
      // the last warp done with stage st refills it with tile it+NSTG: nobody waits
      __syncwarp();
      if (lane == 0 && atom_add_shared_u32(&done[st], 1u) == NT / 32 - 1) {
        done[st] = 0;  // (every warp has arrived for this use; the next use follows the refill)
        if (t + NSTG < t_end) stage_tile2<S>(p, &maps, stg(st), pf.row, pf.u0, pf.tout(p) + w - 1, &bars[st]);
      }
      pf.advance(p);
      if (g.rp > 0) {
        cx = Ord<T>::mx(cx, dgx);
        cn = Ord<T>::mn(cn, dgn);
      }
    } else {
#if MM_MED_SPLIT
    __syncwarp();
    if (lane == 0) mbar_arrive1(&bars[2 + st]);  // this warp is done with the stage
    mbar_wait(&bars[4], it & 1);                 // every warp's ring entries of this tile
#else
    far_blocks_before();
    __syncthreads();
    if (NSTG == 3) {  // every warp is done with stage st: refill it with tile it+3
      if (tid == 0 && t + NSTG < t_end) stage_tile2<S>(p, &maps, stg(st), pf.row, pf.u0, pf.tout(p) + w - 1, &bars[st]);
      pf.advance(p);
    }
#endif

    // ---------------------------------------------------------- gap
    if (g.qp > 0 || g.rp > 0) {
      const int64_t b0 = ab0 + grp - g.qp - 1;  // far block F_{g-q'-1}
      T mx, mn;
      if (g.rp > 0) {
        mx = Rhx[b0 & RMASK];
        mn = Rhn[b0 & RMASK];
      } else {
        mx = Rgx[(b0 + 1) & RMASK];
        mn = Rgn[(b0 + 1) & RMASK];
      }
      for (int s = 1; s <= g.qp; ++s) {
        mx = Ord<T>::mx(mx, Rgx[(b0 + s) & RMASK]);
        mn = Ord<T>::mn(mn, Rgn[(b0 + s) & RMASK]);
      }
      cx = Ord<T>::mx(cx, mx);
      cn = Ord<T>::mn(cn, mn);
    }
    }  // !DIRECT
    // ---------------------------------------------------------- out
    const int c0 = tid * E;
    {
      T ox[E], on[E];
#pragma unroll
      for (int k = 0; k < E; ++k) {
        ox[k] = Ord<T>::mx(ux[k], cx);
        on[k] = Ord<T>::mn(un[k], cn);
      }
      epi(p, row, u0 + c0, tout - c0, ox, on);  // (every thread: the epilogue may be collective)
    }
    // No barrier needed before the next tile in steady state: stage st was last
    // read before this tile's barrier (the prefetch into it is issued after it),
    // and the ring holds >= V + 2*NT/G entries, so the next tile's writes never
    // alias this tile's reads.  A fresh next tile rewrites the V entries before
    // it: wait for this tile's readers first.
    if (!DIRECT && t + 1 < t_end && g.V > 0 && (t + 1 - t_begin < g.need || nxt.u0 / TILE < g.need))
      __syncthreads();
    cur = nxt;
  }
  (void)NG;
}

}  // namespace mm

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
    default: break;
  }
#undef MM_SUF_CASE
}

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

template <typename T, int W>
__global__ void __launch_bounds__(NT) k1d_small(Rows p, const __grid_constant__ CUtensorMap map) {
  using Lay = SmallLayout<T, W>;
  constexpr int E = Lay::E;
  constexpr int VEC = Chunk<T>::VEC;
  constexpr int TILE = Lay::TILE;
  constexpr int NXT = (W - 1 + VEC - 1) / VEC * VEC;  // elements read from the next chunk
  constexpr int K = W >= 16 ? 4 : W >= 8 ? 3 : W >= 4 ? 2 : 1;
  constexpr int SPAN = 1 << K;
  static_assert(W >= 2 && W <= E, "small path: 2 <= W <= E");

  extern __shared__ unsigned char smem_raw[];
  unsigned char *base = reinterpret_cast<unsigned char *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  auto stg = [&](int i) { return base + i * Lay::STAGE; };
  uint64_t *bars = reinterpret_cast<uint64_t *>(base + 2 * Lay::STAGE);
  const int tid = threadIdx.x;

  if (tid == 0) {
    prefetch_tmap(&map);
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t grid = gridDim.x;
  if (tid == 0 && (int64_t)blockIdx.x < p.ntiles) {
    int64_t row, u0;
    int tout;
    tile_coords<TILE>(p, blockIdx.x, row, u0, tout);
    stage_tile<T>(p, &map, stg(0), row, u0, tout + W - 1, &bars[0]);
  }
  int it = 0;
  for (int64_t t = blockIdx.x; t < p.ntiles; t += grid, ++it) {
    const int st = it & 1;
    unsigned char *X = stg(st);
    if (tid == 0 && t + grid < p.ntiles) {  // prefetch the next tile into the other stage
      int64_t row, u0;
      int tout;
      tile_coords<TILE>(p, t + grid, row, u0, tout);
      stage_tile<T>(p, &map, stg(st ^ 1), row, u0, tout + W - 1, &bars[st ^ 1]);
    }
    int64_t row, u0;
    int tout;
    tile_coords<TILE>(p, t, row, u0, tout);
    mbar_wait(&bars[st], (it >> 1) & 1);
    if (patch_tail<T>(p, X, row, u0, tout + W - 1, tid)) __syncthreads();

    const int c0 = tid * E;
    if (c0 < tout) {
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
      store_out<T, E>(p, row, u0 + c0, tout - c0, ox, on);
    }
    __syncthreads();  // stage st is free for the prefetch of iteration it+1
  }
}

// ==================================================================== medium
// Runtime w with E < w <= kHaloMax+1.  Block B = E*G (G lanes, a power of two,
// B <= w-1; B = 32E when w-1 >= 32E).  Thread t owns the near chunk [tE, tE+E)
// of outputs and the far chunk [tE+w-1, tE+w-1+E) of inputs; group g = t/G owns
// near block [gB, gB+B) and far block F_g = [gB+w-1, gB+B+w-1).  With D = w-1-B
// = q'B + r', the gap [gB+B, gB+w-1) of every window of near block g is
//   the last r' elements of F_{g-q'-1}  and  F_{g-q'} .. F_{g-1},
// so out = max(s_local, p_local, C_t), C_t = max(S-carry, P-carry, gap) is one
// per-thread constant.  Far blocks g' in [-(q'+1), -1] lie inside the halo and
// are reduced by the CTA ("virtual" blocks).
struct MedGeom {
  int G;   // lanes per block
  int lgG;
  int B;   // E * G
  int qp;  // q'
  int rp;  // r'
  int V;   // virtual blocks = q' + 1
};

template <typename T>
struct MedLayout {
  static constexpr int E = Chunk<T>::E;
  static constexpr int TILE = NT * E;
  static constexpr int RW = Rowing<T>::RW;
  static constexpr int GHN = NT + kHaloMax / 8 + 8;  // table entries (virtual + real blocks)
  __host__ __device__ static int rows(int64_t w) {
    int r = (int)((TILE + w - 1 + 16 + RW - 1) / RW);  // + margin for shifted 16-B reads
    return (r + kBoxRows - 1) / kBoxRows * kBoxRows;
  }
  __host__ __device__ static size_t stage_bytes(int64_t w) { return (size_t)rows(w) * 128; }
  __host__ __device__ static size_t bytes(int64_t w) {
    return 1024 + 2 * stage_bytes(w) + 4 * sizeof(T) * (size_t)GHN + 64;
  }
};

template <typename T>
__global__ void __launch_bounds__(NT, 2) k1d_medium(Rows p, MedGeom g, const __grid_constant__ CUtensorMap map) {
  using Lay = MedLayout<T>;
  constexpr int E = Lay::E;
  constexpr int TILE = Lay::TILE;
  const int w = (int)p.w;
  const size_t SB = Lay::stage_bytes(w);

  extern __shared__ unsigned char smem_raw[];
  unsigned char *base = reinterpret_cast<unsigned char *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  auto stg = [&](int i) { return base + i * SB; };
  T *GGx = reinterpret_cast<T *>(base + 2 * SB);
  T *GGn = GGx + Lay::GHN;
  T *HHx = GGn + Lay::GHN;
  T *HHn = HHx + Lay::GHN;
  uint64_t *bars = reinterpret_cast<uint64_t *>(HHn + Lay::GHN + 1);
  bars = reinterpret_cast<uint64_t *>((reinterpret_cast<uintptr_t>(bars) + 15) & ~uintptr_t(15));

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int G = g.G, B = g.B;
  const int gl = lane & (G - 1);
  const int grp = tid >> g.lgG;
  const int gbase = lane & ~(G - 1);  // first lane of this lane's group (in the warp)
  // H range inside a far block: block offsets [B - r', B)
  const int hstart = B - g.rp;
  const int h_lane = hstart / E, h_off = hstart - (hstart / E) * E;

  if (tid == 0) {
    prefetch_tmap(&map);
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t grid = gridDim.x;
  if (tid == 0 && (int64_t)blockIdx.x < p.ntiles) {
    int64_t row, u0;
    int tout;
    tile_coords<TILE>(p, blockIdx.x, row, u0, tout);
    stage_tile<T>(p, &map, stg(0), row, u0, tout + w - 1, &bars[0]);
  }

  // group reductions / scans over G lanes
  auto grp_reduce = [&](T &vx, T &vn) {
    for (int d = 1; d < G; d <<= 1) {
      vx = Ord<T>::mx(vx, __shfl_xor_sync(0xffffffffu, vx, d));
      vn = Ord<T>::mn(vn, __shfl_xor_sync(0xffffffffu, vn, d));
    }
  };

  int it = 0;
  for (int64_t t = blockIdx.x; t < p.ntiles; t += grid, ++it) {
    const int st = it & 1;
    const unsigned char *X = stg(st);
    if (tid == 0 && t + grid < p.ntiles) {
      int64_t row, u0;
      int tout;
      tile_coords<TILE>(p, t + grid, row, u0, tout);
      stage_tile<T>(p, &map, stg(st ^ 1), row, u0, tout + w - 1, &bars[st ^ 1]);
    }
    int64_t row, u0;
    int tout;
    tile_coords<TILE>(p, t, row, u0, tout);
    mbar_wait(&bars[st], (it >> 1) & 1);
    if (patch_tail<T>(p, stg(st), row, u0, tout + w - 1, tid)) __syncthreads();

    // ------------------------------------------------- far chunk: prefix
    // ux/un end up as max(P, S) per element: local prefix of the far chunk
    // folded with the local suffix of the near chunk (carries go into cx/cn)
    T ux[E], un[E];
    T cx, cn;
    {
      T y[E];
      lds_swz<T, E>(X, tid * E + w - 1, y);
      ux[0] = un[0] = y[0];
#pragma unroll
      for (int k = 1; k < E; ++k) {
        ux[k] = Ord<T>::mx(ux[k - 1], y[k]);
        un[k] = Ord<T>::mn(un[k - 1], y[k]);
      }
      // H part of this lane: max of y[k] over block offsets >= hstart
      T hx, hn;
      const T bl = __shfl_sync(0xffffffffu, y[E - 1], gbase + G - 1);  // block's last element
      hx = hn = bl;
      if (g.rp > 0) {
        if (gl > h_lane) {
          hx = Ord<T>::mx(hx, ux[E - 1]);
          hn = Ord<T>::mn(hn, un[E - 1]);
        } else if (gl == h_lane) {
          T vx, vn;
          suffix_from<T, E>(y, h_off, vx, vn);
          hx = Ord<T>::mx(hx, vx);
          hn = Ord<T>::mn(hn, vn);
        }
      }
      grp_reduce(hx, hn);
      T ax = ux[E - 1], an = un[E - 1];  // group-inclusive prefix of chunk maxima
      for (int d = 1; d < G; d <<= 1) {
        T vx = shfl_up(ax, d), vn = shfl_up(an, d);
        if (gl >= d) {
          ax = Ord<T>::mx(ax, vx);
          an = Ord<T>::mn(an, vn);
        }
      }
      cx = shfl_up(ax, 1);
      cn = shfl_up(an, 1);
      if (gl == 0) {  // nothing before: an element inside every window
        cx = y[0];
        cn = y[0];
      }
      if (gl == G - 1) {  // publish far block aggregates G_g, H_g
        GGx[grp + g.V] = ax;
        GGn[grp + g.V] = an;
        HHx[grp + g.V] = hx;
        HHn[grp + g.V] = hn;
      }
    }

    // ------------------------------------------------ near chunk: suffix
    {
      T x[E];
      lds_swz_aligned<T, E>(X, tid * E, x);
      T sx = x[E - 1], sn = x[E - 1];
      ux[E - 1] = Ord<T>::mx(ux[E - 1], sx);
      un[E - 1] = Ord<T>::mn(un[E - 1], sn);
#pragma unroll
      for (int k = E - 2; k >= 0; --k) {
        sx = Ord<T>::mx(sx, x[k]);
        sn = Ord<T>::mn(sn, x[k]);
        ux[k] = Ord<T>::mx(ux[k], sx);
        un[k] = Ord<T>::mn(un[k], sn);
      }
      T bx = sx, bn = sn;  // group-inclusive suffix of chunk maxima
      for (int d = 1; d < G; d <<= 1) {
        T dx = shfl_down(bx, d), dn = shfl_down(bn, d);
        if (gl + d < G) {
          bx = Ord<T>::mx(bx, dx);
          bn = Ord<T>::mn(bn, dn);
        }
      }
      T ex = shfl_down(bx, 1), en = shfl_down(bn, 1);
      if (gl == G - 1) {  // nothing after: an element inside every window of the chunk
        ex = x[E - 1];
        en = x[E - 1];
      }
      cx = Ord<T>::mx(cx, ex);
      cn = Ord<T>::mn(cn, en);
    }

    // --------------------------------------- virtual far blocks g' < 0
    {
      const int nv = g.V * G;  // chunks of virtual blocks
      for (int r0 = 0; r0 < nv; r0 += NT) {
        const int vc = r0 + tid;
        if (r0 + (tid & ~31) >= nv) break;  // whole warp idle (warp-uniform)
        const int vcc = vc < nv ? vc : nv - 1;
        const int gv = vcc >> g.lgG;      // 0 .. V-1  <->  g' = gv - V
        const int pos = (gv - g.V) * B + w - 1 + gl * E;
        T y[E];
        lds_swz<T, E>(X, pos, y);
        T ax = y[0], an = y[0];
#pragma unroll
        for (int k = 1; k < E; ++k) {
          ax = Ord<T>::mx(ax, y[k]);
          an = Ord<T>::mn(an, y[k]);
        }
        T hx, hn;
        const T bl = __shfl_sync(0xffffffffu, y[E - 1], gbase + G - 1);
        hx = hn = bl;
        if (g.rp > 0) {
          if (gl > h_lane) {
            hx = Ord<T>::mx(hx, ax);
            hn = Ord<T>::mn(hn, an);
          } else if (gl == h_lane) {
            T ux, un;
            suffix_from<T, E>(y, h_off, ux, un);
            hx = Ord<T>::mx(hx, ux);
            hn = Ord<T>::mn(hn, un);
          }
        }
        grp_reduce(ax, an);
        grp_reduce(hx, hn);
        if (vc < nv && gl == 0) {
          GGx[gv] = ax;
          GGn[gv] = an;
          HHx[gv] = hx;
          HHn[gv] = hn;
        }
      }
    }
    __syncthreads();

    // ---------------------------------------------------------- gap + out
    if (g.qp > 0 || g.rp > 0) {
      const int b0 = grp - g.qp - 1 + g.V;  // table index of F_{g-q'-1}
      T mx, mn;
      if (g.rp > 0) {
        mx = HHx[b0];
        mn = HHn[b0];
      } else {
        mx = GGx[b0 + 1];
        mn = GGn[b0 + 1];
      }
      for (int s = 1; s <= g.qp; ++s) {
        mx = Ord<T>::mx(mx, GGx[b0 + s]);
        mn = Ord<T>::mn(mn, GGn[b0 + s]);
      }
      cx = Ord<T>::mx(cx, mx);
      cn = Ord<T>::mn(cn, mn);
    }
    const int c0 = tid * E;
    if (c0 < tout) {
      T ox[E], on[E];
#pragma unroll
      for (int k = 0; k < E; ++k) {
        ox[k] = Ord<T>::mx(ux[k], cx);
        on[k] = Ord<T>::mn(un[k], cn);
      }
      store_out<T, E>(p, row, u0 + c0, tout - c0, ox, on);
    }
    __syncthreads();  // stage st and the tables are free for the next iteration
  }
}

// ===================================================================== large
// w-1 > kHaloMax.  CTA tile x owns outputs [u0, u0+T), u0 = xT, and stages
//   near N_x = [u0, u0+T)            -> S(i) = max a[u0+i .. u0+T)   (CTA suffix scan)
//   far  F_x = [u0+w-1, u0+w-1+T)    -> P(i) = max a[u0+w-1 .. u0+w-1+i] (CTA prefix scan)
// so that out[u0+i] = max(S(i), M_x, P(i)) with the fixed gap
//   M_x = max a[u0+T .. u0+w-1).
// With w-1 = qT + r the gap is the last r elements of F_{x-q} followed by the
// whole F_{x-q+1} .. F_{x-1}.  Every tile publishes G_x = max F_x and H_x = max
// of the last r elements of F_x; tile x consumes H_{x-q}, G_{x-q+1..x-1}.
// Tiles x in [-q, -1] exist only to publish (their F lies inside the array).
// Tickets (atomic counter) order the tiles: ticket = (row, x+q) row-major.  A
// CTA publishes before it waits, and waits only on lower tickets; a CTA that
// holds a prefetched next ticket finishes its current one (which only waits on
// lower tickets) first -- deadlock-free for any number of resident CTAs.
struct LargeGeom {
  int q, r;
  int64_t tickets_per_row;  // q + tiles_per_row
  int64_t total;            // batch * tickets_per_row
};

template <typename T>
struct LargeWs {  // workspace carve-up
  __host__ __device__ static size_t bytes(int64_t tickets) {
    return 256 + (size_t)tickets * (4 + 4 * sizeof(T)) + 64;
  }
};

template <typename T>
struct LargeLayout {
  static constexpr int E = Chunk<T>::E;
  static constexpr int TILE = NT * E;
  static constexpr int RW = Rowing<T>::RW;
  static constexpr int NROWS = (TILE / RW + kBoxRows - 1) / kBoxRows * kBoxRows;
  static constexpr int FROWS = ((TILE + RW) / RW + kBoxRows - 1) / kBoxRows * kBoxRows;
  static constexpr size_t NB = (size_t)NROWS * 128, FB = (size_t)FROWS * 128;
  static constexpr size_t STAGE = NB + FB;
  static constexpr size_t BYTES = 1024 + 2 * STAGE + 256;
};

template <typename T>
__global__ void __launch_bounds__(NT, 2) k1d_large(Rows p, LargeGeom g, void *ws,
                                                  const __grid_constant__ CUtensorMap map) {
  using Lay = LargeLayout<T>;
  constexpr int E = Lay::E;
  constexpr int TILE = Lay::TILE;
  constexpr int RW = Lay::RW;

  extern __shared__ unsigned char smem_raw[];
  unsigned char *base = reinterpret_cast<unsigned char *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  auto nearb = [&](int i) { return base + i * Lay::STAGE; };
  auto farb = [&](int i) { return base + i * Lay::STAGE + Lay::NB; };
  __shared__ T wagg[4][NWARP];
  __shared__ T gap[2];
  __shared__ int64_t s_ticket[2];
  __shared__ int s_fshift[2];
  __shared__ __align__(8) uint64_t bars[2];

  uint32_t *counter = reinterpret_cast<uint32_t *>(ws);
  uint32_t *flags = reinterpret_cast<uint32_t *>(static_cast<char *>(ws) + 256);
  T *Gx = reinterpret_cast<T *>((reinterpret_cast<uintptr_t>(flags + g.total) + 15) & ~uintptr_t(15));
  T *Gn = Gx + g.total;
  T *Hx = Gn + g.total;
  T *Hn = Hx + g.total;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t w = p.w;

  // stage ticket tk into stage st (thread 0 only)
  auto stage_ticket = [&](int64_t tk, int st) {
    s_ticket[st] = tk;
    if (tk >= g.total) {
      mbar_arrive_expect_tx(&bars[st], 0);
      return;
    }
    const int64_t row = tk / g.tickets_per_row;
    const int64_t x = tk - row * g.tickets_per_row - g.q;
    const int64_t u0 = x * TILE;
    const int64_t f0 = u0 + w - 1;
    int64_t flen = p.n - f0 < TILE ? p.n - f0 : TILE;
    if (p.has_map) {
      uint32_t bytes = 0;
      const int64_t fr0 = f0 / RW, fr1 = (f0 + flen + RW - 1) / RW;
      const int nfb = (int)((fr1 - fr0 + kBoxRows - 1) / kBoxRows);
      int nnb = 0;
      if (x >= 0) nnb = (TILE / RW + kBoxRows - 1) / kBoxRows;
      bytes = (uint32_t)(nfb + nnb) * kBoxBytes;
      mbar_arrive_expect_tx(&bars[st], bytes);
      for (int k = 0; k < nfb; ++k) tma_box(&map, farb(st) + k * kBoxBytes, (int)(fr0 + k * kBoxRows), (int)row, &bars[st]);
      for (int k = 0; k < nnb; ++k)
        tma_box(&map, nearb(st) + k * kBoxBytes, (int)(u0 / RW + k * kBoxRows), (int)row, &bars[st]);
    } else {
      mbar_arrive_expect_tx(&bars[st], 0);
    }
    s_fshift[st] = (int)(f0 - (f0 / RW) * RW);
  };

  if (tid == 0) {
    prefetch_tmap(&map);
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    stage_ticket((int64_t)atomicAdd(reinterpret_cast<unsigned long long *>(counter), 1ull), 0);
  }
  __syncthreads();

  for (int it = 0;; ++it) {
    const int st = it & 1;
    const int64_t ticket = s_ticket[st];
    if (ticket >= g.total) break;
    if (tid == 0)  // prefetch the next ticket into the other stage
      stage_ticket((int64_t)atomicAdd(reinterpret_cast<unsigned long long *>(counter), 1ull), st ^ 1);
    const int64_t row = ticket / g.tickets_per_row;
    const int64_t x = ticket - row * g.tickets_per_row - g.q;  // may be negative
    const int64_t u0 = x * TILE;
    const int64_t f0 = u0 + w - 1;
    int tout = 0;
    if (x >= 0) {
      int64_t left = p.m - u0;
      tout = left < TILE ? (int)left : TILE;
    }
    const int fshift = s_fshift[st];
    mbar_wait(&bars[st], (it >> 1) & 1);
    {  // partial last 128-B row of the series, if staged
      bool fixed = false;
      const T *srs = series_ptr<T>(p, row);
      const int64_t full = p.has_map ? (p.n / RW) * RW : 0;
      if (full < p.n) {
        const int64_t fa = f0 - fshift;  // absolute start of the far stage
        const int64_t fe = f0 + TILE;
        if (full < fe && p.n > fa) {
          const int64_t lo = full > fa ? full : fa, hi = p.n < fe ? p.n : fe;
          for (int64_t i = lo + tid; i < hi; i += NT) sts_swz<T>(farb(st), (int)(i - fa), srs[i]);
          fixed = true;
        }
        if (x >= 0 && full < u0 + TILE && p.n > u0) {
          const int64_t lo = full > u0 ? full : u0, hi = p.n < u0 + TILE ? p.n : u0 + TILE;
          for (int64_t i = lo + tid; i < hi; i += NT) sts_swz<T>(nearb(st), (int)(i - u0), srs[i]);
          fixed = true;
        }
      }
      if (fixed) __syncthreads();
    }

    // ------------------------------------------- far: CTA prefix scan of F_x
    T px[E], pn[E];
    T hx, hn;
    {
      T v[E];
      lds_swz<T, E>(farb(st), fshift + tid * E, v);
      px[0] = pn[0] = v[0];
#pragma unroll
      for (int k = 1; k < E; ++k) {
        px[k] = Ord<T>::mx(px[k - 1], v[k]);
        pn[k] = Ord<T>::mn(pn[k - 1], v[k]);
      }
      // last r positions of F_x: [TILE - r, TILE); an empty part borrows the
      // element at TILE-1, which belongs to every non-empty H range
      const int hstart = TILE - g.r;
      const T last = lds_one_swz<T>(farb(st), fshift + TILE - 1);  // broadcast read
      hx = hn = last;
      if (tid * E >= hstart) {
        hx = Ord<T>::mx(hx, px[E - 1]);
        hn = Ord<T>::mn(hn, pn[E - 1]);
      } else if (tid * E + E > hstart) {
        T ux, un;
        suffix_from<T, E>(v, hstart - tid * E, ux, un);
        hx = Ord<T>::mx(hx, ux);
        hn = Ord<T>::mn(hn, un);
      }
    }
    T ax = px[E - 1], an = pn[E - 1];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      T ux = shfl_up(ax, d), un = shfl_up(an, d);
      if (lane >= d) {
        ax = Ord<T>::mx(ax, ux);
        an = Ord<T>::mn(an, un);
      }
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {  // warp reduce of the H part
      hx = Ord<T>::mx(hx, __shfl_xor_sync(0xffffffffu, hx, d));
      hn = Ord<T>::mn(hn, __shfl_xor_sync(0xffffffffu, hn, d));
    }
    T cpx = shfl_up(ax, 1), cpn = shfl_up(an, 1);
    if (lane == 0) {
      cpx = px[0];
      cpn = pn[0];
    }
    if (lane == 31) {
      wagg[0][warp] = ax;
      wagg[1][warp] = an;
    }
    if (lane == 0) {
      wagg[2][warp] = hx;
      wagg[3][warp] = hn;
    }
    __syncthreads();
    for (int v = 0; v < warp; ++v) {  // cross-warp carry of the prefix
      cpx = Ord<T>::mx(cpx, wagg[0][v]);
      cpn = Ord<T>::mn(cpn, wagg[1][v]);
    }
    // -------------------------------------------------------------- publish
    if (tid == 0) {
      T gx = wagg[0][0], gn = wagg[1][0], hhx = wagg[2][0], hhn = wagg[3][0];
      for (int v = 1; v < NWARP; ++v) {
        gx = Ord<T>::mx(gx, wagg[0][v]);
        gn = Ord<T>::mn(gn, wagg[1][v]);
        hhx = Ord<T>::mx(hhx, wagg[2][v]);
        hhn = Ord<T>::mn(hhn, wagg[3][v]);
      }
      Gx[ticket] = gx;
      Gn[ticket] = gn;
      Hx[ticket] = hhx;
      Hn[ticket] = hhn;
      __threadfence();
      st_release_u32(flags + ticket, 1u);
    }
    if (x >= 0) {
      // ------------------------------------------ near: CTA suffix scan of N_x
      T sx[E], sn[E];
      {
        T v[E];
        lds_swz_aligned<T, E>(nearb(st), tid * E, v);
        sx[E - 1] = sn[E - 1] = v[E - 1];
#pragma unroll
        for (int k = E - 2; k >= 0; --k) {
          sx[k] = Ord<T>::mx(sx[k + 1], v[k]);
          sn[k] = Ord<T>::mn(sn[k + 1], v[k]);
        }
      }
      T bx = sx[0], bn = sn[0];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        T dx = shfl_down(bx, d), dn = shfl_down(bn, d);
        if (lane + d < 32) {
          bx = Ord<T>::mx(bx, dx);
          bn = Ord<T>::mn(bn, dn);
        }
      }
      __syncthreads();  // wagg reuse
      if (lane == 0) {
        wagg[0][warp] = bx;
        wagg[1][warp] = bn;
      }
      T csx = shfl_down(bx, 1), csn = shfl_down(bn, 1);
      if (lane == 31) {
        csx = sx[E - 1];
        csn = sn[E - 1];
      }
      // --------------------------------------------- gap M_x from the look-back
      for (int s = tid; s < g.q; s += NT) {
        const int64_t src = ticket - g.q + s;  // x' = x - q + s
        uint32_t spins = 0;
        while (ld_acquire_u32(flags + src) == 0u) {
          __nanosleep(64);
          if (++spins > (1u << 26)) __trap();  // a lost publish must fail, never hang
        }
      }
      __syncthreads();
      if (tid == 0) {
        T gxv, gnv;
        const int64_t src0 = ticket - g.q;
        if (g.r > 0) {
          gxv = __ldcg(Hx + src0);
          gnv = __ldcg(Hn + src0);
        } else {  // r == 0: the gap is F_{x-q+1..x-1} only (q >= 2 since w-1 > T)
          gxv = __ldcg(Gx + src0 + 1);
          gnv = __ldcg(Gn + src0 + 1);
        }
        for (int s = 1; s < g.q; ++s) {
          gxv = Ord<T>::mx(gxv, __ldcg(Gx + src0 + s));
          gnv = Ord<T>::mn(gnv, __ldcg(Gn + src0 + s));
        }
        gap[0] = gxv;
        gap[1] = gnv;
      }
      __syncthreads();
      for (int v = warp + 1; v < NWARP; ++v) {
        csx = Ord<T>::mx(csx, wagg[0][v]);
        csn = Ord<T>::mn(csn, wagg[1][v]);
      }
      const T cx = Ord<T>::mx(Ord<T>::mx(csx, cpx), gap[0]);
      const T cn = Ord<T>::mn(Ord<T>::mn(csn, cpn), gap[1]);
      const int c0 = tid * E;
      if (c0 < tout) {
        T ox[E], on[E];
#pragma unroll
        for (int k = 0; k < E; ++k) {
          ox[k] = Ord<T>::mx(Ord<T>::mx(sx[k], px[k]), cx);
          on[k] = Ord<T>::mn(Ord<T>::mn(sn[k], pn[k]), cn);
        }
        store_out<T, E>(p, row, u0 + c0, tout - c0, ox, on);
      }
    }
    __syncthreads();  // stage st, wagg and gap are free for the next iteration
  }
}

}  // namespace mm

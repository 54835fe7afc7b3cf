// k1d.cuh -- 1-D (and batched) running max-min filter kernels for sm_100a.
//
// The operation is PAPER.md:39-42: out_max[j] = max a[j..j+w), out_min[j] =
// min a[j..j+w), j in [0, n-w].  The paper's own algorithm (the monotonic
// wedge, Algorithm 1) is inherently sequential; on the GPU
// the same result is reached by block decompositions of the window, in the
// family of van Herk / Gil-Werman: with blocks of length B
// (a power of two with B <= w-1 < 2B, or B = 32 chunks when w-1 >= 2B),
//
//   out[j] = max( S(j),  A[x+1 .. y-1],  P(j+w-1) )       x = j/B, y = (j+w-1)/B
//
// where S is the suffix max inside j's block, P the prefix max inside the
// block of j+w-1 and A[] the maxima of the whole blocks in between (likewise
// for min).  Three kernels cover every w:
//
//   k1d_small<T,W>   2 <= w <= E: compile-time w ("compiling w in the code",
//                    PAPER.md:528-531), log-step doubling in registers.
//   k1d_medium<T>    E < w <= kHaloMax+1: tile + (w-1) halo staged by TMA in
//                    shared memory; chunk-local scans, warp-shuffle group
//                    scans, block aggregates; 2-stage TMA pipeline, persistent.
//   k1d_large<T>     w-1 > kHaloMax: near tile + far tile per CTA, cross-CTA
//                    look-back on far-tile aggregates published through a
//                    workspace (ticketed, deadlock-free).
//
// Every kernel handles a batch of rows (row b at in + b*in_ld); 1-D is batch 1.
#pragma once

#include "common.cuh"

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
};

// Position of tile `t` of TILE outputs: row, first output u0, output count.
template <int TILE>
__device__ __forceinline__ void tile_coords(const Rows &p, int64_t t, int64_t &row, int64_t &u0,
                                            int &tout) {
  row = t / p.tiles_per_row;
  u0 = (t - row * p.tiles_per_row) * (int64_t)TILE;
  int64_t left = p.m - u0;
  tout = left < TILE ? (int)left : TILE;
}

// Issue the TMA copy of input elements [u0, u0+L) of `row` into `dst`
// (rounded out to the enclosing 16-B granules; the row base is 16-B aligned).
template <typename T>
__device__ __forceinline__ void issue_tile_load(const Rows &p, int64_t row, int64_t u0, int64_t L,
                                                T *dst, uint64_t *bar) {
  const T *base = static_cast<const T *>(p.in) + row * p.in_ld;
  const char *g0 = reinterpret_cast<const char *>(base + u0);
  const char *g1 = reinterpret_cast<const char *>(base + u0 + L);
  g1 = reinterpret_cast<const char *>((reinterpret_cast<uintptr_t>(g1) + 15) & ~uintptr_t(15));
  uint32_t bytes = (uint32_t)(g1 - g0);
  mbar_arrive_expect_tx(bar, bytes);
  bulk_g2s_range(dst, g0, g1, bar);
}

// ===================================================================== small
// 2 <= W <= E.  Thread c owns outputs [cE, cE+E) of the tile and needs inputs
// [cE, cE+E+W-1): its own chunk plus the first W-1 elements of the next one.
// Log-step doubling: after the step of span s, m[p] = max a[p .. p+2s); the
// output is max(m_{2^K}[j], m_{2^K}[j+W-2^K]) (overlap is harmless: max is
// idempotent).  K = floor(log2 W) steps + 1 combine per filter.
template <typename T, int W>
__global__ void __launch_bounds__(NT) k1d_small(Rows p) {
  using C = Chunk<T>;
  constexpr int E = C::E;
  constexpr int VEC = C::VEC;
  constexpr int TILE = NT * E;
  constexpr int XCAP = TILE + E + VEC;  // tile + next-chunk read + 16-B rounding
  constexpr int NXT = (W - 1 + VEC - 1) / VEC;  // 16-B vectors of the next chunk
  constexpr int K = W >= 16 ? 4 : W >= 8 ? 3 : W >= 4 ? 2 : 1;
  constexpr int SPAN = 1 << K;
  static_assert(W >= 2 && W <= E, "small path: 2 <= W <= E");

  extern __shared__ __align__(128) unsigned char smem_raw[];
  T *X0 = reinterpret_cast<T *>(smem_raw);
  T *X1 = X0 + XCAP;
  uint64_t *bars = reinterpret_cast<uint64_t *>(X1 + XCAP);
  const int tid = threadIdx.x;

  if (tid == 0) {
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
    issue_tile_load<T>(p, row, u0, tout + W - 1, X0, &bars[0]);
  }
  int it = 0;
  for (int64_t t = blockIdx.x; t < p.ntiles; t += grid, ++it) {
    const int st = it & 1;
    T *X = st ? X1 : X0;
    if (tid == 0 && t + grid < p.ntiles) {  // prefetch the next tile into the other stage
      int64_t row, u0;
      int tout;
      tile_coords<TILE>(p, t + grid, row, u0, tout);
      issue_tile_load<T>(p, row, u0, tout + W - 1, st ? X0 : X1, &bars[st ^ 1]);
    }
    int64_t row, u0;
    int tout;
    tile_coords<TILE>(p, t, row, u0, tout);
    mbar_wait(&bars[st], (it >> 1) & 1);

    const int c0 = tid * E;
    if (c0 < tout) {
      T v[E + VEC * NXT];
      lds_chunk<T, E>(X + c0, *reinterpret_cast<T(*)[E]>(v));
#pragma unroll
      for (int k = 0; k < NXT; ++k) {
        union {
          uint4 q;
          T t[VEC];
        } u;
        u.q = reinterpret_cast<const uint4 *>(X + c0 + E)[k];
#pragma unroll
        for (int e = 0; e < VEC; ++e) v[E + k * VEC + e] = u.t[e];
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
      T *omx = p.out_max ? static_cast<T *>(p.out_max) + row * p.out_ld + u0 + c0 : nullptr;
      T *omn = p.out_min ? static_cast<T *>(p.out_min) + row * p.out_ld + u0 + c0 : nullptr;
      if (c0 + E <= tout) {
        if (omx) store_chunk<T, E>(omx, ox);
        if (omn) store_chunk<T, E>(omn, on);
      } else {
#pragma unroll
        for (int j = 0; j < E; ++j)
          if (c0 + j < tout) {
            if (omx) omx[j] = ox[j];
            if (omn) omn[j] = on[j];
          }
      }
    }
    __syncthreads();  // stage st is free for the prefetch of iteration it+1
  }
}

// ==================================================================== medium
// Runtime w with E+1 <= w <= kHaloMax+1.  Blocks of B = 2^b elements (b >= log2 E,
// B <= 32E) aligned to the tile start; w-1 = qB + r, q >= 1.  For j = xB + i:
//   i + r <  B :  out[j] = max(S(j), A[x+1..x+q-1], P(j+w-1))
//   i + r >= B :  out[j] = max(S(j), A[x+1..x+q],   P(j+w-1))
// (the A range is empty when q = 1 and i + r < B).  Scan pass: every chunk c of
// the tile + halo computes its chunk-local prefix/suffix, the group of G = B/E
// lanes completes them by shuffle scans, the last lane of a group publishes the
// block aggregate A, and P at positions >= w-1 is parked in shared memory (PP,
// padded layout).  Output pass: thread c combines S (registers), A and P.
struct MedGeom {
  int b;  // log2 B
  int q;  // (w-1) >> b
  int r;  // (w-1) & (B-1)
};

template <typename T>
struct MedLayout {  // shared-memory carve-up, identical on host and device
  static constexpr int E = Chunk<T>::E;
  static constexpr int TILE = NT * E;
  static constexpr int PPN = pad_size<T>(TILE);
  static constexpr int AAN = (TILE + kHaloMax) / E + 16;  // blocks (B >= E)
  __host__ __device__ static int xcap(int64_t w) {  // elements, multiple of E
    int64_t L = TILE + w - 1 + 16;
    return (int)((L + E - 1) / E * E);
  }
  __host__ __device__ static size_t bytes(int64_t w) {
    return sizeof(T) * (2 * (size_t)xcap(w) + 2 * (size_t)PPN + 2 * (size_t)AAN) + 64;
  }
};

template <typename T>
__global__ void __launch_bounds__(NT, 2) k1d_medium(Rows p, MedGeom g) {
  using C = Chunk<T>;
  using Lay = MedLayout<T>;
  constexpr int E = C::E;
  constexpr int TILE = Lay::TILE;
  const int w = (int)p.w;
  const int xcap = Lay::xcap(w);

  extern __shared__ __align__(128) unsigned char smem_raw[];
  T *X0 = reinterpret_cast<T *>(smem_raw);
  T *X1 = X0 + xcap;
  T *PPx = X1 + xcap;
  T *PPn = PPx + Lay::PPN;
  T *AAx = PPn + Lay::PPN;
  T *AAn = AAx + Lay::AAN;
  uint64_t *bars = reinterpret_cast<uint64_t *>(
      (reinterpret_cast<uintptr_t>(AAn + Lay::AAN) + 15) & ~uintptr_t(15));

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int B = 1 << g.b;
  const int G = B / E;  // lanes per block (1..32)
  const int gl = lane & (G - 1);

  if (tid == 0) {
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
    issue_tile_load<T>(p, row, u0, tout + w - 1, X0, &bars[0]);
  }
  int it = 0;
  for (int64_t t = blockIdx.x; t < p.ntiles; t += grid, ++it) {
    const int st = it & 1;
    const T *X = st ? X1 : X0;
    if (tid == 0 && t + grid < p.ntiles) {
      int64_t row, u0;
      int tout;
      tile_coords<TILE>(p, t + grid, row, u0, tout);
      issue_tile_load<T>(p, row, u0, tout + w - 1, st ? X0 : X1, &bars[st ^ 1]);
    }
    int64_t row, u0;
    int tout;
    tile_coords<TILE>(p, t, row, u0, tout);
    const int L = tout + w - 1;          // valid input elements of this tile
    const int nchunk = (L + E - 1) / E;  // scan chunks
    const int npass = (nchunk + NT - 1) / NT;
    mbar_wait(&bars[st], (it >> 1) & 1);

    // ---------------------------------------------------------- scan pass
    T Sx[E], Sn[E];  // suffix (with group carry) of this thread's output chunk
    for (int pass = 0; pass < npass; ++pass) {
      const int c = pass * NT + tid;
      const int cc = c < nchunk ? c : nchunk - 1;  // idle lanes redo the last chunk
      T x[E];
      lds_chunk<T, E>(X + cc * E, x);
      T px[E], pn[E], sx[E], sn[E];
      px[0] = pn[0] = x[0];
#pragma unroll
      for (int k = 1; k < E; ++k) {
        px[k] = Ord<T>::mx(px[k - 1], x[k]);
        pn[k] = Ord<T>::mn(pn[k - 1], x[k]);
      }
      sx[E - 1] = sn[E - 1] = x[E - 1];
#pragma unroll
      for (int k = E - 2; k >= 0; --k) {
        sx[k] = Ord<T>::mx(sx[k + 1], x[k]);
        sn[k] = Ord<T>::mn(sn[k + 1], x[k]);
      }
      // group-inclusive prefix (over lanes gl' <= gl) and suffix (gl' >= gl)
      T ax = px[E - 1], an = pn[E - 1], bx = sx[0], bn = sn[0];
      for (int d = 1; d < G; d <<= 1) {
        T ux = shfl_up(ax, d), un = shfl_up(an, d);
        T dx = shfl_down(bx, d), dn = shfl_down(bn, d);
        if (gl >= d) {
          ax = Ord<T>::mx(ax, ux);
          an = Ord<T>::mn(an, un);
        }
        if (gl + d < G) {
          bx = Ord<T>::mx(bx, dx);
          bn = Ord<T>::mn(bn, dn);
        }
      }
      // exclusive carries; a lane at the block edge substitutes an element
      // that lies inside every window concerned (max/min are idempotent)
      T cpx = shfl_up(ax, 1), cpn = shfl_up(an, 1);
      T csx = shfl_down(bx, 1), csn = shfl_down(bn, 1);
      if (gl == 0) {
        cpx = x[0];
        cpn = x[0];
      }
      if (gl == G - 1) {
        csx = x[E - 1];
        csn = x[E - 1];
      }
      if (c < nchunk) {
        if (gl == G - 1) {  // block aggregate
          AAx[c / G] = ax;
          AAn[c / G] = an;
        }
        // P at positions pos >= w-1 is needed by output j = pos-(w-1)
        const int j0 = c * E - (w - 1);
#pragma unroll
        for (int k = 0; k < E; ++k) {
          const int j = j0 + k;
          if (j >= 0 && j < tout) {
            PPx[pad_idx<T>(j)] = Ord<T>::mx(px[k], cpx);
            PPn[pad_idx<T>(j)] = Ord<T>::mn(pn[k], cpn);
          }
        }
      }
      if (pass == 0) {
#pragma unroll
        for (int k = 0; k < E; ++k) {
          Sx[k] = Ord<T>::mx(sx[k], csx);
          Sn[k] = Ord<T>::mn(sn[k], csn);
        }
      }
    }
    __syncthreads();

    // -------------------------------------------------------- output pass
    const int c0 = tid * E;
    if (c0 < tout) {
      const int xb = c0 >> g.b;
      // K1: middle blocks x+1..x+q-1 (or an in-window element when q == 1)
      T k1x = Sx[E - 1], k1n = Sn[E - 1];
      for (int s = 1; s < g.q; ++s) {
        k1x = Ord<T>::mx(k1x, AAx[xb + s]);
        k1n = Ord<T>::mn(k1n, AAn[xb + s]);
      }
      const T k2x = Ord<T>::mx(k1x, AAx[xb + g.q]);
      const T k2n = Ord<T>::mn(k1n, AAn[xb + g.q]);
      T ox[E], on[E];
#pragma unroll
      for (int k = 0; k < E; ++k) {
        const int i = (c0 + k) & (B - 1);
        const bool far = i + g.r >= B;
        const T mx = Ord<T>::mx(Sx[k], far ? k2x : k1x);
        const T mn = Ord<T>::mn(Sn[k], far ? k2n : k1n);
        ox[k] = Ord<T>::mx(mx, PPx[pad_idx<T>(c0 + k)]);
        on[k] = Ord<T>::mn(mn, PPn[pad_idx<T>(c0 + k)]);
      }
      T *omx = p.out_max ? static_cast<T *>(p.out_max) + row * p.out_ld + u0 + c0 : nullptr;
      T *omn = p.out_min ? static_cast<T *>(p.out_min) + row * p.out_ld + u0 + c0 : nullptr;
      if (c0 + E <= tout) {
        if (omx) store_chunk<T, E>(omx, ox);
        if (omn) store_chunk<T, E>(omn, on);
      } else {
#pragma unroll
        for (int k = 0; k < E; ++k)
          if (c0 + k < tout) {
            if (omx) omx[k] = ox[k];
            if (omn) omn[k] = on[k];
          }
      }
    }
    __syncthreads();  // PP/AA and stage st are free for the next iteration
  }
}

// ===================================================================== large
// w-1 > kHaloMax.  CTA x owns outputs [u0, u0+T), u0 = xT, and loads
//   near N_x = [u0, u0+T)            -> S(i) = max a[u0+i .. u0+T)   (CTA suffix scan)
//   far  F_x = [u0+w-1, u0+w-1+T)    -> P(i) = max a[u0+w-1 .. u0+w-1+i] (CTA prefix scan)
// so that out[u0+i] = max(S(i), M_x, P(i)) with the fixed gap
//   M_x = max a[u0+T .. u0+w-1).
// With w-1 = qT + r the gap is the last r elements of F_{x-q} followed by the
// whole F_{x-q+1} .. F_{x-1}.  Every CTA publishes G_x = max F_x and H_x = max
// of the last r elements of F_x; CTA x consumes H_{x-q}, G_{x-q+1..x-1}.
// Tiles x in [-q, -1] exist only to publish (their F lies inside the array).
// Tickets (atomic counter) order the CTAs: ticket = (row, x+q) row-major, and a
// CTA publishes before it waits, waiting only on lower tickets -- deadlock-free.
struct LargeGeom {
  int q, r;
  int64_t tickets_per_row;  // q + tiles_per_row
};

template <typename T>
struct LargeWs {  // workspace carve-up
  __host__ __device__ static size_t bytes(int64_t tickets) {
    return 256 + (size_t)tickets * (4 + 4 * sizeof(T)) + 64;
  }
};

template <typename T>
__global__ void __launch_bounds__(NT, 2) k1d_large(Rows p, LargeGeom g, void *ws) {
  using C = Chunk<T>;
  constexpr int E = C::E;
  constexpr int VEC = C::VEC;
  constexpr int TILE = NT * E;
  constexpr int FCAP = TILE + 2 * VEC;

  __shared__ __align__(128) T Nb[TILE];
  __shared__ __align__(128) T Fb[FCAP];
  __shared__ T wagg[4][NWARP];
  __shared__ T gap[2];
  __shared__ int64_t s_ticket;
  __shared__ __align__(8) uint64_t bar;

  const int64_t total = p.batch * g.tickets_per_row;
  uint32_t *counter = reinterpret_cast<uint32_t *>(ws);
  uint32_t *flags = reinterpret_cast<uint32_t *>(static_cast<char *>(ws) + 256);
  T *Gx = reinterpret_cast<T *>(
      (reinterpret_cast<uintptr_t>(flags + total) + 15) & ~uintptr_t(15));
  T *Gn = Gx + total;
  T *Hx = Gn + total;
  T *Hn = Hx + total;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    s_ticket = (int64_t)atomicAdd(reinterpret_cast<unsigned long long *>(counter), 1ull);
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t ticket = s_ticket;
  if (ticket >= total) return;
  const int64_t row = ticket / g.tickets_per_row;
  const int64_t x = ticket - row * g.tickets_per_row - g.q;  // may be negative
  const int64_t u0 = x * TILE;
  const T *in = static_cast<const T *>(p.in) + row * p.in_ld;
  const int64_t w = p.w;

  // ---------------------------------------------------------------- loads
  const int64_t f0 = u0 + w - 1;  // >= 0 for x >= -q
  const int64_t f1 = f0 + TILE < p.n ? f0 + TILE : p.n;
  const int64_t f0a = f0 & ~(int64_t)(VEC - 1);  // 16-B aligned start
  const int fshift = (int)(f0 - f0a);
  int tout = 0;
  if (x >= 0) {
    int64_t left = p.m - u0;
    tout = left < TILE ? (int)left : TILE;
  }
  if (tid == 0) {
    const char *g0 = reinterpret_cast<const char *>(in + f0a);
    const char *g1 = reinterpret_cast<const char *>(
        (reinterpret_cast<uintptr_t>(in + f1) + 15) & ~uintptr_t(15));
    uint32_t bytes = (uint32_t)(g1 - g0);
    const char *n0 = nullptr, *n1 = nullptr;
    if (x >= 0) {  // near tile [u0, u0+TILE) lies inside the array (T < w-1)
      n0 = reinterpret_cast<const char *>(in + u0);
      n1 = reinterpret_cast<const char *>(in + u0 + TILE);
      bytes += (uint32_t)(n1 - n0);
    }
    mbar_arrive_expect_tx(&bar, bytes);
    bulk_g2s_range(Fb, g0, g1, &bar);
    if (x >= 0) bulk_g2s_range(Nb, n0, n1, &bar);
  }
  mbar_wait(&bar, 0);

  // ------------------------------------------- far: CTA prefix scan of F_x
  T px[E], pn[E];
  T hx, hn;  // max/min of this chunk's part of the last r elements of F_x
  {
    T v[E];
    lds_chunk_shifted<T, E>(Fb + tid * E, fshift, v);
    px[0] = pn[0] = v[0];
#pragma unroll
    for (int k = 1; k < E; ++k) {
      px[k] = Ord<T>::mx(px[k - 1], v[k]);
      pn[k] = Ord<T>::mn(pn[k - 1], v[k]);
    }
    // last r positions of F_x: [TILE - r, TILE); an empty part borrows the
    // element at TILE-1, which belongs to every non-empty H range
    const int hstart = TILE - g.r;
    T last = Fb[fshift + TILE - 1];
    hx = hn = last;
#pragma unroll
    for (int k = 0; k < E; ++k)
      if (tid * E + k >= hstart) {
        hx = Ord<T>::mx(hx, v[k]);
        hn = Ord<T>::mn(hn, v[k]);
      }
  }
  // warp-inclusive prefix of chunk aggregates
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
  if (lane == 31) {
    wagg[0][warp] = ax;
    wagg[1][warp] = an;
  }
  if (lane == 0) {
    wagg[2][warp] = hx;
    wagg[3][warp] = hn;
  }
  T cpx = shfl_up(ax, 1), cpn = shfl_up(an, 1);
  if (lane == 0) {
    cpx = px[0];
    cpn = pn[0];
  }
  __syncthreads();
  // cross-warp carry for the prefix
  for (int v = 0; v < warp; ++v) {
    cpx = Ord<T>::mx(cpx, wagg[0][v]);
    cpn = Ord<T>::mn(cpn, wagg[1][v]);
  }
#pragma unroll
  for (int k = 0; k < E; ++k) {
    px[k] = Ord<T>::mx(px[k], cpx);
    pn[k] = Ord<T>::mn(pn[k], cpn);
  }
  // ----------------------------------------------------------- publish
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
  if (x < 0) return;  // publishing-only ticket

  // ------------------------------------------ near: CTA suffix scan of N_x
  T sx[E], sn[E];
  {
    T v[E];
    lds_chunk<T, E>(Nb + tid * E, v);
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
  // ----------------------------------------------- gap M_x from the look-back
  // ticket of F_{x'} is ticket - (x - x'); needs x' = x-q (H) and x-q+1..x-1 (G)
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
  const T gx = gap[0], gn = gap[1];
  const int c0 = tid * E;
  if (c0 < tout) {
    T ox[E], on[E];
#pragma unroll
    for (int k = 0; k < E; ++k) {
      ox[k] = Ord<T>::mx(Ord<T>::mx(Ord<T>::mx(sx[k], csx), gx), px[k]);
      on[k] = Ord<T>::mn(Ord<T>::mn(Ord<T>::mn(sn[k], csn), gn), pn[k]);
    }
    T *omx = p.out_max ? static_cast<T *>(p.out_max) + row * p.out_ld + u0 + c0 : nullptr;
    T *omn = p.out_min ? static_cast<T *>(p.out_min) + row * p.out_ld + u0 + c0 : nullptr;
    if (c0 + E <= tout) {
      if (omx) store_chunk<T, E>(omx, ox);
      if (omn) store_chunk<T, E>(omn, on);
    } else {
#pragma unroll
      for (int k = 0; k < E; ++k)
        if (c0 + k < tout) {
          if (omx) omx[k] = ox[k];
          if (omn) omn[k] = on[k];
        }
    }
  }
}

}  // namespace mm

// kwarp.cuh -- window extrema computed by ONE warp over a staged, 128B-swizzled
// shared-memory buffer (k1d_base.cuh's layout).  Used by the warp-autonomous
// kernels: the fused stream push (stream.cu, N2) and the fused morphology
// kernel (morph.cu, N4).
//
// For lane l and k < E the warp computes the 32E consecutive windows starting
// at logical positions p = pos0 + l*E + k:
//     ox[k] = max A[p .. p+w)        on[k] = min B[p .. p+w)
// where a loader supplies A and B (the same staged buffer for the max-min
// filter; the arg filter's (value, position) keys, built on the fly from the
// staged values, for N1).  warp_window_med1 / warp_window_small1: one chain.
//
//   warp_window_med<G>: E <= w-1.  The near/far decomposition of k1d_medium
//     (k1d_medium.cuh, same names): block B = E*G <= w-1, out = max(S, gap, P)
//     with S a near-block suffix, P a far-block prefix and the gap assembled
//     from far-block aggregates G (whole block) and H (its last r' elements).
//     The far blocks before the warp's first block are reduced from the
//     staged halo on every call (the warp carries nothing between calls).
//   warp_window_small: w <= E.  Log-step doubling in registers to the span
//     s = 2^K <= w (max is idempotent: out = max(M_s[p], M_s[p + w - s])),
//     the runtime offset w - s applied by a barrel shift of K stages.
#pragma once

#include "k1d_medium.cuh"

namespace mm {

// cp.async staging for the warp-autonomous kernels: 16-B copies global ->
// shared, committed per segment; a ring of n stages keeps n-1 segments in flight.
__device__ __forceinline__ void cp_async16(void *smem, const void *g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// wait until at most n-1 copy groups are pending (n = 2..4, warp-uniform)
__device__ __forceinline__ void cp_async_wait_ring(int n) {
  if (n >= 4)
    asm volatile("cp.async.wait_group 3;" ::: "memory");
  else if (n == 3)
    asm volatile("cp.async.wait_group 2;" ::: "memory");
  else
    asm volatile("cp.async.wait_group 1;" ::: "memory");
}

// Gap geometry of block B = E*G for window w (E <= w-1): D = w-1-B = q'B + r'.
struct WarpGeom {
  int w;
  int qp, rp, V;       // q', r', far blocks before the first block: q' + (r' > 0)
  int h_lane, h_off;   // chunk and offset where a block's last r' elements start
};

template <int E>
__host__ inline WarpGeom make_warp_geom(int w, int G) {
  WarpGeom g;
  const int B = E * G, D = w - 1 - B;
  g.w = w;
  g.qp = D / B;
  g.rp = D - g.qp * B;
  g.V = g.qp + (g.rp > 0 ? 1 : 0);
  const int hstart = B - g.rp;
  g.h_lane = hstart / E;
  g.h_off = hstart - g.h_lane * E;
  return g;
}

// largest power-of-two G <= 32 with E*G <= w-1 (w-1 >= E)
template <int E>
__host__ inline int warp_group(int64_t w) {
  int G = 1;
  while (G < 32 && (int64_t)E * G * 2 <= w - 1) G *= 2;
  return G;
}

// Aggregate slots of one warp: AGG entries for each of G^max, G^min, H^max, H^min.
template <typename T>
struct WarpAgg {
  static constexpr int AGG = 64;
  T *gx, *gn, *hx, *hn;
  __device__ __forceinline__ explicit WarpAgg(unsigned char *p) {
    gx = reinterpret_cast<T *>(p);
    gn = gx + AGG;
    hx = gn + AGG;
    hn = hx + AGG;
  }
  static constexpr int bytes() { return 4 * AGG * (int)sizeof(T); }
};

// Loaders: ld.load<N>(pos, ya, yb) fills the N values of the max chain (ya) and
// of the min chain (yb) at logical positions pos .. pos+N-1.
template <typename T>
struct PairLoader {  // the max-min filter: both chains read the same staged buffer
  const unsigned char *X;
  static constexpr bool TWO = false;
  template <int N>
  __device__ __forceinline__ void load(int pos, T (&ya)[N], T (&yb)[N]) const {
    lds_swz<T, N>(X, pos, ya);
#pragma unroll
    for (int k = 0; k < N; ++k) yb[k] = ya[k];
  }
};

template <typename T>
struct TwoLoader {  // the max chain over A, the min chain over B
  const unsigned char *A, *B;
  static constexpr bool TWO = true;
  template <int N>
  __device__ __forceinline__ void load(int pos, T (&ya)[N], T (&yb)[N]) const {
    lds_swz<T, N>(A, pos, ya);
    lds_swz<T, N>(B, pos, yb);
  }
};

template <typename T, int E, int G, class Ld>
__device__ __forceinline__ void warp_window_med(const Ld &ld, int pos0, const WarpGeom &g, const WarpAgg<T> &agg,
                                                int lane, T (&ox)[E], T (&on)[E]) {
  constexpr bool TWO = Ld::TWO;
  constexpr int B = E * G;
  const int w = g.w;
  const int gl = lane & (G - 1);
  const int grp = lane / G;
  const int glast = (lane & ~(G - 1)) + G - 1;
  // H (max/min of a block's last r' elements) from a chunk y of the block
  auto h_part = [&](const T (&y)[E], T ax, T an, T bl, T &hx, T &hn) {
    hx = hn = bl;  // the block's last element: inside every non-empty H range
    if (g.rp > 0) {
      if (gl > g.h_lane) {
        hx = Ord<T>::mx(hx, ax);
        hn = Ord<T>::mn(hn, an);
      } else if (gl == g.h_lane) {
        T vx, vn;
        suffix_from<T, E>(y, g.h_off, vx, vn);
        hx = Ord<T>::mx(hx, vx);
        hn = Ord<T>::mn(hn, vn);
      }
    }
  };
  // (max over ya, min over yb) of a far chunk at pos: prefixes, aggregates
  T ux[E], un[E];
  T cx, cn;
  {  // ---- far chunk: prefix
    T ya[E], yb[E];
    ld.template load<E>(pos0 + lane * E + w - 1, ya, yb);
    ux[0] = ya[0];
    un[0] = yb[0];
#pragma unroll
    for (int k = 1; k < E; ++k) {
      ux[k] = Ord<T>::mx(ux[k - 1], ya[k]);
      un[k] = Ord<T>::mn(un[k - 1], yb[k]);
    }
    T hx, hn, tx, tn;
    h_part(ya, ux[E - 1], un[E - 1], __shfl_sync(0xffffffffu, ya[E - 1], glast), hx, tn);
    if (TWO) h_part(yb, ux[E - 1], un[E - 1], __shfl_sync(0xffffffffu, yb[E - 1], glast), tx, hn);
    else hn = tn;
    grp_reduce<T, G>(hx, hn);
    T ax = ux[E - 1], an = un[E - 1];
    grp_scan_up<T, G>(ax, an, gl);
    cx = shfl_up(ax, 1);
    cn = shfl_up(an, 1);
    if (gl == 0) {  // nothing before: an element inside every window
      cx = ya[0];
      cn = yb[0];
    }
    if (gl == G - 1) {
      agg.gx[g.V + grp] = ax;
      agg.gn[g.V + grp] = an;
      agg.hx[g.V + grp] = hx;
      agg.hn[g.V + grp] = hn;
    }
  }
  {  // ---- near chunk: suffix
    T xa[E], xb[E];
    ld.template load<E>(pos0 + lane * E, xa, xb);
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
    T bx = sx, bn = sn;
    grp_scan_down<T, G>(bx, bn, gl);
    T ex = shfl_down(bx, 1), en = shfl_down(bn, 1);
    if (gl == G - 1) {  // nothing after: an element inside every window of the chunk
      ex = xa[E - 1];
      en = xb[E - 1];
    }
    cx = Ord<T>::mx(cx, ex);
    cn = Ord<T>::mn(cn, en);
  }
  if (g.V > 0) {  // ---- far blocks before the first block (from the staged halo)
    const int nv = g.V * G;
    for (int r0 = 0; r0 < nv; r0 += 32) {
      const int vc = r0 + lane;
      const int vcc = vc < nv ? vc : nv - 1;
      const int gv = vcc / G;
      const int pos = pos0 + (gv - g.V) * B + w - 1 + gl * E;
      T ya[E], yb[E];
      ld.template load<E>(pos, ya, yb);
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
        agg.gx[gv] = ax;
        agg.gn[gv] = an;
        agg.hx[gv] = hx;
        agg.hn[gv] = hn;
      }
    }
  }
  __syncwarp();
  if (g.qp > 0 || g.rp > 0) {  // ---- gap
    const int b0 = g.V + grp - g.qp - 1;  // far block F_{g-q'-1}
    T mx, mn;
    if (g.rp > 0) {
      mx = agg.hx[b0];
      mn = agg.hn[b0];
    } else {
      mx = agg.gx[b0 + 1];
      mn = agg.gn[b0 + 1];
    }
    for (int s = 1; s <= g.qp; ++s) {
      mx = Ord<T>::mx(mx, agg.gx[b0 + s]);
      mn = Ord<T>::mn(mn, agg.gn[b0 + s]);
    }
    cx = Ord<T>::mx(cx, mx);
    cn = Ord<T>::mn(cn, mn);
  }
#pragma unroll
  for (int k = 0; k < E; ++k) {
    ox[k] = Ord<T>::mx(ux[k], cx);
    on[k] = Ord<T>::mn(un[k], cn);
  }
  __syncwarp();  // the aggregate slots are rewritten by the next call
}

// ---------------------------------------------------------------- small w
template <typename T, int N, int K, bool MAX>
__device__ __forceinline__ void span_levels(T (&v)[N]) {  // v[p] <- op v[p .. p + 2^K)
#pragma unroll
  for (int l = 0; l < K; ++l) {
#pragma unroll
    for (int p = 0; p + (1 << l) < N; ++p)  // ascending: v[p + 2^l] is still the previous level
      v[p] = MAX ? Ord<T>::mx(v[p], v[p + (1 << l)]) : Ord<T>::mn(v[p], v[p + (1 << l)]);
  }
}
template <typename T, int N, int K>
__device__ __forceinline__ void barrel_shift(T (&v)[N], int d) {  // v[p] <- v[p + d], d < 2^K
#pragma unroll
  for (int b = 0; b < K; ++b) {
    if ((d >> b) & 1) {
#pragma unroll
      for (int p = 0; p + (1 << b) < N; ++p) v[p] = v[p + (1 << b)];
    }
  }
}

template <typename T, int E, int K>
__device__ __forceinline__ void small_k(const T (&va)[2 * E], const T (&vb)[2 * E], int d, T (&ox)[E],
                                        T (&on)[E]) {
  constexpr int N = 2 * E;
  T mx[N], mn[N];
#pragma unroll
  for (int p = 0; p < N; ++p) {
    mx[p] = va[p];
    mn[p] = vb[p];
  }
  span_levels<T, N, K, true>(mx);
  span_levels<T, N, K, false>(mn);
  T sx[N], sn[N];
#pragma unroll
  for (int p = 0; p < N; ++p) {
    sx[p] = mx[p];
    sn[p] = mn[p];
  }
  barrel_shift<T, N, K>(sx, d);
  barrel_shift<T, N, K>(sn, d);
#pragma unroll
  for (int k = 0; k < E; ++k) {
    ox[k] = Ord<T>::mx(mx[k], sx[k]);
    on[k] = Ord<T>::mn(mn[k], sn[k]);
  }
}

template <typename T, int E, class Ld>
__device__ __forceinline__ void warp_window_small(const Ld &ld, int pos0, int w, int lane, T (&ox)[E], T (&on)[E]) {
  static_assert(E <= 16, "span levels up to 2^4");
  T va[2 * E], vb[2 * E];
  ld.template load<2 * E>(pos0 + lane * E, va, vb);
  const int K = 31 - __clz(w);  // 2^K <= w < 2^(K+1), w <= E
  const int d = w - (1 << K);
  switch (K) {  // warp-uniform
    case 0: small_k<T, E, 0>(va, vb, d, ox, on); break;
    case 1: small_k<T, E, 1>(va, vb, d, ox, on); break;
    case 2: small_k<T, E, 2>(va, vb, d, ox, on); break;
    case 3: small_k<T, E, 3>(va, vb, d, ox, on); break;
    default: small_k<T, E, 4>(va, vb, d, ox, on); break;
  }
}

// ------------------------------------------------ one chain (max or min only)
template <typename T, bool MAX>
__device__ __forceinline__ T op1(T a, T b) {
  return MAX ? Ord<T>::mx(a, b) : Ord<T>::mn(a, b);
}

// As warp_window_med, for one operation: out[k] = op X[pos0 + lane*E + k ..+ w).
// (The morphology's second pass: the max over the erosion buffer, then the min
// over the dilation buffer -- half the live registers of the pair version.)
template <typename T, int E, int G, bool MAX>
__device__ __forceinline__ void warp_window_med1(const unsigned char *X, int pos0, const WarpGeom &g,
                                                 const WarpAgg<T> &agg, int lane, T (&out)[E]) {
  constexpr int B = E * G;
  const int w = g.w;
  const int gl = lane & (G - 1);
  const int grp = lane / G;
  const int glast = (lane & ~(G - 1)) + G - 1;
  T *GA = MAX ? agg.gx : agg.gn;
  T *HA = MAX ? agg.hx : agg.hn;
  auto h_part = [&](const T (&y)[E], T a, T bl) {
    T h = bl;
    if (g.rp > 0) {
      if (gl > g.h_lane) {
        h = op1<T, MAX>(h, a);
      } else if (gl == g.h_lane) {
        T vx, vn;
        suffix_from<T, E>(y, g.h_off, vx, vn);
        h = op1<T, MAX>(h, MAX ? vx : vn);
      }
    }
    return h;
  };
  auto reduce = [&](T v) {
#pragma unroll
    for (int d = 1; d < G; d <<= 1) v = op1<T, MAX>(v, __shfl_xor_sync(0xffffffffu, v, d));
    return v;
  };
  T u[E];
  T c;
  {  // far chunk: prefix
    T y[E];
    lds_swz<T, E>(X, pos0 + lane * E + w - 1, y);
    u[0] = y[0];
#pragma unroll
    for (int k = 1; k < E; ++k) u[k] = op1<T, MAX>(u[k - 1], y[k]);
    T h = reduce(h_part(y, u[E - 1], __shfl_sync(0xffffffffu, y[E - 1], glast)));
    T a = u[E - 1];
#pragma unroll
    for (int d = 1; d < G; d <<= 1) {
      a = op1<T, MAX>(a, shfl_up_seg(a, d, G));  // (own value below d: idempotent)
    }
    c = shfl_up(a, 1);
    if (gl == 0) c = y[0];
    if (gl == G - 1) {
      GA[g.V + grp] = a;
      HA[g.V + grp] = h;
    }
  }
  {  // near chunk: suffix
    T x[E];
    lds_swz<T, E>(X, pos0 + lane * E, x);
    T sfx = x[E - 1];
    u[E - 1] = op1<T, MAX>(u[E - 1], sfx);
#pragma unroll
    for (int k = E - 2; k >= 0; --k) {
      sfx = op1<T, MAX>(sfx, x[k]);
      u[k] = op1<T, MAX>(u[k], sfx);
    }
    T b = sfx;
#pragma unroll
    for (int d = 1; d < G; d <<= 1) {
      b = op1<T, MAX>(b, shfl_down_seg(b, d, G));
    }
    T e = shfl_down(b, 1);
    if (gl == G - 1) e = x[E - 1];
    c = op1<T, MAX>(c, e);
  }
  if (g.V > 0) {  // far blocks before the first block
    const int nv = g.V * G;
    for (int r0 = 0; r0 < nv; r0 += 32) {
      const int vc = r0 + lane;
      const int vcc = vc < nv ? vc : nv - 1;
      const int gv = vcc / G;
      T y[E];
      lds_swz<T, E>(X, pos0 + (gv - g.V) * B + w - 1 + gl * E, y);
      T a = y[0];
#pragma unroll
      for (int k = 1; k < E; ++k) a = op1<T, MAX>(a, y[k]);
      T h = reduce(h_part(y, a, __shfl_sync(0xffffffffu, y[E - 1], glast)));
      a = reduce(a);
      if (vc < nv && gl == 0) {
        GA[gv] = a;
        HA[gv] = h;
      }
    }
  }
  __syncwarp();
  if (g.qp > 0 || g.rp > 0) {  // gap
    const int b0 = g.V + grp - g.qp - 1;
    T m = g.rp > 0 ? HA[b0] : GA[b0 + 1];
    for (int s = 1; s <= g.qp; ++s) m = op1<T, MAX>(m, GA[b0 + s]);
    c = op1<T, MAX>(c, m);
  }
#pragma unroll
  for (int k = 0; k < E; ++k) out[k] = op1<T, MAX>(u[k], c);
  __syncwarp();
}

template <typename T, int N, int K, bool MAX>
__device__ __forceinline__ void small1_k(const T (&v)[N], int d, T (&out)[N / 2]) {
  T m[N];
#pragma unroll
  for (int p = 0; p < N; ++p) m[p] = v[p];
  span_levels<T, N, K, MAX>(m);
  T sh[N];
#pragma unroll
  for (int p = 0; p < N; ++p) sh[p] = m[p];
  barrel_shift<T, N, K>(sh, d);
#pragma unroll
  for (int k = 0; k < N / 2; ++k) out[k] = op1<T, MAX>(m[k], sh[k]);
}

template <typename T, int E, bool MAX>
__device__ __forceinline__ void warp_window_small1(const unsigned char *X, int pos0, int w, int lane, T (&out)[E]) {
  T v[2 * E];
  lds_swz<T, 2 * E>(X, pos0 + lane * E, v);
  const int K = 31 - __clz(w);
  const int d = w - (1 << K);
  switch (K) {
    case 0: small1_k<T, 2 * E, 0, MAX>(v, d, out); break;
    case 1: small1_k<T, 2 * E, 1, MAX>(v, d, out); break;
    case 2: small1_k<T, 2 * E, 2, MAX>(v, d, out); break;
    case 3: small1_k<T, 2 * E, 3, MAX>(v, d, out); break;
    default: small1_k<T, 2 * E, 4, MAX>(v, d, out); break;
  }
}

}  // namespace mm

// argfilter.cu -- arg-max / arg-min filter: besides the
// max and min of every window, the position of each (the paper keeps
// locations so they come "with no overhead").  Ties: the
// EARLIEST position for both (reading R17).
//
// Every (value, position) pair travels as one 64-bit key whose order is the
// wanted one, so the argument filter IS a max (min) filter on keys and runs on
// the library's 8-byte kernels unchanged:
//   max side:  kx = ord(v) << 32 | (2^32-1 - i)   max key = max value, then
//                                                   the smallest position
//   min side:  kn = ord(v) << 32 | i               min key = min value, then
//                                                   the smallest position
// with ord() an order-preserving map of the <= 4-byte element type to uint32
// (floats: the sign-magnitude flip; +-0 both map to +0's code, reading R8).
// Paths, in order of preference (the keys never reach memory in the first two):
//   * 8 < w <= 8193, 16-B aligned input rows: k1d_medium itself on 64-bit keys
//     with a source policy (ArgSrc: TMA stages the raw values, the loads build
//     both keys with their row positions) and a decoding epilogue (ArgEpi):
//     the contract's traffic, 4n + 24m bytes for f32;
//   * w-1 <= kArgHMax: the warp-autonomous kernel (k_arg_fused, kwarp.cuh),
//     cp.async staging, keys built in the loads (ArgLoader) -- small windows
//     and unaligned rows;
//   * otherwise the composition: keys (elementwise), the max filter on kx and
//     the min filter on kn (the 8-byte 1-D kernels), decode (elementwise); the
//     keys and the key outputs live in the workspace, ~92 B of HBM traffic per
//     element.
#include "kwarp.cuh"
#include "launch.cuh"

namespace mm {

template <typename T>
__device__ __forceinline__ uint32_t ord32(T v) {
  if constexpr (std::is_same<T, float>::value) {
    uint32_t b = __float_as_uint(v);
    if (v == 0.0f) b = 0u;  // -0 and +0 compare equal: one code
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  } else if constexpr (std::is_signed<T>::value) {
    return (uint32_t)(int32_t)v ^ 0x80000000u;
  } else {
    return (uint32_t)v;
  }
}
template <typename T>
__device__ __forceinline__ T unord32(uint32_t o) {
  if constexpr (std::is_same<T, float>::value) {
    const uint32_t b = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
    return __uint_as_float(b);
  } else if constexpr (std::is_signed<T>::value) {
    return (T)(int32_t)(o ^ 0x80000000u);
  } else {
    return (T)o;
  }
}

// keys of row b, positions [0, n): kx/kn rows of pitch kld (even)
template <typename T>
__global__ void __launch_bounds__(256) k_argkeys(const T *__restrict__ in, int64_t batch, int64_t n,
                                                 int64_t in_ld, uint64_t *__restrict__ kx,
                                                 uint64_t *__restrict__ kn, int64_t kld) {
  const int64_t half = (n + 1) / 2;  // pairs of positions per row
  const int64_t total = batch * half;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / half;
    const int64_t i = 2 * (t - b * half);
    const T *row = in + b * in_ld;
    const uint64_t o0 = (uint64_t)ord32<T>(row[i]) << 32;
    const uint64_t o1 = i + 1 < n ? (uint64_t)ord32<T>(row[i + 1]) << 32 : 0;
    const uint32_t i0 = (uint32_t)i, i1 = (uint32_t)(i + 1);
    const ulonglong2 vx = make_ulonglong2(o0 | (0xffffffffu - i0), o1 | (0xffffffffu - i1));
    const ulonglong2 vn = make_ulonglong2(o0 | i0, o1 | i1);
    *reinterpret_cast<ulonglong2 *>(kx + b * kld + i) = vx;
    *reinterpret_cast<ulonglong2 *>(kn + b * kld + i) = vn;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_argdecode(const uint64_t *__restrict__ okx,
                                                   const uint64_t *__restrict__ okn, int64_t batch,
                                                   int64_t m, int64_t kld, T *out_max, T *out_min,
                                                   int64_t *arg_max, int64_t *arg_min, int64_t out_ld) {
  const int64_t total = batch * m;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / m, j = t - b * m;
    const int64_t o = b * out_ld + j;
    if (okx) {
      const uint64_t k = okx[b * kld + j];
      if (out_max) out_max[o] = unord32<T>((uint32_t)(k >> 32));
      if (arg_max) arg_max[o] = (int64_t)(0xffffffffu - (uint32_t)k);
    }
    if (okn) {
      const uint64_t k = okn[b * kld + j];
      if (out_min) out_min[o] = unord32<T>((uint32_t)(k >> 32));
      if (arg_min) arg_min[o] = (int64_t)(uint32_t)k;
    }
  }
}

namespace {
struct ArgLayout {  // workspace: [kx | kn | okx | okn | inner], 256-B aligned pieces
  int64_t kld, mld;
  size_t keys, outs, inner, total;
};
size_t up256(size_t x) { return (x + 255) & ~size_t(255); }
ArgLayout arg_layout(int64_t batch, int64_t n, int64_t w) {
  ArgLayout L;
  const int64_t m = n - w + 1;
  L.kld = (n + 1) & ~int64_t(1);  // 16-B rows of 8-byte keys
  L.mld = (m + 1) & ~int64_t(1);
  L.keys = up256((size_t)batch * L.kld * 8);
  L.outs = up256((size_t)batch * L.mld * 8);
  L.inner = up256(workspace_1d<uint64_t>(batch, L.kld, w));
  L.total = 2 * L.keys + 2 * L.outs + L.inner;
  return L;
}
int grid_for(int64_t items) {
  int64_t g = (items + 255) / 256;
  const int64_t cap = (int64_t)sm_count() * 8;
  return (int)(g < cap ? (g > 0 ? g : 1) : cap);
}
}  // namespace

constexpr int kArgFusedHMax = 1024;  // = kArgHMax below: the fused path needs no workspace
size_t argfilter_workspace(int64_t batch, int64_t n, int64_t w) {
  const int64_t m = n - w + 1;
  if (w - 1 <= kArgFusedHMax && batch * ((m + 255) / 256) <= 0x7fffffffLL) return 0;
  return arg_layout(batch, n, w).total;
}

template <typename S>
int launch_arg_fused(const void *in, int64_t batch, int64_t n, int64_t in_ld, int64_t w, void *out_max, void *out_min,
                     int64_t *arg_max, int64_t *arg_min, int64_t out_ld, cudaStream_t s);
template <typename S>
int launch_arg_medium(const void *in, int64_t batch, int64_t n, int64_t in_ld, int64_t w, void *out_max,
                      void *out_min, int64_t *arg_max, int64_t *arg_min, int64_t out_ld, cudaStream_t s);

template <typename T>
int launch_argfilter(const void *in, int64_t batch, int64_t n, int64_t in_ld, int64_t w, void *out_max,
                     void *out_min, int64_t *arg_max, int64_t *arg_min, int64_t out_ld, void *ws,
                     size_t ws_bytes, cudaStream_t s) {
  static_assert(sizeof(T) <= 4, "keys hold a 32-bit order code and a 32-bit position");
  if (batch == 0) return kOK;
  {
    int rc = launch_arg_medium<T>(in, batch, n, in_ld, w, out_max, out_min, arg_max, arg_min, out_ld, s);
    if (rc != kErrUnsupported) return rc;
    rc = launch_arg_fused<T>(in, batch, n, in_ld, w, out_max, out_min, arg_max, arg_min, out_ld, s);
    if (rc != kErrUnsupported) return rc;
  }
  const ArgLayout L = arg_layout(batch, n, w);
  if (!ws || ws_bytes < L.total) return kErrWorkspace;
  char *p = static_cast<char *>(ws);
  uint64_t *kx = reinterpret_cast<uint64_t *>(p);
  uint64_t *kn = reinterpret_cast<uint64_t *>(p + L.keys);
  uint64_t *okx = reinterpret_cast<uint64_t *>(p + 2 * L.keys);
  uint64_t *okn = reinterpret_cast<uint64_t *>(p + 2 * L.keys + L.outs);
  void *inner = p + 2 * L.keys + 2 * L.outs;
  const bool want_max = out_max || arg_max, want_min = out_min || arg_min;
  const int64_t m = n - w + 1;
  k_argkeys<T><<<grid_for(batch * ((n + 1) / 2)), 256, 0, s>>>(static_cast<const T *>(in), batch, n, in_ld,
                                                             kx, kn, L.kld);
  int rc = note_cuda(cudaGetLastError());
  if (rc) return rc;
  // the key rows hold n keys at pitch kld: the filter sees rows of length n
  if (want_max) {
    rc = launch_1d<uint64_t>(kx, batch, n, L.kld, w, okx, nullptr, L.mld, inner, L.inner, s);
    if (rc) return rc;
  }
  if (want_min) {
    rc = launch_1d<uint64_t>(kn, batch, n, L.kld, w, nullptr, okn, L.mld, inner, L.inner, s);
    if (rc) return rc;
  }
  k_argdecode<T><<<grid_for(batch * m), 256, 0, s>>>(want_max ? okx : nullptr, want_min ? okn : nullptr,
                                                    batch, m, L.mld, static_cast<T *>(out_max),
                                                    static_cast<T *>(out_min), arg_max, arg_min, out_ld);
  return note_cuda(cudaGetLastError());
}

// ============================================================ fused path
constexpr int kArgHMax = kArgFusedHMax;  // largest w-1 of k_arg_fused
constexpr int kArgWarps = 4;

// the two keys of the staged values at logical positions pos.. (absolute base+pos..)
template <typename S>
struct ArgLoader {
  const unsigned char *X;
  uint32_t base;
  static constexpr bool TWO = true;
  template <int N>
  __device__ __forceinline__ void load(int pos, uint64_t (&ya)[N], uint64_t (&yb)[N]) const {
    S v[N];
    lds_swz<S, N>(X, pos, v);
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const uint64_t o = (uint64_t)ord32<S>(v[k]) << 32;
      const uint32_t i = base + (uint32_t)(pos + k);
      ya[k] = o | (0xffffffffu - i);
      yb[k] = o | i;
    }
  }
};

template <typename S>
struct ArgGeo {
  static constexpr int E = 8;  // 8-byte keys
  static constexpr int SEG = 32 * E;
  static constexpr int VEC = 16 / (int)sizeof(S);
  __host__ __device__ static int stage_bytes(int w) {
    return ((SEG + w - 1 + 2 * E + 2 * VEC + 16) * (int)sizeof(S) + 127) / 128 * 128;
  }
  __host__ __device__ static int warp_bytes(int w, int ns) { return ns * stage_bytes(w) + WarpAgg<uint64_t>::bytes(); }
  __host__ __device__ static size_t cta_bytes(int w, int ns, int nw) { return 1024 + (size_t)nw * warp_bytes(w, ns); }
};

struct ArgArgs {
  const void *in;
  void *out_max, *out_min;
  int64_t *arg_max, *arg_min;
  int64_t n, m, in_ld, out_ld, batch, segs_per_row, nseg;
  WarpGeom g;
  int w, in_vec, out_vec, stage_bytes, warp_bytes, nstages;
};


template <typename S>
__device__ __forceinline__ void arg_stage(const ArgArgs &a, unsigned char *X, int64_t row, int64_t j0, int lane) {
  constexpr int VEC = 16 / (int)sizeof(S);
  const int64_t want = j0 + ArgGeo<S>::SEG + a.w - 1;
  const int64_t end = want < a.n ? want : a.n;
  const int nq = (int)((end - j0 + VEC - 1) / VEC);
  const S *src = static_cast<const S *>(a.in) + row * a.in_ld;
  for (int q = lane; q < nq; q += 32) {
    const int64_t v = j0 + (int64_t)q * VEC;
    unsigned char *dst = X + swz(q);
    if (a.in_vec && v + VEC <= a.n) {
      cp_async16(dst, src + v);
    } else {
      S t[VEC];
#pragma unroll
      for (int k = 0; k < VEC; ++k) t[k] = v + k < a.n ? src[v + k] : S(0);
      uint4 u4;
      memcpy(&u4, t, 16);
      *reinterpret_cast<uint4 *>(dst) = u4;
    }
  }
}

template <typename S, int G>
__global__ void __launch_bounds__(32 * kArgWarps) k_arg_fused(ArgArgs a) {
  using Geo = ArgGeo<S>;
  constexpr int E = Geo::E;
  constexpr int SEG = Geo::SEG;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *base = smem_align1024(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char *wb = base + warp * a.warp_bytes;
  auto stg = [&](int i) { return wb + i * a.stage_bytes; };
  const WarpAgg<uint64_t> agg(wb + a.nstages * a.stage_bytes);
  const int nwb = blockDim.x >> 5;
  const int64_t gw = blockIdx.x * (int64_t)nwb + warp, nw = (int64_t)gridDim.x * nwb;
  auto seg_pos = [&](int64_t sg, int64_t &row, int64_t &j0) {  // nseg < 2^31 (launcher)
    const uint32_t r = (uint32_t)sg / (uint32_t)a.segs_per_row;
    row = r;
    j0 = ((int64_t)sg - (int64_t)r * a.segs_per_row) * SEG;
  };
  const int ns = a.nstages;
  for (int k = 0; k + 1 < ns; ++k) {
    const int64_t sg = gw + k * nw;
    if (sg < a.nseg) {
      int64_t row, j0;
      seg_pos(sg, row, j0);
      arg_stage<S>(a, stg(k), row, j0, lane);
    }
    cp_async_commit();
  }
  int slot = 0;
  for (int64_t sg = gw; sg < a.nseg; sg += nw) {
    {
      const int64_t nx = sg + (ns - 1) * nw;
      if (nx < a.nseg) {
        int64_t row, j0;
        seg_pos(nx, row, j0);
        arg_stage<S>(a, stg(slot + ns - 1 < ns ? slot + ns - 1 : slot - 1), row, j0, lane);
      }
    }
    cp_async_commit();
    cp_async_wait_ring(ns);
    __syncwarp();
    const unsigned char *X = stg(slot);
    slot = slot + 1 < ns ? slot + 1 : 0;
    int64_t row, j0;
    seg_pos(sg, row, j0);
    uint64_t kx[E], kn[E];
    const ArgLoader<S> ld{X, (uint32_t)j0};
    if constexpr (G == 0)
      warp_window_small<uint64_t, E>(ld, 0, a.w, lane, kx, kn);
    else
      warp_window_med<uint64_t, E, G>(ld, 0, a.g, agg, lane, kx, kn);
    const int64_t j = j0 + lane * E;
    const int64_t left = a.m - j;
    if (left > 0) {
      const int64_t o = row * a.out_ld + j;
      S vx[E], vn[E];
      int64_t ix[E], in_[E];
#pragma unroll
      for (int k = 0; k < E; ++k) {
        vx[k] = unord32<S>((uint32_t)(kx[k] >> 32));
        ix[k] = (int64_t)(0xffffffffu - (uint32_t)kx[k]);
        vn[k] = unord32<S>((uint32_t)(kn[k] >> 32));
        in_[k] = (int64_t)(uint32_t)kn[k];
      }
      S *omx = a.out_max ? static_cast<S *>(a.out_max) + o : nullptr;
      S *omn = a.out_min ? static_cast<S *>(a.out_min) + o : nullptr;
      int64_t *oax = a.arg_max ? a.arg_max + o : nullptr;
      int64_t *oan = a.arg_min ? a.arg_min + o : nullptr;
      if (left >= E && a.out_vec) {
        if constexpr ((E * sizeof(S)) % 16 == 0) {
          if (omx) store_chunk<S, E>(omx, vx);
          if (omn) store_chunk<S, E>(omn, vn);
        } else {
#pragma unroll
          for (int k = 0; k < E; ++k) {
            if (omx) omx[k] = vx[k];
            if (omn) omn[k] = vn[k];
          }
        }
        if (oax) store_chunk<int64_t, E>(oax, ix);
        if (oan) store_chunk<int64_t, E>(oan, in_);
      } else {
#pragma unroll
        for (int k = 0; k < E; ++k)
          if (k < left) {
            if (omx) omx[k] = vx[k];
            if (omn) omn[k] = vn[k];
            if (oax) oax[k] = ix[k];
            if (oan) oan[k] = in_[k];
          }
      }
    }
    __syncwarp();
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

template <typename S, int G>
int launch_arg_g(ArgArgs a, cudaStream_t s) {
  using Geo = ArgGeo<S>;
  WarpLaunch L;  // resident warps first
  int rc = warp_launch_choice(reinterpret_cast<const void *>(k_arg_fused<S, G>), a.w, kArgWarps, 1,
                              [](int w, int ns, int nw) { return Geo::cta_bytes(w, ns, nw); }, 1, &L);
  if (rc) return rc;
  a.nstages = L.ns;
  a.stage_bytes = Geo::stage_bytes(a.w);
  a.warp_bytes = Geo::warp_bytes(a.w, L.ns);
  const int64_t want = (a.nseg + L.nw - 1) / L.nw;
  const int64_t cap = (int64_t)sm_count() * L.per_sm;
  k_arg_fused<S, G><<<(int)(want < cap ? want : cap), 32 * L.nw, L.smem, s>>>(a);
  return note_cuda(cudaGetLastError());
}

// ------------------------------------------- CTA path: k1d_medium on keys
// 8 < w <= kHaloMax+1: the library's medium kernel (TMA tiles of 2048 windows,
// far-block aggregates carried across tiles) filters the keys, built from the
// staged values inside its loads (ArgSrc), and the epilogue decodes them.
template <typename V>
struct ArgSrc {
  using S = V;  // staged element type (k1d_medium's Src::S)
  static constexpr bool TWO = true;
  template <int E>
  __device__ __forceinline__ static void keys(const S (&v)[E], int64_t p0, uint64_t (&ya)[E], uint64_t (&yb)[E]) {
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const uint64_t o = (uint64_t)ord32<S>(v[k]) << 32;
      const uint32_t i = (uint32_t)p0 + (uint32_t)k;
      ya[k] = o | (0xffffffffu - i);
      yb[k] = o | i;
    }
  }
  template <int E>
  __device__ __forceinline__ static void load(const unsigned char *X, int pos, int64_t u0, uint64_t (&ya)[E],
                                              uint64_t (&yb)[E]) {
    S v[E];
    lds_swz<S, E>(X, pos, v);
    keys<E>(v, u0 + pos, ya, yb);
  }
  template <int E>
  __device__ __forceinline__ static void load_aligned(const unsigned char *X, int pos, int64_t u0, uint64_t (&ya)[E],
                                                      uint64_t (&yb)[E]) {
    S v[E];
    lds_swz<S, E>(X, pos, v);  // E*sizeof(S) may be < 16 B: the general read
    keys<E>(v, u0 + pos, ya, yb);
  }
};
template <typename S>
struct ArgEpi {
  S *out_max, *out_min;
  int64_t *arg_max, *arg_min;
  int64_t out_ld;
  int vec;  // every output row 16-B aligned
  template <typename T, int E>
  __device__ __forceinline__ void operator()(const Rows &p, int64_t row, int64_t j0, int cnt, const T (&ox)[E],
                                             const T (&on)[E]) const {
    if (cnt <= 0) return;
    S vx[E], vn[E];
    int64_t ix[E], in_[E];
#pragma unroll
    for (int k = 0; k < E; ++k) {
      vx[k] = unord32<S>((uint32_t)(ox[k] >> 32));
      ix[k] = (int64_t)(0xffffffffu - (uint32_t)ox[k]);
      vn[k] = unord32<S>((uint32_t)(on[k] >> 32));
      in_[k] = (int64_t)(uint32_t)on[k];
    }
    const int64_t o = row * out_ld + j0;
    S *omx = out_max ? out_max + o : nullptr;
    S *omn = out_min ? out_min + o : nullptr;
    int64_t *oax = arg_max ? arg_max + o : nullptr;
    int64_t *oan = arg_min ? arg_min + o : nullptr;
    if (cnt >= E && vec) {
      if constexpr ((E * sizeof(S)) % 16 == 0) {
        if (omx) store_chunk<S, E>(omx, vx);
        if (omn) store_chunk<S, E>(omn, vn);
      } else {
#pragma unroll
        for (int k = 0; k < E; ++k) {
          if (omx) omx[k] = vx[k];
          if (omn) omn[k] = vn[k];
        }
      }
      if (oax) store_chunk<int64_t, E>(oax, ix);
      if (oan) store_chunk<int64_t, E>(oan, in_);
    } else {
#pragma unroll
      for (int k = 0; k < E; ++k)
        if (k < cnt) {
          if (omx) omx[k] = vx[k];
          if (omn) omn[k] = vn[k];
          if (oax) oax[k] = ix[k];
          if (oan) oan[k] = in_[k];
        }
    }
  }
};

template <typename S, int G>
int launch_arg_medium_g(const Rows &p, const TmaMaps &maps, const ArgEpi<S> &epi, cudaStream_t s) {
  const MedGeom g = medium_geom<uint64_t>(p.w, G);
  // three stages where the tile carries a gap (launch.cuh, launch_medium_g)
  if (MM_MED_RING3 && (g.qp > 0 || (g.rp > 0 && G >= 8)) &&
      2 * (MedLayoutS<uint64_t, S>::bytes(p.w, g.ring, 3) + 1024) <= 228 * 1024) {
    auto kern = k1d_medium<uint64_t, G, ArgEpi<S>, ArgSrc<S>, false, 3>;
    static size_t attr = 0;
    const size_t smem = MedLayoutS<uint64_t, S>::bytes(p.w, g.ring, 3);
    int rc = set_smem(kern, smem, attr);
    if (rc) return rc;
    int grid = 0;
    rc = occupancy_grid(kern, smem, p.ntiles, grid);
    if (rc) return rc;
    kern<<<grid, NT, smem, s>>>(p, g, maps, epi);
    return note_cuda(cudaGetLastError());
  }
  auto kern = k1d_medium<uint64_t, G, ArgEpi<S>, ArgSrc<S>>;
  static size_t attr = 0;
  const size_t smem = MedLayoutS<uint64_t, S>::bytes(p.w, g.ring);
  int rc = set_smem(kern, smem, attr);
  if (rc) return rc;
  int grid = 0;
  rc = occupancy_grid(kern, smem, p.ntiles, grid);
  if (rc) return rc;
  kern<<<grid, NT, smem, s>>>(p, g, maps, epi);
  return note_cuda(cudaGetLastError());
}

template <typename S>
int launch_arg_medium(const void *in, int64_t batch, int64_t n, int64_t in_ld, int64_t w, void *out_max,
                      void *out_min, int64_t *arg_max, int64_t *arg_min, int64_t out_ld, cudaStream_t s) {
  if (w <= Chunk<uint64_t>::E || w > kHaloMax + 1) return kErrUnsupported;
  if ((reinterpret_cast<uintptr_t>(in) % 16) != 0 || (batch > 1 && (in_ld * (int64_t)sizeof(S)) % 16 != 0))
    return kErrUnsupported;  // TMA rows
  Rows p;
  std::memset(&p, 0, sizeof(p));
  p.in = in;
  p.n = n;
  p.w = w;
  p.m = n - w + 1;
  p.in_ld = in_ld;
  p.out_ld = out_ld;
  p.batch = batch;
  p.tiles_per_row = (p.m + Geo1D<uint64_t>::TILE - 1) / Geo1D<uint64_t>::TILE;
  p.ntiles = batch * p.tiles_per_row;
  TmaMaps maps;
  std::memset(&maps, 0, sizeof(maps));
  const int64_t full_rows = n / Rowing<S>::RW;
  p.has_map = full_rows > 0 ? 1 : 0;
  if (p.has_map) {
    int rc = encode_rows_map(&maps.small, in, (int)sizeof(S), full_rows, batch, in_ld * (int64_t)sizeof(S));
    if (rc) return rc;
    rc = encode_rows_map(&maps.big, in, (int)sizeof(S), full_rows, batch, in_ld * (int64_t)sizeof(S), kBigRows);
    if (rc) return rc;
  }
  ArgEpi<S> epi;
  epi.out_max = static_cast<S *>(out_max);
  epi.out_min = static_cast<S *>(out_min);
  epi.arg_max = arg_max;
  epi.arg_min = arg_min;
  epi.out_ld = out_ld;
  auto al = [](const void *q) { return q == nullptr || reinterpret_cast<uintptr_t>(q) % 16 == 0; };
  // one row: the pitch never enters an address, so only the base pointers matter
  epi.vec = (al(out_max) && al(out_min) && al(arg_max) && al(arg_min) &&
             (batch == 1 || ((out_ld * 8) % 16 == 0 && (out_ld * (int64_t)sizeof(S)) % 16 == 0))) ? 1 : 0;
  switch (medium_G<uint64_t>(w)) {
    case 1: return launch_arg_medium_g<S, 1>(p, maps, epi, s);
    case 2: return launch_arg_medium_g<S, 2>(p, maps, epi, s);
    case 4: return launch_arg_medium_g<S, 4>(p, maps, epi, s);
    case 8: return launch_arg_medium_g<S, 8>(p, maps, epi, s);
    case 16: return launch_arg_medium_g<S, 16>(p, maps, epi, s);
    default: return launch_arg_medium_g<S, 32>(p, maps, epi, s);
  }
}

// kErrUnsupported when the fused path does not apply (the caller composes)
template <typename S>
int launch_arg_fused(const void *in, int64_t batch, int64_t n, int64_t in_ld, int64_t w, void *out_max, void *out_min,
                     int64_t *arg_max, int64_t *arg_min, int64_t out_ld, cudaStream_t s) {
  using Geo = ArgGeo<S>;
  constexpr int E = Geo::E;
  if (w - 1 > kArgHMax) return kErrUnsupported;
  ArgArgs a;
  std::memset(&a, 0, sizeof(a));
  a.in = in;
  a.out_max = out_max;
  a.out_min = out_min;
  a.arg_max = arg_max;
  a.arg_min = arg_min;
  a.n = n;
  a.m = n - w + 1;
  a.in_ld = in_ld;
  a.out_ld = out_ld;
  a.batch = batch;
  a.segs_per_row = (a.m + Geo::SEG - 1) / Geo::SEG;
  a.nseg = batch * a.segs_per_row;
  if (a.nseg > 0x7fffffffLL) return kErrUnsupported;
  a.w = (int)w;
  a.in_vec = (reinterpret_cast<uintptr_t>(in) % 16 == 0 && (batch == 1 || (in_ld * (int64_t)sizeof(S)) % 16 == 0))
                 ? 1 : 0;
  auto al = [](const void *p) { return p == nullptr || reinterpret_cast<uintptr_t>(p) % 16 == 0; };
  a.out_vec = (al(out_max) && al(out_min) && al(arg_max) && al(arg_min) &&
               (batch == 1 || ((out_ld * 8) % 16 == 0 && (out_ld * (int64_t)sizeof(S)) % 16 == 0))) ? 1 : 0;
  if (w - 1 < E) {
    a.g.w = (int)w;
    return launch_arg_g<S, 0>(a, s);
  }
  const int G = warp_group<E>(w);
  a.g = make_warp_geom<E>((int)w, G);
  if (a.g.V + 32 / G > WarpAgg<uint64_t>::AGG) return kErrUnsupported;
  switch (G) {
    case 1: return launch_arg_g<S, 1>(a, s);
    case 2: return launch_arg_g<S, 2>(a, s);
    case 4: return launch_arg_g<S, 4>(a, s);
    case 8: return launch_arg_g<S, 8>(a, s);
    case 16: return launch_arg_g<S, 16>(a, s);
    default: return launch_arg_g<S, 32>(a, s);
  }
}

#define MM_ARG_INST(T)                                                                           \
  template int launch_argfilter<T>(const void *, int64_t, int64_t, int64_t, int64_t, void *, void *, \
                                   int64_t *, int64_t *, int64_t, void *, size_t, cudaStream_t);
MM_ARG_INST(uint8_t)
MM_ARG_INST(int8_t)
MM_ARG_INST(uint16_t)
MM_ARG_INST(int16_t)
MM_ARG_INST(uint32_t)
MM_ARG_INST(int32_t)
MM_ARG_INST(float)

}  // namespace mm

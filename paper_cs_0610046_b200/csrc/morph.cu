// morph.cu -- grayscale opening and closing.
//
// The 2-D application family of the filter: "applied to images ... by first
// applying the unidimensional on rows and then on columns";
// erosion is the min filter, dilation the max filter, and the opening /
// closing are their compositions.  With the structuring element kept inside
// the data (reading R20), for every position i of a row of n:
//   e[j] = min a[j .. j+w),  d[j] = max a[j .. j+w)          j in [0, m), m = n-w+1
//   open[i]  = max e[j] over j in [i-w+1, i] ∩ [0, m)
//   close[i] = min d[j] over the same j
//
// 1-D / batched rows (k_morph_fused): ONE pass -- the input is read once, the
// opening and the closing are written once each.  Warp-autonomous like the
// fused stream push (stream.cu): a warp owns a segment of 32E outputs of one
// row, stages a[j0-(w-1), j0+32E+w-1) with cp.async into its swizzled buffer
// (a ring of segments in flight), computes e and d for the 32E+w-1 positions
// [j0-(w-1), j0+32E) into two on-chip buffers (positions outside [0, m) get
// the identity of the next step: lowest for e, highest for d), then the max
// over e and the min over d (kwarp.cuh: near/far blocks for w-1 >= E,
// log-step + barrel shift for w <= E).  w-1 <= kMorphHMax.
//
// 2-D images (launch_morph_2d): the rectangle opening is not a product of 1-D
// openings (max and min along different axes do not commute), so it runs as a
// composition of the library's 2-D filter: e and d of the valid region into
// the interior of two padded buffers whose (w-1)-wide frames hold the
// identities, then the 2-D max over the padded e and the 2-D min over the
// padded d.  HBM: 1 read + 2 writes + 2 reads + 2 writes (vs 1 + 2 fused).
// 1-byte pixels with the packed kernel's square windows skip the frames: the
// second and third passes read e and ~d through the tensor map's zero frame
// (launch_morph_2d_byte, k2d_byte.cu).
#include "kwarp.cuh"
#include "launch.cuh"

#include <limits>

namespace mm {

constexpr int kMorphWarps = 4;
constexpr int kMorphHMax = 8192;  // largest w-1 of k_morph_fused (past ~1024 a warp stages w-1 twice: few warps fit)

template <typename T>
__device__ __forceinline__ T lowest_value() {
  if constexpr (std::is_floating_point<T>::value) return -std::numeric_limits<T>::infinity();
  else return std::numeric_limits<T>::lowest();
}
template <typename T>
__device__ __forceinline__ T highest_value() {
  if constexpr (std::is_floating_point<T>::value) return std::numeric_limits<T>::infinity();
  else return std::numeric_limits<T>::max();
}

#ifndef MM_MORPH_E
#define MM_MORPH_E 16
#endif
template <typename T>
struct MorphGeo {
  // elements per lane (<= Chunk<T>::E; at least one 16-B unit)
  static constexpr int E = (MM_MORPH_E < Chunk<T>::E ? (MM_MORPH_E * (int)sizeof(T) >= 16 ? MM_MORPH_E : 16 / (int)sizeof(T))
                                                     : Chunk<T>::E);
  static constexpr int VEC = 16 / (int)sizeof(T);
  static constexpr int SEG = 32 * E;
  __host__ __device__ static int round128(int bytes) { return (bytes + 127) / 128 * 128; }
  // offset of position j0 in the erosion / dilation buffers (the w-1 carried before it)
  __host__ __device__ static int off(int w) { return (w - 1 + VEC - 1) / VEC * VEC; }
  // staged input f[j0, j0 + SEG + w - 1) + over-reads
  __host__ __device__ static int stage_bytes(int w) { return round128((SEG + w + E + 2 * VEC) * (int)sizeof(T)); }
  __host__ __device__ static int ebuf_bytes(int w) { return round128((off(w) + SEG + E + 2 * VEC) * (int)sizeof(T)); }
  __host__ __device__ static int warp_bytes(int w, int ns) {
    return ns * stage_bytes(w) + 2 * ebuf_bytes(w) + WarpAgg<T>::bytes();
  }
  __host__ __device__ static size_t cta_bytes(int w, int ns, int warps = kMorphWarps) {
    return 1024 + (size_t)warps * warp_bytes(w, ns);
  }
};

struct MorphArgs {
  const void *in;
  void *out_open;
  void *out_close;
  int64_t n, m, in_ld, out_ld, batch;
  int64_t segs_per_row, nseg;
  WarpGeom g;
  int w;
  int in_vec;  // input rows 16-B aligned
  int stage_bytes, ebuf_bytes, warp_bytes, nstages;
};


// stage f[j0, j0 + SEG + w - 1) of `row` (j0 is a multiple of SEG: 16-B aligned)
template <typename T>
__device__ __forceinline__ void morph_stage(const MorphArgs &a, unsigned char *X, int64_t row, int64_t j0, int lane) {
  constexpr int VEC = 16 / (int)sizeof(T);
  constexpr int SEG = MorphGeo<T>::SEG;
  const int64_t want_end = j0 + SEG + a.w - 1;
  const int64_t end = want_end < a.n ? want_end : a.n;
  const int nq = (int)((end - j0 + VEC - 1) / VEC);
  const T *src = static_cast<const T *>(a.in) + row * a.in_ld;
  for (int q = lane; q < nq; q += 32) {
    const int64_t v = j0 + (int64_t)q * VEC;
    unsigned char *dst = X + swz(q);
    if (a.in_vec && v + VEC <= a.n) {
      cp_async16(dst, src + v);
    } else {
      T t[VEC];
#pragma unroll
      for (int k = 0; k < VEC; ++k) t[k] = v + k < a.n ? src[v + k] : T(0);
      uint4 u4;
      memcpy(&u4, t, 16);
      *reinterpret_cast<uint4 *>(dst) = u4;
    }
  }
}

// E elements at logical position pos (a multiple of E) of a swizzled buffer
template <typename T, int E>
__device__ __forceinline__ void sts_swz_chunk(unsigned char *buf, int pos, const T (&v)[E]) {
  constexpr int VEC = 16 / (int)sizeof(T);
  static_assert((E % VEC) == 0, "whole 16-B units");
#pragma unroll
  for (int u = 0; u < E / VEC; ++u) {
    uint4 q;
    memcpy(&q, &v[u * VEC], 16);
    *reinterpret_cast<uint4 *>(buf + swz(pos / VEC + u)) = q;
  }
}

template <typename T, int E, int G>
__device__ __forceinline__ void morph_window(const unsigned char *X, int pos0, const WarpGeom &g,
                                             const WarpAgg<T> &agg, int lane, T (&ox)[E], T (&on)[E]) {
  if constexpr (G == 0)
    warp_window_small<T, E>(PairLoader<T>{X}, pos0, g.w, lane, ox, on);
  else
    warp_window_med<T, E, G>(PairLoader<T>{X}, pos0, g, agg, lane, ox, on);
}

#ifndef MM_MORPH_P2PAIR
#define MM_MORPH_P2PAIR 1  // pass 2 as one paired call (7% faster than two single chains)
#endif
#ifndef MM_MORPH_MINB
#define MM_MORPH_MINB 1
#endif
template <typename T, int G>
__global__ void __launch_bounds__(32 * kMorphWarps, MM_MORPH_MINB) k_morph_fused(MorphArgs a) {
  using Geo = MorphGeo<T>;
  constexpr int E = Geo::E;
  constexpr int SEG = Geo::SEG;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *base = smem_align1024(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char *wb = base + warp * a.warp_bytes;
  auto stg = [&](int i) { return wb + i * a.stage_bytes; };
  unsigned char *EB = wb + a.nstages * a.stage_bytes;  // erosion at positions j0-(w-1) .. j0+SEG
  unsigned char *DB = EB + a.ebuf_bytes;               // dilation, same positions
  const WarpAgg<T> agg(DB + a.ebuf_bytes);
  const int w = a.w;
  const int OFF = Geo::off(w);  // buffer index of position j0
  const int nwb = blockDim.x >> 5;
  const int64_t gw = blockIdx.x * (int64_t)nwb + warp, NW = (int64_t)gridDim.x * nwb;
  // a contiguous range of segments per warp: the erosion / dilation of the w-1
  // positions before a segment carry over from the one before it
  const int64_t s_begin = a.nseg * gw / NW, s_end = a.nseg * (gw + 1) / NW;
  if (s_begin >= s_end) return;
  auto seg_pos = [&](int64_t sg, int64_t &row, int64_t &j0) {  // nseg < 2^31 (launcher)
    const uint32_t r = (uint32_t)sg / (uint32_t)a.segs_per_row;
    row = r;
    j0 = ((int64_t)sg - (int64_t)r * a.segs_per_row) * SEG;
  };
  int64_t s_first;
  {  // warm-up: the segments whose pass 1 feeds the first segment's carried positions
    int64_t row, j0;
    seg_pos(s_begin, row, j0);
    const int64_t wu = (w - 1 + SEG - 1) / SEG, in_row = j0 / SEG;
    s_first = s_begin - (wu < in_row ? wu : in_row);
  }
  const int ns = a.nstages;
  for (int k = 0; k + 1 < ns; ++k) {
    const int64_t sg = s_first + k;
    if (sg < s_end) {
      int64_t row, j0;
      seg_pos(sg, row, j0);
      morph_stage<T>(a, stg(k), row, j0, lane);
    }
    cp_async_commit();
  }
  int slot = 0;
  for (int64_t sg = s_first; sg < s_end; ++sg) {
    {
      const int64_t nx = sg + ns - 1;
      if (nx < s_end) {
        int64_t row, j0;
        seg_pos(nx, row, j0);
        morph_stage<T>(a, stg(slot + ns - 1 < ns ? slot + ns - 1 : slot - 1), row, j0, lane);
      }
    }
    cp_async_commit();
    cp_async_wait_ring(ns);
    __syncwarp();
    const unsigned char *X = stg(slot);
    slot = slot + 1 < ns ? slot + 1 : 0;
    int64_t row, j0;
    seg_pos(sg, row, j0);
    if (j0 == 0) {  // positions before the row: the identities of pass 2
      for (int t = lane; t < w - 1; t += 32) {
        sts_swz<T>(EB, OFF - (w - 1) + t, lowest_value<T>());
        sts_swz<T>(DB, OFF - (w - 1) + t, highest_value<T>());
      }
    }
    // ---- pass 1: d (max) and e (min) at positions j0 + [0, SEG)
    {
      T ox[E], on[E];
      morph_window<T, E, G>(X, 0, a.g, agg, lane, ox, on);
      const int64_t j = j0 + lane * E;
#pragma unroll
      for (int k = 0; k < E; ++k) {
        if (j + k >= a.m) {
          ox[k] = highest_value<T>();
          on[k] = lowest_value<T>();
        }
      }
      sts_swz_chunk<T, E>(DB, OFF + lane * E, ox);
      sts_swz_chunk<T, E>(EB, OFF + lane * E, on);
    }
    __syncwarp();
    // ---- pass 2: opening = max over e, closing = min over d (outputs j0 + [0, SEG))
    if (sg >= s_begin) {
      T op[E], cl[E];
      if constexpr (G == 0) {
        warp_window_small1<T, E, true>(EB, OFF - (w - 1), w, lane, op);
        warp_window_small1<T, E, false>(DB, OFF - (w - 1), w, lane, cl);
      } else {
#if MM_MORPH_P2PAIR
        warp_window_med<T, E, G>(TwoLoader<T>{EB, DB}, OFF - (w - 1), a.g, agg, lane, op, cl);
#else
        warp_window_med1<T, E, G, true>(EB, OFF - (w - 1), a.g, agg, lane, op);
        warp_window_med1<T, E, G, false>(DB, OFF - (w - 1), a.g, agg, lane, cl);
#endif
      }
      const int64_t i0 = j0 + lane * E;
      const int64_t left = a.n - i0;
      if (left > 0) {
        T *oo = a.out_open ? static_cast<T *>(a.out_open) + row * a.out_ld + i0 : nullptr;
        T *oc = a.out_close ? static_cast<T *>(a.out_close) + row * a.out_ld + i0 : nullptr;
        if (left >= E) {
          if (oo) store_chunk<T, E>(oo, op);
          if (oc) store_chunk<T, E>(oc, cl);
        } else {
#pragma unroll
          for (int k = 0; k < E; ++k)
            if (k < left) {
              if (oo) oo[k] = op[k];
              if (oc) oc[k] = cl[k];
            }
        }
      }
    }
    // ---- carry: the last w-1 positions move in front of the next segment's
    if (sg + 1 < s_end && j0 + SEG < a.n) {
      for (int t0 = 0; t0 < w - 1; t0 += 32) {  // ascending steps: load all, then store
        const int t = t0 + lane;
        T ve = T(0), vd = T(0);
        if (t < w - 1) {
          ve = lds_one_swz<T>(EB, OFF + SEG - (w - 1) + t);
          vd = lds_one_swz<T>(DB, OFF + SEG - (w - 1) + t);
        }
        __syncwarp();
        if (t < w - 1) {
          sts_swz<T>(EB, OFF - (w - 1) + t, ve);
          sts_swz<T>(DB, OFF - (w - 1) + t, vd);
        }
      }
    }
    __syncwarp();  // the buffers are rewritten by the next segment
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

template <typename T, int G>
int launch_morph_g(MorphArgs a, cudaStream_t s) {
  using Geo = MorphGeo<T>;
  // instruction-latency bound: resident warps first, then segments in flight
  WarpLaunch L;
  int rc = warp_launch_choice(reinterpret_cast<const void *>(k_morph_fused<T, G>), a.w, kMorphWarps, 1,
                              [](int w, int ns, int nw) { return Geo::cta_bytes(w, ns, nw); }, 1, &L);
  if (rc) return rc;
  a.nstages = L.ns;
  a.warp_bytes = Geo::warp_bytes(a.w, L.ns);
  const int64_t want = (a.nseg + L.nw - 1) / L.nw;
  const int64_t cap = (int64_t)sm_count() * L.per_sm;
  k_morph_fused<T, G><<<(int)(want < cap ? want : cap), 32 * L.nw, L.smem, s>>>(a);
  return note_cuda(cudaGetLastError());
}

template <typename T>
int launch_morph(const void *in, int64_t batch, int64_t n, int64_t in_ld, int64_t w, void *out_open,
                 void *out_close, int64_t out_ld, cudaStream_t s) {
  using Geo = MorphGeo<T>;
  if (batch == 0) return kOK;
  if (w - 1 > kMorphHMax) return kErrUnsupported;
  MorphArgs a;
  std::memset(&a, 0, sizeof(a));
  a.in = in;
  a.out_open = out_open;
  a.out_close = out_close;
  a.n = n;
  a.m = n - w + 1;
  a.in_ld = in_ld;
  a.out_ld = out_ld;
  a.batch = batch;
  a.segs_per_row = (n + Geo::SEG - 1) / Geo::SEG;
  a.nseg = batch * a.segs_per_row;
  if (a.nseg > 0x7fffffffLL) return kErrUnsupported;
  a.w = (int)w;
  a.in_vec = (reinterpret_cast<uintptr_t>(in) % 16 == 0 && (batch == 1 || (in_ld * (int64_t)sizeof(T)) % 16 == 0))
                 ? 1 : 0;
  a.stage_bytes = Geo::stage_bytes((int)w);
  a.ebuf_bytes = Geo::ebuf_bytes((int)w);
  if (w - 1 < Geo::E) {
    a.g.w = (int)w;
    return launch_morph_g<T, 0>(a, s);
  }
  const int G = warp_group<Geo::E>(w);
  a.g = make_warp_geom<Geo::E>((int)w, G);
  if (a.g.V + 32 / G > WarpAgg<T>::AGG) return kErrUnsupported;
  switch (G) {
    case 1: return launch_morph_g<T, 1>(a, s);
    case 2: return launch_morph_g<T, 2>(a, s);
    case 4: return launch_morph_g<T, 4>(a, s);
    case 8: return launch_morph_g<T, 8>(a, s);
    case 16: return launch_morph_g<T, 16>(a, s);
    default: return launch_morph_g<T, 32>(a, s);
  }
}

// ------------------------------------------------------------------- 2-D
// The identity frames of the two padded buffers: every element outside rows
// [r0, r1) x columns [c0, c1).  One warp per (image, padded row): whole rows
// above and below the interior, the left and right margins beside it.
template <typename T>
__global__ void k_morph_frame(T *pe, T *pd, int64_t batch, int64_t PR, int64_t PC, int64_t ld, int64_t bs,
                              int64_t r0, int64_t r1, int64_t c0, int64_t c1) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const T lo = lowest_value<T>(), hi = highest_value<T>();
  for (int64_t it = warp; it < batch * PR; it += nw) {
    const int64_t b = it / PR, r = it - b * PR;
    T *er = pe + b * bs + r * ld;
    T *dr = pd + b * bs + r * ld;
    if (r < r0 || r >= r1) {
      for (int64_t c = lane; c < PC; c += 32) {
        er[c] = lo;
        dr[c] = hi;
      }
    } else {
      for (int64_t c = lane; c < c0; c += 32) {
        er[c] = lo;
        dr[c] = hi;
      }
      for (int64_t c = c1 + lane; c < PC; c += 32) {
        er[c] = lo;
        dr[c] = hi;
      }
    }
  }
}

// dst[b][r][c] = src[b][r][c] for an R x C block of bytes, twice (the erosion
// and the dilation): source rows 16-B aligned, destination rows misaligned by
// the same D bytes (the interior of a padded frame).  One warp per (image, row)
// walks the row in 512-B steps; lane l writes destination 16-B unit u, whose
// bytes are source bytes [16u-D, 16u-D+16): the tail of source unit u-1 (the
// previous lane's, via a shuffle) and the head of unit u, joined with funnel
// shifts.  The first and last units of a row are partial: byte stores.
__device__ __forceinline__ void place_row(const uint8_t *__restrict__ sr, uint8_t *dr, int64_t C, int D, int lane) {
  uint8_t *A = dr - D;  // 16-B aligned
  const int64_t nu = (D + C + 15) / 16;
  const int P = 16 - D;  // start of the wanted bytes in [unit u-1 | unit u]
  const int wi = P >> 2, sh = (P & 3) * 8;
  uint4 carry = make_uint4(0, 0, 0, 0);
  for (int64_t ub = 0; ub < nu; ub += 32) {
    const int64_t u = ub + lane;
    uint4 cur = make_uint4(0, 0, 0, 0);
    if (u * 16 < C) cur = *reinterpret_cast<const uint4 *>(sr + u * 16);
    uint4 prev;
    prev.x = __shfl_up_sync(0xffffffffu, cur.x, 1);
    prev.y = __shfl_up_sync(0xffffffffu, cur.y, 1);
    prev.z = __shfl_up_sync(0xffffffffu, cur.z, 1);
    prev.w = __shfl_up_sync(0xffffffffu, cur.w, 1);
    if (lane == 0) prev = carry;
    carry.x = __shfl_sync(0xffffffffu, cur.x, 31);
    carry.y = __shfl_sync(0xffffffffu, cur.y, 31);
    carry.z = __shfl_sync(0xffffffffu, cur.z, 31);
    carry.w = __shfl_sync(0xffffffffu, cur.w, 31);
    if (u >= nu) continue;
    const uint32_t W[9] = {prev.x, prev.y, prev.z, prev.w, cur.x, cur.y, cur.z, cur.w, 0u};
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t lo = 0, hi = 0;
#pragma unroll
      for (int q = 0; q < 5; ++q)  // W[wi + k], W[wi + k + 1] with a uniform wi in [0, 4]
        if (q == wi) {
          lo = W[q + k];
          hi = W[q + k + 1];
        }
      o[k] = __funnelshift_r(lo, hi, sh);
    }
    const int64_t t0 = u * 16;  // destination bytes [t0, t0+16) relative to A; valid [D, D+C)
    if (t0 >= D && t0 + 16 <= D + C) {
      *reinterpret_cast<uint4 *>(A + t0) = make_uint4(o[0], o[1], o[2], o[3]);
    } else {
      const uint8_t *ob = reinterpret_cast<const uint8_t *>(o);
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (t0 + k >= D && t0 + k < D + C) A[t0 + k] = ob[k];
    }
  }
}

__global__ void k_morph_place_u8(const uint8_t *__restrict__ se, const uint8_t *__restrict__ sd, int64_t sld,
                                 int64_t sbs, uint8_t *de, uint8_t *dd, int64_t dld, int64_t dbs, int64_t batch,
                                 int64_t R, int64_t C, int D) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t it = warp; it < 2 * batch * R; it += nw) {
    const int which = it >= batch * R ? 1 : 0;
    const int64_t k = it - which * batch * R;
    const int64_t b = k / R, r = k - b * R;
    place_row((which ? sd : se) + b * sbs + r * sld, (which ? dd : de) + b * dbs + r * dld, C, D, lane);
  }
}

template <typename T>
struct Morph2DLayout {  // workspace: [padded e | padded d | (1-byte types) aligned e | aligned d]
  int64_t PR, PC, ld, bs;  // padded frames
  int64_t R, C, eld, ebs;  // aligned valid-region buffers
  size_t frame, valid, sep, total;
  Morph2DLayout(int64_t batch, int64_t rows, int64_t cols, int64_t w_row, int64_t w_col) {
    constexpr int VEC = 16 / (int)sizeof(T);
    auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
    PR = rows + w_col - 1;
    PC = cols + w_row - 1;
    ld = (PC + VEC - 1) / VEC * VEC;
    bs = PR * ld;
    frame = up((size_t)batch * bs * sizeof(T));
    R = rows - w_col + 1;
    C = cols - w_row + 1;
    eld = (C + VEC - 1) / VEC * VEC;
    ebs = R * eld;
    valid = sizeof(T) == 1 ? up((size_t)batch * ebs) : 0;
    // the separable 2-D path's row images (the larger of the two passes' needs)
    const size_t s1 = sep2d_workspace<T>(batch, rows, cols, w_row, w_col);
    const size_t s2 = sep2d_workspace<T>(batch, PR, PC, w_row, w_col);
    sep = up(s1 > s2 ? s1 : s2);
    total = 2 * frame + 2 * valid + sep;
  }
};

template <typename T>
size_t morph_2d_workspace(int64_t batch, int64_t rows, int64_t cols, int64_t w_row, int64_t w_col) {
  return Morph2DLayout<T>(batch, rows, cols, w_row, w_col).total;
}

template <typename T>
int launch_morph_2d(const void *in, int64_t batch, int64_t rows, int64_t cols, int64_t in_ld, int64_t in_bstride,
                    int64_t w_row, int64_t w_col, void *out_open, void *out_close, int64_t out_ld,
                    int64_t out_bstride, void *ws, cudaStream_t s) {
  if (batch == 0) return kOK;
  const Morph2DLayout<T> L(batch, rows, cols, w_row, w_col);
  char *base = static_cast<char *>(ws);
  if constexpr (sizeof(T) == 1) {  // square windows of the packed kernel: three passes, no frames
    if (w_row == w_col) {
      const int rc = launch_morph_2d_byte(std::is_signed<T>::value, in, batch, rows, cols, in_ld, in_bstride, w_row,
                                          out_open, out_close, out_ld, out_bstride, base + 2 * L.frame,
                                          base + 2 * L.frame + L.valid, L.eld, s);
      if (rc != kErrUnsupported) return rc;
    }
  }
  T *pe = reinterpret_cast<T *>(base);
  T *pd = reinterpret_cast<T *>(base + L.frame);
  {
    const int64_t items = batch * L.PR;
    const int64_t blocks = std::min<int64_t>((items + 7) / 8, (int64_t)sm_count() * 8);
    k_morph_frame<T><<<(int)(blocks > 0 ? blocks : 1), 256, 0, s>>>(pe, pd, batch, L.PR, L.PC, L.ld, L.bs, w_col - 1,
                                                                     w_col - 1 + L.R, w_row - 1, w_row - 1 + L.C);
    int rc = note_cuda(cudaGetLastError());
    if (rc) return rc;
  }
  const int64_t off = (w_col - 1) * L.ld + (w_row - 1);
  void *sepws = base + 2 * L.frame + 2 * L.valid;
  int rc;
  if (sizeof(T) == 1) {
    // the packed byte kernel writes 4-B aligned rows only: e and d go to aligned
    // buffers first, then into the frames' (unaligned) interiors
    T *ve = reinterpret_cast<T *>(base + 2 * L.frame);
    T *vd = reinterpret_cast<T *>(base + 2 * L.frame + L.valid);
    rc = launch_2d_best<T>(in, batch, rows, cols, in_ld, in_bstride, w_row, w_col, vd, ve, L.eld, L.ebs, sepws, L.sep,
                           s);
    if (rc) return rc;
    const int64_t items = 2 * batch * L.R;
    const int64_t blocks = std::min<int64_t>((items + 7) / 8, (int64_t)sm_count() * 16);
    const int D = (int)(reinterpret_cast<uintptr_t>(pe + off) & 15);  // same for every row (ld % 16 == 0)
    k_morph_place_u8<<<(int)(blocks > 0 ? blocks : 1), 256, 0, s>>>(
        reinterpret_cast<const uint8_t *>(ve), reinterpret_cast<const uint8_t *>(vd), L.eld, L.ebs,
        reinterpret_cast<uint8_t *>(pe + off), reinterpret_cast<uint8_t *>(pd + off), L.ld, L.bs, batch, L.R, L.C, D);
    rc = note_cuda(cudaGetLastError());
  } else {  // the separable and the generic 2-D paths store at any element alignment
    rc = launch_2d_best<T>(in, batch, rows, cols, in_ld, in_bstride, w_row, w_col, pd + off, pe + off, L.ld, L.bs,
                           sepws, L.sep, s);
  }
  if (rc) return rc;
  if (out_open) {
    rc = launch_2d_best<T>(pe, batch, L.PR, L.PC, L.ld, L.bs, w_row, w_col, out_open, nullptr, out_ld, out_bstride,
                           sepws, L.sep, s);
    if (rc) return rc;
  }
  if (out_close)
    rc = launch_2d_best<T>(pd, batch, L.PR, L.PC, L.ld, L.bs, w_row, w_col, nullptr, out_close, out_ld, out_bstride,
                           sepws, L.sep, s);
  return rc;
}

#define MM_MORPH_INST(T)                                                                                      \
  template int launch_morph<T>(const void *, int64_t, int64_t, int64_t, int64_t, void *, void *, int64_t,    \
                               cudaStream_t);                                                                 \
  template size_t morph_2d_workspace<T>(int64_t, int64_t, int64_t, int64_t, int64_t);                        \
  template int launch_morph_2d<T>(const void *, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t,        \
                                  int64_t, void *, void *, int64_t, int64_t, void *, cudaStream_t);
MM_MORPH_INST(uint8_t)
MM_MORPH_INST(int8_t)
MM_MORPH_INST(uint16_t)
MM_MORPH_INST(int16_t)
MM_MORPH_INST(uint32_t)
MM_MORPH_INST(int32_t)
MM_MORPH_INST(uint64_t)
MM_MORPH_INST(int64_t)
MM_MORPH_INST(float)
MM_MORPH_INST(double)

}  // namespace mm

// stream.cu -- online multi-stream filter.
//
// The paper's setting is a stream: "the stream latency of a filter [is] the
// maximum number of data points required after the window has passed"
// (PAPER.md:68-72), and the monotonic wedge reaches latency 0 with O(w) state
// (Table 1).  On the GPU, thousands of independent streams
// ingest a chunk of c samples each per call, and every window that a chunk
// completes is emitted by that same call (reading R19): zero latency per
// push.  The state of a stream is its last w-1 samples (the wedge's value
// buffer; the extrema are rebuilt from them and the chunk on every push).
//
// Two paths, chosen by w when the state is created:
//
// fused (w-1 <= kStreamHMax; k_stream_fused): ONE kernel per push reads
//   each stream's history and its new chunk, writes the c windows and the new
//   history -- exactly the algorithmic bytes: c + 2c + 2(w-1) per stream.
//   History rows are kept right-aligned in ping-pong buffers of hld =
//   round_up(w-1, 16 B) elements, so the virtual row V' = [hist row | chunk]
//   is 16-B aligned in both parts; window k starts at V'[P + k], P = hld-(w-1).
//   Warps are autonomous: a warp owns a segment of 32E windows of one stream,
//   stages V'[j0, j0 + P + 32E + w - 1) into its own 128B-swizzled buffer with
//   cp.async (double-buffered: the next segment's copy is in flight while this
//   one computes) and runs the near/far block decomposition of k1d_medium
//   (k1d_medium.cuh) within the warp: block B = E*G <= w-1, gap aggregates of
//   the far blocks before the segment are reduced from the staged halo.  The
//   warp holding a stream's last window writes the new history.
//
// composed (w-1 > kStreamHMax): the state row is [history (w-1) | slot (max_chunk)];
//   a push copies the chunk into the slot, runs the batched filter (any 1-D
//   kernel) over [0, w-1+c) and moves the last w-1 samples to the front.
//   HBM bytes: 2c + (w-1+c) + 2c + 2(w-1) per stream.
#include "kwarp.cuh"
#include "launch.cuh"

namespace mm {

// dst[e] = src[e] for e in [d0, d1), one warp; dst is 16-B aligned at element
// 0 (stores are 16-B vectors where whole), src any element alignment.  Each
// 32-vector step loads everything before storing anything, and steps ascend,
// so an overlapping in-row move with src = dst + c (c > 0) is safe.
template <typename T>
__device__ __forceinline__ void warp_copy(T *dst, const T *src, int64_t d0, int64_t d1, int lane) {
  constexpr int VEC = 16 / sizeof(T);
  const int64_t v0 = d0 / VEC, v1 = (d1 + VEC - 1) / VEC;
  for (int64_t vb = v0; vb < v1; vb += 32) {
    const int64_t v = vb + lane;
    const int64_t e0 = v * VEC;
    const bool any = v < v1;
    const bool full = any && e0 >= d0 && e0 + VEC <= d1;
    T buf[VEC];
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
      const int64_t e = e0 + k;
      buf[k] = (any && e >= d0 && e < d1) ? src[e] : T(0);
    }
    __syncwarp();
    if (full) {
      uint4 u;
      memcpy(&u, buf, 16);
      *reinterpret_cast<uint4 *>(dst + e0) = u;
    } else if (any) {
#pragma unroll
      for (int k = 0; k < VEC; ++k) {
        const int64_t e = e0 + k;
        if (e >= d0 && e < d1) dst[e] = buf[k];
      }
    }
  }
}

// Row r: state[r*ld + e] = src[r*src_ld + e - src_shift] for e in [d0, d1).
// ordered: one warp per row walks the whole range in ascending steps (the
// in-row shift with overlap); else every row is cut into segments that warps
// copy independently.
template <typename T>
__global__ void __launch_bounds__(256) k_stream_copy(T *state, int64_t streams, int64_t ld, const T *src,
                                                     int64_t src_ld, int64_t src_shift, int64_t d0, int64_t d1,
                                                     int ordered) {
  constexpr int VEC = 16 / sizeof(T);
  constexpr int64_t SEG = 32 * VEC * 8;  // elements per independent segment (8 warp steps)
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // segments start at 16-B boundaries of the destination row
  const int64_t a0 = d0 / VEC * VEC;
  const int64_t nseg = ordered ? 1 : (d1 - a0 + SEG - 1) / SEG;
  const int64_t items = streams * nseg;
  for (int64_t it = warp; it < items; it += nwarps) {
    const int64_t r = it / nseg, sg = it - r * nseg;
    int64_t s0 = ordered ? d0 : a0 + sg * SEG, s1 = ordered ? d1 : s0 + SEG;
    if (s0 < d0) s0 = d0;
    if (s1 > d1) s1 = d1;
    T *drow = state + r * ld;
    const T *srow = src + r * src_ld - src_shift;
    warp_copy<T>(drow, srow, s0, s1, lane);
  }
}


// ============================================================ fused path
constexpr int kStreamHMax = 1024;  // largest w-1 of the fused kernel
constexpr int kStreamWarps = 4;    // warps per CTA (~136 registers: 3 CTAs per SM)

template <typename T, int E_ = Chunk<T>::E>
struct StreamGeo {
  static constexpr int E = E_;
  static constexpr int VEC = 16 / (int)sizeof(T);
  static constexpr int SEG = 32 * E;  // windows per warp segment
  // staged elements: P + SEG + w - 1, plus the 16-B over-reads of lds_swz
  __host__ __device__ static int stage_bytes(int w) {
    const int elems = VEC + SEG + w - 1 + E + 2 * VEC;
    const int bytes = elems * (int)sizeof(T);
    return (bytes + 1023) / 1024 * 1024;
  }
  __host__ __device__ static int warp_bytes(int w, int ns) { return ns * stage_bytes(w) + WarpAgg<T>::bytes(); }
  __host__ __device__ static size_t cta_bytes(int w, int ns) { return 1024 + (size_t)kStreamWarps * warp_bytes(w, ns); }
};

struct StreamArgs {
  const void *hist_in;  // [streams][hld]: the current history (right-aligned)
  void *hist_out;       // [streams][hld]: receives the new history
  const void *chunk;    // [streams][chunk_ld]: c new samples per stream
  void *out_max;
  void *out_min;
  int64_t hld, chunk_ld, c, out_ld, streams;
  int64_t segs_per_row, nseg;
  int w, P;            // window; pad of the history rows
  WarpGeom g;          // gap geometry of block B = E*G (kwarp.cuh)
  int chunk_vec;       // chunk rows are 16-B aligned (else staged element-wise)
  int stage_bytes, warp_bytes;
  int nstages;         // staging ring per warp: 2..4 (nstages-1 segments in flight)
};


// Stage V'[j0, j0 + len) of `row` into the swizzled buffer X (logical index
// i = V' index - j0).  j0 and hld are multiples of VEC, so every 16-B unit
// comes from one source.
template <typename T>
__device__ __forceinline__ void stream_stage(const StreamArgs &a, unsigned char *X, int64_t row, int64_t j0,
                                             int len, int lane) {
  constexpr int VEC = 16 / (int)sizeof(T);
  const T *hist = static_cast<const T *>(a.hist_in) + row * a.hld;
  const T *chk = static_cast<const T *>(a.chunk) + row * a.chunk_ld;
  const int nq = (len + VEC - 1) / VEC;
  for (int q = lane; q < nq; q += 32) {
    const int64_t v = j0 + (int64_t)q * VEC;
    unsigned char *dst = X + swz(q);
    if (v < a.hld) {
      cp_async16(dst, hist + v);
    } else if (a.chunk_vec && v - a.hld + VEC <= a.c) {
      cp_async16(dst, chk + (v - a.hld));
    } else {
      T t[VEC];
#pragma unroll
      for (int k = 0; k < VEC; ++k) {
        const int64_t u = v - a.hld + k;
        t[k] = u < a.c ? chk[u] : T(0);
      }
      uint4 u4;
      memcpy(&u4, t, 16);
      *reinterpret_cast<uint4 *>(dst) = u4;
    }
  }
}

template <typename T, int EE, int G>
__global__ void __launch_bounds__(32 * kStreamWarps) k_stream_fused(StreamArgs a) {
  using Geo = StreamGeo<T, EE>;
  constexpr int E = Geo::E;
  constexpr int SEG = Geo::SEG;
  constexpr int VEC = Geo::VEC;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *base = smem_align1024(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char *wb = base + warp * a.warp_bytes;
  auto stg = [&](int i) { return wb + i * a.stage_bytes; };
  const WarpAgg<T> agg(wb + a.nstages * a.stage_bytes);  // after the staging ring
  const int w = a.w, P = a.P;
  const int64_t gw = blockIdx.x * (int64_t)kStreamWarps + warp, nw = (int64_t)gridDim.x * kStreamWarps;

  auto seg_pos = [&](int64_t sg, int64_t &row, int64_t &j0) {
    if (a.segs_per_row == 1) {  // chunks of <= SEG samples: a segment is a stream
      row = sg;
      j0 = 0;
    } else {  // nseg < 2^31 (checked by the launcher): 32-bit division
      const uint32_t r = (uint32_t)sg / (uint32_t)a.segs_per_row;
      row = r;
      j0 = ((int64_t)sg - (int64_t)r * a.segs_per_row) * SEG;
    }
  };
  auto seg_len = [&](int64_t j0) {  // staged elements of a segment
    const int64_t want = (int64_t)P + SEG + w - 1;
    const int64_t have = a.hld + a.c - j0;
    return (int)(want < have ? want : have);
  };

  const int ns = a.nstages;
  for (int k = 0; k + 1 < ns; ++k) {  // prologue: the first ns-1 segments in flight
    const int64_t sg = gw + k * nw;
    if (sg < a.nseg) {
      int64_t row, j0;
      seg_pos(sg, row, j0);
      stream_stage<T>(a, stg(k), row, j0, seg_len(j0), lane);
    }
    cp_async_commit();
  }
  int slot = 0;
  for (int64_t sg = gw; sg < a.nseg; sg += nw) {
    {  // keep ns-1 segments in flight
      const int64_t nx = sg + (ns - 1) * nw;
      if (nx < a.nseg) {
        int64_t row, j0;
        seg_pos(nx, row, j0);
        const int sl = slot + ns - 1 < ns ? slot + ns - 1 : slot - 1;
        stream_stage<T>(a, stg(sl), row, j0, seg_len(j0), lane);
      }
    }
    cp_async_commit();
    cp_async_wait_ring(ns);
    __syncwarp();
    const unsigned char *X = stg(slot);
    slot = slot + 1 < ns ? slot + 1 : 0;
    int64_t row, j0;
    seg_pos(sg, row, j0);
    const int64_t left = a.c - j0;
    const int cnt = left < SEG ? (int)left : SEG;
    T ox[E], on[E];
    if constexpr (G == 0)  // w <= E: log-step doubling + barrel shift
      warp_window_small<T, E>(PairLoader<T>{X}, P, w, lane, ox, on);
    else
      warp_window_med<T, E, G>(PairLoader<T>{X}, P, a.g, agg, lane, ox, on);
    const int c0 = lane * E;
    if (c0 < cnt) {
      T *omx = a.out_max ? static_cast<T *>(a.out_max) + row * a.out_ld + j0 + c0 : nullptr;
      T *omn = a.out_min ? static_cast<T *>(a.out_min) + row * a.out_ld + j0 + c0 : nullptr;
      if (c0 + E <= cnt) {
        if (omx) store_chunk<T, E>(omx, ox);
        if (omn) store_chunk<T, E>(omn, on);
      } else {
#pragma unroll
        for (int k = 0; k < E; ++k)
          if (c0 + k < cnt) {
            if (omx) omx[k] = ox[k];
            if (omn) omn[k] = on[k];
          }
      }
    }
    // ---- the stream's last segment writes its new history: V'[c + t], t < hld
    if (left <= SEG) {
      T *ho = static_cast<T *>(a.hist_out) + row * a.hld;
      const int off = (int)(a.c - j0);
      for (int t = lane * VEC; t < a.hld; t += 32 * VEC) {
        T v[VEC];
        lds_swz<T, VEC>(X, off + t, v);
        uint4 u4;
        memcpy(&u4, v, 16);
        *reinterpret_cast<uint4 *>(ho + t) = u4;
      }
    }
    __syncwarp();  // X is restaged by the next iteration
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

namespace {
int copy_grid(int64_t items) {
  const int64_t blocks = (items + 7) / 8;  // 8 warps per block
  const int64_t cap = (int64_t)sm_count() * 8;
  return (int)(blocks < 1 ? 1 : (blocks < cap ? blocks : cap));
}
}  // namespace

template <typename T>
StreamLayout stream_layout(int64_t streams, int64_t w, int64_t max_chunk) {
  constexpr int VEC = 16 / (int)sizeof(T);
  auto up256 = [](size_t x) { return (x + 255) & ~size_t(255); };
  StreamLayout L;
  L.fused = (w - 1 <= kStreamHMax) ? 1 : 0;
  if (L.fused) {  // two history buffers (ping-pong), rows right-aligned
    L.ld = (w - 1 + VEC - 1) / VEC * VEC;
    L.hist_bytes = up256((size_t)streams * L.ld * sizeof(T));
    L.ws_bytes = 0;
    L.total = 2 * L.hist_bytes;
  } else {  // [history | slot] rows + the filter's workspace
    L.ld = (w - 1 + max_chunk + VEC - 1) / VEC * VEC;
    L.hist_bytes = up256((size_t)streams * L.ld * sizeof(T));
    L.ws_bytes = workspace_1d<T>(streams, w - 1 + max_chunk, w);
    L.total = L.hist_bytes + up256(L.ws_bytes);
  }
  return L;
}

template <typename T, int E, int G>
int launch_fused_g(StreamArgs a, cudaStream_t s) {
  using Geo = StreamGeo<T, E>;
  a.segs_per_row = (a.c + Geo::SEG - 1) / Geo::SEG;
  a.nseg = a.streams * a.segs_per_row;
  if (a.nseg > 0x7fffffffLL) return kErrUnsupported;
  if constexpr (G > 0) {
    a.g = make_warp_geom<E>(a.w, G);
    if (a.g.V + 32 / G > WarpAgg<T>::AGG) return kErrUnsupported;
  } else {
    a.g.w = a.w;
  }
  // staging depth: the most segments in flight per SM
  WarpLaunch L;
  int rc = warp_launch_choice(reinterpret_cast<const void *>(k_stream_fused<T, E, G>), a.w, kStreamWarps, kStreamWarps,
                              [](int w, int ns, int) { return Geo::cta_bytes(w, ns); }, 0, &L);
  if (rc) return rc;
  a.nstages = L.ns;
  a.stage_bytes = Geo::stage_bytes(a.w);
  a.warp_bytes = Geo::warp_bytes(a.w, L.ns);
  const int64_t want = (a.nseg + kStreamWarps - 1) / kStreamWarps;
  const int64_t cap = (int64_t)sm_count() * L.per_sm;
  k_stream_fused<T, E, G><<<(int)(want < cap ? want : cap), 32 * kStreamWarps, L.smem, s>>>(a);
  return note_cuda(cudaGetLastError());
}

template <typename T>
int launch_stream_push(void *state, const StreamLayout &L, int64_t streams, int64_t w, int phase, const T *chunk,
                       int64_t c, int64_t chunk_ld, T *out_max, T *out_min, int64_t out_ld, cudaStream_t s) {
  if (streams == 0 || c == 0) return kOK;
  constexpr int VEC = 16 / (int)sizeof(T);
  const int64_t h = w - 1;
  if (L.fused) {
    constexpr int EB = Chunk<T>::E;                     // long chunks
    constexpr int ES = EB / 2 >= VEC ? EB / 2 : EB;     // chunks of <= 32*ES samples: half the lanes' work
    char *base = static_cast<char *>(state);
    StreamArgs a;
    std::memset(&a, 0, sizeof(a));
    a.hist_in = base + (phase ? L.hist_bytes : 0);
    a.hist_out = base + (phase ? 0 : L.hist_bytes);
    a.chunk = chunk;
    a.out_max = out_max;
    a.out_min = out_min;
    a.hld = L.ld;
    a.chunk_ld = chunk_ld;
    a.c = c;
    a.out_ld = out_ld;
    a.streams = streams;
    a.w = (int)w;
    a.P = (int)(L.ld - h);
    a.chunk_vec = (reinterpret_cast<uintptr_t>(chunk) % 16 == 0 &&
                   (streams == 1 || (chunk_ld * (int64_t)sizeof(T)) % 16 == 0)) ? 1 : 0;
    if (h < EB) {  // w <= E: the small-window path
      if (ES < EB && c <= 32 * ES && h < ES) return launch_fused_g<T, ES, 0>(a, s);
      return launch_fused_g<T, EB, 0>(a, s);
    }
    const bool small_e = ES < EB && c <= 32 * ES && h >= ES;
    if (small_e) {
      switch (warp_group<ES>(w)) {
        case 1: return launch_fused_g<T, ES, 1>(a, s);
        case 2: return launch_fused_g<T, ES, 2>(a, s);
        case 4: return launch_fused_g<T, ES, 4>(a, s);
        case 8: return launch_fused_g<T, ES, 8>(a, s);
        case 16: return launch_fused_g<T, ES, 16>(a, s);
        default: return launch_fused_g<T, ES, 32>(a, s);
      }
    }
    switch (warp_group<EB>(w)) {
      case 1: return launch_fused_g<T, EB, 1>(a, s);
      case 2: return launch_fused_g<T, EB, 2>(a, s);
      case 4: return launch_fused_g<T, EB, 4>(a, s);
      case 8: return launch_fused_g<T, EB, 8>(a, s);
      case 16: return launch_fused_g<T, EB, 16>(a, s);
      default: return launch_fused_g<T, EB, 32>(a, s);
    }
  }
  T *rows = static_cast<T *>(state);
  const int64_t ld = L.ld;
  void *ws = L.ws_bytes ? static_cast<char *>(state) + L.hist_bytes : nullptr;
  {  // 1. ingest into the slot [h, h+c)
    const int64_t nseg = (h + c - h / VEC * VEC + 32 * VEC * 8 - 1) / (32 * VEC * 8);
    k_stream_copy<T><<<copy_grid(streams * nseg), 256, 0, s>>>(rows, streams, ld, chunk, chunk_ld, h, h, h + c, 0);
    int rc = note_cuda(cudaGetLastError());
    if (rc) return rc;
  }
  // 2. the filter: rows of n = h + c samples, c windows each
  int rc = launch_1d<T>(rows, streams, h + c, ld, w, out_max, out_min, out_ld, ws, L.ws_bytes, s);
  if (rc) return rc;
  if (h > 0) {  // 3. shift: [c, c+h) -> [0, h)
    const bool ordered = c < h;
    const int64_t items = ordered ? streams : streams * ((h + 32 * VEC * 8 - 1) / (32 * VEC * 8));
    k_stream_copy<T><<<copy_grid(items), 256, 0, s>>>(rows, streams, ld, rows, ld, -c, 0, h, ordered ? 1 : 0);
    rc = note_cuda(cudaGetLastError());
  }
  return rc;
}

#define MM_STREAM_INST(T)                                                                                      \
  template StreamLayout stream_layout<T>(int64_t, int64_t, int64_t);                                           \
  template int launch_stream_push<T>(void *, const StreamLayout &, int64_t, int64_t, int, const T *, int64_t,  \
                                     int64_t, T *, T *, int64_t, cudaStream_t);
MM_STREAM_INST(uint8_t)
MM_STREAM_INST(int8_t)
MM_STREAM_INST(uint16_t)
MM_STREAM_INST(int16_t)
MM_STREAM_INST(uint32_t)
MM_STREAM_INST(int32_t)
MM_STREAM_INST(uint64_t)
MM_STREAM_INST(int64_t)
MM_STREAM_INST(float)
MM_STREAM_INST(double)

}  // namespace mm

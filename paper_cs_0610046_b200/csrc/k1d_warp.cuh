// k1d_warp.cuh -- warp-autonomous single-pass 1-D kernel with look-back, for
// w-1 >= WT and element types of <= 4 bytes.
//
// Same decomposition as k1d_large (see k1d_base.cuh), at warp granularity and
// without a CTA-wide barrier in the steady state:
//   warp-tile x owns outputs [u0, u0+WT), u0 = x*WT, WT = 32*E (512 floats);
//   near N_x = [u0, u0+WT)           -> S(i) = max a[u0+i .. u0+WT)
//   far  F_x = [u0+w-1, u0+w-1+WT)   -> P(i) = max a[u0+w-1 .. u0+w-1+i]
//   out[u0+i] = max(S(i), M_x, P(i)),  M_x = max a[u0+WT .. u0+w-1).
// With w-1 = q*WT + r the gap M_x is the last r elements of F_{x-q} (H_{x-q})
// and the whole F_{x-q+1} .. F_{x-1}.  Every tile publishes G_x = max F_x and
// H_x (max of its last r elements) as soon as its far chunk lands; the last
// tile of every group of K=8 also publishes the group's max of the 8 G's, so a
// gap is at most 2(K-1) tile words + ceil(q/K) group words + one H word: a
// handful of words per lane even at w = 262144.  Tiles x in [-q, -1] exist
// only to publish (their far chunks lie inside the row).
//
// Scheduling.  Tiles come in groups of K=8 consecutive tiles of one row; the
// rows' group sequences are concatenated and cut into one contiguous range per
// CTA, whose 8 warps take one tile of each group.  A gap only reaches back q
// tiles, so everything a range needs lies inside it, except the tiles just
// before its start: a short prologue publishes those (the CTA that owns them
// publishes the same words again -- identical values, so the race is benign).
// Hence no CTA ever waits on another one: no tickets, no atomics, and no
// residency assumption.  Each warp pipelines its jobs: in job i it loads the
// far chunk of job i+2 and the near chunk of job i+1, publishes job i+1 (whose
// far chunk has landed), then processes job i, which waits only on words
// published by the CTA's warps in earlier jobs.  Each warp has its own
// mbarriers, so an SM's 16 warps overlap each other's latencies.
//
// Slots are 64-bit words (1 << 32 | value bits), written and polled with
// relaxed gpu-scope accesses (value and flag in one single-copy-atomic store).
#pragma once

#include "k1d_large.cuh"

#ifndef MM_WARP_CONTIG  // 1: one contiguous group range per CTA (round 1); 0: round-robin groups
#define MM_WARP_CONTIG 0
#endif

namespace mm {

template <typename T>
struct WarpGeo {
  static_assert(sizeof(T) <= 4, "packed 64-bit slots hold <= 4-byte values");
#ifndef MM_WARP_E
#define MM_WARP_E 16
#endif
  static constexpr int E = sizeof(T) == 4 ? MM_WARP_E : Chunk<T>::E;  // elements per lane
  static constexpr int WT = 32 * E;          // outputs per warp-tile
  static constexpr int K = NWARP;            // warp-tiles per ticket (one per warp)
  static constexpr int RW = Rowing<T>::RW;   // elements per 128-B row
  static constexpr int VEC = 16 / (int)sizeof(T);
  static constexpr int NROWS = WT / RW;      // near chunk: 128-B rows
  static constexpr int FROWS = NROWS + 1;    // far chunk (unaligned start)
  static constexpr int NEAR = (NROWS * 128 + 1023) / 1024 * 1024;  // swizzled: 1024-B aligned
  static constexpr int FAR = (FROWS * 128 + 1023) / 1024 * 1024;
  static constexpr int NFAR = 3;             // far chunks: published one job ahead
  static constexpr int NNEAR = 2;
  static constexpr int WARP_SMEM = NFAR * FAR + NNEAR * NEAR;
  static constexpr int NBAR = NFAR + NNEAR;  // mbarriers per warp
  static constexpr size_t BYTES = 1024 + (size_t)NWARP * WARP_SMEM + 1024;
};

struct WarpLB {
  int q, r;           // w-1 = q*WT + r, q >= 1
  int64_t tpr;        // output warp-tiles per row
  int64_t xr;         // q + tpr: warp-tiles per row including publish-only ones
  int64_t kt;         // groups per row = ceil(xr / K)
  int64_t total;      // batch * kt
  int pg;             // groups a range start reaches back: ceil(q / K) + 1
};

template <typename T>
struct WarpWs {  // [256 B][tile slots: batch*xr x 4 words][group slots: total x 2 words]
  __host__ __device__ static size_t tiles_offset() { return 256; }
  __host__ __device__ static size_t groups_offset(const WarpLB &g, int64_t batch) {
    return 256 + (size_t)batch * g.xr * 4 * 8;
  }
  __host__ __device__ static size_t bytes(const WarpLB &g, int64_t batch) {
    return groups_offset(g, batch) + (size_t)g.total * 2 * 8 + 64;
  }
};

// Spin until a published slot's flag is set (a lost publish must trap, not hang).
__device__ __forceinline__ uint64_t wait_slot(const uint64_t *s) {
  uint64_t v = ld_relaxed_u64(s);
  uint32_t spins = 0;
  while ((v >> 32) == 0) {
    __nanosleep(20);
    v = ld_relaxed_u64(s);
    if (++spins > (1u << 26)) __trap();
  }
  return v;
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// E elements at logical position pos = sh + lane*E of a swizzled buffer, with
// the in-vector shift sh % VEC a compile-time constant (SH >= 0) or runtime
template <typename T, int E, int SH>
__device__ __forceinline__ void lds_far(const unsigned char *buf, int pos, T (&v)[E]) {
  constexpr int VEC = 16 / (int)sizeof(T);
  if constexpr (SH < 0) {
    lds_swz<T, E>(buf, pos, v);
  } else if constexpr (SH == 0) {
    lds_swz_aligned<T, E>(buf, pos, v);
  } else {
    constexpr int NQ = E / VEC + 1;
    const int c0 = pos / VEC;
    union {
      T t[NQ * VEC];
      uint4 q[NQ];
    } u;
#pragma unroll
    for (int k = 0; k < NQ; ++k) u.q[k] = *reinterpret_cast<const uint4 *>(buf + swz(c0 + k));
#pragma unroll
    for (int k = 0; k < E; ++k) v[k] = u.t[k + SH];
  }
}

template <typename T, int SH>
#ifndef MM_WARP_MINB
#define MM_WARP_MINB 2
#endif
__global__ void __launch_bounds__(NT, MM_WARP_MINB)
    k1d_warp(Rows p, WarpLB g, void *ws, const __grid_constant__ TmaMaps maps) {
  using Geo = WarpGeo<T>;
  constexpr int E = Geo::E, WT = Geo::WT, K = Geo::K, RW = Geo::RW;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *base = smem_align1024(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char *wbuf = base + (size_t)warp * Geo::WARP_SMEM;
  unsigned char *tail = base + (size_t)NWARP * Geo::WARP_SMEM;
  uint64_t *fbar = reinterpret_cast<uint64_t *>(tail) + warp * Geo::NBAR;  // far stages
  uint64_t *nbar = fbar + Geo::NFAR;                                       // near stages
  auto farb = [&](int s) { return wbuf + s * Geo::FAR; };
  auto nearb = [&](int s) { return wbuf + Geo::NFAR * Geo::FAR + s * Geo::NEAR; };

  uint64_t *tslot = reinterpret_cast<uint64_t *>(static_cast<char *>(ws) + WarpWs<T>::tiles_offset());
  uint64_t *kslot =
      reinterpret_cast<uint64_t *>(static_cast<char *>(ws) + WarpWs<T>::groups_offset(g, p.batch));
  const int64_t w = p.w;
  const int64_t full_el = (p.n / RW) * RW;  // elements covered by the tensor maps
  const int fsh = (int)((w - 1) % RW);      // far chunk offset inside its first 128-B row
  const int hstart = WT - g.r;              // H range of a far chunk: [hstart, WT)
  const int h_lane = hstart / E, h_off = hstart % E;

#if MM_WARP_CONTIG
  // this CTA's groups [gbeg, gend), and the prologue groups [pbeg, gbeg) of
  // the same row that its first gaps reach into
  const int64_t gbeg = g.total * (int64_t)blockIdx.x / gridDim.x;
  const int64_t gend = g.total * ((int64_t)blockIdx.x + 1) / gridDim.x;
  if (gbeg >= gend) return;
  const int64_t row0 = gbeg / g.kt;
  const int64_t pbeg = gbeg - row0 * g.kt >= g.pg ? gbeg - g.pg : row0 * g.kt;
  constexpr int64_t gstep = 1;
#else
  // groups dealt round-robin: CTA b takes b, b + grid, b + 2 grid, ...  The
  // whole grid sweeps the rows as one front, so the near chunk of tile x is
  // read shortly after the far chunk of tile x-q loaded the same bytes (an L2
  // hit), and every group -- the publish-only ones at row starts included --
  // has an owner: no prologue.  Gaps reach into groups of other CTAs; the
  // launch is cooperative (every CTA resident), and a CTA only ever waits on
  // groups below the one it processes, so the lowest unpublished group's owner
  // can always proceed.
  const int64_t gbeg = blockIdx.x, gend = g.total, pbeg = gbeg;
  if (gbeg >= gend) return;
  const int64_t gstep = gridDim.x;
  const int64_t step_rows = gstep / g.kt, step_x = (gstep - step_rows * g.kt) * K;
#endif

  if (threadIdx.x == 0) {
    for (int i = 0; i < NWARP * Geo::NBAR; ++i) mbar_init(reinterpret_cast<uint64_t *>(tail) + i, 1);
    fence_mbar_init();
    prefetch_tmap(&maps.big);
    prefetch_tmap(&maps.small);
  }
  __syncthreads();  // the only CTA-wide barrier

  // a job: group tk of the range, i.e. tile x of row `row` for this warp;
  // advanced incrementally (no divisions per job)
  struct Pos {
    int64_t tk, row;
    int x;
  };
  const int xend = -g.q + (int)g.kt * K;  // first x past a row's last group
  auto pos_at = [&](int64_t tk) {
    Pos q_;
    q_.tk = tk;
    q_.row = tk / g.kt;
    q_.x = -g.q + (int)(tk - q_.row * g.kt) * K + warp;
    return q_;
  };
#if MM_WARP_CONTIG
  auto advance = [&](Pos &q_) {
    ++q_.tk;
    q_.x += K;
    if (q_.x >= xend + warp) {
      ++q_.row;
      q_.x = -g.q + warp;
    }
  };
#else
  auto advance = [&](Pos &q_) {
    q_.tk += gstep;
    q_.row += step_rows;
    q_.x += (int)step_x;
    if (q_.x >= xend + warp) {
      ++q_.row;
      q_.x -= (int)g.kt * K;
    }
  };
#endif
  auto exists = [&](const Pos &q_) { return q_.tk < gend && q_.x < g.tpr; };
  // lane 0: TMA loads of a job's far chunk / near chunk (an absent tile arms
  // the barrier with nothing in flight)
  auto load_far = [&](const Pos &j, int s) {
    if (!exists(j)) {
      mbar_arrive_expect_tx(&fbar[s], 0);
      return;
    }
    mbar_arrive_expect_tx(&fbar[s], Geo::FROWS * 128);
    tma_box(&maps.small, farb(s), (int)(((int64_t)j.x * WT + w - 1) / RW), (int)j.row, &fbar[s]);
  };
  auto load_near = [&](const Pos &j, int s) {
    if (j.tk < gbeg || !exists(j) || j.x < 0) {
      mbar_arrive_expect_tx(&nbar[s], 0);
      return;
    }
    mbar_arrive_expect_tx(&nbar[s], Geo::NROWS * 128);
    tma_box(&maps.big, nearb(s), j.x * (WT / RW), (int)j.row, &nbar[s]);
  };
  // elements at or past full_el are not in the maps: plain loads
  auto patch = [&](unsigned char *buf, int64_t row, int64_t start, int64_t len) {
    const int64_t a0 = start > full_el ? start : full_el;
    const int64_t a1 = p.n < start + len ? p.n : start + len;
    const T *srs = series_ptr<T>(p, row);
    for (int64_t i = a0 + lane; i < a1; i += 32) sts_swz<T>(buf, (int)(i - start), srs[i]);
  };

  // ------------------------------------------------------------ publish
  // G_x, H_x of the job's tile (and, for the last warp, the group word)
  auto publish = [&](const Pos &j, int fs) {
    if (!exists(j)) return;
    const int64_t row = j.row;
    const int x = j.x;
    if (full_el < p.n) {
      patch(farb(fs), row, (int64_t)x * WT + w - 1 - fsh, Geo::FROWS * RW);
      __syncwarp();
    }
    T y[E];
    lds_far<T, E, SH>(farb(fs), fsh + lane * E, y);
    T gx = y[0], gn = y[0];
#pragma unroll
    for (int k = 1; k < E; ++k) {
      gx = Ord<T>::mx(gx, y[k]);
      gn = Ord<T>::mn(gn, y[k]);
    }
    // H: lanes past h_lane whole, lane h_lane from h_off (a uniform offset),
    // the rest borrow the chunk's last element (inside every non-empty H)
    T hx = __shfl_sync(0xffffffffu, y[E - 1], 31), hn = hx;
    T vx, vn;
    suffix_from<T, E>(y, h_off, vx, vn);
    if (lane > h_lane) {
      hx = Ord<T>::mx(hx, gx);
      hn = Ord<T>::mn(hn, gn);
    } else if (lane == h_lane) {
      hx = Ord<T>::mx(hx, vx);
      hn = Ord<T>::mn(hn, vn);
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
      gx = Ord<T>::mx(gx, __shfl_xor_sync(0xffffffffu, gx, d));
      gn = Ord<T>::mn(gn, __shfl_xor_sync(0xffffffffu, gn, d));
      hx = Ord<T>::mx(hx, __shfl_xor_sync(0xffffffffu, hx, d));
      hn = Ord<T>::mn(hn, __shfl_xor_sync(0xffffffffu, hn, d));
    }
    const int64_t si = (row * g.xr + x + g.q) * 4;  // this tile's slots
    if (lane < 4) {
      const T v = lane == 0 ? gx : lane == 1 ? gn : lane == 2 ? hx : hn;
      st_relaxed_u64(tslot + si + lane, pack_slot<T>(v));
    }
    if (warp == K - 1) {  // last tile of its group (complete, since it exists)
      const int kt_in_row = (x + g.q) / K;
      T zx = gx, zn = gn;
      if (lane < 2 * (K - 1)) {
        const uint64_t *sp = tslot + (si - 4 * (K - 1)) + 4 * (lane >> 1) + (lane & 1);
        const T v = unpack_slot<T>(wait_slot(sp));
        if (lane & 1)
          zn = Ord<T>::mn(zn, v);
        else
          zx = Ord<T>::mx(zx, v);
      }
#pragma unroll
      for (int d = 16; d >= 1; d >>= 1) {
        zx = Ord<T>::mx(zx, __shfl_xor_sync(0xffffffffu, zx, d));
        zn = Ord<T>::mn(zn, __shfl_xor_sync(0xffffffffu, zn, d));
      }
      if (lane < 2) st_relaxed_u64(kslot + (row * g.kt + kt_in_row) * 2 + lane, pack_slot<T>(lane ? zn : zx));
    }
  };

  // ------------------------------------------------------------ process
  auto process = [&](const Pos &j, int fs, int ns) {
    if (j.tk < gbeg || !exists(j) || j.x < 0) return;  // prologue: publish only
    const int64_t row = j.row;
    const int x = j.x;
    const int64_t u0 = (int64_t)x * WT;
    if (full_el < p.n) {  // (the far chunk was patched when it was published)
      patch(nearb(ns), row, u0, WT);
      __syncwarp();
    }
    // gap words first (their latency overlaps the scans): H_{x-q}, then G over
    // tiles [x-q+1, x-1] as singles + whole groups + singles
    const int a = x - g.q + 1, b = x - 1;
    const int64_t rbase = row * g.xr + g.q;  // slot index of tile 0 of the row
    int ga = (a + g.q + K - 1) / K, gb = (b + g.q + 1) / K - 1;  // groups inside [a, b]
    int s1a = a, s1b = b, s2a = 0, s2b = -1;
    if (b < a) {
      s1b = a - 1, ga = 0, gb = -1;
    } else if (ga <= gb) {
      s1b = ga * K - g.q - 1;
      s2a = (gb + 1) * K - g.q;
      s2b = b;
    } else {
      ga = 0, gb = -1;
    }
    const int n_h = g.r > 0 ? 1 : 0;
    const int n1 = s1b - s1a + 1, n2 = s2b - s2a + 1, ng = gb - ga + 1;
    const int nent = n_h + n1 + n2 + ng;
    auto entry = [&](int e) -> const uint64_t * {
      if (e < n_h) return tslot + (rbase + x - g.q) * 4 + 2;
      if (e < n_h + n1) return tslot + (rbase + s1a + (e - n_h)) * 4;
      if (e < n_h + n1 + n2) return tslot + (rbase + s2a + (e - n_h - n1)) * 4;
      return kslot + (row * g.kt + ga + (e - n_h - n1 - n2)) * 2;
    };
    uint64_t ra[2], rb[2];
#pragma unroll
    for (int e2 = 0; e2 < 2; ++e2) {  // up to 2 entries per lane in flight
      const int e = lane + 32 * e2;
      ra[e2] = rb[e2] = 0;
      if (e < nent) {
        const uint64_t *sp = entry(e);
        ra[e2] = ld_relaxed_u64(sp);
        rb[e2] = ld_relaxed_u64(sp + 1);
      }
    }

    // far prefix + near suffix scans
    T y[E];
    lds_far<T, E, SH>(farb(fs), fsh + lane * E, y);
    T ux[E], un[E];
    T cx, cn;
    {
      ux[0] = un[0] = y[0];
#pragma unroll
      for (int k = 1; k < E; ++k) {
        ux[k] = Ord<T>::mx(ux[k - 1], y[k]);
        un[k] = Ord<T>::mn(un[k - 1], y[k]);
      }
      T ax = ux[E - 1], an = un[E - 1];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const T vx = shfl_up(ax, d), vn = shfl_up(an, d);
        if (lane >= d) {
          ax = Ord<T>::mx(ax, vx);
          an = Ord<T>::mn(an, vn);
        }
      }
      cx = shfl_up(ax, 1);
      cn = shfl_up(an, 1);
      if (lane == 0) {
        cx = y[0];
        cn = y[0];
      }
    }
    {
      T v[E];
      lds_swz_aligned<T, E>(nearb(ns), lane * E, v);
      T sx = v[E - 1], sn = v[E - 1];
      ux[E - 1] = Ord<T>::mx(ux[E - 1], sx);
      un[E - 1] = Ord<T>::mn(un[E - 1], sn);
#pragma unroll
      for (int k = E - 2; k >= 0; --k) {
        sx = Ord<T>::mx(sx, v[k]);
        sn = Ord<T>::mn(sn, v[k]);
        ux[k] = Ord<T>::mx(ux[k], sx);
        un[k] = Ord<T>::mn(un[k], sn);
      }
      T bx = sx, bn = sn;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const T dx = shfl_down(bx, d), dn = shfl_down(bn, d);
        if (lane + d < 32) {
          bx = Ord<T>::mx(bx, dx);
          bn = Ord<T>::mn(bn, dn);
        }
      }
      T ex = shfl_down(bx, 1), en = shfl_down(bn, 1);
      if (lane == 31) {
        ex = v[E - 1];
        en = v[E - 1];
      }
      cx = Ord<T>::mx(cx, ex);
      cn = Ord<T>::mn(cn, en);
    }

    // gap: collect the words (a[u0+w-1] is inside every window: the seed)
    T mx = __shfl_sync(0xffffffffu, y[0], 0), mn = mx;
#pragma unroll
    for (int e2 = 0; e2 < 2; ++e2) {
      const int e = lane + 32 * e2;
      if (e < nent) {
        if (((ra[e2] & rb[e2]) >> 32) == 0) {  // not yet published: poll (rare)
          const uint64_t *sp = entry(e);
          if ((ra[e2] >> 32) == 0) ra[e2] = wait_slot(sp);
          if ((rb[e2] >> 32) == 0) rb[e2] = wait_slot(sp + 1);
        }
        mx = Ord<T>::mx(mx, unpack_slot<T>(ra[e2]));
        mn = Ord<T>::mn(mn, unpack_slot<T>(rb[e2]));
      }
    }
    for (int e = lane + 64; e < nent; e += 32) {  // very large windows
      const uint64_t *sp = entry(e);
      mx = Ord<T>::mx(mx, unpack_slot<T>(wait_slot(sp)));
      mn = Ord<T>::mn(mn, unpack_slot<T>(wait_slot(sp + 1)));
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
      mx = Ord<T>::mx(mx, __shfl_xor_sync(0xffffffffu, mx, d));
      mn = Ord<T>::mn(mn, __shfl_xor_sync(0xffffffffu, mn, d));
    }
    cx = Ord<T>::mx(cx, mx);
    cn = Ord<T>::mn(cn, mn);

    const int64_t left = p.m - u0;
    const int tout = left < WT ? (int)left : WT;
    const int c0 = lane * E;
    if (c0 < tout) {
      T ox[E], on[E];
#pragma unroll
      for (int k = 0; k < E; ++k) {
        ox[k] = Ord<T>::mx(ux[k], cx);
        on[k] = Ord<T>::mn(un[k], cn);
      }
      store_out<T, E>(p, row, u0 + c0, tout - c0, ox, on);
    }
  };

  // ------------------------------------------------------------ pipeline
  // job i is group pbeg + i; far stage i % NFAR, near stage i % NNEAR
  Pos j0 = pos_at(pbeg), j1 = j0, j2;
  advance(j1);
  j2 = j1;
  advance(j2);
  if (lane == 0) {
    load_far(j0, 0);
    load_far(j1, 1);
    load_near(j0, 0);
  }
  uint32_t fph = 0, nph = 0;  // barrier parities per stage (bit s)
  auto wait_far = [&](int s) {
    mbar_wait(&fbar[s], (fph >> s) & 1u);
    fph ^= 1u << s;
  };
  auto wait_near = [&](int s) {
    mbar_wait(&nbar[s], (nph >> s) & 1u);
    nph ^= 1u << s;
  };
  wait_far(0);
  publish(j0, 0);
  int fs = 0, ns = 0;  // stages of job i
  while (j0.tk < gend) {
    const int fs1 = fs + 1 == Geo::NFAR ? 0 : fs + 1, fs2 = fs1 + 1 == Geo::NFAR ? 0 : fs1 + 1;
    const int ns1 = ns ^ 1;
    if (lane == 0) {
      load_far(j2, fs2);
      load_near(j1, ns1);
    }
    wait_far(fs1);
    publish(j1, fs1);  // job i+1 goes public before job i waits on anything
    wait_near(ns);
    process(j0, fs, ns);
    __syncwarp();  // stages fs and ns are reloaded only after every lane read them
    j0 = j1;
    j1 = j2;
    advance(j2);
    fs = fs1;
    ns = ns1;
  }
}

}  // namespace mm

// k1d_lw.cuh -- the large-window 1-D kernel (w-1 >= WT, element types of <= 4
// bytes): SURVEY.md §8 row A5, "tile decomposition + cross-CTA look-back".
//
// Decomposition (k1d_base.cuh): warp-tile x owns the windows [u0, u0+WT),
// u0 = x*WT, WT = 32*E.  Its near chunk N_x = [u0, u0+WT) gives the suffix
// S(i) = max a[u0+i .. u0+WT), its far chunk F_x = [u0+w-1, u0+w-1+WT) the
// prefix P(i) = max a[u0+w-1 .. u0+w-1+i], and
//     out[u0+i] = max(S(i), M_x, P(i)),   M_x = max a[u0+WT .. u0+w-1).
// With w-1 = q*WT + r, M_x is the last r elements of F_{x-q} (H_{x-q}) and the
// whole F_{x-q+1} .. F_{x-1} (G_{..}).  Tiles x in [-q, -1] exist only to
// publish G/H (their far chunks lie in the row), so every row's gaps are
// complete (and the same for every tile: a per-warp constant word list).
//
// Work split.  Tile t = x+q of a row belongs to group t/8 and warp t%8 of
// whichever CTA owns the group.  Groups (all rows concatenated) are taken in
// increasing order from one atomic ticket counter by the CTAs of a persistent
// grid (warp 0 takes the CTA's tickets three jobs ahead and hands them to its
// siblings through a shared ring), so the whole GPU sweeps the rows as one
// front: the near chunk of tile x re-reads bytes that the far chunks of tiles
// x-q, x-q-1 loaded moments before (an L2 hit: HBM reads equal the
// algorithmic n elements).
//
// Publication.  In job i each warp stages the far chunk of job i+3 and the
// near chunk of job i+1 (TMA, 128-B swizzle), then "publishes" job i+2: G and
// H of its far chunk (warp-wide REDUX on order-preserving integer keys) go to
// a shared-memory group table; the last warp of the CTA to arrive (a shared
// atomic election -- nobody waits) turns the table into the group's 32 global
// words: suffix maxima/minima of the 8 G's and the 8 H's, each a 64-bit
// (flag | value) word written with one relaxed store.  Then it processes job
// i: its gap is the same-group prefix from the table (an mbarrier: every
// warp's publish of job i happened two iterations earlier) plus <= 2 + 2q/8
// global words of earlier groups, loaded before the scans and polled only if
// not yet published.  Every live job waits for its table stage, publish-only
// jobs (tiles before a row's first window) too: that wait is what bounds a
// warp's lead over its siblings to the publication lead, and the table, ticket
// and far rings are sized for that bound (warp 0, the ticketer, has no other
// wait on publish-only jobs).  A CTA only waits on lower groups; their tickets were
// taken earlier by CTAs that are running (a CTA takes tickets only while it
// runs) and that only wait on even lower groups -- no deadlock, no residency
// assumption.
//
// Lead (template parameter L3, picked by the launch for q <= MM_LW_L3_QMAX):
// the variant above publishes two jobs ahead; with L3 a warp stages far chunks
// four jobs ahead and publishes job i+3, the fifth far stage taking the shared
// memory of the second near stage -- the single near stage is reloaded for
// job i+1 once job i's suffix scan has consumed it (k1d_lw).
#pragma once

#include "k1d_warp.cuh"

namespace mm {

// order-preserving int32 keys for warp-wide REDUX max/min
template <typename T>
struct RKey {
  static __device__ __forceinline__ int key(T v) { return (int)v; }  // 8/16-bit, int32
  static __device__ __forceinline__ T val(int k) { return (T)k; }
};
template <>
struct RKey<uint32_t> {
  static __device__ __forceinline__ int key(uint32_t v) { return (int)(v ^ 0x80000000u); }
  static __device__ __forceinline__ uint32_t val(int k) { return (uint32_t)k ^ 0x80000000u; }
};
template <>
struct RKey<float> {  // flip the magnitude bits of negatives: signed-int order == float order (no NaN)
  static __device__ __forceinline__ int key(float v) {
    const int b = __float_as_int(v);
    return b ^ ((b >> 31) & 0x7fffffff);
  }
  static __device__ __forceinline__ float val(int k) { return __int_as_float(k ^ ((k >> 31) & 0x7fffffff)); }
};
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
  return RKey<T>::val(__reduce_max_sync(0xffffffffu, RKey<T>::key(v)));
}
template <typename T>
__device__ __forceinline__ T warp_min(T v) {
  return RKey<T>::val(__reduce_min_sync(0xffffffffu, RKey<T>::key(v)));
}

#ifndef MM_LW_STATS  // 1: count gap polls into the workspace header (diagnostics build)
#define MM_LW_STATS 0
#endif

#ifndef MM_LW_L3_QMAX  // publication lead of three jobs for q <= this (the launch picks L3)
#define MM_LW_L3_QMAX 255
#endif
#ifndef MM_LW_TL3  // L3: tickets put this many jobs ahead (>= 5; slot reuse needs < NTK - 4)
#define MM_LW_TL3 5
#endif
#ifndef MM_LW_TL2  // two-job lead: tickets put this many jobs ahead (>= 4; > 4 takes a 16-slot ring)
#define MM_LW_TL2 4
#endif
#ifndef MM_LW_NW0  // gap words per lane loaded before the scans (nent <= 32*NW0; 4: q <= 504)
#define MM_LW_NW0 4
#endif
#ifndef MM_LW_MINB  // resident CTAs per SM the register budget is sized for
#define MM_LW_MINB 2
#endif

template <typename T, bool L3 = false>
struct LwGeo {
  using W = WarpGeo<T>;
  static constexpr int E = W::E, WT = W::WT, RW = W::RW, VEC = W::VEC;
  static constexpr int NROWS = W::NROWS, NEAR = W::NEAR;
  // far chunk = NROWS swizzled rows (a 1024-B aligned buffer like a near
  // chunk) + the one row past them, staged unswizzled into a shared block of
  // 128-B rows (so four far stages cost what three 17-row buffers would)
  // L3 = false: far chunks three jobs ahead (published two ahead), two near
  // stages (one job ahead); ticket ring of 8, tickets put four jobs ahead.
  // L3 = true: far chunks four jobs ahead (published three ahead) in the same
  // shared memory: one near stage, reloaded for job i+1 as soon as job i has
  // consumed it; ticket ring of 16, tickets put five jobs ahead.  Group-table
  // stages: 8 (a warp leads its CTA by <= 2 or 3 jobs).
  static constexpr int NFAR = L3 ? 5 : 4, NNEAR = L3 ? 1 : 2;
  static constexpr int NTAB = 8;
  static constexpr int NTK = (L3 || MM_LW_TL2 > 4) ? 16 : 8;
  static constexpr int WARP_SMEM = (NFAR + NNEAR) * NEAR;
  static constexpr int XROWS = NWARP * NFAR * 128;  // the extra far rows of every warp and stage
  // tail: per warp NFAR+NNEAR mbarriers; per table stage one mbarrier, one
  // election counter and 8 x {Gmax, Gmin, Hmax, Hmin}; the ticket ring
  static constexpr int TAB_OFF = NWARP * (NFAR + NNEAR) * 8;
  static constexpr int TAB_STAGE = 8 + 8 + NWARP * 4 * 4;
  static constexpr int TK_OFF = TAB_OFF + NTAB * TAB_STAGE;  // NTK mbarriers, then NTK int4 slots
  static constexpr size_t BYTES = 1024 + (size_t)NWARP * WARP_SMEM + XROWS + TK_OFF + NTK * 24 + 64;
};

struct LwArgs {
  int q, r;       // w-1 = q*WT + r, q >= 1
  int64_t tpr;    // output tiles per row
  int64_t kt;     // groups per row = ceil((q + tpr) / 8)
  int64_t total;  // batch * kt
};

template <typename T>
struct LwWs {  // [ticket counter | 256 B][total groups x 32 words]
  __host__ __device__ static size_t bytes(const LwArgs &g) { return 256 + (size_t)g.total * 32 * 8 + 64; }
};

__device__ __forceinline__ uint32_t atom_add_shared(uint32_t *p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.acq_rel.cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(p)), "r"(v) : "memory");
  return old;
}

// wait_slot with optional per-lane counters (polled words, spin iterations,
// cycles), added to the workspace header once per warp at the end
struct LwStats {
  unsigned long long polls = 0, spins = 0, cycles = 0;
};
__device__ __forceinline__ uint64_t lw_wait(const uint64_t *s, LwStats &st) {
#if MM_LW_STATS
  const long long t0 = clock64();
  uint64_t v = ld_relaxed_u64(s);
  unsigned spins = 0;
  while ((v >> 32) == 0) {
    __nanosleep(20);
    v = ld_relaxed_u64(s);
    ++spins;
  }
  st.polls += 1;
  st.spins += spins;
  st.cycles += (unsigned long long)(clock64() - t0);
  return v;
#else
  (void)st;
  return wait_slot(s);
#endif
}

template <typename T, int SH, bool L3>
__global__ void __launch_bounds__(NT, MM_LW_MINB) k1d_lw(Rows p, LwArgs g, void *ws, const __grid_constant__ TmaMaps maps) {
  using Geo = LwGeo<T, L3>;
  constexpr int E = Geo::E, WT = Geo::WT, RW = Geo::RW;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *base = smem_align1024(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char *wbuf = base + (size_t)warp * Geo::WARP_SMEM;
  unsigned char *xrows = base + (size_t)NWARP * Geo::WARP_SMEM + warp * Geo::NFAR * 128;
  unsigned char *tail = base + (size_t)NWARP * Geo::WARP_SMEM + Geo::XROWS;
  uint64_t *fbar = reinterpret_cast<uint64_t *>(tail) + warp * (Geo::NFAR + Geo::NNEAR);
  uint64_t *nbar = fbar + Geo::NFAR;
  unsigned char *tab0 = tail + Geo::TAB_OFF;
  auto tbar = [&](int s) { return reinterpret_cast<uint64_t *>(tab0 + s * Geo::TAB_STAGE); };
  auto tcnt = [&](int s) { return reinterpret_cast<uint32_t *>(tab0 + s * Geo::TAB_STAGE + 8); };
  auto tval = [&](int s) { return reinterpret_cast<T *>(tab0 + s * Geo::TAB_STAGE + 16); };  // [4][8]
  auto tkbar = [&](int s) { return reinterpret_cast<uint64_t *>(tail + Geo::TK_OFF) + s; };
  auto tkval = [&](int s) { return reinterpret_cast<int4 *>(tail + Geo::TK_OFF + Geo::NTK * 8) + s; };
  auto farb = [&](int s) { return wbuf + s * Geo::NEAR; };
  auto farx = [&](int s) { return xrows + s * 128; };
  auto nearb = [&](int s) { return wbuf + (Geo::NFAR + s) * Geo::NEAR; };
  uint64_t *gw = reinterpret_cast<uint64_t *>(static_cast<char *>(ws) + 256);  // group words
  LwStats pst;

  const int64_t w = p.w;
  const int64_t full_el = (p.n / RW) * RW;  // elements covered by the tensor maps
  const int fsh = (int)((w - 1) % RW);      // far chunk offset inside its first 128-B row
  const int q = g.q, r = g.r;
  const int h_lane = (WT - r) / E, h_off = (WT - r) % E;  // H = far chunk [WT-r, WT)

  if (threadIdx.x == 0) {
    for (int i = 0; i < NWARP * (Geo::NFAR + Geo::NNEAR); ++i) mbar_init(reinterpret_cast<uint64_t *>(tail) + i, 1);
    for (int s = 0; s < Geo::NTAB; ++s) {
      mbar_init(tbar(s), NWARP);
      *tcnt(s) = 0;
    }
    for (int s = 0; s < Geo::NTK; ++s) mbar_init(tkbar(s), 1);
    fence_mbar_init();
    prefetch_tmap(&maps.big);
    prefetch_tmap(&maps.small);
  }
  __syncthreads();  // the only CTA-wide barrier

  // ---- the gap's global words: a per-warp constant list relative to the
  // job's group (offsets in words, <= 0), max words first then min words
  // tile t = 8*gi + warp; H of t-q; G of t-q+1 .. 8*gi-1 (earlier groups); the
  // own group's t-q+1 .. t-1 come from the shared table
  const int k = warp;
  const int dh = (q - k + 7) >> 3;  // groups back to tile t-q (0: own group)
  const int hk = ((k - q) % 8 + 8) % 8;
  const int da = (q - 1 - k + 7) >> 3;  // groups back to tile t-q+1 (0: inside the own group)
  const int sa = ((k - q + 1) % 8 + 8) % 8;
  // entries: [H pair if dh > 0 && r > 0][suffix pair of group gi-da if da > 0][Σ0 pair of gi-d, d = 1..da-1]
  const int n_h = (dh > 0 && r > 0) ? 1 : 0;
  const int npair = n_h + (da > 0 ? da : 0);
  const int nent = 2 * npair;
  auto entry_off = [&](int e) -> int {  // word offset relative to the job's group base
    const int pr = e >> 1, mn = e & 1;
    if (pr < n_h) return -dh * 32 + 16 + 8 * mn + hk;
    const int j = pr - n_h;  // 0: the partial group gi-da, then gi-da+1 .. gi-1
    const int d = da - j;
    return -d * 32 + 8 * mn + (j == 0 ? sa : 0);
  };
  // own group: siblings [lo_own, k) give G; sibling k-q gives H when dh == 0
  const int lo_own = k - q + 1 > 0 ? k - q + 1 : 0;
  const int eoff0 = lane < nent ? entry_off(lane) : 0, eoff1 = lane + 32 < nent ? entry_off(lane + 32) : 0;

  // ---- far chunk access: logical element pos of the chunk (0 <= pos < (NROWS+1)*RW)
  constexpr int NMAIN = Geo::NROWS * 8;  // 16-B chunks in the swizzled main rows
  auto far_addr = [&](int s, int c) -> const unsigned char * {
    return c < NMAIN ? farb(s) + swz(c) : farx(s) + ((c - NMAIN) << 4);
  };
  // this lane's far read (elements fsh + lane*E ..): NQ 16-B chunks at fixed
  // offsets, the chunks past the main rows in the extra row (mask xm)
  constexpr int NQF = E / Geo::VEC + 1;
  int foff[NQF];
  uint32_t xm = 0;
  {
    const int c0 = (fsh + lane * E) / Geo::VEC;
#pragma unroll
    for (int kk = 0; kk < NQF; ++kk) {
      const int c = c0 + kk;
      foff[kk] = c < NMAIN ? (int)swz(c) : (c - NMAIN) << 4;
      xm |= (c < NMAIN ? 0u : 1u) << kk;
    }
  }
  auto lds_far2 = [&](int s, T (&v)[E]) {
    constexpr int VEC = Geo::VEC;
    const unsigned char *mb = farb(s), *xb = farx(s);
    union {
      T t[NQF * VEC];
      uint4 q[NQF];
    } u;
#pragma unroll
    for (int kk = 0; kk < NQF; ++kk)
      u.q[kk] = *reinterpret_cast<const uint4 *>(((xm >> kk) & 1u ? xb : mb) + foff[kk]);
    if constexpr (SH >= 0) {
#pragma unroll
      for (int kk = 0; kk < E; ++kk) v[kk] = u.t[kk + SH];
    } else {
      const int sh = (fsh + lane * E) % VEC;
#define MM_LW_SH(S)                                                                     \
  case S:                                                                               \
    if (S < VEC) {                                                                      \
      _Pragma("unroll") for (int kk = 0; kk < E; ++kk) v[kk] = u.t[kk + (S < VEC ? S : 0)]; \
    }                                                                                   \
    break;
      switch (sh) {
        MM_LW_SH(0) MM_LW_SH(1) MM_LW_SH(2) MM_LW_SH(3) MM_LW_SH(4) MM_LW_SH(5) MM_LW_SH(6) MM_LW_SH(7)
        MM_LW_SH(8) MM_LW_SH(9) MM_LW_SH(10) MM_LW_SH(11) MM_LW_SH(12) MM_LW_SH(13) MM_LW_SH(14) MM_LW_SH(15)
        default: break;
      }
#undef MM_LW_SH
    }
  };
  auto sts_far2 = [&](int s, int pos, T v) {  // (tail patch)
    const int c = pos / Geo::VEC;
    *reinterpret_cast<T *>(const_cast<unsigned char *>(far_addr(s, c)) + (pos - c * Geo::VEC) * sizeof(T)) = v;
  };

  // ---- job positions: group tk = row*kt + gi, from the ticket ring.  Warp 0's
  // lane 0 takes the tickets (one atomic per job, issued a job before its
  // result is needed, so its latency hides) and publishes {tk, row, gi} three
  // jobs ahead; every warp derives its tile from them (int32: < 2^31 groups).
  struct Pos {
    int tk, row, x;  // group ticket, row, this warp's tile
    bool live, far, near;
  };
  unsigned int *counter = static_cast<unsigned int *>(ws);
  const int kt32 = (int)g.kt, tpr32 = (int)g.tpr, total32 = (int)g.total;
  auto put_ticket = [&](int64_t job, int tk) {  // warp 0, lane 0
    const int s = (int)(job & (Geo::NTK - 1));
    const int row = tk / kt32;
    *tkval(s) = make_int4(tk, row, tk - row * kt32, 0);
    mbar_arrive1(tkbar(s));
  };
  auto wait_ticket = [&](int64_t job) {  // every lane, once per job (slot reused 8 jobs later)
    mbar_wait(tkbar((int)(job & (Geo::NTK - 1))), (uint32_t)((job / Geo::NTK) & 1));
  };
  auto pos = [&](int64_t job) {  // (after wait_ticket(job))
    const int4 t = *tkval((int)(job & (Geo::NTK - 1)));
    Pos o;
    o.tk = t.x;
    o.row = t.y;
    o.x = t.z * 8 + k - q;
    o.live = o.tk < total32;
    o.far = o.live && o.x < tpr32;
    o.near = o.far && o.x >= 0;
    return o;
  };
  const int far_row0 = (int)((w - 1) / RW);  // tile x's far chunk starts at row x*(WT/RW) + far_row0
  auto load_far = [&](const Pos &j, int s) {
    if (!j.far) {
      mbar_arrive_expect_tx(&fbar[s], 0);
      return;
    }
    mbar_arrive_expect_tx(&fbar[s], (Geo::NROWS + 1) * 128);
    const int r0 = j.x * (WT / RW) + far_row0;
    tma_box(&maps.big, farb(s), r0, j.row, &fbar[s]);
    tma_box(&maps.small, farx(s), r0 + Geo::NROWS, j.row, &fbar[s]);  // one unswizzled row
  };
  auto load_near = [&](const Pos &j, int s) {
    if (!j.near) {
      mbar_arrive_expect_tx(&nbar[s], 0);
      return;
    }
    mbar_arrive_expect_tx(&nbar[s], Geo::NROWS * 128);
    tma_box(&maps.big, nearb(s), j.x * (WT / RW), j.row, &nbar[s]);
  };
  // elements at or past full_el are not in the maps: plain loads
  auto patch = [&](unsigned char *buf, int64_t row, int64_t start, int64_t len) {
    const int64_t a0 = start > full_el ? start : full_el;
    const int64_t a1 = p.n < start + len ? p.n : start + len;
    const T *srs = series_ptr<T>(p, row);
    for (int64_t i = a0 + lane; i < a1; i += 32) sts_swz<T>(buf, (int)(i - start), srs[i]);
  };
  auto patch_far = [&](int s, int64_t row, int64_t start, int64_t len) {
    const int64_t a0 = start > full_el ? start : full_el;
    const int64_t a1 = p.n < start + len ? p.n : start + len;
    const T *srs = series_ptr<T>(p, row);
    for (int64_t i = a0 + lane; i < a1; i += 32) sts_far2(s, (int)(i - start), srs[i]);
  };

  // ------------------------------------------------------------ publish
  auto publish = [&](const Pos &j, int fs, int ts) {
    if (!j.live) return;
    T gx, gn, hx, hn;
#if MM_LW_ABL == 2  // ablation (wrong results): publish constants without reading the far chunk
    if (false) {
#else
    if (j.far) {
#endif
      if (full_el < p.n) {
        patch_far(fs, j.row, (int64_t)j.x * WT + w - 1 - fsh, (Geo::NROWS + 1) * RW);
        __syncwarp();
      }
      T y[E];
      lds_far2(fs, y);
      T ax = y[0], an = y[0];
#pragma unroll
      for (int e = 1; e < E; ++e) {
        ax = Ord<T>::mx(ax, y[e]);
        an = Ord<T>::mn(an, y[e]);
      }
      gx = warp_max(ax);
      gn = warp_min(an);
      if (r > 0) {  // H: lanes past h_lane whole, lane h_lane from h_off, others none
        T vx, vn;
        suffix_from<T, E>(y, h_off, vx, vn);
        int kx = lane > h_lane ? RKey<T>::key(ax) : lane == h_lane ? RKey<T>::key(vx) : INT_MIN;
        int kn = lane > h_lane ? RKey<T>::key(an) : lane == h_lane ? RKey<T>::key(vn) : INT_MAX;
        hx = RKey<T>::val(__reduce_max_sync(0xffffffffu, kx));
        hn = RKey<T>::val(__reduce_min_sync(0xffffffffu, kn));
      } else {
        hx = gx;
        hn = gn;
      }
    } else {  // a tile past the row's last window: never consumed
      gx = gn = hx = hn = T(0);
    }
    T *tv = tval(ts);
    if (lane == 0) {
      tv[0 * NWARP + k] = gx;
      tv[1 * NWARP + k] = gn;
      tv[2 * NWARP + k] = hx;
      tv[3 * NWARP + k] = hn;
    }
    uint32_t last = 0;
    if (lane == 0) {
      mbar_arrive1(tbar(ts));  // release: the entries are visible to the waiters
      last = atom_add_shared(tcnt(ts), 1u) == NWARP - 1;
      if (last) *tcnt(ts) = 0;  // every warp has arrived for this use of the stage
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) return;
    // the last warp of the CTA to arrive writes the group's 32 words
    __syncwarp();
    const int i8 = lane & 7, kind = lane >> 3;  // 0: Σmax, 1: Σmin, 2: Hmax, 3: Hmin
    T v = tv[kind * NWARP + i8];
#pragma unroll
    for (int d = 1; d < 8; d <<= 1) {  // suffix over the 8 G's (octets 0, 1; all lanes shuffle)
      const T o = shfl_down(v, d);
      if (kind < 2 && i8 + d < 8) v = kind == 0 ? Ord<T>::mx(v, o) : Ord<T>::mn(v, o);
    }
    st_relaxed_u64(gw + (int64_t)j.tk * 32 + lane, pack_slot<T>(v));
  };

  // ------------------------------------------------------------ process
  // next_near (LEAD3): after this job's near chunk is in registers, lane 0
  // stages the next job's into the single near stage
  auto process = [&](const Pos &j, int fs, int ns, int ts, const Pos *next_near) {
    if (!j.near) {
      if (next_near && lane == 0) load_near(*next_near, 0);
      return;
    }
    const int64_t row = j.row;
    const int64_t u0 = (int64_t)j.x * WT;
    // gap words first: their latency overlaps the scans
    const uint64_t *gb = gw + (int64_t)j.tk * 32;
    constexpr int NW0 = MM_LW_NW0;  // words per lane held in flight (nent <= 32*NW0)
    uint64_t wv[NW0];
#pragma unroll
    for (int e2 = 0; e2 < NW0; ++e2) {
      const int e = lane + 32 * e2;
      wv[e2] = e < nent ? ld_relaxed_u64(gb + (e2 == 0 ? eoff0 : e2 == 1 ? eoff1 : entry_off(e))) : 0;
    }
    if (full_el < p.n) {  // (the far chunk was patched when it was published)
      patch(nearb(ns), row, u0, WT);
      __syncwarp();
    }
    // far chunk: prefix scan
    T px[E], pn[E];
    lds_far2(fs, px);
    const T seed = __shfl_sync(0xffffffffu, px[0], 0);  // a[u0+w-1]: inside every window of the tile
#pragma unroll
    for (int e = 0; e < E; ++e) pn[e] = px[e];
#pragma unroll
    for (int e = 1; e < E; ++e) {
      px[e] = Ord<T>::mx(px[e - 1], px[e]);
      pn[e] = Ord<T>::mn(pn[e - 1], pn[e]);
    }
    T cx = px[E - 1], cn = pn[E - 1];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      cx = Ord<T>::mx(cx, shfl_up(cx, d));  // (lanes below d get their own value: idempotent)
      cn = Ord<T>::mn(cn, shfl_up(cn, d));
    }
    T Cx = shfl_up(cx, 1), Cn = shfl_up(cn, 1);  // exclusive carries (lane 0: the seed)
    if (lane == 0) Cx = Cn = seed;
    // near chunk: suffix scan in place
    T sx[E], sn[E];
    lds_swz_aligned<T, E>(nearb(ns), lane * E, sx);
#pragma unroll
    for (int e = 0; e < E; ++e) sn[e] = sx[e];
#pragma unroll
    for (int e = E - 2; e >= 0; --e) {
      sx[e] = Ord<T>::mx(sx[e], sx[e + 1]);
      sn[e] = Ord<T>::mn(sn[e], sn[e + 1]);
    }
    {
      T bx = sx[0], bn = sn[0];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        bx = Ord<T>::mx(bx, shfl_down(bx, d));
        bn = Ord<T>::mn(bn, shfl_down(bn, d));
      }
      T ex = shfl_down(bx, 1), en = shfl_down(bn, 1);
      if (lane == 31) ex = en = seed;
      if (next_near) {
        // every lane's near values are consumed (the scan above used them):
        // the single near stage takes the next job's chunk
        __syncwarp();
        if (lane == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          load_near(*next_near, 0);
        }
      }
      Cx = Ord<T>::mx(Cx, ex);
      Cn = Ord<T>::mn(Cn, en);
    }
    // gap: own-group entries from the table, then the global words
    T mx = seed, mn = seed;
    {  // (the caller waited for the table stage)
      const T *tv = tval(ts);
      if (lane < 8 && lane >= lo_own && lane < k) {
        mx = Ord<T>::mx(mx, tv[0 * NWARP + lane]);
        mn = Ord<T>::mn(mn, tv[1 * NWARP + lane]);
      }
      if (dh == 0 && r > 0 && lane == 0) {
        mx = Ord<T>::mx(mx, tv[2 * NWARP + hk]);
        mn = Ord<T>::mn(mn, tv[3 * NWARP + hk]);
      }
    }
    // (entry e of a lane has parity e & 1 == lane & 1: odd lanes hold min words)
#pragma unroll
    for (int e2 = 0; e2 < NW0; ++e2) {
      const int e = lane + 32 * e2;
      if (e < nent) {
        uint64_t v = wv[e2];
#if MM_LW_ABL == 1  // ablation (wrong results): never wait for a word
        if ((v >> 32) == 0) v = pack_slot<T>(seed);
#else
        if ((v >> 32) == 0) v = lw_wait(gb + (e2 == 0 ? eoff0 : e2 == 1 ? eoff1 : entry_off(e)), pst);
#endif
        const T t = unpack_slot<T>(v);
        if (lane & 1)
          mn = Ord<T>::mn(mn, t);
        else
          mx = Ord<T>::mx(mx, t);
      }
    }
    for (int e = lane + 32 * NW0; e < nent; e += 32) {  // very large windows (nent > 32*NW0)
      const T t = unpack_slot<T>(lw_wait(gb + entry_off(e), pst));
      if (lane & 1)
        mn = Ord<T>::mn(mn, t);
      else
        mx = Ord<T>::mx(mx, t);
    }
    mx = warp_max(mx);
    mn = warp_min(mn);
    Cx = Ord<T>::mx(Cx, mx);
    Cn = Ord<T>::mn(Cn, mn);

    const int64_t j0 = u0 + lane * E;
    const int cnt = p.m - j0 < E ? (int)(p.m - j0) : E;
    if (cnt > 0) {
      T ox[E], on[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        ox[e] = Ord<T>::mx(Ord<T>::mx(px[e], sx[e]), Cx);
        on[e] = Ord<T>::mn(Ord<T>::mn(pn[e], sn[e]), Cn);
      }
      const int64_t o = row * p.out_ld + j0;
      T *omx = static_cast<T *>(p.out_max), *omn = static_cast<T *>(p.out_min);
      if (cnt == E) {
        if (omx) store_chunk<T, E>(omx + o, ox);
        if (omn) store_chunk<T, E>(omn + o, on);
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e)
          if (e < cnt) {
            if (omx) omx[o + e] = ox[e];
            if (omn) omn[o + e] = on[e];
          }
      }
    }
  };

  // ------------------------------------------------------------ pipeline
if constexpr (L3) {
  // job i: far stage i%5 (loaded four jobs ahead, published three ahead),
  // the near stage, table stage i%8, ticket slot i%16 (put five jobs ahead)
  const bool ticketer = warp == 0 && lane == 0;
  constexpr int TL = MM_LW_TL3;
  static_assert(TL >= 5 && TL + 4 < Geo::NTK, "ticket lead");
  unsigned int pend = 0;  // warp 0 lane 0: the ticket of job i+TL+1, in flight during job i
  if (ticketer) {
    unsigned t[TL];
#pragma unroll
    for (int i = 0; i < TL; ++i) t[i] = atomicAdd(counter, 1u);
#pragma unroll
    for (int i = 0; i < TL; ++i) put_ticket(i, (int)t[i]);
    pend = atomicAdd(counter, 1u);
  }
  for (int i = 0; i < 5; ++i) wait_ticket(i);
  if (lane == 0) {
    for (int i = 0; i < 4; ++i) load_far(pos(i), i);
    load_near(pos(0), 0);
  }
  uint32_t fph = 0, nph = 0, tph = 0;  // barrier parities per stage (bit s)
  auto wait_far = [&](int s) {
    mbar_wait(&fbar[s], (fph >> s) & 1u);
    fph ^= 1u << s;
  };
  for (int i = 0; i < 3; ++i) {
    wait_far(i);
    publish(pos(i), i, i);
  }
  int64_t job = 0;
  int fs = 0;  // job % 5
  while (pos(job).live) {
    const int ts = (int)(job & 7);
    const int fl = fs == 0 ? 4 : fs - 1;  // (job+4) % 5: job-1's stage, now free
    const int fp = fl == 0 ? 4 : fl - 1;  // (job+3) % 5
    if (ticketer) {
      put_ticket(job + TL, (int)pend);
      pend = atomicAdd(counter, 1u);
    }
    if (lane == 0) load_far(pos(job + 4), fl);
    wait_far(fp);
    publish(pos(job + 3), fp, (int)((job + 3) & 7));  // job i+3 goes public before job i waits on anything
    mbar_wait(&nbar[0], nph);
    nph ^= 1u;
    const Pos j0 = pos(job), j1 = pos(job + 1);
    // every live job waits for its table stage, publish-only ones too: this
    // bounds how far a warp (warp 0 included, which takes no ticket waits) can
    // run ahead of its siblings, so the table, ticket and far rings are never
    // refilled under a slower warp
    mbar_wait(tbar(ts), (tph >> ts) & 1u);
    tph ^= 1u << ts;
    process(j0, fs, 0, ts, &j1);
    __syncwarp();  // stage fs is reloaded only after every lane read it
    ++job;
    fs = fs == 4 ? 0 : fs + 1;
    wait_ticket(job + 4);
  }
} else {
  // job i: far stage i%4, near stage i%2, table stage i%8, ticket slot i%8
  const bool ticketer = warp == 0 && lane == 0;
  constexpr int TL = MM_LW_TL2;
  static_assert(TL >= 4 && TL + 3 < Geo::NTK, "ticket lead");
  unsigned int pend = 0;  // warp 0 lane 0: the ticket of job i+TL+1, in flight during job i
  if (ticketer) {
    unsigned t[TL];
#pragma unroll
    for (int i = 0; i < TL; ++i) t[i] = atomicAdd(counter, 1u);
#pragma unroll
    for (int i = 0; i < TL; ++i) put_ticket(i, (int)t[i]);
    pend = atomicAdd(counter, 1u);
  }
  for (int i = 0; i < 4; ++i) wait_ticket(i);
  if (lane == 0) {
    load_far(pos(0), 0);
    load_far(pos(1), 1);
    load_far(pos(2), 2);
    load_near(pos(0), 0);
  }
  uint32_t fph = 0, nph = 0, tph = 0;  // barrier parities per stage (bit s)
  auto wait_far = [&](int s) {
    mbar_wait(&fbar[s], (fph >> s) & 1u);
    fph ^= 1u << s;
  };
  auto wait_near = [&](int s) {
    mbar_wait(&nbar[s], (nph >> s) & 1u);
    nph ^= 1u << s;
  };
  wait_far(0);
  publish(pos(0), 0, 0);
  wait_far(1);
  publish(pos(1), 1, 1);
  int64_t job = 0;
  while (pos(job).live) {
    const int fs = (int)(job & 3), ns = (int)(job & 1), ts = (int)(job & 7);
    if (ticketer) {
      put_ticket(job + TL, (int)pend);
      pend = atomicAdd(counter, 1u);
    }
    if (lane == 0) {
      load_far(pos(job + 3), (fs + 3) & 3);
      load_near(pos(job + 1), ns ^ 1);
    }
    wait_far((fs + 2) & 3);
    publish(pos(job + 2), (fs + 2) & 3, (ts + 2) & 7);  // job i+2 goes public before job i waits on anything
    wait_near(ns);
    const Pos j0 = pos(job);
    // the table stage of job i is complete once all 8 warps published it; every
    // live job waits for it, publish-only ones too (bounds the warps' spread)
    mbar_wait(tbar(ts), (tph >> ts) & 1u);
    tph ^= 1u << ts;
    process(j0, fs, ns, ts, nullptr);
    __syncwarp();  // stages fs and ns are reloaded only after every lane read them
    ++job;
    wait_ticket(job + 3);
  }
}  // L3
#if MM_LW_STATS
  {
    unsigned long long *st = reinterpret_cast<unsigned long long *>(static_cast<char *>(ws) + 64);
    unsigned long long a = pst.polls, b = pst.spins, c = pst.cycles, mx = pst.cycles;
    for (int d = 16; d >= 1; d >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, d);
      b += __shfl_xor_sync(0xffffffffu, b, d);
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, mx, d);
      mx = o > mx ? o : mx;
    }
    if (lane == 0) {
      atomicAdd(st + 0, a);
      atomicAdd(st + 1, b);
      atomicAdd(st + 2, mx);  // per warp: the busiest lane's wait cycles
      atomicMax(st + 3, mx);
    }
  }
#endif
}

}  // namespace mm

// k1d_large.cuh -- large-window 1-D kernel with cross-CTA look-back (see k1d_base.cuh).
#pragma once

#include "k1d_base.cuh"

#ifndef MM_STAGE_POS
#define MM_STAGE_POS 1  // 0: stage before the publish step, 1: right after it
#endif
#ifndef MM_STAGE_WARP
#define MM_STAGE_WARP 7  // the warp that grabs and stages tickets (not warp 0, which publishes)
#endif
#ifndef MM_LARGE_ISSUE
#define MM_LARGE_ISSUE 1  // 0: lane 0 issues 8-row boxes; 1: lanes issue 32/8-row boxes
#endif

namespace mm {

// ===================================================================== large
// w-1 > kHaloMax.  Tile x owns outputs [u0, u0+T), u0 = xT, and stages
//   near N_x = [u0, u0+T)            -> S(i) = max a[u0+i .. u0+T)       (CTA suffix scan)
//   far  F_x = [u0+w-1, u0+w-1+T)    -> P(i) = max a[u0+w-1 .. u0+w-1+i] (CTA prefix scan)
// so that out[u0+i] = max(S(i), M_x, P(i)) with the fixed gap
//   M_x = max a[u0+T .. u0+w-1).
// With w-1 = qT + r the gap is the last r elements of F_{x-q} followed by the
// whole F_{x-q+1} .. F_{x-1}.  Every tile publishes G_x = max F_x and H_x = max
// of the last r elements of F_x; tile x consumes H_{x-q}, G_{x-q+1..x-1}.
// Tiles x in [-q, -1] exist only to publish (their F lies inside the array).
//
// Tickets (atomic counter) order the tiles: ticket = (row, x+q) row-major, so
// the look-back distance is q tiles of the global stream and F_x is still in L2
// when tile x+q stages it as its near tile.  Each CTA runs a 3-stage TMA ring:
// in iteration i it (1) grabs and stages ticket i+2, (2) publishes the
// aggregates of ticket i+1 (already staged), (3) processes ticket i, whose
// predecessors were published an iteration earlier -- the look-back normally
// finds its values ready and stays off the critical path.  Publishing waits on
// nothing but TMA data and waits only target lower tickets, so the scheme is
// deadlock-free for any number of resident CTAs.
//
// Publication: for element types of <= 4 bytes each aggregate travels as one
// 64-bit word (1 << 32 | bits), written and polled with relaxed gpu-scope
// accesses -- the flag and the value are a single-copy-atomic store.  8-byte
// types use a separate release/acquire flag per ticket.
struct LargeGeom {
  int q, r;
  int64_t tickets_per_row;  // q + tiles_per_row
  int64_t total;            // batch * tickets_per_row
};

template <typename T>
struct LargeWs {  // workspace carve-up: [counter | 256 B][flags (8-B types)][slots]
  static constexpr bool kPacked = sizeof(T) <= 4;
  __host__ __device__ static size_t slots_offset(int64_t tickets) {
    return kPacked ? 256 : ((256 + (size_t)tickets * 4 + 255) & ~size_t(255));
  }
  __host__ __device__ static size_t bytes(int64_t tickets) {
    return slots_offset(tickets) + (size_t)tickets * 4 * 8 + 64;
  }
  // bytes to zero before a launch (counter + flags, or counter + packed slots)
  __host__ __device__ static size_t zero_bytes(int64_t tickets) {
    return kPacked ? 256 + (size_t)tickets * 32 : slots_offset(tickets);
  }
};

template <typename T>
struct LargeLayout {
  static constexpr int E = Chunk<T>::E;
  static constexpr int TILE = NT * E;
  static constexpr int RW = Rowing<T>::RW;
  static constexpr int NSTAGE = 3;
  static constexpr int NROWS = (TILE / RW + kBoxRows - 1) / kBoxRows * kBoxRows;
  static constexpr int FROWS = ((TILE + RW) / RW + kBoxRows - 1) / kBoxRows * kBoxRows;
  static constexpr size_t NB = (size_t)NROWS * 128, FB = (size_t)FROWS * 128;
  static constexpr size_t STAGE = NB + FB;
  static constexpr size_t BYTES = 1024 + NSTAGE * STAGE + 256;
};

template <typename T>
__device__ __forceinline__ uint64_t pack_slot(T v) {
  uint32_t b = 0;
  static_assert(sizeof(T) <= 4, "packed slots hold <= 4-byte values");
  memcpy(&b, &v, sizeof(T));
  return (uint64_t(1) << 32) | b;
}
template <typename T>
__device__ __forceinline__ T unpack_slot(uint64_t s) {
  uint32_t b = (uint32_t)s;
  T v;
  memcpy(&v, &b, sizeof(T));
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t *p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

template <typename T>
__global__ void __launch_bounds__(NT, 2)
    k1d_large(Rows p, LargeGeom g, void *ws, const __grid_constant__ TmaMaps maps) {
  using Lay = LargeLayout<T>;
  using Ws = LargeWs<T>;
  constexpr int E = Lay::E;
  constexpr int TILE = Lay::TILE;
  constexpr int RW = Lay::RW;
  constexpr int NS = Lay::NSTAGE;

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *base = smem_align1024(smem_raw);
  auto nearb = [&](int i) { return base + i * Lay::STAGE; };
  auto farb = [&](int i) { return base + i * Lay::STAGE + Lay::NB; };
  __shared__ T wpub[2][4][NWARP];  // G/H partials of the published ticket (by parity)
  __shared__ T wpre[2][NWARP];     // far prefix warp totals of the processed ticket
  __shared__ T wsuf[2][NWARP];     // near suffix warp totals
  __shared__ T wgap[2][NWARP];     // look-back gap partials
  __shared__ int64_t s_ticket[NS];
  __shared__ int s_fshift[NS];
  __shared__ __align__(8) uint64_t bars[NS];

  unsigned long long *counter = reinterpret_cast<unsigned long long *>(ws);
  uint32_t *flags = reinterpret_cast<uint32_t *>(static_cast<char *>(ws) + 256);  // 8-B types
  uint64_t *slots = reinterpret_cast<uint64_t *>(static_cast<char *>(ws) + Ws::slots_offset(g.total));
  // slot k of ticket t: slots[4t + k], k = 0 Gmax, 1 Gmin, 2 Hmax, 3 Hmin

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t w = p.w;

  auto decode = [&](int64_t tk, int64_t &row, int64_t &x) {
    row = tk / g.tickets_per_row;
    x = tk - row * g.tickets_per_row - g.q;  // may be negative
  };

  // stage ticket tk (grabbed an iteration earlier) into stage st: warp 0, the
  // boxes (32-row "big" ones plus 8-row ones) issued by different lanes
  auto stage_ticket = [&](int64_t tk, int st) {
    if (lane == 0) s_ticket[st] = tk;
    if (tk >= g.total) {
      if (lane == 0) mbar_arrive_expect_tx(&bars[st], 0);
      return;
    }
    int64_t row, x;
    decode(tk, row, x);
    const int64_t u0 = x * TILE;
    const int64_t f0 = u0 + w - 1;
    const int64_t flen = p.n - f0 < TILE ? p.n - f0 : TILE;
    if (lane == 0) s_fshift[st] = (int)(f0 - (f0 / RW) * RW);
    if (p.has_map && MM_LARGE_ISSUE == 0) {  // lane 0 issues 8-row boxes one by one
      if (lane == 0) {
        const int64_t fr0 = f0 / RW, fr1 = (f0 + flen + RW - 1) / RW;
        const int nfb = (int)((fr1 - fr0 + kBoxRows - 1) / kBoxRows);
        const int nnb = x >= 0 ? (TILE / RW + kBoxRows - 1) / kBoxRows : 0;
        mbar_arrive_expect_tx(&bars[st], (uint32_t)(nfb + nnb) * kBoxBytes);
        for (int k = 0; k < nfb; ++k)
          tma_box(&maps.small, farb(st) + k * kBoxBytes, (int)(fr0 + k * kBoxRows), (int)row, &bars[st]);
        for (int k = 0; k < nnb; ++k)
          tma_box(&maps.small, nearb(st) + k * kBoxBytes, (int)(u0 / RW + k * kBoxRows), (int)row,
                  &bars[st]);
      }
    } else if (p.has_map) {
      const int64_t fr0 = f0 / RW, fr1 = (f0 + flen + RW - 1) / RW;
      const int frows = (int)(fr1 - fr0);
      const int nrows = x >= 0 ? TILE / RW : 0;
      const int fbig = frows / kBigRows, fsm = (frows - fbig * kBigRows + kBoxRows - 1) / kBoxRows;
      const int nbig = nrows / kBigRows, nsm = (nrows - nbig * kBigRows + kBoxRows - 1) / kBoxRows;
      if (lane == 0)
        mbar_arrive_expect_tx(&bars[st], (uint32_t)((fbig + nbig) * kBigBytes + (fsm + nsm) * kBoxBytes));
      __syncwarp();
      const int nf = fbig + fsm, ntot = nf + nbig + nsm;
      for (int k = lane; k < ntot; k += 32) {
        if (k < fbig)
          tma_box(&maps.big, farb(st) + k * kBigBytes, (int)(fr0 + k * kBigRows), (int)row, &bars[st]);
        else if (k < nf)
          tma_box(&maps.small, farb(st) + fbig * kBigBytes + (k - fbig) * kBoxBytes,
                  (int)(fr0 + fbig * kBigRows + (k - fbig) * kBoxRows), (int)row, &bars[st]);
        else if (k < nf + nbig)
          tma_box(&maps.big, nearb(st) + (k - nf) * kBigBytes, (int)(u0 / RW + (k - nf) * kBigRows),
                  (int)row, &bars[st]);
        else
          tma_box(&maps.small, nearb(st) + nbig * kBigBytes + (k - nf - nbig) * kBoxBytes,
                  (int)(u0 / RW + nbig * kBigRows + (k - nf - nbig) * kBoxRows), (int)row, &bars[st]);
      }
    } else if (lane == 0) {
      mbar_arrive_expect_tx(&bars[st], 0);
    }
  };

  // after the stage's barrier: patch the partial last 128-B row (all threads);
  // returns whether shared memory was written
  auto patch = [&](int st, int64_t row, int64_t x) -> bool {
    const int64_t full = p.has_map ? (p.n / RW) * RW : 0;
    if (full >= p.n) return false;
    bool fixed = false;
    const T *srs = series_ptr<T>(p, row);
    const int64_t u0 = x * TILE;
    const int64_t f0 = u0 + w - 1;
    const int64_t fa = f0 - s_fshift[st];  // absolute start of the far stage
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
    return fixed;
  };

  // Publish G/H of the ticket staged for iteration `itp` (all threads).  Always
  // ends with one barrier, which also fences the process-step partials.
  auto publish = [&](int itp) {
    const int st = itp % NS;
    const int pb = itp & 1;
    const int64_t tk = s_ticket[st];
    if (tk >= g.total) {  // uniform
      __syncthreads();
      return;
    }
    int64_t row, x;
    decode(tk, row, x);
    mbar_wait(&bars[st], (uint32_t)((itp / NS) & 1));  // stage used once per NS iterations
    if (patch(st, row, x)) __syncthreads();
    const int fshift = s_fshift[st];
    T v[E];
    lds_swz<T, E>(farb(st), fshift + tid * E, v);
    T gx = v[0], gn = v[0];
#pragma unroll
    for (int k = 1; k < E; ++k) {
      gx = Ord<T>::mx(gx, v[k]);
      gn = Ord<T>::mn(gn, v[k]);
    }
    // last r positions of F_x: [TILE - r, TILE); threads outside borrow the
    // element at TILE-1, which belongs to every non-empty H range
    const int hstart = TILE - g.r;
    T hx, hn;
    hx = hn = lds_one_swz<T>(farb(st), fshift + TILE - 1);
    if (tid * E >= hstart) {
      hx = Ord<T>::mx(hx, gx);
      hn = Ord<T>::mn(hn, gn);
    } else if (tid * E + E > hstart) {
      T vx, vn;
      suffix_from<T, E>(v, hstart - tid * E, vx, vn);
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
    if (lane == 0) {
      wpub[pb][0][warp] = gx;
      wpub[pb][1][warp] = gn;
      wpub[pb][2][warp] = hx;
      wpub[pb][3][warp] = hn;
    }
    __syncthreads();
    if (warp == 0) {
      const int vv = lane & (NWARP - 1);
      T a0 = wpub[pb][0][vv], a1 = wpub[pb][1][vv], a2 = wpub[pb][2][vv], a3 = wpub[pb][3][vv];
#pragma unroll
      for (int d = NWARP / 2; d >= 1; d >>= 1) {
        a0 = Ord<T>::mx(a0, __shfl_xor_sync(0xffffffffu, a0, d));
        a1 = Ord<T>::mn(a1, __shfl_xor_sync(0xffffffffu, a1, d));
        a2 = Ord<T>::mx(a2, __shfl_xor_sync(0xffffffffu, a2, d));
        a3 = Ord<T>::mn(a3, __shfl_xor_sync(0xffffffffu, a3, d));
      }
      if constexpr (Ws::kPacked) {
        if (lane < 4) {
          const T val = lane == 0 ? a0 : lane == 1 ? a1 : lane == 2 ? a2 : a3;
          st_relaxed_u64(slots + 4 * tk + lane, pack_slot<T>(val));
        }
      } else {
        if (lane == 0) {
          T *d = reinterpret_cast<T *>(slots + 4 * tk);
          d[0] = a0;
          d[1] = a1;
          d[2] = a2;
          d[3] = a3;
          __threadfence();
          st_release_u32(flags + tk, 1u);
        }
      }
    }
  };

  // ------------------------------------------------------------- prologue
  // warp 0 holds the next ticket number in a register, grabbed one iteration
  // before it is staged (the atomic's latency never sits on the critical path)
  unsigned long long tk_next = 0;
  if (tid == 0) {
    prefetch_tmap(&maps.big);
    prefetch_tmap(&maps.small);
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 0) {
    unsigned long long t0 = 0, t1 = 0;
    if (lane == 0) {
      t0 = atomicAdd(counter, 1ull);
      t1 = atomicAdd(counter, 1ull);
    }
    stage_ticket((int64_t)__shfl_sync(0xffffffffu, t0, 0), 0);
    stage_ticket((int64_t)__shfl_sync(0xffffffffu, t1, 0), 1);
  }
  __syncthreads();
  publish(0);

  for (int it = 0;; ++it) {
    const int st = it % NS;
    const int64_t ticket = s_ticket[st];
    if (ticket >= g.total) break;
    // (1) stage ticket it+2 into the stage of ticket it-1 (its readers have all
    //     passed a barrier since), and grab ticket it+3
    if (MM_STAGE_POS == 0 && warp == MM_STAGE_WARP) {
      if (lane == 0) tk_next = atomicAdd(counter, 1ull);
      stage_ticket((int64_t)__shfl_sync(0xffffffffu, tk_next, 0), (it + 2) % NS);
    }
    int64_t row, x;
    decode(ticket, row, x);
    const int64_t u0 = x * TILE;

    // look-back loads for this ticket, issued first; thread s covers
    // x' = x - q + s (H for s == 0 if r > 0, else G)
    const int64_t lb0 = ticket - g.q;
    uint64_t pa = 0, pbv = 0;
    if constexpr (Ws::kPacked) {
      if (x >= 0 && tid < g.q && !(tid == 0 && g.r == 0)) {
        const int k = tid == 0 ? 2 : 0;
        pa = ld_relaxed_u64(slots + 4 * (lb0 + tid) + k);
        pbv = ld_relaxed_u64(slots + 4 * (lb0 + tid) + k + 1);
      }
    }

    // (2) publish ticket it+1 (staged one iteration ago)
    publish(it + 1);
    if (MM_STAGE_POS == 1 && warp == MM_STAGE_WARP) {
      if (lane == 0) tk_next = atomicAdd(counter, 1ull);
      stage_ticket((int64_t)__shfl_sync(0xffffffffu, tk_next, 0), (it + 2) % NS);
    }

    // (3) process ticket it: published last iteration, its stage is complete
    //     and patched
    if (x < 0) {  // publishing-only ticket (uniform)
      // the stage warp wrote s_ticket/s_fshift of ticket it+2 after publish(it+1)'s
      // barrier; publish(it+2) reads them next iteration, so order the write
      // here just as the process step's barrier does for x >= 0
      __syncthreads();
      continue;
    }
    int tout;
    {
      const int64_t left = p.m - u0;
      tout = left < TILE ? (int)left : TILE;
    }
    const int fshift = s_fshift[st];
    T ux[E], un[E];  // become max(P, S) per element
    T cx, cn;        // per-thread constant: carries and gap
    {  // far: prefix scan of F_x
      T v[E];
      lds_swz<T, E>(farb(st), fshift + tid * E, v);
      ux[0] = un[0] = v[0];
#pragma unroll
      for (int k = 1; k < E; ++k) {
        ux[k] = Ord<T>::mx(ux[k - 1], v[k]);
        un[k] = Ord<T>::mn(un[k - 1], v[k]);
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
      if (lane == 0) {  // an element inside every window of the chunk
        cx = ux[0];
        cn = un[0];
      }
      if (lane == 31) {
        wpre[0][warp] = ax;
        wpre[1][warp] = an;
      }
    }
    T nl;  // the near tile's last element: inside every window of the tile
    {  // near: suffix scan of N_x, folded into ux/un
      T v[E];
      lds_swz_aligned<T, E>(nearb(st), tid * E, v);
      nl = lds_one_swz<T>(nearb(st), TILE - 1);
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
      if (lane == 31) {  // an element inside every window of the chunk
        ex = v[E - 1];
        en = v[E - 1];
      }
      cx = Ord<T>::mx(cx, ex);
      cn = Ord<T>::mn(cn, en);
      if (lane == 0) {  // lane 0 holds the warp total
        wsuf[0][warp] = bx;
        wsuf[1][warp] = bn;
      }
    }
    {  // gap M_x from the look-back
      T mx = nl, mn = nl;
      for (int s = tid; s < g.q; s += NT) {
        if (s == 0 && g.r == 0) continue;  // H_{x-q} is empty
        const int k = s == 0 ? 2 : 0;      // slot pair: H or G
        const int64_t src = lb0 + s;
        T vx, vn;
        if constexpr (Ws::kPacked) {
          uint64_t a = pa, b = pbv;
          if (s != tid) {  // q > NT: later rounds load here
            a = ld_relaxed_u64(slots + 4 * src + k);
            b = ld_relaxed_u64(slots + 4 * src + k + 1);
          }
          uint32_t spins = 0;
          while ((a >> 32) == 0) {
            __nanosleep(32);
            a = ld_relaxed_u64(slots + 4 * src + k);
            if (++spins > (1u << 26)) __trap();  // a lost publish must fail, never hang
          }
          while ((b >> 32) == 0) {
            __nanosleep(32);
            b = ld_relaxed_u64(slots + 4 * src + k + 1);
            if (++spins > (1u << 26)) __trap();
          }
          vx = unpack_slot<T>(a);
          vn = unpack_slot<T>(b);
        } else {
          uint32_t spins = 0;
          while (ld_acquire_u32(flags + src) == 0u) {
            __nanosleep(32);
            if (++spins > (1u << 26)) __trap();
          }
          const T *d = reinterpret_cast<const T *>(slots + 4 * src);
          vx = __ldcg(d + k);
          vn = __ldcg(d + k + 1);
        }
        mx = Ord<T>::mx(mx, vx);
        mn = Ord<T>::mn(mn, vn);
      }
#pragma unroll
      for (int d = 16; d >= 1; d >>= 1) {
        mx = Ord<T>::mx(mx, __shfl_xor_sync(0xffffffffu, mx, d));
        mn = Ord<T>::mn(mn, __shfl_xor_sync(0xffffffffu, mn, d));
      }
      if (lane == 0) {
        wgap[0][warp] = mx;
        wgap[1][warp] = mn;
      }
    }
    __syncthreads();  // warp totals of prefix, suffix and gap are in
    for (int v = 0; v < warp; ++v) {  // cross-warp carry of the far prefix
      cx = Ord<T>::mx(cx, wpre[0][v]);
      cn = Ord<T>::mn(cn, wpre[1][v]);
    }
    for (int v = warp + 1; v < NWARP; ++v) {  // cross-warp carry of the suffix
      cx = Ord<T>::mx(cx, wsuf[0][v]);
      cn = Ord<T>::mn(cn, wsuf[1][v]);
    }
#pragma unroll
    for (int v = 0; v < NWARP; ++v) {
      cx = Ord<T>::mx(cx, wgap[0][v]);
      cn = Ord<T>::mn(cn, wgap[1][v]);
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
    // wpre/wsuf/wgap are rewritten next iteration only after that iteration's
    // publish barrier, which every reader here reaches first
  }
}

}  // namespace mm

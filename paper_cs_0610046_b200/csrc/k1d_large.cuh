// k1d_large.cuh -- large-window 1-D kernel with cross-CTA look-back (see k1d_base.cuh).
#pragma once

#include "k1d_base.cuh"

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
// Tickets (atomic counter) order the tiles: ticket = (row, x+q) row-major, so
// the look-back distance is q tiles of the global stream and F_x is still in L2
// when tile x+q stages it as its near tile.  A CTA publishes before it waits and
// waits only on lower tickets; a CTA holding a prefetched next ticket finishes
// its current one (which only waits on lower tickets) first -- deadlock-free for
// any number of resident CTAs.
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
  static constexpr int NROWS = (TILE / RW + kBoxRows - 1) / kBoxRows * kBoxRows;
  static constexpr int FROWS = ((TILE + RW) / RW + kBoxRows - 1) / kBoxRows * kBoxRows;
  static constexpr size_t NB = (size_t)NROWS * 128, FB = (size_t)FROWS * 128;
  static constexpr size_t STAGE = NB + FB;
  static constexpr size_t BYTES = 1024 + 2 * STAGE + 256;
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
    k1d_large(Rows p, LargeGeom g, void *ws, const __grid_constant__ CUtensorMap map) {
  using Lay = LargeLayout<T>;
  using Ws = LargeWs<T>;
  constexpr int E = Lay::E;
  constexpr int TILE = Lay::TILE;
  constexpr int RW = Lay::RW;

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *base = smem_align1024(smem_raw);
  auto nearb = [&](int i) { return base + i * Lay::STAGE; };
  auto farb = [&](int i) { return base + i * Lay::STAGE + Lay::NB; };
  __shared__ T wagg[4][NWARP];
  __shared__ int64_t s_ticket[2];
  __shared__ int s_fshift[2];
  __shared__ __align__(8) uint64_t bars[2];

  unsigned long long *counter = reinterpret_cast<unsigned long long *>(ws);
  uint32_t *flags = reinterpret_cast<uint32_t *>(static_cast<char *>(ws) + 256);  // 8-B types
  uint64_t *slots = reinterpret_cast<uint64_t *>(static_cast<char *>(ws) + Ws::slots_offset(g.total));
  // slot k of ticket t: slots[4t + k], k = 0 Gmax, 1 Gmin, 2 Hmax, 3 Hmin

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
    const int64_t flen = p.n - f0 < TILE ? p.n - f0 : TILE;
    if (p.has_map) {
      const int64_t fr0 = f0 / RW, fr1 = (f0 + flen + RW - 1) / RW;
      const int nfb = (int)((fr1 - fr0 + kBoxRows - 1) / kBoxRows);
      const int nnb = x >= 0 ? (TILE / RW + kBoxRows - 1) / kBoxRows : 0;
      mbar_arrive_expect_tx(&bars[st], (uint32_t)(nfb + nnb) * kBoxBytes);
      for (int k = 0; k < nfb; ++k)
        tma_box(&map, farb(st) + k * kBoxBytes, (int)(fr0 + k * kBoxRows), (int)row, &bars[st]);
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
    stage_ticket((int64_t)atomicAdd(counter, 1ull), 0);
  }
  __syncthreads();

  for (int it = 0;; ++it) {
    const int st = it & 1;
    const int64_t ticket = s_ticket[st];
    if (ticket >= g.total) break;
    if (tid == 0)  // prefetch the next ticket into the other stage
      stage_ticket((int64_t)atomicAdd(counter, 1ull), st ^ 1);
    const int64_t row = ticket / g.tickets_per_row;
    const int64_t x = ticket - row * g.tickets_per_row - g.q;  // may be negative
    const int64_t u0 = x * TILE;
    const int64_t f0 = u0 + w - 1;
    int tout = 0;
    if (x >= 0) {
      const int64_t left = p.m - u0;
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
    T ux[E], un[E];  // become max(P, S) per element
    T hx, hn;
    {
      T v[E];
      lds_swz<T, E>(farb(st), fshift + tid * E, v);
      ux[0] = un[0] = v[0];
#pragma unroll
      for (int k = 1; k < E; ++k) {
        ux[k] = Ord<T>::mx(ux[k - 1], v[k]);
        un[k] = Ord<T>::mn(un[k - 1], v[k]);
      }
      // last r positions of F_x: [TILE - r, TILE); lanes outside borrow the
      // element at TILE-1, which belongs to every non-empty H range
      const int hstart = TILE - g.r;
      hx = hn = lds_one_swz<T>(farb(st), fshift + TILE - 1);
      if (tid * E >= hstart) {
        hx = Ord<T>::mx(hx, ux[E - 1]);
        hn = Ord<T>::mn(hn, un[E - 1]);
      } else if (tid * E + E > hstart) {
        T vx, vn;
        suffix_from<T, E>(v, hstart - tid * E, vx, vn);
        hx = Ord<T>::mx(hx, vx);
        hn = Ord<T>::mn(hn, vn);
      }
    }
    T ax = ux[E - 1], an = un[E - 1];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      T vx = shfl_up(ax, d), vn = shfl_up(an, d);
      if (lane >= d) {
        ax = Ord<T>::mx(ax, vx);
        an = Ord<T>::mn(an, vn);
      }
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {  // warp reduce of the H part
      hx = Ord<T>::mx(hx, __shfl_xor_sync(0xffffffffu, hx, d));
      hn = Ord<T>::mn(hn, __shfl_xor_sync(0xffffffffu, hn, d));
    }
    T cx = shfl_up(ax, 1), cn = shfl_up(an, 1);
    if (lane == 0) {  // an element inside every window of the chunk
      cx = ux[0];
      cn = un[0];
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
      cx = Ord<T>::mx(cx, wagg[0][v]);
      cn = Ord<T>::mn(cn, wagg[1][v]);
    }
    // -------------------------------------------------------------- publish
    if (warp == 0) {
      T gx = wagg[0][lane & (NWARP - 1)], gn = wagg[1][lane & (NWARP - 1)];
      T hhx = wagg[2][lane & (NWARP - 1)], hhn = wagg[3][lane & (NWARP - 1)];
#pragma unroll
      for (int d = NWARP / 2; d >= 1; d >>= 1) {
        gx = Ord<T>::mx(gx, __shfl_xor_sync(0xffffffffu, gx, d));
        gn = Ord<T>::mn(gn, __shfl_xor_sync(0xffffffffu, gn, d));
        hhx = Ord<T>::mx(hhx, __shfl_xor_sync(0xffffffffu, hhx, d));
        hhn = Ord<T>::mn(hhn, __shfl_xor_sync(0xffffffffu, hhn, d));
      }
      if constexpr (Ws::kPacked) {
        if (lane < 4) {
          const T v = lane == 0 ? gx : lane == 1 ? gn : lane == 2 ? hhx : hhn;
          st_relaxed_u64(slots + 4 * ticket + lane, pack_slot<T>(v));
        }
      } else {
        if (lane == 0) {
          T *d = reinterpret_cast<T *>(slots + 4 * ticket);
          d[0] = gx;
          d[1] = gn;
          d[2] = hhx;
          d[3] = hhn;
          __threadfence();
          st_release_u32(flags + ticket, 1u);
        }
      }
    }
    if (x >= 0) {
      // ------------------------------------------ near: CTA suffix scan of N_x
      T bx, bn;
      {
        T v[E];
        lds_swz_aligned<T, E>(nearb(st), tid * E, v);
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
        bx = sx;
        bn = sn;
        // suffix carry from later lanes of the warp
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          T dx = shfl_down(bx, d), dn = shfl_down(bn, d);
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
      }
      // --------------------------------- gap M_x from the look-back, in parallel
      // thread s < q covers x' = x - q + s: H for s == 0 (if r > 0), else G
      // neutral: the near tile's last element lies inside every window of the tile
      T mx = lds_one_swz<T>(nearb(st), TILE - 1), mn = mx;
      for (int s = tid; s < g.q; s += NT) {
        if (s == 0 && g.r == 0) continue;  // H_{x-q} is empty
        const int64_t src = ticket - g.q + s;
        const int k = s == 0 ? 2 : 0;  // slot pair: H or G
        T vx, vn;
        if constexpr (Ws::kPacked) {
          uint64_t a, b;
          uint32_t spins = 0;
          while (((a = ld_relaxed_u64(slots + 4 * src + k)) >> 32) == 0) {
            __nanosleep(32);
            if (++spins > (1u << 26)) __trap();  // a lost publish must fail, never hang
          }
          while (((b = ld_relaxed_u64(slots + 4 * src + k + 1)) >> 32) == 0) {
            __nanosleep(32);
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
      // CTA reduce of the gap, folded into every thread's constant
#pragma unroll
      for (int d = 16; d >= 1; d >>= 1) {
        mx = Ord<T>::mx(mx, __shfl_xor_sync(0xffffffffu, mx, d));
        mn = Ord<T>::mn(mn, __shfl_xor_sync(0xffffffffu, mn, d));
      }
      __syncthreads();  // wagg reuse (prefix aggregates consumed above)
      if (lane == 0) {
        wagg[0][warp] = bx;  // inclusive warp suffix aggregate (lane 0 holds the warp total)
        wagg[1][warp] = bn;
        wagg[2][warp] = mx;
        wagg[3][warp] = mn;
      }
      __syncthreads();
      for (int v = warp + 1; v < NWARP; ++v) {  // cross-warp carry of the suffix
        cx = Ord<T>::mx(cx, wagg[0][v]);
        cn = Ord<T>::mn(cn, wagg[1][v]);
      }
      if (g.q > 1 || g.r > 0) {
        for (int v = 0; v < NWARP; ++v) {
          cx = Ord<T>::mx(cx, wagg[2][v]);
          cn = Ord<T>::mn(cn, wagg[3][v]);
        }
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
    }
    __syncthreads();  // stage st and wagg are free for the next iteration
  }
}

}  // namespace mm

// k2d_byte.cuh -- fused 2-D separable running max-min for 1-byte pixels (u8, i8).
//
// "The unidimensional max-min filter can be applied to images ... by first
// applying the unidimensional on rows and then on columns".
// Rows first, then columns; valid region only (reading R9).  Windows are
// compile-time constants ("compiling w in the code").
//
// Why a separate kernel for bytes: at one byte per pixel the HBM roofline asks
// for ~7.5 pixels per clock per SM, and a scalar min/max per pixel per level
// cannot keep up.  Two pixels therefore travel in one 32-bit register as the
// HIGH bytes of its two 16-bit lanes, and every max/min is one packed
// VIMNMX(3).U16x2 instruction (full issue rate on sm_100a, measured by
// tools/micro/pipes.cu; ptxas fuses max(max(a,b),c) into the 3-input form).
// Only the high byte of a lane is ever read back, so the low byte may hold
// anything: for lanes 256p+g, max/min order them by p first, and the winner's
// high byte is max/min p whatever g is.  Two consequences:
//   * a raw word [c0 c1 c2 c3] of one row IS a packed word of pixels c1, c3
//     ("O"), and (word << 8) one of c0, c2 ("Ev") -- no unpacking at all for
//     ops between rows (the column pass);
//   * for ops within a row (the row pass) a word pairs the same column of two
//     rows: one PRMT makes it from the two rows' raw words.
//
// Every window is a 3-input sparse table (Plan below): level k+1 of span
// s' <= 3s is max3(M_s[j], M_s[j+d], M_s[j+s'-s]); max/min are idempotent, so
// overlaps are harmless.  For w=15: spans 1 -> 3 -> 9 -> 15, three ops per
// output and filter instead of vHGW's three two-input ops plus halo scans.
//
// Work split: a CTA owns a vertical strip of TW=1024 output columns and a
// contiguous range of output rows (the linearised (image, strip, row) space is
// cut evenly over the persistent grid, so the column halo of w_col-1 rows is
// paid once per range, not per tile).  Input rows stream through a 2-stage ring
// of RB-row stages, each staged by one bulk copy per row (cp.async.bulk,
// mbarrier completion).  Per stage:
//   row pass   : thread item = (row pair, 16 output columns); 2 x (16+wr-1)
//                bytes from shared memory -> paired words -> sparse table ->
//                row max / row min bytes into a double-buffered intermediate;
//   barrier    : (the input stage is free: thread 0 issues stage +2)
//   column pass: thread = 4 adjacent columns, streaming down the rows with the
//                sparse-table levels kept in registers across stages (a ring
//                realised by unrolling the RB rows of a stage); results
//                overwrite the intermediate in place;
//   barrier    : one warp sends every valid output row of the stage to HBM as
//                a bulk copy shared -> global (cp.async.bulk, 1 KB per row and
//                filter), so no thread spends instructions on global addresses.
// Signed bytes are biased by 0x80 on the way in and out (order-preserving).
#pragma once

#include "common.cuh"

namespace mm {
namespace k2b {

constexpr int NTB = 256;   // threads per CTA: warps 0-3 row pass, warps 4-7 column pass
constexpr int NRT = 128;   // row-pass threads
constexpr int NCT = 128;   // column-pass threads
constexpr int TW = 4 * NCT;  // output columns per strip = 4 per column thread
constexpr int RB = 16;     // input rows per stage
constexpr int NSTG = 3;    // input stages (bulk-copy ring)
constexpr int NMID = 3;    // intermediate buffers (row pass -> column pass ring)
constexpr int ER = 32;     // output columns per row-pass item
constexpr int MAXW = 17;   // largest compiled window (either direction)
static_assert((RB / 2) * (TW / ER) == NRT, "one row-pass item per row thread and stage");

// named barriers (0 is __syncthreads)
constexpr int kBarFull = 1;               // + m: intermediate m written   (row arrive, column sync)
constexpr int kBarEmpty = kBarFull + NMID;  // + m: intermediate m released (column warp arrive, row sync)
constexpr int kBarRow = kBarEmpty + NMID;   // row threads among themselves
constexpr int kBarCol = kBarRow + 1;        // column threads among themselves

struct Plan {
  int K;     // levels above the input
  int s[8];  // span of level k (s[0] = 1, s[K] = W)
  int d[8];  // middle offset used to build level k+1
};
__host__ __device__ constexpr Plan make_plan(int W) {
  Plan p{};
  p.K = 0;
  p.s[0] = 1;
  while (p.s[p.K] < W) {
    const int s = p.s[p.K];
    const int s2 = 3 * s < W ? 3 * s : W;
    p.d[p.K] = (s2 - s) / 2;  // any d in [s2-2s, s] covers [j, j+s2)
    p.s[p.K + 1] = s2;
    ++p.K;
  }
  return p;
}

__host__ __device__ constexpr int plan_K(int W) { return make_plan(W).K; }
__host__ __device__ constexpr int plan_s(int W, int k) { return make_plan(W).s[k]; }
__host__ __device__ constexpr int plan_d(int W, int k) { return make_plan(W).d[k]; }

// Shared-memory tiles are TMA boxes: 256 columns x RB rows, row-major, so one
// stage of input is two such boxes plus a 16-column tail box (the row halo,
// wr-1 <= 16 columns), and one filter's intermediate/output is two boxes.
constexpr int BOXW = 256;
constexpr int TAILW = 16;
constexpr int BOX = BOXW * RB;                      // bytes of a 256-wide box
constexpr int STAGE_IN = 2 * BOX + TAILW * RB;      // input stage bytes
static_assert(TW == 2 * BOXW, "a strip is two boxes wide");

template <int WR>
struct RowGeo {
  static constexpr int L = ER + WR - 1;          // input columns of an item
  static constexpr int NCH = (L + 15) / 16;      // 16-B chunks read per row
  static_assert(WR - 1 <= TAILW, "row halo must fit the tail box");
  static_assert(TW - ER + 16 * NCH <= TW + TAILW, "item reads stay inside the stage");
};

template <int WR>
struct Smem {
  static constexpr size_t IN = STAGE_IN;  // one input stage
  static constexpr size_t MID = 2 * BOX;  // one filter's intermediate (two boxes)
  static constexpr size_t BYTES = 1024 + NSTG * IN + NMID * 2 * MID + 64;
};

// byte offset of column c (a multiple of 16, c < TW + TAILW) of stage row r
__device__ __forceinline__ int in_off(int c, int r) {
  return c < TW ? (c >> 8) * BOX + r * BOXW + (c & (BOXW - 1)) : 2 * BOX + r * TAILW + (c - TW);
}
// byte offset of column c (< TW) of row r in a filter's intermediate
__device__ __forceinline__ int mid_off(int c, int r) { return (c >> 8) * BOX + r * BOXW + (c & (BOXW - 1)); }

struct Maps {
  CUtensorMap in_box, in_tail;     // input {cols, rows, batch}: boxes {256, RB, 1} and {16, RB, 1}
  CUtensorMap omx, omx1, omn, omn1;  // outputs {Co16, Ro, batch}: boxes {256, RB, 1} and {256, 1, 1}
};

struct Args {
  const uint8_t *in;
  uint8_t *out_max, *out_min;
  int64_t batch, rows, cols, in_ld, in_bstride, out_ld, out_bstride;
  int64_t Ro, Co;     // valid output extent
  int64_t Co16;       // Co rounded down to 16 (the TMA-stored columns)
  int64_t nstrip;     // strips per image
  int64_t units;      // batch * nstrip * Ro
};

// packed 16x2 max/min (the 3-input form is formed by ptxas)
__device__ __forceinline__ uint32_t vmx(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("max.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t vmn(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("min.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
template <bool MAX>
__device__ __forceinline__ uint32_t op3(uint32_t a, uint32_t b, uint32_t c) {
  return MAX ? vmx(vmx(a, b), c) : vmn(vmn(a, b), c);
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
// bulk copy shared -> global (bulk-group completion), and its group waits
__device__ __forceinline__ void bulk_s2g(void *g, const void *s, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g),
               "r"(smem_u32(s)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void tma_load3(const CUtensorMap *m, void *dst, int c, int r, int b,
                                          uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c), "r"(r), "r"(b), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store3(const CUtensorMap *m, const void *src, int c, int r, int b) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c), "r"(r), "r"(b), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_wait_read_1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Row pass of one item: y[i] = op over x[i .. i+W) for i < ER, computed in
// place level by level (descending j keeps the lower level readable).
// Arrival indexing: after level k, A[j] = op over x[j-s_k+1 .. j].
template <int W, bool MAX, int L, int k = 0>
__device__ __forceinline__ void sparse_row(uint32_t (&A)[L]) {
  if constexpr (k < plan_K(W)) {
    constexpr int s1 = plan_s(W, k + 1), a = s1 - plan_s(W, k), d = plan_d(W, k);
#pragma unroll
    for (int j = L - 1; j >= s1 - 1; --j) A[j] = op3<MAX>(A[j - a], A[j - a + d], A[j]);
    sparse_row<W, MAX, L, k + 1>(A);
  }
}

// Streaming column filter state for one packed word stream: the histories of
// levels 0..K-1 (H_k = s_{k+1} - s_k values each), oldest first.
template <int W>
struct ColRing {
  static constexpr int HT = W - 1 > 0 ? W - 1 : 1;  // sum of histories = W - 1
  uint32_t h[HT];
};

// Feed one new value A_0[t]; returns A_K[t] = op over the last W values (valid
// once W values have been fed since the start of a range).
template <int W, bool MAX, int k = 0>
__device__ __forceinline__ uint32_t ring_push(ColRing<W> &r, uint32_t cur) {
  if constexpr (k < plan_K(W)) {
    constexpr int a = plan_s(W, k + 1) - plan_s(W, k), d = plan_d(W, k);  // 0 <= d < a
    constexpr int o = plan_s(W, k) - 1;  // level k's history: h[o .. o+a) = A_k[t-a .. t-1]
    // A_{k+1}[t] = op(A_k[t-a], A_k[t-a+d], A_k[t])
    const uint32_t nxt = op3<MAX>(r.h[o], r.h[o + d], cur);
    // shift the history and append A_k[t] (register renaming once the stage's
    // rows are unrolled; moves only at the stage loop's back edge)
#pragma unroll
    for (int i = 0; i + 1 < a; ++i) r.h[o + i] = r.h[o + i + 1];
    r.h[o + a - 1] = cur;
    return ring_push<W, MAX, k + 1>(r, nxt);
  } else {
    return cur;
  }
}

template <bool SIGNED, int WR, int WC>
__global__ void __launch_bounds__(NTB, 2) k2d_byte(Args p, const __grid_constant__ Maps maps) {
  using G = RowGeo<WR>;
  using S = Smem<WR>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *base = smem_align1024(smem_raw);
  unsigned char *stage_in = base;          // [NSTG][RB][IW]
  unsigned char *mid = base + NSTG * S::IN;  // [NMID][2 filters][RB][TW]
  uint64_t *bars = reinterpret_cast<uint64_t *>(mid + NMID * 2 * S::MID);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr uint32_t FLIP = SIGNED ? 0x80808080u : 0u;

  // this CTA's slice of the linearised (image, strip, output row) space
  const int64_t G_ = gridDim.x;
  const int64_t u_begin = p.units * (int64_t)blockIdx.x / G_;
  const int64_t u_end = p.units * ((int64_t)blockIdx.x + 1) / G_;
  if (u_begin >= u_end) return;

  if (tid == 0) {
    for (int s = 0; s < NSTG; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();  // the only CTA-wide barrier: the roles split below

  // A cursor over (piece, stage) pairs; a piece is a run of output rows of one
  // strip.  Input rows of a piece: [o0, o1 + WC - 1).
  struct Cursor {
    int64_t u;       // first unit of the current piece
    int64_t o0, o1;  // output rows of the piece
    int64_t nin;     // input rows of the piece
    int64_t st;      // stage index within the piece
    int64_t b, c0;   // image, first column of the strip
  };
  auto open = [&](Cursor &c, int64_t u) {
    c.u = u;
    const int64_t bs = u / p.Ro;  // image * nstrip + strip
    c.o0 = u - bs * p.Ro;
    const int64_t left = u_end - u;
    c.o1 = c.o0 + (p.Ro - c.o0 < left ? p.Ro - c.o0 : left);
    c.nin = c.o1 - c.o0 + WC - 1;
    c.st = 0;
    c.b = bs / p.nstrip;
    c.c0 = (bs - c.b * p.nstrip) * TW;
  };
  auto advance = [&](Cursor &c) -> bool {  // false when the CTA's range is done
    ++c.st;
    if (c.st * RB < c.nin) return true;
    const int64_t nu = c.u + (c.o1 - c.o0);
    if (nu >= u_end) return false;
    open(c, nu);
    return true;
  };
  int64_t nstages = 0;  // stages of the whole range (a handful of pieces)
  {
    Cursor c;
    open(c, u_begin);
    for (;;) {
      nstages += (c.nin + RB - 1) / RB;
      const int64_t nu = c.u + (c.o1 - c.o0);
      if (nu >= u_end) break;
      open(c, nu);
    }
  }

  if (warp < NRT / 32) {
    // ================================================= row-pass warps (0-3)
    Cursor ld;  // loader cursor (warp 0)
    open(ld, u_begin);
    bool ld_live = true;
    int64_t ld_gs = 0;
    auto issue = [&]() {  // warp 0, lane 0: stage ld_gs = three TMA boxes
      const int buf = (int)(ld_gs % NSTG);
      if (lane == 0) {
        unsigned char *dst = stage_in + buf * S::IN;
        const int r0 = (int)(ld.o0 + ld.st * RB), c0 = (int)ld.c0, b = (int)ld.b;
        mbar_arrive_expect_tx(&bars[buf], (uint32_t)STAGE_IN);  // OOB parts are zero-filled
        tma_load3(&maps.in_box, dst, c0, r0, b, &bars[buf]);
        tma_load3(&maps.in_box, dst + BOX, c0 + BOXW, r0, b, &bars[buf]);
        tma_load3(&maps.in_tail, dst + 2 * BOX, c0 + TW, r0, b, &bars[buf]);
      }
      ++ld_gs;
      ld_live = advance(ld);
    };
    if (warp == 0) {
      if (lane == 0) {
        prefetch_tmap(&maps.in_box);
        prefetch_tmap(&maps.in_tail);
      }
      for (int k = 0; k < NSTG && ld_live; ++k) issue();
    }
    Cursor cs;
    open(cs, u_begin);
    const int pr = tid / (TW / ER), g = tid - pr * (TW / ER);  // this thread's item
    for (int64_t gs = 0;; ++gs) {
      const int buf = (int)(gs % NSTG);
      const int mb = (int)(gs % NMID);
      mbar_wait(&bars[buf], (uint32_t)((gs / NSTG) & 1));
      if (gs >= NMID) bar_sync(kBarEmpty + mb, NRT + 32);  // column side released mid[mb]
      const unsigned char *sb = stage_in + buf * S::IN;
      uint32_t x[G::L], y[G::L];
      {
        uint32_t ra[4 * G::NCH], rb[4 * G::NCH];
#pragma unroll
        for (int c = 0; c < G::NCH; ++c) {
          const uint4 va = *reinterpret_cast<const uint4 *>(sb + in_off(g * ER + 16 * c, 2 * pr));
          const uint4 vb = *reinterpret_cast<const uint4 *>(sb + in_off(g * ER + 16 * c, 2 * pr + 1));
          ra[4 * c] = va.x ^ FLIP, ra[4 * c + 1] = va.y ^ FLIP, ra[4 * c + 2] = va.z ^ FLIP,
          ra[4 * c + 3] = va.w ^ FLIP;
          rb[4 * c] = vb.x ^ FLIP, rb[4 * c + 1] = vb.y ^ FLIP, rb[4 * c + 2] = vb.z ^ FLIP,
          rb[4 * c + 3] = vb.w ^ FLIP;
        }
#pragma unroll
        for (int j = 0; j < G::L; ++j) {  // word j: column j of row A (lane 0) and row B (lane 1)
          x[j] = prmt(ra[j >> 2], rb[j >> 2], 0x4400u + 0x1111u * (uint32_t)(j & 3));
          y[j] = x[j];
        }
      }
      sparse_row<WR, true>(x);
      sparse_row<WR, false>(y);
      // column i of the item is A[i + WR - 1]; 4 words -> a row-A and a row-B word
      unsigned char *mx_mid = mid + (size_t)(2 * mb) * S::MID;
      unsigned char *mn_mid = mx_mid + S::MID;
      const int oa = mid_off(g * ER, 2 * pr), ob = mid_off(g * ER, 2 * pr + 1);
#pragma unroll
      for (int h = 0; h < ER / 16; ++h) {  // 16 columns -> one 16-B store per row and filter
        uint32_t oxa[4], oxb[4], ona[4], onb[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = 16 * h + 4 * q + WR - 1;
          uint32_t P = prmt(x[j], x[j + 1], 0x7351u), Q = prmt(x[j + 2], x[j + 3], 0x7351u);
          oxa[q] = prmt(P, Q, 0x5410u);
          oxb[q] = prmt(P, Q, 0x7632u);
          P = prmt(y[j], y[j + 1], 0x7351u), Q = prmt(y[j + 2], y[j + 3], 0x7351u);
          ona[q] = prmt(P, Q, 0x5410u);
          onb[q] = prmt(P, Q, 0x7632u);
        }
        *reinterpret_cast<uint4 *>(mx_mid + oa + 16 * h) = make_uint4(oxa[0], oxa[1], oxa[2], oxa[3]);
        *reinterpret_cast<uint4 *>(mx_mid + ob + 16 * h) = make_uint4(oxb[0], oxb[1], oxb[2], oxb[3]);
        *reinterpret_cast<uint4 *>(mn_mid + oa + 16 * h) = make_uint4(ona[0], ona[1], ona[2], ona[3]);
        *reinterpret_cast<uint4 *>(mn_mid + ob + 16 * h) = make_uint4(onb[0], onb[1], onb[2], onb[3]);
      }
      bar_arrive(kBarFull + mb, NTB);  // hand mid[mb] to the column warps
      bar_sync(kBarRow, NRT);          // every row thread is done with input stage `buf`
      if (warp == 0 && ld_live) issue();
      if (!advance(cs)) break;
    }
  } else {
    // ============================================== column-pass warps (4-7)
    const int ct = tid - NRT;  // 4 columns: [4ct, 4ct+4) of the strip
    Cursor cs;
    open(cs, u_begin);
    ColRing<WC> rxo, rxe, rno, rne;  // rings: max/min x odd/even columns
#pragma unroll
    for (int i = 0; i < ColRing<WC>::HT; ++i) rxo.h[i] = rxe.h[i] = rno.h[i] = rne.h[i] = 0;
    for (int64_t gs = 0;; ++gs) {
      const int mb = (int)(gs % NMID);
      unsigned char *mx_mid = mid + (size_t)(2 * mb) * S::MID;
      unsigned char *mn_mid = mx_mid + S::MID;
      bar_sync(kBarFull + mb, NTB);  // row pass of this stage is in mid[mb]
      {
        // results overwrite the intermediate in place (each thread rewrites
        // the 4 bytes it just read) and leave by bulk copies shared -> global
        unsigned char *px = mx_mid + mid_off(4 * ct, 0), *pn = mn_mid + mid_off(4 * ct, 0);
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          const uint32_t vx = *reinterpret_cast<const uint32_t *>(px + r * BOXW);
          const uint32_t vn = *reinterpret_cast<const uint32_t *>(pn + r * BOXW);
          const uint32_t xo = ring_push<WC, true>(rxo, vx);
          const uint32_t xe = ring_push<WC, true>(rxe, vx << 8);
          const uint32_t no = ring_push<WC, false>(rno, vn);
          const uint32_t ne = ring_push<WC, false>(rne, vn << 8);
          *reinterpret_cast<uint32_t *>(px + r * BOXW) = prmt(xe, xo, 0x7351u) ^ FLIP;
          *reinterpret_cast<uint32_t *>(pn + r * BOXW) = prmt(ne, no, 0x7351u) ^ FLIP;
        }
      }
      fence_proxy_async_smem();  // generic-proxy writes -> visible to the bulk copies
      bar_sync(kBarCol, NCT);    // the stage's outputs are complete in mid[mb]
      const int64_t t0 = cs.st * RB;  // piece-relative input row of stage row 0
      // stage row r holds output row orow0 + r, valid for r in [r_lo, r_hi)
      const int r_lo = t0 >= WC - 1 ? 0 : (int)(WC - 1 - t0);
      const int r_hi = cs.nin - t0 < RB ? (int)(cs.nin - t0) : RB;
      const int64_t orow0 = cs.o0 + t0 - (WC - 1);
      if (warp == NRT / 32) {
        if (lane == 0) {  // TMA stores clip at the image's right and bottom edges
          const int b = (int)cs.b;
          for (int f = 0; f < 2; ++f) {
            if (!(f ? p.out_min : p.out_max)) continue;
            const CUtensorMap *m16 = f ? &maps.omn : &maps.omx;
            const CUtensorMap *m1 = f ? &maps.omn1 : &maps.omx1;
            const unsigned char *src = f ? mn_mid : mx_mid;
            for (int h = 0; h < 2; ++h) {
              const int c = (int)cs.c0 + h * BOXW;
              if (c >= p.Co16) break;
              if (r_lo == 0 && r_hi == RB) {
                tma_store3(m16, src + h * BOX, c, (int)orow0, b);
              } else {
                for (int r = r_lo; r < r_hi; ++r)
                  tma_store3(m1, src + h * BOX + r * BOXW, c, (int)(orow0 + r), b);
              }
            }
          }
          bulk_commit();
          if (gs >= 1) bulk_wait_read_1();  // the previous stage's stores have read their buffer
        }
        __syncwarp();
        // release it -- only if the row warps will wait for it (stage gs-1+NMID exists)
        if (gs >= 1 && gs - 1 + NMID < nstages) bar_arrive(kBarEmpty + (int)((gs - 1) % NMID), NRT + 32);
      }
      // TMA clips the innermost dimension in 16-byte units, so the maps end at
      // Co16 = 16*floor(Co/16) and the last < 16 columns go out as plain stores
      if (p.Co16 < p.Co && cs.c0 <= p.Co16 && p.Co16 < cs.c0 + TW) {
        const int k = ct & 15;
        const int64_t c = p.Co16 + k;
        if (c < p.Co) {
          const int cl = (int)(c - cs.c0);
          for (int r = (ct >> 4) + r_lo; r < r_hi; r += NCT / 16) {
            const int64_t go = cs.b * p.out_bstride + (orow0 + r) * p.out_ld + c;
            if (p.out_max) p.out_max[go] = mx_mid[mid_off(cl & ~15, r) + (cl & 15)];
            if (p.out_min) p.out_min[go] = mn_mid[mid_off(cl & ~15, r) + (cl & 15)];
          }
        }
      }
      if (!advance(cs)) break;
    }
    if (warp == NRT / 32 && lane == 0) bulk_wait_all();  // shared memory must outlive the stores
  }
}

}  // namespace k2b
}  // namespace mm

// k2d_byte.cuh -- fused 2-D separable running max-min for 1-byte pixels (u8, i8).
//
// "The unidimensional max-min filter can be applied to images ... by first
// applying the unidimensional on rows and then on columns".
// Rows first, then columns; valid region only (reading R9).  Windows are
// compile-time constants ("compiling w in the code").
//
// Packed arithmetic.  At one byte per pixel the HBM roofline asks for ~7.5
// pixels per clock per SM, so two pixels travel in one 32-bit register as the
// HIGH bytes of its two 16-bit lanes and every max/min is one packed
// VIMNMX3.U16x2 (ptxas fuses max(max(a,b),c) into the 3-input form; the ALU
// pipe issues 64 of them per clock per SM, tools/micro/pipes.cu).  Only the
// high byte of a lane is ever read back, so the low byte may hold anything:
// for lanes 256p+g, max/min order them by p first, and the winner's high byte
// is max/min p whatever g is.  Hence
//   * a raw word [c0 c1 c2 c3] of one row IS a packed word of pixels c1, c3
//     ("O"), and (word << 8) one of c0, c2 ("Ev") -- no unpacking for ops
//     between rows (the column pass);
//   * for ops within a row (the row pass) a word pairs the same column of two
//     rows: one PRMT makes it from the two rows' raw words.
//
// Every window is a 3-input sparse table (Plan below): level k+1 of span
// s' <= 3s is max3(M_s[j], M_s[j+d], M_s[j+s'-s]); max/min are idempotent, so
// overlaps are harmless.  For w=15: spans 1 -> 3 -> 9 -> 15, i.e. three ops per
// output and filter (plus an 18-op halo per 32-column row item).
//
// Work split.  Tiles are (image, band of BH output rows, strip of TW=512
// output columns), strip fastest, dealt round-robin to a persistent grid, so
// the resident CTAs work on neighbouring strips of the same bands and their
// DRAM traffic covers whole image rows.  A CTA is warp-specialised:
//   warps 0-3 (row pass): input rows arrive by TMA in stages of RB=16 rows x
//     528 columns (three 176-column boxes: the 176-byte row pitch skews
//     consecutive rows across shared-memory banks); thread = (row pair
//     (r, r+8), 32 output columns); 2 x 46 bytes -> paired words -> sparse
//     table -> row-max / row-min bytes into an intermediate ring (pitch 528:
//     again bank-skewed);
//   warps 4-7 (column pass): thread = 4 adjacent columns, streaming down the
//     rows with the sparse-table levels of the column window kept in
//     registers across stages (a ring realised by unrolling a stage's rows);
//     one coalesced 4-byte store per row and filter (a warp writes 128
//     contiguous bytes).
// The two sides hand intermediate buffers over with named barriers
// (FULL: row side arrives, column side waits; EMPTY: the reverse), NMID deep.
// Signed bytes are biased by 0x80 on the way in and out (order-preserving).
#pragma once

#include "common.cuh"

namespace mm {
namespace k2b {

#ifndef MM_K2B_FMA_UNPACK
#define MM_K2B_FMA_UNPACK 0
#endif
#ifndef MM_K2B_ROW_VHGW
#define MM_K2B_ROW_VHGW 1
#endif
#ifndef MM_K2B_NSTG
#define MM_K2B_NSTG 3
#endif
#ifndef MM_K2B_NMID
#define MM_K2B_NMID 4
#endif

constexpr int NTB = 256;      // threads per CTA
constexpr int NRT = 128;      // row-pass threads (warps 0-3)
constexpr int NCT = 128;      // column-pass threads (warps 4-7)
constexpr int TW = 4 * NCT;   // output columns per strip = 4 per column thread
constexpr int RB = 16;        // input rows per stage
constexpr int ER = 32;        // output columns per row-pass item
constexpr int NSTG = MM_K2B_NSTG;  // input stages (TMA ring)
constexpr int NMID = MM_K2B_NMID;  // intermediate buffers (row pass -> column pass)
constexpr int MAXW = 17;      // largest compiled window (either direction)
constexpr int HALO = 16;      // input columns beyond the strip (>= w_row - 1)
constexpr int INW = TW + HALO;             // input columns per stage row: 528
constexpr int BOXW = INW / 3;              // TMA box width: 176 bytes
constexpr int INBOX = BOXW * RB;           // bytes of one input box
constexpr int STAGE_IN = 3 * INBOX;        // input stage bytes
constexpr int MP = INW;                    // intermediate row pitch (528 = 16 mod 128)
constexpr int MID = MP * RB;               // one filter's intermediate
static_assert((RB / 2) * (TW / ER) == NRT, "one row-pass item per row thread and stage");
static_assert(BOXW % 16 == 0 && 3 * BOXW == INW, "three 16-byte-aligned boxes per stage row");

// named barriers (0 is __syncthreads)
constexpr int kBarFull = 1;                 // + m: intermediate m written  (row arrive, column sync)
constexpr int kBarEmpty = kBarFull + NMID;  // + m: intermediate m consumed (column arrive, row sync)
constexpr int kBarRow = kBarEmpty + NMID;   // row threads among themselves
static_assert(kBarRow < 16, "16 hardware barriers per CTA");

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

template <int WR>
struct RowGeo {
  static constexpr int L = ER + WR - 1;      // input columns of an item
  static constexpr int NCH = (L + 15) / 16;  // 16-B chunks read per row
  static_assert(WR - 1 <= HALO, "row halo must fit the stage");
  static_assert(TW - ER + 16 * NCH <= INW, "item reads stay inside the stage");
};

struct Smem {
  static constexpr size_t BYTES = 1024 + (size_t)NSTG * STAGE_IN + (size_t)NMID * 2 * MID + 64;
};

// byte offset of input column c (a multiple of 16) of stage row r
__host__ __device__ constexpr int in_off(int c, int r) { return (c / BOXW) * INBOX + r * BOXW + c % BOXW; }

struct Args {
  uint8_t *out_max, *out_min;
  int64_t batch, rows, cols, out_ld, out_bstride;
  int64_t Ro, Co;     // valid output extent
  int64_t nstrip;     // strips per image
  int64_t BH;         // output rows per band (a tile is one band of one strip)
  int64_t nbands;     // bands per image
  int64_t ntiles;     // batch * nbands * nstrip
  uint32_t one, k8, k16, k24;  // 1, 1 << 8, 1 << 16, 1 << 24 (opaque to the compiler)
  int in_r0;  // input row of output row 0's first window row: 0, or -(w-1) for a framed input (morphology)
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
// p + one * step with `one` a register equal to 1 that the compiler cannot see
// through: one IMAD.WIDE.U32 on the FMA pipe, where a plain 64-bit pointer
// add takes two ALU-pipe instructions (the pipe the packed min/max saturate)
__device__ __forceinline__ uint8_t *ptr_step(uint8_t *p, uint32_t one, uint32_t step) {
  uint64_t a;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(a) : "r"(one), "r"(step), "l"(reinterpret_cast<uint64_t>(p)));
  return reinterpret_cast<uint8_t *>(a);
}
__device__ __forceinline__ uint32_t umulhi(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t umul(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("mul.lo.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t umad(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
__device__ __forceinline__ void st_u32(uint8_t *p, uint32_t v) {
  asm volatile("st.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void tma_load3(const CUtensorMap *m, void *dst, int c, int r, int b,
                                          uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c), "r"(r), "r"(b), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
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

// Row pass of one item, van Herk / Gil-Werman style with a 3-input combine:
// blocks of B = (W+1)/2 columns anchored at the item start, h = suffix within
// a block, g = prefix within a block.  A window [j, j+W) spans two or three
// blocks (W <= 2B+1), so out[j] = op(h[j], g[j+W-1]) or op3(h[j], M, g[j+W-1])
// with M = h at the start of the middle block (the whole middle block).  About
// (2(B-1)/B + 1) ops per output: 93 per filter for W=15 and 32 outputs, against
// 114 for the sparse table.  Unneeded h/g values are dead code after unrolling.
template <int W, bool MAX, int L, int E>
__device__ __forceinline__ void vhgw_row(const uint32_t (&x)[L], uint32_t (&out)[E]) {
  constexpr int B = (W + 1) / 2;
  static_assert(W > B && W <= 2 * B + 1, "a window spans two or three blocks");
  uint32_t h[L], g[L];
#pragma unroll
  for (int j = L - 1; j >= 0; --j)
    h[j] = (j % B == B - 1 || j == L - 1) ? x[j] : (MAX ? vmx(x[j], h[j + 1]) : vmn(x[j], h[j + 1]));
#pragma unroll
  for (int k = 0; k < L; ++k) g[k] = (k % B == 0) ? x[k] : (MAX ? vmx(g[k - 1], x[k]) : vmn(g[k - 1], x[k]));
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const int e = j + W - 1, bj = j / B, be = e / B;
    if (be == bj + 1)
      out[j] = MAX ? vmx(h[j], g[e]) : vmn(h[j], g[e]);
    else
      out[j] = op3<MAX>(h[j], h[(bj + 1) * B], g[e]);
  }
}

// Streaming column filter state for one packed word stream: the histories of
// levels 0..K-1 (s_{k+1} - s_k values each, oldest first; they telescope to
// W - 1 values in all).
template <int W>
struct ColRing {
  static constexpr int HT = W - 1 > 0 ? W - 1 : 1;
  uint32_t h[HT];
};

// Feed one new value A_0[t]; returns A_K[t] = op over the last W values (valid
// once W values have been fed since the start of a tile).
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

// FIN: XOR applied to every input byte (0x80 maps i8 to an order-preserving u8);
// FXO / FNO: XOR applied to the max / min output bytes.  FRAMED: the input is
// read through a (w-1)-wide zero frame on every side and only the max filter is
// computed (the min chain, its intermediate and its stores are compiled out):
// output (r, c) is the max over input rows [r-w+1, r] x columns [c-w+1, c].
// Row coordinates of the frame are negative tensor-map coordinates; columns
// start 16 bytes before the strip (a TMA box's inner start must be 16-B
// aligned), and the row pass reads every item D = 17 - w bytes further in.
// The plain filter is <0,0,0> (u8) or <0x80,0x80,0x80> (i8); the morphology
// passes use the others (launch_morph_2d_byte).
template <uint32_t FIN, uint32_t FXO, uint32_t FNO, bool FRAMED, int WR, int WC>
__global__ void __launch_bounds__(NTB, 2) k2d_byte(Args p, const __grid_constant__ CUtensorMap in_map) {
  using G = RowGeo<WR>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *base = smem_align1024(smem_raw);
  unsigned char *stage_in = base;                // [NSTG][3 boxes][RB][BOXW]
  unsigned char *mid = base + NSTG * STAGE_IN;   // [NMID][2 filters][RB][MP]
  uint64_t *bars = reinterpret_cast<uint64_t *>(mid + NMID * 2 * MID);
  const int tid = threadIdx.x, warp = tid >> 5;
  constexpr uint32_t FLIP = FIN * 0x01010101u, XOUT = FXO * 0x01010101u, NOUT = FNO * 0x01010101u;

  const int64_t G_ = gridDim.x;
  if ((int64_t)blockIdx.x >= p.ntiles) return;
  uint32_t *smem_one = reinterpret_cast<uint32_t *>(bars + NSTG);
  if (tid == 0) {
    for (int s = 0; s < NSTG; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    *smem_one = p.one;
  }
  __syncthreads();  // the only CTA-wide barrier: the roles split below

  // A cursor over (tile, stage) pairs.  Input rows of a tile: [o0, o1 + WC - 1).
  struct Cursor {
    int64_t u;       // tile index
    int64_t o0, o1;  // output rows of the tile
    int64_t nin;     // input rows of the tile
    int64_t st;      // stage index within the tile
    int64_t b, c0;   // image, first column of the strip
  };
  const int64_t per_img = p.nbands * p.nstrip;
  auto open = [&](Cursor &c, int64_t u) {
    c.u = u;
    c.b = u / per_img;
    const int64_t rem = u - c.b * per_img;
    const int64_t band = rem / p.nstrip;
    c.c0 = (rem - band * p.nstrip) * TW;
    c.o0 = band * p.BH;
    c.o1 = c.o0 + (p.Ro - c.o0 < p.BH ? p.Ro - c.o0 : p.BH);
    c.nin = c.o1 - c.o0 + WC - 1;
    c.st = 0;
  };
  auto advance = [&](Cursor &c) {  // next stage (of this tile or the CTA's next tile)
    ++c.st;
    if (c.st * RB < c.nin) return;
    if (c.u + G_ < p.ntiles) open(c, c.u + G_);
  };
  int64_t nstages = 0;  // stages of all this CTA's tiles
  for (int64_t u = blockIdx.x; u < p.ntiles; u += G_) {
    const int64_t o0 = ((u % per_img) / p.nstrip) * p.BH;
    const int64_t nin = (p.Ro - o0 < p.BH ? p.Ro - o0 : p.BH) + WC - 1;
    nstages += (nin + RB - 1) / RB;
  }

  if (warp < NRT / 32) {
    // ================================================= row-pass warps (0-3)
    Cursor ld;  // loader cursor (thread 0)
    open(ld, (int64_t)blockIdx.x);
    int64_t ld_next = 0;  // next stage to load
    int ld_buf = 0;
    auto issue = [&]() {  // three TMA boxes of 176 columns x RB rows
      unsigned char *dst = stage_in + ld_buf * STAGE_IN;
      const int r0 = (int)(ld.o0 + ld.st * RB) + p.in_r0, c0 = (int)ld.c0 - (FRAMED ? 16 : 0), b = (int)ld.b;
      mbar_arrive_expect_tx(&bars[ld_buf], (uint32_t)STAGE_IN);  // OOB parts are zero-filled
#pragma unroll
      for (int k = 0; k < 3; ++k) tma_load3(&in_map, dst + k * INBOX, c0 + k * BOXW, r0, b, &bars[ld_buf]);
      if (++ld_buf == NSTG) ld_buf = 0;
      ++ld_next;
      advance(ld);
    };
    if (tid == 0) {
      prefetch_tmap(&in_map);
      while (ld_next < NSTG && ld_next < nstages) issue();
    }
    // this thread's item: rows (pr, pr + 8) of a stage, output columns
    // [32g, 32g + 32) of the strip; lanes pr = 0..7 of a quarter-warp touch 8
    // different rows, which the 176/528-byte pitches spread over all banks
    const int pr = tid & 7, g = tid >> 3;
    // framed input: the stage starts 16 columns before the strip, the item's
    // first needed column is D bytes into its first chunk, and 32 + w - 1 + D
    // = 48 columns are three chunks for every w
    constexpr int D = FRAMED ? 17 - WR : 0;
    constexpr int NCHR = FRAMED ? 3 : G::NCH;
    static_assert(D + G::L <= 16 * NCHR && TW - ER + 16 * NCHR <= INW, "item reads stay inside the stage");
    int offa[NCHR], offb[NCHR];
#pragma unroll
    for (int c = 0; c < NCHR; ++c) {
      offa[c] = in_off(g * ER + 16 * c, pr);
      offb[c] = in_off(g * ER + 16 * c, pr + 8);
    }
    const int oa = pr * MP + g * ER, ob = (pr + 8) * MP + g * ER;
    int buf = 0, mb = 0;
    uint32_t phase = 0;
    for (int64_t gs = 0; gs < nstages; ++gs) {
      mbar_wait(&bars[buf], phase);
      if (gs >= NMID) bar_sync(kBarEmpty + mb, NTB);  // column side is done with mid[mb]
      const unsigned char *sb = stage_in + buf * STAGE_IN;
      uint32_t x[G::L];
#if !MM_K2B_ROW_VHGW
      uint32_t y[G::L];
#endif
      uint32_t ra[4 * NCHR], rb[4 * NCHR];
#pragma unroll
      for (int c = 0; c < NCHR; ++c) {
        const uint4 va = *reinterpret_cast<const uint4 *>(sb + offa[c]);
        const uint4 vb = *reinterpret_cast<const uint4 *>(sb + offb[c]);
        ra[4 * c] = va.x ^ FLIP, ra[4 * c + 1] = va.y ^ FLIP, ra[4 * c + 2] = va.z ^ FLIP, ra[4 * c + 3] = va.w ^ FLIP;
        rb[4 * c] = vb.x ^ FLIP, rb[4 * c + 1] = vb.y ^ FLIP, rb[4 * c + 2] = vb.z ^ FLIP, rb[4 * c + 3] = vb.w ^ FLIP;
      }
#if MM_K2B_FMA_UNPACK
      static_assert(D == 0, "the IMAD unpack takes unshifted items");
#pragma unroll
      for (int q = 0; q < 4 * NCHR; ++q) {
        // the same words built with IMADs (FMA pipe): [0 A0 0 B0], [A0 A1 B0 B1],
        // [A1 A2 0 B2], [A2 A3 B2 B3] -- bytes 0 and 2 are don't-care
        const uint32_t a = ra[q], b = rb[q];
        const uint32_t hb = umulhi(b, p.k16);
        const uint32_t w[4] = {umad(b, p.k24, umulhi(umul(a, p.k24), p.k16)),
                               umad(b, p.k16, umulhi(umul(a, p.k16), p.k16)),
                               umad(hb, p.k24, umulhi(umul(a, p.k8), p.k16)),
                               umad(hb, p.k16, umulhi(a, p.k16))};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int j = 4 * q + t;
          if (j < G::L) x[j] = w[t];
#if !MM_K2B_ROW_VHGW
          if (j < G::L) y[j] = w[t];
#endif
        }
      }
#else
      // word j: column j of row A in byte 1 (lane 0's high byte), of row B in
      // byte 3 (bytes 0 and 2 repeat them)
#pragma unroll
      for (int j = 0; j < G::L; ++j) {
        const int src = j + D;
        x[j] = prmt(ra[src / 4], rb[src / 4], 0x4400u + 0x1111u * (uint32_t)(src % 4));
#if !MM_K2B_ROW_VHGW
        y[j] = x[j];
#endif
      }
#endif
#if MM_K2B_ROW_VHGW
      uint32_t fx[ER], fn[ER] = {};  // column i of the item
      vhgw_row<WR, true>(x, fx);
      if constexpr (!FRAMED) vhgw_row<WR, false>(x, fn);
      constexpr int F0 = 0;
#else
      sparse_row<WR, true>(x);
      sparse_row<WR, false>(y);
      uint32_t(&fx)[G::L] = x;  // column i of the item is x[i + WR - 1]
      uint32_t(&fn)[G::L] = y;
      constexpr int F0 = WR - 1;
#endif
      // 4 words -> a row-A and a row-B word
      unsigned char *mx_mid = mid + (size_t)(2 * mb) * MID;
      unsigned char *mn_mid = mx_mid + MID;
#pragma unroll
      for (int h = 0; h < ER / 16; ++h) {  // 16 columns -> one 16-B store per row and filter
        uint32_t oxa[4], oxb[4], ona[4], onb[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = 16 * h + 4 * q + F0;
          uint32_t P = prmt(fx[j], fx[j + 1], 0x7351u), Q = prmt(fx[j + 2], fx[j + 3], 0x7351u);
          oxa[q] = prmt(P, Q, 0x5410u);
          oxb[q] = prmt(P, Q, 0x7632u);
          if constexpr (!FRAMED) {
            P = prmt(fn[j], fn[j + 1], 0x7351u), Q = prmt(fn[j + 2], fn[j + 3], 0x7351u);
            ona[q] = prmt(P, Q, 0x5410u);
            onb[q] = prmt(P, Q, 0x7632u);
          }
        }
        *reinterpret_cast<uint4 *>(mx_mid + oa + 16 * h) = make_uint4(oxa[0], oxa[1], oxa[2], oxa[3]);
        *reinterpret_cast<uint4 *>(mx_mid + ob + 16 * h) = make_uint4(oxb[0], oxb[1], oxb[2], oxb[3]);
        if constexpr (!FRAMED) {
          *reinterpret_cast<uint4 *>(mn_mid + oa + 16 * h) = make_uint4(ona[0], ona[1], ona[2], ona[3]);
          *reinterpret_cast<uint4 *>(mn_mid + ob + 16 * h) = make_uint4(onb[0], onb[1], onb[2], onb[3]);
        }
      }
      bar_arrive(kBarFull + mb, NTB);  // hand mid[mb] to the column warps
      bar_sync(kBarRow, NRT);          // every row thread is done with input stage `buf`
      if (tid == 0 && ld_next < nstages) issue();
      if (++buf == NSTG) buf = 0, phase ^= 1u;
      if (++mb == NMID) mb = 0;
    }
  } else {
    // ============================================== column-pass warps (4-7)
    const int ct = tid - NRT;  // columns [4ct, 4ct + 4) of the strip
    ColRing<WC> rxo, rxe, rno, rne;  // rings: max/min x odd/even columns
#pragma unroll
    for (int i = 0; i < ColRing<WC>::HT; ++i) rxo.h[i] = rxe.h[i] = rno.h[i] = rne.h[i] = 0;
    const uint32_t ld = (uint32_t)p.out_ld;
    // a per-thread register holding 1 that the compiler can neither fold nor
    // treat as uniform, so each pointer step stays one vector IMAD.WIDE
    uint32_t one;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(one) : "r"(smem_u32(smem_one)));
    const uint32_t stage_step = (uint32_t)(RB * p.out_ld);
    int mb = 0, left = (int)nstages;
    for (int64_t u = blockIdx.x; u < p.ntiles; u += G_) {
      Cursor cs;
      open(cs, u);
      const int nst = (int)((cs.nin + RB - 1) / RB);
      const int nin = (int)cs.nin;
      const int64_t c = cs.c0 + 4 * ct;
      const int64_t cl = p.Co - c;  // valid columns from c
      // address of stage 0's row 0 (output row o0 - (WC-1): only rows >= r_lo
      // of a stage are ever stored)
      const int64_t o = cs.b * p.out_bstride + (cs.o0 - (WC - 1)) * p.out_ld + c;
      uint8_t *bx = p.out_max ? p.out_max + o : nullptr;
      uint8_t *bn = !FRAMED && p.out_min ? p.out_min + o : nullptr;
      const bool fast_cols = cl >= 4 && bx && (bn || FRAMED);
      for (int st = 0; st < nst; ++st, --left) {
        const unsigned char *mx_mid = mid + (size_t)(2 * mb) * MID + 4 * ct;
        const unsigned char *mn_mid = mx_mid + MID;
        bar_sync(kBarFull + mb, NTB);  // row pass of this stage is in mid[mb]
        uint32_t wx[RB], wn[RB];       // this stage's outputs (natural byte order)
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          const uint32_t vx = *reinterpret_cast<const uint32_t *>(mx_mid + r * MP);
          const uint32_t xo = ring_push<WC, true>(rxo, vx);
          const uint32_t xe = ring_push<WC, true>(rxe, vx << 8);
          wx[r] = prmt(xe, xo, 0x7351u) ^ XOUT;
          if constexpr (!FRAMED) {
            const uint32_t vn = *reinterpret_cast<const uint32_t *>(mn_mid + r * MP);
            const uint32_t no = ring_push<WC, false>(rno, vn);
            const uint32_t ne = ring_push<WC, false>(rne, vn << 8);
            wn[r] = prmt(ne, no, 0x7351u) ^ NOUT;
          } else {
            wn[r] = 0;
          }
        }
        // mid[mb] has been read: release it (only if the row side will wait for it)
        if (left > NMID) bar_arrive(kBarEmpty + mb, NTB);
        if (++mb == NMID) mb = 0;
        // stage row r is output row o0 - (WC-1) + RB*st + r, valid for r in [r_lo, r_hi)
        const int t0 = RB * st;
        const int r_lo = t0 >= WC - 1 ? 0 : WC - 1 - t0;
        const int r_hi = nin - t0 < RB ? nin - t0 : RB;
        if (r_lo == 0 && r_hi == RB && fast_cols) {
          uint8_t *ax = bx, *an = bn;
#pragma unroll
          for (int r = 0; r < RB; ++r) {
            st_u32(ax, wx[r]);
            if constexpr (!FRAMED) st_u32(an, wn[r]);
            ax = ptr_step(ax, one, ld);
            if constexpr (!FRAMED) an = ptr_step(an, one, ld);
          }
        } else if (cl > 0) {  // partial stage or ragged right edge: byte stores
          const int ncol = (int)(cl < 4 ? cl : 4);
#pragma unroll
          for (int r = 0; r < RB; ++r) {
            if (r < r_lo || r >= r_hi) continue;
            for (int k = 0; k < ncol; ++k) {
              if (p.out_max) bx[(int64_t)r * p.out_ld + k] = (uint8_t)(wx[r] >> (8 * k));
              if (!FRAMED && p.out_min) bn[(int64_t)r * p.out_ld + k] = (uint8_t)(wn[r] >> (8 * k));
            }
          }
        }
        // (a missing output's pointer advances too but is never stored through)
        bx = ptr_step(bx, one, stage_step);
        bn = ptr_step(bn, one, stage_step);
      }
    }
  }
}

}  // namespace k2b
}  // namespace mm

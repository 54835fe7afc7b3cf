// k2d.cuh -- fused 2-D separable running max-min filter.
//
// "The unidimensional max-min filter can be applied to images ... by first
// applying the unidimensional on rows and then on columns."  One CTA produces an
// output tile of TH x TW pixels: the (TH+w_col-1) x (TW+w_row-1) input box is
// staged in shared memory by TMA (one bulk copy per box row), the row pass
// (window w_row along each row) and the column pass (window w_col down each
// column) both run on chip, and only the tile's outputs go back to HBM -- one
// read of the input, one write of each output (valid region only, reading R9).
//
// Both passes use log-step doubling on ping-pong shared buffers: after the step
// of span s, M[p] = max a[p .. p+2s); the pass result is max(M[p], M[p+w-2^K])
// with 2^K <= w < 2^(K+1) (max/min are idempotent, so the overlap is harmless).
#pragma once

#include "common.cuh"

namespace mm {

constexpr int NT2 = 256;

template <typename T>
struct K2Tile {
  static constexpr int TW = 256 / (int)sizeof(T);  // output columns per tile (256 B)
  static constexpr int TH = 32;                    // output rows per tile
  static constexpr int VEC = 16 / (int)sizeof(T);
  __host__ __device__ static int pitch(int w_row) {  // box row pitch (elements)
    int bw = TW + w_row - 1;
    return (bw + VEC - 1) / VEC * VEC + VEC;
  }
  __host__ __device__ static size_t bytes(int w_row, int w_col) {
    return sizeof(T) * 4 * (size_t)(TH + w_col - 1) * (size_t)pitch(w_row) + 64;
  }
};

struct Img2D {
  const void *in;
  void *out_max;
  void *out_min;
  int64_t batch, rows, cols, in_ld, in_bstride, out_ld, out_bstride;
  int w_row, w_col;
  int64_t tiles_x, tiles_y;  // tiles along columns / rows
};

template <typename T>
__global__ void __launch_bounds__(NT2) k2d_generic(Img2D p) {
  using Tl = K2Tile<T>;
  constexpr int TW = Tl::TW, TH = Tl::TH;
  const int wr = p.w_row, wc = p.w_col;
  const int P = Tl::pitch(wr);
  const int BH = TH + wc - 1;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  T *Ax = reinterpret_cast<T *>(smem_raw);  // ping (max)
  T *An = Ax + (size_t)BH * P;                // ping (min)
  T *Bx = An + (size_t)BH * P;                // pong (max)
  T *Bn = Bx + (size_t)BH * P;                // pong (min)
  uint64_t *bar = reinterpret_cast<uint64_t *>(
      (reinterpret_cast<uintptr_t>(Bn + (size_t)BH * P) + 15) & ~uintptr_t(15));
  const int tid = threadIdx.x;

  int64_t t = blockIdx.x;
  const int64_t per_img = p.tiles_x * p.tiles_y;
  const int64_t b = t / per_img;
  t -= b * per_img;
  const int64_t ty = t / p.tiles_x, tx = t - ty * p.tiles_x;
  const int64_t r0 = ty * TH, c0 = tx * TW;
  const int64_t Ro = p.rows - wc + 1, Co = p.cols - wr + 1;  // valid output extent
  const int th = (int)(Ro - r0 < TH ? Ro - r0 : TH);
  const int tw = (int)(Co - c0 < TW ? Co - c0 : TW);
  const int bh = th + wc - 1;  // box rows / cols actually inside the image
  const int bw = tw + wr - 1;
  const T *img = static_cast<const T *>(p.in) + b * p.in_bstride;

  // box row r starts at global element rowp(r); its 16-B aligned copy lands at
  // Ax + r*P, so the row's first element sits `shift(r)` elements in.
  auto rowp = [&](int r) { return img + (r0 + r) * p.in_ld + c0; };
  auto shift = [&](int r) { return (int)((reinterpret_cast<uintptr_t>(rowp(r)) & 15) / sizeof(T)); };
  if (tid == 0) {
    mbar_init(bar, 32);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid < 32) {  // one warp issues one bulk copy per box row
    uint32_t mine = 0;
    for (int r = tid; r < bh; r += 32) {
      const uintptr_t g0 = reinterpret_cast<uintptr_t>(rowp(r)) & ~uintptr_t(15);
      const uintptr_t g1 = (reinterpret_cast<uintptr_t>(rowp(r) + bw) + 15) & ~uintptr_t(15);
      mine += (uint32_t)(g1 - g0);
    }
    mbar_arrive_expect_tx(bar, mine);
    for (int r = tid; r < bh; r += 32) {
      const uintptr_t g0 = reinterpret_cast<uintptr_t>(rowp(r)) & ~uintptr_t(15);
      const uintptr_t g1 = (reinterpret_cast<uintptr_t>(rowp(r) + bw) + 15) & ~uintptr_t(15);
      bulk_g2s(Ax + (size_t)r * P, reinterpret_cast<const void *>(g0), (uint32_t)(g1 - g0), bar);
    }
  }
  mbar_wait(bar, 0);

  // ------------------------------------------------------------ row pass
  int K = 0;
  while ((2 << K) <= wr) ++K;
  const T *srcx = Ax, *srcn = Ax;  // first step reads the input for both filters
  T *dstx = Bx, *dstn = Bn;
  bool raw = true;  // src is the raw input box (rows carry their shift)
  int cw = bw;  // valid width of the current level
  for (int s = 1; s < (1 << K); s <<= 1) {
    const int nw = cw - s;
    for (int e = tid; e < bh * nw; e += NT2) {
      const int r = e / nw, c = e - r * nw;
      const size_t o = (size_t)r * P + c;
      const size_t i = o + (raw ? shift(r) : 0);
      dstx[o] = Ord<T>::mx(srcx[i], srcx[i + s]);
      dstn[o] = Ord<T>::mn(srcn[i], srcn[i + s]);
    }
    raw = false;
    __syncthreads();
    cw = nw;
    const T *tx_ = dstx, *tn_ = dstn;
    dstx = (dstx == Bx) ? Ax : Bx;
    dstn = (dstn == Bn) ? An : Bn;
    srcx = tx_;
    srcn = tn_;
  }
  {  // combine: R[r][c] = max(M[r][c], M[r][c + wr - 2^K]), c < tw
    const int off = wr - (1 << K);
    for (int e = tid; e < bh * tw; e += NT2) {
      const int r = e / tw, c = e - r * tw;
      const size_t o = (size_t)r * P + c;
      const size_t i = o + (raw ? shift(r) : 0);
      dstx[o] = Ord<T>::mx(srcx[i], srcx[i + off]);
      dstn[o] = Ord<T>::mn(srcn[i], srcn[i + off]);
    }
    __syncthreads();
    const T *tx_ = dstx, *tn_ = dstn;
    dstx = (dstx == Bx) ? Ax : Bx;
    dstn = (dstn == Bn) ? An : Bn;
    srcx = tx_;
    srcn = tn_;
  }
  // --------------------------------------------------------- column pass
  K = 0;
  while ((2 << K) <= wc) ++K;
  int ch = bh;
  for (int s = 1; s < (1 << K); s <<= 1) {
    const int nh = ch - s;
    for (int e = tid; e < nh * tw; e += NT2) {
      const int r = e / tw, c = e - r * tw;
      const size_t o = (size_t)r * P + c;
      dstx[o] = Ord<T>::mx(srcx[o], srcx[o + (size_t)s * P]);
      dstn[o] = Ord<T>::mn(srcn[o], srcn[o + (size_t)s * P]);
    }
    __syncthreads();
    ch = nh;
    const T *tx_ = dstx, *tn_ = dstn;
    dstx = (dstx == Bx) ? Ax : Bx;
    dstn = (dstn == Bn) ? An : Bn;
    srcx = tx_;
    srcn = tn_;
  }
  const int off = wc - (1 << K);
  T *omx = p.out_max ? static_cast<T *>(p.out_max) + b * p.out_bstride + r0 * p.out_ld + c0 : nullptr;
  T *omn = p.out_min ? static_cast<T *>(p.out_min) + b * p.out_bstride + r0 * p.out_ld + c0 : nullptr;
  for (int e = tid; e < th * tw; e += NT2) {
    const int r = e / tw, c = e - r * tw;
    const size_t o = (size_t)r * P + c;
    if (omx) omx[(size_t)r * p.out_ld + c] = Ord<T>::mx(srcx[o], srcx[o + (size_t)off * P]);
    if (omn) omn[(size_t)r * p.out_ld + c] = Ord<T>::mn(srcn[o], srcn[o + (size_t)off * P]);
  }
}

}  // namespace mm

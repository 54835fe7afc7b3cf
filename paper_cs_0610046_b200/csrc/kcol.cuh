// kcol.cuh -- the running max-min filter down columns, streaming (used by the
// separable 2-D path, sep2d.cu, and the depth pass of the 3-D filter,
// filter3d.cu).
//
// A thread owns one column j (image b, column j % span) over a segment of
// `seg` outputs -- columns alone give too few threads for an image -- and
// walks down its elements (pitch `slice`) in blocks of W (compile time, <= 16;
// a segment re-reads the W-1 rows before its end): van Herk / Gil-Werman along the column -- the
// block's suffix extrema and the next block's running prefix in registers, so
// every element is read once and every output written once, coalesced across
// the warp's adjacent columns.  The max chain reads srcx and the min chain
// srcn (the same array for a plain filter; the row-max and row-min images for
// the second pass of a separable filter).
#pragma once

#include "common.cuh"

#ifndef MM_COL_MINB
#define MM_COL_MINB 2  // 16 warps per SM for <= 4-byte types (8-byte types: 1, they would spill)
#endif

namespace mm {

template <typename T, int W>
__global__ void __launch_bounds__(256, (sizeof(T) >= 8 ? 1 : MM_COL_MINB)) k_col(const T *__restrict__ srcx, const T *__restrict__ srcn,
                                                          int64_t items, int64_t span, int64_t in_bs, int64_t slice,
                                                          int64_t depth, int64_t seg, T *__restrict__ omax,
                                                          T *__restrict__ omin, int64_t out_bs, int64_t oslice) {
  const int64_t D = depth - W + 1;
  const int64_t nseg = (D + seg - 1) / seg;
  const bool same = srcx == srcn;
  const int64_t dn = srcn - srcx;  // the min chain's source, relative to the max chain's
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < items; it += (int64_t)gridDim.x * blockDim.x) {
    // item = (segment, image, column), column fastest: a warp reads adjacent columns
    const int64_t sg = it / (items / nseg), rest = it - sg * (items / nseg);
    const int64_t b = rest / span, j = rest - b * span;
    const int64_t zb = sg * seg, ze = zb + seg < D ? zb + seg : D;  // outputs [zb, ze)
    // running pointers (one 64-bit register each instead of an address per row)
    const T *pin = srcx + b * in_bs + j + zb * slice;
    T *pox = omax ? omax + b * out_bs + j + zb * oslice : nullptr;
    T *pon = omin ? omin + b * out_bs + j + zb * oslice : nullptr;
    T sx[W], sn[W];  // suffix max / min of the current block
#pragma unroll
    for (int t = 0; t < W; ++t, pin += slice) {  // the block [zb, zb + W) (zb + W <= depth)
      sx[t] = pin[0];
      sn[t] = same ? sx[t] : pin[dn];
    }
#pragma unroll
    for (int t = W - 2; t >= 0; --t) {
      sx[t] = Ord<T>::mx(sx[t], sx[t + 1]);
      sn[t] = Ord<T>::mn(sn[t], sn[t + 1]);
    }
    for (int64_t b0 = zb; b0 < ze; b0 += W) {  // outputs b0 .. b0+W-1: block b and block b+1
      T vx[W], vn[W];
      const int64_t avail = depth - (b0 + W);  // rows of block b+1 inside the column
#pragma unroll
      for (int t = 0; t < W; ++t, pin += slice) {
        vx[t] = t < avail ? pin[0] : T(0);
        vn[t] = same ? vx[t] : (t < avail ? pin[dn] : T(0));
      }
      const int64_t nout = ze - b0;  // outputs of this block still in the segment
      T px = vx[0], pn = vn[0];      // after step t: the next block's prefix over [0, t]
#pragma unroll
      for (int t = 0; t < W; ++t) {  // window [b0 + t, b0 + t + W): block b's suffix from t, next block's [0, t)
        if (t < nout) {
          T x = sx[t], n = sn[t];
          if (t > 0) {
            x = Ord<T>::mx(x, px);
            n = Ord<T>::mn(n, pn);
          }
          if (pox) {
            *pox = x;
            pox += oslice;
          }
          if (pon) {
            *pon = n;
            pon += oslice;
          }
        }
        if (t > 0) {
          px = Ord<T>::mx(px, vx[t]);
          pn = Ord<T>::mn(pn, vn[t]);
        }
      }
#pragma unroll
      for (int t = 0; t < W; ++t) {  // the next block's suffixes
        sx[t] = vx[t];
        sn[t] = vn[t];
      }
#pragma unroll
      for (int t = W - 2; t >= 0; --t) {
        sx[t] = Ord<T>::mx(sx[t], sx[t + 1]);
        sn[t] = Ord<T>::mn(sn[t], sn[t + 1]);
      }
    }
  }
}

constexpr int kColMaxW = 16;

// kErrUnsupported (= 10, launch.cuh) for windows longer than kColMaxW
template <typename T>
int launch_col(const T *srcx, const T *srcn, int64_t batch, int64_t span, int64_t in_bs, int64_t slice,
               int64_t depth, int64_t w, T *omax, T *omin, int64_t out_bs, int64_t oslice, int sms, cudaStream_t s);

}  // namespace mm

namespace mm {

// 1-byte pixels, four adjacent columns per thread: one 32-bit load per row,
// split into two words whose u16 lanes carry the pixels in their high bytes
// (odd columns: the word masked; even columns: the word shifted by 8), so
// every max / min is one VIMNMX.U16x2 over two columns (the low bytes are
// zero and never decide).  Signed pixels are biased by 0x80 on the way in
// and out.  Rows, pitches and pointers are 4-byte aligned (the launcher
// checks), span % 4 == 0.
template <int W, bool SIGNED>
__global__ void __launch_bounds__(256) k_col_b8(const uint8_t *__restrict__ srcx, const uint8_t *__restrict__ srcn,
                                                int64_t items, int64_t span4, int64_t in_bs, int64_t slice,
                                                int64_t depth, int64_t seg, uint8_t *__restrict__ omax,
                                                uint8_t *__restrict__ omin, int64_t out_bs, int64_t oslice) {
  const int64_t D = depth - W + 1;
  const int64_t nseg = (D + seg - 1) / seg;
  const bool same = srcx == srcn;
  constexpr uint32_t HI = 0xFF00FF00u, BIAS = SIGNED ? 0x80808080u : 0u;
  auto lo_hi = [&](uint32_t w, uint32_t &ev, uint32_t &od) {
    w ^= BIAS;
    od = w & HI;
    ev = (w << 8) & HI;
  };
  auto pack = [&](uint32_t ev, uint32_t od) { return ((od & HI) | ((ev >> 8) & 0x00FF00FFu)) ^ BIAS; };
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < items; it += (int64_t)gridDim.x * blockDim.x) {
    const int64_t sg = it / (items / nseg), rest = it - sg * (items / nseg);
    const int64_t b = rest / span4, j = (rest - b * span4) * 4;
    const int64_t zb = sg * seg, ze = zb + seg < D ? zb + seg : D;
    const uint8_t *ax = srcx + b * in_bs + j;
    const uint8_t *an = srcn + b * in_bs + j;
    uint8_t *ox_ = omax ? omax + b * out_bs + j : nullptr;
    uint8_t *on_ = omin ? omin + b * out_bs + j : nullptr;
    auto ld = [&](const uint8_t *p, int64_t z) { return *reinterpret_cast<const uint32_t *>(p + z * slice); };
    uint32_t sxe[W], sxo[W], sne[W], sno[W];  // suffix max / min, even / odd columns
#pragma unroll
    for (int t = 0; t < W; ++t) {
      lo_hi(ld(ax, zb + t), sxe[t], sxo[t]);
      if (same) {
        sne[t] = sxe[t];
        sno[t] = sxo[t];
      } else {
        lo_hi(ld(an, zb + t), sne[t], sno[t]);
      }
    }
#pragma unroll
    for (int t = W - 2; t >= 0; --t) {
      sxe[t] = __vmaxu2(sxe[t], sxe[t + 1]);
      sxo[t] = __vmaxu2(sxo[t], sxo[t + 1]);
      sne[t] = __vminu2(sne[t], sne[t + 1]);
      sno[t] = __vminu2(sno[t], sno[t + 1]);
    }
    for (int64_t b0 = zb; b0 < ze; b0 += W) {
      uint32_t vxe[W], vxo[W], vne[W], vno[W];
#pragma unroll
      for (int t = 0; t < W; ++t) {
        const int64_t z = b0 + W + t;
        lo_hi(z < depth ? ld(ax, z) : 0u, vxe[t], vxo[t]);
        if (same) {
          vne[t] = vxe[t];
          vno[t] = vxo[t];
        } else {
          lo_hi(z < depth ? ld(an, z) : 0u, vne[t], vno[t]);
        }
      }
      uint32_t pxe = vxe[0], pxo = vxo[0], pne = vne[0], pno = vno[0];
#pragma unroll
      for (int t = 0; t < W; ++t) {
        const int64_t z0 = b0 + t;
        if (z0 < ze) {
          uint32_t xe = sxe[t], xo = sxo[t], ne = sne[t], no = sno[t];
          if (t > 0) {
            xe = __vmaxu2(xe, pxe);
            xo = __vmaxu2(xo, pxo);
            ne = __vminu2(ne, pne);
            no = __vminu2(no, pno);
          }
          if (ox_) *reinterpret_cast<uint32_t *>(ox_ + z0 * oslice) = pack(xe, xo);
          if (on_) *reinterpret_cast<uint32_t *>(on_ + z0 * oslice) = pack(ne, no);
        }
        if (t > 0) {
          pxe = __vmaxu2(pxe, vxe[t]);
          pxo = __vmaxu2(pxo, vxo[t]);
          pne = __vminu2(pne, vne[t]);
          pno = __vminu2(pno, vno[t]);
        }
      }
#pragma unroll
      for (int t = 0; t < W; ++t) {
        sxe[t] = vxe[t];
        sxo[t] = vxo[t];
        sne[t] = vne[t];
        sno[t] = vno[t];
      }
#pragma unroll
      for (int t = W - 2; t >= 0; --t) {
        sxe[t] = __vmaxu2(sxe[t], sxe[t + 1]);
        sxo[t] = __vmaxu2(sxo[t], sxo[t + 1]);
        sne[t] = __vminu2(sne[t], sne[t + 1]);
        sno[t] = __vminu2(sno[t], sno[t + 1]);
      }
    }
  }
}

}  // namespace mm

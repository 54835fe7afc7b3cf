// sep2d.cu -- the 2-D max-min filter as two streaming passes (PAPER.md:61-63,
// "first on rows and then on columns", taken literally) for the element types
// and windows the fused packed-byte kernel (k2d_byte) does not cover.
//   1. rows: the library's 1-D batched filter (k1d_small / k1d_medium: TMA
//      tiles, 0.85-0.95 of HBM bandwidth) over every image row, the row max and
//      the row min into two scratch images of rows x C' (16-B row pitch);
//   2. columns: the streaming column kernel (kcol.cuh) -- the max down the
//      row-max image and the min down the row-min image, straight into the
//      caller's outputs (valid region only).
// HBM: 1 read + 2 writes + 2 reads + 2 writes per pixel against 1 + 2 for a
// fused tile, but both passes stream at bandwidth, where the fused generic
// kernel (k2d_generic: log-step doubling in shared memory) is
// instruction-bound (0.06 of the roofline for f32 at 5x5).
#include "kcol.cuh"
#include "launch.cuh"

namespace mm {

template <typename T>
int launch_col(const T *srcx, const T *srcn, int64_t batch, int64_t span, int64_t in_bs, int64_t slice,
               int64_t depth, int64_t w, T *omax, T *omin, int64_t out_bs, int64_t oslice, int sms, cudaStream_t s) {
  const int64_t cols_total = batch * span;
  if (cols_total == 0) return kOK;
  const int64_t D = depth - w + 1;
  // segments of outputs per column: enough threads to fill the GPU (~64 K), each
  // segment >= 64 outputs so the W-1 re-read rows stay a small overhead
  int64_t seg = D;
  const int64_t want = (int64_t)sms * 512;
  if (cols_total < want) {
    const int64_t nseg = (want + cols_total - 1) / cols_total;
    seg = (D + nseg - 1) / nseg;
    if (seg < 64) seg = 64;
  }
  if constexpr (sizeof(T) == 1) {  // four columns per thread, packed (k_col_b8)
    auto al4 = [](const void *p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 3) == 0; };
    if (span % 4 == 0 && in_bs % 4 == 0 && slice % 4 == 0 && out_bs % 4 == 0 && oslice % 4 == 0 && al4(srcx) &&
        al4(srcn) && al4(omax) && al4(omin)) {
      const int64_t items4 = cols_total / 4 * ((D + seg - 1) / seg);
      const int64_t blocks4 = std::min<int64_t>((items4 + 255) / 256, (int64_t)sms * 8);
      const int g4 = (int)(blocks4 > 0 ? blocks4 : 1);
      constexpr bool SG = std::is_signed<T>::value;
      const uint8_t *ux = reinterpret_cast<const uint8_t *>(srcx), *un = reinterpret_cast<const uint8_t *>(srcn);
      uint8_t *qx = reinterpret_cast<uint8_t *>(omax), *qn = reinterpret_cast<uint8_t *>(omin);
      switch (w) {
#define MM_COLB_CASE(W)                                                                                           \
  case W:                                                                                                         \
    k_col_b8<W, SG><<<g4, 256, 0, s>>>(ux, un, items4, span / 4, in_bs, slice, depth, seg, qx, qn, out_bs, oslice); \
    return note_cuda(cudaGetLastError());
        MM_COLB_CASE(1) MM_COLB_CASE(2) MM_COLB_CASE(3) MM_COLB_CASE(4) MM_COLB_CASE(5) MM_COLB_CASE(6)
        MM_COLB_CASE(7) MM_COLB_CASE(8) MM_COLB_CASE(9) MM_COLB_CASE(10) MM_COLB_CASE(11) MM_COLB_CASE(12)
        MM_COLB_CASE(13) MM_COLB_CASE(14) MM_COLB_CASE(15) MM_COLB_CASE(16)
#undef MM_COLB_CASE
        default: return kErrUnsupported;
      }
    }
  }
  const int64_t items = cols_total * ((D + seg - 1) / seg);
  const int64_t blocks = std::min<int64_t>((items + 255) / 256, (int64_t)sms * 8);
  const int g = (int)(blocks > 0 ? blocks : 1);
  switch (w) {
#define MM_COL_CASE(W)                                                                                             \
  case W:                                                                                                          \
    k_col<T, W><<<g, 256, 0, s>>>(srcx, srcn, items, span, in_bs, slice, depth, seg, omax, omin, out_bs, oslice); \
    return note_cuda(cudaGetLastError());
    MM_COL_CASE(1) MM_COL_CASE(2) MM_COL_CASE(3) MM_COL_CASE(4) MM_COL_CASE(5) MM_COL_CASE(6) MM_COL_CASE(7)
    MM_COL_CASE(8) MM_COL_CASE(9) MM_COL_CASE(10) MM_COL_CASE(11) MM_COL_CASE(12) MM_COL_CASE(13)
    MM_COL_CASE(14) MM_COL_CASE(15) MM_COL_CASE(16)
#undef MM_COL_CASE
    default: return kErrUnsupported;
  }
}

namespace {
template <typename T>
struct Sep2DLayout {
  int64_t C, tld;
  size_t one, total;
  Sep2DLayout(int64_t batch, int64_t rows, int64_t cols, int64_t w_row) {
    constexpr int VEC = 16 / (int)sizeof(T);
    C = cols - w_row + 1;
    tld = (C + VEC - 1) / VEC * VEC;
    one = w_row > 1 ? (((size_t)batch * rows * tld * sizeof(T) + 255) & ~size_t(255)) : 0;
    total = 2 * one;
  }
};
}  // namespace

template <typename T>
bool sep2d_applies(int64_t w_row, int64_t w_col) {
  return w_col <= kColMaxW && w_row <= kHaloMax + 1;
}

template <typename T>
size_t sep2d_workspace(int64_t batch, int64_t rows, int64_t cols, int64_t w_row, int64_t w_col) {
  if (!sep2d_applies<T>(w_row, w_col)) return 0;
  return Sep2DLayout<T>(batch, rows, cols, w_row).total;
}

template <typename T>
int launch_2d_sep(const void *in, int64_t batch, int64_t rows, int64_t cols, int64_t in_ld, int64_t in_bstride,
                  int64_t w_row, int64_t w_col, void *out_max, void *out_min, int64_t out_ld, int64_t out_bstride,
                  void *ws, size_t ws_bytes, cudaStream_t s) {
  if (!sep2d_applies<T>(w_row, w_col)) return kErrUnsupported;
  const Sep2DLayout<T> L(batch, rows, cols, w_row);
  if (ws_bytes < L.total || (L.total && !ws)) return kErrUnsupported;
  const T *src = static_cast<const T *>(in);
  if (w_row == 1) {  // no row pass: the columns of the input itself
    return launch_col<T>(src, src, batch, cols, batch > 1 ? in_bstride : 0, in_ld, rows, w_col,
                         static_cast<T *>(out_max), static_cast<T *>(out_min), batch > 1 ? out_bstride : 0, out_ld,
                         sm_count(), s);
  }
  // the 1-D kernels stage rows with TMA: 16-B aligned rows
  if ((reinterpret_cast<uintptr_t>(in) & 15) || ((in_ld * (int64_t)sizeof(T)) & 15) ||
      (batch > 1 && ((in_bstride * (int64_t)sizeof(T)) & 15)))
    return kErrUnsupported;
  T *tmax = static_cast<T *>(ws);
  T *tmin = reinterpret_cast<T *>(static_cast<char *>(ws) + L.one);
  int rc;
  if (batch == 1 || in_bstride == rows * in_ld) {
    rc = launch_1d<T>(in, batch * rows, cols, in_ld, w_row, tmax, tmin, L.tld, nullptr, 0, s);
  } else {
    rc = kOK;
    for (int64_t b = 0; b < batch && rc == kOK; ++b)
      rc = launch_1d<T>(src + b * in_bstride, rows, cols, in_ld, w_row, tmax + b * rows * L.tld,
                        tmin + b * rows * L.tld, L.tld, nullptr, 0, s);
  }
  if (rc) return rc;
  return launch_col<T>(tmax, tmin, batch, L.C, rows * L.tld, L.tld, rows, w_col, static_cast<T *>(out_max),
                       static_cast<T *>(out_min), batch > 1 ? out_bstride : 0, out_ld, sm_count(), s);
}

template <typename T>
int launch_2d_best(const void *in, int64_t batch, int64_t rows, int64_t cols, int64_t in_ld, int64_t in_bstride,
                   int64_t w_row, int64_t w_col, void *out_max, void *out_min, int64_t out_ld, int64_t out_bstride,
                   void *ws, size_t ws_bytes, cudaStream_t s) {
  if (batch == 0) return kOK;
  if constexpr (sizeof(T) == 1) {
    const int rc = launch_2d_byte(std::is_signed<T>::value, in, batch, rows, cols, in_ld, in_bstride, w_row, w_col,
                                  out_max, out_min, out_ld, out_bstride, s);
    if (rc != kErrUnsupported) return rc;
  }
  const int rc = launch_2d_sep<T>(in, batch, rows, cols, in_ld, in_bstride, w_row, w_col, out_max, out_min, out_ld,
                                  out_bstride, ws, ws_bytes, s);
  if (rc != kErrUnsupported) return rc;
  return launch_2d<T>(in, batch, rows, cols, in_ld, in_bstride, w_row, w_col, out_max, out_min, out_ld, out_bstride, s);
}

#define MM_SEP_INST(T)                                                                                        \
  template int launch_col<T>(const T *, const T *, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, T *, \
                             T *, int64_t, int64_t, int, cudaStream_t);                                      \
  template size_t sep2d_workspace<T>(int64_t, int64_t, int64_t, int64_t, int64_t);                           \
  template int launch_2d_sep<T>(const void *, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, \
                                void *, void *, int64_t, int64_t, void *, size_t, cudaStream_t);          \
  template int launch_2d_best<T>(const void *, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, \
                                 void *, void *, int64_t, int64_t, void *, size_t, cudaStream_t);
MM_SEP_INST(uint8_t)
MM_SEP_INST(int8_t)
MM_SEP_INST(uint16_t)
MM_SEP_INST(int16_t)
MM_SEP_INST(uint32_t)
MM_SEP_INST(int32_t)
MM_SEP_INST(uint64_t)
MM_SEP_INST(int64_t)
MM_SEP_INST(float)
MM_SEP_INST(double)

}  // namespace mm

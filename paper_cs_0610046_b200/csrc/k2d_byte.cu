// k2d_byte.cu -- instantiation and launchers of the packed 1-byte 2-D kernel
// (k2d_byte.cuh).  Square windows 2..17 are compiled in.  Other shapes, other
// element types and layouts the kernel does not take (the input's rows and
// pitches 16-B aligned for TMA, output rows 4-B aligned for the word stores)
// go to the separable or the generic 2-D kernels.
#include "launch.cuh"
#include "k2d_byte.cuh"

namespace mm {

template <uint32_t FIN, uint32_t FXO, uint32_t FNO, bool MAXONLY, int W>
static int launch_byte(const k2b::Args &a, const CUtensorMap &map, cudaStream_t s) {
  constexpr size_t smem = k2b::Smem::BYTES;
  auto kern = k2b::k2d_byte<FIN, FXO, FNO, MAXONLY, W, W>;
  static size_t attr = 0;
  int rc = set_smem(kern, smem, attr);
  if (rc) return rc;
  int per_sm = 0;
  rc = blocks_per_sm(reinterpret_cast<const void *>(kern), k2b::NTB, smem, &per_sm);
  if (rc) return rc;
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)per_sm * sm_count();
  if (grid > a.ntiles) grid = a.ntiles;
  kern<<<(unsigned)grid, k2b::NTB, smem, s>>>(a, map);
  return note_cuda(cudaGetLastError());
}

bool k2b_supports(int64_t w) {  // the square windows compiled into dispatch_square below
  switch (w) {
    case 2: case 3: case 4: case 5: case 7: case 9: case 11: case 13: case 15: case 16: case 17: return true;
    default: return false;
  }
}

template <uint32_t FIN, uint32_t FXO, uint32_t FNO, bool MAXONLY>
static int dispatch_square(const k2b::Args &a, const CUtensorMap &m, int w, cudaStream_t s) {
  switch (w) {
    case 2: return launch_byte<FIN, FXO, FNO, MAXONLY, 2>(a, m, s);
    case 3: return launch_byte<FIN, FXO, FNO, MAXONLY, 3>(a, m, s);
    case 4: return launch_byte<FIN, FXO, FNO, MAXONLY, 4>(a, m, s);
    case 5: return launch_byte<FIN, FXO, FNO, MAXONLY, 5>(a, m, s);
    case 7: return launch_byte<FIN, FXO, FNO, MAXONLY, 7>(a, m, s);
    case 9: return launch_byte<FIN, FXO, FNO, MAXONLY, 9>(a, m, s);
    case 11: return launch_byte<FIN, FXO, FNO, MAXONLY, 11>(a, m, s);
    case 13: return launch_byte<FIN, FXO, FNO, MAXONLY, 13>(a, m, s);
    case 15: return launch_byte<FIN, FXO, FNO, MAXONLY, 15>(a, m, s);
    case 16: return launch_byte<FIN, FXO, FNO, MAXONLY, 16>(a, m, s);
    case 17: return launch_byte<FIN, FXO, FNO, MAXONLY, 17>(a, m, s);
    default: return kErrUnsupported;
  }
}

// Shape checks and the arguments of one packed-byte launch: the input image
// [in_rows x in_cols] (pitches in_ld / in_bstride), outputs [Ro x Co] whose
// output (0, 0) window starts at input (in_off, in_off) -- 0, or -(w-1) when
// the input is read through a zero frame (the tensor map's out-of-bounds fill;
// the FRAMED kernels).
static int byte_args(const void *in, int64_t batch, int64_t in_rows, int64_t in_cols, int64_t in_ld,
                     int64_t in_bstride, int64_t w, int64_t Ro, int64_t Co, int in_off, void *out_max, void *out_min,
                     int64_t out_ld, int64_t out_bstride, k2b::Args &a, CUtensorMap &m) {
  if (w > k2b::MAXW || !k2b_supports(w)) return kErrUnsupported;
  auto al = [](const void *p, uintptr_t q) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) % q) == 0; };
  if (!al(in, 16) || in_ld % 16 || (batch > 1 && in_bstride % 16)) return kErrUnsupported;
  if (!al(out_max, 4) || !al(out_min, 4) || out_ld % 4 || (batch > 1 && out_bstride % 4)) return kErrUnsupported;
  if (in_cols > 0x7fffffffLL || in_rows > 0x7fffffffLL || Ro + w > 0x7fffffffLL || Co + w > 0x7fffffffLL ||
      batch > 0x7fffffffLL || out_ld > (0xffffffffLL / k2b::RB))
    return kErrUnsupported;
  a.out_max = static_cast<uint8_t *>(out_max);
  a.out_min = static_cast<uint8_t *>(out_min);
  a.batch = batch;
  a.rows = in_rows;
  a.cols = in_cols;
  a.out_ld = out_ld;
  a.out_bstride = batch > 1 ? out_bstride : 0;
  a.Ro = Ro;
  a.Co = Co;
  a.nstrip = (a.Co + k2b::TW - 1) / k2b::TW;
  // bands of BH output rows: BH + w - 1 input rows is a whole number of
  // RB-row stages, so only an image's last band has a partial stage
  a.BH = 32 * k2b::RB - (w - 1);
  a.nbands = (a.Ro + a.BH - 1) / a.BH;
  a.ntiles = batch * a.nbands * a.nstrip;
  a.one = 1u;
  a.k8 = 1u << 8;
  a.k16 = 1u << 16;
  a.k24 = 1u << 24;
  a.in_r0 = in_off;
  // TMA map over the input {cols, rows, batch}, boxes {176, RB, 1}; columns and
  // rows outside the image (the last strip's halo, a zero frame) read as zeros
  std::memset(&m, 0, sizeof(m));
  const int64_t idims[3] = {in_cols, in_rows, batch};
  const int64_t istr[2] = {in_ld, batch > 1 ? in_bstride : in_rows * in_ld};
  const int box[3] = {k2b::BOXW, k2b::RB, 1};
  return encode_u8_map(&m, in, idims, istr, box);
}

int launch_2d_byte(bool is_signed, const void *in, int64_t batch, int64_t rows, int64_t cols,
                   int64_t in_ld, int64_t in_bstride, int64_t w_row, int64_t w_col, void *out_max,
                   void *out_min, int64_t out_ld, int64_t out_bstride, cudaStream_t s) {
  if (w_row != w_col) return kErrUnsupported;
  k2b::Args a;
  CUtensorMap m;
  const int rc = byte_args(in, batch, rows, cols, in_ld, in_bstride, w_row, rows - w_col + 1, cols - w_row + 1, 0,
                           out_max, out_min, out_ld, out_bstride, a, m);
  if (rc) return rc;
  if (a.ntiles == 0) return kOK;
  return is_signed ? dispatch_square<0x80, 0x80, 0x80, false>(a, m, (int)w_row, s)
                   : dispatch_square<0, 0, 0, false>(a, m, (int)w_row, s);
}

// Grayscale opening and closing of 1-byte images by a w x w square (reading
// R20) in three packed passes and no frame copies:
//   1. e = min filter and ~d = complement of the max filter, valid region
//      (R x C), into e_buf / d_buf (pitch buf_ld);
//   2. open = max filter of e read through a (w-1)-wide zero frame (the tensor
//      map's out-of-bounds fill: 0 is the identity of max), all rows x cols;
//   3. close = ~(max filter of ~d through the zero frame) = min filter of d
//      framed by 255 (the identity of min).
// Signed bytes travel biased by 0x80 (order-preserving) and are unbiased on
// the final stores.  HBM: 1 read + 2 writes, then 2 x (1 read + 1 write).
int launch_morph_2d_byte(bool is_signed, const void *in, int64_t batch, int64_t rows, int64_t cols, int64_t in_ld,
                         int64_t in_bstride, int64_t w, void *out_open, void *out_close, int64_t out_ld,
                         int64_t out_bstride, void *e_buf, void *d_buf, int64_t buf_ld, cudaStream_t s) {
  const int64_t R = rows - w + 1, C = cols - w + 1;
  k2b::Args a1, a2, a3;
  CUtensorMap m1, m2, m3;
  int rc = byte_args(in, batch, rows, cols, in_ld, in_bstride, w, R, C, 0, d_buf, e_buf, buf_ld, R * buf_ld, a1, m1);
  if (!rc && out_open)
    rc = byte_args(e_buf, batch, R, C, buf_ld, R * buf_ld, w, rows, cols, (int)(1 - w), out_open, nullptr, out_ld,
                   out_bstride, a2, m2);
  if (!rc && out_close)
    rc = byte_args(d_buf, batch, R, C, buf_ld, R * buf_ld, w, rows, cols, (int)(1 - w), out_close, nullptr, out_ld,
                   out_bstride, a3, m3);
  if (rc) return rc;
  if (a1.ntiles == 0) return kOK;
  const int wi = (int)w;
  rc = is_signed ? dispatch_square<0x80, 0xFF, 0, false>(a1, m1, wi, s) : dispatch_square<0, 0xFF, 0, false>(a1, m1, wi, s);
  if (!rc && out_open)
    rc = is_signed ? dispatch_square<0, 0x80, 0, true>(a2, m2, wi, s) : dispatch_square<0, 0, 0, true>(a2, m2, wi, s);
  if (!rc && out_close)
    rc = is_signed ? dispatch_square<0, 0x7F, 0, true>(a3, m3, wi, s) : dispatch_square<0, 0xFF, 0, true>(a3, m3, wi, s);
  return rc;
}

}  // namespace mm

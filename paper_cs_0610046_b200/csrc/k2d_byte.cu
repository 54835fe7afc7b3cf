// k2d_byte.cu -- instantiation and launcher of the packed 1-byte 2-D kernel
// (k2d_byte.cuh).  Square windows 2..17 are compiled in.  Other shapes, other
// element types and layouts the kernel does not take (the input's rows and
// pitches 16-B aligned for TMA, output rows 4-B aligned for the word stores)
// go to k2d_generic.
#include "launch.cuh"
#include "k2d_byte.cuh"

namespace mm {

template <bool SG, int WR, int WC>
static int launch_byte(const k2b::Args &a, const CUtensorMap &map, cudaStream_t s) {
  constexpr size_t smem = k2b::Smem::BYTES;
  auto kern = k2b::k2d_byte<SG, WR, WC>;
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

template <bool SG>
static int dispatch_square(const k2b::Args &a, const CUtensorMap &m, int w, cudaStream_t s) {
  switch (w) {
    case 2: return launch_byte<SG, 2, 2>(a, m, s);
    case 3: return launch_byte<SG, 3, 3>(a, m, s);
    case 4: return launch_byte<SG, 4, 4>(a, m, s);
    case 5: return launch_byte<SG, 5, 5>(a, m, s);
    case 7: return launch_byte<SG, 7, 7>(a, m, s);
    case 9: return launch_byte<SG, 9, 9>(a, m, s);
    case 11: return launch_byte<SG, 11, 11>(a, m, s);
    case 13: return launch_byte<SG, 13, 13>(a, m, s);
    case 15: return launch_byte<SG, 15, 15>(a, m, s);
    case 16: return launch_byte<SG, 16, 16>(a, m, s);
    case 17: return launch_byte<SG, 17, 17>(a, m, s);
    default: return kErrUnsupported;
  }
}

int launch_2d_byte(bool is_signed, const void *in, int64_t batch, int64_t rows, int64_t cols,
                   int64_t in_ld, int64_t in_bstride, int64_t w_row, int64_t w_col, void *out_max,
                   void *out_min, int64_t out_ld, int64_t out_bstride, cudaStream_t s) {
  if (w_row != w_col || w_row > k2b::MAXW || !k2b_supports(w_row)) return kErrUnsupported;
  auto al = [](const void *p, uintptr_t m) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) % m) == 0; };
  if (!al(in, 16) || in_ld % 16 || (batch > 1 && in_bstride % 16)) return kErrUnsupported;
  if (!al(out_max, 4) || !al(out_min, 4) || out_ld % 4 || (batch > 1 && out_bstride % 4))
    return kErrUnsupported;
  if (cols > 0x7fffffffLL || rows > 0x7fffffffLL || batch > 0x7fffffffLL || out_ld > (0xffffffffLL / k2b::RB))
    return kErrUnsupported;
  k2b::Args a;
  a.out_max = static_cast<uint8_t *>(out_max);
  a.out_min = static_cast<uint8_t *>(out_min);
  a.batch = batch;
  a.rows = rows;
  a.cols = cols;
  a.out_ld = out_ld;
  a.out_bstride = batch > 1 ? out_bstride : 0;
  a.Ro = rows - w_col + 1;
  a.Co = cols - w_row + 1;
  a.nstrip = (a.Co + k2b::TW - 1) / k2b::TW;
  // bands of BH output rows: BH + w_col - 1 input rows is a whole number of
  // RB-row stages, so only an image's last band has a partial stage
  a.BH = 32 * k2b::RB - (w_col - 1);
  a.nbands = (a.Ro + a.BH - 1) / a.BH;
  a.ntiles = batch * a.nbands * a.nstrip;
  a.one = 1u;
  a.k8 = 1u << 8;
  a.k16 = 1u << 16;
  a.k24 = 1u << 24;
  if (a.ntiles == 0) return kOK;
  // TMA map over the input {cols, rows, batch}, boxes {176, RB, 1}; columns
  // past the image (the last strip's halo) read as zeros and are never output
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  const int64_t idims[3] = {cols, rows, batch};
  const int64_t istr[2] = {in_ld, batch > 1 ? in_bstride : rows * in_ld};
  const int box[3] = {k2b::BOXW, k2b::RB, 1};
  const int rc = encode_u8_map(&m, in, idims, istr, box);
  if (rc) return rc;
  return is_signed ? dispatch_square<true>(a, m, (int)w_row, s) : dispatch_square<false>(a, m, (int)w_row, s);
}

}  // namespace mm

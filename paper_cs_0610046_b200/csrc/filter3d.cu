// filter3d.cu -- the max-min filter over 3-D boxes ("N-D
// separable filters").  The paper applies the 1-D filter to images "first on
// rows and then on columns"; a volume adds the depth axis:
//   out(k,i,j) = max / min of a over [k, k+w_z) x [i, i+w_y) x [j, j+w_x)
// for the valid region (D' x R' x C' = depth-w_z+1 x rows-w_y+1 x cols-w_x+1).
//
// Two passes, depth first:
//   1. depth: max and min along depth for every (i, j), into two scratch
//      volumes laid out like the input slices.  For w_z <= 16 the streaming
//      column kernel (kcol.cuh): a thread per element of a slice walks down
//      the slices -- one coalesced read per element and one write per output.
//      Larger w_z: the 2-D kernel on the volume seen as an image whose "rows"
//      are slices (window 1 x w_z).
//   2. rows and columns: the 2-D filter (w_x, w_y) of every scratch slice, the
//      max over the depth-max and the min over the depth-min, straight into the
//      caller's outputs (valid region only).
// HBM: 1 read + 2 writes + 2 reads + 2 writes of a volume (a fused 3-D tile
// would need 1 + 2).  Max and min commute with each other per axis, so the
// order of the axes does not change the result (oracle_separable_3d takes the
// opposite order and is compared bit for bit).
#include "kcol.cuh"
#include "launch.cuh"

namespace mm {

template <typename T>
struct Vol3DLayout {
  int64_t D, span, tsl;  // output depth; elements of one slice's span; scratch slice pitch
  size_t one, sep, total;
  Vol3DLayout(int64_t depth, int64_t rows, int64_t cols, int64_t in_ld, int64_t w_z, int64_t w_x = 1,
              int64_t w_y = 1) {
    constexpr int VEC = 16 / (int)sizeof(T);
    D = depth - w_z + 1;
    span = (rows - 1) * in_ld + cols;
    tsl = (rows * in_ld + VEC - 1) / VEC * VEC;
    one = ((size_t)D * tsl * sizeof(T) + 255) & ~size_t(255);
    sep = (sep2d_workspace<T>(D, rows, cols, w_x, w_y) + 255) & ~size_t(255);  // pass 2's row images
    total = 2 * one + sep;
  }
};

template <typename T>
size_t filter3d_workspace(int64_t depth, int64_t rows, int64_t cols, int64_t in_ld, int64_t w_x, int64_t w_y,
                          int64_t w_z) {
  return Vol3DLayout<T>(depth, rows, cols, in_ld, w_z, w_x, w_y).total;
}

template <typename T>
int launch_3d(const void *in, int64_t depth, int64_t rows, int64_t cols, int64_t in_ld, int64_t in_slice,
              int64_t w_x, int64_t w_y, int64_t w_z, void *out_max, void *out_min, int64_t out_ld, int64_t out_slice,
              void *ws, cudaStream_t s) {
  const Vol3DLayout<T> L(depth, rows, cols, in_ld, w_z, w_x, w_y);
  T *tmax = static_cast<T *>(ws);
  T *tmin = reinterpret_cast<T *>(static_cast<char *>(ws) + L.one);
  void *sepws = static_cast<char *>(ws) + 2 * L.one;
  // 1. depth: the streaming kernel, else the 2-D kernel with rows = slices, window 1 x w_z
  int rc = launch_col<T>(static_cast<const T *>(in), static_cast<const T *>(in), 1, L.span, 0, in_slice, depth, w_z,
                         out_max ? tmax : nullptr, out_min ? tmin : nullptr, 0, L.tsl, sm_count(), s);
  if (rc == kErrUnsupported)
    rc = launch_2d<T>(in, 1, depth, L.span, in_slice, 0, 1, w_z, out_max ? tmax : nullptr,
                      out_min ? tmin : nullptr, L.tsl, 0, s);
  if (rc) return rc;
  // 2. rows and columns of every scratch slice
  if (out_max) {
    rc = launch_2d_best<T>(tmax, L.D, rows, cols, in_ld, L.tsl, w_x, w_y, out_max, nullptr, out_ld, out_slice, sepws,
                           L.sep, s);
    if (rc) return rc;
  }
  if (out_min)
    rc = launch_2d_best<T>(tmin, L.D, rows, cols, in_ld, L.tsl, w_x, w_y, nullptr, out_min, out_ld, out_slice, sepws,
                           L.sep, s);
  return rc;
}

#define MM_3D_INST(T)                                                                                      \
  template size_t filter3d_workspace<T>(int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t);    \
  template int launch_3d<T>(const void *, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t,  \
                            int64_t, void *, void *, int64_t, int64_t, void *, cudaStream_t);
MM_3D_INST(uint8_t)
MM_3D_INST(int8_t)
MM_3D_INST(uint16_t)
MM_3D_INST(int16_t)
MM_3D_INST(uint32_t)
MM_3D_INST(int32_t)
MM_3D_INST(uint64_t)
MM_3D_INST(int64_t)
MM_3D_INST(float)
MM_3D_INST(double)

}  // namespace mm

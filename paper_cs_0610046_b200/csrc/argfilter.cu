// argfilter.cu -- arg-max / arg-min filter: besides the
// max and min of every window, the position of each (the paper keeps
// locations so they come "with no overhead").  Ties: the
// EARLIEST position for both (reading R17).
//
// Every (value, position) pair travels as one 64-bit key whose order is the
// wanted one, so the argument filter IS a max (min) filter on keys and runs on
// the library's 8-byte kernels unchanged:
//   max side:  kx = ord(v) << 32 | (2^32-1 - i)   max key = max value, then
//                                                   the smallest position
//   min side:  kn = ord(v) << 32 | i               min key = min value, then
//                                                   the smallest position
// with ord() an order-preserving map of the <= 4-byte element type to uint32
// (floats: the sign-magnitude flip; +-0 both map to +0's code, reading R8).
// Three steps, all on the GPU: keys (elementwise), the max filter on kx and
// the min filter on kn (k1d_small/medium/large<uint64_t>), decode
// (elementwise).  The keys and the key outputs live in the workspace.  This is
// a composition, not a fused pass: ~92 B of HBM traffic per element against
// ~28 B for a fused kernel (N1).
#include "launch.cuh"

namespace mm {

template <typename T>
__device__ __forceinline__ uint32_t ord32(T v) {
  if constexpr (std::is_same<T, float>::value) {
    uint32_t b = __float_as_uint(v);
    if (v == 0.0f) b = 0u;  // -0 and +0 compare equal: one code
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  } else if constexpr (std::is_signed<T>::value) {
    return (uint32_t)(int32_t)v ^ 0x80000000u;
  } else {
    return (uint32_t)v;
  }
}
template <typename T>
__device__ __forceinline__ T unord32(uint32_t o) {
  if constexpr (std::is_same<T, float>::value) {
    const uint32_t b = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
    return __uint_as_float(b);
  } else if constexpr (std::is_signed<T>::value) {
    return (T)(int32_t)(o ^ 0x80000000u);
  } else {
    return (T)o;
  }
}

// keys of row b, positions [0, n): kx/kn rows of pitch kld (even)
template <typename T>
__global__ void __launch_bounds__(256) k_argkeys(const T *__restrict__ in, int64_t batch, int64_t n,
                                                 int64_t in_ld, uint64_t *__restrict__ kx,
                                                 uint64_t *__restrict__ kn, int64_t kld) {
  const int64_t half = (n + 1) / 2;  // pairs of positions per row
  const int64_t total = batch * half;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / half;
    const int64_t i = 2 * (t - b * half);
    const T *row = in + b * in_ld;
    const uint64_t o0 = (uint64_t)ord32<T>(row[i]) << 32;
    const uint64_t o1 = i + 1 < n ? (uint64_t)ord32<T>(row[i + 1]) << 32 : 0;
    const uint32_t i0 = (uint32_t)i, i1 = (uint32_t)(i + 1);
    const ulonglong2 vx = make_ulonglong2(o0 | (0xffffffffu - i0), o1 | (0xffffffffu - i1));
    const ulonglong2 vn = make_ulonglong2(o0 | i0, o1 | i1);
    *reinterpret_cast<ulonglong2 *>(kx + b * kld + i) = vx;
    *reinterpret_cast<ulonglong2 *>(kn + b * kld + i) = vn;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_argdecode(const uint64_t *__restrict__ okx,
                                                   const uint64_t *__restrict__ okn, int64_t batch,
                                                   int64_t m, int64_t kld, T *out_max, T *out_min,
                                                   int64_t *arg_max, int64_t *arg_min, int64_t out_ld) {
  const int64_t total = batch * m;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / m, j = t - b * m;
    const int64_t o = b * out_ld + j;
    if (okx) {
      const uint64_t k = okx[b * kld + j];
      if (out_max) out_max[o] = unord32<T>((uint32_t)(k >> 32));
      if (arg_max) arg_max[o] = (int64_t)(0xffffffffu - (uint32_t)k);
    }
    if (okn) {
      const uint64_t k = okn[b * kld + j];
      if (out_min) out_min[o] = unord32<T>((uint32_t)(k >> 32));
      if (arg_min) arg_min[o] = (int64_t)(uint32_t)k;
    }
  }
}

namespace {
struct ArgLayout {  // workspace: [kx | kn | okx | okn | inner], 256-B aligned pieces
  int64_t kld, mld;
  size_t keys, outs, inner, total;
};
size_t up256(size_t x) { return (x + 255) & ~size_t(255); }
ArgLayout arg_layout(int64_t batch, int64_t n, int64_t w) {
  ArgLayout L;
  const int64_t m = n - w + 1;
  L.kld = (n + 1) & ~int64_t(1);  // 16-B rows of 8-byte keys
  L.mld = (m + 1) & ~int64_t(1);
  L.keys = up256((size_t)batch * L.kld * 8);
  L.outs = up256((size_t)batch * L.mld * 8);
  L.inner = up256(workspace_1d<uint64_t>(batch, L.kld, w));
  L.total = 2 * L.keys + 2 * L.outs + L.inner;
  return L;
}
int grid_for(int64_t items) {
  int64_t g = (items + 255) / 256;
  const int64_t cap = (int64_t)sm_count() * 8;
  return (int)(g < cap ? (g > 0 ? g : 1) : cap);
}
}  // namespace

size_t argfilter_workspace(int64_t batch, int64_t n, int64_t w) { return arg_layout(batch, n, w).total; }

template <typename T>
int launch_argfilter(const void *in, int64_t batch, int64_t n, int64_t in_ld, int64_t w, void *out_max,
                     void *out_min, int64_t *arg_max, int64_t *arg_min, int64_t out_ld, void *ws,
                     size_t ws_bytes, cudaStream_t s) {
  static_assert(sizeof(T) <= 4, "keys hold a 32-bit order code and a 32-bit position");
  if (batch == 0) return kOK;
  const ArgLayout L = arg_layout(batch, n, w);
  if (!ws || ws_bytes < L.total) return kErrWorkspace;
  char *p = static_cast<char *>(ws);
  uint64_t *kx = reinterpret_cast<uint64_t *>(p);
  uint64_t *kn = reinterpret_cast<uint64_t *>(p + L.keys);
  uint64_t *okx = reinterpret_cast<uint64_t *>(p + 2 * L.keys);
  uint64_t *okn = reinterpret_cast<uint64_t *>(p + 2 * L.keys + L.outs);
  void *inner = p + 2 * L.keys + 2 * L.outs;
  const bool want_max = out_max || arg_max, want_min = out_min || arg_min;
  const int64_t m = n - w + 1;
  k_argkeys<T><<<grid_for(batch * ((n + 1) / 2)), 256, 0, s>>>(static_cast<const T *>(in), batch, n, in_ld,
                                                             kx, kn, L.kld);
  int rc = note_cuda(cudaGetLastError());
  if (rc) return rc;
  // the key rows hold n keys at pitch kld: the filter sees rows of length n
  if (want_max) {
    rc = launch_1d<uint64_t>(kx, batch, n, L.kld, w, okx, nullptr, L.mld, inner, L.inner, s);
    if (rc) return rc;
  }
  if (want_min) {
    rc = launch_1d<uint64_t>(kn, batch, n, L.kld, w, nullptr, okn, L.mld, inner, L.inner, s);
    if (rc) return rc;
  }
  k_argdecode<T><<<grid_for(batch * m), 256, 0, s>>>(want_max ? okx : nullptr, want_min ? okn : nullptr,
                                                    batch, m, L.mld, static_cast<T *>(out_max),
                                                    static_cast<T *>(out_min), arg_max, arg_min, out_ld);
  return note_cuda(cudaGetLastError());
}

#define MM_ARG_INST(T)                                                                           \
  template int launch_argfilter<T>(const void *, int64_t, int64_t, int64_t, int64_t, void *, void *, \
                                   int64_t *, int64_t *, int64_t, void *, size_t, cudaStream_t);
MM_ARG_INST(uint8_t)
MM_ARG_INST(int8_t)
MM_ARG_INST(uint16_t)
MM_ARG_INST(int16_t)
MM_ARG_INST(uint32_t)
MM_ARG_INST(int32_t)
MM_ARG_INST(float)

}  // namespace mm

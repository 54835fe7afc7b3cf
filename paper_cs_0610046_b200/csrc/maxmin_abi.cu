// maxmin_abi.cu -- the C ABI of libmaxmin.so (include/maxmin.h): argument
// validation, dtype dispatch, workspace queries and the host-buffer pipeline.
// No compute happens here; every step of the filter runs in the kernels of
// k1d.cuh / k2d.cuh.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "../../include/maxmin.h"
#include "launch.cuh"

#include <initializer_list>
#include <map>
#include <mutex>
#include <tuple>

namespace mm {

static thread_local int g_last_cuda_error = 0;

int note_cuda(cudaError_t e) {
  if (e == cudaSuccess) return kOK;
  g_last_cuda_error = (int)e;
  return kErrCuda;
}

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    cached[dev] = v;
  }
  return cached[dev];
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3-D map {RW, rows_per_series, batch} of 128-byte rows, boxes {RW, 8, 1},
// 128-byte swizzle, zero fill out of bounds (tma.cuh).
int encode_rows_map(CUtensorMap *map, const void *in, int elem_bytes, int64_t rows_per_series,
                    int64_t batch, int64_t in_ld_bytes, int box_rows, bool swizzle) {
  auto fn = encode_fn();
  if (!fn) return note_cuda(cudaErrorNotSupported);
  CUtensorMapDataType dt = elem_bytes == 1   ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                           : elem_bytes == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                           : elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32
                                             : CU_TENSOR_MAP_DATA_TYPE_UINT64;
  const cuuint64_t RW = 128 / elem_bytes;
  cuuint64_t dims[3] = {RW, (cuuint64_t)rows_per_series, (cuuint64_t)batch};
  cuuint64_t strides[2] = {128, (cuuint64_t)(batch > 1 ? in_ld_bytes : rows_per_series * 128)};
  cuuint32_t box[3] = {(cuuint32_t)RW, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, dt, 3, const_cast<void *>(in), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return note_cuda(cudaErrorInvalidValue);
  return kOK;
}

// Generic 3-D byte-element tiled map (no swizzle, zero fill): dims {d0, d1, d2},
// byte strides {s1, s2} of dims 1 and 2, box {b0, b1, b2}.  Used by the packed
// 1-byte 2-D kernel for its input stages and its output stores (k2d_byte.cu).
int encode_u8_map(CUtensorMap *map, const void *base, const int64_t dims[3], const int64_t strides[2],
                  const int box[3]) {
  auto fn = encode_fn();
  if (!fn) return note_cuda(cudaErrorNotSupported);
  cuuint64_t d[3] = {(cuuint64_t)dims[0], (cuuint64_t)dims[1], (cuuint64_t)dims[2]};
  cuuint64_t st[2] = {(cuuint64_t)strides[0], (cuuint64_t)strides[1]};
  cuuint32_t bx[3] = {(cuuint32_t)box[0], (cuuint32_t)box[1], (cuuint32_t)box[2]};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void *>(base), d, st, bx, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return note_cuda(cudaErrorInvalidValue);
  return kOK;
}

MM_DECLARE_INST(uint8_t)
MM_DECLARE_INST(int8_t)
MM_DECLARE_INST(uint16_t)
MM_DECLARE_INST(int16_t)
MM_DECLARE_INST(uint32_t)
MM_DECLARE_INST(int32_t)
MM_DECLARE_INST(uint64_t)
MM_DECLARE_INST(int64_t)
MM_DECLARE_INST(float)
MM_DECLARE_INST(double)

}  // namespace mm

#define MM_DISPATCH(dt, CALL)                   \
  switch (dt) {                                 \
    case MAXMIN_U8: { using T = uint8_t; CALL; } \
    case MAXMIN_I8: { using T = int8_t; CALL; }  \
    case MAXMIN_U16: { using T = uint16_t; CALL; } \
    case MAXMIN_I16: { using T = int16_t; CALL; }  \
    case MAXMIN_U32: { using T = uint32_t; CALL; } \
    case MAXMIN_I32: { using T = int32_t; CALL; }  \
    case MAXMIN_U64: { using T = uint64_t; CALL; } \
    case MAXMIN_I64: { using T = int64_t; CALL; }  \
    case MAXMIN_F32: { using T = float; CALL; }    \
    case MAXMIN_F64: { using T = double; CALL; }   \
    default: return MAXMIN_ERR_DTYPE;             \
  }

namespace mm {
static std::mutex g_launch_mu;  // guards the two maps below

// dynamic smem limit set so far, per (kernel, device); callers hold g_launch_mu
static int raise_smem_limit_locked(const void *kern, int dev, size_t b) {
  static std::map<std::pair<const void *, int>, size_t> attr;
  size_t &cur = attr[std::make_pair(kern, dev)];
  if (b <= cur) return kOK;
  cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b);
  if (r != cudaSuccess) return note_cuda(r);
  cur = b;
  return kOK;
}

int raise_smem_limit(const void *kern, size_t bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return note_cuda(e);
  std::lock_guard<std::mutex> lock(g_launch_mu);
  return raise_smem_limit_locked(kern, dev, bytes);
}

int blocks_per_sm(const void *kern, int threads, size_t smem, int *per_sm) {
  static std::map<std::tuple<const void *, int, int, size_t>, int> cache;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return note_cuda(e);
  std::lock_guard<std::mutex> lock(g_launch_mu);
  const auto key = std::make_tuple(kern, dev, threads, smem);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *per_sm = it->second;
    return kOK;
  }
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, kern, threads, smem);
  if (e != cudaSuccess) return note_cuda(e);
  cache[key] = *per_sm;
  return kOK;
}

int warp_launch_choice(const void *kern, int w, int max_nw, int min_nw, WarpBytesFn bytes, int prefer_warps,
                       WarpLaunch *out) {
  static std::map<std::pair<const void *, int64_t>, WarpLaunch> cache;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return note_cuda(e);
  std::lock_guard<std::mutex> lock(g_launch_mu);
  const auto key = std::make_pair(kern, (int64_t)w * 1024 + dev);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return kOK;
  }
  auto raise_limit = [&](size_t b) -> int { return raise_smem_limit_locked(kern, dev, b); };
  WarpLaunch best{0, 0, 0, 0};
  int64_t best_score = -1;
  for (int nw = max_nw; nw >= min_nw; nw /= 2) {
    for (int ns = 2; ns <= 4; ++ns) {
      const size_t b = bytes(w, ns, nw);
      if (b > 227 * 1024) continue;
      int rc = raise_limit(b);
      if (rc) return rc;
      int per = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 32 * nw, b);
      if (e != cudaSuccess) return note_cuda(e);
      if (per < 1) continue;
      const int64_t warps = (int64_t)per * nw;
      const int64_t score = prefer_warps ? warps * 8 + (ns - 1) : warps * (ns - 1);
      if (score > best_score) {
        best_score = score;
        best = WarpLaunch{ns, nw, per, b};
      }
    }
  }
  if (best_score < 0) return kErrUnsupported;
  cache[key] = best;
  *out = best;
  return kOK;
}
}  // namespace mm

namespace {

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// [lo, hi) byte ranges overlap?
bool overlap(const void *a, size_t abytes, const void *b, size_t bbytes) {
  uintptr_t a0 = (uintptr_t)a, a1 = a0 + abytes, b0 = (uintptr_t)b, b1 = b0 + bbytes;
  return a0 < b1 && b0 < a1;
}

// extent in bytes of `rows` rows of `len` elements with leading dimension ld
bool extent(int64_t rows, int64_t len, int64_t ld, size_t sz, size_t *bytes) {
  if (rows <= 0 || len <= 0) {
    *bytes = 0;
    return true;
  }
  const int64_t lim = INT64_MAX / (int64_t)sz / 2;
  if (ld > 0 && rows - 1 > lim / ld) return false;
  int64_t e = (rows - 1) * ld;
  if (e > lim - len) return false;
  *bytes = (size_t)(e + len) * sz;
  return true;
}

int validate_batched(int dt, const void *in, int64_t batch, int64_t n, int64_t in_ld, int64_t w,
                     const void *out_max, const void *out_min, int64_t out_ld) {
  const size_t sz = maxmin_dtype_size(dt);
  if (!sz) return MAXMIN_ERR_DTYPE;
  if (!in || (!out_max && !out_min)) return MAXMIN_ERR_NULL;
  if (w < 1) return MAXMIN_ERR_WINDOW;
  if (n < 1 || batch < 0) return MAXMIN_ERR_SHAPE;
  if (w > n) return MAXMIN_ERR_WINDOW_TOO_LARGE;
  const int64_t m = n - w + 1;
  if (in_ld < n || out_ld < m) return MAXMIN_ERR_SHAPE;
  size_t ib, ob;
  if (!extent(batch, n, in_ld, sz, &ib) || !extent(batch, m, out_ld, sz, &ob)) return MAXMIN_ERR_SHAPE;
  if (!aligned16(in) || (out_max && !aligned16(out_max)) || (out_min && !aligned16(out_min)))
    return MAXMIN_ERR_ALIGNMENT;
  if (batch > 1 && (((size_t)in_ld * sz) % 16 != 0 || ((size_t)out_ld * sz) % 16 != 0))
    return MAXMIN_ERR_ALIGNMENT;
  if (batch == 0) return MAXMIN_OK;
  if (out_max && overlap(in, ib, out_max, ob)) return MAXMIN_ERR_ALIAS;
  if (out_min && overlap(in, ib, out_min, ob)) return MAXMIN_ERR_ALIAS;
  if (out_max && out_min && overlap(out_max, ob, out_min, ob)) return MAXMIN_ERR_ALIAS;
  return MAXMIN_OK;
}

// Binds the calling thread to the device that owns every data pointer of one
// call for the duration of the call, and restores the caller's device on every
// exit path (the library links cudart statically, so a switch would otherwise
// leak into the caller's framework).  Pointers on different devices are an
// error, not a silent pick of the last one.
class DeviceScope {
 public:
  DeviceScope() = default;
  DeviceScope(const DeviceScope &) = delete;
  DeviceScope &operator=(const DeviceScope &) = delete;
  ~DeviceScope() {
    if (prev_ >= 0) cudaSetDevice(prev_);
  }
  int bind(std::initializer_list<const void *> ptrs) {
    int dev = -1;
    for (const void *p : ptrs) {
      if (!p) continue;
      cudaPointerAttributes a;
      cudaError_t e = cudaPointerGetAttributes(&a, p);
      if (e != cudaSuccess) {
        cudaGetLastError();
        return mm::note_cuda(e);
      }
      if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) return MAXMIN_ERR_MEMORY;
      if (dev < 0)
        dev = a.device;
      else if (a.device != dev)
        return MAXMIN_ERR_DEVICE;
    }
    if (dev < 0) return MAXMIN_OK;
    int cur = -1;
    cudaError_t e = cudaGetDevice(&cur);
    if (e != cudaSuccess) return mm::note_cuda(e);
    if (cur != dev) {
      e = cudaSetDevice(dev);
      if (e != cudaSuccess) return mm::note_cuda(e);
      prev_ = cur;
    }
    return MAXMIN_OK;
  }

 private:
  int prev_ = -1;
};

}  // namespace

extern "C" {

const char *maxmin_status_str(int status) {
  switch (status) {
    case MAXMIN_OK: return "ok";
    case MAXMIN_ERR_NULL: return "null pointer";
    case MAXMIN_ERR_DTYPE: return "unknown dtype";
    case MAXMIN_ERR_WINDOW: return "window < 1";
    case MAXMIN_ERR_WINDOW_TOO_LARGE: return "window larger than input";
    case MAXMIN_ERR_SHAPE: return "bad shape";
    case MAXMIN_ERR_ALIGNMENT: return "misaligned pointer or leading dimension";
    case MAXMIN_ERR_ALIAS: return "output overlaps input or the other output";
    case MAXMIN_ERR_WORKSPACE: return "workspace missing or too small";
    case MAXMIN_ERR_CUDA: return "CUDA error";
    case MAXMIN_ERR_UNSUPPORTED: return "unsupported by this build";
    case MAXMIN_ERR_MEMORY: return "pointer is not device memory";
    case MAXMIN_ERR_DEVICE: return "data pointers on different devices";
    case MAXMIN_ERR_NCCL: return "NCCL error";
    default: return "unknown status";
  }
}

int maxmin_last_cuda_error(void) { return mm::g_last_cuda_error; }

const char *maxmin_version(void) { return "maxmin-b200 0.1 sm_100a"; }

size_t maxmin_dtype_size(int dt) {
  switch (dt) {
    case MAXMIN_U8:
    case MAXMIN_I8: return 1;
    case MAXMIN_U16:
    case MAXMIN_I16: return 2;
    case MAXMIN_U32:
    case MAXMIN_I32:
    case MAXMIN_F32: return 4;
    case MAXMIN_U64:
    case MAXMIN_I64:
    case MAXMIN_F64: return 8;
    default: return 0;
  }
}

int maxmin_workspace_bytes(int dt, int64_t batch, int64_t n, int64_t w, size_t *bytes) {
  if (!bytes) return MAXMIN_ERR_NULL;
  *bytes = 0;
  if (!maxmin_dtype_size(dt)) return MAXMIN_ERR_DTYPE;
  if (w < 1) return MAXMIN_ERR_WINDOW;
  if (n < 1 || batch < 0) return MAXMIN_ERR_SHAPE;
  if (w > n) return MAXMIN_ERR_WINDOW_TOO_LARGE;
  MM_DISPATCH(dt, { *bytes = mm::workspace_1d<T>(batch, n, w); return MAXMIN_OK; })
}

int maxmin_filter_batched(int dt, const void *in, int64_t batch, int64_t n, int64_t in_ld, int64_t w,
                          void *out_max, void *out_min, int64_t out_ld, void *workspace,
                          size_t workspace_bytes, void *stream) {
  int rc = validate_batched(dt, in, batch, n, in_ld, w, out_max, out_min, out_ld);
  if (rc != MAXMIN_OK) return rc;
  size_t need = 0;
  rc = maxmin_workspace_bytes(dt, batch, n, w, &need);
  if (rc != MAXMIN_OK) return rc;
  if (need > 0 && (!workspace || workspace_bytes < need || !aligned16(workspace)))
    return MAXMIN_ERR_WORKSPACE;
  if (need > 0) {  // the workspace must not alias the data either
    size_t ib = 0;
    extent(batch, n, in_ld, maxmin_dtype_size(dt), &ib);
    if (overlap(workspace, need, in, ib)) return MAXMIN_ERR_ALIAS;
  }
  if (batch == 0) return MAXMIN_OK;
  DeviceScope dev;
  if ((rc = dev.bind({in, out_max, out_min, (need > 0) ? workspace : nullptr})) != MAXMIN_OK) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  MM_DISPATCH(dt, return mm::launch_1d<T>(in, batch, n, in_ld, w, out_max, out_min, out_ld,
                                          workspace, workspace_bytes, s))
}

int maxmin_filter_1d(int dt, const void *in, int64_t n, int64_t w, void *out_max, void *out_min,
                     void *workspace, size_t workspace_bytes, void *stream) {
  const int64_t m = n - w + 1;
  return maxmin_filter_batched(dt, in, 1, n, n, w, out_max, out_min, m > 0 ? m : 1, workspace,
                               workspace_bytes, stream);
}

// ------------------------------------------------------------ N3: LB_Keogh
int maxmin_lb_keogh_batched(int dt, const void *cand, int64_t batch, int64_t n, int64_t ld, const void *query,
                            int64_t r, double *lb, void *stream) {
  if (!maxmin_dtype_size(dt)) return MAXMIN_ERR_DTYPE;
  if (dt != MAXMIN_F32) return MAXMIN_ERR_UNSUPPORTED;
  if (!cand || !query || !lb) return MAXMIN_ERR_NULL;
  if (r < 0) return MAXMIN_ERR_WINDOW;
  if (n < 1 || batch < 0 || ld < n) return MAXMIN_ERR_SHAPE;
  if (2 * r + 1 <= n && 2 * r + 1 > mm::kHaloMax + 1) return MAXMIN_ERR_UNSUPPORTED;
  size_t cb = 0;
  if (!extent(batch, n, ld, 4, &cb)) return MAXMIN_ERR_SHAPE;
  if (!aligned16(cand) || (batch > 1 && (ld * 4) % 16 != 0)) return MAXMIN_ERR_ALIGNMENT;
  if (reinterpret_cast<uintptr_t>(query) % 4 || reinterpret_cast<uintptr_t>(lb) % 8) return MAXMIN_ERR_ALIGNMENT;
  if (batch == 0) return MAXMIN_OK;
  if (overlap(cand, cb, lb, (size_t)batch * 8) || overlap(query, (size_t)n * 4, lb, (size_t)batch * 8))
    return MAXMIN_ERR_ALIAS;
  int rc;
  DeviceScope dev;
  if ((rc = dev.bind({cand, query, lb})) != MAXMIN_OK) return rc;
  return mm::launch_keogh(static_cast<const float *>(cand), batch, n, ld, static_cast<const float *>(query), r,
                          lb, static_cast<cudaStream_t>(stream));
}

// ------------------------------------------------------------ N1: arg filter
int maxmin_argfilter_workspace_bytes(int dt, int64_t batch, int64_t n, int64_t w, size_t *bytes) {
  if (!bytes) return MAXMIN_ERR_NULL;
  *bytes = 0;
  const size_t sz = maxmin_dtype_size(dt);
  if (!sz) return MAXMIN_ERR_DTYPE;
  if (sz > 4) return MAXMIN_ERR_UNSUPPORTED;
  if (w < 1) return MAXMIN_ERR_WINDOW;
  if (n < 1 || batch < 0) return MAXMIN_ERR_SHAPE;
  if (w > n) return MAXMIN_ERR_WINDOW_TOO_LARGE;
  if (n > 0xffffffffLL) return MAXMIN_ERR_UNSUPPORTED;  // positions travel as 32 bits
  *bytes = mm::argfilter_workspace(batch, n, w);
  return MAXMIN_OK;
}

int maxmin_argfilter_batched(int dt, const void *in, int64_t batch, int64_t n, int64_t in_ld, int64_t w,
                             void *out_max, void *out_min, int64_t *arg_max, int64_t *arg_min,
                             int64_t out_ld, void *workspace, size_t workspace_bytes, void *stream) {
  const size_t sz = maxmin_dtype_size(dt);
  if (!sz) return MAXMIN_ERR_DTYPE;
  if (!in || (!out_max && !out_min && !arg_max && !arg_min)) return MAXMIN_ERR_NULL;
  if (w < 1) return MAXMIN_ERR_WINDOW;
  if (n < 1 || batch < 0) return MAXMIN_ERR_SHAPE;
  if (w > n) return MAXMIN_ERR_WINDOW_TOO_LARGE;
  size_t need = 0;
  int rc = maxmin_argfilter_workspace_bytes(dt, batch, n, w, &need);
  if (rc != MAXMIN_OK) return rc;
  const int64_t m = n - w + 1;
  if (in_ld < n || out_ld < m) return MAXMIN_ERR_SHAPE;
  size_t ib, ob, ab;
  if (!extent(batch, n, in_ld, sz, &ib) || !extent(batch, m, out_ld, sz, &ob) ||
      !extent(batch, m, out_ld, 8, &ab))
    return MAXMIN_ERR_SHAPE;
  auto el = [](const void *q, uintptr_t a) { return q == nullptr || (reinterpret_cast<uintptr_t>(q) % a) == 0; };
  if (!el(in, sz) || !el(out_max, sz) || !el(out_min, sz) || !el(arg_max, 8) || !el(arg_min, 8))
    return MAXMIN_ERR_ALIGNMENT;
  if (need > 0 && (!workspace || workspace_bytes < need || !aligned16(workspace))) return MAXMIN_ERR_WORKSPACE;
  if (batch == 0) return MAXMIN_OK;
  if (need == 0) workspace = nullptr;  // the fused path: nothing to check or touch
  const void *outs[4] = {out_max, out_min, arg_max, arg_min};
  const size_t obytes[4] = {ob, ob, ab, ab};
  for (int i = 0; i < 4; ++i) {
    if (!outs[i]) continue;
    if (overlap(in, ib, outs[i], obytes[i]) || (workspace && overlap(workspace, need, outs[i], obytes[i])))
      return MAXMIN_ERR_ALIAS;
    for (int k = i + 1; k < 4; ++k)
      if (outs[k] && overlap(outs[i], obytes[i], outs[k], obytes[k])) return MAXMIN_ERR_ALIAS;
  }
  if (workspace && overlap(workspace, need, in, ib)) return MAXMIN_ERR_ALIAS;
  DeviceScope dev;
  if ((rc = dev.bind({in, outs[0], outs[1], outs[2], outs[3], workspace})) != MAXMIN_OK) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  switch (dt) {
    case MAXMIN_U8: return mm::launch_argfilter<uint8_t>(in, batch, n, in_ld, w, out_max, out_min, arg_max, arg_min, out_ld, workspace, workspace_bytes, s);
    case MAXMIN_I8: return mm::launch_argfilter<int8_t>(in, batch, n, in_ld, w, out_max, out_min, arg_max, arg_min, out_ld, workspace, workspace_bytes, s);
    case MAXMIN_U16: return mm::launch_argfilter<uint16_t>(in, batch, n, in_ld, w, out_max, out_min, arg_max, arg_min, out_ld, workspace, workspace_bytes, s);
    case MAXMIN_I16: return mm::launch_argfilter<int16_t>(in, batch, n, in_ld, w, out_max, out_min, arg_max, arg_min, out_ld, workspace, workspace_bytes, s);
    case MAXMIN_U32: return mm::launch_argfilter<uint32_t>(in, batch, n, in_ld, w, out_max, out_min, arg_max, arg_min, out_ld, workspace, workspace_bytes, s);
    case MAXMIN_I32: return mm::launch_argfilter<int32_t>(in, batch, n, in_ld, w, out_max, out_min, arg_max, arg_min, out_ld, workspace, workspace_bytes, s);
    case MAXMIN_F32: return mm::launch_argfilter<float>(in, batch, n, in_ld, w, out_max, out_min, arg_max, arg_min, out_ld, workspace, workspace_bytes, s);
    default: return MAXMIN_ERR_UNSUPPORTED;
  }
}

namespace {
// argument checks of the 2-D calls; ib / ob: byte extents of the input and of one output
int validate_2d(int dt, const void *in, int64_t batch, int64_t rows, int64_t cols, int64_t in_ld,
                int64_t in_bstride, int64_t w_row, int64_t w_col, const void *out_max, const void *out_min,
                int64_t out_ld, int64_t out_bstride, size_t *ib, size_t *ob) {
  const size_t sz = maxmin_dtype_size(dt);
  if (!sz) return MAXMIN_ERR_DTYPE;
  if (!in || (!out_max && !out_min)) return MAXMIN_ERR_NULL;
  if (w_row < 1 || w_col < 1) return MAXMIN_ERR_WINDOW;
  if (batch < 0 || rows < 1 || cols < 1) return MAXMIN_ERR_SHAPE;
  if (w_row > cols || w_col > rows) return MAXMIN_ERR_WINDOW_TOO_LARGE;
  const int64_t R = rows - w_col + 1, C = cols - w_row + 1;
  if (in_ld < cols || out_ld < C) return MAXMIN_ERR_SHAPE;
  if (batch > 1 && (in_bstride < rows * in_ld || out_bstride < R * out_ld)) return MAXMIN_ERR_SHAPE;
  size_t t1, t2;
  if (!extent(rows, cols, in_ld, sz, &t1) || !extent(R, C, out_ld, sz, &t2)) return MAXMIN_ERR_SHAPE;
  if (!extent(batch, (int64_t)(t1 / sz), batch > 1 ? in_bstride : 0, sz, ib) ||
      !extent(batch, (int64_t)(t2 / sz), batch > 1 ? out_bstride : 0, sz, ob))
    return MAXMIN_ERR_SHAPE;
  // 2-D copies each box row separately (16-B aligned outward), so only element
  // alignment is required of pointers and strides.
  auto el_aligned = [sz](const void *p) { return (reinterpret_cast<uintptr_t>(p) % sz) == 0; };
  if (!el_aligned(in) || (out_max && !el_aligned(out_max)) || (out_min && !el_aligned(out_min)))
    return MAXMIN_ERR_ALIGNMENT;
  if (batch == 0) return MAXMIN_OK;
  if (out_max && overlap(in, *ib, out_max, *ob)) return MAXMIN_ERR_ALIAS;
  if (out_min && overlap(in, *ib, out_min, *ob)) return MAXMIN_ERR_ALIAS;
  if (out_max && out_min && overlap(out_max, *ob, out_min, *ob)) return MAXMIN_ERR_ALIAS;
  return MAXMIN_OK;
}
}  // namespace

int maxmin_filter_2d(int dt, const void *in, int64_t batch, int64_t rows, int64_t cols, int64_t in_ld,
                     int64_t in_bstride, int64_t w_row, int64_t w_col, void *out_max, void *out_min,
                     int64_t out_ld, int64_t out_bstride, void *stream) {
  size_t ib = 0, ob = 0;
  int rc = validate_2d(dt, in, batch, rows, cols, in_ld, in_bstride, w_row, w_col, out_max, out_min, out_ld,
                       out_bstride, &ib, &ob);
  if (rc != MAXMIN_OK || batch == 0) return rc;
  DeviceScope dev;
  if ((rc = dev.bind({in, out_max, out_min})) != MAXMIN_OK) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  MM_DISPATCH(dt, return mm::launch_2d<T>(in, batch, rows, cols, in_ld, in_bstride, w_row, w_col,
                                          out_max, out_min, out_ld, out_bstride, s))
}

int maxmin_filter_2d_workspace_bytes(int dt, int64_t batch, int64_t rows, int64_t cols, int64_t w_row, int64_t w_col,
                                     size_t *bytes) {
  if (!bytes) return MAXMIN_ERR_NULL;
  *bytes = 0;
  const size_t sz = maxmin_dtype_size(dt);
  if (!sz) return MAXMIN_ERR_DTYPE;
  if (w_row < 1 || w_col < 1) return MAXMIN_ERR_WINDOW;
  if (batch < 0 || rows < 1 || cols < 1) return MAXMIN_ERR_SHAPE;
  if (w_row > cols || w_col > rows) return MAXMIN_ERR_WINDOW_TOO_LARGE;
  size_t t;
  if (!extent(batch > 0 ? batch : 1, rows * (cols + 16), rows * (cols + 16), sz, &t)) return MAXMIN_ERR_SHAPE;
  // 1-byte pixels in the packed kernel's domain need no scratch (its alignment
  // rules aside: an unaligned call falls back to the fused generic kernel)
  if (sz == 1 && w_row == w_col && mm::k2b_supports(w_row)) return MAXMIN_OK;
  MM_DISPATCH(dt, { *bytes = mm::sep2d_workspace<T>(batch, rows, cols, w_row, w_col); return MAXMIN_OK; })
}

int maxmin_filter_2d_ws(int dt, const void *in, int64_t batch, int64_t rows, int64_t cols, int64_t in_ld,
                        int64_t in_bstride, int64_t w_row, int64_t w_col, void *out_max, void *out_min,
                        int64_t out_ld, int64_t out_bstride, void *workspace, size_t workspace_bytes, void *stream) {
  size_t ib = 0, ob = 0;
  int rc = validate_2d(dt, in, batch, rows, cols, in_ld, in_bstride, w_row, w_col, out_max, out_min, out_ld,
                       out_bstride, &ib, &ob);
  if (rc != MAXMIN_OK || batch == 0) return rc;
  size_t need = 0;
  if ((rc = maxmin_filter_2d_workspace_bytes(dt, batch, rows, cols, w_row, w_col, &need)) != MAXMIN_OK) return rc;
  if (workspace && !aligned16(workspace)) return MAXMIN_ERR_WORKSPACE;
  const size_t wsb = workspace ? workspace_bytes : 0;
  if (workspace && wsb) {
    if (overlap(workspace, wsb, in, ib) || (out_max && overlap(workspace, wsb, out_max, ob)) ||
        (out_min && overlap(workspace, wsb, out_min, ob)))
      return MAXMIN_ERR_ALIAS;
  }
  DeviceScope dev;
  if ((rc = dev.bind({in, out_max, out_min, (workspace && wsb) ? workspace : nullptr})) != MAXMIN_OK) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // the fused packed-byte kernel, else the separable streaming passes (when the
  // workspace suffices), else the fused generic kernel
  if (maxmin_dtype_size(dt) == 1) {
    rc = mm::launch_2d_byte(dt == MAXMIN_I8, in, batch, rows, cols, in_ld, in_bstride, w_row, w_col, out_max, out_min,
                            out_ld, out_bstride, s);
    if (rc != MAXMIN_ERR_UNSUPPORTED) return rc;
  }
  MM_DISPATCH(dt, {
    rc = mm::launch_2d_sep<T>(in, batch, rows, cols, in_ld, in_bstride, w_row, w_col, out_max, out_min, out_ld,
                              out_bstride, workspace, wsb, s);
    if (rc != MAXMIN_ERR_UNSUPPORTED) return rc;
    return mm::launch_2d<T>(in, batch, rows, cols, in_ld, in_bstride, w_row, w_col, out_max, out_min, out_ld,
                            out_bstride, s);
  })
}

// ------------------------------------------------------------ N2: streams
namespace {
bool stream_lay(int dt, int64_t streams, int64_t w, int64_t max_chunk, mm::StreamLayout *L) {
  const size_t sz = maxmin_dtype_size(dt);
  if (w - 1 > INT64_MAX / 4 - max_chunk) return false;
  size_t hb;
  if (!extent(streams, w - 1 + max_chunk + 16, w - 1 + max_chunk + 16, sz, &hb)) return false;
  MM_DISPATCH(dt, { *L = mm::stream_layout<T>(streams, w, max_chunk); return true; })
}
}  // namespace

int maxmin_stream_state_bytes(int dt, int64_t streams, int64_t w, int64_t max_chunk, size_t *bytes) {
  if (!bytes) return MAXMIN_ERR_NULL;
  *bytes = 0;
  if (!maxmin_dtype_size(dt)) return MAXMIN_ERR_DTYPE;
  if (w < 1) return MAXMIN_ERR_WINDOW;
  if (streams < 0 || max_chunk < 1) return MAXMIN_ERR_SHAPE;
  mm::StreamLayout L;
  if (!stream_lay(dt, streams, w, max_chunk, &L)) return MAXMIN_ERR_SHAPE;
  *bytes = L.total;
  return MAXMIN_OK;
}

int maxmin_stream_init(maxmin_stream *st, int dt, int64_t streams, int64_t w, int64_t max_chunk, void *state,
                       size_t state_bytes, void *stream) {
  if (!st) return MAXMIN_ERR_NULL;
  size_t need = 0;
  int rc = maxmin_stream_state_bytes(dt, streams, w, max_chunk, &need);
  if (rc != MAXMIN_OK) return rc;
  if (streams > 0 && !state) return MAXMIN_ERR_NULL;
  if (state && !aligned16(state)) return MAXMIN_ERR_ALIGNMENT;
  if (state_bytes < need) return MAXMIN_ERR_WORKSPACE;
  mm::StreamLayout L;
  stream_lay(dt, streams, w, max_chunk, &L);
  st->dtype = dt;
  st->phase = 0;
  st->streams = streams;
  st->w = w;
  st->max_chunk = max_chunk;
  st->ld = L.ld;
  st->seen = 0;
  st->state = state;
  st->state_bytes = state_bytes;
  if (streams == 0) return MAXMIN_OK;
  DeviceScope dev;
  if ((rc = dev.bind({state})) != MAXMIN_OK) return rc;
  return mm::note_cuda(cudaMemsetAsync(state, 0, L.fused ? 2 * L.hist_bytes : L.hist_bytes,
                                       static_cast<cudaStream_t>(stream)));
}

int maxmin_stream_push(maxmin_stream *st, const void *chunk, int64_t c, int64_t chunk_ld, void *out_max,
                       void *out_min, int64_t out_ld, int64_t *first_valid, void *stream) {
  if (!st || !first_valid) return MAXMIN_ERR_NULL;
  const int dt = st->dtype;
  const size_t sz = maxmin_dtype_size(dt);
  if (!sz) return MAXMIN_ERR_DTYPE;
  if (c < 0 || c > st->max_chunk || st->streams < 0 || st->w < 1) return MAXMIN_ERR_SHAPE;
  mm::StreamLayout L;
  if (!stream_lay(dt, st->streams, st->w, st->max_chunk, &L) || L.ld != st->ld || st->state_bytes < L.total)
    return MAXMIN_ERR_SHAPE;
  const int64_t h = st->w - 1;
  const int64_t fv = h - st->seen;
  *first_valid = fv < 0 ? 0 : (fv > c ? c : fv);
  if (c == 0 || st->streams == 0) return MAXMIN_OK;
  if (!st->state || !chunk || (!out_max && !out_min)) return MAXMIN_ERR_NULL;
  if (out_ld < c || chunk_ld < c) return MAXMIN_ERR_SHAPE;
  if (!aligned16(out_max) && out_max) return MAXMIN_ERR_ALIGNMENT;
  if (!aligned16(out_min) && out_min) return MAXMIN_ERR_ALIGNMENT;
  if (st->streams > 1 && ((size_t)out_ld * sz) % 16 != 0) return MAXMIN_ERR_ALIGNMENT;
  if (reinterpret_cast<uintptr_t>(chunk) % sz != 0) return MAXMIN_ERR_ALIGNMENT;
  size_t ob = 0, cb = 0;
  if (!extent(st->streams, c, out_ld, sz, &ob) || !extent(st->streams, c, chunk_ld, sz, &cb)) return MAXMIN_ERR_SHAPE;
  const void *regions[4] = {st->state, chunk, out_max, out_min};
  const size_t rbytes[4] = {L.total, cb, ob, ob};
  for (int i = 0; i < 4; ++i)
    for (int k = i + 1; k < 4; ++k)
      if (regions[i] && regions[k] && overlap(regions[i], rbytes[i], regions[k], rbytes[k])) return MAXMIN_ERR_ALIAS;
  int rc;
  DeviceScope dev;
  if ((rc = dev.bind({st->state, chunk, out_max, out_min})) != MAXMIN_OK) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  MM_DISPATCH(dt, {
    rc = mm::launch_stream_push<T>(st->state, L, st->streams, st->w, st->phase, static_cast<const T *>(chunk), c,
                                   chunk_ld, static_cast<T *>(out_max), static_cast<T *>(out_min), out_ld, s);
    break;
  })
  if (rc == MAXMIN_OK) {
    st->seen += c;
    if (L.fused) st->phase ^= 1;
  }
  return rc;
}

// ------------------------------------------------------------ N4: morphology
int maxmin_morph_batched(int dt, const void *in, int64_t batch, int64_t n, int64_t in_ld, int64_t w,
                         void *out_open, void *out_close, int64_t out_ld, void *stream) {
  const size_t sz = maxmin_dtype_size(dt);
  if (!sz) return MAXMIN_ERR_DTYPE;
  if (!in || (!out_open && !out_close)) return MAXMIN_ERR_NULL;
  if (w < 1) return MAXMIN_ERR_WINDOW;
  if (n < 1 || batch < 0) return MAXMIN_ERR_SHAPE;
  if (w > n) return MAXMIN_ERR_WINDOW_TOO_LARGE;
  if (w - 1 > 8192) return MAXMIN_ERR_UNSUPPORTED;  // (and when the staging does not fit shared memory)
  if (in_ld < n || out_ld < n) return MAXMIN_ERR_SHAPE;
  size_t ib, ob;
  if (!extent(batch, n, in_ld, sz, &ib) || !extent(batch, n, out_ld, sz, &ob)) return MAXMIN_ERR_SHAPE;
  if ((reinterpret_cast<uintptr_t>(in) % sz) != 0) return MAXMIN_ERR_ALIGNMENT;
  if ((out_open && !aligned16(out_open)) || (out_close && !aligned16(out_close))) return MAXMIN_ERR_ALIGNMENT;
  if (batch > 1 && ((size_t)out_ld * sz) % 16 != 0) return MAXMIN_ERR_ALIGNMENT;
  if (batch == 0) return MAXMIN_OK;
  if (out_open && overlap(in, ib, out_open, ob)) return MAXMIN_ERR_ALIAS;
  if (out_close && overlap(in, ib, out_close, ob)) return MAXMIN_ERR_ALIAS;
  if (out_open && out_close && overlap(out_open, ob, out_close, ob)) return MAXMIN_ERR_ALIAS;
  int rc;
  DeviceScope dev;
  if ((rc = dev.bind({in, out_open, out_close})) != MAXMIN_OK) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  MM_DISPATCH(dt, return mm::launch_morph<T>(in, batch, n, in_ld, w, out_open, out_close, out_ld, s))
}

int maxmin_morph_2d_workspace_bytes(int dt, int64_t batch, int64_t rows, int64_t cols, int64_t w_row,
                                    int64_t w_col, size_t *bytes) {
  if (!bytes) return MAXMIN_ERR_NULL;
  *bytes = 0;
  if (!maxmin_dtype_size(dt)) return MAXMIN_ERR_DTYPE;
  if (w_row < 1 || w_col < 1) return MAXMIN_ERR_WINDOW;
  if (batch < 0 || rows < 1 || cols < 1) return MAXMIN_ERR_SHAPE;
  if (w_row > cols || w_col > rows) return MAXMIN_ERR_WINDOW_TOO_LARGE;
  size_t t;
  if (!extent(batch, (rows + w_col) * (cols + w_row + 16), (rows + w_col) * (cols + w_row + 16), 8, &t))
    return MAXMIN_ERR_SHAPE;
  MM_DISPATCH(dt, { *bytes = mm::morph_2d_workspace<T>(batch, rows, cols, w_row, w_col); return MAXMIN_OK; })
}

int maxmin_morph_2d(int dt, const void *in, int64_t batch, int64_t rows, int64_t cols, int64_t in_ld,
                    int64_t in_bstride, int64_t w_row, int64_t w_col, void *out_open, void *out_close,
                    int64_t out_ld, int64_t out_bstride, void *workspace, size_t workspace_bytes, void *stream) {
  const size_t sz = maxmin_dtype_size(dt);
  if (!sz) return MAXMIN_ERR_DTYPE;
  if (!in || (!out_open && !out_close)) return MAXMIN_ERR_NULL;
  size_t need = 0;
  int rc = maxmin_morph_2d_workspace_bytes(dt, batch, rows, cols, w_row, w_col, &need);
  if (rc != MAXMIN_OK) return rc;
  if (in_ld < cols || out_ld < cols) return MAXMIN_ERR_SHAPE;
  if (batch > 1 && (in_bstride < rows * in_ld || out_bstride < rows * out_ld)) return MAXMIN_ERR_SHAPE;
  size_t ib, ob, t1, t2;
  if (!extent(rows, cols, in_ld, sz, &t1) || !extent(rows, cols, out_ld, sz, &t2)) return MAXMIN_ERR_SHAPE;
  if (!extent(batch, (int64_t)(t1 / sz), batch > 1 ? in_bstride : 0, sz, &ib) ||
      !extent(batch, (int64_t)(t2 / sz), batch > 1 ? out_bstride : 0, sz, &ob))
    return MAXMIN_ERR_SHAPE;
  auto el = [sz](const void *p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) % sz) == 0; };
  if (!el(in) || !el(out_open) || !el(out_close)) return MAXMIN_ERR_ALIGNMENT;
  if (!workspace || workspace_bytes < need || !aligned16(workspace)) return MAXMIN_ERR_WORKSPACE;
  if (batch == 0) return MAXMIN_OK;
  const void *regs[4] = {in, out_open, out_close, workspace};
  const size_t rb[4] = {ib, ob, ob, need};
  for (int i = 0; i < 4; ++i)
    for (int k = i + 1; k < 4; ++k)
      if (regs[i] && regs[k] && overlap(regs[i], rb[i], regs[k], rb[k])) return MAXMIN_ERR_ALIAS;
  DeviceScope dev;
  if ((rc = dev.bind({in, out_open, out_close, workspace})) != MAXMIN_OK) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  MM_DISPATCH(dt, return mm::launch_morph_2d<T>(in, batch, rows, cols, in_ld, in_bstride, w_row, w_col, out_open,
                                                out_close, out_ld, out_bstride, workspace, s))
}

// ------------------------------------------------------------ N4: 3-D boxes
int maxmin_filter_3d_workspace_bytes(int dt, int64_t depth, int64_t rows, int64_t cols, int64_t in_ld, int64_t w_x,
                                     int64_t w_y, int64_t w_z, size_t *bytes) {
  if (!bytes) return MAXMIN_ERR_NULL;
  *bytes = 0;
  const size_t sz = maxmin_dtype_size(dt);
  if (!sz) return MAXMIN_ERR_DTYPE;
  if (w_x < 1 || w_y < 1 || w_z < 1) return MAXMIN_ERR_WINDOW;
  if (depth < 1 || rows < 1 || cols < 1 || in_ld < cols) return MAXMIN_ERR_SHAPE;
  if (w_z > depth || w_x > cols || w_y > rows) return MAXMIN_ERR_WINDOW_TOO_LARGE;
  size_t t;
  if (!extent(depth, rows * in_ld + 16, rows * in_ld + 16, sz, &t)) return MAXMIN_ERR_SHAPE;
  MM_DISPATCH(dt, {
    *bytes = mm::filter3d_workspace<T>(depth, rows, cols, in_ld, w_x, w_y, w_z);
    return MAXMIN_OK;
  })
}

int maxmin_filter_3d(int dt, const void *in, int64_t depth, int64_t rows, int64_t cols, int64_t in_ld,
                     int64_t in_slice, int64_t w_x, int64_t w_y, int64_t w_z, void *out_max, void *out_min,
                     int64_t out_ld, int64_t out_slice, void *workspace, size_t workspace_bytes, void *stream) {
  const size_t sz = maxmin_dtype_size(dt);
  if (!sz) return MAXMIN_ERR_DTYPE;
  if (!in || (!out_max && !out_min)) return MAXMIN_ERR_NULL;
  if (w_x < 1 || w_y < 1 || w_z < 1) return MAXMIN_ERR_WINDOW;
  if (depth < 1 || rows < 1 || cols < 1) return MAXMIN_ERR_SHAPE;
  if (w_x > cols || w_y > rows || w_z > depth) return MAXMIN_ERR_WINDOW_TOO_LARGE;
  const int64_t D = depth - w_z + 1, R = rows - w_y + 1, C = cols - w_x + 1;
  if (in_ld < cols || out_ld < C || in_slice < rows * in_ld || (D > 1 && out_slice < R * out_ld))
    return MAXMIN_ERR_SHAPE;
  size_t need = 0;
  int rc = maxmin_filter_3d_workspace_bytes(dt, depth, rows, cols, in_ld, w_x, w_y, w_z, &need);
  if (rc != MAXMIN_OK) return rc;
  size_t t1, t2, ib, ob;
  if (!extent(rows, cols, in_ld, sz, &t1) || !extent(R, C, out_ld, sz, &t2)) return MAXMIN_ERR_SHAPE;
  if (!extent(depth, (int64_t)(t1 / sz), in_slice, sz, &ib) || !extent(D, (int64_t)(t2 / sz), D > 1 ? out_slice : 0, sz, &ob))
    return MAXMIN_ERR_SHAPE;
  auto el = [sz](const void *p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) % sz) == 0; };
  if (!el(in) || !el(out_max) || !el(out_min)) return MAXMIN_ERR_ALIGNMENT;
  if (!workspace || workspace_bytes < need || !aligned16(workspace)) return MAXMIN_ERR_WORKSPACE;
  const void *regs[4] = {in, out_max, out_min, workspace};
  const size_t rb[4] = {ib, ob, ob, need};
  for (int i = 0; i < 4; ++i)
    for (int k = i + 1; k < 4; ++k)
      if (regs[i] && regs[k] && overlap(regs[i], rb[i], regs[k], rb[k])) return MAXMIN_ERR_ALIAS;
  DeviceScope dev;
  if ((rc = dev.bind({in, out_max, out_min, workspace})) != MAXMIN_OK) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  MM_DISPATCH(dt, return mm::launch_3d<T>(in, depth, rows, cols, in_ld, in_slice, w_x, w_y, w_z, out_max, out_min,
                                          out_ld, out_slice, workspace, s))
}

// ------------------------------------------------------------ host pipeline
static int64_t default_chunk(int64_t chunk) { return chunk > 0 ? chunk : (int64_t(1) << 24); }

int maxmin_host_workspace_bytes(int dt, int64_t n, int64_t w, int64_t chunk, size_t *bytes) {
  if (!bytes) return MAXMIN_ERR_NULL;
  *bytes = 0;
  const size_t sz = maxmin_dtype_size(dt);
  if (!sz) return MAXMIN_ERR_DTYPE;
  if (w < 1) return MAXMIN_ERR_WINDOW;
  if (n < 1) return MAXMIN_ERR_SHAPE;
  if (w > n) return MAXMIN_ERR_WINDOW_TOO_LARGE;
  const int64_t m = n - w + 1;
  int64_t c = default_chunk(chunk);
  if (c > m) c = m;
  size_t ws = 0;
  int rc = maxmin_workspace_bytes(dt, 1, c + w - 1, w, &ws);
  if (rc) return rc;
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t per = up((size_t)(c + w - 1 + 16) * sz) + 2 * up((size_t)c * sz) + up(ws);
  *bytes = 2 * per;
  return MAXMIN_OK;
}

int maxmin_filter_1d_host(int dt, const void *in, int64_t n, int64_t w, void *out_max, void *out_min,
                          int64_t chunk, void *dev_ws, size_t ws_bytes) {
  const size_t sz = maxmin_dtype_size(dt);
  if (!sz) return MAXMIN_ERR_DTYPE;
  if (!in || (!out_max && !out_min)) return MAXMIN_ERR_NULL;
  size_t need = 0;
  int rc = maxmin_host_workspace_bytes(dt, n, w, chunk, &need);
  if (rc) return rc;
  if (!dev_ws || ws_bytes < need || !aligned16(dev_ws)) return MAXMIN_ERR_WORKSPACE;
  DeviceScope dev;
  if ((rc = dev.bind({dev_ws})) != MAXMIN_OK) return rc;
  const int64_t m = n - w + 1;
  int64_t c = default_chunk(chunk);
  if (c > m) c = m;
  size_t kws = 0;
  maxmin_workspace_bytes(dt, 1, c + w - 1, w, &kws);
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t per = need / 2;
  // two non-blocking streams per (thread, device), created on first use and
  // kept: creating and destroying them cost more than a small call
  thread_local std::map<int, std::pair<cudaStream_t, cudaStream_t>> pool;
  int dev_id = 0;
  cudaError_t ge = cudaGetDevice(&dev_id);
  if (ge != cudaSuccess) return mm::note_cuda(ge);
  auto pit = pool.find(dev_id);
  if (pit == pool.end()) {
    cudaStream_t a = nullptr, b = nullptr;
    if ((ge = cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking)) != cudaSuccess) return mm::note_cuda(ge);
    if ((ge = cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking)) != cudaSuccess) {
      cudaStreamDestroy(a);
      return mm::note_cuda(ge);
    }
    pit = pool.emplace(dev_id, std::make_pair(a, b)).first;
  }
  cudaStream_t st[2] = {pit->second.first, pit->second.second};
  const char *hin = static_cast<const char *>(in);
  int64_t k = 0;
  for (int64_t j0 = 0; j0 < m && rc == MAXMIN_OK; j0 += c, ++k) {
    const int64_t cw = m - j0 < c ? m - j0 : c;  // windows in this chunk
    const int64_t len = cw + w - 1;              // input elements
    char *base = static_cast<char *>(dev_ws) + (k & 1) * per;
    char *din = base;
    char *dmx = din + up((size_t)(c + w - 1 + 16) * sz);
    char *dmn = dmx + up((size_t)c * sz);
    char *dws = dmn + up((size_t)c * sz);
    cudaStream_t s = st[k & 1];
    cudaError_t e = cudaMemcpyAsync(din, hin + (size_t)j0 * sz, (size_t)len * sz, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) { rc = mm::note_cuda(e); break; }
    rc = maxmin_filter_1d(dt, din, len, w, out_max ? dmx : nullptr, out_min ? dmn : nullptr,
                          kws ? dws : nullptr, kws, s);
    if (rc) break;
    if (out_max) {
      e = cudaMemcpyAsync(static_cast<char *>(out_max) + (size_t)j0 * sz, dmx, (size_t)cw * sz,
                          cudaMemcpyDeviceToHost, s);
      if (e != cudaSuccess) { rc = mm::note_cuda(e); break; }
    }
    if (out_min) {
      e = cudaMemcpyAsync(static_cast<char *>(out_min) + (size_t)j0 * sz, dmn, (size_t)cw * sz,
                          cudaMemcpyDeviceToHost, s);
      if (e != cudaSuccess) { rc = mm::note_cuda(e); break; }
    }
  }
  for (auto &s : st) {
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess && rc == MAXMIN_OK) rc = mm::note_cuda(e);
  }
  return rc;
}

}  // extern "C"

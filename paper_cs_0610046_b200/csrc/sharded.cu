// sharded.cu -- the 1-D filter of one array split over ranks (
// include/maxmin.h maxmin_filter_1d_sharded).
//
// Rank r owns the contiguous chunk [c_r, c_{r+1}) of the global array and emits
// every window that STARTS in it.  The windows of the last w-1 starts reach
// into rank r+1's chunk: that rank's first `halo` elements are the only remote
// data, received by one NCCL point-to-point message per boundary (send the own
// first `halo` elements to r-1, receive r+1's into the slot after the chunk),
// on the caller's comm stream.  The interior windows need nothing remote and
// run on the compute stream while the message is in flight; the tail windows
// wait for the receive's event.  Every window of every rank is computed by the
// same kernels as maxmin_filter_1d (this file only orders calls and streams).
//
// NCCL is bound at run time (dlopen): in a PyTorch process the library that
// torch already loaded is reused (RTLD_NOLOAD), so the communicator handle the
// caller passes -- e.g. ProcessGroupNCCL's -- belongs to the same libnccl.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdint>
#include <map>
#include <mutex>

#include "../../include/maxmin.h"

namespace {

struct NcclApi {
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*count)(const ncclComm_t, int *) = nullptr;
  ncclResult_t (*user_rank)(const ncclComm_t, int *) = nullptr;
  bool ok = false;
};

const NcclApi &nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void *h = dlopen("libnccl.so.2", RTLD_LAZY | RTLD_NOLOAD);  // the one already in the process
    if (!h) h = dlopen("libnccl.so.2", RTLD_LAZY | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_LAZY | RTLD_GLOBAL);
    if (!h) return;
    api.group_start = reinterpret_cast<decltype(api.group_start)>(dlsym(h, "ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(api.group_end)>(dlsym(h, "ncclGroupEnd"));
    api.send = reinterpret_cast<decltype(api.send)>(dlsym(h, "ncclSend"));
    api.recv = reinterpret_cast<decltype(api.recv)>(dlsym(h, "ncclRecv"));
    api.count = reinterpret_cast<decltype(api.count)>(dlsym(h, "ncclCommCount"));
    api.user_rank = reinterpret_cast<decltype(api.user_rank)>(dlsym(h, "ncclCommUserRank"));
    api.ok = api.group_start && api.group_end && api.send && api.recv && api.count && api.user_rank;
  });
  return api;
}

thread_local int g_last_nccl_error = 0;

// Two timing-free events per (thread, device), created once: "chunk ready" on
// the compute stream and "halo received" on the comm stream.
int events_for(int dev, cudaEvent_t *ready, cudaEvent_t *halo) {
  thread_local std::map<int, std::pair<cudaEvent_t, cudaEvent_t>> cache;
  auto it = cache.find(dev);
  if (it == cache.end()) {
    cudaEvent_t a = nullptr, b = nullptr;
    if (cudaEventCreateWithFlags(&a, cudaEventDisableTiming) != cudaSuccess) return MAXMIN_ERR_CUDA;
    if (cudaEventCreateWithFlags(&b, cudaEventDisableTiming) != cudaSuccess) {
      cudaEventDestroy(a);
      return MAXMIN_ERR_CUDA;
    }
    it = cache.emplace(dev, std::make_pair(a, b)).first;
  }
  *ready = it->second.first;
  *halo = it->second.second;
  return MAXMIN_OK;
}

// First window start recomputed by the tail call of window w: windows from
// n_local-w+1 on touch the halo; the start is aligned down to 64 elements so
// the input and output pointers of the tail call stay 16-byte aligned (it
// recomputes fewer than 64 interior windows, bit-identically).
int64_t tail_start(int64_t n_local, int64_t w) {
  int64_t first_remote = n_local - w + 1;
  if (first_remote < 0) first_remote = 0;
  return first_remote / 64 * 64;
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

extern "C" {

int maxmin_last_nccl_error(void) { return g_last_nccl_error; }

int maxmin_sharded_workspace_bytes(int dt, int64_t n_local, int64_t halo, const int64_t *windows, int nwin,
                                   size_t *bytes) {
  if (!bytes || (nwin > 0 && !windows)) return MAXMIN_ERR_NULL;
  *bytes = 0;
  if (!maxmin_dtype_size(dt)) return MAXMIN_ERR_DTYPE;
  if (n_local < 1 || halo < 0 || nwin < 0) return MAXMIN_ERR_SHAPE;
  size_t best = 0;
  for (int k = 0; k < nwin; ++k) {
    const int64_t w = windows[k];
    if (w < 1) return MAXMIN_ERR_WINDOW;
    if (w - 1 > halo) return MAXMIN_ERR_WINDOW_TOO_LARGE;
    size_t b = 0;  // the interior call (n_local) and the tail call (< 64 + 2w) share it, in stream order
    int rc = maxmin_workspace_bytes(dt, 1, n_local + w - 1, w, &b);
    if (rc != MAXMIN_OK) return rc;
    if (b > best) best = b;
  }
  *bytes = best;
  return MAXMIN_OK;
}

int maxmin_filter_1d_sharded(int dt, void *local, int64_t n_local, int64_t halo, const int64_t *windows,
                             int nwin, int rank, int nranks, void *nccl_comm, void *const *out_max,
                             void *const *out_min, void *workspace, size_t workspace_bytes, void *stream,
                             void *comm_stream) {
  const size_t sz = maxmin_dtype_size(dt);
  if (!sz) return MAXMIN_ERR_DTYPE;
  if (!local || !windows || !out_max || !out_min) return MAXMIN_ERR_NULL;
  if (nranks < 1 || rank < 0 || rank >= nranks || nwin < 1) return MAXMIN_ERR_SHAPE;
  const bool last = rank == nranks - 1;
  size_t need = 0;
  int rc = maxmin_sharded_workspace_bytes(dt, n_local, halo, windows, nwin, &need);
  if (rc != MAXMIN_OK) return rc;
  if (need > 0 && (!workspace || workspace_bytes < need || !aligned16(workspace))) return MAXMIN_ERR_WORKSPACE;
  for (int k = 0; k < nwin; ++k) {
    if (!out_max[k] && !out_min[k]) return MAXMIN_ERR_NULL;
    if (last && windows[k] > n_local) return MAXMIN_ERR_WINDOW_TOO_LARGE;
  }
  if (!aligned16(local)) return MAXMIN_ERR_ALIGNMENT;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaStream_t cs = static_cast<cudaStream_t>(comm_stream ? comm_stream : stream);
  const bool exchange = nranks > 1 && nccl_comm != nullptr && halo > 0;

  cudaPointerAttributes pa;
  cudaError_t e = cudaPointerGetAttributes(&pa, local);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return MAXMIN_ERR_CUDA;
  }
  if (pa.type != cudaMemoryTypeDevice && pa.type != cudaMemoryTypeManaged) return MAXMIN_ERR_MEMORY;
  int prev = -1;
  if (cudaGetDevice(&prev) != cudaSuccess) return MAXMIN_ERR_CUDA;
  struct Restore {  // the caller's device on every exit path
    int prev, dev;
    ~Restore() {
      if (prev != dev) cudaSetDevice(prev);
    }
  } restore{prev, pa.device};
  if (prev != pa.device && cudaSetDevice(pa.device) != cudaSuccess) return MAXMIN_ERR_CUDA;

  cudaEvent_t ev_ready = nullptr, ev_halo = nullptr;
  if (exchange) {
    const NcclApi &api = nccl();
    if (!api.ok) return MAXMIN_ERR_NCCL;
    ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
    int cn = 0, cr = -1;
    ncclResult_t r = api.count(comm, &cn);
    if (r == ncclSuccess) r = api.user_rank(comm, &cr);
    if (r != ncclSuccess) {
      g_last_nccl_error = (int)r;
      return MAXMIN_ERR_NCCL;
    }
    if (cn != nranks || cr != rank) return MAXMIN_ERR_SHAPE;  // the communicator disagrees with rank/nranks
    if ((rc = events_for(pa.device, &ev_ready, &ev_halo)) != MAXMIN_OK) return rc;
    // the chunk (written by work ordered before this call on `stream`) is ready to send
    if ((e = cudaEventRecord(ev_ready, s)) != cudaSuccess || (e = cudaStreamWaitEvent(cs, ev_ready, 0)) != cudaSuccess)
      return MAXMIN_ERR_CUDA;
    char *base = static_cast<char *>(local);
    r = api.group_start();
    if (r == ncclSuccess && rank > 0) r = api.send(base, (size_t)halo * sz, ncclUint8, rank - 1, comm, cs);
    if (r == ncclSuccess && !last) r = api.recv(base + (size_t)n_local * sz, (size_t)halo * sz, ncclUint8, rank + 1, comm, cs);
    ncclResult_t r2 = api.group_end();
    if (r == ncclSuccess) r = r2;
    if (r != ncclSuccess) {
      g_last_nccl_error = (int)r;
      return MAXMIN_ERR_NCCL;
    }
    if (cudaEventRecord(ev_halo, cs) != cudaSuccess) return MAXMIN_ERR_CUDA;
  }
  // interior: the windows inside the own chunk, while the halo is in flight
  for (int k = 0; k < nwin; ++k) {
    const int64_t w = windows[k];
    if (n_local - w + 1 <= 0) continue;
    rc = maxmin_filter_1d(dt, local, n_local, w, out_max[k], out_min[k], workspace, workspace_bytes, s);
    if (rc != MAXMIN_OK) return rc;
  }
  if (last) return MAXMIN_OK;
  if (exchange && cudaStreamWaitEvent(s, ev_halo, 0) != cudaSuccess) return MAXMIN_ERR_CUDA;
  // tail: the windows that reach into the halo (input [t, n_local + w - 1))
  for (int k = 0; k < nwin; ++k) {
    const int64_t w = windows[k];
    const int64_t t = tail_start(n_local, w);
    const int64_t len = n_local - t + w - 1;
    char *in = static_cast<char *>(local) + (size_t)t * sz;
    char *omx = out_max[k] ? static_cast<char *>(out_max[k]) + (size_t)t * sz : nullptr;
    char *omn = out_min[k] ? static_cast<char *>(out_min[k]) + (size_t)t * sz : nullptr;
    rc = maxmin_filter_1d(dt, in, len, w, omx, omn, workspace, workspace_bytes, s);
    if (rc != MAXMIN_OK) return rc;
  }
  return MAXMIN_OK;
}

}  // extern "C"

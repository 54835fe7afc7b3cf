// keogh.cu -- LB_Keogh fused with the envelope.
//
// "[keogh2005eid] use a precomputed max-min filter to approximate the time
// warping distance between two time series".  For every
// candidate row c (n samples) and one query q, warping radius r:
//   U_i, L_i = max, min of c over [max(0,i-r), min(n-1,i+r)]   (reading R18)
//   lb = sqrt( sum_i (q_i > U_i) ? (q_i-U_i)^2 : (q_i < L_i) ? (L_i-q_i)^2 : 0 )
// The envelope is never written: the interior positions i in [r, n-1-r] are
// the full windows j = i - r of the max-min filter with w = 2r+1, computed by
// the library's k1d_small / k1d_medium kernels with an epilogue that folds
// them into the bound (per warp: a shuffle reduction, one double atomic per
// row); the 2r clipped positions at the two ends of every row are running
// prefix / suffix extrema (k_keogh_ends, one warp per row); a last pass takes
// the square roots.  HBM traffic: the candidates once (+ the 2r end samples of
// every row again) and 8 bytes per row.  Squares and sums are in double: the
// order differs from the oracle's, so parity is to a relative 1e-12.
#include "launch.cuh"

namespace mm {

struct KeoghEpi {
  const float *q;  // query, n samples
  int64_t r;
  double *acc;     // per row: the running sum of squares (the output, pre-sqrt)
  // the excess of q_i over the envelope: the operand pair is selected in float
  // ((q_i, U_i), (L_i, q_i) or (0, 0)), so each element costs one conversion
  // pair and one subtraction in double -- the same value as the branch-wise form
  __device__ __forceinline__ static double diff(float qv, float u, float l) {
    const bool hi = qv > u, lo = qv < l;
    const float a = hi ? qv : (lo ? l : 0.f), b = hi ? u : (lo ? qv : 0.f);
    return (double)a - (double)b;
  }
  __device__ __forceinline__ static double term(float qv, float u, float l) {
    const double d = diff(qv, u, l);
    return d * d;
  }
  __device__ __forceinline__ static double acc_term(double s, float qv, float u, float l) {
    const double d = diff(qv, u, l);
    return fma(d, d, s);  // one DFMA per element
  }
  template <typename T, int E>
  __device__ __forceinline__ void operator()(const Rows &p, int64_t row, int64_t j0, int cnt, const T (&ox)[E],
                                             const T (&on)[E]) const {
    static_assert(sizeof(T) == 4, "float rows");
    double s = 0.0;
    const float *qp = q + j0 + r;  // window j -> position j + r
    if (cnt >= E && (reinterpret_cast<uintptr_t>(qp) & 15) == 0) {  // 16-B query loads
#pragma unroll
      for (int k = 0; k < E; k += 4) {
        const float4 v = __ldg(reinterpret_cast<const float4 *>(qp + k));
        s = acc_term(s, v.x, ox[k], on[k]);
        s = acc_term(s, v.y, ox[k + 1], on[k + 1]);
        s = acc_term(s, v.z, ox[k + 2], on[k + 2]);
        s = acc_term(s, v.w, ox[k + 3], on[k + 3]);
      }
    } else {
#pragma unroll
      for (int k = 0; k < E; ++k)
        if (k < cnt) s = acc_term(s, __ldg(qp + k), ox[k], on[k]);
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
    if ((threadIdx.x & 31) == 0 && s != 0.0) atomicAdd(acc + row, s);
  }
};

// The clipped ends of every row: positions i < r read the prefix extrema of c
// up to min(n-1, i+r); positions i > n-1-r (and i >= r) the suffix extrema of
// c from i-r.  One warp per row; 32-element chunks with shuffle scans.
__global__ void __launch_bounds__(256) k_keogh_ends(const float *__restrict__ c, int64_t batch, int64_t n,
                                                    int64_t ld, const float *__restrict__ q, int64_t r,
                                                    double *acc) {
  const int lane = threadIdx.x & 31;
  const int64_t row = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  if (row >= batch) return;
  const float *x = c + row * ld;
  double s = 0.0;
  if (r == 0) {  // U = L = c
    for (int64_t i = lane; i < n; i += 32) s += KeoghEpi::term(q[i], x[i], x[i]);
  }
  // ---- left: prefix extrema P[e], e in [0, min(n, 2r)); position i = e - r, or
  //      every i in [max(0, n-1-r), min(r, n)) at e = n-1 (windows [0, n-1])
  {
    const int64_t eend = n < 2 * r ? n : 2 * r;
    float cx = -INFINITY, cn = INFINITY;  // carry
    for (int64_t base = 0; base < eend; base += 32) {
      const int64_t e = base + lane;
      float vx = e < eend ? x[e] : -INFINITY, vn = e < eend ? x[e] : INFINITY;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const float ux = __shfl_up_sync(0xffffffffu, vx, d), un = __shfl_up_sync(0xffffffffu, vn, d);
        if (lane >= d) {
          vx = fmaxf(vx, ux);
          vn = fminf(vn, un);
        }
      }
      vx = fmaxf(vx, cx);
      vn = fminf(vn, cn);
      if (e < eend) {
        if (e < n - 1) {
          const int64_t i = e - r;
          if (i >= 0 && i < r) s += KeoghEpi::term(q[i], vx, vn);
        } else {  // e == n-1: windows reaching both ends
          const int64_t i0 = n - 1 - r > 0 ? n - 1 - r : 0, i1 = r < n ? r : n;
          for (int64_t i = i0; i < i1; ++i) s += KeoghEpi::term(q[i], vx, vn);
        }
      }
      cx = __shfl_sync(0xffffffffu, vx, 31);
      cn = __shfl_sync(0xffffffffu, vn, 31);
    }
  }
  // ---- right: suffix extrema S[lo] for lo in [max(0, n-2r), n-1-r]; the
  //      position is i = lo + r (i >= max(r, n-r)); the suffix starts at n-1
  if (n - 1 - r >= 0) {
    const int64_t lo_min = n - 2 * r > 0 ? n - 2 * r : 0;
    const int64_t i_min = r > n - r ? r : n - r;  // positions already done on the left: i < r
    float cx = -INFINITY, cn = INFINITY;
    for (int64_t top = n - 1; top >= lo_min; top -= 32) {
      const int64_t e = top - lane;
      float vx = e >= lo_min ? x[e] : -INFINITY, vn = e >= lo_min ? x[e] : INFINITY;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const float ux = __shfl_up_sync(0xffffffffu, vx, d), un = __shfl_up_sync(0xffffffffu, vn, d);
        if (lane >= d) {
          vx = fmaxf(vx, ux);
          vn = fminf(vn, un);
        }
      }
      vx = fmaxf(vx, cx);
      vn = fminf(vn, cn);
      if (e >= lo_min) {
        const int64_t i = e + r;
        if (i >= i_min && i < n) s += KeoghEpi::term(q[i], vx, vn);
      }
      cx = __shfl_sync(0xffffffffu, vx, 31);
      cn = __shfl_sync(0xffffffffu, vn, 31);
    }
  }
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
  if (lane == 0 && s != 0.0) atomicAdd(acc + row, s);
}

__global__ void k_keogh_sqrt(double *lb, int64_t batch) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < batch; b += (int64_t)gridDim.x * blockDim.x)
    lb[b] = sqrt(lb[b]);
}

int launch_keogh(const float *c, int64_t batch, int64_t n, int64_t ld, const float *q, int64_t r, double *lb,
                 cudaStream_t s) {
  if (batch == 0) return kOK;
  cudaError_t e = cudaMemsetAsync(lb, 0, sizeof(double) * (size_t)batch, s);
  if (e != cudaSuccess) return note_cuda(e);
  const int64_t w = 2 * r + 1;
  if (w <= n && w >= 2) {  // interior: the max-min filter with the bound as epilogue
    Rows p;
    std::memset(&p, 0, sizeof(p));
    p.in = c;
    p.n = n;
    p.w = w;
    p.m = n - w + 1;
    p.in_ld = ld;
    p.out_ld = p.m;
    p.batch = batch;
    p.tiles_per_row = (p.m + Geo1D<float>::TILE - 1) / Geo1D<float>::TILE;
    p.ntiles = batch * p.tiles_per_row;
    CUtensorMap map;
    std::memset(&map, 0, sizeof(map));
    const int64_t full_rows = n / Rowing<float>::RW;
    p.has_map = full_rows > 0 ? 1 : 0;
    if (p.has_map) {
      int rc = encode_rows_map(&map, c, 4, full_rows, batch, ld * 4);
      if (rc) return rc;
    }
    KeoghEpi epi{q, r, lb};
    int rc;
    switch (path_1d<float>(w)) {
      case Path1D::Small:
        rc = launch_small_epi<float>(p, map, s, epi);
        break;
      case Path1D::Medium:
        rc = launch_medium_epi<float>(p, map, s, epi);
        break;
      default:
        rc = kErrUnsupported;  // r > 4096: the look-back kernels have no epilogue yet
    }
    if (rc) return rc;
  }
  {  // the clipped ends (every position when w > n; r == 0: every position, U = L = c)
    const int rows_per_cta = 8;
    k_keogh_ends<<<(unsigned)((batch + rows_per_cta - 1) / rows_per_cta), 32 * rows_per_cta, 0, s>>>(
        c, batch, n, ld, q, r, lb);
    int rc = note_cuda(cudaGetLastError());
    if (rc) return rc;
  }
  k_keogh_sqrt<<<(unsigned)((batch + 255) / 256 < 1024 ? (batch + 255) / 256 : 1024), 256, 0, s>>>(lb, batch);
  return note_cuda(cudaGetLastError());
}

}  // namespace mm

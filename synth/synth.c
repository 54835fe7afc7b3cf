/*
 * synth.c -- seeded synthetic inputs for the max-min filter workloads.
 *
 * This module holds NO arithmetic of the method (no max/min filtering).  It is
 * the one piece shared by the oracle side (tests) and the product side (bench
 * inputs): both consume the arrays it writes.  Every value is a pure function
 * of (seed, stream, counter) through SplitMix64, so any sub-range can be
 * generated independently and in parallel with identical results.
 *
 * Workload recipes (BASELINE.json configs, fixed choices in DESIGN.md "Inputs"):
 *   C1  f64 i.i.d. U[0,1), seed 1.
 *   C2  f32 random walk: z_i ~ N(0,1) (Box-Muller), S_i = sum_{k<=i} z_k in
 *       double, summed sequentially; a_i = (float)S_i.
 *   C3  f32 envelopes: series s has period P_s = 50 + 450*U; a[s][t] =
 *       (float)(sin(2 pi t / P_s) + 0.1*N(0,1)).
 *   C4  u8 images: i.i.d. U{0..255} plus 64 painted axis-aligned rectangles
 *       (height, width uniform in [1,2048], top-left uniform, value uniform).
 *   C5  f32 adversarial mix: cycle [up-run, noise, down-run, noise], every
 *       segment length ~ Geometric(p = 1/1000) on {1,2,...}; up-runs start at a
 *       uniform integer in [0, 2^23) and step +1, down-runs start in
 *       [2^23, 2^24) and step -1; noise = U01_f32 * 2^24.
 * Float outputs never contain NaN or -0 (a -0 is rewritten to +0).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t sm_mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static inline uint64_t stream_key(uint64_t seed, uint64_t stream) {
  return sm_mix(sm_mix(seed) ^ (stream * 0xD1B54A32D192ED03ULL));
}

/* The counter-based generator: value i of stream (seed, stream). */
uint64_t synth_rng(uint64_t seed, uint64_t stream, uint64_t i) {
  return sm_mix(stream_key(seed, stream) + i);
}

static inline double u01_f64(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }
static inline float u01_f32(uint64_t x) { return (float)((double)(x >> 40) * 0x1.0p-24); }
static inline double normal_at(uint64_t key, uint64_t i) {
  uint64_t x1 = sm_mix(key + 2 * i), x2 = sm_mix(key + 2 * i + 1);
  double u1 = ((double)(x1 >> 11) + 1.0) * 0x1.0p-53; /* (0, 1] */
  double u2 = (double)(x2 >> 11) * 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}
static inline float no_negzero_f(float v) { return v == 0.0f ? 0.0f : v; }
static inline double no_negzero_d(double v) { return v == 0.0 ? 0.0 : v; }

void synth_raw_u64(uint64_t seed, uint64_t stream, int64_t offset, int64_t n,
                   uint64_t *out) {
  uint64_t key = stream_key(seed, stream);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = sm_mix(key + (uint64_t)(offset + i));
}

void synth_uniform_f64(uint64_t seed, uint64_t stream, int64_t offset,
                       int64_t n, double *out) {
  uint64_t key = stream_key(seed, stream);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    out[i] = no_negzero_d(u01_f64(sm_mix(key + (uint64_t)(offset + i))));
}

void synth_uniform_f32(uint64_t seed, uint64_t stream, int64_t offset,
                       int64_t n, float *out) {
  uint64_t key = stream_key(seed, stream);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    out[i] = no_negzero_f(u01_f32(sm_mix(key + (uint64_t)(offset + i))));
}

void synth_uniform_u8(uint64_t seed, uint64_t stream, int64_t offset, int64_t n,
                      uint8_t *out) {
  uint64_t key = stream_key(seed, stream);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    out[i] = (uint8_t)(sm_mix(key + (uint64_t)(offset + i)) >> 56);
}

void synth_normal_f64(uint64_t seed, uint64_t stream, int64_t offset, int64_t n,
                      double *out) {
  uint64_t key = stream_key(seed, stream);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = normal_at(key, (uint64_t)(offset + i));
}

/* C1: f64 i.i.d. U[0,1), seed 1, stream 0. */
void synth_c1(int64_t n, double *out) { synth_uniform_f64(1, 0, 0, n, out); }

/* C2: f32 random walk of length n (seed 2, the given stream), starting from
   S_{-1} = 0; the partial sums are accumulated sequentially in double. */
int synth_c2(uint64_t stream, int64_t n, float *out) {
  const int64_t CH = 1 << 20;
  double *z = (double *)malloc(sizeof(double) * (size_t)CH);
  if (!z) return -1;
  uint64_t key = stream_key(2, stream);
  double s = 0.0;
  for (int64_t c0 = 0; c0 < n; c0 += CH) {
    int64_t m = n - c0 < CH ? n - c0 : CH;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) z[i] = normal_at(key, (uint64_t)(c0 + i));
    for (int64_t i = 0; i < m; ++i) {
      s += z[i];
      out[c0 + i] = no_negzero_f((float)s);
    }
  }
  free(z);
  return 0;
}

/* C3: rows [row0, row0+rows) of the envelope batch; row s has `len` samples
   stored at out + (s-row0)*ld.  Period stream 0, noise stream 1 (counter
   s*len + t). */
void synth_c3(int64_t row0, int64_t rows, int64_t len, int64_t ld, float *out) {
  uint64_t kp = stream_key(3, 0), kn = stream_key(3, 1);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r) {
    int64_t s = row0 + r;
    double period = 50.0 + 450.0 * u01_f64(sm_mix(kp + (uint64_t)s));
    float *row = out + r * ld;
    for (int64_t t = 0; t < len; ++t) {
      double v = sin(6.283185307179586 * (double)t / period) +
                 0.1 * normal_at(kn, (uint64_t)(s * len + t));
      row[t] = no_negzero_f((float)v);
    }
  }
}

/* C4: images [img0, img0+count) of size rows x cols (row pitch ld bytes, image
   pitch rows*ld): i.i.d. bytes (stream = image index) then `nrect` painted
   rectangles (stream 1000 + image index, 5 draws per rectangle). */
void synth_c4(int64_t img0, int64_t count, int64_t rows, int64_t cols,
              int64_t ld, int nrect, uint8_t *out) {
  for (int64_t b = 0; b < count; ++b) {
    uint64_t g = (uint64_t)(img0 + b);
    uint64_t key = stream_key(4, g);
    uint8_t *img = out + b * rows * ld;
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < rows; ++r)
      for (int64_t c = 0; c < cols; ++c)
        img[r * ld + c] = (uint8_t)(sm_mix(key + (uint64_t)(r * cols + c)) >> 56);
    uint64_t kr = stream_key(4, 1000 + g);
    for (int k = 0; k < nrect; ++k) {
      uint64_t x0 = sm_mix(kr + 5 * (uint64_t)k), x1 = sm_mix(kr + 5 * (uint64_t)k + 1),
               x2 = sm_mix(kr + 5 * (uint64_t)k + 2), x3 = sm_mix(kr + 5 * (uint64_t)k + 3),
               x4 = sm_mix(kr + 5 * (uint64_t)k + 4);
      int64_t h = 1 + (int64_t)(x0 % 2048), wd = 1 + (int64_t)(x1 % 2048);
      int64_t top = (int64_t)(x2 % (uint64_t)rows), left = (int64_t)(x3 % (uint64_t)cols);
      uint8_t v = (uint8_t)(x4 >> 56);
      int64_t bot = top + h < rows ? top + h : rows;
      int64_t right = left + wd < cols ? left + wd : cols;
#pragma omp parallel for schedule(static)
      for (int64_t r = top; r < bot; ++r)
        memset(img + r * ld + left, v, (size_t)(right - left));
    }
  }
}

/* C5: adversarial mix of length n (seed 5, streams 2*stream for segments and
   2*stream+1 for noise).  Returns the number of segments, or -1. */
int64_t synth_c5(uint64_t stream, int64_t n, float *out) {
  uint64_t ks = stream_key(5, 2 * stream), kz = stream_key(5, 2 * stream + 1);
  const double lq = log(1.0 - 1.0 / 1000.0);
  /* pass 1: segment boundaries (sequential; ~n/1000 segments) */
  int64_t cap = 1024, nseg = 0;
  int64_t *start = (int64_t *)malloc(sizeof(int64_t) * (size_t)cap);
  if (!start) return -1;
  int64_t pos = 0;
  while (pos < n) {
    if (nseg == cap) {
      cap *= 2;
      int64_t *p = (int64_t *)realloc(start, sizeof(int64_t) * (size_t)cap);
      if (!p) { free(start); return -1; }
      start = p;
    }
    start[nseg] = pos;
    double u = ((double)(sm_mix(ks + 2 * (uint64_t)nseg) >> 11) + 1.0) * 0x1.0p-53;
    int64_t len = 1 + (int64_t)floor(log(u) / lq);
    pos += len;
    nseg++;
  }
  /* pass 2: fill every segment (independent) */
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t s = 0; s < nseg; ++s) {
    int64_t b = start[s], e = s + 1 < nseg ? start[s + 1] : n;
    if (e > n) e = n;
    uint64_t x = sm_mix(ks + 2 * (uint64_t)s + 1);
    switch (s & 3) {
      case 0: { /* strictly increasing run of integers */
        int64_t v0 = (int64_t)(x >> 41); /* [0, 2^23) */
        for (int64_t i = b; i < e; ++i) out[i] = no_negzero_f((float)(v0 + (i - b)));
        break;
      }
      case 2: { /* strictly decreasing run of integers */
        int64_t v0 = (1LL << 23) + (int64_t)(x >> 41); /* [2^23, 2^24) */
        for (int64_t i = b; i < e; ++i) out[i] = no_negzero_f((float)(v0 - (i - b)));
        break;
      }
      default: /* i.i.d. noise block */
        for (int64_t i = b; i < e; ++i)
          out[i] = no_negzero_f(u01_f32(sm_mix(kz + (uint64_t)i)) * 16777216.0f);
    }
  }
  free(start);
  return nseg;
}

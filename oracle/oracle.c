/*
 * oracle.c -- CPU oracle for the running max-min filter (arXiv cs/0610046).
 * TEST INFRASTRUCTURE ONLY -- see oracle.h.  Build: gcc -O2 -shared -fPIC.
 * No -ffast-math: comparisons must follow IEEE semantics exactly.
 */
#include "oracle.h"

#include <stdint.h>
#include <math.h>
#include <stdlib.h>

/* A bounded double-ended queue of indices (the paper's U and L, PAPER.md:371;
   the paper notes the deques are bounded by w).  A ring
   buffer with a fixed capacity; push on a full deque is an error. */
typedef struct {
  int64_t *buf;
  int64_t cap, head, size;
} oracle_deque;

static int deque_init(oracle_deque *d, int64_t cap) {
  d->buf = (int64_t *)malloc(sizeof(int64_t) * (size_t)cap);
  d->cap = cap;
  d->head = 0;
  d->size = 0;
  return d->buf ? 0 : 1;
}
static void deque_free(oracle_deque *d) {
  free(d->buf);
  d->buf = NULL;
}
static int deque_push_back(oracle_deque *d, int64_t v) {
  if (d->size == d->cap) return 1;
  d->buf[(d->head + d->size) % d->cap] = v;
  d->size++;
  return 0;
}
static int64_t deque_front(const oracle_deque *d) { return d->buf[d->head]; }
static int64_t deque_back(const oracle_deque *d) {
  return d->buf[(d->head + d->size - 1) % d->cap];
}
static void deque_pop_back(oracle_deque *d) {
  if (d->size > 0) d->size--;
}
static void deque_pop_front(oracle_deque *d) {
  if (d->size > 0) {
    d->head = (d->head + 1) % d->cap;
    d->size--;
  }
}

/* N2: the state of one stream (see oracle_stream_push_* in oracle_body.inc). */
struct oracle_stream {
  int64_t w, next;     /* window; position of the next sample */
  oracle_deque U, L;   /* the wedge: stream positions */
  void *ring;          /* the last w+1 values, position i at ring[i % (w+1)] */
  uint64_t comparisons;
  int64_t peak;
};

void oracle_stream_free(oracle_stream *s) {
  if (!s) return;
  deque_free(&s->U);
  deque_free(&s->L);
  free(s->ring);
  free(s);
}

int oracle_stream_stats(const oracle_stream *s, oracle_stats *st) {
  if (!s || !st) return ORACLE_ERR_SHAPE;
  st->comparisons = s->comparisons;
  st->peak_wedge = s->peak;
  return ORACLE_OK;
}

#define T uint8_t
#define TLOW 0
#define THIGH UINT8_MAX
#define S u8
#include "oracle_body.inc"
#undef T
#undef S
#undef TLOW
#undef THIGH
#define T int8_t
#define TLOW INT8_MIN
#define THIGH INT8_MAX
#define S i8
#include "oracle_body.inc"
#undef T
#undef S
#undef TLOW
#undef THIGH
#define T uint16_t
#define TLOW 0
#define THIGH UINT16_MAX
#define S u16
#include "oracle_body.inc"
#undef T
#undef S
#undef TLOW
#undef THIGH
#define T int16_t
#define TLOW INT16_MIN
#define THIGH INT16_MAX
#define S i16
#include "oracle_body.inc"
#undef T
#undef S
#undef TLOW
#undef THIGH
#define T uint32_t
#define TLOW 0
#define THIGH UINT32_MAX
#define S u32
#include "oracle_body.inc"
#undef T
#undef S
#undef TLOW
#undef THIGH
#define T int32_t
#define TLOW INT32_MIN
#define THIGH INT32_MAX
#define S i32
#include "oracle_body.inc"
#undef T
#undef S
#undef TLOW
#undef THIGH
#define T uint64_t
#define TLOW 0
#define THIGH UINT64_MAX
#define S u64
#include "oracle_body.inc"
#undef T
#undef S
#undef TLOW
#undef THIGH
#define T int64_t
#define TLOW INT64_MIN
#define THIGH INT64_MAX
#define S i64
#include "oracle_body.inc"
#undef T
#undef S
#undef TLOW
#undef THIGH
#define T float
#define TLOW (-INFINITY)
#define THIGH INFINITY
#define S f32
#include "oracle_body.inc"
#undef T
#undef S
#undef TLOW
#undef THIGH
#define T double
#define TLOW (-INFINITY)
#define THIGH INFINITY
#define S f64
#include "oracle_body.inc"
#undef T
#undef S
#undef TLOW
#undef THIGH

/* ------------------------------------------------------------------ N3 ----
 * LB_Keogh (the max-min filter as the
 * envelope that lower-bounds the time-warping distance, [keogh2005eid]).
 * For each candidate row c (n samples, row pitch ld) and the query q (n
 * samples), with warping radius r:
 *   U_i = max c[max(0,i-r) .. min(n-1,i+r)],  L_i = min over the same range
 *     (the running max-min filter with w = 2r+1, windows clipped at both ends:
 *      DESIGN.md reading R18)
 *   lb = sqrt( sum_i  (q_i > U_i) ? (q_i-U_i)^2 : (q_i < L_i) ? (L_i-q_i)^2 : 0 )
 *   in double precision, summed in index order.
 * oracle_keogh_f32 takes the interior of the envelope from oracle_appendix_f32
 * (full windows) and the clipped ends from running prefix / suffix extrema;
 * oracle_keogh_brute_f32 takes every U_i, L_i from its clipped window.
 * U, L (optional, may be NULL) receive the envelope, [batch][n] dense.       */
static double keogh_term(float qv, float u, float l) {
  if (qv > u) return ((double)qv - (double)u) * ((double)qv - (double)u);
  if (qv < l) return ((double)l - (double)qv) * ((double)l - (double)qv);
  return 0.0;
}

int oracle_keogh_brute_f32(const float *c, int64_t batch, int64_t n, int64_t ld, const float *q,
                           int64_t r, double *lb, float *U, float *L) {
  if (batch < 0 || n < 1 || ld < n) return ORACLE_ERR_SHAPE;
  if (r < 0) return ORACLE_ERR_WINDOW;
  for (int64_t b = 0; b < batch; ++b) {
    const float *x = c + b * ld;
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const int64_t lo = i - r > 0 ? i - r : 0, hi = i + r < n - 1 ? i + r : n - 1;
      float u = x[lo], l = x[lo];
      for (int64_t k = lo + 1; k <= hi; ++k) {
        if (x[k] > u) u = x[k];
        if (x[k] < l) l = x[k];
      }
      if (U) U[b * n + i] = u;
      if (L) L[b * n + i] = l;
      s += keogh_term(q[i], u, l);
    }
    lb[b] = sqrt(s);
  }
  return ORACLE_OK;
}

int oracle_keogh_f32(const float *c, int64_t batch, int64_t n, int64_t ld, const float *q, int64_t r,
                     double *lb, float *U, float *L) {
  if (batch < 0 || n < 1 || ld < n) return ORACLE_ERR_SHAPE;
  if (r < 0) return ORACLE_ERR_WINDOW;
  const int64_t w = 2 * r + 1;
  const size_t nb = sizeof(float) * (size_t)n;
  float *fx = (float *)malloc(nb), *fn = (float *)malloc(nb);   /* full windows     */
  float *px = (float *)malloc(nb), *pn = (float *)malloc(nb);   /* prefix extrema   */
  float *sx = (float *)malloc(nb), *sn = (float *)malloc(nb);   /* suffix extrema   */
  int rc = (fx && fn && px && pn && sx && sn) ? ORACLE_OK : ORACLE_ERR_ALLOC;
  for (int64_t b = 0; b < batch && rc == ORACLE_OK; ++b) {
    const float *x = c + b * ld;
    if (w <= n && (rc = oracle_appendix_f32(x, n, w, fx, fn, NULL)) != ORACLE_OK) break;
    px[0] = pn[0] = x[0];
    for (int64_t e = 1; e < n; ++e) {
      px[e] = x[e] > px[e - 1] ? x[e] : px[e - 1];
      pn[e] = x[e] < pn[e - 1] ? x[e] : pn[e - 1];
    }
    sx[n - 1] = sn[n - 1] = x[n - 1];
    for (int64_t e = n - 2; e >= 0; --e) {
      sx[e] = x[e] > sx[e + 1] ? x[e] : sx[e + 1];
      sn[e] = x[e] < sn[e + 1] ? x[e] : sn[e + 1];
    }
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const int64_t lo = i - r > 0 ? i - r : 0, hi = i + r < n - 1 ? i + r : n - 1;
      float u, l;
      if (lo == i - r && hi == i + r) {  /* interior: the full window j = i - r */
        u = fx[lo];
        l = fn[lo];
      } else if (lo == 0) {              /* clipped at the left (maybe both ends) */
        u = px[hi];
        l = pn[hi];
      } else {                           /* clipped at the right */
        u = sx[lo];
        l = sn[lo];
      }
      if (U) U[b * n + i] = u;
      if (L) L[b * n + i] = l;
      acc += keogh_term(q[i], u, l);
    }
    lb[b] = sqrt(acc);
  }
  free(fx), free(fn), free(px), free(pn), free(sx), free(sn);
  return rc;
}

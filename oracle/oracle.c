/*
 * oracle.c -- CPU oracle for the running max-min filter (arXiv cs/0610046).
 * TEST INFRASTRUCTURE ONLY -- see oracle.h.  Build: gcc -O2 -shared -fPIC.
 * No -ffast-math: comparisons must follow IEEE semantics exactly.
 */
#include "oracle.h"

#include <stdint.h>
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

#define T uint8_t
#define S u8
#include "oracle_body.inc"
#undef T
#undef S
#define T int8_t
#define S i8
#include "oracle_body.inc"
#undef T
#undef S
#define T uint16_t
#define S u16
#include "oracle_body.inc"
#undef T
#undef S
#define T int16_t
#define S i16
#include "oracle_body.inc"
#undef T
#undef S
#define T uint32_t
#define S u32
#include "oracle_body.inc"
#undef T
#undef S
#define T int32_t
#define S i32
#include "oracle_body.inc"
#undef T
#undef S
#define T uint64_t
#define S u64
#include "oracle_body.inc"
#undef T
#undef S
#define T int64_t
#define S i64
#include "oracle_body.inc"
#undef T
#undef S
#define T float
#define S f32
#include "oracle_body.inc"
#undef T
#undef S
#define T double
#define S f64
#include "oracle_body.inc"
#undef T
#undef S

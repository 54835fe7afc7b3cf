/*
 * oracle.h -- CPU oracle for the running max-min filter (arXiv cs/0610046).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load liboracle.so.
 * The product path (paper_cs_0610046_b200/, include/maxmin.h, libmaxmin.so)
 * never includes this header and never links this library; the two share no
 * code, headers, tables or helpers.
 *
 * Every function is plain, sequential C written from the paper:
 *   oracle_brute_1d_*     definition, PAPER.md:39-42 ("max/min_{i in [j,j+w)} a_i
 *                          for all j"); Table 1 "naive" row.
 *   oracle_alg1_*         Algorithm 1, literal reading
 *                          (readings R1-R4).
 *   oracle_appendix_*     the appendix C++ listing.
 *   oracle_w3_*           Proposition "smallprop", PAPER.md:302-309 (w = 3).
 *   oracle_vhgw_*         van Herk-Gil-Werman, PAPER.md:108-116, 136 and the
 *                          commented-out section PAPER.md:176-192 (reading R7).
 *   oracle_brute_2d_*     2-D rectangle definition (valid region R9).
 *   oracle_separable_2d_* "first applying the unidimensional on rows and then on
 *                          columns", with oracle_appendix_* as the
 *                          1-D filter.
 *   oracle_batched_*      oracle_appendix_* on each row of a batch.
 *   oracle_windows_at_*   brute force for a list of window starts (spot checks).
 *   oracle_arg_brute_*    N1 arg filter, the definition: earliest position of
 *                          each window's max and min (reading R17).
 *   oracle_arg_wedge_*    N1 arg filter by the paper's wedge (PAPER.md:364-401,
 *                          locations PAPER.md:522-525) with equal values kept.
 *   oracle_keogh_f32      N3 LB_Keogh: envelope = the max-min filter with
 *                          w = 2r+1 clipped at the ends, bound
 *                          summed in double; _brute: every window clipped.
 *
 * Comparison counting follows PAPER.md:73-75: only value-vs-value comparisons
 * (a<b or b<a) are counted; index tests and deque bookkeeping are free.
 *
 * Parity pins: see tests/test_oracle_*.py and DESIGN.md section "Oracle pins".
 * Parity unpinned: none of the functions above (each has at least one pin that
 * does not re-derive it from itself).
 */
#ifndef MAXMIN_ORACLE_H
#define MAXMIN_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (negative = error) */
#define ORACLE_OK 0
#define ORACLE_ERR_WINDOW (-1)          /* w < 1 (or w != 3 for oracle_w3)      */
#define ORACLE_ERR_WINDOW_TOO_LARGE (-2) /* w > n                                */
#define ORACLE_ERR_NAN (-3)             /* a NaN in a floating-point input      */
#define ORACLE_ERR_INVARIANT (-4)       /* a paper invariant failed (deque cap) */
#define ORACLE_ERR_ALLOC (-5)
#define ORACLE_ERR_SHAPE (-6)

typedef struct {
  uint64_t comparisons; /* value comparisons                  */
  int64_t peak_wedge;   /* max over loop tops of size(U)+size(L) (+1 for the  */
                        /* implicit newest element of the appendix variant)    */
} oracle_stats;

/* N2: one stream's wedge (opaque; oracle_stream_new_<S> / _push_<S> / _free). */
typedef struct oracle_stream oracle_stream;
void oracle_stream_free(oracle_stream *s);
int oracle_stream_stats(const oracle_stream *s, oracle_stats *st);

#define ORACLE_DECLARE(S, T)                                                    \
  int oracle_brute_1d_##S(const T *a, int64_t n, int64_t w, T *out_max,         \
                          T *out_min, oracle_stats *st);                        \
  int oracle_alg1_##S(const T *a, int64_t n, int64_t w, T *out_max,             \
                      T *out_min, oracle_stats *st);                            \
  int oracle_appendix_##S(const T *a, int64_t n, int64_t w, T *out_max,         \
                          T *out_min, oracle_stats *st);                        \
  int oracle_w3_##S(const T *a, int64_t n, T *out_max, T *out_min,              \
                    oracle_stats *st);                                          \
  int oracle_vhgw_##S(const T *a, int64_t n, int64_t w, T *out_max,             \
                      T *out_min, oracle_stats *st);                            \
  int oracle_batched_##S(const T *a, int64_t batch, int64_t n, int64_t in_ld,   \
                         int64_t w, T *out_max, T *out_min, int64_t out_ld);    \
  int oracle_brute_2d_##S(const T *a, int64_t batch, int64_t rows,              \
                          int64_t cols, int64_t w_row, int64_t w_col,           \
                          T *out_max, T *out_min);                              \
  int oracle_separable_2d_##S(const T *a, int64_t batch, int64_t rows,          \
                              int64_t cols, int64_t w_row, int64_t w_col,       \
                              T *out_max, T *out_min);                          \
  int oracle_windows_at_##S(const T *a, int64_t n, int64_t w,                   \
                            const int64_t *starts, int64_t k, T *out_max,       \
                            T *out_min);                                        \
  int oracle_arg_brute_##S(const T *a, int64_t n, int64_t w, T *out_max,        \
                           T *out_min, int64_t *arg_max, int64_t *arg_min);     \
  int oracle_arg_wedge_##S(const T *a, int64_t n, int64_t w, T *out_max,        \
                           T *out_min, int64_t *arg_max, int64_t *arg_min);     \
  int oracle_morph_brute_##S(const T *a, int64_t n, int64_t w, T *open,        \
                             T *close);                                         \
  int oracle_morph_##S(const T *a, int64_t n, int64_t w, T *open, T *close);    \
  int oracle_morph_2d_brute_##S(const T *a, int64_t batch, int64_t rows,        \
                                int64_t cols, int64_t w_row, int64_t w_col,     \
                                T *open, T *close);                             \
  int oracle_morph_2d_##S(const T *a, int64_t batch, int64_t rows,              \
                          int64_t cols, int64_t w_row, int64_t w_col,           \
                          T *open, T *close);                                   \
  int oracle_brute_3d_##S(const T *a, int64_t depth, int64_t rows,             \
                          int64_t cols, int64_t w_x, int64_t w_y, int64_t w_z,  \
                          T *out_max, T *out_min);                              \
  int oracle_separable_3d_##S(const T *a, int64_t depth, int64_t rows,         \
                              int64_t cols, int64_t w_x, int64_t w_y,           \
                              int64_t w_z, T *out_max, T *out_min);             \
  int oracle_stream_new_##S(int64_t w, oracle_stream **out);                    \
  int oracle_stream_push_##S(oracle_stream *s, const T *x, int64_t c,           \
                             T *out_max, T *out_min, int64_t *emitted);

ORACLE_DECLARE(u8, uint8_t)
ORACLE_DECLARE(i8, int8_t)
ORACLE_DECLARE(u16, uint16_t)
ORACLE_DECLARE(i16, int16_t)
ORACLE_DECLARE(u32, uint32_t)
ORACLE_DECLARE(i32, int32_t)
ORACLE_DECLARE(u64, uint64_t)
ORACLE_DECLARE(i64, int64_t)
ORACLE_DECLARE(f32, float)
ORACLE_DECLARE(f64, double)

#undef ORACLE_DECLARE

/* N3 LB_Keogh (float candidates and query, double bound; N3, R18). */
int oracle_keogh_f32(const float *c, int64_t batch, int64_t n, int64_t ld, const float *q,
                     int64_t r, double *lb, float *U, float *L);
int oracle_keogh_brute_f32(const float *c, int64_t batch, int64_t n, int64_t ld, const float *q,
                           int64_t r, double *lb, float *U, float *L);

#ifdef __cplusplus
}
#endif
#endif

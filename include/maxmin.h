/*
 * maxmin.h -- C ABI of libmaxmin.so, the B200 (sm_100a) running max-min filter.
 *
 * The operation (arXiv cs/0610046 section 1):
 *   given a_0..a_{n-1} and a window width w, for every j in [0, n-w]
 *     out_max[j] = max_{i in [j, j+w)} a_i      out_min[j] = min_{i in [j, j+w)} a_i
 *   -- "the maximum and the minimum over all windows of size w".  There are
 *   m = n-w+1 windows.  Both filters are produced in one pass that reads the
 *   input once (the running max and min filters alone, are the
 *   same calls with one output pointer NULL).
 * 2-D: "applying the unidimensional [filter] on rows and then
 *   on columns"; only the valid region is produced (reading R9).
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 * - All data pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors)
 *   owned by the caller, except the *_host entry points whose data pointers
 *   are HOST pointers.  The library never allocates or frees caller memory;
 *   scratch space is passed in through `workspace`.
 * - Lengths, counts, leading dimensions and strides are in ELEMENTS (int64).
 * - Work is enqueued asynchronously on `stream` (a cudaStream_t passed as
 *   void*; NULL = legacy default stream), which must belong to the device
 *   that owns the call's data pointers.  All data pointers of one call must
 *   be on one device (else MAXMIN_ERR_DEVICE); the library makes that device
 *   current for the duration of the call and restores the caller's current
 *   device before returning, on every path.  Argument errors are detected
 *   synchronously: nothing is launched and a non-zero status is returned.  A
 *   launch failure returns MAXMIN_ERR_CUDA and maxmin_last_cuda_error()
 *   reports the cudaError_t.
 * - Alignment: data pointers must be 16-byte aligned and every leading
 *   dimension / stride times sizeof(element) must be a multiple of 16 bytes
 *   (else MAXMIN_ERR_ALIGNMENT).  Loads never touch bytes outside the 16-byte
 *   granules that contain input elements.
 * - Outputs must not overlap the input or each other (MAXMIN_ERR_ALIAS).
 * - Preconditions not checked: floating-point inputs contain no NaN; -0.0 and
 *   +0.0 compare equal and either may be returned.  Every output element is a
 *   copy of an input element, so under these preconditions results are
 *   bit-identical to any correct implementation (the CPU oracle).
 * - Thread safety: stateless; concurrent calls on different streams are safe
 *   provided they use distinct workspaces.
 */
#ifndef MAXMIN_H
#define MAXMIN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MAXMIN_U8 = 0,
  MAXMIN_I8 = 1,
  MAXMIN_U16 = 2,
  MAXMIN_I16 = 3,
  MAXMIN_U32 = 4,
  MAXMIN_I32 = 5,
  MAXMIN_U64 = 6,
  MAXMIN_I64 = 7,
  MAXMIN_F32 = 8,
  MAXMIN_F64 = 9
} maxmin_dtype;

typedef enum {
  MAXMIN_OK = 0,
  MAXMIN_ERR_NULL = 1,              /* a required pointer is NULL, or both outputs NULL */
  MAXMIN_ERR_DTYPE = 2,             /* unknown dtype (2-D: see maxmin_filter_2d)       */
  MAXMIN_ERR_WINDOW = 3,            /* w < 1                                           */
  MAXMIN_ERR_WINDOW_TOO_LARGE = 4,  /* w > n (2-D: w_row > cols or w_col > rows)       */
  MAXMIN_ERR_SHAPE = 5,             /* n < 1, batch < 0, ld too small, size overflow   */
  MAXMIN_ERR_ALIGNMENT = 6,         /* pointer / leading dimension not 16-byte aligned  */
  MAXMIN_ERR_ALIAS = 7,             /* an output overlaps the input or the other output */
  MAXMIN_ERR_WORKSPACE = 8,         /* workspace NULL or smaller than required          */
  MAXMIN_ERR_CUDA = 9,              /* a CUDA runtime call failed                       */
  MAXMIN_ERR_UNSUPPORTED = 10,      /* valid request outside this build's limits        */
  MAXMIN_ERR_MEMORY = 11,           /* a data pointer is not device memory (device APIs) */
  MAXMIN_ERR_DEVICE = 12,           /* the data pointers of one call are on different devices */
  MAXMIN_ERR_NCCL = 13              /* NCCL missing or an NCCL call failed (sharded call)  */
} maxmin_status;

/* Human-readable name of a status code (static storage). */
const char *maxmin_status_str(int status);

/* cudaError_t of the last failing CUDA call made by this library in the
   calling thread (0 if none). */
int maxmin_last_cuda_error(void);

/* Library version, e.g. "maxmin-b200 0.1 sm_100a". */
const char *maxmin_version(void);

/* Size in bytes of one element of dtype `dt`, or 0 if unknown. */
size_t maxmin_dtype_size(int dt);

/*
 * Workspace needed by maxmin_filter_1d / maxmin_filter_batched for these
 * arguments, written to *bytes.  It is 0 unless the cross-CTA look-back path
 * runs (w > 8193; <= 4-byte types: DESIGN.md kernel "k1d_lw", a ticket
 * counter + 256 B per 4096 windows of every row; 8-byte types: kernel
 * "large", ~32 B per 2048 windows).  The library zeroes what it
 * needs of it on `stream` at every call.
 */
int maxmin_workspace_bytes(int dt, int64_t batch, int64_t n, int64_t w,
                           size_t *bytes);

/*
 * 1-D running max-min filter.
 *   in        device, n elements of dtype dt (contiguous).
 *   n, w      1 <= w <= n.
 *   out_max   device, n-w+1 elements, or NULL to skip the max filter.
 *   out_min   device, n-w+1 elements, or NULL to skip the min filter.
 *   workspace device scratch of maxmin_workspace_bytes(dt,1,n,w) bytes (may be
 *             NULL when that is 0).  Must not be used concurrently by another
 *             call.  Contents on entry are ignored.
 */
int maxmin_filter_1d(int dt, const void *in, int64_t n, int64_t w,
                     void *out_max, void *out_min, void *workspace,
                     size_t workspace_bytes, void *stream);

/*
 * Batched series: the 1-D filter on each of `batch` independent rows (no halo
 * between rows).  Row b is in + b*in_ld (n elements, in_ld >= n); its outputs
 * are out_* + b*out_ld (n-w+1 elements, out_ld >= n-w+1).  batch == 0 is a
 * no-op.  Workspace as maxmin_workspace_bytes(dt, batch, n, w).
 */
int maxmin_filter_batched(int dt, const void *in, int64_t batch, int64_t n,
                          int64_t in_ld, int64_t w, void *out_max,
                          void *out_min, int64_t out_ld, void *workspace,
                          size_t workspace_bytes, void *stream);

/*
 * 2-D separable max-min filter over `batch` images.
 *   Image b, row r, column c is in[b*in_bstride + r*in_ld + c].
 *   w_row is the window along a row (over columns, 1 <= w_row <= cols),
 *   w_col the window down a column (over rows, 1 <= w_col <= rows).
 *   Output (b, r, c), r in [0, rows-w_col], c in [0, cols-w_row], is the max
 *   (min) over rows [r, r+w_col) x columns [c, c+w_row), stored at
 *   out_*[b*out_bstride + r*out_ld + c].  Only the valid region is written.
 *   Requires in_ld >= cols, out_ld >= cols-w_row+1, in_bstride >= rows*in_ld,
 *   out_bstride >= (rows-w_col+1)*out_ld (or batch == 1).
 *   Unlike the 1-D calls, pointers and strides need only element alignment.
 *   Supported dtypes: all.  The fused single-pass kernel keeps the
 *   (32+w_col-1) x (256/sizeof(T)+w_row-1) input box on chip; requests whose
 *   box exceeds 200 KB of shared memory return MAXMIN_ERR_UNSUPPORTED.
 */
int maxmin_filter_2d(int dt, const void *in, int64_t batch, int64_t rows,
                     int64_t cols, int64_t in_ld, int64_t in_bstride,
                     int64_t w_row, int64_t w_col, void *out_max,
                     void *out_min, int64_t out_ld, int64_t out_bstride,
                     void *stream);

/*
 * Arg-max / arg-min filter (the paper keeps the locations
 * of the extrema).  For every window j of every row:
 *   out_max[j], out_min[j]  as maxmin_filter_batched,
 *   arg_max[j], arg_min[j]  the absolute position (0-based, in [j, j+w)) of
 *                           the max / min in the row; ties -> the EARLIEST
 *                           position, for both (reading R17).
 *   Any of the four outputs may be NULL (at least one must not be); all four
 *   use the row pitch out_ld (elements).  Value outputs need element
 *   alignment, position outputs (int64) 8-byte alignment; in needs element
 *   alignment.  The vector load/store paths need 16-byte base pointers and,
 *   when batch > 1, 16-byte pitches; other layouts take element-wise paths
 *   (same results, slower).  dtypes of <= 4 bytes (else MAXMIN_ERR_UNSUPPORTED) and
 *   n < 2^32.  Workspace: maxmin_argfilter_workspace_bytes (~32 bytes per
 *   element: the 64-bit (value, position) keys and their filtered copies).
 *   Runs as keys -> max/min filters on the keys -> decode, all on the device.
 */
int maxmin_argfilter_workspace_bytes(int dt, int64_t batch, int64_t n, int64_t w,
                                     size_t *bytes);
int maxmin_argfilter_batched(int dt, const void *in, int64_t batch, int64_t n,
                             int64_t in_ld, int64_t w, void *out_max,
                             void *out_min, int64_t *arg_max, int64_t *arg_min,
                             int64_t out_ld, void *workspace,
                             size_t workspace_bytes, void *stream);

/*
 * LB_Keogh lower bound of the time-warping distance, fused with the envelope
 * ([keogh2005eid]).  For every candidate
 * row b (cand + b*ld, n float samples) against the query (n float samples)
 * with warping radius r >= 0:
 *   U_i, L_i = max, min of the row over [max(0,i-r), min(n-1,i+r)]
 *             (the running max-min filter with w = 2r+1, clipped at the ends)
 *   lb[b] = sqrt( sum_i (q_i > U_i) ? (q_i-U_i)^2 : (q_i < L_i) ? (L_i-q_i)^2 : 0 )
 * computed in double (summation order unspecified).  The envelope is never
 * stored.  dtype MAXMIN_F32 only; cand 16-byte aligned with 16-byte row
 * pitch, query 4-byte aligned, lb (batch doubles, device) 8-byte aligned.
 * 2r+1 <= 8193 or 2r+1 > n (else MAXMIN_ERR_UNSUPPORTED).  No workspace.
 */
int maxmin_lb_keogh_batched(int dt, const void *cand, int64_t batch, int64_t n,
                            int64_t ld, const void *query, int64_t r, double *lb,
                            void *stream);

/*
 * Online multi-stream filter.  The paper's setting: a
 * stream, filtered with zero stream latency ("the maximum number of data
 * points required after the window has passed"; Table 1) and
 * O(w) state.  `streams` independent streams ingest c
 * samples each per push; a push emits, for every stream, the windows that its
 * c new samples complete -- in the same call (reading R19).
 *
 * State: device memory of maxmin_stream_state_bytes(...) bytes, 16-byte
 * aligned, owned by the caller, described by a host-side maxmin_stream that
 * maxmin_stream_init fills in (it also zero-fills the device state on
 * `stream`).  Per stream it holds the last w-1 samples (for w-1 <= 1024: two
 * ping-pong rows, and a push is ONE kernel; otherwise a [history | max_chunk
 * slot] row plus filter scratch, and a push is copy-in, filter, shift).  The struct is the caller's; push
 * updates `seen` and `phase`.
 *
 * maxmin_stream_push(st, chunk, c, chunk_ld, out_max, out_min, out_ld,
 *                    first_valid, stream):
 *   0 <= c <= max_chunk new samples per stream from chunk, a device pointer
 *   to [streams][chunk_ld] samples (element aligned, chunk_ld >= c; 16-byte
 *   aligned rows are read with 16-byte copies).  out_max / out_min (either may
 *   be NULL, not both): [streams][out_ld] device arrays, 16-byte aligned with
 *   16-byte row pitch.  Column k in [0, c) receives the max / min of the w
 *   samples ending at the k-th new sample, i.e. stream positions
 *   [seen+k-w+1, seen+k]; columns k < *first_valid = clamp(w-1-seen, 0, c)
 *   (the stream holds fewer than w samples there) are unspecified.  Then
 *   st->seen += c.  Stream-ordered on `stream`: the chunk may be reused by
 *   work ordered after the push.  c == 0 is a no-op.
 *   Errors: MAXMIN_ERR_SHAPE (c out of range, ld), MAXMIN_ERR_ALIGNMENT,
 *   MAXMIN_ERR_ALIAS (state, chunk and outputs must be disjoint).
 */
typedef struct maxmin_stream {
  int32_t dtype;      /* maxmin_dtype */
  int32_t phase;      /* which history buffer is current (fused path) */
  int64_t streams;    /* independent streams */
  int64_t w;          /* window */
  int64_t max_chunk;  /* largest c of one push */
  int64_t ld;         /* elements between state rows */
  int64_t seen;       /* samples each stream has received */
  void *state;        /* device buffer (caller-owned) */
  size_t state_bytes;
} maxmin_stream;

int maxmin_stream_state_bytes(int dt, int64_t streams, int64_t w, int64_t max_chunk,
                              size_t *bytes);
int maxmin_stream_init(maxmin_stream *st, int dt, int64_t streams, int64_t w,
                       int64_t max_chunk, void *state, size_t state_bytes, void *stream);
int maxmin_stream_push(maxmin_stream *st, const void *chunk, int64_t c, int64_t chunk_ld,
                       void *out_max, void *out_min, int64_t out_ld, int64_t *first_valid,
                       void *stream);

/*
 * maxmin_filter_2d with scratch: the same operation and rules, routed to the
 * fastest applicable path -- the fused packed-byte kernel (1-byte pixels,
 * square windows <= 17, 16-B aligned rows), else the separable streaming
 * passes (rows by the 1-D kernels into two scratch images, then a streaming
 * column pass: w_col <= 16, w_row <= 8193, 16-B aligned input rows, and
 * `workspace` of maxmin_filter_2d_workspace_bytes -- 0 for 1-byte pixels with
 * square windows <= 17), else the fused generic kernel.  workspace may be
 * NULL (then no separable path).
 */
int maxmin_filter_2d_workspace_bytes(int dt, int64_t batch, int64_t rows, int64_t cols,
                                     int64_t w_row, int64_t w_col, size_t *bytes);
int maxmin_filter_2d_ws(int dt, const void *in, int64_t batch, int64_t rows, int64_t cols,
                        int64_t in_ld, int64_t in_bstride, int64_t w_row, int64_t w_col,
                        void *out_max, void *out_min, int64_t out_ld, int64_t out_bstride,
                        void *workspace, size_t workspace_bytes, void *stream);

/*
 * Grayscale opening and closing (the image-processing use
 * of the filter: erosion = the min filter, dilation = the max
 * filter).  The flat structuring element (w samples; a w_col x w_row
 * rectangle in 2-D) stays inside the data (reading R20):
 *   open[i]  = max, over the windows inside the row that contain i, of their min
 *   close[i] = min, over the same windows, of their max
 * for EVERY position i: outputs have the input's shape.
 *
 * maxmin_morph_batched: rows b of in + b*in_ld (n samples each); out_open /
 *   out_close (either may be NULL) rows at pitch out_ld, 16-byte aligned with
 *   a 16-byte row pitch when batch > 1 (one row: any pitch, it never enters an
 *   address); in needs element alignment.  w - 1 <= 8192 (else
 *   MAXMIN_ERR_UNSUPPORTED; 8-byte types stop where a warp's staging no longer
 *   fits shared memory, about w - 1 <= 4000).  One fused kernel: the input is read once and
 *   each output written once.  No workspace.
 * maxmin_morph_2d: images as maxmin_filter_2d; outputs [batch][rows][cols]
 *   with pitch out_ld / out_bstride, element alignment.  Device workspace of
 *   maxmin_morph_2d_workspace_bytes (two padded copies of the image: the
 *   erosion and the dilation framed by the identities, and two aligned
 *   valid-region buffers).  Runs as the 2-D filter, then its max over the
 *   padded erosion and min over the padded dilation (the rectangle opening is
 *   not separable into 1-D openings).  1-byte pixels with square windows the
 *   packed kernel takes (2..5, 7, 9, ..., 17; 16-B aligned input rows, 4-B
 *   aligned output rows) run as three packed passes instead: erosion and
 *   complemented dilation into the aligned buffers, then max filters of both
 *   read through the tensor map's zero frame (no frame copies).
 */
int maxmin_morph_batched(int dt, const void *in, int64_t batch, int64_t n, int64_t in_ld,
                         int64_t w, void *out_open, void *out_close, int64_t out_ld,
                         void *stream);
int maxmin_morph_2d_workspace_bytes(int dt, int64_t batch, int64_t rows, int64_t cols,
                                    int64_t w_row, int64_t w_col, size_t *bytes);
int maxmin_morph_2d(int dt, const void *in, int64_t batch, int64_t rows, int64_t cols,
                    int64_t in_ld, int64_t in_bstride, int64_t w_row, int64_t w_col,
                    void *out_open, void *out_close, int64_t out_ld, int64_t out_bstride,
                    void *workspace, size_t workspace_bytes, void *stream);

/*
 * The max-min filter over 3-D boxes ("N-D separable
 * filters"; the paper's rows-then-columns application, with
 * a depth axis): for a volume of `depth` slices of rows x cols (row pitch
 * in_ld, slice pitch in_slice, elements),
 *   out(k,i,j) = max / min over [k, k+w_z) x [i, i+w_y) x [j, j+w_x)
 * for the valid region D' x R' x C' = (depth-w_z+1) x (rows-w_y+1) x
 * (cols-w_x+1); outputs with row pitch out_ld and slice pitch out_slice
 * (either output may be NULL).  Element alignment suffices.  Device
 * workspace of maxmin_filter_3d_workspace_bytes (two scratch volumes of D'
 * slices, plus the row images of the separable 2-D pass).  Runs as a
 * streaming column pass along depth (w_z <= 16; else the 2-D kernel with
 * slices as rows), then the 2-D filter (w_x, w_y) of every scratch slice.
 * MAXMIN_ERR_UNSUPPORTED when the depth window exceeds the 2-D kernel's
 * shared memory (about w_z > 140 for 4-byte types).
 */
int maxmin_filter_3d_workspace_bytes(int dt, int64_t depth, int64_t rows, int64_t cols,
                                     int64_t in_ld, int64_t w_x, int64_t w_y, int64_t w_z,
                                     size_t *bytes);
int maxmin_filter_3d(int dt, const void *in, int64_t depth, int64_t rows, int64_t cols,
                     int64_t in_ld, int64_t in_slice, int64_t w_x, int64_t w_y, int64_t w_z,
                     void *out_max, void *out_min, int64_t out_ld, int64_t out_slice,
                     void *workspace, size_t workspace_bytes, void *stream);

/*
 * End-to-end 1-D call on HOST buffers (in, out_max, out_min are host
 * pointers; page-locked memory gives full PCIe bandwidth).  The input is
 * streamed to the device in chunks (with a (w-1)-element overlap), filtered
 * and streamed back, with copies and kernels of consecutive chunks
 * overlapped on two streams.  `dev_workspace` is device scratch of
 * maxmin_host_workspace_bytes(dt, n, w, chunk) bytes.  `chunk` is the number
 * of windows per chunk (0 = default 2^24).  Returns after the results are in
 * the host buffers (synchronous).
 */
int maxmin_host_workspace_bytes(int dt, int64_t n, int64_t w, int64_t chunk,
                                size_t *bytes);
int maxmin_filter_1d_host(int dt, const void *in, int64_t n, int64_t w,
                          void *out_max, void *out_min, int64_t chunk,
                          void *dev_workspace, size_t workspace_bytes);

/*
 * One 1-D array split over `nranks` processes, one GPU each (
 * the filter of PAPER.md:39-42 on the concatenation of the chunks).  Rank r
 * owns the contiguous chunk [c_r, c_{r+1}) of the global array and emits every
 * window that STARTS in it: n_local windows, or n_local-w+1 on the last rank
 * (rank nranks-1).  The windows of the last w-1 starts need the first w-1
 * elements of rank r+1's chunk -- the halo:
 *   local      device buffer of n_local + halo elements (16-byte aligned):
 *              [own chunk | halo slot].  The slot is overwritten.
 *   halo       >= w-1 for every window; must not exceed the next rank's
 *              n_local (not checkable here: the caller's partition).
 *   windows    host array of nwin windows; out_max[k] / out_min[k] (host
 *              arrays of device pointers; per window either may be NULL, not
 *              both) receive the windows of windows[k]: n_local elements, or
 *              n_local - windows[k] + 1 on the last rank, 16-byte aligned.
 *   nccl_comm  an ncclComm_t whose size is nranks and whose rank is `rank`
 *              (e.g. PyTorch ProcessGroupNCCL._comm_ptr()).  Exchange: one
 *              ncclSend of the own first `halo` elements to rank-1 and one
 *              ncclRecv of rank+1's into the slot, grouped, on comm_stream
 *              (NULL = stream).  The windows inside the own chunk run on
 *              `stream` while the message is in flight; the tail windows
 *              (from the last 64-aligned start before n_local-w+1) wait for
 *              the receive.  Every rank must make the call (NCCL point-to-
 *              point semantics).  NCCL is loaded at run time (the libnccl.so.2
 *              already in the process, else the system's); failure of either
 *              -> MAXMIN_ERR_NCCL, maxmin_last_nccl_error() has ncclResult_t.
 *              nccl_comm == NULL: the slot is taken as already filled by the
 *              caller (its own transport, e.g. peer copies) and no exchange
 *              happens.
 *   workspace  device scratch of maxmin_sharded_workspace_bytes(...).
 * Returns when everything is enqueued; `stream` is ordered after the whole
 * call (including the receive).  The communicator's rank/size must match
 * (else MAXMIN_ERR_SHAPE).
 */
int maxmin_sharded_workspace_bytes(int dt, int64_t n_local, int64_t halo,
                                   const int64_t *windows, int nwin, size_t *bytes);
int maxmin_filter_1d_sharded(int dt, void *local, int64_t n_local, int64_t halo,
                             const int64_t *windows, int nwin, int rank, int nranks,
                             void *nccl_comm, void *const *out_max, void *const *out_min,
                             void *workspace, size_t workspace_bytes, void *stream,
                             void *comm_stream);
/* ncclResult_t of the last failing NCCL call of this library in the calling
   thread (0 if none). */
int maxmin_last_nccl_error(void);

#ifdef __cplusplus
}
#endif
#endif /* MAXMIN_H */

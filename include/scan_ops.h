/*
 * scan_ops.h -- C ABI of the scan-based operators in libscan.so (sm_100a):
 * split / compress (Sec. 5.1-5.2) and the LSB radix sort built from
 * one split per key bit (Sec. 5.3).  Same conventions as scan.h: device
 * pointers on the current device, caller-owned buffers, enqueue-only on
 * `stream`, status codes of scan_status, no aborts, workspace initialised
 * ONCE with scan_workspace_init() and reusable in stream order.
 *
 *   - scan_split: P281 "places all items of x where the corresponding flag is
 *     true at the beginning of the output array, followed by all items where
 *     the corresponding flag is false ... the relative order of the elements
 *     is preserved", and P283 SplitInd "also returns the output indices
 *     corresponding to the original input locations": idx_out[j] = input
 *     position of z[j].  The offsets are those of the exclusive scan of the
 *     mask (P283, P461): true item i -> e_i, false item i -> T + (i - e_i).
 *   - compress != 0: P285 "only the first part of the output elements of the
 *     split are returned" (= torch.masked_select): z and idx_out receive T
 *     items.
 *   - scan_radix_sort: P287 LSB radix sort, one split per key bit with mask =
 *     NOT(bit) of the order-preserving key code ("inverting the MSB of
 *     positive numbers and all the bits of the negative numbers" for floats;
 *     sign bit flipped for signed integers), keys moved unchanged, indices
 *     tracked through every split (P365).  Stable.  descending != 0 uses
 *     mask = bit (1-bits first): the exact reverse order, still stable.
 *
 *   - scan_weighted_sample: App. B.3 (P463) "we scan w, and then, given a
 *     uniform sample theta in [0,1] ... The output is an index i of w with
 *     probability proportional to w_i" (inverse transform sampling): the
 *     inclusive fp32 scan S of w is written to `cdf`, then
 *     *index_out = min{ i : S_i > theta * S_{n-1} } (R14).
 *   - scan_top_p_draw: the nucleus + draw step of top-p sampling (Sec. 5.5,
 *     P299: "applies sort and scan on the token probability vector") on the
 *     row scans C of the DESCENDING-sorted probabilities (scan_rows) and the
 *     sort's permutation `order`: K = 1 + min{ j : C_j >= p } (all columns if
 *     none), t = u_r * C_{K-1}, token = order[min{ k : C_k > t }] (R15).
 *
 * Readings: a flag is true iff its int8 value is nonzero (R12);
 * the float code orders keys by the IEEE total order, -NaN < -inf < ... < -0
 * < +0 < ... < +inf < +NaN (R13).  Indices are int32: n must be < 2^31.
 */
#ifndef PAPER_2505_15112_B200_SCAN_OPS_H
#define PAPER_2505_15112_B200_SCAN_OPS_H

#include "scan.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Key types of scan_radix_sort (raw bits in, raw bits out). */
typedef enum {
    SCAN_KEY_U16 = 0,
    SCAN_KEY_I16 = 1,
    SCAN_KEY_F16 = 2,   /* IEEE binary16 (P287's fp16 sort) */
    SCAN_KEY_U32 = 3,
    SCAN_KEY_I32 = 4,
    SCAN_KEY_F32 = 5
} scan_key_type;

/* Workspace bytes scan_split of n elements needs (0 if n < 0). */
SCAN_API size_t scan_split_workspace_bytes(int64_t n);

/* Split (compress == 0) or compress (compress != 0) of n elements of
 * elem_bytes (1, 2, 4 or 8) bytes each.
 *   x       [n] input elements (device)
 *   flags   [n] int8 mask, nonzero = true (device)
 *   z       [n] (split) or [>= T] (compress) output elements (device)
 *   idx_out NULL or [n] / [>= T] int32: input position of every output
 *   count_out NULL or ONE device int64: T, the number of true flags
 * x and z must not overlap.  16-byte-aligned buffers take the vector path;
 * any alignment is accepted.  Errors: SCAN_ERR_ARG for n < 0, n >= 2^31,
 * a NULL required pointer, elem_bytes not in {1,2,4,8} or overlapping x/z;
 * SCAN_ERR_WORKSPACE for a NULL / misaligned / too small workspace. */
SCAN_API int scan_split(const void* x, const int8_t* flags, void* z, int32_t* idx_out, int64_t n,
                        int elem_bytes, int compress, int64_t* count_out, void* ws, size_t ws_bytes,
                        void* stream);

/* Workspace bytes scan_radix_sort of n keys of key_type needs (it holds one
 * ping-pong copy of the keys and indices plus the split counts). */
SCAN_API size_t scan_radix_sort_workspace_bytes(int64_t n, int key_type);

/* Stable LSB radix sort of n keys (16 splits for 16-bit keys, 32 for 32-bit).
 *   keys     [n] input keys (device, not modified)
 *   keys_out [n] sorted keys (device; must not overlap keys)
 *   idx_out  [n] int32 input position of every sorted key (device)
 * Errors as scan_split; SCAN_ERR_ARG also for an unknown key_type. */
SCAN_API int scan_radix_sort(const void* keys, void* keys_out, int32_t* idx_out, int64_t n, int key_type,
                             int descending, void* ws, size_t ws_bytes, void* stream);

/* Row-batched LSB radix sort: each of the `rows` rows of `cols` contiguous keys
 * (keys + r*cols) is sorted on its own -- the sort of P299's top-p pipeline
 * ("applies sort and scan on the token probability vector"), by the same 8-bit
 * digit passes as scan_radix_sort.  Per pass the per-(row, digit, tile) counts
 * are laid out [row][digit][tile] and ONE exclusive row scan per row
 * (scan_rows, P437) gives every (digit, tile) its start inside the row.
 * keys_out [rows*cols] the sorted rows; idx_out [rows*cols] int32 COLUMN index
 * (within the row) of every sorted key.  Stable; descending != 0: descending,
 * equal keys still in ascending column order (= torch.sort(descending=True,
 * stable=True)).  Key order as scan_radix_sort (R13).  ws:
 * scan_radix_sort_rows_workspace_bytes(rows, cols, key_type) bytes, 256-byte
 * aligned; cols < 2^31.  Errors as scan_radix_sort. */
SCAN_API size_t scan_radix_sort_rows_workspace_bytes(int64_t rows, int64_t cols, int key_type);
SCAN_API int scan_radix_sort_rows(const void* keys, void* keys_out, int32_t* idx_out, int64_t rows, int64_t cols,
                                  int key_type, int descending, void* ws, size_t ws_bytes, void* stream);

/* Weighted sampling (P463).  w [n] fp32 non-negative weights with a positive
 * sum; cdf [n] fp32 device scratch that receives the inclusive scan; ws a scan
 * workspace of scan_workspace_bytes(SCAN_F32_F32, n) bytes; index_out ONE
 * device int64.  theta in [0, 1) is the uniform draw (an input, R16). */
SCAN_API int scan_weighted_sample(const float* w, int64_t n, double theta, int64_t* index_out, float* cdf,
                                  void* ws, size_t ws_bytes, void* stream);

/* Top-p draw on `rows` rows.  cdf: row r at cdf + r*cdf_row_stride, the
 * inclusive scan of row r's probabilities sorted in descending order; order:
 * row r at order + r*order_row_stride, int32 original column of every sorted
 * entry (scan_radix_sort_rows' idx_out); u [rows] fp32 uniform draws in [0, 1);
 * p the nucleus mass.  Outputs: token_out [rows] int64 sampled column, kept_out
 * NULL or [rows] int32 nucleus size K.  Strides are in elements, >= cols. */
SCAN_API int scan_top_p_draw(const float* cdf, const int32_t* order, int64_t rows, int64_t cols,
                             int64_t cdf_row_stride, int64_t order_row_stride, float p, const float* u,
                             int64_t* token_out, int32_t* kept_out, void* stream);

/* Top-p sampling of `rows` rows WITHOUT a full sort (Sec. 5.5, R15): per row,
 * one read gathers the candidates near the row maximum, their exact masses per
 * eighth-octave level locate the level where the nucleus ends, and only that
 * level (and the draw's level) is ordered by (probability descending, column
 * ascending) -- the stable descending order of the full sort; nucleus and draw
 * as in scan_top_p_draw, with exact fp64 prefix sums (fallback: candidates
 * {q >= tau}, tau lowered until their mass reaches p, all sorted).  p is used
 * as given (fp32, widened exactly).  probs: row r at probs + r*row_stride, fp32,
 * non-negative; u [rows] uniform draws.  token_out [rows] int64 (-1: the row
 * needs more than 8192 candidates to reach p -- use the sort path,
 * scan_top_p_draw), kept_out NULL or [rows] int32 nucleus sizes.  Rows are
 * claimed by ticket from a counter in the header of `ws` (a workspace
 * initialised with scan_workspace_init, at least scan_workspace_bytes(dtype, 0)
 * bytes; calls that may run concurrently need distinct workspaces).  Errors:
 * SCAN_ERR_ARG for cols == 0 or >= 2^31 or null pointers (rows > 0),
 * SCAN_ERR_WORKSPACE for a NULL / misaligned / too small ws, SCAN_ERR_CUDA for
 * launch failures. */
SCAN_API int scan_top_p_sample(const float* probs, int64_t rows, int64_t cols, int64_t row_stride, float p,
                               const float* u, int64_t* token_out, int32_t* kept_out, void* ws,
                               size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif

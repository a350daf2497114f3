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

#ifdef __cplusplus
}
#endif

#endif

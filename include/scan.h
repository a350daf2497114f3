/*
 * scan.h -- C ABI of the B200 (sm_100a) device-wide prefix-sum library
 * (libscan.so, built from paper_2505_15112_b200/csrc/).
 *
 * What the calls compute (PAPER.md = arxiv 2505.15112 "Parallel Scan on
 * Ascend AI Accelerators"; "P<line>" cites its line):
 *   - scan_inclusive: P68 (Sec. 2) "The inclusive prefix sum of a sequence
 *     x_1, x_2, x_3, ... is the sequence x_1, x_1+x_2, x_1+x_2+x_3, ...".
 *   - scan_exclusive: P461 (App. B.2) the inclusive output "shifted by one
 *     element, discarding the last value and writing zero to the first
 *     position".
 *   - scan_rows: P437 (App. B.1) "The batched scan computes the prefix sum of
 *     a batch of input arrays of equal length".
 *   - scan_total / scan_carry_from_totals: the reduce step of Reduce-Scan-Scan
 *     (P73, Sec. 2.1) applied at device level, so each GPU of a sharded
 *     array can start its scan from the sum of all lower shards (DESIGN.md
 *     "Multi-GPU").
 *   - Type pairs: int32->int32, fp32->fp32, fp16->fp32 ("float16 (with
 *     float32 output)", P98) and int8->int32 ("input matrices of 8-bit
 *     integers with output/accumulation in 32-bit integers", P459).
 *
 * Arithmetic:
 *   - Integer outputs wrap mod 2^32 (two's complement).  int8 input is summed
 *     as signed values; 0/1 flags are the special case the paper uses.
 *   - Float outputs: elements are summed in fp32 inside a tile and the
 *     cross-tile carry is kept in fp64; each output is rounded to fp32 once
 *     (round to nearest even).  Accuracy contract (BASELINE.json north_star):
 *     |out_i - exact_i| <= 1e-6 * sum_{j<=i}|x_j| + 1e-6.
 *
 * Conventions for every call:
 *   - Pointers named in/out/carry/total/ws are DEVICE pointers on the current
 *     CUDA device.  The caller owns and frees every buffer; the library never
 *     allocates device memory and keeps no pointer after it returns.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  All calls
 *     only enqueue work on it and never synchronize the host.
 *   - n == 0 (or rows == 0 / cols == 0) is a no-op returning SCAN_OK.
 *   - Aliasing: in == out is allowed when input and output elements have the
 *     same size (int32, fp32); any other overlap returns SCAN_ERR_ARG.
 *   - Any element alignment is accepted; 16-byte-aligned arrays (and row
 *     strides that are multiples of 16 bytes) take the TMA fast path.
 *   - Errors: SCAN_ERR_ARG for a bad argument (n < 0, NULL pointer with
 *     n > 0, unknown dtype, bad rank/G), SCAN_ERR_WORKSPACE for a workspace
 *     that is NULL, too small or not 256-byte aligned (an uninitialised
 *     workspace cannot be detected: see scan_workspace_init),
 *     SCAN_ERR_DEVICE if the current device is not sm_100, SCAN_ERR_CUDA if
 *     a CUDA call or launch failed.  Nothing is enqueued when an error is
 *     returned before the launch.  No call aborts or throws.
 *   - Workspace: one caller-owned device buffer of scan_workspace_bytes()
 *     bytes, initialised ONCE with scan_workspace_init() before first use,
 *     then reusable by any number of calls issued in stream order.  Two
 *     calls that may run concurrently must not share a workspace.
 *   - Operators (scan_ops.h: split / compress, radix sort) keep scratch in
 *     the workspace where look-back descriptors live.  The library records
 *     (host side) which workspaces an operator dirtied, and the next
 *     scan_inclusive / scan_exclusive / scan_rows given that workspace zeroes
 *     that range first (one cudaMemsetAsync on its stream).  A CUDA graph that
 *     captured a scan does not see this record: do not share a graph's
 *     workspace with operator calls outside the graph.
 *   - Thread safety: calls are reentrant.  The library's state: per-device
 *     caches of device attributes and kernel attributes (set once per
 *     device), the dirty-workspace record above, and, for scan_host only,
 *     two copy streams per device created on first use and kept for the
 *     life of the process.
 */
#ifndef PAPER_2505_15112_B200_SCAN_H
#define PAPER_2505_15112_B200_SCAN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SCAN_ABI_VERSION 2

#if defined(__GNUC__)
#define SCAN_API __attribute__((visibility("default")))
#else
#define SCAN_API
#endif

/* Input -> output element types. */
typedef enum {
    SCAN_I32_I32 = 0,   /* int32 in, int32 out                 */
    SCAN_F32_F32 = 1,   /* fp32 in, fp32 out                   */
    SCAN_F16_F32 = 2,   /* IEEE binary16 in, fp32 out (P98)    */
    SCAN_I8_I32 = 3     /* int8 in (signed), int32 out (P459)  */
} scan_dtype;

typedef enum {
    SCAN_OK = 0,
    SCAN_ERR_ARG = 1,
    SCAN_ERR_WORKSPACE = 2,
    SCAN_ERR_CUDA = 3,
    SCAN_ERR_DEVICE = 4
} scan_status;

/* SCAN_ABI_VERSION of the loaded library. */
SCAN_API int scan_abi_version(void);

/* Static string for a status code (never NULL). */
SCAN_API const char* scan_status_string(int status);

/* Bytes of workspace a 1-D scan of n elements of `dtype` needs (also enough
 * for scan_total of n elements).  Returns 0 for an invalid dtype or n < 0. */
SCAN_API size_t scan_workspace_bytes(int dtype, int64_t n);

/* Bytes of workspace scan_rows(rows, cols) needs. */
SCAN_API size_t scan_rows_workspace_bytes(int dtype, int64_t rows, int64_t cols);

/* Initialise a workspace of ws_bytes bytes (enqueued on `stream`).  Must be
 * called once after allocation and before the first scan that uses it. */
SCAN_API int scan_workspace_init(void* ws, size_t ws_bytes, void* stream);

/* Inclusive scan (P68): out[i] = c + in[0] + ... + in[i], n elements.
 * carry_in: NULL (c = 0) or a device pointer to ONE value added in front of
 * the sequence: int64_t for integer dtypes (used mod 2^32), double for
 * float dtypes.  It is how a shard of a larger array continues the scan of
 * the shards before it. */
SCAN_API int scan_inclusive(const void* in, void* out, int64_t n, int dtype, const void* carry_in,
                   void* ws, size_t ws_bytes, void* stream);

/* Exclusive scan (P461): out[0] = c, out[i] = c + in[0] + ... + in[i-1].
 * Same arguments as scan_inclusive. */
SCAN_API int scan_exclusive(const void* in, void* out, int64_t n, int dtype, const void* carry_in,
                   void* ws, size_t ws_bytes, void* stream);

/* Row-batched scan (P437): for r in [0, rows), the `cols` elements at
 * in + r*in_row_stride are scanned independently (inclusive, or exclusive if
 * `exclusive` != 0) into out + r*out_row_stride.  Strides are in ELEMENTS of
 * the input / output type and must be >= cols. */
SCAN_API int scan_rows(const void* in, void* out, int64_t rows, int64_t cols, int64_t in_row_stride,
              int64_t out_row_stride, int dtype, int exclusive, void* ws, size_t ws_bytes,
              void* stream);

/* Reduction of n input elements (the "R" of Reduce-Scan-Scan, P73):
 * *total_out = in[0] + ... + in[n-1] as int64_t (integer dtypes, exact) or
 * double (float dtypes, fp64 accumulation in a fixed order, so repeated calls
 * give identical bits).  total_out is a device pointer. */
SCAN_API int scan_total(const void* in, int64_t n, int dtype, void* total_out, void* ws,
               size_t ws_bytes, void* stream);

/* Carry of shard `rank` of G contiguous shards: *carry_out = totals[0] + ...
 * + totals[rank-1], summed in that order (0 for rank 0).  totals holds G
 * device values of the scan_total type (int64_t or double); carry_out gets
 * one value of the same type, ready for scan_inclusive's carry_in. */
SCAN_API int scan_carry_from_totals(const void* totals, int G, int rank, int dtype, void* carry_out,
                           void* stream);

/* Two-pass sharded scan: the per-GPU work of the multi-GPU Reduce-Scan-Scan
 * (P73, Sec. 2.1: "a block-level reduction first, followed by a scan of the
 * block-level reductions and a final scan of each block"), with blocks of
 * 131,072 elements.
 *   scan_shard_reduce: one read of the shard; *total_out = sum of the n
 *     elements (int64 / double, as scan_total, fixed order) and the block sums
 *     and their exclusive prefix are kept in `ws`.
 *   scan_shard_scan: the scan of the SAME shard (same n, dtype and ws, after
 *     scan_shard_reduce in stream order) seeded with carry_in (device pointer,
 *     NULL = 0; the sum of the lower shards, e.g. from scan_carry_from_totals):
 *     every block starts from carry_in + its prefix, so the pass is a pure
 *     stream (the batched row kernel), inclusive or exclusive.  Results equal
 *     scan_inclusive / scan_exclusive with the same carry_in (bit-exact for
 *     integers, within the float tolerance).  Unaligned or in-place buffers
 *     fall back to the single-pass scan.
 * ws: scan_shard_workspace_bytes(dtype, n) bytes, initialised once with
 * scan_workspace_init; one workspace per shard in flight. */
SCAN_API size_t scan_shard_workspace_bytes(int dtype, int64_t n);
SCAN_API int scan_shard_reduce(const void* in, int64_t n, int dtype, void* total_out, void* ws, size_t ws_bytes,
                               void* stream);
SCAN_API int scan_shard_scan(const void* in, void* out, int64_t n, int dtype, int exclusive, const void* carry_in,
                             void* ws, size_t ws_bytes, void* stream);

/* Device-initiated exchange of the shard totals: the NCCL all-gather and the
 * carry kernel of the Reduce-Scan-Scan step folded into the two passes.
 *   Slots: every rank owns a slot array of scan_peer_slots_bytes(G) bytes in
 *   device memory that every other rank can write through a peer mapping
 *   (CUDA IPC / P2P / symmetric memory over NVLink), zeroed once before the
 *   first call.  Rank q's total for call `epoch` is written into EVERY rank's
 *   array as two tagged 8-byte words (epoch << 32 | high / low 32 bits of the
 *   int64 or fp64 total), relaxed system-scope stores (each word carries its
 *   own tag, so no ordering against other memory is needed).
 *   scan_shard_reduce_publish: scan_shard_reduce, then the total goes to every
 *     rank's slots; peer_slots is a DEVICE array of G device pointers,
 *     peer_slots[q] = rank q's slot array as addressed from this GPU.
 *   scan_shard_scan_peers: scan_shard_scan whose carry_in is the sum of ranks
 *     0..rank-1's totals (in rank order, as scan_carry_from_totals), read from
 *     this rank's own slot array `slots` (relaxed loads until both tags match): the row kernel's
 *     compute warps wait for the lower ranks while its producer already loads.
 *   epoch: > 0, the same on every rank for one call, a new value per call
 *     (e.g. a call counter).  Slots are a ring of 64 calls: a rank must not
 *     run 64 or more calls ahead of the slowest rank (any collective or
 *     barrier at least every 63 calls guarantees it).  G <= 32.
 * Errors: SCAN_ERR_ARG for G outside 1..32, rank outside 0..G-1, epoch == 0 or
 * NULL slot pointers; otherwise as scan_shard_reduce / scan_shard_scan.  A rank
 * whose lower peers never publish waits forever: call both on every rank. */
SCAN_API size_t scan_peer_slots_bytes(int G);
SCAN_API int scan_shard_reduce_publish(const void* in, int64_t n, int dtype, void* total_out, void* const* peer_slots,
                                       int G, int rank, uint32_t epoch, void* ws, size_t ws_bytes, void* stream);
SCAN_API int scan_shard_scan_peers(const void* in, void* out, int64_t n, int dtype, int exclusive, const void* slots,
                                   int G, int rank, uint32_t epoch, void* ws, size_t ws_bytes, void* stream);

/* Measurement ceiling (not a scan): out[i] = widen(in[i]) for n elements --
 * exactly the HBM traffic of a scan of the same dtype with no scan arithmetic
 * (a 16-byte streaming copy).  bench.py times it in the same run as the scan
 * (SURVEY 8(d) "matched-traffic widen-copy").  16-byte aligned buffers only
 * (SCAN_ERR_ARG otherwise). */
SCAN_API int scan_widen_copy(const void* in, void* out, int64_t n, int dtype, void* stream);

/* End-to-end scan of an array in HOST memory (pinned for full speed): the
 * array is streamed through the GPU in chunks of `chunk_elems` elements with
 * the host->device copy of chunk i+1, the scan of chunk i and the
 * device->host copy of chunk i-1 overlapped on three streams; the carry of
 * chunk i+1 is the fp64 / int64 running total, kept on the device.  h_in and
 * h_out are host pointers (h_in != h_out); `stage` is a device buffer of
 * scan_host_stage_bytes(dtype, chunk_elems) bytes and `ws` a workspace of
 * scan_workspace_bytes(dtype, chunk_elems) bytes.  Asynchronous with respect
 * to the host: the result is complete when `stream` reaches the point the
 * call enqueued (e.g. after cudaStreamSynchronize(stream)).  Semantics are
 * those of scan_inclusive / scan_exclusive over the whole array, carry 0. */
SCAN_API size_t scan_host_stage_bytes(int dtype, int64_t chunk_elems);
SCAN_API int scan_host(const void* h_in, void* h_out, int64_t n, int dtype, int exclusive,
                       int64_t chunk_elems, void* stage, size_t stage_bytes, void* ws,
                       size_t ws_bytes, void* stream);

/* Kernel launches the library enqueued since load (a process-wide counter;
 * used by the bench to report how many of its own kernels ran). */
SCAN_API uint64_t scan_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* PAPER_2505_15112_B200_SCAN_H */

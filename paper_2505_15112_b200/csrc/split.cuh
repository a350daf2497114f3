// split.cuh -- SplitInd / compress (PAPER Sec. 5.1-5.2, P281-285) and the
// per-bit split of the LSB radix sort (Sec. 5.3, P287) for sm_100a.
//
// The paper's SplitInd runs an exclusive MCScan over the 0/1 mask and gathers
// every element (and its index) to the offset the scan gives it (P283).  On
// B200 the scan of a 1-byte mask is cheap next to the payload, so the split is
// a block-level Reduce-then-Scan (the RSS of P73) with the scatter fused into
// the scan's epilogue:
//
//   k_split_count   one read of the mask (or of the key bit): a WARP per
//                   TILE-element tile with all of its loads in flight at once,
//                   true count per tile; the last CTA to finish scans the
//                   counts into tile offsets and the total T (no extra launch);
//   k_split_scatter per tile: the in-tile exclusive scan of the mask (thread
//                   popc -> warp shuffle scan -> CTA scan) places every element
//                   in a shared-memory staging tile -- trues [0, ct), falses
//                   [ct, m) -- which is then written as two contiguous runs:
//                   z[off_t + r] and z[T + (t*TILE - off_t) + q] (P283's
//                   offsets), coalesced, with the indices beside them.  The
//                   next tile's loads are issued before the current tile's
//                   stores (register double buffering).
//
// HBM bytes per element: mask read twice (1+1), payload read once and written
// once, indices written once (read once when they come from a previous pass).
// No look-back, no grid barrier: both kernels are pure streams.
#pragma once
#include <stdint.h>

#include "ptx.cuh"

namespace scan {
namespace split {

constexpr int kThreads = 512;
constexpr int kPer = 16;                   // contiguous elements per thread
constexpr int kTile = kThreads * kPer;     // 8192 elements per tile
constexpr int kWarps = kThreads / 32;

// Mask source: an int8 flag array (nonzero = true, R12) or bit `bit` of the
// order-preserving key code (P287: floats flip the MSB when positive and every
// bit when negative; signed ints flip the sign bit), inverted for ascending
// order so that 0-bits go first.
enum { SRC_FLAGS = 0, SRC_KEYBIT = 1 };
enum { KEY_U16 = 0, KEY_I16 = 1, KEY_F16 = 2, KEY_U32 = 3, KEY_I32 = 4, KEY_F32 = 5 };

// Code of two 16-bit keys packed in a word (or of one 32-bit key).
template <int KT>
__device__ __forceinline__ uint32_t key_code2(uint32_t w)
{
    if constexpr (KT == KEY_U16 || KT == KEY_U32) return w;
    else if constexpr (KT == KEY_I16) return w ^ 0x80008000u;
    else if constexpr (KT == KEY_I32) return w ^ 0x80000000u;
    else if constexpr (KT == KEY_F16) {
        const uint32_t s = (w >> 15) & 0x00010001u;        // sign of each half
        return w ^ (s * 0x7fffu | 0x80008000u);              // negative: all bits, else the MSB
    } else {
        return w ^ ((uint32_t)((int32_t)w >> 31) | 0x80000000u);
    }
}

struct SplitParams {
    const void* x;          // payload (elem_bytes each); for the sort: the keys
    void* z;                // output payload
    const int8_t* flags;    // SRC_FLAGS
    const int32_t* idx_in;  // nullable: input index of every element (else i)
    int32_t* idx_out;       // nullable
    int64_t* count_out;     // nullable, device: T
    uint32_t* counts;       // [ntiles] true count per tile        (workspace)
    uint32_t* offs;         // [ntiles] exclusive scan of counts   (workspace)
    uint32_t* hdr;          // [0] done counter, [2..3] T as uint64 (workspace)
    int64_t n;
    int ntiles;
    int compress;
    int bit;                // SRC_KEYBIT
    int descending;         // SRC_KEYBIT: 1-bits first
    int aligned;            // x, z, flags, idx 16-byte aligned
};

// True-mask of the 16 elements of one thread (bit j = element e0 + j) from
// its flag words / key words; elements >= m are 0.
template <int SRC, int ES, int KT>
__device__ __forceinline__ uint32_t mask16(const SplitParams& p, const uint4& fq, const uint32_t (&w)[ES * 4], int m)
{
    uint32_t bits = 0;
    if constexpr (SRC == SRC_FLAGS) {
        const uint32_t f[4] = {fq.x, fq.y, fq.z, fq.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            // 0x80 in every nonzero byte; the multiply moves bits 7/15/23/31 to
            // 28/29/30/31 without overlapping partial products (no carries)
            const uint32_t nz = __vcmpne4(f[j], 0u) & 0x80808080u;
            bits |= ((nz * 0x00204081u) >> 28) << (4 * j);
        }
    } else {
        const uint32_t inv = p.descending ? 0u : 1u;
        const int b = p.bit;
#pragma unroll
        for (int i = 0; i < ES * 4; ++i) {
            const uint32_t c = key_code2<KT>(w[i]);
            if constexpr (ES == 2) {
                bits |= ((((c >> b) & 1u) ^ inv) << (2 * i)) | ((((c >> (16 + b)) & 1u) ^ inv) << (2 * i + 1));
            } else {
                bits |= (((c >> b) & 1u) ^ inv) << i;
            }
        }
    }
    return m >= kPer ? bits : (bits & ((1u << m) - 1u));
}

// One thread's 16 elements: flag word, payload words, indices.
template <int ES>
struct Lane16 {
    uint4 fq;
    uint32_t w[ES * 4];
    int32_t ix[kPer];
};

template <int SRC, int ES, bool IDX_IN>
__device__ __forceinline__ void load_lane(const SplitParams& p, int64_t e0, int m, Lane16<ES>& L)
{
    const uint8_t* src = reinterpret_cast<const uint8_t*>(p.x) + e0 * ES;
    if (p.aligned && m >= kPer) {
        if constexpr (SRC == SRC_FLAGS) L.fq = ptx::ld_stream_v4(p.flags + e0);
#pragma unroll
        for (int v = 0; v < ES; ++v) {
            const uint4 q = ptx::ld_stream_v4(src + 16 * v);
            L.w[4 * v] = q.x; L.w[4 * v + 1] = q.y; L.w[4 * v + 2] = q.z; L.w[4 * v + 3] = q.w;
        }
        if constexpr (IDX_IN) {
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const uint4 q = ptx::ld_stream_v4(p.idx_in + e0 + 4 * v);
                L.ix[4 * v] = (int32_t)q.x; L.ix[4 * v + 1] = (int32_t)q.y;
                L.ix[4 * v + 2] = (int32_t)q.z; L.ix[4 * v + 3] = (int32_t)q.w;
            }
        }
    } else {
        uint32_t f[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int i = 0; i < ES * 4; ++i) L.w[i] = 0;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            if (j >= m) break;
            if constexpr (SRC == SRC_FLAGS) f[j >> 2] |= (uint32_t)(uint8_t)p.flags[e0 + j] << (8 * (j & 3));
            if constexpr (ES == 1) L.w[j >> 2] |= (uint32_t)src[j] << (8 * (j & 3));
            else if constexpr (ES == 2) L.w[j >> 1] |= (uint32_t)reinterpret_cast<const uint16_t*>(src)[j] << (16 * (j & 1));
            else if constexpr (ES == 4) L.w[j] = reinterpret_cast<const uint32_t*>(src)[j];
            else {
                L.w[2 * j] = reinterpret_cast<const uint32_t*>(src)[2 * j];
                L.w[2 * j + 1] = reinterpret_cast<const uint32_t*>(src)[2 * j + 1];
            }
            if constexpr (IDX_IN) L.ix[j] = p.idx_in[e0 + j];
        }
        L.fq = make_uint4(f[0], f[1], f[2], f[3]);
    }
    if constexpr (!IDX_IN) {
#pragma unroll
        for (int j = 0; j < kPer; ++j) L.ix[j] = (int32_t)(e0 + j);
    }
}

// ---- pass 1: true count per tile (a warp per tile); last CTA scans the counts ----
template <int SRC, int ES, int KT>
__global__ void __launch_bounds__(kThreads) k_split_count(const SplitParams p)
{
    __shared__ uint32_t s_red[kWarps];
    __shared__ bool s_last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gw = blockIdx.x * kWarps + warp, nw = gridDim.x * kWarps;
    constexpr int SZ = SRC == SRC_FLAGS ? 1 : ES;          // bytes per element read
    constexpr int kVec = kTile * SZ / (32 * 16);           // 16-byte loads per lane per tile
    constexpr int kBatch = kVec < 16 ? kVec : 16;
    const uint8_t* const base_ptr = SRC == SRC_FLAGS ? reinterpret_cast<const uint8_t*>(p.flags)
                                                     : reinterpret_cast<const uint8_t*>(p.x);
    const uint32_t inv = p.descending ? 0u : 1u;
    for (int t = gw; t < p.ntiles; t += nw) {
        const int64_t t0 = (int64_t)t * kTile;
        const int64_t rem = p.n - t0;
        uint32_t c = 0;
        if (p.aligned && rem >= kTile) {
            const uint8_t* tp = base_ptr + t0 * SZ;
#pragma unroll
            for (int b0 = 0; b0 < kVec; b0 += kBatch) {
                uint4 q[kBatch];
#pragma unroll
                for (int k = 0; k < kBatch; ++k) q[k] = ptx::ld_stream_v4(tp + ((b0 + k) * 32 + lane) * 16);
#pragma unroll
                for (int k = 0; k < kBatch; ++k) {
                    const uint32_t wv[4] = {q[k].x, q[k].y, q[k].z, q[k].w};
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        if constexpr (SRC == SRC_FLAGS) {
                            c += __popc((((wv[i] & 0x7f7f7f7fu) + 0x7f7f7f7fu) | wv[i]) & 0x80808080u);
                        } else if constexpr (ES == 2) {
                            const uint32_t cd = key_code2<KT>(wv[i]);
                            c += __popc(((cd >> p.bit) & 0x00010001u) ^ (inv * 0x00010001u));
                        } else {
                            c += ((key_code2<KT>(wv[i]) >> p.bit) & 1u) ^ inv;
                        }
                    }
                }
            }
        } else {
            const int m = rem > kTile ? kTile : (int)rem;
            for (int e = lane; e < m; e += 32) {
                if constexpr (SRC == SRC_FLAGS) {
                    c += p.flags[t0 + e] != 0 ? 1u : 0u;
                } else {
                    uint32_t k;
                    if constexpr (ES == 2) k = reinterpret_cast<const uint16_t*>(p.x)[t0 + e];
                    else k = reinterpret_cast<const uint32_t*>(p.x)[t0 + e];
                    c += ((key_code2<KT>(k) >> p.bit) & 1u) ^ inv;
                }
            }
        }
        c = __reduce_add_sync(0xffffffffu, c);
        if (lane == 0) p.counts[t] = c;
    }
    // last CTA: exclusive scan of the tile counts (fixed order, uint64 running total)
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = ptx::claim_add(&p.hdr[0], 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    uint64_t carry = 0;
    constexpr int kPerT = 16;  // counts per thread per pass (4 x 16-byte loads)
    for (int base = 0; base < p.ntiles; base += kThreads * kPerT) {
        uint32_t v[kPerT];
        uint32_t s = 0;
        const int i0 = base + tid * kPerT;
        if (i0 + kPerT <= p.ntiles) {
#pragma unroll
            for (int k = 0; k < kPerT; k += 4) {
                const uint4 q = __ldcg(reinterpret_cast<const uint4*>(p.counts + i0 + k));
                v[k] = q.x; v[k + 1] = q.y; v[k + 2] = q.z; v[k + 3] = q.w;
            }
        } else {
#pragma unroll
            for (int k = 0; k < kPerT; ++k) v[k] = i0 + k < p.ntiles ? __ldcg(&p.counts[i0 + k]) : 0u;
        }
#pragma unroll
        for (int k = 0; k < kPerT; ++k) s += v[k];
        uint32_t incl = s;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += y;
        }
        __syncthreads();
        if (lane == 31) s_red[warp] = incl;
        __syncthreads();
        uint32_t xw = lane < kWarps ? s_red[lane] : 0u;
        uint32_t xi = xw;
#pragma unroll
        for (int d = 1; d < kWarps; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, xi, d);
            if (lane >= d) xi += y;
        }
        const uint32_t tot = __shfl_sync(0xffffffffu, xi, kWarps - 1);
        const uint32_t wpre = __shfl_sync(0xffffffffu, xi - xw, warp);
        uint64_t run = carry + wpre + (incl - s);
        if (i0 + kPerT <= p.ntiles) {
            uint32_t o[kPerT];
#pragma unroll
            for (int k = 0; k < kPerT; ++k) {
                o[k] = (uint32_t)run;
                run += v[k];
            }
#pragma unroll
            for (int k = 0; k < kPerT; k += 4)
                *reinterpret_cast<uint4*>(p.offs + i0 + k) = make_uint4(o[k], o[k + 1], o[k + 2], o[k + 3]);
        } else {
#pragma unroll
            for (int k = 0; k < kPerT; ++k) {
                if (i0 + k < p.ntiles) p.offs[i0 + k] = (uint32_t)run;
                run += v[k];
            }
        }
        carry += tot;
    }
    if (tid == 0) {
        reinterpret_cast<uint64_t*>(p.hdr)[1] = carry;
        if (p.count_out) *p.count_out = (int64_t)carry;
        p.hdr[0] = 0;  // reset for the next call
    }
}

// ---- pass 2: in-tile scan of the mask, stage, write two contiguous runs ----
template <int SRC, int ES, int KT, bool IDX_IN>
__global__ void __launch_bounds__(kThreads) k_split_scatter(const SplitParams p)
{
    extern __shared__ __align__(16) uint8_t s_stage[];  // kTile * ES payload + kTile * 4 indices
    int32_t* const s_idx = reinterpret_cast<int32_t*>(s_stage + kTile * ES);
    __shared__ uint32_t s_red[kWarps];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t T = reinterpret_cast<const uint64_t*>(p.hdr)[1];
    uint8_t* const zb = reinterpret_cast<uint8_t*>(p.z);

    auto lane_m = [&](int t) {
        const int64_t r = p.n - ((int64_t)t * kTile + (int64_t)tid * kPer);
        return r <= 0 ? 0 : (r > kPer ? kPer : (int)r);
    };

    int t = blockIdx.x;
    Lane16<ES> cur;
    if (t < p.ntiles) {
        const int m = lane_m(t);
        if (m > 0) load_lane<SRC, ES, IDX_IN>(p, (int64_t)t * kTile + (int64_t)tid * kPer, m, cur);
    }
    for (; t < p.ntiles; t += gridDim.x) {
        const int64_t t0 = (int64_t)t * kTile;
        const int m = lane_m(t);
        const int64_t rt = p.n - t0;
        const int mt = rt > kTile ? kTile : (int)rt;  // valid elements in the tile
        const uint32_t bits = m > 0 ? mask16<SRC, ES, KT>(p, cur.fq, cur.w, m) : 0u;

        // in-tile exclusive scan of the true counts (P283's exclusive scan)
        const uint32_t c = __popc(bits);
        uint32_t incl = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += y;
        }
        if (lane == 31) s_red[warp] = incl;
        __syncthreads();
        uint32_t wpre = 0, ct = 0;
#pragma unroll
        for (int k = 0; k < kWarps; ++k) {
            const uint32_t x = s_red[k];
            if (k < warp) wpre += x;
            ct += x;
        }
        const uint32_t lt = wpre + incl - c;              // trues before this thread in the tile
        const uint32_t lf = (uint32_t)(tid * kPer) - lt;  // falses before this thread

        // stage: trues at [0, ct), falses at [ct, mt)
        uint32_t rt_ = lt, rf = ct + lf;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            if (j >= m) break;
            const bool tr = (bits >> j) & 1u;
            const uint32_t pos = tr ? rt_++ : rf++;
            if constexpr (ES == 1) s_stage[pos] = (uint8_t)(cur.w[j >> 2] >> (8 * (j & 3)));
            else if constexpr (ES == 2) reinterpret_cast<uint16_t*>(s_stage)[pos] = (uint16_t)(cur.w[j >> 1] >> (16 * (j & 1)));
            else if constexpr (ES == 4) reinterpret_cast<uint32_t*>(s_stage)[pos] = cur.w[j];
            else reinterpret_cast<uint2*>(s_stage)[pos] = make_uint2(cur.w[2 * j], cur.w[2 * j + 1]);
            s_idx[pos] = cur.ix[j];
        }
        __syncthreads();

        // prefetch the next tile while this one is written out
        const int tn = t + gridDim.x;
        if (tn < p.ntiles) {
            const int mn = lane_m(tn);
            if (mn > 0) load_lane<SRC, ES, IDX_IN>(p, (int64_t)tn * kTile + (int64_t)tid * kPer, mn, cur);
        }

        // two contiguous runs: z[off_t + s] (s < ct), z[T + t0 - off_t + (s - ct)]
        const uint64_t off_t = p.offs[t];
        const uint64_t fbase = T + (uint64_t)t0 - off_t;
        const int lim = p.compress ? (int)ct : mt;
        for (int s = tid; s < lim; s += kThreads) {
            const uint64_t dest = s < (int)ct ? off_t + s : fbase + (uint64_t)(s - (int)ct);
            if constexpr (ES == 1) zb[dest] = s_stage[s];
            else if constexpr (ES == 2) reinterpret_cast<uint16_t*>(zb)[dest] = reinterpret_cast<const uint16_t*>(s_stage)[s];
            else if constexpr (ES == 4) reinterpret_cast<uint32_t*>(zb)[dest] = reinterpret_cast<const uint32_t*>(s_stage)[s];
            else reinterpret_cast<uint2*>(zb)[dest] = reinterpret_cast<const uint2*>(s_stage)[s];
            if (p.idx_out) p.idx_out[dest] = s_idx[s];
        }
        __syncthreads();  // staging reused by the next tile
    }
}

// Write a run of `len` staged elements (staging index s0.., global index g0..,
// s0 == g0 mod 16/ES) with 16-byte stores in the middle, scalar head/tail.
template <int ES>
__device__ __forceinline__ void write_run(uint8_t* z, int32_t* idx, uint64_t g0, const uint8_t* st, const int32_t* sti,
                                          int s0, int len, int tid)
{
    constexpr int VE = 16 / ES;
    int head = (int)((VE - (int)(g0 % VE)) % VE);
    head = head < len ? head : len;
    const int nv = (len - head) / VE;
    const int body_end = head + nv * VE;
    auto scalar = [&](int i) {
        const uint64_t d = g0 + (uint64_t)i;
        if constexpr (ES == 1) z[d] = st[s0 + i];
        else if constexpr (ES == 2) reinterpret_cast<uint16_t*>(z)[d] = reinterpret_cast<const uint16_t*>(st)[s0 + i];
        else reinterpret_cast<uint32_t*>(z)[d] = reinterpret_cast<const uint32_t*>(st)[s0 + i];
        if (idx) idx[d] = sti[s0 + i];
    };
    if (tid < head) scalar(tid);
    const int tail = len - body_end;
    if (tid < tail) scalar(body_end + tid);
    uint4* zv = reinterpret_cast<uint4*>(z + (g0 + head) * ES);
    const uint4* sv = reinterpret_cast<const uint4*>(st + (size_t)(s0 + head) * ES);
    for (int v = tid; v < nv; v += kThreads) zv[v] = sv[v];
    if (idx) {
        uint4* iv = reinterpret_cast<uint4*>(idx + g0 + head);
        const uint4* siv = reinterpret_cast<const uint4*>(sti + s0 + head);
        for (int v = tid; v < nv * (VE / 4); v += kThreads) iv[v] = siv[v];
    }
}

// Packed staging (payload << 16 | local index): write a run of `len` staged
// words (staging index s0.., global index g0.., s0 == g0 mod 4); 4-element
// groups go out as one payload vector (8 B fp16 / 4 B int8) and one 16-byte
// index vector; idx = tile base + local index.
template <int ES>
__device__ __forceinline__ void write_run_packed(uint8_t* z, int32_t* idx, uint64_t g0, int32_t t0, const uint32_t* st,
                                                 int s0, int len, int tid)
{
    int head = (int)((4 - (int)(g0 & 3)) & 3);
    head = head < len ? head : len;
    const int nv = (len - head) >> 2;
    const int body_end = head + nv * 4;
    auto scalar = [&](int i) {
        const uint32_t w = st[s0 + i];
        const uint64_t d = g0 + (uint64_t)i;
        if constexpr (ES == 2) reinterpret_cast<uint16_t*>(z)[d] = (uint16_t)(w >> 16);
        else z[d] = (uint8_t)(w >> 16);
        if (idx) idx[d] = t0 + (int32_t)(w & 0xffffu);
    };
    if (tid < head) scalar(tid);
    const int tail = len - body_end;
    if (tid < tail) scalar(body_end + tid);
    const uint4* sv = reinterpret_cast<const uint4*>(st + s0 + head);
    const uint64_t gb = g0 + head;
    for (int v = tid; v < nv; v += kThreads) {
        const uint4 q = sv[v];
        if constexpr (ES == 2) {
            const uint2 pay = make_uint2(__byte_perm(q.x, q.y, 0x7632), __byte_perm(q.z, q.w, 0x7632));
            *reinterpret_cast<uint2*>(z + (gb + 4 * (uint64_t)v) * 2) = pay;
        } else {
            const uint32_t pay = __byte_perm(__byte_perm(q.x, q.y, 0x0062), __byte_perm(q.z, q.w, 0x0062), 0x5410);
            *reinterpret_cast<uint32_t*>(z + gb + 4 * (uint64_t)v) = pay;
        }
        if (idx) {
            const uint4 iv = make_uint4(t0 + (q.x & 0xffffu), t0 + (q.y & 0xffffu), t0 + (q.z & 0xffffu),
                                        t0 + (q.w & 0xffffu));
            *reinterpret_cast<uint4*>(idx + gb + 4 * (uint64_t)v) = iv;
        }
    }
}

// ---- pass 2, TMA variant: a producer warp streams tiles into a shared-memory
// ring (cp.async.bulk, mbarrier completion), so the HBM latency is hidden by
// the ring depth instead of occupancy; 16 compute warps scan, stage and write.
// One CTA per SM, tiles t = blockIdx.x + k * gridDim.x.  Requires 16-byte
// aligned buffers; the ragged last tile is read straight from global memory.
#ifndef SPLIT_SMEM_KB
#define SPLIT_SMEM_KB 105
#endif
#ifndef SPLIT_CTAS
#define SPLIT_CTAS 2
#endif
template <int SRC, int ES, bool IDX_IN>
struct TmaCfg {
    static constexpr int kNC = kWarps;                        // compute warps (512 threads)
    static constexpr int kThreadsT = (1 + kNC) * 32;          // + producer warp
    static constexpr int kFlagB = SRC == SRC_FLAGS ? kTile : 0;
    static constexpr int kPayB = kTile * ES;
    static constexpr int kIdxB = IDX_IN ? kTile * 4 : 0;
    static constexpr int kSlot = kFlagB + kPayB + kIdxB;
    static constexpr int kSlack = 64;                         // alignment shifts of the two runs
    // !IDX_IN and ES <= 2: one packed word per element, (payload << 16) | local index
    static constexpr bool kPack = !IDX_IN && ES <= 2;
    static constexpr int kStage = kPack ? (kTile + kSlack) * 4 : (kTile + kSlack) * (ES + 4);
    // shared memory per CTA; the packed (!IDX_IN, ES <= 2) variants may run SPLIT_CTAS per SM
    static constexpr int kCtas = (!IDX_IN && ES <= 2) ? SPLIT_CTAS : 1;
    static constexpr int kBudget = (!IDX_IN && ES <= 2) ? SPLIT_SMEM_KB * 1024 : 200 * 1024;
    static constexpr int kNB = (kBudget - kStage) / kSlot > 4 ? 4 : (kBudget - kStage) / kSlot;
    static constexpr size_t kSmem = (size_t)kNB * kSlot + kStage + 128;
};

// CMP: compress -- only the trues are staged and written.
template <int SRC, int ES, int KT, bool IDX_IN, bool CMP = false>
__global__ void __launch_bounds__(TmaCfg<SRC, ES, IDX_IN>::kThreadsT, TmaCfg<SRC, ES, IDX_IN>::kCtas) k_split_scatter_tma(const SplitParams p)
{
    using C = TmaCfg<SRC, ES, IDX_IN>;
    constexpr int NB = C::kNB;
    static_assert(NB >= 2, "ring of at least two tiles");
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* const ring = smem;
    uint8_t* const s_stage = smem + NB * C::kSlot;
    int32_t* const s_idx = reinterpret_cast<int32_t*>(s_stage + (kTile + C::kSlack) * ES);
    __shared__ __align__(8) uint64_t full[NB];
    __shared__ __align__(8) uint64_t empty[NB];
    __shared__ uint32_t s_red[2][kWarps];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t full_tiles = p.n / kTile;  // tiles [0, full_tiles) are whole
    if (tid == 0) {
        for (int s = 0; s < NB; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], C::kNC);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();

    if (warp == 0) {
        // ============ producer ============
        if (lane == 0) {
            const uint64_t pol = ptx::policy_evict_first();
            int s = 0;
            uint32_t ph = 0;
            bool wrapped = false;
            for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
                if (wrapped) ptx::mbar_wait(&empty[s], ph ^ 1u);
                uint8_t* dst = ring + s * C::kSlot;
                const int64_t t0 = (int64_t)t * kTile;
                if (t < full_tiles) {
                    ptx::mbar_arrive_expect_tx(&full[s], (uint32_t)C::kSlot);
                    if constexpr (SRC == SRC_FLAGS) ptx::tma_load_1d(dst, p.flags + t0, kTile, &full[s], pol);
                    ptx::tma_load_1d(dst + C::kFlagB, reinterpret_cast<const uint8_t*>(p.x) + t0 * ES, C::kPayB, &full[s], pol);
                    if constexpr (IDX_IN) ptx::tma_load_1d(dst + C::kFlagB + C::kPayB, p.idx_in + t0, C::kIdxB, &full[s], pol);
                } else {
                    ptx::mbar_arrive(&full[s]);  // ragged tile: compute warps read global memory
                }
                if (++s == NB) {
                    s = 0;
                    ph ^= 1u;
                    wrapped = true;
                }
            }
        }
        return;
    }

    // ============ compute (512 threads) ============
    const int ct_ = tid - 32;  // compute thread 0..511
    const int cw = warp - 1, cl = lane;
    const uint64_t T = reinterpret_cast<const uint64_t*>(p.hdr)[1];
    uint8_t* const zb = reinterpret_cast<uint8_t*>(p.z);
    int s = 0;
    uint32_t ph = 0;
    int par = 0;
    for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x, par ^= 1) {
        const int64_t t0 = (int64_t)t * kTile;
        const int64_t e0 = t0 + (int64_t)ct_ * kPer;
        const int64_t rr = p.n - e0;
        const int m = rr <= 0 ? 0 : (rr > kPer ? kPer : (int)rr);
        const int64_t rt = p.n - t0;
        const int mt = rt > kTile ? kTile : (int)rt;
        ptx::mbar_wait(&full[s], ph);
        Lane16<ES> L;
        if (t < full_tiles) {
            const uint8_t* slot = ring + s * C::kSlot;
            if constexpr (SRC == SRC_FLAGS) L.fq = *reinterpret_cast<const uint4*>(slot + ct_ * 16);
#pragma unroll
            for (int v = 0; v < ES; ++v) {
                const uint4 q = *reinterpret_cast<const uint4*>(slot + C::kFlagB + ct_ * 16 * ES + 16 * v);
                L.w[4 * v] = q.x; L.w[4 * v + 1] = q.y; L.w[4 * v + 2] = q.z; L.w[4 * v + 3] = q.w;
            }
            if constexpr (IDX_IN) {
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const uint4 q = *reinterpret_cast<const uint4*>(slot + C::kFlagB + C::kPayB + ct_ * 64 + 16 * v);
                    L.ix[4 * v] = (int32_t)q.x; L.ix[4 * v + 1] = (int32_t)q.y;
                    L.ix[4 * v + 2] = (int32_t)q.z; L.ix[4 * v + 3] = (int32_t)q.w;
                }
            } else {
#pragma unroll
                for (int j = 0; j < kPer; ++j) L.ix[j] = (int32_t)(e0 + j);
            }
        } else if (m > 0) {
            load_lane<SRC, ES, IDX_IN>(p, e0, m, L);
        }
        __syncwarp();
        if (cl == 0) ptx::mbar_arrive(&empty[s]);  // slot read into registers
        if (++s == NB) {
            s = 0;
            ph ^= 1u;
        }
        const uint32_t bits = m > 0 ? mask16<SRC, ES, KT>(p, L.fq, L.w, m) : 0u;

        // in-tile exclusive scan of the true counts (P283)
        const uint32_t c = __popc(bits);
        uint32_t incl = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
            if (cl >= d) incl += y;
        }
        if (cl == 31) s_red[par][cw] = incl;
        ptx::named_bar_sync(1, kThreads);  // also: the previous tile's staging has been written out
        uint32_t xw = cl < kWarps ? s_red[par][cl] : 0u;  // warp totals, scanned by every warp
        uint32_t xi = xw;
#pragma unroll
        for (int d = 1; d < kWarps; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, xi, d);
            if (cl >= d) xi += y;
        }
        const uint32_t ct = __shfl_sync(0xffffffffu, xi, kWarps - 1);
        const uint32_t wpre = __shfl_sync(0xffffffffu, xi - xw, cw);
        const uint32_t lt = wpre + incl - c;              // trues before this thread in the tile
        const uint32_t lf = (uint32_t)(ct_ * kPer) - lt;  // falses before this thread
        const uint64_t off_t = p.offs[t];
        const uint64_t fbase = T + (uint64_t)t0 - off_t;
        if constexpr (C::kPack) {
            // staging index == global index (mod 4): 4-element groups store as one vector
            uint32_t* const s_pk = reinterpret_cast<uint32_t*>(s_stage);
            const int sh_t = (int)(off_t & 3);
            const int fst = ((sh_t + (int)ct + 3) & ~3) + (int)(fbase & 3);
            const uint32_t tb = sh_t + lt, fb = fst + lf;
#pragma unroll
            for (int j = 0; j < kPer; ++j) {
                if (j >= m) break;
                const uint32_t below = __popc(bits & ((1u << j) - 1u));  // trues before j in this thread
                const bool tr = (bits >> j) & 1u;
                const uint32_t pos = tr ? tb + below : fb + (uint32_t)j - below;
                uint32_t pay;
                if constexpr (ES == 2) pay = (L.w[j >> 1] >> (16 * (j & 1))) & 0xffffu;
                else pay = (L.w[j >> 2] >> (8 * (j & 3))) & 0xffu;
                if (!CMP || tr) s_pk[pos] = (pay << 16) | (uint32_t)(ct_ * kPer + j);
            }
            ptx::named_bar_sync(1, kThreads);
            write_run_packed<ES>(zb, p.idx_out, off_t, (int32_t)t0, s_pk, sh_t, (int)ct, ct_);
            if (!CMP) write_run_packed<ES>(zb, p.idx_out, fbase, (int32_t)t0, s_pk, fst, mt - (int)ct, ct_);
        } else {
            // Staging positions are shifted so that staging index == global index
            // (mod VE): the middle of each run is then written with 16-byte stores.
            constexpr int VE = 16 / ES;  // elements per 16-byte payload vector (ES <= 4)
            const int sh_t = (int)(off_t % VE);
            const int fst = ((sh_t + (int)ct + VE - 1) / VE) * VE + (int)(fbase % VE);
            uint32_t rt_ = sh_t + lt, rf = fst + lf;
#pragma unroll
            for (int j = 0; j < kPer; ++j) {
                if (j >= m) break;
                const bool tr = (bits >> j) & 1u;
                const uint32_t pos = tr ? rt_++ : rf++;
                if constexpr (ES == 1) s_stage[pos] = (uint8_t)(L.w[j >> 2] >> (8 * (j & 3)));
                else if constexpr (ES == 2) reinterpret_cast<uint16_t*>(s_stage)[pos] = (uint16_t)(L.w[j >> 1] >> (16 * (j & 1)));
                else reinterpret_cast<uint32_t*>(s_stage)[pos] = L.w[j];
                s_idx[pos] = L.ix[j];
            }
            ptx::named_bar_sync(1, kThreads);
            write_run<ES>(zb, p.idx_out, off_t, s_stage, s_idx, sh_t, (int)ct, ct_);
            if (!CMP) write_run<ES>(zb, p.idx_out, fbase, s_stage, s_idx, fst, mt - (int)ct, ct_);
        }
        // the next tile's first named barrier orders these staging reads before its writes
    }
}

}  // namespace split
}  // namespace scan

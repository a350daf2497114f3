// radix.cuh -- LSB radix sort with 8-bit digits: the B200-idiomatic
// multi-bit variant of the paper's radix sort by 1-bit splits (Sec. 5.3,
// P286-287).  A 1-bit split is a 2-way stable partition
// whose offsets are an exclusive scan of the mask; an 8-bit digit pass is the
// 256-way stable partition whose offsets are the exclusive scan of the
// per-(digit, tile) counts in digit-major order -- the same scan, over 256
// counters per tile instead of one.  16-bit keys take 2 passes, 32-bit keys 4
// (instead of 16 / 32 splits).
//
// Per pass:
//   k_digit_count    counts[d * ntiles + t] = #elements of tile t with digit d
//                    (warp-private shared-memory histograms, atomics);
//   scan_exclusive   over the 256 * ntiles counts (this library's scan, int32)
//                    -> offs[d * ntiles + t], the global start of (d, t);
//   k_digit_scatter  stable rank of every element among the same digit inside
//                    its tile (warp rounds of 32 consecutive elements,
//                    ballot-based peer groups, warp-private running
//                    histograms, then a CTA prefix over warps and digits),
//                    the tile staged in shared memory in (digit, rank) order
//                    and written out as per-digit runs:
//                    dest = offs[d][t] + rank_in_tile(d).
// The key code is P287's order-preserving encoding (floats: MSB flipped when
// positive, every bit when negative; signed ints: sign bit flipped); keys move
// unchanged.  Stable; descending uses digit' = 255 - digit.
#pragma once
#include <stdint.h>

#include "ptx.cuh"
#include "split.cuh"  // key_code2, KEY_* enums

namespace scan {
namespace radix {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
#ifndef RADIX_ROUNDS
#define RADIX_ROUNDS 16
#endif
#ifndef RADIX_SMEM_KB
#define RADIX_SMEM_KB 200
#endif
#ifndef RADIX_CTAS
#define RADIX_CTAS 1
#endif
constexpr int kRounds = RADIX_ROUNDS;             // rounds of 32 elements per warp
constexpr int kTile = kThreads * kRounds;         // 8192 elements per tile
constexpr int kDigits = 256;

struct DigitParams {
    const void* keys_in;
    void* keys_out;
    const int32_t* idx_in;   // nullable: the identity permutation
    int32_t* idx_out;
    uint32_t* counts;        // [256 * ntiles], digit-major
    const uint32_t* offs;    // [256 * ntiles], per digit: exclusive scan of its tile counts (row scans)
    const uint32_t* dbase;   // [256] exclusive scan of the digit totals
    int64_t n;
    int ntiles;
    int shift;               // digit = (code >> shift) & 0xff
    int descending;
    // Segmented (row-batched) sort: cols > 0 sorts every row of `cols` contiguous
    // keys on its own.  Tiles never cross rows (tpr tiles per row, the last one
    // ragged); counts / offs are laid out [row][digit][tile], so ONE exclusive row
    // scan per row (scan_rows) gives every (digit, tile) its row-local start with
    // the digit bases included; indices are column indices.
    int64_t cols;
    int tpr;
    int count_pf;            // k_digit_count: L2 bulk prefetch of the CTA's next tile (tiles ahead, 0 = off)
};

// Geometry of tile t: first element, element count, the row's first element,
// the counts index of (digit 0, this tile) and the stride between digits.
struct TileGeom {
    int64_t t0, row0, c0;
    int mt;
    int64_t dstride;
};
__device__ __forceinline__ TileGeom tile_geom(const DigitParams& p, int t)
{
    TileGeom g;
    if (p.cols > 0) {
        const int64_t row = t / p.tpr, k = t - row * p.tpr;
        g.row0 = row * p.cols;
        g.t0 = g.row0 + k * kTile;
        const int64_t rem = p.cols - k * kTile;
        g.mt = rem > kTile ? kTile : (int)rem;
        g.c0 = row * (int64_t)kDigits * p.tpr + k;
        g.dstride = p.tpr;
    } else {
        g.row0 = 0;
        g.t0 = (int64_t)t * kTile;
        const int64_t rem = p.n - g.t0;
        g.mt = rem > kTile ? kTile : (int)rem;
        g.c0 = t;
        g.dstride = p.ntiles;
    }
    return g;
}

template <int KT, int ES>
__device__ __forceinline__ uint32_t load_key(const void* base, int64_t i)
{
    if constexpr (ES == 2) return __ldg(reinterpret_cast<const uint16_t*>(base) + i);
    else return __ldg(reinterpret_cast<const uint32_t*>(base) + i);
}

template <int KT>
__device__ __forceinline__ uint32_t digit_of(uint32_t key, int shift, int descending)
{
    const uint32_t d = (split::key_code2<KT>(key) >> shift) & 0xffu;
    return descending ? 255u - d : d;
}

// Lanes of the warp holding the same digit as this lane (among `valid` lanes):
// the AND of 8 bit-wise ballots -- the warp multi-split; on sm_100a this is much
// cheaper than MATCH.ANY (measured: 415 -> 333 us for a 2^24 fp16 sort).
__device__ __forceinline__ uint32_t digit_peers(uint32_t d, bool valid)
{
#ifdef RADIX_MATCH  // A/B build: MATCH.ANY (invalid lanes get a unique value: singletons)
    return __match_any_sync(0xffffffffu, valid ? d : 0x100u | (threadIdx.x & 31u));
#endif
    uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const bool bit = (d & (1u << b)) != 0u;  // one LOP3 to a predicate (was a shift + compare)
        const uint32_t bb = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? bb : ~bb;
    }
    return peers;
}

// ---- counts per (digit, tile) --------------------------------------------------
#ifndef RADIX_COUNT_CTAS
#define RADIX_COUNT_CTAS 3
#endif
template <int KT, int ES>
__global__ void __launch_bounds__(kThreads, RADIX_COUNT_CTAS) k_digit_count(const DigitParams p)
{
    // two warp-private histogram sets, used by alternate tiles: the thread that
    // sums a digit's 16 warp counts clears them for the tile after next, so each
    // tile needs ONE CTA barrier (between its atomics and its sums)
    __shared__ uint32_t s_hist[2][kWarps][kDigits];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // one thread prefetches the CTA's tile count_pf steps ahead into L2, so the
    // next iteration's key loads meet L2 latency instead of HBM latency
    auto prefetch = [&](int tp) {
        if (tp < p.ntiles) {
            const TileGeom pg = tile_geom(p, tp);
            const uintptr_t a = (uintptr_t)p.keys_in + (uintptr_t)(pg.t0 * ES);
            const uintptr_t a0 = (a + 15) & ~(uintptr_t)15, a1 = (a + (uintptr_t)pg.mt * ES) & ~(uintptr_t)15;
            if (a1 > a0) ptx::l2_prefetch_bulk(reinterpret_cast<const void*>(a0), (uint32_t)(a1 - a0));
        }
    };
    if (tid == 0)
        for (int k = 1; k < p.count_pf; ++k) prefetch(blockIdx.x + k * gridDim.x);
    for (int i = tid; i < 2 * kWarps * kDigits; i += kThreads) (&s_hist[0][0][0])[i] = 0;
    __syncthreads();
    int hb = 0;
    for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x, hb ^= 1) {
        if (tid == 0 && p.count_pf > 0) prefetch(t + p.count_pf * gridDim.x);
        const TileGeom tg = tile_geom(p, t);
        uint32_t(&h)[kDigits] = s_hist[hb][warp];
        const char* kb = reinterpret_cast<const char*>(p.keys_in) + tg.t0 * ES;
        if (tg.mt == kTile && ((uintptr_t)kb & 15) == 0) {
            // whole, 16-byte aligned tile: 16-byte loads (counting ignores order)
            constexpr int KPV = 16 / ES;                 // keys per 16-byte vector
            constexpr int NV = kRounds / KPV;            // vectors per thread
            uint4 v[NV];
#pragma unroll
            for (int r = 0; r < NV; ++r) v[r] = __ldg(reinterpret_cast<const uint4*>(kb) + r * kThreads + tid);
#pragma unroll
            for (int r = 0; r < NV; ++r) {
                const uint32_t w[4] = {v[r].x, v[r].y, v[r].z, v[r].w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if constexpr (ES == 4) {
                        atomicAdd(&h[digit_of<KT>(w[j], p.shift, p.descending)], 1u);
                    } else {
                        atomicAdd(&h[digit_of<KT>(w[j] & 0xffffu, p.shift, p.descending)], 1u);
                        atomicAdd(&h[digit_of<KT>(w[j] >> 16, p.shift, p.descending)], 1u);
                    }
                }
            }
        } else {
            const int l0 = warp * (kRounds * 32);
            uint32_t key[kRounds];
#pragma unroll
            for (int r = 0; r < kRounds; ++r) {
                const int li = l0 + r * 32 + lane;
                key[r] = li < tg.mt ? load_key<KT, ES>(p.keys_in, tg.t0 + li) : 0u;
            }
#pragma unroll
            for (int r = 0; r < kRounds; ++r) {
                const int li = l0 + r * 32 + lane;
                if (li < tg.mt) atomicAdd(&h[digit_of<KT>(key[r], p.shift, p.descending)], 1u);
            }
        }
        __syncthreads();
        for (int d = tid; d < kDigits; d += kThreads) {
            uint32_t c = 0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                c += s_hist[hb][w][d];
                s_hist[hb][w][d] = 0;
            }
            p.counts[tg.c0 + (int64_t)d * tg.dstride] = c;
        }
    }
}

// ---- stable 256-way partition of every tile to the scanned offsets ---------------
template <int KT, int ES, bool IDX_IN>
__global__ void __launch_bounds__(kThreads) k_digit_scatter(const DigitParams p)
{
    using K = typename std::conditional<ES == 2, uint16_t, uint32_t>::type;
    __shared__ uint32_t s_hist[kWarps][kDigits];   // per-warp running counts, then prefix over warps
    __shared__ uint32_t s_tdp[kDigits];            // tile-local start of digit d
    __shared__ int64_t s_gb[kDigits];              // global start of digit d minus s_tdp[d]
    __shared__ uint32_t s_wsum[kWarps];
    extern __shared__ __align__(16) uint8_t s_dyn[];
    K* const st_key = reinterpret_cast<K*>(s_dyn);
    int32_t* const st_idx = reinterpret_cast<int32_t*>(s_dyn + kTile * sizeof(K));

    __shared__ uint32_t s_dbase[kDigits];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    // digit bases: exclusive scan over d of the digit totals (last row-scan
    // entry + last tile count of every digit)
    if (tid < kDigits) {
        // (segmented: the row scans already include the digit bases)
        const int64_t last = (int64_t)tid * p.ntiles + p.ntiles - 1;
        const uint32_t tot = p.cols > 0 ? 0u : p.offs[last] + p.counts[last];
        uint32_t incl = tot;
#pragma unroll
        for (int k = 1; k < 32; k <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, k);
            if (lane >= k) incl += y;
        }
        if (lane == 31) s_wsum[warp] = incl;
        s_dbase[tid] = incl - tot;
    }
    __syncthreads();
    if (tid < kDigits) {
        uint32_t off = 0;
        for (int w = 0; w < warp; ++w) off += s_wsum[w];
        s_dbase[tid] += off;
    }
    __syncthreads();
    for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
        const TileGeom tg = tile_geom(p, t);
        const int64_t t0 = tg.t0;
        const int mt = tg.mt;
        const int64_t tend = t0 + mt;
        const uint32_t my_off = tid < kDigits ? __ldg(p.offs + tg.c0 + (int64_t)tid * tg.dstride) : 0u;
        for (int i = tid; i < kWarps * kDigits; i += kThreads) (&s_hist[0][0])[i] = 0;
        __syncthreads();

        // 1. warp rounds: rank among equal digits, in element order
        const int64_t w0 = t0 + warp * (kRounds * 32);
        // ES == 2: key | rank << 16 in one register; ES == 4: key and rank apart
        uint32_t key[kRounds], rank[ES == 2 ? 1 : kRounds];
        int32_t ix[IDX_IN ? kRounds : 1];
#pragma unroll
        for (int r = 0; r < kRounds; ++r) {
            const int64_t e = w0 + r * 32 + lane;
            const bool ok = e < tend;
            key[r] = ok ? load_key<KT, ES>(p.keys_in, e) : 0u;
            if constexpr (IDX_IN) ix[r] = ok ? __ldg(p.idx_in + e) : 0;
        }
#pragma unroll
        for (int r = 0; r < kRounds; ++r) {
            const int64_t e = w0 + r * 32 + lane;
            const bool ok = e < tend;
            const uint32_t d = digit_of<KT>(key[r], p.shift, p.descending);
            const uint32_t peers = digit_peers(d, ok);
            const uint32_t before = __popc(peers & lt_mask);
            uint32_t base = 0;
            if (ok) base = s_hist[warp][d];
            if constexpr (ES == 2) key[r] |= (base + before) << 16;
            else rank[r] = base + before;
            __syncwarp();
            if (ok && before == 0) s_hist[warp][d] = base + __popc(peers);  // group leader
            __syncwarp();
        }
        __syncthreads();

        // 2. prefix over warps per digit, tile counts, exclusive scan over digits
        if (tid < kDigits) {
            uint32_t run = 0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                const uint32_t c = s_hist[w][tid];
                s_hist[w][tid] = run;
                run += c;
            }
            // block-level exclusive scan of run (the tile's digit counts) over 256 digits
            uint32_t incl = run;
#pragma unroll
            for (int dd = 1; dd < 32; dd <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, dd);
                if (lane >= dd) incl += y;
            }
            if (lane == 31) s_wsum[warp] = incl;
            s_tdp[tid] = incl - run;  // within-warp exclusive, warp offset added below
        }
        __syncthreads();
        if (tid < kDigits) {
            uint32_t off = 0;
            for (int w = 0; w < warp; ++w) off += s_wsum[w];
            const uint32_t tdp = s_tdp[tid] + off;
            s_tdp[tid] = tdp;
            s_gb[tid] = tg.row0 + (int64_t)s_dbase[tid] + (int64_t)my_off - (int64_t)tdp;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) s_hist[w][tid] += tdp;  // one staging table
        }
        __syncthreads();

        // 3. stage in (digit, rank) order
#pragma unroll
        for (int r = 0; r < kRounds; ++r) {
            const int64_t e = w0 + r * 32 + lane;
            if (e < tend) {
                const uint32_t k = ES == 2 ? (key[r] & 0xffffu) : key[r];
                const uint32_t rk = ES == 2 ? (key[r] >> 16) : rank[ES == 2 ? 0 : r];
                const uint32_t d = digit_of<KT>(k, p.shift, p.descending);
                const uint32_t s = s_hist[warp][d] + rk;
                st_key[s] = (K)k;
                if constexpr (IDX_IN) st_idx[s] = ix[r];
                else st_idx[s] = (int32_t)(e - tg.row0);  // element (or, segmented, column) index
            }
        }
        __syncthreads();

        // 4. write out: consecutive staging slots of one digit are consecutive in global memory
        K* const ko = reinterpret_cast<K*>(p.keys_out);
        for (int s = tid; s < mt; s += kThreads) {
            const uint32_t k = st_key[s];
            const int64_t dest = s_gb[digit_of<KT>(k, p.shift, p.descending)] + s;
            ko[dest] = (K)k;
            p.idx_out[dest] = st_idx[s];
        }
        __syncthreads();
    }
}

// ---- TMA-ring variant: a producer warp streams key (and index) tiles into a
// shared-memory ring with cp.async.bulk so HBM latency is hidden by the ring
// depth; 16 compute warps rank, stage and write.  One CTA per SM.  Needs
// 16-byte aligned key / index buffers; the ragged last tile is read from
// global memory directly.
template <int ES, bool IDX_IN>
struct DigitTmaCfg {
    static constexpr int kKeyB = kTile * ES;
    static constexpr int kIdxB = IDX_IN ? kTile * 4 : 0;
    static constexpr int kSlot = kKeyB + kIdxB;
    static constexpr int kStage = kTile * (ES + 4);
    // shared memory per CTA: the first pass of 16-bit keys (no index input) may run RADIX_CTAS per SM
#ifdef RADIX_ALL_CTAS  // A/B build: every scatter variant at RADIX_ALL_CTAS CTAs per SM
    static constexpr bool kSmall = true;
    static constexpr int kCtas = RADIX_ALL_CTAS;
#else
    static constexpr bool kSmall = !IDX_IN && ES == 2;
    static constexpr int kCtas = kSmall ? RADIX_CTAS : 1;
#endif
    static constexpr int kBudget = kSmall ? RADIX_SMEM_KB * 1024 : 200 * 1024;
    static constexpr int kNB = (kBudget - kStage) / kSlot > 4 ? 4 : (kBudget - kStage) / kSlot;
    static constexpr size_t kSmem = (size_t)kNB * kSlot + kStage;
    static constexpr int kThreadsT = kThreads + 32;
};

template <int KT, int ES, bool IDX_IN>
__global__ void __launch_bounds__(kThreads + 32, DigitTmaCfg<ES, IDX_IN>::kCtas) k_digit_scatter_tma(const DigitParams p)
{
    using C = DigitTmaCfg<ES, IDX_IN>;
    constexpr int NB = C::kNB;
    static_assert(NB >= 2, "ring of at least two tiles");
    using K = typename std::conditional<ES == 2, uint16_t, uint32_t>::type;
#ifdef RADIX_HIST16  // A/B build: 16-bit per-warp counts (<= kRounds * 32 per warp) -- 8 KB less
    __shared__ uint16_t s_hist[kWarps][kDigits];
#else
    __shared__ uint32_t s_hist[kWarps][kDigits];
#endif
    __shared__ uint32_t s_tdp[kDigits];
    __shared__ int64_t s_gb[kDigits];
    __shared__ uint32_t s_wsum[kWarps];
    __shared__ uint32_t s_dbase[kDigits];
    __shared__ __align__(8) uint64_t full[NB], empty[NB];
    extern __shared__ __align__(16) uint8_t s_dyn[];
    uint8_t* const ring = s_dyn;
    K* const st_key = reinterpret_cast<K*>(s_dyn + NB * C::kSlot);
    int32_t* const st_idx = reinterpret_cast<int32_t*>(s_dyn + NB * C::kSlot + kTile * ES);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // a tile goes through the ring when it is whole and its bulk copies are 16-byte aligned
    auto ring_tile = [&](const TileGeom& tg) {
        return tg.mt == kTile && ((tg.t0 * ES) & 15) == 0 && (!IDX_IN || (tg.t0 & 3) == 0);
    };
    if (tid < kDigits) {  // digit bases (as in k_digit_scatter)
        // (segmented: the row scans already include the digit bases)
        const int64_t last = (int64_t)tid * p.ntiles + p.ntiles - 1;
        const uint32_t tot = p.cols > 0 ? 0u : p.offs[last] + p.counts[last];
        uint32_t incl = tot;
#pragma unroll
        for (int k = 1; k < 32; k <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, k);
            if (lane >= k) incl += y;
        }
        if (lane == 31) s_wsum[warp] = incl;
        s_dbase[tid] = incl - tot;
    }
    if (tid == 0) {
        for (int i = 0; i < NB; ++i) {
            ptx::mbar_init(&full[i], 1);
            ptx::mbar_init(&empty[i], kWarps);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    if (tid < kDigits) {
        uint32_t off = 0;
        for (int w = 0; w < warp; ++w) off += s_wsum[w];
        s_dbase[tid] += off;
    }
    __syncthreads();

    if (warp == kWarps) {
        // ============ producer ============
        if (lane == 0) {
            const uint64_t pol = ptx::policy_evict_first();
            int s = 0;
            uint32_t ph = 0;
            bool wrapped = false;
            for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
                if (wrapped) ptx::mbar_wait(&empty[s], ph ^ 1u);
                uint8_t* dst = ring + s * C::kSlot;
                const TileGeom tg = tile_geom(p, t);
                if (ring_tile(tg)) {
                    const int64_t t0 = tg.t0;
                    ptx::mbar_arrive_expect_tx(&full[s], (uint32_t)C::kSlot);
                    ptx::tma_load_1d(dst, reinterpret_cast<const uint8_t*>(p.keys_in) + t0 * ES, C::kKeyB, &full[s], pol);
                    if constexpr (IDX_IN) ptx::tma_load_1d(dst + C::kKeyB, p.idx_in + t0, C::kIdxB, &full[s], pol);
                } else {
                    ptx::mbar_arrive(&full[s]);
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
    const uint32_t lt_mask = (1u << lane) - 1u;
    int s = 0;
    uint32_t ph = 0;
    for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
        const TileGeom tg = tile_geom(p, t);
        const int64_t t0 = tg.t0;
        const int mt = tg.mt;
        const bool in_ring = ring_tile(tg);
        // this tile's (digit, tile) starts: issued now, consumed after the rank
        // rounds (a dependent L2 round trip per tile otherwise stalls the CTA)
        const uint32_t my_off = tid < kDigits ? __ldg(p.offs + tg.c0 + (int64_t)tid * tg.dstride) : 0u;
        for (int i = tid; i < kWarps * kDigits; i += kThreads) (&s_hist[0][0])[i] = 0;
        ptx::mbar_wait(&full[s], ph);
        const uint8_t* slot = ring + s * C::kSlot;
        const K* sk = reinterpret_cast<const K*>(slot);
        const int32_t* si = reinterpret_cast<const int32_t*>(slot + C::kKeyB);
        ptx::named_bar_sync(1, kThreads);  // s_hist zeroed

        const int l0 = warp * (kRounds * 32);   // tile-local index of this warp's first element
        // 4-byte keys: the in-digit ranks wait for the CTA prefix in shared
        // memory, each over its own element's key word in the ring slot (already
        // in a register; the thread that read it writes it) -- 16 rank registers
        // on top of 16 keys spilled at the 96 registers a 17-warp CTA can have.
        // 2-byte keys pack the rank beside the key.
        uint32_t* const s_rank = reinterpret_cast<uint32_t*>(const_cast<uint8_t*>(slot));
        uint32_t key[kRounds];
#pragma unroll
        for (int r = 0; r < kRounds; ++r) {
            const int li = l0 + r * 32 + lane;
            if (in_ring) key[r] = sk[li];
            else key[r] = li < mt ? load_key<KT, ES>(p.keys_in, t0 + li) : 0u;
        }
        // all 16 peer groups first (independent, long-latency MATCH), then the
        // running per-warp digit counts round by round
#pragma unroll
        for (int r = 0; r < kRounds; ++r) {
            const int li = l0 + r * 32 + lane;
            const bool ok = li < mt;
            const uint32_t d = digit_of<KT>(key[r], p.shift, p.descending);
            const uint32_t peers = digit_peers(d, ok);
            const uint32_t before = __popc(peers & lt_mask);
            uint32_t base = 0;
            if (ok) base = s_hist[warp][d];
            if constexpr (ES == 2) key[r] |= (base + before) << 16;
            else s_rank[li] = base + before;
            __syncwarp();
            if (ok && before == 0) s_hist[warp][d] = base + __popc(peers);
            __syncwarp();
        }
        ptx::named_bar_sync(1, kThreads);
        if (tid < kDigits) {
            uint32_t run = 0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                const uint32_t c = s_hist[w][tid];
                s_hist[w][tid] = run;
                run += c;
            }
            uint32_t incl = run;
#pragma unroll
            for (int dd = 1; dd < 32; dd <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, dd);
                if (lane >= dd) incl += y;
            }
            if (lane == 31) s_wsum[warp] = incl;
            s_tdp[tid] = incl - run;
        }
        ptx::named_bar_sync(1, kThreads);
        if (tid < kDigits) {
            uint32_t off = 0;
            for (int w = 0; w < warp; ++w) off += s_wsum[w];
            const uint32_t tdp = s_tdp[tid] + off;
            s_tdp[tid] = tdp;
            s_gb[tid] = tg.row0 + (int64_t)s_dbase[tid] + (int64_t)my_off - (int64_t)tdp;
            // one staging table: s_hist[w][d] becomes the tile-local start of (warp w,
            // digit d) -- one bank-conflicted shared load per staged element instead of
            // two (measured: row sort 19.89 -> 19.24 ms, fp16 sort 0.335 -> 0.329 ms)
#pragma unroll
            for (int w = 0; w < kWarps; ++w) s_hist[w][tid] += tdp;
        }
        ptx::named_bar_sync(1, kThreads);
#pragma unroll
        for (int r = 0; r < kRounds; ++r) {
            const int li = l0 + r * 32 + lane;
            if (li < mt) {
                const uint32_t k = ES == 2 ? (key[r] & 0xffffu) : key[r];
                const uint32_t rk = ES == 2 ? (key[r] >> 16) : s_rank[li];
                const uint32_t d = digit_of<KT>(k, p.shift, p.descending);
                const uint32_t st = s_hist[warp][d] + rk;
                st_key[st] = (K)k;
                if constexpr (IDX_IN) st_idx[st] = in_ring ? si[li] : p.idx_in[t0 + li];
                else st_idx[st] = (int32_t)(t0 + li - tg.row0);
            }
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&empty[s]);  // this warp is done with the slot
        if (++s == NB) {
            s = 0;
            ph ^= 1u;
        }
        ptx::named_bar_sync(1, kThreads);
        K* const ko = reinterpret_cast<K*>(p.keys_out);
        for (int q = tid; q < mt; q += kThreads) {
            const uint32_t k = st_key[q];
            const int64_t dest = s_gb[digit_of<KT>(k, p.shift, p.descending)] + q;
            ko[dest] = (K)k;
            p.idx_out[dest] = st_idx[q];
        }
        // the next tile's first named barrier orders these reads before its writes
    }
}

// dbase[d] = sum over digits d' < d of the digit totals; the total of digit d
// is its last row-scan entry plus its last tile count.
__global__ void __launch_bounds__(kDigits) k_digit_base(const uint32_t* counts, const uint32_t* offs, int ntiles,
                                                        uint32_t* dbase)
{
    __shared__ uint32_t s_w[kDigits / 32];
    const int d = threadIdx.x, lane = d & 31, warp = d >> 5;
    const int64_t last = (int64_t)d * ntiles + ntiles - 1;
    const uint32_t tot = offs[last] + counts[last];
    uint32_t incl = tot;
#pragma unroll
    for (int k = 1; k < 32; k <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, k);
        if (lane >= k) incl += y;
    }
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    uint32_t off = 0;
    for (int w = 0; w < warp; ++w) off += s_w[w];
    dbase[d] = off + incl - tot;
}

}  // namespace radix
}  // namespace scan

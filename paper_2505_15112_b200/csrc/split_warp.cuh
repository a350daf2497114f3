// split_warp.cuh -- warp-granular split / compress (PAPER Sec. 5.1-5.2,
// P281-285): the second-generation scatter for int8 flags and 1- or 2-byte
// payloads (the paper's SplitInd case: "an array of 16-bit elements and a 0/1
// mask array (flags are stored in int8)", P283).
//
// The block-level kernel (split.cuh) stages every tile in shared memory and
// spends ~34 instructions per element on it.  Here a WARP owns a contiguous
// "warp tile" of kWT elements and writes its outputs straight to global memory:
//   * count pass: true count per warp tile; every CTA owns a contiguous range of
//     warp tiles, scans its counts locally and publishes its total; the last
//     CTA scans the CTA totals (a two-level exclusive scan, no serial pass over
//     all tiles);
//   * scatter pass: per step a warp reads 128 consecutive elements (4 per lane:
//     one 4-byte flag word, one 8-/4-byte payload word), the in-step exclusive
//     scan of the mask is 4 ballots + popcounts (lanes own consecutive
//     elements, so the order of the run is lane-major); the step is staged in
//     output order in a 128-word per-warp buffer and written back by
//     consecutive lanes: trues to off + (trues before), falses to
//     T + (warp tile start - off) + (falses before) -- P283's offsets -- as
//     coalesced runs, no block-level barrier.
// HBM bytes per element as before (mask twice, payload once in and out,
// indices out); instructions per element ~8 instead of ~34.
#pragma once
#include <stdint.h>

#include "ptx.cuh"

namespace scan {
namespace splitw {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kWT = 4096;             // elements per warp tile
constexpr int kStep = 128;            // elements per warp step (4 per lane)
constexpr int kSteps = kWT / kStep;   // 32
constexpr int kAhead = 4;             // steps in flight per warp

struct WParams {
    const void* x;          // payload
    void* z;                // output
    const int8_t* flags;
    int32_t* idx_out;       // nullable
    int64_t* count_out;     // nullable, device: T
    uint32_t* counts;       // [nwt] true count per warp tile
    uint32_t* loff;         // [nwt] exclusive scan of counts within the owning CTA's range
    uint32_t* cta_tot;      // [grid] CTA totals, then (last CTA) their exclusive scan
    uint32_t* hdr;          // [0] done counter, [2..3] T
    int64_t n;
    int nwt;                // warp tiles
    int wpc;                // warp tiles per count CTA (contiguous)
    int compress;
};

__device__ __forceinline__ uint32_t nz_bits4(uint32_t f)
{
    // bit j = byte j of f is nonzero (R12)
    const uint32_t nz = __vcmpne4(f, 0u) & 0x80808080u;
    return (nz * 0x00204081u) >> 28;
}

// ---- count pass ------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_splitw_count(const WParams p)
{
    __shared__ uint32_t s_red[kWarps];
    __shared__ bool s_last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wt0 = blockIdx.x * p.wpc;
    const int wt1 = min(p.nwt, wt0 + p.wpc);
    for (int wt = wt0 + warp; wt < wt1; wt += kWarps) {
        const int64_t e0 = (int64_t)wt * kWT;
        uint32_t c = 0;
        if (e0 + kWT <= p.n) {
            const uint4* v = reinterpret_cast<const uint4*>(p.flags + e0);
            uint4 q[kWT / 512];
#pragma unroll
            for (int k = 0; k < kWT / 512; ++k) q[k] = ptx::ld_stream_v4(v + k * 32 + lane);
#pragma unroll
            for (int k = 0; k < kWT / 512; ++k)
                c += __popc(__vcmpne4(q[k].x, 0u) & 0x01010101u) + __popc(__vcmpne4(q[k].y, 0u) & 0x01010101u) +
                     __popc(__vcmpne4(q[k].z, 0u) & 0x01010101u) + __popc(__vcmpne4(q[k].w, 0u) & 0x01010101u);
        } else {
            for (int64_t e = e0 + lane; e < p.n; e += 32) c += p.flags[e] != 0 ? 1u : 0u;
        }
        c = __reduce_add_sync(0xffffffffu, c);
        if (lane == 0) p.counts[wt] = c;
    }
    __syncthreads();
    // CTA-local exclusive scan of this CTA's contiguous range of counts
    uint32_t carry = 0;
    for (int base = wt0; base < wt1; base += kThreads) {
        const int i = base + tid;
        const uint32_t x = i < wt1 ? p.counts[i] : 0u;
        uint32_t incl = x;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += y;
        }
        if (lane == 31) s_red[warp] = incl;
        __syncthreads();
        uint32_t wpre = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t y = s_red[w];
            if (w < warp) wpre += y;
            tot += y;
        }
        if (i < wt1) p.loff[i] = carry + wpre + incl - x;
        carry += tot;
        __syncthreads();
    }
    if (tid == 0) p.cta_tot[blockIdx.x] = carry;
    // last CTA: exclusive scan of the CTA totals
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = ptx::claim_add(&p.hdr[0], 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    uint64_t run = 0;
    for (int base = 0; base < (int)gridDim.x; base += kThreads) {
        const int i = base + tid;
        const uint32_t x = i < (int)gridDim.x ? __ldcg(&p.cta_tot[i]) : 0u;
        uint32_t incl = x;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += y;
        }
        if (lane == 31) s_red[warp] = incl;
        __syncthreads();
        uint32_t wpre = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t y = s_red[w];
            if (w < warp) wpre += y;
            tot += y;
        }
        __syncthreads();
        if (i < (int)gridDim.x) p.cta_tot[i] = (uint32_t)(run + wpre + incl - x);
        run += tot;
    }
    if (tid == 0) {
        reinterpret_cast<uint64_t*>(p.hdr)[1] = run;
        if (p.count_out) *p.count_out = (int64_t)run;
        p.hdr[0] = 0;
    }
}

// ---- scatter pass: a warp per warp tile, direct predicated stores -------------
template <int ES, bool CMP, bool IDX>
__global__ void __launch_bounds__(kThreads) k_splitw_scatter(const WParams p)
{
    using P = typename std::conditional<ES == 2, uint16_t, uint8_t>::type;
    using PV = typename std::conditional<ES == 2, uint2, uint32_t>::type;  // 4 payload elements
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * kThreads + threadIdx.x) >> 5;
    const int nw = (gridDim.x * kThreads) >> 5;
    const uint64_t T = reinterpret_cast<const uint64_t*>(p.hdr)[1];
    const uint32_t lt = (1u << lane) - 1u;
    P* const z = reinterpret_cast<P*>(p.z);
    __shared__ uint32_t s_wbuf[kWarps][kStep];
    uint32_t* const wbuf = s_wbuf[threadIdx.x >> 5];
    for (int wt = gw; wt < p.nwt; wt += nw) {
        const int64_t e0 = (int64_t)wt * kWT;
        const uint64_t off = (uint64_t)__ldg(&p.cta_tot[wt / p.wpc]) + __ldg(&p.loff[wt]);
        uint64_t tpos = off;                             // next true slot
        uint64_t fpos = T + (uint64_t)e0 - off;          // next false slot
        const bool full = e0 + kWT <= p.n;
        if (full) {
            const uint32_t* fw = reinterpret_cast<const uint32_t*>(p.flags + e0);
            const PV* pw = reinterpret_cast<const PV*>(reinterpret_cast<const P*>(p.x) + e0);
            uint32_t fq[kAhead];
            PV pq[kAhead];
#pragma unroll
            for (int a = 0; a < kAhead; ++a) {
                fq[a] = __ldcs(fw + a * 32 + lane);
                pq[a] = __ldcs(pw + a * 32 + lane);
            }
#pragma unroll 1
            for (int st = 0; st < kSteps; st += kAhead) {
#pragma unroll
                for (int a = 0; a < kAhead; ++a) {
                    const uint32_t f = fq[a];
                    const PV pv = pq[a];
                    const int nx = st + a + kAhead;  // prefetch the step kAhead ahead
                    if (nx < kSteps) {
                        fq[a] = __ldcs(fw + nx * 32 + lane);
                        pq[a] = __ldcs(pw + nx * 32 + lane);
                    }
                    const uint32_t bits = nz_bits4(f);
                    const uint32_t b0 = __ballot_sync(0xffffffffu, bits & 1u);
                    const uint32_t b1 = __ballot_sync(0xffffffffu, bits & 2u);
                    const uint32_t b2 = __ballot_sync(0xffffffffu, bits & 4u);
                    const uint32_t b3 = __ballot_sync(0xffffffffu, bits & 8u);
                    const uint32_t before = __popc(b0 & lt) + __popc(b1 & lt) + __popc(b2 & lt) + __popc(b3 & lt);
                    const uint32_t tot = __popc(b0) + __popc(b1) + __popc(b2) + __popc(b3);
                    uint32_t pw32[2];
                    if constexpr (ES == 2) { pw32[0] = pv.x; pw32[1] = pv.y; }
                    else { pw32[0] = pv; pw32[1] = 0; }
                    // stage the step in output order (trues, then falses) in this
                    // warp's 128-word buffer: (payload << 16) | element-in-step
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        uint32_t val;
                        if constexpr (ES == 2) val = (pw32[j >> 1] >> (16 * (j & 1))) & 0xffffu;
                        else val = (pw32[0] >> (8 * j)) & 0xffu;
                        const uint32_t tb = before + __popc(bits & ((1u << j) - 1u));  // trues before element j
                        const uint32_t slot = ((bits >> j) & 1u) ? tb : tot + (uint32_t)(4 * lane + j) - tb;
                        if (!CMP || ((bits >> j) & 1u)) wbuf[slot] = (val << 16) | (uint32_t)(4 * lane + j);
                    }
                    __syncwarp();
                    // write consecutive slots from consecutive lanes: coalesced runs
                    const int64_t sbase = e0 + (int64_t)(st + a) * kStep;
                    const int lim = CMP ? (int)tot : kStep;
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const int k = r * 32 + lane;
                        if (k < lim) {
                            const uint32_t w = wbuf[k];
                            const uint64_t d = k < (int)tot ? tpos + k : fpos + (uint64_t)(k - (int)tot);
                            z[d] = (P)(w >> 16);
                            if constexpr (IDX) p.idx_out[d] = (int32_t)(sbase + (w & 0xffffu));
                        }
                    }
                    __syncwarp();
                    tpos += tot;
                    fpos += kStep - tot;
                }
            }
        } else {
            // ragged last warp tile: element by element, same order
            for (int64_t s0 = e0; s0 < p.n; s0 += 32) {
                const int64_t e = s0 + lane;
                const bool ok = e < p.n;
                const bool tr = ok && p.flags[e] != 0;
                const P val = ok ? reinterpret_cast<const P*>(p.x)[e] : (P)0;
                const uint32_t bt = __ballot_sync(0xffffffffu, tr);
                const uint32_t bv = __ballot_sync(0xffffffffu, ok);
                if (tr) {
                    const uint64_t d = tpos + __popc(bt & lt);
                    z[d] = val;
                    if constexpr (IDX) p.idx_out[d] = (int32_t)e;
                } else if (ok && !CMP) {
                    const uint64_t d = fpos + __popc(bv & ~bt & lt);
                    z[d] = val;
                    if constexpr (IDX) p.idx_out[d] = (int32_t)e;
                }
                tpos += __popc(bt);
                fpos += __popc(bv & ~bt);
            }
        }
    }
}

// ---- staged split / compress: 16 elements per lane, runs written with 16-byte stores ----
// The scatter above stores every output element on its own (2-byte stores and
// their address arithmetic, ~45 instructions per 128 elements).  Here a warp
// takes 16 consecutive elements per lane per step (512 per warp: one 16-byte flag
// load, one or two 16-byte payload loads), forms the exclusive scan of the
// per-lane true counts with a shuffle scan, and packs trues (and, for split,
// falses -- a lane's falses before it are 16 * lane minus its trues before it)
// into private shared-memory runs whose starts are congruent to their global
// destinations modulo 16 bytes; every kSeg input elements the runs are written
// with aligned 16-byte stores (element stores only for a run's first and last
// partial vectors).  Indices (SplitInd, P283) are staged and written the same way.
#ifndef SPLIT_IDX_SEG
#define SPLIT_IDX_SEG 512
#endif
template <bool CMP, bool IDX>
constexpr int staged_seg() { return CMP && !IDX ? 2048 : (!CMP && IDX ? SPLIT_IDX_SEG : 1024); }
constexpr int kRunPad = 32;  // >= 2 x (elements per 16-byte vector) for any payload / index run
// per warp: the payload run(s), then the index run(s) as 16-bit positions in the warp tile
template <int ES, bool CMP, bool IDX, int NT = kThreads>
constexpr size_t staged_smem_bytes()
{
    return (size_t)(NT / 32) * (CMP ? 1 : 2) * (staged_seg<CMP, IDX>() + kRunPad) * (ES + (IDX ? 2 : 0));
}

// run[shift, shift + cnt) of 16-bit warp-tile positions -> g_aligned[k] = base + run[k]
// (int32 indices), 16-byte stores of 4 indices; shift is the payload's (a multiple of 4
// keeps g_aligned 16-byte aligned)
__device__ __forceinline__ void write_idx_run(int32_t* __restrict__ g_aligned, const uint16_t* __restrict__ run,
                                              int shift, int cnt, int32_t base, int lane)
{
    const int nvec = (shift + cnt + 3) / 4;
    for (int v = lane; v < nvec; v += 32) {
        const int lo = v * 4, hi = lo + 4;
        if (lo >= shift && hi <= shift + cnt) {
            const uint2 w = *reinterpret_cast<const uint2*>(run + lo);
            int4 o;
            o.x = base + (int32_t)(w.x & 0xffffu);
            o.y = base + (int32_t)(w.x >> 16);
            o.z = base + (int32_t)(w.y & 0xffffu);
            o.w = base + (int32_t)(w.y >> 16);
            *reinterpret_cast<int4*>(g_aligned + lo) = o;
        } else {
            const int a0 = lo > shift ? lo : shift, a1 = hi < shift + cnt ? hi : shift + cnt;
            for (int k = a0; k < a1; ++k) g_aligned[k] = base + (int32_t)run[k];
        }
    }
}

template <typename T, int SHIFT_MOD>
__device__ __forceinline__ void write_run(T* __restrict__ g_aligned, const T* __restrict__ run, int shift, int cnt,
                                          int lane)
{
    // run[shift, shift + cnt) -> g_aligned[shift, shift + cnt); g_aligned and run
    // are 16-byte aligned, shift < SHIFT_MOD (a multiple of the vector length)
    constexpr int kVecE = 16 / (int)sizeof(T);
    const int nvec = (shift + cnt + kVecE - 1) / kVecE;
    for (int v = lane; v < nvec; v += 32) {
        const int lo = v * kVecE, hi = lo + kVecE;
        if (lo >= shift && hi <= shift + cnt) {
            *reinterpret_cast<uint4*>(g_aligned + lo) = *reinterpret_cast<const uint4*>(run + lo);
        } else {
            const int a0 = lo > shift ? lo : shift, a1 = hi < shift + cnt ? hi : shift + cnt;
            for (int k = a0; k < a1; ++k) g_aligned[k] = run[k];
        }
    }
}

template <int ES, bool CMP, bool IDX, int NT = kThreads>
__global__ void __launch_bounds__(NT, 1024 / NT) k_splitw_staged(const WParams p)
{
    using P = typename std::conditional<ES == 2, uint16_t, uint8_t>::type;
    constexpr int kSegE = staged_seg<CMP, IDX>();
    constexpr int kRun = kSegE + kRunPad;         // elements per staged run buffer
    constexpr int kMod = 16 / ES;                 // run starts congruent modulo this many elements
    static_assert(kMod % 4 == 0, "index runs (4-byte) stay 16-byte aligned under the payload's shift");
    constexpr int kS16 = 512;                     // elements per warp step
    constexpr int kPW = ES;                       // 16-byte payload vectors per lane per step
    constexpr int kSegSteps = kSegE / kS16;
    constexpr int kTileSteps = kWT / kS16;
    constexpr int kAh = 2;                        // steps in flight (runs may be shorter: written mid-loop)
    static_assert(kTileSteps % kSegSteps == 0 && kTileSteps % kAh == 0, "whole runs and prefetch groups per tile");
    extern __shared__ __align__(16) uint8_t s_raw[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int gw = (blockIdx.x * NT + threadIdx.x) >> 5;
    const int nw = (gridDim.x * NT) >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const uint64_t T = reinterpret_cast<const uint64_t*>(p.hdr)[1];
    P* const z = reinterpret_cast<P*>(p.z);
    // per-warp runs: payload [true run][false run], then indices [true run][false run]
    constexpr int kRuns = CMP ? 1 : 2;
    uint8_t* const wbase = s_raw + (size_t)warp * kRuns * kRun * (ES + (IDX ? 2 : 0));
    P* const runT = reinterpret_cast<P*>(wbase);
    P* const runF = runT + kRun;
    uint16_t* const runTi = reinterpret_cast<uint16_t*>(wbase + (size_t)kRuns * kRun * ES);  // positions in the tile
    uint16_t* const runFi = runTi + kRun;
    for (int wt = gw; wt < p.nwt; wt += nw) {
        const int64_t e0 = (int64_t)wt * kWT;
        const uint64_t off = (uint64_t)__ldg(&p.cta_tot[wt / p.wpc]) + __ldg(&p.loff[wt]);
        uint64_t tpos = off;                     // next true slot
        uint64_t fpos = T + (uint64_t)e0 - off;  // next false slot
        if (e0 + kWT <= p.n) {
            const uint4* fw = reinterpret_cast<const uint4*>(p.flags + e0);
            const uint4* pw = reinterpret_cast<const uint4*>(reinterpret_cast<const P*>(p.x) + e0);
            uint4 fq[kAh], pq[kAh][kPW];
#pragma unroll
            for (int a = 0; a < kAh; ++a) {
                fq[a] = __ldcs(fw + a * 32 + lane);
#pragma unroll
                for (int v = 0; v < kPW; ++v) pq[a][v] = __ldcs(pw + (a * 32 + lane) * kPW + v);
            }
            int shT = (int)(tpos % kMod), shF = (int)(fpos % kMod);
            int cT = 0, sdone = 0;  // trues / elements of the current run so far
#pragma unroll 1
            for (int st0 = 0; st0 < kTileSteps; st0 += kAh) {
#pragma unroll
                for (int a = 0; a < kAh; ++a) {
                    const int st = st0 + a;
                    const uint4 f = fq[a];
                    uint32_t w[4 * kPW];
#pragma unroll
                    for (int v = 0; v < kPW; ++v) {
                        w[4 * v] = pq[a][v].x; w[4 * v + 1] = pq[a][v].y;
                        w[4 * v + 2] = pq[a][v].z; w[4 * v + 3] = pq[a][v].w;
                    }
                    const int nx = st + kAh;
                    if (nx < kTileSteps) {
                        fq[a] = __ldcs(fw + nx * 32 + lane);
#pragma unroll
                        for (int v = 0; v < kPW; ++v) pq[a][v] = __ldcs(pw + (nx * 32 + lane) * kPW + v);
                    }
                    const uint32_t bits = nz_bits4(f.x) | (nz_bits4(f.y) << 4) | (nz_bits4(f.z) << 8) |
                                          (nz_bits4(f.w) << 12);
                    const int c = __popc(bits);
                    int incl = c;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const int y = __shfl_up_sync(0xffffffffu, incl, d);
                        if (lane >= d) incl += y;
                    }
                    const int ex = incl - c;                               // trues before this lane in the step
                    const int tb = shT + cT + ex;                          // this lane's first true slot
                    const int fb = shF + (sdone - cT) + (16 * lane - ex);  // ... first false slot
                    const int i0 = st * kS16 + 16 * lane;                  // position in the warp tile
                    int kt = 0, kf = 0;
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        P v;
                        if constexpr (ES == 2) v = (P)(w[j >> 1] >> (16 * (j & 1)));
                        else v = (P)(w[j >> 2] >> (8 * (j & 3)));
                        if ((bits >> j) & 1u) {
                            runT[tb + kt] = v;
                            if constexpr (IDX) runTi[tb + kt] = (uint16_t)(i0 + j);
                            ++kt;
                        } else if constexpr (!CMP) {
                            runF[fb + kf] = v;
                            if constexpr (IDX) runFi[fb + kf] = (uint16_t)(i0 + j);
                            ++kf;
                        }
                    }
                    cT += __shfl_sync(0xffffffffu, incl, 31);
                    sdone += kS16;
                    if (sdone == kSegE) {  // the run is complete: write it, start the next
                        __syncwarp();
                        write_run<P, kMod>(z + (tpos - (uint64_t)shT), runT, shT, cT, lane);
                        if constexpr (IDX)
                            write_idx_run(p.idx_out + (tpos - (uint64_t)shT), runTi, shT, cT, (int32_t)e0, lane);
                        if constexpr (!CMP) {
                            const int cF = kSegE - cT;
                            write_run<P, kMod>(z + (fpos - (uint64_t)shF), runF, shF, cF, lane);
                            if constexpr (IDX)
                                write_idx_run(p.idx_out + (fpos - (uint64_t)shF), runFi, shF, cF, (int32_t)e0, lane);
                            fpos += (uint64_t)cF;
                        }
                        __syncwarp();
                        tpos += (uint64_t)cT;
                        shT = (int)(tpos % kMod);
                        shF = (int)(fpos % kMod);
                        cT = 0;
                        sdone = 0;
                    }
                }
            }
        } else {
            // ragged last warp tile: element by element, same order
            for (int64_t s0 = e0; s0 < p.n; s0 += 32) {
                const int64_t e = s0 + lane;
                const bool ok = e < p.n;
                const bool tr = ok && p.flags[e] != 0;
                const P val = ok ? reinterpret_cast<const P*>(p.x)[e] : (P)0;
                const uint32_t bt = __ballot_sync(0xffffffffu, tr);
                const uint32_t bv = __ballot_sync(0xffffffffu, ok);
                if (tr) {
                    const uint64_t d = tpos + __popc(bt & lt);
                    z[d] = val;
                    if constexpr (IDX) p.idx_out[d] = (int32_t)e;
                } else if (ok && !CMP) {
                    const uint64_t d = fpos + __popc(bv & ~bt & lt);
                    z[d] = val;
                    if constexpr (IDX) p.idx_out[d] = (int32_t)e;
                }
                tpos += __popc(bt);
                fpos += __popc(bv & ~bt);
            }
        }
    }
}

// ---- single-pass compress (decoupled look-back over warp tiles) ----------------
// The two-pass compress reads the mask twice (5 B/element for 4 algorithmic:
// ceiling 80 %, reached).  Here ONE pass: a warp claims the next 2048-element
// warp tile by ticket (tiles start in order), loads its flags and payload into
// registers, counts its trues, publishes the count (flag A) and looks back over
// its predecessors' descriptors -- 32 at a time, summing aggregates back to the
// nearest inclusive prefix (flag P) -- the decoupled look-back the paper cites
// as the single-pass state of the art (P78-81); then it publishes its own
// inclusive prefix, packs its trues into a shared-memory run aligned to the
// destination (as k_splitw_staged) and writes it with 16-byte stores.  The
// descriptor is one 64-bit word {flag:2 | value:62} (single-copy atomic: no
// fences); the launcher zeroes the descriptors and the ticket on the stream.
// Measured 2.2x SLOWER than the two passes (1.87 vs 0.86 ms at 2^30): with
// ~3,500 warp tiles in flight the nearest published inclusive prefix is
// typically thousands of tiles back, ~100 look-back windows of one L2 round
// trip each -- the look-back distance grows with the concurrency B200 needs to
// fill HBM.  Kept as an A/B (SCAN_COMPRESS_SP=1).
constexpr int kSpWT = 2048;        // elements per warp tile
constexpr int kSpSteps = kSpWT / 512;
constexpr int kSpThreads = 256;
constexpr uint64_t kSpA = 1ull << 62, kSpP = 2ull << 62, kSpVal = (1ull << 62) - 1;
template <int ES>
constexpr size_t compress_sp_smem_bytes() { return (size_t)(kSpThreads / 32) * (kSpWT + 32) * ES; }

template <int ES>
__global__ void __launch_bounds__(kSpThreads, 3) k_compress_sp(const WParams p, uint64_t* desc, unsigned* ticket)
{
    using P = typename std::conditional<ES == 2, uint16_t, uint8_t>::type;
    constexpr int kMod = 16 / ES;  // elements per 16-byte vector
    constexpr int kPW = ES;        // 16-byte payload vectors per lane per 512-element step
    extern __shared__ __align__(16) uint8_t s_raw[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    P* const z = reinterpret_cast<P*>(p.z);
    P* const buf = reinterpret_cast<P*>(s_raw) + warp * (kSpWT + 32);
    const int nwt = (int)((p.n + kSpWT - 1) / kSpWT);
    for (;;) {
        int wt = 0;
        if (lane == 0) wt = (int)ptx::claim_add(ticket, 1u);
        wt = __shfl_sync(0xffffffffu, wt, 0);
        if (wt >= nwt) break;
        const int64_t e0 = (int64_t)wt * kSpWT;
        const bool full = e0 + kSpWT <= p.n;
        uint32_t bits[kSpSteps];
        uint4 pq[kSpSteps][kPW];
        int tot = 0;
        if (full) {
            const uint4* fw = reinterpret_cast<const uint4*>(p.flags + e0);
            const uint4* pw = reinterpret_cast<const uint4*>(reinterpret_cast<const P*>(p.x) + e0);
            uint4 fq[kSpSteps];
#pragma unroll
            for (int k = 0; k < kSpSteps; ++k) {
                fq[k] = __ldcs(fw + k * 32 + lane);
#pragma unroll
                for (int v = 0; v < kPW; ++v) pq[k][v] = __ldcs(pw + (k * 32 + lane) * kPW + v);
            }
            int c = 0;
#pragma unroll
            for (int k = 0; k < kSpSteps; ++k) {
                bits[k] = nz_bits4(fq[k].x) | (nz_bits4(fq[k].y) << 4) | (nz_bits4(fq[k].z) << 8) |
                          (nz_bits4(fq[k].w) << 12);
                c += __popc(bits[k]);
            }
            tot = (int)__reduce_add_sync(0xffffffffu, (unsigned)c);
        } else {
            for (int64_t e = e0 + lane; e < e0 + 32 * ((p.n - e0 + 31) / 32); e += 32)
                tot += __popc(__ballot_sync(0xffffffffu, e < p.n && p.flags[e] != 0));
        }
        // publish, look back, publish the inclusive prefix
        uint64_t excl = 0;
        if (wt == 0) {
            if (lane == 0) ptx::st_relaxed_u64(desc, kSpP | (uint64_t)tot);
        } else {
            if (lane == 0) ptx::st_relaxed_u64(desc + wt, kSpA | (uint64_t)tot);
            int64_t top = wt - 1;
            uint32_t backoff = 16;
            for (;;) {
                const int64_t idx = top - lane;
                const uint64_t d = idx >= 0 ? ptx::ld_relaxed_u64(desc + idx) : kSpP;  // before tile 0: prefix 0
                if (__any_sync(0xffffffffu, (d >> 62) == 0)) {  // a predecessor has not published yet
                    __nanosleep(backoff);
                    backoff = backoff < 256 ? backoff * 2 : 256;
                    continue;
                }
                const uint32_t pm = __ballot_sync(0xffffffffu, (d >> 62) == 2);
                const int pl = pm ? __ffs(pm) - 1 : 32;  // the nearest inclusive prefix
                uint64_t v = lane <= pl ? (d & kSpVal) : 0ull;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                excl += v;
                if (pm) break;
                top -= 32;
            }
            if (lane == 0) ptx::st_relaxed_u64(desc + wt, kSpP | (excl + (uint64_t)tot));
        }
        if (wt == nwt - 1 && lane == 0) {
            reinterpret_cast<uint64_t*>(p.hdr)[1] = excl + (uint64_t)tot;
            if (p.count_out) *p.count_out = (int64_t)(excl + (uint64_t)tot);
        }
        uint64_t tpos = excl;
        if (full) {
            const int shift = (int)(tpos % kMod);
            int cT = 0;
#pragma unroll
            for (int k = 0; k < kSpSteps; ++k) {
                const int c = __popc(bits[k]);
                int incl = c;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, d);
                    if (lane >= d) incl += y;
                }
                uint32_t w[4 * kPW];
#pragma unroll
                for (int v = 0; v < kPW; ++v) {
                    w[4 * v] = pq[k][v].x; w[4 * v + 1] = pq[k][v].y;
                    w[4 * v + 2] = pq[k][v].z; w[4 * v + 3] = pq[k][v].w;
                }
                P* const dst = buf + shift + cT + (incl - c);
                int kk = 0;
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    if ((bits[k] >> j) & 1u) {
                        if constexpr (ES == 2) dst[kk] = (P)(w[j >> 1] >> (16 * (j & 1)));
                        else dst[kk] = (P)(w[j >> 2] >> (8 * (j & 3)));
                        ++kk;
                    }
                }
                cT += __shfl_sync(0xffffffffu, incl, 31);
            }
            __syncwarp();
            write_run<P, kMod>(z + (tpos - (uint64_t)shift), buf, shift, cT, lane);
            __syncwarp();
        } else {
            for (int64_t s0 = e0; s0 < p.n; s0 += 32) {
                const int64_t e = s0 + lane;
                const bool tr = e < p.n && p.flags[e] != 0;
                const uint32_t bt = __ballot_sync(0xffffffffu, tr);
                if (tr) z[tpos + __popc(bt & lt)] = reinterpret_cast<const P*>(p.x)[e];
                tpos += __popc(bt);
            }
        }
    }
}

}  // namespace splitw
}  // namespace scan

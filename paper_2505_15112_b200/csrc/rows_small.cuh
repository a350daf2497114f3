// rows_small.cuh -- batched scan of SHORT rows (P437, App. B.1; SURVEY 8(a)
// row a6: "short rows use warp-per-row"), for sm_100a.
//
// A CTA-per-tile kernel spends 512 threads on a row of 32 elements; here:
//   * cols <= 32: one warp scans 32 / G rows at once, G = next power of two >=
//     cols, one element per lane, a SEGMENTED shuffle scan (`__shfl_up_sync`
//     with width G) -- rows never mix;
//   * 32 < cols <= kMaxCols: one warp per row, segments of 128 elements (4
//     consecutive per lane: sequential prefix, warp shuffle scan of the lane
//     totals, running row carry -- fp64 for float rows, as everywhere).
// Loads / stores are element-wise but warp-contiguous (coalesced); rows may be
// strided.  Floats: fp32 inside a segment, fp64 carry, one fp32 rounding of
// the base per segment (same accuracy contract as the other kernels).
#pragma once
#include <stdint.h>

#include "scan_kernels.cuh"

namespace scan {
namespace rows_small {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int64_t kMaxCols = 8192;

struct SRParams {
    const void* in;
    void* out;
    int64_t rows;
    int64_t cols;
    int64_t in_stride;   // elements
    int64_t out_stride;  // elements
    int exclusive;
};

#ifndef ROWS_TINY_U
#define ROWS_TINY_U 8
#endif
constexpr int kTinyU = ROWS_TINY_U;

template <int DT>
__global__ void __launch_bounds__(kThreads) k_rows_tiny(const SRParams p)
{
    using Tr = Traits<DT>;
    using In = typename Tr::In;
    using Out = typename Tr::Out;
    using Acc = typename Tr::Acc;
    const int lane = threadIdx.x & 31;
    int G = 1;
    while (G < p.cols) G <<= 1;             // lanes per row (power of two, <= 32)
    const int rpw = 32 / G;                 // rows per warp
    const int sub = lane / G, pos = lane % G;
    const int64_t gw = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * kThreads) >> 5;
    const In* in = reinterpret_cast<const In*>(p.in);
    Out* out = reinterpret_cast<Out*>(p.out);
    // kTinyU row groups per warp step: their loads are issued together and their
    // shuffle scans interleave (one load in flight per lane was latency-bound).
    // Measured (strided fp32 / int32 rows of 8-32 columns, same box): U = 1 33-35 %,
    // 4 41-42 %, 8 45-46 % of the copy peak on algorithmic bytes
    constexpr int U = kTinyU;
    for (int64_t r0 = gw * rpw * U; r0 < p.rows; r0 += nw * rpw * U) {
        bool ok[U];
        Acc incl[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t row = r0 + (int64_t)u * rpw + sub;
            ok[u] = row < p.rows && pos < p.cols;
            incl[u] = ok[u] ? widen(in[row * p.in_stride + pos]) : Acc(0);
        }
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const Acc y = __shfl_up_sync(0xffffffffu, incl[u], d, G);
                if (d < G && pos >= d) incl[u] = incl[u] + y;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const Acc e = __shfl_up_sync(0xffffffffu, incl[u], 1, G);  // every lane: the warp stays converged
            if (ok[u]) {
                const int64_t row = r0 + (int64_t)u * rpw + sub;
                const Acc v = p.exclusive ? (pos == 0 ? Acc(0) : e) : incl[u];
                out[row * p.out_stride + pos] = narrow(v, (Out*)nullptr);
            }
        }
    }
}

// Contiguous tiny rows (in_stride == out_stride == cols <= 32, 16-byte aligned
// bases): a tile of kThreads rows = kThreads * cols consecutive elements is
// staged through shared memory with 16-byte loads / stores, and thread t scans
// row t sequentially in the Carry type (fp64 for float rows: exact for <= 32
// terms, one rounding on the store).  Per element: ~4 instructions instead of
// the ~20 of the shuffle kernel, which is issue-bound.  Shared index i is padded
// to i + i/32, so the row-strided accesses of the scan phase spread over banks.
constexpr int kTileMaxCols = 32;
constexpr int kTileWords = kThreads * kTileMaxCols;
__device__ __forceinline__ int pad32(int i) { return i + (i >> 5); }

// STRIDED: rows at any 16-byte-multiple stride (in and out), cols a multiple of
// 16 / sizeof(In) and of 4.  The tile's vector q is vector q % V of its row q / V
// (V vectors per row), so the staged layout -- and the scan phase -- are the same
// as for contiguous rows; a warp's loads cover whole 16-byte-aligned row pieces.
template <int DT, bool STRIDED = false>
__global__ void __launch_bounds__(kThreads) k_rows_tile(const SRParams p)
{
    using Tr = Traits<DT>;
    using In = typename Tr::In;
    using Out = typename Tr::Out;
    using Acc = typename Tr::Acc;
    using Carry = typename Tr::Carry;
    constexpr int kEs = (int)sizeof(In);
    constexpr int kPerVec = 16 / kEs;                       // input elements per 16-byte load
    __shared__ __align__(16) Acc s_v[kTileWords + kTileWords / 32];
    const int tid = threadIdx.x;
    const int cols = (int)p.cols;
    const int64_t total = p.rows * p.cols;
    const int64_t tile_elems = (int64_t)kThreads * cols;
    const int64_t tiles = (p.rows + kThreads - 1) / kThreads;
    const In* in = reinterpret_cast<const In*>(p.in);
    Out* out = reinterpret_cast<Out*>(p.out);
    // the next tile's 16-byte loads are issued into registers before this tile is
    // scanned and stored (a thread holds at most kVPT vectors of a tile)
    constexpr int kVPT = kTileMaxCols * kEs / 16;
    uint4 pf[kVPT];
    const int vin = cols / kPerVec, vout = cols / 4;  // STRIDED: vectors per row in / out
    auto prefetch = [&](int64_t tt) {
        const int64_t g0 = tt * tile_elems;
        const int nv = tt < tiles ? (int)(min(tile_elems, total - g0) / kPerVec) : 0;
#pragma unroll
        for (int v = 0; v < kVPT; ++v) {
            const int q = tid + v * kThreads;
            if constexpr (STRIDED) {
                const int r = q / vin;
                const In* src = in + (tt * kThreads + r) * p.in_stride + (q - r * vin) * kPerVec;
                pf[v] = q < nv ? __ldg(reinterpret_cast<const uint4*>(src)) : make_uint4(0u, 0u, 0u, 0u);
            } else {
                pf[v] = q < nv ? __ldg(reinterpret_cast<const uint4*>(in + g0) + q) : make_uint4(0u, 0u, 0u, 0u);
            }
        }
    };
    prefetch(blockIdx.x);
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int64_t f0 = t * tile_elems;                   // multiple of 16 bytes (kThreads * cols * ES)
        const int ne = (int)min(tile_elems, total - f0);
        // 1. stage: the prefetched vectors, widened into padded shared memory
        const int nvec = ne / kPerVec;
#pragma unroll
        for (int v = 0; v < kVPT; ++v) {
            const int q = tid + v * kThreads;
            if (q < nvec) {
                const In* e = reinterpret_cast<const In*>(&pf[v]);
#pragma unroll
                for (int j = 0; j < kPerVec; ++j) s_v[pad32(q * kPerVec + j)] = widen(e[j]);
            }
        }
        if constexpr (!STRIDED)  // (STRIDED: whole vectors only)
            for (int i = nvec * kPerVec + tid; i < ne; i += kThreads) s_v[pad32(i)] = widen(in[f0 + i]);
        __syncthreads();
        prefetch(t + gridDim.x);
        // 2. thread tid scans row tid of the tile, in place
        if (tid * cols < ne) {
            Carry c = Carry(0);
            for (int j = 0; j < cols; ++j) {
                const int k = pad32(tid * cols + j);
                const Acc x = s_v[k];
                if (p.exclusive) {
                    s_v[k] = Acc(c);
                    c = c + Carry(x);
                } else {
                    c = c + Carry(x);
                    s_v[k] = Acc(c);
                }
            }
        }
        __syncthreads();
        // 3. 16-byte stores (Out is 4 bytes for every dtype)
        const int nvo = ne / 4;
        for (int q = tid; q < nvo; q += kThreads) {
            uint4 w;
            Out* e = reinterpret_cast<Out*>(&w);
#pragma unroll
            for (int j = 0; j < 4; ++j) e[j] = narrow(s_v[pad32(q * 4 + j)], (Out*)nullptr);
            if constexpr (STRIDED) {
                const int r = q / vout;
                *reinterpret_cast<uint4*>(out + (t * kThreads + r) * p.out_stride + (q - r * vout) * 4) = w;
            } else {
                reinterpret_cast<uint4*>(out + f0)[q] = w;
            }
        }
        if constexpr (!STRIDED)
            for (int i = nvo * 4 + tid; i < ne; i += kThreads) out[f0 + i] = narrow(s_v[pad32(i)], (Out*)nullptr);
        __syncthreads();
    }
}

template <int DT>
__global__ void __launch_bounds__(kThreads) k_rows_warp(const SRParams p)
{
    using Tr = Traits<DT>;
    using In = typename Tr::In;
    using Out = typename Tr::Out;
    using Acc = typename Tr::Acc;
    using Carry = typename Tr::Carry;
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * kThreads) >> 5;
    const In* in = reinterpret_cast<const In*>(p.in);
    Out* out = reinterpret_cast<Out*>(p.out);
    for (int64_t row = gw; row < p.rows; row += nw) {
        const In* ri = in + row * p.in_stride;
        Out* ro = out + row * p.out_stride;
        Carry carry = Carry(0);
        for (int64_t s0 = 0; s0 < p.cols; s0 += 128) {
            const int64_t e0 = s0 + 4 * lane;
            Acc v[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = e0 + j < p.cols ? widen(ri[e0 + j]) : Acc(0);
            Acc l[4];
            l[0] = v[0];
#pragma unroll
            for (int j = 1; j < 4; ++j) l[j] = l[j - 1] + v[j];
            const Acc incl = warp_incl_scan(l[3], lane);
            const Acc ex = __shfl_up_sync(0xffffffffu, incl, 1);
            const Acc lane_pre = lane == 0 ? Acc(0) : ex;
            const Acc seg_tot = __shfl_sync(0xffffffffu, incl, 31);
            Acc B;
            if constexpr (Tr::kFloat) B = (float)(carry + (double)lane_pre);
            else B = carry + lane_pre;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (e0 + j < p.cols) {
                    const Acc o = p.exclusive ? (j == 0 ? B : B + l[j - 1]) : B + l[j];
                    ro[e0 + j] = narrow(o, (Out*)nullptr);
                }
            }
            carry = carry + Carry(seg_tot);
        }
    }
}

}  // namespace rows_small
}  // namespace scan

// topp.cuh -- top-p (nucleus) sampling without a full row sort (PAPER Sec.
// 5.5, P298-299).
//
// The paper's top-p is "sort and scan on the token probability vector"
// (P299): sort the row descending, scan it, keep the smallest prefix whose
// mass reaches p, draw from it.  Only the TOP of the order matters: the
// nucleus is a prefix of the descending order, so it lies inside any set
// {tokens with probability >= tau} whose mass reaches p.  One CTA per row:
//   1. ONE read of the row: its maximum m and a candidate superset (every q
//      within ~2^-13.25 of the running maximum, seeded from the row's first
//      2048 elements), then per eighth-octave LEVEL l = (bits(m) - bits(q)) >> 20
//      (monotone in q) the exact mass (u64 fixed point) and count, and the first level L
//      whose cumulative mass reaches p.  Levels < L lie wholly inside the
//      nucleus; the nucleus ends inside level L.
//   2. Only level L is sorted (by q descending, index ascending -- the stable
//      descending order of the full sort; 64-bit keys, P287's code, ~index),
//      K = (count of levels < L) + 1 + min{ j : C_<L + C_L,j >= p }, then
//      t = u * C_{K-1}; the draw's level l* is the first whose cumulative
//      mass exceeds t, and only l* is sorted to find rank = min{ k : C_k > t }.
//      Every C is an exact fp64 sum (at most 8192 fp32 terms within 2^14 of
//      each other: 51 significant bits), so any summation order gives the
//      oracle's left-to-right values bit for bit (R15).
//   3. Fallbacks: a level above kLevCap elements sorts all candidates; a
//      superset overflow or a short mass re-reads the row with candidates
//      {q >= tau}, tau = m * 2^-s, s = 8, 12, ... (then sort + scan of all).
// A row whose candidate set would exceed kCap before reaching mass p is not
// handled here: token_out = -1 and the caller falls back to the sort path.
#pragma once
#include <stdint.h>

namespace scan {
namespace topp {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kCap = 8192;       // candidates per row (64 KB of 64-bit keys)
#ifndef TOPP_UNROLL
#define TOPP_UNROLL 4
#endif
constexpr int kLvlShift = 20;    // level = (bits(m) - bits(q)) >> 20: eighth octaves
constexpr int kLevels = 106;     // levels of the one-pass candidate superset (13.25 octaves)
constexpr int kLevels2 = 96;     // the third attempt's window (12 octaves) after two overflows
constexpr int kLevCap = 2048;    // keys of one level sorted on their own
constexpr size_t kSmemBytes = (size_t)(kCap + kLevCap) * 8;

__device__ __forceinline__ double key_val(unsigned long long k)
{
    return (double)__uint_as_float((uint32_t)(k >> 32) & 0x7fffffffu);
}

// Rank sort of keys[0, n) descending for n <= kLevCap / 2 (keys are distinct:
// the index is part of the key): rank_i = #{ j : key_j > key_i }, computed by
// every thread for its elements against all n (broadcast shared reads), the keys
// placed at their ranks in tmp and copied back -- two barriers instead of the
// bitonic network's log^2 n.
__device__ void block_rank_sort_desc(unsigned long long* keys, int n, unsigned long long* tmp)
{
    const int tid = threadIdx.x;
    for (int i = tid; i < n; i += kThreads) {
        const unsigned long long ki = keys[i];
        int r = 0;
        for (int j = 0; j < n; ++j) r += keys[j] > ki ? 1 : 0;
        tmp[r] = ki;
    }
    __syncthreads();
    for (int i = tid; i < n; i += kThreads) keys[i] = tmp[i];
    __syncthreads();
}

// Bitonic sort of keys[0, n) descending (padded with 0 keys to a power of two).
__device__ void block_sort_desc(unsigned long long* keys, int n)
{
    const int tid = threadIdx.x;
    int N = 1;
    while (N < n) N <<= 1;
    for (int i = n + tid; i < N; i += kThreads) keys[i] = 0ull;
    __syncthreads();
    for (int k = 2; k <= N; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = tid; i < N; i += kThreads) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const unsigned long long a = keys[i], b = keys[ixj];
                    const bool desc = (i & k) == 0;
                    if (desc ? (a < b) : (a > b)) {
                        keys[i] = b;
                        keys[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
}

// First j in [0, n) with base + (sum of keys[0..j]) >= thr (STRICT: > thr), n if
// none; *s_c = that prefix (valid when j < n).  Block-wide, contiguous chunks
// per thread + fp64 block scan.
template <bool STRICT>
__device__ int block_first_crossing(const unsigned long long* keys, int n, double base, double thr, double* s_dred,
                                    unsigned long long* s_min, double* s_c)
{
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = (n + kThreads - 1) / kThreads;
    const int lo = tid * per, hi = min(n, lo + per);
    double run = 0.0;
    for (int i = lo; i < hi; ++i) run += key_val(keys[i]);
    double incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    double ex = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) ex = 0.0;
    __syncthreads();  // s_dred / s_min are free
    if (lane == 31) s_dred[warp] = incl;
    if (tid == 0) *s_min = (unsigned long long)n;
    __syncthreads();
    double wpre = 0.0;
    for (int w = 0; w < warp; ++w) wpre += s_dred[w];
    const double before = base + wpre + ex;
    double c = before;
    for (int i = lo; i < hi; ++i) {
        c += key_val(keys[i]);
        if (STRICT ? c > thr : c >= thr) {
            atomicMin(s_min, (unsigned long long)i);
            break;
        }
    }
    __syncthreads();
    const int j = (int)*s_min;
    if (j < n && j >= lo && j < hi) {
        double cj = before;
        for (int i = lo; i <= j; ++i) cj += key_val(keys[i]);
        *s_c = cj;
    }
    __syncthreads();
    return j;
}

// Copy the keys[0, n) of level lvl (relative to the maximum's bits mb) to dst, in
// any order; returns how many there are (copies at most cap).
__device__ int block_extract_level(const unsigned long long* keys, int n, uint32_t mb, int lvl,
                                   unsigned long long* dst, int cap, unsigned* s_ctr)
{
    const int tid = threadIdx.x, lane = tid & 31;
    if (tid == 0) *s_ctr = 0;
    __syncthreads();
    for (int b0 = 0; b0 < n; b0 += kThreads) {
        const int i = b0 + tid;
        unsigned long long key = 0ull;
        bool take = false;
        if (i < n) {
            key = keys[i];
            take = ((mb - ((uint32_t)(key >> 32) & 0x7fffffffu)) >> kLvlShift) == (uint32_t)lvl;
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, take);
        uint32_t base = 0;
        if (lane == 0 && bal) base = atomicAdd(s_ctr, (unsigned)__popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0) + __popc(bal & ((1u << lane) - 1u));
        if (take && base < (uint32_t)cap) dst[base] = key;
    }
    __syncthreads();
    return (int)*s_ctr;
}

__device__ __forceinline__ float block_max(float v, float* s_red)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) s_red[warp] = v;
    __syncthreads();
    float r = s_red[0];
    for (int w = 1; w < kWarps; ++w) r = fmaxf(r, s_red[w]);
    return r;
}

// Warp-parallel level search (one warp): the first level l < lmax whose cumulative
// mass (levels 0..l) reaches thr (STRICT: exceeds thr), the mass and count of the
// levels before it; l = -1 if none.  Level masses are exact (fixed point), so the
// sums are exact in any order.  Results in *out_l, *out_base, *out_nb (lane owning
// the level, or lane 0 when none).
template <bool STRICT>
__device__ __forceinline__ void warp_first_level(const double* lvl, const unsigned* cnt, int lmax, double thr,
                                                 int* out_l, double* out_base, int* out_nb)
{
    constexpr int kPL = (kLevels + 31) / 32;  // levels per lane, consecutive
    const int lane = threadIdx.x & 31;
    double v[kPL];
    unsigned c[kPL];
    double sv = 0.0;
    unsigned sc = 0u;
#pragma unroll
    for (int k = 0; k < kPL; ++k) {
        const int l = lane * kPL + k;
        v[k] = l < lmax ? lvl[l] : 0.0;
        c[k] = l < lmax ? cnt[l] : 0u;
        sv += v[k];
        sc += c[k];
    }
    double iv = sv;
    unsigned ic = sc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double yv = __shfl_up_sync(0xffffffffu, iv, o);
        const unsigned yc = __shfl_up_sync(0xffffffffu, ic, o);
        if (lane >= o) {
            iv += yv;
            ic += yc;
        }
    }
    double acc = __shfl_up_sync(0xffffffffu, iv, 1);
    unsigned nacc = __shfl_up_sync(0xffffffffu, ic, 1);
    if (lane == 0) {
        acc = 0.0;
        nacc = 0u;
    }
    unsigned first = 0xffffffffu;
    double base = 0.0;
    unsigned nb = 0u;
#pragma unroll
    for (int k = 0; k < kPL; ++k) {
        const int l = lane * kPL + k;
        if (l < lmax && first == 0xffffffffu) {
            const double nx = acc + v[k];
            if (STRICT ? nx > thr : nx >= thr) {
                first = (unsigned)l;
                base = acc;
                nb = nacc;
            } else {
                acc = nx;
                nacc += c[k];
            }
        }
    }
    const unsigned fl = __reduce_min_sync(0xffffffffu, first);
    if (fl == 0xffffffffu) {
        if (lane == 0) {
            *out_l = -1;
            *out_base = 0.0;
            *out_nb = 0;
        }
    } else if (first == fl) {
        *out_l = (int)fl;
        *out_base = base;
        *out_nb = (int)nb;
    }
}

// Row tickets: rows differ a lot in cost (superset size, level sizes, fallbacks),
// so a CTA takes the next row when it is done instead of a fixed share -- with a
// static grid-stride share the slowest CTA ran ~60 % longer than the median.
// The counter lives in the caller's workspace header (the launcher zeroes it on
// the stream before the launch), so concurrent or graph-captured calls with
// distinct workspaces never share it.
constexpr size_t kTicketWsOffset = 200;  // inside the 256-byte workspace header pad (192: shard counter)

__global__ void __launch_bounds__(kThreads, 2) k_top_p(const float* probs, int64_t rows, int64_t cols, int64_t stride,
                                                    float p, const float* u, int64_t* token_out, int32_t* kept_out,
                                                    unsigned int* ticket, int dbg, int pf, int w0)
{
    extern __shared__ __align__(16) unsigned long long s_key[];  // kCap candidate keys, then kLevCap level keys
    unsigned long long* const s_lev = s_key + kCap;
    __shared__ float s_red[kWarps];
    __shared__ double s_dred[kWarps];
    __shared__ unsigned s_cnt;
    __shared__ unsigned s_rmax;
    __shared__ int s_level;
    __shared__ double s_lvl[kLevels];
    __shared__ unsigned s_lcnt[kLevels];
    // per-warp fixed-point level masses as two 32-bit halves (fx >> 19, fx & (2^19 - 1)):
    // each half of a term is < 2^19 and a level has <= 8192 terms, so both sums fit
    // 32 bits -- native 32-bit shared atomics instead of 64-bit ones (measured: the
    // 64-bit atomics made the level-mass step ~35 % of the kernel)
    __shared__ unsigned s_whi[kWarps][kLevels];
    __shared__ unsigned s_wlo[kWarps][kLevels];
    __shared__ unsigned s_wcnt[kWarps][kLevels];
    __shared__ double s_c;
    __shared__ double s_base;
    __shared__ int s_aux[2];
    __shared__ unsigned long long s_min;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool vec = (cols % 4 == 0) && (stride % 4 == 0) && ((reinterpret_cast<uintptr_t>(probs) & 15) == 0);

    __shared__ int64_t s_row;
    // pf > 0: the CTA holds the ticket of its NEXT row too, and prefetches that row's
    // first pf * 32 KB into L2 once the current row's pass is done (its start -- the
    // seed loads and the first iterations -- is then an L2 hit)
    int64_t next_row = -1;
    // a row whose nucleus reached past attempt 0's narrower window is redone from
    // attempt 1 (uniform: every thread sets it from shared state)
    int64_t redo = -1;
    float redo_m = 0.f;  // the redone row's maximum (attempt 1's threshold)
    for (;;) {
        const int first_attempt = redo >= 0 ? 1 : 0;
        if (tid == 0) {
            if (redo >= 0) {
                s_row = redo;
            } else {
                s_row = next_row >= 0 ? next_row : (int64_t)ptx::claim_add(ticket, 1u);
                if (pf > 0) next_row = (int64_t)ptx::claim_add(ticket, 1u);
            }
        }
        redo = -1;
        __syncthreads();
        const int64_t row = s_row;
        __syncthreads();
        if (row >= rows) break;
        const float* q = probs + row * stride;
        auto prefetch_next_row = [&]() {
            if (pf > 0 && vec && tid == 0 && next_row < rows) {
                const int64_t n4 = cols / 4;
                const int64_t e4 = (int64_t)pf * TOPP_UNROLL * kThreads < n4 ? (int64_t)pf * TOPP_UNROLL * kThreads : n4;
                ptx::l2_prefetch_bulk(probs + next_row * stride, (uint32_t)(e4 * 16));
            }
        };
        // 1-2 (fast path, one HBM read of the row): the row maximum and, in the same
        // pass, a candidate SUPERSET -- every q whose bits are within 53 * 2^21 of the
        // running block maximum's (about q >= rmax * 2^-13.25; the running maximum only
        // grows, so this contains every q within that distance of the final m).  Then
        // levels l = (bits(m) - bits(q)) >> 20 (eighth octaves, monotone in q), the
        // exact fp64 mass per level (<= 8192 fp32 terms within 2^14 of each other: no
        // rounding, any order), the smallest level L whose cumulative mass reaches p,
        // and the candidates {l <= L} -- an upward-closed set holding the nucleus.
        int count = 0;
        bool ok = false;
        float m = first_attempt == 1 ? redo_m : 0.f;
        int used_attempt = 0;
        {
            constexpr uint32_t kSpan = (uint32_t)kLevels << kLvlShift;
            // seed the running maximum with the first 4 * kThreads elements' maximum
            // (from 0, the first block-iteration would collect everything)
            float lm = 0.f;
            for (int64_t i = tid; i < cols && i < 4 * kThreads; i += kThreads) lm = fmaxf(lm, __ldg(q + i));
            const float m0 = block_max(lm, s_red);
            bool over = false;
            // attempt 0 collects relative to the running maximum; a superset overflow
            // (the early, low running maximum admits too much) repeats the same pipelined
            // pass with the threshold fixed at the final maximum's window (attempt 1), then
            // with a 12-octave window (attempt 2: levels >= kLevels2 stay empty, so a
            // nucleus reaching past them is a short mass and takes the fallback) -- one or
            // two more row reads instead of the tau-stepping fallback and the host-side sort
            // path (2.7 % of the C4 rows overflowed and took ~45 % of the kernel time)
            uint32_t span = kSpan;
            for (int attempt = first_attempt; attempt < 3; ++attempt) {
            // attempt 0's window (w0 levels, default 12.25 octaves) is narrower than the
            // fixed-threshold retry's: ~30 % fewer candidates (their extraction was ~40 % of
            // the pass's instructions); a nucleus reaching past it redoes the row
            span = attempt == 0 ? ((uint32_t)w0 << kLvlShift)
                                : (attempt == 1 ? kSpan : ((uint32_t)kLevels2 << kLvlShift));
            used_attempt = attempt;
            if (tid == 0) {
                s_cnt = 0;
                s_rmax = __float_as_uint(attempt == 0 ? m0 : m);
            }
            __syncthreads();
            over = false;
            auto collect4 = [&](int64_t i0, const float (&v)[4], int nv) {
                const uint32_t rb = *reinterpret_cast<volatile unsigned*>(&s_rmax);
                const uint32_t thr = rb > span ? rb - span : 1u;  // bits of the collection threshold (> 0)
                uint32_t tk = 0;
                float vm = 0.f;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (j < nv) {
                        vm = fmaxf(vm, v[j]);
                        if (__float_as_uint(v[j]) >= thr && v[j] > 0.f) tk |= 1u << j;
                    }
                }
                lm = fmaxf(lm, vm);
                const uint32_t wmb = __reduce_max_sync(0xffffffffu, __float_as_uint(vm));  // vm >= 0: bits order
                if (lane == 0 && wmb > rb) atomicMax(&s_rmax, wmb);
                const uint32_t c = __popc(tk);
                uint32_t incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                uint32_t base = 0;
                if (lane == 31 && incl) base = atomicAdd(&s_cnt, incl);
                base = __shfl_sync(0xffffffffu, base, 31) + (incl - c);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if ((tk >> j) & 1u) {
                        if (base < (unsigned)kCap) {
                            const uint32_t code = __float_as_uint(v[j]) | 0x80000000u;
                            s_key[base] = ((unsigned long long)code << 32) | (0xffffffffu - (uint32_t)(i0 + j));
                        } else {
                            over = true;
                        }
                        ++base;
                    }
                }
            };
            if (vec) {
                // TOPP_UNROLL 16-byte loads in flight per thread; the values are screened
                // together: one running-max update and (when any lane has a
                // candidate) one warp compaction per 128 * TOPP_UNROLL elements of the warp
                constexpr int kUnroll = TOPP_UNROLL;
                const int64_t n4 = cols / 4;
                // L2 bulk prefetch `pf` iterations (of kUnroll * kThreads float4) ahead of
                // the loads: more bytes in flight than the registers hold
                constexpr int64_t kIt4 = (int64_t)kUnroll * kThreads;
                auto prefetch_it = [&](int64_t it) {
                    const int64_t a4 = it * kIt4;
                    if (a4 < n4) {
                        const int64_t e4 = a4 + kIt4 < n4 ? a4 + kIt4 : n4;
                        ptx::l2_prefetch_bulk(reinterpret_cast<const float4*>(q) + a4, (uint32_t)((e4 - a4) * 16));
                    }
                };
                if (tid == 0)
                    for (int k = 1; k <= pf; ++k) prefetch_it(k);
                // software-pipelined: the next iteration's loads are issued before this
                // iteration's values are screened
                float4 nf[kUnroll];
#pragma unroll
                for (int r = 0; r < kUnroll; ++r) {
                    const int64_t i4 = (int64_t)r * kThreads + tid;
                    nf[r] = i4 < n4 ? __ldcs(reinterpret_cast<const float4*>(q) + i4) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
                for (int64_t base4 = 0; base4 < n4; base4 += kUnroll * kThreads) {
                    if (pf > 0 && tid == 0) prefetch_it(base4 / kIt4 + 1 + pf);
                    float4 f[kUnroll];
#pragma unroll
                    for (int r = 0; r < kUnroll; ++r) {
                        f[r] = nf[r];
                        const int64_t i4 = base4 + kUnroll * kThreads + r * kThreads + tid;
                        nf[r] = i4 < n4 ? __ldcs(reinterpret_cast<const float4*>(q) + i4) : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                    const int rb = (int)*reinterpret_cast<volatile unsigned*>(&s_rmax);
                    const int thr = rb > (int)span ? rb - (int)span : 1;  // bits of the threshold (> 0)
                    float vm = 0.f;
                    uint32_t tk = 0;
#pragma unroll
                    for (int r = 0; r < kUnroll; ++r) {
                        const float v[4] = {f[r].x, f[r].y, f[r].z, f[r].w};
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            vm = fmaxf(vm, v[j]);
                            if (__float_as_int(v[j]) >= thr) tk |= 1u << (4 * r + j);  // negative values: < 0
                        }
                    }
                    lm = fmaxf(lm, vm);
                    const uint32_t wmb = __reduce_max_sync(0xffffffffu, __float_as_uint(vm));  // vm >= 0: bits order
                    if (lane == 0 && wmb > (uint32_t)rb) atomicMax(&s_rmax, wmb);
                    if (__any_sync(0xffffffffu, tk != 0)) {
                        const uint32_t c = __popc(tk);
                        uint32_t incl = c;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                            if (lane >= o) incl += y;
                        }
                        uint32_t base = 0;
                        if (lane == 31 && incl) base = atomicAdd(&s_cnt, incl);
                        base = __shfl_sync(0xffffffffu, base, 31) + (incl - c);
                        while (tk) {
                            const int e = __ffs(tk) - 1;
                            tk &= tk - 1;
                            const int r = e >> 2, j = e & 3;
                            float4 fr = f[0];
#pragma unroll
                            for (int rr = 1; rr < kUnroll; ++rr)
                                if (rr == r) fr = f[rr];
                            const float val = j == 0 ? fr.x : (j == 1 ? fr.y : (j == 2 ? fr.z : fr.w));
                            const uint32_t idx = (uint32_t)((base4 + r * kThreads + tid) * 4 + j);
                            if (base < (unsigned)kCap)
                                s_key[base] = ((unsigned long long)(__float_as_uint(val) | 0x80000000u) << 32) |
                                              (0xffffffffu - idx);
                            else
                                over = true;
                            ++base;
                        }
                    }
                }
            } else {
                for (int64_t b0 = 0; b0 < cols; b0 += 4 * kThreads) {
                    const int64_t i0 = b0 + 4 * tid;
                    float v[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) v[j] = i0 + j < cols ? __ldg(q + i0 + j) : 0.f;
                    const int64_t rem = cols - i0;
                    collect4(i0, v, rem <= 0 ? 0 : (rem > 4 ? 4 : (int)rem));
                }
            }
            m = block_max(lm, s_red);
            over = __syncthreads_or(over);
            count = (int)s_cnt;
            if (attempt == 0) prefetch_next_row();
            if (!over) break;
            }  // attempt
            if (dbg == 1) {  // timing A/B: the pass alone
                if (tid == 0) token_out[row] = count;
                __syncthreads();
                continue;
            }
            if (!over && (__float_as_uint(m) >> 23) >= 15u) {  // fixed-point levels need E_m - 14 >= 1
                const uint32_t mb = __float_as_uint(m);
                // level masses in fixed point: q = mant * 2^(E_q - 150) with E_q >= E_m - 14
                // for every level, so q / 2^(E_m - 164) = mant << (E_q - E_m + 14) < 2^38 is an
                // integer and <= 8192 of them sum below 2^51: exact u64 (per-warp bins, no fp
                // atomics), then one exact conversion per level
                const int Em = (int)(mb >> 23);
                for (int i = tid; i < kWarps * kLevels; i += kThreads) {
                    (&s_whi[0][0])[i] = 0u;
                    (&s_wlo[0][0])[i] = 0u;
                    (&s_wcnt[0][0])[i] = 0u;
                }
                __syncthreads();
                for (int i = tid; i < count; i += kThreads) {
                    const uint32_t code = (uint32_t)(s_key[i] >> 32) & 0x7fffffffu;
                    const uint32_t d = mb - code;  // code <= mb
                    if (d < span) {
                        const int Eq = (int)(code >> 23);
                        const unsigned long long fx = (unsigned long long)((code & 0x7fffffu) | 0x800000u)
                                                      << (Eq - Em + 14);
                        atomicAdd(&s_whi[warp][d >> kLvlShift], (unsigned)(fx >> 19));
                        atomicAdd(&s_wlo[warp][d >> kLvlShift], (unsigned)fx & 0x7ffffu);
                        atomicAdd(&s_wcnt[warp][d >> kLvlShift], 1u);
                    }
                }
                __syncthreads();
                for (int l = tid; l < kLevels; l += kThreads) {
                    unsigned long long sm = 0ull;
                    unsigned c = 0u;
                    for (int w = 0; w < kWarps; ++w) {
                        sm += ((unsigned long long)s_whi[w][l] << 19) + s_wlo[w][l];
                        c += s_wcnt[w][l];
                    }
                    s_lvl[l] = ldexp((double)sm, Em - 164);
                    s_lcnt[l] = c;
                }
                __syncthreads();
                // L = the first level whose cumulative mass reaches p; its base mass / count
                if (warp == 0) warp_first_level<false>(s_lvl, s_lcnt, kLevels, (double)p, &s_level, &s_base, &s_aux[0]);
                __syncthreads();
                const int L = s_level;
                if (L < 0 && used_attempt == 0 && w0 < kLevels) {  // short mass in the narrow window
                    redo = row;
                    redo_m = m;
                    __syncthreads();
                    continue;
                }
                if (dbg == 2) {  // timing A/B: pass + level masses + level search
                    if (tid == 0) token_out[row] = L >= 0 ? (int64_t)s_lcnt[L] : -2;
                    __syncthreads();
                    continue;
                }
                if (L >= 0 && s_lcnt[L] <= (unsigned)kLevCap) {
                    // ---- level path: sort level L only (and the draw's level) ----
                    const int nL = block_extract_level(s_key, count, mb, L, s_lev, kLevCap, &s_cnt);
                    const double baseL = s_base;
                    const int nbefL = s_aux[0];
                    if (nL <= kLevCap / 2) block_rank_sort_desc(s_lev, nL, s_lev + kLevCap / 2);
                    else block_sort_desc(s_lev, nL);
                    const int jL = block_first_crossing<false>(s_lev, nL, baseL, (double)p, s_dred, &s_min, &s_c);
                    if (dbg == 3) {  // timing A/B: ... + level L sorted, K found
                        if (tid == 0) token_out[row] = nL;
                        __syncthreads();
                        continue;
                    }
                    if (jL < nL) {  // always: cum(<= L) >= p
                        const int K = nbefL + jL + 1;
                        const double CK = s_c;
                        const double t = (double)__ldg(u + row) * CK;
                        // the draw's level: the first level (< L) whose cumulative mass exceeds t
                        __syncthreads();  // everyone has read s_base (baseL) above
                        if (warp == 0) warp_first_level<true>(s_lvl, s_lcnt, L, t, &s_aux[1], &s_base, &s_aux[0]);
                        __syncthreads();
                        const int ls = s_aux[1] < 0 ? L : s_aux[1];
                        const double base2 = s_base;
                        int nl = jL + 1;  // level L: only its nucleus part
                        bool lev_ok = true;
                        if (ls != L) {
                            if (s_lcnt[ls] <= (unsigned)kLevCap) {
                                nl = block_extract_level(s_key, count, mb, ls, s_lev, kLevCap, &s_cnt);
                                if (nl <= kLevCap / 2) block_rank_sort_desc(s_lev, nl, s_lev + kLevCap / 2);
                                else block_sort_desc(s_lev, nl);
                            } else {
                                lev_ok = false;
                            }
                        }
                        if (lev_ok) {
                            int r = block_first_crossing<true>(s_lev, nl, ls == L ? baseL : base2, t, s_dred, &s_min,
                                                               &s_c);
                            if (r >= nl) r = nl - 1;  // t within rounding of the level's end: its last element
                            if (tid == 0) {
                                token_out[row] = (int64_t)(0xffffffffu - (uint32_t)(s_lev[r] & 0xffffffffu));
                                if (kept_out) kept_out[row] = K;
                            }
                            __syncthreads();
                            continue;  // next row
                        }
                    }
                }
                if (L >= 0) {
                    // keep {level <= L}: read this thread's contiguous share, then write
                    constexpr int kPer = kCap / kThreads;
                    const int lo = tid * kPer, hi = min(count, lo + kPer);
                    unsigned long long key[kPer];
                    uint32_t keep = 0;  // bit k: key[k] is kept (static indices: registers)
#pragma unroll
                    for (int k = 0; k < kPer; ++k) {
                        key[k] = lo + k < hi ? s_key[lo + k] : 0ull;
                        const uint32_t code = (uint32_t)(key[k] >> 32) & 0x7fffffffu;
                        if (lo + k < hi && ((mb - code) >> kLvlShift) <= (uint32_t)L) keep |= 1u << k;
                    }
                    const int nk = __popc(keep);
                    int incl = nk;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int y = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += y;
                    }
                    if (lane == 31) s_red[warp] = __int_as_float(incl);
                    __syncthreads();
                    int wpre = 0, tot = 0;
                    for (int w = 0; w < kWarps; ++w) {
                        const int y = __float_as_int(s_red[w]);
                        if (w < warp) wpre += y;
                        tot += y;
                    }
                    int ob = wpre + incl - nk;
#pragma unroll
                    for (int k = 0; k < kPer; ++k)
                        if ((keep >> k) & 1u) s_key[ob++] = key[k];
                    count = tot;
                    ok = true;
                    __syncthreads();
                }
            }
        }

        if (dbg == 5) {  // diagnostics: rows the level path did not finish, by cause (-10 - code)
            if (tid == 0) token_out[row] = -10 - (ok ? (count > kLevCap ? 3 : 0) : (count > kCap ? 1 : 2));
            __syncthreads();
            continue;
        }
        if (dbg == 4 && !ok) {  // timing A/B: rows that need the fallback are skipped
            if (tid == 0) token_out[row] = 0;
            __syncthreads();
            continue;
        }
        // 1-2 (fallback): candidates {q >= tau} until their mass reaches p
        for (int sh = 8; !ok && sh <= 160; sh += 4) {
            const float tau = sh >= 150 ? 0.f : ldexpf(m, -sh);
            if (tid == 0) s_cnt = 0;
            __syncthreads();
            double mass = 0.0;
            bool over = false;
            auto take4 = [&](int64_t i0, const float (&v)[4], int nv) {
                uint32_t tk = 0;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (j < nv && v[j] >= tau) tk |= 1u << j;
                const uint32_t c = __popc(tk);
                uint32_t incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                uint32_t base = 0;
                if (lane == 31 && incl) base = atomicAdd(&s_cnt, incl);
                base = __shfl_sync(0xffffffffu, base, 31) + (incl - c);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if ((tk >> j) & 1u) {
                        if (base < (unsigned)kCap) {
                            const uint32_t code = __float_as_uint(v[j]) | 0x80000000u;  // q >= 0: P287 code
                            s_key[base] = ((unsigned long long)code << 32) | (0xffffffffu - (uint32_t)(i0 + j));
                        } else {
                            over = true;
                        }
                        ++base;
                        mass += (double)v[j];
                    }
                }
            };
            if (vec) {
                for (int64_t base4 = 0; base4 < cols / 4; base4 += kThreads) {
                    const int64_t i4 = base4 + tid;
                    float v[4] = {-1.f, -1.f, -1.f, -1.f};
                    if (i4 < cols / 4) {
                        const float4 f = __ldg(reinterpret_cast<const float4*>(q) + i4);
                        v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
                    }
                    take4(i4 * 4, v, i4 < cols / 4 ? 4 : 0);
                }
            } else {
                for (int64_t b0 = 0; b0 < cols; b0 += 4 * kThreads) {
                    const int64_t i0 = b0 + 4 * tid;
                    float v[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) v[j] = i0 + j < cols ? __ldg(q + i0 + j) : -1.f;
                    const int64_t rem = cols - i0;
                    take4(i0, v, rem <= 0 ? 0 : (rem > 4 ? 4 : (int)rem));
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mass += __shfl_xor_sync(0xffffffffu, mass, o);
            __syncthreads();
            if (lane == 0) s_dred[warp] = mass;
            __syncthreads();
            double tot = 0.0;
            for (int w = 0; w < kWarps; ++w) tot += s_dred[w];
            count = (int)s_cnt;
            over = __syncthreads_or(over);
            if (over) break;                                // too many candidates: fallback
            if (tot >= (double)p || tau == 0.f) {           // nucleus inside (or the whole row)
                ok = true;
                break;
            }
        }
        if (!ok) {
            if (tid == 0) {
                token_out[row] = -1;
                if (kept_out) kept_out[row] = -1;
            }
            __syncthreads();
            continue;
        }

        // 3. all candidates sorted, descending by (code, ~index)
        block_sort_desc(s_key, count);
        // 4. K = 1 + min{ j : C_j >= p }, t = u * C_{K-1}, rank = min{ k : C_k > t }
        const int jK = block_first_crossing<false>(s_key, count, 0.0, (double)p, s_dred, &s_min, &s_c);
        int K = count;
        double CK = 0.0;
        if (jK < count) {
            K = jK + 1;
            CK = s_c;
        } else {  // the candidates' whole mass is below p (tau = 0: the whole row)
            if (tid == 0) {
                double c = 0.0;
                for (int i = 0; i < count; ++i) c += key_val(s_key[i]);
                s_c = c;
            }
            __syncthreads();
            CK = s_c;
        }
        const double t = (double)__ldg(u + row) * CK;
        int r = block_first_crossing<true>(s_key, K, 0.0, t, s_dred, &s_min, &s_c);
        if (r >= K) r = K - 1;
        if (tid == 0) {
            token_out[row] = (int64_t)(0xffffffffu - (uint32_t)(s_key[r] & 0xffffffffu));
            if (kept_out) kept_out[row] = K;
        }
        __syncthreads();
    }
}

}  // namespace topp
}  // namespace scan

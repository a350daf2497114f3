// topp.cuh -- top-p (nucleus) sampling without a full row sort (PAPER Sec.
// 5.5, P298-299).
//
// The paper's top-p is "sort and scan on the token probability vector"
// (P299): sort the row descending, scan it, keep the smallest prefix whose
// mass reaches p, draw from it.  Only the TOP of the order matters: the
// nucleus is a prefix of the descending order, so it lies inside any set
// {tokens with probability >= tau} whose mass reaches p.  One CTA per row:
//   1. the row maximum m (one HBM read of the row; the row stays in L2);
//   2. candidates {q >= tau}, tau = m * 2^-s, gathered into shared memory
//      (warp-aggregated compaction) with their exact fp64 mass; if the mass
//      is below p, tau is lowered (s += 8) and the row re-read from L2;
//   3. the candidates sorted by (q descending, index ascending) -- exactly the
//      stable descending order of the full sort -- with a bitonic network in
//      shared memory (64-bit keys: P287's order-preserving code, ~index);
//   4. the inclusive fp64 scan C of the sorted candidates (block scan),
//      K = 1 + min{ j : C_j >= p }, t = u * C_{K-1}, rank = min{ k : C_k > t },
//      token = index of rank (R15 -- the same arithmetic as the oracle, summed
//      in a tree order instead of left to right).
// A row whose candidate set would exceed kCap before reaching mass p is not
// handled here: token_out = -1 and the caller falls back to the sort path.
#pragma once
#include <stdint.h>

namespace scan {
namespace topp {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kCap = 8192;       // candidates per row (64 KB of 64-bit keys)

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

__global__ void __launch_bounds__(kThreads) k_top_p(const float* probs, int64_t rows, int64_t cols, int64_t stride,
                                                    float p, const float* u, int64_t* token_out, int32_t* kept_out)
{
    extern __shared__ __align__(16) unsigned long long s_key[];  // kCap sort keys
    __shared__ float s_red[kWarps];
    __shared__ double s_dred[kWarps];
    __shared__ unsigned s_cnt;
    __shared__ unsigned long long s_min;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool vec = (cols % 4 == 0) && (stride % 4 == 0) && ((reinterpret_cast<uintptr_t>(probs) & 15) == 0);

    for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
        const float* q = probs + row * stride;
        // 1. row maximum
        float m = 0.f;
        if (vec) {
            for (int64_t i = tid; i < cols / 4; i += kThreads) {
                const float4 v = __ldg(reinterpret_cast<const float4*>(q) + i);
                m = fmaxf(m, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
            }
        } else {
            for (int64_t i = tid; i < cols; i += kThreads) m = fmaxf(m, __ldg(q + i));
        }
        m = block_max(m, s_red);

        // 2. candidates {q >= tau} until their mass reaches p
        int count = 0;
        bool ok = false;
        for (int sh = 8; sh <= 160; sh += 4) {
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

        // 3. bitonic sort, descending by (code, ~index), padded to a power of two
        int N = 1;
        while (N < count) N <<= 1;
        for (int i = count + tid; i < N; i += kThreads) s_key[i] = 0ull;
        __syncthreads();
        for (int k = 2; k <= N; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = tid; i < N; i += kThreads) {
                    const int ixj = i ^ j;
                    if (ixj > i) {
                        const unsigned long long a = s_key[i], b = s_key[ixj];
                        const bool desc = (i & k) == 0;
                        if (desc ? (a < b) : (a > b)) {
                            s_key[i] = b;
                            s_key[ixj] = a;
                        }
                    }
                }
                __syncthreads();
            }
        }

        // 4. inclusive fp64 scan over the sorted candidates; nucleus; draw
        const int per = (count + kThreads - 1) / kThreads;  // consecutive elements per thread
        const int lo = tid * per, hi = min(count, lo + per);
        double run = 0.0;
        for (int i = lo; i < hi; ++i) run += (double)__uint_as_float((uint32_t)(s_key[i] >> 32) & 0x7fffffffu);
        double incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_dred[warp] = incl;
        __syncthreads();
        double wpre = 0.0;
        for (int w = 0; w < warp; ++w) wpre += s_dred[w];
        double ex = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane == 0) ex = 0.0;
        const double before = wpre + ex;  // exclusive prefix of this thread's first element
        // K = 1 + min{ j : C_j >= p }
        if (tid == 0) s_min = (unsigned long long)count;
        __syncthreads();
        {
            double c = before;
            for (int i = lo; i < hi; ++i) {
                c += (double)__uint_as_float((uint32_t)(s_key[i] >> 32) & 0x7fffffffu);
                if (c >= (double)p) {
                    atomicMin(&s_min, (unsigned long long)i);
                    break;
                }
            }
        }
        __syncthreads();
        const int jK = (int)s_min;
        const int K = jK < count ? jK + 1 : count;
        __syncthreads();
        // C_{K-1}: the thread owning K-1 publishes it
        if (K - 1 >= lo && K - 1 < hi) {
            double c = before;
            for (int i = lo; i <= K - 1; ++i) c += (double)__uint_as_float((uint32_t)(s_key[i] >> 32) & 0x7fffffffu);
            s_dred[0] = c;
        }
        if (tid == 0) s_min = (unsigned long long)K;
        __syncthreads();
        const double t = (double)__ldg(u + row) * s_dred[0];
        {
            double c = before;
            for (int i = lo; i < hi && i < K; ++i) {
                c += (double)__uint_as_float((uint32_t)(s_key[i] >> 32) & 0x7fffffffu);
                if (c > t) {
                    atomicMin(&s_min, (unsigned long long)i);
                    break;
                }
            }
        }
        __syncthreads();
        if (tid == 0) {
            int r = (int)s_min;
            if (r >= K) r = K - 1;
            token_out[row] = (int64_t)(0xffffffffu - (uint32_t)(s_key[r] & 0xffffffffu));
            if (kept_out) kept_out[row] = K;
        }
        __syncthreads();
    }
}

}  // namespace topp
}  // namespace scan

// sample.cuh -- the inverse-transform draws on top of a prefix sum: weighted
// sampling (PAPER App. B.3, P463) and the nucleus / draw step of top-p
// sampling (Sec. 5.5, P298-299), for sm_100a.
//
// Both reduce to "first index whose cumulative sum exceeds a threshold" on a
// non-decreasing prefix sum that the scan kernels have already written: no
// second pass over the data is needed, a k-ary search does it in O(log_1024 n)
// rounds of coalesced probes (one CTA per search; one CTA per row for top-p).
//   weighted (R14):  S = scan(w); t = theta * S[n-1]; i = min{ i : S_i > t }
//   top-p (R15):     C = row scan of the descending probabilities;
//                    K = 1 + min{ j : C_j >= p }   (all ranks if none)
//                    t = u * C_{K-1};   rank = min{ k : C_k > t };
//                    token = order[rank]
#pragma once
#include <stdint.h>

namespace scan {
namespace sample {

constexpr int kThreads = 256;

// First index i in [0, n) with pred(S[i]) true on a monotone predicate
// (false...false true...true); n if none.  One CTA; k-ary search: every round
// probes kThreads evenly spaced points and keeps the bracket between the last
// false and the first true probe.
template <typename Pred>
__device__ __forceinline__ int64_t first_true(const float* S, int64_t n, Pred pred, int64_t* s_br)
{
    const int tid = threadIdx.x;
    int64_t lo = 0, hi = n;  // answer in [lo, hi]; S[hi] true or hi == n
    while (hi - lo > kThreads) {
        const int64_t span = hi - lo;
        const int64_t idx = lo + (span * (tid + 1)) / (kThreads + 1);  // strictly inside (lo, hi)
        const bool t = pred(__ldg(S + idx));
        // first true probe (its index) and the last false probe before it
        if (tid == 0) s_br[0] = hi;
        __syncthreads();
        if (t) atomicMin(reinterpret_cast<unsigned long long*>(&s_br[0]), (unsigned long long)idx);
        __syncthreads();
        const int64_t first_t = s_br[0];
        if (tid == 0) s_br[1] = lo - 1;
        __syncthreads();
        if (!t && idx < first_t) atomicMax(reinterpret_cast<long long*>(&s_br[1]), (long long)idx);
        __syncthreads();
        const int64_t last_f = s_br[1];
        __syncthreads();
        lo = last_f + 1;
        hi = first_t;
    }
    // linear finish over at most kThreads elements
    if (tid == 0) s_br[0] = hi;
    __syncthreads();
    const int64_t i = lo + tid;
    if (i < hi && pred(__ldg(S + i))) atomicMin(reinterpret_cast<unsigned long long*>(&s_br[0]), (unsigned long long)i);
    __syncthreads();
    const int64_t r = s_br[0];
    __syncthreads();
    return r;
}

// Weighted sampling draw: *out = min{ i : S_i > theta * S[n-1] } (n-1 if none).
__global__ void __launch_bounds__(kThreads) k_weighted_draw(const float* S, int64_t n, double theta, int64_t* out)
{
    __shared__ int64_t s_br[2];
    const double t = theta * (double)__ldg(S + n - 1);
    const int64_t i = first_true(S, n, [t](float v) { return (double)v > t; }, s_br);
    if (threadIdx.x == 0) *out = i < n ? i : n - 1;
}

// Top-p nucleus + draw, one CTA per row of the inclusive scan C of the
// descending-sorted probabilities.
__global__ void __launch_bounds__(kThreads) k_top_p_draw(const float* C, const int32_t* order, int64_t cols,
                                                          int64_t c_stride, int64_t o_stride, float p, const float* u,
                                                          int64_t* token_out, int32_t* kept_out)
{
    __shared__ int64_t s_br[2];
    const int64_t row = blockIdx.x;
    const float* Cr = C + row * c_stride;
    const double pp = (double)p;
    const int64_t j = first_true(Cr, cols, [pp](float v) { return (double)v >= pp; }, s_br);
    const int64_t K = j < cols ? j + 1 : cols;
    const double t = (double)__ldg(u + row) * (double)__ldg(Cr + K - 1);
    int64_t r = first_true(Cr, K, [t](float v) { return (double)v > t; }, s_br);
    if (r >= K) r = K - 1;
    if (threadIdx.x == 0) {
        token_out[row] = (int64_t)__ldg(order + row * o_stride + r);
        if (kept_out) kept_out[row] = (int32_t)K;
    }
}

}  // namespace sample
}  // namespace scan

// shard.cuh -- pass 1 of the sharded (multi-GPU) scan: the block-level
// reduction of Reduce-Scan-Scan (PAPER P73, Sec. 2.1: "a block-level
// reduction first, followed by a scan of the block-level reductions and a
// final scan of each block").
//
// A rank's shard cannot be scanned single-pass before the sums of the lower
// shards are known, so it is read twice anyway.  Doing
// the reduction per BLOCK (not just per shard) makes the second read a pure
// stream: every block's starting value is known (carry of the lower shards +
// exclusive prefix of the block sums), so pass 2 is the batched row kernel
// (rowscan.cuh, one CTA per block-row, no grid barrier, no look-back) instead
// of the single-GPU MCScan with its L2-resident re-read.
//
// k_block_sums: CTA c reduces blocks c, c + grid, ... (highest first, so the
// shard's beginning -- which pass 2 reads first -- is read last and kept in L2
// with evict_last), every element widened exactly to fp64 / int64, fixed
// summation order (identical bits per call).  The last CTA scans the block
// sums into pre[b] = sum of blocks < b and pre[nb] = the shard total.
#pragma once
#include <stdint.h>

#include "ptx.cuh"
#include "scan_kernels.cuh"

namespace scan {
namespace shard {

constexpr int kThreads = 512;

// ---- device-initiated exchange of the shard totals ----
// Rank q's total for call `epoch` lives in every rank's slot array at entry
// (epoch % kPeerRing) * G + q: two 8-byte words (epoch << 32 | high 32 bits of
// the int64 / fp64 bits, epoch << 32 | low 32 bits), each one aligned 8-byte
// store, so a reader that sees its epoch in both words has the whole value --
// no flag, no fence order between the words.  The ring lets a rank run up to
// kPeerRing - 1 calls ahead of the slowest reader.
constexpr int kPeerRing = 64;

struct PeerPub {
    uint64_t* const* peers;  // device array of G pointers: rank q's slot array as seen from this GPU
    int G;
    int rank;
    uint32_t epoch;
};

// The tagged words are self-contained (the value travels inside them), so
// neither side needs ordering against other memory: relaxed system-scope
// accesses.  (A st.release.sys per word measured ~1.7 us each -- 28 us for
// G = 8 -- more than the NCCL all-gather it replaces.)
__device__ __forceinline__ void st_relaxed_sys_u64(uint64_t* p, uint64_t v)
{
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_sys_u64(const uint64_t* p)
{
    uint64_t v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void publish_total(const PeerPub& pp, uint64_t bits)
{
    const uint64_t tag = (uint64_t)pp.epoch << 32;
    const int e = (int)(pp.epoch % kPeerRing) * pp.G + pp.rank;
    for (int q = 0; q < pp.G; ++q) {
        uint64_t* slot = pp.peers[q] + 2 * e;
        st_relaxed_sys_u64(slot, tag | (bits >> 32));
        st_relaxed_sys_u64(slot + 1, tag | (bits & 0xffffffffull));
    }
}

// Warp-wide: wait until ranks 0..rank-1 have published call `epoch` into this
// rank's slot array, then their totals summed in rank order (lane 0's result
// is broadcast).  G <= 32.
template <typename Sum>
__device__ __forceinline__ Sum wait_carry_from_slots(const uint64_t* slots, int G, int rank, uint32_t epoch, int lane)
{
    uint64_t bits = 0;
    if (lane < rank) {
        const uint64_t* e = slots + 2 * ((int)(epoch % kPeerRing) * G + lane);
        uint32_t backoff = 32;
        while (true) {
            const uint64_t hi = ld_relaxed_sys_u64(e), lo = ld_relaxed_sys_u64(e + 1);
            if ((uint32_t)(hi >> 32) == epoch && (uint32_t)(lo >> 32) == epoch) {
                bits = (hi << 32) | (lo & 0xffffffffull);
                break;
            }
            __nanosleep(backoff);
            backoff = backoff < 1024 ? backoff * 2 : 1024;
        }
    }
    Sum c = Sum(0);
    for (int q = 0; q < rank; ++q) {  // fixed order: totals[0] + ... + totals[rank-1]
        const uint64_t b = __shfl_sync(0xffffffffu, bits, q);
        Sum v;
        memcpy(&v, &b, sizeof(v));
        c += v;
    }
    return c;
}

// An empty shard still publishes (its total is 0).
__global__ void k_publish_zero(PeerPub pub)
{
    if (threadIdx.x == 0) publish_total(pub, 0ull);
}

// One warp: the carry of a rank from its slot array (for the paths that do not
// run the row kernel: shards shorter than a block, unaligned shards).
template <typename Sum>
__global__ void k_carry_from_slots(const uint64_t* slots, int G, int rank, uint32_t epoch, Sum* carry_out)
{
    const Sum c = wait_carry_from_slots<Sum>(slots, G, rank, epoch, threadIdx.x & 31);
    if (threadIdx.x == 0) *carry_out = c;
}

template <int DT>
using SumT = typename std::conditional<Traits<DT>::kFloat, double, long long>::type;

template <int DT>
__global__ void __launch_bounds__(kThreads) k_block_sums(const void* in_, int64_t n, int64_t blk, int64_t nb,
                                                         SumT<DT>* bsum, SumT<DT>* pre, void* total_out,
                                                         uint32_t* done, PeerPub pub)
{
    using Tr = Traits<DT>;
    using In = typename Tr::In;
    using Sum = SumT<DT>;
    constexpr int VN = Vec16<In>::kN;  // elements per 16-byte vector
    const In* in = reinterpret_cast<const In*>(in_);
    const uint64_t pol = ptx::policy_evict_last();
    __shared__ Sum s_part[kThreads / 32];
    __shared__ bool s_last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    for (int64_t b = nb - 1 - blockIdx.x; b >= 0; b -= gridDim.x) {
        const int64_t lo = b * blk;
        const int64_t m = n - lo < blk ? n - lo : blk;
        // whole vectors (blocks start 16-byte aligned when the shard does)
        const int64_t nv = (((uintptr_t)in_ & 15u) == 0) ? m / VN : 0;
        const uint4* v = reinterpret_cast<const uint4*>(in + lo);
        Sum acc = 0;
        int64_t i = tid;
        for (; i + 3 * kThreads < nv; i += 4 * kThreads) {
            const uint4 a = ptx::ld_keep_v4(v + i, pol);
            const uint4 b1 = ptx::ld_keep_v4(v + i + kThreads, pol);
            const uint4 c = ptx::ld_keep_v4(v + i + 2 * kThreads, pol);
            const uint4 d = ptx::ld_keep_v4(v + i + 3 * kThreads, pol);
            acc += sum_vec16<DT, Sum>(a);
            acc += sum_vec16<DT, Sum>(b1);
            acc += sum_vec16<DT, Sum>(c);
            acc += sum_vec16<DT, Sum>(d);
        }
        for (; i < nv; i += kThreads) acc += sum_vec16<DT, Sum>(ptx::ld_keep_v4(v + i, pol));
        for (int64_t j = nv * VN + tid; j < m; j += kThreads) acc += to_sum<Sum>(widen(in[lo + j]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        __syncthreads();
        if (lane == 0) s_part[warp] = acc;
        __syncthreads();
        if (tid == 0) {
            Sum t = 0;
            for (int w = 0; w < kThreads / 32; ++w) t += s_part[w];
            bsum[b] = t;
        }
    }
    // last CTA: exclusive scan of the block sums (fixed tree order), total
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = ptx::claim_add(done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    Sum carry = 0;
    for (int64_t base = 0; base < nb; base += kThreads) {
        const int64_t i = base + tid;
        const Sum x = i < nb ? ((volatile Sum*)bsum)[i] : Sum(0);
        Sum incl = x;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const Sum y = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += y;
        }
        __syncthreads();
        if (lane == 31) s_part[warp] = incl;
        __syncthreads();
        Sum wpre = 0, tot = 0;
        for (int w = 0; w < kThreads / 32; ++w) {
            const Sum y = s_part[w];
            if (w < warp) wpre += y;
            tot += y;
        }
        Sum ex = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane == 0) ex = Sum(0);
        if (i < nb) pre[i] = carry + (wpre + ex);
        carry += tot;
    }
    if (tid == 0) {
        pre[nb] = carry;
        *reinterpret_cast<Sum*>(total_out) = carry;
        *done = 0;
        if (pub.peers != nullptr) {  // device-initiated exchange: the total straight into every rank's slots
            uint64_t b;
            memcpy(&b, &carry, sizeof(b));
            publish_total(pub, b);
        }
    }
}

// carry_out = carry_in (nullable) + pre[idx]: the start value of a trailing
// partial block handed to the 1-D scan.
template <typename Sum>
__global__ void k_carry_plus(const Sum* carry_in, const Sum* pre, int64_t idx, Sum* carry_out)
{
    if (threadIdx.x == 0) *carry_out = (carry_in ? *carry_in : Sum(0)) + pre[idx];
}

}  // namespace shard

namespace ceiling {

// The measurement ceiling of a scan: the same bytes (read In, write the widened
// Out) with no arithmetic beyond the widening -- a grid-stride stream of
// 16-byte loads and stores.  Not on any scan path; bench.py reports it next to
// the scan so the roofline fraction can be read against what a pure stream of
// the identical traffic achieves in the same run.
template <int DT>
__global__ void __launch_bounds__(256) k_widen_copy(const void* in_, void* out_, int64_t n)
{
    using Tr = Traits<DT>;
    using In = typename Tr::In;
    constexpr int VN = 16 / (int)sizeof(In);  // elements per 16-byte input vector
    const In* in = reinterpret_cast<const In*>(in_);
    uint32_t* out = reinterpret_cast<uint32_t*>(out_);
    const int64_t nv = n / VN;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    auto emit = [&](int64_t i, const uint4& q) {
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
        uint32_t o[VN];
#pragma unroll
        for (int k = 0; k < VN; ++k) {
            if constexpr (sizeof(In) == 4) o[k] = w[k];
            else if constexpr (sizeof(In) == 2) o[k] = __float_as_uint(__half2float(__ushort_as_half((uint16_t)(w[k >> 1] >> (16 * (k & 1))))));
            else o[k] = (uint32_t)(int32_t)(int8_t)(w[k >> 2] >> (8 * (k & 3)));
        }
#pragma unroll
        for (int k = 0; k < VN; k += 4)
            __stcs(reinterpret_cast<uint4*>(out + i * VN + k), make_uint4(o[k], o[k + 1], o[k + 2], o[k + 3]));
    };
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < nv; i += 4 * stride) {  // four 16-byte loads in flight per thread
        const uint4 a = ptx::ld_stream_v4(reinterpret_cast<const uint4*>(in) + i);
        const uint4 b = ptx::ld_stream_v4(reinterpret_cast<const uint4*>(in) + i + stride);
        const uint4 c = ptx::ld_stream_v4(reinterpret_cast<const uint4*>(in) + i + 2 * stride);
        const uint4 d = ptx::ld_stream_v4(reinterpret_cast<const uint4*>(in) + i + 3 * stride);
        emit(i, a);
        emit(i + stride, b);
        emit(i + 2 * stride, c);
        emit(i + 3 * stride, d);
    }
    for (; i < nv; i += stride) emit(i, ptx::ld_stream_v4(reinterpret_cast<const uint4*>(in) + i));
    for (int64_t j = nv * VN + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
        if constexpr (sizeof(In) == 4) out[j] = reinterpret_cast<const uint32_t*>(in)[j];
        else if constexpr (sizeof(In) == 2) out[j] = __float_as_uint(__half2float(__ushort_as_half(reinterpret_cast<const uint16_t*>(in)[j])));
        else out[j] = (uint32_t)(int32_t)in[j];
    }
}

}  // namespace ceiling
}  // namespace scan

// shard_api.cuh -- C ABI of the two-pass sharded scan (include/scan.h:
// scan_shard_workspace_bytes / scan_shard_reduce / scan_shard_scan), compiled
// into scan_api.cu's translation unit.  Host code only.
#pragma once
#include "shard.cuh"

namespace {

constexpr int64_t kShardBlk = 131072;       // elements per block = one row of pass 2
constexpr size_t kShardDone = 192;          // done counter inside the zeroed header block

size_t up256(size_t b) { return (b + 255) & ~(size_t)255; }

// [0, base): the scan workspace of pass 2 (rows + tail); then pre[nb + 1],
// bsum[nb], one carry scalar.
size_t shard_base(int dt, int64_t n)
{
    const int64_t nfull = n / kShardBlk, tail = n % kShardBlk;
    const size_t a = nfull > 0 ? scan_rows_workspace_bytes(dt, nfull, kShardBlk) : 0;
    const size_t b = scan_workspace_bytes(dt, n);  // also covers the tail and the unaligned fallback
    (void)tail;
    return up256(a > b ? a : b);
}

}  // namespace

extern "C" {

size_t scan_shard_workspace_bytes(int dtype, int64_t n)
{
    if (!valid_dt(dtype) || n < 0) return 0;
    const int64_t nb = (n + kShardBlk - 1) / kShardBlk;
    return shard_base(dtype, n) + (size_t)(2 * nb + 2) * 8 + 64;
}

int scan_shard_reduce(const void* in, int64_t n, int dtype, void* total_out, void* ws, size_t ws_bytes, void* stream)
{
    if (!valid_dt(dtype) || n < 0 || total_out == nullptr) return SCAN_ERR_ARG;
    if (n > 0 && in == nullptr) return SCAN_ERR_ARG;
    if (ws == nullptr || ((uintptr_t)ws & 255u) != 0 || ws_bytes < scan_shard_workspace_bytes(dtype, n))
        return SCAN_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    if (n == 0) return cudaMemsetAsync(total_out, 0, 8, s) == cudaSuccess ? SCAN_OK : SCAN_ERR_CUDA;
    DevInfo di;
    int st = dev_info(di);
    if (st != SCAN_OK) return st;
    const int64_t nb = (n + kShardBlk - 1) / kShardBlk;
    uint8_t* w = (uint8_t*)ws;
    uint8_t* arr = w + shard_base(dtype, n);
    uint32_t* done = reinterpret_cast<uint32_t*>(w + kShardDone);
    const int64_t g = (int64_t)di.sms * 4 < nb ? (int64_t)di.sms * 4 : nb;
    using namespace scan::shard;
    switch (dtype) {
#define SHARD_CASE(DT)                                                                                           \
    case DT: {                                                                                                   \
        using S_ = SumT<DT>;                                                                                     \
        S_* pre = reinterpret_cast<S_*>(arr);                                                                    \
        k_block_sums<DT><<<(unsigned)g, scan::shard::kThreads, 0, s>>>(in, n, kShardBlk, nb, pre + nb + 1, pre, total_out,    \
                                                           done);                                                \
        break;                                                                                                   \
    }
        SHARD_CASE(SCAN_I32_I32)
        SHARD_CASE(SCAN_F32_F32)
        SHARD_CASE(SCAN_F16_F32)
        SHARD_CASE(SCAN_I8_I32)
#undef SHARD_CASE
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError() == cudaSuccess ? SCAN_OK : SCAN_ERR_CUDA;
}

int scan_shard_scan(const void* in, void* out, int64_t n, int dtype, int exclusive, const void* carry_in, void* ws,
                    size_t ws_bytes, void* stream)
{
    if (!valid_dt(dtype) || n < 0) return SCAN_ERR_ARG;
    if (n == 0) return SCAN_OK;
    if (in == nullptr || out == nullptr) return SCAN_ERR_ARG;
    if (overlaps(in, n * in_size(dtype), out, n * out_size(dtype)) && in != out) return SCAN_ERR_ARG;
    if (ws == nullptr || ((uintptr_t)ws & 255u) != 0 || ws_bytes < scan_shard_workspace_bytes(dtype, n))
        return SCAN_ERR_WORKSPACE;
    DevInfo di;
    int st = dev_info(di);
    if (st != SCAN_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    const bool aligned = ((uintptr_t)in & 15u) == 0 && ((uintptr_t)out & 15u) == 0;
    if (!aligned || in == out)  // no row view: the single-pass scan with the carry (block sums unused)
        return scan_1d(in, out, n, dtype, carry_in, ws, ws_bytes, stream, exclusive);
    const int64_t nb = (n + kShardBlk - 1) / kShardBlk, nfull = n / kShardBlk, tail = n % kShardBlk;
    uint8_t* w = (uint8_t*)ws;
    uint8_t* arr = w + shard_base(dtype, n);
    if (nfull > 0) {  // pass 2: every block a row starting from carry_in + pre[block]
        ScanParams p{};
        p.in = in;
        p.out = out;
        p.seg_len = kShardBlk;
        p.num_segs = nfull;
        p.in_stride = kShardBlk;
        p.out_stride = kShardBlk;
        p.carry_in = carry_in;
        p.row_pre = arr;
        p.ws = w;
        p.exclusive = exclusive ? 1 : 0;
        p.tma_in = 1;
        p.tma_out = 1;
        switch (dtype) {
        case SCAN_I32_I32: st = launch_rows<SCAN_I32_I32>(p, s, di); break;
        case SCAN_F32_F32: st = launch_rows<SCAN_F32_F32>(p, s, di); break;
        case SCAN_F16_F32: st = launch_rows<SCAN_F16_F32>(p, s, di); break;
        default: st = launch_rows<SCAN_I8_I32>(p, s, di); break;
        }
        if (st != SCAN_OK) return st;
    }
    if (tail > 0) {  // trailing partial block: 1-D scan from carry_in + pre[nfull]
        uint8_t* carry = arr + (size_t)(2 * nb + 1) * 8;
        if (is_float(dtype))
            scan::shard::k_carry_plus<double><<<1, 32, 0, s>>>((const double*)carry_in, (const double*)arr, nfull,
                                                               (double*)carry);
        else
            scan::shard::k_carry_plus<long long><<<1, 32, 0, s>>>((const long long*)carry_in, (const long long*)arr,
                                                                  nfull, (long long*)carry);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        const size_t isz = in_size(dtype);
        st = scan_1d((const uint8_t*)in + nfull * kShardBlk * isz, (uint8_t*)out + nfull * kShardBlk * 4, tail, dtype,
                     carry, ws, shard_base(dtype, n), stream, exclusive);
    }
    return st;
}

int scan_widen_copy(const void* in, void* out, int64_t n, int dtype, void* stream)
{
    if (!valid_dt(dtype) || n < 0) return SCAN_ERR_ARG;
    if (n == 0) return SCAN_OK;
    if (in == nullptr || out == nullptr || ((uintptr_t)in & 15u) || ((uintptr_t)out & 15u)) return SCAN_ERR_ARG;
    DevInfo di;
    int st = dev_info(di);
    if (st != SCAN_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    const unsigned g = (unsigned)di.sms * 8;
    switch (dtype) {
    case SCAN_I32_I32: scan::ceiling::k_widen_copy<SCAN_I32_I32><<<g, 256, 0, s>>>(in, out, n); break;
    case SCAN_F32_F32: scan::ceiling::k_widen_copy<SCAN_F32_F32><<<g, 256, 0, s>>>(in, out, n); break;
    case SCAN_F16_F32: scan::ceiling::k_widen_copy<SCAN_F16_F32><<<g, 256, 0, s>>>(in, out, n); break;
    default: scan::ceiling::k_widen_copy<SCAN_I8_I32><<<g, 256, 0, s>>>(in, out, n); break;
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError() == cudaSuccess ? SCAN_OK : SCAN_ERR_CUDA;
}

}  // extern "C"

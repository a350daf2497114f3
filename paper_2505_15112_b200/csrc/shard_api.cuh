// shard_api.cuh -- C ABI of the two-pass sharded scan (include/scan.h:
// scan_shard_workspace_bytes / scan_shard_reduce / scan_shard_scan), compiled
// into scan_api.cu's translation unit.  Host code only.
#pragma once
#include "shard.cuh"

namespace {

constexpr int64_t kShardBlk = 131072;       // elements per block = one row of pass 2
constexpr size_t kShardDone = 192;          // done counter inside the zeroed header block
constexpr size_t kShardPeerCarry = 216;     // device-initiated exchange: the carry of the lower ranks (8 B)

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

}  // extern "C"

namespace {

int shard_reduce_impl(const void* in, int64_t n, int dtype, void* total_out, void* ws, size_t ws_bytes, void* stream,
                      scan::shard::PeerPub pub)
{
    if (!valid_dt(dtype) || n < 0 || total_out == nullptr) return SCAN_ERR_ARG;
    if (n > 0 && in == nullptr) return SCAN_ERR_ARG;
    if (ws == nullptr || ((uintptr_t)ws & 255u) != 0 || ws_bytes < scan_shard_workspace_bytes(dtype, n))
        return SCAN_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    if (n == 0) {
        if (cudaMemsetAsync(total_out, 0, 8, s) != cudaSuccess) return SCAN_ERR_CUDA;
        if (pub.peers != nullptr) {
            scan::shard::k_publish_zero<<<1, 32, 0, s>>>(pub);
            g_launches.fetch_add(1, std::memory_order_relaxed);
            if (cudaGetLastError() != cudaSuccess) return SCAN_ERR_CUDA;
        }
        return SCAN_OK;
    }
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
                                                           done, pub);                                           \
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

struct PeerSlots {
    const uint64_t* slots;  // NULL: carry_in as given
    int G, rank;
    uint32_t epoch;
};

int shard_scan_impl(const void* in, void* out, int64_t n, int dtype, int exclusive, const void* carry_in, void* ws,
                    size_t ws_bytes, void* stream, PeerSlots ps)
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
    const int64_t nb = (n + kShardBlk - 1) / kShardBlk, nfull = n / kShardBlk, tail = n % kShardBlk;
    uint8_t* w = (uint8_t*)ws;
    uint8_t* arr = w + shard_base(dtype, n);
    const bool rows_path = aligned && in != out && nfull > 0;
    if (ps.slots != nullptr) {
        // device-initiated exchange: the carry of the lower ranks comes from this
        // rank's slot array -- waited for inside the row kernel, or (no row
        // kernel) by one warp before the 1-D scan; either way it lands in the
        // workspace header for the tail / fallback scan
        void* pc = w + kShardPeerCarry;
        if (!rows_path) {
            if (is_float(dtype))
                scan::shard::k_carry_from_slots<double><<<1, 32, 0, s>>>(ps.slots, ps.G, ps.rank, ps.epoch, (double*)pc);
            else
                scan::shard::k_carry_from_slots<long long><<<1, 32, 0, s>>>(ps.slots, ps.G, ps.rank, ps.epoch,
                                                                            (long long*)pc);
            g_launches.fetch_add(1, std::memory_order_relaxed);
            if (cudaGetLastError() != cudaSuccess) return SCAN_ERR_CUDA;
        }
        carry_in = pc;
    }
    if (!aligned || in == out)  // no row view: the single-pass scan with the carry (block sums unused)
        return scan_1d(in, out, n, dtype, carry_in, ws, ws_bytes, stream, exclusive);
    if (nfull > 0) {  // pass 2: every block a row starting from carry_in + pre[block]
        ScanParams p{};
        p.in = in;
        p.out = out;
        p.seg_len = kShardBlk;
        p.num_segs = nfull;
        p.in_stride = kShardBlk;
        p.out_stride = kShardBlk;
        p.carry_in = ps.slots ? nullptr : carry_in;
        p.row_pre = arr;
        p.ws = w;
        if (ps.slots != nullptr) {
            p.peer_slots = ps.slots;
            p.peer_G = ps.G;
            p.peer_rank = ps.rank;
            p.peer_epoch = ps.epoch;
            p.carry_out = w + kShardPeerCarry;  // for the tail
        }
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

}  // namespace

extern "C" {

int scan_shard_reduce(const void* in, int64_t n, int dtype, void* total_out, void* ws, size_t ws_bytes, void* stream)
{
    return shard_reduce_impl(in, n, dtype, total_out, ws, ws_bytes, stream, scan::shard::PeerPub{nullptr, 0, 0, 0});
}

int scan_shard_scan(const void* in, void* out, int64_t n, int dtype, int exclusive, const void* carry_in, void* ws,
                    size_t ws_bytes, void* stream)
{
    return shard_scan_impl(in, out, n, dtype, exclusive, carry_in, ws, ws_bytes, stream, PeerSlots{nullptr, 0, 0, 0});
}

size_t scan_peer_slots_bytes(int G)
{
    if (G < 1 || G > 32) return 0;
    return (size_t)scan::shard::kPeerRing * (size_t)G * 16;
}

int scan_shard_reduce_publish(const void* in, int64_t n, int dtype, void* total_out, void* const* peer_slots, int G,
                              int rank, uint32_t epoch, void* ws, size_t ws_bytes, void* stream)
{
    if (peer_slots == nullptr || G < 1 || G > 32 || rank < 0 || rank >= G || epoch == 0) return SCAN_ERR_ARG;
    return shard_reduce_impl(in, n, dtype, total_out, ws, ws_bytes, stream,
                             scan::shard::PeerPub{reinterpret_cast<uint64_t* const*>(peer_slots), G, rank, epoch});
}

int scan_shard_scan_peers(const void* in, void* out, int64_t n, int dtype, int exclusive, const void* slots, int G,
                          int rank, uint32_t epoch, void* ws, size_t ws_bytes, void* stream)
{
    if (slots == nullptr || G < 1 || G > 32 || rank < 0 || rank >= G || epoch == 0) return SCAN_ERR_ARG;
    return shard_scan_impl(in, out, n, dtype, exclusive, nullptr, ws, ws_bytes, stream,
                           PeerSlots{reinterpret_cast<const uint64_t*>(slots), G, rank, epoch});
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

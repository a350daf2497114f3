// ops_api.cuh -- C ABI of include/scan_ops.h (split / compress / radix sort),
// compiled into scan_api.cu's translation unit so it shares its device cache
// and launch counter.  Host code only: argument checks and launches.
#pragma once
#include "../../include/scan_ops.h"
#include "sample.cuh"
#include "topp.cuh"
#include "split.cuh"
#include "split_warp.cuh"
#include "radix.cuh"

namespace {

using scan::split::SplitParams;
using scan::split::kThreads;
using scan::split::kTile;
using scan::radix::DigitParams;

constexpr size_t kSplitHdr = 128;              // split header inside the scan header block
constexpr size_t kSplitArrays = kWsDescOffset;  // counts[ntiles] then offs[ntiles]

int64_t split_tiles(int64_t n) { return (n + kTile - 1) / kTile; }

int64_t split_tiles4(int64_t n) { return (split_tiles(n) + 3) & ~(int64_t)3; }  // 16-byte aligned arrays

int64_t split_wtiles(int64_t n) { return (n + scan::splitw::kWT - 1) / scan::splitw::kWT; }

size_t split_ws_bytes(int64_t n)
{
    // block kernel: counts + offs per 8192-tile; warp kernel: counts + loff per
    // 4096-element warp tile + the CTA totals (<= 4096 CTAs)
    const size_t a = (size_t)split_tiles4(n) * 8;
    const size_t b = (size_t)((split_wtiles(n) + 3) & ~(int64_t)3) * 8 + 4096 * 4;
    const size_t c = (size_t)((n + scan::splitw::kSpWT - 1) / scan::splitw::kSpWT) * 8;  // single-pass compress
    const size_t ab = a > b ? a : b;
    return kSplitArrays + (ab > c ? ab : c) + 64;
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

bool overlap(const void* a, size_t na, const void* b, size_t nb)
{
    const uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
    return x < y + nb && y < x + na;
}

template <int SRC, int ES, int KT, bool IDX_IN>
int launch_split_t(SplitParams& p, cudaStream_t s, const DevInfo& di)
{
    using namespace scan::split;
    const size_t smem = (size_t)kTile * (ES + 4);
    static DevOnce once;
    static cudaError_t err = cudaSuccess;
    static int occ = 1;
    dev_call_once(once, [smem] {
        err = cudaFuncSetAttribute(k_split_scatter<SRC, ES, KT, IDX_IN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem);
        if (err == cudaSuccess &&
            (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_split_scatter<SRC, ES, KT, IDX_IN>, kThreads, smem) !=
                 cudaSuccess ||
             occ < 1))
            occ = 1;
    });
    if (err != cudaSuccess) return SCAN_ERR_CUDA;
    // count: a warp per tile, up to 4 CTAs per SM; scatter: every resident CTA slot
    const int64_t want_count = ((int64_t)p.ntiles + kWarps - 1) / kWarps;
    const int64_t g_count = (int64_t)di.sms * 4 < want_count ? (int64_t)di.sms * 4 : want_count;
    const int64_t g_scat = (int64_t)di.sms * occ < p.ntiles ? (int64_t)di.sms * occ : p.ntiles;
    k_split_count<SRC, ES, KT><<<(unsigned)g_count, kThreads, 0, s>>>(p);
    k_split_scatter<SRC, ES, KT, IDX_IN><<<(unsigned)g_scat, kThreads, smem, s>>>(p);
    g_launches.fetch_add(2, std::memory_order_relaxed);
    return cudaGetLastError() == cudaSuccess ? SCAN_OK : SCAN_ERR_CUDA;
}

// TMA-ring scatter (split.cuh k_split_scatter_tma): aligned buffers, ES <= 4.
template <int SRC, int ES, int KT, bool IDX_IN, bool CMP>
int launch_split_tma_c(SplitParams& p, cudaStream_t s, const DevInfo& di)
{
    using namespace scan::split;
    using C = TmaCfg<SRC, ES, IDX_IN>;
    static DevOnce once;
    static cudaError_t err = cudaSuccess;
    dev_call_once(once, [] {
        err = cudaFuncSetAttribute(k_split_scatter_tma<SRC, ES, KT, IDX_IN, CMP>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem);
    });
    if (err != cudaSuccess) return SCAN_ERR_CUDA;
    const int64_t want_count = ((int64_t)p.ntiles + kWarps - 1) / kWarps;
    const int64_t g_count = (int64_t)di.sms * 4 < want_count ? (int64_t)di.sms * 4 : want_count;
    const int64_t g_scat = (int64_t)di.sms * C::kCtas < p.ntiles ? (int64_t)di.sms * C::kCtas : p.ntiles;
    k_split_count<SRC, ES, KT><<<(unsigned)g_count, kThreads, 0, s>>>(p);
    k_split_scatter_tma<SRC, ES, KT, IDX_IN, CMP><<<(unsigned)g_scat, C::kThreadsT, C::kSmem, s>>>(p);
    g_launches.fetch_add(2, std::memory_order_relaxed);
    return cudaGetLastError() == cudaSuccess ? SCAN_OK : SCAN_ERR_CUDA;
}

template <int SRC, int ES, int KT, bool IDX_IN>
int launch_split_tma(SplitParams& p, cudaStream_t s, const DevInfo& di)
{
    if constexpr (SRC == scan::split::SRC_FLAGS && !IDX_IN)
        if (p.compress) return launch_split_tma_c<SRC, ES, KT, IDX_IN, true>(p, s, di);
    return launch_split_tma_c<SRC, ES, KT, IDX_IN, false>(p, s, di);
}

// Warp-granular split / compress (split_warp.cuh): int8 flags, 1- or 2-byte
// payload, 16-byte aligned buffers.
template <int ES>
int launch_split_warp(const SplitParams& sp, cudaStream_t s, const DevInfo& di)
{
    using namespace scan::splitw;  // (kThreads qualified: split::kThreads is also visible)
    WParams p;
    memset(&p, 0, sizeof(p));
    p.x = sp.x;
    p.z = sp.z;
    p.flags = sp.flags;
    p.idx_out = sp.idx_out;
    p.count_out = sp.count_out;
    p.hdr = sp.hdr;
    p.n = sp.n;
    p.nwt = (int)split_wtiles(sp.n);
    p.compress = sp.compress;
    uint32_t* arr = sp.counts;  // the split workspace arrays region
    const int64_t nwt4 = (p.nwt + 3) & ~3;
    p.counts = arr;
    p.loff = arr + nwt4;
    p.cta_tot = arr + 2 * nwt4;
    int grid = di.sms * 4;
    if (grid > 4096) grid = 4096;
    p.wpc = (p.nwt + grid - 1) / grid;
    grid = (p.nwt + p.wpc - 1) / p.wpc;
    if (sp.compress && sp.idx_out == nullptr && getenv("SCAN_SPLIT_DIRECT") == nullptr &&
        env_int("SCAN_COMPRESS_SP", 0)) {
        // A/B only (DESIGN 5.6): single pass, decoupled look-back over 2048-element
        // warp tiles -- 2.2x slower than the two passes (look-back distance ~ tiles in flight)
        const int64_t nwt2 = (sp.n + kSpWT - 1) / kSpWT;
        uint64_t* desc = reinterpret_cast<uint64_t*>(sp.counts);
        unsigned* ticket = sp.hdr + 4;
        if (cudaMemsetAsync(desc, 0, (size_t)nwt2 * 8, s) != cudaSuccess || cudaMemsetAsync(ticket, 0, 4, s) != cudaSuccess)
            return SCAN_ERR_CUDA;
        constexpr size_t smem = compress_sp_smem_bytes<ES>();
        if (cudaFuncSetAttribute(k_compress_sp<ES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return SCAN_ERR_CUDA;
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_compress_sp<ES>, kSpThreads, smem) != cudaSuccess ||
            occ < 1)
            return SCAN_ERR_CUDA;
        const int64_t wantc = (nwt2 + kSpThreads / 32 - 1) / (kSpThreads / 32);
        const int64_t g = (int64_t)di.sms * occ < wantc ? (int64_t)di.sms * occ : wantc;
        k_compress_sp<ES><<<(unsigned)g, kSpThreads, smem, s>>>(p, desc, ticket);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return cudaGetLastError() == cudaSuccess ? SCAN_OK : SCAN_ERR_CUDA;
    }
    k_splitw_count<<<(unsigned)grid, scan::splitw::kThreads, 0, s>>>(p);
    const int64_t want = ((int64_t)p.nwt + kWarps - 1) / kWarps;
    const int64_t g2 = (int64_t)di.sms * 4 < want ? (int64_t)di.sms * 4 : want;
    auto staged = [&](auto kern, size_t smem, int nt) -> int {
        // staged runs + 16-byte stores; CTAs per SM by shared memory
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return SCAN_ERR_CUDA;
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nt, smem) != cudaSuccess || occ < 1)
            return SCAN_ERR_CUDA;
        const int64_t wantc = ((int64_t)p.nwt + nt / 32 - 1) / (nt / 32);
        const int64_t g3 = (int64_t)di.sms * occ < wantc ? (int64_t)di.sms * occ : wantc;
        kern<<<(unsigned)g3, nt, smem, s>>>(p);
        return SCAN_OK;
    };
    const bool direct = getenv("SCAN_SPLIT_DIRECT") != nullptr;
    int st = SCAN_OK;
    if (p.compress) {
        if (direct) {
            if (p.idx_out) k_splitw_scatter<ES, true, true><<<(unsigned)g2, scan::splitw::kThreads, 0, s>>>(p);
            else k_splitw_scatter<ES, true, false><<<(unsigned)g2, scan::splitw::kThreads, 0, s>>>(p);
        } else if (p.idx_out) {
            st = staged(k_splitw_staged<ES, true, true, 256>, staged_smem_bytes<ES, true, true, 256>(), 256);
        } else {
            st = staged(k_splitw_staged<ES, true, false>, staged_smem_bytes<ES, true, false>(), scan::splitw::kThreads);
        }
    } else {
        if (direct) {
            if (p.idx_out) k_splitw_scatter<ES, false, true><<<(unsigned)g2, scan::splitw::kThreads, 0, s>>>(p);
            else k_splitw_scatter<ES, false, false><<<(unsigned)g2, scan::splitw::kThreads, 0, s>>>(p);
        } else if (p.idx_out) {
            st = staged(k_splitw_staged<ES, false, true, 256>, staged_smem_bytes<ES, false, true, 256>(), 256);
        } else {
            st = staged(k_splitw_staged<ES, false, false, 256>, staged_smem_bytes<ES, false, false, 256>(), 256);
        }
    }
    if (st != SCAN_OK) return st;
    g_launches.fetch_add(2, std::memory_order_relaxed);
    return cudaGetLastError() == cudaSuccess ? SCAN_OK : SCAN_ERR_CUDA;
}

template <int SRC, int ES, int KT>
int launch_split(SplitParams& p, cudaStream_t s, const DevInfo& di)
{
    if constexpr (SRC == scan::split::SRC_FLAGS && ES <= 2) {
        // compress: the warp kernel (50 % vs 40 % of peak at 2^30); split with
        // indices keeps the block kernel (67 % vs 53 %) -- measured, bench_ops.py
        const char* e = getenv("SCAN_SPLIT_WARP");
        const bool warp = e ? atoi(e) != 0 : p.compress != 0;
        if (p.aligned && warp) return launch_split_warp<ES>(p, s, di);
    }
    if constexpr (ES <= 4) {
        if (p.aligned && getenv("SCAN_SPLIT_NO_TMA") == nullptr) {
            if constexpr (SRC == scan::split::SRC_KEYBIT)
                if (p.idx_in) return launch_split_tma<SRC, ES, KT, true>(p, s, di);
            return launch_split_tma<SRC, ES, KT, false>(p, s, di);
        }
    }
    return p.idx_in ? launch_split_t<SRC, ES, KT, true>(p, s, di) : launch_split_t<SRC, ES, KT, false>(p, s, di);
}

template <int KT>
int launch_sort_pass(SplitParams& p, cudaStream_t s, const DevInfo& di)
{
    using namespace scan::split;
    return launch_split<SRC_KEYBIT, (KT <= KEY_F16 ? 2 : 4), KT>(p, s, di);
}

void split_ws_setup(SplitParams& p, void* ws, int64_t n)
{
    uint8_t* w = (uint8_t*)ws;
    p.hdr = reinterpret_cast<uint32_t*>(w + kSplitHdr);
    p.counts = reinterpret_cast<uint32_t*>(w + kSplitArrays);
    p.offs = p.counts + split_tiles4(n);
    p.n = n;
    p.ntiles = (int)split_tiles(n);
}

// LSB radix sort with 8-bit digits (radix.cuh): per pass count -> scan of the
// digit-major counts (this library's exclusive scan) -> stable scatter.
// Row-batched (segmented) form: cols > 0 sorts each of the n / cols rows.
int64_t digit_tiles(int64_t n, int64_t cols)
{
    constexpr int64_t kRT = scan::radix::kTile;
    if (cols > 0) return (n / cols) * ((cols + kRT - 1) / kRT);
    return (n + kRT - 1) / kRT;
}

size_t digit_scan_ws(int64_t n, int64_t cols)
{
    const int64_t nt = digit_tiles(n, cols);
    if (cols > 0) {
        const int64_t tpr = (cols + scan::radix::kTile - 1) / scan::radix::kTile;
        return scan_rows_workspace_bytes(SCAN_I32_I32, n / cols, scan::radix::kDigits * tpr);
    }
    return scan_rows_workspace_bytes(SCAN_I32_I32, scan::radix::kDigits, nt > 0 ? nt : 1);
}

template <int KT, int ES>
int sort_digits(const void* keys, void* keys_out, int32_t* idx_out, int64_t n, int descending, uint8_t* w,
                void* tmp_keys, int32_t* tmp_idx, cudaStream_t s, const DevInfo& di, int64_t cols = 0)
{
    using namespace scan::radix;
    // radix tiles (qualified: split::kTile / kThreads are also visible here)
    constexpr int64_t kRT = scan::radix::kTile;
    constexpr int kRThreads = scan::radix::kThreads;
    auto up = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const int64_t nt = digit_tiles(n, cols);
    const int64_t tpr = cols > 0 ? (cols + kRT - 1) / kRT : 0;
    const int64_t nc = nt * kDigits;
    const size_t scan_ws = up(digit_scan_ws(n, cols));
    uint32_t* counts = reinterpret_cast<uint32_t*>(w + scan_ws);
    uint32_t* offs = reinterpret_cast<uint32_t*>(w + scan_ws + up((size_t)nc * 4));
    uint32_t* dbase = reinterpret_cast<uint32_t*>(w + scan_ws + 2 * up((size_t)nc * 4));
    const size_t smem = (size_t)kRT * (ES + 4);
    static DevOnce once;
    static cudaError_t err = cudaSuccess;
    static int occ = 1;
    dev_call_once(once, [smem] {
        err = cudaFuncSetAttribute(k_digit_scatter<KT, ES, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (err == cudaSuccess)
            err = cudaFuncSetAttribute(k_digit_scatter<KT, ES, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
        if (err == cudaSuccess)
            err = cudaFuncSetAttribute(k_digit_scatter_tma<KT, ES, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)DigitTmaCfg<ES, true>::kSmem);
        if (err == cudaSuccess)
            err = cudaFuncSetAttribute(k_digit_scatter_tma<KT, ES, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)DigitTmaCfg<ES, false>::kSmem);
        if (err == cudaSuccess &&
            (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_digit_scatter<KT, ES, true>, kRThreads, smem) !=
                 cudaSuccess ||
             occ < 1))
            occ = 1;
    });
    if (err != cudaSuccess) return SCAN_ERR_CUDA;
    const int passes = ES * 8 / 8;  // 8-bit digits: 2 for 16-bit keys, 4 for 32-bit keys (even)
    DigitParams p;
    memset(&p, 0, sizeof(p));
    p.counts = counts;
    p.offs = offs;
    p.dbase = dbase;
    p.n = n;
    p.ntiles = (int)nt;
    p.descending = descending != 0;
    p.cols = cols;
    p.tpr = (int)tpr;
    p.count_pf = env_int("SCAN_RADIX_PF", 1);  // measured: row sort 18.65 -> 18.55 ms, fp32 2^26 2.428 -> 2.415 ms
    const int64_t g_count = (int64_t)di.sms * RADIX_COUNT_CTAS < nt ? (int64_t)di.sms * RADIX_COUNT_CTAS : nt;
    const int64_t g_scat = (int64_t)di.sms * occ < nt ? (int64_t)di.sms * occ : nt;
    const void* src_k = keys;
    const int32_t* src_i = nullptr;
    for (int ps = 0; ps < passes; ++ps) {
        p.keys_in = src_k;
        p.idx_in = src_i;
        p.keys_out = (ps & 1) ? keys_out : tmp_keys;
        p.idx_out = (ps & 1) ? idx_out : tmp_idx;
        p.shift = 8 * ps;
        k_digit_count<KT, ES><<<(unsigned)g_count, kRThreads, 0, s>>>(p);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        // per digit, the exclusive scan of its tile counts: 256 rows of ntiles (P437 row scan);
        // segmented: per row, one exclusive scan over its [digit][tile] counts
        int st = cols > 0 ? scan_rows(counts, offs, n / cols, kDigits * tpr, kDigits * tpr, kDigits * tpr, SCAN_I32_I32, 1,
                                      w, scan_ws, s)
                          : scan_rows(counts, offs, kDigits, nt, nt, nt, SCAN_I32_I32, 1, w, scan_ws, s);
        if (st != SCAN_OK) return st;
        const bool tma = aligned16(src_k) && (src_i == nullptr || aligned16(src_i)) && getenv("SCAN_SORT_NO_TMA") == nullptr;
        if (tma) {
            const int64_t ct = src_i ? DigitTmaCfg<ES, true>::kCtas : DigitTmaCfg<ES, false>::kCtas;
            const int64_t g = (int64_t)di.sms * ct < nt ? (int64_t)di.sms * ct : nt;
            if (src_i)
                k_digit_scatter_tma<KT, ES, true><<<(unsigned)g, DigitTmaCfg<ES, true>::kThreadsT,
                                                    DigitTmaCfg<ES, true>::kSmem, s>>>(p);
            else
                k_digit_scatter_tma<KT, ES, false><<<(unsigned)g, DigitTmaCfg<ES, false>::kThreadsT,
                                                     DigitTmaCfg<ES, false>::kSmem, s>>>(p);
        } else if (src_i) {
            k_digit_scatter<KT, ES, true><<<(unsigned)g_scat, kRThreads, smem, s>>>(p);
        } else {
            k_digit_scatter<KT, ES, false><<<(unsigned)g_scat, kRThreads, smem, s>>>(p);
        }
        g_launches.fetch_add(1, std::memory_order_relaxed);
        if (cudaGetLastError() != cudaSuccess) return SCAN_ERR_CUDA;
        src_k = p.keys_out;
        src_i = p.idx_out;
    }
    return SCAN_OK;
}

}  // namespace

extern "C" {

size_t scan_split_workspace_bytes(int64_t n)
{
    if (n < 0) return 0;
    return split_ws_bytes(n);
}

int scan_split(const void* x, const int8_t* flags, void* z, int32_t* idx_out, int64_t n, int elem_bytes,
               int compress, int64_t* count_out, void* ws, size_t ws_bytes, void* stream)
{
    if (n < 0 || n >= ((int64_t)1 << 31)) return SCAN_ERR_ARG;
    if (!(elem_bytes == 1 || elem_bytes == 2 || elem_bytes == 4 || elem_bytes == 8)) return SCAN_ERR_ARG;
    if (ws == nullptr || ((uintptr_t)ws & 255u) != 0 || ws_bytes < split_ws_bytes(n)) return SCAN_ERR_WORKSPACE;
    if (n > 0 && (x == nullptr || flags == nullptr || z == nullptr)) return SCAN_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    if (n == 0) {
        if (count_out && cudaMemsetAsync(count_out, 0, sizeof(int64_t), s) != cudaSuccess) return SCAN_ERR_CUDA;
        return SCAN_OK;
    }
    if (overlap(x, (size_t)n * elem_bytes, z, (size_t)n * elem_bytes)) return SCAN_ERR_ARG;
    DevInfo di;
    int st = dev_info(di);
    if (st != SCAN_OK) return st;
    SplitParams p;
    memset(&p, 0, sizeof(p));
    split_ws_setup(p, ws, n);
    p.x = x;
    p.z = z;
    p.flags = flags;
    p.idx_out = idx_out;
    p.count_out = count_out;
    p.compress = compress != 0;
    p.aligned = aligned16(x) && aligned16(z) && aligned16(flags) && (idx_out == nullptr || aligned16(idx_out));
    using namespace scan::split;
    ws_mark_dirty(ws, split_ws_bytes(n));  // tile counts / offsets sit where look-back descriptors go
    switch (elem_bytes) {
    case 1: return launch_split<SRC_FLAGS, 1, 0>(p, s, di);
    case 2: return launch_split<SRC_FLAGS, 2, 0>(p, s, di);
    case 4: return launch_split<SRC_FLAGS, 4, 0>(p, s, di);
    default: return launch_split<SRC_FLAGS, 8, 0>(p, s, di);
    }
}

// 8-bit-digit sort workspace: [scan ws of the 256*ntiles counts][counts][offs]
size_t digit_ws_bytes(int64_t n, int64_t cols = 0)
{
    auto up = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const int64_t nt = digit_tiles(n, cols);
    const int64_t nc = nt * scan::radix::kDigits;
    return up(digit_scan_ws(n, cols)) + 2 * up((size_t)nc * 4) + up(scan::radix::kDigits * 4);
}

size_t scan_radix_sort_workspace_bytes(int64_t n, int key_type)
{
    if (n < 0 || key_type < SCAN_KEY_U16 || key_type > SCAN_KEY_F32) return 0;
    const size_t es = key_type <= SCAN_KEY_F16 ? 2 : 4;
    auto up = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t a = up(split_ws_bytes(n)), b = up(digit_ws_bytes(n));
    return (a > b ? a : b) + up((size_t)n * es) + up((size_t)n * 4);
}

static int radix_sort_impl(const void* keys, void* keys_out, int32_t* idx_out, int64_t n, int key_type,
                           int descending, void* ws, size_t ws_bytes, void* stream);

int scan_radix_sort(const void* keys, void* keys_out, int32_t* idx_out, int64_t n, int key_type, int descending,
                    void* ws, size_t ws_bytes, void* stream)
{
    const int st = radix_sort_impl(keys, keys_out, idx_out, n, key_type, descending, ws, ws_bytes, stream);
    // counts, offsets and the key / index temporaries sit where look-back
    // descriptors go: the next scan call given this workspace clears them
    if (st == SCAN_OK && n > 0) ws_mark_dirty(ws, scan_radix_sort_workspace_bytes(n, key_type));
    return st;
}

static int radix_sort_impl(const void* keys, void* keys_out, int32_t* idx_out, int64_t n, int key_type,
                           int descending, void* ws, size_t ws_bytes, void* stream)
{
    if (n < 0 || n >= ((int64_t)1 << 31) || key_type < SCAN_KEY_U16 || key_type > SCAN_KEY_F32) return SCAN_ERR_ARG;
    const size_t need = scan_radix_sort_workspace_bytes(n, key_type);
    if (ws == nullptr || ((uintptr_t)ws & 255u) != 0 || ws_bytes < need) return SCAN_ERR_WORKSPACE;
    if (n > 0 && (keys == nullptr || keys_out == nullptr || idx_out == nullptr)) return SCAN_ERR_ARG;
    if (n == 0) return SCAN_OK;
    const int es = key_type <= SCAN_KEY_F16 ? 2 : 4;
    if (overlap(keys, (size_t)n * es, keys_out, (size_t)n * es)) return SCAN_ERR_ARG;
    DevInfo di;
    int st = dev_info(di);
    if (st != SCAN_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    auto up = [](size_t b) { return (b + 255) & ~(size_t)255; };
    uint8_t* w = (uint8_t*)ws;
    const size_t head = up(split_ws_bytes(n)) > up(digit_ws_bytes(n)) ? up(split_ws_bytes(n)) : up(digit_ws_bytes(n));
    void* tmp_keys = w + head;
    int32_t* tmp_idx = reinterpret_cast<int32_t*>(w + head + up((size_t)n * es));
    if (env_int("SCAN_SORT_BITS", 8) != 1) {
        switch (key_type) {
        case SCAN_KEY_U16: return sort_digits<scan::split::KEY_U16, 2>(keys, keys_out, idx_out, n, descending, w, tmp_keys, tmp_idx, s, di);
        case SCAN_KEY_I16: return sort_digits<scan::split::KEY_I16, 2>(keys, keys_out, idx_out, n, descending, w, tmp_keys, tmp_idx, s, di);
        case SCAN_KEY_F16: return sort_digits<scan::split::KEY_F16, 2>(keys, keys_out, idx_out, n, descending, w, tmp_keys, tmp_idx, s, di);
        case SCAN_KEY_U32: return sort_digits<scan::split::KEY_U32, 4>(keys, keys_out, idx_out, n, descending, w, tmp_keys, tmp_idx, s, di);
        case SCAN_KEY_I32: return sort_digits<scan::split::KEY_I32, 4>(keys, keys_out, idx_out, n, descending, w, tmp_keys, tmp_idx, s, di);
        default: return sort_digits<scan::split::KEY_F32, 4>(keys, keys_out, idx_out, n, descending, w, tmp_keys, tmp_idx, s, di);
        }
    }
    const int bits = es * 8;  // even: pass 0 writes tmp, the last pass writes keys_out
    SplitParams p;
    memset(&p, 0, sizeof(p));
    split_ws_setup(p, ws, n);
    p.descending = descending != 0;
    const void* src_k = keys;
    const int32_t* src_i = nullptr;  // pass 0: indices are the positions
    for (int b = 0; b < bits; ++b) {
        void* dk = (b & 1) ? keys_out : tmp_keys;
        int32_t* di_ = (b & 1) ? idx_out : tmp_idx;
        p.x = src_k;
        p.z = dk;
        p.idx_in = src_i;
        p.idx_out = di_;
        p.bit = b;
        p.aligned = aligned16(src_k) && aligned16(dk) && aligned16(di_) && (src_i == nullptr || aligned16(src_i));
        switch (key_type) {
        case SCAN_KEY_U16: st = launch_sort_pass<scan::split::KEY_U16>(p, s, di); break;
        case SCAN_KEY_I16: st = launch_sort_pass<scan::split::KEY_I16>(p, s, di); break;
        case SCAN_KEY_F16: st = launch_sort_pass<scan::split::KEY_F16>(p, s, di); break;
        case SCAN_KEY_U32: st = launch_sort_pass<scan::split::KEY_U32>(p, s, di); break;
        case SCAN_KEY_I32: st = launch_sort_pass<scan::split::KEY_I32>(p, s, di); break;
        default: st = launch_sort_pass<scan::split::KEY_F32>(p, s, di); break;
        }
        if (st != SCAN_OK) return st;
        src_k = dk;
        src_i = di_;
    }
    return SCAN_OK;
}

size_t scan_radix_sort_rows_workspace_bytes(int64_t rows, int64_t cols, int key_type)
{
    if (rows < 0 || cols < 0 || key_type < SCAN_KEY_U16 || key_type > SCAN_KEY_F32) return 0;
    const size_t es = key_type <= SCAN_KEY_F16 ? 2 : 4;
    auto up = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const int64_t n = rows * cols;
    return up(digit_ws_bytes(n, cols > 0 ? cols : 1)) + up((size_t)n * es) + up((size_t)n * 4);
}

int scan_radix_sort_rows(const void* keys, void* keys_out, int32_t* idx_out, int64_t rows, int64_t cols, int key_type,
                         int descending, void* ws, size_t ws_bytes, void* stream)
{
    if (rows < 0 || cols < 0 || cols >= ((int64_t)1 << 31) || key_type < SCAN_KEY_U16 || key_type > SCAN_KEY_F32)
        return SCAN_ERR_ARG;
    if (rows == 0 || cols == 0) return SCAN_OK;
    const int64_t n = rows * cols;
    constexpr int64_t kRT = scan::radix::kTile;
    if (rows * ((cols + kRT - 1) / kRT) >= ((int64_t)1 << 31) || rows * scan::radix::kDigits * ((cols + kRT - 1) / kRT) >
                                                                        ((int64_t)1 << 40))
        return SCAN_ERR_ARG;
    const size_t need = scan_radix_sort_rows_workspace_bytes(rows, cols, key_type);
    if (ws == nullptr || ((uintptr_t)ws & 255u) != 0 || ws_bytes < need) return SCAN_ERR_WORKSPACE;
    if (keys == nullptr || keys_out == nullptr || idx_out == nullptr) return SCAN_ERR_ARG;
    const int es = key_type <= SCAN_KEY_F16 ? 2 : 4;
    if (overlap(keys, (size_t)n * es, keys_out, (size_t)n * es)) return SCAN_ERR_ARG;
    DevInfo di;
    int st = dev_info(di);
    if (st != SCAN_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    auto up = [](size_t b) { return (b + 255) & ~(size_t)255; };
    uint8_t* w = (uint8_t*)ws;
    const size_t head = up(digit_ws_bytes(n, cols));
    void* tmp_keys = w + head;
    int32_t* tmp_idx = reinterpret_cast<int32_t*>(w + head + up((size_t)n * es));
    switch (key_type) {
    case SCAN_KEY_U16: st = sort_digits<scan::split::KEY_U16, 2>(keys, keys_out, idx_out, n, descending, w, tmp_keys, tmp_idx, s, di, cols); break;
    case SCAN_KEY_I16: st = sort_digits<scan::split::KEY_I16, 2>(keys, keys_out, idx_out, n, descending, w, tmp_keys, tmp_idx, s, di, cols); break;
    case SCAN_KEY_F16: st = sort_digits<scan::split::KEY_F16, 2>(keys, keys_out, idx_out, n, descending, w, tmp_keys, tmp_idx, s, di, cols); break;
    case SCAN_KEY_U32: st = sort_digits<scan::split::KEY_U32, 4>(keys, keys_out, idx_out, n, descending, w, tmp_keys, tmp_idx, s, di, cols); break;
    case SCAN_KEY_I32: st = sort_digits<scan::split::KEY_I32, 4>(keys, keys_out, idx_out, n, descending, w, tmp_keys, tmp_idx, s, di, cols); break;
    default: st = sort_digits<scan::split::KEY_F32, 4>(keys, keys_out, idx_out, n, descending, w, tmp_keys, tmp_idx, s, di, cols); break;
    }
    if (st == SCAN_OK) ws_mark_dirty(ws, need);
    return st;
}

int scan_weighted_sample(const float* w, int64_t n, double theta, int64_t* index_out, float* cdf, void* ws,
                         size_t ws_bytes, void* stream)
{
    if (n <= 0 || w == nullptr || index_out == nullptr || cdf == nullptr || !(theta >= 0.0 && theta <= 1.0))
        return SCAN_ERR_ARG;
    int st = scan_1d(w, cdf, n, SCAN_F32_F32, nullptr, ws, ws_bytes, stream, 0);
    if (st != SCAN_OK) return st;
    scan::sample::k_weighted_draw<<<1, scan::sample::kThreads, 0, (cudaStream_t)stream>>>(cdf, n, theta, index_out);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError() == cudaSuccess ? SCAN_OK : SCAN_ERR_CUDA;
}

int scan_top_p_draw(const float* cdf, const int32_t* order, int64_t rows, int64_t cols, int64_t cdf_row_stride,
                    int64_t order_row_stride, float p, const float* u, int64_t* token_out, int32_t* kept_out,
                    void* stream)
{
    if (rows < 0 || cols < 0 || cdf_row_stride < cols || order_row_stride < cols) return SCAN_ERR_ARG;
    if (rows == 0) return SCAN_OK;
    if (cols == 0 || cdf == nullptr || order == nullptr || u == nullptr || token_out == nullptr) return SCAN_ERR_ARG;
    if (rows > 0x7fffffff) return SCAN_ERR_ARG;
    DevInfo di;
    int st = dev_info(di);
    if (st != SCAN_OK) return st;
    scan::sample::k_top_p_draw<<<(unsigned)rows, scan::sample::kThreads, 0, (cudaStream_t)stream>>>(
        cdf, order, cols, cdf_row_stride, order_row_stride, p, u, token_out, kept_out);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError() == cudaSuccess ? SCAN_OK : SCAN_ERR_CUDA;
}

int scan_top_p_sample(const float* probs, int64_t rows, int64_t cols, int64_t row_stride, float p, const float* u,
                      int64_t* token_out, int32_t* kept_out, void* ws, size_t ws_bytes, void* stream)
{
    if (rows < 0 || cols < 0 || row_stride < cols) return SCAN_ERR_ARG;
    if (rows == 0) return SCAN_OK;
    if (cols == 0 || cols >= ((int64_t)1 << 31) || probs == nullptr || u == nullptr || token_out == nullptr)
        return SCAN_ERR_ARG;
    if (ws == nullptr || ((uintptr_t)ws & 255u) != 0 || ws_bytes < kWsDescOffset) return SCAN_ERR_WORKSPACE;
    DevInfo di;
    int st = dev_info(di);
    if (st != SCAN_OK) return st;
    using namespace scan::topp;
    const size_t smem = kSmemBytes;
    static DevOnce once;
    static cudaError_t err = cudaSuccess;
    static int occ = 1;
    dev_call_once(once, [smem] {
        err = cudaFuncSetAttribute(k_top_p, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (err == cudaSuccess &&
            (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_top_p, scan::topp::kThreads, smem) != cudaSuccess || occ < 1))
            occ = 1;
    });
    if (err != cudaSuccess) return SCAN_ERR_CUDA;
    const int per_sm = env_int("SCAN_TOPP_CTAS_PER_SM", occ) < occ ? env_int("SCAN_TOPP_CTAS_PER_SM", occ) : occ;
    const int64_t g = (int64_t)di.sms * per_sm < rows ? (int64_t)di.sms * per_sm : rows;
    // the first pass's candidate window in eighth-octave levels (SCAN_TOPP_W0, 8..106)
    int w0 = env_int("SCAN_TOPP_W0", 98);
    w0 = w0 < 8 ? 8 : (w0 > scan::topp::kLevels ? scan::topp::kLevels : w0);
    // row-ticket counter: in the caller's workspace header
    unsigned* ticket = reinterpret_cast<unsigned*>((uint8_t*)ws + scan::topp::kTicketWsOffset);
    if (cudaMemsetAsync(ticket, 0, sizeof(unsigned), (cudaStream_t)stream) != cudaSuccess) return SCAN_ERR_CUDA;
    // SCAN_TOPP_DBG (timing A/B only, profiles/topp_phase.py): 1 stop every row after the
    // candidate pass, 2 after the level masses, 3 after the level-L sort, 4 skip fallback
    // rows, 5 report why a row left the level path.  SCAN_TOPP_PF: L2 bulk prefetch distance
    // in 32-KB pass iterations, and the next row's start (measured 2-5 %, default 3)
    k_top_p<<<(unsigned)g, scan::topp::kThreads, smem, (cudaStream_t)stream>>>(probs, rows, cols, row_stride, p, u, token_out,
                                                                    kept_out, ticket, env_int("SCAN_TOPP_DBG", 0),
                                                                    env_int("SCAN_TOPP_PF", 3),
                                                                    w0);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError() == cudaSuccess ? SCAN_OK : SCAN_ERR_CUDA;
}

}  // extern "C"

// scan_api.cu -- the C ABI declared in include/scan.h: argument checks,
// path selection and kernel launches.  All arithmetic is in
// scan_kernels.cuh; nothing here touches element data.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <atomic>
#include <mutex>

#include "../../include/scan.h"
#include "scan_kernels.cuh"

using namespace scan;

namespace {

std::atomic<uint64_t> g_launches{0};

// Smallest tile any variant uses: workspaces are sized for it so a workspace
// fits every variant (kernel variants are selectable for tuning).
constexpr int64_t kMinTile = 4096;

struct DevInfo {
    int sms = 0;
    int major = 0;
    bool ok = false;
};

int dev_info(DevInfo& out)
{
    static std::mutex mu;
    static DevInfo cache[64];
    static bool have[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return SCAN_ERR_CUDA;
    std::lock_guard<std::mutex> g(mu);
    if (!have[dev]) {
        DevInfo d;
        if (cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&d.major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess)
            return SCAN_ERR_CUDA;
        d.ok = (d.major == 10);
        cache[dev] = d;
        have[dev] = true;
    }
    out = cache[dev];
    return out.ok ? SCAN_OK : SCAN_ERR_DEVICE;
}

bool valid_dt(int dt) { return dt >= 0 && dt <= 3; }
size_t in_size(int dt) { return dt == SCAN_I32_I32 || dt == SCAN_F32_F32 ? 4 : dt == SCAN_F16_F32 ? 2 : 1; }
size_t out_size(int) { return 4; }
bool is_float(int dt) { return dt == SCAN_F32_F32 || dt == SCAN_F16_F32; }
size_t desc_bytes(int dt) { return is_float(dt) ? 32 : 16; }

int variant()
{
    static int v = [] {
        const char* e = getenv("SCAN_VARIANT");
        return e ? atoi(e) : 0;
    }();
    return v;
}

// ---- one kernel instantiation --------------------------------------------------
template <int DT, int TH, int RW, int ST, int OS, int MB>
struct Variant {
    static constexpr int kTile = TileShape<TH, RW>::kTile;
    static constexpr size_t kSmem = scan_smem_bytes<DT, TH, RW, ST, OS>();

    static int occupancy()
    {
        static std::once_flag once;
        static int occ = 0;
        static cudaError_t err = cudaSuccess;
        std::call_once(once, [] {
            auto kern = k_scan_tiles<DT, TH, RW, ST, OS, MB>;
            err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
            if (err == cudaSuccess)
                err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, TH, kSmem);
        });
        return err == cudaSuccess ? occ : -1;
    }

    static int launch(ScanParams p, cudaStream_t s, const DevInfo& di)
    {
        int occ = occupancy();
        if (occ <= 0) return SCAN_ERR_CUDA;
        p.tiles_per_seg = (p.seg_len + kTile - 1) / kTile;
        p.num_tiles = p.tiles_per_seg * p.num_segs;
        p.static_sched = p.tiles_per_seg == 1;
        int64_t grid = (int64_t)di.sms * occ;
        if (grid > p.num_tiles) grid = p.num_tiles;
        k_scan_tiles<DT, TH, RW, ST, OS, MB><<<(unsigned)grid, TH, kSmem, s>>>(p);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return cudaGetLastError() == cudaSuccess ? SCAN_OK : SCAN_ERR_CUDA;
    }
};

// Tuned per dtype; SCAN_VARIANT selects alternatives.
template <int DT>
int launch_dt(ScanParams p, cudaStream_t s, const DevInfo& di, int64_t& tile)
{
    constexpr bool wide_in = (DT == SCAN_I32_I32 || DT == SCAN_F32_F32);
    switch (variant()) {
    case 1:
        tile = Variant<DT, 256, 8, 2, 1, 2>::kTile;
        return Variant<DT, 256, 8, 2, 1, 2>::launch(p, s, di);
    case 2:
        tile = Variant<DT, 512, 4, 3, 2, 1>::kTile;
        return Variant<DT, 512, 4, 3, 2, 1>::launch(p, s, di);
    case 3:
        tile = Variant<DT, 256, 4, 3, 2, 3>::kTile;
        return Variant<DT, 256, 4, 3, 2, 3>::launch(p, s, di);
    default:
        if constexpr (wide_in) {
            tile = Variant<DT, 512, 4, 2, 1, 2>::kTile;
            return Variant<DT, 512, 4, 2, 1, 2>::launch(p, s, di);
        } else {
            tile = Variant<DT, 512, 4, 3, 1, 2>::kTile;
            return Variant<DT, 512, 4, 3, 1, 2>::launch(p, s, di);
        }
    }
}

int launch_any(int dt, ScanParams p, cudaStream_t s, const DevInfo& di)
{
    int64_t tile = 0;
    switch (dt) {
    case SCAN_I32_I32: return launch_dt<0>(p, s, di, tile);
    case SCAN_F32_F32: return launch_dt<1>(p, s, di, tile);
    case SCAN_F16_F32: return launch_dt<2>(p, s, di, tile);
    case SCAN_I8_I32: return launch_dt<3>(p, s, di, tile);
    }
    return SCAN_ERR_ARG;
}

bool overlaps(const void* a, size_t abytes, const void* b, size_t bbytes)
{
    uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
    return x < y + bbytes && y < x + abytes;
}

int64_t tiles_for(int64_t len) { return (len + kMinTile - 1) / kMinTile; }

int check_ws(int dt, void* ws, size_t ws_bytes, int64_t tiles_needed)
{
    if (ws == nullptr || ((uintptr_t)ws & 255u) != 0) return SCAN_ERR_WORKSPACE;
    if (ws_bytes < kWsDescOffset + (size_t)tiles_needed * desc_bytes(dt)) return SCAN_ERR_WORKSPACE;
    return SCAN_OK;
}

int scan_1d(const void* in, void* out, int64_t n, int dt, const void* carry_in, void* ws,
            size_t ws_bytes, void* stream, int exclusive)
{
    if (!valid_dt(dt) || n < 0) return SCAN_ERR_ARG;
    if (n == 0) return SCAN_OK;
    if (in == nullptr || out == nullptr) return SCAN_ERR_ARG;
    if (in != out && overlaps(in, n * in_size(dt), out, n * out_size(dt))) return SCAN_ERR_ARG;
    if (in == out && in_size(dt) != out_size(dt)) return SCAN_ERR_ARG;
    if (tiles_for(n) > 0x7fffffffLL) return SCAN_ERR_ARG;
    DevInfo di;
    int st = dev_info(di);
    if (st != SCAN_OK) return st;
    if (n > kMinTile) {  // more than one tile of the smallest variant: look-back path
        st = check_ws(dt, ws, ws_bytes, tiles_for(n));
        if (st != SCAN_OK) return st;
    }
    ScanParams p{};
    p.in = in;
    p.out = out;
    p.seg_len = n;
    p.num_segs = 1;
    p.in_stride = n;
    p.out_stride = n;
    p.carry_in = carry_in;
    p.ws = (uint8_t*)ws;
    p.exclusive = exclusive;
    p.tma_in = ((uintptr_t)in & 15u) == 0;
    p.tma_out = ((uintptr_t)out & 15u) == 0;
    return launch_any(dt, p, (cudaStream_t)stream, di);
}

}  // namespace

extern "C" {

int scan_abi_version(void) { return SCAN_ABI_VERSION; }

const char* scan_status_string(int status)
{
    switch (status) {
    case SCAN_OK: return "SCAN_OK";
    case SCAN_ERR_ARG: return "SCAN_ERR_ARG: invalid argument";
    case SCAN_ERR_WORKSPACE: return "SCAN_ERR_WORKSPACE: workspace NULL, misaligned or too small";
    case SCAN_ERR_CUDA: return "SCAN_ERR_CUDA: CUDA call or kernel launch failed";
    case SCAN_ERR_DEVICE: return "SCAN_ERR_DEVICE: current device is not sm_100 (B200)";
    }
    return "unknown scan status";
}

size_t scan_workspace_bytes(int dtype, int64_t n)
{
    if (!valid_dt(dtype) || n < 0) return 0;
    return kWsDescOffset + (size_t)tiles_for(n) * desc_bytes(dtype);
}

size_t scan_rows_workspace_bytes(int dtype, int64_t rows, int64_t cols)
{
    if (!valid_dt(dtype) || rows < 0 || cols < 0) return 0;
    return kWsDescOffset + (size_t)(rows * tiles_for(cols)) * desc_bytes(dtype);
}

int scan_workspace_init(void* ws, size_t ws_bytes, void* stream)
{
    if (ws == nullptr || ((uintptr_t)ws & 255u) != 0 || ws_bytes < kWsDescOffset)
        return SCAN_ERR_WORKSPACE;
    DevInfo di;
    int st = dev_info(di);
    if (st != SCAN_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemsetAsync(ws, 0, ws_bytes, s) != cudaSuccess) return SCAN_ERR_CUDA;
    // capacity in tiles of the float descriptor size (the larger one), so the
    // tag-wrap clear never runs past the buffer for any dtype
    size_t cap = (ws_bytes - kWsDescOffset) / 32;
    if (cap > 0xffffffffull) cap = 0xffffffffull;
    k_ws_init<<<1, 32, 0, s>>>((uint8_t*)ws, (uint32_t)cap);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError() == cudaSuccess ? SCAN_OK : SCAN_ERR_CUDA;
}

int scan_inclusive(const void* in, void* out, int64_t n, int dtype, const void* carry_in,
                   void* ws, size_t ws_bytes, void* stream)
{
    return scan_1d(in, out, n, dtype, carry_in, ws, ws_bytes, stream, 0);
}

int scan_exclusive(const void* in, void* out, int64_t n, int dtype, const void* carry_in,
                   void* ws, size_t ws_bytes, void* stream)
{
    return scan_1d(in, out, n, dtype, carry_in, ws, ws_bytes, stream, 1);
}

int scan_rows(const void* in, void* out, int64_t rows, int64_t cols, int64_t in_row_stride,
              int64_t out_row_stride, int dtype, int exclusive, void* ws, size_t ws_bytes,
              void* stream)
{
    if (!valid_dt(dtype) || rows < 0 || cols < 0) return SCAN_ERR_ARG;
    if (rows == 0 || cols == 0) return SCAN_OK;
    if (in == nullptr || out == nullptr) return SCAN_ERR_ARG;
    if (in_row_stride < cols || out_row_stride < cols) return SCAN_ERR_ARG;
    size_t ib = ((size_t)(rows - 1) * in_row_stride + cols) * in_size(dtype);
    size_t ob = ((size_t)(rows - 1) * out_row_stride + cols) * out_size(dtype);
    if (in == out) {
        if (in_size(dtype) != out_size(dtype) || in_row_stride != out_row_stride) return SCAN_ERR_ARG;
    } else if (overlaps(in, ib, out, ob)) {
        return SCAN_ERR_ARG;
    }
    if (rows * tiles_for(cols) > 0x7fffffffLL) return SCAN_ERR_ARG;
    DevInfo di;
    int st = dev_info(di);
    if (st != SCAN_OK) return st;
    if (cols > kMinTile) {
        st = check_ws(dtype, ws, ws_bytes, rows * tiles_for(cols));
        if (st != SCAN_OK) return st;
    }
    ScanParams p{};
    p.in = in;
    p.out = out;
    p.seg_len = cols;
    p.num_segs = rows;
    p.in_stride = in_row_stride;
    p.out_stride = out_row_stride;
    p.carry_in = nullptr;
    p.ws = (uint8_t*)ws;
    p.exclusive = exclusive ? 1 : 0;
    p.tma_in = ((uintptr_t)in & 15u) == 0 && ((in_row_stride * (int64_t)in_size(dtype)) & 15) == 0;
    p.tma_out = ((uintptr_t)out & 15u) == 0 && ((out_row_stride * 4) & 15) == 0;
    return launch_any(dtype, p, (cudaStream_t)stream, di);
}

int scan_total(const void* in, int64_t n, int dtype, void* total_out, void* ws, size_t ws_bytes,
               void* stream)
{
    if (!valid_dt(dtype) || n < 0 || total_out == nullptr) return SCAN_ERR_ARG;
    if (n > 0 && in == nullptr) return SCAN_ERR_ARG;
    DevInfo di;
    int st = dev_info(di);
    if (st != SCAN_OK) return st;
    if (ws == nullptr || ((uintptr_t)ws & 255u) != 0 || ws_bytes < kWsDescOffset)
        return SCAN_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    constexpr int TH = 512;
    int64_t grid = (n + TH * 16 - 1) / (TH * 16);
    int64_t max_grid = (int64_t)di.sms * 4;
    if (grid > max_grid) grid = max_grid;
    if (grid > kMaxTotalCtas) grid = kMaxTotalCtas;
    if (grid < 1) grid = 1;
    uint8_t* w = (uint8_t*)ws;
    switch (dtype) {
    case SCAN_I32_I32: k_total<0, TH><<<(unsigned)grid, TH, 0, s>>>(in, n, total_out, w); break;
    case SCAN_F32_F32: k_total<1, TH><<<(unsigned)grid, TH, 0, s>>>(in, n, total_out, w); break;
    case SCAN_F16_F32: k_total<2, TH><<<(unsigned)grid, TH, 0, s>>>(in, n, total_out, w); break;
    case SCAN_I8_I32: k_total<3, TH><<<(unsigned)grid, TH, 0, s>>>(in, n, total_out, w); break;
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError() == cudaSuccess ? SCAN_OK : SCAN_ERR_CUDA;
}

int scan_carry_from_totals(const void* totals, int G, int rank, int dtype, void* carry_out,
                           void* stream)
{
    if (!valid_dt(dtype) || G < 1 || rank < 0 || rank >= G || carry_out == nullptr ||
        totals == nullptr)
        return SCAN_ERR_ARG;
    DevInfo di;
    int st = dev_info(di);
    if (st != SCAN_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    if (is_float(dtype))
        k_carry_from_totals<double><<<1, 32, 0, s>>>((const double*)totals, rank, (double*)carry_out);
    else
        k_carry_from_totals<long long>
            <<<1, 32, 0, s>>>((const long long*)totals, rank, (long long*)carry_out);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError() == cudaSuccess ? SCAN_OK : SCAN_ERR_CUDA;
}

uint64_t scan_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

}  // extern "C"

// scan_api.cu -- the C ABI declared in include/scan.h: argument checks,
// path selection and kernel launches.  All arithmetic is in
// scan_kernels.cuh; nothing here touches element data.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <mutex>
#include <type_traits>

#include "../../include/scan.h"
#include "scan_kernels.cuh"
#include "scan_ws.cuh"
#include "mcscan.cuh"
#include "rowscan.cuh"
#include "rowscan_tc.cuh"
#include "rows_small.cuh"

using namespace scan;

namespace {

std::atomic<uint64_t> g_launches{0};

int env_int(const char* name, int dflt);  // tuning / A-B knobs (below)

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
#ifdef SCAN_FUZZ
        if (const char* m = getenv("SCAN_FUZZ_MASK")) {  // fault-injection sites to enable (stress build)
            const uint32_t mask = (uint32_t)strtoul(m, nullptr, 0);
            cudaMemcpyToSymbol(scan::ptx::g_fuzz_mask, &mask, sizeof(mask));
        }
#endif
    }
    out = cache[dev];
    return out.ok ? SCAN_OK : SCAN_ERR_DEVICE;
}

// Per-device one-time setup (cudaFuncSetAttribute is a per-device setting: a
// process that drives several GPUs must set it on each of them).
struct DevOnce {
    std::mutex mu;
    bool done[64] = {};
};

template <class F>
void dev_call_once(DevOnce& o, F&& f)
{
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
    std::lock_guard<std::mutex> g(o.mu);
    if (!o.done[dev]) {
        f();
        o.done[dev] = true;
    }
}

// Workspaces whose descriptor region holds operator scratch (split counts,
// radix temporaries) that a later look-back scan could misread as tagged
// descriptors.  The operators register the range they dirtied; the next scan
// entry point that receives the workspace zeroes it (stream-ordered) before
// launching -- a zero slot never carries a live epoch (epochs are >= 1).
struct DirtyWs {
    uintptr_t base;
    size_t bytes;
};
std::mutex g_dirty_mu;
DirtyWs g_dirty[256];
int g_ndirty = 0;

void ws_mark_dirty(void* ws, size_t bytes)
{
    std::lock_guard<std::mutex> g(g_dirty_mu);
    const uintptr_t b = (uintptr_t)ws;
    for (int i = 0; i < g_ndirty; ++i)
        if (g_dirty[i].base == b) {
            if (bytes > g_dirty[i].bytes) g_dirty[i].bytes = bytes;
            return;
        }
    if (g_ndirty == 256) {  // full: forget the oldest (its owner can re-init it)
        memmove(&g_dirty[0], &g_dirty[1], sizeof(DirtyWs) * 255);
        g_ndirty = 255;
    }
    g_dirty[g_ndirty++] = {b, bytes};
}

// Bytes of `ws` (from its start) to zero before a scan, 0 if clean.
size_t ws_take_dirty(const void* ws, size_t ws_bytes)
{
    std::lock_guard<std::mutex> g(g_dirty_mu);
    const uintptr_t b = (uintptr_t)ws;
    for (int i = 0; i < g_ndirty; ++i)
        if (g_dirty[i].base == b) {
            const size_t d = g_dirty[i].bytes < ws_bytes ? g_dirty[i].bytes : ws_bytes;
            g_dirty[i] = g_dirty[--g_ndirty];
            return d;
        }
    return 0;
}

bool valid_dt(int dt) { return dt >= 0 && dt <= 3; }
size_t in_size(int dt) { return dt == SCAN_I32_I32 || dt == SCAN_F32_F32 ? 4 : dt == SCAN_F16_F32 ? 2 : 1; }
size_t out_size(int) { return 4; }
bool is_float(int dt) { return dt == SCAN_F32_F32 || dt == SCAN_F16_F32; }
size_t desc_bytes(int dt) { return is_float(dt) ? 32 : 16; }

int debug_bits()
{
    static int v = [] {
        const char* e = getenv("SCAN_DEBUG");
        return e ? atoi(e) : 0;
    }();
    return v;
}

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
        static DevOnce once;
        static int occ = 0;
        static cudaError_t err = cudaSuccess;
        dev_call_once(once, [] {
            auto kern = k_scan_tiles<DT, TH, RW, ST, OS, MB>;
            err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
            if (err == cudaSuccess)
                err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, TH, kSmem);
        });
        return err == cudaSuccess ? occ : -1;
    }

    // Small 1-D n (2..16 tiles): one cluster, one tile per CTA, DSMEM carries.
    static int launch_cluster(ScanParams p, cudaStream_t s)
    {
        static DevOnce once;
        static cudaError_t err = cudaSuccess;
        auto kern = k_scan_tiles<DT, TH, RW, ST, OS, MB>;
        dev_call_once(once, [&] {
            err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
            if (err == cudaSuccess)
                err = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        });
        if (err != cudaSuccess) return SCAN_ERR_CUDA;
        p.tiles_per_seg = (p.seg_len + kTile - 1) / kTile;
        p.num_tiles = p.tiles_per_seg;
        p.static_sched = 1;
        p.cluster = (int)p.num_tiles;
        p.cl_push = env_int("SCAN_CLUSTER_PUSH", 1);  // measured: C1 3.5 -> 3.2 us per scan
        p.debug = 0;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)p.num_tiles);
        cfg.blockDim = dim3(TH);
        cfg.dynamicSmemBytes = kSmem;
        cfg.stream = s;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)p.num_tiles;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        // programmatic dependent launch: this (latency-bound) launch overlaps the
        // tail of the previous kernel in the stream; the kernel waits for it
        // (griddepcontrol.wait) before touching global memory
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = env_int("SCAN_PDL", 1) ? 2 : 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return e == cudaSuccess ? SCAN_OK : SCAN_ERR_CUDA;
    }

    static int launch(ScanParams p, cudaStream_t s, const DevInfo& di)
    {
        int occ = occupancy();
        if (occ <= 0) return SCAN_ERR_CUDA;
        p.tiles_per_seg = (p.seg_len + kTile - 1) / kTile;
        p.num_tiles = p.tiles_per_seg * p.num_segs;
        p.static_sched = p.tiles_per_seg == 1;
        p.cluster = 0;
        p.debug = debug_bits();
        int64_t grid = (int64_t)di.sms * occ;
        if (grid > p.num_tiles) grid = p.num_tiles;
        if (grid <= di.sms && env_int("SCAN_PDL", 1)) {
            // one wave of a latency-bound launch: programmatic dependent launch, as
            // for the cluster path (the kernel waits before touching global memory)
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)grid);
            cfg.blockDim = dim3(TH);
            cfg.dynamicSmemBytes = kSmem;
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            const cudaError_t e = cudaLaunchKernelEx(&cfg, k_scan_tiles<DT, TH, RW, ST, OS, MB>, p);
            g_launches.fetch_add(1, std::memory_order_relaxed);
            return e == cudaSuccess ? SCAN_OK : SCAN_ERR_CUDA;
        }
        k_scan_tiles<DT, TH, RW, ST, OS, MB><<<(unsigned)grid, TH, kSmem, s>>>(p);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return cudaGetLastError() == cudaSuccess ? SCAN_OK : SCAN_ERR_CUDA;
    }
};

// Warp-specialized multi-tile kernel (scan_ws.cuh): one CTA per SM.
template <int DT, int NC, int NL, int RW, int NBI, int NBO>
struct WsVariant {
    using Cfg = WsCfg<DT, NC, NL, RW, NBI, NBO>;
    static constexpr int kTile = Cfg::kTile;

    static int ready()
    {
        static DevOnce once;
        static cudaError_t err = cudaSuccess;
        dev_call_once(once, [] {
            err = cudaFuncSetAttribute(k_scan_ws<DT, NC, NL, RW, NBI, NBO>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmem);
        });
        return err == cudaSuccess;
    }

    static int launch(ScanParams p, cudaStream_t s, const DevInfo& di)
    {
        if (!ready()) return SCAN_ERR_CUDA;
        p.tiles_per_seg = (p.seg_len + kTile - 1) / kTile;
        p.num_tiles = p.tiles_per_seg * p.num_segs;
        p.static_sched = 0;
        p.debug = debug_bits();
        int64_t grid = di.sms;
        if (grid > p.num_tiles) grid = p.num_tiles;
        k_scan_ws<DT, NC, NL, RW, NBI, NBO><<<(unsigned)grid, Cfg::kThreads, Cfg::kSmem, s>>>(p);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return cudaGetLastError() == cudaSuccess ? SCAN_OK : SCAN_ERR_CUDA;
    }
};

// Persistent cooperative MCScan with L2 splitting (mcscan.cuh): 1-D scans.
int env_int(const char* name, int dflt)
{
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}

constexpr int kMaxGrid = 192;
constexpr size_t kWsHeadCarry = 208;  // header pad: the body carry of an unaligned 1-D scan (8 B)  // workspace sizing bound on the CTA count (B200: 148)
constexpr int64_t kMcMinElems = 1 << 20;  // below this the look-back kernel wins (one chunk)

// ---- TMA tensor maps (driver entry point, no libcuda link dependency) ----------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn()
{
    static EncodeTiledFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (EncodeTiledFn) nullptr;
        return (EncodeTiledFn)f;
    }();
    return fn;
}

// [rows x 128 B] view of a 16-byte-aligned array, 256-row boxes, 128 B swizzle.
bool encode_rows128(CUtensorMap* tm, const void* base, int64_t rows, int elem_bytes, int box_rows)
{
    EncodeTiledFn fn = encode_fn();
    if (!fn || rows < 1) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)(128 / elem_bytes), (cuuint64_t)rows};
    const cuuint64_t strides[1] = {128};
    const cuuint32_t box[2] = {(cuuint32_t)(128 / elem_bytes), (cuuint32_t)box_rows};
    const cuuint32_t es[2] = {1, 1};
    const CUtensorMapDataType dt = elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_UINT16;
    return fn(tm, dt, 2, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Second-generation MCScan: 16 contiguous elements per lane (mcscan16.cuh).
template <int DT, int NC, int GPW, int NBI, int NBO, bool SEG = false, int SH = 0>
struct Mc16Variant {
    static constexpr bool SHIFT = SH > 0;
    using Cfg = Mc16Cfg<DT, NC, GPW, NBI, NBO, SHIFT>;
    static constexpr int kTile = Cfg::kTile;

    // segmented: sp's contiguous rows as one segmented scan (row length a whole
    // number of tiles; carries reset at row starts).
    static int launch(const ScanParams& sp, cudaStream_t s, const DevInfo& di, int bt, int ahead)
    {
        constexpr bool segmented = SEG;
        using In = typename Traits<DT>::In;
        if constexpr (Cfg::kSmem > 232448) return SCAN_ERR_ARG;  // tuning variant does not fit this dtype
        // segmented: rows of >= one tile (at most one row start per tile); the
        // in-place ring would let a split tile's first pass overwrite its inputs
        if (segmented && (sp.seg_len < kTile || Cfg::kUni)) return SCAN_ERR_ARG;
        static DevOnce once;
        static cudaError_t err = cudaSuccess;
        dev_call_once(once, [] {
            err = cudaFuncSetAttribute(k_mcscan16<DT, NC, GPW, NBI, NBO, SEG, SH>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmem);
        });
        if (err != cudaSuccess) return SCAN_ERR_CUDA;
        McParams16 p;
        memset(&p, 0, sizeof(p));
        const int64_t n = segmented ? sp.seg_len * sp.num_segs : sp.seg_len;
        const int64_t rows_out = n / 32;
        if (!encode_rows128(&p.tm_out, sp.out, rows_out, 4, Cfg::kBoxRowsOut)) return SCAN_ERR_CUDA;
        // SHIFT: the input views start at the 16-byte boundary `d` elements below
        // `in`; n_tma_in counts the elements of `in` those views cover
        const int d = SHIFT ? sp.shift : 0;
        const void* in_al = (const uint8_t*)sp.in - (int64_t)d * (int64_t)sizeof(In);
        p.shift = d;
        if constexpr (sizeof(In) == 1) {
            p.n_tma_in = ((n + d) & ~(int64_t)15) - d;
        } else {
            const int64_t rows_in = (n + d) / Cfg::kRowElemsIn;
            if (!encode_rows128(&p.tm_in, in_al, rows_in, (int)sizeof(In), Cfg::kBoxRowsIn)) return SCAN_ERR_CUDA;
            if (SHIFT && !encode_rows128(&p.tm_in1, in_al, rows_in, (int)sizeof(In), 1)) return SCAN_ERR_CUDA;
            p.n_tma_in = rows_in * Cfg::kRowElemsIn - d;
        }
        p.n_tma_out = rows_out * 32;
        p.in = sp.in;
        p.out = sp.out;
        p.carry_in = sp.carry_in;
        p.ws = sp.ws;
        p.exclusive = sp.exclusive;
        p.debug = debug_bits();
        p.ahead = ahead < 1 ? 1 : (ahead > 4 ? 4 : ahead);
        // L2 policy of the Phase-I read: evict_last for 1- and 2-byte inputs; 4-byte
        // inputs take evict_normal (bit 0) since the lighter compute path (DESIGN 8.1:
        // C5 burst 90.6 -> 91.9 %, sustained 91.7 -> 91.5 %; C2 / C3 lose 0.4-0.6 with it)
        p.l2 = env_int("SCAN_MC_L2", sizeof(In) == 4 ? 1 : 0);
        // mbarrier waits (measured, DESIGN 5.1): the producer / storer sleep in
        // the barrier unit instead of spinning, and for 1- and 2-byte inputs (more
        // instructions per byte) the compute warps too; SCAN_MC_WAIT overrides
        p.wait_mode = env_int("SCAN_MC_WAIT", sizeof(In) < 4 ? 3 : 1);
        p.bar_mode = env_int("SCAN_MC_BAR", 0);
        p.lazy_carry = env_int("SCAN_MC_LAZY", 0);  // A/B: measured +1.8 points at ahead 1, none at the default
        p.seg_len = segmented ? sp.seg_len : 0;
        p.gm.n = n;
        p.gm.g = di.sms < kMaxGrid ? di.sms : kMaxGrid;
        const int64_t ntiles = (n + kTile - 1) / kTile;
        int64_t lim = n < p.n_tma_in ? n : p.n_tma_in;
        lim = lim < p.n_tma_out ? lim : p.n_tma_out;
        p.gm.ntiles = (int)ntiles;
        p.gm.full_tiles = (int)(lim / kTile);
        const int64_t per_cta = (ntiles + p.gm.g - 1) / p.gm.g;
        int64_t bt64 = bt < per_cta ? bt : (per_cta < 1 ? 1 : per_cta);
        if ((ntiles + (int64_t)p.gm.g * bt64 - 1) / ((int64_t)p.gm.g * bt64) > kMaxChunks)  // counters must fit
            bt64 = (ntiles + (int64_t)kMaxChunks * p.gm.g - 1) / ((int64_t)kMaxChunks * p.gm.g);
        p.gm.bt = (int)bt64;
        p.gm.chunk_tiles = p.gm.g * p.gm.bt;
        p.gm.chunks = (int)((ntiles + p.gm.chunk_tiles - 1) / p.gm.chunk_tiles);
        void* args[] = {&p};
        cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_mcscan16<DT, NC, GPW, NBI, NBO, SEG, SH>,
                                                    dim3(p.gm.g), dim3(Cfg::kThreads), args, Cfg::kSmem, s);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return e == cudaSuccess ? SCAN_OK : SCAN_ERR_CUDA;
    }
};

// Workspace bytes the MCScan path needs for n elements (tile >= 8192, bt >= 1):
// r[c][b] (8 B) per block; barrier counters live in the fixed header region.
size_t mc_workspace_bytes(int64_t n)
{
    const int64_t blocks = (n + 8191) / 8192 + kMaxGrid;  // r[c][b] entries, upper bound
    return kWsDescOffset + (size_t)blocks * 16 + 64;       // up to 2 tagged words each
}

// Chunk = G blocks of bt tiles.  Reductions run `ahead` chunks ahead of the
// scans, so (ahead + 1) chunks of input must stay resident in L2 between
// their HBM read (Phase I) and their re-read (Phase II).  Measured on B200
// (DESIGN.md section 8): the re-read stays in L2 while that footprint is about
// 32 MB (126 MB L2 split over two dies, output streaming through it), and
// bt >= 2 tiles per block keeps the per-chunk coordination (grid barrier,
// 148 block sums per CTA) off the critical path; ahead = 2 absorbs barrier skew.
template <typename V, int DT>
int launch_mc_sized(const ScanParams& p, cudaStream_t s, const DevInfo& di)
{
    using In = typename Traits<DT>::In;
    const int64_t tile_bytes = (int64_t)V::kTile * (int64_t)sizeof(In);
    // int8 inputs (16-KB tiles): reductions one chunk ahead with 4-tile blocks
    // (19 MB resident) -- measured 101.8 % of the copy peak on C3 against 92.6 %
    // at the 4-byte setting (ahead 2, 32 MB); DESIGN 5.1
    // shifted fp16 (4 + 1 ring slots): one chunk ahead, 3-tile blocks -- 82.4 % on
    // C2 x[1:] against 78.4 % at the default
    const bool one_ahead = sizeof(In) == 1 || (V::SHIFT && sizeof(In) == 2);
    const int ahead = env_int("SCAN_MC_AHEAD", one_ahead ? 1 : 2);
    const int64_t resident =
        (int64_t)env_int("SCAN_MC_RESIDENT_MB", sizeof(In) == 1 ? 19 : (one_ahead ? 29 : 32)) << 20;
    const int64_t per_bt = (int64_t)(ahead + 1) * di.sms * tile_bytes;
    int64_t bt = (resident + per_bt / 2) / per_bt;
    bt = bt < 2 ? 2 : bt;
    return V::launch(p, s, di, env_int("SCAN_MC_BT", (int)bt), ahead);
}

// Default variant per dtype (warps, groups per warp, input slots, output slots;
// 0 output slots = outputs in place in the input ring); SCAN_MC selects
// alternatives for tuning runs.
// Shifted-input MCScan (default warp / ring configuration): one instantiation
// per whole-word part of the shift, SH - 1 = (shift * sizeof(In)) / 4.
template <int DT, int SH>
int launch_mc_shift_sh(const ScanParams& p, cudaStream_t s, const DevInfo& di)
{
    constexpr bool wide_in = (DT == SCAN_I32_I32 || DT == SCAN_F32_F32);
    if constexpr (wide_in && SH == 1) {
        return SCAN_ERR_ARG;  // 4-byte elements: a nonzero shift is >= 1 whole word
    } else if constexpr (wide_in) {
        return launch_mc_sized<Mc16Variant<DT, 12, 2, 3, 1, false, SH>, DT>(p, s, di);
    } else if constexpr (DT == SCAN_F16_F32) {
        // the extra rows must fit: 4 input + 1 output slots (measured 74.5 % of peak
        // on C2 x[1:]; 2 + 2 slots: 69 %)
        return launch_mc_sized<Mc16Variant<DT, 16, 2, 4, 1, false, SH>, DT>(p, s, di);
    } else {
        // 5 input + 2 output slots (82 % on C3 x[1:]; 8 + 1: 80 %)
        return launch_mc_sized<Mc16Variant<DT, 16, 2, 5, 2, false, SH>, DT>(p, s, di);
    }
}

template <int DT>
int launch_mc_shift(const ScanParams& p, cudaStream_t s, const DevInfo& di)
{
    using In = typename Traits<DT>::In;
    switch ((p.shift * (int)sizeof(In)) >> 2) {
    case 0: return launch_mc_shift_sh<DT, 1>(p, s, di);
    case 1: return launch_mc_shift_sh<DT, 2>(p, s, di);
    case 2: return launch_mc_shift_sh<DT, 3>(p, s, di);
    default: return launch_mc_shift_sh<DT, 4>(p, s, di);
    }
}

template <int DT>
int launch_mc(const ScanParams& p, cudaStream_t s, const DevInfo& di)
{
    constexpr bool wide_in = (DT == SCAN_I32_I32 || DT == SCAN_F32_F32);
    if (p.shift != 0)  // input not on a 16-byte boundary (the output is): shifted slots
        return launch_mc_shift<DT>(p, s, di);
    switch (env_int("SCAN_MC", 0)) {
    case 1:
        if constexpr (wide_in) return launch_mc_sized<Mc16Variant<DT, 16, 2, 2, 1>, DT>(p, s, di);
        else return launch_mc_sized<Mc16Variant<DT, 16, 2, 4, 2>, DT>(p, s, di);
    case 7: return launch_mc_sized<Mc16Variant<DT, 16, 2, 3, 0>, DT>(p, s, di);   // unified in-place ring
    case 20: {  // A/B: the segmented instantiation on one row
        using V = std::conditional_t<wide_in, Mc16Variant<DT, 12, 2, 3, 1, true>,
                                     std::conditional_t<DT == SCAN_F16_F32, Mc16Variant<DT, 16, 2, 3, 2, true>,
                                                        Mc16Variant<DT, 16, 2, 6, 2, true>>>;
        return launch_mc_sized<V, DT>(p, s, di);
    }
    default:
        if constexpr (wide_in) return launch_mc_sized<Mc16Variant<DT, 12, 2, 3, 1>, DT>(p, s, di);
        else if constexpr (DT == SCAN_F16_F32) return launch_mc_sized<Mc16Variant<DT, 16, 2, 3, 2>, DT>(p, s, di);
        else return launch_mc_sized<Mc16Variant<DT, 16, 2, 6, 2>, DT>(p, s, di);
    }
}

// Few long contiguous rows as ONE segmented MCScan over the whole matrix (rows
// of at least one tile); -1 when the rows are shorter than the variant's tile.
template <int DT>
int launch_mc_rows(const ScanParams& p, cudaStream_t s, const DevInfo& di)
{
    constexpr bool wide_in = (DT == SCAN_I32_I32 || DT == SCAN_F32_F32);
    using V = std::conditional_t<wide_in, Mc16Variant<DT, 12, 2, 3, 1, true>,
                                 std::conditional_t<DT == SCAN_F16_F32, Mc16Variant<DT, 16, 2, 3, 2, true>,
                                                    Mc16Variant<DT, 16, 2, 6, 2, true>>>;
    if (p.seg_len < V::kTile) return -1;
    return launch_mc_sized<V, DT>(p, s, di);
}

// ---- batched rows of many tiles: one CTA per row (rowscan.cuh) -------------------
bool encode_rows3d(CUtensorMap* tm, const void* base, int64_t rows, int64_t cols, int64_t stride_elems,
                   int elem_bytes, int box_rows)
{
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)(128 / elem_bytes), (cuuint64_t)(cols * elem_bytes / 128),
                                (cuuint64_t)rows};
    const cuuint64_t strides[2] = {128, (cuuint64_t)(stride_elems * elem_bytes)};
    const cuuint32_t box[3] = {(cuuint32_t)(128 / elem_bytes), (cuuint32_t)box_rows, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    const CUtensorMapDataType dt = elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_UINT16;
    return fn(tm, dt, 3, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int DT, int NC, int GPW, int NB>
struct RowVariant {
    using Cfg = RowCfg<DT, NC, GPW, NB>;
    static int launch(const ScanParams& sp, cudaStream_t s, const DevInfo& di)
    {
        using In = typename Traits<DT>::In;
        static DevOnce once;
        static cudaError_t err = cudaSuccess;
        dev_call_once(once, [] {
            err = cudaFuncSetAttribute(k_rowscan16<DT, NC, GPW, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)Cfg::kSmem);
        });
        if (err != cudaSuccess) return SCAN_ERR_CUDA;
        RowParams p;
        memset(&p, 0, sizeof(p));
        if constexpr (sizeof(In) != 1) {
            if (!encode_rows3d(&p.tm_in, sp.in, sp.num_segs, sp.seg_len, sp.in_stride, (int)sizeof(In),
                               Cfg::kBoxRowsIn))
                return SCAN_ERR_CUDA;
        }
        if (!encode_rows3d(&p.tm_out, sp.out, sp.num_segs, sp.seg_len, sp.out_stride, 4, Cfg::kBoxRowsOut))
            return SCAN_ERR_CUDA;
        p.in = sp.in;
        p.out = sp.out;
        p.ws = sp.ws;
        p.rows = sp.num_segs;
        p.cols = sp.seg_len;
        p.in_stride = sp.in_stride;
        p.tiles_per_row = (int)((sp.seg_len + Cfg::kTile - 1) / Cfg::kTile);
        p.exclusive = sp.exclusive;
        p.row_pre = sp.row_pre;
        p.carry_in = sp.row_pre ? sp.carry_in : nullptr;
        p.peer_slots = sp.peer_slots;
        p.peer_G = sp.peer_G;
        p.peer_rank = sp.peer_rank;
        p.peer_epoch = sp.peer_epoch;
        p.carry_out = sp.carry_out;
        int64_t grid = di.sms;
        if (grid > sp.num_segs) grid = sp.num_segs;
        k_rowscan16<DT, NC, GPW, NB><<<(unsigned)grid, Cfg::kThreads, Cfg::kSmem, s>>>(p);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return cudaGetLastError() == cudaSuccess ? SCAN_OK : SCAN_ERR_CUDA;
    }
};

template <int DT>
bool rowscan_ok(const ScanParams& p)
{
    using In = typename Traits<DT>::In;
    return p.num_segs > 1 && p.tma_in && p.tma_out && (p.seg_len * (int64_t)sizeof(In)) % 128 == 0 &&
           (p.seg_len * 4) % 128 == 0 && p.num_segs < (1ll << 31) && env_int("SCAN_NO_ROWSCAN", 0) == 0;
}

// Tensor-core local scan (rowscan_tc.cuh), the A/B of SURVEY 8(f) row 2:
// fp16 rows of exactly 16,384 elements, inclusive, selected by SCAN_ROWS_TC=1.
template <int ES>
int launch_rows_tc(const ScanParams& sp, cudaStream_t s, const DevInfo& di)
{
    using Cfg = scan::tc::TcCfg<ES>;
    static DevOnce once;
    static cudaError_t err = cudaSuccess;
    dev_call_once(once, [] {
        err = cudaFuncSetAttribute(scan::tc::k_rowscan_tc<ES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)Cfg::kSmem);
    });
    if (err != cudaSuccess) return SCAN_ERR_CUDA;
    EncodeTiledFn fn = encode_fn();
    if (!fn) return SCAN_ERR_CUDA;
    scan::tc::TcParams p;
    memset(&p, 0, sizeof(p));
    // [rows][128 chunks][128 elements] view, boxes of one 128-byte K block x 128 chunks
    const cuuint64_t dims[3] = {128, 128, (cuuint64_t)sp.num_segs};
    const cuuint64_t strides[2] = {128 * ES, (cuuint64_t)(sp.in_stride * ES)};
    const cuuint32_t box[3] = {128 / ES, 128, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    if (fn(&p.tm_in, ES == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_UINT8, 3,
           const_cast<void*>(sp.in), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return SCAN_ERR_CUDA;
    p.out = sp.out;
    p.rows = sp.num_segs;
    p.out_stride = sp.out_stride;
    const int64_t grid = di.sms < sp.num_segs ? di.sms : sp.num_segs;
    scan::tc::k_rowscan_tc<ES><<<(unsigned)grid, scan::tc::kThreads, Cfg::kSmem, s>>>(p);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError() == cudaSuccess ? SCAN_OK : SCAN_ERR_CUDA;
}

template <int DT>
int launch_rows(const ScanParams& p, cudaStream_t s, const DevInfo& di)
{
    if constexpr (DT == SCAN_F16_F32 || DT == SCAN_I8_I32) {  // tensor-core A/B (SCAN_ROWS_TC=1)
        if (p.seg_len == scan::tc::kCols && !p.exclusive && p.row_pre == nullptr && env_int("SCAN_ROWS_TC", 0) != 0)
            return launch_rows_tc<DT == SCAN_F16_F32 ? 2 : 1>(p, s, di);
    }
    switch (env_int("SCAN_ROWS", 0)) {
    case 1: return RowVariant<DT, 16, 1, 6>::launch(p, s, di);
    case 2: return RowVariant<DT, 16, 2, 2>::launch(p, s, di);
    default: return RowVariant<DT, 16, 2, 3>::launch(p, s, di);
    }
}

// Single-tile-per-segment (static) and tuning-alternative kernels; the default
// path for multi-tile segments is the warp-specialized kernel.  SCAN_VARIANT
// selects alternatives for experiments.
template <int DT>
int launch_rows_small(const ScanParams& sp, cudaStream_t s, const DevInfo& di)
{
    using namespace scan::rows_small;
    SRParams p;
    p.in = sp.in;
    p.out = sp.out;
    p.rows = sp.num_segs;
    p.cols = sp.seg_len;
    p.in_stride = sp.in_stride;
    p.out_stride = sp.out_stride;
    p.exclusive = sp.exclusive;
    const bool contig = sp.in_stride == sp.seg_len && sp.out_stride == sp.seg_len &&
                        ((reinterpret_cast<uintptr_t>(sp.in) | reinterpret_cast<uintptr_t>(sp.out)) & 15) == 0;
    // strided rows of whole 16-byte vectors (every row start 16-byte aligned, in and out)
    // and at least 64 bytes of input per row: measured (profiles/r02c_rows_tiny.txt) fp32 x 32
    // 45 -> 50 %, int32 x 32 44 -> 55 %, fp16 x 32 36 -> 61 % of the copy peak against the
    // shuffle kernel, fp32 x 16 even, fp32 x 8 (32-byte rows) 45 -> 36 % (kept on the shuffles)
    constexpr int kEsIn = (int)sizeof(typename Traits<DT>::In);
    const bool strided_vec = !contig && sp.seg_len * kEsIn >= 64 && sp.seg_len % (16 / kEsIn) == 0 &&
                             sp.seg_len % 4 == 0 &&
                             (sp.in_stride * kEsIn) % 16 == 0 && (sp.out_stride * 4) % 16 == 0 &&
                             ((reinterpret_cast<uintptr_t>(sp.in) | reinterpret_cast<uintptr_t>(sp.out)) & 15) == 0 &&
                             env_int("SCAN_ROWS_TILE_STRIDED", 1);
    if (sp.seg_len <= kTileMaxCols && (contig || strided_vec) && env_int("SCAN_ROWS_TILE", 1)) {
        int64_t grid = (sp.num_segs + kThreads - 1) / kThreads;
        const int64_t cap = (int64_t)di.sms * 6;  // 34 KB of shared memory per CTA
        if (grid > cap) grid = cap;
        if (contig)
            k_rows_tile<DT><<<(unsigned)grid, kThreads, 0, s>>>(p);
        else
            k_rows_tile<DT, true><<<(unsigned)grid, kThreads, 0, s>>>(p);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return cudaGetLastError() == cudaSuccess ? SCAN_OK : SCAN_ERR_CUDA;
    }
    int64_t warps_needed;
    if (sp.seg_len <= 32) {
        int G = 1;
        while (G < sp.seg_len) G <<= 1;
        warps_needed = (sp.num_segs + (32 / G) - 1) / (32 / G);
    } else {
        warps_needed = sp.num_segs;
    }
    int64_t grid = (warps_needed + kWarps - 1) / kWarps;
    const int64_t cap = (int64_t)di.sms * 8;  // 8 CTAs of 8 warps per SM
    if (grid > cap) grid = cap;
    if (sp.seg_len <= 32) k_rows_tiny<DT><<<(unsigned)grid, kThreads, 0, s>>>(p);
    else k_rows_warp<DT><<<(unsigned)grid, kThreads, 0, s>>>(p);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError() == cudaSuccess ? SCAN_OK : SCAN_ERR_CUDA;
}

template <int DT>
int launch_dt(ScanParams p, cudaStream_t s, const DevInfo& di)
{
    constexpr bool wide_in = (DT == SCAN_I32_I32 || DT == SCAN_F32_F32);
    using Small = Variant<DT, 512, 4, 2, 1, 2>;  // 8192-element tiles
    const int v = variant();
    // batched short rows: a warp (or a fraction of one) per row -- SURVEY 8(a) a6
    if (p.num_segs > 1 && p.seg_len <= env_int("SCAN_ROWS_WARP_MAX", 4096) && p.carry_in == nullptr &&
        p.row_pre == nullptr && v == 0)
        return launch_rows_small<DT>(p, s, di);
    if (v == 0 || p.seg_len <= Small::kTile) {
        if (p.seg_len <= Small::kTile) return Small::launch(p, s, di);
        if (p.num_segs == 1 && p.seg_len <= 16 * (int64_t)Small::kTile && env_int("SCAN_NO_CLUSTER", 0) == 0) {
            // n <= 65,536 (C1): 4096-element tiles, up to 16 CTAs in the cluster --
            // half the per-CTA latency of 8192-element tiles (C1 step 12.1 -> 9-10 us)
            using Small4 = Variant<DT, 256, 4, 2, 1, 2>;
            if (env_int("SCAN_SMALL4", 1) != 0 && p.seg_len <= 16 * (int64_t)Small4::kTile)
                return Small4::launch_cluster(p, s);
            return Small::launch_cluster(p, s);
        }
        if (p.num_segs == 1 && p.tma_in && p.tma_out && p.seg_len >= kMcMinElems &&
            env_int("SCAN_NO_MC", 0) == 0)
            return launch_mc<DT>(p, s, di);
        // few long rows (fewer than half the SMs, >= 2^22 elements each): one
        // full-GPU MCScan per row instead of one CTA per row -- SURVEY 8(a) a6
        const int few = env_int("SCAN_FEW_ROWS", 0);
        // at most half as many rows as SMs (a CTA per row would leave the GPU
        // half idle), contiguous, tile-multiple length: one segmented MCScan over
        // all rows (the whole GPU on every row, L2 splitting intact)
        if (p.num_segs > 1 && p.num_segs * 2 <= (int64_t)di.sms * env_int("SCAN_SEG_MC_X2", 1) &&
            p.in_stride == p.seg_len && p.out_stride == p.seg_len && p.num_segs * p.seg_len >= kMcMinElems &&
            p.tma_in && p.tma_out && p.row_pre == nullptr && p.carry_in == nullptr &&
            env_int("SCAN_NO_MC", 0) == 0 && few == 0) {
            const int st = launch_mc_rows<DT>(p, s, di);
            if (st != -1) return st;
        }
        if (p.num_segs > 1 && p.num_segs * 2 <= di.sms && p.seg_len >= ((int64_t)1 << 22) && p.tma_in &&
            p.tma_out && p.row_pre == nullptr && env_int("SCAN_NO_MC", 0) == 0 && few == 0) {
            using In = typename Traits<DT>::In;
            for (int64_t r = 0; r < p.num_segs; ++r) {
                ScanParams q = p;
                q.in = (const uint8_t*)p.in + r * p.in_stride * (int64_t)sizeof(In);
                q.out = (uint8_t*)p.out + r * p.out_stride * 4;
                q.num_segs = 1;
                q.in_stride = q.out_stride = p.seg_len;
                q.carry_in = nullptr;
                const int st = launch_mc<DT>(q, s, di);
                if (st != SCAN_OK) return st;
            }
            return SCAN_OK;
        }
        if (rowscan_ok<DT>(p) && !(few == 1 && p.num_segs < di.sms)) return launch_rows<DT>(p, s, di);
        if constexpr (wide_in) {
            return WsVariant<DT, 16, 3, 8, 3, 3>::launch(p, s, di);
        } else if constexpr (DT == SCAN_F16_F32) {
            return WsVariant<DT, 16, 3, 4, 4, 3>::launch(p, s, di);
        } else {
            return WsVariant<DT, 16, 2, 8, 3, 2>::launch(p, s, di);
        }
    }
#define SCAN_VARIANT_CASE(ID, TH, RW, ST, OS, MB) \
    case ID: return Variant<DT, TH, RW, ST, OS, MB>::launch(p, s, di);
    switch (v) {
        SCAN_VARIANT_CASE(1, 256, 8, 2, 1, 2)
        SCAN_VARIANT_CASE(2, 512, 4, 1, 1, 2)
        SCAN_VARIANT_CASE(4, 256, 8, 1, 1, 2)
        SCAN_VARIANT_CASE(5, 128, 8, 1, 1, 6)
    case 10:
        if constexpr (wide_in) return WsVariant<DT, 16, 1, 8, 3, 3>::launch(p, s, di);
        else return WsVariant<DT, 16, 1, 8, 3, 2>::launch(p, s, di);
    case 11:
        if constexpr (wide_in) return WsVariant<DT, 16, 2, 4, 6, 6>::launch(p, s, di);
        else return WsVariant<DT, 16, 2, 4, 4, 4>::launch(p, s, di);
    case 12:
        if constexpr (wide_in) return WsVariant<DT, 16, 3, 4, 6, 6>::launch(p, s, di);
        else return WsVariant<DT, 16, 3, 4, 4, 3>::launch(p, s, di);
    case 14:
        if constexpr (wide_in) return WsVariant<DT, 16, 2, 8, 2, 2>::launch(p, s, di);
        else return WsVariant<DT, 16, 2, 8, 3, 2>::launch(p, s, di);
    case 13:
        if constexpr (wide_in) return WsVariant<DT, 16, 6, 4, 6, 6>::launch(p, s, di);
        else return WsVariant<DT, 16, 4, 4, 4, 4>::launch(p, s, di);
    default:
        return Small::launch(p, s, di);
    }
#undef SCAN_VARIANT_CASE
}

int launch_any(int dt, ScanParams p, cudaStream_t s, const DevInfo& di)
{
    switch (dt) {
    case SCAN_I32_I32: return launch_dt<0>(p, s, di);
    case SCAN_F32_F32: return launch_dt<1>(p, s, di);
    case SCAN_F16_F32: return launch_dt<2>(p, s, di);
    case SCAN_I8_I32: return launch_dt<3>(p, s, di);
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

// Zero the operator scratch a previous split / sort left in `ws` (see DirtyWs).
int ws_clean(void* ws, size_t ws_bytes, cudaStream_t s)
{
    if (ws == nullptr) return SCAN_OK;
    const size_t d = ws_take_dirty(ws, ws_bytes);
    if (d > kWsDescOffset && cudaMemsetAsync((uint8_t*)ws + kWsDescOffset, 0, d - kWsDescOffset, s) != cudaSuccess)
        return SCAN_ERR_CUDA;
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
    if ((st = ws_clean(ws, ws_bytes, (cudaStream_t)stream)) != SCAN_OK) return st;
    if (!(p.tma_in && p.tma_out) && n >= kMcMinElems + 16 && ((uintptr_t)out & 3u) == 0 &&
        ((uintptr_t)in % in_size(dt)) == 0 && variant() == 0 && env_int("SCAN_NO_MC", 0) == 0 &&
        env_int("SCAN_NO_SHIFT", 0) == 0) {
        // Unaligned 1-D array: the <= 3-element head up to the output's next 16-byte
        // boundary is scanned on its own (k_scan_head: head outputs, and carry_in +
        // head sum into the workspace header), then the MCScan runs on the rest with
        // an aligned output and, if the input is still off a 16-byte boundary, the
        // shifted-slot instantiation (its TMA views start at the boundary below).
        const int h = (int)(((16u - ((uintptr_t)out & 15u)) & 15u) / 4u);
        cudaStream_t s = (cudaStream_t)stream;
        const void* carry = carry_in;
        if (h > 0) {
            void* slot = (uint8_t*)ws + kWsHeadCarry;
            switch (dt) {
            case SCAN_I32_I32: k_scan_head<0><<<1, 32, 0, s>>>(in, out, h, carry_in, exclusive, slot); break;
            case SCAN_F32_F32: k_scan_head<1><<<1, 32, 0, s>>>(in, out, h, carry_in, exclusive, slot); break;
            case SCAN_F16_F32: k_scan_head<2><<<1, 32, 0, s>>>(in, out, h, carry_in, exclusive, slot); break;
            default: k_scan_head<3><<<1, 32, 0, s>>>(in, out, h, carry_in, exclusive, slot); break;
            }
            g_launches.fetch_add(1, std::memory_order_relaxed);
            if (cudaGetLastError() != cudaSuccess) return SCAN_ERR_CUDA;
            carry = slot;
        }
        const uint8_t* body_in = (const uint8_t*)in + (int64_t)h * (int64_t)in_size(dt);
        p.in = body_in;
        p.out = (uint8_t*)out + (int64_t)h * 4;
        p.seg_len = p.in_stride = p.out_stride = n - h;
        p.carry_in = carry;
        p.tma_in = p.tma_out = 1;
        p.shift = (int)(((uintptr_t)body_in & 15u) / in_size(dt));
        return launch_any(dt, p, s, di);
    }
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
    const size_t lb = kWsDescOffset + (size_t)tiles_for(n) * desc_bytes(dtype);
    const size_t mc = mc_workspace_bytes(n);
    return lb > mc ? lb : mc;
}

size_t scan_rows_workspace_bytes(int dtype, int64_t rows, int64_t cols)
{
    if (!valid_dt(dtype) || rows < 0 || cols < 0) return 0;
    const size_t lb = kWsDescOffset + (size_t)(rows * tiles_for(cols)) * desc_bytes(dtype);
    const size_t mc = mc_workspace_bytes(rows * cols);  // few long rows: one segmented MCScan
    return lb > mc ? lb : mc;
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
    if ((st = ws_clean(ws, ws_bytes, (cudaStream_t)stream)) != SCAN_OK) return st;
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

// ---- host streaming (end-to-end) ----------------------------------------------------
// Stage layout: in[2] (chunk x in_size), out[2] (chunk x 4), then a ring of 3
// carry triples {carry_i, total_i, unused} (8 bytes each, 256-aligned).
size_t scan_host_stage_bytes(int dtype, int64_t chunk_elems)
{
    if (!valid_dt(dtype) || chunk_elems <= 0) return 0;
    auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
    return 2 * up((size_t)chunk_elems * in_size(dtype)) + 2 * up((size_t)chunk_elems * 4) + 256;
}

int scan_host(const void* h_in, void* h_out, int64_t n, int dtype, int exclusive, int64_t chunk_elems,
              void* stage, size_t stage_bytes, void* ws, size_t ws_bytes, void* stream)
{
    if (!valid_dt(dtype) || n < 0 || chunk_elems <= 0) return SCAN_ERR_ARG;
    if (n == 0) return SCAN_OK;
    if (h_in == nullptr || h_out == nullptr || stage == nullptr || h_in == h_out) return SCAN_ERR_ARG;
    if (stage_bytes < scan_host_stage_bytes(dtype, chunk_elems)) return SCAN_ERR_ARG;
    DevInfo di;
    int st = dev_info(di);
    if (st != SCAN_OK) return st;
    int dev = 0;
    cudaGetDevice(&dev);
    // two copy streams per device, created once (the library's only cached resource besides attributes)
    static std::mutex mu;
    static cudaStream_t copy_streams[64][2] = {};
    {
        std::lock_guard<std::mutex> g(mu);
        if (copy_streams[dev][0] == nullptr) {
            for (int k = 0; k < 2; ++k)
                if (cudaStreamCreateWithFlags(&copy_streams[dev][k], cudaStreamNonBlocking) != cudaSuccess)
                    return SCAN_ERR_CUDA;
        }
    }
    cudaStream_t s_c = (cudaStream_t)stream, s_in = copy_streams[dev][0], s_out = copy_streams[dev][1];
    auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t isz = in_size(dtype), in_b = up((size_t)chunk_elems * isz), out_b = up((size_t)chunk_elems * 4);
    uint8_t* base = (uint8_t*)stage;
    uint8_t* d_in[2] = {base, base + in_b};
    uint8_t* d_out[2] = {base + 2 * in_b, base + 2 * in_b + out_b};
    uint8_t* trip = base + 2 * in_b + 2 * out_b;  // 3 x {carry, total, unused} x 8 B
    const int64_t nchunks = (n + chunk_elems - 1) / chunk_elems;

    cudaEvent_t ev_start, ev_in[2], ev_comp[2], ev_out[2];
    auto mk = [](cudaEvent_t* e) { return cudaEventCreateWithFlags(e, cudaEventDisableTiming) == cudaSuccess; };
    if (!mk(&ev_start)) return SCAN_ERR_CUDA;
    for (int k = 0; k < 2; ++k)
        if (!mk(&ev_in[k]) || !mk(&ev_comp[k]) || !mk(&ev_out[k])) return SCAN_ERR_CUDA;
    int rc = SCAN_OK;
    // order after everything already on the caller's stream
    if (cudaEventRecord(ev_start, s_c) != cudaSuccess) rc = SCAN_ERR_CUDA;
    cudaStreamWaitEvent(s_in, ev_start, 0);
    cudaStreamWaitEvent(s_out, ev_start, 0);
    if (cudaMemsetAsync(trip, 0, 24, s_c) != cudaSuccess) rc = SCAN_ERR_CUDA;  // carry_0 = 0
    auto h2d = [&](int64_t i) {
        const int64_t off = i * chunk_elems, cnt = n - off < chunk_elems ? n - off : chunk_elems;
        if (i >= 2) cudaStreamWaitEvent(s_in, ev_comp[i & 1], 0);  // scan of chunk i-2 has read the buffer
        cudaMemcpyAsync(d_in[i & 1], (const uint8_t*)h_in + off * isz, cnt * isz, cudaMemcpyHostToDevice, s_in);
        cudaEventRecord(ev_in[i & 1], s_in);
    };
    h2d(0);
    for (int64_t i = 0; i < nchunks && rc == SCAN_OK; ++i) {
        if (i + 1 < nchunks) h2d(i + 1);
        const int64_t off = i * chunk_elems, cnt = n - off < chunk_elems ? n - off : chunk_elems;
        cudaStreamWaitEvent(s_c, ev_in[i & 1], 0);
        if (i >= 2) cudaStreamWaitEvent(s_c, ev_out[i & 1], 0);  // d_out[i&1] copied out
        uint8_t* tr = trip + 24 * (i % 3);
        uint8_t* tr_next = trip + 24 * ((i + 1) % 3);
        rc = scan_1d(d_in[i & 1], d_out[i & 1], cnt, dtype, tr, ws, ws_bytes, stream, exclusive);
        if (rc == SCAN_OK && i + 1 < nchunks) {
            rc = scan_total(d_in[i & 1], cnt, dtype, tr + 8, ws, ws_bytes, stream);       // total_i
            if (rc == SCAN_OK) rc = scan_carry_from_totals(tr, 3, 2, dtype, tr_next, stream);  // carry + total
        }
        cudaEventRecord(ev_comp[i & 1], s_c);
        cudaStreamWaitEvent(s_out, ev_comp[i & 1], 0);
        cudaMemcpyAsync((uint8_t*)h_out + off * 4, d_out[i & 1], cnt * 4, cudaMemcpyDeviceToHost, s_out);
        cudaEventRecord(ev_out[i & 1], s_out);
    }
    // the caller's stream resumes after the last copy out
    cudaStreamWaitEvent(s_c, ev_out[(nchunks - 1) & 1], 0);
    if (nchunks >= 2) cudaStreamWaitEvent(s_c, ev_out[(nchunks - 2) & 1], 0);
    cudaEventDestroy(ev_start);
    for (int k = 0; k < 2; ++k) {
        cudaEventDestroy(ev_in[k]);
        cudaEventDestroy(ev_comp[k]);
        cudaEventDestroy(ev_out[k]);
    }
    if (rc == SCAN_OK && cudaGetLastError() != cudaSuccess) rc = SCAN_ERR_CUDA;
    return rc;
}

}  // extern "C"

// ---- scan-based operators (include/scan_ops.h) ----
#include "ops_api.cuh"
// ---- two-pass sharded scan (multi-GPU Reduce-Scan-Scan, include/scan.h) ----
#include "shard_api.cuh"

// scan_kernels.cuh -- sm_100a kernels of the device-wide prefix sum.
//
// What is computed (PAPER.md, "P<line>"): the inclusive prefix sum of P68
// (Sec. 2), the exclusive one of P461 (App. B.2), the batched row scan of
// P437 (App. B.1), with the P98/P459 type pairs.
//
// How: the paper's multi-core MCScan (Alg. 3, P229-261)
// reads the input twice and writes it twice across a SyncAll barrier (3N+2N
// traffic).  On B200 we use the single-pass "decoupled look-back" strategy
// that the paper itself names as the GPU state of the art (P78-81, Sec. 2.1:
// "require only ~2N data movement"):
//
//   a1  persistent CTAs claim tiles in order with a global atomic ticket;
//   a2  a producer thread streams each tile HBM -> shared memory with a TMA
//       1-D bulk copy (cp.async.bulk + mbarrier), STAGES tiles ahead;
//   a3  the tile is scanned in registers: 4 elements per lane per 128-element
//       row, a warp shuffle scan per row, rows chained within the warp, and
//       a block scan of the warp totals (the analog of the cube's A@U_s
//       row-local scans plus the vector unit's `partial` propagation of
//       Alg. 1, P145-155);
//   a4  warp 0 publishes the tile aggregate, looks back over the predecessor
//       descriptors (32 per step, one per lane) until it meets an inclusive
//       prefix, and publishes its own inclusive prefix (this replaces
//       SyncAll + "Sum first i entries of r", P245-248);
//   a5  outputs = carry + local prefix are written to a shared staging buffer
//       and streamed back with a TMA bulk store.
//
// Integer tiles use uint32 arithmetic (wraps mod 2^32).  Float tiles use fp32
// in-tile sums and an fp64 carry; an output is fl32(P_hi + fl32(base + l))
// where (P_hi, P_lo) is the double-float split of the fp64 prefix folded
// into the per-row base (an fp32 carry chain fails C2).
//
// Descriptor protocol (no fences needed): every 8-byte descriptor slot holds
// (epoch << 32 | 32 payload bits) and is written once per call, so a reader
// that sees its own epoch in a slot has a complete value.  fp64 values use
// two slots (hi/lo words).  The epoch lives in the workspace header and is
// advanced by the last CTA to finish, which also resets the ticket counter,
// so no memset is needed between calls.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include <type_traits>

#include "ptx.cuh"

namespace scan {

// ---------------------------------------------------------------- workspace
constexpr uint32_t kWsMagic = 0x5CA7B200u;
constexpr size_t kWsPartialsOffset = 256;         // scan_total per-CTA partials
constexpr int kMaxTotalCtas = 4096;
constexpr int kMaxGridPerLane = 6;   // k_mcscan coordinator: up to 192 CTAs
constexpr size_t kWsBarOffset = kWsPartialsOffset + 8 * kMaxTotalCtas;   // 33024: MCScan barriers
constexpr int kMaxChunks = 8192;                                            // u32 counter per chunk
constexpr size_t kWsDescOffset = kWsBarOffset + 4 * kMaxChunks;            // 65792

struct WsHeader {
    uint32_t magic;
    uint32_t epoch;         // tag of the current call's descriptors (>= 1)
    uint32_t ticket;        // next tile to claim
    uint32_t done;          // CTAs finished in the current call
    uint32_t capacity;      // descriptor slots (tiles) the workspace holds
    uint32_t total_done;    // scan_total: CTAs finished
    uint32_t error;         // set if a kernel found a bad header
    uint32_t pad[57];
};
static_assert(sizeof(WsHeader) == 256, "header is 256 bytes");

// ---------------------------------------------------------------- type traits
template <int DT>
struct Traits;

template <>
struct Traits<0> {  // SCAN_I32_I32
    using In = int32_t;
    using Out = int32_t;
    using Acc = uint32_t;
    using Carry = uint32_t;
    static constexpr bool kFloat = false;
};
template <>
struct Traits<1> {  // SCAN_F32_F32
    using In = float;
    using Out = float;
    using Acc = float;
    using Carry = double;
    static constexpr bool kFloat = true;
};
template <>
struct Traits<2> {  // SCAN_F16_F32 (raw binary16 bits in)
    using In = uint16_t;
    using Out = float;
    using Acc = float;
    using Carry = double;
    static constexpr bool kFloat = true;
};
template <>
struct Traits<3> {  // SCAN_I8_I32
    using In = int8_t;
    using Out = int32_t;
    using Acc = uint32_t;
    using Carry = uint32_t;
    static constexpr bool kFloat = false;
};

// ---- widening loads of 4 consecutive input elements (exact conversions) ----
__device__ __forceinline__ void unpack4(const int32_t* s, uint32_t (&v)[4])
{
    uint4 q = *reinterpret_cast<const uint4*>(s);
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
}
__device__ __forceinline__ void unpack4(const float* s, float (&v)[4])
{
    float4 q = *reinterpret_cast<const float4*>(s);
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
}
__device__ __forceinline__ void unpack4(const uint16_t* s, float (&v)[4])
{
    uint2 q = *reinterpret_cast<const uint2*>(s);
    __half2 a = *reinterpret_cast<__half2*>(&q.x);
    __half2 b = *reinterpret_cast<__half2*>(&q.y);
    float2 fa = __half22float2(a), fb = __half22float2(b);
    v[0] = fa.x; v[1] = fa.y; v[2] = fb.x; v[3] = fb.y;
}
__device__ __forceinline__ void unpack4(const int8_t* s, uint32_t (&v)[4])
{
    uint32_t w = *reinterpret_cast<const uint32_t*>(s);
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = (uint32_t)(int32_t)(int8_t)(w >> (8 * k));
}
__device__ __forceinline__ uint32_t widen(int32_t x) { return (uint32_t)x; }
__device__ __forceinline__ uint32_t widen(int8_t x) { return (uint32_t)(int32_t)x; }
__device__ __forceinline__ float widen(float x) { return x; }
__device__ __forceinline__ float widen(uint16_t x) { return __half2float(__ushort_as_half(x)); }

__device__ __forceinline__ void store4(int32_t* d, const uint32_t (&o)[4])
{
    *reinterpret_cast<uint4*>(d) = make_uint4(o[0], o[1], o[2], o[3]);
}
__device__ __forceinline__ void store4(float* d, const float (&o)[4])
{
    *reinterpret_cast<float4*>(d) = make_float4(o[0], o[1], o[2], o[3]);
}
__device__ __forceinline__ int32_t narrow(uint32_t x, int32_t*) { return (int32_t)x; }
__device__ __forceinline__ float narrow(float x, float*) { return x; }

// ---- warp primitives -------------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T x, int lane)
{
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x = x + y;
    }
    return x;
}

__device__ __forceinline__ uint32_t warp_sum(uint32_t x) { return __reduce_add_sync(0xffffffffu, x); }
__device__ __forceinline__ double warp_sum(double x)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// Butterfly reduction over the warp (fixed order: every lane gets the same bits).
template <typename T>
__device__ __forceinline__ T warp_reduce_fixed(T x)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = x + __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// Carry <-> 64-bit storage word.
__device__ __forceinline__ uint64_t carry_bits(uint32_t v) { return v; }
__device__ __forceinline__ uint64_t carry_bits(double v) { return (uint64_t)__double_as_longlong(v); }
template <typename C>
__device__ __forceinline__ C carry_from_bits(uint64_t b);
template <>
__device__ __forceinline__ uint32_t carry_from_bits<uint32_t>(uint64_t b) { return (uint32_t)b; }
template <>
__device__ __forceinline__ double carry_from_bits<double>(uint64_t b) { return __longlong_as_double((long long)b); }

// ---- thread-block cluster helpers (small-n path) ----
__device__ __forceinline__ uint32_t cluster_ctarank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Split cluster barrier: arrive early (every CTA has started), wait later.
__device__ __forceinline__ void cluster_arrive_relaxed()
{
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait()
{
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}
// Write a 64-bit word into the shared memory of CTA `rank` of this cluster.
__device__ __forceinline__ void st_dsmem_u64(void* local_smem_ptr, uint32_t rank, uint64_t v)
{
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(ptx::smem_u32(local_smem_ptr)), "r"(rank));
    asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(remote), "l"(v) : "memory");
}
// Read a 64-bit word from the shared memory of CTA `rank` of this cluster.
__device__ __forceinline__ uint64_t ld_dsmem_u64(const void* local_smem_ptr, uint32_t rank)
{
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(ptx::smem_u32(local_smem_ptr)), "r"(rank));
    uint64_t v;
    asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(remote) : "memory");
    return v;
}

using ptx::ld_acquire_u32;
using ptx::ld_acquire_u64;
using ptx::ld_relaxed_u64;
using ptx::named_bar_sync;

// ---- look-back descriptors -------------------------------------------------
// int: 2 slots per tile {aggregate, inclusive}; fp64: 4 slots {agg hi, agg lo,
// incl hi, incl lo}.  Slot = (epoch << 32) | payload.
template <typename Carry>
struct Desc;

template <>
struct Desc<uint32_t> {
    static constexpr int kSlots = 2;
    static __device__ __forceinline__ void publish(uint64_t* d, bool inclusive, uint32_t tag,
                                                   uint32_t v)
    {
        ptx::st_relaxed_u64(d + (inclusive ? 1 : 0), ((uint64_t)tag << 32) | v);
    }
    // status: 2 = inclusive prefix, 1 = aggregate, 0 = not ready.
    static __device__ __forceinline__ int read(const uint64_t* d, uint32_t tag, uint32_t& v)
    {
        uint64_t a, i;
        ptx::ld_relaxed_v2u64(d, a, i);
        if ((uint32_t)(i >> 32) == tag) { v = (uint32_t)i; return 2; }
        if ((uint32_t)(a >> 32) == tag) { v = (uint32_t)a; return 1; }
        v = 0;
        return 0;
    }
};

template <>
struct Desc<double> {
    static constexpr int kSlots = 4;
    static __device__ __forceinline__ void publish(uint64_t* d, bool inclusive, uint32_t tag,
                                                   double v)
    {
        uint64_t b = (uint64_t)__double_as_longlong(v);
        uint64_t t = (uint64_t)tag << 32;
        ptx::st_relaxed_v2u64(d + (inclusive ? 2 : 0), t | (b >> 32), t | (b & 0xffffffffull));
    }
    static __device__ __forceinline__ int read(const uint64_t* d, uint32_t tag, double& v)
    {
        uint64_t ah, al, ih, il;
        ptx::ld_relaxed_v2u64(d, ah, al);
        ptx::ld_relaxed_v2u64(d + 2, ih, il);
        if ((uint32_t)(ih >> 32) == tag && (uint32_t)(il >> 32) == tag) {
            v = __longlong_as_double((long long)((ih << 32) | (il & 0xffffffffull)));
            return 2;
        }
        if ((uint32_t)(ah >> 32) == tag && (uint32_t)(al >> 32) == tag) {
            v = __longlong_as_double((long long)((ah << 32) | (al & 0xffffffffull)));
            return 1;
        }
        v = 0.0;
        return 0;
    }
};

// Warp-cooperative decoupled look-back for tile t.  `lo` < t is a tile whose
// inclusive prefix `lo_val` is already known to the caller: either the CTA's
// own previously processed tile (tiles are claimed in increasing order, so it
// is always below t) or the virtual tile before the segment (value = the
// segment's carry-in).  The warp therefore only has to sum the aggregates of
// tiles lo+1..t-1, stopping early at the nearest inclusive prefix.  Each lane
// reads BATCH descriptors per round (idx = hi - lane - 32 r), so one L2 round
// trip covers 32*BATCH predecessors instead of 32.
template <typename Carry, int BATCH>
__device__ __forceinline__ Carry lookback(const uint64_t* desc, int64_t t, int64_t lo, Carry lo_val,
                                          uint32_t tag, int lane, uint32_t backoff,
                                          unsigned long long* stats = nullptr)
{
    using D = Desc<Carry>;
    Carry acc = Carry(0);
    int64_t hi = t - 1;  // highest tile not yet accounted for
    while (true) {
        int st[BATCH];
        Carry v[BATCH];
#pragma unroll
        for (int r = 0; r < BATCH; ++r) {
            int64_t idx = hi - lane - 32 * r;
            if (idx > lo) {
                st[r] = D::read(desc + idx * D::kSlots, tag, v[r]);
            } else {
                st[r] = 2;
                v[r] = (idx == lo) ? lo_val : Carry(0);
            }
        }
        bool progressed = false;
        if (stats && lane == 0) atomicAdd(&stats[0], 1ull);  // rounds
#pragma unroll
        for (int r = 0; r < BATCH; ++r) {
            uint32_t pm = __ballot_sync(0xffffffffu, st[r] == 2);
            uint32_t xm = __ballot_sync(0xffffffffu, st[r] == 0);
            uint32_t need = pm ? ((pm & (0u - pm)) << 1) - 1u : 0xffffffffu;  // lanes 0..first P
            if (xm & need) break;  // a needed predecessor has not published yet
            Carry c = ((need >> lane) & 1u) ? v[r] : Carry(0);
            acc = acc + warp_sum(c);
            if (stats && lane == 0) atomicAdd(&stats[7], 1ull);  // windows consumed (s_prof[11])
            if (pm) return acc;
            hi -= 32;
            progressed = true;
        }
        if (stats && lane == 0 && !progressed) stats[1] += 1;  // stalled rounds (s_prof[5])
        if (!progressed && backoff) {
            __nanosleep(backoff);
            backoff = backoff < 512 ? backoff * 2 : 512;
        }
    }
}

// Range look-back used by the warp-specialized kernel.  Walks tiles t-1,
// t-2, ... down to the nearest inclusive prefix (P) or to tile `lo`, which is
// treated as a P whose value the CALLER adds afterwards (it may not be known
// yet: `lo` is this CTA's previous tile, resolved by another look-back warp).
// Returns the sum of the aggregates above the stop point plus, if the stop
// was a real P, its value; *hit_lo tells whether the stop was `lo`.
template <typename Carry, int BATCH>
__device__ __forceinline__ Carry lookback_range(const uint64_t* desc, int64_t t, int64_t lo,
                                                uint32_t tag, int lane, uint32_t backoff,
                                                bool* hit_lo, unsigned long long* stats)
{
    using D = Desc<Carry>;
    Carry acc = Carry(0);
    int64_t hi = t - 1;
    while (true) {
        int st[BATCH];
        Carry v[BATCH];
#pragma unroll
        for (int r = 0; r < BATCH; ++r) {
            const int64_t idx = hi - lane - 32 * r;
            st[r] = 2;
            v[r] = Carry(0);
            if (idx > lo) st[r] = D::read(desc + idx * D::kSlots, tag, v[r]);
        }
        if (stats && lane == 0) atomicAdd(&stats[0], 1ull);
        int consumed = 0;
        bool blocked = false;
#pragma unroll
        for (int r = 0; r < BATCH; ++r) {
            if (blocked) continue;
            const uint32_t pm = __ballot_sync(0xffffffffu, st[r] == 2);
            const uint32_t xm = __ballot_sync(0xffffffffu, st[r] == 0);
            const uint32_t need = pm ? ((pm & (0u - pm)) << 1) - 1u : 0xffffffffu;
            if (xm & need) {  // a needed predecessor has not published yet
                blocked = true;
                continue;
            }
            const Carry c = ((need >> lane) & 1u) ? v[r] : Carry(0);
            acc = acc + warp_sum(c);
            if (stats && lane == 0) atomicAdd(&stats[7], 1ull);
            if (pm) {
                const int64_t stop = hi - 32 * r - (__ffs(pm) - 1);
                *hit_lo = stop <= lo;
                return acc;
            }
            ++consumed;
        }
        hi -= 32 * consumed;
        if (consumed == 0) {
            if (stats && lane == 0) atomicAdd(&stats[1], 1ull);
            if (backoff) __nanosleep(backoff);
        }
    }
}

// ---------------------------------------------------------------- parameters
struct ScanParams {
    const void* in;
    void* out;
    int64_t seg_len;        // elements per segment (n for 1-D, cols for rows)
    int64_t num_segs;       // 1 for 1-D, rows for scan_rows
    int64_t in_stride;      // elements between segment starts (input)
    int64_t out_stride;     // elements between segment starts (output)
    int64_t tiles_per_seg;
    int64_t num_tiles;
    const void* carry_in;   // nullable; applies to segment 0 (1-D API only; rows: added to row_pre)
    const void* row_pre;    // nullable; rows kernel: per-row start value (sharded scan pass 2)
    uint8_t* ws;            // workspace (unused when static_sched)
    int exclusive;
    int tma_in;             // segment bases and strides 16-byte aligned (input)
    int tma_out;            // same for output
    int static_sched;       // one tile per segment: no tickets, no look-back
    int cluster;            // > 0: small-n mode, one tile per CTA of ONE cluster, carries via DSMEM
    int cl_push;            // cluster mode: aggregates pushed to the higher CTAs (one cluster barrier)
    int debug;              // bit 0: skip look-back (timing only; wrong results); bit 1: spin without
                            // nanosleep; bit 2: per-CTA stall counters into the workspace
    int shift;              // MCScan SHIFT: `in` is this many elements past a 16-byte boundary
    // rows kernel, sharded pass 2 with the device-initiated exchange (shard.cuh)
    const uint64_t* peer_slots;
    int peer_G, peer_rank;
    uint32_t peer_epoch;
    void* carry_out;
};

template <int THREADS, int ROWS>
struct TileShape {
    static constexpr int kWarps = THREADS / 32;
    static constexpr int kRowElems = 128;                 // 32 lanes x 4 elements
    static constexpr int kWarpElems = ROWS * kRowElems;
    static constexpr int kTile = kWarps * kWarpElems;     // elements per tile
};

// Dynamic shared memory of k_scan_tiles.
template <int DT, int THREADS, int ROWS, int STAGES, int OSTAGES>
constexpr size_t scan_smem_bytes()
{
    using T = Traits<DT>;
    return (size_t)STAGES * TileShape<THREADS, ROWS>::kTile * sizeof(typename T::In) +
           (size_t)OSTAGES * TileShape<THREADS, ROWS>::kTile * sizeof(typename T::Out);
}

// ---------------------------------------------------------------- the kernel
template <int DT, int THREADS, int ROWS, int STAGES, int OSTAGES, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) k_scan_tiles(const ScanParams p)
{
    using Tr = Traits<DT>;
    using In = typename Tr::In;
    using Out = typename Tr::Out;
    using Acc = typename Tr::Acc;
    using Carry = typename Tr::Carry;
    using Shape = TileShape<THREADS, ROWS>;
    constexpr int NW = Shape::kWarps;
    constexpr int TILE = Shape::kTile;

    extern __shared__ __align__(128) uint8_t smem[];
    In* const in_stage = reinterpret_cast<In*>(smem);
    Out* const out_stage = reinterpret_cast<Out*>(smem + (size_t)STAGES * TILE * sizeof(In));

    __shared__ __align__(8) uint64_t full_bar[STAGES];
    __shared__ int64_t s_ticket[STAGES];
    __shared__ int s_tma[STAGES];
    __shared__ Acc s_warp_tot[NW];
    __shared__ Acc s_warp_pref[NW];
    __shared__ Carry s_prefix;
    __shared__ uint32_t s_epoch;
    __shared__ uint64_t s_cl_agg;  // cluster mode: this CTA's tile aggregate (Carry bits)
    __shared__ uint64_t s_cl_in[16];  // cluster push mode: slot r = the aggregate of CTA r < this CTA

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;

    WsHeader* hdr = reinterpret_cast<WsHeader*>(p.ws);
    uint64_t* desc = reinterpret_cast<uint64_t*>(p.ws + kWsDescOffset);
    const In* gin = reinterpret_cast<const In*>(p.in);
    Out* gout = reinterpret_cast<Out*>(p.out);

    const uint64_t pol_in = ptx::policy_evict_first();
    const uint64_t pol_out = ptx::policy_evict_first();

    // Claim this CTA's q-th tile and, if it can go by TMA, start streaming it
    // into stage s.  Called by one thread (tid 0 in the prologue, tid 32 --
    // warp 1, so the look-back warp never waits on the ticket atomic -- later).
    auto issue = [&](int s, int64_t q) {
        int64_t t;
        if (p.static_sched) {
            t = (int64_t)blockIdx.x + q * gridDim.x;
        } else {
            t = (int64_t)ptx::claim_add(&hdr->ticket, 1u);
        }
        s_ticket[s] = t;
        int tma = 0;
        if (t < p.num_tiles) {
            int64_t seg = t / p.tiles_per_seg;
            int64_t k = t - seg * p.tiles_per_seg;
            int64_t m = p.seg_len - k * TILE;
            if (m > TILE) m = TILE;
            uint32_t bytes = (uint32_t)(m * (int64_t)sizeof(In));
            if (p.tma_in && (bytes & 15u) == 0) {
                tma = 1;
                ptx::mbar_arrive_expect_tx(&full_bar[s], bytes);
                ptx::tma_load_1d(in_stage + (size_t)s * TILE, gin + seg * p.in_stride + k * TILE, bytes,
                                 &full_bar[s], pol_in);
            }
        }
        s_tma[s] = tma;
    };

    // Programmatic dependent launch (cluster launches of small n): the next kernel
    // in the stream may start launching now; it waits in ITS griddepcontrol.wait
    // until this grid has completed and flushed.  No-ops without the attribute.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // cluster push mode: announce this CTA has started (its shared memory may
    // receive the lower CTAs' aggregates once every CTA has announced)
    if (p.cluster && p.cl_push) cluster_arrive_relaxed();
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) ptx::mbar_init(&full_bar[s], 1);
        ptx::fence_mbar_init();
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous kernel's writes are visible
    if (tid == 0) {
        if (!p.static_sched) {
            if (hdr->magic != kWsMagic) hdr->error = 1;
            s_epoch = hdr->epoch;
        }
        for (int s = 0; s < STAGES; ++s) issue(s, s);
    }
    __syncthreads();
    const uint32_t tag = s_epoch;

    uint32_t phases = 0;  // bit s = parity of the next wait on full_bar[s]
    int ostage = 0;
    int64_t last_t = -1;       // warp 0: this CTA's previous tile and its inclusive prefix
    Carry last_incl = Carry(0);
    for (int64_t iter = 0;; ++iter) {
        const int s = (int)(iter % STAGES);
        const int64_t t = s_ticket[s];
        if (t >= p.num_tiles) break;
        const int tma = s_tma[s];
        const int64_t seg = t / p.tiles_per_seg;
        const int64_t k = t - seg * p.tiles_per_seg;
        int64_t m64 = p.seg_len - k * TILE;
        const int m = (int)(m64 > TILE ? TILE : m64);
        const bool full = (m == TILE);
        const In* src = gin + seg * p.in_stride + k * TILE;
        Out* dst = gout + seg * p.out_stride + k * TILE;

        // ---- a2: load the tile into registers (4 elements per lane per row)
        Acc v[ROWS][4];
        const int wbase = warp * Shape::kWarpElems + 4 * lane;
        if (tma) {
            ptx::mbar_wait(&full_bar[s], (phases >> s) & 1u);
            phases ^= 1u << s;
            const In* st = in_stage + (size_t)s * TILE;
#pragma unroll
            for (int j = 0; j < ROWS; ++j) unpack4(st + wbase + j * 128, v[j]);
            if (!full) {
#pragma unroll
                for (int j = 0; j < ROWS; ++j)
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (wbase + j * 128 + q >= m) v[j][q] = Acc(0);
            }
        } else {
#pragma unroll
            for (int j = 0; j < ROWS; ++j)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    int e = wbase + j * 128 + q;
                    v[j][q] = e < m ? widen(src[e]) : Acc(0);
                }
        }

        // ---- a3: thread-local, warp and row scans
        Acc lane_excl[ROWS];
        Acc row_tot[ROWS];
#pragma unroll
        for (int j = 0; j < ROWS; ++j) {
            v[j][1] = v[j][0] + v[j][1];
            v[j][2] = v[j][1] + v[j][2];
            v[j][3] = v[j][2] + v[j][3];
            Acc incl = warp_incl_scan(v[j][3], lane);
            Acc ex = __shfl_up_sync(0xffffffffu, incl, 1);
            lane_excl[j] = lane == 0 ? Acc(0) : ex;
            row_tot[j] = __shfl_sync(0xffffffffu, incl, 31);
        }
        Acc row_pref[ROWS];
        Acc wsum = Acc(0);
#pragma unroll
        for (int j = 0; j < ROWS; ++j) {
            row_pref[j] = wsum;
            wsum = wsum + row_tot[j];
        }
        if (lane == 0) s_warp_tot[warp] = wsum;
        __syncthreads();  // [A] stage s fully read; warp totals visible

        // STAGES > 1: refill stage s with the next claimed tile while we finish
        // this one.  (That tile's aggregate then waits for this tile's
        // look-back: a chain.  STAGES == 1 claims after the look-back instead.)
        if (STAGES > 1 && tid == 32) issue(s, iter + STAGES);

        // ---- a4: block scan of warp totals + decoupled look-back (warp 0)
        if (warp == 0) {
            Acc x = lane < NW ? s_warp_tot[lane] : Acc(0);
            Acc xi = warp_incl_scan(x, lane);
            Acc xe = __shfl_up_sync(0xffffffffu, xi, 1);
            if (lane < NW) s_warp_pref[lane] = lane == 0 ? Acc(0) : xe;
            const Acc agg = __shfl_sync(0xffffffffu, xi, NW - 1);
            Carry carry_seg = Carry(0);
            if (seg == 0 && p.carry_in != nullptr) {
                if constexpr (Tr::kFloat)
                    carry_seg = *reinterpret_cast<const double*>(p.carry_in);
                else
                    carry_seg = (uint32_t)(uint64_t)(*reinterpret_cast<const int64_t*>(p.carry_in));
            }
            Carry prefix;
            if (p.cluster) {
                prefix = carry_seg;  // + lower CTAs' aggregates, added after the cluster barrier
                if (lane == 0) s_cl_agg = carry_bits(Carry(agg));
            } else if (k == 0) {
                prefix = carry_seg;
                if (!p.static_sched && p.tiles_per_seg > 1 && lane == 0)
                    Desc<Carry>::publish(desc + t * Desc<Carry>::kSlots, true, tag,
                                         carry_seg + Carry(agg));
            } else {
                if (lane == 0)
                    Desc<Carry>::publish(desc + t * Desc<Carry>::kSlots, false, tag, Carry(agg));
                const int64_t seg_first = t - k;
                const bool own = last_t >= seg_first;
                if (p.debug & 1)
                    prefix = Carry(0);
                else
                    prefix = lookback<Carry, 8>(desc, t, own ? last_t : seg_first - 1,
                                                own ? last_incl : carry_seg, tag, lane,
                                                (p.debug & 2) ? 0u : 32u);
                if (lane == 0 && k + 1 < p.tiles_per_seg)
                    Desc<Carry>::publish(desc + t * Desc<Carry>::kSlots, true, tag,
                                         prefix + Carry(agg));
            }
            last_t = t;
            last_incl = prefix + Carry(agg);
            if (lane == 0) s_prefix = prefix;
        }
        if (p.cluster) {
            // Small n: the tiles are the CTAs of one cluster.  Every CTA posts
            // its aggregate in its own shared memory; after a cluster barrier
            // warp 0 sums the aggregates of the lower-ranked CTAs over DSMEM
            // (fixed lane-tree order) -- no global descriptors, no atomics.
            if (p.cl_push) {
                // push: every CTA of the cluster has started (the early arrive's
                // phase), so lane q > rank of warp 0 stores this CTA's aggregate
                // into CTA q's slot; after ONE barrier the lower aggregates are
                // local, and no CTA touches another's shared memory afterwards
                cluster_wait();
                if (warp == 0) {
                    __syncwarp();
                    const uint32_t rank = cluster_ctarank();
                    if ((uint32_t)lane > rank && lane < p.cluster)
                        st_dsmem_u64(&s_cl_in[rank], (uint32_t)lane, s_cl_agg);
                }
                cluster_sync_all();
                if (warp == 0) {
                    const uint32_t rank = cluster_ctarank();
                    Carry v = Carry(0);
                    if ((uint32_t)lane < rank) v = carry_from_bits<Carry>(s_cl_in[lane]);
                    v = warp_reduce_fixed(v);
                    if (lane == 0) s_prefix = s_prefix + v;
                }
            } else {
                cluster_sync_all();
                if (warp == 0) {
                    const uint32_t rank = cluster_ctarank();
                    Carry v = Carry(0);
                    if ((uint32_t)lane < rank) v = carry_from_bits<Carry>(ld_dsmem_u64(&s_cl_agg, (uint32_t)lane));
                    v = warp_reduce_fixed(v);
                    if (lane == 0) s_prefix = s_prefix + v;
                }
                cluster_sync_all();  // no CTA leaves while another may still read its shared memory
            }
        }
        // The output staging buffer we are about to fill must no longer be
        // read by the bulk store issued OSTAGES tiles ago.
        if (tid == 0 && p.tma_out) ptx::bulk_wait_read<OSTAGES - 1>();
        __syncthreads();  // [B] prefix and warp prefixes visible

        // STAGES == 1: claim the next tile only now, when this CTA is free to
        // process it right after its data lands, so its aggregate is published
        // one load latency after the claim, independent of any look-back.
        if (STAGES == 1 && tid == 32) issue(0, iter + 1);

        // ---- a5: epilogue
        const Carry P = s_prefix;
        const Acc wpref = s_warp_pref[warp];
        const bool use_tma_out = p.tma_out && ((m * (int)sizeof(Out)) & 15) == 0;
        Out* ost = out_stage + (size_t)ostage * TILE;
#pragma unroll
        for (int j = 0; j < ROWS; ++j) {
            Acc o[4];
            if constexpr (Tr::kFloat) {
                const float P_hi = (float)P;
                const float P_lo = isfinite(P_hi) ? (float)(P - (double)P_hi) : 0.f;  // inf carry: no inf - inf (R8)
                const float base = P_lo + ((wpref + row_pref[j]) + lane_excl[j]);
                if (p.exclusive) {
                    o[0] = P_hi + base;
                    o[1] = P_hi + (base + v[j][0]);
                    o[2] = P_hi + (base + v[j][1]);
                    o[3] = P_hi + (base + v[j][2]);
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) o[q] = P_hi + (base + v[j][q]);
                }
            } else {
                const Acc base = P + wpref + row_pref[j] + lane_excl[j];
                if (p.exclusive) {
                    o[0] = base;
                    o[1] = base + v[j][0];
                    o[2] = base + v[j][1];
                    o[3] = base + v[j][2];
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) o[q] = base + v[j][q];
                }
            }
            const int e = wbase + j * 128;
            if (use_tma_out) {
                store4(ost + e, o);
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (e + q < m) dst[e + q] = narrow(o[q], (Out*)nullptr);
            }
        }
        if (use_tma_out) {
            ptx::fence_proxy_async_smem();
            __syncthreads();  // [C] staging buffer complete
            if (tid == 0) {
                ptx::tma_store_1d(dst, ost, (uint32_t)(m * (int)sizeof(Out)), pol_out);
                ptx::bulk_commit();
            }
            ostage = (ostage + 1) % OSTAGES;
        } else {
            __syncthreads();  // keep the per-tile barrier count uniform
        }
    }

    if (tid == 0) {
        ptx::bulk_wait<0>();  // all stores done before the CTA (and its smem) retires
        if (!p.static_sched) {
            __threadfence();
            uint32_t prev = ptx::claim_add(&hdr->done, 1u);
            if (prev == gridDim.x - 1) {
                // Last CTA: every other CTA has claimed its final ticket and
                // read the epoch.  Reset the counters and advance the epoch.
                hdr->ticket = 0;
                hdr->done = 0;
                uint32_t e = hdr->epoch + 1;
                if (e == 0) {
                    // Tag wrap (once per 2^32 calls): clear every slot so no
                    // stale tag can match a recycled epoch.
                    uint64_t nslots = (uint64_t)hdr->capacity * (Tr::kFloat ? 4 : 2);
                    for (uint64_t i = 0; i < nslots; ++i) desc[i] = 0;
                    e = 1;
                }
                hdr->epoch = e;
                __threadfence();
            }
        }
    }
}

// ---------------------------------------------------------------- reduction
// scan_total: every thread streams 16-byte vectors (4-deep, so ~64 B per thread are in flight)
// of its chunk in a fixed order, widening every element exactly to int64 /
// fp64 (so |error| <= n 2^-53 sum|x| for floats); then a fixed-order block reduction, and the
// last CTA adds the per-CTA partials in index order (identical bits per call).
template <typename In>
struct Vec16;
template <> struct Vec16<int32_t> { static constexpr int kN = 4; };
template <> struct Vec16<float> { static constexpr int kN = 4; };
template <> struct Vec16<uint16_t> { static constexpr int kN = 8; };
template <> struct Vec16<int8_t> { static constexpr int kN = 16; };

template <typename Sum>
__device__ __forceinline__ Sum to_sum(uint32_t x) { return (Sum)(int32_t)x; }  // ints: sign of the wrap type
template <typename Sum>
__device__ __forceinline__ Sum to_sum(float x) { return (Sum)x; }

template <int DT, typename Sum>
__device__ __forceinline__ Sum sum_vec16(const uint4& q)
{
    using In = typename Traits<DT>::In;
    constexpr int N = Vec16<In>::kN;
    if constexpr (sizeof(In) == 1) {
        // 16 signed bytes: four dp4a (4-way byte dot product with 1,1,1,1)
        int t = __dp4a((int)q.x, 0x01010101, 0);
        t = __dp4a((int)q.y, 0x01010101, t);
        t = __dp4a((int)q.z, 0x01010101, t);
        t = __dp4a((int)q.w, 0x01010101, t);
        return (Sum)t;
    }
    const In* e = reinterpret_cast<const In*>(&q);
    Sum s = 0;
#pragma unroll
    for (int k = 0; k < N; k += 2) {
        if constexpr (Traits<DT>::kFloat)
            s += (double)widen(e[k]) + (double)widen(e[k + 1]);  // every element widened exactly to fp64
        else
            s += (long long)(int32_t)widen(e[k]) + (long long)(int32_t)widen(e[k + 1]);
    }
    return s;
}

template <int DT, int THREADS>
__global__ void __launch_bounds__(THREADS) k_total(const void* in_, int64_t n, void* total_out,
                                                   uint8_t* ws)
{
    using Tr = Traits<DT>;
    using In = typename Tr::In;
    using Sum = typename std::conditional<Tr::kFloat, double, long long>::type;
    constexpr int VN = Vec16<In>::kN;
    const In* in = reinterpret_cast<const In*>(in_);
    WsHeader* hdr = reinterpret_cast<WsHeader*>(ws);
    Sum* partials = reinterpret_cast<Sum*>(ws + kWsPartialsOffset);

    // chunk boundaries in whole 16-byte vectors (the unaligned head goes to CTA 0,
    // the tail past the last whole vector to the last CTA)
    const int64_t head = (int64_t)((16 - ((uintptr_t)in & 15)) & 15) / (int64_t)sizeof(In);
    const int64_t h = head < n ? head : n;
    const int64_t nvec = (n - h) / VN;
    const uint4* vin = reinterpret_cast<const uint4*>(in + h);
    // Grid-stride BACKWARDS from the end of the array with an L2 evict_last
    // hint: the bytes read last are the array's beginning, which the scan
    // that follows (multi-GPU RSS: total, then scan of the same shard) reads
    // first -- up to ~100 MB of the shard is then served by L2, not HBM.
    const uint64_t pol = ptx::policy_evict_last();
    const int64_t T = (int64_t)gridDim.x * THREADS;
    Sum acc = 0;
    int64_t i = nvec - 1 - ((int64_t)blockIdx.x * THREADS + threadIdx.x);
    for (; i - 3 * T >= 0; i -= 4 * T) {
        const uint4 a = ptx::ld_keep_v4(vin + i, pol);
        const uint4 b = ptx::ld_keep_v4(vin + i - T, pol);
        const uint4 c = ptx::ld_keep_v4(vin + i - 2 * T, pol);
        const uint4 d = ptx::ld_keep_v4(vin + i - 3 * T, pol);
        acc += sum_vec16<DT, Sum>(a);
        acc += sum_vec16<DT, Sum>(b);
        acc += sum_vec16<DT, Sum>(c);
        acc += sum_vec16<DT, Sum>(d);
    }
    for (; i >= 0; i -= T) acc += sum_vec16<DT, Sum>(ptx::ld_keep_v4(vin + i, pol));
    if (blockIdx.x == 0)
        for (int64_t j = threadIdx.x; j < h; j += THREADS) acc += to_sum<Sum>(widen(in[j]));
    if (blockIdx.x == gridDim.x - 1)
        for (int64_t j = h + nvec * VN + threadIdx.x; j < n; j += THREADS) acc += to_sum<Sum>(widen(in[j]));
    // block reduction (fixed order)
    __shared__ Sum s_part[THREADS / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        Sum b = 0;
        for (int w = 0; w < THREADS / 32; ++w) b += s_part[w];
        partials[blockIdx.x] = b;
        __threadfence();
        uint32_t prev = ptx::claim_add(&hdr->total_done, 1u);
        if (prev == gridDim.x - 1) {
            __threadfence();
            Sum t = 0;
            for (unsigned c = 0; c < gridDim.x; ++c) t += ((volatile Sum*)partials)[c];
            *reinterpret_cast<Sum*>(total_out) = t;
            hdr->total_done = 0;
        }
    }
}

// carry_r = totals[0] + ... + totals[rank-1], in that order.
template <typename Sum>
__global__ void k_carry_from_totals(const Sum* totals, int rank, Sum* carry_out)
{
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        Sum c = 0;
        for (int r = 0; r < rank; ++r) c += totals[r];
        *carry_out = c;
    }
}

// The <= 15-element head of a 1-D scan whose output is not 16-byte aligned
// (scan_1d then runs the MCScan on the aligned rest): one thread scans it
// sequentially from carry_in (P68 / P461) and leaves carry_in + sum(head) in
// *carry_out (int64 / fp64, the carry_in type) for the body.
template <int DT>
__global__ void k_scan_head(const void* in, void* out, int h, const void* carry_in, int exclusive, void* carry_out)
{
    using Tr = Traits<DT>;
    using In = typename Tr::In;
    using Out = typename Tr::Out;
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const In* x = reinterpret_cast<const In*>(in);
    Out* y = reinterpret_cast<Out*>(out);
    if constexpr (Tr::kFloat) {
        double c = carry_in ? *reinterpret_cast<const double*>(carry_in) : 0.0;
        for (int i = 0; i < h; ++i) {
            double xi;
            if constexpr (sizeof(In) == 2) xi = (double)__half2float(__ushort_as_half(x[i]));  // raw binary16 bits
            else xi = (double)x[i];
            if (exclusive) {
                y[i] = (float)c;
                c = c + xi;
            } else {
                c = (i == 0 && !carry_in) ? xi : c + xi;
                y[i] = (float)c;
            }
        }
        *reinterpret_cast<double*>(carry_out) = c;
    } else {
        uint32_t c = carry_in ? (uint32_t)(uint64_t)*reinterpret_cast<const int64_t*>(carry_in) : 0u;
        for (int i = 0; i < h; ++i) {
            const uint32_t xi = (uint32_t)(int32_t)x[i];
            if (exclusive) {
                y[i] = (int32_t)c;
                c += xi;
            } else {
                c += xi;
                y[i] = (int32_t)c;
            }
        }
        *reinterpret_cast<int64_t*>(carry_out) = (int64_t)(int32_t)c;
    }
}

__global__ void k_ws_init(uint8_t* ws, uint32_t capacity)
{
    WsHeader* hdr = reinterpret_cast<WsHeader*>(ws);
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        hdr->magic = kWsMagic;
        hdr->epoch = 1;
        hdr->ticket = 0;
        hdr->done = 0;
        hdr->capacity = capacity;
        hdr->total_done = 0;
        hdr->error = 0;
    }
}

}  // namespace scan

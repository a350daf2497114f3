// mcscan.cuh -- the paper's multi-core scan (MCScan, Alg. 3, P229-261) with
// its "L2 cache splitting" optimisation (Sec. 6.1.1, P332), re-designed for
// B200 (sm_100a) as ONE persistent, cooperative kernel.
//
// Alg. 3 runs Phase I (per block: local scans + a recomputed block reduction
// r_i, P235-243), a SyncAll barrier (P245), and Phase II (per block: partial =
// sum of the first i entries of r, then propagate it through the block,
// P247-254).  L2 splitting (P332) "splits the input into consecutive chunks so
// that the input and intermediate arrays fit in the L2 cache during the
// processing of each chunk ... the last value of each chunk is propagated to
// the next chunk".  On B200 we keep the idea and change the mechanics:
//
//   * a chunk is G contiguous blocks of BT tiles, one block per CTA (G = SMs);
//   * Phase I (job R(c)): each CTA streams its block HBM -> smem with TMA
//     (L2 policy evict_last, so the bytes stay in the 126 MB L2) and reduces
//     it to r[c][b];  it then arrives on the chunk's grid barrier;
//   * Phase II (job S(c)): after the barrier, each CTA forms its carry
//     (chunk carry + r[c][0..b-1] in a fixed order), re-reads its block -- now
//     from L2 -- scans every tile in registers, adds the running carry and
//     streams the result out with TMA bulk stores.  No local scans are ever
//     written to global memory (Alg. 3 writes them to y in Phase I and reads
//     them back in Phase II: 3N+2N traffic; here HBM sees N reads + N writes);
//   * jobs run in the order R(0) R(1) S(0) R(2) S(1) ..., so the barrier of
//     chunk c is normally complete long before S(c) needs it.
//
// Lanes: every compute lane owns 16 CONTIGUOUS elements, so one warp shuffle
// scan serves 16 elements and the epilogue is one add per element.  Conflict-
// free shared-memory access to 64 contiguous bytes per lane needs a swizzled
// layout: 4-byte and 2-byte inputs (and all 4-byte outputs) move through TMA
// *tensor* copies (cp.async.bulk.tensor.2d) over a [rows x 128 B] view of the
// array with CU_TENSOR_MAP_SWIZZLE_128B, which stores 16-byte chunk c of tile
// row R at chunk c ^ (R & 7).  int8 inputs (16 bytes per lane) use plain 1-D
// bulk copies.  Elements past the last full 128-byte row are read / written
// directly by the lanes that own them.
//
// Warp roles: warp 0 producer (TMA loads of the job sequence), warp 1 storer
// (TMA stores), warp 2 coordinator (publishes r[c][b], waits for each chunk's
// barrier and forms the block carries ahead of time), warps 3.. compute
// (reductions and scans).  Carries: uint32 (ints, wraps mod 2^32) or fp64
// (floats), as in k_scan_tiles.
//
// Grid barrier: one u32 arrival counter per chunk in a workspace region only
// this kernel uses (zeroed by scan_workspace_init, reset by the last CTA).
#pragma once
#include <cuda.h>

#include "scan_kernels.cuh"
#include "scan_ws.cuh"  // mbar_wait_prof

namespace scan {

#ifdef SCAN_MC_PROF
constexpr int kMcProf = 25;  // [21..24] (prof build): globaltimer at entry, first tile in, last job done, exit
#else
constexpr int kMcProf = 21;  // [18..20]: coordinator publish -> complete, complete -> sums loaded, chunks
#endif

// Block reductions live in the workspace after the header: r[c][b] (8 bytes
// each, chunk-major); barrier counters in their own region (kWsBarOffset).
// Geometry in TILE units (32-bit: n <= 2^32 elements is <= 2^19 tiles).
struct McGeom {
    int64_t n;          // elements
    int ntiles;         // ceil(n / TILE)
    int full_tiles;     // tiles [0, full_tiles) are whole and inside both TMA views
    int bt;             // tiles per block
    int chunk_tiles;    // g * bt
    int chunks;         // number of chunks
    int g;              // CTAs (blocks per chunk)
};

// Job q of a CTA's sequence with reductions running `ahead` chunks ahead of
// scans: R(0)..R(ahead), then S(0) R(ahead+1) S(1) R(ahead+2) ..., then the
// remaining S jobs.  Returns the chunk and whether it is a scan (S) job.
__device__ __forceinline__ void mc_job(int q, int chunks, int ahead, int& c, bool& is_scan)
{
    const int F = chunks < ahead + 1 ? chunks : ahead + 1;  // leading reductions
    if (q < F) {
        c = q;
        is_scan = false;
        return;
    }
    const int qq = q - F;
    const int P = chunks - F;  // (S, R) pairs
    if (qq < 2 * P) {
        c = (qq & 1) ? (qq >> 1) + F : (qq >> 1);
        is_scan = (qq & 1) == 0;
    } else {
        c = P + (qq - 2 * P);
        is_scan = true;
    }
}

// Ring position: slot index and the parity of its current use.
template <int NB>
struct Ring {
    int s = 0;
    uint32_t ph = 0;
    bool wrapped = false;  // true once every slot has been used at least once
    __device__ __forceinline__ void next()
    {
        if (++s == NB) {
            s = 0;
            ph ^= 1u;
            wrapped = true;
        }
    }
};

struct McParams16 {
    CUtensorMap tm_in;      // 2-D [rows x 128 B] view of the input (unused for int8)
    CUtensorMap tm_out;     // 2-D [rows x 128 B] view of the output
    const void* in;
    void* out;
    const void* carry_in;   // nullable: int64 (ints) / double (floats)
    uint8_t* ws;
    McGeom gm;
    int64_t n_tma_in;       // elements covered by tm_in (full rows) / by bulk copies
    int64_t n_tma_out;      // elements covered by tm_out (full rows)
    int exclusive;
    int debug;
    int ahead;              // reduce jobs run this many chunks ahead of scan jobs (1..4)
    int l2;                 // L2 policies: bits 0-1 Phase-I read, bits 2-3 Phase-II re-read (0 = default),
                            // bits 4-5 after the re-read: 1 discard / 2 demote the tile's lines,
                            // bits 6-7 the output stores' policy (0 evict_first)
    int64_t seg_len;        // > 0: segmented scan of contiguous rows of seg_len >= TILE elements
                            // (carries reset at every row start); 0: one 1-D scan
    int lazy_carry;         // Phase II waits for the block carry only at the first tile's emit
    int bar_mode;           // chunk barrier: 0 = release-add counter per chunk, then the block sums;
                            // 1 = block sums as epoch-tagged words polled directly (one L2 round
                            // trip after the last publish instead of two)
    int wait_mode;          // mbarrier waits: bit 0 producer / storer, bit 1 compute warps sleep in the
                            // barrier unit (suspend-time hint) instead of spinning
    int shift;              // SHIFT instantiation: the input starts `shift` elements past a 16-byte
                            // boundary; tm_in / the bulk copies address that aligned-down base
    CUtensorMap tm_in1;     // SHIFT, 2-/4-byte inputs: the same view with a one-row box (the row
                            // after a tile, which holds its last `shift` elements)
};

template <int DT, int NC, int GPW, int NB_IN, int NB_OUT, bool SHIFT = false>
struct Mc16Cfg {
    using Tr = Traits<DT>;
    using In = typename Tr::In;
    static constexpr int kThreads = (3 + NC) * 32;
    static constexpr int kTile = NC * GPW * 512;  // 32 lanes x 16 elements per group
    static constexpr size_t kInSlot = (size_t)kTile * sizeof(In);
    static constexpr size_t kOutSlot = (size_t)kTile * 4;
    static constexpr int kRowElemsIn = 128 / (int)sizeof(In);          // elements per 128-B row
    // TMA boxes: up to 256 rows of 128 B each (the box-dimension limit)
    static constexpr int box_rows(size_t rows)
    {
        for (int k = 1; k <= 64; ++k)
            if (rows % k == 0 && rows / k <= 256 && (rows / k) % 8 == 0) return (int)(rows / k);
        return 0;
    }
    static constexpr int kBoxRowsIn = box_rows(kInSlot / 128);
    static constexpr int kBoxRowsOut = box_rows(kOutSlot / 128);
    static constexpr int kBoxesIn = sizeof(In) == 1 ? 0 : (int)(kInSlot / (kBoxRowsIn * 128));
    static constexpr int kBoxesOut = (int)(kOutSlot / (kBoxRowsOut * 128));
    static_assert(sizeof(In) == 1 || kInSlot % (kBoxRowsIn * 128) == 0, "whole TMA boxes per tile");
    static_assert(kOutSlot % (kBoxRowsOut * 128) == 0, "whole TMA boxes per tile");
    static_assert(sizeof(In) == 1 || kBoxRowsIn > 0, "input boxes of whole 1024-B swizzle phases");
    static_assert(kBoxRowsOut > 0, "output boxes of whole 1024-B swizzle phases");
    // NB_OUT == 0: unified ring -- NB_IN slots of kOutSlot bytes; a scan tile's
    // outputs are written in place over its input after the per-tile named
    // barrier, and the storer frees the slot once its store has read it.
    static constexpr bool kUni = NB_OUT == 0;
    // SHIFT: a tile also needs the 128-B row after it (its last `shift`
    // elements).  1-byte inputs (linear slots): each slot is 128 B longer.
    // 2-/4-byte inputs (swizzled slots): the extra rows sit together after the
    // ring, row s for slot s, so every slot keeps its 1024-B swizzle phase.
    static constexpr size_t kRingSlot = kUni ? kOutSlot : kInSlot + ((SHIFT && sizeof(In) == 1) ? 128 : 0);
    static constexpr size_t up1k(size_t b) { return (b + 1023) & ~(size_t)1023; }
    static constexpr size_t kExtraOff = up1k(NB_IN * kRingSlot);
    static constexpr size_t kOutOff = kUni ? 0 : up1k(kExtraOff + ((SHIFT && sizeof(In) > 1) ? NB_IN * 128 : 0));
    static constexpr size_t kSmem = kUni ? NB_IN * kOutSlot + 1024 : kOutOff + NB_OUT * kOutSlot + 1024;
    static_assert(!(SHIFT && kUni), "shifted input needs a separate input ring");
    static_assert(!SHIFT || NB_IN <= 8, "extra rows: one swizzle phase");
};

// ---- 16 contiguous elements of lane-offset e0 from a swizzled slot -----------
// 4-byte elements: row R = e0/32, half h = (e0/16)&1, chunks 4h..4h+3.
__device__ __forceinline__ uint32_t swz4(int e0, int j)
{
    const int R = e0 >> 5;
    return (uint32_t)(R * 128 + ((((e0 >> 2) & 7) + j) ^ (R & 7)) * 16);
}
// 2-byte elements: row R = e0/64, quarter q = (e0/16)&3, chunks 2q, 2q+1.
__device__ __forceinline__ uint32_t swz2(int e0, int j)
{
    const int R = e0 >> 6;
    return (uint32_t)(R * 128 + ((((e0 >> 3) & 7) + j) ^ (R & 7)) * 16);
}
// Byte offset of ONE element e (any e) in a swizzled slot.
template <int SZ>
__device__ __forceinline__ uint32_t swz_elem(int e)
{
    if constexpr (SZ == 4) {
        const int R = e >> 5;
        return (uint32_t)(R * 128 + ((((e >> 2) & 7)) ^ (R & 7)) * 16 + (e & 3) * 4);
    } else if constexpr (SZ == 2) {
        const int R = e >> 6;
        return (uint32_t)(R * 128 + ((((e >> 3) & 7)) ^ (R & 7)) * 16 + (e & 7) * 2);
    } else {
        return (uint32_t)e;
    }
}

// ---- one lane's group of 16 contiguous elements, as raw input words ------------
// SZ = sizeof(In): 16 words (4-byte), 8 words (fp16 pairs) or 4 words (int8 quads).
template <int SZ>
struct Grp {
    uint32_t w[4 * SZ];
};

// Full group from a swizzled (4-/2-byte) or linear (1-byte) ring slot.
template <int SZ>
__device__ __forceinline__ void grp_load(const uint8_t* slot, int e0, Grp<SZ>& g)
{
#pragma unroll
    for (int j = 0; j < SZ; ++j) {
        uint32_t off;
        if constexpr (SZ == 4) off = swz4(e0, j);
        else if constexpr (SZ == 2) off = swz2(e0, j);
        else off = (uint32_t)e0;
        const uint4 q = *reinterpret_cast<const uint4*>(slot + off);
        g.w[4 * j] = q.x; g.w[4 * j + 1] = q.y; g.w[4 * j + 2] = q.z; g.w[4 * j + 3] = q.w;
    }
}

// Ragged group: element e0+k is read from the slot below m_tma, from global
// memory below m, and is 0 (the identity) beyond.
template <int SZ>
__device__ __forceinline__ uint32_t raw_bits(const void* p)
{
    if constexpr (SZ == 4) return *reinterpret_cast<const uint32_t*>(p);
    else if constexpr (SZ == 2) return *reinterpret_cast<const uint16_t*>(p);
    else return *reinterpret_cast<const uint8_t*>(p);
}
// SHIFT, swizzled slots: byte address of slot position `pos` -- positions past
// the tile (pos >= tile) live in the slot's extra row `xrow`, whose swizzle
// phase is the slot index xs (extra rows are 128 B apart from a 1-KB boundary).
template <int SZ>
__device__ __forceinline__ const uint8_t* shift_elem(const uint8_t* slot, const uint8_t* xrow, int xs, int pos, int tile)
{
    if (SZ == 1 || pos < tile) return slot + swz_elem<SZ>(pos);
    const int r = pos - tile;  // position within the extra row
    constexpr int EPC = 16 / SZ;
    return xrow + (((r / EPC) ^ xs) * 16) + (r % EPC) * SZ;
}

template <int SZ>
__device__ __forceinline__ void grp_load_tail(const uint8_t* slot, const uint8_t* gin_tile, int e0, int m,
                                              int m_tma, Grp<SZ>& g, int shift = 0, const uint8_t* xrow = nullptr,
                                              int xs = 0, int tile = 1 << 30)
{
#pragma unroll
    for (int j = 0; j < 4 * SZ; ++j) g.w[j] = 0u;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int e = e0 + k;
        uint32_t bits = 0u;
        if (e < m_tma) bits = raw_bits<SZ>(shift_elem<SZ>(slot, xrow, xs, e + shift, tile));
        else if (e < m) bits = raw_bits<SZ>(gin_tile + (size_t)e * SZ);
        g.w[(k * SZ) / 4] |= bits << ((k * SZ * 8) & 31);
    }
}

// fp16 (raw binary16 in the low / high half of w) + fp32 -> fp32 with ONE
// rounding: sm_100's mixed-precision add (SASS FHADD, .H1 operand select), so
// widening costs no instruction of its own.
__device__ __forceinline__ float fhadd_lo(uint32_t w, float c)
{
    float d;
    asm("{.reg .f16 l, h; mov.b32 {l, h}, %1; add.rn.f32.f16 %0, l, %2;}" : "=f"(d) : "r"(w), "f"(c));
    return d;
}
__device__ __forceinline__ float fhadd_hi(uint32_t w, float c)
{
    float d;
    asm("{.reg .f16 l, h; mov.b32 {l, h}, %1; add.rn.f32.f16 %0, h, %2;}" : "=f"(d) : "r"(w), "f"(c));
    return d;
}

// int8: c + (signed byte sum of w selected by mask), exact mod 2^32 (IDP.4A).
__device__ __forceinline__ uint32_t dp4(uint32_t w, uint32_t mask, uint32_t c)
{
    return (uint32_t)__dp4a((int)w, (int)mask, (int)c);
}

// Reduction of a group (Phase I).  Floats: fp32 partials, widened to the fp64 carry.
__device__ __forceinline__ uint32_t grp_sum(const Grp<4>& g, const int32_t*)
{
    uint32_t s[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) s[j] = (g.w[4 * j] + g.w[4 * j + 1]) + (g.w[4 * j + 2] + g.w[4 * j + 3]);
    return (s[0] + s[1]) + (s[2] + s[3]);
}
__device__ __forceinline__ double grp_sum(const Grp<4>& g, const float*)
{
    float s8[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) s8[k] = __uint_as_float(g.w[2 * k]) + __uint_as_float(g.w[2 * k + 1]);
    const float a = (s8[0] + s8[1]) + (s8[2] + s8[3]);
    const float b = (s8[4] + s8[5]) + (s8[6] + s8[7]);
    return (double)(a + b);
}
__device__ __forceinline__ double grp_sum(const Grp<2>& g, const uint16_t*)
{
    float a = -0.0f, b = -0.0f;  // two independent FHADD chains (elements 0-7, 8-15)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        a = fhadd_hi(g.w[j], fhadd_lo(g.w[j], a));
        b = fhadd_hi(g.w[4 + j], fhadd_lo(g.w[4 + j], b));
    }
    return (double)(a + b);
}
__device__ __forceinline__ uint32_t grp_sum(const Grp<1>& g, const int8_t*)
{
    uint32_t s = 0u;
#pragma unroll
    for (int j = 0; j < 4; ++j) s = dp4(g.w[j], 0x01010101u, s);
    return s;
}

// In-lane inclusive prefix v[k] = x_0 + ... + x_k (4- and 2-byte inputs).
__device__ __forceinline__ void grp_prefix(const Grp<4>& g, uint32_t (&v)[16], const int32_t*)
{
    v[0] = g.w[0];
#pragma unroll
    for (int k = 1; k < 16; ++k) v[k] = v[k - 1] + g.w[k];
}
__device__ __forceinline__ void grp_prefix(const Grp<4>& g, float (&v)[16], const float*)
{
    v[0] = __uint_as_float(g.w[0]);
#pragma unroll
    for (int k = 1; k < 16; ++k) v[k] = v[k - 1] + __uint_as_float(g.w[k]);
}
__device__ __forceinline__ void grp_prefix(const Grp<2>& g, float (&v)[16], const uint16_t*)
{
    v[0] = fhadd_lo(g.w[0], -0.0f);  // exact widening (x + -0 == x, -0 kept)
    v[1] = fhadd_hi(g.w[0], v[0]);
#pragma unroll
    for (int j = 1; j < 8; ++j) {
        v[2 * j] = fhadd_lo(g.w[j], v[2 * j - 1]);
        v[2 * j + 1] = fhadd_hi(g.w[j], v[2 * j]);
    }
}

// int8 epilogue straight from the raw bytes: out = base + prefix of the bytes,
// one IDP.4A per element (masks select bytes 0..k of the word).
__device__ __forceinline__ void grp_emit_i8(const Grp<1>& g, uint32_t B, bool exclusive, uint32_t (&o)[16])
{
    uint32_t b = B;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (exclusive) {
            o[4 * j] = b;
            o[4 * j + 1] = dp4(g.w[j], 0x00000001u, b);
            o[4 * j + 2] = dp4(g.w[j], 0x00000101u, b);
            o[4 * j + 3] = dp4(g.w[j], 0x00010101u, b);
            b = dp4(g.w[j], 0x01010101u, b);
        } else {
            o[4 * j] = dp4(g.w[j], 0x00000001u, b);
            o[4 * j + 1] = dp4(g.w[j], 0x00000101u, b);
            o[4 * j + 2] = dp4(g.w[j], 0x00010101u, b);
            o[4 * j + 3] = dp4(g.w[j], 0x01010101u, b);
            b = o[4 * j + 3];
        }
    }
}

// Zero (the identity, as raw bits) the elements e0+k of a group outside [lo, hi).
template <int SZ>
__device__ __forceinline__ void grp_mask(Grp<SZ>& g, int e0, int lo, int hi)
{
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int e = e0 + k;
        if (e < lo || e >= hi) {
            if constexpr (SZ == 4) g.w[k] = 0u;
            else if constexpr (SZ == 2) g.w[k >> 1] &= (k & 1) ? 0x0000ffffu : 0xffff0000u;
            else g.w[k >> 2] &= ~(0xffu << (8 * (k & 3)));
        }
    }
}

// Segmented scans (rows of seg_len >= TILE elements: at most one row start per
// tile).  A CTA's jobs of one phase visit its block of chunks 0, 1, 2, ... in
// order, so the block start modulo seg_len advances by a constant per job: no
// 64-bit division in the job loop (a division per job cost ~10 % of the kernel).
template <int TILE>
struct SegCursor {
    int64_t rem = 0;        // (first element of this CTA's block in the next job's chunk) mod seg_len
    int tile = 0x7fffffff;  // tile of the next row start in the current job (INT_MAX: none before n)
    int off = 0;            // its offset in that tile
    __device__ __forceinline__ void init(int b, int bt, int64_t seg_len) { rem = ((int64_t)b * bt * TILE) % seg_len; }
    __device__ __forceinline__ void set(int64_t next, int64_t n)
    {
        tile = next < n ? (int)(next / TILE) : 0x7fffffff;
        off = (int)(next - (int64_t)tile * TILE);
    }
    // at the start of a job whose first tile is t0; dchunk = (chunk_tiles * TILE) mod seg_len
    __device__ __forceinline__ void job(int t0, int64_t seg_len, int64_t dchunk, int64_t n)
    {
        set((int64_t)t0 * TILE + (rem == 0 ? 0 : seg_len - rem), n);
        rem += dchunk;
        if (rem >= seg_len) rem -= seg_len;
    }
    // after the row start in `tile` has been consumed
    __device__ __forceinline__ void advance(int64_t seg_len, int64_t n) { set((int64_t)tile * TILE + off + seg_len, n); }
};

// One lane's 16 elements through a tile scan: load raw words, form the lane
// total (int8: IDP.4A byte sums; others: the in-lane inclusive prefix v), then
// emit base + local prefix.  Used by k_mcscan16 and k_rowscan16.
template <int DT>
struct LaneScan {
    using Tr = Traits<DT>;
    using In = typename Tr::In;
    using Acc = typename Tr::Acc;
    static constexpr int SZ = (int)sizeof(In);
    static constexpr bool kBytes = SZ == 1;
    Grp<SZ> g;
    Acc v[kBytes ? 1 : 16];

    __device__ __forceinline__ Acc prefix()
    {
        if constexpr (kBytes) {
            return grp_sum(g, (const In*)nullptr);
        } else {
            grp_prefix(g, v, (const In*)nullptr);
            return v[15];
        }
    }
    __device__ __forceinline__ void emit(Acc B, bool exclusive, Acc (&o)[16]) const
    {
        if constexpr (kBytes) {
            grp_emit_i8(g, B, exclusive, o);
        } else if (exclusive) {
            o[0] = B;
#pragma unroll
            for (int k = 1; k < 16; ++k) o[k] = B + v[k - 1];
        } else {
#pragma unroll
            for (int k = 0; k < 16; ++k) o[k] = B + v[k];
        }
    }
};

template <typename A>
__device__ __forceinline__ void store16(uint8_t* slot, int e0, const A (&o)[16])
{
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        static_assert(sizeof(A) == 4, "4-byte outputs");
        uint4 q;
        q.x = *reinterpret_cast<const uint32_t*>(&o[4 * j]);
        q.y = *reinterpret_cast<const uint32_t*>(&o[4 * j + 1]);
        q.z = *reinterpret_cast<const uint32_t*>(&o[4 * j + 2]);
        q.w = *reinterpret_cast<const uint32_t*>(&o[4 * j + 3]);
        *reinterpret_cast<uint4*>(slot + swz4(e0, j)) = q;
    }
}

// ---- TMA tensor copies -----------------------------------------------------------
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* tm, int x, int y,
                                            uint64_t* bar, uint64_t policy)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(ptx::smem_u32(smem_dst)),
        "l"(tm), "r"(x), "r"(y), "r"(ptx::smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* tm, int x, int y, const void* smem_src,
                                             uint64_t policy)
{
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;" ::"l"(
                     tm),
                 "r"(x), "r"(y), "r"(ptx::smem_u32(smem_src)), "l"(policy)
                 : "memory");
}

// Per-lane byte offsets of the 16-byte chunks of a lane's group 0 inside a
// ring slot; group g of the same lane sits g * kGrp bytes further (the
// swizzle phase R & 7 is the same for every group, 512 elements apart).
template <int SZ>
struct LaneOffsets {
    static constexpr uint32_t kGrpIn = SZ == 4 ? 2048u : (SZ == 2 ? 1024u : 512u);
    static constexpr uint32_t kGrpOut = 2048u;
    uint32_t in[SZ];
    uint32_t out[4];
    __device__ __forceinline__ explicit LaneOffsets(int e0)
    {
#pragma unroll
        for (int j = 0; j < SZ; ++j) in[j] = SZ == 4 ? swz4(e0, j) : (SZ == 2 ? swz2(e0, j) : (uint32_t)e0);
#pragma unroll
        for (int j = 0; j < 4; ++j) out[j] = swz4(e0, j);
    }
};

template <int SZ>
__device__ __forceinline__ void grp_load_off(const uint8_t* base, const uint32_t (&off)[SZ], Grp<SZ>& g)
{
#pragma unroll
    for (int j = 0; j < SZ; ++j) {
        const uint4 q = *reinterpret_cast<const uint4*>(base + off[j]);
        g.w[4 * j] = q.x; g.w[4 * j + 1] = q.y; g.w[4 * j + 2] = q.z; g.w[4 * j + 3] = q.w;
    }
}

// Full group of a SHIFTED slot: the lane's 16 elements sit at slot positions
// e0 + d .. e0 + d + 15 (d = the input's element offset from a 16-byte
// boundary, warp-uniform).  Loads the 16-byte chunks they touch (5 / 3 / 2 for
// 4- / 2- / 1-byte elements, swizzled as the TMA wrote them) and funnel-shifts
// the words into place.
__device__ __forceinline__ uint32_t chunk_off(int q, int SZ)
{
    if (SZ == 1) return (uint32_t)q * 16;
    const int R = q >> 3;
    return (uint32_t)(R * 128 + ((q & 7) ^ (R & 7)) * 16);
}
// DW = whole words to skip (compile time: the word selection is register
// renaming), sh = the remaining bit offset (0 / 8 / 16 / 24, one funnel shift
// per word; always 0 for 4-byte elements).
template <int SZ, int DW>
__device__ __forceinline__ void grp_load_shift(const uint8_t* slot, int e0, uint32_t sh, Grp<SZ>& g,
                                               const uint8_t* xrow, int xs, int tile)
{
    constexpr int EPC = 16 / SZ;              // elements per 16-byte chunk
    constexpr int NQ = SZ == 4 ? 5 : (SZ == 2 ? 3 : 2);
    uint32_t W[4 * NQ];
    const int q0 = e0 / EPC;                  // e0 is a multiple of 16 elements
    const int qt = tile / EPC;                // first chunk past the tile (swizzled slots: the extra row)
    // 32-bit shared-window addresses and explicit ld.shared.v4 (a select between
    // two generic pointers made the compiler fall back to split generic loads)
    const uint32_t s_slot = ptx::smem_u32(slot), s_x = ptx::smem_u32(xrow);
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
        const int q = q0 + j;
        const uint32_t a = (SZ > 1 && q >= qt) ? s_x + (uint32_t)(((q - qt) ^ xs) * 16) : s_slot + chunk_off(q, SZ);
        uint4 v;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "r"(a));
        W[4 * j] = v.x; W[4 * j + 1] = v.y; W[4 * j + 2] = v.z; W[4 * j + 3] = v.w;
    }
    constexpr int NW = 4 * SZ;                // words of the group
    static_assert(DW + NW < 4 * NQ + 1, "chunks cover the shifted group");
    if constexpr (SZ == 4) {
#pragma unroll
        for (int k = 0; k < NW; ++k) g.w[k] = W[DW + k];
    } else {
#pragma unroll
        for (int k = 0; k < NW; ++k) g.w[k] = __funnelshift_r(W[DW + k], (DW + k + 1 < 4 * NQ) ? W[DW + k + 1] : 0u, sh);
    }
}

template <typename A>
__device__ __forceinline__ void store16_off(uint8_t* base, const uint32_t (&off)[4], const A (&o)[16])
{
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        uint4 q;
        q.x = *reinterpret_cast<const uint32_t*>(&o[4 * j]);
        q.y = *reinterpret_cast<const uint32_t*>(&o[4 * j + 1]);
        q.z = *reinterpret_cast<const uint32_t*>(&o[4 * j + 2]);
        q.w = *reinterpret_cast<const uint32_t*>(&o[4 * j + 3]);
        *reinterpret_cast<uint4*>(base + off[j]) = q;
    }
}

// ---- segmented scans: the tile holding a row start at offset ro > 0 -------------
// Phase I: this lane's share of the sum of the tile's elements [ro, TILE).
template <int DT, int GPW>
__device__ __forceinline__ typename Traits<DT>::Carry mc_split_sum(const uint8_t* slot, const uint8_t* gin_tile, int e0_base,
                                                                int m, int m_in, int ro)
{
    using Tr = Traits<DT>;
    using Carry = typename Tr::Carry;
    constexpr int SZ = (int)sizeof(typename Tr::In);
    Carry sum = Carry(0);
#pragma unroll 1
    for (int g = 0; g < GPW; ++g) {
        Grp<SZ> gr;
        grp_load_tail(slot, gin_tile, e0_base + 512 * g, m, m_in, gr);
        grp_mask(gr, e0_base + 512 * g, ro, 1 << 30);
        sum = sum + Carry(grp_sum(gr, (const typename Tr::In*)nullptr));
    }
    return sum;
}

// Phase II: two masked passes over the slot -- [0, ro) with the running carry,
// [ro, TILE) from 0 -- each a full tile scan (NC compute warps, named barrier 1,
// s_wt[(s_count + pass) & 1]); outputs stored element-wise.  Returns the
// aggregate of [ro, TILE), the new row's running sum.
template <int DT, int NC, int GPW, int TILE>
__device__ __forceinline__ typename Traits<DT>::Acc mc_split_tile(
    const uint8_t* slot, uint8_t* ost, const uint8_t* gin_tile, typename Traits<DT>::Out* gout_tile, bool full, int m,
    int m_in, int m_out, int ro, typename Traits<DT>::Carry carry, bool exclusive, int e0_base,
    const LaneOffsets<(int)sizeof(typename Traits<DT>::In)> off, typename Traits<DT>::Acc* s_wt, int s_count, int lane,
    int cw)
{
    using Tr = Traits<DT>;
    using Acc = typename Tr::Acc;
    using Carry = typename Tr::Carry;
    using Out = typename Tr::Out;
    constexpr int SZ = (int)sizeof(typename Tr::In);
    constexpr uint32_t GI = LaneOffsets<SZ>::kGrpIn;
    Acc agg = Acc(0);
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
        const int lo = pass ? ro : 0, hi = pass ? TILE : ro;
        const Carry cin = pass ? Carry(0) : carry;
        LaneScan<DT> ls[GPW];
        Acc ex[GPW], gp[GPW];
        Acc wsum = Acc(0);
#pragma unroll
        for (int g = 0; g < GPW; ++g) {
            if (full)
                grp_load_off(slot + g * GI, off.in, ls[g].g);
            else
                grp_load_tail(slot, gin_tile, e0_base + 512 * g, m, m_in, ls[g].g);
            grp_mask(ls[g].g, e0_base + 512 * g, lo, hi);
            ex[g] = ls[g].prefix();
        }
#pragma unroll
        for (int g = 0; g < GPW; ++g) {
            const Acc incl = warp_incl_scan(ex[g], lane);
            const Acc e1 = __shfl_up_sync(0xffffffffu, incl, 1);
            ex[g] = lane == 0 ? Acc(0) : e1;
            gp[g] = wsum;
            wsum = wsum + __shfl_sync(0xffffffffu, incl, 31);
        }
        Acc* wt = s_wt + ((s_count + pass) & 1) * NC;
        if (lane == 0) wt[cw] = wsum;
        named_bar_sync(1, NC * 32);
        const Acc x = lane < NC ? wt[lane] : Acc(0);
        const Acc xi = warp_incl_scan(x, lane);
        const Acc xe = __shfl_up_sync(0xffffffffu, xi, 1);
        const Acc wpref = __shfl_sync(0xffffffffu, lane == 0 ? Acc(0) : xe, cw);
        agg = __shfl_sync(0xffffffffu, xi, NC - 1);
#pragma unroll
        for (int g = 0; g < GPW; ++g) {
            Acc B;
            if constexpr (Tr::kFloat)
                B = (float)(cin + (double)((wpref + gp[g]) + ex[g]));
            else
                B = cin + wpref + gp[g] + ex[g];
            Acc o16[16];
            ls[g].emit(B, exclusive, o16);
            const int e0 = e0_base + 512 * g;
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const int e = e0 + k;
                if (e < lo || e >= hi) continue;
                if (e < m_out)
                    *reinterpret_cast<Acc*>(ost + swz_elem<4>(e)) = o16[k];
                else if (e < m)
                    gout_tile[e] = narrow(o16[k], (Out*)nullptr);
            }
        }
    }
    return agg;
}

// SEG: segmented scan of contiguous rows (p.seg_len); a separate instantiation so
// the 1-D kernels carry none of its code.
// SH > 0: the input starts p.shift elements past a 16-byte boundary, with
// (p.shift * sizeof(In)) / 4 == SH - 1 whole words (one instantiation each).
template <int DT, int NC, int GPW, int NB_IN, int NB_OUT, bool SEG = false, int SH = 0>
__global__ void __launch_bounds__((3 + NC) * 32, 1) k_mcscan16(const __grid_constant__ McParams16 p)
{
    constexpr bool SHIFT = SH > 0;
    constexpr int DW = SH > 0 ? SH - 1 : 0;
    static_assert(!(SEG && SHIFT), "shifted input: 1-D scans only");
    using Cfg = Mc16Cfg<DT, NC, GPW, NB_IN, NB_OUT, SHIFT>;
    using Tr = Traits<DT>;
    using In = typename Tr::In;
    using Out = typename Tr::Out;
    using Acc = typename Tr::Acc;
    using Carry = typename Tr::Carry;
    constexpr int TILE = Cfg::kTile;
    constexpr int SZ = (int)sizeof(In);
    constexpr int KC = 8;  // carry ring (ahead <= 4)
    constexpr int RS = 8;  // reduce-sum hand-off ring (ahead <= 4)

    extern __shared__ uint8_t smem_raw[];
    // 1024-B aligned ring base.  By pointer arithmetic the compiler keeps the
    // shared-memory provenance (LDS / STS on 32-bit addresses); through an integer
    // round trip it loses it and emits generic LD.E / ST.E with 64-bit address
    // math for every slot access.  Measured (DESIGN 5.1, same box, 3 runs each):
    // shared C2 83.0 -> 86.6 %, C3 90.5 -> 91.5 %, shifted C5 -> 91.1 %.  The
    // aligned 4-byte kernel (C5) kept the generic form until the fourth session of
    // round 2 because it is 1.5 points faster in a burst (92.1 vs 90.6 %); under
    // the power cap the lighter form holds 91.6 % where the generic one falls to
    // 82-88 % (DESIGN 8.1), so every instantiation now takes the shared form
    // (-DSCAN_MC_GENERIC4 restores the old one for A/B).
#ifdef SCAN_MC_GENERIC4
    constexpr bool kGenericBase = (SZ == 4 && SH == 0 && !SEG);
#else
    constexpr bool kGenericBase = false;
#endif
    uint8_t* const smem =
        kGenericBase ? reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023)
                     : smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    constexpr bool UNI = Cfg::kUni;
    constexpr int NSR = UNI ? NB_IN : NB_OUT;  // store_ready / out slots
    uint8_t* const in_ring = smem;
    uint8_t* const out_ring = UNI ? smem : smem + Cfg::kOutOff;
    uint8_t* const extra_rows = smem + Cfg::kExtraOff;  // SHIFT, 2-/4-byte inputs: row s for slot s

    __shared__ __align__(8) uint64_t in_full[NB_IN];
    __shared__ __align__(8) uint64_t in_empty[NB_IN];
    __shared__ __align__(8) uint64_t store_ready[NSR];
    __shared__ __align__(8) uint64_t out_empty[NSR];
    __shared__ __align__(8) uint64_t carry_ready[KC];
    __shared__ __align__(8) uint64_t rsum_ready[RS];
    __shared__ Acc s_wt[2][NC];
    __shared__ Carry s_job_sum[RS][NC];
    __shared__ Carry s_carry[KC];
    __shared__ unsigned long long s_prof[kMcProf];

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const McGeom& gm = p.gm;
    const int b = blockIdx.x;
    const int njobs = gm.chunks * 2;
    // Per-CTA stall counters (SCAN_DEBUG=4).  Their clock reads cost ~14
    // instructions per 1,024 elements even when off (C2 84.2 -> 86.6 % without
    // them), so they are compiled in only with -DSCAN_MC_PROF (profiles/
    // mc_counters.py, mc_timeline.py) or, for the aligned 4-byte kernel, with
    // -DSCAN_MC_GENERIC4 (the pre-8.1 form of that kernel, which kept them).
#ifdef SCAN_MC_GENERIC4
    constexpr bool kProfRuntime = (sizeof(In) == 4 && SH == 0 && !SEG);
#else
    constexpr bool kProfRuntime = false;
#endif
#ifdef SCAN_MC_PROF
    const bool prof = (p.debug & 4) != 0;
#else
    const bool prof = kProfRuntime && (p.debug & 4) != 0;
#endif
    const long long t_start = clock64();
#ifdef SCAN_MC_PROF
    const unsigned long long g_entry = ptx::globaltimer();
#endif

    WsHeader* hdr = reinterpret_cast<WsHeader*>(p.ws);
    uint64_t* r_all = reinterpret_cast<uint64_t*>(p.ws + kWsDescOffset);
    uint32_t* bar = reinterpret_cast<uint32_t*>(p.ws + kWsBarOffset);
    const In* gin = reinterpret_cast<const In*>(p.in);
    Out* gout = reinterpret_cast<Out*>(p.out);

    if (tid < kMcProf) s_prof[tid] = 0;
#ifdef SCAN_MC_PROF
    if (tid == 0) s_prof[21] = g_entry;
#endif
    if (tid == 0) {
        for (int s = 0; s < NB_IN; ++s) {
            ptx::mbar_init(&in_full[s], 1);
            ptx::mbar_init(&in_empty[s], NC);
        }
        for (int o = 0; o < NSR; ++o) {
            ptx::mbar_init(&store_ready[o], NC);
            ptx::mbar_init(&out_empty[o], 1);
        }
        for (int k = 0; k < KC; ++k) ptx::mbar_init(&carry_ready[k], 1);
        for (int k = 0; k < RS; ++k) ptx::mbar_init(&rsum_ready[k], NC);
        ptx::fence_mbar_init();
    }
    __syncthreads();

    // Tiles [t0, t1) of block b of chunk c.
    auto block_tiles = [&](int c, int& t0, int& t1) {
        t0 = c * gm.chunk_tiles + b * gm.bt;
        t1 = t0 + gm.bt;
        if (t0 > gm.ntiles) t0 = gm.ntiles;
        if (t1 > gm.ntiles) t1 = gm.ntiles;
    };

    if (warp == 0) {
        // =========================== producer ===========================
        if (lane == 0) {
            // L2 policy of the Phase-I read (kept for the Phase-II re-read) and
            // of the re-read (dead afterwards); p.l2 selects alternatives (A/B)
            uint64_t pol_keep, pol_drop;
            switch (p.l2 & 3) {
            case 1: pol_keep = ptx::policy_evict_normal(); break;
            case 2: pol_keep = ptx::policy_evict_last_frac(0.5f); break;
            case 3: pol_keep = ptx::policy_evict_unchanged(); break;
            default: pol_keep = ptx::policy_evict_last(); break;
            }
            switch ((p.l2 >> 2) & 3) {
            case 1: pol_drop = ptx::policy_evict_normal(); break;
            case 2: pol_drop = ptx::policy_evict_unchanged(); break;
            default: pol_drop = ptx::policy_evict_first(); break;
            }
            Ring<NB_IN> rin;
            for (int q = 0; q < njobs; ++q) {
                int c, t0, t1;
                bool is_scan;
                mc_job(q, gm.chunks, p.ahead, c, is_scan);
                block_tiles(c, t0, t1);
                const uint64_t pol = is_scan ? pol_drop : pol_keep;
                for (int t = t0; t < t1; ++t, rin.next()) {
                    if (rin.wrapped) {
                        if (p.wait_mode & 1)
                            ptx::mbar_wait_sleep(&in_empty[rin.s], rin.ph ^ 1u);
                        else
                            ptx::mbar_wait(&in_empty[rin.s], rin.ph ^ 1u);
                    }
                    uint8_t* dst = in_ring + rin.s * Cfg::kRingSlot;
                    if constexpr (SZ == 1) {
                        // SHIFT: bytes from the 16-byte boundary below the tile's first
                        // element, up to 16 past its end (all 16-byte multiples)
                        const int64_t g0 = (int64_t)t * TILE;
                        int64_t m_tma = p.n_tma_in + (SHIFT ? p.shift : 0) - g0;
                        const int64_t cap = SHIFT ? TILE + 16 : TILE;
                        m_tma = m_tma < 0 ? 0 : (m_tma > cap ? cap : m_tma);
                        if (m_tma > 0) {
                            ptx::mbar_arrive_expect_tx(&in_full[rin.s], (uint32_t)m_tma);
                            ptx::tma_load_1d(dst, gin + g0 - (SHIFT ? p.shift : 0), (uint32_t)m_tma, &in_full[rin.s],
                                             pol);
                        } else {
                            ptx::mbar_arrive(&in_full[rin.s]);
                        }
                    } else {
                        ptx::mbar_arrive_expect_tx(&in_full[rin.s], (uint32_t)Cfg::kInSlot + (SHIFT ? 128u : 0u));
                        const int y0 = t * (TILE / Cfg::kRowElemsIn);
#pragma unroll
                        for (int k = 0; k < Cfg::kBoxesIn; ++k)
                            tma_load_2d(dst + k * Cfg::kBoxRowsIn * 128, &p.tm_in, 0, y0 + Cfg::kBoxRowsIn * k,
                                        &in_full[rin.s], pol);
                        if constexpr (SHIFT)  // the row after the tile (its last `shift` elements)
                            tma_load_2d(extra_rows + rin.s * 128, &p.tm_in1, 0, y0 + TILE / Cfg::kRowElemsIn,
                                        &in_full[rin.s], pol);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // =========================== storer ===========================
        if (lane == 0) {
            // output stores: evict_first (default); p.l2 bits 6-7 = 1 evict_normal,
            // 2 evict_unchanged, 3 evict_last (A/B of the L2 residency of the re-read)
            const int sp_ = (p.l2 >> 6) & 3;
            const uint64_t pol = sp_ == 1 ? ptx::policy_evict_normal()
                                 : sp_ == 2 ? ptx::policy_evict_unchanged()
                                 : sp_ == 3 ? ptx::policy_evict_last()
                                            : ptx::policy_evict_first();
            Ring<NB_IN> rin;    // UNI: outputs sit in the input slots
            Ring<NSR> rout;
            uint32_t sparity = 0;  // UNI: bit s = parity of the next store_ready[s] phase (S tiles only)
            int pend = -1;         // slot whose store may still be reading shared memory
            auto release = [&](int slot) {
                if (UNI)
                    ptx::mbar_arrive_cnt(&in_empty[slot], NC);  // counts as the NC compute arrivals
                else
                    ptx::mbar_arrive(&out_empty[slot]);
            };
            for (int q = 0; q < njobs; ++q) {
                int c, t0, t1;
                bool is_scan;
                mc_job(q, gm.chunks, p.ahead, c, is_scan);
                block_tiles(c, t0, t1);
                if (!is_scan) {
                    if (UNI)
                        for (int t = t0; t < t1; ++t) rin.next();
                    continue;
                }
                for (int t = t0; t < t1; ++t, rin.next(), rout.next()) {
                    const int o = UNI ? rin.s : rout.s;
                    const uint32_t par = UNI ? ((sparity >> o) & 1u) : rout.ph;
                    if (pend >= 0 && !ptx::mbar_try_wait(&store_ready[o], par)) {
                        // about to block: release the pending slot first
                        ptx::bulk_wait_read<0>();
                        release(pend);
                        pend = -1;
                    }
                    mbar_wait_prof(&store_ready[o], par, prof, &s_prof[5], (p.wait_mode & 1) != 0);
                    if (UNI) sparity ^= 1u << o;
                    if ((int64_t)t * TILE < p.n_tma_out) {
                        const int y0 = t * (TILE / 32);
#pragma unroll
                        for (int k = 0; k < Cfg::kBoxesOut; ++k)
                            tma_store_2d(&p.tm_out, 0, y0 + Cfg::kBoxRowsOut * k,
                                         out_ring + o * Cfg::kOutSlot + k * Cfg::kBoxRowsOut * 128, pol);
                        ptx::bulk_commit();
                        if (pend >= 0) {  // keep two stores in flight; retire the older one
                            const long long w0 = prof ? clock64() : 0;
                            ptx::bulk_wait_read<1>();
                            if (prof) atomicAdd(&s_prof[6], (unsigned long long)(clock64() - w0));
                            release(pend);
                        }
                        pend = o;
                    } else {
                        release(o);
                    }
                }
            }
            ptx::bulk_wait<0>();
        }
    } else if (warp == 2) {
        // ========================= coordinator =========================
        Carry chunk_carry = Carry(0);
        if (p.carry_in != nullptr) {
            if constexpr (Tr::kFloat)
                chunk_carry = *reinterpret_cast<const double*>(p.carry_in);
            else
                chunk_carry = (uint32_t)(uint64_t)(*reinterpret_cast<const int64_t*>(p.carry_in));
        }
        constexpr int RPL = kMaxGridPerLane;
        // Event loop: publish r[c][b] as soon as the compute warps' reduction
        // of chunk c is in (fixed-order sum of their sums, release-add on the
        // chunk barrier), and form the carry of chunk c as soon as its barrier
        // is complete (SyncAll P245; partial = sum of the first b entries of r,
        // P248) -- whichever is ready first, so neither waits on the other.
        int next_pub = 0, next_car = 0;
        uint32_t backoff = 32;
        // tagged mode: block sums are (call epoch << 32 | payload) words, 2 per sum for
        // fp64 (high / low halves); the epoch is the workspace's call counter, advanced
        // by the last CTA, so no word of an earlier call carries it
        const bool tagged = p.bar_mode == 1;
        long long t_pub[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // prof: clock at the publish of chunk c (c % 8)
        constexpr int RW = Tr::kFloat ? 2 : 1;
        const uint64_t tagw = (uint64_t)hdr->epoch << 32;
        int64_t seg_rem[SEG ? RPL : 1], seg_dc = 0;  // SEG: (start of block lane+32k of chunk next_car) mod seg_len
        if constexpr (SEG) {
            seg_dc = ((int64_t)gm.chunk_tiles * TILE) % p.seg_len;
#pragma unroll
            for (int k = 0; k < RPL; ++k) seg_rem[k] = ((int64_t)(lane + 32 * k) * gm.bt * TILE) % p.seg_len;
        }
        long long spin0 = 0;
        while (next_car < gm.chunks) {
            bool progressed = false;
            // lane 0's poll decides for the warp: every branch below must be
            // warp-uniform (lanes polling on their own can disagree, and then
            // the shuffles / __syncwarp further down diverge -- found by the
            // fault-injection build, tests/test_gpu_fuzz.py)
            bool rs_ready = false;
            if (next_pub < gm.chunks && lane == 0)
                rs_ready = ptx::mbar_try_wait(&rsum_ready[next_pub % RS], (uint32_t)(next_pub / RS) & 1u);
            rs_ready = __shfl_sync(0xffffffffu, rs_ready, 0);
            if (rs_ready) {
                if (lane == 0) {
                    Carry t = Carry(0);
                    for (int w = 0; w < NC; ++w) t = t + s_job_sum[next_pub % RS][w];
                    if (tagged) {
                        // self-contained tagged words: no fence, no counter
                        const uint64_t bits = carry_bits(t);
                        uint64_t* e = r_all + ((int64_t)next_pub * gm.g + b) * RW;
                        if (RW == 2) {
                            ptx::st_relaxed_u64(e, tagw | (bits >> 32));
                            ptx::st_relaxed_u64(e + 1, tagw | (bits & 0xffffffffull));
                        } else {
                            ptx::st_relaxed_u64(e, tagw | (bits & 0xffffffffull));
                        }
                    } else {
                        r_all[(int64_t)next_pub * gm.g + b] = carry_bits(t);
                        ptx::red_release_add_u32(&bar[next_pub], 1u);  // orders the r store before the arrival
                    }
                }
                __syncwarp();
                if (prof) t_pub[next_pub & 7] = clock64();
                ++next_pub;
                progressed = true;
            }
            if (next_car < next_pub) {
                uint64_t rb[RPL];
                bool ready;
                if (tagged) {
                    // every block sum of chunk next_car, tags checked: all present -> ready
                    bool mine = true;
#pragma unroll
                    for (int k = 0; k < RPL; ++k) {
                        const int bb = lane + 32 * k;
                        rb[k] = 0ull;
                        if (bb < gm.g) {
                            const uint64_t* e = r_all + ((int64_t)next_car * gm.g + bb) * RW;
                            const uint64_t w0 = ld_relaxed_u64(e);
                            const uint64_t w1 = RW == 2 ? ld_relaxed_u64(e + 1) : tagw;
                            mine = mine && (w0 >> 32) == (tagw >> 32) && (w1 >> 32) == (tagw >> 32);
                            rb[k] = RW == 2 ? ((w0 << 32) | (w1 & 0xffffffffull)) : (w0 & 0xffffffffull);
                        }
                    }
                    ready = __all_sync(0xffffffffu, mine);
                } else {
                    uint32_t arrived = lane == 0 ? ld_acquire_u32(&bar[next_car]) : 0u;
                    arrived = __shfl_sync(0xffffffffu, arrived, 0);
                    ready = arrived >= (uint32_t)gm.g;
                    const long long t_rdy = prof ? clock64() : 0;
                    if (ready) {
#pragma unroll
                        for (int k = 0; k < RPL; ++k) {
                            const int bb = lane + 32 * k;
                            rb[k] = bb < gm.g ? ld_relaxed_u64(&r_all[(int64_t)next_car * gm.g + bb]) : 0ull;
                        }
                        if (prof) {
                            uint64_t acc = 0;
#pragma unroll
                            for (int k = 0; k < RPL; ++k) acc ^= rb[k];
                            acc = __shfl_sync(0xffffffffu, acc, 0);  // the loads have landed
                            if (lane == 0) {
                                const long long t_val = clock64() + (long long)(acc & 0);
                                s_prof[18] += (unsigned long long)(t_rdy - t_pub[next_car & 7]);
                                s_prof[19] += (unsigned long long)(t_val - t_rdy);
                                s_prof[20] += 1;
                            }
                        }
                    }
                }
                if (ready) {
                    const int c = next_car;
                    // Segmented (rows): a block holding a row start contributes only its
                    // sum from its last row start (Phase I), and the sums before the last
                    // such block -- and the chunk carry -- do not reach later blocks.
                    int lh_below = -1, lh_all = -1;
                    if constexpr (SEG) {
#pragma unroll
                        for (int k = 0; k < RPL; ++k) {
                            const int bb = lane + 32 * k;
                            const int u0 = c * gm.chunk_tiles + bb * gm.bt;
                            const int u1 = u0 + gm.bt < gm.ntiles ? u0 + gm.bt : gm.ntiles;
                            const int64_t e0 = (int64_t)u0 * TILE;
                            // first row start at or after e0 (seg_rem[k] = e0 mod seg_len)
                            const int64_t first = e0 + (seg_rem[k] == 0 ? 0 : p.seg_len - seg_rem[k]);
                            if (bb < gm.g && u0 < u1 && first < (int64_t)u1 * TILE && first < gm.n) {
                                lh_all = bb;
                                if (bb < b) lh_below = bb;
                            }
                            seg_rem[k] += seg_dc;  // the same block of the next chunk
                            if (seg_rem[k] >= p.seg_len) seg_rem[k] -= p.seg_len;
                        }
                        lh_all = __reduce_max_sync(0xffffffffu, lh_all);
                        lh_below = __reduce_max_sync(0xffffffffu, lh_below);
                    }
                    Carry below = Carry(0), total = Carry(0);
#pragma unroll
                    for (int k = 0; k < RPL; ++k) {
                        const int bb = lane + 32 * k;
                        const Carry v = bb < gm.g ? carry_from_bits<Carry>(rb[k]) : Carry(0);
                        if (bb >= lh_all) total = total + v;
                        if (bb < b && bb >= lh_below) below = below + v;
                    }
                    below = warp_reduce_fixed(below);
                    total = warp_reduce_fixed(total);
                    if (lane == 0) {
                        s_carry[c % KC] = (lh_below < 0 ? chunk_carry : Carry(0)) + below;
                        ptx::mbar_arrive(&carry_ready[c % KC]);
                    }
                    __syncwarp();
                    chunk_carry = (lh_all < 0 ? chunk_carry : Carry(0)) + total;
                    ++next_car;
                    progressed = true;
                }
            }
            if (progressed) {
                backoff = 32;
                if (prof && lane == 0 && spin0) {
                    s_prof[4] += (unsigned long long)(clock64() - spin0);
                    spin0 = 0;
                }
            } else {
                if (prof && lane == 0 && !spin0) spin0 = clock64();
                __nanosleep(backoff);
                backoff = backoff < 256 ? backoff * 2 : 256;
            }
        }
    } else {
        // =========================== compute ===========================
        const int cw = warp - 3;
        const int e0_base = cw * GPW * 512 + 16 * lane;  // group g: + 512 g
        const LaneOffsets<SZ> off(e0_base);
        constexpr uint32_t GI = LaneOffsets<SZ>::kGrpIn, GO = LaneOffsets<SZ>::kGrpOut;
        const uint8_t* const gin_b = reinterpret_cast<const uint8_t*>(p.in);
        const bool csleep = (p.wait_mode & 2) != 0;
        // L2 maintenance after the re-read (A/B, p.l2 bits 4-5); an in-place scan
        // never discards (its output lands on the same lines)
        int l2_after = (p.l2 >> 4) & 3;
        const uint32_t sh_bits = (uint32_t)((p.shift * SZ) & 3) * 8;  // SHIFT: bits past the DW words
        if (l2_after == 1 && p.in == (const void*)p.out) l2_after = 2;
        const bool exclusive = p.exclusive != 0;
        const bool prof0 = prof && cw == 0 && lane == 0;
        Ring<NB_IN> rin;
        Ring<NSR> rout;  // !UNI only
        int s_count = 0;

        // Valid elements m and TMA-covered elements m_tma of a ragged tile t.
        auto ragged = [&](int t, int& m, int& m_in, int& m_out) {
            const int64_t g0 = (int64_t)t * TILE;
            const int64_t r = gm.n - g0, ri = p.n_tma_in - g0, ro = p.n_tma_out - g0;
            m = (int)(r < TILE ? r : TILE);
            m_in = (int)(ri < 0 ? 0 : (ri > m ? m : ri));
            m_out = (int)(ro < 0 ? 0 : (ro > m ? m : ro));
        };

        SegCursor<TILE> seg_r, seg_s;  // SEG: row starts of the Phase-I / Phase-II jobs
        int64_t seg_dc = 0;
        if constexpr (SEG) {
            seg_r.init(b, gm.bt, p.seg_len);
            seg_s.init(b, gm.bt, p.seg_len);
            seg_dc = ((int64_t)gm.chunk_tiles * TILE) % p.seg_len;
        }
        for (int q = 0; q < njobs; ++q) {
            int c, t0, t1;
            bool is_scan;
            mc_job(q, gm.chunks, p.ahead, c, is_scan);
            block_tiles(c, t0, t1);
            if (!is_scan) {
                // ---------------- Phase I: block reduction r[c][b] ----------------
                Carry jsum = Carry(0);
                if constexpr (SEG) seg_r.job(t0, p.seg_len, seg_dc, gm.n);
                for (int t = t0; t < t1; ++t, rin.next()) {
                    mbar_wait_prof(&in_full[rin.s], rin.ph, prof0, &s_prof[1], csleep);
#ifdef SCAN_MC_PROF
                    if (prof0 && s_prof[22] == 0) s_prof[22] = ptx::globaltimer();
#endif
                    const long long tr0 = prof ? clock64() : 0;
                    const uint8_t* slot = in_ring + rin.s * Cfg::kRingSlot;
                    if (SEG && t == seg_r.tile) {
                        // a row starts in this tile: drop the sums before it (cold path)
                        const int ro = seg_r.off;
                        seg_r.advance(p.seg_len, gm.n);
                        int m = TILE, m_in = TILE, m_out = TILE;
                        if (t >= gm.full_tiles) ragged(t, m, m_in, m_out);
                        jsum = mc_split_sum<DT, GPW>(slot, gin_b + (int64_t)t * TILE * SZ, e0_base, m, m_in, ro);
                    } else if (t < gm.full_tiles) {
#pragma unroll
                        for (int g = 0; g < GPW; ++g) {
                            Grp<SZ> gr;
                            if (SHIFT && !(p.debug & 8))
                                grp_load_shift<SZ, DW>(slot, e0_base + 512 * g, sh_bits, gr,
                                                       extra_rows + rin.s * 128, rin.s, TILE);
                            else
                                grp_load_off(slot + g * GI, off.in, gr);
                            jsum = jsum + Carry(grp_sum(gr, (const In*)nullptr));
                        }
                    } else {
                        int m, m_in, m_out;
                        ragged(t, m, m_in, m_out);
#pragma unroll
                        for (int g = 0; g < GPW; ++g) {
                            Grp<SZ> gr;
                            grp_load_tail(slot, gin_b + (int64_t)t * TILE * SZ, e0_base + 512 * g, m, m_in, gr,
                                          SHIFT ? p.shift : 0, extra_rows + rin.s * 128, rin.s, TILE);
                            jsum = jsum + Carry(grp_sum(gr, (const In*)nullptr));
                        }
                    }
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&in_empty[rin.s]);
                    if (prof0) {
                        s_prof[8] += 1;
                        s_prof[10] += (unsigned long long)(clock64() - tr0);
                    }
                }
                jsum = warp_reduce_fixed(jsum);
                if (lane == 0) {
                    s_job_sum[c % RS][cw] = jsum;
                    ptx::mbar_arrive(&rsum_ready[c % RS]);
                }
            } else {
                // ---------------- Phase II: scan with the block carry ----------------
                // The carry is first needed at the first tile's emit: the tile's loads, lane
                // prefixes and shuffle / warp-total scans run before the wait (lazy carry),
                // hiding the chunk barrier's latency behind them.  Segmented scans take it
                // up front (their split-tile path needs it earlier).
                Carry carry = Carry(0);
                bool have_carry = false;
                auto get_carry = [&]() {
                    if (!have_carry) {
                        mbar_wait_prof(&carry_ready[c % KC], (uint32_t)(c / KC) & 1u, prof0, &s_prof[0], csleep);
                        carry = s_carry[c % KC];
                        have_carry = true;
                    }
                };
                if (SEG || !(p.lazy_carry)) get_carry();
                if constexpr (SEG) seg_s.job(t0, p.seg_len, seg_dc, gm.n);
                for (int t = t0; t < t1; ++t, rin.next(), rout.next(), ++s_count) {
                    const int s = rin.s;
                    const int o = UNI ? s : rout.s;
                    mbar_wait_prof(&in_full[s], rin.ph, prof0, &s_prof[2], csleep);
                    const long long ts0 = prof ? clock64() : 0;
                    const bool full = t < gm.full_tiles;  // warp-uniform
                    int m = TILE, m_in = TILE, m_out = TILE;
                    if (!full) ragged(t, m, m_in, m_out);
                    const uint8_t* slot = in_ring + s * Cfg::kRingSlot;
                    int ro = 0;
                    if (SEG && t == seg_s.tile) {
                        ro = seg_s.off;
                        seg_s.advance(p.seg_len, gm.n);
                        if (ro == 0) carry = Carry(0);  // a row starts with this tile
                    }
                    if (SEG && ro > 0) {
                        // A row starts inside this tile (rare: once per row): cold path.
                        if (!UNI && rout.wrapped) mbar_wait_prof(&out_empty[o], rout.ph ^ 1u, prof0, &s_prof[3], csleep);
                        const Acc agg = mc_split_tile<DT, NC, GPW, TILE>(
                            slot, out_ring + o * Cfg::kOutSlot, gin_b + (int64_t)t * TILE * SZ, gout + (int64_t)t * TILE,
                            full, m, m_in, m_out, ro, carry, exclusive, e0_base, off, &s_wt[0][0], s_count, lane, cw);
                        s_count += 2;
                        __syncwarp();
                        if (!UNI && lane == 0) ptx::mbar_arrive(&in_empty[s]);  // both passes have read the slot
                        ptx::fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive(&store_ready[o]);
                        carry = Carry(agg);  // the new row's running sum
                        --s_count;           // the loop increment counts one pass
                    } else {
                    LaneScan<DT> ls[GPW];
                    Acc ex[GPW], gp[GPW];
                    Acc wsum = Acc(0);
#pragma unroll
                    for (int g = 0; g < GPW; ++g) {
                        if (full && SHIFT && !(p.debug & 8))  // debug bit 3: unshifted loads (timing only)
                            grp_load_shift<SZ, DW>(slot, e0_base + 512 * g, sh_bits, ls[g].g, extra_rows + s * 128,
                                                   s, TILE);
                        else if (full)
                            grp_load_off(slot + g * GI, off.in, ls[g].g);
                        else
                            grp_load_tail(slot, gin_b + (int64_t)t * TILE * SZ, e0_base + 512 * g, m, m_in,
                                          ls[g].g, SHIFT ? p.shift : 0, extra_rows + s * 128, s, TILE);
                        ex[g] = ls[g].prefix();  // lane total (held in ex until the shuffle scan)
                    }
                    if (!UNI) {  // unified ring: the storer frees the slot after the store
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive(&in_empty[s]);
                    }
                    if (l2_after && full) {
                        // the re-read was this tile's last use of its input: release its
                        // L2 lines (one 128-byte line per compute thread) so the lines of
                        // the chunks still waiting for their re-read stay resident
                        const uintptr_t tb = (uintptr_t)(gin_b + (int64_t)t * TILE * SZ);
                        const uintptr_t a1 = (tb + (uintptr_t)TILE * SZ) & ~(uintptr_t)127;
                        for (uintptr_t a = ((tb + 127) & ~(uintptr_t)127) + (uintptr_t)(cw * 32 + lane) * 128; a < a1;
                             a += (uintptr_t)NC * 32 * 128) {
                            if (l2_after == 1)
                                ptx::l2_discard_line(reinterpret_cast<const void*>(a));
                            else
                                ptx::l2_demote_line(reinterpret_cast<const void*>(a));
                        }
                    }
#pragma unroll
                    for (int g = 0; g < GPW; ++g) {
                        const Acc incl = warp_incl_scan(ex[g], lane);
                        const Acc e1 = __shfl_up_sync(0xffffffffu, incl, 1);
                        ex[g] = lane == 0 ? Acc(0) : e1;
                        gp[g] = wsum;
                        wsum = wsum + __shfl_sync(0xffffffffu, incl, 31);
                    }
                    if (lane == 0) s_wt[s_count & 1][cw] = wsum;
                    const long long ts1 = prof ? clock64() : 0;
                    named_bar_sync(1, NC * 32);
                    const long long ts2 = prof ? clock64() : 0;
                    const Acc x = lane < NC ? s_wt[s_count & 1][lane] : Acc(0);
                    const Acc xi = warp_incl_scan(x, lane);
                    const Acc xe = __shfl_up_sync(0xffffffffu, xi, 1);
                    const Acc wpref = __shfl_sync(0xffffffffu, lane == 0 ? Acc(0) : xe, cw);
                    const Acc agg = __shfl_sync(0xffffffffu, xi, NC - 1);
                    get_carry();
                    const long long te0 = prof ? clock64() : 0;
                    if (!UNI && rout.wrapped) mbar_wait_prof(&out_empty[o], rout.ph ^ 1u, prof0, &s_prof[3], csleep);
                    uint8_t* ost = out_ring + o * Cfg::kOutSlot;
                    const long long te1 = prof ? clock64() : 0;
#pragma unroll
                    for (int g = 0; g < GPW; ++g) {
                        Acc B;
                        if constexpr (Tr::kFloat)
                            B = (float)(carry + (double)((wpref + gp[g]) + ex[g]));
                        else
                            B = carry + wpref + gp[g] + ex[g];
                        Acc o16[16];
                        ls[g].emit(B, exclusive, o16);
                        if (full) {
                            store16_off(ost + g * GO, off.out, o16);
                        } else {
                            const int e0 = e0_base + 512 * g;
#pragma unroll
                            for (int k = 0; k < 16; ++k) {
                                if (e0 + k < m_out)
                                    *reinterpret_cast<Acc*>(ost + swz_elem<4>(e0 + k)) = o16[k];
                                else if (e0 + k < m)
                                    gout[(int64_t)t * TILE + e0 + k] = narrow(o16[k], (Out*)nullptr);
                            }
                        }
                    }
                    const long long te2 = prof ? clock64() : 0;
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&store_ready[o]);
                    carry = carry + Carry(agg);
                    if (prof0) {
                        const long long te3 = clock64();
                        s_prof[14] += (unsigned long long)(te0 - ts2);
                        s_prof[15] += (unsigned long long)(te1 - te0);
                        s_prof[16] += (unsigned long long)(te2 - te1);
                        s_prof[17] += (unsigned long long)(te3 - te2);
                        s_prof[9] += 1;
                        s_prof[11] += (unsigned long long)(ts1 - ts0);
                        s_prof[12] += (unsigned long long)(ts2 - ts1);
                        s_prof[13] += (unsigned long long)(te3 - ts2);
                    }
                    }  // row start inside the tile / not
                }
            }
        }
    }

#ifdef SCAN_MC_PROF
    if (prof && warp == 3 && lane == 0) s_prof[23] = ptx::globaltimer();  // compute warp 0 done
#endif
    __syncthreads();
    if (prof && tid == 0) s_prof[7] = (unsigned long long)(clock64() - t_start);
#ifdef SCAN_MC_PROF
    if (prof && tid == 0) s_prof[24] = ptx::globaltimer();
#endif
    __syncthreads();
    if (prof && tid < kMcProf && (blockIdx.x + 1) * kMcProf * 8 <= (int)(kWsBarOffset - kWsPartialsOffset))
        reinterpret_cast<unsigned long long*>(p.ws + kWsPartialsOffset)[blockIdx.x * kMcProf + tid] = s_prof[tid];
    if (tid == 0) {
        __threadfence();
        const uint32_t prev = ptx::claim_add(&hdr->done, 1u);
        if (prev == gridDim.x - 1) {
            // every CTA is past every barrier: reset the counters for the next call
            if (p.bar_mode == 1) {
                uint32_t e = hdr->epoch + 1;
                if (e == 0) {  // tag wrap (once per 2^32 calls): no stale word may match
                    const int64_t nw = (int64_t)gm.chunks * gm.g * (Tr::kFloat ? 2 : 1);
                    for (int64_t i = 0; i < nw; ++i) r_all[i] = 0ull;
                    e = 1;
                }
                hdr->epoch = e;
            } else {
                for (int c = 0; c < gm.chunks; ++c) bar[c] = 0;
            }
            hdr->done = 0;
            __threadfence();
        }
    }
}

}  // namespace scan

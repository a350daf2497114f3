// rowscan.cuh -- batched row scan (P437, App. B.1: "the prefix sum of a batch
// of input arrays of equal length") for rows of many tiles.
//
// The paper's batched ScanUL1 assigns "a separate array in the batch" to each
// AI core (P447) and ScanU's vector unit carries a running `partial` across
// the tiles of an array (Alg. 1, P145-155).  The B200 version does exactly
// that at CTA granularity: a persistent CTA claims whole rows with an atomic
// ticket and streams each row's tiles through shared memory in order,
// carrying the row prefix in a register (fp64 for float rows) -- no look-back
// and no grid barrier, so the only cost is the HBM stream.
//
// Rows move through TMA *tensor* copies over a 3-D view [rows][cols*sz/128][128 B]
// (row stride arbitrary, multiple of 16 B) with 128-byte swizzle; every lane
// owns 16 contiguous elements (one shuffle scan per 512 elements, see
// mcscan.cuh).  Outputs are written in place into the tile's slot after the
// per-tile named barrier and stored back with TMA tensor stores.
// Requirements (checked on the host, else the look-back kernel runs):
// cols*sizeof(In) and cols*4 multiples of 128 bytes, strides multiples of 16 B.
#pragma once
#include "mcscan.cuh"
#include "shard.cuh"  // device-initiated totals exchange (wait_carry_from_slots)

namespace scan {

struct RowParams {
    CUtensorMap tm_in;   // 3-D view of the input rows (int8: unused, 1-D bulk copies)
    CUtensorMap tm_out;  // 3-D view of the output rows
    const void* in;
    void* out;
    uint8_t* ws;         // header ticket / done counter
    int64_t rows;
    int64_t cols;
    int64_t in_stride;   // elements
    int tiles_per_row;
    int exclusive;
    // Sharded scan pass 2 (shard.cuh): row r starts from carry_in + row_pre[r]
    // (int64 for integer dtypes, double for floats); both NULL for plain rows.
    const void* row_pre;
    const void* carry_in;
    // Device-initiated exchange (sharded pass 2 without NCCL): if non-NULL the
    // carry is the sum of ranks 0..peer_rank-1's totals, read from this rank's
    // slot array (shard.cuh) by every compute warp before its first row -- the
    // producer's first loads overlap the wait; CTA 0 leaves it in carry_out.
    const uint64_t* peer_slots;
    int peer_G;
    int peer_rank;
    uint32_t peer_epoch;
    void* carry_out;
};

template <int DT, int NC, int GPW, int NB>
struct RowCfg {
    using Tr = Traits<DT>;
    using In = typename Tr::In;
    static constexpr int kThreads = (2 + NC) * 32;
    static constexpr int kTile = NC * GPW * 512;
    static constexpr size_t kInBytes = (size_t)kTile * sizeof(In);
    static constexpr size_t kSlot = (size_t)kTile * 4;  // outputs in place
    static constexpr int kRowElemsIn = 128 / (int)sizeof(In);
    static constexpr int box_rows(size_t r)
    {
        for (int k = 1; k <= 64; ++k)
            if (r % k == 0 && r / k <= 256 && (r / k) % 8 == 0) return (int)(r / k);
        return 0;
    }
    static constexpr int kBoxRowsIn = box_rows(kInBytes / 128);
    static constexpr int kBoxRowsOut = box_rows(kSlot / 128);
    static constexpr int kBoxesIn = (int)(kInBytes / 128 / (kBoxRowsIn ? kBoxRowsIn : 1));
    static constexpr int kBoxesOut = (int)(kSlot / 128 / kBoxRowsOut);
    static_assert(kBoxRowsOut > 0 && (sizeof(In) == 1 || kBoxRowsIn > 0), "whole swizzle phases per box");
    static constexpr size_t kSmem = NB * kSlot + 1024;
};

__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* tm, int x, int y, int z,
                                            uint64_t* bar, uint64_t policy)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(ptx::smem_u32(smem_dst)),
        "l"(tm), "r"(x), "r"(y), "r"(z), "r"(ptx::smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* tm, int x, int y, int z, const void* smem_src,
                                             uint64_t policy)
{
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2, %3}], [%4], %5;" ::"l"(
                     tm),
                 "r"(x), "r"(y), "r"(z), "r"(ptx::smem_u32(smem_src)), "l"(policy)
                 : "memory");
}

template <int DT, int NC, int GPW, int NB>
__global__ void __launch_bounds__((2 + NC) * 32, 1) k_rowscan16(const __grid_constant__ RowParams p)
{
    using Cfg = RowCfg<DT, NC, GPW, NB>;
    using Tr = Traits<DT>;
    using In = typename Tr::In;
    using Acc = typename Tr::Acc;
    using Carry = typename Tr::Carry;
    constexpr int TILE = Cfg::kTile;

    extern __shared__ uint8_t smem_raw[];
    // 1024-B aligned through an integer round trip (generic slot accesses); the
    // provenance-keeping form (LDS / STS) measured 100.5 -> 99.9 % on C4
    uint8_t* const ring = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);

    __shared__ __align__(8) uint64_t in_full[NB];
    __shared__ __align__(8) uint64_t in_empty[NB];
    __shared__ __align__(8) uint64_t store_ready[NB];
    __shared__ int64_t s_row[NB];   // row of the tile in each slot (-1: end of stream)
    __shared__ int s_k[NB];         // tile index within the row
    __shared__ Acc s_wt[2][NC];

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    WsHeader* hdr = reinterpret_cast<WsHeader*>(p.ws);
    const int tpr = p.tiles_per_row;

    if (tid == 0) {
        for (int s = 0; s < NB; ++s) {
            ptx::mbar_init(&in_full[s], 1);
            ptx::mbar_init(&in_empty[s], 1);
            ptx::mbar_init(&store_ready[s], NC);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();

    if (warp == 0) {
        // ============ producer: claim rows, stream their tiles ============
        if (lane == 0) {
            const uint64_t pol = ptx::policy_evict_first();
            int64_t q = 0;
            while (true) {
                const int64_t row = (int64_t)ptx::claim_add(&hdr->ticket, 1u);
                const bool end = row >= p.rows;
                for (int k = 0; k < (end ? 1 : tpr); ++k, ++q) {
                    const int s = (int)(q % NB);
                    const uint32_t use = (uint32_t)(q / NB);
                    if (use > 0) ptx::mbar_wait(&in_empty[s], (use - 1) & 1u);
                    s_row[s] = end ? -1 : row;
                    s_k[s] = k;
                    if (end) {
                        ptx::mbar_arrive(&in_full[s]);
                        break;
                    }
                    uint8_t* dst = ring + s * Cfg::kSlot;
                    const int64_t c0 = (int64_t)k * TILE;
                    if constexpr (sizeof(In) == 1) {
                        const int64_t m = p.cols - c0 < TILE ? p.cols - c0 : TILE;
                        ptx::mbar_arrive_expect_tx(&in_full[s], (uint32_t)m);
                        ptx::tma_load_1d(dst, reinterpret_cast<const In*>(p.in) + row * p.in_stride + c0,
                                         (uint32_t)m, &in_full[s], pol);
                    } else {
                        ptx::mbar_arrive_expect_tx(&in_full[s], (uint32_t)Cfg::kInBytes);
                        const int y0 = (int)(c0 / Cfg::kRowElemsIn);
#pragma unroll
                        for (int bx = 0; bx < Cfg::kBoxesIn; ++bx)
                            tma_load_3d(dst + bx * Cfg::kBoxRowsIn * 128, &p.tm_in, 0, y0 + Cfg::kBoxRowsIn * bx,
                                        (int)row, &in_full[s], pol);
                    }
                }
                if (end) break;
            }
        }
    } else if (warp == 1) {
        // ============ storer ============
        if (lane == 0) {
            const uint64_t pol = ptx::policy_evict_first();
            int pend = -1;
            for (int64_t q = 0;; ++q) {
                const int s = (int)(q % NB);
                const uint32_t par = (uint32_t)(q / NB) & 1u;
                if (pend >= 0 && !ptx::mbar_try_wait(&store_ready[s], par)) {
                    ptx::bulk_wait_read<0>();
                    ptx::mbar_arrive(&in_empty[pend]);
                    pend = -1;
                }
                ptx::mbar_wait(&store_ready[s], par);
                const int64_t row = s_row[s];
                if (row < 0) break;
                const int y0 = s_k[s] * (TILE / 32);
#pragma unroll
                for (int bx = 0; bx < Cfg::kBoxesOut; ++bx)
                    tma_store_3d(&p.tm_out, 0, y0 + Cfg::kBoxRowsOut * bx, (int)row,
                                 ring + s * Cfg::kSlot + bx * Cfg::kBoxRowsOut * 128, pol);
                ptx::bulk_commit();
                if (pend >= 0) {
                    ptx::bulk_wait_read<1>();
                    ptx::mbar_arrive(&in_empty[pend]);
                }
                pend = s;
            }
            ptx::bulk_wait<0>();
        }
    } else {
        // ============ compute: one tile at a time, running row carry ============
        const int cw = warp - 2;
        Carry carry = Carry(0);
        using Sum64 = typename std::conditional<Tr::kFloat, double, long long>::type;
        Sum64 c_in = Sum64(0);  // carry of the lower shards (sharded pass 2)
        if (p.peer_slots != nullptr) {
            c_in = shard::wait_carry_from_slots<Sum64>(p.peer_slots, p.peer_G, p.peer_rank, p.peer_epoch, lane);
            if (blockIdx.x == 0 && cw == 0 && lane == 0 && p.carry_out) *reinterpret_cast<Sum64*>(p.carry_out) = c_in;
        } else if (p.row_pre != nullptr && p.carry_in != nullptr) {
            c_in = *reinterpret_cast<const Sum64*>(p.carry_in);
        }
        for (int64_t q = 0;; ++q) {
            const int s = (int)(q % NB);
            ptx::mbar_wait(&in_full[s], (uint32_t)(q / NB) & 1u);
            const int64_t row = s_row[s];
            if (row < 0) {
                if (lane == 0) ptx::mbar_arrive(&store_ready[s]);  // let the storer see the end
                break;
            }
            const int k = s_k[s];
            if (k == 0) {  // a new row starts from zero (P437) or from its block prefix (sharded pass 2)
                carry = Carry(0);
                if (p.row_pre != nullptr) {
                    if constexpr (Tr::kFloat)
                        carry = c_in + reinterpret_cast<const double*>(p.row_pre)[row];
                    else
                        carry = (Carry)(uint32_t)(uint64_t)(c_in + reinterpret_cast<const long long*>(p.row_pre)[row]);
                }
            }
            const int m = (int)(p.cols - (int64_t)k * TILE < TILE ? p.cols - (int64_t)k * TILE : TILE);
            uint8_t* const slot = ring + s * Cfg::kSlot;

            LaneScan<DT> ls[GPW];
            Acc ex[GPW], gp[GPW];
            Acc wsum = Acc(0);
            const bool full = m == TILE;  // warp-uniform
#pragma unroll
            for (int g = 0; g < GPW; ++g) {
                const int e0 = (cw * GPW + g) * 512 + 16 * lane;
                if (full || e0 + 16 <= m)
                    grp_load(slot, e0, ls[g].g);
                else
                    grp_load_tail(slot, slot, e0, m, m, ls[g].g);
                ex[g] = ls[g].prefix();  // lane total until the shuffle scan
            }
#pragma unroll
            for (int g = 0; g < GPW; ++g) {
                const Acc incl = warp_incl_scan(ex[g], lane);
                const Acc e1 = __shfl_up_sync(0xffffffffu, incl, 1);
                ex[g] = lane == 0 ? Acc(0) : e1;
                gp[g] = wsum;
                wsum = wsum + __shfl_sync(0xffffffffu, incl, 31);
            }
            if (lane == 0) s_wt[q & 1][cw] = wsum;
            named_bar_sync(1, NC * 32);  // totals visible; every warp has read its input
            const Acc x = lane < NC ? s_wt[q & 1][lane] : Acc(0);
            const Acc xi = warp_incl_scan(x, lane);
            const Acc xe = __shfl_up_sync(0xffffffffu, xi, 1);
            const Acc wpref = __shfl_sync(0xffffffffu, lane == 0 ? Acc(0) : xe, cw);
            const Acc agg = __shfl_sync(0xffffffffu, xi, NC - 1);
            const bool exclusive = p.exclusive != 0;
#pragma unroll
            for (int g = 0; g < GPW; ++g) {
                const int e0 = (cw * GPW + g) * 512 + 16 * lane;
                Acc B;
                if constexpr (Tr::kFloat)
                    B = (float)(carry + (double)((wpref + gp[g]) + ex[g]));
                else
                    B = carry + wpref + gp[g] + ex[g];
                Acc o16[16];
                ls[g].emit(B, exclusive, o16);
                store16(slot, e0, o16);  // columns past `cols` fall outside the tensor: not stored
            }
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&store_ready[s]);
            carry = carry + Carry(agg);
        }
    }

    __syncthreads();
    if (tid == 0) {
        __threadfence();
        const uint32_t prev = ptx::claim_add(&hdr->done, 1u);
        if (prev == gridDim.x - 1) {
            hdr->ticket = 0;
            hdr->done = 0;
            __threadfence();
        }
    }
}

}  // namespace scan

// scan_ws.cuh -- warp-specialized single-pass scan for multi-tile segments.
//
// Same method as k_scan_tiles (decoupled look-back, P78-81; tile-local scans
// as the analog of Alg. 1's A@U_s + `partial`, P145-155), re-timed so the
// look-back round trips through L2 never stall the streaming warps.  One CTA
// per SM; roles synchronised with mbarriers over a ring of tile slots:
//
//   warp 0     producer   claims tiles (global ticket) and streams them into
//                         the input ring with TMA 1-D bulk copies;
//   warp 1     storer     streams finished tiles back with TMA bulk stores and
//                         frees their slots once the store has read them;
//   warps 2..  look-back  NL warps, tile j handled by warp j % NL: walk the
//                         predecessor descriptors down to the nearest inclusive
//                         prefix or to this CTA's previous tile (whose
//                         inclusive prefix another look-back warp hands over
//                         through shared memory), publish the inclusive prefix;
//   the rest   compute    NC warps: scan their rows of tile i in place (local
//                         inclusive sums in the output slot); the last warp to
//                         finish publishes the tile aggregate at once; then
//                         they finish tile i-1 (add its prefix: epilogue).
//
// A tile's aggregate never waits for the look-back of an older tile of the
// same CTA, and NL look-backs are in flight per CTA, so the L2 round-trip
// latency of a look-back is overlapped instead of serialised (DESIGN.md
// "Kernels"; measured stall counters in profiles/).
#pragma once
#include "scan_kernels.cuh"

namespace scan {

constexpr int64_t kEndTile = INT64_MAX;
constexpr int kNumProf = 12;  // per-CTA stall counters (debug bit 2), in the partials area

// Timed mbarrier wait: adds the cycles spent waiting to *acc when profiling.
__device__ __forceinline__ void mbar_wait_prof(uint64_t* bar, uint32_t parity, bool prof,
                                               unsigned long long* acc, bool sleep = false)
{
    if (!prof) {
        if (sleep)
            ptx::mbar_wait_sleep(bar, parity);
        else
            ptx::mbar_wait(bar, parity);
        return;
    }
    if (ptx::mbar_try_wait(bar, parity)) return;
    long long t0 = clock64();
    ptx::mbar_wait(bar, parity);
    atomicAdd(acc, (unsigned long long)(clock64() - t0));
}

template <int DT, int NC, int NL, int ROWS, int NB_IN, int NB_OUT>
struct WsCfg {
    using Tr = Traits<DT>;
    using In = typename Tr::In;
    using Out = typename Tr::Out;
    static constexpr bool kInPlace = sizeof(In) == sizeof(Out);
    static constexpr int kThreads = (2 + NL + NC) * 32;
    static constexpr int kTile = NC * ROWS * 128;
    static constexpr size_t kInSlot = (size_t)kTile * sizeof(In);
    static constexpr size_t kOutSlot = (size_t)kTile * sizeof(Out);
    static constexpr int kChain = 2 * NB_OUT;  // hand-off ring of inclusive prefixes
    static_assert(!kInPlace || NB_IN == NB_OUT, "in-place rings share slots");
    static_assert(NB_OUT % NL == 0, "a slot is always revisited by the same look-back warp");
    static_assert(NC <= 32, "warp totals are scanned by one warp");
    static constexpr size_t kSmem = kInPlace ? NB_OUT * kOutSlot : NB_IN * kInSlot + NB_OUT * kOutSlot;
};

template <int DT, int NC, int NL, int ROWS, int NB_IN, int NB_OUT>
__global__ void __launch_bounds__((2 + NL + NC) * 32, 1) k_scan_ws(const ScanParams p)
{
    using Cfg = WsCfg<DT, NC, NL, ROWS, NB_IN, NB_OUT>;
    using Tr = Traits<DT>;
    using In = typename Tr::In;
    using Out = typename Tr::Out;
    using Acc = typename Tr::Acc;
    using Carry = typename Tr::Carry;
    using Lane4 = typename std::conditional<Tr::kFloat, float, int32_t>::type;
    constexpr int TILE = Cfg::kTile;
    constexpr bool INPLACE = Cfg::kInPlace;
    constexpr int KCH = Cfg::kChain;

    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* const in_ring = smem;
    uint8_t* const out_ring = INPLACE ? smem : smem + NB_IN * Cfg::kInSlot;

    __shared__ __align__(8) uint64_t in_full[NB_IN];
    __shared__ __align__(8) uint64_t in_empty[NB_IN];
    __shared__ __align__(8) uint64_t local_done[NB_OUT];
    __shared__ __align__(8) uint64_t prefix_ready[NB_OUT];
    __shared__ __align__(8) uint64_t store_ready[NB_OUT];
    __shared__ __align__(8) uint64_t out_empty[NB_OUT];
    __shared__ int64_t s_tile_in[NB_IN];
    __shared__ int s_tma_in[NB_IN];
    __shared__ int64_t s_tile_out[NB_OUT];
    __shared__ Acc s_warp_tot[NB_OUT][NC];
    __shared__ Acc s_warp_pref[NB_OUT][NC];
    __shared__ Carry s_prefix[NB_OUT];
    __shared__ Acc s_agg[NB_OUT];
    __shared__ int s_cnt[NB_OUT];
    __shared__ int64_t s_tix[KCH];             // tile index of this CTA's j-th tile
    __shared__ volatile int64_t s_chain_seq[KCH];
    __shared__ Carry s_chain_incl[KCH];        // inclusive prefix of this CTA's j-th tile
    __shared__ volatile int64_t s_end;         // index j of the end-of-stream marker
    __shared__ unsigned long long s_prof[kNumProf];

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const bool prof = (p.debug & 4) != 0;

    WsHeader* hdr = reinterpret_cast<WsHeader*>(p.ws);
    uint64_t* desc = reinterpret_cast<uint64_t*>(p.ws + kWsDescOffset);
    const In* gin = reinterpret_cast<const In*>(p.in);
    Out* gout = reinterpret_cast<Out*>(p.out);

    if (tid < kNumProf) s_prof[tid] = 0;
    if (tid < KCH) s_chain_seq[tid] = -1;
    if (tid == 0) {
        s_end = kEndTile;
        for (int s = 0; s < NB_IN; ++s) {
            ptx::mbar_init(&in_full[s], 1);
            ptx::mbar_init(&in_empty[s], NC);
        }
        for (int o = 0; o < NB_OUT; ++o) {
            ptx::mbar_init(&local_done[o], 1);  // arrived by the last compute warp
            s_cnt[o] = 0;
            ptx::mbar_init(&prefix_ready[o], 1);
            ptx::mbar_init(&store_ready[o], NC);
            ptx::mbar_init(&out_empty[o], 1);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    const uint32_t tag = hdr->epoch;

    // Geometry of tile t: segment, tile-in-segment, valid elements.
    auto geom = [&](int64_t t, int64_t& seg, int64_t& k, int& m) {
        seg = t / p.tiles_per_seg;
        k = t - seg * p.tiles_per_seg;
        const int64_t mm = p.seg_len - k * TILE;
        m = (int)(mm > TILE ? TILE : mm);
    };
    auto carry_of = [&](int64_t seg) -> Carry {
        if (seg == 0 && p.carry_in != nullptr) {
            if constexpr (Tr::kFloat)
                return *reinterpret_cast<const double*>(p.carry_in);
            else
                return (uint32_t)(uint64_t)(*reinterpret_cast<const int64_t*>(p.carry_in));
        }
        return Carry(0);
    };

    if (warp == 0) {
        // =========================== producer ===========================
        if (lane == 0) {
            const uint64_t pol = ptx::policy_evict_first();
            for (int64_t q = 0;; ++q) {
                const int s = (int)(q % NB_IN);
                const uint32_t use = (uint32_t)(q / NB_IN);
                if (use > 0) {
                    // INPLACE: free once the storer has read it out; otherwise
                    // once the compute warps have read the input.
                    if (INPLACE)
                        mbar_wait_prof(&out_empty[s], (use - 1) & 1u, prof, &s_prof[6]);
                    else
                        mbar_wait_prof(&in_empty[s], (use - 1) & 1u, prof, &s_prof[6]);
                }
                int64_t t = (int64_t)ptx::claim_add(&hdr->ticket, 1u);
                if (t >= p.num_tiles) t = kEndTile;
                s_tile_in[s] = t;
                int tma = 0;
                if (t != kEndTile) {
                    int64_t seg, k;
                    int m;
                    geom(t, seg, k, m);
                    const uint32_t bytes = (uint32_t)(m * (int)sizeof(In));
                    if (p.tma_in && (bytes & 15u) == 0) {
                        tma = 1;
                        s_tma_in[s] = 1;
                        ptx::mbar_arrive_expect_tx(&in_full[s], bytes);
                        ptx::tma_load_1d(in_ring + s * Cfg::kInSlot, gin + seg * p.in_stride + k * TILE,
                                         bytes, &in_full[s], pol);
                    }
                }
                if (!tma) {
                    s_tma_in[s] = 0;
                    ptx::mbar_arrive(&in_full[s]);
                }
                if (t == kEndTile) break;
            }
        }
    } else if (warp == 1) {
        // =========================== storer ===========================
        if (lane == 0) {
            const uint64_t pol = ptx::policy_evict_first();
            for (int64_t j = 0;; ++j) {
                const int o = (int)(j % NB_OUT);
                mbar_wait_prof(&store_ready[o], (uint32_t)(j / NB_OUT) & 1u, prof, &s_prof[8]);
                const int64_t t = s_tile_out[o];
                if (t == kEndTile) break;
                int64_t seg, k;
                int m;
                geom(t, seg, k, m);
                const uint32_t bytes = (uint32_t)(m * (int)sizeof(Out));
                if (p.tma_out && (bytes & 15u) == 0) {
                    ptx::tma_store_1d(gout + seg * p.out_stride + k * TILE, out_ring + o * Cfg::kOutSlot,
                                      bytes, pol);
                    ptx::bulk_commit();
                    const long long w0 = prof ? clock64() : 0;
                    ptx::bulk_wait_read<0>();
                    if (prof) atomicAdd(&s_prof[9], (unsigned long long)(clock64() - w0));
                }
                ptx::mbar_arrive(&out_empty[o]);
            }
            ptx::bulk_wait<0>();  // every store has landed before the CTA retires
        }
    } else if (warp < 2 + NL) {
        // =========================== look-back ===========================
        const int lw = warp - 2;
        for (int64_t j = lw;; j += NL) {
            const int o = (int)(j % NB_OUT);
            const uint32_t par = (uint32_t)(j / NB_OUT) & 1u;
            // lane 0 waits and decides for the warp (warp-uniform control flow
            // for the collectives below); __syncwarp orders its acquire before
            // the other lanes' shared-memory reads
            int ended = 0;
            if (lane == 0 && !ptx::mbar_try_wait(&local_done[o], par)) {
                const long long w0 = prof ? clock64() : 0;
                while (!ptx::mbar_try_wait(&local_done[o], par)) {
                    if (s_end <= j) {
                        ended = 1;
                        break;
                    }
                }
                if (prof) atomicAdd(&s_prof[3], (unsigned long long)(clock64() - w0));
            }
            ended = __shfl_sync(0xffffffffu, ended, 0);
            __syncwarp();
            if (ended) break;
            const int64_t t = s_tile_out[o];
            if (t == kEndTile) break;
            const Acc agg = s_agg[o];
            int64_t seg, k;
            int m;
            geom(t, seg, k, m);
            const Carry carry_seg = carry_of(seg);
            Carry prefix;
            if (k == 0) {
                prefix = carry_seg;  // inclusive prefix already published by the compute side
            } else {
                const long long lb0 = prof ? clock64() : 0;
                const int64_t seg_first = t - k;
                const int64_t t_prev = j > 0 ? s_tix[(j - 1) % KCH] : -1;
                const bool own = t_prev >= seg_first;
                const int64_t lo = own ? t_prev : seg_first - 1;
                if (p.debug & 1) {
                    prefix = Carry(0);
                } else {
                    bool hit_lo = false;
                    prefix = lookback_range<Carry, 8>(desc, t, lo, tag, lane, (p.debug & 2) ? 0u : 32u,
                                                      &hit_lo, prof ? &s_prof[4] : nullptr);
                    if (hit_lo) {
                        if (own) {
                            // inclusive prefix of this CTA's previous tile, from the
                            // look-back warp that resolved it
                            const int c = (int)((j - 1) % KCH);
                            while (s_chain_seq[c] != j - 1) {
                            }
                            __threadfence_block();
                            prefix = prefix + s_chain_incl[c];
                        } else {
                            prefix = prefix + carry_seg;
                        }
                    }
                }
                if (lane == 0 && k + 1 < p.tiles_per_seg)
                    Desc<Carry>::publish(desc + t * Desc<Carry>::kSlots, true, tag, prefix + Carry(agg));
                if (prof && lane == 0) {
                    atomicAdd(&s_prof[2], (unsigned long long)(clock64() - lb0));
                    atomicAdd(&s_prof[10], (unsigned long long)(t - lo));
                }
            }
            if (lane == 0) {
                const int c = (int)(j % KCH);
                s_chain_incl[c] = prefix + Carry(agg);
                s_prefix[o] = prefix;
                __threadfence_block();
                s_chain_seq[c] = j;
                ptx::mbar_arrive(&prefix_ready[o]);
            }
            __syncwarp();
        }
    } else {
        // =========================== compute ===========================
        const int cw = warp - 2 - NL;
        const int wbase = cw * ROWS * 128 + 4 * lane;  // element offset of this lane's row 0

        // Epilogue of tile j (slot o): out = prefix + warp prefix + local.
        auto epilogue = [&](int64_t j) {
            const int o = (int)(j % NB_OUT);
            mbar_wait_prof(&prefix_ready[o], (uint32_t)(j / NB_OUT) & 1u, prof && cw == 0 && lane == 0,
                           &s_prof[1]);
            const int64_t t = s_tile_out[o];
            int64_t seg, k;
            int m;
            geom(t, seg, k, m);
            const bool tma_out = p.tma_out && ((m * (int)sizeof(Out)) & 15) == 0;
            const Carry P = s_prefix[o];
            const Acc wpref = s_warp_pref[o][cw];
            Acc* slot = reinterpret_cast<Acc*>(out_ring + o * Cfg::kOutSlot);
            Out* dst = gout + seg * p.out_stride + k * TILE;
            float P_hi = 0.f, base_f = 0.f;
            if constexpr (Tr::kFloat) {
                P_hi = (float)P;
                const float P_lo = isfinite(P_hi) ? (float)(P - (double)P_hi) : 0.f;  // inf carry: no inf - inf (R8)
                base_f = P_lo + wpref;
            }
#pragma unroll 4
            for (int r = 0; r < ROWS; ++r) {
                const int e = wbase + r * 128;
                Acc l[4];
                unpack4(reinterpret_cast<const Lane4*>(slot + e), l);
                Acc o4[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if constexpr (Tr::kFloat)
                        o4[q] = P_hi + (base_f + l[q]);
                    else
                        o4[q] = P + wpref + l[q];
                }
                if (tma_out) {
                    store4(reinterpret_cast<Out*>(slot) + e, o4);
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (e + q < m) dst[e + q] = narrow(o4[q], (Out*)nullptr);
                }
            }
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&store_ready[o]);
        };

        int64_t i = 0;
        for (;; ++i) {
            const int s = (int)(i % NB_IN);
            const int o = (int)(i % NB_OUT);
            mbar_wait_prof(&in_full[s], (uint32_t)(i / NB_IN) & 1u, prof && cw == 0 && lane == 0,
                           &s_prof[0]);
            const int64_t t = s_tile_in[s];
            // The output slot must have been stored out (INPLACE: guaranteed by
            // the producer, which refilled the slot only after out_empty).
            if (!INPLACE && i >= NB_OUT) ptx::mbar_wait(&out_empty[o], (uint32_t)(i / NB_OUT - 1) & 1u);
            if (t == kEndTile) break;
            if (prof && cw == 0 && lane == 0) s_prof[7] += 1;
            int64_t seg, k;
            int m;
            geom(t, seg, k, m);
            const bool full = m == TILE;
            const In* in_slot = reinterpret_cast<const In*>(in_ring + s * Cfg::kInSlot);
            Acc* out_slot = reinterpret_cast<Acc*>(out_ring + o * Cfg::kOutSlot);
            const In* src = gin + seg * p.in_stride + k * TILE;
            const bool tma_in = s_tma_in[s] != 0;

            // ---- local scan: rows of 128 elements, chained within the warp
            Acc wsum = Acc(0);
#pragma unroll 4
            for (int r = 0; r < ROWS; ++r) {
                const int e = wbase + r * 128;
                Acc v[4];
                if (tma_in) {
                    unpack4(in_slot + e, v);
                    if (!full) {
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            if (e + q >= m) v[q] = Acc(0);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) v[q] = e + q < m ? widen(src[e + q]) : Acc(0);
                }
                v[1] = v[0] + v[1];
                v[2] = v[1] + v[2];
                v[3] = v[2] + v[3];
                const Acc incl = warp_incl_scan(v[3], lane);
                Acc ex = __shfl_up_sync(0xffffffffu, incl, 1);
                ex = lane == 0 ? Acc(0) : ex;
                const Acc rt = __shfl_sync(0xffffffffu, incl, 31);
                const Acc base = wsum + ex;
                Acc l[4];
                if (p.exclusive) {
                    l[0] = base;
                    l[1] = base + v[0];
                    l[2] = base + v[1];
                    l[3] = base + v[2];
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) l[q] = base + v[q];
                }
                store4(reinterpret_cast<Lane4*>(out_slot + e), l);
                wsum = wsum + rt;
            }

            // ---- the last warp to finish publishes the tile aggregate at once
            int last = 0;
            if (lane == 0) {
                s_warp_tot[o][cw] = wsum;
                __threadfence_block();
                last = atomicAdd(&s_cnt[o], 1) == NC - 1;
                if (!INPLACE) ptx::mbar_arrive(&in_empty[s]);
            }
            last = __shfl_sync(0xffffffffu, last, 0);
            if (last) {
                __threadfence_block();
                const Acc x = lane < NC ? ((volatile Acc*)s_warp_tot[o])[lane] : Acc(0);
                const Acc xi = warp_incl_scan(x, lane);
                const Acc xe = __shfl_up_sync(0xffffffffu, xi, 1);
                if (lane < NC) s_warp_pref[o][lane] = lane == 0 ? Acc(0) : xe;
                const Acc agg = __shfl_sync(0xffffffffu, xi, NC - 1);
                if (lane == 0) {
                    uint64_t* d = desc + t * Desc<Carry>::kSlots;
                    if (k == 0)
                        Desc<Carry>::publish(d, true, tag, carry_of(seg) + Carry(agg));
                    else
                        Desc<Carry>::publish(d, false, tag, Carry(agg));
                    s_agg[o] = agg;
                    s_tile_out[o] = t;
                    s_tix[i % KCH] = t;
                    s_cnt[o] = 0;
                }
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&local_done[o]);
            }
            // ---- epilogue of the previous tile (its look-back overlapped our scan)
            if (i > 0) epilogue(i - 1);
        }
        // drain: finish the last tile, then mark the end of the stream for the
        // look-back warps and the storer (slot o is free: checked above).
        if (i > 0) epilogue(i - 1);
        const int o = (int)(i % NB_OUT);
        int last = 0;
        if (lane == 0) last = atomicAdd(&s_cnt[o], 1) == NC - 1;
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last && lane == 0) {
            s_tile_out[o] = kEndTile;
            s_end = i;
            __threadfence_block();
            ptx::mbar_arrive(&local_done[o]);
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&store_ready[o]);
    }

    __syncthreads();
    if (prof && tid < kNumProf && (blockIdx.x + 1) * kNumProf <= kMaxTotalCtas)
        reinterpret_cast<unsigned long long*>(p.ws + kWsPartialsOffset)[blockIdx.x * kNumProf + tid] = s_prof[tid];
    if (tid == 0) {
        __threadfence();
        const uint32_t prev = ptx::claim_add(&hdr->done, 1u);
        if (prev == gridDim.x - 1) {
            hdr->ticket = 0;
            hdr->done = 0;
            uint32_t e = hdr->epoch + 1;
            if (e == 0) {
                const uint64_t nslots = (uint64_t)hdr->capacity * 4;
                for (uint64_t q = 0; q < nslots; ++q) desc[q] = 0;
                e = 1;
            }
            hdr->epoch = e;
            __threadfence();
        }
    }
}

}  // namespace scan

// ptx.cuh -- thin inline-PTX wrappers for sm_100a used by the scan kernels:
// TMA 1-D bulk copies (cp.async.bulk) with mbarrier completion, bulk-group
// stores, proxy fences, and relaxed gpu-scope loads/stores for the look-back
// descriptors.  Nothing here is scan arithmetic.
#pragma once
#include <stdint.h>

namespace scan {
namespace ptx {

// Nanosecond device timer (profiling builds).
__device__ __forceinline__ unsigned long long globaltimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- fault injection (the T2 stress tier; libscan_fuzz.so only) ---------------
// With -DSCAN_FUZZ every hand-off between warps, CTAs and the async proxy
// (mbarrier arrivals, release arrivals on the grid barriers, look-back
// descriptor publishes, ticket claims, bulk-store commits) first sleeps a
// pseudo-random 0-4 us in about one call of four, so orderings that the normal
// schedule never produces get exercised.  The product build compiles it away.
#ifdef SCAN_FUZZ
__device__ uint32_t g_fuzz_mask = 0xffffffffu;  // sites enabled (SCAN_FUZZ_MASK, set by the launcher)

__device__ __forceinline__ void fuzz_delay(uint32_t site)
{
    if (((*(volatile uint32_t*)&g_fuzz_mask >> site) & 1u) == 0) return;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    uint32_t h = (uint32_t)(t ^ (t >> 23)) * 0x9E3779B1u;
    h ^= blockIdx.x * 0x85EBCA6Bu ^ threadIdx.x * 0xC2B2AE35u ^ site * 0x27D4EB2Fu;
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    if ((h & 3u) == 0) __nanosleep(h >> 20);
}
#define SCAN_FUZZ_POINT(site) ::scan::ptx::fuzz_delay(site)
#else
#define SCAN_FUZZ_POINT(site) ((void)0)
#endif

// A ticket / completion-counter claim (a fault-injection point in the fuzz build).
__device__ __forceinline__ unsigned int claim_add(unsigned int* p, unsigned int v)
{
    SCAN_FUZZ_POINT(8);
    return atomicAdd(p, v);
}

// ---- mbarrier ---------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes)
{
    SCAN_FUZZ_POINT(1);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity)
{
    uint32_t ok;
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar)
{
    SCAN_FUZZ_POINT(2);
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_cnt(uint64_t* bar, uint32_t count)
{
    SCAN_FUZZ_POINT(3);
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity);

// Blocking wait.  SCAN_WAIT_SLEEP (A/B build flag): every plain wait sleeps.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
#ifdef SCAN_WAIT_SLEEP
    mbar_wait_sleep(bar, parity);
#else
    while (!mbar_try_wait(bar, parity)) {
    }
#endif
}

// Blocking wait with a suspend-time hint: the warp sleeps in the barrier unit
// until the phase completes (up to ~10 ms per try) instead of re-issuing the
// test, so it takes no issue slots from the warps of its SM sub-partition (the
// C2 source view counted ~50 SYNCS tests per 1,024 elements); the wake-up can
// be later than a spinning test would notice the phase.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity)
{
    uint32_t ok;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity), "r"(0x989680u)
            : "memory");
    } while (!ok);
}

// Bulk prefetch of [p, p + bytes) into L2 (16-byte aligned, bytes a multiple of 16):
// one instruction, no registers or shared memory held while the lines arrive.
__device__ __forceinline__ void l2_prefetch_bulk(const void* p, uint32_t bytes)
{
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// ---- TMA 1-D bulk copies -------------------------------------------------------
__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ uint64_t policy_evict_last()
{
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ uint64_t policy_evict_normal()
{
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ uint64_t policy_evict_unchanged()
{
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// evict_last on `fraction` of the accessed lines, priority unchanged on the rest
// L2 line maintenance after a line's last use: drop it (clean input only: the
// line's contents become undefined) or demote it to normal eviction priority.
__device__ __forceinline__ void l2_discard_line(const void* p128)
{
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p128) : "memory");
}
__device__ __forceinline__ void l2_demote_line(const void* p128)
{
    asm volatile("applypriority.global.L2::evict_normal [%0], 128;" ::"l"(p128) : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_last_frac(float fraction)
{
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_unchanged.b64 %0, %1;" : "=l"(pol) : "f"(fraction));
    return pol;
}

// global -> shared, completion signalled on `bar` (complete_tx of `bytes`).
__device__ __forceinline__ void tma_load_1d(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                            uint64_t* bar, uint64_t policy)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(smem_dst)),
        "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// shared -> global, tracked by the issuing thread's bulk async-group.
__device__ __forceinline__ void tma_store_1d(void* gmem_dst, const void* smem_src, uint32_t bytes,
                                             uint64_t policy)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                     gmem_dst),
                 "r"(smem_u32(smem_src)), "r"(bytes), "l"(policy)
                 : "memory");
}

__device__ __forceinline__ void bulk_commit() {
    SCAN_FUZZ_POINT(5); asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

// Wait until at most N committed bulk groups still READ shared memory.
template <int N>
__device__ __forceinline__ void bulk_wait_read()
{
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

// Wait until at most N committed bulk groups are incomplete (writes done).
template <int N>
__device__ __forceinline__ void bulk_wait()
{
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// Make this thread's generic-proxy shared-memory writes visible to the async
// proxy (TMA store) -- needed before a bulk store reads what threads wrote.
__device__ __forceinline__ void fence_proxy_async_smem()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- relaxed gpu-scope accesses for look-back descriptors -----------------------
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v)
{
    SCAN_FUZZ_POINT(6);
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void st_relaxed_v2u64(uint64_t* p, uint64_t a, uint64_t b)
{
    SCAN_FUZZ_POINT(7);
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

__device__ __forceinline__ void ld_relaxed_v2u64(const uint64_t* p, uint64_t& a, uint64_t& b)
{
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p)
{
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint64_t ld_acquire_u64(const uint64_t* p)
{
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p)
{
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Release-ordered add without a return value (publish + arrive in one op).
__device__ __forceinline__ void red_release_add_u32(uint32_t* p, uint32_t v)
{
    SCAN_FUZZ_POINT(4);
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Named barrier over `count` threads (id 0 is __syncthreads).
__device__ __forceinline__ void named_bar_sync(int id, int count)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// ---- streaming global loads (non-TMA paths) ---------------------------------------
// 16-byte read-only load kept in L2 with the given policy (e.g. evict_last).
__device__ __forceinline__ uint4 ld_keep_v4(const void* p, uint64_t policy)
{
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(policy));
    return r;
}

__device__ __forceinline__ uint4 ld_stream_v4(const void* p)
{
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

}  // namespace ptx
}  // namespace scan

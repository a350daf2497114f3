// rowscan_tc.cuh -- the paper's cube-unit local scan (Eq. eqn:scan, P165-177;
// ScanU / ScanUL1, Alg. 1, P141-163) on B200's 5th-generation tensor cores,
// built for the A/B the north_star asks for ("tensor cores are used only if an
// ncu-backed A/B test shows a triangular-matmul local scan beating the
// CUDA-core path").  Batched fp16 -> fp32 rows of exactly 16,384 = 128 x 128
// elements (one tile per row, the batched-scan case of P437/P447).
//
// The paper multiplies a tile A (s x s, row-major chunk of the input) by the
// upper-triangular all-ones U_s: (A U_s)[m][j] = sum_{k<=j} A[m][k], the
// inclusive scan of every row of the tile; the row totals are then combined
// (L^-_s A 1_s, P167).  Here the product is issued TRANSPOSED so that the TMEM
// lane is the position j within a 128-element chunk and the TMEM column is the
// chunk index m:
//     D[j][m] = sum_k T[j][k] * X[m][k],   T[j][k] = (k <= j)   (= U_s^T),
// with T as the K-major A operand (constant, in shared memory) and the tile X
// (chunk m = elements 128m .. 128m+127) as the K-major B operand, streamed by
// TMA with 128-byte swizzle.  M = N = K = 128: 8 tcgen05.mma.kind::f16
// (K = 16 each) into 128 fp32 TMEM columns; two accumulator buffers.
// Epilogue (4 warps, thread = TMEM lane j): tcgen05.ld 128 columns, the chunk
// totals D[127][m] are exclusive-scanned over m by one warp (the L^-_s A 1_s
// term), out[128m + j] = base[m] + D[j][m] -- consecutive threads store
// consecutive addresses.
//
// Warp roles: 0 TMA producer, 1 MMA issuer (one lane) + TMEM owner, 2..5
// epilogue.  One CTA per SM, rows claimed statically (row = blockIdx.x + k*grid).
#pragma once
#include <cuda.h>
#include <stdint.h>

#include "ptx.cuh"

namespace scan {
namespace tc {

constexpr int kCols = 16384;       // elements per row = one 128 x 128 tile
constexpr int kNA = 2;             // input tile ring
constexpr int kThreads = 10 * 32;  // TMA, MMA, two epilogue groups of 4 warps
constexpr uint32_t kKBlock = 128 * 128;         // one 128-byte-wide K block: [128 rows x 128 B]
constexpr uint32_t kOutBytes = kCols * 4;       // 64 KB fp32 / int32 output tile (staging)
// ES = 2: fp16 in (kind::f16, 2 K blocks of 64, 8 MMAs of K = 16);
// ES = 1: int8 in (kind::i8, 1 K block of 128, 4 MMAs of K = 32), exact int32 sums.
template <int ES>
struct TcCfg {
    static constexpr uint32_t kTileBytes = kCols * ES;
    static constexpr int kKBlocks = ES;                 // 128-byte K blocks per tile row
    static constexpr int kKPerMma = 16 * (3 - ES);      // 16 (f16) / 32 (i8) elements
    static constexpr int kMmaPerBlock = 128 / ES / kKPerMma;  // 4 per K block
    static constexpr size_t kSmem = kTileBytes /*T*/ + kNA * kTileBytes + 2 * kOutBytes;
};
constexpr uint32_t kTileBytes = kCols * 2;    // fp16 (kept for the host launcher)
constexpr size_t kSmem = TcCfg<2>::kSmem;

struct TcParams {
    CUtensorMap tm_in;   // 3-D {128 fp16, 128 chunks, rows}, box {64, 128, 1}, SWIZZLE_128B
    void* out;           // fp32 (fp16 input) or int32 (int8 input)
    int64_t rows;
    int64_t out_stride;  // elements
};

__device__ __forceinline__ uint64_t sw128_desc(uint32_t smem_addr)
{
    // K-major, SWIZZLE_128B: start >> 4, LBO (ignored) = 1, SBO = 1024 B between
    // 8-row core-matrix groups, descriptor version 1 (sm_100), layout 2.
    uint64_t d = 0;
    d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);
    d |= (uint64_t)1u << 16;
    d |= (uint64_t)(1024u >> 4) << 32;
    d |= (uint64_t)1u << 46;
    d |= (uint64_t)2u << 61;
    return d;
}

// Instruction descriptors, both operands K-major, N = M = 128:
// kind::f16: D fp32 (c_format 1), A/B fp16 (format 0);
// kind::i8:  D s32 (c_format 2), A/B signed int8 (format 1).
constexpr uint32_t kIdesc = (1u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
constexpr uint32_t kIdescI8 = (2u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(kIdescI8), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     ptx::smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32])
{
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = r[i];
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tma_load_3d_tc(void* dst, const CUtensorMap* tm, int x, int y, int z, uint64_t* bar,
                                               uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(ptx::smem_u32(dst)),
        "l"(tm), "r"(x), "r"(y), "r"(z), "r"(ptx::smem_u32(bar)), "l"(pol)
        : "memory");
}

template <typename V>
struct alignas(16) V4 {
    V x, y, z, w;
};

template <int ES>
__global__ void __launch_bounds__(kThreads, 1) k_rowscan_tc(const __grid_constant__ TcParams p)
{
    using C = TcCfg<ES>;
    using V = typename std::conditional<ES == 2, float, uint32_t>::type;  // accumulator / output type
    constexpr uint32_t kTB = C::kTileBytes;
    extern __shared__ __align__(1024) uint8_t smem_raw[];  // SWIZZLE_128B operands need 1024-B alignment
    uint8_t* const base = smem_raw;
    uint8_t* const sT = base;                  // T = U^T operand, ES K-blocks of 16 KB
    uint8_t* const sX = base + kTB;            // kNA input tiles
    V* const sO0 = reinterpret_cast<V*>(base + kTB + kNA * kTB);  // output staging x2

    __shared__ __align__(8) uint64_t a_full[kNA], a_empty[kNA], t_full[2], t_empty[2];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(16) V s_tot[2][128];   // per epilogue group
    __shared__ __align__(16) V s_base[2][128];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    // T[j][k] = (k <= j) as fp16, K-major SW128: K block kb = k / 64, row j at
    // j*128 B, 16-byte chunk c = (k%64)/8 stored at chunk c ^ (j % 8).
    for (int e = tid; e < 128 * 128; e += kThreads) {
        const int j = e >> 7, k = e & 127;
        if constexpr (ES == 2) {  // fp16 1.0, K blocks of 64 elements
            const int kb = k >> 6, kk = k & 63;
            const uint32_t off = kb * kKBlock + j * 128 + ((((kk >> 3) ^ (j & 7)) << 4)) + (kk & 7) * 2;
            *reinterpret_cast<uint16_t*>(sT + off) = (k <= j) ? (uint16_t)0x3C00 : (uint16_t)0;
        } else {                  // int8 1, one K block of 128 elements
            const uint32_t off = j * 128 + ((((k >> 4) ^ (j & 7)) << 4)) + (k & 15);
            sT[off] = (k <= j) ? (uint8_t)1 : (uint8_t)0;
        }
    }
    if (tid == 0) {
        for (int s = 0; s < kNA; ++s) {
            ptx::mbar_init(&a_full[s], 1);
            ptx::mbar_init(&a_empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&t_full[b], 1);
            ptx::mbar_init(&t_empty[b], 128);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) {  // TMEM: 2 accumulator buffers x 128 columns
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(ptx::smem_u32(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // generic-proxy writes of T must be visible to the tensor core (async proxy)
    ptx::fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;

    if (warp == 0) {
        // ============ TMA producer ============
        if (lane == 0) {
            const uint64_t pol = ptx::policy_evict_first();
            int s = 0;
            uint32_t ph = 0;
            bool wrapped = false;
            for (int64_t r = blockIdx.x; r < p.rows; r += gridDim.x) {
                if (wrapped) ptx::mbar_wait(&a_empty[s], ph ^ 1u);
                uint8_t* dst = sX + s * kTB;
                ptx::mbar_arrive_expect_tx(&a_full[s], kTB);
#pragma unroll
                for (int kb = 0; kb < C::kKBlocks; ++kb)
                    tma_load_3d_tc(dst + kb * kKBlock, &p.tm_in, kb * (128 / ES), 0, (int)r, &a_full[s], pol);
                if (++s == kNA) {
                    s = 0;
                    ph ^= 1u;
                    wrapped = true;
                }
            }
        }
    } else if (warp == 1) {
        // ============ MMA issuer ============
        if (lane == 0) {
            const uint32_t t_addr = ptx::smem_u32(sT);
            int s = 0;
            uint32_t ph = 0;
            int64_t i = 0;
            for (int64_t r = blockIdx.x; r < p.rows; r += gridDim.x, ++i) {
                const int b = (int)(i & 1);
                if (i >= 2) ptx::mbar_wait(&t_empty[b], (uint32_t)((i >> 1) - 1) & 1u);
                ptx::mbar_wait(&a_full[s], ph);
                tc_fence_after();
                const uint32_t x_addr = ptx::smem_u32(sX + s * kTB);
                const uint32_t d = tmem + (uint32_t)(b * 128);
#pragma unroll
                for (int kb = 0; kb < C::kKBlocks; ++kb) {
#pragma unroll
                    for (int k = 0; k < C::kMmaPerBlock; ++k) {  // 32 bytes of K per MMA
                        const uint64_t a = sw128_desc(t_addr + kb * kKBlock + k * 32);
                        const uint64_t bb = sw128_desc(x_addr + kb * kKBlock + k * 32);
                        if constexpr (ES == 2) mma_f16(d, a, bb, (kb | k) != 0);
                        else mma_i8(d, a, bb, (kb | k) != 0);
                    }
                }
                mma_commit(&a_empty[s]);  // input slot free once these MMAs have read it
                mma_commit(&t_full[b]);   // accumulator ready
                if (++s == kNA) {
                    s = 0;
                    ph ^= 1u;
                }
            }
        }
    } else {
        // ============ epilogue: thread = TMEM lane j ============
        // Two groups of 4 warps take alternate tiles (group g <-> TMEM buffer g),
        // so one group stages / stores while the other loads its accumulator.
        const int q = warp & 3;                // TMEM lane quarter this warp may access
        const int j = q * 32 + lane;           // position within a 128-element chunk
        const int g = (warp - 2) >> 2;         // epilogue group
        const int ew = (warp - 2) & 3;         // warp within the group
        const int bar_id = 1 + g;
        V* const sO = sO0 + g * (kOutBytes / 4);  // this group's two 32 KB half-tile buffers
        int hb = 0;                                    // next half buffer
        int64_t i = g;
        for (int64_t r = blockIdx.x + (int64_t)g * gridDim.x; r < p.rows; r += 2 * (int64_t)gridDim.x, i += 2) {
            const int b = g;
            ptx::mbar_wait(&t_full[b], (uint32_t)(i >> 1) & 1u);
            tc_fence_after();
            V v[128];
            const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * 128);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t w[32];
                tmem_ld32(ta + c * 32, w);
#pragma unroll
                for (int t = 0; t < 32; ++t) {
                    if constexpr (ES == 2) v[c * 32 + t] = __uint_as_float(w[t]);
                    else v[c * 32 + t] = w[t];
                }
            }
            tmem_wait_ld();
            tc_fence_before();
            ptx::mbar_arrive(&t_empty[b]);
            // chunk totals D[127][m] -> exclusive scan over m (the L^- A 1 term)
            if (j == 127) {
#pragma unroll
                for (int m = 0; m < 128; m += 4)
                    *reinterpret_cast<V4<V>*>(&s_tot[b][m]) = V4<V>{v[m], v[m + 1], v[m + 2], v[m + 3]};
            }
            ptx::named_bar_sync(bar_id, 128);
            if (ew == 0) {
                const V4<V> t4 = *reinterpret_cast<const V4<V>*>(&s_tot[b][lane * 4]);
                const V l0 = t4.x, l1 = l0 + t4.y, l2 = l1 + t4.z, l3 = l2 + t4.w;
                V incl = l3;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const V y = __shfl_up_sync(0xffffffffu, incl, d);
                    if (lane >= d) incl += y;
                }
                V ex = __shfl_up_sync(0xffffffffu, incl, 1);
                if (lane == 0) ex = V(0);
                *reinterpret_cast<V4<V>*>(&s_base[b][lane * 4]) = V4<V>{ex, ex + l0, ex + l1, ex + l2};
                if (lane == 0) ptx::bulk_wait_read<1>();  // buffer hb's previous store has read it
            }
            ptx::named_bar_sync(bar_id, 128);
            // out[128 m + j] = base[m] + D[j][m]: consecutive threads, consecutive
            // words; staged and stored in two halves of 64 chunks (32 KB each)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (h == 1) {  // buffer hb was last read by the store issued two stores ago
                    if (ew == 0 && lane == 0) ptx::bulk_wait_read<1>();
                    ptx::named_bar_sync(bar_id, 128);
                }
                V* const buf = sO + hb * (kOutBytes / 8);
#pragma unroll
                for (int m = 64 * h; m < 64 * h + 64; m += 4) {
                    const V4<V> bs = *reinterpret_cast<const V4<V>*>(&s_base[b][m]);
                    const int mm = m - 64 * h;
                    buf[(mm + 0) * 128 + j] = bs.x + v[m + 0];
                    buf[(mm + 1) * 128 + j] = bs.y + v[m + 1];
                    buf[(mm + 2) * 128 + j] = bs.z + v[m + 2];
                    buf[(mm + 3) * 128 + j] = bs.w + v[m + 3];
                }
                ptx::fence_proxy_async_smem();
                ptx::named_bar_sync(bar_id, 128);
                if (ew == 0 && lane == 0) {
                    ptx::tma_store_1d(reinterpret_cast<V*>(p.out) + r * p.out_stride + h * 64 * 128, buf, kOutBytes / 2,
                                      ptx::policy_evict_first());
                    ptx::bulk_commit();
                }
                hb ^= 1;
            }
        }
        if (ew == 0 && lane == 0) ptx::bulk_wait<0>();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
    }
}

}  // namespace tc
}  // namespace scan

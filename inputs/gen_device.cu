/*
 * gen_device.cu -- device fill of the seeded input recipes in recipe.h, so
 * the bench can materialise multi-GiB inputs in HBM quickly.  Test/bench
 * infrastructure: no scan arithmetic here.  Built with -fmad=false so every
 * recipe evaluates exactly as gen_host.c does (bit-identical, pinned by
 * tests/test_inputs_gpu.py).
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include "recipe.h"
#include "softmax.h"

template <typename T, typename F>
__global__ void k_fill(T* __restrict__ out, uint64_t seed, uint64_t start, uint64_t n, F f)
{
    uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = f(seed, start + i);
}

struct FI32U100 { __device__ int32_t operator()(uint64_t s, uint64_t i) const { return inputs_i32_u100(s, i); } };
struct FI8Flag { __device__ int8_t operator()(uint64_t s, uint64_t i) const { return inputs_i8_flag(s, i); } };
struct FF16U01 { __device__ uint16_t operator()(uint64_t s, uint64_t i) const { return inputs_f16_u01(s, i); } };
struct FF32Normal { __device__ float operator()(uint64_t s, uint64_t i) const { return inputs_f32_normal(s, i); } };
struct FI32Full { __device__ int32_t operator()(uint64_t s, uint64_t i) const { return inputs_i32_full(s, i); } };
struct FI8Full { __device__ int8_t operator()(uint64_t s, uint64_t i) const { return inputs_i8_full(s, i); } };
struct FF32U01 { __device__ float operator()(uint64_t s, uint64_t i) const { return inputs_f32_u01(s, i); } };
struct FF32PM1 { __device__ float operator()(uint64_t s, uint64_t i) const { return inputs_f32_pm1(s, i); } };
struct FF16Normal { __device__ uint16_t operator()(uint64_t s, uint64_t i) const { return inputs_f16_normal(s, i); } };

/* One warp per row: lane L owns partial_L (softmax.h's fixed order). */
__global__ void k_softmax_stats(uint64_t seed, uint64_t row0, uint64_t rows, uint64_t cols,
                                float* __restrict__ mrow, double* __restrict__ srow)
{
    uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t lane = threadIdx.x & 31;
    if (warp >= rows) return;
    uint64_t row = row0 + warp;
    float m = -INFINITY;
    for (uint64_t c = lane; c < cols; c += 32) {
        float l = inputs_softmax_logit(seed, row, cols, c);
        m = l > m ? l : m;
    }
    for (int o = 16; o > 0; o >>= 1) {
        float other = __shfl_xor_sync(0xffffffffu, m, o);
        m = other > m ? other : m;
    }
    double part = inputs_softmax_lane_partial(seed, row, cols, lane, m);
    double S = 0.0;
    for (int L = 0; L < 32; ++L) S = S + __shfl_sync(0xffffffffu, part, L);
    if (lane == 0) { mrow[warp] = m; srow[warp] = S; }
}

__global__ void k_softmax_fill(uint64_t seed, uint64_t row0, uint64_t rows, uint64_t cols,
                               const float* __restrict__ mrow, const double* __restrict__ srow,
                               float* __restrict__ out)
{
    uint64_t total = rows * cols;
    uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        uint64_t r = i / cols, c = i - r * cols;
        out[i] = inputs_softmax_value(seed, row0 + r, cols, c, mrow[r], srow[r]);
    }
}

template <typename T, typename F>
static int launch(void* out, uint64_t seed, uint64_t start, uint64_t n, cudaStream_t s, F f)
{
    if (n == 0) return 0;
    uint64_t blocks = (n + 255) / 256;
    if (blocks > 148ull * 64) blocks = 148ull * 64;
    k_fill<T, F><<<(unsigned)blocks, 256, 0, s>>>((T*)out, seed, start, n, f);
    return (int)cudaGetLastError();
}

/* Same contract as inputs_fill_host; `out` is a device pointer; asynchronous
 * on `stream`.  Returns 0 or a cudaError_t / -1 (unknown kind). */
extern "C" int inputs_fill_device(int kind, uint64_t seed, uint64_t start, uint64_t n,
                                  uint64_t cols, void* out, void* stream)
{
    cudaStream_t s = (cudaStream_t)stream;
    switch (kind) {
    case INPUTS_I32_U100: return launch<int32_t>(out, seed, start, n, s, FI32U100{});
    case INPUTS_I8_FLAG: return launch<int8_t>(out, seed, start, n, s, FI8Flag{});
    case INPUTS_F16_U01: return launch<uint16_t>(out, seed, start, n, s, FF16U01{});
    case INPUTS_F32_NORMAL: return launch<float>(out, seed, start, n, s, FF32Normal{});
    case INPUTS_I32_FULL: return launch<int32_t>(out, seed, start, n, s, FI32Full{});
    case INPUTS_I8_FULL: return launch<int8_t>(out, seed, start, n, s, FI8Full{});
    case INPUTS_F32_U01: return launch<float>(out, seed, start, n, s, FF32U01{});
    case INPUTS_F32_PM1: return launch<float>(out, seed, start, n, s, FF32PM1{});
    case INPUTS_F16_NORMAL: return launch<uint16_t>(out, seed, start, n, s, FF16Normal{});
    case INPUTS_F32_SOFTMAX: {
        if (n == 0 || cols == 0) return 0;
        float* m = nullptr; double* S = nullptr;
        int e = (int)cudaMallocAsync((void**)&m, n * sizeof(float), s); if (e) return e;
        e = (int)cudaMallocAsync((void**)&S, n * sizeof(double), s); if (e) return e;
        uint64_t threads = n * 32;
        k_softmax_stats<<<(unsigned)((threads + 127) / 128), 128, 0, s>>>(seed, start, n, cols, m, S);
        uint64_t total = n * cols;
        uint64_t blocks = (total + 255) / 256;
        if (blocks > 148ull * 64) blocks = 148ull * 64;
        k_softmax_fill<<<(unsigned)blocks, 256, 0, s>>>(seed, start, n, cols, m, S, (float*)out);
        e = (int)cudaGetLastError(); if (e) return e;
        cudaFreeAsync(m, s); cudaFreeAsync(S, s);
        return (int)cudaGetLastError(); }
    default: return -1;
    }
}

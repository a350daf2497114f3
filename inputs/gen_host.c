/*
 * gen_host.c -- host (CPU) fill of the seeded input recipes in recipe.h.
 * Test/bench infrastructure: no scan arithmetic here.  Single-threaded; inputs/__init__.py splits large fills over threads (ctypes drops the GIL).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include "recipe.h"
#include "softmax.h"

/* Fill out[0..n) with recipe `kind`, elements start..start+n of the stream.
 * For INPUTS_F32_SOFTMAX, start/n count ROWS of `cols` floats.
 * Returns 0, or -1 for an unknown kind. */
int inputs_fill_host(int kind, uint64_t seed, uint64_t start, uint64_t n, uint64_t cols,
                     void* out)
{
    int64_t N = (int64_t)n;
    switch (kind) {
    case INPUTS_I32_U100: {
        int32_t* o = (int32_t*)out;
        for (int64_t i = 0; i < N; ++i) o[i] = inputs_i32_u100(seed, start + (uint64_t)i);
        return 0; }
    case INPUTS_I8_FLAG: {
        int8_t* o = (int8_t*)out;
        for (int64_t i = 0; i < N; ++i) o[i] = inputs_i8_flag(seed, start + (uint64_t)i);
        return 0; }
    case INPUTS_F16_U01: {
        uint16_t* o = (uint16_t*)out;
        for (int64_t i = 0; i < N; ++i) o[i] = inputs_f16_u01(seed, start + (uint64_t)i);
        return 0; }
    case INPUTS_F32_NORMAL: {
        float* o = (float*)out;
        for (int64_t i = 0; i < N; ++i) o[i] = inputs_f32_normal(seed, start + (uint64_t)i);
        return 0; }
    case INPUTS_I32_FULL: {
        int32_t* o = (int32_t*)out;
        for (int64_t i = 0; i < N; ++i) o[i] = inputs_i32_full(seed, start + (uint64_t)i);
        return 0; }
    case INPUTS_I8_FULL: {
        int8_t* o = (int8_t*)out;
        for (int64_t i = 0; i < N; ++i) o[i] = inputs_i8_full(seed, start + (uint64_t)i);
        return 0; }
    case INPUTS_F32_U01: {
        float* o = (float*)out;
        for (int64_t i = 0; i < N; ++i) o[i] = inputs_f32_u01(seed, start + (uint64_t)i);
        return 0; }
    case INPUTS_F32_PM1: {
        float* o = (float*)out;
        for (int64_t i = 0; i < N; ++i) o[i] = inputs_f32_pm1(seed, start + (uint64_t)i);
        return 0; }
    case INPUTS_F16_NORMAL: {
        uint16_t* o = (uint16_t*)out;
        for (int64_t i = 0; i < N; ++i) o[i] = inputs_f16_normal(seed, start + (uint64_t)i);
        return 0; }
    case INPUTS_F32_SOFTMAX: {
        float* o = (float*)out;
        int64_t C = (int64_t)cols;
        for (int64_t rr = 0; rr < N; ++rr) {
            uint64_t row = start + (uint64_t)rr;
            float m = -INFINITY;
            for (int64_t c = 0; c < C; ++c) {
                float l = inputs_softmax_logit(seed, row, cols, (uint64_t)c);
                if (l > m) m = l;
            }
            double S = 0.0;
            for (uint32_t lane = 0; lane < 32; ++lane)
                S = S + inputs_softmax_lane_partial(seed, row, cols, lane, m);
            for (int64_t c = 0; c < C; ++c)
                o[rr * C + c] = inputs_softmax_value(seed, row, cols, (uint64_t)c, m, S);
        }
        return 0; }
    default:
        return -1;
    }
}

/*
 * recipe.h -- seeded synthetic input recipes for the five BASELINE.json
 * configs (C1..C5) and the parity tests.
 *
 * This module holds NONE of the scan's arithmetic: it only draws input
 * values.  It is the one piece of code that serves both sides of a parity
 * check: gen_host.c (gcc, for the oracle and the CPU
 * tests) and gen_device.cu (nvcc, to fill device buffers for the bench) both
 * include this header, so every recipe is a single source.  Both are built
 * without FMA contraction (gcc -ffp-contract=off, nvcc -fmad=false) and use
 * only correctly-rounded IEEE operations (+ - * / sqrt, floor), so host and
 * device produce bit-identical values (pinned by tests/test_inputs*.py).
 *
 * Counter-based generator: element i of a stream
 * with seed s is a pure function  h = splitmix64((s << 48) | i).
 *
 * Recipes:
 *   I32_U100    C1: int32 uniform in [-100, 100]   ((h>>32)*201)>>32 - 100
 *   I8_FLAG     C3: int8 Bernoulli(0.5) flag        h >> 63
 *   F16_U01     C2: U[0,1) with 24 bits, k*2^-24, rounded to fp16 (RNE)
 *   F32_NORMAL  C5: N(0,1) by Box-Muller on two 24-bit uniforms in fp64,
 *               rounded once to fp32
 *   F32_SOFTMAX C4: per row r of `cols`, z = F32_NORMAL at index r*cols+c,
 *               p = softmax(4 z) in fp64 (sequential row sum), rounded once
 *   I32_FULL, I8_FULL, F32_U01, F32_PM1, F16_NORMAL: extra test recipes.
 */
#ifndef SCAN_INPUTS_RECIPE_H
#define SCAN_INPUTS_RECIPE_H

#include <stdint.h>

#ifdef __CUDACC__
#define INPUTS_HD __host__ __device__ __forceinline__
#else
#define INPUTS_HD static inline
#endif

enum inputs_kind {
    INPUTS_I32_U100 = 0,
    INPUTS_I8_FLAG = 1,
    INPUTS_F16_U01 = 2,
    INPUTS_F32_NORMAL = 3,
    INPUTS_F32_SOFTMAX = 4,
    INPUTS_I32_FULL = 5,   /* all 2^32 int32 values, exercises wrap-around */
    INPUTS_I8_FULL = 6,    /* all 256 int8 values                         */
    INPUTS_F32_U01 = 7,    /* k * 2^-24, exact in fp32                    */
    INPUTS_F32_PM1 = 8,    /* {-1, 0, +1}: every prefix exact in fp32     */
    INPUTS_F16_NORMAL = 9  /* N(0,1) rounded to fp16                      */
};

INPUTS_HD uint64_t inputs_splitmix64(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

INPUTS_HD uint64_t inputs_hash(uint64_t seed, uint64_t i)
{
    return inputs_splitmix64((seed << 48) | (i & 0xFFFFFFFFFFFFull));
}

INPUTS_HD uint64_t inputs_dbits(double d)
{
    union { double d; uint64_t u; } c; c.d = d; return c.u;
}
INPUTS_HD double inputs_bitsd(uint64_t u)
{
    union { double d; uint64_t u; } c; c.u = u; return c.d;
}
INPUTS_HD uint32_t inputs_fbits(float f)
{
    union { float f; uint32_t u; } c; c.f = f; return c.u;
}

/* float -> IEEE binary16 bits, round to nearest even, in integer arithmetic. */
INPUTS_HD uint16_t inputs_f32_to_f16(float f)
{
    uint32_t x = inputs_fbits(f);
    uint32_t sign = (x >> 16) & 0x8000u;
    uint32_t ax = x & 0x7FFFFFFFu;
    if (ax >= 0x7F800000u) return (uint16_t)(sign | (ax > 0x7F800000u ? 0x7E00u : 0x7C00u));
    if (ax >= 0x477FF000u) return (uint16_t)(sign | 0x7C00u);     /* >= 65520 -> inf */
    if (ax <= 0x33000000u) return (uint16_t)sign;                 /* <= 2^-25 -> 0   */
    uint32_t e = ax >> 23;
    uint32_t mant = (ax & 0x7FFFFFu) | 0x800000u;
    if (e < 113u) {                                               /* half subnormal  */
        uint32_t shift = 126u - e;
        uint32_t k = mant >> shift;
        uint32_t rem = mant & ((1u << shift) - 1u);
        uint32_t half = 1u << (shift - 1u);
        if (rem > half || (rem == half && (k & 1u))) ++k;
        return (uint16_t)(sign | k);
    }
    uint32_t h = ((e - 112u) << 10) | ((mant & 0x7FFFFFu) >> 13);
    uint32_t rnd = ax & 0x1FFFu;
    if (rnd > 0x1000u || (rnd == 0x1000u && (h & 1u))) ++h;
    return (uint16_t)(sign | h);
}

/* ln(u) for a normal double u > 0: u = m 2^e, m in (sqrt(1/2), sqrt(2)],
 * ln m = 2 atanh(s), s = (m-1)/(m+1), |s| < 0.172, series to s^23. */
INPUTS_HD double inputs_ln(double u)
{
    uint64_t b = inputs_dbits(u);
    int e = (int)((b >> 52) & 0x7FF) - 1023;
    double m = inputs_bitsd((b & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull);
    if (m > 1.4142135623730951) { m = m * 0.5; e = e + 1; }
    double s = (m - 1.0) / (m + 1.0);
    double s2 = s * s;
    double p = 1.0 / 23.0;
    p = p * s2 + 1.0 / 21.0;
    p = p * s2 + 1.0 / 19.0;
    p = p * s2 + 1.0 / 17.0;
    p = p * s2 + 1.0 / 15.0;
    p = p * s2 + 1.0 / 13.0;
    p = p * s2 + 1.0 / 11.0;
    p = p * s2 + 1.0 / 9.0;
    p = p * s2 + 1.0 / 7.0;
    p = p * s2 + 1.0 / 5.0;
    p = p * s2 + 1.0 / 3.0;
    p = p * s2 + 1.0;
    return (double)e * 0.6931471805599453 + 2.0 * s * p;
}

/* cos(x) and sin(x) for |x| <= pi/4 by Taylor series (terms to x^20). */
INPUTS_HD double inputs_cos_small(double x)
{
    double x2 = x * x;
    double p = 1.0 / 2432902008176640000.0;        /* 1/20! */
    p = -p * x2 + 1.0 / 6402373705728000.0;        /* 1/18! */
    p = -p * x2 + 1.0 / 20922789888000.0;          /* 1/16! */
    p = -p * x2 + 1.0 / 87178291200.0;             /* 1/14! */
    p = -p * x2 + 1.0 / 479001600.0;               /* 1/12! */
    p = -p * x2 + 1.0 / 3628800.0;                 /* 1/10! */
    p = -p * x2 + 1.0 / 40320.0;                   /* 1/8!  */
    p = -p * x2 + 1.0 / 720.0;                     /* 1/6!  */
    p = -p * x2 + 1.0 / 24.0;                      /* 1/4!  */
    p = -p * x2 + 1.0 / 2.0;                       /* 1/2!  */
    p = -p * x2 + 1.0;
    return p;
}
INPUTS_HD double inputs_sin_small(double x)
{
    double x2 = x * x;
    double p = 1.0 / 121645100408832000.0;         /* 1/19! */
    p = -p * x2 + 1.0 / 355687428096000.0;         /* 1/17! */
    p = -p * x2 + 1.0 / 1307674368000.0;           /* 1/15! */
    p = -p * x2 + 1.0 / 6227020800.0;              /* 1/13! */
    p = -p * x2 + 1.0 / 39916800.0;                /* 1/11! */
    p = -p * x2 + 1.0 / 362880.0;                  /* 1/9!  */
    p = -p * x2 + 1.0 / 5040.0;                    /* 1/7!  */
    p = -p * x2 + 1.0 / 120.0;                     /* 1/5!  */
    p = -p * x2 + 1.0 / 6.0;                       /* 1/3!  */
    p = -p * x2 + 1.0;
    return p * x;
}

/* cos(2 pi t) for t = k 2^-24 in [0, 1): exact octant reduction. */
INPUTS_HD double inputs_cos2pi(double t)
{
    double sign = 1.0;
    if (t > 0.5) t = 1.0 - t;                    /* cos(2pi t) = cos(2pi (1-t)) */
    if (t > 0.25) { t = 0.5 - t; sign = -1.0; }  /* cos(2pi t) = -cos(2pi (1/2-t)) */
    double c;
    if (t <= 0.125) c = inputs_cos_small(6.283185307179586 * t);
    else c = inputs_sin_small(6.283185307179586 * (0.25 - t));
    return sign * c;
}

/* exp(x) for -700 < x <= 0: x = k ln2 + r, |r| <= ln2/2, Taylor to r^18. */
INPUTS_HD double inputs_exp(double x)
{
    double kd = (double)(int64_t)(x * 1.4426950408889634 - 0.5);  /* round(x/ln2), x <= 0 */
    double r = x - kd * 0.6931471803691238;       /* ln2 high part (exact product) */
    r = r - kd * 1.9082149292705877e-10;          /* ln2 low part                  */
    double p = 1.0 / 6402373705728000.0;          /* 1/18! */
    p = p * r + 1.0 / 355687428096000.0;          /* 1/17! */
    p = p * r + 1.0 / 20922789888000.0;           /* 1/16! */
    p = p * r + 1.0 / 1307674368000.0;            /* 1/15! */
    p = p * r + 1.0 / 87178291200.0;              /* 1/14! */
    p = p * r + 1.0 / 6227020800.0;               /* 1/13! */
    p = p * r + 1.0 / 479001600.0;                /* 1/12! */
    p = p * r + 1.0 / 39916800.0;                 /* 1/11! */
    p = p * r + 1.0 / 3628800.0;                  /* 1/10! */
    p = p * r + 1.0 / 362880.0;                   /* 1/9!  */
    p = p * r + 1.0 / 40320.0;                    /* 1/8!  */
    p = p * r + 1.0 / 5040.0;                     /* 1/7!  */
    p = p * r + 1.0 / 720.0;                      /* 1/6!  */
    p = p * r + 1.0 / 120.0;                      /* 1/5!  */
    p = p * r + 1.0 / 24.0;                       /* 1/4!  */
    p = p * r + 1.0 / 6.0;                        /* 1/3!  */
    p = p * r + 0.5;
    p = p * r + 1.0;
    p = p * r + 1.0;
    int64_t k = (int64_t)kd;
    return p * inputs_bitsd((uint64_t)(k + 1023) << 52);
}

/* ---- per-element recipes ------------------------------------------- */

INPUTS_HD int32_t inputs_i32_u100(uint64_t seed, uint64_t i)
{
    uint64_t h = inputs_hash(seed, i);
    return (int32_t)(((h >> 32) * 201ull) >> 32) - 100;
}

INPUTS_HD int8_t inputs_i8_flag(uint64_t seed, uint64_t i)
{
    return (int8_t)(inputs_hash(seed, i) >> 63);
}

INPUTS_HD uint16_t inputs_f16_u01(uint64_t seed, uint64_t i)
{
    uint64_t h = inputs_hash(seed, i);
    float u = (float)(uint32_t)(h >> 40) * 5.9604644775390625e-08f;  /* k * 2^-24, exact */
    return inputs_f32_to_f16(u);
}

INPUTS_HD double inputs_normal64(uint64_t seed, uint64_t i)
{
    uint64_t h = inputs_hash(seed, i);
    double u1 = (double)((h >> 40) + 1ull) * 5.9604644775390625e-08;          /* (0,1] */
    double t = (double)((h >> 16) & 0xFFFFFFull) * 5.9604644775390625e-08;    /* [0,1) */
    double r = -2.0 * inputs_ln(u1);
    if (r < 0.0) r = 0.0;                        /* ln(1) = 0 exactly; guard -0 */
    return sqrt(r) * inputs_cos2pi(t);
}

INPUTS_HD float inputs_f32_normal(uint64_t seed, uint64_t i)
{
    return (float)inputs_normal64(seed, i);
}

INPUTS_HD int32_t inputs_i32_full(uint64_t seed, uint64_t i)
{
    return (int32_t)(uint32_t)(inputs_hash(seed, i) >> 32);
}

INPUTS_HD int8_t inputs_i8_full(uint64_t seed, uint64_t i)
{
    return (int8_t)(uint8_t)(inputs_hash(seed, i) >> 56);
}

INPUTS_HD float inputs_f32_u01(uint64_t seed, uint64_t i)
{
    return (float)(uint32_t)(inputs_hash(seed, i) >> 40) * 5.9604644775390625e-08f;
}

INPUTS_HD float inputs_f32_pm1(uint64_t seed, uint64_t i)
{
    return (float)((int)((inputs_hash(seed, i) >> 32) % 3ull) - 1);
}

INPUTS_HD uint16_t inputs_f16_normal(uint64_t seed, uint64_t i)
{
    return inputs_f32_to_f16(inputs_f32_normal(seed, i));
}

/* C4 softmax rows: logit l_c = 4 * z_c (exact in fp32). */
INPUTS_HD float inputs_softmax_logit(uint64_t seed, uint64_t row, uint64_t cols, uint64_t c)
{
    return 4.0f * inputs_f32_normal(seed, row * cols + c);
}

#endif /* SCAN_INPUTS_RECIPE_H */

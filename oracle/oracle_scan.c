/*
 * oracle_scan.c -- plain sequential CPU oracle for the prefix sum (scan).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load or call this code.
 * The product path (paper_2505_15112_b200/) never links, imports or executes
 * anything under oracle/, and this file shares no code, header, table or
 * constant with the CUDA kernels.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, "P<line>"):
 *   - P68 (Sec. 2, Background): "The inclusive prefix sum of a sequence of
 *     elements x_1, x_2, x_3, ... equipped with a binary associative operator
 *     (.) is the sequence x_1, x_1 (.) x_2, x_1 (.) x_2 (.) x_3, ...".  Here
 *     (.) is addition.  Written out: y_1 = x_1, y_i = y_{i-1} + x_i.
 *   - P461 (App. B.2, "Exclusive and int8 scan"): the exclusive scan is the
 *     inclusive output "shifted by one element, discarding the last value and
 *     writing zero to the first position".  Written out: e_1 = 0,
 *     e_i = y_{i-1}.
 *   - P98 (Sec. 3.1) and P459 (App. B.2): fp16 input with fp32 output and
 *     int8 input with int32 output ("input matrices of 8-bit integers with
 *     output/accumulation in 32-bit integers").
 *   - P437 (App. B.1): a batched scan is the scan of every row independently.
 *   - P73 (Sec. 2.1, RSS): a block-level *reduction* (total) of a range.
 *
 * Readings where the paper is silent (DESIGN.md "Readings" R1..R8):
 *   R1 integer overflow wraps mod 2^32 (two's complement); accumulation is
 *      done in uint32_t, which C defines to wrap.
 *   R2 int8 values are summed as signed integers (flags are the 0/1 case).
 *   R3 a carry-in c (0 by default) is added in front of the sequence:
 *      inclusive y_i = c + sum_{j<=i} x_j, exclusive e_i = c + sum_{j<i} x_j.
 *      With no carry and no previous chunk the first inclusive value is x_1
 *      itself (P68), so the sign of -0.0 is kept.
 *   R4 floating point: every input is widened exactly to double and the
 *      running sum is kept in double, sequentially, in index order; the fp32
 *      result is ONE round-to-nearest-even conversion of that double.  The
 *      tolerance weight A_i = sum_{j<=i} |x_j| (BASELINE.json north_star) is
 *      accumulated beside it, also in double.
 *   R6 with a carry-in c (which stands for the sum of the elements before
 *      this array, e.g. lower shards) the weight starts at |c|:
 *      A_i = |c| + sum_{j<=i} |x_j|, a lower bound of the weight the same
 *      element has in the unsharded array.
 *   R5 fp16 is decoded from its IEEE-754 binary16 bit layout here (sign,
 *      5-bit exponent, 10-bit fraction, subnormals, inf/NaN) so the oracle
 *      does not depend on any CUDA conversion routine.
 *
 * Streaming: every scan function takes a state struct carried from one chunk
 * to the next, so arrays larger than host RAM can be checked piecewise; a
 * single call over the whole array and any chunking give identical results
 * (tests/test_oracle.py pins this).
 *
 * Build: gcc -O2 -fno-fast-math -ffp-contract=off (no reassociation, no FMA
 * contraction) -- see oracle/Makefile.
 */
#include <stdint.h>
#include <string.h>
#include <math.h>

/* ------------------------------------------------------------------ */
/* Integer state: running sum mod 2^32 (R1).                           */
/* ------------------------------------------------------------------ */
typedef struct {
    uint32_t sum;      /* c + sum of all elements seen so far, mod 2^32 */
    int64_t  count;    /* elements seen so far                          */
} oracle_istate;

void oracle_istate_init(oracle_istate* st, int64_t carry_in)
{
    st->sum = (uint32_t)(uint64_t)carry_in;   /* carry taken mod 2^32 */
    st->count = 0;
}

/* P68 inclusive / P461 exclusive over int32 input, int32 output. */
void oracle_scan_i32(const int32_t* x, int64_t n, int exclusive,
                     oracle_istate* st, int32_t* y)
{
    for (int64_t i = 0; i < n; ++i) {
        uint32_t before = st->sum;
        st->sum = before + (uint32_t)x[i];
        y[i] = (int32_t)(exclusive ? before : st->sum);
    }
    st->count += n;
}

/* P459: int8 input (signed, R2), int32 accumulation and output. */
void oracle_scan_i8(const int8_t* x, int64_t n, int exclusive,
                    oracle_istate* st, int32_t* y)
{
    for (int64_t i = 0; i < n; ++i) {
        uint32_t before = st->sum;
        st->sum = before + (uint32_t)(int32_t)x[i];   /* sign-extend */
        y[i] = (int32_t)(exclusive ? before : st->sum);
    }
    st->count += n;
}

/* ------------------------------------------------------------------ */
/* Floating-point state: fp64 running sum and |x| sum (R4).            */
/* ------------------------------------------------------------------ */
typedef struct {
    double  sum;       /* c + sum_{j<i} x_j in double                    */
    double  abs_sum;   /* sum_{j<i} |x_j| in double (tolerance weight)   */
    int64_t count;     /* elements seen so far                           */
    int     has_carry; /* 1 if a carry-in was given (R3)                 */
} oracle_fstate;

void oracle_fstate_init(oracle_fstate* st, double carry_in, int has_carry)
{
    st->sum = has_carry ? carry_in : 0.0;
    st->abs_sum = has_carry ? fabs(carry_in) : 0.0;   /* R6: the carry stands for the
                                                         elements before this array */
    st->count = 0;
    st->has_carry = has_carry;
}

/* R5: IEEE-754 binary16 -> double, from the bit layout. */
double oracle_f16_to_f64(uint16_t h)
{
    int sign = (h >> 15) & 1;
    int exponent = (h >> 10) & 0x1f;
    int fraction = h & 0x3ff;
    double v;
    if (exponent == 0) {
        v = ldexp((double)fraction, -24);                 /* subnormal: f * 2^-24 */
    } else if (exponent == 31) {
        v = fraction ? NAN : INFINITY;
    } else {
        v = ldexp((double)(1024 + fraction), exponent - 25);  /* (1 + f/1024) 2^(e-15) */
    }
    return sign ? -v : v;
}

/* One element of the float scan: shared by the fp32 and fp16 paths below. */
static void fstep(double xi, int exclusive, oracle_fstate* st,
                  double* y64, double* a64, float* y32, int64_t i)
{
    double before = st->sum;
    double inc;
    if (st->count == 0 && i == 0 && !st->has_carry)
        inc = xi;                          /* P68: y_1 = x_1 */
    else
        inc = before + xi;
    double out = exclusive ? before : inc;
    st->abs_sum = st->abs_sum + fabs(xi);
    st->sum = inc;
    if (y64) y64[i] = out;
    if (a64) a64[i] = st->abs_sum;        /* A_i = sum_{j<=i} |x_j| */
    if (y32) y32[i] = (float)out;         /* one RNE rounding (R4)  */
}

/* fp32 input; outputs (any may be NULL): the fp64 prefix, the tolerance
 * weight A_i, and the once-rounded fp32 prefix. */
void oracle_scan_f32(const float* x, int64_t n, int exclusive, oracle_fstate* st,
                     double* y64, double* a64, float* y32)
{
    for (int64_t i = 0; i < n; ++i)
        fstep((double)x[i], exclusive, st, y64, a64, y32, i);
    st->count += n;
}

/* fp16 input (raw binary16 bits), fp32 output (P98). */
void oracle_scan_f16(const uint16_t* x, int64_t n, int exclusive, oracle_fstate* st,
                     double* y64, double* a64, float* y32)
{
    for (int64_t i = 0; i < n; ++i)
        fstep(oracle_f16_to_f64(x[i]), exclusive, st, y64, a64, y32, i);
    st->count += n;
}

/* ------------------------------------------------------------------ */
/* Totals (RSS "reduce", P73): plain sequential sums.                  */
/* ------------------------------------------------------------------ */
int64_t oracle_total_i32(const int32_t* x, int64_t n)
{
    int64_t s = 0;
    for (int64_t i = 0; i < n; ++i) s += x[i];
    return s;
}

int64_t oracle_total_i8(const int8_t* x, int64_t n)
{
    int64_t s = 0;
    for (int64_t i = 0; i < n; ++i) s += x[i];
    return s;
}

double oracle_total_f32(const float* x, int64_t n)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += (double)x[i];
    return s;
}

double oracle_total_f16(const uint16_t* x, int64_t n)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += oracle_f16_to_f64(x[i]);
    return s;
}

/* ------------------------------------------------------------------ */
/* Tolerance check (BASELINE.json north_star):                         */
/*   |gpu_i - oracle_i| <= 1e-6 * A_i + 1e-6                           */
/* Returns the number of violations; *worst gets max err/tol and        */
/* *worst_at its index.  NaN/inf: the same class is required (R8).      */
/* ------------------------------------------------------------------ */
int64_t oracle_check_f32(const float* got, const double* ref, const double* abs_w,
                         int64_t n, double rel, double abs_tol,
                         double* worst, int64_t* worst_at)
{
    int64_t bad = 0;
    double w = 0.0;
    int64_t at = n > 0 ? 0 : -1;
    for (int64_t i = 0; i < n; ++i) {
        double g = (double)got[i];
        double r = ref[i];
        double ratio;
        if (isnan(r) || isnan(g)) {
            ratio = (isnan(r) && isnan(g)) ? 0.0 : INFINITY;
        } else if (isinf(r) || isinf(g)) {
            ratio = (g == r) ? 0.0 : INFINITY;
        } else {
            double tol = rel * abs_w[i] + abs_tol;
            ratio = fabs(g - r) / tol;
        }
        if (ratio > 1.0) ++bad;
        if (ratio > w) { w = ratio; at = i; }
    }
    if (worst) *worst = w;
    if (worst_at) *worst_at = at;
    return bad;
}

/* Rows (P437): each row of `cols` elements scanned independently, row r
 * starting at x + r*in_stride and written to y + r*out_stride.  Only the
 * int32 and fp32 row types that the configs use need a dedicated entry;
 * other types are checked row by row from Python. */
void oracle_rows_f32(const float* x, int64_t rows, int64_t cols, int64_t in_stride,
                     int64_t out_stride, int exclusive,
                     double* y64, double* a64, float* y32)
{
    for (int64_t r = 0; r < rows; ++r) {
        oracle_fstate st;
        oracle_fstate_init(&st, 0.0, 0);
        oracle_scan_f32(x + r * in_stride, cols, exclusive, &st,
                        y64 ? y64 + r * out_stride : 0,
                        a64 ? a64 + r * out_stride : 0,
                        y32 ? y32 + r * out_stride : 0);
    }
}

void oracle_rows_i32(const int32_t* x, int64_t rows, int64_t cols, int64_t in_stride,
                     int64_t out_stride, int exclusive, int32_t* y)
{
    for (int64_t r = 0; r < rows; ++r) {
        oracle_istate st;
        oracle_istate_init(&st, 0);
        oracle_scan_i32(x + r * in_stride, cols, exclusive, &st, y + r * out_stride);
    }
}

int oracle_abi_version(void) { return 1; }

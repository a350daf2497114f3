/*
 * oracle_threaded.c -- the all-core CPU BASELINE of SURVEY.md 8(c5)/8(d):
 * the sequential oracle of oracle_scan.c split over T host threads.
 *
 * TEST INFRASTRUCTURE ONLY (same rule as oracle_scan.c): only bench.py's
 * cpu_baseline leg and tests/ call it.  It is a reported baseline, never a
 * checker: validation always uses the single-thread functions.
 *
 * What it computes: the scan of P68 / P461 over n elements cut into T
 * contiguous chunks -- the Reduce-Scan-Scan structure of P73 (Sec. 2.1) with
 * threads as the blocks:
 *   pass 1  every thread sums its chunk (oracle_total_*),
 *   carry   chunk c starts from the sum of chunks 0..c-1, added in order,
 *   pass 2  every thread scans its chunk from its carry (oracle_scan_*).
 * Integers wrap mod 2^32 exactly as the sequential scan, so the result is
 * bit-identical to it (tests/test_oracle.py pins this).  Floats: chunk totals
 * and carries in fp64, so the result differs from the sequential fp64 sum
 * only by reassociation at T-1 chunk boundaries (within the tolerance; pinned
 * in the same test).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

/* oracle_scan.c */
typedef struct {
    uint32_t sum;
    int64_t count;
} oracle_istate;
typedef struct {
    double sum;
    double abs_sum;
    int64_t count;
    int has_carry;
} oracle_fstate;
void oracle_istate_init(oracle_istate* st, int64_t carry_in);
void oracle_fstate_init(oracle_fstate* st, double carry_in, int has_carry);
void oracle_scan_i32(const int32_t* x, int64_t n, int exclusive, oracle_istate* st, int32_t* y);
void oracle_scan_i8(const int8_t* x, int64_t n, int exclusive, oracle_istate* st, int32_t* y);
void oracle_scan_f32(const float* x, int64_t n, int exclusive, oracle_fstate* st, double* y64, double* a64,
                     float* y32);
void oracle_scan_f16(const uint16_t* x, int64_t n, int exclusive, oracle_fstate* st, double* y64, double* a64,
                     float* y32);
int64_t oracle_total_i32(const int32_t* x, int64_t n);
int64_t oracle_total_i8(const int8_t* x, int64_t n);
double oracle_total_f32(const float* x, int64_t n);
double oracle_total_f16(const uint16_t* x, int64_t n);

/* dt: 0 int32, 1 fp32, 2 fp16 (raw bits), 3 int8 -- the order of scan.h's scan_dtype */
typedef struct {
    const void* x;
    void* y;
    int64_t lo, hi;
    int dt, exclusive, pass;
    int64_t itot, icarry;
    double ftot, fcarry;
    int first;
} job_t;

static void* run(void* arg)
{
    job_t* j = (job_t*)arg;
    const int64_t n = j->hi - j->lo;
    if (j->pass == 1) {
        switch (j->dt) {
        case 0: j->itot = oracle_total_i32((const int32_t*)j->x + j->lo, n); break;
        case 3: j->itot = oracle_total_i8((const int8_t*)j->x + j->lo, n); break;
        case 1: j->ftot = oracle_total_f32((const float*)j->x + j->lo, n); break;
        default: j->ftot = oracle_total_f16((const uint16_t*)j->x + j->lo, n); break;
        }
        return 0;
    }
    if (j->dt == 0 || j->dt == 3) {
        oracle_istate st;
        oracle_istate_init(&st, j->icarry);
        if (j->dt == 0)
            oracle_scan_i32((const int32_t*)j->x + j->lo, n, j->exclusive, &st, (int32_t*)j->y + j->lo);
        else
            oracle_scan_i8((const int8_t*)j->x + j->lo, n, j->exclusive, &st, (int32_t*)j->y + j->lo);
    } else {
        oracle_fstate st;
        oracle_fstate_init(&st, j->fcarry, !j->first);
        if (j->dt == 1)
            oracle_scan_f32((const float*)j->x + j->lo, n, j->exclusive, &st, 0, 0, (float*)j->y + j->lo);
        else
            oracle_scan_f16((const uint16_t*)j->x + j->lo, n, j->exclusive, &st, 0, 0, (float*)j->y + j->lo);
    }
    return 0;
}

/* y: int32 (integer dtypes) or fp32 (float dtypes), n elements.  Returns 0, or
 * -1 for bad arguments / thread creation failure. */
int oracle_scan_threaded(const void* x, int64_t n, int dt, int exclusive, int threads, void* y)
{
    if (n < 0 || dt < 0 || dt > 3 || threads < 1) return -1;
    if (n == 0) return 0;
    if (threads > n) threads = (int)n;
    job_t* jobs = (job_t*)calloc((size_t)threads, sizeof(job_t));
    pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    if (!jobs || !th) {
        free(jobs);
        free(th);
        return -1;
    }
    const int64_t per = (n + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        jobs[t].x = x;
        jobs[t].y = y;
        jobs[t].lo = (int64_t)t * per < n ? (int64_t)t * per : n;
        jobs[t].hi = jobs[t].lo + per < n ? jobs[t].lo + per : n;
        jobs[t].dt = dt;
        jobs[t].exclusive = exclusive;
        jobs[t].first = t == 0;
    }
    int rc = 0;
    for (int pass = 1; pass <= 2 && rc == 0; ++pass) {
        if (pass == 2) { /* chunk carries, in chunk order */
            int64_t ic = 0;
            double fc = 0.0;
            for (int t = 0; t < threads; ++t) {
                jobs[t].icarry = ic;
                jobs[t].fcarry = fc;
                ic += jobs[t].itot;
                fc += jobs[t].ftot;
            }
        }
        int started = 0;
        for (int t = 0; t < threads; ++t) {
            jobs[t].pass = pass;
            if (pthread_create(&th[t], 0, run, &jobs[t]) != 0) {
                rc = -1;
                break;
            }
            ++started;
        }
        for (int t = 0; t < started; ++t) pthread_join(th[t], 0);
    }
    free(jobs);
    free(th);
    return rc;
}

/* Rows (P437) on T threads: thread t scans rows [t*R/T, (t+1)*R/T) with the
 * sequential row oracle -- rows are independent, so the result is identical to
 * the single-thread row scan for every type. */
typedef struct {
    const void* x;
    void* y;
    int64_t r0, r1, cols;
    int dt, exclusive;
} rjob_t;

static void* run_rows(void* arg)
{
    rjob_t* j = (rjob_t*)arg;
    for (int64_t r = j->r0; r < j->r1; ++r) {
        const int64_t o = r * j->cols;
        if (j->dt == 0 || j->dt == 3) {
            oracle_istate st;
            oracle_istate_init(&st, 0);
            if (j->dt == 0)
                oracle_scan_i32((const int32_t*)j->x + o, j->cols, j->exclusive, &st, (int32_t*)j->y + o);
            else
                oracle_scan_i8((const int8_t*)j->x + o, j->cols, j->exclusive, &st, (int32_t*)j->y + o);
        } else {
            oracle_fstate st;
            oracle_fstate_init(&st, 0.0, 0);
            if (j->dt == 1)
                oracle_scan_f32((const float*)j->x + o, j->cols, j->exclusive, &st, 0, 0, (float*)j->y + o);
            else
                oracle_scan_f16((const uint16_t*)j->x + o, j->cols, j->exclusive, &st, 0, 0, (float*)j->y + o);
        }
    }
    return 0;
}

int oracle_rows_threaded(const void* x, int64_t rows, int64_t cols, int dt, int exclusive, int threads, void* y)
{
    if (rows < 0 || cols < 0 || dt < 0 || dt > 3 || threads < 1) return -1;
    if (rows == 0 || cols == 0) return 0;
    if (threads > rows) threads = (int)rows;
    rjob_t* jobs = (rjob_t*)calloc((size_t)threads, sizeof(rjob_t));
    pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    if (!jobs || !th) {
        free(jobs);
        free(th);
        return -1;
    }
    int rc = 0, started = 0;
    for (int t = 0; t < threads; ++t) {
        jobs[t] = (rjob_t){x, y, rows * t / threads, rows * (t + 1) / threads, cols, dt, exclusive};
        if (pthread_create(&th[t], 0, run_rows, &jobs[t]) != 0) {
            rc = -1;
            break;
        }
        ++started;
    }
    for (int t = 0; t < started; ++t) pthread_join(th[t], 0);
    free(jobs);
    free(th);
    return rc;
}

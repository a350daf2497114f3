/*
 * oracle_ops.c -- plain sequential CPU oracle for the scan-based operators of
 * PAPER.md Sec. 5 ("Parallel scan applications") and App. B.3.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load or call this code.
 * The product path (paper_2505_15112_b200/) never links, imports or executes
 * anything under oracle/, and this file shares no code, header, table or
 * constant with the CUDA kernels.
 *
 * Each operator follows the paper's own formulation step by step, on top of
 * the plain exclusive scan (P461) written out here as a running sum:
 *
 *   - Split / SplitInd (P281-283, Sec. 5.1): "places all items of x where the
 *     corresponding flag is true at the beginning of the output array,
 *     followed by all items where the corresponding flag is false ... the
 *     relative order of the elements is preserved"; SplitInd "executes an
 *     exclusive scan ... on the mask array.  Afterwards, it gathers the
 *     correct input elements and their indices ... and stores them in global
 *     memory at the offsets calculated by the scan".  With e_i the exclusive
 *     scan of the 0/1 mask b and T its total, item i goes to e_i if b_i,
 *     else to T + (i - e_i); idx[dest] = i.
 *   - Compress (P285, Sec. 5.2): "only the first part of the output elements
 *     of the split are returned" (= torch.masked_select).
 *   - Radix sort (P287, Sec. 5.3): LSB radix sort; each iteration "executes a
 *     split where the mask is obtained by reading the corresponding bit" --
 *     mask = NOT(bit) ("ShiftRight and Not"), so 0-bits go first; floats are
 *     pre-encoded by "inverting the Most Significant Bit (MSB) of positive
 *     numbers and all the bits of the negative numbers" and the sorted keys
 *     are decoded back.  Indices are tracked through every split (P365).
 *   - Weighted sampling (P463, App. B.3): scan the weights, draw theta in
 *     [0,1), the sample is the index whose cumulative interval contains
 *     theta * sum(w) (inverse transform sampling).
 *   - Top-p / nucleus sampling (P298-299, Sec. 5.5): sort the probabilities
 *     (descending), scan them, keep the nucleus, sample from it by the
 *     inverse transform on the same scan.
 *
 * Readings where the paper is silent (R12-R16):
 *   R12 a flag is true iff its int8 value is nonzero (P283 stores 0/1 flags in
 *       int8; other values are treated as true, not summed).
 *   R13 the float encoding (P287) orders keys by the IEEE total order:
 *       -NaN < -inf < ... < -0 < +0 < ... < +inf < +NaN; -0 sorts before +0.
 *       Signed integers flip the sign bit; unsigned keys are used as is.
 *       Descending = the same LSB splits with mask = bit (1-bits first), which
 *       is the exact reverse order of the keys and still stable (equal keys
 *       keep their input order, as torch.sort(stable=True, descending=True)).
 *   R14 weighted sampling returns min{ i : S_i > theta * S_{n-1} } with S the
 *       inclusive fp64 scan (equivalently the last i whose exclusive prefix is
 *       <= theta * S_{n-1} for positive weights; P463's SplitInd formulation).
 *   R15 the nucleus is the smallest prefix of the descending order whose mass
 *       reaches p (Holtzman et al.): keep rank k iff k == 0 or E_k < p, with
 *       E_k the exclusive scan of the sorted probabilities; the sample is drawn
 *       from the kept ranks renormalised, t = u * C_K, first kept k with C_k > t.
 *   R16 the uniform numbers (theta, u) are inputs, not drawn here.
 *
 * Build: gcc -O2 -fno-fast-math -ffp-contract=off (oracle/Makefile).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* double value of an IEEE binary16 (defined in oracle_scan.c, R5). */
double oracle_f16_to_f64(uint16_t h);

/* ------------------------------------------------------------------ */
/* Split / SplitInd / Compress (P281-285)                               */
/* ------------------------------------------------------------------ */
/* Returns T (number of true flags).  z holds n elements (split) or T
 * (compress); idx (nullable) the input index of every output element. */
int64_t oracle_split(const void* x, const int8_t* flags, int64_t n, int elem_bytes, int compress,
                     void* z, int32_t* idx)
{
    /* step 1: exclusive scan of the 0/1 mask (P461), kept as e_i */
    int64_t* e = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    int64_t run = 0;
    for (int64_t i = 0; i < n; ++i) {
        e[i] = run;
        run += flags[i] != 0 ? 1 : 0;
    }
    const int64_t T = run;
    /* step 2: gather every item to the offset the scan gives it (P283) */
    const uint8_t* xs = (const uint8_t*)x;
    uint8_t* zs = (uint8_t*)z;
    for (int64_t i = 0; i < n; ++i) {
        int64_t dest;
        if (flags[i] != 0)
            dest = e[i];
        else if (compress)
            continue;
        else
            dest = T + (i - e[i]);
        memcpy(zs + dest * elem_bytes, xs + i * elem_bytes, (size_t)elem_bytes);
        if (idx) idx[dest] = (int32_t)i;
    }
    free(e);
    return T;
}

/* ------------------------------------------------------------------ */
/* Radix sort by LSB splits (P286-287)                                  */
/* ------------------------------------------------------------------ */
enum { ORACLE_U16 = 0, ORACLE_I16 = 1, ORACLE_F16 = 2, ORACLE_U32 = 3, ORACLE_I32 = 4, ORACLE_F32 = 5 };

static int key_bits(int kt) { return kt <= ORACLE_F16 ? 16 : 32; }

/* P287 pre-processing (and R13 for integers). */
uint32_t oracle_sort_encode(uint32_t k, int kt)
{
    switch (kt) {
    case ORACLE_U16: return k & 0xffffu;
    case ORACLE_I16: return (k ^ 0x8000u) & 0xffffu;
    case ORACLE_F16: return (k & 0x8000u) ? (~k & 0xffffu) : (k | 0x8000u);
    case ORACLE_U32: return k;
    case ORACLE_I32: return k ^ 0x80000000u;
    default: return (k & 0x80000000u) ? ~k : (k | 0x80000000u);
    }
}

static uint32_t load_key(const void* keys, int64_t i, int kt)
{
    if (key_bits(kt) == 16) return ((const uint16_t*)keys)[i];
    return ((const uint32_t*)keys)[i];
}

/* Sorts keys (as raw bits) into keys_out, input index of each output into
 * idx_out.  The keys are moved unchanged: encoding the key for the mask and
 * decoding it back afterwards (P287) leaves the bits as they were. */
void oracle_radix_sort(const void* keys, int64_t n, int kt, int descending, void* keys_out, int32_t* idx_out)
{
    const int B = key_bits(kt);
    const int eb = B / 8;
    uint8_t* cur = (uint8_t*)malloc((size_t)(n > 0 ? n : 1) * eb);
    uint8_t* nxt = (uint8_t*)malloc((size_t)(n > 0 ? n : 1) * eb);
    int32_t* ci = (int32_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
    int32_t* ni = (int32_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
    int32_t* gi = (int32_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
    int8_t* f = (int8_t*)malloc((size_t)(n > 0 ? n : 1));
    memcpy(cur, keys, (size_t)n * eb);
    for (int64_t i = 0; i < n; ++i) ci[i] = (int32_t)i;
    for (int b = 0; b < B; ++b) {
        /* RadixSingle: mask = NOT(bit b of the encoded key) (ascending) */
        for (int64_t i = 0; i < n; ++i) {
            const uint32_t bit = (oracle_sort_encode(load_key(cur, i, kt), kt) >> b) & 1u;
            f[i] = (int8_t)(descending ? bit : (bit ^ 1u));
        }
        /* SplitInd on the keys; gi = position in `cur` of every output */
        oracle_split(cur, f, n, eb, 0, nxt, gi);
        for (int64_t j = 0; j < n; ++j) ni[j] = ci[gi[j]];
        uint8_t* t = cur; cur = nxt; nxt = t;
        int32_t* u = ci; ci = ni; ni = u;
    }
    memcpy(keys_out, cur, (size_t)n * eb);
    if (idx_out) memcpy(idx_out, ci, (size_t)n * sizeof(int32_t));
    free(cur); free(nxt); free(ci); free(ni); free(gi); free(f);
}

/* ------------------------------------------------------------------ */
/* Weighted sampling (P463) and top-p sampling (P298-299)               */
/* ------------------------------------------------------------------ */
/* R14: first i with S_i > theta * S_{n-1}; S the inclusive fp64 scan of w. */
int64_t oracle_weighted_sample(const float* w, int64_t n, double theta)
{
    if (n <= 0) return -1;
    double* S = (double*)malloc((size_t)n * sizeof(double));
    double run = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        run += (double)w[i];
        S[i] = run;
    }
    const double t = theta * S[n - 1];
    int64_t pick = n - 1;
    for (int64_t i = 0; i < n; ++i)
        if (S[i] > t) {
            pick = i;
            break;
        }
    free(S);
    return pick;
}

/* R15: nucleus of mass >= p in descending order, inverse transform with u.
 * Writes the nucleus size to *kept (nullable). */
int64_t oracle_top_p_sample(const float* probs, int64_t n, double p, double u, int64_t* kept)
{
    if (n <= 0) return -1;
    float* q = (float*)malloc((size_t)n * sizeof(float));
    int32_t* order = (int32_t*)malloc((size_t)n * sizeof(int32_t));
    oracle_radix_sort(probs, n, ORACLE_F32, 1, q, order);  /* sort (P299) */
    double* C = (double*)malloc((size_t)n * sizeof(double));
    double run = 0.0;
    int64_t K = 0;  /* ranks 0..K-1 are kept */
    for (int64_t k = 0; k < n; ++k) {
        const double E = run;  /* exclusive scan of the sorted probabilities */
        run += (double)q[k];
        C[k] = run;
        if (k == 0 || E < p) K = k + 1;
    }
    const double t = u * C[K - 1];
    int64_t pick = K - 1;
    for (int64_t k = 0; k < K; ++k)
        if (C[k] > t) {
            pick = k;
            break;
        }
    const int64_t tok = order[pick];
    if (kept) *kept = K;
    free(q); free(order); free(C);
    return tok;
}

int oracle_ops_abi_version(void) { return 1; }

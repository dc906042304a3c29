/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, fp64 CPU reference for the one hot path this repo builds:
 * Hetis' head-granular decode Attention over a head-granular paged KV cache
 * (arXiv 2509.08309).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / `--impl reference` legs may load this library.  It shares no
 * code, header, table or helper with paper_2509_08309_b200/ (the CUDA path),
 * and neither side imports the other.
 *
 * Citations are PAPER.md line numbers with the
 * section / equation they fall in; "reading N" refers to the numbered list of
 * readings in DESIGN.md §3 (same numbering as SURVEY.md §8(c)).
 *
 *   oracle_decode_f64        Eq. 2b (§4.2) for every query head
 *                            of every request, placed at its global head index
 *                            (Eq. 2a Concat; reading 4).  K and V
 *                            are read through head-granular block tables: one
 *                            page = page_size tokens of ONE kv head (PAPER.md:539,
 *                            §6 "split cache blocks on the head dimension").
 *   oracle_decode_pairs_f64  the same value for a list of (seq, head) pairs
 *                            (used to sample outputs at full size).
 *   oracle_kv_append         head-granular store "via the combination of sequence
 *                            id, position within the sequence, and head id"
 *                            (§6).
 *   oracle_lse_merge_f64     merge of attention results over disjoint token
 *                            subsets by log-sum-exp weights.  The paper does not
 *                            state it (reading 12); it is the textbook identity
 *                            softmax over a union = weighted softmaxes.
 *
 * Pins (tests/test_oracle.py): mpmath brute force on tiny inputs, torch fp64
 * scaled_dot_product_attention, the closed forms L=1 / L=2 / uniform keys /
 * affine equivariance / peaked limit, page-permutation / head-partition /
 * token-permutation / GQA==expanded-MHA invariants, and a hand-worked golden
 * example (tests/golden/).
 *
 * Arithmetic: everything in double.  bf16 inputs are widened exactly
 * (bits << 16 reinterpreted as binary32, then to binary64); fp32 inputs are
 * widened exactly.  No blocking, fusion or reordering: tokens are summed in
 * ascending order t = 0 .. L-1, dimensions in ascending order k = 0 .. D-1.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_F32 0
#define ORACLE_BF16 1

#define ORACLE_OK 0
#define ORACLE_E_ARG (-1)      /* null pointer / bad shape                          */
#define ORACLE_E_EMPTY (-2)    /* seq_len < 1: softmax over the empty set (reading 10) */
#define ORACLE_E_PAGE (-3)     /* page id outside [0, num_pages)                    */
#define ORACLE_E_LEN (-4)      /* seq_len > max_pages * page_size                   */

/* Exact widening of one stored element to double. */
static double load_elem(const void *base, int dtype, int64_t idx) {
    if (dtype == ORACLE_BF16) {
        uint16_t b = ((const uint16_t *)base)[idx];
        uint32_t w = ((uint32_t)b) << 16;
        float f;
        memcpy(&f, &w, sizeof f);
        return (double)f;
    }
    return (double)((const float *)base)[idx];
}

typedef struct {
    int B, H, Hkv, D, P, dtype;
    const void *q, *k_pool, *v_pool;
    int64_t num_pages;
    const int32_t *block_table;
    int max_pages;
    const int32_t *seq_lens;
} problem;

/*
 * result_{j,h} = softmax(q_{j,h} . K_{j,g}^T / sqrt(d)) . V_{j,g}   (Eq. 2b)
 * with g = floor(h / r), r = H / Hkv (reading 5), d = head_dim (reading 1),
 * and the token-t row of K/V found at page bt[j][g][t / P], slot t mod P
 * (reading 11).  Writes D doubles to out.
 */
static int decode_one(const problem *pb, int j, int h, double *out, double *scores) {
    const int r = pb->H / pb->Hkv;
    const int g = h / r;
    const int L = pb->seq_lens[j];
    if (L < 1) return ORACLE_E_EMPTY;
    if (L > pb->max_pages * pb->P) return ORACLE_E_LEN;
    const int32_t *bt = pb->block_table + ((int64_t)j * pb->Hkv + g) * pb->max_pages;
    const int64_t q_off = ((int64_t)j * pb->H + h) * pb->D;
    const double inv_sqrt_d = 1.0 / sqrt((double)pb->D);

    /* s_t = (sum_k q_k K_t,k) / sqrt(d) */
    for (int t = 0; t < L; ++t) {
        const int32_t page = bt[t / pb->P];
        if (page < 0 || page >= pb->num_pages) return ORACLE_E_PAGE;
        const int64_t row = ((int64_t)page * pb->P + (t % pb->P)) * pb->D;
        double dot = 0.0;
        for (int k = 0; k < pb->D; ++k)
            dot += load_elem(pb->q, pb->dtype, q_off + k) * load_elem(pb->k_pool, pb->dtype, row + k);
        scores[t] = dot * inv_sqrt_d;
    }
    /* softmax with max subtraction (mathematically identical, reading 16) */
    double m = scores[0];
    for (int t = 1; t < L; ++t)
        if (scores[t] > m) m = scores[t];
    double Z = 0.0;
    for (int t = 0; t < L; ++t) {
        scores[t] = exp(scores[t] - m);
        Z += scores[t];
    }
    /* O = sum_t w_t V_t / Z */
    for (int k = 0; k < pb->D; ++k) out[k] = 0.0;
    for (int t = 0; t < L; ++t) {
        const int32_t page = bt[t / pb->P];
        const int64_t row = ((int64_t)page * pb->P + (t % pb->P)) * pb->D;
        for (int k = 0; k < pb->D; ++k)
            out[k] += scores[t] * load_elem(pb->v_pool, pb->dtype, row + k);
    }
    for (int k = 0; k < pb->D; ++k) out[k] /= Z;
    return ORACLE_OK;
}

static int check_problem(const problem *pb) {
    if (!pb->q || !pb->k_pool || !pb->v_pool || !pb->block_table || !pb->seq_lens) return ORACLE_E_ARG;
    if (pb->B < 0 || pb->H < 1 || pb->Hkv < 1 || pb->D < 1 || pb->P < 1 || pb->max_pages < 1) return ORACLE_E_ARG;
    if (pb->H % pb->Hkv != 0) return ORACLE_E_ARG;
    if (pb->dtype != ORACLE_F32 && pb->dtype != ORACLE_BF16) return ORACLE_E_ARG;
    return ORACLE_OK;
}

/* Largest seq_len among the pairs that will be evaluated (scratch sizing). */
static int max_len(const problem *pb) {
    int m = 1;
    for (int j = 0; j < pb->B; ++j)
        if (pb->seq_lens[j] > m) m = pb->seq_lens[j];
    return m;
}

/*
 * Evaluate n_pairs (seq, head) outputs; pairs[2i] = seq, pairs[2i+1] = global
 * query head.  out is [n_pairs][D].  nthreads <= 0 means "OpenMP default".
 * The per-output arithmetic is identical for any thread count (each output is
 * computed by one thread, in the fixed order above).
 */
int oracle_decode_pairs_f64(int B, int H, int Hkv, int D, int P, int dtype,
                            const void *q, const void *k_pool, const void *v_pool, int64_t num_pages,
                            const int32_t *block_table, int max_pages, const int32_t *seq_lens,
                            int64_t n_pairs, const int32_t *pairs, double *out, int nthreads) {
    problem pb = {B, H, Hkv, D, P, dtype, q, k_pool, v_pool, num_pages, block_table, max_pages, seq_lens};
    int st = check_problem(&pb);
    if (st != ORACLE_OK) return st;
    if (n_pairs > 0 && (!pairs || !out)) return ORACLE_E_ARG;
    for (int64_t i = 0; i < n_pairs; ++i)
        if (pairs[2 * i] < 0 || pairs[2 * i] >= B || pairs[2 * i + 1] < 0 || pairs[2 * i + 1] >= H) return ORACLE_E_ARG;
    const int Lmax = max_len(&pb);
    int err = ORACLE_OK;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel
    {
        double *scores = (double *)malloc(sizeof(double) * (size_t)Lmax);
        int local = scores ? ORACLE_OK : ORACLE_E_ARG;
#pragma omp for schedule(dynamic, 1)
        for (int64_t i = 0; i < n_pairs; ++i) {
            if (local != ORACLE_OK) continue;
            int s = decode_one(&pb, pairs[2 * i], pairs[2 * i + 1], out + i * D, scores);
            if (s != ORACLE_OK) local = s;
        }
#pragma omp critical
        {
            if (local != ORACLE_OK && err == ORACLE_OK) err = local;
        }
        free(scores);
    }
    return err;
}

/* Full output [B][H][D] at global head index (Eq. 2a Concat, reading 4). */
int oracle_decode_f64(int B, int H, int Hkv, int D, int P, int dtype,
                      const void *q, const void *k_pool, const void *v_pool, int64_t num_pages,
                      const int32_t *block_table, int max_pages, const int32_t *seq_lens,
                      double *out, int nthreads) {
    problem pb = {B, H, Hkv, D, P, dtype, q, k_pool, v_pool, num_pages, block_table, max_pages, seq_lens};
    int st = check_problem(&pb);
    if (st != ORACLE_OK) return st;
    if (!out) return ORACLE_E_ARG;
    const int Lmax = max_len(&pb);
    const int64_t n = (int64_t)B * H;
    int err = ORACLE_OK;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel
    {
        double *scores = (double *)malloc(sizeof(double) * (size_t)Lmax);
        int local = scores ? ORACLE_OK : ORACLE_E_ARG;
#pragma omp for schedule(dynamic, 1)
        for (int64_t i = 0; i < n; ++i) {
            if (local != ORACLE_OK) continue;
            int s = decode_one(&pb, (int)(i / H), (int)(i % H), out + i * D, scores);
            if (s != ORACLE_OK) local = s;
        }
#pragma omp critical
        {
            if (local != ORACLE_OK && err == ORACLE_OK) err = local;
        }
        free(scores);
    }
    return err;
}

/*
 * Head-granular store (§6): for each request j and each kv head
 * g, the new token's K/V row goes to position L_j - 1 (seq_lens are lengths
 * AFTER the append, reading 6): page bt[j][g][(L_j-1) / P], slot (L_j-1) mod P.
 * Pure byte copy of elem_bytes * D bytes per row; pools are
 * [num_pages][P][D], new rows are [B][Hkv][D].
 */
int oracle_kv_append(int B, int Hkv, int D, int P, int elem_bytes,
                     const void *k_new, const void *v_new, void *k_pool, void *v_pool, int64_t num_pages,
                     const int32_t *block_table, int max_pages, const int32_t *seq_lens) {
    if (!k_new || !v_new || !k_pool || !v_pool || !block_table || !seq_lens) return ORACLE_E_ARG;
    if (B < 0 || Hkv < 1 || D < 1 || P < 1 || max_pages < 1 || (elem_bytes != 2 && elem_bytes != 4)) return ORACLE_E_ARG;
    const size_t row_bytes = (size_t)D * (size_t)elem_bytes;
    for (int j = 0; j < B; ++j) {
        const int L = seq_lens[j];
        if (L < 1) return ORACLE_E_EMPTY;
        if (L > max_pages * P) return ORACLE_E_LEN;
        const int pos = L - 1;
        for (int g = 0; g < Hkv; ++g) {
            const int32_t page = block_table[((int64_t)j * Hkv + g) * max_pages + pos / P];
            if (page < 0 || page >= num_pages) return ORACLE_E_PAGE;
            const size_t dst = ((size_t)page * P + (size_t)(pos % P)) * row_bytes;
            const size_t src = ((size_t)j * Hkv + g) * row_bytes;
            memcpy((char *)k_pool + dst, (const char *)k_new + src, row_bytes);
            memcpy((char *)v_pool + dst, (const char *)v_new + src, row_bytes);
        }
    }
    return ORACLE_OK;
}

/*
 * Merge S partial attention results of one head over disjoint token subsets:
 * given o_s = softmax-weighted mean of V over subset s and
 * lse_s = log(sum_{t in s} exp(score_t)), the result over the union is
 *   lse = log(sum_s exp(lse_s)),  o = sum_s exp(lse_s - lse) * o_s.
 * (Not stated in the paper -- reading 12; this is the identity that makes any
 * token split exact.)  o_parts is [S][D], lse_parts is [S]; out is [D].
 */
int oracle_lse_merge_f64(int S, int D, const double *o_parts, const double *lse_parts, double *out, double *lse_out) {
    if (S < 1 || D < 1 || !o_parts || !lse_parts || !out) return ORACLE_E_ARG;
    double m = lse_parts[0];
    for (int s = 1; s < S; ++s)
        if (lse_parts[s] > m) m = lse_parts[s];
    double z = 0.0;
    for (int s = 0; s < S; ++s) z += exp(lse_parts[s] - m);
    const double lse = m + log(z);
    for (int k = 0; k < D; ++k) out[k] = 0.0;
    for (int s = 0; s < S; ++s) {
        const double w = exp(lse_parts[s] - lse);
        for (int k = 0; k < D; ++k) out[k] += w * o_parts[(int64_t)s * D + k];
    }
    if (lse_out) *lse_out = lse;
    return ORACLE_OK;
}

/* lse of one head over tokens [t0, t1) -- the natural-log normaliser used with
 * oracle_lse_merge_f64 in the split tests.  Same definitions as decode_one. */
int oracle_decode_range_f64(int B, int H, int Hkv, int D, int P, int dtype,
                            const void *q, const void *k_pool, const void *v_pool, int64_t num_pages,
                            const int32_t *block_table, int max_pages, const int32_t *seq_lens,
                            int j, int h, int t0, int t1, double *out, double *lse_out) {
    problem pb = {B, H, Hkv, D, P, dtype, q, k_pool, v_pool, num_pages, block_table, max_pages, seq_lens};
    int st = check_problem(&pb);
    if (st != ORACLE_OK) return st;
    if (j < 0 || j >= B || h < 0 || h >= H || !out || !lse_out) return ORACLE_E_ARG;
    if (t0 < 0 || t1 <= t0 || t1 > seq_lens[j]) return ORACLE_E_ARG;
    const int r = H / Hkv, g = h / r;
    const int32_t *bt = block_table + ((int64_t)j * Hkv + g) * max_pages;
    const int64_t q_off = ((int64_t)j * H + h) * D;
    const double inv_sqrt_d = 1.0 / sqrt((double)D);
    double *scores = (double *)malloc(sizeof(double) * (size_t)(t1 - t0));
    if (!scores) return ORACLE_E_ARG;
    for (int t = t0; t < t1; ++t) {
        const int32_t page = bt[t / P];
        if (page < 0 || page >= num_pages) {
            free(scores);
            return ORACLE_E_PAGE;
        }
        const int64_t row = ((int64_t)page * P + (t % P)) * D;
        double dot = 0.0;
        for (int k = 0; k < D; ++k) dot += load_elem(q, dtype, q_off + k) * load_elem(k_pool, dtype, row + k);
        scores[t - t0] = dot * inv_sqrt_d;
    }
    double m = scores[0];
    for (int t = 1; t < t1 - t0; ++t)
        if (scores[t] > m) m = scores[t];
    double Z = 0.0;
    for (int t = 0; t < t1 - t0; ++t) {
        scores[t] = exp(scores[t] - m);
        Z += scores[t];
    }
    for (int k = 0; k < D; ++k) out[k] = 0.0;
    for (int t = t0; t < t1; ++t) {
        const int64_t row = ((int64_t)bt[t / P] * P + (t % P)) * D;
        for (int k = 0; k < D; ++k) out[k] += scores[t - t0] * load_elem(v_pool, dtype, row + k);
    }
    for (int k = 0; k < D; ++k) out[k] /= Z;
    *lse_out = m + log(Z);
    free(scores);
    return ORACLE_OK;
}

/*
 * Head-granular KV migration (the Hauler, "only partial cache
 * transmission", :545): the cache of one (request, kv head) is the token rows
 * its block-table row lists.  For every entry e = (src_row, dst_row, n) and
 * every token t < n, the destination row's token t receives the source row's
 * token t:
 *   dst_pool[dst_bt[dst_row][t / P]][t mod P][:] = src_pool[src_bt[src_row][t / P]][t mod P][:]
 * for the K and the V pool.  Token-by-token byte copy (slots past n untouched).
 * entries: [num_entries][3] int32.
 */
int oracle_kv_migrate(int num_entries, const int32_t *entries, int D, int P, int elem_bytes,
                      const void *src_k, const void *src_v, int64_t src_pages, const int32_t *src_bt,
                      int src_max_pages, void *dst_k, void *dst_v, int64_t dst_pages, const int32_t *dst_bt,
                      int dst_max_pages) {
    if (num_entries < 0 || D < 1 || P < 1 || (elem_bytes != 2 && elem_bytes != 4)) return ORACLE_E_ARG;
    if (num_entries == 0) return ORACLE_OK;
    if (!entries || !src_k || !src_v || !src_bt || !dst_k || !dst_v || !dst_bt) return ORACLE_E_ARG;
    const size_t row_bytes = (size_t)D * (size_t)elem_bytes;
    for (int e = 0; e < num_entries; ++e) {
        const int src_row = entries[3 * e], dst_row = entries[3 * e + 1], n = entries[3 * e + 2];
        if (src_row < 0 || dst_row < 0 || n < 0) return ORACLE_E_ARG;
        if (n > src_max_pages * P || n > dst_max_pages * P) return ORACLE_E_LEN;
        for (int t = 0; t < n; ++t) {
            const int32_t sp = src_bt[(int64_t)src_row * src_max_pages + t / P];
            const int32_t dp = dst_bt[(int64_t)dst_row * dst_max_pages + t / P];
            if (sp < 0 || sp >= src_pages || dp < 0 || dp >= dst_pages) return ORACLE_E_PAGE;
            const size_t so = ((size_t)sp * P + (size_t)(t % P)) * row_bytes;
            const size_t d0 = ((size_t)dp * P + (size_t)(t % P)) * row_bytes;
            memcpy((char *)dst_k + d0, (const char *)src_k + so, row_bytes);
            memcpy((char *)dst_v + d0, (const char *)src_v + so, row_bytes);
        }
    }
    return ORACLE_OK;
}

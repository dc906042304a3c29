/*
 * c_decode.c -- the C ABI of libhetis.so used from plain C (no Python, no torch).
 *
 * One decode step of one layer on one device for a small GQA batch: plan,
 * workspace query, then the step as two kernels (attention with the kv_append
 * fused, then the split combine), results read back and checked against two
 * closed forms of Eq. 2b:
 *   request 0 has L = 1      -> O = the new token's V row, bit for bit;
 *   request 1 has all keys 0 -> softmax is uniform -> O = mean of V over its tokens.
 *
 *   gcc -O2 -std=c11 -Iinclude examples/c_decode.c -Lpaper_2509_08309_b200 -lhetis \
 *       -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_2509_08309_b200 -lm -o c_decode
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "hetis.h"

#define CHECK(x)                                                                                   \
    do {                                                                                           \
        hetis_status s_ = (x);                                                                     \
        if (s_ != HETIS_OK) {                                                                      \
            fprintf(stderr, "%s failed: %s (%s)\n", #x, hetis_status_str(s_), hetis_last_error()); \
            return 1;                                                                              \
        }                                                                                          \
    } while (0)
#define CUDA(x)                                                                     \
    do {                                                                            \
        cudaError_t e_ = (x);                                                       \
        if (e_ != cudaSuccess) {                                                    \
            fprintf(stderr, "%s failed: %s\n", #x, cudaGetErrorString(e_));         \
            return 1;                                                               \
        }                                                                           \
    } while (0)

/* bf16 <-> float on the host (round to nearest even) */
static uint16_t f2bf(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}
static float bf2f(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

int main(void) {
    enum { H = 16, HKV = 2, D = 128, P = 16, B = 2 };
    const int lens[B] = {1, 300};                 /* lengths AFTER this step's append */
    const int max_len = 300, max_pages = (max_len + P - 1) / P;
    hetis_shape shape = {H, HKV, D, P, HETIS_BF16, HETIS_BF16, HETIS_F32};

    /* plan: one device owns every head (Eq. 5: sum x = H) */
    int32_t x[1] = {H};
    hetis_plan *plan = NULL;
    CHECK(hetis_plan_create(&shape, 1, B, x, 0, &plan));

    /* pages: request j, kv head g uses pages [base, base + ceil(L/P)), identity layout */
    int num_pages = 0;
    int32_t bt[B][HKV][(300 + P - 1) / P];
    for (int j = 0; j < B; ++j)
        for (int g = 0; g < HKV; ++g)
            for (int k = 0; k < max_pages; ++k) bt[j][g][k] = k < (lens[j] + P - 1) / P ? num_pages++ : -1;

    /* host data: q and V random-ish; K of request 1 all zero (uniform softmax) */
    size_t pool_elems = (size_t)num_pages * P * D;
    uint16_t *hk = calloc(pool_elems, 2), *hv = calloc(pool_elems, 2);
    uint16_t *hq = malloc((size_t)B * H * D * 2), *hkn = malloc((size_t)B * HKV * D * 2),
             *hvn = malloc((size_t)B * HKV * D * 2);
    unsigned seed = 12345u;
    for (size_t i = 0; i < (size_t)B * H * D; ++i) hq[i] = f2bf((float)((seed = seed * 1103515245u + 12345u) % 2001) / 1000.f - 1.f);
    for (size_t i = 0; i < pool_elems; ++i) {
        hv[i] = f2bf((float)((seed = seed * 1103515245u + 12345u) % 2001) / 1000.f - 1.f);
        hk[i] = f2bf((float)((seed = seed * 1103515245u + 12345u) % 2001) / 1000.f - 1.f);
    }
    for (size_t i = 0; i < (size_t)B * HKV * D; ++i) {
        hkn[i] = f2bf((float)((seed = seed * 1103515245u + 12345u) % 2001) / 1000.f - 1.f);
        hvn[i] = f2bf((float)((seed = seed * 1103515245u + 12345u) % 2001) / 1000.f - 1.f);
    }
    for (int g = 0; g < HKV; ++g) {          /* request 1: every key (history and new) = 0 */
        for (int k = 0; k < (lens[1] + P - 1) / P; ++k) memset(hk + (size_t)bt[1][g][k] * P * D, 0, P * D * 2);
        memset(hkn + ((size_t)1 * HKV + g) * D, 0, D * 2);
    }

    /* device buffers (the caller owns all of them) */
    void *dq, *dk, *dv, *dkn, *dvn, *dbt, *dsl, *dout, *dws;
    CUDA(cudaMalloc(&dq, (size_t)B * H * D * 2));
    CUDA(cudaMalloc(&dk, pool_elems * 2));
    CUDA(cudaMalloc(&dv, pool_elems * 2));
    CUDA(cudaMalloc(&dkn, (size_t)B * HKV * D * 2));
    CUDA(cudaMalloc(&dvn, (size_t)B * HKV * D * 2));
    CUDA(cudaMalloc(&dbt, sizeof bt));
    CUDA(cudaMalloc(&dsl, sizeof lens));
    CUDA(cudaMalloc(&dout, (size_t)B * H * D * 4));
    CUDA(cudaMemcpy(dq, hq, (size_t)B * H * D * 2, cudaMemcpyHostToDevice));
    CUDA(cudaMemcpy(dk, hk, pool_elems * 2, cudaMemcpyHostToDevice));
    CUDA(cudaMemcpy(dv, hv, pool_elems * 2, cudaMemcpyHostToDevice));
    CUDA(cudaMemcpy(dkn, hkn, (size_t)B * HKV * D * 2, cudaMemcpyHostToDevice));
    CUDA(cudaMemcpy(dvn, hvn, (size_t)B * HKV * D * 2, cudaMemcpyHostToDevice));
    CUDA(cudaMemcpy(dbt, bt, sizeof bt, cudaMemcpyHostToDevice));
    CUDA(cudaMemcpy(dsl, lens, sizeof lens, cudaMemcpyHostToDevice));

    /* workspace: sized by the library, zero-filled once */
    size_t ws_bytes = 0;
    CHECK(hetis_attn_decode_workspace(&shape, B, H, max_len, &ws_bytes));
    CUDA(cudaMalloc(&dws, ws_bytes));
    CUDA(cudaMemset(dws, 0, ws_bytes));

    int32_t q_begin = 0, q_count = 0;
    CHECK(hetis_plan_heads(plan, 0, 0, &q_begin, &q_count));
    CHECK(hetis_attn_decode_append(&shape, B, q_begin, q_count, dq, dkn, dvn, dk, dv, num_pages, dbt, max_pages,
                                   dsl, max_len, dout, dws, ws_bytes, 0u, NULL));
    CUDA(cudaDeviceSynchronize());

    float *ho = malloc((size_t)B * H * D * 4);
    CUDA(cudaMemcpy(ho, dout, (size_t)B * H * D * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int h = 0; h < H; ++h) {
        const int g = h / (H / HKV);
        for (int k = 0; k < D; ++k) {
            /* request 0, L = 1: the new V row exactly */
            if (ho[((size_t)0 * H + h) * D + k] != bf2f(hvn[((size_t)0 * HKV + g) * D + k])) ++bad;
            /* request 1: uniform weights -> mean of V over its 300 tokens (299 history + the new row) */
            double mean = bf2f(hvn[((size_t)1 * HKV + g) * D + k]);
            for (int t = 0; t < lens[1] - 1; ++t) mean += bf2f(hv[((size_t)bt[1][g][t / P] * P + t % P) * D + k]);
            mean /= lens[1];
            if (fabs(ho[((size_t)1 * H + h) * D + k] - mean) > 2e-3) ++bad;
        }
    }
    hetis_plan_destroy(plan);
    printf("c example: %d mismatches, %llu library kernels launched\n", bad, (unsigned long long)hetis_launch_count());
    if (bad == 0) printf("c example ok\n");
    return bad != 0;
}

// combine_fold.cuh -- the split-KV merge arithmetic (a5), shared by the combine kernels
// (small_kernels.cu) and the merge fused into the per-warp attention kernel
// (attn_decode.cu), so every path produces the same bits for a (request, head) pair.
//
// o = sum_s 2^(lse_s - M) o_s / sum_s 2^(lse_s - M), M = max_s lse_s (lse in log2 units).
// A lane owns 4 dims of the row (d4); D/4 lanes cover it.  Splits are folded in chunks of
// kCombineChunk: the chunk's lse and o rows are loaded together (one memory round trip per
// chunk) and accumulated with an online max (rescale by 2^(M_old - M_new)).  The result of a
// pair depends on its split count ns only (hence on L_j only), never on the launch shape:
//   ns <= kNarrowSplits: s = 0 .. ns-1 in one fold;
//   ns >  kNarrowSplits: G = D/4-lane groups of a 128-thread block fold s = k, k + G, ... and
//                        the G states are merged in ascending k (merge_groups).
// Every multiply-add is an explicit _rn intrinsic: no fp-contraction decision of the compiler
// can differ between the call sites.  With one split, w = 2^0 = 1 and every other term is an
// exact zero, so o = o_0 bit for bit.
#pragma once

#include <cuda_bf16.h>
#include <stdint.h>

#include "device_utils.cuh"

namespace hetis {

constexpr int kCombineThreads = 128;
#ifndef HETIS_COMBINE_CHUNK
#define HETIS_COMBINE_CHUNK 8
#endif
constexpr int kCombineChunk = HETIS_COMBINE_CHUNK;
constexpr int kNarrowSplits = 16;

struct FoldState {
    float M, wsum;
    float4 acc;
};

__device__ __forceinline__ float4 scale4(float4 a, float s) {
    return make_float4(__fmul_rn(a.x, s), __fmul_rn(a.y, s), __fmul_rn(a.z, s), __fmul_rn(a.w, s));
}
__device__ __forceinline__ float4 fma4(float w, float4 v, float4 a) {
    return make_float4(__fmaf_rn(w, v.x, a.x), __fmaf_rn(w, v.y, a.y), __fmaf_rn(w, v.z, a.z),
                       __fmaf_rn(w, v.w, a.w));
}

// CG: read through L2 only (ld.global.cg) -- for partials written by other CTAs of the SAME
// launch (the fused merge); the combine kernels read a finished predecessor's output.
template <bool CG>
__device__ __forceinline__ float ld_f(const float *p) {
    return CG ? __ldcg(p) : *p;
}
template <bool CG>
__device__ __forceinline__ float4 ld_f4(const float *p) {
    return CG ? __ldcg(reinterpret_cast<const float4 *>(p)) : *reinterpret_cast<const float4 *>(p);
}

// fold splits s = first, first + step, ... < ns; load(s, l, v) fetches split s's log2-sum-exp and
// this lane's 4 dims of its partial row (from global memory, or from a shared-memory staging copy --
// the arithmetic below is the same code either way)
template <class Load>
__device__ __forceinline__ FoldState fold_splits_with(int first, int step, int ns, Load load) {
    constexpr int U = kCombineChunk;
    FoldState f{-INFINITY, 0.f, make_float4(0.f, 0.f, 0.f, 0.f)};
    for (int base = first; base < ns; base += step * U) {
        float l[U];
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int sp = base + u * step;
            if (sp < ns) {
                load(sp, l[u], v[u]);
            } else {
                l[u] = -INFINITY;
                v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        float mc = l[0];  // finite: split `base` exists
#pragma unroll
        for (int u = 1; u < U; ++u) mc = fmaxf(mc, l[u]);
        const float Mn = fmaxf(f.M, mc);
        const float alpha = dev::ex2(f.M - Mn);  // 0 on the first chunk (M = -inf)
        f.wsum = __fmul_rn(f.wsum, alpha);
        f.acc = scale4(f.acc, alpha);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const float w = dev::ex2(l[u] - Mn);  // 0 for the padding (l = -inf)
            f.wsum = __fadd_rn(f.wsum, w);
            f.acc = fma4(w, v[u], f.acc);
        }
        f.M = Mn;
    }
    return f;
}

// split s's partial row of row rr of kv head g, request split offset s0: ((s0 + s) * kv_heads + g) * r + rr
template <int D, bool CG = false>
__device__ __forceinline__ FoldState fold_splits(int first, int step, int ns, int s0, int kv_heads, int g, int r,
                                                 int rr, const float *part_lse, const float *part_o, int d4) {
    return fold_splits_with(first, step, ns, [&](int sp, float &l, float4 &v) {
        const size_t rw = ((size_t)(s0 + sp) * kv_heads + g) * r + rr;
        l = ld_f<CG>(part_lse + rw);
        v = ld_f4<CG>(part_o + rw * D + 4 * d4);
    });
}

// NR rows at once (rows rr0 .. rr0 + NR - 1 of the same pair, lane d4 of each): the loads of every
// row's chunk are issued together (one memory round trip for NR rows); each row's arithmetic is
// exactly fold_splits(0, 1, ns, ...) -- the narrow fold.
template <int D, bool CG, int NR>
__device__ __forceinline__ void fold_rows_narrow(int ns, int s0, int kv_heads, int g, int r, int rr0,
                                                 const float *part_lse, const float *part_o, int d4,
                                                 FoldState (&f)[NR]) {
    constexpr int U = kCombineChunk;
#pragma unroll
    for (int k = 0; k < NR; ++k) f[k] = FoldState{-INFINITY, 0.f, make_float4(0.f, 0.f, 0.f, 0.f)};
    for (int base = 0; base < ns; base += U) {
        float l[NR][U];
        float4 v[NR][U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int sp = base + u;
#pragma unroll
            for (int k = 0; k < NR; ++k) {
                if (sp < ns) {
                    const size_t rw = ((size_t)(s0 + sp) * kv_heads + g) * r + rr0 + k;
                    l[k][u] = ld_f<CG>(part_lse + rw);
                    v[k][u] = ld_f4<CG>(part_o + rw * D + 4 * d4);
                } else {
                    l[k][u] = -INFINITY;
                    v[k][u] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            float mc = l[k][0];
#pragma unroll
            for (int u = 1; u < U; ++u) mc = fmaxf(mc, l[k][u]);
            const float Mn = fmaxf(f[k].M, mc);
            const float alpha = dev::ex2(f[k].M - Mn);
            f[k].wsum = __fmul_rn(f[k].wsum, alpha);
            f[k].acc = scale4(f[k].acc, alpha);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const float w = dev::ex2(l[k][u] - Mn);
                f[k].wsum = __fadd_rn(f[k].wsum, w);
                f[k].acc = fma4(w, v[k][u], f[k].acc);
            }
            f[k].M = Mn;
        }
    }
}

// merge of the G group states of a wide fold, in ascending group order (every group holds >= 1 split)
template <int G>
__device__ __forceinline__ FoldState merge_groups(const float (&m)[G], const float (&w)[G], const float4 (&a)[G]) {
    float Mall = m[0];
#pragma unroll
    for (int k = 1; k < G; ++k) Mall = fmaxf(Mall, m[k]);
    FoldState t;
    const float f0 = dev::ex2(m[0] - Mall);
    t.acc = scale4(a[0], f0);
    t.wsum = __fmul_rn(f0, w[0]);
#pragma unroll
    for (int k = 1; k < G; ++k) {
        const float fk = dev::ex2(m[k] - Mall);
        t.acc = fma4(fk, a[k], t.acc);
        t.wsum = __fmaf_rn(fk, w[k], t.wsum);
    }
    t.M = Mall;
    return t;
}

__device__ __forceinline__ float4 finish(const FoldState &f, float *lse2_out) {
    *lse2_out = f.M + log2f(f.wsum);
    return make_float4(__fdiv_rn(f.acc.x, f.wsum), __fdiv_rn(f.acc.y, f.wsum), __fdiv_rn(f.acc.z, f.wsum),
                       __fdiv_rn(f.acc.w, f.wsum));
}

// The whole merge of one row by ONE lane group (d4 = its lane index in the row): the narrow fold,
// or the wide one with its G group states computed one after the other -- the same states and
// the same merge as the G groups of a wide combine block.  ns >= 1.
template <int D, bool CG>
__device__ __forceinline__ float4 fold_row(int ns, int s0, int kv_heads, int g, int r, int rr, const float *part_lse,
                                           const float *part_o, int d4, float *lse2_out) {
    constexpr int G = kCombineThreads / (D / 4);
    if (ns <= kNarrowSplits)
        return finish(fold_splits<D, CG>(0, 1, ns, s0, kv_heads, g, r, rr, part_lse, part_o, d4), lse2_out);
    float m[G], w[G];
    float4 a[G];
#pragma unroll
    for (int k = 0; k < G; ++k) {
        const FoldState f = fold_splits<D, CG>(k, G, ns, s0, kv_heads, g, r, rr, part_lse, part_o, d4);
        m[k] = f.M;
        w[k] = f.wsum;
        a[k] = f.acc;
    }
    return finish(merge_groups<G>(m, w, a), lse2_out);
}

template <int OUT_BF16>
__device__ __forceinline__ void store_row4(void *o, size_t idx, float4 acc) {
    if (OUT_BF16) {
        uint2 pk;
        pk.x = dev::pack_bf16x2(acc.x, acc.y);
        pk.y = dev::pack_bf16x2(acc.z, acc.w);
        *reinterpret_cast<uint2 *>(static_cast<__nv_bfloat16 *>(o) + idx) = pk;
    } else {
        *reinterpret_cast<float4 *>(static_cast<float *>(o) + idx) = acc;
    }
}

}  // namespace hetis

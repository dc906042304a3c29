// seq_split.cu -- sequence-wise split of decode attention across devices (row f3).
//
// The paper's rejected alternative to head-wise dispatch (PAPER.md:292-304,
// :356-358 `fig:head_wise_advantage`): every device attends ALL heads over a
// subset of each request's tokens, and the results are aggregated with the
// global softmax attributes (the per-head log-sum-exp).  Layout (DESIGN.md
// reading f3): page k of every (request, kv head) lives on device k mod N
// ("page striping"), so the new token always lands on the device holding the
// last page and no page ever moves as the request grows.
//
//   seq_split_lens_kernel : global L_j -> this device's token count l_j and the
//                           length to append with (l_j on the owner of the
//                           last page, 0 elsewhere).  Integer, bit-exact.
//   seq_merge_kernel      : O = sum_p e^(lse_p - lse) o_p over the devices' partial
//                           results in ascending device order (the union-of-
//                           subsets identity oracle_lse_merge_f64 states).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "device_utils.cuh"
#include "hetis_internal.h"

namespace hetis {

namespace {

__global__ void seq_split_lens_kernel(int num_ranks, int rank, int page_size, int num_seqs, const int32_t *seq_lens,
                                      int32_t *local_lens, int32_t *append_lens) {
    // no early release: these lengths are the seq_lens the attention kernel reads in its
    // prologue before it waits, so dependents may only start once this kernel is complete
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= num_seqs) return;
    const int L = seq_lens[j];
    const int np = (L + page_size - 1) / page_size;  // pages 0 .. np-1; page k on device k mod N
    const int mine = np > rank ? (np - 1 - rank) / num_ranks + 1 : 0;
    const bool owns_last = np > 0 && (np - 1) % num_ranks == rank;
    // every page is full except the last one, which holds L - (np - 1) P tokens
    const int l = mine * page_size - (owns_last ? np * page_size - L : 0);
    local_lens[j] = l;
    if (append_lens) append_lens[j] = owns_last ? l : 0;
}

// One group of D/4 threads per (request, head); each thread owns 4 dims.
// lse_p in natural log; -inf marks a device that holds none of the request.
template <int D, int OUT_BF16>
__global__ void seq_merge_kernel(int num_parts, int num_seqs, int q_heads, const float *o_parts, int64_t o_part_stride,
                                 const float *lse_parts, int64_t lse_part_stride, void *o, int64_t o_seq_stride) {
    dev::pdl_wait_then_release();
    constexpr int TPH = D / 4;
    const int heads_per_block = blockDim.x / TPH;
    const int hl = threadIdx.x / TPH, d4 = threadIdx.x % TPH;
    const int64_t flat = (int64_t)blockIdx.x * heads_per_block + hl;
    if (flat >= (int64_t)num_seqs * q_heads) return;
    const int j = (int)(flat / q_heads), h = (int)(flat - (int64_t)j * q_heads);
    constexpr float kLog2e = 1.4426950408889634f;
    float M = -INFINITY;
    for (int p = 0; p < num_parts; ++p) M = fmaxf(M, lse_parts[p * lse_part_stride + flat] * kLog2e);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (M != -INFINITY) {
        float wsum = 0.f;
        for (int p = 0; p < num_parts; ++p) {
            const float x = lse_parts[p * lse_part_stride + flat] * kLog2e;
            if (x == -INFINITY) continue;  // that device holds no token of request j (its o_p is 0)
            const float w = dev::ex2(x - M);  // the largest part gets 2^0 = 1 exactly
            const float4 v = reinterpret_cast<const float4 *>(o_parts + p * o_part_stride + flat * D)[d4];
            wsum += w;
            acc.x = fmaf(w, v.x, acc.x);
            acc.y = fmaf(w, v.y, acc.y);
            acc.z = fmaf(w, v.z, acc.z);
            acc.w = fmaf(w, v.w, acc.w);
        }
        acc.x = __fdiv_rn(acc.x, wsum);
        acc.y = __fdiv_rn(acc.y, wsum);
        acc.z = __fdiv_rn(acc.z, wsum);
        acc.w = __fdiv_rn(acc.w, wsum);
    }
    const size_t idx = (size_t)j * o_seq_stride + (size_t)h * D + 4 * d4;
    if (OUT_BF16) {
        uint2 pk;
        pk.x = dev::pack_bf16x2(acc.x, acc.y);
        pk.y = dev::pack_bf16x2(acc.z, acc.w);
        *reinterpret_cast<uint2 *>(static_cast<__nv_bfloat16 *>(o) + idx) = pk;
    } else {
        *reinterpret_cast<float4 *>(static_cast<float *>(o) + idx) = acc;
    }
}

}  // namespace

cudaError_t launch_seq_split_lens(int num_ranks, int rank, int page_size, int num_seqs, const int32_t *seq_lens,
                                  int32_t *local_lens, int32_t *append_lens, cudaStream_t s) {
    if (num_seqs == 0) return cudaSuccess;
    const int threads = 128;
    return launch_pdl(seq_split_lens_kernel, dim3((num_seqs + threads - 1) / threads), dim3(threads), 0, s,
                      num_ranks, rank, page_size, num_seqs, seq_lens, local_lens, append_lens);
}

cudaError_t launch_seq_merge(int num_parts, int num_seqs, int q_heads, int head_dim, const float *o_parts,
                             int64_t o_part_stride, const float *lse_parts, int64_t lse_part_stride, void *o,
                             int o_dtype, int64_t o_seq_stride, cudaStream_t s) {
    const int64_t heads = (int64_t)num_seqs * q_heads;
    if (heads == 0) return cudaSuccess;
    const int threads = 128;
    const int hpb = threads / (head_dim / 4);
    const int64_t blocks = (heads + hpb - 1) / hpb;
    auto kern = head_dim == 128 ? (o_dtype == HETIS_BF16 ? seq_merge_kernel<128, 1> : seq_merge_kernel<128, 0>)
                                : (o_dtype == HETIS_BF16 ? seq_merge_kernel<64, 1> : seq_merge_kernel<64, 0>);
    return launch_pdl(kern, dim3((unsigned)blocks), dim3(threads), 0, s, num_parts, num_seqs, q_heads, o_parts,
                      o_part_stride, lse_parts, lse_part_stride, o, o_seq_stride);
}

}  // namespace hetis

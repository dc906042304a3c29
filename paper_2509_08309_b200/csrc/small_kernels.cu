// small_kernels.cu -- the non-attention kernels of the step:
//   kv_append    head-granular store of the new token's K/V rows (a3)
//   combine      LSE merge of the split-KV partials in ascending split order (a5)
//   head slice / place: strided [B][H][d] <-> dense [B][x][d] shard copies around
//                the NCCL scatter / gather (a2, a6; Eq. 2a Concat)
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <set>
#include <utility>

#include "combine_fold.cuh"
#include "peer_sync.cuh"
#include "device_utils.cuh"
#include "hetis_internal.h"

namespace hetis {

namespace {
std::atomic<uint64_t> g_launches{0};

// ---------------------------------------------------------------- kv append
// One warp per (request j, kv head g); lanes move 16-byte chunks of the K and V rows.
__global__ void kv_append_kernel(int num_seqs, int kv_heads, int row_bytes, int page_size, const uint8_t *k_new,
                                 const uint8_t *v_new, uint8_t *k_pool, uint8_t *v_pool, const int32_t *block_table,
                                 int max_pages, const int32_t *seq_lens) {
    // release first: the attention kernel that follows may run its prologue (q, seq_lens and
    // block tables only -- no library kernel that releases early writes those) while this
    // kernel waits for its predecessor; its page copies wait for this kernel to complete
    dev::pdl_release_then_wait();
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= num_seqs * kv_heads) return;
    const int j = warp / kv_heads, g = warp - j * kv_heads;
    const int pos = seq_lens[j] - 1;
    if (pos < 0) return;  // seq_lens[j] == 0: nothing appended for request j on this device (sequence split)
    const int32_t page = block_table[((size_t)j * kv_heads + g) * max_pages + pos / page_size];
    const size_t dst = ((size_t)page * page_size + (size_t)(pos % page_size)) * row_bytes;
    const size_t src = (size_t)warp * row_bytes;
    for (int c = lane * 16; c < row_bytes; c += 32 * 16) {
        *reinterpret_cast<uint4 *>(k_pool + dst + c) = *reinterpret_cast<const uint4 *>(k_new + src + c);
        *reinterpret_cast<uint4 *>(v_pool + dst + c) = *reinterpret_cast<const uint4 *>(v_new + src + c);
    }
}

// ---------------------------------------------------------------- combine
// The merge arithmetic lives in combine_fold.cuh (shared with the merge fused into the per-warp
// attention kernel).  Launch shapes: when every request of the batch has <= kNarrowSplits splits,
// a block serves G pairs (one group each: few blocks, one round trip per pair); otherwise a block
// serves one pair and its G groups fold it together.
#ifndef HETIS_COMBINE_DISCARD
#define HETIS_COMBINE_DISCARD 0
#endif

// Narrow pair: folded by ONE group (the calling group); no block barrier.
template <int D>
__device__ __forceinline__ float4 combine_narrow(int j, int h, int q_heads, int r, const int32_t *split_off,
                                                 const float *part_lse, const float *part_o, int d4,
                                                 float *lse2_out, bool sole_reader = true) {
    const int kv_heads = q_heads / r, g = h / r, rr = h - g * r;
    const int s0 = split_off[j], ns = split_off[j + 1] - s0;
    if (ns == 0) {  // no tokens (a device holding none of request j under a sequence split): o = 0, lse = -inf
        *lse2_out = -INFINITY;
        return make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const FoldState f = fold_splits<D>(0, 1, ns, s0, kv_heads, g, r, rr, part_lse, part_o, d4);
#if HETIS_COMBINE_DISCARD
    // the partial rows are dead once folded: drop their (dirty) L2 lines instead of writing them back
    constexpr int TPH = D / 4, LINES = D * 4 / 128;
    const unsigned lane = threadIdx.x & 31;
    const unsigned gmask = (TPH == 32 ? 0xffffffffu : ((1u << TPH) - 1u) << (lane & ~(unsigned)(TPH - 1)));
    __syncwarp(gmask);
    for (int i = sole_reader ? d4 : ns * LINES; i < ns * LINES; i += TPH) {
        const int sp = i / LINES, ln = i % LINES;
        const float *line = part_o + (((size_t)(s0 + sp) * kv_heads + g) * r + rr) * D + ln * 32;
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(line) : "memory");
    }
#endif
    return finish(f, lse2_out);
}

// Wide launch: the whole 128-thread block serves one pair.  Result valid in group 0.
template <int D>
__device__ __forceinline__ float4 combine_wide(int j, int h, int q_heads, int r, const int32_t *split_off,
                                               const float *part_lse, const float *part_o, float *lse2_out) {
    constexpr int TPH = D / 4, G = kCombineThreads / TPH;
    __shared__ float4 s_acc[G][TPH];
    __shared__ float s_m[G], s_w[G];
    const int tid = threadIdx.x, grp = tid / TPH, d4 = tid % TPH;
    const int kv_heads = q_heads / r, g = h / r, rr = h - g * r;
    const int s0 = split_off[j], ns = split_off[j + 1] - s0;
    if (ns <= kNarrowSplits)  // block-uniform; every group folds the same pair, so none may discard
        return combine_narrow<D>(j, h, q_heads, r, split_off, part_lse, part_o, d4, lse2_out, false);
    const FoldState f = fold_splits<D>(grp, G, ns, s0, kv_heads, g, r, rr, part_lse, part_o, d4);
    s_acc[grp][d4] = f.acc;
    if (d4 == 0) {
        s_m[grp] = f.M;
        s_w[grp] = f.wsum;
    }
    __syncthreads();
    float m[G], w[G];
    float4 a[G];
#pragma unroll
    for (int k = 0; k < G; ++k) {
        m[k] = s_m[k];
        w[k] = s_w[k];
        a[k] = s_acc[k][d4];
    }
    return finish(merge_groups<G>(m, w, a), lse2_out);
}

// lse (optional, natural log, [num_seqs][q_heads]): ln sum_t exp(q.k_t / sqrt(d)) of
// the head over the tokens this launch saw -- the input of the cross-device merge
// of a sequence split (seq_split.cu).
#ifndef HETIS_COMBINE_MIN_BLOCKS
#define HETIS_COMBINE_MIN_BLOCKS 1
#endif
#ifndef HETIS_COMBINE_STAGED
#define HETIS_COMBINE_STAGED 1
#endif
template <int D, int OUT_BF16, bool WIDE>
__global__ void __launch_bounds__(kCombineThreads, HETIS_COMBINE_MIN_BLOCKS) combine_kernel(int num_seqs, int q_heads, int r,
                                                                  const int32_t *seq_lens, const int32_t *split_off,
                                                                  const float *part_lse, const float *part_o, void *o,
                                                                  int64_t o_seq_stride, float *lse,
                                                                  const int32_t *units) {
    dev::pdl_release_then_wait();
    constexpr int TPH = D / 4, G = kCombineThreads / TPH;
    const int grp = threadIdx.x / TPH, d4 = threadIdx.x % TPH;
    const int64_t flat = WIDE ? (int64_t)blockIdx.x : (int64_t)blockIdx.x * G + grp;
    if (flat >= (int64_t)num_seqs * q_heads) return;  // narrow launches only (wide grids are exact)
    const int j = (int)(flat / q_heads), h = (int)(flat - (int64_t)j * q_heads);
    float lse2;
    const float4 acc = WIDE ? combine_wide<D>(j, h, q_heads, r, split_off, part_lse, part_o, &lse2)
                            : combine_narrow<D>(j, h, q_heads, r, split_off, part_lse, part_o, d4, &lse2);
    if (WIDE && grp != 0) return;
    // units (per-request plans): launch row j is (request units[2j], global kv head units[2j+1]) and
    // h < r its query head within the group -> row units[2j] of o, global head units[2j+1] * r + h
    const size_t orow = units != nullptr ? (size_t)units[2 * j] * o_seq_stride + ((size_t)units[2 * j + 1] * r + h) * D
                                         : (size_t)j * o_seq_stride + (size_t)h * D;
    store_row4<OUT_BF16>(o, orow + 4 * d4, acc);
    if (lse != nullptr && d4 == 0) lse[flat] = lse2 * 0.69314718055994531f;  // log2 -> natural log
}

// ---------------------------------------------------------------- exchanges over peer memory
// (system-scope epoch helpers: peer_sync.cuh)

// Combine fused with the all-gather over peer memory: each merged O row is
// stored straight into every target rank's o_full at its GLOBAL head index
// (Eq. 2a Concat), after that rank has acknowledged it consumed the previous
// step's o_full; then the last block publishes the epoch into every target's
// state slot kStOut + rank with a system-scope release store.
template <int D, int OUT_BF16, bool WIDE>
__global__ void __launch_bounds__(kCombineThreads) combine_peers_kernel(int num_seqs, int q_heads, int r,
                                                                        const int32_t *split_off,
                                                                        const float *part_lse, const float *part_o,
                                                                        PeerGroupDev g) {
    dev::pdl_wait_then_release();
    const int64_t e = current_epoch(g);
    constexpr int TPH = D / 4, G = kCombineThreads / TPH;
    const int grp = threadIdx.x / TPH, d4 = threadIdx.x % TPH;
    // rank p may still read the previous step's o_full until it acknowledges (its scatter_pull of this step)
    if (threadIdx.x < g.n && peer_is_target(g, threadIdx.x)) spin_until_geq(g.state[g.rank] + kStAck + threadIdx.x, e - 1);
    __syncthreads();
    // one row per group (narrow) or per block (wide); the grid-stride loop only matters for huge launches
    const int64_t total = (int64_t)num_seqs * q_heads;
    const int64_t first = WIDE ? (int64_t)blockIdx.x : (int64_t)blockIdx.x * G + grp;
    const int64_t stride = WIDE ? (int64_t)gridDim.x : (int64_t)gridDim.x * G;
    for (int64_t flat = first; WIDE ? flat < total : true; flat += stride) {
        if (!WIDE && flat >= total) break;
        const int j = (int)(flat / q_heads);
        const int h = (int)(flat - (int64_t)j * q_heads);
        float lse2;
        const float4 acc = WIDE ? combine_wide<D>(j, h, q_heads, r, split_off, part_lse, part_o, &lse2)
                                : combine_narrow<D>(j, h, q_heads, r, split_off, part_lse, part_o, d4, &lse2);
        if (!WIDE || grp == 0) {
            const size_t idx = (size_t)j * g.o_seq_stride + (size_t)(g.head0 + h) * D + 4 * d4;
            for (int p = 0; p < g.n; ++p)
                if (peer_is_target(g, p)) store_row4<OUT_BF16>(g.o[p], idx, acc);
        }
        if (WIDE) __syncthreads();  // combine_wide's shared state is reused by the next row
    }
    // no per-block completion protocol: hetis_peer_wait, the next kernel on this rank's stream, publishes
    // the epoch after this grid has completed (one system-scope fence per step instead of one per block)
}

// The step's last kernel.  Every rank first publishes that its rows of this
// epoch are in every target's o_full: the kernel that stored them (the combine,
// or the attention kernel with the merge fused) has completed before
// griddepcontrol.wait returns, so its stores happen-before this thread's
// system-scope fence, which orders them before the release stores of the epoch
// into the targets' kStOut slots.  A target rank then waits (acquire, bounded)
// until every rank has published, and every rank records the step as completed
// (the next step's kernels derive their epoch from it).
__global__ void peer_wait_kernel(PeerGroupDev g) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL launch: the combine before it has completed
    const int64_t e = current_epoch(g);
    if (threadIdx.x == 0) {
        peer_publish_fence();
        for (int p = 0; p < g.n; ++p)
            if (peer_is_target(g, p)) st_release_sys(g.state[p] + kStOut + g.rank, e);
    }
    if ((int)threadIdx.x < g.n && peer_is_target(g, g.rank)) spin_until_geq(g.state[g.rank] + kStOut + threadIdx.x, e);
    __syncthreads();
    if (threadIdx.x == 0) g.state[g.rank][kStStep] = e;
}

// ---------------------------------------------------------------- table validation (debug)
// Counts contract violations of the device-side data the decode kernels trust without
// checking (include/hetis.h): 1 <= seq_lens[j] <= max_pages * P, and every page id a
// kernel will read (pages 0 .. ceil(L_j / P) - 1 of each (request, kv head)) in [0, num_pages).
__global__ void check_tables_kernel(int num_seqs, int kv_heads, int page_size, int64_t num_pages,
                                    const int32_t *block_table, int max_pages, const int32_t *seq_lens,
                                    int32_t *violations) {
    const int64_t total = (int64_t)num_seqs * kv_heads * max_pages;
    int bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(i % max_pages);
        const int64_t row = i / max_pages;
        const int j = (int)(row / kv_heads);
        const int L = seq_lens[j];
        if (k == 0 && row % kv_heads == 0 && (L < 1 || (int64_t)L > (int64_t)max_pages * page_size)) ++bad;
        const int np = L < 1 ? 0 : (L + page_size - 1) / page_size;
        if (k < np) {
            const int32_t pid = block_table[i];
            if (pid < 0 || (int64_t)pid >= num_pages) ++bad;
        }
    }
    if (bad) atomicAdd(violations, bad);
}

// ---------------------------------------------------------------- scatter over peer memory
// Pull this rank's shard of the step's inputs straight from the root's buffers
// (mapped over NVLink).  Block 0 first publishes, system-wide: on the root, the
// epoch into every rank's kStIn (everything before this kernel on the root's
// stream -- the writes of q_full, k_new_full, v_new_full -- is visible); on
// every rank, its acknowledgement (kStAck + rank = e - 1: everything before this
// kernel on its stream, including the consumer of the previous step's o_full,
// has completed).  Every block's thread 0 then waits (acquire, bounded) for the
// root's epoch and the block copies 16-byte chunks of
//   q      [B][H][d]     heads [q0, q0 + nq)   -> q_shard [B][nq][d]
//   k, v   [B][Hkv][d]   heads [k0, k0 + nk)   -> k/v_shard [B][nk][d]
__global__ void scatter_pull_kernel(PeerGroupDev g, int num_seqs, int H, int Hkv, int q0, int nq, int k0, int nk,
                                    int qrow, int kvrow, uint8_t *q_dst, uint8_t *k_dst, uint8_t *v_dst) {
    // PDL launch: wait for the previous step's peer_wait (which wrote the step counter), then let the
    // attention kernel launch at once -- its prologue overlaps this copy; it reads the shards only
    // after its own griddepcontrol.wait, i.e. after this kernel has completed.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int64_t e = current_epoch(g);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        peer_publish_fence();
        for (int p = 0; p < g.n; ++p) {
            st_release_sys(g.state[p] + kStAck + g.rank, e - 1);
            if (g.rank == g.root) st_release_sys(g.state[p] + kStIn, e);
        }
    }
    // the Primary's own inputs were written before griddepcontrol.wait returned: it has nothing to wait for
    if (threadIdx.x == 0 && g.rank != g.root) spin_until_geq(g.state[g.rank] + kStIn, e);
    __syncthreads();
    const int qc = qrow / 16, kc = kvrow / 16;
    const int64_t nq_chunks = (int64_t)num_seqs * nq * qc, nk_chunks = (int64_t)num_seqs * nk * kc;
    const int64_t total = nq_chunks + 2 * nk_chunks;
    auto addr = [&](int64_t i, const uint8_t *&src, uint8_t *&dst) {
        if (i < nq_chunks) {
            const int c = (int)(i % qc);
            const int64_t row = i / qc;
            const int h = (int)(row % nq), j = (int)(row / nq);
            src = g.q_root + ((size_t)j * H + q0 + h) * qrow + 16 * c;
            dst = q_dst + ((size_t)j * nq + h) * qrow + 16 * c;
        } else {
            const int64_t ii = (i - nq_chunks) % nk_chunks;
            const bool is_v = (i - nq_chunks) >= nk_chunks;
            const int c = (int)(ii % kc);
            const int64_t row = ii / kc;
            const int h = (int)(row % nk), j = (int)(row / nk);
            src = (is_v ? g.v_root : g.k_root) + ((size_t)j * Hkv + k0 + h) * kvrow + 16 * c;
            dst = (is_v ? v_dst : k_dst) + ((size_t)j * nk + h) * kvrow + 16 * c;
        }
    };
    // the root's epoch was acquired above (thread 0, then the barrier): plain L2 loads (.cg, never a stale L1
    // line of the previous step), four 16-byte chunks in flight per thread
    constexpr int U = 4;
    const int64_t step = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < total; i0 += U * step) {
        uint4 v[U];
        uint8_t *dst[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + u * step;
            dst[u] = nullptr;
            if (i < total) {
                const uint8_t *src;
                addr(i, src, dst[u]);
                v[u] = __ldcg(reinterpret_cast<const uint4 *>(src));
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (dst[u] != nullptr) *reinterpret_cast<uint4 *>(dst[u]) = v[u];
    }
}

// ---------------------------------------------------------------- shard copies
// Strided [B][H][d] <-> dense [B][x][d] head copies around the NCCL scatter /
// gather, every rank's (and tensor's) segment in one launch.
// Batched version: chunk i belongs to the segment whose prefix range holds it
// (linear search: at most 3 N segments).
__global__ void head_copies_kernel(const CopySegs c) {
    const int64_t total = c.start[c.count];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int k = 0;
        while (i >= c.start[k + 1]) ++k;
        const CopySeg &g = c.seg[k];
        const int chunks = g.row_bytes / 16;
        const int64_t li = i - c.start[k];
        const int ch = (int)(li % chunks);
        const int64_t rowi = li / chunks;
        const int hh = (int)(rowi % g.n);
        const int j = (int)(rowi / g.n);
        const uint4 v =
            *reinterpret_cast<const uint4 *>(g.src + (((size_t)j * g.src_heads + g.hs + hh) * g.row_bytes) + 16 * ch);
        *reinterpret_cast<uint4 *>(g.dst + (((size_t)j * g.dst_heads + g.hd + hh) * g.row_bytes) + 16 * ch) = v;
    }
}

}  // namespace

cudaError_t launch_head_copies(CopySegs &c, cudaStream_t s) {
    c.start[0] = 0;
    for (int k = 0; k < c.count; ++k)
        c.start[k + 1] = c.start[k] + (int64_t)c.num_seqs * c.seg[k].n * (c.seg[k].row_bytes / 16);
    const int64_t total = c.start[c.count];
    if (total == 0) return cudaSuccess;
    const int threads = 256;
    int64_t blocks = (total + threads - 1) / threads;
    if (blocks > 4 * num_sms()) blocks = 4 * num_sms();
    head_copies_kernel<<<(unsigned)blocks, threads, 0, s>>>(c);
    note_launch();
    return cudaGetLastError();
}

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void prefer_max_smem_once(const void *kern) {
    static std::mutex mu;
    static std::set<std::pair<int, const void *>> seen;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    if (seen.insert({dev, kern}).second)
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}
uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

int num_sms() {
    static std::atomic<int> cache[64];  // per device; 0 = not queried yet
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if ((n = cache[dev & 63].load(std::memory_order_relaxed)) > 0) return n;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) return 148;
    cache[dev & 63].store(n, std::memory_order_relaxed);
    return n;
}

cudaError_t launch_kv_append(int num_seqs, int kv_heads, int head_dim, int page_size, int elem_bytes,
                             const void *k_new, const void *v_new, void *k_pool, void *v_pool,
                             const int32_t *block_table, int max_pages, const int32_t *seq_lens, cudaStream_t s) {
    const int rows = num_seqs * kv_heads;
    if (rows == 0) return cudaSuccess;
    const int threads = 256;
    const int blocks = (rows * 32 + threads - 1) / threads;
    return launch_pdl(kv_append_kernel, dim3(blocks), dim3(threads), 0, s, num_seqs, kv_heads, head_dim * elem_bytes,
                      page_size, static_cast<const uint8_t *>(k_new), static_cast<const uint8_t *>(v_new),
                      static_cast<uint8_t *>(k_pool), static_cast<uint8_t *>(v_pool), block_table, max_pages,
                      seq_lens);
}

// Narrow combine with the partials staged in shared memory: lane 0 of a warp issues one bulk copy
// (cp.async.bulk, completion on an mbarrier) per split row of the warp's rows, the row's lanes < ns
// copy the split lse values, and the fold reads shared memory.  No register staging, so ~4 KiB of
// loads per row are in flight with ~40 registers per thread: c3's 8192 rows fit in one wave (the
// register-staged kernel needs 72 registers per thread and two waves).  Same fold code, same order:
// bit-identical to combine_kernel.
constexpr int kStagedWarps = 4;
template <int D, int OUT_BF16>
__global__ void __launch_bounds__(32 * kStagedWarps) combine_staged_kernel(
    int num_seqs, int q_heads, int r, int ns_max, const int32_t *split_off, const float *part_lse,
    const float *part_o, void *o, int64_t o_seq_stride, float *lse, const int32_t *units) {
    constexpr int TPH = D / 4, RPW = 32 / TPH;  // lanes per row, rows per warp
    extern __shared__ __align__(128) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, sub = lane / TPH, d4 = lane % TPH;
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
    float *stage = reinterpret_cast<float *>(smem + 128) + (size_t)warp * RPW * ns_max * (D + 4);
    float *rowbuf = stage + (size_t)sub * ns_max * (D + 4);  // [ns_max][D] partial rows, then [ns_max] lse
    float *lsebuf = rowbuf + (size_t)ns_max * D;
    if (threadIdx.x < kStagedWarps) dev::mbar_init(&bar[threadIdx.x], 1);
    dev::fence_barrier_init();
    __syncthreads();
    dev::pdl_release_then_wait();
    const int64_t total = (int64_t)num_seqs * q_heads;
    const int64_t flat = ((int64_t)blockIdx.x * kStagedWarps + warp) * RPW + sub;
    const bool live = flat < total;
    int j = 0, h = 0, s0 = 0, ns = 0, kv_heads = q_heads / r, g = 0, rr = 0;
    if (live) {
        j = (int)(flat / q_heads);
        h = (int)(flat - (int64_t)j * q_heads);
        g = h / r;
        rr = h - g * r;
        s0 = split_off[j];
        ns = split_off[j + 1] - s0;
    }
    // bytes of the warp's rows (lane 0 of each row group reports its row's count)
    uint32_t bytes = (live && d4 == 0) ? (uint32_t)ns * D * 4 : 0u;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, off);
    if (lane == 0) dev::mbar_arrive_expect_tx(&bar[warp], bytes);
    __syncwarp();
    if (live && d4 < ns) {  // lane d4 < ns: split d4's bulk copy and lse (ns <= kNarrowSplits <= TPH)
        const size_t rw = ((size_t)(s0 + d4) * kv_heads + g) * r + rr;
        dev::bulk_g2s(rowbuf + (size_t)d4 * D, part_o + rw * D, D * 4, &bar[warp], dev::policy_evict_first());
        lsebuf[d4] = part_lse[rw];
    }
    dev::mbar_wait(&bar[warp], 0);
    __syncwarp();
    if (!live) return;
    float4 acc;
    float lse2;
    if (ns == 0) {  // a device holding none of request j's tokens (sequence split): o = 0, lse = -inf
        acc = make_float4(0.f, 0.f, 0.f, 0.f);
        lse2 = -INFINITY;
    } else {
        acc = finish(fold_splits_with(0, 1, ns,
                                      [&](int sp, float &l, float4 &v) {
                                          l = lsebuf[sp];
                                          v = *reinterpret_cast<const float4 *>(rowbuf + (size_t)sp * D + 4 * d4);
                                      }),
                     &lse2);
    }
    const size_t orow = units != nullptr ? (size_t)units[2 * j] * o_seq_stride + ((size_t)units[2 * j + 1] * r + h) * D
                                         : (size_t)j * o_seq_stride + (size_t)h * D;
    store_row4<OUT_BF16>(o, orow + 4 * d4, acc);
    if (lse != nullptr && d4 == 0) lse[flat] = lse2 * 0.69314718055994531f;  // log2 -> natural log
}

cudaError_t launch_combine(int num_seqs, int q_heads, int r, int head_dim, const int32_t *seq_lens,
                           const int32_t *split_off, const float *part_lse, const float *part_o, void *o,
                           int o_dtype, int64_t o_seq_stride, cudaStream_t s, float *lse, int max_seq_len,
                           const int32_t *units) {
    const int64_t pairs = (int64_t)num_seqs * q_heads;
    if (pairs == 0) return cudaSuccess;
    const int ns_max = (max_seq_len + kSplitTokens - 1) / kSplitTokens;
    const bool wide = ns_max > kNarrowSplits;
#if HETIS_COMBINE_STAGED
    // shared-memory staged fold when the register-staged kernel would need more than one wave (~7 of its
    // 4-row blocks fit an SM at 72 registers per thread): c3 at N = 1, 8192 rows, -1 us per step; for
    // one-wave launches the bulk-copy round trip is the slower one (c3's 8-GPU share: +1.7 us)
    if (!wide && pairs > (int64_t)7 * 4 * num_sms()) {
        const int rpw = 32 / (head_dim / 4);
        const size_t smem = 128 + (size_t)kStagedWarps * rpw * ns_max * (head_dim + 4) * sizeof(float);
        const int64_t warps = (pairs + rpw - 1) / rpw;
        const int64_t blocks = (warps + kStagedWarps - 1) / kStagedWarps;
        const bool bf = o_dtype == HETIS_BF16;
        decltype(&combine_staged_kernel<128, 0>) kern =
            head_dim == 128 ? (bf ? combine_staged_kernel<128, 1> : combine_staged_kernel<128, 0>)
                            : (bf ? combine_staged_kernel<64, 1> : combine_staged_kernel<64, 0>);
        return launch_pdl(kern, dim3((unsigned)blocks), dim3(32 * kStagedWarps), smem, s, num_seqs, q_heads, r,
                          ns_max, split_off, part_lse, part_o, o, o_seq_stride, lse, units);
    }
#endif
    const int g = kCombineThreads / (head_dim / 4);
    const int64_t blocks = wide ? pairs : (pairs + g - 1) / g;
    const bool bf = o_dtype == HETIS_BF16;
    decltype(&combine_kernel<128, 0, false>) kern;
    if (head_dim == 128)
        kern = wide ? (bf ? combine_kernel<128, 1, true> : combine_kernel<128, 0, true>)
                    : (bf ? combine_kernel<128, 1, false> : combine_kernel<128, 0, false>);
    else
        kern = wide ? (bf ? combine_kernel<64, 1, true> : combine_kernel<64, 0, true>)
                    : (bf ? combine_kernel<64, 1, false> : combine_kernel<64, 0, false>);
    return launch_pdl(kern, dim3((unsigned)blocks), dim3(kCombineThreads), 0, s, num_seqs, q_heads, r, seq_lens,
                      split_off, part_lse, part_o, o, o_seq_stride, lse, units);
}

cudaError_t launch_combine_peers(int num_seqs, int q_heads, int r, int head_dim, const int32_t *split_off,
                                 const float *part_lse, const float *part_o, int o_dtype, const PeerGroupDev &g,
                                 cudaStream_t s, int max_seq_len) {
    const int64_t pairs = (int64_t)num_seqs * q_heads;
    const bool wide = (max_seq_len + kSplitTokens - 1) / kSplitTokens > kNarrowSplits;
    const int gsz = kCombineThreads / (head_dim / 4);
    int64_t blocks = wide ? pairs : (pairs + gsz - 1) / gsz;  // every row in flight at once (one fold each)
    if (blocks < 1) blocks = 1;
    const bool bf = o_dtype == HETIS_BF16;
    decltype(&combine_peers_kernel<128, 0, false>) kern;
    if (head_dim == 128)
        kern = wide ? (bf ? combine_peers_kernel<128, 1, true> : combine_peers_kernel<128, 0, true>)
                    : (bf ? combine_peers_kernel<128, 1, false> : combine_peers_kernel<128, 0, false>);
    else
        kern = wide ? (bf ? combine_peers_kernel<64, 1, true> : combine_peers_kernel<64, 0, true>)
                    : (bf ? combine_peers_kernel<64, 1, false> : combine_peers_kernel<64, 0, false>);
    return launch_pdl(kern, dim3((unsigned)blocks), dim3(kCombineThreads), 0, s, num_seqs, q_heads, r, split_off,
                      part_lse, part_o, g);
}

cudaError_t launch_peer_wait(const PeerGroupDev &g, cudaStream_t s) {
    return launch_pdl(peer_wait_kernel, dim3(1), dim3(32), 0, s, g);
}

cudaError_t launch_check_tables(int num_seqs, int kv_heads, int page_size, int64_t num_pages,
                                const int32_t *block_table, int max_pages, const int32_t *seq_lens,
                                int32_t *violations, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(violations, 0, sizeof(int32_t), s);
    if (e != cudaSuccess) return e;
    const int64_t total = (int64_t)num_seqs * kv_heads * max_pages;
    if (total == 0) return cudaSuccess;
    const int threads = 256;
    int64_t blocks = (total + threads - 1) / threads;
    if (blocks > 4 * num_sms()) blocks = 4 * num_sms();
    check_tables_kernel<<<(unsigned)blocks, threads, 0, s>>>(num_seqs, kv_heads, page_size, num_pages, block_table,
                                                             max_pages, seq_lens, violations);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_scatter_pull(const PeerGroupDev &g, int num_seqs, int H, int Hkv, int q0, int nq, int k0, int nk,
                                int qrow, int kvrow, void *q_dst, void *k_dst, void *v_dst, cudaStream_t s) {
    const int64_t total = (int64_t)num_seqs * (nq * (qrow / 16) + 2 * nk * (kvrow / 16));
    const int threads = 256;
    int64_t blocks = (total + threads - 1) / threads;
    if (blocks > 2 * num_sms()) blocks = 2 * num_sms();
    if (blocks < 1) blocks = 1;  // nothing to copy still publishes the signal and the acknowledgement
    return launch_pdl(scatter_pull_kernel, dim3((unsigned)blocks), dim3(threads), 0, s, g, num_seqs, H, Hkv, q0,
                      nq, k0, nk, qrow, kvrow, static_cast<uint8_t *>(q_dst), static_cast<uint8_t *>(k_dst),
                      static_cast<uint8_t *>(v_dst));
}

}  // namespace hetis

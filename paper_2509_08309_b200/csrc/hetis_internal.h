// hetis_internal.h -- host-side declarations shared by the library's .cu/.cpp
// files (never installed, never seen by the oracle).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "hetis.h"

namespace hetis {

// split-KV chunk C in tokens (reading 12): fixed, a multiple of the page size.
constexpr int kSplitTokens = 256;
constexpr int kPageSize = 16;

// Everything a decode-attention launch needs, validated by the API layer.
struct AttnArgs {
    int num_seqs;
    int q_heads;       // local query heads x
    int kv_heads;      // local kv heads x / r
    int r;
    int head_dim;
    int dtype;         // hetis_dtype of q / kv
    const void *q;
    const void *k_pool;
    const void *v_pool;
    int64_t num_pages;
    const int32_t *block_table;
    int max_pages;
    const int32_t *seq_lens;
    int max_seq_len;
    // workspace carve-up
    int32_t *split_off;   // [num_seqs + 1]
    float *part_lse;      // [max_items][r]
    float *part_o;        // [max_items][r][head_dim]
    int64_t max_items;
    uint32_t flags;       // HETIS_ATTN_*
    int32_t *counters;    // [2] work-claim and CTA-finish counters; zero between launches
    const void *k_new;    // fused append: new rows [num_seqs][kv_heads][head_dim], or nullptr
    const void *v_new;
    // per-request plans (hetis_attn_decode_units): launch row j = unit (units[2j], units[2j+1]) =
    // (request, GLOBAL kv head), kv_heads == 1, q / k_new / block-table rows in the full
    // [requests][row_kv_heads] layout.  nullptr: launch row j = request j.
    const int32_t *units;
    int row_kv_heads;
    // merge fused into the per-warp kernel: O rows of every (request, kv head) pair written by the
    // pair's last split (nullptr: partials only, hetis_attn_combine merges)
    void *o_out;
    int64_t o_seq_stride;
    int o_dtype;
    int32_t *pair_cnt;    // [num_seqs * kv_heads], zero between launches (self-cleaning)
    // fused merge + gather over peer memory: the rows go to every target rank's o_full (nullptr: o_out)
    const struct PeerGroupDev *peer;
    // pull mode: q / k_new / v_new are the Primary's buffers (offset to this rank's heads), in_kv_stride
    // kv rows per request; the kernel does the scatter's synchronisation (nullptr: ordinary launch)
    const struct PeerGroupDev *pull;
    int in_kv_stride;     // 0 = kv_heads (dense shards)
};

struct WorkspaceLayout {
    size_t split_off_offset, lse_offset, o_offset, counter_offset, pair_cnt_offset, total;
    int64_t max_items;
};

WorkspaceLayout workspace_layout(int num_seqs, int kv_heads, int r, int head_dim, int max_seq_len);

// launchers (return cudaError_t of the launch)
cudaError_t launch_attn_simt(const AttnArgs &a, cudaStream_t s);
cudaError_t launch_attn_tc(const AttnArgs &a, cudaStream_t s, std::string *err);
// Group mode of the merge-fused per-warp kernel (attn_decode.cu, Params::group_mode): launches with
// at most one (request, kv head) pair per SM and at most HETIS_TC_NW splits per pair, not pipelined,
// not device-claimed, not HETIS_ATTN_NO_GROUP_MODE.  The decode calls fuse the merge for such launches
// even without HETIS_ATTN_FUSED_MERGE (measured faster: c3 8-GPU share 27.9 vs 29.0 us per step).
bool group_mode_qualifies(int64_t pairs, int max_seq_len, uint32_t flags);
cudaError_t launch_combine(int num_seqs, int q_heads, int r, int head_dim, const int32_t *seq_lens,
                           const int32_t *split_off, const float *part_lse, const float *part_o, void *o,
                           int o_dtype, int64_t o_seq_stride, cudaStream_t s, float *lse, int max_seq_len,
                           const int32_t *units = nullptr);
cudaError_t launch_kv_append(int num_seqs, int kv_heads, int head_dim, int page_size, int elem_bytes,
                             const void *k_new, const void *v_new, void *k_pool, void *v_pool,
                             const int32_t *block_table, int max_pages, const int32_t *seq_lens, cudaStream_t s);
// Up to kMaxCopySegs strided head copies in ONE launch (the scatter's pack on the
// root and the gather's placement: one kernel instead of one per rank and tensor).
// Segment k copies, for every request j, heads [hs, hs + n) of src rows
// [num_seqs][src_heads] to heads [hd, hd + n) of dst rows [num_seqs][dst_heads].
constexpr int kMaxCopySegs = 48;
struct CopySeg {
    const uint8_t *src;
    uint8_t *dst;
    int src_heads, hs, dst_heads, hd, n, row_bytes;
};
struct CopySegs {
    CopySeg seg[kMaxCopySegs];
    int64_t start[kMaxCopySegs + 1];  // prefix of 16-byte chunks per segment
    int count;
    int num_seqs;
};
cudaError_t launch_head_copies(CopySegs &c, cudaStream_t s);

// ---------------------------------------------------------------- exchanges over peer memory
// Device-resident exchange state of one rank (hetis_peer_state_bytes; the
// caller zero-fills it once).  int64 slots; every epoch lives in device memory,
// so a step's kernels take no per-step host argument and a captured CUDA graph
// replays any number of steps.  Epoch of the step in flight = state[kStStep] + 1
// (read after stream ordering); hetis_peer_wait, the step's last kernel, stores it.
constexpr int kMaxPeers = 8;
constexpr int kStStep = 0;     // steps this rank has completed (written only by its own peer_wait)
constexpr int kStDone = 8;     // reserved (was combine_peers' block counter; peer_wait publishes now)
constexpr int kStIn = 16;      // the root's latest published input epoch
constexpr int kStOut = 32;     // [kMaxPeers] epoch of rank p's rows now in this rank's o_full
constexpr int kStAck = 48;     // [kMaxPeers] rank p has consumed its o_full through this epoch
constexpr int kStSlots = 64;   // 512 bytes
struct PeerGroupDev {
    int64_t *state[kMaxPeers];  // every rank's state as mapped in this process ([rank] = own)
    void *o[kMaxPeers];         // every rank's o_full [num_seqs][H][d] (o_dtype), mapped here
    const uint8_t *q_root, *k_root, *v_root;  // the root's q_full / k_new_full / v_new_full, mapped here
    int n, rank, root;
    int gather_root;            // -1: every rank receives O (all-gather); >= 0: only that rank
    int head0;                  // this rank's first global query head
    int64_t o_seq_stride;       // elements between requests in o_full (>= H * d)
};
// O rows of this rank's heads go to rank p iff gather_root < 0 or p == gather_root
__host__ __device__ inline bool peer_is_target(const PeerGroupDev &g, int p) {
    return g.gather_root < 0 || p == g.gather_root;
}
cudaError_t launch_combine_peers(int num_seqs, int q_heads, int r, int head_dim, const int32_t *split_off,
                                 const float *part_lse, const float *part_o, int o_dtype, const PeerGroupDev &g,
                                 cudaStream_t s, int max_seq_len);
cudaError_t launch_scatter_pull(const PeerGroupDev &g, int num_seqs, int H, int Hkv, int q0, int nq, int k0, int nk,
                                int qrow, int kvrow, void *q_dst, void *k_dst, void *v_dst, cudaStream_t s);
cudaError_t launch_peer_wait(const PeerGroupDev &g, cudaStream_t s);
// sequence-wise split (row f3, seq_split.cu)
cudaError_t launch_seq_split_lens(int num_ranks, int rank, int page_size, int num_seqs, const int32_t *seq_lens,
                                  int32_t *local_lens, int32_t *append_lens, cudaStream_t s);
cudaError_t launch_seq_merge(int num_parts, int num_seqs, int q_heads, int head_dim, const float *o_parts,
                             int64_t o_part_stride, const float *lse_parts, int64_t lse_part_stride, void *o,
                             int o_dtype, int64_t o_seq_stride, cudaStream_t s);
cudaError_t launch_check_tables(int num_seqs, int kv_heads, int page_size, int64_t num_pages,
                                const int32_t *block_table, int max_pages, const int32_t *seq_lens,
                                int32_t *violations, cudaStream_t s);
cudaError_t launch_kv_migrate(int num_entries, const hetis_migration_entry *entries, int page_size, int page_bytes,
                              const void *src_k, const void *src_v, const int32_t *src_bt, int src_max_pages,
                              void *dst_k, void *dst_v, const int32_t *dst_bt, int dst_max_pages, int max_ctas,
                              cudaStream_t s);

void note_launch();
int num_sms();

// Launch with programmatic dependent launch (PDL): the kernel may be scheduled
// while the previous kernel in the stream is still running; every kernel of
// this library executes griddepcontrol.wait before its first global-memory
// access (so stream order is preserved) and then griddepcontrol.launch_dependents,
// which hides launch latency and CTA scheduling between the step's kernels.
// Every kernel of the library prefers the maximum shared-memory carveout: the
// persistent attention kernel needs ~217 KB per SM, and a small kernel (append,
// combine, migration on a side stream) that lands first on an SM with a smaller
// carveout would keep the attention CTA off that SM until it drains.
void prefer_max_smem_once(const void *kern);  // small_kernels.cu: once per kernel (and device)

template <typename... KArgs>
void prefer_max_smem(void (*kern)(KArgs...)) {
    prefer_max_smem_once(reinterpret_cast<const void *>(kern));
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args &&...args) {
    prefer_max_smem(kern);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
    note_launch();
    return e;
}

}  // namespace hetis

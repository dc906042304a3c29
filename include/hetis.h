/*
 * hetis.h -- C ABI of libhetis.so: the B200 (sm_100a) hot path of Hetis
 * (arXiv 2509.08309), head-granular distributed decode Attention over a
 * head-granular paged KV cache.
 *
 * Citations: "PAPER.md:N" = /root/reference/PAPER.md line N (section /
 * equation given alongside); "reading N" = DESIGN.md §3 (the readings taken
 * where the paper is silent or ambiguous).
 *
 * One decode step of one layer on device i:
 *   hetis_plan_*      head -> device assignment x_i (Eq. 5)
 *   hetis_scatter_q   primary -> attention workers: q of the device's heads and
 *                     the new token's k, v (Eq. 4 traffic)
 *   hetis_kv_append   head-granular store of the new K/V rows
 *   hetis_attn_decode result_{i,j} = softmax(q K^T / sqrt(d)) V for the device's
 *                     heads (Eq. 2b) = hetis_attn_partial (split-KV
 *                     partial attention) + hetis_attn_combine (LSE merge)
 *   hetis_gather      Attention_j = Concat_i result_{i,j} (Eq. 2a)
 * Over peer memory (NVLink, no NCCL; the bench default at N > 1):
 *   hetis_attn_partial_pull -> hetis_attn_combine_peers -> hetis_peer_wait
 *                     (the scatter folded into the attention kernel, the gather
 *                     into the combine; hetis_scatter_pull is the standalone pull)
 * Per-request plans (Eq. 7, x_i^j varying with j): hetis_attn_decode_units.
 *
 * Conventions
 * -----------
 * - Every call returns hetis_status; nothing throws, aborts or prints.  On a
 *   validation error nothing is launched.  hetis_last_error() gives a
 *   thread-local one-line detail of the last failure.
 * - The caller owns every device buffer, stream and NCCL communicator.  The
 *   library owns only plans (freed by hetis_plan_destroy); it never allocates
 *   device memory (TMA descriptors are built per call on the host and passed
 *   as kernel parameters).
 *   Workspace is sized by the *_workspace queries.
 * - All device work is asynchronous and ordered on the given stream
 *   (cudaStream_t; NULL = legacy default stream).
 * - "Local" indexing: on a device holding query heads [b, b + x) the q / o
 *   shards are [num_seqs][x][head_dim] with local head h - b, and the block
 *   table is [num_seqs][x / r][max_pages] with local kv head g - b / r.
 *   Global head ids appear only in plans, scatter and gather.
 * - Device-data contracts (not checked per call, as in vLLM): every page id a
 *   kernel reads is in [0, num_pages); 0 <= seq_lens[j] <= min(max_seq_len,
 *   max_pages * page_size).  Table entries past ceil(L_j / page_size) and
 *   pool slots past L_j are never read into a result (they may hold NaN).
 *   L_j = 0 is meaningful only on a device that holds none of request j's
 *   tokens under a sequence split (row f3): kv_append skips the request, the
 *   combine writes o = 0 (and lse = -inf).  Softmax over no token is
 *   undefined (reading 10), so a whole-request result needs L_j >= 1.
 * - Stream ordering: kernels are launched with programmatic dependent launch
 *   (PDL).  Each waits (griddepcontrol.wait) for its predecessor before it
 *   touches anything a predecessor writes, so results follow stream order.
 *   Callers may rely on: the attention kernels read seq_lens and block tables
 *   before that wait (none of this library's kernels that let their successor
 *   start early writes those -- hetis_seq_split_lens and hetis_kv_migrate
 *   never do) and q only after it (hetis_scatter_pull, which writes q shards,
 *   releases its successor before its copy completes); with
 *   HETIS_ATTN_PIPELINED they read q and the cache pages other than each
 *   request's last two positions early, so a pipelined step's q must not come
 *   from hetis_scatter_pull.  Work the
 *   caller enqueues itself (copies, torch kernels) is ordinary stream order.
 * - Builds: head_dim in {64, 128}; page_size 16; kv/q dtype in {bf16, f32}
 *   with q_dtype == kv_dtype; o_dtype in {f32, bf16}; r = H / H_kv in
 *   {1, 2, 4, 8}.  Anything else -> HETIS_E_UNSUPPORTED.  bf16 with r > 1
 *   runs on tensor cores (mma.sync m16n8k16); everything else on CUDA cores.
 */
#ifndef HETIS_H_
#define HETIS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 4: hetis_attn_decode_launches_for; hetis_attn_decode(_append) / _units fuse the merge automatically in
 * group mode; hetis_attn_decode_peers' pull form (q_shard NULL); flags NO_GROUP_MODE, STATIC_DEAL. */
#define HETIS_ABI_VERSION 4

#if defined(__GNUC__)
#define HETIS_API __attribute__((visibility("default")))
#else
#define HETIS_API
#endif

typedef struct CUstream_st *hetis_stream_t; /* == cudaStream_t */

typedef enum {
    HETIS_OK = 0,
    HETIS_E_INVALID = 1,        /* null / misaligned pointer, bad size or shape              */
    HETIS_E_HEAD_INTEGRITY = 2, /* Eq. 5: sum_i x_i^j != H                    */
    HETIS_E_GROUP_ALIGN = 3,    /* x_i^j / r not integral, or a head range    */
                                /* that does not start/end on a kv-group boundary            */
    HETIS_E_CAPACITY = 4,       /* Eq. 6 in pages: sum_j ceil(L_j/P) x_i^j/r  */
                                /*  > free_pages_i (reading 13)                              */
    HETIS_E_UNSUPPORTED = 5,    /* dtype / head_dim / page_size / r / batch not built        */
    HETIS_E_WORKSPACE = 6,      /* workspace too small or misaligned                         */
    HETIS_E_CUDA = 7,           /* a CUDA runtime call or launch failed                      */
    HETIS_E_NCCL = 8            /* NCCL missing or an NCCL call failed                       */
} hetis_status;

typedef enum { HETIS_F32 = 0, HETIS_BF16 = 1 } hetis_dtype;

/* Model-side attention shape (D9).  H = num_q_heads (the "H" of Eq. 5),
 * r = num_q_heads / num_kv_heads, head_dim = the d of Eq. 2b
 * (reading 1), page_size = tokens per head-granular block. */
typedef struct {
    int32_t num_q_heads;
    int32_t num_kv_heads;
    int32_t head_dim;
    int32_t page_size;
    int32_t kv_dtype; /* hetis_dtype of K/V pools and of new K/V rows */
    int32_t q_dtype;  /* hetis_dtype of q; must equal kv_dtype        */
    int32_t o_dtype;  /* hetis_dtype of o: HETIS_F32 or HETIS_BF16    */
} hetis_shape;

/* Flags for hetis_attn_partial(_append) / hetis_attn_decode(_append).  None of
 * them changes a result bit: an item's arithmetic depends on L_j only. */
#define HETIS_ATTN_FORCE_SIMT 0x1u /* bf16 GQA on CUDA cores instead of tensor cores */
/* The shared page ring with a per-item CTA merge instead of the per-warp
 * kernel (whose default gives every consumer warp whole items and its own
 * sub-ring): for bf16 GQA on tensor cores, and for bf16 MHA on CUDA cores
 * (bf16 MHA defaults to the per-warp kernel with a CUDA-core consumer; its
 * pipelined launches always run the shared-ring kernel, so they are
 * bit-identical to serial launches WITH this flag, and within tolerance of
 * the default). */
#define HETIS_ATTN_TC_SHARED_RING 0x2u
/* Per-warp kernel (bf16 GQA; bf16 MHA on its CUDA-core consumer): claim work
 * items device-wide (the first round
 * dealt round-robin, every later claim from a device-wide counter).  The
 * DEFAULT of that kernel for every launch that is neither pipelined nor in
 * group mode (with the consumer refill it measured faster: c3 attention
 * 171 -> 163 us); it also keeps decode fast beside another kernel (e.g.
 * hetis_kv_migrate on a low-priority stream, the Hauler: slowed SMs take
 * fewer items).  Passing the flag forces it and turns group mode off.
 * Ignored with HETIS_ATTN_PIPELINED. */
#define HETIS_ATTN_DEVICE_CLAIM 0x4u
/* The CTA-local deal instead of the default device-wide claiming (95% of the
 * items dealt to CTAs round-robin, the rest stolen at the end; the default
 * before round 2's consumer refill).  For A/B measurements. */
#define HETIS_ATTN_STATIC_DEAL 0x80u
/* bf16 MHA (r = 1) with the per-warp kernel's tensor-core consumer (one valid
 * MMA row) instead of its CUDA-core consumer (the default; c2 attention 751 vs
 * 746 us: no gain -- decode MHA is HBM-bound, not a dense contraction). */
#define HETIS_ATTN_MHA_TC 0x8u
/* Pipelined steps: the caller passes two workspaces alternately to consecutive
 * steps on the stream (at most one kv_append -- fused or not -- per step).
 * The attention kernel then streams cache pages while the previous step's
 * combine and attention tail still run: it waits for them only before a page
 * holding one of the last two positions of a request, and before it ends.
 * Measured before round 2's consumer refill: it paid when a device had about
 * one work item per warp (c3 8-GPU share -12%).  With the final kernels the
 * plain launches are faster everywhere (c3: 170.7 vs 195.8 us at N = 1, the
 * 8-GPU share 26.6 us in group mode vs 30.1 pipelined), because pipelined
 * launches keep the producer-issued pages and the CTA-local deal; kept as an
 * option.  No work stealing in this mode.
 * Safety rests on at most ONE attention CTA per SM (step t + 1 reaches an SM
 * only after step t's CTA there, which waits for combine t - 1, has left):
 * pipelined launches reserve > 114 KiB of shared memory per CTA and the
 * launcher checks the occupancy (HETIS_E_CUDA if it is not exactly 1). */
#define HETIS_ATTN_PIPELINED 0x10u
/* hetis_attn_decode / _decode_append / _decode_units / _decode_peers with the
 * per-warp tensor-core kernel: fold each (request, kv head) pair's splits in
 * the attention kernel itself (the warp that finishes the pair's last split;
 * the combine's arithmetic, bit-identical) -- ONE launch per step, and over
 * peer memory the merged rows go straight into every rank's o_full.  Measured
 * SLOWER than the separate combine on B200 (c3: 200 vs 188 us at N = 1, 33.1
 * vs 30.7 us for the 8-GPU share; without the fold 182 / 27.7 us -- the fold's
 * L2 round trips under a saturated memory system stall the merging warp), so
 * opt-in -- except for launches in group mode (below), where the
 * merge runs in shared memory, is faster, and is the default. */
#define HETIS_ATTN_FUSED_MERGE 0x20u
/* Merge-fused launches (above) run in GROUP MODE when they have at most one
 * (request, kv head) pair per SM and at most 8 splits per pair (max_seq_len <=
 * 2048), e.g. the LLaMA-70B GQA share of one of 8 GPUs: CTA c runs pair c,
 * consumer warp w its split w, the warps stage their partials in shared memory
 * and fold them there after one CTA barrier (the combine's arithmetic, same
 * order: bit-identical).  This flag turns group mode off (the last-arriver
 * merge through L2 instead). */
#define HETIS_ATTN_NO_GROUP_MODE 0x40u
/* Diagnostic only: stream every K/V page through the shared-memory ring but
 * skip the math (partials are left unwritten).  Measures the memory-system
 * ceiling of the pipeline; every kernel honours it. */
#define HETIS_ATTN_DIAG_STREAM_ONLY 0x100u

/* ---- status ------------------------------------------------------------ */
HETIS_API const char *hetis_status_str(hetis_status s);
HETIS_API const char *hetis_last_error(void);
HETIS_API int32_t hetis_abi_version(void);
/* Tokens per split-KV chunk C (reading 12): a constant, so the chunking of a
 * sequence depends on its length only -- partition invariance is bit-exact. */
HETIS_API int32_t hetis_split_tokens(void);

/* ---- plan: head -> device assignment (Eq. 5) --------- */
typedef struct hetis_plan hetis_plan; /* opaque, immutable after create */

/* x (host): per_request == 0: [num_devices] counts shared by every request;
 *           per_request != 0: [num_seqs][num_devices] counts x_i^j.
 * Validates x >= 0, x mod r == 0 (-> HETIS_E_GROUP_ALIGN) and sum_i x = H for
 * every request (-> HETIS_E_HEAD_INTEGRITY; Eq. 7c uses "= H", reading 14).
 * Device i gets the contiguous global head range [b_i, b_i + x_i), b_i =
 * sum_{i' < i} x_i' (reading 3).  On success *out owns a new plan. */
HETIS_API hetis_status hetis_plan_create(const hetis_shape *shape, int32_t num_devices, int32_t num_seqs,
                               const int32_t *x, int32_t per_request, hetis_plan **out);
HETIS_API void hetis_plan_destroy(hetis_plan *plan);
/* Head range of request `seq` (ignored for global plans) on `device`. */
HETIS_API hetis_status hetis_plan_heads(const hetis_plan *plan, int32_t device, int32_t seq, int32_t *q_begin,
                              int32_t *q_count);
HETIS_API int32_t hetis_plan_num_devices(const hetis_plan *plan);
/* Work units of `device`: one unit = one (request j, kv head g) pair the device
 * owns, i.e. r query heads of one request.  A per-request plan (x_i^j varying
 * with j, the dispatcher's output, Eq. 7) is executed by the unchanged kernels
 * by treating each unit as a request with ONE kv head: q, o as [U][r][head_dim],
 * block table [U][1][max_pages], seq_lens[u] = L_j of the unit's request, and
 * the shape's head range = (0, r).  The chunking of a unit depends on L_j only,
 * so results are bit-identical to the uniform-plan path.
 *   units: host int32 [2 * U] receiving (request, GLOBAL kv head) pairs in the
 *          device's order (requests ascending, kv heads ascending), or NULL to
 *          query the count; *num_units: in = capacity in units (ignored when
 *          units is NULL), out = U.  Too small a capacity -> HETIS_E_INVALID. */
HETIS_API hetis_status hetis_plan_units(const hetis_plan *plan, int32_t device, int32_t *units, int32_t *num_units);
/* Eq. 6 in pages (reading 13): for every device i,
 *   sum_j ceil(seq_lens[j] / P) * x_i^j / r <= free_pages[i].
 * seq_lens_host: [num_seqs] lengths the requests will have (num_seqs must equal
 * the plan's for per-request plans); free_pages: [N]. */
HETIS_API hetis_status hetis_plan_check_capacity(const hetis_plan *plan, int32_t num_seqs,
                                                 const int32_t *seq_lens_host, const int64_t *free_pages);

/* ---- kv append: head-granular store --------------------- */
/* For every request j and local kv head g: the new row goes to page
 * block_table[j][g][(L_j - 1) / P], slot (L_j - 1) mod P, L_j = seq_lens[j]
 * (length AFTER the append, reading 6).  A bit-exact copy.  L_j = 0: nothing
 * is stored for request j (a device that does not own the request's newest
 * page under a sequence split, see hetis_seq_split_lens).
 *   k_new, v_new : device [num_seqs][kv_head_count][head_dim], kv_dtype
 *   k_pool, v_pool: device [num_pages][page_size][head_dim], 16-B aligned
 *   block_table  : device int32 [num_seqs][kv_head_count][max_pages]
 *   seq_lens     : device int32 [num_seqs]
 * The caller must have placed a valid page at (L_j - 1) / P beforehand (a new
 * page is needed exactly when (L_j - 1) mod P == 0). */
HETIS_API hetis_status hetis_kv_append(const hetis_shape *shape, int32_t num_seqs, int32_t kv_head_count,
                             const void *k_new, const void *v_new, void *k_pool, void *v_pool, int64_t num_pages,
                             const int32_t *block_table, int32_t max_pages, const int32_t *seq_lens,
                             hetis_stream_t stream);

/* ---- debug validation of the device-data contracts -------------------- */
/* Counts, into *violations (device int32, overwritten), the contract
 * violations the decode kernels trust not to happen: seq_lens[j] outside
 * [1, max_pages * P] (reading 10: an empty request has no softmax), and page
 * ids of pages 0 .. ceil(L_j / P) - 1 of every (request, local kv head)
 * outside [0, num_pages).  Stream-ordered; read *violations after it.  For
 * debugging only -- it reads the whole block table. */
HETIS_API hetis_status hetis_check_tables(const hetis_shape *shape, int32_t num_seqs, int32_t kv_head_count,
                                          int64_t num_pages, const int32_t *block_table, int32_t max_pages,
                                          const int32_t *seq_lens, int32_t *violations, hetis_stream_t stream);

/* ---- decode attention (Eq. 2b) --------------------------- */
/* Workspace bytes for num_seqs requests of length <= max_seq_len and
 * q_head_count local heads (partials of every split + the split offsets). */
HETIS_API hetis_status hetis_attn_decode_workspace(const hetis_shape *shape, int32_t num_seqs, int32_t q_head_count,
                                         int32_t max_seq_len, size_t *bytes);

/* Kernel 1 (a4): split-KV partial attention.  For every (request j, local kv
 * head g, split s covering tokens [s C, min((s+1) C, L_j))) and each of the r
 * query heads of g: o_s = softmax-weighted mean of V over the split and its
 * log2-sum-exp, written to the workspace.  Arguments:
 *   q_head_begin, q_head_count: this device's global head range (multiples
 *       of r; only validated -- indexing is local)
 *   q          : device [num_seqs][q_head_count][head_dim], q_dtype
 *   k_pool, v_pool, num_pages, block_table, max_pages, seq_lens: as in
 *       hetis_kv_append with kv_head_count = q_head_count / r
 *   max_seq_len: upper bound of seq_lens (workspace sizing)
 *   workspace  : device, >= hetis_attn_decode_workspace bytes, 256-B aligned,
 *                ZERO-filled before its first use (it ends in two work-claim
 *                counters that every completed launch returns to zero)
 *   flags      : HETIS_ATTN_* */
HETIS_API hetis_status hetis_attn_partial(const hetis_shape *shape, int32_t num_seqs, int32_t q_head_begin,
                                int32_t q_head_count, const void *q, const void *k_pool, const void *v_pool,
                                int64_t num_pages, const int32_t *block_table, int32_t max_pages,
                                const int32_t *seq_lens, int32_t max_seq_len, void *workspace,
                                size_t workspace_bytes, uint32_t flags, hetis_stream_t stream);

/* hetis_kv_append fused into hetis_attn_partial: ONE kernel whose warp that
 * owns request j's newest page takes the new K/V row of each local kv head
 * from k_new / v_new (device [num_seqs][q_head_count / r][head_dim]) straight
 * into its shared-memory copy of the page -- the new token never round-trips
 * through HBM before it is used -- and stores it into the pool slot
 * (page block_table[j][g][(L_j - 1) / P], slot (L_j - 1) mod P) for later
 * steps.  Results and pools are bit-identical to hetis_kv_append followed by
 * hetis_attn_partial (same arguments otherwise); seq_lens must be >= 1. */
HETIS_API hetis_status hetis_attn_partial_append(const hetis_shape *shape, int32_t num_seqs, int32_t q_head_begin,
                                                 int32_t q_head_count, const void *q, const void *k_new,
                                                 const void *v_new, void *k_pool, void *v_pool, int64_t num_pages,
                                                 const int32_t *block_table, int32_t max_pages,
                                                 const int32_t *seq_lens, int32_t max_seq_len, void *workspace,
                                                 size_t workspace_bytes, uint32_t flags, hetis_stream_t stream);

/* Kernel 2 (a5): o = sum_s 2^(lse_s - lse) o_s in ascending s (fixed order).
 *   o : device [num_seqs][q_head_count][head_dim] (o_dtype), rows of request j
 *       start at o + j * o_seq_stride elements (o_seq_stride >= q_head_count *
 *       head_dim; pass q_head_count * head_dim for a dense shard). */
HETIS_API hetis_status hetis_attn_combine(const hetis_shape *shape, int32_t num_seqs, int32_t q_head_count,
                                const int32_t *seq_lens, int32_t max_seq_len, void *o, int64_t o_seq_stride,
                                const void *workspace, size_t workspace_bytes, hetis_stream_t stream);

/* hetis_attn_combine that also returns, per head, the natural-log normaliser
 * over the tokens this device holds (the "global softmax attribute" a sequence
 * split must aggregate):
 *   lse[j][h] = ln sum_{t < L_j} exp(q_{j,h} . k_t / sqrt(d))
 * (-inf and o = 0 when L_j = 0).  lse: device float [num_seqs][q_head_count]. */
HETIS_API hetis_status hetis_attn_combine_lse(const hetis_shape *shape, int32_t num_seqs, int32_t q_head_count,
                                              const int32_t *seq_lens, int32_t max_seq_len, void *o,
                                              int64_t o_seq_stride, float *lse, const void *workspace,
                                              size_t workspace_bytes, hetis_stream_t stream);

/* The whole per-device step (a3 + a4 + a5) with a dense o shard: results
 * bit-identical to hetis_attn_partial_append followed by hetis_attn_combine.
 * With HETIS_ATTN_FUSED_MERGE and the per-warp tensor-core kernel (bf16 and
 * r > 1, or HETIS_ATTN_MHA_TC; not with HETIS_ATTN_FORCE_SIMT /
 * _TC_SHARED_RING / _PIPELINED / _DIAG_STREAM_ONLY) it is ONE kernel: the warp
 * that finishes the last split of a (request, kv head) pair folds the pair's
 * splits (the combine's arithmetic, same order) and stores its r rows; a
 * one-split pair stores its rows straight from registers.  Launches that
 * qualify for group mode (see hetis_attn_decode_launches_for) are one kernel
 * without the flag.  Otherwise two kernels.  o must be 16-byte aligned for
 * the one-kernel form (8-byte for the two-kernel form). */
HETIS_API hetis_status hetis_attn_decode_append(const hetis_shape *shape, int32_t num_seqs, int32_t q_head_begin,
                                                int32_t q_head_count, const void *q, const void *k_new,
                                                const void *v_new, void *k_pool, void *v_pool, int64_t num_pages,
                                                const int32_t *block_table, int32_t max_pages,
                                                const int32_t *seq_lens, int32_t max_seq_len, void *o,
                                                void *workspace, size_t workspace_bytes, uint32_t flags,
                                                hetis_stream_t stream);

/* hetis_attn_partial followed by hetis_attn_combine with a dense o shard (one
 * kernel under the same conditions as hetis_attn_decode_append). */
HETIS_API hetis_status hetis_attn_decode(const hetis_shape *shape, int32_t num_seqs, int32_t q_head_begin,
                               int32_t q_head_count, const void *q, const void *k_pool, const void *v_pool,
                               int64_t num_pages, const int32_t *block_table, int32_t max_pages,
                               const int32_t *seq_lens, int32_t max_seq_len, void *o, void *workspace,
                               size_t workspace_bytes, uint32_t flags, hetis_stream_t stream);

/* Kernels hetis_attn_decode / _decode_append / _decode_units launch for this
 * shape and these flags: 1 (merge fused into the attention kernel) or 2
 * (attention + combine); -1 for an invalid shape.  Launches in group mode
 * (HETIS_ATTN_NO_GROUP_MODE above) are always 1: use
 * hetis_attn_decode_launches_for for the count of one concrete launch. */
HETIS_API int32_t hetis_attn_decode_launches(const hetis_shape *shape, uint32_t flags);

/* Kernels one hetis_attn_decode / _decode_append launch of num_seqs requests,
 * q_head_count local query heads and seq_lens <= max_seq_len runs, for a
 * 16-byte aligned o (for _decode_units pass num_seqs = num_units and
 * q_head_count = r): 1 when the merge is fused -- HETIS_ATTN_FUSED_MERGE, or
 * automatically in group mode (<= one (request, kv head) pair per SM and
 * max_seq_len <= 2048 on the per-warp tensor-core kernel, where one kernel is
 * measured faster: the LLaMA-70B GQA 8-GPU share 27.9 vs 29.0 us per step) --
 * else 2; -1 for invalid arguments. */
HETIS_API int32_t hetis_attn_decode_launches_for(const hetis_shape *shape, int32_t num_seqs, int32_t q_head_count,
                                                 int32_t max_seq_len, uint32_t flags);

/* A per-request plan (f2: x_i^j varying with request j, the Eq. 7 dispatcher's
 * output) executed by ONE attention launch and ONE
 * combine on the original layouts -- no caller-side gathers of q or o.  The
 * device's work is its unit list (hetis_plan_units: unit = one (request j,
 * GLOBAL kv head g) it owns = the r query heads g r .. g r + r - 1 of j), held
 * in device memory; each unit is chunked by L_j exactly as in the uniform path,
 * so every result is bit-identical to hetis_attn_decode(_append) of the same
 * heads.  Arguments:
 *   num_seqs   : requests B (rows of q, o, block_table, seq_lens)
 *   num_units, units: device int32 [num_units][2] (j, g), 0 <= j < num_seqs,
 *                0 <= g < H_kv, no pair twice (a device-data contract); any order
 *   q          : device [num_seqs][H][head_dim] (q_dtype), ALL heads' rows
 *                (only the units' heads are read)
 *   k_new, v_new: device [num_seqs][H_kv][head_dim] new rows, or both NULL.
 *                Given: the append is fused (hetis_attn_partial_append) for the
 *                units' (j, g); NULL: the pools already hold the new tokens
 *   block_table: device int32 [num_seqs][H_kv][max_pages], global kv index
 *                (rows of kv heads the device does not own are never read)
 *   o          : device [num_seqs][H][head_dim] (o_dtype), rows of request j
 *                at o + j * o_seq_stride elements; only the units' heads are
 *                written, at their GLOBAL head index
 *   workspace  : >= hetis_attn_decode_workspace(shape, num_units, r,
 *                max_seq_len) bytes, 256-B aligned, zero-filled before first use
 *   flags      : HETIS_ATTN_* except HETIS_ATTN_PIPELINED (-> UNSUPPORTED)
 * One kernel when hetis_attn_decode_launches says 1 and o rows are 16-byte
 * aligned; else two.  num_units == 0 launches nothing. */
HETIS_API hetis_status hetis_attn_decode_units(const hetis_shape *shape, int32_t num_seqs, int32_t num_units,
                                               const int32_t *units, const void *q, const void *k_new,
                                               const void *v_new, void *k_pool, void *v_pool, int64_t num_pages,
                                               const int32_t *block_table, int32_t max_pages,
                                               const int32_t *seq_lens, int32_t max_seq_len, void *o,
                                               int64_t o_seq_stride, void *workspace, size_t workspace_bytes,
                                               uint32_t flags, hetis_stream_t stream);

/* ---- the step's exchanges over peer memory (NVLink 5 / NVSwitch) -------- */
/* The scatter (a2) and the gather (a6, Eq. 2a Concat) without
 * NCCL: every rank pulls its shard of the step's inputs straight from the
 * Primary's buffers, and the combine kernel stores every merged O row straight
 * into every receiving rank's o_full.  One step on every rank is
 *     hetis_scatter_pull -> hetis_attn_partial(_append) -> hetis_attn_combine_peers
 *     -> hetis_peer_wait
 * (the Primary writes q_full, k_new_full, v_new_full before its scatter_pull).
 * Synchronisation lives in device memory: each rank owns a STATE of
 * hetis_peer_state_bytes() (zero-filled once by the caller, 64-byte aligned)
 * holding its step counter and the epochs its peers publish (system-scope
 * release stores, acquire loads).  No call takes a per-step host argument, so
 * a step -- or many -- can be captured once in a CUDA graph and replayed.
 * Every rank must run the same sequence of steps.  Reuse rules enforced on the
 * device: a rank's O rows go into a peer's o_full only after that peer's
 * scatter_pull of the same step acknowledged (everything it enqueued before,
 * i.e. the consumer of the previous step's o_full, has completed); the
 * Primary's scatter_pull of step e + 1 follows its peer_wait of step e, so the
 * Primary may overwrite its input buffers after hetis_peer_wait returns on its
 * stream (every rank has pulled by then).  Bounded waits: a peer that never
 * publishes makes the waiting kernel trap after ~10 s (HETIS_E_CUDA on the
 * stream) instead of hanging the device. */
HETIS_API size_t hetis_peer_state_bytes(void);
/* Let kernels on the CURRENT device dereference memory of peer_device (NVLink
 * peer access; needed for the peer pointers of a group whose ranks sit on
 * other GPUs of the box).  OK when already enabled or peer_device is the
 * current device; HETIS_E_UNSUPPORTED when the devices cannot access each
 * other.  Host-side, once per pair. */
HETIS_API hetis_status hetis_peer_access(int32_t peer_device);
typedef struct hetis_peer_group hetis_peer_group; /* opaque, immutable after create */
/* plan         : global plan (per_request == 0) of num_devices <= 8 ranks
 * rank, root   : this rank; the Primary holding the step's inputs
 * gather_root  : -1 = every rank receives O (all-gather, north star); >= 0 =
 *                only that rank does (gather to the Primary)
 * state_peers  : host array [N] of device pointers, rank p's state as mapped
 *                in THIS process ([rank] = own; peers via cudaIpcOpenMemHandle
 *                or any other peer mapping)
 * o_full_peers : host array [N], rank p's o_full [num_seqs][H][head_dim]
 *                (o_dtype) mapped here; rows o_seq_stride elements apart,
 *                16-byte aligned.  Entries of non-receiving ranks may be NULL.
 * q_full_root, k_new_full_root, v_new_full_root : the Primary's [num_seqs][H][d]
 *                and [num_seqs][H_kv][d] input buffers mapped here
 * The group copies the pointers; the caller keeps the memory alive. */
HETIS_API hetis_status hetis_peer_group_create(const hetis_plan *plan, int32_t rank, int32_t root,
                                               int32_t gather_root, int64_t *const *state_peers,
                                               void *const *o_full_peers, int64_t o_seq_stride,
                                               const void *q_full_root, const void *k_new_full_root,
                                               const void *v_new_full_root, hetis_peer_group **out);
HETIS_API void hetis_peer_group_destroy(hetis_peer_group *group);
/* a2: on the Primary, first publish this step's epoch (its inputs are written);
 * on every rank, acknowledge the previous step's o_full, wait (acquire) for
 * the Primary's epoch, then copy this rank's plan range straight from the
 * Primary's buffers:
 *   q_full_root [num_seqs][H][d] heads [b, b + x)       -> q_shard [num_seqs][x][d]
 *   k/v_new_full_root [num_seqs][H_kv][d] [b/r, (b+x)/r) -> k/v_new_shard [num_seqs][x/r][d]
 * One kernel; the same bytes as hetis_scatter_q. */
HETIS_API hetis_status hetis_scatter_pull(const hetis_peer_group *group, int32_t num_seqs, void *q_shard,
                                          void *k_new_shard, void *v_new_shard, hetis_stream_t stream);
/* a5 + a6 in ONE kernel: the split combine of this rank's heads (same
 * arithmetic as hetis_attn_combine) storing every row o[j][h] at its GLOBAL
 * head index into every receiving rank's o_full (after that rank acknowledged
 * the previous step).  workspace: this step's hetis_attn_partial workspace. */
HETIS_API hetis_status hetis_attn_combine_peers(const hetis_peer_group *group, int32_t num_seqs,
                                                const int32_t *seq_lens, int32_t max_seq_len, void *workspace,
                                                size_t workspace_bytes, hetis_stream_t stream);
/* a2 + a3 + a4 in ONE kernel (the scatter folded into the attention): the
 * split-KV partial attention of this rank's heads with the append fused, whose
 * producers copy each work item's q rows, and whose consumers take the new
 * token's k, v rows, straight from the Primary's q_full / k_new_full /
 * v_new_full (peer memory: NVLink loads, pipelined with the K/V pages) -- no
 * shard copy.  Its first steps after griddepcontrol.wait are hetis_scatter_pull's
 * synchronisation: CTA 0 publishes this rank's acknowledgement of the previous
 * o_full (and, on the Primary, the input epoch), every CTA waits (bounded) for
 * the Primary's epoch.  Pools, block table, seq_lens and workspace as in
 * hetis_attn_partial_append for this rank's heads.  One step per rank is then
 *     hetis_attn_partial_pull -> hetis_attn_combine_peers -> hetis_peer_wait.
 * Results bit-identical to hetis_scatter_pull + hetis_attn_partial_append.
 * A rank without heads, or num_seqs == 0 -> HETIS_E_UNSUPPORTED (use
 * hetis_scatter_pull, which takes part in the protocol without a shard);
 * HETIS_ATTN_PIPELINED / _DIAG_STREAM_ONLY / _FUSED_MERGE -> UNSUPPORTED. */
HETIS_API hetis_status hetis_attn_partial_pull(const hetis_peer_group *group, int32_t num_seqs, void *k_pool,
                                               void *v_pool, int64_t num_pages, const int32_t *block_table,
                                               int32_t max_pages, const int32_t *seq_lens, int32_t max_seq_len,
                                               void *workspace, size_t workspace_bytes, uint32_t flags,
                                               hetis_stream_t stream);

/* a3 + a4 + a5 + a6 in ONE kernel: this rank's attention over its shard
 * (hetis_attn_partial_append when k/v_new_shard are given, else
 * hetis_attn_partial; q_shard [num_seqs][x][d], block table / pools / seq_lens
 * as there) whose merge of each (request, kv head) pair's splits (the
 * combine's arithmetic) stores the pair's rows straight into every receiving
 * rank's o_full at the GLOBAL head index, after that rank acknowledged the
 * previous step -- the work of hetis_attn_partial(_append) +
 * hetis_attn_combine_peers, bit-identical, one launch.  One step per rank is
 * then
 *     hetis_scatter_pull -> hetis_attn_decode_peers -> hetis_peer_wait.
 * It belongs to a step: before its first O store it waits (bounded, traps after
 * ~10 s) for every receiving rank's acknowledgement published by that rank's
 * hetis_scatter_pull of the same step, so it cannot be replayed alone.
 * Only where hetis_attn_decode_launches(shape, flags | HETIS_ATTN_FUSED_MERGE)
 * == 1 (the per-warp tensor-core kernel; the flag is implied) and the rank
 * holds >= 1 head and >= 1 request; else HETIS_E_UNSUPPORTED (use the
 * two-kernel path).  o_full rows 16-B aligned.
 * q_shard == NULL (then k_new_shard and v_new_shard NULL too): PULL form -- the
 * kernel reads q and the new k, v rows from the Primary's buffers as
 * hetis_attn_partial_pull does (its acknowledgement / epoch protocol, the
 * append fused), so one step per rank is TWO kernels
 *     hetis_attn_decode_peers(q_shard = NULL) -> hetis_peer_wait;
 * the group needs the Primary's mappings.  Launches that qualify for group mode
 * (hetis_attn_decode_launches_for) merge in shared memory (the default N > 1
 * step for such shares, e.g. LLaMA-70B GQA on 8 GPUs). */
HETIS_API hetis_status hetis_attn_decode_peers(const hetis_peer_group *group, int32_t num_seqs, const void *q_shard,
                                               const void *k_new_shard, const void *v_new_shard, void *k_pool,
                                               void *v_pool, int64_t num_pages, const int32_t *block_table,
                                               int32_t max_pages, const int32_t *seq_lens, int32_t max_seq_len,
                                               void *workspace, size_t workspace_bytes, uint32_t flags,
                                               hetis_stream_t stream);
/* The step's last kernel: every rank publishes (one system-scope fence, then
 * release stores) that the rows the previous kernel stored are in every
 * receiving rank's o_full; a receiving rank then waits until every rank has
 * published; every rank records the step as completed.  Work enqueued after it
 * on the stream may read o_full. */
HETIS_API hetis_status hetis_peer_wait(const hetis_peer_group *group, hetis_stream_t stream);

/* ---- scatter / gather over NCCL ------------------- */
/* nccl_comm is an ncclComm_t (e.g. torch ProcessGroupNCCL._comm_ptr()) whose
 * ranks are the plan's devices.  libnccl.so.2 is resolved at first use from
 * the process (dlopen by soname); absent -> HETIS_E_NCCL.  Only global plans
 * (per_request == 0) are supported here -> else HETIS_E_UNSUPPORTED.
 *
 * Staging bytes needed on `rank` by scatter and gather with this plan. */
HETIS_API hetis_status hetis_comm_workspace(const hetis_plan *plan, int32_t rank, int32_t num_seqs, size_t *bytes);

/* Root holds q_full [num_seqs][H][d] and k_new_full, v_new_full
 * [num_seqs][H_kv][d] (q/kv dtypes); every rank receives its shards
 * q_shard [num_seqs][x_rank][d] and k/v_new_shard [num_seqs][x_rank/r][d].
 * Non-root ranks may pass NULL for the *_full pointers. */
HETIS_API hetis_status hetis_scatter_q(const hetis_plan *plan, void *nccl_comm, int32_t rank, int32_t root,
                             int32_t num_seqs, const void *q_full, const void *k_new_full,
                             const void *v_new_full, void *q_shard, void *k_new_shard, void *v_new_shard,
                             void *workspace, size_t workspace_bytes, hetis_stream_t stream);

/* o_shard [num_seqs][x_rank][d] (o_dtype) from every rank -> o_full
 * [num_seqs][H][d] with each head at its GLOBAL index (reading 4).
 * root == -1: every rank receives o_full (all-gather, north star);
 * root >= 0: only root does (gather to the Primary worker). */
HETIS_API hetis_status hetis_gather(const hetis_plan *plan, void *nccl_comm, int32_t rank, int32_t root, int32_t num_seqs,
                          const void *o_shard, void *o_full, void *workspace, size_t workspace_bytes,
                          hetis_stream_t stream);

/* ---- sequence-wise split across devices (row f3) ------------------------ */
/* The alternative the paper argues against (PAPER.md:292-304 `fig:head_wise_
 * advantage`, :356-358): every device attends ALL heads over a subset of each
 * request's tokens; the partial results are merged with their log-sum-exp
 * ("aggregate global softmax attributes").  Layout (reading f3):
 * page k of every (request, kv head) lives on device k mod N ("page striping"):
 * the device's block table lists its pages k = rank, rank + N, ... in order, so
 * only its last page can be partial, and the newest token always lands on the
 * device holding page ceil(L_j / P) - 1.  Nothing moves as a request grows.
 *
 * From global lengths L_j (after the append), this device's token count
 *   local_lens[j]  = sum over its pages of the tokens they hold
 * and the length to pass to hetis_kv_append (append_lens may be NULL)
 *   append_lens[j] = local_lens[j] if it owns page ceil(L_j / P) - 1, else 0.
 * seq_lens, local_lens, append_lens: device int32 [num_seqs].  Integer; exact. */
HETIS_API hetis_status hetis_seq_split_lens(int32_t num_ranks, int32_t rank, int32_t page_size, int32_t num_seqs,
                                            const int32_t *seq_lens, int32_t *local_lens, int32_t *append_lens,
                                            hetis_stream_t stream);
/* O[j][h] = sum_p e^(lse_p - lse) o_p[j][h], lse = ln sum_p e^(lse_p), over the
 * num_parts devices' partial results in ascending p (the union-of-subsets
 * identity; a part with lse = -inf holds no token and is skipped).  One part
 * reproduces its o bit for bit.
 *   o_parts   : device float, part p at o_parts + p * o_part_stride, layout
 *               [num_seqs][q_head_count][head_dim]; 16-byte aligned
 *   lse_parts : device float, part p at lse_parts + p * lse_part_stride,
 *               [num_seqs][q_head_count] (natural log, hetis_attn_combine_lse)
 *   o         : device [num_seqs][q_head_count][head_dim] (o_dtype), rows of
 *               request j at o + j * o_seq_stride elements */
HETIS_API hetis_status hetis_seq_merge(const hetis_shape *shape, int32_t num_parts, int32_t num_seqs,
                                       int32_t q_head_count, const float *o_parts, int64_t o_part_stride,
                                       const float *lse_parts, int64_t lse_part_stride, void *o,
                                       int64_t o_seq_stride, hetis_stream_t stream);
/* The sequence split's input exchange: every device needs q of ALL heads (and
 * the new k, v rows, which only the owner of the newest page stores): NCCL
 * broadcast of q [num_seqs][H][d] and k_new, v_new [num_seqs][H_kv][d] from
 * root, in place.  nccl_comm: ncclComm_t of num_ranks ranks, this one `rank`. */
HETIS_API hetis_status hetis_seq_broadcast_q(const hetis_shape *shape, void *nccl_comm, int32_t num_ranks,
                                             int32_t rank, int32_t root, int32_t num_seqs, void *q, void *k_new,
                                             void *v_new, hetis_stream_t stream);
/* The sequence split's output exchange: all-gather every device's record
 *   part = [ o [num_seqs][H][d] float | lse [num_seqs][H] float ]
 * (hetis_attn_combine_lse with q_head_count = H) into staging [num_ranks][record]
 * (NCCL, num_seqs * H must be a multiple of 4), then hetis_seq_merge -> o
 * [num_seqs][H][d] (o_dtype) on every rank. */
HETIS_API hetis_status hetis_seq_allgather_merge(const hetis_shape *shape, void *nccl_comm, int32_t num_ranks,
                                                 int32_t rank, int32_t num_seqs, const float *part, float *staging,
                                                 void *o, int64_t o_seq_stride, hetis_stream_t stream);

/* ---- head-granular KV migration (the Hauler) ------- */
/* Re-dispatching a request moves only the kv-head groups whose device changes
 * ("only partial cache transmission"): each moved (request, kv
 * head) is a block-table ROW on the source and one on the destination, and its
 * cache is the ceil(num_tokens / P) pages those rows list.  For every entry e
 * and page k < ceil(entries[e].num_tokens / P):
 *   dst_pool[dst_block_table[dst_row][k]] <- src_pool[src_block_table[src_row][k]]
 * for both the K and the V pool -- a bit-exact copy of whole pages (the slots
 * past num_tokens in the last page receive the source page's bytes).
 *   entries        : device [num_entries] hetis_migration_entry; src_row indexes
 *                    the rows of src_block_table ([rows][src_max_pages]), dst_row
 *                    those of dst_block_table ([rows][dst_max_pages])
 *   src_*_pool     : [pages][page_size][head_dim] kv_dtype, 16-B aligned, readable
 *                    by the executing device (local, or a peer mapping: pull)
 *   dst_*_pool     : same layout, writable by the executing device (local, or a
 *                    peer mapping over NVLink: push)
 *   the tables and entries must be readable by the executing device; the
 *   destination pages are allocated by the caller (as for kv_append) and must
 *   not overlap any source page of the same call.
 *   max_ctas       : CTAs the copy may occupy (0 = 2 per SM).  The Hauler runs
 *                    this on a low-priority stream while decode runs (PAPER.md:
 *                    545); max_ctas bounds its share of the SMs.
 * num_entries <= 16384 (else HETIS_E_INVALID); 0 launches nothing.  Row and
 * page ids are contracts on device data (not checked). */
typedef struct {
    int32_t src_row;     /* row of src_block_table */
    int32_t dst_row;     /* row of dst_block_table */
    int32_t num_tokens;  /* cached tokens of this (request, kv head): L_j */
} hetis_migration_entry;
HETIS_API hetis_status hetis_kv_migrate(const hetis_shape *shape, int32_t num_entries,
                                        const hetis_migration_entry *entries, const void *src_k_pool,
                                        const void *src_v_pool, const int32_t *src_block_table,
                                        int32_t src_max_pages, void *dst_k_pool, void *dst_v_pool,
                                        const int32_t *dst_block_table, int32_t dst_max_pages, int32_t max_ctas,
                                        hetis_stream_t stream);

/* Number of kernels this library has launched in the calling process (all
 * threads) -- for the bench's gpu_launches accounting. */
HETIS_API uint64_t hetis_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* HETIS_H_ */
